"""GPU parity of the 2-D Tsallis path
against the CPU oracle, through the C ABI (-m gpu).

Bar (as the 1-D path): mean image, 2-D histogram, status
and labels bit-exact; (t, s) bit-exact unless the oracle's distinct-partition
gap is < 1e-12, in which case the GPU pair must be a near-tie member under the
oracle; objective within 1e-12 relative."""
import numpy as np
import pytest
import torch

import oracle
import phantom
import paper_2012_10684_b200 as tsa

pytestmark = pytest.mark.gpu
REL = 1e-12
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def c2_slab(nz, z_first):
    return phantom.make_volume(phantom.CONFIGS["c2"], nz=nz, z_first=z_first)


def check_pair(h, q, t, s, phi, ref, where):
    if ref["status"] != oracle.OK:
        assert (t, s) == (-1, -1) and np.isnan(phi), where
        return
    if (t, s) != (ref["t"], ref["s"]):
        assert ref["gap"] < REL, (where, (t, s), ref)
        v = oracle.phi2d_at(h, q, t, s)
        assert v is not None and v >= ref["phi"] - REL * abs(ref["phi"]), (where, v, ref)
        assert abs(phi - v) <= REL * abs(v), (where, phi, v)
    else:
        assert abs(phi - ref["phi"]) <= REL * abs(ref["phi"]) + (REL if ref["phi"] == 0 else 0), \
            (where, phi, ref["phi"])


def run_and_check(vol, bins, q, slices=None, cluster=0, threads=None):
    out = tsa.tsa2d_segment(to_dev(vol), bins, q, histogram=True, cluster=cluster)
    torch.cuda.synchronize()
    hist = out["histogram"].cpu().numpy().astype(np.uint32)
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    st = out["status"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    zs = range(vol.shape[0]) if slices is None else slices
    for z in zs:
        h_ref, st_ref = oracle.hist2d(vol[z], bins)
        np.testing.assert_array_equal(hist[z], h_ref, err_msg=f"hist2d z={z}")
        if st_ref != oracle.OK:
            assert st[z] == st_ref and tuple(thr[z]) == (-1, -1) and (lab[z] == 0).all()
            continue
        ref = oracle.search2d(h_ref, q, threads=threads or oracle.max_threads())
        assert st[z] == ref["status"], (z, st[z], ref)
        check_pair(h_ref, q, int(thr[z][0]), int(thr[z][1]), float(phi[z]), ref, f"z={z} q={q}")
        if ref["status"] == oracle.OK:
            np.testing.assert_array_equal(lab[z], oracle.label(vol[z], 1, (int(thr[z][0]),)),
                                          err_msg=f"labels z={z}")
        else:
            assert (lab[z] == 0).all()
    return out


# --------------------------------------------------------------- mean image
@pytest.mark.parametrize("shape", [(512, 512), (7, 11), (4, 4), (1, 8), (9, 1), (33, 36)])
def test_mean3x3_bitexact(shape):
    rng = np.random.default_rng(sum(shape))
    vol = rng.integers(0, 256, size=(2,) + shape).astype(np.uint8)
    if shape == (512, 512):
        vol = c2_slab(2, 120)
    g = tsa.tsa2d_mean3x3(to_dev(vol)).cpu().numpy()
    for z in range(vol.shape[0]):
        np.testing.assert_array_equal(g[z], oracle.mean3x3(vol[z]), err_msg=f"{shape} z={z}")


# ----------------------------------------------------------- 2-D histogram
@pytest.mark.parametrize("cluster", [0, 4, 5, 6, 7, 8])
def test_hist2d_bitexact_phantom(cluster):
    vol = c2_slab(6, 100)
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 256, cluster=cluster)
    torch.cuda.synchronize()
    h = hist.cpu().numpy().astype(np.uint32)
    for z in range(vol.shape[0]):
        ref, st_ref = oracle.hist2d(vol[z], 256)
        assert st[z].item() == st_ref
        np.testing.assert_array_equal(h[z], ref, err_msg=f"cluster={cluster} z={z}")


def test_hist2d_full_bench_volume():
    """Every slice of the bench volume (c2, 512x512x300) in the bench launch configuration."""
    vol = phantom.make_volume(phantom.CONFIGS["c2"])
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 256)
    torch.cuda.synchronize()
    h = hist.cpu().numpy().astype(np.uint32)
    assert (st.cpu().numpy() == 0).all()
    for z in range(vol.shape[0]):
        ref, _ = oracle.hist2d(vol[z], 256)
        np.testing.assert_array_equal(h[z], ref, err_msg=f"z={z}")


@pytest.mark.parametrize("shape", [(1024, 1024), (700, 333), (3, 5), (1, 1), (2000, 64)])
def test_hist2d_shapes_and_rounds(shape):
    """Odd widths (scalar path), tall slices (several counting rounds per CTA),
    slices smaller than the cluster."""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    vol = rng.integers(0, 256, size=(2,) + shape).astype(np.uint8)
    vol[1, : shape[0] // 2] = 17  # a large uniform region: warp-uniform shortcut
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 256)
    torch.cuda.synchronize()
    h = hist.cpu().numpy().astype(np.uint32)
    for z in range(2):
        ref, _ = oracle.hist2d(vol[z], 256)
        np.testing.assert_array_equal(h[z], ref, err_msg=f"{shape} z={z}")


def test_hist2d_constant_slice_counts_past_16_bits():
    """A constant 512x512 slice puts 262144 pixels in one cell: the 16-bit private
    counters never see more than 65535 per round, the merged band is u32."""
    vol = np.full((1, 512, 512), 200, np.uint8)
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 256)
    h = hist.cpu().numpy()
    assert h[0, 200, 200] == 512 * 512 and h.sum() == 512 * 512


def test_hist2d_level_overflow():
    rng = np.random.default_rng(5)
    vol = rng.integers(0, 32, size=(3, 64, 64)).astype(np.uint8)
    vol[1, 10, 10] = 40  # f >= L
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 32)
    st = st.cpu().numpy()
    h = hist.cpu().numpy().astype(np.uint32)
    for z in range(3):
        ref, st_ref = oracle.hist2d(vol[z], 32)
        assert st[z] == st_ref
        np.testing.assert_array_equal(h[z], ref)
    assert st[1] == oracle.LEVEL_OVERFLOW


# -------------------------------------------------------------- whole path
@pytest.mark.parametrize("L", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.3, 2.0])
def test_segment2d_random_small_levels(L, q):
    rng = np.random.default_rng(L * 100 + int(q * 10))
    vol = rng.integers(0, L, size=(3, 40, 48)).astype(np.uint8)
    vol[1] = (vol[1] // 2) * 2  # empty odd rows / columns: equivalent candidates
    vol[2, :20] = rng.integers(0, 3, size=(20, 48))
    run_and_check(vol, L, q)


@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.5])
def test_segment2d_phantom_reduced_levels(q):
    """Phantom slices quantised to 64 levels (oracle in well under a second)."""
    vol = (c2_slab(4, 80) >> 2).astype(np.uint8)
    run_and_check(vol, 64, q)


def test_segment2d_phantom_full_size_sampled():
    """The bench configuration (c2 volume, 256 levels, q = 0.8): histograms and
    labels of every slice bit-exact; the oracle's exhaustive search on sampled
    slices; phi(t*,s*) from the definition on every slice."""
    vol = phantom.make_volume(phantom.CONFIGS["c2"])
    run_and_check(vol, 256, 0.8, slices=[0, 120, 217, 299])
    out = tsa.tsa2d_segment(to_dev(vol), 256, 0.8)
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    for z in range(0, vol.shape[0], 7):
        h, _ = oracle.hist2d(vol[z], 256)
        v = oracle.phi2d_at(h, 0.8, int(thr[z][0]), int(thr[z][1]))
        assert abs(v - phi[z]) <= REL * abs(v), z
        np.testing.assert_array_equal(lab[z], oracle.label(vol[z], 1, (int(thr[z][0]),)))


@pytest.mark.parametrize("cluster", [4, 5, 6, 8])
def test_segment2d_cluster_sizes_agree(cluster):
    vol = c2_slab(3, 150)
    a = tsa.tsa2d_segment(to_dev(vol), 256, 0.8, cluster=cluster)
    b = tsa.tsa2d_segment(to_dev(vol), 256, 0.8)
    assert torch.equal(a["thresholds"], b["thresholds"])
    assert torch.equal(a["labels"], b["labels"])
    np.testing.assert_allclose(a["objective"].cpu().numpy(), b["objective"].cpu().numpy(),
                               rtol=1e-13)


def test_segment2d_degenerate():
    vol = np.zeros((4, 32, 32), np.uint8)
    vol[0] = 9                      # one cell: no (t,s) with two non-empty classes
    vol[1, :, :16] = 3              # two flat regions: cells (3,3),(9,9) + edge cells
    vol[1, :, 16:] = 9
    vol[2, ::2, ::2] = 15           # checkerboard-ish
    vol[3] = np.arange(32, dtype=np.uint8)[None, :] % 16
    run_and_check(vol, 16, 0.8)
    out = tsa.tsa2d_segment(to_dev(vol[:1]), 16, 0.8)
    assert out["status"].item() == oracle.NO_VALID_SPLIT
    assert (out["labels"] == 0).all()


def test_segment2d_level_overflow_slice():
    rng = np.random.default_rng(8)
    vol = rng.integers(0, 16, size=(2, 24, 24)).astype(np.uint8)
    vol[0, 3, 3] = 200
    run_and_check(vol, 16, 1.2)


def test_segment2d_graph_capture():
    vol = to_dev(c2_slab(8, 40))
    out = tsa.tsa2d_segment(vol, 256, 0.8)
    ws = tsa.tsa2d_workspace(tsa.make_problem2d(vol, 256, 0.8), DEV)
    outs = {k: torch.empty_like(v) if v is not None else None for k, v in out.items()}
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa2d_segment(vol, 256, 0.8, out=outs, workspace=ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    for k in ("thresholds", "objective", "status", "labels"):
        assert torch.equal(outs[k], out[k]), k


def test_segment2d_small_levels_any_cluster():
    """Small L fits any cluster size (4..8): identical results."""
    rng = np.random.default_rng(12)
    vol = to_dev(rng.integers(0, 32, size=(4, 64, 64)).astype(np.uint8))
    ref = tsa.tsa2d_segment(vol, 32, 0.7, cluster=8)
    for c in (4, 5, 6, 7):
        o = tsa.tsa2d_segment(vol, 32, 0.7, cluster=c)
        assert torch.equal(o["thresholds"], ref["thresholds"]), c
        np.testing.assert_allclose(o["objective"].cpu().numpy(), ref["objective"].cpu().numpy(),
                                   rtol=1e-13)


@pytest.mark.parametrize("bins", [64, 256])
def test_hist2d_65536_pixel_rounds(bins):
    """4-CTA clusters on 512x512 count exactly 65536 pixels per CTA in one
    round: a CTA whose whole band falls in one cell wraps its 16-bit counter
    (low half: the carry lands in the neighbour cell; high half: lost) and is
    repaired at the merge; near misses (one pixel off, out-of-range pixels)
    must not be taken for a wrap."""
    rng = np.random.default_rng(bins)
    vol = rng.integers(0, bins, size=(5, 512, 512)).astype(np.uint8)
    vol[0, :129] = 40                   # CTA 0 uniform, even cell (low half)
    vol[1, 127:257] = 41                # CTA 1 uniform (its 3x3 halo too), odd cell
    vol[2, :] = 7
    vol[2, 300, 5] = 9                  # CTA 2 one pixel off uniform, the rest uniform
    vol[3, :129] = 40
    vol[3, 0, 0] = 255                  # pixel (0, 0) out of range at 64 levels
    vol[4, 128:, :] = 63                # CTAs 1-3 uniform, one cell across bands
    hist, st = tsa.tsa2d_histogram(to_dev(vol), bins, cluster=4)
    torch.cuda.synchronize()
    h = hist.cpu().numpy().astype(np.uint32)
    for z in range(vol.shape[0]):
        ref, st_ref = oracle.hist2d(vol[z], bins)
        assert st[z].item() == st_ref, z
        np.testing.assert_array_equal(h[z], ref, err_msg=f"z={z}")
    run_and_check(vol[[0, 1, 4]], bins, 0.8, cluster=4)


@pytest.mark.parametrize("shape", [(256, 1024), (1024, 256), (128, 512)])
def test_hist2d_65536_pixel_rounds_other_shapes(shape):
    """Other shapes whose 4-CTA bands hold exactly 65536 pixels (ny x nx with
    ceil(ny/4) * nx = 65536), with uniform bands in even and odd cells; (128,
    512) is below the bound (no band reaches 65536)."""
    ny, nx = shape
    rng = np.random.default_rng(ny + nx)
    vol = rng.integers(0, 256, size=(2, ny, nx)).astype(np.uint8)
    q = (ny + 3) // 4
    vol[0, : q + 1] = 122
    vol[1, q - 1: 2 * q + 1] = 33
    hist, st = tsa.tsa2d_histogram(to_dev(vol), 256, cluster=4)
    torch.cuda.synchronize()
    h = hist.cpu().numpy().astype(np.uint32)
    for z in range(2):
        ref, st_ref = oracle.hist2d(vol[z], 256)
        assert st[z].item() == st_ref
        np.testing.assert_array_equal(h[z], ref, err_msg=f"{shape} z={z}")


def test_segment2d_multiround_full_search():
    """1024x1024 slices (several counting rounds per CTA, static bands) with the
    whole search checked against the oracle (64 levels keep it quick)."""
    vol = phantom.generate(1024, 1024, 2, "u8", seed=phantom.SEED_BASE + 9, z_first=100, z_total=300)
    vol = (vol >> 2).astype(np.uint8)
    run_and_check(vol, 64, 0.8)


@pytest.mark.parametrize("q", [0.1, 0.3, 3.0, 5.0])
def test_segment2d_extreme_q(q):
    rng = np.random.default_rng(int(q * 10))
    vol = rng.integers(0, 24, size=(3, 48, 64)).astype(np.uint8)
    vol[1, 10:30, 10:40] = 20
    run_and_check(vol, 24, q)


@pytest.mark.parametrize("L", [2, 3])
def test_segment2d_minimum_levels(L):
    rng = np.random.default_rng(L)
    vol = rng.integers(0, L, size=(4, 16, 32)).astype(np.uint8)
    vol[3] = 0
    run_and_check(vol, L, 0.8)
