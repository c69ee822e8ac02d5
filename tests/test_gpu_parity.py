"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (-m gpu).  Bar (BASELINE.json:north_star, DESIGN.md
"Parity"): histograms and labels bit-exact; thresholds bit-exact unless the
oracle's top-two distinct-partition gap is < 1e-12, in which case the GPU tuple
must be a near-tie member; objective within 1e-12 relative."""
import numpy as np
import pytest
import torch

import oracle
import phantom
import paper_2012_10684_b200 as tsa
from tests import _pins

pytestmark = pytest.mark.gpu
REL = 1e-12
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def check_slice(hist, k, q, obj, t_gpu, phi_gpu, ref, where=""):
    """Acceptance rule for one slice; ref is oracle.search()."""
    if ref["status"] != 0:
        assert tuple(t_gpu) == (-1,) * k and np.isnan(phi_gpu), where
        return
    ok, why = _pins.accept(hist, k, q, t_gpu, ref, objective=obj, rel=REL,
                           phi_fn=lambda h, t: oracle.phi_at(h, k, q, t, obj))
    assert ok, f"{where}: {why}"
    if tuple(t_gpu) == tuple(ref["t"]):
        assert abs(phi_gpu - ref["phi"]) <= REL * abs(ref["phi"]) + (REL if ref["phi"] == 0 else 0), \
            (where, phi_gpu, ref["phi"])
    else:
        v = oracle.phi_at(hist, k, q, t_gpu, obj)
        assert abs(phi_gpu - v) <= REL * abs(v), where


def run_and_check(vol, bins, k, q, obj=0, enumeration="canonical", units=0, slices=None):
    out = tsa.tsa_segment(to_dev(vol), bins, k, q, objective=obj, enumeration=enumeration,
                          units=units)
    torch.cuda.synchronize()
    hist = out["histogram"].cpu().numpy().astype(np.uint32)
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    st = out["status"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    zs = range(vol.shape[0]) if slices is None else slices
    for z in zs:
        h_ref, st_ref = oracle.histogram(vol[z], bins)
        np.testing.assert_array_equal(hist[z], h_ref, err_msg=f"hist z={z}")
        if st_ref != 0:
            assert st[z] == st_ref
            assert (lab[z] == 0).all()
            continue
        ref = oracle.search(h_ref, k, q, objective=obj)
        assert st[z] == ref["status"], (z, st[z], ref)
        check_slice(h_ref, k, q, obj, thr[z], phi[z], ref, where=f"z={z} k={k} q={q} obj={obj}")
        if ref["status"] == 0:
            np.testing.assert_array_equal(lab[z], oracle.label(vol[z], k, thr[z]), err_msg=f"labels z={z}")
        else:
            assert (lab[z] == 0).all()
    return out


# ------------------------------------------------------------- histogram
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_histogram_bitexact_full_config(name):
    cfg = phantom.CONFIGS[name]
    vol = phantom.make_volume(cfg)
    hist, st = tsa.tsa_histogram(to_dev(vol), cfg.bins)
    torch.cuda.synchronize()
    h = hist.cpu().numpy()
    for z in range(vol.shape[0]):
        np.testing.assert_array_equal(h[z], np.bincount(vol[z].ravel(), minlength=cfg.bins))
    assert (st.cpu().numpy() == 0).all()


def test_histogram_u16_overflow_and_ragged():
    rng = np.random.default_rng(7)
    vol = rng.integers(0, 4096, size=(5, 37, 53)).astype(np.uint16)  # odd sizes: unaligned slices
    vol[2, 5, 7] = 4096
    vol[4, 36, 52] = 65535
    hist, st = tsa.tsa_histogram(to_dev(vol), 4096)
    torch.cuda.synchronize()
    h, s = hist.cpu().numpy(), st.cpu().numpy()
    for z in range(5):
        hr, sr = oracle.histogram(vol[z], 4096)
        np.testing.assert_array_equal(h[z], hr)
        assert s[z] == sr
    assert list(s) == [0, 0, 2, 0, 2]


def test_histogram_u8_small_bins_overflow_and_runs():
    vol = np.zeros((3, 64, 64), np.uint8)
    vol[0] = 7  # one long run: fast path only
    vol[1, :, :32] = 3
    vol[1, :, 32:] = np.arange(32, dtype=np.uint8)[None, :]
    vol[2] = 200  # >= bins for bins=100
    hist, st = tsa.tsa_histogram(to_dev(vol), 100)
    torch.cuda.synchronize()
    for z in range(3):
        hr, sr = oracle.histogram(vol[z], 100)
        np.testing.assert_array_equal(hist.cpu().numpy()[z], hr)
        assert st.cpu().numpy()[z] == sr


# --------------------------------------------------------------- labels
@pytest.mark.parametrize("dtype,bins", [("u8", 256), ("u16", 4096)])
def test_labels_bitexact_given_thresholds(dtype, bins):
    rng = np.random.default_rng(3)
    npdt = np.uint8 if dtype == "u8" else np.uint16
    vol = rng.integers(0, bins, size=(6, 48, 80)).astype(npdt)
    for k in (1, 2, 3, 4):
        thr = np.sort(rng.choice(bins - 1, size=(6, k), replace=True), axis=1).astype(np.int32)
        status = np.zeros(6, np.int32)
        status[3] = 3
        lab = tsa.tsa_label(to_dev(vol), to_dev(thr), to_dev(status), bins=bins).cpu().numpy()
        for z in range(6):
            ref = np.zeros_like(lab[z]) if status[z] else oracle.label(vol[z], k, thr[z])
            np.testing.assert_array_equal(lab[z], ref)


# ----------------------------------------------------- search: small cases
def random_hist_volume(seed, nz, L, zero_frac, side=24):
    """Slices whose histograms are random small-L histograms with empty bins."""
    rng = np.random.default_rng(seed)
    vols = []
    for _ in range(nz):
        p = rng.random(L) * (rng.random(L) > zero_frac)
        if p.sum() == 0:
            p[rng.integers(L)] = 1
        p /= p.sum()
        vols.append(rng.choice(L, size=(side, side), p=p))
    return np.stack(vols).astype(np.uint8)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.3, 2.0])
@pytest.mark.parametrize("obj", [0, 1])
def test_search_tiny_random_histograms(k, q, obj):
    L = 14
    vol = random_hist_volume(17 * k + int(q * 10) + obj, 40, L, zero_frac=0.3)
    for enumeration in ("canonical", "full"):
        run_and_check(vol, L, k, q, obj, enumeration=enumeration)


def test_degenerate_slices():
    L = 256
    vol = np.zeros((6, 32, 32), np.uint8)
    vol[0] = 9                       # constant: NO_VALID_SPLIT
    vol[1, :16] = 40; vol[1, 16:] = 200  # two point masses: t = 40, phi = 0
    vol[2].flat[:4] = [10, 90, 91, 250]; vol[2].flat[4:] = 10  # exactly k+1 non-empty for k=3
    vol[3] = np.arange(32 * 32).reshape(32, 32) % 256   # uniform-ish
    vol[4, :, :] = 0; vol[4, 0, :3] = [1, 2, 3]
    vol[5] = (np.arange(32 * 32).reshape(32, 32) * 7) % 251
    for k in (1, 3):
        for q in (0.8, 1.0, 1.5):
            run_and_check(vol, L, k, q)


def test_k_equals_bins_minus_one():
    vol = random_hist_volume(5, 8, 5, zero_frac=0.0, side=16)
    run_and_check(vol, 5, 4, 0.7)
    run_and_check(vol, 5, 4, 0.7, enumeration="full")


# ------------------------------------------------ search: phantom slabs
@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.2, 1.5])
def test_phantom_slab_k123(k, q):
    cfg = phantom.CONFIGS["c2"]
    vol = phantom.make_volume(cfg, nz=6, z_first=60 + 30 * k)
    run_and_check(vol, 256, k, q)


def test_phantom_slab_k4():
    cfg = phantom.CONFIGS["c4"]
    vol = phantom.make_volume(cfg, nz=3, z_first=140)
    run_and_check(vol, 256, 4, 0.8)
    run_and_check(vol, 256, 4, 0.8, enumeration="full", slices=[0])


def test_sum_plus_product_slab():
    vol = phantom.make_volume(phantom.CONFIGS["c3"], nz=4, z_first=300)
    for k in (2, 3):
        for q in (0.7, 1.0, 1.3):
            run_and_check(vol, 256, k, q, obj=1)


# ---------------------------------------- invariances (exact, bit for bit)
def _search_all(vol, bins, k, q, units, enumeration="canonical", obj=0, split=None):
    v = to_dev(vol)
    hist, st = tsa.tsa_histogram(v, bins)
    n = vol.shape[1] * vol.shape[2]
    if split is None:
        ps, pk = tsa.tsa_search(hist, st, n, k, q, obj, enumeration, units=units)
    else:
        parts = []
        for (a, b) in split:
            parts.append(tsa.tsa_search(hist, st.clone(), n, k, q, obj, enumeration, units=units,
                                        unit_begin=a, unit_end=b))
        ps = torch.cat([p[0] for p in parts])
        pk = torch.cat([p[1] for p in parts])
    s, key = tsa.tsa_merge(ps, pk)
    torch.cuda.synchronize()
    return s.cpu().numpy(), key.cpu().numpy()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_partition_invariance(k):
    """Any unit count, unit split (= fake multi-rank) or enumeration mode gives
    bit-identical (score, key) per slice."""
    vol = phantom.make_volume(phantom.CONFIGS["c2"], nz=5, z_first=100)
    base = _search_all(vol, 256, k, 0.8, units=1)
    for units in (3, 16):
        s, key = _search_all(vol, 256, k, 0.8, units=units)
        np.testing.assert_array_equal(s, base[0])
        np.testing.assert_array_equal(key, base[1])
    s, key = _search_all(vol, 256, k, 0.8, units=16, split=[(0, 5), (5, 11), (11, 16)])
    np.testing.assert_array_equal(s, base[0])
    np.testing.assert_array_equal(key, base[1])
    s, key = _search_all(vol, 256, k, 0.8, units=4, enumeration="full")
    np.testing.assert_array_equal(s, base[0])
    np.testing.assert_array_equal(key, base[1])


# --------------------------------------- full-size configs, sampled slices
FULL_SAMPLES = {"c2": [0, 77, 150, 299], "c3": [0, 310, 599], "c4": [40, 200], "c5": [0, 500]}


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_full_config_sampled(name):
    """Whole config in the bench's launch configuration (default units);
    histograms and labels checked for every slice, the search on samples."""
    cfg = phantom.CONFIGS[name]
    vol = phantom.make_volume(cfg)
    out = tsa.tsa_segment(to_dev(vol), cfg.bins, cfg.k, cfg.qs[0])
    torch.cuda.synchronize()
    hist = out["histogram"].cpu().numpy()
    thr = out["thresholds"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    for z in range(vol.shape[0]):
        np.testing.assert_array_equal(hist[z], np.bincount(vol[z].ravel(), minlength=cfg.bins))
        lz = (vol[z][..., None] > thr[z][None, None, :]).sum(-1).astype(np.uint8)
        np.testing.assert_array_equal(lab[z], lz)
    for z in FULL_SAMPLES.get(name, [0]):
        ref = oracle.search(hist[z].astype(np.uint32), cfg.k, cfg.qs[0])
        check_slice(hist[z].astype(np.uint32), cfg.k, cfg.qs[0], 0, thr[z], phi[z], ref, f"{name} z={z}")


def test_c3_q_sweep_sampled():
    cfg = phantom.CONFIGS["c3"]
    vol = phantom.make_volume(cfg)
    v = to_dev(vol)
    for q in cfg.qs:
        out = tsa.tsa_segment(v, cfg.bins, cfg.k, q, labels=False)
        torch.cuda.synchronize()
        hist = out["histogram"].cpu().numpy().astype(np.uint32)
        thr = out["thresholds"].cpu().numpy()
        phi = out["objective"].cpu().numpy()
        for z in FULL_SAMPLES["c3"]:
            ref = oracle.search(hist[z], cfg.k, q)
            check_slice(hist[z], cfg.k, q, 0, thr[z], phi[z], ref, f"c3 q={q} z={z}")


def test_c5_sampled():
    cfg = phantom.CONFIGS["c5"]
    vol = phantom.make_volume(cfg)
    out = tsa.tsa_segment(to_dev(vol), cfg.bins, cfg.k, cfg.qs[0])
    torch.cuda.synchronize()
    hist = out["histogram"].cpu().numpy()
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    lab = out["labels"]
    for z in range(0, cfg.nz, 111):
        np.testing.assert_array_equal(hist[z], np.bincount(vol[z].ravel(), minlength=cfg.bins))
        np.testing.assert_array_equal(lab[z].cpu().numpy(), oracle.label(vol[z], cfg.k, thr[z]))
    assert int(hist.sum()) == vol.size
    for z in FULL_SAMPLES["c5"]:
        ref = oracle.search(hist[z].astype(np.uint32), cfg.k, cfg.qs[0])
        check_slice(hist[z].astype(np.uint32), cfg.k, cfg.qs[0], 0, thr[z], phi[z], ref, f"c5 z={z}")


def test_host_buffer_path_matches_device_path():
    cfg = phantom.CONFIGS["c2"]
    vol = phantom.make_volume(cfg, nz=40, z_first=50)
    dev = tsa.tsa_segment(to_dev(vol), 256, 2, 0.8)
    host = tsa.tsa_segment_host(torch.from_numpy(vol).pin_memory(), 256, 2, 0.8, slab=16)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host["thresholds"].numpy(), dev["thresholds"].cpu().numpy())
    np.testing.assert_array_equal(host["objective"].numpy(), dev["objective"].cpu().numpy())
    np.testing.assert_array_equal(host["labels"].numpy(), dev["labels"].cpu().numpy())


def test_cuda_graph_capture():
    """tsa_segment is capturable (no sync / alloc inside) and replays exactly."""
    cfg = phantom.CONFIGS["c2"]
    vol = to_dev(phantom.make_volume(cfg, nz=8, z_first=100))
    p = tsa.make_problem(vol, 256, 2, 0.8)
    ws = tsa.workspace_for(p, DEV)
    ref = tsa.tsa_segment(vol, 256, 2, 0.8, workspace=ws)
    out = {k: torch.empty_like(v) for k, v in ref.items()}
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa_segment(vol, 256, 2, 0.8, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    for key in ref:
        assert torch.equal(out[key], ref[key]), key


# ------------------------------------------- fused pipeline == staged kernels
@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.3])
def test_fused_pipeline_bitexact_vs_staged(k, q):
    """The persistent fused kernel (k <= 2) and the one-kernel-per-stage path
    produce bit-identical histograms, thresholds, objectives, status and labels."""
    cfg = phantom.CONFIGS["c2"]
    vol = to_dev(phantom.make_volume(cfg, nz=37, z_first=20))
    b = tsa.tsa_segment(vol, 256, k, q, pipeline="staged")
    for pipe in ("fused", "compact"):
        a = tsa.tsa_segment(vol, 256, k, q, pipeline=pipe, slab_slices=4, label_lag=3)
        torch.cuda.synchronize()
        for key in ("histogram", "thresholds", "status", "labels"):
            assert torch.equal(a[key], b[key]), (pipe, key)
        assert torch.equal(a["objective"].view(torch.int64), b["objective"].view(torch.int64)), pipe


def test_fused_pipeline_parity_and_errors():
    """Fused path vs oracle, including overflow and no-valid-split slices."""
    vol = phantom.make_volume(phantom.CONFIGS["c2"], nz=12, z_first=150).copy()
    vol[3] = 77                      # constant slice: NO_VALID_SPLIT
    vol[5, 10, 10] = 255             # fine for bins = 256
    out = tsa.tsa_segment(to_dev(vol), 256, 2, 0.8, pipeline="fused", slab_slices=5, label_lag=3)
    torch.cuda.synchronize()
    st = out["status"].cpu().numpy()
    assert st[3] == 3
    run_and_check(vol, 256, 2, 0.8)   # auto = fused for this shape
    # overflow (u16 data above bins) through the fused path
    v16 = (vol.astype(np.uint16) * 3)
    v16[7, 0, 0] = 1000
    for pipe in ("fused", "compact"):
        out = tsa.tsa_segment(to_dev(v16), 1000, 1, 0.8, pipeline=pipe)
        torch.cuda.synchronize()
        assert out["status"].cpu().numpy()[7] == 2
    run_and_check(v16, 1000, 1, 0.8)


@pytest.mark.parametrize("sb,dl", [(1, 3), (3, 3), (16, 6), (64, 9)])
def test_fused_schedule_invariance(sb, dl):
    vol = to_dev(phantom.make_volume(phantom.CONFIGS["c2"], nz=50, z_first=100))
    ref = tsa.tsa_segment(vol, 256, 2, 0.8, pipeline="staged")
    out = tsa.tsa_segment(vol, 256, 2, 0.8, pipeline="fused", slab_slices=sb, label_lag=dl)
    torch.cuda.synchronize()
    for key in ("histogram", "thresholds", "labels", "status"):
        assert torch.equal(out[key], ref[key]), key
