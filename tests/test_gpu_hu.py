"""GPU parity of the HU path: pre-processing (readings
DESIGN.md R23-R25) fused into the histogram and label passes of the 1-D path
(SURVEY.md §8(f) row 2), against oracle.preprocess + the 1-D oracle (-m gpu).
Bar: the 8-bit image, its histograms and the labels bit-exact; thresholds and
objective under the 1-D acceptance rule."""
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


def check(vol, k, q, bg=-2000, slices=None, obj=0):
    out = tsa.tsa_hu_segment(to_dev(vol), k, q, background=bg, objective=obj)
    torch.cuda.synchronize()
    gray, lo, hi = oracle.preprocess(vol, bg)
    assert tuple(out["window"].cpu().tolist()) == (lo, hi) or (vol == bg).all()
    hist = out["histogram"].cpu().numpy().astype(np.uint32)
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    st = out["status"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    for z in (range(vol.shape[0]) if slices is None else slices):
        h_ref, _ = oracle.histogram(gray[z], 256)
        np.testing.assert_array_equal(hist[z], h_ref, err_msg=f"hist z={z}")
        ref = oracle.search(h_ref, k, q, objective=obj)
        assert st[z] == ref["status"], (z, st[z], ref["status"])
        if ref["status"] != oracle.OK:
            assert (lab[z] == 0).all()
            continue
        ok, why = _pins.accept(h_ref, k, q, thr[z], ref, objective=obj, rel=REL,
                               phi_fn=lambda h, t: oracle.phi_at(h, k, q, t, obj))
        assert ok, (z, why)
        v = ref["phi"] if tuple(thr[z]) == tuple(ref["t"]) else oracle.phi_at(h_ref, k, q, thr[z], obj)
        assert abs(phi[z] - v) <= REL * abs(v) + (REL if v == 0 else 0), z
        np.testing.assert_array_equal(lab[z], oracle.label(gray[z], k, thr[z]), err_msg=f"labels z={z}")
    return out


def test_preprocess_bitexact_phantom():
    vol = phantom.make_volume(phantom.CONFIGS["f2"], nz=12, z_first=80)
    gray, win = tsa.tsa_hu_preprocess(to_dev(vol))
    ref, lo, hi = oracle.preprocess(vol)
    assert tuple(win.cpu().tolist()) == (lo, hi)
    np.testing.assert_array_equal(gray.cpu().numpy(), ref)


@pytest.mark.parametrize("seed", range(5))
def test_preprocess_bitexact_random(seed):
    rng = np.random.default_rng(seed)
    lo, hi = sorted(rng.integers(-4096, 4096, size=2))
    vol = rng.integers(lo, hi + 1, size=(3, 16, 32)).astype(np.int16)
    bg = int(rng.integers(-4096, 4096)) if seed % 2 else -2000
    vol[rng.random(vol.shape) < 0.3] = bg
    gray, win = tsa.tsa_hu_preprocess(to_dev(vol), background=bg)
    ref, rlo, rhi = oracle.preprocess(vol, bg)
    np.testing.assert_array_equal(gray.cpu().numpy(), ref)


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("q", [0.8, 1.0, 1.3])
def test_segment_hu_phantom(k, q):
    vol = phantom.make_volume(phantom.CONFIGS["f2"], nz=6, z_first=110)
    check(vol, k, q)


def test_segment_hu_full_workload_sampled():
    """The f2 workload (512x512x300 HU): histograms and labels of every slice,
    the exhaustive search on every 10th slice."""
    vol = phantom.make_volume(phantom.CONFIGS["f2"])
    out = check(vol, 2, 0.8, slices=range(0, 300, 10))
    gray, _, _ = oracle.preprocess(vol)
    hist = out["histogram"].cpu().numpy().astype(np.uint32)
    lab = out["labels"].cpu().numpy()
    thr = out["thresholds"].cpu().numpy()
    for z in range(300):
        np.testing.assert_array_equal(hist[z], oracle.histogram(gray[z], 256)[0])
        np.testing.assert_array_equal(lab[z], oracle.label(gray[z], 2, thr[z]))


def test_fused_equals_preprocess_then_u8_path():
    """tsa_hu_segment == tsa_segment(tsa_hu_preprocess(vol)) bit for bit."""
    vol = to_dev(phantom.make_volume(phantom.CONFIGS["f2"], nz=20, z_first=60))
    a = tsa.tsa_hu_segment(vol, 2, 0.8)
    gray, _ = tsa.tsa_hu_preprocess(vol)
    b = tsa.tsa_segment(gray, 256, 2, 0.8)
    for key in ("thresholds", "histogram", "status", "labels"):
        assert torch.equal(a[key], b[key]), key
    assert torch.equal(a["objective"], b["objective"])


@pytest.mark.parametrize("k", [1, 2, 4])
def test_segment_hu_random_and_cutoff_edges(k):
    """Random HU with a background value inside the data range and windows whose
    label cutoffs land on -1 HU, on the background value and past the int16 range."""
    rng = np.random.default_rng(40 + k)
    vol = rng.integers(-300, 300, size=(4, 32, 32)).astype(np.int16)
    vol[0] = rng.integers(-256, 255, size=(32, 32))  # window [-256, 254]: a cutoff can be -1
    vol[1, :8] = -40  # background value inside the window
    vol[2] = rng.choice([-1000, -1, 0, 700], size=(32, 32))
    check(vol, k, 0.7, bg=-40)


def test_segment_hu_overflow_and_degenerate():
    vol = np.full((4, 16, 16), -2000, np.int16)
    vol[1] = np.arange(256, dtype=np.int16).reshape(16, 16) * 3 - 300
    vol[2] = vol[1]
    vol[2, 0, 0] = 5000  # outside [-4096, 4095]: LEVEL_OVERFLOW for slice 2
    vol[3, :, :8] = 100
    out = tsa.tsa_hu_segment(to_dev(vol), 1, 0.8)
    st = out["status"].cpu().numpy()
    assert st[2] == oracle.LEVEL_OVERFLOW
    assert st[0] == oracle.NO_VALID_SPLIT  # all background: one 8-bit level
    assert (out["labels"][2] == 0).all() and (out["labels"][0] == 0).all()
    gray, lo, hi = oracle.preprocess(vol)
    assert tuple(out["window"].cpu().tolist()) == (lo, hi) == (-300, 5000)
    for z in (1, 3):
        h, _ = oracle.histogram(gray[z], 256)
        np.testing.assert_array_equal(out["histogram"][z].cpu().numpy().astype(np.uint32), h)


def test_all_background_volume():
    vol = np.full((2, 16, 16), -2000, np.int16)
    out = tsa.tsa_hu_segment(to_dev(vol), 2, 0.8)
    assert (out["status"].cpu().numpy() == oracle.NO_VALID_SPLIT).all()
    gray, _ = tsa.tsa_hu_preprocess(to_dev(vol))
    assert (gray == 0).all()


def test_two_phase_slabs_equal_whole_volume():
    """Slices split into slabs: phase 1 per slab, the window reduced (min lo,
    max hi -- what dist.reduce_window all-reduces across ranks), phase 2 per
    slab: bit-identical to tsa_hu_segment of the whole volume."""
    vol = to_dev(phantom.make_volume(phantom.CONFIGS["f2"], nz=30, z_first=50))
    ref = tsa.tsa_hu_segment(vol, 2, 0.8)
    slabs = [vol[:11], vol[11:12], vol[12:]]
    ph1 = [tsa.tsa_hu_histogram(s.contiguous(), 2, 0.8) for s in slabs]
    wins = torch.stack([w for w, _ in ph1]).cpu()
    win = torch.tensor([int(wins[:, 0].min()), int(wins[:, 1].max())], dtype=torch.int32).to(DEV)
    outs = [tsa.tsa_hu_finish(s.contiguous(), 2, 0.8, win, ws) for s, (_, ws) in zip(slabs, ph1)]
    for key in ("thresholds", "objective", "histogram", "status", "labels"):
        assert torch.equal(torch.cat([o[key] for o in outs]), ref[key]), key
    assert torch.equal(win, ref["window"])


def _hu_worker(rank, world, port, ret):
    import os
    import sys

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import phantom as ph
    from paper_2012_10684_b200.dist import hu_segment_slabs, slab_range

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        vol = ph.make_volume(ph.CONFIGS["f2"], nz=9, z_first=120)
        z0, z1 = slab_range(9, world, rank)
        out = hu_segment_slabs(torch.from_numpy(np.ascontiguousarray(vol[z0:z1])).cuda(), 2, 0.8)
        torch.cuda.synchronize()
        ret[rank] = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    finally:
        dist.destroy_process_group()


def test_hu_segment_slabs_two_ranks():
    """dist.hu_segment_slabs on 2 gloo ranks (both on cuda:0) == one GPU."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    ps = [ctx.Process(target=_hu_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    vol = phantom.make_volume(phantom.CONFIGS["f2"], nz=9, z_first=120)
    ref = tsa.tsa_hu_segment(to_dev(vol), 2, 0.8)
    for key in ("thresholds", "objective", "labels", "histogram"):
        got = np.concatenate([ret[0][key], ret[1][key]])
        np.testing.assert_array_equal(got, ref[key].cpu().numpy(), err_msg=key)
    np.testing.assert_array_equal(ret[0]["window"], ref["window"].cpu().numpy())
