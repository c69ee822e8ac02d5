"""Exhaustive parity on the five BASELINE.json configs (-m gpu).

Every slice of every config, in the launch configuration bench.py times
(tsa_segment with its default pipeline and work units), against the CPU
oracle on all host threads (oracle.segment: histogram, Level-1 exhaustive
search, labels).  Acceptance rule of BASELINE.json:north_star:
histograms and labels bit-exact, thresholds bit-exact unless the oracle's
top-two distinct-partition gap is < 1e-12 relative (then the GPU tuple must be
a near-tie member and its labels equal the oracle's labels at the GPU tuple),
objective within 1e-12 relative.

Sizes: c1 1 slice, c2 300, c3 600 x 11 q (labels every q), c4 300 (canonical)
plus 10 seeded slices in FULL enumeration, c5 all 1000 slices (~150 s of
oracle time on 16 host threads; PAPER.md:593-597 defines the argmax pinned).
"""
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


def compare_volume(vol, bins, k, q, gpu, ref, where, labels=True):
    """gpu: tsa_segment outputs (device tensors); ref: oracle.segment dict."""
    hist = gpu["histogram"].cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(hist, ref["hist"], err_msg=f"{where}: histograms")
    st = gpu["status"].cpu().numpy()
    np.testing.assert_array_equal(st, ref["status"], err_msg=f"{where}: status")
    thr = gpu["thresholds"].cpu().numpy()
    phi = gpu["objective"].cpu().numpy()
    lab = gpu["labels"].cpu().numpy() if labels else None
    exact = 0
    for z in range(vol.shape[0]):
        tag = f"{where} z={z}"
        if ref["status"][z] != 0:
            assert (thr[z] == -1).all() and np.isnan(phi[z]), tag
            if labels:
                assert not lab[z].any(), tag
            continue
        r = {"t": tuple(int(x) for x in ref["thresholds"][z]), "phi": float(ref["phi"][z]),
             "gap": float(ref["gap"][z])}
        ok, why = _pins.accept(hist[z], k, q, thr[z], r, rel=REL,
                               phi_fn=lambda h, t: oracle.phi_at(h, k, q, t))
        assert ok, f"{tag}: {why}"
        same = tuple(int(x) for x in thr[z]) == r["t"]
        v = r["phi"] if same else oracle.phi_at(hist[z], k, q, thr[z])
        assert abs(phi[z] - v) <= REL * abs(v) + (REL if v == 0 else 0), (tag, phi[z], v)
        if labels:
            want = ref["labels"][z] if same else oracle.label(vol[z], k, thr[z])
            np.testing.assert_array_equal(lab[z], want, err_msg=f"{tag}: labels")
        exact += same
    return exact


def gpu_segment(vol_dev, cfg, q, labels=True, **kw):
    out = tsa.tsa_segment(vol_dev, cfg.bins, cfg.k, q, labels=labels, **kw)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_every_slice(name):
    cfg = phantom.CONFIGS[name]
    vol = phantom.make_volume(cfg)
    q = cfg.qs[0]
    gpu = gpu_segment(torch.from_numpy(vol).to(DEV), cfg, q)
    ref = oracle.segment(vol, cfg.bins, cfg.k, q)
    exact = compare_volume(vol, cfg.bins, cfg.k, q, gpu, ref, name)
    assert exact >= 0.9 * (ref["status"] == 0).sum()


def test_c3_every_slice_every_q():
    """c3 as specified: one volume, the search and the labels for each of the
    11 q in {0.5, ..., 1.5} (q = 1 takes the Shannon branch, R6)."""
    cfg = phantom.CONFIGS["c3"]
    vol = phantom.make_volume(cfg)
    v = torch.from_numpy(vol).to(DEV)
    assert len(cfg.qs) == 11
    outs = tsa.tsa_segment_sweep(v, cfg.bins, cfg.k, cfg.qs)  # the bench's c3 step
    torch.cuda.synchronize()
    for q, gpu in zip(cfg.qs, outs):
        gpu = dict(gpu, histogram=outs[0]["histogram"])
        ref = oracle.segment(vol, cfg.bins, cfg.k, q)
        compare_volume(vol, cfg.bins, cfg.k, q, gpu, ref, f"c3 q={q}")


@pytest.mark.parametrize("name,nz", [("c3", 24), ("c2", 16), ("c5", 6)])
def test_sweep_equals_per_q_segment(name, nz):
    """tsa_segment_sweep == one tsa_segment per q, bit for bit."""
    cfg = phantom.CONFIGS[name]
    v = torch.from_numpy(phantom.make_volume(cfg, nz=nz, z_first=cfg.nz // 3)).to(DEV)
    qs = (0.5, 0.8, 1.0, 1.3)
    outs = tsa.tsa_segment_sweep(v, cfg.bins, cfg.k, qs)
    for q, o in zip(qs, outs):
        ref = tsa.tsa_segment(v, cfg.bins, cfg.k, q)
        torch.cuda.synchronize()
        for key in ("thresholds", "status", "labels"):
            assert torch.equal(o[key], ref[key]), (q, key)
        assert torch.equal(o["objective"].view(torch.int64), ref["objective"].view(torch.int64)), q
    assert torch.equal(outs[0]["histogram"], ref["histogram"])


def test_c4_full_enumeration_sample():
    """FULL enumeration (all C(255,4) tuples per slice) on 10 seeded slices of c4."""
    cfg = phantom.CONFIGS["c4"]
    rng = np.random.default_rng(cfg.seed)
    zs = np.sort(rng.choice(cfg.nz, size=10, replace=False))
    vol = np.ascontiguousarray(phantom.make_volume(cfg)[zs])
    q = cfg.qs[0]
    gpu = gpu_segment(torch.from_numpy(vol).to(DEV), cfg, q, enumeration="full")
    ref = oracle.segment(vol, cfg.bins, cfg.k, q)
    compare_volume(vol, cfg.bins, cfg.k, q, gpu, ref, f"c4 full {list(zs)}")


def test_c5_every_slice():
    """c5 (1024 x 1024 x 1000 u16, 4096 bins, k = 2): all 1000 slices."""
    cfg = phantom.CONFIGS["c5"]
    vol = phantom.make_volume(cfg)
    q = cfg.qs[0]
    gpu = gpu_segment(torch.from_numpy(vol).to(DEV), cfg, q)
    ref = oracle.segment(vol, cfg.bins, cfg.k, q)
    compare_volume(vol, cfg.bins, cfg.k, q, gpu, ref, "c5")
