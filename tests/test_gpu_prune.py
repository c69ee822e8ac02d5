"""The bounded k = 2 search (k_search.cuh k2_tile PRUNE, k_k2_seed) against
the plain exhaustive kernel (TSA_K2_PRUNE=0) and the oracle (-m gpu).

The pruned search skips a group of tuples only when an upper bound of every
value in it is strictly below a score already reached, so thresholds,
objective and labels must be bit-identical to the exhaustive kernel's -- also
on inputs built to tie (uniform and mirror-symmetric histograms, where the
lowest tuple among equal scores must win) and on every q < 1 the library
prunes for.  PAPER.md:593-597 (the argmax of the pseudo-additive objective).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import phantom
import paper_2012_10684_b200 as tsa
from tests import _pins

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(vol, bins, q, prune, **kw):
    old = os.environ.get("TSA_K2_PRUNE")
    os.environ["TSA_K2_PRUNE"] = "1" if prune else "0"
    try:
        out = tsa.tsa_segment(vol, bins, 2, q, **kw)
        torch.cuda.synchronize()
    finally:
        if old is None:
            del os.environ["TSA_K2_PRUNE"]
        else:
            os.environ["TSA_K2_PRUNE"] = old
    return {k: v.cpu().numpy() for k, v in out.items() if v is not None}


def _same(a, b, where):
    for key in ("thresholds", "status", "labels", "histogram"):
        if key in a:
            np.testing.assert_array_equal(a[key], b[key], err_msg=f"{where}: {key}")
    # objective bit-identical (NaN where no split)
    oa, ob = a["objective"].view(np.uint64), b["objective"].view(np.uint64)
    np.testing.assert_array_equal(oa, ob, err_msg=f"{where}: objective bits")


@pytest.mark.parametrize("q", [0.3, 0.5, 0.8, 0.95])
def test_c5_slab_pruned_equals_exhaustive(q):
    cfg = phantom.CONFIGS["c5"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=24, z_first=300)).to(DEV)
    _same(_run(vol, cfg.bins, q, True, pipeline="staged"), _run(vol, cfg.bins, q, False, pipeline="staged"),
          f"c5 q={q}")


@pytest.mark.parametrize("q", [0.5, 0.8])
def test_c2_staged_pruned_equals_exhaustive(q):
    cfg = phantom.CONFIGS["c2"]
    vol = torch.from_numpy(phantom.make_volume(cfg, nz=40, z_first=100)).to(DEV)
    _same(_run(vol, cfg.bins, q, True, pipeline="staged"), _run(vol, cfg.bins, q, False, pipeline="staged"),
          f"c2 q={q}")


def _from_hist(h, nx):
    """A slice (u16) whose histogram is exactly h (values laid out in order)."""
    v = np.repeat(np.arange(len(h), dtype=np.uint16), h)
    assert v.size == nx * nx
    return v.reshape(nx, nx)


@pytest.mark.parametrize("bins", [256, 4096])
def test_ties_lowest_tuple(bins):
    nx = 256
    rng = np.random.default_rng(7)
    slices = []
    # uniform over every bin (all class sizes multiples: many exact ties)
    h = np.zeros(bins, np.int64)
    used = min(bins, 256)
    h[:used] = nx * nx // used
    slices.append(_from_hist(h, nx))
    # mirror-symmetric two-mode histogram
    h = np.zeros(bins, np.int64)
    half = np.array([40, 200, 900, 2000, 5000, 2000, 900, 200, 40] * 2)
    pos = np.linspace(0, bins - 1, half.size).astype(int)
    h[pos] = half
    h[pos[0]] += nx * nx - h.sum()
    slices.append(_from_hist(h, nx))
    # four equal spikes
    h = np.zeros(bins, np.int64)
    h[np.linspace(3, bins - 4, 4).astype(int)] = nx * nx // 4
    slices.append(_from_hist(h, nx))
    # random sparse histogram
    h = np.zeros(bins, np.int64)
    idx = rng.choice(bins, size=min(bins, 700), replace=False)
    h[idx] = rng.integers(1, 60, size=idx.size)
    h[idx[0]] += nx * nx - h.sum()
    slices.append(_from_hist(h, nx))
    vol_np = np.stack(slices)
    vol = torch.from_numpy(vol_np).to(DEV)
    for q in (0.5, 0.8):
        a = _run(vol, bins, q, True, pipeline="staged")
        b = _run(vol, bins, q, False, pipeline="staged")
        _same(a, b, f"ties bins={bins} q={q}")
        ref = oracle.segment(vol_np, bins, 2, q)
        for z in range(vol_np.shape[0]):
            if ref["status"][z] != 0:
                continue
            r = {"t": tuple(int(x) for x in ref["thresholds"][z]), "phi": float(ref["phi"][z]),
                 "gap": float(ref["gap"][z])}
            ok, why = _pins.accept(ref["hist"][z], 2, q, a["thresholds"][z], r, rel=1e-12,
                                   phi_fn=lambda hh, t: oracle.phi_at(hh, 2, q, t))
            assert ok, f"bins={bins} q={q} z={z}: {why}"


def _tie_volume(nx=128):
    """u8 slices built to tie: uniform over 64 / 90 levels, mirror-symmetric
    modes, equal spikes."""
    out = []
    for used in (64, 90):
        h = np.zeros(256, np.int64)
        lv = np.linspace(0, 255, used).astype(int)
        h[lv] = nx * nx // used
        h[lv[0]] += nx * nx - h.sum()
        out.append(h)
    h = np.zeros(256, np.int64)
    half = np.array([30, 100, 400, 900, 2000, 900, 400, 100, 30] * 3)
    pos = np.linspace(2, 250, half.size).astype(int)
    h[pos] = half
    h[pos[0]] += nx * nx - h.sum()
    out.append(h)
    h = np.zeros(256, np.int64)
    h[np.linspace(5, 250, 6).astype(int)] = nx * nx // 6
    h[5] += nx * nx - h.sum()
    out.append(h)
    return np.stack([np.repeat(np.arange(256, dtype=np.uint8), hh).reshape(nx, nx) for hh in out])


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("q", [0.6, 1.0, 1.4])
def test_tri_pruned_ties_equal_full(k, q):
    """k >= 3: the chunk-bounded canonical search (k_search_tri) against the
    unpruned FULL enumeration (k_search_rows), bit for bit, on tie-heavy
    histograms (the lowest tuple among equal scores must win)."""
    vol_np = _tie_volume()
    vol = torch.from_numpy(vol_np).to(DEV)
    a = tsa.tsa_segment(vol, 256, k, q)
    b = tsa.tsa_segment(vol, 256, k, q, enumeration="full")
    torch.cuda.synchronize()
    for key in ("thresholds", "status", "labels"):
        np.testing.assert_array_equal(a[key].cpu().numpy(), b[key].cpu().numpy(), err_msg=f"k={k} q={q} {key}")
    np.testing.assert_array_equal(a["objective"].cpu().numpy().view(np.uint64),
                                  b["objective"].cpu().numpy().view(np.uint64))


@pytest.mark.parametrize("q", [0.4, 0.8])
def test_k2_many_bins_unstaged_seed(q):
    """M > 1024 non-empty bins (k_k2_seed reads the rows from global memory,
    16-row bound records near the slice end) and small M (< 32 rows)."""
    rng = np.random.default_rng(11)
    nx = 256
    slices = []
    for used in (2500, 1100, 20, 5):
        h = np.zeros(4096, np.int64)
        idx = np.sort(rng.choice(4096, size=used, replace=False))
        h[idx] = rng.integers(1, max(2, 2 * nx * nx // used), size=used)
        scale = (nx * nx - used) / max(1, h.sum() - used)
        h[idx] = 1 + np.floor((h[idx] - 1) * min(1.0, scale)).astype(np.int64)
        h[idx[0]] += nx * nx - h.sum()
        slices.append(_from_hist(h, nx))
    vol = torch.from_numpy(np.stack(slices)).to(DEV)
    _same(_run(vol, 4096, q, True, pipeline="staged"), _run(vol, 4096, q, False, pipeline="staged"),
          f"many bins q={q}")


@pytest.mark.parametrize("q", [0.5, 0.8])
def test_k2_full_enumeration_equals_canonical(q):
    """FULL enumeration (positions = every bin, empty ones included; the
    unpruned kernel) against the pruned canonical search, L = 256 with ~90
    non-empty bins and L = 4096 (12-bit): the same thresholds and objective."""
    for name, nz in (("c2", 6), ("c5", 2)):
        cfg = phantom.CONFIGS[name]
        vol = torch.from_numpy(phantom.make_volume(cfg, nz=nz, z_first=150)).to(DEV)
        a = _run(vol, cfg.bins, q, True, pipeline="staged")
        b = _run(vol, cfg.bins, q, True, pipeline="staged", enumeration="full")
        _same(a, b, f"{name} full vs canonical q={q}")
