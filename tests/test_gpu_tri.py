"""k_search_tri (canonical k >= 3 with per-item class-term tables in shared
memory, global fallback for large slices) against the FULL-enumeration
kernels (k_rtable + k_search_rows) bit for bit, and against the oracle, for
slices whose non-empty bin count m is below, at and far above the shared-
memory capacity (-m gpu)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_10684_b200 as tsa
from tests import _pins

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def volume_with_m(ms, seed=7, n=128):
    """[len(ms)][n][n] u8 slices, slice i with exactly ms[i] non-empty bins
    (random levels, random skewed counts)."""
    rng = np.random.default_rng(seed)
    out = np.empty((len(ms), n, n), np.uint8)
    for i, m in enumerate(ms):
        levels = np.sort(rng.choice(256, size=m, replace=False)).astype(np.uint8)
        w = rng.gamma(0.7, size=m) + 0.05
        v = rng.choice(levels, size=n * n, p=w / w.sum())
        v[:m] = levels  # every level present
        out[i] = rng.permutation(v).reshape(n, n)
    return out


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("q", [0.6, 1.0, 1.4])
def test_tri_equals_full_enumeration(k, q):
    ms = [5, 40, 90, 113, 114, 115, 130] + ([200, 256] if k == 3 else [160])
    vol = torch.from_numpy(volume_with_m(ms, seed=k * 10 + int(q * 10))).to(DEV)
    a = tsa.tsa_segment(vol, 256, k, q)                      # canonical: k_search_tri
    b = tsa.tsa_segment(vol, 256, k, q, enumeration="full")  # k_rtable + k_search_rows
    torch.cuda.synchronize()
    for key in ("thresholds", "status", "labels", "histogram"):
        assert torch.equal(a[key], b[key]), key
    assert torch.equal(a["objective"].view(torch.int64), b["objective"].view(torch.int64))


@pytest.mark.parametrize("k", [3, 4])
def test_tri_units_and_oracle(k):
    ms = [12, 95, 120]
    vh = volume_with_m(ms, seed=3 + k)
    vol = torch.from_numpy(vh).to(DEV)
    ref = tsa.tsa_segment(vol, 256, k, 0.8, units=1)
    for u in (2, 7):
        out = tsa.tsa_segment(vol, 256, k, 0.8, units=u)
        torch.cuda.synchronize()
        assert torch.equal(out["thresholds"], ref["thresholds"]), u
    hist = ref["histogram"].cpu().numpy().astype(np.uint32)
    thr = ref["thresholds"].cpu().numpy()
    for z in range(len(ms)):
        r = oracle.search(hist[z], k, 0.8)
        ok, why = _pins.accept(hist[z], k, 0.8, thr[z], r, phi_fn=lambda h, t: oracle.phi_at(h, k, 0.8, t))
        assert ok, (z, why)
