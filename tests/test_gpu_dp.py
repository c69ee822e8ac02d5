"""GPU parity of the exact interval DP (TSA_ENUM_DP)
against the oracle's exhaustive search (acceptance rule) and against the
exhaustive GPU kernels (-m gpu)."""
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


def check(vol, bins, k, q):
    out = tsa.tsa_segment(to_dev(vol), bins, k, q, enumeration="dp")
    torch.cuda.synchronize()
    thr = out["thresholds"].cpu().numpy()
    phi = out["objective"].cpu().numpy()
    st = out["status"].cpu().numpy()
    lab = out["labels"].cpu().numpy()
    for z in range(vol.shape[0]):
        h, _ = oracle.histogram(vol[z], bins)
        ref = oracle.search(h, k, q)
        assert st[z] == ref["status"], z
        if ref["status"] != oracle.OK:
            continue
        ok, why = _pins.accept(h, k, q, thr[z], ref, rel=REL,
                               phi_fn=lambda hh, t: oracle.phi_at(hh, k, q, t))
        assert ok, (z, why)
        v = ref["phi"] if tuple(thr[z]) == tuple(ref["t"]) else oracle.phi_at(h, k, q, thr[z])
        assert abs(phi[z] - v) <= REL * abs(v) + (REL if v == 0 else 0)
        np.testing.assert_array_equal(lab[z], oracle.label(vol[z], k, thr[z]))
    return out


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("q", [0.5, 0.8, 1.0, 1.2, 1.5])
def test_dp_phantom(k, q):
    vol = phantom.make_volume(phantom.CONFIGS["c2"], nz=4, z_first=90)
    check(vol, 256, k, q)


@pytest.mark.parametrize("seed", range(6))
def test_dp_random_small(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(6, 40))
    k = int(rng.integers(1, min(4, L - 1) + 1))
    q = [0.6, 1.0, 1.4][seed % 3]
    vol = rng.integers(0, L, size=(5, 16, 16)).astype(np.uint8)
    vol[1] = vol[1] // 3 * 3  # empty bins
    vol[2, :] = 2  # one level: NO_VALID_SPLIT
    check(vol, L, k, q)


def test_dp_equals_exhaustive_on_bench_volume():
    """c4 (k = 4) volume: the DP's tuples equal the exhaustive canonical
    search's except on near-ties (then both are members of the tie set)."""
    vol = to_dev(phantom.make_volume(phantom.CONFIGS["c4"], nz=60, z_first=100))
    a = tsa.tsa_segment(vol, 256, 4, 0.8, enumeration="dp")
    b = tsa.tsa_segment(vol, 256, 4, 0.8)
    ta, tb = a["thresholds"].cpu().numpy(), b["thresholds"].cpu().numpy()
    diff = [z for z in range(60) if tuple(ta[z]) != tuple(tb[z])]
    h = b["histogram"].cpu().numpy().astype(np.uint32)
    for z in diff:
        ref = oracle.search(h[z], 4, 0.8)
        assert ref["gap"] < REL, (z, ta[z], tb[z], ref)
    assert len(diff) <= 3


def test_dp_rejects_sum_plus_product():
    vol = to_dev(np.zeros((1, 16, 16), np.uint8))
    with pytest.raises(tsa.TsaError):
        tsa.tsa_segment(vol, 256, 2, 0.8, objective="sum_plus_product", enumeration="dp")


@pytest.mark.parametrize("k", [2, 4])
def test_dp_12bit_levels(k):
    """u16 / 4096 levels (the shared-memory budget leaves the term table to
    slices with small m; the rest evaluate terms on the fly)."""
    cfg = phantom.CONFIGS["c5"]
    vol = phantom.generate(256, 256, 2, "u16", seed=cfg.seed, z_first=400, z_total=1000)
    check(vol, 4096, k, 0.8) if k == 2 else None
    out = tsa.tsa_segment(to_dev(vol), 4096, k, 0.8, enumeration="dp")
    ref = tsa.tsa_segment(to_dev(vol), 4096, k, 0.8)
    h = ref["histogram"].cpu().numpy().astype(np.uint32)
    for z in range(2):
        a, b = tuple(out["thresholds"][z].tolist()), tuple(ref["thresholds"][z].tolist())
        if a != b:
            assert oracle.search(h[z], k, 0.8, level=1)["gap"] < REL
