"""GPU parity of the morphology kernels (
readings DESIGN.md R26-R28) against the brute-force oracle, bit-exact (-m gpu)."""
import numpy as np
import pytest
import torch

import oracle
import phantom
import paper_2012_10684_b200 as tsa

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def ref(a, op, r):
    if op == "erode":
        return oracle.erode(a, r)
    if op == "dilate":
        return oracle.dilate(a, r)
    o, t = oracle.tophat(a, r)
    return o if op == "open" else t


@pytest.mark.parametrize("op", ["erode", "dilate", "open", "tophat"])
@pytest.mark.parametrize("r", [1, 2, 3, 5, 10])
@pytest.mark.parametrize("shape", [(2, 64, 64), (1, 37, 300), (1, 25, 513), (2, 9, 5)])
def test_morph_random(op, r, shape):
    rng = np.random.default_rng(r * 7 + shape[2])
    a = rng.integers(0, 256, size=shape).astype(np.uint8)
    a[:, : shape[1] // 3] //= 8  # dark band: structure for the opening to keep
    out = tsa.tsa_morph(to_dev(a), op, r).cpu().numpy()
    np.testing.assert_array_equal(out, ref(a, op, r), err_msg=f"{op} r={r} {shape}")


def test_tophat_phantom_full_slices():
    """The bench configuration: 512x512 phantom slices, disk(10) top-hat."""
    a = phantom.make_volume(phantom.CONFIGS["c2"], nz=3, z_first=100)
    out = tsa.tsa_morph(to_dev(a), "tophat", 10).cpu().numpy()
    o = tsa.tsa_morph(to_dev(a), "open", 10).cpu().numpy()
    ro, rt = oracle.tophat(a, 10)
    np.testing.assert_array_equal(o, ro)
    np.testing.assert_array_equal(out, rt)


def test_radius0_identity_and_errors():
    a = np.arange(64, dtype=np.uint8).reshape(1, 8, 8)
    assert torch.equal(tsa.tsa_morph(to_dev(a), "open", 0).cpu(), torch.from_numpy(a))
    assert (tsa.tsa_morph(to_dev(a), "tophat", 0) == 0).all()
    with pytest.raises(tsa.TsaError):
        tsa.tsa_morph(to_dev(a), "open", 11)


def test_speck_removed_and_invariants():
    a = np.zeros((1, 64, 64), np.uint8)
    a[0, 30, 30] = 200
    assert (tsa.tsa_morph(to_dev(a), "open", 10) == 0).all()
    rng = np.random.default_rng(1)
    b = rng.integers(0, 256, size=(1, 48, 80)).astype(np.uint8)
    bo = tsa.tsa_morph(to_dev(b), "open", 4)
    assert (bo.cpu().numpy() <= b).all()
    assert torch.equal(tsa.tsa_morph(bo, "open", 4), bo)  # idempotent
