"""Pins for the morphology oracle (
readings DESIGN.md R26-R28 after SPEC.md:118-166)."""
import numpy as np
import pytest

import oracle


def disk_offsets(r):
    return [(dy, dx) for dy in range(-r, r + 1) for dx in range(-r, r + 1) if dy * dy + dx * dx <= r * r]


def np_morph(a, r, is_max):
    """Independent: numpy padded shifts with the neutral border value."""
    pad = 0 if is_max else 255
    p = np.pad(a.astype(np.int32), r, constant_values=pad)
    acc = np.full(a.shape, pad, np.int32)
    for dy, dx in disk_offsets(r):
        sh = p[r + dy:r + dy + a.shape[0], r + dx:r + dx + a.shape[1]]
        acc = np.maximum(acc, sh) if is_max else np.minimum(acc, sh)
    return acc.astype(np.uint8)


def test_disk_sizes():
    """disk(0) = 1, disk(1) = 5, disk(2) = 13 offsets; disk(10) = 317."""
    assert [len(disk_offsets(r)) for r in (0, 1, 2, 10)] == [1, 5, 13, 317]


def test_single_pixel_dilates_to_plus():
    a = np.zeros((7, 7), np.uint8)
    a[3, 3] = 255
    d = oracle.dilate(a, 1)
    assert d.sum() == 5 * 255 and d[3, 2] == d[2, 3] == d[3, 4] == d[4, 3] == 255


@pytest.mark.parametrize("r", [0, 1, 2, 3, 10])
def test_matches_numpy_random(r):
    rng = np.random.default_rng(r)
    a = rng.integers(0, 256, size=(23, 31)).astype(np.uint8)
    np.testing.assert_array_equal(oracle.erode(a, r), np_morph(a, r, False))
    np.testing.assert_array_equal(oracle.dilate(a, r), np_morph(a, r, True))


def test_invariants():
    rng = np.random.default_rng(5)
    a = rng.integers(0, 256, size=(2, 40, 36)).astype(np.uint8)
    r = 3
    op, th = oracle.tophat(a, r)
    np.testing.assert_array_equal(op, oracle.dilate(oracle.erode(a, r), r))
    assert (op <= a).all()  # anti-extensive
    np.testing.assert_array_equal(oracle.tophat(op, r)[0], op)  # idempotent
    np.testing.assert_array_equal(th, (a.astype(int) - op).clip(0).astype(np.uint8))
    # duality with neutral borders
    np.testing.assert_array_equal(oracle.erode(a, r), 255 - oracle.dilate(255 - a, r))
    # monotone
    b = np.maximum(a, rng.integers(0, 256, size=a.shape).astype(np.uint8))
    assert (oracle.tophat(b, r)[0] >= op).all()


def test_constant_and_speck():
    c = np.full((30, 30), 77, np.uint8)
    np.testing.assert_array_equal(oracle.tophat(c, 10)[0], c)
    assert (oracle.tophat(c, 10)[1] == 0).all()
    s = np.zeros((41, 41), np.uint8)
    s[20, 20] = 200  # a speck smaller than disk(10): removed by the opening
    op, th = oracle.tophat(s, 10)
    assert (op == 0).all() and th[20, 20] == 200
