"""Pins for the pre-processing oracle (
readings DESIGN.md R23-R25 after SPEC.md:73-81)."""
import numpy as np
import pytest

import oracle
import phantom


def test_spec_worked_example():
    """[-2000, 0, 500], background -2000 -> [0, 0, 255]."""
    g, lo, hi = oracle.preprocess(np.array([-2000, 0, 500], np.int16))
    assert g.tolist() == [0, 0, 255] and (lo, hi) == (0, 500)


def test_constant_and_all_background():
    assert oracle.preprocess(np.full(4, 7, np.int16))[0].tolist() == [0, 0, 0, 0]
    assert oracle.preprocess(np.full(5, -2000, np.int16))[0].tolist() == [0] * 5


@pytest.mark.parametrize("seed", range(6))
def test_matches_float_formula_and_invariants(seed):
    """Independent: numpy float64 floor(255 (v - lo)/(hi - lo) + 1/2) (the
    quotient never rounds across a half: its distance to one is >= 1/(2(hi-lo)));
    output range, min -> 0, max -> 255, monotone in HU, background -> 0."""
    rng = np.random.default_rng(seed)
    v = rng.integers(-1500, 3000, size=5000).astype(np.int16)
    v[rng.random(5000) < 0.2] = -2000
    if seed == 1:
        v[::7] = 17  # many exact ties of the rounding
    g, lo, hi = oracle.preprocess(v)
    nb = v[v != -2000].astype(np.int64)
    assert (lo, hi) == (nb.min(), nb.max())
    ref = np.floor(255.0 * (np.where(v == -2000, lo, v).astype(np.int64) - lo) / (hi - lo) + 0.5)
    np.testing.assert_array_equal(g, ref.astype(np.uint8))
    assert g.min() == 0 and g.max() == 255
    assert (g[v == -2000] == 0).all()
    o = np.argsort(v, kind="stable")
    assert (np.diff(g[o][v[o] != -2000].astype(int)) >= 0).all()


def test_half_ties_round_away_from_zero():
    """hi - lo = 510: v - lo = 1 gives 255/510 = 0.5 exactly -> 1."""
    v = np.array([0, 1, 3, 510], np.int16)
    g, lo, hi = oracle.preprocess(v, background=-2000)
    assert g.tolist() == [0, 1, 2, 255]  # 0.5 -> 1, 1.5 -> 2


def test_phantom_hu_window():
    """The HU phantom: background exactly -2000 outside the FOV, window from
    the data, every non-background voxel mapped into 0..255."""
    v = phantom.make_volume(phantom.CONFIGS["f2"], nz=3, z_first=100)
    g, lo, hi = oracle.preprocess(v)
    assert lo > -2000 and hi > lo
    assert (g[v == -2000] == 0).all()
