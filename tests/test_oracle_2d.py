"""Pins for the 2-D Tsallis oracle."""
import itertools

import mpmath
import numpy as np
import pytest

import oracle
import phantom

mpmath.mp.dps = 50


def np_mean3x3(f):
    """Independent: numpy edge padding + nine shifted sums, floor division."""
    p = np.pad(f.astype(np.int64), 1, mode="edge")
    s = sum(p[1 + dy:1 + dy + f.shape[0], 1 + dx:1 + dx + f.shape[1]]
            for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    return (s // 9).astype(np.uint8)


def test_mean3x3_and_hist2d_match_numpy():
    f = phantom.make_volume(phantom.CONFIGS["c2"], nz=1, z_first=120)[0]
    g = oracle.mean3x3(f)
    np.testing.assert_array_equal(g, np_mean3x3(f))
    h, st = oracle.hist2d(f, 256)
    assert st == oracle.OK
    ref = np.bincount(f.astype(np.int64).ravel() * 256 + g.astype(np.int64).ravel(),
                      minlength=256 * 256).reshape(256, 256)
    np.testing.assert_array_equal(h, ref)
    # odd sizes exercise the replicate border on every side
    rng = np.random.default_rng(0)
    f2 = rng.integers(0, 256, size=(7, 11)).astype(np.uint8)
    np.testing.assert_array_equal(oracle.mean3x3(f2), np_mean3x3(f2))


def test_hist2d_overflow():
    f = np.full((8, 8), 10, np.uint8)
    f[3, 3] = 200
    h, st = oracle.hist2d(f, 64)
    assert st == oracle.LEVEL_OVERFLOW


def mp_phi2d(h, t, s, q):
    """Composition identity phi = (A1 A2 - 1)/(1 - q) (Shannon sum at q = 1), 50 digits."""
    h = np.asarray(h, dtype=np.int64)
    L = h.shape[0]
    q = mpmath.mpf(q)
    classes = [h[:t + 1, :s + 1], h[t + 1:, s + 1:]]
    A, S = [], []
    for c in classes:
        n = int(c.sum())
        if n == 0:
            return None
        cells = [int(x) for x in c.ravel() if x]
        if q == 1:
            S.append(mpmath.log(n) - sum(mpmath.mpf(x) * mpmath.log(x) for x in cells) / n)
        else:
            A.append(sum((mpmath.mpf(x) / n) ** q for x in cells))
    if q == 1:
        return S[0] + S[1]
    return (A[0] * A[1] - 1) / (1 - q)


@pytest.mark.parametrize("seed", range(12))
def test_2d_bruteforce_mpmath(seed):
    rng = np.random.default_rng(50 + seed)
    L = int(rng.integers(3, 8))
    q = [0.5, 0.8, 1.0, 1.3, 2.0, 0.7][seed % 6]
    h = rng.integers(0, 20, size=(L, L)).astype(np.uint32)
    h[rng.random((L, L)) < 0.4] = 0
    vals = {}
    for t, s in itertools.product(range(L - 1), range(L - 1)):
        v = mp_phi2d(h, t, s, q)
        if v is not None:
            vals[(t, s)] = v
            o = oracle.phi2d_at(h, q, t, s)
            assert abs(o - float(v)) <= 1e-13 * max(1.0, abs(float(v)))
        else:
            assert oracle.phi2d_at(h, q, t, s) is None
    r = oracle.search2d(h, q)
    if not vals:
        assert r["status"] == oracle.NO_VALID_SPLIT
        return
    best = max(vals.values())
    ties = {k for k, v in vals.items() if v >= best - abs(best) * 1e-13}
    assert (r["t"], r["s"]) in ties
    if len(ties) == 1:
        assert (r["t"], r["s"]) == min(ties)


@pytest.mark.parametrize("q", [0.6, 1.0, 1.4])
def test_diagonal_2d_equals_1d(q):
    """A diagonal 2-D histogram (g == f) with s = t is the 1-D problem: phi2d(t,t) = phi1d(t)."""
    rng = np.random.default_rng(9)
    L = 24
    d = rng.integers(0, 50, size=L).astype(np.uint32)
    d[::5] = 0
    h = np.diag(d).astype(np.uint32)
    for t in range(L - 1):
        a = oracle.phi2d_at(h, q, t, t)
        b = oracle.phi_at(d, 1, q, (t,))
        assert (a is None) == (b is None)
        if a is not None:
            assert abs(a - b) <= 1e-13 * max(1.0, abs(b))


def test_2d_point_masses():
    h = np.zeros((16, 16), np.uint32)
    h[3, 3] = 40
    h[12, 12] = 40
    for q in (0.5, 1.0, 1.5):
        r = oracle.search2d(h, q)
        assert (r["t"], r["s"]) == (3, 3) and r["phi"] == 0.0


def test_2d_transpose_symmetry():
    rng = np.random.default_rng(4)
    h = rng.integers(0, 30, size=(12, 12)).astype(np.uint32)
    for q in (0.7, 1.0, 1.3):
        for t, s in [(2, 5), (7, 1), (4, 4), (9, 10)]:
            a = oracle.phi2d_at(h, q, t, s)
            b = oracle.phi2d_at(h.T.copy(), q, s, t)
            assert abs(a - b) <= 1e-13 * abs(a)


def _partition(h, t, s):
    """The classes of (t,s) as sets of non-empty cells (independent of the oracle)."""
    nz = {(int(i), int(j)) for i, j in zip(*np.nonzero(h))}
    return (frozenset(c for c in nz if c[0] <= t and c[1] <= s),
            frozenset(c for c in nz if c[0] > t and c[1] > s))


@pytest.mark.parametrize("seed", range(6))
def test_2d_gap_over_distinct_partitions(seed):
    """Runner-up = best value over candidates whose cell partition differs from
    t*'s (50-digit values, partitions as explicit cell sets)."""
    rng = np.random.default_rng(300 + seed)
    L = int(rng.integers(5, 9))
    q = [0.6, 1.0, 1.4][seed % 3]
    h = rng.integers(0, 15, size=(L, L)).astype(np.uint32)
    h[rng.integers(0, L, 2), :] = 0  # empty rows and columns make equivalent candidates
    h[:, rng.integers(0, L, 2)] = 0
    r = oracle.search2d(h, q)
    if r["status"] != oracle.OK:
        return
    best_part = _partition(h, r["t"], r["s"])
    others = [mp_phi2d(h, t, s, q) for t, s in itertools.product(range(L - 1), range(L - 1))
              if _partition(h, t, s) != best_part]
    others = [v for v in others if v is not None]
    if not others:
        assert r["gap"] == float("inf")
        return
    phi2 = max(others)
    gap = (mpmath.mpf(r["phi"]) - phi2) / abs(mpmath.mpf(r["phi"]))
    assert abs(r["gap"] - float(gap)) <= 1e-12 * max(1.0, abs(float(gap))) + 1e-13


def test_2d_equivalent_candidates_tie_exactly_and_lowest_wins():
    """Empty rows/columns between candidates leave the partition unchanged, so
    their values tie bit for bit and the lowest candidate (non-empty row and
    column) is returned -- the reading the canonical GPU search relies on."""
    rng = np.random.default_rng(77)
    L = 10
    h = rng.integers(1, 9, size=(L, L)).astype(np.uint32)
    h[4:7, :] = 0
    h[:, 2:5] = 0
    for t in range(L - 1):
        for s in range(L - 1):
            a = oracle.phi2d_at(h, 0.7, t, s)
            tt = t if not 4 <= t <= 6 else 3
            ss = s if not 2 <= s <= 4 else 1
            assert (a is None) == (oracle.phi2d_at(h, 0.7, tt, ss) is None)
            if a is not None:
                assert a == oracle.phi2d_at(h, 0.7, tt, ss)
    for q in (0.5, 1.0, 1.5):
        r = oracle.search2d(h, q)
        assert r["t"] not in (4, 5, 6) and r["s"] not in (2, 3, 4)


def test_2d_point_masses_gap():
    h = np.zeros((16, 16), np.uint32)
    h[3, 3] = 40
    h[12, 12] = 40
    r = oracle.search2d(h, 0.8)
    assert r["gap"] == float("inf")  # a single distinct valid partition


def test_2d_thread_count_invariant():
    f = phantom.make_volume(phantom.CONFIGS["c2"], nz=1, z_first=60)[0][::4, ::4].copy()
    h, _ = oracle.hist2d(f, 256)
    hs = h[::4, ::4].copy()  # 64 levels keeps the O(L^4) search quick
    a = oracle.search2d(hs, 0.8, threads=1)
    b = oracle.search2d(hs, 0.8, threads=4)
    assert a == b
