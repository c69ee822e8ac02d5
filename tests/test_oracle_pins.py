"""Pins for the CPU oracle (-m "not gpu").  Each test pins the oracle to
something other than itself: a library routine, a closed form, exact
arithmetic, a textbook limit, an independent algorithm or an invariant
(DESIGN.md "Oracle pins").  Citations are PAPER.md v2 lines."""
import itertools
import math

import mpmath
import numpy as np
import pytest

import oracle
import phantom
from tests import _pins

QS = [0.5, 0.8, 1.0, 1.2, 1.5]


def rng_hist(rng, L, zero_frac=0.3, hi=50):
    h = rng.integers(1, hi, size=L)
    h[rng.random(L) < zero_frac] = 0
    return h.astype(np.uint32)


@pytest.fixture(scope="module")
def ct_slices():
    cfg = phantom.CONFIGS["c2"]
    return phantom.make_volume(cfg, nz=4, z_first=110)


# ---------------------------------------------------------------- histogram
def test_histogram_matches_bincount(ct_slices):
    """per-slice brightness histogram == numpy.bincount."""
    for s in ct_slices:
        h, st = oracle.histogram(s, 256)
        assert st == oracle.OK
        np.testing.assert_array_equal(h, np.bincount(s.ravel(), minlength=256))
        assert int(h.sum()) == s.size


def test_histogram_u16_and_overflow():
    rng = np.random.default_rng(1)
    s = rng.integers(0, 4096, size=(64, 64)).astype(np.uint16)
    h, st = oracle.histogram(s, 4096)
    assert st == oracle.OK
    np.testing.assert_array_equal(h, np.bincount(s.ravel(), minlength=4096))
    s[3, 5] = 4096  # one voxel >= bins: LEVEL_OVERFLOW, never clamped (R13)
    h, st = oracle.histogram(s, 4096)
    assert st == oracle.LEVEL_OVERFLOW
    assert int(h.sum()) == s.size - 1


# ----------------------------------------------------------- class entropy
@pytest.mark.parametrize("q", QS + [0.3, 2.0, 3.0])
def test_class_entropy_closed_forms(q):
    """PAPER.md:581-585.  A single-bin class has S = 0 exactly; a uniform m-bin
    class has S = (1 - m^(1-q)) / (q - 1) (Shannon: ln m)."""
    L = 64
    p = np.zeros(L)
    p[10] = 0.25
    p[20:28] = 0.75 / 8
    assert oracle.class_entropy(p, 5, 15, q) == 0.0
    assert oracle.class_entropy(p, 30, 40, q) is None  # empty class
    s = oracle.class_entropy(p, 16, 31, q)  # uniform over 8 non-empty bins
    m = mpmath.mpf(8)
    ref = mpmath.log(m) if q == 1.0 else (1 - m ** (1 - mpmath.mpf(q))) / (mpmath.mpf(q) - 1)
    assert abs(s - float(ref)) <= 1e-14 * abs(float(ref))


# --------------------------------------------------- uniform closed forms
@pytest.mark.parametrize("q", [0.8, 1.2, 0.5, 1.5])
def test_uniform_histogram_k1(q):
    """Uniform L=256, k=1: t* = 127 and phi = (128^(2(1-q)) - 1)/(1 - q)
    (composition of two uniform 128-bin classes)."""
    r = oracle.search(np.full(256, 1000), 1, q)
    assert r["status"] == 0 and r["t"] == (127,)
    ref = (mpmath.mpf(128) ** (2 * (1 - mpmath.mpf(q))) - 1) / (1 - mpmath.mpf(q))
    assert abs(r["phi"] - float(ref)) <= 1e-13 * float(ref)
    if q == 0.8:
        assert abs(r["phi"] - 29.822022531844958) <= 1e-13 * 29.8


@pytest.mark.parametrize("q", [0.8, 1.2, 1.0])
def test_uniform_histogram_k3(q):
    """Uniform L=256, k=3: t* = (63,127,191), phi = (64^(4(1-q)) - 1)/(1-q);
    q = 1: 4 ln 64."""
    r = oracle.search(np.full(256, 7), 3, q)
    assert r["t"] == (63, 127, 191)
    if q == 1.0:
        ref = 4 * mpmath.log(64)
    else:
        ref = (mpmath.mpf(64) ** (4 * (1 - mpmath.mpf(q))) - 1) / (1 - mpmath.mpf(q))
    assert abs(r["phi"] - float(ref)) <= 1e-13 * float(ref)


# ------------------------------------------------ exact rationals at q = 2
@pytest.mark.parametrize("seed", range(12))
def test_q2_exact_rationals(seed):
    """q = 2: A_j = sum c^2 / n_j^2 is rational, so Fraction arithmetic gives the
    exact argmax, tie set and objective (composition identity, not the fold)."""
    rng = np.random.default_rng(100 + seed)
    L = int(rng.integers(5, 12))
    k = int(rng.integers(1, 4))
    h = rng_hist(rng, L, zero_frac=0.25, hi=9)
    if (h > 0).sum() < k + 1:
        h[: k + 1] = 1
    best, tstar, vals = _pins.exhaustive(h, k, _pins.frac_phi_q2)
    r = oracle.search(h, k, 2.0)
    assert r["status"] == 0
    exact_ties = {t for t, v in vals.items() if v == best}
    if tstar == r["t"]:
        pass
    else:  # only a mathematically exact tie between distinct partitions may differ
        assert r["t"] in exact_ties
    assert abs(r["phi"] - float(best)) <= 1e-14 * max(1.0, abs(float(best)))
    for t in list(vals)[:40]:
        v = oracle.phi_at(h, k, 2.0, t)
        assert abs(v - float(vals[t])) <= 1e-14 * max(1.0, abs(float(vals[t])))


# ------------------------------------- brute force in 50-digit arithmetic
@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("objective", [0, 1])
def test_bruteforce_mpmath(seed, objective):
    """Tiny random histograms with zeros, L <= 12, k <= 4, all q: oracle argmax
    equals the 50-digit argmax unless the distinct-partition gap < 1e-12, and
    phi agrees to 1e-13."""
    rng = np.random.default_rng(seed)
    L = int(rng.integers(4, 13))
    k = int(rng.integers(1, min(4, L - 1) + 1))
    q = [0.5, 0.8, 1.0, 1.2, 1.5, 2.5][seed % 6]
    h = rng_hist(rng, L, zero_frac=0.3, hi=40)
    best, tstar, vals = _pins.exhaustive(h, k, lambda hh, t: _pins.mp_phi(hh, t, q, objective))
    r = oracle.search(h, k, q, objective=objective)
    if best is None:
        assert r["status"] == oracle.NO_VALID_SPLIT
        return
    gap = _pins.distinct_gap(h, vals, tstar)
    if gap >= 1e-12:
        assert r["t"] == tstar, (r, tstar, float(gap))
    else:
        assert vals[r["t"]] >= best - abs(best) * 1e-12
    assert abs(r["phi"] - float(best)) <= 1e-13 * max(1.0, abs(float(best)))
    # oracle's own gap report agrees with the high-precision one
    if gap != mpmath.inf and gap > 1e-10:
        assert abs(r["gap"] - float(gap)) <= 1e-6 * float(gap) + 1e-13


@pytest.mark.parametrize("seed", range(10))
def test_level0_equals_level1_bitexact(seed):
    """Level 1 (memoised by class content) is bit-identical to Level 0."""
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.integers(6, 17))
    k = int(rng.integers(1, 5))
    h = rng_hist(rng, L, zero_frac=0.35, hi=1000)
    for q in (0.7, 1.0, 1.3):
        for obj in (0, 1):
            a = oracle.search(h, k, q, objective=obj, level=0)
            b = oracle.search(h, k, q, objective=obj, level=1)
            assert a["t"] == b["t"] and a["status"] == b["status"]
            if a["status"] == 0:
                assert a["phi"] == b["phi"] and a["gap"] == b["gap"]
                assert a["tuples_valid"] == b["tuples_valid"]


# ------------------------------------------------------ textbook: Kapur
def test_kapur_closed_form_q1(ct_slices):
    """q = 1, k = 1 is Kapur-Sahoo-Wong maximum-entropy thresholding."""
    h = np.bincount(ct_slices[0].ravel(), minlength=256)
    nzb = np.nonzero(h)[0]
    vals = {}
    for t in range(255):
        v = _pins.kapur_k1(h, t)
        if v is None:
            continue
        vals[t] = v
        o = oracle.phi_at(h, 1, 1.0, (t,))
        assert abs(o - float(v)) <= 1e-13 * float(v)
    best = max(vals.values())
    tstar = min(t for t, v in vals.items() if v == best)
    r = oracle.search(h, 1, 1.0)
    assert r["t"] == (int(nzb[nzb <= tstar].max()),) or r["t"] == (tstar,)


# ------------------------------------------------------- special cases
def test_point_masses():
    """Two equal point masses at 40/200: every t in [40,199]
    gives phi = 0 and the lowest wins; exactly k+1 non-empty bins give the unique
    partition; <= k non-empty bins give NO_VALID_SPLIT."""
    h = np.zeros(256, np.uint32)
    h[40] = h[200] = 5000
    for q in QS:
        r = oracle.search(h, 1, q)
        assert r["t"] == (40,) and r["phi"] == 0.0
    h = np.zeros(256, np.uint32)
    h[[10, 90, 91, 250]] = [7, 3, 11, 2]
    r = oracle.search(h, 3, 0.8)
    assert r["t"] == (10, 90, 91) and r["phi"] == 0.0 and r["gap"] == math.inf
    r = oracle.search(h, 4, 0.8)
    assert r["status"] == oracle.NO_VALID_SPLIT
    h = np.zeros(256, np.uint32)
    h[17] = 100
    assert oracle.search(h, 1, 0.8)["status"] == oracle.NO_VALID_SPLIT
    assert oracle.search(np.zeros(256, np.uint32), 1, 0.8)["status"] == oracle.NO_VALID_SPLIT


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("q", [0.5, 0.7, 0.8, 1.0, 1.2, 1.5])
def test_gap_phantoms(k, q):
    """k+1 equal-mass, equal-width uniform clusters separated by empty gaps:
    prod A_j = (prod m_j)^(1-q) is optimised only by the equal split, i.e. by
    t_j = last bin of cluster j (checks the class-boundary convention R4 and
    the direction of the argmax for q < 1, q = 1 and q > 1)."""
    L, w = 256, 16
    starts = np.linspace(8, L - w - 8, k + 1).astype(int)
    h = np.zeros(L, np.uint32)
    for s in starts:
        h[s:s + w] = 37
    r = oracle.search(h, k, q)
    assert r["t"] == tuple(int(s + w - 1) for s in starts[:-1])
    assert r["gap"] > 1e-6


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("k", [1, 2, 3])
def test_mirror_symmetry(seed, k):
    """h[i] = h[L-1-i]  =>  phi(mirror(t*)) = phi(t*) with
    mirror(t)_j = L-2-t_{k+1-j}; which of the two is chosen is an fp near-tie."""
    rng = np.random.default_rng(seed)
    L = 64
    half = rng_hist(rng, L // 2, zero_frac=0.2, hi=200)
    h = np.concatenate([half, half[::-1]])
    for q in (0.6, 1.0, 1.4):
        r = oracle.search(h, k, q)
        m = tuple(sorted(L - 2 - x for x in r["t"]))
        pm = oracle.phi_at(h, k, q, m)
        assert abs(pm - r["phi"]) <= 1e-12 * r["phi"]


@pytest.mark.parametrize("q", QS)
def test_scale_invariance(ct_slices, q):
    """Counts x 7 leave the partition unchanged, absent near-ties."""
    h = np.bincount(ct_slices[1].ravel(), minlength=256)
    for k in (1, 2):
        a = oracle.search(h, k, q)
        b = oracle.search(h * 7, k, q)
        if a["gap"] > 1e-9:
            assert a["t"] == b["t"]
            assert abs(a["phi"] - b["phi"]) <= 1e-12 * a["phi"]


@pytest.mark.parametrize("q", QS)
@pytest.mark.parametrize("k", [1, 2, 3])
def test_dp_independent_algorithm(ct_slices, q, k):
    """A log-domain DP over class intervals finds the same partition as the
    exhaustive oracle (absent near-ties)."""
    h = np.bincount(ct_slices[2].ravel(), minlength=256)
    r = oracle.search(h, k, q)
    t_dp, _ = _pins.dp_argmax(h, k, q)
    if r["gap"] > 1e-9:
        assert r["t"] == t_dp


def test_q_to_one_continuity(ct_slices):
    """t*(q = 1 +- 1e-6) = t*(q = 1) when the gap is large (Shannon limit, R6)."""
    h = np.bincount(ct_slices[3].ravel(), minlength=256)
    for k in (1, 2):
        r1 = oracle.search(h, k, 1.0)
        assert r1["gap"] > 1e-6
        for q in (1 - 1e-6, 1 + 1e-6):
            assert oracle.search(h, k, q)["t"] == r1["t"]


def test_canonical_runner_up_and_tstar(ct_slices):
    """t* is canonical (every t_j a non-empty bin), the runner-up is a different
    partition, and phi2 <= phi*."""
    h = np.bincount(ct_slices[0].ravel(), minlength=256)
    for k in (1, 2, 3):
        r = oracle.search(h, k, 0.8)
        assert all(h[x] > 0 for x in r["t"])
        assert r["t2"] != r["t"] and r["phi2"] <= r["phi"]
        assert r["phi2"] == oracle.phi_at(h, k, 0.8, r["t2"])


# ------------------------------------------------------------- labels
def test_labels_counts_and_algorithm1(ct_slices):
    """label = #{j : v > t_j}: count of label j == n_j from the histogram at t*;
    k = 1 is Algorithm 1 ('>= T') with T = t + 1."""
    s = ct_slices[0]
    h = np.bincount(s.ravel(), minlength=256)
    for k in (1, 2, 3):
        r = oracle.search(h, k, 0.8)
        lab = oracle.label(s, k, r["t"])
        bounds = _pins.classes(r["t"], 256)
        for j, (a, b) in enumerate(bounds):
            assert int((lab == j).sum()) == int(h[a:b + 1].sum())
        if k == 1:
            np.testing.assert_array_equal(lab, (s >= r["t"][0] + 1).astype(np.uint8))


def test_segment_matches_per_slice_calls(ct_slices):
    out = oracle.segment(ct_slices, 256, 2, 0.8, threads=2)
    for z, s in enumerate(ct_slices):
        r = oracle.search(np.bincount(s.ravel(), minlength=256), 2, 0.8)
        assert tuple(out["thresholds"][z]) == r["t"]
        assert out["phi"][z] == r["phi"] and out["gap"][z] == r["gap"]
        np.testing.assert_array_equal(out["labels"][z], oracle.label(s, 2, r["t"]))
    # thread count does not change results
    out1 = oracle.segment(ct_slices, 256, 2, 0.8, threads=1)
    np.testing.assert_array_equal(out1["thresholds"], out["thresholds"])
    np.testing.assert_array_equal(out1["phi"], out["phi"])


def test_sum_plus_product_k1_equals_fold():
    """For two classes both objectives are the paper's H1 + H2 + (1-a) H1 H2."""
    rng = np.random.default_rng(5)
    h = rng_hist(rng, 40, hi=300)
    for q in (0.6, 1.4):
        a = oracle.search(h, 1, q, objective=0)
        b = oracle.search(h, 1, q, objective=1)
        assert a["t"] == b["t"]
        assert abs(a["phi"] - b["phi"]) <= 1e-14 * a["phi"]
