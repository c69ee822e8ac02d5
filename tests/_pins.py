"""Independent references used to pin the oracle (and, through it, the CUDA
path).  Nothing here calls oracle/ or the CUDA package.

* ``mp_phi``: the objective from the Tsallis *composition* identity
  phi = (prod_j A_j - 1) / (1 - q),  A_j = sum_{i in C_j} (c_i / n_j)^q
  (pseudo-additive), in mpmath at 50 digits -- a different formula for the same
  quantity the oracle folds left to right, so a dropped term,
  wrong sign or wrong index in the oracle's fold shows up here.
  q == 1: sum_j (ln n_j - (1/n_j) sum c ln c)  (Shannon / Kapur, R6).
* ``frac_phi_q2``: the same identity at q = 2 in exact rationals.
* ``kapur_k1``: Kapur-Sahoo-Wong closed form for k = 1, q = 1.
* ``dp_argmax``: log-domain dynamic programme over class intervals (an
  independent exact algorithm for the pseudo-additive objective).
* ``accept``: BASELINE.json:north_star acceptance rule.
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import mpmath
import numpy as np

mpmath.mp.dps = 50

PSEUDO_ADDITIVE, SUM_PLUS_PRODUCT = 0, 1


def classes(t, L):
    lo = [0] + [x + 1 for x in t]
    hi = list(t) + [L - 1]
    return list(zip(lo, hi))


def tuples(L, k):
    return itertools.combinations(range(L - 1), k)


def mp_phi(hist, t, q, objective=PSEUDO_ADDITIVE):
    """High-precision objective at t, or None if some class is empty."""
    c = [int(x) for x in hist]
    L = len(c)
    q = mpmath.mpf(q)
    A, S = [], []
    for a, b in classes(t, L):
        n = sum(c[a:b + 1])
        if n == 0:
            return None
        if q == 1:
            s = mpmath.log(n) - sum(mpmath.mpf(x) * mpmath.log(x) for x in c[a:b + 1] if x) / n
            S.append(s)
            A.append(None)
        else:
            a_j = sum((mpmath.mpf(x) / n) ** q for x in c[a:b + 1] if x)
            A.append(a_j)
            S.append((1 - a_j) / (q - 1))
    if objective == SUM_PLUS_PRODUCT:
        prod = mpmath.mpf(1)
        for s in S:
            prod *= s
        return sum(S) + (1 - q) * prod
    if q == 1:
        return sum(S)
    prod = mpmath.mpf(1)
    for a_j in A:
        prod *= a_j
    return (prod - 1) / (1 - q)


def frac_phi_q2(hist, t):
    """Exact rational pseudo-additive objective at q = 2: phi = 1 - prod A_j."""
    c = [int(x) for x in hist]
    prod = Fraction(1)
    for a, b in classes(t, len(c)):
        n = sum(c[a:b + 1])
        if n == 0:
            return None
        prod *= Fraction(sum(x * x for x in c[a:b + 1]), n * n)
    return 1 - prod


def exhaustive(hist, k, value_fn):
    """(best value, lowest tuple among exact maxima, all values dict)."""
    L = len(hist)
    vals = {}
    for t in tuples(L, k):
        v = value_fn(hist, t)
        if v is not None:
            vals[t] = v
    if not vals:
        return None, None, vals
    best = max(vals.values())
    tstar = min(t for t, v in vals.items() if v == best)
    return best, tstar, vals


def canonical(hist, t):
    """Lowest tuple giving the same partition: each t_j -> last non-empty bin <= t_j."""
    out = []
    for x in t:
        y = x
        while y > 0 and hist[y] == 0:
            y -= 1
        out.append(y)
    return tuple(out)


def distinct_gap(hist, vals, tstar):
    """Relative gap between the best value and the best *different partition*."""
    best = vals[tstar]
    others = [v for t, v in vals.items() if canonical(hist, t) != canonical(hist, tstar)]
    if not others:
        return mpmath.inf
    second = max(others)
    if best == 0:
        return mpmath.inf if second != 0 else 0
    return (best - second) / abs(best)


def kapur_k1(hist, t):
    """Kapur, Sahoo & Wong (1985): psi(t) = ln(P_t (1-P_t)) + H_t/P_t + (H_n-H_t)/(1-P_t)."""
    c = [mpmath.mpf(int(x)) for x in hist]
    N = sum(c)
    p = [x / N for x in c]
    Pt = sum(p[: t + 1])
    if Pt == 0 or Pt == 1:
        return None
    Ht = -sum(x * mpmath.log(x) for x in p[: t + 1] if x)
    Hn = -sum(x * mpmath.log(x) for x in p if x)
    return mpmath.log(Pt * (1 - Pt)) + Ht / Pt + (Hn - Ht) / (1 - Pt)


def dp_argmax(hist, k, q):
    """Log-domain DP for the pseudo-additive objective (independent algorithm).

    Maximises sum_j g(C_j) with g = sign * ln A_j (q != 1; sign +1 for q < 1,
    -1 for q > 1 since phi = (prod A - 1)/(1 - q)) or g = S_j (q == 1).
    Returns the canonical tuple of one optimum."""
    c = np.asarray(hist, dtype=np.float64)
    L = c.size
    NEG = -np.inf
    g = np.full((L, L), NEG)
    for a in range(L):
        seg = c[a:]
        n = np.cumsum(seg)
        if q == 1.0:
            clc = np.cumsum(np.where(seg > 0, seg * np.log(np.where(seg > 0, seg, 1)), 0.0))
            with np.errstate(divide="ignore", invalid="ignore"):
                val = np.log(n) - clc / n
        else:
            w = np.cumsum(np.where(seg > 0, seg ** q, 0.0))
            with np.errstate(divide="ignore", invalid="ignore"):
                val = np.log(w) - q * np.log(n)
            val = val if q < 1 else -val
        val = np.where(n > 0, val, NEG)
        g[a, a:] = val
    # best[j][b]: best score of splitting [0, b] into j+1 classes
    best = np.full((k + 1, L), NEG)
    arg = np.zeros((k + 1, L), dtype=np.int64)
    best[0] = g[0]
    for j in range(1, k + 1):
        for b in range(j, L):
            cand = best[j - 1][: b] + g[1: b + 1, b]  # previous class ends at a-1 = 0..b-1
            a = int(np.argmax(cand))
            best[j][b] = cand[a]
            arg[j][b] = a  # previous class ends at a
    t = []
    b = L - 1
    for j in range(k, 0, -1):
        a = int(arg[j][b])
        t.append(a)
        b = a
    t = tuple(reversed(t))
    return canonical(hist, t), float(best[k][L - 1])


def accept(hist, k, q, t_test, ref, objective=PSEUDO_ADDITIVE, rel=1e-12, phi_fn=None):
    """North-star acceptance rule.  ref: oracle.search() dict.  phi_fn(hist, t)
    evaluates the oracle objective at another tuple (for the near-tie clause).
    Returns (ok, reason)."""
    t_test = tuple(int(x) for x in t_test)
    if t_test == tuple(ref["t"]):
        return True, "exact"
    gap = ref["gap"]
    if gap is not None and gap >= rel:
        return False, f"threshold mismatch {t_test} vs {ref['t']} with gap {gap:.3e}"
    v = phi_fn(hist, t_test)
    if v is None:
        return False, f"{t_test} is not a valid tuple"
    if v >= ref["phi"] * (1 - rel) - (rel if ref["phi"] == 0 else 0):
        return True, "near-tie"
    return False, f"near-tie member check failed {v} < {ref['phi']}"
