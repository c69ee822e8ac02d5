"""CPU oracle for the Tsallis multilevel-thresholding hot path (arXiv 2012.10684).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs, never by the product
package.  Thin ctypes wrapper over ``tsallis_oracle.c`` (which documents every
step with its PAPER.md citation); shares nothing with the CUDA path.

Parity pins: every function here is pinned by tests/test_oracle_*.py against
closed forms, exact rationals, textbook limits, brute force and invariants (see
DESIGN.md "Oracle pins").  ``phi_at``/``search`` on the paper's own (private)
data are "parity unpinned": the paper prints no threshold or objective values.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "tsallis_oracle.c")

OK, INVALID_ARG, LEVEL_OVERFLOW, NO_VALID_SPLIT = 0, 1, 2, 3
PSEUDO_ADDITIVE, SUM_PLUS_PRODUCT = 0, 1
KMAX = 4
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


class _Result(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("t", ctypes.c_int32 * KMAX),
        ("phi", ctypes.c_double),
        ("has_runner_up", ctypes.c_int32),
        ("t2", ctypes.c_int32 * KMAX),
        ("phi2", ctypes.c_double),
        ("gap", ctypes.c_double),
        ("tuples_valid", ctypes.c_int64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        lib.oracle_histogram.restype = I
        lib.oracle_histogram.argtypes = [P, I, I64, I, P]
        lib.oracle_class_entropy.restype = D
        lib.oracle_class_entropy.argtypes = [P, I, I, D, ctypes.POINTER(I)]
        lib.oracle_phi_at.restype = D
        lib.oracle_phi_at.argtypes = [P, I, I, D, I, P, ctypes.POINTER(I)]
        lib.oracle_search.restype = I
        lib.oracle_search.argtypes = [P, I, I, D, I, I, ctypes.POINTER(_Result)]
        lib.oracle_label.restype = None
        lib.oracle_label.argtypes = [P, I, I64, I, P, P]
        lib.oracle_segment.restype = I
        lib.oracle_segment.argtypes = [P, I, I64, I64, I64, I64, I64, I, I, D, I, I, I,
                                       P, P, P, P, P, P]
        lib.oracle_max_threads.restype = I
        lib.oracle_mean3x3.restype = None
        lib.oracle_mean3x3.argtypes = [P, I64, I64, P]
        lib.oracle_hist2d.restype = I
        lib.oracle_hist2d.argtypes = [P, I64, I64, I, P]
        lib.oracle_phi2d_at.restype = D
        lib.oracle_phi2d_at.argtypes = [P, I, D, I, I, ctypes.POINTER(I)]
        lib.oracle_erode.restype = None
        lib.oracle_erode.argtypes = [P, I64, I64, I, P]
        lib.oracle_dilate.restype = None
        lib.oracle_dilate.argtypes = [P, I64, I64, I, P]
        lib.oracle_tophat.restype = None
        lib.oracle_tophat.argtypes = [P, I64, I64, I, P, P]
        lib.oracle_preprocess.restype = None
        lib.oracle_preprocess.argtypes = [P, I64, I, P, P, P]
        lib.oracle_search2d_n.restype = I
        lib.oracle_search2d_n.argtypes = [P, I, D, I, P, P, P, P]
        _lib = lib
    return _lib


def _u32(h):
    h = np.ascontiguousarray(h, dtype=np.uint32)
    return h


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def histogram(slice_, bins):
    """(hist u32[bins], status) of one slice (any shape)."""
    a = np.ascontiguousarray(slice_)
    h = np.zeros(bins, np.uint32)
    st = _load().oracle_histogram(a.ctypes.data, a.dtype.itemsize, a.size, bins, h.ctypes.data)
    return h, int(st)


def class_entropy(p, a, b, q):
    """S of class [a,b] from probabilities p (None if the class is empty)."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    v = ctypes.c_int(0)
    s = _load().oracle_class_entropy(p.ctypes.data, a, b, q, ctypes.byref(v))
    return s if v.value else None


def phi_at(hist, k, q, t, objective=PSEUDO_ADDITIVE):
    """Objective at tuple t from the definition (None if invalid)."""
    h = _u32(hist)
    tt = np.ascontiguousarray(t, dtype=np.int32)
    assert tt.size == k
    v = ctypes.c_int(0)
    r = _load().oracle_phi_at(h.ctypes.data, h.size, k, q, objective, tt.ctypes.data,
                              ctypes.byref(v))
    return r if v.value else None


def search(hist, k, q, objective=PSEUDO_ADDITIVE, level=1):
    """Exhaustive argmax.  Returns dict(status, t, phi, t2, phi2, gap, tuples_valid)."""
    h = _u32(hist)
    r = _Result()
    _load().oracle_search(h.ctypes.data, h.size, k, q, objective, level, ctypes.byref(r))
    return {
        "status": int(r.status),
        "t": tuple(int(x) for x in r.t[:k]),
        "phi": float(r.phi),
        "t2": tuple(int(x) for x in r.t2[:k]) if r.has_runner_up else None,
        "phi2": float(r.phi2) if r.has_runner_up else None,
        "gap": float(r.gap),
        "tuples_valid": int(r.tuples_valid),
    }


def label(slice_, k, t):
    a = np.ascontiguousarray(slice_)
    tt = np.ascontiguousarray(t, dtype=np.int32)
    out = np.empty(a.shape, np.uint8)
    _load().oracle_label(a.ctypes.data, a.dtype.itemsize, a.size, k, tt.ctypes.data,
                         out.ctypes.data)
    return out


def segment(vol, bins, k, q, objective=PSEUDO_ADDITIVE, level=1, z0=0, z1=None,
            threads=None, labels=True):
    """Whole path for slices [z0, z1) of vol[nz][ny][nx].  Arrays are indexed by
    absolute slice; entries outside [z0, z1) are left zero/NaN."""
    v = np.ascontiguousarray(vol)
    nz, ny, nx = v.shape
    z1 = nz if z1 is None else z1
    hist = np.zeros((nz, bins), np.uint32)
    thr = np.full((nz, k), -1, np.int32)
    phi = np.full(nz, np.nan)
    gap = np.full(nz, np.nan)
    status = np.full(nz, -1, np.int32)
    lab = np.zeros(v.shape, np.uint8) if labels else None
    threads = threads or max_threads()
    _load().oracle_segment(v.ctypes.data, v.dtype.itemsize, nx, ny, nz, z0, z1, bins, k, q,
                           objective, level, threads, hist.ctypes.data, thr.ctypes.data,
                           phi.ctypes.data, gap.ctypes.data, status.ctypes.data,
                           lab.ctypes.data if labels else None)
    return {"hist": hist, "thresholds": thr, "phi": phi, "gap": gap, "status": status,
            "labels": lab}


# ---------------------------------------------------------------- 2-D (f1)
def mean3x3(slice_u8):
    """3x3 floor mean with replicate border (R18/R19)."""
    f = np.ascontiguousarray(slice_u8, dtype=np.uint8)
    g = np.empty_like(f)
    _load().oracle_mean3x3(f.ctypes.data, f.shape[1], f.shape[0], g.ctypes.data)
    return g


def hist2d(slice_u8, bins):
    """(h [bins][bins] u32 with h[i][j] = #{f=i, g=j}, status)."""
    f = np.ascontiguousarray(slice_u8, dtype=np.uint8)
    h = np.zeros((bins, bins), np.uint32)
    st = _load().oracle_hist2d(f.ctypes.data, f.shape[1], f.shape[0], bins, h.ctypes.data)
    return h, int(st)


def phi2d_at(h, q, t, s):
    h = np.ascontiguousarray(h, dtype=np.uint32)
    v = ctypes.c_int(0)
    r = _load().oracle_phi2d_at(h.ctypes.data, h.shape[0], q, t, s, ctypes.byref(v))
    return r if v.value else None


def search2d(h, q, threads=1):
    """Exhaustive Level-0 2-D argmax (O(L^4); rows of candidates on `threads`
    OpenMP threads -- the result does not depend on the thread count).
    Returns dict(status, t, s, phi, gap); gap is over distinct partitions."""
    h = np.ascontiguousarray(h, dtype=np.uint32)
    t = np.zeros(1, np.int32)
    s = np.zeros(1, np.int32)
    phi = np.zeros(1)
    gap = np.zeros(1)
    st = _load().oracle_search2d_n(h.ctypes.data, h.shape[0], q, int(threads), t.ctypes.data,
                                    s.ctypes.data, phi.ctypes.data, gap.ctypes.data)
    return {"status": int(st), "t": int(t[0]), "s": int(s[0]), "phi": float(phi[0]),
            "gap": float(gap[0])}


def segment2d(vol, bins, q, z_list=None, threads=None, labels=True):
    """2-D path for the slices in z_list (default all) of a u8 vol[nz][ny][nx]:
    hist2d -> search2d -> labels = f > t ("only t is used").
    Arrays are indexed by absolute slice; slices not in z_list stay -1/NaN/0."""
    v = np.ascontiguousarray(vol, dtype=np.uint8)
    nz = v.shape[0]
    z_list = range(nz) if z_list is None else z_list
    threads = threads or max_threads()
    hist = np.zeros((nz, bins, bins), np.uint32)
    thr = np.full((nz, 2), -1, np.int32)
    phi = np.full(nz, np.nan)
    gap = np.full(nz, np.nan)
    status = np.full(nz, -1, np.int32)
    lab = np.zeros(v.shape, np.uint8) if labels else None
    for z in z_list:
        h, st = hist2d(v[z], bins)
        hist[z] = h
        if st == OK:
            r = search2d(h, q, threads)
            st = r["status"]
            if st == OK:
                thr[z] = (r["t"], r["s"])
                phi[z] = r["phi"]
                gap[z] = r["gap"]
                if labels:
                    lab[z] = label(v[z], 1, (r["t"],))
        status[z] = st
    return {"hist": hist, "thresholds": thr, "phi": phi, "gap": gap, "status": status,
            "labels": lab}


# -------------------------------------------------------- pre-processing (f2)
def preprocess(vol_i16, background=-2000):
    """HU int16 volume -> (u8 volume, lo, hi): PAPER.md:514-516 with the
    volume-wide window of DESIGN.md R23-R25."""
    v = np.ascontiguousarray(vol_i16, dtype=np.int16)
    out = np.empty(v.shape, np.uint8)
    lo = np.zeros(1, np.int32)
    hi = np.zeros(1, np.int32)
    _load().oracle_preprocess(v.ctypes.data, v.size, int(background), out.ctypes.data,
                              lo.ctypes.data, hi.ctypes.data)
    return out, int(lo[0]), int(hi[0])


# ------------------------------------------------------------ morphology (f3)
def _slicewise(fn, a, r):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    two = a.ndim == 2
    a3 = a[None] if two else a
    out = np.empty_like(a3)
    for z in range(a3.shape[0]):
        fn(a3[z].ctypes.data, a3.shape[2], a3.shape[1], int(r), out[z].ctypes.data)
    return out[0] if two else out


def erode(a, r):
    """Grayscale erosion by disk(r), outside = 255 (R26-R27)."""
    return _slicewise(_load().oracle_erode, a, r)


def dilate(a, r):
    """Grayscale dilation by disk(r), outside = 0 (R26-R27)."""
    return _slicewise(_load().oracle_dilate, a, r)


def tophat(a, r):
    """(opening, white top-hat) of every slice (R28)."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    two = a.ndim == 2
    a3 = a[None] if two else a
    op = np.empty_like(a3)
    th = np.empty_like(a3)
    for z in range(a3.shape[0]):
        _load().oracle_tophat(a3[z].ctypes.data, a3.shape[2], a3.shape[1], int(r),
                              op[z].ctypes.data, th[z].ctypes.data)
    return (op[0], th[0]) if two else (op, th)
