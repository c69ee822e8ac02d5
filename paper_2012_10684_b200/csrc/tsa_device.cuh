// tsa_device.cuh -- device-side helpers shared by the libtsa kernels (sm_100a).
//
// Arithmetic rules: every quantity that can
// decide an argmax is computed with explicit __dadd_rn/__dsub_rn/__dmul_rn so
// nvcc cannot contract or re-associate it; the same device function produces a
// class term wherever it is needed (tables, on-the-fly search), so a tuple's
// value is a pure function of the tuple, identical across kernels, launch
// configurations, unit partitions and GPUs.
#pragma once
#include <cstdint>
#include <math_constants.h>

namespace tsa {

constexpr int kKMax = 4;
constexpr uint64_t kKeyNone = 0xFFFFFFFFFFFFFFFFull;

// status values (mirror tsa_status in include/tsa.h)
constexpr int kOK = 0, kLevelOverflow = 2, kNoValidSplit = 3;

// ---------------------------------------------------------------- dd helpers
// Double-double (unevaluated sum hi + lo) prefix sums keep every class sum
// accurate to ~1 ulp after the prefix difference (plain fp64
// prefix differences lose up to 9e-10 relative).
struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double e = __dsub_rn(b, __dsub_rn(s, a));
  return {s, e};
}

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  dd s = two_sum(a.hi, b);
  s.lo = __dadd_rn(s.lo, a.lo);
  return fast_two_sum(s.hi, s.lo);
}

// (b - a) rounded to double: exact hi difference whenever the two prefixes are
// close (Sterbenz), otherwise the lost bits are < 1/2 ulp of the result.
__device__ __forceinline__ double dd_diff(double bhi, double blo, double ahi, double alo) {
  return __dadd_rn(__dsub_rn(bhi, ahi), __dsub_rn(blo, alo));
}

// --------------------------------------------------------------- term modes
// PROD_MAX / PROD_MIN: pseudo-additive, q != 1: score = +/- prod_j A_j, since
//   phi = (prod_j A_j - 1)/(1 - q) (Tsallis composition, R1) is
//   increasing in prod A for q < 1 and decreasing for q > 1.
// SUM: pseudo-additive at q == 1: score = sum_j S_j (Shannon/Kapur, R6).
// SPP: sum-plus-product objective, score = phi itself.
enum Mode { PROD_MAX = 0, PROD_MIN = 1, SUM = 2, SPP = 3 };

// Per-slice tables, entry e = position + 1, entry 0 = sentinel (C = 0, W = 0).
struct SliceTables {
  const uint32_t *C;   // inclusive prefix counts
  const double *Whi;   // dd inclusive prefix of w_i = c_i^q (or c_i ln c_i at q == 1)
  const double *Wlo;
  const double *Asuf;  // Asuf[i] = T(i+1, M-1), i in [0, M-2]
};

struct Luts {
  const double *ipow;  // ipow[n] = 1 / n^q, ipow[0] = NaN   (q != 1)
  const double *lnn;   // lnn[n] = ln n, lnn[0] = NaN        (q == 1)
  const double *rcp;   // rcp[n] = 1 / n                     (q == 1)
  double iqm1;         // 1 / (q - 1)
  double omq;          // 1 - q
  int shannon;         // q == 1
};

// Class term T(a, b) of the class made of table positions [a, b]:
//   q != 1, pseudo-additive: A = W / n^q = sum_{i in C} (c_i / n)^q
//   q == 1:                  S = ln n - (sum c ln c) / n
//   sum-plus-product:        S = (1 - A) / (q - 1)  (or the q == 1 S)
// An empty class (n == 0, FULL enumeration only) yields NaN, which never wins a
// comparison, so invalid tuples are skipped without a branch.
template <int MODE>
__device__ __forceinline__ double class_term(const SliceTables &t, const Luts &l, int a, int b) {
  // generic loads: the tables may be staged in shared memory
  const uint32_t n = t.C[b + 1] - t.C[a];
  const double w = dd_diff(t.Whi[b + 1], t.Wlo[b + 1], t.Whi[a], t.Wlo[a]);
  if (MODE == PROD_MAX || MODE == PROD_MIN) {
    return __dmul_rn(w, __ldg(l.ipow + n));
  } else if (MODE == SUM) {
    return __dsub_rn(__ldg(l.lnn + n), __dmul_rn(w, __ldg(l.rcp + n)));
  } else {
    if (l.shannon) return __dsub_rn(__ldg(l.lnn + n), __dmul_rn(w, __ldg(l.rcp + n)));
    const double A = __dmul_rn(w, __ldg(l.ipow + n));
    return __dmul_rn(__dsub_rn(1.0, A), l.iqm1);
  }
}

template <int MODE>
__device__ __forceinline__ double combine(double x, double y) {
  if (MODE == SUM) return __dadd_rn(x, y);
  return __dmul_rn(x, y);
}

// ------------------------------------------------------------- binomials
__device__ __forceinline__ uint64_t binom(uint64_t n, int r) {
  if (r == 0) return 1;
  if (n < (uint64_t)r) return 0;
  if (r == 1) return n;
  if (r == 2) return n * (n - 1) / 2;
  if (r == 3) return n * (n - 1) / 2 * (n - 2) / 3;  // n(n-1)/2 is exact; times (n-2) divisible by 3 jointly
  // r == 4
  return binom(n, 3) * (n - 3) / 4;
}

// Unrank lex rank r among R-combinations of [0, P): idx[0] < ... < idx[R-1].
template <int R>
__device__ __forceinline__ void unrank_comb(uint64_t r, int P, int *idx) {
  int x = 0;
#pragma unroll
  for (int j = 0; j < R; j++) {
    const int rem = R - 1 - j;
    for (;;) {
      const uint64_t cnt = binom((uint64_t)(P - 1 - x), rem);
      if (r < cnt) {
        idx[j] = x;
        x++;
        break;
      }
      r -= cnt;
      x++;
    }
  }
}

// Lex successor of an R-combination of [0, P); returns false at the end.
template <int R>
__device__ __forceinline__ bool next_comb(int *idx, int P) {
  int j = R - 1;
  while (j >= 0 && idx[j] == P - R + j) j--;
  if (j < 0) return false;
  idx[j]++;
  for (int jj = j + 1; jj < R; jj++) idx[jj] = idx[jj - 1] + 1;
  return true;
}

// Total order of partial results: higher score first, then lower key.
__device__ __forceinline__ bool better(double s1, uint64_t k1, double s0, uint64_t k0) {
  return s1 > s0 || (s1 == s0 && k1 < k0);
}

__device__ __forceinline__ void warp_argmax(double &s, uint64_t &k) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, s, off);
    const uint64_t ok = __shfl_xor_sync(0xffffffffu, k, off);
    if (better(os, ok, s, k)) {
      s = os;
      k = ok;
    }
  }
}

}  // namespace tsa

namespace tsa {

// Block-wide exclusive scan of per-thread (m, n, w): m, n exact integers and w
// a double-double.  Warp shuffle scans, then one warp scans the warp totals.
// Every kernel that builds prefix tables uses this one function with the same
// block size, so tables (and hence every tuple value) are bit-identical
// across the staged, compact and fused paths.  scratch: >= 32 * 24 bytes.
__device__ __forceinline__ void block_scan_mnw(uint32_t m, uint32_t n, dd w, uint32_t &m_ex,
                                               uint32_t &n_ex, dd &w_ex, uint32_t &m_tot,
                                               uint32_t &n_tot, char *scratch, int nthreads) {
  // threads >= nthreads must pass zeros; only the first nthreads/32 warps are scanned
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (nthreads + 31) >> 5;
  uint32_t mi = m, ni = n;
  dd wi = w;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t om = __shfl_up_sync(0xffffffffu, mi, off);
    const uint32_t on = __shfl_up_sync(0xffffffffu, ni, off);
    const double oh = __shfl_up_sync(0xffffffffu, wi.hi, off);
    const double ol = __shfl_up_sync(0xffffffffu, wi.lo, off);
    if (lane >= off) {
      mi += om;
      ni += on;
      wi = dd_add({oh, ol}, wi);
    }
  }
  uint32_t *sm = reinterpret_cast<uint32_t *>(scratch);
  uint32_t *sn = sm + 32;
  double *sh = reinterpret_cast<double *>(scratch + 256);
  double *sl = sh + 32;
  if (lane == 31 && warp < nw) {
    sm[warp] = mi;
    sn[warp] = ni;
    sh[warp] = wi.hi;
    sl[warp] = wi.lo;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t a = lane < nw ? sm[lane] : 0u, b = lane < nw ? sn[lane] : 0u;
    dd c = lane < nw ? dd{sh[lane], sl[lane]} : dd{0.0, 0.0};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t oa = __shfl_up_sync(0xffffffffu, a, off);
      const uint32_t ob = __shfl_up_sync(0xffffffffu, b, off);
      const double oh = __shfl_up_sync(0xffffffffu, c.hi, off);
      const double ol = __shfl_up_sync(0xffffffffu, c.lo, off);
      if (lane >= off) {
        a += oa;
        b += ob;
        c = dd_add({oh, ol}, c);
      }
    }
    // store inclusive warp prefixes; slot nw.. holds the totals
    __syncwarp();
    if (lane < nw) {
      sm[lane] = a;
      sn[lane] = b;
      sh[lane] = c.hi;
      sl[lane] = c.lo;
    }
  }
  __syncthreads();
  m_tot = sm[nw - 1];
  n_tot = sn[nw - 1];
  // exclusive prefix of this thread = (warp exclusive) + (lane exclusive)
  const uint32_t wm = warp ? sm[warp - 1] : 0u, wn = warp ? sn[warp - 1] : 0u;
  const dd ww = warp ? dd{sh[warp - 1], sl[warp - 1]} : dd{0.0, 0.0};
  const uint32_t lm = mi - m, ln = ni - n;
  dd lw;
  lw.hi = __shfl_up_sync(0xffffffffu, wi.hi, 1);
  lw.lo = __shfl_up_sync(0xffffffffu, wi.lo, 1);
  if (lane == 0) lw = {0.0, 0.0};
  m_ex = wm + lm;
  n_ex = wn + ln;
  w_ex = dd_add(ww, lw);
  __syncthreads();  // scratch reusable after return
}

}  // namespace tsa
