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

// Class-term constants without an N-sized table.  A class of n voxels needs
// n^-q (or ln n and 1/n at q == 1) for integer n in [1, 2^31).  Round 1 read
// them from an (N+1)-entry table: at 12-bit CT (N = 2^20, 8 MB) every k = 2
// tuple paid an L2 gather.  Here n = 2^s (j + r 2^-s) with j = n >> s in
// [2^10, 2^11) (s = 0 and r = 0 for n <= 2^11), d = r / (j 2^s) in [0, 2^-10):
//   n^-q = j^-q * 2^(-s q) * (1 + d)^-q,    (1 + d)^-q = sum_k binom(-q, k) d^k
//   ln n = ln j + s ln 2 + d * P(d),         P(d) = log1p(d)/d
//   1/n  = (1/j) 2^-s * (1 + d)^-1
// from a 32 KB table (j^-q or ln j, 1/j for j <= 2^11), 2^(-s q) or s ln 2 (in
// the kernel parameters) and
// a Horner polynomial in registers.  Degree 5 (q <= 2), 6 (q <= 10) or 12
// keeps the truncation below 2^-56 relative for q <= 256; n <= 2^11 reads the table
// entry itself (d = 0 makes the polynomial exactly 1).  Every kernel uses this
// one function, so a tuple's value is still a pure function of the tuple.
constexpr int kSB = 11;               // table bits
constexpr int kSN = (1 << kSB) + 1;   // entries j = 0 .. 2^kSB
constexpr int kSmallLut = 2 * kSN;  // doubles in the small table

// One table position of a slice, packed for the k = 2 search (two 16-byte
// loads): W = dd prefix of w at the position, as = Asuf[e-1] = T(e, M-1),
// c = prefix count, bin = the bin of the position.
struct __align__(16) K2Row {
  double wh, wl, as;
  uint32_t c;
  int32_t bin;
};

// Bound record of the pruned k = 2 search (k2_tile PRUNE, one 16-byte load):
// wub >= the exact W (dd hi + lo, rounded up) at the record's last row, amax
// >= max Asuf over its rows (rounded up to float), c = C at its first row.
struct __align__(16) K2Chk {
  double wub;
  float amax;
  uint32_t c;
};

struct Luts {
  const double *sp;  // [kSN] j^-q (ln j at q == 1) | [kSN] 1/j; entry j = 0: NaN
  double p2[32];     // 2^(-s q) (q == 1: ln 2^s), s = 0..31, from the host (kernel parameter:
                     // constant cache, off the shared-memory path)
  double c[13];      // binom(-q, k), k = 0..12 (q == 1: (-1)^k)
  double lc[7];      // log1p(d)/d = sum_k lc[k] d^k = sum (-1)^k d^k / (k+1)
  int deg;           // 5, 6 or 12 (c[deg+1..] are zero up to c[6])
  double iqm1;       // 1 / (q - 1)
  double omq;        // 1 - q
  int shannon;       // q == 1
};

// Table access of the class-size constants: the global layout of Luts::sp
// ([kSN] j^-q | [kSN] 1/j | [32] 2^(-s q)); kernels that stage the table in
// shared memory use an interleaved {j^-q, 1/j} layout (one 16-byte load) with
// the same arithmetic, so every kernel computes bit-identical values.
// p2(s): 2^(-s q) (Luts::p2) from a shared-memory copy -- the k = 2 kernels
// index it per lane, and a lane-divergent index into the kernel-parameter
// copy serialises in the constant cache (ncu: LDC in the k = 2 hot loop).
#ifdef TSA_TRACE
// debug builds only: 8 phase timestamps per slice of a per-slice kernel
// (k_mid: tools/fused_trace.py; k_scan_seed: tools/scan_trace.py)
__device__ unsigned long long g_mphase[8 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TSA_MPHASE(z, i) \
  if (threadIdx.x == 0 && (z) < 4096) g_mphase[8 * (z) + (i)] = gtimer();
// inside the table build (scan_slice / build_tables): tools/scan_trace.py
__device__ unsigned long long g_sphase[8 * 4096];
#define TSA_SPHASE(z, i) \
  if (threadIdx.x == 0 && (z) < 4096) g_sphase[8 * (z) + (i)] = gtimer();
#else
#define TSA_MPHASE(z, i)
#define TSA_SPHASE(z, i)
#endif

struct SpGlobal {
  const double *sp;
  const double *p2s = nullptr;  // shared copy of Luts::p2 (k2_term users only)
  const double *k1q = nullptr;  // (the pruned k = 2 search only; unused here)
  __device__ __forceinline__ double2 jr(uint32_t j) const { return make_double2(sp[j], sp[kSN + j]); }
  __device__ __forceinline__ double p2(int s) const { return p2s[s]; }
};
struct SpPair {  // shared-memory staging: jr[j] = {j^-q or ln j, 1/j}
  const double2 *jrt;
  const double *p2s;  // shared copy of Luts::p2
  const double *k1q = nullptr;  // [kK1Q] k^(1-q) (the pruned k = 2 search only)
  __device__ __forceinline__ double2 jr(uint32_t j) const { return jrt[j]; }
  __device__ __forceinline__ double p2(int s) const { return p2s[s]; }
};

// n = 2^s (j + r 2^-s): table index j, exponent s and d = r / (j 2^s)
__device__ __forceinline__ void nsplit_idx(uint32_t n, uint32_t &j, int &s, uint32_t &r) {
  s = max(0, 32 - kSB - __clz(n));
  j = n >> s;
  r = n - (j << s);
}
__device__ __forceinline__ double two_pow_neg(int s) { return __hiloint2double((1023 - s) << 20, 0); }

__device__ __forceinline__ double horner_c(const Luts &l, double d) {
  double p = l.c[5];
  if (l.deg > 6) {  // uniform branches
    double h = l.c[12];
#pragma unroll
    for (int k = 11; k >= 6; k--) h = __fma_rn(h, d, l.c[k]);
    p = __fma_rn(h, d, l.c[5]);
  } else if (l.deg == 6) {
    p = __fma_rn(l.c[6], d, l.c[5]);
  }
#pragma unroll
  for (int k = 4; k >= 0; k--) p = __fma_rn(p, d, l.c[k]);
  return p;
}

// horner_c with the degree fixed at compile time (DEG = l.deg): the same
// operations, for kernels specialised on the degree.
template <int DEG>
__device__ __forceinline__ double horner_c_deg(const Luts &l, double d) {
  double p = l.c[5];
  if (DEG > 6) {
    double h = l.c[12];
#pragma unroll
    for (int k = 11; k >= 6; k--) h = __fma_rn(h, d, l.c[k]);
    p = __fma_rn(h, d, l.c[5]);
  } else if (DEG == 6) {
    p = __fma_rn(l.c[6], d, l.c[5]);
  }
#pragma unroll
  for (int k = 4; k >= 0; k--) p = __fma_rn(p, d, l.c[k]);
  return p;
}

// d = (r * (1/j)) * 2^-s with the exact power-of-two scaling done on the
// exponent field (r >= 1: r/j >= 2^-11, so the result stays normal); equal to
// __dmul_rn(x, two_pow_neg(s)) bit for bit.
__device__ __forceinline__ double scale_pow2_neg(double x, int s, uint32_t r) {
  const int hi = __double2hiint(x) - (s << 20);
  return r ? __hiloint2double(hi, __double2loint(x)) : 0.0;
}

// n^-q (q != 1); NaN at n = 0
template <class Tab>
__device__ __forceinline__ double ipow_t(const Luts &l, const Tab &tab, uint32_t n) {
  uint32_t j, r;
  int s;
  nsplit_idx(n, j, s, r);
  const double2 e = tab.jr(j);
  const double d = __dmul_rn(__dmul_rn((double)r, e.y), two_pow_neg(s));
  return __dmul_rn(__dmul_rn(e.x, tab.p2s ? tab.p2s[s] : l.p2[s]), horner_c(l, d));
}

// Shannon class term S = ln n - w / n (q == 1); NaN at n = 0
template <class Tab>
__device__ __forceinline__ double shannon_t(const Luts &l, const Tab &tab, uint32_t n, double w) {
  uint32_t j, r;
  int s;
  nsplit_idx(n, j, s, r);
  const double2 e = tab.jr(j);
  const double two_ms = two_pow_neg(s);
  const double d = __dmul_rn(__dmul_rn((double)r, e.y), two_ms);
  double p = l.lc[6];
#pragma unroll
  for (int k = 5; k >= 0; k--) p = __fma_rn(p, d, l.lc[k]);
  const double lnn = __dadd_rn(__dadd_rn(e.x, tab.p2s ? tab.p2s[s] : l.p2[s]), __dmul_rn(d, p));
  const double rcp = __dmul_rn(__dmul_rn(e.y, two_ms), horner_c(l, d));
  return __dsub_rn(lnn, __dmul_rn(w, rcp));
}

__device__ __forceinline__ double ipow_n(const Luts &l, uint32_t n) { return ipow_t(l, SpGlobal{l.sp}, n); }
__device__ __forceinline__ double shannon_term(const Luts &l, uint32_t n, double w) {
  return shannon_t(l, SpGlobal{l.sp}, n, w);
}

// The class term from its count n and weight w (see class_term).
template <int MODE, class Tab>
__device__ __forceinline__ double class_term_nw(const Luts &l, const Tab &tab, uint32_t n, double w) {
  if (MODE == PROD_MAX || MODE == PROD_MIN) {
    return __dmul_rn(w, ipow_t(l, tab, n));
  } else if (MODE == SUM) {
    return shannon_t(l, tab, n, w);
  } else {
    if (l.shannon) return shannon_t(l, tab, n, w);
    const double A = __dmul_rn(w, ipow_t(l, tab, n));
    return __dmul_rn(__dsub_rn(1.0, A), l.iqm1);
  }
}

// Class term T(a, b) of the class made of table positions [a, b]:
//   q != 1, pseudo-additive: A = W / n^q = sum_{i in C} (c_i / n)^q
//   q == 1:                  S = ln n - (sum c ln c) / n
//   sum-plus-product:        S = (1 - A) / (q - 1)  (or the q == 1 S)
// An empty class (n == 0, FULL enumeration only) yields NaN, which never wins a
// comparison, so invalid tuples are skipped without a branch.
// p2s: a shared-memory copy of Luts::p2 (stage_p2) -- the index s differs
// across lanes, and lane-divergent indices into the kernel-parameter copy
// serialise in the constant cache; null reads the parameter copy (same values).
template <int MODE>
__device__ __forceinline__ double class_term(const SliceTables &t, const Luts &l, int a, int b,
                                             const double *p2s = nullptr) {
  // generic loads: the tables may be staged in shared memory
  const uint32_t n = t.C[b + 1] - t.C[a];
  const double w = dd_diff(t.Whi[b + 1], t.Wlo[b + 1], t.Whi[a], t.Wlo[a]);
  return class_term_nw<MODE>(l, SpGlobal{l.sp, p2s}, n, w);
}

// Luts::p2 into shared memory (threads 0..31; the caller synchronises).
__device__ __forceinline__ void stage_p2(const Luts &l, double *p2s) {
  if (threadIdx.x < 32) p2s[threadIdx.x] = l.p2[threadIdx.x];
}

// Entry e of the small table (Luts::sp layout).
__device__ __forceinline__ double small_lut_entry(int e, double q, int shannon) {
  if (e < kSN) {
    const double x = (double)e;
    return e == 0 ? CUDART_NAN : (shannon ? log(x) : __drcp_rn(pow(x, q)));
  }
  const int j = e - kSN;
  return j == 0 ? CUDART_NAN : __drcp_rn((double)j);
}

// Fills the small table of Luts::sp (kSmallLut doubles); any grid.
__global__ void k_small_luts(double *sp, double q, int shannon) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kSmallLut; e += gridDim.x * blockDim.x)
    sp[e] = small_lut_entry(e, q, shannon);
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

// ------------------------------------------------ TMA bulk staging (1-D)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace tsa
