// k_tables.cuh -- SURVEY.md §8 row a2: the prefix-scan tables that make every
// class term O(1) (north star (2): "a prefix-scan of p_i and p_i^q").
//
//   k_small_luts (tsa_device.cuh) the 33 KB table behind n^-q / ln n / 1/n
//            (j^-q for j <= 2^11, 1/j, 2^(-s q)); no N-sized table
//   k_scan   per slice: compaction of the non-empty bins, exact prefix counts
//            C, double-double prefix sums W of w_i = c_i^q (c_i ln c_i at q=1),
//            and the last-class terms Asuf[i] = T(i+1, M-1)
//   k_rtable per slice (k >= 3): R[a][b] = T(a+1,b) (x) T(b+1,M-1)
//
// The objective is invariant to N (A_j = sum c^q / n_j^q, R11), so
// tables are in counts; p_i = c_i/N only appears in the definitional
// recomputation of phi(t*) (k_finalize).
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

struct ScanArgs {
  const uint32_t *hist;  // [nz][L]
  int32_t *status;       // [nz]
  int64_t nz;
  int L, E, k;           // E = L + 1 (entries per slice incl. sentinel)
  double q;
  int shannon;           // w = c ln c instead of c^q
  int full;              // FULL enumeration: tables over all L bins
  uint32_t *cC;          // canonical (compacted) tables [nz][E]
  double *cWhi, *cWlo;
  int32_t *cBin;
  uint32_t *fC;          // full tables [nz][E] (only when full)
  double *fWhi, *fWlo;
  int32_t *fBin;
  double *Asuf;          // [nz][L]
  int32_t *M;            // [nz] entries used by the search (m or L)
  int32_t *mmax;         // max over slices of M (atomicMax; zeroed before launch) or null
  K2Row *rows;           // [nz][RE] packed positions for the k = 2 search, or null
  int RE;                // row stride of `rows`
  Luts luts;
};

// Canonical prefix tables of one slice, built by the whole CTA (any block
// size; every caller uses kTableThreads so the rounding is identical):
//   w_i = c_i^q (c_i ln c_i at q == 1) for all bins, lane-strided (independent
//   pow calls overlap); thread t then owns the contiguous bins
//   [t*per, (t+1)*per): local double-double prefix, a block scan of
//   (#non-empty, count, W) gives its offsets, and it writes its entries
//   e = rank + 1:  C[e] (exact prefix count), Whi/Wlo[e], Bin[e]; entry 0 is
//   the sentinel (0, 0, -1).  Returns m (non-empty bins) and N (total count).
constexpr int kTableThreads = 256;

__device__ __forceinline__ void build_tables(const uint32_t *h, int L, double q, int shannon,
                                             double *wsh, uint32_t *C, double *Whi, double *Wlo,
                                             int32_t *Bin, char *scratch, int &m_out,
                                             uint32_t &n_out, const int zt = 1 << 30) {
  // exactly kTableThreads threads do the work whatever the block size (>= it),
  // so every kernel produces bit-identical tables
  const int tid = threadIdx.x, T = kTableThreads;
  const int per = (L + T - 1) / T;
  const int i0 = tid < T ? min(L, tid * per) : L, i1 = tid < T ? min(L, i0 + per) : L;
  // (a compacted variant -- listing the non-empty bins first so the pow calls
  // spread evenly -- measured slower on c5: 84 vs 63 us)
  {
    for (int i = tid; i < L; i += blockDim.x) {
      const uint32_t c = h[i];
      const double x = (double)c;
      wsh[i] = c == 0 ? 0.0 : (shannon ? __dmul_rn(x, log(x)) : pow(x, q));
    }
  }
  __syncthreads();
  TSA_SPHASE(zt, 1)
  uint32_t m_l = 0, n_l = 0;
  dd w_l = {0.0, 0.0};
  for (int i = i0; i < i1; i++) {
    const uint32_t c = h[i];
    if (c) {
      m_l++;
      n_l += c;
      w_l = dd_add_d(w_l, wsh[i]);
    }
  }
  uint32_t m_ex, n_ex, m_tot, n_tot;
  dd w_ex;
  TSA_SPHASE(zt, 2)
  block_scan_mnw(m_l, n_l, w_l, m_ex, n_ex, w_ex, m_tot, n_tot, scratch, T);
  TSA_SPHASE(zt, 3)
  if (tid == 0) {
    C[0] = 0;
    Whi[0] = 0.0;
    Wlo[0] = 0.0;
    Bin[0] = -1;
  }
  uint32_t e = m_ex + 1, ncum = n_ex;
  dd wl = {0.0, 0.0};
  for (int i = i0; i < i1; i++) {
    const uint32_t c = h[i];
    if (c) {
      ncum += c;
      wl = dd_add_d(wl, wsh[i]);
      const dd W = dd_add(w_ex, wl);
      C[e] = ncum;
      Whi[e] = W.hi;
      Wlo[e] = W.lo;
      Bin[e] = i;
      e++;
    }
  }
  __syncthreads();
  m_out = (int)m_tot;
  n_out = n_tot;
}

// One CTA (kTableThreads) per slice: canonical tables via build_tables; FULL
// tables copy the canonical entry of the last non-empty bin <= i, so tuples
// that differ only by empty bins read identical table values and evaluate
// bit-identically; then Asuf.
// The per-slice body of k_scan (also run by the stream pipeline's histogram
// tasks, k_stream.cuh): h = the slice's histogram (global or shared), wsh =
// [L] doubles + 1 KB of shared scratch, blockDim.x == kTableThreads.
template <int MODE>
__device__ void scan_slice(const ScanArgs &g, const int64_t z, const uint32_t *h, double *wsh) {
  __shared__ double s_p2[32];  // Luts::p2 (read before: build_tables synchronises)
  stage_p2(g.luts, s_p2);
  const int tid = threadIdx.x;
  const int L = g.L, E = g.E;
  char *scratch = reinterpret_cast<char *>(wsh + L);
  uint32_t *cC = g.cC + z * E;
  double *cWhi = g.cWhi + z * E, *cWlo = g.cWlo + z * E;
  int32_t *cBin = g.cBin + z * E;
  int m;
  uint32_t ntot;
  TSA_SPHASE(z, 0)
  build_tables(h, L, g.q, g.shannon, wsh, cC, cWhi, cWlo, cBin, scratch, m, ntot, (int)z);
  TSA_SPHASE(z, 4)
  int status = g.status[z];
  if (status == kOK && m < g.k + 1) status = kNoValidSplit;
  __syncthreads();
  if (tid == 0) g.status[z] = status;
  const uint32_t *tC = cC;
  const double *tWhi = cWhi, *tWlo = cWlo;
  int M = m;
  if (g.full) {
    uint32_t *fC = g.fC + z * E;
    double *fWhi = g.fWhi + z * E, *fWlo = g.fWlo + z * E;
    int32_t *fBin = g.fBin + z * E;
    // rank of bin i among non-empty bins: binary search in the canonical list
    for (int i = tid; i <= L; i += blockDim.x) {
      if (i == 0) {
        fC[0] = 0;
        fWhi[0] = 0.0;
        fWlo[0] = 0.0;
        fBin[0] = -1;
        continue;
      }
      const int bin = i - 1;
      int lo = 0, hi = m;  // largest r in [0, m] with cBin[r] <= bin (cBin[0] = -1)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cBin[mid] <= bin) lo = mid;
        else hi = mid - 1;
      }
      fC[i] = cC[lo];
      fWhi[i] = cWhi[lo];
      fWlo[i] = cWlo[lo];
      fBin[i] = bin;
    }
    __syncthreads();
    tC = fC;
    tWhi = fWhi;
    tWlo = fWlo;
    M = L;
  }
  if (tid == 0) {
    g.M[z] = M;
    if (g.mmax) atomicMax(g.mmax, M);
  }
  if (status != kOK) return;
  const int32_t *tBin = g.full ? g.fBin + z * E : cBin;
  // canonical tables back into shared memory (wsh is free now) for the Asuf
  // class terms and the packed rows: one coalesced pass instead of scattered
  // L2 reads of the tables just written (round 2: 6.4 us of a c5 slice's
  // 26 us table build, profiles/r2zz3); same values
  if (!g.full && (size_t)(M + 1) * 24 <= (size_t)L * 8) {
    double *sWhi = wsh, *sWlo = wsh + (M + 1);
    uint32_t *sC = reinterpret_cast<uint32_t *>(sWlo + (M + 1));
    int32_t *sBin = reinterpret_cast<int32_t *>(sC + (M + 1));
    for (int e = tid; e <= M; e += blockDim.x) {
      sWhi[e] = tWhi[e];
      sWlo[e] = tWlo[e];
      sC[e] = tC[e];
      sBin[e] = tBin[e];
    }
    __syncthreads();
    tC = sC;
    tWhi = sWhi;
    tWlo = sWlo;
    tBin = sBin;
  }
  SliceTables t{tC, tWhi, tWlo, nullptr};
  double *Asuf = g.Asuf + z * L;
  K2Row *rows = g.rows ? g.rows + z * g.RE : nullptr;
  TSA_SPHASE(z, 5)
  for (int i = tid; i <= M - 2; i += blockDim.x) {
    const double as = class_term<MODE>(t, g.luts, i + 1, M - 1, s_p2);
    Asuf[i] = as;
    if (rows) rows[i + 1] = K2Row{tWhi[i + 1], tWlo[i + 1], as, tC[i + 1], tBin[i + 1]};
  }
  TSA_SPHASE(z, 6)
}

template <int MODE>
__global__ void __launch_bounds__(kTableThreads) k_scan(ScanArgs g) {
  // [L] doubles + 1 KB scan scratch, then the slice's histogram [L] u32: the
  // per-thread bin loops of build_tables read it from shared memory (round 1
  // read it from global memory with dependent branches: latency-bound, 74 us
  // on c5)
  extern __shared__ __align__(16) double wsh[];
  uint32_t *hs = reinterpret_cast<uint32_t *>(wsh + g.L + 128);
  const uint4 *h4 = reinterpret_cast<const uint4 *>(g.hist + (int64_t)blockIdx.x * g.L);
  if ((g.L & 3) == 0 && (reinterpret_cast<uintptr_t>(g.hist) & 15) == 0)
    for (int i = threadIdx.x; i < g.L / 4; i += blockDim.x) reinterpret_cast<uint4 *>(hs)[i] = __ldg(h4 + i);
  else
    for (int i = threadIdx.x; i < g.L; i += blockDim.x) hs[i] = g.hist[(int64_t)blockIdx.x * g.L + i];
  __syncthreads();
  scan_slice<MODE>(g, blockIdx.x, hs, wsh);
}

// R[a][b] = combine(T(a+1, b), Asuf[b]) for 0 <= a < b <= M-2 (k >= 3,
// pseudo-additive): the last two classes of a tuple, so the search's inner
// loop is one multiply (or add) and one compare per tuple.  Entries b > M-2
// of each row are padded with NaN (never selected) up to the row stride RS.
// (See k_rtable below for the three tables.)
template <int MODE>
__global__ void __launch_bounds__(256) k_rtable(const uint32_t *C, const double *Whi,
                                                const double *Wlo, const double *Asuf,
                                                const int32_t *Mz, const int32_t *status,
                                                double *R, double *PP, double *AI, int E, int L,
                                                int RS, Luts luts) {
  // row x = blockIdx.x of the three k >= 3 tables (row stride RS, NaN padding):
  //   R[x][y]  = T(x+1, y) (x) T(y+1, M-1)   last two classes,      x < y <= M-2
  //   PP[x][y] = T(0, x) (x) T(x+1, y)        first two classes,    x < y <= M-2
  //   AI[x][y] = T(x, y)                      one interval (k = 4), x <= y <= M-2
  // each the same expression as the on-the-fly fold, so values are identical
  // one CTA per slice, threads over the flattened (row, column) entries
  const int z = blockIdx.x;
  if (status[z] != kOK) return;
  const int M = Mz[z];
  SliceTables t{C + (size_t)z * E, Whi + (size_t)z * E, Wlo + (size_t)z * E, nullptr};
  const double *as = Asuf + (size_t)z * L;
  const int rows = M - 1;  // a in [0, M-2]
  for (int64_t e = threadIdx.x; e < (int64_t)rows * RS; e += blockDim.x) {
    const int a = (int)(e / RS), b = (int)(e % RS);
    double r = CUDART_NAN, pp = CUDART_NAN, ai = CUDART_NAN;
    if (b <= M - 2) {
      if (b > a) {
        const double mid = class_term<MODE>(t, luts, a + 1, b);
        r = combine<MODE>(mid, __ldg(as + b));
        pp = combine<MODE>(class_term<MODE>(t, luts, 0, a), mid);
      }
      if (AI && b >= a) ai = class_term<MODE>(t, luts, a, b);
    }
    const size_t o = ((size_t)z * L + a) * RS + b;
    R[o] = r;
    PP[o] = pp;
    if (AI) AI[o] = ai;
  }
}

// tsa_class_consts (testing): the class-size constants exactly as the search
// kernels compute them -- q != 1: a = n^-q; q == 1: a = ln n (S with w = 0),
// b = 1/n (from S with w = -1: S = ln n + 1/n, minus ln n, would round; use
// the same pieces directly instead).
__global__ void k_class_consts(const uint32_t *n, int64_t count, Luts l, double *a, double *b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = n[i];
    if (!l.shannon) {
      a[i] = ipow_n(l, v);
    } else {
      a[i] = shannon_term(l, v, 0.0);
      uint32_t j, r;
      int s;
      nsplit_idx(v, j, s, r);
      const double two_ms = two_pow_neg(s);
      const double d = __dmul_rn(__dmul_rn((double)r, l.sp[kSN + j]), two_ms);
      if (b) b[i] = __dmul_rn(__dmul_rn(l.sp[kSN + j], two_ms), horner_c(l, d));
    }
  }
}

}  // namespace tsa
