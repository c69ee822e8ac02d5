// k_tables.cuh -- SURVEY.md §8 row a2: the prefix-scan tables that make every
// class term O(1) (north star (2): "a prefix-scan of p_i and p_i^q").
//
//   k_luts   n-indexed 1/n^q (or ln n, 1/n at q == 1), n in [0, N], shared by
//            all slices of a call (N+1 pow instead of one pow per class term)
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

__global__ void k_luts(double *ipow, double *lnn, double *rcp, int64_t N, double q, int shannon) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n <= N;
       n += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)n;
    if (shannon) {
      lnn[n] = n == 0 ? CUDART_NAN : log(x);
      rcp[n] = n == 0 ? CUDART_NAN : __drcp_rn(x);
    }
    if (ipow) ipow[n] = n == 0 ? CUDART_NAN : __drcp_rn(pow(x, q));
  }
}

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
  Luts luts;
};

// One warp (one CTA) per slice.  Lane l owns the contiguous bins
// [l*L/32, (l+1)*L/32): it forms w_i (pow or c ln c) once into shared memory,
// a local double-double prefix, and a warp shuffle scan of (m, n, W) gives its
// offsets.  FULL tables copy the canonical entry of the last non-empty bin <= i,
// so tuples that differ only by empty bins read identical table values and
// evaluate bit-identically.
template <int MODE>
__global__ void __launch_bounds__(32) k_scan(ScanArgs g) {
  extern __shared__ double wsh[];  // [L]
  const int lane = threadIdx.x;
  const int64_t z = blockIdx.x;
  const int L = g.L, E = g.E;
  const uint32_t *h = g.hist + z * L;
  const int per = (L + 31) / 32;
  const int i0 = min(L, lane * per), i1 = min(L, i0 + per);
  // w_i for all bins, lane-strided: independent pow/log calls overlap
#pragma unroll 4
  for (int i = lane; i < L; i += 32) {
    const uint32_t c = __ldg(h + i);
    const double x = (double)c;
    wsh[i] = c == 0 ? 0.0 : (g.shannon ? __dmul_rn(x, log(x)) : pow(x, g.q));
  }
  __syncwarp();
  uint32_t m_l = 0, n_l = 0;
  dd w_l = {0.0, 0.0};
  for (int i = i0; i < i1; i++) {
    const uint32_t c = __ldg(h + i);
    if (c) {
      m_l++;
      n_l += c;
      w_l = dd_add_d(w_l, wsh[i]);
    }
  }
  uint32_t m_inc = m_l, n_inc = n_l;
  dd w_inc = w_l;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t om = __shfl_up_sync(0xffffffffu, m_inc, off);
    const uint32_t on = __shfl_up_sync(0xffffffffu, n_inc, off);
    const double oh = __shfl_up_sync(0xffffffffu, w_inc.hi, off);
    const double ol = __shfl_up_sync(0xffffffffu, w_inc.lo, off);
    if (lane >= off) {
      m_inc += om;
      n_inc += on;
      w_inc = dd_add({oh, ol}, w_inc);
    }
  }
  const uint32_t m_tot = __shfl_sync(0xffffffffu, m_inc, 31);
  const uint32_t m_ex = m_inc - m_l, n_ex = n_inc - n_l;
  dd w_ex;
  w_ex.hi = __shfl_up_sync(0xffffffffu, w_inc.hi, 1);
  w_ex.lo = __shfl_up_sync(0xffffffffu, w_inc.lo, 1);
  uint32_t *cC = g.cC + z * E;
  double *cWhi = g.cWhi + z * E, *cWlo = g.cWlo + z * E;
  int32_t *cBin = g.cBin + z * E;
  if (lane == 0) {
    cC[0] = 0;
    cWhi[0] = 0.0;
    cWlo[0] = 0.0;
    cBin[0] = -1;
  }
  {
    uint32_t e = m_ex + 1, ncum = n_ex;
    dd wl = {0.0, 0.0};
    for (int i = i0; i < i1; i++) {
      const uint32_t c = __ldg(h + i);
      if (c) {
        ncum += c;
        wl = dd_add_d(wl, wsh[i]);
        const dd W = lane == 0 ? wl : dd_add(w_ex, wl);
        cC[e] = ncum;
        cWhi[e] = W.hi;
        cWlo[e] = W.lo;
        cBin[e] = i;
        e++;
      }
    }
  }
  __syncwarp();
  int status = g.status[z];
  if (status == kOK && (int)m_tot < g.k + 1) status = kNoValidSplit;
  if (lane == 0) g.status[z] = status;
  const uint32_t *tC = cC;
  const double *tWhi = cWhi, *tWlo = cWlo;
  int M = (int)m_tot;
  if (g.full) {
    uint32_t *fC = g.fC + z * E;
    double *fWhi = g.fWhi + z * E, *fWlo = g.fWlo + z * E;
    int32_t *fBin = g.fBin + z * E;
    if (lane == 0) {
      fC[0] = 0;
      fWhi[0] = 0.0;
      fWlo[0] = 0.0;
      fBin[0] = -1;
    }
    uint32_t r = m_ex;
    for (int i = i0; i < i1; i++) {
      if (__ldg(h + i)) r++;
      fC[i + 1] = cC[r];
      fWhi[i + 1] = cWhi[r];
      fWlo[i + 1] = cWlo[r];
      fBin[i + 1] = i;
    }
    __syncwarp();
    tC = fC;
    tWhi = fWhi;
    tWlo = fWlo;
    M = L;
  }
  if (lane == 0) g.M[z] = M;
  if (status != kOK) return;
  SliceTables t{tC, tWhi, tWlo, nullptr};
  double *Asuf = g.Asuf + z * L;
  for (int i = lane; i <= M - 2; i += 32) Asuf[i] = class_term<MODE>(t, g.luts, i + 1, M - 1);
}

// R[a][b] = combine(T(a+1, b), Asuf[b]) for 0 <= a < b <= M-2 (k >= 3,
// pseudo-additive): the last two classes of a tuple, so the search's inner
// loop is one multiply (or add) and one compare per tuple.  Entries b > M-2
// of each row are padded with NaN (never selected) up to the row stride RS.
template <int MODE>
__global__ void __launch_bounds__(256) k_rtable(const uint32_t *C, const double *Whi,
                                                const double *Wlo, const double *Asuf,
                                                const int32_t *Mz, const int32_t *status,
                                                double *R, int E, int L, int RS, Luts luts) {
  const int z = blockIdx.y;
  const int a = blockIdx.x;
  if (status[z] != kOK) return;
  const int M = Mz[z];
  if (a > M - 3) return;
  SliceTables t{C + (size_t)z * E, Whi + (size_t)z * E, Wlo + (size_t)z * E, nullptr};
  const double *as = Asuf + (size_t)z * L;
  double *row = R + ((size_t)z * L + a) * RS;
  for (int b = threadIdx.x; b < RS; b += blockDim.x) {
    double v = CUDART_NAN;
    if (b > a && b <= M - 2) v = combine<MODE>(class_term<MODE>(t, luts, a + 1, b), __ldg(as + b));
    row[b] = v;
  }
}

}  // namespace tsa
