// tsa_kernels.cuh -- the libtsa kernels (sm_100a), one per SURVEY.md §8(a) row:
//   a1 k_histogram   per-slice gray-level histogram
//   a2 k_luts/k_scan prefix tables of c and c^q
//      k_rtable      last-two-class table (k >= 3)
//   a3 k_search      exhaustive tuple search, fp64
//   a4 k_merge/k_finalize  argmax + phi(t*) recompute
//   a5 k_label       Algorithm 1 generalised to k classes PAPER.md:464-477
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

// =============================================================== a1: histogram
// One CTA per (slice chunk, slice).  Per-warp (or per-group) privatised
// shared-memory bins, 128-bit coalesced loads, and a run fast path: a 16-byte
// vector whose bytes are all equal (the constant -2000 HU background outside
// the field of view, ~21 % of a CT slice) costs one shared
// atomic instead of 16.  Out-of-range voxels (>= bins) set the slice's
// LEVEL_OVERFLOW status and are not counted.
struct HistArgs {
  const uint8_t *vol;  // byte pointer to the volume
  uint32_t *hist;      // [nz][L], zeroed before launch
  int32_t *status;     // [nz], zeroed before launch
  int64_t n;           // voxels per slice
  int L;
  int replicas;        // number of smem copies of the bins
  int chunks;          // CTAs per slice (gridDim.x)
};

template <typename T>
__global__ void __launch_bounds__(512) k_histogram(HistArgs g) {
  extern __shared__ uint32_t sh[];
  const int z = blockIdx.y;
  const int L = g.L;
  const int nthr = blockDim.x;
  const int rep = (threadIdx.x >> 5) % g.replicas;
  for (int i = threadIdx.x; i < L * g.replicas; i += nthr) sh[i] = 0;
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  uint32_t *bins = sh + rep * L;
  const T *slice = reinterpret_cast<const T *>(g.vol) + (size_t)z * g.n;
  constexpr int VEC = 16 / sizeof(T);
  // aligned middle part of this slice
  const uintptr_t base = reinterpret_cast<uintptr_t>(slice);
  int64_t head = (int64_t)(((16 - (base & 15)) & 15) / sizeof(T));
  if (head > g.n) head = g.n;
  const int64_t nvec = (g.n - head) / VEC;
  const int64_t tail0 = head + nvec * VEC;
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice + head);
  // chunk of vectors for this CTA
  const int64_t per = (nvec + g.chunks - 1) / g.chunks;
  const int64_t v0 = per * blockIdx.x;
  const int64_t v1 = min(nvec, v0 + per);
  int ovf = 0;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += nthr) {
    const uint4 w = __ldcs(v4 + i);  // streamed once: evict-first
    if (sizeof(T) == 1) {
      const uint32_t b0 = w.x & 0xffu;
      if (w.x == w.y && w.x == w.z && w.x == w.w && w.x == b0 * 0x01010101u) {
        if (b0 < (uint32_t)L) atomicAdd(bins + b0, 16u);
        else ovf = 1;
      } else {
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t b = (ws[q] >> (8 * j)) & 0xffu;
            if (b < (uint32_t)L) atomicAdd(bins + b, 1u);
            else ovf = 1;
          }
        }
      }
    } else {
      const uint32_t b0 = w.x & 0xffffu;
      if (w.x == w.y && w.x == w.z && w.x == w.w && w.x == b0 * 0x00010001u) {
        if (b0 < (uint32_t)L) atomicAdd(bins + b0, 8u);
        else ovf = 1;
      } else {
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
#pragma unroll
          for (int j = 0; j < 2; j++) {
            const uint32_t b = (ws[q] >> (16 * j)) & 0xffffu;
            if (b < (uint32_t)L) atomicAdd(bins + b, 1u);
            else ovf = 1;
          }
        }
      }
    }
  }
  // unaligned head / tail: chunk 0 handles them
  if (blockIdx.x == 0) {
    for (int64_t i = threadIdx.x; i < head; i += nthr) {
      const uint32_t b = slice[i];
      if (b < (uint32_t)L) atomicAdd(bins + b, 1u);
      else ovf = 1;
    }
    for (int64_t i = tail0 + threadIdx.x; i < g.n; i += nthr) {
      const uint32_t b = slice[i];
      if (b < (uint32_t)L) atomicAdd(bins + b, 1u);
      else ovf = 1;
    }
  }
  if (ovf) overflow = 1;
  __syncthreads();
  uint32_t *out = g.hist + (size_t)z * L;
  for (int b = threadIdx.x; b < L; b += nthr) {
    uint32_t s = 0;
    for (int r = 0; r < g.replicas; r++) s += sh[r * L + b];
    if (s) atomicAdd(out + b, s);
  }
  if (threadIdx.x == 0 && overflow) g.status[z] = kLevelOverflow;
}

// ================================================================ a2: tables
// n-indexed lookup tables shared by all slices of a call: 1/n^q (q != 1) or
// ln n and 1/n (q == 1), n in [0, N].  N+1 pow calls per call replace one pow
// per class term in the search.
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
  // canonical (compacted) tables [nz][E]
  uint32_t *cC;
  double *cWhi, *cWlo;
  int32_t *cBin;
  // full tables [nz][E] (only when full)
  uint32_t *fC;
  double *fWhi, *fWlo;
  int32_t *fBin;
  double *Asuf;  // [nz][L]
  int32_t *M;    // [nz] entries used by the search (m or L)
  Luts luts;
  int mode;
};

// One warp per slice.  Lane l owns the contiguous bins [l*L/32, (l+1)*L/32):
// it compacts its non-empty bins, forms c^q with pow (or c ln c), and a local
// double-double prefix; a warp shuffle scan of the lane totals gives each lane
// its dd offset.  FULL tables copy the canonical entry of the last non-empty
// bin <= i, so tuples that differ only by empty bins read identical table
// values and evaluate bit-identically.
template <int MODE>
__global__ void __launch_bounds__(128) k_scan(ScanArgs g) {
  const int lane = threadIdx.x & 31;
  const int64_t z = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (z >= g.nz) return;
  const int L = g.L, E = g.E;
  const uint32_t *h = g.hist + z * L;
  const int per = (L + 31) / 32;
  const int i0 = min(L, lane * per), i1 = min(L, i0 + per);
  uint32_t m_l = 0, n_l = 0;
  dd w_l = {0.0, 0.0};
  for (int i = i0; i < i1; i++) {
    const uint32_t c = __ldg(h + i);
    if (c) {
      m_l++;
      n_l += c;
      const double x = (double)c;
      w_l = dd_add_d(w_l, g.shannon ? __dmul_rn(x, log(x)) : pow(x, g.q));
    }
  }
  // warp inclusive scans of (m, n, w)
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
  uint32_t m_ex = m_inc - m_l, n_ex = n_inc - n_l;
  dd w_ex;
  w_ex.hi = __shfl_up_sync(0xffffffffu, w_inc.hi, 1);
  w_ex.lo = __shfl_up_sync(0xffffffffu, w_inc.lo, 1);
  if (lane == 0) w_ex = {0.0, 0.0};
  uint32_t *cC = g.cC + z * E;
  double *cWhi = g.cWhi + z * E, *cWlo = g.cWlo + z * E;
  int32_t *cBin = g.cBin + z * E;
  if (lane == 0) {
    cC[0] = 0;
    cWhi[0] = 0.0;
    cWlo[0] = 0.0;
    cBin[0] = -1;
  }
  // second pass: write canonical entries
  {
    uint32_t e = m_ex + 1, ncum = n_ex;
    dd wl = {0.0, 0.0};
    for (int i = i0; i < i1; i++) {
      const uint32_t c = __ldg(h + i);
      if (c) {
        ncum += c;
        const double x = (double)c;
        wl = dd_add_d(wl, g.shannon ? __dmul_rn(x, log(x)) : pow(x, g.q));
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
  if (lane == 0) {
    g.status[z] = status;
  }
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
    uint32_t r = m_ex;  // canonical entries before bin i0
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
// loop is one multiply (or add) and one compare per tuple.
template <int MODE>
__global__ void __launch_bounds__(256) k_rtable(const uint32_t *C, const double *Whi,
                                                const double *Wlo, const double *Asuf,
                                                const int32_t *Mz, const int32_t *status,
                                                double *R, int E, int L, Luts luts) {
  const int z = blockIdx.y;
  const int a = blockIdx.x;
  if (status[z] != kOK) return;
  const int M = Mz[z];
  if (a > M - 3) return;
  SliceTables t{C + (size_t)z * E, Whi + (size_t)z * E, Wlo + (size_t)z * E, nullptr};
  const double *as = Asuf + (size_t)z * L;
  double *row = R + ((size_t)z * L + a) * L;
  for (int b = a + 1 + threadIdx.x; b <= M - 2; b += blockDim.x)
    row[b] = combine<MODE>(class_term<MODE>(t, luts, a + 1, b), __ldg(as + b));
}

// ================================================================ a3: search
struct SearchArgs {
  const uint32_t *C;
  const double *Whi, *Wlo, *Asuf, *R;
  const int32_t *Bin, *Mz, *status;
  double *part_score;  // [nunits][nz]
  uint64_t *part_key;
  Luts luts;
  int64_t nz;
  int E, L, units, unit_begin;
};

// Exhaustive search.  The tuple space of slice z is enumerated as "rows": a
// row is a lex-ranked (k-1)-combination (t_1..t_{k-1}) of positions [0, M-2];
// its tuples are t_k = b in (t_{k-1}, M-2].  Unit u of U covers rows
// [NR*u/U, NR*(u+1)/U).  Warps take rows round-robin, lanes take b with stride
// 32, so every lane visits its tuples in increasing lex order and a strict '>'
// keeps the lowest tuple among equal scores.  Value of a tuple:
//   Pre = T(0,t_1) x T(t_1+1,t_2) x ... x T(t_{k-2}+1, t_{k-1})   (left fold)
//   v   = Pre x R(t_{k-1}, t_k),  R(a,b) = T(a+1,b) x T(b+1,M-1)
// (x = * or +; sum-plus-product keeps (sum, prod) pairs), one expression tree
// for every tuple.
template <int K, int MODE, bool RT>
__global__ void __launch_bounds__(256) k_search(SearchArgs g) {
  const int z = blockIdx.y;
  const int u = g.unit_begin + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double best = -CUDART_INF;
  uint64_t brow = 0;
  int bb = -1;
  const int st = g.status[z];
  const int M = g.Mz[z];
  const int P = M - 1;  // positions 0..M-2
  SliceTables t{g.C + (size_t)z * g.E, g.Whi + (size_t)z * g.E, g.Wlo + (size_t)z * g.E,
                g.Asuf + (size_t)z * g.L};
  int idx[kKMax];
  if (st == kOK && P >= K) {
    const uint64_t NR = binom((uint64_t)P, K - 1);
    const uint64_t r0 = NR * (uint64_t)u / (uint64_t)g.units;
    const uint64_t r1 = NR * (uint64_t)(u + 1) / (uint64_t)g.units;
    uint64_t r = r0 + warp;
    if (r < r1) {
      if (K > 1) unrank_comb<(K > 1 ? K - 1 : 1)>(r, P, idx);
      for (; r < r1; r += nw) {
        const int a = K > 1 ? idx[K - 2] : -1;
        if (a <= M - 3) {
          if (MODE == SPP) {
            double sum = 0.0, prod = 1.0;
            int lo = 0;
#pragma unroll
            for (int j = 0; j < K - 1; j++) {
              const double s = class_term<MODE>(t, g.luts, lo, idx[j]);
              sum = __dadd_rn(sum, s);
              prod = __dmul_rn(prod, s);
              lo = idx[j] + 1;
            }
            for (int b = a + 1 + lane; b <= M - 2; b += 32) {
              const double s1 = class_term<MODE>(t, g.luts, a + 1, b);
              const double s2 = __ldg(t.Asuf + b);
              const double v = __dadd_rn(__dadd_rn(sum, __dadd_rn(s1, s2)),
                                         __dmul_rn(g.luts.omq, __dmul_rn(prod, __dmul_rn(s1, s2))));
              if (v > best) {
                best = v;
                brow = r;
                bb = b;
              }
            }
          } else {
            double pre = MODE == SUM ? 0.0 : 1.0;
            int lo = 0;
#pragma unroll
            for (int j = 0; j < K - 1; j++) {
              pre = combine<MODE>(pre, class_term<MODE>(t, g.luts, lo, idx[j]));
              lo = idx[j] + 1;
            }
            constexpr bool kRT = RT && K >= 3;
            const double *Rrow = kRT ? g.R + ((size_t)z * g.L + (size_t)a) * g.L : nullptr;
            for (int b = a + 1 + lane; b <= M - 2; b += 32) {
              const double R = kRT ? __ldg(Rrow + b)
                                  : combine<MODE>(class_term<MODE>(t, g.luts, a + 1, b),
                                                  __ldg(t.Asuf + b));
              double v = combine<MODE>(pre, R);
              if (MODE == PROD_MIN) v = -v;
              if (v > best) {
                best = v;
                brow = r;
                bb = b;
              }
            }
          }
        }
        if (K > 1) {
          bool ok = true;
          for (int s = 0; s < nw && ok; s++) ok = next_comb<(K > 1 ? K - 1 : 1)>(idx, P);
          if (!ok) break;
        }
      }
    }
  }
  // key of the lane's best tuple
  uint64_t key = kKeyNone;
  if (bb >= 0) {
    if (K > 1) unrank_comb<(K > 1 ? K - 1 : 1)>(brow, P, idx);
    const int32_t *bin = g.Bin + (size_t)z * g.E;
    key = 0;
#pragma unroll
    for (int j = 0; j < K - 1; j++) key = (key << 12) | (uint64_t)__ldg(bin + idx[j] + 1);
    key = (key << 12) | (uint64_t)__ldg(bin + bb + 1);
  }
  warp_argmax(best, key);
  __shared__ double ss[32];
  __shared__ uint64_t sk[32];
  if (lane == 0) {
    ss[warp] = best;
    sk[warp] = key;
  }
  __syncthreads();
  if (warp == 0) {
    best = lane < nw ? ss[lane] : -CUDART_INF;
    key = lane < nw ? sk[lane] : kKeyNone;
    warp_argmax(best, key);
    if (lane == 0) {
      g.part_score[(size_t)blockIdx.x * g.nz + z] = best;
      g.part_key[(size_t)blockIdx.x * g.nz + z] = key;
    }
  }
}

// ================================================================ a4: argmax
__global__ void k_merge(const double *ps, const uint64_t *pk, int nparts, int64_t nz,
                        double *s_out, uint64_t *k_out) {
  const int64_t z = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (z >= nz) return;
  double s = -CUDART_INF;
  uint64_t k = kKeyNone;
  for (int p = lane; p < nparts; p += 32) {
    const double os = ps[(size_t)p * nz + z];
    const uint64_t ok = pk[(size_t)p * nz + z];
    if (better(os, ok, s, k)) {
      s = os;
      k = ok;
    }
  }
  warp_argmax(s, k);
  if (lane == 0) {
    s_out[z] = s;
    k_out[z] = k;
  }
}

struct FinalizeArgs {
  const uint32_t *hist;
  const int32_t *status_in;
  const double *ps;
  const uint64_t *pk;
  int nparts;
  int64_t nz;
  int L, k, objective;
  double q;
  int32_t *thresholds;
  double *objective_out;
  int32_t *status_out;
};

// One warp per slice: merge the partials, decode t*, and recompute phi(t*) in
// the definition's order (sequential ascending sums of p_i = c_i/N, P_j and
// (p_i/P_j)^q, then the left-to-right fold) so the reported objective agrees
// with the definition to ~1e-16 regardless of how the search scored tuples.
// The pow/log terms run lane-parallel; the sums are sequential on lane 0.
__global__ void __launch_bounds__(32) k_finalize(FinalizeArgs g) {
  extern __shared__ double term[];  // [L]
  const int64_t z = blockIdx.x;
  const int lane = threadIdx.x;
  double s = -CUDART_INF;
  uint64_t key = kKeyNone;
  for (int p = lane; p < g.nparts; p += 32) {
    const double os = g.ps[(size_t)p * g.nz + z];
    const uint64_t ok = g.pk[(size_t)p * g.nz + z];
    if (better(os, ok, s, key)) {
      s = os;
      key = ok;
    }
  }
  warp_argmax(s, key);
  int st = g.status_in[z];
  if (st == kOK && key == kKeyNone) st = kNoValidSplit;
  const int k = g.k, L = g.L;
  if (st != kOK) {
    if (lane < k) g.thresholds[z * k + lane] = -1;
    if (lane == 0) {
      if (g.objective_out) g.objective_out[z] = CUDART_NAN;
      if (g.status_out) g.status_out[z] = st;
    }
    return;
  }
  int t[kKMax + 1];
  for (int j = 0; j < k; j++) t[j] = (int)((key >> (12 * (k - 1 - j))) & 0xFFFull);
  if (lane < k) g.thresholds[z * k + lane] = t[lane];
  if (!g.objective_out && !g.status_out) return;
  const uint32_t *h = g.hist + z * L;
  const double q = g.q;
  const int shannon = q == 1.0;
  __shared__ double Pc[kKMax + 1];
  __shared__ double Nsh;
  if (lane == 0) {
    double N = 0.0;
    for (int i = 0; i < L; i++) N = __dadd_rn(N, (double)h[i]);
    Nsh = N;
    int lo = 0;
    for (int j = 0; j <= k; j++) {
      const int hi = j < k ? t[j] : L - 1;
      double P = 0.0;
      for (int i = lo; i <= hi; i++) {
        const uint32_t c = h[i];
        if (c) P = __dadd_rn(P, __ddiv_rn((double)c, N));
      }
      Pc[j] = P;
      lo = hi + 1;
    }
  }
  __syncwarp();
  const double N = Nsh;
  // class of bin i
  for (int i = lane; i < L; i += 32) {
    const uint32_t c = h[i];
    double v = 0.0;
    if (c) {
      int j = 0;
      while (j < k && i > t[j]) j++;
      const double r = __ddiv_rn(__ddiv_rn((double)c, N), Pc[j]);
      v = shannon ? __dmul_rn(r, log(r)) : pow(r, q);
    }
    term[i] = v;
  }
  __syncwarp();
  if (lane == 0) {
    double S[kKMax + 1];
    int lo = 0;
    for (int j = 0; j <= k; j++) {
      const int hi = j < k ? t[j] : L - 1;
      double A = 0.0;
      for (int i = lo; i <= hi; i++)
        if (h[i]) A = shannon ? __dsub_rn(A, term[i]) : __dadd_rn(A, term[i]);
      S[j] = shannon ? A : __ddiv_rn(__dsub_rn(1.0, A), __dsub_rn(q, 1.0));
      lo = hi + 1;
    }
    double phi;
    if (g.objective == 1) {
      double sum = 0.0, prod = 1.0;
      for (int j = 0; j <= k; j++) sum = __dadd_rn(sum, S[j]);
      for (int j = 0; j <= k; j++) prod = __dmul_rn(prod, S[j]);
      phi = __dadd_rn(sum, __dmul_rn(__dsub_rn(1.0, q), prod));
    } else {
      phi = S[0];
      for (int j = 1; j <= k; j++)
        phi = __dadd_rn(__dadd_rn(phi, S[j]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, q), phi), S[j]));
    }
    if (g.objective_out) g.objective_out[z] = phi;
    if (g.status_out) g.status_out[z] = kOK;
  }
}

// ================================================================ a5: labels
// label(v) = #{j : v > t_j}.  u8: SWAR -- one __vcmpgtu4 per threshold per 4
// voxels, 16-byte loads and stores.  u16: 8 voxels per 16-byte load.
struct LabelArgs {
  const uint8_t *vol;
  uint8_t *labels;
  const int32_t *thr;     // [nz][k]
  const int32_t *status;  // [nz] or null
  int64_t n;              // voxels per slice
  int k;
  int chunks;
};

template <typename T>
__global__ void __launch_bounds__(256) k_label(LabelArgs g) {
  const int z = blockIdx.y;
  const T *slice = reinterpret_cast<const T *>(g.vol) + (size_t)z * g.n;
  uint8_t *out = g.labels + (size_t)z * g.n;
  const bool ok = g.status == nullptr || g.status[z] == kOK;
  int t[kKMax] = {0, 0, 0, 0};
  for (int j = 0; j < g.k; j++) t[j] = g.thr[z * g.k + j];
  // element range of this CTA: multiples of 16 elements
  const int64_t n16 = g.n / 16;
  const int64_t per = (n16 + g.chunks - 1) / g.chunks;
  const int64_t c0 = per * blockIdx.x, c1 = min(n16, c0 + per);
  const bool aligned = ((reinterpret_cast<uintptr_t>(slice) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (aligned) {
    if (sizeof(T) == 1) {
      uint32_t tb[kKMax];
      for (int j = 0; j < kKMax; j++) tb[j] = (uint32_t)(t[j] & 0xff) * 0x01010101u;
      const uint4 *src = reinterpret_cast<const uint4 *>(slice);
      uint4 *dst = reinterpret_cast<uint4 *>(out);
      for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
        const uint4 w = __ldcs(src + i);
        uint4 o = {0u, 0u, 0u, 0u};
        if (ok) {
          for (int j = 0; j < g.k; j++) {
            o.x += __vcmpgtu4(w.x, tb[j]) & 0x01010101u;
            o.y += __vcmpgtu4(w.y, tb[j]) & 0x01010101u;
            o.z += __vcmpgtu4(w.z, tb[j]) & 0x01010101u;
            o.w += __vcmpgtu4(w.w, tb[j]) & 0x01010101u;
          }
        }
        __stcs(dst + i, o);
      }
    } else {
      const uint4 *src = reinterpret_cast<const uint4 *>(slice);
      uint2 *dst = reinterpret_cast<uint2 *>(out);
      for (int64_t i = 2 * c0 + threadIdx.x; i < 2 * c1; i += blockDim.x) {
        const uint4 w = __ldcs(src + i);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        uint32_t o[2] = {0u, 0u};
        if (ok) {
#pragma unroll
          for (int e = 0; e < 8; e++) {
            const int v = (int)((ws[e >> 1] >> (16 * (e & 1))) & 0xffffu);
            uint32_t l = 0;
            for (int j = 0; j < g.k; j++) l += v > t[j];
            o[e >> 2] |= l << (8 * (e & 3));
          }
        }
        __stcs(dst + i, make_uint2(o[0], o[1]));
      }
    }
  } else {
    for (int64_t i = c0 * 16 + threadIdx.x; i < c1 * 16; i += blockDim.x) {
      const int v = (int)slice[i];
      uint32_t l = 0;
      if (ok)
        for (int j = 0; j < g.k; j++) l += v > t[j];
      out[i] = (uint8_t)l;
    }
  }
  if (blockIdx.x == gridDim.x - 1) {
    for (int64_t i = n16 * 16 + threadIdx.x; i < g.n; i += blockDim.x) {
      const int v = (int)slice[i];
      uint32_t l = 0;
      if (ok)
        for (int j = 0; j < g.k; j++) l += v > t[j];
      out[i] = (uint8_t)l;
    }
  }
}

}  // namespace tsa
