// k_search.cuh -- SURVEY.md §8 row a3: exhaustive search over ordered
// threshold tuples t_1 < ... < t_k maximising the pseudo-additive Tsallis
// objective (folded over k+1 classes, R1), fp64,
// with a deterministic lowest-tuple tie-break (R8).
//
// Enumeration.  The tuple space of slice z (positions [0, M-2] of its table,
// M = non-empty bins for CANONICAL, L for FULL) is split into "rows": a row is
// a lex-ranked (k-1)-combination (t_1..t_{k-1}) and holds the tuples
// (t_1..t_{k-1}, b), b in (t_{k-1}, M-2].  Unit u of U covers rows
// [NR*u/U, NR*(u+1)/U) (NR = C(M-1, k-1)), a rank-independent partition, so
// disjoint unit ranges on different GPUs partition the tuple space.  Warps
// take rows round-robin (successor stepping, unranked once), lanes take b
// with stride 32: every lane visits its tuples in increasing lex order and a
// strict '>' keeps its lowest tuple among equal scores; the cross-lane,
// cross-warp, cross-CTA and cross-rank merges use the total order
// (score desc, key asc), so the result is independent of the partition.
//
// Value of a tuple (one expression tree for every tuple, explicit _rn ops):
//   Pre = T(0,t_1) x T(t_1+1,t_2) x ... x T(t_{k-2}+1, t_{k-1})   (left fold)
//   v   = Pre x R(t_{k-1}, b),  R(a,b) = T(a+1,b) x T(b+1,M-1)
// with x = * (pseudo-additive, score = +-v) or + (q == 1), and (sum, prod)
// pairs for sum-plus-product.  R comes from the k_rtable table when present.
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

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

// STAGE: copy the slice's C/W/Asuf tables to shared memory first (L <= 1024).
template <int K, int MODE, bool RT, bool STAGE>
__global__ void __launch_bounds__(256) k_search(SearchArgs g) {
  extern __shared__ double ssh[];
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
  if (STAGE && st == kOK) {
    double *sWhi = ssh, *sWlo = ssh + g.E, *sAsuf = ssh + 2 * g.E;
    uint32_t *sC = reinterpret_cast<uint32_t *>(ssh + 2 * g.E + g.L);
    for (int i = threadIdx.x; i <= M; i += blockDim.x) {
      sWhi[i] = t.Whi[i];
      sWlo[i] = t.Wlo[i];
      sC[i] = t.C[i];
      if (i <= M - 2) sAsuf[i] = t.Asuf[i];
    }
    __syncthreads();
    t = SliceTables{sC, sWhi, sWlo, sAsuf};
  }
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
              const double s2 = t.Asuf[b];
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
                                   : combine<MODE>(class_term<MODE>(t, g.luts, a + 1, b), t.Asuf[b]);
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

}  // namespace tsa
