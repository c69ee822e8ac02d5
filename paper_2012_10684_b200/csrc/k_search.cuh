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
  const double *PP, *AI;  // k >= 3 prefix tables (k_rtable): PP[x][y] = T(0,x) (x) T(x+1,y), AI[x][y] = T(x,y)
  const int32_t *Bin, *Mz, *status;
  int32_t *counter;    // dynamic item counter (k >= 3 rows kernel, k = 2 block kernel), zeroed before launch
  const int32_t *mmax; // max over slices of M (k_scan), k = 2 block kernel
  double *item_score;  // [nbmax][nz] per-(a-block, slice) partials of the k = 2 block kernel
  uint64_t *item_key;
  const K2Row *rows;   // [nz][RE] packed positions (k_scan) for the k = 2 block kernel
  int RE;
  double *part_score;  // [nunits][nz]
  uint64_t *part_key;
  Luts luts;
  int64_t nz;
  int E, L, RS, units, unit_begin;  // RS: R-table row stride (>= L + 8, even)
  int nunits;                        // units in this launch (unit_end - unit_begin)
  int ss;                            // k_search_tri: CTA entries per slice
  int32_t *ccur;                     // k_search_tri: [nz] per-slice chunk counters, zeroed
  double *seed;                      // [nz] seed scores of the pruned k = 2 search (k_k2_seed)
  K2Chk *chk;                        // [2][nz][RE] bound records of the pruned k = 2 search (k_k2_seed)
  int64_t TS;                        // k_tri_tables / k_search_tri: doubles per slice region (tri_slice_stride)
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
            const double *Rrow = kRT ? g.R + ((size_t)z * g.L + (size_t)a) * g.RS : nullptr;
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

namespace tsa {

// Colex unranking of an R-combination (R = 2 or 3): the combination of rank r
// in colexicographic order (last element major).  Closed-form estimate plus
// exact integer correction.
template <int R>
__device__ __forceinline__ void unrank_colex(uint64_t r, int *idx) {
  if (R == 1) {
    idx[0] = (int)r;
    return;
  }
  if (R == 2) {
    int a = (int)((1.0 + sqrt(1.0 + 8.0 * (double)r)) * 0.5);
    while (a > 1 && binom((uint64_t)a, 2) > r) a--;
    while (binom((uint64_t)a + 1, 2) <= r) a++;
    idx[1] = a;
    idx[0] = (int)(r - binom((uint64_t)a, 2));
    return;
  }
  // R == 3
  int a = (int)cbrt(6.0 * (double)r) + 1;
  while (a > 2 && binom((uint64_t)a, 3) > r) a--;
  while (binom((uint64_t)a + 1, 3) <= r) a++;
  idx[2] = a;
  r -= binom((uint64_t)a, 3);
  int b = (int)((1.0 + sqrt(1.0 + 8.0 * (double)r)) * 0.5);
  while (b > 1 && binom((uint64_t)b, 2) > r) b--;
  while (binom((uint64_t)b + 1, 2) <= r) b++;
  idx[1] = b;
  idx[0] = (int)(r - binom((uint64_t)b, 2));
}

// hit |= any(pre (x) r_i >= best) over 4 columns, as 4 DMUL/DADD + 4 setp.ge.or
// into one predicate (2 FP64-pipe instructions per tuple; the compiler would
// otherwise turn the OR of compares into a DSETP.MAX chain).
template <int MODE>
__device__ __forceinline__ unsigned cmp4(unsigned hit, double pre, double2 x, double2 y, double best) {
  if (MODE == SUM) {
    asm("{\n\t.reg .pred p;\n\t.reg .f64 t0, t1, t2, t3;\n\t"
        "setp.ne.u32 p, %0, 0;\n\t"
        "add.rn.f64 t0, %1, %2;\n\tadd.rn.f64 t1, %1, %3;\n\t"
        "add.rn.f64 t2, %1, %4;\n\tadd.rn.f64 t3, %1, %5;\n\t"
        "setp.ge.or.f64 p, t0, %6, p;\n\tsetp.ge.or.f64 p, t1, %6, p;\n\t"
        "setp.ge.or.f64 p, t2, %6, p;\n\tsetp.ge.or.f64 p, t3, %6, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "+r"(hit)
        : "d"(pre), "d"(x.x), "d"(x.y), "d"(y.x), "d"(y.y), "d"(best));
  } else {
    asm("{\n\t.reg .pred p;\n\t.reg .f64 t0, t1, t2, t3;\n\t"
        "setp.ne.u32 p, %0, 0;\n\t"
        "mul.rn.f64 t0, %1, %2;\n\tmul.rn.f64 t1, %1, %3;\n\t"
        "mul.rn.f64 t2, %1, %4;\n\tmul.rn.f64 t3, %1, %5;\n\t"
        "setp.ge.or.f64 p, t0, %6, p;\n\tsetp.ge.or.f64 p, t1, %6, p;\n\t"
        "setp.ge.or.f64 p, t2, %6, p;\n\tsetp.ge.or.f64 p, t3, %6, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "+r"(hit)
        : "d"(pre), "d"(x.x), "d"(x.y), "d"(y.x), "d"(y.y), "d"(best));
  }
  return hit;
}

// hit |= any(pre (x) x_i >= best) over 8 columns: 8 DMUL/DADD and 8 DSETP into
// independent predicates (no serial predicate chain), OR-ed by a PLOP3 tree.
template <int MODE>
__device__ __forceinline__ unsigned cmp8(unsigned hit, double pre, double2 x0, double2 x1, double2 x2,
                                         double2 x3, double best) {
#define TSA_CMP8_BODY(OP)                                                                        \
  asm("{\n\t.reg .pred p0, p1, p2, p3, p4, p5, p6, p7, ph;\n\t"                                  \
      ".reg .f64 t0, t1, t2, t3, t4, t5, t6, t7;\n\t" OP " t0, %1, %2;\n\t" OP " t1, %1, %3;\n\t" \
      OP " t2, %1, %4;\n\t" OP " t3, %1, %5;\n\t" OP " t4, %1, %6;\n\t" OP " t5, %1, %7;\n\t"     \
      OP " t6, %1, %8;\n\t" OP " t7, %1, %9;\n\t"                                                 \
      "setp.ge.f64 p0, t0, %10;\n\tsetp.ge.f64 p1, t1, %10;\n\t"                                  \
      "setp.ge.f64 p2, t2, %10;\n\tsetp.ge.f64 p3, t3, %10;\n\t"                                  \
      "setp.ge.f64 p4, t4, %10;\n\tsetp.ge.f64 p5, t5, %10;\n\t"                                  \
      "setp.ge.f64 p6, t6, %10;\n\tsetp.ge.f64 p7, t7, %10;\n\t"                                  \
      "setp.ne.u32 ph, %0, 0;\n\t"                                                                \
      "or.pred p0, p0, p1;\n\tor.pred p2, p2, p3;\n\tor.pred p4, p4, p5;\n\t"                     \
      "or.pred p6, p6, p7;\n\tor.pred p0, p0, p2;\n\tor.pred p4, p4, p6;\n\t"                     \
      "or.pred p0, p0, p4;\n\tor.pred p0, p0, ph;\n\t"                                            \
      "selp.u32 %0, 1, 0, p0;\n\t}"                                                               \
      : "+r"(hit)                                                                                 \
      : "d"(pre), "d"(x0.x), "d"(x0.y), "d"(x1.x), "d"(x1.y), "d"(x2.x), "d"(x2.y), "d"(x3.x),    \
        "d"(x3.y), "d"(best))
  if (MODE == SUM) {
    TSA_CMP8_BODY("add.rn.f64");
  } else {
    TSA_CMP8_BODY("mul.rn.f64");
  }
#undef TSA_CMP8_BODY
  return hit;
}

// Two prefixes against the same 8 columns: 16 DMUL/DADD + 16 DSETP into
// independent predicates, one PLOP3 tree (the column loads are shared).
template <int MODE>
__device__ __forceinline__ unsigned cmp8x2(unsigned hit, double p0, double p1, double2 x0, double2 x1,
                                           double2 x2, double2 x3, double best) {
#define TSA_CMP16_BODY(OP)                                                                        \
  asm("{\n\t.reg .pred q0, q1, q2, q3, q4, q5, q6, q7, q8, q9, q10, q11, q12, q13, q14, q15, qh;\n\t" \
      ".reg .f64 t0, t1, t2, t3, t4, t5, t6, t7, u0, u1, u2, u3, u4, u5, u6, u7;\n\t"               \
      OP " t0, %1, %3;\n\t" OP " t1, %1, %4;\n\t" OP " t2, %1, %5;\n\t" OP " t3, %1, %6;\n\t"        \
      OP " t4, %1, %7;\n\t" OP " t5, %1, %8;\n\t" OP " t6, %1, %9;\n\t" OP " t7, %1, %10;\n\t"       \
      OP " u0, %2, %3;\n\t" OP " u1, %2, %4;\n\t" OP " u2, %2, %5;\n\t" OP " u3, %2, %6;\n\t"        \
      OP " u4, %2, %7;\n\t" OP " u5, %2, %8;\n\t" OP " u6, %2, %9;\n\t" OP " u7, %2, %10;\n\t"       \
      "setp.ge.f64 q0, t0, %11;\n\tsetp.ge.f64 q1, t1, %11;\n\tsetp.ge.f64 q2, t2, %11;\n\t"        \
      "setp.ge.f64 q3, t3, %11;\n\tsetp.ge.f64 q4, t4, %11;\n\tsetp.ge.f64 q5, t5, %11;\n\t"        \
      "setp.ge.f64 q6, t6, %11;\n\tsetp.ge.f64 q7, t7, %11;\n\tsetp.ge.f64 q8, u0, %11;\n\t"        \
      "setp.ge.f64 q9, u1, %11;\n\tsetp.ge.f64 q10, u2, %11;\n\tsetp.ge.f64 q11, u3, %11;\n\t"      \
      "setp.ge.f64 q12, u4, %11;\n\tsetp.ge.f64 q13, u5, %11;\n\tsetp.ge.f64 q14, u6, %11;\n\t"     \
      "setp.ge.f64 q15, u7, %11;\n\tsetp.ne.u32 qh, %0, 0;\n\t"                                     \
      "or.pred q0, q0, q1;\n\tor.pred q2, q2, q3;\n\tor.pred q4, q4, q5;\n\tor.pred q6, q6, q7;\n\t"  \
      "or.pred q8, q8, q9;\n\tor.pred q10, q10, q11;\n\tor.pred q12, q12, q13;\n\t"                  \
      "or.pred q14, q14, q15;\n\tor.pred q0, q0, q2;\n\tor.pred q4, q4, q6;\n\t"                     \
      "or.pred q8, q8, q10;\n\tor.pred q12, q12, q14;\n\tor.pred q0, q0, q4;\n\t"                    \
      "or.pred q8, q8, q12;\n\tor.pred q0, q0, q8;\n\tor.pred q0, q0, qh;\n\t"                       \
      "selp.u32 %0, 1, 0, q0;\n\t}"                                                                 \
      : "+r"(hit)                                                                                  \
      : "d"(p0), "d"(p1), "d"(x0.x), "d"(x0.y), "d"(x1.x), "d"(x1.y), "d"(x2.x), "d"(x2.y),          \
        "d"(x3.x), "d"(x3.y), "d"(best))
  if (MODE == SUM) {
    TSA_CMP16_BODY("add.rn.f64");
  } else {
    TSA_CMP16_BODY("mul.rn.f64");
  }
#undef TSA_CMP16_BODY
  return hit;
}

// Colex successor of an R-combination (no upper bound check: callers bound
// the rank range).
template <int R>
__device__ __forceinline__ void next_colex(int *idx) {
  // explicit per R (a loop with an early return kept idx[] in local memory)
  if (R == 1) {
    idx[0]++;
  } else if (R == 2) {
    if (idx[0] + 1 < idx[1]) {
      idx[0]++;
    } else {
      idx[1]++;
      idx[0] = 0;
    }
  } else {
    if (idx[0] + 1 < idx[1]) {
      idx[0]++;
    } else if (idx[1] + 1 < idx[2]) {
      idx[1]++;
      idx[0] = 0;
    } else {
      idx[2]++;
      idx[0] = 0;
      idx[1] = 1;
    }
  }
}

// One row of the k >= 3 search: tuples (prefix, b), b in (a, M-2], value
// pre (x) R[a][b].  Fast path: 8 columns per step, 2 FP64 instructions per
// tuple (DMUL + DSETP.GE.OR into one predicate), next group's loads in flight
// while the current one is compared.  Only if some value >= best is the row
// rescanned under the exact (score, key) order.
// 16-byte row loads: read-only cache path (global tables) or generic (tables
// in shared memory, k_search_tri)
template <bool NC>
__device__ __forceinline__ double2 ldrow(const double2 *p) {
  if (NC) return __ldg(p);
  return *p;
}

template <int MODE, int R, bool NC = true>
__device__ __forceinline__ void search_row(const double *row, int a, int M, double pre, const int *idx,
                                           const int32_t *bin, double &best, uint64_t &bestkey) {
  // columns [a+1, M-2]; entries outside are NaN, so 8-column groups from the
  // even column at or below a+1 need no bounds checks (row stride RS >= L+8)
  const double2 *rp = reinterpret_cast<const double2 *>(row + ((a + 1) & ~1));
  int ng = (M - 1 - ((a + 1) & ~1) + 7) >> 3;  // 8-column groups (>= 1)
  unsigned hit = 0;
  // two register buffers alternate (no copies): loads of group g+1 are in
  // flight while group g is compared
  double2 x0 = ldrow<NC>(rp), x1 = ldrow<NC>(rp + 1), x2 = ldrow<NC>(rp + 2), x3 = ldrow<NC>(rp + 3);
  double2 y0, y1, y2, y3;
  for (;;) {
    if (ng > 1) {
      y0 = ldrow<NC>(rp + 4);
      y1 = ldrow<NC>(rp + 5);
      y2 = ldrow<NC>(rp + 6);
      y3 = ldrow<NC>(rp + 7);
    }
    hit = cmp8<MODE>(hit, pre, x0, x1, x2, x3, best);
    if (--ng == 0) break;
    rp += 4;
    if (ng > 1) {
      x0 = ldrow<NC>(rp + 4);
      x1 = ldrow<NC>(rp + 5);
      x2 = ldrow<NC>(rp + 6);
      x3 = ldrow<NC>(rp + 7);
    }
    hit = cmp8<MODE>(hit, pre, y0, y1, y2, y3, best);
    if (--ng == 0) break;
    rp += 4;
  }
  if (hit) {
    uint64_t kp = 0;
#pragma unroll
    for (int j = 0; j < R; j++) kp = (kp << 12) | (uint64_t)bin[idx[j] + 1];
    for (int b = a + 1; b <= M - 2; b++) {
      const double v = combine<MODE>(pre, row[b]);
      if (v >= best) {
        const uint64_t key = (kp << 12) | (uint64_t)bin[b + 1];
        if (better(v, key, best, bestkey)) {
          best = v;
          bestkey = key;
        }
      }
    }
  }
}

// Two rows sharing a (consecutive colex ranks): the 8-column loads serve both.
template <int MODE, int R, bool NC = true>
__device__ __forceinline__ void search_row2(const double *row, int a, int M, double pre0, double pre1,
                                            const int *idx0, const int *idx1, const int32_t *bin,
                                            double &best, uint64_t &bestkey) {
  const double2 *rp = reinterpret_cast<const double2 *>(row + ((a + 1) & ~1));
  int ng = (M - 1 - ((a + 1) & ~1) + 7) >> 3;
  unsigned hit = 0;
  double2 x0 = ldrow<NC>(rp), x1 = ldrow<NC>(rp + 1), x2 = ldrow<NC>(rp + 2), x3 = ldrow<NC>(rp + 3);
  double2 y0, y1, y2, y3;
  for (;;) {
    if (ng > 1) {
      y0 = ldrow<NC>(rp + 4);
      y1 = ldrow<NC>(rp + 5);
      y2 = ldrow<NC>(rp + 6);
      y3 = ldrow<NC>(rp + 7);
    }
    hit = cmp8x2<MODE>(hit, pre0, pre1, x0, x1, x2, x3, best);
    if (--ng == 0) break;
    rp += 4;
    if (ng > 1) {
      x0 = ldrow<NC>(rp + 4);
      x1 = ldrow<NC>(rp + 5);
      x2 = ldrow<NC>(rp + 6);
      x3 = ldrow<NC>(rp + 7);
    }
    hit = cmp8x2<MODE>(hit, pre0, pre1, y0, y1, y2, y3, best);
    if (--ng == 0) break;
    rp += 4;
  }
  if (hit) {  // exact rescan, lower-lex row first
    for (int which = 0; which < 2; which++) {
      const int *idx = which == 0 ? idx0 : idx1;
      const double pre = which == 0 ? pre0 : pre1;
      uint64_t kp = 0;
#pragma unroll
      for (int j = 0; j < R; j++) kp = (kp << 12) | (uint64_t)bin[idx[j] + 1];
      for (int b = a + 1; b <= M - 2; b++) {
        const double v = combine<MODE>(pre, row[b]);
        if (v >= best) {
          const uint64_t key = (kp << 12) | (uint64_t)bin[b + 1];
          if (better(v, key, best, bestkey)) {
            best = v;
            bestkey = key;
          }
        }
      }
    }
  }
}

__device__ __forceinline__ void block_argmax(double &best, uint64_t &key) {
  __shared__ double ss[32];
  __shared__ uint64_t sk[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  warp_argmax(best, key);
  __syncthreads();  // previous users of ss/sk are done
  if (lane == 0) {
    ss[warp] = best;
    sk[warp] = key;
  }
  __syncthreads();
  best = lane < nw ? ss[lane] : -CUDART_INF;
  key = lane < nw ? sk[lane] : kKeyNone;
  warp_argmax(best, key);  // every warp reduces the same values: all threads agree
}

// Exhaustive search for k >= 3 with the R/PP/AI tables (pseudo-additive, q != 1
// or q == 1).  Persistent: CTA b handles work items (slice z, unit u) b, b+G,
// ...; in an item each thread walks CH consecutive colex rows (prefixes ending
// at a = t_{k-1}; unrank once, then successor), so the 32*CH rows of a warp
// share a and read the same R row (L1 broadcast).  Pre comes from the tables
// (no class-term gathers).  After every thread's first chunk the CTA's best so
// far seeds all threads, so later rows rarely need the exact rescan.
template <int K, int MODE>
__global__ void __launch_bounds__(256, 3) k_search_rows(SearchArgs g) {
  static_assert(K >= 3 && K <= 4, "rows kernel is for k = 3, 4");
  constexpr int R = K - 1;
  constexpr int CH = 8;
  const int64_t items = g.nz * (int64_t)g.nunits;
  __shared__ int s_item;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(g.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= items) break;
    const int z = (int)(item / g.nunits);
    const int ul = (int)(item % g.nunits);
    const int u = g.unit_begin + ul;
    double best = -CUDART_INF;
    uint64_t bestkey = kKeyNone;
    const int st = g.status[z];
    const int M = g.Mz[z];
    const int P = M - 1;
    const int32_t *bin = g.Bin + (size_t)z * g.E;
    const bool active = st == kOK && P >= K;
    uint64_t r0 = 0, r1 = 0;
    if (active) {
      const uint64_t NR = binom((uint64_t)P, R);
      r0 = NR * (uint64_t)u / (uint64_t)g.units;
      r1 = NR * (uint64_t)(u + 1) / (uint64_t)g.units;
    }
    const double *PPz = g.PP + (size_t)z * g.L * g.RS;
    const double *AIz = K == 4 ? g.AI + (size_t)z * g.L * g.RS : nullptr;
    const double *Rz = g.R + (size_t)z * g.L * g.RS;
    // uniform chunk count for the CTA: after every chunk the CTA's best so far
    // is shared (one block reduction per 4 rows per thread), so a thread only
    // rescans a row that may beat the best any thread has seen
    const uint64_t span = (uint64_t)blockDim.x * CH;
    const uint64_t nchunks = r1 > r0 ? (r1 - r0 + span - 1) / span : 0;
    for (uint64_t ci = 0; ci < nchunks; ci++) {
      const uint64_t rb = r0 + ci * span + (uint64_t)threadIdx.x * CH;
      if (rb < r1) {
        int idx[R];
        unrank_colex<R>(rb, idx);
        const uint64_t re_ = min(r1, rb + CH);
        // software pipeline across rows: the next row's Pre loads are issued
        // before the current row's compare loop
        auto pre_of = [&](const int *id) -> double {
          const double p = K == 3 ? __ldg(PPz + (size_t)id[0] * g.RS + id[R - 1])
                                  : combine<MODE>(__ldg(PPz + (size_t)id[0] * g.RS + id[1]),
                                                  __ldg(AIz + (size_t)(id[1] + 1) * g.RS + id[R - 1]));
          return MODE == PROD_MIN ? -p : p;  // (-pre)*R == -(pre*R) exactly
        };
        for (uint64_t r = rb; r < re_;) {
          int nidx[R];
#pragma unroll
          for (int j = 0; j < R; j++) nidx[j] = idx[j];
          next_colex<R>(nidx);
          const int a = idx[R - 1];
          // Pre = (1 (x) T(0,t1)) (x) T(t1+1,t2) [(x) T(t2+1,a)] from the tables
          if (r + 1 < re_ && nidx[R - 1] == a && a <= M - 3) {
            search_row2<MODE, R>(Rz + (size_t)a * g.RS, a, M, pre_of(idx), pre_of(nidx), idx, nidx, bin,
                                 best, bestkey);
#pragma unroll
            for (int j = 0; j < R; j++) idx[j] = nidx[j];
            next_colex<R>(idx);
            r += 2;
          } else {
            if (a <= M - 3) search_row<MODE, R>(Rz + (size_t)a * g.RS, a, M, pre_of(idx), idx, bin, best, bestkey);
#pragma unroll
            for (int j = 0; j < R; j++) idx[j] = nidx[j];
            r += 1;
          }
        }
      }
      block_argmax(best, bestkey);
    }
    block_argmax(best, bestkey);
    if (threadIdx.x == 0) {
      g.part_score[(size_t)ul * g.nz + z] = best;
      g.part_key[(size_t)ul * g.nz + z] = bestkey;
    }
  }
}

// k_search_tri helpers (see the kernel below)
__device__ __forceinline__ int tri_idx(int i, int j) { return j * (j + 1) / 2 + i; }
constexpr int kTriMaxRows = 128;                 // positions staged in static shared memory
constexpr int kTriCum = 512 + 2;                 // item prefix sums, one per t_{k-1} (M <= bins <= 512)
constexpr int kTri3Cols = 96;                    // k = 3: last thresholds per item (3 per lane)
#ifndef TSA_TRI_SEED_PASSES
#define TSA_TRI_SEED_PASSES 3  // coordinate-ascent rounds of the k >= 3 seed (tri_seed)
#endif
#ifndef TSA_TRI4_Q
#define TSA_TRI4_Q 16
#endif
// k = 4: tiles of 4 prefixes per lane per item (32 * 4 * Q prefixes per item).
// With the exact item bound almost every item is dropped by its bound check,
// so larger items mean fewer checks (Q = 4 -> 16: the check was 67 % of the
// kernel's instructions on c4)
constexpr int kTri4Q = TSA_TRI4_Q;
#ifndef TSA_TRI_MINB
#define TSA_TRI_MINB 2  // CTAs per SM of k_search_tri (register cap; A/B builds)
#endif
// dynamic tables: 104 KB at two CTAs per SM, 72 KB (M <= 93) at three
constexpr size_t kTriSmemBytes = TSA_TRI_MINB >= 3 ? 72 * 1024 : 104 * 1024;

// doubles needed for the tables of a slice with M positions (rows packed)
// R row a of k_search_tri: columns from sa = (a+1) & ~1 in whole 4-column
// steps up to M-2 (NaN outside (a, M-2])
__host__ __device__ __forceinline__ int tri_row_len(int M, int a) { return 4 * ((M + 2 - ((a + 1) & ~1)) >> 2); }
// Chunk bounds (round 2, exact pruning of the k >= 3 search): RB[a][c] bounds
// the 16 packed columns [16c, 16c+16) of R row a (max; min in PROD_MIN, where
// prefixes are <= 0), PB[a][c] the sign-adjusted k = 3 prefix values
// combine(T(0, t1), T(t1+1, a)) for t1 in [8c, 8c+8) (max).  NaN entries are
// skipped (fmax / fmin); a chunk with no entry is NaN, which never passes a test.
__host__ __device__ __forceinline__ int tri_rbs(int M) { return (tri_row_len(M, 0) + 15) >> 4; }
__host__ __device__ __forceinline__ int tri_pbs(int M) { return (M + 7) >> 3; }
__host__ __device__ __forceinline__ int64_t tri_table_doubles(int M) {
  int64_t r = 0;
  for (int a = 0; a <= M - 3; a++) r += tri_row_len(M, a);
  return r + (int64_t)(M - 1) * M / 2 + (int64_t)(M - 2) * (tri_rbs(M) + tri_pbs(M)) + 2 * (int64_t)M;
}
// After RB and PB: QB[j] = max_c PB[j][c] (the sign-adjusted first-two-class
// prefix bound for t_{k-2} = j, any t_1 < j) and RA[a] = the bound of the
// whole R row a (max_c RB[a][c]; min in PROD_MIN), M doubles each: item-level
// bounds of the k >= 3 search.
__host__ __device__ __forceinline__ int64_t tri_qb_off(int M) {
  return (int64_t)(M - 1) * M / 2 + (int64_t)(M - 2) * (tri_rbs(M) + tri_pbs(M));
}

// Per-slice table region of k_search_tri (doubles): row offsets (M-1 ints,
// padded to an even number of doubles so the rows stay 16-byte aligned), then
// the packed R rows, then the triangular T table.
// (the last double of the offsets area holds the slice's seed score, tri_seed)
__host__ __device__ __forceinline__ int tri_roff_doubles(int M) { return (((M + 1) / 2) + 2) & ~1; }
// After the tables: the slice's item prefix counts cum[0..na] (ints, na = M-3-(k-2)+1;
// tri_items_warp), written once by k_tri_tables instead of per search entry.
__host__ __device__ __forceinline__ int64_t tri_cum_doubles(int M) { return (M + 3) / 2; }
__host__ __device__ __forceinline__ int64_t tri_region_doubles(int M) {
  return tri_roff_doubles(M) + tri_table_doubles(M) + tri_cum_doubles(M);
}
// Offset (doubles) of cum from the region start; tbase = roff[M-2] (the R rows' length)
__host__ __device__ __forceinline__ int64_t tri_cum_off(int M, int tbase) {
  return tri_roff_doubles(M) + tbase + tri_qb_off(M) + 2 * (int64_t)M;
}
// Per-slice region stride (host): room for any M <= L, even (16-byte aligned
// regions for the bulk copy).
inline int64_t tri_slice_stride(int L) { return (tri_region_doubles(L) + 1) & ~(int64_t)1; }

// Build the tables of slice z into `base`: roff[a] (start of R row a;
// roff[M-2] = start of T), T, then -- warp 0 computing the slice's seed score
// from T (tri_seed, concurrently) -- the R rows and the chunk bounds RB / PB
// (warps 1..; a named barrier orders RB / PB after the R rows).  Same
// expressions as k_rtable.  s_roff: shared copy of roff (M <= kTriMaxRows)
// for the row search of the flattened R loop, else null.
template <int K, int MODE>
__device__ double tri_seed(const int M, const double *Tt, const double *asz);
template <int K>
__device__ __forceinline__ int tri_items_warp(const int M, const uint64_t r0, const uint64_t r1, int *cum);

template <int K, int MODE>
__device__ void tri_build(const SearchArgs &g, const int z, const int M, const SliceTables &t, double *base,
                          int *s_roff) {
  int *roff = reinterpret_cast<int *>(base);
  double *Rt = base + tri_roff_doubles(M);
  const double *asz = g.Asuf + (size_t)z * g.L;
  __shared__ double s_p2[32];
  stage_p2(g.luts, s_p2);
  if (threadIdx.x == 0) {
    int o = 0;
    for (int a = 0; a <= M - 3; a++) {
      roff[a] = o;
      if (s_roff) s_roff[a] = o;
      o += tri_row_len(M, a);
    }
    roff[M - 2] = o;  // start of the T table
    if (s_roff) s_roff[M - 2] = o;
  }
  __syncthreads();
  const int *ro = s_roff ? s_roff : roff;
  const int tbase = ro[M - 2];
  double *Tt = Rt + tbase;
  // flattened over all entries (every thread busy; round 2's first version
  // looped over rows with at most M threads active and was latency-bound)
  const int ntri = (M - 1) * M / 2;
  for (int e = threadIdx.x; e < ntri; e += blockDim.x) {
    int j = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);  // e = j(j+1)/2 + i, i <= j
    while (j * (j + 1) / 2 > e) j--;
    while ((j + 1) * (j + 2) / 2 <= e) j++;
    Tt[e] = class_term<MODE>(t, g.luts, e - j * (j + 1) / 2, j, s_p2);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // warp 0: the seed (reads T and Asuf only)
    if (M - 1 >= K) {
      const double seed = tri_seed<K, MODE>(M, Tt, asz);
      if (threadIdx.x == 0) base[tri_roff_doubles(M) - 1] = seed;
    }
    return;  // no further block-wide barrier in the caller before its __syncthreads
  }
  const int tid = threadIdx.x - 32, nth = blockDim.x - 32;
  if (tid < 32 && M - 1 >= K) {  // warp 1: the item prefix counts of the search (tri_items_warp)
    const uint64_t NR = binom((uint64_t)(M - 1), K - 1);
    const uint64_t r0 = NR * (uint64_t)g.unit_begin / (uint64_t)g.units;
    const uint64_t r1 = NR * (uint64_t)(g.unit_begin + g.nunits) / (uint64_t)g.units;
    tri_items_warp<K>(M, r0, r1, reinterpret_cast<int *>(base + tri_cum_off(M, tbase)));
  }
  {  // R rows, a warp per row (lanes over its columns; a flattened loop
     // needed a binary search of roff per entry: ncu, the top stall)
    const int lane = threadIdx.x & 31, nwr = nth >> 5;
    for (int a = tid >> 5; a <= M - 3; a += nwr) {
      const int sa = (a + 1) & ~1, len = tri_row_len(M, a);
      double *row = Rt + ro[a];
      for (int u = lane; u < len; u += 32) {
        const int b = sa + u;
        row[u] = (b > a && b <= M - 2) ? combine<MODE>(Tt[tri_idx(a + 1, b)], __ldg(asz + b)) : CUDART_NAN;
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nth) : "memory");  // warps 1.. only
  double *RB = Tt + ntri;
  const int rbs = tri_rbs(M), pbs = tri_pbs(M);
  double *PB = RB + (M - 2) * rbs;
  for (int e = tid; e < (M - 2) * rbs; e += nth) {
    const int a = e / rbs, c = e - a * rbs;
    const double *row = Rt + ro[a];
    const int u1 = min(tri_row_len(M, a), 16 * c + 16);
    double v = CUDART_NAN;
    for (int u = 16 * c; u < u1; u++) v = MODE == PROD_MIN ? fmin(v, row[u]) : fmax(v, row[u]);
    RB[e] = v;
  }
  for (int e = tid; e < (M - 2) * pbs; e += nth) {
    const int a = e / pbs, c = e - a * pbs;
    double v = CUDART_NAN;
    for (int t1 = 8 * c; t1 < min(a, 8 * c + 8); t1++) {
      double pre = combine<MODE>(Tt[tri_idx(0, t1)], Tt[tri_idx(t1 + 1, a)]);
      if (MODE == PROD_MIN) pre = -pre;
      v = fmax(v, pre);
    }
    PB[e] = v;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nth) : "memory");
  double *QB = PB + (M - 2) * pbs, *RA = QB + M;
  for (int j = tid; j <= M - 3; j += nth) {
    double qv = CUDART_NAN, rv = CUDART_NAN;
    for (int c = 0; c < pbs; c++) qv = fmax(qv, PB[j * pbs + c]);
    for (int c = 0; c < rbs; c++) rv = MODE == PROD_MIN ? fmin(rv, RB[j * rbs + c]) : fmax(rv, RB[j * rbs + c]);
    QB[j] = qv;
    RA[j] = rv;
  }
}

// hit |= any(p_i (x) x_c >= best), i < 4 prefixes, c < 4 columns (x01, x23):
// 16 DMUL/DADD + 16 DSETP in four predicate chains of four (2 FP64
// instructions per tuple, ~85 % of the issued instructions on the FP64 pipe).
template <int MODE>
__device__ __forceinline__ unsigned cmp_p4c4(unsigned hit, const double *p, double2 x01, double2 x23,
                                             double best) {
#define TSA_CMP_P4C4(OP)                                                                          \
  asm("{\n\t.reg .pred a, b, c, d;\n\t.reg .f64 t<16>;\n\t"                                      \
      "setp.ne.u32 a, %0, 0;\n\t"                                                                 \
      OP " t0, %1, %5;\n\t" OP " t1, %1, %6;\n\t" OP " t2, %1, %7;\n\t" OP " t3, %1, %8;\n\t"    \
      OP " t4, %2, %5;\n\t" OP " t5, %2, %6;\n\t" OP " t6, %2, %7;\n\t" OP " t7, %2, %8;\n\t"    \
      OP " t8, %3, %5;\n\t" OP " t9, %3, %6;\n\t" OP " t10, %3, %7;\n\t" OP " t11, %3, %8;\n\t"  \
      OP " t12, %4, %5;\n\t" OP " t13, %4, %6;\n\t" OP " t14, %4, %7;\n\t" OP " t15, %4, %8;\n\t" \
      "setp.ge.f64 b, t1, %9;\n\tsetp.ge.f64 c, t2, %9;\n\tsetp.ge.f64 d, t3, %9;\n\t"           \
      "setp.ge.or.f64 a, t0, %9, a;\n\tsetp.ge.or.f64 b, t5, %9, b;\n\t"                          \
      "setp.ge.or.f64 c, t6, %9, c;\n\tsetp.ge.or.f64 d, t7, %9, d;\n\t"                          \
      "setp.ge.or.f64 a, t4, %9, a;\n\tsetp.ge.or.f64 b, t9, %9, b;\n\t"                          \
      "setp.ge.or.f64 c, t10, %9, c;\n\tsetp.ge.or.f64 d, t11, %9, d;\n\t"                        \
      "setp.ge.or.f64 a, t8, %9, a;\n\tsetp.ge.or.f64 b, t13, %9, b;\n\t"                         \
      "setp.ge.or.f64 c, t14, %9, c;\n\tsetp.ge.or.f64 d, t15, %9, d;\n\t"                        \
      "setp.ge.or.f64 a, t12, %9, a;\n\t"                                                         \
      "or.pred a, a, b;\n\tor.pred c, c, d;\n\tor.pred a, a, c;\n\tselp.u32 %0, 1, 0, a;\n\t}"    \
      : "+r"(hit)                                                                                 \
      : "d"(p[0]), "d"(p[1]), "d"(p[2]), "d"(p[3]), "d"(x01.x), "d"(x01.y), "d"(x23.x), "d"(x23.y), \
        "d"(best))
  if (MODE == SUM) {
    TSA_CMP_P4C4("add.rn.f64");
  } else {
    TSA_CMP_P4C4("mul.rn.f64");
  }
#undef TSA_CMP_P4C4
  return hit;
}

// One prefix value against the lane's three columns (k = 3 tiles).
template <int MODE>
__device__ __forceinline__ unsigned cmp_p1c3(unsigned hit, double p, const double *x, double best) {
#define TSA_CMP_P1C3(OP)                                                                          \
  asm("{\n\t.reg .pred a;\n\t.reg .f64 t<3>;\n\t"                                                \
      "setp.ne.u32 a, %0, 0;\n\t"                                                                 \
      OP " t0, %1, %2;\n\t" OP " t1, %1, %3;\n\t" OP " t2, %1, %4;\n\t"                          \
      "setp.ge.or.f64 a, t0, %5, a;\n\tsetp.ge.or.f64 a, t1, %5, a;\n\t"                          \
      "setp.ge.or.f64 a, t2, %5, a;\n\tselp.u32 %0, 1, 0, a;\n\t}"                                \
      : "+r"(hit)                                                                                 \
      : "d"(p), "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(best))
  if (MODE == SUM) {
    TSA_CMP_P1C3("add.rn.f64");
  } else {
    TSA_CMP_P1C3("mul.rn.f64");
  }
#undef TSA_CMP_P1C3
  return hit;
}

// One prefix, four columns (k = 3: a prefix row is short, one per lane).
template <int MODE>
__device__ __forceinline__ unsigned cmp_p1c4(unsigned hit, double p, double2 x01, double2 x23, double best) {
#define TSA_CMP_P1C4(OP)                                                                          \
  asm("{\n\t.reg .pred a, b;\n\t.reg .f64 t<4>;\n\t"                                             \
      "setp.ne.u32 a, %0, 0;\n\t"                                                                 \
      OP " t0, %1, %2;\n\t" OP " t1, %1, %3;\n\t" OP " t2, %1, %4;\n\t" OP " t3, %1, %5;\n\t"    \
      "setp.ge.f64 b, t1, %6;\n\tsetp.ge.or.f64 a, t0, %6, a;\n\t"                               \
      "setp.ge.or.f64 b, t3, %6, b;\n\tsetp.ge.or.f64 a, t2, %6, a;\n\t"                         \
      "or.pred a, a, b;\n\tselp.u32 %0, 1, 0, a;\n\t}"                                            \
      : "+r"(hit)                                                                                 \
      : "d"(p), "d"(x01.x), "d"(x01.y), "d"(x23.x), "d"(x23.y), "d"(best))
  if (MODE == SUM) {
    TSA_CMP_P1C4("add.rn.f64");
  } else {
    TSA_CMP_P1C4("mul.rn.f64");
  }
#undef TSA_CMP_P1C4
  return hit;
}

// One CTA's share of slice z, register-tiled like a GEMM micro-kernel with
// (max, x): items are (a, chunk) -- a = t_{k-1}, a chunk = 32 P consecutive
// prefixes ending at a (P = 4 for k = 4, 1 for k = 3); a lane holds P prefix
// values and streams the shared row R[a][*] four columns at a time (one
// broadcast 32-byte shared load serves 4P tuples), testing value >= best in
// predicate chains.  Only a lane whose tile produced a hit rescans its rows
// exactly (the staged kernels' value, (score desc, key asc) order).  Items are
// claimed from the slice's counter by warps of every CTA on the slice.
// A lower bound for the slice's best score, to seed the rescan test: the
// value (same expression tree as the search) of a tuple found by coordinate
// ascent from evenly spaced thresholds (3 passes, one warp; any valid tuple's
// value is a valid seed -- a good one makes exact rescans rare and the chunk
// bounds effective).  The R entry of (a, b) is formed from T and Asuf exactly
// as tri_build forms it, so the seed runs next to the R build.  The search
// then compares against it with key = none, so the tuples scoring >= it,
// the argmax among them, are all still found exactly.  Returns the seed in
// every lane.
template <int K, int MODE>
__device__ double tri_seed(const int M, const double *Tt, const double *asz) {
  constexpr int R = K - 1;
  const int lane = threadIdx.x & 31;
  auto val = [&](const int *t) -> double {  // t[0..K-1] strictly increasing in [0, M-2]
    const double p01 = combine<MODE>(Tt[tri_idx(0, t[0])], Tt[tri_idx(t[0] + 1, t[1])]);
    double pre = K == 3 ? p01 : combine<MODE>(p01, Tt[tri_idx(t[1] + 1, t[R - 1])]);
    if (MODE == PROD_MIN) pre = -pre;
    const int a = t[R - 1], b = t[K - 1];
    return combine<MODE>(pre, combine<MODE>(Tt[tri_idx(a + 1, b)], __ldg(asz + b)));
  };
  int t[K];
#pragma unroll
  for (int j = 0; j < K; j++) t[j] = (int)((int64_t)(j + 1) * (M - 1) / (K + 1)) - 1 + (j == 0);
#pragma unroll
  for (int j = 1; j < K; j++) t[j] = max(t[j], t[j - 1] + 1);  // strictly increasing
  double best = val(t);
  for (int pass = 0; pass < TSA_TRI_SEED_PASSES; pass++) {
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int lo = j == 0 ? 0 : t[j - 1] + 1, hi = j == K - 1 ? M - 2 : t[j + 1] - 1;
      double bv = -CUDART_INF;
      int bx = t[j];
      // independent candidates: unrolled so their table loads overlap
#pragma unroll 4
      for (int x = lo + lane; x <= hi; x += 32) {
        int u[K];
#pragma unroll
        for (int i = 0; i < K; i++) u[i] = i == j ? x : t[i];
        const double v = val(u);
        if (v > bv || (v == bv && x < bx)) {
          bv = v;
          bx = x;
        }
      }
      uint64_t key = (uint64_t)bx;
      warp_argmax(bv, key);
      if (bv > best) {
        best = bv;
        t[j] = (int)key;
      }
    }
  }
  return best;
}

// Items of a slice: for a in [R-1, M-3] the prefixes ending at a have colex
// ranks [C(a, R), C(a+1, R)); intersected with [r0, r1) and cut into chunks of
// G; s_cum[a - (R-1) + 1] = items up to a (thread 0; returns the total).
template <int K>
__device__ __forceinline__ int tri_items(const int M, const uint64_t r0, const uint64_t r1, int *s_cum) {
  constexpr int R = K - 1, G = 32 * (K == 4 ? 4 * kTri4Q : 1);  // = tri_search's 32 P Q
  const int a0 = R - 1;
  if (threadIdx.x < 32) {  // warp 0: per-a item counts and their prefix sums
    const int lane = threadIdx.x;
    int base = 0;
    for (int as = a0; as <= M - 3; as += 32) {
      const int a = as + lane;
      int cnt = 0;
      if (a <= M - 3) {
        const uint64_t lo = max(binom((uint64_t)a, R), r0), hi = min(binom((uint64_t)a + 1, R), r1);
        if (hi > lo) cnt = K == 3 ? (M - 2 - a + kTri3Cols - 1) / kTri3Cols : (int)((hi - lo + G - 1) / G);
      }
      int x = cnt;  // inclusive warp scan
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (a <= M - 3) s_cum[a - a0 + 1] = base + x;
      base += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      s_cum[0] = 0;
      s_cum[kTriCum - 1] = base;
    }
  }
  __syncthreads();
  return s_cum[kTriCum - 1];
}

// tri_items for one warp (no block barrier): cum[a - (R-1) + 1] = items up to
// a, cum[0] = 0; returns the total (every lane).
template <int K>
__device__ __forceinline__ int tri_items_warp(const int M, const uint64_t r0, const uint64_t r1, int *cum) {
  constexpr int R = K - 1, G = 32 * (K == 4 ? 4 * kTri4Q : 1);
  const int a0 = R - 1, lane = threadIdx.x & 31;
  int base = 0;
  for (int as = a0; as <= M - 3; as += 32) {
    const int a = as + lane;
    int cnt = 0;
    if (a <= M - 3) {
      const uint64_t lo = max(binom((uint64_t)a, R), r0), hi = min(binom((uint64_t)a + 1, R), r1);
      if (hi > lo) cnt = K == 3 ? (M - 2 - a + kTri3Cols - 1) / kTri3Cols : (int)((hi - lo + G - 1) / G);
    }
    int x = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (a <= M - 3) cum[a - a0 + 1] = base + x;
    base += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) cum[0] = 0;
  return base;
}

template <int K, int MODE>
__device__ __forceinline__ void tri_search(const SearchArgs &g, const int M, const uint64_t r0, const uint64_t r1,
                                           const double *base, const int32_t *bin, int32_t *ccur,
                                           const int *s_cum, const int nitems, double &best,
                                           uint64_t &bestkey) {
  constexpr int R = K - 1;           // prefix length (t_1 .. t_{k-1}, t_{k-1} = a)
  constexpr int P = K == 4 ? 4 : 1;  // prefixes per register tile
  constexpr int Q = K == 4 ? kTri4Q : 1;  // tiles per lane per item
  constexpr int G = 32 * P * Q;      // prefixes per item
  const int *roff = reinterpret_cast<const int *>(base);
  const double *Rt = base + tri_roff_doubles(M);
  const double *Tt = Rt + roff[M - 2];
  const int a0 = R - 1, na = M - 3 - a0 + 1;  // a in [R-1, M-3]; items: s_cum (tri_items)
  const int lane = threadIdx.x & 31;
  bool first = true;
  // item claims run one item ahead (the atomic's round trip overlaps the
  // current item instead of stalling the warp before it)
  int cn = 0;
  if (lane == 0) cn = atomicAdd(ccur, 1);
  for (;;) {
    const int c = __shfl_sync(0xffffffffu, cn, 0);
    if (c >= nitems) break;
    if (lane == 0) cn = atomicAdd(ccur, 1);
    int lo_i = 0, hi_i = na - 1;  // the a whose items contain c
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i + 1) >> 1;
      if (s_cum[mid] <= c) lo_i = mid;
      else hi_i = mid - 1;
    }
    const int a = a0 + lo_i;
    const uint64_t lo = max(binom((uint64_t)a, R), r0), hi = min(binom((uint64_t)a + 1, R), r1);
    if (K == 3) {
      // lanes over the last threshold b (3 columns each), loop over t_1:
      // the prefix value (one per t_1) is a broadcast, the R values stay in
      // registers: 2 FP64 instructions per tuple + 1 DMUL per t_1
      const int sa = (a + 1) & ~1;
      const double *row = Rt + roff[a] - sa;
      const int bb = a + 1 + (c - s_cum[lo_i]) * kTri3Cols + lane;
      double rv[3];
#pragma unroll
      for (int u = 0; u < 3; u++) {
        const int b = bb + 32 * u;
        rv[u] = b <= M - 2 ? row[b] : CUDART_NAN;
      }
      const int t1lo = (int)(lo - binom((uint64_t)a, 2)), t1hi = (int)(hi - binom((uint64_t)a, 2));
      unsigned hit = 0;
      // chunks of 8 t_1: skipped by the whole warp when no lane's bound
      // combine(PB[a][chunk], bound of its 3 columns) reaches its best
      // (value = combine(pre, R) is monotone in both and rounding is
      // monotone, so a skipped tuple scores <= the bound < best: exact)
      const double rbl = MODE == PROD_MIN ? fmin(fmin(rv[0], rv[1]), rv[2]) : fmax(fmax(rv[0], rv[1]), rv[2]);
      const double *pbr = Tt + (M - 1) * M / 2 + (M - 2) * tri_rbs(M) + a * tri_pbs(M);
      // the whole item first: QB[a] bounds every prefix ending at a
      const bool live = __any_sync(0xffffffffu, combine<MODE>(Tt[tri_qb_off(M) + a], rbl) >= best);
      for (int t1c = live ? t1lo : t1hi; t1c < t1hi;) {
        const int cend = min(t1hi, (t1c & ~7) + 8);
        if (__any_sync(0xffffffffu, combine<MODE>(pbr[t1c >> 3], rbl) >= best))
          for (int t1 = t1c; t1 < cend; t1++) {
            double pre = combine<MODE>(Tt[tri_idx(0, t1)], Tt[tri_idx(t1 + 1, a)]);
            if (MODE == PROD_MIN) pre = -pre;
            hit = cmp_p1c3<MODE>(hit, pre, rv, best);
          }
        t1c = cend;
      }
      if (hit) {  // exact rescan of this lane's tuples in lex order (t_1, then b)
        for (int t1 = t1lo; t1 < t1hi; t1++) {
          double pre = combine<MODE>(Tt[tri_idx(0, t1)], Tt[tri_idx(t1 + 1, a)]);
          if (MODE == PROD_MIN) pre = -pre;
          const uint64_t kp = ((uint64_t)bin[t1 + 1] << 12) | (uint64_t)bin[a + 1];
#pragma unroll
          for (int u = 0; u < 3; u++) {
            const int b = bb + 32 * u;
            const double v = combine<MODE>(pre, rv[u]);
            if (b <= M - 2 && v >= best) {
              const uint64_t key = (kp << 12) | (uint64_t)bin[b + 1];
              if (better(v, key, best, bestkey)) {
                best = v;
                bestkey = key;
              }
            }
          }
        }
      }
      if (first) {
        warp_argmax(best, bestkey);
        first = false;
      }
      continue;
    }
    const uint64_t ib = lo + (uint64_t)(c - s_cum[lo_i]) * G;  // the item's ranks [ib, min(hi, ib + G))
    if (K == 4) {
      // item bound: prefixes (t_1, j, a) score <= combine(QB[j], T(j+1, a))
      // (QB: the max of the first two classes over t_1), rows <= RA[a]; the
      // item is dropped when that is below every lane's best
      const uint64_t base_a = binom((uint64_t)a, 3);
      auto jof = [&](uint64_t r) -> int {  // t_2 of colex offset r within a: C(j,2) <= r < C(j+1,2)
        int j = (int)((1.0 + sqrt(1.0 + 8.0 * (double)r)) * 0.5);
        while (j > 1 && binom((uint64_t)j, 2) > r) j--;
        while (binom((uint64_t)j + 1, 2) <= r) j++;
        return j;
      };
      const int jlo = jof(ib - base_a), jhi = jof(min(hi, ib + G) - 1 - base_a);
      const double *QB = Tt + tri_qb_off(M);
      double vb = -CUDART_INF;
      for (int j = jlo + lane; j <= jhi; j += 32) vb = fmax(vb, combine<MODE>(QB[j], Tt[tri_idx(j + 1, a)]));
      double bmin = best;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        vb = fmax(vb, __shfl_xor_sync(0xffffffffu, vb, off));
        bmin = fmin(bmin, __shfl_xor_sync(0xffffffffu, bmin, off));
      }
      if (!(combine<MODE>(vb, QB[M + a]) >= bmin)) {
        if (first) {
          warp_argmax(best, bestkey);
          first = false;
        }
        continue;
      }
    }
    uint64_t rb = ib + (uint64_t)lane * (P * Q);
    {  // the whole warp runs the tiles (lanes past hi hold NaN prefixes), so
       // the chunk votes below are converged
      const int sa = (a + 1) & ~1;
      const double *row = Rt + roff[a] - sa;  // row[b], b in [sa, sa + tri_row_len)
      const double2 *rp = reinterpret_cast<const double2 *>(Rt + roff[a]);
      const int nsteps = tri_row_len(M, a) >> 2;  // 4-column steps
      const double *rbr = Tt + (M - 1) * M / 2 + a * tri_rbs(M);  // chunk bounds of row a
      int idx[R];
      unrank_colex<R>(rb, idx);
#pragma unroll 1
      for (int q = 0; q < Q; q++) {
        if (!__any_sync(0xffffffffu, rb < hi)) break;
        // this tile's prefixes rb .. rb+P-1 (< hi), all ending at a
        double pre[P];
        int tid0[P], tid1[P];
        int nv = 0;
#pragma unroll
        for (int i = 0; i < P; i++) {
          if (i > 0) next_colex<R>(idx);
          const bool v = rb + i < hi;
          nv += v;
          tid0[i] = idx[0];
          tid1[i] = idx[R - 2];
          const double p01 = combine<MODE>(Tt[tri_idx(0, idx[0])], Tt[tri_idx(idx[0] + 1, idx[1])]);
          double pv = K == 3 ? p01 : combine<MODE>(p01, Tt[tri_idx(idx[1] + 1, a)]);
          if (MODE == PROD_MIN) pv = -pv;  // (-pre)*R == -(pre*R) exactly
          pre[i] = v ? pv : CUDART_NAN;    // NaN never compares >= best
        }
        unsigned hit = 0;
        // 16-column chunks of the row, skipped by the (active) warp when no
        // lane's bound combine(max of its P prefixes, RB[a][chunk]) reaches
        // its best: exact, as for k = 3 (NaN prefixes are ignored by fmax)
        double pm = pre[0];
#pragma unroll
        for (int i = 1; i < P; i++) pm = fmax(pm, pre[i]);
        for (int c0 = 0; c0 < nsteps; c0 += 4) {
          if (!__any_sync(0xffffffffu, combine<MODE>(pm, rbr[c0 >> 2]) >= best)) continue;
          const int s1 = min(nsteps, c0 + 4);
          for (int s = c0; s < s1; s++) {
            const double2 x01 = rp[2 * s], x23 = rp[2 * s + 1];
            if (P == 4) hit = cmp_p4c4<MODE>(hit, pre, x01, x23, best);
            else hit = cmp_p1c4<MODE>(hit, pre[0], x01, x23, best);
          }
        }
        if (hit) {  // exact rescan of this tile's rows, lower-lex prefix first
          // unrolled over the constant P with a guard: a dynamic index into
          // pre / tid0 / tid1 put them in local memory (ncu: STL/LDL per tile)
#pragma unroll
          for (int i = 0; i < P; i++) {
            if (i >= nv) break;
            uint64_t kp = (uint64_t)bin[tid0[i] + 1];
            if (K == 4) kp = (kp << 12) | (uint64_t)bin[tid1[i] + 1];
            kp = (kp << 12) | (uint64_t)bin[a + 1];
            for (int b = a + 1; b <= M - 2; b++) {
              const double v = combine<MODE>(pre[i], row[b]);
              if (v >= best) {
                const uint64_t key = (kp << 12) | (uint64_t)bin[b + 1];
                if (better(v, key, best, bestkey)) {
                  best = v;
                  bestkey = key;
                }
              }
            }
          }
        }
        next_colex<R>(idx);  // first prefix of the next tile
        rb += P;
      }
    }
    if (first) {  // the warp's best so far seeds every lane's test
      warp_argmax(best, bestkey);
      first = false;
    }
  }
}

// Tables of every slice (one CTA per slice) into the per-slice global regions,
// and the slice's seed score (tri_seed) in the last double of the offsets.
template <int K, int MODE>
__global__ void __launch_bounds__(256) k_tri_tables(SearchArgs g) {
  __shared__ uint32_t s_C[kTriMaxRows + 2];
  __shared__ double s_Wh[kTriMaxRows + 2], s_Wl[kTriMaxRows + 2];
  const int z = blockIdx.x;
  const int M = g.Mz[z];
  if (g.status[z] != kOK || M < 4) return;
  const uint32_t *gC = g.C + (size_t)z * g.E;
  const double *gWh = g.Whi + (size_t)z * g.E, *gWl = g.Wlo + (size_t)z * g.E;
  const bool stage = M + 1 <= kTriMaxRows + 2;
  if (stage)
    for (int e = threadIdx.x; e <= M; e += blockDim.x) {
      s_C[e] = gC[e];
      s_Wh[e] = gWh[e];
      s_Wl[e] = gWl[e];
    }
  __syncthreads();
  const SliceTables t{stage ? s_C : gC, stage ? s_Wh : gWh, stage ? s_Wl : gWl, nullptr};
  double *region = const_cast<double *>(g.R) + (size_t)z * g.TS;
  __shared__ int s_roff[kTriMaxRows + 2];
  tri_build<K, MODE>(g, z, M, t, region, M <= kTriMaxRows ? s_roff : nullptr);
}

// Exhaustive search for k >= 3 over per-slice class-term tables (round 2;
// replaces k_rtable's three L x (L+8) HBM tables per slice):
//   T(i, j), 0 <= i <= j <= M-2      every class term (triangular, j(j+1)/2 + i)
//   R[a][b] = T(a+1, b) (x) Asuf[b]  the last two classes, rows a <= M-3 stored
//                                    from column (a+1) & ~1 in whole 8-column
//                                    groups (NaN outside (a, M-2]), packed
// built once per slice by k_tri_tables (M^2 doubles: ~70 KB at m ~ 90) and
// copied into shared memory by every CTA that searches the slice when they
// fit (M <= ~115 at two CTAs per SM: every slice of the 8-bit configs), else
// read from the global region.  Prefix values are the staged tables'
// expressions: K = 3: PP[t1][a] = T(0,t1) (x) T(t1+1,a); K = 4:
// PP[t1][t2] (x) T(t2+1,a); the compare loop is search_row / search_row2, so
// every tuple's value is bit-identical to k_search_rows' (tested).
// Work: entries e = z * ss + j (slices in order, ss entries each) from a
// global counter; the CTAs on a slice share its prefix rows [r0, r1) (the
// launch's units, one contiguous colex range) through a per-slice chunk
// counter, so a slice's work spreads over up to ss CTAs and no CTA waits on a
// long last item.  Entry results go to slot [j][z]; k_fold_slots merges.
template <int K, int MODE>
__global__ void __launch_bounds__(256, TSA_TRI_MINB) k_search_tri(SearchArgs g, int smem_doubles) {
  static_assert(K >= 3 && K <= 4, "k = 3, 4");
  constexpr int R = K - 1;
  extern __shared__ __align__(16) double tsm[];
  __shared__ int s_item;
  __shared__ int32_t s_bin[kTriMaxRows + 2];
  __shared__ __align__(8) uint64_t s_bar;  // the tables' bulk copy (TMA)
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const int64_t items = g.nz * (int64_t)g.ss;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(g.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= items) break;
    const int z = (int)(item / g.ss);
    const int j = (int)(item % g.ss);
    double best = -CUDART_INF;
    uint64_t bestkey = kKeyNone;
    const int st = g.status[z];
    const int M = g.Mz[z];
    const int P = M - 1;
    int32_t *ccur = g.ccur + z;
    if (st == kOK && P >= K) {
      const uint64_t NR = binom((uint64_t)P, R);
      const uint64_t r0 = NR * (uint64_t)g.unit_begin / (uint64_t)g.units;
      const uint64_t r1 = NR * (uint64_t)(g.unit_begin + g.nunits) / (uint64_t)g.units;
      // item prefix counts from k_tri_tables (tri_items_warp), total cum[na]
      const double *region = g.R + (size_t)z * g.TS;
      const int tbase = reinterpret_cast<const int *>(region)[M - 2];
      const int64_t coff = tri_cum_off(M, tbase);
      const int nitems = reinterpret_cast<const int *>(region + coff)[M - 3 - (R - 1) + 1];
      // skip the copy when the slice's items are already all claimed
      if (*((volatile int32_t *)ccur) < nitems) {
        const int32_t *gB = g.Bin + (size_t)z * g.E;
        const bool stage = M + 1 <= kTriMaxRows + 2;
        if (stage)
          for (int e = threadIdx.x; e <= M; e += blockDim.x) s_bin[e] = gB[e];
        const int64_t nd = coff + tri_cum_doubles(M);
        if (M <= kTriMaxRows && nd <= smem_doubles) {
          // the slice's tables into shared memory: one TMA bulk copy (the
          // previous entry's generic reads are ordered before it by the
          // barrier at the top of the loop and the proxy fence)
          if (threadIdx.x == 0) {
            const uint32_t bytes = (uint32_t)(((nd + 1) / 2) * 16);
            fence_proxy_async_smem();
            mbar_expect_tx(&s_bar, bytes);
            bulk_g2s(tsm, region, bytes, &s_bar);
          }
          mbar_wait(&s_bar, phase);
          phase ^= 1u;
          __syncthreads();
          best = tsm[tri_roff_doubles(M) - 1];  // the slice's seed (k_tri_tables)
          tri_search<K, MODE>(g, M, r0, r1, tsm, stage ? s_bin : gB, ccur,
                              reinterpret_cast<const int *>(tsm + coff), nitems, best, bestkey);
        } else {
          __syncthreads();
          best = region[tri_roff_doubles(M) - 1];
          tri_search<K, MODE>(g, M, r0, r1, region, stage ? s_bin : gB, ccur,
                              reinterpret_cast<const int *>(region + coff), nitems, best, bestkey);
        }
      }
    }
    block_argmax(best, bestkey);
    if (threadIdx.x == 0) {
      g.item_score[(size_t)j * g.nz + z] = best;
      g.item_key[(size_t)j * g.nz + z] = bestkey;
    }
  }
}

// Slots [ss][nz] of k_search_tri -> part[0][z] (merged), part[1..nu-1][z] = none.
__global__ void k_fold_slots(const double *is, const uint64_t *ik, int ss, int64_t nz, int nu, double *ps,
                             uint64_t *pk) {
  const int64_t z = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (z >= nz) return;
  double s = -CUDART_INF;
  uint64_t k = kKeyNone;
  for (int j = lane; j < ss; j += 32) {
    const double os = is[(size_t)j * nz + z];
    const uint64_t ok = ik[(size_t)j * nz + z];
    if (better(os, ok, s, k)) {
      s = os;
      k = ok;
    }
  }
  warp_argmax(s, k);
  for (int u = lane; u < nu; u += 32) {
    ps[(size_t)u * nz + z] = u == 0 ? s : -CUDART_INF;
    pk[(size_t)u * nz + z] = u == 0 ? k : kKeyNone;
  }
}

}  // namespace tsa

namespace tsa {

// Chunks of the k <= 2 tuple space of a slice with M canonical positions
// (P = M - 1 threshold positions): k = 1, chunk c = thresholds [c*CH, c*CH+CH);
// k = 2, row b (a = 0..b-1) is split into ceil(b/CH) chunks of CH consecutive
// a, rows in order: off(b) = sum_{j<b} ceil(j/CH).
template <int K, int CH>
__host__ __device__ __forceinline__ int k12_off(int b) {
  const int n = b - 1, Q = n / CH, Rr = n % CH;
  return b <= 0 ? 0 : CH * Q * (Q + 1) / 2 + (Q + 1) * Rr;
}
template <int K, int CH>
__host__ __device__ __forceinline__ int k12_chunks(int M) {
  const int P = M - 1;
  if (P <= 0) return 0;
  return K == 1 ? (P + CH - 1) / CH : k12_off<K, CH>(P);
}

// Row-chunked exhaustive search for k <= 2: chunks [cbeg, cend) of the slice,
// dealt to threads tid, tid + nth, ...  No tuple is unranked (no FP64 sqrt)
// and a thread keeps CH independent class terms in flight.  Value of tuple
// (a, b): (1 (x) Apre[a]) (x) (T(a+1, b) (x) Asuf[b]) (k = 2), 1 (x) (T(0, b)
// (x) Asuf[b]) (k = 1) -- the expression tree of every other search kernel --
// and candidates are compared under the full (score, key) order, so any
// chunk partition gives the same result.
template <int K, int MODE, int CH = 16>
__device__ __forceinline__ void search_rows_k12(const SliceTables &t, const double *Apre, const Luts &l,
                                                const int32_t *bin, int M, int cbeg, int cend, int tid,
                                                int nth, double &best, uint64_t &bestkey,
                                                const double *p2s = nullptr) {
  const double ident = MODE == SUM ? 0.0 : 1.0;
  const int P = M - 1;  // positions 0 .. M-2
  if (K == 1) {
    for (int c = cbeg + tid; c < cend; c += nth) {
      const int b0 = c * CH;
      double v[CH];
#pragma unroll
      for (int u = 0; u < CH; u++) {
        const int b = min(b0 + u, P - 1);
        v[u] = combine<MODE>(ident, combine<MODE>(class_term<MODE>(t, l, 0, b, p2s), t.Asuf[b]));
        if (MODE == PROD_MIN) v[u] = -v[u];
      }
#pragma unroll
      for (int u = 0; u < CH; u++) {
        const int b = b0 + u;
        if (b < P && v[u] >= best) {
          const uint64_t key = (uint64_t)bin[b + 1];
          if (better(v[u], key, best, bestkey)) {
            best = v[u];
            bestkey = key;
          }
        }
      }
    }
    return;
  }
  for (int c = cbeg + tid; c < cend; c += nth) {
    // row b: largest b with off(b) <= c (rows 1 .. P-1 hold tuples)
    int lo = 1, hi = P - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (k12_off<K, CH>(mid) <= c) lo = mid;
      else hi = mid - 1;
    }
    const int b = lo, a0 = (c - k12_off<K, CH>(b)) * CH;
    const double R0 = t.Asuf[b];
    double v[CH];
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int a = min(a0 + u, b - 1);
      const double R = combine<MODE>(class_term<MODE>(t, l, a + 1, b, p2s), R0);
      v[u] = combine<MODE>(combine<MODE>(ident, Apre[a]), R);
      if (MODE == PROD_MIN) v[u] = -v[u];
    }
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int a = a0 + u;
      if (a < b && v[u] >= best) {
        const uint64_t key = ((uint64_t)bin[a + 1] << 12) | (uint64_t)bin[b + 1];
        if (better(v[u], key, best, bestkey)) {
          best = v[u];
          bestkey = key;
        }
      }
    }
  }
}

// Staged-path kernel for k <= 2 (not sum-plus-product): CTA (unit, slice)
// stages the slice's canonical tables, Apre and the small class-term table in
// shared memory, then searches its chunk range [NC*u/U, NC*(u+1)/U) with
// search_rows_k12 (NC = k12_chunks(M)).
constexpr int kK12Chunk = 16;

template <int K, int MODE, int NT>
__global__ void __launch_bounds__(NT) k_search_flat(SearchArgs g) {
  extern __shared__ double ssh[];
  const int z = blockIdx.y;
  const int u = g.unit_begin + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double best = -CUDART_INF;
  uint64_t bestkey = kKeyNone;
  const int st = g.status[z];
  const int M = g.Mz[z];
  const int P = M - 1;
  if (st == kOK && P >= K) {
    SliceTables t{g.C + (size_t)z * g.E, g.Whi + (size_t)z * g.E, g.Wlo + (size_t)z * g.E,
                  g.Asuf + (size_t)z * g.L};
    double *sWhi = ssh, *sWlo = ssh + g.E, *sAsuf = ssh + 2 * g.E, *sApre = ssh + 2 * g.E + g.L;
    double *sSp = ssh + 2 * g.E + 2 * g.L;  // small class-term table (kSmallLut)
    uint32_t *sC = reinterpret_cast<uint32_t *>(sSp + kSmallLut);
    for (int i = threadIdx.x; i <= M; i += blockDim.x) {
      sWhi[i] = t.Whi[i];
      sWlo[i] = t.Wlo[i];
      sC[i] = t.C[i];
      if (i <= M - 2) sAsuf[i] = t.Asuf[i];
    }
    for (int i = threadIdx.x; i < kSmallLut; i += blockDim.x) sSp[i] = g.luts.sp[i];
    __shared__ double s_p2[32];
    stage_p2(g.luts, s_p2);
    __syncthreads();
    const SliceTables ts{sC, sWhi, sWlo, sAsuf};
    Luts ls = g.luts;
    ls.sp = sSp;
    if (K == 2)
      for (int i = threadIdx.x; i <= M - 2; i += blockDim.x) sApre[i] = class_term<MODE>(ts, ls, 0, i, s_p2);
    __syncthreads();
    const int64_t NC = k12_chunks<K, kK12Chunk>(M);
    const int c0 = (int)(NC * u / g.units), c1 = (int)(NC * (u + 1) / g.units);
    search_rows_k12<K, MODE, kK12Chunk>(ts, sApre, ls, g.Bin + (size_t)z * g.E, M, c0, c1, threadIdx.x,
                                        blockDim.x, best, bestkey, s_p2);
  }
  warp_argmax(best, bestkey);
  __shared__ double ss[32];
  __shared__ uint64_t sk[32];
  if (lane == 0) {
    ss[warp] = best;
    sk[warp] = bestkey;
  }
  __syncthreads();
  if (warp == 0) {
    best = lane < nw ? ss[lane] : -CUDART_INF;
    bestkey = lane < nw ? sk[lane] : kKeyNone;
    warp_argmax(best, bestkey);
    if (lane == 0) {
      g.part_score[(size_t)blockIdx.x * g.nz + z] = best;
      g.part_key[(size_t)blockIdx.x * g.nz + z] = bestkey;
    }
  }
}

// ---------------------------------------------------------------------------
// k = 2 exhaustive search, warp per a-block (pseudo-additive or q == 1).
//
// Work item (i, z): slice z, a-block i = lanes a = 32 i + lane (t_1 = position
// a).  The warp walks every row b = t_2 in (32 i, M-2]; lane a evaluates
// (a, b) when a < b.  The lane's own quantities (C[a+1], W[a+1], Apre[a] =
// T(0, a)) stay in registers for the whole item and the row's (C[b+1], W[b+1],
// Asuf[b]) are warp-uniform loads, so the only per-tuple memory access is the
// {j^-q, 1/j} entry of the class-size table, staged once per CTA in shared
// memory (one 16-byte load; n = C[b+1] - C[a+1] is sorted across the lanes,
// so the loads mostly fall in distinct banks).  Value of (a, b):
//   (1 (x) T(0, a)) (x) (T(a+1, b) (x) Asuf[b])     -- the expression tree of
// every other search kernel, class terms from the same arithmetic.
// Items are claimed per warp from a global counter in (i-major, z) order, so
// the large early blocks go first (LPT) and the small late ones fill the tail.
// Unit u of U owns the a-blocks i == u (mod U): a rank-independent partition.
// Each item writes its own (score, key) partial to item_score/key[i][z];
// k_merge_items folds them per (unit, slice) under the total order.
constexpr int kK2Rows = 4;  // rows in flight per lane (tables are padded by >= kK2Rows entries)
constexpr int kK1Q = 128;   // k^(1-q) table of the pruned k = 2 search (classes of < 128 bins)

// The class term of the k = 2 kernel: class_term_nw<MODE> with the polynomial
// degree fixed at compile time and the 2^-s scaling on the exponent field --
// bit-identical values (same operations, same order).
template <int MODE, int DEG, class Tab>
__device__ __forceinline__ double k2_term(const Luts &l, const Tab &tab, uint32_t n, double w) {
  uint32_t j, r;
  int s;
  nsplit_idx(n, j, s, r);
  const double2 e = tab.jr(j);
  if (MODE == PROD_MAX || MODE == PROD_MIN) {
    const double d = scale_pow2_neg(__dmul_rn((double)r, e.y), s, r);
    const double ip = __dmul_rn(__dmul_rn(e.x, tab.p2(s)), horner_c_deg<DEG>(l, d));
    return __dmul_rn(w, ip);
  } else {
    return shannon_t(l, tab, n, w);
  }
}

// One warp's tile of slice positions (k = 2): lane l owns a = 32 i + l and
// walks b in [max(32 i + 1, blo), min(M - 2, bhi)] kK2Rows rows at a time;
// returns the lane's best (score, key) (not yet warp-reduced).  rz = the
// slice's K2Row table.  Every k = 2 kernel (k_search_k2: whole a-blocks; the
// stream pipeline: 2-D tiles) runs this body, so a tuple's value is the same
// expression tree everywhere.
//
// PRUNE (PROD_MAX only, i.e. pseudo-additive with q < 1; `best` enters as
// the slice's seed score): before a bulk group of kK2Rows rows b0..b0+3 is
// evaluated, each lane bounds its four values from above by
//   Apre[a] * (W[b0+3] - W[a]) * ub(n(a, b0)^-q) * max_r Asuf[b0+r]
// -- W is non-decreasing in b, n(a, b) = C[b+1] - C[a+1] is increasing, so
// n^-q is decreasing (q > 0), and ub(n^-q) = j^-q 2^(-s q) >= n^-q drops the
// (1 + d)^-q <= 1 factor of k2_term (a 0.1 % looser bound for one DMUL
// instead of a degree-5..12 polynomial) -- and the warp skips the group when
// no lane's bound, widened by 2^-20 relative (far above the few-ulp rounding
// of either side), reaches the lane's best.  A skipped tuple therefore scores
// strictly below a score some evaluated tuple (or the seed tuple) reaches, so
// it is neither the argmax nor tied with it: the result is the exhaustive
// search's, bit for bit.  The first 32 columns (lanes with a >= b) and the
// last partial group are always evaluated.
// The bound's inputs come from per-slice records (k_k2_seed, K2Chk: one
// 16-byte load): ck4[b0+1] = {W at row b0+3 rounded up, max Asuf over rows
// b0..b0+3 rounded up to float, C at row b0} for a group and
// ck16[b0+1] the same over rows b0..b0+15, checked first for every 16 rows
// (two 16-byte loads per check instead of the group's eight row loads: the
// first pruned version was L1-bound, ncu 93 % L1/TEX throughput).
template <int MODE, int DEG, bool NC = true, bool PRUNE = false, class Tab = SpPair>
__device__ __forceinline__ void k2_tile(const K2Row *rz, const int M, const int i, const int blo, const int bhi,
                                        const int lane, const Luts &l, const Tab &tab, double &best,
                                        uint64_t &bestkey, const K2Chk *ck4 = nullptr,
                                        const K2Chk *ck16 = nullptr) {
  static_assert(!PRUNE || MODE == PROD_MAX, "k = 2 pruning bounds the product form with q < 1");
  const double ident = MODE == SUM ? 0.0 : 1.0;
  const int a = 32 * i + lane;
  const int ac = min(a, M - 3);  // lanes past the slice stay idle (masked below)
  const K2Row ra = rz[ac + 1];
  const uint32_t Ca = ra.c;
  const double Wah = ra.wh, Wal = ra.wl;
  // Apre[a] = T(0, a) = class term of positions [0, a]: n = C[a+1], w = W[a+1];
  // lanes past the slice (a > M-3) get NaN, which never compares >= best
  const double pre0 = combine<MODE>(ident, k2_term<MODE, DEG>(l, tab, Ca, dd_diff(Wah, Wal, 0.0, 0.0)));
  const double pre = a <= M - 3 ? pre0 : CUDART_NAN;
  const int bend = min(M - 2, bhi);
  // one group of kK2Rows second thresholds b0 .. b0+kK2Rows-1; CHK: test
  // a < b and b <= bend per tuple (the first 32 columns of the block, where
  // some lanes have a >= b, and the last partial group), else none
  const double preub = PRUNE ? __dmul_rn(pre, 1.0 + 0x1p-20) : 0.0;
  // some lane's bound over the rows of record ck reaches its best
  // (NaN -- lanes past the slice -- never asks for the rows)
  // In the first 32 columns (chk groups) a lane's valid rows are b > a: for
  // a >= b0 the smallest class is n(a, a+1) (nfirst), and a lane with
  // a >= b0 + 3 has none.
  const uint32_t nfirst = PRUNE ? rz[min(ac + 2, M - 1)].c - Ca : 0u;
  // x = W at the record's last row, y = (max Asuf, (C at its first row, -))
  // Near the diagonal the middle class holds few non-empty bins and the
  // W-based bound is loose; there the power-mean inequality
  // sum_{i in C} c_i^q <= k^(1-q) (sum c_i)^q, k = #bins of C (q < 1), bounds
  // the middle class term by k^(1-q) <= kmax^(1-q), kmax = b0 + span - 1 - a
  // (tab.k1q, one shared load), and the smaller bound is used.
  // x = the record as {wub, (amax float bits | c << 32)} (K2Chk)
  auto live_xy = [&](const double2 x, const bool chk, const int b0, const int span) -> bool {
    uint32_t j, rr, n = (uint32_t)__double2hiint(x.y) - Ca;
    if (chk && a >= b0) n = nfirst;
    int s;
    nsplit_idx(n, j, s, rr);
    const double amax = (double)__int_as_float(__double2loint(x.y));
    const double ipub = __dmul_rn(tab.jr(j).x, tab.p2(s));
    double bound = __dmul_rn(__dmul_rn(preub, ipub), __dmul_rn(dd_diff(x.x, 0.0, Wah, Wal), amax));
    const int kmax = b0 + span - 1 - a;
    if (kmax < kK1Q) bound = fmin(bound, __dmul_rn(__dmul_rn(preub, tab.k1q[max(kmax, 0)]), amax));
    return __any_sync(0xffffffffu, (!chk || a < b0 + span - 1) && bound >= best);
  };
  auto live = [&](const K2Chk *ck, const bool chk, const int b0) -> bool {
    return live_xy(ldrow<NC>(reinterpret_cast<const double2 *>(ck)), chk, b0, kK2Rows);
  };
  // chkd: the group's bound was already checked (PRUNE) by the caller
  auto group = [&](const int b0, const bool chk, const bool chkd = false) {
    if (PRUNE && !chkd && !live(ck4 + b0 + 1, chk, b0)) return;
    const K2Row *pr = rz + b0 + 1;
    double vb[kK2Rows];
    double2 yv[kK2Rows], xv[kK2Rows];
#pragma unroll
    for (int r = 0; r < kK2Rows; r++) {
      xv[r] = ldrow<NC>(reinterpret_cast<const double2 *>(pr + r));      // wh, wl
      yv[r] = ldrow<NC>(reinterpret_cast<const double2 *>(pr + r) + 1);  // as, (c, bin)
    }
#pragma unroll
    for (int r = 0; r < kK2Rows; r++) {
      const double2 x = xv[r], y = yv[r];
      const uint32_t n = (uint32_t)__double2loint(y.y) - Ca;
      const double wm = dd_diff(x.x, x.y, Wah, Wal);
      const double R = combine<MODE>(k2_term<MODE, DEG>(l, tab, n, wm), y.x);
      double v = combine<MODE>(pre, R);
      if (MODE == PROD_MIN) v = -v;
      vb[r] = v;
    }
    // one predicate for the group (the exact update is rare once best is
    // good): no per-tuple branch / reconvergence (ncu: ~5 instructions per
    // tuple)
    bool any = false;
#pragma unroll
    for (int r = 0; r < kK2Rows; r++) any |= vb[r] >= best;
    if (!any) return;
#pragma unroll
    for (int r = 0; r < kK2Rows; r++) {
      const int b = b0 + r;
      if (vb[r] >= best && (!chk || (a < b && b <= bend))) {
        const uint64_t key = ((uint64_t)ra.bin << 12) | (uint64_t)__double2hiint(yv[r].y);
        if (better(vb[r], key, best, bestkey)) {
          best = vb[r];
          bestkey = key;
        }
      }
    }
  };
  int b0 = max(32 * i + 1, blo);
  for (; b0 <= bend && b0 < 32 * i + 32; b0 += kK2Rows) group(b0, true);
  if (PRUNE && b0 + 15 <= bend) {
    // records one 16-row block ahead (their L1/L2 latency was the top stall);
    // inside a live block the four group records are loaded together
    double2 nx = ldrow<NC>(reinterpret_cast<const double2 *>(ck16 + b0 + 1));
    for (; b0 + 15 <= bend; b0 += 16) {
      const double2 x = nx;
      if (b0 + 31 <= bend) nx = ldrow<NC>(reinterpret_cast<const double2 *>(ck16 + b0 + 17));
      if (live_xy(x, false, b0, 16)) {
        double2 gx[4];
#pragma unroll
        for (int g = 0; g < 4; g++) gx[g] = ldrow<NC>(reinterpret_cast<const double2 *>(ck4 + b0 + 4 * g + 1));
        unsigned lv = 0;
#pragma unroll
        for (int g = 0; g < 4; g++) lv |= live_xy(gx[g], false, b0 + 4 * g, kK2Rows) ? 1u << g : 0u;
#pragma unroll 1
        for (int g = 0; g < 4; g++)
          if (lv >> g & 1u) group(b0 + 4 * g, false, true);
      }
    }
  }
  for (; b0 + kK2Rows - 1 <= bend; b0 += kK2Rows) group(b0, false);
  if (b0 <= bend) group(b0, true);
}

template <int MODE, int DEG>
__device__ __forceinline__ void k2_block(const K2Row *rz, const int M, const int i, const int lane,
                                         const Luts &l, const SpPair &tab, double &best, uint64_t &bestkey) {
  k2_tile<MODE, DEG>(rz, M, i, 32 * i + 1, M - 2, lane, l, tab, best, bestkey);
}

#ifndef TSA_K2_MINB
#define TSA_K2_MINB 4  // minimum CTAs per SM of k_search_k2 (register cap: 64)
#endif
// k = 2 search: warp items (slice z, a-block i, b-tile t) from a global
// counter, a-block-major (longest blocks first), so every item is at most
// kK2Tile second thresholds long (a whole a-block is ~M per lane: round 1's
// items made the last ones a latency tail, and small slabs latency-bound).
// Tile partials go to item_score/key[(i * nbt + t)][z], nbt = tiles per block
// of the widest slice (from mmax); k_merge_items folds them per (unit, slice).
constexpr int kK2Tile = 4096;  // one tile per a-block: 128-wide tiles measured 7 % slower on c5 (606 vs 564 us)
__host__ __device__ __forceinline__ int k2_tiles(int m) { return m >= 3 ? (m - 2) / kK2Tile + 1 : 1; }

template <int MODE, int DEG, bool PRUNE = false>
__global__ void __launch_bounds__(256, TSA_K2_MINB) k_search_k2(SearchArgs g) {
  __shared__ double2 s_jr[kSN];
  __shared__ double s_p2[32];
  __shared__ double s_k1q[PRUNE ? kK1Q : 1];
  for (int i = threadIdx.x; i < kSN; i += blockDim.x) s_jr[i] = make_double2(g.luts.sp[i], g.luts.sp[kSN + i]);
  if (threadIdx.x < 32) s_p2[threadIdx.x] = g.luts.p2[threadIdx.x];
  if (PRUNE)  // k^(1-q): within an ulp (the bound's 2^-20 widening covers it)
    for (int k = threadIdx.x; k < kK1Q; k += blockDim.x) s_k1q[k] = pow((double)k, g.luts.omq);
  __syncthreads();
  const SpPair tab{s_jr, s_p2, s_k1q};
  const Luts &l = g.luts;
  const int lane = threadIdx.x & 31;
  const int mmax = *g.mmax;
  const int nbmax = mmax >= 3 ? (mmax - 3) / 32 + 1 : 0;  // a-blocks: a <= M-3
  const int nbt = k2_tiles(mmax);
  const int w = g.nunits, U = g.units, u0 = g.unit_begin;
  // blocks of this launch: i = (t / w) * U + u0 + t % w, t < nbl
  const int nbl = nbmax <= u0 ? 0 : ((nbmax - u0) / U) * w + min(w, (nbmax - u0) % U);
  const uint32_t nz = (uint32_t)g.nz;
  const uint32_t items = (uint32_t)nbl * nbt * nz;
  uint32_t itn = 0;  // claims one item ahead
  if (lane == 0) itn = (uint32_t)atomicAdd(g.counter, 1);
  for (;;) {
    const uint32_t it = __shfl_sync(0xffffffffu, itn, 0);
    if (it >= items) break;
    if (lane == 0) itn = (uint32_t)atomicAdd(g.counter, 1);
    const int tt = (int)(it / nz);
    const int z = (int)(it - (uint32_t)tt * nz);
    const int tb = tt / nbt, bt = tt - tb * nbt;
    const int i = (tb / w) * U + u0 + tb % w;
    const int M = g.Mz[z];
    const int blo = bt * kK2Tile, bhi = blo + kK2Tile - 1;
    // PRUNE: the seed enters with key none, so tuples scoring == seed are still taken
    double best = -CUDART_INF;
    uint64_t bestkey = kKeyNone;
    if (g.status[z] == kOK && 32 * i <= M - 3 && bhi >= 32 * i + 1 && blo <= M - 2) {
      if (PRUNE) best = g.seed[z];
      const K2Chk *ck = PRUNE ? g.chk + (size_t)z * g.RE : nullptr;
      k2_tile<MODE, DEG, true, PRUNE>(g.rows + (size_t)z * g.RE, M, i, blo, bhi, lane, l, tab, best, bestkey, ck,
                                      PRUNE ? ck + (size_t)g.nz * g.RE : nullptr);
      warp_argmax(best, bestkey);
    }
    if (lane == 0) {
      g.item_score[(size_t)(i * nbt + bt) * g.nz + z] = best;
      g.item_key[(size_t)(i * nbt + bt) * g.nz + z] = bestkey;
    }
  }
}

// Seed score of the pruned k = 2 search (k_search_k2<PROD_MAX, DEG, true>):
// one CTA per slice evaluates a coarse grid of tuples (a, b) = (S i, S j),
// S = ceil((M-1)/32), then one round of coordinate ascent (the best a for
// the grid's b over every position, then the best b for that a), and stores
// the value of the best tuple found (on the c5 phantom within ~1e-5 of the
// maximum; a third pass reaches it, but costs a block-wide step of latency
// for little extra pruning).  Values are k2_tile's expression tree
// (k2_value), so the seed equals that tuple's score in the search bit for
// bit, and the search, starting from (seed, key none), still finds every
// tuple scoring >= it.  The slice's packed rows are staged in shared memory
// when they fit (M <= kK2SeedRows).  Slices that are not searched get -inf.
template <int MODE, int DEG, class Tab>
__device__ __forceinline__ double k2_value(const K2Row *rz, const int a, const int b, const Luts &l, const Tab &tab) {
  const double ident = MODE == SUM ? 0.0 : 1.0;
  const K2Row ra = rz[a + 1], rb = rz[b + 1];
  const double pre = combine<MODE>(ident, k2_term<MODE, DEG>(l, tab, ra.c, dd_diff(ra.wh, ra.wl, 0.0, 0.0)));
  const double wm = dd_diff(rb.wh, rb.wl, ra.wh, ra.wl);
  const double R = combine<MODE>(k2_term<MODE, DEG>(l, tab, rb.c - ra.c, wm), rb.as);
  double v = combine<MODE>(pre, R);
  if (MODE == PROD_MIN) v = -v;
  return v;
}

constexpr int kK2SeedRows = 1024;  // rows staged in shared memory (32 KB)
#ifndef TSA_K2_SEED_GRID
#define TSA_K2_SEED_GRID 32  // side of the seed's coarse grid of (a, b)
#endif

// The per-slice body (k_k2_seed, and k_scan_seed after the slice's tables):
// srow = shared staging for up to `cap` rows; the early return is CTA-uniform.
template <int MODE, int DEG>
__device__ void k2_seed_body(const SearchArgs &g, const int z, K2Row *srow, const int cap) {
  const int M = g.Mz[z];
  if (g.status[z] != kOK || M < 3) {
    if (threadIdx.x == 0) g.seed[z] = -CUDART_INF;
    return;
  }
  const K2Row *rz = g.rows + (size_t)z * g.RE;
  if (M <= cap) {  // entries 0 .. M-1 (a + 1, b + 1 <= M - 1)
    for (int e = threadIdx.x; e < M; e += blockDim.x) srow[e] = rz[e];
    rz = srow;
  }
  __shared__ double s_p2[32];
  if (threadIdx.x < 32) s_p2[threadIdx.x] = g.luts.p2[threadIdx.x];
  __syncthreads();
  TSA_MPHASE(z, 3)
  // bound records of the search (k2_tile PRUNE): entry e = b0 + 1 covers rows
  // b0 .. b0+3 (chk4) / b0 .. b0+15 (chk16), clipped to the slice's last row
  // M-1 (records reaching past it are never read)
  {
    K2Chk *c4 = g.chk + (size_t)z * g.RE, *c16 = c4 + (size_t)g.nz * g.RE;
    for (int e = 1 + threadIdx.x; e <= M - 1; e += blockDim.x) {
      const int e4 = min(e + 3, M - 1), e16 = min(e + 15, M - 1);
      double m4 = rz[e].as, m16;
      for (int x = e + 1; x <= e4; x++) m4 = fmax(m4, rz[x].as);
      m16 = m4;
      for (int x = e4 + 1; x <= e16; x++) m16 = fmax(m16, rz[x].as);
      // upper bounds: W rounded up from its dd (hi + lo), Asuf max rounded up to float
      c4[e] = K2Chk{__dadd_ru(rz[e4].wh, rz[e4].wl), __double2float_ru(m4), rz[e].c};
      c16[e] = K2Chk{__dadd_ru(rz[e16].wh, rz[e16].wl), __double2float_ru(m16), rz[e].c};
    }
  }
  const SpGlobal tab{g.luts.sp, s_p2};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double ss[32];
  __shared__ uint64_t sk[32];
  // block argmax of (value desc, key asc); key = a << 16 | b
  auto reduce = [&](double v, uint64_t key) -> uint64_t {
    warp_argmax(v, key);
    __syncthreads();  // previous round's readers are done
    if (lane == 0) {
      ss[warp] = v;
      sk[warp] = key;
    }
    __syncthreads();
    v = lane < nw ? ss[lane] : -CUDART_INF;
    key = lane < nw ? sk[lane] : kKeyNone;
    warp_argmax(v, key);
    return key;  // every warp reduces the same entries: block-uniform
  };
  constexpr int GS = TSA_K2_SEED_GRID, GU = (GS * GS + 255) / 256;  // grid side, points per thread
  const int S = (M - 1 + GS - 1) / GS;
  double v = -CUDART_INF;
  uint64_t key = kKeyNone;
  {  // grid: GS x GS points, independent (their loads overlap)
    double x[GU];
    uint64_t kx[GU];
#pragma unroll
    for (int u = 0; u < GU; u++) {
      const int e = threadIdx.x + u * 256;
      const int a = S * (e / GS), b = S * (e % GS);
      const bool ok = e < GS * GS && a < b && b <= M - 2;
      x[u] = ok ? k2_value<MODE, DEG>(rz, a, b, g.luts, tab) : -CUDART_INF;
      kx[u] = ok ? (((uint64_t)a << 16) | (uint64_t)b) : kKeyNone;
    }
#pragma unroll
    for (int u = 0; u < GU; u++)
      if (better(x[u], kx[u], v, key)) {
        v = x[u];
        key = kx[u];
      }
  }
  TSA_MPHASE(z, 4)
  key = reduce(v, key);
  TSA_MPHASE(z, 5)
  int ta = key == kKeyNone ? 0 : (int)(key >> 16), tb = key == kKeyNone ? 1 : (int)(key & 0xffff);
  for (int pass = 0; pass < 2; pass++) {
    const bool move_a = pass == 0;
    const int lo = move_a ? 0 : ta + 1, hi = move_a ? tb - 1 : M - 2;
    v = -CUDART_INF;
    key = kKeyNone;
#pragma unroll 4
    for (int x = lo + threadIdx.x; x <= hi; x += blockDim.x) {
      const int a = move_a ? x : ta, b = move_a ? tb : x;
      const double y = k2_value<MODE, DEG>(rz, a, b, g.luts, tab);
      const uint64_t ky = ((uint64_t)a << 16) | (uint64_t)b;
      if (better(y, ky, v, key)) {
        v = y;
        key = ky;
      }
    }
    key = reduce(v, key);
    ta = (int)(key >> 16);
    tb = (int)(key & 0xffff);
  }
  TSA_MPHASE(z, 6)
  if (threadIdx.x == 0) g.seed[z] = k2_value<MODE, DEG>(rz, ta, tb, g.luts, tab);
}

template <int MODE, int DEG>
__global__ void __launch_bounds__(256) k_k2_seed(SearchArgs g) {
  __shared__ K2Row srow[kK2SeedRows];
  k2_seed_body<MODE, DEG>(g, blockIdx.x, srow, kK2SeedRows);
}

// Per (unit u in [u0, u1), slice z), one warp: fold the k = 2 tile partials of
// the blocks i == u (mod U), i < nblocks(z), tiles t < nbt(z), into
// part[u - u0][z] under the total order.
__global__ void k_merge_items(const double *is, const uint64_t *ik, const int32_t *Mz, const int32_t *status,
                              const int32_t *mmax, int64_t nz, int U, int u0, int nu, double *ps, uint64_t *pk) {
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nz * nu) return;  // warp-uniform
  const int64_t z = t % nz;
  const int u = u0 + (int)(t / nz);
  const int M = Mz[z];
  const int nb = (status[z] == kOK && M >= 3) ? (M - 3) / 32 + 1 : 0;
  const int nbt = k2_tiles(*mmax), nbz = k2_tiles(M);  // slot stride, tiles of this slice
  double s = -CUDART_INF;
  uint64_t k = kKeyNone;
  const int nblk = nb > u ? (nb - u + U - 1) / U : 0;  // blocks u, u + U, ...
  for (int e = lane; e < nblk * nbz; e += 32) {
    const int i = u + (e / nbz) * U, bt = e % nbz;
    const size_t o = (size_t)(i * nbt + bt) * nz + z;
    if (bt * kK2Tile + kK2Tile - 1 < 32 * i + 1) continue;  // a tile below the block: not written
    const double os = is[o];
    const uint64_t ok = ik[o];
    if (better(os, ok, s, k)) {
      s = os;
      k = ok;
    }
  }
  warp_argmax(s, k);
  if (lane == 0) {
    ps[(size_t)(u - u0) * nz + z] = s;
    pk[(size_t)(u - u0) * nz + z] = k;
  }
}

}  // namespace tsa
