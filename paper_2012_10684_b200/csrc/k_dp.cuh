// k_dp.cuh -- SURVEY.md §8(f) NEXT row 4: an exact algorithmic variant of the
// a3 search for the pseudo-additive objective.  The fold is a product over
// classes, phi = (prod_j A_j - 1)/(1 - q) (R1), so the argmax over tuples is
// the argmax of sum_j g(C_j) with g = +ln A (q < 1), -ln A (q > 1), or the
// Shannon S (q == 1, phi = sum S_j): a shortest-path / interval DP
//   suf_k(a) = g([a, M-1]),   suf_j(a) = max_{b} g([a, b]) + suf_{j+1}(b+1)
// over the m canonical positions (non-empty bins; every class non-empty), in
// O(k m^2) class terms instead of C(m-1, k) tuples.  The tuple is rebuilt
// left to right taking the SMALLEST b whose (recomputed, bit-identical) value
// equals the optimum, i.e. the lexicographically smallest optimum of the DP
// objective.  It equals the exhaustive argmax except where two partitions'
// objectives differ only by rounding (the near-tie exception of the parity
// rule; tested against the oracle and the exhaustive kernels).
// The result goes to the same (score, key) partials as the exhaustive search,
// so tsa_finalize recomputes phi(t*) from the histogram as usual.
// Not applicable to SUM_PLUS_PRODUCT (not a sum over classes).
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

template <int MODE>
__device__ __forceinline__ double dp_term(const SliceTables &t, const Luts &l, int a, int b) {
  if (MODE == SUM) return class_term<SUM>(t, l, a, b);
  const double A = class_term<PROD_MAX>(t, l, a, b);  // W / n^q > 0
  return MODE == PROD_MAX ? log(A) : -log(A);
}

// Triangular table of the class terms g([a, b]), 0 <= a <= b < M, row a at
// offset a*M - a*(a-1)/2 (each term -- a double-double difference, a LUT
// gather and a log -- evaluated once, all in parallel).
__device__ __forceinline__ int tri_off(int a, int M) { return a * M - a * (a - 1) / 2; }

constexpr size_t kDpTableMax = 64 * 1024;  // term-table bytes (m <= 127; several CTAs per SM)

__host__ __device__ inline size_t dp_table_bytes(int M) { return (size_t)M * (M + 1) / 2 * sizeof(double); }

// One CTA per slice; dynamic shared memory: (k+1) * (L+1) doubles for the
// suffix values, then (when it fits the launch's tab_max <= kDpTableMax bytes)
// the term table; otherwise terms are evaluated on the fly in the level loops.
template <int MODE>
__global__ void __launch_bounds__(256) k_search_dp(SearchArgs g, int k, size_t tab_max) {
  extern __shared__ double suf[];  // suf[j * (L+1) + a], then the table
  const int z = blockIdx.x;
  const int st = g.status[z];
  const int M = g.Mz[z];
  const int S = g.L + 1;
  double *ps = g.part_score + z;
  uint64_t *pk = g.part_key + z;
  if (st != kOK || M < k + 1) {
    if (threadIdx.x == 0) {
      *ps = -CUDART_INF;
      *pk = kKeyNone;
    }
    return;
  }
  SliceTables t{g.C + (size_t)z * g.E, g.Whi + (size_t)z * g.E, g.Wlo + (size_t)z * g.E, nullptr};
  double *T = suf + (size_t)(k + 1) * S;
  const bool tab = dp_table_bytes(M) <= tab_max;
  if (tab) {
    const int ntri = M * (M + 1) / 2;
    for (int e = threadIdx.x; e < ntri; e += blockDim.x) {
      // invert e -> (a, b): row a holds M - a entries
      int a = (int)((2.0 * M + 1.0 - sqrt((2.0 * M + 1.0) * (2.0 * M + 1.0) - 8.0 * e)) / 2.0);
      while (a > 0 && tri_off(a, M) > e) a--;
      while (a + 1 < M && tri_off(a + 1, M) <= e) a++;
      const int b = a + (e - tri_off(a, M));
      T[e] = dp_term<MODE>(t, g.luts, a, b);
    }
    __syncthreads();
  }
  auto term = [&](int a, int b) -> double {
    return tab ? T[tri_off(a, M) + (b - a)] : dp_term<MODE>(t, g.luts, a, b);
  };
  // last class: [a, M-1], a >= k (classes 0..k-1 need a position each)
  for (int a = threadIdx.x; a < M; a += blockDim.x)
    suf[k * S + a] = a >= k ? term(a, M - 1) : -CUDART_INF;
  __syncthreads();
  for (int j = k - 1; j >= 0; j--) {
    // class j = [a, b] with a >= j and b <= M-1-(k-j); j == 0 only needs a == 0
    const int amax = j == 0 ? 0 : M - 1 - (k - j);
    for (int a = j + threadIdx.x; a <= amax; a += blockDim.x) {
      double best = -CUDART_INF;
      for (int b = a; b <= M - 1 - (k - j); b++) {
        const double v = __dadd_rn(term(a, b), suf[(j + 1) * S + b + 1]);
        if (v > best) best = v;
      }
      suf[j * S + a] = best;
    }
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    // lexicographically smallest optimum: the smallest b reproducing the
    // value (a warp checks 32 candidates per ballot)
    const int lane = threadIdx.x;
    uint64_t key = 0;
    int a = 0;
    for (int j = 0; j < k; j++) {
      const double target = suf[j * S + a];
      const int bmax = M - 1 - (k - j);
      int bsel = -1;
      for (int b0 = a; b0 <= bmax && bsel < 0; b0 += 32) {
        const int b = b0 + lane;
        const bool hit = b <= bmax && __dadd_rn(term(a, b), suf[(j + 1) * S + b + 1]) == target;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (m) bsel = b0 + __ffs(m) - 1;
      }
      const int bin = g.Bin[(size_t)z * g.E + bsel + 1];  // table entry = position + 1
      key = (key << 12) | (uint64_t)bin;
      a = bsel + 1;
    }
    if (lane == 0) {
      *ps = suf[0];
      *pk = key;
    }
  }
}

}  // namespace tsa
