// k_finalize.cuh -- SURVEY.md §8 row a4: argmax across work units (and ranks)
// under the total order (score desc, key asc), decode of t*, and phi(t*)
// recomputed from the histogram in the definition's order:
//   N = sum c_i; p_i = c_i / N; P_j = sequential sum of p_i over C_j;
//   A_j = sequential sum of (p_i/P_j)^q (q == 1: S_j = -sum r ln r);
//   S_j = (1 - A_j)/(q - 1); phi = left fold x (+) y = x + y + (1-q) x y
//   (or sum S + (1-q) prod S).
// Sums skip empty bins (adding +0.0 is exact) and run sequentially in ascending
// bin order on one lane; the pow/log terms run lane-parallel.  So the
// reported objective matches the oracle's to the last ulps of pow/log,
// whatever expression the search used to rank tuples.
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

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
  int32_t *status_out2;
};

__device__ __forceinline__ int class_of(int i, int t0, int t1, int t2, int t3) {
  return (i > t0) + (i > t1) + (i > t2) + (i > t3);
}

// One warp per slice.  Lane c <= k owns class c: it sums P_c and then A_c
// sequentially over the class's non-empty bins in ascending order (the
// definition's order); the p_i and pow/log terms are computed lane-parallel.
__global__ void __launch_bounds__(32) k_finalize(FinalizeArgs g) {
  extern __shared__ double fsh[];  // [L] p then terms, followed by int [L] bin list
  int *lst = reinterpret_cast<int *>(fsh + g.L);
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
      if (g.status_out2) g.status_out2[z] = st;
    }
    return;
  }
  // thresholds beyond k are "L": no bin is above them
  const int t0 = (int)((key >> (12 * (k - 1))) & 0xFFFull);
  const int t1 = k > 1 ? (int)((key >> (12 * (k - 2))) & 0xFFFull) : L;
  const int t2 = k > 2 ? (int)((key >> (12 * (k - 3))) & 0xFFFull) : L;
  const int t3 = k > 3 ? (int)(key & 0xFFFull) : L;
  if (lane < k) {
    const int tl = lane == 0 ? t0 : lane == 1 ? t1 : lane == 2 ? t2 : t3;
    g.thresholds[z * k + lane] = tl;
  }
  if (lane == 0) {
    if (g.status_out) g.status_out[z] = kOK;
    if (g.status_out2) g.status_out2[z] = kOK;
  }
  if (!g.objective_out) return;
  const uint32_t *h = g.hist + z * L;
  // N, the ordered list of non-empty bins, and per-class list lengths
  uint64_t nsum = 0;
  int m = 0;
  int cnt_mine = 0;  // lane c: number of non-empty bins in class c
  for (int i0 = 0; i0 < L; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t c = i < L ? __ldg(h + i) : 0u;
    nsum += c;
    const unsigned bal = __ballot_sync(0xffffffffu, c != 0);
    if (c) lst[m + __popc(bal & ((1u << lane) - 1u))] = i;
    m += __popc(bal);
    const int cls = c ? class_of(i, t0, t1, t2, t3) : -1;
#pragma unroll
    for (int cc = 0; cc <= kKMax; cc++) {
      const int n_c = __popc(__ballot_sync(0xffffffffu, cls == cc));
      if (lane == cc) cnt_mine += n_c;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, off);
  const double N = (double)nsum;  // exact: the oracle's sequential double sum of integers
  int start = cnt_mine;           // exclusive prefix of class lengths over lanes 0..k
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, start, off);
    if (lane >= off) start += o;
  }
  start -= cnt_mine;
  __syncwarp();
  for (int j = lane; j < m; j += 32) fsh[j] = __ddiv_rn((double)__ldg(h + lst[j]), N);
  __syncwarp();
  double P = 0.0;
  if (lane <= k)
    for (int j = start; j < start + cnt_mine; j++) P = __dadd_rn(P, fsh[j]);
  __syncwarp();
  const double q = g.q;
  const bool shannon = q == 1.0;
  __shared__ double Psh[kKMax + 1];
  if (lane <= k) Psh[lane] = P;
  __syncwarp();
  for (int j = lane; j < m; j += 32) {
    const int cls = class_of(lst[j], t0, t1, t2, t3);
    const double r = __ddiv_rn(fsh[j], Psh[cls]);
    fsh[j] = shannon ? __dmul_rn(r, log(r)) : pow(r, q);
  }
  __syncwarp();
  double A = 0.0;
  if (lane <= k)
    for (int j = start; j < start + cnt_mine; j++)
      A = shannon ? __dsub_rn(A, fsh[j]) : __dadd_rn(A, fsh[j]);
  const double Sl = shannon ? A : __ddiv_rn(__dsub_rn(1.0, A), __dsub_rn(q, 1.0));
  double S[kKMax + 1];
#pragma unroll
  for (int j = 0; j <= kKMax; j++) S[j] = __shfl_sync(0xffffffffu, Sl, j);
  if (lane == 0) {
    double phi;
    if (g.objective == 1) {
      double sum = 0.0, prod = 1.0;
#pragma unroll
      for (int j = 0; j <= kKMax; j++)
        if (j <= k) sum = __dadd_rn(sum, S[j]);
#pragma unroll
      for (int j = 0; j <= kKMax; j++)
        if (j <= k) prod = __dmul_rn(prod, S[j]);
      phi = __dadd_rn(sum, __dmul_rn(__dsub_rn(1.0, q), prod));
    } else {
      phi = S[0];
#pragma unroll
      for (int j = 1; j <= kKMax; j++)
        if (j <= k)
          phi = __dadd_rn(__dadd_rn(phi, S[j]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, q), phi), S[j]));
    }
    g.objective_out[z] = phi;
  }
}

}  // namespace tsa
