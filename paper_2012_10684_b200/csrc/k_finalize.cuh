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

// One CTA (kFinThreads) per slice.  Warp 0 merges the partials; the CTA
// builds the ascending list of non-empty bins (per-thread bin ranges + a block
// scan), computes p_i = c_i/N and the pow/log terms thread-parallel, and
// thread c <= k sums P_c and then A_c sequentially over its class's list
// segment in ascending bin order (the definition's order).
constexpr int kFinThreads = 256;

// The per-slice body (also run by the stream pipeline's label tasks, k_stream.cuh):
// fsh = [L] doubles followed by [L] ints of shared memory; blockDim.x ==
// kFinThreads; the early returns are CTA-uniform.
// phi_only: thresholds and statuses were written by k_decide (same merge,
// same decisions); only the objective is written.
__device__ void finalize_slice(const FinalizeArgs &g, const int64_t z, double *fsh, uint32_t *hsm = nullptr,
                               const bool phi_only = false) {
  int *lst = reinterpret_cast<int *>(fsh + g.L);
  __shared__ double s_best[1];
  __shared__ uint64_t s_key[1];
  __shared__ int s_cnt[kFinThreads / 32 + 1];
  __shared__ unsigned long long s_n[kFinThreads / 32];
  __shared__ int s_start[kKMax + 2];
  __shared__ double Psh[kKMax + 1], Ssh[kKMax + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kFinThreads / 32;
  if (warp == 0) {
    double s = -CUDART_INF;
    uint64_t key = kKeyNone;
    // L2 loads: in the stream pipeline these come from another CTA of a
    // running kernel (no stale L1 lines of neighbouring slices)
    for (int p = lane; p < g.nparts; p += 32) {
      const double os = __ldcg(g.ps + (size_t)p * g.nz + z);
      const uint64_t ok = __ldcg(g.pk + (size_t)p * g.nz + z);
      if (better(os, ok, s, key)) {
        s = os;
        key = ok;
      }
    }
    warp_argmax(s, key);
    if (lane == 0) {
      s_best[0] = s;
      s_key[0] = key;
    }
  }
  __syncthreads();
  const uint64_t key = s_key[0];
  int st = __ldcg(g.status_in + z);
  if (st == kOK && key == kKeyNone) st = kNoValidSplit;
  const int k = g.k, L = g.L;
  if (st != kOK) {
    if (tid < k && !phi_only) g.thresholds[z * k + tid] = -1;
    if (tid == 0) {
      if (g.objective_out) g.objective_out[z] = CUDART_NAN;
      if (g.status_out && !phi_only) g.status_out[z] = st;
      if (g.status_out2 && !phi_only) g.status_out2[z] = st;
    }
    return;
  }
  // thresholds beyond k are "L": no bin is above them
  const int t0 = (int)((key >> (12 * (k - 1))) & 0xFFFull);
  const int t1 = k > 1 ? (int)((key >> (12 * (k - 2))) & 0xFFFull) : L;
  const int t2 = k > 2 ? (int)((key >> (12 * (k - 3))) & 0xFFFull) : L;
  const int t3 = k > 3 ? (int)(key & 0xFFFull) : L;
  if (tid < k && !phi_only) {
    const int tl = tid == 0 ? t0 : tid == 1 ? t1 : tid == 2 ? t2 : t3;
    g.thresholds[z * k + tid] = tl;
  }
  if (tid == 0 && !phi_only) {
    if (g.status_out) g.status_out[z] = kOK;
    if (g.status_out2) g.status_out2[z] = kOK;
  }
  if (!g.objective_out) return;
  // the histogram: staged into shared memory when the caller gives room
  // (k_finalize), else read through L2
  const uint32_t *h = g.hist + z * L;
  if (hsm) {
    for (int i = tid; i < L; i += kFinThreads) hsm[i] = __ldcg(h + i);
    __syncthreads();
    h = hsm;
  }
  auto ldh = [&](int i) -> uint32_t { return hsm ? hsm[i] : __ldcg(h + i); };
  // ordered list of non-empty bins: thread t owns bins [t*per, (t+1)*per)
  const int per = (L + kFinThreads - 1) / kFinThreads;
  const int i0 = min(L, tid * per), i1 = min(L, i0 + per);
  // L = 1024 / 4096 (per = 4 / 16) from global memory: the thread's bins in
  // registers from up to four 16-byte loads issued together (round 1 walked
  // them with one dependent L2 round trip per bin: ~half of the c5 finalize)
  const bool vec = !hsm && (per == 4 || per == 16) && L == per * kFinThreads &&
                   (reinterpret_cast<uintptr_t>(h) & 15) == 0;
  uint32_t cv[16];
  if (vec) {
    const uint4 *h4 = reinterpret_cast<const uint4 *>(h + i0);
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const uint4 x = v < per / 4 ? __ldcg(h4 + v) : make_uint4(0u, 0u, 0u, 0u);
      cv[4 * v] = x.x;
      cv[4 * v + 1] = x.y;
      cv[4 * v + 2] = x.z;
      cv[4 * v + 3] = x.w;
    }
  }
  int cnt = 0;
  unsigned long long nsum = 0;
  if (vec) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      cnt += cv[u] != 0;
      nsum += cv[u];
    }
  } else {
    for (int i = i0; i < i1; i++) {
      const uint32_t c = ldh(i);
      cnt += c != 0;
      nsum += c;
    }
  }
  int ex = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, ex, off);
    if (lane >= off) ex += o;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, off);
  if (lane == 31) s_cnt[warp] = ex;
  if (lane == 0) s_n[warp] = nsum;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < NW; w++) {
      const int c = s_cnt[w];
      s_cnt[w] = acc;
      acc += c;
    }
    s_cnt[NW] = acc;
    unsigned long long n = 0;
    for (int w = 0; w < NW; w++) n += s_n[w];
    s_n[0] = n;
  }
  __syncthreads();
  const int m = s_cnt[NW];
  int e = s_cnt[warp] + ex - cnt;
  // the list entry and its count (fsh is free until p is formed)
  if (vec) {
#pragma unroll
    for (int u = 0; u < 16; u++)
      if (cv[u]) {
        lst[e] = i0 + u;
        fsh[e++] = (double)cv[u];
      }
  } else {
    for (int i = i0; i < i1; i++) {
      const uint32_t c = ldh(i);
      if (c) {
        lst[e] = i;
        fsh[e++] = (double)c;
      }
    }
  }
  const double N = (double)s_n[0];  // exact: the oracle's sequential double sum of integers
  __syncthreads();
  // class c = list segment [start_c, start_{c+1}): first entry with bin > t_{c-1}
  if (tid <= k + 1) {
    int tv = tid == 0 ? -1 : tid == 1 ? t0 : tid == 2 ? t1 : tid == 3 ? t2 : t3;
    if (tid == k + 1) tv = L;  // end
    int lo = 0, hi = m;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lst[mid] > tv) hi = mid;
      else lo = mid + 1;
    }
    s_start[tid] = tid == k + 1 ? m : lo;
  }
  for (int j = tid; j < m; j += kFinThreads) fsh[j] = __ddiv_rn(fsh[j], N);
  __syncthreads();
  // sequential sums in ascending order; the shared loads of 8 terms are
  // issued ahead of their 8 dependent adds (round 2: one load latency per
  // term made the k = 2 c5 finalize 51 us) -- the same additions in the same order
  auto seqsum = [&](const int j0, const int j1, const bool neg) -> double {
    double acc = 0.0;
    int j = j0;
    for (; j + 8 <= j1; j += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; u++) x[u] = fsh[j + u];
#pragma unroll
      for (int u = 0; u < 8; u++) acc = neg ? __dsub_rn(acc, x[u]) : __dadd_rn(acc, x[u]);
    }
    for (; j < j1; j++) acc = neg ? __dsub_rn(acc, fsh[j]) : __dadd_rn(acc, fsh[j]);
    return acc;
  };
  if (tid <= k) Psh[tid] = seqsum(s_start[tid], s_start[tid + 1], false);
  __syncthreads();
  const double q = g.q;
  const bool shannon = q == 1.0;
  for (int j = tid; j < m; j += kFinThreads) {
    const int cls = class_of(lst[j], t0, t1, t2, t3);
    const double r = __ddiv_rn(fsh[j], Psh[cls]);
    fsh[j] = shannon ? __dmul_rn(r, log(r)) : pow(r, q);
  }
  __syncthreads();
  if (tid <= k) {
    const double A = seqsum(s_start[tid], s_start[tid + 1], shannon);
    Ssh[tid] = shannon ? A : __ddiv_rn(__dsub_rn(1.0, A), __dsub_rn(q, 1.0));
  }
  __syncthreads();
  if (tid == 0) {
    double phi;
    if (g.objective == 1) {
      double sum = 0.0, prod = 1.0;
      for (int j = 0; j <= k; j++) sum = __dadd_rn(sum, Ssh[j]);
      for (int j = 0; j <= k; j++) prod = __dmul_rn(prod, Ssh[j]);
      phi = __dadd_rn(sum, __dmul_rn(__dsub_rn(1.0, q), prod));
    } else {
      phi = Ssh[0];
      for (int j = 1; j <= k; j++)
        phi = __dadd_rn(__dadd_rn(phi, Ssh[j]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, q), phi), Ssh[j]));
    }
    g.objective_out[z] = phi;
  }
}

// The staged step with labels splits k_finalize: k_decide (one warp per
// slice: the merge, t* and the statuses -- all the labels need), then the
// label kernel launched with Programmatic Dependent Launch, and
// k_finalize_phi (phi(t*) only) as ITS dependent: it needs nothing from the
// labels, so its CTAs run next to the label CTAs (which leave one CTA slot
// per SM, tsa_api.cu) instead of before them, and it ends with
// griddepcontrol.wait so its completion implies the labels' (later stream
// work stays ordered after both).
__global__ void k_decide(FinalizeArgs g) {
  const int64_t z = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (z >= g.nz) return;  // warp-uniform
  double sc = -CUDART_INF;
  uint64_t key = kKeyNone;
  for (int p = lane; p < g.nparts; p += 32) {
    const double os = g.ps[(size_t)p * g.nz + z];
    const uint64_t ok = g.pk[(size_t)p * g.nz + z];
    if (better(os, ok, sc, key)) {
      sc = os;
      key = ok;
    }
  }
  warp_argmax(sc, key);
  int st = g.status_in[z];
  if (st == kOK && key == kKeyNone) st = kNoValidSplit;
  const int k = g.k;
  if (lane < k) {
    int tl = -1;
    if (st == kOK) tl = (int)((key >> (12 * (k - 1 - lane))) & 0xFFFull);
    g.thresholds[z * k + lane] = tl;
  }
  __syncwarp();
  if (lane == 0) {
    if (g.status_out) g.status_out[z] = st;
    if (g.status_out2) g.status_out2[z] = st;
  }
}

__global__ void __launch_bounds__(kFinThreads) k_finalize_phi(FinalizeArgs g) {
  extern __shared__ double fsh[];
  finalize_slice(g, blockIdx.x, fsh, nullptr, true);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // completion implies the primary's (labels)
}

__global__ void __launch_bounds__(kFinThreads) k_finalize(FinalizeArgs g) {
  extern __shared__ double fsh[];  // [L] p then terms, int [L] bin list
  // (staging the histogram in shared memory as well measured slower on c5,
  // 57 vs 52 us: 64 KB per CTA leaves 3 CTAs per SM instead of 4)
  finalize_slice(g, blockIdx.x, fsh);
}

}  // namespace tsa
