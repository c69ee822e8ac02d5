// k_histogram.cuh -- SURVEY.md §8 row a1: per-slice gray-level histogram
// ("histogram of the brightness level"; c_i = #{v == i}).
//
// Design (measured on B200, profiles/r1_hist_variants.md): shared-memory
// atomics are the only per-voxel operation.  Each warp owns a private copy of
// the bins (no inter-warp contention), loads are 128-bit and coalesced, and
// the u8 / 256-bin case drops every range check (a u8 voxel is always < 256).
// Lane-private counters, thread-private u16 counters, __match_any_sync
// aggregation and zero-skipping were all measured slower.  The kernel is
// bound by shared-atomic throughput (~10 lane-atomics/clk/SM), not by HBM; the
// step hides this by overlapping it with the HBM-bound label pass.
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

struct HistArgs {
  const uint8_t *vol;  // byte pointer to the volume
  uint32_t *hist;      // [nz][L], zeroed before launch
  int32_t *status;     // [nz], zeroed before launch
  int64_t n;           // voxels per slice
  int64_t z0;          // first slice of this launch (slab pipelining)
  int L;
  int replicas;        // smem copies of the bins (<= warps per CTA)
  int chunks;          // CTAs per slice (gridDim.x)
};

template <typename T, bool CHECK>
__device__ __forceinline__ void hist_word(uint32_t *bins, uint32_t w, int L, int &ovf) {
  constexpr int PER = 4 / sizeof(T);
#pragma unroll
  for (int j = 0; j < PER; j++) {
    const uint32_t b = sizeof(T) == 1 ? (w >> (8 * j)) & 0xffu : (w >> (16 * j)) & 0xffffu;
    if (!CHECK) {
      atomicAdd(bins + b, 1u);
    } else if (b < (uint32_t)L) {
      atomicAdd(bins + b, 1u);
    } else {
      ovf = 1;
    }
  }
}

// CHECK = false only for u8 with L == 256.
template <typename T, bool CHECK>
__global__ void __launch_bounds__(512) k_histogram(HistArgs g) {
  extern __shared__ uint32_t sh[];
  const int z = (int)(g.z0 + blockIdx.y);
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
  const uintptr_t base = reinterpret_cast<uintptr_t>(slice);
  int64_t head = (int64_t)(((16 - (base & 15)) & 15) / sizeof(T));
  if (head > g.n) head = g.n;
  const int64_t nvec = (g.n - head) / VEC;
  const int64_t tail0 = head + nvec * VEC;
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice + head);
  const int64_t per = (nvec + g.chunks - 1) / g.chunks;
  const int64_t v0 = per * blockIdx.x;
  const int64_t v1 = min(nvec, v0 + per);
  int ovf = 0;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += nthr) {
    const uint4 w = __ldcs(v4 + i);
    hist_word<T, CHECK>(bins, w.x, L, ovf);
    hist_word<T, CHECK>(bins, w.y, L, ovf);
    hist_word<T, CHECK>(bins, w.z, L, ovf);
    hist_word<T, CHECK>(bins, w.w, L, ovf);
  }
  if (blockIdx.x == 0) {  // unaligned head / tail
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

// u16 data, large L (12-bit CT, 4096 bins): per-warp copies of 16-bit counters
// packed two per word (atomicAdd of 1 or 1<<16), so every warp gets its own
// copy within 128 KB of shared memory; a warp counts at most
// (slice / chunks) / warps < 65536 voxels, so no half-word overflows.
__global__ void __launch_bounds__(512) k_histogram_p16(HistArgs g) {
  extern __shared__ uint32_t sh[];
  const int z = (int)(g.z0 + blockIdx.y);
  const int L = g.L, LW = (L + 1) / 2;
  const int nthr = blockDim.x;
  const int rep = (threadIdx.x >> 5) % g.replicas;
  for (int i = threadIdx.x; i < LW * g.replicas; i += nthr) sh[i] = 0;
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  uint32_t *bins = sh + rep * LW;
  const uint16_t *slice = reinterpret_cast<const uint16_t *>(g.vol) + (size_t)z * g.n;
  const uintptr_t base = reinterpret_cast<uintptr_t>(slice);
  int64_t head = (int64_t)(((16 - (base & 15)) & 15) / 2);
  if (head > g.n) head = g.n;
  const int64_t nvec = (g.n - head) / 8;
  const int64_t tail0 = head + nvec * 8;
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice + head);
  const int64_t per = (nvec + g.chunks - 1) / g.chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec, v0 + per);
  int ovf = 0;
  auto add = [&](uint32_t b) {
    if (b < (uint32_t)L) atomicAdd(bins + (b >> 1), 1u << ((b & 1u) << 4));
    else ovf = 1;
  };
  for (int64_t i = v0 + threadIdx.x; i < v1; i += nthr) {
    const uint4 w = __ldcs(v4 + i);
    add(w.x & 0xffffu); add(w.x >> 16);
    add(w.y & 0xffffu); add(w.y >> 16);
    add(w.z & 0xffffu); add(w.z >> 16);
    add(w.w & 0xffffu); add(w.w >> 16);
  }
  if (blockIdx.x == 0) {
    for (int64_t i = threadIdx.x; i < head; i += nthr) add(slice[i]);
    for (int64_t i = tail0 + threadIdx.x; i < g.n; i += nthr) add(slice[i]);
  }
  if (ovf) overflow = 1;
  __syncthreads();
  uint32_t *out = g.hist + (size_t)z * L;
  for (int b = threadIdx.x; b < L; b += nthr) {
    uint32_t s = 0;
    for (int r = 0; r < g.replicas; r++) s += (sh[r * LW + (b >> 1)] >> ((b & 1) << 4)) & 0xffffu;
    if (s) atomicAdd(out + b, s);
  }
  if (threadIdx.x == 0 && overflow) g.status[z] = kLevelOverflow;
}

}  // namespace tsa
