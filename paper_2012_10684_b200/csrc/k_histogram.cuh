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

// u16 data (12-bit CT, up to 4096 bins), round 2.  One copy of the bins per
// CTA plus an overflow slot [L]: every v >= L is counted there (a branch-free
// range check; LEVEL_OVERFLOW iff the slot is non-zero), so each voxel is
// extract + min + one shared reduction (red.shared.add.u32 -> ATOMS.POPC.INC,
// which merges same-address lanes of a warp).  ~128 K voxels per CTA.
// Round 1's kernel spent more issue slots on zeroing/flushing four 16 KB bin
// copies per 64 KB chunk and on a branch per voxel than on the atomics (ncu:
// 25 instructions per voxel, issue-bound at 2.6 TB/s on c5).
__device__ __forceinline__ void red_inc(uint32_t base, uint32_t v, uint32_t L) {
  const uint32_t addr = base + 4u * min(v, L);
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}

__global__ void __launch_bounds__(512) k_hist16(HistArgs g) {
  extern __shared__ uint32_t sh[];  // [L + 1]
  const int z = (int)(g.z0 + blockIdx.y);
  const int L = g.L;
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sh);
  const uint16_t *slice = reinterpret_cast<const uint16_t *>(g.vol) + (size_t)z * g.n;
  const uintptr_t addr0 = reinterpret_cast<uintptr_t>(slice);
  int64_t head = (int64_t)(((16 - (addr0 & 15)) & 15) / 2);
  if (head > g.n) head = g.n;
  const int64_t nvec = (g.n - head) / 8;
  const int64_t tail0 = head + nvec * 8;
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice + head);
  const int64_t per = (nvec + g.chunks - 1) / g.chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec, v0 + per);
  const uint32_t UL = (uint32_t)L;
  constexpr int U = 2;
  for (int64_t i0 = v0 + threadIdx.x; i0 < v1; i0 += (int64_t)U * blockDim.x) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      if (i < v1) w[u] = __ldcs(v4 + i);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (i0 + (int64_t)u * blockDim.x >= v1) break;
      red_inc(base, w[u].x & 0xffffu, UL);
      red_inc(base, w[u].x >> 16, UL);
      red_inc(base, w[u].y & 0xffffu, UL);
      red_inc(base, w[u].y >> 16, UL);
      red_inc(base, w[u].z & 0xffffu, UL);
      red_inc(base, w[u].z >> 16, UL);
      red_inc(base, w[u].w & 0xffffu, UL);
      red_inc(base, w[u].w >> 16, UL);
    }
  }
  if (blockIdx.x == 0) {  // unaligned head / tail
    for (int64_t i = threadIdx.x; i < head; i += blockDim.x) red_inc(base, slice[i], UL);
    for (int64_t i = tail0 + threadIdx.x; i < g.n; i += blockDim.x) red_inc(base, slice[i], UL);
  }
  __syncthreads();
  uint32_t *out = g.hist + (size_t)z * L;
  for (int b = threadIdx.x; b < L; b += blockDim.x) {
    const uint32_t c = sh[b];
    if (c) atomicAdd(out + b, c);
  }
  if (threadIdx.x == 0 && sh[L]) g.status[z] = kLevelOverflow;
}

}  // namespace tsa
