// tools/hist_variants.cu -- micro-benchmark of u8 histogram / label kernel
// variants on a real phantom volume (design exploration; the product kernels
// live in paper_2012_10684_b200/csrc).  Usage: hist_variants <raw u8 file> nz ny nx
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// (a) per-warp replicas, ATOMS, no range checks (L = 256), uniform fast path
template <bool FAST>
__global__ void __launch_bounds__(512) h_atoms(const uint4 *v, uint32_t *hist, int64_t nvec_slice, int chunks) {
  __shared__ uint32_t sh[16][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t *b = sh[threadIdx.x >> 5];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + chunks - 1) / chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    const uint4 w = s[i];
    if (FAST && w.x == w.y && w.x == w.z && w.x == w.w && w.x == (w.x & 0xff) * 0x01010101u) {
      atomicAdd(b + (w.x & 0xff), 16u);
      continue;
    }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int j = 0; j < 4; j++) atomicAdd(b + ((ws[q] >> (8 * j)) & 0xff), 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}

// (b) thread-private u16 counters [bin][T] (T = 128), persistent contiguous
// ranges with flush at slice boundaries, uniform fast path, UNROLL loads.
template <int T, int UNROLL, bool FAST>
__global__ void __launch_bounds__(T) h_private(const uint8_t *vol, uint32_t *hist, int64_t n, int64_t nz) {
  extern __shared__ uint16_t cnt[];  // [256][T]
  const int tid = threadIdx.x;
  const int64_t total16 = n * nz / 16;
  const int64_t a = total16 * blockIdx.x / gridDim.x, bnd = total16 * (blockIdx.x + 1) / gridDim.x;
  const int64_t per_slice16 = n / 16;
  for (int i = tid; i < 256 * T / 8; i += T) reinterpret_cast<uint4 *>(cnt)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  int64_t i = a;
  const uint4 *v4 = reinterpret_cast<const uint4 *>(vol);
  while (i < bnd) {
    const int64_t z = i / per_slice16;
    const int64_t e = min(bnd, (z + 1) * per_slice16);
    // main loop over [i, e)
    int64_t j = i + tid;
    for (; j + (UNROLL - 1) * T < e; j += UNROLL * T) {
      uint4 w[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; u++) w[u] = __ldcs(v4 + j + u * T);
#pragma unroll
      for (int u = 0; u < UNROLL; u++) {
        if (FAST && w[u].x == w[u].y && w[u].x == w[u].z && w[u].x == w[u].w &&
            w[u].x == (w[u].x & 0xff) * 0x01010101u) {
          uint16_t *c = cnt + (w[u].x & 0xff) * T + tid;
          *c = *c + 16;
          continue;
        }
        const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            uint16_t *c = cnt + ((ws[q] >> (8 * jj)) & 0xff) * T + tid;
            *c = *c + 1;
          }
      }
    }
    for (; j < e; j += T) {
      const uint4 w = __ldcs(v4 + j);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          uint16_t *c = cnt + ((ws[q] >> (8 * jj)) & 0xff) * T + tid;
          *c = *c + 1;
        }
    }
    __syncthreads();
    // flush: thread b sums bins b, b+T, ... over all T counters (rotated to avoid conflicts)
    for (int bin = tid; bin < 256; bin += T) {
      const uint32_t *row = reinterpret_cast<const uint32_t *>(cnt + bin * T);
      uint32_t s = 0;
      for (int c = 0; c < T / 2; c++) {
        const uint32_t x = row[(c + tid) % (T / 2)];
        s += (x & 0xffff) + (x >> 16);
      }
      if (s) atomicAdd(hist + z * 256 + bin, s);
    }
    __syncthreads();
    if (e < bnd) {
      for (int q = tid; q < 256 * T / 8; q += T) reinterpret_cast<uint4 *>(cnt)[q] = make_uint4(0, 0, 0, 0);
      __syncthreads();
    }
    i = e;
  }
}


// V1/V2: SWAR zero count in a register, atomics only for non-zero bytes; V2 adds
// a warp-uniform skip of all-zero vectors.  COPIES per warp: 1 or 2 (half-warps).
__device__ __forceinline__ uint32_t zero_bytes(uint32_t w) {
  uint32_t t = (w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
  t = ~(t | w | 0x7F7F7F7Fu);
  return __popc(t);
}
template <int MODE, int COPIES>
__global__ void __launch_bounds__(512) h_atoms2(const uint4 *v, uint32_t *hist, int64_t nvec_slice, int chunks) {
  __shared__ uint32_t sh[16 * COPIES][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * COPIES * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t *b = sh[(threadIdx.x >> 5) * COPIES + (COPIES == 2 ? (lane >> 4) : 0)];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + chunks - 1) / chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  uint32_t zeros = 0;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    const uint4 w = s[i];
    if (MODE == 0) {
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int j = 0; j < 4; j++) atomicAdd(b + ((ws[q] >> (8 * j)) & 0xff), 1u);
      continue;
    }
    const bool allzero = (w.x | w.y | w.z | w.w) == 0;
    if (MODE == 2 && __all_sync(0xffffffffu, allzero)) { zeros += 16; continue; }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      zeros += zero_bytes(ws[q]);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t x = (ws[q] >> (8 * j)) & 0xff;
        if (x) atomicAdd(b + x, 1u);
      }
    }
  }
  atomicAdd(b, zeros);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16 * COPIES; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}
// V6: __match_any_sync aggregation per byte slot
__global__ void __launch_bounds__(512) h_match(const uint4 *v, uint32_t *hist, int64_t nvec_slice, int chunks) {
  __shared__ uint32_t sh[16][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t *b = sh[threadIdx.x >> 5];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + chunks - 1) / chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  for (int64_t i0 = v0; i0 < v1; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool act = i < v1;
    const uint4 w = act ? s[i] : make_uint4(0, 0, 0, 0);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t x = act ? ((ws[q] >> (8 * j)) & 0xff) : 0x100u + lane;
        const uint32_t m = __match_any_sync(0xffffffffu, x);
        if (act && (__ffs(m) - 1) == lane) atomicAdd(b + x, (uint32_t)__popc(m));
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}
// hist with L2 evict_last loads (leave the volume in L2 for the label pass)
__global__ void __launch_bounds__(512) h_atoms_keep(const uint4 *v, uint32_t *hist, int64_t nvec_slice, int chunks) {
  __shared__ uint32_t sh[16][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t *b = sh[threadIdx.x >> 5];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + chunks - 1) / chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    uint4 w;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(s + i), "l"(pol));
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int j = 0; j < 4; j++) atomicAdd(b + ((ws[q] >> (8 * j)) & 0xff), 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}


// V7: lane-private packed u16x2 counters [bin/2][lane] (16 KB per warp), ATOMS
// (no same-address or bank conflicts by construction), warp-contiguous ranges
// over the whole volume, flush at slice boundaries.
template <int WARPS, int UNROLL>
__global__ void __launch_bounds__(WARPS * 32) h_lane(const uint8_t *vol, uint32_t *hist, int64_t n, int64_t nz) {
  extern __shared__ uint32_t smc[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *c = smc + wid * (128 * 32);
  const int64_t W = (int64_t)gridDim.x * WARPS;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + wid;
  const int64_t total16 = n * nz / 16, per16 = n / 16;
  const int64_t a = total16 * gw / W, bnd = total16 * (gw + 1) / W;
  for (int r = lane; r < 128 * 32 / 4; r += 32) reinterpret_cast<uint4 *>(c)[r] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  const uint4 *v4 = reinterpret_cast<const uint4 *>(vol);
  int64_t i = a;
  while (i < bnd) {
    const int64_t z = i / per16;
    const int64_t e = min(bnd, (z + 1) * per16);
    int64_t j = i + lane;
    for (; j + (UNROLL - 1) * 32 < e; j += UNROLL * 32) {
      uint4 w[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; u++) w[u] = __ldcs(v4 + j + u * 32);
#pragma unroll
      for (int u = 0; u < UNROLL; u++) {
        const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            const uint32_t x = (ws[q] >> (8 * jj)) & 0xff;
            atomicAdd(c + (x >> 1) * 32 + lane, 1u << ((x & 1) * 16));
          }
      }
    }
    for (; j < e; j += 32) {
      const uint4 w = __ldcs(v4 + j);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          const uint32_t x = (ws[q] >> (8 * jj)) & 0xff;
          atomicAdd(c + (x >> 1) * 32 + lane, 1u << ((x & 1) * 16));
        }
    }
    __syncwarp();
    // flush: lane l owns bin pairs r = l, l+32, l+64, l+96; rotated column reads
    for (int r = lane; r < 128; r += 32) {
      uint32_t lo = 0, hi = 0;
      for (int cc = 0; cc < 32; cc++) {
        const uint32_t x = c[r * 32 + ((cc + lane) & 31)];
        lo += x & 0xffff;
        hi += x >> 16;
      }
      if (lo) atomicAdd(hist + z * 256 + 2 * r, lo);
      if (hi) atomicAdd(hist + z * 256 + 2 * r + 1, hi);
    }
    __syncwarp();
    if (e < bnd) {
      for (int r = lane; r < 128 * 32 / 4; r += 32) reinterpret_cast<uint4 *>(c)[r] = make_uint4(0, 0, 0, 0);
      __syncwarp();
    }
    i = e;
  }
}


// V8: predicated red.shared (no branches) for non-zero bytes, zero bytes
// counted with SWAR in a register (bin 0 is ~31% of a CT slice and its
// same-address atomics serialise).
__device__ __forceinline__ void red_nz(uint32_t *bins, uint32_t x) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], 1;\n\t}"
               :: "r"((uint32_t)__cvta_generic_to_shared(bins + x)), "r"(x) : "memory");
}
template <int CH>
__global__ void __launch_bounds__(512) h_prednz(const uint4 *v, uint32_t *hist, int64_t nvec_slice) {
  __shared__ uint32_t sh[16][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t *b = sh[threadIdx.x >> 5];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + CH - 1) / CH;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  uint32_t zeros = 0;
  for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    const uint4 w = s[i];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      zeros += zero_bytes(ws[q]);
#pragma unroll
      for (int j = 0; j < 4; j++) red_nz(b, (ws[q] >> (8 * j)) & 0xff);
    }
  }
  atomicAdd(b, zeros);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}
// V9: plain red.shared for every byte (baseline for V8)
__device__ __forceinline__ void red_all(uint32_t *bins, uint32_t x) {
  asm volatile("red.shared.add.u32 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(bins + x)) : "memory");
}
template <int CH>
__global__ void __launch_bounds__(512) h_redall(const uint4 *v, uint32_t *hist, int64_t nvec_slice) {
  __shared__ uint32_t sh[16][256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t *b = sh[threadIdx.x >> 5];
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + CH - 1) / CH;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    const uint4 w = s[i];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int j = 0; j < 4; j++) red_all(b, (ws[q] >> (8 * j)) & 0xff);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t t = 0;
    for (int r = 0; r < 16; r++) t += sh[r][i];
    if (t) atomicAdd(hist + z * 256 + i, t);
  }
}

// label kernels
template <int UNROLL>
__global__ void __launch_bounds__(256) l_swar(const uint4 *v, uint4 *out, int64_t nvec, int64_t per_slice,
                                              const int *thr, int k) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nvec; i0 += stride * UNROLL) {
    uint4 w[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      const int64_t i = i0 + u * stride;
      if (i < nvec) w[u] = __ldcs(v + i);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      const int z = (int)(i / per_slice);
      uint4 o = make_uint4(0, 0, 0, 0);
      for (int j = 0; j < k; j++) {
        const uint32_t tb = (uint32_t)thr[z * k + j] * 0x01010101u;
        o.x += __vcmpgtu4(w[u].x, tb) & 0x01010101u;
        o.y += __vcmpgtu4(w[u].y, tb) & 0x01010101u;
        o.z += __vcmpgtu4(w[u].z, tb) & 0x01010101u;
        o.w += __vcmpgtu4(w[u].w, tb) & 0x01010101u;
      }
      __stcs(out + i, o);
    }
  }
}


// (p) pair histogram: one shared atomic per TWO pixels into 65536 packed u16
// counters H2[a][b] (128 KB), then h[a] += row sum a + column sum a.  A CTA
// counts <= 65535 pairs, so neither a counter nor a packed column/row sum wraps.
template <bool FAST>
__global__ void __launch_bounds__(512) h_pair(const uint4 *v, uint32_t *hist, int64_t nvec_slice, int chunks) {
  extern __shared__ uint32_t H2[];  // 32768 words
  __shared__ uint32_t hs[256];
  const int z = blockIdx.y;
  for (int i = threadIdx.x; i < 8192; i += 512) reinterpret_cast<uint4 *>(H2)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 256) hs[threadIdx.x] = 0;
  __syncthreads();
  const uint4 *s = v + z * nvec_slice;
  const int64_t per = (nvec_slice + chunks - 1) / chunks;
  const int64_t v0 = per * blockIdx.x, v1 = min(nvec_slice, v0 + per);
  auto pairs = [&](uint32_t x) {
    if (FAST && x == (x & 0xffu) * 0x01010101u) {
      const uint32_t k = (x & 0xffu) * 257u;
      atomicAdd(H2 + (k >> 1), 2u << ((k & 1u) << 4));
      return;
    }
    const uint32_t k0 = __byte_perm(x, 0, 0x4401), k1 = __byte_perm(x, 0, 0x4423);  // (b0<<8|b1), (b2<<8|b3)
    atomicAdd(H2 + (k0 >> 1), 1u << ((k0 & 1u) << 4));
    atomicAdd(H2 + (k1 >> 1), 1u << ((k1 & 1u) << 4));
  };
  int64_t i = v0 + threadIdx.x;
  for (; i + 3 * 512 < v1; i += 4 * 512) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; u++) w[u] = __ldcs(s + i + u * 512);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      pairs(w[u].x);
      pairs(w[u].y);
      pairs(w[u].z);
      pairs(w[u].w);
    }
  }
  for (; i < v1; i += 512) {
    const uint4 w = s[i];
    pairs(w.x);
    pairs(w.y);
    pairs(w.z);
    pairs(w.w);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // row sums: warp per row (first byte a)
  for (int a = warp; a < 256; a += 16) {
    uint32_t t = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) t += H2[a * 128 + lane + 32 * j];
    t = (t & 0xffffu) + (t >> 16);
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) hs[a] = t;
  }
  __syncthreads();
  // column sums: 4 threads per word column (second byte 2w, 2w+1), 64 rows each
  {
    const int w = threadIdx.x & 127, a0 = (threadIdx.x >> 7) * 64;
    uint32_t t = 0;
#pragma unroll 16
    for (int a = 0; a < 64; a++) t += H2[(a0 + a) * 128 + w];
    atomicAdd(&hs[2 * w], t & 0xffffu);
    atomicAdd(&hs[2 * w + 1], t >> 16);
  }
  __syncthreads();
  if (threadIdx.x < 256 && hs[threadIdx.x]) atomicAdd(hist + z * 256 + threadIdx.x, hs[threadIdx.x]);
}

__global__ void flush_l2(uint4 *buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4(i, 0, 0, 0);
}

int main(int argc, char **argv) {
  if (argc < 5) return 1;
  const int64_t nz = atoll(argv[2]), ny = atoll(argv[3]), nx = atoll(argv[4]);
  const int64_t n = nx * ny, total = n * nz;
  std::vector<uint8_t> h(total);
  FILE *f = fopen(argv[1], "rb");
  if (!f || fread(h.data(), 1, total, f) != (size_t)total) { printf("read fail\n"); return 1; }
  fclose(f);
  std::vector<uint32_t> ref(nz * 256, 0);
  for (int64_t z = 0; z < nz; z++) for (int64_t i = 0; i < n; i++) ref[z * 256 + h[z * n + i]]++;
  uint8_t *d; uint32_t *hist; uint4 *fl; uint8_t *lab; int *thr;
  CK(cudaMalloc(&d, total)); CK(cudaMalloc(&lab, total)); CK(cudaMalloc(&hist, nz * 256 * 4));
  const int64_t flN = 512ll << 20; CK(cudaMalloc(&fl, flN));
  CK(cudaMalloc(&thr, nz * 2 * 4));
  std::vector<int> th(nz * 2); for (int64_t z = 0; z < nz; z++) { th[z * 2] = 26; th[z * 2 + 1] = 138; }
  CK(cudaMemcpy(thr, th.data(), nz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d, h.data(), total, cudaMemcpyHostToDevice));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch, double bytes, bool check) {
    float best = 1e9, sum = 0; int reps = 10;
    for (int r = 0; r < reps + 2; r++) {
      flush_l2<<<sms * 4, 256>>>(fl, flN / 16);
      CK(cudaMemset(hist, 0, nz * 256 * 4));
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
    }
    bool ok = true;
    if (check) {
      std::vector<uint32_t> g(nz * 256);
      CK(cudaMemcpy(g.data(), hist, nz * 1024, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < g.size(); i++) if (g[i] != ref[i]) { ok = false; break; }
    }
    printf("{\"variant\": \"%s\", \"best_us\": %.2f, \"mean_us\": %.2f, \"gbs_best\": %.1f, \"ok\": %s}\n", name,
           best * 1e3, sum / reps * 1e3, bytes / (best * 1e-3) / 1e9, ok ? "true" : "false");
  };
  const int64_t nvs = n / 16;
  for (int chunks : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "atoms_fast_c%d", chunks);
    timeit(nm, [&] { h_atoms<true><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    snprintf(nm, 64, "atoms_nofast_c%d", chunks);
    timeit(nm, [&] { h_atoms<false><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
  }
  {
    const int T = 128; const size_t smem = 256 * T * 2;
    cudaFuncSetAttribute(h_private<T, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(h_private<T, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(h_private<T, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int per_sm : {2, 3}) {
      char nm[64];
      snprintf(nm, 64, "private_T128_u4_fast_g%d", per_sm);
      timeit(nm, [&] { h_private<T, 4, true><<<sms * per_sm, T, smem>>>(d, hist, n, nz); }, total, true);
      snprintf(nm, 64, "private_T128_u8_fast_g%d", per_sm);
      timeit(nm, [&] { h_private<T, 8, true><<<sms * per_sm, T, smem>>>(d, hist, n, nz); }, total, true);
      snprintf(nm, 64, "private_T128_u8_nofast_g%d", per_sm);
      timeit(nm, [&] { h_private<T, 8, false><<<sms * per_sm, T, smem>>>(d, hist, n, nz); }, total, true);
    }
  }
  {
    const int T = 256; const size_t smem = 256 * T * 2;
    cudaFuncSetAttribute(h_private<T, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timeit("private_T256_u8_fast_g1", [&] { h_private<T, 8, true><<<sms, T, smem>>>(d, hist, n, nz); }, total, true);
  }
  for (int per_sm : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "label_u1_g%d", per_sm);
    timeit(nm, [&] { l_swar<1><<<sms * per_sm, 256>>>((const uint4 *)d, (uint4 *)lab, total / 16, nvs, thr, 2); }, 2.0 * total, false);
    snprintf(nm, 64, "label_u4_g%d", per_sm);
    timeit(nm, [&] { l_swar<4><<<sms * per_sm, 256>>>((const uint4 *)d, (uint4 *)lab, total / 16, nvs, thr, 2); }, 2.0 * total, false);
  }

  for (int chunks : {4}) {
    timeit("atoms2_plain_1copy", [&] { h_atoms2<0, 1><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    timeit("atoms2_zeroskip_1copy", [&] { h_atoms2<1, 1><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    timeit("atoms2_zeroskip_warpskip_1copy", [&] { h_atoms2<2, 1><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    timeit("atoms2_plain_2copy", [&] { h_atoms2<0, 2><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    timeit("atoms2_zeroskip_warpskip_2copy", [&] { h_atoms2<2, 2><<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    timeit("match_any", [&] { h_match<<<dim3(chunks, nz), 512>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
  }
  {
    // hist (evict_last) followed by label: label time measured separately
    float tl = 0, th = 0; int reps = 10;
    cudaEvent_t e2; cudaEventCreate(&e2);
    for (int r = 0; r < reps + 2; r++) {
      flush_l2<<<sms * 4, 256>>>(fl, flN / 16);
      cudaMemset(hist, 0, nz * 1024);
      cudaEventRecord(e0);
      h_atoms_keep<<<dim3(4, nz), 512>>>((const uint4 *)d, hist, nvs, 4);
      cudaEventRecord(e1);
      l_swar<1><<<sms * 8, 256>>>((const uint4 *)d, (uint4 *)lab, total / 16, nvs, thr, 2);
      cudaEventRecord(e2);
      cudaEventSynchronize(e2);
      float a, b2; cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b2, e1, e2);
      if (r >= 2) { th += a; tl += b2; }
    }
    printf("{\"variant\": \"hist_keepL2_then_label\", \"hist_us\": %.2f, \"label_us\": %.2f, \"label_gbs_alg\": %.1f}\n",
           th / reps * 1e3, tl / reps * 1e3, 2.0 * total / (tl / reps * 1e-3) / 1e9);
  }

  {
    auto runl = [&](auto kern, int warps, int ctas_per_sm, const char *nm) {
      const size_t smem = (size_t)warps * 16384;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      timeit(nm, [&] { kern<<<sms * ctas_per_sm, warps * 32, smem>>>(d, hist, n, nz); }, total, true);
    };
    runl(h_lane<4, 4>, 4, 3, "lane_w4_u4_g3");
    runl(h_lane<4, 2>, 4, 3, "lane_w4_u2_g3");
    runl(h_lane<2, 4>, 2, 7, "lane_w2_u4_g7");
    runl(h_lane<2, 8>, 2, 6, "lane_w2_u8_g6");
    runl(h_lane<8, 2>, 8, 1, "lane_w8_u2_g1");
    runl(h_lane<4, 4>, 4, 6, "lane_w4_u4_g6x(2waves)");
  }

  {
    const size_t smem = 131072;
    cudaFuncSetAttribute(h_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(h_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int chunks : {3, 4, 6, 8}) {
      char nm[64];
      snprintf(nm, 64, "pair_fast_c%d", chunks);
      timeit(nm, [&] { h_pair<true><<<dim3(chunks, nz), 512, smem>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
      snprintf(nm, 64, "pair_nofast_c%d", chunks);
      timeit(nm, [&] { h_pair<false><<<dim3(chunks, nz), 512, smem>>>((const uint4 *)d, hist, nvs, chunks); }, total, true);
    }
  }
  timeit("prednz_c4", [&] { h_prednz<4><<<dim3(4, nz), 512>>>((const uint4 *)d, hist, nvs); }, total, true);
  timeit("prednz_c8", [&] { h_prednz<8><<<dim3(8, nz), 512>>>((const uint4 *)d, hist, nvs); }, total, true);
  timeit("redall_c4", [&] { h_redall<4><<<dim3(4, nz), 512>>>((const uint4 *)d, hist, nvs); }, total, true);
  // copy reference: a plain D2D copy of the same bytes
  timeit("memcpy_d2d", [&] { cudaMemcpyAsync(lab, d, total, cudaMemcpyDeviceToDevice); }, 2.0 * total, false);
  return 0;
}
