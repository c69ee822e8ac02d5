// k_label.cuh -- SURVEY.md §8 row a5: relabel every voxel by class,
// label(v) = #{j : v > t*_j}.  For k = 1 this is Algorithm 1 (PAPER.md:464-477,
// "image(x,y) >= T -> 1") with T = t* + 1, t* being the last level of the
// lower class (R4); for k > 1 the same rule per threshold.
//
// HBM-bound streaming kernel: flat grid-stride over the slab in 16-byte
// vectors (u8: 16 voxels -> 16 labels, SWAR compare with __vcmpgtu4; u16: 8
// voxels -> 8 labels), streaming (evict-first) loads and stores, grid sized as
// a multiple of the SM count.  Slices whose status is not OK get label 0.
#pragma once
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

struct LabelArgs {
  const uint8_t *vol;
  uint8_t *labels;
  const int32_t *thr;     // [nz][k]
  const int32_t *status;  // [nz] or null
  int64_t n;              // voxels per slice
  int64_t z0, z1;         // slab [z0, z1)
  int k;
};

__device__ __forceinline__ uint32_t swar_label4(uint32_t w, const uint32_t *tb, int k) {
  uint32_t o = 0;
  for (int j = 0; j < k; j++) o += __vcmpgtu4(w, tb[j]) & 0x01010101u;
  return o;
}

// Fast path: n % 16 == 0 and 16-byte aligned volume/labels (the common case).
template <typename T>
__global__ void __launch_bounds__(256) k_label_flat(LabelArgs g) {
  const int64_t per = g.n / 16;  // 16-voxel groups per slice
  const int64_t i0 = g.z0 * per, i1 = g.z1 * per;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4 *src = reinterpret_cast<const uint4 *>(g.vol);
  uint4 *dst = reinterpret_cast<uint4 *>(g.labels);
  int zc = -1;
  bool ok = false;
  uint32_t tb[kKMax];
  int t[kKMax];
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i1; i += stride) {
    const int z = (int)(i / per);
    if (z != zc) {
      zc = z;
      ok = g.status == nullptr || g.status[z] == kOK;
#pragma unroll
      for (int j = 0; j < kKMax; j++) {
        t[j] = j < g.k ? g.thr[z * g.k + j] : 0;
        tb[j] = (uint32_t)(t[j] & 0xff) * 0x01010101u;
      }
    }
    if (sizeof(T) == 1) {
      const uint4 w = __ldcs(src + i);
      uint4 o = make_uint4(0u, 0u, 0u, 0u);
      if (ok) {
        o.x = swar_label4(w.x, tb, g.k);
        o.y = swar_label4(w.y, tb, g.k);
        o.z = swar_label4(w.z, tb, g.k);
        o.w = swar_label4(w.w, tb, g.k);
      }
      __stcs(dst + i, o);
    } else {
      const uint4 wa = __ldcs(src + 2 * i), wb = __ldcs(src + 2 * i + 1);
      const uint32_t ws[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      uint32_t o[4] = {0u, 0u, 0u, 0u};
      if (ok) {
#pragma unroll
        for (int e = 0; e < 16; e++) {
          const int v = (int)((ws[e >> 1] >> (16 * (e & 1))) & 0xffffu);
          uint32_t l = 0;
          for (int j = 0; j < g.k; j++) l += v > t[j];
          o[e >> 2] |= l << (8 * (e & 3));
        }
      }
      __stcs(dst + i, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

// General path (any n, any alignment): one CTA row per slice, scalar.
template <typename T>
__global__ void __launch_bounds__(256) k_label_generic(LabelArgs g) {
  const int64_t z = g.z0 + blockIdx.y;
  const T *slice = reinterpret_cast<const T *>(g.vol) + (size_t)z * g.n;
  uint8_t *out = g.labels + (size_t)z * g.n;
  const bool ok = g.status == nullptr || g.status[z] == kOK;
  int t[kKMax] = {0, 0, 0, 0};
  for (int j = 0; j < g.k; j++) t[j] = g.thr[z * g.k + j];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)slice[i];
    uint32_t l = 0;
    if (ok)
      for (int j = 0; j < g.k; j++) l += v > t[j];
    out[i] = (uint8_t)l;
  }
}

}  // namespace tsa
