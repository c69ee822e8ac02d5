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

// Thresholds beyond k are set to 255 (u8) / 65535 (u16): "v > t" is then never
// true, so the unrolled 4-way compare needs no k-dependent control flow.
__device__ __forceinline__ uint32_t swar_label4(uint32_t w, uint32_t t0, uint32_t t1, uint32_t t2,
                                                uint32_t t3) {
  return (__vcmpgtu4(w, t0) & 0x01010101u) + (__vcmpgtu4(w, t1) & 0x01010101u) +
         (__vcmpgtu4(w, t2) & 0x01010101u) + (__vcmpgtu4(w, t3) & 0x01010101u);
}

template <int KT>
__device__ __forceinline__ uint32_t swar_labelk(uint32_t w, uint32_t t0, uint32_t t1, uint32_t t2,
                                                uint32_t t3) {
  uint32_t o = __vcmpgtu4(w, t0) & 0x01010101u;
  if (KT > 1) o += __vcmpgtu4(w, t1) & 0x01010101u;
  if (KT > 2) o += __vcmpgtu4(w, t2) & 0x01010101u;
  if (KT > 3) o += __vcmpgtu4(w, t3) & 0x01010101u;
  return o;
}

template <int KT>
__device__ __forceinline__ uint32_t label_ofk(int v, int t0, int t1, int t2, int t3) {
  uint32_t l = (uint32_t)(v > t0);
  if (KT > 1) l += (uint32_t)(v > t1);
  if (KT > 2) l += (uint32_t)(v > t2);
  if (KT > 3) l += (uint32_t)(v > t3);
  return l;
}

__device__ __forceinline__ uint32_t label_of(int v, int t0, int t1, int t2, int t3) {
  return (uint32_t)(v > t0) + (uint32_t)(v > t1) + (uint32_t)(v > t2) + (uint32_t)(v > t3);
}

// Fast path: n % 16 == 0 and 16-byte aligned volume/labels (the common case).
// KT = k (compile-time: only k SWAR compares per word; thresholds >= k unused).
template <typename T, int KT>
__global__ void __launch_bounds__(256) k_label_flat(LabelArgs g) {
  // a PDL-launched dependent (k_finalize_phi in the staged step) may start
  // now: it reads nothing this kernel writes (no effect without one)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t per = g.n / 16;  // 16-voxel groups per slice
  const int64_t i0 = g.z0 * per, i1 = g.z1 * per;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4 *src = reinterpret_cast<const uint4 *>(g.vol);
  uint4 *dst = reinterpret_cast<uint4 *>(g.labels);
  const int64_t i_first = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int z = (int)(i_first / per);
  int64_t zend = (int64_t)(z + 1) * per;  // first group of the next slice
  const int tmax = sizeof(T) == 1 ? 255 : 65535;
  int t0 = tmax, t1 = tmax, t2 = tmax, t3 = tmax;
  bool ok = false;
  bool fresh = true;
  for (int64_t i = i_first; i < i1; i += stride) {
    if (i >= zend || fresh) {  // slice change: at most once or twice per thread
      if (!fresh) {
        z = (int)(i / per);
        zend = (int64_t)(z + 1) * per;
      }
      fresh = false;
      ok = g.status == nullptr || g.status[z] == kOK;
      const int32_t *tz = g.thr + z * g.k;
      t0 = tz[0];
      t1 = g.k > 1 ? tz[1] : tmax;
      t2 = g.k > 2 ? tz[2] : tmax;
      t3 = g.k > 3 ? tz[3] : tmax;
    }
    if (sizeof(T) == 1) {
      const uint4 w = __ldcs(src + i);
      uint4 o = make_uint4(0u, 0u, 0u, 0u);
      if (ok) {
        const uint32_t b0 = (uint32_t)t0 * 0x01010101u, b1 = (uint32_t)t1 * 0x01010101u;
        const uint32_t b2 = (uint32_t)t2 * 0x01010101u, b3 = (uint32_t)t3 * 0x01010101u;
        o.x = swar_labelk<KT>(w.x, b0, b1, b2, b3);
        o.y = swar_labelk<KT>(w.y, b0, b1, b2, b3);
        o.z = swar_labelk<KT>(w.z, b0, b1, b2, b3);
        o.w = swar_labelk<KT>(w.w, b0, b1, b2, b3);
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
          o[e >> 2] |= label_ofk<KT>(v, t0, t1, t2, t3) << (8 * (e & 3));
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
  const int tmax = 65535;
  const int32_t *tz = g.thr + z * g.k;
  const int t0 = tz[0], t1 = g.k > 1 ? tz[1] : tmax, t2 = g.k > 2 ? tz[2] : tmax;
  const int t3 = g.k > 3 ? tz[3] : tmax;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = ok ? (uint8_t)label_of((int)slice[i], t0, t1, t2, t3) : (uint8_t)0;
  }
}

// q sweep (tsa_segment_sweep): the labels of every q from ONE read of the
// volume (round 2; the sweep labelled the same volume 11 times).  A failed
// slice of a q has thresholds -1 and gets labels 0 for that q.  Grid (chunk,
// slice); the packed thresholds of the slice for every q are staged in shared
// memory.  n % 16 == 0, 16-byte aligned volume and labels.
constexpr int kSweepMaxQ = 16;  // q values per launch
struct LabelSweepArgs {
  const uint8_t *vol;
  int64_t n;  // voxels per slice
  int k, nq;
  const int32_t *thr[kSweepMaxQ];  // [nz][k] per q
  uint8_t *lab[kSweepMaxQ];        // [nz][n] per q
};

template <typename T, int KT>
__global__ void __launch_bounds__(256) k_label_sweep(LabelSweepArgs g) {
  __shared__ uint32_t s_b[kSweepMaxQ][4];  // u8: thresholds replicated in 4 bytes; u16: the value
  __shared__ int s_ok[kSweepMaxQ];
  const int64_t z = blockIdx.y;
  if (threadIdx.x < g.nq) {
    const int32_t *tz = g.thr[threadIdx.x] + z * g.k;
    const int t0 = tz[0];
    s_ok[threadIdx.x] = t0 >= 0;
    const int tmax = sizeof(T) == 1 ? 255 : 65535;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int t = j < KT ? tz[j] : tmax;
      s_b[threadIdx.x][j] = sizeof(T) == 1 ? (uint32_t)(t & 0xff) * 0x01010101u : (uint32_t)t;
    }
  }
  __syncthreads();
  const int64_t groups = g.n / 16;
  const int64_t per = (groups + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = z * groups + per * blockIdx.x, i1 = z * groups + min(groups, per * (blockIdx.x + 1));
  const uint4 *src = reinterpret_cast<const uint4 *>(g.vol);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    if (sizeof(T) == 1) {
      const uint4 w = __ldcs(src + i);
      for (int qi = 0; qi < g.nq; qi++) {
        uint4 o = make_uint4(0u, 0u, 0u, 0u);
        if (s_ok[qi]) {
          const uint32_t b0 = s_b[qi][0], b1 = s_b[qi][1], b2 = s_b[qi][2], b3 = s_b[qi][3];
          o.x = swar_labelk<KT>(w.x, b0, b1, b2, b3);
          o.y = swar_labelk<KT>(w.y, b0, b1, b2, b3);
          o.z = swar_labelk<KT>(w.z, b0, b1, b2, b3);
          o.w = swar_labelk<KT>(w.w, b0, b1, b2, b3);
        }
        __stcs(reinterpret_cast<uint4 *>(g.lab[qi]) + i, o);
      }
    } else {
      const uint4 wa = __ldcs(src + 2 * i), wb = __ldcs(src + 2 * i + 1);
      const uint32_t ws[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      for (int qi = 0; qi < g.nq; qi++) {
        uint32_t o[4] = {0u, 0u, 0u, 0u};
        if (s_ok[qi]) {
          const int t0 = (int)s_b[qi][0], t1 = (int)s_b[qi][1], t2 = (int)s_b[qi][2], t3 = (int)s_b[qi][3];
#pragma unroll
          for (int e = 0; e < 16; e++) {
            const int v = (int)((ws[e >> 1] >> (16 * (e & 1))) & 0xffffu);
            o[e >> 2] |= label_ofk<KT>(v, t0, t1, t2, t3) << (8 * (e & 3));
          }
        }
        __stcs(reinterpret_cast<uint4 *>(g.lab[qi]) + i, make_uint4(o[0], o[1], o[2], o[3]));
      }
    }
  }
}

}  // namespace tsa
