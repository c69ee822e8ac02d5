// k_hu.cuh -- SURVEY.md §8(f) NEXT row 2: pre-processing (PAPER.md:514-516,
// "change the value of -2000 ... to 0. Then all intensity levels are linearly
// transformed to the range 0 to 255") fused into the histogram and label
// passes of the 1-D path, on raw int16 HU input (readings DESIGN.md R23-R25):
//   lo, hi   = volume-wide min / max of the non-background voxels
//   g(v)     = 0 for the background; else round-half-away(255 (v - lo) / (hi - lo))
//            = floor((510 (v - lo) + (hi - lo)) / (2 (hi - lo)));  hi == lo -> 0
//
// The volume is read twice (histogram pass, label pass) instead of three times
// plus a write of the 8-bit image:
//   k_hu_hist   per-slice HU histograms over 8192 bins (HU in [-4096, 4095],
//               else LEVEL_OVERFLOW)
//   k_hu_window the volume-wide window from the histograms' non-empty bins
//   k_hu_glut   g over the 8192 HU bins (one exact division each)
//   k_hu_remap  per slice, the 8-bit histogram c_b = sum_{v : g(v) = b} h_v
//               (exact: g is a function of v) -> the usual search / finalize
//   k_label_hu  labels straight from HU: g is non-decreasing, so
//               g(v) > t  <=>  v >= lo + ceil((2t + 1)(hi - lo) / 510)
//               (background voxels excluded), compared two voxels per
//               instruction with signed 16-bit SIMD compares
//   k_hu_map    the standalone 8-bit image (tsa_hu_preprocess), per-CTA LUT
#pragma once
#include <climits>
#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

constexpr int kHuBins = 8192;  // HU histogram bins: v + 4096
constexpr int kHuOff = 4096;

struct HuArgs {
  const int16_t *vol;  // [nz][n]
  int64_t n, nz;
  int bg;              // background HU
  uint32_t *hu_hist;   // [nz][8192] (zeroed) or null (window only)
  int32_t *win;        // [0] lo, [1] hi, [2] / [3] min / max of the out-of-range voxels
  int32_t *status;     // [nz] (zeroed)
  int chunks;
};

// window slots start at (INT_MAX, INT_MIN) for (lo, hi) and for the
// out-of-range voxels' (min, max)
__global__ void k_hu_init(int32_t *win) {
  win[0] = INT_MAX;
  win[1] = INT_MIN;
  win[2] = INT_MAX;
  win[3] = INT_MIN;
}

// g(v) for a non-background voxel (exact integer arithmetic)
__device__ __forceinline__ uint32_t hu_gray(int v, int lo, int hi) {
  if (hi <= lo) return 0u;
  const int64_t num = 510 * (int64_t)(v - lo) + (hi - lo);
  return (uint32_t)(num / (2 * (int64_t)(hi - lo)));
}

// HU histogram of a (slice, chunk).  Four copies of the 8192 bins as 16-bit
// counters packed two per word (4 x 16 KB, so several CTAs share an SM; warps
// w, w+4, ... share copy w % 4; a counter sees < 65536 voxels: the host keeps
// chunks at <= 128 K voxels).  The background (a fifth of a CT slice, all in
// one bin: 32-way same-address atomics) is counted in a register and added to
// global memory once per warp.  The window comes from the histograms
// (k_hu_window); only voxels outside the bins (LEVEL_OVERFLOW, rare) update it
// here directly.
__global__ void __launch_bounds__(512) k_hu_hist(HuArgs g) {
  extern __shared__ uint32_t hsh[];
  const int z = blockIdx.y, c = blockIdx.x;
  constexpr int REP = 4, HW = kHuBins / 2;
  for (int i = threadIdx.x; i < HW * REP / 4; i += blockDim.x)
    reinterpret_cast<uint4 *>(hsh)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  // 32-bit shared address of this warp's copy (computed once: the compiler
  // otherwise re-derives the generic->shared window per atomic)
  const uint32_t sbase =
      (uint32_t)__cvta_generic_to_shared(hsh + ((threadIdx.x >> 5) % REP) * HW);
  const int16_t *slice = g.vol + (size_t)z * g.n;
  const int64_t nvec = g.n / 8;  // 16-byte vectors (n % 16 == 0, aligned: checked by the host)
  const int64_t per = (nvec + g.chunks - 1) / g.chunks;
  const int64_t v0 = per * c, v1 = min(nvec, v0 + per);
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice);
  const int bg = g.bg;
  uint32_t nbg = 0;
  int ovf = 0, omn = INT_MAX, omx = INT_MIN;  // out-of-range voxels (window only)
  // every voxel issues one shared reduction; the background (always inside
  // the bins, checked by the host) and out-of-range voxels add 0 to a
  // lane-private word of bins 0..63 (HU -4096..-4033: adding 0 changes
  // nothing and the 32 lanes hit 32 banks), so no predicate splits the warp.
  // Two voxels per 32-bit word: b = v + 4096 for both lanes in one
  // VIADD.16x2; the range and background tests are masks (the 16-bit SIMD
  // compares are emulated on sm_100a).
  const uint32_t lane_addr = sbase + 4u * (threadIdx.x & 31);
  const uint32_t bg2 = ((uint32_t)(uint16_t)bg) * 0x00010001u;
  auto red = [&](uint32_t addr, uint32_t inc) {
    asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(addr), "r"(inc) : "memory");
  };
  auto word = [&](uint32_t w) {
    const uint32_t b2 = __vadd2(w, 0x10001000u);  // both lanes + 4096 (mod 2^16)
    if (__builtin_expect((b2 & 0xE000E000u) != 0u, 0)) {  // a lane outside [-4096, 4095] (rare)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int v = (int)(int16_t)((w >> (16 * h)) & 0xffffu);
        const uint32_t b = (b2 >> (16 * h)) & 0xffffu;
        if (b >= (uint32_t)kHuBins) {
          ovf = 1;
          if (v != bg) {
            omn = min(omn, v);
            omx = max(omx, v);
          }
          red(lane_addr, 0u);
        } else if (v == bg) {
          nbg++;
          red(lane_addr, 0u);
        } else {
          red(sbase + ((b << 1) & 0x3ffcu), (b & 1u) ? 0x10000u : 1u);
        }
      }
      return;
    }
    const uint32_t x = w ^ bg2;
    const bool bg0 = (x & 0xffffu) == 0u, bg1 = (x >> 16) == 0u;
    nbg += (bg0 ? 1u : 0u) + (bg1 ? 1u : 0u);
    const uint32_t a0 = bg0 ? lane_addr : sbase + ((b2 << 1) & 0x3ffcu);
    const uint32_t i0 = bg0 ? 0u : ((b2 & 1u) ? 0x10000u : 1u);
    const uint32_t a1 = bg1 ? lane_addr : sbase + ((b2 >> 15) & 0x3ffcu);
    const uint32_t i1 = bg1 ? 0u : ((b2 & 0x10000u) ? 0x10000u : 1u);
    red(a0, i0);
    red(a1, i1);
  };
  constexpr int U = 4;  // 16-byte loads in flight per thread
  for (int64_t i0 = v0 + threadIdx.x; i0 < v1; i0 += (int64_t)U * blockDim.x) {
    uint4 wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      if (i < v1) wv[u] = __ldcs(v4 + i);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (i0 + (int64_t)u * blockDim.x >= v1) break;
      word(wv[u].x);
      word(wv[u].y);
      word(wv[u].z);
      word(wv[u].w);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    nbg += __shfl_xor_sync(0xffffffffu, nbg, off);
    omn = min(omn, __shfl_xor_sync(0xffffffffu, omn, off));
    omx = max(omx, __shfl_xor_sync(0xffffffffu, omx, off));
  }
  ovf = __any_sync(0xffffffffu, ovf);
  uint32_t *out = g.hu_hist + (size_t)z * kHuBins;
  if ((threadIdx.x & 31) == 0) {
    if (nbg) atomicAdd(out + (uint32_t)(bg + kHuOff), nbg);
    if (ovf) {
      if (omn != INT_MAX) atomicMin(g.win + 2, omn);
      if (omx != INT_MIN) atomicMax(g.win + 3, omx);
      g.status[z] = kLevelOverflow;
    }
  }
  __syncthreads();
  // flush: 4 words (8 bins) of every copy per 16-byte load
  for (int q = threadIdx.x; q < HW / 4; q += blockDim.x) {
    uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int r = 0; r < REP; r++) {
      const uint4 w = reinterpret_cast<const uint4 *>(hsh + r * HW)[q];
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; e++) {
        lo[e] += ws[e] & 0xffffu;
        hi[e] += ws[e] >> 16;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int b = 8 * q + 2 * e;
      if (lo[e]) atomicAdd(out + b, lo[e]);
      if (hi[e]) atomicAdd(out + b + 1, hi[e]);
    }
  }
}

// The volume-wide window from the HU histograms: (lo, hi) = the lowest / highest
// non-empty bin other than the background over every slice, merged with the
// out-of-range voxels' min / max (win[2], win[3]).  Grid over the bins, each
// thread ORs its bin over the slices.
__global__ void __launch_bounds__(256) k_hu_window(const uint32_t *hu_hist, int64_t nz, int bg, int32_t *win) {
  // grid (bins / 256, slice chunks): each thread ORs its bin over its slices
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t zc = (nz + gridDim.y - 1) / gridDim.y;
  const int64_t z0 = zc * blockIdx.y, z1 = min(nz, z0 + zc);
  uint32_t any = 0;
  if (b < kHuBins && b - kHuOff != bg)
    for (int64_t z = z0; z < z1; z++) any |= __ldcs(hu_hist + (size_t)z * kHuBins + b);
  int mn = any ? b - kHuOff : INT_MAX, mx = any ? b - kHuOff : INT_MIN;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (mn != INT_MAX) atomicMin(win, mn);
    if (mx != INT_MIN) atomicMax(win + 1, mx);
  }
}

// fold the out-of-range extremes into (lo, hi) (one thread, after k_hu_window)
__global__ void k_hu_window_fold(int32_t *win) {
  if (win[2] != INT_MAX) win[0] = min(win[0], win[2]);
  if (win[3] != INT_MIN) win[1] = max(win[1], win[3]);
}

// g over the HU bins (one exact division per bin, once per call)
__global__ void k_hu_glut(const int32_t *win, int bg, uint8_t *glut) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= kHuBins) return;
  const int lo = win[0], hi = win[1], v = b - kHuOff;
  glut[b] = (uint8_t)((v == bg || lo == INT_MAX) ? 0u : min(hu_gray(v, lo, hi), 255u));
}

// 8-bit histogram of a slice from its HU histogram: grid (4, nz), each CTA a
// quarter of the HU bins into shared bins, then added into hist (zeroed).
__global__ void __launch_bounds__(256) k_hu_remap(const uint32_t *hu_hist, const uint8_t *glut,
                                                  uint32_t *hist) {
  __shared__ uint32_t b8[256];
  const int z = blockIdx.y, q = blockIdx.x;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) b8[i] = 0u;
  __syncthreads();
  const uint4 *h4 = reinterpret_cast<const uint4 *>(hu_hist + (size_t)z * kHuBins) + q * (kHuBins / 16);
  const uint32_t *g4 = reinterpret_cast<const uint32_t *>(glut) + q * (kHuBins / 16);
  for (int i = threadIdx.x; i < kHuBins / 16; i += blockDim.x) {
    const uint4 c = __ldcs(h4 + i);
    if ((c.x | c.y | c.z | c.w) == 0u) continue;
    const uint32_t gg = g4[i];
    if (c.x) atomicAdd(b8 + (gg & 0xffu), c.x);
    if (c.y) atomicAdd(b8 + ((gg >> 8) & 0xffu), c.y);
    if (c.z) atomicAdd(b8 + ((gg >> 16) & 0xffu), c.z);
    if (c.w) atomicAdd(b8 + (gg >> 24), c.w);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (b8[i]) atomicAdd(hist + (size_t)z * 256 + i, b8[i]);
}

// Smallest HU v with g(v) > t (t an 8-bit threshold); INT_MAX if none.
__device__ __forceinline__ int hu_cut(int t, int lo, int hi) {
  if (t < 0) return INT_MIN;
  if (t >= 255 || hi <= lo) return INT_MAX;
  const int64_t d = (int64_t)(2 * t + 1) * (hi - lo);
  return lo + (int)((d + 509) / 510);  // ceil((2t+1)(hi-lo)/510)
}

// labels[z][i] = #{ j : g(v) > t_j } for non-background voxels, 0 for the
// background and for failed slices.  Grid (chunks, nz): a CTA labels a
// contiguous part of one slice (its cutoffs computed once), 16 voxels (two
// 16-byte loads, one 16-byte store) per item, two items in flight per thread.
template <int KT>
__global__ void __launch_bounds__(256) k_label_hu(const int16_t *vol, uint8_t *labels, const int32_t *thr,
                                                  const int32_t *status, const int32_t *win, int bg,
                                                  int64_t n, int k) {
  const int z = blockIdx.y;
  const int64_t per = n / 16;
  const int64_t cp = (per + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)z * per + cp * blockIdx.x;
  const int64_t i1 = (int64_t)z * per + min(per, cp * (blockIdx.x + 1));
  const uint4 *src = reinterpret_cast<const uint4 *>(vol);
  uint4 *dst = reinterpret_cast<uint4 *>(labels);
  const int lo = win[0], hi = win[1];
  const uint32_t bg2 = ((uint32_t)(uint16_t)bg) * 0x00010001u;
  const bool ok = status == nullptr || status[z] == kOK;
  const int32_t *tz = thr + (size_t)z * k;
  // cutoffs clamped to the int16 range (every int16 >= -32768); "never" when
  // the cutoff is above every int16
  bool nv[4] = {true, true, true, true};
  uint32_t cc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < KT; j++) {
    const int c = hu_cut(tz[j], lo, hi);
    nv[j] = c > 32767;
    const int c16 = c > 32767 ? 32767 : (c < -32768 ? -32768 : c);
    cc[j] = ((uint32_t)(uint16_t)c16) * 0x00010001u;
  }
  for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += 2 * (int64_t)blockDim.x) {
    uint4 wa[2], wb[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int64_t it = ib + (int64_t)u * blockDim.x;
      if (it < i1) {
        wa[u] = __ldcs(src + 2 * it);
        wb[u] = __ldcs(src + 2 * it + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int64_t it = ib + (int64_t)u * blockDim.x;
      if (it >= i1) break;
      const uint32_t ws[8] = {wa[u].x, wa[u].y, wa[u].z, wa[u].w, wb[u].x, wb[u].y, wb[u].z, wb[u].w};
      uint32_t o[4] = {0u, 0u, 0u, 0u};
      if (ok) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
          // per 16-bit lane: 1 where v >= cut (signed), masked by v != bg
          const uint32_t w = ws[e];
          uint32_t l = 0u;
#pragma unroll
          for (int j = 0; j < KT; j++)
            if (!nv[j]) l += __vcmpges2(w, cc[j]) & 0x00010001u;
          l &= __vcmpne2(w, bg2);
          // two 16-bit lanes -> two bytes of the output word
          o[e >> 1] |= __byte_perm(l, 0u, 0x4420) << (16 * (e & 1));
        }
      }
      __stcs(dst + it, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

// Standalone 8-bit image (tsa_hu_preprocess): a per-CTA LUT over the HU bins.
__global__ void __launch_bounds__(256) k_hu_map(const int16_t *vol, uint8_t *gray, const int32_t *win,
                                                int bg, int64_t total) {
  __shared__ uint8_t lut[kHuBins];
  const int lo = win[0], hi = win[1];
  for (int b = threadIdx.x; b < kHuBins; b += blockDim.x) {
    const int v = b - kHuOff;
    lut[b] = (uint8_t)((v == bg || lo == INT_MAX) ? 0u : min(hu_gray(v, lo, hi), 255u));
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = vol[i];
    const uint32_t b = (uint32_t)(v + kHuOff);
    gray[i] = b < (uint32_t)kHuBins ? lut[b] : (uint8_t)0;
  }
}

}  // namespace tsa
