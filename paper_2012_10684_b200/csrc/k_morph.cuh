// k_morph.cuh -- SURVEY.md §8(f) NEXT row 3: grayscale morphology with a
// disk structuring element (readings DESIGN.md R26-R28):
//   erode(a)(y,x)  = min_{dy^2+dx^2 <= r^2} a(y+dy, x+dx), outside = 255
//   dilate(a)(y,x) = max over the same disk, outside = 0
//   open = dilate(erode(a)),  tophat = max(a - open, 0)
//
// Decomposition (exact): the disk is the union of the horizontal segments
// |dx| <= w(dy) = floor(sqrt(r^2 - dy^2)), so
//   erode(a)(y, x) = min_dy H_{w(dy)}(y + dy, x),   H_w(y, x) = min_{|dx| <= w} a(y, x+dx).
// One CTA streams a 256-pixel column strip of a slice top to bottom, four rows
// per step (a thread = 4 pixels of a row): each new row's H_w for w = 0..r is
// a cascade H_w = min(H_{w-1}, a(x-w), a(x+w)) in 16-bit lanes (two pixels per
// VIMNMX.U16x2; the 8-bit SIMD forms are emulated on sm_100a), the distinct
// widths the disk uses (7 for r = 10) are kept in a ring of 2r+4 rows in
// shared memory (88 KB: two CTAs per SM), and each output row (r rows behind)
// is the min over the 2r+1 ring rows of its disk.  The input is read
// once per pass (plus a 2r-pixel halo per strip row), the output written once.
#pragma once
#include <cmath>
#include <cstdint>

namespace tsa {

constexpr int kMorphStrip = 256;   // pixels per CTA column strip
constexpr int kMorphRows = 4;      // rows per step
constexpr int kMorphTpr = kMorphStrip / 4;  // threads per row (4 pixels each)
constexpr int kMorphThreads = kMorphRows * kMorphTpr;
constexpr int kMorphRmax = 10;

struct MorphArgs {
  const uint8_t *src;   // [nz][ny][nx]
  const uint8_t *orig;  // top-hat minuend (TOPHAT) or null
  uint8_t *dst;
  int64_t nx, ny, nz;
};

// distinct half-widths of disk(R): w(dy) = floor(sqrt(R^2 - dy^2)) (integer)
__host__ __device__ constexpr int isqrt_c(int v) {
  int s = 0;
  while ((s + 1) * (s + 1) <= v) s++;
  return s;
}
template <int R>
__host__ __device__ constexpr int halfw(int dy) {
  return isqrt_c(R * R - dy * dy);
}
// index of width w among the distinct widths (ascending dy from 0 gives
// descending widths); -1 if the disk has no row of that width
template <int R>
__host__ __device__ constexpr int widx(int w) {
  int k = 0, prev = -1;
  for (int dy = R; dy >= 0; dy--) {
    const int h = halfw<R>(dy);
    if (h != prev) {
      if (h == w) return k;
      k++;
      prev = h;
    }
  }
  return -1;
}
template <int R>
__host__ __device__ constexpr int nwidths() {
  int k = 0, prev = -1;
  for (int dy = R; dy >= 0; dy--) {
    const int h = halfw<R>(dy);
    if (h != prev) {
      k++;
      prev = h;
    }
  }
  return k;
}

template <bool MAX>
__device__ __forceinline__ uint32_t vop(uint32_t a, uint32_t b) {
  return MAX ? __vmaxu2(a, b) : __vminu2(a, b);
}

// pixel pair (u16 index k, k+1) of a thread's register window (word j holds
// u16 indices 2j, 2j+1): a word, or one PRMT across two words for odd k
template <int K>
__device__ __forceinline__ uint32_t pairk(const uint32_t *win) {
  if (K % 2 == 0) return win[K / 2];
  return __byte_perm(win[K / 2], win[K / 2 + 1], 0x5432);
}

template <int R, bool MAX, int P, int D>
__device__ __forceinline__ void cascade_step(const uint32_t *win, uint32_t &m) {
  // widen the window of the pair at pixel offset P by displacement D
  m = vop<MAX>(m, pairk<(R + R % 2) + P + D>(win));
}

template <int R, bool MAX, int W>
struct Cascade {
  // m0 / m1: the two pairs' running H_{W-1}; apply width W, store, recurse
  __device__ __forceinline__ static void run(const uint32_t *win, uint32_t &m0, uint32_t &m1,
                                             uint32_t *slot, int t) {
    cascade_step<R, MAX, 0, -W>(win, m0);
    cascade_step<R, MAX, 0, W>(win, m0);
    cascade_step<R, MAX, 2, -W>(win, m1);
    cascade_step<R, MAX, 2, W>(win, m1);
    if (widx<R>(W) >= 0)
      *reinterpret_cast<uint2 *>(slot + widx<R>(W) * (kMorphStrip / 2) + 2 * t) = make_uint2(m0, m1);
    Cascade<R, MAX, W + 1>::run(win, m0, m1, slot, t);
  }
};
template <int R, bool MAX>
struct Cascade<R, MAX, R + 1> {
  __device__ __forceinline__ static void run(const uint32_t *, uint32_t &, uint32_t &, uint32_t *, int) {}
};

template <int R, bool MAX, bool TOPHAT>
__global__ void __launch_bounds__(kMorphThreads) k_morph(MorphArgs g) {
  constexpr int NW = nwidths<R>();
  constexpr int PADL = R + R % 2;                  // even left pad (u16 pixels)
  constexpr int RS = 2 * R + kMorphRows;           // ring rows
  constexpr int PW = kMorphStrip / 2;              // pair words per strip row
  constexpr int BW = (kMorphStrip + 2 * PADL + 4) / 2;  // row buffer words (u16 pixels)
  constexpr int WINW = (2 * PADL + 4) / 2 + 1;     // register window words
  constexpr uint32_t NEUT = MAX ? 0u : 255u;
  constexpr uint32_t NEUT2 = NEUT * 0x00010001u;
  extern __shared__ __align__(16) uint32_t msm[];
  uint32_t *ring = msm;                            // [RS][NW][PW]
  uint32_t *rowbuf = msm + RS * NW * PW;           // [kMorphRows][BW]
  const int z = blockIdx.y;
  const int64_t x0 = (int64_t)blockIdx.x * kMorphStrip;
  const int64_t nx = g.nx, ny = g.ny;
  const uint8_t *src = g.src + (size_t)z * nx * ny;
  const int rr = threadIdx.x / kMorphTpr;          // which of the step's rows
  const int t = threadIdx.x % kMorphTpr;           // 4-pixel group in the strip
  const int64_t xp = x0 + 4 * t;
  const int steps = (int)((ny + R + kMorphRows - 1) / kMorphRows);
  for (int s = 0; s <= steps; s++) {
    // ---- S1: the step's input rows (strip + halo) into rowbuf as u16 pixels
    {
      const int64_t y = (int64_t)s * kMorphRows + rr;
      uint16_t *rb = reinterpret_cast<uint16_t *>(rowbuf + rr * BW);
      if (y < ny)
        for (int i = t; i < kMorphStrip + 2 * PADL + 4; i += kMorphTpr) {
          const int64_t x = x0 - PADL + i;
          rb[i] = (x >= 0 && x < nx) ? (uint16_t)__ldg(src + y * nx + x) : (uint16_t)NEUT;
        }
    }
    __syncthreads();
    // ---- S2: H_w cascade (w = 0..R) of the new rows into the ring
    {
      const int64_t y = (int64_t)s * kMorphRows + rr;
      if (y < ny) {
        uint32_t win[WINW];
        const uint32_t *rb = rowbuf + rr * BW + 2 * t;
#pragma unroll
        for (int j = 0; j < WINW; j++) win[j] = rb[j];
        uint32_t *slot = ring + ((int)y % RS) * NW * PW;
        uint32_t m0 = pairk<PADL>(win), m1 = pairk<PADL + 2>(win);
        if (widx<R>(0) >= 0)
          *reinterpret_cast<uint2 *>(slot + widx<R>(0) * PW + 2 * t) = make_uint2(m0, m1);
        Cascade<R, MAX, 1>::run(win, m0, m1, slot, t);
      }
    }
    __syncthreads();
    // ---- S3: output row y = (input row) - R: vertical min/max over the disk
    {
      const int64_t y = (int64_t)s * kMorphRows + rr - R;
      if (y >= 0 && y < ny && xp < nx) {
        uint32_t a0 = NEUT2, a1 = NEUT2;
#pragma unroll
        for (int dy = -R; dy <= R; dy++) {
          const int64_t yy = y + dy;
          if (yy < 0 || yy >= ny) continue;  // outside the slice: neutral
          const int wi = widx<R>(halfw<R>(dy < 0 ? -dy : dy));
          const uint2 v = *reinterpret_cast<const uint2 *>(ring + (((int)yy % RS) * NW + wi) * PW + 2 * t);
          a0 = vop<MAX>(a0, v.x);
          a1 = vop<MAX>(a1, v.y);
        }
        const int64_t o = ((size_t)z * ny + y) * nx + xp;
        const bool full = xp + 3 < nx &&
                          ((reinterpret_cast<uintptr_t>(g.dst + o) |
                            (TOPHAT ? reinterpret_cast<uintptr_t>(g.orig + o) : 0u)) & 3u) == 0;
        if (TOPHAT) {
          // max(orig - open, 0) per 16-bit lane = max(orig, open) - open
          uint32_t ow = 0u;
          if (full) {
            ow = *reinterpret_cast<const uint32_t *>(g.orig + o);
          } else {
            for (int e = 0; e < 4; e++)
              if (xp + e < nx) ow |= (uint32_t)g.orig[o + e] << (8 * e);
          }
          const uint32_t o0 = __byte_perm(ow, 0u, 0x4140), o1 = __byte_perm(ow, 0u, 0x4342);
          a0 = __vmaxu2(o0, a0) - a0;
          a1 = __vmaxu2(o1, a1) - a1;
        }
        const uint32_t packed = __byte_perm(a0, a1, 0x6420);  // bytes 0,2 of a0 then of a1
        if (full) {
          *reinterpret_cast<uint32_t *>(g.dst + o) = packed;
        } else {
          for (int e = 0; e < 4; e++)
            if (xp + e < nx) g.dst[o + e] = (uint8_t)((packed >> (8 * e)) & 0xffu);
        }
      }
    }
  }
}

template <int R>
__host__ inline size_t morph_smem() {
  constexpr int NW = nwidths<R>();
  constexpr int PADL = R + R % 2;
  return (size_t)(2 * R + kMorphRows) * NW * (kMorphStrip / 2) * 4 +
         (size_t)kMorphRows * ((kMorphStrip + 2 * PADL + 4) / 2) * 4;
}

}  // namespace tsa
