// k_morph.cuh -- SURVEY.md §8(f) NEXT row 3: grayscale morphology with a
// disk structuring element (readings DESIGN.md R26-R28):
//   erode(a)(y,x)  = min_{dy^2+dx^2 <= r^2} a(y+dy, x+dx), outside = 255
//   dilate(a)(y,x) = max over the same disk, outside = 0
//   open = dilate(erode(a)),  tophat = max(a - open, 0)
//
// Decomposition (exact): the disk is the union of the horizontal segments
// |dx| <= w(dy) = floor(sqrt(r^2 - dy^2)), so
//   erode(a)(y, x) = min_dy H_{w(dy)}(y + dy, x),   H_w(y, x) = min_{|dx| <= w} a(y, x+dx).
// A CTA streams a 256-pixel column strip of 128 output rows of a slice top to
// bottom (plus r halo rows each side); a thread owns 4 pixel columns.  For
// each input row the thread computes its H_w, w = 0..r, as a cascade H_w =
// min(H_{w-1}, a(x-w), a(x+w)) in 16-bit lanes (two pixels per VIMNMX.U16x2;
// the 8-bit SIMD forms are emulated on sm_100a) from a shared-memory copy of
// the row, and folds them into REGISTER accumulators of the 2r+1 output rows
// the input row touches (slot j = output row y-r+j); the completed output
// row (r rows behind) is written and the slots shift by one.  No vertical gather, no shared-memory ring.  The input is read
// once per pass (plus a 2r-pixel halo per strip row), the output written once.
#pragma once
#include <cmath>
#include <cstdint>
#include <type_traits>

namespace tsa {

constexpr int kMorphStrip = 256;                // pixels per CTA column strip
constexpr int kMorphThreads = kMorphStrip / 4;  // a thread = 4 pixel columns
constexpr int kMorphChunk = 128;                // output rows per CTA
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

// Register accumulators of the 2R+1 pending output rows of a thread's 4
// columns (two 16-bit-lane words each); slot j holds output row y-R+j while
// input row y is processed.
constexpr int kMorphGroup = 2;  // input rows per accumulator shift (4: 124 registers, slower)

template <int R>
struct Acc {
  uint32_t a[2 * R + kMorphGroup][2];
};

// The H_w cascade of one input row for the thread's two pixel pairs: hw[w]
// for w = 0..R (only the widths the disk uses are read by the caller).
template <int R, bool MAX, int W>
__device__ __forceinline__ void cascade(const uint32_t *win, uint32_t (&h0)[R + 1], uint32_t (&h1)[R + 1]) {
  if constexpr (W == 0) {
    h0[0] = pairk<R + R % 2>(win);
    h1[0] = pairk<R + R % 2 + 2>(win);
  } else {
    h0[W] = vop<MAX>(vop<MAX>(h0[W - 1], pairk<R + R % 2 - W>(win)), pairk<R + R % 2 + W>(win));
    h1[W] = vop<MAX>(vop<MAX>(h1[W - 1], pairk<R + R % 2 + 2 - W>(win)), pairk<R + R % 2 + 2 + W>(win));
  }
  if constexpr (W < R) cascade<R, MAX, W + 1>(win, h0, h1);
}

// Rows come in groups of kMorphGroup; input row y+OFF contributes H_{w(R-j)} to the
// pending output row y+OFF-R+j held in slot j+OFF, j = 0..2R; output row
// y+OFF-R (slot OFF) is then complete and written (if it is one of this CTA's
// rows).  After the group the slots shift down by kMorphGroup (register moves:
// a short loop body instead of a (2R+1)-phase unrolled one, which overflowed
// the instruction cache; groups divide the moves per row).
template <int R, bool MAX, bool TOPHAT, int OFF>
__device__ __forceinline__ void morph_row(Acc<R> &acc, const uint32_t *win, bool real, int64_t y,
                                          int64_t ylo, int64_t yhi, const MorphArgs &g, int z,
                                          int64_t xp, bool full) {
  if (real) {
    uint32_t h0[R + 1], h1[R + 1];
    cascade<R, MAX, 0>(win, h0, h1);
#pragma unroll
    for (int j = 0; j <= 2 * R; j++) {
      const int w = halfw<R>(R - j < 0 ? j - R : R - j);
      acc.a[j + OFF][0] = vop<MAX>(acc.a[j + OFF][0], h0[w]);
      acc.a[j + OFF][1] = vop<MAX>(acc.a[j + OFF][1], h1[w]);
    }
  }
  const int64_t yo = y - R;
  if (yo >= ylo && yo < yhi && xp < g.nx) {
    uint32_t a0 = acc.a[OFF][0], a1 = acc.a[OFF][1];
    const int64_t o = ((size_t)z * g.ny + yo) * g.nx + xp;
    if (TOPHAT) {
      // max(orig - open, 0) per 16-bit lane = max(orig, open) - open
      uint32_t ow = 0u;
      if (full) {
        ow = *reinterpret_cast<const uint32_t *>(g.orig + o);
      } else {
        for (int e = 0; e < 4; e++)
          if (xp + e < g.nx) ow |= (uint32_t)g.orig[o + e] << (8 * e);
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
        if (xp + e < g.nx) g.dst[o + e] = (uint8_t)((packed >> (8 * e)) & 0xffu);
    }
  }
}

template <int R, bool MAX>
__device__ __forceinline__ void shiftg(Acc<R> &acc) {
  constexpr uint32_t NEUT2 = (MAX ? 0u : 255u) * 0x00010001u;
  constexpr int G = kMorphGroup;
#pragma unroll
  for (int j = 0; j < 2 * R + G; j++) {
    acc.a[j][0] = j + G < 2 * R + G ? acc.a[j + G][0] : NEUT2;
    acc.a[j][1] = j + G < 2 * R + G ? acc.a[j + G][1] : NEUT2;
  }
}

// Row y's strip segment (pixels x0-PADL .. x0+kMorphStrip+PADL+3) as u16
// pixels: fetched into registers first (the loads fly while the current row
// is computed), stored into the idle row buffer afterwards.
template <int R>
struct RowFetch {
  static constexpr int PADL = R + R % 2;
  static constexpr int N = kMorphStrip + 2 * PADL + 4;
  static constexpr int PER = (N + kMorphThreads - 1) / kMorphThreads;
  uint16_t v[PER];
};

template <int R, bool MAX>
__device__ __forceinline__ void fetch_row(const uint8_t *src, int64_t y, int64_t x0, int64_t nx,
                                          RowFetch<R> &f) {
  constexpr uint16_t NEUT = MAX ? 0 : 255;
#pragma unroll
  for (int k = 0; k < RowFetch<R>::PER; k++) {
    const int i = threadIdx.x + k * kMorphThreads;
    const int64_t x = x0 - RowFetch<R>::PADL + i;
    f.v[k] = (i < RowFetch<R>::N && x >= 0 && x < nx) ? (uint16_t)__ldg(src + y * nx + x) : NEUT;
  }
}

template <int R>
__device__ __forceinline__ void store_row(const RowFetch<R> &f, uint16_t *rb) {
#pragma unroll
  for (int k = 0; k < RowFetch<R>::PER; k++) {
    const int i = threadIdx.x + k * kMorphThreads;
    if (i < RowFetch<R>::N) rb[i] = f.v[k];
  }
}

template <int R, bool MAX, bool TOPHAT>
__global__ void __launch_bounds__(kMorphThreads) k_morph(MorphArgs g) {
  constexpr int PADL = R + R % 2;
  constexpr int BW = (kMorphStrip + 2 * PADL + 4) / 2;
  constexpr int NS = 2 * R + 1;
  constexpr uint32_t NEUT2 = (MAX ? 0u : 255u) * 0x00010001u;
  __shared__ __align__(16) uint16_t bufs[2 * 2 * BW];
  const int z = blockIdx.z;
  const int64_t x0 = (int64_t)blockIdx.x * kMorphStrip;
  const int64_t ylo = (int64_t)blockIdx.y * kMorphChunk, yhi = min(g.ny, ylo + kMorphChunk);
  const uint8_t *src = g.src + (size_t)z * g.nx * g.ny;
  const int64_t xp = x0 + 4 * threadIdx.x;
  Acc<R> acc;
#pragma unroll
  for (int k = 0; k < NS + kMorphGroup - 1; k++) acc.a[k][0] = acc.a[k][1] = NEUT2;
  // input rows ylo-R .. yhi+R-1 (outside the slice: no contribution)
  constexpr int WINW = PADL + 3;
  int64_t y = ylo - R;
  const int64_t yend = yhi + R;
  // 16-byte... 4-byte aligned output (and top-hat input) words for the whole walk
  const bool full = xp + 3 < g.nx && (g.nx & 3) == 0 &&
                    ((reinterpret_cast<uintptr_t>(g.dst) |
                      (TOPHAT ? reinterpret_cast<uintptr_t>(g.orig) : 0u)) & 3u) == 0;
  int cur = 0;
  if (y >= 0 && y < g.ny) {
    RowFetch<R> f0;
    fetch_row<R, MAX>(src, y, x0, g.nx, f0);
    store_row<R>(f0, bufs);
  }
  __syncthreads();
  auto row = [&](auto off_tag) {
    constexpr int OFF = decltype(off_tag)::value;
    // the next row's pixels are fetched before this row is computed and
    // stored into the other buffer after it
    RowFetch<R> nf;
    const bool nxt = y + 1 < yend && y + 1 >= 0 && y + 1 < g.ny;
    if (nxt) fetch_row<R, MAX>(src, y + 1, x0, g.nx, nf);
    const bool real = y < yend && y >= 0 && y < g.ny;
    uint32_t win[WINW];
    const uint32_t *rb = reinterpret_cast<const uint32_t *>(bufs + cur * 2 * BW) + 2 * threadIdx.x;
#pragma unroll
    for (int j = 0; j < WINW; j++) win[j] = real ? rb[j] : 0u;
    morph_row<R, MAX, TOPHAT, OFF>(acc, win, real, y, ylo, yhi, g, z, xp, full);
    if (nxt) store_row<R>(nf, bufs + (cur ^ 1) * 2 * BW);
    __syncthreads();  // the other buffer is complete; this one may be overwritten
    cur ^= 1;
    y++;
  };
  while (y < yend) {
    row(std::integral_constant<int, 0>{});
    row(std::integral_constant<int, 1>{});
    if constexpr (kMorphGroup == 4) {
      row(std::integral_constant<int, 2>{});
      row(std::integral_constant<int, 3>{});
    }
    shiftg<R, MAX>(acc);
  }
}

}  // namespace tsa
