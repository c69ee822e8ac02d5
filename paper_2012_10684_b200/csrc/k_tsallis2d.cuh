// k_tsallis2d.cuh -- SURVEY.md §8(f) NEXT row 1: the paper's own 2-D Tsallis
// thresholding, one thread-block cluster per slice.
//
//   g(x,y)  = floor(sum_{3x3} f / 9), replicate border            PAPER.md:566-570 (R18, R19)
//   h(i,j)  = #{f = i, g = j}
//   class 1 = {i <= t, j <= s}, class 2 = {i > t, j > s}           PAPER.md:578-591 (R20)
//   A_c     = sum_{class c} (h / n_c)^q,  phi = (A_1 A_2 - 1)/(1 - q)  (q == 1: S_1 + S_2)
//   (t*,s*) = argmax phi over [0, L-2]^2, lowest (t,s) on exact ties  PAPER.md:593-597 (R21)
//   label   = [f > t*]  ("only t is used")                          PAPER.md:597 (R22)
//
// B200 design.  The 2-D histogram of an 8-bit slice is 256 x 256 u32 = 256 KB,
// more than one SM's shared memory, so a slice is owned by a cluster of CL
// CTAs (one per SM, ~210 KB of shared memory each) and never leaves the chip:
//   1. histogram: CTA c reads image rows [c ny/CL, (c+1) ny/CL) (16-pixel
//      items, 16-bit-lane SWAR 3x3 box sums, exact floor(v/9) = (7282 v) >> 16,
//      a register ring keeping 4 rows of loads in flight) and counts (f,g)
//      codes into a PRIVATE full L x L histogram of 16-bit counters packed two
//      per word (a CTA counts <= 65535 pixels per round, so no counter can
//      wrap); uniform items add 16, warp-uniform ones 16 x lanes at once.
//   2. merge over DSMEM: the non-empty f-rows (union of the CTAs' row masks)
//      are split evenly over the cluster in row order; CTA r sums its rows of
//      all CL private histograms into compacted u32 rows (several counting
//      rounds, for slices over CL x 65535 pixels: static bands of R rows).
//   3. band column sums are exchanged over DSMEM: every CTA gets the
//      column totals of the bands below / above it (the SAT boundary values).
//   4. prefix walk: groups of rows (as many as the free shared memory holds),
//      one warp per row scans the row (lane = 8 contiguous columns, warp scan
//      of lane totals), then thread s walks the rows adding the row prefix to
//      its running (n_1, W_1) = summed-area table value at (t, s) and stores
//      A_1(t,s) = W_1 / n_1^q in shared memory.
//   5. suffix walk: the same from the top row down with row suffixes, giving
//      (n_2, W_2) of class 2 directly (sums of non-negative terms, no prefix
//      differences, no cancellation), the score A_1 A_2 (+-, or S_1 + S_2 at
//      q = 1) and a running (score, key = t L + s) best.
//   6. argmax: warp shuffles, block, then over the cluster via DSMEM, carrying
//      the winner's class terms, from which phi(t*,s*) = H_1 + H_2 +
//      (1-q) H_1 H_2 is formed (2-D objective).
// Only canonical candidates -- row t and column s non-empty -- are scored:
// every other candidate describes the same partition as a canonical one and
// the lowest member of each class is canonical (R21), so the result
// equals the exhaustive argmax and the summation order of the tables need not
// make equivalent candidates tie bit for bit.  w(c) = c^q (c ln c at q = 1)
// and 1/n^q (ln n, 1/n) come from n-indexed tables (k2d_luts).
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

#include "tsa_device.cuh"

namespace tsa {

namespace cg = cooperative_groups;

constexpr int k2dThreads = 256;  // CTA size of the cluster kernel
constexpr int k2dGroup = k2dThreads / 32;  // rows per walk group (one warp per row)
constexpr int k2dMaxCL = 8;
constexpr int kStageChunks = 8;  // bulk copies (mbarriers) staging a CTA's image rows

struct Tsa2dArgs {
  const uint8_t *vol;     // [nz][ny][nx]
  int64_t nx, ny, nz;
  int L, LP;              // bins, even row pitch of the 2-D tables
  int CL, R;              // CTAs per cluster, f-rows per band (R = ceil(L / CL))
  int rr;                 // image rows per counting round (rr * nx <= 65535; one round: <= 65536)
  int rounds;             // counting rounds (same for every CTA of a cluster)
  int vec;                // 16-pixel SWAR path (nx % 16 == 0, 16-byte aligned slices)
  double q;
  int mode;               // PROD_MAX / PROD_MIN / SUM (q == 1)
  const double *wlut;     // [N+1] w(c): c^q, or c ln c at q == 1; w(0) = 0
  const double *ipow;     // [N+1] 1/n^q (NaN at 0)          (q != 1)
  const double *lnn;      // [N+1] ln n (NaN at 0)            (q == 1)
  const double *rcp;      // unused (null): S = ln n - W / n
  int32_t *thresholds;    // [nz][2] (t, s), -1 on error
  int32_t *tlab;          // [nz] t for the label kernel (-1 on error)
  double *objective;      // [nz] or null
  uint32_t *hist;         // [nz][L][L] or null
  int32_t *status;        // [nz] (workspace, read by the label kernel)
  int32_t *status2;       // [nz] or null (caller's copy)
  int hist_only;          // stop after the histogram (tsa2d_histogram)
};

// ------------------------------------------------------------------ luts
__global__ void k2d_luts(double *wlut, double *ipow, double *lnn, double *rcp, int64_t N, double q,
                         int shannon) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n <= N;
       n += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)n;
    if (shannon) {
      wlut[n] = n == 0 ? 0.0 : __dmul_rn(x, log(x));
      lnn[n] = n == 0 ? CUDART_NAN : log(x);
      if (rcp) rcp[n] = n == 0 ? CUDART_NAN : __drcp_rn(x);
    } else {
      const double pw = pow(x, q);
      wlut[n] = n == 0 ? 0.0 : pw;
      ipow[n] = n == 0 ? CUDART_NAN : __drcp_rn(pw);
    }
  }
}

// ------------------------------------------------------- 3x3 mean helpers
// 16-bit-lane horizontal 3-sums of the 4 pixels of word w (bytes b0..b3 =
// pixels x..x+3), lb = pixel x-1, rb = pixel x+4 (already border-replicated):
//   lo = (lb+b0+b1, b0+b1+b2), hi = (b1+b2+b3, b2+b3+rb)   (each <= 765)
__device__ __forceinline__ void hsum4(uint32_t w, uint32_t lb, uint32_t rb, uint32_t &lo,
                                      uint32_t &hi) {
  const uint32_t pL0 = __byte_perm(w, lb, 0x5054);  // (lb, b0)
  const uint32_t p01 = __byte_perm(w, 0u, 0x4140);  // (b0, b1)
  const uint32_t p12 = __byte_perm(w, 0u, 0x4241);  // (b1, b2)
  const uint32_t p23 = __byte_perm(w, 0u, 0x4342);  // (b2, b3)
  const uint32_t p3R = __byte_perm(w, rb, 0x5453);  // (b3, rb)
  lo = pL0 + p01 + p12;
  hi = p12 + p23 + p3R;
}

// floor(v / 9) for 0 <= v <= 2295 (= 9 * 255): (7282 v) >> 16 is exact on that range
__device__ __forceinline__ uint32_t div9(uint32_t v) { return (v * 7282u) >> 16; }

__device__ __forceinline__ uint32_t ldg_u8(const uint8_t *p) { return (uint32_t)__ldg(p); }

// image row y's word gx plus its border-replicated neighbour pixels
__device__ __forceinline__ void load_row4(const uint8_t *row, int64_t gx, int64_t G4, uint32_t &w,
                                          uint32_t &lb, uint32_t &rb) {
  w = __ldg(reinterpret_cast<const uint32_t *>(row) + gx);
  lb = gx > 0 ? ldg_u8(row + 4 * gx - 1) : (w & 0xffu);
  rb = gx < G4 - 1 ? ldg_u8(row + 4 * gx + 4) : (w >> 24);
}

// --------------------------------------------------------- stage: g image
// tsa2d_mean3x3: g for every pixel (the same SWAR arithmetic as the cluster
// kernel when vec, else scalar).  grid (x-chunks, nz), 256 threads.
__global__ void __launch_bounds__(256) k2d_mean(const uint8_t *vol, uint8_t *g, int64_t nx,
                                                int64_t ny, int vec) {
  const int64_t z = blockIdx.y;
  const uint8_t *f = vol + z * nx * ny;
  uint8_t *gz = g + z * nx * ny;
  if (vec) {
    const int64_t G4 = nx / 4;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < G4 * ny;
         it += (int64_t)gridDim.x * blockDim.x) {
      const int64_t y = it / G4, gx = it % G4;
      uint32_t lo = 0, hi = 0;
      for (int dy = -1; dy <= 1; dy++) {
        const int64_t yy = min(max(y + dy, (int64_t)0), ny - 1);
        uint32_t w, lb, rb, l, h;
        load_row4(f + yy * nx, gx, G4, w, lb, rb);
        hsum4(w, lb, rb, l, h);
        lo += l;
        hi += h;
      }
      const uint32_t out = div9(lo & 0xffffu) | div9(lo >> 16) << 8 | div9(hi & 0xffffu) << 16 |
                           div9(hi >> 16) << 24;
      *reinterpret_cast<uint32_t *>(gz + y * nx + 4 * gx) = out;
    }
  } else {
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nx * ny;
         it += (int64_t)gridDim.x * blockDim.x) {
      const int64_t y = it / nx, x = it % nx;
      uint32_t v = 0;
      for (int dy = -1; dy <= 1; dy++)
        for (int dx = -1; dx <= 1; dx++) {
          const int64_t yy = min(max(y + dy, (int64_t)0), ny - 1);
          const int64_t xx = min(max(x + dx, (int64_t)0), nx - 1);
          v += f[yy * nx + xx];
        }
      gz[it] = (uint8_t)div9(v);
    }
  }
}

// ------------------------------------------------------------ block scans
// inclusive scan over the CTA (one element per thread, thread order) of an
// exact count and a double; scratch >= 32 * 16 bytes.  Fixed tree: results
// are a pure function of the inputs.
__device__ __forceinline__ void block_incl_scan(uint32_t &n, double &w, char *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t on = __shfl_up_sync(0xffffffffu, n, off);
    const double ow = __shfl_up_sync(0xffffffffu, w, off);
    if (lane >= off) {
      n += on;
      w = __dadd_rn(ow, w);
    }
  }
  uint32_t *sn = reinterpret_cast<uint32_t *>(scratch);
  double *sw = reinterpret_cast<double *>(scratch + 256);
  if (lane == 31) {
    sn[warp] = n;
    sw[warp] = w;
  }
  __syncthreads();
  uint32_t bn = 0;
  double bw = 0.0;
  for (int i = 0; i < warp && i < nw; i++) {
    bn += sn[i];
    bw = __dadd_rn(bw, sw[i]);
  }
  n += bn;
  w = __dadd_rn(bw, w);
  __syncthreads();
}

// exclusive SUFFIX scan (sum over threads > this one)
__device__ __forceinline__ void block_excl_suffix_scan(uint32_t &n, double &w, char *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t in = n;
  double iw = w;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t on = __shfl_down_sync(0xffffffffu, in, off);
    const double ow = __shfl_down_sync(0xffffffffu, iw, off);
    if (lane + off < 32) {
      in += on;
      iw = __dadd_rn(iw, ow);
    }
  }
  uint32_t *sn = reinterpret_cast<uint32_t *>(scratch);
  double *sw = reinterpret_cast<double *>(scratch + 256);
  if (lane == 0) {
    sn[warp] = in;
    sw[warp] = iw;
  }
  __syncthreads();
  uint32_t bn = 0;
  double bw = 0.0;
  for (int i = nw - 1; i > warp; i--) {
    bn += sn[i];
    bw = __dadd_rn(bw, sw[i]);
  }
  // exclusive within the warp: inclusive of the next lane
  uint32_t xn = __shfl_down_sync(0xffffffffu, in, 1);
  double xw = __shfl_down_sync(0xffffffffu, iw, 1);
  if (lane == 31) {
    xn = 0;
    xw = 0.0;
  }
  n = xn + bn;
  w = __dadd_rn(xw, bw);
  __syncthreads();
}

// class term of a (count, W) rectangle: A = W / n^q, or S = ln n - W / n at
// q == 1 (Shannon, R6); NaN if n == 0 (the LUTs hold NaN at 0)
template <int MODE>
__device__ __forceinline__ double term2d(uint32_t n, double W, const Tsa2dArgs &a) {
  if (MODE == SUM) return __dsub_rn(__ldg(a.lnn + n), __ddiv_rn(W, (double)n));
  return __dmul_rn(W, __ldg(a.ipow + n));
}

// the same term from an already gathered LUT value g (ipow[n] or lnn[n])
template <int MODE>
__device__ __forceinline__ double term2d_g(uint32_t n, double W, double g) {
  if (MODE == SUM) return __dsub_rn(g, __ddiv_rn(W, (double)n));
  return __dmul_rn(W, g);
}

// 8-byte global -> shared async copy (zero-fill when !valid), LDGSTS
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int MODE>
__device__ __forceinline__ double score2d(double t1, double t2) {
  if (MODE == SUM) return __dadd_rn(t1, t2);
  const double p = __dmul_rn(t1, t2);
  return MODE == PROD_MAX ? p : -p;
}

// -------------------------------------------------------------- the kernel
// Shared-memory layout (bytes, every offset 16-aligned).  Band-row tables use
// the pitch PP = LP rounded up to 8 with column j at j ^ ((j >> 5) & 7) (an
// XOR swizzle inside each aligned 8-column group), so a lane reading 8
// contiguous columns and a thread reading column s are both bank-conflict
// free, without the 12.5 % of a padded pitch.
//   A      max(L*LP*2, R*LP*8): private u16 histogram; later A_1 / S_1 [nrl][LP]
//          f64 and, in the tail, walk buffers for as many rows as fit
//   Hb     R*PP*4              merged u32 rows of the band (compacted)
//   gN     G*PP*4, gW G*PP*8   fallback walk buffers (G = 8 rows)
//   colN   LP*4, colW LP*8     band column sums (read by the other CTAs)
//   rla    R*4, rlh R*4        absolute f-row / Hb row of each non-empty band row
//   msk    16 words            non-empty f-rows (own private histogram, then all);
//                              words 8.. the cluster's wrapped cells (Xch::extra)
//   xch    128                 exchange slots (flags, mask, argmax + payload)
//   bar    64                  mbarriers of the staged image rows
//   scr    1024                scan scratch
struct Smem2d {
  size_t A, Abytes, Hb, gN, gW, colN, colW, rla, rlh, msk, xch, bar, scr, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline int pitch2d(int LP) { return (LP + 7) & ~7; }

__host__ __device__ inline Smem2d smem2d_layout(int L, int LP, int R) {
  Smem2d s;
  const int PP = pitch2d(LP);
  size_t o = 0;
  s.A = o;
  const size_t a1 = (size_t)L * LP * 2, a2 = (size_t)R * LP * 8;
  s.Abytes = al16(a1 > a2 ? a1 : a2);
  o += s.Abytes;
  s.Hb = o;
  o += al16((size_t)R * PP * 4);
  s.gN = o;
  o += al16((size_t)k2dGroup * PP * 4);
  s.gW = o;
  o += al16((size_t)k2dGroup * PP * 8);
  s.colN = o;
  o += al16((size_t)LP * 4);
  s.colW = o;
  o += al16((size_t)LP * 8);
  s.rla = o;
  o += al16((size_t)R * 4);
  s.rlh = o;
  o += al16((size_t)R * 4);
  s.msk = o;
  o += 64;
  s.xch = o;
  o += 128;
  s.bar = o;
  o += 8 * kStageChunks;
  s.scr = o;
  o += 1024;
  s.total = o;
  return s;
}

__device__ __forceinline__ int pj(int j) { return j ^ ((j >> 5) & 7); }

// exchange slots read by the other CTAs of the cluster
struct Xch {
  int flags;           // LEVEL_OVERFLOW seen
  int extra;           // single round: f << 16 | g if all 65536 pixels fell in that cell, else -1
  uint32_t mask[8];    // non-empty f-rows of this CTA's private histogram (L <= 256)
  double score;        // CTA best (score, key) and its two class terms
  uint64_t key;
  double t1, t2;
};

// one image row's 16-pixel item: pixels x0..x0+15 (uint4) and the
// border-replicated neighbours x0-1, x0+16
struct Raw16 {
  uint4 w;
  uint32_t lb, rb;
};

__device__ __forceinline__ Raw16 load16(const uint8_t *row, int64_t gx, int64_t G16) {
  Raw16 r;
  r.w = __ldg(reinterpret_cast<const uint4 *>(row) + gx);
  r.lb = gx > 0 ? ldg_u8(row + 16 * gx - 1) : (r.w.x & 0xffu);
  r.rb = gx < G16 - 1 ? ldg_u8(row + 16 * gx + 16) : (r.w.w >> 24);
  return r;
}

// horizontal 3-sums of the 16 pixels: 8 words of two 16-bit lanes
__device__ __forceinline__ void hsum16(const Raw16 &r, uint32_t *hs) {
  hsum4(r.w.x, r.lb, r.w.y & 0xffu, hs[0], hs[1]);
  hsum4(r.w.y, r.w.x >> 24, r.w.z & 0xffu, hs[2], hs[3]);
  hsum4(r.w.z, r.w.y >> 24, r.w.w & 0xffu, hs[4], hs[5]);
  hsum4(r.w.w, r.w.z >> 24, r.rb, hs[6], hs[7]);
}

// Private-histogram cell (f, g): 16-bit counter (g & 1) of word
//   f * rw + 4 * ((g >> 3) ^ (f & 7)) + ((g >> 1) & 3)         (rw = LP/2 words per row)
// The XOR swizzle of 16-byte chunks by f spreads the rows of one g column over
// 8 bank groups (unswizzled, a row pitch of 128 words puts every f of a column
// in the same bank and the noisy tissue pixels' atomics collide ~11-way).
// Applied when rw % 32 == 0 (then the swizzled chunk stays inside the row).
__device__ __forceinline__ uint32_t cell_word(uint32_t f, uint32_t g, uint32_t rw, bool swz) {
  const uint32_t ch = swz ? ((g >> 3) ^ (f & 7u)) : (g >> 3);
  return f * rw + (ch << 2) + ((g >> 1) & 3u);
}

// L = 256 fast encoding of the same layout with a 32-chunk swizzle: pixel with
// f (as f8 = f << 8) and box sum v (from h2 = umulhi(v << 16, 14564) =
// floor(v * 7282 / 2^15) = 2 g or 2 g + 1) has byte offset
//   f * 512 + ((h2 ^ 16 f) & 0x1fc)     (chunk ((g >> 3) ^ f) & 31, word (g >> 1) & 3)
// and counter half (h2 >> 1) & 1 = g & 1.  ~9 integer instructions per pixel.
__device__ __forceinline__ void add256(char *hpb, uint32_t f8, uint32_t h2, uint32_t n) {
  const uint32_t off = f8 * 2u + ((h2 ^ (f8 >> 4)) & 0x1fcu);
  atomicAdd(reinterpret_cast<uint32_t *>(hpb + off), n << ((h2 & 2u) << 3));
}
// cell word of the L = 256 layout (merge side)
__device__ __forceinline__ uint32_t cell_word256(uint32_t f, uint32_t g) {
  return f * 128u + 4u * (((g >> 3) ^ f) & 31u) + ((g >> 1) & 3u);
}

__device__ __forceinline__ void add_code(uint32_t *hp, uint32_t f, uint32_t g, uint32_t rw, bool swz,
                                         uint32_t n) {
  // rw == 128 (L = 256): the 32-chunk layout of add256 / cell_word256
  const uint32_t w = rw == 128u ? cell_word256(f, g) : cell_word(f, g, rw, swz);
  atomicAdd(hp + w, n << ((g & 1u) << 4));
}

// (TMA bulk staging helpers: tsa_device.cuh)

// Rows [Y0, Y1) of the slice staged in shared memory by kStageChunks bulk
// copies, chunk c = rows [Y0 + c cr, Y0 + (c+1) cr), each with its mbarrier.
struct Stage {
  const uint8_t *buf;  // shared memory holding row Y0 at offset 0
  uint64_t *bar;       // [kStageChunks]
  int64_t Y0, Y1, cr;
};

// Count the (f, g) codes of image rows [ya, yb) into the packed u16 histogram.
// VEC: items of 16 pixels (nx % 16 == 0, 16-byte aligned slices); each item
// walks a stripe of rows.  STAGED: rows come from the shared-memory stage
// (the stripe first waits for the chunks it needs); otherwise from global
// memory through a register ring prefetching kPF rows ahead.
constexpr int kPF = 4;

template <bool STAGED>
__device__ __forceinline__ Raw16 row16(const uint8_t *f, const Stage &sg, int64_t y, int64_t nx,
                                       int64_t gx, int64_t G16) {
  if (STAGED) {
    const uint8_t *row = sg.buf + (y - sg.Y0) * nx;
    Raw16 r;
    r.w = *reinterpret_cast<const uint4 *>(row + 16 * gx);
    r.lb = gx > 0 ? (uint32_t)row[16 * gx - 1] : (r.w.x & 0xffu);
    r.rb = gx < G16 - 1 ? (uint32_t)row[16 * gx + 16] : (r.w.w >> 24);
    return r;
  }
  return load16(f + y * nx, gx, G16);
}

template <bool VEC, bool CHECK, bool STAGED, int LT>
__device__ __forceinline__ void count_round(const Tsa2dArgs &a, const uint8_t *f, const Stage &sg,
                                            int64_t ya, int64_t yb, uint32_t *hp, int &ovf) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t nx = a.nx, ny = a.ny;
  const int LP = LT ? LT : a.LP, L = LT ? LT : a.L;
  const uint32_t rw = (uint32_t)LP / 2;
  const bool swz = (rw & 31u) == 0;
  if (yb <= ya) return;
  if (VEC) {
    const int64_t G16 = nx / 16;
    const int64_t S = G16 >= k2dThreads ? 1 : k2dThreads / G16;  // row stripes
    const int64_t rows = yb - ya, per = (rows + S - 1) / S;
    for (int64_t item = tid; item < G16 * S; item += k2dThreads) {
      const int64_t gx = item % G16, st = item / G16;
      const int64_t ys = ya + st * per, ye = min(yb, ys + per);
      if (ys >= ye) continue;
      if (STAGED) {
        const int64_t r0 = max(ys - 1, (int64_t)0), r1 = min(ye, ny - 1);
        for (int64_t c = (r0 - sg.Y0) / sg.cr; c <= (r1 - sg.Y0) / sg.cr; c++) mbar_wait(sg.bar + c, 0);
      }
      uint32_t hp_[8], hc[8], hn[8];
      {
        const Raw16 r0 = row16<STAGED>(f, sg, max(ys - 1, (int64_t)0), nx, gx, G16);
        hsum16(r0, hp_);
      }
      Raw16 cur = row16<STAGED>(f, sg, ys, nx, gx, G16);
      hsum16(cur, hc);
      Raw16 ring[kPF];
#pragma unroll
      for (int d = 0; d < kPF; d++)
        if (ys + 1 + d <= ye) ring[d] = row16<STAGED>(f, sg, min(ys + 1 + d, ny - 1), nx, gx, G16);
      for (int64_t y = ys; y < ye; y += kPF) {
#pragma unroll
        for (int d = 0; d < kPF; d++) {
          if (y + d < ye) {
            const Raw16 nxt = ring[d];
            const int64_t yl = y + d + 1 + kPF;  // row kept in this slot next
            if (yl <= ye) ring[d] = row16<STAGED>(f, sg, min(yl, ny - 1), nx, gx, G16);
            hsum16(nxt, hn);
            uint32_t box[8];
#pragma unroll
            for (int e = 0; e < 8; e++) box[e] = hp_[e] + hc[e] + hn[e];
            const uint32_t fw[4] = {cur.w.x, cur.w.y, cur.w.z, cur.w.w};
            if (!CHECK) {
              const uint32_t f0 = fw[0] & 0xffu;
              bool uni = fw[0] == f0 * 0x01010101u && fw[1] == fw[0] && fw[2] == fw[0] &&
                         fw[3] == fw[0];
              const uint32_t b0 = box[0] & 0xffffu;
#pragma unroll
              for (int e = 0; e < 8; e++) uni = uni && box[e] == (b0 | (b0 << 16));
              const uint32_t g0 = div9(b0);
              const uint32_t c0 = f0 * LP + g0;
              const unsigned m = __activemask();
              const int leader = __ffs(m) - 1;
              const uint32_t cl = __shfl_sync(m, c0, leader);
              if (__all_sync(m, uni && c0 == cl)) {
                if (lane == leader) add_code(hp, f0, g0, rw, swz, 16u * __popc(m));
              } else if (uni) {
                add_code(hp, f0, g0, rw, swz, 16u);
              } else if (LT == 256) {
                char *hpb = reinterpret_cast<char *>(hp);
#pragma unroll
                for (int e = 0; e < 16; e++) {
                  const uint32_t f8 = __byte_perm(fw[e >> 2], 0u, 0x4404u | ((e & 3) << 4));
                  const uint32_t vs = (e & 1) ? (box[e >> 1] & 0xffff0000u) : (box[e >> 1] << 16);
                  add256(hpb, f8, __umulhi(vs, 14564u), 1u);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 16; e++) {
                  const uint32_t fv = (fw[e >> 2] >> (8 * (e & 3))) & 0xffu;
                  const uint32_t bv = (box[e >> 1] >> (16 * (e & 1))) & 0xffffu;
                  add_code(hp, fv, div9(bv), rw, swz, 1u);
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; e++) {
                const uint32_t fv = (fw[e >> 2] >> (8 * (e & 3))) & 0xffu;
                const uint32_t gv = div9((box[e >> 1] >> (16 * (e & 1))) & 0xffffu);
                if (fv >= (uint32_t)L || gv >= (uint32_t)L) {
                  ovf = 1;
                  continue;
                }
                add_code(hp, fv, gv, rw, swz, 1u);
              }
            }
#pragma unroll
            for (int e = 0; e < 8; e++) {
              hp_[e] = hc[e];
              hc[e] = hn[e];
            }
            cur = nxt;
          }
        }
      }
    }
  } else {
    const int64_t npx = (yb - ya) * nx;
    for (int64_t it = tid; it < npx; it += k2dThreads) {
      const int64_t y = ya + it / nx, x = it % nx;
      uint32_t v = 0;
      for (int dy = -1; dy <= 1; dy++)
        for (int dx = -1; dx <= 1; dx++) {
          const int64_t yy = min(max(y + dy, (int64_t)0), ny - 1);
          const int64_t xx = min(max(x + dx, (int64_t)0), nx - 1);
          v += ldg_u8(f + yy * nx + xx);
        }
      const uint32_t fv = ldg_u8(f + y * nx + x), gv = div9(v);
      if (CHECK && (fv >= (uint32_t)L || gv >= (uint32_t)L)) {
        ovf = 1;
        continue;
      }
      add_code(hp, fv, gv, rw, swz, 1u);
    }
    (void)lane;
  }
}

// Single round of 65536 pixels (kept out of line: rarely taken, and inlined
// it costs the kernel registers).  Only a cell holding all 65536 pixels can
// wrap its 16-bit counter, and then it is the cell of pixel (ya, 0): counted,
// yet reading 0.  The word is cleared (a low-half wrap carried into the other
// half), the f-row kept in the mask; returns f << 16 | g, else -1.
__device__ __noinline__ int wrap_check(const uint8_t *f, int64_t nx, int64_t ny, int64_t ya,
                                       const uint8_t *buf, uint64_t *bar, int64_t Y0,
                                       uint32_t *hp, int L, int rw, bool swz, uint32_t *msk) {
  // the rows are in the CTA's region, whose chunks have all landed (the
  // waits complete at once; no 64-bit index division on this path)
  if (buf)
    for (int c = 0; c < kStageChunks; c++) mbar_wait(bar + c, 0);
  const int64_t y0 = max(ya - 1, (int64_t)0), y2 = min(ya + 1, ny - 1), x1 = min((int64_t)1, nx - 1);
  const int64_t rows[3] = {y0, ya, y2}, cols[3] = {0, 0, x1};
  uint32_t px[9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      px[i * 3 + j] = buf ? (uint32_t)buf[(rows[i] - Y0) * nx + cols[j]] : ldg_u8(f + rows[i] * nx + cols[j]);
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < 9; j++) v += px[j];
  const uint32_t fv = px[4];
  const uint32_t gv = div9(v);
  if (fv >= (uint32_t)L || gv >= (uint32_t)L) return -1;
  uint32_t *wp = hp + (rw == 128 ? cell_word256(fv, gv) : cell_word(fv, gv, (uint32_t)rw, swz));
  if (((*wp >> ((gv & 1u) << 4)) & 0xffffu) != 0u) return -1;
  *wp = 0u;
  atomicOr(&msk[fv >> 5], 1u << (fv & 31));
  return (int)(fv << 16 | gv);
}

// adds the 65536 pixels of a wrapped cell e to this CTA's band if its row is
// one of the band's compacted rows (the band = union ranks [k0, k1))
__device__ __noinline__ void wrap_add(uint32_t *Hb, const uint32_t *msk, int e, int r, int CL, int NW,
                                      int PP) {
  const int fe = e >> 16, ge = e & 0xffff;
  int mf = 0, rank = __popc(msk[fe >> 5] & ((1u << (fe & 31)) - 1u));
  for (int w = 0; w < NW; w++) {
    const int pc = __popc(msk[w]);
    mf += pc;
    if (w < (fe >> 5)) rank += pc;
  }
  const int k0 = r * mf / CL, k1 = (r + 1) * mf / CL;
  if (rank >= k0 && rank < k1) atomicAdd(&Hb[(rank - k0) * PP + pj(ge)], 65536u);
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// argmax with the winning candidate's two class terms as payload
__device__ __forceinline__ void warp_argmax4(double &s, uint64_t &k, double &t1, double &t2) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, s, off);
    const uint64_t ok = __shfl_xor_sync(0xffffffffu, k, off);
    const double o1 = __shfl_xor_sync(0xffffffffu, t1, off);
    const double o2 = __shfl_xor_sync(0xffffffffu, t2, off);
    if (better(os, ok, s, k)) {
      s = os;
      k = ok;
      t1 = o1;
      t2 = o2;
    }
  }
}

// LT = 256: the paper's 8-bit case with every table dimension a compile-time
// constant (L = LP = PP = 256, 8 columns per lane); LT = 0: any L.
template <int MODE, bool VEC, bool CHECK, int LT>
__global__ void __launch_bounds__(k2dThreads, 1) k_tsallis2d(Tsa2dArgs a) {
  extern __shared__ __align__(16) char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = a.CL, r = (int)cluster.block_rank();
  const int64_t z = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = LT ? LT : a.L, LP = LT ? LT : a.LP, R = a.R;
  const int PP = LT ? LT : pitch2d(LP);
  const int NW = (L + 31) / 32;  // mask words
  const Smem2d lay = smem2d_layout(L, LP, R);
  uint32_t *hp = reinterpret_cast<uint32_t *>(smem + lay.A);  // packed u16 private histogram
  double *A1 = reinterpret_cast<double *>(smem + lay.A);
  uint32_t *Hb = reinterpret_cast<uint32_t *>(smem + lay.Hb);
  uint32_t *colN = reinterpret_cast<uint32_t *>(smem + lay.colN);
  double *colW = reinterpret_cast<double *>(smem + lay.colW);
  int *rla = reinterpret_cast<int *>(smem + lay.rla);
  int *rlh = reinterpret_cast<int *>(smem + lay.rlh);
  uint32_t *msk = reinterpret_cast<uint32_t *>(smem + lay.msk);
  Xch *xch = reinterpret_cast<Xch *>(smem + lay.xch);
  char *scr = smem + lay.scr;
  const uint8_t *f = a.vol + z * a.nx * a.ny;
  const bool single = a.rounds == 1;  // balanced, compacted bands

  // ---- 1 + 2: counting, then the band rows of every private histogram merged
  // over DSMEM.  Single round: the non-empty f-rows (union of the CTAs' masks)
  // are split evenly over the cluster in row order and stored compacted.
  // Several rounds: band r = f-rows [r R, (r+1) R), accumulated per round.
  if (tid == 0) xch->flags = 0;
  const int row0 = r * R, nrows_static = max(0, min(L, row0 + R) - row0);
  if (!single)
    for (int i = tid; i < nrows_static * PP; i += k2dThreads) Hb[i] = 0u;
  int ovf = 0;
  int nst = 0;  // Hb rows in use
  const int64_t ya0 = (int64_t)r * a.ny / CL, yb0 = (int64_t)(r + 1) * a.ny / CL;
  // a CTA of the cluster may count 65536 pixels in its single round (cluster-uniform)
  const bool wrap_possible = a.rounds == 1 && (a.ny + CL - 1) / CL * a.nx == 65536;
  const int hw = L * LP / 2;  // words of the private histogram
  const int rw = LP / 2;      // words per private-histogram row
  const bool swz = (rw & 31) == 0;  // cell_word's chunk swizzle
  // single round, 16-pixel path: stage the CTA's image rows (plus the halo
  // rows) in the shared memory the band tables use later (Hb .. colN)
  Stage sg;
  sg.Y0 = max(ya0 - 1, (int64_t)0);
  sg.Y1 = min(yb0 + 1, a.ny);
  sg.cr = max((int64_t)1, (sg.Y1 - sg.Y0 + kStageChunks - 1) / kStageChunks);
  sg.buf = reinterpret_cast<const uint8_t *>(smem + lay.Hb);
  sg.bar = reinterpret_cast<uint64_t *>(smem + lay.bar);
  const bool staged = VEC && single && yb0 > ya0 &&
                      (size_t)(sg.Y1 - sg.Y0) * (size_t)a.nx <= lay.colN - lay.Hb;
  if (staged && tid == 0) {
    for (int c = 0; c < kStageChunks; c++) mbar_init(sg.bar + c, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int c = 0; c < kStageChunks; c++) {
      const int64_t r0 = sg.Y0 + c * sg.cr, r1 = min(sg.Y1, r0 + sg.cr);
      const uint32_t bytes = r1 > r0 ? (uint32_t)((r1 - r0) * a.nx) : 0u;
      mbar_expect_tx(sg.bar + c, bytes);
      if (bytes)
        bulk_g2s(smem + lay.Hb + (r0 - sg.Y0) * a.nx, f + r0 * a.nx, bytes, sg.bar + c);
    }
  }
  for (int rd = 0; rd < a.rounds; rd++) {
    uint4 *hp4 = reinterpret_cast<uint4 *>(hp);
    for (int i = tid; i < (hw + 3) / 4; i += k2dThreads) hp4[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid < 8) msk[tid] = 0u;
    __syncthreads();
    const int64_t ya = min(yb0, ya0 + (int64_t)rd * a.rr), yb = min(yb0, ya + a.rr);
    if (staged) count_round<VEC, CHECK, true, LT>(a, f, sg, ya, yb, hp, ovf);
    else count_round<VEC, CHECK, false, LT>(a, f, sg, ya, yb, hp, ovf);
    cluster.sync();  // every private histogram of this round complete
    if (single) {
      // own non-empty rows -> mask -> cluster union
      if ((rw & 3) == 0) {
        const uint4 *h4 = reinterpret_cast<const uint4 *>(hp);
        const int r4 = rw / 4;
#pragma unroll 4
        for (int i = warp; i < L; i += k2dThreads / 32) {
          uint32_t any = 0;
          for (int w = lane; w < r4; w += 32) {
            const uint4 v = h4[i * r4 + w];
            any |= v.x | v.y | v.z | v.w;
          }
          if (__any_sync(0xffffffffu, any != 0) && lane == 0) atomicOr(&msk[i >> 5], 1u << (i & 31));
        }
      } else {
        for (int i = warp; i < L; i += k2dThreads / 32) {
          uint32_t any = 0;
          for (int w = lane; w < rw; w += 32) any |= hp[i * rw + w];
          if (__any_sync(0xffffffffu, any != 0) && lane == 0) atomicOr(&msk[i >> 5], 1u << (i & 31));
        }
      }
      __syncthreads();
      if (wrap_possible) {
        // A single round may count 65536 pixels (one more than a 16-bit
        // counter holds); only a cell holding all of them can wrap, leaving
        // at most one non-empty row.  Then wrap_check clears the word, keeps
        // the row in the mask and publishes the cell; its band owner adds 65536.
        if (tid == 0) {
          int e = -1;
          if ((yb - ya) * a.nx == 65536) {
            int pc = 0;
            for (int w = 0; w < NW; w++) pc += __popc(msk[w]);
            if (pc <= 1) e = wrap_check(f, a.nx, a.ny, ya, staged ? sg.buf : nullptr, sg.bar, sg.Y0, hp, L, rw, swz, msk);
          }
          xch->extra = e;
        }
        __syncthreads();
      }
      if (tid < 8) xch->mask[tid] = msk[tid];
      cluster.sync();
      if (tid < NW) {
        uint32_t m = 0;
        for (int c = 0; c < CL; c++) m |= cluster.map_shared_rank(xch, c)->mask[tid];
        msk[tid] = m;
      }
      if (wrap_possible && tid < CL) msk[8 + tid] = (uint32_t)cluster.map_shared_rank(xch, tid)->extra;
      __syncthreads();
      int mf = 0, below = 0;
      for (int w = 0; w < NW; w++) {
        const int pc = __popc(msk[w]);
        if (w < (tid >> 5)) below += pc;
        mf += pc;
      }
      const int k0 = r * mf / CL, k1 = (r + 1) * mf / CL;
      nst = k1 - k0;
      if (tid < L && ((msk[tid >> 5] >> (tid & 31)) & 1u)) {
        const int rank = below + __popc(msk[tid >> 5] & ((1u << (tid & 31)) - 1u));
        if (rank >= k0 && rank < k1) {
          rla[rank - k0] = tid;
          rlh[rank - k0] = rank - k0;
        }
      }
      __syncthreads();
      // pull the nst rows (8 cells per item) from every private histogram
      const int cpr = (LP + 7) / 8;  // 8-cell chunks per row
      for (int it = tid; it < nst * cpr; it += k2dThreads) {
        const int kk = it / cpr, j = (it - kk * cpr) * 8, i = rla[kk];
        uint32_t o[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        if ((LP & 7) == 0) {
          // physical word of the chunk (swizzle of cell_word)
          const int pch = rw == 128 ? 4 * (((j >> 3) ^ i) & 31) : 4 * (swz ? ((j >> 3) ^ (i & 7)) : (j >> 3));
          uint4 v[k2dMaxCL];
#pragma unroll
          for (int c = 0; c < k2dMaxCL; c++)
            if (c < CL)
              v[c] = *reinterpret_cast<const uint4 *>(cluster.map_shared_rank(hp, c) + i * rw + pch);
#pragma unroll
          for (int c = 0; c < k2dMaxCL; c++)
            if (c < CL) {
              o[0] += v[c].x & 0xffffu;
              o[1] += v[c].x >> 16;
              o[2] += v[c].y & 0xffffu;
              o[3] += v[c].y >> 16;
              o[4] += v[c].z & 0xffffu;
              o[5] += v[c].z >> 16;
              o[6] += v[c].w & 0xffffu;
              o[7] += v[c].w >> 16;
            }
        } else {
          for (int c = 0; c < CL; c++) {
            const uint32_t *src = cluster.map_shared_rank(hp, c);
            for (int e = 0; e < 8 && j + e < LP; e += 2) {
              const uint32_t v = src[rw == 128 ? cell_word256(i, j + e) : cell_word(i, j + e, rw, swz)];
              o[e] += v & 0xffffu;
              o[e + 1] += v >> 16;
            }
          }
        }
        uint32_t *dst = Hb + kk * PP;
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (j + e < LP) dst[pj(j + e)] = o[e];
      }
    } else {
      for (int c = 0; c < CL; c++) {
        const uint32_t *src = cluster.map_shared_rank(hp, c);
        for (int i = tid; i < nrows_static * rw; i += k2dThreads) {
          const int ri = i / rw, j = 2 * (i - ri * rw);
          const uint32_t v = src[rw == 128 ? cell_word256(row0 + ri, j) : cell_word(row0 + ri, j, rw, swz)];
          if (v) {
            Hb[ri * PP + pj(j)] += v & 0xffffu;
            Hb[ri * PP + pj(j + 1)] += v >> 16;
          }
        }
      }
    }
    if (single && wrap_possible) {
      bool wrapped = false;
      for (int c = 0; c < CL; c++) wrapped |= (int)msk[8 + c] >= 0;
      if (wrapped) {  // rare: a CTA's whole round in one cell
        __syncthreads();
        if (tid < CL && (int)msk[8 + tid] >= 0) wrap_add(Hb, msk, (int)msk[8 + tid], r, CL, NW, PP);
      }
    }
    cluster.sync();  // all reads of the private histograms done before reuse
  }
  if (CHECK && ovf) atomicOr(&xch->flags, 1);
  if (!single) {
    // compacted list of the band's non-empty rows
    nst = nrows_static;
    for (int i = warp; i < nrows_static; i += k2dThreads / 32) {
      uint32_t any = 0;
      for (int j = lane; j < L; j += 32) any |= Hb[i * PP + pj(j)];
      any = __any_sync(0xffffffffu, any != 0);
      if (lane == 0) rlh[i] = any ? 1 : 0;
    }
    __syncthreads();
    if (warp == 0) {
      int cnt = 0;
      for (int b = 0; b < nrows_static; b += 32) {
        const int i = b + lane;
        const bool fl = i < nrows_static && rlh[i];
        const unsigned m = __ballot_sync(0xffffffffu, fl);
        __syncwarp();
        if (fl) {
          const int pos = cnt + __popc(m & ((1u << lane) - 1u));
          rlh[pos] = i;
          rla[pos] = row0 + i;
        }
        cnt += __popc(m);
        __syncwarp();
      }
      if (lane == 0) msk[8] = cnt;
    }
  }
  // optional histogram output: non-empty rows from Hb, the CTA's share of the
  // empty rows as zeros
  if (a.hist) {
    __syncthreads();
    uint32_t *hz = a.hist + (size_t)z * L * L;
    const int nl = single ? nst : (int)msk[8];
    for (int kk = warp; kk < nl; kk += k2dThreads / 32) {
      const int i = rla[kk], h = rlh[kk];
      for (int j = lane; j < L; j += 32) hz[(size_t)i * L + j] = Hb[h * PP + pj(j)];
    }
    const int e0 = r * L / CL, e1 = (r + 1) * L / CL;
    for (int i = e0 + warp; i < e1; i += k2dThreads / 32) {
      const bool empty = single ? !((msk[i >> 5] >> (i & 31)) & 1u) : false;
      if (empty)
        for (int j = lane; j < L; j += 32) hz[(size_t)i * L + j] = 0u;
    }
    if (!single) {  // static bands: empty band rows
      for (int i = warp; i < nrows_static; i += k2dThreads / 32) {
        bool any = false;
        for (int j = lane; j < L; j += 32) any |= Hb[i * PP + pj(j)] != 0u;
        if (!__any_sync(0xffffffffu, any))
          for (int j = lane; j < L; j += 32) hz[(size_t)(row0 + i) * L + j] = 0u;
      }
    }
  }

  // ---- 3: band column sums and the exchange
  const int s = tid;  // column owned in the walks (L <= 256 = k2dThreads)
  {
    uint32_t n = 0;
    double W = 0.0;
    if (s < L) {
#pragma unroll 4
      for (int i = 0; i < nst; i++) {
        const uint32_t h = Hb[i * PP + pj(s)];
        n += h;
        W = __dadd_rn(W, h ? __ldg(a.wlut + h) : 0.0);
      }
    }
    if (s < LP) {
      colN[s] = n;
      colW[s] = W;
    }
  }
  __syncthreads();
  cluster.sync();
  const int nrl = single ? nst : (int)msk[8];
  int any_ovf = 0;
  uint32_t lowN = 0, upN = 0, allN = 0;
  double lowW = 0.0, upW = 0.0;
  {
    uint32_t cn[k2dMaxCL];
    double cw[k2dMaxCL];
#pragma unroll
    for (int c = 0; c < k2dMaxCL; c++) {
      if (c < CL) {
        cn[c] = s < L ? cluster.map_shared_rank(colN, c)[s] : 0u;
        cw[c] = s < L ? cluster.map_shared_rank(colW, c)[s] : 0.0;
        if (CHECK) any_ovf |= cluster.map_shared_rank(&xch->flags, c)[0];
      }
    }
#pragma unroll
    for (int c = 0; c < k2dMaxCL; c++) {
      if (c < CL) {
        allN += cn[c];
        if (c < r) {
          lowN += cn[c];
          lowW = __dadd_rn(lowW, cw[c]);
        }
      }
    }
#pragma unroll
    for (int c = k2dMaxCL - 1; c >= 0; c--) {
      if (c < CL && c > r) {
        upN += cn[c];
        upW = __dadd_rn(upW, cw[c]);
      }
    }
  }
  const bool colnz = s < L && allN > 0;
  // prefix base B(s) = sum_{j <= s} low(j); suffix base B'(s) = sum_{j > s} up(j)
  block_incl_scan(lowN, lowW, scr);
  block_excl_suffix_scan(upN, upW, scr);
  double best = -CUDART_INF, bt1 = CUDART_NAN, bt2 = CUDART_NAN;
  uint64_t bkey = kKeyNone;
  if (!a.hist_only && !any_ovf && nrl > 0) {
    const int CPL = (L + 31) / 32;
    const int j0 = LT ? lane * (LT / 32) : min(L, lane * CPL);
    const int jn = LT ? LT / 32 : max(0, min(L, j0 + CPL) - j0);
    // walk buffers: the tail of region A behind A1[nrl][LP] if it holds at
    // least k2dGroup rows, else the fixed k2dGroup-row buffers
    const size_t a1b = al16((size_t)nrl * LP * 8);
    int G = (int)((lay.Abytes - a1b) / ((size_t)PP * 12));
    uint32_t *gN;
    double *gW;
    if (G >= k2dGroup) {
      G = min(G, nrl);
      gW = reinterpret_cast<double *>(smem + lay.A + a1b);
      gN = reinterpret_cast<uint32_t *>(smem + lay.A + a1b + (size_t)G * PP * 8);
    } else {
      G = k2dGroup;
      gW = reinterpret_cast<double *>(smem + lay.gW);
      gN = reinterpret_cast<uint32_t *>(smem + lay.gN);
    }
    // ---- 4: prefix walk over the non-empty rows: A_1 / S_1 of every (t, s)
    // with column s non-empty into A1[k][s] (k = compacted row index).  Empty
    // rows add nothing and are never canonical.
    uint32_t accN = lowN;
    double accW = lowW;
    for (int g0 = 0; g0 < nrl; g0 += G) {
      const int ge = min(G, nrl - g0);
      // w(h) of every cell of the warp's rows gathered into gW by async copies
      // (one L2 round trip for all of them), then the scans read them back
      for (int w = warp; w < ge; w += k2dThreads / 32) {
        const int i = rlh[g0 + w];
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (e < jn) {
            const uint32_t h = Hb[i * PP + pj(j0 + e)];
            cp_async8(gW + w * PP + pj(j0 + e), a.wlut + h, h != 0u);
          }
      }
      cp_async_wait_all();
      for (int w = warp; w < ge; w += k2dThreads / 32) {
        const int i = rlh[g0 + w];
        uint32_t hv[8];
        double wv[8];
#pragma unroll
        for (int e = 0; e < 8; e++) hv[e] = e < jn ? Hb[i * PP + pj(j0 + e)] : 0u;
#pragma unroll
        for (int e = 0; e < 8; e++) wv[e] = e < jn ? gW[w * PP + pj(j0 + e)] : 0.0;
        uint32_t ln = 0;
        double lw = 0.0;
#pragma unroll
        for (int e = 0; e < 8; e++) {
          ln += hv[e];
          lw = __dadd_rn(lw, wv[e]);
        }
        uint32_t xn = ln;
        double xw = lw;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t on = __shfl_up_sync(0xffffffffu, xn, off);
          const double ow = __shfl_up_sync(0xffffffffu, xw, off);
          if (lane >= off) {
            xn += on;
            xw = __dadd_rn(ow, xw);
          }
        }
        xn -= ln;  // exclusive count (exact)
        xw = __shfl_up_sync(0xffffffffu, xw, 1);
        if (lane == 0) xw = 0.0;
#pragma unroll
        for (int e = 0; e < 8; e++) {
          xn += hv[e];
          xw = __dadd_rn(xw, wv[e]);
          if (e < jn) {
            gN[w * PP + pj(j0 + e)] = xn;
            gW[w * PP + pj(j0 + e)] = xw;
          }
        }
      }
      __syncthreads();
      if (s < L) {
        // running (n_1, W_1) of every row of the group back into this column's
        // gN / gW slots, the 1/n^q (ln n) gathers straight into A1 by async
        // copies (one L2 round trip per group), then A_1 = W_1 / n_1^q in place
        const double *lut = MODE == SUM ? a.lnn : a.ipow;
        for (int w = 0; w < ge; w++) {
          const int c = w * PP + pj(s);
          accN += gN[c];
          accW = __dadd_rn(accW, gW[c]);
          gN[c] = accN;
          gW[c] = accW;
          cp_async8(A1 + (g0 + w) * LP + s, lut + accN, colnz);
        }
        cp_async_wait_all();
        for (int w = 0; w < ge; w++) {
          const int c = w * PP + pj(s);
          double *d = A1 + (g0 + w) * LP + s;
          *d = colnz ? term2d_g<MODE>(gN[c], gW[c], *d) : CUDART_NAN;
        }
      }
      __syncthreads();
    }
    // ---- 5: suffix walk (top row down), scores and the running best
    uint32_t sN = upN;
    double sW = upW;
    for (int g1 = nrl; g1 > 0; g1 -= G) {
      const int ge = min(G, g1);  // rows g1-1 down to g1-ge
      for (int w = warp; w < ge; w += k2dThreads / 32) {
        const int i = rlh[g1 - 1 - w];
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (e < jn) {
            const uint32_t h = Hb[i * PP + pj(j0 + e)];
            cp_async8(gW + w * PP + pj(j0 + e), a.wlut + h, h != 0u);
          }
      }
      cp_async_wait_all();
      for (int w = warp; w < ge; w += k2dThreads / 32) {
        const int i = rlh[g1 - 1 - w];
        uint32_t hv[8];
        double wv[8];
#pragma unroll
        for (int e = 0; e < 8; e++) hv[e] = e < jn ? Hb[i * PP + pj(j0 + e)] : 0u;
#pragma unroll
        for (int e = 0; e < 8; e++) wv[e] = e < jn ? gW[w * PP + pj(j0 + e)] : 0.0;
        uint32_t ln = 0;
        double lw = 0.0;
#pragma unroll
        for (int e = 7; e >= 0; e--) {
          ln += hv[e];
          lw = __dadd_rn(lw, wv[e]);
        }
        uint32_t xn = ln;
        double xw = lw;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t on = __shfl_down_sync(0xffffffffu, xn, off);
          const double ow = __shfl_down_sync(0xffffffffu, xw, off);
          if (lane + off < 32) {
            xn += on;
            xw = __dadd_rn(xw, ow);
          }
        }
        uint32_t cn = __shfl_down_sync(0xffffffffu, xn, 1);
        double cw = __shfl_down_sync(0xffffffffu, xw, 1);
        if (lane == 31) {
          cn = 0;
          cw = 0.0;
        }
        // row suffix at column j = sum over columns > j
#pragma unroll
        for (int e = 7; e >= 0; e--) {
          if (e < jn) {
            gN[w * PP + pj(j0 + e)] = cn;
            gW[w * PP + pj(j0 + e)] = cw;
          }
          cn += hv[e];
          cw = __dadd_rn(cw, wv[e]);
        }
      }
      __syncthreads();
      if (s < L) {
        for (int w0 = 0; w0 < ge; w0 += 8) {
          uint32_t nn[8];
          double wwv[8];
#pragma unroll
          for (int w = 0; w < 8; w++) {
            // (sN, sW) before the row is added = class 2 of (t, s): rows > t, columns > s
            nn[w] = sN;
            wwv[w] = sW;
            if (w0 + w < ge) {
              sN += gN[(w0 + w) * PP + pj(s)];
              sW = __dadd_rn(sW, gW[(w0 + w) * PP + pj(s)]);
            }
          }
#pragma unroll
          for (int w = 0; w < 8; w++) {
            const int kk = g1 - 1 - (w0 + w);
            if (w0 + w < ge && colnz && s <= L - 2) {
              const int t = rla[kk];
              if (t <= L - 2) {
                const double c1 = A1[kk * LP + s], c2 = term2d<MODE>(nn[w], wwv[w], a);
                const double sc = score2d<MODE>(c1, c2);
                const uint64_t key = (uint64_t)t * (uint64_t)L + (uint64_t)s;
                if (better(sc, key, best, bkey)) {
                  best = sc;
                  bkey = key;
                  bt1 = c1;
                  bt2 = c2;
                }
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }
  // ---- 6: argmax over the CTA, then the cluster
  warp_argmax4(best, bkey, bt1, bt2);
  double *ws = reinterpret_cast<double *>(scr);
  uint64_t *wk = reinterpret_cast<uint64_t *>(scr + 256);
  double *w1 = reinterpret_cast<double *>(scr + 512);
  double *w2 = reinterpret_cast<double *>(scr + 768);
  if (lane == 0) {
    ws[warp] = best;
    wk[warp] = bkey;
    w1[warp] = bt1;
    w2[warp] = bt2;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < k2dThreads / 32; w++)
      if (better(ws[w], wk[w], best, bkey)) {
        best = ws[w];
        bkey = wk[w];
        bt1 = w1[w];
        bt2 = w2[w];
      }
    xch->score = best;
    xch->key = bkey;
    xch->t1 = bt1;
    xch->t2 = bt2;
  }
  __syncthreads();
  cluster.sync();
  if (r == 0 && tid == 0) {
    best = -CUDART_INF;
    bkey = kKeyNone;
    for (int c = 0; c < CL; c++) {
      const Xch *x = cluster.map_shared_rank(xch, c);
      const double sc = x->score;
      const uint64_t k = x->key;
      if (better(sc, k, best, bkey)) {
        best = sc;
        bkey = k;
        bt1 = x->t1;
        bt2 = x->t2;
      }
    }
    if (CHECK) any_ovf = 0;
    if (CHECK)
      for (int c = 0; c < CL; c++) any_ovf |= cluster.map_shared_rank(&xch->flags, c)[0];
  }
  cluster_arrive();  // remote reads done: the other CTAs may leave once we all arrive
  if (r == 0 && tid == 0) {
    const bool found = bkey != kKeyNone;
    const int tb = found ? (int)(bkey / (uint64_t)L) : -1;
    const int sb = found ? (int)(bkey % (uint64_t)L) : -1;
    int st = kOK;
    if (CHECK && any_ovf) st = kLevelOverflow;
    else if (!found) st = kNoValidSplit;
    // phi(t*, s*) = H_1 + H_2 + (1 - q) H_1 H_2 from the
    // winning candidate's class terms (A_c = W_c / n_c^q, or S_c at q == 1)
    double phi = CUDART_NAN;
    if (st == kOK && !a.hist_only) {
      if (MODE == SUM) {
        phi = __dadd_rn(bt1, bt2);
      } else {
        const double H1 = __ddiv_rn(__dsub_rn(1.0, bt1), __dsub_rn(a.q, 1.0));
        const double H2 = __ddiv_rn(__dsub_rn(1.0, bt2), __dsub_rn(a.q, 1.0));
        phi = __dadd_rn(__dadd_rn(H1, H2), __dmul_rn(__dmul_rn(__dsub_rn(1.0, a.q), H1), H2));
      }
    }
    const bool ok = st == kOK && !a.hist_only;
    if (a.thresholds) {
      a.thresholds[2 * z] = ok ? tb : -1;
      a.thresholds[2 * z + 1] = ok ? sb : -1;
    }
    if (a.tlab) a.tlab[z] = ok ? tb : -1;
    if (a.objective) a.objective[z] = ok ? phi : CUDART_NAN;
    const int sth = CHECK && any_ovf ? kLevelOverflow : kOK;
    if (a.status) a.status[z] = a.hist_only ? sth : st;
    if (a.status2) a.status2[z] = a.hist_only ? sth : st;
  }
  cluster_wait();  // no CTA leaves while its shared memory may still be read
}

}  // namespace tsa
