// k_stream.cuh -- the "stream" pipeline of tsa_segment for k = 2 at large bin
// counts (the c5 regime: 1024^2 x 1000 u16 slices, 4096 bins): the whole hot
// path in ONE persistent kernel, so the HBM-bound
// stages of some slices run next to the FP64-bound search of others.
//
// Two roles (per 4 consecutive blockIdx: nio io CTAs, the rest search CTAs):
//   io      claims tasks from the io queue, in order; round r holds
//             H(r, c)      c < HC: histogram chunk c of slice r into shared
//                          bins (+ overflow slot), flushed with global atomics
//             L(r-Dl, c)   c < LC: labels of chunk c of slice r-Dl once t* is
//                          known.  The slice was read Dl rounds earlier, so
//                          the label pass mostly re-reads it from L2.
//           and joins the search role when the queue is empty.
//   search  claims slices in order (SS CTAs per slice) and works on them.
// Working on slice z (work_slice, either role):
//   scan    claimed by one CTA once all HC chunks are in: prefix tables
//           (scan_slice, the staged k_scan body) -> sst[z] = done
//   tiles   every warp claims tiles (a-block x 128 second thresholds) from the
//           slice's counter and runs k2_tile (the staged k_search_k2 body);
//           the warp finishing the last tile merges the partials, writes t* and sets mdone[z], and its
//           CTA then recomputes phi(t*) in the definition's order
//           (finalize_slice, the staged k_finalize body).
// An io CTA whose label task finds t* missing works on that slice itself, so
// no wait depends on a CTA that might not be running: the kernel cannot
// deadlock, even when a profiler serialises it or only part of it is resident.
// Every value comes from the staged kernels' own device functions (same
// expression trees and block sizes): results are bit-identical to the staged
// pipeline (tested).
#pragma once
#include <cstdint>

#include "k_finalize.cuh"
#include "k_fused.cuh"  // label16, wait_ge
#include "k_histogram.cuh"
#include "k_search.cuh"
#include "k_tables.cuh"
#include "tsa_device.cuh"

namespace tsa {

constexpr int kStThreads = 256;  // == kTableThreads == kFinThreads
constexpr int kStTileB = 128;    // second-threshold span of a search tile

struct StreamArgs {
  const uint8_t *vol;   // [nz][n] T
  int64_t n, nz;
  int L, k;
  uint32_t *hist;       // [nz][L], zeroed before launch
  int32_t *status;      // [nz] working status (scan / merge / finalize)
  int32_t *thresholds;  // [nz][2]
  uint8_t *labels;      // [nz][n] or null
  double *item_score;   // [nz][NB] per-tile partials
  uint64_t *item_key;
  int NB;               // tiles per slice at most: a-blocks x second-threshold tiles
  double *ps;           // [nz] merged partial (finalize input)
  uint64_t *pk;
  int32_t *ctr;         // zeroed: [0..1] io head (u64), [2] search head,
                        // then per slice (nz each): hcnt, sst, bcur, bdone, mdone, ovf
  ScanArgs scan;        // tables (status, cC.., Asuf, M, rows, luts) as the staged scan
  FinalizeArgs fin;     // objective recomputation (hist, status, ps/pk, nparts = 1)
  int HC, LC, SS, Dl;   // chunks per slice (histogram, labels), search CTAs per slice, label lag
  int nio;              // io CTAs per 4 consecutive blockIdx
  int ltasks;           // 1 = label tasks (labels requested)
};

enum { kHcnt = 0, kSst = 1, kBcur = 2, kBdone = 3, kMdone = 4, kOvf = 5 };
constexpr int kStCounters = 6;  // per-slice counters (+ 3 global)
__device__ __forceinline__ int32_t *st_cnt(const StreamArgs &g, int which, int64_t z) {
  return g.ctr + 3 + which * g.nz + z;
}

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// io task t -> (is_label, z, chunk).  Rounds r: H(r, 0..HC-1) if r < nz, then
// L(r-Dl, 0..LC-1) if ltasks and 0 <= r-Dl < nz.
__device__ __forceinline__ void st_task(const StreamArgs &g, int64_t t, bool &lab, int64_t &z, int &c) {
  const int64_t nz = g.nz;
  if (!g.ltasks) {
    lab = false;
    z = t / g.HC;
    c = (int)(t % g.HC);
    return;
  }
  const int64_t D = min((int64_t)g.Dl, nz);
  const int64_t a = D * g.HC;
  if (t < a) {
    lab = false;
    z = t / g.HC;
    c = (int)(t % g.HC);
    return;
  }
  t -= a;
  const int64_t per = g.HC + g.LC, nb = nz - D;
  if (t < nb * per) {
    const int64_t r = D + t / per;
    const int o = (int)(t % per);
    lab = o >= g.HC;
    z = lab ? r - D : r;
    c = lab ? o - g.HC : o;
    return;
  }
  t -= nb * per;
  lab = true;
  z = nz - D + t / g.LC;
  c = (int)(t % g.LC);
}

// H task: chunk c of slice z -> shared bins [L] + overflow slot [L] -> global atomics
template <typename T>
__device__ void st_hist(const StreamArgs &g, const int64_t z, const int c, uint32_t *sh) {
  const int L = g.L;
  const uint32_t UL = (uint32_t)L;
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sh);
  constexpr int VEC = 16 / sizeof(T);
  const int64_t nvec = g.n / VEC;
  const int64_t per = (nvec + g.HC - 1) / g.HC;
  const int64_t v0 = per * c, v1 = min(nvec, v0 + per);
  const uint4 *v4 = reinterpret_cast<const uint4 *>(g.vol) + z * nvec;
  constexpr int U = 4;  // 64 bytes in flight per thread
  for (int64_t i0 = v0 + threadIdx.x; i0 < v1; i0 += (int64_t)U * blockDim.x) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      if (i < v1) w[u] = __ldg(v4 + i);  // default policy: stays in L2 for the label pass
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (i0 + (int64_t)u * blockDim.x >= v1) break;
      const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
      for (int e = 0; e < 4; e++) {
        if (sizeof(T) == 2) {
          red_inc(base, ws[e] & 0xffffu, UL);
          red_inc(base, ws[e] >> 16, UL);
        } else {
          red_inc(base, ws[e] & 0xffu, UL);
          red_inc(base, (ws[e] >> 8) & 0xffu, UL);
          red_inc(base, (ws[e] >> 16) & 0xffu, UL);
          red_inc(base, ws[e] >> 24, UL);
        }
      }
    }
  }
  __syncthreads();
  uint32_t *out = g.hist + z * L;
  for (int b = threadIdx.x; b < L; b += blockDim.x) {
    const uint32_t cnt = sh[b];
    if (cnt) atomicAdd(out + b, cnt);
  }
  if (threadIdx.x == 0 && sh[L]) atomicOr(st_cnt(g, kOvf, z), 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(st_cnt(g, kHcnt, z), 1);
  }
}

// The slice's tables, by the CTA that claimed the scan: histogram through L2
// into shared memory, histogram status, scan_slice (exactly k_scan's body).
template <int MODE>
__device__ void st_scan(const StreamArgs &g, const int64_t z, uint32_t *sh, double *wsh) {
  const int L = g.L;
  const uint32_t *h = g.hist + z * L;
  for (int b = threadIdx.x; b < L; b += blockDim.x) sh[b] = __ldcg(h + b);
  if (threadIdx.x == 0) g.status[z] = __ldcg(st_cnt(g, kOvf, z)) ? kLevelOverflow : kOK;
  __syncthreads();
  scan_slice<MODE>(g.scan, z, sh, wsh);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(st_cnt(g, kSst, z), 2);
  }
}

// Work on slice z until none of its jobs is left to claim: the scan (once all
// histogram chunks are in), then a-blocks.  If one of this CTA's warps
// completes the slice, the CTA recomputes phi(t*).  Returns when the slice
// has no unclaimed work (other warps may still be finishing a-blocks).
template <int MODE, int DEG>
__device__ void work_slice(const StreamArgs &g, const int64_t z, double *smem) {
  __shared__ int s_job, s_M, s_st, s_done;
  __shared__ double s_p2[32];
  double2 *s_jr = reinterpret_cast<double2 *>(smem);
  const int lane = threadIdx.x & 31;
  bool jr_ok = false;  // the class-size table is staged in smem (CTA-uniform)
  for (;;) {
    __syncthreads();  // every thread has read the previous s_job / s_M / s_st (racecheck)
    // 0 = finished, 1 = scan claimed, 2 = search, 3 = wait
    if (threadIdx.x == 0) {
      int job = 3;
      if (ld_acquire(st_cnt(g, kMdone, z))) {
        job = 0;
      } else {
        const int sst = ld_acquire(st_cnt(g, kSst, z));
        if (sst == 2) {
          job = 2;
        } else if (sst == 0 && ld_acquire(st_cnt(g, kHcnt, z)) == g.HC &&
                   atomicCAS(st_cnt(g, kSst, z), 0, 1) == 0) {
          __threadfence();
          job = 1;
        }
      }
      if (job == 2) {
        s_M = __ldcg(g.scan.M + z);
        s_st = __ldcg(g.status + z);
      }
      if (job == 3) __nanosleep(256);
      s_job = job;
      s_done = 0;
    }
    __syncthreads();
    const int job = s_job;
    if (job == 0) return;
    if (job == 3) continue;
    if (job == 1) {
      st_scan<MODE>(g, z, reinterpret_cast<uint32_t *>(smem), smem + ((g.L + 2) / 2 + 1));
      jr_ok = false;
      continue;
    }
    // search: stage the class-size table, then claim a-blocks
    if (!jr_ok) {
      for (int i = threadIdx.x; i < kSN; i += blockDim.x)
        s_jr[i] = make_double2(g.scan.luts.sp[i], g.scan.luts.sp[kSN + i]);
      if (threadIdx.x < 32) s_p2[threadIdx.x] = g.scan.luts.p2[threadIdx.x];
      __syncthreads();
      jr_ok = true;
    }
    const int M = s_M, st = s_st;
    // 2-D tiles: a-block i (32 first thresholds) x kStTileB second thresholds,
    // so no single item is long (a whole a-block is ~M tuples per lane)
    const int nb = (st == kOK && M >= 3) ? (M - 3) / 32 + 1 : 0;
    const int nbt = M >= 3 ? (M - 2) / kStTileB + 1 : 1;
    const int nbe = max(nb * nbt, 1);
    const SpPair tab{s_jr, s_p2};
    const Luts &l = g.scan.luts;
    for (;;) {
      int c = 0;
      if (lane == 0) c = atomicAdd(st_cnt(g, kBcur, z), 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nbe) break;
      double best = -CUDART_INF;
      uint64_t bestkey = kKeyNone;
      if (nb > 0) {
        const int i = c / nbt, blo = (c % nbt) * kStTileB;
        if (blo + kStTileB - 1 >= 32 * i + 1) {
          k2_tile<MODE, DEG>(g.scan.rows + z * g.scan.RE, M, i, blo, blo + kStTileB - 1, lane, l, tab, best,
                             bestkey);
          warp_argmax(best, bestkey);
        }
      }
      int last = 0;
      if (lane == 0) {
        g.item_score[z * g.NB + c] = best;
        g.item_key[z * g.NB + c] = bestkey;
        __threadfence();
        last = atomicAdd(st_cnt(g, kBdone, z), 1) == nbe - 1;
        if (last) __threadfence();
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (!last) continue;
      // the slice's last a-block: merge its partials under (score desc, key asc)
      double s = -CUDART_INF;
      uint64_t key = kKeyNone;
      for (int i = lane; i < nbe; i += 32) {
        const double os = __ldcg(g.item_score + z * g.NB + i);
        const uint64_t ok = __ldcg(g.item_key + z * g.NB + i);
        if (better(os, ok, s, key)) {
          s = os;
          key = ok;
        }
      }
      warp_argmax(s, key);
      if (lane == 0) {
        g.ps[z] = s;
        g.pk[z] = key;
        int sz = st;
        if (sz == kOK && key == kKeyNone) sz = kNoValidSplit;
        const bool ok = sz == kOK;
        g.thresholds[2 * z] = ok ? (int)((key >> 12) & 0xFFFull) : -1;
        g.thresholds[2 * z + 1] = ok ? (int)(key & 0xFFFull) : -1;
        g.status[z] = sz;
        if (g.fin.status_out2) g.fin.status_out2[z] = sz;
        __threadfence();
        atomicExch(st_cnt(g, kMdone, z), 1);
        s_done = 1;
      }
    }
    __syncthreads();
    if (s_done && g.fin.objective_out) finalize_slice(g.fin, z, smem);
    __syncthreads();
    return;
  }
}

// L task: labels of chunk c of slice z; works on the slice itself while t* is missing.
template <typename T, int MODE, int DEG>
__device__ void st_label(const StreamArgs &g, const int64_t z, const int c, double *smem) {
  work_slice<MODE, DEG>(g, z, smem);
  if (threadIdx.x == 0) wait_ge(st_cnt(g, kMdone, z), 1);
  __syncthreads();
  const int64_t groups = g.n / 16;
  const int64_t per = (groups + g.LC - 1) / g.LC;
  const int64_t i0 = z * groups + per * c;
  const int64_t i1 = z * groups + min(groups, per * (c + 1));
  const uint4 *src = reinterpret_cast<const uint4 *>(g.vol);
  uint4 *dst = reinterpret_cast<uint4 *>(g.labels);
  const bool ok = __ldcg(g.status + z) == kOK;
  const int t0 = __ldcg(g.thresholds + 2 * z), t1 = __ldcg(g.thresholds + 2 * z + 1);
  const uint32_t b0 = (uint32_t)(t0 & 0xff) * 0x01010101u, b1 = (uint32_t)(t1 & 0xff) * 0x01010101u;
  constexpr int U = 4;
  for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += (int64_t)U * blockDim.x) {
    uint4 o[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = ib + (int64_t)u * blockDim.x;
      if (i < i1) o[u] = label16<T>(src, i, ok, t0, t1, b0, b1);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = ib + (int64_t)u * blockDim.x;
      if (i < i1) __stcs(dst + i, o[u]);
    }
  }
}

template <typename T, int MODE, int DEG>
__global__ void __launch_bounds__(kStThreads, 4) k_stream(StreamArgs g) {
  // one shared buffer for every job: H [L+1] u32 bins; scan [L] u32 + [L]
  // doubles + 1 KB; finalize [L] doubles + [L] ints; search [kSN] double2
  extern __shared__ __align__(16) double st_smem[];
  __shared__ int64_t s_t;
  const bool io = (int)(blockIdx.x & 3) < g.nio;
  if (io) {
    const int64_t ntasks = g.nz * (int64_t)(g.HC + (g.ltasks ? g.LC : 0));
    for (;;) {
      __syncthreads();  // shared memory of the previous task is free
      if (threadIdx.x == 0) s_t = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(g.ctr), 1ull);
      __syncthreads();
      const int64_t t = s_t;
      if (t >= ntasks) break;
      bool lab;
      int64_t z;
      int c;
      st_task(g, t, lab, z, c);
      if (lab) st_label<T, MODE, DEG>(g, z, c, st_smem);
      else st_hist<T>(g, z, c, reinterpret_cast<uint32_t *>(st_smem));
    }
  }
  // search role (and io CTAs once their queue is empty): slices in order
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = atomicAdd(g.ctr + 2, 1);
    __syncthreads();
    const int64_t z = s_t / g.SS;
    if (z >= g.nz) break;
    work_slice<MODE, DEG>(g, z, st_smem);
  }
}

}  // namespace tsa
