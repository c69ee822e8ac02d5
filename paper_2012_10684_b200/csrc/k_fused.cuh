// k_fused.cuh -- the whole hot path as ONE
// persistent kernel for k <= 2, bins <= 1024, canonical enumeration (the c1/c2
// workloads).  Separate kernels leave the GPU idle between phases: the
// histogram is bound by shared-memory atomics, the per-slice search/finalize
// by latency, the labelling by HBM.  Here they overlap.
//
// Task queue (claimed in order with one global atomic; every dependency points
// to an earlier queue position, so a CTA waiting on one waits on a task some
// running CTA already holds -- no deadlock):
//   LUT tasks                               1/n^q table chunks
//   round r = 0 .. nslab + DL - 1:
//     H(r)       slab r: (slice, chunk) histogram partials (no atomics to HBM)
//     M(r - 1)   slab r-1: per slice, sum partials -> histogram, prefix tables,
//                exhaustive search, argmax, phi(t*) in the definition's order
//     L(r - DL)  slab r-DL: (slice, chunk) labels, DL rounds behind so M is
//                done; the slab's voxels are still in L2 (126 MB), so the
//                label pass re-reads them from L2, not HBM.
// Completion counters (hdone[z], mdone[z], lutdone) use release/acquire
// (__threadfence + atomic / volatile poll + __threadfence).
#pragma once
#include <cstdint>

#include "k_histogram.cuh"
#include "k_label.cuh"
#include "k_search.cuh"
#include "k_tables.cuh"
#include "tsa_device.cuh"

namespace tsa {

#ifdef TSA_TRACE
// debug builds only (tools/fused_trace.py): per-task (type, z, smid, t0, t1)
__device__ unsigned long long g_trace[5 * 65536];
__device__ int g_trace_n;
#endif
// TSA_MPHASE / g_mphase / gtimer: tsa_device.cuh

struct FusedArgs {
  const uint8_t *vol;
  int dtype_bytes;
  int64_t n;  // voxels per slice
  int64_t nz;
  int L, k;
  double q;
  int mode;
  // outputs
  int32_t *thresholds;  // [nz][k]
  double *objective;    // [nz] or null
  uint32_t *hist;       // [nz][L]
  int32_t *status;      // [nz]
  int32_t *status2;     // [nz] or null (user copy)
  uint8_t *labels;      // [nz][n] or null
  // workspace
  uint32_t *partial;    // [nz][HC][L]
  int32_t *povf;        // [nz][HC]
  double *sp;           // [kSmallLut] small table of Luts (k_small_luts layout)
  int32_t *counters;    // [0] head, [1] lutdone, [2 .. 2+nz) hdone, [2+nz .. 2+2nz) mdone
  Luts luts;
  // schedule
  int HC, LC, SB, DM, DL, nslab, nlut;
  int64_t lut_per;
};

__device__ __forceinline__ void wait_ge(const int32_t *p, int target) {
  if (*((volatile const int32_t *)p) >= target) {
    __threadfence();
    return;
  }
  unsigned ns = 32;
  while (*((volatile const int32_t *)p) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns *= 2;
  }
  __threadfence();
}

__device__ __forceinline__ void signal_add(int32_t *p, int v) {
  __threadfence();
  atomicAdd(p, v);
}

// ---------------------------------------------------------------- H task
template <typename T>
__device__ void fused_hist(const FusedArgs &g, int z, int c, uint32_t *sh) {
  const int L = g.L;
  const int warps = blockDim.x >> 5;
  for (int i = threadIdx.x; i < L * warps; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t *bins = sh + (threadIdx.x >> 5) * L;
  const T *slice = reinterpret_cast<const T *>(g.vol) + (size_t)z * g.n;
  constexpr int VEC = 16 / sizeof(T);
  const int64_t nvec = g.n / VEC;
  const int64_t per = (nvec + g.HC - 1) / g.HC;
  const int64_t v0 = per * c, v1 = min(nvec, v0 + per);
  const uint4 *v4 = reinterpret_cast<const uint4 *>(slice);
  int ovf = 0;
  const bool nocheck = sizeof(T) == 1 && L == 256;
  constexpr int U = 4;  // 4 x 16-byte loads in flight per thread
  for (int64_t i0 = v0 + threadIdx.x; i0 < v1; i0 += (int64_t)U * blockDim.x) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      w[u] = i < v1 ? __ldg(v4 + i) : make_uint4(0u, 0u, 0u, 0u);  // default policy: stays in L2
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (i0 + (int64_t)u * blockDim.x >= v1) break;
      if (nocheck) {
        hist_word<T, false>(bins, w[u].x, L, ovf);
        hist_word<T, false>(bins, w[u].y, L, ovf);
        hist_word<T, false>(bins, w[u].z, L, ovf);
        hist_word<T, false>(bins, w[u].w, L, ovf);
      } else {
        hist_word<T, true>(bins, w[u].x, L, ovf);
        hist_word<T, true>(bins, w[u].y, L, ovf);
        hist_word<T, true>(bins, w[u].z, L, ovf);
        hist_word<T, true>(bins, w[u].w, L, ovf);
      }
    }
  }
  __shared__ int s_ovf;
  if (threadIdx.x == 0) s_ovf = 0;
  __syncthreads();
  if (ovf) s_ovf = kLevelOverflow;
  uint32_t *out = g.partial + ((size_t)z * g.HC + c) * L;
  for (int b = threadIdx.x; b < L; b += blockDim.x) {
    uint32_t s = 0;
    for (int r = 0; r < warps; r++) s += sh[r * L + b];
    out[b] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    g.povf[(size_t)z * g.HC + c] = s_ovf;
    if (g.counters) signal_add(g.counters + 2 + z, 1);
  }
}

// ---------------------------------------------------------------- L task
template <typename T>
__device__ __forceinline__ uint4 label16(const uint4 *src, int64_t i, bool ok, int t0, int t1,
                                         uint32_t b0, uint32_t b1) {
  if (sizeof(T) == 1) {
    const uint4 w = __ldcs(src + i);
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (ok) {
      o.x = (__vcmpgtu4(w.x, b0) & 0x01010101u) + (__vcmpgtu4(w.x, b1) & 0x01010101u);
      o.y = (__vcmpgtu4(w.y, b0) & 0x01010101u) + (__vcmpgtu4(w.y, b1) & 0x01010101u);
      o.z = (__vcmpgtu4(w.z, b0) & 0x01010101u) + (__vcmpgtu4(w.z, b1) & 0x01010101u);
      o.w = (__vcmpgtu4(w.w, b0) & 0x01010101u) + (__vcmpgtu4(w.w, b1) & 0x01010101u);
    }
    return o;
  } else {
    const uint4 wa = __ldcs(src + 2 * i), wb = __ldcs(src + 2 * i + 1);
    const uint32_t ws[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    if (ok) {
#pragma unroll
      for (int e = 0; e < 16; e++) {
        const int v = (int)((ws[e >> 1] >> (16 * (e & 1))) & 0xffffu);
        o[e >> 2] |= ((uint32_t)(v > t0) + (uint32_t)(v > t1)) << (8 * (e & 3));
      }
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
}

template <typename T>
__device__ void fused_label(const FusedArgs &g, int z, int c) {
  const int64_t groups = g.n / 16;
  const int64_t per = (groups + g.LC - 1) / g.LC;
  const int64_t i0 = (int64_t)z * groups + per * c;
  const int64_t i1 = (int64_t)z * groups + min(groups, per * (c + 1));
  const uint4 *src = reinterpret_cast<const uint4 *>(g.vol);
  uint4 *dst = reinterpret_cast<uint4 *>(g.labels);
  // touch this thread's first input vectors before waiting (the volume does
  // not depend on the search): the wait then overlaps the L2 latency
  for (int64_t i = i0 + threadIdx.x; i < i1; i += 4 * (int64_t)blockDim.x) {
    if (sizeof(T) == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(src + i));
    else asm volatile("prefetch.global.L1 [%0];" ::"l"(src + 2 * i));
  }
  if (threadIdx.x == 0) wait_ge(g.counters + 2 + g.nz + z, 1);
  __syncthreads();
  // data written by another CTA in this launch: read through L2 (__ldcg)
  const bool ok = __ldcg(g.status + z) == kOK;
  const int tmax = sizeof(T) == 1 ? 255 : 65535;
  const int32_t *tz = g.thresholds + z * g.k;
  const int t0 = __ldcg(tz), t1 = g.k > 1 ? __ldcg(tz + 1) : tmax;
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

// ---------------------------------------------------------------- M task
// One CTA per slice: histogram from partials, prefix tables (canonical), the
// exhaustive search for k <= 2, argmax, phi(t*) in the definition's order.
template <int K, int MODE>
__device__ void fused_mid(const FusedArgs &g, int z, char *smem) {
  const int L = g.L, E = L + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  uint32_t *hs = reinterpret_cast<uint32_t *>(smem);            // [L]
  double *wsh = reinterpret_cast<double *>(hs + ((L + 1) & ~1)); // [L]
  double *tWhi = wsh + L;                                       // [E]
  double *tWlo = tWhi + E;                                      // [E]
  double *Asuf = tWlo + E;                                      // [L]
  double *fsh = Asuf + L;                                       // [L]
  uint32_t *tC = reinterpret_cast<uint32_t *>(fsh + L);         // [E]
  int32_t *tBin = reinterpret_cast<int32_t *>(tC + E);          // [E]
  __shared__ int s_status, s_M;
  __shared__ double s_red[32], s_P[kKMax + 1], s_S[kKMax + 1];
  __shared__ uint64_t s_key[32];
  __shared__ __align__(16) double s_scan[128];  // build_tables scratch: 1 KB
  __shared__ double s_p2[32];  // Luts::p2 for the class terms (synchronised below)
  stage_p2(g.luts, s_p2);
  TSA_MPHASE(z, 0)
  if (tid == 0 && g.counters) {
    wait_ge(g.counters + 1, g.nlut);
    wait_ge(g.counters + 2 + z, g.HC);
  }
  __syncthreads();
  TSA_MPHASE(z, 1)
  // histogram = sum of chunk partials; overflow flag
  int ovf = 0;
  // only LEVEL_OVERFLOW counts (the HU path passes its slice status here,
  // which may hold NO_VALID_SPLIT from an earlier finish on the same workspace)
  for (int c = tid; c < g.HC; c += blockDim.x) ovf |= __ldcg(g.povf + (size_t)z * g.HC + c) == kLevelOverflow;
  if (tid == 0) s_status = 0;
  __syncthreads();
  if (ovf) s_status = kLevelOverflow;
  for (int i = tid; i < L; i += blockDim.x) {
    uint32_t s = 0;
    for (int c = 0; c < g.HC; c++) s += __ldcg(g.partial + ((size_t)z * g.HC + c) * L + i);
    hs[i] = s;
    g.hist[(size_t)z * L + i] = s;
  }
  __syncthreads();
  TSA_MPHASE(z, 2)
  // prefix tables (the same block-wide construction as k_scan: bit-identical)
  {
    int m;
    uint32_t ntot;
    build_tables(hs, L, g.q, g.luts.shannon, wsh, tC, tWhi, tWlo, tBin,
                 reinterpret_cast<char *>(s_scan), m, ntot);
    if (tid == 0) {
      s_M = m;
      if (s_status == kOK && m < K + 1) s_status = kNoValidSplit;
    }
    __syncthreads();
  }
  TSA_MPHASE(z, 3)
  const int M = s_M;
  int st = s_status;
  const SliceTables t{tC, tWhi, tWlo, Asuf};
  double best = -CUDART_INF;
  uint64_t key = kKeyNone;
  if (st == kOK) {
    // Asuf[i] = T(i+1, M-1) and Apre[i] = T(0, i) (in fsh, free until the finalize
    // step) in one pass so their gathers overlap
    for (int i = tid; i <= M - 2; i += blockDim.x) {
      const double as = class_term<MODE>(t, g.luts, i + 1, M - 1, s_p2);
      const double ap = K == 2 ? class_term<MODE>(t, g.luts, 0, i, s_p2) : 0.0;
      Asuf[i] = as;
      if (K == 2) fsh[i] = ap;
    }
    __syncthreads();
    TSA_MPHASE(z, 4)
    // exhaustive search over all C(M-1, K) tuples, row chunks over the CTA
    search_rows_k12<K, MODE, 16>(t, fsh, g.luts, tBin, M, 0, k12_chunks<K, 16>(M), tid, blockDim.x, best, key,
                                 s_p2);
    __syncthreads();  // fsh is reused below
  }
  warp_argmax(best, key);
  if (lane == 0) {
    s_red[warp] = best;
    s_key[warp] = key;
  }
  __syncthreads();
  if (warp == 0) {
    best = lane < nw ? s_red[lane] : -CUDART_INF;
    key = lane < nw ? s_key[lane] : kKeyNone;
    warp_argmax(best, key);
    if (lane == 0) {
      if (st == kOK && key == kKeyNone) st = kNoValidSplit;
      s_status = st;
      s_key[0] = key;
    }
  }
  __syncthreads();
  TSA_MPHASE(z, 5)
  st = s_status;
  key = s_key[0];
  int32_t *thr = g.thresholds + (size_t)z * g.k;
  const int t0 = (int)((key >> (12 * (K - 1))) & 0xFFFull);
  const int t1 = K > 1 ? (int)(key & 0xFFFull) : L;
  if (st != kOK) {
    if (tid < g.k) thr[tid] = -1;
    if (tid == 0) {
      if (g.objective) g.objective[z] = CUDART_NAN;
      g.status[z] = st;
      if (g.status2) g.status2[z] = st;
    }
  } else {
    if (tid < K) thr[tid] = tid == 0 ? t0 : t1;
    if (tid == 0) {
      g.status[z] = kOK;
      if (g.status2) g.status2[z] = kOK;
    }
  }
  __syncthreads();
  TSA_MPHASE(z, 6)
  // t* and the status release the slice's labelling now; phi(t*) (only the
  // host reads it) is computed after the signal, off the labels' critical path
  if (tid == 0 && g.counters) signal_add(g.counters + 2 + g.nz + z, 1);
  if (st == kOK) {
    // phi(t*) in the definition's order (k_finalize): p over the canonical list
    if (g.objective) {
      // N = total count (the last prefix count; exact)
      const double N = (double)tC[M];
      for (int j = tid; j < M; j += blockDim.x) fsh[j] = __ddiv_rn((double)(tC[j + 1] - tC[j]), N);
      __syncthreads();
      // class c = canonical-list range [cs, ce): boundaries by binary search
      auto first_above = [&](int tv) {  // smallest j in [0, M] with j == M or bin_j > tv
        int lo = 0, hi = M;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (tBin[mid + 1] > tv) hi = mid;
          else lo = mid + 1;
        }
        return lo;
      };
      int cs = 0, ce = M;
      if (tid <= K) {
        cs = tid == 0 ? 0 : first_above(tid == 1 ? t0 : t1);
        ce = tid == K ? M : first_above(tid == 0 ? t0 : t1);
      }
      // sequential sums in ascending bin order (the definition's order),
      // loads batched four at a time
      auto seq_sum = [&](bool sub) {
        double acc = 0.0;
        int j = cs;
        for (; j + 4 <= ce; j += 4) {
          const double x0 = fsh[j], x1 = fsh[j + 1], x2 = fsh[j + 2], x3 = fsh[j + 3];
          if (sub) {
            acc = __dsub_rn(acc, x0);
            acc = __dsub_rn(acc, x1);
            acc = __dsub_rn(acc, x2);
            acc = __dsub_rn(acc, x3);
          } else {
            acc = __dadd_rn(acc, x0);
            acc = __dadd_rn(acc, x1);
            acc = __dadd_rn(acc, x2);
            acc = __dadd_rn(acc, x3);
          }
        }
        for (; j < ce; j++) acc = sub ? __dsub_rn(acc, fsh[j]) : __dadd_rn(acc, fsh[j]);
        return acc;
      };
      if (tid <= K) s_P[tid] = seq_sum(false);
      __syncthreads();
      const bool shannon = g.luts.shannon;
      for (int j = tid; j < M; j += blockDim.x) {
        const int cls = (tBin[j + 1] > t0) + (K > 1 && tBin[j + 1] > t1);
        const double r = __ddiv_rn(fsh[j], s_P[cls]);
        fsh[j] = shannon ? __dmul_rn(r, log(r)) : pow(r, g.q);
      }
      __syncthreads();
      if (tid <= K) {
        const double A = seq_sum(shannon);
        s_S[tid] = shannon ? A : __ddiv_rn(__dsub_rn(1.0, A), __dsub_rn(g.q, 1.0));
      }
      __syncthreads();
      if (tid == 0) {
        double phi = s_S[0];
        for (int j = 1; j <= K; j++)
          phi = __dadd_rn(__dadd_rn(phi, s_S[j]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, g.q), phi), s_S[j]));
        g.objective[z] = phi;
      }
    }
  }
}

// Task index -> (type, slice, chunk).  Queue: LUT tasks, then rounds r:
// H(slab r), M(slab r - DM), L(slab r - DL) (empty parts are skipped, so the
// queue has no no-op tasks).  Returns 0 LUT, 1 H, 2 M, 3 L, -1 past the end.
__device__ __forceinline__ int decode_task(const FusedArgs &g, int64_t t, int &z, int &c) {
  if (t < g.nlut) {
    z = (int)t;
    return 0;
  }
  t -= g.nlut;
  const int nH = g.SB * g.HC, nM = g.SB, nL = g.SB * g.LC;
  for (int r = 0; r < g.nslab + g.DL; r++) {
    const int h = r < g.nslab ? nH : 0;
    const int m = (r - g.DM >= 0 && r - g.DM < g.nslab) ? nM : 0;
    const int l = (r - g.DL >= 0 && r - g.DL < g.nslab) ? nL : 0;
    if (t < h) {
      z = r * g.SB + (int)(t / g.HC);
      c = (int)(t % g.HC);
      return 1;
    }
    t -= h;
    if (t < m) {
      z = (r - g.DM) * g.SB + (int)t;
      c = 0;
      return 2;
    }
    t -= m;
    if (t < l) {
      z = (r - g.DL) * g.SB + (int)(t / g.LC);
      c = (int)(t % g.LC);
      return 3;
    }
    t -= l;
  }
  return -1;
}

template <typename T, int K, int MODE>
__global__ void __launch_bounds__(512, 2) k_fused(FusedArgs g) {
  extern __shared__ __align__(16) char fsm[];
  __shared__ int s_type, s_z, s_c;
  for (;;) {
    if (threadIdx.x == 0) {
      const int task = atomicAdd(g.counters, 1);
      int z = 0, c = 0;
      s_type = decode_task(g, task, z, c);
      s_z = z;
      s_c = c;
    }
    __syncthreads();
    const int type = s_type, z = s_z, c = s_c;
    __syncthreads();
    if (type < 0) break;
#ifdef TSA_TRACE
    unsigned long long tr0 = 0;
    if (threadIdx.x == 0) tr0 = gtimer();
    const int tr_type = type, tr_z = z;
#endif
    if (type == 0) {
      const int64_t a = (int64_t)z * g.lut_per, b = min((int64_t)kSmallLut, a + g.lut_per);
      for (int64_t e = a + threadIdx.x; e < b; e += blockDim.x) g.sp[e] = small_lut_entry((int)e, g.q, g.luts.shannon);
      __syncthreads();
      if (threadIdx.x == 0) signal_add(g.counters + 1, 1);
    } else if (z < g.nz) {
      if (type == 1) fused_hist<T>(g, z, c, reinterpret_cast<uint32_t *>(fsm));
      else if (type == 2) fused_mid<K, MODE>(g, z, fsm);
      else if (g.labels) fused_label<T>(g, z, c);
    }
#ifdef TSA_TRACE
    if (threadIdx.x == 0) {
      const int slot = atomicAdd(&g_trace_n, 1);
      if (slot < 65536) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[5 * slot + 0] = tr_type;
        g_trace[5 * slot + 1] = (unsigned long long)tr_z;
        g_trace[5 * slot + 2] = smid;
        g_trace[5 * slot + 3] = tr0;
        g_trace[5 * slot + 4] = gtimer();
      }
    }
#endif
  }
}

// ---------------------------------------------------------------------------
// Compact path (default for the same eligible problems): the fused kernel's
// task bodies as three kernels chained with Programmatic Dependent Launch.
// Each kernel lets its dependent launch as soon as all its CTAs are running
// (griddepcontrol.launch_dependents), and dependents wait per slice on the
// release/acquire counters instead of on whole-grid completion, so the
// latency-bound per-slice search overlaps the atomics-bound histogram and the
// HBM-bound labelling of other slices.  (A dependent grid only launches once
// every CTA of its primary has started, so spinning dependents can never
// starve the CTAs they wait for.)
//   k_lut_part    the small class-term table (Luts::sp); signals lutdone
//   k_hist_part   persistent, slice-ordered (slice, chunk) histogram partials;
//                 signals hdone[z]
//   k_mid         one CTA per slice: waits lutdone, hdone[z]; tables, search,
//                 argmax, phi(t*); signals mdone[z]
//   k_label_part  (chunk, slice): waits mdone[z]; labels
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Last statement of every PDL-launched kernel of the chain: an early-triggering
// primary's dependents must execute griddepcontrol.wait (PTX ISA), and with it
// a grid completes only after its primary has, so later stream work (a D2H
// of the objective, the next captured node) is ordered after the whole chain.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifdef TSA_TRACE
__device__ __forceinline__ void trace_rec(int type, int z, unsigned long long t0) {
  if (threadIdx.x != 0) return;
  const int slot = atomicAdd(&g_trace_n, 1);
  if (slot < 65536) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[5 * slot + 0] = type;
    g_trace[5 * slot + 1] = (unsigned long long)z;
    g_trace[5 * slot + 2] = smid;
    g_trace[5 * slot + 3] = t0;
    g_trace[5 * slot + 4] = gtimer();
  }
}
#define TRACE_T0 const unsigned long long _t0 = gtimer();
#define TRACE_END(type, z) trace_rec(type, z, _t0);
#else
#define TRACE_T0
#define TRACE_END(type, z)
#endif

template <typename T>
__global__ void __launch_bounds__(512) k_hist_part(FusedArgs g) {
  extern __shared__ __align__(16) char fsm[];
  TRACE_T0
  pdl_trigger();  // one wave: the per-slice kernel can launch right away
  const int64_t G = gridDim.x;
  // persistent over (slice, chunk) items in slice order, so early slices
  // complete first and their per-slice work can start while later slices are
  // still being counted
  const int64_t items = g.nz * (int64_t)g.HC;
  for (int64_t it = blockIdx.x; it < items; it += G) {
    __syncthreads();  // shared bins of the previous item are flushed
    fused_hist<T>(g, (int)(it / g.HC), (int)(it % g.HC), reinterpret_cast<uint32_t *>(fsm));
  }
  TRACE_END(1, blockIdx.x)
  pdl_wait();
}

// The small class-term table (Luts::sp, 33 KB), PDL primary of k_hist_part;
// every CTA signals the LUT counter that k_mid waits on.
__global__ void __launch_bounds__(256) k_lut_part(FusedArgs g) {
  pdl_trigger();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kSmallLut; e += gridDim.x * blockDim.x)
    g.sp[e] = small_lut_entry(e, g.q, g.luts.shannon);
  __syncthreads();
  if (threadIdx.x == 0 && g.counters) signal_add(g.counters + 1, 1);
}

// per-slice kernel of the compact path: 256 threads, 3 CTAs per SM (measured
// on c2: 256 -> 70.9 us/step, 512 -> 89.2, 1024 -> 102.7; more threads per
// slice cost more co-residency with the histogram / label CTAs than they save)
constexpr int kMidThreads = 256;

template <int K, int MODE>
__global__ void __launch_bounds__(kMidThreads, 3) k_mid(FusedArgs g) {
  extern __shared__ __align__(16) char fsm[];
  TRACE_T0
  pdl_trigger();
  fused_mid<K, MODE>(g, blockIdx.x, fsm);
  TRACE_END(2, blockIdx.x)
  pdl_wait();
}

template <typename T>
__global__ void __launch_bounds__(256) k_label_part(FusedArgs g) {
  TRACE_T0
  fused_label<T>(g, blockIdx.y, blockIdx.x);
  TRACE_END(3, blockIdx.y)
  pdl_wait();
}

}  // namespace tsa
