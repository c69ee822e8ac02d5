// k_scan_seed.cuh -- the pruned k = 2 search's prologue in one kernel: per
// slice CTA, the prefix tables (k_scan's body) and then
// the seed score and bound records (k_k2_seed's body), the
// slice's packed rows staged in the dynamic shared memory the scan used.
// One launch and one latency chain per slice instead of two (each ~2 waves
// of 1000 CTAs on c5).
#pragma once
#include "k_search.cuh"
#include "k_tables.cuh"

namespace tsa {

template <int DEG>
__global__ void __launch_bounds__(kTableThreads) k_scan_seed(ScanArgs g, SearchArgs sa, int smem_bytes) {
  extern __shared__ __align__(16) double wsh[];
  TSA_MPHASE(blockIdx.x, 0)
  uint32_t *hs = reinterpret_cast<uint32_t *>(wsh + g.L + 128);
  const uint4 *h4 = reinterpret_cast<const uint4 *>(g.hist + (int64_t)blockIdx.x * g.L);
  if ((g.L & 3) == 0 && (reinterpret_cast<uintptr_t>(g.hist) & 15) == 0)
    for (int i = threadIdx.x; i < g.L / 4; i += blockDim.x) reinterpret_cast<uint4 *>(hs)[i] = __ldg(h4 + i);
  else
    for (int i = threadIdx.x; i < g.L; i += blockDim.x) hs[i] = g.hist[(int64_t)blockIdx.x * g.L + i];
  __syncthreads();
  TSA_MPHASE(blockIdx.x, 1)
  scan_slice<PROD_MAX>(g, blockIdx.x, hs, wsh);
  __syncthreads();  // the slice's rows / M / status are written (global, this CTA)
  TSA_MPHASE(blockIdx.x, 2)
  k2_seed_body<PROD_MAX, DEG>(sa, blockIdx.x, reinterpret_cast<K2Row *>(wsh), smem_bytes / (int)sizeof(K2Row));
  TSA_MPHASE(blockIdx.x, 7)
}

}  // namespace tsa
