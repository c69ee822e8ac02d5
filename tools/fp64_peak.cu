// tools/fp64_peak.cu -- FP64 pipe peak micro-benchmark.
// MEASURED_PEAKS.json has no FP64 figure, so the search kernel's roofline
// denominator is measured here: independent DFMA / DMUL chains on every SM,
// CUDA-event timed, printed as one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>
#include <cstdio>

template <bool FMA>
__global__ void __launch_bounds__(256) k_fp64(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = FMA ? fma(x[j], a, b) : x[j] * a;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += x[j];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best_fma = 0, best_mul = 0;
  for (int rep = 0; rep < 6; rep++) {
    for (int f = 0; f < 2; f++) {
      cudaEventRecord(e0);
      if (f == 0)
        k_fp64<true><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
      else
        k_fp64<false><<<blocks, threads>>>(out, iters, 0.999999, 0.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;  // instructions (lane-ops)
      const double rate = ops / (ms * 1e-3);
      if (f == 0) best_fma = rate > best_fma ? rate : best_fma;
      else best_mul = rate > best_mul ? rate : best_mul;
    }
  }
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_lane_ops_per_s\": %.4e, \"dfma_tflops\": %.3f, "
         "\"dmul_lane_ops_per_s\": %.4e, \"fp64_lanes_per_sm_per_clk_at_attr_clock\": %.2f}\n",
         sms, clk / 1e3, best_fma, 2 * best_fma / 1e12, best_mul, best_fma / sms / (clk * 1e3));
  return 0;
}
