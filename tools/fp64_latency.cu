// FP64 dependent-chain latency on one warp (cycles per DADD / DMUL / dd_add)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, int n, double a) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = __dadd_rn(x, a);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < n; i++) y = __dmul_rn(y, a);
  long long t2 = clock64();
  double hi = y, lo = 0;
  for (int i = 0; i < n; i++) {  // dd_add_d chain
    double s = __dadd_rn(hi, a), bb = __dsub_rn(s, hi);
    double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(a, bb));
    e = __dadd_rn(e, lo);
    hi = __dadd_rn(s, e);
    lo = __dsub_rn(e, __dsub_rn(hi, s));
  }
  long long t3 = clock64();
  double p = hi;
  for (int i = 0; i < 64; i++) p = pow(p * 1e-3 + 1.5, 0.8);
  long long t4 = clock64();
  out[threadIdx.x] = x + y + hi + lo + p;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double *o; long long *c, h[4];
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 32);
  int n = 4096;
  k<<<1, 32>>>(o, c, n, 1.0000001); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n, 1.0000001); cudaDeviceSynchronize();
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("{\"dadd_latency_cyc\": %.2f, \"dmul_latency_cyc\": %.2f, \"dd_add_d_cyc\": %.2f, \"pow_cyc\": %.1f}\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / 64);
  return 0;
}
