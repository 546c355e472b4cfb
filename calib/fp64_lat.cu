// Diagnostic: dependent-chain latency (cycles) of fp64 ops on this GPU.  Not part of the library.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int n) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = 1.5 / x + 0.5;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-12;
  long long t4 = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-7f);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x) + 0.5;
  long long t7 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, c, 1.3, n);
    long long h[7]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("per op (cycles, dependent chain): dfma %.1f  sqrt+add %.1f  div+add %.1f  shfl.f64+add %.1f  ffma %.1f  dmul %.1f  drcp_rn+add %.1f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n, h[6] / (double)n);
  }
  return 0;
}
