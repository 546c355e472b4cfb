// L0 calibration: FP64 DMMA (mma.sync m8n8k4) vs DFMA throughput, FP32 FFMA, on one B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o calib calib.cu
// Prints one JSON object on stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_bench(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_bench(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void ffma_bench(float* out, int iters) {
  float a = 1.0f + threadIdx.x * 1e-7f, b = 1.0f - threadIdx.x * 1e-7f;
  float c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fmaf(c[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456f) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* dout; float* fout;
  CK(cudaMalloc(&dout, 1024 * sizeof(double))); CK(cudaMalloc(&fout, 1024 * sizeof(float)));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, sms, clk_khz);
  // DMMA: each warp-instruction = 8*8*4 = 256 FMA = 512 flop.
  for (int wpb : {4, 8, 16}) {
    const int iters = 20000;
    int grid = sms * 2, block = 32 * wpb;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dmma_bench<8><<<grid, block>>>(dout, iters); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_bench<8><<<grid, block>>>(dout, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
    }
    double flops = (double)grid * wpb * iters * 8 * 512.0;
    printf(", \"dmma_tflops_wpb%d\": %.3f", wpb, flops / (best * 1e-3) / 1e12);
  }
  for (int wpb : {8, 16, 32}) {
    const int iters = 20000;
    int grid = sms * 2, block = 32 * wpb;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dfma_bench<8><<<grid, block>>>(dout, iters); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_bench<8><<<grid, block>>>(dout, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
    }
    double flops = (double)grid * block * iters * 8 * 2.0;
    printf(", \"dfma_tflops_wpb%d\": %.3f", wpb, flops / (best * 1e-3) / 1e12);
  }
  for (int wpb : {16, 32}) {
    const int iters = 20000;
    int grid = sms * 2, block = 32 * wpb;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    ffma_bench<8><<<grid, block>>>(fout, iters); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); ffma_bench<8><<<grid, block>>>(fout, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
    }
    double flops = (double)grid * block * iters * 8 * 2.0;
    printf(", \"ffma_tflops_wpb%d\": %.3f", wpb, flops / (best * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
