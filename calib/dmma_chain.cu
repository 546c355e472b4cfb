// dmma_chain.cu — DMMA.8x8x4 dependent-chain latency and the rate vs. independent
// accumulator chains per SM sub-partition (DESIGN.md §5 K1s: why a 1-CTA/SM short-K flush
// with 16 chains per warp ran at half rate).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_chain dmma_chain.cu && ./dmma_chain
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// CH independent accumulators per warp, ITER sequential DMMAs on each
template <int CH>
__global__ void chain_kernel(double* out, long long* cyc, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x + 1), b = 1e-3 * (threadIdx.x + 2);
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run(int warps_per_cta, double* out, long long* cyc) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148;   // one CTA per SM
  chain_kernel<CH><<<grid, 32 * warps_per_cta>>>(out, cyc, 16);
  cudaEventRecord(e0);
  chain_kernel<CH><<<grid, 32 * warps_per_cta>>>(out, cyc, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 8 * 8 * 4 * (double)CH * iters * warps_per_cta * grid;
  printf("{\"chains_per_warp\": %d, \"warps_per_sm\": %d, \"chains_per_smsp\": %d, \"cycles_per_dmma_per_chain\": %.1f, "
         "\"tflops\": %.2f}\n",
         CH, warps_per_cta, CH * warps_per_cta / 4, (double)c / iters, flops / ms / 1e9);
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  run<1>(1, out, cyc);      // pure latency
  run<2>(1, out, cyc);
  run<4>(1, out, cyc);
  run<8>(4, out, cyc);
  run<16>(4, out, cyc);
  run<32>(4, out, cyc);
  run<16>(8, out, cyc);
  run<32>(8, out, cyc);
  run<16>(16, out, cyc);
  run<64>(4, out, cyc);
  run<32>(16, out, cyc);
  return 0;
}
