// Cluster barrier latency: 8 CTAs x 256 threads, 1000 barriers; optionally a global store in
// flight before each barrier (what the MGS exchange has: its LL words).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 calib/cbar_probe.cu -o calib/cbar_probe
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void bar_kernel(int iters, int mode, int st, long long* out, unsigned long long* g) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sm[threadIdx.x] = i;
    if (st && threadIdx.x < 8) g[blockIdx.x * 64 + threadIdx.x * 8] = i;   // global stores in flight
    if (mode == 0) cl.sync();
    else if (mode == 1) {
      asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    } else if (mode == 2) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 0) sm[300] += cl.map_shared_rank(sm, (blockIdx.x + 1) % 8)[5];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  unsigned long long* g; cudaMalloc(&g, 1 << 20);
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* nm[] = {"cg sync", "fence.acq_rel.cluster+relaxed", "arrive.release/wait.acquire", "relaxed only"};
  for (int st = 0; st < 2; ++st) for (int mode = 0; mode < 4; ++mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 8192;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, bar_kernel, 1000, mode, st, d, g);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
    printf("global stores %d, %-32s: %.1f cycles per iteration (%s)\n", st, nm[mode], h[0] / 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
