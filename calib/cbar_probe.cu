// Cluster barrier latency: 8 CTAs x 256 threads (98 KB dyn smem each), 1000 cluster.sync().
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 calib/cbar_probe.cu -o calib/cbar_probe
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void bar_kernel(int iters, int mode, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) cl.sync();
    else if (mode == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    } else __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sm[threadIdx.x] = 0;
}
int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int cs : {2, 4, 8}) for (int mode = 0; mode < 3; ++mode) for (int dyn : {4096, 98 * 1024}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, bar_kernel, 1000, mode, d);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
    printf("cluster %d mode %d (%s) dyn %6d: %.1f cycles per barrier (%s)\n", cs, mode,
           mode == 0 ? "cg sync" : mode == 1 ? "relaxed" : "syncthreads", dyn, h[0] / 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
