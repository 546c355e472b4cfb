// Diagnostic: one-way inter-SM latency of a global-memory flag (ping-pong / 2), cluster
// barrier latency, DSMEM load latency.  Not part of the library.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ int ldv(const int* p) { int v; asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void stv(int* p, int v) { asm volatile("st.volatile.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ int lda(const int* p) { int v; asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(int* p, int v) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

template <int MODE>
__global__ void pingpong(int* f, int rounds, int other, unsigned long long* out) {
  // block 0 and block `other` (grid = other+1; the rest idle)
  const int b = blockIdx.x;
  if (threadIdx.x != 0 || (b != 0 && b != other)) return;
  int* mine = f + (b == 0 ? 0 : 64);
  int* peer = f + (b == 0 ? 64 : 0);
  unsigned long long t0 = gtime();
  for (int i = 1; i <= rounds; ++i) {
    if (b == 0) {
      if (MODE == 0) stv(mine, i); else str(mine, i);
      if (MODE == 0) { while (ldv(peer) != i) {} } else { while (lda(peer) != i) {} }
    } else {
      if (MODE == 0) { while (ldv(peer) != i) {} } else { while (lda(peer) != i) {} }
      if (MODE == 0) stv(mine, i); else str(mine, i);
    }
  }
  if (b == 0) out[0] = gtime() - t0;
}

__global__ void clusterbar(int rounds, unsigned long long* out, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[256];
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  unsigned long long t0 = gtime();
  for (int i = 0; i < rounds; ++i) cl.sync();
  unsigned long long t1 = gtime();
  double a = 0;
  for (int i = 0; i < rounds; ++i) {
    const double* r = cl.map_shared_rank(buf, (cl.block_rank() + 1 + i) % cl.num_blocks());
    a += r[(threadIdx.x + (int)a) & 255];   // dependent chain of DSMEM loads
  }
  unsigned long long t2 = gtime();
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[1] = t1 - t0; out[2] = t2 - t1; }
  if (a == -1) sink[0] = a;
}

int main() {
  int* f; unsigned long long* out; double* sink;
  cudaMalloc(&f, 4096); cudaMalloc(&out, 64); cudaMalloc(&sink, 64);
  const int rounds = 10000;
  for (int other : {1, 2, 37, 74, 100, 147}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(f, 0, 4096);
      if (mode == 0) pingpong<0><<<other + 1, 32>>>(f, rounds, other, out); else pingpong<1><<<other + 1, 32>>>(f, rounds, other, out);
      unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      printf("pingpong block0<->block%d %s: one-way %.3f us  (%s)\n", other, mode ? "release/acquire" : "volatile", h / 1e3 / rounds / 2, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int csz : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(csz * 4); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(clusterbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, clusterbar, 1000, out, sink);
    cudaDeviceSynchronize();
    unsigned long long h[3]; cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    printf("cluster %2d: cluster.sync %.3f us, dependent DSMEM load %.3f us (%s)\n", csz, h[1] / 1e3 / 1000, h[2] / 1e3 / 1000, cudaGetErrorString(e));
  }
  return 0;
}
