// Microbenchmark: cost of one grid-wide exchange round among G co-resident CTAs.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ int ld_acq(const int* p) { int v; asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ int ld_rlx(const int* p) { int v; asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(int* p, int v) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

template <int MODE, int READ>
__global__ void xbench(int* flags, unsigned* bar, double* part, int rounds, int spread) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  cg::grid_group grid = cg::this_grid();
  double acc = 0;
  for (int it = 1; it <= rounds; ++it) {
    if (tid < 64) part[(size_t)(it & 1) * G * 64 + tid * G + g] = it + tid;
    if (MODE == 3) { grid.sync(); }
    else if (MODE == 2) {
      __syncthreads();
      if (tid == 0) {
        unsigned g0 = *(volatile unsigned*)(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == G - 1) { bar[0] = 0; __threadfence(); atomicAdd(bar + 1, 1u); }
        else while (*(volatile unsigned*)(bar + 1) == g0) {}
        __threadfence();
      }
      __syncthreads();
    } else {
      __syncthreads();
      if (tid == 0) { if (MODE == 0) __threadfence(); st_rel(flags + (it & 1) * G * spread + g * spread, it); }
      if (tid < 32) {
        for (;;) {
          bool all = true;
          for (int h = lane; h < G; h += 32) all &= ((MODE == 0 ? ld_acq(flags + (it & 1) * G * spread + h * spread) : ld_rlx(flags + (it & 1) * G * spread + h * spread)) >= it);
          if (__all_sync(0xffffffffu, all)) break;
        }
        if (MODE == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
    }
    // read partials of 64 columns (one warp-row per column)
    if (spread < 0) { double s = 0; for (int h = 0; h < G; ++h) s += __ldcg(part + (size_t)(it & 1) * G * 64 + tid * G + h); acc += s; }
    else if (READ) {  // warp per column, lanes over CTAs, 8 columns per warp, all loads in flight
      const int warp = tid >> 5;
      double a[8];
      for (int t = 0; t < 8; ++t) a[t] = 0;
      for (int h = lane; h < G; h += 32)
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] += __ldcg(part + (size_t)(it & 1) * G * 64 + (warp + 8 * t) * G + h);
#pragma unroll
      for (int t = 0; t < 8; ++t) { for (int o = 16; o; o >>= 1) a[t] += __shfl_xor_sync(0xffffffffu, a[t], o); acc += a[t]; }
    }
  }
  if (acc == -1.0) part[0] = acc;
}

template <int RD> void run(int* flags, unsigned* bar, double* part, int rounds);
int main() {
  int *flags; unsigned* bar; double* part;
  cudaMalloc(&flags, 1 << 20); cudaMalloc(&bar, 64); cudaMalloc(&part, 1 << 24);
  const int rounds = 2000;
  run<0>(flags, bar, part, rounds); run<1>(flags, bar, part, rounds);
  return 0;
}
template <int RD> void run(int* flags, unsigned* bar, double* part, int rounds) {
  for (int G : {16, 32, 64, 128}) for (int mode = 0; mode < 4; ++mode) for (int spread : {1}) {
    cudaMemset(flags, 0, 1 << 20); cudaMemset(bar, 0, 64);
    void* args[] = {&flags, &bar, &part, (void*)&rounds, &spread};
    const void* k = mode == 0 ? (const void*)xbench<0, RD> : mode == 1 ? (const void*)xbench<1, RD> : mode == 2 ? (const void*)xbench<2, RD> : (const void*)xbench<3, RD>;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel(k, G, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(flags, 0, 1 << 20); cudaMemset(bar, 0, 64);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel(k, G, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("READ=%d G=%3d mode=%d (%s) spread=%2d: %.3f us/round %s\n", RD, G, mode, mode==0?"fence+release/acquire":mode==1?"release/relaxed+fence":mode==2?"atomic barrier":"cg grid.sync", spread, ms * 1e3 / rounds, cudaGetErrorString(err));
  }
}
