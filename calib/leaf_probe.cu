// Diagnostic: phase timing (%clock64) of the right-looking register Cholesky leaf (w = 32):
// diagonal load, Crout, row loads, barrier, substitution.  Not part of the library.
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
constexpr unsigned kFull = 0xffffffffu;
template <int W, int NT, int VAR>
__global__ void __launch_bounds__(NT) leaf(int64_t m, int w, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                           int64_t ldd, long long* stamps) {
  __shared__ double Ls[W][W + 1];
  __shared__ double inv[W];
  __shared__ double lc[2][W];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (warp == 0) {
    double a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k <= lane && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : 0.0;
    if (VAR == 1) { double s = 0; for (int k = 0; k < W; ++k) s += a[k]; if (s == 12345.0) a[0] = 1; }   // force loads complete
    t1 = clock64();
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const double d = __shfl_sync(kFull, a[c], c);
      const double Lcc = sqrt(d);
      double l;
      if (VAR == 3) {
        const double ri = 1.0 / Lcc;          // uniform across the warp
        l = (lane == c) ? Lcc : a[c] * ri;
        if (lane == c) inv[c] = ri;
      } else if (VAR == 4) {
        const double ri = 1.0 / Lcc;
        l = (lane == c) ? Lcc : a[c] / Lcc;   // division kept, reciprocal uniform (no divergent second division)
        if (lane == c) inv[c] = ri;
      } else {
        l = (lane == c) ? Lcc : a[c] / Lcc;
        if (lane == c) inv[c] = 1.0 / Lcc;
      }
      a[c] = l;
      if (lane < W) lc[c & 1][lane] = l;
      __syncwarp();
#pragma unroll
      for (int j = c + 1; j < W; ++j) a[j] = fma(-l, lc[c & 1][j], a[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) if (lane < W) Ls[lane][k] = (k <= lane) ? a[k] : 0.0;
    t2 = clock64();
  }
  double x[W];
  if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : 0.0;
  }
  long long t3 = clock64();
  __syncthreads();
  long long t4 = clock64();
  if (r < m) {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      x[c] = x[c] * inv[c];
#pragma unroll
      for (int j = c + 1; j < W; ++j) x[j] = fma(-x[c], Ls[j][c], x[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) if (k < w) dst[r + (int64_t)k * ldd] = x[k];
  }
  long long t5 = clock64();
  if (blockIdx.x == 0 && (tid == 0 || tid == 32)) {
    long long* o = stamps + (tid == 0 ? 0 : 8);
    o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t0; o[3] = t4 - t0; o[4] = t5 - t4; o[5] = t5 - t0;
  }
}
template <int W, int NT>
__global__ void __launch_bounds__(NT) leaf_rot(int64_t m, int w, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                               int64_t ldd, long long* stamps) {
  __shared__ double Ls[2 * W][W + 1];   // rows >= W stay zero (shifted reads past the block)
  __shared__ double inv[W];
  __shared__ double lc[2][2 * W];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  for (int idx = tid; idx < W * (W + 1); idx += NT) Ls[W + idx / (W + 1)][idx % (W + 1)] = 0.0;
  if (tid < 2 * W) { lc[0][tid] = 0.0; lc[1][tid] = 0.0; }
  __syncthreads();
  if (warp == 0) {
    double a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k <= lane && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : 0.0;
    t1 = clock64();
#pragma unroll 1
    for (int c = 0; c < w; ++c) {
      const double d = __shfl_sync(kFull, a[0], c);
      const double Lcc = sqrt(d);
      const double l = (lane == c) ? Lcc : a[0] / Lcc;
      if (lane == c) inv[c] = 1.0 / Lcc;
      if (lane < W) { Ls[lane][c] = (lane >= c) ? l : 0.0; lc[c & 1][lane] = (lane > c) ? l : 0.0; }
      __syncwarp();
      const double* lcc = &lc[c & 1][c];
#pragma unroll
      for (int j = 1; j < W; ++j) a[j - 1] = fma(-l, lcc[j], a[j]);
      a[W - 1] = 0.0;
    }
    t2 = clock64();
  }
  double x[W];
  if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : 0.0;
  }
  long long t3 = clock64();
  __syncthreads();
  long long t4 = clock64();
  if (r < m) {
#pragma unroll 1
    for (int c = 0; c < w; ++c) {
      const double xc = x[0] * inv[c];
      dst[r + (int64_t)c * ldd] = xc;
#pragma unroll
      for (int j = 1; j < W; ++j) x[j - 1] = fma(-xc, Ls[c + j][c], x[j]);
      x[W - 1] = 0.0;
    }
  }
  long long t5 = clock64();
  if (blockIdx.x == 0 && (tid == 0 || tid == 32)) {
    long long* o = stamps + (tid == 0 ? 0 : 8);
    o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t0; o[3] = t4 - t0; o[4] = t5 - t4; o[5] = t5 - t0;
  }
}

// rcp + transposed L (Lt[c][j] = L_jc, contiguous for the substitution) + pipelined:
// the row substitutions consume column c as soon as warp 0 has published it.
template <int W, int NT>
__global__ void __launch_bounds__(NT) leaf_pipe(int64_t m, int w, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                                int64_t ldd, long long* stamps) {
  __shared__ __align__(16) double Lt[W][W + 2];   // Lt[c][j] = L_jc (even stride: 16-byte rows)
  __shared__ double inv[W];
  __shared__ double lc[2][W];
  __shared__ volatile int ready;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (tid == 0) ready = 0;
  __syncthreads();
  double x[W];
  if (warp == 0) {
    double a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k <= lane && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : 0.0;
    t1 = clock64();
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const double d = __shfl_sync(kFull, a[c], c);
      const double Lcc = sqrt(d);
      const double ri = 1.0 / Lcc;
      const double l = (lane == c) ? Lcc : a[c] * ri;
      a[c] = l;
      if (lane < W) { lc[c & 1][lane] = l; Lt[c][lane] = (lane >= c) ? l : 0.0; }
      if (lane == c) inv[c] = ri;
      __syncwarp();
      if (lane == 0) { __threadfence_block(); ready = c + 1; }
#pragma unroll
      for (int j = c + 1; j < W; ++j) a[j] = fma(-l, lc[c & 1][j], a[j]);
    }
    t2 = clock64();
  }
  if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : 0.0;
  }
  long long t3 = clock64();
  long long t4 = t3;
  if (r < m) {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (warp != 0) { while (ready <= c) {} __threadfence_block(); }
      x[c] = x[c] * inv[c];
      const double* lt = &Lt[c][0];
#pragma unroll
      for (int j = c + 1; j < W; ++j) x[j] = fma(-x[c], lt[j], x[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) if (k < w) dst[r + (int64_t)k * ldd] = x[k];
  }
  long long t5 = clock64();
  if (blockIdx.x == 0 && (tid == 0 || tid == 32)) {
    long long* o = stamps + (tid == 0 ? 0 : 8);
    o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t0; o[3] = t4 - t0; o[4] = t5 - t4; o[5] = t5 - t0;
  }
}

// rolled + rotated registers + reciprocal + shifted (16-byte aligned) broadcast vectors
template <int W, int NT>
__global__ void __launch_bounds__(NT) leaf_rot2(int64_t m, int w, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                                int64_t ldd, long long* stamps) {
  __shared__ __align__(16) double Lr[W][W];   // Lr[c][j] = L_{c+1+j, c} (0 past the block)
  __shared__ double inv[W];
  __shared__ double Ld[W][W + 1];             // the block itself, for the write-out
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (warp == 0) {
    double a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k <= lane && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : 0.0;
    t1 = clock64();
#pragma unroll 1
    for (int c = 0; c < w; ++c) {
      const double d = __shfl_sync(kFull, a[0], c);     // a[0] = current column of my row
      const double Lcc = sqrt(d);
      const double ri = 1.0 / Lcc;
      const double l = (lane == c) ? Lcc : a[0] * ri;
      if (lane < W) {
        Ld[lane][c] = (lane >= c) ? l : 0.0;
        Lr[c][lane] = 0.0;
      }
      __syncwarp();
      if (lane > c && lane < W) Lr[c][lane - c - 1] = l;
      if (lane == c) inv[c] = ri;
      __syncwarp();
      const double* v = &Lr[c][0];
#pragma unroll
      for (int j = 1; j < W; ++j) a[j - 1] = fma(-l, v[j - 1], a[j]);
      a[W - 1] = 0.0;
    }
    t2 = clock64();
  }
  double x[W];
  if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : 0.0;
  }
  long long t3 = clock64();
  __syncthreads();
  long long t4 = clock64();
  if (r < m) {
#pragma unroll 1
    for (int c = 0; c < w; ++c) {
      const double xc = x[0] * inv[c];
      dst[r + (int64_t)c * ldd] = xc;
      const double* v = &Lr[c][0];
#pragma unroll
      for (int j = 1; j < W; ++j) x[j - 1] = fma(-xc, v[j - 1], x[j]);
      x[W - 1] = 0.0;
    }
  }
  long long t5 = clock64();
  if (blockIdx.x == 0 && (tid == 0 || tid == 32)) {
    long long* o = stamps + (tid == 0 ? 0 : 8);
    o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t0; o[3] = t4 - t0; o[4] = t5 - t4; o[5] = t5 - t0;
  }
}

template <int VAR>
void run(const char* name, int64_t m, double* src, double* dst, long long* st) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = (int)((m - 32 + 127) / 128);
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0);
    if (VAR == 6) leaf_rot2<32, 128><<<grid, 128>>>(m, 32, src, m, dst, m, st); else if (VAR == 5) leaf_pipe<32, 128><<<grid, 128>>>(m, 32, src, m, dst, m, st); else if (VAR == 2) leaf_rot<32, 128><<<grid, 128>>>(m, 32, src, m, dst, m, st); else leaf<32, 128, VAR><<<grid, 128>>>(m, 32, src, m, dst, m, st);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
  }
  long long h[16]; cudaMemcpy(h, st, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s m=%lld: %.1f us | warp0: diagload %lld crout %lld rowsload-end %lld barrier-end %lld subst %lld total %lld | warp1: rowsload-end %lld barrier-end %lld subst %lld total %lld cycles (%s)\n",
         name, (long long)m, best * 1e3, h[0], h[1], h[2], h[3], h[4], h[5], h[10], h[11], h[12], h[13], cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int64_t m = 65536;
  std::vector<double> hv(m * 32);
  for (int64_t i = 0; i < m * 32; ++i) hv[i] = 0.01 * (rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < 32; ++i) hv[i + i * m] += 4.0;
  double *src, *dst; long long* st;
  cudaMalloc(&src, m * 32 * 8); cudaMalloc(&dst, m * 32 * 8); cudaMalloc(&st, 256);
  cudaMemcpy(src, hv.data(), m * 32 * 8, cudaMemcpyHostToDevice);
  for (int64_t mm : {2000, 16384, 65536}) { run<0>("rl", mm, src, dst, st); run<2>("rot", mm, src, dst, st); run<3>("rl-rcp", mm, src, dst, st); run<6>("rot2", mm, src, dst, st); }
  // check rot == rl output
  {
    int64_t mm = 16384; std::vector<double> o1(mm * 32), o2(mm * 32);
    run<3>("rl-rcp", mm, src, dst, st); cudaMemcpy(o1.data(), dst, mm * 32 * 8, cudaMemcpyDeviceToHost);
    cudaMemset(dst, 0, mm * 32 * 8);
    run<6>("rot2", mm, src, dst, st); cudaMemcpy(o2.data(), dst, mm * 32 * 8, cudaMemcpyDeviceToHost);
    double md = 0; for (int64_t i = 32; i < mm; ++i) for (int k = 0; k < 32; ++k) { double dd = fabs(o1[i + k * mm] - o2[i + k * mm]); if (dd > md) md = dd; }
    printf("max |rl - rot| rows below = %g\n", md);
  }
  return 0;
}
