// panels.cu — the s-column panel recurrences of Algorithms 1-3
// plus small utilities.  Templated on the storage type (double for the fp64 path, float for
// the fp32 path).
//
// Cholesky leaf: for each column c of the leaf
//     L_cc = sqrt(A_cc - sum_k L_ck^2),   L_ic = (A_ic - sum_k L_ik L_ck) / L_cc
// The k-sums run over the leaf's earlier columns; earlier columns of the same panel were
// folded in by the driver's sub-panel correction (same terms, grouped), earlier panels by
// the flushes.  Restructured for the GPU (same arithmetic per element, reassociated sums):
// every CTA factors the w x w diagonal block redundantly in shared memory (one warp, a lane
// per row), then each thread runs an independent forward substitution for one row below
// (rows are coalesced across a warp because the matrix is column-major).
//
// LU leaf: L_ic = A_ic - sum_k L_ik U_kc ; U_ci = (A_ci - sum_k L_ck U_ki)/L_cc
// diagonal block Crout in shared memory, then L rows below and U columns to the right are
// independent substitutions (thread per row / per column).
//
// QR MGS panel: v = M[:,c]; v -= q_j (q_j^T v) for j in [z, c); q_c = v/||v||.
// Right-looking form (each column sees the same projections in the same order): when q_c
// is done every later panel column is projected once.  The norm of v_c and its dot
// products with the later columns come from ONE grid-wide reduction (Gram row), so the
// persistent cooperative kernel needs one grid barrier per column.
#include <cooperative_groups.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace sf {

template <typename T> __device__ __forceinline__ T dsqrt(T x);
template <> __device__ __forceinline__ double dsqrt<double>(double x) { return sqrt(x); }
template <> __device__ __forceinline__ float dsqrt<float>(float x) { return sqrtf(x); }

__device__ __forceinline__ void record_fail(long long* fail, long long col1) {
  atomicMin((unsigned long long*)fail, (unsigned long long)col1);
}

// =============================================================== Cholesky leaf
constexpr int kLeafThreads = 128;

template <typename T, int W>
__global__ void __launch_bounds__(kLeafThreads) chol_leaf_kernel(int64_t m, int w, const T* __restrict__ src,
                                                                 int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                                 int64_t col0, long long* fail) {
  if (failed(fail)) return;
  __shared__ T D[W][W + 1];
  __shared__ T inv[W];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) bad = 0;
  for (int idx = tid; idx < w * w; idx += kLeafThreads) {
    const int i = idx % w, j = idx / w;
    if (i >= j) D[i][j] = src[i + (int64_t)j * lds];
  }
  __syncthreads();
  if (tid < 32) {
    // one warp; lane owns rows lane and lane+32 (W <= 64)
    for (int c = 0; c < w; ++c) {
      T t[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        t[h] = T(0);
        if (i >= c && i < w) {
          T a0 = D[i][c], a1 = T(0), a2 = T(0), a3 = T(0);
          int k = 0;
          for (; k + 4 <= c; k += 4) {
            a0 = fma(-D[i][k], D[c][k], a0);
            a1 = fma(-D[i][k + 1], D[c][k + 1], a1);
            a2 = fma(-D[i][k + 2], D[c][k + 2], a2);
            a3 = fma(-D[i][k + 3], D[c][k + 3], a3);
          }
          for (; k < c; ++k) a0 = fma(-D[i][k], D[c][k], a0);
          t[h] = (a0 + a1) + (a2 + a3);
        }
      }
      const T d = __shfl_sync(0xffffffffu, (c >> 5) ? t[1] : t[0], c & 31);
      if (!(d > T(0))) {  // not positive definite (or NaN) at column col0 + c
        if (lane == 0) { bad = 1; if (blockIdx.x == 0) record_fail(fail, col0 + c + 1); }
        break;
      }
      const T Lcc = dsqrt(d);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (i == c) D[c][c] = Lcc;
        else if (i > c && i < w) D[i][c] = t[h] / Lcc;
      }
      if (lane == 0) inv[c] = T(1) / Lcc;
      __syncwarp();
    }
  }
  __syncthreads();
  if (bad) return;
  if (blockIdx.x == 0) {
    for (int idx = tid; idx < w * w; idx += kLeafThreads) {
      const int i = idx % w, j = idx / w;
      if (i >= j) dst[i + (int64_t)j * ldd] = D[i][j];
    }
  }
  // rows below the diagonal block: independent forward substitutions
  const int64_t r = w + (int64_t)blockIdx.x * kLeafThreads + tid;
  if (r >= m) return;
  T x[W];
#pragma unroll
  for (int k = 0; k < W; ++k) x[k] = (k < w) ? src[r + (int64_t)k * lds] : T(0);
#pragma unroll
  for (int c = 0; c < W; ++c) {
    if (c < w) {
      T a0 = x[c], a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
      for (int k = 0; k + 4 <= c; k += 4) {
        a0 = fma(-x[k], D[c][k], a0);
        a1 = fma(-x[k + 1], D[c][k + 1], a1);
        a2 = fma(-x[k + 2], D[c][k + 2], a2);
        a3 = fma(-x[k + 3], D[c][k + 3], a3);
      }
#pragma unroll
      for (int k = c & ~3; k < c; ++k) a0 = fma(-x[k], D[c][k], a0);
      x[c] = ((a0 + a1) + (a2 + a3)) * inv[c];
    }
  }
#pragma unroll
  for (int k = 0; k < W; ++k)
    if (k < w) dst[r + (int64_t)k * ldd] = x[k];
}

template <typename T>
cudaError_t chol_leaf(int64_t m, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                      long long* fail, cudaStream_t st) {
  if (w <= 0 || m <= 0) return cudaSuccess;
  const int64_t below = m - w;
  const int grid = below > 0 ? (int)((below + kLeafThreads - 1) / kLeafThreads) : 1;
  if (w <= 16) chol_leaf_kernel<T, 16><<<grid, kLeafThreads, 0, st>>>(m, w, src, lds, dst, ldd, col0, fail);
  else if (w <= 32) chol_leaf_kernel<T, 32><<<grid, kLeafThreads, 0, st>>>(m, w, src, lds, dst, ldd, col0, fail);
  else if (w <= 64) chol_leaf_kernel<T, 64><<<grid, kLeafThreads, 0, st>>>(m, w, src, lds, dst, ldd, col0, fail);
  else return cudaErrorInvalidValue;
  count_launch();
  return cudaGetLastError();
}

// =============================================================== LU leaf
template <typename T, int W>
__global__ void __launch_bounds__(kLeafThreads) lu_leaf_kernel(int64_t m, int64_t ncr, int w,
                                                               const T* __restrict__ src, int64_t lds,
                                                               T* __restrict__ dst, int64_t ldd, int64_t col0,
                                                               const T* tolp, long long* fail, int nrow_blocks) {
  if (failed(fail)) return;
  __shared__ T D[W][W + 1];
  __shared__ T inv[W];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31;
  const T tol = *tolp;
  if (tid == 0) bad = 0;
  for (int idx = tid; idx < w * w; idx += kLeafThreads) {
    const int i = idx % w, j = idx / w;
    D[i][j] = src[i + (int64_t)j * lds];
  }
  __syncthreads();
  if (tid < 32) {
    for (int c = 0; c < w; ++c) {
      T tl[2], tu[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        tl[h] = T(0); tu[h] = T(0);
        if (i >= c && i < w) {
          // L_ic = A_ic - sum_k L_ik U_kc
          T a0 = D[i][c], a1 = T(0);
          int k = 0;
          for (; k + 2 <= c; k += 2) { a0 = fma(-D[i][k], D[k][c], a0); a1 = fma(-D[i][k + 1], D[k + 1][c], a1); }
          if (k < c) a0 = fma(-D[i][k], D[k][c], a0);
          tl[h] = a0 + a1;
        }
        if (i > c && i < w) {
          // U_ci * L_cc = A_ci - sum_k L_ck U_ki
          T a0 = D[c][i], a1 = T(0);
          int k = 0;
          for (; k + 2 <= c; k += 2) { a0 = fma(-D[c][k], D[k][i], a0); a1 = fma(-D[c][k + 1], D[k + 1][i], a1); }
          if (k < c) a0 = fma(-D[c][k], D[k][i], a0);
          tu[h] = a0 + a1;
        }
      }
      const T Lcc = __shfl_sync(0xffffffffu, (c >> 5) ? tl[1] : tl[0], c & 31);
      if (!(fabs(Lcc) >= tol)) {
        if (lane == 0) { bad = 1; if (blockIdx.x == 0) record_fail(fail, col0 + c + 1); }
        break;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (i >= c && i < w) D[i][c] = tl[h];
        if (i > c && i < w) D[c][i] = tu[h] / Lcc;
      }
      if (lane == 0) inv[c] = T(1) / Lcc;
      __syncwarp();
    }
  }
  __syncthreads();
  if (bad) return;
  if (blockIdx.x == 0) {
    for (int idx = tid; idx < w * w; idx += kLeafThreads) {
      const int i = idx % w, j = idx / w;
      dst[i + (int64_t)j * ldd] = D[i][j];
    }
  }
  if ((int)blockIdx.x < nrow_blocks) {
    // L rows below: L_rc = A_rc - sum_{k<c} L_rk U_kc
    const int64_t r = w + (int64_t)blockIdx.x * kLeafThreads + tid;
    if (r >= m) return;
    T x[W];
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? src[r + (int64_t)k * lds] : T(0);
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (c < w) {
        T a0 = x[c], a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
        for (int k = 0; k + 4 <= c; k += 4) {
          a0 = fma(-x[k], D[k][c], a0);
          a1 = fma(-x[k + 1], D[k + 1][c], a1);
          a2 = fma(-x[k + 2], D[k + 2][c], a2);
          a3 = fma(-x[k + 3], D[k + 3][c], a3);
        }
#pragma unroll
        for (int k = c & ~3; k < c; ++k) a0 = fma(-x[k], D[k][c], a0);
        x[c] = (a0 + a1) + (a2 + a3);
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) dst[r + (int64_t)k * ldd] = x[k];
  } else {
    // U columns to the right: U_cj = (A_cj - sum_{k<c} L_ck U_kj) / L_cc
    const int64_t j = w + (int64_t)(blockIdx.x - nrow_blocks) * kLeafThreads + tid;
    if (j >= w + ncr) return;
    const T* col = src + j * lds;
    T y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) y[k] = (k < w) ? col[k] : T(0);
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (c < w) {
        T a0 = y[c], a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
        for (int k = 0; k + 4 <= c; k += 4) {
          a0 = fma(-D[c][k], y[k], a0);
          a1 = fma(-D[c][k + 1], y[k + 1], a1);
          a2 = fma(-D[c][k + 2], y[k + 2], a2);
          a3 = fma(-D[c][k + 3], y[k + 3], a3);
        }
#pragma unroll
        for (int k = c & ~3; k < c; ++k) a0 = fma(-D[c][k], y[k], a0);
        y[c] = ((a0 + a1) + (a2 + a3)) * inv[c];
      }
    }
    T* out = dst + j * ldd;
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) out[k] = y[k];
  }
}

template <typename T>
cudaError_t lu_leaf(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                    const T* tol, long long* fail, cudaStream_t st) {
  if (w <= 0 || m <= 0) return cudaSuccess;
  const int64_t below = m - w;
  const int nrb = below > 0 ? (int)((below + kLeafThreads - 1) / kLeafThreads) : 0;
  const int ncb = ncr > 0 ? (int)((ncr + kLeafThreads - 1) / kLeafThreads) : 0;
  int grid = nrb + ncb;
  if (grid == 0) grid = 1;
  if (w <= 16) lu_leaf_kernel<T, 16><<<grid, kLeafThreads, 0, st>>>(m, ncr, w, src, lds, dst, ldd, col0, tol, fail, nrb);
  else if (w <= 32) lu_leaf_kernel<T, 32><<<grid, kLeafThreads, 0, st>>>(m, ncr, w, src, lds, dst, ldd, col0, tol, fail, nrb);
  else if (w <= 64) lu_leaf_kernel<T, 64><<<grid, kLeafThreads, 0, st>>>(m, ncr, w, src, lds, dst, ldd, col0, tol, fail, nrb);
  else return cudaErrorInvalidValue;
  count_launch();
  return cudaGetLastError();
}

// =============================================================== QR MGS panel
constexpr int kMgsThreads = 256;

struct MgsGeom { int G; int RB; size_t smem; };

static MgsGeom mgs_geom(int64_t n, int w, int elt) {
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  MgsGeom g;
  g.G = (int)((n + 63) / 64);
  if (g.G > sms) g.G = sms;
  if (g.G < 1) g.G = 1;
  g.RB = (int)((n + g.G - 1) / g.G);
  g.smem = (size_t)elt * ((size_t)g.RB * w + 2 * (size_t)w + 64);
  return g;
}

size_t qr_mgs_work_elems(int64_t n, int w) {
  MgsGeom g = mgs_geom(n, w, 8);
  return 2 * (size_t)g.G * (size_t)w;
}

template <typename T>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                             int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                             int64_t col0, const T* tolp, T* work,
                                                             long long* fail) {
  if (failed(fail)) return;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  T* V = reinterpret_cast<T*>(smraw);          // V[c * RB + r]: this CTA's rows of the panel
  T* gsum = V + (size_t)RB * w;                // reduced Gram row for the current column
  T* dcoef = gsum + w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kMgsThreads / 32;
  const int G = gridDim.x, g = blockIdx.x;
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = *tolp;

  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    V[idx] = (r < rows) ? src[r0 + r + (int64_t)c * lds] : T(0);
  }
  __syncthreads();

  bool ok = true;
  for (int c = 0; c < w; ++c) {
    T* part = work + (size_t)(c & 1) * G * w;
    // 1) partial Gram row: <v_c, v_c'> over this CTA's rows, c' in [c, w)
    const T* vc = V + (size_t)c * RB;
    for (int cp = c + warp; cp < w; cp += nwarps) {
      const T* v2 = V + (size_t)cp * RB;
      T acc = T(0);
      for (int r = lane; r < RB; r += 32) acc = fma(vc[r], v2[r], acc);
      acc = warp_sum(acc);
      if (lane == 0) part[(size_t)g * w + cp] = acc;
    }
    grid.sync();
    // 2) every CTA reduces the partials in the same fixed order
    for (int cp = c + tid; cp < w; cp += kMgsThreads) {
      T s = T(0);
      for (int h = 0; h < G; ++h) s += part[(size_t)h * w + cp];
      gsum[cp] = s;
    }
    __syncthreads();
    const T nv = dsqrt(gsum[c]);
    if (!(nv >= tol)) {
      if (g == 0 && tid == 0) record_fail(fail, col0 + c + 1);
      ok = false;
      break;
    }
    for (int cp = c + 1 + tid; cp < w; cp += kMgsThreads) dcoef[cp] = gsum[cp] / nv;   // q_c^T v_c'
    for (int r = tid; r < RB; r += kMgsThreads) V[(size_t)c * RB + r] = vc[r] / nv;     // q_c = v_c/||v_c||
    __syncthreads();
    // 3) project q_c out of every later panel column
    const int rem = w - c - 1;
    for (int idx = tid; idx < RB * rem; idx += kMgsThreads) {
      const int r = idx % RB, cp = c + 1 + idx / RB;
      V[(size_t)cp * RB + r] = fma(-vc[r], dcoef[cp], V[(size_t)cp * RB + r]);
    }
    __syncthreads();
  }
  if (!ok) return;
  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    if (r < rows) dst[r0 + r + (int64_t)c * ldd] = V[idx];
  }
}

template <typename T>
cudaError_t qr_mgs_panel(int64_t n, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                         const T* tol, T* work, long long* fail, cudaStream_t st) {
  if (w <= 0) return cudaSuccess;
  MgsGeom g = mgs_geom(n, w, (int)sizeof(T));
  if (g.smem > 220 * 1024) return cudaErrorInvalidValue;   // caller splits wider panels
  auto k = qr_mgs_kernel<T>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  if (e != cudaSuccess) return e;
  int RB = g.RB;
  void* args[] = {(void*)&n, (void*)&w, (void*)&RB, (void*)&src, (void*)&lds, (void*)&dst, (void*)&ldd,
                  (void*)&col0, (void*)&tol, (void*)&work, (void*)&fail};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k, dim3(g.G), dim3(kMgsThreads), args, g.smem, st);
}

int qr_mgs_max_width(int64_t n, int elt) {
  MgsGeom g = mgs_geom(n, 1, elt);
  int64_t w = (220 * 1024 / elt - 64) / (g.RB + 2);
  return (int)(w > 4096 ? 4096 : w);
}

// =============================================================== utilities
template <typename T>
__global__ void sumsq_partial(int64_t n, const T* A, int64_t lda, double* part) {
  double acc = 0.0;
  const int64_t total = n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)A[(t % n) + (t / n) * lda];
    acc = fma(v, v, acc);
  }
  __shared__ double red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

template <typename T>
__global__ void sumsq_final(int64_t n, const double* part, int np, T* tol_out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += part[i];
    tol_out[0] = (T)(1e-12 * sqrt(s) / (double)n);
  }
}

template <typename T>
cudaError_t frob_norm_tol(int64_t n, const T* A, int64_t lda, T* tol_out, double* part, cudaStream_t st) {
  const int np = 512;
  sumsq_partial<T><<<np, 256, 0, st>>>(n, A, lda, part); count_launch();
  sumsq_final<T><<<1, 32, 0, st>>>(n, part, np, tol_out); count_launch();
  return cudaGetLastError();
}

__global__ void init_fail_kernel(long long* fail) { *fail = kNoFail; }
__global__ void finish_info_kernel(const long long* fail, int64_t* info) {
  const long long f = *fail;
  *info = (f == kNoFail) ? 0 : (int64_t)f;
}
cudaError_t init_fail(long long* fail, cudaStream_t st) {
  init_fail_kernel<<<1, 1, 0, st>>>(fail); count_launch();
  return cudaGetLastError();
}
cudaError_t finish_info(const long long* fail, int64_t* d_info, cudaStream_t st) {
  finish_info_kernel<<<1, 1, 0, st>>>(fail, d_info); count_launch();
  return cudaGetLastError();
}

template <typename T>
__global__ void zero_lower_kernel(int64_t n, T* R, int64_t ldr) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = j + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      R[i + j * ldr] = T(0);
}
template <typename T>
cudaError_t zero_strict_lower(int64_t n, T* R, int64_t ldr, cudaStream_t st) {
  zero_lower_kernel<T><<<dim3(4, 1024), 256, 0, st>>>(n, R, ldr); count_launch();
  return cudaGetLastError();
}

template <typename T>
__global__ void copy_kernel(int64_t m, int64_t n, const T* src, int64_t lds, T* dst, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      dst[i + j * ldd] = src[i + j * lds];
}
template <typename T>
cudaError_t copy_matrix(int64_t m, int64_t n, const T* src, int64_t lds, T* dst, int64_t ldd, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  copy_kernel<T><<<dim3((unsigned)((m + 255) / 256 > 8 ? 8 : (m + 255) / 256), 2048), 256, 0, st>>>(m, n, src, lds, dst, ldd); count_launch();
  return cudaGetLastError();
}

#define SF_INST(T)                                                                                             \
  template cudaError_t chol_leaf<T>(int64_t, int, const T*, int64_t, T*, int64_t, int64_t, long long*,        \
                                    cudaStream_t);                                                            \
  template cudaError_t lu_leaf<T>(int64_t, int64_t, int, const T*, int64_t, T*, int64_t, int64_t, const T*,  \
                                  long long*, cudaStream_t);                                                  \
  template cudaError_t qr_mgs_panel<T>(int64_t, int, const T*, int64_t, T*, int64_t, int64_t, const T*, T*,  \
                                       long long*, cudaStream_t);                                             \
  template cudaError_t frob_norm_tol<T>(int64_t, const T*, int64_t, T*, double*, cudaStream_t);                   \
  template cudaError_t zero_strict_lower<T>(int64_t, T*, int64_t, cudaStream_t);                             \
  template cudaError_t copy_matrix<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t);
SF_INST(double)
SF_INST(float)

}  // namespace sf
