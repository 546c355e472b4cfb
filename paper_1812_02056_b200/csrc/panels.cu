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
#include <math.h>

#include "common.cuh"
#include "kernels.h"


namespace sf {

template <typename T> __device__ __forceinline__ T dsqrt(T x);
template <> __device__ __forceinline__ double dsqrt<double>(double x) { return sqrt(x); }
template <> __device__ __forceinline__ float dsqrt<float>(float x) { return sqrtf(x); }

__device__ __forceinline__ void record_fail(long long* fail, long long col1) {
  atomicMin((unsigned long long*)fail, (unsigned long long)col1);
}

// =============================================================== QR MGS panel
constexpr int kMgsThreads = 256;

struct MgsGeom { int G; int RB; size_t smem; };

static MgsGeom mgs_geom(int64_t n, int w, int elt) {
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  MgsGeom g;
  g.G = (int)((n + 127) / 128);
  if (g.G > sms) g.G = sms;
  if (g.G < 1) g.G = 1;
  g.RB = (int)((n + g.G - 1) / g.G);
  g.smem = (size_t)elt * ((size_t)g.RB * w + 2 * (size_t)w + 64);
  return g;
}

size_t qr_mgs_work_elems(int64_t n, int w) {
  MgsGeom g = mgs_geom(n, w, 8);
  return (size_t)g.G + 2 * (size_t)g.G * (size_t)w + 2;   // flags[2][G] + partials[2][w][G]
}

// Inter-CTA exchange for a cooperative (co-resident) grid, without atomics: CTA g publishes
// its partial Gram row for column c into slot part[c&1] and then raises flag[c&1][g] = c+1
// (release); readers poll all G flags of that parity (acquire) and then read the partials
// bypassing L1.  Double buffering by column parity is safe: a CTA writes parity c&1 again
// only at column c+2, after it has seen every CTA's flag for column c+1, i.e. after every
// CTA finished reading the column-c partials.
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kMgsMaxT = 16;   // columns per warp whose partial sums are fetched together

template <typename T>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                             int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                             int64_t col0, const T* tolp, T* work,
                                                             long long* fail) {
  if (failed(fail)) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* V = reinterpret_cast<T*>(smraw);          // V[c * RB + r]: this CTA's rows of the panel
  T* gsum = V + (size_t)RB * w;                // reduced Gram row for the current column
  T* dcoef = gsum + w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kMgsThreads / 32;
  const int G = gridDim.x, g = blockIdx.x;
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = __ldcg(tolp);
  int* flags = reinterpret_cast<int*>(work);                                   // flags[2][G]
  T* partbase = work + (2 * G * sizeof(int) + sizeof(T) - 1) / sizeof(T);     // part[2][w][G]

  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    V[idx] = (r < rows) ? __ldcg(src + r0 + r + (int64_t)c * lds) : T(0);   // L2, never a stale L1 line
  }
  __syncthreads();

  bool ok = true;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    T* part = partbase + (size_t)buf * G * w;
    // 1) partial Gram row over this CTA's rows: <v_c, v_c'> for c' in [c, w)
    const T* vc = V + (size_t)c * RB;
    for (int cp = c + warp; cp < w; cp += nwarps) {
      const T* v2 = V + (size_t)cp * RB;
      T acc = T(0);
      for (int r = lane; r < RB; r += 32) acc = fma(vc[r], v2[r], acc);
      acc = warp_sum(acc);
      if (lane == 0) part[(size_t)cp * G + g] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_s32(flags + buf * G + g, (int)(col0 + c + 1));   // epochs grow across launches
    }
    // 2) wait until every CTA has published column c
    if (warp == 0) {
      for (;;) {
        bool mine = true;
        for (int h = lane; h < G; h += 32) mine &= (ld_acquire_s32(flags + buf * G + h) >= (int)(col0 + c + 1));
        if (__all_sync(0xffffffffu, mine)) break;
      }
    }
    __syncthreads();
    // 3) every CTA reduces the partials in the same fixed order (warp per column,
    //    coalesced over the CTA index; deterministic shuffle tree), all loads in flight
    for (int cb = c + warp; cb < w; cb += nwarps * kMgsMaxT) {
      T acc[kMgsMaxT];
#pragma unroll
      for (int t = 0; t < kMgsMaxT; ++t) acc[t] = T(0);
      for (int h = lane; h < G; h += 32) {
#pragma unroll
        for (int t = 0; t < kMgsMaxT; ++t) {
          const int cp = cb + t * nwarps;
          if (cp < w) acc[t] += __ldcg(part + (size_t)cp * G + h);
        }
      }
#pragma unroll
      for (int t = 0; t < kMgsMaxT; ++t) {
        const int cp = cb + t * nwarps;
        const T v = warp_sum(acc[t]);
        if (lane == 0 && cp < w) gsum[cp] = v;
      }
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
    // 4) project q_c out of every later panel column
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

__global__ void init_fail_kernel(long long* fail) { fail[0] = kNoFail; fail[1] = 0; }
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
      dst[i + j * ldd] = __ldcg(src + i + j * lds);
}
template <typename T>
cudaError_t copy_matrix(int64_t m, int64_t n, const T* src, int64_t lds, T* dst, int64_t ldd, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  copy_kernel<T><<<dim3((unsigned)((m + 255) / 256 > 8 ? 8 : (m + 255) / 256), 2048), 256, 0, st>>>(m, n, src, lds, dst, ldd); count_launch();
  return cudaGetLastError();
}

#define SF_INST(T)                                                                                             \
  template cudaError_t qr_mgs_panel<T>(int64_t, int, const T*, int64_t, T*, int64_t, int64_t, const T*, T*,  \
                                       long long*, cudaStream_t);                                             \
  template cudaError_t frob_norm_tol<T>(int64_t, const T*, int64_t, T*, double*, cudaStream_t);                   \
  template cudaError_t zero_strict_lower<T>(int64_t, T*, int64_t, cudaStream_t);                             \
  template cudaError_t copy_matrix<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t);
SF_INST(double)
SF_INST(float)

}  // namespace sf
