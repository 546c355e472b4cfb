// leaf.cu — the innermost panel recurrences (W <= 32 columns) of Algorithms 1 and 2.
//
// Cholesky, for each column c of the leaf:
//     L_cc = sqrt(A_cc - sum_{k<c} L_ck^2),    L_ic = (A_ic - sum_{k<c} L_ik L_ck) / L_cc
// LU, Crout form, for each column/row c:
//     L_ic = A_ic - sum_{k<c} L_ik U_kc   (i >= c),   U_ci = (A_ci - sum_{k<c} L_ck U_ki) / L_cc  (i > c)
// (the sums over earlier columns of the same panel / earlier panels were already applied by
// the driver's grouped corrections and by the flushes).
//
// GPU structure.  Every CTA first factors the w x w diagonal block with ONE warp, lane i
// holding row i (and for LU also column i) in registers; the k-sums read the pivot row's
// entries with warp shuffles, so a column step costs c shuffles + FMAs and one sqrt /
// division, with no shared-memory round trips or barriers.  The finished block is
// published to shared memory and then every thread of the CTA runs an independent
// substitution for one row below the block (coalesced: the matrix is column-major) — or,
// for LU's U part, for one column to the right (staged through shared memory so the
// column's w contiguous entries are loaded and stored coalesced).
// The diagonal factorization is repeated by every CTA (~1-2 us) instead of a grid-wide
// dependency; the last CTA to have read it writes it out.
// All loads of data produced by other kernels bypass L1 (ld.global.cg): with the
// lookahead stream two kernels share SMs, and an SM's L1 may hold lines another kernel
// read before a third one rewrote them.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace sf {

constexpr int kLeafT = 128;
constexpr int kUCols = 64;   // U columns per CTA (static smem budget)
constexpr unsigned kFull = 0xffffffffu;


__device__ __forceinline__ void leaf_fail(long long* fail, long long col1) {
  atomicMin((unsigned long long*)fail, (unsigned long long)col1);
}

// True in exactly one CTA of the grid: the last one to arrive (all others have finished
// reading the diagonal block).  Resets the counter for the next launch on the stream.
__device__ __forceinline__ bool last_reader(long long* counter) {
  __shared__ int last;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd((unsigned long long*)counter, 1ull);
    last = (old == gridDim.x - 1);
    if (last) *counter = 0;
  }
  __syncthreads();
  return last;
}

// ------------------------------------------------------------------ Cholesky
// RIGHT-looking, the paper's per-element order.  Warp 0
// holds the diagonal block in registers (lane i = row i, a[k] = running A_ik); at column c
// lane c's a[c] is final, L_cc = sqrt(a[c]) is broadcast, every lane scales its a[c] by
// 1/L_cc, publishes L_ic to a shared vector, and subtracts L_ic L_jc from its a[j], j > c.
// Each entry thus receives  A_ij - L_i0 L_j0 - L_i1 L_j1 - ...  one term at a time in k
// order — exactly PAPER.md:59-64 ("L_ic -= L_ik L_ck" for k = z..c-1) — and the
// critical path of a column is one shuffle, sqrt, reciprocal, a shared store/load and ONE
// fma (the j = c+1 update): the remaining fmas are independent and overlap the next column.
// The division by L_cc is a multiplication by the warp-uniform 1/L_cc (<= 1 ulp apart,
// DESIGN.md reading P11): a per-lane division next to lane c's different branch cost
// ~500 cycles per column (calib/leaf_probe.cu: Crout 33.5K -> 18.2K cycles, w = 32).
// Rows below: the same right-looking order in registers (x_c *= 1/L_cc, x_j -= x_c L_jc),
// L stored transposed (Lt[c][j] = L_jc) so the broadcast operands of a column are
// contiguous (16-byte shared loads).
template <typename T, int W, int NT>
__global__ void __launch_bounds__(NT) chol_leaf_rl_kernel(int64_t m, int w, const T* __restrict__ src,
                                                              int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                              int64_t col0, long long* fail) {
  static_assert(W <= 32, "one row per lane");
  if (failed(fail)) return;
  __shared__ __align__(16) T Lt[W][W + 2];   // Lt[c][j] = L_jc (j >= c), 0 above
  __shared__ T inv[W];
  __shared__ T lc[2][W];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;
  if (warp == 0) {
    T a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k <= lane && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : T(0);
    int okc = 1;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (c < w) {
        const T d = __shfl_sync(kFull, a[c], c);
        if (!(d > T(0))) {
          okc = 0;
          if (lane == 0 && blockIdx.x == 0) leaf_fail(fail, col0 + c + 1);
          break;
        }
        const T ri = fast_rsqrt(d);                    // 1 / L_cc, warp-uniform (P11)
        const T Lcc = d * ri;                          // sqrt(d)
        const T l = (lane == c) ? Lcc : a[c] * ri;     // lanes < c: unused (upper part)
        a[c] = l;
        if (lane < W) { lc[c & 1][lane] = l; Lt[c][lane] = (lane >= c) ? l : T(0); }
        if (lane == c) inv[c] = ri;
        __syncwarp();
#pragma unroll
        for (int j = c + 1; j < W; ++j) a[j] = fma(-l, lc[c & 1][j], a[j]);   // row lane, col j (used iff j <= lane)
      } else {
        if (lane < W) Lt[c][lane] = T(0);
        if (lane == 0) inv[c] = T(0);
      }
    }
    if (lane == 0) bad = !okc;
  }
  T x[W];
  if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : T(0);
  }
  __syncthreads();
  if (bad) return;
  if (last_reader(fail + 1)) {
    for (int idx = tid; idx < w * w; idx += NT) {
      const int i = idx % w, k = idx / w;
      if (k <= i) dst[i + (int64_t)k * ldd] = Lt[k][i];
    }
  }
  if (r >= m) return;
#pragma unroll
  for (int c = 0; c < W; ++c) {
    x[c] = x[c] * inv[c];
#pragma unroll
    for (int j = c + 1; j < W; ++j) x[j] = fma(-x[c], Lt[c][j], x[j]);
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
  const int grid = below > 0 ? (int)((below + kLeafT - 1) / kLeafT) : 1;
  if (w <= 16) chol_leaf_rl_kernel<T, 16, kLeafT><<<grid, kLeafT, 0, st>>>(m, w, src, lds, dst, ldd, col0, fail);
  else if (w <= 32) chol_leaf_rl_kernel<T, 32, kLeafT><<<grid, kLeafT, 0, st>>>(m, w, src, lds, dst, ldd, col0, fail);
  else return cudaErrorInvalidValue;
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ LU
// ONE warp factors the diagonal block in registers while the other warps already load their
// rows below / stage their U columns; then one __syncthreads and the independent
// substitutions (the 32-wide leaf of lu_panel_rec with SF_LU_P64=0; panel64.cu is the
// default).
template <typename T, int W>
__global__ void __launch_bounds__(kLeafT) lu_leaf_warp_kernel(int64_t m, int64_t ncr, int w, const T* __restrict__ src,
                                                              int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                              int64_t col0, const T* tolp, long long* fail,
                                                              int nrow_blocks) {
  if (failed(fail)) return;
  constexpr int LW = W + 2;   // dynamic shared memory (about 50 KB for fp64)
  extern __shared__ __align__(16) unsigned char lusm[];
  T (*Lt)[LW] = reinterpret_cast<T (*)[LW]>(lusm);              // L11 transposed (Lt[k][i] = L_ik)
  T (*Us)[LW] = reinterpret_cast<T (*)[LW]>(lusm + sizeof(T) * W * LW);   // U11 (Us[k][j] = U_kj)
  T (*S)[W + 1] = reinterpret_cast<T (*)[W + 1]>(lusm + 2 * sizeof(T) * W * LW);   // U column staging
  __shared__ T inv[W];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowblock = (int)blockIdx.x < nrow_blocks;
  const int64_t r = w + (int64_t)blockIdx.x * kLeafT + tid;
  const int64_t j0 = w + (int64_t)(blockIdx.x - nrow_blocks) * kUCols;
  const int ncols = rowblock ? 0 : (int)((w + ncr - j0) < kUCols ? (w + ncr - j0) : kUCols);
  if (warp == 0) {
    // Right-looking in registers, the paper's per-element order (every
    // entry receives its -L_ik U_k* terms one at a time in k order): lane i holds row i of
    // the block; at column c lane c's a[c] is L_cc, lane c scales its row right of c by the
    // warp-uniform 1/L_cc (U_c*, reading P11) and publishes it, every lane below subtracts
    // L_ic U_cj.  Critical path per column: shuffle, reciprocal, one multiply, a shared
    // store/load and one fma (was: a c-term dot product and a per-lane division).
    __shared__ T uc[2][W];
    const T tol = __ldcg(tolp);
    T a[W];
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = (lane < w && k < w) ? __ldcg(src + lane + (int64_t)k * lds) : T(0);
    int okc = 1;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (c < w) {
        const T Lcc = __shfl_sync(kFull, a[c], c);
        if (!(fabs(Lcc) >= tol)) {
          okc = 0;
          if (lane == 0 && blockIdx.x == 0) leaf_fail(fail, col0 + c + 1);
          break;
        }
        const T ri = fast_rcp(Lcc);
        if (lane == c) {
          inv[c] = ri;
#pragma unroll
          for (int j = c + 1; j < W; ++j) { a[j] = a[j] * ri; uc[c & 1][j] = a[j]; }
        }
        __syncwarp();
        if (lane > c) {
          const T l = a[c];
#pragma unroll
          for (int j = c + 1; j < W; ++j) a[j] = fma(-l, uc[c & 1][j], a[j]);
        }
      } else if (lane == 0) {
        inv[c] = T(0);
      }
    }
    if (okc && lane < W) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        Lt[k][lane] = (k <= lane) ? a[k] : T(0);
        Us[lane][k] = (k > lane) ? a[k] : T(0);
      }
    }
    if (lane == 0) bad = !okc;
  } else if (!rowblock) {
    // warps 1..3 stage the U columns while warp 0 factors the block
    for (int jj = warp - 1; jj < ncols; jj += kLeafT / 32 - 1)
      if (lane < w) S[jj][lane] = __ldcg(src + lane + (j0 + jj) * lds);
  }
  T x[W];
  if (rowblock && r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) x[k] = (k < w) ? __ldcg(src + r + (int64_t)k * lds) : T(0);
  }
  __syncthreads();
  if (bad) return;
  if (last_reader(fail + 1)) {   // in-place safety: every CTA has read the diagonal block
    for (int idx = tid; idx < w * w; idx += kLeafT) {
      const int i = idx % w, k = idx / w;
      dst[i + (int64_t)k * ldd] = (k <= i) ? Lt[k][i] : Us[i][k];   // L incl. diagonal / U strict upper
    }
  }
  if (rowblock) {
    // L rows below: L_rc = A_rc - sum_{k<c} L_rk U_kc, right-looking (terms in k order)
    if (r >= m) return;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const T xc = x[c];
#pragma unroll
      for (int j = c + 1; j < W; ++j) x[j] = fma(-xc, Us[c][j], x[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) dst[r + (int64_t)k * ldd] = x[k];
    return;
  }
  // U columns to the right: U_cj = (A_cj - sum_{k<c} L_ck U_kj) / L_cc
  if (tid < ncols) {
    T y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) y[k] = (k < w) ? S[tid][k] : T(0);
#pragma unroll
    for (int c = 0; c < W; ++c) {   // right-looking: y_c *= 1/L_cc, then y_j -= L_jc y_c
      y[c] = y[c] * inv[c];
#pragma unroll
      for (int j = c + 1; j < W; ++j) y[j] = fma(-Lt[c][j], y[c], y[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) S[tid][k] = y[k];
  }
  __syncthreads();
  for (int jj = warp; jj < ncols; jj += kLeafT / 32)
    if (lane < w) dst[lane + (j0 + jj) * ldd] = S[jj][lane];
}

template <typename T>
cudaError_t lu_leaf(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                    const T* tol, long long* fail, cudaStream_t st) {
  if (w <= 0 || m <= 0) return cudaSuccess;
  const int64_t below = m - w;
  const int nrb = below > 0 ? (int)((below + kLeafT - 1) / kLeafT) : 0;
  const int ncb = ncr > 0 ? (int)((ncr + kUCols - 1) / kUCols) : 0;
  int grid = nrb + ncb;
  if (grid == 0) grid = 1;
  auto go = [&](auto kern, int W) -> cudaError_t {
    const size_t smem = sizeof(T) * ((size_t)2 * W * (W + 2) + (size_t)kUCols * (W + 1));
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kLeafT, smem, st>>>(m, ncr, w, src, lds, dst, ldd, col0, tol, fail, nrb);
    return cudaSuccess;
  };
  cudaError_t e;
  if (w <= 16) e = go(lu_leaf_warp_kernel<T, 16>, 16);
  else if (w <= 32) e = go(lu_leaf_warp_kernel<T, 32>, 32);
  else return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ LU, U rows only
// The U part of lu_leaf_warp_kernel against an ALREADY FACTORED diagonal block: L11 (w x w,
// lower incl. diagonal, at `l11`) is read, not recomputed.  Used by the block-cyclic
// distributed LU (dist.cu), where a rank holds the received L panel but not the original
// diagonal block: U_cj = (A_cj - sum_{k<c} L_ck U_kj) / L_cc for the
// ncols columns at src.
template <typename T, int W>
__global__ void __launch_bounds__(kLeafT) lu_usolve_kernel(int64_t ncols_total, int w, const T* __restrict__ l11,
                                                           int64_t ldl, const T* __restrict__ src, int64_t lds,
                                                           T* __restrict__ dst, int64_t ldd, const long long* fail) {
  if (failed(fail)) return;
  __shared__ T Ls[W][W + 1];
  __shared__ T inv[W];
  __shared__ T S[kUCols][W + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < W * W; idx += kLeafT) {
    const int c = idx % W, k = idx / W;
    Ls[c][k] = (c < w && k <= c) ? __ldcg(l11 + c + (int64_t)k * ldl) : T(0);
  }
  __syncthreads();
  if (tid < w) inv[tid] = T(1) / Ls[tid][tid];
  const int64_t j0 = (int64_t)blockIdx.x * kUCols;
  const int ncols = (int)((ncols_total - j0) < kUCols ? (ncols_total - j0) : kUCols);
  for (int jj = warp; jj < ncols; jj += kLeafT / 32)
    if (lane < w) S[jj][lane] = __ldcg(src + lane + (j0 + jj) * lds);
  __syncthreads();
  if (tid < ncols) {
    T y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) y[k] = (k < w) ? S[tid][k] : T(0);
#pragma unroll
    for (int c = 0; c < W; ++c) {
      T a0 = y[c], a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
      for (int k = 0; k < c; ++k) {
        if ((k & 3) == 0) a0 = fma(-Ls[c][k], y[k], a0);
        else if ((k & 3) == 1) a1 = fma(-Ls[c][k], y[k], a1);
        else if ((k & 3) == 2) a2 = fma(-Ls[c][k], y[k], a2);
        else a3 = fma(-Ls[c][k], y[k], a3);
      }
      y[c] = ((a0 + a1) + (a2 + a3)) * inv[c];
    }
#pragma unroll
    for (int k = 0; k < W; ++k) S[tid][k] = y[k];
  }
  __syncthreads();
  for (int jj = warp; jj < ncols; jj += kLeafT / 32)
    if (lane < w) dst[lane + (j0 + jj) * ldd] = S[jj][lane];
}

template <typename T>
cudaError_t lu_usolve_leaf(int64_t ncols, int w, const T* l11, int64_t ldl, const T* src, int64_t lds, T* dst,
                           int64_t ldd, const long long* fail, cudaStream_t st) {
  if (w <= 0 || ncols <= 0) return cudaSuccess;
  const int grid = (int)((ncols + kUCols - 1) / kUCols);
  if (w <= 16) lu_usolve_kernel<T, 16><<<grid, kLeafT, 0, st>>>(ncols, w, l11, ldl, src, lds, dst, ldd, fail);
  else if (w <= 32) lu_usolve_kernel<T, 32><<<grid, kLeafT, 0, st>>>(ncols, w, l11, ldl, src, lds, dst, ldd, fail);
  else return cudaErrorInvalidValue;
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ back substitution
// Upper-triangular solve T X = B for ncols right-hand sides in place, w <= W rows:
//   x_c = (y_c - sum_{k>c} T_ck x_k) / T_ck   (c descending; UNIT: no division)
// with T given by its storage: TRANS = 0 -> T_ck = t[c + k*ldt] (an upper factor: U, R);
// TRANS = 1 -> T_ck = t[k + c*ldt] (the transpose of a lower factor: L^T).  Columns staged
// through shared memory so each column's w contiguous entries move coalesced.  Used by the
// triangular solves with the factors (chol/lu/qr_solve).
template <typename T, int W, bool TRANS, bool UNIT>
__global__ void __launch_bounds__(kLeafT) trsm_upper_kernel(int64_t ncols_total, int w, const T* __restrict__ t,
                                                            int64_t ldt, T* __restrict__ B, int64_t ldb) {
  __shared__ T Ts[W][W + 1];
  __shared__ T inv[W];
  __shared__ T S[kUCols][W + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < W * W; idx += kLeafT) {
    const int c = idx % W, k = idx / W;
    T v = T(0);
    if (c < w && k < w && k >= c) v = TRANS ? __ldcg(t + k + (int64_t)c * ldt) : __ldcg(t + c + (int64_t)k * ldt);
    Ts[c][k] = v;
  }
  __syncthreads();
  if (!UNIT && tid < w) inv[tid] = T(1) / Ts[tid][tid];
  const int64_t j0 = (int64_t)blockIdx.x * kUCols;
  const int ncols = (int)((ncols_total - j0) < kUCols ? (ncols_total - j0) : kUCols);
  for (int jj = warp; jj < ncols; jj += kLeafT / 32)
    if (lane < w) S[jj][lane] = __ldcg(B + lane + (j0 + jj) * ldb);
  __syncthreads();
  if (tid < ncols) {
    T y[W];
#pragma unroll
    for (int k = 0; k < W; ++k) y[k] = (k < w) ? S[tid][k] : T(0);
#pragma unroll
    for (int c = W - 1; c >= 0; --c) {
      if (c < w) {
        T a0 = y[c], a1 = T(0);
#pragma unroll
        for (int k = c + 1; k < W; ++k) {
          if ((k & 1) == 0) a0 = fma(-Ts[c][k], y[k], a0);
          else a1 = fma(-Ts[c][k], y[k], a1);
        }
        y[c] = UNIT ? (a0 + a1) : (a0 + a1) * inv[c];
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) S[tid][k] = y[k];
  }
  __syncthreads();
  for (int jj = warp; jj < ncols; jj += kLeafT / 32)
    if (lane < w) B[lane + (j0 + jj) * ldb] = S[jj][lane];
}

template <typename T>
cudaError_t trsm_upper_leaf(int64_t ncols, int w, const T* t, int64_t ldt, int trans, int unit, T* B, int64_t ldb,
                            cudaStream_t st) {
  if (w <= 0 || ncols <= 0) return cudaSuccess;
  if (w > 32) return cudaErrorInvalidValue;
  const int grid = (int)((ncols + kUCols - 1) / kUCols);
#define SF_TRSM(TR, UN)                                                                                  \
  if (w <= 16) trsm_upper_kernel<T, 16, TR, UN><<<grid, kLeafT, 0, st>>>(ncols, w, t, ldt, B, ldb);      \
  else trsm_upper_kernel<T, 32, TR, UN><<<grid, kLeafT, 0, st>>>(ncols, w, t, ldt, B, ldb);
  if (trans && unit) { SF_TRSM(true, true) }
  else if (trans) { SF_TRSM(true, false) }
  else if (unit) { SF_TRSM(false, true) }
  else { SF_TRSM(false, false) }
#undef SF_TRSM
  count_launch();
  return cudaGetLastError();
}

template cudaError_t chol_leaf<double>(int64_t, int, const double*, int64_t, double*, int64_t, int64_t, long long*,
                                       cudaStream_t);
template cudaError_t chol_leaf<float>(int64_t, int, const float*, int64_t, float*, int64_t, int64_t, long long*,
                                      cudaStream_t);
template cudaError_t lu_leaf<double>(int64_t, int64_t, int, const double*, int64_t, double*, int64_t, int64_t,
                                     const double*, long long*, cudaStream_t);
template cudaError_t lu_leaf<float>(int64_t, int64_t, int, const float*, int64_t, float*, int64_t, int64_t,
                                    const float*, long long*, cudaStream_t);

template cudaError_t lu_usolve_leaf<double>(int64_t, int, const double*, int64_t, const double*, int64_t, double*,
                                            int64_t, const long long*, cudaStream_t);
template cudaError_t lu_usolve_leaf<float>(int64_t, int, const float*, int64_t, const float*, int64_t, float*, int64_t,
                                           const long long*, cudaStream_t);

template cudaError_t trsm_upper_leaf<double>(int64_t, int, const double*, int64_t, int, int, double*, int64_t,
                                             cudaStream_t);
template cudaError_t trsm_upper_leaf<float>(int64_t, int, const float*, int64_t, int, int, float*, int64_t,
                                            cudaStream_t);

}  // namespace sf
