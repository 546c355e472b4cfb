// panel64.cu — a whole panel of width w <= 64 in ONE launch.
//
// LU, Crout form, for each column c of the panel:
//     L_ic = A_ic - sum_{k<c} L_ik U_kc   (i >= c),   U_ci = (A_ci - sum_{k<c} L_ck U_ki) / L_cc  (i > c)
// Cholesky:
//     L_cc = sqrt(A_cc - sum_{k<c} L_ck^2),    L_ic = (A_ic - sum_{k<c} L_ik L_ck) / L_cc
// where k runs over the panel's earlier columns (earlier panels were applied by the flushes).
//
// Why one launch.  The recursive panel (drv.cuh lu_panel_rec / chol_panel_rec) factors a
// 64-wide panel as leaf(32) -> GEMM -> [GEMM] -> leaf(32): four dependent launches, each
// waiting for a flush CTA to retire before it gets an SM (the lookahead panel runs beside
// flush part 2), then paying its launch and cold instruction fetch.  For narrow panels
// (cfg2 LU: s = 64) that chain IS the critical path of the factorization.
//
// Structure.  Grid = row blocks (128 rows of L below the panel's diagonal block each) +
// column blocks (LU only: 128 columns of U right of the panel each).  Every CTA factors the
// w x w diagonal block itself in shared memory (no grid-wide dependency; identical
// operations in every CTA, so identical bits), blocked 2 x 2 in 32 x 32 quarters:
//   1. warp 0: D11, right-looking in registers (lane = row; per column one shuffle, one
//      reciprocal, one broadcast row and one fma per entry — DESIGN.md reading P11);
//   2. warp 1: the rows 32..w-1 of the block against U11 (L21); warp 2 (LU): the columns
//      32..w-1 against L11 (U12) — one forward substitution per lane;
//   3. all warps: D22 -= L21 U12 (Cholesky: L21 L21^T), terms one at a time in k order;
//   4. warp 0: D22 as in 1.
// while the CTA's own rows (or columns) are prefetched into L2.  Then each thread finishes its row (L_i* against U, right-looking: x_j -= x_c U_cj
// for c ascending, i.e. the paper's per-element order of terms) or its column of U.  Every
// entry receives the same terms in the same k order as the paper's loops (grouping-free);
// only the reciprocal multiply (P11) and fma rounding differ from the oracle.
// The last CTA to have read the diagonal block writes it (in-place safety).
// Loads of data produced by other kernels bypass L1 (ld.global.cg), see leaf.cu.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace sf {

namespace p64 {
constexpr int NT = 128;     // threads per CTA = rows / columns per CTA
constexpr int W = 64;       // maximum panel width
constexpr int H = 32;       // quarter size
constexpr int LD = W + 2;   // smem row stride (16-byte aligned rows)
constexpr unsigned kFull = 0xffffffffu;
}  // namespace p64

template <typename T> __device__ __forceinline__ T p64_sqrt(T x);
template <> __device__ __forceinline__ double p64_sqrt<double>(double x) { return sqrt(x); }
template <> __device__ __forceinline__ float p64_sqrt<float>(float x) { return sqrtf(x); }

__device__ __forceinline__ void p64_fail(long long* fail, long long col1) {
  atomicMin((unsigned long long*)fail, (unsigned long long)col1);
}

__device__ __forceinline__ bool p64_last_reader(long long* counter) {
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

// Factor the H x H quarter D[o:o+H, o:o+H] in place with warp `warp` (lane = row o+lane),
// right-looking.  LU: D <- L (lower incl. diagonal) and U (strict upper, scaled by 1/L_cc);
// Cholesky: D <- L (lower incl. diagonal), upper part untouched.  inv[o+c] = 1 / L_cc.
// Returns false (in every lane) on R3 failure, after recording column col0+o+c+1.
template <typename T, bool LU>
__device__ __forceinline__ bool p64_factor_quarter(T (*D)[p64::LD], T* inv, T (*buf)[p64::H], int o, int wq,
                                                   T tol, int64_t col0, long long* fail, int lane) {
  using namespace p64;
  T a[H];
#pragma unroll
  for (int k = 0; k < H; ++k) a[k] = D[o + lane][o + k];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < H; ++c) {
    if (c < wq) {
      const T d = __shfl_sync(kFull, a[c], c);
      if (LU ? !(fabs(d) >= tol) : !(d > T(0))) {
        ok = false;
        if (lane == 0 && blockIdx.x == 0) p64_fail(fail, col0 + o + c + 1);
        break;
      }
      if (LU) {
        const T ri = T(1) / d;
        if (lane == c) {
          inv[o + c] = ri;
#pragma unroll
          for (int j = c + 1; j < H; ++j) { a[j] = a[j] * ri; buf[c & 1][j] = a[j]; }
        }
        __syncwarp();
        if (lane > c) {
          const T l = a[c];
#pragma unroll
          for (int j = c + 1; j < H; ++j) a[j] = fma(-l, buf[c & 1][j], a[j]);
        }
      } else {
        const T Lcc = p64_sqrt(d);
        const T ri = T(1) / Lcc;
        const T l = (lane == c) ? Lcc : a[c] * ri;
        a[c] = l;
        buf[c & 1][lane] = l;
        if (lane == c) inv[o + c] = ri;
        __syncwarp();
        if (lane > c) {
#pragma unroll
          for (int j = c + 1; j < H; ++j) a[j] = fma(-l, buf[c & 1][j], a[j]);
        }
      }
    }
  }
  if (ok) {
#pragma unroll
    for (int k = 0; k < H; ++k)
      if (LU || k <= lane) D[o + lane][o + k] = a[k];
  }
  return __all_sync(kFull, ok);
}

// One launch per panel of width w <= 64.  LU: rows [0, m) from the diagonal down, ncr
// columns of U right of the panel; Cholesky: ncr = 0.  Blocks [0, nrb) own 128 rows below
// the diagonal block each, blocks [nrb, grid) 128 columns of U each.
template <typename T, bool LU>
__global__ void __launch_bounds__(p64::NT) panel64_kernel(int64_t m, int64_t ncr, int w, const T* __restrict__ src,
                                                          int64_t lds, T* __restrict__ dst, int64_t ldd, int64_t col0,
                                                          const T* tolp, long long* fail, int nrb) {
  using namespace p64;
  if (failed(fail)) return;
  __shared__ __align__(16) T D[W][LD];
  __shared__ T inv[W];
  __shared__ T buf[2][H];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowblock = (int)blockIdx.x < nrb;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;                       // my row (row blocks)
  const int64_t jc = w + (int64_t)((int)blockIdx.x - nrb) * NT + tid;         // my U column (column blocks)
  const bool mine = rowblock ? r < m : jc < w + ncr;

  // warm L2 with this CTA's rows / columns (512 lines of 128 B) while the diagonal block is
  // factored; they are loaded into registers after it (holding them through the diagonal
  // steps would spill)
  for (int l = tid; l < 512; l += NT) {
    if (rowblock) {
      const int k = l >> 3;   // column k, 16-row line (l & 7) of this CTA's 128 rows
      const int64_t rr = w + (int64_t)blockIdx.x * NT + (l & 7) * 16;
      if (k < w && rr < m) prefetch_l2(src + rr + (int64_t)k * lds);
    } else {
      const int64_t j = w + (int64_t)((int)blockIdx.x - nrb) * NT + (l >> 2);   // column, 16-row line (l & 3)
      if (j < w + ncr && (l & 3) * 16 < w) prefetch_l2(src + (l & 3) * 16 + j * lds);
    }
  }
  for (int idx = tid; idx < W * W; idx += NT) {
    const int i = idx % W, j = idx / W;
    D[i][j] = (i < w && j < w && (LU || j <= i)) ? __ldcg(src + i + (int64_t)j * lds) : T(0);
  }
  const T tol = LU ? __ldcg(tolp) : T(0);
  if (tid < W) inv[tid] = T(0);
  if (tid == 0) bad = 0;
  __syncthreads();

  const int w1 = w < H ? w : H, w2 = w - w1;
  // 1. D11
  if (warp == 0 && !p64_factor_quarter<T, LU>(D, inv, buf, 0, w1, tol, col0, fail, lane) && lane == 0) bad = 1;
  __syncthreads();
  if (bad) return;
  if (w2 > 0) {
    // 2. L21 = D21 U11^-1 (LU) / D21 L11^-T (Cholesky): lane = row 32 + lane
    if (warp == 1) {
      T y[H];
#pragma unroll
      for (int k = 0; k < H; ++k) y[k] = D[H + lane][k];
#pragma unroll
      for (int c = 0; c < H; ++c) {
        if (!LU) y[c] = y[c] * inv[c];
#pragma unroll
        for (int j = c + 1; j < H; ++j) y[j] = fma(-y[c], LU ? D[c][j] : D[j][c], y[j]);
      }
      if (lane < w2) {
#pragma unroll
        for (int k = 0; k < H; ++k) D[H + lane][k] = y[k];
      }
    } else if (LU && warp == 2) {
      // U12 = L11^-1 D12, scaled: lane = column 32 + lane
      T y[H];
#pragma unroll
      for (int k = 0; k < H; ++k) y[k] = D[k][H + lane];
#pragma unroll
      for (int c = 0; c < H; ++c) {
        y[c] = y[c] * inv[c];
#pragma unroll
        for (int k = c + 1; k < H; ++k) y[k] = fma(-D[k][c], y[c], y[k]);
      }
      if (lane < w2) {
#pragma unroll
        for (int k = 0; k < H; ++k) D[k][H + lane] = y[k];
      }
    }
    __syncthreads();
    // 3. D22 -= L21 U12 (Cholesky: L21 L21^T, lower part), one term at a time in k order
#pragma unroll
    for (int e = 0; e < H * H / NT; ++e) {
      const int idx = tid + e * NT, i = idx % H, j = idx / H;
      if (i < w2 && j < w2 && (LU || j <= i)) {
        T v = D[H + i][H + j];
#pragma unroll
        for (int k = 0; k < H; ++k) v = fma(-D[H + i][k], LU ? D[k][H + j] : D[H + j][k], v);
        D[H + i][H + j] = v;
      }
    }
    __syncthreads();
    // 4. D22
    if (warp == 0 && !p64_factor_quarter<T, LU>(D, inv, buf, H, w2, tol, col0, fail, lane) && lane == 0) bad = 1;
    __syncthreads();
    if (bad) return;
  }
  if (p64_last_reader(fail + 1)) {
    for (int idx = tid; idx < w * w; idx += NT) {
      const int i = idx % w, k = idx / w;
      if (LU || k <= i) dst[i + (int64_t)k * ldd] = D[i][k];
    }
  }
  if (!mine) return;
  T x[W];
#pragma unroll
  for (int k = 0; k < W; ++k)
    x[k] = (k < w) ? (rowblock ? __ldcg(src + r + (int64_t)k * lds) : __ldcg(src + k + jc * lds)) : T(0);
  if (rowblock) {
    // row r: L_rc = A_rc - sum_{k<c} L_rk U_kc (Cholesky: (A_rc - sum L_rk L_ck) / L_cc)
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (!LU) x[c] = x[c] * inv[c];
#pragma unroll
      for (int j = c + 1; j < W; ++j) x[j] = fma(-x[c], LU ? D[c][j] : D[j][c], x[j]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) dst[r + (int64_t)k * ldd] = x[k];
  } else {
    // U column jc: U_cj = (A_cj - sum_{k<c} L_ck U_kj) / L_cc
#pragma unroll
    for (int c = 0; c < W; ++c) {
      x[c] = x[c] * inv[c];
#pragma unroll
      for (int k = c + 1; k < W; ++k) x[k] = fma(-D[k][c], x[c], x[k]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) dst[k + jc * ldd] = x[k];
  }
}

template <typename T, bool LU>
static cudaError_t launch_panel64(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd,
                                  int64_t col0, const T* tol, long long* fail, cudaStream_t st) {
  if (w <= 0 || m <= 0) return cudaSuccess;
  if (w > p64::W) return cudaErrorInvalidValue;
  const int64_t below = m - w;
  const int nrb = below > 0 ? (int)((below + p64::NT - 1) / p64::NT) : 0;
  const int ncb = (LU && ncr > 0) ? (int)((ncr + p64::NT - 1) / p64::NT) : 0;
  int grid = nrb + ncb;
  if (grid == 0) grid = 1;
  panel64_kernel<T, LU><<<grid, p64::NT, 0, st>>>(m, LU ? ncr : 0, w, src, lds, dst, ldd, col0, tol, fail, nrb);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t lu_panel64(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                       const T* tol, long long* fail, cudaStream_t st) {
  return launch_panel64<T, true>(m, ncr, w, src, lds, dst, ldd, col0, tol, fail, st);
}
template <typename T>
cudaError_t chol_panel64(int64_t m, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                         long long* fail, cudaStream_t st) {
  return launch_panel64<T, false>(m, 0, w, src, lds, dst, ldd, col0, nullptr, fail, st);
}

template cudaError_t lu_panel64<double>(int64_t, int64_t, int, const double*, int64_t, double*, int64_t, int64_t,
                                        const double*, long long*, cudaStream_t);
template cudaError_t lu_panel64<float>(int64_t, int64_t, int, const float*, int64_t, float*, int64_t, int64_t,
                                       const float*, long long*, cudaStream_t);
template cudaError_t chol_panel64<double>(int64_t, int, const double*, int64_t, double*, int64_t, int64_t, long long*,
                                          cudaStream_t);
template cudaError_t chol_panel64<float>(int64_t, int, const float*, int64_t, float*, int64_t, int64_t, long long*,
                                         cudaStream_t);

}  // namespace sf
