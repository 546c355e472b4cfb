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
//   1. warp 0: D11, right-looking in registers (2-D lane layout, see p64_factor_quarter):
//      per column c the pivot by one shuffle, its reciprocal, and a rank-1 update whose
//      operands arrive by 12 warp shuffles (no shared-memory round trip);
//   2. warp 1: the rows 32..w-1 of the block against U11 (L21); warp 2 (LU): the columns
//      32..w-1 against L11 (U12) — one forward substitution per lane;
//   3. all warps: D22 -= L21 U12 (Cholesky: L21 L21^T), terms one at a time in k order;
//   4. warp 0: D22 as in 1,
// while the CTA's own rows (or columns) are prefetched into L2.  Then each thread finishes its
// row of L (against U, right-looking: x_j -= x_c U_cj for c ascending — the paper's per-entry
// order of terms) or its column of U.  Reading P11: a division by L_cc is a
// multiplication by the (warp-uniform) reciprocal; in the LU diagonal block the update term
// L_ic U_cj is formed as (L_ic / L_cc) * (L_cc U_cj) — same terms, reassociated, <= 1 ulp.
// The last CTA to have read the diagonal block writes it (in-place safety).
// Loads of data produced by other kernels bypass L1 (ld.global.cg), see leaf.cu.
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace sf {

// SF_P64_TIMING (calib/p64_probe.cu only): CTA 0 thread 0 records %globaltimer at phase ends
#ifdef SF_P64_TIMING
__device__ unsigned long long p64_times[16];
__device__ unsigned long long p64_times_col[16];   // the first column-block CTA (blockIdx.x == nrb)
#define P64_T(k) do { if ((blockIdx.x == 0 || (int)blockIdx.x == nrb) && threadIdx.x == 0) { unsigned long long t; \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); (blockIdx.x == 0 ? p64_times : p64_times_col)[k] = t; } } while (0)
// [10] earliest CTA start, [11] latest thread end, [12] latest row-block end
#define P64_EDGE(k, op) do { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); \
  op(&p64_times[k], t); } while (0)
#else
#define P64_T(k) do {} while (0)
#define P64_EDGE(k, op) do {} while (0)
#endif

namespace p64 {
constexpr int NT = 128;     // threads per CTA = rows / columns per CTA
constexpr int W = 64;       // maximum panel width
constexpr int H = 32;       // quarter size
// Shared-memory matrices are W rows x DS columns: the substitution's register window covers
// columns c0 .. c0+63 (c0 <= 56), so rows are zero padded (to 120 columns; DS even keeps
// rows 16-byte aligned for paired loads).
constexpr int DS = W + 56 + 2;
constexpr unsigned kFull = 0xffffffffu;
}  // namespace p64

template <typename T> struct T2s;
template <> struct T2s<double> { using type = double2; };
template <> struct T2s<float> { using type = float2; };
template <typename T> using T2 = typename T2s<T>::type;

__device__ __forceinline__ void p64_fail(long long* fail, long long col1) {
  atomicMin((unsigned long long*)fail, (unsigned long long)col1);
}

__device__ __forceinline__ bool p64_last_reader(long long* counter) {
  __shared__ int last;
  if (threadIdx.x == 0) {
    // this CTA's reads of the diagonal block have completed (their values are in shared
    // memory), so no fence is needed before announcing it
    const unsigned long long old = atomicAdd((unsigned long long*)counter, 1ull);
    last = (old == gridDim.x - 1);
    if (last) *counter = 0;
  }
  __syncthreads();
  return last;
}

// Factor the H x H quarter D[o:o+H, o:o+H] in place with ONE warp, right-looking.  LU:
// D <- L (lower incl. diagonal) and U (strict upper, scaled by 1/L_cc); Cholesky: D <- L
// (lower incl. diagonal), upper part untouched.  inv[o+c] = 1 / L_cc.  Returns false (in
// every lane) on R3 failure, after recording column col0+o+c+1.
// 2-D register layout: lane = 4p + q holds the 4 x 8 block of rows 4p..4p+3, columns
// 8q..8q+7, so the rank-1 update of column c needs only 4 multipliers (from the lane holding
// column c of my rows) and 8 pivot-row entries (from the lane holding row c of my columns)
// by shuffle — 12 values instead of a whole row per lane.  Masked entries get a zero
// multiplier (fma(-0, u, a) == a exactly), so the update itself is branch-free.  The column
// loop is rolled in chunks of 8 (static register indices), and the reciprocal is a
// call-free Newton iteration (p64_rcp): an IEEE division subroutine would make the
// compiler save the whole register block around every call.
template <typename T, bool LU>
__device__ __forceinline__ bool p64_factor_quarter(T* D, T* inv, int o, int wq, T tol, int64_t col0, long long* fail,
                                                   int lane) {
  using namespace p64;
  const int p = lane >> 2, q = lane & 3;
  T blk[4][8];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) blk[ii][jj] = D[(o + 4 * p + ii) * DS + o + 8 * q + jj];
  int bad_col = -1;   // warp-uniform
#pragma unroll 1
  for (int cb = 0; cb < H / 8; ++cb) {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int c = 8 * cb + cc;
      const int pi = cc & 3, pr = 2 * cb + (cc >> 2);   // row c = 4 pr + pi, column c = 8 cb + cc
      const int src_d = 4 * pr + cb;
      const T d0 = __shfl_sync(kFull, blk[pi][cc], src_d);
      const bool live = c < wq;
      if (live && bad_col < 0 && (LU ? !(fabs(d0) >= tol) : !(d0 > T(0)))) bad_col = c;
      const T d = live ? d0 : T(1);
      T l[4], u[8];
      if (LU) {
        const T ri = fast_rcp(d);
        // multipliers L_ic of my rows (lane (p, cb)); pivot row U_cj = A_cj / L_cc of my
        // columns (lane (pr, q))
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) l[ii] = __shfl_sync(kFull, blk[ii][cc], 4 * p + cb);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) u[jj] = __shfl_sync(kFull, blk[pi][jj], 4 * pr + q) * ri;
        if (lane == src_d) inv[o + c] = live ? ri : T(0);
        if (p == pr) {   // row c keeps U_cj (scaled) right of the diagonal
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) blk[pi][jj] = (8 * q + jj > c) ? u[jj] : blk[pi][jj];
        }
      } else {
        const T ri = fast_rsqrt(d);   // 1 / L_cc
        const T Lcc = d * ri;
        // L_ic of my rows (lane (p, cb)); L_jc of my columns j = 8q + jj, row j held by lane
        // (2q + jj/4, cb) at row slot jj % 4
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) l[ii] = __shfl_sync(kFull, blk[ii][cc], 4 * p + cb) * ri;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) u[jj] = __shfl_sync(kFull, blk[jj & 3][cc], 4 * (2 * q + (jj >> 2)) + cb) * ri;
        if (lane == src_d) inv[o + c] = live ? ri : T(0);
        if (q == cb) {   // column c keeps L_ic below the diagonal, L_cc on it
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int i = 4 * p + ii;
            blk[ii][cc] = (i > c) ? l[ii] : (i == c ? Lcc : blk[ii][cc]);
          }
        }
      }
      // rank-1 update of rows i > c, columns j > c (Cholesky: j <= i)
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) l[ii] = (4 * p + ii > c) ? l[ii] : T(0);
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) u[jj] = (8 * q + jj > c) ? u[jj] : T(0);
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (LU || 8 * q + jj <= 4 * p + ii) blk[ii][jj] = fma(-l[ii], u[jj], blk[ii][jj]);
        }
    }
  }
  const bool ok = bad_col < 0;
  if (!ok && lane == 0 && blockIdx.x == 0) p64_fail(fail, col0 + o + bad_col + 1);
  if (ok) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (LU || 8 * q + jj <= 4 * p + ii) D[(o + 4 * p + ii) * DS + o + 8 * q + jj] = blk[ii][jj];
  }
  return ok;
}

// One 8-column block of the row / column substitution (see the kernel): x[0..JN) is the
// register window for columns c0..c0+JN-1; on return it has moved on by 8 columns.
template <typename T, int JN>
__device__ __forceinline__ void p64_subst_block(T (&x)[p64::W], const T* Op, const T* inv, bool use_u, int c0, int w,
                                                T* out, int64_t ostride, float* sh = nullptr, float* sl = nullptr) {
  using namespace p64;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const T* Mr = Op + (c0 + c) * DS + c0;   // 16-byte aligned (DS, c0 even)
    if (!use_u) x[c] = x[c] * inv[c0 + c];
    if ((c + 1) & 1) x[c + 1] = fma(-x[c], Mr[c + 1], x[c + 1]);
#pragma unroll
    for (int jj = (c + 2) & ~1; jj < JN; jj += 2) {
      const T2<T> mv = *reinterpret_cast<const T2<T>*>(Mr + jj);
      x[jj] = fma(-x[c], mv.x, x[jj]);
      x[jj + 1] = fma(-x[c], mv.y, x[jj + 1]);
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c0 + c < w) out[(int64_t)(c0 + c) * ostride] = x[c];
  if constexpr (std::is_same<T, float>::value) {
    // fp32 Cholesky rows: the 3xTF32 split of the final values, K-major (what split_tf32
    // would produce from `out` afterwards, computed from the same registers)
    if (sh) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c0 + c < w) {
          const float hi = tf32_rna(x[c]);
          sh[c0 + c] = hi;
          sl[c0 + c] = tf32_rna(x[c] - hi);
        }
    }
  }
#pragma unroll
  for (int j = 0; j < JN - 8; ++j) x[j] = x[j + 8];
#pragma unroll
  for (int j = JN - 8; j < JN; ++j) x[j] = T(0);
}

// One launch per panel of width w <= 64.  LU: rows [0, m) from the diagonal down, ncr
// columns of U right of the panel; Cholesky: ncr = 0.  Blocks [0, nrb) own 128 rows below
// the diagonal block each, blocks [nrb, grid) 128 columns of U each.
template <typename T, bool LU>
__global__ void __launch_bounds__(p64::NT) panel64_kernel(int64_t m, int64_t ncr, int w, const T* __restrict__ src,
                                                          int64_t lds, T* __restrict__ dst, int64_t ldd, int64_t col0,
                                                          const T* tolp, long long* fail, int nrb, float* sph,
                                                          float* spl, int64_t spld) {
  using namespace p64;
  if (threadIdx.x == 0) P64_EDGE(10, atomicMin);
  if (failed(fail)) return;
  extern __shared__ __align__(16) unsigned char p64_dyn[];
  T* D = reinterpret_cast<T*>(p64_dyn);            // the diagonal block, W x DS (zero padded)
  T* Mt = D + W * DS;                              // L^T for the L-against-L^T substitutions
  __shared__ T inv[W];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowblock = (int)blockIdx.x < nrb;
  const int64_t r = w + (int64_t)blockIdx.x * NT + tid;                       // my row (row blocks)
  const int64_t jc = w + (int64_t)((int)blockIdx.x - nrb) * NT + tid;         // my U column (column blocks)
  const bool mine = rowblock ? r < m : jc < w + ncr;
  // which operator the substitution applies: U (LU rows) or L^T (LU columns, Cholesky rows)
  const bool use_u = LU && rowblock;

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
  {
    // the diagonal block (column j: lanes over rows, coalesced), then the zero padding
    T v[W / 4][2];
#pragma unroll
    for (int jj = 0; jj < W / 4; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h, j = warp + 4 * jj;
        v[jj][h] = (i < w && j < w && (LU || j <= i)) ? __ldcg(src + i + (int64_t)j * lds) : T(0);
      }
#pragma unroll
    for (int jj = 0; jj < W / 4; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) D[(lane + 32 * h) * DS + warp + 4 * jj] = v[jj][h];
    for (int i = warp; i < W; i += NT / 32)
      for (int j = W + lane; j < DS; j += 32) D[i * DS + j] = T(0);
  }
  const T tol = LU ? __ldcg(tolp) : T(0);
  if (tid < W) inv[tid] = T(0);
  if (tid == 0) bad = 0;
  P64_T(0);
  __syncthreads();
  P64_T(1);

  const int w1 = w < H ? w : H, w2 = w - w1;
  // 1.-4.: the two diagonal quarters share ONE copy of the quarter code (a rolled loop): the
  // second pass finds it in the instruction cache
#pragma unroll 1
  for (int qi = 0; qi < 2; ++qi) {
    if (qi == 1) {
      if (w2 <= 0) break;
      // 2. L21 = D21 U11^-1 (LU) / D21 L11^-T (Cholesky): lane = row 32 + lane
      if (warp == 1) {
        T y[H];
        T* row = D + (H + lane) * DS;
#pragma unroll
        for (int k = 0; k < H; ++k) y[k] = row[k];
#pragma unroll
        for (int c = 0; c < H; ++c) {
          if (!LU) y[c] = y[c] * inv[c];
#pragma unroll
          for (int j = c + 1; j < H; ++j) y[j] = fma(-y[c], LU ? D[c * DS + j] : D[j * DS + c], y[j]);
        }
        if (lane < w2) {
#pragma unroll
          for (int k = 0; k < H; ++k) row[k] = y[k];
        }
      } else if (LU && warp == 2) {
        // U12 = L11^-1 D12, scaled: lane = column 32 + lane
        T y[H];
#pragma unroll
        for (int k = 0; k < H; ++k) y[k] = D[k * DS + H + lane];
#pragma unroll
        for (int c = 0; c < H; ++c) {
          y[c] = y[c] * inv[c];
#pragma unroll
          for (int k = c + 1; k < H; ++k) y[k] = fma(-D[k * DS + c], y[c], y[k]);
        }
        if (lane < w2) {
#pragma unroll
          for (int k = 0; k < H; ++k) D[k * DS + H + lane] = y[k];
        }
      }
      __syncthreads();
      P64_T(3);
      // 3. D22 -= L21 U12 (Cholesky: L21 L21^T, lower part), one term at a time in k order;
      //    lane = column (contiguous across the warp), rows warp-uniform (broadcast operands);
      //    the k loop is rolled (one short body)
      {
        T v[H * H / NT];
        const int j = lane;
#pragma unroll
        for (int e = 0; e < H * H / NT; ++e) v[e] = D[(H + warp + 4 * e) * DS + H + j];
#pragma unroll 1
        for (int k = 0; k < H; ++k) {
          const T ukj = LU ? D[k * DS + H + j] : D[(H + j) * DS + k];
#pragma unroll
          for (int e = 0; e < H * H / NT; ++e) v[e] = fma(-D[(H + warp + 4 * e) * DS + k], ukj, v[e]);
        }
#pragma unroll
        for (int e = 0; e < H * H / NT; ++e) {
          const int i = warp + 4 * e;
          if (i < w2 && j < w2 && (LU || j <= i)) D[(H + i) * DS + H + j] = v[e];
        }
      }
      __syncthreads();
      P64_T(4);
    }
    if (warp == 0 && !p64_factor_quarter<T, LU>(D, inv, H * qi, qi ? w2 : w1, tol, col0, fail, lane) && lane == 0)
      bad = 1;
    __syncthreads();
    if (qi == 0) P64_T(2);
    if (bad) return;
  }
  P64_T(5);
  // 5. L^T for the substitutions that need it: Mt[k][j] = L_jk (j > k), zero elsewhere
  if (!use_u) {
    if (tid < DS) {
#pragma unroll 4
      for (int k = 0; k < W; ++k) Mt[k * DS + tid] = (tid > k && tid < W) ? D[tid * DS + k] : T(0);
    }
    __syncthreads();
  }
  P64_T(6);
  if (p64_last_reader(fail + 1)) {
    for (int idx = tid; idx < w * w; idx += NT) {
      const int i = idx % w, k = idx / w;
      if (LU || k <= i) dst[i + (int64_t)k * ldd] = D[i * DS + k];
    }
  }
  P64_T(7);
  if (!mine) return;
  // my row r (x_k = A_rk) or my U column jc (x_k = A_kjc), k < w
  T x[W];
#pragma unroll
  for (int k = 0; k < W; ++k)
    x[k] = (k < w) ? (rowblock ? __ldcg(src + r + (int64_t)k * lds) : __ldcg(src + k + jc * lds)) : T(0);
  P64_T(8);
  // right-looking substitution, terms one at a time in k order (x_j -= x_k M_kj for k
  // ascending; M = U for LU rows, L^T otherwise, whose x_k is first scaled by 1/L_kk), in
  // blocks of 8 columns: the register window x[] holds columns c0..c0+63 and rotates by 8
  // per block, so a loop body is one block's code (a fully unrolled 64-column substitution
  // is several thousand instructions executed once).  Blocks with c0 >= 32 only touch the
  // window's first 32 columns (the rest is past the panel) and run a half-width body.
  const T* Op = use_u ? D : Mt;
  T* out = rowblock ? dst + r : dst + jc * ldd;
  const int64_t ostride = rowblock ? ldd : 1;
  const int nb = (w + 7) / 8;
  const int nb1 = nb < 4 ? nb : 4;
  // fp32 Cholesky: this row's split (hi / lo, K-major, row r of the panel below the block)
  float* sh = (!LU && rowblock && sph) ? sph + r * spld : nullptr;
  float* sl = sh ? spl + r * spld : nullptr;
#pragma unroll 1
  for (int b = 0; b < nb1; ++b) p64_subst_block<T, 64>(x, Op, inv, use_u, 8 * b, w, out, ostride, sh, sl);
#pragma unroll 1
  for (int b = 4; b < nb; ++b) p64_subst_block<T, 32>(x, Op, inv, use_u, 8 * b, w, out, ostride, sh, sl);
  P64_T(9);
  P64_EDGE(11, atomicMax);
  if (rowblock) P64_EDGE(12, atomicMax);
}

template <typename T, bool LU>
static cudaError_t launch_panel64(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd,
                                  int64_t col0, const T* tol, long long* fail, cudaStream_t st, float* sph = nullptr,
                                  float* spl = nullptr, int64_t spld = 0) {
  if (w <= 0 || m <= 0) return cudaSuccess;
  if (w > p64::W) return cudaErrorInvalidValue;
  const int64_t below = m - w;
  const int nrb = below > 0 ? (int)((below + p64::NT - 1) / p64::NT) : 0;
  const int ncb = (LU && ncr > 0) ? (int)((ncr + p64::NT - 1) / p64::NT) : 0;
  int grid = nrb + ncb;
  if (grid == 0) grid = 1;
  constexpr size_t dyn = sizeof(T) * 2 * p64::W * p64::DS;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(panel64_kernel<T, LU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  panel64_kernel<T, LU><<<grid, p64::NT, dyn, st>>>(m, LU ? ncr : 0, w, src, lds, dst, ldd, col0, tol, fail, nrb, sph,
                                                     spl, spld);
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
                         long long* fail, cudaStream_t st, float* sph, float* spl, int64_t spld) {
  return launch_panel64<T, false>(m, 0, w, src, lds, dst, ldd, col0, nullptr, fail, st, sph, spl, spld);
}

template cudaError_t lu_panel64<double>(int64_t, int64_t, int, const double*, int64_t, double*, int64_t, int64_t,
                                        const double*, long long*, cudaStream_t);
template cudaError_t lu_panel64<float>(int64_t, int64_t, int, const float*, int64_t, float*, int64_t, int64_t,
                                       const float*, long long*, cudaStream_t);
template cudaError_t chol_panel64<double>(int64_t, int, const double*, int64_t, double*, int64_t, int64_t, long long*,
                                          cudaStream_t, float*, float*, int64_t);
template cudaError_t chol_panel64<float>(int64_t, int, const float*, int64_t, float*, int64_t, int64_t, long long*,
                                         cudaStream_t, float*, float*, int64_t);

}  // namespace sf
