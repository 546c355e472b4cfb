// kernels.h — internal launch interface between the drivers (driver.cu) and the kernels.
// Not part of the public C ABI (include/stepfact.h).  All matrices column-major.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tiles.cuh"

namespace sf {

// process-wide count of kernel launches enqueued by the library (sf_launch_counter)
void count_launch(int n = 1);


// C(MxN) = (beta ? Cin : 0) + alpha * op(A)(MxK) * op(B)(KxN)
//   op(A)(i,k) = a_kcontig ? A[k + i*lda] : A[i + k*lda]
//   op(B)(k,j) = b_kcontig ? B[k + j*ldb] : B[j + k*ldb]
//   mask: write only i >= j (lower) / i <= j (upper) of C
//   splits > 1: split-K with a fixed-order reduction through `work` (splits*M*N doubles)
struct GemmF64 {
  int64_t M, N, K;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  const double* Cin; int64_t ldcin;
  double* C; int64_t ldc;
  double alpha;
  int beta;
  int splits;
  double* work;
  const long long* fail;   // device "first failed column" word; kernels exit early if set
  int64_t off = 0;         // mask diagonal offset: lower keeps i >= j + off, upper i <= j + off
  Raster rs;               // tile rasterization (filled by the launcher)
  int max_ctas = 0;        // > 0: at most this many CTAs, each looping over tiles (leaves SMs free)
  int ntiles = 0;          // set by the launcher
};
cudaError_t gemm_f64(GemmF64 p, int a_kcontig, int b_kcontig, int mask, cudaStream_t st);

// Grouped launch: `count` independent blocks C_g(M_g x N_g) = Cin_g + alpha op(A_g) op(B_g),
// sharing K, lda/ldb/ldc/ldcin, alpha/beta and the mask (each with its own diagonal offset)
// — one grid for all of them (p's M, N, A, B, Cin, C, off are ignored; splits = 1).
struct GemmGroup {
  int64_t M, N, off;
  const double* A; const double* B; const double* Cin; double* C;
  int tile0;   // set by the launcher
};
constexpr int kMaxGroups = 16;
struct GemmGroups { int count; GemmGroup g[kMaxGroups]; };
cudaError_t gemm_f64_grouped(GemmF64 p, const GemmGroup* groups, int count, int a_kcontig, int b_kcontig, int mask,
                             cudaStream_t st);

// ---------------------------------------------------------------- fp32: 3xTF32 on tcgen05
// C(M x N) = Cin - A B^T with A, B given by their 3xTF32 split (x_hi, x_lo) in K-major
// layout (row i of A: K contiguous floats at Ah + i*ldk_a).  mask / off as for GemmF64.
// Bases 16-byte aligned, ldk multiples of 4 (TMA).
struct Tf32Gemm {
  int64_t M, N, K;
  const float* Ah; const float* Al; int64_t ldk_a;
  const float* Bh; const float* Bl; int64_t ldk_b;
  const float* Cin; int64_t ldcin;
  float* C; int64_t ldc;
  int mask; int64_t off;
  const long long* fail;
  float alpha = -1.f;   // C = (beta ? Cin : 0) + alpha * A B^T
  int beta = 1;
};
cudaError_t gemm_tf32x3(const Tf32Gemm& g, cudaStream_t st);
// column-major X (m x k, ld) -> K-major hi/lo split (row i at H + i*ldk)
cudaError_t split_tf32(int64_t m, int64_t k, const float* X, int64_t ld, float* H, float* L, int64_t ldk,
                       cudaStream_t st);
// K-major X (row i: k contiguous at X + i*ld) -> K-major hi/lo split (no transpose)
cudaError_t split_tf32_kmajor(int64_t m, int64_t k, const float* X, int64_t ld, float* H, float* L, int64_t ldk,
                              cudaStream_t st);

// ---------------------------------------------------------------- panels (templated T)
// Cholesky leaf (Alg. 1 inner loops) on columns [0,w) of the m x w block
// whose top-left corner is the diagonal entry (z',z').  src may equal dst.
// D = a op(X) + b op(Y) with zero padding outside each operand's extent (Strassen block sums)
template <typename T>
cudaError_t comb(int64_t rows, int64_t cols, T a, const T* X, int64_t ldx, int xkc, int64_t xr, int64_t xc, T b,
                 const T* Y, int64_t ldy, int ykc, int64_t yr, int64_t yc, T* D, int64_t ldd, cudaStream_t st);

template <typename T>
cudaError_t chol_leaf(int64_t m, int w, const T* src, int64_t lds, T* dst, int64_t ldd,
                      int64_t col0, long long* fail, cudaStream_t st);

// LU leaf (Alg. 2 inner loops): diagonal w x w block, the L rows below
// it (m-w rows) and the U columns right of it (ncols_right columns), all in place/out.
template <typename T>
cudaError_t lu_leaf(int64_t m, int64_t ncols_right, int w, const T* src, int64_t lds, T* dst,
                    int64_t ldd, int64_t col0, const T* tol, long long* fail, cudaStream_t st);

// Per-device chaining of persistent MGS grids across streams (panels.cu MgsOrder), for
// whole replayed QR graphs: wait before the launch, record after it.
void mgs_order_before(cudaStream_t st);
void mgs_order_after(cudaStream_t st);

// A whole panel of width w <= 64 in one launch (panel64.cu): LU — the diagonal block, the L
// rows below it and the U columns right of it (ncr columns); Cholesky — the diagonal block
// and the L rows below it.  Same arguments as lu_leaf / chol_leaf.
template <typename T>
cudaError_t lu_panel64(int64_t m, int64_t ncr, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                       const T* tol, long long* fail, cudaStream_t st);
// Whole Cholesky of a small matrix (n <= 256, s | 32) in one thread-block cluster, the
// matrix resident in shared memory (small.cu).
bool chol_small_applies(int64_t n, int64_t s, int elt);
cudaError_t chol_small(int64_t n, int64_t s, const double* A, int64_t lda, double* L, int64_t ldl, long long* fail,
                       cudaStream_t st);
// sph / spl (fp32 only, may be NULL): also write the 3xTF32 split (hi / lo) of the rows below
// the diagonal block, K-major with row stride spld, row r of the panel at sph + r*spld.
template <typename T>
cudaError_t chol_panel64(int64_t m, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                         long long* fail, cudaStream_t st, float* sph = nullptr, float* spl = nullptr,
                         int64_t spld = 0);

// LU U rows only, against an already factored diagonal block L11 (ldl): the U part of
// lu_leaf for ncols columns (block-cyclic distributed LU).
template <typename T>
cudaError_t lu_usolve_leaf(int64_t ncols, int w, const T* l11, int64_t ldl, const T* src, int64_t lds, T* dst,
                           int64_t ldd, const long long* fail, cudaStream_t st);

// Upper-triangular solve T X = B in place (ncols right-hand sides, w <= 32 rows): trans = 0:
// T_ck = t[c + k*ldt]; trans = 1: T_ck = t[k + c*ldt] (L^T of a lower L); unit: T_cc = 1.
template <typename T>
cudaError_t trsm_upper_leaf(int64_t ncols, int w, const T* t, int64_t ldt, int trans, int unit, T* B, int64_t ldb,
                            cudaStream_t st);

// QR panel, modified Gram-Schmidt (Alg. 3) on n x w columns.
template <typename T>
cudaError_t qr_mgs_panel(int64_t n, int w, const T* src, int64_t lds, T* dst, int64_t ldd,
                         int64_t col0, const T* tol, T* work, long long* fail, cudaStream_t st);
size_t qr_mgs_work_elems(int64_t n, int w, int elt);   // in units of the element type
int qr_mgs_max_width(int64_t n, int elt);   // widest panel the smem-resident MGS kernel takes

// utilities
template <typename T>
cudaError_t frob_norm_tol(int64_t n, const T* A, int64_t lda, T* tol_out, double* work, cudaStream_t st);  // work: 512 doubles
cudaError_t init_fail(long long* fail, cudaStream_t st);
cudaError_t finish_info(const long long* fail, int64_t* d_info, cudaStream_t st);
template <typename T>
cudaError_t zero_strict_lower(int64_t n, T* R, int64_t ldr, cudaStream_t st);
template <typename T>
cudaError_t copy_matrix(int64_t m, int64_t n, const T* src, int64_t lds, T* dst, int64_t ldd, cudaStream_t st);

}  // namespace sf
