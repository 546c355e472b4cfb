/*
 * stepfact.h — C ABI of libstepfact, a B200 (sm_100a) implementation of the step-s
 * Cholesky / LU / QR algorithms of C. Camarero, arXiv 1812.02056 ("the paper";
 * PAPER.md:<line> cites /root/reference/PAPER.md).
 *
 * Problem statement: given A, find triangular L (and U) with A = L L^T /
 * A = L U, or orthogonal Q and upper triangular R with A = Q R.  The step size s
 * is the number of columns factored between two trailing updates
 * ("flushes"): a flush fires when c = z + s and subtracts ONE
 * rectangular product from the trailing matrix.
 *
 * Conventions for every entry point
 *   - Matrices are column-major: element (i,j) of an n x n matrix X with leading
 *     dimension ldx >= n lives at X[i + j*ldx] (0-based i, j).  Pointers to device memory
 *     are prefixed d, host memory h.  The caller owns every matrix and the info word; the
 *     library owns only temporary workspace, taken from the CUDA stream-ordered allocator
 *     on `stream` and released before the call's work completes.
 *   - Device entry points are asynchronous and stream-ordered on `stream` (a
 *     cudaStream_t; NULL = the legacy default stream).  They never synchronize.
 *   - Numerical failure is NOT a return code: it is written, stream-ordered, to the device
 *     int64 *d_info: 0 = success, k >= 1 = the first (1-based) column
 *     at which the algorithm could not continue (see each function).  The outputs are then
 *     unspecified from the first column of the panel (step) containing column k on; the
 *     panels before it hold their final values (cf. LAPACK/cuSOLVER devInfo semantics).
 *   - Return codes (sf_status) report argument / resource / launch errors, synchronously;
 *     on SF_EINVAL nothing has been enqueued.  sf_last_error() gives a one-line detail.
 *   - dtype: SF_F64 (double storage and arithmetic; the update runs on the FP64 tensor
 *     cores, DMMA) or SF_F32 (float storage; see each function).
 *   - Alignment: any; 16-byte aligned pointers with even ld take the vectorised path.
 *   - Threads: every entry point may be called from any host thread; calls are serialized
 *     on the host while they enqueue (the library's side streams and caches are shared),
 *     the device work stays asynchronous.
 */
#ifndef STEPFACT_H
#define STEPFACT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sf_dtype { SF_F64 = 0, SF_F32 = 1 };
enum sf_status { SF_OK = 0, SF_EINVAL = 1, SF_ENOTSUP = 2, SF_ENOMEM = 3, SF_ECUDA = 4, SF_ENCCL = 5 };

/* Algorithm 1, "A fast Cholesky decomposition algorithm".
 *   n      order of A, n >= 1
 *   s      step size, 1 <= s <= n
 *   dA     n x n symmetric positive definite input, leading dimension lda >= n; ONLY its
 *          lower triangle (incl. diagonal) is read.  Read-only unless dA == dL.
 *   dL     n x n output, leading dimension ldl >= n: the lower triangle (incl. diagonal)
 *          receives L with A = L L^T and L_cc > 0; the strict upper triangle of dL is
 *          never written (so dA == dL factors in place, "could be done in
 *          place of A").  dL may alias dA only exactly (dA == dL, lda == ldl).
 *   d_info device int64: 0, or k if the value under the square root at column k
 *           was <= 0 or NaN.
 * Per panel p (columns [p*s, min((p+1)*s, n))): panel recurrences PAPER.md:53-67, then, if a
 * later panel exists, the flush A[c:n,c:n] -= R R^T with R = L[c:n, z:c),
 * lower triangle only (Alg. 1 never reads the upper part of A). */
int chol_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dL, int64_t ldl,
                int64_t* d_info, void* stream);

/* Algorithm 2, "A fast LU decomposition algorithm", no pivoting, Crout
 * normalisation: L lower triangular with its own diagonal, U unit upper triangular
 * (U_cc = L_cc / L_cc = 1 exactly).
 *   dA     n x n input with nonzero leading principal minors, read-only
 *          unless dA == dLU.
 *   dLU    n x n output: lower triangle incl. diagonal = L, strict upper triangle = U
 *          (the unit diagonal of U is implicit, not stored).  dLU == dA factors in place.
 *   d_info 0, or k if |L_kk| < 1e-12 * ||A||_F / n (||A||_F of the input; R3).
 * Flush: A[c:n,c:n] -= R_L R_U, R_L = L[c:n, z:c), R_U = U[z:c, c:n). */
int lu_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dLU, int64_t ldlu,
              int64_t* d_info, void* stream);

/* Algorithm 3, "A fast QR decomposition algorithm", modified
 * Gram-Schmidt inside the panel, block projection at each flush.
 *   dA     n x n input of full rank, read-only (it is needed again for R := Q^T A, :170)
 *   dQ     n x n output, orthonormal columns; also used as the working matrix M
 *          (columns < c hold Q, columns >= c hold M).  Must not alias dA.
 *   dR     n x n output: R = Q^T A on and above the diagonal, exact zeros below
 *          (R5).  Must not alias dA or dQ.
 *   d_info 0, or k if ||v_k|| < 1e-12 * ||A||_F / n (R3).
 * Flush: C = B_Q^T B_M, S = B_Q C, M[:, c:n] -= S over all rows. */
int qr_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dQ, int64_t ldq,
              void* dR, int64_t ldr, int64_t* d_info, void* stream);

/* Variable step: PAPER.md:194 notes that "the s parameter could be varied
 * during the execution".  steps[0..nsteps) is a HOST array of panel widths s_0, s_1, ...
 * (each >= 1; the last repeats if the sequence ends before column n; the final panel is
 * clipped at n): panel p covers [z_p, z_p + s_p) and is flushed (one rectangular product)
 * before panel p+1 — Algorithms 1-3 with the flush condition c = z + s_p (R11).
 * A constant sequence is the fixed-s call.  Everything else as for the fixed-s entry points. */
int chol_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dL,
                      int64_t ldl, int64_t* d_info, void* stream);
int lu_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dLU,
                    int64_t ldlu, int64_t* d_info, void* stream);
int qr_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dQ,
                    int64_t ldq, void* dR, int64_t ldr, int64_t* d_info, void* stream);

/* Solving with the factors ("used everywhere to solve linear systems",
 * PAPER.md:16): A X = B for nrhs right-hand sides, B (n x nrhs, column-major, ldb >= n,
 * device) overwritten by X.  Triangular solves by recursive halving: 32-row substitution
 * leaves plus tensor-core GEMMs for the couplings.  Stream-ordered; no pivoting, no
 * singularity checks (the factorization's info covers that).
 *   chol_solve: dL from chol_factor (lower triangle read): L Y = B, L^T X = Y.
 *   lu_solve:   dLU from lu_factor: L Y = B (L with its diagonal), U X = Y (U unit upper).
 *   qr_solve:   dQ, dR from qr_factor: X = R^-1 (Q^T B). */
int chol_solve(int64_t n, int64_t nrhs, int dtype, const void* dL, int64_t ldl, void* dB, int64_t ldb, void* stream);
int lu_solve(int64_t n, int64_t nrhs, int dtype, const void* dLU, int64_t ldlu, void* dB, int64_t ldb, void* stream);
int qr_solve(int64_t n, int64_t nrhs, int dtype, const void* dQ, int64_t ldq, const void* dR, int64_t ldr, void* dB,
             int64_t ldb, void* stream);

/* Host-buffer variants (the end-to-end path): same arguments with HOST matrices (pinned
 * memory recommended) and a host info word.  The library copies A to the device, runs
 * the factorization on an internal stream, copies the outputs back and synchronizes
 * before returning.  Outputs may alias the input exactly (in place).
 * chol_factor_host moves only the lower triangle (incl. diagonal), panel by panel, and
 * copies each panel of L back as soon as it is final, overlapped with the remaining
 * flushes.  The strict upper triangle of hL is unspecified out of place (entries inside the
 * s x s diagonal blocks receive A's values); in place (hL == hA) it keeps A's values.
 * lu_factor_host copies each panel's L columns and U rows back as soon as the panel is
 * factored, qr_factor_host each panel of Q (R, computed last, follows), overlapped with
 * the remaining work. */
int chol_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hL, int64_t ldl,
                     int64_t* info);
int lu_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hLU, int64_t ldlu,
                   int64_t* info);
int qr_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hQ, int64_t ldq,
                   void* hR, int64_t ldr, int64_t* info);

/* Building blocks — one call per hot-path step, exposed so
 * each step can be parity-tested and timed on its own.  All device, column-major,
 * stream-ordered; `fail`-style numerical errors go to *d_info as above (column indices
 * relative to the block's first column + col0).
 *
 * sf_chol_panel: PAPER.md:53-67 on the m x w block dP (top-left = the panel's diagonal
 *   entry), in place; the block's earlier-panel contributions must already be subtracted.
 * sf_syrk_sub:   PAPER.md:43-50: C(m x m, lower incl. diagonal) -= R R^T, R m x k.
 * sf_gemm_sub:   C(m x n) -= op(A) op(B), op(A)(i,k) = ta ? A[k + i*lda] : A[i + k*lda],
 *                op(B)(k,j) = tb ? B[j + k*ldb] : B[k + j*ldb]  (the LU/QR flush products).
 * sf_lu_panel:   PAPER.md:105-121 on the panel with top-left (z,z): m = n - z rows, w
 *   columns for L, and ncols_right = n - z - w further columns for U, in place.
 * sf_qr_panel:   PAPER.md:158-168, MGS of the n x w columns dV in place (-> Q columns). */
int sf_chol_panel(int64_t m, int64_t w, int dtype, void* dP, int64_t ld, int64_t col0, int64_t* d_info, void* stream);
int sf_syrk_sub(int64_t m, int64_t k, int dtype, const void* dR, int64_t ldr, void* dC, int64_t ldc, void* stream);
int sf_gemm_sub(int64_t m, int64_t n, int64_t k, int dtype, const void* dA, int64_t lda, int ta,
                const void* dB, int64_t ldb, int tb, void* dC, int64_t ldc, void* stream);
int sf_lu_panel(int64_t m, int64_t w, int64_t ncols_right, int dtype, void* dP, int64_t ld, int64_t col0,
                double tol, int64_t* d_info, void* stream);
int sf_qr_panel(int64_t n, int64_t w, int dtype, void* dV, int64_t ld, int64_t col0, double tol,
                int64_t* d_info, void* stream);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU, one process per GPU (BASELINE.json north_star (3)).
 *
 * Block-cyclic column layout: panel p (columns [p*s, min((p+1)*s, n)), the paper's step,
 * PAPER.md:31) lives on rank p % nranks at local slot p / nranks; a rank stores its panels
 * full height, column-major, side by side: local column (slot*s + k) is global column
 * (p*s + k), ld_local >= n, sf_local_cols(n, s, nranks, rank) columns in total.  Per panel
 * the owner factors it and broadcasts it; each rank then
 * applies the flush to the local columns right of it.
 * The results are the single-GPU results, distributed the same way.
 *
 * Communicators: sf_comm_init wraps an NCCL communicator (collective over the nranks
 * processes; rank 0 makes the id with sf_get_unique_id and ships it, e.g. through
 * torch.distributed).  sf_comm_init_loopback makes ONE process drive all nranks ranks on
 * its current device (each rank with its own buffers and streams; the broadcast is a device
 * copy) — the single-GPU test harness of the distributed schedule.
 *
 * Pointer arrays: the dist entry points take arrays with sf_comm_local_ranks(comm) entries
 * (1 for an NCCL communicator: this process's rank; nranks for loopback: rank 0..nranks-1),
 * each a DEVICE pointer to that rank's local storage or info word.  A rank with no columns
 * (nranks > number of panels) may pass NULL matrices.  d_info receives the GLOBAL first
 * failing column (all-reduce min over ranks), 0 on success.  Ownership, stream semantics
 * and error returns as for the single-GPU calls; NCCL failures return SF_ENCCL.
 * ------------------------------------------------------------------------------------- */
typedef struct sf_comm_* sf_comm_t;
int sf_get_unique_id(uint8_t id[128]);                                          /* NCCL id, rank 0 */
int sf_comm_init(sf_comm_t* comm, int nranks, int rank, const uint8_t id[128]);  /* collective; current device */
int sf_comm_init_loopback(sf_comm_t* comm, int nranks);
int sf_comm_destroy(sf_comm_t comm);
int sf_comm_size(sf_comm_t comm);
/* Panel transport.  on = 0 (default): the owner packs each factored panel
 * and it travels by ncclBroadcast (loopback: a device copy) on a communication stream.
 * on = 1: device-initiated push — ONE kernel on the owner's panel stream reads the factored
 * panel and stores it packed into every rank's receive buffer (NCCL: through the peers'
 * load/store pointers into a symmetric window, ncclMemAlloc + ncclCommWindowRegister,
 * allocated collectively at the first dist call that needs it and freed by
 * sf_comm_destroy), then raises each rank's ready flag (release); receivers wait on their
 * flag on the device before the flush and signal every rank when done with the buffer.
 * Cholesky and LU (QR keeps the broadcast of whole Q panels).  Same bytes, same results
 * (bitwise).  Every rank must set the same mode.  SF_EINVAL for a NULL comm, on not in
 * {0, 1}, or more than 16 ranks; NCCL window failures surface as SF_ENCCL at the dist call. */
int sf_comm_set_push(sf_comm_t comm, int on);
/* Payload bytes of every panel message this communicator has broadcast so far (cumulative):
 * panel p of a Cholesky / LU run sends rows [p*s, n) of its w columns, packed ((n - p*s) * w
 * elements; the last panel, never flushed, is not sent); QR sends whole Q panels (n * w).
 * -1 for a NULL comm. */
int64_t sf_comm_bcast_bytes(sf_comm_t comm);
int sf_comm_local_ranks(sf_comm_t comm);
int64_t sf_local_cols(int64_t n, int64_t s, int nranks, int rank);

/* Algorithm 1 distributed: dA_local[i] (input, lower triangle of the local columns read)
 * and dL_local[i] (output L, lower triangle; may equal dA_local[i] for in place). */
int chol_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dL_local,
                     int64_t ld_local, int64_t* const* d_info, void* stream);
/* Algorithm 2 distributed, Crout L (with diagonal) / unit U, packed as in lu_factor. */
int lu_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dLU_local,
                   int64_t ld_local, int64_t* const* d_info, void* stream);
/* Algorithm 3 distributed: local columns of Q and of R = Q^T A (exact zeros below the
 * diagonal).  Every rank keeps a full n x n copy of Q as workspace (R needs all of it). */
int qr_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dQ_local,
                   void* const* dR_local, int64_t ld_local, int64_t* const* d_info, void* stream);

/* Fast multiplication in the flush ("using a fast
 * rectangular matrix multiplication algorithm", 186-190: the paper used 2-3 recursions).
 * levels = L in 1..3: fp64 flushes whose two output sides are >= min_dim use Strassen-
 * Winograd (7 half-size products, operand/output block sums elementwise; uneven halves
 * zero-padded), the half-size products recursing while they still meet min_dim, at most L
 * levels deep — LU's A -= R_L R_U, QR's M -= B_Q C, and the off-diagonal half of Cholesky's
 * A -= R R^T.  levels = 0 (default): classical products only.  Process-wide, single-GPU
 * drivers, fp64; clears the library's captured CUDA graphs.  Rounding differs from the
 * classical product (normwise error bound, not componentwise).  Errors: SF_EINVAL if levels
 * not in 0..3 or min_dim < 64. */
int sf_set_strassen(int levels, int64_t min_dim);

/* Number of flushes the c = z+s schedule performs: floor((n-1)/s). */
int64_t sf_flush_count(int64_t n, int64_t s);
/* The schedule the drivers run (row a1; PAPER.md:36-52, 87-104, 139-157 and, for a step
 * sequence, PAPER.md:194 / reading R11): writes the 0-based columns c at which the flushes
 * fire (c = z + s_p, then z := c; never at c = n) to flush_cols[0 .. min(count, cap)) and
 * returns the count.  nsteps == 1: the fixed step steps[0] (the chol/lu/qr_factor schedule);
 * nsteps > 1: the *_factor_steps schedule, the last step repeating.  Host only, no GPU.
 * Returns -1 if n < 1, nsteps < 1, steps is NULL or a step is < 1; flush_cols may be NULL
 * when cap == 0. */
int64_t sf_schedule(int64_t n, int64_t nsteps, const int64_t* steps, int64_t* flush_cols, int64_t cap);
/* Cumulative number of kernel launches this library has enqueued in this process
 * (launch accounting for benchmarks: read it before and after a timed region). */
int64_t sf_launch_counter(void);

/* Profiling hook.  sf_profile_enable(1) makes the drivers record a CUDA event pair on the
 * factorization stream around every flush (kind 0: the trailing-update kernel launches),
 * every panel (kind 1), QR's R := Q^T A (kind 2) and, in the distributed drivers, every
 * NCCL panel broadcast on the rank's comm stream (kind 3).  sf_profile_collect synchronizes
 * on the recorded events and returns, per kind, total device milliseconds, number of
 * bracketed regions and the algorithmic flops they performed (SURVEY.md §8(d) formulas:
 * Cholesky flush s*m*(m+1), LU flush 2*s*m^2, QR flush 4*n*s*m, R n^2*(n+1); kind 3:
 * bytes); arrays of length 4; then it clears the record.  Not for use during graph capture. */
void sf_profile_enable(int on);
int sf_profile_collect(double* ms, int64_t* count, double* flops);
/* Per kind, the wall-clock milliseconds covered by the union of the regions the last
 * sf_profile_collect summed (regions on different streams may overlap: LU's lookahead flush
 * part on the panel stream beside the rest of the flush).  ms_union: 4 doubles.  SF_EINVAL
 * for NULL. */
int sf_profile_union(double* ms_union);

const char* sf_strerror(int status);
const char* sf_last_error(void);
int sf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STEPFACT_H */
