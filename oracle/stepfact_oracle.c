/*
 * stepfact_oracle.c — CPU ORACLE for the step-s Cholesky / LU / QR algorithms of
 * C. Camarero, "fast Cholesky/LU/QR decomposition algorithms", arXiv 1812.02056
 * (text in /root/reference/PAPER.md, cited below as PAPER.md:<line>).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or helper with the CUDA path (paper_1812_02056_b200/csrc), and neither
 * includes nor links the other.
 *
 * Style: the paper's Algorithms 1-3 written out step by step, in the paper's order and
 * notation, translated from 1-based inclusive ranges to 0-based half-open
 * ones.  fp64 throughout; compile with -O2 -ffp-contract=off -fno-fast-math so every
 * `a - b*c` rounds twice exactly as written (no FMA contraction).  Loops over rows /
 * columns whose iterations are independent may run under OpenMP; that never changes a
 * single rounding.  No blocking, fusion or reordering beyond what the algorithms state.
 *
 * Storage: all matrices column-major, element (i,j) at p[i + j*ld].
 *
 * Readings where the paper is silent (listed in DESIGN.md §3):
 *   R1  flush fires exactly when c == z+s at the top of the loop body; the last panel is
 *       never flushed.
 *   R2  S := R R^T is formed by summing k ascending first, then subtracted
 *       (PAPER.md:44-50); in-panel corrections subtract one term at a time (PAPER.md:55-56,
 *       63-64, 110, 118).
 *   R3  failure thresholds: Cholesky fails when the value under the sqrt is not > 0
 *       (incl. NaN); LU fails when |L_cc| < tol, QR when ||v|| < tol, tol = 1e-12*||A||_F/n.
 *       info = first failing column, 1-based; 0 = success.
 *   R4  v/||v|| is an elementwise division; ||v|| = sqrt(sum v_i^2) unscaled.
 *   R5  R := Q^T A is formed in full, the mass of its strict lower part is
 *       reported, then the strict lower part is set to 0.
 *   R11 variable step ("the s parameter could be varied during the
 *       execution"): with a step sequence s_0, s_1, ..., panel p flushes when c = z + s_p;
 *       the *_steps entry points.  A constant sequence is bitwise the fixed-s algorithm.
 *
 * Restricted variants: every routine takes `kcols` (K).  With K = n it is the verbatim
 * algorithm.  With K < n it produces only the first K columns of L (Cholesky), the first
 * K columns of L and K rows of U (LU), the first K columns of Q and K rows of R (QR): the
 * loop over c stops at K and each flush only updates the entries those outputs later
 * read.  Every retained entry undergoes the same operations in the same order as in the
 * full run, so it is bitwise equal to it (pinned by tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AT(p, ld, i, j) (p)[(size_t)(i) + (size_t)(j) * (size_t)(ld)]

static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

void orc_set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ||A||_F of the input, summed column by column (used only for the R3 thresholds). */
double orc_frobenius(int64_t n, const double* A, int64_t lda) {
  double acc = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) acc += AT(A, lda, i, j) * AT(A, lda, i, j);
  return sqrt(acc);
}

/* Step sequence.  The paper fixes one s and notes that "the s parameter could
 * be varied during the execution": with a sequence s_0, s_1, ... the flush
 * condition of the current panel is c = z + s_p and p advances at each flush (reading R11).
 * steps == NULL means the constant s. */
typedef struct { const int64_t* steps; int64_t nsteps, s, p; } Steps;
static int64_t step_now(const Steps* st) {
  if (!st->steps) return st->s;
  return st->p < st->nsteps ? st->steps[st->p] : st->steps[st->nsteps - 1];
}
static void step_next(Steps* st) { st->p++; }
static int64_t step_max(const Steps* st) {
  if (!st->steps) return st->s;
  int64_t m = 1;
  for (int64_t i = 0; i < st->nsteps; ++i) if (st->steps[i] > m) m = st->steps[i];
  return m;
}

/* Flush trace (test hook, tests/test_oracle.py): while armed, every flush of Algorithms 1-3
 * records the 0-based column c at which it fires (the `if c = z+s` of PAPER.md:41, 91, 143),
 * so the schedule each algorithm actually runs can be pinned against hand-worked lists. */
static int64_t* g_trace = NULL;
static int64_t g_trace_cap = 0, g_trace_n = 0;
void orc_trace_flushes(int64_t* buf, int64_t cap) { g_trace = buf; g_trace_cap = cap; g_trace_n = 0; }
int64_t orc_trace_count(void) { return g_trace_n; }
static void trace_flush(int64_t c) {
  if (g_trace && g_trace_n < g_trace_cap) g_trace[g_trace_n] = c;
  g_trace_n++;
}

/* Number of flushes the schedule of Algorithms 1-3 performs (R1). */
int64_t orc_flush_count(int64_t n, int64_t s) {
  int64_t z = 0, flushes = 0;
  for (int64_t c = 0; c < n; ++c) {
    if (c == z + s) { ++flushes; z = c; }
  }
  return flushes;
}

/*
 * Algorithm 1, "A fast Cholesky decomposition algorithm".
 *   A: n x n SPD input (read only; the algorithm's mutations of A go to a private copy W)
 *   L: n x n output, lower triangular; entries never written stay 0
 *   With K < n only the first K columns of A are read and of L written (n x K blocks).
 * Returns info (0 or 1-based failing column).
 */
static int64_t chol_core(int64_t n, Steps sp, int64_t kcols, const double* A, int64_t lda,
                         double* L, int64_t ldl) {
  const int64_t K = min64(kcols, n);
  /* the paper's A (mutated by the flushes); a restricted run only ever touches columns < K,
     so only those are copied (A and L may then be n x K blocks) */
  double* W = (double*)malloc(sizeof(double) * (size_t)n * (size_t)K);
  if (!W) return -1;
  for (int64_t j = 0; j < K; ++j)
    for (int64_t i = 0; i < n; ++i) { AT(W, n, i, j) = AT(A, lda, i, j); AT(L, ldl, i, j) = 0.0; }

  int64_t info = 0;
  int64_t z = 0;                                             /* z := 1            (:37) */
  for (int64_t c = 0; c < K; ++c) {                          /* for c from 1 to n (:39) */
    if (c == z + step_now(&sp)) {                            /* if c = z+s        (:41) */
      trace_flush(c);
      /* R := L[c..n, z..c-1] (:42); S := R R^T (:43); A_ij := A_ij - S (:44-50).
         Columns j >= K of W are never read again in a restricted run. */
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t j = c; j < K; ++j) {
        for (int64_t i = c; i < n; ++i) {
          double S = 0.0;
          for (int64_t k = z; k < c; ++k) S += AT(L, ldl, i, k) * AT(L, ldl, j, k);
          AT(W, n, i, j) = AT(W, n, i, j) - S;
        }
      }
      z = c;                                                 /* z := c            (:51) */
      step_next(&sp);
    }
    double d = AT(W, n, c, c);                               /* L_cc := A_cc      (:53) */
    for (int64_t k = z; k < c; ++k)                          /* (:54-57) */
      d = d - AT(L, ldl, c, k) * AT(L, ldl, c, k);
    if (!(d > 0.0)) { info = c + 1; break; }                 /* R3 */
    const double Lcc = sqrt(d);                              /* (:58) */
    AT(L, ldl, c, c) = Lcc;
#pragma omp parallel for schedule(static)
    for (int64_t i = c + 1; i < n; ++i) {                    /* (:59-67) */
      double t = AT(W, n, i, c);
      for (int64_t k = z; k < c; ++k) t = t - AT(L, ldl, i, k) * AT(L, ldl, c, k);
      AT(L, ldl, i, c) = t / Lcc;
    }
  }
  free(W);
  return info;
}

int64_t orc_chol(int64_t n, int64_t s, int64_t kcols, const double* A, int64_t lda, double* L, int64_t ldl) {
  Steps sp = {NULL, 0, s, 0};
  return chol_core(n, sp, kcols, A, lda, L, ldl);
}
int64_t orc_chol_steps(int64_t n, int64_t nsteps, const int64_t* steps, int64_t kcols, const double* A, int64_t lda,
                       double* L, int64_t ldl) {
  Steps sp = {steps, nsteps, steps[0], 0};
  return chol_core(n, sp, kcols, A, lda, L, ldl);
}

/*
 * Algorithm 2, "A fast LU decomposition algorithm".  Crout form:
 * L lower with its own diagonal, U unit upper.
 *   L, U: n x n outputs; entries never written stay 0.
 *   tol: R3 threshold 1e-12*||A||_F/n (pass <= 0 to compute it here).
 */
static int64_t lu_core(int64_t n, Steps sp, int64_t kcols, const double* A, int64_t lda,
                       double* L, int64_t ldl, double* U, int64_t ldu, double tol) {
  const int64_t K = min64(kcols, n);
  if (tol <= 0.0) tol = 1e-12 * orc_frobenius(n, A, lda) / (double)n;
  double* W = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!W) return -1;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      AT(W, n, i, j) = AT(A, lda, i, j); AT(L, ldl, i, j) = 0.0; AT(U, ldu, i, j) = 0.0;
    }

  int64_t info = 0;
  int64_t z = 0;
  for (int64_t c = 0; c < K; ++c) {
    if (c == z + step_now(&sp)) {                            /* (:91) */
      trace_flush(c);
      /* R_L := L[c..n, z..c-1], R_U := U[z..c-1, c..n], S := R_L R_U, A -= S (:92-103).
         A restricted run only ever reads W[i][j] with j < K (L columns) or i < K (U rows). */
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t j = c; j < n; ++j) {
        for (int64_t i = c; i < n; ++i) {
          if (j >= K && i >= K) continue;
          double S = 0.0;
          for (int64_t k = z; k < c; ++k) S += AT(L, ldl, i, k) * AT(U, ldu, k, j);
          AT(W, n, i, j) = AT(W, n, i, j) - S;
        }
      }
      z = c;
      step_next(&sp);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = c; i < n; ++i) {                        /* L column (:105-112) */
      double t = AT(W, n, i, c);
      for (int64_t k = z; k < c; ++k) t = t - AT(L, ldl, i, k) * AT(U, ldu, k, c);
      AT(L, ldl, i, c) = t;
    }
    const double Lcc = AT(L, ldl, c, c);
    if (!(fabs(Lcc) >= tol)) { info = c + 1; break; }        /* R3 */
#pragma omp parallel for schedule(static)
    for (int64_t i = c; i < n; ++i) {                        /* U row (:113-121) */
      double t = AT(W, n, c, i);
      for (int64_t k = z; k < c; ++k) t = t - AT(L, ldl, c, k) * AT(U, ldu, k, i);
      AT(U, ldu, c, i) = t / Lcc;
    }
  }
  free(W);
  return info;
}

int64_t orc_lu(int64_t n, int64_t s, int64_t kcols, const double* A, int64_t lda, double* L, int64_t ldl, double* U,
               int64_t ldu, double tol) {
  Steps sp = {NULL, 0, s, 0};
  return lu_core(n, sp, kcols, A, lda, L, ldl, U, ldu, tol);
}
int64_t orc_lu_steps(int64_t n, int64_t nsteps, const int64_t* steps, int64_t kcols, const double* A, int64_t lda,
                     double* L, int64_t ldl, double* U, int64_t ldu, double tol) {
  Steps sp = {steps, nsteps, steps[0], 0};
  return lu_core(n, sp, kcols, A, lda, L, ldl, U, ldu, tol);
}

/*
 * Algorithm 3, "A fast QR decomposition algorithm".
 *   Q: n x n output (orthonormal columns);  R: n x n output (upper; strict lower zeroed, R5)
 *   *lower_mass: ||tril(Q^T A, -1)||_F before zeroing (rows < K only in a restricted run)
 *   tol: R3 threshold (<= 0: computed here).
 */
static int64_t qr_core(int64_t n, Steps sp, int64_t kcols, const double* A, int64_t lda,
                       double* Q, int64_t ldq, double* R, int64_t ldr, double tol, double* lower_mass) {
  const int64_t s = step_max(&sp);
  const int64_t K = min64(kcols, n);
  if (tol <= 0.0) tol = 1e-12 * orc_frobenius(n, A, lda) / (double)n;
  double* M = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);  /* M := copy of A */
  double* C = (double*)malloc(sizeof(double) * (size_t)(s > 0 ? s : 1) * (size_t)n);
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  if (!M || !C || !v) { free(M); free(C); free(v); return -1; }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      AT(M, n, i, j) = AT(A, lda, i, j); AT(Q, ldq, i, j) = 0.0; AT(R, ldr, i, j) = 0.0;
    }

  int64_t info = 0;
  int64_t z = 0;
  for (int64_t c = 0; c < K; ++c) {
    if (c == z + step_now(&sp)) {                            /* (:143) */
      trace_flush(c);
      const int64_t w = c - z;
      const int64_t jend = K;  /* a restricted run never reads M columns >= K */
      /* B_Q := Q[1..n, z..c-1], B_M := M[1..n, c..n] (:145-146); C := B_Q^T B_M (:147) */
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t j = c; j < jend; ++j)
        for (int64_t k = z; k < c; ++k) {
          double t = 0.0;
          for (int64_t i = 0; i < n; ++i) t += AT(Q, ldq, i, k) * AT(M, n, i, j);
          AT(C, w, k - z, j) = t;
        }
      /* S := B_Q C (:148); M_ij := M_ij - S_ij for all rows i (:149-155) */
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t j = c; j < jend; ++j)
        for (int64_t i = 0; i < n; ++i) {
          double S = 0.0;
          for (int64_t k = z; k < c; ++k) S += AT(Q, ldq, i, k) * AT(C, w, k - z, j);
          AT(M, n, i, j) = AT(M, n, i, j) - S;
        }
      z = c;                                                 /* (:156) */
      step_next(&sp);
    }
    for (int64_t i = 0; i < n; ++i) v[i] = AT(M, n, i, c);   /* v := column c of M (:158) */
    for (int64_t j = z; j < c; ++j) {                        /* (:159-163) */
      double t = 0.0;                                        /* u := column j of Q; u^T v */
      for (int64_t i = 0; i < n; ++i) t += AT(Q, ldq, i, j) * v[i];
      for (int64_t i = 0; i < n; ++i) v[i] = v[i] - AT(Q, ldq, i, j) * t;
    }
    double nv2 = 0.0;
    for (int64_t i = 0; i < n; ++i) nv2 += v[i] * v[i];
    const double nv = sqrt(nv2);
    if (!(nv >= tol)) { info = c + 1; break; }               /* R3 */
    for (int64_t i = 0; i < n; ++i) AT(Q, ldq, i, c) = v[i] / nv;  /* (:164-168), R4 */
  }
  if (info == 0) {
    /* R := Q^T A (:170), rows < K */
    double mass = 0.0;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = 0; k < K; ++k) {
        double t = 0.0;
        for (int64_t i = 0; i < n; ++i) t += AT(Q, ldq, i, k) * AT(A, lda, i, j);
        AT(R, ldr, k, j) = t;
      }
    for (int64_t j = 0; j < n; ++j)                          /* R5 */
      for (int64_t k = j + 1; k < K; ++k) { mass += AT(R, ldr, k, j) * AT(R, ldr, k, j); AT(R, ldr, k, j) = 0.0; }
    if (lower_mass) *lower_mass = sqrt(mass);
  }
  free(M); free(C); free(v);
  return info;
}

int64_t orc_qr(int64_t n, int64_t s, int64_t kcols, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
               int64_t ldr, double tol, double* lower_mass) {
  Steps sp = {NULL, 0, s, 0};
  return qr_core(n, sp, kcols, A, lda, Q, ldq, R, ldr, tol, lower_mass);
}
int64_t orc_qr_steps(int64_t n, int64_t nsteps, const int64_t* steps, int64_t kcols, const double* A, int64_t lda,
                     double* Q, int64_t ldq, double* R, int64_t ldr, double tol, double* lower_mass) {
  Steps sp = {steps, nsteps, steps[0], 0};
  return qr_core(n, sp, kcols, A, lda, Q, ldq, R, ldr, tol, lower_mass);
}

/*
 * Solving with the factors ("used everywhere to solve linear systems"): plain
 * forward / back substitution, column by column of B (n x nrhs, in place), fp64.
 *   kind 0: A = L L^T   (F1 = L, lower):      L y = b (forward, / L_ii), L^T x = y (backward)
 *   kind 1: A = L U     (F1 = L\U packed):    L y = b (forward, / L_ii), U x = y (unit, backward)
 *   kind 2: A = Q R     (F1 = Q, F2 = R):     y = Q^T b, R x = y (backward, / R_ii)
 */
void orc_solve(int64_t kind, int64_t n, int64_t nrhs, const double* F1, int64_t ld1, const double* F2, int64_t ld2,
               double* B, int64_t ldb) {
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  if (!y) return;
  for (int64_t j = 0; j < nrhs; ++j) {
    double* b = B + (size_t)j * (size_t)ldb;
    if (kind == 2) {
      for (int64_t i = 0; i < n; ++i) {                       /* y = Q^T b */
        double t = 0.0;
        for (int64_t k = 0; k < n; ++k) t += AT(F1, ld1, k, i) * b[k];
        y[i] = t;
      }
      for (int64_t i = n - 1; i >= 0; --i) {                  /* R x = y */
        double t = y[i];
        for (int64_t k = i + 1; k < n; ++k) t = t - AT(F2, ld2, i, k) * b[k];
        b[i] = t / AT(F2, ld2, i, i);
      }
      continue;
    }
    for (int64_t i = 0; i < n; ++i) {                         /* L y = b */
      double t = b[i];
      for (int64_t k = 0; k < i; ++k) t = t - AT(F1, ld1, i, k) * b[k];
      b[i] = t / AT(F1, ld1, i, i);
    }
    for (int64_t i = n - 1; i >= 0; --i) {                    /* L^T x = y  or  U x = y */
      double t = b[i];
      for (int64_t k = i + 1; k < n; ++k)
        t = t - (kind == 0 ? AT(F1, ld1, k, i) : AT(F1, ld1, i, k)) * b[k];
      b[i] = kind == 0 ? t / AT(F1, ld1, i, i) : t;
    }
  }
  free(y);
}
