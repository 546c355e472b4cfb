// small.cu — the whole step-s Cholesky of a small matrix (n <= 256) inside ONE thread-block
// cluster, every value resident in shared memory (SURVEY.md §8 a1-a3 at BASELINE.json
// configs[0]: n = 256, s = 16).
//
// At n = 256 the general driver is launch-latency bound: 16 panels x (panel leaf + two flush
// launches), ~7 us each, ~0.34 ms per factorization for 5.6 MFLOP.  Here CTA k of a cluster
// of ceil(n/32) CTAs owns the 32 columns [32k, 32k+32) (rows >= the column: the lower
// triangle Algorithm 1 reads) in its shared memory, and the paper's
// schedule runs with one cluster barrier per step:
//
//   for each panel p = [z, z+w)   (w = s; 32 % s == 0, so a panel lies in one CTA)
//     owner CTA: the panel recurrences, right-looking over the panel's
//       columns — per column c: L_cc = sqrt(d), L_ic = x_ic / L_cc (x 1/L_cc, reading P11),
//       then x_ij -= L_ic L_jc for the panel's later columns j, one term at a time in k order
//     cluster barrier (the factored panel is visible through distributed shared memory)
//     flush, when c = z + w < n: every CTA copies the panel rows it needs
//       (rows >= c) into its own shared memory and applies A[i, j] -= sum_k L_ik L_jk
//       (k = z .. c-1 ascending, one fused multiply-add per term) to its columns j >= c,
//       rows i >= j
//
// A failed pivot (R3: the value under the square root not > 0, incl. NaN) is recorded as the
// first failed column and stops every CTA of the cluster after the same barrier.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace sf {

// SF_SMALL_TIMING (calib/small_probe.cu only): thread 0 of every CTA accumulates clock64
// cycles per phase: [k][0] load, [1] panel, [2] barrier after the panel, [3] panel copy,
// [4] flush, [5] end-of-step barrier, [6] write-back
#ifdef SF_SMALL_TIMING
__device__ unsigned long long small_times[8][16][8];   // [warp][cta][phase] (lane 0)
__device__ unsigned long long small_steps[8][40][3];   // [cta][step][phase 1,2,5 end], warp 0
__device__ unsigned long long small_cols[40][4];    // owner thread 0: per column step of panel 0: start, after sync, after rsqrt, end
#define SM_T0() long long sm_t = clock64(); long long sm_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define SM_T(ph) do { long long t = clock64(); sm_acc[ph] += t - sm_t; sm_t = t; \
  if (threadIdx.x == 0 && (ph == 1 || ph == 2 || ph == 5)) small_steps[k][z / s][ph == 1 ? 0 : ph == 2 ? 1 : 2] = t; } while (0)
#define SM_TC(q) do { if (z == 0 && threadIdx.x == 0) small_cols[c][q] = clock64(); } while (0)
#define SM_TEND() do { if ((threadIdx.x & 31) == 0) \
  for (int q = 0; q < 8; ++q) small_times[threadIdx.x >> 5][k][q] = sm_acc[q]; } while (0)
#else
#define SM_T0() do {} while (0)
#define SM_T(ph) do {} while (0)
#define SM_TEND() do {} while (0)
#define SM_TC(q) do {} while (0)
#endif

template <typename T> struct T2s_;
template <> struct T2s_<double> { using type = double2; };
template <> struct T2s_<float> { using type = float2; };
template <typename T> using T2v = typename T2s_<T>::type;

namespace small {
constexpr int CW = 32;        // columns per CTA
constexpr int NT = 256;       // threads per CTA: one row each
constexpr int NMAX = 256;     // rows (one per thread) = columns (8 CTAs x 32)
}  // namespace small

// smem: X[jl * NP + i] (own columns, column-major, rows >= the column valid), then the panel
// copy P[k * NP + i] (k < s) used by the flush.
template <typename T, int S>
__global__ void __launch_bounds__(small::NT) chol_small_cluster_kernel(int n, int s_, const T* __restrict__ A,
                                                                       int64_t lda, T* __restrict__ L, int64_t ldl,
                                                                       long long* fail) {
  using namespace small;
  constexpr int s = S;   // the step, a compile-time constant (s | 32): register windows of s
  (void)s_;
  cg::cluster_group cluster = cg::this_cluster();
  const int k = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int NP = (n + 1) & ~1;   // even column stride: 16-byte aligned pairs
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* X = reinterpret_cast<T*>(sm_raw);
  T* P = X + CW * NP;
  __shared__ int badcol;     // first failed column (1-based) this CTA met, 0 = none
  __shared__ __align__(16) T piv[2][S < 2 ? 2 : S];   // owner: the diagonal block's column c (double-buffered)
  const int j0 = k * CW;
  const int ncol = (n - j0 < CW) ? n - j0 : CW;
  if (tid == 0) badcol = 0;
  SM_T0();
  // load my columns, rows >= column (coalesced: a warp covers 32 consecutive rows)
  for (int jl = 0; jl < ncol; ++jl) {
    const int j = j0 + jl;
    for (int i = j + tid; i < n; i += NT) X[jl * NP + i] = __ldg(A + i + (int64_t)j * lda);
  }
  cluster.sync();
  { const int z = 0; SM_T(0); }
  const int i = tid;   // my row

  // ---- the panel recurrences of [z, z+w) by its owner, right-looking, one
  // term at a time in k order, in a rotating register window: at column step c, x[0] is my
  // row's column c, x[q] its column c + q.  The rows of the diagonal block publish their
  // x[0] (double-buffered, one barrier per column); per column: L_cc = sqrt(d), L_ic = x_ic /
  // L_cc (x 1/L_cc, reading P11), x_{i,c+q} -= L_ic L_{c+q,c} (a zero multiplier where
  // c+q > i: fma(-0, u, x) == x exactly), then the window moves on by one column —
  // compile-time register indices in a rolled loop (a version indexing registers by the
  // runtime column compiled to ~1450 instructions per column and ran 1.2 us a column).
  auto factor = [&](int z, int w) {
    T* Xp = X + (size_t)(z - j0) * NP;   // panel column cc at Xp[cc * NP]
    T x[S];
#pragma unroll
    for (int q = 0; q < S; ++q) x[q] = (q < w && i >= z + q && i < n) ? Xp[q * NP + i] : T(0);
    for (int c = 0; c < w; ++c) {
      const int col = z + c;
      T* pv = piv[c & 1];
      if (i >= col && i < z + w) pv[i - col] = x[0];   // row col + q publishes x_{col+q, col}
      __syncthreads();
      const T d = pv[0];
      if (!(d > T(0))) {                // R3: incl. NaN
        if (tid == 0) { badcol = col + 1; atomicMin((unsigned long long*)fail, (unsigned long long)(col + 1)); }
        break;
      }
      const T r = fast_rsqrt(d);        // 1 / L_cc
      if (i >= col && i < n) {
        const T l = (i == col) ? d * r : x[0] * r;
        Xp[c * NP + i] = l;
        T u[S];   // the pivot rows' column c, all loads issued before the first use
        if constexpr (S >= 2) {
#pragma unroll
          for (int q = 0; q < S; q += 2) {
            const T2v<T> v = *reinterpret_cast<const T2v<T>*>(pv + q);
            u[q] = v.x; u[q + 1] = v.y;
          }
        } else {
          u[0] = pv[0];
        }
        const int qmax = (i > col) ? min(w - c - 1, i - col) : 0;   // c + q < w, col + q <= i
#pragma unroll
        for (int q = 1; q < S; ++q) {
          const T lq = (q <= qmax) ? l : T(0);
          x[q] = fma(-lq, u[q] * r, x[q]);
        }
      }
#pragma unroll
      for (int q = 0; q + 1 < S; ++q) x[q] = x[q + 1];
      x[S - 1] = T(0);
    }
    __syncthreads();
  };

  // ---- flush of the panel copied into P (w columns, rows >= r0) into my
  // local columns [ja, jb) (all >= c): A[i, j] -= sum_k L_ik L_jk for rows i >= j, k
  // ascending.  Item = (row, group of 8 columns): 8 independent accumulators; lanes run over
  // rows, so the group's panel rows are broadcasts (two per 16-byte load).
  auto flush = [&](int w, int r0, int ja, int jb) {
    const int ga = ja / 8, gb = (jb + 7) / 8, nr = n - r0;
    const int nitems = nr * (gb - ga);
    for (int it = tid; it < nitems; it += NT) {
      const int ii = r0 + it % nr, g = ga + it / nr;
      if (j0 + 8 * g > ii) continue;   // group entirely above the diagonal
      T acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = T(0);
#pragma unroll 2
      for (int kk = 0; kk < w; ++kk) {
        const T lik = P[kk * NP + ii];
        const T* pj = P + kk * NP + j0 + 8 * g;
        T2v<T> v[4];   // all loads of the step issued before the first use
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = *reinterpret_cast<const T2v<T>*>(pj + 2 * q);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = fma(lik, v[q].x, acc[2 * q]);              // S_ij, k ascending
          acc[2 * q + 1] = fma(lik, v[q].y, acc[2 * q + 1]);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int jl = 8 * g + q;
        if (jl >= ja && jl < jb && j0 + jl <= ii) X[jl * NP + ii] -= acc[q];
      }
    }
  };

  // Schedule with lookahead: in step p, the owner of panel p+1 first applies flush p to
  // that panel's columns, factors it, then flushes its other columns, while the other CTAs
  // apply flush p to theirs; one cluster barrier per step (panel p+1 final, panel p read).
  if (k == 0) factor(0, s < n ? s : n);
  { const int z = 0; SM_T(1); }
  cluster.sync();
  { const int z = 0; SM_T(2); }
  for (int z = 0; z < n; z += s) {
    const int w = (s < n - z) ? s : n - z;
    const int owner = z / CW;
    // a failure in panel p (its owner's first failed column lies in [z, z+w)) stops everyone
    // here; a failure its owner already met in panel p+1 is acted on one step later
    const int ob = *cluster.map_shared_rank(&badcol, owner);
    if (ob != 0 && ob <= z + w) break;
    const int c = z + w;
    if (c >= n) break;
    const int w2 = (s < n - c) ? s : n - c;
    const int owner2 = c / CW;
    if (j0 + ncol > c) {
      // copy panel p's rows >= r0 from its owner (all loads of a thread in flight first)
      const T* OX = cluster.map_shared_rank(X, owner) + (size_t)(z - owner * CW) * NP;
      const int r0 = (c > j0) ? c : j0;
      for (int r = r0 + tid; r < n; r += NT) {
        T v[S];
#pragma unroll
        for (int kk = 0; kk < S; ++kk) v[kk] = kk < w ? OX[kk * NP + r] : T(0);
#pragma unroll
        for (int kk = 0; kk < S; ++kk)
          if (kk < w) P[kk * NP + r] = v[kk];
      }
      __syncthreads();
      SM_T(3);
      const int jlo = (c > j0) ? c - j0 : 0;
      if (k == owner2) {
        const int pa = c - j0, pb = pa + w2;   // panel p+1's local columns
        flush(w, r0, pa, pb);
        __syncthreads();
        factor(c, w2);
        if (pb < ncol) flush(w, r0, pb, ncol);
        (void)jlo;
      } else {
        flush(w, r0, jlo, ncol);
      }
    }
    SM_T(4);
    cluster.sync();   // panel p+1 final; every CTA done with panel p and its failure flag
    SM_T(5);
  }
  // write my columns, rows >= column (the strict upper part of L is not touched)
  for (int jl = 0; jl < ncol; ++jl) {
    const int j = j0 + jl;
    for (int r = j + tid; r < n; r += NT) L[r + (int64_t)j * ldl] = X[jl * NP + r];
  }
  { const int z = 0; SM_T(6); }
  SM_TEND();
  cluster.sync();   // no CTA leaves while a peer may still read its shared memory
}

bool chol_small_applies(int64_t n, int64_t s, int elt) {
  static const int on = [] { const char* e = getenv("SF_CHOL_SMALL"); return e ? atoi(e) : 1; }();
  return on && elt == 8 && n >= 1 && n <= small::NMAX && s >= 1 && small::CW % s == 0;
}

cudaError_t chol_small(int64_t n, int64_t s, const double* A, int64_t lda, double* L, int64_t ldl, long long* fail,
                       cudaStream_t st) {
  using namespace small;
  const int nc = (int)((n + CW - 1) / CW);
  const int64_t np = (n + 1) & ~(int64_t)1;
  const size_t dyn = sizeof(double) * ((size_t)CW * np + (size_t)s * np + CW);   // + the last CTA's overrun of P
  const void* fn = nullptr;
  switch (s) {
    case 1: fn = (const void*)chol_small_cluster_kernel<double, 1>; break;
    case 2: fn = (const void*)chol_small_cluster_kernel<double, 2>; break;
    case 4: fn = (const void*)chol_small_cluster_kernel<double, 4>; break;
    case 8: fn = (const void*)chol_small_cluster_kernel<double, 8>; break;
    case 16: fn = (const void*)chol_small_cluster_kernel<double, 16>; break;
    case 32: fn = (const void*)chol_small_cluster_kernel<double, 32>; break;
    default: return cudaErrorInvalidValue;
  }
  static bool attr[33] = {};
  if (!attr[s]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(double) * (2 * CW * NMAX + CW)));
    if (e != cudaSuccess) return e;
    attr[s] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  count_launch();
  int n_ = (int)n, s_ = (int)s;
  void* args[] = {(void*)&n_, (void*)&s_, (void*)&A, (void*)&lda, (void*)&L, (void*)&ldl, (void*)&fail};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace sf
