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
// persistent kernel needs one grid-wide exchange per column (qr_mgs_ll_kernel below: two-level,
// through distributed shared memory within clusters and epoch-tagged words across them).
#include <math.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include <stdio.h>

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
  g.smem = (size_t)elt * ((size_t)g.RB * w + (size_t)w + 64);
  return g;
}

size_t qr_mgs_work_elems(int64_t n, int w, int elt) {
  MgsGeom g = mgs_geom(n, w, elt);
  // flags[2][G] (int) + partials[2][w][G] (T), in units of T
  const size_t flag = (2 * (size_t)g.G * sizeof(int) + elt - 1) / elt + 2 * (size_t)g.G * (size_t)w + 2;
  // LL exchange: words[2][Q][w] of 16 (fp64) / 8 (fp32) bytes, Q <= ceil(n / 128) clusters, + alignment
  const size_t Q = (size_t)((n + 127) / 128);
  const size_t ll = (2 * Q * (size_t)w * (elt == 8 ? 16 : 8) + 256) / elt;
  return flag > ll ? flag : ll;
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
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until flags[0..G) >= epoch (warp 0 of the CTA polls; relaxed loads with a short
// back-off, one acquire fence at the end), then make the CTA wait for warp 0.
__device__ __forceinline__ void wait_flags(const int* flags, int G, int epoch) {
  if ((threadIdx.x >> 5) == 0) {
    const int lane = threadIdx.x & 31;
    for (;;) {
      bool all = true;
      for (int hh = lane; hh < G; hh += 32) all &= (ld_relaxed_s32(flags + hh) >= epoch);
      if (__all_sync(0xffffffffu, all)) break;
      __nanosleep(64);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

constexpr int kMgsMaxT = 16;   // columns per warp whose partial sums are fetched together
constexpr int kMgsRJ = 16;     // max rows per lane (RB <= 512, i.e. n <= 75776 on 148 SMs)

template <typename T>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                             int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                             int64_t col0, const T* tolp, T* work,
                                                             long long* fail) {
  if (failed(fail)) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* V = reinterpret_cast<T*>(smraw);          // V[c * RB + r]: this CTA's rows of the panel
  T* gsum = V + (size_t)RB * w;                // reduced Gram row for the current column
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kMgsThreads / 32;
  const int G = gridDim.x, g = blockIdx.x;
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = __ldcg(tolp);
  int* flags = reinterpret_cast<int*>(work);                                   // flags[2][G]
  T* partbase = work + (2 * G * sizeof(int) + sizeof(T) - 1) / sizeof(T);     // part[2][w][G]
  const int RJ = (RB + 31) / 32;               // rows per lane (RB <= 32 * kMgsRJ)

  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    V[idx] = (r < rows) ? __ldcg(src + r0 + r + (int64_t)c * lds) : T(0);   // L2, never a stale L1 line
  }
  __syncthreads();

  // partial Gram row of column 0: <v_0, v_cp> over this CTA's rows
  {
    T v0[kMgsRJ];
#pragma unroll
    for (int j = 0; j < kMgsRJ; ++j) v0[j] = (j < RJ && lane + 32 * j < RB) ? V[lane + 32 * j] : T(0);
    for (int cp = warp; cp < w; cp += nwarps) {
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < kMgsRJ; ++j)
        if (j < RJ && lane + 32 * j < RB) acc = fma(v0[j], V[(size_t)cp * RB + lane + 32 * j], acc);
      acc = warp_sum(acc);
      if (lane == 0) partbase[(size_t)cp * G + g] = acc;
    }
  }

  bool ok = true;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    T* part = partbase + (size_t)buf * G * w;
    // 1) publish this CTA's partial Gram row of column c, wait for everybody's
    __syncthreads();
    if (tid == 0) { __threadfence(); st_release_s32(flags + buf * G + g, (int)(col0 + c + 1)); }   // epochs grow across launches
    wait_flags(flags + buf * G, G, (int)(col0 + c + 1));
    // 2) fixed-order reduction of the partials (warp per column, coalesced over CTAs)
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
    // 3) q_c = v_c / ||v_c|| (every warp keeps its lane's rows in registers), the next
    //    column updated first (redundantly in every warp), then each warp projects q_c out
    //    of its columns and immediately forms their partial dot with v_{c+1}: the update
    //    of column c and the partial Gram row of column c+1 are one pass over shared memory.
    T q[kMgsRJ], vn[kMgsRJ];
    const T cn = (c + 1 < w) ? gsum[c + 1] / nv : T(0);
#pragma unroll
    for (int j = 0; j < kMgsRJ; ++j) {
      const int r = lane + 32 * j;
      const bool in = j < RJ && r < RB;
      q[j] = in ? V[(size_t)c * RB + r] / nv : T(0);
      vn[j] = (in && c + 1 < w) ? fma(-q[j], cn, V[(size_t)(c + 1) * RB + r]) : T(0);
    }
    __syncthreads();   // everybody has read v_c and v_{c+1}
    if (warp == 0) {
#pragma unroll
      for (int j = 0; j < kMgsRJ; ++j) {
        const int r = lane + 32 * j;
        if (j < RJ && r < RB) V[(size_t)c * RB + r] = q[j];
      }
    }
    T* pnext = partbase + (size_t)(buf ^ 1) * G * w;
    for (int cp = c + 1 + warp; cp < w; cp += nwarps) {
      const T coef = gsum[cp] / nv;                 // q_c^T v_cp
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < kMgsRJ; ++j) {
        const int r = lane + 32 * j;
        if (j < RJ && r < RB) {
          const T nvp = (cp == c + 1) ? vn[j] : fma(-q[j], coef, V[(size_t)cp * RB + r]);
          V[(size_t)cp * RB + r] = nvp;
          acc = fma(vn[j], nvp, acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) pnext[(size_t)cp * G + g] = acc;
    }
  }
  if (!ok) return;
  __syncthreads();
  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    if (r < rows) dst[r0 + r + (int64_t)c * ldd] = V[idx];
  }
}

// Register-resident variant for the common case w <= 128, RB <= 2*kMgsRPT: thread t owns
// column t>>1 and half t&1 of this CTA's rows (kMgsRPT values in registers), so a column
// step is one pass of register FMAs against two broadcast vectors in shared memory (q_c and
// v_{c+1}), with the two halves of each dot combined by a shuffle.
constexpr int kMgsRPT = 64;

template <typename T>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_reg_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                                 int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                                 int64_t col0, const T* tolp, T* work,
                                                                 long long* fail) {
  if (failed(fail)) return;
  constexpr int QP = kMgsRPT + 2;              // half stride in the broadcast vectors (bank spread)
  __shared__ T qs[2 * QP], vs[2 * QP];
  __shared__ T gsum[128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kMgsThreads / 32;
  const int G = gridDim.x, g = blockIdx.x;
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = __ldcg(tolp);
  int* flags = reinterpret_cast<int*>(work);
  T* partbase = work + (2 * G * sizeof(int) + sizeof(T) - 1) / sizeof(T);
  const int cp = tid >> 1, h = tid & 1;        // my column and half
  const int rbase = h * kMgsRPT;
  const bool mine = cp < w;
  T x[kMgsRPT];
#pragma unroll
  for (int r = 0; r < kMgsRPT; ++r) {
    const int rr = rbase + r;
    x[r] = (mine && rr < rows) ? __ldcg(src + r0 + rr + (int64_t)cp * lds) : T(0);
  }
  // partial Gram row of column 0
  if (cp == 0) {
#pragma unroll
    for (int r = 0; r < kMgsRPT; ++r) vs[h * QP + r] = x[r];
  }
  __syncthreads();
  {
    T acc = T(0);
#pragma unroll
    for (int r = 0; r < kMgsRPT; ++r) acc = fma(vs[h * QP + r], x[r], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (mine && h == 0) partbase[(size_t)cp * G + g] = acc;
  }

  bool ok = true;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    T* part = partbase + (size_t)buf * G * w;
    __syncthreads();
    if (tid == 0) { __threadfence(); st_release_s32(flags + buf * G + g, (int)(col0 + c + 1)); }
    wait_flags(flags + buf * G, G, (int)(col0 + c + 1));
    for (int cb = c + warp; cb < w; cb += nwarps * kMgsMaxT) {
      T acc[kMgsMaxT];
#pragma unroll
      for (int t = 0; t < kMgsMaxT; ++t) acc[t] = T(0);
      for (int hh = lane; hh < G; hh += 32) {
#pragma unroll
        for (int t = 0; t < kMgsMaxT; ++t) {
          const int cc = cb + t * nwarps;
          if (cc < w) acc[t] += __ldcg(part + (size_t)cc * G + hh);
        }
      }
#pragma unroll
      for (int t = 0; t < kMgsMaxT; ++t) {
        const int cc = cb + t * nwarps;
        const T v = warp_sum(acc[t]);
        if (lane == 0 && cc < w) gsum[cc] = v;
      }
    }
    __syncthreads();
    const T nv = dsqrt(gsum[c]);
    if (!(nv >= tol)) {
      if (g == 0 && tid == 0) record_fail(fail, col0 + c + 1);
      ok = false;
      break;
    }
    // q_c = v_c / ||v_c|| (owner threads), v_{c+1} before its update (owner threads)
    const T rnv = T(1) / nv;   // q_c = v_c * (1/||v_c||): one division per CTA instead of one per row
    if (cp == c) {
#pragma unroll
      for (int r = 0; r < kMgsRPT; ++r) { x[r] = x[r] * rnv; qs[h * QP + r] = x[r]; }
    }
    if (cp == c + 1) {
#pragma unroll
      for (int r = 0; r < kMgsRPT; ++r) vs[h * QP + r] = x[r];
    }
    __syncthreads();
    const bool act = mine && cp > c;
    T acc = T(0);
    if (act) {
      const T coef = gsum[cp] * rnv;                        // q_c^T v_cp
      const T cn = (c + 1 < w) ? gsum[c + 1] * rnv : T(0);  // q_c^T v_{c+1}
#pragma unroll
      for (int r = 0; r < kMgsRPT; ++r) {
        const T qr = qs[h * QP + r];
        x[r] = fma(-qr, coef, x[r]);                         // v_cp -= q_c (q_c^T v_cp)
        acc = fma(fma(-qr, cn, vs[h * QP + r]), x[r], acc);  // <v_{c+1}, v_cp> (both updated)
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);             // all lanes take part
    if (act && h == 0 && c + 1 < w) partbase[(size_t)(buf ^ 1) * G * w + (size_t)cp * G + g] = acc;
  }
  if (!ok || !mine) return;
#pragma unroll
  for (int r = 0; r < kMgsRPT; ++r) {
    const int rr = rbase + r;
    if (rr < rows) dst[r0 + rr + (int64_t)cp * ldd] = x[r];
  }
}

// ---------------------------------------------------------------- cluster + LL exchange
// The variant used whenever it fits (w <= 128, <= 128 rows per CTA, the clusters
// co-resident): the same register-resident column step as qr_mgs_reg_kernel, but the
// Gram-row exchange is two-level.
//   1. inside a thread-block cluster of CL CTAs the partial rows meet in distributed shared
//      memory: after a cluster barrier, CTA k of the cluster sums (in rank order) the CL
//      partials of columns j = c + k (mod CL) and publishes the cluster sum;
//   2. the Q = G / CL cluster sums go through global memory as "LL" words: each 64-bit word
//      carries 32 data bits and the 32-bit epoch (col0 + c + 1) of the column they belong
//      to, so a reader polls the data itself — a word whose epoch matches is valid (64-bit
//      accesses are single-copy atomic), no separate flag, no fence, one L2 round trip.
//      Every CTA reads all Q sums of every remaining column and adds them in cluster order,
//      so all CTAs hold bitwise the same Gram row (and take the same break decision).
// Measured on B200 (calib/mgs_probe.cu, n = 8192, w = 128): 3.8 us per column against
// 5.6 us for the flag exchange of qr_mgs_reg_kernel (its partial reads alone took 2.8 us).
// Buffer reuse: slot (c & 1, q, j) is rewritten at column c + 2 only after the writer's
// cluster passed the cluster barrier of column c + 2, i.e. after every CTA of every cluster
// polled column c + 1, hence finished reading column c.  Epochs grow across the launches of
// one factorization and the buffer is zeroed at its start, so a stale word never matches.
template <typename T> struct LL;
template <> struct LL<double> {
  static constexpr int kWords = 2;
  static __device__ __forceinline__ void put(unsigned long long* p, double v, unsigned ep) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long w0 = ((unsigned long long)ep << 32) | (b & 0xffffffffull);
    const unsigned long long w1 = ((unsigned long long)ep << 32) | (b >> 32);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
  }
  static __device__ __forceinline__ bool get(const unsigned long long* p, unsigned ep, double& v) {
    unsigned long long w0, w1;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if ((unsigned)(w0 >> 32) != ep || (unsigned)(w1 >> 32) != ep) return false;
    v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
    return true;
  }
};
template <> struct LL<float> {
  static constexpr int kWords = 1;
  static __device__ __forceinline__ void put(unsigned long long* p, float v, unsigned ep) {
    const unsigned long long w0 = ((unsigned long long)ep << 32) | (unsigned long long)__float_as_uint(v);
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(w0) : "memory");
  }
  static __device__ __forceinline__ bool get(const unsigned long long* p, unsigned ep, float& v) {
    unsigned long long w0;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w0) : "l"(p) : "memory");
    if ((unsigned)(w0 >> 32) != ep) return false;
    v = __uint_as_float((unsigned)(w0 & 0xffffffffull));
    return true;
  }
};

// Gather the Q cluster sums of columns c..w-1 (cnt = Q * wc LL words, poll until each carries
// epoch ep) into cval[qq * w + j].  A thread's words are requested 4 at a time before any is
// checked, so a poll pass costs one L2 round trip, not one per word (a thread owns up to
// ceil(Q*w / 256) words).
template <typename T>
__device__ __forceinline__ void ll_gather(const unsigned long long* ll, int buf, int Q, int w, int c, int wc, int cnt,
                                          unsigned ep, T* cval, int tid) {
  constexpr int B = 4;
  for (int base = tid; base < cnt; base += B * kMgsThreads) {
    T v[B];
    bool got[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int idx = base + u * kMgsThreads;
      got[u] = idx >= cnt;
      if (!got[u]) {
        const int qq = idx / wc, j = c + idx % wc;
        got[u] = LL<T>::get(ll + LL<T>::kWords * ((size_t)(buf * Q + qq) * w + j), ep, v[u]);
      }
    }
    bool all = true;
#pragma unroll
    for (int u = 0; u < B; ++u) all = all && got[u];
    while (!all) {
      all = true;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (!got[u]) {
          const int idx = base + u * kMgsThreads, qq = idx / wc, j = c + idx % wc;
          got[u] = LL<T>::get(ll + LL<T>::kWords * ((size_t)(buf * Q + qq) * w + j), ep, v[u]);
          all = all && got[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int idx = base + u * kMgsThreads;
      if (idx < cnt) cval[(idx / wc) * w + c + idx % wc] = v[u];
    }
  }
}

// Gather + sum in one pass: thread t polls the Q cluster sums of column j = c + t (all its
// words requested before any is checked, one L2 round trip per poll pass) and adds them in
// cluster order q = 0, 1, ... (the order of the two-pass gather + sum: the same bits), so the
// Gram row needs no staging buffer and one CTA barrier instead of two.
template <typename T>
__device__ __forceinline__ void ll_gather_sum(const unsigned long long* ll, int buf, int Q, int w, int c, unsigned ep,
                                              T* gsum, int tid) {
  for (int j = c + tid; j < w; j += kMgsThreads) {
    T a = T(0);
    for (int q0 = 0; q0 < Q; q0 += 8) {   // 8 words in flight (registers, static indices)
      T v[8];
      unsigned pending = 0;                // bit u: word q0 + u not yet valid
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = T(0);
        if (q0 + u < Q && !LL<T>::get(ll + LL<T>::kWords * ((size_t)(buf * Q + q0 + u) * w + j), ep, v[u]))
          pending |= 1u << u;
      }
      while (pending) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if ((pending >> u) & 1u)
            if (LL<T>::get(ll + LL<T>::kWords * ((size_t)(buf * Q + q0 + u) * w + j), ep, v[u])) pending &= ~(1u << u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + u < Q) a += v[u];
    }
    gsum[j] = a;
  }
}

// RPT = rows of its column half a thread owns (the CTA holds 2 * RPT rows), NR of them in
// registers and RPT - NR in shared memory (xs, one slot per thread: conflict-free).
// RPT = 128, NR = 64 halves the number of CTAs (SMs) the panel occupies at the same register
// use per CTA, so the concurrent flush keeps more SMs (measured: DESIGN.md §5 K7).
// SF_MGS_TIMING (calib/mgs_ll_probe.cu only): thread 0 of every CTA accumulates clock64
// cycles per phase of the column step: [0] cluster barrier, [1] DSMEM sum + LL put,
// [2] LL gather, [3] Gram row sum (2 CTA barriers), [4] scale q_c / publish (1 barrier),
// [5] projections + partial Gram row of c+1
#ifdef SF_MGS_TIMING
__device__ unsigned long long mgs_times[256][8];
#define MG_T0() long long mg_t = clock64(); long long mg_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define MG_T(ph) do { long long t_ = clock64(); mg_acc[ph] += t_ - mg_t; mg_t = t_; } while (0)
#define MG_TEND() do { if (threadIdx.x == 0) for (int q_ = 0; q_ < 8; ++q_) mgs_times[blockIdx.x & 255][q_] = mg_acc[q_]; } while (0)
#else
#define MG_T0() do {} while (0)
#define MG_T(ph) do {} while (0)
#define MG_TEND() do {} while (0)
#endif

template <typename T, int RPT, int NR>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_ll_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                                int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                                int64_t col0, const T* tolp,
                                                                unsigned long long* ll, long long* fail,
                                                                int mgs_two_pass) {
  if (failed(fail)) return;      // stable during the launch: every CTA of a cluster agrees
  constexpr int QP = RPT + 2;
  __shared__ T qs[2 * QP], vs[2 * QP];
  __shared__ T gsum[128];
  __shared__ T mypart[2][128];
  extern __shared__ __align__(16) unsigned char smraw[];
  T* cval = reinterpret_cast<T*>(smraw);   // cval[q * w + j]: cluster q's sum for column j
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), k = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int G = gridDim.x, g = blockIdx.x, Q = G / CL, q = g / CL;
  T* xs = cval + (((size_t)Q * w + 1) & ~(size_t)1);   // rows NR.. of each thread: xs[(r - NR) * kMgsThreads + tid]
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = __ldcg(tolp);
  const int cp = tid >> 1, h = tid & 1;        // my column and half
  const int rbase = h * RPT;
  const bool mine = cp < w;
  T x[NR];
  auto X = [&](int r) -> T& { return r < NR ? x[r < NR ? r : 0] : xs[(size_t)(r - NR) * kMgsThreads + tid]; };
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int rr = rbase + r;
    X(r) = (mine && rr < rows) ? __ldcg(src + r0 + rr + (int64_t)cp * lds) : T(0);
  }
  if (cp == 0) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) vs[h * QP + r] = X(r);
  }
  __syncthreads();
  {
    // four interleaved partial sums: the dot product's dependency chain is RPT/4 fmas deep
    T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r & 3] = fma(vs[h * QP + r], X(r), acc[r & 3]);
    T a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    a += __shfl_xor_sync(0xffffffffu, a, 1);
    if (mine && h == 0) mypart[0][cp] = a;
  }

  bool ok = true;
  MG_T0();
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    const unsigned ep = (unsigned)(col0 + c + 1);
    cluster.sync();   // every CTA of the cluster wrote its partial row of column c
    MG_T(0);
    for (int j = c + k + CL * tid; j < w; j += CL * kMgsThreads) {
      T a = T(0);
      for (int rr = 0; rr < CL; ++rr) a += cluster.map_shared_rank(&mypart[buf][0], rr)[j];
      LL<T>::put(ll + LL<T>::kWords * ((size_t)(buf * Q + q) * w + j), a, ep);
    }
    MG_T(1);
    if (Q <= 32 && !mgs_two_pass) {
      ll_gather_sum<T>(ll, buf, Q, w, c, ep, gsum, tid);
      MG_T(2);
    } else {
      const int wc = w - c, cnt = Q * wc;
      ll_gather<T>(ll, buf, Q, w, c, wc, cnt, ep, cval, tid);
      MG_T(2);
      __syncthreads();
      for (int j = c + tid; j < w; j += kMgsThreads) {
        T a = T(0);
        for (int qq = 0; qq < Q; ++qq) a += cval[qq * w + j];
        gsum[j] = a;
      }
    }
    __syncthreads();
    MG_T(3);
    // 1/||v_c|| without the IEEE sqrt / division subroutines (reading P11); ||v_c|| for R3
    const T rnv = fast_rsqrt(gsum[c]);
    const T nv = gsum[c] * rnv;
    if (!(nv >= tol)) {
      if (g == 0 && tid == 0) record_fail(fail, col0 + c + 1);
      ok = false;
      break;
    }
    if (cp == c) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) { X(r) = X(r) * rnv; qs[h * QP + r] = X(r); }
    }
    if (cp == c + 1) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) vs[h * QP + r] = X(r);
    }
    __syncthreads();
    MG_T(4);
    const bool act = mine && cp > c;
    T acc[4] = {T(0), T(0), T(0), T(0)};   // interleaved partial sums (short dependency chains)
    if (act) {
      const T coef = gsum[cp] * rnv;                        // q_c^T v_cp
      const T cn = (c + 1 < w) ? gsum[c + 1] * rnv : T(0);  // q_c^T v_{c+1}
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const T qr = qs[h * QP + r];
        const T xr = fma(-qr, coef, X(r));                   // v_cp -= q_c (q_c^T v_cp)
        X(r) = xr;
        acc[r & 3] = fma(fma(-qr, cn, vs[h * QP + r]), xr, acc[r & 3]);   // <v_{c+1}, v_cp>
      }
    }
    T a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    a += __shfl_xor_sync(0xffffffffu, a, 1);
    if (act && h == 0 && c + 1 < w) mypart[buf ^ 1][cp] = a;
    MG_T(5);
  }
  MG_TEND();
  cluster.sync();   // no CTA leaves while a cluster peer may still read its shared memory
  if (!ok || !mine) return;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int rr = rbase + r;
    if (rr < rows) dst[r0 + rr + (int64_t)cp * ldd] = X(r);
  }
}

// Shared-memory-resident variant of the cluster + LL exchange for panels wider than 128
// columns (or more rows per CTA than the register variant holds): the panel rows live in
// shared memory as in qr_mgs_kernel (a warp per column, lanes over rows), the Gram-row
// exchange is the two-level one of qr_mgs_ll_kernel.
template <typename T>
__global__ void __launch_bounds__(kMgsThreads) qr_mgs_ll_smem_kernel(int64_t n, int w, int RB, const T* __restrict__ src,
                                                                     int64_t lds, T* __restrict__ dst, int64_t ldd,
                                                                     int64_t col0, const T* tolp,
                                                                     unsigned long long* ll, long long* fail) {
  if (failed(fail)) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* V = reinterpret_cast<T*>(smraw);          // V[c * RB + r]: this CTA's rows of the panel
  T* gsum = V + (size_t)RB * w;                // reduced Gram row of the current column
  T* mypart = gsum + w;                        // [2][w] this CTA's partial Gram rows
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), k = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kMgsThreads / 32;
  const int G = gridDim.x, g = blockIdx.x, Q = G / CL, q = g / CL;
  T* cval = mypart + 2 * w;                    // [Q][w] cluster sums
  T* qs = cval + (size_t)Q * w;                // [RB] q_c of this CTA's rows
  T* vs = qs + RB;                             // [RB] updated v_{c+1}
  const int64_t r0 = (int64_t)g * RB;
  const int rows = (int)((r0 + RB <= n) ? RB : (n > r0 ? n - r0 : 0));
  const T tol = __ldcg(tolp);
  const int RJ = (RB + 31) / 32;

  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    V[idx] = (r < rows) ? __ldcg(src + r0 + r + (int64_t)c * lds) : T(0);
  }
  __syncthreads();
  {
    T v0[kMgsRJ];
#pragma unroll
    for (int j = 0; j < kMgsRJ; ++j) v0[j] = (j < RJ && lane + 32 * j < RB) ? V[lane + 32 * j] : T(0);
    for (int cp = warp; cp < w; cp += nwarps) {
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < kMgsRJ; ++j)
        if (j < RJ && lane + 32 * j < RB) acc = fma(v0[j], V[(size_t)cp * RB + lane + 32 * j], acc);
      acc = warp_sum(acc);
      if (lane == 0) mypart[cp] = acc;
    }
  }

  bool ok = true;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    const unsigned ep = (unsigned)(col0 + c + 1);
    cluster.sync();
    for (int j = c + k + CL * tid; j < w; j += CL * kMgsThreads) {
      T a = T(0);
      for (int rr = 0; rr < CL; ++rr) a += cluster.map_shared_rank(mypart + buf * w, rr)[j];
      LL<T>::put(ll + LL<T>::kWords * ((size_t)(buf * Q + q) * w + j), a, ep);
    }
    const int wc = w - c, cnt = Q * wc;
    ll_gather<T>(ll, buf, Q, w, c, wc, cnt, ep, cval, tid);
    __syncthreads();
    for (int j = c + tid; j < w; j += kMgsThreads) {
      T a = T(0);
      for (int qq = 0; qq < Q; ++qq) a += cval[qq * w + j];
      gsum[j] = a;
    }
    __syncthreads();
    // 1/||v_c|| without the IEEE sqrt / division subroutines (reading P11); ||v_c|| for R3
    const T rnv = fast_rsqrt(gsum[c]);
    const T nv = gsum[c] * rnv;
    if (!(nv >= tol)) {
      if (g == 0 && tid == 0) record_fail(fail, col0 + c + 1);
      ok = false;
      break;
    }
    // q_c = v_c / ||v_c|| and the updated v_{c+1} as shared vectors, then a THREAD per later
    // column (no per-column warp reduction): v_cp -= q_c (q_c^T v_cp) row by row, with its
    // dot against the updated v_{c+1} formed in the same pass (the next partial Gram row)
    const T cn = (c + 1 < w) ? gsum[c + 1] * rnv : T(0);
    for (int r = tid; r < RB; r += kMgsThreads) {
      const T qr = V[(size_t)c * RB + r] * rnv;
      qs[r] = qr;
      V[(size_t)c * RB + r] = qr;
      vs[r] = (c + 1 < w) ? fma(-qr, cn, V[(size_t)(c + 1) * RB + r]) : T(0);
    }
    __syncthreads();
    for (int cp = c + 1 + tid; cp < w; cp += kMgsThreads) {
      const T coef = gsum[cp] * rnv;
      T* col = V + (size_t)cp * RB;
      T acc = T(0);
      if (cp == c + 1) {
        for (int r = 0; r < RB; ++r) { const T v = vs[r]; col[r] = v; acc = fma(v, v, acc); }
      } else {
#pragma unroll 4
        for (int r = 0; r < RB; ++r) {
          const T v = fma(-qs[r], coef, col[r]);
          col[r] = v;
          acc = fma(vs[r], v, acc);
        }
      }
      mypart[(buf ^ 1) * w + cp] = acc;
    }
    __syncthreads();
  }
  cluster.sync();
  if (!ok) return;
  __syncthreads();
  for (int idx = tid; idx < RB * w; idx += kMgsThreads) {
    const int r = idx % RB, c = idx / RB;
    if (r < rows) dst[r0 + r + (int64_t)c * ldd] = V[idx];
  }
}

struct LLGeom { int G = 0, CL = 0, RB = 0; size_t dyn = 0; };

// The MGS grids are persistent: their CTAs wait on each other, so two of them running at
// once on one device (two QR calls on different streams) could each hold part of the SMs
// and wait forever for the rest.  Eager launches are therefore chained per device: a launch
// on another stream than the previous one first waits for the previous launch's event.
// (Launches recorded into a CUDA graph are not chained; DESIGN.md §5 K7.)
struct MgsOrder {
  static constexpr int kMaxDev = 64;
  static cudaEvent_t ev[kMaxDev];
  static cudaStream_t last[kMaxDev];
  int dev = -1;
  cudaStream_t st;
  explicit MgsOrder(cudaStream_t s) : st(s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (getenv("SF_MGS_NOORDER") != nullptr) return;   // experiment switch only
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) { cudaGetLastError(); return; }
    if (cs != cudaStreamCaptureStatusNone || cudaGetDevice(&dev) != cudaSuccess || dev >= kMaxDev) { dev = -1; return; }
    if (ev[dev] != nullptr && last[dev] != st) cudaStreamWaitEvent(st, ev[dev], 0);
  }
  ~MgsOrder() {
    if (dev < 0) return;
    if (ev[dev] == nullptr && cudaEventCreateWithFlags(&ev[dev], cudaEventDisableTiming) != cudaSuccess) { ev[dev] = nullptr; return; }
    cudaEventRecord(ev[dev], st);
    last[dev] = st;
  }
};
cudaEvent_t MgsOrder::ev[MgsOrder::kMaxDev] = {};
cudaStream_t MgsOrder::last[MgsOrder::kMaxDev] = {};

// A replayed CUDA graph of a QR factorization contains MGS panel launches: chain whole
// graph launches the same way (driver.cu run_graph), so replays on two streams never run
// two persistent MGS grids at once.
void mgs_order_before(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= MgsOrder::kMaxDev) return;
  if (MgsOrder::ev[dev] != nullptr && MgsOrder::last[dev] != st) cudaStreamWaitEvent(st, MgsOrder::ev[dev], 0);
}
void mgs_order_after(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= MgsOrder::kMaxDev) return;
  if (MgsOrder::ev[dev] == nullptr &&
      cudaEventCreateWithFlags(&MgsOrder::ev[dev], cudaEventDisableTiming) != cudaSuccess) {
    MgsOrder::ev[dev] = nullptr;
    return;
  }
  cudaEventRecord(MgsOrder::ev[dev], st);
  MgsOrder::last[dev] = st;
}

// Cooperative launch (guaranteed co-residency of the persistent grid, e.g. under MPS or
// beside another process) by default; not under a profiler (CUDA_INJECTION64_PATH is set by
// Nsight Compute / Systems, which reject cooperative cluster launches) or with SF_MGS_COOP=0.
// Measured neutral: cfg4 80.04 (cooperative) vs 80.96 ms.
static bool mgs_cooperative() {
  static const bool on = [] {
    const char* e = getenv("SF_MGS_COOP");
    if (e) return atoi(e) != 0;
    return getenv("CUDA_INJECTION64_PATH") == nullptr;
  }();
  return on;
}

// Grid for the LL kernels, or G = 0 when they do not apply (then the flag-exchange kernels).
// reg: the register-resident variant (w <= 128, <= 128 rows per CTA); otherwise the
// shared-memory one (the panel rows + exchange buffers within 220 KB per CTA).
// rows per thread of the LL kernel (SF_MGS_RPT: 64 = all in registers, 128 = half in shared
// memory: twice the rows per CTA, half the CTAs)
// SF_MGS_TWO_PASS (default 1): the gather spreads the Q x (w - c) words over all threads,
// stages them, then sums per column.  0: one pass, thread t polls and sums column c + t
// (measured slower: 3.0 vs 1.4 us per column in the gather — half the threads idle, twice the
// words per poller; cfg4 80.8 vs 76.4 ms).
static int mgs_two_pass() {
  static const int v = [] { const char* e = getenv("SF_MGS_TWO_PASS"); return e ? atoi(e) : 1; }();
  return v;
}
static int mgs_rpt() {
  static const int v = [] { const char* e = getenv("SF_MGS_RPT"); return (e && atoi(e) == 128) ? 128 : 64; }();
  return v;
}
// rows of the 64 a thread owns that stay in registers (SF_MGS_NR: 64, or 32 = half in shared
// memory: ~half the registers per CTA, so two flush CTAs share the panel CTA's SM)
static int mgs_nr() {
  static const int v = [] { const char* e = getenv("SF_MGS_NR"); return (e && atoi(e) == 32) ? 32 : 64; }();
  return v;
}
template <typename T>
static const void* mgs_ll_reg_fn() {
  if (mgs_rpt() == 128) return (const void*)qr_mgs_ll_kernel<T, 128, 64>;
  return mgs_nr() == 32 ? (const void*)qr_mgs_ll_kernel<T, 64, 32> : (const void*)qr_mgs_ll_kernel<T, 64, 64>;
}

template <typename T>
static LLGeom ll_geom(int64_t n, int w, bool reg) {
  LLGeom r;
  const int rpt = reg ? mgs_rpt() : kMgsRPT;
  if (getenv("SF_MGS_NOLL") != nullptr) return r;
  if (reg && w > 128) return r;
  const int64_t G0 = (n + 2 * rpt - 1) / (2 * rpt);
  static int maxcl[2][17] = {{-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
                             {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}};
  auto dyn_for = [&](int G, int CL) -> size_t {
    if (reg) return sizeof(T) * (((size_t)(G / CL) * (size_t)w + 1) / 2 * 2 + (size_t)(rpt - (rpt == 64 ? mgs_nr() : 64)) * kMgsThreads);
    const int RB = (int)((n + G - 1) / G);
    return sizeof(T) * ((size_t)RB * w + 3 * (size_t)w + (size_t)(G / CL) * w + 2 * (size_t)RB);
  };
  auto fits = [&](int CL, int G) -> bool {
    const size_t dyn = dyn_for(G, CL);
    if (dyn > (reg ? 200 : 220) * 1024) return false;
    int& mc = maxcl[reg ? 0 : 1][CL];
    if (mc < 0 || !reg) {   // the shared-memory variant's occupancy depends on its size
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(kMgsThreads);
      cfg.dynamicSmemBytes = dyn;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const void* kf = reg ? mgs_ll_reg_fn<T>() : (const void*)qr_mgs_ll_smem_kernel<T>;
      // (the register variant's dynamic size varies a little with G: allow up to 200 KB)
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, reg ? 200 * 1024 : (int)dyn);
      if (CL > 8) cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int m = 0;
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&m, kf, &cfg);
      if (getenv("SF_MGS_DEBUG"))
        fprintf(stderr, "mgs geom: reg %d rpt %d CL %d G %d dyn %zu -> max clusters %d (%s)\n", (int)reg, rpt, CL, G,
                dyn, m, cudaGetErrorString(oe));
      if (oe != cudaSuccess) { cudaGetLastError(); m = 0; }
      if (reg) mc = m;
      else return G / CL <= m;
    }
    return G / CL <= mc;
  };
  int G = 0, CL = 0;
  if (G0 <= 8) {
    if (fits((int)G0, (int)G0)) { G = (int)G0; CL = (int)G0; }
  } else {
    // SF_MGS_CL16: try non-portable 16-CTA clusters first (half as many clusters to exchange
    // through global memory, twice the partial rows summed in distributed shared memory)
    static const bool cl16 = getenv("SF_MGS_CL16") && atoi(getenv("SF_MGS_CL16"));
    for (int cl : {16, 8, 4}) {
      if (cl == 16 && !cl16) continue;
      const int g = (int)((G0 + cl - 1) / cl * cl);
      if (fits(cl, g)) { G = g; CL = cl; break; }
    }
  }
  if (G == 0) return r;
  r.G = G; r.CL = CL;
  r.RB = (int)((n + G - 1) / G);
  if (r.RB > (reg ? 2 * rpt : 32 * kMgsRJ)) return LLGeom{};
  r.dyn = dyn_for(G, CL);
  return r;
}

template <typename T>
cudaError_t qr_mgs_panel(int64_t n, int w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                         const T* tol, T* work, long long* fail, cudaStream_t st) {
  if (w <= 0) return cudaSuccess;
  MgsOrder order(st);
  LLGeom lg = ll_geom<T>(n, w, true);
  const bool lreg = lg.G > 0;
  if (!lreg) lg = ll_geom<T>(n, w, false);
  if (lg.G > 0) {
    unsigned long long* ll = reinterpret_cast<unsigned long long*>(((uintptr_t)work + 255) & ~(uintptr_t)255);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lg.G);
    cfg.blockDim = dim3(kMgsThreads);
    cfg.dynamicSmemBytes = lg.dyn;
    cfg.stream = st;
    // Every cluster waits on every other, so all must be co-resident: ll_geom admits the grid
    // only if cudaOccupancyMaxActiveClusters says they all fit, and eager launches are chained
    // (MgsOrder).  Not launched cooperative: Nsight Compute rejects cooperative cluster launches.
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = lg.CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = mgs_cooperative() ? 2 : 1;
    int RB = lg.RB;
    count_launch();
    if (lreg && mgs_rpt() == 64 && mgs_nr() == 32)
      return cudaLaunchKernelEx(&cfg, qr_mgs_ll_kernel<T, 64, 32>, n, w, RB, src, lds, dst, ldd, col0, tol, ll, fail,
                                mgs_two_pass());
    if (lreg && mgs_rpt() == 64)
      return cudaLaunchKernelEx(&cfg, qr_mgs_ll_kernel<T, 64, 64>, n, w, RB, src, lds, dst, ldd, col0, tol, ll, fail,
                                mgs_two_pass());
    if (lreg)
      return cudaLaunchKernelEx(&cfg, qr_mgs_ll_kernel<T, 128, 64>, n, w, RB, src, lds, dst, ldd, col0, tol, ll, fail,
                                mgs_two_pass());
    return cudaLaunchKernelEx(&cfg, qr_mgs_ll_smem_kernel<T>, n, w, RB, src, lds, dst, ldd, col0, tol, ll, fail);
  }
  MgsGeom g = mgs_geom(n, w, (int)sizeof(T));
  if (g.smem > 220 * 1024) return cudaErrorInvalidValue;   // caller splits wider panels
  if (g.RB > 32 * kMgsRJ) return cudaErrorNotSupported;     // rows per CTA beyond the register budget
  const bool reg = w <= 128 && g.RB <= 2 * kMgsRPT && getenv("SF_MGS_SMEM") == nullptr;
  auto k = reg ? qr_mgs_reg_kernel<T> : qr_mgs_kernel<T>;
  const size_t dyn = reg ? 0 : g.smem;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int RB = g.RB;
  void* args[] = {(void*)&n, (void*)&w, (void*)&RB, (void*)&src, (void*)&lds, (void*)&dst, (void*)&ldd,
                  (void*)&col0, (void*)&tol, (void*)&work, (void*)&fail};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k, dim3(g.G), dim3(kMgsThreads), args, dyn, st);
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

// D(i, j) = a X(i, j) + b Y(i, j) over rows x cols; X(i, j) = 0 outside its xr x xc extent
// (zero padding of the uneven Strassen blocks), op(X)(i, j) = xkc ? X[j + i ldx] : X[i + j ldx]
// (Y likewise).  Memory-bound elementwise pass (the Strassen-Winograd block sums, f1).
template <typename T>
__global__ void comb_kernel(int64_t rows, int64_t cols, T a, const T* X, int64_t ldx, int xkc, int64_t xr, int64_t xc,
                            T b, const T* Y, int64_t ldy, int ykc, int64_t yr, int64_t yc, T* D, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
      const T x = (X && i < xr && j < xc) ? __ldcg(X + (xkc ? j + i * ldx : i + j * ldx)) : T(0);
      const T y = (Y && i < yr && j < yc) ? __ldcg(Y + (ykc ? j + i * ldy : i + j * ldy)) : T(0);
      D[i + j * ldd] = a * x + b * y;
    }
}
template <typename T>
cudaError_t comb(int64_t rows, int64_t cols, T a, const T* X, int64_t ldx, int xkc, int64_t xr, int64_t xc, T b,
                 const T* Y, int64_t ldy, int ykc, int64_t yr, int64_t yc, T* D, int64_t ldd, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const unsigned gx = (unsigned)((rows + 255) / 256 > 4 ? 4 : (rows + 255) / 256);
  const unsigned gy = (unsigned)(cols < 4096 ? cols : 4096);
  comb_kernel<T><<<dim3(gx, gy), 256, 0, st>>>(rows, cols, a, X, ldx, xkc, xr, xc, b, Y, ldy, ykc, yr, yc, D, ldd);
  count_launch();
  return cudaGetLastError();
}

#define SF_INST(T)                                                                                             \
  template cudaError_t qr_mgs_panel<T>(int64_t, int, const T*, int64_t, T*, int64_t, int64_t, const T*, T*,  \
                                       long long*, cudaStream_t);                                             \
  template cudaError_t frob_norm_tol<T>(int64_t, const T*, int64_t, T*, double*, cudaStream_t);                   \
  template cudaError_t zero_strict_lower<T>(int64_t, T*, int64_t, cudaStream_t);                             \
  template cudaError_t copy_matrix<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t);             \
  template cudaError_t comb<T>(int64_t, int64_t, T, const T*, int64_t, int, int64_t, int64_t, T, const T*, int64_t, int, \
                               int64_t, int64_t, T*, int64_t, cudaStream_t);
SF_INST(double)
SF_INST(float)

}  // namespace sf
