// drv.cuh — host-side pieces shared by the single-GPU drivers (driver.cu) and the
// block-cyclic multi-GPU drivers (dist.cu): workspace, lookahead streams, the GEMM
// dispatch and the recursive panel factorizations.
#pragma once
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/stepfact.h"
#include "kernels.h"

namespace sf {

int fail_with(int code, const char* fmt, ...);

// Host-side serialization of the public entry points: the drivers share per-device side
// streams, events, graph and stream caches, so concurrent calls from several host threads
// enqueue one at a time (the GPU work itself stays asynchronous).
std::recursive_mutex& api_mutex();
#define SF_API_LOCK std::lock_guard<std::recursive_mutex> sf_api_lock_(sf::api_mutex())

// ------------------------------------------------------------------ profiling hook
// When enabled, CUDA event pairs are recorded on the factorization stream around every
// flush (trailing update) and every panel, so a benchmark can measure the update
// kernels' own device time inside its timed region (sf_profile_collect).
struct ProfRec { cudaEvent_t a, b; int kind; double flops; };
extern bool g_prof;
extern std::vector<ProfRec> g_prof_recs;
cudaEvent_t pool_event();
struct ProfScope {
  ProfRec r{}; cudaStream_t st; bool on;
  ProfScope(int kind, double flops, cudaStream_t s) : st(s), on(g_prof) {
    if (!on) return;
    r.a = pool_event(); r.b = pool_event(); r.kind = kind; r.flops = flops;
    cudaEventRecord(r.a, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(r.b, st);
    g_prof_recs.push_back(r);
  }
};

#define SF_CUDA(expr)                                                                               \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess) return fail_with(SF_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                                           __FILE__, __LINE__);                                     \
  } while (0)

inline int leaf_width() {
  static int w = [] {
    const char* e = getenv("SF_LEAF");
    int v = e ? atoi(e) : 32;
    if (v != 16 && v != 32) v = 32;
    return v;
  }();
  return w;
}

// Cholesky leaf width of the recursive panel: 32 (default) or 16 (SF_CHOL_LEAF).
inline int chol_leaf_width() {
  static int w = [] {
    const char* e = getenv("SF_CHOL_LEAF");
    int v = e ? atoi(e) : 32;
    if (v != 16 && v != 32) v = 32;
    return v;
  }();
  return w;
}

// One-launch 64-wide panels (panel64.cu).  LU: on by default (SF_LU_P64=0 -> the 32-wide
// leaf recursion).  Cholesky: for panels whose height m is at most SF_CHOL_P64_MAXM (the
// fused leaf doubles the SIMT flops of the rows below — the 32-wide recursion moves half of
// them to the tensor cores — so it pays only where launch latency dominates).
inline bool lu_p64_on() {
  static const int on = [] { const char* e = getenv("SF_LU_P64"); return e ? atoi(e) : 1; }();
  return on != 0;
}
inline int64_t chol_p64_maxm() {
  static const int64_t v = [] { const char* e = getenv("SF_CHOL_P64_MAXM"); return e ? (int64_t)atoll(e) : (int64_t)0; }();
  return v;
}
// fp32 Cholesky panels: the one-launch leaf is measured faster (cfg3 fp32 24.3 -> 23.1 ms)
inline int64_t chol32_p64_maxm() {
  static const int64_t v = [] {
    const char* e = getenv("SF_CHOL32_P64_MAXM");
    return e ? (int64_t)atoll(e) : (int64_t)1 << 40;
  }();
  return v;
}

inline int64_t half_of(int64_t w, int leaf) {
  int64_t h = (w / 2 + leaf - 1) / leaf * leaf;
  if (h >= w) h = w - leaf;
  if (h <= 0) h = w / 2;
  return h;
}

// ------------------------------------------------------------------ workspace
// Stream-ordered scratch, freed on `st` when the driver returns — on every path, including
// an error return in the middle of the factorization: streams registered with join() (the
// lookahead side stream, the QR early-R stream) are joined into `st` first, so no kernel
// still queued there can touch the freed block.
struct Workspace {
  char* base = nullptr;
  size_t off = 0, cap = 0;
  cudaStream_t st = nullptr;
  cudaStream_t joins[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaError_t init(size_t bytes, cudaStream_t s) {
    st = s;
    cap = bytes;
    keep_pool();
    return cudaMallocAsync((void**)&base, bytes, s);
  }
  void join(cudaStream_t s) {
    for (auto& j : joins)
      if (!j || j == s) { j = s; return; }
  }
  // keep freed workspace in the device's stream-ordered pool (the default release
  // threshold of 0 would unmap it at every synchronization and remap it next call)
  static void keep_pool() {
    static bool done[16] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || done[dev & 15]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev & 15] = true;
  }
  template <typename U>
  U* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    U* p = (U*)(base + off);
    off += n * sizeof(U);
    return p;
  }
  ~Workspace() {
    if (!base) return;
    for (cudaStream_t j : joins) {
      if (!j || j == st) continue;
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(e, j);
        cudaStreamWaitEvent(st, e, 0);
        cudaEventDestroy(e);
      }
    }
    cudaFreeAsync(base, st);
  }
};

// ------------------------------------------------------------------ schedule (a1)
// Panel boundaries of the step-s schedule: panel p = columns
// [z(p), z(p) + w(p)); a flush follows every panel but the last.  Fixed s, or a step
// sequence s_0, s_1, ... ("the s parameter could be varied during the execution",
// PAPER.md:194, reading R11; the last step repeats if the sequence is short).
struct Sched {
  int64_t n;
  std::vector<int64_t> start;   // panel starts, then n
  Sched(int64_t n_, int64_t s) : n(n_) {
    for (int64_t z = 0; z < n; z += s) start.push_back(z);
    start.push_back(n);
  }
  Sched(int64_t n_, const int64_t* steps, int64_t nsteps) : n(n_) {
    int64_t z = 0, p = 0;
    while (z < n) {
      start.push_back(z);
      z += steps[p < nsteps ? p : nsteps - 1];
      ++p;
    }
    start.push_back(n);
  }
  int64_t P() const { return (int64_t)start.size() - 1; }
  int64_t z(int64_t p) const { return start[p]; }
  int64_t w(int64_t p) const { return start[p + 1] - start[p]; }
  // the step if every panel but the last has the same width (and the last is not wider), else 0
  int64_t fixed() const {
    const int64_t s = w(0);
    for (int64_t p = 0; p + 1 < P(); ++p) if (w(p) != s) return 0;
    return w(P() - 1) <= s ? s : 0;
  }
  int64_t maxw() const {
    int64_t m = 1;
    for (int64_t p = 0; p < P(); ++p) m = w(p) > m ? w(p) : m;
    return m;
  }
};

// ------------------------------------------------------------------ panel completion hook
// Called (on the host, while enqueueing) after the work that finishes panel [z, z+w) has
// been enqueued on stream `st`: the end-to-end host path uses it to start the device->host
// copy of each finished panel while the later flushes run.
struct PanelHook {
  virtual ~PanelHook() {}
  virtual cudaError_t done(int64_t z, int64_t w, cudaStream_t st) = 0;
};

// ------------------------------------------------------------------ lookahead streams
// Panel p+1 is factored on a high-priority side stream while the rest of flush p runs on
// the caller's stream (classic lookahead): the caller's stream first updates only the
// columns of panel p+1, signals, then updates the remainder of the trailing matrix.
inline bool lookahead_on() {
  static int on = [] { const char* e = getenv("SF_LOOKAHEAD"); return e ? atoi(e) : 1; }();
  return on != 0;
}
struct Side {
  cudaStream_t st = nullptr;
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  // events are re-recorded round-robin: a stream wait captures the event's state at the
  // time cudaStreamWaitEvent is called, so re-recording afterwards is safe
  cudaEvent_t event() { return ev[next++ % ev.size()]; }
};
inline cudaError_t side_stream(Side*& out) {
  static Side sides[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Side& sd = sides[dev & 15];
  if (!sd.st) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&sd.st, cudaStreamNonBlocking, hi);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < 8; ++i) { cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); sd.ev.push_back(ev); }
  }
  out = &sd;
  return cudaSuccess;
}
// A second, LOW-priority side stream: background work that only fills SM slots the
// factorization's own kernels leave free (QR's early R row blocks).
inline cudaError_t low_stream(Side*& out) {
  static Side sides[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Side& sd = sides[dev & 15];
  if (!sd.st) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&sd.st, cudaStreamNonBlocking, lo);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < 8; ++i) { cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); sd.ev.push_back(ev); }
  }
  out = &sd;
  return cudaSuccess;
}
// record on `from`, make `to` wait
inline cudaError_t fork_join(Side& sd, cudaStream_t from, cudaStream_t to) {
  cudaEvent_t e = sd.event();
  cudaError_t r = cudaEventRecord(e, from);
  if (r != cudaSuccess) return r;
  return cudaStreamWaitEvent(to, e, 0);
}

// ------------------------------------------------------------------ GEMM dispatch per dtype
template <typename T>
struct Gemm {
  int64_t M, N, K;
  const T* A; int64_t lda; int ak;
  const T* B; int64_t ldb; int bk;
  const T* Cin; int64_t ldcin;
  T* C; int64_t ldc;
  double alpha; int beta; int mask;
  int splits; T* work;
  const long long* fail;
  int64_t off = 0;   // mask diagonal offset (lower: i >= j + off, upper: i <= j + off)
  int max_ctas = 0;  // fp64: bounded grid (0 = one CTA per tile)
};

inline cudaError_t run_gemm(const Gemm<double>& g, cudaStream_t st) {
  GemmF64 p{g.M, g.N, g.K, g.A, g.lda, g.B, g.ldb, g.Cin, g.ldcin, g.C, g.ldc,
            g.alpha, g.beta, g.splits, g.work, g.fail};
  p.off = g.off;
  p.max_ctas = g.max_ctas;
  return gemm_f64(p, g.ak, g.bk, g.mask, st);
}
// fp32: split op(A) and op(B) once into K-major hi/lo copies (stream-ordered scratch), then
// ONE 3xTF32 tcgen05 GEMM (gemm_tf32.cu); split-K requests are served unsplit.
inline cudaError_t run_gemm(const Gemm<float>& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.K <= 0) {
    if (g.beta && g.Cin == g.C && g.ldcin == g.ldc) return cudaSuccess;
    return cudaErrorNotSupported;
  }
  const int64_t ldk = (g.K + 3) / 4 * 4;
  float* buf = nullptr;
  const size_t elems = 2 * (size_t)(g.M + g.N) * ldk;
  cudaError_t e = cudaMallocAsync((void**)&buf, elems * sizeof(float) + 64, st);
  if (e != cudaSuccess) return e;
  float* Ah = buf; float* Al = Ah + (size_t)g.M * ldk;
  float* Bh = Al + (size_t)g.M * ldk; float* Bl = Bh + (size_t)g.N * ldk;
  // op(A)(i,k): ak ? A[k + i*lda] (K-major) : A[i + k*lda] (column-major)
  e = g.ak ? split_tf32_kmajor(g.M, g.K, g.A, g.lda, Ah, Al, ldk, st) : split_tf32(g.M, g.K, g.A, g.lda, Ah, Al, ldk, st);
  // op(B)(k,j): bk ? B[k + j*ldb] (row j of B^T is K-major) : B[j + k*ldb]
  if (e == cudaSuccess)
    e = g.bk ? split_tf32_kmajor(g.N, g.K, g.B, g.ldb, Bh, Bl, ldk, st) : split_tf32(g.N, g.K, g.B, g.ldb, Bh, Bl, ldk, st);
  if (e == cudaSuccess) {
    Tf32Gemm t{g.M, g.N, g.K, Ah, Al, ldk, Bh, Bl, ldk, g.Cin, g.ldcin, g.C, g.ldc, g.mask, g.off, g.fail};
    t.alpha = (float)g.alpha;
    t.beta = g.beta;
    e = gemm_tf32x3(t, st);
  }
  cudaError_t e2 = cudaFreeAsync(buf, st);
  return e != cudaSuccess ? e : e2;
}

// C -= op(A) op(B) with C read from Cin (may differ) : common "subtract" form
template <typename T>
inline cudaError_t gemm_sub(int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, int ak, const T* B,
                            int64_t ldb, int bk, const T* Cin, int64_t ldcin, T* C, int64_t ldc, int mask,
                            const long long* fail, cudaStream_t st, int max_ctas = 0) {
  Gemm<T> g{M, N, K, A, lda, ak, B, ldb, bk, Cin, ldcin, C, ldc, -1.0, 1, mask, 1, nullptr, fail};
  g.max_ctas = max_ctas;
  return run_gemm(g, st);
}

// ------------------------------------------------------------------ f1: Strassen-Winograd flush
// the step-s method is "fast" because the rectangular product of
// each flush can use a fast matrix multiplication.  Optional (sf_set_strassen; off by
// default): ONE Strassen-Winograd level for fp64 flushes whose sides are >= min_dim —
// 7 half-size DMMA products instead of 8 plus 8 operand block sums and 4 output block
// sums (elementwise, HBM-bound).  Uneven halves are zero-padded (ceil/floor split).  On
// B200 the flush is tensor-bound with a ridge near 6 flop/B, so the saved 1/8 of the flops
// costs ~12 extra passes over half-size blocks (DESIGN.md §9 f1 has the measurement).
struct StrassenCfg { int levels = 0; int64_t min_dim = 4096; };
inline StrassenCfg& strassen_cfg() { static StrassenCfg c; return c; }

// op(X) sub-block at (r0, c0): element (i, k) of op(X) is X[kc ? k + i*ld : i + k*ld]
template <typename T>
inline const T* opblk(const T* X, int64_t ld, int kc, int64_t r0, int64_t c0) {
  return X + (kc ? c0 + r0 * ld : r0 + c0 * ld);
}

inline bool strassen_applies(int64_t M, int64_t N, int64_t K);

// C = beta*Cin + alpha*op(A) op(B) (alpha = +-1, beta in {0, 1}) by Strassen-Winograd, `depth`
// levels deep (PAPER.md:186-190 used 2-3 recursions): the 7 half-size products recurse while
// they still meet the size threshold.  fp64.  C may equal Cin (in place); beta = 0 never reads Cin.
template <typename T>
inline cudaError_t strassen_gen(int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda, int ak, const T* B,
                                int64_t ldb, int bk, int beta, const T* Cin, int64_t ldcin, T* C, int64_t ldc,
                                const long long* fail, cudaStream_t st, int depth) {
  const int64_t m1 = (M + 1) / 2, m2 = M - m1, k1 = (K + 1) / 2, k2 = K - k1, n1 = (N + 1) / 2, n2 = N - n1;
  // op(B)(k, j): bk ? B[k + j*ldb] : B[j + k*ldb]  ->  as an "op(X)(row k, col j)" with kc = !bk
  const int bkc = bk ? 0 : 1;
  const T *A11 = opblk(A, lda, ak, 0, 0), *A12 = opblk(A, lda, ak, 0, k1), *A21 = opblk(A, lda, ak, m1, 0),
          *A22 = opblk(A, lda, ak, m1, k1);
  const T *B11 = opblk(B, ldb, bkc, 0, 0), *B12 = opblk(B, ldb, bkc, 0, n1), *B21 = opblk(B, ldb, bkc, k1, 0),
          *B22 = opblk(B, ldb, bkc, k1, n1);
  Workspace ws;
  cudaError_t e = ws.init(sizeof(T) * (size_t)(4 * m1 * k1 + 4 * k1 * n1 + 3 * m1 * n1) + 16 * 256, st);
  if (e != cudaSuccess) return e;
  T *S1 = ws.take<T>(m1 * k1), *S2 = ws.take<T>(m1 * k1), *S3 = ws.take<T>(m1 * k1), *S4 = ws.take<T>(m1 * k1);
  T *T1 = ws.take<T>(k1 * n1), *T2 = ws.take<T>(k1 * n1), *T3 = ws.take<T>(k1 * n1), *T4 = ws.take<T>(k1 * n1);
  T *W = ws.take<T>(m1 * n1), *V = ws.take<T>(m1 * n1), *X = ws.take<T>(m1 * n1);
  const T one = T(1), mone = T(-1);
  const T* cin = beta ? Cin : nullptr;   // beta = 0: the block sums read zeros, not Cin
#define SF_TRY(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  // operand block sums (zero padded to m1 x k1 / k1 x n1)
  SF_TRY(comb<T>(m1, k1, one, A21, lda, ak, m2, k1, one, A22, lda, ak, m2, k2, S1, m1, st));   // S1 = A21 + A22
  SF_TRY(comb<T>(m1, k1, one, S1, m1, 0, m1, k1, mone, A11, lda, ak, m1, k1, S2, m1, st));     // S2 = S1 - A11
  SF_TRY(comb<T>(m1, k1, one, A11, lda, ak, m1, k1, mone, A21, lda, ak, m2, k1, S3, m1, st));  // S3 = A11 - A21
  SF_TRY(comb<T>(m1, k1, one, A12, lda, ak, m1, k2, mone, S2, m1, 0, m1, k1, S4, m1, st));     // S4 = A12 - S2
  SF_TRY(comb<T>(k1, n1, one, B12, ldb, bkc, k1, n2, mone, B11, ldb, bkc, k1, n1, T1, k1, st)); // T1 = B12 - B11
  SF_TRY(comb<T>(k1, n1, one, B22, ldb, bkc, k2, n2, mone, T1, k1, 0, k1, n1, T2, k1, st));     // T2 = B22 - T1
  SF_TRY(comb<T>(k1, n1, one, B22, ldb, bkc, k2, n2, mone, B12, ldb, bkc, k1, n2, T3, k1, st)); // T3 = B22 - B12
  SF_TRY(comb<T>(k1, n1, one, T2, k1, 0, k1, n1, mone, B21, ldb, bkc, k2, n1, T4, k1, st));     // T4 = T2 - B21
  // c = beta_p*cin + alpha_p*op(a) op(b): one more Strassen level while the product is large
  auto prod = [&](int64_t mm, int64_t nn, int64_t kk, const T* a, int64_t la, int aak, const T* b, int64_t lb, int bbk,
                  double alpha_p, int beta_p, const T* ci, int64_t lci, T* c, int64_t lc) -> cudaError_t {
    if (mm <= 0 || nn <= 0) return cudaSuccess;
    if (depth > 1 && strassen_applies(mm, nn, kk))
      return strassen_gen<T>(mm, nn, kk, (T)alpha_p, a, la, aak, b, lb, bbk, beta_p, ci, lci, c, lc, fail, st, depth - 1);
    Gemm<T> g{mm, nn, kk, a, la, aak, b, lb, bbk, ci, lci, c, lc, alpha_p, beta_p, kMaskNone, 1, nullptr, fail};
    return run_gemm(g, st);
  };
  const double al = (double)alpha;
  // products (gemm operands: plain temps are idx-contiguous: ak = 0; as B: bk = 1 means B[k + j*ld])
  SF_TRY(prod(m1, n1, k1, A11, lda, ak, B11, ldb, bk, 1.0, 0, nullptr, 0, W, m1));  // W = P1
  SF_TRY(comb<T>(m1, n1, one, cin, ldcin, 0, m1, n1, alpha, W, m1, 0, m1, n1, C, ldc, st));           // C11 = b Cin11 + a P1
  SF_TRY(prod(m1, n1, k2, A12, lda, ak, B21, ldb, bk, al, 1, C, ldc, C, ldc));      // C11 += a P2
  SF_TRY(prod(m1, n1, k1, S2, m1, 0, T2, k1, 1, 1.0, 1, W, m1, W, m1));             // W = U2
  SF_TRY(prod(m1, n1, k1, S3, m1, 0, T3, k1, 1, 1.0, 1, W, m1, V, m1));             // V = U3
  SF_TRY(prod(m1, n1, k1, S1, m1, 0, T1, k1, 1, 1.0, 0, nullptr, 0, X, m1));        // X = P5
  T* C21 = C + m1;
  const T* Cin21 = cin ? cin + m1 : nullptr;
  SF_TRY(comb<T>(m2, n1, one, Cin21, ldcin, 0, m2, n1, alpha, V, m1, 0, m1, n1, C21, ldc, st));        // C21 = b Cin21 + a U3
  SF_TRY(prod(m2, n1, k2, A22, lda, ak, T4, k1, 1, -al, 1, C21, ldc, C21, ldc));   // C21 -= a P4
  SF_TRY(comb<T>(m1, n1, one, V, m1, 0, m1, n1, one, X, m1, 0, m1, n1, V, m1, st));                    // V = U7
  SF_TRY(comb<T>(m2, n2, one, cin ? Cin21 + n1 * ldcin : nullptr, ldcin, 0, m2, n2, alpha, V, m1, 0, m1, n1,
                 C21 + n1 * ldc, ldc, st));                                                            // C22
  SF_TRY(comb<T>(m1, n1, one, W, m1, 0, m1, n1, one, X, m1, 0, m1, n1, W, m1, st));                    // W = U4
  SF_TRY(comb<T>(m1, n2, one, cin ? cin + n1 * ldcin : nullptr, ldcin, 0, m1, n2, alpha, W, m1, 0, m1, n1,
                 C + n1 * ldc, ldc, st));                                                              // C12 = b Cin12 + a U4
  SF_TRY(prod(m1, n2, k2, S4, m1, 0, B22, ldb, bk, al, 1, C + n1 * ldc, ldc, C + n1 * ldc, ldc));      // C12 += a P3
#undef SF_TRY
  return cudaSuccess;
}

// C = Cin - op(A) op(B) by Strassen-Winograd (the flush; strassen_cfg().levels levels).
template <typename T>
inline cudaError_t strassen_sub(int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, int ak, const T* B,
                                int64_t ldb, int bk, const T* Cin, int64_t ldcin, T* C, int64_t ldc,
                                const long long* fail, cudaStream_t st) {
  return strassen_gen<T>(M, N, K, T(-1), A, lda, ak, B, ldb, bk, 1, Cin, ldcin, C, ldc, fail, st, strassen_cfg().levels);
}

inline bool strassen_applies(int64_t M, int64_t N, int64_t K) {
  const StrassenCfg& c = strassen_cfg();
  return c.levels > 0 && M >= c.min_dim && N >= c.min_dim && K >= 32;
}

// The flush C = Cin - op(A) op(B) (no mask): LU's A[c:n,c:n] -= R_L R_U, QR's M -= B_Q C.
template <typename T>
inline cudaError_t flush_general(int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, int ak, const T* B,
                                 int64_t ldb, int bk, const T* Cin, int64_t ldcin, T* C, int64_t ldc,
                                 const long long* fail, cudaStream_t st, int max_ctas = 0) {
  if (sizeof(T) == 8 && strassen_applies(M, N, K))
    return strassen_sub<T>(M, N, K, A, lda, ak, B, ldb, bk, Cin, ldcin, C, ldc, fail, st);
  return gemm_sub<T>(M, N, K, A, lda, ak, B, ldb, bk, Cin, ldcin, C, ldc, kMaskNone, fail, st, max_ctas);
}

// The Cholesky flush C = Cin - R R^T on the lower triangle.  With Strassen on: the two
// diagonal halves stay lower-masked SYRKs, the off-diagonal block C21 -= R2 R1^T is the
// Strassen product.
template <typename T>
inline cudaError_t flush_lower(int64_t M, int64_t K, const T* R, int64_t ldr, const T* Cin, int64_t ldcin, T* C,
                               int64_t ldc, const long long* fail, cudaStream_t st, int max_ctas = 0) {
  const int64_t h = (M + 1) / 2;
  if (!(sizeof(T) == 8 && strassen_applies(M - h, h, K)))
    return gemm_sub<T>(M, M, K, R, ldr, 0, R, ldr, 0, Cin, ldcin, C, ldc, kMaskLower, fail, st, max_ctas);
  cudaError_t e = gemm_sub<T>(h, h, K, R, ldr, 0, R, ldr, 0, Cin, ldcin, C, ldc, kMaskLower, fail, st);
  if (e != cudaSuccess) return e;
  e = strassen_sub<T>(M - h, h, K, R + h, ldr, 0, R, ldr, 0, Cin + h, ldcin, C + h, ldc, fail, st);
  if (e != cudaSuccess) return e;
  return gemm_sub<T>(M - h, M - h, K, R + h, ldr, 0, R + h, ldr, 0, Cin + h + h * ldcin, ldcin, C + h + h * ldc, ldc,
                     kMaskLower, fail, st);
}

// SM reservation for the lookahead panel.  The flush's second part runs concurrently with
// the factorization of the next panel; the panel is a chain of ~30 short dependent kernels,
// and when the flush holds every SM each of them waits for a flush CTA to retire.  When the
// remaining flush is small (its flops per panel-step below SF_RESERVE_FLOPS, default 4e10,
// i.e. ~1.5 ms), the flush can run on a bounded grid that leaves SF_PANEL_SMS SMs to the
// panel stream.  Off by default: measured on cfg2/cfg3/cfg5 it changes the time by < 1%
// (the panel chain is bound by its own latency, not by waiting for SMs) and costs cfg2 3%.
// Returns the CTA bound for gemm_sub (0 = unbounded).
inline int flush_ctas_for_panel(double flush_flops) {
  static const int reserve = [] { const char* e = getenv("SF_PANEL_SMS"); return e ? atoi(e) : 0; }();
  static const double thresh = [] { const char* e = getenv("SF_RESERVE_FLOPS"); return e ? atof(e) : 4e10; }();
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  if (reserve <= 0 || flush_flops > thresh || reserve >= sms) return 0;
  return 2 * (sms - reserve);   // two CTAs per SM on the others
}

// ------------------------------------------------------------------ Cholesky
template <typename T>
inline cudaError_t chol_panel_rec(int64_t m, int64_t w, const T* src, int64_t lds, T* dst, int64_t ldd,
                                  int64_t col0, long long* fail, cudaStream_t st) {
  const bool p64 = m <= chol_p64_maxm();
  const int leaf = p64 ? 64 : chol_leaf_width();
  if (w <= leaf)
    return p64 ? chol_panel64<T>(m, (int)w, src, lds, dst, ldd, col0, fail, st)
               : chol_leaf<T>(m, (int)w, src, lds, dst, ldd, col0, fail, st);
  const int64_t h = half_of(w, leaf);
  cudaError_t e = chol_panel_rec<T>(m, h, src, lds, dst, ldd, col0, fail, st);
  if (e != cudaSuccess) return e;
  // columns [h, w), rows [h, m):  X -= L[h:m, 0:h] * L[h:w, 0:h]^T  (lower part only)
  e = gemm_sub<T>(m - h, w - h, h, dst + h, ldd, 0, dst + h, ldd, 0, src + h + h * lds, lds, dst + h + h * ldd, ldd,
                  kMaskLower, fail, st);
  if (e != cudaSuccess) return e;
  return chol_panel_rec<T>(m - h, w - h, dst + h + h * ldd, ldd, dst + h + h * ldd, ldd, col0 + h, fail, st);
}

// ------------------------------------------------------------------ fp32 Cholesky panel
// K-major 3xTF32 split of one panel (hi / lo), row r / column k relative to the panel's
// top-left entry: element at h[r*ldk + k].
struct SplitBuf {
  float* h; float* l; int64_t ldk;
  SplitBuf at(int64_t r, int64_t k) const { return SplitBuf{h + r * ldk + k, l + r * ldk + k, ldk}; }
};

inline cudaError_t syrk_tf32(int64_t M, int64_t N, int64_t K, const SplitBuf& a, const SplitBuf& b, const float* Cin,
                             int64_t ldcin, float* C, int64_t ldc, const long long* fail, cudaStream_t st) {
  Tf32Gemm g{M, N, K, a.h, a.l, a.ldk, b.h, b.l, b.ldk, Cin, ldcin, C, ldc, kMaskLower, 0, fail};
  return gemm_tf32x3(g, st);
}

// Same recursion as chol_panel_rec; the left half's columns are split (hi/lo, K-major) into
// `sb` before the 3xTF32 correction of the right half.  On return the panel's columns are
// split for rows [w, m) only up to the last left half: the caller splits the whole panel
// for the flush.
// fp32 panels whose leaves are one-launch panels (panel64) write the split of every row below
// their diagonal blocks themselves (the substitution's final registers), so neither the
// recursion nor the caller needs a separate split pass over those rows.
inline bool chol32_fused_split(int64_t m) {
  // measured slower (cfg3 fp32 23.2 vs 22.3 ms, cfg5 fp32 ~499 vs ~494 ms): each thread stores
  // its own row's split (one sector per lane) where split_tf32 transposes through shared memory
  static const int on = [] { const char* e = getenv("SF_CHOL32_FUSED_SPLIT"); return e ? atoi(e) : 0; }();
  return on && m <= chol32_p64_maxm();
}

inline cudaError_t chol_panel_rec_f32(int64_t m, int64_t w, const float* src, int64_t lds, float* dst, int64_t ldd,
                                      int64_t col0, SplitBuf sb, long long* fail, cudaStream_t st) {
  const bool p64 = m <= chol32_p64_maxm();
  const int leaf = p64 ? 64 : chol_leaf_width();
  if (w <= leaf)
    return p64 ? chol_panel64<float>(m, (int)w, src, lds, dst, ldd, col0, fail, st,
                                     chol32_fused_split(m) ? sb.h : nullptr, sb.l, sb.ldk)
               : chol_leaf<float>(m, (int)w, src, lds, dst, ldd, col0, fail, st);
  const int64_t h = half_of(w, leaf);
  cudaError_t e = chol_panel_rec_f32(m, h, src, lds, dst, ldd, col0, sb, fail, st);
  if (e != cudaSuccess) return e;
  if (!chol32_fused_split(m)) e = split_tf32(m - h, h, dst + h, ldd, sb.at(h, 0).h, sb.at(h, 0).l, sb.ldk, st);
  if (e != cudaSuccess) return e;
  const SplitBuf lh = sb.at(h, 0);
  e = syrk_tf32(m - h, w - h, h, lh, lh, src + h + h * lds, lds, dst + h + h * ldd, ldd, fail, st);
  if (e != cudaSuccess) return e;
  return chol_panel_rec_f32(m - h, w - h, dst + h + h * ldd, ldd, dst + h + h * ldd, ldd, col0 + h, sb.at(h, h), fail,
                            st);
}

// ------------------------------------------------------------------ LU
template <typename T>
inline cudaError_t lu_panel_rec(int64_t m, int64_t w, int64_t ncr, const T* src, int64_t lds, T* dst, int64_t ldd,
                                int64_t col0, const T* tol, long long* fail, cudaStream_t st) {
  const bool p64 = lu_p64_on();
  const int leaf = p64 ? 64 : leaf_width();
  if (w <= leaf)
    return p64 ? lu_panel64<T>(m, ncr, (int)w, src, lds, dst, ldd, col0, tol, fail, st)
               : lu_leaf<T>(m, ncr, (int)w, src, lds, dst, ldd, col0, tol, fail, st);
  const int64_t h = half_of(w, leaf);
  cudaError_t e = lu_panel_rec<T>(m, h, ncr + (w - h), src, lds, dst, ldd, col0, tol, fail, st);
  if (e != cudaSuccess) return e;
  // L part and U11 part of the right half: rows [h, m), cols [h, w) -= L[h:m, 0:h] U[0:h, h:w]
  e = gemm_sub<T>(m - h, w - h, h, dst + h, ldd, 0, dst + h * ldd, ldd, 1, src + h + h * lds, lds, dst + h + h * ldd,
                  ldd, kMaskNone, fail, st);
  if (e != cudaSuccess) return e;
  // U rows [h, w) of the columns right of the panel: -= L[h:w, 0:h] U[0:h, w:w+ncr]
  if (ncr > 0) {
    e = gemm_sub<T>(w - h, ncr, h, dst + h, ldd, 0, dst + w * ldd, ldd, 1, src + h + w * lds, lds, dst + h + w * ldd,
                    ldd, kMaskNone, fail, st);
    if (e != cudaSuccess) return e;
  }
  return lu_panel_rec<T>(m - h, w - h, ncr, dst + h + h * ldd, ldd, dst + h + h * ldd, ldd, col0 + h, tol, fail, st);
}

// U rows [0, w) of ncols columns (at U, ldu; in place) against the factored w x w diagonal
// block L11 (at l11, ldl): the U part of lu_panel_rec alone, with the same halving, so
// every element sees the same grouped corrections in the same order.
template <typename T>
inline cudaError_t lu_usolve_rec(int64_t w, int64_t ncols, const T* l11, int64_t ldl, T* U, int64_t ldu,
                                 long long* fail, cudaStream_t st) {
  const int leaf = leaf_width();
  if (w <= leaf) return lu_usolve_leaf<T>(ncols, (int)w, l11, ldl, U, ldu, U, ldu, fail, st);
  const int64_t h = half_of(w, leaf);
  cudaError_t e = lu_usolve_rec<T>(h, ncols, l11, ldl, U, ldu, fail, st);
  if (e != cudaSuccess) return e;
  // U rows [h, w) -= L[h:w, 0:h] U[0:h, :]
  e = gemm_sub<T>(w - h, ncols, h, l11 + h, ldl, 0, U, ldu, 1, U + h, ldu, U + h, ldu, kMaskNone, fail, st);
  if (e != cudaSuccess) return e;
  return lu_usolve_rec<T>(w - h, ncols, l11 + h + h * ldl, ldl, U + h, ldu, fail, st);
}

// ------------------------------------------------------------------ triangular solves (f4)
// Forward: L X = B, L lower non-unit (w x w at l, ldl), B w x ncols in place — the U-row
// solve of the LU panel is exactly this (lu_usolve_rec).
// Backward: T X = B, T upper (trans = 0: T = U or R as stored; trans = 1: T = L^T), unit or
// not; recursive halving, bottom half first, the coupling by one GEMM.
template <typename T>
inline cudaError_t trsm_upper_rec(int64_t w, int64_t ncols, const T* t, int64_t ldt, int trans, int unit, T* B,
                                  int64_t ldb, cudaStream_t st) {
  const int leaf = leaf_width();
  if (w <= leaf) return trsm_upper_leaf<T>(ncols, (int)w, t, ldt, trans, unit, B, ldb, st);
  const int64_t h = half_of(w, leaf);
  // bottom rows [h, w): T22 at (h, h)
  cudaError_t e = trsm_upper_rec<T>(w - h, ncols, t + h + h * ldt, ldt, trans, unit, B + h, ldb, st);
  if (e != cudaSuccess) return e;
  // B[0:h] -= T12 X2,  T12(i, k) = T(i, h + k): trans 0 -> t[i + (h+k)*ldt] ; trans 1 -> t[(h+k) + i*ldt]
  if (trans) e = gemm_sub<T>(h, ncols, w - h, t + h, ldt, 1, B + h, ldb, 1, B, ldb, B, ldb, kMaskNone, nullptr, st);
  else e = gemm_sub<T>(h, ncols, w - h, t + h * ldt, ldt, 0, B + h, ldb, 1, B, ldb, B, ldb, kMaskNone, nullptr, st);
  if (e != cudaSuccess) return e;
  return trsm_upper_rec<T>(h, ncols, t, ldt, trans, unit, B, ldb, st);
}

// ------------------------------------------------------------------ QR
inline int splitk_for(int64_t M, int64_t N, int64_t K) {
  // long-K products run on the 64 x 64 DMMA tiles, 4 CTAs per SM: aim at two waves
  const int64_t tiles = ((M + 63) / 64) * ((N + 63) / 64);
  int64_t sp = (8 * 148 + tiles - 1) / tiles;
  const int64_t maxsp = K / 256 > 1 ? K / 256 : 1;
  if (sp > maxsp) sp = maxsp;
  if (sp > 16) sp = 16;
  return (int)(sp < 1 ? 1 : sp);
}

struct QrWork {
  void* cw; void* split; void* mgs;
  int64_t split_elems;
};

// Project the columns [0, wc) of V (n rows) against the orthonormal columns Qb (n x k):
//   C = Qb^T V ; V = Vin - Qb C   (PAPER.md:147-155 restricted to the given columns)
template <typename T>
inline cudaError_t qr_project(int64_t n, int64_t k, int64_t wc, const T* Qb, int64_t ldq, const T* Vin, int64_t ldvin,
                              T* V, int64_t ldv, T* Cw, T* split, int64_t split_elems, long long* fail,
                              cudaStream_t st) {
  int sp = splitk_for(k, wc, n);
  while (sp > 1 && (int64_t)sp * k * wc > split_elems) --sp;
  Gemm<T> g1{k, wc, n, Qb, ldq, 1, Vin, ldvin, 1, nullptr, 0, Cw, k, 1.0, 0, kMaskNone, sp, split, fail};
  cudaError_t e = run_gemm(g1, st);
  if (e != cudaSuccess) return e;
  return flush_general<T>(n, wc, k, Qb, ldq, 0, Cw, k, 1, Vin, ldvin, V, ldv, fail, st);
}

template <typename T>
inline cudaError_t qr_panel(int64_t n, int64_t w, const T* src, int64_t lds, T* dst, int64_t ldd, int64_t col0,
                           const T* tol, T* mgswork, T* Cw, T* split, int64_t split_elems, long long* fail,
                           cudaStream_t st) {
  const int64_t wmax = qr_mgs_max_width(n, (int)sizeof(T));
  if (w <= wmax) return qr_mgs_panel<T>(n, (int)w, src, lds, dst, ldd, col0, tol, mgswork, fail, st);
  // panel wider than one cooperative MGS launch holds: chunks, projected against the
  // finished chunks of the same panel (DESIGN.md §3 reading R12)
  for (int64_t z0 = 0; z0 < w; z0 += wmax) {
    const int64_t wc = (wmax < w - z0) ? wmax : w - z0;
    const T* vin = src + z0 * lds;
    int64_t ldvin = lds;
    if (z0 > 0) {
      cudaError_t e = qr_project<T>(n, z0, wc, dst, ldd, vin, ldvin, dst + z0 * ldd, ldd, Cw, split, split_elems, fail, st);
      if (e != cudaSuccess) return e;
      vin = dst + z0 * ldd;
      ldvin = ldd;
    }
    cudaError_t e = qr_mgs_panel<T>(n, (int)wc, vin, ldvin, dst + z0 * ldd, ldd, col0 + z0, tol, mgswork, fail, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sf
