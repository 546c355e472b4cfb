// driver.cu — the step-s schedule and the C ABI (include/stepfact.h).
//
// Schedule: z := 0; for c in 0..n-1: if c == z+s then
// flush and z := c.  In panel terms: panels p = [p*s, min((p+1)s, n)) are factored in
// order; after every panel except the last, ONE rectangular product updates the trailing
// matrix.  Flush count = floor((n-1)/s).
//
// Out-of-place support: every kernel reads from `src` and writes to `dst`.  The first
// panel and the first flush read the caller's A; from then on everything lives in the
// output buffer (the first flush rewrites the whole trailing lower triangle / square), so
// A is never modified unless the caller passes dA == dOut.
//
// Panels wider than the leaf width are factored recursively: factor the left half,
// subtract its contribution from the right half with one GEMM (the same terms the paper's
// k-loops subtract, grouped), factor the right half.  DESIGN.md §5 discusses why.
#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "drv.cuh"

namespace sf {

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local char g_last_error[512] = "";

// profiling hook state (drv.cuh ProfScope)
bool g_prof = false;
std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_event_pool;
cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) { cudaEvent_t e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
  cudaEvent_t e; cudaEventCreate(&e); return e;
}


std::recursive_mutex& api_mutex() {
  static std::recursive_mutex m;
  return m;
}

int fail_with(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}






template <typename T>
static int chol_run(int64_t n, const Sched& S, const T* A, int64_t lda, T* L, int64_t ldl, int64_t* d_info,
                    cudaStream_t st, PanelHook* hook = nullptr) {
  Workspace ws;
  SF_CUDA(ws.init(4096, st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  SF_CUDA(init_fail(fail, st));
  if constexpr (std::is_same<T, double>::value) {
    // small n: the whole schedule in one thread-block cluster, shared-memory resident (small.cu)
    if (S.fixed() && chol_small_applies(n, S.fixed(), 8)) {
      {
        ProfScope ps(1, 0.0, st);
        SF_CUDA(chol_small(n, S.fixed(), A, lda, L, ldl, fail, st));
      }
      if (hook) SF_CUDA(hook->done(0, n, st));
      SF_CUDA(finish_info(fail, d_info, st));
      return SF_OK;
    }
  }
  Side* sd = nullptr;
  const bool la = lookahead_on() && S.P() > 1;
  if (la) { SF_CUDA(side_stream(sd)); ws.join(sd->st); }
  {
    ProfScope ps(1, 0.0, st);
    const int64_t w0 = S.w(0);
    SF_CUDA(chol_panel_rec<T>(n, w0, A, lda, L, ldl, 0, fail, st));
    if (hook) SF_CUDA(hook->done(0, w0, st));
  }
  for (int64_t p = 0; p + 1 < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p), c = z + w;
    const int64_t w2 = S.w(p + 1), m = n - c;
    const T* src = (z == 0) ? A : L;
    const int64_t lds = (z == 0) ? lda : ldl;
    const T* R = L + c + z * ldl;   // R = L[c:n, z:c)
    if (la) {
      {  // flush, part 1: the columns of the next panel
        ProfScope ps(0, (double)w * ((double)m * (m + 1) - (double)(m - w2) * (m - w2 + 1)), st);
        SF_CUDA(gemm_sub<T>(m, w2, w, R, ldl, 0, R, ldl, 0, src + c + c * lds, lds, L + c + c * ldl, ldl, kMaskLower,
                            fail, st));
      }
      SF_CUDA(fork_join(*sd, st, sd->st));
      {
        ProfScope ps(1, 0.0, sd->st);
        SF_CUDA(chol_panel_rec<T>(m, w2, L + c + c * ldl, ldl, L + c + c * ldl, ldl, c, fail, sd->st));
        if (hook) SF_CUDA(hook->done(c, w2, sd->st));
      }
      if (m > w2) {  // flush, part 2: the rest of the trailing matrix, concurrently with the panel
        const int64_t c2 = c + w2;
        const double fl = (double)w * (double)(m - w2) * (double)(m - w2 + 1);
        ProfScope ps(0, fl, st);
        SF_CUDA(flush_lower<T>(m - w2, w, R + w2, ldl, src + c2 + c2 * lds, lds, L + c2 + c2 * ldl, ldl, fail, st,
                               flush_ctas_for_panel(fl)));
      }
      SF_CUDA(fork_join(*sd, sd->st, st));
    } else {
      {  // flush: A[c:n,c:n] -= R R^T
        ProfScope ps(0, (double)w * (double)m * (double)(m + 1), st);
        SF_CUDA(flush_lower<T>(m, w, R, ldl, src + c + c * lds, lds, L + c + c * ldl, ldl, fail, st));
      }
      ProfScope ps(1, 0.0, st);
      SF_CUDA(chol_panel_rec<T>(m, w2, L + c + c * ldl, ldl, L + c + c * ldl, ldl, c, fail, st));
      if (hook) SF_CUDA(hook->done(c, w2, st));
    }
  }
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}


// fp32 Cholesky: fp32 storage and panel, 3xTF32 tcgen05 flush.  Same
// schedule and lookahead as chol_run; each panel's split (hi/lo) lives in one of two
// buffers so the side stream can split panel p+1 while the flush of panel p reads panel p's.
static int chol_run_f32(int64_t n, const Sched& S, const float* A, int64_t lda, float* L, int64_t ldl,
                        int64_t* d_info, cudaStream_t st, PanelHook* hook = nullptr) {
  const int64_t ldk = (S.maxw() + 3) / 4 * 4;
  Workspace ws;
  SF_CUDA(ws.init(4096 + 4 * sizeof(float) * (size_t)n * ldk + 4 * 256, st));
  long long* fail = ws.take<long long>(2);
  SplitBuf sb[2];
  for (int b = 0; b < 2; ++b) {
    sb[b].h = ws.take<float>((size_t)n * ldk);
    sb[b].l = ws.take<float>((size_t)n * ldk);
    sb[b].ldk = ldk;
  }
  SF_CUDA(init_fail(fail, st));
  Side* sd = nullptr;
  const bool la = lookahead_on() && S.P() > 1;
  if (la) { SF_CUDA(side_stream(sd)); ws.join(sd->st); }
  {
    ProfScope ps(1, 0.0, st);
    const int64_t w0 = S.w(0);
    SF_CUDA(chol_panel_rec_f32(n, w0, A, lda, L, ldl, 0, sb[0], fail, st));
    if (hook) SF_CUDA(hook->done(0, w0, st));
    if (w0 < n && !chol32_fused_split(n))
      SF_CUDA(split_tf32(n - w0, w0, L + w0, ldl, sb[0].at(w0, 0).h, sb[0].at(w0, 0).l, ldk, st));
  }
  for (int64_t p = 0; p + 1 < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p), c = z + w;
    const int64_t w2 = S.w(p + 1), m = n - c;
    const float* src = (z == 0) ? A : L;
    const int64_t lds = (z == 0) ? lda : ldl;
    const SplitBuf R = sb[p & 1].at(w, 0);       // R = L[c:n, z:c), split
    SplitBuf& nxt = sb[(p + 1) & 1];
    cudaStream_t pst = la ? sd->st : st;
    if (la) {
      ProfScope ps(0, 3.0 * w * ((double)m * (m + 1) - (double)(m - w2) * (m - w2 + 1)), st);
      SF_CUDA(syrk_tf32(m, w2, w, R, R, src + c + c * lds, lds, L + c + c * ldl, ldl, fail, st));
      SF_CUDA(fork_join(*sd, st, pst));
    } else {
      ProfScope ps(0, 3.0 * w * (double)m * (double)(m + 1), st);
      SF_CUDA(syrk_tf32(m, m, w, R, R, src + c + c * lds, lds, L + c + c * ldl, ldl, fail, st));
    }
    {
      ProfScope ps(1, 0.0, pst);
      SF_CUDA(chol_panel_rec_f32(m, w2, L + c + c * ldl, ldl, L + c + c * ldl, ldl, c, nxt, fail, pst));
      if (hook) SF_CUDA(hook->done(c, w2, pst));
      if (w2 < m && !chol32_fused_split(m))
        SF_CUDA(split_tf32(m - w2, w2, L + c + w2 + c * ldl, ldl, nxt.at(w2, 0).h, nxt.at(w2, 0).l, ldk, pst));
    }
    if (la) {
      if (m > w2) {
        const int64_t c2 = c + w2;
        ProfScope ps(0, 3.0 * w * (double)(m - w2) * (double)(m - w2 + 1), st);
        SF_CUDA(syrk_tf32(m - w2, m - w2, w, R.at(w2, 0), R.at(w2, 0), src + c2 + c2 * lds, lds, L + c2 + c2 * ldl, ldl,
                          fail, st));
      }
      SF_CUDA(fork_join(*sd, pst, st));
    }
  }
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}

static bool lu_part1_grouped() {
  static const int on = [] { const char* e = getenv("SF_LU_PART1_GROUPED"); return e ? atoi(e) : 1; }();
  return on != 0;
}

template <typename T>
static int64_t lu_la_min_m() {
  // fp64 default 0 (always: the first flush part is one grouped launch); fp32 keeps two
  // launches for it, where lookahead loses below m = 4096 (cfg2 fp32 8.7 vs 10.7 ms)
  static const int64_t v = [] {
    const char* e = getenv("SF_LU_LA_MIN_M");
    return e ? (int64_t)atoll(e) : (int64_t)(std::is_same<T, double>::value ? 0 : 4096);
  }();
  return v;
}

// Two-deep lookahead for LU (SF_LU_LA2; default on for fp64: cfg2 6.21 -> 5.57 ms, bench).  The flush of panel p is split three ways:
//   F1(p): the L-shaped region panel p+1 reads (its columns, rows >= c; its U rows, columns
//          right of it) — on the panel stream, right before panel p+1;
//   F2(p): the L-shaped region of panel p+2 — first on the main stream, so F1(p+1) (same
//          region, next contribution) can start as soon as it and panel p+1 are done;
//   F3(p): the rest, rows and columns >= the start of panel p+3 — main stream, overlapping
//          the panel chain.
// The critical chain is panel(p) -> F1(p) -> panel(p+1) -> ...; it no longer waits behind the
// bulk of the previous flush as in the one-deep scheme (where part 1 of flush p+1 queued
// behind all of part 2 of flush p).  Every element still receives the flushes p = 0, 1, ...
// in order, each from one tile with the same K order: the result is bitwise the same.
// fp32 keeps the one-deep scheme: its small L-shaped products each pay a 3xTF32 operand
// split and a workspace allocation on the critical path (cfg2 fp32: 9.48 vs 6.39 ms).
template <typename T>
static bool lu_la2_on() {
  static const int on = [] {
    const char* e = getenv("SF_LU_LA2");
    return e ? atoi(e) : (std::is_same<T, double>::value ? 1 : 0);
  }();
  return on != 0;
}

template <typename T>
static int lu_run_la2(int64_t n, const Sched& S, const T* A, int64_t lda, T* LU, int64_t ldd, int64_t* d_info,
                      cudaStream_t st, PanelHook* hook, long long* fail, T* tol) {
  Side* sd = nullptr;
  SF_CUDA(side_stream(sd));
  cudaStream_t ps = sd->st;
  SF_CUDA(fork_join(*sd, st, ps));
  {
    ProfScope pr(1, 0.0, ps);
    const int64_t w0 = S.w(0);
    SF_CUDA(lu_panel_rec<T>(n, w0, n - w0, A, lda, LU, ldd, 0, tol, fail, ps));
    if (hook) SF_CUDA(hook->done(0, w0, ps));
  }
  cudaEvent_t ev_pan = sd->event();
  SF_CUDA(cudaEventRecord(ev_pan, ps));
  cudaEvent_t ev_f2 = nullptr;   // F2(p-1) done (main stream)
  for (int64_t p = 0; p + 1 < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p), c = z + w;
    const int64_t w2 = S.w(p + 1), c2 = c + w2;
    const int64_t w3 = (p + 2 < S.P()) ? S.w(p + 2) : 0, c3 = c2 + w3;
    const T* src = (z == 0) ? A : LU;
    const int64_t lds = (z == 0) ? lda : ldd;
    const T* RL = LU + c + z * ldd;   // R_L = L[c:n, z:c)
    const T* RU = LU + z + c * ldd;   // R_U = U[z:c, c:n)
    // the L-shaped region of the panel [a, a + wl): its columns (rows >= a) and its U rows
    // (columns >= a + wl), as ONE grouped launch (fp64) — flush p restricted to it
    auto lshape = [&](int64_t a, int64_t wl, cudaStream_t s) -> int {
      if (wl <= 0) return SF_OK;
      const int64_t ma = n - a;
      ProfScope pf(0, 2.0 * w * ((double)ma * wl + (double)wl * (ma - wl)), s);
      const T* ra = RL + (a - c);
      if constexpr (std::is_same<T, double>::value) {
        GemmGroup g[2] = {};
        int ng = 0;
        g[ng].M = ma; g[ng].N = wl; g[ng].A = ra; g[ng].B = RU + (a - c) * ldd;
        g[ng].Cin = src + a + a * lds; g[ng].C = LU + a + a * ldd; ++ng;
        if (ma > wl) {
          g[ng].M = wl; g[ng].N = ma - wl; g[ng].A = ra; g[ng].B = RU + (a + wl - c) * ldd;
          g[ng].Cin = src + a + (a + wl) * lds; g[ng].C = LU + a + (a + wl) * ldd; ++ng;
        }
        GemmF64 p64{0, 0, w, nullptr, ldd, nullptr, ldd, nullptr, lds, nullptr, ldd, -1.0, 1, 1, nullptr, fail};
        SF_CUDA(gemm_f64_grouped(p64, g, ng, 0, 1, kMaskNone, s));
      } else {
        SF_CUDA(gemm_sub<T>(ma, wl, w, ra, ldd, 0, RU + (a - c) * ldd, ldd, 1, src + a + a * lds, lds,
                            LU + a + a * ldd, ldd, kMaskNone, fail, s));
        if (ma > wl)
          SF_CUDA(gemm_sub<T>(wl, ma - wl, w, ra, ldd, 0, RU + (a + wl - c) * ldd, ldd, 1, src + a + (a + wl) * lds,
                              lds, LU + a + (a + wl) * ldd, ldd, kMaskNone, fail, s));
      }
      return SF_OK;
    };
    // panel stream: F1(p) (after F2(p-1) wrote the same region), then panel p+1
    if (ev_f2) SF_CUDA(cudaStreamWaitEvent(ps, ev_f2, 0));
    if (int rc = lshape(c, w2, ps)) return rc;
    {
      ProfScope pr(1, 0.0, ps);
      SF_CUDA(lu_panel_rec<T>(n - c, w2, n - c2, LU + c + c * ldd, ldd, LU + c + c * ldd, ldd, c, tol, fail, ps));
      if (hook) SF_CUDA(hook->done(c, w2, ps));
    }
    // main stream: F2(p), F3(p) once panel p is final
    SF_CUDA(cudaStreamWaitEvent(st, ev_pan, 0));
    ev_pan = sd->event();
    SF_CUDA(cudaEventRecord(ev_pan, ps));   // panel p+1 final (read by F2/F3(p+1))
    if (int rc = lshape(c2, w3, st)) return rc;
    ev_f2 = sd->event();
    SF_CUDA(cudaEventRecord(ev_f2, st));
    if (c3 < n) {
      const int64_t m3 = n - c3;
      const double fl = 2.0 * w * (double)m3 * (double)m3;
      ProfScope pf(0, fl, st);
      SF_CUDA(flush_general<T>(m3, m3, w, RL + (c3 - c), ldd, 0, RU + (c3 - c) * ldd, ldd, 1, src + c3 + c3 * lds, lds,
                               LU + c3 + c3 * ldd, ldd, fail, st));
    }
  }
  SF_CUDA(fork_join(*sd, ps, st));
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}

template <typename T>
static int lu_run(int64_t n, const Sched& S, const T* A, int64_t lda, T* LU, int64_t ldd, int64_t* d_info,
                  cudaStream_t st, PanelHook* hook = nullptr) {
  Workspace ws;
  SF_CUDA(ws.init(16384, st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  T* tol = ws.take<T>(1);
  double* part = ws.take<double>(512);
  SF_CUDA(init_fail(fail, st));
  SF_CUDA(frob_norm_tol<T>(n, A, lda, tol, part, st));
  Side* sd = nullptr;
  const bool la = lookahead_on() && S.P() > 1;
  if (la) { SF_CUDA(side_stream(sd)); ws.join(sd->st); }
  if (la && lu_la2_on<T>()) return lu_run_la2<T>(n, S, A, lda, LU, ldd, d_info, st, hook, fail, tol);
  {
    ProfScope ps(1, 0.0, st);
    const int64_t w0 = S.w(0);
    SF_CUDA(lu_panel_rec<T>(n, w0, n - w0, A, lda, LU, ldd, 0, tol, fail, st));
    if (hook) SF_CUDA(hook->done(0, w0, st));   // L[0:n, 0:w0) and U[0:w0, w0:n) are final
  }
  for (int64_t p = 0; p + 1 < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p), c = z + w;
    const int64_t w2 = S.w(p + 1), m = n - c;
    const T* src = (z == 0) ? A : LU;
    const int64_t lds = (z == 0) ? lda : ldd;
    const T* RL = LU + c + z * ldd;   // R_L = L[c:n, z:c)
    const T* RU = LU + z + c * ldd;   // R_U = U[z:c, c:n)
    // SF_LU_LA_MIN_M: lookahead only while the trailing matrix is larger (default 0 =
    // always).  With the L-shaped first flush part as two launches, lookahead lost at
    // n = 4096 (6.44 vs 6.26 ms without); as ONE grouped launch it wins everywhere
    // (n = 4096: 5.94 ms; n = 8192 s = 64: 23.44 vs 24.47; n = 16384: 122.3 vs 123.3)
    const bool lap = la && m > lu_la_min_m<T>();
    cudaStream_t pst = lap ? sd->st : st;
    if (lap) {
      ProfScope ps(0, 2.0 * w * ((double)m * m - (double)(m - w2) * (m - w2)), st);
      // flush, part 1: columns [c, c+w2) (all rows >= c) and rows [c, c+w2) right of them —
      // fp64: the two blocks of the L-shaped region in ONE grouped launch
      bool done1 = false;
      if constexpr (std::is_same<T, double>::value) {
        if (lu_part1_grouped()) {
          GemmGroup g[2] = {};
          int ng = 0;
          g[ng].M = m; g[ng].N = w2; g[ng].off = 0; g[ng].A = RL; g[ng].B = RU;
          g[ng].Cin = src + c + c * lds; g[ng].C = LU + c + c * ldd; ++ng;
          if (m > w2) {
            const int64_t c2 = c + w2;
            g[ng].M = w2; g[ng].N = m - w2; g[ng].off = 0; g[ng].A = RL; g[ng].B = RU + w2 * ldd;
            g[ng].Cin = src + c + c2 * lds; g[ng].C = LU + c + c2 * ldd; ++ng;
          }
          GemmF64 p64{0, 0, w, nullptr, ldd, nullptr, ldd, nullptr, lds, nullptr, ldd, -1.0, 1, 1, nullptr, fail};
          SF_CUDA(gemm_f64_grouped(p64, g, ng, 0, 1, kMaskNone, st));
          done1 = true;
        }
      }
      if (!done1) {
        SF_CUDA(gemm_sub<T>(m, w2, w, RL, ldd, 0, RU, ldd, 1, src + c + c * lds, lds, LU + c + c * ldd, ldd, kMaskNone,
                            fail, st));
        if (m > w2) {
          const int64_t c2 = c + w2;
          SF_CUDA(gemm_sub<T>(w2, m - w2, w, RL, ldd, 0, RU + w2 * ldd, ldd, 1, src + c + c2 * lds, lds,
                              LU + c + c2 * ldd, ldd, kMaskNone, fail, st));
        }
      }
      SF_CUDA(fork_join(*sd, st, pst));
    } else {
      ProfScope ps(0, 2.0 * w * (double)m * (double)m, st);
      SF_CUDA(flush_general<T>(m, m, w, RL, ldd, 0, RU, ldd, 1, src + c + c * lds, lds, LU + c + c * ldd, ldd, fail,
                               st));
    }
    {
      ProfScope ps(1, 0.0, pst);
      SF_CUDA(lu_panel_rec<T>(m, w2, m - w2, LU + c + c * ldd, ldd, LU + c + c * ldd, ldd, c, tol, fail, pst));
      if (hook) SF_CUDA(hook->done(c, w2, pst));
    }
    if (lap) {
      if (m > w2) {  // flush, part 2: the remaining trailing block, concurrently with the panel
        const int64_t c2 = c + w2;
        const double fl = 2.0 * w * (double)(m - w2) * (double)(m - w2);
        ProfScope ps(0, fl, st);
        SF_CUDA(flush_general<T>(m - w2, m - w2, w, RL + w2, ldd, 0, RU + w2 * ldd, ldd, 1, src + c2 + c2 * lds, lds,
                                 LU + c2 + c2 * ldd, ldd, fail, st, flush_ctas_for_panel(fl)));
      }
      SF_CUDA(fork_join(*sd, pst, st));
    }
  }
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}


// Early R row blocks on a low-priority stream (SF_QR_EARLY_R=1): measured slower — the
// long-K R tiles hold SM slots the flushes need (cfg4 89.3 vs 83.8 ms) — off by default.
static bool qr_early_r_on() {
  static const int on = [] { const char* e = getenv("SF_QR_EARLY_R"); return e ? atoi(e) : 0; }();
  return on != 0;
}

template <typename T>
static int qr_run(int64_t n, const Sched& S, const T* A, int64_t lda, T* Q, int64_t ldq, T* R, int64_t ldr,
                  int64_t* d_info, cudaStream_t st, PanelHook* hook = nullptr) {
  const int64_t s = S.maxw();
  const int64_t wmax = qr_mgs_max_width(n, (int)sizeof(T));
  const int64_t wcap = s < wmax ? s : wmax;
  const size_t mgs_elems = qr_mgs_work_elems(n, (int)wcap, (int)sizeof(T)) + 64;
  const int64_t cw_elems = s * n;
  int64_t split_elems = 0;
  for (int64_t p = 0; p < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p);
    if (z + w < n) {
      const int sp = splitk_for(w, n - z - w, n);
      if ((int64_t)sp * w * (n - z - w) > split_elems) split_elems = (int64_t)sp * w * (n - z - w);
    }
  }
  if (s > wmax) {
    const int sp = splitk_for(s, wmax, n);
    if ((int64_t)sp * s * wmax > split_elems) split_elems = (int64_t)sp * s * wmax;
  }
  Workspace ws;
  SF_CUDA(ws.init(sizeof(T) * (mgs_elems + 2 * cw_elems + 2 * split_elems) + 16384 + 8 * 256, st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  T* tol = ws.take<T>(1);
  double* part = ws.take<double>(512);
  T* mgsw = ws.take<T>(mgs_elems);
  T* Cw = ws.take<T>(cw_elems);
  T* split = ws.take<T>(split_elems > 0 ? split_elems : 1);
  // the side stream's wide-panel chunk projections get their own scratch
  T* Cw2 = s > wmax ? ws.take<T>(cw_elems) : Cw;
  T* split2 = s > wmax ? ws.take<T>(split_elems > 0 ? split_elems : 1) : split;
  SF_CUDA(init_fail(fail, st));
  SF_CUDA(cudaMemsetAsync(mgsw, 0, sizeof(T) * mgs_elems, st));   // MGS flags (epochs start at 0)
  SF_CUDA(frob_norm_tol<T>(n, A, lda, tol, part, st));
  Side* sd = nullptr;
  const bool la = lookahead_on() && S.P() > 1;
  if (la) { SF_CUDA(side_stream(sd)); ws.join(sd->st); }
  // R := Q^T A by row blocks as soon as their Q columns are final: the
  // rows [z, z+w) of R need only Q[:, z:z+w) (later flushes never touch it), so each block
  // runs on a low-priority stream in the SM slots the short-K flushes leave idle, instead
  // of one n^3 product after the last panel.  Every element is the same K-ordered dot
  // product as in the one-shot product (tile-local DMMA accumulation over k = 0..n-1).
  Side* rs = nullptr;
  const bool early_r = qr_early_r_on();
  if (early_r) {
    SF_CUDA(low_stream(rs));
    ws.join(rs->st);
    SF_CUDA(fork_join(*rs, st, rs->st));
    SF_CUDA(zero_strict_lower<T>(n, R, ldr, rs->st));
  }
  auto r_rows = [&](int64_t z, int64_t w, cudaStream_t from) -> int {
    if (!early_r) return SF_OK;
    SF_CUDA(fork_join(*rs, from, rs->st));
    ProfScope ps(2, (double)w * (double)n * (double)(2 * (n - z) - w + 1), rs->st);
    Gemm<T> g{w, n - z, n, Q + z * ldq, ldq, 1, A + z * lda, lda, 1, nullptr, 0, R + z + z * ldr, ldr, 1.0, 0,
              kMaskUpper, 1, nullptr, fail};
    SF_CUDA(run_gemm(g, rs->st));
    return SF_OK;
  };
  {
    ProfScope ps(1, 0.0, st);
    const int64_t w0 = S.w(0);
    SF_CUDA(qr_panel<T>(n, w0, A, lda, Q, ldq, 0, tol, mgsw, Cw, split, split_elems, fail, st));
    if (hook) SF_CUDA(hook->done(0, w0, st));   // Q[:, 0:w0) is final
  }
  if (int rc = r_rows(0, S.w(0), st)) return rc;
  for (int64_t p = 0; p + 1 < S.P(); ++p) {
    const int64_t z = S.z(p), w = S.w(p), c = z + w;
    const int64_t w2 = S.w(p + 1), m = n - c;
    const T* src = (z == 0) ? A : Q;           // M := copy of A lives in Q
    const int64_t lds = (z == 0) ? lda : ldq;
    const T* BQ = Q + z * ldq;                 // B_Q = Q[:, z:c)
    // flush: C = B_Q^T B_M, M[:, c:n] -= B_Q C over all rows.  With
    // lookahead the columns of the next panel go first, the rest overlaps that panel.
    const int64_t first = la ? w2 : m;
    {
      ProfScope ps(0, 4.0 * (double)n * (double)w * (double)first, st);
      SF_CUDA(qr_project<T>(n, w, first, BQ, ldq, src + c * lds, lds, Q + c * ldq, ldq, Cw, split, split_elems,
                            fail, st));
    }
    cudaStream_t pst = st;
    if (la) { SF_CUDA(fork_join(*sd, st, sd->st)); pst = sd->st; }
    {
      ProfScope ps(1, 0.0, pst);
      SF_CUDA(qr_panel<T>(n, w2, Q + c * ldq, ldq, Q + c * ldq, ldq, c, tol, mgsw, Cw2, split2, split_elems, fail,
                          pst));
      if (hook) SF_CUDA(hook->done(c, w2, pst));
    }
    if (int rc = r_rows(c, w2, pst)) return rc;
    if (la) {
      if (m > w2) {
        const int64_t c2 = c + w2;
        ProfScope ps(0, 4.0 * (double)n * (double)w * (double)(m - w2), st);
        SF_CUDA(qr_project<T>(n, w, m - w2, BQ, ldq, src + c2 * lds, lds, Q + c2 * ldq, ldq, Cw, split, split_elems,
                              fail, st));
      }
      SF_CUDA(fork_join(*sd, sd->st, st));
    }
  }
  if (early_r) {
    SF_CUDA(fork_join(*rs, rs->st, st));   // the caller's stream waits for the last R block
  } else {
    // R := Q^T A: upper triangle on the tensor cores, exact zeros below
    SF_CUDA(zero_strict_lower<T>(n, R, ldr, st));
    ProfScope ps(2, (double)n * (double)n * (double)(n + 1), st);
    Gemm<T> g{n, n, n, Q, ldq, 1, A, lda, 1, nullptr, 0, R, ldr, 1.0, 0, kMaskUpper, 1, nullptr, fail};
    SF_CUDA(run_gemm(g, st));
  }
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}

// ------------------------------------------------------------------ argument checks
static int check_common(int64_t n, int64_t s, int dtype, const void* a, int64_t lda, const void* o, int64_t ldo) {
  if (n < 1) return fail_with(SF_EINVAL, "n=%lld < 1", (long long)n);
  if (s < 1 || s > n) return fail_with(SF_EINVAL, "step s=%lld outside [1, n=%lld]", (long long)s, (long long)n);
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  if (!a || !o) return fail_with(SF_EINVAL, "null matrix pointer");
  if (lda < n || ldo < n) return fail_with(SF_EINVAL, "leading dimension < n");
  const size_t elt = dtype == SF_F64 ? 8 : 4;
  if (((uintptr_t)a % elt) || ((uintptr_t)o % elt)) return fail_with(SF_EINVAL, "misaligned matrix pointer");
  if (a != o) {
    // out of place: the two n x n extents must not overlap
    const char* pa = (const char*)a; const char* po = (const char*)o;
    const char* ea = pa + elt * (size_t)(lda * (n - 1) + n);
    const char* eo = po + elt * (size_t)(ldo * (n - 1) + n);
    if (pa < eo && po < ea) return fail_with(SF_EINVAL, "input and output overlap without being identical");
  } else if (lda != ldo) {
    return fail_with(SF_EINVAL, "in-place call with lda != ld_out");
  }
  return SF_OK;
}

// ------------------------------------------------------------------ CUDA graphs
// A factorization is a fixed sequence of ~3 launches per panel for given (n, s, pointers),
// so repeated calls replay one captured CUDA graph instead of re-launching every kernel —
// the small configs (n = 256 .. 4096) are launch-bound.  The first call with a key runs
// eagerly (it also performs one-time setup: function attributes, streams, module loading),
// the second captures and instantiates, later ones replay.  Off when profiling is enabled,
// on the legacy default stream, inside a caller's own capture, or with SF_GRAPH=0.
struct GraphKey {
  int kind, dtype;
  int64_t n, s, lda, ld1, ld2;
  const void *a, *o1, *o2;
  int64_t* info;
  cudaStream_t st;
  bool operator==(const GraphKey& o) const {
    return kind == o.kind && dtype == o.dtype && n == o.n && s == o.s && lda == o.lda && ld1 == o.ld1 &&
           ld2 == o.ld2 && a == o.a && o1 == o.o1 && o2 == o.o2 && info == o.info && st == o.st;
  }
};
struct GraphEntry { GraphKey key; cudaGraphExec_t exec = nullptr; long long launches = 0; uint64_t used = 0; };
static std::vector<GraphEntry> g_graphs;
static uint64_t g_graph_clock = 0;
static bool graphs_on() {
  static int on = [] { const char* e = getenv("SF_GRAPH"); return e ? atoi(e) : 1; }();
  return on != 0;
}

template <typename F>
static int run_graph(const GraphKey& key, cudaStream_t st, F&& body) {
  if (!graphs_on() || g_prof || st == nullptr) return body();
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return body();
  GraphEntry* e = nullptr;
  for (auto& g : g_graphs)
    if (g.key == key) e = &g;
  if (!e) {   // first sighting: eager run, remember the key
    if (g_graphs.size() >= 8) {   // evict the least recently used
      size_t lru = 0;
      for (size_t i = 1; i < g_graphs.size(); ++i)
        if (g_graphs[i].used < g_graphs[lru].used) lru = i;
      if (g_graphs[lru].exec) cudaGraphExecDestroy(g_graphs[lru].exec);
      g_graphs.erase(g_graphs.begin() + lru);
    }
    GraphEntry ne;
    ne.key = key;
    ne.used = ++g_graph_clock;
    g_graphs.push_back(ne);
    return body();
  }
  e->used = ++g_graph_clock;
  if (!e->exec) {
    const long long l0 = g_launches.load();
    SF_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    const int rc = body();
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &g);
    const long long nl = g_launches.load() - l0;
    g_launches.fetch_sub(nl);   // captured, not launched
    if (rc != SF_OK || ec != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      if (rc != SF_OK) return rc;
      return fail_with(SF_ECUDA, "graph capture: %s", cudaGetErrorString(ec));
    }
    const cudaError_t ei = cudaGraphInstantiateWithFlags(&e->exec, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) { e->exec = nullptr; return fail_with(SF_ECUDA, "graph instantiate: %s", cudaGetErrorString(ei)); }
    e->launches = nl;
  }
  if (key.kind == 2) mgs_order_before(st);   // QR: persistent MGS grids never overlap
  SF_CUDA(cudaGraphLaunch(e->exec, st));
  if (key.kind == 2) mgs_order_after(st);
  count_launch((int)e->launches);
  return SF_OK;
}

template <typename T>
static int solve_run(int kind, int64_t n, int64_t nrhs, const T* F1, int64_t ld1, const T* F2, int64_t ld2, T* B,
                     int64_t ldb, cudaStream_t st) {
  if (nrhs == 0) return SF_OK;
  Workspace ws;
  SF_CUDA(ws.init(4096 + (kind == 2 ? sizeof(T) * (size_t)n * (size_t)nrhs + 256 : 0), st));
  long long* fail = ws.take<long long>(2);
  SF_CUDA(init_fail(fail, st));
  if (kind == 0) {          // A = L L^T: L Y = B, then L^T X = Y
    SF_CUDA(lu_usolve_rec<T>(n, nrhs, F1, ld1, B, ldb, fail, st));
    SF_CUDA(trsm_upper_rec<T>(n, nrhs, F1, ld1, 1, 0, B, ldb, st));
  } else if (kind == 1) {   // A = L U (U unit upper): L Y = B, then U X = Y
    SF_CUDA(lu_usolve_rec<T>(n, nrhs, F1, ld1, B, ldb, fail, st));
    SF_CUDA(trsm_upper_rec<T>(n, nrhs, F1, ld1, 0, 1, B, ldb, st));
  } else {                  // A = Q R: Y = Q^T B, R X = Y
    T* Y = ws.take<T>((size_t)n * nrhs);
    Gemm<T> g{n, nrhs, n, F1, ld1, 1, B, ldb, 1, nullptr, 0, Y, n, 1.0, 0, kMaskNone, 1, nullptr, fail};
    SF_CUDA(run_gemm(g, st));
    SF_CUDA(trsm_upper_rec<T>(n, nrhs, F2, ld2, 0, 0, Y, n, st));
    SF_CUDA(copy_matrix<T>(n, nrhs, Y, n, B, ldb, st));
  }
  return SF_OK;
}

}  // namespace sf

using namespace sf;

extern "C" {

int chol_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dL, int64_t ldl, int64_t* d_info,
                void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, s, dtype, dA, lda, dL, ldl);
  if (rc) return rc;
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const GraphKey key{0, dtype, n, s, lda, ldl, 0, dA, dL, nullptr, d_info, st};
  return run_graph(key, st, [&]() {
    const Sched S(n, s);
    if (dtype == SF_F64) return chol_run<double>(n, S, (const double*)dA, lda, (double*)dL, ldl, d_info, st);
    return chol_run_f32(n, S, (const float*)dA, lda, (float*)dL, ldl, d_info, st);
  });
}

int lu_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dLU, int64_t ldlu, int64_t* d_info,
              void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, s, dtype, dA, lda, dLU, ldlu);
  if (rc) return rc;
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const GraphKey key{1, dtype, n, s, lda, ldlu, 0, dA, dLU, nullptr, d_info, st};
  return run_graph(key, st, [&]() {
    const Sched S(n, s);
    if (dtype == SF_F32) return lu_run<float>(n, S, (const float*)dA, lda, (float*)dLU, ldlu, d_info, st);
    return lu_run<double>(n, S, (const double*)dA, lda, (double*)dLU, ldlu, d_info, st);
  });
}

int qr_factor(int64_t n, int64_t s, int dtype, const void* dA, int64_t lda, void* dQ, int64_t ldq, void* dR,
              int64_t ldr, int64_t* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, s, dtype, dA, lda, dQ, ldq);
  if (rc) return rc;
  rc = check_common(n, s, dtype, dA, lda, dR, ldr);
  if (rc) return rc;
  if (dA == dQ || dA == dR || dQ == dR) return fail_with(SF_EINVAL, "qr_factor outputs must not alias");
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const GraphKey key{2, dtype, n, s, lda, ldq, ldr, dA, dQ, dR, d_info, st};
  return run_graph(key, st, [&]() {
    const Sched S(n, s);
    if (dtype == SF_F32) return qr_run<float>(n, S, (const float*)dA, lda, (float*)dQ, ldq, (float*)dR, ldr, d_info, st);
    return qr_run<double>(n, S, (const double*)dA, lda, (double*)dQ, ldq, (double*)dR, ldr, d_info, st);
  });
}

// ------------------------------------------------------------------ variable step (R11)
static int check_steps(int64_t nsteps, const int64_t* steps) {
  if (nsteps < 1 || !steps) return fail_with(SF_EINVAL, "empty step sequence");
  for (int64_t i = 0; i < nsteps; ++i)
    if (steps[i] < 1) return fail_with(SF_EINVAL, "step %lld of the sequence is < 1", (long long)i);
  return SF_OK;
}

int chol_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dL,
                      int64_t ldl, int64_t* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, 1, dtype, dA, lda, dL, ldl);
  if (!rc) rc = check_steps(nsteps, steps);
  if (rc) return rc;
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const Sched S(n, steps, nsteps);
  if (dtype == SF_F64) return chol_run<double>(n, S, (const double*)dA, lda, (double*)dL, ldl, d_info, st);
  return chol_run_f32(n, S, (const float*)dA, lda, (float*)dL, ldl, d_info, st);
}

int lu_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dLU,
                    int64_t ldlu, int64_t* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, 1, dtype, dA, lda, dLU, ldlu);
  if (!rc) rc = check_steps(nsteps, steps);
  if (rc) return rc;
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const Sched S(n, steps, nsteps);
  if (dtype == SF_F32) return lu_run<float>(n, S, (const float*)dA, lda, (float*)dLU, ldlu, d_info, st);
  return lu_run<double>(n, S, (const double*)dA, lda, (double*)dLU, ldlu, d_info, st);
}

int qr_factor_steps(int64_t n, int64_t nsteps, const int64_t* steps, int dtype, const void* dA, int64_t lda, void* dQ,
                    int64_t ldq, void* dR, int64_t ldr, int64_t* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_common(n, 1, dtype, dA, lda, dQ, ldq);
  if (!rc) rc = check_common(n, 1, dtype, dA, lda, dR, ldr);
  if (!rc) rc = check_steps(nsteps, steps);
  if (rc) return rc;
  if (dA == dQ || dA == dR || dQ == dR) return fail_with(SF_EINVAL, "qr_factor outputs must not alias");
  if (!d_info) return fail_with(SF_EINVAL, "null d_info");
  cudaStream_t st = (cudaStream_t)stream;
  const Sched S(n, steps, nsteps);
  if (dtype == SF_F32) return qr_run<float>(n, S, (const float*)dA, lda, (float*)dQ, ldq, (float*)dR, ldr, d_info, st);
  return qr_run<double>(n, S, (const double*)dA, lda, (double*)dQ, ldq, (double*)dR, ldr, d_info, st);
}

// ------------------------------------------------------------------ solves with the factors (f4)
static int check_solve(int64_t n, int64_t nrhs, int dtype, const void* f, int64_t ldf, const void* b, int64_t ldb) {
  if (n < 1 || nrhs < 0) return fail_with(SF_EINVAL, "bad solve sizes");
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  if (!f || !b || ldf < n || ldb < n) return fail_with(SF_EINVAL, "bad solve pointers / leading dimensions");
  return SF_OK;
}

int chol_solve(int64_t n, int64_t nrhs, int dtype, const void* dL, int64_t ldl, void* dB, int64_t ldb, void* stream) {
  SF_API_LOCK;
  int rc = check_solve(n, nrhs, dtype, dL, ldl, dB, ldb);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SF_F32) return solve_run<float>(0, n, nrhs, (const float*)dL, ldl, nullptr, 0, (float*)dB, ldb, st);
  return solve_run<double>(0, n, nrhs, (const double*)dL, ldl, nullptr, 0, (double*)dB, ldb, st);
}

int lu_solve(int64_t n, int64_t nrhs, int dtype, const void* dLU, int64_t ldlu, void* dB, int64_t ldb, void* stream) {
  SF_API_LOCK;
  int rc = check_solve(n, nrhs, dtype, dLU, ldlu, dB, ldb);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SF_F32) return solve_run<float>(1, n, nrhs, (const float*)dLU, ldlu, nullptr, 0, (float*)dB, ldb, st);
  return solve_run<double>(1, n, nrhs, (const double*)dLU, ldlu, nullptr, 0, (double*)dB, ldb, st);
}

int qr_solve(int64_t n, int64_t nrhs, int dtype, const void* dQ, int64_t ldq, const void* dR, int64_t ldr, void* dB,
             int64_t ldb, void* stream) {
  SF_API_LOCK;
  int rc = check_solve(n, nrhs, dtype, dQ, ldq, dB, ldb);
  if (!rc) rc = check_solve(n, nrhs, dtype, dR, ldr, dB, ldb);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SF_F32)
    return solve_run<float>(2, n, nrhs, (const float*)dQ, ldq, (const float*)dR, ldr, (float*)dB, ldb, st);
  return solve_run<double>(2, n, nrhs, (const double*)dQ, ldq, (const double*)dR, ldr, (double*)dB, ldb, st);
}

// ------------------------------------------------------------------ host-buffer variants
// Host buffers the caller did not pin are registered (page-locked) for the duration of the
// call: the per-panel device->host copies must be asynchronous, or enqueueing would stall
// at every panel until that panel is factored and the lookahead overlap would be lost.
struct HostPin {
  void* ptr[3] = {nullptr, nullptr, nullptr};
  int n = 0;
  cudaError_t pin(const void* p, size_t bytes) {
    for (int i = 0; i < n; ++i)
      if (ptr[i] == p) return cudaSuccess;
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) cudaGetLastError();
    if (e == cudaSuccess && at.type != cudaMemoryTypeUnregistered) return cudaSuccess;   // pinned / managed already
    e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) { cudaGetLastError(); return cudaSuccess; }
    if (e != cudaSuccess) return e;
    ptr[n++] = const_cast<void*>(p);
    return cudaSuccess;
  }
  ~HostPin() {
    for (int i = 0; i < n; ++i) cudaHostUnregister(ptr[i]);
  }
};

static int host_body(int kind, int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hO1, int64_t ld1,
                     void* hO2, int64_t ld2, int64_t* info, char* d, int64_t* dinfo, cudaStream_t st,
                     cudaStream_t cs, cudaEvent_t ev) {
  const size_t elt = dtype == SF_F64 ? 8 : 4;
  const size_t bytes = elt * (size_t)n * (size_t)n;
  // the copy stream must not run ahead of the previous call
  SF_CUDA(cudaEventRecord(ev, st));
  SF_CUDA(cudaStreamWaitEvent(cs, ev, 0));
  const Sched S(n, s);
  int rc = SF_OK;
  if (kind == 0) {
    // Cholesky reads and writes only the lower triangle: copy it panel by panel (half the
    // bytes), and return each panel of L as soon as it is final, on the copy stream, while
    // the later flushes run (the device->host copy hides behind the factorization).
    for (int64_t z = 0; z < n; z += s) {
      const int64_t w = (s < n - z) ? s : n - z;
      SF_CUDA(cudaMemcpy2DAsync(d + elt * (z + z * n), n * elt, (const char*)hA + elt * (z + z * lda), lda * elt,
                                (n - z) * elt, w, cudaMemcpyHostToDevice, st));
    }
    struct D2H : PanelHook {
      int64_t n, ldh; size_t elt; const char* dev; char* host; cudaStream_t cs; cudaEvent_t ev;
      cudaError_t done(int64_t z, int64_t w, cudaStream_t pst) override {
        cudaError_t r = cudaEventRecord(ev, pst);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(cs, ev, 0);
        if (r == cudaSuccess)
          r = cudaMemcpy2DAsync(host + elt * (z + z * ldh), ldh * elt, dev + elt * (z + z * n), n * elt,
                                (n - z) * elt, w, cudaMemcpyDeviceToHost, cs);
        return r;
      }
    } hook;
    hook.n = n; hook.ldh = ld1; hook.elt = elt; hook.dev = d; hook.host = (char*)hO1; hook.cs = cs; hook.ev = ev;
    rc = dtype == SF_F64 ? chol_run<double>(n, S, (const double*)d, n, (double*)d, n, dinfo, st, &hook)
                         : chol_run_f32(n, S, (const float*)d, n, (float*)d, n, dinfo, st, &hook);
  } else if (kind == 1) {
    SF_CUDA(cudaMemcpy2DAsync(d, n * elt, hA, lda * elt, n * elt, n, cudaMemcpyHostToDevice, st));
    // LU: each panel's L columns [z, z+w) (rows >= z) and U rows [z, z+w) (columns >= z+w)
    // are final once the panel is factored; returned on the copy stream as for Cholesky.
    struct LuD2H : PanelHook {
      int64_t n, ldh; size_t elt; const char* dev; char* host; cudaStream_t cs; cudaEvent_t ev;
      cudaError_t done(int64_t z, int64_t w, cudaStream_t pst) override {
        cudaError_t r = cudaEventRecord(ev, pst);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(cs, ev, 0);
        if (r == cudaSuccess)   // L columns (incl. the diagonal block's U part)
          r = cudaMemcpy2DAsync(host + elt * (z + z * ldh), ldh * elt, dev + elt * (z + z * n), n * elt,
                                (n - z) * elt, w, cudaMemcpyDeviceToHost, cs);
        if (r == cudaSuccess && z + w < n)   // U rows right of the panel
          r = cudaMemcpy2DAsync(host + elt * (z + (z + w) * ldh), ldh * elt, dev + elt * (z + (z + w) * n), n * elt,
                                w * elt, n - z - w, cudaMemcpyDeviceToHost, cs);
        return r;
      }
    } hook;
    hook.n = n; hook.ldh = ld1; hook.elt = elt; hook.dev = d; hook.host = (char*)hO1; hook.cs = cs; hook.ev = ev;
    rc = dtype == SF_F64 ? lu_run<double>(n, S, (const double*)d, n, (double*)d, n, dinfo, st, &hook)
                         : lu_run<float>(n, S, (const float*)d, n, (float*)d, n, dinfo, st, &hook);
  } else {
    SF_CUDA(cudaMemcpy2DAsync(d, n * elt, hA, lda * elt, n * elt, n, cudaMemcpyHostToDevice, st));
    // QR: Q[:, z:z+w) is final once panel p's MGS is done (later flushes touch columns >= z+w
    // only): returned on the copy stream while the factorization continues; R (one product
    // at the end) follows.
    struct QD2H : PanelHook {
      int64_t n, ldh; size_t elt; const char* dev; char* host; cudaStream_t cs; cudaEvent_t ev;
      cudaError_t done(int64_t z, int64_t w, cudaStream_t pst) override {
        cudaError_t r = cudaEventRecord(ev, pst);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(cs, ev, 0);
        if (r == cudaSuccess)
          r = cudaMemcpy2DAsync(host + elt * (z * ldh), ldh * elt, dev + elt * (z * n), n * elt, n * elt, w,
                                cudaMemcpyDeviceToHost, cs);
        return r;
      }
    } hook;
    hook.n = n; hook.ldh = ld1; hook.elt = elt; hook.dev = d + bytes; hook.host = (char*)hO1; hook.cs = cs; hook.ev = ev;
    rc = dtype == SF_F64 ? qr_run<double>(n, S, (const double*)d, n, (double*)(d + bytes), n,
                                          (double*)(d + 2 * bytes), n, dinfo, st, &hook)
                         : qr_run<float>(n, S, (const float*)d, n, (float*)(d + bytes), n, (float*)(d + 2 * bytes), n,
                                         dinfo, st, &hook);
    if (!rc)
      SF_CUDA(cudaMemcpy2DAsync(hO2, ld2 * elt, d + 2 * bytes, n * elt, n * elt, n, cudaMemcpyDeviceToHost, st));
  }
  if (rc) return rc;
  SF_CUDA(cudaMemcpyAsync(info, dinfo, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  return SF_OK;
}

static int host_call(int kind, int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hO1, int64_t ld1,
                     void* hO2, int64_t ld2, int64_t* info) {
  SF_API_LOCK;
  if (n < 1 || !hA || !hO1 || !info || (kind == 2 && !hO2)) return fail_with(SF_EINVAL, "bad host arguments");
  if (lda < n || ld1 < n || (kind == 2 && ld2 < n)) return fail_with(SF_EINVAL, "leading dimension < n");
  if (s < 1 || s > n) return fail_with(SF_EINVAL, "step s=%lld outside [1, n=%lld]", (long long)s, (long long)n);
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  const size_t elt = dtype == SF_F64 ? 8 : 4;
  const size_t bytes = elt * (size_t)n * (size_t)n;
  int devh = 0;
  SF_CUDA(cudaGetDevice(&devh));
  // per-device internal compute stream + copy stream / event (created once)
  static cudaStream_t streams[16] = {}, cstreams[16] = {};
  static cudaEvent_t cevents[16] = {};
  if (!streams[devh & 15]) {
    SF_CUDA(cudaStreamCreateWithFlags(&streams[devh & 15], cudaStreamNonBlocking));
    SF_CUDA(cudaStreamCreateWithFlags(&cstreams[devh & 15], cudaStreamNonBlocking));
    SF_CUDA(cudaEventCreateWithFlags(&cevents[devh & 15], cudaEventDisableTiming));
  }
  cudaStream_t st = streams[devh & 15], cs = cstreams[devh & 15];
  cudaEvent_t ev = cevents[devh & 15];
  Workspace::keep_pool();   // repeated calls reuse the device block from the stream-ordered pool
  HostPin pins;
  SF_CUDA(pins.pin(hA, elt * ((size_t)lda * (n - 1) + n)));
  SF_CUDA(pins.pin(hO1, elt * ((size_t)ld1 * (n - 1) + n)));
  if (kind == 2) SF_CUDA(pins.pin(hO2, elt * ((size_t)ld2 * (n - 1) + n)));
  char* d = nullptr;
  const int nbuf = kind == 2 ? 3 : 1;
  if (cudaMallocAsync((void**)&d, nbuf * bytes + 256, st) != cudaSuccess) {
    cudaGetLastError();
    return fail_with(SF_ENOMEM, "device allocation of %zu bytes failed", nbuf * bytes + 256);
  }
  int64_t* dinfo = (int64_t*)(d + nbuf * bytes);
  const int rc = host_body(kind, n, s, dtype, hA, lda, hO1, ld1, hO2, ld2, info, d, dinfo, st, cs, ev);
  // on every path: join the copy stream (it reads d), free d, wait for the call's work
  cudaError_t ej = cudaEventRecord(ev, cs);
  if (ej == cudaSuccess) ej = cudaStreamWaitEvent(st, ev, 0);
  cudaFreeAsync(d, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  if (rc) return rc;
  if (ej != cudaSuccess) return fail_with(SF_ECUDA, "copy stream join: %s", cudaGetErrorString(ej));
  if (es != cudaSuccess) return fail_with(SF_ECUDA, "stream sync: %s", cudaGetErrorString(es));
  return SF_OK;
}

int chol_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hL, int64_t ldl,
                     int64_t* info) {
  return host_call(0, n, s, dtype, hA, lda, hL, ldl, nullptr, 0, info);
}
int lu_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hLU, int64_t ldlu,
                   int64_t* info) {
  return host_call(1, n, s, dtype, hA, lda, hLU, ldlu, nullptr, 0, info);
}
int qr_factor_host(int64_t n, int64_t s, int dtype, const void* hA, int64_t lda, void* hQ, int64_t ldq, void* hR,
                   int64_t ldr, int64_t* info) {
  return host_call(2, n, s, dtype, hA, lda, hQ, ldq, hR, ldr, info);
}

// ------------------------------------------------------------------ building blocks
int sf_chol_panel(int64_t m, int64_t w, int dtype, void* dP, int64_t ld, int64_t col0, int64_t* d_info, void* stream) {
  SF_API_LOCK;
  if (m < 1 || w < 1 || w > m || ld < m || !dP || !d_info) return fail_with(SF_EINVAL, "bad panel arguments");
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ldk = (w + 3) / 4 * 4;
  Workspace ws;
  SF_CUDA(ws.init(256 + (dtype == SF_F32 ? 2 * sizeof(float) * (size_t)m * ldk + 512 : 0), st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  SF_CUDA(init_fail(fail, st));
  if (dtype == SF_F64) {
    SF_CUDA(chol_panel_rec<double>(m, w, (double*)dP, ld, (double*)dP, ld, col0, fail, st));
  } else {
    SplitBuf sb{ws.take<float>((size_t)m * ldk), nullptr, ldk};
    sb.l = ws.take<float>((size_t)m * ldk);
    SF_CUDA(chol_panel_rec_f32(m, w, (float*)dP, ld, (float*)dP, ld, col0, sb, fail, st));
  }
  SF_CUDA(finish_info(fail, d_info, st));
  return SF_OK;
}

int sf_syrk_sub(int64_t m, int64_t k, int dtype, const void* dR, int64_t ldr, void* dC, int64_t ldc, void* stream) {
  SF_API_LOCK;
  if (m < 0 || k < 0 || !dR || !dC || ldr < m || ldc < m) return fail_with(SF_EINVAL, "bad syrk arguments");
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SF_F64) {
    const double* R = (const double*)dR;
    SF_CUDA(gemm_sub<double>(m, m, k, R, ldr, 0, R, ldr, 0, (double*)dC, ldc, (double*)dC, ldc, kMaskLower, nullptr, st));
    return SF_OK;
  }
  if (m == 0 || k == 0) return SF_OK;
  // fp32: split R once (3xTF32, K-major), then the tcgen05 update
  const int64_t ldk = (k + 3) / 4 * 4;
  Workspace ws;
  SF_CUDA(ws.init(2 * sizeof(float) * (size_t)m * ldk + 1024, st));
  SplitBuf sb{ws.take<float>((size_t)m * ldk), nullptr, ldk};
  sb.l = ws.take<float>((size_t)m * ldk);
  SF_CUDA(split_tf32(m, k, (const float*)dR, ldr, sb.h, sb.l, ldk, st));
  SF_CUDA(syrk_tf32(m, m, k, sb, sb, (float*)dC, ldc, (float*)dC, ldc, nullptr, st));
  return SF_OK;
}

int sf_gemm_sub(int64_t m, int64_t n, int64_t k, int dtype, const void* dA, int64_t lda, int ta, const void* dB,
                int64_t ldb, int tb, void* dC, int64_t ldc, void* stream) {
  SF_API_LOCK;
  if (m < 0 || n < 0 || k < 0 || !dA || !dB || !dC || ldc < m) return fail_with(SF_EINVAL, "bad gemm arguments");
  if (dtype != SF_F64) return fail_with(SF_ENOTSUP, "fp64 only");
  SF_CUDA(gemm_sub<double>(m, n, k, (const double*)dA, lda, ta ? 1 : 0, (const double*)dB, ldb, tb ? 0 : 1,
                           (double*)dC, ldc, (double*)dC, ldc, kMaskNone, nullptr, (cudaStream_t)stream));
  return SF_OK;
}

int sf_lu_panel(int64_t m, int64_t w, int64_t ncr, int dtype, void* dP, int64_t ld, int64_t col0, double tol,
                int64_t* d_info, void* stream) {
  SF_API_LOCK;
  if (m < 1 || w < 1 || w > m || ncr < 0 || ld < m || !dP || !d_info) return fail_with(SF_EINVAL, "bad panel arguments");
  if (dtype != SF_F64) return fail_with(SF_ENOTSUP, "fp64 only");
  cudaStream_t st = (cudaStream_t)stream;
  Workspace ws;
  SF_CUDA(ws.init(512, st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  double* dtol = ws.take<double>(1);
  SF_CUDA(init_fail(fail, st));
  SF_CUDA(cudaMemcpyAsync(dtol, &tol, sizeof(double), cudaMemcpyHostToDevice, st));
  SF_CUDA(lu_panel_rec<double>(m, w, ncr, (double*)dP, ld, (double*)dP, ld, col0, dtol, fail, st));
  SF_CUDA(finish_info(fail, d_info, st));
  SF_CUDA(cudaStreamSynchronize(st));  // tol lives in pageable host memory
  return SF_OK;
}

int sf_qr_panel(int64_t n, int64_t w, int dtype, void* dV, int64_t ld, int64_t col0, double tol, int64_t* d_info,
                void* stream) {
  SF_API_LOCK;
  if (n < 1 || w < 1 || w > n || ld < n || !dV || !d_info) return fail_with(SF_EINVAL, "bad panel arguments");
  if (dtype != SF_F64) return fail_with(SF_ENOTSUP, "fp64 only");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t wmax = qr_mgs_max_width(n, 8);
  const int64_t wcap = w < wmax ? w : wmax;
  const int sp = splitk_for(w, wcap, n);
  const int64_t split_elems = (int64_t)sp * w * wcap;
  const size_t mgs = qr_mgs_work_elems(n, (int)wcap, 8) + 64;
  Workspace ws;
  SF_CUDA(ws.init(8 * (mgs + w * wcap + split_elems) + 4096, st));
  long long* fail = ws.take<long long>(2);   // [0] first failed column, [1] leaf counter
  double* dtol = ws.take<double>(1);
  double* mgsw = ws.take<double>(mgs);
  double* Cw = ws.take<double>(w * wcap);
  double* split = ws.take<double>(split_elems);
  SF_CUDA(init_fail(fail, st));
  SF_CUDA(cudaMemsetAsync(mgsw, 0, sizeof(double) * mgs, st));
  SF_CUDA(cudaMemcpyAsync(dtol, &tol, sizeof(double), cudaMemcpyHostToDevice, st));
  SF_CUDA(qr_panel<double>(n, w, (double*)dV, ld, (double*)dV, ld, col0, dtol, mgsw, Cw, split, split_elems, fail, st));
  SF_CUDA(finish_info(fail, d_info, st));
  SF_CUDA(cudaStreamSynchronize(st));
  return SF_OK;
}

int64_t sf_flush_count(int64_t n, int64_t s) {
  if (n < 1 || s < 1) return 0;
  int64_t f = 0;
  for (int64_t z = 0; z < n; z += s)
    if (z + s < n) ++f;
  return f;
}

int64_t sf_schedule(int64_t n, int64_t nsteps, const int64_t* steps, int64_t* flush_cols, int64_t cap) {
  if (n < 1 || nsteps < 1 || !steps) return -1;
  for (int64_t i = 0; i < nsteps; ++i)
    if (steps[i] < 1) return -1;
  const Sched S = nsteps == 1 ? Sched(n, steps[0]) : Sched(n, steps, nsteps);
  const int64_t count = S.P() - 1;   // a flush follows every panel but the last
  for (int64_t p = 0; p < count && p < cap; ++p) flush_cols[p] = S.z(p + 1);
  return count;
}

int64_t sf_launch_counter(void) { return g_launches.load(); }

int sf_set_strassen(int levels, int64_t min_dim) {
  SF_API_LOCK;
  if (levels < 0 || levels > 3 || min_dim < 64) return fail_with(SF_EINVAL, "strassen: levels must be 0..3, min_dim >= 64");
  strassen_cfg().levels = levels;
  strassen_cfg().min_dim = min_dim;
  for (auto& g : g_graphs)   // captured factorizations embed the old choice
    if (g.exec) cudaGraphExecDestroy(g.exec);
  g_graphs.clear();
  return SF_OK;
}

void sf_profile_enable(int on) {
  SF_API_LOCK;
  g_prof = on != 0;
}

static double g_prof_union[4] = {0.0, 0.0, 0.0, 0.0};

int sf_profile_collect(double* ms, int64_t* count, double* flops) {
  SF_API_LOCK;
  for (int k = 0; k < 4; ++k) { ms[k] = 0.0; count[k] = 0; flops[k] = 0.0; g_prof_union[k] = 0.0; }
  int rc = SF_OK;
  // per kind: the intervals on a common time axis (relative to the first recorded event), so
  // that regions running concurrently on two streams (LU's two-deep lookahead: F1 on the
  // panel stream beside F2/F3) are also reported as their wall-clock union
  std::vector<std::pair<double, double>> iv[4];
  const cudaEvent_t ref = g_prof_recs.empty() ? nullptr : g_prof_recs.front().a;
  for (auto& r : g_prof_recs) {
    if (r.kind < 0 || r.kind > 3) continue;
    float t = 0.f, t0 = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t0, ref, r.a);
    if (e != cudaSuccess) rc = fail_with(SF_ECUDA, "profile events: %s", cudaGetErrorString(e));
    ms[r.kind] += t; count[r.kind] += 1; flops[r.kind] += r.flops;
    iv[r.kind].push_back({(double)t0, (double)t0 + t});
  }
  for (int k = 0; k < 4; ++k) {
    std::sort(iv[k].begin(), iv[k].end());
    double cur_a = 0.0, cur_b = -1.0;
    for (auto& x : iv[k]) {
      if (x.first > cur_b) { if (cur_b > cur_a) g_prof_union[k] += cur_b - cur_a; cur_a = x.first; cur_b = x.second; }
      else if (x.second > cur_b) cur_b = x.second;
    }
    if (cur_b > cur_a) g_prof_union[k] += cur_b - cur_a;
  }
  for (auto& r : g_prof_recs) { g_event_pool.push_back(r.a); g_event_pool.push_back(r.b); }
  g_prof_recs.clear();
  return rc;
}

int sf_profile_union(double* ms_union) {
  SF_API_LOCK;
  if (!ms_union) return fail_with(SF_EINVAL, "sf_profile_union: null output");
  for (int k = 0; k < 4; ++k) ms_union[k] = g_prof_union[k];
  return SF_OK;
}

const char* sf_strerror(int status) {
  switch (status) {
    case SF_OK: return "success";
    case SF_EINVAL: return "invalid argument";
    case SF_ENOTSUP: return "not supported";
    case SF_ENOMEM: return "out of device memory";
    case SF_ECUDA: return "CUDA error";
    case SF_ENCCL: return "NCCL error";
    default: return "unknown status";
  }
}
const char* sf_last_error(void) { return g_last_error; }
int sf_version(void) { return 1; }

}  // extern "C"
