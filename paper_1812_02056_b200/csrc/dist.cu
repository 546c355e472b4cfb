// dist.cu — block-cyclic multi-GPU drivers (BASELINE.json north_star (3)).
//
// One process per GPU.  The n x n matrix is split into panels of s columns (the paper's
// step); panel p = columns [p*s, min((p+1)s, n)) lives on rank
// p % G at local slot p / G, stored full height (local column-major storage, ld >= n).  The
// schedule is the paper's (flush when c = z + s) with ONE exchange per
// panel: the owner factors the panel (the s-column recurrences) and broadcasts it; every
// rank then applies the flush to the columns it owns.  Per rank and panel p:
//
//   Cholesky  Lp = L[ps:n, panel p] broadcast (in place from the owner);
//                              each local panel q > p:  A[qs:n, q] -= Lp[qs:n] Lp[q]^T
//                              (lower part; one grouped launch over all local panels)
//   LU       Lp = L[ps:n, panel p] (U11 in its strict upper block);
//                              local columns right of p: U rows [ps, ps+w) = L11^-1 A
//                              (Crout U rows, / L_cc), then A[ps+w:n, cols] -= L21 U12
//   QR      Q panel broadcast into a full n x n copy of Q on every
//                              rank; local columns right of p: C = B_Q^T M, M -= B_Q C;
//                              finally R[:, local] = Q^T A[:, local] (upper part).
//
// Lookahead: the owner of panel p+1 first applies panel p to panel p+1 only, factors p+1
// on a high-priority stream and broadcasts it on a third stream while the rest of the
// flush p runs — the broadcast and the next panel overlap the update, tile for tile the
// same arithmetic as the single-GPU driver (driver.cu), so for Cholesky the distributed
// result is bitwise equal to the single-GPU one.
//
// Transport: NCCL (ncclBroadcast over NVLink / NVSwitch) for a real communicator; a
// LOOPBACK communicator runs all G ranks of the schedule in this process on one GPU (each
// rank with its own buffers and streams, the broadcast a device copy), which is how the
// multi-rank path is parity-tested on a single B200.
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>
#include <map>
#include <type_traits>

#include "common.cuh"
#include "drv.cuh"

struct sf_comm_ {
  int nranks = 1;
  int rank = 0;        // ignored for loopback
  int device = 0;
  ncclComm_t nccl = nullptr;
  int64_t bcast_bytes = 0;   // payload of every panel message sent so far (sf_comm_bcast_bytes)
  // f3 (sf_comm_set_push): device-initiated panel push instead of ncclBroadcast.  NCCL: the
  // receive buffers and flags live in a symmetric window (ncclMemAlloc +
  // ncclCommWindowRegister), peers addressed by their load/store (LSA) pointers.
  int push = 0;
  uint64_t calls = 0;        // dist calls so far: the high half of the push flag tags
  void* win_base = nullptr;
  size_t win_bytes = 0;
  ncclWindow_t win = nullptr;
  std::vector<char*> peer_base;   // every rank's window base, as addressable from this GPU
  bool loopback() const { return nccl == nullptr; }
  int nlocal() const { return loopback() ? nranks : 1; }
  int local_rank(int i) const { return loopback() ? i : rank; }
};

namespace sf {

// ------------------------------------------------------------------ block-cyclic layout
struct Cyclic {
  int64_t n, s, P;
  int G;
  Cyclic(int64_t n_, int64_t s_, int G_) : n(n_), s(s_), P((n_ + s_ - 1) / s_), G(G_) {}
  int64_t width(int64_t p) const { return (s < n - p * s) ? s : n - p * s; }
  int owner(int64_t p) const { return (int)(p % G); }
  int64_t slot(int64_t p) const { return p / G; }
  int64_t local_cols(int r) const {
    int64_t c = 0;
    for (int64_t p = r; p < P; p += G) c += width(p);
    return c;
  }
  // first local slot of rank r whose global panel is > p
  int64_t first_slot_after(int64_t p, int r) const { return p < r ? 0 : (p - r) / G + 1; }
  int64_t panel_of(int64_t slot_, int r) const { return slot_ * G + r; }
};

// ------------------------------------------------------------------ per-rank state
struct RankStreams { cudaStream_t mn = nullptr, pan = nullptr, com = nullptr; };
static cudaError_t rank_streams(int dev, int idx, RankStreams& out) {
  static std::map<std::pair<int, int>, RankStreams> cache;
  auto key = std::make_pair(dev, idx);
  auto it = cache.find(key);
  if (it != cache.end()) { out = it->second; return cudaSuccess; }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  RankStreams rs;
  cudaError_t e = cudaStreamCreateWithPriority(&rs.mn, cudaStreamNonBlocking, lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&rs.pan, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&rs.com, cudaStreamNonBlocking, hi);
  if (e != cudaSuccess) return e;
  cache[key] = rs;
  out = rs;
  return cudaSuccess;
}

struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() { for (auto e : ev) cudaEventDestroy(e); }
  cudaError_t make(size_t n) {
    ev.resize(n, nullptr);
    for (auto& e : ev) {
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  }
  cudaEvent_t operator[](size_t i) const { return ev[i]; }
};

template <typename T>
struct Rank {
  int r = 0;
  const T* A = nullptr;   // local input
  T* X = nullptr;         // local output: L (Cholesky), LU, Q = working M (QR)
  T* R = nullptr;         // QR: local R
  int64_t* d_info = nullptr;
  RankStreams st;
  Workspace ws;
  long long* fail = nullptr;
  T* tol = nullptr;
  double* part = nullptr;
  double* sumsq = nullptr;
  T* buf[2] = {nullptr, nullptr};   // Cholesky / LU: panel receive buffers (Span layout)
  T* qfull = nullptr;               // QR: every panel of Q, n x n, ld n
  T* mgsw = nullptr; T* cw = nullptr; T* split = nullptr; T* cw2 = nullptr; T* split2 = nullptr;
  int64_t split_elems = 0;
  SplitBuf sb_upd{}, sb_pan{};      // fp32 Cholesky: 3xTF32 split of the received / own panel
  Events recv, ready, done, la;
};

template <typename T> inline ncclDataType_t nccl_type();
template <> inline ncclDataType_t nccl_type<double>() { return ncclFloat64; }
template <> inline ncclDataType_t nccl_type<float>() { return ncclFloat32; }

#define SF_NCCL(expr)                                                                              \
  do {                                                                                             \
    ncclResult_t _r = (expr);                                                                      \
    if (_r != ncclSuccess) return fail_with(SF_ENCCL, "%s: %s", #expr, ncclGetErrorString(_r));   \
  } while (0)

__global__ void min_into_kernel(long long* dst, const long long* src) {
  if (*src < *dst) *dst = *src;
}
__global__ void add_into_kernel(double* dst, const double* src) { *dst += *src; }

template <typename T>
__global__ void sumsq_cols_kernel(int64_t m, int64_t ncols, const T* A, int64_t lda, double* part) {
  double acc = 0.0;
  const int64_t total = m * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)A[(t % m) + (t / m) * lda];
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
__global__ void sum_parts_kernel(const double* part, int np, double* out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += part[i];
    *out = s;
  }
}
// tol = 1e-12 * ||A||_F / n  (R3), from the global sum of squares
template <typename T>
__global__ void tol_from_sumsq_kernel(int64_t n, const double* sumsq, T* tol) {
  if (threadIdx.x == 0) *tol = (T)(1e-12 * sqrt(*sumsq) / (double)n);
}

// R's strict lower part (rows > global column) of the local columns := 0
template <typename T>
__global__ void zero_lower_cyclic_kernel(int64_t n, int64_t s, int G, int r, int64_t nloc, T* R, int64_t ld) {
  for (int64_t jl = blockIdx.y; jl < nloc; jl += gridDim.y) {
    const int64_t g = (jl / s) * G * s + (int64_t)r * s + jl % s;
    for (int64_t i = g + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      R[i + jl * ld] = T(0);
  }
}

template <typename T>
static cudaError_t sumsq_local(int64_t n, int64_t nloc, const T* A, int64_t ld, double* part, double* out,
                               cudaStream_t st) {
  const int np = 512;
  if (nloc > 0) {
    sumsq_cols_kernel<T><<<np, 256, 0, st>>>(n, nloc, A, ld, part);
    count_launch();
    sum_parts_kernel<<<1, 32, 0, st>>>(part, np, out);
  } else {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    sum_parts_kernel<<<1, 32, 0, st>>>(part, 0, out);
  }
  count_launch();
  return cudaGetLastError();
}

static cudaError_t wait_on(cudaStream_t waiter, cudaEvent_t ev) { return cudaStreamWaitEvent(waiter, ev, 0); }

// The exchange of panel p: after it, on rank r's comm stream (event recv[p]), the panel
// is at `dst(r)` (the owner's own storage on the owner); `count` elements.  Non-owners first wait for
// `free_ev(r)` (the buffer's previous contents are no longer read), the owner for ready[p].
template <typename T, typename DstF, typename FreeF>
static int exchange(sf_comm_t comm, std::vector<Rank<T>>& rk, int64_t p, int owner, size_t count, DstF dst,
                    FreeF free_ev) {
  comm->bcast_bytes += (int64_t)(count * sizeof(T));
  if (!comm->loopback()) {
    Rank<T>& me = rk[0];
    if (me.r == owner) SF_CUDA(wait_on(me.st.com, me.ready[p]));
    else if (cudaEvent_t fe = free_ev(me)) SF_CUDA(wait_on(me.st.com, fe));
    static const bool skip1 = getenv("SF_DIST_SKIP1") && atoi(getenv("SF_DIST_SKIP1"));
    if (!(skip1 && comm->nranks == 1)) {
      T* b = dst(me);
      ProfScope pb(3, (double)(count * sizeof(T)), me.st.com);
      SF_NCCL(ncclBroadcast(b, b, count, nccl_type<T>(), owner, comm->nccl, me.st.com));
      count_launch();
    }
    SF_CUDA(cudaEventRecord(me.recv[p], me.st.com));
    return SF_OK;
  }
  Rank<T>& o = rk[owner];
  for (auto& x : rk) {
    SF_CUDA(wait_on(x.st.com, o.ready[p]));
    if (x.r != owner) {
      if (cudaEvent_t fe = free_ev(x)) SF_CUDA(wait_on(x.st.com, fe));
      SF_CUDA(cudaMemcpyAsync(dst(x), dst(o), count * sizeof(T), cudaMemcpyDeviceToDevice, x.st.com));
    }
    SF_CUDA(cudaEventRecord(x.recv[p], x.st.com));
  }
  return SF_OK;
}

// ------------------------------------------------------------------ f3: device-initiated push
// SURVEY.md §8 f3.  Instead of pack (device copy) + ncclBroadcast on a third stream, the
// owner of panel q runs ONE kernel right after the panel's last kernel on its panel stream:
// it reads the factored panel (rows [qs, n) of its w columns, strided, from its own storage)
// and stores it packed into EVERY rank's receive buffer for slot q & 1 — through the peers'
// load/store-accessible window pointers (NVLink / NVSwitch) for an NCCL communicator, plain
// device pointers for loopback — then the last CTA, after a system-scope fence, raises each
// rank's `ready[slot]` flag (release) to the panel's tag.  A receiver's main stream runs a
// one-thread wait (acquire) before its flush of panel p, and after that flush writes its
// `consumed` tag into every rank's flags; the owner of panel q waits until all ranks consumed
// panel q-2 (same slot) before pushing.  No host, NCCL call or stream event on the data path;
// same bytes as the packed broadcast, same operands for the flush (results bitwise equal).
constexpr int kMaxPushRanks = 16;
struct PushFlags {
  unsigned long long ready[2];                 // tag of the panel in slot 0 / 1
  unsigned long long consumed[kMaxPushRanks];  // tag of the last panel rank r finished flushing
  unsigned long long counter;                  // CTA arrivals of the running push kernel
  unsigned long long pad[13];
};
struct PushTargets {
  void* dst[kMaxPushRanks];
  unsigned long long* flag[kMaxPushRanks];
  int G;
};
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// packed element (i, k) of the panel (i < m rows from its first row, k < w) -> dst[i + k*m]
template <typename T>
__global__ void __launch_bounds__(256) push_panel_kernel(const T* __restrict__ src, int64_t ld, int64_t m, int w,
                                                         PushTargets tg, unsigned long long tag,
                                                         unsigned long long* counter) {
  const int64_t total = m * (int64_t)w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % m, k = t / m;
    const T v = __ldcg(src + i + k * ld);
    for (int r = 0; r < tg.G; ++r) __stcg(static_cast<T*>(tg.dst[r]) + t, v);
  }
  __threadfence_system();   // this CTA's stores are performed for every observer
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long old = atomicAdd(counter, 1ull);
    if (old == gridDim.x - 1) {   // the last CTA: all CTAs' stores are fenced
      *counter = 0;
      __threadfence_system();
      for (int r = 0; r < tg.G; ++r) st_release_sys(tg.flag[r], tag);
    }
  }
}
// one thread per flag: spin (acquire) until every flag reaches the tag
__global__ void wait_flags_kernel(PushTargets tg, unsigned long long tag) {
  if ((int)threadIdx.x < tg.G)
    while (ld_acquire_sys(tg.flag[threadIdx.x]) < tag) __nanosleep(100);
}
__global__ void signal_flags_kernel(PushTargets tg, unsigned long long tag) {
  if ((int)threadIdx.x < tg.G) st_release_sys(tg.flag[threadIdx.x], tag);
}
__global__ void lsa_pointers_kernel(ncclWindow_t w, int G, char** out) {
  if ((int)threadIdx.x < G) out[threadIdx.x] = (char*)ncclGetPeerPointer(w, 0, (int)threadIdx.x);
}

// The symmetric window of an NCCL communicator, per rank: [PushFlags (4 KB) | slot 0 | slot 1]
// — the flags at a fixed offset, so their tags carry over between calls of any size.
// Collective (every rank calls the dist entry point with the same sizes).
constexpr size_t kFlagBytes = 4096;
static_assert(sizeof(PushFlags) <= kFlagBytes, "flag block");
static int ensure_window(sf_comm_t comm, size_t buf_bytes) {
  const size_t need = kFlagBytes + 2 * buf_bytes;
  if (comm->win && comm->win_bytes >= need) return SF_OK;
  if (comm->win) {
    SF_CUDA(cudaDeviceSynchronize());
    SF_NCCL(ncclCommWindowDeregister(comm->nccl, comm->win));
    SF_NCCL(ncclMemFree(comm->win_base));
    comm->win = nullptr; comm->win_base = nullptr; comm->win_bytes = 0;
  }
  const size_t bytes = (need + (size_t(1) << 21) - 1) & ~((size_t(1) << 21) - 1);
  SF_NCCL(ncclMemAlloc(&comm->win_base, bytes));
  SF_CUDA(cudaMemset(comm->win_base, 0, bytes));
  SF_NCCL(ncclCommWindowRegister(comm->nccl, comm->win_base, bytes, &comm->win, NCCL_WIN_COLL_SYMMETRIC));
  comm->win_bytes = bytes;
  char** d = nullptr;
  SF_CUDA(cudaMalloc(&d, sizeof(char*) * comm->nranks));
  lsa_pointers_kernel<<<1, 32>>>(comm->win, comm->nranks, d);
  comm->peer_base.assign(comm->nranks, nullptr);
  cudaError_t e = cudaMemcpy(comm->peer_base.data(), d, sizeof(char*) * comm->nranks, cudaMemcpyDeviceToHost);
  cudaFree(d);
  SF_CUDA(e);
  return SF_OK;
}

// info: all-reduce(min) of the first failed column over ranks, then per-rank d_info
template <typename T>
static int finish_dist(sf_comm_t comm, std::vector<Rank<T>>& rk, cudaStream_t caller) {
  if (!comm->loopback()) {
    Rank<T>& me = rk[0];
    SF_NCCL(ncclAllReduce(me.fail, me.fail, 1, ncclInt64, ncclMin, comm->nccl, me.st.mn));
    count_launch();
    SF_CUDA(finish_info(me.fail, me.d_info, me.st.mn));
    cudaEvent_t e = pool_event();
    SF_CUDA(cudaEventRecord(e, me.st.mn));
    SF_CUDA(wait_on(caller, e));
    return SF_OK;
  }
  for (auto& x : rk) {
    cudaEvent_t e = pool_event();
    SF_CUDA(cudaEventRecord(e, x.st.mn));
    SF_CUDA(wait_on(caller, e));
  }
  for (size_t i = 1; i < rk.size(); ++i) { min_into_kernel<<<1, 1, 0, caller>>>(rk[0].fail, rk[i].fail); count_launch(); }
  for (size_t i = 1; i < rk.size(); ++i)
    SF_CUDA(cudaMemcpyAsync(rk[i].fail, rk[0].fail, sizeof(long long), cudaMemcpyDeviceToDevice, caller));
  for (auto& x : rk) SF_CUDA(finish_info(x.fail, x.d_info, caller));
  return SF_OK;
}

// global tolerance for LU / QR: sum of squares of every rank's local columns of A
template <typename T>
static int dist_tol(sf_comm_t comm, std::vector<Rank<T>>& rk, const Cyclic& cy, int64_t ld, cudaStream_t caller) {
  for (auto& x : rk) SF_CUDA(sumsq_local<T>(cy.n, cy.local_cols(x.r), x.A, ld, x.part, x.sumsq, caller));
  if (!comm->loopback()) {
    SF_NCCL(ncclAllReduce(rk[0].sumsq, rk[0].sumsq, 1, ncclFloat64, ncclSum, comm->nccl, caller));
    count_launch();
  } else {
    for (size_t i = 1; i < rk.size(); ++i) { add_into_kernel<<<1, 1, 0, caller>>>(rk[0].sumsq, rk[i].sumsq); count_launch(); }
    for (size_t i = 1; i < rk.size(); ++i)
      SF_CUDA(cudaMemcpyAsync(rk[i].sumsq, rk[0].sumsq, sizeof(double), cudaMemcpyDeviceToDevice, caller));
  }
  for (auto& x : rk) { tol_from_sumsq_kernel<T><<<1, 32, 0, caller>>>(cy.n, x.sumsq, x.tol); count_launch(); }
  return SF_OK;
}

template <typename T>
static int setup_ranks(sf_comm_t comm, std::vector<Rank<T>>& rk, const Cyclic& cy, void* const* dA, void* const* dX,
                       void* const* dR, int64_t* const* d_info, size_t buf_elems, size_t qfull_elems,
                       size_t extra_elems, cudaStream_t caller) {
  const int nl = comm->nlocal();
  rk.resize(nl);
  cudaEvent_t fork = pool_event();
  SF_CUDA(cudaEventRecord(fork, caller));
  for (int i = 0; i < nl; ++i) {
    Rank<T>& x = rk[i];
    x.r = comm->local_rank(i);
    x.A = (const T*)dA[i];
    x.X = (T*)dX[i];
    x.R = dR ? (T*)dR[i] : nullptr;
    x.d_info = d_info[i];
    SF_CUDA(rank_streams(comm->device, i, x.st));
    SF_CUDA(x.ws.init(sizeof(T) * (2 * buf_elems + qfull_elems + extra_elems) + 64 * 1024, caller));
    x.ws.join(x.st.mn); x.ws.join(x.st.pan); x.ws.join(x.st.com);
    x.fail = x.ws.template take<long long>(2);
    x.tol = x.ws.template take<T>(1);
    x.sumsq = x.ws.template take<double>(1);
    x.part = x.ws.template take<double>(512);
    if (buf_elems) { x.buf[0] = x.ws.template take<T>(buf_elems); x.buf[1] = x.ws.template take<T>(buf_elems); }
    if (qfull_elems) x.qfull = x.ws.template take<T>(qfull_elems);
    SF_CUDA(init_fail(x.fail, caller));
    SF_CUDA(x.recv.make(cy.P)); SF_CUDA(x.ready.make(cy.P)); SF_CUDA(x.done.make(cy.P)); SF_CUDA(x.la.make(cy.P));
    SF_CUDA(wait_on(x.st.mn, fork)); SF_CUDA(wait_on(x.st.pan, fork)); SF_CUDA(wait_on(x.st.com, fork));
  }
  return SF_OK;
}

// join a rank's panel and comm streams into its main stream
template <typename T>
static int join_rank(Rank<T>& x) {
  cudaEvent_t a = pool_event(), b = pool_event();
  SF_CUDA(cudaEventRecord(a, x.st.pan)); SF_CUDA(cudaEventRecord(b, x.st.com));
  SF_CUDA(wait_on(x.st.mn, a)); SF_CUDA(wait_on(x.st.mn, b));
  return SF_OK;
}

// ------------------------------------------------------------------ Cholesky
// Flush of panel p into rank x's local panels in slots [j_begin, j_end): for each, rows
// [qs, n) of its columns -= Lp[qs-ps : n-ps] Lp[qs-ps : qs-ps+wq]^T, lower part;
// one grouped launch.  Adds the algorithmic flops to *flops.
static cudaError_t chol_update_slots(const Cyclic& cy, Rank<double>& x, int64_t p, int64_t j_begin, int64_t j_end,
                                     const double* Lp, int64_t ldp, int64_t ld, double* flops, cudaStream_t st) {
  std::vector<GemmGroup> gs;
  const int64_t ps = p * cy.s, wp = cy.width(p);
  const double* src = (p == 0) ? x.A : x.X;   // out of place: the first flush reads A
  for (int64_t j = j_begin; j < j_end; ++j) {
    const int64_t q = cy.panel_of(j, x.r), qs = q * cy.s, wq = cy.width(q);
    GemmGroup g{};
    g.M = cy.n - qs; g.N = wq; g.off = 0;
    g.A = (const double*)(Lp + (qs - ps)); g.B = g.A;
    g.Cin = (const double*)(src + qs + j * cy.s * ld); g.C = (double*)(x.X + qs + j * cy.s * ld);
    gs.push_back(g);
    *flops += 2.0 * wp * ((double)wq * (double)g.M - 0.5 * (double)wq * (double)(wq - 1));
  }
  if (gs.empty()) return cudaSuccess;
  GemmF64 p64{0, 0, wp, nullptr, ldp, nullptr, ldp, nullptr, ld, nullptr, ld, -1.0, 1, 1, nullptr, x.fail};
  return gemm_f64_grouped(p64, gs.data(), (int)gs.size(), 0, 0, kMaskLower, st);
}

// fp32: the received panel's rows [c, n) were split once into x.sb_upd (chol_split_panel);
// one 3xTF32 tcgen05 launch per local panel.
static cudaError_t chol_update_slots(const Cyclic& cy, Rank<float>& x, int64_t p, int64_t j_begin, int64_t j_end,
                                     const float*, int64_t, int64_t ld, double* flops, cudaStream_t st) {
  const int64_t c = p * cy.s + cy.width(p), wp = cy.width(p);
  const float* src = (p == 0) ? x.A : x.X;
  for (int64_t j = j_begin; j < j_end; ++j) {
    const int64_t q = cy.panel_of(j, x.r), qs = q * cy.s, wq = cy.width(q), M = cy.n - qs;
    const SplitBuf R = x.sb_upd.at(qs - c, 0);
    cudaError_t e = syrk_tf32(M, wq, wp, R, R, src + qs + j * cy.s * ld, ld, x.X + qs + j * cy.s * ld, ld, x.fail, st);
    if (e != cudaSuccess) return e;
    *flops += 3.0 * 2.0 * wp * ((double)wq * (double)M - 0.5 * (double)wq * (double)(wq - 1));
  }
  return cudaSuccess;
}
static cudaError_t chol_split_panel(const Cyclic&, Rank<double>&, int64_t, const double*, int64_t, cudaStream_t) {
  return cudaSuccess;
}
static cudaError_t chol_split_panel(const Cyclic& cy, Rank<float>& x, int64_t p, const float* Lp, int64_t ld,
                                    cudaStream_t st) {
  const int64_t wp = cy.width(p), c = p * cy.s + wp;
  if (c >= cy.n) return cudaSuccess;
  return split_tf32(cy.n - c, wp, Lp + wp, ld, x.sb_upd.h, x.sb_upd.l, x.sb_upd.ldk, st);
}
static cudaError_t chol_panel_any(Rank<double>& x, int64_t m, int64_t w, const double* src, int64_t lds, double* dst,
                                  int64_t ldd, int64_t col0, cudaStream_t st) {
  return chol_panel_rec<double>(m, w, src, lds, dst, ldd, col0, x.fail, st);
}
static cudaError_t chol_panel_any(Rank<float>& x, int64_t m, int64_t w, const float* src, int64_t lds, float* dst,
                                  int64_t ldd, int64_t col0, cudaStream_t st) {
  return chol_panel_rec_f32(m, w, src, lds, dst, ldd, col0, x.sb_pan, x.fail, st);
}

// Panel p as broadcast: rows [ps, n) of its w columns, packed (ld = n - ps) into the rank's
// receive buffer buf[p & 1] — on the owner by one strided device copy right after the panel
// is factored, on the others by the broadcast.  Rows [0, ps) are never sent: an in-place
// broadcast of the owner's storage would move the contiguous span from (ps, first column)
// to (n-1, last column), about twice the bytes (n*w instead of (n - ps)*w).  Every rank,
// the owner included, then flushes from the packed copy (same operations, only the operand
// leading dimension differs: results bitwise equal).
template <typename T>
struct Span {
  const Cyclic& cy; int64_t ld;
  int64_t ldp(int64_t p) const { return cy.n - p * cy.s; }
  size_t count(int64_t p) const { return (size_t)ldp(p) * (size_t)cy.width(p); }
  T* at(Rank<T>& x, int64_t p) const { return x.buf[p & 1]; }
  // owner: copy the factored panel into its packed buffer; `prev` = the buffer's last reader
  int pack(Rank<T>& x, int64_t p, cudaEvent_t prev, cudaStream_t st) const {
    if (prev) SF_CUDA(cudaStreamWaitEvent(st, prev, 0));
    const T* src = x.X + p * cy.s + cy.slot(p) * cy.s * ld;
    SF_CUDA(cudaMemcpy2DAsync(at(x, p), sizeof(T) * ldp(p), src, sizeof(T) * ld, sizeof(T) * ldp(p), cy.width(p),
                              cudaMemcpyDeviceToDevice, st));
    return SF_OK;
  }
};

// Panel exchange of the Span-packed drivers (Cholesky, LU): the broadcast (pack + NCCL /
// loopback copy) or the push (f3).  send() after the owner factored panel q (panel stream),
// recv(p) before the flushes of panel p (leaves recv[p] recorded where the flush waits),
// consumed() after a rank's flush of panel p (main stream).
template <typename T>
struct PanelXfer {
  sf_comm_t comm;
  std::vector<Rank<T>>& rk;
  const Span<T>& sp;
  bool push = false;
  unsigned long long call = 0;
  std::vector<T*> gbuf[2];               // every rank's receive buffer per slot (device addresses)
  std::vector<PushFlags*> gflags;        // every rank's flags
  std::vector<PushFlags*> lflags;        // the local ranks' own flags

  PanelXfer(sf_comm_t c, std::vector<Rank<T>>& r, const Span<T>& s) : comm(c), rk(r), sp(s) {}
  unsigned long long tag(int64_t p) const { return (call << 32) | (unsigned long long)(p + 1); }

  int setup(size_t buf_elems, cudaStream_t caller) {
    push = comm->push != 0;
    call = ++comm->calls;
    if (!push) return SF_OK;
    const int G = comm->nranks;
    if (G > kMaxPushRanks) return fail_with(SF_EINVAL, "push transport supports at most %d ranks", kMaxPushRanks);
    gbuf[0].assign(G, nullptr); gbuf[1].assign(G, nullptr); gflags.assign(G, nullptr);
    if (comm->loopback()) {
      for (auto& x : rk) {
        PushFlags* f = x.ws.template take<PushFlags>(1);
        SF_CUDA(cudaMemsetAsync(f, 0, sizeof(PushFlags), caller));
        gbuf[0][x.r] = x.buf[0]; gbuf[1][x.r] = x.buf[1]; gflags[x.r] = f;
        lflags.push_back(f);
      }
    } else {
      const size_t bb = (buf_elems * sizeof(T) + 255) & ~(size_t)255;
      if (int rc = ensure_window(comm, bb)) return rc;
      Rank<T>& me = rk[0];
      me.buf[0] = (T*)((char*)comm->win_base + kFlagBytes);
      me.buf[1] = (T*)((char*)comm->win_base + kFlagBytes + bb);
      for (int r = 0; r < G; ++r) {
        gflags[r] = (PushFlags*)comm->peer_base[r];
        gbuf[0][r] = (T*)(comm->peer_base[r] + kFlagBytes);
        gbuf[1][r] = (T*)(comm->peer_base[r] + kFlagBytes + bb);
      }
      lflags.push_back((PushFlags*)comm->win_base);   // tags grow across calls: no reset
    }
    cudaEvent_t e = pool_event();   // the rank streams see the zeroed flags
    SF_CUDA(cudaEventRecord(e, caller));
    for (auto& x : rk) { SF_CUDA(wait_on(x.st.mn, e)); SF_CUDA(wait_on(x.st.pan, e)); }
    return SF_OK;
  }
  PushFlags* own(const Rank<T>& x) const { return comm->loopback() ? lflags[x.r] : lflags[0]; }

  int send(Rank<T>& x, int64_t q, cudaEvent_t prev, cudaStream_t st) {
    if (!push) return sp.pack(x, q, prev, st);
    const int G = comm->nranks;
    if (q >= 2) {   // every rank finished flushing panel q-2 out of this slot
      PushTargets w{};
      w.G = G;
      for (int r = 0; r < G; ++r) w.flag[r] = &own(x)->consumed[r];
      wait_flags_kernel<<<1, 32, 0, st>>>(w, tag(q - 2));
      count_launch();
    }
    const int slot = (int)(q & 1);
    PushTargets tg{};
    tg.G = G;
    for (int r = 0; r < G; ++r) { tg.dst[r] = gbuf[slot][r]; tg.flag[r] = &gflags[r]->ready[slot]; }
    const int64_t m = sp.ldp(q);
    const T* src = x.X + q * sp.cy.s + sp.cy.slot(q) * sp.cy.s * sp.ld;
    const int64_t total = m * sp.cy.width(q);
    int grid = (int)((total + 255) / 256);
    if (grid > 4 * 148) grid = 4 * 148;
    push_panel_kernel<T><<<grid, 256, 0, st>>>(src, sp.ld, m, (int)sp.cy.width(q), tg, tag(q), &own(x)->counter);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? SF_OK : fail_with(SF_ECUDA, "push_panel_kernel launch");
  }
  template <typename FreeF>
  int recv(int64_t p, int owner, FreeF free_ev) {
    if (!push)
      return exchange<T>(comm, rk, p, owner, sp.count(p), [&](Rank<T>& x) { return sp.at(x, p); }, free_ev);
    comm->bcast_bytes += (int64_t)(sp.count(p) * sizeof(T));
    for (auto& x : rk) {
      PushTargets w{};
      w.G = 1;
      w.flag[0] = &own(x)->ready[p & 1];
      ProfScope pb(3, (double)(sp.count(p) * sizeof(T)), x.st.mn);
      wait_flags_kernel<<<1, 32, 0, x.st.mn>>>(w, tag(p));
      count_launch();
      SF_CUDA(cudaEventRecord(x.recv[p], x.st.mn));
    }
    return SF_OK;
  }
  int consumed(Rank<T>& x, int64_t p, cudaStream_t st) {
    if (!push) return SF_OK;
    PushTargets w{};
    w.G = comm->nranks;
    for (int r = 0; r < w.G; ++r) w.flag[r] = &gflags[r]->consumed[x.r];
    signal_flags_kernel<<<1, 32, 0, st>>>(w, tag(p));
    count_launch();
    return SF_OK;
  }
};

template <typename T>
static int chol_dist_run(sf_comm_t comm, int64_t n, int64_t s, void* const* dA, void* const* dL, int64_t ld,
                         int64_t* const* d_info, cudaStream_t caller) {
  const Cyclic cy(n, s, comm->nranks);
  std::vector<Rank<T>> rk;
  const int64_t ldk = (s + 3) / 4 * 4;
  const size_t split_elems = std::is_same<T, float>::value ? 4 * (size_t)n * ldk + 1024 : 0;
  int rc = setup_ranks<T>(comm, rk, cy, dA, dL, nullptr, d_info, (size_t)s * ld, 0, split_elems, caller);
  if (rc) return rc;
  if (std::is_same<T, float>::value) {
    for (auto& x : rk) {
      x.sb_upd = SplitBuf{(float*)x.ws.template take<T>((size_t)n * ldk), nullptr, ldk};
      x.sb_upd.l = (float*)x.ws.template take<T>((size_t)n * ldk);
      x.sb_pan = SplitBuf{(float*)x.ws.template take<T>((size_t)n * ldk), nullptr, ldk};
      x.sb_pan.l = (float*)x.ws.template take<T>((size_t)n * ldk);
    }
  }
  const Span<T> sp{cy, ld};
  PanelXfer<T> xf(comm, rk, sp);
  rc = xf.setup((size_t)s * ld, caller);
  if (rc) return rc;
  // prologue: panel 0 on its owner, out of place from A
  for (auto& o : rk) {
    if (o.r != 0) continue;
    {
      ProfScope ps(1, 0.0, o.st.pan);
      SF_CUDA(chol_panel_any(o, n, cy.width(0), o.A, ld, o.X, ld, 0, o.st.pan));
    }
    if (cy.P > 1) { rc = xf.send(o, 0, nullptr, o.st.pan); if (rc) return rc; }
    SF_CUDA(cudaEventRecord(o.ready[0], o.st.pan));
  }
  for (int64_t p = 0; p + 1 < cy.P; ++p) {   // the last panel is never flushed: not sent
    rc = xf.recv(p, cy.owner(p), [&](Rank<T>& x) -> cudaEvent_t { return p >= 2 ? x.done[p - 2] : nullptr; });
    if (rc) return rc;
    for (auto& x : rk) {
      SF_CUDA(wait_on(x.st.mn, x.recv[p]));
      const T* Lp = sp.at(x, p);
      const int64_t ldp = sp.ldp(p);
      const int64_t nslots = (cy.local_cols(x.r) + s - 1) / s;
      SF_CUDA(chol_split_panel(cy, x, p, Lp, ldp, x.st.mn));
      int64_t j0 = cy.first_slot_after(p, x.r);
      if (cy.owner(p + 1) == x.r) {
        // lookahead: flush into panel p+1 first, factor it while the rest of the flush runs
        const int64_t q = p + 1, qs = q * s, wq = cy.width(q), j = cy.slot(q);
        {
          double fl = 0.0;
          ProfScope pf(0, 0.0, x.st.mn);
          SF_CUDA(chol_update_slots(cy, x, p, j, j + 1, Lp, ldp, ld, &fl, x.st.mn));
          pf.r.flops = fl;
        }
        j0 = j + 1;
        SF_CUDA(cudaEventRecord(x.la[q], x.st.mn));
        SF_CUDA(wait_on(x.st.pan, x.la[q]));
        {
          ProfScope pp(1, 0.0, x.st.pan);
          T* P0 = x.X + qs + j * s * ld;
          SF_CUDA(chol_panel_any(x, n - qs, wq, P0, ld, P0, ld, qs, x.st.pan));
        }
        if (q + 1 < cy.P) { rc = xf.send(x, q, q >= 2 ? x.done[q - 2] : nullptr, x.st.pan); if (rc) return rc; }
        SF_CUDA(cudaEventRecord(x.ready[q], x.st.pan));
      }
      {
        double fl = 0.0;
        ProfScope pf(0, 0.0, x.st.mn);
        SF_CUDA(chol_update_slots(cy, x, p, j0, nslots, Lp, ldp, ld, &fl, x.st.mn));
        pf.r.flops = fl;
      }
      SF_CUDA(cudaEventRecord(x.done[p], x.st.mn));
      rc = xf.consumed(x, p, x.st.mn);
      if (rc) return rc;
    }
  }
  for (auto& x : rk) { rc = join_rank<T>(x); if (rc) return rc; }
  return finish_dist<T>(comm, rk, caller);
}

// ------------------------------------------------------------------ LU
// Flush of panel p into rank x's local columns [c0, c1) (all right of panel p):
// U rows [ps, ps+wp) := L11^-1 (rows) with the Crout division, then
// rows [ps+wp, n) -= L21 U12.
template <typename T>
static cudaError_t lu_update_cols(const Cyclic& cy, Rank<T>& x, int64_t p, int64_t c0, int64_t c1, const T* Lp,
                                  int64_t ldp, int64_t ld, double* flops, cudaStream_t st) {
  if (c1 <= c0) return cudaSuccess;
  const int64_t ps = p * cy.s, wp = cy.width(p), nc = c1 - c0;
  T* U = x.X + ps + c0 * ld;
  cudaError_t e = lu_usolve_rec<T>(wp, nc, Lp, ldp, U, ld, x.fail, st);
  if (e != cudaSuccess) return e;
  const int64_t m = cy.n - ps - wp;
  *flops += 2.0 * (double)wp * (double)m * (double)nc;
  return gemm_sub<T>(m, nc, wp, Lp + wp, ldp, 0, U, ld, 1, U + wp, ld, U + wp, ld, kMaskNone, x.fail, st);
}

template <typename T>
static int lu_dist_run(sf_comm_t comm, int64_t n, int64_t s, void* const* dA, void* const* dLU, int64_t ld,
                       int64_t* const* d_info, cudaStream_t caller) {
  const Cyclic cy(n, s, comm->nranks);
  std::vector<Rank<T>> rk;
  int rc = setup_ranks<T>(comm, rk, cy, dA, dLU, nullptr, d_info, (size_t)s * ld, 0, 0, caller);
  if (rc) return rc;
  rc = dist_tol<T>(comm, rk, cy, ld, caller);
  if (rc) return rc;
  // out of place: the whole local matrix is rewritten, so start from a copy of A
  for (auto& x : rk) {
    if (x.A != x.X) SF_CUDA(copy_matrix<T>(n, cy.local_cols(x.r), x.A, ld, x.X, ld, caller));
    cudaEvent_t e = pool_event();
    SF_CUDA(cudaEventRecord(e, caller));
    SF_CUDA(wait_on(x.st.mn, e)); SF_CUDA(wait_on(x.st.pan, e)); SF_CUDA(wait_on(x.st.com, e));
  }
  const Span<T> sp{cy, ld};   // the L panel incl. U11 in its diagonal block
  PanelXfer<T> xf(comm, rk, sp);
  rc = xf.setup((size_t)s * ld, caller);
  if (rc) return rc;
  for (auto& o : rk) {
    if (o.r != 0) continue;
    {
      ProfScope ps(1, 0.0, o.st.pan);
      SF_CUDA(lu_panel_rec<T>(n, cy.width(0), 0, o.X, ld, o.X, ld, 0, o.tol, o.fail, o.st.pan));
    }
    if (cy.P > 1) { rc = xf.send(o, 0, nullptr, o.st.pan); if (rc) return rc; }
    SF_CUDA(cudaEventRecord(o.ready[0], o.st.pan));
  }
  for (int64_t p = 0; p + 1 < cy.P; ++p) {   // the last panel is never flushed: not sent
    rc = xf.recv(p, cy.owner(p), [&](Rank<T>& x) -> cudaEvent_t { return p >= 2 ? x.done[p - 2] : nullptr; });
    if (rc) return rc;
    for (auto& x : rk) {
      SF_CUDA(wait_on(x.st.mn, x.recv[p]));
      const T* Lp = sp.at(x, p);
      const int64_t ldp = sp.ldp(p);
      const int64_t nloc = cy.local_cols(x.r);
      int64_t c0 = cy.first_slot_after(p, x.r) * s;
      if (cy.owner(p + 1) == x.r) {
        const int64_t q = p + 1, qs = q * s, wq = cy.width(q), j = cy.slot(q);
        {
          double fl = 0.0;
          ProfScope pf(0, 0.0, x.st.mn);
          SF_CUDA(lu_update_cols<T>(cy, x, p, j * s, j * s + wq, Lp, ldp, ld, &fl, x.st.mn));
          pf.r.flops = fl;
        }
        c0 = j * s + wq;
        SF_CUDA(cudaEventRecord(x.la[q], x.st.mn));
        SF_CUDA(wait_on(x.st.pan, x.la[q]));
        {
          ProfScope pp(1, 0.0, x.st.pan);
          T* P0 = x.X + qs + j * s * ld;
          SF_CUDA(lu_panel_rec<T>(n - qs, wq, 0, P0, ld, P0, ld, qs, x.tol, x.fail, x.st.pan));
        }
        if (q + 1 < cy.P) { rc = xf.send(x, q, q >= 2 ? x.done[q - 2] : nullptr, x.st.pan); if (rc) return rc; }
        SF_CUDA(cudaEventRecord(x.ready[q], x.st.pan));
      }
      {
        double fl = 0.0;
        ProfScope pf(0, 0.0, x.st.mn);
        SF_CUDA(lu_update_cols<T>(cy, x, p, c0, nloc, Lp, ldp, ld, &fl, x.st.mn));
        pf.r.flops = fl;
      }
      SF_CUDA(cudaEventRecord(x.done[p], x.st.mn));
      rc = xf.consumed(x, p, x.st.mn);
      if (rc) return rc;
    }
  }
  for (auto& x : rk) { rc = join_rank<T>(x); if (rc) return rc; }
  return finish_dist<T>(comm, rk, caller);
}

// ------------------------------------------------------------------ QR
template <typename T>
static int qr_dist_run(sf_comm_t comm, int64_t n, int64_t s, void* const* dA, void* const* dQ, void* const* dR,
                       int64_t ld, int64_t* const* d_info, cudaStream_t caller) {
  const Cyclic cy(n, s, comm->nranks);
  const int64_t wmax = qr_mgs_max_width(n, (int)sizeof(T));
  const int64_t wcap = s < wmax ? s : wmax;
  const size_t mgs_elems = qr_mgs_work_elems(n, (int)wcap, (int)sizeof(T)) + 64;
  const int64_t cw_elems = s * n;
  int64_t split_elems = 1;
  for (int64_t p = 0; p + 1 < cy.P; ++p) {
    for (int r = 0; r < cy.G; ++r) {
      const int64_t nc = cy.local_cols(r) - cy.first_slot_after(p, r) * s;
      if (nc <= 0) continue;
      const int sp = splitk_for(cy.width(p), nc, n);
      if ((int64_t)sp * cy.width(p) * nc > split_elems) split_elems = (int64_t)sp * cy.width(p) * nc;
    }
  }
  if (s > wmax) {
    const int sp = splitk_for(s, wmax, n);
    if ((int64_t)sp * s * wmax > split_elems) split_elems = (int64_t)sp * s * wmax;
  }
  std::vector<Rank<T>> rk;
  const size_t extra = mgs_elems + 2 * cw_elems + 2 * split_elems + 1024;
  int rc = setup_ranks<T>(comm, rk, cy, dA, dQ, dR, d_info, 0, (size_t)n * n, extra, caller);
  if (rc) return rc;
  for (auto& x : rk) {
    x.mgsw = x.ws.template take<T>(mgs_elems);
    x.cw = x.ws.template take<T>(cw_elems); x.cw2 = x.ws.template take<T>(cw_elems);
    x.split = x.ws.template take<T>(split_elems); x.split2 = x.ws.template take<T>(split_elems);
    x.split_elems = split_elems;
    SF_CUDA(cudaMemsetAsync(x.mgsw, 0, sizeof(T) * mgs_elems, caller));   // MGS flags (epochs start at 0)
  }
  rc = dist_tol<T>(comm, rk, cy, ld, caller);
  if (rc) return rc;
  for (auto& x : rk) {   // M := A lives in Q
    SF_CUDA(copy_matrix<T>(n, cy.local_cols(x.r), x.A, ld, x.X, ld, caller));
    cudaEvent_t e = pool_event();
    SF_CUDA(cudaEventRecord(e, caller));
    SF_CUDA(wait_on(x.st.mn, e)); SF_CUDA(wait_on(x.st.pan, e)); SF_CUDA(wait_on(x.st.com, e));
  }
  for (auto& o : rk) {
    if (o.r != 0) continue;
    ProfScope ps(1, 0.0, o.st.pan);
    const int64_t w0 = cy.width(0);
    SF_CUDA(qr_panel<T>(n, w0, o.X, ld, o.X, ld, 0, o.tol, o.mgsw, o.cw2, o.split2, o.split_elems, o.fail, o.st.pan));
    SF_CUDA(cudaMemcpy2DAsync(o.qfull, n * sizeof(T), o.X, ld * sizeof(T), n * sizeof(T), w0,
                              cudaMemcpyDeviceToDevice, o.st.pan));
    SF_CUDA(cudaEventRecord(o.ready[0], o.st.pan));
  }
  for (int64_t p = 0; p < cy.P; ++p) {
    rc = exchange<T>(comm, rk, p, cy.owner(p), (size_t)n * cy.width(p),
                     [&](Rank<T>& x) { return x.qfull + p * s * n; },
                     [&](Rank<T>&) -> cudaEvent_t { return nullptr; });
    if (rc) return rc;
    if (p + 1 == cy.P) break;
    const int64_t wp = cy.width(p);
    for (auto& x : rk) {
      SF_CUDA(wait_on(x.st.mn, x.recv[p]));
      const T* BQ = x.qfull + p * s * n;   // B_Q = Q[:, z:c)
      const int64_t nloc = cy.local_cols(x.r);
      int64_t c0 = cy.first_slot_after(p, x.r) * s;
      if (cy.owner(p + 1) == x.r) {
        const int64_t q = p + 1, qs = q * s, wq = cy.width(q), j = cy.slot(q);
        T* V = x.X + j * s * ld;
        {
          ProfScope pf(0, 4.0 * (double)n * wp * wq, x.st.mn);
          SF_CUDA(qr_project<T>(n, wp, wq, BQ, n, V, ld, V, ld, x.cw, x.split, x.split_elems, x.fail, x.st.mn));
        }
        c0 = j * s + wq;
        SF_CUDA(cudaEventRecord(x.la[q], x.st.mn));
        SF_CUDA(wait_on(x.st.pan, x.la[q]));
        {
          ProfScope pp(1, 0.0, x.st.pan);
          SF_CUDA(qr_panel<T>(n, wq, V, ld, V, ld, qs, x.tol, x.mgsw, x.cw2, x.split2, x.split_elems, x.fail,
                              x.st.pan));
          SF_CUDA(cudaMemcpy2DAsync(x.qfull + qs * n, n * sizeof(T), V, ld * sizeof(T), n * sizeof(T), wq,
                                    cudaMemcpyDeviceToDevice, x.st.pan));
        }
        SF_CUDA(cudaEventRecord(x.ready[q], x.st.pan));
      }
      if (nloc > c0) {
        ProfScope pf(0, 4.0 * (double)n * wp * (double)(nloc - c0), x.st.mn);
        T* V = x.X + c0 * ld;
        SF_CUDA(qr_project<T>(n, wp, nloc - c0, BQ, n, V, ld, V, ld, x.cw, x.split, x.split_elems, x.fail, x.st.mn));
      }
      SF_CUDA(cudaEventRecord(x.done[p], x.st.mn));
    }
  }
  // R := Q^T A on the local columns: upper part of each local panel, one
  // grouped launch over the slots (the full Q is on every rank), exact zeros below
  for (auto& x : rk) {
    rc = join_rank<T>(x);
    if (rc) return rc;
    const int64_t nloc = cy.local_cols(x.r);
    if (nloc == 0) continue;
    zero_lower_cyclic_kernel<T><<<dim3(4, 1024), 256, 0, x.st.mn>>>(n, s, cy.G, x.r, nloc, x.R, ld);
    count_launch();
    std::vector<GemmGroup> gs;
    double fl = 0.0;
    for (int64_t j = 0; j * s < nloc; ++j) {
      const int64_t q = cy.panel_of(j, x.r), qs = q * s, wq = cy.width(q);
      GemmGroup g{};
      g.M = qs + wq; g.N = wq; g.off = qs;
      g.A = (const double*)x.qfull; g.B = (const double*)(x.A + j * s * ld);
      g.Cin = nullptr; g.C = (double*)(x.R + j * s * ld);
      gs.push_back(g);
      fl += 2.0 * n * ((double)wq * qs + 0.5 * (double)wq * (wq + 1));
    }
    ProfScope pr(2, fl, x.st.mn);
    if (std::is_same<T, double>::value) {
      GemmF64 p64{0, n, n, nullptr, n, nullptr, ld, nullptr, 0, nullptr, ld, 1.0, 0, 1, nullptr, x.fail};
      SF_CUDA(gemm_f64_grouped(p64, gs.data(), (int)gs.size(), 1, 1, kMaskUpper, x.st.mn));
    } else {
      for (int64_t j = 0; j * s < nloc; ++j) {   // fp32: one 3xTF32 launch per local panel
        const int64_t q = cy.panel_of(j, x.r), qs = q * s, wq = cy.width(q);
        Gemm<T> g{qs + wq, wq, n, x.qfull, n, 1, x.A + j * s * ld, ld, 1, nullptr, 0, x.R + j * s * ld, ld,
                  1.0, 0, kMaskUpper, 1, nullptr, x.fail};
        g.off = qs;
        SF_CUDA(run_gemm(g, x.st.mn));
      }
    }
  }
  return finish_dist<T>(comm, rk, caller);
}

}  // namespace sf

using namespace sf;

extern "C" {

int sf_get_unique_id(uint8_t id[128]) {
  if (!id) return fail_with(SF_EINVAL, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  SF_NCCL(ncclGetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return SF_OK;
}

int sf_comm_init(sf_comm_t* comm, int nranks, int rank, const uint8_t id[128]) {
  SF_API_LOCK;
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail_with(SF_EINVAL, "bad communicator arguments");
  sf_comm_* c = new sf_comm_();
  c->nranks = nranks; c->rank = rank;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) { delete c; return fail_with(SF_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e)); }
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) { delete c; return fail_with(SF_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)); }
  *comm = c;
  return SF_OK;
}

int sf_comm_init_loopback(sf_comm_t* comm, int nranks) {
  SF_API_LOCK;
  if (!comm || nranks < 1) return fail_with(SF_EINVAL, "bad communicator arguments");
  sf_comm_* c = new sf_comm_();
  c->nranks = nranks; c->rank = 0;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) { delete c; return fail_with(SF_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e)); }
  *comm = c;
  return SF_OK;
}

int sf_comm_destroy(sf_comm_t comm) {
  SF_API_LOCK;
  if (!comm) return SF_OK;
  int rc = SF_OK;
  if (comm->win) {
    cudaDeviceSynchronize();
    ncclCommWindowDeregister(comm->nccl, comm->win);
    ncclMemFree(comm->win_base);
  }
  if (comm->nccl) {
    ncclResult_t r = ncclCommDestroy(comm->nccl);
    if (r != ncclSuccess) rc = fail_with(SF_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  }
  delete comm;
  return rc;
}

int sf_comm_set_push(sf_comm_t comm, int on) {
  SF_API_LOCK;
  if (!comm || (on != 0 && on != 1)) return fail_with(SF_EINVAL, "sf_comm_set_push: bad arguments");
  if (on && comm->nranks > sf::kMaxPushRanks) return fail_with(SF_EINVAL, "push transport: at most %d ranks", sf::kMaxPushRanks);
  comm->push = on;
  return SF_OK;
}
int sf_comm_size(sf_comm_t comm) { return comm ? comm->nranks : 0; }
int64_t sf_comm_bcast_bytes(sf_comm_t comm) { return comm ? comm->bcast_bytes : -1; }
int sf_comm_local_ranks(sf_comm_t comm) { return comm ? comm->nlocal() : 0; }

int64_t sf_local_cols(int64_t n, int64_t s, int nranks, int rank) {
  if (n < 1 || s < 1 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
  return Cyclic(n, s, nranks).local_cols(rank);
}

static int check_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* a, void* const* o, int64_t ld,
                      int64_t* const* info) {
  if (!comm) return fail_with(SF_EINVAL, "null communicator");
  if (n < 1) return fail_with(SF_EINVAL, "n=%lld < 1", (long long)n);
  if (s < 1 || s > n) return fail_with(SF_EINVAL, "step s=%lld outside [1, n=%lld]", (long long)s, (long long)n);
  if (dtype != SF_F64 && dtype != SF_F32) return fail_with(SF_EINVAL, "unknown dtype %d", dtype);
  if (ld < n) return fail_with(SF_EINVAL, "ld_local < n");
  if (!a || !o || !info) return fail_with(SF_EINVAL, "null pointer array");
  for (int i = 0; i < comm->nlocal(); ++i) {
    const int64_t nl = sf_local_cols(n, s, comm->nranks, comm->local_rank(i));
    if (!info[i]) return fail_with(SF_EINVAL, "null d_info");
    if (nl > 0 && (!a[i] || !o[i])) return fail_with(SF_EINVAL, "null local matrix");
  }
  return SF_OK;
}

int chol_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dL_local,
                     int64_t ld_local, int64_t* const* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_dist(comm, n, s, dtype, dA_local, dL_local, ld_local, d_info);
  if (rc) return rc;
  if (dtype == SF_F32) return chol_dist_run<float>(comm, n, s, dA_local, dL_local, ld_local, d_info, (cudaStream_t)stream);
  return chol_dist_run<double>(comm, n, s, dA_local, dL_local, ld_local, d_info, (cudaStream_t)stream);
}

int lu_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dLU_local,
                   int64_t ld_local, int64_t* const* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_dist(comm, n, s, dtype, dA_local, dLU_local, ld_local, d_info);
  if (rc) return rc;
  if (dtype == SF_F32) return lu_dist_run<float>(comm, n, s, dA_local, dLU_local, ld_local, d_info, (cudaStream_t)stream);
  return lu_dist_run<double>(comm, n, s, dA_local, dLU_local, ld_local, d_info, (cudaStream_t)stream);
}

int qr_factor_dist(sf_comm_t comm, int64_t n, int64_t s, int dtype, void* const* dA_local, void* const* dQ_local,
                   void* const* dR_local, int64_t ld_local, int64_t* const* d_info, void* stream) {
  SF_API_LOCK;
  int rc = check_dist(comm, n, s, dtype, dA_local, dQ_local, ld_local, d_info);
  if (rc) return rc;
  if (!dR_local) return fail_with(SF_EINVAL, "null pointer array");
  for (int i = 0; i < comm->nlocal(); ++i)
    if (sf_local_cols(n, s, comm->nranks, comm->local_rank(i)) > 0 &&
        (!dR_local[i] || dR_local[i] == dQ_local[i] || dR_local[i] == dA_local[i] || dQ_local[i] == dA_local[i]))
      return fail_with(SF_EINVAL, "qr_factor_dist outputs must not alias");
  if (dtype == SF_F32)
    return qr_dist_run<float>(comm, n, s, dA_local, dQ_local, dR_local, ld_local, d_info, (cudaStream_t)stream);
  return qr_dist_run<double>(comm, n, s, dA_local, dQ_local, dR_local, ld_local, d_info, (cudaStream_t)stream);
}

}  // extern "C"
