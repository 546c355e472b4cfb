// Diagnostic: where does a column step of the register-resident MGS panel kernel spend its
// time?  A copy of qr_mgs_reg_kernel's loop with %globaltimer stamps per phase (CTA 0 and
// the last CTA, thread 0).  Not part of the library.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_relaxed_s32(const int* p) { int v; asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_release_s32(int* p, int v) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <typename T> __device__ __forceinline__ T warp_sum(T v) { for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }

constexpr int NT = 256, RPT = 64, MAXT = 16;
// FENCE: 0 = __threadfence + st.release, 1 = st.release only
template <int FENCE, int SLEEP>
__global__ void __launch_bounds__(NT) mgs(int n, int w, int RB, double* V, int* flags, double* partbase, unsigned long long* stamps) {
  constexpr int QP = RPT + 2;
  __shared__ double qs[2 * QP], vs[2 * QP], gsum[128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT / 32;
  const int G = gridDim.x, g = blockIdx.x;
  const int r0 = g * RB, rows = min(RB, n - r0);
  const int cp = tid >> 1, h = tid & 1, rbase = h * RPT;
  const bool mine = cp < w;
  double x[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) x[r] = (mine && rbase + r < rows) ? V[r0 + rbase + r + (size_t)cp * n] : 0.0;
  if (cp == 0) for (int r = 0; r < RPT; ++r) vs[h * QP + r] = x[r];
  __syncthreads();
  { double acc = 0; for (int r = 0; r < RPT; ++r) acc = fma(vs[h * QP + r], x[r], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1); if (mine && h == 0) partbase[(size_t)cp * G + g] = acc; }
  unsigned long long tw = 0, tr = 0, tc = 0, t0, t1;
  const bool rec = (g == 0 || g == G - 1) && tid == 0;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    double* part = partbase + (size_t)buf * G * w;
    __syncthreads();
    t0 = gtime();
    if (tid == 0) { if (FENCE == 0) __threadfence(); st_release_s32(flags + buf * G + g, c + 1); }
    if (warp == 0) {
      for (;;) { bool all = true; for (int hh = lane; hh < G; hh += 32) all &= ld_relaxed_s32(flags + buf * G + hh) >= c + 1;
        if (__all_sync(0xffffffffu, all)) break; if (SLEEP) __nanosleep(SLEEP); }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    t1 = gtime(); tw += t1 - t0; t0 = t1;
    for (int cb = c + warp; cb < w; cb += nwarps * MAXT) {
      double acc[MAXT];
      for (int t = 0; t < MAXT; ++t) acc[t] = 0;
      for (int hh = lane; hh < G; hh += 32)
#pragma unroll
        for (int t = 0; t < MAXT; ++t) { const int cc = cb + t * nwarps; if (cc < w) acc[t] += __ldcg(part + (size_t)cc * G + hh); }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) { const int cc = cb + t * nwarps; const double v = warp_sum(acc[t]); if (lane == 0 && cc < w) gsum[cc] = v; }
    }
    __syncthreads();
    t1 = gtime(); tr += t1 - t0; t0 = t1;
    const double nv = sqrt(gsum[c]), rnv = 1.0 / nv;
    if (cp == c) for (int r = 0; r < RPT; ++r) { x[r] *= rnv; qs[h * QP + r] = x[r]; }
    if (cp == c + 1) for (int r = 0; r < RPT; ++r) vs[h * QP + r] = x[r];
    __syncthreads();
    const bool act = mine && cp > c;
    double acc = 0;
    if (act) {
      const double coef = gsum[cp] * rnv, cn = (c + 1 < w) ? gsum[c + 1] * rnv : 0.0;
#pragma unroll
      for (int r = 0; r < RPT; ++r) { const double qr = qs[h * QP + r]; x[r] = fma(-qr, coef, x[r]); acc = fma(fma(-qr, cn, vs[h * QP + r]), x[r], acc); }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (act && h == 0 && c + 1 < w) partbase[(size_t)(buf ^ 1) * G * w + (size_t)cp * G + g] = acc;
    t1 = gtime(); tc += t1 - t0;
  }
  if (rec) { const int k = g == 0 ? 0 : 3; stamps[k] = tw; stamps[k + 1] = tr; stamps[k + 2] = tc; }
  if (mine) for (int r = 0; r < RPT; ++r) if (rbase + r < rows) V[r0 + rbase + r + (size_t)cp * n] = x[r];
}


#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ void st_ll(unsigned long long* p, double v, unsigned ep) {
  const unsigned long long b = __double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)ep << 32) | (b & 0xffffffffull), w1 = ((unsigned long long)ep << 32) | (b >> 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ bool ld_ll(const unsigned long long* p, unsigned ep, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  if ((unsigned)(w0 >> 32) != ep || (unsigned)(w1 >> 32) != ep) return false;
  v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return true;
}
// LL exchange: cluster-level reduction through DSMEM, then one 16-byte {data, epoch} word per
// (cluster, column) in global memory that readers poll directly (no separate flag).
template <int CL, int POLL>
__global__ void __launch_bounds__(NT) mgs_ll(int n, int w, int RB, double* V, int* flags, double* partbase, unsigned long long* stamps) {
  constexpr int QP = RPT + 2;
  __shared__ double qs[2 * QP], vs[2 * QP], gsum[128];
  __shared__ double mypart[2][128];
  __shared__ double cval[40][128];
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x;
  const int G = gridDim.x, g = blockIdx.x, Q = G / CL, q = g / CL, k = (int)cluster.block_rank();
  unsigned long long* ll = reinterpret_cast<unsigned long long*>(partbase);   // [2][Q][w] x 2 words
  const int r0 = g * RB, rows = min(RB, n - r0);
  const int cp = tid >> 1, h = tid & 1, rbase = h * RPT;
  const bool mine = cp < w;
  double x[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) x[r] = (mine && rbase + r < rows) ? V[r0 + rbase + r + (size_t)cp * n] : 0.0;
  if (cp == 0) for (int r = 0; r < RPT; ++r) vs[h * QP + r] = x[r];
  __syncthreads();
  { double acc = 0; for (int r = 0; r < RPT; ++r) acc = fma(vs[h * QP + r], x[r], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1); if (mine && h == 0) mypart[0][cp] = acc; }
  unsigned long long tw = 0, tr = 0, tc = 0, t0, t1;
  const bool rec = (g == 0 || g == G - 1) && tid == 0;
  for (int c = 0; c < w; ++c) {
    const int buf = c & 1;
    const unsigned ep = c + 1;
    t0 = gtime();
    cluster.sync();
    // cluster sum of columns j = c + k + CL*i (fixed rank order), published as LL words
    for (int j = c + k + CL * tid; j < w; j += CL * NT) {
      double a = 0;
      for (int rr = 0; rr < CL; ++rr) a += cluster.map_shared_rank(&mypart[buf][0], rr)[j];
      st_ll(ll + 2 * ((size_t)(buf * Q + q) * w + j), a, ep);
    }
    t1 = gtime(); tw += t1 - t0; t0 = t1;
    // poll: thread j-c owns column j and loads all Q cluster words of it at once
    if (POLL == 1) {
      const int j = c + tid;
      if (j < w) {
        double v[16];
        bool okq[16];
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) okq[qq] = qq >= Q;
        for (long long spins = 0;; ++spins) {
          bool all = true;
#pragma unroll
          for (int qq = 0; qq < 16; ++qq)
            if (!okq[qq]) { okq[qq] = ld_ll(ll + 2 * ((size_t)(buf * Q + qq) * w + j), ep, v[qq]); all &= okq[qq]; }
          if (all) break;
          if (spins > (1 << 22)) { stamps[7] = 1000000ull * c + j; break; }
        }
        double a = 0;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) if (qq < Q) a += v[qq];
        gsum[j] = a;
      }
      __syncthreads();
    } else if (POLL == 2) {
      if ((tid >> 5) == 0) {
        const int lane = tid & 31;
        const int cnt = Q * (w - c);
        for (int base = 0; base < cnt; base += 32 * 8) {
          double v[8]; bool okk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) okk[i] = base + lane + 32 * i >= cnt;
          for (long long spins = 0;; ++spins) {
            bool all = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int idx = base + lane + 32 * i;
              if (!okk[i]) { const int qq = idx / (w - c), j = c + idx % (w - c); okk[i] = ld_ll(ll + 2 * ((size_t)(buf * Q + qq) * w + j), ep, v[i]); all &= okk[i]; }
            }
            if (all) break;
            if (spins > (1 << 22)) { stamps[7] = 1; break; }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) { const int idx = base + lane + 32 * i; if (idx < cnt) cval[idx / (w - c)][c + idx % (w - c)] = v[i]; }
        }
      }
      __syncthreads();
      for (int j = c + tid; j < w; j += NT) { double a = 0; for (int qq = 0; qq < Q; ++qq) a += cval[qq][j]; gsum[j] = a; }
      __syncthreads();
    } else {
    const int cnt = Q * (w - c);
    for (int idx = tid; idx < cnt; idx += NT) {
      const int qq = idx / (w - c), j = c + idx % (w - c);
      double v;
      const unsigned long long* p = ll + 2 * ((size_t)(buf * Q + qq) * w + j);
      long long spins = 0;
      while (!ld_ll(p, ep, v)) { if (POLL == 3) __nanosleep(64); if (++spins > (1 << 22)) { stamps[7] = 1000000ull * c + 1000ull * qq + j; v = 0; break; } }
      cval[qq][j] = v;
    }
    __syncthreads();
    for (int j = c + tid; j < w; j += NT) { double a = 0; for (int qq = 0; qq < Q; ++qq) a += cval[qq][j]; gsum[j] = a; }
    __syncthreads();
    }
    t1 = gtime(); tr += t1 - t0; t0 = t1;
    const double nv = sqrt(gsum[c]), rnv = 1.0 / nv;
    if (cp == c) for (int r = 0; r < RPT; ++r) { x[r] *= rnv; qs[h * QP + r] = x[r]; }
    if (cp == c + 1) for (int r = 0; r < RPT; ++r) vs[h * QP + r] = x[r];
    __syncthreads();
    const bool act = mine && cp > c;
    double acc = 0;
    if (act) {
      const double coef = gsum[cp] * rnv, cn = (c + 1 < w) ? gsum[c + 1] * rnv : 0.0;
#pragma unroll
      for (int r = 0; r < RPT; ++r) { const double qr = qs[h * QP + r]; x[r] = fma(-qr, coef, x[r]); acc = fma(fma(-qr, cn, vs[h * QP + r]), x[r], acc); }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (act && h == 0 && c + 1 < w) mypart[buf ^ 1][cp] = acc;
    t1 = gtime(); tc += t1 - t0;
  }
  if (rec) { const int kk = g == 0 ? 0 : 3; stamps[kk] = tw; stamps[kk + 1] = tr; stamps[kk + 2] = tc; }
  cluster.sync();
  if (mine) for (int r = 0; r < RPT; ++r) if (rbase + r < rows) V[r0 + rbase + r + (size_t)cp * n] = x[r];
}

template <int CL, int POLL>
void run_ll(const char* name, int n, int w, double* V, int* flags, double* part, unsigned long long* st, bool coop) {
  int G = n / 128; if (G > 148) G = 148; int RB = (n + G - 1) / G;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = 0; cfg.stream = 0;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
  cfg.attrs = at; cfg.numAttrs = coop ? 2 : 1;
  int ncl = -1; cudaOccupancyMaxActiveClusters(&ncl, (void*)mgs_ll<CL, POLL>, &cfg);
  if (ncl < G / CL) { printf("%-22s n=%d: %d clusters > max %d, skipped\n", name, n, G / CL, ncl); return; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9; cudaError_t err = cudaSuccess;
  for (int it = 0; it < 6; ++it) {
    cudaMemset(part, 0, 1 << 22);
    cudaEventRecord(e0);
    err = cudaLaunchKernelEx(&cfg, mgs_ll<CL, POLL>, n, w, RB, V, flags, part, st);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    if (err != cudaSuccess) break;
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
  }
  unsigned long long hh[8]; cudaMemcpy(hh, st, sizeof hh, cudaMemcpyDeviceToHost);
  if (hh[7]) printf("poll timeout at c=%llu q=%llu j=%llu\n", hh[7] / 1000000, hh[7] / 1000 % 1000, hh[7] % 1000);
  printf("%-22s n=%d w=%d G=%d maxclusters=%d coop=%d: %.1f us/panel = %.2f us/col | cta0 clus %.2f poll %.2f comp %.2f | ctaL %.2f %.2f %.2f  %s/%s\n",
         name, n, w, G, ncl, (int)coop, best * 1e3, best * 1e3 / w, hh[0] / 1e3 / w, hh[1] / 1e3 / w, hh[2] / 1e3 / w, hh[3] / 1e3 / w, hh[4] / 1e3 / w, hh[5] / 1e3 / w,
         cudaGetErrorString(err), cudaGetErrorString(cudaGetLastError()));
}

template <int F, int S>
void run(const char* name, int n, int w, double* V, int* flags, double* part, unsigned long long* st) {
  int G = n / 128; if (G > 148) G = 148; int RB = (n + G - 1) / G;
  void* args[] = {&n, &w, &RB, &V, &flags, &part, &st};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    cudaMemset(flags, 0, 4096);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)mgs<F, S>, G, NT, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
  }
  unsigned long long h[6]; cudaMemcpy(h, st, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-22s n=%d w=%d G=%d: %.1f us/panel = %.2f us/col | cta0 wait %.2f red %.2f comp %.2f | ctaL wait %.2f red %.2f comp %.2f us/col  %s\n",
         name, n, w, G, best * 1e3, best * 1e3 / w, h[0] / 1e3 / w, h[1] / 1e3 / w, h[2] / 1e3 / w, h[3] / 1e3 / w, h[4] / 1e3 / w, h[5] / 1e3 / w,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int n = 8192, w = 128;
  double *V, *part; int* flags; unsigned long long* st;
  cudaMalloc(&V, sizeof(double) * 16384 * w); cudaMalloc(&part, 1 << 22); cudaMalloc(&flags, 4096); cudaMalloc(&st, 64); cudaMemset(st, 0, 64);
  std::vector<double> hv((size_t)16384 * w); for (auto& v : hv) v = rand() / (double)RAND_MAX - 0.5;
  cudaFuncSetAttribute(mgs_ll<16, 0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int nn : {8192, 16384, 4096}) {
    cudaMemcpy(V, hv.data(), sizeof(double) * nn * w, cudaMemcpyHostToDevice);
    run<1, 64>("rel sleep64", nn, w, V, flags, part, st);
    run<1, 0>("rel nosleep", nn, w, V, flags, part, st);
    run_ll<8, 0>("ll cl8", nn, w, V, flags, part, st, false);
    run_ll<8, 2>("ll cl8 warppoll", nn, w, V, flags, part, st, false);
    run_ll<8, 3>("ll cl8 sleep", nn, w, V, flags, part, st, false);
    run_ll<16, 0>("ll cl16", nn, w, V, flags, part, st, false);
    run_ll<4, 0>("ll cl4", nn, w, V, flags, part, st, false);
  }
  return 0;
}
