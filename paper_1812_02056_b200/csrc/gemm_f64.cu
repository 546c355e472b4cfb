// gemm_f64.cu — FP64 tensor-core (DMMA.8x8x4) GEMM / SYRK with the trailing-matrix
// subtraction fused into the epilogue.
//
// Serves every dense contraction of the three algorithms:
//   Cholesky flush   A[c:n,c:n] -= R R^T,      R = L[c:n, z:c)
//   LU flush         A[c:n,c:n] -= R_L R_U
//   QR flush         C = B_Q^T B_M ; M[:,c:n] -= B_Q C
//   QR R             R = Q^T A  (upper tiles only)
//   in-panel corrections of the recursive panel (same formulas, narrower N).
// The product S is never materialised: each 128x64 tile of C is read, decremented by the
// accumulator and written once (Cin may differ from C: out-of-place first step).  MASK
// restricts work to the lower (Cholesky) or upper (R) triangle of C.
//
// Design (DESIGN.md §5 K1/K2): 128x64 CTA tile, 128 threads = 4 warps as 2 (i) x 2 (j); warp
// tile 64x32 = 8x4 DMMA atoms (64 fp64 accumulators per lane); 3-stage cp.async pipeline of
// BK=16 operand slices (smem layouts padded so every fragment load is bank-conflict free);
// two CTAs per SM (92 KB smem each) so one CTA's epilogue overlaps the other's MMAs; the
// D fragment is used transposed (D = C^T).  Epilogue: the accumulator tile is parked in
// the (now idle) pipeline shared memory, then every warp streams whole 1 KB columns of C:
// all loads of a thread are issued before the first store, in 16-byte vectors, so the
// read-modify-write costs about one L2/HBM round trip per tile instead of one per atom.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "tiles.cuh"

namespace sf {

namespace g64 {
// CTA tile BM (i) x BN (j), 4 warps as 2 (i) x 2 (j), warp tile 64 x 32.  ~92 KB of shared
// memory and <= 255 registers per thread, so TWO CTAs share an SM: one CTA's prologue /
// epilogue overlaps the other's DMMA main loop (a single 1-CTA/SM kernel leaves the tensor
// pipe idle during every epilogue).
constexpr int BM = 128, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int PAD_KI = BK + 4;    // smem row stride (doubles) for k-contiguous slices (== 4 mod 16)
template <int NIDX> struct Slice {
  static constexpr int PAD_IK = NIDX + 4;   // row stride for idx-contiguous slices (== 4 mod 16)
  static constexpr int ELEMS = (BK * PAD_IK > NIDX * PAD_KI) ? BK * PAD_IK : NIDX * PAD_KI;
  template <int NT> static constexpr int chunks() { return NIDX * BK / 2 / NT; }   // 16-byte chunks per thread
};
constexpr int OPER_A = Slice<BM>::ELEMS, OPER_B = Slice<BN>::ELEMS;
constexpr int STAGE = OPER_A + OPER_B;
constexpr int CPAD = BM + 2;      // epilogue staging column stride
constexpr size_t SMEM_PIPE = sizeof(double) * (size_t)STAGE * STAGES;
constexpr size_t SMEM_EPI = sizeof(double) * (size_t)BN * CPAD;
constexpr size_t SMEM = SMEM_PIPE > SMEM_EPI ? SMEM_PIPE : SMEM_EPI;
static_assert(2 * SMEM <= 227 * 1024, "two CTAs per SM");
}  // namespace g64

// Load an NIDX (idx) x BK (k) slice of op(X) into shared memory.
//  KC=false: op(X)(idx,k) = X[idx + k*ld]  (idx contiguous)  -> Xs[k*PAD_IK + idx]
//  KC=true : op(X)(idx,k) = X[k + idx*ld]  (k contiguous)    -> Xs[idx*PAD_KI + k]
template <int NIDX, bool KC, bool V16, int NT = g64::THREADS>
__device__ __forceinline__ void load_slice(double* Xs, const double* __restrict__ X, int64_t ld,
                                           int64_t idx0, int64_t nidx, int64_t k0, int64_t K, int tid) {
  using namespace g64;
  using S = Slice<NIDX>;
#pragma unroll
  for (int r = 0; r < S::template chunks<NT>(); ++r) {
    const int id = tid + r * NT;
    int64_t idx, kg;
    double* dst;
    if (!KC) {
      const int kk = id / (NIDX / 2), ch = id % (NIDX / 2);
      idx = idx0 + 2 * ch; kg = k0 + kk;
      dst = Xs + kk * S::PAD_IK + 2 * ch;
      const bool kin = kg < K;
      if (V16) {
        const int bytes = (!kin || idx >= nidx) ? 0 : (idx + 1 >= nidx ? 8 : 16);
        cp_async16(dst, bytes ? X + idx + kg * ld : X, bytes);
      } else {
        const int b0 = (kin && idx < nidx) ? 8 : 0, b1 = (kin && idx + 1 < nidx) ? 8 : 0;
        dst[0] = b0 ? __ldcg(X + idx + kg * ld) : 0.0;       // unaligned operand: L2-only loads
        dst[1] = b1 ? __ldcg(X + idx + 1 + kg * ld) : 0.0;
      }
    } else {
      const int ii = id / (BK / 2), ch = id % (BK / 2);
      idx = idx0 + ii; kg = k0 + 2 * ch;
      dst = Xs + ii * PAD_KI + 2 * ch;
      const bool iin = idx < nidx;
      if (V16) {
        const int bytes = (!iin || kg >= K) ? 0 : (kg + 1 >= K ? 8 : 16);
        cp_async16(dst, bytes ? X + kg + idx * ld : X, bytes);
      } else {
        const int b0 = (iin && kg < K) ? 8 : 0, b1 = (iin && kg + 1 < K) ? 8 : 0;
        dst[0] = b0 ? __ldcg(X + kg + idx * ld) : 0.0;
        dst[1] = b1 ? __ldcg(X + kg + 1 + idx * ld) : 0.0;
      }
    }
  }
}

// The same slice for a tile that lies wholly inside the operand and the K range (no zero
// fill): `g` is this thread's first 16-byte chunk in global memory, `xs` its place in the
// slot; the thread's other chunks sit at compile-time row steps from both.  A handful of
// integer instructions per stage instead of the generic path's per-chunk index / bound /
// address arithmetic, which each warp otherwise executes between its DMMA groups.
template <int NIDX, bool KC, int NT>
constexpr bool slice_full_ok() { return KC ? NT % (g64::BK / 2) == 0 : NT % (NIDX / 2) == 0; }
template <int NIDX, bool KC, int NT>
__device__ __forceinline__ void load_slice_full(double* xs, const double* __restrict__ g, int64_t ld) {
  using namespace g64;
  using S = Slice<NIDX>;
  constexpr int RS = KC ? NT / (BK / 2) : NT / (NIDX / 2);   // rows (idx | k) between a thread's chunks
  static_assert(slice_full_ok<NIDX, KC, NT>(), "chunk rows");
  const unsigned sb = (unsigned)__cvta_generic_to_shared(xs);
#pragma unroll
  for (int r = 0; r < S::template chunks<NT>(); ++r) {
    const unsigned d = sb + (unsigned)(r * RS * (KC ? PAD_KI : S::PAD_IK) * sizeof(double));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g + (int64_t)(r * RS) * ld));
  }
}
// this thread's first chunk of the slice at (idx0, k0): offset in the operand / in the slot
template <int NIDX, bool KC, int NT>
__device__ __forceinline__ int64_t slice_goff(int64_t ld, int64_t idx0, int64_t k0, int tid) {
  using namespace g64;
  if (!KC) return idx0 + 2 * (tid % (NIDX / 2)) + (k0 + tid / (NIDX / 2)) * ld;
  return k0 + 2 * (tid % (BK / 2)) + (idx0 + tid / (BK / 2)) * ld;
}
template <int NIDX, bool KC, int NT>
__device__ __forceinline__ int slice_soff(int tid) {
  using namespace g64;
  if (!KC) return (tid / (NIDX / 2)) * Slice<NIDX>::PAD_IK + 2 * (tid % (NIDX / 2));
  return (tid / (BK / 2)) * PAD_KI + 2 * (tid % (BK / 2));
}

template <int NIDX, bool KC>
__device__ __forceinline__ double frag(const double* Xs, int base, int kk, int lane) {
  using namespace g64;
  if (!KC) return Xs[(kk * 4 + (lane & 3)) * Slice<NIDX>::PAD_IK + base + (lane >> 2)];
  return Xs[(base + (lane >> 2)) * PAD_KI + kk * 4 + (lane & 3)];
}

using T64 = Tiles<g64::BM, g64::BN>;
// rasterization: tile columns in groups of 32 (2048 C columns); see Tiles::tile_of_grouped
constexpr int kGroupCols = 32;
__host__ __device__ __forceinline__ int first_lower(int tj, int64_t off = 0) { return T64::first_lower(tj, off); }
__host__ __device__ __forceinline__ int masked_tiles(int mask, int TM, int TN, int64_t off) {
  return T64::count(mask, TM, TN, off);
}

// bulk-async reduction of a shared-memory column segment into global memory (in-place epilogues)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_reduce_add_f64(double* gdst, const double* ssrc, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(gdst), "r"(s),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

template <bool AK, bool BKC, bool V16, int MASK, int NT = g64::THREADS>
__device__ __forceinline__ void gemm_f64_body(const GemmF64& p, int bid, int vecC, int bulk = 0) {
  using namespace g64;
  // NT = 128: 4 warps as 2 (i) x 2 (j), warp tile 64 x 32; NT = 256 (short K): 8 warps as
  // 4 x 2, warp tile 32 x 32 — twice the issuing warps per SM sub-partition
  constexpr int NWARP = NT / 32, WARPS_M = NWARP / 2, WTM = BM / WARPS_M, ATM = WTM / 8;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                       // [STAGES][OPER_A]
  double* Bs = smem + STAGES * OPER_A;     // [STAGES][OPER_B]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + BN - 1) / BN);
  int ti, tj;
  if (p.rs.ngroups > 0) T64::tile_of_raster(MASK, bid, TM, p.off, p.rs, ti, tj);
  else T64::tile_of(MASK, bid, TM, TN, p.off, ti, tj);
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * BN;

  // K range of this split
  const int sp = blockIdx.y;
  int64_t kchunk = (p.K + p.splits - 1) / p.splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int64_t kbeg = (int64_t)sp * kchunk;
  const int64_t kend = (kbeg + kchunk < p.K) ? kbeg + kchunk : p.K;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  // Warm L2 with the C tile we will read-modify-write in the epilogue.
  if (p.beta && p.splits == 1) {
#pragma unroll
    for (int r = 0; r < BN * 8 / NT; ++r) {
      const int id = tid + r * NT;           // BN columns x 8 lines of 128 B
      const int64_t jj = j0 + (id >> 3), ii = i0 + (id & 7) * 16;
      if (jj < p.N && ii < p.M) prefetch_l2(p.Cin + ii + jj * p.ldcin);
    }
  }

  double acc[ATM][4][2];
#pragma unroll
  for (int a = 0; a < ATM; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // interior tiles: running per-thread source pointers (load_slice_full)
  // (not for the lower-masked instantiation: it only serves SYRK flushes with K <= 64, where
  // the pointer set-up cost more than it saved: m = 16384, K = 64 0.783 -> 0.842 ms)
  constexpr bool FULL_OK = slice_full_ok<BM, AK, NT>() && slice_full_ok<BN, BKC, NT>() && MASK != kMaskLower;
  const bool full = FULL_OK && V16 && i0 + BM <= p.M && j0 + BN <= p.N;
  const double* ga = p.A + slice_goff<BM, AK, NT>(p.lda, i0, kbeg, tid);
  const double* gb = p.B + slice_goff<BN, BKC, NT>(p.ldb, j0, kbeg, tid);
  const int soa = slice_soff<BM, AK, NT>(tid), sob = slice_soff<BN, BKC, NT>(tid);
  auto issue = [&](int kb) {
    if (kb < nk) {
      const int slot = kb % STAGES;
      const int64_t k0 = kbeg + (int64_t)kb * BK;
      if (full && k0 + BK <= kend) {
        if constexpr (FULL_OK) {
          load_slice_full<BM, AK, NT>(As + slot * OPER_A + soa, ga, p.lda);
          load_slice_full<BN, BKC, NT>(Bs + slot * OPER_B + sob, gb, p.ldb);
        }
      } else {
        load_slice<BM, AK, V16, NT>(As + slot * OPER_A, p.A, p.lda, i0, p.M, k0, kend, tid);
        load_slice<BN, BKC, V16, NT>(Bs + slot * OPER_B, p.B, p.ldb, j0, p.N, k0, kend, tid);
      }
      ga += AK ? (int64_t)BK : (int64_t)BK * p.lda;    // issue() runs for kb = 0, 1, 2, ... in order
      gb += BKC ? (int64_t)BK : (int64_t)BK * p.ldb;
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);

  for (int kb = 0; kb < nk; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue(kb + STAGES - 1);
    const double* as = As + (kb % STAGES) * OPER_A;
    const double* bs = Bs + (kb % STAGES) * OPER_B;
    double fa[2][ATM], fb[2][4];
#pragma unroll
    for (int a = 0; a < ATM; ++a) fa[0][a] = frag<BM, AK>(as, wm * WTM + a * 8, 0, lane);
#pragma unroll
    for (int b = 0; b < 4; ++b) fb[0][b] = frag<BN, BKC>(bs, wn * 32 + b * 8, 0, lane);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int cur = kk & 1, nxt = cur ^ 1;
      if (kk + 1 < BK / 4) {
#pragma unroll
        for (int a = 0; a < ATM; ++a) fa[nxt][a] = frag<BM, AK>(as, wm * WTM + a * 8, kk + 1, lane);
#pragma unroll
        for (int b = 0; b < 4; ++b) fb[nxt][b] = frag<BN, BKC>(bs, wn * 32 + b * 8, kk + 1, lane);
      }
#pragma unroll
      for (int a = 0; a < ATM; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          // D = C^T: the MMA's A operand is op(B) (rows j), its B operand is op(A) (cols i)
          dmma_8x8x4(acc[a][b][0], acc[a][b][1], fb[cur][b], fa[cur][a]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- epilogue, step 1: park the accumulator tile in shared memory, Cs[j*CPAD + i]
  double* Cs = smem;
  const int64_t rows = (p.M - i0 < BM) ? p.M - i0 : BM;
  // in place (Cin == C): add alpha*acc to C in L2 by one bulk reduction per column (as the
  // v2 tile), -0.0 where the mask excludes an entry (x + -0.0 == x: bit-identical)
  const bool use_bulk = bulk && p.splits == 1 && (rows & 1) == 0;
#pragma unroll
  for (int a = 0; a < ATM; ++a) {
    const int il = wm * WTM + a * 8 + 2 * (lane & 3);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jl = wn * 32 + b * 8 + (lane >> 2);
      double v0 = acc[a][b][0], v1 = acc[a][b][1];
      if (use_bulk) {
        const int64_t i = i0 + il, jd = j0 + jl + p.off;
        const bool in0 = MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i <= jd);
        const bool in1 = MASK == kMaskNone || (MASK == kMaskLower ? i + 1 >= jd : i + 1 <= jd);
        v0 = in0 ? p.alpha * v0 : -0.0;
        v1 = in1 ? p.alpha * v1 : -0.0;
      }
      *reinterpret_cast<double2*>(Cs + jl * CPAD + il) = make_double2(v0, v1);
    }
  }
  if (use_bulk) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid < BN) {
      const int64_t j = j0 + tid;
      if (j < p.N) bulk_reduce_add_f64(p.C + i0 + j * p.ldc, Cs + tid * CPAD, (int)(rows * 8));
      bulk_commit();
      bulk_wait_read0();
    }
    return;
  }
  __syncthreads();

  // ---- step 2: each warp streams BN/4 whole columns; lane owns rows 2*lane+{0,1} and
  //      64+2*lane+{0,1} (each warp instruction covers 512 contiguous bytes of a column)
  constexpr int COLS = BN / NWARP;
  if (p.splits > 1) {
    double* W = p.work + (int64_t)sp * p.M * p.N;
    for (int q = 0; q < COLS; ++q) {
      const int jl = warp * COLS + q;
      const int64_t j = j0 + jl;
      if (j >= p.N) break;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int il = 64 * h + 2 * lane + e;
          if (i0 + il < p.M) W[j * p.M + i0 + il] = Cs[jl * CPAD + il];
        }
    }
    return;
  }
  double cin[COLS][2][2];
  if (p.beta) {
#pragma unroll
    for (int q = 0; q < COLS; ++q) {
      const int64_t j = j0 + warp * COLS + q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = i0 + 64 * h + 2 * lane;
        const double* src = p.Cin + i + j * p.ldcin;
        if (vecC && j < p.N && i + 1 < p.M) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(src));
          cin[q][h][0] = v.x; cin[q][h][1] = v.y;
        } else {
          cin[q][h][0] = (j < p.N && i < p.M) ? __ldcg(src) : 0.0;
          cin[q][h][1] = (j < p.N && i + 1 < p.M) ? __ldcg(src + 1) : 0.0;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < COLS; ++q) {
    const int jl = warp * COLS + q;
    const int64_t j = j0 + jl;
    if (j >= p.N) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int il = 64 * h + 2 * lane;
      const int64_t i = i0 + il;
      const double2 d = *reinterpret_cast<const double2*>(Cs + jl * CPAD + il);
      double v0 = p.alpha * d.x, v1 = p.alpha * d.y;
      if (p.beta) { v0 += cin[q][h][0]; v1 += cin[q][h][1]; }
      double* dst = p.C + i + j * p.ldc;
      const int64_t jd = j + p.off;   // diagonal position of column j
      const bool pair_in = (i + 1 < p.M) && (MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i + 1 <= jd));
      if (pair_in && vecC) {
        __stcg(reinterpret_cast<double2*>(dst), make_double2(v0, v1));
      } else {
        if (i < p.M && (MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i <= jd))) dst[0] = v0;
        if (i + 1 < p.M && (MASK == kMaskNone || (MASK == kMaskLower ? i + 1 >= jd : i + 1 <= jd))) dst[1] = v1;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// v2 tile (DESIGN.md §5 K1): BM x 64 CTA tile, 4 warps as 2 x 2 (warp tile BM/2 x 32),
// MINB CTAs per SM.  Differences from gemm_f64_body:
//  * paired fragment loads: for an idx-contiguous operand the two atoms 2b, 2b+1 of a warp
//    tile interleave their rows (atom 2b row r = logical row 16b + 2r, atom 2b+1 = 16b+2r+1),
//    so ONE 16-byte shared load feeds both DMMA operands — half the LDS instructions per DMMA;
//  * BM = 96 with 3 CTAs per SM (12 warps, 3 per SM sub-partition): while one CTA is in its
//    prologue / epilogue the other two still keep two warps per sub-partition issuing DMMA;
//  * in-place epilogue by bulk reduction: the tile (alpha * acc, -0.0 where masked) is
//    parked in shared memory and added to C in L2 by `cp.reduce.async.bulk .add.f64`, one
//    column per lane — no C load on the CTA's critical path.  fl(C + alpha*acc) is the same
//    IEEE operation as the load/add/store epilogue; x + (-0.0) == x for every x, so masked
//    entries are unchanged bit for bit.
namespace g64v2 {
using g64::BK;
using g64::PAD_KI;
template <int NIDX, bool KC> constexpr int slice_elems() { return KC ? NIDX * PAD_KI : BK * (NIDX + 4); }
template <int BM, bool AK, bool BKC> constexpr int stage_elems() { return slice_elems<BM, AK>() + slice_elems<64, BKC>(); }
template <int BM, bool AK, bool BKC> constexpr size_t smem_bytes() {
  const size_t pipe = sizeof(double) * (size_t)stage_elems<BM, AK, BKC>() * g64::STAGES;
  const size_t epi = sizeof(double) * (size_t)64 * (BM + 2);
  return pipe > epi ? pipe : epi;
}
}  // namespace g64v2


template <int BM, bool PAIR, bool AK, bool BKC, bool V16, int MASK>
__device__ __forceinline__ void gemm_f64_body2(const GemmF64& p, int bid, int vecC, int bulk) {
  using namespace g64;
  constexpr int NT = 128, WTM = BM / 2, ATM = WTM / 8;
  static_assert(ATM % 2 == 0, "paired atoms");
  constexpr bool PA_ = PAIR && !AK, PB_ = PAIR && !BKC;   // paired fragment loads per operand
  constexpr int SA = g64v2::slice_elems<BM, AK>(), SB = g64v2::slice_elems<64, BKC>();
  constexpr int PA = BM + 4, PB = 64 + 4;   // idx-contiguous row strides (== 4 mod 16 doubles)
  constexpr int CP = BM + 2;
  using TT = Tiles<BM, 64>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * SA;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + 63) / 64);
  int ti, tj;
  if (p.rs.ngroups > 0) TT::tile_of_raster(MASK, bid, TM, p.off, p.rs, ti, tj);
  else TT::tile_of(MASK, bid, TM, TN, p.off, ti, tj);
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * 64;

  const int sp = blockIdx.y;
  int64_t kchunk = (p.K + p.splits - 1) / p.splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int64_t kbeg = (int64_t)sp * kchunk;
  const int64_t kend = (kbeg + kchunk < p.K) ? kbeg + kchunk : p.K;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  if (p.beta && p.splits == 1) {
#pragma unroll
    for (int r = 0; r < 64 * 8 / NT; ++r) {
      const int id = tid + r * NT;
      const int64_t jj = j0 + (id >> 3), ii = i0 + (id & 7) * 16;
      if (jj < p.N && ii < p.M) prefetch_l2(p.Cin + ii + jj * p.ldcin);
    }
  }

  double acc[ATM][4][2];
#pragma unroll
  for (int a = 0; a < ATM; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // interior tiles (all of the big flushes but their last tile row / column): running
  // per-thread source pointers, see load_slice_full
  constexpr bool FULL_OK = slice_full_ok<BM, AK, NT>() && slice_full_ok<64, BKC, NT>();
  const bool full = FULL_OK && V16 && i0 + BM <= p.M && j0 + 64 <= p.N;
  const double* ga = p.A + slice_goff<BM, AK, NT>(p.lda, i0, kbeg, tid);
  const double* gb = p.B + slice_goff<64, BKC, NT>(p.ldb, j0, kbeg, tid);
  const int soa = slice_soff<BM, AK, NT>(tid), sob = slice_soff<64, BKC, NT>(tid);
  auto issue = [&](int kb) {
    if (kb < nk) {
      const int slot = kb % STAGES;
      const int64_t k0 = kbeg + (int64_t)kb * BK;
      if (full && k0 + BK <= kend) {
        if constexpr (FULL_OK) {
          load_slice_full<BM, AK, NT>(As + slot * SA + soa, ga, p.lda);
          load_slice_full<64, BKC, NT>(Bs + slot * SB + sob, gb, p.ldb);
        }
      } else {
        load_slice<BM, AK, V16, NT>(As + slot * SA, p.A, p.lda, i0, p.M, k0, kend, tid);
        load_slice<64, BKC, V16, NT>(Bs + slot * SB, p.B, p.ldb, j0, p.N, k0, kend, tid);
      }
      ga += AK ? (int64_t)BK : (int64_t)BK * p.lda;    // issue() runs for kb = 0, 1, 2, ... in order
      gb += BKC ? (int64_t)BK : (int64_t)BK * p.ldb;
    }
    cp_async_commit();
  };
  // fragments of step kk: A atoms (i), B atoms (j)
  auto load_frags = [&](const double* as, const double* bs, int kk, double (&fa)[ATM], double (&fb)[4]) {
    if (PA_) {
#pragma unroll
      for (int b2 = 0; b2 < ATM / 2; ++b2) {
        const double2 v = *reinterpret_cast<const double2*>(as + (kk * 4 + (lane & 3)) * PA + wm * WTM + 16 * b2 +
                                                            2 * (lane >> 2));
        fa[2 * b2] = v.x; fa[2 * b2 + 1] = v.y;
      }
    } else if (AK) {
#pragma unroll
      for (int a = 0; a < ATM; ++a) fa[a] = as[(wm * WTM + a * 8 + (lane >> 2)) * PAD_KI + kk * 4 + (lane & 3)];
    } else {
#pragma unroll
      for (int a = 0; a < ATM; ++a) fa[a] = as[(kk * 4 + (lane & 3)) * PA + wm * WTM + a * 8 + (lane >> 2)];
    }
    if (PB_) {
#pragma unroll
      for (int b2 = 0; b2 < 2; ++b2) {
        const double2 v = *reinterpret_cast<const double2*>(bs + (kk * 4 + (lane & 3)) * PB + wn * 32 + 16 * b2 +
                                                            2 * (lane >> 2));
        fb[2 * b2] = v.x; fb[2 * b2 + 1] = v.y;
      }
    } else if (BKC) {
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = bs[(wn * 32 + b * 8 + (lane >> 2)) * PAD_KI + kk * 4 + (lane & 3)];
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = bs[(kk * 4 + (lane & 3)) * PB + wn * 32 + b * 8 + (lane >> 2)];
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);

  for (int kb = 0; kb < nk; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue(kb + STAGES - 1);
    const double* as = As + (kb % STAGES) * SA;
    const double* bs = Bs + (kb % STAGES) * SB;
    double fa[2][ATM], fb[2][4];
    load_frags(as, bs, 0, fa[0], fb[0]);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int cur = kk & 1, nxt = cur ^ 1;
      if (kk + 1 < BK / 4) load_frags(as, bs, kk + 1, fa[nxt], fb[nxt]);
#pragma unroll
      for (int a = 0; a < ATM; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], fb[cur][b], fa[cur][a]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- park the tile in shared memory, Cs[j*CP + i] (logical tile coordinates)
  double* Cs = smem;
  const int64_t rows = (p.M - i0 < BM) ? p.M - i0 : BM;
  const bool use_bulk = bulk && p.splits == 1 && (rows & 1) == 0;
  const double alpha = p.alpha;
  const bool neg = alpha == -1.0;
  // logical i of atom a, MMA column c (0..7); logical j of atom b, MMA row r
  auto li = [&](int a, int c) { return !PA_ ? wm * WTM + 8 * a + c : wm * WTM + 16 * (a >> 1) + 2 * c + (a & 1); };
  auto lj = [&](int b, int r) { return !PB_ ? wn * 32 + 8 * b + r : wn * 32 + 16 * (b >> 1) + 2 * r + (b & 1); };
#pragma unroll
  for (int a = 0; a < ATM; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jl = lj(b, lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int il = li(a, 2 * (lane & 3) + e);
        double v = acc[a][b][e];
        if (use_bulk) {
          const int64_t i = i0 + il, jd = j0 + jl + p.off;
          const bool in = MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i <= jd);
          // alpha = -1 (every flush): a sign flip on the integer pipe, not a DMUL on the FP64
          // pipe the co-resident CTAs' DMMAs are using (bit-identical to alpha * v)
          v = in ? (neg ? __longlong_as_double(__double_as_longlong(v) ^ (long long)0x8000000000000000ULL) : alpha * v)
                 : -0.0;
        }
        Cs[jl * CP + il] = v;
      }
    }
  if (use_bulk) {
    fence_proxy_async_smem();
    __syncthreads();
    // one 16-byte-multiple column segment per lane: rows [i0, i0+rows) of column j
    if (tid < 64) {
      const int64_t j = j0 + tid;
      if (j < p.N) bulk_reduce_add_f64(p.C + i0 + j * p.ldc, Cs + tid * CP, (int)(rows * 8));
      bulk_commit();
      bulk_wait_read0();
    }
    return;
  }
  __syncthreads();

  constexpr int COLS = 64 / 4;
  if (p.splits > 1) {
    double* W = p.work + (int64_t)sp * p.M * p.N;
    for (int q = 0; q < COLS; ++q) {
      const int jl = warp * COLS + q;
      const int64_t j = j0 + jl;
      if (j >= p.N) break;
      for (int il = lane; il < BM; il += 32)
        if (i0 + il < p.M) W[j * p.M + i0 + il] = Cs[jl * CP + il];
    }
    return;
  }
  // load/add/store epilogue: lane owns rows 2*lane+{0,1} (+64 for BM = 128) of each column
  constexpr int H = (BM + 63) / 64;
  double cin[COLS][H][2];
  if (p.beta) {
#pragma unroll
    for (int q = 0; q < COLS; ++q) {
      const int64_t j = j0 + warp * COLS + q;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int il = 64 * h + 2 * lane;
        const int64_t i = i0 + il;
        const double* src = p.Cin + i + j * p.ldcin;
        if (il < BM && vecC && j < p.N && i + 1 < p.M) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(src));
          cin[q][h][0] = v.x; cin[q][h][1] = v.y;
        } else {
          cin[q][h][0] = (il < BM && j < p.N && i < p.M) ? __ldcg(src) : 0.0;
          cin[q][h][1] = (il < BM && j < p.N && i + 1 < p.M) ? __ldcg(src + 1) : 0.0;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < COLS; ++q) {
    const int jl = warp * COLS + q;
    const int64_t j = j0 + jl;
    if (j >= p.N) break;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int il = 64 * h + 2 * lane;
      if (il >= BM) continue;
      const int64_t i = i0 + il;
      const double2 d = *reinterpret_cast<const double2*>(Cs + jl * CP + il);
      double v0 = alpha * d.x, v1 = alpha * d.y;
      if (p.beta) { v0 += cin[q][h][0]; v1 += cin[q][h][1]; }
      double* dst = p.C + i + j * p.ldc;
      const int64_t jd = j + p.off;
      const bool pair_in = (i + 1 < p.M) && (MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i + 1 <= jd));
      if (pair_in && vecC) {
        __stcg(reinterpret_cast<double2*>(dst), make_double2(v0, v1));
      } else {
        if (i < p.M && (MASK == kMaskNone || (MASK == kMaskLower ? i >= jd : i <= jd))) dst[0] = v0;
        if (i + 1 < p.M && (MASK == kMaskNone || (MASK == kMaskLower ? i + 1 >= jd : i + 1 <= jd))) dst[1] = v1;
      }
    }
  }
}

template <int BM, int MINB, bool PAIR, bool AK, bool BKC, bool V16, int MASK>
__global__ void __launch_bounds__(128, MINB) gemm_f64v2_kernel(GemmF64 p, int vecC, int bulk) {
  if (p.fail && failed(p.fail)) return;
  gemm_f64_body2<BM, PAIR, AK, BKC, V16, MASK>(p, blockIdx.x, vecC, bulk);
}

template <bool AK, bool BKC, bool V16, int MASK, int NT = g64::THREADS>
__global__ void __launch_bounds__(NT, 2) gemm_f64_kernel(GemmF64 p, int vecC, int bulk) {
  if (p.fail && failed(p.fail)) return;
  gemm_f64_body<AK, BKC, V16, MASK, NT>(p, blockIdx.x, vecC, bulk);
}

// Bounded grid (max_ctas > 0): each CTA loops over tiles, leaving SMs to a concurrent stream.
template <bool AK, bool BKC, bool V16, int MASK>
__global__ void __launch_bounds__(g64::THREADS, 2) gemm_f64_loop_kernel(GemmF64 p, int vecC) {
  if (p.fail && failed(p.fail)) return;
#pragma unroll 1
  for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    gemm_f64_body<AK, BKC, V16, MASK>(p, t, vecC);
    __syncthreads();   // shared memory is reused by the next tile
  }
}

// Grouped launch: several independent C blocks sharing K, the operand leading dimensions
// and the mask, one CTA grid (the block-cyclic distributed updates).
template <bool AK, bool BKC, bool V16, int MASK, int NT = g64::THREADS>
__global__ void __launch_bounds__(NT, 2) gemm_f64_grouped_kernel(GemmF64 p, GemmGroups gs, int vecC, int bulk) {
  if (p.fail && failed(p.fail)) return;
  int g = 0;
  while (g + 1 < gs.count && (int)blockIdx.x >= gs.g[g + 1].tile0) ++g;
  p.M = gs.g[g].M; p.N = gs.g[g].N; p.off = gs.g[g].off; p.rs.ngroups = 0;
  p.A = gs.g[g].A; p.B = gs.g[g].B; p.Cin = gs.g[g].Cin; p.C = gs.g[g].C;
  gemm_f64_body<AK, BKC, V16, MASK, NT>(p, (int)blockIdx.x - gs.g[g].tile0, vecC, bulk);
}

// Fixed-order split-K reduction: C = (beta ? Cin : 0) + alpha * sum_sp work[sp].
__global__ void splitk_reduce_f64(GemmF64 p) {
  if (p.fail && failed(p.fail)) return;
  const int64_t total = p.M * p.N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % p.M, j = t / p.M;
    double s = 0.0;
    for (int sp = 0; sp < p.splits; ++sp) s += p.work[(int64_t)sp * total + t];
    const double v = p.alpha * s;
    p.C[i + j * p.ldc] = p.beta ? p.Cin[i + j * p.ldcin] + v : v;
  }
}

static cudaError_t splitk_reduce(const GemmF64& p, cudaStream_t st) {
  const int64_t total = p.M * p.N;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  splitk_reduce_f64<<<blocks, 256, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// K1s — chunked short-K flush (K <= 64, in place, no mask; DESIGN.md §5 K1s).  The LU flush
// at s = 64 (A[c:n,c:n] -= R_L R_U with K = s) is 1 MFLOP per 128x64 tile:
// with one tile per CTA the operand fill and the epilogue are as long as the 2048 DMMAs.
// Here a CTA owns a CHUNK of consecutive tiles of one row block: the 128 x K block of R_L is
// loaded ONCE (bulk copies, mbarrier-tracked), the K x 64 blocks of R_U stream through a
// double buffer, and the result of tile t is added to C in L2 by bulk reductions issued by a
// producer warp while the 8 consumer warps already run the DMMAs of tile t+1.  No CTA-wide
// barrier in the main loop: consumers and producer meet only on mbarriers.
//   warps 0-7 : consumers, 4 (i) x 2 (j), warp tile 32 x 32 (4 x 4 DMMA atoms)
//   warp 8    : producer (operand bulk copies, C bulk reductions)
// Every element gets the same DMMA chain as gemm_f64_kernel (k in ascending groups of 4,
// accumulator from 0, then C + (-acc) by the bulk reduction): bitwise the same result.
namespace g64s {
constexpr int BM = 128, BN = 64, KMAX = 64, NCW = 8, NT = (NCW + 1) * 32;
constexpr int PA = BM + 4;     // As[k*PA + i]   (idx-contiguous rows, == 4 mod 16 doubles)
constexpr int PB = KMAX + 4;   // Bs[j*PB + k]   (k-contiguous rows)
constexpr int CP = BM + 2;     // Cs[j*CP + i]   (staging for the column bulk reductions)
constexpr size_t A_BYTES = sizeof(double) * KMAX * PA;
constexpr size_t B_BYTES = sizeof(double) * BN * PB;
constexpr size_t C_BYTES = sizeof(double) * BN * CP;
constexpr size_t SMEM = A_BYTES + 2 * B_BYTES + C_BYTES + 64;
static_assert(SMEM <= 227 * 1024, "one CTA per SM");

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
}  // namespace g64s

// C[i0:i0+rows, j] += alpha * sum_k A[i, k] B[k, j]   (A idx-contiguous, B k-contiguous)
__global__ void __launch_bounds__(g64s::NT, 1) gemm_f64_chunk_kernel(GemmF64 p, int TN, int chunk, int cpr) {
  using namespace g64s;
  extern __shared__ __align__(128) unsigned char g64s_raw[];
  double* As = reinterpret_cast<double*>(g64s_raw);
  double* Bs = reinterpret_cast<double*>(g64s_raw + A_BYTES);   // [2][BN * PB]
  double* Cs = reinterpret_cast<double*>(g64s_raw + A_BYTES + 2 * B_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(g64s_raw + A_BYTES + 2 * B_BYTES + C_BYTES);
  uint64_t* full = bars;        // [2] operands of the tile in B buffer b have landed
  uint64_t* empty = bars + 2;   // [2] the consumers are done reading B buffer b
  uint64_t* parked = bars + 4;  // the tile's result is in Cs
  uint64_t* stgfree = bars + 5; // the bulk reductions have read Cs
  __shared__ int skip;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    skip = (p.fail && failed(p.fail)) ? 1 : 0;   // one CTA-uniform decision
    mb_init(&full[0], 1); mb_init(&full[1], 1);
    mb_init(&empty[0], NCW); mb_init(&empty[1], NCW);
    mb_init(parked, NCW); mb_init(stgfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (skip) return;
  const int ti = (int)blockIdx.x / cpr, tj0 = ((int)blockIdx.x % cpr) * chunk;
  const int T = (TN - tj0 < chunk) ? TN - tj0 : chunk;
  const int64_t i0 = (int64_t)ti * BM;
  const int rows = (p.M - i0 < BM) ? (int)(p.M - i0) : BM;   // even (launcher: M even)
  const int K = (int)p.K;                                       // multiple of 4, <= KMAX
  auto cols_of = [&](int t) {
    const int64_t j0 = (int64_t)(tj0 + t) * BN;
    return (p.N - j0 < BN) ? (int)(p.N - j0) : BN;
  };

  if (warp == NCW) {   // ---------------- producer
    // tile t's R_U block into B buffer t & 1 (tile 0: together with the R_L block)
    auto load = [&](int t) {
      const int b = t & 1, cols = cols_of(t);
      const int64_t j0 = (int64_t)(tj0 + t) * BN;
      const uint32_t abytes = t == 0 ? (uint32_t)(K * rows * 8) : 0u;
      if (lane == 0) mb_expect_tx(&full[b], abytes + (uint32_t)(cols * K * 8));
      __syncwarp();
      if (t == 0)
        for (int k = lane; k < K; k += 32) bulk_g2s(As + k * PA, p.A + i0 + (int64_t)k * p.lda, rows * 8, &full[0]);
      for (int j = lane; j < cols; j += 32) bulk_g2s(Bs + b * (BN * PB) + j * PB, p.B + (j0 + j) * p.ldb, K * 8, &full[b]);
    };
    load(0);
    if (T > 1) load(1);
    for (int t = 0; t < T; ++t) {
      if (t + 2 < T) {
        mb_wait(&empty[t & 1], (t >> 1) & 1);
        load(t + 2);
      }
      mb_wait(parked, t & 1);
      const int cols = cols_of(t);
      const int64_t j0 = (int64_t)(tj0 + t) * BN;
      for (int j = lane; j < cols; j += 32) bulk_reduce_add_f64(p.C + i0 + (j0 + j) * p.ldc, Cs + j * CP, rows * 8);
      bulk_commit();
      bulk_wait_read0();
      __syncwarp();
      if (lane == 0) mb_arrive(stgfree);
    }
    bulk_wait_all();
    return;
  }
  // ---------------- consumers
  const int wm = warp & 3, wn = warp >> 2, q = lane & 3, r = lane >> 2;
  const int nk = K / 4;
  const double alpha = p.alpha;
  const bool neg = alpha == -1.0;
  for (int t = 0; t < T; ++t) {
    const int b = t & 1;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    mb_wait(&full[b], (t >> 1) & 1);
    const double* bs = Bs + b * (BN * PB) + (wn * 32 + r) * PB + q;
    const double* as = As + q * PA + wm * 32 + 2 * r;
#pragma unroll
    for (int kk = 0; kk < KMAX / 4; ++kk) {
      if (kk >= nk) break;
      double fa[4], fb[4];
#pragma unroll
      for (int b2 = 0; b2 < 2; ++b2) {
        // paired atoms: atom 2b2 row r = logical row 16 b2 + 2r, atom 2b2+1 = 16 b2 + 2r + 1
        const double2 v = *reinterpret_cast<const double2*>(as + kk * 4 * PA + 16 * b2);
        fa[2 * b2] = v.x; fa[2 * b2 + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) fb[c] = bs[c * 8 * PB + kk * 4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma_8x8x4(acc[a][c][0], acc[a][c][1], fb[c], fa[a]);
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[b]);
    if (t > 0) mb_wait(stgfree, (t - 1) & 1);
    // park alpha * acc (D = C^T: MMA row = j, MMA column = i); alpha = -1 is a sign flip
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int jl = wn * 32 + 8 * c + r;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int il = wm * 32 + 16 * (a >> 1) + 2 * (2 * q + e) + (a & 1);
          const double v = acc[a][c][e];
          Cs[jl * CP + il] =
              neg ? __longlong_as_double(__double_as_longlong(v) ^ (long long)0x8000000000000000ULL) : alpha * v;
        }
      }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mb_arrive(parked);
  }
}

// SF_DMMA_CHUNK=0 disables K1s; SF_DMMA_CHUNK_MIN = fewest tiles for which it is used;
// SF_DMMA_CHUNK_T = fixed chunk length (tiles per CTA)
static bool chunk_on() {
  static const int on = [] { const char* e = getenv("SF_DMMA_CHUNK"); return e ? atoi(e) : 0; }();
  return on != 0;
}
static int chunk_min_tiles() {
  static const int v = [] { const char* e = getenv("SF_DMMA_CHUNK_MIN"); return e ? atoi(e) : 444; }();
  return v;
}
static int chunk_fixed() {
  static const int v = [] { const char* e = getenv("SF_DMMA_CHUNK_T"); return e ? atoi(e) : 0; }();
  return v;
}

// true if gemm_f64_chunk_kernel serves this product
static bool chunk_eligible(const GemmF64& p, int a_kcontig, int b_kcontig, int mask) {
  if (!chunk_on() || mask != kMaskNone || p.splits != 1 || p.max_ctas > 0 || a_kcontig || !b_kcontig) return false;
  if (p.K <= 0 || p.K > g64s::KMAX || (p.K & 3) || (p.M & 1) || !p.beta || p.Cin != p.C || p.ldcin != p.ldc)
    return false;
  auto al = [](const void* q, int64_t ld) { return (((uintptr_t)q) & 15) == 0 && (ld % 2) == 0; };
  if (!al(p.A, p.lda) || !al(p.B, p.ldb) || !al(p.C, p.ldc)) return false;
  const int64_t tiles = ((p.M + g64s::BM - 1) / g64s::BM) * ((p.N + g64s::BN - 1) / g64s::BN);
  return tiles >= chunk_min_tiles();
}

static cudaError_t launch_chunk(const GemmF64& p, cudaStream_t st) {
  const int TM = (int)((p.M + g64s::BM - 1) / g64s::BM), TN = (int)((p.N + g64s::BN - 1) / g64s::BN);
  // about two waves of one-CTA-per-SM chunks; chunks of a row balanced to equal length
  int chunk = chunk_fixed();
  if (chunk <= 0) chunk = (int)(((int64_t)TM * TN + 2 * 148 - 1) / (2 * 148));
  if (chunk < 1) chunk = 1;
  if (chunk > TN) chunk = TN;
  const int cpr = (TN + chunk - 1) / chunk;
  chunk = (TN + cpr - 1) / cpr;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_f64_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)g64s::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gemm_f64_chunk_kernel<<<TM * cpr, g64s::NT, g64s::SMEM, st>>>(p, TN, chunk, cpr);
  count_launch();
  return cudaGetLastError();
}

static bool short_k_wide() {
  static const int on = [] { const char* e = getenv("SF_GEMM_SHORTK8"); return e ? atoi(e) : 1; }();
  return on != 0;
}
static int64_t short_k_max() {
  static const int64_t k = [] { const char* e = getenv("SF_GEMM_SHORTK8_MAXK"); return e ? (int64_t)atoll(e) : (int64_t)256; }();
  return k;
}

static bool grouped_short_k8() {
  // measured neutral at cfg2 (5.19 vs 5.14 ms without): off by default
  static const int on = [] { const char* e = getenv("SF_GROUPED_SHORTK8"); return e ? atoi(e) : 0; }();
  return on != 0;
}

template <bool AK, bool BKC, bool V16, int MASK>
static cudaError_t launch_t(const GemmF64& p, const GemmGroups* gs, int ntiles, int vecC, int bulk, cudaStream_t st) {
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_f64_kernel<AK, BKC, V16, MASK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g64::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_f64_grouped_kernel<AK, BKC, V16, MASK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g64::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_f64_loop_kernel<AK, BKC, V16, MASK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g64::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_f64_kernel<AK, BKC, V16, MASK, 256>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g64::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_f64_grouped_kernel<AK, BKC, V16, MASK, 256>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g64::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(ntiles, p.splits);
  if (gs && p.K <= short_k_max() && short_k_wide() && grouped_short_k8())
    // the short-K grouped launches (LU's L-shaped lookahead flush part, K = s = 64) sit on the
    // panel chain: 8 warps per CTA keep two issuing warps per SM sub-partition on an SM of
    // its own (one 4-warp CTA issues DMMA at about half rate)
    gemm_f64_grouped_kernel<AK, BKC, V16, MASK, 256><<<grid, 256, g64::SMEM, st>>>(p, *gs, vecC, bulk);
  else if (gs) gemm_f64_grouped_kernel<AK, BKC, V16, MASK><<<grid, g64::THREADS, g64::SMEM, st>>>(p, *gs, vecC, bulk);
  else if (p.max_ctas > 0 && p.max_ctas < ntiles) {
    grid.x = p.max_ctas;
    gemm_f64_loop_kernel<AK, BKC, V16, MASK><<<grid, g64::THREADS, g64::SMEM, st>>>(p, vecC);
  } else if (p.K <= short_k_max() && short_k_wide()) {
    // short K: the per-tile prologue/epilogue is a large share of each tile; 8-warp CTAs keep
    // two issuing warps per SM sub-partition through the co-resident CTA's epilogue
    gemm_f64_kernel<AK, BKC, V16, MASK, 256><<<grid, 256, g64::SMEM, st>>>(p, vecC, bulk);
  } else gemm_f64_kernel<AK, BKC, V16, MASK><<<grid, g64::THREADS, g64::SMEM, st>>>(p, vecC, bulk);
  count_launch();
  return cudaGetLastError();
}

template <bool AK, bool BKC, bool V16>
static cudaError_t launch_mask(const GemmF64& p, const GemmGroups* gs, int mask, int ntiles, int vecC, int bulk,
                               cudaStream_t st) {
  switch (mask) {
    case kMaskLower: return launch_t<AK, BKC, V16, kMaskLower>(p, gs, ntiles, vecC, bulk, st);
    case kMaskUpper: return launch_t<AK, BKC, V16, kMaskUpper>(p, gs, ntiles, vecC, bulk, st);
    default: return launch_t<AK, BKC, V16, kMaskNone>(p, gs, ntiles, vecC, bulk, st);
  }
}

static bool aligned16(const void* ptr, int64_t ld) {
  return (((uintptr_t)ptr) & 15) == 0 && (ld % 2) == 0;
}

static cudaError_t launch_key(const GemmF64& p, const GemmGroups* gs, int a_kcontig, int b_kcontig, bool v16, int mask,
                              int ntiles, int vecC, cudaStream_t st, int bulk = 0) {
  const int key = (a_kcontig ? 1 : 0) | (b_kcontig ? 2 : 0) | (v16 ? 4 : 0);
  switch (key) {
    case 0: return launch_mask<false, false, false>(p, gs, mask, ntiles, vecC, bulk, st);
    case 1: return launch_mask<true, false, false>(p, gs, mask, ntiles, vecC, bulk, st);
    case 2: return launch_mask<false, true, false>(p, gs, mask, ntiles, vecC, bulk, st);
    case 3: return launch_mask<true, true, false>(p, gs, mask, ntiles, vecC, bulk, st);
    case 4: return launch_mask<false, false, true>(p, gs, mask, ntiles, vecC, bulk, st);
    case 5: return launch_mask<true, false, true>(p, gs, mask, ntiles, vecC, bulk, st);
    case 6: return launch_mask<false, true, true>(p, gs, mask, ntiles, vecC, bulk, st);
    default: return launch_mask<true, true, true>(p, gs, mask, ntiles, vecC, bulk, st);
  }
}

// Tile variant per K (DESIGN.md §5 K1, measured: profiles/r02_dmma_variants.txt):
//   K <= 64        gemm_f64_kernel, 8 warps (the 128x64 short-K tile)
//   64 < K <= 128  v2, 64x64 tiles, 4 CTAs/SM, plain fragment loads
//   K > 128        v2, 64x64 tiles, 4 CTAs/SM, paired fragment loads
// SF_DMMA / SF_DMMA_SHORTK override (0 = gemm_f64_kernel, 1 = v2 128x64 paired 2/SM, 2 = 96x64
// paired 3/SM, 3 = 96x64 3/SM, 4 = 128x64 2/SM, 5 = 64x64 4/SM, 6 = 64x64 paired 4/SM) for
// the long- (K > 256) and short-K (K <= 256) products; SF_DMMA_BULK=0 disables the
// bulk-reduce epilogue.
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int dmma_variant_for(int64_t K) {
  static const int lk = env_int("SF_DMMA", -1), sk = env_int("SF_DMMA_SHORTK", -1);
  if (K > 256) return lk >= 0 ? lk : 6;
  if (sk >= 0) return sk;
  return K <= 64 ? 0 : (K <= 128 ? 5 : 6);
}
static bool dmma_bulk() {
  static const int v = env_int("SF_DMMA_BULK", 1);
  return v != 0;
}

template <int BM, int MINB, bool PAIR, bool AK, bool BKC, bool V16, int MASK>
static cudaError_t launch_v2_t(const GemmF64& p, int ntiles, int vecC, int bulk, cudaStream_t st) {
  constexpr size_t SM = g64v2::smem_bytes<BM, AK, BKC>();
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_f64v2_kernel<BM, MINB, PAIR, AK, BKC, V16, MASK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(ntiles, p.splits);
  gemm_f64v2_kernel<BM, MINB, PAIR, AK, BKC, V16, MASK><<<grid, 128, SM, st>>>(p, vecC, bulk);
  count_launch();
  return cudaGetLastError();
}
template <int BM, int MINB, bool PAIR, bool AK, bool BKC, bool V16>
static cudaError_t launch_v2_mask(const GemmF64& p, int mask, int ntiles, int vecC, int bulk, cudaStream_t st) {
  switch (mask) {
    case kMaskLower: return launch_v2_t<BM, MINB, PAIR, AK, BKC, V16, kMaskLower>(p, ntiles, vecC, bulk, st);
    case kMaskUpper: return launch_v2_t<BM, MINB, PAIR, AK, BKC, V16, kMaskUpper>(p, ntiles, vecC, bulk, st);
    default: return launch_v2_t<BM, MINB, PAIR, AK, BKC, V16, kMaskNone>(p, ntiles, vecC, bulk, st);
  }
}
template <int BM, int MINB, bool PAIR>
static cudaError_t launch_v2(GemmF64 p, int a_kcontig, int b_kcontig, bool v16, int mask, int vecC, int bulk,
                             cudaStream_t st) {
  using TT = Tiles<BM, 64>;
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + 63) / 64);
  const int ntiles = (int)TT::count(mask, TM, TN, p.off);
  if (ntiles == 0) return cudaSuccess;
  TT::make_raster(mask, TM, TN, p.off, kGroupCols, p.rs);
  p.ntiles = ntiles;
  const int key = (a_kcontig ? 1 : 0) | (b_kcontig ? 2 : 0) | (v16 ? 4 : 0);
  switch (key) {
    case 0: return launch_v2_mask<BM, MINB, PAIR, false, false, false>(p, mask, ntiles, vecC, bulk, st);
    case 1: return launch_v2_mask<BM, MINB, PAIR, true, false, false>(p, mask, ntiles, vecC, bulk, st);
    case 2: return launch_v2_mask<BM, MINB, PAIR, false, true, false>(p, mask, ntiles, vecC, bulk, st);
    case 3: return launch_v2_mask<BM, MINB, PAIR, true, true, false>(p, mask, ntiles, vecC, bulk, st);
    case 4: return launch_v2_mask<BM, MINB, PAIR, false, false, true>(p, mask, ntiles, vecC, bulk, st);
    case 5: return launch_v2_mask<BM, MINB, PAIR, true, false, true>(p, mask, ntiles, vecC, bulk, st);
    case 6: return launch_v2_mask<BM, MINB, PAIR, false, true, true>(p, mask, ntiles, vecC, bulk, st);
    default: return launch_v2_mask<BM, MINB, PAIR, true, true, true>(p, mask, ntiles, vecC, bulk, st);
  }
}

cudaError_t gemm_f64(GemmF64 p, int a_kcontig, int b_kcontig, int mask, cudaStream_t st) {
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  if (p.K <= 0) {
    // nothing to subtract: C = beta ? Cin : 0 (only needed out of place)
    if (p.beta && p.Cin == p.C && p.ldcin == p.ldc) return cudaSuccess;
    p.K = 0;
  }
  if (p.splits < 1) p.splits = 1;
  if (chunk_eligible(p, a_kcontig, b_kcontig, mask)) return launch_chunk(p, st);
  {
    const int var = dmma_variant_for(p.K);
    if (var > 0 && p.max_ctas == 0 && p.K > 0) {
      const bool v16 = aligned16(p.A, p.lda) && aligned16(p.B, p.ldb);
      const int vecC = aligned16(p.C, p.ldc) && (!p.beta || aligned16(p.Cin, p.ldcin));
      const int bulk = dmma_bulk() && p.splits == 1 && p.beta && vecC && p.Cin == p.C && p.ldcin == p.ldc;
      cudaError_t e;
      switch (var) {
        case 1: e = launch_v2<128, 2, true>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
        case 2: e = launch_v2<96, 3, true>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
        case 3: e = launch_v2<96, 3, false>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
        case 5: e = launch_v2<64, 4, false>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
        case 6: e = launch_v2<64, 4, true>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
        default: e = launch_v2<128, 2, false>(p, a_kcontig, b_kcontig, v16, mask, vecC, bulk, st); break;
      }
      if (e != cudaSuccess || p.splits == 1) return e;
      return splitk_reduce(p, st);
    }
  }
  const int TM = (int)((p.M + g64::BM - 1) / g64::BM), TN = (int)((p.N + g64::BN - 1) / g64::BN);
  const int ntiles = masked_tiles(mask, TM, TN, p.off);
  if (ntiles == 0) return cudaSuccess;
  T64::make_raster(mask, TM, TN, p.off, kGroupCols, p.rs);
  p.ntiles = ntiles;
  const bool v16 = aligned16(p.A, p.lda) && aligned16(p.B, p.ldb);
  const int vecC = aligned16(p.C, p.ldc) && (!p.beta || aligned16(p.Cin, p.ldcin));
  const int bulk = dmma_bulk() && p.splits == 1 && p.beta && vecC && p.Cin == p.C && p.ldcin == p.ldc;
  cudaError_t e = launch_key(p, nullptr, a_kcontig, b_kcontig, v16, mask, ntiles, vecC, st, bulk);
  if (e != cudaSuccess || p.splits == 1) return e;
  return splitk_reduce(p, st);
}

cudaError_t gemm_f64_grouped(GemmF64 p, const GemmGroup* groups, int count, int a_kcontig, int b_kcontig, int mask,
                             cudaStream_t st) {
  // groups with an empty block are dropped; one launch per kMaxGroups groups
  if (p.K <= 0) return cudaErrorInvalidValue;
  p.rs.ngroups = 0;
  bool v16 = (p.lda % 2) == 0 && (p.ldb % 2) == 0;
  int vecC = (p.ldc % 2) == 0 && (!p.beta || (p.ldcin % 2) == 0);
  p.splits = 1;
  GemmGroups gs{};
  int ntiles = 0;
  bool inplace = p.beta && p.ldcin == p.ldc;
  for (int i = 0; i < count; ++i) {
    const GemmGroup& g = groups[i];
    if (g.M <= 0 || g.N <= 0) continue;
    v16 = v16 && aligned16(g.A, p.lda) && aligned16(g.B, p.ldb);
    vecC = vecC && aligned16(g.C, p.ldc) && (!p.beta || aligned16(g.Cin, p.ldcin));
    inplace = inplace && g.Cin == g.C;
  }
  const int bulk = dmma_bulk() && inplace && vecC;
  for (int i = 0; i < count; ++i) {
    GemmGroup g = groups[i];
    if (g.M <= 0 || g.N <= 0) continue;
    const int TM = (int)((g.M + g64::BM - 1) / g64::BM), TN = (int)((g.N + g64::BN - 1) / g64::BN);
    const int nt = masked_tiles(mask, TM, TN, g.off);
    if (nt == 0) continue;
    if (gs.count == kMaxGroups) {
      cudaError_t e = launch_key(p, &gs, a_kcontig, b_kcontig, v16, mask, ntiles, vecC, st, bulk);
      if (e != cudaSuccess) return e;
      gs.count = 0; ntiles = 0;
    }
    g.tile0 = ntiles;
    gs.g[gs.count++] = g;
    ntiles += nt;
  }
  if (gs.count == 0) return cudaSuccess;
  return launch_key(p, &gs, a_kcontig, b_kcontig, v16, mask, ntiles, vecC, st, bulk);
}

}  // namespace sf
