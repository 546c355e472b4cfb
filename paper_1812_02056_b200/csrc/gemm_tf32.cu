// gemm_tf32.cu — the fp32 trailing update on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with the 3xTF32 split, accumulators in TMEM, operands staged by TMA
// (BASELINE.json north_star (1)).
//
//   C(M x N) = Cin - A B^T     (Cholesky flush PAPER.md:42-50: A = B = R = L[c:n, z:c);
//                               in-panel corrections of the fp32 panel recursion)
//
// 3xTF32 (DESIGN.md §5 K5): every fp32 operand x is split once into x_hi = rna_tf32(x) and
// x_lo = rna_tf32(x - x_hi) (split_tf32 below, K-major copies), and
//   A B^T ~= A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T
// is ONE tcgen05 GEMM over K' = 3K (the lo*lo term, ~2^-22 relative, is dropped).  x_hi and
// x_lo have zero low mantissa bits, so the hardware's TF32 operand truncation is exact and
// the products accumulate in fp32 in TMEM.
//
// Kernel (one 128 x BN tile per CTA, BN = 256 for the flush, 64/128 for the narrow in-panel
// corrections; two CTAs per SM, 6 warps):
//   warp 0     TMA producer (one lane): per BK = 16 slice the four operand tiles A_hi, A_lo
//              (128 x 16), B_hi, B_lo (BN x 16) — 64-byte rows, 64B swizzle — into a ring of
//              96 KB, mbarrier complete_tx; lanes 1-31 first warm L2 with the C tile
//   warp 1     MMA issuer (one lane): per 8-wide k-step hi.hi, hi.lo, lo.hi tcgen05.mma
//              (M = 128, N = BN) into one TMEM accumulator; tcgen05.commit frees the stage
//   warps 2-5  epilogue: tcgen05.ld 32 lanes x 32 columns at a time, C = Cin - acc, masked
//              store (column-major C: a warp's 32 rows of one column are one 128-byte line)
// Non-persistent on purpose: the lookahead stream's panel kernels get SMs between CTAs, and
// the second CTA on the SM overlaps this one's epilogue (DESIGN.md §5 K5).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace sf {

namespace t32 {
constexpr int BM = 128, BK = 16;                 // BK fp32 = 64 bytes = one 64B-swizzle row
constexpr int UMMA_K = 8;                        // kind::tf32: K = 8 per instruction (32 bytes)
constexpr int THREADS = 192;
template <int BN> struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;                 // one of A_hi / A_lo: 8 KB
  static constexpr int B_BYTES = BN * BK * 4;                 // one of B_hi / B_lo
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (96 * 1024) / STAGE_BYTES;    // 96 KB of stages: two CTAs per SM
  static constexpr int TMEM_COLS = BN;                        // one fp32 accumulator
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  using TT = Tiles<BM, BN>;
};
}  // namespace t32

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)map) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// K-major, 64B-swizzled operand tile: rows of 64 bytes (16 fp32), 8-row atoms 512 bytes apart.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                           // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;                  // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                           // descriptor version (tcgen05)
  d |= (uint64_t)4 << 61;                           // layout: SWIZZLE_64B
  return d;
}
// Instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major, M = 128, N = BN.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)                 // D format f32
         | (2u << 7)               // A format tf32
         | (2u << 10)              // B format tf32
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ the kernel
struct Tf32Params {
  int64_t M, N, K;          // C is M x N, products over K (the split operands have K columns)
  const float* Cin; int64_t ldcin;
  float* C; int64_t ldc;
  int64_t off;              // mask diagonal offset
  int mask;
  const long long* fail;
  float alpha;              // C = (beta ? Cin : 0) + alpha * acc
  int beta;
};

// One 128 x BN tile per CTA, two CTAs per SM (96 KB of stages each): one CTA's epilogue
// overlaps the other's MMAs, and between CTAs the lookahead stream's panel kernels get SMs.
// Each stage holds one BK = 16 slice of all four operands (A_hi, A_lo, B_hi, B_lo), so the
// three products of a slice are issued back to back and every operand byte fetched from L2
// feeds 1.5 MMAs on average (3 products from 4 tiles).
template <int BN>
__global__ void __launch_bounds__(t32::THREADS, 2)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                   const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, Tf32Params p) {
  using namespace t32;
  using C_ = Cfg<BN>;
  constexpr int STAGES = C_::STAGES, A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES;
  if (p.fail && failed(p.fail)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);   // swizzle atoms aligned
  uint64_t* full = (uint64_t*)(smem + STAGES * C_::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
  auto sAh = [&](int s) { return smem + s * C_::STAGE_BYTES; };
  auto sAl = [&](int s) { return smem + s * C_::STAGE_BYTES + A_BYTES; };
  auto sBh = [&](int s) { return smem + s * C_::STAGE_BYTES + 2 * A_BYTES; };
  auto sBl = [&](int s) { return smem + s * C_::STAGE_BYTES + 2 * A_BYTES + B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + BN - 1) / BN);
  int ti, tj;
  // column order (not the DMMA kernel's rasterized order): the CTAs running at once then
  // read the same B slices (2/3 of the operand bytes), which L2 serves as one request
  C_::TT::tile_of(p.mask, blockIdx.x, TM, TN, p.off, ti, tj);
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * BN;
  const int nkb = (int)((p.K + BK - 1) / BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh); tma_prefetch_desc(&mAl); tma_prefetch_desc(&mBh); tma_prefetch_desc(&mBl);
  } else if (warp == 0) {
    // warm L2 with this tile's C columns for the epilogue's read-modify-write
    for (int u = lane - 1; u < BN * 4; u += 31) {
      const int64_t j = j0 + (u >> 2), i = i0 + (u & 3) * 32;
      if (p.beta && j < p.N && i < p.M) prefetch_l2(p.Cin + i + j * p.ldcin);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(C_::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: one BK slice of A_hi, A_lo, B_hi, B_lo per stage
      const int ya = (int)i0, yb = (int)j0;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], C_::STAGE_BYTES);
        tma_load_2d(sAh(s), &mAh, &full[s], kb * BK, ya);
        tma_load_2d(sAl(s), &mAl, &full[s], kb * BK, ya);
        tma_load_2d(sBh(s), &mBh, &full[s], kb * BK, yb);
        tma_load_2d(sBl(s), &mBl, &full[s], kb * BK, yb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: per k-step hi.hi, hi.lo, lo.hi into one accumulator
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sAh(s)), al = smem_u32(sAl(s)), bh = smem_u32(sBh(s)), bl = smem_u32(sBl(s));
#pragma unroll
        for (int k = 0; k < BK / UMMA_K; ++k) {
          const uint32_t o = k * UMMA_K * 4;   // 32 bytes along K inside the swizzled row
          umma_tf32(tmem, umma_desc_sw64(ah + o), umma_desc_sw64(bh + o), idesc, (kb | k) != 0);
          umma_tf32(tmem, umma_desc_sw64(ah + o), umma_desc_sw64(bl + o), idesc, 1);
          umma_tf32(tmem, umma_desc_sw64(al + o), umma_desc_sw64(bh + o), idesc, 1);
        }
        umma_commit(&empty[s]);                // frees the stage when these MMAs retire
      }
      umma_commit(tfull);                      // accumulator complete
    }
  } else {
    // ---------------- epilogue: warps 2..5 -> TMEM lanes 32*(warp%4) .. +31
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int64_t i = i0 + q * 32 + lane;
    for (int c = 0; c < BN; c += 32) {
      if (j0 + c >= p.N) break;
      float v[32];
      tmem_ld32(tmem + lane_base + (uint32_t)c, v);
      if (i < p.M) {
        float cin[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int64_t j = j0 + c + u;
          const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
          cin[u] = (in && p.beta) ? __ldcg(p.Cin + i + j * p.ldcin) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int64_t j = j0 + c + u;
          const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
          if (in) __stcg(p.C + i + j * p.ldc, fmaf(p.alpha, v[u], cin[u]));
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C_::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with M = 256
// MMAs issued by the leader (rank 0).  Each CTA stages only ITS half of the operands — A rows
// [rank*128, +128) and B rows [rank*128, +128) — so an SM receives 2 x 32 KB per BK slice
// instead of 48 KB for the same MMA work (the single-CTA kernel is bound by that operand
// traffic).  Protocol (the leader's barriers coordinate both CTAs):
//   full[s]   (leader)   1 arrival (leader's expect_tx of both CTAs' bytes) + the tx of both
//                        CTAs' TMA (cta_group::2 form, barrier address with the peer bit
//                        cleared -> the leader's barrier)
//   empty[s]  (each CTA) the leader's tcgen05.commit multicast to both CTAs
//   tfull     (each CTA) likewise, after the last MMA; each CTA then drains its own TMEM
//                        (its 128 rows of D)
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;   // shared::cluster address of the rank-0 CTA

namespace t32p {
constexpr int BM = 256, BN = 256, HALF = 128, BK = 16;
constexpr int TILE = HALF * BK * 4;                 // one operand tile per CTA: 8 KB
constexpr int STAGE_BYTES = 4 * TILE;               // A_hi, A_lo, B_hi, B_lo halves: 32 KB
constexpr int STAGES = 3;                           // 96 KB: two CTAs (of different pairs) per SM
constexpr int TMEM_COLS = BN;
constexpr int ECOLS = 64;                           // epilogue C chunk: 128 rows x 64 columns = 32 KB
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
static_assert(3 * HALF * ECOLS * 4 <= STAGES * STAGE_BYTES, "epilogue ring fits in the stage buffers");
using TT = Tiles<BM, BN>;
}  // namespace t32p

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// One 256 x 256 tile per pair, two CTAs per SM.  Epilogue: when the CTA's 128 x 256 block of
// C lies inside the mask with whole 16-byte columns, C is fetched with bulk async copies
// (cp.async.bulk, 512 B per column) through a 3-deep ring of 64-column chunks in the idle
// stage buffers — the epilogue is latency-bound otherwise (32 scalar loads in flight per
// thread) — and results are stored straight from registers.  Other blocks (the diagonal,
// ragged edges, unaligned C) take the per-element path.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(t32::THREADS, 2)
gemm_tf32x3_pair_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                        const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, Tf32Params p,
                        int vecC, const __grid_constant__ Raster rs) {
  using namespace t32p;
  // no early exit on p.fail here: both CTAs of the pair must reach every cluster barrier
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* cbar = tfull + 1;           // [3] epilogue chunk ring
  uint32_t* tmem_slot = (uint32_t*)(cbar + 3);
  auto sAh = [&](int s) { return smem + s * STAGE_BYTES; };
  auto sAl = [&](int s) { return smem + s * STAGE_BYTES + TILE; };
  auto sBh = [&](int s) { return smem + s * STAGE_BYTES + 2 * TILE; };
  auto sBl = [&](int s) { return smem + s * STAGE_BYTES + 3 * TILE; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + BN - 1) / BN);
  int ti, tj;
  if (rs.ngroups > 0) TT::tile_of_raster(p.mask, blockIdx.x >> 1, TM, p.off, rs, ti, tj);
  else TT::tile_of(p.mask, blockIdx.x >> 1, TM, TN, p.off, ti, tj);
  const int64_t i0 = (int64_t)ti * BM, j0 = (int64_t)tj * BN;
  const int64_t r0 = i0 + rank * HALF;    // this CTA's first C row
  const int nkb = (int)((p.K + BK - 1) / BK);
  const bool skip = p.fail && failed(p.fail);
  // bulk epilogue: the whole 128 x 256 block is inside M, N and the mask
  const int64_t jl = j0 + BN - 1;
  const bool inside = (r0 + HALF <= p.M) && (j0 + BN <= p.N) &&
                      (p.mask == kMaskNone || (p.mask == kMaskLower ? r0 >= jl + p.off : r0 + HALF - 1 <= j0 + p.off));
  const bool bulk = vecC && inside && !skip && p.beta;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    for (int c = 0; c < 3; ++c) mbar_init(&cbar[c], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh); tma_prefetch_desc(&mAl); tma_prefetch_desc(&mBh); tma_prefetch_desc(&mBl);
  } else if (warp == 0) {
    for (int u = lane - 1; u < BN * 4; u += 31) {   // warm L2 with this CTA's C rows
      const int64_t j = j0 + (u >> 2), i = r0 + (u & 3) * 32;
      if (p.beta && j < p.N && i < p.M) prefetch_l2(p.Cin + i + j * p.ldcin);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();   // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const int ya = (int)r0, yb = (int)(j0 + rank * HALF);
      const uint32_t lbar0 = smem_u32(&full[0]) & kPeerMask;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
        const uint32_t lbar = lbar0 + s * 8;
        tma_load_2d_pair(sAh(s), &mAh, lbar, kb * BK, ya);
        tma_load_2d_pair(sAl(s), &mAl, lbar, kb * BK, ya);
        tma_load_2d_pair(sBh(s), &mBh, lbar, kb * BK, yb);
        tma_load_2d_pair(sBl(s), &mBl, lbar, kb * BK, yb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sAh(s)), al = smem_u32(sAl(s)), bh = smem_u32(sBh(s)), bl = smem_u32(sBl(s));
#pragma unroll
        for (int k = 0; k < BK / t32::UMMA_K; ++k) {
          const uint32_t o = k * t32::UMMA_K * 4;
          umma_tf32_pair(tmem, umma_desc_sw64(ah + o), umma_desc_sw64(bh + o), idesc, (kb | k) != 0);
          umma_tf32_pair(tmem, umma_desc_sw64(ah + o), umma_desc_sw64(bl + o), idesc, 1);
          umma_tf32_pair(tmem, umma_desc_sw64(al + o), umma_desc_sw64(bh + o), idesc, 1);
        }
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(tfull);
    }
  } else {
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int row = q * 32 + lane;          // this thread's row inside the CTA's 128 rows
    const int64_t i = r0 + row;
    mbar_wait(tfull, 0);                    // all MMAs done: the stage buffers are free
    tc_fence_after();
    if (bulk) {
      float* ring = (float*)smem;           // [3][ECOLS][HALF], column-major chunks
      constexpr int NCH = BN / ECOLS;
      auto issue = [&](int ch) {            // warp 2 fetches chunk ch into ring slot ch % 3
        float* dst = ring + (ch % 3) * ECOLS * HALF;
        if (lane == 0) mbar_expect_tx(&cbar[ch % 3], ECOLS * HALF * 4);
        __syncwarp();
        for (int u = lane; u < ECOLS; u += 32)
          bulk_g2s(dst + u * HALF, p.Cin + r0 + (j0 + ch * ECOLS + u) * p.ldcin, HALF * 4, &cbar[ch % 3]);
      };
      if (warp == 2)
        for (int ch = 0; ch < 3 && ch < NCH; ++ch) issue(ch);
      for (int ch = 0; ch < NCH; ++ch) {
        mbar_wait(&cbar[ch % 3], (ch / 3) & 1);
        const float* src = ring + (ch % 3) * ECOLS * HALF;
#pragma unroll
        for (int c = 0; c < ECOLS; c += 32) {
          float v[32];
          tmem_ld32(tmem + lane_base + (uint32_t)(ch * ECOLS + c), v);
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int64_t j = j0 + ch * ECOLS + c + u;
            __stcg(p.C + i + j * p.ldc, fmaf(p.alpha, v[u], src[(c + u) * HALF + row]));
          }
        }
        epi_bar_sync();                     // all four epilogue warps are done with slot ch % 3
        if (warp == 2 && ch + 3 < NCH) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic reads before async writes
          issue(ch + 3);
        }
      }
    } else {
      for (int c = 0; c < BN; c += 32) {
        if (j0 + c >= p.N) break;
        float v[32];
        tmem_ld32(tmem + lane_base + (uint32_t)c, v);
        if (i < p.M && !skip) {
          float cin[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int64_t j = j0 + c + u;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            cin[u] = (in && p.beta) ? __ldcg(p.Cin + i + j * p.ldcin) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int64_t j = j0 + c + u;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            if (in) __stcg(p.C + i + j * p.ldc, fmaf(p.alpha, v[u], cin[u]));
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  cluster_sync_all();   // the peer's TMEM / smem stay live until the leader's MMAs are done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ persistent CTA-pair variant
// One CTA pair per pair of SMs walks the tiles (static round-robin over the rasterized
// order) with TWO TMEM accumulators (2 x 256 columns = all 512): the leader's MMAs for tile
// t+1 run while both CTAs' epilogue warps drain tile t, so no tile pays its epilogue (or the
// pipeline fill: the producer runs ahead into the next tile's slices) on the tensor pipe.
// In-place tiles inside M, N (the flushes after the first) are added to C by bulk reduction
// (cp.reduce.async.bulk .add.f32, one 512-byte column per lane from a double-buffered staging
// chunk; masked entries add -0.0, which leaves every value bit-identical); other tiles take
// the per-element load/add/store path.  fl(C + alpha*acc) is the same IEEE operation either way.
// Barriers (leader-owned unless noted):
//   full[s] / empty[s] (each CTA)   as in gemm_tf32x3_pair_kernel, slice counter across tiles
//   tfull[a]  (each CTA)            the leader's commit after a tile's last MMA into accumulator a
//   tempty[a] (leader)              8 arrivals: the 4 epilogue warps of each CTA, after reading a
namespace t32q {
constexpr int BM = 256, BN = 256, HALF = 128, BK = 16;
constexpr int TILE = HALF * BK * 4;                 // one operand tile per CTA: 8 KB
constexpr int STAGE_BYTES = 4 * TILE;               // 32 KB
constexpr int STAGES = 5;
constexpr int ECOLS = 32;                           // staging chunk: 128 rows x 32 columns = 16 KB
constexpr int STG_BYTES = HALF * ECOLS * 4;
constexpr int TMEM_COLS = 2 * BN;
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 2 * STG_BYTES + 1024 + 256;
using TT = Tiles<BM, BN>;
}  // namespace t32q

__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, const float* ssrc, int bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(t32::THREADS, 1)
gemm_tf32x3_pair_persist_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                                const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                                Tf32Params p, int vecC, int ntiles, int tpc, const __grid_constant__ Raster rs) {
  using namespace t32q;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* stg = (float*)(smem + STAGES * STAGE_BYTES);           // [2][ECOLS][HALF]
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES + 2 * STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;     // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  auto sAh = [&](int s) { return smem + s * STAGE_BYTES; };
  auto sAl = [&](int s) { return smem + s * STAGE_BYTES + TILE; };
  auto sBh = [&](int s) { return smem + s * STAGE_BYTES + 2 * TILE; };
  auto sBl = [&](int s) { return smem + s * STAGE_BYTES + 3 * TILE; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // tiles of this pair: tpc > 0 -> the contiguous run [pair*tpc, +tpc) of the rasterized order
  // (pairs retire every tpc tiles, so the lookahead stream's panel kernels get SMs); tpc = 0
  // -> every npairs-th tile (fully persistent)
  const int t_first = tpc ? pair * tpc : pair, t_step = tpc ? 1 : npairs;
  const int t_end = tpc ? min(ntiles, (pair + 1) * tpc) : ntiles;
  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + BN - 1) / BN);
  const int nkb = (int)((p.K + BK - 1) / BK);
  const bool skip = p.fail && failed(p.fail);   // both CTAs still pass every barrier
  auto tile_ij = [&](int t, int64_t& i0, int64_t& j0) {
    int ti, tj;
    if (rs.ngroups > 0) TT::tile_of_raster(p.mask, t, TM, p.off, rs, ti, tj);
    else TT::tile_of(p.mask, t, TM, TN, p.off, ti, tj);
    i0 = (int64_t)ti * BM; j0 = (int64_t)tj * BN;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh); tma_prefetch_desc(&mAl); tma_prefetch_desc(&mBh); tma_prefetch_desc(&mBl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (each CTA: its halves of A and B), running ahead across tiles
      const uint32_t lbar0 = smem_u32(&full[0]) & kPeerMask;
      int g = 0;
      for (int t = t_first; t < t_end; t += t_step) {
        int64_t i0, j0;
        tile_ij(t, i0, j0);
        const int ya = (int)(i0 + rank * HALF), yb = (int)(j0 + rank * HALF);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
          const uint32_t lbar = lbar0 + s * 8;
          tma_load_2d_pair(sAh(s), &mAh, lbar, kb * BK, ya);
          tma_load_2d_pair(sAl(s), &mAl, lbar, kb * BK, ya);
          tma_load_2d_pair(sBh(s), &mBh, lbar, kb * BK, yb);
          tma_load_2d_pair(sBl(s), &mBl, lbar, kb * BK, yb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader): tile it into accumulator it & 1
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      int g = 0, it = 0;
      for (int t = t_first; t < t_end; t += t_step, ++it) {
        const int a = it & 1, u = it >> 1;
        mbar_wait(&tempty[a], (u & 1) ^ 1);   // both CTAs' epilogues have drained accumulator a
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(a * BN);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t ah = smem_u32(sAh(s)), al = smem_u32(sAl(s)), bh = smem_u32(sBh(s)), bl = smem_u32(sBl(s));
#pragma unroll
          for (int k = 0; k < BK / t32::UMMA_K; ++k) {
            const uint32_t o = k * t32::UMMA_K * 4;
            umma_tf32_pair(d, umma_desc_sw64(ah + o), umma_desc_sw64(bh + o), idesc, (kb | k) != 0);
            umma_tf32_pair(d, umma_desc_sw64(ah + o), umma_desc_sw64(bl + o), idesc, 1);
            umma_tf32_pair(d, umma_desc_sw64(al + o), umma_desc_sw64(bh + o), idesc, 1);
          }
          umma_commit_pair(&empty[s]);
        }
        umma_commit_pair(&tfull[a]);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 -> TMEM lanes 32*(warp%4) .. +31 = CTA rows
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int row = q * 32 + lane;
    const uint32_t tempty_leader = smem_u32(&tempty[0]) & kPeerMask;
    int it = 0, nchunk = 0;
    for (int t = t_first; t < t_end; t += t_step, ++it) {
      const int a = it & 1, u = it >> 1;
      int64_t i0, j0;
      tile_ij(t, i0, j0);
      const int64_t r0 = i0 + rank * HALF, i = r0 + row;
      const bool bulk = vecC && !skip && (r0 + HALF <= p.M) && (j0 + BN <= p.N);
      mbar_wait(&tfull[a], u & 1);
      tc_fence_after();
      const uint32_t tacc = tmem + lane_base + (uint32_t)(a * BN);
      for (int c = 0; c < BN; c += ECOLS) {
        if (!bulk && j0 + c >= p.N) break;
        float v[32];
        tmem_ld32(tacc + (uint32_t)c, v);
        if (bulk) {
          float* buf = stg + (nchunk & 1) * (ECOLS * HALF);
          if (nchunk >= 2) {
            if (warp == 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");   // buf's last reduce has read it
            epi_bar_sync();
          }
#pragma unroll
          for (int uu = 0; uu < 32; ++uu) {
            const int64_t j = j0 + c + uu;
            const bool in = p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off);
            buf[uu * HALF + row] = in ? p.alpha * v[uu] : -0.f;
          }
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          epi_bar_sync();
          if (warp == 2) {
            bulk_reduce_add_f32(p.C + r0 + (j0 + c + lane) * p.ldc, buf + lane * HALF, HALF * 4);
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          }
          ++nchunk;
        } else if (i < p.M && !skip) {
          float cin[32];
#pragma unroll
          for (int uu = 0; uu < 32; ++uu) {
            const int64_t j = j0 + c + uu;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            cin[uu] = (in && p.beta) ? __ldcg(p.Cin + i + j * p.ldcin) : 0.f;
          }
#pragma unroll
          for (int uu = 0; uu < 32; ++uu) {
            const int64_t j = j0 + c + uu;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            if (in) __stcg(p.C + i + j * p.ldc, fmaf(p.alpha, v[uu], cin[uu]));
          }
        }
      }
      // accumulator a is free once every epilogue warp of both CTAs has read it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + a * 8);
    }
    if (warp == 2) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ split kernel
// x -> (rna_tf32(x), rna_tf32(x - hi)), transposed from column-major (m x k, ld) to K-major
// (row i: k contiguous values at H + i*ldk).  32 x 32 tiles through shared memory.
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void split_tf32_kernel(int64_t m, int64_t k, const float* __restrict__ X, int64_t ld, float* __restrict__ H,
                                  float* __restrict__ L, int64_t ldk) {
  __shared__ float t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + tx, kk = k0 + r;
    t[r][tx] = (i < m && kk < k) ? __ldcg(X + i + kk * ld) : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, kk = k0 + tx;
    if (i < m && kk < k) {
      const float x = t[tx][r];
      const float hi = rna_tf32(x);
      H[i * ldk + kk] = hi;
      L[i * ldk + kk] = rna_tf32(x - hi);
    }
  }
}

cudaError_t split_tf32(int64_t m, int64_t k, const float* X, int64_t ld, float* H, float* L, int64_t ldk,
                       cudaStream_t st) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)((k + 31) / 32));
  split_tf32_kernel<<<grid, 256, 0, st>>>(m, k, X, ld, H, L, ldk);
  count_launch();
  return cudaGetLastError();
}

__global__ void split_tf32_kmajor_kernel(int64_t m, int64_t k, const float* __restrict__ X, int64_t ld,
                                         float* __restrict__ H, float* __restrict__ L, int64_t ldk) {
  const int64_t total = m * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k, kk = t % k;
    const float x = __ldcg(X + i * ld + kk);
    const float hi = rna_tf32(x);
    H[i * ldk + kk] = hi;
    L[i * ldk + kk] = rna_tf32(x - hi);
  }
}

cudaError_t split_tf32_kmajor(int64_t m, int64_t k, const float* X, int64_t ld, float* H, float* L, int64_t ldk,
                              cudaStream_t st) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  int64_t blocks = (m * k + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  split_tf32_kmajor_kernel<<<(unsigned)blocks, 256, 0, st>>>(m, k, X, ld, H, L, ldk);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)f;
  }();
  return fn;
}

// 2-D map over a K-major fp32 operand: `rows` rows of `k` valid columns, row stride ldk;
// box = BK columns x box_rows rows, 64-byte swizzle; out-of-range elements read as zero.
static cudaError_t make_map(CUtensorMap* map, const float* base, int64_t k, int64_t rows, int64_t ldk, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldk * 4};
  cuuint32_t box[2] = {(cuuint32_t)t32::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN>
static cudaError_t launch_bn(const Tf32Gemm& g, cudaStream_t st) {
  using namespace t32;
  using C_ = Cfg<BN>;
  const int TM = (int)((g.M + BM - 1) / BM), TN = (int)((g.N + BN - 1) / BN);
  const int ntiles = C_::TT::count(g.mask, TM, TN, g.off);
  if (ntiles == 0) return cudaSuccess;
  CUtensorMap mAh, mAl, mBh, mBl;
  cudaError_t e;
  // the maps start at the operands' first rows; TMA rows beyond M / N and columns beyond K
  // read zeros
  if ((e = make_map(&mAh, g.Ah, g.K, g.M, g.ldk_a, BM)) != cudaSuccess) return e;
  if ((e = make_map(&mAl, g.Al, g.K, g.M, g.ldk_a, BM)) != cudaSuccess) return e;
  if ((e = make_map(&mBh, g.Bh, g.K, g.N, g.ldk_b, BN)) != cudaSuccess) return e;
  if ((e = make_map(&mBl, g.Bl, g.K, g.N, g.ldk_b, BN)) != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(gemm_tf32x3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  Tf32Params p{g.M, g.N, g.K, g.Cin, g.ldcin, g.C, g.ldc, g.off, g.mask, g.fail, g.alpha, g.beta};
  gemm_tf32x3_kernel<BN><<<ntiles, THREADS, C_::SMEM, st>>>(mAh, mAl, mBh, mBl, p);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_pair(const Tf32Gemm& g, cudaStream_t st) {
  using namespace t32p;
  const int TM = (int)((g.M + BM - 1) / BM), TN = (int)((g.N + BN - 1) / BN);
  const int ntiles = TT::count(g.mask, TM, TN, g.off);
  if (ntiles == 0) return cudaSuccess;
  CUtensorMap mAh, mAl, mBh, mBl;
  cudaError_t e;
  if ((e = make_map(&mAh, g.Ah, g.K, g.M, g.ldk_a, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mAl, g.Al, g.K, g.M, g.ldk_a, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mBh, g.Bh, g.K, g.N, g.ldk_b, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mBl, g.Bl, g.K, g.N, g.ldk_b, HALF)) != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(gemm_tf32x3_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  Tf32Params p{g.M, g.N, g.K, g.Cin, g.ldcin, g.C, g.ldc, g.off, g.mask, g.fail, g.alpha, g.beta};
  static int bulk_on = [] { const char* e = getenv("SF_TF32_BULKEPI"); return e ? atoi(e) : 1; }();
  const int vecC = bulk_on && g.beta && (g.ldc % 4) == 0 && (g.ldcin % 4) == 0 && ((uintptr_t)g.Cin % 16) == 0 &&
                   ((uintptr_t)g.C % 16) == 0;
  // tile order: rasterized in groups of `gb` tile columns when the operands exceed what L2
  // keeps (SF_TF32_RASTER overrides; 0 = column order)
  static int gb_env = [] { const char* e = getenv("SF_TF32_RASTER"); return e ? atoi(e) : -1; }();
  Raster rs;
  const int gb = gb_env >= 0 ? gb_env : 8;
  if (gb > 0) TT::make_raster(g.mask, TM, TN, g.off, gb, rs);
  gemm_tf32x3_pair_kernel<<<2 * ntiles, t32::THREADS, SMEM, st>>>(mAh, mAl, mBh, mBl, p, vecC, rs);
  count_launch();
  return cudaGetLastError();
}

// persistent pairs for flushes of at least SF_TF32_PERSIST_MIN tiles (0 = always; -1 = never)
static bool persist_for(int ntiles) {
  static int mn = [] { const char* e = getenv("SF_TF32_PERSIST_MIN"); return e ? atoi(e) : 0; }();
  return mn >= 0 && ntiles >= mn;
}

static cudaError_t launch_pair_persist(const Tf32Gemm& g, cudaStream_t st) {
  using namespace t32q;
  const int TM = (int)((g.M + BM - 1) / BM), TN = (int)((g.N + BN - 1) / BN);
  const int ntiles = TT::count(g.mask, TM, TN, g.off);
  if (ntiles == 0) return cudaSuccess;
  CUtensorMap mAh, mAl, mBh, mBl;
  cudaError_t e;
  if ((e = make_map(&mAh, g.Ah, g.K, g.M, g.ldk_a, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mAl, g.Al, g.K, g.M, g.ldk_a, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mBh, g.Bh, g.K, g.N, g.ldk_b, HALF)) != cudaSuccess) return e;
  if ((e = make_map(&mBl, g.Bl, g.K, g.N, g.ldk_b, HALF)) != cudaSuccess) return e;
  static bool attr = false;
  static int sms = 148;
  if (!attr) {
    e = cudaFuncSetAttribute(gemm_tf32x3_pair_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  Tf32Params p{g.M, g.N, g.K, g.Cin, g.ldcin, g.C, g.ldc, g.off, g.mask, g.fail, g.alpha, g.beta};
  // bulk-reduce epilogue: in place, 16-byte aligned columns
  const int vecC = g.beta && g.Cin == g.C && g.ldcin == g.ldc && (g.ldc % 4) == 0 && ((uintptr_t)g.C % 16) == 0;
  static int gb_env = [] { const char* e = getenv("SF_TF32_RASTER"); return e ? atoi(e) : -1; }();
  Raster rs;
  const int gb = gb_env >= 0 ? gb_env : 8;
  if (gb > 0) TT::make_raster(g.mask, TM, TN, g.off, gb, rs);
  static int tpc = [] { const char* e = getenv("SF_TF32_TPC"); return e ? atoi(e) : 0; }();
  // SF_TF32_RESERVE SMs are left to concurrent work (the lookahead panel) in persistent mode
  // (measured: 16 -> cfg5 fp32 505 ms, cfg3 fp32 22.1 ms; 0 -> 505 / 23.4; 32 -> 518 / 21.6)
  static int reserve = [] { const char* e = getenv("SF_TF32_RESERVE"); return e ? atoi(e) : 16; }();
  int maxp = (sms - reserve) / 2;
  if (maxp < 1) maxp = 1;
  const int npairs = tpc > 0 ? (ntiles + tpc - 1) / tpc : (ntiles < maxp ? ntiles : maxp);
  gemm_tf32x3_pair_persist_kernel<<<2 * npairs, t32::THREADS, SMEM, st>>>(mAh, mAl, mBh, mBl, p, vecC, ntiles, tpc,
                                                                          rs);
  count_launch();
  return cudaGetLastError();
}

static bool pair_on() {
  static int on = [] { const char* e = getenv("SF_TF32_PAIR"); return e ? atoi(e) : 1; }();
  return on != 0;
}

cudaError_t gemm_tf32x3(const Tf32Gemm& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaSuccess;
  if ((g.ldk_a % 4) || (g.ldk_b % 4) || ((uintptr_t)g.Ah % 16) || ((uintptr_t)g.Al % 16) || ((uintptr_t)g.Bh % 16) ||
      ((uintptr_t)g.Bl % 16))
    return cudaErrorInvalidValue;   // TMA: 16-byte aligned bases and row strides
  // narrow updates (the panel recursion's corrections) take a narrower tile
  if (g.N <= 64) return launch_bn<64>(g, st);
  if (g.N <= 128) return launch_bn<128>(g, st);
  if (pair_on()) {   // wide flushes: CTA pairs
    const int ntiles = t32p::TT::count(g.mask, (int)((g.M + 255) / 256), (int)((g.N + 255) / 256), g.off);
    return persist_for(ntiles) ? launch_pair_persist(g, st) : launch_pair(g, st);
  }
  return launch_bn<256>(g, st);
}

}  // namespace sf
