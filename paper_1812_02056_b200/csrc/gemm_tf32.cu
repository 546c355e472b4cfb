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
// Kernel (persistent, one CTA per SM, 6 warps):
//   warp 0     TMA producer (one lane): per k-block a 128 x 32 A tile and a 256 x 32 B tile
//              (128-byte rows, 128B swizzle) into a 4-stage ring, mbarrier complete_tx
//   warp 1     MMA issuer (one lane): 4 x tcgen05.mma 128x256x8 per k-block into one of two
//              TMEM accumulators (2 x 256 of the 512 columns), tcgen05.commit releases the
//              smem stage / publishes the accumulator
//   warps 2-5  epilogue: tcgen05.ld 32 lanes x 32 columns at a time, C = Cin - acc, masked
//              store (column-major C: a warp's 32 rows of one column are one 128-byte line);
//              the next tile's MMAs run meanwhile in the other accumulator
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace sf {

namespace t32 {
constexpr int BM = 128, BN = 256, BK = 32;      // BK fp32 = 128 bytes = one swizzle row
constexpr int STAGES = 4;
constexpr int UMMA_K = 8;                       // kind::tf32: K = 8 per instruction (32 bytes)
constexpr int A_BYTES = BM * BK * 4;            // 16 KB
constexpr int B_BYTES = BN * BK * 4;            // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 192;
constexpr int TMEM_COLS = 512;
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
using TT = Tiles<BM, BN>;
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

// K-major, 128B-swizzled operand tile: rows of 128 bytes, 8-row atoms 1024 bytes apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                           // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                 // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                           // descriptor version (tcgen05)
  d |= (uint64_t)2 << 61;                           // layout: SWIZZLE_128B
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
  int64_t a_row0, b_row0;   // first row of A / B in their tensor maps
  const float* Cin; int64_t ldcin;
  float* C; int64_t ldc;
  int64_t off;              // mask diagonal offset
  int mask;
  int ntiles;
  const long long* fail;
};

__global__ void __launch_bounds__(t32::THREADS, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                   const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, Tf32Params p) {
  using namespace t32;
  if (p.fail && failed(p.fail)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);   // SW128 atoms: 1 KB aligned
  uint8_t* sA = smem;                                   // [STAGES][A_BYTES]
  uint8_t* sB = smem + STAGES * A_BYTES;                // [STAGES][B_BYTES]
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;                     // [2]
  uint64_t* tempty = tfull + 2;                         // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh); tma_prefetch_desc(&mAl); tma_prefetch_desc(&mBh); tma_prefetch_desc(&mBl);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int TM = (int)((p.M + BM - 1) / BM), TN = (int)((p.N + BN - 1) / BN);
  const int nkb = (int)((p.K + BK - 1) / BK);          // k-blocks per product
  const int nkb3 = 3 * nkb;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        int ti, tj;
        TT::tile_of(p.mask, t, TM, TN, p.off, ti, tj);
        const int ya = (int)(p.a_row0 + (int64_t)ti * BM), yb = (int)(p.b_row0 + (int64_t)tj * BN);
        for (int kb = 0; kb < nkb3; ++kb) {
          const int prod = kb / nkb, kx = (kb - prod * nkb) * BK;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          // products: hi*hi, hi*lo, lo*hi
          tma_load_2d(sA + stage * A_BYTES, prod < 2 ? &mAh : &mAl, &full[stage], kx, ya);
          tma_load_2d(sB + stage * B_BYTES, prod == 1 ? &mBl : &mBh, &full[stage], kx, yb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      int stage = 0; uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t use = (uint32_t)(local >> 1) & 1;
        mbar_wait(&tempty[acc], use ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nkb3; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES), b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            // advance along K inside the 128-byte swizzle row: 32 bytes per instruction
            umma_tf32(d, umma_desc_sw128(a0 + k * UMMA_K * 4), umma_desc_sw128(b0 + k * UMMA_K * 4), idesc,
                      (kb | k) != 0);
          }
          umma_commit(&empty[stage]);          // frees the smem stage when these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);              // accumulator complete
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 -> TMEM lanes 32*(warp%4) .. +31
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int local = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++local) {
      int ti, tj;
      TT::tile_of(p.mask, t, TM, TN, p.off, ti, tj);
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1) & 1;
      mbar_wait(&tfull[acc], use);
      tc_fence_after();
      const int64_t i = (int64_t)ti * BM + q * 32 + lane;
      const int64_t j0 = (int64_t)tj * BN;
      for (int c = 0; c < BN; c += 32) {
        if (j0 + c >= p.N) break;
        float v[32];
        tmem_ld32(tmem + lane_base + (uint32_t)(acc * BN + c), v);
        if (i < p.M) {
          float cin[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int64_t j = j0 + c + u;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            cin[u] = in ? __ldcg(p.Cin + i + j * p.ldcin) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int64_t j = j0 + c + u;
            const bool in = j < p.N && (p.mask == kMaskNone || (p.mask == kMaskLower ? i >= j + p.off : i <= j + p.off));
            if (in) __stcg(p.C + i + j * p.ldc, cin[u] - v[u]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
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
// box = BK columns x box_rows rows, 128-byte swizzle; out-of-range elements read as zero.
static cudaError_t make_map(CUtensorMap* map, const float* base, int64_t k, int64_t rows, int64_t ldk, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldk * 4};
  cuuint32_t box[2] = {(cuuint32_t)t32::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t gemm_tf32x3(const Tf32Gemm& g, cudaStream_t st) {
  using namespace t32;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaSuccess;
  if ((g.ldk_a % 4) || (g.ldk_b % 4) || ((uintptr_t)g.Ah % 16) || ((uintptr_t)g.Al % 16) || ((uintptr_t)g.Bh % 16) ||
      ((uintptr_t)g.Bl % 16))
    return cudaErrorInvalidValue;   // TMA: 16-byte aligned bases and row strides
  const int TM = (int)((g.M + BM - 1) / BM), TN = (int)((g.N + BN - 1) / BN);
  const int ntiles = TT::count(g.mask, TM, TN, g.off);
  if (ntiles == 0) return cudaSuccess;
  CUtensorMap mAh, mAl, mBh, mBl;
  cudaError_t e;
  // the maps start at the operands' first rows; TMA rows beyond M / N read zeros
  if ((e = make_map(&mAh, g.Ah, g.K, g.M, g.ldk_a, BM)) != cudaSuccess) return e;
  if ((e = make_map(&mAl, g.Al, g.K, g.M, g.ldk_a, BM)) != cudaSuccess) return e;
  if ((e = make_map(&mBh, g.Bh, g.K, g.N, g.ldk_b, BN)) != cudaSuccess) return e;
  if ((e = make_map(&mBl, g.Bl, g.K, g.N, g.ldk_b, BN)) != cudaSuccess) return e;
  static int sms = 0;
  static bool attr = false;
  if (!attr) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  Tf32Params p{g.M, g.N, g.K, 0, 0, g.Cin, g.ldcin, g.C, g.ldc, g.off, g.mask, ntiles, g.fail};
  const int grid = ntiles < sms ? ntiles : sms;
  gemm_tf32x3_kernel<<<grid, THREADS, SMEM, st>>>(mAh, mAl, mBh, mBl, p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace sf
