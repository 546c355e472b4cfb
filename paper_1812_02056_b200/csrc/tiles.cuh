// tiles.cuh — enumeration of the C tiles a masked (triangular) update visits, shared by the
// FP64 DMMA kernel (gemm_f64.cu) and the TF32 tcgen05 kernel (gemm_tf32.cu).
//
// Tiles are BM x BN and enumerated column by column; tile column tj covers C columns
// [tj*BN, tj*BN+BN), tile row ti rows [ti*BM, ti*BM+BM).  The mask is relative to a diagonal
// offset `off` >= 0: lower keeps i >= j + off, upper keeps i <= j + off.
#pragma once
#include <stdint.h>

namespace sf {

enum { kMaskNone = 0, kMaskLower = 1, kMaskUpper = 2 };

// sum_{i=0}^{n-1} floor((a*i + b) / m) for a, b >= 0, m > 0 (Euclid-like reduction, O(log m)).
__host__ __device__ __forceinline__ int64_t floor_sum(int64_t n, int64_t m, int64_t a, int64_t b) {
  int64_t ans = 0;
  while (n > 0) {
    if (a >= m) { ans += (n - 1) * n / 2 * (a / m); a %= m; }
    if (b >= m) { ans += n * (b / m); b %= m; }
    const int64_t y = a * n + b;
    if (y < m) break;
    n = y / m; b = y % m;
    const int64_t t = m; m = a; a = t;
  }
  return ans;
}

template <int BM, int BN>
struct Tiles {
  // first tile row of tile column tj that meets the lower mask
  __host__ __device__ static __forceinline__ int first_lower(int tj, int64_t off) {
    const int64_t r = ((int64_t)tj * BN + off) / BM;
    return r > 0 ? (int)r : 0;
  }
  // number of tile rows of tile column tj that meet the upper mask
  __host__ __device__ static __forceinline__ int count_upper(int tj, int TM, int64_t off) {
    const int64_t c = ((int64_t)tj * BN + BN - 1 + off) / BM + 1;
    return c < TM ? (int)c : TM;
  }
  // masked tiles in tile columns [0, j): O(log), so a CTA finds its tile by binary search
  __host__ __device__ static __forceinline__ int64_t prefix(int mask, int64_t j, int TM, int TN, int64_t off) {
    if (j > TN) j = TN;
    if (mask == kMaskNone) return j * TM;
    if (mask == kMaskLower) {
      int64_t J = ((int64_t)TM * BM - off + BN - 1) / BN;   // columns with first_lower < TM
      if (J < 0) J = 0;
      if (J > TN) J = TN;
      if (j > J) j = J;
      return j * TM - floor_sum(j, BM, BN, off);
    }
    const int64_t num = (int64_t)(TM - 1) * BM - BN + 1 - off;   // h(t) >= TM  <=>  t*BN >= num
    int64_t t1 = num <= 0 ? 0 : (num + BN - 1) / BN;
    if (t1 > TN) t1 = TN;
    if (j <= t1) return floor_sum(j, BM, BN, BN - 1 + off) + j;
    return floor_sum(t1, BM, BN, BN - 1 + off) + t1 + (j - t1) * TM;
  }
  __host__ __device__ static __forceinline__ int count(int mask, int TM, int TN, int64_t off) {
    return (int)prefix(mask, TN, TM, TN, off);
  }
  __host__ __device__ static __forceinline__ void tile_of(int mask, int bid, int TM, int TN, int64_t off, int& ti,
                                                          int& tj) {
    if (mask == kMaskNone) { ti = bid % TM; tj = bid / TM; return; }
    int lo = 0, hi = TN;   // largest j with prefix(j) <= bid
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix(mask, mid, TM, TN, off) <= bid) lo = mid; else hi = mid;
    }
    tj = lo;
    const int r = bid - (int)prefix(mask, lo, TM, TN, off);
    ti = (mask == kMaskLower) ? first_lower(lo, off) + r : r;
  }
};

}  // namespace sf
