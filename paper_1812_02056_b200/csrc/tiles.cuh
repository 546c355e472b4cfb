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

// Host-built rasterization table (Tiles::make_raster): tile columns in groups of gb, gp[g] =
// number of masked tiles in columns [0, g*gb).  ngroups = 0: plain column order.
constexpr int kMaxRaster = 64;
struct Raster {
  int ngroups = 0, gb = 1, last_w = 1;
  int gp[kMaxRaster + 1];
};

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

  // Rasterized order for L2 reuse: tile columns in groups of GB; inside a group, row by
  // row.  The CTAs running at the same time then cover a compact band of ~(resident/GB)
  // tile rows x GB tile columns, so each operand row block fetched from HBM is reused by
  // GB tiles from L2 instead of being re-fetched for every tile column (the R rows of a
  // flush are far larger than L2 at n = 65536).  Same tile set as tile_of.
  __host__ __device__ static __forceinline__ bool needed(int mask, int ti, int tj, int TM, int64_t off) {
    if (mask == kMaskLower) return ti >= first_lower(tj, off);
    if (mask == kMaskUpper) return ti < count_upper(tj, TM, off);
    return true;
  }
  __host__ __device__ static __forceinline__ int rows_below(int mask, int R, int tj, int TM, int64_t off) {
    if (R > TM) R = TM;
    if (mask == kMaskLower) { const int f = first_lower(tj, off); return R > f ? R - f : 0; }
    if (mask == kMaskUpper) { const int c = count_upper(tj, TM, off); return R < c ? R : c; }
    return R;
  }
  __host__ __device__ static __forceinline__ int64_t cdiv(int64_t a, int64_t b) {   // ceil(a/b), b > 0
    return a >= 0 ? (a + b - 1) / b : -((-a) / b);
  }
  __host__ __device__ static __forceinline__ int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
  }
  // tiles of the group's columns [tj0, tj1) in rows < R — O(log) via floor_sum
  __host__ __device__ static __forceinline__ int64_t group_rows_prefix(int mask, int64_t R, int tj0, int tj1, int TM,
                                                                       int64_t off) {
    if (R > TM) R = TM;
    if (R <= 0) return 0;
    if (mask == kMaskNone) return R * (tj1 - tj0);
    if (mask == kMaskLower) {
      // columns with first_lower(j) < R form the prefix [tj0, js)
      const int64_t js = clampi(cdiv(R * BM - off, BN), tj0, tj1);
      return (js - tj0) * R - (floor_sum(js, BM, BN, off) - floor_sum(tj0, BM, BN, off));
    }
    // upper: min(R, count_upper(j)); columns with h(j) < R form the prefix [tj0, j1)
    const int64_t j1 = clampi(cdiv((R - 1) * BM - BN + 1 - off, BN), tj0, tj1);
    const int64_t sh = floor_sum(j1, BM, BN, BN - 1 + off) - floor_sum(tj0, BM, BN, BN - 1 + off) + (j1 - tj0);
    return sh + (tj1 - j1) * R;
  }
  __host__ __device__ static __forceinline__ void tile_of_grouped(int mask, int bid, int TM, int TN, int64_t off, int GB,
                                                                  int& ti, int& tj) {
    const int ngroups = (TN + GB - 1) / GB;
    int lo = 0, hi = ngroups;   // group: largest g with prefix(g*GB) <= bid
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix(mask, (int64_t)mid * GB, TM, TN, off) <= bid) lo = mid; else hi = mid;
    }
    const int tj0 = lo * GB, tj1 = (tj0 + GB < TN) ? tj0 + GB : TN;
    const int64_t b = bid - prefix(mask, tj0, TM, TN, off);
    int rl = 0, rh = TM;        // row: largest R with P(R) <= b
    while (rh - rl > 1) {
      const int mid = (rl + rh) >> 1;
      if (group_rows_prefix(mask, mid, tj0, tj1, TM, off) <= b) rl = mid; else rh = mid;
    }
    ti = rl;
    const int64_t k = b - group_rows_prefix(mask, rl, tj0, tj1, TM, off);
    // needed columns of row ti inside the group: a prefix (lower), a suffix (upper) or all
    int64_t first = tj0;
    if (mask == kMaskUpper) first = clampi(cdiv((int64_t)ti * BM - BN + 1 - off, BN), tj0, tj1);
    tj = (int)(first + k);
  }

  // ---- the same rasterized order with a host-built table of group prefixes: the kernel's
  // lookup is a short search plus <= ~GB*BN/BM rows of 32-bit arithmetic (no 64-bit
  // divisions on the CTA's critical path).
  __host__ __device__ static __forceinline__ int row_count(int mask, int r, int tj0, int W, int64_t off) {
    if (mask == kMaskLower) {   // needed columns: j <= tmax(r)
      const int64_t tmax = ((int64_t)(r + 1) * BM - off - 1);
      const int64_t c = (tmax < 0 ? -1 : tmax / BN) - tj0 + 1;
      return c < 0 ? 0 : (c > W ? W : (int)c);
    }
    if (mask == kMaskUpper) {   // needed columns: j >= tmin(r)
      int64_t tmin = cdiv((int64_t)r * BM - BN + 1 - off, BN);
      if (tmin < tj0) tmin = tj0;
      const int64_t c = tj0 + W - tmin;
      return c < 0 ? 0 : (int)c;
    }
    return W;
  }
  __host__ __device__ static __forceinline__ void tile_of_raster(int mask, int bid, int TM, int64_t off, const Raster& rs,
                                                        int& ti, int& tj) {
    int g = 0;
    while (g + 1 < rs.ngroups && rs.gp[g + 1] <= bid) ++g;
    const int tj0 = g * rs.gb;
    const int W = rs.gp[g + 1] == rs.gp[g] ? 1 : ((g + 1 == rs.ngroups) ? rs.last_w : rs.gb);
    int b = bid - rs.gp[g];
    if (mask == kMaskNone) { ti = b / W; tj = tj0 + b % W; return; }
    if (mask == kMaskLower) {
      int r = first_lower(tj0, off);
      const int rfull = first_lower(tj0 + W - 1, off);   // rows from here on are full
      for (; r < rfull; ++r) {
        const int c = row_count(mask, r, tj0, W, off);
        if (b < c) { ti = r; tj = tj0 + b; return; }
        b -= c;
      }
      ti = rfull + b / W; tj = tj0 + b % W;
      return;
    }
    // upper: full rows first, then the tail
    int64_t rf = ((int64_t)tj0 * BN + BN - 1 + off) / BM + 1;   // rows [0, rf) are full
    if (rf > TM) rf = TM;
    if (b < rf * W) { ti = b / W; tj = tj0 + b % W; return; }
    b -= (int)(rf * W);
    for (int r = (int)rf; r < TM; ++r) {
      const int c = row_count(mask, r, tj0, W, off);
      if (b < c) { ti = r; tj = tj0 + W - c + b; return; }
      b -= c;
    }
    ti = TM - 1; tj = tj0;   // unreachable for bid < count
  }
  static inline void make_raster(int mask, int TM, int TN, int64_t off, int gb, Raster& rs) {
    if ((TN + gb - 1) / gb > kMaxRaster) gb = (TN + kMaxRaster - 1) / kMaxRaster;
    rs.gb = gb;
    rs.ngroups = (TN + gb - 1) / gb;
    rs.last_w = TN - (rs.ngroups - 1) * gb;
    for (int g = 0; g <= rs.ngroups; ++g) rs.gp[g] = (int)prefix(mask, (int64_t)g * gb, TM, TN, off);
  }
};

}  // namespace sf
