// GPU access recorder / block occupancy (analyzer.py:31-116).
//
// The paper's Suppl. Table 1 study from real centroid traces, at any size:
// a (source, target) cell is touched iff some bilinear tap corner with
// nonzero weight lands on it in some iteration — offsets -r..r+1 around the
// level floor, the last row / column only when the fractional part is > 0,
// clipped to the (unpadded) level grid (analyzer.py:31-80).
//   * cvb_access_union: per query, the number of distinct touched cells
//     over all iterations (each window's cells not covered by an earlier
//     window of the same query), summed; optionally split by the iteration
//     that first touched them.  Equals the size of the reference AccessLog.
//   * cvb_access_blocks: ORs one iteration's touched (source group, target
//     group) pairs into a bitmask for a block size and layout
//     (row-major: B^2 consecutive raster indices; patch-major: B x B spatial
//     tiles, analyzer.py:83-97) — occupancy = popcount / positions.
#include "common.cuh"

namespace cvb {

struct Win {
  int y0, y1, x0, x1;  // inclusive touched rows / cols (clipped)
};

__device__ __forceinline__ Win touched_window(const void* coords, bool f64, int64_t p, int level,
                                              int r, int th, int tw, bool trim) {
  double x, y;
  load_coord(coords, f64, p, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const long long ylo = lp.y0 - r, xlo = lp.x0 - r;
  long long yhi = lp.y0 + r + 1, xhi = lp.x0 + r + 1;
  if (trim && !(lp.fy > 0.0)) --yhi;
  if (trim && !(lp.fx > 0.0)) --xhi;
  Win w;
  w.y0 = (int)max(ylo, 0LL);
  w.y1 = (int)min(yhi, (long long)th - 1);
  w.x0 = (int)max(xlo, 0LL);
  w.x1 = (int)min(xhi, (long long)tw - 1);
  return w;
}

struct Coords8 {
  const void* it[64];
};

__global__ void __launch_bounds__(256) access_union_kernel(Coords8 C, int n_iter, bool f64,
                                                           int64_t p_total, int level, int r,
                                                           int th, int tw, bool trim,
                                                           unsigned long long* first_touch) {
  __shared__ unsigned long long s_cnt[64];
  for (int i = threadIdx.x; i < n_iter; i += blockDim.x) s_cnt[i] = 0ULL;
  __syncthreads();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < p_total;
       p += (int64_t)gridDim.x * blockDim.x) {
    Win prev[64];
    for (int it = 0; it < n_iter; ++it) {
      const Win w = touched_window(C.it[it], f64, p, level, r, th, tw, trim);
      unsigned long long fresh = 0;
      if (w.y0 <= w.y1 && w.x0 <= w.x1) {
        for (int cy = w.y0; cy <= w.y1; ++cy)
          for (int cx = w.x0; cx <= w.x1; ++cx) {
            bool seen = false;
            for (int k = 0; k < it && !seen; ++k)
              seen = cy >= prev[k].y0 && cy <= prev[k].y1 && cx >= prev[k].x0 && cx <= prev[k].x1;
            fresh += !seen;
          }
      }
      prev[it] = w;
      if (fresh) atomicAdd(&s_cnt[it], fresh);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_iter; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(first_touch + i, s_cnt[i]);
}

__global__ void __launch_bounds__(256) access_blocks_kernel(const void* coords, bool f64, int h1,
                                                            int w1, int level, int r, int th,
                                                            int tw, int block, bool patch,
                                                            bool trim, uint32_t* mask,
                                                            int64_t wpr) {
  const int64_t p_total = (int64_t)h1 * w1;
  const int tiles_x_src = (w1 + block - 1) / block, tiles_x_tgt = (tw + block - 1) / block;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < p_total;
       p += (int64_t)gridDim.x * blockDim.x) {
    const Win w = touched_window(coords, f64, p, level, r, th, tw, trim);
    if (w.y0 > w.y1 || w.x0 > w.x1) continue;
    const int py = (int)(p / w1), px = (int)(p % w1);
    const int64_t gs = patch ? (int64_t)(py / block) * tiles_x_src + px / block
                             : p / ((int64_t)block * block);
    uint32_t* row = mask + gs * wpr;
    for (int cy = w.y0; cy <= w.y1; ++cy) {
      if (patch) {
        // one bit per touched target tile of this row
        const int t0 = w.x0 / block, t1 = w.x1 / block;
        for (int tx = t0; tx <= t1; ++tx) {
          const int64_t gt = (int64_t)(cy / block) * tiles_x_tgt + tx;
          atomicOr(row + (gt >> 5), 1u << (gt & 31));
        }
      } else {
        const int64_t b2 = (int64_t)block * block;
        const int64_t g0 = ((int64_t)cy * tw + w.x0) / b2, g1 = ((int64_t)cy * tw + w.x1) / b2;
        for (int64_t gt = g0; gt <= g1; ++gt) atomicOr(row + (gt >> 5), 1u << (gt & 31));
      }
    }
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_access_union(const void* const* coords_iters_host, int32_t n_iter, int32_t h1, int32_t w1,
                     int32_t level, int32_t radius, int32_t th, int32_t tw, int32_t flags,
                     unsigned long long* first_touch, void* stream) {
  CVB_REQUIRE(coords_iters_host && first_touch, "access_union: null pointer");
  CVB_REQUIRE(n_iter >= 1 && n_iter <= 64, "access_union: 1..64 iterations");
  CVB_REQUIRE(level >= 0 && level < 62 && radius >= 0 && th >= 1 && tw >= 1,
              "access_union: bad geometry");
  Coords8 C;
  for (int i = 0; i < n_iter; ++i) {
    CVB_REQUIRE(coords_iters_host[i], "access_union: null iteration pointer");
    C.it[i] = coords_iters_host[i];
  }
  const int64_t p = (int64_t)h1 * w1;
  if (p == 0) return CVB_OK;
  int64_t g = ceil_div(p, 256);
  if (g > 148 * 8) g = 148 * 8;
  access_union_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(
      C, n_iter, flags & CVB_COORDS_F64, p, level, radius, th, tw, !(flags & CVB_ACCESS_NO_TRIM),
      first_touch);
  return check_launch("access_union");
}

int cvb_access_blocks(const void* coords, int32_t h1, int32_t w1, int32_t level, int32_t radius,
                      int32_t th, int32_t tw, int32_t block, int32_t patch_major, int32_t flags,
                      uint32_t* mask, int64_t words_per_row, void* stream) {
  CVB_REQUIRE(coords && mask, "access_blocks: null pointer");
  CVB_REQUIRE(block >= 1 && level >= 0 && level < 62 && radius >= 0 && th >= 1 && tw >= 1,
              "access_blocks: bad geometry");
  const int64_t p = (int64_t)h1 * w1;
  if (p == 0) return CVB_OK;
  int64_t g = ceil_div(p, 256);
  if (g > 148 * 8) g = 148 * 8;
  access_blocks_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(
      coords, flags & CVB_COORDS_F64, h1, w1, level, radius, th, tw, block, patch_major != 0,
      !(flags & CVB_ACCESS_NO_TRIM), mask, words_per_row);
  return check_launch("access_blocks");
}

}  // extern "C"
