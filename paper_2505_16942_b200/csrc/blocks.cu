// Reference block-sparse state on the GPU (the paper's own pipeline,
// PAPER.md:938-974; corrvol sparse.py:262-408):
//   mask scatter  -> per query, the B-tile rectangle its support touches on
//                    the PADDED target grid, OR-ed into a per-source-tile
//                    bitmask row (<= 9 atomics per query instead of (2r+2)^2);
//   block indices -> newly = mask & ~cum, popcount + exclusive scan gives
//                    row-major ids appended after the store's `used`;
//   sampled MMM   -> one 64x64 SIMT tile per (block, sub-tile), padded
//                    patch-major tiles formed on the fly (zero rows);
//   gather+sample -> proxy (2r+2)^2 patch from the store, canonical combine.
// Used for reference-compatible state/counters and as the paper-literal
// partial mode; bit-exact with the reference in STRICT mode.
#include "gemm.cuh"

namespace cvb {

__global__ void mask_kernel(const void* __restrict__ coords, bool f64, int h1, int w1, int level,
                            int radius, int block, int pth, int ptw, int tiles_x_src,
                            int tiles_x_tgt, uint32_t* __restrict__ mask, int64_t wpr) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= (int64_t)h1 * w1) return;
  const int py = (int)(p / w1), px = (int)(p % w1);
  double x, y;
  load_coord(coords, f64, p, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const long long ylo = max(lp.y0 - radius, 0LL), yhi = min(lp.y0 + radius + 1, (long long)pth - 1);
  const long long xlo = max(lp.x0 - radius, 0LL), xhi = min(lp.x0 + radius + 1, (long long)ptw - 1);
  if (ylo > yhi || xlo > xhi) return;
  const int64_t s = (int64_t)(py / block) * tiles_x_src + px / block;
  uint32_t* row = mask + s * wpr;
  for (long long by = ylo / block; by <= yhi / block; ++by)
    for (long long bx = xlo / block; bx <= xhi / block; ++bx) {
      const int64_t t = by * tiles_x_tgt + bx;
      atomicOr(row + (t >> 5), 1u << (t & 31));
    }
}

constexpr int SCAN_BLOCK = 1024;

__global__ void popc_reduce_kernel(const uint32_t* __restrict__ mask,
                                   const uint32_t* __restrict__ cum, int64_t n,
                                   long long* __restrict__ block_sums) {
  __shared__ long long s[SCAN_BLOCK / 32];
  const int64_t i = blockIdx.x * (int64_t)SCAN_BLOCK + threadIdx.x;
  long long c = (i < n) ? __popc(mask[i] & ~cum[i]) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    c = s[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = c;
  }
}

// exclusive scan of block sums in place (single CTA, sequential carry); total -> *count_out
__global__ void scan_sums_kernel(long long* __restrict__ sums, int64_t nb,
                                 long long* __restrict__ count_out) {
  __shared__ long long s[SCAN_BLOCK];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += SCAN_BLOCK) {
    const int64_t i = base + threadIdx.x;
    const long long v = (i < nb) ? sums[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < SCAN_BLOCK; o <<= 1) {
      const long long t = (threadIdx.x >= o) ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) sums[i] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += s[SCAN_BLOCK - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count_out = carry;
}

__global__ void assign_ids_kernel(const uint32_t* __restrict__ mask, uint32_t* __restrict__ cum,
                                  int64_t n, int64_t wpr, int64_t n_tgt, int64_t used,
                                  const long long* __restrict__ block_offs,
                                  long long* __restrict__ block_ids,
                                  long long* __restrict__ positions, int64_t max_positions) {
  __shared__ long long s[SCAN_BLOCK];
  const int64_t i = blockIdx.x * (int64_t)SCAN_BLOCK + threadIdx.x;
  const uint32_t m = (i < n) ? mask[i] : 0u;
  uint32_t newly = (i < n) ? (m & ~cum[i]) : 0u;
  const long long c = __popc(newly);
  s[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < SCAN_BLOCK; o <<= 1) {
    const long long t = (threadIdx.x >= o) ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i >= n) return;
  long long rank = block_offs[blockIdx.x] + s[threadIdx.x] - c;
  const int64_t row = i / wpr, word = i % wpr;
  while (newly) {
    const int b = __ffs(newly) - 1;
    newly &= newly - 1;
    const int64_t pos = row * n_tgt + word * 32 + b;
    block_ids[pos] = used + rank;
    if (rank < max_positions) positions[rank] = pos;
    ++rank;
  }
  cum[i] |= m;
}

template <bool STRICT>
__global__ void __launch_bounds__(GEMM_THREADS)
    sampled_mmm_kernel(const float* __restrict__ f1, int h1, int w1, int d,
                       const float* __restrict__ f2l, int th, int tw, int block, int tiles_x_src,
                       int tiles_x_tgt, int64_t n_tgt, const long long* __restrict__ positions,
                       float* __restrict__ store, int64_t first_id, int sub_n, bool vec) {
  __shared__ __align__(16) float smem[GEMM_SMEM_FLOATS];
  const int64_t i = blockIdx.x;
  const int sub = blockIdx.y;
  const int su = sub / sub_n, sv = sub % sub_n;
  const long long pos = positions[i];
  const int64_t s = pos / n_tgt, t = pos % n_tgt;
  const int sy = (int)(s / tiles_x_src), sx = (int)(s % tiles_x_src);
  const int ty = (int)(t / tiles_x_tgt), tx = (int)(t % tiles_x_tgt);
  const int b2 = block * block;
  const float* rowsA[2];
  const float* rowsB[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int r = (threadIdx.x >> 3) + 32 * k;
    const int u = su * GT + r, v = sv * GT + r;
    rowsA[k] = nullptr;
    rowsB[k] = nullptr;
    if (u < b2) {
      const int py = sy * block + u / block, px = sx * block + u % block;
      if (py < h1 && px < w1) rowsA[k] = f1 + ((int64_t)py * w1 + px) * d;
    }
    if (v < b2) {
      const int cy = ty * block + v / block, cx = tx * block + v % block;
      if (cy < th && cx < tw) rowsB[k] = f2l + ((int64_t)cy * tw + cx) * d;
    }
  }
  float acc[4][4];
  gemm_tile_64x64<STRICT>(rowsA, rowsB, d, vec, smem, acc);
  float* out = store + (first_id + i) * (int64_t)b2 * b2;
  const int tcol = threadIdx.x & 15, trow = threadIdx.x >> 4;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int u = su * GT + trow * 4 + a;
    if (u >= b2) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int v = sv * GT + tcol * 4 + b;
      if (v < b2) out[(int64_t)u * b2 + v] = acc[a][b];
    }
  }
}

template <bool STRICT>
__global__ void __launch_bounds__(128)
    block_gather_kernel(const void* __restrict__ coords, bool f64, int h1, int w1, int level,
                        int levels, int radius, int block, int pth, int ptw, int tiles_x_src,
                        int tiles_x_tgt, int64_t n_tgt, const long long* __restrict__ block_ids,
                        const float* __restrict__ store, float scale, bool normalize,
                        float* __restrict__ out, int* __restrict__ miss_flag) {
  extern __shared__ float bg_smem[];
  const int S = 2 * radius + 2, K = 2 * radius + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 4 + warp;
  if (p >= (int64_t)h1 * w1) return;
  float* patch = bg_smem + warp * S * S;
  const int py = (int)(p / w1), px = (int)(p % w1);
  const int64_t s = (int64_t)(py / block) * tiles_x_src + px / block;
  const int src_inner = (py % block) * block + px % block;
  const int64_t b2 = (int64_t)block * block;
  double x, y;
  load_coord(coords, f64, p, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const int ax = clamp_anchor(lp.x0, radius, ptw), ay = clamp_anchor(lp.y0, radius, pth);
  for (int c = lane; c < S * S; c += 32) {
    const int ty = ay - radius + c / S, tx = ax - radius + c % S;
    float v = 0.f;
    if (ty >= 0 && ty < pth && tx >= 0 && tx < ptw) {
      const int64_t tb = (int64_t)(ty / block) * tiles_x_tgt + tx / block;
      const long long bid = block_ids[s * n_tgt + tb];
      if (bid < 0) {
        atomicExch(miss_flag, 1);
      } else {
        v = __ldg(store + bid * b2 * b2 + (int64_t)src_inner * b2 + (ty % block) * block +
                  tx % block);
      }
    }
    patch[c] = v;
  }
  __syncwarp();
  const Weights64 w64 = weights64(lp.fx, lp.fy);
  const Weights32 w32 = weights32(lp.fx, lp.fy);
  float* o = out + (p * levels + level) * (int64_t)(K * K);
  for (int t = lane; t < K * K; t += 32)
    o[t] = tap_from_patch<STRICT>(patch, S, t / K, t % K, w64, w32, scale, normalize);
}

// Reference-model block accounting for the tile path (sparse.py:293-309 and
// :426-430 without the ids): newly = mask & ~cum (cum cleared first when the
// cache is off), cum |= mask, union |= mask; the newly bits are added to the
// run total and to the level's store count.  One warp-reduced atomic per warp.
__global__ void __launch_bounds__(256)
    mask_accumulate_kernel(const uint32_t* __restrict__ mask, uint32_t* __restrict__ cum,
                           uint32_t* __restrict__ uni, int64_t n, bool reset,
                           unsigned long long* __restrict__ total,
                           unsigned long long* __restrict__ level_used) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t m = mask[i];
    const uint32_t old = reset ? 0u : cum[i];
    c += __popc(m & ~old);
    cum[i] = old | m;
    if (uni != nullptr) uni[i] |= m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c != 0) {
    if (total != nullptr) atomicAdd(total, c);
    if (level_used != nullptr) atomicAdd(level_used, c);
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_computation_mask(const void* coords, int32_t h1, int32_t w1, int32_t level, int32_t radius,
                         int32_t block, int32_t pth, int32_t ptw, int32_t flags, uint32_t* mask,
                         int64_t words_per_row, void* stream) {
  CVB_REQUIRE(block >= 1 && radius >= 0 && level >= 0, "bad block/radius/level");
  CVB_REQUIRE(pth % block == 0 && ptw % block == 0, "padded extents must be multiples of block");
  const int64_t n_tgt = (int64_t)(pth / block) * (ptw / block);
  CVB_REQUIRE(words_per_row * 32 >= n_tgt, "mask row too short");
  const int64_t p = (int64_t)h1 * w1;
  if (p == 0) return CVB_OK;
  CVB_REQUIRE(coords && mask, "computation_mask: null pointer");
  const int tiles_x_src = (int)ceil_div(w1, block);
  mask_kernel<<<(unsigned)ceil_div(p, 256), 256, 0, as_stream(stream)>>>(
      coords, flags & CVB_COORDS_F64, h1, w1, level, radius, block, pth, ptw, tiles_x_src,
      ptw / block, mask, words_per_row);
  return check_launch("computation_mask");
}

int cvb_mask_accumulate(const uint32_t* mask, uint32_t* mask_cum, uint32_t* mask_union,
                        int64_t n_words, int32_t reset_cum, unsigned long long* total_count,
                        unsigned long long* level_count, void* stream) {
  CVB_REQUIRE(n_words >= 0, "mask_accumulate: bad size");
  cudaStream_t s = as_stream(stream);
  if (reset_cum && level_count != nullptr) cudaMemsetAsync(level_count, 0, sizeof(*level_count), s);
  if (n_words == 0) return check_launch("mask_accumulate");
  CVB_REQUIRE(mask && mask_cum, "mask_accumulate: null pointer");
  const int64_t blocks = ceil_div(n_words, 256);
  mask_accumulate_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, s>>>(
      mask, mask_cum, mask_union, n_words, reset_cum != 0, total_count, level_count);
  return check_launch("mask_accumulate");
}

int64_t cvb_block_indices_workspace(int64_t total_words) {
  return (ceil_div(total_words, SCAN_BLOCK) + 1) * (int64_t)sizeof(long long);
}

int cvb_block_indices(const uint32_t* mask, uint32_t* cum, int64_t rows, int64_t words_per_row,
                      int64_t n_tgt, int64_t used, int64_t* block_ids, int64_t* positions,
                      int64_t max_positions, int64_t* count_out, void* scan_ws, void* stream) {
  CVB_REQUIRE(rows >= 0 && words_per_row >= 0 && used >= 0, "block_indices: bad sizes");
  CVB_REQUIRE(words_per_row * 32 >= n_tgt, "mask row too short");
  CVB_REQUIRE(count_out && scan_ws, "block_indices: null pointer");
  const int64_t n = rows * words_per_row;
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    cudaMemsetAsync(count_out, 0, sizeof(int64_t), s);
    return check_launch("block_indices");
  }
  CVB_REQUIRE(mask && cum && block_ids, "block_indices: null pointer");
  const int64_t nb = ceil_div(n, SCAN_BLOCK);
  long long* sums = reinterpret_cast<long long*>(scan_ws);
  popc_reduce_kernel<<<(unsigned)nb, SCAN_BLOCK, 0, s>>>(mask, cum, n, sums);
  int st = check_launch("block_indices/reduce");
  if (st != CVB_OK) return st;
  scan_sums_kernel<<<1, SCAN_BLOCK, 0, s>>>(sums, nb, reinterpret_cast<long long*>(count_out));
  st = check_launch("block_indices/scan");
  if (st != CVB_OK) return st;
  assign_ids_kernel<<<(unsigned)nb, SCAN_BLOCK, 0, s>>>(
      mask, cum, n, words_per_row, n_tgt, used, sums, reinterpret_cast<long long*>(block_ids),
      reinterpret_cast<long long*>(positions), positions ? max_positions : 0);
  return check_launch("block_indices/assign");
}

int cvb_sampled_block_mmm(const float* f1, int32_t h1, int32_t w1, int32_t d, const float* f2l,
                          int32_t th, int32_t tw, int32_t block, int32_t tiles_x_src,
                          int32_t tiles_x_tgt, int64_t n_tgt, const int64_t* positions, int64_t k,
                          float* store, int64_t first_id, int32_t flags, void* stream) {
  CVB_REQUIRE(block >= 1 && d >= 1, "sampled_block_mmm: bad block/dims");
  if (k == 0) return CVB_OK;
  CVB_REQUIRE(f1 && f2l && positions && store, "sampled_block_mmm: null pointer");
  CVB_REQUIRE(k <= 2147483647LL, "too many blocks in one call");
  const int b2 = block * block;
  const int sub_n = (int)ceil_div(b2, GT);
  CVB_REQUIRE(sub_n * sub_n <= 65535, "block too large");
  const bool vec = (d % 4 == 0) && (((uintptr_t)f1 & 15) == 0) && (((uintptr_t)f2l & 15) == 0);
  dim3 grid((unsigned)k, (unsigned)(sub_n * sub_n));
  cudaStream_t s = as_stream(stream);
  const long long* pos = reinterpret_cast<const long long*>(positions);
  if (flags & CVB_STRICT)
    sampled_mmm_kernel<true><<<grid, GEMM_THREADS, 0, s>>>(f1, h1, w1, d, f2l, th, tw, block,
                                                           tiles_x_src, tiles_x_tgt, n_tgt, pos,
                                                           store, first_id, sub_n, vec);
  else
    sampled_mmm_kernel<false><<<grid, GEMM_THREADS, 0, s>>>(f1, h1, w1, d, f2l, th, tw, block,
                                                            tiles_x_src, tiles_x_tgt, n_tgt, pos,
                                                            store, first_id, sub_n, vec);
  return check_launch("sampled_block_mmm");
}

int cvb_block_gather_sample(const void* coords, int32_t h1, int32_t w1, int32_t level,
                            int32_t levels, int32_t radius, int32_t block, int32_t pth,
                            int32_t ptw, int32_t tiles_x_src, int32_t tiles_x_tgt, int64_t n_tgt,
                            const int64_t* block_ids, const float* store, float scale, float* out,
                            int32_t* miss_flag, int32_t flags, void* stream) {
  CVB_REQUIRE(radius >= 0 && radius <= 30 && block >= 1, "bad radius/block");
  CVB_REQUIRE(level >= 0 && level < levels, "bad level");
  const int64_t p = (int64_t)h1 * w1;
  if (p == 0) return CVB_OK;
  CVB_REQUIRE(coords && block_ids && out && miss_flag, "block_gather_sample: null pointer");
  const int S = 2 * radius + 2;
  const size_t smem = (size_t)4 * S * S * sizeof(float);
  const unsigned grid = (unsigned)ceil_div(p, 4);
  const bool f64 = flags & CVB_COORDS_F64;
  const long long* ids = reinterpret_cast<const long long*>(block_ids);
  cudaStream_t s = as_stream(stream);
  if (flags & CVB_STRICT)
    block_gather_kernel<true><<<grid, 128, smem, s>>>(coords, f64, h1, w1, level, levels, radius,
                                                      block, pth, ptw, tiles_x_src, tiles_x_tgt,
                                                      n_tgt, ids, store, scale, scale != 1.0f,
                                                      out, miss_flag);
  else
    block_gather_kernel<false><<<grid, 128, smem, s>>>(coords, f64, h1, w1, level, levels, radius,
                                                       block, pth, ptw, tiles_x_src, tiles_x_tgt,
                                                       n_tgt, ids, store, scale, scale != 1.0f,
                                                       out, miss_flag);
  return check_launch("block_gather_sample");
}

}  // extern "C"
