// Partial (incremental) correlation-volume sampler — the north-star path.
//
// Replaces the per-iteration body of sample_iteration (sparse.py:411-452):
//   mask scatter -> block ids -> sampled block MMM -> proxy gather -> combine
// with a B200-first decomposition over 8x8 query tiles:
//
//  K1 partial_contract_kernel   (north-star subsystems 2, 3, 4)
//     window-union tiler: per (tile, level) the bounding box B_t of the
//     tile's (2r+2)^2 supports (offsets -r..r+1 around floor(x/2^l),
//     sparse.py:279) clipped to the level grid — cells outside the grid are
//     dots with zero vectors, i.e. exactly 0 (layout.py:1-14), so they are
//     never computed.  Incremental cache: only B_t \ B_{t-1} (<= 4
//     rectangles) is contracted, as a dense [64 queries x 64 cells x D] tile
//     GEMM; results go to a toroidal cap_h x cap_w slot window
//     slot(y,x) = (y mod cap_h)*cap_w + (x mod cap_w), 64 query floats per
//     slot.  Cells of B_t ∩ B_{t-1} keep their slots (two distinct cells of a
//     box that fits the cap never share a slot), so the cache needs no copy
//     when the window slides.  Boxes that exceed the cap are flagged and
//     evaluated directly by K2.
//  K2 partial_sample_kernel     (north-star subsystem 5)
//     per query row of the tile (one warp, 8 queries): the union of the 8
//     supports is streamed from the cache in 32-byte sectors (8 queries x
//     4 B per slot), scattered into per-query (2r+2)^2 patches in shared
//     memory, and combined into (2r+1)^2 taps (canonical fp64 association
//     in STRICT mode, _pykernels.py:99-115), written coalesced per query.
#include "gemm.cuh"

namespace cvb {

constexpr int TQH = CVB_TILE_H, TQW = CVB_TILE_W, TQ = TQH * TQW;  // 64 queries
constexpr int ST_OK = 0, ST_OVERFLOW = 1, ST_EMPTY = 2;

struct PartialParams {
  const float* f1;
  int h1, w1, d, levels, radius;
  const float* f2[CVB_MAX_LEVELS];
  float* cache[CVB_MAX_LEVELS];
  int th[CVB_MAX_LEVELS], tw[CVB_MAX_LEVELS], ch[CVB_MAX_LEVELS], cw[CVB_MAX_LEVELS];
  const void* coords;
  int32_t* meta;
  unsigned long long* counters;
  int tiles_x;
  int64_t n_tiles;
  float scale;
  bool f64, normalize, no_cache, vec;
};

struct Box {
  int ylo, yhi, xlo, xhi;
  __device__ bool empty() const { return ylo > yhi || xlo > xhi; }
  __device__ int h() const { return yhi - ylo + 1; }
  __device__ int w() const { return xhi - xlo + 1; }
  __device__ int64_t area() const { return empty() ? 0 : (int64_t)h() * w(); }
};

// idx-th cell of B \ I in a fixed order (top band, bottom band, left, right).
// I is empty or contained in B.
__device__ __forceinline__ void new_cell(const Box& B, const Box& I, bool has_i, int idx, int& cy,
                                         int& cx) {
  const int wB = B.w();
  if (!has_i) {
    cy = B.ylo + idx / wB;
    cx = B.xlo + idx % wB;
    return;
  }
  const int n1 = (I.ylo - B.ylo) * wB;
  if (idx < n1) {
    cy = B.ylo + idx / wB;
    cx = B.xlo + idx % wB;
    return;
  }
  idx -= n1;
  const int n2 = (B.yhi - I.yhi) * wB;
  if (idx < n2) {
    cy = I.yhi + 1 + idx / wB;
    cx = B.xlo + idx % wB;
    return;
  }
  idx -= n2;
  const int wl = I.xlo - B.xlo;
  const int n3 = I.h() * wl;
  if (idx < n3) {
    cy = I.ylo + idx / wl;
    cx = B.xlo + idx % wl;
    return;
  }
  idx -= n3;
  const int wr = B.xhi - I.xhi;
  cy = I.ylo + idx / wr;
  cx = I.xhi + 1 + idx % wr;
}

__device__ __forceinline__ int slot_of(int cy, int cx, int ch, int cw) {
  return (cy % ch) * cw + (cx % cw);
}

template <bool STRICT>
__global__ void __launch_bounds__(GEMM_THREADS) partial_contract_kernel(PartialParams P) {
  __shared__ __align__(16) float smem[GEMM_SMEM_FLOATS];
  __shared__ int s_red[4];  // min_ay, max_ay, min_ax, max_ax
  __shared__ int s_nvalid;
  __shared__ Box s_B, s_I;
  __shared__ int s_has_i, s_n_new;

  const int64_t tile = blockIdx.x;
  const int level = blockIdx.y;
  const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
  const int th = P.th[level], tw = P.tw[level], r = P.radius;
  const int tid = threadIdx.x;

  if (tid == 0) {
    s_red[0] = INT_MAX;
    s_red[1] = INT_MIN;
    s_red[2] = INT_MAX;
    s_red[3] = INT_MIN;
    s_nvalid = 0;
  }
  __syncthreads();
  if (tid < TQ) {
    const int py = tile_y * TQH + tid / TQW, px = tile_x * TQW + tid % TQW;
    if (py < P.h1 && px < P.w1) {
      double x, y;
      load_coord(P.coords, P.f64, (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, level);
      const int ay = clamp_anchor(lp.y0, r, th), ax = clamp_anchor(lp.x0, r, tw);
      atomicMin(&s_red[0], ay);
      atomicMax(&s_red[1], ay);
      atomicMin(&s_red[2], ax);
      atomicMax(&s_red[3], ax);
      atomicAdd(&s_nvalid, 1);
    }
  }
  __syncthreads();
  int32_t* meta = P.meta + (tile * P.levels + level) * CVB_META_INTS;
  if (tid == 0) {
    Box B;
    B.ylo = max(s_red[0] - r, 0);
    B.yhi = min(s_red[1] + r + 1, th - 1);
    B.xlo = max(s_red[2] - r, 0);
    B.xhi = min(s_red[3] + r + 1, tw - 1);
    int status = ST_OK;
    if (s_nvalid == 0 || B.empty()) {
      status = ST_EMPTY;
      B = Box{1, 0, 1, 0};
    } else if (B.h() > P.ch[level] || B.w() > P.cw[level]) {
      status = ST_OVERFLOW;
    }
    Box prev{meta[0], meta[1], meta[2], meta[3]};
    const bool prev_ok = !P.no_cache && meta[4] == ST_OK && !prev.empty();
    Box I{max(B.ylo, prev.ylo), min(B.yhi, prev.yhi), max(B.xlo, prev.xlo),
          min(B.xhi, prev.xhi)};
    const bool has_i = status == ST_OK && prev_ok && !I.empty();
    const int n_new = status == ST_OK ? (int)(B.area() - (has_i ? I.area() : 0)) : 0;
    s_B = B;
    s_I = I;
    s_has_i = has_i;
    s_n_new = n_new;
    meta[0] = B.ylo;
    meta[1] = B.yhi;
    meta[2] = B.xlo;
    meta[3] = B.xhi;
    meta[4] = status;
    meta[5] = n_new;
    if (P.counters != nullptr) {
      if (n_new > 0) {
        atomicAdd(P.counters + 0, (unsigned long long)n_new * s_nvalid);
        atomicAdd(P.counters + 1, (unsigned long long)n_new);
      }
      if (status == ST_OVERFLOW) atomicAdd(P.counters + 2, 1ULL);
      if (status == ST_EMPTY) atomicAdd(P.counters + 3, 1ULL);
    }
  }
  __syncthreads();
  const int n_new = s_n_new;
  if (n_new == 0) return;
  const Box B = s_B, I = s_I;
  const bool has_i = s_has_i;
  const int ch = P.ch[level], cw = P.cw[level];
  const float* f2 = P.f2[level];
  float* cache = P.cache[level] + tile * (int64_t)(ch * cw) * TQ;
  const int d = P.d;

  const float* rowsA[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int q = (tid >> 3) + 32 * s;
    const int py = tile_y * TQH + q / TQW, px = tile_x * TQW + q % TQW;
    rowsA[s] = (py < P.h1 && px < P.w1) ? P.f1 + ((int64_t)py * P.w1 + px) * d : nullptr;
  }
  const int tx = tid & 15, ty = tid >> 4;
  for (int c0 = 0; c0 < n_new; c0 += GT) {
    const float* rowsB[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int idx = c0 + (tid >> 3) + 32 * s;
      rowsB[s] = nullptr;
      if (idx < n_new) {
        int cy, cx;
        new_cell(B, I, has_i, idx, cy, cx);
        rowsB[s] = f2 + ((int64_t)cy * tw + cx) * d;
      }
    }
    float acc[4][4];
    gemm_tile_64x64<STRICT>(rowsA, rowsB, d, P.vec, smem, acc);
    // acc[i][j]: query ty*4+i, cell c0 + tx*4 + j
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = c0 + tx * 4 + j;
      if (idx >= n_new) continue;
      int cy, cx;
      new_cell(B, I, has_i, idx, cy, cx);
      float4 v = make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
      *reinterpret_cast<float4*>(cache + (int64_t)slot_of(cy, cx, ch, cw) * TQ + ty * 4) = v;
    }
  }
}

template <bool STRICT>
__global__ void __launch_bounds__(256) partial_sample_kernel(PartialParams P, float* out) {
  extern __shared__ __align__(16) float ps_smem[];
  const int r = P.radius, S = 2 * r + 2, K = 2 * r + 1, SS = S * S, KK = K * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = blockIdx.x;
  const int level = blockIdx.y;
  const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
  const int th = P.th[level], tw = P.tw[level];
  const int py = tile_y * TQH + warp;
  if (py >= P.h1) return;  // warp-uniform

  // per-warp shared state: patches [8][SS], anchors, weights
  float* patch = ps_smem + warp * (TQW * SS);
  int* s_ay = reinterpret_cast<int*>(ps_smem + 8 * TQW * SS) + warp * (4 * TQW);
  int* s_ax = s_ay + TQW;
  int* s_valid = s_ax + TQW;
  double* s_fx = reinterpret_cast<double*>(ps_smem + 8 * TQW * SS + 8 * 4 * TQW) + warp * 2 * TQW;
  double* s_fy = s_fx + TQW;

  for (int c = lane; c < TQW * SS; c += 32) patch[c] = 0.f;
  int ay = 0, ax = 0, valid = 0;
  if (lane < TQW) {
    const int px = tile_x * TQW + lane;
    valid = px < P.w1;
    if (valid) {
      double x, y;
      load_coord(P.coords, P.f64, (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, level);
      ay = clamp_anchor(lp.y0, r, th);
      ax = clamp_anchor(lp.x0, r, tw);
      s_fx[lane] = lp.fx;
      s_fy[lane] = lp.fy;
    }
    s_ay[lane] = ay;
    s_ax[lane] = ax;
    s_valid[lane] = valid;
  }
  // warp union of supports, clipped to the grid
  int ylo = valid ? ay - r : INT_MAX, yhi = valid ? ay + r + 1 : INT_MIN;
  int xlo = valid ? ax - r : INT_MAX, xhi = valid ? ax + r + 1 : INT_MIN;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
    yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
    xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
    xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, o));
  }
  __syncwarp();
  const int32_t* meta = P.meta + (tile * P.levels + level) * CVB_META_INTS;
  const int status = meta[4];
  const int q = lane & 7, sub = lane >> 3;
  const int qay = s_ay[q], qax = s_ax[q], qvalid = s_valid[q];
  ylo = max(ylo, 0);
  yhi = min(yhi, th - 1);
  xlo = max(xlo, 0);
  xhi = min(xhi, tw - 1);
  if (status == ST_OK && ylo <= yhi && xlo <= xhi) {
    const int ch = P.ch[level], cw = P.cw[level];
    const float* cache = P.cache[level] + tile * (int64_t)(ch * cw) * TQ + warp * TQW;
    const int rw = xhi - xlo + 1;
    const int n = (yhi - ylo + 1) * rw;
    for (int c = sub; c < n; c += 4) {
      const int cy = ylo + c / rw, cx = xlo + c % rw;
      const float v = __ldg(cache + (int64_t)slot_of(cy, cx, ch, cw) * TQ + q);
      const int j = cy - (qay - r), i = cx - (qax - r);
      if (qvalid && j >= 0 && j < S && i >= 0 && i < S) patch[q * SS + j * S + i] = v;
    }
  } else if (status == ST_OVERFLOW) {
    // direct evaluation of each query's in-grid support cells
    const int d = P.d;
    const float* f2 = P.f2[level];
    for (int e = lane; e < TQW * SS; e += 32) {
      const int qq = e / SS, c = e % SS;
      if (!s_valid[qq]) continue;
      const int cy = s_ay[qq] - r + c / S, cx = s_ax[qq] - r + c % S;
      if (cy < 0 || cy >= th || cx < 0 || cx >= tw) continue;
      const float* a = P.f1 + ((int64_t)py * P.w1 + tile_x * TQW + qq) * d;
      const float* b = f2 + ((int64_t)cy * tw + cx) * d;
      float acc = 0.f;
      for (int k = 0; k < d; ++k) acc = mac<STRICT>(acc, __ldg(a + k), __ldg(b + k));
      patch[e] = acc;
    }
  }
  __syncwarp();
  const int64_t row0 = (int64_t)py * P.w1 + tile_x * TQW;
  for (int e = lane; e < TQW * KK; e += 32) {
    const int qq = e / KK, t = e % KK;
    if (!s_valid[qq]) continue;
    const Weights64 w64 = weights64(s_fx[qq], s_fy[qq]);
    const Weights32 w32 = weights32(s_fx[qq], s_fy[qq]);
    out[((row0 + qq) * P.levels + level) * (int64_t)KK + t] = tap_from_patch<STRICT>(
        patch + qq * SS, S, t / K, t % K, w64, w32, P.scale, P.normalize);
  }
}

static size_t sample_smem_bytes(int radius) {
  const int S = 2 * radius + 2;
  return (size_t)8 * TQW * S * S * sizeof(float) + (size_t)8 * 4 * TQW * sizeof(int) +
         (size_t)8 * 2 * TQW * sizeof(double);
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_partial_sizes(const cvb_partial_desc* desc, int64_t* n_tiles, int64_t* meta_ints,
                      int64_t* cache_floats_per_level) {
  CVB_REQUIRE(desc, "partial_sizes: null desc");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  const int64_t nt = ceil_div(desc->h1, TQH) * ceil_div(desc->w1, TQW);
  if (n_tiles) *n_tiles = nt;
  if (meta_ints) *meta_ints = nt * desc->levels * CVB_META_INTS;
  if (cache_floats_per_level)
    for (int l = 0; l < desc->levels; ++l)
      cache_floats_per_level[l] = nt * (int64_t)desc->cap_h[l] * desc->cap_w[l] * TQ;
  return CVB_OK;
}

__global__ void reset_meta_kernel(int32_t* meta, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t* m = meta + i * CVB_META_INTS;
  m[0] = 1;
  m[1] = 0;
  m[2] = 1;
  m[3] = 0;
  m[4] = ST_EMPTY;
  m[5] = 0;
  m[6] = 0;
  m[7] = 0;
}

int cvb_partial_reset(const cvb_partial_desc* desc, int32_t* meta, void* stream) {
  int64_t nt = 0;
  int st = cvb_partial_sizes(desc, &nt, nullptr, nullptr);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(meta, "partial_reset: null meta");
  const int64_t n = nt * desc->levels;
  if (n == 0) return CVB_OK;
  reset_meta_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(meta, n);
  return check_launch("partial_reset");
}

static int build_params(const cvb_partial_desc* desc, const float* f1,
                        const float* const* f2_levels_host, const void* coords, float scale,
                        int32_t* meta, float* const* cache_levels_host,
                        unsigned long long* counters, int32_t flags, PartialParams& P) {
  CVB_REQUIRE(desc && f2_levels_host && cache_levels_host, "partial_sample: null argument");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  CVB_REQUIRE(desc->radius >= 0 && desc->radius <= 8, "partial sampler radius must be <= 8");
  CVB_REQUIRE(desc->d >= 1, "feature dims must be >= 1");
  CVB_REQUIRE(desc->h1 >= 0 && desc->w1 >= 0, "bad source dims");
  CVB_REQUIRE(f1 && coords && meta, "partial_sample: null pointer");
  P.f1 = f1;
  P.h1 = desc->h1;
  P.w1 = desc->w1;
  P.d = desc->d;
  P.levels = desc->levels;
  P.radius = desc->radius;
  bool vec = (desc->d % 4 == 0) && (((uintptr_t)f1 & 15) == 0);
  for (int l = 0; l < CVB_MAX_LEVELS; ++l) {
    const bool used = l < desc->levels;
    P.f2[l] = used ? f2_levels_host[l] : nullptr;
    P.cache[l] = used ? cache_levels_host[l] : nullptr;
    P.th[l] = used ? desc->th[l] : 0;
    P.tw[l] = used ? desc->tw[l] : 0;
    P.ch[l] = used ? desc->cap_h[l] : 1;
    P.cw[l] = used ? desc->cap_w[l] : 1;
    if (used) {
      CVB_REQUIRE(P.f2[l] && P.cache[l], "partial_sample: null level pointer");
      CVB_REQUIRE(P.th[l] >= 1 && P.tw[l] >= 1, "empty target level %d", l);
      CVB_REQUIRE(P.ch[l] >= 1 && P.cw[l] >= 1, "bad cache window at level %d", l);
      vec = vec && (((uintptr_t)P.f2[l] & 15) == 0);
    }
  }
  P.coords = coords;
  P.meta = meta;
  P.counters = counters;
  P.tiles_x = (int)ceil_div(desc->w1, TQW);
  P.n_tiles = ceil_div(desc->h1, TQH) * (int64_t)P.tiles_x;
  P.scale = scale;
  P.f64 = flags & CVB_COORDS_F64;
  P.normalize = scale != 1.0f;
  P.no_cache = flags & CVB_NO_CACHE;
  P.vec = vec;
  CVB_REQUIRE(P.n_tiles <= 2147483647LL, "too many tiles");
  return CVB_OK;
}

static int launch_contract(const PartialParams& P, int32_t flags, cudaStream_t s) {
  if (P.n_tiles == 0) return CVB_OK;
  dim3 grid((unsigned)P.n_tiles, (unsigned)P.levels);
  if (flags & CVB_STRICT)
    partial_contract_kernel<true><<<grid, GEMM_THREADS, 0, s>>>(P);
  else
    partial_contract_kernel<false><<<grid, GEMM_THREADS, 0, s>>>(P);
  return check_launch("partial_contract");
}

static int launch_gather(const PartialParams& P, float* out, int32_t flags, cudaStream_t s) {
  if (P.n_tiles == 0) return CVB_OK;
  CVB_REQUIRE(out, "partial_sample: null output");
  dim3 grid((unsigned)P.n_tiles, (unsigned)P.levels);
  const size_t smem = sample_smem_bytes(P.radius);
  if (flags & CVB_STRICT) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(partial_sample_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    partial_sample_kernel<true><<<grid, 256, smem, s>>>(P, out);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(partial_sample_kernel<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    partial_sample_kernel<false><<<grid, 256, smem, s>>>(P, out);
  }
  return check_launch("partial_sample");
}

int cvb_partial_sample(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       int32_t* meta, float* const* cache_levels_host, float* out,
                       unsigned long long* counters, int32_t flags, void* stream) {
  PartialParams P;
  int st = build_params(desc, f1, f2_levels_host, coords, scale, meta, cache_levels_host,
                        counters, flags, P);
  if (st != CVB_OK) return st;
  st = launch_contract(P, flags, as_stream(stream));
  if (st != CVB_OK) return st;
  return launch_gather(P, out, flags, as_stream(stream));
}

int cvb_partial_contract(const cvb_partial_desc* desc, const float* f1,
                         const float* const* f2_levels_host, const void* coords, int32_t* meta,
                         float* const* cache_levels_host, unsigned long long* counters,
                         int32_t flags, void* stream) {
  PartialParams P;
  int st = build_params(desc, f1, f2_levels_host, coords, 1.0f, meta, cache_levels_host,
                        counters, flags, P);
  if (st != CVB_OK) return st;
  return launch_contract(P, flags, as_stream(stream));
}

int cvb_partial_gather(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       const int32_t* meta, float* const* cache_levels_host, float* out,
                       int32_t flags, void* stream) {
  PartialParams P;
  int st = build_params(desc, f1, f2_levels_host, coords, scale, const_cast<int32_t*>(meta),
                        cache_levels_host, nullptr, flags, P);
  if (st != CVB_OK) return st;
  return launch_gather(P, out, flags, as_stream(stream));
}

}  // extern "C"
