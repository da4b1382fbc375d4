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
#include "partial.cuh"

namespace cvb {

template <bool STRICT>
__global__ void __launch_bounds__(GEMM_THREADS) partial_contract_kernel(PartialParams P) {
  __shared__ __align__(16) float smem[GEMM_SMEM_FLOATS];
  __shared__ int s_red[5];
  __shared__ TilePlan s_plan;

  const int64_t tile = P.tile0 + blockIdx.x;
  const int level = blockIdx.y;
  const TileRef tr = tile_ref(P, tile);
  const int tile_y = tr.ty, tile_x = tr.tx;
  const int tw = P.tw[level];
  const int tid = threadIdx.x;
  plan_tile_level(P, tile, level, &s_plan, s_red);
  const int n_new = s_plan.n_new;
  if (n_new == 0) return;
  const Box B = s_plan.B, I = s_plan.I;
  const bool has_i = s_plan.has_i;
  const int ch = P.ch[level], cw = P.cw[level];
  const float* f2 = P.f2[level] + tr.pair * P.f2_pp[level];
  float* cache = P.cache[level] + tile * (int64_t)(ch * cw) * TQ;
  const int d = P.d;

  const float* rowsA[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int q = (tid >> 3) + 32 * s;
    const int py = tile_y * TQH + q / TQW, px = tile_x * TQW + q % TQW;
    rowsA[s] = (py < P.h1 && px < P.w1) ? P.f1 + (tr.pix + (int64_t)py * P.w1 + px) * d : nullptr;
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
      // queries ty*4..ty*4+3: tile row ty>>1, columns (ty&1)*4..+3 -> one
      // group, 4 consecutive group indices (cache layout [group][slot][8])
      const int qy = ty >> 1, qx0 = (ty & 1) * 4;
      *reinterpret_cast<float4*>(
          cache + ((int64_t)qgroup(qy, qx0) * (ch * cw) + slot_of(cy, cx, ch, cw)) * QG +
          qindex(qy, qx0)) = v;
    }
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_partial_sizes(const cvb_partial_desc* desc, int64_t* n_tiles, int64_t* meta_ints,
                      int64_t* cache_floats_per_level) {
  CVB_REQUIRE(desc, "partial_sizes: null desc");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  CVB_REQUIRE(desc->batch >= 0, "bad batch");
  const int64_t nt = ceil_div(desc->h1, TQH) * ceil_div(desc->w1, TQW) * batch_of(desc);
  if (n_tiles) *n_tiles = nt;
  // per-level metadata, then one plan record per tile (tensor-core path)
  // (plus one record's worth of ints for the contraction's tile counter)
  if (meta_ints) *meta_ints = nt * desc->levels * CVB_META_INTS + (nt + 1) * PLAN_INTS;
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

__attribute__((visibility("hidden"))) int cvb_internal_build_params(
    const cvb_partial_desc* desc, const float* f1,
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
  P.batch = batch_of(desc);
  P.tiles_pp = ceil_div(desc->h1, TQH) * (int64_t)P.tiles_x;
  P.n_tiles = P.tiles_pp * P.batch;
  P.plans = meta + P.n_tiles * desc->levels * CVB_META_INTS;
  for (int l = 0; l < CVB_MAX_LEVELS; ++l)
    P.f2_pp[l] = l < desc->levels ? (int64_t)desc->th[l] * desc->tw[l] * desc->d : 0;
  P.scale = scale;
  P.f64 = flags & CVB_COORDS_F64;
  P.normalize = scale != 1.0f;
  P.no_cache = flags & CVB_NO_CACHE;
  P.out_raft = flags & CVB_OUT_RAFT;
  P.vec = vec;
  CVB_REQUIRE(P.n_tiles <= 2147483647LL, "too many tiles");
  P.tile0 = desc->tile_begin > 0 ? desc->tile_begin : 0;
  const int64_t tend = desc->tile_end > desc->tile_begin ? desc->tile_end : P.n_tiles;
  CVB_REQUIRE(P.tile0 <= P.n_tiles && tend <= P.n_tiles, "tile range outside the frame");
  P.ntile = tend > P.tile0 ? tend - P.tile0 : 0;
  return CVB_OK;
}

static int launch_contract(const PartialParams& P, int32_t flags, cudaStream_t s) {
  if (P.ntile == 0) return CVB_OK;
  dim3 grid((unsigned)P.ntile, (unsigned)P.levels);
  if (flags & CVB_STRICT)
    partial_contract_kernel<true><<<grid, GEMM_THREADS, 0, s>>>(P);
  else
    partial_contract_kernel<false><<<grid, GEMM_THREADS, 0, s>>>(P);
  return check_launch("partial_contract");
}

static int launch_gather(const PartialParams& P, float* out, int32_t flags, cudaStream_t s) {
  if (P.ntile == 0) return CVB_OK;
  CVB_REQUIRE(out, "partial_sample: null output");
  return launch_gather_kernel(P, out, flags & CVB_STRICT, s);
}

int cvb_partial_sample(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       int32_t* meta, float* const* cache_levels_host, float* out,
                       unsigned long long* counters, int32_t flags, void* stream) {
  PartialParams P;
  int st = cvb_internal_build_params(desc, f1, f2_levels_host, coords, scale, meta, cache_levels_host,
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
  int st = cvb_internal_build_params(desc, f1, f2_levels_host, coords, 1.0f, meta, cache_levels_host,
                        counters, flags, P);
  if (st != CVB_OK) return st;
  return launch_contract(P, flags, as_stream(stream));
}

int cvb_partial_gather(const cvb_partial_desc* desc, const float* f1,
                       const float* const* f2_levels_host, const void* coords, float scale,
                       const int32_t* meta, float* const* cache_levels_host, float* out,
                       int32_t flags, void* stream) {
  PartialParams P;
  int st = cvb_internal_build_params(desc, f1, f2_levels_host, coords, scale, const_cast<int32_t*>(meta),
                        cache_levels_host, nullptr, flags, P);
  if (st != CVB_OK) return st;
  return launch_gather(P, out, flags, as_stream(stream));
}

}  // extern "C"
