// Shared definitions of the partial sampler's tile path (csrc/partial.cu,
// csrc/partial_tc.cu): query tiles, the window-union tiler and the toroidal
// tile-cache addressing.  See partial.cu for the design.
#pragma once
#include "common.cuh"

namespace cvb {

constexpr int TQH = CVB_TILE_H, TQW = CVB_TILE_W, TQ = TQH * TQW;  // 64 queries
constexpr int ST_OK = 0, ST_OVERFLOW = 1, ST_EMPTY = 2;

// Tile-cache sectors: each cached cell holds its 64 query costs as 8 groups of
// 8 (32 bytes), a group being 2 query rows x 4 query columns of the tile.  A
// sampler reading one group's windows fetches the union of 8 windows shifted
// by (0..1, 0..3) cells — 10-13% fewer sectors than 8 queries of one row.
// Cache layout per level: [tile][group][cap_h * cap_w slots][8 queries].
constexpr int QG = 8;
__host__ __device__ __forceinline__ int qgroup(int qy, int qx) { return (qy >> 1) * 2 + (qx >> 2); }
__host__ __device__ __forceinline__ int qindex(int qy, int qx) { return (qy & 1) * 4 + (qx & 3); }
__host__ __device__ __forceinline__ int group_qy(int g, int i) { return 2 * (g >> 1) + (i >> 2); }
__host__ __device__ __forceinline__ int group_qx(int g, int i) { return 4 * (g & 1) + (i & 3); }

struct PartialParams {
  const float* f1;
  int h1, w1, d, levels, radius;
  const float* f2[CVB_MAX_LEVELS];
  float* cache[CVB_MAX_LEVELS];
  int th[CVB_MAX_LEVELS], tw[CVB_MAX_LEVELS], ch[CVB_MAX_LEVELS], cw[CVB_MAX_LEVELS];
  const void* coords;
  int32_t* meta;
  int32_t* plans;        // PlanRec per tile (after the per-level meta, same buffer)
  unsigned long long* counters;
  int tiles_x;
  int64_t n_tiles;       // all tiles of the frame (of every pair of the batch)
  int batch;             // image pairs sharing one launch (>= 1)
  int64_t tiles_pp;      // tiles per pair: pair b owns tiles [b*tiles_pp, (b+1)*tiles_pp)
  int64_t f2_pp[CVB_MAX_LEVELS];  // floats between consecutive pairs' level-l maps
  int64_t tile0, ntile;  // range handled by this launch
  float scale;
  bool f64, normalize, no_cache, vec;
  bool out_raft;         // CVB_OUT_RAFT output layout
};

// Where a (global) tile lives: its pair, its tile row / column within the
// pair's frame, and the pair's first pixel in f1 / coords / the cost map
// ([B, H, W, ...] layouts).  A batch of one reduces to the single-pair frame.
struct TileRef {
  int pair, ty, tx;
  int64_t pix;
};
__device__ __forceinline__ TileRef tile_ref(const PartialParams& P, int64_t tile) {
  TileRef t;
  t.pair = P.batch > 1 ? (int)(tile / P.tiles_pp) : 0;
  const int64_t lt = tile - (int64_t)t.pair * P.tiles_pp;
  t.ty = (int)(lt / P.tiles_x);
  t.tx = (int)(lt - (int64_t)t.ty * P.tiles_x);
  t.pix = (int64_t)t.pair * P.h1 * P.w1;
  return t;
}

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

// Result of the window-union tiler for one (tile, level).
struct TilePlan {
  Box B, I;
  int has_i, n_new, nvalid, status;
};

// All-level plan of one tile as the tensor-core contraction consumes it: one
// 16-byte-aligned record per tile, copied into shared memory with one bulk
// async copy (csrc/partial_tc.cu).
struct alignas(16) PlanRec {
  TilePlan plan[CVB_MAX_LEVELS];
  int prefix[CVB_MAX_LEVELS + 1];  // cells of levels < l in the tile's new-cell list
  int n_cells;
  int tile;    // the record's tile (-1: end of the work list)
  int pad;
};
constexpr int PLAN_INTS = (int)(sizeof(PlanRec) / 4);

// Window-union tiler for one (tile, level); every thread of the CTA must call
// it (blockDim >= 64).  Bounding box of the tile's (2r+2)^2 supports (offsets
// -r..r+1 around floor(x/2^l), sparse.py:279) clipped to the level grid;
// compares with the previous box in `meta`, decides OK / OVERFLOW / EMPTY,
// writes the new meta and counters.  `plan` and `red` are shared memory.
__device__ __forceinline__ void plan_tile_level(const PartialParams& P, int64_t tile, int level,
                                                TilePlan* plan, int* red) {
  const TileRef tr = tile_ref(P, tile);
  const int tile_y = tr.ty, tile_x = tr.tx;
  const int th = P.th[level], tw = P.tw[level], r = P.radius;
  const int tid = threadIdx.x;
  if (tid == 0) {
    red[0] = INT_MAX;
    red[1] = INT_MIN;
    red[2] = INT_MAX;
    red[3] = INT_MIN;
    red[4] = 0;
  }
  __syncthreads();
  if (tid < TQ) {
    const int py = tile_y * TQH + tid / TQW, px = tile_x * TQW + tid % TQW;
    if (py < P.h1 && px < P.w1) {
      double x, y;
      load_coord(P.coords, P.f64, tr.pix + (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, level);
      const int ay = clamp_anchor(lp.y0, r, th), ax = clamp_anchor(lp.x0, r, tw);
      atomicMin(&red[0], ay);
      atomicMax(&red[1], ay);
      atomicMin(&red[2], ax);
      atomicMax(&red[3], ax);
      atomicAdd(&red[4], 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int32_t* meta = P.meta + (tile * P.levels + level) * CVB_META_INTS;
    const int nvalid = red[4];
    Box B;
    B.ylo = max(red[0] - r, 0);
    B.yhi = min(red[1] + r + 1, th - 1);
    B.xlo = max(red[2] - r, 0);
    B.xhi = min(red[3] + r + 1, tw - 1);
    int status = ST_OK;
    if (nvalid == 0 || B.empty()) {
      status = ST_EMPTY;
      B = Box{1, 0, 1, 0};
    } else if (B.h() > P.ch[level] || B.w() > P.cw[level]) {
      status = ST_OVERFLOW;
    }
    const Box prev{meta[0], meta[1], meta[2], meta[3]};
    const bool prev_ok = !P.no_cache && meta[4] == ST_OK && !prev.empty();
    const Box I{max(B.ylo, prev.ylo), min(B.yhi, prev.yhi), max(B.xlo, prev.xlo),
                min(B.xhi, prev.xhi)};
    const bool has_i = status == ST_OK && prev_ok && !I.empty();
    const int n_new = status == ST_OK ? (int)(B.area() - (has_i ? I.area() : 0)) : 0;
    plan->B = B;
    plan->I = I;
    plan->has_i = has_i;
    plan->n_new = n_new;
    plan->nvalid = nvalid;
    plan->status = status;
    meta[0] = B.ylo;
    meta[1] = B.yhi;
    meta[2] = B.xlo;
    meta[3] = B.xhi;
    meta[4] = status;
    meta[5] = n_new;
    if (P.counters != nullptr) {
      if (n_new > 0) {
        atomicAdd(P.counters + 0, (unsigned long long)n_new * nvalid);
        atomicAdd(P.counters + 1, (unsigned long long)n_new);
      }
      if (status == ST_OVERFLOW) atomicAdd(P.counters + 2, 1ULL);
      if (status == ST_EMPTY) atomicAdd(P.counters + 3, 1ULL);
    }
  }
  __syncthreads();
}

// gather/sampler launch (csrc/gather.cu)
int launch_gather_kernel(const PartialParams& P, float* out, bool strict, cudaStream_t s);
// fast-arithmetic r=4 sampler (csrc/gather_fast.cu)
int launch_gather_fast_r4(const PartialParams& P, float* out, cudaStream_t s);

}  // namespace cvb

extern "C" int cvb_internal_build_params(const cvb_partial_desc* desc, const float* f1,
                                         const float* const* f2_levels_host, const void* coords,
                                         float scale, int32_t* meta,
                                         float* const* cache_levels_host,
                                         unsigned long long* counters, int32_t flags,
                                         cvb::PartialParams& P);
