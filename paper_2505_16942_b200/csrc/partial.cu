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

  const int64_t tile = blockIdx.x;
  const int level = blockIdx.y;
  const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
  const int tw = P.tw[level];
  const int tid = threadIdx.x;
  plan_tile_level(P, tile, level, &s_plan, s_red);
  const int n_new = s_plan.n_new;
  if (n_new == 0) return;
  const Box B = s_plan.B, I = s_plan.I;
  const bool has_i = s_plan.has_i;
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
      // cache layout [query row][slot][8 queries]; queries ty*4..ty*4+3
      *reinterpret_cast<float4*>(
          cache + ((int64_t)(ty >> 1) * (ch * cw) + slot_of(cy, cx, ch, cw)) * TQW + (ty & 1) * 4) = v;
    }
  }
}

// K2: one warp per query row of the tile (8 queries); 4 warps per CTA, so a
// tile is two CTAs.  The union of the 8 supports (unclipped) is staged into
// shared memory as region[ry][rx][8 queries] with 16-byte loads of the cache
// (each cell holds the 8 queries' costs in one 32-byte sector); cells outside
// the grid stay zero, so every tap reads its 4 corners without bounds tests.
// Oversized regions and overflowed tiles take a per-query fallback.
constexpr int K2_WARPS = 4;
constexpr int K2_REGION_CELLS = 256;  // per warp: 256 cells x 8 queries x 4 B = 8 KB
constexpr int K2_MAX_TAPS = 81;       // staged outputs per query (r <= 4); larger r: fallback

template <bool STRICT>
__device__ __forceinline__ void emit_taps(const float* __restrict__ R, int stride_cell, int rw,
                                          int oy, int ox, int K, int t0, int tstep, double fx,
                                          double fy, float scale, bool normalize,
                                          float* __restrict__ o) {
  const Weights64 w64 = weights64(fx, fy);
  const Weights32 w32 = weights32(fx, fy);
  int dy = t0 / K, dx = t0 % K;
  const int row = rw * stride_cell;
  for (int t = t0; t < K * K; t += tstep) {
    const float* c = R + ((oy + dy) * rw + (ox + dx)) * stride_cell;
    const float v00 = c[0], v01 = c[stride_cell], v10 = c[row], v11 = c[row + stride_cell];
    float v = STRICT ? combine64(v00, v01, v10, v11, w64) : combine32(v00, v01, v10, v11, w32);
    if (normalize) v = __fmul_rn(v, scale);
    o[t] = v;
    dx += tstep;
    while (dx >= K) {
      dx -= K;
      ++dy;
    }
  }
}

template <bool STRICT>
__global__ void __launch_bounds__(K2_WARPS * 32) partial_sample_kernel(PartialParams P, float* out) {
  __shared__ __align__(16) float s_region[K2_WARPS][K2_REGION_CELLS * TQW];
  __shared__ int s_ay[K2_WARPS][TQW], s_ax[K2_WARPS][TQW], s_valid[K2_WARPS][TQW];
  __shared__ double s_fx[K2_WARPS][TQW], s_fy[K2_WARPS][TQW];
  __shared__ Weights64 s_w64[K2_WARPS][TQW];
  __shared__ Weights32 s_w32[K2_WARPS][TQW];
  __shared__ __align__(16) float s_out[K2_WARPS][TQW * K2_MAX_TAPS];
  __shared__ __align__(8) uint64_t s_bar[K2_WARPS];

  const int r = P.radius, S = 2 * r + 2, K = 2 * r + 1, KK = K * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = blockIdx.x >> 1;
  const int level = blockIdx.y;
  const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
  const int th = P.th[level], tw = P.tw[level];
  const int qrow = (blockIdx.x & 1) * K2_WARPS + warp;  // query row inside the tile
  const int py = tile_y * TQH + qrow;
  if (py >= P.h1) return;  // warp-uniform
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_bar[warp]))
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  int ay = 0, ax = 0, valid = 0;
  if (lane < TQW) {
    const int px = tile_x * TQW + lane;
    valid = px < P.w1;
    double fx = 0.0, fy = 0.0;
    if (valid) {
      double x, y;
      load_coord(P.coords, P.f64, (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, level);
      ay = clamp_anchor(lp.y0, r, th);
      ax = clamp_anchor(lp.x0, r, tw);
      fx = lp.fx;
      fy = lp.fy;
    }
    s_ay[warp][lane] = ay;
    s_ax[warp][lane] = ax;
    s_valid[warp][lane] = valid;
    s_fx[warp][lane] = fx;
    s_fy[warp][lane] = fy;
    s_w64[warp][lane] = weights64(fx, fy);
    s_w32[warp][lane] = weights32(fx, fy);
  }
  __syncwarp();
  const int32_t* meta = P.meta + (tile * P.levels + level) * CVB_META_INTS;
  const int status = meta[4];
  const int ch = P.ch[level], cw = P.cw[level];
  // this warp's plane of the tile cache: [slot][8 queries]
  const float* cache = P.cache[level] + (tile * TQH + qrow) * (int64_t)(ch * cw) * TQW;
  const int64_t row0 = (int64_t)py * P.w1 + tile_x * TQW;
  float* R = s_region[warp];
  float* O = s_out[warp];
  const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(R);
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar[warp]);
  const unsigned valid_mask = __ballot_sync(0xffffffffu, valid) & 0xFFu;
  unsigned done = ~valid_mask & 0xFFu;  // invalid queries need nothing
  uint32_t phase = 0;

  // Fast path over query groups: all 8 queries share one staged region; if
  // their union does not fit, two groups of 4 (divergent flow), then the
  // per-query fallback below.
  if (status != ST_OVERFLOW && KK <= K2_MAX_TAPS) {
    for (int gsz = TQW; gsz >= 4 && done != 0xFFu; gsz >>= 1) {
      for (int g0 = 0; g0 < TQW; g0 += gsz) {
        const unsigned gmask = ((1u << gsz) - 1u) << g0;
        const unsigned todo = gmask & ~done;
        if (todo == 0) continue;
        const bool mine = lane < TQW && ((todo >> lane) & 1u);
        int ylo = mine ? ay : INT_MAX, yhi = mine ? ay : INT_MIN;
        int xlo = mine ? ax : INT_MAX, xhi = mine ? ax : INT_MIN;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
          yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
          xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
          xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, o));
        }
        // unclipped union of the group's supports
        ylo -= r;
        yhi += r + 1;
        xlo -= r;
        xhi += r + 1;
        const int rh = yhi - ylo + 1, rw = xhi - xlo + 1;
        if (rh * rw > K2_REGION_CELLS) continue;  // try smaller groups
        // ---- stage the region: each in-grid region row is one contiguous run
        // of slots in this warp's cache plane (two if it wraps the toroidal
        // column), fetched with one bulk async copy per run; cells outside the
        // grid are zero-filled first.  In-grid cells of the region lie in the
        // tile box B (<= cap): slot = first in-grid slot + offset < cap.
        const bool ok = status == ST_OK;
        const int gy0 = max(ylo, 0), gy1 = min(yhi, th - 1);
        const int gx0 = max(xlo, 0), gx1 = min(xhi, tw - 1);
        const bool any = ok && gy0 <= gy1 && gx0 <= gx1;
        const bool full = any && gy0 == ylo && gy1 == yhi && gx0 == xlo && gx1 == xhi;
        if (!full) {
          float4* z = reinterpret_cast<float4*>(R);
          for (int i = lane; i < rh * rw * 2; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (any) {
          const int nrow = gy1 - gy0 + 1, ncol = gx1 - gx0 + 1;
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"((uint32_t)(nrow * ncol * TQW * 4))
                         : "memory");
          __syncwarp();
          const int ym = gy0 % ch, xm = gx0 % cw;
          const int n1 = min(ncol, cw - xm);  // cells before the column wrap
          for (int i = lane; i < nrow; i += 32) {
            int srow = ym + i;
            if (srow >= ch) srow -= ch;
            const float* src = cache + (int64_t)(srow * cw + xm) * TQW;
            const uint32_t dst =
                rbase + (uint32_t)(((gy0 - ylo + i) * rw + (gx0 - xlo)) * TQW * 4);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(dst),
                "l"(src), "r"((uint32_t)(n1 * TQW * 4)), "r"(bar)
                : "memory");
            if (ncol > n1)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                  "%2, [%3];" ::"r"(dst + (uint32_t)(n1 * TQW * 4)),
                  "l"(cache + (int64_t)(srow * cw) * TQW), "r"((uint32_t)((ncol - n1) * TQW * 4)),
                  "r"(bar)
                  : "memory");
          }
          asm volatile(
              "{\n\t.reg .pred P1;\n"
              "LAB_WAIT:\n\t"
              "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
              "@P1 bra.uni DONE;\n\t"
              "bra.uni LAB_WAIT;\n"
              "DONE:\n\t}\n" ::"r"(bar),
              "r"(phase)
              : "memory");
          phase ^= 1u;
        }
        // ---- taps: one (query, tap row) per lane-iteration; the two region
        // rows a tap row needs are read once (K+1 cells each) and combined in
        // registers; results staged in shared memory for coalesced stores.
        for (int e = lane; e < TQW * K; e += 32) {
          const int q = e & (TQW - 1), dy = e >> 3;
          if (!((todo >> q) & 1u)) continue;
          const float* a =
              R + ((s_ay[warp][q] - r - ylo + dy) * rw + (s_ax[warp][q] - r - xlo)) * TQW + q;
          const float* b = a + rw * TQW;
          const Weights32 w32 = s_w32[warp][q];
          const Weights64 w64 = s_w64[warp][q];
          float* o = O + q * KK + dy * K;
          float a0 = a[0], b0 = b[0];
          for (int i = 0; i < K; ++i) {
            const float a1 = a[(i + 1) * TQW], b1 = b[(i + 1) * TQW];
            float v = STRICT ? combine64(a0, a1, b0, b1, w64) : combine32(a0, a1, b0, b1, w32);
            if (P.normalize) v = __fmul_rn(v, P.scale);
            o[i] = v;
            a0 = a1;
            b0 = b1;
          }
        }
        __syncwarp();
        for (int q = g0; q < g0 + gsz; ++q) {
          if (!((todo >> q) & 1u)) continue;
          float* dst = out + ((row0 + q) * P.levels + level) * (int64_t)KK;
          for (int t = lane; t < KK; t += 32) dst[t] = O[q * KK + t];
        }
        __syncwarp();
        done |= todo;
      }
    }
  }
  if (done == 0xFFu) return;

  // ---- fallback: one query at a time through a (2r+2)^2 patch ----
  const int d = P.d;
  const float* f2 = P.f2[level];
  for (int q = 0; q < TQW; ++q) {
    if ((done >> q) & 1u) continue;
    const int qay = s_ay[warp][q], qax = s_ax[warp][q];
    const float* a = P.f1 + (row0 + q) * d;
    for (int c = lane; c < S * S; c += 32) {
      const int cy = qay - r + c / S, cx = qax - r + c % S;
      float v = 0.f;
      if (cy >= 0 && cy < th && cx >= 0 && cx < tw) {
        if (status == ST_OK) {
          v = __ldg(cache + (int64_t)slot_of(cy, cx, ch, cw) * TQW + q);
        } else if (status == ST_OVERFLOW) {
          const float* b = f2 + ((int64_t)cy * tw + cx) * d;
          float acc = 0.f;
          if (P.vec) {
            for (int k = 0; k < d; k += 4) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(a + k));
              const float4 y = __ldg(reinterpret_cast<const float4*>(b + k));
              acc = mac<STRICT>(acc, x.x, y.x);
              acc = mac<STRICT>(acc, x.y, y.y);
              acc = mac<STRICT>(acc, x.z, y.z);
              acc = mac<STRICT>(acc, x.w, y.w);
            }
          } else {
            for (int k = 0; k < d; ++k) acc = mac<STRICT>(acc, __ldg(a + k), __ldg(b + k));
          }
          v = acc;
        }
      }
      R[c] = v;
    }
    __syncwarp();
    emit_taps<STRICT>(R, 1, S, 0, 0, K, lane, 32, s_fx[warp][q], s_fy[warp][q], P.scale,
                      P.normalize, out + ((row0 + q) * P.levels + level) * (int64_t)KK);
    __syncwarp();
  }
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
  dim3 grid((unsigned)(2 * P.n_tiles), (unsigned)P.levels);
  if (flags & CVB_STRICT)
    partial_sample_kernel<true><<<grid, K2_WARPS * 32, 0, s>>>(P, out);
  else
    partial_sample_kernel<false><<<grid, K2_WARPS * 32, 0, s>>>(P, out);
  return check_launch("partial_sample");
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
