// (5) Gather / bilinear sampler, fast-arithmetic r=4 path (RAFT / SEA-RAFT).
//
// Same contract as gather_kernel (gather.cu) — taps from the tile cache,
// zero padding outside the level grid, fp32 bilinear weights — restructured
// for instruction economy, since the sampler is issue-bound, not HBM-bound,
// when every lane does its own staging arithmetic:
//   * one warp per query row of a tile (8 queries), all levels (<= 4 per
//     launch); lane (q, l) = (lane & 7, lane >> 3) derives the anchor and
//     weights of query q at level l once, so the four levels' centroid math
//     and union rectangles are computed in parallel (3 shuffle rounds);
//   * the union of the 8 supports of a level is staged from the cache plane
//     ([slot][8 queries], 32 B per cell) with one cp.async.bulk per in-grid
//     region row, issued by a single lane from warp-uniform row parameters,
//     into a double-buffered region (level l+1 in flight while level l is
//     combined); the region row stride is odd so the three tap-row groups
//     read distinct banks;
//   * taps: lane (q, p), p < 3, computes tap rows p, p+3, p+6 of query q
//     (canonical fp32 combine, pre-scaled weights) into a per-level output
//     stage, written back as 81 contiguous floats per query.
// Levels whose box overflowed the cache window, or whose union does not fit
// the region buffer, take the per-query path (gather.cu semantics).
#include "partial.cuh"

namespace cvb {
namespace gfast {

constexpr int WARPS = 4;
constexpr int R = 4, K = 9, KK = 81, S = 10;
constexpr int REG_CELLS = 240;  // 240 cells x 8 queries x 4 B = 7.5 KB per buffer

struct Shared {
  float region[WARPS][2][REG_CELLS * TQW];
  float outs[WARPS][TQW * KK];
  float patch[WARPS][S * S];
  uint64_t bar[WARPS][2];
};

__device__ __forceinline__ void bulk_copy(uint32_t dst, const float* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra.uni DONE;\n\t"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Staged region of one level (warp-uniform).
struct Region {
  int ylo, xlo, rh, rw, ld;  // ld: odd row stride in cells
  bool fast, copies;
};

__global__ void __launch_bounds__(WARPS * 32, 3) gather_fast_kernel(PartialParams P, float* out,
                                                                 int level0, int nlev) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  Shared& sm = *reinterpret_cast<Shared*>(g_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = P.tile0 + (blockIdx.x >> 1);
  const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
  const int qrow = (blockIdx.x & 1) * WARPS + warp;
  const int py = tile_y * TQH + qrow;
  if (py >= P.h1) return;  // warp-uniform

  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t bar1 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][1]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- lane (q, l): anchor and weights of query q at level level0 + l ----
  const int q = lane & 7, li = lane >> 3;
  const int px = tile_x * TQW + q;
  const bool qvalid = px < P.w1;
  const unsigned vmask = __ballot_sync(0xffffffffu, qvalid) & 0xFFu;
  int ay = 0, ax = 0;
  Weights32 w{0.f, 0.f, 0.f, 0.f};
  double fx = 0.0, fy = 0.0;
  int status = ST_EMPTY;
  if (li < nlev) {
    const int l = level0 + li;
    status = P.meta[(tile * P.levels + l) * CVB_META_INTS + 4];
    if (qvalid) {
      double x, y;
      load_coord(P.coords, P.f64, (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, l);
      ay = clamp_anchor(lp.y0, R, P.th[l]);
      ax = clamp_anchor(lp.x0, R, P.tw[l]);
      fx = lp.fx;
      fy = lp.fy;
      w = weights32(lp.fx, lp.fy);
      const float sc = P.normalize ? P.scale : 1.0f;
      w.w00 *= sc;
      w.w01 *= sc;
      w.w10 *= sc;
      w.w11 *= sc;
    }
  }
  // union rectangle of the level's 8 anchors (lanes of one level group)
  int uylo = qvalid ? ay : INT_MAX, uyhi = qvalid ? ay : INT_MIN;
  int uxlo = qvalid ? ax : INT_MAX, uxhi = qvalid ? ax : INT_MIN;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    uylo = min(uylo, __shfl_xor_sync(0xffffffffu, uylo, o));
    uyhi = max(uyhi, __shfl_xor_sync(0xffffffffu, uyhi, o));
    uxlo = min(uxlo, __shfl_xor_sync(0xffffffffu, uxlo, o));
    uxhi = max(uxhi, __shfl_xor_sync(0xffffffffu, uxhi, o));
  }
  __syncwarp();
  if (vmask == 0) return;
  const int64_t row0 = (int64_t)py * P.w1 + tile_x * TQW;
  float* O = sm.outs[warp];
  uint32_t phase0 = 0u, phase1 = 0u;

  auto plane_of = [&](int l) {
    const int64_t cap = (int64_t)P.ch[l] * P.cw[l];
    return P.cache[l] + (tile * TQH + qrow) * cap * TQW;
  };

  // stage level li's region into buffer b (warp-uniform control flow)
  auto issue = [&](int li_, int b) -> Region {
    Region g{0, 0, 0, 0, 0, false, false};
    const int st = __shfl_sync(0xffffffffu, status, 8 * li_);
    if (st == ST_OVERFLOW) return g;
    const int ylo = __shfl_sync(0xffffffffu, uylo, 8 * li_) - R;
    const int yhi = __shfl_sync(0xffffffffu, uyhi, 8 * li_) + R + 1;
    const int xlo = __shfl_sync(0xffffffffu, uxlo, 8 * li_) - R;
    const int xhi = __shfl_sync(0xffffffffu, uxhi, 8 * li_) + R + 1;
    g.ylo = ylo;
    g.xlo = xlo;
    g.rh = yhi - ylo + 1;
    g.rw = xhi - xlo + 1;
    g.ld = g.rw | 1;
    if (g.rh * g.ld > REG_CELLS) return g;
    g.fast = true;
    const int l = level0 + li_;
    const int th = P.th[l], tw = P.tw[l], ch = P.ch[l], cw = P.cw[l];
    float* Rb = sm.region[warp][b];
    const int gy0 = max(ylo, 0), gy1 = min(yhi, th - 1);
    const int gx0 = max(xlo, 0), gx1 = min(xhi, tw - 1);
    const bool any = st == ST_OK && gy0 <= gy1 && gx0 <= gx1;
    const bool full = any && gy0 == ylo && gy1 == yhi && gx0 == xlo && gx1 == xhi;
    if (!full) {
      float4* z = reinterpret_cast<float4*>(Rb);
      for (int i = lane; i < g.rh * g.ld * 2; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (!any) return g;
    g.copies = true;
    if (lane == 0) {
      const int nrow = gy1 - gy0 + 1, ncol = gx1 - gx0 + 1;
      const uint32_t bar = b ? bar1 : bar0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(nrow * ncol * TQW * 4))
                   : "memory");
      // in-grid cells lie in the tile box (<= cap): slot = first in-grid slot +
      // an offset < cap, one conditional subtraction
      const float* plane = plane_of(l);
      const int xm = gx0 % cw;
      const int n1 = min(ncol, cw - xm);
      const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(Rb) +
                             (uint32_t)(((gy0 - ylo) * g.ld + (gx0 - xlo)) * TQW * 4);
      int srow = gy0 % ch;
      for (int i = 0; i < nrow; ++i) {
        const uint32_t dst = rbase + (uint32_t)(i * g.ld * TQW * 4);
        const float* src = plane + (int64_t)(srow * cw) * TQW;
        bulk_copy(dst, src + xm * TQW, (uint32_t)(n1 * TQW * 4), bar);
        if (ncol > n1) bulk_copy(dst + (uint32_t)(n1 * TQW * 4), src, (uint32_t)((ncol - n1) * TQW * 4), bar);
        if (++srow == ch) srow = 0;
      }
    }
    return g;
  };

  // per-query fallback (overflowed box or oversized union): (2r+2)^2 patch
  // from the cache, or direct dot products when the box overflowed
  auto slow_level = [&](int li_) {
    const int l = level0 + li_;
    const int st = __shfl_sync(0xffffffffu, status, 8 * li_);
    const int th = P.th[l], tw = P.tw[l], ch = P.ch[l], cw = P.cw[l];
    const float* plane = plane_of(l);
    const float* f2 = P.f2[l];
    const int d = P.d;
    float* patch = sm.patch[warp];
    for (int qq = 0; qq < TQW; ++qq) {
      const int src_lane = 8 * li_ + qq;
      const int qay = __shfl_sync(0xffffffffu, ay, src_lane);
      const int qax = __shfl_sync(0xffffffffu, ax, src_lane);
      const double qfx = __shfl_sync(0xffffffffu, fx, src_lane);
      const double qfy = __shfl_sync(0xffffffffu, fy, src_lane);
      if (!((vmask >> qq) & 1u)) continue;
      const float* a = P.f1 + (row0 + qq) * d;
      for (int c = lane; c < S * S; c += 32) {
        const int cy = qay - R + c / S, cx = qax - R + c % S;
        float v = 0.f;
        if (cy >= 0 && cy < th && cx >= 0 && cx < tw) {
          if (st == ST_OK) {
            v = __ldg(plane + (int64_t)slot_of(cy, cx, ch, cw) * TQW + qq);
          } else if (st == ST_OVERFLOW) {
            const float* bb = f2 + ((int64_t)cy * tw + cx) * d;
            float acc = 0.f;
            for (int k = 0; k < d; ++k) acc = fmaf(__ldg(a + k), __ldg(bb + k), acc);
            v = acc;
          }
        }
        patch[c] = v;
      }
      __syncwarp();
      const Weights64 w64 = weights64(qfx, qfy);
      const Weights32 w32 = weights32(qfx, qfy);
      float* o = out + ((row0 + qq) * P.levels + l) * (int64_t)KK;
      for (int t = lane; t < KK; t += 32)
        o[t] = tap_from_patch<false>(patch, S, t / K, t % K, w64, w32, P.scale, P.normalize);
      __syncwarp();
    }
  };

  Region pend0 = issue(0, 0), pend1{0, 0, 0, 0, 0, false, false};
  if (nlev > 1) pend1 = issue(1, 1);
  const int p = lane >> 3;  // tap-row group (lanes 24..31 idle in the combine)
  for (int li_ = 0; li_ < nlev; ++li_) {
    const int b = li_ & 1;
    const Region g = b ? pend1 : pend0;
    const int l = level0 + li_;
    if (g.fast) {
      // this lane's query at level li_
      const int src_lane = 8 * li_ + q;
      const int qay = __shfl_sync(0xffffffffu, ay, src_lane);
      const int qax = __shfl_sync(0xffffffffu, ax, src_lane);
      Weights32 qw;
      qw.w00 = __shfl_sync(0xffffffffu, w.w00, src_lane);
      qw.w01 = __shfl_sync(0xffffffffu, w.w01, src_lane);
      qw.w10 = __shfl_sync(0xffffffffu, w.w10, src_lane);
      qw.w11 = __shfl_sync(0xffffffffu, w.w11, src_lane);
      if (g.copies) {
        uint32_t& ph = b ? phase1 : phase0;
        bar_wait(b ? bar1 : bar0, ph);
        ph ^= 1u;
      }
      if (p < 3 && ((vmask >> q) & 1u)) {
        const float* Rb = sm.region[warp][b];
        const float* base = Rb + ((qay - R - g.ylo) * g.ld + (qax - R - g.xlo)) * TQW + q;
        float* o = O + q * KK;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int dy = p + 3 * j;
          const float* r0 = base + dy * g.ld * TQW;
          const float* r1 = r0 + g.ld * TQW;
          float a0 = r0[0], b0 = r1[0];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const float a1 = r0[(i + 1) * TQW], b1 = r1[(i + 1) * TQW];
            o[dy * K + i] = combine32(a0, a1, b0, b1, qw);
            a0 = a1;
            b0 = b1;
          }
        }
      }
      __syncwarp();
      // 81 contiguous floats per query
#pragma unroll 1
      for (int qq = 0; qq < TQW; ++qq) {
        if (!((vmask >> qq) & 1u)) continue;
        float* dst = out + ((row0 + qq) * P.levels + l) * (int64_t)KK;
        const float* src = O + qq * KK;
        dst[lane] = src[lane];
        dst[lane + 32] = src[lane + 32];
        if (lane < KK - 64) dst[lane + 64] = src[lane + 64];
      }
      __syncwarp();
    } else {
      slow_level(li_);
    }
    if (li_ + 2 < nlev) {
      if (b)
        pend1 = issue(li_ + 2, 1);
      else
        pend0 = issue(li_ + 2, 0);
    }
  }
}

}  // namespace gfast

int launch_gather_fast_r4(const PartialParams& P, float* out, cudaStream_t s) {
  static bool attr = false;
  const int smem = (int)sizeof(gfast::Shared);
  if (!attr) {
    cudaFuncSetAttribute(gfast::gather_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr = true;
  }
  for (int l0 = 0; l0 < P.levels; l0 += 4) {
    const int nl = min(4, P.levels - l0);
    gfast::gather_fast_kernel<<<(unsigned)(2 * P.ntile), gfast::WARPS * 32, smem, s>>>(P, out, l0,
                                                                                      nl);
    const int st = check_launch("partial_gather_fast");
    if (st != CVB_OK) return st;
  }
  return CVB_OK;
}

}  // namespace cvb
