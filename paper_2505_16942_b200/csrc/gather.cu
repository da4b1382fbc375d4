// (5) Gather / bilinear sampler of the partial path, reading the tile cache:
// the reference-exact (strict, fp64 combine) sampler and the fast sampler for
// radii other than 4 (fast r=4 is gather_fast.cu).
//
// One warp per query group of a tile (2 rows x 4 columns, the 8 queries of a
// cache sector) handles ALL levels, so the centroids are read once and the
// levels pipeline: while level l's taps are combined, level l+1's cache region
// is already in flight.
//   * staging: the union of the 8 supports of a level is a rectangle of
//     cells; in the warp's cache plane ([slot][8 queries], 32 B per cell)
//     every in-grid row of it is one contiguous run of slots (two if it wraps
//     the toroidal column), fetched with one cp.async.bulk per run into a
//     double-buffered shared-memory region; cells outside the grid are
//     zero-filled (dots with the zero padding, layout.py:1-14);
//   * taps: one (query, tap row) per lane-iteration; the two region rows a tap
//     row needs are read once and combined in registers with the canonical
//     association (fp64 in strict mode, _pykernels.py:99-115); the radius is a
//     template constant for strict r=4 so the loops unroll;
//   * outputs are staged per level in shared memory and written per query as
//     81 contiguous floats.
// Groups whose 8 supports do not fit one region (divergent flow) are processed
// as two groups of 4, then per query; tiles whose box overflowed the cache
// window are evaluated directly (dot products) — all bit-identical in strict
// mode.
#include <stdlib.h>

#include "partial.cuh"

namespace cvb {
namespace gather {

constexpr int WARPS = 4;
constexpr int MAXL = 4;          // levels per launch (the host loops for more)
constexpr int REG_CELLS = 224;   // per region buffer: 224 cells x 8 queries x 4 B = 7 KB
constexpr int MAX_TAPS = 81;     // r <= 4 for the staged-output path

struct QInfo {
  int ay, ax;
  double fx, fy;
  Weights32 w32;   // fp32 weights (the 1/sqrt(D) scale is applied after the combine)
};

struct Shared {
  float region[WARPS][2][REG_CELLS * TQW];
  float outs[WARPS][TQW * MAX_TAPS];
  QInfo q[WARPS][MAXL][TQW];
  int status[WARPS][MAXL];
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

// Pending staged region of one level (warp-uniform).
struct Region {
  int ylo, xlo, rh, rw;
  bool fast, copies;
};

// Union rectangle of the supports of the queries in `todo` at level l.
__device__ __forceinline__ void union_rect(const QInfo* qi, unsigned todo, int lane, int r,
                                           int& ylo, int& yhi, int& xlo, int& xhi) {
  const bool mine = lane < TQW && ((todo >> lane) & 1u);
  ylo = mine ? qi[lane].ay : INT_MAX;
  yhi = mine ? qi[lane].ay : INT_MIN;
  xlo = mine ? qi[lane].ax : INT_MAX;
  xhi = mine ? qi[lane].ax : INT_MIN;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
    yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
    xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
    xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, o));
  }
  ylo -= r;
  yhi += r + 1;
  xlo -= r;
  xhi += r + 1;
}

// Zero-fill (when needed) and issue the bulk copies of a region rectangle.
// Returns whether any copy was issued (then `bar` completes one phase).
__device__ __forceinline__ bool stage_region(float* R, uint32_t bar, const float* plane, int th,
                                             int tw, int ch, int cw, bool ok, int ylo, int yhi,
                                             int xlo, int xhi, int lane) {
  const int rh = yhi - ylo + 1, rw = xhi - xlo + 1;
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
  if (!any) return false;
  const int nrow = gy1 - gy0 + 1, ncol = gx1 - gx0 + 1;
  if (lane == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)(nrow * ncol * TQW * 4))
                 : "memory");
  __syncwarp();
  // In-grid cells of the region lie in the tile box (<= cap): slot = first
  // in-grid slot + an offset < cap, one conditional subtraction.
  const int ym = gy0 % ch, xm = gx0 % cw;
  const int n1 = min(ncol, cw - xm);  // cells before the column wrap
  const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(R);
  for (int i = lane; i < nrow; i += 32) {
    int srow = ym + i;
    if (srow >= ch) srow -= ch;
    const uint32_t dst = rbase + (uint32_t)(((gy0 - ylo + i) * rw + (gx0 - xlo)) * TQW * 4);
    bulk_copy(dst, plane + (int64_t)(srow * cw + xm) * TQW, (uint32_t)(n1 * TQW * 4), bar);
    if (ncol > n1)
      bulk_copy(dst + (uint32_t)(n1 * TQW * 4), plane + (int64_t)(srow * cw) * TQW,
                (uint32_t)((ncol - n1) * TQW * 4), bar);
  }
  return true;
}

// Taps of the queries in `todo` from a staged region into outs[q][K*K].
template <bool STRICT, int K_>
__device__ __forceinline__ void region_taps(const float* __restrict__ R, const QInfo* qi,
                                            unsigned todo, int ylo, int xlo, int rw, int r, int K,
                                            float scale, bool normalize, float* __restrict__ O,
                                            int lane) {
  const int KK = K * K;
  for (int e = lane; e < TQW * K; e += 32) {
    const int q = e & (TQW - 1), dy = e >> 3;
    if (!((todo >> q) & 1u)) continue;
    const float* a = R + ((qi[q].ay - r - ylo + dy) * rw + (qi[q].ax - r - xlo)) * TQW + q;
    const float* b = a + rw * TQW;
    const Weights32 w32 = qi[q].w32;
    Weights64 w64;
    if (STRICT) w64 = weights64(qi[q].fx, qi[q].fy);
    float* o = O + q * KK + dy * K;
    float a0 = a[0], b0 = b[0];
    if (K_ > 0) {
#pragma unroll
      for (int i = 0; i < K_; ++i) {
        const float a1 = a[(i + 1) * TQW], b1 = b[(i + 1) * TQW];
        float v = STRICT ? combine64(a0, a1, b0, b1, w64) : combine32(a0, a1, b0, b1, w32);
        if (normalize) v = __fmul_rn(v, scale);
        o[i] = v;
        a0 = a1;
        b0 = b1;
      }
    } else {
      for (int i = 0; i < K; ++i) {
        const float a1 = a[(i + 1) * TQW], b1 = b[(i + 1) * TQW];
        float v = STRICT ? combine64(a0, a1, b0, b1, w64) : combine32(a0, a1, b0, b1, w32);
        if (normalize) v = __fmul_rn(v, scale);
        o[i] = v;
        a0 = a1;
        b0 = b1;
      }
    }
  }
}

// Pixel of query i of the warp's group: pix0 + (i >> 2) * w1 + (i & 3).
template <int KK_>
__device__ __forceinline__ void write_outs(const float* O, unsigned todo, float* out,
                                           int64_t pix0, int w1, int levels, int level, int KK,
                                           int lane) {
  if (KK_ > 0 && todo == 0xFFu) {  // flat loop over the 8 queries' outputs
    for (int e = lane; e < QG * KK_; e += 32) {
      const int q = e / KK_, t = e - q * KK_;
      const int64_t pix = pix0 + (q >> 2) * (int64_t)w1 + (q & 3);
      out[(pix * levels + level) * (int64_t)KK_ + t] = O[e];
    }
    return;
  }
  for (int q = 0; q < QG; ++q) {
    if (!((todo >> q) & 1u)) continue;
    const int64_t pix = pix0 + (q >> 2) * (int64_t)w1 + (q & 3);
    float* dst = out + (pix * levels + level) * (int64_t)KK;
    for (int t = lane; t < KK; t += 32) dst[t] = O[q * KK + t];
  }
}

template <bool STRICT>
__device__ __forceinline__ void emit_patch_taps(const float* __restrict__ patch, int S, int K,
                                                const QInfo& qi, float scale, bool normalize,
                                                float* __restrict__ o, int lane) {
  const Weights64 w64 = weights64(qi.fx, qi.fy);
  for (int t = lane; t < K * K; t += 32) {
    const int j = t / K, i = t % K;
    o[t] = tap_from_patch<STRICT>(patch, S, j, i, w64, qi.w32, scale, normalize);
  }
}

template <bool STRICT, int RADIUS>
__global__ void __launch_bounds__(WARPS * 32)
    gather_kernel(PartialParams P, float* out, int level0, int nlev) {
  extern __shared__ __align__(128) uint8_t g_smem[];
  Shared& sm = *reinterpret_cast<Shared*>(g_smem);
  const int r = RADIUS >= 0 ? RADIUS : P.radius;
  const int K = 2 * r + 1, KK = K * K, S = 2 * r + 2;
  constexpr int K_ = RADIUS >= 0 ? 2 * RADIUS + 1 : -1;
  constexpr int KK_ = K_ > 0 ? K_ * K_ : -1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = P.tile0 + (blockIdx.x >> 1);
  const TileRef tr = tile_ref(P, tile);
  const int tile_y = tr.ty, tile_x = tr.tx;
  const int grp = (blockIdx.x & 1) * WARPS + warp;  // query group (2 rows x 4 columns)
  const int py0 = tile_y * TQH + group_qy(grp, 0), px0 = tile_x * TQW + group_qx(grp, 0);
  if (py0 >= P.h1) return;  // warp-uniform

  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t bar1 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][1]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- centroids once, per-level anchors and weights ----
  bool valid = false;
  if (lane < QG) {
    const int py = py0 + (lane >> 2), px = px0 + (lane & 3);
    valid = py < P.h1 && px < P.w1;
    double x = 0.0, y = 0.0;
    if (valid) load_coord(P.coords, P.f64, tr.pix + (int64_t)py * P.w1 + px, x, y);
    for (int li = 0; li < nlev; ++li) {
      const int l = level0 + li;
      QInfo qi{0, 0, 0.0, 0.0, Weights32{0.f, 0.f, 0.f, 0.f}};
      if (valid) {
        const LevelPos lp = level_pos(x, y, l);
        qi.ay = clamp_anchor(lp.y0, r, P.th[l]);
        qi.ax = clamp_anchor(lp.x0, r, P.tw[l]);
        qi.fx = lp.fx;
        qi.fy = lp.fy;
        qi.w32 = weights32(lp.fx, lp.fy);
      }
      sm.q[warp][li][lane] = qi;
    }
  } else if (lane < TQW + nlev) {
    const int li = lane - TQW;
    sm.status[warp][li] = P.meta[(tile * P.levels + level0 + li) * CVB_META_INTS + 4];
  }
  const unsigned vmask = __ballot_sync(0xffffffffu, valid) & 0xFFu;
  __syncwarp();
  if (vmask == 0) return;
  const int64_t pix0 = tr.pix + (int64_t)py0 * P.w1 + px0;
  auto pix = [&](int q) { return pix0 + (q >> 2) * (int64_t)P.w1 + (q & 3); };
  float* O = sm.outs[warp];
  uint32_t phase0 = 0u, phase1 = 0u;

  auto plane_of = [&](int l) {
    const int64_t cap = (int64_t)P.ch[l] * P.cw[l];
    return P.cache[l] + (tile * QG + grp) * cap * QG;
  };

  // issue the staged region of level index li into buffer b
  auto issue = [&](int li, int b) -> Region {
    Region g{0, 0, 0, 0, false, false};
    const int l = level0 + li;
    const int status = sm.status[warp][li];
    if (status == ST_OVERFLOW || KK > MAX_TAPS) return g;
    int ylo, yhi, xlo, xhi;
    union_rect(sm.q[warp][li], vmask, lane, r, ylo, yhi, xlo, xhi);
    g.ylo = ylo;
    g.xlo = xlo;
    g.rh = yhi - ylo + 1;
    g.rw = xhi - xlo + 1;
    if (g.rh * g.rw > REG_CELLS) return g;
    g.fast = true;
    g.copies = stage_region(sm.region[warp][b], b ? bar1 : bar0, plane_of(l), P.th[l], P.tw[l],
                            P.ch[l], P.cw[l], status == ST_OK, ylo, yhi, xlo, xhi, lane);
    return g;
  };

  // synchronous path for a level that did not fit one staged region
  auto slow_level = [&](int li, int b) {
    const int l = level0 + li;
    const int status = sm.status[warp][li];
    const int th = P.th[l], tw = P.tw[l], ch = P.ch[l], cw = P.cw[l];
    const float* plane = plane_of(l);
    float* R = sm.region[warp][b];
    const uint32_t bar = b ? bar1 : bar0;
    const QInfo* qi = sm.q[warp][li];
    unsigned done = ~vmask & 0xFFu;
    if (status != ST_OVERFLOW && KK <= MAX_TAPS) {
      for (int g0 = 0; g0 < TQW; g0 += 4) {  // groups of 4 queries
        const unsigned todo = (0xFu << g0) & ~done;
        if (todo == 0) continue;
        int ylo, yhi, xlo, xhi;
        union_rect(qi, todo, lane, r, ylo, yhi, xlo, xhi);
        const int rw = xhi - xlo + 1;
        if ((yhi - ylo + 1) * rw > REG_CELLS) continue;
        if (stage_region(R, bar, plane, th, tw, ch, cw, status == ST_OK, ylo, yhi, xlo, xhi,
                         lane)) {
          uint32_t& ph = b ? phase1 : phase0;
          bar_wait(bar, ph);
          ph ^= 1u;
        }
        region_taps<STRICT, K_>(R, qi, todo, ylo, xlo, rw, r, K, P.scale, P.normalize, O, lane);
        __syncwarp();
        write_outs<KK_>(O, todo, out, pix0, P.w1, P.levels, l, KK, lane);
        __syncwarp();
        done |= todo;
      }
    }
    // per query: (2r+2)^2 patch from the cache, or direct dots if overflowed
    const int d = P.d;
    const float* f2 = P.f2[l] + tr.pair * P.f2_pp[l];
    for (int q = 0; q < TQW; ++q) {
      if ((done >> q) & 1u) continue;
      const float* a = P.f1 + pix(q) * d;
      for (int c = lane; c < S * S; c += 32) {
        const int cy = qi[q].ay - r + c / S, cx = qi[q].ax - r + c % S;
        float v = 0.f;
        if (cy >= 0 && cy < th && cx >= 0 && cx < tw) {
          if (status == ST_OK) {
            v = __ldg(plane + (int64_t)slot_of(cy, cx, ch, cw) * TQW + q);
          } else if (status == ST_OVERFLOW) {
            const float* bb = f2 + ((int64_t)cy * tw + cx) * d;
            float acc = 0.f;
            if (P.vec) {
              for (int k = 0; k < d; k += 4) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(a + k));
                const float4 y = __ldg(reinterpret_cast<const float4*>(bb + k));
                acc = mac<STRICT>(acc, x.x, y.x);
                acc = mac<STRICT>(acc, x.y, y.y);
                acc = mac<STRICT>(acc, x.z, y.z);
                acc = mac<STRICT>(acc, x.w, y.w);
              }
            } else {
              for (int k = 0; k < d; ++k) acc = mac<STRICT>(acc, __ldg(a + k), __ldg(bb + k));
            }
            v = acc;
          }
        }
        R[c] = v;
      }
      __syncwarp();
      emit_patch_taps<STRICT>(R, S, K, qi[q], P.scale, P.normalize,
                              out + (pix(q) * P.levels + l) * (int64_t)KK, lane);
      __syncwarp();
    }
  };

  // ---- level pipeline: regions of levels li+1 (and li+2 after consuming li)
  // are in flight while level li's taps are combined ----
  Region pend0 = issue(0, 0), pend1{0, 0, 0, 0, false, false};
  if (nlev > 1) pend1 = issue(1, 1);
  for (int li = 0; li < nlev; ++li) {
    const int b = li & 1;
    const Region g = b ? pend1 : pend0;
    if (g.fast) {
      if (g.copies) {
        uint32_t& ph = b ? phase1 : phase0;
        bar_wait(b ? bar1 : bar0, ph);
        ph ^= 1u;
      }
      region_taps<STRICT, K_>(sm.region[warp][b], sm.q[warp][li], vmask, g.ylo, g.xlo, g.rw, r,
                              K, P.scale, P.normalize, O, lane);
      __syncwarp();
      write_outs<KK_>(O, vmask, out, pix0, P.w1, P.levels, level0 + li, KK, lane);
      __syncwarp();
    } else {
      slow_level(li, b);
    }
    if (li + 2 < nlev) {
      if (b)
        pend1 = issue(li + 2, 1);
      else
        pend0 = issue(li + 2, 0);
    }
  }
}

}  // namespace gather

template <bool STRICT, int RADIUS>
static void launch_one(const PartialParams& P, float* out, int l0, int nl, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  const int smem = (int)sizeof(gather::Shared);
  ensure_max_smem(attr, gather::gather_kernel<STRICT, RADIUS>, smem);
  gather::gather_kernel<STRICT, RADIUS>
      <<<(unsigned)(2 * P.ntile), gather::WARPS * 32, smem, s>>>(P, out, l0, nl);
}

int launch_gather_kernel(const PartialParams& P, float* out, bool strict, cudaStream_t s) {
  // fast arithmetic at r=4 (RAFT / SEA-RAFT): the register-direct sampler
  if (!strict && P.radius == 4) return launch_gather_fast_r4(P, out, s);
  CVB_REQUIRE(!P.out_raft, "CVB_OUT_RAFT needs the fast-arithmetic r=4 sampler");
  for (int l0 = 0; l0 < P.levels; l0 += gather::MAXL) {
    const int nl = min(gather::MAXL, P.levels - l0);
    if (strict && P.radius == 4)
      launch_one<true, 4>(P, out, l0, nl, s);
    else if (strict)
      launch_one<true, -1>(P, out, l0, nl, s);
    else
      launch_one<false, -1>(P, out, l0, nl, s);
    const int st = check_launch("partial_gather");
    if (st != CVB_OK) return st;
  }
  return CVB_OK;
}

}  // namespace cvb
