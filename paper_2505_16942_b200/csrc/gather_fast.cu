// (5) Gather / bilinear sampler, fast-arithmetic r=4 path (RAFT / SEA-RAFT).
//
// Same contract as gather_kernel (gather.cu) — taps from the tile cache, zero
// padding outside the level grid, fp32 bilinear weights — but without a
// shared-memory region stage: the sampler is bound by instructions and
// latency, not bytes, when every lane computes staging addresses, so each lane
// reads exactly the cache sectors its taps need straight into registers.
//   * one warp per query group of a tile (2 rows x 4 columns = the 8 queries
//     of one 32-byte cache sector), two groups per CTA, all levels (<= 4 per
//     launch); lane
//     (q, l) = (lane & 7, lane >> 3) derives the anchor and weights of query
//     q at level l once (the four levels in parallel);
//   * taps: lane (q, l) owns query q at level l: two passes of 5 and 4 tap
//     rows, each loading the 6 x 10 / 4 x 10 patch values it needs from the
//     cache plane
//     ([slot][8 queries], 32-byte sectors shared by the row's queries through
//     L1) into registers, zero outside the level grid, and combining them
//     (canonical fp32 combine, pre-scaled weights);
//   * the group's outputs (two rows of 4 queries x L levels x 81 taps, two
//     contiguous blocks of the [H,W,L,9,9] cost map) are staged in shared
//     memory and written with 128-bit stores.
// Levels whose box overflowed the cache window are evaluated by direct dot
// products, the warp cooperating on each query's window (gather.cu semantics).
#include <stdlib.h>

#include "partial.cuh"

namespace cvb {
namespace gfast {

// two query groups (a quarter tile) per CTA, 8 CTAs per SM: the same 16
// resident warps per SM as whole-tile CTAs (registers bind at 126), but small
// CTAs retire and refill independently (-6% sampler time at C4)
constexpr int WARPS = 2;
constexpr int CTAS_PER_TILE = (TQ / QG) / WARPS;  // 8 query groups per tile
constexpr int MAXL = 4;    // levels per launch
constexpr int R = 4, K = 9, KK = 81, S = 10;

struct Shared {
  float outs[WARPS][QG * MAXL * KK];   // 10,368 B per warp
  float patch[WARPS][S * S];           // overflow path: one query's window
};

// Overflowed tile-level (its box exceeded the cache window): the warp
// evaluates each query's (2r+2)^2 window by direct dot products — lanes split
// the 100 cells, four independent 128-bit-load dot chains per lane — then
// combines the taps from the staged patch (gather.cu semantics, fmaf dots).
__device__ __noinline__ void overflow_level(const float* f1, const float* f2, int th, int tw,
                                            int d, bool vec, int64_t pix0, int w1, unsigned vmask,
                                            int ay, int ax, Weights32 w, int l_, int nlev,
                                            float* patch, float* O, int lane) {
  for (int qq = 0; qq < QG; ++qq) {
    const int src = 8 * l_ + qq;
    const int qay = __shfl_sync(0xffffffffu, ay, src), qax = __shfl_sync(0xffffffffu, ax, src);
    Weights32 qw;
    qw.w00 = __shfl_sync(0xffffffffu, w.w00, src);
    qw.w01 = __shfl_sync(0xffffffffu, w.w01, src);
    qw.w10 = __shfl_sync(0xffffffffu, w.w10, src);
    qw.w11 = __shfl_sync(0xffffffffu, w.w11, src);
    if (!((vmask >> qq) & 1u)) continue;
    const float* a = f1 + (pix0 + (qq >> 2) * (int64_t)w1 + (qq & 3)) * (int64_t)d;
    const float* b[4];
    bool in[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = lane + 32 * j;
      const int cy = qay - R + c / S, cx = qax - R + c % S;
      in[j] = c < S * S && cy >= 0 && cy < th && cx >= 0 && cx < tw;
      b[j] = in[j] ? f2 + ((int64_t)cy * tw + cx) * d : a;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (vec) {
      for (int k = 0; k < d; k += 4) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(a + k));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 y = __ldg(reinterpret_cast<const float4*>(b[j] + k));
          acc[j] = fmaf(x.x, y.x, acc[j]);
          acc[j] = fmaf(x.y, y.y, acc[j]);
          acc[j] = fmaf(x.z, y.z, acc[j]);
          acc[j] = fmaf(x.w, y.w, acc[j]);
        }
      }
    } else {
      for (int k = 0; k < d; ++k) {
        const float x = __ldg(a + k);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = fmaf(x, __ldg(b[j] + k), acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (lane + 32 * j < S * S) patch[lane + 32 * j] = in[j] ? acc[j] : 0.f;
    __syncwarp();
    float* o = O + (qq * nlev + l_) * KK;
    for (int t = lane; t < KK; t += 32) {
      const int dy = t / K, dx = t - dy * K;
      o[t] = combine32(patch[dy * S + dx], patch[dy * S + dx + 1], patch[(dy + 1) * S + dx],
                       patch[(dy + 1) * S + dx + 1], qw);
    }
    __syncwarp();
  }
}

template <int NPASS>
__global__ void __launch_bounds__(WARPS * 32, NPASS >= 3 ? 16 / WARPS : (NPASS == 2 ? 7 : 6))
    gather_fast_kernel(PartialParams P, float* out, int level0, int nlev, bool reverse) {
  extern __shared__ __align__(16) uint8_t g_smem[];
  Shared& sm = *reinterpret_cast<Shared*>(g_smem);
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tiles in reverse order: the contraction claims tiles in increasing order,
  // so the last tiles' new cells are the likeliest to still be in L2 (-1.1%
  // per C4 step, A/B; CVB_GF_REVERSE=0 restores the forward order)
  const int64_t ti = blockIdx.x / CTAS_PER_TILE;
  const int64_t tile = P.tile0 + (reverse ? P.ntile - 1 - ti : ti);
  const TileRef tr = tile_ref(P, tile);
  const int tile_y = tr.ty, tile_x = tr.tx;
  // query group: tile rows 2(g>>1)..+1, columns 4(g&1)..+3
  const int grp = (int)(blockIdx.x % CTAS_PER_TILE) * WARPS + warp;
  const int py0 = tile_y * TQH + group_qy(grp, 0), px0 = tile_x * TQW + group_qx(grp, 0);
  if (py0 >= P.h1) return;  // warp-uniform

  // ---- lane (q, l): anchor, fractions and weights of query q at level l ----
  const int q = lane & 7, li = lane >> 3;
  const int py = py0 + (q >> 2), px = px0 + (q & 3);
  const bool qvalid = py < P.h1 && px < P.w1;
  const unsigned vmask = __ballot_sync(0xffffffffu, qvalid) & 0xFFu;
  int ay = 0, ax = 0, status = ST_EMPTY;
  Weights32 w{0.f, 0.f, 0.f, 0.f};
  if (li < nlev) {
    const int l = level0 + li;
    status = P.meta[(tile * P.levels + l) * CVB_META_INTS + 4];
    if (qvalid) {
      double x, y;
      load_coord(P.coords, P.f64, tr.pix + (int64_t)py * P.w1 + px, x, y);
      const LevelPos lp = level_pos(x, y, l);
      ay = clamp_anchor(lp.y0, R, P.th[l]);
      ax = clamp_anchor(lp.x0, R, P.tw[l]);
      w = weights32(lp.fx, lp.fy);
      const float sc = P.normalize ? P.scale : 1.0f;
      w.w00 *= sc;
      w.w01 *= sc;
      w.w10 *= sc;
      w.w11 *= sc;
    }
  }
  if (vmask == 0) return;
  // pixel of query i (within the pair's frame): pix0 + (i>>2)*W + (i&3)
  const int64_t pix0 = (int64_t)py0 * P.w1 + px0;
  float* O = sm.outs[warp];  // [q][nlev][81]
  // overflowed levels: warp-cooperative direct dots (warp-uniform loop)
  for (int l_ = 0; l_ < nlev; ++l_) {
    if (__shfl_sync(0xffffffffu, status, 8 * l_) == ST_OVERFLOW)
      overflow_level(P.f1 + tr.pix * P.d, P.f2[level0 + l_] + tr.pair * P.f2_pp[level0 + l_],
                     P.th[level0 + l_], P.tw[level0 + l_], P.d, P.vec,
                     pix0, P.w1, vmask, ay, ax, w, l_, nlev, sm.patch[warp], O, lane);
  }
  // every lane (q, l) combines the 81 taps of query q at level l, TPP tap
  // rows per pass from (TPP + 1) x 10 cache values loaded into registers
  if (li < nlev && qvalid && status != ST_OVERFLOW) {
    const int l = level0 + li;
    const int th = P.th[l], tw = P.tw[l], ch = P.ch[l], cw = P.cw[l];
    const float* plane = P.cache[l] + ((tile * QG + grp) * (int64_t)(ch * cw)) * QG + q;
    const int x0 = ax - R;
    int xs = x0 % cw;
    if (xs < 0) xs += cw;
    // toroidal slot offsets and in-grid flags of the 10 patch columns
    int colofs[S];
    bool colin[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      colofs[i] = xs * QG;
      colin[i] = x0 + i >= 0 && x0 + i < tw;
      if (++xs == cw) xs = 0;
    }
    float* o = O + (q * nlev + li) * KK;
    // NPASS passes of TPP tap rows (TPP + 1 patch rows in registers): a pass's
    // last row is the next pass's first, carried in registers (each cache row
    // is loaded once); fewer passes = fewer dependent load round trips, more
    // registers
    constexpr int TPP = (K + NPASS - 1) / NPASS;
    float v[TPP + 1][S];
    int sy = (ay - R) % ch;
    if (sy < 0) sy += ch;
#pragma unroll 1
    for (int pass = 0; pass < NPASS; ++pass) {
      const int t0 = TPP * pass, nt = min(TPP, K - t0);
      const int y0 = ay - R + t0;
      if (pass > 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) v[0][i] = v[TPP][i];
      }
#pragma unroll
      for (int j = 0; j <= TPP; ++j) {
        if ((pass > 0 && j == 0) || j > nt) continue;
        const int gy = y0 + j;
        const bool rin = status == ST_OK && gy >= 0 && gy < th;
        const float* prow = plane + (int64_t)(sy * cw) * QG;
#pragma unroll
        for (int i = 0; i < S; ++i) v[j][i] = (rin && colin[i]) ? __ldg(prow + colofs[i]) : 0.f;
        if (++sy == ch) sy = 0;
      }
#pragma unroll
      for (int j = 0; j < TPP; ++j)
        if (j < nt)
#pragma unroll
          for (int i = 0; i < K; ++i)
            o[(t0 + j) * K + i] = combine32(v[j][i], v[j][i + 1], v[j + 1][i], v[j + 1][i + 1], w);
    }
  }
  __syncwarp();
  // ---- write back: the group's two rows of 4 queries ----
  if (P.out_raft) {
    // RAFT CorrBlock layout: out[(l * 81 + dx * 9 + dy) * H * W + pixel]; per
    // window index each row of the group is 16 contiguous bytes
    const int64_t hw = (int64_t)P.h1 * P.w1;
    float* out_pair = out + tr.pair * (int64_t)P.levels * KK * hw;  // [B, L*81, H, W]
    for (int e = lane; e < nlev * KK * 2; e += 32) {
      const int hq = e & 1, lt = e >> 1;
      const int l_ = lt / KK, t = lt - l_ * KK;
      const int dy = t / K, dx = t - dy * K;
      const unsigned rowmask = (vmask >> (4 * hq)) & 0xFu;
      float* dst = out_pair + ((int64_t)(level0 + l_) * KK + dx * K + dy) * hw + pix0 + hq * P.w1;
      const float* src = O + (4 * hq) * nlev * KK + lt;
      if (rowmask == 0xFu && (((uintptr_t)dst) & 15) == 0) {
        *reinterpret_cast<float4*>(dst) =
            make_float4(src[0], src[nlev * KK], src[2 * nlev * KK], src[3 * nlev * KK]);
      } else {
        for (int k = 0; k < 4; ++k)
          if ((rowmask >> k) & 1u) dst[k] = src[k * nlev * KK];
      }
    }
  } else {
    for (int hq = 0; hq < 2; ++hq) {
      const unsigned rowmask = (vmask >> (4 * hq)) & 0xFu;
      const float* src = O + 4 * hq * nlev * KK;
      float* dst = out + (tr.pix + pix0 + hq * P.w1) * (int64_t)(P.levels * KK);
      if (rowmask == 0xFu && nlev == P.levels && (((uintptr_t)dst) & 15) == 0) {
        // 4 consecutive pixels x L x 81 floats: one contiguous block
        const int n4 = 4 * nlev * KK / 4;
        for (int i = lane; i < n4; i += 32)
          reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
      } else {
        for (int k = 0; k < 4; ++k) {
          if (!((rowmask >> k) & 1u)) continue;
          for (int e = lane; e < nlev * KK; e += 32) {
            const int l_ = e / KK, t = e - l_ * KK;
            dst[(int64_t)k * P.levels * KK + (level0 + l_) * KK + t] = src[k * nlev * KK + e];
          }
        }
      }
    }
  }
}

}  // namespace gfast

int launch_gather_fast_r4(const PartialParams& P, float* out, cudaStream_t s) {
  // tap-row passes per query: 2 (patch rows 0-5, then 5-9; 128 registers,
  // the occupancy of 3 passes of 3 rows, one dependent load round trip
  // fewer: -1.8% sampler time at C4, A/B); CVB_GF_PASSES=1|3 for A/B
  static int npass = -1;
  if (npass < 0) {
    const char* e = getenv("CVB_GF_PASSES");
    npass = e ? atoi(e) : 2;
    if (npass != 1 && npass != 3) npass = 2;
  }
  auto kernel = npass == 1 ? gfast::gather_fast_kernel<1>
                           : (npass == 2 ? gfast::gather_fast_kernel<2> : gfast::gather_fast_kernel<3>);
  static std::atomic<uint64_t> attr{0};
  static int reverse = -1;
  if (reverse < 0) {
    const char* e = getenv("CVB_GF_REVERSE");
    reverse = !e || atoi(e) != 0;
  }
  const int smem = (int)sizeof(gfast::Shared);
  ensure_max_smem(attr, kernel, smem);
  // Shared-memory carveout 65%: the taps re-read each cache sector ~3x through
  // L1, so L1 capacity matters more than the last CTA slot per SM (measured:
  // 65% is 1-2% faster than the default 200 KB carveout; 100% halves the
  // speed).  CVB_GF_CARVEOUT overrides (percent; -1 = driver default).
  static std::atomic<uint64_t> carved{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(carved.load() & bit)) {
    const char* e = getenv("CVB_GF_CARVEOUT");
    const int carve = e ? atoi(e) : 65;
    if (carve >= 0)
      cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    carved.fetch_or(bit);
  }
  for (int l0 = 0; l0 < P.levels; l0 += gfast::MAXL) {
    const int nl = min(gfast::MAXL, P.levels - l0);
    launch_pdl_phase(kernel, dim3((unsigned)(gfast::CTAS_PER_TILE * P.ntile)), dim3(gfast::WARPS * 32), smem,
               s, P, out, l0, nl, reverse != 0);
    const int st = check_launch("partial_gather_fast");
    if (st != CVB_OK) return st;
  }
  return CVB_OK;
}

}  // namespace cvb
