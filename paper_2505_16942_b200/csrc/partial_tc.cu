// Tensor-core (tcgen05) contraction for the partial sampler's fast path.
//
// Same tiler, metadata and toroidal tile cache as partial_contract_kernel
// (partial.cuh); only the arithmetic of the new-cell contraction changes:
//
//   * one CTA per 8x8 query tile handles ALL levels: the new cells of every
//     level are concatenated and contracted in chunks of 128 cells;
//   * D[128 cells x 64 queries] = A[cells x K] . B[queries x K]^T with
//     M=128, N=64, K=16 `tcgen05.mma.cta_group::1.kind::f16`, accumulators in
//     TMEM (128 lanes x 64 fp32 columns, two of them);
//   * split precision: every fp32 value x (pre-scaled by a per-tensor power of
//     two so it sits in fp16 range) is stored as hi = fp16(x) and
//     lo = fp16((x - hi) * 2^11); x*y = hi_x*hi_y + 2^-11 (hi_x*lo_y + lo_x*hi_y)
//     + O(2^-22).  Three MMAs per K-step (main += hi.hi; corr += hi.lo;
//     corr += lo.hi) keep ~22 significant bits per product at 2x the TF32
//     tensor rate, well inside the fp32 tolerance (products of two fp16 are
//     exact in the fp32 accumulator);
//   * operands are pre-split once per image pair (cvb_tc_prepare): the F1
//     tile is one contiguous 64 KB image of its shared-memory layout, fetched
//     with a single bulk async copy (cp.async.bulk + mbarrier complete_tx);
//     A rows (gathered bbox cells) stream through a 2-stage cp.async ring in
//     the canonical K-major no-swizzle core-matrix layout (8 rows x 16 B);
//   * the epilogue reads TMEM with tcgen05.ld, combines main + 2^-11 corr,
//     removes the power-of-two scales and writes each cell's 64 query costs
//     (256 contiguous bytes) into its cache slot.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "partial.cuh"

namespace cvb {
namespace tc {

constexpr int THREADS = 128;
constexpr int M = 128;         // cells per MMA chunk (TMEM lanes)
constexpr int N = 64;          // queries per tile
constexpr int KS = 32;         // K per pipeline stage
constexpr int NST = 2;         // pipeline stages
constexpr int A_HALF = M * KS * 2;       // 8 KB (hi or lo)
constexpr int A_STAGE = 2 * A_HALF;      // 16 KB
constexpr int MAX_DP = 256;
constexpr int LOG2_LO = 11;              // lo part scale
constexpr int TARGET_EXP = 14;           // max |x * 2^e| < 2^14

// instruction descriptor: D f32, A/B f16, both K-major, N=64, M=128
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, SWIZZLE_NONE shared-memory matrix descriptor (sm100 version 1):
// core matrices of 8 rows x 16 B; LBO = byte step between the two 8-element
// K halves of a K=16 slice, SBO = byte step between 8-row groups.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra.uni DONE;\n\t"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N_>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// power-of-two exponent e with max * 2^e < 2^TARGET_EXP (0 for an all-zero tensor)
__device__ __forceinline__ int scale_exp(uint32_t maxbits) {
  const float m = __uint_as_float(maxbits);
  if (!(m > 0.f) || !isfinite(m)) return 0;
  int k;
  frexpf(m, &k);  // m < 2^k
  int e = TARGET_EXP - k;
  return e < -60 ? -60 : (e > 60 ? 60 : e);
}

__device__ __forceinline__ void split8(const float (&x)[8], float s, uint4& hi, uint4& lo) {
  __half h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float v = x[i] * s;
    h[i] = __float2half_rn(v);
    l[i] = __float2half_rn((v - __half2float(h[i])) * (float)(1 << LOG2_LO));
  }
  hi = *reinterpret_cast<uint4*>(h);
  lo = *reinterpret_cast<uint4*>(l);
}

struct TcParams {
  PartialParams P;
  const uint8_t* f1s;                  // [tiles][2][8 rg][dp/8 kg][8][8] fp16
  const __half* f2s[CVB_MAX_LEVELS];   // hi plane [th*tw][dp]; lo = hi + plane
  int64_t plane[CVB_MAX_LEVELS];
  const uint32_t* maxbits;             // [0] max|F1|, [1] max|F2|
  int dp;
};

__global__ void absmax_kernel(const float* __restrict__ x, int64_t n, uint32_t* out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(__ldg(x + i)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// F1 -> per-tile image of the B operand: [2][8 rowgroups][dp/8][8 rows][8]
__global__ void split_f1_kernel(const float* __restrict__ f1, int h1, int w1, int d, int dp,
                                int tiles_x, int64_t n_tiles, const uint32_t* maxbits,
                                uint8_t* __restrict__ out) {
  const int kgs = dp / 8;
  const int64_t total = n_tiles * N * kgs;
  const float s = ldexpf(1.f, scale_exp(maxbits[0]));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kg = (int)(i % kgs);
    const int q = (int)((i / kgs) % N);
    const int64_t tile = i / ((int64_t)kgs * N);
    const int py = (int)(tile / tiles_x) * TQH + q / TQW, px = (int)(tile % tiles_x) * TQW + q % TQW;
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kg * 8 + j;
      x[j] = (py < h1 && px < w1 && k < d) ? __ldg(f1 + ((int64_t)py * w1 + px) * d + k) : 0.f;
    }
    uint4 hi, lo;
    split8(x, s, hi, lo);
    const int64_t half_bytes = (int64_t)N * dp * 2;
    uint8_t* base = out + tile * 2 * half_bytes + (q / 8) * (kgs * 128) + kg * 128 + (q % 8) * 16;
    *reinterpret_cast<uint4*>(base) = hi;
    *reinterpret_cast<uint4*>(base + half_bytes) = lo;
  }
}

// F2 level -> hi/lo planes [cells][dp] fp16
__global__ void split_f2_kernel(const float* __restrict__ f2, int64_t cells, int d, int dp,
                                const uint32_t* maxbits, __half* __restrict__ out) {
  const int kgs = dp / 8;
  const int64_t total = cells * kgs;
  const float s = ldexpf(1.f, scale_exp(maxbits[1]));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kg = (int)(i % kgs);
    const int64_t c = i / kgs;
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kg * 8 + j;
      x[j] = k < d ? __ldg(f2 + c * d + k) : 0.f;
    }
    uint4 hi, lo;
    split8(x, s, hi, lo);
    *reinterpret_cast<uint4*>(out + c * dp + kg * 8) = hi;
    *reinterpret_cast<uint4*>(out + cells * dp + c * dp + kg * 8) = lo;
  }
}

struct CellRef {
  int level, cy, cx;
};

__device__ __forceinline__ CellRef cell_of(int g, const TilePlan* plans, const int* prefix,
                                           int levels) {
  int l = 0;
  while (l + 1 < levels && g >= prefix[l + 1]) ++l;
  CellRef c;
  c.level = l;
  new_cell(plans[l].B, plans[l].I, plans[l].has_i, g - prefix[l], c.cy, c.cx);
  return c;
}

__global__ void __launch_bounds__(THREADS) partial_contract_tc_kernel(TcParams T) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[NST + 2];  // stage_free[NST], acc_full, b_full
  __shared__ uint32_t s_tmem;
  __shared__ TilePlan s_plan[CVB_MAX_LEVELS];
  __shared__ int s_red[CVB_MAX_LEVELS][2][4];
  __shared__ int s_nvalid;
  __shared__ int s_prefix[CVB_MAX_LEVELS + 1];

  const PartialParams& P = T.P;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t tile = P.tile0 + blockIdx.x;
  const int dp = T.dp;
  const uint32_t half_bytes = (uint32_t)N * dp * 2;  // one of hi / lo
  const uint32_t b_bytes = 2 * half_bytes;
  const uint32_t sB = smem_u32(smem);
  const uint32_t sA = sB + b_bytes;
  const uint32_t bar_stage = smem_u32(&bars[0]);
  const uint32_t bar_acc = smem_u32(&bars[NST]);
  const uint32_t bar_b = smem_u32(&bars[NST + 1]);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    s_nvalid = 0;
    for (int i = 0; i < NST + 2; ++i) mbar_init(bar_stage + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t d_main = tmem, d_corr = tmem + 64;

  // B operand: the pre-split F1 tile image, one bulk async copy
  if (tid == 0) {
    mbar_expect_tx(bar_b, b_bytes);
    const uint8_t* src = T.f1s + tile * (int64_t)b_bytes;
    const uint32_t piece = b_bytes / 4;
    for (int i = 0; i < 4; ++i) bulk_g2s(sB + i * piece, src + i * piece, piece, bar_b);
  }

  // window-union tiler for every level (overlaps the B copy)
  plan_tile_all_levels(P, tile, s_plan, s_red, &s_nvalid);
  if (tid == 0) {
    s_prefix[0] = 0;
    for (int l = 0; l < P.levels; ++l) s_prefix[l + 1] = s_prefix[l] + s_plan[l].n_new;
  }
  __syncthreads();
  const int n_cells = s_prefix[P.levels];
  const int n_chunks = (n_cells + M - 1) / M;
  const int n_ks = dp / KS;
  const int n_steps = n_chunks * n_ks;

  const int rg = tid >> 3, r8 = tid & 7;
  const uint32_t row_off = rg * (KS / 8) * 128 + r8 * 16;  // A: SBO = 512 B
  int load_chunk = -1;
  const __half* src_hi = nullptr;
  const __half* src_lo = nullptr;

  auto issue_loads = [&](int c, int ks, int st) {
    if (c != load_chunk) {
      load_chunk = c;
      src_hi = nullptr;
      const int g = c * M + tid;
      if (g < n_cells) {
        const CellRef cr = cell_of(g, s_plan, s_prefix, P.levels);
        src_hi = T.f2s[cr.level] + ((int64_t)cr.cy * P.tw[cr.level] + cr.cx) * dp;
        src_lo = src_hi + T.plane[cr.level];
      }
    }
    if (src_hi != nullptr) {
      const uint32_t dst = sA + st * A_STAGE + row_off;
#pragma unroll
      for (int j = 0; j < KS / 8; ++j) {
        cp_async16(dst + j * 128, src_hi + ks * KS + j * 8);
        cp_async16(dst + A_HALF + j * 128, src_lo + ks * KS + j * 8);
      }
    }
    cp_async_commit();
  };

  if (n_steps > 0) issue_loads(0, 0, 0);
  if (tid == 0) mbar_wait(bar_b, 0);
  const float s_main = ldexpf(1.f, -(scale_exp(T.maxbits[0]) + scale_exp(T.maxbits[1])));
  const float s_corr = s_main * (1.f / (float)(1 << LOG2_LO));

  // step i = (chunk c, k-slice ks) uses stage st = i % NST; its n-th use
  // (n = i / NST) completes phase n of stage_free[st]
  int c = 0, ks = 0, st = 0;
  int nc = 0, nks = 1, nst = 1 % NST, nuse = (1 >= NST) ? 1 : 0;  // next step, stage use count
  if (nks == n_ks) {
    nks = 0;
    ++nc;
  }
  for (int i = 0; i < n_steps; ++i) {
    if (i + 1 < n_steps) {
      if (i + 1 >= NST) mbar_wait(bar_stage + 8 * nst, (nuse - 1) & 1);
      issue_loads(nc, nks, nst);
      cp_async_wait<1>();
      if (++nks == n_ks) {
        nks = 0;
        ++nc;
      }
      if (++nst == NST) {
        nst = 0;
        ++nuse;
      }
    } else {
      cp_async_wait<0>();
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_hi = sA + st * A_STAGE, a_lo = a_hi + A_HALF;
#pragma unroll
      for (int s = 0; s < KS / 16; ++s) {
        const uint32_t kstep = ks * (KS / 16) + s;
        const uint64_t dah = make_desc(a_hi + s * 256, 128, (KS / 8) * 128);
        const uint64_t dal = make_desc(a_lo + s * 256, 128, (KS / 8) * 128);
        const uint64_t dbh = make_desc(sB + kstep * 256, 128, (dp / 8) * 128);
        const uint64_t dbl = make_desc(sB + half_bytes + kstep * 256, 128, (dp / 8) * 128);
        const uint32_t acc = (ks > 0 || s > 0) ? 1u : 0u;
        mma_f16(d_main, dah, dbh, acc);
        mma_f16(d_corr, dah, dbl, acc);
        mma_f16(d_corr, dal, dbh, 1u);
      }
      mma_commit(bar_stage + 8 * st);
      if (ks == n_ks - 1) mma_commit(bar_acc);
    }
    if (ks == n_ks - 1) {
      // ---- epilogue of chunk c ----
      mbar_wait(bar_acc, c & 1);
      tc_fence_after();
      const int g = c * M + tid;
      const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
      float vm[32], vc[32];
      float* dst = nullptr;  // tile block of the cell's level: [query row][slot][8]
      int64_t plane = 0, slot = 0;
      if (g < n_cells) {
        const CellRef cr = cell_of(g, s_plan, s_prefix, P.levels);
        const int ch = P.ch[cr.level], cw = P.cw[cr.level];
        plane = (int64_t)ch * cw * TQW;
        slot = slot_of(cr.cy, cr.cx, ch, cw);
        dst = P.cache[cr.level] + tile * plane * TQH + slot * TQW;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(d_main + lane_base + h * 32, vm);
        tmem_ld32(d_corr + lane_base + h * 32, vc);
        if (dst != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o;
            o.x = fmaf(vc[j + 0], s_corr, vm[j + 0] * s_main);
            o.y = fmaf(vc[j + 1], s_corr, vm[j + 1] * s_main);
            o.z = fmaf(vc[j + 2], s_corr, vm[j + 2] * s_main);
            o.w = fmaf(vc[j + 3], s_corr, vm[j + 3] * s_main);
            const int q = h * 32 + j;  // queries q..q+3 share query row q/8
            *reinterpret_cast<float4*>(dst + (q >> 3) * plane + (q & 7)) = o;
          }
        }
      }
      tc_fence_before();
      __syncthreads();
    }
    if (++ks == n_ks) {
      ks = 0;
      ++c;
    }
    if (++st == NST) st = 0;
  }
  if (n_steps == 0 && tid == 0) mbar_wait(bar_b, 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
  }
}

}  // namespace tc

// ---------------------------------------------------------------------------
// Persistent, warp-specialised variant (default).  One CTA per SM walks the
// tiles blockIdx.x, blockIdx.x + gridDim.x, ...; the roles communicate only
// through mbarrier rings, so the next tile's planning, B image and A rows are
// in flight while the current tile's MMAs run and the previous chunk's
// accumulators drain:
//   warp 0       B producer: one 64 KB bulk copy per tile into a 2-deep ring
//   warp 1       MMA issuer (one thread): 3 tcgen05.mma per K=16 step
//   warps 2-3    planner: the window-union tiler for every level of a tile
//   warps 4-7    A producers: one A row (cell) per thread, cp.async into a
//                4-stage ring, fence.proxy.async + arrive once a stage landed
//   warps 8-11   epilogue: tcgen05.ld of a 2-deep TMEM accumulator ring,
//                main + 2^-11 corr, cache-slot stores
// ---------------------------------------------------------------------------
namespace tcp {

constexpr int NST = 4;   // A stages
constexpr int NB = 2;    // B buffers
constexpr int NPL = 4;   // plan slots (the planner runs up to 3 tiles ahead)
constexpr int THREADS = 384;
constexpr uint32_t SPIN_LIMIT = 1u << 24;  // watchdog: trap instead of hanging

struct PlanSlot {
  TilePlan plan[CVB_MAX_LEVELS];
  int prefix[CVB_MAX_LEVELS + 1];
  int n_cells;
};

struct Ctl {
  uint64_t plan_full[NPL], plan_empty[NPL];
  uint64_t b_full[NB], b_empty[NB];
  uint64_t a_full[NST], a_empty[NST];
  uint64_t acc_full[2], acc_empty[2];
  PlanSlot slot[NPL];
  int red[CVB_MAX_LEVELS][2][4];
  int nv[2];
  uint32_t tmem;
};

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// full barriers: the k-th completion has parity k&1; empty barriers: the
// producer's k-th wait passes on parity (k&1)^1 (a fresh barrier counts as
// having completed the phase before phase 0).
__device__ __forceinline__ void wait_full(uint32_t bar, uint32_t k) {
  for (uint32_t n = 0; !mbar_try(bar, k & 1u); ++n)
    if (n > SPIN_LIMIT) __trap();
}
__device__ __forceinline__ void wait_empty(uint32_t bar, uint32_t k) {
  for (uint32_t n = 0; !mbar_try(bar, (k & 1u) ^ 1u); ++n)
    if (n > SPIN_LIMIT) __trap();
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1) partial_contract_tcp_kernel(tc::TcParams T) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const PartialParams& P = T.P;
  const int dp = T.dp;
  const uint32_t half_bytes = (uint32_t)tc::N * dp * 2;
  const uint32_t b_bytes = 2 * half_bytes;
  uint8_t* sB = smem;                                   // NB x b_bytes
  uint8_t* sA = smem + NB * b_bytes;                    // NST x A_STAGE
  Ctl& C = *reinterpret_cast<Ctl*>(sA + NST * tc::A_STAGE);
  const uint32_t uB = tc::smem_u32(sB), uA = tc::smem_u32(sA);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_ks = dp / tc::KS;
  auto U = [](const uint64_t& b) { return tc::smem_u32(&b); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     tc::smem_u32(&C.tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < NPL; ++i) {
      tc::mbar_init(U(C.plan_full[i]), 64);
      tc::mbar_init(U(C.plan_empty[i]), 1 + 1 + 128 + 128);
    }
    for (int i = 0; i < NB; ++i) {
      tc::mbar_init(U(C.b_full[i]), 1);
      tc::mbar_init(U(C.b_empty[i]), 1);
    }
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(U(C.a_full[i]), 128);
      tc::mbar_init(U(C.a_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(U(C.acc_full[i]), 1);
      tc::mbar_init(U(C.acc_empty[i]), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = C.tmem;

  if (warp == 0) {
    // ---------------- B producer ----------------
    if (lane == 0) {
      uint32_t kb = 0;
      for (int64_t it = 0;; ++it) {
        const int64_t t = blockIdx.x + it * gridDim.x;
        if (t >= P.ntile) break;
        const int s = (int)(it % NPL);
        wait_full(U(C.plan_full[s]), (uint32_t)(it / NPL));
        if (C.slot[s].n_cells > 0) {
          const int tb = kb % NB;
          wait_empty(U(C.b_empty[tb]), kb / NB);
          tc::mbar_expect_tx(U(C.b_full[tb]), b_bytes);
          const uint8_t* src = T.f1s + (P.tile0 + t) * (int64_t)b_bytes;
          const uint32_t piece = b_bytes / 4;
          for (int i = 0; i < 4; ++i)
            tc::bulk_g2s(uB + tb * b_bytes + i * piece, src + i * piece, piece, U(C.b_full[tb]));
          ++kb;
        }
        arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t kb = 0, g = 0, cg = 0;
      for (int64_t it = 0;; ++it) {
        const int64_t t = blockIdx.x + it * gridDim.x;
        if (t >= P.ntile) break;
        const int s = (int)(it % NPL);
        wait_full(U(C.plan_full[s]), (uint32_t)(it / NPL));
        const int n = C.slot[s].n_cells;
        if (n > 0) {
          const int tb = kb % NB;
          wait_full(U(C.b_full[tb]), kb / NB);
          const uint32_t bh = uB + tb * b_bytes, bl = bh + half_bytes;
          const int n_chunks = (n + tc::M - 1) / tc::M;
          for (int c = 0; c < n_chunks; ++c, ++cg) {
            const int ab = cg & 1;
            wait_empty(U(C.acc_empty[ab]), cg >> 1);
            tc::tc_fence_after();
            const uint32_t d_main = tmem + ab * 128, d_corr = d_main + 64;
            for (int ks = 0; ks < n_ks; ++ks, ++g) {
              const int st = g % NST;
              wait_full(U(C.a_full[st]), g / NST);
              tc::tc_fence_after();
              const uint32_t a_hi = uA + st * tc::A_STAGE, a_lo = a_hi + tc::A_HALF;
#pragma unroll
              for (int k2 = 0; k2 < tc::KS / 16; ++k2) {
                const uint32_t kstep = ks * (tc::KS / 16) + k2;
                const uint64_t dah = tc::make_desc(a_hi + k2 * 256, 128, (tc::KS / 8) * 128);
                const uint64_t dal = tc::make_desc(a_lo + k2 * 256, 128, (tc::KS / 8) * 128);
                const uint64_t dbh = tc::make_desc(bh + kstep * 256, 128, (dp / 8) * 128);
                const uint64_t dbl = tc::make_desc(bl + kstep * 256, 128, (dp / 8) * 128);
                const uint32_t acc = (ks > 0 || k2 > 0) ? 1u : 0u;
                tc::mma_f16(d_main, dah, dbh, acc);
                tc::mma_f16(d_corr, dah, dbl, acc);
                tc::mma_f16(d_corr, dal, dbh, 1u);
              }
              tc::mma_commit(U(C.a_empty[st]));
            }
            tc::mma_commit(U(C.acc_full[ab]));
          }
          tc::mma_commit(U(C.b_empty[tb]));
          ++kb;
        }
        arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp < 4) {
    // ---------------- planner (64 threads) ----------------
    const int pt = tid - 64, pw = pt >> 5;
    const int r = P.radius;
    for (int64_t it = 0;; ++it) {
      const int64_t t = blockIdx.x + it * gridDim.x;
      if (t >= P.ntile) break;
      const int64_t tile = P.tile0 + t;
      const int s = (int)(it % NPL);
      wait_empty(U(C.plan_empty[s]), (uint32_t)(it / NPL));
      const int tile_y = (int)(tile / P.tiles_x), tile_x = (int)(tile % P.tiles_x);
      const int py = tile_y * TQH + pt / TQW, px = tile_x * TQW + pt % TQW;
      const bool valid = py < P.h1 && px < P.w1;
      double x = 0.0, y = 0.0;
      if (valid) load_coord(P.coords, P.f64, (int64_t)py * P.w1 + px, x, y);
      const unsigned vote = __ballot_sync(0xffffffffu, valid);
      if (lane == 0) C.nv[pw] = __popc(vote);
      for (int l = 0; l < P.levels; ++l) {
        int ylo = INT_MAX, yhi = INT_MIN, xlo = INT_MAX, xhi = INT_MIN;
        if (valid) {
          const LevelPos lp = level_pos(x, y, l);
          ylo = yhi = clamp_anchor(lp.y0, r, P.th[l]);
          xlo = xhi = clamp_anchor(lp.x0, r, P.tw[l]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
          yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
          xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
          xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, o));
        }
        if (lane == 0) {
          C.red[l][pw][0] = ylo;
          C.red[l][pw][1] = yhi;
          C.red[l][pw][2] = xlo;
          C.red[l][pw][3] = xhi;
        }
      }
      named_sync(1, 64);
      PlanSlot& S = C.slot[s];
      if (pt < P.levels) {
        const int level = pt;
        const int th = P.th[level], tw = P.tw[level];
        int32_t* meta = P.meta + (tile * P.levels + level) * CVB_META_INTS;
        const int nv = C.nv[0] + C.nv[1];
        Box B;
        B.ylo = max(min(C.red[level][0][0], C.red[level][1][0]) - r, 0);
        B.yhi = min(max(C.red[level][0][1], C.red[level][1][1]) + r + 1, th - 1);
        B.xlo = max(min(C.red[level][0][2], C.red[level][1][2]) - r, 0);
        B.xhi = min(max(C.red[level][0][3], C.red[level][1][3]) + r + 1, tw - 1);
        int status = ST_OK;
        if (nv == 0 || B.empty()) {
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
        S.plan[level] = TilePlan{B, I, (int)has_i, n_new, nv, status};
        meta[0] = B.ylo;
        meta[1] = B.yhi;
        meta[2] = B.xlo;
        meta[3] = B.xhi;
        meta[4] = status;
        meta[5] = n_new;
        if (P.counters != nullptr) {
          if (n_new > 0) {
            atomicAdd(P.counters + 0, (unsigned long long)n_new * nv);
            atomicAdd(P.counters + 1, (unsigned long long)n_new);
          }
          if (status == ST_OVERFLOW) atomicAdd(P.counters + 2, 1ULL);
          if (status == ST_EMPTY) atomicAdd(P.counters + 3, 1ULL);
        }
      }
      named_sync(1, 64);
      if (pt == 0) {
        S.prefix[0] = 0;
        for (int l = 0; l < P.levels; ++l) S.prefix[l + 1] = S.prefix[l] + S.plan[l].n_new;
        S.n_cells = S.prefix[P.levels];
      }
      named_sync(1, 64);
      arrive(U(C.plan_full[s]));
    }
  } else if (warp < 8) {
    // ---------------- A producers (128 threads, one A row each) ----------------
    const int ap = tid - 128;
    const uint32_t row_off = (ap >> 3) * (tc::KS / 8) * 128 + (ap & 7) * 16;
    uint32_t g = 0;
    for (int64_t it = 0;; ++it) {
      const int64_t t = blockIdx.x + it * gridDim.x;
      if (t >= P.ntile) break;
      const int s = (int)(it % NPL);
      wait_full(U(C.plan_full[s]), (uint32_t)(it / NPL));
      const PlanSlot& S = C.slot[s];
      const int n = S.n_cells;
      const int n_chunks = (n + tc::M - 1) / tc::M;
      // stages issued but not yet published (at most NST-1 in flight)
      int n_pend = 0;
      uint32_t pend_st0 = 0, pend_st1 = 0;
      for (int c = 0; c < n_chunks; ++c) {
        const __half* src_hi = nullptr;
        const __half* src_lo = nullptr;
        const int gi = c * tc::M + ap;
        if (gi < n) {
          const tc::CellRef cr = tc::cell_of(gi, S.plan, S.prefix, P.levels);
          src_hi = T.f2s[cr.level] + ((int64_t)cr.cy * P.tw[cr.level] + cr.cx) * dp;
          src_lo = src_hi + T.plane[cr.level];
        }
        for (int ks = 0; ks < n_ks; ++ks, ++g) {
          const int st = g % NST;
          wait_empty(U(C.a_empty[st]), g / NST);
          if (src_hi != nullptr) {
            const uint32_t dst = uA + st * tc::A_STAGE + row_off;
#pragma unroll
            for (int j = 0; j < tc::KS / 8; ++j) {
              tc::cp_async16(dst + j * 128, src_hi + ks * tc::KS + j * 8);
              tc::cp_async16(dst + tc::A_HALF + j * 128, src_lo + ks * tc::KS + j * 8);
            }
          }
          tc::cp_async_commit();
          if (n_pend == 2) {  // the oldest stage landed: publish it to the tensor core
            tc::cp_async_wait<2>();
            tc::fence_proxy_async();
            arrive(U(C.a_full[pend_st0]));
            pend_st0 = pend_st1;
            pend_st1 = st;
          } else if (n_pend == 1) {
            pend_st1 = st;
            n_pend = 2;
          } else {
            pend_st0 = st;
            n_pend = 1;
          }
        }
      }
      if (n_pend == 2) {
        tc::cp_async_wait<1>();
        tc::fence_proxy_async();
        arrive(U(C.a_full[pend_st0]));
        pend_st0 = pend_st1;
        n_pend = 1;
      }
      if (n_pend == 1) {
        tc::cp_async_wait<0>();
        tc::fence_proxy_async();
        arrive(U(C.a_full[pend_st0]));
      }
      arrive(U(C.plan_empty[s]));
    }
  } else {
    // ---------------- epilogue (128 threads = TMEM lanes) ----------------
    const int ep = tid - 256;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const float s_main =
        ldexpf(1.f, -(tc::scale_exp(T.maxbits[0]) + tc::scale_exp(T.maxbits[1])));
    const float s_corr = s_main * (1.f / (float)(1 << tc::LOG2_LO));
    uint32_t cg = 0;
    for (int64_t it = 0;; ++it) {
      const int64_t t = blockIdx.x + it * gridDim.x;
      if (t >= P.ntile) break;
      const int64_t tile = P.tile0 + t;
      const int s = (int)(it % NPL);
      wait_full(U(C.plan_full[s]), (uint32_t)(it / NPL));
      const PlanSlot& S = C.slot[s];
      const int n = S.n_cells;
      const int n_chunks = (n + tc::M - 1) / tc::M;
      for (int c = 0; c < n_chunks; ++c, ++cg) {
        const int ab = cg & 1;
        wait_full(U(C.acc_full[ab]), cg >> 1);
        tc::tc_fence_after();
        const int gi = c * tc::M + ep;
        float* dst = nullptr;
        int64_t plane = 0;
        if (gi < n) {
          const tc::CellRef cr = tc::cell_of(gi, S.plan, S.prefix, P.levels);
          const int ch = P.ch[cr.level], cw = P.cw[cr.level];
          plane = (int64_t)ch * cw * TQW;
          dst = P.cache[cr.level] + tile * plane * TQH +
                (int64_t)slot_of(cr.cy, cr.cx, ch, cw) * TQW;
        }
        float vm[32], vc[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tc::tmem_ld32(tmem + ab * 128 + lane_base + h * 32, vm);
          tc::tmem_ld32(tmem + ab * 128 + 64 + lane_base + h * 32, vc);
          if (dst != nullptr) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o;
              o.x = fmaf(vc[j + 0], s_corr, vm[j + 0] * s_main);
              o.y = fmaf(vc[j + 1], s_corr, vm[j + 1] * s_main);
              o.z = fmaf(vc[j + 2], s_corr, vm[j + 2] * s_main);
              o.w = fmaf(vc[j + 3], s_corr, vm[j + 3] * s_main);
              const int q = h * 32 + j;
              *reinterpret_cast<float4*>(dst + (q >> 3) * plane + (q & 7)) = o;
            }
          }
        }
        tc::tc_fence_before();
        arrive(U(C.acc_empty[ab]));
      }
      arrive(U(C.plan_empty[s]));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

size_t smem_bytes(int dp) {
  return (size_t)NB * 2 * tc::N * dp * 2 + (size_t)NST * tc::A_STAGE + sizeof(Ctl) + 1024;
}

}  // namespace tcp

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_tc_sizes(const cvb_partial_desc* desc, int64_t* f1_split_bytes,
                 int64_t* f2_split_bytes_per_level) {
  CVB_REQUIRE(desc, "tc_sizes: null desc");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  const int dp = (int)ceil_div(desc->d, tc::KS) * tc::KS;
  CVB_REQUIRE(dp <= tc::MAX_DP, "tensor-core path supports D <= %d", tc::MAX_DP);
  const int64_t nt = ceil_div(desc->h1, TQH) * ceil_div(desc->w1, TQW);
  if (f1_split_bytes) *f1_split_bytes = nt * 2 * tc::N * dp * 2;
  if (f2_split_bytes_per_level)
    for (int l = 0; l < desc->levels; ++l)
      f2_split_bytes_per_level[l] = 2 * (int64_t)desc->th[l] * desc->tw[l] * dp * 2;
  return CVB_OK;
}

int cvb_tc_prepare(const cvb_partial_desc* desc, const float* f1,
                   const float* const* f2_levels_host, void* f1_split,
                   void* const* f2_split_host, uint32_t* maxbits, void* stream) {
  int64_t f1b = 0;
  int st = cvb_tc_sizes(desc, &f1b, nullptr);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(f1 && f2_levels_host && f1_split && f2_split_host && maxbits,
              "tc_prepare: null pointer");
  cudaStream_t s = as_stream(stream);
  const int dp = (int)ceil_div(desc->d, tc::KS) * tc::KS;
  const int64_t n1 = (int64_t)desc->h1 * desc->w1 * desc->d;
  const int64_t n2 = (int64_t)desc->th[0] * desc->tw[0] * desc->d;
  cudaMemsetAsync(maxbits, 0, 2 * sizeof(uint32_t), s);
  tc::absmax_kernel<<<148 * 4, 256, 0, s>>>(f1, n1, maxbits);
  if ((st = check_launch("tc_absmax")) != CVB_OK) return st;
  tc::absmax_kernel<<<148 * 4, 256, 0, s>>>(f2_levels_host[0], n2, maxbits + 1);
  if ((st = check_launch("tc_absmax")) != CVB_OK) return st;
  const int tiles_x = (int)ceil_div(desc->w1, TQW);
  const int64_t n_tiles = ceil_div(desc->h1, TQH) * tiles_x;
  tc::split_f1_kernel<<<148 * 8, 256, 0, s>>>(f1, desc->h1, desc->w1, desc->d, dp, tiles_x,
                                              n_tiles, maxbits,
                                              reinterpret_cast<uint8_t*>(f1_split));
  if ((st = check_launch("tc_split_f1")) != CVB_OK) return st;
  for (int l = 0; l < desc->levels; ++l) {
    CVB_REQUIRE(f2_levels_host[l] && f2_split_host[l], "tc_prepare: null level pointer");
    tc::split_f2_kernel<<<148 * 8, 256, 0, s>>>(
        f2_levels_host[l], (int64_t)desc->th[l] * desc->tw[l], desc->d, dp, maxbits,
        reinterpret_cast<__half*>(f2_split_host[l]));
    if ((st = check_launch("tc_split_f2")) != CVB_OK) return st;
  }
  return CVB_OK;
}

int cvb_partial_contract_tc(const cvb_partial_desc* desc, const float* f1,
                            const float* const* f2_levels_host, const void* f1_split,
                            const void* const* f2_split_host, const uint32_t* maxbits,
                            const void* coords, int32_t* meta, float* const* cache_levels_host,
                            unsigned long long* counters, int32_t flags, void* stream) {
  tc::TcParams T;
  int st = cvb_internal_build_params(desc, f1, f2_levels_host, coords, 1.0f, meta,
                                     cache_levels_host, counters, flags, T.P);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(!(flags & CVB_STRICT), "tensor-core contraction has no strict mode");
  CVB_REQUIRE(f1_split && f2_split_host && maxbits, "partial_contract_tc: null pointer");
  T.dp = (int)ceil_div(desc->d, tc::KS) * tc::KS;
  CVB_REQUIRE(T.dp <= tc::MAX_DP, "tensor-core path supports D <= %d", tc::MAX_DP);
  T.f1s = reinterpret_cast<const uint8_t*>(f1_split);
  T.maxbits = maxbits;
  for (int l = 0; l < CVB_MAX_LEVELS; ++l) {
    const bool used = l < desc->levels;
    T.f2s[l] = used ? reinterpret_cast<const __half*>(f2_split_host[l]) : nullptr;
    T.plane[l] = used ? (int64_t)desc->th[l] * desc->tw[l] * T.dp : 0;
    if (used) CVB_REQUIRE(T.f2s[l], "partial_contract_tc: null level pointer");
  }
  if (T.P.ntile == 0) return CVB_OK;
  static int persistent = -1;
  if (persistent < 0) {
    const char* e = getenv("CVB_TC_PERSISTENT");
    persistent = (e == nullptr || e[0] != '0') ? 1 : 0;
  }
  if (persistent) {
    static int n_sms = 0;
    static bool attr_p = false;
    if (n_sms == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const size_t smem = tcp::smem_bytes(T.dp);
    if (!attr_p) {
      cudaFuncSetAttribute(tcp::partial_contract_tcp_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcp::smem_bytes(tc::MAX_DP));
      attr_p = true;
    }
    const int64_t grid = T.P.ntile < n_sms ? T.P.ntile : n_sms;
    tcp::partial_contract_tcp_kernel<<<(unsigned)grid, tcp::THREADS, smem, as_stream(stream)>>>(T);
    return check_launch("partial_contract_tcp");
  }
  const size_t smem = (size_t)2 * tc::N * T.dp * 2 + (size_t)tc::NST * tc::A_STAGE;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc::partial_contract_tc_kernel,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(tc::MAX_DP * 2 * 2 * tc::N + tc::NST * tc::A_STAGE));
    attr_set = true;
  }
  tc::partial_contract_tc_kernel<<<(unsigned)T.P.ntile, tc::THREADS, smem, as_stream(stream)>>>(T);
  return check_launch("partial_contract_tc");
}

}  // extern "C"
