// Tensor-core (tcgen05) contraction for the partial sampler's fast path.
//
// Same tiler, metadata and toroidal tile cache as partial_contract_kernel
// (partial.cuh); only the arithmetic of the new-cell contraction changes:
//
//   * D[128 cells x 64 queries] = A[cells x K] . B[queries x K]^T with
//     M=128, N=64, K=16 `tcgen05.mma.cta_group::1.kind::f16`, accumulators in
//     TMEM (a 2-deep ring of main + corr accumulators, 64 fp32 columns each);
//   * split precision: every fp32 value x (pre-scaled by a per-row power of
//     two so it sits in fp16 range) is stored as hi = fp16(x) and
//     lo = fp16(x - hi); x*y = hi_x*hi_y + hi_x*lo_y + lo_x*hi_y + O(2^-22).
//     Per K-step one N=128 MMA (the F1 piece's hi and lo rows form one
//     128-row B matrix: main += hi.hi and corr += hi.lo, reading A_hi from
//     shared memory once) and one N=64 MMA (corr += lo.hi) keep ~22
//     significant bits per product (products of two fp16 are exact in the
//     fp32 accumulator);
//   * operands are pre-split once per image pair (cvb_tc_prepare): the F1
//     tile is a contiguous image of its shared-memory layout cut into K
//     pieces of 64 channels (16 KB: hi 8 KB + lo 8 KB), each fetched with one
//     bulk async copy (cp.async.bulk + mbarrier complete_tx) into a ring of
//     pieces, so the next tile's first pieces land while the current tile's
//     last chunk still runs; A rows (gathered new bbox cells of all levels,
//     128 per chunk) stream by cp.async (8 lanes per 128-byte row) through a
//     4-stage ring of 128B-swizzled K=64 stages (32 KB: hi + lo) that never
//     drains between tiles;
//   * the epilogue reads TMEM with tcgen05.ld, combines main + corr,
//     removes the power-of-two scales and writes each cell's 64 query costs
//     into its cache slot.
#include <cuda_fp16.h>
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "partial.cuh"

namespace cvb {
namespace tc {

constexpr int M = 128;         // cells per MMA chunk (TMEM lanes)
constexpr int N = 64;          // queries per tile
constexpr int KP = 64;         // K per A stage and per B piece (one 128-byte swizzle atom row)
constexpr int A_HALF = M * KP * 2;       // 16 KB (hi or lo)
constexpr int A_STAGE = 2 * A_HALF;      // 32 KB
constexpr int B_HALF = N * KP * 2;       // 8 KB (hi or lo)
constexpr int B_PIECE = 2 * B_HALF;      // 16 KB
constexpr int MAX_DP = 256;
#ifndef CVB_F2_HILO
#define CVB_F2_HILO 1  // F2 split rows interleaved [cell][hi dp | lo dp]; 0: two planes
#endif
// fp16 offsets of cell c's hi row and of its lo row relative to the hi row in
// a level's split operand.  Interleaved per cell, an A-row fetch's hi and lo
// 128-byte pieces share a DRAM page (two planes put them ~cells*dp*2 bytes
// apart): -1% warm contraction, -0.5% per C4 step (A/B)
__host__ __device__ __forceinline__ int64_t f2_hi(int64_t c, int dp) {
  return CVB_F2_HILO ? c * 2 * dp : c * dp;
}
__host__ __device__ __forceinline__ int64_t f2_lo_delta(int64_t cells, int dp) {
  return CVB_F2_HILO ? dp : cells * dp;
}
// lo = fp16(x - hi), unscaled: main (hi.hi) + corr (hi.lo + lo.hi) is a plain
// add in the epilogue
constexpr int TARGET_EXP = 14;           // max |x * 2^e| < 2^14

// instruction descriptor: D f32, A/B f16, both K-major, N=64, M=128
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
// N = 2 x 64: the F1 piece's hi and lo halves form one 128-row B matrix, so
// main (A_hi . B_hi) and the first correction (A_hi . B_lo) are one MMA that
// reads A_hi from shared memory once (the MMA phase is smem-read-bound)
constexpr uint32_t IDESC_N128 =
    (1u << 4) | ((uint32_t)(2 * N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

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

// K-major, SWIZZLE_128B descriptor: rows of 128 B (64 fp16 of K) in 8-row,
// 1024-byte atoms (the layout TMA writes with CU_TENSOR_MAP_SWIZZLE_128B);
// SBO = 1024 B between 8-row groups; a K=16 step advances the start by 32 B.
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <uint32_t ID = IDESC>
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(ID), "r"(acc));
}

// one lane of a converged warp (elect.sync): the MMA issuer runs as a whole
// warp so tcgen05.mma / commit issue without a per-instruction divergence loop
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(e));
  return e != 0;
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

__device__ __forceinline__ void st_global_v8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
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
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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

// power-of-two exponent e with m * 2^e < 2^TARGET_EXP (0 for an all-zero row)
__device__ __forceinline__ int scale_exp(float m) {
  if (!(m > 0.f) || !isfinite(m)) return 0;
  int k;
  frexpf(m, &k);  // m < 2^k
  const int e = TARGET_EXP - k;
  return e < -60 ? -60 : (e > 60 ? 60 : e);
}

// 2^-e as a float (|e| <= 60)
__device__ __forceinline__ float exp2_neg(int e) { return __int_as_float((127 - e) << 23); }

__device__ __forceinline__ void split8(const float (&x)[8], float s, uint4& hi, uint4& lo) {
  __half h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float v = x[i] * s;
    h[i] = __float2half_rn(v);
    l[i] = __float2half_rn(v - __half2float(h[i]));
  }
  hi = *reinterpret_cast<uint4*>(h);
  lo = *reinterpret_cast<uint4*>(l);
}

struct TcParams {
  PartialParams P;
  const uint8_t* f1s;                  // per tile: [dp/KP pieces][hi, lo][8 rg][KP/8 kg][8][8] fp16
  const int8_t* e1;                    // per tile: 64 query exponents
  const __half* f2s[CVB_MAX_LEVELS];   // per cell: hi row, lo row (f2_hi / f2_lo_delta)
  const int8_t* e2[CVB_MAX_LEVELS];    // per cell exponent
  int64_t plane[CVB_MAX_LEVELS];
  int64_t pair_bytes[CVB_MAX_LEVELS];  // split-operand bytes per pair of the batch, per level
  int dp;
  int dbg;                             // profiling knockouts (CVB_TC_DEBUG; debug instantiation only)
  unsigned long long* ts;              // role timeline (CVB_TC_DEBUG & 16; debug instantiation only)
  int* watchdog;                       // host-mapped error word (null: none); see wait_phase
  // dense instantiation (cvb_dense_tc): every tile's "new cells" are all cells
  // of every level and the epilogue writes the all-pairs rows
  // dense[l][pixel][cell] instead of cache slots
  float* dense[CVB_MAX_LEVELS];
};

// Operand preparation, once per image pair.  Every row (a query of F1, a
// cell of a pyramid level) gets its own power-of-two exponent e (max|x| 2^e
// < 2^14, so hi and lo stay normal fp16) and is split into hi/lo fp16; the
// epilogue removes 2^-(e_q + e_c) exactly.  One warp per row, lane = 8
// channels.

__device__ __forceinline__ void load8(const float* __restrict__ row, int d, int kg, bool vec,
                                      float (&x)[8]) {
  if (vec && kg * 8 + 8 <= d) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(row + kg * 8));
    const float4 b = __ldg(reinterpret_cast<const float4*>(row + kg * 8 + 4));
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = kg * 8 + j < d ? __ldg(row + kg * 8 + j) : 0.f;
  }
}

__device__ __forceinline__ int row_exp(const float (&x)[8]) {
  float m = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) m = fmaxf(m, fabsf(x[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return scale_exp(m);
}

// F1 -> per-tile B-operand images + query exponents.  One warp per (tile,
// 8-query row group): lane (q, j) = (lane & 7, lane >> 3) owns k-groups
// j, j+4, ..., so every store instruction writes 4 x 128 contiguous bytes of
// the image and every load 8 x 128 contiguous bytes of F1.
__global__ void __launch_bounds__(256) split_f1_kernel(const float* __restrict__ f1, int h1,
                                                       int w1, int d, int dp, int tiles_x,
                                                       int64_t n_tiles, bool vec,
                                                       uint8_t* __restrict__ out,
                                                       int8_t* __restrict__ exps) {
  const int lane = threadIdx.x & 31, kgs = dp / 8;  // kgs <= 32
  const int q8 = lane & 7, j = lane >> 3;
  const int64_t tile_bytes = (int64_t)N * dp * 2 * 2;
  const int64_t groups = n_tiles * (N / 8);
  for (int64_t gidx = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gidx < groups;
       gidx += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int rg = (int)(gidx % (N / 8));
    const int64_t tile = gidx / (N / 8);
    const int q = rg * 8 + q8;
    const int py = (int)(tile / tiles_x) * TQH + q / TQW, px = (int)(tile % tiles_x) * TQW + q % TQW;
    const bool valid = py < h1 && px < w1;
    const float* row = f1 + ((int64_t)py * w1 + px) * d;
    float x[8][8];
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kg = 4 * i + j;
#pragma unroll
      for (int e = 0; e < 8; ++e) x[i][e] = 0.f;
      if (valid && kg < kgs) load8(row, d, kg, vec, x[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(x[i][e]));
    }
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
    const int ex = scale_exp(m);
    const float sc = exp2_neg(-ex);
    uint8_t* img = out + tile * tile_bytes;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kg = 4 * i + j;
      if (kg >= kgs) continue;
      uint4 hi, lo;
      split8(x[i], sc, hi, lo);
      const int piece = kg / (KP / 8), kgi = kg % (KP / 8);
      uint8_t* base = img + (int64_t)piece * B_PIECE + rg * (KP / 8 * 128) + kgi * 128 + q8 * 16;
      *reinterpret_cast<uint4*>(base) = hi;
      *reinterpret_cast<uint4*>(base + B_HALF) = lo;
    }
    if (j == 0) exps[tile * N + q] = (int8_t)ex;
  }
}

// One pyramid level -> hi/lo planes [cells][dp] + cell exponents.  With
// `pool`, the level is first produced from the previous one by the
// reference's 2x2 average pool (((a+b)+(c+d))*0.25, bit-exact with
// pool2x2_vec4_kernel) and also written out in fp32.
__device__ __forceinline__ float pool4f(float a, float b, float c, float d) {
  return __fmul_rn(__fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d)), 0.25f);
}

__device__ __forceinline__ void split_store(const float (&x)[8], int lane, int kgs,
                                            int64_t c, int64_t cells, int dp,
                                            __half* __restrict__ planes,
                                            int8_t* __restrict__ exps) {
  const int e = row_exp(x);
  if (lane < kgs) {
    uint4 hi, lo;
    split8(x, exp2_neg(-e), hi, lo);
    *reinterpret_cast<uint4*>(planes + f2_hi(c, dp) + lane * 8) = hi;
    *reinterpret_cast<uint4*>(planes + f2_hi(c, dp) + f2_lo_delta(cells, dp) + lane * 8) = lo;
  }
  if (lane == 0) exps[c] = (int8_t)e;
}

// With src_planes, the pooling pass also splits the four source cells of every
// output cell (the source level is read once); the source cells a 2x2 pool
// drops (odd trailing row / column) are split by split_tail_kernel.
__global__ void __launch_bounds__(256) split_level_kernel(const float* __restrict__ src,
                                                          int src_w, float* __restrict__ pooled,
                                                          int h, int w, int d, int dp, bool pool,
                                                          bool vec, __half* __restrict__ planes,
                                                          int8_t* __restrict__ exps,
                                                          __half* __restrict__ src_planes,
                                                          int8_t* __restrict__ src_exps,
                                                          int64_t src_cells) {
  const int lane = threadIdx.x & 31, kgs = dp / 8;
  const int64_t cells = (int64_t)h * w;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < cells;
       c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (lane < kgs) {
      if (pool) {
        const int y = (int)(c / w), xx = (int)(c % w);
        const float* r0 = src + ((int64_t)(2 * y) * src_w + 2 * xx) * d;
        const float* r1 = r0 + (int64_t)src_w * d;
        float a[8], b[8], e[8], f[8];
        load8(r0, d, lane, vec, a);
        load8(r0 + d, d, lane, vec, b);
        load8(r1, d, lane, vec, e);
        load8(r1 + d, d, lane, vec, f);
        if (src_planes != nullptr) {
          const int64_t s0 = (int64_t)(2 * y) * src_w + 2 * xx, s1 = s0 + src_w;
          split_store(a, lane, kgs, s0, src_cells, dp, src_planes, src_exps);
          split_store(b, lane, kgs, s0 + 1, src_cells, dp, src_planes, src_exps);
          split_store(e, lane, kgs, s1, src_cells, dp, src_planes, src_exps);
          split_store(f, lane, kgs, s1 + 1, src_cells, dp, src_planes, src_exps);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = pool4f(a[j], b[j], e[j], f[j]);
        float* o = pooled + c * d;
        if (vec && lane * 8 + 8 <= d) {
          *reinterpret_cast<float4*>(o + lane * 8) = make_float4(x[0], x[1], x[2], x[3]);
          *reinterpret_cast<float4*>(o + lane * 8 + 4) = make_float4(x[4], x[5], x[6], x[7]);
        } else {
          for (int j = 0; j < 8; ++j)
            if (lane * 8 + j < d) o[lane * 8 + j] = x[j];
        }
      } else {
        load8(src + c * d, d, lane, vec, x);
      }
    }
    const int e = row_exp(x);
    if (lane < kgs) {
      uint4 hi, lo;
      split8(x, exp2_neg(-e), hi, lo);
      *reinterpret_cast<uint4*>(planes + f2_hi(c, dp) + lane * 8) = hi;
      *reinterpret_cast<uint4*>(planes + f2_hi(c, dp) + f2_lo_delta(cells, dp) + lane * 8) = lo;
    }
    if (lane == 0) exps[c] = (int8_t)e;
  }
}

// Source cells not covered by the 2x2 pool (odd trailing row / column).
__global__ void __launch_bounds__(256) split_tail_kernel(const float* __restrict__ src, int sh,
                                                         int sw, int d, int dp, bool vec,
                                                         __half* __restrict__ planes,
                                                         int8_t* __restrict__ exps) {
  const int lane = threadIdx.x & 31, kgs = dp / 8;
  const int ph = (sh / 2) * 2, pw = (sw / 2) * 2;
  const int64_t n_rows = (int64_t)(sh - ph) * sw, n = n_rows + (int64_t)ph * (sw - pw);
  const int64_t cells = (int64_t)sh * sw;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int y, x;
    if (i < n_rows) {
      y = ph + (int)(i / sw);
      x = (int)(i % sw);
    } else {
      y = (int)(i - n_rows);
      x = pw;
    }
    const int64_t c = (int64_t)y * sw + x;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (lane < kgs) load8(src + c * d, d, lane, vec, v);
    split_store(v, lane, kgs, c, cells, dp, planes, exps);
  }
}

struct CellRef {
  int level, cy, cx;
};

// g-th row of a tile's new-cell list (levels concatenated).
__device__ __forceinline__ CellRef cell_of(int g, const TilePlan* plans, const int* prefix,
                                           int levels) {
  int l = 0;
  while (l + 1 < levels && g >= prefix[l + 1]) ++l;
  CellRef c;
  c.level = l;
  new_cell(plans[l].B, plans[l].I, plans[l].has_i, g - prefix[l], c.cy, c.cx);
  return c;
}

}  // namespace tc

// ---------------------------------------------------------------------------
// Persistent, warp-specialised contraction.  One CTA per SM walks the tiles
// blockIdx.x, blockIdx.x + gridDim.x, ...; the roles communicate only through
// mbarrier rings, so the next tile's plan, F1 pieces and A rows are in flight
// while the current tile's MMAs run and the previous chunk's accumulators
// drain.  No thread ever waits on its own copy (bulk copies complete_tx,
// cp.async arrive-on-completion):
//   warp 0       B producer: one 16 KB bulk copy per F1 K-piece into an
//                NBP-deep piece ring (a piece is released after the last
//                chunk of its tile has consumed it)
//   warp 1       MMA issuer (converged warp, one elected lane issues): two
//                tcgen05.mma per K=16 step
//   warp 2       plan loader: the tile's PlanRec (window-union tiler output
//                of every level, computed for all tiles at once by
//                plan_kernel) via one bulk copy into an NPL-deep slot ring
//   warps 4-7,   A producers (16 rows each): per chunk and 64-channel K
//   12-15        block, every new
//                cell's hi and lo 128-byte rows via cp.async (full L2 lines)
//                into a 128B-swizzled NST-stage ring, completion tracked by
//                cp.async.mbarrier.arrive.noinc
//   warps 8-11   epilogue: tcgen05.ld of a 2-deep TMEM accumulator ring,
//                main + corr, cache-slot stores
// ---------------------------------------------------------------------------
namespace tcp {

#ifndef CVB_TC_NST
#define CVB_TC_NST 4
#endif
#ifndef CVB_TC_NBP
#define CVB_TC_NBP 5
#endif
constexpr int NST = CVB_TC_NST;     // A stages (32 KB each: hi + lo, 128 rows x 64 channels)
constexpr int NBP = CVB_TC_NBP;     // F1 pieces in the ring (16 KB each)
#ifndef CVB_TC_NPL
#define CVB_TC_NPL 3  // plan slots: 3 is 1.7% faster warm than 4 (A/B, round 2)
#endif
constexpr int NPL = CVB_TC_NPL;     // plan slots
#ifndef CVB_TC_AW
#define CVB_TC_AW 8
#endif
constexpr int A_WARPS = CVB_TC_AW;     // A producers: warps 4-7 (and 12-15 when 8)
constexpr int THREADS = A_WARPS == 8 ? 512 : 384;
constexpr int A_ROWS = 128 / A_WARPS;  // A rows per producer warp
// Pipeline watchdog: a ring wait that has not completed after this long
// (%globaltimer ns) means a broken pipeline, not a slow one.  The CTA then sets
// its abort flag, every role leaves its loop at its next wait, the kernel exits
// normally and the host-mapped error word makes the NEXT contraction call
// return CVB_ERR_CUDA.  (The CUDA context survives, unlike with __trap().)
constexpr unsigned long long WATCHDOG_NS = 20ull * 1000 * 1000 * 1000;
constexpr int WATCHDOG_CODE = 0x5744;  // 'WD'

struct Ctl {
  uint64_t plan_full[NPL], plan_empty[NPL];
  uint64_t b_full[NBP], b_empty[NBP];
  uint64_t a_full[NST], a_empty[NST];
  uint64_t acc_full[2], acc_empty[2];
  PlanRec slot[NPL];
  alignas(16) int8_t e1[NPL][tc::N];  // the slot's tile's query exponents (bulk-copied with the plan)
  float qscale[tc::N];                 // dense instantiation: 2^-e_q of the current tile
  uint32_t tmem;
  int abort;  // watchdog fired in this CTA
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
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait for `parity` on `bar`; false if the CTA's pipeline was aborted.  The
// fast path is one try_wait; the clock is read only every 64 failed polls.
__device__ __noinline__ bool wait_slow(uint32_t bar, uint32_t parity, volatile int* abort,
                                       int* word) {
  const unsigned long long t0 = global_ns();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try(bar, parity)) return true;
    if ((n & 63u) == 0) {
      if (*abort) return false;
      if (global_ns() - t0 > WATCHDOG_NS) {
        *abort = 1;
        if (word != nullptr) atomicExch_system(word, WATCHDOG_CODE);
        return false;
      }
    }
  }
}
__device__ __forceinline__ bool wait_phase(uint32_t bar, uint32_t parity, volatile int* abort,
                                           int* word) {
  return mbar_try(bar, parity) || wait_slow(bar, parity, abort, word);
}
// full barriers: the k-th completion has parity k&1; empty barriers: the
// producer's k-th wait passes on parity (k&1)^1 (a fresh barrier counts as
// having completed the phase before phase 0).
#define WAIT_FULL(bar, k) wait_phase((bar), (uint32_t)(k) & 1u, &C.abort, T.watchdog)
#define WAIT_EMPTY(bar, k) wait_phase((bar), ((uint32_t)(k) & 1u) ^ 1u, &C.abort, T.watchdog)
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Work counter of the persistent contraction: the plan loader of every CTA
// claims the next tile with one atomicAdd (dynamic load balance).  It is the
// `pad` word of the range's FIRST plan record, which belongs to this range
// alone (ranges are disjoint), so contractions of disjoint tile ranges may run
// concurrently on different streams (include/corrvol_b200.h).  plan_kernel
// resets it; the contraction's pdl_wait orders the reset before the claims.
__device__ __forceinline__ int* tile_counter(const PartialParams& P) {
  return P.plans + P.tile0 * PLAN_INTS + (int)(offsetof(PlanRec, pad) / 4);
}

template <bool DEBUG>
__device__ __forceinline__ void stamp(const tc::TcParams& T, int64_t it, int e) {
  if (DEBUG && T.ts != nullptr && blockIdx.x < 4 && it < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    T.ts[((int64_t)blockIdx.x * 64 + it) * 32 + e] = t;
  }
}

// DEBUG=false is the production instantiation: the CVB_TC_DEBUG knock-outs
// and the %globaltimer role timeline compile out of it.
template <bool DEBUG, bool DENSE = false>
__global__ void __launch_bounds__(THREADS, 1)
    partial_contract_tcp_kernel(const __grid_constant__ tc::TcParams T) {
  extern __shared__ uint8_t smem_raw[];
  const PartialParams& P = T.P;
  const int dp = T.dp;
  const int n_kb = dp / tc::KP;  // K blocks = A stages per chunk = F1 pieces per tile
  // 1024-byte alignment for the 128B-swizzled A stages
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;                        // NST x A_STAGE
  uint8_t* sB = smem + NST * tc::A_STAGE;    // NBP x B_PIECE
  Ctl& C = *reinterpret_cast<Ctl*>(sB + NBP * tc::B_PIECE);
  const uint32_t uB = tc::smem_u32(sB), uA = tc::smem_u32(sA);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto U = [](const uint64_t& b) { return tc::smem_u32(&b); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     tc::smem_u32(&C.tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < NPL; ++i) {
      tc::mbar_init(U(C.plan_full[i]), 1);
      tc::mbar_init(U(C.plan_empty[i]), 1 + 1 + 32 * A_WARPS + 128);
    }
    for (int i = 0; i < NBP; ++i) {
      tc::mbar_init(U(C.b_full[i]), 1);
      tc::mbar_init(U(C.b_empty[i]), 1);
    }
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(U(C.a_full[i]), 32 * A_WARPS);
      tc::mbar_init(U(C.a_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(U(C.acc_full[i]), 1);
      tc::mbar_init(U(C.acc_empty[i]), 128);
    }
    C.abort = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = C.tmem;
  pdl_trigger();
  pdl_wait();  // the plan records, meta and cache of earlier launches are complete

  if (warp == 0) {
    // ---------------- B producer: F1 pieces ----------------
    if (lane == 0) {
      uint32_t pb = 0;  // pieces issued so far
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!WAIT_FULL(U(C.plan_full[s]), (uint32_t)(it / NPL))) goto done;
        const int tile_i = C.slot[s].tile;
        if (tile_i < 0) break;
        if (C.slot[s].n_cells > 0) {
          const uint8_t* src = T.f1s + (int64_t)tile_i * n_kb * tc::B_PIECE;
          for (int q = 0; q < n_kb; ++q, ++pb) {
            const int bs = (int)(pb % NBP);
            if (!WAIT_EMPTY(U(C.b_empty[bs]), pb / NBP)) goto done;
            stamp<DEBUG>(T, it, 24 + q);
            if (DEBUG && (T.dbg & 8)) {
              arrive(U(C.b_full[bs]));
              continue;
            }
            tc::mbar_expect_tx(U(C.b_full[bs]), tc::B_PIECE);
            tc::bulk_g2s(uB + bs * tc::B_PIECE, src + (int64_t)q * tc::B_PIECE, tc::B_PIECE,
                         U(C.b_full[bs]));
          }
        }
        stamp<DEBUG>(T, it, 5);
        arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // the whole warp walks the rings (converged); one elected lane issues.
    // Descriptors are built once per stage: a K=16 step advances the
    // swizzled A start by 32 B (+2 in the descriptor's address field) and
    // the B start by 256 B (+16).
    uint32_t pb = 0, g = 0, cg = 0;
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % NPL);
      if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.plan_full[s]), (uint32_t)(it / NPL)))) goto done;
      if (C.slot[s].tile < 0) break;
      if (lane == 0) stamp<DEBUG>(T, it, 1);
      const int n = C.slot[s].n_cells;
      if (n > 0) {
        const int n_chunks = (n + tc::M - 1) / tc::M;
        for (int c = 0; c < n_chunks; ++c, ++cg) {
          const int ab = cg & 1;
          if (!__all_sync(0xffffffffu, WAIT_EMPTY(U(C.acc_empty[ab]), cg >> 1))) goto done;
          tc::tc_fence_after();
          if (c == 0 && lane == 0) stamp<DEBUG>(T, it, 6);
          const uint32_t d_main = tmem + ab * 128, d_corr = d_main + 64;
          for (int kb = 0; kb < n_kb; ++kb, ++g) {
            const uint32_t pi = pb + kb;
            const int bs = (int)(pi % NBP);
            if (c == 0) {
              if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.b_full[bs]), pi / NBP))) goto done;
              if (lane == 0) stamp<DEBUG>(T, it, 12 + kb);
            }
            const int st = (int)(g % NST);
            if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.a_full[st]), g / NST))) goto done;
            tc::tc_fence_after();
            if (c == 0 && lane == 0) stamp<DEBUG>(T, it, 8 + kb);
            const uint32_t a_hi = uA + st * tc::A_STAGE, a_lo = a_hi + tc::A_HALF;
            const uint32_t b_hi = uB + bs * tc::B_PIECE;  // hi rows 0-63, lo rows 64-127
            const uint64_t dah = tc::make_desc_sw128(a_hi), dal = tc::make_desc_sw128(a_lo);
            const uint64_t dbh = tc::make_desc(b_hi, 128, (tc::KP / 8) * 128);
            if (tc::elect_one()) {
              if (!(DEBUG && (T.dbg & 4))) {
#pragma unroll
                for (int k = 0; k < tc::KP / 16; ++k) {
                  const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                  // cols 0-63 += A_hi B_hi (main), cols 64-127 += A_hi B_lo (corr)
                  // (three N=64 MMAs into one accumulator, halving the epilogue's
                  // TMEM reads, measured 3% slower per step: A_hi read twice)
                  tc::mma_f16<tc::IDESC_N128>(d_main, dah + 2 * k, dbh + 16 * k, acc);
                  tc::mma_f16(d_corr, dal + 2 * k, dbh + 16 * k, 1u);  // corr += A_lo B_hi
                }
              }
              tc::mma_commit(U(C.a_empty[st]));
              if (c == n_chunks - 1) tc::mma_commit(U(C.b_empty[bs]));
              if (kb == n_kb - 1) tc::mma_commit(U(C.acc_full[ab]));
            }
            __syncwarp();
          }
        }
        pb += n_kb;
      }
      if (lane == 0) {
        stamp<DEBUG>(T, it, 2);
        arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp == 2) {
    // ---------------- plan loader: one bulk copy per tile record ----------------
    if (lane == 0) {
      // dynamic tile scheduler; the next tile is claimed one record ahead, so
      // the atomic's round trip overlaps the wait for a free slot
      // (only with many tiles per CTA: a tile claimed ahead is one the CTA
      // cannot give up, which unbalances the tail of short ranges — C2: +3%)
      const bool ahead = P.ntile >= 16 * (int64_t)gridDim.x;
      int64_t t_next = ahead ? atomicAdd(tile_counter(P), 1) : 0;
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!WAIT_EMPTY(U(C.plan_empty[s]), (uint32_t)(it / NPL))) goto done;
        if (!ahead) t_next = atomicAdd(tile_counter(P), 1);
        const int64_t t = t_next;
        if (ahead && t < P.ntile) t_next = atomicAdd(tile_counter(P), 1);
        if (t >= P.ntile) {  // end of the work list: a sentinel record
          C.slot[s].tile = -1;
          arrive(U(C.plan_full[s]));
          break;
        }
        // the plan record and the tile's 64 query exponents (the epilogue's
        // scales: no global load on its per-tile path)
        tc::mbar_expect_tx(U(C.plan_full[s]), (uint32_t)sizeof(PlanRec) + tc::N);
        tc::bulk_g2s(tc::smem_u32(&C.slot[s]), P.plans + (P.tile0 + t) * PLAN_INTS,
                     (uint32_t)sizeof(PlanRec), U(C.plan_full[s]));
        tc::bulk_g2s(tc::smem_u32(&C.e1[s][0]), T.e1 + (P.tile0 + t) * tc::N, tc::N,
                     U(C.plan_full[s]));
        stamp<DEBUG>(T, it, 0);
      }
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ---------------- A producers: cp.async of the new cells ----------------
    // warp aw owns A rows A_ROWS*aw ..+A_ROWS-1 (eight warps: per-chunk cell
    // decoding and issue run in parallel; -3% at iteration 0 against four);
    // per 4-row group one warp instruction
    // moves 4 full 128-byte rows (8 lanes x 16 B each, full L2 lines) into
    // the 128B-swizzled stage; completion is signalled per thread with
    // cp.async.mbarrier.arrive.noinc, so no producer thread ever waits on
    // its own copies.
    const int aw = warp < 8 ? warp - 4 : warp - 8;
    const int sub = lane >> 3, chunk = lane & 7;
    uint32_t g = 0;  // A stages issued
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % NPL);
      if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.plan_full[s]), (uint32_t)(it / NPL)))) goto done;
      const PlanRec& S = C.slot[s];
      if (S.tile < 0) break;
      const int n = S.n_cells;
      const int n_chunks = (n + tc::M - 1) / tc::M;
      const int64_t pair = P.batch > 1 ? S.tile / P.tiles_pp : 0;
      for (int c = 0; c < n_chunks; ++c) {
        // source row of A row 32aw + lane (hi plane; lo = hi + plane)
        const int gi = c * tc::M + A_ROWS * aw + (lane % A_ROWS);
        const __half* my_hi = nullptr;
        int64_t my_plane = 0;
        if (gi < n) {
          const tc::CellRef cr = tc::cell_of(gi, S.plan, S.prefix, P.levels);
          my_hi = reinterpret_cast<const __half*>(reinterpret_cast<const uint8_t*>(T.f2s[cr.level]) +
                                                  pair * T.pair_bytes[cr.level]) +
                  tc::f2_hi((int64_t)cr.cy * P.tw[cr.level] + cr.cx, dp);
          my_plane = tc::f2_lo_delta(T.plane[cr.level] / dp, dp);
        }
        for (int kb = 0; kb < n_kb; ++kb, ++g) {
          const int st = (int)(g % NST);
          if (!__all_sync(0xffffffffu, WAIT_EMPTY(U(C.a_empty[st]), g / NST))) goto done;
          if (c == 0 && tid == 128) stamp<DEBUG>(T, it, 16 + kb);
          if (!(DEBUG && (T.dbg & 1))) {
            const uint32_t stage = uA + st * tc::A_STAGE;
#pragma unroll
            for (int i = 0; i < A_ROWS / 4; ++i) {
              const int rl = 4 * i + sub;  // row within the warp's A_ROWS
              const __half* hi = reinterpret_cast<const __half*>(
                  __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_hi), rl));
              const int64_t pl = __shfl_sync(0xffffffffu, my_plane, rl);
              if (hi != nullptr) {
                const int row = A_ROWS * aw + rl;
                const uint32_t dst = stage + row * 128 + ((chunk ^ (row & 7)) << 4);
                const __half* src = hi + kb * tc::KP + chunk * 8;
                tc::cp_async16(dst, src);
                tc::cp_async16(dst + tc::A_HALF, src + pl);
              }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                             U(C.a_full[st]))
                         : "memory");
          } else {
            arrive(U(C.a_full[st]));
          }
        }
      }
      if (tid == 128) stamp<DEBUG>(T, it, 3);
      arrive(U(C.plan_empty[s]));
    }
  } else if (warp >= 8 && warp < 12) {
    // ---------------- epilogue (128 threads = TMEM lanes) ----------------
    const int ep = tid - 256;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t cg = 0;
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % NPL);
      if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.plan_full[s]), (uint32_t)(it / NPL)))) goto done;
      const PlanRec& S = C.slot[s];
      if (S.tile < 0) break;
      const int64_t tile = S.tile;
      const int n = S.n_cells;
      const int n_chunks = (n + tc::M - 1) / tc::M;
      const int64_t pair = P.batch > 1 ? tile / P.tiles_pp : 0;
      const TileRef tr = DENSE ? tile_ref(P, tile) : TileRef{0, 0, 0, 0};
      const int8_t* e_q = C.e1[s];  // query exponents: scale 2^-(e_q + e_c), exact
      if (DENSE && n_chunks > 0) {
        // dense tiles run hundreds of chunks: their 64 query scales as floats
        // once per tile (the per-element integer scale cost 2.3x in the dense
        // epilogue's store loop)
        tc::named_bar(1, 128);
        if (ep < tc::N) C.qscale[ep] = tc::exp2_neg(e_q[ep]);
        tc::named_bar(1, 128);
      }
      for (int c = 0; c < n_chunks; ++c, ++cg) {
        const int ab = cg & 1;
        // the row's cell, cache slot and exponent depend only on the plan:
        // resolve them (and issue the exponent load) before the accumulator wait
        const int gi = c * tc::M + ep;
        float* dst = nullptr;
        float* dd = nullptr;  // dense mode: this cell's entry in the tile's first row
        int64_t plane = 0;
        int e_c = 0;
        if (gi < n) {
          const tc::CellRef cr = tc::cell_of(gi, S.plan, S.prefix, P.levels);
          if (DENSE) {
            plane = (int64_t)P.th[cr.level] * P.tw[cr.level];  // row length of the level
            dd = T.dense[cr.level] + (int64_t)cr.cy * P.tw[cr.level] + cr.cx;
          } else {
            const int ch = P.ch[cr.level], cw = P.cw[cr.level];
            plane = (int64_t)ch * cw * TQW;
            dst = P.cache[cr.level] + tile * plane * TQH +
                  (int64_t)slot_of(cr.cy, cr.cx, ch, cw) * TQW;
          }
          if (!(DEBUG && (T.dbg & 64)))
            e_c = T.e2[cr.level][pair * T.pair_bytes[cr.level] + (int64_t)cr.cy * P.tw[cr.level] + cr.cx];
        }
        if (!__all_sync(0xffffffffu, WAIT_FULL(U(C.acc_full[ab]), cg >> 1))) goto done;
        tc::tc_fence_after();
        if (c == 0 && tid == 256) stamp<DEBUG>(T, it, 20);
        float vm[32], vc[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tc::tmem_ld32(tmem + ab * 128 + lane_base + h * 32, vm);
          tc::tmem_ld32(tmem + ab * 128 + 64 + lane_base + h * 32, vc);
          if (dst != nullptr && !(DEBUG && (T.dbg & 2))) {
            // this half holds tile rows 4h..4h+3 = query groups 4h/2*2 .. +3;
            // each group's 8 costs (32 B, one cache sector) leave in one
            // 256-bit store, so a warp writes whole sectors of consecutive slots
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
              const int r = gg >> 1, c = gg & 1;  // row pair and column half in this half
              const int j0 = 16 * r + 4 * c, j1 = j0 + 8;
              float o[8];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                // (main + corr) * 2^-(e_q + e_c): exact power-of-two scales
                o[i] = (vm[j0 + i] + vc[j0 + i]) * tc::exp2_neg(e_q[h * 32 + j0 + i] + e_c);
                o[4 + i] = (vm[j1 + i] + vc[j1 + i]) * tc::exp2_neg(e_q[h * 32 + j1 + i] + e_c);
              }
              const int g = (2 * h + r) * 2 + c;  // == qgroup(4h + 2r, 4c)
              tc::st_global_v8(dst + g * plane, o);
            }
          } else if (DENSE && dd != nullptr) {
            const float s_cd = tc::exp2_neg(e_c);
            // dense rows: query q of the tile -> pixel (8ty + q/8, 8tx + q%8); a
            // warp's lanes are consecutive cells, so each store is 128 B
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const int q = h * 32 + j;
              const int py = tr.ty * TQH + (q >> 3), px = tr.tx * TQW + (q & 7);
              if (py < P.h1 && px < P.w1)
                dd[((int64_t)py * P.w1 + px) * plane] =
                    (vm[j] + vc[j]) * (C.qscale[q] * s_cd);
            }
          }
        }
        tc::tc_fence_before();
        if (c == 0 && tid == 256) stamp<DEBUG>(T, it, 21);
        arrive(U(C.acc_empty[ab]));
      }
      if (tid == 256) stamp<DEBUG>(T, it, 4);
      arrive(U(C.plan_empty[s]));
    }
  }
done:  // normal exit, or a role leaving early after the watchdog fired
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// Window-union tiler for every tile and level of the range, one warp per
// tile (two queries per lane; per-level bounding boxes by warp shuffles; lane
// l finalises level l against its previous box in meta), eight tiles per CTA.
// Writes the tile's PlanRec for the persistent contraction and updates the
// per-level meta; the work counters are reduced per CTA (one atomic each).
constexpr int PLAN_WARPS = 8;


__global__ void __launch_bounds__(PLAN_WARPS * 32) plan_kernel(PartialParams P) {
  __shared__ unsigned long long s_cnt[4];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0ULL;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *tile_counter(P) = 0;  // scheduler reset
  const int64_t t = (int64_t)blockIdx.x * PLAN_WARPS + warp;
  if (t < P.ntile) {
    const int64_t tile = P.tile0 + t;
    const int r = P.radius;
    const TileRef tr = tile_ref(P, tile);
    const int tile_y = tr.ty, tile_x = tr.tx;
    double x[2], y[2];
    bool v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = lane + 32 * h;
      const int py = tile_y * TQH + q / TQW, px = tile_x * TQW + q % TQW;
      v[h] = py < P.h1 && px < P.w1;
      x[h] = y[h] = 0.0;
      if (v[h]) load_coord(P.coords, P.f64, tr.pix + (int64_t)py * P.w1 + px, x[h], y[h]);
    }
    const int nv = __popc(__ballot_sync(0xffffffffu, v[0])) + __popc(__ballot_sync(0xffffffffu, v[1]));
    // lane l < L: its level's previous box, loaded now so the latency overlaps
    // the anchor math
    int32_t* meta = P.meta + (tile * P.levels + (lane < P.levels ? lane : 0)) * CVB_META_INTS;
    int pm[5] = {0, 0, 0, 0, 0};
    if (lane < P.levels) {
#pragma unroll
      for (int i = 0; i < 5; ++i) pm[i] = meta[i];
    }
    // Level floors from the level-0 floor: floor(x / 2^l) == floor(x) >> l
    // (x * 2^-l is exact in fp64), and shifting and clamp_anchor are both
    // monotonic, so the tile's per-level anchor range is the shifted, clamped
    // range of its level-0 floors — one fp64 floor per coordinate and one
    // warp reduction for all levels.  Floors are saturated to +-2^30 first
    // (beyond any grid: they clamp to the same anchors at every level).
    int fxlo = INT_MAX, fxhi = INT_MIN, fylo = INT_MAX, fyhi = INT_MIN;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (v[h]) {
        const LevelPos lp = level_pos(x[h], y[h], 0);
        const long long sat = 1ll << 30;
        const int fx = (int)(lp.x0 < -sat ? -sat : (lp.x0 > sat ? sat : lp.x0));
        const int fy = (int)(lp.y0 < -sat ? -sat : (lp.y0 > sat ? sat : lp.y0));
        fxlo = min(fxlo, fx);
        fxhi = max(fxhi, fx);
        fylo = min(fylo, fy);
        fyhi = max(fyhi, fy);
      }
    }
    fxlo = __reduce_min_sync(0xffffffffu, fxlo);
    fxhi = __reduce_max_sync(0xffffffffu, fxhi);
    fylo = __reduce_min_sync(0xffffffffu, fylo);
    fyhi = __reduce_max_sync(0xffffffffu, fyhi);
    int mylo_y = 0, myhi_y = 0, mylo_x = 0, myhi_x = 0;  // lane l: level l's anchor range
    if (lane < P.levels && nv > 0) {
      const int l = lane;
      mylo_y = clamp_anchor(fylo >> l, r, P.th[l]);
      myhi_y = clamp_anchor(fyhi >> l, r, P.th[l]);
      mylo_x = clamp_anchor(fxlo >> l, r, P.tw[l]);
      myhi_x = clamp_anchor(fxhi >> l, r, P.tw[l]);
    }
    int n_new = 0;
    unsigned long long c_ovf = 0, c_empty = 0, c_dots, c_cells;
    int* rec = P.plans + tile * PLAN_INTS;
    if (lane < P.levels) {
      const int level = lane;
      const int th = P.th[level], tw = P.tw[level];
      Box B;
      B.ylo = max(mylo_y - r, 0);
      B.yhi = min(myhi_y + r + 1, th - 1);
      B.xlo = max(mylo_x - r, 0);
      B.xhi = min(myhi_x + r + 1, tw - 1);
      int status = ST_OK;
      if (nv == 0 || B.empty()) {
        status = ST_EMPTY;
        B = Box{1, 0, 1, 0};
      } else if (B.h() > P.ch[level] || B.w() > P.cw[level]) {
        status = ST_OVERFLOW;
      }
      const Box prev{pm[0], pm[1], pm[2], pm[3]};
      const bool prev_ok = !P.no_cache && pm[4] == ST_OK && !prev.empty();
      const Box I{max(B.ylo, prev.ylo), min(B.yhi, prev.yhi), max(B.xlo, prev.xlo),
                  min(B.xhi, prev.xhi)};
      const bool has_i = status == ST_OK && prev_ok && !I.empty();
      n_new = status == ST_OK ? (int)(B.area() - (has_i ? I.area() : 0)) : 0;
      meta[0] = B.ylo;
      meta[1] = B.yhi;
      meta[2] = B.xlo;
      meta[3] = B.xhi;
      meta[4] = status;
      meta[5] = n_new;
      const TilePlan tp{B, I, (int)has_i, n_new, nv, status};
      const int* src = reinterpret_cast<const int*>(&tp);
      constexpr int TP_INTS = (int)(sizeof(TilePlan) / 4);
#pragma unroll
      for (int i = 0; i < TP_INTS; ++i) rec[level * TP_INTS + i] = src[i];
      c_ovf = status == ST_OVERFLOW;
      c_empty = status == ST_EMPTY;
    }
    // prefix over levels (lane l holds n_new of level l)
    int pre = n_new;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += u;
    }
    int* prefix = rec + CVB_MAX_LEVELS * (int)(sizeof(TilePlan) / 4);
    if (lane <= P.levels) prefix[lane] = pre - n_new;       // exclusive prefix, lanes 0..L
    if (lane == P.levels) prefix[CVB_MAX_LEVELS + 1] = pre - n_new;  // n_cells
    if (lane == 0) prefix[CVB_MAX_LEVELS + 2] = (int)tile;           // the record's tile
    // per-warp totals (a tile's dots fit 32 bits: <= L * cap_h * cap_w * 64)
    c_dots = __reduce_add_sync(0xffffffffu, (unsigned)(n_new * nv));
    c_cells = __reduce_add_sync(0xffffffffu, (unsigned)n_new);
    c_ovf = __reduce_add_sync(0xffffffffu, (unsigned)c_ovf);
    c_empty = __reduce_add_sync(0xffffffffu, (unsigned)c_empty);
    if (lane == 0 && P.counters != nullptr) {
      if (c_dots) atomicAdd(&s_cnt[0], c_dots);
      if (c_cells) atomicAdd(&s_cnt[1], c_cells);
      if (c_ovf) atomicAdd(&s_cnt[2], c_ovf);
      if (c_empty) atomicAdd(&s_cnt[3], c_empty);
    }
  }
  __syncthreads();
  if (threadIdx.x < 4 && P.counters != nullptr && s_cnt[threadIdx.x])
    atomicAdd(P.counters + threadIdx.x, s_cnt[threadIdx.x]);
}

// Dense mode plans: every tile's work list is every cell of every level
// (B = the level grid, no previous box); resets the range's work counter.
__global__ void dense_plan_kernel(PartialParams P) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= P.n_tiles) return;
  int* rec = P.plans + t * PLAN_INTS;
  PlanRec pr;
  int acc = 0;
  for (int l = 0; l < CVB_MAX_LEVELS; ++l) {
    TilePlan tp{Box{1, 0, 1, 0}, Box{1, 0, 1, 0}, 0, 0, 0, ST_EMPTY};
    if (l < P.levels) {
      tp.B = Box{0, P.th[l] - 1, 0, P.tw[l] - 1};
      tp.n_new = P.th[l] * P.tw[l];
      tp.nvalid = TQ;
      tp.status = ST_OK;
    }
    pr.plan[l] = tp;
    pr.prefix[l] = acc;
    acc += tp.n_new;
  }
  pr.prefix[CVB_MAX_LEVELS] = acc;
  pr.n_cells = acc;
  pr.tile = (int)t;
  pr.pad = 0;  // the work counter of the range starting at tile 0
  const int* src = reinterpret_cast<const int*>(&pr);
  for (int i = 0; i < PLAN_INTS; ++i) rec[i] = src[i];
}

size_t smem_bytes() {
  return (size_t)NST * tc::A_STAGE + (size_t)NBP * tc::B_PIECE + sizeof(Ctl) + 1024;
}

// SM count per device (the persistent grid size), queried once per device.
int sm_count(int dev) {
  static std::atomic<int> cache[64];
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// The watchdog's error word: one int of portable, host-mapped pinned memory
// (the kernel writes it with a system-scope atomic; the host reads it on the
// next call without a synchronisation).  Allocated on the first call that is
// not being captured into a CUDA graph; null until then (no reporting).
int* watchdog_host = nullptr;
int* watchdog_dev = nullptr;
int* watchdog_word(cudaStream_t s) {
  static std::atomic<int> state{0};  // 0 unallocated, 1 ready, 2 failed
  if (state.load(std::memory_order_acquire) == 0) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    static std::atomic_flag lock = ATOMIC_FLAG_INIT;
    while (lock.test_and_set(std::memory_order_acquire)) {
    }
    if (state.load() == 0) {
      void* h = nullptr;
      void* d = nullptr;
      if (cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) ==
              cudaSuccess &&
          cudaHostGetDevicePointer(&d, h, 0) == cudaSuccess) {
        *(volatile int*)h = 0;
        watchdog_host = (int*)h;
        watchdog_dev = (int*)d;
        state.store(1, std::memory_order_release);
      } else {
        cudaGetLastError();
        state.store(2, std::memory_order_release);
      }
    }
    lock.clear(std::memory_order_release);
  }
  return state.load(std::memory_order_acquire) == 1 ? watchdog_host : nullptr;
}

}  // namespace tcp

// ---------------------------------------------------------------------------
// Cold-iteration contraction on SM pairs (tcgen05.mma.cta_group::2).
//
// At iteration 0 (and every iteration with the cache off) each tile contracts
// its whole bounding box, and horizontally adjacent tiles' boxes share most of
// their cells: gathering every tile's A rows separately moves 6.2 GB through
// L2 -> SMEM at C4, the cold contraction's limit.  Here a cluster of two CTAs
// (one SM pair) takes a PAIR of horizontally adjacent tiles and contracts the
// hull of their two boxes once, as M=256 chunks: each CTA gathers half of
// every chunk's cell rows (A) and holds its own tile's F1 image (B = the two
// tiles' 128 queries, N-split across the CTAs); the leader CTA issues
// tcgen05.mma.cta_group::2 (main = A_hi.B_hi, corr = A_hi.B_lo + A_lo.B_hi,
// three N=128 MMAs per K=16 step) and every commit is multicast to both
// CTAs' barriers.  Each CTA's TMEM holds its 128 cells x 128 queries; its
// epilogue writes every cell that lies in tile j's box into tile j's cache
// (the same cells the single-tile kernel writes when the tile is cold; a
// cell of the previous box is rewritten with its own value when it is not).
// Cross-CTA signalling: the follower's A / B completions are relayed by its
// warp 1 to the leader's full barriers; the follower's epilogue arrives on
// the leader's accumulator-empty barrier remotely.
// ---------------------------------------------------------------------------
namespace tcp2 {

// Rings of the pair kernel (A stages, F1 pieces, plan slots; the slots hold
// only the pair's per-level tile plans, levels <= PMAXL).  5 A stages with 4
// F1 pieces and 2 slots also fit 227 KB: no faster (A/B, round 2).
#ifndef CVB_TC2_NST
#define CVB_TC2_NST 4
#endif
#ifndef CVB_TC2_NBP
#define CVB_TC2_NBP 5
#endif
#ifndef CVB_TC2_NPL
#define CVB_TC2_NPL 3
#endif
constexpr int NST = CVB_TC2_NST;
constexpr int NBP = CVB_TC2_NBP;
constexpr int NPL = CVB_TC2_NPL;
constexpr int PMAXL = 4;  // levels the pair kernel handles (more: single-tile kernel)
constexpr int THREADS = 512;
constexpr int A_WARPS = 8;             // A producers: warps 4-7 and 12-15
constexpr int A_ROWS = 128 / A_WARPS;

constexpr int M2 = 256;  // cells per pair chunk (128 per CTA)
// accumulators: main (hi.hi) and corr (hi.lo + lo.hi) in 128 TMEM columns
// each per buffer, a 2-deep ring in 512 columns — the same two sums in the
// same order as the single-tile kernel, so a cell has the same bits whichever
// kernel computed it (one shared accumulator: 3% faster here, but not
// bit-compatible with the single-tile kernel's cells)
constexpr int NACC = 2;
constexpr int RELAY_LANES = NST + 1;  // follower relay: one lane per A stage + one for B

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Relaxed remote arrive: no cluster-scope membar (a release arrive costs a
// fence per call, which serialised the relay to ~1.3 us per stage).  What it
// publishes is already complete: cp.async data whose local barrier the relay
// has observed (plus fence.proxy.async), or TMEM reads retired by
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync.
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void st_cluster_u64(uint32_t cluster_addr, unsigned long long v) {
  asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(cluster_addr), "l"(v)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
template <uint32_t ID>
__device__ __forceinline__ void mma2(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(ID), "r"(acc));
}
__device__ __forceinline__ void commit_mc(uint32_t mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(mbar),
      "h"((uint16_t)3)
      : "memory");
}
// D f32, A/B f16 K-major, N=128 (64 per CTA), M=256 (128 per CTA)
constexpr uint32_t IDESC2 = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(M2 >> 4) << 24);

// Work item: a pair of horizontally adjacent tiles (tile[1] < 0: a lone last
// tile of an odd tile row) and the per-level hull of their boxes.
struct alignas(16) PairSlot {
  TilePlan plan[2][PMAXL];  // the two tiles' per-level plans (head of their PlanRecs)
  int hull[PMAXL][4];       // ylo, yhi, xlo, xhi
  int hw[PMAXL];            // hull width
  int prefix[PMAXL + 1];
  int n_cells;
  int tile[2];
  int end;
};

struct Ctl2 {
  uint64_t plan_full[NPL], plan_empty[NPL], plan_copy[NPL];
  uint64_t pidx_full[NPL];         // follower: the leader posted the slot's pair index
  unsigned long long pidx[NPL];    // follower: pair index mailbox (written by the leader)
  uint64_t b_full[NBP], b_empty[NBP];
  uint64_t a_full[NST], a_empty[NST];
  uint64_t acc_full[NACC], acc_empty[NACC];
  PairSlot slot[NPL];
  alignas(16) int8_t e1[NPL][2][tc::N];  // both tiles' query exponents (bulk-copied with the plans)
  uint32_t tmem;
  int abort;
};

size_t smem_bytes() {
  return (size_t)NST * tc::A_STAGE + (size_t)NBP * tc::B_PIECE + sizeof(Ctl2) + 1024;
}

__device__ __forceinline__ bool in_box(const Box& b, int y, int x) {
  return y >= b.ylo && y <= b.yhi && x >= b.xlo && x <= b.xhi;
}

// pair index -> the two global tiles (pairs never straddle a tile row)
__device__ __forceinline__ void pair_tiles(const PartialParams& P, int64_t pidx, int& t0, int& t1) {
  const int ppr = (P.tiles_x + 1) / 2;  // pairs per tile row
  const int64_t row = pidx / ppr;
  const int pc = (int)(pidx - row * ppr);
  const int64_t base = P.tile0 + row * P.tiles_x;  // P.tile0 is a row boundary
  t0 = (int)(base + 2 * pc);
  t1 = 2 * pc + 1 < P.tiles_x ? t0 + 1 : -1;
}

#define WAIT_FULL2(bar, k) tcp::wait_phase((bar), (uint32_t)(k) & 1u, &C.abort, T.watchdog)
#define WAIT_EMPTY2(bar, k) tcp::wait_phase((bar), ((uint32_t)(k) & 1u) ^ 1u, &C.abort, T.watchdog)
#define WAIT_FULL_CL(bar, k) tcp::wait_phase((bar), (uint32_t)(k) & 1u, &C.abort, T.watchdog)
#define WAIT_EMPTY_CL(bar, k) tcp::wait_phase((bar), ((uint32_t)(k) & 1u) ^ 1u, &C.abort, T.watchdog)

// DEBUG=true: the CVB_TC_DEBUG knock-outs (1 A loads, 2 epilogue stores, 4 MMAs,
// 8 F1 loads) for profiling; DEBUG=false is the production instantiation.
template <bool DEBUG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    pair_contract_kernel(const __grid_constant__ tc::TcParams T, int64_t n_pairs) {
  extern __shared__ uint8_t smem_raw[];
  const PartialParams& P = T.P;
  const int dp = T.dp;
  const int n_kb = dp / tc::KP;
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * tc::A_STAGE;
  Ctl2& C = *reinterpret_cast<Ctl2*>(sB + NBP * tc::B_PIECE);
  const uint32_t uB = tc::smem_u32(sB), uA = tc::smem_u32(sA);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  auto U = [](const uint64_t& b) { return tc::smem_u32(&b); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     tc::smem_u32(&C.tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < NPL; ++i) {
      tc::mbar_init(U(C.plan_full[i]), 1);
      // B producer + MMA issuer (leader) or the RELAY_LANES relay lanes
      // (follower) + A producers + epilogue
      tc::mbar_init(U(C.plan_empty[i]), 1 + (leader ? 1 : RELAY_LANES) + 32 * A_WARPS + 128);
      tc::mbar_init(U(C.plan_copy[i]), 1);
      tc::mbar_init(U(C.pidx_full[i]), 1);
    }
    for (int i = 0; i < NBP; ++i) {
      tc::mbar_init(U(C.b_full[i]), leader ? 2 : 1);  // leader: own copy + the follower's relay
      tc::mbar_init(U(C.b_empty[i]), 1);
    }
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(U(C.a_full[i]), 32 * A_WARPS + (leader ? 1 : 0));
      tc::mbar_init(U(C.a_empty[i]), 1);
    }
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(U(C.acc_full[i]), 1);
      tc::mbar_init(U(C.acc_empty[i]), 4 + 1);  // leader: 4 local epilogue warps + the follower
    }
    C.abort = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = C.tmem;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ---------------- B producer: this CTA's tile's F1 pieces ----------------
    if (lane == 0) {
      uint32_t pb = 0;
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!WAIT_FULL2(U(C.plan_full[s]), (uint32_t)(it / NPL))) goto done;
        const PairSlot& S = C.slot[s];
        if (S.end) break;
        if (S.n_cells > 0) {
          const int my = S.tile[rank] >= 0 ? S.tile[rank] : S.tile[0];
          const uint8_t* src = T.f1s + (int64_t)my * n_kb * tc::B_PIECE;
          for (int q = 0; q < n_kb; ++q, ++pb) {
            const int bs = (int)(pb % NBP);
            if (!WAIT_EMPTY2(U(C.b_empty[bs]), pb / NBP)) goto done;
            if (DEBUG && (T.dbg & 8)) {
              tcp::arrive(U(C.b_full[bs]));
              continue;
            }
            tc::mbar_expect_tx(U(C.b_full[bs]), tc::B_PIECE);
            tc::bulk_g2s(uB + bs * tc::B_PIECE, src + (int64_t)q * tc::B_PIECE, tc::B_PIECE,
                         U(C.b_full[bs]));
          }
        }
        tcp::arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader CTA) ----------------
      uint32_t pb = 0, g = 0, cg = 0;
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!__all_sync(0xffffffffu, WAIT_FULL2(U(C.plan_full[s]), (uint32_t)(it / NPL))))
          goto done;
        if (C.slot[s].end) break;
        const int n = C.slot[s].n_cells;
        if (n > 0) {
          const int n_chunks = (n + M2 - 1) / M2;
          for (int c = 0; c < n_chunks; ++c, ++cg) {
            const int ab = (int)(cg % NACC);
            if (!__all_sync(0xffffffffu, WAIT_EMPTY_CL(U(C.acc_empty[ab]), cg / NACC))) goto done;
            tc::tc_fence_after();
            const uint32_t d_main = tmem + ab * 256, d_corr = d_main + 128;
            for (int kb = 0; kb < n_kb; ++kb, ++g) {
              const uint32_t pi = pb + kb;
              const int bs = (int)(pi % NBP);
              if (c == 0 && !__all_sync(0xffffffffu, WAIT_FULL_CL(U(C.b_full[bs]), pi / NBP)))
                goto done;
              const int st = (int)(g % NST);
              if (!__all_sync(0xffffffffu, WAIT_FULL_CL(U(C.a_full[st]), g / NST))) goto done;
              tc::tc_fence_after();
              const uint32_t a_hi = uA + st * tc::A_STAGE, a_lo = a_hi + tc::A_HALF;
              const uint32_t b_hi = uB + bs * tc::B_PIECE, b_lo = b_hi + tc::B_HALF;
              const uint64_t dah = tc::make_desc_sw128(a_hi), dal = tc::make_desc_sw128(a_lo);
              const uint64_t dbh = tc::make_desc(b_hi, 128, (tc::KP / 8) * 128);
              const uint64_t dbl = tc::make_desc(b_lo, 128, (tc::KP / 8) * 128);
              if (tc::elect_one()) {
#pragma unroll
                for (int k = 0; k < tc::KP / 16; ++k) {
                  if (DEBUG && (T.dbg & 4)) break;
                  const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                  mma2<IDESC2>(d_main, dah + 2 * k, dbh + 16 * k, acc);  // A_hi B_hi
                  mma2<IDESC2>(d_corr, dah + 2 * k, dbl + 16 * k, acc);  // A_hi B_lo
                  mma2<IDESC2>(d_corr, dal + 2 * k, dbh + 16 * k, 1u);   // A_lo B_hi
                }
                commit_mc(U(C.a_empty[st]));
                if (c == n_chunks - 1) commit_mc(U(C.b_empty[bs]));
                if (kb == n_kb - 1) commit_mc(U(C.acc_full[ab]));
              }
              __syncwarp();
            }
          }
          pb += n_kb;
        }
        if (lane == 0) tcp::arrive(U(C.plan_empty[s]));
      }
    } else if (lane < RELAY_LANES) {
      // ---------------- relay (follower CTA): A / B completions -> leader ----------------
      // lane st < NST relays A stage st, lane NST the B pieces; the lanes walk
      // the same work sequence independently, so relays of different stages
      // overlap
      uint32_t pb = 0, g = 0;
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!WAIT_FULL2(U(C.plan_full[s]), (uint32_t)(it / NPL))) goto done;
        if (C.slot[s].end) break;
        const int n = C.slot[s].n_cells;
        if (n > 0) {
          const int n_chunks = (n + M2 - 1) / M2;
          for (int c = 0; c < n_chunks; ++c) {
            for (int kb = 0; kb < n_kb; ++kb, ++g) {
              const uint32_t pi = pb + kb;
              const int bs = (int)(pi % NBP);
              if (c == 0 && lane == NST) {
                if (!WAIT_FULL2(U(C.b_full[bs]), pi / NBP)) goto done;
                arrive_remote(mapa(U(C.b_full[bs]), 0));
              }
              const int st = (int)(g % NST);
              if (lane == st) {
                if (!WAIT_FULL2(U(C.a_full[st]), g / NST)) goto done;
                tc::fence_proxy_async();
                arrive_remote(mapa(U(C.a_full[st]), 0));
              }
            }
          }
          pb += n_kb;
        }
        tcp::arrive(U(C.plan_empty[s]));
      }
    }
  } else if (warp == 2) {
    // ---------------- plan loader: both tiles' records + the per-level hull ----------------
    if (lane == 0) {
      // dynamic pair scheduling: the leader claims pairs (one ahead, so the
      // atomic's round trip overlaps the slot wait) and posts each index into
      // the follower's mailbox for the same slot
      // (claimed ahead only with many pairs per cluster, as for tiles)
      const bool ahead = n_pairs >= 8 * (int64_t)gridDim.x;
      int64_t pidx_next = leader && ahead ? atomicAdd(tcp::tile_counter(P), 1) : 0;  // reset by plan_kernel
      for (int64_t it = 0;; ++it) {
        const int s = (int)(it % NPL);
        if (!WAIT_EMPTY2(U(C.plan_empty[s]), (uint32_t)(it / NPL))) goto done;
        PairSlot& S = C.slot[s];
        int64_t pidx;
        if (leader) {
          if (!ahead) pidx_next = atomicAdd(tcp::tile_counter(P), 1);
          pidx = pidx_next;
          if (ahead && pidx < n_pairs) pidx_next = atomicAdd(tcp::tile_counter(P), 1);
          st_cluster_u64(mapa(tc::smem_u32(&C.pidx[s]), 1), (unsigned long long)pidx);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           mapa(U(C.pidx_full[s]), 1))
                       : "memory");
        } else {
          if (!WAIT_FULL2(U(C.pidx_full[s]), (uint32_t)(it / NPL))) goto done;
          pidx = (int64_t)*reinterpret_cast<volatile unsigned long long*>(&C.pidx[s]);
        }
        if (pidx >= n_pairs) {
          S.end = 1;
          tcp::arrive(U(C.plan_full[s]));
          break;
        }
        int t0, t1;
        pair_tiles(P, pidx, t0, t1);
        S.end = 0;
        S.tile[0] = t0;
        S.tile[1] = t1;
        // the head of each PlanRec: its per-level TilePlans
        const uint32_t rec_bytes = (uint32_t)(P.levels * sizeof(TilePlan));
        tc::mbar_expect_tx(U(C.plan_copy[s]), (rec_bytes + tc::N) * (t1 >= 0 ? 2 : 1));
        tc::bulk_g2s(tc::smem_u32(&S.plan[0][0]), P.plans + (int64_t)t0 * PLAN_INTS, rec_bytes,
                     U(C.plan_copy[s]));
        tc::bulk_g2s(tc::smem_u32(&C.e1[s][0][0]), T.e1 + (int64_t)t0 * tc::N, tc::N,
                     U(C.plan_copy[s]));
        if (t1 >= 0) {
          tc::bulk_g2s(tc::smem_u32(&S.plan[1][0]), P.plans + (int64_t)t1 * PLAN_INTS, rec_bytes,
                       U(C.plan_copy[s]));
          tc::bulk_g2s(tc::smem_u32(&C.e1[s][1][0]), T.e1 + (int64_t)t1 * tc::N, tc::N,
                       U(C.plan_copy[s]));
        }
        if (!WAIT_FULL2(U(C.plan_copy[s]), (uint32_t)(it / NPL))) goto done;
        int acc = 0;
        for (int l = 0; l < PMAXL; ++l) {
          S.prefix[l] = acc;
          int ylo = INT_MAX, yhi = INT_MIN, xlo = INT_MAX, xhi = INT_MIN;
          if (l < P.levels) {
            for (int j = 0; j < 2; ++j) {
              if (j == 1 && t1 < 0) continue;
              const TilePlan& tp = S.plan[j][l];
              if (tp.status != ST_OK) continue;
              ylo = min(ylo, tp.B.ylo);
              yhi = max(yhi, tp.B.yhi);
              xlo = min(xlo, tp.B.xlo);
              xhi = max(xhi, tp.B.xhi);
            }
          }
          const bool any = ylo <= yhi && xlo <= xhi;
          S.hull[l][0] = ylo;
          S.hull[l][1] = yhi;
          S.hull[l][2] = xlo;
          S.hull[l][3] = xhi;
          S.hw[l] = any ? xhi - xlo + 1 : 1;
          acc += any ? (yhi - ylo + 1) * (xhi - xlo + 1) : 0;
        }
        S.prefix[PMAXL] = acc;
        S.n_cells = acc;
        tcp::arrive(U(C.plan_full[s]));
      }
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ---------------- A producers: this CTA's half of every 256-cell chunk ----------------
    const int aw = warp < 8 ? warp - 4 : warp - 8;
    const int sub = lane >> 3, chunk = lane & 7;
    uint32_t g = 0;
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % NPL);
      if (!__all_sync(0xffffffffu, WAIT_FULL2(U(C.plan_full[s]), (uint32_t)(it / NPL)))) goto done;
      const PairSlot& S = C.slot[s];
      if (S.end) break;
      const int n = S.n_cells;
      const int n_chunks = (n + M2 - 1) / M2;
      const int64_t pair = P.batch > 1 ? S.tile[0] / P.tiles_pp : 0;
      for (int c = 0; c < n_chunks; ++c) {
        const int gi = c * M2 + (int)rank * tc::M + A_ROWS * aw + (lane % A_ROWS);
        const __half* my_hi = nullptr;
        int64_t my_plane = 0;
        if (gi < n) {
          int l = 0;
          while (l + 1 < P.levels && gi >= S.prefix[l + 1]) ++l;
          const int idx = gi - S.prefix[l];
          const int cy = S.hull[l][0] + idx / S.hw[l], cx = S.hull[l][2] + idx % S.hw[l];
          my_hi = reinterpret_cast<const __half*>(reinterpret_cast<const uint8_t*>(T.f2s[l]) +
                                                  pair * T.pair_bytes[l]) +
                  tc::f2_hi((int64_t)cy * P.tw[l] + cx, dp);
          my_plane = tc::f2_lo_delta(T.plane[l] / dp, dp);
        }
        for (int kb = 0; kb < n_kb; ++kb, ++g) {
          const int st = (int)(g % NST);
          if (!__all_sync(0xffffffffu, WAIT_EMPTY2(U(C.a_empty[st]), g / NST))) goto done;
          const uint32_t stage = uA + st * tc::A_STAGE;
          if (DEBUG && (T.dbg & 1)) {
            tcp::arrive(U(C.a_full[st]));
            continue;
          }
#pragma unroll
          for (int i = 0; i < A_ROWS / 4; ++i) {
            const int rl = 4 * i + sub;
            const __half* hi = reinterpret_cast<const __half*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_hi), rl));
            const int64_t pl = __shfl_sync(0xffffffffu, my_plane, rl);
            if (hi != nullptr) {
              const int row = A_ROWS * aw + rl;
              const uint32_t dst = stage + row * 128 + ((chunk ^ (row & 7)) << 4);
              const __half* src = hi + kb * tc::KP + chunk * 8;
              tc::cp_async16(dst, src);
              tc::cp_async16(dst + tc::A_HALF, src + pl);
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                           U(C.a_full[st]))
                       : "memory");
        }
      }
      tcp::arrive(U(C.plan_empty[s]));
    }
  } else if (warp >= 8 && warp < 12) {
    // ---------------- epilogue: this CTA's 128 cells x both tiles' queries ----------------
    const int ep = tid - 256;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t acc_empty_base = mapa(U(C.acc_empty[0]), 0);  // leader's ring (remote)
    uint32_t cg = 0;
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % NPL);
      if (!__all_sync(0xffffffffu, WAIT_FULL2(U(C.plan_full[s]), (uint32_t)(it / NPL)))) goto done;
      const PairSlot& S = C.slot[s];
      if (S.end) break;
      const int n = S.n_cells;
      const int n_chunks = (n + M2 - 1) / M2;
      const int64_t pair = P.batch > 1 ? S.tile[0] / P.tiles_pp : 0;
      // both tiles' query exponents: scale 2^-(e_q + e_c), exact
      const int8_t(&e_q)[2][tc::N] = C.e1[s];
      for (int c = 0; c < n_chunks; ++c, ++cg) {
        const int ab = (int)(cg % NACC);
        const int gi = c * M2 + (int)rank * tc::M + ep;
        float* dst[2] = {nullptr, nullptr};
        int64_t plane = 0;
        int e_c = 0;
        if (gi < n) {
          int l = 0;
          while (l + 1 < P.levels && gi >= S.prefix[l + 1]) ++l;
          const int idx = gi - S.prefix[l];
          const int cy = S.hull[l][0] + idx / S.hw[l], cx = S.hull[l][2] + idx % S.hw[l];
          const int ch = P.ch[l], cw = P.cw[l];
          plane = (int64_t)ch * cw * TQW;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (S.tile[j] < 0) continue;
            const TilePlan& tp = S.plan[j][l];
            if (tp.status == ST_OK && in_box(tp.B, cy, cx))
              dst[j] = P.cache[l] + (int64_t)S.tile[j] * plane * TQH +
                       (int64_t)slot_of(cy, cx, ch, cw) * TQW;
          }
          if (!(DEBUG && (T.dbg & 64))) e_c = T.e2[l][pair * T.pair_bytes[l] + (int64_t)cy * P.tw[l] + cx];
        }
        if (!__all_sync(0xffffffffu, WAIT_FULL2(U(C.acc_full[ab]), cg / NACC))) goto done;
        tc::tc_fence_after();
        float vm[32], vc[32];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t col = (uint32_t)(j * 64 + h * 32);
            tc::tmem_ld32(tmem + ab * 256 + lane_base + col, vm);
            tc::tmem_ld32(tmem + ab * 256 + 128 + lane_base + col, vc);
            if (dst[j] != nullptr && !(DEBUG && (T.dbg & 2))) {
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) {
                const int r = gg >> 1, cc = gg & 1;
                const int j0 = 16 * r + 4 * cc, j1 = j0 + 8;
                float o[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  o[i] = (vm[j0 + i] + vc[j0 + i]) * tc::exp2_neg(e_q[j][h * 32 + j0 + i] + e_c);
                  o[4 + i] = (vm[j1 + i] + vc[j1 + i]) * tc::exp2_neg(e_q[j][h * 32 + j1 + i] + e_c);
                }
                const int grp = (2 * h + r) * 2 + cc;
                tc::st_global_v8(dst[j] + grp * plane, o);
              }
            }
          }
        }
        tc::tc_fence_before();
        if (leader) {
          __syncwarp();
          if (lane == 0) tcp::arrive(U(C.acc_empty[ab]));
        } else {
          tc::named_bar(2, 128);
          if (ep == 0) arrive_remote(acc_empty_base + ab * (uint32_t)sizeof(uint64_t));
        }
      }
      tcp::arrive(U(C.plan_empty[s]));
    }
  }
done:
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace tcp2

}  // namespace cvb

using namespace cvb;


extern "C" {

// split-operand bytes of one pair at level l: hi plane, lo plane, exponents
static int64_t tc_pair_bytes(const cvb_partial_desc* desc, int l, int dp) {
  const int64_t cells = (int64_t)desc->th[l] * desc->tw[l];
  return 4 * cells * dp + ceil_div(cells, 16) * 16;
}

int cvb_tc_sizes(const cvb_partial_desc* desc, int64_t* f1_split_bytes,
                 int64_t* f2_split_bytes_per_level) {
  CVB_REQUIRE(desc, "tc_sizes: null desc");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  const int dp = (int)ceil_div(desc->d, tc::KP) * tc::KP;
  CVB_REQUIRE(dp <= tc::MAX_DP, "tensor-core path supports D <= %d", tc::MAX_DP);
  const int64_t nt = ceil_div(desc->h1, TQH) * ceil_div(desc->w1, TQW) * batch_of(desc);
  // F1: per-tile B images (tiles of every pair), then one exponent byte per query
  if (f1_split_bytes) *f1_split_bytes = nt * tc::N * dp * 4 + nt * tc::N;
  // per level and pair: hi plane, lo plane, then one exponent byte per cell
  if (f2_split_bytes_per_level)
    for (int l = 0; l < desc->levels; ++l)
      f2_split_bytes_per_level[l] = tc_pair_bytes(desc, l, dp) * batch_of(desc);
  return CVB_OK;
}

static int prep_grid(int64_t rows) {
  const int64_t g = ceil_div(rows, 8);
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

int cvb_tc_prepare(const cvb_partial_desc* desc, const float* f1, float* const* f2_levels_host,
                   void* f1_split, void* const* f2_split_host, int32_t flags, void* stream) {
  int64_t f1b = 0;
  int st = cvb_tc_sizes(desc, &f1b, nullptr);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(f1 && f2_levels_host && f1_split && f2_split_host, "tc_prepare: null pointer");
  cudaStream_t s = as_stream(stream);
  const int d = desc->d;
  const int dp = (int)ceil_div(d, tc::KP) * tc::KP;
  const int tiles_x = (int)ceil_div(desc->w1, TQW);
  const int64_t tiles_pp = ceil_div(desc->h1, TQH) * tiles_x;
  const int batch = batch_of(desc);
  const int64_t n_all = tiles_pp * batch;
  const int64_t tile_bytes = (int64_t)tc::N * dp * 4;
  const bool pool = flags & CVB_PREP_POOL;
  for (int l = 0; l < desc->levels; ++l)
    CVB_REQUIRE(f2_levels_host[l] && f2_split_host[l], "tc_prepare: null level pointer");
  auto aligned = [&](const void* p) { return d % 4 == 0 && ((uintptr_t)p & 15) == 0; };
  // level 0 is split by the level-1 pooling pass when there is one
  const bool fuse01 = pool && desc->levels > 1;
  for (int b = 0; b < batch; ++b) {  // pair-major buffers: one pass per pair
    const float* f1b_ = f1 + (int64_t)b * desc->h1 * desc->w1 * d;
    uint8_t* f1s = reinterpret_cast<uint8_t*>(f1_split);
    tc::split_f1_kernel<<<prep_grid(tiles_pp * (tc::N / 8)), 256, 0, s>>>(
        f1b_, desc->h1, desc->w1, d, dp, tiles_x, tiles_pp, aligned(f1b_),
        f1s + b * tiles_pp * tile_bytes,
        reinterpret_cast<int8_t*>(f1s + n_all * tile_bytes + b * tiles_pp * tc::N));
    if ((st = check_launch("tc_split_f1")) != CVB_OK) return st;
    auto level_of = [&](int l) {
      return f2_levels_host[l] + (int64_t)b * desc->th[l] * desc->tw[l] * d;
    };
    auto planes_of = [&](int l) {
      return reinterpret_cast<__half*>(reinterpret_cast<uint8_t*>(f2_split_host[l]) +
                                       b * tc_pair_bytes(desc, l, dp));
    };
    auto exps_of = [&](int l) {
      return reinterpret_cast<int8_t*>(planes_of(l) + 2 * (int64_t)desc->th[l] * desc->tw[l] * dp);
    };
    for (int l = 0; l < desc->levels; ++l) {
      const int h = desc->th[l], w = desc->tw[l];
      const int64_t cells = (int64_t)h * w;
      if (l == 0 && fuse01) {
        const int64_t tail = cells - (int64_t)(h / 2) * 2 * ((w / 2) * 2);
        if (tail > 0) {
          tc::split_tail_kernel<<<prep_grid(tail), 256, 0, s>>>(
              level_of(0), h, w, d, dp, aligned(level_of(0)), planes_of(0), exps_of(0));
          if ((st = check_launch("tc_split_tail")) != CVB_OK) return st;
        }
        continue;
      }
      const bool pool_l = pool && l > 0;
      if (pool_l)
        CVB_REQUIRE(desc->th[l - 1] / 2 == h && desc->tw[l - 1] / 2 == w,
                    "tc_prepare: level %d dims are not the 2x2 pool of level %d", l, l - 1);
      const float* src = pool_l ? level_of(l - 1) : level_of(l);
      const bool v = aligned(src) && aligned(level_of(l));
      const bool split_src = fuse01 && l == 1;
      tc::split_level_kernel<<<prep_grid(cells), 256, 0, s>>>(
          src, pool_l ? desc->tw[l - 1] : w, level_of(l), h, w, d, dp, pool_l, v, planes_of(l),
          exps_of(l), split_src ? planes_of(0) : nullptr, split_src ? exps_of(0) : nullptr,
          (int64_t)desc->th[0] * desc->tw[0]);
      if ((st = check_launch("tc_split_level")) != CVB_OK) return st;
    }
  }
  return CVB_OK;
}

int64_t cvb_dense_tc_workspace(const cvb_partial_desc* desc) {
  if (desc == nullptr) return 0;
  const int64_t nt = ceil_div(desc->h1, TQH) * ceil_div(desc->w1, TQW);
  return (nt + 1) * PLAN_INTS * (int64_t)sizeof(int);
}

int cvb_dense_tc(const cvb_partial_desc* desc, const void* f1_split,
                 const void* const* f2_split_host, void* workspace, float* const* out_levels_host,
                 void* stream) {
  CVB_REQUIRE(desc && f1_split && f2_split_host && workspace && out_levels_host,
              "dense_tc: null argument");
  CVB_REQUIRE(desc->levels >= 1 && desc->levels <= CVB_MAX_LEVELS, "bad level count");
  CVB_REQUIRE(desc->batch <= 1, "dense_tc: one image pair");
  CVB_REQUIRE(desc->h1 >= 1 && desc->w1 >= 1 && desc->d >= 1, "bad source dims");
  tc::TcParams T;
  memset(&T, 0, sizeof(T));
  PartialParams& P = T.P;
  P.h1 = desc->h1;
  P.w1 = desc->w1;
  P.d = desc->d;
  P.levels = desc->levels;
  P.radius = desc->radius;
  P.tiles_x = (int)ceil_div(desc->w1, TQW);
  P.batch = 1;
  P.tiles_pp = ceil_div(desc->h1, TQH) * (int64_t)P.tiles_x;
  P.n_tiles = P.tiles_pp;
  P.tile0 = 0;
  P.ntile = P.n_tiles;
  P.plans = reinterpret_cast<int32_t*>(workspace);
  T.dp = (int)ceil_div(desc->d, tc::KP) * tc::KP;
  CVB_REQUIRE(T.dp <= tc::MAX_DP, "tensor-core path supports D <= %d", tc::MAX_DP);
  T.f1s = reinterpret_cast<const uint8_t*>(f1_split);
  T.e1 = reinterpret_cast<const int8_t*>(T.f1s + P.n_tiles * tc::N * T.dp * 4);
  for (int l = 0; l < desc->levels; ++l) {
    P.th[l] = desc->th[l];
    P.tw[l] = desc->tw[l];
    P.ch[l] = P.cw[l] = 1;
    CVB_REQUIRE(P.th[l] >= 1 && P.tw[l] >= 1, "empty target level %d", l);
    CVB_REQUIRE((int64_t)P.th[l] * P.tw[l] < (1LL << 28), "dense_tc: level too large");
    CVB_REQUIRE(f2_split_host[l] && out_levels_host[l], "dense_tc: null level pointer");
    T.f2s[l] = reinterpret_cast<const __half*>(f2_split_host[l]);
    T.plane[l] = (int64_t)desc->th[l] * desc->tw[l] * T.dp;
    T.pair_bytes[l] = 0;
    T.e2[l] = reinterpret_cast<const int8_t*>(T.f2s[l] + 2 * T.plane[l]);
    T.dense[l] = out_levels_host[l];
  }
  cudaStream_t s = as_stream(stream);
  int* word = tcp::watchdog_word(s);
  T.watchdog = word != nullptr ? tcp::watchdog_dev : nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  const int n_sms = tcp::sm_count(dev);
  const size_t smem = tcp::smem_bytes();
  static std::atomic<uint64_t> attr{0};
  ensure_max_smem(attr, tcp::partial_contract_tcp_kernel<false, true>, (int)smem);
  tcp::dense_plan_kernel<<<(unsigned)ceil_div(P.n_tiles, 128), 128, 0, s>>>(P);
  int st = check_launch("dense_plan");
  if (st != CVB_OK) return st;
  const int64_t grid = P.ntile < n_sms ? P.ntile : n_sms;
  launch_pdl(tcp::partial_contract_tcp_kernel<false, true>, dim3((unsigned)grid),
             dim3(tcp::THREADS), smem, s, T);
  return check_launch("dense_tc");
}

int cvb_partial_contract_tc(const cvb_partial_desc* desc, const float* f1,
                            const float* const* f2_levels_host, const void* f1_split,
                            const void* const* f2_split_host, const void* coords, int32_t* meta,
                            float* const* cache_levels_host, unsigned long long* counters,
                            int32_t flags, void* stream) {
  tc::TcParams T;
  memset(&T, 0, sizeof(T));
  int st = cvb_internal_build_params(desc, f1, f2_levels_host, coords, 1.0f, meta,
                                     cache_levels_host, counters, flags, T.P);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(!(flags & CVB_STRICT), "tensor-core contraction has no strict mode");
  CVB_REQUIRE(f1_split && f2_split_host, "partial_contract_tc: null pointer");
  T.dp = (int)ceil_div(desc->d, tc::KP) * tc::KP;
  CVB_REQUIRE(T.dp <= tc::MAX_DP, "tensor-core path supports D <= %d", tc::MAX_DP);
  T.f1s = reinterpret_cast<const uint8_t*>(f1_split);
  const int64_t n_tiles_all = T.P.n_tiles;
  T.e1 = reinterpret_cast<const int8_t*>(T.f1s + n_tiles_all * tc::N * T.dp * 4);
  for (int l = 0; l < CVB_MAX_LEVELS; ++l) {
    const bool used = l < desc->levels;
    T.f2s[l] = used ? reinterpret_cast<const __half*>(f2_split_host[l]) : nullptr;
    T.plane[l] = used ? (int64_t)desc->th[l] * desc->tw[l] * T.dp : 0;
    T.pair_bytes[l] = used ? tc_pair_bytes(desc, l, T.dp) : 0;
    T.e2[l] = used ? reinterpret_cast<const int8_t*>(T.f2s[l] + 2 * T.plane[l]) : nullptr;
    if (used) CVB_REQUIRE(T.f2s[l], "partial_contract_tc: null level pointer");
  }
  // a watchdog abort of an earlier launch (its outputs are invalid) surfaces here
  int* word = tcp::watchdog_word(as_stream(stream));
  if (word != nullptr && *(volatile int*)word != 0) {
    *(volatile int*)word = 0;
    set_error("partial_contract_tc: a previous contraction launch was aborted by its pipeline "
              "watchdog (a ring wait exceeded %llu s); its cache and outputs are invalid",
              tcp::WATCHDOG_NS / 1000000000ull);
    return CVB_ERR_CUDA;
  }
  T.watchdog = word != nullptr ? tcp::watchdog_dev : nullptr;
  if (T.P.ntile == 0) return CVB_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const int n_sms = tcp::sm_count(dev);
  static int dbg = -1;  // CVB_TC_DEBUG: profiling knock-outs / timeline (debug kernel)
  if (dbg < 0) {
    const char* e = getenv("CVB_TC_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  T.dbg = dbg;
  static unsigned long long* ts_buf = nullptr;
  T.ts = nullptr;
  if (dbg & 16) {
    if (ts_buf == nullptr) cudaMalloc(&ts_buf, 4 * 64 * 32 * sizeof(unsigned long long));
    cudaMemsetAsync(ts_buf, 0, 4 * 64 * 32 * sizeof(unsigned long long), as_stream(stream));
    T.ts = ts_buf;
  }
  const size_t smem = tcp::smem_bytes();
  auto kernel = dbg ? tcp::partial_contract_tcp_kernel<true> : tcp::partial_contract_tcp_kernel<false>;
  static std::atomic<uint64_t> attr_prod{0}, attr_dbg{0};
  ensure_max_smem(dbg ? attr_dbg : attr_prod, kernel, (int)smem);
  launch_pdl(tcp::plan_kernel, dim3((unsigned)ceil_div(T.P.ntile, tcp::PLAN_WARPS)),
             dim3(tcp::PLAN_WARPS * 32), 0, as_stream(stream), T.P);
  if ((st = check_launch("partial_plan")) != CVB_OK) return st;
  // cold iterations on SM pairs: every tile row of the range is whole
  const bool rows_whole = T.P.tile0 % T.P.tiles_x == 0 && T.P.ntile % T.P.tiles_x == 0;
  // (CVB_TC_DEBUG: the single-tile debug kernel, or with bit 256 the pair
  // kernel's debug instantiation)
  if ((flags & CVB_TC_PAIRS) && (!dbg || (dbg & 256)) && rows_whole && n_sms >= 2 &&
      T.P.levels <= tcp2::PMAXL) {
    const int64_t n_pairs = T.P.ntile / T.P.tiles_x * ((T.P.tiles_x + 1) / 2);
    const size_t smem2 = tcp2::smem_bytes();
    auto kernel2 = dbg ? tcp2::pair_contract_kernel<true> : tcp2::pair_contract_kernel<false>;
    static std::atomic<uint64_t> attr2{0}, attr2_dbg{0};
    ensure_max_smem(dbg ? attr2_dbg : attr2, kernel2, (int)smem2);
    const int64_t max_cl = n_sms / 2;
    const int64_t grid2 = 2 * (n_pairs < max_cl ? n_pairs : max_cl);
    launch_pdl_phase(kernel2, dim3((unsigned)grid2), dim3(tcp2::THREADS), smem2,
               as_stream(stream), T, n_pairs);
    return check_launch("partial_contract_tcp2");
  }
  const int64_t grid = T.P.ntile < n_sms ? T.P.ntile : n_sms;
  launch_pdl_phase(kernel, dim3((unsigned)grid), dim3(tcp::THREADS), smem, as_stream(stream), T);
  if (T.ts != nullptr) {  // debug timeline dump (CTA 0..3, first 64 tiles, 32 events), ns
    static unsigned long long h[4 * 64 * 32];
    cudaStreamSynchronize(as_stream(stream));
    cudaMemcpy(h, T.ts, sizeof(h), cudaMemcpyDeviceToHost);
    static int call = 0;
    ++call;
    const char* path = getenv("CVB_TC_TS_FILE");
    if (path != nullptr) {
      FILE* f = fopen(path, call == 1 ? "wb" : "ab");
      if (f) {
        fwrite(h, sizeof(h), 1, f);
        fclose(f);
      }
    }
  }
  return check_launch("partial_contract_tcp");
}

}  // extern "C"
