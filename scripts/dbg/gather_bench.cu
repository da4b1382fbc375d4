// Microbenchmark: A-operand row gather into a 4-stage 128B-swizzled smem ring
// (128 rows x 64 fp16, hi and lo planes = 32 KB per stage), LDGSTS (cp.async,
// 8 lanes per row, noinc arrive) vs TMA tile::gather4 (one tensor map over
// the hi/lo row planes).  The consumer just releases stages.  Reports GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void arrive(uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory"); }
__device__ __forceinline__ uint32_t hashu(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
constexpr int NST = 4, STAGE = 32768, HALF = 16384;
// row of chunk c, slot r: random within [0, span) around a CTA-dependent base
__device__ __forceinline__ int row_of(int cta, int c, int r, int nrows, int span) {
  const int base = (int)((hashu(cta * 7919 + c) % (uint32_t)nrows));
  return (base + (int)(hashu(cta * 131071 + c * 977 + r) % (uint32_t)span)) % nrows;
}
template <int MODE>
__global__ void __launch_bounds__(384, 1) k(const __half* f2, const __grid_constant__ CUtensorMap tm, int nrows,
                                            int span, int nchunks, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(MODE == 1 || MODE == 3 ? 1 : MODE == 4 ? 129 : MODE == 5 ? 256 : 128) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t uA = su32(sm);
  const long long t0 = clock64();
  const int64_t plane = (int64_t)nrows * 256;
  if (warp == 1) {  // consumer
    if (lane == 0) {
      for (int g = 0; g < nchunks * 4; ++g) {
        const int s = g % NST;
        while (!tryw(su32(&full[s]), (g / NST) & 1)) {}
        arrive(su32(&empty[s]));
      }
      out[blockIdx.x] = clock64() - t0;
    }
  } else if (MODE == 0 && warp >= 4 && warp < 8) {
    const int aw = warp - 4, sub = lane >> 3, chunk = lane & 7;
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int my_row = row_of(blockIdx.x, c, 32 * aw + lane, nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        const uint32_t stage = uA + st * STAGE;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = 4 * i + sub;
          const int r = __shfl_sync(0xffffffffu, my_row, rl);
          const int row = 32 * aw + rl;
          const uint32_t dst = stage + row * 128 + ((chunk ^ (row & 7)) << 4);
          const __half* src = f2 + (int64_t)r * 256 + kb * 64 + chunk * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + HALF), "l"(src + plane) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
      }
    }
  } else if (MODE == 2 && warp >= 4 && warp < 8) {
    // LDG.128 into registers (8 lanes per row), then st.shared into the swizzled stage
    const int aw = warp - 4, sub = lane >> 3, chunk = lane & 7;
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int my_row = row_of(blockIdx.x, c, 32 * aw + lane, nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        uint4 vh[8], vl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = 4 * i + sub;
          const int r = __shfl_sync(0xffffffffu, my_row, rl);
          const __half* src = f2 + (int64_t)r * 256 + kb * 64 + chunk * 8;
          vh[i] = __ldg(reinterpret_cast<const uint4*>(src));
          vl[i] = __ldg(reinterpret_cast<const uint4*>(src + plane));
        }
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        uint8_t* stage = sm + st * STAGE;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = 32 * aw + 4 * i + sub;
          *reinterpret_cast<uint4*>(stage + row * 128 + ((chunk ^ (row & 7)) << 4)) = vh[i];
          *reinterpret_cast<uint4*>(stage + HALF + row * 128 + ((chunk ^ (row & 7)) << 4)) = vl[i];
        }
        arrive(su32(&full[st]));
      }
    }
  } else if (MODE == 3 && warp >= 4 && warp < 8) {
    // TMA gather4 issued by 8 lanes of each of 4 warps (4 rows per lane)
    const int aw = warp - 4;
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = row_of(blockIdx.x, c, 32 * aw + 4 * (lane & 7) + j, nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        if (aw == 0 && lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(STAGE) : "memory");
        if (lane < 8) {
          const uint32_t dst = uA + st * STAGE + (32 * aw + 4 * lane) * 128;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(&tm), "r"(kb * 64), "r"(r[0]), "r"(r[1]),
              "r"(r[2]), "r"(r[3]), "r"(su32(&full[st])) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst + HALF), "l"(&tm), "r"(kb * 64), "r"(r[0] + nrows),
              "r"(r[1] + nrows), "r"(r[2] + nrows), "r"(r[3] + nrows), "r"(su32(&full[st])) : "memory");
        }
      }
    }
  } else if (MODE == 5 && (warp >= 4)) {
    // LDGSTS from 8 warps (warps 4-11), 16 rows each
    const int aw = warp - 4, sub = lane >> 3, chunk = lane & 7;
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int my_row = row_of(blockIdx.x, c, 16 * aw + (lane & 15), nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        const uint32_t stage = uA + st * STAGE;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rl = 4 * i + sub;
          const int r = __shfl_sync(0xffffffffu, my_row, rl);
          const int row = 16 * aw + rl;
          const uint32_t dst = stage + row * 128 + ((chunk ^ (row & 7)) << 4);
          const __half* src = f2 + (int64_t)r * 256 + kb * 64 + chunk * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + HALF), "l"(src + plane) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
      }
    }
  } else if (MODE == 4 && warp >= 4 && warp < 8) {
    // hi half by TMA gather4 (lanes 0-7), lo half by LDGSTS (all lanes, noinc)
    const int aw = warp - 4, sub = lane >> 3, chunk = lane & 7;
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = row_of(blockIdx.x, c, 32 * aw + 4 * (lane & 7) + j, nrows, span);
      const int my_row = row_of(blockIdx.x, c, 32 * aw + lane, nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        if (aw == 0 && lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(HALF) : "memory");
        const uint32_t stage = uA + st * STAGE;
        if (lane < 8) {
          const uint32_t dst = stage + (32 * aw + 4 * lane) * 128;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(&tm), "r"(kb * 64), "r"(r[0]), "r"(r[1]),
              "r"(r[2]), "r"(r[3]), "r"(su32(&full[st])) : "memory");
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = 4 * i + sub;
          const int rr = __shfl_sync(0xffffffffu, my_row, rl);
          const int row = 32 * aw + rl;
          const uint32_t dst = stage + HALF + row * 128 + ((chunk ^ (row & 7)) << 4);
          const __half* src = f2 + (int64_t)rr * 256 + kb * 64 + chunk * 8 + plane;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
      }
    }
  } else if (MODE == 1 && warp == 4) {
    int g = 0;
    for (int c = 0; c < nchunks; ++c) {
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = row_of(blockIdx.x, c, 4 * lane + j, nrows, span);
      for (int kb = 0; kb < 4; ++kb, ++g) {
        const int st = g % NST;
        while (!tryw(su32(&empty[st]), ((g / NST) & 1) ^ 1)) {}
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(STAGE) : "memory");
        __syncwarp();
        const uint32_t dst = uA + st * STAGE + lane * 512;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(&tm), "r"(kb * 64), "r"(r[0]), "r"(r[1]),
            "r"(r[2]), "r"(r[3]), "r"(su32(&full[st])) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst + HALF), "l"(&tm), "r"(kb * 64), "r"(r[0] + nrows),
            "r"(r[1] + nrows), "r"(r[2] + nrows), "r"(r[3] + nrows), "r"(su32(&full[st])) : "memory");
      }
    }
  }
}
// check: gather4 writes the same bytes as the cp.async path (first stage of CTA 0)
__global__ void check(const __half* f2, const __grid_constant__ CUtensorMap tm, int nrows, int* bad) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  int r[4];
  for (int j = 0; j < 4; ++j) r[j] = (int)(hashu(4 * lane + j) % (uint32_t)nrows);
  if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(HALF) : "memory");
  __syncwarp();
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(sm) + lane * 512), "l"(&tm), "r"(64), "r"(r[0]), "r"(r[1]),
      "r"(r[2]), "r"(r[3]), "r"(su32(&bar)) : "memory");
  while (!tryw(su32(&bar), 0)) {}
  int nb = 0;
  for (int j = 0; j < 4; ++j) {
    const int row = 4 * lane + j;
    for (int ch = 0; ch < 8; ++ch) {
      const uint4 a = *reinterpret_cast<const uint4*>(sm + row * 128 + ((ch ^ (row & 7)) << 4));
      const uint4 b = *reinterpret_cast<const uint4*>(f2 + (int64_t)r[j] * 256 + 64 + ch * 8);
      nb += (a.x != b.x) + (a.y != b.y) + (a.z != b.z) + (a.w != b.w);
    }
  }
  atomicAdd(bad, nb);
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int nrows = 518400;
  __half* f2; cudaMalloc(&f2, (size_t)nrows * 256 * 2 * 2);
  std::vector<uint16_t> h((size_t)nrows * 512);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  cudaMemcpy(f2, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {256, (cuuint64_t)nrows * 2}, strides[1] = {512};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, f2, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)rc);
  int* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  check<<<1, 32, 20000>>>(f2, tm, nrows, bad);
  int hb = -1; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("gather4 layout check: %d mismatching words (%s)\n", hb, cudaGetErrorString(cudaGetLastError()));
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  unsigned long long hh[148];
  const int smem = NST * STAGE + 1024, nch = 400;
  for (int span : {1 << 30, 4096, 512}) {
    for (int tma = 0; tma < 6; ++tma) {
      if (tma == 2 || tma == 1 || tma == 4) continue;
      auto kern = tma == 0 ? k<0> : tma == 1 ? k<1> : tma == 2 ? k<2> : tma == 3 ? k<3> : tma == 4 ? k<4> : k<5>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      kern<<<148, 384, smem>>>(f2, tm, nrows, span > nrows ? nrows : span, nch, d);
      cudaEventRecord(e0);
      kern<<<148, 384, smem>>>(f2, tm, nrows, span > nrows ? nrows : span, nch, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = 148.0 * nch * 4 * STAGE;
      printf("%s span %8d rows: %.3f ms, %.0f GB/s into smem (%s)\n", tma == 1 ? "TMA gather4" : tma == 2 ? "LDG+STS    " : tma == 3 ? "gather4 x32" : tma == 4 ? "hi TMA+lo LDGSTS" : tma == 5 ? "LDGSTS 8 warps" : "LDGSTS     ",
             span > nrows ? nrows : span, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
