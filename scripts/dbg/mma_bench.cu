// Microbenchmark: tcgen05.mma (kind::f16, SS operands, M=128) issue/execute
// rate for the contraction's per-stage MMA mix, one CTA per SM, one issuing
// thread, a commit per stage.  Prints cycles per stage (4 K16 steps).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t dsw128(uint32_t a) {
  return (uint64_t)((a & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t dnone(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <uint32_t N>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t ID = (1u << 4) | ((N >> 3) << 17) | ((128u >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(ID), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
template <uint32_t N>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  constexpr uint32_t ID = (1u << 4) | ((N >> 3) << 17) | ((128u >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(ID), "r"(acc));
}
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int n) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tm;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < (4 * 32768 + 5 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tm;
  const uint32_t uA = su32(sm), uB = uA + 4 * 32768;
  if (MODE >= 10 ? threadIdx.x < 32 : threadIdx.x == 0) {
    long long t0 = clock64();
    for (int g = 0; g < n; ++g) {
      const int st = g & 3, bs = g % 5;
      if (g >= 4) while (!tryw(su32(&bar[st]), ((g >> 2) - 1) & 1)) {}  // stage reuse (ring of 4)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = uA + st * 32768, a_lo = a_hi + 16384, b = uB + bs * 16384;
      const uint32_t dm = tmem + (g & 1) * 128, dc = dm + 64;
      if (MODE == 0 || MODE == 4) {  // kernel mix: N128 (A_hi, B hi+lo) + N64 (A_lo, B_hi), B no-swizzle
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bh = MODE == 0 ? dnone(b + kk * 256, 128, 1024) : dsw128(b + kk * 32);
          mma<128>(dm, dsw128(a_hi + kk * 32), bh, kk > 0);
          mma<64>(dc, dsw128(a_lo + kk * 32), bh, 1);
        }
      } else if (MODE == 5) {  // kernel mix, MMA2 into its own 64 columns (two independent chains)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bh = dnone(b + kk * 256, 128, 1024);
          mma<128>(tmem + (g & 1) * 192, dsw128(a_hi + kk * 32), bh, kk > 0);
          mma<64>(tmem + (g & 1) * 192 + 128, dsw128(a_lo + kk * 32), bh, kk > 0);
        }
      } else if (MODE == 6) {  // N128 only, two accumulators alternating by K step
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma<128>(tmem + (kk & 1) * 128, dsw128(a_hi + kk * 32), dnone(b + kk * 256, 128, 1024), kk > 1);
      } else if (MODE == 7 || MODE == 8) {  // kernel mix, A from TMEM (cols 256..511: 4 stages x 64 cols)
        const uint32_t ta = tmem + 256 + st * 64;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bh = dnone(b + kk * 256, 128, 1024);
          mma_ts<128>(dm, ta + kk * 8, bh, kk > 0);
          if (MODE == 7) mma_ts<64>(dc, ta + 32 + kk * 8, bh, 1);
        }
      } else if (MODE == 11 || MODE == 12) {  // warp-converged; 11: both N128; 12: 16 MMAs (K=128) per stage
        const uint64_t dah = dsw128(a_hi), dal = dsw128(a_lo), db = dnone(b, 128, 1024);
        uint32_t e;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
        if (e) {
#pragma unroll
          for (int kk = 0; kk < (MODE == 12 ? 8 : 4); ++kk) {
            mma<128>(dm, dah + 2 * (kk & 3), db + 16 * (kk & 3), kk > 0);
            if (MODE == 11) mma<128>(dm, dal + 2 * kk, db + 16 * kk, 1);
            else mma<64>(dc, dal + 2 * (kk & 3), db + 16 * (kk & 3), 1);
          }
        }
        __syncwarp();
      } else if (MODE == 9 || MODE == 10) {  // kernel mix, descriptors = base + constant
        const uint64_t dah = dsw128(a_hi), dal = dsw128(a_lo), db = dnone(b, 128, 1024);
        uint32_t e = 1;
        if (MODE == 10) asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
        if (e) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma<128>(dm, dah + 2 * kk, db + 16 * kk, kk > 0);
            mma<64>(dc, dal + 2 * kk, db + 16 * kk, 1);
          }
        }
        if (MODE == 10) __syncwarp();
      } else if (MODE == 1) {  // N128 only
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma<128>(dm, dsw128(a_hi + kk * 32), dnone(b + kk * 256, 128, 1024), kk > 0);
      } else if (MODE == 2) {  // N64 only
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma<64>(dc, dsw128(a_lo + kk * 32), dnone(b + kk * 256, 128, 1024), kk > 0);
      } else if (MODE == 3) {  // N256 only (B = 256 rows: reads A stage as B)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma<256>(tmem, dsw128(a_hi + kk * 32), dsw128(uA + ((st + 1) & 3) * 32768 + kk * 32), kk > 0);
      }
      if (MODE >= 10) {
        uint32_t e;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
        if (e) commit(su32(&bar[st]));
        __syncwarp();
      } else {
        commit(su32(&bar[st]));
      }
    }
    for (int g = n - 4; g < n; ++g) while (!tryw(su32(&bar[g & 3]), (g >> 2) & 1)) {}
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  const int n = 4000, smem = 4 * 32768 + 5 * 16384 + 1024;
  auto run = [&](auto kern, const char* name, double floor) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, 128, smem>>>(d, n);
    kern<<<148, 128, smem>>>(d, n);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
    printf("%-44s %7.1f cycles/stage (floor %.0f) %s\n", name, m / n, floor, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0>, "kernel mix N128+N64, B no-swizzle", 384);
  run(k<4>, "kernel mix N128+N64, B sw128", 384);
  run(k<5>, "kernel mix, MMA2 own columns", 384);
  run(k<6>, "N128 only, 2 alternating accumulators", 256);
  run(k<7>, "kernel mix, A in TMEM (TS)", 384);
  run(k<8>, "N128 only, A in TMEM (TS)", 256);
  run(k<9>, "kernel mix, base+offset descriptors", 384);
  run(k<10>, "kernel mix, base+offset, warp-converged elect", 384);
  run(k<11>, "warp elect, 2xN128 per K16", 512);
  run(k<12>, "warp elect, mix, 16 MMAs per stage", 768);
  run(k<1>, "N128 only", 256);
  run(k<2>, "N64 only", 128);
  run(k<3>, "N256 only", 512);
}
