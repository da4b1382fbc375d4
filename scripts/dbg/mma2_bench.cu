// Microbenchmark: tcgen05.mma.cta_group::2 (M=256 across an SM pair, kind::f16,
// SS operands) issue rate for the contraction's per-stage mix (N=128 + N=64 per
// K=16 step, 4 steps per stage), one issuing warp in the leader CTA, a
// multicast commit per stage.  Compare with mma_bench (cta_group::1: 603
// cycles per stage for half the rows).
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
template <uint32_t M, uint32_t N, int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t ID = (1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);
  if (CG == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(ID), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(ID), "r"(acc));
}
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ bool elect() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
  return e;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k2(unsigned long long* out, int n) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tm;
  const uint32_t rank = cta_rank();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < (4 * 32768 + 5 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tm;
  const uint32_t uA = su32(sm), uB = uA + 4 * 32768;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int g = 0; g < n; ++g) {
      const int st = g & 3, bs = g % 5;
      if (g >= 4) while (!tryw(su32(&bar[st]), ((g >> 2) - 1) & 1)) {}
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (rank == 0) {
        const uint32_t a_hi = uA + st * 32768, a_lo = a_hi + 16384, b = uB + bs * 16384;
        const uint32_t dm = tmem + (g & 1) * 128, dc = dm + 64;
        const uint64_t dah = dsw128(a_hi), dal = dsw128(a_lo), db = dnone(b, 128, 1024);
        if (elect()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma<256, 128, 2>(dm, dah + 2 * kk, db + 16 * kk, kk > 0);
            mma<256, 64, 2>(dc, dal + 2 * kk, db + 16 * kk, 1);
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(su32(&bar[st])), "h"((uint16_t)3) : "memory");
        }
        __syncwarp();
      }
    }
    for (int g = n - 4; g < n; ++g) while (!tryw(su32(&bar[g & 3]), (g >> 2) & 1)) {}
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  const int n = 4000, smem = 4 * 32768 + 5 * 16384 + 1024;
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k2<<<148, 128, smem>>>(d, n);
  k2<<<148, 128, smem>>>(d, n);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 148; i += 2) m += h[i]; m /= 74;
  printf("cta_group::2 M=256 mix N128+N64: %.1f cycles/stage per SM pair (%s)\n", m / n, cudaGetErrorString(e));
}
