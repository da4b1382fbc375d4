// Microbenchmark: latency of tcgen05.commit -> mbarrier completion, and issue cost.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(unsigned long long* out, int n) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // round trip: commit then wait for the phase to flip
    unsigned long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)(i & 1)) : "memory");
      }
    }
    unsigned long long t1 = clock64();
    // plain arrive round trip for comparison
    for (int i = 0; i < n; ++i) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)((n + i) & 1)) : "memory");
      }
    }
    unsigned long long t2 = clock64();
    out[0] = (t1 - t0) / n;
    out[1] = (t2 - t1) / n;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm) : "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  k<<<1, 128>>>(d, 1000);
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("commit->complete round trip %llu cycles, arrive->complete %llu cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
}
