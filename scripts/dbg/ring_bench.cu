// Microbenchmark: throughput of an mbarrier ring between one consumer thread
// (the MMA issuer's role) and 4 producer warps (the A producers' role), the
// synchronisation skeleton of partial_contract_tcp_kernel.  Cycles per stage.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
template <int NS, bool AGG>
__global__ void ring(unsigned long long* out, int n) {
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(AGG ? 4 : 128) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      for (int g = 0; g < n; ++g) {
        const int s = g % NS;
        while (!tryw(su32(&full[s]), (g / NS) & 1)) {}
        arrive(su32(&empty[s]));
      }
      out[blockIdx.x] = (clock64() - t0);
    }
  } else if (warp >= 4 && warp < 8) {
    for (int g = 0; g < n; ++g) {
      const int s = g % NS;
      while (!tryw(su32(&empty[s]), ((g / NS) & 1) ^ 1)) {}
      if (AGG) { __syncwarp(); if (lane == 0) arrive(su32(&full[s])); }
      else arrive(su32(&full[s]));
    }
  }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  const int n = 20000;
  auto run = [&](auto kern, const char* name) {
    kern<<<148, 384>>>(d, n);
    kern<<<148, 384>>>(d, n);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/stage (%s)\n", name, (double)h[0] / n, cudaGetErrorString(cudaGetLastError()));
  };
  run(ring<4, false>, "4 slots, 128 arrivals");
  run(ring<4, true>, "4 slots, 4 elected arrivals");
  run(ring<8, false>, "8 slots, 128 arrivals");
  run(ring<2, false>, "2 slots, 128 arrivals");
}
