// DRAM traffic of scattered partial-line WRITES (run under ncu with
// dram__bytes_read.sum, dram__bytes_write.sum): each probe writes to every
// 128-byte line of a 2 GB buffer in hashed order (16M lines, footprint >> L2):
//   probe 0: one 32-byte sector per line (st.global.v8.f32 by one lane)  0.5 GB
//   probe 1: two adjacent sectors (64 B) per line                        1 GB
//   probe 2: the whole line (128 B)                                       2 GB
// Written bytes beyond the requested ones (or DRAM reads) mean line-granular
// write-back or fills.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; return x;
}
__device__ __forceinline__ void st8(float* p, float v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
template <int P>
__global__ void probe(float* p, int64_t lines) {
  const int64_t n = lines;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = (int64_t)(mix(i) % (uint64_t)n);
    float* l = p + line * 32;
    st8(l + 8, 1.f);
    if (P >= 1) st8(l + 16, 1.f);
    if (P >= 2) { st8(l, 1.f); st8(l + 24, 1.f); }
  }
}
int main() {
  const int64_t bytes = 1ll << 31, lines = bytes / 128;
  float* p;
  cudaMalloc(&p, bytes);
  cudaMemset(p, 0, bytes);
  cudaDeviceSynchronize();
  probe<0><<<148 * 16, 256>>>(p, lines);
  probe<1><<<148 * 16, 256>>>(p, lines);
  probe<2><<<148 * 16, 256>>>(p, lines);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
