// DRAM fill size vs the ld prefetch-size hint (run under ncu with
// dram__bytes_read.sum): every probe reads ONE 32-byte sector (8 lanes x 4 B)
// from 1/8 of the 128-byte lines of a 2 GB buffer in hashed (scattered) order
// (requested 0.067 GB):
//   probe 0: ld.global.nc                (no hint)
//   probe 1: ld.global.nc.L2::64B
//   probe 2: ld.global.nc.L2::256B
//   probe 3: ld.global (coherent) .L2::64B
//   probe 4: ld.global.nc.L1::no_allocate.L2::64B
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; return x;
}
template <int P>
__global__ void probe(const float* p, int64_t lines, float* out) {
  float acc = 0.f;
  const int lane = threadIdx.x & 31;
  const int64_t units = lines / 32;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < units;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = w * 4 + (lane >> 3);
    const int64_t line = (int64_t)(mix(i) % (uint64_t)(lines / 8)) * 8;
    const float* l = p + line * 32 + 8 + (lane & 7);
    float v;
    if (P == 0) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(l));
    if (P == 1) asm volatile("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(l));
    if (P == 2) asm volatile("ld.global.nc.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(l));
    if (P == 3) asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(l));
    if (P == 4) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(l));
    acc += v;
  }
  if (acc == 123.f) out[0] = acc;
}
int main() {
  const int64_t bytes = 1ll << 31, lines = bytes / 128;
  float* p;
  float* o;
  cudaMalloc(&p, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(p, 0, bytes);
  probe<0><<<148 * 16, 256>>>(p, lines, o);
  probe<1><<<148 * 16, 256>>>(p, lines, o);
  probe<2><<<148 * 16, 256>>>(p, lines, o);
  probe<3><<<148 * 16, 256>>>(p, lines, o);
  probe<4><<<148 * 16, 256>>>(p, lines, o);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
