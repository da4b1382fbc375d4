// DRAM fetch granularity probe (run under ncu with dram__bytes_read.sum and
// lts__t_sectors_srcunit_tex_op_read.sum).  Each probe reads ONE 32-byte
// sector from each of N lines (8 lanes x 4 B):
//   probe 0: every line, in order (streaming)           requested 0.537 GB
//   probe 1: every 8th line, in order                    requested 0.067 GB
//   probe 2: 1/8 of the lines, hashed (scattered) order  requested 0.067 GB
//   probe 3: every line, hashed order                    requested 0.537 GB
//   probe 4: 2 adjacent sectors (64 B) of every 8th line requested 0.134 GB
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; return x;
}
template <int P>
__global__ void probe(const float* p, int64_t lines, float* out) {
  float acc = 0.f;
  const int lane = threadIdx.x & 31;
  const int64_t units = (P == 0 || P == 3) ? lines / 4 : lines / 32;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < units;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t i = w * 4 + (lane >> 3);  // access index
    int64_t line;
    if (P == 0) line = i;
    else if (P == 1 || P == 4) line = i * 8;
    else if (P == 2) line = (int64_t)(mix(i) % (uint64_t)(lines / 8)) * 8;
    else line = (int64_t)(mix(i) % (uint64_t)lines);
    const float* l = p + line * 32;
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(l + 8 + (lane & 7)));
    acc += v;
    if (P == 4) {
      asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(l + 16 + (lane & 7)));
      acc += v;
    }
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
  printf("done\n");
  return 0;
}
