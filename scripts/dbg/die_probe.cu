// Which die serves which address?  One warp on SM s chases dependent loads
// (L2-missing, 1 line each) through a buffer laid out so every access is to a
// chosen 4 KB page; the average latency per page, measured from SMs spread over
// the chip, shows whether a page is "near" or "far" for each SM.
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__global__ void probe(const uint64_t* buf, int64_t pages, int reps, unsigned long long* out, int target_sm) {
  if (smid() != (unsigned)target_sm || threadIdx.x != 0) return;
  for (int64_t p = 0; p < pages; ++p) {
    const uint64_t* base = buf + p * 512;  // 4 KB page = 512 x 8 B
    // touch 16 different lines of the page, dependent chain, flush by stride
    unsigned long long t0 = clock64();
    uint64_t idx = 0;
    for (int r = 0; r < reps; ++r) {
      idx = __ldcg(base + ((idx + r * 16) & 511));
    }
    unsigned long long t1 = clock64();
    out[(int64_t)target_sm * pages + p] = (t1 - t0) + (idx & 1);
  }
}
int main() {
  const int64_t pages = 4096;  // 16 MB
  uint64_t* buf;
  cudaMalloc(&buf, pages * 4096);
  cudaMemset(buf, 0, pages * 4096);
  unsigned long long* out;
  int nsm = 148;
  cudaMalloc(&out, nsm * pages * sizeof(unsigned long long));
  cudaMemset(out, 0, nsm * pages * sizeof(unsigned long long));
  const int sms[4] = {0, 40, 80, 120};
  for (int k = 0; k < 4; ++k) {
    // flush L2 between probes
    uint64_t* big; cudaMalloc(&big, 512ll << 20); cudaMemset(big, 1, 512ll << 20); cudaFree(big);
    probe<<<nsm * 4, 32>>>(buf, pages, 32, out, sms[k]);
  }
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(nsm * pages);
  cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  for (int k = 0; k < 4; ++k) {
    printf("sm %3d:", sms[k]);
    for (int p = 0; p < 64; ++p) printf(" %4llu", h[(int64_t)sms[k] * pages + p] / 32);
    printf("\n");
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
