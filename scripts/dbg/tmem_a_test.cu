// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (layout check).
// A[128][K] fp16 written to TMEM lane m, column k/2 (two fp16 per 32-bit
// column, low half = even k); B[64][K] fp16 in smem (K-major, no swizzle core
// matrices); D = A.B^T [128][64] fp32 in TMEM, read back and compared on host.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
constexpr int M = 128, N = 64, K = 64;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__global__ void k(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) __half sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B -> smem K-major no-swizzle: core matrix (8 rows x 8 k) contiguous 128 B;
  // [row group][k group][8][8]: LBO (k step) = 128 B, SBO (8-row step) = (K/8)*128
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, kk = i % K;
    sB[((n / 8) * (K / 8) + kk / 8) * 64 + (n % 8) * 8 + kk % 8] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tm;
  const uint32_t a_col = 128;  // A at columns 128.. (D at 0..63)
  // each thread = TMEM lane (row m); store its row's K values, 2 fp16 per column
  {
    const int m = warp * 32 + lane;
    uint32_t r[32];
    for (int c = 0; c < K / 2; ++c) {
      __half2 h = __halves2half2(A[m * K + 2 * c], A[m * K + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + a_col;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t db = make_desc(su32(sB) + s * 256, 128, (K / 8) * 128);
      const uint32_t acc = s > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "r"(tmem + a_col + s * 8), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int m = warp * 32 + lane;
    uint32_t r[32];
    for (int h = 0; h < 2; ++h) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + h * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) D[m * N + h * 32 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}
int main() {
  __half hA[M * K], hB[N * K]; float fA[M * K], fB[N * K];
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 4.0f; hA[i] = __float2half(v); fA[i] = v; }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 13 - 6) / 2.0f; hB[i] = __float2half(v); fB[i] = v; }
  __half *dA, *dB; float* dD; cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  float hD[M * N]; cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
  printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
  int bad = 0; double maxerr = 0;
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
    double ref = 0; for (int kk = 0; kk < K; ++kk) ref += (double)fA[m * K + kk] * fB[n * K + kk];
    double e = fabs(ref - hD[m * N + n]); maxerr = fmax(maxerr, e); if (e > 1e-3) ++bad;
    if (bad && bad < 4 && e > 1e-3) printf("m %d n %d ref %f got %f\n", m, n, ref, hD[m * N + n]);
  }
  printf("A-from-TMEM probe: %d mismatches, max err %g\n", bad, maxerr);
}
