// Kernel lane on the GPU: corr_pairs, corr_gather, block_mmm
// (_ckernels.pyx:17-70, _pykernels.py:18-58).  Also the dense-variant level
// volume builder (build_dense_volume, dense.py:27-45 calls corr_pairs).
#include "gemm.cuh"

namespace cvb {

template <bool STRICT>
__global__ void __launch_bounds__(GEMM_THREADS)
    pairs_kernel(const float* __restrict__ a, int64_t n, const float* __restrict__ b, int64_t m,
                 int d, float* __restrict__ out, int64_t a_bstride, int64_t b_bstride,
                 int64_t o_bstride, bool vec) {
  __shared__ __align__(16) float smem[GEMM_SMEM_FLOATS];
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  const int64_t batch = blockIdx.z;
  a += batch * a_bstride;
  b += batch * b_bstride;
  out += batch * o_bstride;
  const float* rowsA[2];
  const float* rowsB[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int r = (threadIdx.x >> 3) + 32 * s;
    rowsA[s] = (i0 + r < n) ? a + (i0 + r) * d : nullptr;
    rowsB[s] = (j0 + r < m) ? b + (j0 + r) * d : nullptr;
  }
  float acc[4][4];
  gemm_tile_64x64<STRICT>(rowsA, rowsB, d, vec, smem, acc);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = i0 + ty * 4 + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = j0 + tx * 4 + j;
      if (c < m) out[r * m + c] = acc[i][j];
    }
  }
}

template <bool STRICT>
__global__ void __launch_bounds__(256)
    gather_kernel(const float* __restrict__ f1, int64_t p, const float* __restrict__ f2, int d,
                  const int64_t* __restrict__ idx, const uint8_t* __restrict__ valid,
                  float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p) return;
  if (!valid[i]) {
    out[i] = 0.f;
    return;
  }
  const float* x = f1 + i * d;
  const float* y = f2 + idx[i] * d;
  float acc = 0.f;
  for (int k = 0; k < d; ++k) acc = mac<STRICT>(acc, __ldg(x + k), __ldg(y + k));
  out[i] = acc;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

int launch_pairs(const float* a, int64_t n, const float* b, int64_t m, int d, float* out,
                 int64_t batches, int64_t a_bs, int64_t b_bs, int64_t o_bs, bool strict,
                 cudaStream_t s) {
  if (n == 0 || m == 0 || batches == 0) return CVB_OK;
  const bool vec = (d % 4 == 0) && aligned16(a) && aligned16(b) && (a_bs % 4 == 0) &&
                   (b_bs % 4 == 0);
  const int64_t gy = ceil_div(n, GT), gx = ceil_div(m, GT);
  if (gy > 65535 || gx > 2147483647LL || batches > 65535) {
    set_error("corr_pairs: problem too large for one launch");
    return CVB_ERR_INVALID;
  }
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)batches);
  if (strict)
    pairs_kernel<true><<<grid, GEMM_THREADS, 0, s>>>(a, n, b, m, d, out, a_bs, b_bs, o_bs, vec);
  else
    pairs_kernel<false><<<grid, GEMM_THREADS, 0, s>>>(a, n, b, m, d, out, a_bs, b_bs, o_bs, vec);
  return check_launch("corr_pairs");
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_corr_pairs(const float* a, int64_t n, const float* b, int64_t m, int32_t d, float* out,
                   int32_t flags, void* stream) {
  CVB_REQUIRE(d >= 1, "channel counts must be >= 1");
  CVB_REQUIRE(n >= 0 && m >= 0, "negative row count");
  CVB_REQUIRE((a && b && out) || n == 0 || m == 0, "corr_pairs: null pointer");
  return launch_pairs(a, n, b, m, d, out, 1, 0, 0, 0, flags & CVB_STRICT, as_stream(stream));
}

int cvb_block_mmm(const float* at, const float* bt, int64_t k, int32_t n, int32_t m, int32_t d,
                  float* out, int32_t flags, void* stream) {
  CVB_REQUIRE(d >= 1 && n >= 0 && m >= 0 && k >= 0, "block_mmm: bad dims");
  CVB_REQUIRE((at && bt && out) || k == 0 || n == 0 || m == 0, "block_mmm: null pointer");
  cudaStream_t s = as_stream(stream);
  // batch in slices of 65535 (grid.z limit)
  for (int64_t q0 = 0; q0 < k; q0 += 65535) {
    const int64_t kb = (k - q0) < 65535 ? (k - q0) : 65535;
    const int st = launch_pairs(at + q0 * n * d, n, bt + q0 * m * d, m, d, out + q0 * n * m, kb,
                                (int64_t)n * d, (int64_t)m * d, (int64_t)n * m,
                                flags & CVB_STRICT, s);
    if (st != CVB_OK) return st;
  }
  return CVB_OK;
}

int cvb_corr_gather(const float* f1, int64_t p, const float* f2, int64_t rows2, int32_t d,
                    const int64_t* idx, const uint8_t* valid, float* out, int32_t flags,
                    void* stream) {
  CVB_REQUIRE(d >= 1 && p >= 0 && rows2 >= 0, "corr_gather: bad dims");
  if (p == 0) return CVB_OK;
  CVB_REQUIRE(f1 && f2 && idx && valid && out, "corr_gather: null pointer");
  const unsigned grid = (unsigned)ceil_div(p, 256);
  if (flags & CVB_STRICT)
    gather_kernel<true><<<grid, 256, 0, as_stream(stream)>>>(f1, p, f2, d, idx, valid, out);
  else
    gather_kernel<false><<<grid, 256, 0, as_stream(stream)>>>(f1, p, f2, d, idx, valid, out);
  return check_launch("corr_gather");
}

}  // extern "C"
