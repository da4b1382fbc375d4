// (1) fmap2 avg-pool pyramid and dense-volume pooling — HBM-bound, bit-exact.
//
// pool2x2 (_pykernels.py:65-81): out = ((a+b)+(c+d))*0.25 in fp32 with floor
// dims.  The multiply by 0.25 is exact, so the association is the only
// rounding choice; __fadd_rn pins it.  Each thread moves one float4 of
// channels: a warp reads 4 x 512 contiguous bytes and writes 512, so the
// kernel streams at HBM rate (reads 4 B/elt-out * 4, writes 4 B/elt-out).
#include "common.cuh"

namespace cvb {

__device__ __forceinline__ float pool4(float a, float b, float c, float d) {
  return __fmul_rn(__fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d)), 0.25f);
}

__global__ void __launch_bounds__(256) pool2x2_vec4_kernel(const float4* __restrict__ in,
                                                           int w, int d4, float4* __restrict__ out,
                                                           int ho, int wo) {
  const int64_t total = (int64_t)ho * wo * d4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % d4);
    const int64_t cell = i / d4;
    const int x = (int)(cell % wo), y = (int)(cell / wo);
    const int64_t r0 = ((int64_t)(2 * y) * w + 2 * x) * d4 + c;
    const int64_t r1 = r0 + (int64_t)w * d4;
    const float4 a = __ldg(in + r0), b = __ldg(in + r0 + d4);
    const float4 e = __ldg(in + r1), f = __ldg(in + r1 + d4);
    float4 o;
    o.x = pool4(a.x, b.x, e.x, f.x);
    o.y = pool4(a.y, b.y, e.y, f.y);
    o.z = pool4(a.z, b.z, e.z, f.z);
    o.w = pool4(a.w, b.w, e.w, f.w);
    out[i] = o;
  }
}

__global__ void __launch_bounds__(256) pool2x2_scalar_kernel(const float* __restrict__ in, int w,
                                                             int d, float* __restrict__ out,
                                                             int ho, int wo) {
  const int64_t total = (int64_t)ho * wo * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % d);
    const int64_t cell = i / d;
    const int x = (int)(cell % wo), y = (int)(cell / wo);
    const int64_t r0 = ((int64_t)(2 * y) * w + 2 * x) * d + c;
    const int64_t r1 = r0 + (int64_t)w * d;
    out[i] = pool4(__ldg(in + r0), __ldg(in + r0 + d), __ldg(in + r1), __ldg(in + r1 + d));
  }
}

static int grid_for(int64_t work) {
  // 148 SMs x 8 resident 256-thread CTAs, grid-stride beyond that.
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 8 * 4) g = 148 * 8 * 4;
  return (int)(g < 1 ? 1 : g);
}

static int pool2x2_launch(const float* in, int h, int w, int d, float* out, cudaStream_t s) {
  const int ho = h / 2, wo = w / 2;
  const bool vec = (d % 4 == 0) && ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (vec) {
    const int d4 = d / 4;
    pool2x2_vec4_kernel<<<grid_for((int64_t)ho * wo * d4), 256, 0, s>>>(
        reinterpret_cast<const float4*>(in), w, d4, reinterpret_cast<float4*>(out), ho, wo);
  } else {
    pool2x2_scalar_kernel<<<grid_for((int64_t)ho * wo * d), 256, 0, s>>>(in, w, d, out, ho, wo);
  }
  return check_launch("pool2x2");
}

// pool_volume (dense.py:48-60): pools the target grid of every source row.
__global__ void __launch_bounds__(256) pool_volume_kernel(const float* __restrict__ mat,
                                                          int64_t p1, int th, int tw,
                                                          float* __restrict__ out) {
  const int ho = th / 2, wo = tw / 2;
  const int64_t per = (int64_t)ho * wo;
  const int64_t total = p1 * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / per;
    const int64_t cell = i % per;
    const int x = (int)(cell % wo), y = (int)(cell / wo);
    const float* m = mat + row * (int64_t)th * tw;
    const int64_t a = (int64_t)(2 * y) * tw + 2 * x;
    out[i] = pool4(__ldg(m + a), __ldg(m + a + 1), __ldg(m + a + tw), __ldg(m + a + tw + 1));
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_pool2x2(const float* in, int32_t h, int32_t w, int32_t d, float* out, void* stream) {
  CVB_REQUIRE(in && out, "pool2x2: null pointer");
  CVB_REQUIRE(h >= 2 && w >= 2 && d >= 1,
              "cannot 2x2-pool dims (%d, %d); both must be >= 2", (int)h, (int)w);
  return pool2x2_launch(in, h, w, d, out, as_stream(stream));
}

int cvb_build_pyramid(const float* f2, int32_t h, int32_t w, int32_t d, int32_t levels,
                      float* const* out_levels_host, void* stream) {
  CVB_REQUIRE(f2 && out_levels_host, "build_pyramid: null pointer");
  CVB_REQUIRE(levels >= 1 && levels <= CVB_MAX_LEVELS, "levels must be in [1, %d]",
              CVB_MAX_LEVELS);
  int hh = h, ww = w;
  for (int l = 1; l < levels; ++l) hh /= 2, ww /= 2;
  CVB_REQUIRE(hh >= 1 && ww >= 1,
              "pyramid of %d levels on %dx%d would produce an empty level", (int)levels, (int)h,
              (int)w);
  const float* cur = f2;
  hh = h;
  ww = w;
  for (int l = 1; l < levels; ++l) {
    CVB_REQUIRE(out_levels_host[l], "build_pyramid: null level pointer");
    const int st = pool2x2_launch(cur, hh, ww, d, out_levels_host[l], as_stream(stream));
    if (st != CVB_OK) return st;
    cur = out_levels_host[l];
    hh /= 2;
    ww /= 2;
  }
  return CVB_OK;
}

int cvb_pool_volume(const float* mat, int64_t p1, int32_t th, int32_t tw, float* out,
                    void* stream) {
  CVB_REQUIRE(mat && out, "pool_volume: null pointer");
  CVB_REQUIRE(th >= 2 && tw >= 2, "cannot 2x2-pool dims (%d, %d); both must be >= 2", (int)th,
              (int)tw);
  const int64_t total = p1 * (int64_t)(th / 2) * (tw / 2);
  if (total == 0) return CVB_OK;
  pool_volume_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(mat, p1, th, tw, out);
  return check_launch("pool_volume");
}

}  // extern "C"
