// Cascaded-init flow resample (flowio.py:151-199).
//
// The step before the lookup in SEA-RAFT's cascade: a quarter-resolution
// pass's flow is resampled onto the full-resolution pass's eighth-resolution
// grid.  A different sampling convention from the cost lookup: output pixel
// centres map to input pixel centres, src = (out + 0.5) / scale - 0.5, with
// edge CLAMPING (not zero padding), and magnitudes are multiplied by scale.
// One thread per output pixel (both vector components); every operation is the
// reference's fp64 expression with explicit rounding (no contraction), so the
// result is bit-identical to numpy's.
#include "common.cuh"

namespace cvb {

__global__ void __launch_bounds__(256) resample_flow_kernel(const float* __restrict__ in, int h,
                                                            int w, double scale,
                                                            float* __restrict__ out, int oh,
                                                            int ow) {
  const int64_t n = (int64_t)oh * ow;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int oy = (int)(i / ow), ox = (int)(i % ow);
    double sy = __dsub_rn(__ddiv_rn(__dadd_rn((double)oy, 0.5), scale), 0.5);
    double sx = __dsub_rn(__ddiv_rn(__dadd_rn((double)ox, 0.5), scale), 0.5);
    sy = fmin(fmax(sy, 0.0), (double)h - 1.0);
    sx = fmin(fmax(sx, 0.0), (double)w - 1.0);
    const int y0 = (int)floor(sy), x0 = (int)floor(sx);
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    const double fy = __dsub_rn(sy, (double)y0), fx = __dsub_rn(sx, (double)x0);
    const double wy0 = __dsub_rn(1.0, fy), wx0 = __dsub_rn(1.0, fx);
    const double w00 = __dmul_rn(wy0, wx0), w01 = __dmul_rn(wy0, fx);
    const double w10 = __dmul_rn(fy, wx0), w11 = __dmul_rn(fy, fx);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double v00 = in[((int64_t)y0 * w + x0) * 2 + c], v01 = in[((int64_t)y0 * w + x1) * 2 + c];
      const double v10 = in[((int64_t)y1 * w + x0) * 2 + c], v11 = in[((int64_t)y1 * w + x1) * 2 + c];
      double acc = __dadd_rn(__dmul_rn(v00, w00), __dmul_rn(v01, w01));
      acc = __dadd_rn(acc, __dmul_rn(v10, w10));
      acc = __dadd_rn(acc, __dmul_rn(v11, w11));
      out[i * 2 + c] = __double2float_rn(__dmul_rn(acc, scale));
    }
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_resample_dims(int32_t h, int32_t w, double scale, int32_t* out_h, int32_t* out_w) {
  CVB_REQUIRE(out_h && out_w, "resample_dims: null pointer");
  CVB_REQUIRE(isfinite(scale) && scale > 0.0,
              "scale must be a positive finite number, got %g", scale);
  const double oh = floor((double)h * scale + 0.5), ow = floor((double)w * scale + 0.5);
  CVB_REQUIRE(oh >= 1.0 && ow >= 1.0, "scale %g collapses %dx%d to %.0fx%.0f", scale, (int)h,
              (int)w, oh, ow);
  CVB_REQUIRE(oh < 2147483647.0 && ow < 2147483647.0, "resampled dims overflow");
  *out_h = (int32_t)oh;
  *out_w = (int32_t)ow;
  return CVB_OK;
}

int cvb_resample_flow(const float* in, int32_t h, int32_t w, double scale, float* out,
                      int32_t out_h, int32_t out_w, void* stream) {
  CVB_REQUIRE(in && out, "resample_flow: null pointer");
  CVB_REQUIRE(h >= 1 && w >= 1, "resample_flow: empty field");
  int32_t eh = 0, ew = 0;
  const int st = cvb_resample_dims(h, w, scale, &eh, &ew);
  if (st != CVB_OK) return st;
  CVB_REQUIRE(eh == out_h && ew == out_w, "resample_flow: output must be %dx%d", (int)eh, (int)ew);
  const int64_t n = (int64_t)out_h * out_w;
  int64_t g = ceil_div(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  resample_flow_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(in, h, w, scale, out, out_h,
                                                                    out_w);
  return check_launch("resample_flow");
}

}  // extern "C"
