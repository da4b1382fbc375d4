// Index stage exports, dense-variant lookup and on-demand variant.
//
// Index stage: _level_centroid_floors (sparse.py:251-259) and the support
// validity used by _corner_patches (dense.py:163-185), lookup_on_demand
// (ondemand.py:71-83) and _gather_patches (sparse.py:349-375).
//
// Dense lookup: per query, the (2r+2)^2 corner patch of row p of the level
// volume, zero outside the UNPADDED grid, combined into (2r+1)^2 taps.
//
// On-demand: per query, each in-bounds support cell is one fresh length-D dot
// (the reference evaluates 4 corner dots per tap; every corner value equals
// the unique cell's dot bit for bit, so evaluating each cell once yields the
// identical result).  One warp per query: F1 row staged in shared memory
// (broadcast reads), F2 rows streamed through L1/L2 with 16-byte loads.
#include "common.cuh"

namespace cvb {

__global__ void floors_kernel(const void* __restrict__ coords, bool f64, int64_t p, int level,
                              long long* __restrict__ x0, long long* __restrict__ y0,
                              double* __restrict__ fx, double* __restrict__ fy) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p) return;
  double x, y;
  load_coord(coords, f64, i, x, y);
  const LevelPos q = level_pos(x, y, level);
  x0[i] = q.x0;
  y0[i] = q.y0;
  fx[i] = q.fx;
  fy[i] = q.fy;
}

__global__ void support_valid_kernel(const void* __restrict__ coords, bool f64, int64_t p,
                                     int level, int radius, int gh, int gw,
                                     uint8_t* __restrict__ out) {
  const int S = 2 * radius + 2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p * S * S) return;
  const int64_t q = i / (S * S);
  const int c = (int)(i % (S * S));
  double x, y;
  load_coord(coords, f64, q, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const long long ty = lp.y0 - radius + c / S, tx = lp.x0 - radius + c % S;
  out[i] = (ty >= 0 && ty < gh && tx >= 0 && tx < gw) ? 1 : 0;
}

constexpr int LK_WARPS = 4;

template <bool STRICT>
__global__ void __launch_bounds__(LK_WARPS * 32)
    lookup_dense_kernel(const float* __restrict__ mat, int64_t p1, int th, int tw,
                        const void* __restrict__ coords, bool f64, int level, int levels,
                        int radius, float scale, bool normalize, float* __restrict__ out) {
  extern __shared__ float lk_smem[];
  const int S = 2 * radius + 2, K = 2 * radius + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * LK_WARPS + warp;
  if (p >= p1) return;
  float* patch = lk_smem + warp * S * S;
  double x, y;
  load_coord(coords, f64, p, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const int ax = clamp_anchor(lp.x0, radius, tw), ay = clamp_anchor(lp.y0, radius, th);
  const float* row = mat + p * (int64_t)th * tw;
  for (int c = lane; c < S * S; c += 32) {
    const int ty = ay - radius + c / S, tx = ax - radius + c % S;
    float v = 0.f;
    if (ty >= 0 && ty < th && tx >= 0 && tx < tw) v = __ldg(row + (int64_t)ty * tw + tx);
    patch[c] = v;
  }
  __syncwarp();
  const Weights64 w64 = weights64(lp.fx, lp.fy);
  const Weights32 w32 = weights32(lp.fx, lp.fy);
  float* o = out + (p * levels + level) * (int64_t)(K * K);
  for (int t = lane; t < K * K; t += 32)
    o[t] = tap_from_patch<STRICT>(patch, S, t / K, t % K, w64, w32, scale, normalize);
}

template <bool STRICT>
__global__ void __launch_bounds__(LK_WARPS * 32)
    lookup_on_demand_kernel(const float* __restrict__ f1, int64_t p1, int d,
                            const float* __restrict__ f2l, int th, int tw,
                            const void* __restrict__ coords, bool f64, int level, int levels,
                            int radius, float scale, bool normalize, float* __restrict__ out,
                            unsigned long long* __restrict__ counters, bool vec) {
  extern __shared__ __align__(16) float od_smem[];
  const int S = 2 * radius + 2, K = 2 * radius + 1;
  const int dpad = (d + 3) & ~3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * LK_WARPS + warp;
  if (p >= p1) return;
  float* frow = od_smem + warp * (dpad + S * S);
  float* patch = frow + dpad;
  for (int k = lane; k < d; k += 32) frow[k] = __ldg(f1 + p * d + k);
  __syncwarp();
  double x, y;
  load_coord(coords, f64, p, x, y);
  const LevelPos lp = level_pos(x, y, level);
  const int ax = clamp_anchor(lp.x0, radius, tw), ay = clamp_anchor(lp.y0, radius, th);
  unsigned long long n_exec = 0, n_model = 0;
  for (int c = lane; c < S * S; c += 32) {
    const int j = c / S, i = c % S;
    const int ty = ay - radius + j, tx = ax - radius + i;
    float acc = 0.f;
    if (ty >= 0 && ty < th && tx >= 0 && tx < tw) {
      const float* g = f2l + ((int64_t)ty * tw + tx) * d;
      if (vec) {
        for (int k = 0; k < d; k += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(g + k));
          const float4 a = *reinterpret_cast<const float4*>(frow + k);
          acc = mac<STRICT>(acc, a.x, b.x);
          acc = mac<STRICT>(acc, a.y, b.y);
          acc = mac<STRICT>(acc, a.z, b.z);
          acc = mac<STRICT>(acc, a.w, b.w);
        }
      } else {
        for (int k = 0; k < d; ++k) acc = mac<STRICT>(acc, frow[k], __ldg(g + k));
      }
      n_exec += 1;
      // taps using support cell (j, i): 1 at the border rows/cols, else 2 per axis
      n_model += (unsigned long long)((j >= 1) + (j <= K - 1)) * ((i >= 1) + (i <= K - 1));
    }
    patch[c] = acc;
  }
  __syncwarp();
  if (counters != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n_exec += __shfl_xor_sync(0xffffffffu, n_exec, o);
      n_model += __shfl_xor_sync(0xffffffffu, n_model, o);
    }
    if (lane == 0) {
      atomicAdd(counters + 0, n_exec);
      atomicAdd(counters + 1, n_model);
    }
  }
  const Weights64 w64 = weights64(lp.fx, lp.fy);
  const Weights32 w32 = weights32(lp.fx, lp.fy);
  float* o = out + (p * levels + level) * (int64_t)(K * K);
  for (int t = lane; t < K * K; t += 32)
    o[t] = tap_from_patch<STRICT>(patch, S, t / K, t % K, w64, w32, scale, normalize);
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cvb_level_floors(const void* coords, int64_t p, int32_t level, int32_t flags, int64_t* x0,
                     int64_t* y0, double* fx, double* fy, void* stream) {
  CVB_REQUIRE(level >= 0 && level < 62, "bad level %d", (int)level);
  if (p == 0) return CVB_OK;
  CVB_REQUIRE(coords && x0 && y0 && fx && fy, "level_floors: null pointer");
  floors_kernel<<<(unsigned)ceil_div(p, 256), 256, 0, as_stream(stream)>>>(
      coords, flags & CVB_COORDS_F64, p, level, reinterpret_cast<long long*>(x0),
      reinterpret_cast<long long*>(y0), fx, fy);
  return check_launch("level_floors");
}

int cvb_support_valid(const void* coords, int64_t p, int32_t level, int32_t radius, int32_t gh,
                      int32_t gw, int32_t flags, uint8_t* out, void* stream) {
  CVB_REQUIRE(radius >= 0 && radius <= 64 && level >= 0, "bad radius/level");
  if (p == 0) return CVB_OK;
  CVB_REQUIRE(coords && out, "support_valid: null pointer");
  const int64_t S = 2 * radius + 2;
  support_valid_kernel<<<(unsigned)ceil_div(p * S * S, 256), 256, 0, as_stream(stream)>>>(
      coords, flags & CVB_COORDS_F64, p, level, radius, gh, gw, out);
  return check_launch("support_valid");
}

int cvb_lookup_dense(const float* level_mat, int32_t h1, int32_t w1, int32_t th, int32_t tw,
                     const void* coords, int32_t level, int32_t levels, int32_t radius,
                     float scale, float* out, int32_t flags, void* stream) {
  CVB_REQUIRE(radius >= 0 && radius <= 30, "radius must be in [0, 30]");
  CVB_REQUIRE(level >= 0 && level < levels, "bad level");
  CVB_REQUIRE(th >= 1 && tw >= 1, "empty target level");
  const int64_t p1 = (int64_t)h1 * w1;
  if (p1 == 0) return CVB_OK;
  CVB_REQUIRE(level_mat && coords && out, "lookup_dense: null pointer");
  const int S = 2 * radius + 2;
  const size_t smem = (size_t)LK_WARPS * S * S * sizeof(float);
  const unsigned grid = (unsigned)ceil_div(p1, LK_WARPS);
  const bool f64 = flags & CVB_COORDS_F64;
  const bool norm = scale != 1.0f;
  if (flags & CVB_STRICT)
    lookup_dense_kernel<true><<<grid, LK_WARPS * 32, smem, as_stream(stream)>>>(
        level_mat, p1, th, tw, coords, f64, level, levels, radius, scale, norm, out);
  else
    lookup_dense_kernel<false><<<grid, LK_WARPS * 32, smem, as_stream(stream)>>>(
        level_mat, p1, th, tw, coords, f64, level, levels, radius, scale, norm, out);
  return check_launch("lookup_dense");
}

int cvb_lookup_on_demand(const float* f1, int32_t h1, int32_t w1, int32_t d, const float* f2l,
                         int32_t th, int32_t tw, const void* coords, int32_t level,
                         int32_t levels, int32_t radius, float scale, float* out,
                         unsigned long long* counters, int32_t flags, void* stream) {
  CVB_REQUIRE(radius >= 0 && radius <= 30, "radius must be in [0, 30]");
  CVB_REQUIRE(level >= 0 && level < levels, "bad level");
  CVB_REQUIRE(d >= 1 && d <= 8192, "feature dims must be in [1, 8192]");
  CVB_REQUIRE(th >= 1 && tw >= 1, "empty target level");
  const int64_t p1 = (int64_t)h1 * w1;
  if (p1 == 0) return CVB_OK;
  CVB_REQUIRE(f1 && f2l && coords && out, "lookup_on_demand: null pointer");
  const int S = 2 * radius + 2;
  const int dpad = (d + 3) & ~3;
  const size_t smem = (size_t)LK_WARPS * (dpad + S * S) * sizeof(float);
  CVB_REQUIRE(smem <= 200 * 1024, "lookup_on_demand: D/radius too large");
  const bool vec = (d % 4 == 0) && (((uintptr_t)f2l & 15) == 0);
  const unsigned grid = (unsigned)ceil_div(p1, LK_WARPS);
  const bool f64 = flags & CVB_COORDS_F64;
  const bool norm = scale != 1.0f;
  cudaStream_t s = as_stream(stream);
  if (flags & CVB_STRICT) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(lookup_on_demand_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lookup_on_demand_kernel<true><<<grid, LK_WARPS * 32, smem, s>>>(
        f1, p1, d, f2l, th, tw, coords, f64, level, levels, radius, scale, norm, out, counters,
        vec);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(lookup_on_demand_kernel<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lookup_on_demand_kernel<false><<<grid, LK_WARPS * 32, smem, s>>>(
        f1, p1, d, f2l, th, tw, coords, f64, level, levels, radius, scale, norm, out, counters,
        vec);
  }
  return check_launch("lookup_on_demand");
}

}  // extern "C"
