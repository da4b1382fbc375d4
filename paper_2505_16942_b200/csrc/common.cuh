// Shared device helpers for libcorrvol_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <utility>

#include "../../include/corrvol_b200.h"

namespace cvb {

// ---- host-side status plumbing -------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);  // cudaGetLastError -> status, counts launches
void note_launch();

#define CVB_REQUIRE(cond, ...)          \
  do {                                  \
    if (!(cond)) {                      \
      ::cvb::set_error(__VA_ARGS__);    \
      return CVB_ERR_INVALID;           \
    }                                   \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) -------------------------------------
// The per-iteration kernels (plan -> contraction -> sampler -> next plan) are
// launched with programmatic stream serialization: a kernel may be scheduled
// while its predecessor drains, runs its prologue, and blocks in
// pdl_wait() until the predecessor grid has completed and flushed memory.
// Every kernel calls pdl_wait() before touching global memory that any earlier
// stream work produces or reads, so results are exactly those of plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();    // opt-in: CVB_PDL=1 (every per-iteration edge)
bool pdl_in_phase();   // default (CVB_PDL unset or 2): the tiler -> contraction -> sampler edges

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_if(bool allow, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                        size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = allow ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t s, Args&&... args) {
  return launch_pdl_if(pdl_enabled(), kernel, grid, block, smem, s, std::forward<Args>(args)...);
}
// a launch that depends on the previous kernel of the same iteration
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_phase(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                           size_t smem, cudaStream_t s, Args&&... args) {
  return launch_pdl_if(pdl_enabled() || pdl_in_phase(), kernel, grid, block, smem, s,
                       std::forward<Args>(args)...);
}
static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// image pairs described by a partial-sampler descriptor (0 means 1)
static inline int batch_of(const cvb_partial_desc* d) { return d->batch > 1 ? d->batch : 1; }

// Function attributes live in the current device's context: opt each kernel
// into its dynamic shared memory once per device (call sites keep `done`).
template <typename Kernel>
static inline void ensure_max_smem(std::atomic<uint64_t>& done, Kernel kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
  }
}

// ---- arithmetic ------------------------------------------------------------
// Reference dot arithmetic: fp32, ascending channel, every multiply and add
// rounded separately (no FMA): _ckernels.pyx:27-31 built with -ffp-contract=off.
template <bool STRICT>
__device__ __forceinline__ float mac(float acc, float a, float b) {
  if (STRICT) return __fadd_rn(acc, __fmul_rn(a, b));
  return fmaf(a, b, acc);
}

// ---- index stage -------------------------------------------------------------
// Level position of a level-0 centroid: xl = x/2^l, x0 = floor(xl), fx = xl-x0,
// all in fp64 (sparse.py:251-259; dense.py:214-217; ondemand.py:63-70).
// Division by 2^l equals multiplication by 2^-l exactly (both are the correctly
// rounded value of the same real number).
struct LevelPos {
  long long x0, y0;  // true floors (int64, as the reference)
  double fx, fy;
  bool finite;
};

__device__ __forceinline__ void load_coord(const void* coords, bool f64, int64_t p, double& x,
                                           double& y) {
  if (f64) {
    const double* c = reinterpret_cast<const double*>(coords);
    x = c[2 * p];
    y = c[2 * p + 1];
  } else {
    const float* c = reinterpret_cast<const float*>(coords);
    x = (double)c[2 * p];
    y = (double)c[2 * p + 1];
  }
}

__device__ __forceinline__ LevelPos level_pos(double x, double y, int level) {
  LevelPos r;
  r.finite = isfinite(x) && isfinite(y);
  if (!r.finite) {  // the reference rejects non-finite centroids; keep kernels safe
    x = -1.0e12;
    y = -1.0e12;
  }
  // exact 2^-level from the exponent field (level < 1023)
  const double s = __longlong_as_double((long long)(1023 - level) << 52);
  const double xl = __dmul_rn(x, s), yl = __dmul_rn(y, s);
  const double flx = floor(xl), fly = floor(yl);
  r.x0 = (long long)flx;
  r.y0 = (long long)fly;
  r.fx = __dsub_rn(xl, flx);
  r.fy = __dsub_rn(yl, fly);
  return r;
}

// Window anchor clamped into int32 range without changing in/out-of-bounds
// status of any support cell: a window that lies wholly outside the grid stays
// wholly outside.  Support cells are anchor-r .. anchor+r+1.
__device__ __forceinline__ int clamp_anchor(long long v, int radius, int extent) {
  const long long lo = -(long long)radius - 2;
  const long long hi = (long long)extent + radius + 2;
  return (int)(v < lo ? lo : (v > hi ? hi : v));
}

// Canonical bilinear combination (combine_corners, _pykernels.py:84-96):
// ((v00*w00 + v01*w01) + v10*w10) + v11*w11 in fp64, weights w_ab = wy_a*wx_b.
struct Weights64 {
  double w00, w01, w10, w11;
};
__device__ __forceinline__ Weights64 weights64(double fx, double fy) {
  const double wx1 = fx, wx0 = __dsub_rn(1.0, fx);
  const double wy1 = fy, wy0 = __dsub_rn(1.0, fy);
  Weights64 w;
  w.w00 = __dmul_rn(wy0, wx0);
  w.w01 = __dmul_rn(wy0, wx1);
  w.w10 = __dmul_rn(wy1, wx0);
  w.w11 = __dmul_rn(wy1, wx1);
  return w;
}
__device__ __forceinline__ float combine64(float v00, float v01, float v10, float v11,
                                           const Weights64& w) {
  double acc = __dadd_rn(__dmul_rn((double)v00, w.w00), __dmul_rn((double)v01, w.w01));
  acc = __dadd_rn(acc, __dmul_rn((double)v10, w.w10));
  acc = __dadd_rn(acc, __dmul_rn((double)v11, w.w11));
  return __double2float_rn(acc);
}
struct Weights32 {
  float w00, w01, w10, w11;
};
__device__ __forceinline__ Weights32 weights32(double fx, double fy) {
  const Weights64 w = weights64(fx, fy);
  return Weights32{(float)w.w00, (float)w.w01, (float)w.w10, (float)w.w11};
}
__device__ __forceinline__ float combine32(float v00, float v01, float v10, float v11,
                                           const Weights32& w) {
  return fmaf(v11, w.w11, fmaf(v10, w.w10, fmaf(v01, w.w01, v00 * w.w00)));
}

// Tap value for (dy+r, dx+r) from a (2r+2)^2 patch with row stride `ld`,
// then the optional 1/sqrt(D) fp32 multiply (sparse.py:445-446).
template <bool STRICT>
__device__ __forceinline__ float tap_from_patch(const float* patch, int ld, int j, int i,
                                                const Weights64& w64, const Weights32& w32,
                                                float scale, bool normalize) {
  const float v00 = patch[j * ld + i], v01 = patch[j * ld + i + 1];
  const float v10 = patch[(j + 1) * ld + i], v11 = patch[(j + 1) * ld + i + 1];
  float t = STRICT ? combine64(v00, v01, v10, v11, w64) : combine32(v00, v01, v10, v11, w32);
  if (normalize) t = __fmul_rn(t, scale);
  return t;
}

}  // namespace cvb
