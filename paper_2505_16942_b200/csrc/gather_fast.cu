// (5) Gather / bilinear sampler, fast-arithmetic r=4 path (RAFT / SEA-RAFT):
// the standalone sampler kernel.  The per-query-group body (design notes) is
// gfast::sample_group in gather_fast.cuh, shared with the sampler warps of the
// fused warm contraction (partial_tc.cu).
#include <stdlib.h>

#include "gather_fast.cuh"

namespace cvb {
namespace gfast {

// two query groups (a quarter tile) per CTA, 8 CTAs per SM: the same 16
// resident warps per SM as whole-tile CTAs (registers bind at 126), but small
// CTAs retire and refill independently (-6% sampler time at C4)
constexpr int WARPS = 2;
constexpr int CTAS_PER_TILE = (TQ / QG) / WARPS;  // 8 query groups per tile

__global__ void __launch_bounds__(WARPS * 32, 16 / WARPS) gather_fast_kernel(PartialParams P, float* out,
                                                                    int level0, int nlev) {
  extern __shared__ __align__(16) uint8_t g_smem[];
  WarpStage* stage = reinterpret_cast<WarpStage*>(g_smem);
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = P.tile0 + blockIdx.x / CTAS_PER_TILE;
  const int grp = (int)(blockIdx.x % CTAS_PER_TILE) * WARPS + warp;
  const int li = lane >> 3;
  const int status = li < nlev ? P.meta[(tile * P.levels + level0 + li) * CVB_META_INTS + 4] : ST_EMPTY;
  sample_group<true>(P, tile, grp, status, out, level0, nlev, stage[warp], lane);
}

}  // namespace gfast

int launch_gather_fast_r4(const PartialParams& P, float* out, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  const int smem = (int)(gfast::WARPS * sizeof(gfast::WarpStage));
  ensure_max_smem(attr, gfast::gather_fast_kernel, smem);
  // Shared-memory carveout 65%: the taps re-read each cache sector ~3x through
  // L1, so L1 capacity matters more than the last CTA slot per SM (measured:
  // 65% is 1-2% faster than the default 200 KB carveout; 100% halves the
  // speed).  CVB_GF_CARVEOUT overrides (percent; -1 = driver default).
  static std::atomic<uint64_t> carved{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(carved.load() & bit)) {
    const char* e = getenv("CVB_GF_CARVEOUT");
    const int carve = e ? atoi(e) : 65;
    if (carve >= 0)
      cudaFuncSetAttribute(gfast::gather_fast_kernel,
                           cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    carved.fetch_or(bit);
  }
  for (int l0 = 0; l0 < P.levels; l0 += gfast::MAXL) {
    const int nl = min(gfast::MAXL, P.levels - l0);
    launch_pdl(gfast::gather_fast_kernel, dim3((unsigned)(gfast::CTAS_PER_TILE * P.ntile)), dim3(gfast::WARPS * 32), smem,
               s, P, out, l0, nl);
    const int st = check_launch("partial_gather_fast");
    if (st != CVB_OK) return st;
  }
  return CVB_OK;
}

}  // namespace cvb
