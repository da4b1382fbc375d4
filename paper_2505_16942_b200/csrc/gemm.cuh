// SIMT register-blocked 64x64 dot-product tile (FP32 pipe).
//
// Computes acc[i][j] (i over 4 rows of the thread, j over 4 cols) of a 64x64
// output tile C[r][c] = sum_k A_r[k] * B_c[k].  Each output is owned by one
// thread and accumulated over k in ascending order, so with STRICT the value
// is bit-identical to the reference's sequential fp32 loop
// (_ckernels.pyx:27-31); trailing zero padding adds +-0 and never changes it.
// Operand rows are fetched through row-pointer functors so the same tile
// serves dense GEMM rows, batched block pairs and gathered bbox cells.
#pragma once
#include "common.cuh"

namespace cvb {

constexpr int GT = 64;        // tile edge
constexpr int GKC = 32;       // k chunk
constexpr int GLD = GT + 4;   // smem leading dim (16B-aligned rows)
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_SMEM_FLOATS = 2 * GKC * GLD;

// Loads this thread's two float4 slots of a [64 rows x GKC] chunk into the
// k-major smem tile S[k][row].
__device__ __forceinline__ void load_chunk(float* __restrict__ S, const float* const (&rows)[2],
                                           int k0, int d, bool vec) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int f = tid + GEMM_THREADS * s;
    const int row = f >> 3;
    const int k4 = f & 7;
    const int k = k0 + 4 * k4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* p = rows[s];
    if (p != nullptr) {
      if (vec) {
        if (k < d) v = __ldg(reinterpret_cast<const float4*>(p + k));
      } else {
        if (k + 0 < d) v.x = __ldg(p + k + 0);
        if (k + 1 < d) v.y = __ldg(p + k + 1);
        if (k + 2 < d) v.z = __ldg(p + k + 2);
        if (k + 3 < d) v.w = __ldg(p + k + 3);
      }
    }
    S[(4 * k4 + 0) * GLD + row] = v.x;
    S[(4 * k4 + 1) * GLD + row] = v.y;
    S[(4 * k4 + 2) * GLD + row] = v.z;
    S[(4 * k4 + 3) * GLD + row] = v.w;
  }
}

// rowsA/rowsB: this thread's loader rows (tile rows tid/8 and tid/8+32),
// nullptr for zero rows.  vec: every non-null row is 16B aligned and d%4==0.
template <bool STRICT>
__device__ __forceinline__ void gemm_tile_64x64(const float* const (&rowsA)[2],
                                                const float* const (&rowsB)[2], int d, bool vec,
                                                float* __restrict__ smem, float (&acc)[4][4]) {
  float* As = smem;
  float* Bs = smem + GKC * GLD;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < d; k0 += GKC) {
    load_chunk(As, rowsA, k0, d, vec);
    load_chunk(Bs, rowsB, k0, d, vec);
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GKC; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(As + kk * GLD + ty * 4);
      const float4 b = *reinterpret_cast<const float4*>(Bs + kk * GLD + tx * 4);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = mac<STRICT>(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }
}

}  // namespace cvb
