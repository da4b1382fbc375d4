/*
 * TEST INFRASTRUCTURE ONLY — part of the CPU oracle (oracle/), never linked
 * into or called by the product path.
 *
 * Sequential fp32 dot products in ascending channel order with every multiply
 * and add rounded separately, restating the reference kernel lane
 * (corrvol _ckernels.pyx:27-31 / _pykernels.py:18-58, built with
 * -ffp-contract=off, setup.py:19).  Build with -ffp-contract=off.
 * Pairs are independent, so OpenMP over pairs leaves each dot unchanged.
 */
#include <stdint.h>

void oracle_pair_dots(const float* a, const float* b, const int64_t* ia, const int64_t* ib,
                      int64_t n, int32_t d, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    const float* x = a + ia[k] * (int64_t)d;
    const float* y = b + ib[k] * (int64_t)d;
    float acc = 0.0f;
    for (int32_t c = 0; c < d; ++c) {
      const float p = x[c] * y[c];
      acc = acc + p;
    }
    out[k] = acc;
  }
}
