// KL scoring primitives (similarity.py:101-106):
//   D(x||y) = xlogx[x] - sum_j x_j * log y_j
// exact: fp64 logs, fp64 accumulation (left to right, FMA)
// screen: fp32 logs, fp32 FMA, plus sum_j |x_j * log y_j| for the error bound
#pragma once

#include "common.cuh"

namespace knnd {

// exact fp64 score; x64 may live in shared memory (broadcast reads)
__device__ __forceinline__ double exact_score(const double *x64, const double *__restrict__ lrow,
                                              int d, double xl) {
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= d; j += 4) {
    double l0 = __ldg(lrow + j), l1 = __ldg(lrow + j + 1), l2 = __ldg(lrow + j + 2), l3 = __ldg(lrow + j + 3);
    acc = fma(x64[j], l0, acc);
    acc = fma(x64[j + 1], l1, acc);
    acc = fma(x64[j + 2], l2, acc);
    acc = fma(x64[j + 3], l3, acc);
  }
  for (; j < d; ++j) acc = fma(x64[j], __ldg(lrow + j), acc);
  return xl - acc;
}

}  // namespace knnd
