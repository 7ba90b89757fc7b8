// Scoring primitives.  Both metrics are "anchor constant + row extra - scale *
// sum_j x_j * row_j", so one screen and one fp64 rescoring serve both:
//   KL  (similarity.py:101-106)  D(x||y) = xlogx[x] - sum_j x_j * log y_j
//        fp64 table: log rows (d);            anchor constant: xlogx[x]
//   L2  (similarity.py:135-140)  d2(x,y) = max(sq[x] + sq[y] - 2 * sum_j y_j x_j, 0)
//        fp64 table: vector rows + |y|^2 (d+1); anchor constant: sq[x]
// exact: fp64, left-to-right FMA accumulation of the dot product
// screen: fp32 over padded rows (join.cu), with a rigorous error band
#pragma once

#include "common.cuh"

namespace knnd {

constexpr int METRIC_KL = 0, METRIC_L2 = 1;

// the metric's fp64 value from the anchor constant, the row extra and the dot
__device__ __forceinline__ double finish_score(int metric, double xl, double extra, double acc) {
  if (metric == METRIC_L2) return fmax((xl + extra) - 2.0 * acc, 0.0);
  return xl - acc;
}

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

// either metric; lrow has d (KL) or d + 1 (L2: the squared norm last) entries
__device__ __forceinline__ double exact_score_m(const double *x64, const double *__restrict__ lrow, int d,
                                                double xl, int metric) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) acc = fma(x64[j], __ldg(lrow + j), acc);
  return finish_score(metric, xl, metric == METRIC_L2 ? __ldg(lrow + d) : 0.0, acc);
}

}  // namespace knnd
