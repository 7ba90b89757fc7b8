// The local join's fp32, K in 33..64 kernel family (join_impl.cuh; host side in join.cu).
#include "join_impl.cuh"

namespace knnd {

int join_dispatch_f32k2(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                        int64_t m, int32_t *slabs, cudaStream_t st) {
  return dispatch_class_family<FAM_F32K2>(P, i, p, lists, counts, m, slabs, st);
}

}  // namespace knnd

KNND_CHECK_READER(join_f32k2, 7)
