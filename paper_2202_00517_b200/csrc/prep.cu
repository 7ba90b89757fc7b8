// Per-run precompute (KlRankingSystem.__init__), the batch_scores operator,
// the initial row sort (K6) and the friend-clustering-rate count (K5).
#include "common.cuh"
#include "score.cuh"

namespace knnd {

// ---------------------------------------------------------------------------
// similarity.py:87-95 — log table (fp64 + padded fp32 copy) and row entropy.
// One warp per point row.
__global__ void kl_prepare_kernel(const double *__restrict__ pts, int64_t n, int d, int ld,
                                  float *__restrict__ log32, double *__restrict__ log64,
                                  double *__restrict__ xlogx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    double part = 0.0;
    for (int j = lane; j < ld; j += 32) {
      float l32 = 0.f;
      if (j < d) {
        double x = pts[r * d + j];
        double l = log(x);
        log64[r * d + j] = l;
        l32 = (float)l;
        part = fma(x, l, part);
      }
      log32[r * ld + j] = l32;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if (lane == 0) xlogx[r] = part;
  }
}

// core.py:97-103 / similarity.py:101-106 — exact scores of ids against anchor x
__global__ void batch_scores_kernel(const double *__restrict__ pts, const double *__restrict__ log64,
                                    const double *__restrict__ xlogx, int d, int64_t x,
                                    const int32_t *__restrict__ ids, int64_t m, double *__restrict__ out) {
  extern __shared__ double xs[];
  for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = pts[x * d + j];
  __syncthreads();
  const double xl = xlogx[x];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int y = ids[i];
    out[i] = exact_score(xs, log64 + (int64_t)y * d, d, xl);
  }
}

// descent.py:163-174 — each initial row sorted by (score, draw position).
// One warp per row, K <= 64 (two keys per lane above 32).
template <int KPL>
__global__ void sort_rows_kernel(const double *__restrict__ pts, const double *__restrict__ log64,
                                 const double *__restrict__ xlogx, int d, int K, int64_t lo, int64_t hi,
                                 const int32_t *__restrict__ draws, int32_t *__restrict__ out_ids,
                                 double *__restrict__ out_kl) {
  extern __shared__ double sx[];  // per warp: d doubles
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  double *x64 = sx + (size_t)w * d;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t x = lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + w; x < hi; x += warps) {
    const int64_t xr = x - lo;
    for (int j = lane; j < d; j += 32) x64[j] = pts[x * d + j];
    __syncwarp();
    const double xl = xlogx[x];
    KeyD key[KPL];
    int idv[KPL];
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      int pos = q * 32 + lane;
      key[q] = KeyD::inf();
      idv[q] = -1;
      if (pos < K) {
        int y = draws[xr * K + pos];
        idv[q] = y;
        key[q] = {exact_score(x64, log64 + (int64_t)y * d, d, xl), pos};
      }
    }
    // sort keys; the tie field is the draw position (stable argsort)
    key[0] = warp_sort32(key[0], lane);
    if (KPL == 2) {
      key[KPL - 1] = warp_sort32(key[KPL - 1], lane);
      KeyD r = key[KPL - 1].shfl(31 - lane);
      KeyD lo_ = kmin(key[0], r), hi_ = kmax(key[0], r);
      key[0] = warp_merge32(lo_, lane);
      key[KPL - 1] = warp_merge32(hi_, lane);
    }
    // gather ids by sorted position
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      int i = q * 32 + lane;
      int pos = key[q].id;
      // fetch id at draw position `pos` (held by lane pos%32, register pos/32)
      int src = pos & 31;
      int y0 = __shfl_sync(FULL, idv[0], src);
      int y = y0;
      if (KPL == 2) {
        int y1 = __shfl_sync(FULL, idv[KPL - 1], src);
        if (pos >= 32) y = y1;
      }
      if (i < K) {
        out_ids[xr * K + i] = y;
        if (out_kl) out_kl[xr * K + i] = key[q].s;
      }
    }
    __syncwarp();
  }
}

// descent.py:317-338 — count of adjacent sampled friend pairs
__global__ void fcc_kernel(const int32_t *__restrict__ F, int K, const int32_t *__restrict__ xs,
                           const int32_t *__restrict__ is, const int32_t *__restrict__ js, int S,
                           int32_t *__restrict__ out_count) {
  int local = 0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    int64_t x = xs[s];
    int y = F[x * K + is[s]];
    int z = F[x * K + js[s]];
    bool adj = false;
    const int32_t *fz = F + (int64_t)z * K;
    const int32_t *fy = F + (int64_t)y * K;
    for (int t = 0; t < K; ++t) adj |= (fz[t] == y) | (fy[t] == z);
    local += adj ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(FULL, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(out_count, local);
}

}  // namespace knnd

using namespace knnd;

extern "C" {

int knnd_kl_prepare(const double *points, int64_t n, int32_t d, int32_t ld32, float *log32,
                    double *log64, double *xlogx, void *stream) {
  KNND_CHECK_ARG(points && log32 && log64 && xlogx, "knnd_kl_prepare: null pointer");
  KNND_CHECK_ARG(n >= 1 && d >= 1, "knnd_kl_prepare: bad shape n=%lld d=%d", (long long)n, d);
  KNND_CHECK_ARG(ld32 >= d && ld32 % 4 == 0, "knnd_kl_prepare: ld32=%d must be >= d and a multiple of 4", ld32);
  const int threads = 256;
  int64_t blocks = (n + 7) / 8;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  kl_prepare_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(points, n, d, ld32, log32, log64, xlogx);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_batch_scores(const double *points, const double *log64, const double *xlogx, int64_t n,
                      int32_t d, int64_t x, const int32_t *ids, int64_t m, double *out, void *stream) {
  KNND_CHECK_ARG(points && log64 && xlogx && out, "knnd_batch_scores: null pointer");
  KNND_CHECK_ARG(x >= 0 && x < n, "knnd_batch_scores: anchor %lld out of range", (long long)x);
  KNND_CHECK_ARG(m >= 0, "knnd_batch_scores: m < 0");
  if (m == 0) return KNND_OK;
  KNND_CHECK_ARG(ids != nullptr, "knnd_batch_scores: null ids");
  const int threads = 256;
  int64_t blocks = (m + threads - 1) / threads;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  batch_scores_kernel<<<(unsigned)blocks, threads, d * sizeof(double), as_stream(stream)>>>(
      points, log64, xlogx, d, x, ids, m, out);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_sort_rows(const double *points, const double *log64, const double *xlogx, int64_t n,
                   int32_t d, int32_t k, int64_t row_lo, int64_t row_hi, const int32_t *draws,
                   int32_t *out_ids, double *out_kl, void *stream) {
  KNND_CHECK_ARG(points && log64 && xlogx && draws && out_ids, "knnd_sort_rows: null pointer");
  KNND_CHECK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= n, "knnd_sort_rows: bad row range");
  if (k < 1 || k > 64) {
    set_error("knnd_sort_rows: K=%d unsupported (1..64)", k);
    return KNND_EUNSUPPORTED;
  }
  if (row_hi == row_lo) return KNND_OK;
  const int threads = 256, wpb = threads / 32;
  int64_t rows = row_hi - row_lo;
  int64_t blocks = (rows + wpb - 1) / wpb;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  size_t smem = (size_t)wpb * d * sizeof(double);
  if (k <= 32)
    sort_rows_kernel<1><<<(unsigned)blocks, threads, smem, as_stream(stream)>>>(
        points, log64, xlogx, d, k, row_lo, row_hi, draws, out_ids, out_kl);
  else
    sort_rows_kernel<2><<<(unsigned)blocks, threads, smem, as_stream(stream)>>>(
        points, log64, xlogx, d, k, row_lo, row_hi, draws, out_ids, out_kl);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_fcc(const int32_t *friends, int64_t n, int32_t k, const int32_t *xs, const int32_t *is,
             const int32_t *js, int32_t s_count, int32_t *out_count, void *stream) {
  KNND_CHECK_ARG(friends && xs && is && js && out_count, "knnd_fcc: null pointer");
  KNND_CHECK_ARG(n >= 1 && k >= 2 && s_count >= 1, "knnd_fcc: bad sizes n=%lld k=%d S=%d", (long long)n, k, s_count);
  cudaStream_t st = as_stream(stream);
  KNND_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int32_t), st));
  const int threads = 256;
  int blocks = (s_count + threads - 1) / threads;
  if (blocks > num_sms() * 4) blocks = num_sms() * 4;
  fcc_kernel<<<blocks, threads, 0, st>>>(friends, k, xs, is, js, s_count, out_count);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

}  // extern "C"
