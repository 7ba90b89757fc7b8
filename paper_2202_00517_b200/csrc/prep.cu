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

// column minima / maxima of the log table (the Q23 screen's quantisation ranges)
__device__ __forceinline__ unsigned long long ord_f64(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return b ^ ((unsigned long long)((long long)b >> 63) | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_f64(unsigned long long u) {
  const unsigned long long b = u ^ ((unsigned long long)((long long)~u >> 63) | 0x8000000000000000ull);
  return __longlong_as_double((long long)b);
}

__global__ void col_minmax_kernel(const double *__restrict__ log64, int64_t n, int d,
                                  unsigned long long *__restrict__ mm) {  // [2d]: min, then max (ordered bits)
  const int rows_per = blockDim.x / d;  // column j = thread % d of rows_per rows at a time
  if ((int)threadIdx.x >= rows_per * d) return;
  const int j = threadIdx.x % d;
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t r = (int64_t)blockIdx.x * rows_per + threadIdx.x / d; r < n; r += (int64_t)gridDim.x * rows_per) {
    const unsigned long long u = ord_f64(log64[r * d + j]);
    lo = u < lo ? u : lo;
    hi = u > hi ? u : hi;
  }
  atomicMin(mm + j, lo);
  atomicMax(mm + d + j, hi);
}

// The 23-bit fixed-point log table of the join's Q23 screen (join.cu): per
// column j, h_j = (max - min) / (2^23 - 1), q = round((max - log) / h_j),
// 3 bytes per entry (little endian) at byte 3 j of a row of row_bytes bytes.
// One thread per 4-byte word of the table; its bytes come from the (at most
// two) entries that overlap it.
__global__ void q23_quantize_kernel(const double *__restrict__ log64, int64_t n, int d, int row_bytes,
                                    const unsigned long long *__restrict__ mm, uint32_t *__restrict__ q23,
                                    float *__restrict__ qh) {
  const int wpr = row_bytes >> 2;  // words per row
  const int64_t total = n * wpr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / wpr;
    const int w = (int)(i - r * wpr);
    uint32_t word = 0;
    for (int j = (4 * w) / 3; 3 * j < 4 * w + 4; ++j) {  // entries overlapping bytes [4w, 4w+4)
      if (j >= d) break;
      const double lo = unord_f64(mm[j]), hi = unord_f64(mm[d + j]);
      const double h = (hi - lo) / 8388607.0;
      unsigned q = 0;
      if (h > 0.0) {
        double t = rint((hi - log64[r * d + j]) / h);
        t = t < 0.0 ? 0.0 : (t > 8388607.0 ? 8388607.0 : t);
        q = (unsigned)t;
      }
      const int sh = 8 * (3 * j - 4 * w);  // bit offset of the entry inside this word (may be negative)
      word |= sh >= 0 ? (q << sh) : (q >> (-sh));
    }
    q23[i] = word;
    if (r == 0) {
      for (int j = w; j < row_bytes / 3; j += wpr) {  // row 0's threads also write qh
        float hv = 0.f;
        if (j < d) hv = (float)((unord_f64(mm[d + j]) - unord_f64(mm[j])) / 8388607.0);
        qh[j] = hv;
      }
    }
  }
}

// core.py:97-103 / similarity.py:101-106 — exact scores of ids against anchor x
// (L2: similarity.py:135-140, pts = log64 = the vector rows with |v|^2 appended)
__global__ void batch_scores_kernel(const double *__restrict__ pts, int pstride, const double *__restrict__ log64,
                                    int d64, const double *__restrict__ xlogx, int d, int metric, int64_t x,
                                    const int32_t *__restrict__ ids, int64_t m, double *__restrict__ out) {
  extern __shared__ double xs[];
  for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = pts[x * pstride + j];
  __syncthreads();
  const double xl = xlogx[x];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int y = ids[i];
    out[i] = exact_score_m(xs, log64 + (int64_t)y * d64, d, xl, metric);
  }
}

// similarity.py:126-128 + the L2 screen tables: rows64 = [v, |v|^2] (the squared
// norm computed by the caller with numpy's einsum, as the reference does),
// cand32 = [v - mu, |v - mu|^2, 0...], anchor32 = [2 (v - mu), -1, 0...]: the
// screen's -sum anchor32 * cand32 = |y - mu|^2 - 2 (x - mu).(y - mu) is d2(x, y)
// minus a per-anchor constant.  One warp per row.
__global__ void l2_prepare_kernel(const double *__restrict__ vecs, const double *__restrict__ sq, int64_t n, int d,
                                  int ld, const double *__restrict__ center, float *__restrict__ cand32,
                                  float *__restrict__ anchor32, double *__restrict__ rows64) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    double part = 0.0;
    for (int j = lane; j < ld; j += 32) {
      float c32 = 0.f, a32 = 0.f;
      if (j < d) {
        const double v = vecs[r * d + j];
        const double c = v - center[j];
        rows64[r * (d + 1) + j] = v;
        c32 = (float)c;
        a32 = (float)(2.0 * c);
        part = fma(c, c, part);
      }
      if (j != d) {
        cand32[r * ld + j] = c32;
        anchor32[r * ld + j] = a32;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if (lane == 0) {
      cand32[r * ld + d] = (float)part;
      anchor32[r * ld + d] = -1.f;
      rows64[r * (d + 1) + d] = sq[r];
    }
  }
}

// descent.py:163-174 — each initial row sorted by (score, draw position).
// One warp per row, K <= 64 (two keys per lane above 32).
template <int KPL>
__global__ void sort_rows_kernel(const double *__restrict__ pts, int pstride, const double *__restrict__ log64,
                                 int d64, const double *__restrict__ xlogx, int d, int metric, int K, int64_t lo,
                                 int64_t hi, const int32_t *__restrict__ draws, int32_t *__restrict__ out_ids,
                                 double *__restrict__ out_kl, int staged) {
  // per warp: d doubles (the anchor), then (staged) K rows of d64 doubles at an
  // odd stride: the K candidate rows are copied in row-contiguous 8 B chunks
  // (cp.async) instead of one lane reading one scattered row
  extern __shared__ double sx[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int sd = d64 | 1;
  const size_t per_warp = (size_t)d + (staged ? (size_t)K * sd : 0);
  double *x64 = sx + (size_t)w * per_warp;
  double *stage = x64 + d;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t x = lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + w; x < hi; x += warps) {
    const int64_t xr = x - lo;
    for (int j = lane; j < d; j += 32) x64[j] = pts[x * pstride + j];
    __syncwarp();
    const double xl = xlogx[x];
    KeyD key[KPL];
    int idv[KPL];
    KNND_DCHECK((size_t)(w + 1) * per_warp * 8 <= (size_t)dyn_smem_bytes());
    if (KPL == 1 && staged) {
      const int y = lane < K ? draws[xr * K + lane] : 0;
      KNND_DCHECK(lane >= K || y >= 0);
      idv[0] = lane < K ? y : -1;
      const int nchunk = K * d64;
      int r = lane / d64, j = lane - (lane / d64) * d64;
      const int rq = 32 / d64, rr = 32 - rq * d64;
      for (int c0 = 0; c0 < nchunk; c0 += 32) {
        const int yr = __shfl_sync(FULL, y, r & 31);
        if (c0 + lane < nchunk) cp_async8(stage + r * sd + j, log64 + (int64_t)yr * d64 + j);
        r += rq;
        j += rr;
        if (j >= d64) {
          j -= d64;
          ++r;
        }
      }
      cp_async_wait_all();
      __syncwarp();
      key[0] = KeyD::inf();
      if (lane < K) {  // exact_score_m's arithmetic, from the staged row
        const double *row = stage + lane * sd;
        double acc = 0.0;
        for (int jj = 0; jj < d; ++jj) acc = fma(x64[jj], row[jj], acc);
        key[0] = {finish_score(metric, xl, metric == METRIC_L2 ? row[d] : 0.0, acc), lane};
      }
    } else {
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        int pos = q * 32 + lane;
        key[q] = KeyD::inf();
        idv[q] = -1;
        if (pos < K) {
          int y = draws[xr * K + pos];
          KNND_DCHECK(y >= 0);
          idv[q] = y;
          key[q] = {exact_score_m(x64, log64 + (int64_t)y * d64, d, xl, metric), pos};
        }
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

size_t knnd_kl_q23_workspace_bytes(int32_t d) { return d < 1 ? 0 : align_up((size_t)d * 16, 256); }

int knnd_kl_q23_prepare(const double *log64, int64_t n, int32_t d, int32_t row_bytes, uint8_t *q23, float *qh,
                        void *ws, size_t ws_bytes, void *stream) {
  KNND_CHECK_ARG(log64 && q23 && qh, "knnd_kl_q23_prepare: null pointer");
  KNND_CHECK_ARG(n >= 1 && d >= 1 && d <= 256, "knnd_kl_q23_prepare: bad shape n=%lld d=%d", (long long)n, d);
  KNND_CHECK_ARG(row_bytes >= 3 * d && row_bytes % 16 == 0,
                 "knnd_kl_q23_prepare: row_bytes=%d must be >= 3 d and a multiple of 16", row_bytes);
  if (!ws || ws_bytes < knnd_kl_q23_workspace_bytes(d)) {
    set_error("knnd_kl_q23_prepare: workspace %zu < %zu bytes", ws_bytes, knnd_kl_q23_workspace_bytes(d));
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  unsigned long long *mm = static_cast<unsigned long long *>(ws);
  KNND_CUDA(cudaMemsetAsync(mm, 0xFF, (size_t)d * 8, st));
  KNND_CUDA(cudaMemsetAsync(mm + d, 0x00, (size_t)d * 8, st));
  const int threads = (256 / d) * d > 0 ? (256 / d) * d : d;
  col_minmax_kernel<<<num_sms() * 4, threads, 0, st>>>(log64, n, d, mm);
  KNND_LAUNCHED(1);
  int64_t blocks = (n * (row_bytes / 4) + 255) / 256;
  if (blocks > (int64_t)num_sms() * 32) blocks = (int64_t)num_sms() * 32;
  q23_quantize_kernel<<<(unsigned)blocks, 256, 0, st>>>(log64, n, d, row_bytes, mm,
                                                        reinterpret_cast<uint32_t *>(q23), qh);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_l2_prepare(const double *vectors, const double *sq64, int64_t n, int32_t d, int32_t ld32,
                    const double *center, float *cand32, float *anchor32, double *rows64, void *stream) {
  KNND_CHECK_ARG(vectors && sq64 && center && cand32 && anchor32 && rows64, "knnd_l2_prepare: null pointer");
  KNND_CHECK_ARG(n >= 1 && d >= 1, "knnd_l2_prepare: bad shape n=%lld d=%d", (long long)n, d);
  KNND_CHECK_ARG(ld32 >= d + 1 && ld32 % 4 == 0, "knnd_l2_prepare: ld32=%d must be >= d+1 and a multiple of 4",
                 ld32);
  int64_t blocks = (n + 7) / 8;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  l2_prepare_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(vectors, sq64, n, d, ld32, center, cand32,
                                                                      anchor32, rows64);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

static int batch_scores_impl(const char *who, const double *pts, int pstride, const double *log64, int d64,
                             const double *xlogx, int64_t n, int32_t d, int metric, int64_t x, const int32_t *ids,
                             int64_t m, double *out, void *stream) {
  KNND_CHECK_ARG(pts && log64 && xlogx && out, "%s: null pointer", who);
  KNND_CHECK_ARG(x >= 0 && x < n, "%s: anchor %lld out of range", who, (long long)x);
  KNND_CHECK_ARG(m >= 0, "%s: m < 0", who);
  if (m == 0) return KNND_OK;
  KNND_CHECK_ARG(ids != nullptr, "%s: null ids", who);
  const int threads = 256;
  int64_t blocks = (m + threads - 1) / threads;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  batch_scores_kernel<<<(unsigned)blocks, threads, d * sizeof(double), as_stream(stream)>>>(
      pts, pstride, log64, d64, xlogx, d, metric, x, ids, m, out);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_batch_scores(const double *points, const double *log64, const double *xlogx, int64_t n,
                      int32_t d, int64_t x, const int32_t *ids, int64_t m, double *out, void *stream) {
  return batch_scores_impl("knnd_batch_scores", points, d, log64, d, xlogx, n, d, METRIC_KL, x, ids, m, out, stream);
}

int knnd_l2_batch_scores(const double *rows64, const double *sq64, int64_t n, int32_t d, int64_t x,
                         const int32_t *ids, int64_t m, double *out, void *stream) {
  return batch_scores_impl("knnd_l2_batch_scores", rows64, d + 1, rows64, d + 1, sq64, n, d, METRIC_L2, x, ids, m,
                           out, stream);
}

static int sort_rows_impl(const char *who, const double *pts, int pstride, const double *log64, int d64,
                          const double *xlogx, int64_t n, int32_t d, int metric, int32_t k, int64_t row_lo,
                          int64_t row_hi, const int32_t *draws, int32_t *out_ids, double *out_kl, void *stream) {
  KNND_CHECK_ARG(pts && log64 && xlogx && draws && out_ids, "%s: null pointer", who);
  KNND_CHECK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= n, "%s: bad row range", who);
  if (k < 1 || k > 64) {
    set_error("%s: K=%d unsupported (1..64)", who, k);
    return KNND_EUNSUPPORTED;
  }
  if (row_hi == row_lo) return KNND_OK;
  const int threads = 256, wpb = threads / 32;
  int64_t rows = row_hi - row_lo;
  int64_t blocks = (rows + wpb - 1) / wpb;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  const size_t staged_smem = (size_t)wpb * (d + (size_t)k * (d64 | 1)) * sizeof(double);
  const int staged = (k <= 32 && staged_smem <= 160 * 1024) ? 1 : 0;
  size_t smem = staged ? staged_smem : (size_t)wpb * d * sizeof(double);
  if (k <= 32) {
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void *)sort_rows_kernel<1>, 256, smem, &per_sm)) return rc;
    sort_rows_kernel<1><<<(unsigned)blocks, threads, smem, as_stream(stream)>>>(
        pts, pstride, log64, d64, xlogx, d, metric, k, row_lo, row_hi, draws, out_ids, out_kl, staged);
  } else {
    sort_rows_kernel<2><<<(unsigned)blocks, threads, smem, as_stream(stream)>>>(
        pts, pstride, log64, d64, xlogx, d, metric, k, row_lo, row_hi, draws, out_ids, out_kl, staged);
  }
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_sort_rows(const double *points, const double *log64, const double *xlogx, int64_t n,
                   int32_t d, int32_t k, int64_t row_lo, int64_t row_hi, const int32_t *draws,
                   int32_t *out_ids, double *out_kl, void *stream) {
  return sort_rows_impl("knnd_sort_rows", points, d, log64, d, xlogx, n, d, METRIC_KL, k, row_lo, row_hi, draws,
                        out_ids, out_kl, stream);
}

int knnd_l2_sort_rows(const double *rows64, const double *sq64, int64_t n, int32_t d, int32_t k, int64_t row_lo,
                      int64_t row_hi, const int32_t *draws, int32_t *out_ids, double *out_d2, void *stream) {
  return sort_rows_impl("knnd_l2_sort_rows", rows64, d + 1, rows64, d + 1, sq64, n, d, METRIC_L2, k, row_lo,
                        row_hi, draws, out_ids, out_d2, stream);
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

KNND_CHECK_READER(prep, 4)
