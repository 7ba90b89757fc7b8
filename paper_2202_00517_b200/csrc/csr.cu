// K1 — co-friend CSR (the transpose of the friends digraph) for the targets a
// rank owns; replaces _transpose_csr (descent.py:151-160).
//
//   count   : one thread per source row, atomic in-degree histogram (int32)
//   reduce  : per 4096-tile sums + global max in-degree
//   partials: exclusive scan of tile sums (single block)
//   apply   : per-tile exclusive scan -> indptr (int64) and fill cursor
//   fill    : one thread per source row, atomic cursor -> indices[pos] = source
//
// Segment order is unspecified (the local join is order-independent: it
// dedups through a hash table and ranks by the (score, id) total order).
#include "common.cuh"

namespace knnd {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void csr_count_kernel(const int32_t *__restrict__ F, int64_t n, int K, int64_t lo, int64_t m,
                                 int32_t *__restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * K; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = (int64_t)__ldg(F + e) - lo;
    if ((uint64_t)t < (uint64_t)m) atomicAdd(cnt + t, 1);
  }
}

__device__ __forceinline__ int block_excl_scan(int v, int *warp_sums, int &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) warp_sums[w] = inc;
  __syncthreads();
  if (w == 0) {
    int s = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0;
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(FULL, si, o);
      if (lane >= o) si += u;
    }
    warp_sums[lane] = si - s;  // exclusive
    if (lane == 31) warp_sums[32] = si;
  }
  __syncthreads();
  int r = warp_sums[w] + inc - v;
  total = warp_sums[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) csr_reduce_kernel(const int32_t *__restrict__ cnt, int64_t m,
                                                                  int64_t *__restrict__ tile_sums,
                                                                  int32_t *__restrict__ max_out) {
  __shared__ int red[33];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int s = 0, mx = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < m) {
      int c = cnt[idx];
      s += c;
      mx = max(mx, c);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(FULL, s, o);
    mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  if ((threadIdx.x & 31) == 0 && max_out) atomicMax(max_out, mx);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) csr_partials_kernel(int64_t *__restrict__ tile_sums, int64_t ntiles,
                                                                    int64_t *__restrict__ indptr, int64_t m) {
  __shared__ long long ws[33];
  long long carry = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = 0; b < ntiles; b += SCAN_THREADS) {
    int64_t i = b + threadIdx.x;
    long long v = i < ntiles ? tile_sums[i] : 0;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long u = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      long long s = ws[lane], si = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long u = __shfl_up_sync(FULL, si, o);
        if (lane >= o) si += u;
      }
      ws[lane] = si - s;
      if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    if (i < ntiles) tile_sums[i] = carry + ws[w] + inc - v;
    carry += ws[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) indptr[m] = carry;
}

__global__ void __launch_bounds__(SCAN_THREADS) csr_apply_kernel(int32_t *__restrict__ cnt_cursor, int64_t m,
                                                                 const int64_t *__restrict__ tile_offsets,
                                                                 int64_t *__restrict__ indptr) {
  __shared__ int ws[33];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < m) ? cnt_cursor[base + i] : 0;
    s += v[i];
  }
  int total;
  int ex = block_excl_scan(s, ws, total);
  const long long off = tile_offsets[blockIdx.x];
  long long run = off + ex;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < m) {
      indptr[base + i] = run;
      cnt_cursor[base + i] = (int32_t)run;
    }
    run += v[i];
  }
}

__global__ void csr_fill_kernel(const int32_t *__restrict__ F, int64_t n, int K, int64_t lo, int64_t m,
                                int32_t *__restrict__ cursor, int32_t *__restrict__ indices) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t *row = F + s * K;
    for (int j = 0; j < K; ++j) {
      int64_t t = (int64_t)__ldg(row + j) - lo;
      if ((uint64_t)t < (uint64_t)m) {
        int pos = atomicAdd(cursor + t, 1);
        KNND_DCHECK(pos >= 0 && (int64_t)pos < n * K);
        indices[pos] = (int32_t)s;
      }
    }
  }
}

}  // namespace knnd

using namespace knnd;

extern "C" {

size_t knnd_csr_workspace_bytes(int64_t n, int32_t k, int64_t row_lo, int64_t row_hi) {
  (void)n;
  (void)k;
  int64_t m = row_hi > row_lo ? row_hi - row_lo : 0;
  int64_t tiles = (m + SCAN_TILE - 1) / SCAN_TILE;
  return align_up((size_t)m * 4, 256) + align_up((size_t)(tiles + 1) * 8, 256);
}

int knnd_csr_build(const int32_t *friends, int64_t n, int32_t k, int64_t row_lo, int64_t row_hi, int64_t *indptr,
                   int32_t *indices, int32_t *max_indeg, void *ws, size_t ws_bytes, void *stream) {
  return knnd_csr_build_ev(friends, n, k, row_lo, row_hi, indptr, indices, max_indeg, ws, ws_bytes, stream, nullptr);
}

int knnd_csr_build_ev(const int32_t *friends, int64_t n, int32_t k, int64_t row_lo, int64_t row_hi, int64_t *indptr,
                      int32_t *indices, int32_t *max_indeg, void *ws, size_t ws_bytes, void *stream,
                      void *counted_event) {
  KNND_CHECK_ARG(friends && indptr && indices, "knnd_csr_build: null pointer");
  KNND_CHECK_ARG(n >= 1 && k >= 1, "knnd_csr_build: bad sizes");
  KNND_CHECK_ARG(n * (int64_t)k < ((int64_t)1 << 31), "knnd_csr_build: n*K must be < 2^31");
  KNND_CHECK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= n, "knnd_csr_build: bad row range");
  size_t need = knnd_csr_workspace_bytes(n, k, row_lo, row_hi);
  if (ws_bytes < need || (need && !ws)) {
    set_error("knnd_csr_build: workspace %zu < %zu bytes", ws_bytes, need);
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t m = row_hi - row_lo;
  if (max_indeg) KNND_CUDA(cudaMemsetAsync(max_indeg, 0, sizeof(int32_t), st));
  if (m == 0) {
    KNND_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int64_t), st));
    if (counted_event) KNND_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(counted_event), st));
    return KNND_OK;
  }
  int32_t *cnt = static_cast<int32_t *>(ws);
  int64_t *tiles = reinterpret_cast<int64_t *>(static_cast<char *>(ws) + align_up((size_t)m * 4, 256));
  const int64_t ntiles = (m + SCAN_TILE - 1) / SCAN_TILE;
  const int sms = num_sms();

  KNND_CUDA(cudaMemsetAsync(cnt, 0, (size_t)m * 4, st));
  {
    int64_t blocks = (n * k + 255) / 256;
    if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
    csr_count_kernel<<<(unsigned)blocks, 256, 0, st>>>(friends, n, k, row_lo, m, cnt);
    KNND_LAUNCHED(1);
  }
  csr_reduce_kernel<<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(cnt, m, tiles, max_indeg);
  KNND_LAUNCHED(1);
  // max_indeg is final here: a caller that only waits for it (the round's stop test and the
  // next join's plan) need not wait for the scan and the fill — two thirds of the build
  if (counted_event) KNND_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(counted_event), st));
  csr_partials_kernel<<<1, SCAN_THREADS, 0, st>>>(tiles, ntiles, indptr, m);
  KNND_LAUNCHED(1);
  csr_apply_kernel<<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(cnt, m, tiles, indptr);
  KNND_LAUNCHED(1);
  {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
    csr_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(friends, n, k, row_lo, m, cnt, indices);
    KNND_LAUNCHED(1);
  }
  return KNND_OK;
}

}  // extern "C"

KNND_CHECK_READER(csr, 3)
