// Device replica of the initial random K-out draws (descent.py:194-197):
//   draws = Generator(PCG64).integers(0, n - 1, size=(n, K), dtype=int64)
//   draws += draws >= row
// bit-identical to numpy.  numpy's path for a range below 2^32
// (random_bounded_uint64_fill -> buffered_bounded_lemire_uint32) consumes
// the PCG64 stream as 32-bit halves (low half of each 64-bit output first),
// and Lemire's rejection of a 32-bit value v depends on v alone:
//   m = v * excl; reject iff (m mod 2^32) < (2^32 - excl) mod excl
// so the draws are a stream compaction of accepted values: every thread jumps
// the 128-bit LCG ahead to its slice (O(log) multiplications), counts its
// accepted values, an exclusive scan gives output positions, and a second pass
// writes (m >> 32) plus the row shift.  The kernel also reports how many
// 32-bit values were consumed, so the host can continue the numpy stream for
// the rejection redraws of rows with duplicates (descent.py:198-205).
#include <cmath>

#include "common.cuh"

namespace knnd {

typedef unsigned __int128 u128;

constexpr int RNG_OUT_PER_THREAD = 8;  // 64-bit outputs per thread = 16 u32 values
constexpr int RNG_THREADS = 256;

struct Jump {
  unsigned long long a_lo[64], a_hi[64], c_lo[64], c_hi[64];  // state_{i+2^b} = A_b * state_i + C_b
};

__device__ __forceinline__ u128 mk(unsigned long long hi, unsigned long long lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  const unsigned long long x = hi ^ lo;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct RngArgs {
  unsigned long long s_hi, s_lo, inc_hi, inc_lo;
  unsigned long long mult_hi, mult_lo;
  unsigned excl, thresh;
  int has_u32;
  unsigned u32_buffered;
  long long nthreads;  // threads covering the generated block
  long long out_base;  // 64-bit output index of this block's first output (0-based)
};

// state after `j` more outputs
__device__ __forceinline__ u128 jump(const Jump *__restrict__ J, u128 s, unsigned long long j) {
  for (int b = 0; j; ++b, j >>= 1) {
    if (j & 1ull) s = mk(J->a_hi[b], J->a_lo[b]) * s + mk(J->c_hi[b], J->c_lo[b]);
  }
  return s;
}

// the 16 u32 values of thread t: outputs out_base + t*8 + 0..7, low half first
template <bool WRITE>
__global__ void __launch_bounds__(RNG_THREADS) rng_pass_kernel(RngArgs a, const Jump *__restrict__ J,
                                                               int *__restrict__ counts,
                                                               const long long *__restrict__ offsets,
                                                               long long u32_base, long long N, int K,
                                                               int32_t *__restrict__ out,
                                                               unsigned long long *__restrict__ consumed) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nthreads) return;
  const u128 mult = mk(a.mult_hi, a.mult_lo), inc = mk(a.inc_hi, a.inc_lo);
  u128 s = jump(J, mk(a.s_hi, a.s_lo), (unsigned long long)(a.out_base + t * RNG_OUT_PER_THREAD));
  long long pos = WRITE ? offsets[t] : 0;
  KNND_DCHECK(pos >= 0);
  int cnt = 0;
#pragma unroll
  for (int o = 0; o < RNG_OUT_PER_THREAD; ++o) {
    s = s * mult + inc;
    const unsigned long long v64 = pcg_out(s);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned v = h ? (unsigned)(v64 >> 32) : (unsigned)v64;
      const unsigned long long m = (unsigned long long)v * a.excl;
      if ((unsigned)m >= a.thresh) {
        if (WRITE) {
          if (pos < N) {
            const long long row = (long long)((int)pos / K);
            const long long val = (long long)(m >> 32);
            out[pos] = (int32_t)(val + (val >= row ? 1 : 0));
            if (pos == N - 1)  // index of this u32 in the whole stream, +1
              *consumed = (unsigned long long)(u32_base + t * 2 * RNG_OUT_PER_THREAD + 2 * o + h + 1);
          }
          ++pos;
        } else {
          ++cnt;
        }
      }
    }
  }
  if (!WRITE) counts[t] = cnt;
}

// the buffered high half (has_uint32) is the stream's first value
__global__ void rng_buffered_kernel(RngArgs a, long long N, int32_t *__restrict__ out,
                                    unsigned long long *__restrict__ consumed, long long *__restrict__ first) {
  const unsigned long long m = (unsigned long long)a.u32_buffered * a.excl;
  long long acc = 0;
  if ((unsigned)m >= a.thresh) {
    const long long val = (long long)(m >> 32);
    out[0] = (int32_t)(val + (val >= 0 ? 1 : 0));
    acc = 1;
    if (N == 1) *consumed = 1;
  }
  *first = acc;
}

// exclusive scan of counts (single block, chunked) + base
__global__ void __launch_bounds__(1024) rng_scan_kernel(const int *__restrict__ counts, long long nthreads,
                                                        long long *__restrict__ offsets,
                                                        const long long *__restrict__ base,
                                                        long long *__restrict__ total) {
  __shared__ long long ws[33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long carry = *base;
  for (long long b0 = 0; b0 < nthreads; b0 += 1024) {
    const long long i = b0 + threadIdx.x;
    const long long v = i < nthreads ? counts[i] : 0;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      const long long sv = ws[lane];
      long long si = sv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(FULL, si, o);
        if (lane >= o) si += u;
      }
      ws[lane] = si - sv;
      if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    if (i < nthreads) offsets[i] = carry + ws[w] + inc - v;
    carry += ws[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// rows with a repeated id (descent.py:199-200) -> bad list (unordered)
__global__ void dup_rows_kernel(const int32_t *__restrict__ T, long long n, int K, int32_t *__restrict__ bad,
                                int *__restrict__ nbad) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int32_t *row = T + r * K;
    bool dup = false;
    for (int i = 1; i < K && !dup; ++i) {
      const int32_t v = row[i];
      for (int j = 0; j < i; ++j) dup |= row[j] == v;
    }
    if (dup) {
      const int at = atomicAdd(nbad, 1);
      KNND_DCHECK(at >= 0 && at < n);
      bad[at] = (int32_t)r;
    }
  }
}

}  // namespace knnd

using namespace knnd;

extern "C" {

// generator threads the workspace has room for: a rejection rate up to 1/2
// (the worst case for a range below 2^31) plus margins
static long long rng_ws_threads(int64_t n, int32_t k) {
  const long long N = n * (long long)k;
  return (N * 21 / 10 + 8192) / (2 * RNG_OUT_PER_THREAD) + 64;
}

size_t knnd_random_kout_workspace_bytes(int64_t n, int32_t k) {
  const long long nthreads = rng_ws_threads(n, k);
  return align_up(sizeof(Jump), 256) + align_up((size_t)nthreads * 4, 256) + align_up((size_t)nthreads * 8, 256) +
         256;
}

int knnd_random_kout(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int32_t has_uint32,
                     uint32_t uinteger, int64_t n, int32_t k, int32_t *out, uint64_t *consumed, int32_t *bad,
                     int32_t *nbad, void *ws, size_t ws_bytes, void *stream) {
  KNND_CHECK_ARG(out && consumed && bad && nbad, "knnd_random_kout: null pointer");
  KNND_CHECK_ARG(n >= 3 && k >= 1 && n * (int64_t)k < ((int64_t)1 << 31) && n - 1 <= 0xFFFFFFFFll,
                 "knnd_random_kout: bad sizes n=%lld k=%d", (long long)n, k);
  const size_t need = knnd_random_kout_workspace_bytes(n, k);
  if (!ws || ws_bytes < need) {
    set_error("knnd_random_kout: workspace %zu < %zu bytes", ws_bytes, need);
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  unsigned long long *consumed_d = reinterpret_cast<unsigned long long *>(consumed);
  const long long N = n * (long long)k;
  // integers(0, n-1): numpy's rng = n - 2, rng_excl = n - 1
  const unsigned excl = (unsigned)(n - 1);
  const unsigned thresh = (unsigned)((0xFFFFFFFFull - (unsigned long long)(n - 2)) % excl);

  // jump table on the host (128-bit LCG powers)
  Jump J;
  const unsigned __int128 MULT = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  const unsigned __int128 INC = ((unsigned __int128)inc_hi << 64) | inc_lo;
  unsigned __int128 A = MULT, C = INC;
  for (int b = 0; b < 64; ++b) {
    J.a_lo[b] = (unsigned long long)A;
    J.a_hi[b] = (unsigned long long)(A >> 64);
    J.c_lo[b] = (unsigned long long)C;
    J.c_hi[b] = (unsigned long long)(C >> 64);
    C = A * C + C;  // (A, C) o (A, C)
    A = A * A;
  }
  char *w = static_cast<char *>(ws);
  Jump *dJ = reinterpret_cast<Jump *>(w);
  w += align_up(sizeof(Jump), 256);
  // the layout of knnd_random_kout_workspace_bytes exactly (deriving the count
  // back from the byte total overshot it by the alignment padding, and the
  // scan's two scalars then landed up to ~0.5 KB past the workspace)
  const long long cap_threads = rng_ws_threads(n, k);
  int *counts = reinterpret_cast<int *>(w);
  w += align_up((size_t)cap_threads * 4, 256);
  long long *offsets = reinterpret_cast<long long *>(w);
  w += align_up((size_t)cap_threads * 8, 256);
  long long *scal = reinterpret_cast<long long *>(w);  // [0] base, [1] total
  KNND_CUDA(cudaMemcpyAsync(dJ, &J, sizeof(Jump), cudaMemcpyHostToDevice, st));
  KNND_CUDA(cudaMemsetAsync(nbad, 0, sizeof(int32_t), st));
  KNND_CUDA(cudaMemsetAsync(consumed, 0, sizeof(uint64_t), st));

  RngArgs a;
  a.s_hi = state_hi;
  a.s_lo = state_lo;
  a.inc_hi = inc_hi;
  a.inc_lo = inc_lo;
  a.mult_hi = (unsigned long long)(MULT >> 64);
  a.mult_lo = (unsigned long long)MULT;
  a.excl = excl;
  a.thresh = thresh;
  a.has_u32 = has_uint32;
  a.u32_buffered = uinteger;
  // generate enough u32 values for N accepted ones with overwhelming margin:
  // expected rejections N*p (p = thresh / 2^32); the margin covers 8 sigma + 1%
  const double p = (double)thresh / 4294967296.0;
  const double need_u32 = (double)N / (1.0 - p);
  const long long want_u32 = (long long)(need_u32 * 1.01 + 8.0 * sqrt(need_u32 * (p + 1e-9)) + 1024.0);
  long long nthreads = (want_u32 + 2 * RNG_OUT_PER_THREAD - 1) / (2 * RNG_OUT_PER_THREAD);
  if (nthreads > cap_threads) {
    set_error("knnd_random_kout: rejection rate too high for the workspace (p=%g)", p);
    return KNND_EUNSUPPORTED;
  }
  a.nthreads = nthreads;
  a.out_base = 0;
  const long long u32_base = has_uint32 ? 1 : 0;
  if (has_uint32) {
    rng_buffered_kernel<<<1, 1, 0, st>>>(a, N, out, consumed_d, scal);
    KNND_LAUNCHED(1);
  } else {
    KNND_CUDA(cudaMemsetAsync(scal, 0, sizeof(long long), st));
  }
  const unsigned blocks = (unsigned)((nthreads + RNG_THREADS - 1) / RNG_THREADS);
  rng_pass_kernel<false><<<blocks, RNG_THREADS, 0, st>>>(a, dJ, counts, nullptr, u32_base, N, k, out, consumed_d);
  KNND_LAUNCHED(1);
  rng_scan_kernel<<<1, 1024, 0, st>>>(counts, nthreads, offsets, scal, scal + 1);
  KNND_LAUNCHED(1);
  rng_pass_kernel<true><<<blocks, RNG_THREADS, 0, st>>>(a, dJ, counts, offsets, u32_base, N, k, out, consumed_d);
  KNND_LAUNCHED(1);
  dup_rows_kernel<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(out, n, k, bad, nbad);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

}  // extern "C"

KNND_CHECK_READER(rng, 5)
