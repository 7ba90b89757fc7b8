// Shared helpers for the knnd sm_100a kernels: error slot, launch accounting,
// warp-level (key) sorting networks used by the top-K selections.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/knnd.h"

namespace knnd {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// host-side error slot / launch counter (defined in abi.cu)
void set_error(const char *fmt, ...);
void count_launch(unsigned n = 1);
int num_sms();
// blocks of `kern` resident per SM at (block threads, dynamic smem) on the current
// device, raising the kernel's dynamic-smem limit to `smem` when needed; memoised
// per (device, kernel, block, smem), so a round's launches make no attribute or
// occupancy API calls after the first time (abi.cu).  Returns a KNND_* status.
int kernel_occupancy(const void *kern, int block, size_t smem, int *per_sm);

#define KNND_CHECK_ARG(cond, ...)            \
  do {                                       \
    if (!(cond)) {                           \
      ::knnd::set_error(__VA_ARGS__);        \
      return KNND_EINVAL;                    \
    }                                        \
  } while (0)

#define KNND_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::knnd::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                     \
      return KNND_ECUDA;                                                         \
    }                                                                            \
  } while (0)

#define KNND_LAUNCHED(n)                                                          \
  do {                                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess) {                                                      \
      ::knnd::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                      \
      return KNND_ECUDA;                                                          \
    }                                                                             \
    ::knnd::count_launch(n);                                                      \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Checked build (-DKNND_CHECKED -> libknnd_checked.so; the stand-in for
// compute-sanitizer, which this GPU pool keeps closed): device-side bounds
// checks on the hand-computed indices — shared-memory slab layouts, hash
// table / list / staging capacities, workspace offsets, id ranges.  A failed
// check counts itself and records its source line (the first one wins) in a
// per-file device word; knnd_check_failures() reads and clears them all.  The
// product build compiles every check away.
#ifdef KNND_CHECKED
static __device__ unsigned long long g_check[2];  // [0] failures, [1] first failing line
#define KNND_DCHECK(cond)                                                                 \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      if (atomicAdd(&::knnd::g_check[0], 1ull) == 0ull) ::knnd::g_check[1] = __LINE__;    \
    }                                                                                     \
  } while (0)
// one reader per source file (file id * 100000 + line identifies a failure)
#define KNND_CHECK_READER(NAME, FILE_ID)                                                   \
  namespace knnd {                                                                        \
  int check_read_##NAME(unsigned long long *count, unsigned long long *first) {          \
    unsigned long long h[2] = {0, 0}, z[2] = {0, 0};                                      \
    if (cudaMemcpyFromSymbol(h, g_check, sizeof(h)) != cudaSuccess) return KNND_ECUDA;    \
    if (cudaMemcpyToSymbol(g_check, z, sizeof(z)) != cudaSuccess) return KNND_ECUDA;      \
    if (h[0] && !*first) *first = (unsigned long long)(FILE_ID) * 100000ull + h[1];      \
    *count += h[0];                                                                       \
    return KNND_OK;                                                                       \
  }                                                                                       \
  }
int check_read_abi(unsigned long long *, unsigned long long *);
int check_read_join(unsigned long long *, unsigned long long *);
int check_read_join_f32k2(unsigned long long *, unsigned long long *);
int check_read_join_q23(unsigned long long *, unsigned long long *);
int check_read_exact(unsigned long long *, unsigned long long *);
int check_read_csr(unsigned long long *, unsigned long long *);
int check_read_prep(unsigned long long *, unsigned long long *);
int check_read_rng(unsigned long long *, unsigned long long *);
#else
#define KNND_DCHECK(cond) \
  do {                    \
  } while (0)
#define KNND_CHECK_READER(NAME, FILE_ID)
#endif

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// keys for the warp sorting networks

// approximate screening key: a float, ascending
struct KeyF {
  float v;
  __device__ __forceinline__ static KeyF inf() { return {__int_as_float(0x7f800000)}; }
  __device__ __forceinline__ bool lt(const KeyF &o) const { return v < o.v; }
  __device__ __forceinline__ KeyF shfl(int src) const { return {__shfl_sync(FULL, v, src)}; }
  __device__ __forceinline__ KeyF shfl_xor(int m) const { return {__shfl_xor_sync(FULL, v, m)}; }
};

// exact key: (fp64 score, tie id) lexicographic — the ScoredRankingSystem
// total order (core.py:83-90); for the initial row sort the tie field is the
// draw position (descent.py:168-169, stable argsort).
struct KeyD {
  double s;
  int id;
  __device__ __forceinline__ static KeyD inf() { return {__longlong_as_double(0x7ff0000000000000ll), 0x7fffffff}; }
  __device__ __forceinline__ bool lt(const KeyD &o) const { return s < o.s || (s == o.s && id < o.id); }
  __device__ __forceinline__ KeyD shfl(int src) const {
    return {__shfl_sync(FULL, s, src), __shfl_sync(FULL, id, src)};
  }
  __device__ __forceinline__ KeyD shfl_xor(int m) const {
    return {__shfl_xor_sync(FULL, s, m), __shfl_xor_sync(FULL, id, m)};
  }
};

template <class Key>
__device__ __forceinline__ Key kmin(const Key &a, const Key &b) { return b.lt(a) ? b : a; }
template <class Key>
__device__ __forceinline__ Key kmax(const Key &a, const Key &b) { return a.lt(b) ? b : a; }

// One bitonic compare-exchange with the partner lane (lane ^ j): keep the
// smaller key, or the larger when keep_max — one comparison, one select.
// (screened value, id) packed into one orderable 64-bit integer: the same
// order as (value, id) lexicographic with a single 64-bit comparison (used to
// certify a row without fp64)
struct KeyU {
  unsigned long long k;
  __device__ __forceinline__ static unsigned ord(float f) {
    const unsigned b = __float_as_uint(f);
    return b ^ ((unsigned)((int)b >> 31) | 0x80000000u);
  }
  __device__ __forceinline__ static KeyU make(float v, int id) {
    return {((unsigned long long)ord(v) << 32) | (unsigned)id};
  }
  __device__ __forceinline__ static KeyU inf() { return make(__int_as_float(0x7f800000), 0x7fffffff); }
  __device__ __forceinline__ float v() const {
    const unsigned u = (unsigned)(k >> 32);
    return __uint_as_float(u ^ ((unsigned)((int)~u >> 31) | 0x80000000u));
  }
  __device__ __forceinline__ int id() const { return (int)(unsigned)k; }
  __device__ __forceinline__ bool lt(const KeyU &o) const { return k < o.k; }
  __device__ __forceinline__ KeyU shfl(int src) const { return {__shfl_sync(FULL, k, src)}; }
  __device__ __forceinline__ KeyU shfl_xor(int m) const { return {__shfl_xor_sync(FULL, k, m)}; }
};

template <class Key>
__device__ __forceinline__ Key cmpx(Key v, int j, bool keep_max) {
  const Key o = v.shfl_xor(j);
  return (o.lt(v) != keep_max) ? o : v;
}

// sort one key per lane ascending (desc: descending) across the warp
// (bitonic, 15 exchanges)
template <class Key, bool DESC = false>
__device__ __forceinline__ Key warp_sort32(Key v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) v = cmpx(v, j, (((lane & k) != 0) != ((lane & j) != 0)) != DESC);
  }
  return v;
}

template <class Key>
__device__ __forceinline__ Key warp_sort32_desc(Key v, int lane) {
  return warp_sort32<Key, true>(v, lane);
}

// sort a bitonic sequence (one key per lane) ascending (5 exchanges)
template <class Key>
__device__ __forceinline__ Key warp_merge32(Key v, int lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) v = cmpx(v, j, (lane & j) != 0);
  return v;
}

// Warp-wide running top-(32*KPL) buffer, element i at lane i%32, register i/32,
// kept sorted ascending.  Only the first K entries are guaranteed exact (entries
// between K and 32*KPL may be stale because inserts are filtered by the K-th).
template <class Key, int KPL>
struct WarpTopK {
  Key b[KPL];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int q = 0; q < KPL; ++q) b[q] = Key::inf();
  }
  __device__ __forceinline__ Key get(int i) const {
    Key r = b[0];
    if (KPL > 1 && i >= 32) r = b[KPL - 1];
    return r.shfl(i & 31);
  }
  // the first batch into an empty buffer: just sort it
  __device__ __forceinline__ void first(Key v, int lane) {
    b[0] = warp_sort32(v, lane);
#pragma unroll
    for (int q = 1; q < KPL; ++q) b[q] = Key::inf();
  }
  // insert one candidate per lane (pass Key::inf() for "none")
  __device__ __forceinline__ void insert(Key v, int K, int lane) {
    Key kth = get(K - 1);
    bool pass = v.lt(kth);
    if (!__any_sync(FULL, pass)) return;
    if (!pass) v = Key::inf();
    v = warp_sort32(v, lane);
    Key r = v.shfl(31 - lane);
    if (KPL == 1) {
      b[0] = warp_merge32(kmin(b[0], r), lane);
    } else {
      Key m = warp_merge32(kmin(b[KPL - 1], r), lane);  // 32 smallest of b1 u v
      Key r2 = m.shfl(31 - lane);
      Key lo = kmin(b[0], r2), hi = kmax(b[0], r2);
      b[0] = warp_merge32(lo, lane);
      b[KPL - 1] = warp_merge32(hi, lane);
    }
  }
};

__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace knnd

namespace knnd {

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) gathers into shared memory.  Rows are copied in
// row-contiguous 16 B (or 8 B) chunks so one warp instruction touches a few
// 128 B lines instead of 32 scattered ones (L1TEX wavefronts, not DRAM, bound
// a lane-per-row gather).
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

}  // namespace knnd
