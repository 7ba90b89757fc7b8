// Probe: TMA tile::gather4 row gathers vs cp.async (LDGSTS) 16-B chunk gathers
// of random 80-B fp32 rows into shared memory, the staging step of the
// local join's screen.  (1) correctness at 16-B and 128-B aligned
// destinations, (2) rows/s of each with a light consumer (sum of the row).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

#ifndef PROBE_CP
#define PROBE_CP "cp.async.cg"
#endif
#ifndef PROBE_LD
#define PROBE_LD 20
#endif
constexpr int LD = PROBE_LD;
constexpr int WARPS = 4;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *tm, int r0, int r1, int r2, int r3,
                                        uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(su32(dst)),
      "l"((uint64_t)tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}

// each warp: `batches` batches of 32 rows (ids[] per warp), staged, then each lane sums its row
template <bool TMA>
__global__ void __launch_bounds__(WARPS * 32) stage_kernel(const __grid_constant__ CUtensorMap tm, const float *tab,
                                                           const int *ids, int batches, int align_off, float *out,
                                                           int check, int gs) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slab = 2 * (8 * 384 + 256);  // two buffers of 8 groups (<= 384 B each)
  unsigned char *base = sm + warp * (slab + 128);
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);  // 2 barriers
  float *stage0 = reinterpret_cast<float *>(base + 128 + align_off);
  const int bstride = 8 * 96 + 64;  // floats per buffer
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * WARPS + warp;
  const int *wids = ids + (size_t)gw * batches * 32;
  float acc = 0.f;
  unsigned phase = 0;
  auto issue = [&](int b, int buf) {
    float *st = stage0 + buf * bstride;
    const int my = wids[b * 32 + lane];
    if (TMA) {
      const int i0 = __shfl_sync(0xffffffffu, my, (lane * 4) & 31);
      const int i1 = __shfl_sync(0xffffffffu, my, (lane * 4 + 1) & 31);
      const int i2 = __shfl_sync(0xffffffffu, my, (lane * 4 + 2) & 31);
      const int i3 = __shfl_sync(0xffffffffu, my, (lane * 4 + 3) & 31);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_expect(bar + buf, 32 * LD * 4);
      __syncwarp();
      if (lane < 8) gather4(st + lane * gs, &tm, i0, i1, i2, i3, bar + buf);
    } else {
      constexpr int NV4 = LD / 4, RPI = 32 / NV4;
      const int r0 = lane / NV4, part = lane - r0 * NV4;
#pragma unroll
      for (int t = 0; t < (32 + RPI - 1) / RPI; ++t) {
        const int r = r0 + t * RPI;
        const int y = __shfl_sync(0xffffffffu, my, r & 31);
        if (r0 < RPI && r < 32)
          asm volatile(PROBE_CP ".shared.global [%0], [%1], 16;" ::"r"(su32(st + r * LD + part * 4)),
                       "l"(tab + (size_t)y * LD + part * 4)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  issue(0, 0);
  for (int b = 0; b < batches; ++b) {
    const int buf = b & 1;
    if (b + 1 < batches) issue(b + 1, buf ^ 1);
    if (TMA) {
      mbar_wait(bar + buf, (phase >> buf) & 1);
      phase ^= 1u << buf;
    } else {
      if (b + 1 < batches)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const float *row = stage0 + buf * bstride + (TMA ? (lane >> 2) * gs + (lane & 3) * LD : lane * LD);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < LD; ++j) s += row[j];
    if (check) {
      const int y = wids[b * 32 + lane];
      float t = 0.f;
      for (int j = 0; j < LD; ++j) t += tab[(size_t)y * LD + j];
      if (t != s) atomicAdd(out + 1, 1.f);
    }
    acc += s;
    __syncwarp();
  }
  atomicAdd(out, acc);
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 1000000;
  const int batches = argc > 2 ? atoi(argv[2]) : 256;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks_per_sm = argc > 4 ? atoi(argv[4]) : 4;
  const int grid = sms * blocks_per_sm;
  const long nw = (long)grid * WARPS;
  float *tab;
  int *ids;
  float *out;
  CK(cudaMalloc(&tab, n * LD * 4));
  CK(cudaMalloc(&ids, nw * batches * 32 * 4));
  CK(cudaMalloc(&out, 8));
  {
    float *h = (float *)malloc(n * LD * 4);
    for (long i = 0; i < n * LD; ++i) h[i] = (float)((i * 2654435761u) % 1000) * 0.001f;
    CK(cudaMemcpy(tab, h, n * LD * 4, cudaMemcpyHostToDevice));
    free(h);
    int *hi = (int *)malloc(nw * batches * 32 * 4);
    uint64_t s = 88172645463325252ull;
    for (long i = 0; i < nw * batches * 32; ++i) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      hi[i] = (int)(s % n);
    }
    CK(cudaMemcpy(ids, hi, nw * batches * 32 * 4, cudaMemcpyHostToDevice));
    free(hi);
  }
  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)LD, (cuuint64_t)n};
  cuuint64_t gstr[1] = {(cuuint64_t)LD * 4};
  cuuint32_t box[2] = {(cuuint32_t)LD, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);
  const int smem = WARPS * (2 * (8 * 384 + 256) + 128) + 1024;
  CK(cudaFuncSetAttribute(stage_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(stage_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  float h[2];
  // correctness at 16-B and 128-B aligned destinations
  const int offs[3] = {0, 0, 16}, gss[3] = {96, 80, 96};
  const int which = argc > 3 ? atoi(argv[3]) : 0;
  {
    const int off = offs[which], gs = gss[which];
    CK(cudaMemset(out, 0, 8));
    stage_kernel<true><<<grid, WARPS * 32, smem>>>(tm, tab, ids, 8, off, out, 1, gs);
    cudaError_t e = cudaDeviceSynchronize();
    CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
    printf("tma align_off=%d gs=%d: err=%s mismatches=%.0f\n", off, gs, cudaGetErrorString(e), h[1]);
    if (e != cudaSuccess) return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep)
    for (int tma = 0; tma < 2; ++tma) {
      CK(cudaMemset(out, 0, 8));
      cudaEventRecord(e0);
      if (tma)
        stage_kernel<true><<<grid, WARPS * 32, smem>>>(tm, tab, ids, batches, 0, out, 0, 96);
      else
        stage_kernel<false><<<grid, WARPS * 32, smem>>>(tm, tab, ids, batches, 0, out, 0, 96);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double rows = (double)nw * batches * 32;
      printf("%s n=%ld: %.3f ms, %.3e rows/s, %.1f GB/s (80 B rows)\n", tma ? "tma-gather4" : "cp.async16 ", n, ms,
             rows / (ms * 1e-3), rows * 80 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
