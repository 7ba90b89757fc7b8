// Probe: random-row gather rate by row size (16 .. 80 B rows = 1 .. 3 sectors),
// cp.async.cg 16-B chunks into a per-warp double buffer, a light consumer
// (sum of the row's words).  Which term sets the join's staging rate at the C3
// (L2-resident) and C5 (DRAM) table sizes: rows or sectors?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DPROBE_LD=8 -o tools/row_probe8 tools/row_probe.cu
// Run:   row_probe<LD> n batches blocks_per_sm
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

#ifndef PROBE_LD
#define PROBE_LD 20
#endif
constexpr int LD = PROBE_LD;  // floats per row
constexpr int WARPS = 4;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(WARPS * 32) stage_kernel(const float *tab, const int *ids, int batches, float *out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float *stage0 = reinterpret_cast<float *>(sm) + warp * (2 * 32 * LD);
  const int gw = blockIdx.x * WARPS + warp;
  const int *wids = ids + (size_t)gw * batches * 32;
  float acc = 0.f;
  auto issue = [&](int b, int buf) {
    float *st = stage0 + buf * 32 * LD;
    const int my = wids[b * 32 + lane];
    constexpr int NV4 = LD / 4, RPI = 32 / NV4;
    const int r0 = lane / NV4, part = lane - r0 * NV4;
#pragma unroll
    for (int t = 0; t < (32 + RPI - 1) / RPI; ++t) {
      const int r = r0 + t * RPI;
      const int y = __shfl_sync(0xffffffffu, my, r & 31);
      if (r0 < RPI && r < 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(st + r * LD + part * 4)),
                     "l"(tab + (size_t)y * LD + part * 4)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0, 0);
  for (int b = 0; b < batches; ++b) {
    const int buf = b & 1;
    if (b + 1 < batches) issue(b + 1, buf ^ 1);
    if (b + 1 < batches)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const float4 *row = reinterpret_cast<const float4 *>(stage0 + buf * 32 * LD + lane * LD);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < LD / 4; ++j) {
      const float4 v = row[j];
      s += (v.x + v.y) + (v.z + v.w);
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
  const int blocks_per_sm = argc > 3 ? atoi(argv[3]) : 4;
  {  // argv[4]: cudaLimitMaxL2FetchGranularity (bytes; a hint the platform may clamp)
    size_t g0 = 0, g1 = 0;
    cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
    if (argc > 4) {
      cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[4]));
      cudaDeviceGetLimit(&g1, cudaLimitMaxL2FetchGranularity);
      printf("L2 fetch granularity: default %zu, asked %s -> %zu (%s)\n", g0, argv[4], g1, cudaGetErrorString(e));
    } else {
      printf("L2 fetch granularity: %zu\n", g0);
    }
  }
  const int grid = sms * blocks_per_sm;
  const long nw = (long)grid * WARPS;
  float *tab, *out;
  int *ids;
  CK(cudaMalloc(&tab, n * LD * 4));
  CK(cudaMalloc(&ids, nw * batches * 32 * 4));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(tab, 0, n * LD * 4));
  {
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
  const int smem = WARPS * 2 * 32 * LD * 4;
  CK(cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_kernel, WARPS * 32, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemset(out, 0, 8));
    cudaEventRecord(e0);
    stage_kernel<<<grid, WARPS * 32, smem>>>(tab, ids, batches, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double rows = (double)nw * batches * 32;
  printf("row %3d B  n=%-9ld warps/SM=%-2d (resident blocks/SM %d): %.3e rows/s  %.0f GB/s\n", LD * 4, n,
         blocks_per_sm * WARPS, per_sm, rows / (best * 1e-3), rows * LD * 4 / (best * 1e-3) / 1e9);
  return 0;
}
