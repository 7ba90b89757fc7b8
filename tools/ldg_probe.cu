// Probe: random 64-byte row gather by LDG.128 straight into registers (4 lanes per
// row, one 16-byte chunk each, partial sums reduced by two butterflies) against the
// cp.async staging of tools/row_probe.cu.  Same ids, same consumer (sum of the row).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ldg_probe tools/ldg_probe.cu
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

constexpr int LD = 16;  // floats per row (64 B)
constexpr int WARPS = 4;

template <int DEPTH>  // batches (of 32 rows) in flight per warp
__global__ void __launch_bounds__(WARPS * 32) ldg_kernel(const float *tab, const int *ids, int batches, float *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * WARPS + warp;
  const int *wids = ids + (size_t)gw * batches * 32;
  const int part = lane & 3, r0 = lane >> 2;
  float acc = 0.f;
  float4 buf[DEPTH][4];
  auto issue = [&](int b, float4 (&dst)[4]) {
    const int my = wids[b * 32 + lane];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int y = __shfl_sync(0xffffffffu, my, r0 + 8 * t);
      const float4 *src = reinterpret_cast<const float4 *>(tab + (size_t)y * LD) + part;
      asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(dst[t].x), "=f"(dst[t].y), "=f"(dst[t].z), "=f"(dst[t].w)
                   : "l"(src));
    }
  };
#pragma unroll
  for (int i = 0; i < DEPTH - 1; ++i)
    if (i < batches) issue(i, buf[i]);
#pragma unroll 1
  for (int b0 = 0; b0 < batches; b0 += DEPTH) {
#pragma unroll
    for (int i = 0; i < DEPTH; ++i) {
      const int b = b0 + i;
      if (b + DEPTH - 1 < batches) issue(b + DEPTH - 1, buf[(i + DEPTH - 1) % DEPTH]);
      if (b < batches) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float4 v = buf[i][t];
          float s = (v.x + v.y) + (v.z + v.w);
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          s += __shfl_xor_sync(0xffffffffu, s, 2);
          acc += part == (t & 3) ? s : 0.f;
        }
      }
    }
  }
  atomicAdd(out, acc);
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 1000000;
  const int batches = argc > 2 ? atoi(argv[2]) : 256;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks_per_sm = argc > 3 ? atoi(argv[3]) : 4;
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
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int depth = 2; depth <= 4; ++depth) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemset(out, 0, 8));
      cudaEventRecord(e0);
      if (depth == 2) ldg_kernel<2><<<grid, WARPS * 32>>>(tab, ids, batches, out);
      if (depth == 3) ldg_kernel<3><<<grid, WARPS * 32>>>(tab, ids, batches, out);
      if (depth == 4) ldg_kernel<4><<<grid, WARPS * 32>>>(tab, ids, batches, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double rows = (double)nw * batches * 32;
    printf("LDG.128 64-B rows n=%-9ld warps/SM=%-2d depth %d: %.3e rows/s\n", n, blocks_per_sm * WARPS, depth,
           rows / (best * 1e-3));
  }
  return 0;
}
