// Probe: FFMA throughput with a denormal multiplicand vs a normal one (the Q23 screen's F_j = q 2^-149)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float *out, unsigned bits, int iters) {
  float f = __uint_as_float(bits + threadIdx.x);
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
  float w = 1.5f + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(w, f, a0); a1 = fmaf(w, f, a1); a2 = fmaf(w, f, a2); a3 = fmaf(w, f, a3);
    a4 = fmaf(w, f, a4); a5 = fmaf(w, f, a5); a6 = fmaf(w, f, a6); a7 = fmaf(w, f, a7);
    w += 1e-3f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
}
int main() {
  float *o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const unsigned pats[3] = {0x3F800000u, 0x00123456u, 0x00800000u};
  const char *names[3] = {"normal 1.0", "denormal", "min normal"};
  for (int rep = 0; rep < 2; ++rep)
    for (int p = 0; p < 3; ++p) {
      cudaEventRecord(e0);
      k<<<148 * 8, 256>>>(o, pats[p], 100000);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-12s %.3f ms  %.2f TFMA/s\n", names[p], ms, 148.0 * 8 * 256 * 8 * 100000 / (ms * 1e-3) / 1e12);
    }
  return 0;
}
