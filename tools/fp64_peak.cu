// DFMA throughput microbenchmark: independent FMA chains per thread, all SMs.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; cudaMalloc(&out, 8);
  const int CH = 8, iters = 1 << 16;
  int blocks = p.multiProcessorCount * 8, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<CH><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * CH * (double)iters * blocks * threads;
    printf("rep %d: %.3f ms  %.2f TFLOP/s fp64\n", rep, ms, flops / ms / 1e9);
  }
  return 0;
}
