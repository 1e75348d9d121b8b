// Microbenchmark: dependent DFMA chain latency and DFMA throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = fma(acc, a, b);
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void tput(double* out, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 8);
  int n = 1 << 16;
  chain<<<1, 32>>>(out, 1.0000001, 1e-9, n, cyc); cudaDeviceSynchronize();
  chain<<<1, 32>>>(out, 1.0000001, 1e-9, n, cyc); cudaDeviceSynchronize();
  printf("dependent DFMA latency: %.2f cycles\n", (double)*cyc / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256, m = 4096;
  tput<<<blocks, threads>>>(out, 1.0000001, 1e-9, m);
  cudaEventRecord(e0);
  tput<<<blocks, threads>>>(out, 1.0000001, 1e-9, m);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)blocks * threads * m * 8;
  printf("DFMA throughput: %.2f TFMA/s (%.1f TFLOPS fp64)\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  return 0;
}
