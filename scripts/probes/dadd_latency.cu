// Microbenchmark: dependent DADD vs DFMA chain latency (cycles per step).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void chain(const double* in, double* out, int n, long long* cyc) {
  double acc = in[threadIdx.x];
  const double p = in[threadIdx.x + 32];
  const double q = in[threadIdx.x + 64];
  long long t0 = clock64();
  if (MODE == 0) {
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, p);
  } else {
    for (int i = 0; i < n; ++i) acc = __fma_rn(q, p, acc);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *in, *out; long long* cyc;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 8);
  cudaMemset(in, 0, 4096);
  int n = 1 << 16;
  for (int r = 0; r < 2; ++r) {
    chain<0><<<1, 32>>>(in, out, n, cyc); cudaDeviceSynchronize(); if (r) printf("DADD chain: %.2f cyc/step\n", (double)*cyc / n);
    chain<1><<<1, 32>>>(in, out, n, cyc); cudaDeviceSynchronize(); if (r) printf("DFMA chain: %.2f cyc/step\n", (double)*cyc / n);
  }
  return 0;
}
