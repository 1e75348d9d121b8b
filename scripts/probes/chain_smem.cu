// Microbenchmark: per-step latency of a sequential fp64 FMA chain whose operands
// come from shared memory (x broadcast, w per-lane), as in the router kernel.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int K = 2048;
template <int MODE>
__global__ void chain(const double* __restrict__ gx, const double* __restrict__ gw, double* out, long long* cyc) {
  __shared__ double sx[K];
  __shared__ double sw[K];
  for (int i = threadIdx.x; i < K; i += blockDim.x) { sx[i] = gx[i]; sw[i] = gw[i]; }
  __syncthreads();
  double acc = -0.0;
  long long t0 = clock64();
  if (MODE == 0) {  // plain loop, compiler scheduling
#pragma unroll 16
    for (int k = 0; k < K; ++k) acc = __fma_rn(sx[k], sw[k] * (1 + threadIdx.x * 0), acc);
  } else if (MODE == 1) {  // operands in registers (upper bound)
    double a = sx[threadIdx.x], b = sw[threadIdx.x];
#pragma unroll 16
    for (int k = 0; k < K; ++k) acc = __fma_rn(a, b, acc);
  } else {  // explicit 16-deep register prefetch
    double xa[16], wa[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) { xa[u] = sx[u]; wa[u] = sw[u]; }
    for (int k = 0; k < K; k += 16) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double x = xa[u], w = wa[u];
        if (k + 16 + u < K) { xa[u] = sx[k + 16 + u]; wa[u] = sw[k + 16 + u]; }
        acc = __fma_rn(x, w, acc);
      }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *gx, *gw, *out; long long* cyc;
  cudaMalloc(&gx, K * 8); cudaMalloc(&gw, K * 8); cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 8);
  cudaMemset(gx, 0, K * 8); cudaMemset(gw, 0, K * 8);
  for (int rep = 0; rep < 2; ++rep) {
    chain<0><<<1, 32>>>(gx, gw, out, cyc); cudaDeviceSynchronize(); if (rep) printf("mode0 plain   : %.2f cyc/step\n", (double)*cyc / K);
    chain<1><<<1, 32>>>(gx, gw, out, cyc); cudaDeviceSynchronize(); if (rep) printf("mode1 regs    : %.2f cyc/step\n", (double)*cyc / K);
    chain<2><<<1, 32>>>(gx, gw, out, cyc); cudaDeviceSynchronize(); if (rep) printf("mode2 prefetch: %.2f cyc/step\n", (double)*cyc / K);
  }
  return 0;
}
