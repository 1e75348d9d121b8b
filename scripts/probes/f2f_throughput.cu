// Probe: per-SM throughput of F2F.F64.F32 vs DFMA vs DADD (independent ops, many warps).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const float* in, double* out, int n, long long* cyc) {
  float f[8]; double a[8];
  for (int i = 0; i < 8; ++i) { f[i] = in[(threadIdx.x + i) & 255]; a[i] = f[i]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] += static_cast<double>(f[i]);           // F2F + DADD
      else if (MODE == 1) a[i] = __fma_rn(a[i], 1.0000001, 0.5);  // DFMA
      else if (MODE == 2) a[i] = __dadd_rn(a[i], 0.5);            // DADD
      else { f[i] = __uint_as_float(__float_as_uint(f[i]) + 1u); a[i] = __dadd_rn(a[i], static_cast<double>(f[i])); }
    }
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4); cudaMalloc(&out, 148 * 1024 * 8); cudaMallocManaged(&cyc, 8);
  const int n = 4096, th = 1024;
  const char* names[4] = {"F2F+DADD", "DFMA", "DADD", "int+F2F+DADD"};
  for (int m = 0; m < 4; ++m) {
    for (int r = 0; r < 2; ++r) {
      if (m == 0) k<0><<<148, th>>>(in, out, n, cyc);
      if (m == 1) k<1><<<148, th>>>(in, out, n, cyc);
      if (m == 2) k<2><<<148, th>>>(in, out, n, cyc);
      if (m == 3) k<3><<<148, th>>>(in, out, n, cyc);
      cudaDeviceSynchronize();
    }
    const double ops = (double)th * n * 8;  // per SM
    printf("%-14s %.1f ops/clk/SM\n", names[m], ops / *cyc);
  }
  return 0;
}
