// Probe: per-SM throughput of the segment router's phase-1 instruction mixes
// (16 independent chains per thread, 256 threads, one CTA per SM).
//   A: 16 DFMA + 16 DADD              (no conversions)
//   B: A + 8 F2F.F64.F32              (current router step)
//   C: 16 DFMA + 8 F2F + 16 FFMA.RU   (magnitude bound in fp32)
//   D: 16 DFMA + 8 F2F                (no magnitude)
//   E: 16 DFMA                        (pipe floor)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const float* in, double* out, int n, long long* cyc) {
  float xf[4], wf[4];
  for (int i = 0; i < 4; ++i) { xf[i] = in[(threadIdx.x + i) & 255]; wf[i] = in[(threadIdx.x + 7 * i) & 255]; }
  double acc[16], mag[16];
  float mf[16];
  for (int i = 0; i < 16; ++i) { acc[i] = 0; mag[i] = 0; mf[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    double xd[4], wd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (MODE == 0 || MODE == 4) { xd[i] = 1.0000001 + it; wd[i] = 0.999 * it; }
      else { xd[i] = static_cast<double>(xf[i]); wd[i] = static_cast<double>(wf[i]); }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i * 4 + j] = __fma_rn(xd[i], wd[j], acc[i * 4 + j]);
        if (MODE <= 1) mag[i * 4 + j] = __dadd_rn(mag[i * 4 + j], fabs(acc[i * 4 + j]));
        if (MODE == 2) mf[i * 4 + j] = __fmaf_ru(fabsf(xf[i]), fabsf(wf[j]), mf[i * 4 + j]);
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) { xf[i] = __uint_as_float(__float_as_uint(xf[i]) ^ 1u); wf[i] = __uint_as_float(__float_as_uint(wf[i]) ^ 2u); }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i] + mag[i] + mf[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4); cudaMalloc(&out, 148 * 256 * 8); cudaMallocManaged(&cyc, 8);
  const int n = 2048;
  const char* names[5] = {"A 16DFMA+16DADD", "B +8F2F (router)", "C 16DFMA+8F2F+16FFMA.RU", "D 16DFMA+8F2F", "E 16DFMA"};
  for (int m = 0; m < 5; ++m) {
    for (int r = 0; r < 2; ++r) {
      switch (m) {
        case 0: k<0><<<148, 256>>>(in, out, n, cyc); break;
        case 1: k<1><<<148, 256>>>(in, out, n, cyc); break;
        case 2: k<2><<<148, 256>>>(in, out, n, cyc); break;
        case 3: k<3><<<148, 256>>>(in, out, n, cyc); break;
        default: k<4><<<148, 256>>>(in, out, n, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    printf("%-26s %.1f cycles per step (256 threads, 16 chains each)\n", names[m], (double)*cyc / n);
  }
  return 0;
}
