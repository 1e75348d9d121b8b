// Probe: fp64 register-tiled chains with operands staged in shared memory as
// fp64 (LDS.128 pairs, broadcast across lanes), the candidate inner loop of
// the round-3 router.  Lane = (token pair group, expert pair group): 8 x 4.
// Each lane owns TT tokens x TE experts; warps share the token slice and own
// disjoint expert slices.  SEG adds the magnitude DADD (certified segments).
// Prints cycles per k step and DFMA per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KC = 128;

template <int TT, int TE, int NW, bool SEG>
__global__ void __launch_bounds__(NW * 32, 1) k(const double* gx, const double* gw, double* out, int n, long long* cyc) {
  constexpr int TW = 8 * TT;          // tokens per warp (== per CTA)
  constexpr int EW = 4 * TE;          // experts per warp
  extern __shared__ __align__(16) double sm[];
  double* sx = sm;                    // [KC][TW]
  double* sw = sm + KC * TW;          // [KC][NW*EW]
  for (int i = threadIdx.x; i < KC * TW; i += blockDim.x) sx[i] = gx[i];
  for (int i = threadIdx.x; i < KC * NW * EW; i += blockDim.x) sw[i] = gw[i];
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tg = lane % 8, eg = lane / 8;
  const double* px = sx + tg * TT;
  const double* pw = sw + warp * EW + eg * TE;
  double acc[TT][TE], mag[TT][TE];
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TE; ++j) { acc[i][j] = -0.0; mag[i][j] = 0.0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll 8
    for (int kk = 0; kk < KC; ++kk) {
      double xv[TT], wv[TE];
#pragma unroll
      for (int i = 0; i < TT; i += 2) {
        double2 v = *reinterpret_cast<const double2*>(px + kk * TW + i);
        xv[i] = v.x; xv[i + 1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < TE; j += 2) {
        double2 v = *reinterpret_cast<const double2*>(pw + kk * NW * EW + j);
        wv[j] = v.x; wv[j + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TE; ++j) {
          acc[i][j] = __fma_rn(xv[i], wv[j], acc[i][j]);
          if (SEG) mag[i][j] = __dadd_rn(mag[i][j], fabs(acc[i][j]));
        }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TE; ++j) s += acc[i][j] + mag[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int TT, int TE, int NW, bool SEG>
void run(const char* name, double* gx, double* gw, double* out, long long* cyc) {
  const int n = 64;
  const size_t smem = (size_t)KC * (8 * TT + NW * 4 * TE) * 8;
  cudaFuncSetAttribute(k<TT, TE, NW, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int r = 0; r < 2; ++r) {
    k<TT, TE, NW, SEG><<<148, NW * 32, smem>>>(gx, gw, out, n, cyc);
    cudaDeviceSynchronize();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  const double steps = (double)n * KC;
  const double per = (double)*cyc / steps;
  const double dfma = (double)NW * 32 * TT * TE / per;
  printf("%-34s %6.2f cyc/step  %5.1f DFMA/clk/SM (+%s)\n", name, per, dfma, SEG ? "DADD" : "none");
}

int main() {
  double *gx, *gw, *out;
  long long* cyc;
  cudaMalloc(&gx, 1 << 20);
  cudaMalloc(&gw, 1 << 22);
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 8);
  {
    double h[1 << 17];
    for (int i = 0; i < (1 << 17); ++i) h[i] = 1.0 + 1e-7 * (i % 977);
    cudaMemcpy(gx, h, sizeof(double) * (1 << 17), cudaMemcpyHostToDevice);
    cudaMemcpy(gw, h, sizeof(double) * (1 << 17), cudaMemcpyHostToDevice);
    cudaMemcpy(gw + (1 << 17), h, sizeof(double) * (1 << 17), cudaMemcpyHostToDevice);
  }
  run<2, 2, 4, false>("TT2 TE2 4w exact", gx, gw, out, cyc);
  run<2, 2, 8, false>("TT2 TE2 8w exact", gx, gw, out, cyc);
  run<2, 2, 16, false>("TT2 TE2 16w exact", gx, gw, out, cyc);
  run<2, 4, 4, false>("TT2 TE4 4w exact", gx, gw, out, cyc);
  run<2, 4, 8, false>("TT2 TE4 8w exact", gx, gw, out, cyc);
  run<4, 2, 4, false>("TT4 TE2 4w exact", gx, gw, out, cyc);
  run<4, 2, 8, false>("TT4 TE2 8w exact", gx, gw, out, cyc);
  run<4, 4, 4, false>("TT4 TE4 4w exact", gx, gw, out, cyc);
  run<4, 4, 8, false>("TT4 TE4 8w exact", gx, gw, out, cyc);
  run<2, 2, 8, true>("TT2 TE2 8w seg", gx, gw, out, cyc);
  run<2, 2, 16, true>("TT2 TE2 16w seg", gx, gw, out, cyc);
  run<2, 4, 8, true>("TT2 TE4 8w seg", gx, gw, out, cyc);
  run<4, 4, 8, true>("TT4 TE4 8w seg", gx, gw, out, cyc);
  return 0;
}
