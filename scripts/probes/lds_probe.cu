// Probe: shared-memory load cost (cycles per warp instruction, per SM) by
// width and address pattern, 8 warps per SM, 148 CTAs.  The results fix the
// operand-delivery model of the fp64 router tiles.
#include <cstdio>
#include <cuda_runtime.h>

// PAT: 0 all lanes same address; 1 lane%8 distinct (quarter-warp broadcast);
// 2 lane/8 distinct (8 lanes share); 3 all 32 distinct consecutive;
// 4 lane%16 distinct; 5 lane/4 distinct
template <int W, int PAT>
__global__ void __launch_bounds__(256, 1) k(double* out, int n, long long* cyc) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i;
  __syncthreads();
  const int lane = threadIdx.x % 32;
  int idx;
  switch (PAT) {
    case 0: idx = 0; break;
    case 1: idx = (lane % 8); break;
    case 2: idx = (lane / 8); break;
    case 3: idx = lane; break;
    case 4: idx = lane % 16; break;
    default: idx = lane / 4; break;
  }
  idx *= W / 8;  // element stride = access width
  double acc0 = 0, acc1 = 0;
  const long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int o = ((it * 16 + u) & 63) * 64 + idx;
      if (W == 4) {
        acc0 += reinterpret_cast<const float*>(sm)[o];
      } else if (W == 8) {
        acc0 += sm[o];
      } else {
        const double2 v = *reinterpret_cast<const double2*>(sm + o);
        acc0 += v.x;
        acc1 += v.y;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int W, int PAT>
void run(const char* name, double* out, long long* cyc) {
  const int n = 256;
  for (int r = 0; r < 2; ++r) { k<W, PAT><<<148, 256>>>(out, n, cyc); cudaDeviceSynchronize(); }
  // 8 warps x n*16 loads per SM
  printf("LDS.%-3d %-22s %5.2f cyc/warp-instr (SM)\n", W * 8, name, (double)*cyc / (8.0 * n * 16));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 8);
  run<4, 0>("same addr", out, cyc);
  run<4, 3>("32 distinct", out, cyc);
  run<8, 0>("same addr", out, cyc);
  run<8, 1>("lane%8 distinct", out, cyc);
  run<8, 2>("lane/8 distinct", out, cyc);
  run<8, 4>("lane%16 distinct", out, cyc);
  run<8, 5>("lane/4 distinct", out, cyc);
  run<8, 3>("32 distinct", out, cyc);
  run<16, 0>("same addr", out, cyc);
  run<16, 1>("lane%8 distinct", out, cyc);
  run<16, 2>("lane/8 distinct", out, cyc);
  run<16, 4>("lane%16 distinct", out, cyc);
  run<16, 5>("lane/4 distinct", out, cyc);
  run<16, 3>("32 distinct", out, cyc);
  return 0;
}
