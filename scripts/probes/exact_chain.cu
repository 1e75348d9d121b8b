// Probe: cycles per step of the warp-cooperative exact fallback chain
// (router.cuh exact_chain_logit_warp) and of a bare dependent DADD chain.
#include <cstdio>
#include <vector>
#include "../../paper_2605_23911_b200/csrc/router.cuh"
using namespace moe;
__global__ void probe(RouterParams p, long long* cyc, float* out) {
  __shared__ double win[kChainWin];
  const int lane = threadIdx.x;
  long long t0 = clock64();
  float v = exact_chain_logit_warp<true>(p, 3, 5, lane, win);
  long long t1 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; out[0] = v; }
  // bare chain
  double acc = 0.0, q = 1e-3 * lane;
  t0 = clock64();
  for (int i = 0; i < 4096; ++i) acc = __dadd_rn(acc, q);
  t1 = clock64();
  if (lane == 0) { cyc[1] = t1 - t0; out[1] = (float)acc; }
}
int main() {
  const int B = 8, d = 2048, E = 60;
  std::vector<uint16_t> hx(B * d, 0x3f80);
  std::vector<float> hw(d * E, 0.5f);
  void *x, *w; long long* cyc; float* out;
  cudaMalloc(&x, hx.size() * 2); cudaMalloc(&w, hw.size() * 4);
  cudaMemcpy(x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(w, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice);
  cudaMallocManaged(&cyc, 16); cudaMallocManaged(&out, 8);
  RouterParams p{}; p.x = x; p.wr = (const float*)w; p.d = d; p.E = E; p.B = B;
  for (int r = 0; r < 3; ++r) { probe<<<1, 32>>>(p, cyc, out); cudaDeviceSynchronize(); }
  printf("exact chain d=%d: %lld cycles, %.2f cyc/step (v=%f); bare DADD chain %.2f cyc/step\n", d, cyc[0],
         (double)cyc[0] / d, out[0], (double)cyc[1] / 4096);
  return 0;
}
