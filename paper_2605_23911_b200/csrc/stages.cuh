// stages.cuh — device kernels behind the reference's stage-level API
// (moeperf/__init__.py:56-78): gate_scores / topk_select on caller-given
// logits and scores (router.py:61-113), the numpy-exact sigmoid / silu
// (linalg.py:71-86), the canonical fp64-fold dense_matmul (linalg.py:45-68)
// and the exact fp32 row gather of permute_tokens (pipeline.py:165-183).
// The fused layer forward does not use them; they give the stage functions a
// GPU implementation with the reference's arithmetic, bit for bit.
#pragma once

#include "common.cuh"
#include "router.cuh"

namespace moe {

constexpr int kStageWarps = 8;

// One warp per row: router.py:69-84 on caller-given logits (B, E) fp32.
//   softmax: s = fp32(l - max), e = exp64(s), S = numpy pairwise fp64 sum,
//            score = fp32(e / S)
//   sigmoid: the numpy-SIMD-expf split-form logistic (np_sigmoid)
// Any non-finite logit sets *flag (require_finite, router.py:80).
__global__ void __launch_bounds__(kStageWarps * 32)
gate_scores_kernel(const float* __restrict__ logits, float* __restrict__ scores, int B, int E, int gating,
                   uint32_t* __restrict__ flag) {
  extern __shared__ __align__(16) double gs_row[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  double* row = gs_row + (size_t)warp * E;
  for (int t = blockIdx.x * kStageWarps + warp; t < B; t += gridDim.x * kStageWarps) {
    const float* l = logits + (size_t)t * E;
    float* out = scores + (size_t)t * E;
    bool bad = false;
    float m = -__int_as_float(0x7f800000);
    for (int e = lane; e < E; e += 32) {
      const float v = l[e];
      bad |= !isfinite(v);
      m = fmaxf(m, v);
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(flag, 1u);
      continue;
    }
    if (gating == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      for (int e = lane; e < E; e += 32) row[e] = np_exp64(static_cast<double>(__fsub_rn(l[e], m)));
      __syncwarp();
      const double S = pairwise_sum_warp<double>(row, E, lane);
      for (int e = lane; e < E; e += 32) out[e] = __double2float_rn(__ddiv_rn(row[e], S));
      __syncwarp();
    } else {
      for (int e = lane; e < E; e += 32) out[e] = np_sigmoid(l[e]);
    }
  }
}

// numpy argmax "first maximum" rule over (value, index) pairs: a NaN beats
// everything (the first NaN wins), otherwise the larger value, ties to the
// lower index.
MOE_DEVICE bool argmax_better(float v, int i, float bv, int bi) {
  const bool vn = isnan(v), bn = isnan(bv);
  if (bn) return vn && i < bi;
  if (vn) return true;
  return v > bv || (v == bv && i < bi);
}

// One warp per row: router.py:87-113 on caller-given scores (B, E) fp32,
// literally: k rounds of numpy argmax, the selected entry set to -1.0 in the
// work copy, weights = the ORIGINAL scores of the picks; sigmoid mode
// renormalises by the fp32 pairwise sum (1/k when it is zero).
__global__ void __launch_bounds__(kStageWarps * 32)
topk_select_kernel(const float* __restrict__ scores, int32_t* __restrict__ idx, float* __restrict__ w, int B, int E,
                   int k, int gating) {
  extern __shared__ __align__(16) float tk_work[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* work = tk_work + (size_t)warp * (E + k);
  float* wsel = work + E;
  for (int t = blockIdx.x * kStageWarps + warp; t < B; t += gridDim.x * kStageWarps) {
    const float* s = scores + (size_t)t * E;
    for (int e = lane; e < E; e += 32) work[e] = s[e];
    __syncwarp();
    for (int j = 0; j < k; ++j) {
      float bv = -__int_as_float(0x7f800000);
      int bi = 0x7fffffff;
      for (int e = lane; e < E; e += 32)
        if (bi == 0x7fffffff || argmax_better(work[e], e, bv, bi)) { bv = work[e]; bi = e; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi != 0x7fffffff && (bi == 0x7fffffff || argmax_better(ov, oi, bv, bi))) { bv = ov; bi = oi; }
      }
      __syncwarp();
      if (lane == 0) {
        idx[(size_t)t * k + j] = bi;
        wsel[j] = s[bi];
        work[bi] = -1.0f;
      }
      __syncwarp();
    }
    if (gating == 1) {
      float S = 0.0f;
      if (lane == 0) S = pairwise_sum<float>(wsel, k);
      S = __shfl_sync(0xffffffffu, S, 0);
      const float uni = __double2float_rn(1.0 / static_cast<double>(k));
      for (int j = lane; j < k; j += 32) w[(size_t)t * k + j] = (S == 0.0f) ? uni : __fdiv_rn(wsel[j], S);
    } else {
      for (int j = lane; j < k; j += 32) w[(size_t)t * k + j] = wsel[j];
    }
    __syncwarp();
  }
}

// numpy's float64 exp (np_exp64) over n values: the exhaustive check of the
// port the softmax uses (tests/test_gpu_stage_api.py).
__global__ void __launch_bounds__(256)
np_exp64_kernel(const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    y[i] = np_exp64(x[i]);
}

// linalg.py:71-86, elementwise, bit-exact with numpy's float32 arithmetic.
template <bool kSilu>
__global__ void __launch_bounds__(256)
sigmoid_kernel(const float* __restrict__ x, float* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const float v = x[i];
    const float s = np_sigmoid(v);
    y[i] = kSilu ? __fmul_rn(v, s) : s;
  }
}

// linalg.py:45-68 dot_accumulate: c[i, j] = fp32(sum_k a[i,k] * b[k,j]) with
// exact fp64 products folded strictly in ascending k (the fold is seeded with
// the first product, as np.add.accumulate is).  One thread per output.
__global__ void __launch_bounds__(256)
dense_matmul_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ c, int m, int K,
                    int n) {
  const long long total = (long long)m * n;
  for (long long o = (long long)blockIdx.x * 256 + threadIdx.x; o < total; o += (long long)gridDim.x * 256) {
    const int i = static_cast<int>(o / n), j = static_cast<int>(o % n);
    const float* ar = a + (size_t)i * K;
    double acc = static_cast<double>(ar[0]) * static_cast<double>(b[j]);
    for (int kk = 1; kk < K; ++kk)
      acc = __fma_rn(static_cast<double>(ar[kk]), static_cast<double>(b[(size_t)kk * n + j]), acc);
    c[o] = __double2float_rn(acc);
  }
}

// pipeline.py:165-183: dst[r] = src[fwd[r] / k], rows of row_bytes (a
// multiple of 16), copied exactly.
__global__ void __launch_bounds__(256)
permute_rows_kernel(const uint8_t* __restrict__ src, const int32_t* __restrict__ fwd, int k, uint8_t* __restrict__ dst,
                    int n_rows, int row_bytes) {
  const int vpr = row_bytes / 16;
  const long long total = (long long)n_rows * vpr;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    const int r = static_cast<int>(i / vpr), v = static_cast<int>(i % vpr);
    const int t = fwd[r] / k;
    reinterpret_cast<int4*>(dst + (size_t)r * row_bytes)[v] =
        __ldg(reinterpret_cast<const int4*>(src + (size_t)t * row_bytes) + v);
  }
}

// fp32 -> bf16 (round to nearest even), the operand cast of the stage GEMMs.
__global__ void __launch_bounds__(256)
f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    y[i] = __float2bfloat16_rn(x[i]);
}

}  // namespace moe
