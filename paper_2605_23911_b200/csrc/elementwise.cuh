// elementwise.cuh — HBM-bound row kernels: the expert-major gather
// (pipeline.py:165-183 permute_tokens, fused fp32->bf16 cast) and the
// deterministic k-slot combine (pipeline.py:396-399, ascending j, fp32).
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kRowThreads = 256;

// xp[r, :] = bf16(x[fwd[r] / k, :]); 16-byte vectors.  One CTA per row block.
template <bool kBf16In>
__global__ void __launch_bounds__(kRowThreads)
permute_kernel(const void* __restrict__ x, const int32_t* __restrict__ fwd,
               __nv_bfloat16* __restrict__ xp, int T, int k, int d) {
  const int vec_per_row = d / 8;  // 8 bf16 = 16 B out
  const long total = (long)T * vec_per_row;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int r = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    const int t = __ldg(fwd + r) / k;
    int4 out;
    if (kBf16In) {
      out = __ldg(reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(x) + (size_t)t * d) + v);
    } else {
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(x) + (size_t)t * d) + 2 * v;
      float4 a = __ldg(src), b = __ldg(src + 1);
      __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y);
      __nv_bfloat162 p3 = __floats2bfloat162_rn(b.z, b.w);
      out.x = *reinterpret_cast<int*>(&p0);
      out.y = *reinterpret_cast<int*>(&p1);
      out.z = *reinterpret_cast<int*>(&p2);
      out.w = *reinterpret_cast<int*>(&p3);
    }
    reinterpret_cast<int4*>(xp + (size_t)r * d)[v] = out;
  }
}

// y[t, :] = sum_{j<k} ys[t*k + j, :], ascending j in fp32, starting from
// +0 like the reference's zero-initialised accumulator.  float4 vectors.
template <bool kBf16Out>
__global__ void __launch_bounds__(kRowThreads)
combine_kernel(const float* __restrict__ ys, void* __restrict__ y, int B, int k, int d) {
  const int vec_per_row = d / 4;
  const long total = (long)B * vec_per_row;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int t = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    const float4* src = reinterpret_cast<const float4*>(ys + (size_t)t * k * d) + v;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      float4 a = __ldg(src + (size_t)j * (d / 4));
      acc.x = __fadd_rn(acc.x, a.x);
      acc.y = __fadd_rn(acc.y, a.y);
      acc.z = __fadd_rn(acc.z, a.z);
      acc.w = __fadd_rn(acc.w, a.w);
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
}

// Fused-forward combine: the down tiles wrote raw K-split partials P[s] at
// the expanded slot.  y[t] = sum_j fl(w[t,j] * (sum_s P[s][t*k+j])),
// ascending j and s, fp32 — the reference's out += w_j * g_j order
// (pipeline.py:396-399) with g_j's K-split summed first.
template <bool kBf16Out>
__global__ void __launch_bounds__(kRowThreads)
combine_partials_kernel(const float* __restrict__ ys, int splits, size_t split_stride,
                        const float* __restrict__ topk_w, void* __restrict__ y, int B, int k, int d) {
  const int vec_per_row = d / 4;
  const long total = (long)B * vec_per_row;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int t = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const size_t row = (size_t)t * k + j;
      const float w = __ldg(topk_w + row);
      const float4* src = reinterpret_cast<const float4*>(ys + row * d) + v;
      float4 g = __ldg(src);
      for (int s = 1; s < splits; ++s) {
        float4 a = __ldg(src + s * (split_stride / 4));
        g.x = __fadd_rn(g.x, a.x); g.y = __fadd_rn(g.y, a.y);
        g.z = __fadd_rn(g.z, a.z); g.w = __fadd_rn(g.w, a.w);
      }
      acc.x = __fadd_rn(acc.x, __fmul_rn(w, g.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w, g.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w, g.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w, g.w));
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
}

// Fused-forward combine over the tiled down partials
//   ys[s][feat/256][(feat/128)%2][prow][feat%128]   (prow = padded permuted row)
// y[t] = sum_j fl(w[t,j] * (sum_s P_s)), ascending j and s, fp32 — the
// reference's out += w_j * g_j order (pipeline.py:396-399).  Each warp reads
// one contiguous 512 B row segment per (slot, split).
template <bool kBf16Out>
__global__ void __launch_bounds__(kRowThreads)
combine_tiled_kernel(const float* __restrict__ ys, int splits, int n_dp, int T_pad,
                     const int32_t* __restrict__ prow, const float* __restrict__ topk_w,
                     void* __restrict__ y, int B, int k, int d) {
  pdl_wait();
  const int vec_per_row = d / 4;
  const long total = (long)B * vec_per_row;
  const size_t half_stride = (size_t)T_pad * 128;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int t = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    const int feat = v * 4;
    const size_t blk = (size_t)(feat >> 8) * 2 + ((feat >> 7) & 1);  // (d-pair, half)
    const int col = feat & 127;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const int x = t * k + j;
      const float w = __ldg(topk_w + x);
      const int prow_x = __ldg(prow + x);
      if (prow_x < 0) continue;  // dropped slot (out-of-range routing override)
      const size_t row = (size_t)prow_x;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < splits; ++s) {
        const float* src = ys + ((size_t)s * n_dp * 2 + blk) * half_stride + row * 128 + col;
        const float4 a = __ldg(reinterpret_cast<const float4*>(src));
        if (s == 0) {
          g = a;
        } else {
          g.x = __fadd_rn(g.x, a.x); g.y = __fadd_rn(g.y, a.y);
          g.z = __fadd_rn(g.z, a.z); g.w = __fadd_rn(g.w, a.w);
        }
      }
      acc.x = __fadd_rn(acc.x, __fmul_rn(w, g.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w, g.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w, g.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w, g.w));
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
}

// Fused-forward combine, one CTA per token: the k slots' padded rows and
// routing weights are read once into shared memory, and every thread keeps
// all k x S partial loads of its 16-byte columns in flight.
//   y[t] = sum_j fl(w[t,j] * (sum_s P_s[prow(t*k+j)])), ascending j and s,
// fp32 from +0 — the reference's out += w_j * g_j (pipeline.py:396-399).
constexpr int kCombineMaxKS = 16;  // k * S register budget (else the generic loop)
// kNV: 16-byte columns per thread (k * S <= kCombineMaxKS / kNV partials each)
template <bool kBf16Out, int kS, int kNV>
__global__ void __launch_bounds__(kRowThreads)
combine_token_kernel(const float* __restrict__ ys, int n_dp, int T_pad,
                     const int32_t* __restrict__ prow, const float* __restrict__ topk_w,
                     void* __restrict__ y, int B, int k, int d) {
  __shared__ int32_t s_row[kCombineMaxKS];
  __shared__ float s_w[kCombineMaxKS];
  // grid (B, ceil(d / 4 / (kRowThreads * kNV))): up to kNV
  // 16-byte columns of one token per thread, every partial load issued before
  // the first add (one L2 round trip after the row ids)
  const int t = blockIdx.x;
  // PDL: griddepcontrol.wait only orders this grid after its immediate
  // predecessor (the FFN); the row ids / weights come from the router and the
  // dispatch, two launches earlier, so they too are read after the wait.
  pdl_wait();
  if (threadIdx.x < k) {
    s_row[threadIdx.x] = prow[(size_t)t * k + threadIdx.x];
    s_w[threadIdx.x] = topk_w[(size_t)t * k + threadIdx.x];
  }
  __syncthreads();
  const size_t half_stride = (size_t)T_pad * 128;
  constexpr int kSlots = kCombineMaxKS / kNV;
  constexpr int kMaxK = kSlots / kS;
  const int ks = k * kS;
  const int v0 = blockIdx.y * kRowThreads * kNV + threadIdx.x;
  float4 a[kNV][kSlots];
#pragma unroll
  for (int c = 0; c < kNV; ++c) {
    const int v = v0 + c * kRowThreads;
    const int feat = v * 4;
    const size_t blk = (size_t)(feat >> 8) * 2 + ((feat >> 7) & 1);  // (d-pair, half)
    const int col = feat & 127;
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
      if (i < ks && v < d / 4) {
        const int j = i / kS, s = i % kS;
        if (s_row[j] < 0) { a[c][i] = make_float4(0.f, 0.f, 0.f, 0.f); continue; }  // dropped slot
        const float* src = ys + ((size_t)s * n_dp * 2 + blk) * half_stride + (size_t)s_row[j] * 128 + col;
        a[c][i] = __ldg(reinterpret_cast<const float4*>(src));
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kNV; ++c) {
    const int v = v0 + c * kRowThreads;
    if (v >= d / 4) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j < k && s_row[j] >= 0) {
        float4 g = a[c][j * kS];
#pragma unroll
        for (int s = 1; s < kS; ++s) {
          const float4 b = a[c][j * kS + s];
          g.x = __fadd_rn(g.x, b.x); g.y = __fadd_rn(g.y, b.y);
          g.z = __fadd_rn(g.z, b.z); g.w = __fadd_rn(g.w, b.w);
        }
        const float w = s_w[j];
        acc.x = __fadd_rn(acc.x, __fmul_rn(w, g.x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(w, g.y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(w, g.z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(w, g.w));
      }
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
}

// The combine overlapped with the FFN's tail: combine_token_kernel's
// arithmetic (identical bits), but launched right behind the FFN with
// programmatic dependent launch and WITHOUT griddepcontrol.wait -- its CTAs
// start on SMs the persistent FFN grid releases and each spins (acquire) on
// the arrival counters of its token's 256-column blocks (ffn.cuh
// FfnParams::arrive) until all k * S partial rows are in, then combines and
// resets the counters.  The FFN's last down tiles and this grid overlap, so
// only the last tokens' combine is exposed after the FFN.
template <bool kBf16Out, int kS, int kNV>
__global__ void __launch_bounds__(kRowThreads)
combine_flag_kernel(const float* __restrict__ ys, int n_dp, int T_pad, const int32_t* __restrict__ prow,
                    const float* __restrict__ topk_w, void* __restrict__ y, int B, int k, int d,
                    int32_t* __restrict__ arrive, int S) {
  __shared__ int32_t s_row[kCombineMaxKS];
  __shared__ float s_w[kCombineMaxKS];
  const int t = blockIdx.x;
  const int c_lo = blockIdx.y * kRowThreads * kNV * 4;                // first column of this CTA
  const int mt_lo = c_lo / 256, mt_hi = min(n_dp, (c_lo + kRowThreads * kNV * 4 + 255) / 256);
  const int target = k * S;
  if (threadIdx.x < mt_hi - mt_lo) {
    const int32_t* a = arrive + (size_t)t * n_dp + mt_lo + threadIdx.x;
    int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
      if (v >= target) break;
      __nanosleep(128);
    }
  }
  if (threadIdx.x < k) {
    s_row[threadIdx.x] = __ldcg(prow + (size_t)t * k + threadIdx.x);
    s_w[threadIdx.x] = __ldcg(topk_w + (size_t)t * k + threadIdx.x);
  }
  __syncthreads();
  const size_t half_stride = (size_t)T_pad * 128;
  constexpr int kSlots = kCombineMaxKS / kNV;
  constexpr int kMaxK = kSlots / kS;
  const int ks = k * kS;
  const int v0 = blockIdx.y * kRowThreads * kNV + threadIdx.x;
  float4 a[kNV][kSlots];
#pragma unroll
  for (int c = 0; c < kNV; ++c) {
    const int v = v0 + c * kRowThreads;
    const int feat = v * 4;
    const size_t blk = (size_t)(feat >> 8) * 2 + ((feat >> 7) & 1);
    const int col = feat & 127;
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
      if (i < ks && v < d / 4) {
        const int j = i / kS, s = i % kS;
        if (s_row[j] < 0) { a[c][i] = make_float4(0.f, 0.f, 0.f, 0.f); continue; }
        const float* src = ys + ((size_t)s * n_dp * 2 + blk) * half_stride + (size_t)s_row[j] * 128 + col;
        a[c][i] = __ldcg(reinterpret_cast<const float4*>(src));
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kNV; ++c) {
    const int v = v0 + c * kRowThreads;
    if (v >= d / 4) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j < k && s_row[j] >= 0) {
        float4 g = a[c][j * kS];
#pragma unroll
        for (int s = 1; s < kS; ++s) {
          const float4 b = a[c][j * kS + s];
          g.x = __fadd_rn(g.x, b.x); g.y = __fadd_rn(g.y, b.y);
          g.z = __fadd_rn(g.z, b.z); g.w = __fadd_rn(g.w, b.w);
        }
        const float w = s_w[j];
        acc.x = __fadd_rn(acc.x, __fmul_rn(w, g.x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(w, g.y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(w, g.z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(w, g.w));
      }
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
  __syncthreads();  // every partial of this CTA's blocks is read: reset their counters
  if (threadIdx.x < mt_hi - mt_lo) arrive[(size_t)t * n_dp + mt_lo + threadIdx.x] = 0;
}

// Unfused ablation (pipeline.py:316-370 unfused_gate_up): the separate
// activation pass h = bf16(silu(g) * u) over the tiled fp32 projections
// [proj][f/128][T_pad][128] -> tiled bf16 h [f/128][T_pad][128], with the
// fused epilogue's exact formula (silu_mul, ffn.cuh) so h is bit-identical.
__global__ void __launch_bounds__(kRowThreads)
swiglu_tiled_kernel(const float* __restrict__ gu32, __nv_bfloat16* __restrict__ h, size_t n_per_proj) {
  pdl_wait();
  const size_t n4 = n_per_proj / 4;
  for (size_t i = (size_t)blockIdx.x * kRowThreads + threadIdx.x; i < n4; i += (size_t)gridDim.x * kRowThreads) {
    const float4 g = __ldg(reinterpret_cast<const float4*>(gu32) + i);
    const float4 u = __ldg(reinterpret_cast<const float4*>(gu32 + n_per_proj) + i);
    const __nv_bfloat162 a = __floats2bfloat162_rn(silu_mul(g.x, u.x), silu_mul(g.y, u.y));
    const __nv_bfloat162 b = __floats2bfloat162_rn(silu_mul(g.z, u.z), silu_mul(g.w, u.w));
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&a);
    o.y = *reinterpret_cast<const uint32_t*>(&b);
    reinterpret_cast<uint2*>(h)[i] = o;
  }
}

// Expert-parallel helpers --------------------------------------------------

// dst[r, :] = src[idx[r], :] for rows of `row_bytes` (multiple of 16) bytes.
__global__ void __launch_bounds__(kRowThreads)
gather_rows_kernel(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx,
                   uint8_t* __restrict__ dst, int n_rows, int row_bytes) {
  const int vec_per_row = row_bytes / 16;
  const long total = (long)n_rows * vec_per_row;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int r = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    const int4 val = __ldg(reinterpret_cast<const int4*>(src + (size_t)__ldg(idx + r) * row_bytes) + v);
    reinterpret_cast<int4*>(dst + (size_t)r * row_bytes)[v] = val;
  }
}

// Schedule for rows that arrive already grouped by (local) expert: counts ->
// offsets, 16-aligned padded offsets, FFN chunk table and the padded row map.
// One CTA (E_local <= 1024).  Mirrors the scheduler half of the router kernel.
__global__ void __launch_bounds__(256)
schedule_from_counts_kernel(const int32_t* __restrict__ counts, int E, int chunk_rows,
                            int32_t* __restrict__ offsets, int4* __restrict__ chunk_tab, int2* __restrict__ chunk_grp,
                            int32_t* __restrict__ n_chunks, int32_t* __restrict__ prow) {
  __shared__ int32_t s_off[1025], s_off16[1025], s_cpre[1025];
  if (threadIdx.x == 0) {
    int a = 0, b = 0, c = 0;
    for (int e = 0; e < E; ++e) {
      s_off[e] = a; s_off16[e] = b; s_cpre[e] = c;
      const int n = counts[e];
      a += n; b += (n + 15) & ~15; c += (n + chunk_rows - 1) / chunk_rows;
    }
    s_off[E] = a; s_off16[E] = b; s_cpre[E] = c;
    *n_chunks = c;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += blockDim.x) offsets[e] = s_off[e];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int n = counts[e];
    const int nch_e = (n + chunk_rows - 1) / chunk_rows;
    for (int c = 0; c < nch_e; ++c) {
      const int r0 = c * chunk_rows;
      chunk_tab[s_cpre[e] + c] = make_int4(e, s_off[e] + r0, min(chunk_rows, n - r0), s_off16[e] + r0);
      chunk_grp[s_cpre[e] + c] = make_int2(s_cpre[e], nch_e);
    }
  }
  // padded row of every (expert-major) row
  const int T = s_off[E];
  for (int r = threadIdx.x; r < T; r += blockDim.x) {
    int lo = 0, hi = E - 1;  // expert of row r: last e with off[e] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    prow[r] = s_off16[lo] + (r - s_off[lo]);
  }
}

// Unweighted per-row expert output: out[r] = sum_s P_s[prow[r]] (fp32, ascending s)
__global__ void __launch_bounds__(kRowThreads)
row_reduce_kernel(const float* __restrict__ ys, int splits, int n_dp, int T_pad,
                  const int32_t* __restrict__ prow, float* __restrict__ out, int T, int d) {
  const int vec_per_row = d / 4;
  const long total = (long)T * vec_per_row;
  const size_t half_stride = (size_t)T_pad * 128;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int r = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    const int feat = v * 4;
    const size_t blk = (size_t)(feat >> 8) * 2 + ((feat >> 7) & 1);
    const size_t row = (size_t)__ldg(prow + r);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(ys + ((size_t)s * n_dp * 2 + blk) * half_stride + row * 128 + (feat & 127)));
      if (s == 0) { g = a; } else {
        g.x = __fadd_rn(g.x, a.x); g.y = __fadd_rn(g.y, a.y);
        g.z = __fadd_rn(g.z, a.z); g.w = __fadd_rn(g.w, a.w);
      }
    }
    reinterpret_cast<float4*>(out + (size_t)r * d)[v] = g;
  }
}

// Home-rank combine of expert-parallel results: rows come back in the local
// expert-major order; y[t] = sum_j fl(w[t,j] * rows[inv[t*k+j]]), ascending j.
template <bool kBf16Out>
__global__ void __launch_bounds__(kRowThreads)
combine_rows_kernel(const float* __restrict__ rows, const int32_t* __restrict__ inv,
                    const float* __restrict__ topk_w, void* __restrict__ y, int B, int k, int d) {
  const int vec_per_row = d / 4;
  const long total = (long)B * vec_per_row;
  for (long i = (long)blockIdx.x * kRowThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kRowThreads) {
    const int t = static_cast<int>(i / vec_per_row);
    const int v = static_cast<int>(i % vec_per_row);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const int x = t * k + j;
      const float w = __ldg(topk_w + x);
      const float4 g = __ldg(reinterpret_cast<const float4*>(rows + (size_t)__ldg(inv + x) * d) + v);
      acc.x = __fadd_rn(acc.x, __fmul_rn(w, g.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w, g.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w, g.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w, g.w));
    }
    if (kBf16Out) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&p0);
      o.y = *reinterpret_cast<uint32_t*>(&p1);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(y) + (size_t)t * d)[v] = o;
    } else {
      reinterpret_cast<float4*>(static_cast<float*>(y) + (size_t)t * d)[v] = acc;
    }
  }
}

}  // namespace moe
