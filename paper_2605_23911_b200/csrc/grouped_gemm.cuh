// grouped_gemm.cuh — persistent, warp-specialised tcgen05 grouped GEMMs for
// the expert FFN (reference pipeline.py:186-313).
//
// Both projections run "swap-AB": the expert WEIGHT tile is the MMA's M side
// (128 output features per tile) and the routed TOKENS are the N side
// (16..BN rows of one expert chunk).  Small per-expert token counts (16 for
// DeepSeek, ~34 for Qwen, ~128 for Mixtral at 512 tokens) therefore map onto
// a legal N without padding M, and every weight byte is streamed from HBM
// exactly once per chunk — the layer is HBM-bound on that stream at <= 512
// tokens.
//
// Operands are consumed in the reference's stacked layout with no repack:
//   gate/up (E*d, f) and down (E*f, d) are N-contiguous, i.e. the weight
//   tile is MN-major for tcgen05 (A operand, SWIZZLE_128B, LBO = 8 KB between
//   the two 64-wide M halves, SBO = 1 KB between 8-row K groups);
//   activations (rows x K, K-contiguous) are the K-major B operand.
//
// Roles (256 threads, 1 CTA per SM):
//   warp 0   : TMA producer (one elected lane), mbarrier full/empty ring
//   warp 1   : tcgen05.mma issuer (one elected lane)
//   warp 2   : TMEM allocator
//   warps 4-7: epilogue — tcgen05.ld the accumulators, fused math, store
// Gate+up keeps two TMEM accumulators fed from the SAME staged token tile,
// and applies SiLU(g)*u in registers before the bf16 store (pipeline.py:289-296).
// The down projection's epilogue multiplies by the fp32 routing weight and
// scatters each row to its expanded slot t*k+j (pipeline.py:396-399, first
// half); the ordered k-sum happens in the combine kernel.
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kGemmThreads = 256;
constexpr int kBM = 128;        // weight rows (output features) per tile
constexpr int kBK = 64;         // K per stage (one 128-byte swizzle row of bf16)
constexpr int kBoxRows = 32;    // token rows per TMA box

struct GemmParams {
  const int4* chunk_tab;   // {expert, row0, nrows, 0} per token chunk
  const int32_t* n_chunks; // device count of chunks
  int n_mtiles;            // ceil(out_features / 128)
  int K;                   // reduction dim (d for gate/up, f for down)
  int out_features;        // f for gate/up, d for down
  // gate+up epilogue
  __nv_bfloat16* h;        // (T, f)
  // down epilogue
  float* ys;               // (T, d)
  const float* topk_w;     // (B*k) flat
  const int32_t* fwd;      // (T)
};

template <int kBN, bool kGateUp>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;                 // 16 KB per weight matrix
  static constexpr int kNumA = kGateUp ? 2 : 1;
  static constexpr int kBBytes = kBN * kBK * 2;                 // token tile
  static constexpr int kStageBytes = kNumA * kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes;
  static constexpr int kAccCols = kGateUp ? 2 * kBN : kBN;
  static constexpr uint32_t kTmemCols = kAccCols <= 32 ? 32 : kAccCols <= 64 ? 64 : kAccCols <= 128 ? 128 : kAccCols <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(kStages >= 2, "pipeline depth");
  static_assert(kAccCols <= 512, "TMEM columns");
};

MOE_DEVICE float silu_mul(float g, float u) {
  // silu(g) * u in fp32 (fast exp; tolerance path, pipeline.py:294)
  return __fdividef(g, 1.0f + __expf(-g)) * u;
}

template <int kBN, bool kGateUp>
__global__ void __launch_bounds__(kGemmThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tm_a0,
                    const __grid_constant__ CUtensorMap tm_a1,
                    const __grid_constant__ CUtensorMap tm_b, const GemmParams p) {
  using C = GemmCfg<kBN, kGateUp>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tmem_full = empty_bar + C::kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a0);
    if (kGateUp) tma_prefetch_desc(&tm_a1);
    tma_prefetch_desc(&tm_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(full_bar + s, 1);
      mbar_init(empty_bar + s, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  const int total_tiles = __ldg(p.n_chunks) * p.n_mtiles;
  const int num_kb = (p.K + kBK - 1) / kBK;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int4 ch = __ldg(p.chunk_tab + tile / p.n_mtiles);
        const int mt = tile % p.n_mtiles;
        const int n_mma = max(16, (ch.z + 15) & ~15);
        const int nbox = (n_mma + kBoxRows - 1) / kBoxRows;
        const uint32_t bytes = C::kNumA * C::kABytes + nbox * kBoxRows * kBK * 2;
        const int a_col = mt * kBM;
        const int a_row0 = ch.x * p.K;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(empty_bar + stage, phase ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          mbar_arrive_expect_tx(full_bar + stage, bytes);
          const int krow = a_row0 + kb * kBK;
          tma_load_2d_hint(&tm_a0, full_bar + stage, st, a_col, krow, pol_w);
          tma_load_2d_hint(&tm_a0, full_bar + stage, st + C::kABytes / 2, a_col + 64, krow, pol_w);
          if (kGateUp) {
            tma_load_2d_hint(&tm_a1, full_bar + stage, st + C::kABytes, a_col, krow, pol_w);
            tma_load_2d_hint(&tm_a1, full_bar + stage, st + C::kABytes + C::kABytes / 2, a_col + 64,
                             krow, pol_w);
          }
          uint8_t* sb = st + C::kNumA * C::kABytes;
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(&tm_b, full_bar + stage, sb + b * kBoxRows * kBK * 2, kb * kBK,
                        ch.y + b * kBoxRows);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int4 ch = __ldg(p.chunk_tab + tile / p.n_mtiles);
      const int n_mma = max(16, (ch.z + 15) & ~15);
      const uint32_t idesc = make_idesc_bf16(kBM, n_mma, /*a MN-major*/ 1, /*b K-major*/ 0);
      mbar_wait(tmem_empty, acc_phase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(full_bar + stage, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t st = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = st + C::kNumA * C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t bdesc = make_smem_desc_sw128(sb + kk * 32, 16, 1024);
            const uint64_t adesc0 = make_smem_desc_sw128(st + kk * 2048, C::kABytes / 2, 1024);
            const uint32_t acc = (kb | kk) != 0;
            mma_bf16(tmem_base, adesc0, bdesc, idesc, acc);
            if (kGateUp) {
              const uint64_t adesc1 =
                  make_smem_desc_sw128(st + C::kABytes + kk * 2048, C::kABytes / 2, 1024);
              mma_bf16(tmem_base + kBN, adesc1, bdesc, idesc, acc);
            }
          }
          mma_commit(empty_bar + stage);
          if (kb == num_kb - 1) mma_commit(tmem_full);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ============================ epilogue ================================
    const int wq = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int4 ch = __ldg(p.chunk_tab + tile / p.n_mtiles);
      const int mt = tile % p.n_mtiles;
      const int feat = mt * kBM + wq * 32 + lane;  // output feature owned by this thread
      const bool feat_ok = feat < p.out_features;
      mbar_wait(tmem_full, acc_phase);
      tc_fence_after();
      for (int c0 = 0; c0 < ch.z; c0 += 32) {
        uint32_t a[32];
        tmem_ld_32x32b_x32(tmem_base + lane_base + c0, a);
        if (kGateUp) {
          uint32_t b[32];
          tmem_ld_32x32b_x32(tmem_base + lane_base + kBN + c0, b);
          tmem_wait_ld();
          if (feat_ok) {
            __nv_bfloat16* hp = p.h + (size_t)(ch.y + c0) * p.out_features + feat;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              if (c0 + c < ch.z) {
                float v = silu_mul(__uint_as_float(a[c]), __uint_as_float(b[c]));
                hp[(size_t)c * p.out_features] = __float2bfloat16_rn(v);
              }
            }
          }
        } else {
          tmem_wait_ld();
          if (feat_ok) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              if (c0 + c < ch.z) {
                const int xid = __ldg(p.fwd + ch.y + c0 + c);
                const float w = __ldg(p.topk_w + xid);
                p.ys[(size_t)xid * p.out_features + feat] = __fmul_rn(__uint_as_float(a[c]), w);
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tmem_empty);
      acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

}  // namespace moe
