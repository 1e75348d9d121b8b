// ffn.cuh — persistent, warp-specialised tcgen05 expert FFN for sm_100a
// (reference pipeline.py:186-313: fused_gate_up + grouped_gemm(down)).
//
// ONE kernel streams both projections.  Its dynamic work queue holds
//   [gate+up tiles]  (chunk c, 128 ffn rows)       for c in chunks
//   [down tiles]     (chunk c, 128 hidden rows, K split s)
// and every CTA (one per SM) pulls the next tile with an atomic.  A down tile
// of chunk c waits on a per-chunk counter that the chunk's gate+up tiles
// release once their h rows are globally visible, so the down projection of
// early experts overlaps the gate+up tail of late ones: the whole layer's
// expert weights (6·A·d·f bytes) become one HBM stream with a single tail,
// instead of two kernels each paying a wave-quantisation tail.
//
// Swap-AB: expert WEIGHTS are the MMA's M side (128 output features per
// tile) and the routed TOKENS are N (16..BN rows of one expert chunk), so
// 16-token DeepSeek experts and 128-token Mixtral experts both map onto a
// legal N without padding M, and each weight byte is read once per chunk.
// Weights are consumed in the reference's stacked layout (model.py:119-165):
// gate/up (E*d, f) and down (E*f, d) are N-contiguous, i.e. MN-major A
// operands (SWIZZLE_128B; LBO 8 KB between the two 64-wide M halves, SBO 1 KB
// between 8-row K groups).  Tokens (rows x K, K-contiguous) are the K-major
// B operand.
//
// Roles (256 threads): warp 0 = scheduler + TMA producer, warp 1 = MMA
// issuer (one lane), warp 2 = TMEM allocator, warps 4-7 = epilogue.
// Gate+up keeps two TMEM accumulators fed from the SAME staged token tile
// and applies SiLU(g)*u in registers before the bf16 store (pipeline.py:289-296).
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kFfnThreads = 256;
constexpr int kBM = 128;        // weight rows (output features) per tile
constexpr int kBK = 64;         // K per stage: one 128-byte swizzle row of bf16
constexpr int kBoxRows = 32;    // token rows per TMA box
constexpr int kSchedSlots = 4;  // tile-id ring between scheduler and consumers
constexpr int kPrefetchBytes = 256 * 1024;  // L2 prefetch distance of the weight stream per SM

struct FfnParams {
  const int4* chunk_tab;     // {expert, row0, nrows, 0} per token chunk
  const int32_t* n_chunks;   // device count of chunks
  int n_mt_gu;               // gate+up tiles per chunk (ceil(f/128)); 0 = none
  int n_mt_dn;               // down tiles per chunk (ceil(d/128)); 0 = none
  int splits;                // K splits of a down tile
  int kb_per_split;          // k-blocks per down split
  int d, f;
  int T;                     // expanded rows B*k
  __nv_bfloat16* h;          // (T, f) SwiGLU intermediate
  float* ys;                 // down output; split s at ys + s*T*d
  const float* topk_w;       // (B*k) routing weights, flat
  const int32_t* fwd;        // (T) permuted row -> expanded id
  int scale_by_w;            // 1: ys[xid] = w*acc (stage API); 0: raw partials
  int gu_wait;               // down tiles wait for their chunk's gate+up tiles
  int32_t* work_counter;     // self-resetting
  int32_t* exit_counter;     // self-resetting
  int32_t* gu_done;          // per-chunk completed gate+up tiles, self-resetting
  unsigned long long* trace; // optional (debug): per tile {sm, t_fetch, t_first_load, t_done}
};

MOE_DEVICE unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
MOE_DEVICE uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

struct FfnCfg {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB: one 128x64 weight tile
  static constexpr int kBBytes = 256 * kBK * 2;  // 32 KB: up to 256 token rows
  static constexpr int kStageBytes = 2 * kABytes + kBBytes;
  static constexpr int kStages = 3;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 512 /*barriers*/;
};

MOE_DEVICE float silu_mul(float g, float u) {
  // silu(g) * u in fp32 (fast exp; tolerance path, pipeline.py:294)
  return __fdividef(g, 1.0f + __expf(-g)) * u;
}

MOE_DEVICE int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
MOE_DEVICE void red_release_gpu_add(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MOE_DEVICE void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
MOE_DEVICE void epi_bar_sync() {  // the 128 epilogue threads only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

struct TileInfo {
  int is_gu, chunk, mt, split;
};

MOE_DEVICE TileInfo decode_tile(const FfnParams& p, int tile) {
  TileInfo t;
  const int n_gu_per = p.n_mt_gu;
  const int per_dn = p.n_mt_dn * p.splits;
  // gate+up tiles occupy [0, n_chunks*n_mt_gu)
  const int nch = __ldg(p.n_chunks);
  const int n_gu = nch * n_gu_per;
  if (tile < n_gu) {
    t.is_gu = 1;
    t.chunk = tile / n_gu_per;
    t.mt = tile % n_gu_per;
    t.split = 0;
  } else {
    const int q = tile - n_gu;
    t.is_gu = 0;
    t.chunk = q / per_dn;
    const int r = q % per_dn;
    t.mt = r / p.splits;
    t.split = r % p.splits;
  }
  return t;
}

__global__ void __launch_bounds__(kFfnThreads, 1)
ffn_kernel(const __grid_constant__ CUtensorMap tm_wg, const __grid_constant__ CUtensorMap tm_wu,
           const __grid_constant__ CUtensorMap tm_xp, const __grid_constant__ CUtensorMap tm_wd,
           const __grid_constant__ CUtensorMap tm_h, const FfnParams p) {
  using C = FfnCfg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tmem_full = empty_bar + C::kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint64_t* sched_full = tmem_empty + 1;
  uint64_t* sched_empty = sched_full + kSchedSlots;
  int32_t* sched_tile = reinterpret_cast<int32_t*>(sched_empty + kSchedSlots);
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(sched_tile + kSchedSlots);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_wg);
    tma_prefetch_desc(&tm_wu);
    tma_prefetch_desc(&tm_xp);
    tma_prefetch_desc(&tm_wd);
    tma_prefetch_desc(&tm_h);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(full_bar + s, 1);
      mbar_init(empty_bar + s, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    for (int s = 0; s < kSchedSlots; ++s) {
      mbar_init(sched_full + s, 1);
      mbar_init(sched_empty + s, 1 + 4);  // MMA lane + one lane per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  const int nch = __ldg(p.n_chunks);
  const int total_tiles = nch * (p.n_mt_gu + p.n_mt_dn * p.splits);
  const int nkb_gu = (p.d + kBK - 1) / kBK;
  const int nkb_dn = (p.f + kBK - 1) / kBK;

  if (warp == 0) {
    // ====================== scheduler + TMA producer ========================
    // Tile ids are fetched one tile ahead so the weight stream of the next
    // tile is already being prefetched into L2 while this one finishes: the
    // weight tensor is streamed with cp.async.bulk.prefetch.tensor ~kPrefetchBytes
    // ahead of the smem TMA loads, which raises the bytes in flight per SM far
    // beyond the 3 smem stages (HBM latency x 44 GB/s per SM).
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      int slot = 0;
      uint32_t sphase = 0;
      auto fetch = [&]() -> int {
        const int t = atomicAdd(p.work_counter, 1);
        if (p.trace && t < total_tiles) {
          p.trace[t * 4 + 0] = smid();
          p.trace[t * 4 + 1] = globaltimer();
        }
        return t < total_tiles ? t : -1;
      };
      auto kb_range = [&](const TileInfo& ti, int& kb0, int& kb1) {
        if (ti.is_gu) { kb0 = 0; kb1 = nkb_gu; }
        else { kb0 = ti.split * p.kb_per_split; kb1 = min(nkb_dn, kb0 + p.kb_per_split); }
      };
      // L2 prefetch of the weight boxes of k-block kb of a tile
      auto prefetch_w = [&](const TileInfo& ti, const int4& ch, int kb) {
        const int a_col = ti.mt * kBM;
        if (ti.is_gu) {
          const int krow = ch.x * p.d + kb * kBK;
          tma_prefetch_l2_2d(&tm_wg, a_col, krow);
          tma_prefetch_l2_2d(&tm_wg, a_col + 64, krow);
          tma_prefetch_l2_2d(&tm_wu, a_col, krow);
          tma_prefetch_l2_2d(&tm_wu, a_col + 64, krow);
        } else {
          const int krow = ch.x * p.f + kb * kBK;
          tma_prefetch_l2_2d(&tm_wd, a_col, krow);
          tma_prefetch_l2_2d(&tm_wd, a_col + 64, krow);
        }
      };
      int tile = fetch();
      TileInfo ti{};
      int4 ch{};
      int kb0 = 0, kb1 = 0;
      if (tile >= 0) {
        ti = decode_tile(p, tile);
        ch = __ldg(p.chunk_tab + ti.chunk);
        kb_range(ti, kb0, kb1);
      }
      auto pd_for = [&](const TileInfo& t) {
        return t.is_gu ? kPrefetchBytes / (2 * FfnCfg::kABytes) : kPrefetchBytes / FfnCfg::kABytes;
      };
      int pd = tile >= 0 ? pd_for(ti) : 0;  // prefetch distance (k-blocks) of the current tile
      int pf_cur = 0;                          // blocks of the current tile already prefetched
      while (true) {
        mbar_wait(sched_empty + slot, sphase ^ 1);
        sched_tile[slot] = tile;
        mbar_arrive(sched_full + slot);
        if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
        if (tile < 0) break;
        // the next tile is claimed only when the prefetch front reaches the end of
        // this one, so tiles are not reserved long before a CTA can start them
        int nxt = -2;
        TileInfo tn{};
        int4 cn{};
        int nk0 = 0, nk1 = 0;
        auto claim_next = [&]() {
          nxt = fetch();
          if (nxt >= 0) {
            tn = decode_tile(p, nxt);
            cn = __ldg(p.chunk_tab + tn.chunk);
            kb_range(tn, nk0, nk1);
          }
        };
        const int n_mma = max(16, (ch.z + 15) & ~15);
        const int nbox = (n_mma + kBoxRows - 1) / kBoxRows;
        const uint32_t b_bytes = nbox * kBoxRows * kBK * 2;
        const int a_col = ti.mt * kBM;
        if (!ti.is_gu && p.gu_wait) {
          // h rows of this chunk are complete once all its gate+up tiles released
          while (ld_acquire_gpu(p.gu_done + ti.chunk) < p.n_mt_gu) __nanosleep(64);
          fence_proxy_async_global();
        }
        if (p.trace) p.trace[tile * 4 + 2] = globaltimer();
        const int len = kb1 - kb0;
        int pf_nxt = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          // keep the L2 prefetch front pd blocks ahead, running into the next tile
          const int target = kb - kb0 + pd + 1;
          while (pf_cur < min(len, target)) prefetch_w(ti, ch, kb0 + pf_cur++);
          if (target > len) {
            if (nxt == -2) claim_next();
            if (nxt >= 0) {
              const int extra = min(min(nk1 - nk0, pd_for(tn)), target - len);
              while (pf_nxt < extra) prefetch_w(tn, cn, nk0 + pf_nxt++);
            }
          }
          mbar_wait(empty_bar + stage, phase ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          uint8_t* sb = st + 2 * C::kABytes;
          if (ti.is_gu) {
            mbar_arrive_expect_tx(full_bar + stage, 2 * C::kABytes + b_bytes);
            const int krow = ch.x * p.d + kb * kBK;
            tma_load_2d_hint(&tm_wg, full_bar + stage, st, a_col, krow, pol_w);
            tma_load_2d_hint(&tm_wg, full_bar + stage, st + C::kABytes / 2, a_col + 64, krow, pol_w);
            tma_load_2d_hint(&tm_wu, full_bar + stage, st + C::kABytes, a_col, krow, pol_w);
            tma_load_2d_hint(&tm_wu, full_bar + stage, st + C::kABytes + C::kABytes / 2, a_col + 64, krow, pol_w);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d(&tm_xp, full_bar + stage, sb + b * kBoxRows * kBK * 2, kb * kBK, ch.y + b * kBoxRows);
          } else {
            mbar_arrive_expect_tx(full_bar + stage, C::kABytes + b_bytes);
            const int krow = ch.x * p.f + kb * kBK;
            tma_load_2d_hint(&tm_wd, full_bar + stage, st, a_col, krow, pol_w);
            tma_load_2d_hint(&tm_wd, full_bar + stage, st + C::kABytes / 2, a_col + 64, krow, pol_w);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d(&tm_h, full_bar + stage, sb + b * kBoxRows * kBK * 2, kb * kBK, ch.y + b * kBoxRows);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if (nxt == -2) claim_next();
        pf_cur = pf_nxt;
        tile = nxt;
        ti = tn;
        ch = cn;
        kb0 = nk0;
        kb1 = nk1;
        pd = nxt >= 0 ? pd_for(tn) : 0;
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc_phase = 0;
    int slot = 0;
    uint32_t sphase = 0;
    while (true) {
      mbar_wait(sched_full + slot, sphase);
      const int tile = sched_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty + slot);
      if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
      if (tile < 0) break;
      const TileInfo ti = decode_tile(p, tile);
      const int4 ch = __ldg(p.chunk_tab + ti.chunk);
      const int n_mma = max(16, (ch.z + 15) & ~15);
      const uint32_t idesc = make_idesc_bf16(kBM, n_mma, /*a MN-major*/ 1, /*b K-major*/ 0);
      int kb0, kb1;
      if (ti.is_gu) {
        kb0 = 0; kb1 = nkb_gu;
      } else {
        kb0 = ti.split * p.kb_per_split;
        kb1 = min(nkb_dn, kb0 + p.kb_per_split);
      }
      mbar_wait(tmem_empty, acc_phase ^ 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(full_bar + stage, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t st = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = st + 2 * C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t bdesc = make_smem_desc_sw128(sb + kk * 32, 16, 1024);
            const uint64_t adesc0 = make_smem_desc_sw128(st + kk * 2048, C::kABytes / 2, 1024);
            const uint32_t acc = (kb > kb0 || kk > 0) ? 1u : 0u;
            mma_bf16(tmem_base, adesc0, bdesc, idesc, acc);
            if (ti.is_gu) {
              const uint64_t adesc1 = make_smem_desc_sw128(st + C::kABytes + kk * 2048, C::kABytes / 2, 1024);
              mma_bf16(tmem_base + 256, adesc1, bdesc, idesc, acc);
            }
          }
          mma_commit(empty_bar + stage);
          if (kb == kb1 - 1) mma_commit(tmem_full);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // =============================== epilogue ===============================
    const int wq = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    uint32_t acc_phase = 0;
    int slot = 0;
    uint32_t sphase = 0;
    while (true) {
      mbar_wait(sched_full + slot, sphase);
      const int tile = sched_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty + slot);
      if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
      if (tile < 0) break;
      const TileInfo ti = decode_tile(p, tile);
      const int4 ch = __ldg(p.chunk_tab + ti.chunk);
      const int feat = ti.mt * kBM + wq * 32 + lane;  // output feature of this thread
      mbar_wait(tmem_full, acc_phase);
      tc_fence_after();
      if (ti.is_gu) {
        const bool ok = feat < p.f;
        for (int c0 = 0; c0 < ch.z; c0 += 32) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(tmem_base + lane_base + c0, g);
          tmem_ld_32x32b_x32(tmem_base + lane_base + 256 + c0, u);
          tmem_wait_ld();
          if (ok) {
            __nv_bfloat16* hp = p.h + (size_t)(ch.y + c0) * p.f + feat;
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c0 + c < ch.z)
                hp[(size_t)c * p.f] = __float2bfloat16_rn(silu_mul(__uint_as_float(g[c]), __uint_as_float(u[c])));
          }
        }
        tc_fence_before();
        mbar_arrive(tmem_empty);
        if (p.gu_wait) {
          // publish: every epilogue thread's h stores, then one release increment
          __threadfence();
          fence_proxy_async_global();
          epi_bar_sync();
          if (wq == 0 && lane == 0) red_release_gpu_add(p.gu_done + ti.chunk, 1);
        }
      } else {
        const bool ok = feat < p.d;
        float* out = p.ys + (size_t)ti.split * p.T * p.d;
        for (int c0 = 0; c0 < ch.z; c0 += 32) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(tmem_base + lane_base + c0, a);
          tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              if (c0 + c < ch.z) {
                const int xid = __ldg(p.fwd + ch.y + c0 + c);
                float v = __uint_as_float(a[c]);
                if (p.scale_by_w) v = __fmul_rn(v, __ldg(p.topk_w + xid));
                out[(size_t)xid * p.d + feat] = v;
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(tmem_empty);
      }
      if (p.trace && wq == 0 && lane == 0) p.trace[tile * 4 + 3] = globaltimer();
      acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) {
    // last CTA out resets the queue and the per-chunk counters for the next launch
    __threadfence();
    const int prev = atomicAdd(p.exit_counter, 1);
    if (prev == static_cast<int>(gridDim.x) - 1) {
      *p.work_counter = 0;
      for (int c = 0; c < nch; ++c) p.gu_done[c] = 0;
      __threadfence();
      *p.exit_counter = 0;
    }
  }
}

}  // namespace moe
