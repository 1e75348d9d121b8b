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
// Roles (384 threads): warp 0 = scheduler + TMA producer, warp 1 = MMA
// issuer (one lane), warp 2 = TMEM allocator, warps 4-11 = epilogue in two
// groups of four (warp w reads TMEM lanes 32*(w%4)..+31); 32-row token chunks
// alternate between the groups so the TMEM drain (SiLU on MUFU) runs on 8
// warps and the next tile's MMAs start sooner.
// Gate+up keeps two TMEM accumulators fed from the SAME staged token tile
// and applies SiLU(g)*u in registers before the bf16 store (pipeline.py:289-296).
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kFfnThreads = 384;
constexpr int kEpiWarps = 8;    // warps 4..11: two groups of 4 (one warp per TMEM lane quadrant)
constexpr int kEpiGroups = 2;   // 32-row chunks alternate between the groups
constexpr int kBM = 128;        // weight rows (output features) per tile
constexpr uint32_t kAcc2 = 256; // TMEM column offset of a tile's second accumulator (up / down half 1)
constexpr int kBK = 64;         // K per stage: one 128-byte swizzle row of bf16
#ifndef MOE_B200_BOX_ROWS
#define MOE_B200_BOX_ROWS 32
#endif
constexpr int kBoxRows = MOE_B200_BOX_ROWS;  // token rows per TMA box
constexpr int kSchedSlots = 4;  // tile-id ring between scheduler and consumers

struct FfnParams {
  // down weights as a 3-D view with a 4-block box: a down tile's two adjacent
  // 128-row hidden tiles (two ring slots, 512 contiguous bytes per row) in one
  // TMA request when the slots are adjacent in the ring (w3d only)
  alignas(64) CUtensorMap tm_wd4;
  const int4* chunk_tab;     // {expert, row0, nrows, padded row0} per token chunk
  const int2* chunk_grp;     // {first chunk, chunks} of the chunk's expert
  const int32_t* n_chunks;   // device count of chunks
  int n_mt_gu;               // gate+up tiles per chunk (ceil(f/128)); 0 = none
  int n_mt_dn;               // down tiles per chunk (ceil(d/256): pairs of 128 rows); 0 = none
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
  int gu_unfused;            // 1: gate and up as separate tiles, fp32 out (pipeline.py:316-370 ablation)
  float* gu32;               // unfused output: tiled [proj][f/128][T_pad][128] fp32
  int pair;                  // 1: launched as CTA pairs (clusters of 2) sharing token loads
  int tiled;                 // 1: h / ys in the tiled padded-row layouts (fused forward)
  int T_pad;                 // padded-row capacity of the tiled layouts
  unsigned long long* trace; // optional (debug): 8 u64 per tile {sm, fetch, first load, epi done, epi start, mma start}
  // Overlapped combine (elementwise.cuh combine_flag_kernel): arrive != null:
  // once a down tile's K-split partial rows are globally visible, its
  // epilogue adds 1 to arrive[t][mt] for every row (token t = expanded id / k,
  // mt its 256-column block); the combine grid, launched behind this one with
  // programmatic dependent launch, starts on the SMs this grid releases and
  // combines each (token, block) as soon as its k * splits arrivals are in.
  int tmem_db;               // 1: chunks of <= 128 rows alternate two TMEM accumulator slots
  int32_t* arrive;           // (B, n_mt_dn) arrival counters, reset by the combine
  int k;                     // top-k: slot j of token t is expanded id t * k + j
  int w3d;                   // 1: tm_wg / tm_wu / tm_wd are 3-D [64-col block][row][64 col] views (one load per slot)
  int wd4;                   // 1: tm_wd4 is valid (down tiles load both hidden halves in one request)
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

// Shared memory: a ring of 16 KB weight slots (one 128 x 64 bf16 MN-major
// tile each) decoupled from a ring of token slots (kBN x 64 bf16).  A
// gate+up k-block takes two weight slots and one token slot, a down k-block
// one of each, so the weight bytes in flight per SM (the HBM-latency x
// bandwidth product) no longer shrink with the token tile: 8-10 slots keep
// 128-160 KB of weights outstanding for either tile type.
// Epilogue stores go through shared-memory staging buffers and asynchronous
// bulk copies (one 256 B / 512 B row segment per copy, issued by one lane),
// so the output stream never competes with the weight stream as thousands of
// scattered STGs.  kV selects the ring/staging split (tuning).
template <int kBN, int kV, bool k2 = false>
struct FfnCfg {
  static constexpr int kABytes = kBM * kBK * 2;      // 16 KB weight slot
  static constexpr int kBRows = k2 ? kBN / 2 : kBN;  // cta_group::2: each CTA holds half the token rows
  static constexpr int kBBytes = kBRows * kBK * 2;   // token slot
  static constexpr int kStgBytes = 32 * kBM * 4;     // 32 rows x 128 fp32 (16 KB)
  static constexpr int kStgBufs = kEpiGroups;  // one staging buffer per epilogue group
  // kV 2: balanced rings; kV 3: deeper weight ring (more HBM bytes in flight
  // per SM), shallower token ring (tokens are L2-resident)
  // k2: the halved token slots buy a deeper weight ring (8 A / 4 B for BN=256)
  static constexpr int kAStages = k2 ? (kBN == 256 ? 8 : 10) : kBN == 256 ? (kV == 3 ? 8 : 6) : (kV == 3 ? 10 : 8);
  static constexpr int kBStages = k2 ? 4 : kBN == 256 ? (kV == 3 ? 2 : 3) : (kV == 3 ? 2 : 4);
  static constexpr int kRingBytes = kAStages * kABytes + kBStages * kBBytes;
  static constexpr int kDataBytes = kRingBytes + kStgBufs * kStgBytes;
  // 512 columns: two accumulators (gate / up, or the two down halves) at
  // +0 and +kAcc2, each holding up to 256 token columns -- or, for token
  // chunks of <= 128 rows, TWO such pairs (slots at +0 and +128): the next
  // tile's MMAs run into the other slot while this tile's epilogue drains
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kSmemBytes = kDataBytes + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(kSmemBytes <= 232448, "shared memory");
};

MOE_DEVICE void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
MOE_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
MOE_DEVICE void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
MOE_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
MOE_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
MOE_DEVICE void epi_bar_sync(int group) {  // the 128 threads of one epilogue group
  asm volatile("bar.sync %0, 128;" ::"r"(1 + group) : "memory");
}

struct TileInfo {
  int is_gu, chunk, mt, split;
  int dummy;  // pair mode: the pair's second weight tile does not exist (odd tile count)
};

// Tile order.  Gate+up tiles come first, then down tiles.  Within each, an
// expert's tiles are contiguous (chunk-major over experts, so the down tiles
// of early experts are ready early), and when an expert spans several token
// chunks (a hot expert under routing skew) its tiles are ordered weight-tile
// major, chunk minor: the chunks' reads of the SAME weight tile are adjacent
// in the queue, run concurrently on different SMs and are served once from
// HBM (L2 de-duplicates), keeping the weight stream near one pass.
// Pair mode (CTA pairs sharing token loads, see ffn_kernel): a tile id names a
// PAIR of adjacent weight tiles of the same chunk; CTA rank r takes weight
// tile 2 * pair + r.
MOE_DEVICE TileInfo decode_tile(const FfnParams& p, int tile, int rank = 0) {
  TileInfo t;
  t.dummy = 0;
  const int mt_gu = p.pair ? (p.n_mt_gu + 1) / 2 : p.n_mt_gu;
  const int mt_dn = p.pair ? (p.n_mt_dn + 1) / 2 : p.n_mt_dn;
  const int per_gu = mt_gu * (p.gu_unfused ? 2 : 1);
  const int per_dn = mt_dn * p.splits;
  const int nch = __ldg(p.n_chunks);
  const int n_gu = nch * per_gu;
  int q, per;
  if (tile < n_gu) {
    t.is_gu = 1;
    q = tile;
    per = per_gu;
  } else {
    t.is_gu = 0;
    q = tile - n_gu;
    per = per_dn;
  }
  const int c0 = q / per;
  const int2 g = __ldg(p.chunk_grp + c0);  // {first chunk of the expert, chunks of the expert}
  const int r = q - g.x * per;              // position within the expert's tiles
  const int wt = r / g.y;                   // weight tile (gate+up: mt; down: mt * splits + split)
  t.chunk = g.x + r % g.y;
  if (t.is_gu) {
    // unfused: weight tiles (mt, projection) with split = 0 gate / 1 up
    t.mt = p.gu_unfused ? (wt >> 1) : wt;
    t.split = p.gu_unfused ? (wt & 1) : 0;
  } else {
    t.mt = wt / p.splits;
    t.split = wt % p.splits;
  }
  if (p.pair) {
    t.mt = 2 * t.mt + rank;
    t.dummy = t.mt >= (t.is_gu ? p.n_mt_gu : p.n_mt_dn);
  }
  return t;
}

// kPM: 0 single CTAs; 1 and 2 CTA pairs (clusters of two CTAs on one TPC)
// that process the two halves of a pair tile (adjacent weight tiles of the
// same token chunk).  Mode 2 is the default for 256-row token chunks.
//
// kPM == 1 (multicast pairs): each CTA
// streams its own weights, but the shared token k-blocks are loaded ONCE per
// pair: each CTA loads half the 32-row boxes with TMA multicast into both CTAs'
// token slots, and each MMA releases a token slot in both CTAs (multicast
// commit), halving the token traffic per SM.  Rank 0 owns the tile queue and
// hands each pair tile to rank 1 through distributed shared memory.
//
// kPM == 2 (cta_group::2): the pair's two weight tiles form ONE MMA of
// M = 256 issued by rank 0; each CTA stages its own 128 weight rows and HALF
// of the token rows (rank r: rows [r N/2, (r+1) N/2)), so every token byte is
// fetched once per pair with no multicast, and the halved token slots buy a
// deeper weight ring.  Both producers signal rank 0's full barriers; rank 0's
// commits multicast to both CTAs' empty / TMEM-full barriers; both CTAs'
// epilogue warps release rank 0's TMEM-empty barrier.
template <int kBN, int kV, int kPM = 0>
__global__ void __launch_bounds__(kFfnThreads, 1)
ffn_kernel(const __grid_constant__ CUtensorMap tm_wg, const __grid_constant__ CUtensorMap tm_wu,
           const __grid_constant__ CUtensorMap tm_xp, const __grid_constant__ CUtensorMap tm_wd,
           const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ FfnParams p) {
  constexpr bool kPair = kPM != 0;
  constexpr bool k2 = kPM == 2;
  using C = FfnCfg<kBN, kV, k2>;
  const int rank = kPair ? static_cast<int>(cluster_ctarank()) : 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_ring = smem;
  uint8_t* b_ring = smem + C::kAStages * C::kABytes;
  uint8_t* stg = smem + C::kRingBytes;  // epilogue staging buffers
  uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + C::kDataBytes);
  uint64_t* a_empty = a_full + C::kAStages;
  uint64_t* b_full = a_empty + C::kAStages;
  uint64_t* b_empty = b_full + C::kBStages;
  uint64_t* tmem_full = b_empty + C::kBStages;  // [2]: per accumulator slot
  uint64_t* tmem_empty = tmem_full + 2;         // [2]
  uint64_t* sched_full = tmem_empty + 2;
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
    if (p.wd4) tma_prefetch_desc(&p.tm_wd4);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kAStages; ++s) {
      mbar_init(a_full + s, k2 ? 2 : 1);  // k2 (rank 0's): both producers
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < C::kBStages; ++s) {
      mbar_init(b_full + s, k2 ? 2 : 1);
      mbar_init(b_empty + s, kPM == 1 ? 2 : 1);  // pair: both CTAs' MMAs release the shared slot
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tmem_full + s, 1);
      mbar_init(tmem_empty + s, (k2 ? 2 : 1) * kEpiWarps);  // one arrival per epilogue warp (k2: of both CTAs)
    }
    for (int s = 0; s < kSchedSlots; ++s) {
      mbar_init(sched_full + s, 1);
      // MMA lane + one lane per epilogue warp (pair: of both CTAs, plus rank 1's producer)
      mbar_init(sched_empty + s, kPair ? 2 * (1 + kEpiWarps) + 1 : 1 + kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (k2) tmem_alloc2<C::kTmemCols>(tmem_base_smem);
    else tmem_alloc<C::kTmemCols>(tmem_base_smem);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // peer barriers initialised before any remote access
  else __syncthreads();
  tc_fence_after();
  // pair: remote (peer-rank) addresses of the scheduler ring
  const uint32_t peer = static_cast<uint32_t>(rank ^ 1);
  const uint32_t r_sched_empty0 = kPair ? map_to_rank(smem_u32(sched_empty), 0) : 0;  // rank 0's ring
  const uint32_t r_sched_full1 = kPair ? map_to_rank(smem_u32(sched_full), 1) : 0;    // rank 1's ring
  const uint32_t r_sched_tile1 = kPair ? map_to_rank(smem_u32(sched_tile), 1) : 0;
  (void)peer;
  // k2: rank 0's full / TMEM-empty barriers (cluster addresses)
  const uint32_t lead_a_full = k2 ? map_to_rank(smem_u32(a_full), 0) : 0;
  const uint32_t lead_b_full = k2 ? map_to_rank(smem_u32(b_full), 0) : 0;
  const uint32_t lead_tmem_empty = k2 ? map_to_rank(smem_u32(tmem_empty), 0) : 0;
  // consumer side of the scheduler ring: read slot, release it (pair: on rank 0)
  auto sched_read = [&](int slot, uint32_t sphase, bool release_lane, bool warp_sync) -> int {
    if (kPair && rank == 1) mbar_wait_cluster(sched_full + slot, sphase);
    else mbar_wait(sched_full + slot, sphase);
    // (the mbarrier pair orders the slot; the shared atomics also make that
    // visible to compute-sanitizer racecheck, which does not model mbarriers)
    const int t = atomicAdd(sched_tile + slot, 0);
    if (warp_sync) __syncwarp();
    if (release_lane) {
      if (kPair && rank == 1) mbar_arrive_cluster(r_sched_empty0 + slot * 8);
      else mbar_arrive(sched_empty + slot);
    }
    return t;
  };
  const uint32_t tmem_base = *tmem_base_smem;
  // prologue done: wait for the dispatch (chunk table, permuted tokens) to be
  // complete and visible, THEN let the combine grid queue up: the overlapped
  // combine reads prow / topk_w (dispatch and router outputs) without a
  // griddepcontrol.wait of its own, so with MOE_B200_PDL=1 it must not launch
  // before every FFN CTA has seen the dispatch complete
  pdl_wait();
  pdl_launch_dependents();

  const int nch = __ldg(p.n_chunks);
  const int mt_gu_q = kPair ? (p.n_mt_gu + 1) / 2 : p.n_mt_gu;  // queue entries per chunk
  const int mt_dn_q = kPair ? (p.n_mt_dn + 1) / 2 : p.n_mt_dn;
  const int total_tiles = nch * (mt_gu_q * (p.gu_unfused ? 2 : 1) + mt_dn_q * p.splits);
  const int nkb_gu = (p.d + kBK - 1) / kBK;
  const int nkb_dn = (p.f + kBK - 1) / kBK;

  if (warp == 0) {
    // ====================== scheduler + TMA producer ========================
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_t = policy_evict_last();  // k2 token loads: reused by the chunk's tiles
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      int slot = 0;
      uint32_t sphase = 0;
      while (true) {
        int tile;
        if (!kPair || rank == 0) {
          tile = atomicAdd(p.work_counter, 1);
          if (p.trace && tile < total_tiles) {
            p.trace[tile * 8 + 0] = smid();
            p.trace[tile * 8 + 1] = globaltimer();
          }
          const int v = tile < total_tiles ? tile : -1;
          mbar_wait(sched_empty + slot, sphase ^ 1);
          atomicExch(sched_tile + slot, v);
          if constexpr (kPair) {  // hand the pair tile to rank 1 through DSMEM
            st_cluster_u32(r_sched_tile1 + slot * 4, static_cast<uint32_t>(v));
            mbar_arrive_cluster(r_sched_full1 + slot * 8);
          }
          mbar_arrive(sched_full + slot);
        } else {
          tile = sched_read(slot, sphase, true, false);
          if (tile < 0) tile = total_tiles;
        }
        if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
        if (tile >= total_tiles) break;
        const TileInfo ti = decode_tile(p, tile, rank);
        const int4 ch = __ldg(p.chunk_tab + ti.chunk);
        const int n_mma = max(16, (ch.z + 15) & ~15);
        // k2: this CTA's half of the token rows
        const int b_row0 = k2 ? rank * (n_mma / 2) : 0;
        const int b_rows = k2 ? n_mma / 2 : n_mma;
        const int nbox = (b_rows + kBoxRows - 1) / kBoxRows;
        const uint32_t b_bytes = nbox * kBoxRows * kBK * 2;
        // k2, missing second weight tile: stream a valid tile (results discarded)
        const int mt_ld = (k2 && ti.dummy) ? (ti.is_gu ? p.n_mt_gu : p.n_mt_dn) - 1 : ti.mt;
        const int a_col = ti.is_gu ? mt_ld * kBM : mt_ld * 2 * kBM;
        // one 16 KB weight slot: two 64-column boxes
        auto load_a = [&](const CUtensorMap* m, int col, int krow) {
          mbar_wait(a_empty + as, aph ^ 1);
          uint8_t* sa = a_ring + as * C::kABytes;
          if constexpr (k2) {
            const uint32_t bar = lead_a_full + as * 8;
            mbar_arrive_expect_tx_cluster(bar, C::kABytes);
            if (p.w3d) {
              tma_load_3d_2sm(m, bar, sa, 0, krow, col / 64, pol_w);
            } else {
              tma_load_2d_2sm(m, bar, sa, col, krow, pol_w);
              tma_load_2d_2sm(m, bar, sa + C::kABytes / 2, col + 64, krow, pol_w);
            }
          } else {
            mbar_arrive_expect_tx(a_full + as, C::kABytes);
            if (p.w3d) {
              tma_load_3d_hint(m, a_full + as, sa, 0, krow, col / 64, pol_w);
            } else {
              tma_load_2d_hint(m, a_full + as, sa, col, krow, pol_w);
              tma_load_2d_hint(m, a_full + as, sa + C::kABytes / 2, col + 64, krow, pol_w);
            }
          }
          if (++as == C::kAStages) { as = 0; aph ^= 1; }
        };
        // a down tile's two hidden halves: one 32 KB request into two adjacent
        // ring slots (the first slot's full barrier carries the bytes; the MMA
        // waits it before the second, which gets a plain arrival)
        auto load_a_pair = [&](int col, int krow) {
          // (single-CTA tiles only: with cta_group::2 pairs the 32 KB requests measured
          // far slower, Mixtral-512 553 -> 740 us)
          if (!p.wd4 || k2 || as + 1 >= C::kAStages) {
            load_a(&tm_wd, col, krow);
            load_a(&tm_wd, col + kBM, krow);
            return;
          }
          mbar_wait(a_empty + as, aph ^ 1);
          mbar_wait(a_empty + as + 1, aph ^ 1);
          uint8_t* sa = a_ring + as * C::kABytes;
          if constexpr (k2) {
            const uint32_t bar = lead_a_full + as * 8;
            mbar_arrive_expect_tx_cluster(bar, 2 * C::kABytes);
            tma_load_3d_2sm(&p.tm_wd4, bar, sa, 0, krow, col / 64, pol_w);
            mbar_arrive_cluster(lead_a_full + (as + 1) * 8);
          } else {
            mbar_arrive_expect_tx(a_full + as, 2 * C::kABytes);
            tma_load_3d_hint(&p.tm_wd4, a_full + as, sa, 0, krow, col / 64, pol_w);
            mbar_arrive(a_full + as + 1);
          }
          as += 2;
          if (as == C::kAStages) { as = 0; aph ^= 1; }
        };
        int kb0, kb1;
        if (ti.is_gu) {
          kb0 = 0; kb1 = nkb_gu;
        } else {
          kb0 = ti.split * p.kb_per_split;
          kb1 = min(nkb_dn, kb0 + p.kb_per_split);
          if (p.gu_wait) {
            // h rows of this chunk are complete once all its gate+up tiles released
            while (ld_acquire_gpu(p.gu_done + ti.chunk) < p.n_mt_gu * kEpiGroups) __nanosleep(64);
            fence_proxy_async_global();
          }
        }
        if (p.trace) p.trace[tile * 8 + 2] = globaltimer();
        for (int kb = kb0; kb < kb1; ++kb) {
          if (ti.dummy && !k2) {
            // pair mode 1, missing second tile: no weights; still supply this
            // CTA's half of the shared token k-block below
          } else if (ti.is_gu && p.gu_unfused) {
            // one projection per tile: a single weight slot per k-block
            load_a(ti.split ? &tm_wu : &tm_wg, a_col, ch.x * p.d + kb * kBK);
          } else if (ti.is_gu) {
            const int krow = ch.x * p.d + kb * kBK;
            load_a(&tm_wg, a_col, krow);
            load_a(&tm_wu, a_col, krow);
          } else {
            // a down tile is a PAIR of 128-row hidden tiles sharing the token slot
            const int krow = ch.x * p.f + kb * kBK;
            load_a_pair(a_col, krow);
          }
          mbar_wait(b_empty + bs, bph ^ 1);
          uint8_t* sb = b_ring + bs * C::kBBytes;
          const bool tok_rows = ti.is_gu || !p.tiled;
          const CUtensorMap* tb = ti.is_gu ? &tm_xp : &tm_h;
          // token row coordinate of box 0 and the k column within the map
          const int r0 = tok_rows ? ch.y + b_row0 : (kb >> 1) * p.T_pad + ch.w + b_row0;
          const int kc = tok_rows ? kb * kBK : (kb & 1) * kBK;  // tiled h: [f-tile][padded row][128]
          if constexpr (k2) {
            const uint32_t bar = lead_b_full + bs * 8;
            mbar_arrive_expect_tx_cluster(bar, b_bytes);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d_2sm(tb, bar, sb + b * kBoxRows * kBK * 2, kc, r0 + b * kBoxRows, pol_t);
          } else {
            mbar_arrive_expect_tx(b_full + bs, b_bytes);
            for (int b = 0; b < nbox; ++b) {
              if constexpr (kPair) {  // this CTA's half of the boxes, into both CTAs' slot
                if ((b & 1) == rank)
                  tma_load_2d_mc(tb, b_full + bs, sb + b * kBoxRows * kBK * 2, kc, r0 + b * kBoxRows, 3);
              } else {
                tma_load_2d(tb, b_full + bs, sb + b * kBoxRows * kBK * 2, kc, r0 + b * kBoxRows);
              }
            }
          }
          if (++bs == C::kBStages) { bs = 0; bph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    int as = 0, bs = 0;
    uint32_t aph = 0, bph = 0;
    uint32_t eph = 0;          // TMEM-empty phases of the two accumulator slots (bits 0, 1)
    int next_acc = 0;          // accumulator slot of the next narrow tile
    int slot = 0;
    uint32_t sphase = 0;
    while (true) {
      const int tile = sched_read(slot, sphase, lane == 0, true);
      if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
      if (tile < 0) break;
      if (k2 && rank == 1) continue;  // k2: rank 0 issues the pair's MMAs
      const TileInfo ti = decode_tile(p, tile, rank);
      const int4 ch = __ldg(p.chunk_tab + ti.chunk);
      const int n_mma = max(16, (ch.z + 15) & ~15);
      const uint32_t idesc = make_idesc_bf16(k2 ? 2 * kBM : kBM, n_mma, /*a MN-major*/ 1, /*b K-major*/ 0);
      int kb0, kb1;
      if (ti.is_gu) {
        kb0 = 0; kb1 = nkb_gu;
      } else {
        kb0 = ti.split * p.kb_per_split;
        kb1 = min(nkb_dn, kb0 + p.kb_per_split);
      }
      // narrow tile (<= 128 token columns): one accumulator slot, alternating;
      // wide: both slots (its accumulators span 256 columns each)
      const bool narrow = p.tmem_db && n_mma <= 128;
      const int acc_slot = next_acc;
      if (narrow) {
        next_acc ^= 1;
        mbar_wait(tmem_empty + acc_slot, ((eph >> acc_slot) & 1u) ^ 1u);
      } else {
        mbar_wait(tmem_empty, (eph & 1u) ^ 1u);
        mbar_wait(tmem_empty + 1, ((eph >> 1) & 1u) ^ 1u);
      }
      const uint32_t acc_lo = tmem_base + (narrow ? acc_slot * 128u : 0u);
      uint64_t* full_bar = tmem_full + (narrow ? acc_slot : 0);
      tc_fence_after();
      if (p.trace && lane == 0) p.trace[tile * 8 + 5] = globaltimer();
      for (int kb = kb0; kb < kb1; ++kb) {
        if constexpr (!k2) {
          if (ti.dummy) {
            // pair mode 1, missing second tile: consume and release the shared token slot
            mbar_wait(b_full + bs, bph);
            tc_fence_after();
            if (elect_one()) {
              mma_commit_mc(b_empty + bs, 3);
              if (kb == kb1 - 1) {
                mma_commit(full_bar);
                if (!narrow) mma_commit(tmem_full + 1);
              }
            }
            __syncwarp();
            if (++bs == C::kBStages) { bs = 0; bph ^= 1; }
            continue;
          }
        }
        const bool single = ti.is_gu && p.gu_unfused;  // one weight slot, one accumulator
        // (k2: the full barriers complete with the peer's TMA bytes too; the
        // transaction completion makes them visible, a CTA-scope wait suffices)
        auto wait_full = [&](uint64_t* bar, uint32_t ph) { mbar_wait(bar, ph); };
        const int as0 = as;
        wait_full(a_full + as, aph);
        if (++as == C::kAStages) { as = 0; aph ^= 1; }
        const int as1 = as;  // second weight slot: up (gate+up) or hidden rows +128 (down)
        if (!single) {
          wait_full(a_full + as, aph);
          if (++as == C::kAStages) { as = 0; aph ^= 1; }
        }
        wait_full(b_full + bs, bph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa0 = smem_u32(a_ring + as0 * C::kABytes);
          const uint32_t sb = smem_u32(b_ring + bs * C::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t bdesc = make_smem_desc_sw128(sb + kk * 32, 16, 1024);
            const uint64_t adesc0 = make_smem_desc_sw128(sa0 + kk * 2048, C::kABytes / 2, 1024);
            const uint32_t acc = (kb > kb0 || kk > 0) ? 1u : 0u;
            if constexpr (k2) mma_bf16_2sm(acc_lo, adesc0, bdesc, idesc, acc);
            else mma_bf16(acc_lo, adesc0, bdesc, idesc, acc);
            if (!single) {
              const uint32_t sa1 = smem_u32(a_ring + as1 * C::kABytes);
              const uint64_t adesc1 = make_smem_desc_sw128(sa1 + kk * 2048, C::kABytes / 2, 1024);
              if constexpr (k2) mma_bf16_2sm(acc_lo + kAcc2, adesc1, bdesc, idesc, acc);
              else mma_bf16(acc_lo + kAcc2, adesc1, bdesc, idesc, acc);
            }
          }
          if constexpr (k2) {  // release both CTAs' slots; both epilogues start
            mma_commit2_mc(a_empty + as0, 3);
            if (!single) mma_commit2_mc(a_empty + as1, 3);
            mma_commit2_mc(b_empty + bs, 3);
            if (kb == kb1 - 1) {
              mma_commit2_mc(full_bar, 3);
              if (!narrow) mma_commit2_mc(tmem_full + 1, 3);
            }
          } else {
            mma_commit(a_empty + as0);
            if (!single) mma_commit(a_empty + as1);
            if constexpr (kPair) mma_commit_mc(b_empty + bs, 3);  // the slot is shared by the pair
            else mma_commit(b_empty + bs);
            if (kb == kb1 - 1) {
              mma_commit(full_bar);
              if (!narrow) mma_commit(tmem_full + 1);
            }
          }
        }
        __syncwarp();
        if (++bs == C::kBStages) { bs = 0; bph ^= 1; }
      }
      eph ^= narrow ? (1u << acc_slot) : 3u;
    }
  } else if (warp >= 4) {
    // =============================== epilogue ===============================
    const int wq = warp & 3;                 // TMEM lane quadrant
    const int grp = (warp - 4) >> 2;         // chunk group: 32-row chunks q with q % 2 == grp
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const bool issuer = (wq == 0 && lane == 0);  // one bulk-copy issuer per group
    uint8_t* stg_g = stg + grp * C::kStgBytes;
    // accumulator slots: the same narrow / wide sequence as the MMA issuer
    uint32_t fph = 0;  // TMEM-full phases of the two slots (bits 0, 1)
    int next_acc = 0;
    bool narrow = true;
    int acc_slot = 0;
    // release the accumulator: one arrival per warp (k2: on rank 0's barrier)
    auto release_tmem = [&]() {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        for (int s = narrow ? acc_slot : 0; s < (narrow ? acc_slot + 1 : 2); ++s) {
          if constexpr (k2) mbar_arrive_cluster(lead_tmem_empty + s * 8);
          else mbar_arrive(tmem_empty + s);
        }
      }
    };
    int slot = 0;
    uint32_t sphase = 0;
    while (true) {
      const int tile = sched_read(slot, sphase, lane == 0, true);
      if (++slot == kSchedSlots) { slot = 0; sphase ^= 1; }
      if (tile < 0) break;
      const TileInfo ti = decode_tile(p, tile, rank);
      const int4 ch = __ldg(p.chunk_tab + ti.chunk);
      narrow = p.tmem_db && max(16, (ch.z + 15) & ~15) <= 128;
      acc_slot = next_acc;
      if (narrow) {
        next_acc ^= 1;
        mbar_wait(tmem_full + acc_slot, (fph >> acc_slot) & 1u);
        fph ^= 1u << acc_slot;
      } else {
        mbar_wait(tmem_full, fph & 1u);
        mbar_wait(tmem_full + 1, (fph >> 1) & 1u);
        fph ^= 3u;
      }
      const uint32_t acc_lo = tmem_base + (narrow ? acc_slot * 128u : 0u);
      tc_fence_after();
      if (ti.dummy) {  // pair mode, missing second tile: nothing to write
        release_tmem();
        continue;
      }
      if (p.trace && warp == 4 && lane == 0) p.trace[tile * 8 + 4] = globaltimer();
      // Staged store protocol, per 32-row chunk of this group: (issuer) make the
      // staging buffer free -> group barrier -> every thread writes its feature
      // column -> proxy fence -> group barrier -> issuer bulk-copies the rows.
      if (ti.is_gu && p.gu_unfused) {
        // unfused ablation: store the raw fp32 projection (gate or up) tiled
        // [proj][f-tile][padded row][128]; the activation runs in a separate pass
        const int nq = (ch.z + 31) / 32;
        const int my_last = (nq - 1 - grp) >= 0 ? (nq - 1 - ((nq - 1 - grp) % kEpiGroups)) : -1;
        for (int q = grp; q < nq; q += kEpiGroups) {
          const int c0 = q * 32;
          uint32_t a[32];
          tmem_ld_32x32b_x32(acc_lo + lane_base + c0, a);
          tmem_wait_ld();
          if (q == my_last) release_tmem();
          float* sbuf = reinterpret_cast<float*>(stg_g);
          if (issuer) bulk_wait_read<0>();
          epi_bar_sync(grp);
          const int fl = wq * 32 + lane;
#pragma unroll
          for (int c = 0; c < 32; ++c) sbuf[c * kBM + fl] = __uint_as_float(a[c]);
          fence_proxy_async_smem();
          epi_bar_sync(grp);
          if (issuer) {
            const int rows = min(32, ch.z - c0);
            float* dst = p.gu32 + (((size_t)ti.split * p.n_mt_gu + ti.mt) * p.T_pad + ch.w + c0) * kBM;
            bulk_store(dst, sbuf, rows * kBM * 4);
            bulk_commit();
          }
        }
        if (my_last < 0) release_tmem();
        if (issuer) bulk_wait_all();
      } else if (ti.is_gu) {
        const int f0 = ti.mt * kBM;
        const int nvalid_f = min(kBM, p.f - f0);
        // Phase 1 (TMEM critical path): drain both accumulators, apply SiLU(g)*u and
        // keep h as packed bf16 pairs in registers, then release TMEM so the next
        // tile's MMAs start while this tile's h is still being written out.
        constexpr int kMaxChunks = kBN / 32 / kEpiGroups;
        uint32_t hp[kMaxChunks][16];
#pragma unroll
        for (int qq = 0; qq < kMaxChunks; ++qq) {
          const int q = qq * kEpiGroups + grp;
          if (q * 32 < ch.z) {
            uint32_t g[32], u[32];
            tmem_ld_32x32b_x32(acc_lo + lane_base + q * 32, g);
            tmem_ld_32x32b_x32(acc_lo + lane_base + kAcc2 + q * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float h0 = silu_mul(__uint_as_float(g[2 * i]), __uint_as_float(u[2 * i]));
              const float h1 = silu_mul(__uint_as_float(g[2 * i + 1]), __uint_as_float(u[2 * i + 1]));
              __nv_bfloat162 pk = __floats2bfloat162_rn(h0, h1);
              hp[qq][i] = *reinterpret_cast<uint32_t*>(&pk);
            }
          }
        }
        release_tmem();
        if (p.trace && warp == 4 && lane == 0) p.trace[tile * 8 + 6] = globaltimer();
        // Phase 2: stage 32-row chunks in smem and bulk-copy them out.
        const int fl = wq * 32 + lane;  // feature within the tile
#pragma unroll
        for (int qq = 0; qq < kMaxChunks; ++qq) {
          const int q = qq * kEpiGroups + grp;
          const int c0 = q * 32;
          if (c0 < ch.z) {
            __nv_bfloat16* sbuf = reinterpret_cast<__nv_bfloat16*>(stg_g);
            if (issuer) bulk_wait_read<0>();
            epi_bar_sync(grp);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t w = hp[qq][i];
              reinterpret_cast<uint16_t*>(sbuf)[(2 * i) * kBM + fl] = static_cast<uint16_t>(w & 0xFFFFu);
              reinterpret_cast<uint16_t*>(sbuf)[(2 * i + 1) * kBM + fl] = static_cast<uint16_t>(w >> 16);
            }
            fence_proxy_async_smem();
            epi_bar_sync(grp);
            if (issuer) {
              const int rows = min(32, ch.z - c0);
              if (p.tiled) {
                // one contiguous block: rows x 128 features of this f-tile
                bulk_store(p.h + ((size_t)ti.mt * p.T_pad + ch.w + c0) * kBM, sbuf, rows * kBM * 2);
              } else {
                for (int c = 0; c < rows; ++c)
                  bulk_store(p.h + (size_t)(ch.y + c0 + c) * p.f + f0, sbuf + c * kBM, nvalid_f * 2);
              }
              bulk_commit();
            }
          }
        }
        if (p.gu_wait && issuer) {
          // publish this group's h rows: bulk writes complete, then one release increment
          bulk_wait_all();
          fence_proxy_async_global();
          __threadfence();
          red_release_gpu_add(p.gu_done + ti.chunk, 1);
        }
      } else {
        // down tile: two 128-row halves; 32-row chunks alternate between the groups
        const int nq = (ch.z + 31) / 32;
        // overlapped combine: tokens of this group's rows (lane: row q * 32 + lane
        // of each of the group's chunks q), loaded now, used after the stores
        constexpr int kRowsPerLane = kBN / 32 / kEpiGroups;
        int arr_tok[kRowsPerLane];
#pragma unroll
        for (int i = 0; i < kRowsPerLane; ++i) {
          const int c = (grp + kEpiGroups * i) * 32 + lane;
          arr_tok[i] = (p.arrive && wq == 0 && c < ch.z) ? __ldg(p.fwd + ch.y + c) / p.k : -1;
        }
        const int my_last = (nq - 1 - grp) >= 0 ? (nq - 1 - ((nq - 1 - grp) % kEpiGroups)) : -1;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int d0 = ti.mt * 2 * kBM + half * kBM;
          const int nvalid_d = min(kBM, p.d - d0);
          for (int q = grp; q < nq; q += kEpiGroups) {
            const int c0 = q * 32;
            uint32_t a[32];
            tmem_ld_32x32b_x32(acc_lo + lane_base + half * kAcc2 + c0, a);
            tmem_wait_ld();
            if (half == 1 && q == my_last) release_tmem();
            float* sbuf = reinterpret_cast<float*>(stg_g);
            if (issuer) bulk_wait_read<0>();
            epi_bar_sync(grp);
            const int fl = wq * 32 + lane;
#pragma unroll
            for (int c = 0; c < 32; ++c) sbuf[c * kBM + fl] = __uint_as_float(a[c]);
            fence_proxy_async_smem();
            epi_bar_sync(grp);
            if (p.tiled) {
              // one contiguous block in ys[split][d-pair][half][padded row][128]
              if (issuer) {
                const int rows = min(32, ch.z - c0);
                float* dst = p.ys + ((((size_t)ti.split * p.n_mt_dn + ti.mt) * 2 + half) * p.T_pad + ch.w + c0) * kBM;
                bulk_store(dst, sbuf, rows * kBM * 4);
                bulk_commit();
              }
            } else if (wq == 0 && nvalid_d > 0) {
              // lane c looks up row c's expanded slot; lane 0 issues all copies (scatter)
              const int rows = min(32, ch.z - c0);
              // expanded slot of row c (fwd == null: the grouped-GEMM stage, rows stay in place)
              const int xid = lane < rows ? (p.fwd ? __ldg(p.fwd + ch.y + c0 + lane) : ch.y + c0 + lane) : 0;
              if (p.scale_by_w && lane < rows) {
                const float w = __ldg(p.topk_w + xid);
                for (int qv = 0; qv < kBM; ++qv) sbuf[lane * kBM + qv] = __fmul_rn(sbuf[lane * kBM + qv], w);
                fence_proxy_async_smem();
              }
              __syncwarp();
              for (int c = 0; c < rows; ++c) {
                const int xc = __shfl_sync(0xffffffffu, xid, c);
                if (lane == 0) bulk_store(p.ys + (size_t)xc * p.d + d0, sbuf + c * kBM, nvalid_d * 4);
              }
              if (lane == 0) bulk_commit();
            }
          }
        }
        if (my_last < 0) release_tmem();  // this group had no chunk: still release TMEM
        if (issuer) bulk_wait_all();
        if (p.arrive && p.tiled && wq == 0) {
          // publish this group's partial rows to the overlapped combine: the
          // issuer (lane 0) waited for its bulk writes above; proxy + gpu
          // fences, then one relaxed arrival per row (the fence orders them)
          if (lane == 0) {
            fence_proxy_async_global();
            __threadfence();
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < kRowsPerLane; ++i) {
            if (arr_tok[i] >= 0) atomicAdd(p.arrive + (size_t)arr_tok[i] * p.n_mt_dn + ti.mt, 1);
          }
        }
      }
      if (p.trace && warp == 4 && lane == 0) p.trace[tile * 8 + 3] = globaltimer();
    }
  }

  if ((warp == 4 || warp == 8) && lane == 0) bulk_wait_all();
  tc_fence_before();
  // pair: neither CTA leaves while its peer may still multicast into its
  // shared memory or arrive on its barriers
  if constexpr (kPair) cluster_sync_all();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (k2) tmem_dealloc2<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
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
