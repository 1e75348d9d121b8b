// dispatch.cuh — scheduler + permute in one fully parallel launch
// (scheduler.py:78-117 and pipeline.py:165-183).
//
// Each CTA owns kDispRows consecutive expanded rows i = t*k + j (id order).
// It streams all T routing indices (L2-resident, <= 128 KB) once and builds in
// shared memory
//   tot[e]    = #rows routed to e                   (expert_histogram, :78-82)
//   before[e] = #rows i' < r0 routed to e
// so the stable expert-major position of each of its rows is
//   pos(i) = off[e] + before[e] + #{i' in [r0, i) : idx[i'] = e}
// (argsort(kind="stable"), :97-103; off = exclusive scan of tot, :85-94).
// No CTA waits for another: there is no serial scheduler section.  CTA 0 also
// writes counts, offsets, and the FFN chunk table (the device form of
// build_block_schedule, :106-117).  With xp != nullptr it gathers its rows:
// xp[pos(i)] = bf16(x[i / k])  (pipeline.py:182, fused fp32 -> bf16 cast).
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kDispThreads = 256;
constexpr int kDispRows = 8;         // expanded rows per CTA
constexpr int kDispSmemT = 8192;     // up to this many rows, every CTA stages all indices in smem

struct DispatchParams {
  const int32_t* topk_idx;  // (T) expert of expanded row i = t*k + j
  int T, k, E, d;
  int chunk_rows;           // FFN chunk cap (BN)
  const void* x;            // (B, d) fp32 or bf16 (gather source), may be null
  __nv_bfloat16* xp;        // (T, d) permuted tokens, null: no gather
  int32_t* counts;          // (E)
  int32_t* offsets;         // (E+1)
  int32_t* fwd;             // (T) permuted row -> expanded id
  int32_t* inv;             // (T) expanded id -> permuted row
  int32_t* prow;            // (T) expanded id -> padded permuted row (experts start 16-aligned)
  int4* chunk_tab;          // {expert, row0, nrows, padded row0}
  int2* chunk_grp;          // {first chunk of the expert, chunks of the expert}
  int32_t* n_chunks;        // [1]
  uint32_t* flags;          // bit 4: an index outside [0, E) (row dropped)
  // overlapped combine (elementwise.cuh combine_flag_kernel): a dropped row
  // pre-arrives on its token's counters with its S splits
  int32_t* tok_cnt;         // (B, n_dp) or null
  int n_dp, splits;
  unsigned long long* trace;  // debug: 16 u64 per CTA (globaltimer start, clock64 phase deltas)
};

template <bool kXBf16>
MOE_DEVICE int4 load_bf16x8(const void* x, size_t t, int d, int q) {
  if (kXBf16) return __ldg(reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(x) + t * d) + q);
  const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(x) + t * d) + 2 * q;
  const float4 a = __ldg(src), b = __ldg(src + 1);
  __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
  __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
  int4 out;
  out.x = *reinterpret_cast<int*>(&h0);
  out.y = *reinterpret_cast<int*>(&h1);
  out.z = *reinterpret_cast<int*>(&h2);
  out.w = *reinterpret_cast<int*>(&h3);
  return out;
}

// kSmemIdx (T <= kDispSmemT): all T indices are staged in shared memory with
// one round of 16-byte loads and counted with plain shared atomics; the CTA's
// own rows read their experts from that copy.  Otherwise they are streamed
// (four loads in flight per thread, warp-aggregated atomics).
template <bool kXBf16, bool kSmemIdx>
__global__ void __launch_bounds__(kDispThreads) dispatch_kernel(const DispatchParams p) {
  extern __shared__ __align__(16) int32_t dsm[];
  int32_t* tot = dsm;                  // [E]
  int32_t* before = tot + p.E;         // [E]
  int32_t* off = before + p.E;         // [E+1]
  int32_t* off16 = off + p.E + 1;      // [E+1]
  int32_t* cpre = off16 + p.E + 1;     // [E+1]
  int32_t* idx_s = dsm + ((5 * p.E + 3 + 3) & ~3);  // [T] (kSmemIdx), 16-byte aligned
  __shared__ int32_t s_pos[kDispRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * kDispRows;
  const int r1 = min(p.T, r0 + kDispRows);
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  const long long c_start = clock64();
  auto stamp = [&](int i) { if (tr && threadIdx.x == 0) tr[i] = clock64() - c_start; };
  if (tr && tid == 0) { tr[0] = globaltimer_ns(); tr[15] = smid_u32(); }

  for (int e = tid; e < p.E; e += kDispThreads) {
    tot[e] = 0;
    before[e] = 0;
  }
  // gather: warp w copies expanded row r0 + w (token (r0 + w) / k).  The
  // sources are known now: put the first loads of the row in flight before the
  // histogram, store them once the positions are known
  static_assert(kDispRows == kDispThreads / 32, "one warp per gathered row");
  const int vpr = p.d / 8;                 // 16-byte vectors per row
  const bool has_row = r0 + warp < r1;
  const int src_tok = (r0 + warp) / p.k;
  constexpr int kPre = 8;
  int4 pre[kPre];
  if (p.xp != nullptr && has_row) {
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int q = lane + 32 * u;
      if (q < vpr) pre[u] = load_bf16x8<kXBf16>(p.x, (size_t)src_tok, p.d, q);
    }
  }
  pdl_launch_dependents();
  pdl_wait();  // routing indices of the router grid
  constexpr int U = 4;
  if (kSmemIdx) {
    if ((reinterpret_cast<uintptr_t>(p.topk_idx) & 15) == 0) {
      const int nv = p.T >> 2;
#pragma unroll 4
      for (int v = tid; v < nv; v += kDispThreads)
        reinterpret_cast<int4*>(idx_s)[v] = __ldg(reinterpret_cast<const int4*>(p.topk_idx) + v);
      for (int i = 4 * nv + tid; i < p.T; i += kDispThreads) idx_s[i] = __ldg(p.topk_idx + i);
    } else {
#pragma unroll 4
      for (int i = tid; i < p.T; i += kDispThreads) idx_s[i] = __ldg(p.topk_idx + i);
    }
  }
  __syncthreads();
  stamp(1);
  if (kSmemIdx) {
    // histogram of all rows and of the rows before r0 (shared atomics)
    for (int i = tid; i < p.T; i += kDispThreads) {
      const int e = idx_s[i];
      if (e < 0 || e >= p.E) {  // routing override out of range: drop the row
        if (blockIdx.x == 0 && p.flags) atomicOr(p.flags, 4u);
        continue;
      }
      atomicAdd(&tot[e], 1);
      if (i < r0) atomicAdd(&before[e], 1);
    }
  }
  // histogram of all rows and of the rows before r0 (warp-aggregated smem
  // atomics); four index loads in flight per thread
  for (int base0 = warp * 32; !kSmemIdx && base0 < p.T; base0 += U * kDispThreads) {
    int ev[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base0 + u * kDispThreads + lane;
      ev[u] = i < p.T ? __ldg(p.topk_idx + i) : -1 - lane;
      if (i < p.T && (ev[u] < 0 || ev[u] >= p.E)) {  // routing override out of range: drop the row
        if (blockIdx.x == 0 && p.flags) atomicOr(p.flags, 4u);
        ev[u] = -1 - lane;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base0 + u * kDispThreads + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, ev[u]);
      const uint32_t peers_before = peers & __ballot_sync(0xffffffffu, i < r0);
      if (i < p.T && ev[u] >= 0 && (__ffs(peers) - 1) == lane) {
        atomicAdd(&tot[ev[u]], __popc(peers));
        if (peers_before) atomicAdd(&before[ev[u]], __popc(peers_before));
      }
    }
  }
  __syncthreads();
  stamp(2);
  // exclusive scans: offsets, 16-aligned padded offsets, chunk counts (warp 0)
  // (cold code, run once per CTA: kept small -- instruction fetch, not
  // arithmetic, bounds these short phases; chunk_rows is a power of two)
  const int cshift = __ffs(p.chunk_rows) - 1;
  if (warp == 0) {
    const int per = (p.E + 31) / 32;
    const int lo = lane * per, hi = min(p.E, lo + per);
    int sc = 0, s16 = 0, sch = 0;
#pragma unroll 1
    for (int e = lo; e < hi; ++e) {
      const int n = tot[e];
      sc += n;
      s16 += (n + 15) & ~15;
      sch += (n + p.chunk_rows - 1) >> cshift;
    }
    int ic = sc, i16 = s16, ich = sch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ic, o);
      const int b = __shfl_up_sync(0xffffffffu, i16, o);
      const int c = __shfl_up_sync(0xffffffffu, ich, o);
      if (lane >= o) { ic += a; i16 += b; ich += c; }
    }
    int rc = ic - sc, r16 = i16 - s16, rch = ich - sch;
#pragma unroll 1
    for (int e = lo; e < hi; ++e) {
      off[e] = rc; off16[e] = r16; cpre[e] = rch;
      const int n = tot[e];
      rc += n;
      r16 += (n + 15) & ~15;
      rch += (n + p.chunk_rows - 1) >> cshift;
    }
    if (lane == 31) { off[p.E] = ic; off16[p.E] = i16; cpre[p.E] = ich; }
  }
  stamp(6);
  __syncthreads();
  stamp(7);
  if (blockIdx.x == 0) {
#pragma unroll 1
    for (int e = tid; e < p.E; e += kDispThreads) {
      p.counts[e] = tot[e];
      p.offsets[e] = off[e];
      const int n = tot[e];
      const int nch_e = (n + p.chunk_rows - 1) >> cshift;
#pragma unroll 1
      for (int c = 0; c < nch_e; ++c) {
        const int rr = c * p.chunk_rows;
        p.chunk_tab[cpre[e] + c] = make_int4(e, off[e] + rr, min(p.chunk_rows, n - rr), off16[e] + rr);
        p.chunk_grp[cpre[e] + c] = make_int2(cpre[e], nch_e);
      }
    }
    if (tid == 0) {
      p.offsets[p.E] = off[p.E];
      p.n_chunks[0] = cpre[p.E];
    }
  }
  stamp(8);
  // stable positions of this CTA's rows (one warp; kDispRows <= 32)
  if (warp == 0) {
    const int i = r0 + lane;
    const bool valid = lane < kDispRows && i < r1;
    int e = valid ? (kSmemIdx ? idx_s[i] : __ldg(p.topk_idx + i)) : -1 - lane;
    if (e < 0 || e >= p.E) e = -1 - lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    if (valid && e >= 0) {
      const int rank = before[e] + __popc(peers & ((1u << lane) - 1u));
      const int pos = off[e] + rank;
      p.fwd[pos] = i;
      p.inv[i] = pos;
      p.prow[i] = off16[e] + rank;
      s_pos[lane] = pos;
    } else if (valid) {  // dropped (out-of-range override index): no permuted row
      p.inv[i] = -1;
      p.prow[i] = -1;
      s_pos[lane] = -1;
      if (p.tok_cnt) {  // the overlapped combine counts this slot's S partials as arrived
        const int t = i / p.k;
        for (int mt = 0; mt < p.n_dp; ++mt) atomicAdd(p.tok_cnt + (size_t)t * p.n_dp + mt, p.splits);
      }
    }
  }
  stamp(3);
  if (p.xp == nullptr) return;
  __syncthreads();
  stamp(4);
  // gather: xp[pos(i)] = bf16(x[i / k]), 16-byte vectors, warp w -> row r0 + w
  const int dst_row = has_row ? s_pos[warp] : -1;
  if (dst_row >= 0) {
    int4* dst = reinterpret_cast<int4*>(p.xp + (size_t)dst_row * p.d);
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int q = lane + 32 * u;
      if (q < vpr) dst[q] = pre[u];
    }
#pragma unroll 1
    for (int q0 = lane + 32 * kPre; q0 < vpr; q0 += 32 * U) {
      int4 out[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads first: U vectors in flight per lane
        const int q = q0 + 32 * u;
        if (q < vpr) out[u] = load_bf16x8<kXBf16>(p.x, (size_t)src_tok, p.d, q);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + 32 * u;
        if (q < vpr) dst[q] = out[u];
      }
    }
  }
  __syncthreads();
  stamp(5);
}

// Small-batch dispatch inside the router (T = B*k <= kFuseMaxT rows): run
// by the last router CTA to finish phase 2 once every routing index is
// written (router_seg_kernel, fuse_dispatch), so the forward has no separate
// dispatch launch at decode-like batch sizes.  Same outputs as
// dispatch_kernel: counts, offsets, stable permutation (fwd, inv, padded
// rows), the FFN chunk table and the bf16 gather of the T rows.  sm: at least
// 4E + 3 + 2 kFuseMaxT ints of shared memory.
constexpr int kFuseMaxT = 16;

template <bool kXBf16>
MOE_DEVICE void dispatch_small_cta(const int32_t* topk_idx, int T, int k, int E, int d, int chunk_rows,
                                   const void* x, __nv_bfloat16* xp, int32_t* counts, int32_t* offsets,
                                   int32_t* fwd, int32_t* inv, int32_t* prow, int4* chunk_tab, int2* chunk_grp,
                                   int32_t* n_chunks, int32_t* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  int32_t* tot = sm;
  int32_t* off = tot + E;
  int32_t* off16 = off + E + 1;
  int32_t* cpre = off16 + E + 1;
  int32_t* idx_s = cpre + E + 1;
  int32_t* pos_s = idx_s + kFuseMaxT;
#pragma unroll 1
  for (int e = tid; e < E; e += blockDim.x) tot[e] = 0;
  if (tid < T) idx_s[tid] = __ldcg(topk_idx + tid);  // other CTAs' phase-2 writes: through L2
  __syncthreads();
  if (tid < T) atomicAdd(&tot[idx_s[tid]], 1);  // (router indices are in [0, E))
  __syncthreads();
  const int cshift = __ffs(chunk_rows) - 1;
  if (warp == 0) {  // exclusive scans (as dispatch_kernel)
    const int per = (E + 31) / 32;
    const int lo = lane * per, hi = min(E, lo + per);
    int sc = 0, s16 = 0, sch = 0;
#pragma unroll 1
    for (int e = lo; e < hi; ++e) {
      const int n = tot[e];
      sc += n;
      s16 += (n + 15) & ~15;
      sch += (n + chunk_rows - 1) >> cshift;
    }
    int ic = sc, i16 = s16, ich = sch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ic, o);
      const int b = __shfl_up_sync(0xffffffffu, i16, o);
      const int c = __shfl_up_sync(0xffffffffu, ich, o);
      if (lane >= o) { ic += a; i16 += b; ich += c; }
    }
    int rc = ic - sc, r16 = i16 - s16, rch = ich - sch;
#pragma unroll 1
    for (int e = lo; e < hi; ++e) {
      off[e] = rc; off16[e] = r16; cpre[e] = rch;
      const int n = tot[e];
      rc += n;
      r16 += (n + 15) & ~15;
      rch += (n + chunk_rows - 1) >> cshift;
    }
    if (lane == 31) { off[E] = ic; off16[E] = i16; cpre[E] = ich; }
  }
  __syncthreads();
#pragma unroll 1
  for (int e = tid; e < E; e += blockDim.x) {
    counts[e] = tot[e];
    offsets[e] = off[e];
    const int n = tot[e];
    const int nch_e = (n + chunk_rows - 1) >> cshift;
#pragma unroll 1
    for (int c = 0; c < nch_e; ++c) {
      const int rr = c * chunk_rows;
      chunk_tab[cpre[e] + c] = make_int4(e, off[e] + rr, min(chunk_rows, n - rr), off16[e] + rr);
      chunk_grp[cpre[e] + c] = make_int2(cpre[e], nch_e);
    }
  }
  if (tid == 0) {
    offsets[E] = off[E];
    n_chunks[0] = cpre[E];
  }
  if (tid < T) {  // stable rank among the earlier rows of the same expert (scheduler.py:97-103)
    const int e = idx_s[tid];
    int rank = 0;
#pragma unroll 1
    for (int i = 0; i < tid; ++i) rank += idx_s[i] == e;
    const int pos = off[e] + rank;
    fwd[pos] = tid;
    inv[tid] = pos;
    prow[tid] = off16[e] + rank;
    pos_s[tid] = pos;
  }
  if (xp == nullptr) return;
  __syncthreads();
  const int vpr = d / 8;  // 16-byte vectors per row
#pragma unroll 1
  for (int i = warp; i < T; i += nwarps) {
    int4* dst = reinterpret_cast<int4*>(xp + (size_t)pos_s[i] * d);
    const int t = i / k;
#pragma unroll 1
    for (int q0 = lane; q0 < vpr; q0 += 32 * 4) {
      int4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + 32 * u < vpr) v[u] = load_bf16x8<kXBf16>(x, (size_t)t, d, q0 + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + 32 * u < vpr) dst[q0 + 32 * u] = v[u];
    }
  }
}

}  // namespace moe
