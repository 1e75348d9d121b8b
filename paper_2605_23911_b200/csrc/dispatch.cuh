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
constexpr int kDispRows = 8;  // expanded rows per CTA

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

template <bool kXBf16>
__global__ void __launch_bounds__(kDispThreads) dispatch_kernel(const DispatchParams p) {
  extern __shared__ __align__(16) int32_t dsm[];
  int32_t* tot = dsm;                  // [E]
  int32_t* before = tot + p.E;         // [E]
  int32_t* off = before + p.E;         // [E+1]
  int32_t* off16 = off + p.E + 1;      // [E+1]
  int32_t* cpre = off16 + p.E + 1;     // [E+1]
  __shared__ int32_t s_pos[kDispRows], s_tok[kDispRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * kDispRows;
  const int r1 = min(p.T, r0 + kDispRows);

  for (int e = tid; e < p.E; e += kDispThreads) {
    tot[e] = 0;
    before[e] = 0;
  }
  // the gather sources (token i / k) are known now: put the first batch of row
  // loads in flight before the histogram, store them once positions are known
  const int vpr = p.d / 8;
  const int nvec = (r1 - r0) * vpr;
  constexpr int kPre = 8;
  int4 pre[kPre];
  if (p.xp != nullptr) {
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int v = tid + u * kDispThreads;
      if (v < nvec) pre[u] = load_bf16x8<kXBf16>(p.x, (size_t)((r0 + v / vpr) / p.k), p.d, v % vpr);
    }
  }
  pdl_launch_dependents();
  pdl_wait();  // routing indices of the router grid
  __syncthreads();
  // histogram of all rows and of the rows before r0 (warp-aggregated smem
  // atomics); four index loads in flight per thread
  constexpr int U = 4;
  for (int base0 = warp * 32; base0 < p.T; base0 += U * kDispThreads) {
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
  // exclusive scans: offsets, 16-aligned padded offsets, chunk counts (warp 0)
  if (warp == 0) {
    const int per = (p.E + 31) / 32;
    const int lo = lane * per, hi = min(p.E, lo + per);
    int sc = 0, s16 = 0, sch = 0;
    for (int e = lo; e < hi; ++e) {
      const int n = tot[e];
      sc += n;
      s16 += (n + 15) & ~15;
      sch += (n + p.chunk_rows - 1) / p.chunk_rows;
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
    for (int e = lo; e < hi; ++e) {
      off[e] = rc; off16[e] = r16; cpre[e] = rch;
      const int n = tot[e];
      rc += n;
      r16 += (n + 15) & ~15;
      rch += (n + p.chunk_rows - 1) / p.chunk_rows;
    }
    if (lane == 31) { off[p.E] = ic; off16[p.E] = i16; cpre[p.E] = ich; }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int e = tid; e < p.E; e += kDispThreads) {
      p.counts[e] = tot[e];
      p.offsets[e] = off[e];
      const int n = tot[e];
      const int nch_e = (n + p.chunk_rows - 1) / p.chunk_rows;
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
  // stable positions of this CTA's rows (one warp; kDispRows <= 32)
  if (warp == 0) {
    const int i = r0 + lane;
    const bool valid = lane < kDispRows && i < r1;
    int e = valid ? __ldg(p.topk_idx + i) : -1 - lane;
    if (e < 0 || e >= p.E) e = -1 - lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    if (valid && e >= 0) {
      const int rank = before[e] + __popc(peers & ((1u << lane) - 1u));
      const int pos = off[e] + rank;
      p.fwd[pos] = i;
      p.inv[i] = pos;
      p.prow[i] = off16[e] + rank;
      s_pos[lane] = pos;
      s_tok[lane] = i / p.k;
    } else if (valid) {  // dropped (out-of-range override index): in-bounds placeholders
      p.inv[i] = -1;
      p.prow[i] = 0;
      s_pos[lane] = -1;
      s_tok[lane] = i / p.k;
    }
  }
  if (p.xp == nullptr) return;
  __syncthreads();
  // gather: xp[pos(i)] = bf16(x[i / k]), 16-byte vectors
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const int v = tid + u * kDispThreads;
    if (v < nvec && s_pos[v / vpr] >= 0) reinterpret_cast<int4*>(p.xp + (size_t)s_pos[v / vpr] * p.d)[v % vpr] = pre[u];
  }
  for (int v0 = tid + kPre * kDispThreads; v0 < nvec; v0 += U * kDispThreads) {
    int4 out[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // all loads first: U vectors in flight per thread
      const int v = v0 + u * kDispThreads;
      if (v < nvec) out[u] = load_bf16x8<kXBf16>(p.x, (size_t)s_tok[v / vpr], p.d, v % vpr);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * kDispThreads;
      if (v < nvec && s_pos[v / vpr] >= 0) reinterpret_cast<int4*>(p.xp + (size_t)s_pos[v / vpr] * p.d)[v % vpr] = out[u];
    }
  }
}

}  // namespace moe
