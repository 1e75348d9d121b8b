// ep_p2p.cuh — expert-parallel exchanges over peer memory.
//
// Every rank's exchange buffers are mapped into every other rank's address
// space (NVLink P2P on a node; CUDA IPC handles), so the data path writes rows
// straight into the destination rank's buffer instead of staging them for a
// library all-to-all:
//   1. counts all-gather   every rank writes its per-expert row counts into
//                          counts[me][:] of every rank;
//   2. dispatch            rows go straight from the local permuted order into
//                          the destination's expert-major receive buffer, at
//                          the position the single-GPU permutation would give
//                          them (experts ascending, then source rank, then the
//                          source's stable order), with their {source, expanded
//                          id}; fused with the local gather x[id / k];
//   3. return              every received row's expert output goes back into
//                          its home rank's buffer at its expanded id.
// Each step publishes with a system-scope fence and a release store of an
// epoch counter (one flag per source); consumers acquire-spin on the flags.
// Epochs only grow, so nothing is ever reset.
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kEpMaxRanks = 16;
constexpr int kEpFlagSets = 3;  // counts, rows, returns

struct EpPeers {
  int32_t* counts[kEpMaxRanks];              // rank r: [n][E] counts[src][e]
  unsigned long long* flags[kEpMaxRanks];    // rank r: [3][n] epoch flags per source
  __nv_bfloat16* rows[kEpMaxRanks];          // rank r: [R_max][d] expert-major received rows
  int2* ids[kEpMaxRanks];                    // rank r: [R_max] {source rank, expanded id}
  float* home[kEpMaxRanks];                  // rank r: [T_max][d] returned outputs by expanded id
  int expert_lo[kEpMaxRanks + 1];            // rank r owns experts [lo[r], lo[r+1])
  int n, me;
  unsigned long long* epoch_dev;             // local {counter, current}: device epochs (launch epoch 0)
};

// The epoch of this forward: the launch argument, or (0) the device-side one
// that ep_counts_kernel advanced -- so a captured CUDA graph replays correctly.
MOE_DEVICE unsigned long long ep_epoch(const EpPeers& P, unsigned long long epoch) {
  return epoch ? epoch : *reinterpret_cast<volatile unsigned long long*>(P.epoch_dev + 1);
}

MOE_DEVICE void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
MOE_DEVICE unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 of the CTA waits until flags[0 .. n) >= epoch, then the CTA proceeds
MOE_DEVICE void ep_wait_all(const unsigned long long* flags, int n, unsigned long long epoch) {
  if (threadIdx.x == 0)
    for (int s = 0; s < n; ++s)
      while (ld_acquire_sys_u64(flags + s) < epoch) __nanosleep(256);
  __syncthreads();
}
MOE_DEVICE int ep_owner(const EpPeers& P, int e) {
  int r = 0;
  while (r + 1 < P.n && e >= P.expert_lo[r + 1]) ++r;
  return r;
}

// 1. counts all-gather (one CTA): local histogram of the routing, written
// into every rank's counts[me][:], then flag set 0.
__global__ void __launch_bounds__(256) ep_counts_kernel(const int32_t* __restrict__ topk_idx, int T, int E,
                                                        EpPeers P, unsigned long long epoch) {
  extern __shared__ int32_t hist[];
  if (epoch == 0) {  // device epochs: this forward's = counter + 1 (the first kernel of the forward)
    __shared__ unsigned long long s_ep;
    if (threadIdx.x == 0) {
      s_ep = P.epoch_dev[0] + 1;
      P.epoch_dev[0] = s_ep;
      P.epoch_dev[1] = s_ep;
    }
    __syncthreads();
    epoch = s_ep;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const int e = __ldg(topk_idx + i);
    if (e >= 0 && e < E) atomicAdd(&hist[e], 1);
  }
  __syncthreads();
  for (int r = 0; r < P.n; ++r)
    for (int e = threadIdx.x; e < E; e += blockDim.x) P.counts[r][(size_t)P.me * E + e] = hist[e];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < P.n; ++r) st_release_sys_u64(P.flags[r] + 0 * P.n + P.me, epoch);
}

// wait until every source's flag of `set` reached `epoch` (one thread)
__global__ void ep_wait_kernel(EpPeers P, int set, unsigned long long epoch) {
  ep_wait_all(P.flags[P.me] + (size_t)set * P.n, P.n, ep_epoch(P, epoch));
}

// 2. dispatch: local permuted row p (expert-major, stable) -> destination.
// x is bf16 (B, d); counts of every source are in this rank's counts buffer.
__global__ void __launch_bounds__(256) ep_dispatch_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const int32_t* __restrict__ topk_idx,
                                                          const int32_t* __restrict__ fwd,
                                                          const int32_t* __restrict__ offsets, int T, int k,
                                                          int E, int d, EpPeers P, int32_t* done_counter,
                                                          unsigned long long epoch) {
  extern __shared__ int32_t ep_sm[];
  int32_t* dest0 = ep_sm;  // [E]: destination row of this source's first row of expert e
  const int32_t* cnt = P.counts[P.me];
  epoch = ep_epoch(P, epoch);
  ep_wait_all(P.flags[P.me] + 0 * P.n, P.n, epoch);
  // dest0[e] = (rows of the owner's experts before e, all sources) + (rows of e
  //            from sources before me)
  if (threadIdx.x == 0) {
    int r = 0, run = 0;
    for (int e = 0; e < E; ++e) {
      while (r + 1 < P.n && e >= P.expert_lo[r + 1]) { ++r; run = 0; }
      int tot = 0, pre = 0;
      for (int s = 0; s < P.n; ++s) {
        const int c = __ldcg(cnt + (size_t)s * E + e);
        tot += c;
        if (s < P.me) pre += c;
      }
      dest0[e] = run + pre;
      run += tot;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nwarps = gridDim.x * (blockDim.x / 32);
  const int vpr = d / 8;  // 16-byte vectors per row
  for (int p = blockIdx.x * (blockDim.x / 32) + warp; p < T; p += nwarps) {
    const int xid = __ldg(fwd + p);
    const int e = __ldg(topk_idx + xid);
    const int rnk = p - __ldg(offsets + e);
    const int r = ep_owner(P, e);
    const int pos = dest0[e] + rnk;
    const int4* src = reinterpret_cast<const int4*>(x + (size_t)(xid / k) * d);
    int4* dst = reinterpret_cast<int4*>(P.rows[r] + (size_t)pos * d);
    for (int q = lane; q < vpr; q += 32) dst[q] = __ldg(src + q);
    if (lane == 0) P.ids[r][pos] = make_int2(P.me, xid);
  }
  // publish: the last CTA to finish signals every destination
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(done_counter, 1);
    if (prev == static_cast<int>(gridDim.x) - 1) {
      __threadfence_system();
      *done_counter = 0;
      for (int r = 0; r < P.n; ++r) st_release_sys_u64(P.flags[r] + 1 * P.n + P.me, epoch);
    }
  }
}

// 3. return: received row p's expert output (fp32, local) -> home rank's
// home[xid]; flag set 2 of every source once all rows are out.
__global__ void __launch_bounds__(256) ep_return_kernel(const float* __restrict__ out, const int2* __restrict__ ids,
                                                        int R, int d, EpPeers P, int32_t* done_counter,
                                                        unsigned long long epoch) {
  epoch = ep_epoch(P, epoch);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nwarps = gridDim.x * (blockDim.x / 32);
  const int vpr = d / 4;
  for (int p = blockIdx.x * (blockDim.x / 32) + warp; p < R; p += nwarps) {
    const int2 id = ids[p];
    const float4* src = reinterpret_cast<const float4*>(out + (size_t)p * d);
    float4* dst = reinterpret_cast<float4*>(P.home[id.x] + (size_t)id.y * d);
    for (int q = lane; q < vpr; q += 32) dst[q] = src[q];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(done_counter, 1);
    if (prev == static_cast<int>(gridDim.x) - 1) {
      __threadfence_system();
      *done_counter = 0;
      for (int r = 0; r < P.n; ++r) st_release_sys_u64(P.flags[r] + 2 * P.n + P.me, epoch);
    }
  }
}

// 3'. return fused with the FFN's K-split reduction: received row p's output
// = sum over the down splits of its partials (ascending split order, exactly
// row_reduce_kernel's sum), written straight into home[source][id] of its
// home rank; then flag set 2 of every source.  Partials are in the FFN's
// tiled layout ys[split][d-pair][half][padded row][128] (prow: row -> padded row).
__global__ void __launch_bounds__(256) ep_reduce_return_kernel(const float* __restrict__ ys, int splits, int n_dp,
                                                               int T_pad, const int32_t* __restrict__ prow,
                                                               const int2* __restrict__ ids, int R,
                                                               const int32_t* __restrict__ R_dev, int d,
                                                               EpPeers P, int32_t* done_counter,
                                                               unsigned long long epoch) {
  if (R_dev) R = *R_dev;  // received rows counted on the device (no host sync)
  epoch = ep_epoch(P, epoch);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nwarps = gridDim.x * (blockDim.x / 32);
  const size_t half_stride = (size_t)T_pad * 128;
  for (int p = blockIdx.x * (blockDim.x / 32) + warp; p < R; p += nwarps) {
    const int2 id = ids[p];
    const size_t row = (size_t)__ldg(prow + p);
    float4* dst = reinterpret_cast<float4*>(P.home[id.x] + (size_t)id.y * d);
    for (int v = lane; v < d / 4; v += 32) {
      const int feat = v * 4;
      const size_t blk = (size_t)(feat >> 8) * 2 + ((feat >> 7) & 1);
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < splits; ++s) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(ys + ((size_t)s * n_dp * 2 + blk) * half_stride +
                                                               row * 128 + (feat & 127)));
        if (s == 0) {
          g = a;
        } else {
          g.x = __fadd_rn(g.x, a.x); g.y = __fadd_rn(g.y, a.y);
          g.z = __fadd_rn(g.z, a.z); g.w = __fadd_rn(g.w, a.w);
        }
      }
      dst[v] = g;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(done_counter, 1);
    if (prev == static_cast<int>(gridDim.x) - 1) {
      __threadfence_system();
      *done_counter = 0;
      for (int r = 0; r < P.n; ++r) st_release_sys_u64(P.flags[r] + 2 * P.n + P.me, epoch);
    }
  }
}

// Local per-expert row counts from the all-gathered matrix, once the rows of
// every source are in (flag set 1): counts_out[e] = sum_s counts[s][lo + e].
__global__ void __launch_bounds__(256) ep_local_counts_kernel(EpPeers P, int E, int lo, int E_local,
                                                              int32_t* __restrict__ counts_out,
                                                              unsigned long long epoch) {
  ep_wait_all(P.flags[P.me] + 1 * P.n, P.n, ep_epoch(P, epoch));
  const int32_t* cnt = P.counts[P.me];
  for (int e = threadIdx.x; e < E_local; e += blockDim.x) {
    int c = 0;
    for (int s = 0; s < P.n; ++s) c += __ldcg(cnt + (size_t)s * E + lo + e);
    counts_out[e] = c;
  }
}

}  // namespace moe
