// router_seg.cuh — router for the latency regime (few token x expert chains,
// e.g. Mixtral / Qwen at <= 512 tokens): certified split-K fp64 logits.
//
// The reference logit is ONE sequential fp64 fold over d (linalg.py:45-57):
// a_i = fl(a_{i-1} + p_i), p_i = x_i * w_i exact in fp64.  Run as written that
// is d x DFMA latency (17 us at d = 4096) on a handful of SMs.  Here every
// chain is cut into segments of L steps that run in parallel:
//   segment s:  b_j = fl(b_{j-1} + p_{sL+j}) from -0,  c_s = b_L,
//               m_s = sum_j |b_j|                    (DADD, off the chain)
// and the sequential result is bracketed rigorously.  Each rounding of the
// reference fold errs by at most u|a_i| (u = 2^-53), so
//   |a_d - sum p| <= u * sum_i |a_i|,   |a_i| <= |C_s| + |b_j| + O(u),
// with C_s the prefix of the segment totals; the segment sums themselves err
// by at most u * m_s.  Hence with
//   A = sum_s (L_s |C_s| + m_s),   s^ = sum_s c_s
// the reference value lies in [s^ - D, s^ + D] for D = u A (2 + 12/L)(1 + 2^-20) + 8u|s^|:
//   u A        bounds the reference fold's own rounding (|a_i| <= |C_s| + |b_j|),
//   u sum m_s  (<= u A) the segment folds' rounding,
//   u sum |C_node| over the merge tree (<= 5 warp-tree levels plus the
//              sequential cross-warp / cross-k-block prefixes, each level
//              <= 2A/L) the merges' rounding of the interior prefixes, and
//   8u|s^|     the rightmost nodes' (<= 7 merges -- 5 tree levels, the last
//              warp, the last k-block -- end at the total, which is not a
//              segment boundary, so A/L does not bound it),
// and (1 + 2^-20) covers the O(d u) second-order terms and the rounding of A
// itself (tests/test_certificate.py restates this arithmetic in numpy and
// checks it on random and adversarial inputs).  The fp32 rounding of every point of that interval
// is the certified logit interval {lo, hi}; lo == hi almost always.  Phase 2
// (router.cuh route_scores_tokens) checks whether the outputs depend on the
// remaining uncertainty and recomputes only those logits with the exact
// sequential chain.  A == 0 (all products zero: the sign of a zero sum
// depends on the order) is always recomputed.
//
// Grid: (token blocks of 4) x (expert blocks of expc) x (k-blocks of kr).
// 256 threads = S segments x G expert groups; each thread owns a 4 x 4
// (token x expert) register tile over one segment, with operands streamed
// straight from global memory one 8-step block ahead.  Segment partials are
// merged in k order (warp shuffles, then across warps) into per-k-block
// {C_b, A_b}; the last k-block CTA of a (token block, expert block) combines
// them in k order, the last expert block of a token block runs phase 2
// (scores + top-k).  The scheduler runs in the dispatch kernel
// (dispatch.cuh).  All counters self-reset.
#pragma once

#include <type_traits>

#include "dispatch.cuh"
#include "router.cuh"

namespace moe {

constexpr int kSegThreads = 256;
constexpr int kSegTT = 4;  // tokens per CTA (and per thread tile)
constexpr int kSegTE = 4;  // experts per thread tile

// Non-finite inputs (require_finite, linalg.py:38-42): finite fp32 operands
// cannot make the fp64 fold non-finite (|x w| <= 1.2e77, d < 2^20 terms), so a
// non-finite sum means the token row or the expert column holds an Inf / NaN.
// Only then are both scanned to set the right flag (off the hot loop).
template <bool kXBf16>
MOE_DEVICE void flag_nonfinite_inputs(const RouterParams& p, int t, int e) {
  bool bad_x = false, bad_w = false;
  for (int k = 0; k < p.d; ++k) {
    const float xv = kXBf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p.x)[(size_t)t * p.d + k])
                            : static_cast<const float*>(p.x)[(size_t)t * p.d + k];
    bad_x |= !isfinite(xv);
    bad_w |= !isfinite(p.wr[(size_t)k * p.E + e]);
  }
  if (bad_x) atomicOr(p.flags, 1u);
  if (bad_w) atomicOr(p.flags, 2u);
}

template <bool kXBf16>
MOE_DEVICE void seg_finalize(const RouterParams& p, int t, int e, double s, double A) {
  if (t >= p.B || e >= p.E) return;
  if (!isfinite(s) || !isfinite(A)) flag_nonfinite_inputs<kXBf16>(p, t, e);
  float2 r;
  if (!(A > 0.0) || !isfinite(s) || p.force_exact) {
    r = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));  // unknown: recompute exactly
  } else {
    // + 8 u |s|: the merges' roundings of the running total itself (the
    // rightmost node of each merge level sums up to the whole chain)
    const double D = __dadd_ru(__dmul_ru(A, p.cert_coef), __dmul_ru(fabs(s), 0x1p-50));
    r = make_float2(__double2float_rn(__dsub_rd(s, D)), __double2float_rn(__dadd_ru(s, D)));
  }
  p.lbuf[(size_t)t * p.E + e] = r;
}

// kTT: tokens per CTA / thread tile (4; 1- and 2-token batches use 1 / 2, so
// no thread folds padding rows and the CTA reduction moves less data)
template <bool kXBf16, bool kWVec, bool kW64 = false, int kTT = kSegTT>
__global__ void __launch_bounds__(kSegThreads, 1) router_seg_kernel(const __grid_constant__ RouterParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TT = kTT, TE = kSegTE;
  const int tid = threadIdx.x;
  const int kb = blockIdx.x % p.n_kb;
  const int rest = blockIdx.x / p.n_kb;
  const int eb = rest % p.n_eblocks;
  const int tb = rest / p.n_eblocks;
  const int t0 = tb * TT, e0 = eb * p.expc;
  const int G = p.expc / TE;        // expert groups per segment: 1, 2, 4, 8, 16
  const int g = tid % G, s = tid / G;
  const int kbeg = kb * p.kr + s * p.seg_len;
  const int kend = min(p.d, kbeg + p.seg_len);
  const int ebase = e0 + g * TE;
  // debug timeline: 16 u64 per CTA {globaltimer start, clock64 deltas of the
  // phase boundaries [1..9], smid, exact-chain counts [11], [12]}
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  const long long c_start = clock64();
  auto stamp = [&](int i) { if (tr && threadIdx.x == 0) tr[i] = clock64() - c_start; };
  if (tr && tid == 0) { tr[0] = globaltimer_ns(); tr[10] = smid_u32(); }

  pdl_launch_dependents();  // the dispatch grid may queue up (it waits for this grid)

  // ------------------------------ phase 1 -----------------------------------
  double acc[TT][TE], mag[TT][TE];
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TE; ++j) {
      acc[i][j] = -0.0;
      mag[i][j] = 0.0;
    }
  bool tok_ok[TT];
#pragma unroll
  for (int i = 0; i < TT; ++i) tok_ok[i] = (t0 + i) < p.B;
  bool ex_ok[TE];
#pragma unroll
  for (int j = 0; j < TE; ++j) ex_ok[j] = (ebase + j) < p.E;

  using WT = typename std::conditional<kW64, double, float>::type;
  auto load_blk = [&](int k, float (&xb)[TT][8], WT (&wb)[8][TE]) {
#pragma unroll
    for (int i = 0; i < TT; ++i) {
      if (tok_ok[i]) {
        load_x8<kXBf16>(p.x, (size_t)(t0 + i) * p.d + k, xb[i]);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) xb[i][q] = 0.0f;
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if constexpr (kW64) {
        const double* wrow = p.wlin64 + (size_t)(k + r) * p.E + ebase;
        if (kWVec) {  // E % 4 == 0: two 16-byte loads
          double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
          if (ex_ok[0]) { a = __ldg(reinterpret_cast<const double2*>(wrow)); b = __ldg(reinterpret_cast<const double2*>(wrow) + 1); }
          wb[r][0] = a.x; wb[r][1] = a.y; wb[r][2] = b.x; wb[r][3] = b.y;
        } else {
#pragma unroll
          for (int j = 0; j < TE; ++j) wb[r][j] = ex_ok[j] ? __ldg(wrow + j) : 0.0;
        }
        continue;
      }
      const float* wrow = p.wr + (size_t)(k + r) * p.E + ebase;
      if (kWVec) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ex_ok[0]) v = __ldg(reinterpret_cast<const float4*>(wrow));
        wb[r][0] = static_cast<WT>(v.x); wb[r][1] = static_cast<WT>(v.y);
        wb[r][2] = static_cast<WT>(v.z); wb[r][3] = static_cast<WT>(v.w);
      } else {
#pragma unroll
        for (int j = 0; j < TE; ++j) wb[r][j] = ex_ok[j] ? static_cast<WT>(__ldg(wrow + j)) : WT(0);
      }
    }
  };

  if (kbeg < kend) {
    float xc[TT][8];
    WT wc[8][TE];
    load_blk(kbeg, xc, wc);
    for (int k = kbeg; k < kend; k += 8) {
      float xn[TT][8];
      WT wn[8][TE];
      if (k + 8 < kend) load_blk(k + 8, xn, wn);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        double xd[TT], wd[TE];
#pragma unroll
        for (int i = 0; i < TT; ++i) xd[i] = static_cast<double>(xc[i][r]);
#pragma unroll
        for (int j = 0; j < TE; ++j) wd[j] = static_cast<double>(wc[r][j]);
#pragma unroll
        for (int i = 0; i < TT; ++i)
#pragma unroll
          for (int j = 0; j < TE; ++j) {
            acc[i][j] = __fma_rn(xd[i], wd[j], acc[i][j]);
            mag[i][j] = __dadd_rn(mag[i][j], fabs(acc[i][j]));
          }
      }
#pragma unroll
      for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) xc[i][q] = xn[i][q];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < TE; ++j) wc[r][j] = wn[r][j];
    }
  }

  stamp(2);
  // ---- per-chain reduction of the segment partials --------------------------
  // Merge of adjacent ranges (left l, right r) of the k order:
  //   C = C_l + C_r,  A = A_l + A_r + K_r |C_l|,  K = K_l + K_r
  // (the right range's prefixes are shifted by C_l; |C_l + c| <= |C_l| + |c|).
  // A single segment starts as {c_s, m_s, L_s}.  Ordered tree over the lanes
  // of a warp (lane = s_lo * G + g), then over the 8 warps in order.
  const int warp = tid / 32, lane = tid % 32;
  const int chains = TT * p.expc;
  double K = static_cast<double>(max(0, kend - kbeg));
  // (levels not unrolled: this code runs once per CTA from a cold
  // instruction cache, so every unrolled level would be fetched from L2)
#pragma unroll 1
  for (int off = G; off < 32; off <<= 1) {
    const double Kr = __shfl_down_sync(0xffffffffu, K, off);
    const bool left = ((lane / G) & (2 * off / G - 1)) == 0;
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
      for (int j = 0; j < TE; ++j) {
        const double Cr = __shfl_down_sync(0xffffffffu, acc[i][j], off);
        const double Ar = __shfl_down_sync(0xffffffffu, mag[i][j], off);
        if (left) {
          mag[i][j] = mag[i][j] + Ar + Kr * fabs(acc[i][j]);
          acc[i][j] = acc[i][j] + Cr;
        }
      }
    if (left) K += Kr;
  }
  // warp results -> smem red[warp][chain] = {C, A}; wk[warp] = K
  double2* red = reinterpret_cast<double2*>(smem);
  double* wk = reinterpret_cast<double*>(smem + (size_t)(kSegThreads / 32) * chains * 16);
  if (lane < G) {
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
      for (int j = 0; j < TE; ++j) red[(size_t)warp * chains + i * p.expc + g * TE + j] = make_double2(acc[i][j], mag[i][j]);
    if (lane == 0) wk[warp] = K;
  }
  __syncthreads();
  const bool single_kb = (p.n_kb == 1);
  double2* gpart = reinterpret_cast<double2*>(p.gpart);
  for (int c = tid; c < chains; c += kSegThreads) {
    double C = 0.0, A = 0.0;
    for (int w = 0; w < kSegThreads / 32; ++w) {
      const double2 v = red[(size_t)w * chains + c];
      A = A + v.y + wk[w] * fabs(C);
      C = C + v.x;
    }
    const int t = t0 + c / p.expc, e = e0 + c % p.expc;
    if (single_kb) {
      seg_finalize<kXBf16>(p, t, e, C, A);
    } else {
      gpart[((size_t)(tb * p.n_eblocks + eb) * p.n_kb + kb) * chains + c] = make_double2(C, A);
    }
  }
  stamp(3);
  if (!single_kb) {
    // last k-block CTA of this (token block, expert block) combines in k order
    if (!cta_arrive_last(p.blk_counter + tb * p.n_eblocks + eb, p.n_kb)) return;
    stamp(4);
    for (int c = tid; c < chains; c += kSegThreads) {
      double Gs = 0.0, A = 0.0;
      for (int b = 0; b < p.n_kb; ++b) {
        const double2 v = __ldcg(gpart + ((size_t)(tb * p.n_eblocks + eb) * p.n_kb + b) * chains + c);
        const int Kb = max(0, min(p.kr, p.d - b * p.kr));
        A += v.y + static_cast<double>(Kb) * fabs(Gs);
        Gs += v.x;
      }
      seg_finalize<kXBf16>(p, t0 + c / p.expc, e0 + c % p.expc, Gs, A);
    }
    if (tid == 0) p.blk_counter[tb * p.n_eblocks + eb] = 0;
    stamp(5);
  }

  // ------------------ phase 2: last expert block of the token block ----------
  if (p.n_eblocks > 1) {
    if (!cta_arrive_last(p.tb_counter + tb, p.n_eblocks)) return;
    if (tid == 0) p.tb_counter[tb] = 0;
  } else {
    __syncthreads();  // lbuf of this token block was written by this CTA
  }
  stamp(6);
  route_scores_tokens<kXBf16>(p, t0, min(t0 + TT, p.B), smem);
  stamp(7);
  if (p.fuse_dispatch) {
    // small batch: the last token block to finish phase 2 schedules and
    // gathers all B*k rows (no dispatch launch)
    if (p.n_tblocks > 1) {
      if (!cta_arrive_last(p.disp_counter, p.n_tblocks)) return;
      if (tid == 0) *p.disp_counter = 0;
    } else {
      __syncthreads();
    }
    dispatch_small_cta<kXBf16>(p.topk_idx, p.B * p.k, p.k, p.E, p.d, p.chunk_rows, p.x, p.xp, p.counts,
                               p.offsets, p.fwd, p.inv, p.prow, p.chunk_tab, p.chunk_grp, p.n_chunks,
                               reinterpret_cast<int32_t*>(smem));
  }
}

}  // namespace moe
