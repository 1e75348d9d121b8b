// router_screen.cuh — router for sigmoid gating at large B x E (the
// throughput regime: DeepSeek-V3, 256 experts x 512 tokens = 131K logits of
// d = 7168 steps each).  Same outputs as router_kernel / router_seg_kernel
// (bit-exact routing, reference router.py:88-133 + linalg.py:45-57), a
// fraction of the fp64 work.
//
// With sigmoid gating a token's outputs depend only on the logits that can
// reach its top-k: score_e = sigmoid32(l_e) is a per-expert function, the
// top-k keeps the k largest (score, lowest index) keys and the weights
// renormalise the k selected scores (router.py:99-112).  So every logit gets a
// cheap, rigorous interval first, and only the few that can still matter are
// computed to the reference's fp32 bits:
//
//  1. screen (INT8 tensor cores, tcgen05 kind::i8).  Each token row and each
//     expert column is scaled by a power of two (2^F > max|v|) and rounded to a
//     20-bit integer Q = rint(v 2^(19-F)), split into three balanced base-128
//     digits (|D| <= 64) stored as int8 planes.  Q_x Q_w = sum_{s,t} D_s G_t
//     128^(4-s-t): the digit-plane products of weight class c = s + t are
//     accumulated EXACTLY in int32 TMEM columns [128c, 128c+128) -- one
//     tcgen05.mma of N = 256 writes the planes [G0 G1] of a token plane into
//     two adjacent classes -- and class 4 (D2 G2, weight 1) is dropped into the
//     error bound.  K is split across CTAs; the int32 partials are combined as
//     exact int64.  The interval adds (all rounded up): the quantisation error
//     err_x sum|w| + err_w sum|x^| (err = half a unit, 2^(u-1)), the dropped
//     class 64 min(sum|D2|, sum|G2|), and the reference fold's own rounding
//     d u sum|x||w| (the sums per row / column from the prep kernels;
//     tests/test_screen_bound.py restates the bound in exact rationals).  Its
//     fp32 rounding [lo, hi] contains the reference logit.
//  2. select: per token the k-th largest lower score bound S_k; experts whose
//     upper score bound is below S_k can never be selected (their score is
//     strictly below k others').  The rest (~k per token) are candidates.
//  3. refine: the candidates' logits with the certified split-K fp64 fold of
//     router_seg.cuh (segments of the d axis across CTAs, W slice in shared
//     memory, one thread folds its segment of up to 8 candidate chains).
//  4. phase 2 (router.cuh route_scores_tokens, screen mode): the segment
//     partials are merged in k order (sequential within a lane, then a warp
//     tree), the certified interval is intersected with the screen interval,
//     the non-candidates are excluded and the usual certification (exact
//     chain for whatever still matters) + top-k + renormalisation run.
//
// Sigmoid bounds: numpy's float32 logistic (np_sigmoid) is accurate to a few
// ulps but not monotone at the ulp level, so score bounds carry a 2^-20
// relative margin (and 2^-126 absolute), and nothing is excluded when S_k is
// below 2^-100 (subnormal scores).
#pragma once

#include "router.cuh"

namespace moe {

constexpr int kScrPlanes = 3;
constexpr int kScrBits = 19;     // Q = rint(v * 2^(19 - F)), |Q| <= 2^19 for 2^F > max|v|
constexpr int kScrM = 128;       // tokens per GEMM tile (TMEM lanes)
constexpr int kScrN = 128;       // experts per GEMM tile
constexpr int kScrKB = 128;      // K per shared-memory block (one 128-byte swizzle row of int8)
constexpr int kScrStages = 2;
constexpr int kScrThreads = 192; // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int kScrMaxCand = 32;  // candidates refined per token (more: exact fallback)
constexpr int kScrRefThreads = 512;
constexpr int kScrPh2Tok = 4;    // tokens per phase-2 CTA
constexpr int kScrPh2Threads = 512;
constexpr uint32_t kScrPlaneBytes = kScrM * kScrKB;                // 16 KB
constexpr uint32_t kScrStageBytes = 2 * kScrPlanes * kScrPlaneBytes;  // A + B planes: 96 KB
constexpr size_t kScrGemmSmem = kScrStages * kScrStageBytes + 1024 + 256;

struct ScreenParams {
  const void* x;
  const float* wr;
  int B, d, E, k;
  int B_pad, E_pad, d_pad;
  int n_ks, kb_per_split;
  int8_t* xq;               // [3][B_pad][d_pad] token digit planes (plane 0 most significant)
  int8_t* wq;               // [3][E_pad][d_pad] expert digit planes (K-major rows)
  int4* xst;                // per token {unit exponent, err bound 2^(ue-1) (float bits), sum |D2|, 0}
  long long* xqs;           // per token sum |Q|
  uint32_t* wmax;           // per expert max |w| (float bits), header, self-resetting
  uint32_t* wg2;            // per expert sum |G2|
  unsigned long long* wrs;  // per expert sum |Q|
  long long* spart;         // [n_ks][B_pad][E_pad] int64 partials (units 2^(ux + uw))
  int32_t* cand;            // [B][kScrMaxCand]
  int32_t* ncand;           // [B]; -1: too many candidates (phase 2 resolves exactly)
  int32_t* ecount;          // per expert: candidate chains listed (header, self-resetting)
  int32_t* elist;           // [E][B] candidate chains of expert e: t * kScrMaxCand + slot (any order)
  double2* rpart;           // [n_rs][B][kScrMaxCand] {C, A} segment partials
  int n_rs, rs_len, rs_first;
  float2* lbuf;
  uint32_t* flags;
};

// ---------------------------------------------------------------------------
// digit decomposition.  Q = rint(v 2^-ue) with the power-of-two scaling in
// fp32 (exact, split in two factors when 2^-ue exceeds fp32's range; a product
// that underflows is < 1/2 and rounds to 0 like the exact one), balanced
// base-128 digits.  The quantisation error is at most half a unit, 2^(ue-1)
// (0 for an all-zero row or column).
// ---------------------------------------------------------------------------
MOE_DEVICE int scr_unit_exp(float vmax) {  // unit exponent u: v^ = Q 2^u
  if (!(vmax > 0.0f)) return 0;
  int e;
  frexpf(vmax, &e);  // vmax = m 2^e, m in [0.5, 1): vmax < 2^e
  return e - kScrBits;
}
MOE_DEVICE double scr_pow2(int n) {  // 2^n, n in [-1022, 1023]
  return __longlong_as_double(static_cast<long long>(n + 1023) << 52);
}
MOE_DEVICE float scr_pow2f(int n) {  // 2^n, n in [-126, 127]
  return __int_as_float((n + 127) << 23);
}
struct ScrScale {
  float s1, s2;
};
MOE_DEVICE ScrScale scr_scale(int ue) {  // 2^-ue = s1 s2, both normal fp32
  const int n = -ue;
  const int a = max(-126, min(126, n));
  return {scr_pow2f(a), scr_pow2f(n - a)};
}
struct ScrDigits {
  int q, d0, d1, d2;
};
MOE_DEVICE ScrDigits scr_digits(float v, ScrScale s) {
  ScrDigits r;
  r.q = __float2int_rn(__fmul_rn(__fmul_rn(v, s.s1), s.s2));
  r.d2 = ((r.q + 64) & 127) - 64;
  const int q1 = (r.q - r.d2) >> 7;
  r.d1 = ((q1 + 64) & 127) - 64;
  r.d0 = (q1 - r.d1) >> 7;  // |d0| <= 33
  return r;
}
MOE_DEVICE uint32_t scr_pack(int a, int b, int c, int d) {
  return (static_cast<uint32_t>(a) & 0xFFu) | ((static_cast<uint32_t>(b) & 0xFFu) << 8) |
         ((static_cast<uint32_t>(c) & 0xFFu) << 16) | (static_cast<uint32_t>(d) << 24);
}

template <bool kXBf16>
MOE_DEVICE float scr_load_x(const void* x, size_t i) {
  if constexpr (kXBf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
  else return static_cast<const float*>(x)[i];
}
// 4 consecutive elements (i % 4 == 0, row-aligned)
template <bool kXBf16>
MOE_DEVICE float4 scr_load_x4(const void* x, size_t i) {
  if constexpr (kXBf16) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(x) + i));
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xFFFF0000u));
  } else {
    return __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(x) + i));
  }
}

// ---------------------------------------------------------------------------
// K1: per-expert max |w| (atomicMax on the bits of a non-negative float).
// Grid (ceil(d / 64), ceil(E / 32)); lane = expert, warp = row phase.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) screen_wmax_kernel(const ScreenParams p) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.y * 32 + lane;
  const int r0 = blockIdx.x * 64;
  float m = 0.0f;
  bool bad = false;
  if (e < p.E) {
#pragma unroll 4
    for (int i = warp; i < 64; i += 8) {
      const int k = r0 + i;
      if (k < p.d) {
        const float v = __ldg(p.wr + (size_t)k * p.E + e);
        if (isfinite(v)) m = fmaxf(m, fabsf(v));
        else bad = true;
      }
    }
  }
  if (bad) atomicOr(p.flags, 2u);
  red[warp][lane] = m;
  __syncthreads();
  if (warp == 0 && e < p.E) {
    for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w][lane]);
    if (m > 0.0f) atomicMax(p.wmax + e, __float_as_uint(m));
  }
}

// ---------------------------------------------------------------------------
// K2: digit planes.  CTAs [0, B): one token row each (the row is held in
// registers, 8 x 4 elements per thread, for d <= 8192; longer rows are read
// twice).  CTAs past B: one (128-row k tile, 32 experts) tile of W each,
// transposed through shared memory into K-major expert rows.  Padding
// (k >= d, experts >= E) is written as 0.  Non-finite inputs set the flags
// (NonFiniteInput) and digitise as 0.
// ---------------------------------------------------------------------------
constexpr int kScrRowRegs = 8;  // float4 per thread held in registers

template <bool kXBf16>
__global__ void __launch_bounds__(256) screen_digits_kernel(const ScreenParams p) {
  __shared__ float s_red[8];
  __shared__ long long s_q[8];
  __shared__ int s_d2[8];
  __shared__ uint32_t s_dig[kScrPlanes][32][33];  // packed 4 k per word, padded rows
  __shared__ unsigned long long s_wq[8][32];
  __shared__ uint32_t s_wg2[8][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x < static_cast<unsigned>(p.B)) {
    // ------------------------------ token row ------------------------------
    const int t = blockIdx.x;
    const size_t row = (size_t)t * p.d;
    const int n4 = p.d / 4;  // d % 8 == 0
    float4 v[kScrRowRegs];
    float m = 0.0f;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < kScrRowRegs; ++i) {
      const int j = tid + 256 * i;
      v[i] = j < n4 ? scr_load_x4<kXBf16>(p.x, row + 4 * (size_t)j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto acc_max = [&](float4& a) {
      const float c[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (isfinite(c[q])) m = fmaxf(m, fabsf(c[q]));
        else bad = true;
      }
    };
#pragma unroll
    for (int i = 0; i < kScrRowRegs; ++i) acc_max(v[i]);
    for (int j = tid + 256 * kScrRowRegs; j < n4; j += 256) {
      float4 a = scr_load_x4<kXBf16>(p.x, row + 4 * (size_t)j);
      acc_max(a);
    }
    if (bad) atomicOr(p.flags, 1u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    m = s_red[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, s_red[w]);
    const int ue = scr_unit_exp(m);
    const ScrScale sc = scr_scale(ue);
    long long qs = 0;
    int d2s = 0;
    int8_t* q0 = p.xq + (size_t)t * p.d_pad;
    const size_t plane = (size_t)p.B_pad * p.d_pad;
    auto emit = [&](int j, float4 a) {  // 4 elements k = 4j .. 4j+3
      const float c[4] = {a.x, a.y, a.z, a.w};
      ScrDigits g[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        g[q] = scr_digits(isfinite(c[q]) ? c[q] : 0.0f, sc);
        qs += abs(g[q].q);
        d2s += abs(g[q].d2);
      }
      reinterpret_cast<uint32_t*>(q0)[j] = scr_pack(g[0].d0, g[1].d0, g[2].d0, g[3].d0);
      reinterpret_cast<uint32_t*>(q0 + plane)[j] = scr_pack(g[0].d1, g[1].d1, g[2].d1, g[3].d1);
      reinterpret_cast<uint32_t*>(q0 + 2 * plane)[j] = scr_pack(g[0].d2, g[1].d2, g[2].d2, g[3].d2);
    };
#pragma unroll
    for (int i = 0; i < kScrRowRegs; ++i) {
      const int j = tid + 256 * i;
      if (j < n4) emit(j, v[i]);
    }
    for (int j = tid + 256 * kScrRowRegs; j < n4; j += 256) emit(j, scr_load_x4<kXBf16>(p.x, row + 4 * (size_t)j));
    for (int j = n4 + tid; j < p.d_pad / 4; j += 256) {  // zero padding k >= d
      reinterpret_cast<uint32_t*>(q0)[j] = 0;
      reinterpret_cast<uint32_t*>(q0 + plane)[j] = 0;
      reinterpret_cast<uint32_t*>(q0 + 2 * plane)[j] = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      qs += __shfl_xor_sync(0xffffffffu, qs, o);
      d2s += __shfl_xor_sync(0xffffffffu, d2s, o);
    }
    if (lane == 0) { s_q[warp] = qs; s_d2[warp] = d2s; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < 8; ++w) { qs += s_q[w]; d2s += s_d2[w]; }
      const float err = m > 0.0f ? scr_pow2f(max(-126, ue - 1)) : 0.0f;  // (>= 2^(ue-1))
      p.xst[t] = make_int4(ue, __float_as_int(err), d2s, 0);
      p.xqs[t] = qs;
    }
    return;
  }
  // ------------------------------- W tile ----------------------------------
  const int wb = blockIdx.x - p.B;
  const int n_eg = p.E_pad / 32;
  const int kt = wb / n_eg, eg = wb % n_eg;
  const int k0 = kt * kScrKB, e = eg * 32 + lane;
  const bool ev = e < p.E;
  const ScrScale sc = scr_scale(ev ? scr_unit_exp(__uint_as_float(p.wmax[e])) : 0);
  unsigned long long qs = 0;
  uint32_t g2 = 0;
  // warp w: rows 16w .. 16w+15 of the tile, packed 4 per word
  float v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int k = k0 + warp * 16 + r;
    v[r] = (ev && k < p.d) ? __ldg(p.wr + (size_t)k * p.E + e) : 0.0f;
  }
#pragma unroll
  for (int r4 = 0; r4 < 4; ++r4) {
    ScrDigits g[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float c = v[r4 * 4 + j];
      g[j] = scr_digits(isfinite(c) ? c : 0.0f, sc);
      qs += static_cast<unsigned long long>(abs(g[j].q));
      g2 += static_cast<uint32_t>(abs(g[j].d2));
    }
    s_dig[0][lane][warp * 4 + r4] = scr_pack(g[0].d0, g[1].d0, g[2].d0, g[3].d0);
    s_dig[1][lane][warp * 4 + r4] = scr_pack(g[0].d1, g[1].d1, g[2].d1, g[3].d1);
    s_dig[2][lane][warp * 4 + r4] = scr_pack(g[0].d2, g[1].d2, g[2].d2, g[3].d2);
  }
  s_wq[warp][lane] = qs;
  s_wg2[warp][lane] = g2;
  __syncthreads();
  if (warp == 0 && ev) {
    for (int w = 1; w < 8; ++w) { qs += s_wq[w][lane]; g2 += s_wg2[w][lane]; }
    atomicAdd(p.wrs + e, qs);
    atomicAdd(p.wg2 + e, g2);
  }
  // write 3 planes x 32 expert rows x 128 bytes: one word per thread per pass
  const size_t plane = (size_t)p.E_pad * p.d_pad;
  for (int i = tid; i < kScrPlanes * 32 * 32; i += 256) {
    const int pl = i / (32 * 32), r = (i / 32) % 32, wd = i % 32;
    reinterpret_cast<uint32_t*>(p.wq + pl * plane + (size_t)(eg * 32 + r) * p.d_pad + k0)[wd] = s_dig[pl][r][wd];
  }
}

// ---------------------------------------------------------------------------
// K3: screen GEMM (tcgen05 kind::i8).  CTA = (128 tokens, 128 experts, one K
// split).  TMEM: class c at columns [128c, 128c + 128), c = 0..3.  Per
// 32-element k step, five MMAs: (x plane s) x (w planes [G0 G1], N = 256)
// into classes s, s+1 for s = 0, 1, 2, and (x plane s) x G2 (N = 128) into
// class s + 2 for s = 0, 1.  The first k step orders them so that every class
// is first written with accumulate = 0.  Epilogue: V = sum_c class_c 2^(7(4-c))
// as int64 per (token, expert), stored to this split's partial slab.
// ---------------------------------------------------------------------------
MOE_DEVICE uint32_t make_idesc_s8(uint32_t m, uint32_t n) {
  uint32_t d = 0;
  d |= 2u << 4;   // D: s32
  d |= 1u << 7;   // A: s8
  d |= 1u << 10;  // B: s8
  d |= ((n >> 3) & 0x3Fu) << 17;
  d |= ((m >> 4) & 0x1Fu) << 24;
  return d;
}
MOE_DEVICE void mma_s8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(kScrThreads, 1)
screen_gemm_kernel(const __grid_constant__ CUtensorMap tm_xq, const __grid_constant__ CUtensorMap tm_wq,
                   const ScreenParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kScrStages * kScrStageBytes);
  uint64_t* empty = full + kScrStages;
  uint64_t* done = empty + kScrStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_eb = p.E_pad / kScrN;
  const int ks = blockIdx.x % p.n_ks;
  const int rest = blockIdx.x / p.n_ks;
  const int eb = rest % n_eb, tt = rest / n_eb;
  const int nkb = p.d_pad / kScrKB;
  const int kb0 = ks * p.kb_per_split, kb1 = min(nkb, kb0 + p.kb_per_split);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_xq);
    tma_prefetch_desc(&tm_wq);
    for (int s = 0; s < kScrStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0; kb < kb1; ++kb) {
        const int i = kb - kb0, s = i % kScrStages;
        mbar_wait(empty + s, ((i / kScrStages) & 1) ^ 1);
        uint8_t* st = smem + s * kScrStageBytes;
        mbar_arrive_expect_tx(full + s, kScrStageBytes);
        for (int pl = 0; pl < kScrPlanes; ++pl) {
          tma_load_2d(&tm_xq, full + s, st + pl * kScrPlaneBytes, kb * kScrKB, pl * p.B_pad + tt * kScrM);
          tma_load_2d(&tm_wq, full + s, st + (kScrPlanes + pl) * kScrPlaneBytes, kb * kScrKB,
                      pl * p.E_pad + eb * kScrN);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id256 = make_idesc_s8(kScrM, 2 * kScrN), id128 = make_idesc_s8(kScrM, kScrN);
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0, s = i % kScrStages;
      mbar_wait(full + s, (i / kScrStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a0 = smem_u32(smem + s * kScrStageBytes);
        const uint32_t b0 = a0 + kScrPlanes * kScrPlaneBytes;
#pragma unroll
        for (int kk = 0; kk < kScrKB / 32; ++kk) {
          auto ad = [&](int pl) { return make_smem_desc_sw128(a0 + pl * kScrPlaneBytes + kk * 32, 16, 1024); };
          const uint64_t b01 = make_smem_desc_sw128(b0 + kk * 32, 16, 1024);
          const uint64_t b2 = make_smem_desc_sw128(b0 + 2 * kScrPlaneBytes + kk * 32, 16, 1024);
          const uint32_t f = (kb > kb0 || kk > 0) ? 1u : 0u;  // first k step: initialise every class once
          mma_s8(tmem + 0 * kScrN, ad(0), b01, id256, f);      // classes 0, 1
          mma_s8(tmem + 2 * kScrN, ad(0), b2, id128, f);       // class 2
          mma_s8(tmem + 3 * kScrN, ad(1), b2, id128, f);       // class 3
          mma_s8(tmem + 1 * kScrN, ad(1), b01, id256, 1u);     // classes 1, 2
          mma_s8(tmem + 2 * kScrN, ad(2), b01, id256, 1u);     // classes 2, 3
        }
        mma_commit(empty + s);
        if (kb == kb1 - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (one token row per lane)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int t = tt * kScrM + r;
    mbar_wait(done, 0);
    tc_fence_after();
    long long* dst = p.spart + ((size_t)ks * p.B_pad + t) * p.E_pad + eb * kScrN;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    for (int j = 0; j < kScrN / 32; ++j) {
      uint32_t c0[32], c1[32], c2[32], c3[32];
      tmem_ld_32x32b_x32(tmem + lane_base + 0 * kScrN + 32 * j, c0);
      tmem_ld_32x32b_x32(tmem + lane_base + 1 * kScrN + 32 * j, c1);
      tmem_ld_32x32b_x32(tmem + lane_base + 2 * kScrN + 32 * j, c2);
      tmem_ld_32x32b_x32(tmem + lane_base + 3 * kScrN + 32 * j, c3);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        longlong2 v;
        v.x = (static_cast<long long>(static_cast<int>(c0[i])) << 28) +
              (static_cast<long long>(static_cast<int>(c1[i])) << 21) +
              (static_cast<long long>(static_cast<int>(c2[i])) << 14) +
              (static_cast<long long>(static_cast<int>(c3[i])) << 7);
        v.y = (static_cast<long long>(static_cast<int>(c0[i + 1])) << 28) +
              (static_cast<long long>(static_cast<int>(c1[i + 1])) << 21) +
              (static_cast<long long>(static_cast<int>(c2[i + 1])) << 14) +
              (static_cast<long long>(static_cast<int>(c3[i + 1])) << 7);
        reinterpret_cast<longlong2*>(dst + 32 * j)[i / 2] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// K4: screen intervals + candidates; one CTA per token, one thread per expert.
// The interval of (t, e): V = sum of the splits' int64 partials (exact), value
// V 2^(ux+uw), radius (rounded up) err_x sum|w| + err_w sum|x^| +
// 64 min(sum|D2|, sum|G2|) 2^(ux+uw) + d u' sum|x| max|w|, with
// sum|w| <= sum|w^| + d err_w and sum|x| <= sum|x^| + d err_x.
// ---------------------------------------------------------------------------
constexpr int kScrSelThreads = 256;

MOE_DEVICE float2 scr_interval(const ScreenParams& p, long long V, int e, int ux, double xerr, int xd2, double sum_xh,
                               double sum_x, double gam, double dd) {
  const float wm = __uint_as_float(p.wmax[e]);
  const int uw = scr_unit_exp(wm);
  const double sc2 = scr_pow2(ux + uw);
  const double werr = wm > 0.0f ? scr_pow2(uw - 1) : 0.0;
  const double sum_w = __dadd_ru(__dmul_ru(static_cast<double>(p.wrs[e]), scr_pow2(uw)), __dmul_ru(dd, werr));
  double R = __dmul_ru(xerr, sum_w);
  R = __dadd_ru(R, __dmul_ru(werr, sum_xh));
  R = __dadd_ru(R, __dmul_ru(64.0 * static_cast<double>(min(xd2, static_cast<int>(p.wg2[e]))), sc2));
  R = __dadd_ru(R, __dmul_ru(__dmul_ru(sum_x, static_cast<double>(wm)), gam));
  R = __dmul_ru(R, 1.0 + 0x1p-40);
  const double v_lo = __dsub_rd(__dmul_rd(__ll2double_rd(V), sc2), R);
  const double v_hi = __dadd_ru(__dmul_ru(__ll2double_ru(V), sc2), R);
  return make_float2(__double2float_rn(v_lo), __double2float_rn(v_hi));
}

__global__ void __launch_bounds__(kScrSelThreads) screen_select_kernel(const ScreenParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* sc = reinterpret_cast<float*>(smem);  // lower score bounds (scratch)
  float* sh = sc + p.E;                        // upper score bounds
  const int t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid % 32;
  const int4 xs = p.xst[t];
  const int ux = xs.x;
  const double xerr = static_cast<double>(__int_as_float(xs.y));
  const double dd = static_cast<double>(p.d);
  const double sum_xh = static_cast<double>(p.xqs[t]) * scr_pow2(ux);  // sum |x^| (exact)
  const double sum_x = __dadd_ru(sum_xh, __dmul_ru(dd, xerr));        // >= sum |x|
  const double gam = __dmul_ru(dd, 0x1.02p-53);                       // fold: (d-1) u (1 + ...)
  for (int e = tid; e < p.E; e += kScrSelThreads) {
    long long V = 0;
    const long long* col = p.spart + (size_t)t * p.E_pad + e;
    const size_t slab = (size_t)p.B_pad * p.E_pad;
#pragma unroll 8
    for (int s = 0; s < p.n_ks; ++s) V += __ldcg(col + s * slab);
    const float2 r = scr_interval(p, V, e, ux, xerr, xs.z, sum_xh, sum_x, gam, dd);
    p.lbuf[(size_t)t * p.E + e] = r;
    sc[e] = scr_score_lo(r.x);
    sh[e] = scr_score_hi(r.y);
  }
  __syncthreads();
  if (tid >= 32) return;
  const float Sk = scr_kth_largest(sc, p.E, p.k, lane);
  const bool exclude = Sk >= 0x1p-100f;
  int n = 0;
  for (int e0 = 0; e0 < p.E; e0 += 32) {
    const int e = e0 + lane;
    const bool c = e < p.E && (!exclude || !(sh[e] < Sk));
    const uint32_t bal = __ballot_sync(0xffffffffu, c);
    const int pos = n + __popc(bal & ((1u << lane) - 1u));
    if (c && pos < kScrMaxCand) p.cand[(size_t)t * kScrMaxCand + pos] = e;
    n += __popc(bal);
  }
  if (lane == 0) p.ncand[t] = n <= kScrMaxCand ? n : -1;
  if (n <= kScrMaxCand && lane < n) {
    // the refinement runs expert-major: list this chain under its expert
    const int e = p.cand[(size_t)t * kScrMaxCand + lane];
    const int pos = atomicAdd(p.ecount + e, 1);
    p.elist[(size_t)e * p.B + pos] = t * kScrMaxCand + lane;
  }
}

// ---------------------------------------------------------------------------
// K5: refine.  CTA j folds segment j of the d axis (k in [k0, k0 + len)) for
// every candidate chain, from -0, tracking m = sum |partial| (router_seg.cuh's
// segment step).  The segment's W rows and the token rows' segment (per token
// group) are staged in shared memory with cp.async (all in flight at once).
// A thread takes tokens t = tid, tid + 256, ... and runs up to 8 of a token's
// chains together (the x value is shared).  CTA 0 also resets the per-expert
// screen statistics for the next forward (K2 / K4 are complete).
// ---------------------------------------------------------------------------
MOE_DEVICE void cp_async_4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

template <bool kXBf16>
__global__ void __launch_bounds__(kScrRefThreads) screen_refine_kernel(const ScreenParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kEs = kXBf16 ? 2 : 4;
  const int j = blockIdx.x;
  const int k0 = j == 0 ? 0 : p.rs_first + (j - 1) * p.rs_len;
  const int len = j == 0 ? p.rs_first : p.rs_len;  // both even (d, rs_len even)
  const int row_words = (p.rs_len * kEs / 4) | 1;   // odd word stride
  const int words = len * kEs / 4;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  double* ws = reinterpret_cast<double*>(smem);     // W rows of the segment, widened to fp64 (exact)
  uint32_t* xs = reinterpret_cast<uint32_t*>(ws + (size_t)p.rs_len * p.E);  // token rows' segment (all B)
  int* uoff = reinterpret_cast<int*>(xs + max((size_t)p.B * row_words, (size_t)p.rs_len * p.E));  // list offsets [E + 1]
  float* wraw = reinterpret_cast<float*>(xs);       // (W staging before the x rows land)
  if (j == 0)
    for (int e = threadIdx.x; e < p.E; e += blockDim.x) { p.wmax[e] = 0; p.wg2[e] = 0; p.wrs[e] = 0; }
  const float* src = p.wr + (size_t)k0 * p.E;
  for (int i = threadIdx.x; i < len * p.E; i += blockDim.x) cp_async_4(wraw + i, src + i);
  cp_async_commit();
  // expert-major flattened chain list: exclusive prefix of the list counts (warp 0)
  if (warp == 0) {
    int run = 0;
    for (int e0 = 0; e0 < p.E; e0 += 32) {
      const int e = e0 + lane;
      const int u = e < p.E ? p.ecount[e] : 0;
      int s = u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += v;
      }
      if (e < p.E) uoff[e] = run + s - u;
      run += __shfl_sync(0xffffffffu, s, 31);
    }
    if (lane == 0) uoff[p.E] = run;
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int i = threadIdx.x; i < len * p.E; i += blockDim.x) ws[i] = static_cast<double>(wraw[i]);
  __syncthreads();  // (wraw consumed before the x rows overwrite it)
  const uint8_t* xb = static_cast<const uint8_t*>(p.x);
  for (int i = threadIdx.x; i < p.B * words; i += blockDim.x) {
    const int r = i / words, c = i % words;
    cp_async_4(xs + r * row_words + c, xb + ((size_t)r * p.d + k0) * kEs + 4 * c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int n_pairs = uoff[p.E];
  // chain q of the flattened list -> (expert, token row offset in xs, rpart slot)
  auto chain = [&](int q, int& e, int& xo, size_t& out) -> bool {
    if (q >= n_pairs) { e = 0; xo = 0; return false; }
    int lo = 0, hi = p.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (uoff[mid] <= q) lo = mid; else hi = mid - 1;
    }
    e = lo;
    const int id = __ldg(p.elist + (size_t)lo * p.B + (q - uoff[lo]));
    const int t = id / kScrMaxCand;
    xo = t * row_words;
    out = ((size_t)j * p.B + t) * kScrMaxCand + id % kScrMaxCand;
    return true;
  };
  // two chains per lane (independent folds); a warp's 32 consecutive list
  // entries span 1-3 experts, so each W read is a broadcast of few words
  const int stride = 2 * 32 * nw;
  for (int q0 = warp * 64; q0 < n_pairs; q0 += stride) {
    int ea, eb, xa, xbo;
    size_t oa = 0, ob = 0;
    const bool va = chain(q0 + lane, ea, xa, oa);
    const bool vb = chain(q0 + 32 + lane, eb, xbo, ob);
    double acc_a = -0.0, mag_a = 0.0, acc_b = -0.0, mag_b = 0.0;
    // two k steps per iteration (len is even): one word holds both bf16 x values
    const double* wa = ws + ea;
    const double* wb = ws + eb;
    const uint32_t* pa = xs + xa;
    const uint32_t* pb = xs + xbo;
#pragma unroll 2
    for (int kk = 0; kk < len; kk += 2) {
      float xa0, xa1, xb0, xb1;
      if constexpr (kXBf16) {
        const uint32_t ua = pa[kk >> 1], ub = pb[kk >> 1];
        xa0 = __uint_as_float(ua << 16); xa1 = __uint_as_float(ua & 0xFFFF0000u);
        xb0 = __uint_as_float(ub << 16); xb1 = __uint_as_float(ub & 0xFFFF0000u);
      } else {
        xa0 = __uint_as_float(pa[kk]); xa1 = __uint_as_float(pa[kk + 1]);
        xb0 = __uint_as_float(pb[kk]); xb1 = __uint_as_float(pb[kk + 1]);
      }
      const double w_a0 = wa[(size_t)kk * p.E], w_a1 = wa[(size_t)(kk + 1) * p.E];
      const double w_b0 = wb[(size_t)kk * p.E], w_b1 = wb[(size_t)(kk + 1) * p.E];
      acc_a = __fma_rn(static_cast<double>(xa0), w_a0, acc_a);
      acc_b = __fma_rn(static_cast<double>(xb0), w_b0, acc_b);
      mag_a = __dadd_rn(mag_a, fabs(acc_a));
      mag_b = __dadd_rn(mag_b, fabs(acc_b));
      acc_a = __fma_rn(static_cast<double>(xa1), w_a1, acc_a);
      acc_b = __fma_rn(static_cast<double>(xb1), w_b1, acc_b);
      mag_a = __dadd_rn(mag_a, fabs(acc_a));
      mag_b = __dadd_rn(mag_b, fabs(acc_b));
    }
    if (va) p.rpart[oa] = make_double2(acc_a, mag_a);
    if (vb) p.rpart[ob] = make_double2(acc_b, mag_b);
  }
}

// ---------------------------------------------------------------------------
// K6: merge + phase 2.  First every warp merges candidate chains of the CTA's
// tokens (lane l folds segments [l J, (l+1) J) in order, then a shuffle tree
// over the lanes: the merge rule of router_seg.cuh), certifies the result and
// intersects it with the screen interval.  Then one warp per token, lane c =
// candidate c: the k-th largest lower score bound S_k over the candidates
// (the k largest lower bounds of all experts are candidates), exclusion, top-k
// over (score, index) keys, renormalisation (router.py:99-112, the same
// operations as eval_route_outputs).  A token with an unknown or unsure
// non-excluded logit, too many candidates or S_k < 2^-100 takes the general
// path (route_scores_tokens in screen mode: exact chains for what matters).
// ---------------------------------------------------------------------------
MOE_DEVICE void scr_merge(double& C, double& A, double& K, double Cr, double Ar, double Kr) {
  A = A + Ar + Kr * fabs(C);
  C = C + Cr;
  K = K + Kr;
}

template <bool kXBf16>
__global__ void __launch_bounds__(kScrPh2Threads) screen_phase2_kernel(const __grid_constant__ ScreenParams sp,
                                                                       const __grid_constant__ RouterParams p,
                                                                       double cert_coef) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int t0 = blockIdx.x * kScrPh2Tok, t1 = min(sp.B, t0 + kScrPh2Tok);
  // debug timeline (p.trace): per CTA {globaltimer at entry, clock64 deltas}
  unsigned long long* tr = (p.trace && threadIdx.x == 0) ? p.trace + 64 + (size_t)blockIdx.x * 8 : nullptr;
  const long long c_start = clock64();
  if (tr) { tr[0] = globaltimer_ns(); }
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < sp.E; e += blockDim.x) sp.ecount[e] = 0;
  const int J = (sp.n_rs + 31) / 32;
  int nch[kScrPh2Tok] = {};
  int total = 0;
#pragma unroll
  for (int i = 0; i < kScrPh2Tok; ++i) {
    nch[i] = (t0 + i < t1) ? max(0, sp.ncand[t0 + i]) : 0;
    total += nch[i];
  }
  const int j0 = lane * J, j1 = min(sp.n_rs, j0 + J);
  // this warp's chains (ci = warp, warp + nw, ...): the first two chains'
  // partials are loaded together (<= 4 segments per lane each)
  double2 pre[2][4];
  auto chain_of = [&](int ci, int& t, int& c) {
    int ti = 0;
    c = ci;
    while (c >= nch[ti]) { c -= nch[ti]; ++ti; }
    t = t0 + ti;
  };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ci = warp + q * nw;
    if (ci < total) {
      int t, c;
      chain_of(ci, t, c);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < j1) pre[q][u] = __ldcg(sp.rpart + ((size_t)(j0 + u) * sp.B + t) * kScrMaxCand + c);
    }
  }
  for (int ci = warp, q = 0; ci < total; ci += nw, ++q) {
    int t, c;
    chain_of(ci, t, c);
    double C = -0.0, A = 0.0, K = 0.0;
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u < j1) {
        if (q == 0) v[u] = pre[0][u];
        else if (q == 1) v[u] = pre[1][u];
        else v[u] = __ldcg(sp.rpart + ((size_t)(j0 + u) * sp.B + t) * kScrMaxCand + c);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < j1) scr_merge(C, A, K, v[u].x, v[u].y, static_cast<double>(j0 + u == 0 ? sp.rs_first : sp.rs_len));
    for (int jj = j0 + 4; jj < j1; ++jj) {  // (J > 4: more than 128 segments)
      const double2 w = __ldcg(sp.rpart + ((size_t)jj * sp.B + t) * kScrMaxCand + c);
      scr_merge(C, A, K, w.x, w.y, static_cast<double>(sp.rs_len));
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double Cr = __shfl_down_sync(0xffffffffu, C, off);
      const double Ar = __shfl_down_sync(0xffffffffu, A, off);
      const double Kr = __shfl_down_sync(0xffffffffu, K, off);
      if ((lane & (2 * off - 1)) == 0) scr_merge(C, A, K, Cr, Ar, Kr);
    }
    if (lane == 0) {
      const int e = sp.cand[(size_t)t * kScrMaxCand + c];
      const float2 s = sp.lbuf[(size_t)t * sp.E + e];
      float2 r = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
      if (A > 0.0 && isfinite(C) && isfinite(A)) {
        // u A (2 + 12/L)(1 + 2^-20) + 8 u |s| (the merges' roundings of the total)
        const double D = __dadd_ru(__dmul_ru(A, cert_coef), __dmul_ru(fabs(C), 0x1p-50));
        const float lo = fmaxf(s.x, __double2float_rn(__dsub_rd(C, D)));
        const float hi = fminf(s.y, __double2float_rn(__dadd_ru(C, D)));
        if (lo <= hi) r = make_float2(lo, hi);
        if (p.trace && !(lo <= hi)) atomicAdd(p.trace + 1, 1ull);  // debug: empty intersection
        if (p.trace && lo < hi) atomicAdd(p.trace + 2, 1ull);      // debug: refined width > 0
      } else if (p.trace) {
        atomicAdd(p.trace + 0, 1ull);  // debug: refinement inconclusive (A == 0 / non-finite)
      }
      sp.lbuf[(size_t)t * sp.E + e] = r;
    }
  }
  if (tr) tr[1] = clock64() - c_start;
  __syncthreads();
  if (tr) tr[2] = clock64() - c_start;
  // ---- selection, one warp per token
  const int t = t0 + warp;
  if (warp >= kScrPh2Tok || t >= t1) return;
  const int nc = sp.ncand[t];
  bool general = nc <= 0;
  int e = 0;
  float lo = 0.0f, hi = 0.0f, slo = -1.0f, shi = -1.0f;
  if (!general && lane < nc) {
    e = sp.cand[(size_t)t * kScrMaxCand + lane];
    const float2 r = __ldcg(sp.lbuf + (size_t)t * sp.E + e);
    lo = r.x; hi = r.y;
    slo = scr_score_lo(lo);
    shi = scr_score_hi(hi);
  }
  float Sk = 0.0f;
  if (!general) {
    // k-th largest lower bound over the candidate lanes (one instance removed per round)
    float v = slo;
    for (int j = 0; j < p.k; ++j) {
      float m = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const uint32_t own = __ballot_sync(0xffffffffu, v == m);
      if (lane == __ffs(own) - 1) v = -1.0f;
      Sk = m;
    }
    general = !(Sk >= 0x1p-100f);
  }
  const bool alive = !general && lane < nc && !(shi < Sk);
  float score = -1.0f;
  if (alive) {
    // the logit must give one certain score (every candidate fp32 value between lo and hi)
    bool sure = !isnan(lo) && !isnan(hi);
    if (sure) {
      score = np_sigmoid(lo);
      if (!same_bits(lo, hi) && !(lo >= 18.0f)) {
        float c = lo;
        int steps = 0;
        while (sure && !same_bits(c, hi)) {
          c = nextafterf(c, hi);
          sure = (++steps <= 8) && same_bits(np_sigmoid(c), score);
        }
      }
    }
    general = !sure;
  }
  general = __any_sync(0xffffffffu, general);
  if (p.trace && lane == 0) {  // debug: why the general path
    if (nc <= 0) atomicAdd(p.trace + 3, 1ull);
    else if (!(Sk >= 0x1p-100f)) atomicAdd(p.trace + 4, 1ull);
    else if (general) atomicAdd(p.trace + 5, 1ull);
    else atomicAdd(p.trace + 6, 1ull);
  }
  if (general) {
    route_scores_tokens<kXBf16>(p, t, t + 1, smem + (size_t)warp * (sp.E * 16 + kChainWin * 8), warp);
    return;
  }
  // top-k over keys (score bits desc, expert index asc); scores >= +0
  uint32_t key = alive ? ((score == 0.0f ? 0u : __float_as_uint(score)) + 1u) : 0u;
  float wsel = 0.0f;
  int isel = 0;
  for (int j = 0; j < p.k; ++j) {
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
    const int eb = static_cast<int>(__reduce_min_sync(0xffffffffu, key == kmax ? static_cast<uint32_t>(e) : 0xFFFFFFFFu));
    if (key == kmax && e == eb) key = 0u;
    if (lane == j) { wsel = __uint_as_float(kmax - 1u); isel = eb; }
  }
  // renormalise with numpy's fp32 pairwise sum over the k selected (selection order)
  float* wrow = reinterpret_cast<float*>(smem + (size_t)kScrPh2Tok * (sp.E * 16 + kChainWin * 8)) + warp * 32;
  if (lane < p.k) wrow[lane] = wsel;
  __syncwarp();
  float S = 0.0f;
  if (lane == 0) S = pairwise_sum<float>(wrow, p.k);
  S = __shfl_sync(0xffffffffu, S, 0);
  const float uni = __double2float_rn(1.0 / static_cast<double>(p.k));
  if (lane < p.k) {
    p.topk_idx[(size_t)t * p.k + lane] = isel;
    p.topk_w[(size_t)t * p.k + lane] = (S == 0.0f) ? uni : __fdiv_rn(wsel, S);
  }
  if (tr) { tr[3] = clock64() - c_start; tr[4] = globaltimer_ns(); }
}

}  // namespace moe
