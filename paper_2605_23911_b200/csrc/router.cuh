// router.cuh — bit-exact router + scheduler, one launch.
//
// Reference semantics (cited per step):
//   logits  = tokens @ W_r, fp64 exact products, ascending-k fold, one fp32
//             rounding                          (linalg.py:45-57, router.py:131)
//   softmax = fp32 max-subtract, fp64 exp, numpy pairwise fp64 row sum,
//             fp64 divide, fp32 round           (router.py:78-83)
//   sigmoid = float32 split-form logistic with numpy's SIMD expf
//                                                 (linalg.py:71-80)
//   top-k   = k rounds of argmax, lowest index on ties, -1.0 masking
//             == k largest keys (score desc, index asc) (router.py:99-107)
//   sigmoid renormalisation by the fp32 pairwise sum, 1/k on zero sum
//                                                 (router.py:108-112)
//   histogram / offsets / stable permutation    (scheduler.py:78-103)
//   block schedule (device tile table)          (scheduler.py:106-117)
//
// Launch structure: grid = (token blocks) x (expert blocks).  Phase 1: every
// CTA runs TOKC x EXPC sequential fp64 FMA chains (TG chains per thread for
// ILP), staging x / W_r chunks through a cp.async ring and an fp64 smem
// buffer.  Phase 2: the last CTA to finish a token block (atomic counter)
// computes scores and top-k for it, one warp per token.  Phase 3: the last
// token block to finish builds counts, offsets, the stable permutation and
// the GEMM tile table in one CTA.  All counters self-reset.
#pragma once

#include "common.cuh"

namespace moe {

constexpr int kRouterKC = 128;     // W64 padding granularity (max k-chunk)
constexpr int kMaxExperts = 1024;

struct RouterParams {
  const void* x;        // (B, d) fp32 or bf16
  const float* wr;      // (d, E) fp32
  const double* w64;    // prepared W64[eb][d_pad][expc] (router_prep_kernel)
  int x_bf16;
  int B, d, E, k, gating;
  int tokc, expc;       // CTA tile: tokc tokens x expc experts
  int stages;           // smem pipeline depth
  int n_eblocks, n_tblocks;
  int chunk_rows;       // GEMM row-chunk cap (BN)
  float* logits;        // (B, E) fp32
  int32_t* topk_idx;    // (B, k)
  float* topk_w;        // (B, k)
  int32_t* counts;      // (E)
  int32_t* offsets;     // (E+1)
  int32_t* fwd;         // (T)
  int32_t* inv;         // (T)
  int4* chunk_tab;      // (max_chunks) {expert, row0, nrows, padded row0}
  int32_t* prow;        // (T) expanded id -> padded permuted row (experts start 16-aligned)
  int32_t* n_chunks;    // [1]
  int32_t* tb_counter;  // (n_tblocks) self-resetting
  int32_t* done_counter;// [1] self-resetting
  uint32_t* flags;      // [1]
  unsigned long long* trace;  // debug: CTA 0 per-chunk {issue, rawfull seen, full seen, compute done}
};

// ---------------------------------------------------------------------------
// numpy-compatible pairwise sum (numpy loops_utils pairwise_sum; verified
// against ndarray.sum in tests/test_host.py for every n used here).
// ---------------------------------------------------------------------------
template <typename T>
MOE_DEVICE T pairwise_sum_block(const T* a, int n) {
  // n <= 128
  if (n < 8) {
    T res = T(0);
    for (int i = 0; i < n; ++i) res = res + a[i];
    return res;
  }
  T r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = r0 + a[i + 0]; r1 = r1 + a[i + 1]; r2 = r2 + a[i + 2]; r3 = r3 + a[i + 3];
    r4 = r4 + a[i + 4]; r5 = r5 + a[i + 5]; r6 = r6 + a[i + 6]; r7 = r7 + a[i + 7];
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + a[i];
  return res;
}

template <typename T>
MOE_DEVICE T pairwise_sum(const T* a, int n) {
  // Iterative form of numpy's recursion: n > 128 splits at n2 = n/2 - (n/2)%8.
  // Depth is at most 3 for n <= 1024; an explicit stack keeps it non-recursive.
  if (n <= 128) return pairwise_sum_block(a, n);
  struct Frame { int lo, n, state; T left; };
  Frame st[8];
  int sp = 0;
  st[0] = {0, n, 0, T(0)};
  T ret = T(0);
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_sum_block(a + f.lo, f.n);
      --sp;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.lo, n2, 0, T(0)};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + n2, f.n - n2, 0, T(0)};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

// ---------------------------------------------------------------------------
// numpy float32 exp (AVX512F/AVX2 SIMD kernel), reconstructed per SURVEY
// Appendix A step 3 and checked against np.exp (tests).  Every operation is
// an explicit round-to-nearest intrinsic so nvcc cannot contract it.
// ---------------------------------------------------------------------------
MOE_DEVICE float np_expf(float x) {
  if (x <= -103.97208404541015625f) return 0.0f;
  if (x >= 88.72283935546875f) return __int_as_float(0x7f800000);
  float q = __fmul_rn(x, 1.442695040888963407359924681001892137f);
  q = __fsub_rn(__fadd_rn(q, 0x1.8p+23f), 0x1.8p+23f);
  float r = __fmaf_rn(q, -6.93145752e-1f, x);
  r = __fmaf_rn(q, -1.42860677e-6f, r);
  r = __fmaf_rn(q, 0.0f, r);
  float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
  num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
  num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
  num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
  num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);
  float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
  den = __fmaf_rn(den, r, 1.0f);
  float p = __fdiv_rn(num, den);
  // p * 2^q with a single rounding (scalef): exact in fp64, then one fp32 rounding.
  const long long qe = static_cast<long long>(static_cast<int>(q) + 1023) << 52;  // 2^q, q in [-150, 128]
  return __double2float_rn(static_cast<double>(p) * __longlong_as_double(qe));
}

MOE_DEVICE unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

MOE_DEVICE float np_sigmoid(float x) {
  float t = np_expf(-fabsf(x));
  float den = __fadd_rn(1.0f, t);
  return x >= 0.0f ? __fdiv_rn(1.0f, den) : __fdiv_rn(t, den);
}

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
MOE_DEVICE uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v), m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), m);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

MOE_DEVICE void cp_async_16(void* smem, const void* gmem, bool valid) {
  uint32_t s = smem_u32(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz)
               : "memory");
}
MOE_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MOE_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kRouterProducers = 128;  // 4 warps: W bulk copies + x fp64 conversion
constexpr int kRouterMaxStages = 12;

// ---------------------------------------------------------------------------
// Router weight preparation (once per weight): W64[eb][k][expc] fp64, the
// exact widening of the fp32 router weight, zero-padded to whole k-chunks and
// expert blocks, so a chunk of an expert block is ONE contiguous bulk copy.
// Non-finite entries set flag bit 2 (NonFiniteInput on router_weight).
// ---------------------------------------------------------------------------
__global__ void router_prep_kernel(const float* __restrict__ wr, double* __restrict__ w64, int d, int E,
                                   int expc, int d_pad, int n_eblocks, uint32_t* flags) {
  const long total = (long)n_eblocks * d_pad * expc;
  bool bad = false;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int el = static_cast<int>(i % expc);
    const long r = i / expc;
    const int k = static_cast<int>(r % d_pad);
    const int eb = static_cast<int>(r / d_pad);
    const int e = eb * expc + el;
    float v = 0.0f;
    if (k < d && e < E) {
      v = __ldg(wr + (size_t)k * E + e);
      if (!isfinite(v)) bad = true;
    }
    w64[i] = static_cast<double>(v);
  }
  if (bad) atomicOr(flags, 2u);
}

MOE_DEVICE void bulk_load_smem(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------------------
// Shared memory of phase 1: p.stages x {W chunk (KC x expc fp64),
// x chunk (tokc x (KC+1) fp64)} + mbarriers full[s], empty[s].
// ---------------------------------------------------------------------------
struct RouterSmem {
  static __host__ __device__ size_t w_bytes(int expc, int kc) { return (size_t)kc * expc * 8; }
  static __host__ __device__ size_t x_bytes(int tokc, int kc) { return ((size_t)tokc * (kc + 1) * 8 + 127) / 128 * 128; }
  static __host__ __device__ size_t raw_bytes(int tokc, int xb, int kc) { return ((size_t)tokc * kc * xb + 127) / 128 * 128; }
  static __host__ __device__ size_t stage_bytes(int tokc, int expc, int xb, int kc) {
    return w_bytes(expc, kc) + x_bytes(tokc, kc) + raw_bytes(tokc, xb, kc);
  }
  static __host__ __device__ size_t total_bytes(int tokc, int expc, int xb, int E, int nthreads, int stages, int kc) {
    size_t ph1 = stages * stage_bytes(tokc, expc, xb, kc) + 3 * stages * 8;
    size_t ph2 = (size_t)(nthreads / 32) * E * sizeof(double);
    size_t ph3 = ((size_t)(nthreads / 32) + 5) * E * sizeof(int32_t) + 512;
    size_t m = ph1 > ph2 ? ph1 : ph2;
    return m > ph3 ? m : ph3;
  }
};

// Launch shape: blockDim = n_compute + kRouterProducers.  Compute threads own a
// kTE x kTT register tile of independent sequential fp64 chains; the producer
// warps fill stage s: one elected thread bulk-copies the W64 chunk (tx-count on
// full[s]), all 128 convert the x chunk to fp64 (one arrival each).  Compute
// warps release stages through empty[s] (one arrival per warp).
template <bool kXBf16, int kTE, int kTT, int kKC>
__global__ void __launch_bounds__(384)
router_kernel(const __grid_constant__ CUtensorMap tm_x, const RouterParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int n_compute = nthreads - kRouterProducers;
  const int n_cwarps = n_compute / 32;
  const int tb = blockIdx.x / p.n_eblocks;
  const int eb = blockIdx.x % p.n_eblocks;
  const int t0 = tb * p.tokc;
  const int e0 = eb * p.expc;

  // ------------------------------- phase 1: logits ---------------------------
  const int xb = kXBf16 ? 2 : 4;
  const size_t wbytes = RouterSmem::w_bytes(p.expc, kKC);
  const size_t xbytes = RouterSmem::x_bytes(p.tokc, kKC);
  const size_t sbytes = RouterSmem::stage_bytes(p.tokc, p.expc, xb, kKC);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * sbytes);
  uint64_t* empty = full + p.stages;
  uint64_t* rawfull = empty + p.stages;
  const int nch = (p.d + kKC - 1) / kKC;
  const int d_pad = (p.d + kRouterKC - 1) / kRouterKC * kRouterKC;
  const int ntok = min(p.tokc, p.B - t0);  // valid token rows of this block
  if (p.trace && threadIdx.x == 0) p.trace[4096 * 4 + 2048 * 4 + blockIdx.x] = globaltimer_ns();
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, kRouterProducers + 1);
      mbar_init(empty + s, n_cwarps);
      mbar_init(rawfull + s, 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (tid >= n_compute) {
    // ============================ producers ================================
    // The elected producer keeps p.stages-1 chunks of async copies in
    // flight (W64 chunk -> full[s], raw x rows -> rawfull[s]); all producers
    // convert each landed raw x chunk to fp64 and arrive on full[s].
    const int ptid = tid - n_compute;
    bool nonfinite_x = false;
    const double* wsrc = p.w64 + (size_t)eb * d_pad * p.expc;
    auto issue = [&](int c) {
      const int s = c % p.stages;
      const uint32_t ph = (c / p.stages) & 1;
      mbar_wait(empty + s, ph ^ 1);
      uint8_t* st = smem + s * sbytes;
      mbar_arrive_expect_tx(full + s, static_cast<uint32_t>(wbytes));
      if (p.trace && blockIdx.x == 0) p.trace[c * 4 + 0] = clock64();
      bulk_load_smem(st, wsrc + (size_t)c * kKC * p.expc, static_cast<uint32_t>(wbytes), full + s);
      // one 2-D TMA tile (KC x tokc, OOB rows/cols zero-filled) per chunk
      mbar_arrive_expect_tx(rawfull + s, static_cast<uint32_t>(p.tokc * kKC * xb));
      tma_load_2d(&tm_x, rawfull + s, st + wbytes + xbytes, c * kKC, t0);
    };
    if (ptid == 0)
      for (int c = 0; c < min(nch, p.stages - 1); ++c) issue(c);
    const int nx = p.tokc * kKC;
    for (int c = 0; c < nch; ++c) {
      const int s = c % p.stages;
      const uint32_t ph = (c / p.stages) & 1;
      mbar_wait(rawfull + s, ph);
      if (p.trace && blockIdx.x == 0 && ptid == 0) p.trace[c * 4 + 1] = clock64();
      uint8_t* st = smem + s * sbytes;
      double* dx = reinterpret_cast<double*>(st + wbytes);
      const uint8_t* raw = st + wbytes + xbytes;
      const int kv = min(kKC, p.d - c * kKC);
      for (int i = ptid; i < nx; i += kRouterProducers) {
        const int row = i / kKC, kk = i % kKC;
        float v = 0.0f;
        if (row < ntok && kk < kv) {
          if (kXBf16) v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(raw)[i]);
          else v = reinterpret_cast<const float*>(raw)[i];
          if (!isfinite(v)) nonfinite_x = true;
        }
        dx[row * (kKC + 1) + kk] = static_cast<double>(v);
      }
      mbar_arrive(full + s);
      // refill: chunk c+S-1 goes into the stage of chunk c-1 once compute released it
      if (ptid == 0 && c + p.stages - 1 < nch) issue(c + p.stages - 1);
    }
    if (nonfinite_x) atomicOr(p.flags, 1u);
  } else {
    // ============================ compute chains ===========================
    // Experts e0 + eg + i*n_eg, tokens t0 + tg + j*n_tg: the warp's W loads are
    // contiguous and its x loads near-broadcast; operands are register
    // double-buffered U steps ahead of the dependent FMA chain.
    const int n_eg = p.expc / kTE;
    const int n_tg = p.tokc / kTT;
    const int eg = tid % n_eg;
    const int tg = tid / n_eg;
    const bool active = tg < n_tg;
    double acc[kTE][kTT];
#pragma unroll
    for (int i = 0; i < kTE; ++i)
#pragma unroll
      for (int j = 0; j < kTT; ++j) acc[i][j] = -0.0;  // fma(a,b,-0) == a*b exactly, sign included
    constexpr int XS = kKC + 1;  // padded fp64 x row
    const int lane = tid & 31;
    for (int c = 0; c < nch; ++c) {
      const int s = c % p.stages;
      const uint32_t ph = (c / p.stages) & 1;
      mbar_wait(full + s, ph);
      if (p.trace && blockIdx.x == 0 && tid == 0) p.trace[c * 4 + 2] = clock64();
      if (active) {
        const uint8_t* st = smem + s * sbytes;
        const double* dw = reinterpret_cast<const double*>(st) + eg;
        const double* dx = reinterpret_cast<const double*>(st + wbytes) + (size_t)tg * XS;
        const int xstep = n_tg * XS;
        // the last chunk may be partial: only k < d is folded, like the reference
        // plain loop: the compiler keeps operand loads ~6 steps ahead of the chain
        // without register-reuse (WAR) stalls (probe: 10.3 vs 13.9 cycles/step)
        const int kvalid = min(kKC, p.d - c * kKC);
        if (kvalid == kKC) {
#pragma unroll 16
          for (int kk = 0; kk < kKC; ++kk) {
#pragma unroll
            for (int i = 0; i < kTE; ++i) {
              const double w = dw[kk * p.expc + i * n_eg];
#pragma unroll
              for (int j = 0; j < kTT; ++j) acc[i][j] = __fma_rn(dx[j * xstep + kk], w, acc[i][j]);
            }
          }
        } else {
          for (int kk = 0; kk < kvalid; ++kk) {
#pragma unroll
            for (int i = 0; i < kTE; ++i) {
              const double w = dw[kk * p.expc + i * n_eg];
#pragma unroll
              for (int j = 0; j < kTT; ++j) acc[i][j] = __fma_rn(dx[j * xstep + kk], w, acc[i][j]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (p.trace && blockIdx.x == 0 && tid == 0) p.trace[c * 4 + 3] = clock64();
    }
    if (active) {
#pragma unroll
      for (int i = 0; i < kTE; ++i) {
        const int e = e0 + eg + i * n_eg;
#pragma unroll
        for (int j = 0; j < kTT; ++j) {
          const int t = t0 + tg + j * n_tg;
          if (t < p.B && e < p.E && eg + i * n_eg < p.expc)
            p.logits[(size_t)t * p.E + e] = __double2float_rn(acc[i][j]);
        }
      }
    }
  }

  if (p.trace && tid == 0) p.trace[4096 * 4 + blockIdx.x * 4 + 0] = globaltimer_ns();
  // --------------------- phase 2: scores + top-k (last CTA of block) --------
  __shared__ int s_flag;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int prev = atomicAdd(p.tb_counter + tb, 1);
    s_flag = (prev == p.n_eblocks - 1);
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();

  {
    const int warp = tid / 32, lane = tid % 32;
    double* row = reinterpret_cast<double*>(smem) + (size_t)warp * p.E;
    const int tend = min(t0 + p.tokc, p.B);
    for (int t = t0 + warp; t < tend; t += nthreads / 32) {
      const float* lg = p.logits + (size_t)t * p.E;
      // scores -> row (as double for softmax, float bits stored in double for sigmoid)
      if (p.gating == 0) {
        float m = -__int_as_float(0x7f800000);
        for (int e = lane; e < p.E; e += 32) m = fmaxf(m, __ldcg(lg + e));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        for (int e = lane; e < p.E; e += 32) {
          float s = __fsub_rn(__ldcg(lg + e), m);
          row[e] = exp(static_cast<double>(s));
        }
        __syncwarp();
        double S = 0.0;
        if (lane == 0) S = pairwise_sum<double>(row, p.E);
        S = __shfl_sync(0xffffffffu, S, 0);
        __syncwarp();
        for (int e = lane; e < p.E; e += 32) {
          float sc = __double2float_rn(__ddiv_rn(row[e], S));
          row[e] = static_cast<double>(sc);
        }
      } else {
        for (int e = lane; e < p.E; e += 32) row[e] = static_cast<double>(np_sigmoid(__ldcg(lg + e)));
      }
      __syncwarp();
      // top-k over keys (score bits desc, index asc); scores are >= +0.
      float wsel = 0.0f;
      int isel = 0;
      for (int j = 0; j < p.k; ++j) {
        uint64_t best = 0;
        for (int e = lane; e < p.E; e += 32) {
          float sc = static_cast<float>(row[e]);
          if (sc < 0.0f) continue;  // already selected (marked -1)
          uint32_t bits = (sc == 0.0f) ? 0u : __float_as_uint(sc);
          uint64_t key = (static_cast<uint64_t>(bits) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(e));
          best = key > best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          uint64_t other = shfl_xor_u64(best, o);
          best = other > best ? other : best;
        }
        int e_best = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFu));
        float s_best = __uint_as_float(static_cast<uint32_t>(best >> 32));
        __syncwarp();
        if (lane == (e_best & 31)) row[e_best] = -1.0;
        __syncwarp();
        if (lane == j) { wsel = s_best; isel = e_best; }
        if (j >= 32) {  // k > 32: write directly (rare)
          if (lane == 0) {
            p.topk_idx[(size_t)t * p.k + j] = e_best;
            p.topk_w[(size_t)t * p.k + j] = s_best;
          }
        }
      }
      __syncwarp();
      if (p.gating == 1) {
        // renormalise over the selected k with numpy's fp32 pairwise sum
        float* wrow = reinterpret_cast<float*>(row);
        if (lane < p.k && lane < 32) wrow[lane] = wsel;
        __syncwarp();
        if (p.k > 32 && lane == 0) {
          for (int j = 32; j < p.k; ++j) wrow[j] = p.topk_w[(size_t)t * p.k + j];
        }
        __syncwarp();
        float S = 0.0f;
        if (lane == 0) S = pairwise_sum<float>(wrow, p.k);
        S = __shfl_sync(0xffffffffu, S, 0);
        const float uni = __double2float_rn(1.0 / static_cast<double>(p.k));
        if (lane < p.k) wsel = (S == 0.0f) ? uni : __fdiv_rn(wsel, S);
        if (p.k > 32 && lane == 0) {
          for (int j = 32; j < p.k; ++j) {
            float v = wrow[j];
            p.topk_w[(size_t)t * p.k + j] = (S == 0.0f) ? uni : __fdiv_rn(v, S);
          }
        }
        __syncwarp();
      }
      if (lane < p.k) {
        p.topk_idx[(size_t)t * p.k + lane] = isel;
        p.topk_w[(size_t)t * p.k + lane] = wsel;
      }
      __syncwarp();
    }
  }

  if (p.trace && tid == 0) p.trace[4096 * 4 + blockIdx.x * 4 + 1] = globaltimer_ns();
  // -------------------- phase 3: scheduler (last token block) ---------------
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    p.tb_counter[tb] = 0;  // every CTA of this block has arrived: reset for the next launch
    int prev = atomicAdd(p.done_counter, 1);
    s_flag = (prev == p.n_tblocks - 1);
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();

  {
    const int nw = nthreads / 32;
    const int warp = tid / 32, lane = tid % 32;
    const int T = p.B * p.k;
    const int E = p.E;
    int32_t* hist = reinterpret_cast<int32_t*>(smem);       // [nw][E] -> per-warp base
    int32_t* s_cnt = hist + (size_t)nw * E;                  // [E]
    int32_t* s_off = s_cnt + E;                              // [E+1]
    int32_t* s_cpre = s_off + E + 1;                         // [E+1] chunk prefix
    int32_t* s_off16 = s_cpre + E + 1;                       // [E+1] 16-padded offsets
    for (int i = tid; i < nw * E; i += nthreads) hist[i] = 0;
    __syncthreads();
    const int seg = (T + nw - 1) / nw;
    const int s0 = warp * seg, s1 = min(T, s0 + seg);
    for (int i = s0 + lane; i < s1; i += 32) atomicAdd(&hist[warp * E + __ldcg(p.topk_idx + i)], 1);
    __syncthreads();
    // per-expert totals and per-warp exclusive bases
    for (int e = tid; e < E; e += nthreads) {
      int run = 0;
      for (int w = 0; w < nw; ++w) {
        int h = hist[w * E + e];
        hist[w * E + e] = run;
        run += h;
      }
      s_cnt[e] = run;
    }
    __syncthreads();
    // warp 0: exclusive scans of counts and of chunk counts
    if (warp == 0) {
      const int per = (E + 31) / 32;
      const int lo = lane * per, hi = min(E, lo + per);
      int sum_c = 0, sum_ch = 0, sum_16 = 0;
      for (int e = lo; e < hi; ++e) {
        sum_c += s_cnt[e];
        sum_ch += (s_cnt[e] + p.chunk_rows - 1) / p.chunk_rows;
        sum_16 += (s_cnt[e] + 15) & ~15;
      }
      int inc_c = sum_c, inc_ch = sum_ch, inc_16 = sum_16;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(0xffffffffu, inc_c, o);
        int b = __shfl_up_sync(0xffffffffu, inc_ch, o);
        int c = __shfl_up_sync(0xffffffffu, inc_16, o);
        if (lane >= o) { inc_c += a; inc_ch += b; inc_16 += c; }
      }
      int run_c = inc_c - sum_c, run_ch = inc_ch - sum_ch, run_16 = inc_16 - sum_16;
      for (int e = lo; e < hi; ++e) {
        s_off[e] = run_c;
        s_cpre[e] = run_ch;
        s_off16[e] = run_16;
        run_c += s_cnt[e];
        run_ch += (s_cnt[e] + p.chunk_rows - 1) / p.chunk_rows;
        run_16 += (s_cnt[e] + 15) & ~15;
      }
      if (lane == 31) {
        s_off[E] = inc_c;
        s_cpre[E] = inc_ch;
        s_off16[E] = inc_16;
      }
    }
    __syncthreads();
    for (int e = tid; e < E; e += nthreads) {
      p.counts[e] = s_cnt[e];
      p.offsets[e] = s_off[e];
      const int n_e = s_cnt[e];
      const int nchunk = (n_e + p.chunk_rows - 1) / p.chunk_rows;
      for (int c = 0; c < nchunk; ++c) {
        int r0 = c * p.chunk_rows;
        p.chunk_tab[s_cpre[e] + c] = make_int4(e, s_off[e] + r0, min(p.chunk_rows, n_e - r0), s_off16[e] + r0);
      }
    }
    if (tid == 0) {
      p.offsets[E] = s_off[E];
      p.n_chunks[0] = s_cpre[E];
    }
    // stable counting sort: warp w walks its segment in id order
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int base = s0; base < s1; base += 32) {
      int i = base + lane;
      bool valid = i < s1;
      int e = valid ? __ldcg(p.topk_idx + i) : -1 - lane;  // unique sentinel per invalid lane
      uint32_t peers = __match_any_sync(0xffffffffu, e);
      if (valid) {
        int rank = __popc(peers & lt_mask);
        int pos = s_off[e] + hist[warp * E + e] + rank;
        p.fwd[pos] = i;
        p.inv[i] = pos;
        if (p.prow) p.prow[i] = s_off16[e] + (pos - s_off[e]);
      }
      __syncwarp();
      if (valid && (__ffs(peers) - 1) == static_cast<int>(lane)) hist[warp * E + e] += __popc(peers);
      __syncwarp();
    }
    if (tid == 0) *p.done_counter = 0;
    if (p.trace && tid == 0) {
      p.trace[4096 * 4 + blockIdx.x * 4 + 2] = 1;
      p.trace[4096 * 4 + blockIdx.x * 4 + 3] = globaltimer_ns();
    }
  }
}

}  // namespace moe
