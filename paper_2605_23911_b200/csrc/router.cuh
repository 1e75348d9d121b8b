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
//   (histogram / offsets / stable permutation / schedule: dispatch.cuh)
//
// Two phase-1 kernels produce certified logit intervals (lbuf):
//  * router_kernel (this file, throughput regime): grid = (token blocks) x
//    (expert blocks); every CTA runs TOKC x EXPC exact sequential fp64 FMA
//    chains (register tiles for ILP), staging x / W_r chunks through an
//    mbarrier ring and an fp64 smem buffer; intervals have zero width.
//  * router_seg_kernel (router_seg.cuh, latency regime): certified split-K.
// Phase 2 (route_scores_tokens): the last CTA to finish a token block (atomic
// counter) computes scores and top-k for it, one warp per token.  All
// counters self-reset.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace moe {

constexpr int kRouterKC = 128;     // W64 padding granularity (max k-chunk)
constexpr int kMaxExperts = 1024;
constexpr int kChainWin = 128;  // exact fallback: steps per shared-memory product window

struct RouterParams {
  const void* x;        // (B, d) fp32 or bf16
  const float* wr;      // (d, E) fp32
  const double* w64;    // prepared W64[eb][d_pad][expc] (router_prep_kernel)
  const double* wlin64; // segment kernel, W widened to fp64 in its (d, E) layout (widen_f64_kernel)
  int x_bf16;
  int B, d, E, k, gating;
  int tokc, expc;       // CTA tile: tokc tokens x expc experts
  int stages;           // smem pipeline depth
  int n_eblocks, n_tblocks;
  int chunk_rows;       // GEMM row-chunk cap (BN)
  float* logits;        // (B, E) fp32 exact logits, written only when want_logits
  float2* lbuf;         // (B, E) certified logit interval {lo, hi} (fp32); lo = NaN: unknown
  int want_logits;      // 1: resolve every logit exactly and write `logits`
  int force_exact;      // test hook: certificates report "unknown" (exact fallback for every logit)
  double cert_coef;     // segment kernel: D = A * cert_coef = u (2 + 12/L)(1 + 2^-20)
  int kr, seg_len, n_kb;// segment kernel: k-range per CTA, segment length, k-blocks
  int32_t* blk_counter; // (n_tblocks * n_eblocks) self-resetting (segment kernel)
  void* gpart;          // segment kernel: per (block, k-block, chain) {C_b, A_b} fp64
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
  uint32_t* flags;      // [1]
  unsigned long long* trace;  // debug: CTA 0 per-chunk {issue, rawfull seen, full seen, compute done}
  // small batches (segment kernel, B*k <= kFuseMaxT): the last phase-2 CTA
  // also runs the dispatch (dispatch.cuh dispatch_small_cta)
  int fuse_dispatch;
  __nv_bfloat16* xp;    // permuted-token gather target (null: no gather)
  int2* chunk_grp;      // {first chunk of the expert, chunks of the expert}
  int32_t* disp_counter;// self-resetting (token blocks that finished phase 2)
  // screen mode (router_screen.cuh): lbuf holds screen intervals (refined for
  // the candidates); phase 2 first excludes the experts that cannot reach the top-k
  int screen;
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

// Warp-cooperative form of the same sum (identical bits, every add in the same
// order): for a block of n <= 128 values, lanes 0..7 run the eight strided
// accumulators r[j] = a[j] + a[j+8] + ... in parallel, the fixed
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree runs on shuffles, and the tail is
// added in order; n <= 256 splits once at numpy's n2 (the halves on lanes
// 0..7 and 8..15).  All lanes return the sum.  Larger n: one lane, serially.
template <typename T>
MOE_DEVICE T pairwise_block_warp(const T* a, int n, int lane, int base) {
  // lanes base..base+7 hold the strided accumulators of a[0 .. n)
  const int j = lane - base;
  T r = T(0);
  if (n >= 8 && j >= 0 && j < 8) {
    r = a[j];
    for (int i = 8 + j; i < n - (n % 8); i += 8) r = r + a[i];
  }
  // tree over lanes base..base+7 (other lanes compute garbage, unused)
  const T r1 = __shfl_down_sync(0xffffffffu, r, 1);
  const T p01 = r + r1;                          // valid at even j: r_j + r_{j+1}
  const T q = __shfl_down_sync(0xffffffffu, p01, 2);
  const T p0123 = p01 + q;                       // valid at j % 4 == 0
  const T h = __shfl_down_sync(0xffffffffu, p0123, 4);
  T res = p0123 + h;                             // valid at j == 0
  res = __shfl_sync(0xffffffffu, res, base);
  if (n < 8) {
    res = T(0);
    for (int i = 0; i < n; ++i) res = res + a[i];
    return res;
  }
  for (int i = n - (n % 8); i < n; ++i) res = res + a[i];
  return res;
}

template <typename T>
MOE_DEVICE T pairwise_sum_warp(const T* a, int n, int lane) {
  if (n <= 128) return pairwise_block_warp(a, n, lane, 0);
  if (n <= 256) {
    int n2 = n / 2;
    n2 -= n2 % 8;  // both halves <= 128 for n <= 256
    const T left = pairwise_block_warp(a, n2, lane, 0);
    const T right = pairwise_block_warp(a + n2, n - n2, lane, 8);
    return left + right;
  }
  T s = T(0);
  if (lane == 0) s = pairwise_sum(a, n);
  return __shfl_sync(0xffffffffu, s, 0);
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

// numpy's float64 exp on x86-64 with AVX-512 (SIMD dispatch to Intel SVML's
// __svml_exp8_ha, vendored in numpy), reconstructed from its machine code and
// constant tables and checked bit-exact against np.exp on every float32 input
// in (-707.70, 0] (tests/test_gpu_stage_api.py, on the box's own numpy).
// Tang-style: n = RZ(x / ln2 * 16) with a shifter, j = n mod 16, r = x - n ln2/16
// (two-part ln2), degree-6 polynomial, 2^(j/16) as top + tail, scalef by
// floor(n / 16).  The softmax (router.py:78-83) only ever feeds it
// s = fp32(l - max) <= 0; for s <= -707.70 (SVML's separate rare path) it
// returns +0: such terms (< 2^-1000) never change the pairwise sum (which
// holds exp(0) = 1) nor their own fp32 score (0) -- the softmax's bits are
// those of numpy either way.
__device__ __constant__ uint64_t kNpExpTop[16] = {
    0x3ff0000000000000ull, 0x3ff0b5586cf9890full, 0x3ff172b83c7d517bull, 0x3ff2387a6e756238ull,
    0x3ff306fe0a31b715ull, 0x3ff3dea64c123422ull, 0x3ff4bfdad5362a27ull, 0x3ff5ab07dd485429ull,
    0x3ff6a09e667f3bcdull, 0x3ff7a11473eb0187ull, 0x3ff8ace5422aa0dbull, 0x3ff9c49182a3f090ull,
    0x3ffae89f995ad3adull, 0x3ffc199bdd85529cull, 0x3ffd5818dcfba487ull, 0x3ffea4afa2a490daull};
__device__ __constant__ uint64_t kNpExpTail[16] = {
    0x0000000000000000ull, 0x3c979aa65d837b6dull, 0xbc801b15eaa59348ull, 0x3c968efde3a8a894ull,
    0x3c834d754db0abb6ull, 0x3c859f48a72a4c6dull, 0x3c7690cebb7aafb0ull, 0x3c9063e1e21c5409ull,
    0xbc93b3efbf5e2228ull, 0xbc7b32dcb94da51dull, 0x3c8db72fc1f0eab4ull, 0x3c71affc2b91ce27ull,
    0x3c8c1a7792cb3387ull, 0x3c736eae30af0cb3ull, 0x3c74a385a63d07a7ull, 0xbc8ff7128fd391f0ull};

MOE_DEVICE double np_exp64(double x) {
  if (!(fabs(x) < 707.7032713517042)) return x < 0.0 ? 0.0 : exp(x);  // (softmax: x <= 0 always)
  const double inv_ln2 = __longlong_as_double(0x3ff71547652b82feLL);
  const double shifter = __longlong_as_double(0x42f8000000003ff0LL);
  const double ln2_hi = __longlong_as_double(0x3fe62e42fefa39efLL);
  const double ln2_lo = __longlong_as_double(0x3c7abc9e3b39803fLL);
  const double c6 = __longlong_as_double(0x3f57411836940c04LL), c5 = __longlong_as_double(0x3f81101cbbc265c0LL);
  const double c4 = __longlong_as_double(0x3fa55557242d68feLL), c3 = __longlong_as_double(0x3fc5555553939732LL);
  const double c2 = __longlong_as_double(0x3fe000000000d008LL), c1 = __longlong_as_double(0x3fefffffffffff70LL);
  const double t = __fma_rz(x, inv_ln2, shifter);
  const double n = __dsub_rn(t, shifter);
  const int j = static_cast<int>(__double_as_longlong(t) & 15);
  double r = __fma_rn(-n, ln2_hi, x);
  r = __fma_rn(-ln2_lo, n, r);
  r = __longlong_as_double(__double_as_longlong(r) & 0xbfffffffffffffffLL);
  const double r2 = __dmul_rn(r, r);
  double a = __fma_rn(c6, r, c5);
  const double b = __fma_rn(c4, r, c3);
  const double c = __fma_rn(c2, r, c1);
  a = __fma_rn(r2, a, b);
  a = __fma_rn(r2, a, c);
  const double top = __longlong_as_double(static_cast<long long>(kNpExpTop[j]));
  const double p = __fma_rn(a, r, __longlong_as_double(static_cast<long long>(kNpExpTail[j])));
  const double res = __fma_rn(top, p, top);
  // scalef(res, floor(n)): exact -- res * 2^m stays normal for |x| < 707.7
  const int m = static_cast<int>(floor(n));
  return __dmul_rn(res, __longlong_as_double(static_cast<long long>(m + 1023) << 52));
}

// np_exp64 for a whole warp (every lane calls it, uniform control flow): the
// 2^(j/16) table entries come from lanes j of (top_i, tail_i) by shuffles
// instead of divergent constant-cache reads (16 distinct addresses serialise).
// Same operations, same bits as np_exp64.
MOE_DEVICE double np_exp64_warp(double x, double top_i, double tail_i) {
  const bool big = !(fabs(x) < 707.7032713517042);
  const double xs = big ? 0.0 : x;
  const double inv_ln2 = __longlong_as_double(0x3ff71547652b82feLL);
  const double shifter = __longlong_as_double(0x42f8000000003ff0LL);
  const double ln2_hi = __longlong_as_double(0x3fe62e42fefa39efLL);
  const double ln2_lo = __longlong_as_double(0x3c7abc9e3b39803fLL);
  const double c6 = __longlong_as_double(0x3f57411836940c04LL), c5 = __longlong_as_double(0x3f81101cbbc265c0LL);
  const double c4 = __longlong_as_double(0x3fa55557242d68feLL), c3 = __longlong_as_double(0x3fc5555553939732LL);
  const double c2 = __longlong_as_double(0x3fe000000000d008LL), c1 = __longlong_as_double(0x3fefffffffffff70LL);
  const double t = __fma_rz(xs, inv_ln2, shifter);
  const double n = __dsub_rn(t, shifter);
  const int j = static_cast<int>(__double_as_longlong(t) & 15);
  const double top = __shfl_sync(0xffffffffu, top_i, j);
  const double tail = __shfl_sync(0xffffffffu, tail_i, j);
  double r = __fma_rn(-n, ln2_hi, xs);
  r = __fma_rn(-ln2_lo, n, r);
  r = __longlong_as_double(__double_as_longlong(r) & 0xbfffffffffffffffLL);
  const double r2 = __dmul_rn(r, r);
  double a = __fma_rn(c6, r, c5);
  const double b = __fma_rn(c4, r, c3);
  const double c = __fma_rn(c2, r, c1);
  a = __fma_rn(r2, a, b);
  a = __fma_rn(r2, a, c);
  const double pp = __fma_rn(a, r, tail);
  const double res = __fma_rn(top, pp, top);
  const int m = static_cast<int>(floor(n));
  if (big) return x < 0.0 ? 0.0 : exp(x);
  return __dmul_rn(res, __longlong_as_double(static_cast<long long>(m + 1023) << 52));
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
// W (d, E) fp32 -> fp64, same layout: the segment router's operand, so its
// hot loop converts only the token values (F2F.F64.F32 runs at a quarter of
// the DFMA rate).
__global__ void __launch_bounds__(256) widen_f64_kernel(const float* __restrict__ w, double* __restrict__ o, long n) {
  for (long i = (long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long)gridDim.x * 256)
    o[i] = static_cast<double>(w[i]);
}

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
  // fp64 x chunk: token-major rows of kc + 1 (padded), or k-major rows of
  // tokc + 2 (the 4 x 2 quarter-warp tile layout); sized for either
  static __host__ __device__ size_t x_bytes(int tokc, int kc) {
    const size_t a = (size_t)tokc * (kc + 1), b = (size_t)kc * (tokc + 2);
    return ((a > b ? a : b) * 8 + 127) / 128 * 128;
  }
  static __host__ __device__ size_t raw_bytes(int tokc, int xb, int kc) { return ((size_t)tokc * kc * xb + 127) / 128 * 128; }
  static __host__ __device__ size_t stage_bytes(int tokc, int expc, int xb, int kc) {
    return w_bytes(expc, kc) + x_bytes(tokc, kc) + raw_bytes(tokc, xb, kc);
  }
  static __host__ __device__ size_t total_bytes(int tokc, int expc, int xb, int E, int nthreads, int stages, int kc) {
    size_t ph1 = stages * stage_bytes(tokc, expc, xb, kc) + 3 * stages * 8;
    size_t ph2 = (size_t)(nthreads / 32) * (E * 16 + kChainWin * 8);  // scores row (fp64) + logit interval + window
    return ph1 > ph2 ? ph1 : ph2;
  }
};

// ---------------------------------------------------------------------------
// Operand helpers: 8 consecutive x values of one token row as fp32.
// ---------------------------------------------------------------------------
MOE_DEVICE void unpack_bf16x8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <bool kXBf16>
MOE_DEVICE void load_x8(const void* x, size_t off, float (&f)[8]) {
  if constexpr (kXBf16) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + off));
    unpack_bf16x8(v, f);
  } else {
    const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(x) + off);
    const float4 a = __ldg(q), b = __ldg(q + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
}

// Last-arriver election across CTAs: every thread's prior global writes are
// ordered before thread 0's release (bar.sync + fence.acq_rel.gpu, as in a
// cooperative grid sync); the last CTA's reads follow its acquire and go
// through L2 (__ldcg).  Returns true in the CTA that arrives n-th.
MOE_DEVICE bool cta_arrive_last(int32_t* counter, int n) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const int prev = atomicAdd(counter, 1);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_last = (prev == n - 1);
  }
  __syncthreads();
  return s_last != 0;
}

// Exact logit: ONE sequential fp64 FMA chain in ascending k, rounded once to
// fp32 (linalg.py:45-57 dot_accumulate; fp32 x fp32 products are exact in
// fp64, so fma == the reference's multiply-then-add).  Used by the certified
// segment path only for the rare logits whose certificate is inconclusive.
// Warp-cooperative: lanes stream 32-step windows of x[t, :] and
// W_r[:, e] (4 windows in flight, hiding L2 latency), every lane runs the same
// dependent fold on shuffled operands (identical result in all lanes).
template <bool kXBf16>
__device__ __noinline__ float exact_chain_logit_warp(const RouterParams& p, int t, int e, int lane, double* win) {
  // fma(x, w, a) == fl(x*w + a) because x*w is exact in fp64: the lanes form
  // the products of a 128-step window (4 each, operands loaded one window
  // ahead), the window goes through shared memory, and every lane folds it
  // with broadcast loads — one dependent DADD per step.
  const size_t xrow = (size_t)t * p.d;
  const int nwin = (p.d + kChainWin - 1) / kChainWin;
  // volatile loads with a memory clobber: issued where written (one window
  // ahead), never sunk below the shared-memory fold of the current window
  auto ld = [&](int w, float (&xv)[4], float (&wv)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = min(w * kChainWin + i * 32 + lane, p.d - 1);
      if constexpr (kXBf16) {
        unsigned short b;
        asm volatile("ld.global.nc.u16 %0, [%1];"
                     : "=h"(b) : "l"(static_cast<const __nv_bfloat16*>(p.x) + xrow + k) : "memory");
        xv[i] = __uint_as_float(static_cast<uint32_t>(b) << 16);
      } else {
        asm volatile("ld.global.nc.f32 %0, [%1];"
                     : "=f"(xv[i]) : "l"(static_cast<const float*>(p.x) + xrow + k) : "memory");
      }
      asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(wv[i]) : "l"(p.wr + (size_t)k * p.E + e) : "memory");
    }
  };
  float xa[4], wa[4], xb[4], wb[4];
  ld(0, xa, wa);
  double acc = -0.0;  // fl(p + -0) == p, sign included, like fma(x, w, -0)
  for (int w = 0; w < nwin; ++w) {
    if (w + 1 < nwin) ld(w + 1, xb, wb);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // steps past d (clamped loads) are never folded: n below stops at d
      win[i * 32 + lane] = static_cast<double>(xa[i]) * static_cast<double>(wa[i]);
    }
    __syncwarp();
    const int n = min(kChainWin, p.d - w * kChainWin);
    if (n == kChainWin) {
#pragma unroll
      for (int j = 0; j < kChainWin; ++j) acc = __dadd_rn(acc, win[j]);
    } else {
      for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, win[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) { xa[i] = xb[i]; wa[i] = wb[i]; }
  }
  __syncwarp();
  return __double2float_rn(acc);
}

MOE_DEVICE bool same_bits(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }

// warp max of floats (no NaN among the inputs: the logits are finite here)
MOE_DEVICE float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Screen mode (router_screen.cuh, sigmoid gating): score bounds of a logit
// interval.  np_sigmoid is accurate to a few ulps but not monotone at the
// ulp level: the bounds carry a 2^-20 relative (and 2^-126 absolute) margin.
// logit >= l, upper bound for a logit <= l
MOE_DEVICE float scr_score_lo(float l) {
  if (isnan(l)) return 0.0f;
  return __fmul_rd(np_sigmoid(l), 1.0f - 0x1p-20f);
}
MOE_DEVICE float scr_score_hi(float l) {
  if (isnan(l)) return 2.0f;
  return __fmaf_ru(np_sigmoid(l), 1.0f + 0x1p-20f, 0x1p-126f);
}

// k-th largest of v[0..n) (a warp; destroys v): k rounds of warp max, each
// removing one instance
MOE_DEVICE float scr_kth_largest(float* v, int n, int k, int lane) {
  float m = 0.0f;
  for (int j = 0; j < k; ++j) {
    float bm = -1.0f;
    int bi = 0x7fffffff;
    for (int e = lane; e < n; e += 32)
      if (v[e] > bm) { bm = v[e]; bi = e; }
    m = bm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int owner = __reduce_min_sync(0xffffffffu, bm == m ? bi : 0x7fffffff);
    __syncwarp();
    if (lane == (owner & 31) && owner < n) v[owner] = -1.0f;
    __syncwarp();
  }
  return m;
}

constexpr int kTopkRegs = 8;  // phase-2 top-k keeps E <= 256 scores in registers

// Scores (softmax: numpy float64 exp of the fp32-shifted logits, pairwise
// sum, divide; sigmoid: numpy float32 logistic) and top-k of one token from
// the logits lo[] (shared memory, one warp): lane j < min(k, 32) returns
// selection j in (isel, wsel); for k > 32 the selections past 31 are written
// to the outputs of token t directly (t < 0: not supported, callers check).
// Used by phase 2 and by the certification's candidate enumeration.
MOE_DEVICE void eval_route_outputs(const RouterParams& p, int t, const float* lo, float m, double* row, int lane,
                                   int& isel_out, float& wsel_out) {
  // ---- scores (lo is a representative: every candidate gives the same bits)
  if (p.gating == 0) {
    const double top_i = __longlong_as_double(static_cast<long long>(kNpExpTop[lane & 15]));
    const double tail_i = __longlong_as_double(static_cast<long long>(kNpExpTail[lane & 15]));
    for (int e0 = 0; e0 < p.E; e0 += 32) {
      const int e = e0 + lane;
      const double v = np_exp64_warp(e < p.E ? static_cast<double>(__fsub_rn(lo[e], m)) : 0.0, top_i, tail_i);
      if (e < p.E) row[e] = v;
    }
    __syncwarp();
    const double S = pairwise_sum_warp<double>(row, p.E, lane);
    __syncwarp();
    for (int e = lane; e < p.E; e += 32) {
      float sc = __double2float_rn(__ddiv_rn(row[e], S));
      row[e] = static_cast<double>(sc);
    }
  } else {
    for (int e = lane; e < p.E; e += 32) row[e] = static_cast<double>(np_sigmoid(lo[e]));
  }
  __syncwarp();
    // top-k over keys (score bits desc, index asc); scores are >= +0.
    float wsel = 0.0f;
    int isel = 0;
    if (p.E <= 32 * kTopkRegs) {
      // the lane's scores e = lane + 32 i in registers (ascending i: the
      // first max within the lane is its lowest index); k rounds of two
      // warp reductions, the winner's owner marks it selected
      float sc[kTopkRegs];
#pragma unroll
      for (int i = 0; i < kTopkRegs; ++i) {
        const int e = lane + 32 * i;
        sc[i] = e < p.E ? static_cast<float>(row[e]) : -1.0f;
      }
      for (int j = 0; j < p.k; ++j) {
        uint32_t kb = 0, kidx = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < kTopkRegs; ++i) {
          const float v = sc[i];
          if (!(v < 0.0f)) {
            const uint32_t key = ((v == 0.0f) ? 0u : __float_as_uint(v)) + 1u;
            if (key > kb) { kb = key; kidx = static_cast<uint32_t>(lane + 32 * i); }
          }
        }
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, kb);
        const int e_best = static_cast<int>(__reduce_min_sync(0xffffffffu, kb == kmax ? kidx : 0xFFFFFFFFu));
        const float s_best = __uint_as_float(kmax - 1u);
        if (lane == (e_best & 31)) {
#pragma unroll
          for (int i = 0; i < kTopkRegs; ++i)
            if (i == (e_best >> 5)) sc[i] = -1.0f;
        }
        if (lane == j) { wsel = s_best; isel = e_best; }
        if (j >= 32 && lane == 0) {  // k > 32: write directly (rare)
          p.topk_idx[(size_t)t * p.k + j] = e_best;
          p.topk_w[(size_t)t * p.k + j] = s_best;
        }
      }
    }
    for (int j = 0; j < (p.E <= 32 * kTopkRegs ? 0 : p.k); ++j) {
      // largest key (score bits desc, index asc) in two warp reductions: the
      // max of score bits + 1 (0: no candidate), then the lowest index holding it
      uint32_t kb = 0, kidx = 0xFFFFFFFFu;
      for (int e = lane; e < p.E; e += 32) {  // ascending e: the first max is the lowest index
        float sc = static_cast<float>(row[e]);
        if (sc < 0.0f) continue;  // already selected (marked -1)
        const uint32_t key = ((sc == 0.0f) ? 0u : __float_as_uint(sc)) + 1u;
        if (key > kb) { kb = key; kidx = static_cast<uint32_t>(e); }
      }
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, kb);
      const int e_best = static_cast<int>(__reduce_min_sync(0xffffffffu, kb == kmax ? kidx : 0xFFFFFFFFu));
      const float s_best = __uint_as_float(kmax - 1u);
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
  isel_out = isel;
  wsel_out = wsel;
}

// Certification of one token's logit intervals (phase 2's slow path, taken
// only when some interval is unknown or has nonzero width): resolves, with
// the exact sequential chain, every logit the outputs depend on and returns
// the (certain) row max for the softmax.  Out of line: the common path stays
// a short straight run of code (the router executes it once per CTA, from a
// cold instruction cache).
template <bool kXBf16>
__device__ __noinline__ float certify_token(const RouterParams& p, int t, float* lo, float* hi, double* win,
                                            double* row, int lane) {
  float m = 0.0f;
  for (int round = 0; round < 2; ++round) {
    bool any = false;
    if (round == 1 && p.gating == 0 && !p.want_logits && p.k <= 32) {
      // Enumeration certificate (softmax): when at most two logits still have
      // an uncertain shifted value fp32(l - m), each with exactly two fp32
      // candidates {lo, hi = nextafter(lo)}, evaluate the token's outputs
      // (top-k indices and weight bits) for every combination of candidates.
      // If they all agree, the outputs do not depend on which value the
      // reference fold rounds to: no exact recompute is needed (the exact
      // chain costs d x 8 cycles of latency).
      int nf = 0, fe[2] = {0, 0};
      bool ok = true;
      for (int e0 = 0; e0 < p.E && ok; e0 += 32) {
        const int e = e0 + lane;
        bool f = false, two = true;
        if (e < p.E) {
          const float a = lo[e], b = hi[e];
          f = !same_bits(a, b) && !same_bits(__fsub_rn(a, m), __fsub_rn(b, m));
          two = !f || same_bits(nextafterf(a, __int_as_float(0x7f800000)), b);
        }
        uint32_t bal = __ballot_sync(0xffffffffu, f);
        ok = __all_sync(0xffffffffu, two) && ok;
        while (bal && ok) {
          if (nf == 2) { ok = false; break; }
          fe[nf++] = e0 + __ffs(bal) - 1;
          bal &= bal - 1;
        }
      }
      if (ok && nf > 0) {
        float orig[2] = {lo[fe[0]], lo[fe[1]]};
        int i0 = 0, i1 = 0;
        float w0 = 0.0f, w1 = 0.0f;
        eval_route_outputs(p, t, lo, m, row, lane, i0, w0);
        bool same = true;
        for (int c = 1; c < (1 << nf) && same; ++c) {
          __syncwarp();
          if (lane == 0)
            for (int q = 0; q < nf; ++q) lo[fe[q]] = ((c >> q) & 1) ? hi[fe[q]] : orig[q];
          __syncwarp();
          eval_route_outputs(p, t, lo, m, row, lane, i1, w1);
          same = __all_sync(0xffffffffu, lane >= p.k || (i1 == i0 && same_bits(w1, w0)));
        }
        __syncwarp();
        if (lane == 0)
          for (int q = 0; q < nf; ++q) {
            lo[fe[q]] = orig[q];
            if (same) hi[fe[q]] = orig[q];  // certified: lo is a valid representative
          }
        __syncwarp();
        if (same && p.trace && p.seg_len && lane == 0) atomicAdd(p.trace + (size_t)blockIdx.x * 16 + 12, 1ull << 32);
      }
    }
    for (int e0 = 0; e0 < p.E; e0 += 32) {
      const int e = e0 + lane;
      bool nd = false;
      if (e < p.E) {
        const float a = lo[e], b = hi[e];
        const bool unsure = !same_bits(a, b);
        if (round == 0) {
          nd = isnan(a) || (p.want_logits && unsure);
        } else if (unsure) {
          if (p.gating == 0) {
            nd = !same_bits(__fsub_rn(a, m), __fsub_rn(b, m));
          } else {
            const float sa = np_sigmoid(a);
            float c = a;
            int steps = 0;
            // every logit >= 18 scores exactly 1.0f (expf(-18) < 2^-25: 1 + t rounds to 1)
            if (a >= 18.0f) c = b;
            while (!nd && !same_bits(c, b)) {
              c = nextafterf(c, b);
              nd = (++steps > 8) || !same_bits(np_sigmoid(c), sa);
            }
          }
        }
      }
      // resolve the flagged logits of this 32-wide slice one at a time, warp-wide
      uint32_t todo = __ballot_sync(0xffffffffu, nd);
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const float v = exact_chain_logit_warp<kXBf16>(p, t, e0 + j, lane, win);
        if (lane == j) {
          lo[e] = v;
          hi[e] = v;
        }
        if (p.trace && p.seg_len && lane == 0) atomicAdd(p.trace + (size_t)blockIdx.x * 16 + 11, 1ull);
      }
      any |= nd;
    }
    __syncwarp();
    if (round == 0 && p.gating == 0) {
      // the row max must be certain; otherwise resolve every unsure logit
      float mlo = -__int_as_float(0x7f800000), mhi = mlo;
      for (int e = lane; e < p.E; e += 32) {
        mlo = fmaxf(mlo, lo[e]);
        mhi = fmaxf(mhi, hi[e]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mlo = fmaxf(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
        mhi = fmaxf(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
      }
      if (mlo != mhi) {
        for (int e0 = 0; e0 < p.E; e0 += 32) {
          const int e = e0 + lane;
          uint32_t todo = __ballot_sync(0xffffffffu, e < p.E && !same_bits(lo[e], hi[e]));
          while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const float v = exact_chain_logit_warp<kXBf16>(p, t, e0 + j, lane, win);
            if (lane == j) {
              lo[e] = v;
              hi[e] = v;
            }
            if (p.trace && p.seg_len && lane == 0) atomicAdd(p.trace + (size_t)blockIdx.x * 16 + 12, 1ull);
          }
        }
        __syncwarp();
        mlo = -__int_as_float(0x7f800000);
        for (int e = lane; e < p.E; e += 32) mlo = fmaxf(mlo, lo[e]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mlo = fmaxf(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
      }
      m = mlo;
    }
    (void)any;
  }
  return m;
}

// ---------------------------------------------------------------------------
// Phase 2 (one warp per token): scores + top-k + sigmoid renormalisation from
// the certified logit intervals.  A logit interval [lo, hi] holds every fp32
// value the reference's sequential fold can round to.  Only the quantities
// the outputs depend on must be certain:
//   softmax: m = max logit, and s_e = fp32(l_e - m) for every e
//            (router.py:78-83; exp64 and the division are then fixed);
//   sigmoid: score_e = sigmoid32(l_e)                (linalg.py:71-80).
// Both are checked over the interval (subtraction is monotone; the sigmoid is
// evaluated at every candidate, at most 8), and any logit that still matters
// is recomputed with the exact sequential chain.  want_logits resolves all.
// ---------------------------------------------------------------------------
template <bool kXBf16>
MOE_DEVICE void route_scores_tokens(const RouterParams& p, int t_begin, int t_end, uint8_t* smem,
                                    int warp_override = -1) {
  const int tid = threadIdx.x;
  // warp_override >= 0: only the calling warp, on token t_begin, with its
  // scratch at smem (the screening router's per-token fallback)
  const int nwarps = warp_override >= 0 ? 1 : blockDim.x / 32;
  const int warp = warp_override >= 0 ? 0 : tid / 32, lane = tid % 32;
  uint8_t* base = smem + (size_t)warp * (p.E * 16 + kChainWin * 8);
  double* row = reinterpret_cast<double*>(base);
  float* lo = reinterpret_cast<float*>(base + (size_t)p.E * 8);
  float* hi = lo + p.E;
  double* win = reinterpret_cast<double*>(base + (size_t)p.E * 16);  // exact-chain window
  // debug timeline (segment kernel): phase-2 sub-steps of the CTA's first token
  // as clock64 deltas from phase-2 entry in slots 8, 9, 13, 14
  unsigned long long* tr2 = (p.trace && p.seg_len && tid == 0) ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  const long long c2 = clock64();
  auto stamp2 = [&](int i) { if (tr2) tr2[i] = clock64() - c2; };
  for (int t = t_begin + warp; t < t_end; t += nwarps) {
    const float2* lb = p.lbuf + (size_t)t * p.E;
    for (int e = lane; e < p.E; e += 32) {
      const float2 v = __ldcg(lb + e);
      lo[e] = v.x;
      hi[e] = v.y;
    }
    __syncwarp();
    if (p.screen) {
      // exclusion: an expert whose upper score bound is below the k-th largest
      // lower bound has k experts strictly above it and is never selected;
      // its logit becomes a certain -FLT_MAX (score 0 < S_k)
      float* sl = reinterpret_cast<float*>(row);
      for (int e = lane; e < p.E; e += 32) sl[e] = scr_score_lo(lo[e]);
      __syncwarp();
      const float Sk = scr_kth_largest(sl, p.E, p.k, lane);
      if (Sk >= 0x1p-100f)
        for (int e = lane; e < p.E; e += 32)
          if (scr_score_hi(hi[e]) < Sk) { lo[e] = -FLT_MAX; hi[e] = -FLT_MAX; }
      __syncwarp();
    }
    stamp2(8);
    // ---- certification; `round` 0: unknown (+ everything if want_logits),
    //      1: whatever the outputs still depend on.  Fast path: every interval
    //      has zero width (the common case) -- nothing to resolve, m = max.
    bool unsure_any = false;
    for (int e = lane; e < p.E; e += 32) unsure_any |= isnan(lo[e]) || !same_bits(lo[e], hi[e]);
    unsure_any = __any_sync(0xffffffffu, unsure_any);
    float m = 0.0f;
    if (!unsure_any && p.gating == 0) {
      float mx = -__int_as_float(0x7f800000);
      for (int e = lane; e < p.E; e += 32) mx = fmaxf(mx, lo[e]);
      m = warp_max_f32(mx);
    }
    if (unsure_any) m = certify_token<kXBf16>(p, t, lo, hi, win, row, lane);
    stamp2(9);
    if (p.want_logits)
      for (int e = lane; e < p.E; e += 32) p.logits[(size_t)t * p.E + e] = lo[e];
    int isel = 0;
    float wsel = 0.0f;
    eval_route_outputs(p, t, lo, m, row, lane, isel, wsel);
    stamp2(14);
      if (lane < p.k) {
        p.topk_idx[(size_t)t * p.k + lane] = isel;
        p.topk_w[(size_t)t * p.k + lane] = wsel;
      }
      __syncwarp();
      tr2 = nullptr;  // (debug timeline: the first token only)
    }
}

// Launch shape: blockDim = n_compute + kRouterProducers.  Compute threads own a
// kTE x kTT register tile of independent sequential fp64 chains; the producer
// warps fill stage s: one elected thread bulk-copies the W64 chunk (tx-count on
// full[s]), all 128 convert the x chunk to fp64 (one arrival each).  Compute
// warps release stages through empty[s] (one arrival per warp).
template <bool kXBf16, int kTE, int kTT, int kKC>
__global__ void __launch_bounds__(384)
router_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ RouterParams p) {
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
  // 4 x 2 quarter-warp tiles (32 x 32 CTA block, 4 compute warps; host-checked)
  constexpr bool kQ = (kTE == 4 && kTT == 2);
  constexpr int kQTok = 32, kQExp = 32;
  if (p.trace && threadIdx.x == 0) p.trace[4096 * 4 + 2048 * 4 + blockIdx.x] = globaltimer_ns();
  pdl_launch_dependents();
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
        if constexpr (kQ) dx[kk * (kQTok + 2) + row] = static_cast<double>(v);  // k-major (see compute)
        else dx[row * (kKC + 1) + kk] = static_cast<double>(v);
      }
      mbar_arrive(full + s);
      // refill: chunk c+S-1 goes into the stage of chunk c-1 once compute released it
      if (ptid == 0 && c + p.stages - 1 < nch) issue(c + p.stages - 1);
    }
    if (nonfinite_x) atomicOr(p.flags, 1u);
  } else if constexpr (kQ) {
    // ===================== compute chains, quarter-warp tiles ================
    // 32 tokens x 32 experts per CTA, 4 warps of 16 x 16 chains; lane = 8
    // token pairs (lane % 8) x 4 expert quads (lane / 8), 4 x 2 chains each.
    // Shared-memory operand cost per step (LDS.128, measured on B200,
    // scripts/probes/lds_probe.cu): x pair distinct within each quarter-warp
    // 4 cycles, W quads uniform within each quarter-warp 2 + 2 cycles -- 8
    // cycles per 8 DFMA per warp (the 2 x 2 / 2 x 4 strided tiles: 9-10
    // cycles per 4-8 DFMA).  x is k-major fp64 in the stage (kQTok + 2 row
    // stride: 16-byte aligned pairs, 2-way store conflicts for the producers).
    const int cw = tid / 32, lane = tid & 31;
    const int tok0 = 16 * (cw >> 1) + 2 * (lane & 7);
    const int ex0 = 16 * (cw & 1) + 4 * (lane >> 3);
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) { acc[i][0] = -0.0; acc[i][1] = -0.0; }
    for (int c = 0; c < nch; ++c) {
      const int s = c % p.stages;
      const uint32_t ph = (c / p.stages) & 1;
      mbar_wait(full + s, ph);
      const uint8_t* st = smem + s * sbytes;
      const double* dw = reinterpret_cast<const double*>(st) + ex0;
      const double* dx = reinterpret_cast<const double*>(st + wbytes) + tok0;
      const int kvalid = min(kKC, p.d - c * kKC);
      auto step = [&](int kk) {
        const double2 xv = *reinterpret_cast<const double2*>(dx + kk * (kQTok + 2));
        const double2 wa = *reinterpret_cast<const double2*>(dw + kk * kQExp);
        const double2 wb = *reinterpret_cast<const double2*>(dw + kk * kQExp + 2);
        acc[0][0] = __fma_rn(xv.x, wa.x, acc[0][0]); acc[0][1] = __fma_rn(xv.y, wa.x, acc[0][1]);
        acc[1][0] = __fma_rn(xv.x, wa.y, acc[1][0]); acc[1][1] = __fma_rn(xv.y, wa.y, acc[1][1]);
        acc[2][0] = __fma_rn(xv.x, wb.x, acc[2][0]); acc[2][1] = __fma_rn(xv.y, wb.x, acc[2][1]);
        acc[3][0] = __fma_rn(xv.x, wb.y, acc[3][0]); acc[3][1] = __fma_rn(xv.y, wb.y, acc[3][1]);
      };
      if (kvalid == kKC) {
#pragma unroll 16
        for (int kk = 0; kk < kKC; ++kk) step(kk);
      } else {
        for (int kk = 0; kk < kvalid; ++kk) step(kk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = e0 + ex0 + i;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int t = t0 + tok0 + j;
        if (t < p.B && e < p.E) {
          const float l = __double2float_rn(acc[i][j]);
          p.lbuf[(size_t)t * p.E + e] = make_float2(l, l);  // exact: a zero-width interval
        }
      }
    }
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
          if (t < p.B && e < p.E && eg + i * n_eg < p.expc) {
            const float l = __double2float_rn(acc[i][j]);
            p.lbuf[(size_t)t * p.E + e] = make_float2(l, l);  // exact: a zero-width interval
          }
        }
      }
    }
  }

  if (p.trace && tid == 0) p.trace[4096 * 4 + blockIdx.x * 4 + 0] = globaltimer_ns();
  // --------------------- phase 2: scores + top-k (last CTA of block) --------
  if (p.n_eblocks > 1) {
    if (!cta_arrive_last(p.tb_counter + tb, p.n_eblocks)) return;
    if (tid == 0) p.tb_counter[tb] = 0;  // every CTA of this block has arrived: reset for the next launch
  } else {
    __syncthreads();
  }
  route_scores_tokens<kXBf16>(p, t0, min(t0 + p.tokc, p.B), smem);
  if (p.trace && tid == 0) p.trace[4096 * 4 + blockIdx.x * 4 + 1] = globaltimer_ns();
}

}  // namespace moe
