// moe_b200.cu — C-ABI entry points (include/moe_b200.h): argument checks,
// workspace layout, TMA descriptor encoding and kernel launches.
#include "../../include/moe_b200.h"

#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "elementwise.cuh"
#include "ffn.cuh"
#include "router.cuh"
#include "router_seg.cuh"
#include "router_screen.cuh"
#include "dispatch.cuh"
#include "ep_p2p.cuh"
#include "stages.cuh"

using namespace moe;

namespace {

// NVTX ranges per stage (host-side launch regions; nsys / ncu correlate them
// with the kernels launched inside).  Header-only NVTX3: without an attached
// tool a push / pop is a null-pointer check.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

thread_local std::string g_last_error;

int cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  g_last_error = buf;
  cudaGetLastError();  // reported here: do not leave a (non-sticky) error for the next launch check
  return MOE_B200_ERR_CUDA;
}

// Event record that also works inside stream capture: there it becomes an
// external event-record node, so streams outside the graph can wait on it.
cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  return cudaEventRecord(ev, s);
}

#define MOE_CUDA(call)                                \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

#define MOE_LAUNCH_CHECK(what)                          \
  do {                                                  \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return cuda_fail(_e, what);  \
  } while (0)

constexpr size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Tuning / test hooks (MOE_B200_* environment variables).  Read once, off the
// forward path: at the first use, at every moe_b200_workspace_init and by
// moe_b200_tuning_reload (tests that flip a hook on an existing layer call it).
// -1 / 0 mean "not set" (the built-in rule applies).
struct Tuning {
  int chunk_rows = 0;        // MOE_B200_CHUNK_ROWS (128 | 256)
  int down_splits = 0;       // MOE_B200_DOWN_SPLITS
  int seg_wide = -1;         // MOE_B200_SEG_WIDE (0: never 64-wide expert blocks)
  long long seg_max_chains = 64LL * 1024;  // MOE_B200_SEG_MAX_CHAINS
  int seg_len = 0;           // MOE_B200_SEG_LEN
  int pdl = 0;               // MOE_B200_PDL
  int rx_te = 0, rx_tt = 0, rx_tokc = 0;  // MOE_B200_RX_TILE "te,tt,tokc"
  int ffn_pair = -1;         // MOE_B200_FFN_PAIR (0 | 1 | 2)
  int ffn_variant = 2;       // MOE_B200_FFN_VARIANT
  int force_exact = 0;       // MOE_B200_ROUTER_FORCE_EXACT
  int io_graphs = 1;         // MOE_B200_IO_GRAPHS
  int fused_combine = 1;     // MOE_B200_FUSED_COMBINE (0: separate combine launch)
  int carveout = -1;         // MOE_B200_CARVEOUT: shared-memory carveout (%) of the small kernels
  int tmem_db = 1;           // MOE_B200_TMEM_DB: double-buffered TMEM accumulators for <= 128-row chunks
  int seg_w64 = 0;           // MOE_B200_SEG_W64: segment router reads W pre-widened to fp64
  int rx_quarter = 1;        // MOE_B200_RX_QUARTER: 4 x 2 quarter-warp tiles in the exact router (0: 2 x 4)
  int fuse_dispatch = 1;     // MOE_B200_FUSE_DISPATCH: small batches dispatch inside the router (0: separate launch)
  int screen = -1;           // MOE_B200_SCREEN: sigmoid router via the INT8 screen (-1 auto, 0 off, 1 always)
  int w3d = 2;               // MOE_B200_W3D: 3-D TMA weight loads, 1 = one per 16 KB slot, 2 = + a down tile's two slots in one (single-CTA tiles); 0: 2-D
  int seg_tt1 = 1;           // MOE_B200_SEG_TT1: 1- and 2-token batches use 1- / 2-token segment tiles (0: 4-token tiles)
};
Tuning g_tune;
std::mutex g_tune_mu;
std::atomic<bool> g_tune_loaded{false};

void load_tuning_locked() {
  Tuning t;
  auto geti = [](const char* name, int def) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : def;
  };
  t.chunk_rows = geti("MOE_B200_CHUNK_ROWS", 0);
  t.down_splits = geti("MOE_B200_DOWN_SPLITS", 0);
  t.seg_wide = geti("MOE_B200_SEG_WIDE", -1);
  if (const char* v = getenv("MOE_B200_SEG_MAX_CHAINS")) t.seg_max_chains = atoll(v);
  t.seg_len = geti("MOE_B200_SEG_LEN", 0);
  t.pdl = geti("MOE_B200_PDL", 0);
  if (const char* v = getenv("MOE_B200_RX_TILE")) {
    if (sscanf(v, "%d,%d,%d", &t.rx_te, &t.rx_tt, &t.rx_tokc) != 3) t.rx_te = t.rx_tt = t.rx_tokc = 0;
  }
  t.ffn_pair = geti("MOE_B200_FFN_PAIR", -1);
  t.ffn_variant = geti("MOE_B200_FFN_VARIANT", 2);
  t.force_exact = geti("MOE_B200_ROUTER_FORCE_EXACT", 0);
  t.io_graphs = geti("MOE_B200_IO_GRAPHS", 1);
  t.fused_combine = geti("MOE_B200_FUSED_COMBINE", 1);
  t.carveout = geti("MOE_B200_CARVEOUT", -1);
  t.tmem_db = geti("MOE_B200_TMEM_DB", 1);
  t.seg_w64 = geti("MOE_B200_SEG_W64", 0);
  t.rx_quarter = geti("MOE_B200_RX_QUARTER", 1);
  t.fuse_dispatch = geti("MOE_B200_FUSE_DISPATCH", 1);
  t.screen = geti("MOE_B200_SCREEN", -1);
  t.w3d = geti("MOE_B200_W3D", 2);
  t.seg_tt1 = geti("MOE_B200_SEG_TT1", 1);
  g_tune = t;
  g_tune_loaded = true;
}

const Tuning& tuning() {
  if (!g_tune_loaded) {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    if (!g_tune_loaded) load_tuning_locked();
  }
  return g_tune;
}

void reload_tuning() {
  std::lock_guard<std::mutex> lock(g_tune_mu);
  load_tuning_locked();
}

constexpr int kTbCap = 4096;      // max router token blocks per launch
constexpr int kChunkCap = 8192;   // max expert row-chunks per launch
constexpr int kBlkCap = 16384;    // max (token block x expert block) counters (segment router)

// Fixed header at the start of the workspace (zeroed by workspace_init; every
// kernel leaves its counters zeroed again):
//   [0] flags  [1] router done counter  [2] n_chunks  [3] ffn work counter
//   [4] ffn exit counter  [5] fused small-batch dispatch counter
//   [16, 16+kTbCap) router token-block counters
//   [16+kTbCap, 16+kTbCap+kChunkCap) per-chunk gate+up completion counters
//   [.., +kBlkCap) segment-router (token block, expert block) counters
constexpr int kHdrDisp = 5;  // [5] fused small-batch dispatch: token blocks past phase 2
constexpr int kHdrTb = 16;
constexpr int kHdrGuDone = 16 + kTbCap;
constexpr int kHdrBlk = 16 + kTbCap + kChunkCap;
// arrival counters of the combine overlapped with the FFN tail, (token,
// 256-column block); overlapped while B * ceil(d / 256) <= kTokCntCap (every
// BASELINE config), else the combine simply runs after the FFN
constexpr int kTokCntCap = 64 * 1024;
constexpr int kHdrTok = 16 + kTbCap + kChunkCap + kBlkCap;
// per-expert statistics of the screening router (router_screen.cuh; max |w|,
// max quantisation error, sum |G2| as u32, sum |Q| as u64), self-resetting
constexpr int kHdrScr = 16 + kTbCap + kChunkCap + kBlkCap + kTokCntCap;
static_assert(kHdrScr % 2 == 0, "u64 alignment of the screen statistics");
constexpr size_t kHeaderBytes = align256((kHdrScr + 5 * kMaxExperts) * sizeof(int32_t));

struct Layout {
  size_t logits, lbuf, gpart, w64, chunk_tab, prow, xp, h, ys, rt_idx, rt_w, rt_misc, gu32, total;
  size_t s_xq, s_wq, s_xst, s_xqs, s_part, s_cand, s_ncand, s_elist, s_rpart;  // screening router (0: unused)
  int max_chunks, splits, kb_per_split, T_pad, n_ft, n_dp;
};

int chunk_rows_for(const moe_b200_config& c, int64_t B) {
  // Tokens per expert on average; big chunks keep one weight pass per expert
  // (Mixtral), small chunks for many-expert layers (DeepSeek / Qwen).
  const int64_t T = B * c.top_k;
  const int v = tuning().chunk_rows;
  if (v == 128 || v == 256) return v;  // tuning hook (the FFN templates are BN 128 / 256)
  return (T > 96LL * c.num_experts) ? 256 : 128;
}

// Expected number of experts with at least one routed row under uniform top-k
// routing: E (1 - (1 - k/E)^B).
double expected_active_experts(const moe_b200_config& c, int64_t B) {
  const double E = c.num_experts;
  return std::max(1.0, E * (1.0 - std::pow(1.0 - c.top_k / E, static_cast<double>(B))));
}

// K splits of a down tile (a pair of 128-row hidden tiles).  Large batches:
// S = round(f/2d), i.e. down tiles stream about twice the weight bytes of a
// gate+up tile (measured best on Mixtral-512: S=2 beats 3 and 4 once the
// partial-sum traffic of the combine is counted).  Small batches have few
// active experts, so few down tiles: split until about 256 down tiles (~1.7
// waves) exist, keeping >= 6 k-blocks per split (measured Mixtral B=1/2/4:
// S=8/6/4 -> 161->131, 203->182, 248->229 us; B=16 keeps S=2; Qwen B=1/4:
// S=4 -> 59->53, 82->76 us).  Partials are reduced deterministically in
// combine.  MOE_B200_DOWN_SPLITS overrides (tuning).
int down_split_count(const moe_b200_config& c, int64_t B, int force) {
  const int nkb = (c.ffn_dim + kBK - 1) / kBK;
  const int n_dp = (c.hidden_dim + 2 * kBM - 1) / (2 * kBM);
  int s = static_cast<int>((c.ffn_dim + c.hidden_dim) / (2 * c.hidden_dim));  // round(f / 2d)
  const int fill = static_cast<int>(std::lround(256.0 / (n_dp * expected_active_experts(c, B))));
  s = std::max(s, std::min(fill, nkb / 6));
  if (force > 0) s = force;  // 0: the rule above
  s = std::max(1, std::min(s, 16));
  return std::min(s, nkb);
}

// s_force > 0: a caller-chosen count (the expert-parallel ranks use the global
// layer's count so their rows match the single-GPU forward bit for bit)
void down_splits(const moe_b200_config& c, int64_t B, int* splits, int* kb_per_split, int s_force = 0) {
  const int nkb = (c.ffn_dim + kBK - 1) / kBK;
  const int s = s_force > 0 ? std::min(std::min(s_force, 16), nkb) : down_split_count(c, B, tuning().down_splits);
  int kps = (nkb + s - 1) / s;
  *kb_per_split = kps;
  *splits = (nkb + kps - 1) / kps;
}

// The combine runs overlapped with the FFN's tail (combine_flag_kernel behind
// the FFN with programmatic dependent launch, driven by per-(token, block)
// arrival counters) unless MOE_B200_FUSED_COMBINE=0, the batch exceeds the
// counter capacity, or the K split is outside the combine kernels' register
// budget (then the combine launches after the FFN as before; same bits).
bool combine_overlapped(const moe_b200_config& c, int64_t B) {
  const int64_t n_dp = (c.hidden_dim + 2 * kBM - 1) / (2 * kBM);
  if (tuning().fused_combine == 0 || B < 1 || B * n_dp > kTokCntCap) return false;
  int S = 0, kps = 0;
  down_splits(c, B, &S, &kps);
  return S <= 8 && c.top_k * S <= kCombineMaxKS;
}

// ---- segment (certified split-K) router plan --------------------------------
// Experts per CTA block (a multiple of the 4-expert thread tile).  Up to 64
// experts go in one 64-wide block (16 lanes per segment) when 32-wide blocks
// would need more than one wave of CTAs (a 202-register CTA runs alone on an
// SM): Qwen-60 at 512 tokens, 256 CTAs in two waves -> 128 CTAs in one.
int seg_expc(int E, int64_t B) {
  if (E <= 4) return 4;
  if (E <= 8) return 8;
  if (E <= 16) return 16;
  if (E <= 32) return 32;
  const int64_t n_tb = (B + kSegTT - 1) / kSegTT;
  // MOE_B200_SEG_WIDE=0: never 64-wide (A/B)
  if (E <= 64 && n_tb * ((E + 31) / 32) > kNumSMs && tuning().seg_wide != 0) return 64;
  return 32;
}

// The segment router runs up to this many tokens (B*E chains <= 64K, tunable
// via MOE_B200_SEG_MAX_CHAINS); larger problems are fp64-throughput bound and
// use the exact kernel (no magnitude DADD: half the fp64 work; measured
// DeepSeek-V3 B=512: 257 us exact vs 430 us segment).
int64_t seg_max_tokens(const moe_b200_config& c) {
  const int64_t chains = tuning().seg_max_chains;
  return chains / std::max(1, c.num_experts);
}

struct SegPlan {
  int tt, expc, n_eb, n_tb, n_kb, seg_len, kr, grid;
  size_t smem;
};

SegPlan plan_seg(const moe_b200_config& c, int64_t B) {
  SegPlan q{};
  q.expc = seg_expc(c.num_experts, B);
  q.n_eb = (c.num_experts + q.expc - 1) / q.expc;
  q.tt = (B <= 2 && tuning().seg_tt1 != 0 && !tuning().seg_w64) ? static_cast<int>(B) : kSegTT;  // tokens per CTA
  q.n_tb = static_cast<int>((B + q.tt - 1) / q.tt);
  const int G = q.expc / kSegTE;
  const int S = kSegThreads / G;
  // k-blocks: one when the (token, expert) blocks alone fill >= 3/4 of the
  // SMs (long segments amortise the per-CTA reduction / arrival overhead;
  // a segment of L steps costs ~8L cycles of latency), otherwise enough
  // k-blocks for ~1.5 waves, with segments of at least 8 steps
  const long base = (long)q.n_tb * q.n_eb;
  const int max_kb = std::max(1, (c.hidden_dim + S * 8 - 1) / (S * 8));
  int n_kb = base * 4 >= kNumSMs * 3 ? 1 : static_cast<int>(std::min<long>(max_kb, (kNumSMs * 3 / 2 + base - 1) / base));
  if (q.expc > 32) n_kb = 1;  // (64-wide blocks only when they fill the SMs; keeps n_kb <= d/256)
  q.seg_len = ((c.hidden_dim + (long)n_kb * S - 1) / ((long)n_kb * S) + 7) / 8 * 8;
  if (tuning().seg_len > 0 && q.expc <= 32) q.seg_len = std::max(8, tuning().seg_len / 8 * 8);
  q.kr = S * q.seg_len;
  q.n_kb = (c.hidden_dim + q.kr - 1) / q.kr;
  q.grid = q.n_tb * q.n_eb * q.n_kb;
  const size_t part = (size_t)(kSegThreads / 32) * q.tt * q.expc * 16 + 64;  // warp partials
  const size_t ph2 = (size_t)(kSegThreads / 32) * (c.num_experts * 16 + kChainWin * 8);
  q.smem = std::max(part, ph2);
  return q;
}

// ---- screening router plan (router_screen.cuh) --------------------------------
// Sigmoid gating in the exact router's regime (B x E above the segment
// router's chain budget): INT8 screen + candidate refinement.
// MOE_B200_SCREEN=0 keeps the exact router, =1 uses the screen for every
// sigmoid batch (tests / A/B).
bool screen_applies(const moe_b200_config& c, int64_t B) {
  const int v = tuning().screen;
  if (v == 0 || c.gating != MOE_B200_GATING_SIGMOID_NORMALIZED || c.top_k > kScrMaxCand || B < 1) return false;
  // the refinement keeps the segment's W rows and every token row in shared memory
  if ((size_t)2 * c.num_experts * 12 + (size_t)B * 12 > (size_t)220 * 1024) return false;
  if (v == 1) return true;
  return B > seg_max_tokens(c);
}

struct ScreenPlan {
  int B_pad, E_pad, d_pad, n_tt, n_eb, nkb, n_ks, kbps, n_rs, rs_len, rs_first;
  size_t ref_smem, sel_smem, ph2_smem;
};

int screen_splits(int nkb, long tiles, int* kbps) {
  const int want = static_cast<int>(std::max(1L, std::min<long>(nkb, kNumSMs / std::max(1L, tiles))));
  *kbps = (nkb + want - 1) / want;
  return (nkb + *kbps - 1) / *kbps;
}

ScreenPlan plan_screen(const moe_b200_config& c, int64_t B) {
  ScreenPlan q{};
  const int E = c.num_experts, d = c.hidden_dim;
  q.B_pad = static_cast<int>((B + kScrM - 1) / kScrM * kScrM);
  q.E_pad = (E + kScrN - 1) / kScrN * kScrN;
  q.d_pad = (d + kScrKB - 1) / kScrKB * kScrKB;
  q.n_tt = q.B_pad / kScrM;
  q.n_eb = q.E_pad / kScrN;
  q.nkb = q.d_pad / kScrKB;
  q.n_ks = screen_splits(q.nkb, (long)q.n_tt * q.n_eb, &q.kbps);
  // refine: ~128 segments of the d axis (one per CTA), the W rows of a
  // segment in shared memory (<= 200 KB); segment 0 takes the remainder
  // x rows of the segment staged per token group (odd row stride)
  // (even lengths: the token rows are staged as 4-byte words, bf16 pairs;
  // the W rows are widened to fp64; W rows + all B token rows of the segment
  // + the unit offsets fit in shared memory)
  auto smem_for = [&](int l) {
    const size_t x = std::max((size_t)B * (size_t)(l | 1) * 4, (size_t)l * E * 4);  // (W staging reuses the x area)
    return (size_t)l * E * 8 + x + (size_t)(E + 1) * 4;
  };
  int len = std::max(8, (d + kNumSMs - 5) / (kNumSMs - 4));  // one wave of segments
  len = (len + 1) & ~1;
  while (len > 2 && smem_for(len) > (size_t)220 * 1024) len -= 2;
  q.rs_len = len;
  q.n_rs = (d + len - 1) / len;
  q.rs_first = d - (q.n_rs - 1) * len;
  q.ref_smem = smem_for(len);
  q.sel_smem = (size_t)2 * E * sizeof(float);
  q.ph2_smem = (size_t)kScrPh2Tok * (E * 16 + kChainWin * 8) + kScrPh2Tok * 32 * sizeof(float);
  return q;
}

// rows of the screen's split-K partial slab for any batch <= B (the split
// count falls as the token tiles grow, not monotonically in B)
size_t screen_part_rows(const moe_b200_config& c, int64_t B) {
  const ScreenPlan q = plan_screen(c, B);
  size_t rows = 0;
  for (int tt = 1; tt <= q.n_tt; ++tt) {
    int kbps = 0;
    const int ks = screen_splits(q.nkb, (long)tt * q.n_eb, &kbps);
    rows = std::max(rows, (size_t)ks * tt * kScrM);
  }
  return rows;
}

Layout layout_for(const moe_b200_config& c, int64_t B, int s_force = 0) {
  Layout L{};
  const int64_t T = B * c.top_k;
  const int bn = chunk_rows_for(c, B);
  L.max_chunks = static_cast<int>(std::min<int64_t>(c.num_experts, T) + T / bn + 1);
  down_splits(c, B, &L.splits, &L.kb_per_split, s_force);
  // tiled layouts: experts start 16-row aligned in a padded row space
  L.T_pad = static_cast<int>(((T + 15LL * std::min<int64_t>(c.num_experts, T)) + 15) / 16 * 16);
  L.n_ft = (c.ffn_dim + kBM - 1) / kBM;
  L.n_dp = (c.hidden_dim + 2 * kBM - 1) / (2 * kBM);
  const size_t h_rows = (size_t)T * c.ffn_dim * 2;
  const size_t h_tiled = (size_t)L.n_ft * L.T_pad * kBM * 2;
  const size_t ys_tiled = (size_t)L.splits * L.n_dp * 2 * L.T_pad * kBM * sizeof(float);
  size_t off = kHeaderBytes;
  L.logits = off;    off = align256(off + (size_t)B * c.num_experts * sizeof(float));
  L.lbuf = off;      off = align256(off + (size_t)B * c.num_experts * sizeof(float2));
  {
    // segment router partials: (B rounded to token blocks) x (E rounded to
    // expert blocks) chains x at most ceil(d / 256) k-blocks (S >= 32, L >= 8)
    const int64_t bseg = (std::min<int64_t>(B, seg_max_tokens(c)) + kSegTT - 1) / kSegTT * kSegTT;
    const int expc = seg_expc(c.num_experts, 1);  // 32-wide padding >= the 64-wide one (E <= 64)
    const int64_t epad = (c.num_experts + expc - 1) / expc * expc;
    const int64_t nkb = (c.hidden_dim + 255) / 256;
    L.gpart = off;   off = align256(off + (size_t)(bseg * epad * nkb) * 16);
  }
  {
    const int expc = std::min(c.num_experts, 32);
    const size_t neb = (c.num_experts + expc - 1) / expc;
    const size_t d_pad = (c.hidden_dim + kRouterKC - 1) / kRouterKC * kRouterKC;
    L.w64 = off;     off = align256(off + neb * d_pad * expc * sizeof(double));
  }
  // chunk table {expert, row0, nrows, padded row0} followed by the per-chunk
  // expert group {first chunk of the expert, chunks of the expert}
  L.chunk_tab = off; off = align256(off + (size_t)L.max_chunks * (sizeof(int4) + sizeof(int2)));
  L.prow = off;      off = align256(off + (size_t)T * sizeof(int32_t));
  L.xp = off;        off = align256(off + (size_t)T * c.hidden_dim * 2);
  L.h = off;         off = align256(off + std::max(h_rows, h_tiled));
  L.ys = off;        off = align256(off + std::max((size_t)T * c.hidden_dim * sizeof(float), ys_tiled));
  // scratch routing outputs for moe_b200_forward_routed's discarded router run
  L.rt_idx = off;    off = align256(off + (size_t)T * sizeof(int32_t));
  L.rt_w = off;      off = align256(off + (size_t)T * sizeof(float));
  L.rt_misc = off;   off = align256(off + (size_t)(2 * c.num_experts + 1 + 2 * T) * sizeof(int32_t));
  // unfused ablation: tiled fp32 gate and up projections [2][f/128][T_pad][128]
  L.gu32 = off;      off = align256(off + (size_t)2 * L.n_ft * L.T_pad * kBM * sizeof(float));
  if (screen_applies(c, B)) {
    const ScreenPlan q = plan_screen(c, B);
    L.s_xq = off;     off = align256(off + (size_t)kScrPlanes * q.B_pad * q.d_pad);
    L.s_wq = off;     off = align256(off + (size_t)kScrPlanes * q.E_pad * q.d_pad);
    L.s_xst = off;    off = align256(off + (size_t)B * sizeof(int4));
    L.s_xqs = off;    off = align256(off + (size_t)B * sizeof(long long));
    L.s_part = off;   off = align256(off + screen_part_rows(c, B) * q.E_pad * sizeof(long long));
    L.s_cand = off;   off = align256(off + (size_t)B * kScrMaxCand * sizeof(int32_t));
    L.s_ncand = off;  off = align256(off + (size_t)B * sizeof(int32_t));
    L.s_elist = off;  off = align256(off + (size_t)c.num_experts * B * sizeof(int32_t));
    L.s_rpart = off;  off = align256(off + (size_t)q.n_rs * B * kScrMaxCand * sizeof(double2));
  }
  L.total = off;
  return L;
}

int check_config(const moe_b200_config* c) {
  if (!c) return MOE_B200_ERR_INVALID_VALUE;
  if (c->num_experts < 1 || c->hidden_dim < 1 || c->ffn_dim < 1) return MOE_B200_ERR_INVALID_VALUE;
  if (c->top_k < 1 || c->top_k > c->num_experts) return MOE_B200_ERR_INVALID_K;
  if (c->gating != MOE_B200_GATING_SOFTMAX && c->gating != MOE_B200_GATING_SIGMOID_NORMALIZED)
    return MOE_B200_ERR_INVALID_VALUE;
  if (c->num_experts > kMaxExperts) return MOE_B200_ERR_UNSUPPORTED;
  if (c->hidden_dim % 8 || c->ffn_dim % 8) return MOE_B200_ERR_UNSUPPORTED;
  return MOE_B200_OK;
}

int check_ws(const moe_b200_config* c, int64_t B, void* ws, size_t ws_bytes, Layout* L, int s_force = 0) {
  *L = layout_for(*c, B, s_force);
  if (!ws || ws_bytes < L->total) {
    g_last_error = "workspace too small";
    return MOE_B200_ERR_WORKSPACE;
  }
  if (reinterpret_cast<uintptr_t>(ws) % 256) {
    g_last_error = "workspace must be 256-byte aligned";
    return MOE_B200_ERR_WORKSPACE;
  }
  return MOE_B200_OK;
}

// --------------------------- TMA descriptor encoding --------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int get_encoder() {
  std::call_once(g_encode_once, []() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    g_last_error = "cuTensorMapEncodeTiled unavailable";
    return MOE_B200_ERR_CUDA;
  }
  return MOE_B200_OK;
}

// Host cost per forward: encoded tensor maps are cached by their inputs (the
// weight stacks and workspace regions of a layer repeat call after call), so
// the common case is a lookup, not an encode.
struct MapKey {
  const void* base;
  uint64_t rows, cols;
  uint32_t box_cols, box_rows;
  uint32_t blocks;  // 0: 2-D map; > 0: 3-D weight view with this many 64-column blocks per box
  bool operator==(const MapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && box_cols == o.box_cols &&
           box_rows == o.box_rows && blocks == o.blocks;
  }
};
constexpr int kMapCache = 64;
struct MapCache {
  std::mutex mu;
  MapKey key[kMapCache];
  CUtensorMap map[kMapCache];
  int n = 0, next = 0;
};
MapCache g_maps;

int encode_map_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                    uint32_t box_rows);

// Row-major bf16 matrix (rows x cols), box (box_cols x box_rows), 128B swizzle.
int make_map_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                  uint32_t box_cols, uint32_t box_rows) {
  const MapKey k{base, rows, cols, box_cols, box_rows, 0};
  std::lock_guard<std::mutex> lock(g_maps.mu);
  for (int i = 0; i < g_maps.n; ++i)
    if (g_maps.key[i] == k) {
      *m = g_maps.map[i];
      return MOE_B200_OK;
    }
  const int rc = encode_map_bf16(m, base, rows, cols, box_cols, box_rows);
  if (rc) return rc;
  const int slot = g_maps.n < kMapCache ? g_maps.n++ : (g_maps.next++ % kMapCache);
  g_maps.key[slot] = k;
  g_maps.map[slot] = *m;
  return MOE_B200_OK;
}

int encode_map_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                    uint32_t box_rows) {
  int rc = get_encoder();
  if (rc) return rc;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d)", (int)r);
    g_last_error = buf;
    return MOE_B200_ERR_CUDA;
  }
  return MOE_B200_OK;
}

// A weight matrix (rows x cols bf16, cols % 64 == 0) as a 3-D tensor
// [cols / 64][rows][64]: box {64, box_rows, 2} loads two adjacent 64-column
// halves -- one 16 KB weight slot -- in one TMA instruction, in the same
// shared-memory layout as two 2-D boxes.
int encode_map_w3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                   uint32_t box_blocks = 2) {
  int rc = get_encoder();
  if (rc) return rc;
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_blocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_last_error = "cuTensorMapEncodeTiled(3-D weights) failed";
    return MOE_B200_ERR_CUDA;
  }
  return MOE_B200_OK;
}

// encode_map_w3d through the map cache (every launch_ffn call asks for them)
int make_map_w3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                 uint32_t box_blocks) {
  const MapKey k{base, rows, cols, 64, box_rows, box_blocks};
  std::lock_guard<std::mutex> lock(g_maps.mu);
  for (int i = 0; i < g_maps.n; ++i)
    if (g_maps.key[i] == k) {
      *m = g_maps.map[i];
      return MOE_B200_OK;
    }
  const int rc = encode_map_w3d(m, base, rows, cols, box_rows, box_blocks);
  if (rc) return rc;
  const int slot = g_maps.n < kMapCache ? g_maps.n++ : (g_maps.next++ % kMapCache);
  g_maps.key[slot] = k;
  g_maps.map[slot] = *m;
  return MOE_B200_OK;
}

// Largest dynamic shared memory already granted per (kernel, device):
// cudaFuncSetAttribute is a driver call, so it runs only when a launch needs more.
cudaError_t ensure_dyn_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& g : granted)
    if (g.first.first == kern && g.first.second == dev) {
      if (bytes <= g.second) return cudaSuccess;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
      if (e == cudaSuccess) g.second = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) granted.push_back({{kern, dev}, bytes});
  return e;
}

// Preferred shared-memory carveout of the small kernels (router, dispatch,
// combine): the persistent FFN runs at the maximum carveout, so kernels that
// ask for a different L1 / shared split make the SMs reconfigure at every
// boundary.  MOE_B200_CARVEOUT (percent) sets it; once per (kernel, value).
void apply_carveout(const void* kern) {
  const int v = tuning().carveout;
  if (v < 0) return;
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& d : done)
    if (d.first == kern && d.second == v) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaGetLastError();
  done.push_back({kern, v});
}

// ------------------------------- launches --------------------------------------
// Launch with programmatic stream serialization (PDL) when MOE_B200_PDL=1:
// the kernel may start while its predecessor finishes and calls pdl_wait()
// before reading the predecessor's outputs (common.cuh).  Off by default: it
// measured no gain on the graph-replayed forward (A/B 510 vs 508 us, Mixtral;
// on the FFN -> combine edge alone 601 vs 600 us Mixtral, 209 vs 209 us Qwen;
// round 2, all edges: Mixtral-512 562 vs 575, Qwen 200.9 vs 200.7, DeepSeek
// 3394 vs 3392, skew64 574.5 vs 580.9 us).  (Its one failure -- the overlapped
// combine launched before the dispatch finished, ffn.cuh -- is fixed; the GPU
// suites pass with it on.)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool on, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args&&... args) {
  const bool disabled = !on;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = disabled ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  return launch_pdl_if(tuning().pdl != 0, kern, grid, block, smem, s, std::forward<Args>(args)...);
}



unsigned long long* g_ffn_trace = nullptr;  // debug: per-tile timeline of the next ffn launches
unsigned long long* g_dispatch_trace = nullptr;  // debug: per-CTA dispatch timeline
unsigned long long* g_router_trace = nullptr;  // debug: CTA-0 per-chunk router timeline
struct RouterPlan {
  int expc, te, tt, tokc, n_eblocks, n_tblocks, threads, d_pad, stages, kc;
  size_t smem;
};

// Router CTA shape: expc experts x tokc tokens; each compute thread owns a
// te x tt register tile of sequential fp64 chains; 4 producer warps stage
// operands.  Large B*E (DeepSeek) is fp64-throughput bound: 2x4 tiles keep
// shared-memory wavefronts under the DFMA rate.  Small B*E (Mixtral, Qwen)
// is chain-latency bound (d x 8.2 cycles): 1x1 tiles and few tokens per CTA
// spread the chains over >= ~120 SMs.
RouterPlan plan_router(const moe_b200_config& c, int64_t B, int x_bf16) {
  RouterPlan r{};
  const int E = c.num_experts;
  r.expc = std::min(E, 32);
  r.n_eblocks = (E + r.expc - 1) / r.expc;
  r.d_pad = (c.hidden_dim + kRouterKC - 1) / kRouterKC * kRouterKC;
  const int64_t target = (kNumSMs * 4) / 5;
  const int64_t chains = B * (int64_t)E;
  if (chains >= 64LL * 1024 && r.expc % 2 == 0) {
    // 32 x 32 blocks: 4 experts x 2 tokens per thread in the quarter-warp
    // layout (router_kernel kQ) when the expert block is 32 wide; else 2 x 4
    // strided tiles (DeepSeek-512 A/B of the strided tiles: 2x2 within
    // +-0.5%, 4x4 +9%, 2x1 over 16-token blocks +4%)
    r.te = 2; r.tt = 4; r.tokc = 32;
    if (r.expc == 32 && tuning().rx_quarter != 0) r.te = 4, r.tt = 2;
    {  // tuning: MOE_B200_RX_TILE="te,tt,tokc"
      const int te = tuning().rx_te, tt = tuning().rx_tt, tokc = tuning().rx_tokc;
      if (te > 0 &&
          ((te == 2 && (tt == 2 || tt == 4)) || (te == 4 && tt == 4) ||
           (te == 4 && tt == 2 && tokc == 32 && r.expc == 32)) &&
          tokc >= tt && tokc % tt == 0 && r.expc % te == 0 &&
          (r.expc / te) * (tokc / tt) + kRouterProducers <= 384) {  // router_kernel's launch bound
        r.te = te; r.tt = tt; r.tokc = tokc;
      }
    }
  } else {
    r.te = 1; r.tt = 1;
    int g = 1;
    while (g * 2 * r.expc <= 256 && g * 2 <= 64 && ((B + g * 2 - 1) / (g * 2)) * r.n_eblocks >= target) g *= 2;
    r.tokc = g;
  }
  const int compute = ((r.expc / r.te) * (r.tokc / r.tt) + 31) / 32 * 32;
  r.threads = compute + kRouterProducers;
  r.n_tblocks = static_cast<int>((B + r.tokc - 1) / r.tokc);
  const int xb = x_bf16 ? 2 : 4;
  // latency regime: long k-chunks amortise the per-chunk barrier cost;
  // throughput regime: 64-wide chunks keep >= 4 stages of 2x4-tile operands
  r.kc = r.te == 1 ? 128 : 64;
  const size_t sb = RouterSmem::stage_bytes(r.tokc, r.expc, xb, r.kc);
  r.stages = static_cast<int>(std::min<size_t>(kRouterMaxStages, (180u * 1024) / sb));
  r.stages = std::max(r.stages, 2);
  r.smem = RouterSmem::total_bytes(r.tokc, r.expc, xb, E, r.threads, r.stages, r.kc);
  return r;
}

template <bool kBf16, int kTE, int kTT, int kKC>
int launch_router_t(const CUtensorMap& tmx, const RouterParams& p, const RouterPlan& plan, cudaStream_t s) {
  auto kern = router_kernel<kBf16, kTE, kTT, kKC>;
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(kern), plan.smem));
  kern<<<plan.n_tblocks * plan.n_eblocks, plan.threads, plan.smem, s>>>(tmx, p);
  MOE_LAUNCH_CHECK("router_kernel");
  return MOE_B200_OK;
}

template <bool kBf16>
int launch_router_x(const CUtensorMap& tmx, const RouterParams& p, const RouterPlan& plan, cudaStream_t s) {
  if (plan.te == 4 && plan.tt == 2) return launch_router_t<kBf16, 4, 2, 64>(tmx, p, plan, s);
  if (plan.te == 4) return launch_router_t<kBf16, 4, 4, 64>(tmx, p, plan, s);
  if (plan.te == 2 && plan.tt == 2) return launch_router_t<kBf16, 2, 2, 64>(tmx, p, plan, s);
  if (plan.te == 2) return launch_router_t<kBf16, 2, 4, 64>(tmx, p, plan, s);
  return launch_router_t<kBf16, 1, 1, 128>(tmx, p, plan, s);
}

template <int kBN, int kV, int kPM = 0>
int launch_ffn_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& cm, const CUtensorMap& dm,
                 const CUtensorMap& e, const FfnParams& p, int grid, cudaStream_t s) {
  constexpr bool kPair = kPM != 0;
  using C = FfnCfg<kBN, kV, kPM == 2>;
  auto kern = ffn_kernel<kBN, kV, kPM>;
  static bool attr_set[64] = {};
  int dev = 0;
  MOE_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    MOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaError_t err;
  if constexpr (kPair) {
    // clusters of two CTAs (same TPC) sharing token loads
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFfnThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelEx(&cfg, kern, a, b, cm, dm, e, p);
  } else {
    err = launch_pdl(kern, dim3(grid), dim3(kFfnThreads), C::kSmemBytes, s, a, b, cm, dm, e, p);
  }
  if (err != cudaSuccess) return cuda_fail(err, "ffn launch");
  return MOE_B200_OK;
}

int launch_ffn_kernel(int bn, int variant, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& cm,
                      const CUtensorMap& dm, const CUtensorMap& e, const FfnParams& p, int grid,
                      cudaStream_t s) {
  if (p.pair == 2) {  // cta_group::2 pairs
    return bn == 256 ? launch_ffn_t<256, 2, 2>(a, b, cm, dm, e, p, grid, s)
                     : launch_ffn_t<128, 2, 2>(a, b, cm, dm, e, p, grid, s);
  }
  if (p.pair) {
    return bn == 256 ? launch_ffn_t<256, 2, 1>(a, b, cm, dm, e, p, grid, s)
                     : launch_ffn_t<128, 2, 1>(a, b, cm, dm, e, p, grid, s);
  }
  if (bn == 256)
    return variant == 3 ? launch_ffn_t<256, 3>(a, b, cm, dm, e, p, grid, s) : launch_ffn_t<256, 2>(a, b, cm, dm, e, p, grid, s);
  return variant == 3 ? launch_ffn_t<128, 3>(a, b, cm, dm, e, p, grid, s) : launch_ffn_t<128, 2>(a, b, cm, dm, e, p, grid, s);
}

// FFN launch modes: kFfnFused = gate+up and down in one launch over the tiled
// layouts (down tiles wait on per-chunk gate+up release); kFfnStaged = one
// projection per launch over row layouts (stage API); kFfnUnfusedGU = gate and
// up as separate tiles writing fp32 (ablation); kFfnTiledDown = down tiles
// only over the tiled h (after the ablation's activation pass).
enum FfnMode { kFfnFused = 0, kFfnStaged = 1, kFfnUnfusedGU = 2, kFfnTiledDown = 3 };

int launch_ffn(const moe_b200_config& c, int64_t B, const Layout& L, void* ws, const void* xp,
               const void* w_gate, const void* w_up, const void* w_down, void* h, float* ys,
               const float* topk_w, const int32_t* fwd, bool do_gu, bool do_dn, int mode,
               cudaStream_t s, float* gu32 = nullptr, int32_t* arrive = nullptr) {
  NvtxRange nvtx("moe_b200.ffn");
  const bool fused = (mode != kFfnStaged);  // tiled padded-row layouts
  const int E = c.num_experts, d = c.hidden_dim, f = c.ffn_dim;
  const int64_t T = B * c.top_k;
  CUtensorMap m_wg, m_wu, m_xp, m_wd, m_h;
  int rc;
  const void* any_w = do_gu ? w_gate : w_down;
  // 3-D weight views (one TMA per 16 KB weight slot) when every weight's
  // column count is a multiple of 64 (else the 2-D maps zero-fill the tail)
  const bool w3d = tuning().w3d != 0 && f % 64 == 0 && d % 64 == 0;
  auto wmap = [&](CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
    return w3d ? make_map_w3d(m, base, rows, cols, 64, 2) : make_map_bf16(m, base, rows, cols, 64, 64);
  };
  if ((rc = wmap(&m_wg, do_gu ? w_gate : any_w, do_gu ? (uint64_t)E * d : (uint64_t)E * f, do_gu ? f : d))) return rc;
  if ((rc = wmap(&m_wu, do_gu ? w_up : any_w, do_gu ? (uint64_t)E * d : (uint64_t)E * f, do_gu ? f : d))) return rc;
  if ((rc = wmap(&m_wd, do_dn ? w_down : any_w, do_dn ? (uint64_t)E * f : (uint64_t)E * d, do_dn ? d : f))) return rc;
  if ((rc = make_map_bf16(&m_xp, do_gu ? xp : h, T, do_gu ? d : f, 64, kBoxRows))) return rc;
  if (fused) {
    // tiled h: [n_ft * T_pad rows][128 cols]
    if ((rc = make_map_bf16(&m_h, h, (uint64_t)L.n_ft * L.T_pad, kBM, 64, kBoxRows))) return rc;
  } else if ((rc = make_map_bf16(&m_h, do_dn ? h : xp, T, do_dn ? f : d, 64, kBoxRows))) {
    return rc;
  }
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  FfnParams p{};
  p.chunk_tab = reinterpret_cast<const int4*>(static_cast<uint8_t*>(ws) + L.chunk_tab);
  p.chunk_grp = reinterpret_cast<const int2*>(p.chunk_tab + L.max_chunks);
  p.n_chunks = hdr + 2;
  p.n_mt_gu = do_gu ? (f + kBM - 1) / kBM : 0;
  p.n_mt_dn = do_dn ? (d + 2 * kBM - 1) / (2 * kBM) : 0;
  p.splits = fused ? L.splits : 1;
  p.kb_per_split = fused ? L.kb_per_split : (f + kBK - 1) / kBK;
  p.d = d; p.f = f; p.T = static_cast<int>(T);
  p.h = static_cast<__nv_bfloat16*>(h);
  p.ys = ys;
  p.topk_w = topk_w;
  p.fwd = fwd;
  p.scale_by_w = (!fused && topk_w) ? 1 : 0;
  p.gu_wait = (mode == kFfnFused && do_gu && do_dn) ? 1 : 0;
  p.gu_unfused = (mode == kFfnUnfusedGU) ? 1 : 0;
  p.gu32 = gu32;
  p.work_counter = hdr + 3;
  p.exit_counter = hdr + 4;
  p.gu_done = hdr + kHdrGuDone;
  p.tiled = fused ? 1 : 0;
  p.T_pad = L.T_pad;
  p.tmem_db = tuning().tmem_db != 0;
  p.w3d = w3d ? 1 : 0;
  if (w3d && do_dn && tuning().w3d > 1) {  // down tiles' two slots in one request (not for CTA pairs)
    if ((rc = make_map_w3d(&p.tm_wd4, w_down, (uint64_t)E * f, d, 64, 4))) return rc;
    p.wd4 = 1;
  }
  if (arrive && mode == kFfnFused && do_gu && do_dn) {
    // the down epilogue publishes per-(token, block) arrivals for the combine
    // grid that runs overlapped with this grid's tail
    p.arrive = arrive;
    p.k = c.top_k;
  }
  p.trace = g_ffn_trace;
  const int bn = chunk_rows_for(c, B);
  // CTA pairs for large token chunks, where token re-reads are a real share of
  // the L2 -> SM traffic: one cta_group::2 MMA per pair, each CTA holding half
  // the token rows (mode 2; under the 1 kW cap Mixtral-512 ~6% faster than the
  // multicast pair, mode 1, from the saved data movement; a tie uncapped).
  // MOE_B200_FFN_PAIR=0/1/2 forces a mode (all bit-identical).
  p.pair = (mode == kFfnFused && bn == 256) ? 2 : 0;
  if (tuning().ffn_pair >= 0) p.pair = mode == kFfnFused ? std::min(2, tuning().ffn_pair) : 0;
  long max_tiles = (long)L.max_chunks * (p.n_mt_gu * (p.gu_unfused ? 2 : 1) + p.n_mt_dn * p.splits);
  int grid = static_cast<int>(std::max(1L, std::min<long>(kNumSMs, max_tiles)));
  if (p.pair) grid = std::max(2, grid & ~1);  // whole clusters
  const int variant = tuning().ffn_variant;
  return launch_ffn_kernel(bn, variant, m_wg, m_wu, m_xp, m_wd, m_h, p, grid, s);
}

int grid_for_rows(long total_vec) {
  long blocks = (total_vec + kRowThreads - 1) / kRowThreads;
  long cap = (long)kNumSMs * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

uint8_t* ws8(void* ws) { return static_cast<uint8_t*>(ws); }

int launch_router_exact(const moe_b200_config& c, int64_t B, const void* x, int xb, const float* w_router,
                        const Layout& L, void* ws, RouterParams& p, cudaStream_t s) {
  const moe_b200_config* cfg = &c;
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  RouterPlan plan = plan_router(c, B, xb);
  if (plan.n_tblocks > kTbCap) return MOE_B200_ERR_UNSUPPORTED;
  double* w64 = reinterpret_cast<double*>(ws8(ws) + L.w64);
  {
    // exact fp32 -> fp64 widening of W_r into the chunked expert-block layout
    const long total = (long)plan.n_eblocks * plan.d_pad * plan.expc;
    const int grid = static_cast<int>(std::min<long>((total + 255) / 256, (long)kNumSMs * 8));
    router_prep_kernel<<<grid, 256, 0, s>>>(w_router, w64, cfg->hidden_dim, cfg->num_experts, plan.expc,
                                           plan.d_pad, plan.n_eblocks, reinterpret_cast<uint32_t*>(hdr));
    MOE_LAUNCH_CHECK("router_prep_kernel");
  }
  p.w64 = w64;
  p.tokc = plan.tokc; p.expc = plan.expc;
  p.n_eblocks = plan.n_eblocks; p.n_tblocks = plan.n_tblocks;
  p.stages = plan.stages;
  CUtensorMap tmx;
  {
    int rc2 = get_encoder();
    if (rc2) return rc2;
    cuuint64_t dims[2] = {(cuuint64_t)cfg->hidden_dim, (cuuint64_t)B};
    cuuint64_t strides[1] = {(cuuint64_t)cfg->hidden_dim * (xb ? 2 : 4)};
    cuuint32_t box[2] = {(cuuint32_t)plan.kc, (cuuint32_t)plan.tokc};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(&tmx, xb ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                          const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      g_last_error = "cuTensorMapEncodeTiled(x) failed";
      return MOE_B200_ERR_CUDA;
    }
  }
  return xb ? launch_router_x<true>(tmx, p, plan, s) : launch_router_x<false>(tmx, p, plan, s);
}


int launch_combine(const moe_b200_config& c, int64_t B, const Layout& L, void* ws, const float* topk_w, void* y,
                   int y_dtype, cudaStream_t s, int32_t* arrive = nullptr) {
  NvtxRange nvtx("moe_b200.combine");
  if (y_dtype != MOE_B200_DTYPE_F32 && y_dtype != MOE_B200_DTYPE_BF16) return MOE_B200_ERR_INVALID_VALUE;
  const int d = c.hidden_dim, k = c.top_k;
  const float* ys = reinterpret_cast<const float*>(ws8(ws) + L.ys);
  const int32_t* prow = reinterpret_cast<const int32_t*>(ws8(ws) + L.prow);
  const bool bf = y_dtype == MOE_B200_DTYPE_BF16;
  const int S = L.splits;
  cudaError_t e;
  if (arrive) {
    // overlapped with the FFN's tail: programmatic dependent launch, the
    // CTAs wait on the FFN's per-(token, block) arrival counters
    using K = void (*)(const float*, int, int, const int32_t*, const float*, void*, int, int, int, int32_t*, int);
    const bool wide = k * S <= kCombineMaxKS / 4;
    K kern;
#define MOE_COMBINE_PICK(SS)                                                                   \
  kern = wide ? (bf ? combine_flag_kernel<true, SS, 4> : combine_flag_kernel<false, SS, 4>) \
              : (bf ? combine_flag_kernel<true, SS, 1> : combine_flag_kernel<false, SS, 1>)
    switch (S) {  // (small batches: S up to 8 with k * S <= kCombineMaxKS)
      case 1: MOE_COMBINE_PICK(1); break;
      case 2: MOE_COMBINE_PICK(2); break;
      case 3: MOE_COMBINE_PICK(3); break;
      case 4: MOE_COMBINE_PICK(4); break;
      case 5: MOE_COMBINE_PICK(5); break;
      case 6: MOE_COMBINE_PICK(6); break;
      case 7: MOE_COMBINE_PICK(7); break;
      default: MOE_COMBINE_PICK(8); break;
    }
#undef MOE_COMBINE_PICK
    const int nv = wide ? 4 : 1;
    const unsigned col_blocks = (unsigned)((d / 4 + kRowThreads * nv - 1) / (kRowThreads * nv));
    apply_carveout(reinterpret_cast<const void*>(kern));
    e = launch_pdl_if(true, kern, dim3((unsigned)B, col_blocks), dim3(kRowThreads), 0, s, ys, L.n_dp, L.T_pad, prow,
                      topk_w, y, (int)B, k, d, arrive, S);
  } else if (S <= 4 && k * S <= kCombineMaxKS) {
    using K = void (*)(const float*, int, int, const int32_t*, const float*, void*, int, int, int);
    const bool wide = k * S <= kCombineMaxKS / 4;  // 4 columns per thread
    K kern;
#define MOE_COMBINE_PICK(SS)                                                                   \
  kern = wide ? (bf ? combine_token_kernel<true, SS, 4> : combine_token_kernel<false, SS, 4>) \
              : (bf ? combine_token_kernel<true, SS, 1> : combine_token_kernel<false, SS, 1>)
    switch (S) {
      case 1: MOE_COMBINE_PICK(1); break;
      case 2: MOE_COMBINE_PICK(2); break;
      case 3: MOE_COMBINE_PICK(3); break;
      default: MOE_COMBINE_PICK(4); break;
    }
#undef MOE_COMBINE_PICK
    const int nv = wide ? 4 : 1;
    const unsigned col_blocks = (unsigned)((d / 4 + kRowThreads * nv - 1) / (kRowThreads * nv));
    e = launch_pdl(kern, dim3((unsigned)B, col_blocks), dim3(kRowThreads), 0, s, ys, L.n_dp, L.T_pad, prow, topk_w, y,
                   (int)B, k, d);
  } else {
    const int grid = grid_for_rows((long)B * (d / 4));
    e = launch_pdl(bf ? combine_tiled_kernel<true> : combine_tiled_kernel<false>, dim3(grid), dim3(kRowThreads), 0, s,
                   ys, S, L.n_dp, L.T_pad, prow, topk_w, y, (int)B, k, d);
  }
  if (e != cudaSuccess) return cuda_fail(e, "combine launch");
  return MOE_B200_OK;
}

int launch_dispatch(const moe_b200_config& c, int64_t B, const void* x, int xb, const int32_t* topk_idx,
                    int32_t* counts, int32_t* offsets, int32_t* fwd, int32_t* inv, int32_t* prow, int4* chunk_tab,
                    int32_t* n_chunks, void* xp, cudaStream_t s, uint32_t* flags = nullptr,
                    int32_t* tok_cnt = nullptr, int splits = 1) {
  NvtxRange nvtx("moe_b200.dispatch");
  DispatchParams q{};
  q.tok_cnt = tok_cnt;
  q.n_dp = (c.hidden_dim + 2 * kBM - 1) / (2 * kBM);
  q.splits = splits;
  q.trace = g_dispatch_trace;
  q.flags = flags;
  q.topk_idx = topk_idx;
  q.T = static_cast<int>(B * c.top_k); q.k = c.top_k; q.E = c.num_experts; q.d = c.hidden_dim;
  q.chunk_rows = chunk_rows_for(c, B);
  q.x = x; q.xp = static_cast<__nv_bfloat16*>(xp);
  q.counts = counts; q.offsets = offsets; q.fwd = fwd; q.inv = inv; q.prow = prow;
  q.chunk_tab = chunk_tab; q.n_chunks = n_chunks;
  q.chunk_grp = reinterpret_cast<int2*>(chunk_tab + layout_for(c, B).max_chunks);
  const int grid = (q.T + kDispRows - 1) / kDispRows;
  const bool smem_idx = q.T <= kDispSmemT;
  const size_t smem = (((5 * c.num_experts + 3 + 3) & ~3) + (smem_idx ? ((q.T + 3) & ~3) : 0)) * sizeof(int32_t);
  auto kern = xb ? (smem_idx ? dispatch_kernel<true, true> : dispatch_kernel<true, false>)
                 : (smem_idx ? dispatch_kernel<false, true> : dispatch_kernel<false, false>);
  if (smem > 48 * 1024) MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  apply_carveout(reinterpret_cast<const void*>(kern));
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kDispThreads), smem, s, q);
  if (e != cudaSuccess) return cuda_fail(e, "dispatch launch");
  return MOE_B200_OK;
}


}  // namespace

// ================================ C ABI =======================================
extern "C" {

const char* moe_b200_version(void) { return "moe_b200 0.2.0 (sm_100a)"; }

int moe_b200_record_event(void* event, void* stream) {
  if (!event) return MOE_B200_ERR_INVALID_VALUE;
  MOE_CUDA(record_event(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)));
  return MOE_B200_OK;
}

int moe_b200_combine_overlapped(const moe_b200_config* cfg, int64_t num_tokens) {
  if (check_config(cfg)) return 0;
  return combine_overlapped(*cfg, num_tokens) ? 1 : 0;
}

int moe_b200_tuning_reload(void) {
  reload_tuning();
  return MOE_B200_OK;
}

// Debug hook (not part of the public header): record a per-tile timeline of
// subsequent ffn launches into a device buffer of 4 u64 per tile, or NULL to stop.
void moe_b200_debug_set_ffn_trace(unsigned long long* dev_buf) { g_ffn_trace = dev_buf; }
void moe_b200_debug_set_router_trace(unsigned long long* dev_buf) { g_router_trace = dev_buf; }
void moe_b200_debug_set_dispatch_trace(unsigned long long* dev_buf) { g_dispatch_trace = dev_buf; }

const char* moe_b200_last_error_detail(void) { return g_last_error.c_str(); }

// Debug hook (not part of the public header): byte offset of the certified
// logit-interval buffer (float2 per (token, expert)) inside the workspace.
size_t moe_b200_debug_lbuf_offset(const moe_b200_config* cfg, int64_t max_tokens) {
  return layout_for(*cfg, max_tokens).lbuf;
}

const char* moe_b200_strerror(int status) {
  switch (status) {
    case MOE_B200_OK: return "ok";
    case MOE_B200_ERR_NON_FINITE_INPUT: return "NonFiniteInput: input contains NaN or infinity";
    case MOE_B200_ERR_SHAPE_MISMATCH: return "ShapeMismatch: operand shapes are inconsistent";
    case MOE_B200_ERR_INVALID_K: return "InvalidK: top_k outside [1, num_experts]";
    case MOE_B200_ERR_INDEX_OUT_OF_RANGE: return "IndexOutOfRange: index outside its valid range";
    case MOE_B200_ERR_INVALID_BLOCK_M: return "InvalidBlockM: block_m must be a positive integer";
    case MOE_B200_ERR_SCHEDULE_MISMATCH: return "ScheduleMismatch: schedule does not tile offsets";
    case MOE_B200_ERR_INVALID_VALUE: return "ValueError: invalid configuration value";
    case MOE_B200_ERR_WORKSPACE: return "workspace too small or misaligned";
    case MOE_B200_ERR_UNSUPPORTED: return "unsupported shape for the sm_100a path";
    case MOE_B200_ERR_CUDA: return "CUDA error";
    case MOE_B200_ERR_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

int moe_b200_workspace_size(const moe_b200_config* cfg, int64_t max_tokens, size_t* bytes) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (max_tokens < 0 || !bytes) return MOE_B200_ERR_INVALID_VALUE;
  reload_tuning();  // (the hooks shape the layout: size and init read the same values)
  // the down-split count falls as B grows (down_split_count) while the padded
  // row space grows: size for the largest B of every split count <= max_tokens
  size_t total = layout_for(*cfg, max_tokens).total;
  const int force = tuning().down_splits;
  const int s_last = down_split_count(*cfg, max_tokens, force);
  int s_prev = down_split_count(*cfg, 1, force);
  for (int64_t b = 2; b <= max_tokens && s_prev > s_last; ++b) {
    const int s_b = down_split_count(*cfg, b, force);
    if (s_b != s_prev) total = std::max(total, layout_for(*cfg, b - 1).total);
    s_prev = s_b;
  }
  *bytes = total;
  return MOE_B200_OK;
}

int moe_b200_workspace_init(const moe_b200_config* cfg, int64_t max_tokens, void* ws,
                            size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (!ws || ws_bytes < kHeaderBytes) return MOE_B200_ERR_WORKSPACE;
  (void)max_tokens;
  reload_tuning();  // the MOE_B200_* hooks are read here, not on the forward path
  MOE_CUDA(cudaMemsetAsync(ws, 0, kHeaderBytes, static_cast<cudaStream_t>(stream)));
  return MOE_B200_OK;
}

int moe_b200_read_flags(const moe_b200_config* cfg, int64_t max_tokens, void* ws, size_t ws_bytes,
                        uint32_t* flags, void* stream) {
  (void)cfg; (void)max_tokens;
  if (!ws || ws_bytes < kHeaderBytes || !flags) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MOE_CUDA(cudaMemcpyAsync(flags, ws, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaMemsetAsync(ws, 0, sizeof(uint32_t), s));
  MOE_CUDA(cudaStreamSynchronize(s));
  return MOE_B200_OK;
}

// Screening router (router_screen.cuh): W max -> digit planes -> INT8 screen
// GEMM -> intervals + candidates -> candidate refinement -> merge + phase 2.
int launch_router_screen(const moe_b200_config& c, int64_t B, const void* x, int xb, const float* w_router,
                         const Layout& L, void* ws, RouterParams& p, cudaStream_t s) {
  const ScreenPlan q = plan_screen(c, B);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  ScreenParams sp{};
  sp.x = x; sp.wr = w_router;
  sp.B = static_cast<int>(B); sp.d = c.hidden_dim; sp.E = c.num_experts; sp.k = c.top_k;
  sp.B_pad = q.B_pad; sp.E_pad = q.E_pad; sp.d_pad = q.d_pad;
  sp.n_ks = q.n_ks; sp.kb_per_split = q.kbps;
  sp.xq = reinterpret_cast<int8_t*>(ws8(ws) + L.s_xq);
  sp.wq = reinterpret_cast<int8_t*>(ws8(ws) + L.s_wq);
  sp.xst = reinterpret_cast<int4*>(ws8(ws) + L.s_xst);
  sp.xqs = reinterpret_cast<long long*>(ws8(ws) + L.s_xqs);
  uint32_t* st = reinterpret_cast<uint32_t*>(hdr + kHdrScr);
  sp.wmax = st; sp.ecount = reinterpret_cast<int32_t*>(st + kMaxExperts); sp.wg2 = st + 2 * kMaxExperts;
  sp.wrs = reinterpret_cast<unsigned long long*>(st + 3 * kMaxExperts);
  sp.spart = reinterpret_cast<long long*>(ws8(ws) + L.s_part);
  sp.cand = reinterpret_cast<int32_t*>(ws8(ws) + L.s_cand);
  sp.ncand = reinterpret_cast<int32_t*>(ws8(ws) + L.s_ncand);
  sp.elist = reinterpret_cast<int32_t*>(ws8(ws) + L.s_elist);
  sp.rpart = reinterpret_cast<double2*>(ws8(ws) + L.s_rpart);
  sp.n_rs = q.n_rs; sp.rs_len = q.rs_len; sp.rs_first = q.rs_first;
  sp.lbuf = p.lbuf;
  sp.flags = p.flags;
  // TMA maps over the stacked digit planes (rows: plane-major)
  CUtensorMap tmx, tmw;
  {
    int rc = get_encoder();
    if (rc) return rc;
    auto enc = [&](CUtensorMap* m, void* base, int rows) -> bool {
      cuuint64_t dims[2] = {(cuuint64_t)q.d_pad, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)q.d_pad};
      cuuint32_t box[2] = {(cuuint32_t)kScrKB, (cuuint32_t)kScrM};
      cuuint32_t estr[2] = {1, 1};
      return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!enc(&tmx, sp.xq, kScrPlanes * q.B_pad) || !enc(&tmw, sp.wq, kScrPlanes * q.E_pad)) {
      g_last_error = "cuTensorMapEncodeTiled(screen digits) failed";
      return MOE_B200_ERR_CUDA;
    }
  }
  screen_wmax_kernel<<<dim3((c.hidden_dim + 63) / 64, (c.num_experts + 31) / 32), 256, 0, s>>>(sp);
  MOE_LAUNCH_CHECK("screen_wmax_kernel");
  const int n_wtiles = (q.d_pad / kScrKB) * (q.E_pad / 32);
  if (xb) screen_digits_kernel<true><<<static_cast<unsigned>(B + n_wtiles), 256, 0, s>>>(sp);
  else screen_digits_kernel<false><<<static_cast<unsigned>(B + n_wtiles), 256, 0, s>>>(sp);
  MOE_LAUNCH_CHECK("screen_digits_kernel");
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(screen_gemm_kernel), kScrGemmSmem));
  screen_gemm_kernel<<<q.n_tt * q.n_eb * q.n_ks, kScrThreads, kScrGemmSmem, s>>>(tmx, tmw, sp);
  MOE_LAUNCH_CHECK("screen_gemm_kernel");
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(screen_select_kernel), q.sel_smem));
  screen_select_kernel<<<static_cast<unsigned>(B), kScrSelThreads, q.sel_smem, s>>>(sp);
  MOE_LAUNCH_CHECK("screen_select_kernel");
  auto ref = xb ? screen_refine_kernel<true> : screen_refine_kernel<false>;
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(ref), q.ref_smem));
  ref<<<q.n_rs, kScrRefThreads, q.ref_smem, s>>>(sp);
  MOE_LAUNCH_CHECK("screen_refine_kernel");
  p.screen = 1;
  p.seg_len = 0;
  const double coef = ldexp((2.0 + 12.0 / q.rs_len) * (1.0 + ldexp(1.0, -20)), -53);
  auto ph2 = xb ? screen_phase2_kernel<true> : screen_phase2_kernel<false>;
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(ph2), q.ph2_smem));
  ph2<<<static_cast<unsigned>((B + kScrPh2Tok - 1) / kScrPh2Tok), kScrPh2Threads, q.ph2_smem, s>>>(sp, p, coef);
  MOE_LAUNCH_CHECK("screen_phase2_kernel");
  return MOE_B200_OK;
}

// route + dispatch; xp != nullptr also gathers the permuted bf16 tokens
static int route_impl(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                      const float* w_router, int32_t* topk_idx, float* topk_w, int32_t* counts,
                      int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, float* logits,
                      void* ws, size_t ws_bytes, void* stream, void* xp, void* mid_event = nullptr) {
  NvtxRange nvtx("moe_b200.route");
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B < 0) return MOE_B200_ERR_SHAPE_MISMATCH;
  if (x_dtype != MOE_B200_DTYPE_F32 && x_dtype != MOE_B200_DTYPE_BF16) return MOE_B200_ERR_INVALID_VALUE;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  if (B == 0) {
    MOE_CUDA(cudaMemsetAsync(counts, 0, cfg->num_experts * sizeof(int32_t), s));
    MOE_CUDA(cudaMemsetAsync(offsets, 0, (cfg->num_experts + 1) * sizeof(int32_t), s));
    MOE_CUDA(cudaMemsetAsync(hdr + 2, 0, sizeof(int32_t), s));
    return MOE_B200_OK;
  }
  if (!x || !w_router || !topk_idx || !topk_w || !counts || !offsets || !perm_fwd || !perm_inv)
    return MOE_B200_ERR_INVALID_VALUE;
  const int xb = x_dtype == MOE_B200_DTYPE_BF16;
  RouterParams p{};
  p.x = x; p.wr = w_router; p.x_bf16 = xb;
  p.B = static_cast<int>(B); p.d = cfg->hidden_dim; p.E = cfg->num_experts; p.k = cfg->top_k;
  p.gating = cfg->gating;
  p.chunk_rows = chunk_rows_for(*cfg, B);
  p.logits = logits;
  p.want_logits = logits != nullptr;
  p.force_exact = tuning().force_exact;
  p.lbuf = reinterpret_cast<float2*>(ws8(ws) + L.lbuf);
  p.topk_idx = topk_idx; p.topk_w = topk_w; p.counts = counts; p.offsets = offsets;
  p.fwd = perm_fwd; p.inv = perm_inv;
  p.chunk_tab = reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab);
  p.prow = reinterpret_cast<int32_t*>(ws8(ws) + L.prow);
  p.n_chunks = hdr + 2;
  p.tb_counter = hdr + kHdrTb;
  p.flags = reinterpret_cast<uint32_t*>(hdr);
  p.trace = g_router_trace;

  bool fused_disp = false;
  const bool use_screen = screen_applies(*cfg, B) && !p.want_logits && !p.force_exact;
  if (B <= seg_max_tokens(*cfg) && !use_screen) {
    // latency regime: certified split-K segments (router_seg.cuh)
    const SegPlan q = plan_seg(*cfg, B);
    if (q.n_tb > kTbCap || (long)q.n_tb * q.n_eb > kBlkCap) return MOE_B200_ERR_UNSUPPORTED;
    p.tokc = q.tt; p.expc = q.expc;
    p.n_eblocks = q.n_eb; p.n_tblocks = q.n_tb;
    p.kr = q.kr; p.seg_len = q.seg_len; p.n_kb = q.n_kb;
    p.cert_coef = ldexp((2.0 + 12.0 / q.seg_len) * (1.0 + ldexp(1.0, -20)), -53);
    p.blk_counter = hdr + kHdrBlk;
    p.gpart = ws8(ws) + L.gpart;
    // small batch: the router's last phase-2 CTA runs the dispatch too
    // (one token block: with two, the last-arriver hand-off and the single-CTA
    // gather cost more than the dispatch launch -- Mixtral B=8 +1.4 us)
    fused_disp = B <= kSegTT && B * cfg->top_k <= kFuseMaxT && tuning().fuse_dispatch != 0 &&
                 L.max_chunks <= kChunkCap;
    p.fuse_dispatch = fused_disp;
    p.xp = static_cast<__nv_bfloat16*>(xp);
    p.chunk_grp = reinterpret_cast<int2*>(reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab) + L.max_chunks);
    p.disp_counter = hdr + kHdrDisp;
    const int grid = q.grid;
    const bool wvec = (cfg->num_experts % 4) == 0;
    void (*kern)(RouterParams) = xb ? (wvec ? router_seg_kernel<true, true> : router_seg_kernel<true, false>)
                                    : (wvec ? router_seg_kernel<false, true> : router_seg_kernel<false, false>);
    if (q.tt == 1)
      kern = xb ? (wvec ? router_seg_kernel<true, true, false, 1> : router_seg_kernel<true, false, false, 1>)
                : (wvec ? router_seg_kernel<false, true, false, 1> : router_seg_kernel<false, false, false, 1>);
    else if (q.tt == 2)
      kern = xb ? (wvec ? router_seg_kernel<true, true, false, 2> : router_seg_kernel<true, false, false, 2>)
                : (wvec ? router_seg_kernel<false, true, false, 2> : router_seg_kernel<false, false, false, 2>);
    if (tuning().seg_w64) {
      // W widened to fp64 once per call (the hot loop then converts only x)
      double* w64 = reinterpret_cast<double*>(ws8(ws) + L.w64);
      const long n = (long)cfg->hidden_dim * cfg->num_experts;
      widen_f64_kernel<<<static_cast<int>(std::min<long>((n + 255) / 256, (long)kNumSMs * 8)), 256, 0, s>>>(
          w_router, w64, n);
      MOE_LAUNCH_CHECK("widen_f64_kernel");
      p.wlin64 = w64;
      kern = xb ? (wvec ? router_seg_kernel<true, true, true> : router_seg_kernel<true, false, true>)
                : (wvec ? router_seg_kernel<false, true, true> : router_seg_kernel<false, false, true>);
    }
    MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(kern), q.smem));
    apply_carveout(reinterpret_cast<const void*>(kern));
    kern<<<grid, kSegThreads, q.smem, s>>>(p);
    MOE_LAUNCH_CHECK("router_seg_kernel");
  } else if (use_screen) {
    if ((rc = launch_router_screen(*cfg, B, x, xb, w_router, L, ws, p, s))) return rc;
  } else if ((rc = launch_router_exact(*cfg, B, x, xb, w_router, L, ws, p, s))) {
    return rc;
  }
  if (mid_event) MOE_CUDA(record_event(static_cast<cudaEvent_t>(mid_event), s));
  if (fused_disp) return MOE_B200_OK;
  return launch_dispatch(*cfg, B, x, xb, topk_idx, counts, offsets, perm_fwd, perm_inv,
                         reinterpret_cast<int32_t*>(ws8(ws) + L.prow), reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                         hdr + 2, xp, s);
}

int moe_b200_route(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                   const float* w_router, int32_t* topk_idx, float* topk_w, int32_t* counts,
                   int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, float* logits,
                   void* ws, size_t ws_bytes, void* stream) {
  return route_impl(cfg, B, x, x_dtype, w_router, topk_idx, topk_w, counts, offsets, perm_fwd, perm_inv,
                    logits, ws, ws_bytes, stream, nullptr);
}

// throughput regime: exact sequential chains, register-tiled (router.cuh)
int moe_b200_permute(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                     const int32_t* perm_fwd, void* xp, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!x || !perm_fwd || !xp) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int T = static_cast<int>(B * cfg->top_k);
  const int d = cfg->hidden_dim;
  const int grid = grid_for_rows((long)T * (d / 8));
  if (x_dtype == MOE_B200_DTYPE_BF16)
    permute_kernel<true><<<grid, kRowThreads, 0, s>>>(x, perm_fwd, static_cast<__nv_bfloat16*>(xp), T, cfg->top_k, d);
  else if (x_dtype == MOE_B200_DTYPE_F32)
    permute_kernel<false><<<grid, kRowThreads, 0, s>>>(x, perm_fwd, static_cast<__nv_bfloat16*>(xp), T, cfg->top_k, d);
  else
    return MOE_B200_ERR_INVALID_VALUE;
  MOE_LAUNCH_CHECK("permute_kernel");
  return MOE_B200_OK;
}

int moe_b200_gate_up(const moe_b200_config* cfg, int64_t B, const void* xp, const void* w_gate,
                     const void* w_up, void* h, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!xp || !w_gate || !w_up || !h) return MOE_B200_ERR_INVALID_VALUE;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (L.max_chunks > kChunkCap) return MOE_B200_ERR_UNSUPPORTED;
  return launch_ffn(*cfg, B, L, ws, xp, w_gate, w_up, nullptr, h, nullptr, nullptr, nullptr,
                    /*gu*/ true, /*dn*/ false, kFfnStaged, s);
}

int moe_b200_down_scatter(const moe_b200_config* cfg, int64_t B, const void* h, const void* w_down,
                          const float* topk_w, const int32_t* perm_fwd, float* ys, void* ws,
                          size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!h || !w_down || !topk_w || !perm_fwd || !ys) return MOE_B200_ERR_INVALID_VALUE;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (L.max_chunks > kChunkCap) return MOE_B200_ERR_UNSUPPORTED;
  return launch_ffn(*cfg, B, L, ws, nullptr, nullptr, nullptr, w_down, const_cast<void*>(h), ys,
                    topk_w, perm_fwd, /*gu*/ false, /*dn*/ true, kFfnStaged, s);
}

int moe_b200_combine(const moe_b200_config* cfg, int64_t B, const float* ys, void* y, int y_dtype,
                     void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!ys || !y) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = cfg->hidden_dim;
  const int grid = grid_for_rows((long)B * (d / 4));
  if (y_dtype == MOE_B200_DTYPE_F32)
    combine_kernel<false><<<grid, kRowThreads, 0, s>>>(ys, y, (int)B, cfg->top_k, d);
  else if (y_dtype == MOE_B200_DTYPE_BF16)
    combine_kernel<true><<<grid, kRowThreads, 0, s>>>(ys, y, (int)B, cfg->top_k, d);
  else
    return MOE_B200_ERR_INVALID_VALUE;
  MOE_LAUNCH_CHECK("combine_kernel");
  return MOE_B200_OK;
}

static int forward_impl(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                     const float* w_router, const void* w_gate, const void* w_up,
                     const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                     int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                     void* ws, size_t ws_bytes, void* stream, void** events, bool unfused = false) {
  NvtxRange nvtx("moe_b200.forward");
  int rc = check_config(cfg);
  if (rc) return rc;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto mark = [&](int i) -> int {
    if (events && events[i]) MOE_CUDA(record_event(static_cast<cudaEvent_t>(events[i]), s));
    return MOE_B200_OK;
  };
  if ((rc = mark(0))) return rc;
  void* xp = ws8(ws) + L.xp;
  void* h = ws8(ws) + L.h;
  float* ys = reinterpret_cast<float*>(ws8(ws) + L.ys);
  // router, then dispatch (scheduler + permute gather) — events[1] between them
  if ((rc = route_impl(cfg, B, x, x_dtype, w_router, topk_idx, topk_w, counts, offsets, perm_fwd, perm_inv,
                       nullptr, ws, ws_bytes, stream, xp, events ? events[1] : nullptr)))
    return rc;
  if (B == 0) return events ? mark(1) : MOE_B200_OK;
  if ((rc = mark(2))) return rc;
  if (L.max_chunks > kChunkCap) return MOE_B200_ERR_UNSUPPORTED;
  const bool overlap = !unfused && combine_overlapped(*cfg, B);
  int32_t* arrive = overlap ? reinterpret_cast<int32_t*>(ws) + kHdrTok : nullptr;
  if (y_dtype != MOE_B200_DTYPE_F32 && y_dtype != MOE_B200_DTYPE_BF16) return MOE_B200_ERR_INVALID_VALUE;
  if (!unfused) {
    if ((rc = launch_ffn(*cfg, B, L, ws, xp, w_gate, w_up, w_down, h, ys, topk_w, perm_fwd,
                         /*gu*/ true, /*dn*/ true, kFfnFused, s, nullptr, arrive)))
      return rc;
  } else {
    // ablation (pipeline.py:316-370): gate and up GEMMs as separate tiles
    // (fp32 out), a separate activation pass, then the down projection
    float* gu32 = reinterpret_cast<float*>(ws8(ws) + L.gu32);
    if ((rc = launch_ffn(*cfg, B, L, ws, xp, w_gate, w_up, w_down, h, ys, topk_w, perm_fwd,
                         /*gu*/ true, /*dn*/ false, kFfnUnfusedGU, s, gu32)))
      return rc;
    const size_t n_per_proj = (size_t)L.n_ft * L.T_pad * kBM;
    const int grid = grid_for_rows((long)(n_per_proj / 4));
    cudaError_t e = launch_pdl(swiglu_tiled_kernel, dim3(grid), dim3(kRowThreads), 0, s, (const float*)gu32,
                               static_cast<__nv_bfloat16*>(h), n_per_proj);
    if (e != cudaSuccess) return cuda_fail(e, "swiglu launch");
    if ((rc = launch_ffn(*cfg, B, L, ws, xp, w_gate, w_up, w_down, h, ys, topk_w, perm_fwd,
                         /*gu*/ false, /*dn*/ true, kFfnTiledDown, s)))
      return rc;
  }
  if (overlap) {
    // no event between the FFN and the overlapped combine (it would serialise
    // them): the "ffn" interval covers both, the "combine" one is empty
    if ((rc = launch_combine(*cfg, B, L, ws, topk_w, y, y_dtype, s, arrive))) return rc;
    if ((rc = mark(3))) return rc;
  } else {
    if ((rc = mark(3))) return rc;
    if ((rc = launch_combine(*cfg, B, L, ws, topk_w, y, y_dtype, s))) return rc;
  }
  return mark(4);
}

int moe_b200_forward(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                     const float* w_router, const void* w_gate, const void* w_up,
                     const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                     int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                     void* ws, size_t ws_bytes, void* stream) {
  return forward_impl(cfg, B, x, x_dtype, w_router, w_gate, w_up, w_down, y, y_dtype, topk_idx, topk_w, counts,
                      offsets, perm_fwd, perm_inv, ws, ws_bytes, stream, nullptr);
}

int moe_b200_forward_unfused(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                             const float* w_router, const void* w_gate, const void* w_up,
                             const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                             int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                             void* ws, size_t ws_bytes, void* stream) {
  return forward_impl(cfg, B, x, x_dtype, w_router, w_gate, w_up, w_down, y, y_dtype, topk_idx, topk_w, counts,
                      offsets, perm_fwd, perm_inv, ws, ws_bytes, stream, nullptr, /*unfused*/ true);
}

int moe_b200_forward_routed(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                            const int32_t* topk_idx, const float* topk_w, const float* w_router,
                            const void* w_gate, const void* w_up, const void* w_down, void* y, int y_dtype,
                            int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, void* ws,
                            size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B < 0) return MOE_B200_ERR_SHAPE_MISMATCH;
  if (x_dtype != MOE_B200_DTYPE_F32 && x_dtype != MOE_B200_DTYPE_BF16) return MOE_B200_ERR_INVALID_VALUE;
  if (y_dtype != MOE_B200_DTYPE_F32 && y_dtype != MOE_B200_DTYPE_BF16) return MOE_B200_ERR_INVALID_VALUE;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!x || !topk_idx || !topk_w || !w_gate || !w_up || !w_down || !y || !counts || !offsets || !perm_fwd ||
      !perm_inv)
    return MOE_B200_ERR_INVALID_VALUE;
  if (L.max_chunks > kChunkCap) return MOE_B200_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  if (w_router) {
    // the paper's override still runs the router projection: route into scratch, discard
    int32_t* r_idx = reinterpret_cast<int32_t*>(ws8(ws) + L.rt_idx);
    float* r_w = reinterpret_cast<float*>(ws8(ws) + L.rt_w);
    int32_t* r_misc = reinterpret_cast<int32_t*>(ws8(ws) + L.rt_misc);
    const int T = static_cast<int>(B * cfg->top_k);
    if ((rc = route_impl(cfg, B, x, x_dtype, w_router, r_idx, r_w, r_misc, r_misc + cfg->num_experts,
                         r_misc + 2 * cfg->num_experts + 1, r_misc + 2 * cfg->num_experts + 1 + T, nullptr, ws,
                         ws_bytes, stream, nullptr)))
      return rc;
  }
  void* xp = ws8(ws) + L.xp;
  void* h = ws8(ws) + L.h;
  float* ys = reinterpret_cast<float*>(ws8(ws) + L.ys);
  const bool overlap = combine_overlapped(*cfg, B);
  int32_t* arrive = overlap ? reinterpret_cast<int32_t*>(ws) + kHdrTok : nullptr;
  if ((rc = launch_dispatch(*cfg, B, x, x_dtype == MOE_B200_DTYPE_BF16, topk_idx, counts, offsets, perm_fwd, perm_inv,
                            reinterpret_cast<int32_t*>(ws8(ws) + L.prow), reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                            hdr + 2, xp, s, reinterpret_cast<uint32_t*>(hdr),
                            arrive, L.splits)))
    return rc;
  if ((rc = launch_ffn(*cfg, B, L, ws, xp, w_gate, w_up, w_down, h, ys, topk_w, perm_fwd,
                       /*gu*/ true, /*dn*/ true, kFfnFused, s, nullptr, arrive)))
    return rc;
  return launch_combine(*cfg, B, L, ws, topk_w, y, y_dtype, s, arrive);
}

int moe_b200_forward_timed(const moe_b200_config* cfg, int64_t B, const void* x, int x_dtype,
                           const float* w_router, const void* w_gate, const void* w_up,
                           const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                           int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                           void* ws, size_t ws_bytes, void* stream, void** events) {
  return forward_impl(cfg, B, x, x_dtype, w_router, w_gate, w_up, w_down, y, y_dtype, topk_idx, topk_w, counts,
                      offsets, perm_fwd, perm_inv, ws, ws_bytes, stream, events);
}

// ----------------------- host-buffer (end-to-end) forward -----------------------

}  // extern "C"

// Host-buffer I/O context.  The compute of a forward is captured once per
// (staging slot, batch, buffer pointers) as a CUDA graph on a private stream
// and replayed on the caller's stream: a graph launch instead of four kernel
// launches with their descriptor / attribute set-up per call (host cost per
// forward ~24 -> a few us).  MOE_B200_* tuning variables are read at capture.
struct IoGraph {
  int slot;
  int64_t B;
  const void* ptrs[12];
  cudaGraphExec_t exec;
};
constexpr int kIoGraphs = 16;

struct moe_b200_io {
  moe_b200_config cfg;
  int64_t max_tokens;
  int x_dtype, y_dtype;
  size_t x_bytes, y_bytes;
  void* x_dev[2];
  void* y_dev[2];
  cudaStream_t s_in, s_out, s_cap;
  cudaEvent_t in_done[2], disp_done[2], comp_done[2], out_done[2];
  int64_t count;
  std::vector<IoGraph> graphs;
  int graphs_off;  // MOE_B200_IO_GRAPHS=0: eager launches
};

extern "C" {

int moe_b200_io_create(const moe_b200_config* cfg, int64_t max_tokens, int x_dtype, int y_dtype,
                       moe_b200_io** io_out) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (!io_out || max_tokens < 1) return MOE_B200_ERR_INVALID_VALUE;
  if ((x_dtype != MOE_B200_DTYPE_F32 && x_dtype != MOE_B200_DTYPE_BF16) ||
      (y_dtype != MOE_B200_DTYPE_F32 && y_dtype != MOE_B200_DTYPE_BF16))
    return MOE_B200_ERR_INVALID_VALUE;
  moe_b200_io* io = new moe_b200_io{};
  io->cfg = *cfg;
  io->max_tokens = max_tokens;
  io->x_dtype = x_dtype;
  io->y_dtype = y_dtype;
  io->x_bytes = (size_t)max_tokens * cfg->hidden_dim * (x_dtype == MOE_B200_DTYPE_BF16 ? 2 : 4);
  io->y_bytes = (size_t)max_tokens * cfg->hidden_dim * (y_dtype == MOE_B200_DTYPE_BF16 ? 2 : 4);
  auto fail = [&](cudaError_t e, const char* what) {
    moe_b200_io_destroy(io);
    return cuda_fail(e, what);
  };
  cudaError_t e;
  for (int i = 0; i < 2; ++i) {
    if ((e = cudaMalloc(&io->x_dev[i], io->x_bytes)) != cudaSuccess) return fail(e, "io x staging");
    if ((e = cudaMalloc(&io->y_dev[i], io->y_bytes)) != cudaSuccess) return fail(e, "io y staging");
    for (cudaEvent_t* ev : {&io->in_done[i], &io->disp_done[i], &io->comp_done[i], &io->out_done[i]})
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "io event");
  }
  if ((e = cudaStreamCreateWithFlags(&io->s_in, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "io stream");
  if ((e = cudaStreamCreateWithFlags(&io->s_out, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "io stream");
  if ((e = cudaStreamCreateWithFlags(&io->s_cap, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "io stream");
  io->graphs_off = tuning().io_graphs == 0;
  *io_out = io;
  return MOE_B200_OK;
}

int moe_b200_io_destroy(moe_b200_io* io) {
  if (!io) return MOE_B200_OK;
  if (io->s_in) cudaStreamSynchronize(io->s_in);
  if (io->s_out) cudaStreamSynchronize(io->s_out);
  for (int i = 0; i < 2; ++i) {
    if (io->x_dev[i]) cudaFree(io->x_dev[i]);
    if (io->y_dev[i]) cudaFree(io->y_dev[i]);
    for (cudaEvent_t ev : {io->in_done[i], io->disp_done[i], io->comp_done[i], io->out_done[i]})
      if (ev) cudaEventDestroy(ev);
  }
  for (IoGraph& g : io->graphs) cudaGraphExecDestroy(g.exec);
  if (io->s_in) cudaStreamDestroy(io->s_in);
  if (io->s_out) cudaStreamDestroy(io->s_out);
  if (io->s_cap) cudaStreamDestroy(io->s_cap);
  delete io;
  return MOE_B200_OK;
}

int moe_b200_forward_host(moe_b200_io* io, int64_t B, const void* x_host, void* y_host, const float* w_router,
                          const void* w_gate, const void* w_up, const void* w_down, int32_t* topk_idx,
                          float* topk_w, int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                          void* ws, size_t ws_bytes, void* stream) {
  if (!io) return MOE_B200_ERR_INVALID_VALUE;
  if (B < 0 || B > io->max_tokens) return MOE_B200_ERR_SHAPE_MISMATCH;
  if (B > 0 && (!x_host || !y_host)) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int slot = static_cast<int>(io->count & 1);
  const size_t xb = (size_t)B * io->cfg.hidden_dim * (io->x_dtype == MOE_B200_DTYPE_BF16 ? 2 : 4);
  const size_t yb = (size_t)B * io->cfg.hidden_dim * (io->y_dtype == MOE_B200_DTYPE_BF16 ? 2 : 4);
  const bool reuse = io->count >= 2;  // this slot's buffers were used by batch count-2
  // copy-in: x_dev[slot] is free once batch count-2's router + dispatch read it
  if (reuse) MOE_CUDA(cudaStreamWaitEvent(io->s_in, io->disp_done[slot], 0));
  if (xb) MOE_CUDA(cudaMemcpyAsync(io->x_dev[slot], x_host, xb, cudaMemcpyHostToDevice, io->s_in));
  MOE_CUDA(cudaEventRecord(io->in_done[slot], io->s_in));
  // compute: after the copy-in, and after batch count-2's copy-out released y_dev[slot]
  MOE_CUDA(cudaStreamWaitEvent(s, io->in_done[slot], 0));
  if (reuse) MOE_CUDA(cudaStreamWaitEvent(s, io->out_done[slot], 0));
  // events[2] is recorded after the dispatch (the last reader of x)
  void* evs[5] = {nullptr, nullptr, io->disp_done[slot], nullptr, nullptr};
  auto run = [&](cudaStream_t st) {
    return forward_impl(&io->cfg, B, io->x_dev[slot], io->x_dtype, w_router, w_gate, w_up, w_down, io->y_dev[slot],
                        io->y_dtype, topk_idx, topk_w, counts, offsets, perm_fwd, perm_inv, ws, ws_bytes, st, evs);
  };
  const void* key[12] = {w_router, w_gate, w_up, w_down, topk_idx, topk_w, counts, offsets, perm_fwd, perm_inv, ws,
                         reinterpret_cast<const void*>(ws_bytes)};
  cudaGraphExec_t exec = nullptr;
  if (!io->graphs_off && B > 0) {
    for (IoGraph& g : io->graphs)
      if (g.slot == slot && g.B == B && memcmp(g.ptrs, key, sizeof(key)) == 0) exec = g.exec;
    if (!exec) {
      // capture this slot / batch once on the private stream (the kernels and
      // the mid-forward event record become graph nodes)
      cudaGraph_t graph = nullptr;
      int rc = MOE_B200_OK;
      if (cudaStreamBeginCapture(io->s_cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        rc = run(io->s_cap);
        const cudaError_t ce = cudaStreamEndCapture(io->s_cap, &graph);
        if (rc == MOE_B200_OK && ce == cudaSuccess && graph &&
            cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess)
          exec = nullptr;
        if (graph) cudaGraphDestroy(graph);
        if (rc) return rc;  // a validation error is reported, not retried
      }
      cudaGetLastError();  // a failed capture leaves no sticky error: run eagerly below
      if (exec) {
        if ((int)io->graphs.size() >= kIoGraphs) {
          cudaGraphExecDestroy(io->graphs.front().exec);
          io->graphs.erase(io->graphs.begin());
        }
        IoGraph g{slot, B, {}, exec};
        memcpy(g.ptrs, key, sizeof(key));
        io->graphs.push_back(g);
      }
    }
  }
  if (exec) {
    MOE_CUDA(cudaGraphLaunch(exec, s));
  } else {
    const int rc = run(s);
    if (rc) return rc;
  }
  MOE_CUDA(cudaEventRecord(io->comp_done[slot], s));
  // copy-out
  MOE_CUDA(cudaStreamWaitEvent(io->s_out, io->comp_done[slot], 0));
  if (yb) MOE_CUDA(cudaMemcpyAsync(y_host, io->y_dev[slot], yb, cudaMemcpyDeviceToHost, io->s_out));
  MOE_CUDA(cudaEventRecord(io->out_done[slot], io->s_out));
  ++io->count;
  return MOE_B200_OK;
}

int moe_b200_io_record(moe_b200_io* io, void* event) {
  if (!io || !event) return MOE_B200_ERR_INVALID_VALUE;
  MOE_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), io->s_out));
  return MOE_B200_OK;
}

int moe_b200_io_wait(moe_b200_io* io, void* event) {
  if (!io || !event) return MOE_B200_ERR_INVALID_VALUE;
  MOE_CUDA(cudaStreamWaitEvent(io->s_in, static_cast<cudaEvent_t>(event), 0));
  MOE_CUDA(cudaStreamWaitEvent(io->s_out, static_cast<cudaEvent_t>(event), 0));
  return MOE_B200_OK;
}

int moe_b200_launches_per_forward(const moe_b200_config* cfg, int64_t B) {
  if (check_config(cfg)) return -1;
  if (B <= 0) return 0;
  // the forward's router path (route_impl): INT8 screen (6 launches), segment
  // router (1; the small-batch dispatch runs inside it), or weight prep + exact
  // router (2); then dispatch, FFN and the combine
  const bool screen = screen_applies(*cfg, B) && !tuning().force_exact;
  const bool seg = !screen && B <= seg_max_tokens(*cfg);
  const bool fused_disp = seg && B <= kSegTT && B * cfg->top_k <= kFuseMaxT && tuning().fuse_dispatch != 0 &&
                          layout_for(*cfg, B).max_chunks <= kChunkCap;
  return (screen ? 6 : seg ? 1 : 2) + (fused_disp ? 0 : 1) + 2;
}

int moe_b200_io_sync(moe_b200_io* io) {
  if (!io) return MOE_B200_ERR_INVALID_VALUE;
  MOE_CUDA(cudaStreamSynchronize(io->s_in));
  MOE_CUDA(cudaStreamSynchronize(io->s_out));
  return MOE_B200_OK;
}

// --------------------------- expert parallelism --------------------------------

int moe_b200_down_splits(const moe_b200_config* cfg, int64_t num_tokens, int* splits) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (num_tokens < 0 || !splits) return MOE_B200_ERR_INVALID_VALUE;
  int kps = 0;
  down_splits(*cfg, std::max<int64_t>(num_tokens, 1), splits, &kps);
  return MOE_B200_OK;
}

int moe_b200_expert_ffn_workspace_size(const moe_b200_config* cfg, int64_t max_rows, int down_splits_max,
                                       size_t* bytes) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (max_rows < 0 || down_splits_max < 0 || !bytes) return MOE_B200_ERR_INVALID_VALUE;
  moe_b200_config c1 = *cfg;
  c1.top_k = 1;
  if (down_splits_max == 0) return moe_b200_workspace_size(&c1, max_rows, bytes);
  *bytes = layout_for(c1, std::max<int64_t>(max_rows, 1), down_splits_max).total;
  return MOE_B200_OK;
}

int moe_b200_expert_ffn(const moe_b200_config* cfg, int64_t n_rows, int down_splits, const int32_t* counts,
                        const void* xp, const void* w_gate, const void* w_up, const void* w_down,
                        float* out_rows, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (n_rows < 0) return MOE_B200_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return MOE_B200_OK;
  if (!counts || !xp || !w_gate || !w_up || !w_down || !out_rows) return MOE_B200_ERR_INVALID_VALUE;
  // the FFN works on T = n_rows rows: lay the workspace out as B = n_rows tokens with k = 1
  moe_b200_config c1 = *cfg;
  c1.top_k = 1;
  Layout L;
  if (down_splits < 0) return MOE_B200_ERR_INVALID_VALUE;
  if ((rc = check_ws(&c1, n_rows, ws, ws_bytes, &L, down_splits))) return rc;
  if (L.max_chunks > kChunkCap || c1.num_experts > 1024) return MOE_B200_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* offsets = reinterpret_cast<int32_t*>(ws8(ws) + L.logits);  // scratch: E+1 ints
  int32_t* prow = reinterpret_cast<int32_t*>(ws8(ws) + L.prow);
  schedule_from_counts_kernel<<<1, 256, 0, s>>>(counts, c1.num_experts, chunk_rows_for(c1, n_rows), offsets,
                                                reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                                                reinterpret_cast<int2*>(ws8(ws) + L.chunk_tab) + 2 * L.max_chunks,
                                                hdr + 2, prow);
  MOE_LAUNCH_CHECK("schedule_from_counts_kernel");
  void* h = ws8(ws) + L.h;
  float* ys = reinterpret_cast<float*>(ws8(ws) + L.ys);
  if ((rc = launch_ffn(c1, n_rows, L, ws, xp, w_gate, w_up, w_down, h, ys, nullptr, nullptr,
                       /*gu*/ true, /*dn*/ true, kFfnFused, s)))
    return rc;
  const int d = c1.hidden_dim;
  row_reduce_kernel<<<grid_for_rows((long)n_rows * (d / 4)), kRowThreads, 0, s>>>(
      ys, L.splits, L.n_dp, L.T_pad, prow, out_rows, static_cast<int>(n_rows), d);
  MOE_LAUNCH_CHECK("row_reduce_kernel");
  return MOE_B200_OK;
}

static int ep_peers_from(const moe_b200_ep_peers* in, moe::EpPeers* out);

int moe_b200_ep_p2p_ffn_return(const moe_b200_config* cfg, int64_t n_rows, int down_splits, const int32_t* counts,
                               const void* xp, const void* w_gate, const void* w_up, const void* w_down,
                               const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch, void* ws,
                               size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  moe::EpPeers P{};
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (n_rows < 0 || down_splits < 0) return MOE_B200_ERR_INVALID_VALUE;
  if (!done_counter) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  moe_b200_config c1 = *cfg;
  c1.top_k = 1;
  const int d = c1.hidden_dim;
  if (d % 4) return MOE_B200_ERR_UNSUPPORTED;
  if (n_rows == 0) {  // nothing received: still publish the (empty) return
    ep_reduce_return_kernel<<<1, 256, 0, s>>>(nullptr, 1, 1, 1, nullptr, nullptr, 0, nullptr, d, P, done_counter,
                                              epoch);
    MOE_LAUNCH_CHECK("ep_reduce_return_kernel");
    return MOE_B200_OK;
  }
  if (!counts || !xp || !w_gate || !w_up || !w_down) return MOE_B200_ERR_INVALID_VALUE;
  Layout L;
  if ((rc = check_ws(&c1, n_rows, ws, ws_bytes, &L, down_splits))) return rc;
  if (L.max_chunks > kChunkCap || c1.num_experts > 1024) return MOE_B200_ERR_UNSUPPORTED;
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* offsets = reinterpret_cast<int32_t*>(ws8(ws) + L.logits);  // scratch: E+1 ints
  int32_t* prow = reinterpret_cast<int32_t*>(ws8(ws) + L.prow);
  schedule_from_counts_kernel<<<1, 256, 0, s>>>(counts, c1.num_experts, chunk_rows_for(c1, n_rows), offsets,
                                                reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                                                reinterpret_cast<int2*>(ws8(ws) + L.chunk_tab) + 2 * L.max_chunks,
                                                hdr + 2, prow);
  MOE_LAUNCH_CHECK("schedule_from_counts_kernel");
  void* h = ws8(ws) + L.h;
  float* ys = reinterpret_cast<float*>(ws8(ws) + L.ys);
  if ((rc = launch_ffn(c1, n_rows, L, ws, xp, w_gate, w_up, w_down, h, ys, nullptr, nullptr,
                       /*gu*/ true, /*dn*/ true, kFfnFused, s)))
    return rc;
  const int grid = std::max(1, std::min<int>(static_cast<int>((n_rows + 7) / 8), kNumSMs * 4));
  ep_reduce_return_kernel<<<grid, 256, 0, s>>>(ys, L.splits, L.n_dp, L.T_pad, prow, P.ids[P.me],
                                               static_cast<int>(n_rows), nullptr, d, P, done_counter, epoch);
  MOE_LAUNCH_CHECK("ep_reduce_return_kernel");
  return MOE_B200_OK;
}

int moe_b200_ep_p2p_ffn_return_async(const moe_b200_config* cfg, int64_t max_rows, int down_splits,
                                     const void* xp, const void* w_gate, const void* w_up, const void* w_down,
                                     const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                                     void* ws, size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  moe::EpPeers P{};
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (max_rows < 1 || down_splits < 0 || !done_counter || !xp || !w_gate || !w_up || !w_down)
    return MOE_B200_ERR_INVALID_VALUE;
  const int lo = P.expert_lo[P.me], E_local = P.expert_lo[P.me + 1] - lo, E = P.expert_lo[P.n];
  if (E_local != cfg->num_experts) return MOE_B200_ERR_SHAPE_MISMATCH;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  moe_b200_config c1 = *cfg;
  c1.top_k = 1;
  const int d = c1.hidden_dim;
  if (d % 4) return MOE_B200_ERR_UNSUPPORTED;
  // the layout (and the FFN grid) for the worst case; the actual rows come
  // from the device-side counts through the chunk table
  Layout L;
  if ((rc = check_ws(&c1, max_rows, ws, ws_bytes, &L, down_splits))) return rc;
  if (L.max_chunks > kChunkCap || c1.num_experts > 1024) return MOE_B200_ERR_UNSUPPORTED;
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* counts = reinterpret_cast<int32_t*>(ws8(ws) + L.rt_misc);    // scratch: E_local ints
  int32_t* offsets = reinterpret_cast<int32_t*>(ws8(ws) + L.logits);    // scratch: E_local + 1 ints
  int32_t* prow = reinterpret_cast<int32_t*>(ws8(ws) + L.prow);
  ep_local_counts_kernel<<<1, 256, 0, s>>>(P, E, lo, E_local, counts, epoch);
  MOE_LAUNCH_CHECK("ep_local_counts_kernel");
  schedule_from_counts_kernel<<<1, 256, 0, s>>>(counts, c1.num_experts, chunk_rows_for(c1, max_rows), offsets,
                                                reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                                                reinterpret_cast<int2*>(ws8(ws) + L.chunk_tab) + 2 * L.max_chunks,
                                                hdr + 2, prow);
  MOE_LAUNCH_CHECK("schedule_from_counts_kernel");
  void* h = ws8(ws) + L.h;
  float* ys = reinterpret_cast<float*>(ws8(ws) + L.ys);
  if ((rc = launch_ffn(c1, max_rows, L, ws, xp, w_gate, w_up, w_down, h, ys, nullptr, nullptr,
                       /*gu*/ true, /*dn*/ true, kFfnFused, s)))
    return rc;
  const int grid = std::max(1, std::min<int>(static_cast<int>((max_rows + 7) / 8), kNumSMs * 4));
  ep_reduce_return_kernel<<<grid, 256, 0, s>>>(ys, L.splits, L.n_dp, L.T_pad, prow, P.ids[P.me],
                                               static_cast<int>(max_rows), offsets + E_local, d, P, done_counter,
                                               epoch);
  MOE_LAUNCH_CHECK("ep_reduce_return_kernel");
  return MOE_B200_OK;
}

int moe_b200_gather_rows(int64_t n_rows, int64_t row_bytes, const void* src, const int32_t* idx,
                         void* dst, void* stream) {
  if (n_rows < 0 || row_bytes <= 0 || row_bytes % 16) return MOE_B200_ERR_INVALID_VALUE;
  if (n_rows == 0) return MOE_B200_OK;
  if (!src || !idx || !dst) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  gather_rows_kernel<<<grid_for_rows((long)n_rows * (row_bytes / 16)), kRowThreads, 0, s>>>(
      static_cast<const uint8_t*>(src), idx, static_cast<uint8_t*>(dst), static_cast<int>(n_rows),
      static_cast<int>(row_bytes));
  MOE_LAUNCH_CHECK("gather_rows_kernel");
  return MOE_B200_OK;
}

int moe_b200_ipc_alloc(size_t bytes, void** ptr, void* handle64) {
  if (!ptr || !handle64 || bytes == 0) return MOE_B200_ERR_INVALID_VALUE;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  MOE_CUDA(cudaMalloc(ptr, bytes));
  MOE_CUDA(cudaMemset(*ptr, 0, bytes));
  cudaIpcMemHandle_t h;
  MOE_CUDA(cudaIpcGetMemHandle(&h, *ptr));
  memcpy(handle64, &h, sizeof(h));
  return MOE_B200_OK;
}

int moe_b200_ipc_open(const void* handle64, void** ptr) {
  if (!ptr || !handle64) return MOE_B200_ERR_INVALID_VALUE;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  MOE_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MOE_B200_OK;
}

int moe_b200_ipc_close(void* ptr) {
  MOE_CUDA(cudaIpcCloseMemHandle(ptr));
  return MOE_B200_OK;
}

int moe_b200_ipc_free(void* ptr) {
  MOE_CUDA(cudaFree(ptr));
  return MOE_B200_OK;
}

static int ep_peers_from(const moe_b200_ep_peers* in, moe::EpPeers* out) {
  if (!in || in->n < 1 || in->n > kEpMaxRanks || in->me < 0 || in->me >= in->n) return MOE_B200_ERR_INVALID_VALUE;
  for (int r = 0; r < in->n; ++r) {
    out->counts[r] = static_cast<int32_t*>(in->counts[r]);
    out->flags[r] = static_cast<unsigned long long*>(in->flags[r]);
    out->rows[r] = static_cast<__nv_bfloat16*>(in->rows[r]);
    out->ids[r] = static_cast<int2*>(in->ids[r]);
    out->home[r] = static_cast<float*>(in->home[r]);
  }
  for (int r = 0; r <= in->n; ++r) out->expert_lo[r] = in->expert_lo[r];
  out->n = in->n;
  out->me = in->me;
  out->epoch_dev = static_cast<unsigned long long*>(in->epoch_dev);
  return MOE_B200_OK;
}

int moe_b200_ep_p2p_counts(const moe_b200_config* cfg, int64_t num_rows, const int32_t* topk_idx,
                           const moe_b200_ep_peers* peers, uint64_t epoch, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  moe::EpPeers P{};
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (num_rows < 0 || (num_rows > 0 && !topk_idx)) return MOE_B200_ERR_INVALID_VALUE;
  if (epoch == 0 && !P.epoch_dev) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = (size_t)cfg->num_experts * sizeof(int32_t);
  ep_counts_kernel<<<1, 256, smem, s>>>(topk_idx, static_cast<int>(num_rows), cfg->num_experts, P, epoch);
  MOE_LAUNCH_CHECK("ep_counts_kernel");
  return MOE_B200_OK;
}

int moe_b200_ep_p2p_wait(const moe_b200_ep_peers* peers, int set, uint64_t epoch, void* stream) {
  moe::EpPeers P{};
  int rc;
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (set < 0 || set >= kEpFlagSets) return MOE_B200_ERR_INVALID_VALUE;
  if (epoch == 0 && !P.epoch_dev) return MOE_B200_ERR_INVALID_VALUE;
  ep_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(P, set, epoch);
  MOE_LAUNCH_CHECK("ep_wait_kernel");
  return MOE_B200_OK;
}

int moe_b200_ep_p2p_dispatch(const moe_b200_config* cfg, int64_t num_tokens, const void* x_bf16,
                             const int32_t* topk_idx, const int32_t* perm_fwd, const int32_t* offsets,
                             const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                             void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  moe::EpPeers P{};
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (!done_counter || (num_tokens > 0 && (!x_bf16 || !topk_idx || !perm_fwd || !offsets)))
    return MOE_B200_ERR_INVALID_VALUE;
  if (cfg->hidden_dim % 8) return MOE_B200_ERR_UNSUPPORTED;
  const int T = static_cast<int>(num_tokens * cfg->top_k);
  const int grid = std::max(1, std::min((T + 7) / 8, kNumSMs));
  const size_t smem = (size_t)cfg->num_experts * sizeof(int32_t);
  ep_dispatch_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x_bf16), topk_idx, perm_fwd, offsets, T, cfg->top_k, cfg->num_experts,
      cfg->hidden_dim, P, done_counter, epoch);
  MOE_LAUNCH_CHECK("ep_dispatch_kernel");
  return MOE_B200_OK;
}

int moe_b200_ep_p2p_return(const moe_b200_config* cfg, int64_t num_rows, const float* out_rows,
                           const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                           void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  moe::EpPeers P{};
  if ((rc = ep_peers_from(peers, &P))) return rc;
  if (!done_counter || (num_rows > 0 && !out_rows)) return MOE_B200_ERR_INVALID_VALUE;
  if (cfg->hidden_dim % 4) return MOE_B200_ERR_UNSUPPORTED;
  const int grid = std::max(1, std::min<int>(static_cast<int>((num_rows + 7) / 8), kNumSMs));
  ep_return_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out_rows, P.ids[P.me], static_cast<int>(num_rows), cfg->hidden_dim, P, done_counter, epoch);
  MOE_LAUNCH_CHECK("ep_return_kernel");
  return MOE_B200_OK;
}

// ------------------------- reference stage API ----------------------------------
// Device implementations of the stage functions the reference exports
// (moeperf/__init__.py:56-78) for callers that run the pipeline stage by stage.

static int stage_grid(long long n, int per_block) {
  const long long b = (n + per_block - 1) / per_block;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, (long long)kNumSMs * 16)));
}

int moe_b200_gate_scores(int64_t B, int E, int gating, const float* logits, float* scores, uint32_t* flag,
                         void* stream) {
  if (B < 0 || E < 1 || E > kMaxExperts) return E > kMaxExperts ? MOE_B200_ERR_UNSUPPORTED : MOE_B200_ERR_INVALID_VALUE;
  if (gating != MOE_B200_GATING_SOFTMAX && gating != MOE_B200_GATING_SIGMOID_NORMALIZED)
    return MOE_B200_ERR_INVALID_VALUE;
  if (B == 0) return MOE_B200_OK;
  if (!logits || !scores || !flag) return MOE_B200_ERR_INVALID_VALUE;
  const size_t smem = (size_t)kStageWarps * E * sizeof(double);
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(gate_scores_kernel), smem));
  gate_scores_kernel<<<stage_grid(B, kStageWarps), kStageWarps * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      logits, scores, static_cast<int>(B), E, gating, flag);
  MOE_LAUNCH_CHECK("gate_scores_kernel");
  return MOE_B200_OK;
}

int moe_b200_topk_select(int64_t B, int E, int k, int gating, const float* scores, int32_t* idx, float* w,
                         void* stream) {
  if (B < 0 || E < 1) return MOE_B200_ERR_INVALID_VALUE;
  if (k < 1 || k > E) return MOE_B200_ERR_INVALID_K;
  if (E > kMaxExperts) return MOE_B200_ERR_UNSUPPORTED;
  if (gating != MOE_B200_GATING_SOFTMAX && gating != MOE_B200_GATING_SIGMOID_NORMALIZED)
    return MOE_B200_ERR_INVALID_VALUE;
  if (B == 0) return MOE_B200_OK;
  if (!scores || !idx || !w) return MOE_B200_ERR_INVALID_VALUE;
  const size_t smem = (size_t)kStageWarps * (E + k) * sizeof(float);
  MOE_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(topk_select_kernel), smem));
  topk_select_kernel<<<stage_grid(B, kStageWarps), kStageWarps * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      scores, idx, w, static_cast<int>(B), E, k, gating);
  MOE_LAUNCH_CHECK("topk_select_kernel");
  return MOE_B200_OK;
}

int moe_b200_sigmoid(int64_t n, const float* x, float* y, int silu, void* stream) {
  if (n < 0) return MOE_B200_ERR_INVALID_VALUE;
  if (n == 0) return MOE_B200_OK;
  if (!x || !y) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (silu) sigmoid_kernel<true><<<stage_grid(n, 256), 256, 0, s>>>(x, y, n);
  else sigmoid_kernel<false><<<stage_grid(n, 256), 256, 0, s>>>(x, y, n);
  MOE_LAUNCH_CHECK("sigmoid_kernel");
  return MOE_B200_OK;
}

int moe_b200_np_exp64(int64_t n, const double* x, double* y, void* stream) {
  if (n < 0) return MOE_B200_ERR_INVALID_VALUE;
  if (n == 0) return MOE_B200_OK;
  if (!x || !y) return MOE_B200_ERR_INVALID_VALUE;
  np_exp64_kernel<<<stage_grid(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n);
  MOE_LAUNCH_CHECK("np_exp64_kernel");
  return MOE_B200_OK;
}

int moe_b200_dense_matmul(int64_t m, int64_t K, int64_t n, const float* a, const float* b, float* c, void* stream) {
  if (m < 0 || K < 0 || n < 0 || m > INT32_MAX || K > INT32_MAX || n > INT32_MAX) return MOE_B200_ERR_INVALID_VALUE;
  if (m == 0 || n == 0) return MOE_B200_OK;
  if (!c || (K > 0 && (!a || !b))) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (K == 0) {
    MOE_CUDA(cudaMemsetAsync(c, 0, (size_t)m * n * sizeof(float), s));
    return MOE_B200_OK;
  }
  dense_matmul_kernel<<<stage_grid(m * n, 256), 256, 0, s>>>(a, b, c, static_cast<int>(m), static_cast<int>(K),
                                                              static_cast<int>(n));
  MOE_LAUNCH_CHECK("dense_matmul_kernel");
  return MOE_B200_OK;
}

int moe_b200_permute_rows(int64_t n_rows, int64_t row_bytes, const void* src, const int32_t* perm_fwd, int k,
                          void* dst, void* stream) {
  if (n_rows < 0 || row_bytes <= 0 || row_bytes % 16 || k < 1) return MOE_B200_ERR_INVALID_VALUE;
  if (n_rows == 0) return MOE_B200_OK;
  if (!src || !perm_fwd || !dst) return MOE_B200_ERR_INVALID_VALUE;
  permute_rows_kernel<<<stage_grid(n_rows * (row_bytes / 16), 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), perm_fwd, k, static_cast<uint8_t*>(dst), static_cast<int>(n_rows),
      static_cast<int>(row_bytes));
  MOE_LAUNCH_CHECK("permute_rows_kernel");
  return MOE_B200_OK;
}

int moe_b200_cast_bf16(int64_t n, const float* x, void* y, void* stream) {
  if (n < 0) return MOE_B200_ERR_INVALID_VALUE;
  if (n == 0) return MOE_B200_OK;
  if (!x || !y) return MOE_B200_ERR_INVALID_VALUE;
  f32_to_bf16_kernel<<<stage_grid(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, static_cast<__nv_bfloat16*>(y), n);
  MOE_LAUNCH_CHECK("f32_to_bf16_kernel");
  return MOE_B200_OK;
}

int moe_b200_swiglu(int64_t n, const float* gu, void* h, void* stream) {
  if (n < 0 || n % 4) return MOE_B200_ERR_INVALID_VALUE;
  if (n == 0) return MOE_B200_OK;
  if (!gu || !h) return MOE_B200_ERR_INVALID_VALUE;
  swiglu_tiled_kernel<<<grid_for_rows(n / 4), kRowThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      gu, static_cast<__nv_bfloat16*>(h), static_cast<size_t>(n));
  MOE_LAUNCH_CHECK("swiglu_kernel");
  return MOE_B200_OK;
}

int moe_b200_schedule(const moe_b200_config* cfg, int64_t B, const int32_t* topk_idx, int32_t* counts,
                      int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, void* ws, size_t ws_bytes,
                      void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B < 0) return MOE_B200_ERR_SHAPE_MISMATCH;
  Layout L;
  if ((rc = check_ws(cfg, B, ws, ws_bytes, &L))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  if (B == 0) {
    MOE_CUDA(cudaMemsetAsync(counts, 0, cfg->num_experts * sizeof(int32_t), s));
    MOE_CUDA(cudaMemsetAsync(offsets, 0, (cfg->num_experts + 1) * sizeof(int32_t), s));
    return MOE_B200_OK;
  }
  if (!topk_idx || !counts || !offsets || !perm_fwd || !perm_inv) return MOE_B200_ERR_INVALID_VALUE;
  return launch_dispatch(*cfg, B, nullptr, 0, topk_idx, counts, offsets, perm_fwd, perm_inv,
                         reinterpret_cast<int32_t*>(ws8(ws) + L.prow), reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                         hdr + 2, nullptr, s, reinterpret_cast<uint32_t*>(hdr));
}

// expert-grouped rows (counts[e] rows for expert e, ascending e): the chunk
// table from the counts, then one FFN launch in row-layout (staged) mode
static int grouped_ffn(const moe_b200_config* cfg, int64_t n_rows, const int32_t* counts, const void* xp,
                       const void* w_gate, const void* w_up, const void* w_down, void* h, float* out, void* ws,
                       size_t ws_bytes, void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (n_rows < 0) return MOE_B200_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return MOE_B200_OK;
  moe_b200_config c1 = *cfg;
  c1.top_k = 1;
  Layout L;
  if ((rc = check_ws(&c1, n_rows, ws, ws_bytes, &L))) return rc;
  if (L.max_chunks > kChunkCap || c1.num_experts > 1024) return MOE_B200_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  schedule_from_counts_kernel<<<1, 256, 0, s>>>(counts, c1.num_experts, chunk_rows_for(c1, n_rows),
                                                reinterpret_cast<int32_t*>(ws8(ws) + L.logits),
                                                reinterpret_cast<int4*>(ws8(ws) + L.chunk_tab),
                                                reinterpret_cast<int2*>(ws8(ws) + L.chunk_tab) + 2 * L.max_chunks,
                                                hdr + 2, reinterpret_cast<int32_t*>(ws8(ws) + L.prow));
  MOE_LAUNCH_CHECK("schedule_from_counts_kernel");
  const bool gu = w_down == nullptr;
  return launch_ffn(c1, n_rows, L, ws, xp, w_gate, w_up, w_down, gu ? h : const_cast<void*>(xp), out, nullptr,
                    nullptr, /*gu*/ gu, /*dn*/ !gu, kFfnStaged, s);
}

int moe_b200_grouped_gate_up(const moe_b200_config* cfg, int64_t n_rows, const int32_t* counts, const void* xp,
                             const void* w_gate, const void* w_up, void* h, void* ws, size_t ws_bytes, void* stream) {
  if (n_rows > 0 && (!counts || !xp || !w_gate || !w_up || !h)) return MOE_B200_ERR_INVALID_VALUE;
  return grouped_ffn(cfg, n_rows, counts, xp, w_gate, w_up, nullptr, h, nullptr, ws, ws_bytes, stream);
}

int moe_b200_grouped_gemm(const moe_b200_config* cfg, int64_t n_rows, const int32_t* counts, const void* a,
                          const void* w_stack, float* out, void* ws, size_t ws_bytes, void* stream) {
  if (n_rows > 0 && (!counts || !a || !w_stack || !out)) return MOE_B200_ERR_INVALID_VALUE;
  return grouped_ffn(cfg, n_rows, counts, a, nullptr, nullptr, w_stack, nullptr, out, ws, ws_bytes, stream);
}

int moe_b200_combine_rows(const moe_b200_config* cfg, int64_t B, const float* rows,
                          const int32_t* perm_inv, const float* topk_w, void* y, int y_dtype,
                          void* stream) {
  int rc = check_config(cfg);
  if (rc) return rc;
  if (B == 0) return MOE_B200_OK;
  if (!rows || !perm_inv || !topk_w || !y) return MOE_B200_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = cfg->hidden_dim;
  const int grid = grid_for_rows((long)B * (d / 4));
  if (y_dtype == MOE_B200_DTYPE_F32)
    combine_rows_kernel<false><<<grid, kRowThreads, 0, s>>>(rows, perm_inv, topk_w, y, (int)B, cfg->top_k, d);
  else if (y_dtype == MOE_B200_DTYPE_BF16)
    combine_rows_kernel<true><<<grid, kRowThreads, 0, s>>>(rows, perm_inv, topk_w, y, (int)B, cfg->top_k, d);
  else
    return MOE_B200_ERR_INVALID_VALUE;
  MOE_LAUNCH_CHECK("combine_rows_kernel");
  return MOE_B200_OK;
}

}  // extern "C"
