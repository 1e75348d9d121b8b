/*
 * moe_b200.h — C-ABI of the B200-native fused MoE-layer forward.
 *
 * Drop-in boundary for the reference `moeperf` hot path
 * (/root/reference/pkg/src/moeperf/pipeline.py:572 `moe_forward`).  The
 * reference has no FFI of its own (it is pure Python/numpy), so the entry
 * points below are exactly the stage functions its Python API exports
 * (moeperf/__init__.py:56-78); each one cites the reference function it
 * replaces.  The Python host mirror (paper_2605_23911_b200/) binds them with
 * ctypes; INTEGRATION.md shows the binding a maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All tensor pointers are DEVICE pointers
 *    (cudaMalloc'd or torch-owned), row-major and contiguous.
 *  - The caller owns every buffer, including the workspace; the library
 *    never allocates in the forward path.
 *  - All calls are asynchronous on `stream` (a cudaStream_t passed as void*),
 *    never synchronise the host, and are CUDA-graph capturable.
 *  - Return value: MOE_B200_OK (0) or one status code per reference
 *    exception class (moeperf/errors.py:9-50) plus CUDA / unsupported codes.
 *  - Expert weights use the reference's stacked layout (moeperf/model.py:119-165):
 *        gate, up : (E*d, f)  bf16, expert e owns rows [e*d, (e+1)*d)
 *        down     : (E*f, d)  bf16, expert e owns rows [e*f, (e+1)*f)
 *    The router weight is (d, E) fp32 (model/router.py:116-133).
 *  - Routing indices are int32 on device (the reference's int64 values fit).
 *  - d and f must be multiples of 8 (16-byte TMA row pitch).
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  Names follow moeperf/errors.py. */
typedef enum moe_b200_status {
  MOE_B200_OK = 0,
  MOE_B200_ERR_NON_FINITE_INPUT = 1,   /* NonFiniteInput      errors.py:13 */
  MOE_B200_ERR_SHAPE_MISMATCH = 2,     /* ShapeMismatch       errors.py:17 */
  MOE_B200_ERR_INVALID_K = 3,          /* InvalidK            errors.py:21 */
  MOE_B200_ERR_INDEX_OUT_OF_RANGE = 4, /* IndexOutOfRange     errors.py:25 */
  MOE_B200_ERR_INVALID_BLOCK_M = 5,    /* InvalidBlockM       errors.py:29 */
  MOE_B200_ERR_SCHEDULE_MISMATCH = 6,  /* ScheduleMismatch    errors.py:33 */
  MOE_B200_ERR_INVALID_VALUE = 7,      /* ValueError (ModelConfig/PipelineParams) */
  MOE_B200_ERR_WORKSPACE = 8,          /* workspace too small / misaligned */
  MOE_B200_ERR_UNSUPPORTED = 9,        /* shape the sm_100a path does not take */
  MOE_B200_ERR_CUDA = 10,              /* CUDA runtime/driver failure */
  MOE_B200_ERR_NCCL = 11               /* expert-parallel collective failure */
} moe_b200_status;

/* Gating mode (moeperf/model.py:14-18). */
#define MOE_B200_GATING_SOFTMAX 0
#define MOE_B200_GATING_SIGMOID_NORMALIZED 1

/* Element dtypes for activations. */
#define MOE_B200_DTYPE_F32 0
#define MOE_B200_DTYPE_BF16 1

/* Static layer shape (moeperf/model.py:21-48 ModelConfig). */
typedef struct moe_b200_config {
  int32_t num_experts; /* E */
  int32_t top_k;       /* k, 1 <= k <= E */
  int32_t hidden_dim;  /* d */
  int32_t ffn_dim;     /* f */
  int32_t gating;      /* MOE_B200_GATING_* */
} moe_b200_config;

/* Device-side status bits, readable with moe_b200_read_flags. */
#define MOE_B200_FLAG_NONFINITE_TOKENS 1u
#define MOE_B200_FLAG_NONFINITE_ROUTER 2u
#define MOE_B200_FLAG_INDEX_OUT_OF_RANGE 4u

/* Bytes of workspace needed for up to `max_tokens` tokens.  The workspace
 * holds the router logits, schedule tables, the permuted bf16 tokens, the
 * bf16 SwiGLU intermediate and the per-slot fp32 expert outputs. */
int moe_b200_workspace_size(const moe_b200_config* cfg, int64_t max_tokens, size_t* bytes);

/* Zero the workspace's self-resetting counters and flags.  Call once after
 * allocating a workspace (the kernels leave them zeroed afterwards). */
int moe_b200_workspace_init(const moe_b200_config* cfg, int64_t max_tokens, void* ws,
                            size_t ws_bytes, void* stream);

/* Router + scheduler, one launch.
 * Replaces router.py:116 `route` (logits, gate_scores, topk_select) and
 * scheduler.py:78-117 (`expert_histogram`, `expert_offsets`,
 * `build_permutation`, `build_block_schedule` as a device tile table).
 * Bit-exact with the reference: fp64 ascending-k logits, numpy pairwise
 * softmax sum / numpy-SIMD sigmoid, lowest-index tie-break, stable sort.
 *   x        (B, d)   fp32 or bf16 (x_dtype)
 *   w_router (d, E)   fp32
 *   topk_idx (B, k)   int32   out: expert ids, descending score
 *   topk_w   (B, k)   fp32    out: combine weights
 *   counts   (E)      int32   out: expert histogram
 *   offsets  (E+1)    int32   out: exclusive prefix sum
 *   perm_fwd (B*k)    int32   out: permuted row -> expanded id t*k+j
 *   perm_inv (B*k)    int32   out: expanded id -> permuted row
 *   logits   (B, E)   fp32    out, optional (NULL): router logits        */
int moe_b200_route(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                   const float* w_router, int32_t* topk_idx, float* topk_w, int32_t* counts,
                   int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, float* logits,
                   void* ws, size_t ws_bytes, void* stream);

/* Gather expert-major rows (pipeline.py:165-183 `permute_tokens`), cast to
 * bf16.  xp (B*k, d) bf16 out. */
int moe_b200_permute(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                     const int32_t* perm_fwd, void* xp, void* stream);

/* Fused gate+up grouped GEMM with SiLU*up epilogue (pipeline.py:250-313
 * `fused_gate_up`): h (B*k, f) bf16 out.  Uses the tile table written by
 * moe_b200_route into `ws`. */
int moe_b200_gate_up(const moe_b200_config* cfg, int64_t num_tokens, const void* xp,
                     const void* w_gate, const void* w_up, void* h, void* ws, size_t ws_bytes,
                     void* stream);

/* Down-projection grouped GEMM (pipeline.py:186-247 `grouped_gemm`) whose
 * epilogue multiplies by the routing weight and scatters each row to its
 * expanded slot (the first half of pipeline.py:373-399):
 *   ys (B*k, d) fp32 out, row t*k+j = w[t,j] * (h_row @ W_down_e). */
int moe_b200_down_scatter(const moe_b200_config* cfg, int64_t num_tokens, const void* h,
                          const void* w_down, const float* topk_w, const int32_t* perm_fwd,
                          float* ys, void* ws, size_t ws_bytes, void* stream);

/* Deterministic combine (second half of pipeline.py:373-399):
 *   y[t] = sum_{j=0..k-1} ys[t*k+j], ascending j, fp32.  y (B, d). */
int moe_b200_combine(const moe_b200_config* cfg, int64_t num_tokens, const float* ys, void* y,
                     int y_dtype, void* stream);

/* Whole layer (pipeline.py:572-615 `moe_forward`): route, dispatch (histogram,
 * offsets, stable permutation, schedule, gather), ONE persistent FFN launch
 * (gate+up and down), and the deterministic weighted unpermute-combine,
 * overlapped with the FFN's tail (moe_b200_combine_overlapped) -- four
 * launches (five with the exact router's weight prep; nine when a sigmoid
 * router above 64K logits runs the INT8 screen), no host synchronisation.
 * Intermediates live in `ws`; routing outputs are written to the caller's
 * buffers so the host can build the trace lazily from `counts`. */
int moe_b200_forward(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                     const float* w_router, const void* w_gate, const void* w_up,
                     const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                     int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                     void* ws, size_t ws_bytes, void* stream);

/* The same layer with the reference's unfused gate+up (pipeline.py:316-370,
 * PipelineParams.fused = False): gate and up as separate grouped GEMMs
 * writing fp32, a separate SiLU*up pass, then the down projection.  The
 * fusion ablation; results are bit-identical to moe_b200_forward. */
int moe_b200_forward_unfused(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                             const float* w_router, const void* w_gate, const void* w_up,
                             const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                             int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                             void* ws, size_t ws_bytes, void* stream);

/* Whole layer with the routing given (the paper's router override for the
 * routing-skew study; tables from moeperf/skew.py:74-105):
 * topk_idx (B, k) int32 and topk_w (B, k) fp32 are INPUTS on the device.
 * Runs dispatch (histogram, offsets, stable permutation, schedule, gather),
 * the fused FFN and the combine.  If w_router is non-NULL the router kernel
 * also runs (its result is discarded), so a timing includes the projection as
 * in the paper's experiment.  Indices outside [0, E) set
 * MOE_B200_FLAG_INDEX_OUT_OF_RANGE and those rows are dropped. */
int moe_b200_forward_routed(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                            const int32_t* topk_idx, const float* topk_w, const float* w_router,
                            const void* w_gate, const void* w_up, const void* w_down, void* y,
                            int y_dtype, int32_t* counts, int32_t* offsets, int32_t* perm_fwd,
                            int32_t* perm_inv, void* ws, size_t ws_bytes, void* stream);

/* Same as moe_b200_forward, recording five cudaEvent_t (events[0..4]) on
 * `stream` around the stages: [route | permute | fused FFN | combine].  Used
 * by the benchmark to time the dominant kernel inside the real forward. */
int moe_b200_forward_timed(const moe_b200_config* cfg, int64_t num_tokens, const void* x, int x_dtype,
                           const float* w_router, const void* w_gate, const void* w_up,
                           const void* w_down, void* y, int y_dtype, int32_t* topk_idx, float* topk_w,
                           int32_t* counts, int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv,
                           void* ws, size_t ws_bytes, void* stream, void** events);

/* --------------------- host-buffer (end-to-end) forward ---------------------
 * The reference API takes and returns host arrays (pipeline.py:572-578:
 * numpy in, numpy out).  An I/O context owns double-buffered device staging
 * for x and y and two copy streams, so that consecutive calls overlap the
 * host<->device copies of one batch with the compute of its neighbours:
 *   copy-in stream:  x_host -> x_dev[i % 2]      (waits for batch i-2's dispatch)
 *   compute stream:  moe_b200_forward(x_dev, y_dev[i % 2])  (waits for copy-in
 *                    and for batch i-2's copy-out of y_dev)
 *   copy-out stream: y_dev[i % 2] -> y_host       (waits for the compute)
 * x_host / y_host should be pinned (page-locked) for the copies to be
 * asynchronous; the caller keeps them untouched until moe_b200_io_sync.
 * The context allocates its staging buffers once (moe_b200_io_create); the
 * forward path itself never allocates. */
typedef struct moe_b200_io moe_b200_io;

int moe_b200_io_create(const moe_b200_config* cfg, int64_t max_tokens, int x_dtype, int y_dtype,
                       moe_b200_io** io);
int moe_b200_io_destroy(moe_b200_io* io);

/* Asynchronous: returns once the copies and launches are enqueued. */
int moe_b200_forward_host(moe_b200_io* io, int64_t num_tokens, const void* x_host, void* y_host,
                          const float* w_router, const void* w_gate, const void* w_up,
                          const void* w_down, int32_t* topk_idx, float* topk_w, int32_t* counts,
                          int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, void* ws,
                          size_t ws_bytes, void* stream);

/* Record `event` (a cudaEvent_t) on the copy-out stream after the last
 * enqueued batch's y copy; make both copy streams wait for `event` (e.g. a
 * timing start recorded on the compute stream); wait for everything. */
int moe_b200_io_record(moe_b200_io* io, void* event);
int moe_b200_io_wait(moe_b200_io* io, void* event);
int moe_b200_io_sync(moe_b200_io* io);

/* Number of kernel launches one moe_b200_forward of `num_tokens` tokens makes
 * (router [+ weight prep], dispatch, FFN, combine). */
int moe_b200_launches_per_forward(const moe_b200_config* cfg, int64_t num_tokens);

/* ---------------------------- expert parallelism ------------------------------
 * The reference has no multi-GPU path ("planned
 * follow-up").  These two entry points are the local compute of an
 * expert-parallel layer whose dispatch/combine all-to-alls run over NCCL
 * (paper_2605_23911_b200/ep.py).  cfg describes the LOCAL expert slice.
 *
 * moe_b200_expert_ffn: rows already grouped by local expert (counts[e] rows for
 * expert e, ascending e) -> unweighted expert outputs, fp32, same row order:
 *   out_rows[r] = silu(x_r Wg_e) * (x_r Wu_e) @ Wd_e   (pipeline.py:250-313, 186-247)
 * Bit-identical, row by row, to the single-GPU forward's per-slot expert output.
 *   counts   (E_local) int32 device; xp (n_rows, d) bf16; out_rows (n_rows, d) fp32
 * down_splits: the K-split count of the down projection (its fp32 partial
 * sums are added in split order, so a row's bits depend on it).  Pass
 * moe_b200_down_splits(global cfg, global token count) to reproduce the
 * single-GPU forward bit for bit; 0 derives it from (cfg, n_rows).
 * Workspace: moe_b200_expert_ffn_workspace_size(cfg, max rows, largest
 * down_splits passed). */
int moe_b200_expert_ffn(const moe_b200_config* cfg, int64_t n_rows, int down_splits, const int32_t* counts,
                        const void* xp, const void* w_gate, const void* w_up, const void* w_down,
                        float* out_rows, void* ws, size_t ws_bytes, void* stream);

/* Workspace bytes for moe_b200_expert_ffn over up to max_rows rows with
 * split counts up to down_splits_max (0: the count derived from cfg). */
int moe_b200_expert_ffn_workspace_size(const moe_b200_config* cfg, int64_t max_rows, int down_splits_max,
                                       size_t* bytes);

/* The K-split count of the down projection that moe_b200_forward uses for
 * num_tokens tokens (more splits for small batches, where few experts are
 * active and the down tiles would otherwise not fill the SMs). */
int moe_b200_down_splits(const moe_b200_config* cfg, int64_t num_tokens, int* splits);

/* Row gather dst[r] = src[idx[r]] (row_bytes a multiple of 16): the reorder
 * between the all-to-all layout (source-major) and expert-major rows. */
int moe_b200_gather_rows(int64_t n_rows, int64_t row_bytes, const void* src, const int32_t* idx,
                         void* dst, void* stream);

/* Home-rank combine (pipeline.py:373-399): rows (B*k, d) fp32 in the local
 * permuted order; y[t] = sum_j fl(w[t,j] * rows[perm_inv[t*k+j]]), ascending j. */
int moe_b200_combine_rows(const moe_b200_config* cfg, int64_t num_tokens, const float* rows,
                          const int32_t* perm_inv, const float* topk_w, void* y, int y_dtype,
                          void* stream);

/* ---- expert parallelism over peer memory (NVLink P2P / CUDA IPC) ----------
 * Replaces the library all-to-alls of the expert-parallel layer (
 * paper_2605_23911_b200/ep.py) with direct writes into the peer ranks' buffers.
 * Buffers are allocated with moe_b200_ipc_alloc, their handles exchanged by the
 * caller (any host transport) and mapped with moe_b200_ipc_open.  Per rank r:
 *   counts[r]  int32 [n][E]          all-gathered per-expert row counts
 *   flags[r]   uint64 [3][n]         epoch flags (counts, rows, returns) per source, zeroed once
 *   rows[r]    bf16 [R_max][d]       expert-major received rows
 *   ids[r]     int32x2 [R_max]       {source rank, expanded id} of each received row
 *   home[r]    fp32 [T_max][d]       returned expert outputs by expanded id
 * `epoch` grows by one per forward (or pass 0 everywhere and give epoch_dev:
 * device-side epochs); flags are never reset. */
#define MOE_B200_EP_MAX_RANKS 16
typedef struct {
  void* counts[MOE_B200_EP_MAX_RANKS];
  void* flags[MOE_B200_EP_MAX_RANKS];
  void* rows[MOE_B200_EP_MAX_RANKS];
  void* ids[MOE_B200_EP_MAX_RANKS];
  void* home[MOE_B200_EP_MAX_RANKS];
  int expert_lo[MOE_B200_EP_MAX_RANKS + 1]; /* rank r owns experts [lo[r], lo[r+1]) */
  int n, me;
  /* local device uint64[2] {counter, current}, zeroed once: with epoch = 0 in
   * every call, moe_b200_ep_p2p_counts advances it on the device and the other
   * steps read it, so a captured CUDA graph of the forward replays correctly */
  void* epoch_dev;
} moe_b200_ep_peers;

/* cudaMalloc + IPC handle (64 bytes, opaque) of the allocation. */
int moe_b200_ipc_alloc(size_t bytes, void** ptr, void* handle64);
/* Map another process's allocation from its handle. */
int moe_b200_ipc_open(const void* handle64, void** ptr);
int moe_b200_ipc_close(void* ptr);
int moe_b200_ipc_free(void* ptr);

/* 1. Counts all-gather: histogram of topk_idx (T = B*k entries, global expert
 *    ids) written into counts[r][me][:] of every rank r, then flag set 0. */
int moe_b200_ep_p2p_counts(const moe_b200_config* cfg, int64_t num_rows, const int32_t* topk_idx,
                           const moe_b200_ep_peers* peers, uint64_t epoch, void* stream);
/* Wait (on the device) until flag set `set` of every source reached `epoch`. */
int moe_b200_ep_p2p_wait(const moe_b200_ep_peers* peers, int set, uint64_t epoch, void* stream);
/* 2. Dispatch: the local permuted rows (perm_fwd / offsets of the local
 *    route) of x (bf16, num_tokens x d) go into the owners' rows / ids at the
 *    single-GPU permutation's expert-major order, then flag set 1.  Waits for
 *    flag set 0 itself.  done_counter: one int32 of device memory, zeroed once. */
int moe_b200_ep_p2p_dispatch(const moe_b200_config* cfg, int64_t num_tokens, const void* x_bf16,
                             const int32_t* topk_idx, const int32_t* perm_fwd, const int32_t* offsets,
                             const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                             void* stream);
/* 3. Return: the num_rows received rows' outputs (fp32, num_rows x d) into
 *    home[source][expanded id], then flag set 2 of every source. */
int moe_b200_ep_p2p_return(const moe_b200_config* cfg, int64_t num_rows, const float* out_rows,
                           const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                           void* stream);

/* 3'. The local expert FFN over the num_rows received rows (expert-major,
 *     counts per local expert; cfg describes the LOCAL expert slice, as for
 *     moe_b200_expert_ffn) with the return fused into its K-split reduction:
 *     each row's output goes straight into home[source][expanded id] of its
 *     home rank, then flag set 2.  Workspace as moe_b200_expert_ffn. */
int moe_b200_ep_p2p_ffn_return(const moe_b200_config* cfg, int64_t num_rows, int down_splits,
                               const int32_t* counts, const void* xp, const void* w_gate, const void* w_up,
                               const void* w_down, const moe_b200_ep_peers* peers, int32_t* done_counter,
                               uint64_t epoch, void* ws, size_t ws_bytes, void* stream);

/* 3'' The same with no host synchronisation: waits for flag set 1 itself,
 *     takes the local per-expert counts from the all-gathered matrix on the
 *     device, and lays the workspace out for up to max_rows received rows
 *     (moe_b200_expert_ffn_workspace_size(cfg, max_rows, down_splits)).  With
 *     moe_b200_ep_p2p_counts / _dispatch / _wait and moe_b200_combine_rows the
 *     whole expert-parallel forward runs without a host synchronisation. */
int moe_b200_ep_p2p_ffn_return_async(const moe_b200_config* cfg, int64_t max_rows, int down_splits,
                                     const void* xp, const void* w_gate, const void* w_up, const void* w_down,
                                     const moe_b200_ep_peers* peers, int32_t* done_counter, uint64_t epoch,
                                     void* ws, size_t ws_bytes, void* stream);

/* ------------------------------ stage API -----------------------------------
 * Device implementations of the reference's stage-level functions
 * (moeperf/__init__.py:56-78) for callers that run the pipeline stage by
 * stage.  The one-call forward above does not use them. */

/* router.py:69-84 `gate_scores` on caller-given logits (B, E) fp32 -> scores
 * (B, E) fp32, bit-exact (numpy pairwise fp64 softmax sum; numpy-SIMD-expf
 * sigmoid).  A non-finite logit sets *flag (device uint32) to 1 and leaves its
 * row unwritten (require_finite, router.py:80). */
int moe_b200_gate_scores(int64_t num_tokens, int num_experts, int gating, const float* logits, float* scores,
                         uint32_t* flag, void* stream);

/* router.py:87-113 `topk_select`: k rounds of numpy argmax (first maximum,
 * NaN first) with -1.0 masking; weights are the picked scores, renormalised
 * by their fp32 pairwise sum in sigmoid mode (1/k when the sum is zero).
 * idx (B, k) int32, w (B, k) fp32.  MOE_B200_ERR_INVALID_K unless 1 <= k <= E. */
int moe_b200_topk_select(int64_t num_tokens, int num_experts, int k, int gating, const float* scores,
                         int32_t* idx, float* w, void* stream);

/* linalg.py:71-80 `sigmoid` (silu = 0) or linalg.py:83-86 `silu` (silu = 1),
 * elementwise over n fp32 values, bit-exact with numpy's float32 path. */
int moe_b200_sigmoid(int64_t n, const float* x, float* y, int silu, void* stream);

/* numpy's float64 exp as the softmax computes it (router.py:65, :82:
 * np.exp on float64; on AVX-512 hosts numpy dispatches to SVML's
 * __svml_exp8_ha, which this reproduces bit for bit for |x| < 707.7; beyond,
 * x < 0 gives +0 -- see router.cuh np_exp64).  Elementwise over n doubles. */
int moe_b200_np_exp64(int64_t n, const double* x, double* y, void* stream);

/* linalg.py:45-68 `dense_matmul`: c (m, n) = a (m, K) @ b (K, n), fp32 in and
 * out, exact fp64 products folded in ascending K (bit-exact). */
int moe_b200_dense_matmul(int64_t m, int64_t K, int64_t n, const float* a, const float* b, float* c,
                          void* stream);

/* scheduler.py:78-103 `expert_histogram` + `expert_offsets` +
 * `build_permutation` from given routing indices (B, k) int32 (no gather).
 * Indices outside [0, E) set MOE_B200_FLAG_INDEX_OUT_OF_RANGE. */
int moe_b200_schedule(const moe_b200_config* cfg, int64_t num_tokens, const int32_t* topk_idx, int32_t* counts,
                      int32_t* offsets, int32_t* perm_fwd, int32_t* perm_inv, void* ws, size_t ws_bytes,
                      void* stream);

/* pipeline.py:165-183 `permute_tokens`, exact: dst[r] = src[perm_fwd[r] / k]
 * for rows of row_bytes (a multiple of 16) bytes. */
int moe_b200_permute_rows(int64_t n_rows, int64_t row_bytes, const void* src, const int32_t* perm_fwd, int k,
                          void* dst, void* stream);

/* fp32 -> bf16 (round to nearest even): the operand cast of the stage GEMMs. */
int moe_b200_cast_bf16(int64_t n, const float* x, void* y, void* stream);

/* pipeline.py:250-313 `fused_gate_up` over expert-grouped rows (counts[e]
 * rows of expert e, ascending e; cfg->top_k ignored):
 *   h (n_rows, f) bf16 = silu(xp Wg_e) * (xp Wu_e)   (tcgen05, fp32 accumulate)
 * Workspace: moe_b200_expert_ffn_workspace_size(cfg, n_rows, 0). */
int moe_b200_grouped_gate_up(const moe_b200_config* cfg, int64_t n_rows, const int32_t* counts, const void* xp,
                             const void* w_gate, const void* w_up, void* h, void* ws, size_t ws_bytes, void* stream);

/* pipeline.py:186-247 `grouped_gemm` over expert-grouped rows: out (n_rows, N)
 * fp32 = a (n_rows, K) bf16 @ W_e, W the flat (E*K, N) bf16 stack; cfg gives
 * E, hidden_dim = N and ffn_dim = K.  Workspace as moe_b200_grouped_gate_up. */
int moe_b200_grouped_gemm(const moe_b200_config* cfg, int64_t n_rows, const int32_t* counts, const void* a,
                          const void* w_stack, float* out, void* ws, size_t ws_bytes, void* stream);

/* The activation pass of pipeline.py:316-370 `unfused_gate_up`:
 * h[i] = bf16(silu(g[i]) * u[i]) with gu = [g (n) | u (n)] fp32, the fused
 * epilogue's exact formula (so fused == unfused bit for bit). */
int moe_b200_swiglu(int64_t n, const float* gu, void* h, void* stream);

/* Copy the device status flags (MOE_B200_FLAG_*) to the host and clear them.
 * Synchronises `stream`. */
int moe_b200_read_flags(const moe_b200_config* cfg, int64_t max_tokens, void* ws,
                        size_t ws_bytes, uint32_t* flags, void* stream);

/* Record `event` (a cudaEvent_t) on `stream`; inside a stream capture it
 * becomes an external event-record node (a timing point of every replay). */
int moe_b200_record_event(void* event, void* stream);

/* 1 when a forward of num_tokens tokens overlaps the weighted
 * unpermute-combine with the FFN's tail: the FFN's down epilogue publishes
 * per-(token, 256-column block) arrivals and the combine grid, launched behind
 * it with programmatic dependent launch, combines each token as soon as its
 * partial rows are in (default while num_tokens * ceil(d / 256) <= 65536 and
 * the down K split is <= 4; MOE_B200_FUSED_COMBINE=0 runs the combine after
 * the FFN -- bit-identical either way). */
int moe_b200_combine_overlapped(const moe_b200_config* cfg, int64_t num_tokens);

/* Re-read the MOE_B200_* tuning / test hooks from the environment.  They are
 * read once (first use) and at every moe_b200_workspace_init, never on the
 * forward path. */
int moe_b200_tuning_reload(void);

/* Human-readable status. */
const char* moe_b200_strerror(int status);

/* Last CUDA error string recorded by the library (thread-local). */
const char* moe_b200_last_error_detail(void);

/* Library version string. */
const char* moe_b200_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MOE_B200_H */
