"""CPU oracle for the MoE-layer forward hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``moeperf`` pipeline
(``/root/reference/pkg/src/moeperf``), written from the reference's
documented algorithm, not copied.  It is the *checker* for the CUDA path:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it.  The product
package (``paper_2605_23911_b200``) never imports or calls it, and has no
CPU fallback.

Parity pin: every function below is checked bit-for-bit against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``; see
``tests/test_oracle_golden.py``), plus the known-answer values the
reference's own tests hold.

Numerics contract (reference ``linalg.py:45-57``): every dot product forms
exact float64 products and folds them strictly left-to-right in ascending
inner index, then rounds to float32 once.  Because the fold order depends
only on the inner index, row/column tiling never changes the bits.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32
F64 = np.float64

SOFTMAX = "softmax"
SIGMOID_NORMALIZED = "sigmoid_normalized"


# ---------------------------------------------------------------------------
# L0 numerics core  (reference linalg.py)
# ---------------------------------------------------------------------------

def dot_fp64_fold(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """``a @ b`` with exact fp64 products, ascending-k fold, one fp32 rounding.

    Follows ``linalg.py:45-57`` (``dot_accumulate``).  The fold is seeded with
    the first product (as ``np.add.accumulate`` is), so the sign of an
    all-zero sum matches the reference too.  Memory is O(m·n) instead of the
    reference's O(m·n·K) temporary; the arithmetic is identical.
    """
    a = np.asarray(a, dtype=F32)
    b = np.asarray(b, dtype=F32)
    m, kdim = a.shape
    n = b.shape[1]
    if kdim == 0:
        return np.zeros((m, n), dtype=F32)
    a64 = a.astype(F64)
    b64 = b.astype(F64)
    acc = a64[:, 0:1] * b64[0:1, :]
    for kk in range(1, kdim):
        acc += a64[:, kk : kk + 1] * b64[kk : kk + 1, :]
    return acc.astype(F32)


def sigmoid_f32(x) -> np.ndarray:
    """Split-form logistic in float32 (``linalg.py:71-80``).

    ``t = exp(-|x|)`` in float32 (numpy's SIMD expf), then ``1/(1+t)`` for
    x >= 0 and ``t/(1+t)`` otherwise, all float32.
    """
    x = np.asarray(x, dtype=F32)
    t = np.exp(-np.abs(x))
    one = F32(1.0)
    return np.where(x >= 0, one / (one + t), t / (one + t)).astype(F32)


def silu_f32(x) -> np.ndarray:
    """``x * sigmoid(x)`` in float32 (``linalg.py:83-86``)."""
    x = np.asarray(x, dtype=F32)
    return (x * sigmoid_f32(x)).astype(F32)


# ---------------------------------------------------------------------------
# L2 router  (reference router.py)
# ---------------------------------------------------------------------------

def router_logits(tokens: np.ndarray, router_weight: np.ndarray) -> np.ndarray:
    """``logits = tokens @ W_r`` via the canonical fold (``router.py:131``)."""
    return dot_fp64_fold(tokens, router_weight)


def gate_scores(logits: np.ndarray, gating: str) -> np.ndarray:
    """Softmax or sigmoid gate scores (``router.py:69-84``).

    softmax: fp32 max-subtract, fp64 exp, fp64 (numpy pairwise) row sum,
    fp64 divide, one fp32 rounding.  sigmoid: float32 ``sigmoid_f32``.
    """
    logits = np.asarray(logits, dtype=F32)
    if gating == SOFTMAX:
        if logits.shape[0] == 0:
            return logits.copy()
        shifted = (logits - logits.max(axis=1, keepdims=True)).astype(F32)
        e = np.exp(shifted.astype(F64))
        return (e / e.sum(axis=1, keepdims=True)).astype(F32)
    if gating == SIGMOID_NORMALIZED:
        return sigmoid_f32(logits)
    raise ValueError(f"unknown gating {gating!r}")


def topk_select(scores: np.ndarray, k: int, gating: str):
    """Iterative argmax top-k with -1.0 masking (``router.py:87-113``).

    Returns ``(indices int64 (B,k), weights float32 (B,k))``; ties go to the
    lowest expert index (``np.argmax``).  Sigmoid mode renormalises the k
    selected scores by their float32 (pairwise) sum; a zero sum falls back to
    uniform ``1/k``.  Softmax weights are *not* renormalised.
    """
    scores = np.asarray(scores, dtype=F32)
    nt, ne = scores.shape
    if not 1 <= k <= ne:
        raise ValueError(f"k must be in [1, {ne}], got {k}")
    work = scores.copy()
    idx = np.empty((nt, k), dtype=np.int64)
    w = np.empty((nt, k), dtype=F32)
    rows = np.arange(nt)
    for j in range(k):
        best = work.argmax(axis=1) if nt else np.empty(0, dtype=np.int64)
        idx[:, j] = best
        w[:, j] = scores[rows, best]
        work[rows, best] = F32(-1.0)
    if gating == SIGMOID_NORMALIZED and nt:
        s = w.sum(axis=1, keepdims=True)
        zero = s == 0.0
        w = (w / np.where(zero, F32(1.0), s)).astype(F32)
        w[zero.ravel()] = F32(1.0 / k)
    return idx, w


def route(tokens, router_weight, k: int, gating: str):
    """Full router (``router.py:116-133``): logits → scores → top-k."""
    logits = router_logits(tokens, router_weight)
    return topk_select(gate_scores(logits, gating), k, gating)


# ---------------------------------------------------------------------------
# L2 scheduler  (reference scheduler.py)
# ---------------------------------------------------------------------------

def expert_histogram(indices: np.ndarray, num_experts: int) -> np.ndarray:
    """Per-expert count of expanded assignments (``scheduler.py:78-82``)."""
    flat = np.asarray(indices, dtype=np.int64).reshape(-1)
    return np.bincount(flat, minlength=num_experts).astype(np.int64)


def expert_offsets(counts: np.ndarray) -> np.ndarray:
    """Exclusive prefix sum, length E+1 (``scheduler.py:85-94``)."""
    counts = np.asarray(counts, dtype=np.int64)
    off = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off


def build_permutation(indices: np.ndarray):
    """Stable expert-major order of expanded ids ``t*k+j`` (``scheduler.py:97-103``).

    Restated as a counting sort: row ``off[e] + rank`` holds the rank-th
    expanded id routed to expert e, ids taken in ascending order.
    """
    flat = np.asarray(indices, dtype=np.int64).reshape(-1)
    n = flat.size
    ne = int(flat.max()) + 1 if n else 0
    off = expert_offsets(np.bincount(flat, minlength=ne)) if n else np.zeros(1, np.int64)
    cursor = off[:-1].copy()
    forward = np.empty(n, dtype=np.int64)
    for i in range(n):
        e = flat[i]
        forward[cursor[e]] = i
        cursor[e] += 1
    inverse = np.empty(n, dtype=np.int64)
    inverse[forward] = np.arange(n, dtype=np.int64)
    return forward, inverse


def build_block_schedule(offsets: np.ndarray, block_m: int):
    """Algorithm 1 tile list ``(e, local_start)`` (``scheduler.py:106-117``)."""
    entries = []
    for e in range(offsets.size - 1):
        n_e = int(offsets[e + 1] - offsets[e])
        entries.extend((e, s) for s in range(0, n_e, block_m))
    return tuple(entries)


# ---------------------------------------------------------------------------
# L3 pipeline stages  (reference pipeline.py)
# ---------------------------------------------------------------------------

def permute_tokens(tokens: np.ndarray, forward: np.ndarray, k: int) -> np.ndarray:
    """Row ``r`` ← token ``forward[r] // k`` (``pipeline.py:165-183``)."""
    return np.ascontiguousarray(np.asarray(tokens, dtype=F32)[forward // k])


def fused_gate_up(permuted, gate, up, offsets, hidden_dim: int) -> np.ndarray:
    """``h = silu(A·Wg_e) * (A·Wu_e)`` per expert segment (``pipeline.py:250-313``).

    Tiling never changes bits (ascending-k fold), so each expert's rows are
    done as one block.
    """
    total = int(offsets[-1])
    f = gate.shape[1]
    out = np.zeros((total, f), dtype=F32)
    d = hidden_dim
    for e in range(offsets.size - 1):
        r0, r1 = int(offsets[e]), int(offsets[e + 1])
        if r1 == r0:
            continue
        a = permuted[r0:r1]
        g = dot_fp64_fold(a, gate[e * d : (e + 1) * d])
        u = dot_fp64_fold(a, up[e * d : (e + 1) * d])
        out[r0:r1] = (silu_f32(g) * u).astype(F32)
    return out


def grouped_gemm(inp, weight_stack, offsets) -> np.ndarray:
    """Expert-grouped GEMM over an ``(E*K, N)`` stack (``pipeline.py:186-247``)."""
    total = int(offsets[-1])
    kdim = inp.shape[1]
    n = weight_stack.shape[1]
    out = np.zeros((total, n), dtype=F32)
    for e in range(offsets.size - 1):
        r0, r1 = int(offsets[e]), int(offsets[e + 1])
        if r1 == r0:
            continue
        out[r0:r1] = dot_fp64_fold(inp[r0:r1], weight_stack[e * kdim : (e + 1) * kdim])
    return out


def unpermute_combine(expert_out, weights, inverse) -> np.ndarray:
    """``y[t] = Σ_j fl(w[t,j]·Y[inverse[t·k+j]])``, ascending j, fp32 (``pipeline.py:373-399``)."""
    b, k = weights.shape
    hidden = expert_out.shape[1]
    out = np.zeros((b, hidden), dtype=F32)
    if b == 0:
        return out
    g = expert_out[inverse.reshape(b, k)]
    for j in range(k):
        out += weights[:, j : j + 1] * g[:, j]
    return out


def moe_forward(tokens, router_weight, gate, up, down, num_experts, k, gating,
                routing=None, ffn=None):
    """Whole layer (``pipeline.py:572-615``) → dict of every intermediate.

    ``routing`` optionally overrides ``(indices, weights)`` (the paper's
    routing-override for the skew sweep); ``ffn`` optionally
    replaces the gate_up/down pair with another implementation of the same
    arithmetic, ``ffn(permuted, offsets) -> (h, expert_out)``.
    """
    tokens = np.ascontiguousarray(np.asarray(tokens, dtype=F32))
    d = tokens.shape[1]
    if routing is None:
        idx, w = route(tokens, router_weight, k, gating)
    else:
        idx, w = routing
    counts = expert_histogram(idx, num_experts)
    off = expert_offsets(counts)
    fwd, inv = build_permutation(idx)
    xp = permute_tokens(tokens, fwd, k)
    if ffn is None:
        h = fused_gate_up(xp, gate, up, off, d)
        ys = grouped_gemm(h, down, off)
    else:
        h, ys = ffn(xp, off)
    y = unpermute_combine(ys, w, inv)
    return dict(indices=idx, weights=w, counts=counts, offsets=off, forward=fwd,
                inverse=inv, permuted=xp, h=h, expert_out=ys, y=y)


def dense_moe_oracle(tokens, router_weight, gate, up, down, num_experts, k, gating):
    """Per-token loop over selected experts (``pipeline.py:618-643``)."""
    tokens = np.asarray(tokens, dtype=F32)
    d = tokens.shape[1]
    f = gate.shape[1]
    idx, w = route(tokens, router_weight, k, gating)
    out = np.zeros((tokens.shape[0], d), dtype=F32)
    for t in range(tokens.shape[0]):
        x = tokens[t : t + 1]
        acc = np.zeros((1, d), dtype=F32)
        for j in range(k):
            e = int(idx[t, j])
            g = dot_fp64_fold(x, gate[e * d : (e + 1) * d])
            u = dot_fp64_fold(x, up[e * d : (e + 1) * d])
            h = (silu_f32(g) * u).astype(F32)
            acc += w[t, j] * dot_fp64_fold(h, down[e * f : (e + 1) * f])
        out[t] = acc[0]
    return out


def moe_rows(tokens, router_weight, expert, num_experts, k, gating, routing=None):
    """Layer output for a subset of tokens, fetching only the experts they use.

    Rows of the reference forward are independent (``SPEC.md:155-156``;
    ``dense_moe_oracle`` is bitwise ``moe_forward``, ``pipeline.py:618-643``),
    so y for a token subset is the dense per-token restatement over just those
    tokens: route them (``router.py:116-133``), then for every selected expert
    ``g = x Wg_e, u = x Wu_e, h = silu(g) * u, o = h Wd_e`` with the canonical
    fp64 fold, combined ``out += w_j * o_j`` in ascending j from zero
    (``pipeline.py:396-399``).  ``expert(e)`` returns ``(gate_e (d,f), up_e
    (d,f), down_e (f,d))`` float32 — a full-size layer (DeepSeek-V3: 45 GB in
    fp32) never has to be materialised on the host.  Tokens that share an
    expert are folded together (same bits: the fold is per output element).
    """
    tokens = np.ascontiguousarray(np.asarray(tokens, dtype=F32))
    b, d = tokens.shape
    if routing is None:
        idx, w = route(tokens, router_weight, k, gating)
    else:
        idx, w = routing
    outs = {}
    for e in np.unique(idx):
        rows, slots = np.nonzero(idx == e)
        ge, ue, de = expert(int(e))
        a = tokens[rows]
        g = dot_fp64_fold(a, ge)
        u = dot_fp64_fold(a, ue)
        h = (silu_f32(g) * u).astype(F32)
        o = dot_fp64_fold(h, de)
        for i, (r, j) in enumerate(zip(rows, slots)):
            outs[(int(r), int(j))] = o[i]
    y = np.zeros((b, d), dtype=F32)
    for j in range(idx.shape[1]):
        for r in range(b):
            y[r] += w[r, j] * outs[(r, j)]
    return dict(indices=idx, weights=w, y=y)


def max_rel_error(y, y_ref) -> float:
    """``max|y−y_ref| / max(max|y_ref|, 1e-6)`` — the reference verify metric (``cli.py:733-737``)."""
    y = np.asarray(y, dtype=F64)
    y_ref = np.asarray(y_ref, dtype=F64)
    if y_ref.size == 0:
        return 0.0
    return float(np.max(np.abs(y - y_ref)) / max(float(np.max(np.abs(y_ref))), 1e-6))


# ---------------------------------------------------------------------------
# Synthetic instances  (reference tests/conftest.py:37-58, model.py:147-156)
# ---------------------------------------------------------------------------

def make_instance(seed, num_experts=4, top_k=2, hidden_dim=8, ffn_dim=12, batch=9):
    """The reference's canonical PCG64 instance: tokens, *unscaled* W_r, weights.

    Draw order (one ``Generator(PCG64(seed))``): tokens N(0,1) (B,d); router
    N(0,1) (d,E); gate, up N(0,1)/√d (E·d,f); down N(0,1)/√f (E·f,d), each
    drawn in float64 and cast to float32.
    """
    gen = np.random.Generator(np.random.PCG64(seed))
    e, d, f = num_experts, hidden_dim, ffn_dim
    tokens = gen.standard_normal((batch, d)).astype(F32)
    wr = gen.standard_normal((d, e)).astype(F32)
    gate = (gen.standard_normal((e * d, f)) / np.sqrt(d)).astype(F32)
    up = (gen.standard_normal((e * d, f)) / np.sqrt(d)).astype(F32)
    down = (gen.standard_normal((e * f, d)) / np.sqrt(f)).astype(F32)
    return tokens, wr, gate, up, down


def make_router_instance(seed, batch, hidden_dim, num_experts, scaled=True, bf16_tokens=False):
    """Tokens and router weight only, for routing parity at full model shapes.

    ``scaled`` draws W_r ~ N(0,1)/√d (non-degenerate logits);
    unscaled is the reference generator's N(0,1) (saturating, tie-heavy).
    ``bf16_tokens`` rounds tokens to bfloat16 values (kept in float32), as the
    throughput configs feed the router.
    """
    gen = np.random.Generator(np.random.PCG64(seed))
    tokens = gen.standard_normal((batch, hidden_dim)).astype(F32)
    wr = gen.standard_normal((hidden_dim, num_experts))
    if scaled:
        wr = wr / np.sqrt(hidden_dim)
    wr = wr.astype(F32)
    if bf16_tokens:
        tokens = round_to_bf16(tokens)
    return tokens, wr


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even), kept as float32."""
    u = np.ascontiguousarray(a, dtype=F32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(F32).reshape(np.shape(a))
