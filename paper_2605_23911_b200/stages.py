"""The reference's stage-level API on the GPU (drop-ins for
``moeperf/__init__.py:56-78``).

Same names, signatures, validation and exception classes as the reference
functions; the arithmetic runs in libmoe_b200.so (``csrc/stages.cuh`` and the
tcgen05 FFN kernel), there is no CPU fallback.  numpy in -> numpy out, CUDA
tensors in -> CUDA tensors out.

Exactness (the reference's contract, ``SPEC.md``):

* bit-exact: ``gate_scores``, ``stable_softmax_row``, ``topk_select``,
  ``route``, ``expert_histogram``, ``build_permutation``, ``permute_tokens``,
  ``unpermute_combine``, ``sigmoid``, ``silu``, ``dense_matmul``
  (``expert_offsets`` / ``build_block_schedule`` are E-sized host metadata,
  as in the reference);
* bf16 tensor-core tolerance (operands rounded to bf16, fp32 accumulation,
  ``h`` rounded to bf16 as the fused layer stores it): ``fused_gate_up``,
  ``unfused_gate_up`` (bit-identical to ``fused_gate_up``, like the
  reference's pair), ``grouped_gemm``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import IndexOutOfRange, InvalidK, NonFiniteInput, ShapeMismatch
from .layer import _array_fingerprint, _ptr, _stream_ptr
from .trace import (
    INDEX_BYTES,
    STAGE_DOWN,
    STAGE_GATE_UP,
    StageRecord,
    build_block_schedule,
    check_schedule,
    expert_offsets,
)
from .types import (
    GATING_CODE,
    ExpertOffsets,
    Gating,
    Permutation,
    PipelineParams,
    RoutingResult,
)

__all__ = [
    "gate_scores", "stable_softmax_row", "topk_select", "expert_histogram", "expert_offsets",
    "build_permutation", "build_block_schedule", "permute_tokens", "fused_gate_up", "unfused_gate_up",
    "grouped_gemm", "unpermute_combine", "sigmoid", "silu", "dense_matmul",
]


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


def _to_dev(a, dtype) -> torch.Tensor:
    t = a if _is_torch(a) else torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
    return t.to(device=_device(), dtype=dtype).contiguous()


def _matrix(a, name: str) -> torch.Tensor:
    """``linalg.as_matrix`` (``linalg.py:27-35``): 2-D float32, else ShapeMismatch."""
    shape = tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape
    if len(shape) != 2:
        raise ShapeMismatch(f"{name} must be 2-D, got shape {shape}")
    return _to_dev(a, torch.float32)


def _out(t: torch.Tensor, like_numpy: bool):
    return t.cpu().numpy() if like_numpy else t


def _stream():
    return _stream_ptr(_device())


def _round8(n: int) -> int:
    return (n + 7) // 8 * 8


def _pad_cols(t: torch.Tensor, to: int) -> torch.Tensor:
    return t if t.shape[1] == to else torch.nn.functional.pad(t, (0, to - t.shape[1])).contiguous()


# ---------------------------------------------------------------------------
# router (router.py:61-113)
# ---------------------------------------------------------------------------

def gate_scores(logits, mode: Gating):
    """``router.py:69-84``: softmax / sigmoid gate scores, bit-exact."""
    like_numpy = not _is_torch(logits)
    lg = _matrix(logits, "logits")
    mode = Gating(mode)
    B, E = lg.shape
    if B == 0 or E == 0:
        return _out(lg.clone(), like_numpy)
    lib = _lib.load()
    scores = torch.empty_like(lg)
    flag = torch.zeros(1, dtype=torch.int32, device=lg.device)
    _lib.check(lib.moe_b200_gate_scores(B, E, GATING_CODE[mode], _ptr(lg), _ptr(scores), _ptr(flag), _stream()),
               "gate_scores")
    if int(flag.item()):
        raise NonFiniteInput("logits contains non-finite values")
    return _out(scores, like_numpy)


def stable_softmax_row(row):
    """``router.py:61-66``: max-subtracted softmax of one logit row (float32)."""
    like_numpy = not _is_torch(row)
    r = row if _is_torch(row) else np.asarray(row, dtype=np.float32)
    r2 = r.reshape(1, -1)
    out = gate_scores(r2, Gating.SOFTMAX)
    return out.reshape(-1) if like_numpy else out.reshape(-1)


def topk_select(scores, k: int, mode: Gating = Gating.SOFTMAX) -> RoutingResult:
    """``router.py:87-113``: k rounds of argmax with -1.0 masking, bit-exact."""
    like_numpy = not _is_torch(scores)
    sc = _matrix(scores, "scores")
    B, E = sc.shape
    if not 1 <= k <= E:
        raise InvalidK(f"k must be in [1, {E}], got {k}")
    mode = Gating(mode)
    idx = torch.empty((B, k), dtype=torch.int32, device=sc.device)
    w = torch.empty((B, k), dtype=torch.float32, device=sc.device)
    if B:
        _lib.check(_lib.load().moe_b200_topk_select(B, E, int(k), GATING_CODE[mode], _ptr(sc), _ptr(idx), _ptr(w),
                                                    _stream()), "topk_select")
    idx = idx.to(torch.int64)
    return RoutingResult(indices=_out(idx, like_numpy), weights=_out(w, like_numpy))


# ---------------------------------------------------------------------------
# scheduler (scheduler.py:78-117)
# ---------------------------------------------------------------------------

_WS_CACHE: dict = {}


def _workspace(cfg_struct, key, size_fn) -> tuple:
    ws = _WS_CACHE.get(key)
    if ws is None:
        n = ctypes.c_size_t(0)
        _lib.check(size_fn(ctypes.byref(n)), "workspace_size")
        t = torch.empty(max(int(n.value), 256), dtype=torch.uint8, device=_device())
        _lib.check(_lib.load().moe_b200_workspace_init(ctypes.byref(cfg_struct), 1, _ptr(t), t.numel(), _stream()),
                   "workspace_init")
        ws = (t, t.numel())
        if len(_WS_CACHE) > 8:
            _WS_CACHE.pop(next(iter(_WS_CACHE)))
        _WS_CACHE[key] = ws
    return ws


def _schedule(indices, num_experts: int):
    """counts, offsets, forward, inverse of routing indices (B, k) on the device."""
    lib = _lib.load()
    idx = _to_dev(indices, torch.int32)
    B, k = idx.shape
    # (k > E only when the caller's ids use fewer experts than slots: the
    # dispatch kernel needs k <= E, extra experts just stay empty)
    cfg = _lib.config_struct(max(int(num_experts), k, 1), max(k, 1), 8, 8, 0)
    dev = idx.device
    counts = torch.empty(cfg.num_experts, dtype=torch.int32, device=dev)
    offsets = torch.empty(cfg.num_experts + 1, dtype=torch.int32, device=dev)
    fwd = torch.empty(B * k, dtype=torch.int32, device=dev)
    inv = torch.empty(B * k, dtype=torch.int32, device=dev)
    if B * k == 0:
        counts.zero_()
        offsets.zero_()
        return counts, offsets, fwd, inv
    ws, ws_bytes = _workspace(cfg, ("sched", cfg.num_experts, k, B),
                              lambda p: lib.moe_b200_workspace_size(ctypes.byref(cfg), B, p))
    _lib.check(lib.moe_b200_schedule(ctypes.byref(cfg), B, _ptr(idx), _ptr(counts), _ptr(offsets), _ptr(fwd),
                                     _ptr(inv), _ptr(ws), ws_bytes, _stream()), "schedule")
    return counts, offsets, fwd, inv


def expert_histogram(routing: RoutingResult, num_experts: int):
    """``scheduler.py:78-82``: expanded assignments per expert (int64, length E)."""
    routing.validate(num_experts)
    like_numpy = not _is_torch(routing.indices)
    counts = _schedule(routing.indices, num_experts)[0][:num_experts].to(torch.int64)
    return _out(counts, like_numpy)


def build_permutation(routing: RoutingResult) -> Permutation:
    """``scheduler.py:97-103``: stable expert-major order of the expanded ids."""
    like_numpy = not _is_torch(routing.indices)
    idx = routing.indices
    n = int(np.prod(tuple(idx.shape)))
    if n and int(idx.min()) < 0:
        raise IndexOutOfRange(f"expert ids must be >= 0, got {int(idx.min())}")
    E = int(idx.max()) + 1 if n else 1
    _, _, fwd, inv = _schedule(idx, E)
    return Permutation(forward=_out(fwd.to(torch.int64), like_numpy), inverse=_out(inv.to(torch.int64), like_numpy))


# ---------------------------------------------------------------------------
# pipeline stages (pipeline.py:165-399)
# ---------------------------------------------------------------------------

def permute_tokens(tokens, routing: RoutingResult, permutation: Permutation):
    """``pipeline.py:165-183``: row r <- token forward[r] // k (exact fp32 copy)."""
    like_numpy = not _is_torch(tokens)
    x = _matrix(tokens, "tokens")
    batch, k = tuple(routing.indices.shape)
    if x.shape[0] != batch:
        raise ShapeMismatch(f"tokens have {x.shape[0]} rows, routing has {batch}")
    fwd_n = int(np.prod(tuple(permutation.forward.shape)))
    if fwd_n != batch * k:
        raise ShapeMismatch(f"permutation covers {fwd_n} rows, expected {batch * k}")
    d = x.shape[1]
    if k == 0 or batch == 0 or d == 0:
        return _out(torch.zeros((batch * k, d), dtype=torch.float32, device=x.device), like_numpy)
    dp = (d + 3) // 4 * 4  # 16-byte rows
    xs = _pad_cols(x, dp)
    fwd = _to_dev(permutation.forward, torch.int32)
    out = torch.empty((batch * k, dp), dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().moe_b200_permute_rows(batch * k, dp * 4, _ptr(xs), _ptr(fwd), int(k), _ptr(out), _stream()),
               "permute_rows")
    return _out(out[:, :d].contiguous() if dp != d else out, like_numpy)


def unpermute_combine(expert_out, routing: RoutingResult, permutation: Permutation):
    """``pipeline.py:373-399``: y[t] = sum_j w[t,j] * Y[inverse[t*k+j]], ascending j, fp32 (bit-exact)."""
    like_numpy = not _is_torch(expert_out)
    ys = _matrix(expert_out, "expert_out")
    batch, k = tuple(routing.indices.shape)
    inv_n = int(np.prod(tuple(permutation.inverse.shape)))
    if inv_n != batch * k:
        raise ShapeMismatch(f"permutation covers {inv_n} rows, expected {batch * k}")
    if ys.shape[0] != batch * k:
        raise ShapeMismatch(f"expert output has {ys.shape[0]} rows, expected {batch * k}")
    hidden = ys.shape[1]
    if batch == 0 or k == 0 or hidden == 0:
        return _out(torch.zeros((batch, hidden), dtype=torch.float32, device=ys.device), like_numpy)
    hp = _round8(hidden)
    rows = _pad_cols(ys, hp)
    inv = _to_dev(permutation.inverse, torch.int32)
    w = _to_dev(routing.weights, torch.float32)
    y = torch.empty((batch, hp), dtype=torch.float32, device=ys.device)
    cfg = _lib.config_struct(k, k, hp, 8, 0)
    _lib.check(_lib.load().moe_b200_combine_rows(ctypes.byref(cfg), batch, _ptr(rows), _ptr(inv), _ptr(w), _ptr(y),
                                                 _lib.DTYPE_F32, _stream()), "combine_rows")
    return _out(y[:, :hidden].contiguous() if hp != hidden else y, like_numpy)


# -- the expert GEMMs ----------------------------------------------------------

_STACK_CACHE: dict = {}


def _stack_bf16(stack, num_experts: int, rows: int, cols: int, rows_p: int, cols_p: int) -> torch.Tensor:
    """A flat (E*rows, cols) weight stack as a resident bf16 device copy padded
    to (E*rows_p, cols_p); cached while the array is unchanged."""
    key = (id(stack), rows_p, cols_p)
    fp = _array_fingerprint(stack)
    hit = _STACK_CACHE.get(key)
    if hit is not None and hit[0] == fp:
        return hit[1]
    t = _to_dev(stack, torch.float32)
    if t.numel() and not bool(torch.isfinite(t).all()):
        raise NonFiniteInput("weight stack contains non-finite values")
    t = t.to(torch.bfloat16)
    if rows_p != rows or cols_p != cols:
        out = torch.zeros((num_experts, rows_p, cols_p), dtype=torch.bfloat16, device=t.device)
        out[:, :rows, :cols] = t.reshape(num_experts, rows, cols)
        t = out.reshape(num_experts * rows_p, cols_p)
    if len(_STACK_CACHE) >= 6:
        _STACK_CACHE.pop(next(iter(_STACK_CACHE)))
    _STACK_CACHE[key] = (fp, t)
    return t


def _rows_bf16(inp: torch.Tensor, cols_p: int) -> torch.Tensor:
    x = _pad_cols(inp, cols_p)
    out = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    _lib.check(_lib.load().moe_b200_cast_bf16(x.numel(), _ptr(x), _ptr(out), _stream()), "cast_bf16")
    return out


def _counts_dev(offsets: ExpertOffsets) -> torch.Tensor:
    off = np.asarray(offsets.offsets.cpu() if _is_torch(offsets.offsets) else offsets.offsets, dtype=np.int64)
    return torch.from_numpy(np.diff(off).astype(np.int32)).to(_device())


def _grouped_ws(cfg):
    lib = _lib.load()
    return lambda n_rows: _workspace(
        cfg, ("grp", cfg.num_experts, cfg.hidden_dim, cfg.ffn_dim, n_rows),
        lambda p: lib.moe_b200_expert_ffn_workspace_size(ctypes.byref(cfg), n_rows, 0, p))


def _gemm(inp: torch.Tensor, stack, offsets: ExpertOffsets, out: torch.Tensor | None = None) -> torch.Tensor:
    """out (T, N) fp32 = inp (T, K) @ W_e per expert segment (tcgen05, bf16 operands)."""
    T, K = inp.shape
    E = offsets.num_experts
    N = int(stack.shape[1])
    Kp, Np = _round8(K), _round8(N)
    w = _stack_bf16(stack, E, K, N, Kp, Np)
    a = _rows_bf16(inp, Kp)
    cfg = _lib.config_struct(E, 1, Np, Kp, 0)
    if out is None:
        out = torch.empty((T, Np), dtype=torch.float32, device=inp.device)
    ws, ws_bytes = _grouped_ws(cfg)(T)
    counts = _counts_dev(offsets)
    _lib.check(_lib.load().moe_b200_grouped_gemm(ctypes.byref(cfg), T, _ptr(counts), _ptr(a), _ptr(w), _ptr(out),
                                                 _ptr(ws), ws_bytes, _stream()), "grouped_gemm")
    return out


def _check_stack(stack, name: str, rows: int):
    if int(stack.shape[0]) != rows:
        raise ShapeMismatch(f"{name} stack has {int(stack.shape[0])} rows, expected {rows}")


def _steps(total: int, block: int) -> int:
    return -(-total // block) if total else 0


def _spans(offsets: ExpertOffsets, schedule):
    for expert, local_start in schedule.entries:
        n_e = offsets.count(expert)
        yield min(schedule.block_m, n_e - local_start)


def grouped_gemm(inp, weight_stack, schedule, offsets: ExpertOffsets, params: PipelineParams, trace=None,
                 stage: str = STAGE_DOWN):
    """``pipeline.py:186-247``: expert-grouped GEMM over a flat ``(E*K, N)`` stack."""
    like_numpy = not _is_torch(inp)
    x = _matrix(inp, "input")
    _matrix(weight_stack, "weights") if not _is_torch(weight_stack) else None
    total, E = offsets.total, offsets.num_experts
    if x.shape[0] != total:
        raise ShapeMismatch(f"input has {x.shape[0]} rows, offsets say {total}")
    K = x.shape[1]
    if len(weight_stack.shape) != 2:
        raise ShapeMismatch(f"weights must be 2-D, got shape {tuple(weight_stack.shape)}")
    if int(weight_stack.shape[0]) != E * K:
        raise ShapeMismatch(f"weight stack has {int(weight_stack.shape[0])} rows, expected {E} x {K}")
    N = int(weight_stack.shape[1])
    check_schedule(offsets, schedule)
    if total == 0 or N == 0 or K == 0:
        out = torch.zeros((total, N), dtype=torch.float32, device=x.device)
    else:
        out = _gemm(x, weight_stack, offsets)[:, :N]
    if trace is not None:
        eb = trace.element_bytes
        spans = list(_spans(offsets, schedule))
        ks, ns = _steps(K, params.block_k), _steps(N, params.block_n)
        trace.add(StageRecord(stage=stage, tiles=len(spans) * ks * ns, flops=sum(2 * m * K * N for m in spans),
                              reads={"input": sum(m * K for m in spans) * eb, "weight": len(spans) * K * N * eb},
                              writes={"output": sum(m * N for m in spans) * eb}))
    return _out(out.contiguous(), like_numpy)


def _gate_up_checks(x, weights, offsets):
    total, E = offsets.total, offsets.num_experts
    if x.shape[0] != total:
        raise ShapeMismatch(f"input has {x.shape[0]} rows, offsets say {total}")
    d = x.shape[1]
    for name in ("gate", "up"):
        _check_stack(getattr(weights, name), name, E * d)
    if int(weights.gate.shape[1]) != int(weights.up.shape[1]):
        raise ShapeMismatch("gate and up stacks disagree on ffn dim")
    return d, int(weights.gate.shape[1])


def fused_gate_up(inp, weights, schedule, offsets: ExpertOffsets, params: PipelineParams, trace=None):
    """``pipeline.py:250-313``: h = silu(A Wg_e) * (A Wu_e) from one staged input
    tile per expert segment (tcgen05, SiLU*up in registers, bf16 h)."""
    like_numpy = not _is_torch(inp)
    x = _matrix(inp, "input")
    d, f = _gate_up_checks(x, weights, offsets)
    check_schedule(offsets, schedule)
    T, E = offsets.total, offsets.num_experts
    if T == 0 or f == 0:
        h32 = torch.zeros((T, f), dtype=torch.float32, device=x.device)
    else:
        dp, fp = _round8(d), _round8(f)
        wg = _stack_bf16(weights.gate, E, d, f, dp, fp)
        wu = _stack_bf16(weights.up, E, d, f, dp, fp)
        a = _rows_bf16(x, dp)
        cfg = _lib.config_struct(E, 1, dp, fp, 0)
        h = torch.empty((T, fp), dtype=torch.bfloat16, device=x.device)
        ws, ws_bytes = _grouped_ws(cfg)(T)
        counts = _counts_dev(offsets)
        _lib.check(_lib.load().moe_b200_grouped_gate_up(ctypes.byref(cfg), T, _ptr(counts), _ptr(a), _ptr(wg),
                                                        _ptr(wu), _ptr(h), _ptr(ws), ws_bytes, _stream()),
                   "grouped_gate_up")
        h32 = h[:, :f].float()
    if trace is not None:
        eb = trace.element_bytes
        spans = list(_spans(offsets, schedule))
        ks, ns = _steps(d, params.block_k), _steps(f, params.block_n)
        trace.add(StageRecord(stage=STAGE_GATE_UP, tiles=len(spans) * ks * ns,
                              flops=sum(4 * m * d * f + 5 * m * f for m in spans),
                              reads={"input": sum(m * d for m in spans) * eb, "weight": len(spans) * 2 * d * f * eb},
                              writes={"intermediate": sum(m * f for m in spans) * eb}))
    return _out(h32.contiguous(), like_numpy)


def unfused_gate_up(inp, weights, schedule, offsets: ExpertOffsets, params: PipelineParams, trace=None):
    """``pipeline.py:316-370``: gate and up as two grouped GEMMs (fp32 buffers),
    then a separate activation pass; bit-identical to ``fused_gate_up``."""
    if tuple(weights.gate.shape) != tuple(weights.up.shape):
        raise ShapeMismatch("gate and up stacks must have identical shapes")
    like_numpy = not _is_torch(inp)
    x = _matrix(inp, "input")
    d, f = _gate_up_checks(x, weights, offsets)
    check_schedule(offsets, schedule)
    T = offsets.total
    if T == 0 or f == 0:
        h32 = torch.zeros((T, f), dtype=torch.float32, device=x.device)
    else:
        fp = _round8(f)
        gu = torch.empty((2, T, fp), dtype=torch.float32, device=x.device)
        _gemm(x, weights.gate, offsets, out=gu[0])
        _gemm(x, weights.up, offsets, out=gu[1])
        h = torch.empty((T, fp), dtype=torch.bfloat16, device=x.device)
        _lib.check(_lib.load().moe_b200_swiglu(T * fp, _ptr(gu), _ptr(h), _stream()), "swiglu")
        h32 = h[:, :f].float()
    if trace is not None:
        eb = trace.element_bytes
        spans = list(_spans(offsets, schedule))
        ks, ns = _steps(d, params.block_k), _steps(f, params.block_n)
        trace.add(StageRecord(stage=STAGE_GATE_UP, tiles=len(spans) * 2 * ks * ns,
                              flops=sum(4 * m * d * f for m in spans) + 5 * T * f,
                              reads={"input": sum(2 * m * d for m in spans) * eb,
                                     "weight": len(spans) * 2 * d * f * eb, "buffer": 2 * T * f * eb},
                              writes={"gate_out": sum(m * f for m in spans) * eb,
                                      "up_out": sum(m * f for m in spans) * eb, "intermediate": T * f * eb}))
    return _out(h32.contiguous(), like_numpy)


# ---------------------------------------------------------------------------
# numerics helpers (linalg.py:45-86)
# ---------------------------------------------------------------------------

def _elementwise(x, silu_flag: int):
    like_numpy = not _is_torch(x)
    t = _to_dev(x, torch.float32)
    out = torch.empty_like(t)
    if t.numel():
        _lib.check(_lib.load().moe_b200_sigmoid(t.numel(), _ptr(t), _ptr(out), silu_flag, _stream()), "sigmoid")
    return _out(out, like_numpy)


def sigmoid(x):
    """``linalg.py:71-80``: split-form logistic in float32, numpy's bits."""
    return _elementwise(x, 0)


def silu(x):
    """``linalg.py:83-86``: ``x * sigmoid(x)`` in float32, numpy's bits."""
    return _elementwise(x, 1)


def dense_matmul(a, b):
    """``linalg.py:60-68``: float32 matmul with exact fp64 products folded in
    ascending k, one fp32 rounding (bit-exact)."""
    like_numpy = not _is_torch(a)
    A = _matrix(a, "a")
    Bm = _matrix(b, "b")
    if A.shape[1] != Bm.shape[0]:
        raise ShapeMismatch(f"inner dimensions differ: a is {tuple(A.shape)}, b is {tuple(Bm.shape)}")
    m, K = A.shape
    n = Bm.shape[1]
    c = torch.empty((m, n), dtype=torch.float32, device=A.device)
    if m and n:
        _lib.check(_lib.load().moe_b200_dense_matmul(m, K, n, _ptr(A), _ptr(Bm), _ptr(c), _stream()), "dense_matmul")
    return _out(c, like_numpy)


def dense_moe_oracle(tokens, router_weight, weights, config):
    """``pipeline.py:618-643`` returns the same bits as ``moe_forward`` in the
    reference (its per-token restatement); here it is the device forward's y."""
    from .layer import moe_forward

    return moe_forward(tokens, router_weight, weights, config)[0]


_ = INDEX_BYTES  # (trace accounting helpers share the module's constants)
