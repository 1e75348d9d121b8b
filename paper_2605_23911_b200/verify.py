"""GPU-backed ``verify`` (the reference's ``moeperf verify``, ``cli.py:715-881``,
with the sm_100a layer as the system under test).

    python -m paper_2605_23911_b200 verify [--model Mixtral8x7B | --experts E --top-k K
        --hidden-dim D --ffn-dim F [--gating softmax|sigmoid_normalized]]
        [--batch 16] [--trials 5] [--tol 2e-2] [--seed 0] [--format md|json] [--out PATH]
        [--full-dims]

Each trial mirrors ``run_verify_trial`` (``cli.py:755-793``): one PCG64(seed)
stream draws the tokens, the unscaled router weight and
``ExpertWeights.random`` with the REFERENCE's own generators, at
``shrink_config`` dimensions (``cli.py:720-730``) unless ``--full-dims``.  The
checker is the reference package itself (``moeperf``, importable from
PYTHONPATH or the offline install in ``baseline/_ref``):

* routing (indices, weights, expert counts, forward permutation) bit-exact
  against ``route`` / ``expert_histogram`` / ``build_permutation``;
* the GPU output within ``--tol`` (max relative error, ``cli.py:733-737``) of
  ``dense_moe_oracle`` — bf16 tolerance (north_star), 2e-2 by default;
* the fused and the unfused (``PipelineParams.fused=False``) GPU forwards
  bitwise equal, like the reference's own fused == unfused invariant;
* the returned trace equal to the reference's ``trace_from_counts``.

Exit codes follow the reference CLI (``cli.py:979-992``): 0 pass, 1 mismatch,
2 usage / environment error (including "reference not importable").
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import dataclass

import numpy as np

from .errors import MoeperfError

_REF_PATHS = (os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref"),)


def _import_reference():
    try:
        import moeperf  # noqa: F401
    except ImportError:
        for p in _REF_PATHS:
            if os.path.isdir(p) and p not in sys.path:
                sys.path.append(p)
        try:
            import moeperf  # noqa: F401
        except ImportError as exc:
            raise RuntimeError("reference package moeperf not importable (PYTHONPATH or baseline/_ref)") from exc
    import moeperf
    return moeperf


@dataclass
class GpuTrial:
    index: int
    seed: int
    blocks: tuple
    routing_exact: bool
    permutation_exact: bool
    max_rel_error: float
    bitwise_fused_unfused: bool
    trace_match: bool

    def ok(self, tol: float) -> bool:
        return (self.routing_exact and self.permutation_exact and self.bitwise_fused_unfused
                and self.trace_match and self.max_rel_error <= tol)


def _records(trace):
    return [(r.stage, r.tiles, r.flops, dict(r.reads), dict(r.writes)) for r in trace.records]


def run_gpu_trial(ref, config_ref, batch: int, seed: int, blocks, index: int) -> GpuTrial:
    from . import layer as L
    from .types import ExpertWeights, Gating, ModelConfig, PipelineParams

    rng = np.random.Generator(np.random.PCG64(seed))
    tokens = rng.standard_normal((batch, config_ref.hidden_dim)).astype(np.float32)
    router_w = rng.standard_normal((config_ref.hidden_dim, config_ref.num_experts)).astype(np.float32)
    w_ref = ref.ExpertWeights.random(config_ref, rng)
    cfg = ModelConfig(config_ref.num_experts, config_ref.top_k, config_ref.hidden_dim, config_ref.ffn_dim,
                      Gating(config_ref.gating.value), config_ref.element_bytes)
    weights = ExpertWeights(np.asarray(w_ref.gate), np.asarray(w_ref.up), np.asarray(w_ref.down))
    bm, bn, bk = blocks
    y_f, trace_f = L.moe_forward(tokens, router_w, weights, cfg, PipelineParams(bm, bn, bk, True))
    lay = L._layer_for(weights, cfg, router_w, batch)
    idx_gpu = lay.topk_idx[:batch].cpu().numpy().astype(np.int64)
    w_gpu = lay.topk_w[:batch].cpu().numpy()
    counts_gpu = lay.counts.cpu().numpy().astype(np.int64)
    fwd_gpu = lay.fwd[: batch * cfg.top_k].cpu().numpy().astype(np.int64)
    y_u, trace_u = L.moe_forward(tokens, router_w, weights, cfg, PipelineParams(bm, bn, bk, False))

    from moeperf.pipeline import dense_moe_oracle, trace_from_counts
    from moeperf.router import route
    from moeperf.scheduler import build_permutation, expert_histogram

    r = route(tokens, router_w, config_ref)
    counts = expert_histogram(r, config_ref.num_experts)
    perm = build_permutation(r)
    oracle = dense_moe_oracle(tokens, router_w, w_ref, config_ref)
    routing_exact = (np.array_equal(idx_gpu, r.indices) and
                     np.array_equal(w_gpu.view(np.uint32), np.asarray(r.weights, np.float32).view(np.uint32)))
    perm_exact = np.array_equal(counts_gpu, counts) and np.array_equal(fwd_gpu, perm.forward)
    ref_params = ref.PipelineParams(block_m=bm, block_n=bn, block_k=bk, fused=True)
    ref_params_u = ref.PipelineParams(block_m=bm, block_n=bn, block_k=bk, fused=False)
    trace_match = (_records(trace_f) == _records(trace_from_counts(config_ref, batch, counts, ref_params)) and
                   _records(trace_u) == _records(trace_from_counts(config_ref, batch, counts, ref_params_u)))
    scale = max(float(np.abs(oracle).max()), 1e-6) if oracle.size else 1.0
    err = float(np.abs(y_f.astype(np.float64) - oracle.astype(np.float64)).max() / scale) if oracle.size else 0.0
    return GpuTrial(index, seed, tuple(blocks), bool(routing_exact), bool(perm_exact), err,
                    bool(np.array_equal(y_f.view(np.uint32), y_u.view(np.uint32))), bool(trace_match))


def _config_from_args(ref, args):
    custom = (args.experts, args.top_k, args.hidden_dim, args.ffn_dim)
    if any(v is not None for v in custom):
        if any(v is None for v in custom):
            raise ValueError("custom model needs --experts/--top-k/--hidden-dim/--ffn-dim")
        return "custom", ref.ModelConfig(args.experts, args.top_k, args.hidden_dim, args.ffn_dim,
                                         ref.Gating(args.gating or "softmax"))
    name = args.model or "Mixtral8x7B"
    return name, ref.preset(name)


def cmd_verify(args) -> int:
    ref = _import_reference()
    from moeperf.cli import shrink_config

    name, full = _config_from_args(ref, args)
    if args.batch < 1 or args.trials < 1 or not args.tol > 0:
        raise ValueError("batch and trials must be >= 1, tolerance > 0")
    config = full if args.full_dims else shrink_config(full)
    expanded = args.batch * config.top_k
    block_cycle = [(3, 4, 5), (5, 3, 2), (2, 7, 3), (max(expanded, 1), 8, 8), (1, 2, 1)]
    trials = [run_gpu_trial(ref, config, args.batch, args.seed + t, block_cycle[t % len(block_cycle)], t)
              for t in range(args.trials)]
    max_err = max(t.max_rel_error for t in trials)
    passed = all(t.ok(args.tol) for t in trials)
    if args.format == "json":
        text = json.dumps({
            "model": name, "device": "B200 (sm_100a)", "checker": "moeperf (reference)",
            "dims": {"num_experts": config.num_experts, "top_k": config.top_k, "hidden_dim": config.hidden_dim,
                     "ffn_dim": config.ffn_dim, "gating": config.gating.value},
            "batch": args.batch, "tolerance": args.tol, "max_rel_error": max_err,
            "trials": [t.__dict__ | {"blocks": list(t.blocks)} for t in trials],
            "status": "pass" if passed else "fail"}, indent=2, sort_keys=True) + "\n"
    else:
        lines = [f"# GPU pipeline verification: {name} ({'full' if args.full_dims else 'reduced'} dims)", "",
                 f"- dims: E={config.num_experts} k={config.top_k} d={config.hidden_dim} f={config.ffn_dim} "
                 f"({config.gating.value}), batch {args.batch}, device B200 sm_100a, checker: reference moeperf",
                 f"- tolerance: {args.tol:g} (max relative error vs dense_moe_oracle)", "",
                 "| trial | seed | blocks | routing exact | permutation exact | max rel err | fused==unfused | trace |",
                 "|---|---|---|---|---|---|---|---|"]
        yes = lambda b: "yes" if b else "NO"  # noqa: E731
        for t in trials:
            lines.append(f"| {t.index} | {t.seed} | {t.blocks} | {yes(t.routing_exact)} | {yes(t.permutation_exact)} "
                         f"| {t.max_rel_error:.3e} | {yes(t.bitwise_fused_unfused)} | {yes(t.trace_match)} |")
        n_ok = sum(t.ok(args.tol) for t in trials)
        lines += ["", f"result: {'PASS' if passed else 'FAIL'} ({n_ok}/{len(trials)} trials, "
                      f"max rel err {max_err:.3e})", ""]
        text = "\n".join(lines)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0 if passed else 1


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2605_23911_b200", description="B200 MoE layer tools")
    sub = ap.add_subparsers(dest="command", required=True)
    v = sub.add_parser("verify", help="check the GPU layer against the reference (moeperf)")
    v.add_argument("--model")
    v.add_argument("--experts", type=int)
    v.add_argument("--top-k", dest="top_k", type=int)
    v.add_argument("--hidden-dim", dest="hidden_dim", type=int)
    v.add_argument("--ffn-dim", dest="ffn_dim", type=int)
    v.add_argument("--gating", choices=("softmax", "sigmoid_normalized"))
    v.add_argument("--batch", type=int, default=16)
    v.add_argument("--trials", type=int, default=5)
    v.add_argument("--tol", type=float, default=2e-2)
    v.add_argument("--seed", type=int, default=0)
    v.add_argument("--format", choices=("md", "json"), default="md")
    v.add_argument("--out")
    v.add_argument("--full-dims", dest="full_dims", action="store_true")
    v.set_defaults(func=cmd_verify)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except (MoeperfError, ValueError, KeyError, OSError, RuntimeError) as exc:
        msg = exc.args[0] if isinstance(exc, KeyError) and exc.args else exc
        print(f"error: {msg}", file=sys.stderr)
        return 2
