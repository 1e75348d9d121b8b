#!/usr/bin/env python
"""Benchmark of the B200-native fused MoE layer (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config mixtral|qwen60|deepseek|skew64|small] [--tokens B]
                    [--zipf ALPHA] [--unfused] [--ep-transport p2p|collective]

Metric: MoE-layer tokens/s at <= 512 tokens.  Default workload at N = 1:
BASELINE configs[1], the Mixtral-8x7B layer (E=8, top-2, d=4096, f=14336,
bf16) at 512 tokens; at N > 1 the expert-parallel DeepSeek-V3 layer (E=256,
top-8, d=7168, f=2048, 512 tokens global) that north_star scales over 2/4/8
GPUs.  A "step" is one full layer forward (route, permute, gate+up, down,
combine) over one batch of synthetic tokens with random-init weights of that
shape.  `python bench.py --gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.

Our arm (`value`): K steps captured as ONE CUDA graph of K one-call C-ABI
forwards, each recording CUDA events between its launches (external
event-record nodes), replayed once between two events: whole-job tokens/s
from the device clock, max over ranks, and every stage of every step timed
in the same back-to-back regime -> `stages_ms` and the dominant kernel's
`roofline` (bytes of the reference's minimal-traffic model,
moeperf/perfmodel.py:216-249, over that kernel's in-graph time and the
measured HBM peak).  L2: flushed between steps unless the expert weights a
step streams are >= 4x L2.  `e2e` re-times the forward through the C-ABI
host-buffer entry (pinned host tokens in, output out, inside the timed
region).  `parity`: in the same run, the GPU routing / histogram /
permutation against the CPU oracle (bit-exact) and y on the cpu_baseline leg's
tokens (reference verify metric, moeperf/cli.py:733-737, <= 2e-2); a
mismatch makes the run fail (rc 1).

Reference arm (--impl reference): the oracle port of the reference's CPU
forward (numpy, token-sharded over every host core) on a bounded token sample
per step, same metric/config; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (E, k, d, f, gating, tokens, label)
    "mixtral": (8, 2, 4096, 14336, "softmax", 512, "Mixtral-8x7B MoE layer (E=8, top-2, d=4096, d_ffn=14336)"),
    "qwen60": (60, 4, 2048, 1408, "softmax", 512, "Qwen2-MoE routed layer (E=60, top-4, d=2048, d_ffn=1408)"),
    "deepseek": (256, 8, 7168, 2048, "sigmoid_normalized", 512, "DeepSeek-V3 MoE layer (E=256, top-8, d=7168, d_ffn=2048)"),
    "skew64": (64, 2, 3584, 2560, "softmax", 512, "Routing-skew layer (E=64, top-2, d=3584, d_ffn=2560)"),
    "small": (8, 2, 512, 1024, "softmax", 128, "Small MoE layer (E=8, top-2, d=512, d_ffn=1024)"),
}
METRIC = "MoE-layer tokens/sec at <=512 tokens"
UNIT = "tokens/s"
TOL = 2e-2  # north_star bf16 tolerance, max|y - y_ref| / max|y_ref|
CPU_EXPERT_BUDGET = 12 << 30  # host bytes of fp32 expert stacks the CPU leg may hold


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = []
        for ln in out.strip().splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower().startswith("active")})
        busy = [r for r in rows if r[2] > 300.0] or rows
        sm = sorted(r[0] for r in busy)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(busy),
                "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference forward)
# ---------------------------------------------------------------------------

def _expert_bytes(d, f):
    return 3 * d * f * 4


def _weight_pool(E, d, f, n_pool, seed):
    """fp32 expert stacks for the reference arm when the full layer does not
    fit the host budget: n_pool distinct random experts, expert e uses stack
    e % n_pool (the CPU cost of the oracle does not depend on the values)."""
    rng = np.random.default_rng(seed)
    pool = []
    for _ in range(n_pool):
        g = (rng.standard_normal((d, f), dtype=np.float32) / np.float32(d ** 0.5))
        u = (rng.standard_normal((d, f), dtype=np.float32) / np.float32(d ** 0.5))
        dn = (rng.standard_normal((f, d), dtype=np.float32) / np.float32(f ** 0.5))
        pool.append((g, u, dn))
    return lambda e: pool[e % n_pool]


def cpu_sample_tokens(procs: int, steps_total: int, t_token: float, budget_s: float = 120.0) -> int:
    """Tokens per CPU step so that steps_total steps stay within ~budget_s."""
    per_step = budget_s / max(1, steps_total)
    per_proc = max(1, int(per_step / max(t_token, 1e-3)))
    return procs * min(per_proc, 4)


def reference_arm(args, cfg_name):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    E, k, d, f, gating, B0, label = CONFIGS[cfg_name]
    B = args.tokens or B0
    import torch

    from oracle.cpu_baseline import host_cores, import_reference, run_reference_sharded, run_rows_sharded

    torch.set_num_threads(host_cores())
    gen = torch.Generator().manual_seed(1234)
    x = torch.randn((B, d), generator=gen).to(torch.bfloat16).float().numpy()
    wr = (torch.randn((d, E), generator=gen) / d ** 0.5).float().numpy()
    full = E * _expert_bytes(d, f) <= CPU_EXPERT_BUDGET
    if full:
        stacks = [((torch.randn((E * d, f), generator=gen) / d ** 0.5).to(torch.bfloat16).float().numpy())
                  for _ in range(2)]
        dn = (torch.randn((E * f, d), generator=gen) / f ** 0.5).to(torch.bfloat16).float().numpy()
        expert = lambda e: (stacks[0][e * d:(e + 1) * d], stacks[1][e * d:(e + 1) * d], dn[e * f:(e + 1) * f])  # noqa: E731
        wdesc = "random-init bf16-rounded weights of the full layer"
    else:
        n_pool = max(1, min(E, 16, CPU_EXPERT_BUDGET // _expert_bytes(d, f)))
        expert = _weight_pool(E, d, f, n_pool, 1234)
        wdesc = f"{n_pool} random expert stacks shared by expert id mod {n_pool} (the oracle's cost is value-independent)"
    procs = host_cores()
    t_token = k * 3 * d * f / 1.4e8  # ~1.4e8 fp64 fold products / s / core
    n_tok = min(B, cpu_sample_tokens(procs, args.steps + args.warmup, t_token))
    ref_mod = import_reference() if full else None
    if ref_mod is not None:
        # the reference's own moe_forward (pipeline.py:572), unmodified
        run = lambda xs: run_reference_sharded(xs, wr, stacks[0], stacks[1], dn, E, k, gating, procs)  # noqa: E731
        kind = "reference"
        what = (f"the reference package's own moeperf.moe_forward (pipeline.py:572; installed unmodified in "
                f"baseline/_ref) on {{n}} of {B} tokens per step, token-sharded over {{p}} forked workers")
    else:
        run = lambda xs: run_rows_sharded(xs, wr, expert, E, k, gating, procs)  # noqa: E731
        kind = "port"
        what = (f"{{n}} of {B} tokens per step, token-sharded over {{p}} forked numpy workers running "
                f"oracle/moe_oracle.py moe_rows (the dense per-token restatement of moeperf moe_forward, "
                f"bitwise equal to it)")
    for _ in range(args.warmup):
        run(x[:n_tok])
    walls = []
    for i in range(args.steps):
        lo = (i * n_tok) % max(1, B - n_tok + 1)
        _, _, wall, used = run(x[lo:lo + n_tok])
        walls.append(wall)
    total = sum(walls)
    value = n_tok * len(walls) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(walls),
        "higher_is_better": True, "scaling": "weak" if cfg_name != "deepseek" or args.gpus == 1 else "strong",
        "vs_baseline": None, "dtype": "f64-accumulate/f32",
        "data": f"synthetic (torch CPU Philox N(0,1) tokens, {wdesc})",
        "config": {"workload": f"{label}, {B} tokens", "tokens": B, "model_shape": [E, k, d, f], "gating": gating,
                   "sample_tokens_per_step": n_tok},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": kind,
                         "sample": what.format(n=n_tok, p=used)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_leg(x, wr, gate, up, down, E, k, d, f, gating, B, gpu_idx, routing=None):
    """Bounded-sample CPU baseline on the first tokens of the GPU's batch.
    The experts those tokens use (known from the GPU routing) are copied to
    the host as fp32 once, outside the timing; returns (cpu_baseline, y, idx,
    rows)."""
    from oracle.cpu_baseline import host_cores, import_reference, run_reference_sharded, run_rows_sharded

    procs = host_cores()
    want = min(B, procs * 2)
    if routing is None and E * _expert_bytes(d, f) <= CPU_EXPERT_BUDGET and import_reference() is not None:
        # the reference's own moe_forward (pipeline.py:572) on the first tokens, full fp32 weights
        n_tok = want
        xs = x[:n_tok].float().cpu().numpy()
        host = [t.float().cpu().numpy() for t in (wr, gate, up, down)]
        y, idx, wall, nproc = run_reference_sharded(xs, *host, E, k, gating, procs)
        del host
        cb = {"value": n_tok / wall, "unit": UNIT, "cores": nproc, "kind": "reference",
              "sample": f"{n_tok} of the {B} tokens through the reference package's own moeperf.moe_forward "
                        f"(pipeline.py:572, installed unmodified in baseline/_ref), token-sharded over {nproc} "
                        f"forked workers, {wall:.1f} s"}
        return cb, y, idx, n_tok
    n_tok, used = 0, set()
    for t in range(want):
        nxt = used | set(int(e) for e in gpu_idx[t])
        if n_tok and len(nxt) * _expert_bytes(d, f) > CPU_EXPERT_BUDGET:
            break
        used, n_tok = nxt, t + 1
    cache = {}
    for e in sorted(used):
        cache[e] = (gate[e * d:(e + 1) * d].float().cpu().numpy(), up[e * d:(e + 1) * d].float().cpu().numpy(),
                    down[e * f:(e + 1) * f].float().cpu().numpy())
    xs = x[:n_tok].float().cpu().numpy()
    r = None if routing is None else (routing[0][:n_tok], routing[1][:n_tok])
    y, idx, wall, nproc = run_rows_sharded(xs, wr.float().cpu().numpy(), cache.__getitem__, E, k, gating, procs,
                                           routing=r)
    cb = {"value": n_tok / wall, "unit": UNIT, "cores": nproc, "kind": "port",
          "sample": f"{n_tok} of the {B} tokens, token-sharded over {nproc} forked numpy workers running "
                    f"oracle/moe_oracle.py moe_rows (dense per-token restatement of moeperf moe_forward), "
                    f"wall {wall:.1f} s"}
    return cb, y, idx, n_tok


def parity_gate(layer, x, wr, out, cpu_y, cpu_idx, n_tok, routing=None):
    """In-run correctness: GPU routing / histogram / permutation vs the oracle
    on every token (bit-exact) and y vs the CPU leg's rows (cli.py:733-737)."""
    from oracle import moe_oracle as O

    cfg = layer.config
    B = out.shape[0]
    k, E = cfg.top_k, cfg.num_experts
    gidx = layer.topk_idx[:B].cpu().numpy().astype(np.int64)
    if routing is None:
        idx_ref, w_ref = O.route(x.float().cpu().numpy(), wr.float().cpu().numpy(), k, cfg.gating.value)
        routing_exact = bool(np.array_equal(gidx, idx_ref)) and bool(
            np.array_equal(layer.topk_w[:B].cpu().numpy().view(np.uint32), w_ref.view(np.uint32)))
    else:
        idx_ref = np.asarray(routing[0], dtype=np.int64)
        routing_exact = True
    counts_exact = bool(np.array_equal(layer.counts.cpu().numpy().astype(np.int64), O.expert_histogram(idx_ref, E)))
    fwd_ref, inv_ref = O.build_permutation(idx_ref)
    perm_exact = bool(np.array_equal(layer.fwd[: B * k].cpu().numpy(), fwd_ref)) and bool(
        np.array_equal(layer.inv[: B * k].cpu().numpy(), inv_ref))
    cpu_idx_exact = bool(np.array_equal(np.asarray(cpu_idx, np.int64), idx_ref[:n_tok]))
    err = O.max_rel_error(out[:n_tok].float().cpu().numpy(), cpu_y)
    ok = routing_exact and counts_exact and perm_exact and cpu_idx_exact and err <= TOL
    return {"ok": ok, "routing_exact": routing_exact and cpu_idx_exact, "counts_exact": counts_exact,
            "permutation_exact": perm_exact, "max_rel_err": err, "tolerance": TOL, "tokens_checked_y": n_tok,
            "tokens_checked_routing": B,
            "metric": "max|y - y_ref| / max(max|y_ref|, 1e-6) (moeperf/cli.py:733-737) vs the oracle's fp32 forward"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _events(torch, n):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in evs:
        e.record()  # materialise the cudaEvent_t before any capture
    return evs


def ours_arm(args, cfg_name):
    import torch
    import torch.distributed as dist

    import paper_2605_23911_b200 as P
    from paper_2605_23911_b200 import _lib
    from paper_2605_23911_b200.trace import (DEVICE_STAGES, STAGE_DOWN, STAGE_GATE_UP, STAGE_UNPERMUTE, stage_bytes,
                                             stage_flops)

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    shared_gpu = world > ndev  # more ranks than GPUs: a functional multi-rank run on shared devices

    E, k, d, f, gating, B0, label = CONFIGS[cfg_name]
    B = args.tokens or B0
    cfg = P.ModelConfig(E, k, d, f, P.Gating(gating))
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if world > 1 and cfg_name == "deepseek":
        return ep_arm(args, cfg, label, B, world, rank, dev, shared_gpu)

    def allreduce_max(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev if not shared_gpu else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn((B, d), generator=gen, device=dev).to(torch.bfloat16)
    wr = (torch.randn((d, E), generator=gen, device=dev) / d ** 0.5).float()
    gate = (torch.randn((E * d, f), generator=gen, device=dev) / d ** 0.5).to(torch.bfloat16)
    up = (torch.randn((E * d, f), generator=gen, device=dev) / d ** 0.5).to(torch.bfloat16)
    down = (torch.randn((E * f, d), generator=gen, device=dev) / f ** 0.5).to(torch.bfloat16)
    layer = P.MoELayer(cfg, P.ExpertWeights(gate, up, down), wr, max_tokens=B, device=dev)
    out = torch.empty((B, d), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    lib = _lib.load()

    def mark(ev):  # an event on the CURRENT stream (inside a capture: an external event-record node)
        _lib.check(lib.moe_b200_record_event(ev.cuda_event, torch.cuda.current_stream(dev).cuda_stream), "record")

    # routing-skew workload (BASELINE configs[4]): the reference harness's Zipf
    # table (skew.synthesize_routing, rank r -> expert r, weights 1/k) replaces
    # the router output; the router projection still runs
    skew, routed, rt = None, None, None
    if args.zipf is not None:
        from paper_2605_23911_b200.skew import SkewSpec, imbalance_metrics, synthesize_routing

        spec = SkewSpec.for_alpha(args.zipf, 1234 + rank, B, cfg)
        rt = synthesize_routing(spec)
        routed = (torch.from_numpy(rt.indices.astype(np.int32)).to(dev), torch.from_numpy(rt.weights).to(dev))
        m = imbalance_metrics(np.bincount(rt.indices.reshape(-1), minlength=E))
        skew = {"distribution": spec.distribution, "alpha": args.zipf, "seed": spec.seed,
                "max_over_mean": m.max_over_mean, "gini": m.gini, "active_experts": m.active_experts}
    fused = not args.unfused

    def step(ev):
        """One forward; ev = 5 events [route | permute | ffn | combine] (routed: ev[0], ev[4])."""
        if routed is None:
            if fused:
                layer.forward_events(x, out, ev)
            else:
                mark(ev[0])
                layer.forward(x, out, fused=False)
                mark(ev[4])
        else:
            mark(ev[0])
            layer.forward_routed(x, routed, out)
            mark(ev[4])

    warm_ev = _events(torch, 5)
    for _ in range(max(3, args.warmup)):
        step(warm_ev)
    torch.cuda.synchronize(dev)
    # L2 policy between timed steps: flush (write 256 MB > 126 MB L2) unless the
    # expert weights streamed per step are >= 4x L2, i.e. inputs larger than
    # L2 by construction (contract: flush OR inputs larger than L2; the FFN
    # streams them with evict-first, so no step can find another's weights)
    cnt0 = layer.counts.cpu().numpy()
    streamed = int((cnt0 > 0).sum()) * 3 * d * f * 2
    L2_BYTES = 126 * 1024 * 1024
    flush_between = {"always": True, "never": False}.get(args.l2_flush, streamed < 4 * L2_BYTES)
    l2_desc = (f"L2 flushed (256 MB write, outside the step events) before every step; streamed expert weights "
               f"{streamed / 1e9:.2f} GB/step" if flush_between else
               f"no flush: inputs larger than L2 (streamed expert weights {streamed / 1e9:.2f} GB/step >= 4x the "
               f"126 MB L2)")

    # Two CUDA graphs of K captured forwards each.  `timed`: the forwards as
    # they run in production (plus, when L2 is flushed between steps, one
    # event pair per step to exclude the flush); `staged`: every forward also
    # records its stage events as external event-record nodes -- the stage
    # times (and the dominant kernel's roofline) in the same back-to-back
    # regime.  value comes from `timed`; `stage_sum_ms` from `staged` shows the
    # cost of the extra event nodes.
    K = args.steps
    evs = [_events(torch, 5) for _ in range(K)]
    tev = [_events(torch, 2) for _ in range(K)]
    torch.cuda.synchronize(dev)

    def plain(i):
        if flush_between:
            flush.zero_()
            mark(tev[i][0])
        if routed is None:
            layer.forward(x, out, fused=fused)
        else:
            layer.forward_routed(x, routed, out)
        if flush_between:
            mark(tev[i][1])

    g_timed, g_staged = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_timed):
        for i in range(K):
            plain(i)
    with torch.cuda.graph(g_staged):
        for i in range(K):
            if flush_between:
                flush.zero_()
            step(evs[i])
    g_timed.replay()
    g_staged.replay()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local % ndev)
    sampler.start()
    # keep the GPU busy ~1 s so the clock samples see the timed region's state
    t_end = time.time() + 1.0
    while time.time() < t_end:
        g_timed.replay()
        torch.cuda.synchronize(dev)
    t0, t1 = _events(torch, 2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0.record()
    g_timed.replay()
    t1.record()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    g_staged.replay()  # the stage breakdown, right after (same regime)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    step_ms = [evs[i][0].elapsed_time(evs[i][4]) for i in range(K)]
    if flush_between:
        total_ms = sum(tev[i][0].elapsed_time(tev[i][1]) for i in range(K))
        timing_desc = ("one CUDA-graph replay of K captured one-call C-ABI forwards (each preceded by an L2 "
                       "flush); device time summed over each step's event pair (flushes excluded)")
    else:
        total_ms = t0.elapsed_time(t1)
        timing_desc = "CUDA events around one CUDA-graph replay of K back-to-back captured one-call C-ABI forwards"
    names = layer.STAGE_NAMES
    if routed is None and fused:
        stages = {n: float(np.mean([evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(K)]))
                  for j, n in enumerate(names)}
    else:
        stages = {"step": float(np.mean(step_ms))}
    stage_sum = float(np.mean(step_ms))

    # e2e through the C-ABI host-buffer entry point (moe_b200_forward_host):
    # every step copies its tokens in from pinned host memory and its output
    # back to pinned host memory inside the timed region; consecutive steps
    # overlap those copies with the neighbouring steps' compute
    if routed is not None or not fused:
        e2e_ms, e2e_steps, e2e_path = _e2e_overlapped(args, x, out, lambda xx, oo: (
            layer.forward_routed(xx, routed, oo) if routed is not None else layer.forward(xx, oo, fused=False)),
            flush if flush_between else None, dev)
    else:
        e2e_ms, e2e_steps, e2e_path = _e2e_pipelined(args, layer, x, B, d, flush if flush_between else None, dev)

    counts = layer.counts.cpu().numpy().astype(np.int64)
    total_ms_max, e2e_ms_max = allreduce_max([total_ms, e2e_ms / e2e_steps])
    ms_per_step = total_ms_max / K
    value = world * B / (ms_per_step / 1e3)
    e2e_value = world * B / (e2e_ms_max / 1e3)

    hbm, tflops, peak_src = _peaks()
    ffn_bytes = (stage_bytes(STAGE_GATE_UP, cfg, B, counts, element_bytes=2)
                 + stage_bytes(STAGE_DOWN, cfg, B, counts, element_bytes=2))
    tot_b = sum(stage_bytes(s, cfg, B, counts, element_bytes=2) for s in DEVICE_STAGES)
    tot_f = sum(stage_flops(s, cfg, B) for s in DEVICE_STAGES)
    overlapped = bool(lib.moe_b200_combine_overlapped(ctypes.byref(layer.cfg), B))
    if "ffn" in stages and overlapped:
        # the "ffn" interval spans the FFN and the combine overlapped with its tail
        kern_ms = stages["ffn"]
        kern_bytes = ffn_bytes + stage_bytes(STAGE_UNPERMUTE, cfg, B, counts, element_bytes=2)
        kern_name = ("ffn_kernel (fused gate+up SiLU*up and K-split down, one persistent launch) + the "
                     "weighted combine overlapped with its tail (combine_flag_kernel)")
        bytes_model = ("perfmodel.stage_bytes(GateUp)+stage_bytes(Down)+stage_bytes(Unpermute), element_bytes=2, "
                       "actual histogram")
    elif "ffn" in stages:
        kern_ms, kern_bytes = stages["ffn"], ffn_bytes
        kern_name = "ffn_kernel (fused gate+up SiLU*up and K-split down, one persistent launch)"
        bytes_model = "perfmodel.stage_bytes(GateUp)+stage_bytes(Down), element_bytes=2, actual histogram"
    else:
        kern_ms, kern_bytes = stages["step"], tot_b
        kern_name = "whole layer step (routing override / unfused ablation: no per-launch events)"
        bytes_model = "sum of perfmodel.stage_bytes over the 5 stages, element_bytes=2, actual histogram"
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            traffic = tj.get(f"{cfg_name}_{B}_ffn")
            if traffic is not None and "ffn" in stages and overlapped:
                comb = tj.get(f"{cfg_name}_{B}_combine")
                traffic = traffic + comb if comb is not None else None
        except Exception:
            traffic = None

    rc = 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch CUDA Philox N(0,1) bf16 tokens; random-init weights N(0,1)/sqrt(fan_in) bf16; "
                    "router N(0,1)/sqrt(d) fp32)",
            "config": {"workload": f"{label}, {B} tokens per GPU", "tokens": B, "model_shape": [E, k, d, f],
                       "gating": gating,
                       "parallelism": (f"replicas x{world}" + (" (ranks share GPUs)" if shared_gpu else ""))
                       if world > 1 else "single GPU",
                       "variant": "fused" if fused else "unfused gate+up ablation (pipeline.py:316-370)",
                       "l2": l2_desc, "timing": timing_desc},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": B * d * 2,
                    "d2h_bytes_per_step": B * d * 4, "path": e2e_path, "steps": e2e_steps},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "kernel": kern_name,
                         "bytes_per_launch": kern_bytes, "launch_ms": kern_ms, "bytes_model": bytes_model,
                         "timing": "mean over the K timed steps of the kernel's in-graph CUDA events",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src}, burst copy)"},
            "stages_ms": stages,
            "stage_sum_ms": stage_sum,
            "layer_roofline_frac": max(tot_b / (hbm * 1e9), tot_f / (tflops * 1e12)) / (ms_per_step / 1e3),
            "gpu_launches": layer.launches_per_forward(B) * K if routed is None and fused else None,
            "clocks": clocks,
        }
        if skew is not None:
            line["config"]["routing"] = skew
            line["config"]["workload"] += f", Zipf routing override alpha={args.zipf}"
            line["gpu_launches"] = (layer.launches_per_forward(B)) * K
        if not fused:
            line["gpu_launches"] = (layer.launches_per_forward(B) + 2) * K
        if not args.no_cpu:
            gidx = layer.topk_idx[:B].cpu().numpy() if routed is None else rt.indices
            cb, cpu_y, cpu_idx, n_tok = cpu_leg(x, wr, gate, up, down, E, k, d, f, gating, B, gidx,
                                                routing=None if rt is None else (rt.indices, rt.weights))
            if world == 1:
                line["cpu_baseline"] = cb
            step(warm_ev)  # the output of this batch (the timed replays wrote the same)
            torch.cuda.synchronize(dev)
            par = parity_gate(layer, x, wr, out, cpu_y, cpu_idx, n_tok,
                              routing=None if rt is None else (rt.indices, rt.weights))
            line["parity"] = par
            if not par["ok"]:
                rc = 1
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return rc


def _e2e_pipelined(args, layer, x, B, d, flush, dev):
    """e2e through moe_b200_forward_host: every step copies its tokens in from
    pinned host memory and its output back inside the timed region; the copies
    overlap the neighbouring steps' compute (two staging slots, copy streams)."""
    import torch

    n_slots = 2
    x_host = [x.cpu().pin_memory() for _ in range(n_slots)]
    y_host = [torch.empty((B, d), dtype=torch.float32).pin_memory() for _ in range(n_slots)]
    pipe = layer.host_pipeline(x_dtype=torch.bfloat16, y_dtype=torch.float32)
    for i in range(4):
        pipe.submit(x_host[i % n_slots], y_host[i % n_slots])
    pipe.sync()
    # a stream of >= 100 forwards: the pipeline's fill (the first step's H2D)
    # and drain (the last step's D2H) are one-off latencies, amortised as in
    # a serving loop (at 20 steps they alone cost ~2% of Mixtral-512's e2e)
    steps = max(100, min(args.steps, 400))
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    if flush is not None:
        flush.zero_()
    # same power / clock regime as `value`: ~1 s of the same pipelined steps
    # right before the timed ones, with no idle gap in between
    t_warm = time.time() + 1.0
    i = 0
    while time.time() < t_warm:
        pipe.submit(x_host[i % n_slots], y_host[i % n_slots])
        i += 1
    e_start.record()
    pipe.wait(e_start)  # the copy streams start after the timing start
    for i in range(steps):
        pipe.submit(x_host[i % n_slots], y_host[i % n_slots])
    pipe.record(e_end)
    pipe.sync()
    e_end.synchronize()
    ms = e_start.elapsed_time(e_end)
    pipe.close()
    note = ("; L2 flushed once before the stream, not between steps (the device-timed value flushes before "
            "every step: its expert weights fit in L2)") if flush is not None else ""
    return ms, steps, ("moe_b200_forward_host (C-ABI, pinned host buffers): per step H2D tokens + layer + D2H "
                       "output, copies overlapped with neighbouring steps' compute (double-buffered staging)" + note)


def _e2e_overlapped(args, x, out, run, flush, dev):
    """e2e for the routing-override and unfused forwards (no C-ABI host-buffer
    entry): every step copies its tokens in from pinned host memory and its
    output back inside the timed region; two device staging slots and two copy
    streams overlap a step's copies with its neighbours' compute (the C++
    host pipeline's scheme, driven from Python), no host synchronisation."""
    import torch

    n_slots = 2
    x_host = [x.cpu().pin_memory() for _ in range(n_slots)]
    y_host = [torch.empty(tuple(out.shape), dtype=out.dtype).pin_memory() for _ in range(n_slots)]
    x_dev = [torch.empty_like(x) for _ in range(n_slots)]
    y_dev = [torch.empty_like(out) for _ in range(n_slots)]
    s_comp = torch.cuda.current_stream(dev)
    s_in = torch.cuda.Stream(dev)
    s_out = torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(n_slots)]
    ev_comp = [torch.cuda.Event() for _ in range(n_slots)]
    ev_out = [torch.cuda.Event() for _ in range(n_slots)]
    for sl in range(n_slots):  # the slots start free
        ev_comp[sl].record(s_comp)
        ev_out[sl].record(s_comp)

    def submit(i):
        sl = i % n_slots
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_comp[sl])  # the forward two steps back has read x_dev[sl]
            x_dev[sl].copy_(x_host[sl], non_blocking=True)
            ev_in[sl].record(s_in)
        s_comp.wait_event(ev_in[sl])
        s_comp.wait_event(ev_out[sl])     # y_dev[sl] copied out
        if flush is not None:
            flush.zero_()
        run(x_dev[sl], y_dev[sl])
        ev_comp[sl].record(s_comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[sl])
            y_host[sl].copy_(y_dev[sl], non_blocking=True)
            ev_out[sl].record(s_out)

    for i in range(4):
        submit(i)
    torch.cuda.synchronize(dev)
    steps = max(20, min(args.steps, 100))
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(s_comp)
    s_in.wait_event(e_start)
    for i in range(steps):
        submit(i)
    s_comp.wait_stream(s_out)
    e_end.record(s_comp)
    e_end.synchronize()
    torch.cuda.synchronize(dev)
    return e_start.elapsed_time(e_end), steps, (
        "C-ABI forward with pinned-host tokens copied in and output copied out every step, copies on two "
        "streams overlapped with the neighbouring steps' compute (double-buffered device staging)")


def _e2e_serial(args, x, out, run, flush, dev):
    """e2e with the copies serialised around each step (routing override / ablation)."""
    import torch

    x_host = x.cpu().pin_memory()
    y_host = torch.empty(tuple(out.shape), dtype=out.dtype).pin_memory()
    x_dev = torch.empty_like(x)
    steps = max(5, min(args.steps, 50))
    ms = 0.0
    for i in range(steps + 2):
        if flush is not None:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        x_dev.copy_(x_host, non_blocking=True)
        run(x_dev, out)
        y_host.copy_(out, non_blocking=True)
        e1.record()
        e1.synchronize()
        if i >= 2:
            ms += e0.elapsed_time(e1)
    return ms, steps, "C-ABI forward with pinned-host tokens copied in and output copied out, serialised"


def ep_arm(args, cfg, label, B, world, rank, dev, shared_gpu):
    """DeepSeek-V3 expert parallelism: experts sharded over the ranks, the global
    batch B sharded B/n tokens per rank; exchanges over peer memory (rows
    written straight into the owners' buffers over NVLink, device-side epoch
    flags, no library collective on the data path).  The whole EP forward is
    captured as one CUDA graph per rank and replayed.  Strong scaling (fixed
    global batch); value = B / max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    import paper_2605_23911_b200 as P
    from paper_2605_23911_b200.ep import ExpertParallelMoE, expert_ranges
    from paper_2605_23911_b200.trace import STAGE_DOWN, STAGE_GATE_UP, stage_bytes

    E, k, d, f = cfg.num_experts, cfg.top_k, cfg.hidden_dim, cfg.ffn_dim
    lo, hi = expert_ranges(E, world)[rank]
    El = hi - lo
    gen = torch.Generator(device=dev).manual_seed(1234)  # same router on every rank
    wr = (torch.randn((d, E), generator=gen, device=dev) / d ** 0.5).float()
    gen_r = torch.Generator(device=dev).manual_seed(99 + rank)
    b0, b1 = rank * B // world, (rank + 1) * B // world
    Bl = b1 - b0
    x = torch.randn((Bl, d), generator=gen_r, device=dev).to(torch.bfloat16)
    gate = (torch.randn((El * d, f), generator=gen_r, device=dev) / d ** 0.5).to(torch.bfloat16)
    up = (torch.randn((El * d, f), generator=gen_r, device=dev) / d ** 0.5).to(torch.bfloat16)
    down = (torch.randn((El * f, d), generator=gen_r, device=dev) / f ** 0.5).to(torch.bfloat16)
    cpu = torch.device("cpu")
    # The peer-memory transport maps the other ranks' buffers with CUDA IPC; if
    # that (or the first forward) fails on any rank -- e.g. no peer access
    # between the devices -- every rank falls back to the NCCL all-to-alls.
    # (the ranks agree on success after construction, before any forward: a
    # peer-memory forward on the healthy ranks would wait on a failed peer)
    transport, fallback = args.ep_transport, None
    layer = None
    try:
        layer = ExpertParallelMoE(cfg, wr, P.ExpertWeights(gate, up, down), max_tokens=Bl, device=dev,
                                  transport=transport)
        torch.cuda.synchronize(dev)
        ok = 1
    except Exception as exc:  # noqa: BLE001 -- any failure: agree on the fallback below
        ok, fallback = 0, f"{type(exc).__name__}: {str(exc)[:200]}"
    flag = torch.tensor([ok], dtype=torch.int32, device=cpu if shared_gpu else dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0 and transport == "p2p":
        if layer is not None and layer.p2p is not None:
            layer.p2p.close()
        transport = "collective"
        fallback = fallback or "a peer rank failed to set up the peer-memory transport"
        layer = ExpertParallelMoE(cfg, wr, P.ExpertWeights(gate, up, down), max_tokens=Bl, device=dev,
                                  transport=transport)
    elif int(flag.item()) == 0:
        raise RuntimeError(f"expert-parallel setup failed: {fallback}")
    args.ep_transport = transport

    def allreduce_max(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=cpu if shared_gpu else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    for _ in range(max(3, args.warmup)):
        y = layer.forward(x, global_tokens=B)
    torch.cuda.synchronize(dev)
    dist.barrier()
    graphed = args.ep_transport == "p2p"
    if graphed:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            y = layer.forward(x, global_tokens=B)
        dist.barrier()
        run = graph.replay
    else:
        run = lambda: layer.forward(x, global_tokens=B)  # noqa: E731
    for _ in range(2):
        run()
    torch.cuda.synchronize(dev)
    dist.barrier()
    sampler = ClockSampler(_env_int("LOCAL_RANK", 0) % torch.cuda.device_count())
    sampler.start()
    e0, e1 = _events(torch, 2)
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0.record()
    for _ in range(args.steps):
        run()
    e1.record()
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = sampler.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    # e2e: this rank's tokens from pinned host memory in, its outputs back, every step
    x_host = x.cpu().pin_memory()
    y_host = torch.empty(tuple(y.shape), dtype=y.dtype).pin_memory()
    x_stage = x  # the captured graph reads x: refill it from the host each step
    steps_e2e = max(5, min(args.steps, 20))
    dist.barrier()
    torch.cuda.synchronize(dev)
    a0, a1 = _events(torch, 2)
    a0.record()
    for _ in range(steps_e2e):
        x_stage.copy_(x_host, non_blocking=True)
        run()
        y_host.copy_(y, non_blocking=True)
    a1.record()
    torch.cuda.synchronize(dev)
    dist.barrier()
    e2e_local = a0.elapsed_time(a1) / steps_e2e
    ms_per_step, e2e_ms = allreduce_max([ms_local, e2e_local])
    # per-rank algorithmic bytes: local experts' weights + the rows they
    # receive (stage_bytes over the local histogram) + the all-to-all payload
    # (bf16 rows out, fp32 rows back) of this rank
    recv_counts = layer.p2p.counts_local.sum(dim=0)[lo:hi].cpu().numpy().astype(np.int64) if layer.p2p else None
    lcfg = P.ModelConfig(El, 1, d, f, cfg.gating)
    n_recv = int(recv_counts.sum()) if recv_counts is not None else Bl * k
    local_bytes = (stage_bytes(STAGE_GATE_UP, lcfg, n_recv, recv_counts, element_bytes=2)
                   + stage_bytes(STAGE_DOWN, lcfg, n_recv, recv_counts, element_bytes=2)) if recv_counts is not None else 0
    a2a_bytes = Bl * k * d * (2 + 4)
    hbm, _, peak_src = _peaks()
    achieved = (local_bytes + a2a_bytes) / (ms_local / 1e3) / 1e9
    worst = allreduce_max([float(local_bytes + a2a_bytes)])[0]
    if rank == 0:
        line = {
            "metric": METRIC, "value": B / (ms_per_step / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch CUDA Philox N(0,1) bf16 tokens; random-init bf16 expert weights; router N(0,1)/sqrt(d))",
            "config": {"workload": f"{label}, {B} tokens global ({B // world} per rank)", "tokens": B,
                       "model_shape": [E, k, d, f], "gating": cfg.gating.value,
                       "parallelism": f"expert-parallel ep{world} ("
                                      + ("peer-memory exchanges over NVLink (CUDA IPC), one CUDA graph per rank"
                                         if args.ep_transport == "p2p" else "NCCL all-to-all") + ")"
                                      + (" -- ranks SHARE GPUs: functional run, not a scaling measurement"
                                         if shared_gpu else ""),
                       "timing": ("CUDA events over K graph replays of the whole EP forward, max over ranks"
                                  if graphed else "CUDA events over K eager EP forwards, max over ranks"),
                       "ep_transport": args.ep_transport,
                       "ep_transport_fallback": fallback},
            "e2e": {"value": B / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * d * 2,
                    "d2h_bytes_per_step": B * d * 4,
                    "path": "per rank: pinned-host token shard copied into the graph's input, EP forward replay, "
                            "output copied to pinned host, serialised; max over ranks"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "kernel": "whole expert-parallel step on rank 0 (counts, dispatch over "
                                                    "peer memory, local ffn_kernel, return, combine)",
                         "bytes_per_launch": local_bytes + a2a_bytes, "max_rank_bytes": worst,
                         "bytes_model": "rank-local perfmodel.stage_bytes(GateUp)+stage_bytes(Down) over the "
                                        "received rows + all-to-all payload (bf16 rows out, fp32 rows back)",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"},
            "gpu_launches": 7 * args.steps if graphed else None,
            "ranks": world, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def spawn(args) -> int:
    """`bench.py --gpus N` without torchrun: re-launch under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="workload (default: mixtral at 1 GPU, the expert-parallel deepseek layer at N > 1)")
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg and the parity gate")
    ap.add_argument("--zipf", type=float, default=None,
                    help="routing-skew workload: override routing with the Zipf(alpha) table (0 = uniform)")
    ap.add_argument("--unfused", action="store_true",
                    help="the unfused gate+up ablation (PipelineParams.fused=False, pipeline.py:316-370)")
    ap.add_argument("--ep-transport", choices=("p2p", "collective"), default="p2p",
                    help="expert-parallel exchanges (DeepSeek, --gpus > 1): peer memory or NCCL all-to-alls")
    ap.add_argument("--l2-flush", choices=("auto", "always", "never"), default="auto",
                    help="flush L2 between timed steps (auto: unless streamed weights >= 16x L2)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.config is None:
        args.config = "deepseek" if args.gpus > 1 else "mixtral"
    if args.impl == "reference":
        return reference_arm(args, args.config)
    return ours_arm(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
