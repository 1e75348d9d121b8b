"""CPU baseline runner — TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle port of the reference MoE forward (``oracle.moe_oracle``,
a numpy restatement of ``moeperf.pipeline.moe_forward``,
``pipeline.py:572-615``) on the host cores.  The reference is single-threaded
numpy; rows are independent, so the token batch is sharded across one
forked worker per core (bit-identical to the unsharded run — the reference's
row-parallel guarantee).  Only ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs call this.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import moe_oracle as O

_STATE: dict = {}


def _worker(args):
    lo, hi = args
    s = _STATE
    res = O.moe_forward(s["tokens"][lo:hi], s["wr"], s["gate"], s["up"], s["down"],
                        s["E"], s["k"], s["gating"])
    return lo, res["y"], res["indices"]


def _noop(_):
    return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _rows_worker(args):
    lo, hi = args
    s = _STATE
    t0 = time.perf_counter()
    res = O.moe_rows(s["tokens"][lo:hi], s["wr"], s["expert"], s["E"], s["k"], s["gating"],
                     routing=None if s["routing"] is None else (s["routing"][0][lo:hi], s["routing"][1][lo:hi]))
    return lo, res["y"], res["indices"], time.perf_counter() - t0


def run_rows_sharded(tokens, wr, expert, num_experts, k, gating, procs=None, routing=None):
    """``O.moe_rows`` over ``tokens`` sharded across forked workers; ``expert(e)``
    returns expert e's fp32 stacks (shared with the workers through fork).
    Returns ``(y, indices, wall_seconds, procs)``."""
    procs = procs or host_cores()
    B = tokens.shape[0]
    procs = max(1, min(procs, B))
    _STATE.update(tokens=tokens, wr=wr, expert=expert, E=num_experts, k=k, gating=gating, routing=routing)
    bounds = np.linspace(0, B, procs + 1).astype(int)
    jobs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs) if bounds[i + 1] > bounds[i]]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(jobs)) as pool:
        pool.map(_noop, range(len(jobs)))
        t0 = time.perf_counter()
        parts = pool.map(_rows_worker, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    parts.sort(key=lambda p: p[0])
    y = np.concatenate([p[1] for p in parts])
    idx = np.concatenate([p[2] for p in parts])
    _STATE.clear()
    return y, idx, wall, len(jobs)


REF_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def import_reference():
    """The UNMODIFIED reference package (``moeperf``, installed into
    ``baseline/_ref`` from /root/reference with pip --target), or None."""
    import sys
    try:
        import moeperf  # noqa: F401
    except ImportError:
        if os.path.isdir(REF_PATH) and REF_PATH not in sys.path:
            sys.path.append(REF_PATH)
        try:
            import moeperf  # noqa: F401
        except ImportError:
            return None
    import moeperf
    return moeperf


def _ref_worker(args):
    lo, hi = args
    s = _STATE
    m = s["moeperf"]
    t0 = time.perf_counter()
    y, _ = m.moe_forward(s["tokens"][lo:hi], s["wr"], s["weights"], s["config"], m.PipelineParams())
    t_fwd = time.perf_counter() - t0
    r = m.route(s["tokens"][lo:hi], s["wr"], s["config"])  # (indices for the parity check; not timed)
    return lo, y, r.indices, t_fwd


def run_reference_sharded(tokens, wr, gate, up, down, num_experts, k, gating, procs=None):
    """The reference's own ``moe_forward`` (``pipeline.py:572``) over
    ``tokens``, token-sharded across forked workers (rows are independent:
    the sharded output is bitwise the unsharded one).  Returns ``(y, indices,
    seconds, procs)`` -- seconds = the slowest worker's moe_forward time (the
    workers run concurrently; the indices for the parity check come from a
    separate, untimed ``route`` call) -- or None when the reference is not
    installed."""
    m = import_reference()
    if m is None:
        return None
    procs = procs or host_cores()
    B, d = tokens.shape
    procs = max(1, min(procs, B))
    f = gate.shape[1]
    config = m.ModelConfig(num_experts, k, d, f, m.Gating(gating))
    weights = m.ExpertWeights(gate=gate, up=up, down=down)
    _STATE.update(tokens=tokens, wr=wr, weights=weights, config=config, moeperf=m)
    bounds = np.linspace(0, B, procs + 1).astype(int)
    jobs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs) if bounds[i + 1] > bounds[i]]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(jobs)) as pool:
        pool.map(_noop, range(len(jobs)))
        parts = pool.map(_ref_worker, jobs, chunksize=1)
    parts.sort(key=lambda p: p[0])
    y = np.concatenate([p[1] for p in parts])
    idx = np.concatenate([p[2] for p in parts])
    _STATE.clear()
    return y, idx, max(p[3] for p in parts), len(jobs)


def run_sharded(tokens, wr, gate, up, down, num_experts, k, gating, procs=None):
    """Oracle forward over ``tokens`` sharded across ``procs`` forked workers.

    Returns ``(y, indices, wall_seconds, procs)``.  Weight arrays are shared
    with the workers through fork (copy-on-write, never written).
    """
    procs = procs or host_cores()
    B = tokens.shape[0]
    procs = max(1, min(procs, B))
    _STATE.update(tokens=tokens, wr=wr, gate=gate, up=up, down=down, E=num_experts, k=k, gating=gating)
    bounds = np.linspace(0, B, procs + 1).astype(int)
    jobs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs) if bounds[i + 1] > bounds[i]]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(jobs)) as pool:
        pool.map(_noop, range(len(jobs)))  # workers forked and ready before timing
        t0 = time.perf_counter()
        parts = pool.map(_worker, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    parts.sort(key=lambda p: p[0])
    y = np.concatenate([p[1] for p in parts]) if parts else np.zeros((0, tokens.shape[1]), np.float32)
    idx = np.concatenate([p[2] for p in parts]) if parts else np.zeros((0, k), np.int64)
    _STATE.clear()
    return y, idx, wall, len(jobs)
