"""Expert-parallel host logic on CPU: world_size 2 over gloo.

The EP layer (paper_2605_23911_b200/ep.py) runs its all-to-alls through
torch.distributed; here its row compute is replaced by an oracle-backed ops
object (test infrastructure), so the partition, split sizes, source/expert
reorders and the home-rank combine order are checked on CPU: EP=2 must equal
the single-process oracle forward BIT-FOR-BIT.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O


class OracleOps:
    """Reference arithmetic on CPU tensors (fp32 h, fp64-fold GEMMs)."""

    def __init__(self, tokens_all, wr, gate, up, down, E, k, d, f, gating, lo, hi):
        self.wr, self.gate, self.up, self.down = wr, gate, up, down
        self.E, self.k, self.d, self.f, self.gating = E, k, d, f, gating
        self.lo, self.hi = lo, hi

    def route(self, x):
        idx, w = O.route(x.numpy(), self.wr, self.k, self.gating)
        counts = O.expert_histogram(idx, self.E)
        fwd, inv = O.build_permutation(idx)
        return (torch.from_numpy(idx), torch.from_numpy(w), torch.from_numpy(counts),
                torch.from_numpy(fwd), torch.from_numpy(inv))

    def permute(self, x, fwd, k):
        return x[fwd // k].clone()

    def gather_rows(self, src, idx):
        return src[idx.long()].clone()

    def expert_ffn(self, counts, xp, global_tokens):
        self.global_tokens = global_tokens
        out = torch.zeros((xp.shape[0], self.d), dtype=torch.float32)
        d, f = self.d, self.f
        r = 0
        for el, c in enumerate(counts.tolist()):
            if c:
                e = self.lo + el
                a = xp[r:r + c].numpy()
                g = O.dot_fp64_fold(a, self.gate[e * d:(e + 1) * d])
                u = O.dot_fp64_fold(a, self.up[e * d:(e + 1) * d])
                h = (O.silu_f32(g) * u).astype(np.float32)
                out[r:r + c] = torch.from_numpy(O.dot_fp64_fold(h, self.down[e * f:(e + 1) * f]))
            r += c
        return out

    def combine(self, rows, inv, w, B):
        return torch.from_numpy(O.unpermute_combine(rows.numpy(), w.numpy(), inv.numpy()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_23911_b200.ep import ExpertParallelMoE, expert_ranges
        from paper_2605_23911_b200.types import Gating, ModelConfig

        seed, E, k, d, f, B, gating = case
        tokens, wr, gate, up, down = O.make_instance(seed, E, k, d, f, B)
        cfg = ModelConfig(E, k, d, f, Gating(gating))
        lo, hi = expert_ranges(E, world)[rank]
        b0, b1 = rank * B // world, (rank + 1) * B // world
        ops = OracleOps(tokens, wr, gate, up, down, E, k, d, f, gating, lo, hi)
        layer = ExpertParallelMoE(cfg, wr, None, max_tokens=B, device="cpu", ops=ops)
        y = layer.forward(torch.from_numpy(tokens[b0:b1]))
        # the counts exchange also carries every rank's token count: each rank
        # sees the global batch (it fixes the down K-split count)
        assert ops.global_tokens == B, (ops.global_tokens, B)
        q.put((rank, b0, y.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (0, 8, 2, 16, 24, 13, "softmax"),
    (1, 16, 4, 32, 16, 20, "sigmoid_normalized"),
    (2, 6, 2, 8, 12, 9, "softmax"),   # uneven expert blocks (6 experts over 2 ranks -> 3+3)
])
def test_expert_parallel_world2_matches_single_process_bitwise(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    y_ep = np.concatenate([t[2] for t in parts])
    seed, E, k, d, f, B, gating = case
    tokens, wr, gate, up, down = O.make_instance(seed, E, k, d, f, B)
    ref = O.moe_forward(tokens, wr, gate, up, down, E, k, gating)
    np.testing.assert_array_equal(y_ep.view(np.uint32), ref["y"].view(np.uint32))


def test_expert_ranges_and_reorder():
    from paper_2605_23911_b200.ep import expert_ranges, source_major_to_expert_major

    assert expert_ranges(256, 8) == [(32 * r, 32 * (r + 1)) for r in range(8)]
    assert expert_ranges(60, 8)[0] == (0, 8) and expert_ranges(60, 8)[-1][1] == 60
    for E, n in ((60, 8), (7, 3), (256, 4)):
        owner = [e * n // E for e in range(E)]
        rng = expert_ranges(E, n)
        assert all(rng[owner[e]][0] <= e < rng[owner[e]][1] for e in range(E))
    rc = np.array([[2, 0, 1], [1, 3, 0]])  # src x expert
    # source-major rows: s0:e0(0,1) e2(2) | s1:e0(3) e1(4,5,6)
    assert source_major_to_expert_major(rc).tolist() == [0, 1, 3, 4, 5, 6, 2]
