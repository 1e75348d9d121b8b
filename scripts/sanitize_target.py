"""Small workloads for compute-sanitizer (tests/test_gpu_sanitizers.py): every
kernel of the library on small shapes.  Usage:
    python scripts/sanitize_target.py layer|pairs|stages|ep"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_23911_b200 as P  # noqa: E402
from oracle import moe_oracle as O  # noqa: E402


def layer_case(e, k, d, f, b, g, routed=False, unfused=False, y_bf16=False):
    tokens, wr, gate, up, down = O.make_instance(11, e, k, d, f, b)
    out = torch.bfloat16 if y_bf16 else torch.float32
    layer = P.MoELayer(P.ModelConfig(e, k, d, f, P.Gating(g)), P.ExpertWeights(gate, up, down), wr, max_tokens=b,
                       out_dtype=out)
    x = torch.from_numpy(tokens).cuda()
    layer.forward(x)
    layer.forward(x[: max(1, b // 2)])
    if unfused:
        layer.forward(x, fused=False)
    if routed:
        idx = np.stack([np.random.default_rng(t).permutation(e)[:k] for t in range(b)])
        w = np.full((b, k), 1.0 / k, np.float32)
        layer.forward_routed(x, (idx, w))
    torch.cuda.synchronize()


def main(which):
    if which == "layer":
        layer_case(8, 2, 256, 512, 64, "softmax", routed=True, unfused=True)      # segment router, 128-row chunks
        layer_case(16, 4, 128, 256, 48, "sigmoid_normalized", y_bf16=True)
        layer_case(256, 8, 64, 64, 300, "sigmoid_normalized")                     # INT8 screen router (> 64K chains)
        layer_case(256, 8, 64, 64, 300, "softmax")                                # exact router (> 64K chains)
    elif which == "pairs":
        layer_case(4, 2, 256, 384, 512, "softmax")                                # 256-row chunks: cta_group::2 pairs
    elif which == "stages":
        tokens, wr, gate, up, down = O.make_instance(5, 8, 2, 64, 96, 40)
        cfg = P.ModelConfig(8, 2, 64, 96)
        r = P.route(tokens, wr, cfg)
        perm = P.build_permutation(r)
        off = P.expert_offsets(P.expert_histogram(r, 8))
        sch = P.build_block_schedule(off, 64)
        xp = P.permute_tokens(tokens, r, perm)
        w = P.ExpertWeights(gate, up, down)
        h = P.fused_gate_up(xp, w, sch, off, P.PipelineParams())
        P.unfused_gate_up(xp, w, sch, off, P.PipelineParams())
        ys = P.grouped_gemm(h, down, sch, off, P.PipelineParams())
        P.unpermute_combine(ys, r, perm)
        s = P.gate_scores(np.random.default_rng(0).standard_normal((33, 60)).astype(np.float32), P.Gating.SOFTMAX)
        P.topk_select(s, 4)
        P.silu(np.linspace(-120, 120, 1000, dtype=np.float32))
        P.dense_matmul(tokens, wr)
        torch.cuda.synchronize()
    elif which == "ep":
        from paper_2605_23911_b200.ep import ExpertParallelMoE
        tokens, wr, gate, up, down = O.make_instance(9, 16, 4, 128, 256, 32)
        cfg = P.ModelConfig(16, 4, 128, 256, P.Gating.SIGMOID_NORMALIZED)
        ep = ExpertParallelMoE(cfg, wr, P.ExpertWeights(gate, up, down), max_tokens=32, transport="p2p")
        for _ in range(2):
            ep.forward(torch.from_numpy(tokens).cuda())
        torch.cuda.synchronize()
        ep.p2p.close()
    print("sanitize target done:", which)


if __name__ == "__main__":
    main(sys.argv[1])
