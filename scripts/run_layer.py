"""Minimal driver for ncu captures: build a layer of a BASELINE config and run
N forwards (no timing).
Usage: python scripts/run_layer.py [config] [tokens] [iters] [fused|unfused]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_23911_b200 as P  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
E, k, d, f, gating, B0, _ = CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else B0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
fused = (sys.argv[4] if len(sys.argv) > 4 else "fused") != "unfused"
for _ in range(iters):
    layer.forward(x, fused=fused)
torch.cuda.synchronize()
print("counts", layer.counts.tolist())
