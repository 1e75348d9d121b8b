"""Warm per-launch times inside the one-call forward (layer.device_trace)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_23911_b200 as P
from bench import CONFIGS
for name in sys.argv[1:] or ["qwen60", "mixtral"]:
    E, k, d, f, gating, B, _ = CONFIGS[name]
    B = int(os.environ.get("ST_B", B))
    gen = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
    wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
    gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
    layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
    for _ in range(3):
        layer.forward(x)
    tr = layer.device_trace(x, iters=20)
    print(name, B, " | ".join(f"{r['launch']}: {r['time_us']:.1f} us" for r in tr))
    del layer, gate, up, down
    torch.cuda.empty_cache()
