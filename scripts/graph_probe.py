"""Probe: where does the graph-replayed step time go?  Times (a) graph replay
with and without an L2 flush between steps, (b) per-stage times with the
library's events captured INSIDE the graph.  Usage: python scripts/graph_probe.py [config] [tokens]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
E, k, d, f, gating, B, _ = CONFIGS[name]
if len(sys.argv) > 2:
    B = int(sys.argv[2])
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
out = torch.empty((B, d), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    layer.forward(x, out)
torch.cuda.synchronize()
def capture(env):
    for k_, v_ in env.items():
        os.environ[k_] = v_
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.forward(x, out)
    for k_ in env:
        os.environ.pop(k_, None)
    return g
variants = {"pdl": capture({}), "no_pdl": capture({"MOE_B200_NO_PDL": "1"})}
torch.cuda.synchronize()
def run(graph, n, do_flush):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        if do_flush: flush.zero_()
        st[i].record(); graph.replay(); en[i].record()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in zip(st, en)]) * 1e3
res = {k: [] for k in variants}
for rnd in range(8):  # alternate variants to cancel drift in clocks / power
    for kname, g in variants.items():
        res[kname].append(run(g, 10, True))
line = f"{name} B={B}: graph step us (flush, alternating A/B):"
for kname, v in res.items():
    v = np.concatenate(v)
    line += f" {kname} med {np.median(v):.1f} min {v.min():.1f} |"
print(line)
