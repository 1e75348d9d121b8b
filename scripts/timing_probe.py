"""Probe: sustained µs/step of the same layer under different launch/timing
methods, alternated to cancel power/clock drift.  Usage: python scripts/timing_probe.py [config]"""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
E, k, d, f, gating, B, _ = CONFIGS[name]
dev = torch.device("cuda")
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
out = torch.empty((B, d), dtype=torch.float32, device="cuda")
for _ in range(3):
    layer.forward(x, out)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    layer.forward(x, out)
torch.cuda.synchronize()
def smi():
    r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"], capture_output=True, text=True)
    return r.stdout.strip()
def loop_graph(n):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): g.replay()
    b.record(); b.synchronize(); return a.elapsed_time(b) * 1e3 / n
def loop_direct(n):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): layer.forward(x, out)
    b.record(); b.synchronize(); return a.elapsed_time(b) * 1e3 / n
def loop_graph_events(n):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]; en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        st[i].record(); g.replay(); en[i].record()
    torch.cuda.synchronize(); return float(np.mean([s.elapsed_time(e) for s, e in zip(st, en)])) * 1e3
def loop_graph_events_gaps(n):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]; en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        st[i].record(); g.replay(); en[i].record()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n
methods = {"graph_b2b": loop_graph, "direct_b2b": loop_direct, "graph_per_step_events": loop_graph_events,
           "graph_events_wall": loop_graph_events_gaps}
res = {m: [] for m in methods}
t_end = time.time() + 2.0
while time.time() < t_end:
    loop_graph(20)
for rnd in range(4):
    for m, fn in methods.items():
        res[m].append(fn(40))
    print("round", rnd, smi(), flush=True)
for m, v in res.items():
    print(f"{name}: {m:24s} us/step: " + " ".join(f"{t:.1f}" for t in v))
