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
s = torch.cuda.Stream()
# graph with the library's stage events inside
lib = layer.lib
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for e in ev:
    e.record()
torch.cuda.synchronize()
arr = (ctypes.c_void_p * 5)(*[e.cuda_event for e in ev])
xp, xdt = layer._prep_x(x)
def fwd_timed():
    rc = lib.moe_b200_forward_timed(ctypes.byref(layer.cfg), B, xp.data_ptr(), xdt, layer.router_weight.data_ptr(),
        layer.weights.gate.data_ptr(), layer.weights.up.data_ptr(), layer.weights.down.data_ptr(), out.data_ptr(), 0,
        layer.topk_idx.data_ptr(), layer.topk_w.data_ptr(), layer.counts.data_ptr(), layer.offsets.data_ptr(),
        layer.fwd.data_ptr(), layer.inv.data_ptr(), layer.ws.data_ptr(), layer.ws_bytes, torch.cuda.current_stream().cuda_stream, arr)
    assert rc == 0, rc
g_plain = torch.cuda.CUDAGraph()
with torch.cuda.graph(g_plain):
    layer.forward(x, out)
g_timed = torch.cuda.CUDAGraph()
with torch.cuda.graph(g_timed):
    fwd_timed()
torch.cuda.synchronize()
def run(graph, n, do_flush):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        if do_flush: flush.zero_()
        st[i].record(); graph.replay(); en[i].record()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in zip(st, en)]) * 1e3
for _ in range(2):
    a = run(g_plain, 30, True); b = run(g_plain, 30, False)
    print(f"{name} B={B}: graph step us: flush med {np.median(a):.1f} min {a.min():.1f} | no-flush med {np.median(b):.1f} min {b.min():.1f}")
names = ["route", "dispatch", "ffn", "combine"]
acc = np.zeros(4)
n = 20
for i in range(n):
    flush.zero_()
    g_timed.replay()
    torch.cuda.synchronize()
    acc += np.array([ev[j].elapsed_time(ev[j + 1]) for j in range(4)]) * 1e3
print("  in-graph stages us: " + " ".join(f"{nm}={v/n:.1f}" for nm, v in zip(names, acc)) + f" sum={acc.sum()/n:.1f}")
