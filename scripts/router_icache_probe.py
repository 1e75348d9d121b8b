"""Debug: segment-router phase timeline with the L2 warm (router run back to
back) vs flushed (a 512 MB write between routes, as the FFN's weight stream
does inside a forward): is phase 2 paying for cold instruction / data fetch?
Usage: python scripts/router_icache_probe.py [config] [tokens]"""
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
z = np.zeros((E * d, 8), np.float32)
layer = P.MoELayer(P.ModelConfig(E, k, d, 8, P.Gating(gating)), P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    layer.route(x)
torch.cuda.synchronize()
lib = _lib.load()
lib.moe_b200_debug_set_router_trace.argtypes = [ctypes.c_void_p]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for mode in ("warm", "flushed"):
    ts, rows = [], []
    for it in range(12):
        buf = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
        if mode == "flushed":
            flush.fill_(it & 255)
        else:
            layer.route(x)
        traced = it >= 6
        if traced:
            lib.moe_b200_debug_set_router_trace(buf.data_ptr())
        ev[0].record(); layer.route(x); ev[1].record(); torch.cuda.synchronize()
        if traced:
            lib.moe_b200_debug_set_router_trace(None)
            t = buf.view(-1, 16).cpu().numpy()
            rows.append(t[t[:, 0] > 0])
        else:
            ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    t = np.concatenate(rows)
    print(f"{name} B={B} {mode}: route us (untraced) median {np.median(ts):.1f}")
    for i, nm in ((2, "part-store"), (3, "cta-reduce"), (6, "arrive2"), (7, "phase2-end")):
        v = t[:, i][t[:, i] > 0]
        if len(v):
            print(f"  {nm:12s} cycles med {int(np.median(v))}")
    for i, nm in ((8, "p2 lbuf"), (9, "p2 certified"), (14, "p2 topk")):
        v = t[:, i][t[:, i] > 0]
        if len(v):
            print(f"  {nm:12s} cycles from phase-2 entry med {int(np.median(v))}")
