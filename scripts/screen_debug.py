"""Debug: the screening router's phase-2 path counters (router_screen.cuh, via
the router trace hook) and route() times.  Usage: python scripts/screen_debug.py [config] [tokens]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "deepseek"
E, k, d, f, gating, B, _ = CONFIGS[name]
if len(sys.argv) > 2:
    B = int(sys.argv[2])
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
z = np.zeros((E * d, 8), np.float32)
layer = P.MoELayer(P.ModelConfig(E, k, d, 8, P.Gating(gating)), P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
for _ in range(3):
    layer.route(x)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(20):
    ev[0].record(); layer.route(x); ev[1].record(); torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
lib = _lib.load()
buf = torch.zeros(16 * 65536, dtype=torch.int64, device="cuda")
lib.moe_b200_debug_set_router_trace.argtypes = [ctypes.c_void_p]
lib.moe_b200_debug_set_router_trace(buf.data_ptr())
layer.route(x)
torch.cuda.synchronize()
lib.moe_b200_debug_set_router_trace(None)
c = buf[:8].cpu().numpy()
tl = buf[64:64 + 8 * 1024].view(-1, 8).cpu().numpy()
tl = tl[tl[:, 0] > 0]
if len(tl):
    g0 = (tl[:, 0] - tl[:, 0].min()) / 1e3
    g1 = (tl[:, 4] - tl[:, 0].min()) / 1e3
    print(f"  phase-2 CTAs {len(tl)}: start spread us {g0.max():.1f}, end us med {np.median(g1):.1f} max {g1.max():.1f}")
    for i, nm in ((1, "merged"), (2, "synced"), (3, "selected")):
        print(f"    {nm:9s} cycles med {np.median(tl[:, i]):.0f} max {tl[:, i].max():.0f}")
print(f"{name} B={B}: route us median {np.median(ts):.1f} min {min(ts):.1f}")
print("  chains: inconclusive", c[0], "empty-intersection", c[1], "width>0", c[2])
print("  tokens: general(no cand)", c[3], "general(Sk tiny)", c[4], "general(unsure)", c[5], "lean", c[6])
