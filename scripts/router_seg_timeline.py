"""Debug: per-CTA timeline of the segment router (globaltimer) + exact-chain
fallback counts, and route() times under env variants.
Usage: python scripts/router_seg_timeline.py [config] [tokens]"""
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
t = buf.view(-1, 16).cpu().numpy()
n = int((t[:, 0] > 0).sum())
t = t[:n]
print(f"{name} B={B}: route us median {np.median(ts):.1f} min {min(ts):.1f}; CTAs {n}")
g0 = (t[:, 0] - t[:, 0].min()) / 1e3
print(f"  CTA start spread us: med {np.median(g0):.1f} max {g0.max():.1f}")
names = ["", "phase1", "part-store", "cta-reduce", "arrive1", "finalize", "arrive2", "phase2", "arrive3", "phase3"]
for i in range(2, 8):
    v = t[:, i][t[:, i] > 0]
    if len(v):
        print(f"  {names[i]:10s} n={len(v):5d} cycles min/med/max {v.min()}/{int(np.median(v))}/{v.max()}")
for i, nm in ((8, "p2 lbuf"), (9, "p2 certified"), (15, "p2 exp"), (1, "p2 sum"), (13, "p2 scores"), (14, "p2 topk")):
    v = t[:, i][t[:, i] > 0]
    if len(v):
        print(f"  {nm:12s} n={len(v):5d} cycles from phase-2 entry min/med/max {v.min()}/{int(np.median(v))}/{v.max()}")
print(f"  exact chains: certify-round {int(t[:, 11].sum())}, max-uncertain {int((t[:, 12] & 0xFFFFFFFF).sum())}; "
      f"enumeration-certified tokens {int((t[:, 12] >> 32).sum())}; logits {B*E}")
