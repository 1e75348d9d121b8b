"""Debug: per-CTA timeline of the dispatch kernel (globaltimer start + clock64
phase deltas).  Usage: python scripts/dispatch_timeline.py [config] [tokens]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "qwen60"
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
lib = _lib.load()
buf = torch.zeros(16 * 8192, dtype=torch.int64, device="cuda")
lib.moe_b200_debug_set_dispatch_trace.argtypes = [ctypes.c_void_p]
lib.moe_b200_debug_set_dispatch_trace(buf.data_ptr())
layer.route(x)
torch.cuda.synchronize()
lib.moe_b200_debug_set_dispatch_trace(None)
t = buf.view(-1, 16).cpu().numpy()
n = int((t[:, 0] > 0).sum())
t = t[:n]
g0 = (t[:, 0] - t[:, 0].min()) / 1e3
print(f"{name} B={B}: dispatch CTAs {n}; start spread us med {np.median(g0):.2f} max {g0.max():.2f}")
for i, nm in [(1, "idx staged"), (2, "histogram"), (6, "scan (warp0)"), (7, "sync"), (8, "cta0 tables"), (3, "positions"), (4, "sync"), (5, "gather")]:
    v = t[:, i]
    print(f"  {nm:18s} cycles min/med/max {v.min()}/{int(np.median(v))}/{v.max()}")
