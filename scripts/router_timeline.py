"""Debug: CTA-0 per-chunk timeline of the router kernel (clock64 cycles)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
E, k, d, f, gating, B, _ = CONFIGS[name]
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
z = np.zeros((E * d, 8), np.float32)
layer = P.MoELayer(P.ModelConfig(E, k, d, 8, P.Gating(gating)), P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
for _ in range(3):
    layer.route(x)
lib = _lib.load()
buf = torch.zeros(4 * 4096 + 4 * 2048 + 2048, dtype=torch.int64, device="cuda")
lib.moe_b200_debug_set_router_trace.argtypes = [ctypes.c_void_p]
lib.moe_b200_debug_set_router_trace(buf.data_ptr())
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); layer.route(x); e1.record()
torch.cuda.synchronize()
lib.moe_b200_debug_set_router_trace(None)
raw = buf.cpu().numpy()
ph = raw[4 * 4096: 4 * 4096 + 4 * 2048].reshape(-1, 4)
st = raw[4 * 4096 + 4 * 2048:]
t = raw[:4 * 4096].reshape(-1, 4)
n = int((t[:, 3] > 0).sum())
t = t[:n] - t[0, 0]
print(name, "route ms", e0.elapsed_time(e1), "chunks", n)
print("chunk issue rawfull full done (cycles rel. to first issue)")
for c in list(range(min(n, 12))) + list(range(max(12, n - 4), n)):
    print(c, t[c].tolist(), "copy lat", t[c, 1] - t[c, 0], "compute", t[c, 3] - t[c, 2], "wait full", t[c, 2] - (t[c - 1, 3] if c else 0))

nb = int((ph[:, 0] > 0).sum())
t0 = st[:nb].min()
p1 = (ph[:nb, 0] - t0) / 1e3
p2 = (ph[:nb, 1] - t0) / 1e3
who = np.where(ph[:nb, 2] == 1)[0]
print("CTAs", nb, "start spread us", (st[:nb].max() - t0) / 1e3, "phase1 end min/med/max us", p1.min(), np.median(p1), p1.max())
p2v = p2[p2 > -1e5]
print("phase2 end (for CTAs that ran it) max us", p2v[p2v > 0].max() if (p2v > 0).any() else None)
if len(who):
    print("phase3 CTA", who[0], "end us", (ph[who[0], 3] - t0) / 1e3)
