"""Debug: list the logits whose certified interval is not a single fp32 value
after route() (segment router), with the exact value.  Usage: python scripts/lbuf_debug.py [config]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from bench import CONFIGS
from oracle import moe_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "qwen60"
E, k, d, f, gating, B, _ = CONFIGS[name]
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
z = np.zeros((E * d, 8), np.float32)
layer = P.MoELayer(P.ModelConfig(E, k, d, 8, P.Gating(gating)), P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
layer.route(x)
torch.cuda.synchronize()
lib = layer.lib
lib.moe_b200_debug_lbuf_offset.restype = ctypes.c_size_t
off = lib.moe_b200_debug_lbuf_offset(ctypes.byref(layer.cfg), B)
lb = layer.ws[off: off + B * E * 8].view(torch.float32).view(B, E, 2).cpu().numpy()
lo, hi = lb[..., 0], lb[..., 1]
bad = np.argwhere(~(lo.view(np.uint32) == hi.view(np.uint32)))
xs = x.float().cpu().numpy().astype(np.float64); ws = wr.cpu().numpy().astype(np.float64)
print(name, "uncertain logits:", len(bad), "of", B * E)
for t, e in bad[:10]:
    p = xs[t] * ws[:, e]
    seq = np.add.accumulate(p)[-1]
    print(f"  t={t} e={e} lo={lo[t,e]!r} hi={hi[t,e]!r} exact={np.float32(seq)!r} seq={seq!r} "
          f"ulp32={np.spacing(np.float32(seq))!r} width={float(hi[t,e]) - float(lo[t,e])!r}")
