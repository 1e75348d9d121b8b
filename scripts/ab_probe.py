"""A/B probe under sustained load: capture one CUDA graph of the layer per env
variant, then alternate back-to-back replay rounds (cancels clock / power
drift).  Usage: python scripts/ab_probe.py <config> VAR=a,b [VAR2=..]
e.g.  python scripts/ab_probe.py mixtral MOE_B200_FFN_VARIANT=2,3"""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS
name = sys.argv[1]
tokens = None
variants = [{}]
for a in sys.argv[2:]:
    if a.startswith("B="):
        tokens = int(a[2:])
        continue
    k_, vals = a.split("=")
    sep = "|" if "|" in vals else ","  # '|' separates variants whose values contain commas
    variants = [dict(v, **{k_: x}) for v in variants for x in vals.split(sep)]
E, k, d, f, gating, B, _ = CONFIGS[name]
B = tokens or B
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
# workspace sized with every router path enabled (the variants may switch paths)
os.environ["MOE_B200_SEG_MAX_CHAINS"] = str(1 << 30)
os.environ["MOE_B200_DOWN_SPLITS"] = "16"
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
os.environ.pop("MOE_B200_SEG_MAX_CHAINS")
os.environ.pop("MOE_B200_DOWN_SPLITS")
_lib.reload_tuning()  # the library reads the hooks at workspace init / reload only
out = torch.empty((B, d), dtype=torch.float32, device="cuda")
graphs = []
for v in variants:
    os.environ.update(v)
    _lib.reload_tuning()
    for _ in range(2):
        layer.forward(x, out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.forward(x, out)
    graphs.append(g)
    for k_ in v:
        os.environ.pop(k_)
    _lib.reload_tuning()
torch.cuda.synchronize()
def run(g, n):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): g.replay()
    b.record(); b.synchronize(); return a.elapsed_time(b) * 1e3 / n
t_end = time.time() + 2.0
while time.time() < t_end:
    run(graphs[0], 10)
res = [[] for _ in variants]
for rnd in range(6):
    for i, g in enumerate(graphs):
        res[i].append(run(g, 20))
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                     capture_output=True, text=True).stdout.strip()
for v, r in zip(variants, res):
    print(f"{name} B={B} {v}: us/step med {np.median(r):.1f} min {min(r):.1f}  rounds " + " ".join(f"{t:.0f}" for t in r))
print("clock,power after:", clk)
