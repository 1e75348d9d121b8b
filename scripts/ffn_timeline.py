"""Debug: per-tile timeline of the fused FFN kernel (globaltimer) for one config."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_23911_b200 as P
from paper_2605_23911_b200 import _lib
from bench import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
tag = sys.argv[2] if len(sys.argv) > 2 else name
E, k, d, f, gating, B, _ = CONFIGS[name]
B = int(os.environ.get("TL_B", B))
gen = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
gate = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
up = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
down = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(gate, up, down), wr, max_tokens=B)
for _ in range(3):
    layer.forward(x)
lib = _lib.load()
buf = torch.zeros(8 * 200000, dtype=torch.int64, device="cuda")
lib.moe_b200_debug_set_ffn_trace.argtypes = [ctypes.c_void_p]
lib.moe_b200_debug_set_ffn_trace(buf.data_ptr())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); flush.zero_()
torch.cuda.synchronize()
layer.forward(x)
torch.cuda.synchronize()
lib.moe_b200_debug_set_ffn_trace(None)
t = buf.view(-1, 8).cpu().numpy()
n = int((t[:, 1] > 0).sum())
t = t[:n]
t0 = t[:, 1].min()
rel = (t[:, 1:] - t0) / 1e3
out = {"config": name, "counts": layer.counts.tolist(), "tiles": n,
       "sm": t[:, 0].tolist(), "fetch_us": rel[:, 0].tolist(), "load_us": rel[:, 1].tolist(), "done_us": rel[:, 2].tolist(),
       "epi_start_us": rel[:, 3].tolist(), "mma_start_us": rel[:, 4].tolist(), "gu_release_us": rel[:, 5].tolist()}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/timeline_{tag}.json", "w"))
print(name, "tiles", n, "span_us", rel[:, 2].max())
raw = buf.view(-1, 8).cpu().numpy()[:n]
if len(sys.argv) > 3:
    np.save(f"gpurun_out/timeline_raw_{tag}.npy", raw)
