"""Probe: host cost of one eager layer.forward (C-ABI call from Python) vs the
device time of the same forward under graph replay."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_23911_b200 as P
from bench import CONFIGS
for name, B in (("small", 128), ("mixtral", 1), ("mixtral", 512)):
    E, k, d, f, gating, _, _ = CONFIGS[name]
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
    wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
    g = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    u = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    dn = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
    layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(g, u, dn), wr, max_tokens=B)
    out = torch.empty((B, d), dtype=torch.float32, device="cuda")
    for _ in range(5):
        layer.forward(x, out)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        layer.forward(x, out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        layer.forward(x, out)
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        gr.replay()
    b.record(); torch.cuda.synchronize()
    print(f"{name} B={B}: host per eager call {1e6 * (t1 - t0) / n:.1f} us, eager wall per step {1e6 * (t2 - t0) / n:.1f} us, "
          f"graph replay per step {1e3 * a.elapsed_time(b) / n:.1f} us")
    del layer, g, u, dn
    torch.cuda.empty_cache()

# split: the C-ABI call alone (pointers computed once) vs layer.forward
import ctypes
from paper_2605_23911_b200 import _lib
from paper_2605_23911_b200.layer import _ptr, _stream_ptr
E, k, d, f, gating, _, _ = CONFIGS["small"]
B = 128
gen = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((B, d), generator=gen, device="cuda").to(torch.bfloat16)
wr = (torch.randn((d, E), generator=gen, device="cuda") / d ** 0.5).float()
g = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
u = (torch.randn((E * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
dn = (torch.randn((E * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
layer = P.MoELayer(P.ModelConfig(E, k, d, f, P.Gating(gating)), P.ExpertWeights(g, u, dn), wr, max_tokens=B)
out = torch.empty((B, d), dtype=torch.float32, device="cuda")
layer.forward(x, out)
args = (ctypes.byref(layer.cfg), B, _ptr(x), _lib.DTYPE_BF16, _ptr(layer.router_weight), _ptr(layer.weights.gate),
        _ptr(layer.weights.up), _ptr(layer.weights.down), _ptr(out), _lib.DTYPE_F32, _ptr(layer.topk_idx),
        _ptr(layer.topk_w), _ptr(layer.counts), _ptr(layer.offsets), _ptr(layer.fwd), _ptr(layer.inv), _ptr(layer.ws),
        layer.ws_bytes, _stream_ptr(layer.device))
fn = layer.lib.moe_b200_forward
for _ in range(10):
    fn(*args)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    fn(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"small: direct C-ABI call {1e6 * (t1 - t0) / n:.1f} us host")
t0 = time.perf_counter()
for _ in range(n):
    layer.forward(x, out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"small: layer.forward {1e6 * (t1 - t0) / n:.1f} us host")

# host cost per forward_host submission (pinned host buffers), graphs off / on
for gflag in ("0", "1"):
    os.environ["MOE_B200_IO_GRAPHS"] = gflag
    xh = [x.cpu().pin_memory() for _ in range(2)]
    yh = [torch.empty((B, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    pipe = layer.host_pipeline(x_dtype=torch.bfloat16, y_dtype=torch.float32)
    for i in range(6):
        pipe.submit(xh[i % 2], yh[i % 2])
    pipe.sync()
    n = 500
    t0 = time.perf_counter()
    for i in range(n):
        pipe.submit(xh[i % 2], yh[i % 2])
    t1 = time.perf_counter()
    pipe.sync()
    t2 = time.perf_counter()
    print(f"small: forward_host graphs={gflag}: host {1e6 * (t1 - t0) / n:.1f} us per submit, wall {1e6 * (t2 - t0) / n:.1f} us per step")
    pipe.close()
