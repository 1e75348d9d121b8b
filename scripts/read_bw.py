"""Probe: pure-read HBM bandwidth (sum over a large bf16 tensor) vs copy."""
import torch
x = torch.empty(2 << 30, dtype=torch.bfloat16, device="cuda").normal_()  # 4 GiB
y = torch.empty_like(x)
for name, fn, nbytes in (("sum (read)", lambda: x.sum(dtype=torch.float32), x.numel() * 2),
                         ("amax (read)", lambda: x.abs().amax() if False else torch.amax(x), x.numel() * 2),
                         ("copy (r+w)", lambda: y.copy_(x), x.numel() * 4)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{name}: best {nbytes / min(ts) / 1e6:.0f} GB/s, median {nbytes / sorted(ts)[5] / 1e6:.0f} GB/s")
