"""Exhaustive check of oracle/np_exp64.c (the C restatement of numpy's float64
exp) against this host's np.exp on every float32 input in (-707.7, 0]
(1.144e9 values, ~1 minute).  Usage: python scripts/check_np_exp64.py"""
import ctypes, os, subprocess, tempfile, time
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(tempfile.mkdtemp(), "np_exp64.so")
subprocess.run(["gcc", "-O2", "-mfma", "-frounding-math", "-shared", "-fPIC", "-o", so,
                os.path.join(ROOT, "oracle", "np_exp64.c"), "-lm"], check=True)
lib = ctypes.CDLL(so)
lib.np_exp64_array.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
hi = int(np.array([-707.70327], np.float32).view(np.uint32)[0])
chunk = 1 << 26
t0, bad, n = time.time(), 0, 0
for c0 in range(0x80000000, hi + 1, chunk):
    c1 = min(hi + 1, c0 + chunk)
    x = np.arange(c0, c1, dtype=np.uint64).astype(np.uint32).view(np.float32).astype(np.float64)
    x = x[np.abs(x) < 707.7032713517042]
    y = np.empty_like(x)
    lib.np_exp64_array(x.ctypes.data, y.ctypes.data, x.size)
    bad += int((y.view(np.uint64) != np.exp(x).view(np.uint64)).sum())
    n += x.size
print("checked", n, "mismatches", bad, "secs", round(time.time() - t0, 1))
