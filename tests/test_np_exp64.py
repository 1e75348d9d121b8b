"""The C restatement of numpy's float64 exp (oracle/np_exp64.c; the softmax's
np.exp, router.py:65 / :82) against this host's np.exp: a stratified sample of
float32 inputs in (-707.7, 0].  (The device port, csrc/router.cuh np_exp64,
follows the restatement op for op; tests/test_gpu_stage_api.py checks it
exhaustively against the GPU box's own numpy.)  Skips on hosts whose numpy
does not dispatch float64 exp to AVX-512 SVML."""

from __future__ import annotations

import ctypes
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cport(tmp_path_factory):
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("gcc not available")
    so = tmp_path_factory.mktemp("npexp") / "np_exp64.so"
    subprocess.run([cc, "-O2", "-mfma", "-frounding-math", "-shared", "-fPIC", "-o", str(so),
                    os.path.join(ROOT, "oracle", "np_exp64.c"), "-lm"], check=True)
    lib = ctypes.CDLL(str(so))
    lib.np_exp64_array.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
    return lib


def _run(lib, x):
    y = np.empty_like(x)
    lib.np_exp64_array(x.ctypes.data, y.ctypes.data, x.size)
    return y


def test_np_exp64_restatement_matches_numpy(cport):
    probe = np.linspace(-700, 0, 4096)
    if not np.array_equal(_run(cport, probe).view(np.uint64), np.exp(probe).view(np.uint64)):
        pytest.skip("this host's numpy float64 exp is not the AVX-512 SVML kernel")
    rng = np.random.default_rng(0)
    bits = rng.integers(0x80000000, 0xC430EDA0, 4_000_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32).astype(np.float64)
    x = x[np.abs(x) < 707.7032713517042]
    for lo in (-1e-6, -1e-3, -1.0, -20.0):
        x = np.concatenate([x, np.random.default_rng(1).uniform(lo, 0, 200_000).astype(np.float32).astype(np.float64)])
    y = _run(cport, x)
    bad = np.nonzero(y.view(np.uint64) != np.exp(x).view(np.uint64))[0]
    assert bad.size == 0, (bad.size, x[bad[:5]])
