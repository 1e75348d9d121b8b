"""CPU tests of the host logic and the C-ABI library surface (no GPU calls)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from golden_util import golden_meta
from oracle import moe_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------------------
# numpy pairwise summation: the algorithm the router kernel implements
# (csrc/router.cuh pairwise_sum) restated here and pinned to ndarray.sum.
# ---------------------------------------------------------------------------

def _pairwise_block(a, n, dt):
    if n < 8:
        r = dt(0)
        for i in range(n):
            r = dt(r + a[i])
        return r
    r = [a[j] for j in range(8)]
    i = 8
    while i < n - (n % 8):
        for j in range(8):
            r[j] = dt(r[j] + a[i + j])
        i += 8
    res = dt(dt(dt(r[0] + r[1]) + dt(r[2] + r[3])) + dt(dt(r[4] + r[5]) + dt(r[6] + r[7])))
    while i < n:
        res = dt(res + a[i])
        i += 1
    return res


def _pairwise(a, n, dt):
    if n <= 128:
        return _pairwise_block(a, n, dt)
    n2 = n // 2
    n2 -= n2 % 8
    return dt(_pairwise(a[:n2], n2, dt) + _pairwise(a[n2:], n - n2, dt))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pairwise_sum_matches_numpy(dtype):
    rng = np.random.default_rng(0)
    for n in list(range(1, 140)) + [200, 255, 256, 257, 300, 512, 1024]:
        rows = (rng.random((4, n)) * rng.choice([1e-3, 1.0, 1e3], size=(4, 1))).astype(dtype)
        ref = rows.sum(axis=1)
        for r in range(4):
            got = _pairwise(list(rows[r]), n, dtype)
            assert got == ref[r], (n, got, ref[r])


# ---------------------------------------------------------------------------
# trace replay against the reference's executed traces
# ---------------------------------------------------------------------------

def test_trace_from_counts_matches_reference_golden(golden):
    from paper_2605_23911_b200 import Gating, ModelConfig, PipelineParams, trace_from_counts

    for _, name, seed, e, k, d, f, b, g in [m for m in golden_meta(golden) if m[0] == "fwd"]:
        cfg = ModelConfig(e, k, d, f, Gating(g))
        counts = golden[f"fwd/{name}/counts"]
        tr = trace_from_counts(cfg, b, counts, PipelineParams())
        np.testing.assert_array_equal([r.flops for r in tr.records], golden[f"fwd/{name}/trace_flops"])
        np.testing.assert_array_equal([r.total_bytes for r in tr.records], golden[f"fwd/{name}/trace_bytes"])
        np.testing.assert_array_equal([r.tiles for r in tr.records], golden[f"fwd/{name}/trace_tiles"])
        assert [r.stage for r in tr.records] == ["Router", "HostSchedule", "Permute", "GateUp", "Down", "Unpermute"]


def test_host_schedule_and_errors():
    import paper_2605_23911_b200 as P

    off = P.expert_offsets([5, 0, 7])
    assert off.offsets.tolist() == [0, 5, 5, 12]
    assert P.build_block_schedule(off, 4).entries == ((0, 0), (0, 4), (2, 0), (2, 4))
    for bad in (0, -1, 2.5, True):
        with pytest.raises(P.InvalidBlockM):
            P.build_block_schedule(off, bad)
    with pytest.raises(P.IndexOutOfRange):
        P.expert_offsets([2, -1])
    with pytest.raises(ValueError):
        P.ModelConfig(4, 5, 8, 8)
    with pytest.raises(ValueError):
        P.PipelineParams(block_m=0)
    with pytest.raises(KeyError):
        P.preset("nope")
    assert P.preset("DeepSeekV3").gating is P.Gating.SIGMOID_NORMALIZED


# ---------------------------------------------------------------------------
# C-ABI surface: the library loads and exports every declared symbol
# ---------------------------------------------------------------------------

def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "moe_b200.h")).read()
    return sorted(set(re.findall(r"\b(moe_b200_[a-z_]+)\s*\(", src)))


def test_header_declares_the_stage_entry_points():
    syms = _declared_symbols()
    for s in ("moe_b200_route", "moe_b200_permute", "moe_b200_gate_up", "moe_b200_down_scatter",
              "moe_b200_combine", "moe_b200_forward", "moe_b200_workspace_size", "moe_b200_strerror"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2605_23911_b200 import _lib

    lib = _lib.load()
    for s in _declared_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, s
    assert lib.moe_b200_version().startswith(b"moe_b200")
    assert lib.moe_b200_strerror(2).startswith(b"ShapeMismatch")


def test_workspace_size_and_config_validation_without_gpu():
    from paper_2605_23911_b200 import _lib

    lib = _lib.load()
    n = ctypes.c_size_t(0)
    cfg = _lib.config_struct(8, 2, 4096, 14336, 0)
    assert lib.moe_b200_workspace_size(ctypes.byref(cfg), 512, ctypes.byref(n)) == 0
    T = 512 * 2
    assert n.value >= T * 4096 * 2 + T * 14336 * 2 + T * 4096 * 4
    bad = _lib.config_struct(8, 9, 4096, 14336, 0)
    assert lib.moe_b200_workspace_size(ctypes.byref(bad), 512, ctypes.byref(n)) == 3  # InvalidK
    odd = _lib.config_struct(8, 2, 4095, 14336, 0)
    assert lib.moe_b200_workspace_size(ctypes.byref(odd), 512, ctypes.byref(n)) == 9  # unsupported pitch


def test_down_split_rule_and_workspace_monotonicity_without_gpu():
    """The down K-split count (a function of config and batch only, so EP
    ranks can reproduce the single-GPU bits): ~256 down tiles at small
    batches, round(f/2d) at large ones; the workspace for max_tokens covers
    every smaller batch's layout."""
    from paper_2605_23911_b200 import _lib

    lib = _lib.load()

    def splits(e, k, d, f, b):
        c = _lib.config_struct(e, k, d, f, 0)
        s = ctypes.c_int(0)
        assert lib.moe_b200_down_splits(ctypes.byref(c), b, ctypes.byref(s)) == 0
        return s.value

    mixtral = (8, 2, 4096, 14336)
    assert [splits(*mixtral, b) for b in (1, 2, 4, 8, 32, 512)] == [8, 5, 3, 2, 2, 2]
    assert splits(60, 4, 2048, 1408, 1) == 3 and splits(60, 4, 2048, 1408, 512) == 1
    assert splits(256, 8, 7168, 2048, 512) == 1
    prev = None
    for b in range(1, 600):  # non-increasing in the batch
        s = splits(*mixtral, b)
        assert prev is None or s <= prev
        prev = s
    n_max, n_b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    cfg = _lib.config_struct(*mixtral, 0)
    assert lib.moe_b200_workspace_size(ctypes.byref(cfg), 512, ctypes.byref(n_max)) == 0
    for b in (1, 2, 3, 5, 17, 300, 512):
        assert lib.moe_b200_workspace_size(ctypes.byref(cfg), b, ctypes.byref(n_b)) == 0
        assert n_b.value <= n_max.value


def test_status_codes_map_to_reference_exceptions():
    from paper_2605_23911_b200 import _lib, errors

    with pytest.raises(errors.ShapeMismatch):
        _lib.check(2, "x")
    with pytest.raises(errors.NonFiniteInput):
        _lib.check(1, "x")
    with pytest.raises(errors.InvalidK):
        _lib.check(3, "x")
    _lib.check(0, "x")


def test_product_package_never_imports_the_oracle():
    """The product package never imports, loads or executes the repo's oracle/
    (test infrastructure).  verify.py uses the REFERENCE package's own
    dense_moe_oracle as its checker, which is allowed."""
    pkg = os.path.join(ROOT, "paper_2605_23911_b200")
    bad = re.compile(r"^\s*(from|import)\s+oracle\b|['\"]oracle[/.]|sys\.path.*oracle|\bmoe_oracle\b|\bcpu_baseline\b",
                     re.M)
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = re.sub(r"#.*|//.*", "", open(os.path.join(dirpath, fn)).read())
                assert not bad.search(src), (fn, bad.search(src))


def test_verify_cli_usage_errors_exit_2():
    """Usage errors map to exit code 2 like the reference CLI (cli.py:979-992)."""
    from paper_2605_23911_b200.verify import main
    assert main(["verify", "--model", "NoSuchModel"]) == 2
    assert main(["verify", "--experts", "4"]) == 2
    assert main(["verify", "--batch", "0"]) == 2
    assert main(["nope"]) == 2
