"""ctypes binding of libmoe_b200.so (the C-ABI in include/moe_b200.h).

There is deliberately no fallback: if the library is missing or fails to
load, every entry point raises ``NativeLibraryMissing``.  Status codes map
onto the reference's exception classes (``moeperf/errors.py:9-50``).
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

LIB_NAME = "libmoe_b200.so"
LIB_PATH = os.environ.get("MOE_B200_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OK = 0
STATUS_TO_EXC = {
    1: errors.NonFiniteInput,
    2: errors.ShapeMismatch,
    3: errors.InvalidK,
    4: errors.IndexOutOfRange,
    5: errors.InvalidBlockM,
    6: errors.ScheduleMismatch,
    7: ValueError,
    8: errors.DeviceError,
    9: errors.DeviceError,
    10: errors.DeviceError,
    11: errors.DeviceError,
}

DTYPE_F32 = 0
DTYPE_BF16 = 1


class Config(ctypes.Structure):
    _fields_ = [
        ("num_experts", ctypes.c_int32),
        ("top_k", ctypes.c_int32),
        ("hidden_dim", ctypes.c_int32),
        ("ffn_dim", ctypes.c_int32),
        ("gating", ctypes.c_int32),
    ]


EP_MAX_RANKS = 16


class EpPeers(ctypes.Structure):
    """moe_b200_ep_peers: per-rank buffer pointers mapped in this process."""
    _fields_ = [
        ("counts", ctypes.c_void_p * EP_MAX_RANKS),
        ("flags", ctypes.c_void_p * EP_MAX_RANKS),
        ("rows", ctypes.c_void_p * EP_MAX_RANKS),
        ("ids", ctypes.c_void_p * EP_MAX_RANKS),
        ("home", ctypes.c_void_p * EP_MAX_RANKS),
        ("expert_lo", ctypes.c_int32 * (EP_MAX_RANKS + 1)),
        ("n", ctypes.c_int32),
        ("me", ctypes.c_int32),
        ("epoch_dev", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_CFG = ctypes.POINTER(Config)
_SZ = ctypes.c_size_t

#: symbol -> (restype, argtypes); every symbol declared in include/moe_b200.h
_PEERS = ctypes.POINTER(EpPeers)
_U64 = ctypes.c_uint64
SIGNATURES = {
    "moe_b200_ipc_alloc": (_INT, [_SZ, ctypes.POINTER(_P), _P]),
    "moe_b200_ipc_open": (_INT, [_P, ctypes.POINTER(_P)]),
    "moe_b200_ipc_close": (_INT, [_P]),
    "moe_b200_ipc_free": (_INT, [_P]),
    "moe_b200_ep_p2p_counts": (_INT, [_CFG, _I64, _P, _PEERS, _U64, _P]),
    "moe_b200_ep_p2p_wait": (_INT, [_PEERS, _INT, _U64, _P]),
    "moe_b200_ep_p2p_dispatch": (_INT, [_CFG, _I64, _P, _P, _P, _P, _PEERS, _P, _U64, _P]),
    "moe_b200_ep_p2p_return": (_INT, [_CFG, _I64, _P, _PEERS, _P, _U64, _P]),
    "moe_b200_ep_p2p_ffn_return_async": (_INT, [_CFG, _I64, ctypes.c_int, _P, _P, _P, _P, _PEERS, _P, _U64, _P,
                                                _SZ, _P]),
    "moe_b200_ep_p2p_ffn_return": (_INT, [_CFG, _I64, ctypes.c_int, _P, _P, _P, _P, _P, _PEERS, _P, _U64, _P,
                                          _SZ, _P]),
    "moe_b200_workspace_size": (_INT, [_CFG, _I64, ctypes.POINTER(_SZ)]),
    "moe_b200_workspace_init": (_INT, [_CFG, _I64, _P, _SZ, _P]),
    "moe_b200_route": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_permute": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P]),
    "moe_b200_gate_up": (_INT, [_CFG, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_down_scatter": (_INT, [_CFG, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_combine": (_INT, [_CFG, _I64, _P, _P, _INT, _P]),
    "moe_b200_forward": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_forward_unfused": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _P, _P, _P,
                                        _SZ, _P]),
    "moe_b200_forward_routed": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _P,
                                       _SZ, _P]),
    "moe_b200_forward_timed": (_INT, [_CFG, _I64, _P, _INT, _P, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _P, _P, _P, _SZ, _P,
                                      ctypes.POINTER(ctypes.c_void_p)]),
    "moe_b200_expert_ffn": (_INT, [_CFG, _I64, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_expert_ffn_workspace_size": (_INT, [_CFG, _I64, ctypes.c_int, ctypes.POINTER(_SZ)]),
    "moe_b200_down_splits": (_INT, [_CFG, _I64, ctypes.POINTER(ctypes.c_int)]),
    "moe_b200_gather_rows": (_INT, [_I64, _I64, _P, _P, _P, _P]),
    "moe_b200_combine_rows": (_INT, [_CFG, _I64, _P, _P, _P, _P, _INT, _P]),
    "moe_b200_read_flags": (_INT, [_CFG, _I64, _P, _SZ, ctypes.POINTER(ctypes.c_uint32), _P]),
    "moe_b200_io_create": (_INT, [_CFG, _I64, _INT, _INT, ctypes.POINTER(ctypes.c_void_p)]),
    "moe_b200_io_destroy": (_INT, [_P]),
    "moe_b200_forward_host": (_INT, [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_io_record": (_INT, [_P, _P]),
    "moe_b200_io_wait": (_INT, [_P, _P]),
    "moe_b200_launches_per_forward": (_INT, [_CFG, _I64]),
    "moe_b200_io_sync": (_INT, [_P]),
    "moe_b200_tuning_reload": (_INT, []),
    "moe_b200_record_event": (_INT, [_P, _P]),
    "moe_b200_combine_overlapped": (_INT, [_CFG, _I64]),
    "moe_b200_gate_scores": (_INT, [_I64, _INT, _INT, _P, _P, _P, _P]),
    "moe_b200_topk_select": (_INT, [_I64, _INT, _INT, _INT, _P, _P, _P, _P]),
    "moe_b200_sigmoid": (_INT, [_I64, _P, _P, _INT, _P]),
    "moe_b200_dense_matmul": (_INT, [_I64, _I64, _I64, _P, _P, _P, _P]),
    "moe_b200_np_exp64": (_INT, [_I64, _P, _P, _P]),
    "moe_b200_schedule": (_INT, [_CFG, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_permute_rows": (_INT, [_I64, _I64, _P, _P, _INT, _P, _P]),
    "moe_b200_cast_bf16": (_INT, [_I64, _P, _P, _P]),
    "moe_b200_grouped_gate_up": (_INT, [_CFG, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_grouped_gemm": (_INT, [_CFG, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "moe_b200_swiglu": (_INT, [_I64, _P, _P, _P]),
    "moe_b200_strerror": (ctypes.c_char_p, [_INT]),
    "moe_b200_last_error_detail": (ctypes.c_char_p, []),
    "moe_b200_version": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the ctypes library handle."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise errors.NativeLibraryMissing(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        try:
            lib = ctypes.CDLL(p)
        except OSError as exc:  # pragma: no cover - environment specific
            raise errors.NativeLibraryMissing(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int, what: str) -> None:
    """Raise the reference exception class for a non-zero status."""
    if status == OK:
        return
    lib = load()
    msg = lib.moe_b200_strerror(status).decode()
    detail = lib.moe_b200_last_error_detail().decode()
    exc = STATUS_TO_EXC.get(status, errors.DeviceError)
    raise exc(f"{what}: {msg}" + (f" ({detail})" if detail else ""))


def reload_tuning() -> None:
    """Re-read the MOE_B200_* tuning / test hooks (the library reads them once,
    and at every workspace init, never on the forward path)."""
    check(load().moe_b200_tuning_reload(), "tuning_reload")


def config_struct(num_experts, top_k, hidden_dim, ffn_dim, gating_code) -> Config:
    return Config(num_experts, top_k, hidden_dim, ffn_dim, gating_code)
