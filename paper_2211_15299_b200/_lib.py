"""ctypes binding of the C-ABI in include/structfft_b200.h.

This is the binding a maintainer of the reference would add.
The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute call raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (BudgetExceededError, ContractViolationError, DeviceError,
                     InvalidInputError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFFT_LIB") or os.path.join(_HERE, "libsfft_b200.so")

OK, ERR_INVALID, ERR_CONTRACT, ERR_BUDGET, ERR_CUDA, ERR_UNSUPPORTED = 0, 2, 3, 4, 5, 6
C64, C128 = 0, 1
OUT_NODES, OUT_DFT, OUT_SAS, OUT_SLOTS = 0, 1, 2, 3
ORDER_SLOT, ORDER_PATTERN = 0, 1

_c = ctypes
_P = _c.c_void_p
_I64 = _c.c_int64
_I32 = _c.c_int32


class PlanInfo(_c.Structure):
    _fields_ = [("M", _c.c_int), ("dtype", _c.c_int), ("n_r", _c.c_int), ("height", _c.c_int),
                ("s", _c.c_int), ("level", _c.c_int), ("homogeneous", _c.c_int),
                ("per_signal", _c.c_int), ("k", _I64), ("A", _I64), ("n_nodes", _I64),
                ("mu_star", _I64), ("pivot_mask", _c.c_uint64), ("used", _I32 * 32)]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = [
    ("sfft_version", _c.c_char_p, []),
    ("sfft_last_error", _c.c_char_p, []),
    ("sfft_device_ok", _c.c_int, []),
    ("sfft_analyze", _c.c_int, [_P, _I64, _c.c_int, _P, _P, _P]),
    ("sfft_pivoted_pattern", _c.c_int, [_P, _c.c_int, _c.c_int, _P, _P]),
    ("sfft_plan_create", _c.c_int, [_P, _I64, _c.c_int, _P, _c.c_int, _c.c_int, _c.c_int, _P,
                                    _c.POINTER(_P)]),
    ("sfft_plan_destroy", _c.c_int, [_P]),
    ("sfft_plan_get_info", _c.c_int, [_P, _c.POINTER(PlanInfo)]),
    ("sfft_plan_tables", _c.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    ("sfft_hidft", _c.c_int, [_P, _P, _I64, _I64, _I64, _c.c_int, _P, _I64, _P, _I64, _P]),
    ("sfft_hidft_gathered", _c.c_int, [_P, _P, _I64, _I64, _c.c_int, _P, _I64, _P, _I64, _P]),
    ("sfft_plan_apply_map", _c.c_int, [_P, _c.c_int, _P, _I64, _I64, _P, _I64, _P]),
    ("sfft_synthesize", _c.c_int, [_P, _P, _I64, _c.c_int, _P, _I64, _P, _P]),
    ("sfft_prefix_weights", _c.c_int, [_P, _I64, _c.c_int, _P, _c.c_int, _P, _P, _P]),
    ("sfft_plan_nodes", _c.c_int, [_P, _P, _P, _P]),
    ("sfft_tree_build", _c.c_int, [_P, _I64, _c.c_int, _c.c_int, _c.c_int, _P, _P, _P, _P]),
    ("sfft_hidft_shifts", _c.c_int, [_P, _P, _I64, _I64, _c.c_int, _I64, _I64, _c.c_int, _P, _I64, _P]),
    ("sfft_sas_decode", _c.c_int, [_P, _P, _I64, _c.c_int, _I64, _I64, _c.c_double, _P, _I64, _c.c_int, _P, _P,
                                   _P, _I64, _P, _P, _I64, _P, _P, _P, _P, _P]),
    ("sfft_host_gather", _c.c_int, [_P, _I64, _I64, _c.c_int, _P, _I64, _P, _c.c_int]),
    ("sfft_plan_batched", _c.c_int, [_P, _I64, _I64, _c.c_int, _c.c_int, _P, _P]),
    ("sfft_launch_count", _c.c_int, [_P, _I64, _P]),
    ("sfft_hidft_interleaved", _c.c_int, [_P, _P, _I64, _I64, _I64, _c.c_int, _P, _I64, _P]),
    ("sfft_stream_chain", _c.c_int, [_P, _c.c_int]),
    ("sfft_hidft_to_dft_fused_host", _c.c_int, [_P, _I64, _c.c_int, _P, _I64, _I64, _c.c_int, _P, _I64,
                                                _c.c_int, _P]),
    ("sfft_hidft_host", _c.c_int, [_P, _P, _I64, _I64, _I64, _c.c_int, _P, _I64, _P, _I64, _I64, _c.c_int, _P]),
    ("sfft_host_stage", _c.c_int, [_P, _P, _I64, _I64, _c.c_int, _I64, _I64, _c.c_int, _c.c_int, _P, _I64,
                                   _c.c_int, _P]),
    ("sfft_hidft_staged", _c.c_int, [_P, _P, _I64, _I64, _c.c_int, _c.c_int, _P, _I64, _P, _I64, _P]),
    ("sfft_hidft_to_dft_fused", _c.c_int, [_P, _I64, _I64, _c.c_int, _P, _I64, _I64, _c.c_int, _P,
                                           _I64, _P, _P]),
    ("sfft_probe_fma_peak", _c.c_int, [_c.c_int, _c.POINTER(_c.c_double), _P]),
    ("sfft_peer_alloc", _c.c_int, [_I64, _c.POINTER(_P), _P]),
    ("sfft_peer_free", _c.c_int, [_P]),
    ("sfft_peer_open", _c.c_int, [_P, _c.POINTER(_P)]),
    ("sfft_peer_close", _c.c_int, [_P]),
]
IPC_HANDLE_BYTES = 64

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (no GPU needed); raise DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = _c.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().sfft_last_error().decode(errors="replace")
    if rc == ERR_INVALID:
        raise InvalidInputError(msg)
    if rc == ERR_CONTRACT:
        raise ContractViolationError(msg)
    if rc == ERR_BUDGET:
        raise BudgetExceededError(msg)
    raise DeviceError(f"status {rc}: {msg}")


def require_device():
    """The torch device this call runs on; fails loudly without a B200."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("structfft_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return t.data_ptr()
