"""ctypes loader for libmsn_pkm.so (the C ABI of include/msn_pkm.h).

Argument marshalling only.  There is no fallback: if the CUDA library is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MSN_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("MSN_LIB", os.path.join(_HERE, "libmsn_pkm.so"))

ABI_VERSION = 2
MAX_WORLD = 8
MSN_F32, MSN_BF16 = 0, 1
FLAG_ATOMIC_BWD = 0x1
FLAG_GROUP_TABLES = 0x2
FLAG_DQ_QK_DTYPE = 0x4
FLAG_VALIDATE = 0x8
GATES = {"tanh": 1, "sigmoid": 2, "identity": 3}  # msn_gate (include/msn_pkm.h)
UPDATES = {"sgd": 1, "adagrad": 2}                # msn_update

STATUS = {0: "MSN_OK", 1: "MSN_ERR_INVALID_ARG", 2: "MSN_ERR_UNSUPPORTED", 3: "MSN_ERR_CUDA",
          5: "MSN_ERR_WORKSPACE", 6: "MSN_ERR_INTERNAL"}


class MsnError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("heads", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("d_half", ctypes.c_int32),
                ("d_value", ctypes.c_int32), ("k", ctypes.c_int32),
                ("max_batch", ctypes.c_int64), ("qk_dtype", ctypes.c_int32),
                ("value_dtype", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("head_groups", ctypes.c_int32), ("row_begin", ctypes.c_int64),
                ("row_end", ctypes.c_int64), ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32)]


# msn_pkm_exchange (a9, the row-sharded table's record exchange)
XCHG_PEER, XCHG_STAGED = 0, 1
XREG = ["IN_ROW", "IN_W", "IN_CNT", "PART_IN", "DOUT", "DW_IN", "POS", "CTL",
        "OUT_ROW", "OUT_W", "OUT_CNT", "PART_OUT", "DOUT_ALL", "DW_OUT"]


class Exchange(ctypes.Structure):
    _fields_ = [("transport", ctypes.c_int32), ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("local_batch", ctypes.c_int64), ("base", ctypes.c_void_p * MAX_WORLD)]


# name -> argtypes (all return msn_status except where noted)
_P, _I64, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
SIGNATURES = {
    "msn_pkm_create": [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_void_p)],
    "msn_pkm_destroy": [_P],
    "msn_pkm_workspace_size": [_P, _I64, _I64, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ)],
    "msn_pkm_forward": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_forward_qln": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_forward_gated": [_P, _P, _I64, _P, _P, _P, _P, ctypes.c_int32, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_gate_backward": [_P, _P, _I64, ctypes.c_int32, _P, _P, _P, _P, _P],
    "msn_pkm_layernorm": [_P, _P, _I64, _P, _P],
    "msn_pkm_layernorm_backward": [_P, _P, _I64, _P, _P, _P],
    "msn_pkm_key_transform": [_P, _P, _P, _P, _P],
    "msn_pkm_key_transform_backward": [_P, _P, _P, _P, _P, _P, _P],
    "msn_pkm_scatter_update": [_P, _P, _I64, _P, _P, _P, _P, ctypes.c_int32, ctypes.c_float,
                               ctypes.c_float, _P, _P, _P, _SZ],
    "msn_pkm_backward": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_select": [_P, _P, _I64, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_gather": [_P, _P, _I64, _P, _P, _P, _P],
    "msn_pkm_exchange_layout": [_P, _I64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_SZ)],
    "msn_pkm_forward_sharded": [_P, _P, _I64, _P, _P, _P, ctypes.POINTER(Exchange), _P, _P, _P, _P, _SZ],
    "msn_pkm_backward_sharded": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, ctypes.POINTER(Exchange), _P, _P, _P,
                                 _P, _P, _SZ],
    "msn_pkm_exchange_select": [_P, _P, _P, _P, _P, ctypes.POINTER(Exchange), _P, _P, _P, _P, _SZ],
    "msn_pkm_exchange_gather": [_P, _P, _P, ctypes.POINTER(Exchange)],
    "msn_pkm_exchange_combine": [_P, _P, ctypes.POINTER(Exchange), _P],
    "msn_pkm_exchange_scatter": [_P, _P, _P, _P, ctypes.POINTER(Exchange), _P, _SZ],
    "msn_pkm_exchange_collect": [_P, _P, _P, ctypes.POINTER(Exchange), _P],
    "msn_pkm_exchange_barrier": [_P, _P, ctypes.POINTER(Exchange)],
    "msn_pkm_validate_tape": [_P, _P, _I64, _P, _P, _P],
    "msn_pkm_scatter": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_backward_keys": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ],
    "msn_pkm_last_launch_count": [_P],
    "msn_pkm_set_trace_events": [_P, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32],
    "msn_pkm_status_string": [ctypes.c_int],
    "msn_pkm_last_error": [],
}
_RESTYPE = {"msn_pkm_last_launch_count": ctypes.c_int32,
            "msn_pkm_status_string": ctypes.c_char_p,
            "msn_pkm_last_error": ctypes.c_char_p}

_lib = None


def load(path: str = LIB_PATH):
    """Load the library (raises if absent: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run __graft_entry__.build() "
                               "(the PKM path has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def check(status: int):
    if status != 0:
        detail = load().msn_pkm_last_error().decode(errors="replace")
        raise MsnError(status, detail)
