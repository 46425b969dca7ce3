"""ctypes wrapper around oracle/pkm_oracle.c (fp64 PKM oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Inputs are numpy arrays
or CPU torch tensors holding the exact stored values (fp32, bf16 or fp64);
bf16 tensors are passed as their raw 16-bit patterns and widened in C.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pkm_oracle.c")
_LIB = os.path.join(_HERE, "libpkm_oracle.so")

DT_F32, DT_BF16, DT_F64 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        _lib.pkm_oracle_forward.argtypes = [I64, I32, I32, I32, I32, I32,
                                            P, I32, P, I32, P, I32,
                                            P, P, P, P, P, P, P, P, P, I32]
        _lib.pkm_oracle_forward.restype = I32
        _lib.pkm_oracle_slot_scores.argtypes = [I64, I32, I32, I32, P, I32, P, I32, P, I32, P, I32]
        _lib.pkm_oracle_slot_scores.restype = I32
        _lib.pkm_oracle_backward.argtypes = [I64, I32, I32, I32, I32, I32,
                                             P, I32, P, I32, P, I32,
                                             P, P, P, P, P, P, I64, P, P, I32]
        _lib.pkm_oracle_backward.restype = I32
    return _lib


def _as_stored(x):
    """-> (contiguous numpy array of the stored bits, dtype code)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().contiguous()
            if x.dtype == torch.bfloat16:
                return x.view(torch.int16).numpy().view(np.uint16), DT_BF16
            if x.dtype == torch.float32:
                return x.numpy(), DT_F32
            if x.dtype == torch.float64:
                return x.numpy(), DT_F64
            raise TypeError(f"unsupported dtype {x.dtype}")
    except ImportError:  # pragma: no cover
        pass
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return x, DT_F32
    if x.dtype == np.float64:
        return x, DT_F64
    if x.dtype == np.uint16:
        return x, DT_BF16
    raise TypeError(f"unsupported dtype {x.dtype}")


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _threads(nthreads):
    return int(nthreads) if nthreads else len(os.sched_getaffinity(0))


def forward(Q, K, V, k: int, nthreads: int = 0, per_head: bool = False):
    """PKM forward (pkm_oracle_forward).  Q [B,H,2,d_h], K [H,2,n_sub,d_h],
    V [n_sub^2, d_v].  Returns a dict of fp64 / int64 numpy arrays:
    I, J, s1, s2 (per-half top-k), idx, c, w [B,H,k], out [B,d_v]
    (and out_ph [B,H,d_v] when per_head)."""
    q, qdt = _as_stored(Q)
    kk, kdt = _as_stored(K)
    v, vdt = _as_stored(V)
    B, H, two, d_h = q.shape
    assert two == 2 and kk.shape[0] == H and kk.shape[1] == 2 and kk.shape[3] == d_h
    n_sub = kk.shape[2]
    d_v = v.shape[1]
    assert v.shape[0] == n_sub * n_sub
    r = {name: np.empty((B, H, k), np.int64) for name in ("I", "J", "idx")}
    r.update({name: np.empty((B, H, k), np.float64) for name in ("s1", "s2", "c", "w")})
    r["out"] = np.empty((B, d_v), np.float64)
    r["out_ph"] = np.empty((B, H, d_v), np.float64) if per_head else None
    rc = lib().pkm_oracle_forward(B, H, n_sub, d_h, d_v, k, _p(q), qdt, _p(kk), kdt, _p(v), vdt,
                                  _p(r["I"]), _p(r["J"]), _p(r["s1"]), _p(r["s2"]),
                                  _p(r["idx"]), _p(r["c"]), _p(r["w"]), _p(r["out"]),
                                  _p(r["out_ph"]), _threads(nthreads))
    if rc != 0:
        raise ValueError(f"pkm_oracle_forward failed ({rc})")
    return r


def slot_scores(Q, K, slots: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """fp64 S1[i]+S2[j] for slots [B,H,m] (flat ids i*n_sub+j)."""
    q, qdt = _as_stored(Q)
    kk, kdt = _as_stored(K)
    B, H, _, d_h = q.shape
    n_sub = kk.shape[2]
    s = np.ascontiguousarray(slots, dtype=np.int64)
    assert s.shape[:2] == (B, H)
    out = np.empty(s.shape, np.float64)
    rc = lib().pkm_oracle_slot_scores(B, H, n_sub, d_h, _p(q), qdt, _p(kk), kdt, _p(s), s.shape[2],
                                      _p(out), _threads(nthreads))
    if rc != 0:
        raise ValueError("pkm_oracle_slot_scores failed")
    return out


def backward(Q, K, V, idx: np.ndarray, dOut, rows: Optional[np.ndarray] = None,
             nthreads: int = 0, want_dense_dv: bool = True):
    """PKM backward at the selection idx [B,H,k] for L = <dOut, out>.
    Returns dict dQ [B,H,2,d_h], dK [H,2,n_sub,d_h], dV (compact [len(rows),d_v]
    over the sorted unique rows, or dense [n,d_v]), rows, dw, ds [B,H,k]."""
    q, qdt = _as_stored(Q)
    kk, kdt = _as_stored(K)
    v, vdt = _as_stored(V)
    B, H, _, d_h = q.shape
    n_sub = kk.shape[2]
    d_v = v.shape[1]
    ix = np.ascontiguousarray(idx, dtype=np.int64)
    k = ix.shape[2]
    try:
        import torch
        if isinstance(dOut, torch.Tensor):
            dOut = dOut.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    d = np.ascontiguousarray(dOut, dtype=np.float64)
    assert d.shape == (B, d_v)
    if rows is None and not want_dense_dv:
        rows = np.unique(ix)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        dV = np.empty((rows.shape[0], d_v), np.float64)
    else:
        dV = np.empty((n_sub * n_sub, d_v), np.float64)
    dQ = np.empty((B, H, 2, d_h), np.float64)
    dK = np.empty((H, 2, n_sub, d_h), np.float64)
    dw = np.empty((B, H, k), np.float64)
    ds = np.empty((B, H, k), np.float64)
    rc = lib().pkm_oracle_backward(B, H, n_sub, d_h, d_v, k, _p(q), qdt, _p(kk), kdt, _p(v), vdt,
                                   _p(ix), _p(d), _p(dQ), _p(dK), _p(dV), _p(rows),
                                   0 if rows is None else rows.shape[0], _p(dw), _p(ds),
                                   _threads(nthreads))
    if rc != 0:
        raise ValueError(f"pkm_oracle_backward failed ({rc})")
    return {"dQ": dQ, "dK": dK, "dV": dV, "rows": rows, "dw": dw, "ds": ds}
