"""Fused sparse optimiser update in fp64 -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's Sparse-Gather op "fuses sparse access, weight computation, and
gradient updates into a unified kernel" (sec. 3.6).  Reading
R20: the update is applied to the touched value rows only, with
g_r = dV[r] = sum over the contributions to row r of w * d_out[b] (the value
gradient the backward computes, PAPER.md:229 differentiated):

    SGD      V[r] <- V[r] - lr * g_r
    Adagrad  s[r] <- s[r] + g_r^2 ;  V[r] <- V[r] - lr * g_r / (sqrt(s[r]) + eps)

elementwise; untouched rows and their state are left alone (the sparse /
lazy form of both optimisers).  Plain numpy on the oracle's dV rows.
"""
from __future__ import annotations

import numpy as np

UPDATES = ("sgd", "adagrad")


def apply(V, rows: np.ndarray, dV_rows: np.ndarray, kind: str, lr: float, eps: float = 1e-10,
          state=None):
    """V [n, d_v] (any float, widened to fp64), rows [m] unique touched row ids,
    dV_rows [m, d_v] their gradients.  Returns (V_new fp64, state_new fp64 or None)."""
    Vn = np.array(V, dtype=np.float64, copy=True)
    g = np.asarray(dV_rows, dtype=np.float64)
    rows = np.asarray(rows, dtype=np.int64)
    if kind == "sgd":
        Vn[rows] -= lr * g
        return Vn, None
    if kind == "adagrad":
        s = np.array(state, dtype=np.float64, copy=True)
        s[rows] += g * g
        Vn[rows] -= lr * g / (np.sqrt(s[rows]) + eps)
        return Vn, s
    raise ValueError(kind)
