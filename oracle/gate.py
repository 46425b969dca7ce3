"""Memory-gated fusion in fp64 -- TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).

    x~ = x_in (.) g(v_o)        Eq. gating, PAPER.md:318-322 [sec. 3.5]

with g = tanh (the paper's choice) or, as in the gating
ablation, sigmoid or the identity ("removing the activation entirely",
PAPER.md:492).  v_o is the memory output (the PKM lookup's out, summed over
heads, reading R7); x_in has the same width.  For a loss with upstream
gradient dx~ (product rule, elementwise):

    dx_in = dx~ (.) g(v_o)
    dv_o  = dx~ (.) x_in (.) g'(v_o),   g' = 1 - tanh^2 | s (1 - s) | 1

dv_o is the d_out that the PKM backward consumes.  Plain numpy, elementwise.
"""
from __future__ import annotations

import numpy as np

GATES = ("tanh", "sigmoid", "identity")


def _g(v: np.ndarray, gate: str) -> np.ndarray:
    if gate == "tanh":
        return np.tanh(v)
    if gate == "sigmoid":
        return 1.0 / (1.0 + np.exp(-v))
    if gate == "identity":
        return v.copy()
    raise ValueError(gate)


def _dg(v: np.ndarray, gate: str) -> np.ndarray:
    if gate == "tanh":
        t = np.tanh(v)
        return 1.0 - t * t
    if gate == "sigmoid":
        s = 1.0 / (1.0 + np.exp(-v))
        return s * (1.0 - s)
    if gate == "identity":
        return np.ones_like(v)
    raise ValueError(gate)


def _f64(a) -> np.ndarray:
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a, dtype=np.float64)


def forward(v_o, x_in, gate: str = "tanh") -> np.ndarray:
    """x~ = x_in * g(v_o)."""
    v, x = _f64(v_o), _f64(x_in)
    assert v.shape == x.shape
    return x * _g(v, gate)


def backward(v_o, x_in, d_xt, gate: str = "tanh"):
    """-> (dx_in, dv_o) for the upstream gradient d_xt."""
    v, x, d = _f64(v_o), _f64(x_in), _f64(d_xt)
    assert v.shape == x.shape == d.shape
    return d * _g(v, gate), d * x * _dg(v, gate)
