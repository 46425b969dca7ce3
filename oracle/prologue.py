"""Query / key prologue of the lookup in fp64 --
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Layer normalisation of the query and sub-key vectors before the similarity
  computation (sec. 3.4.1): per row of width d,
      x_hat = (x - mean(x)) / sqrt(var(x) + eps),  var = mean((x - mean)^2),
  reading R23: no learned affine (gamma, beta) -- for the keys the
  over-parameterisation Theta that follows subsumes a per-feature scale --
  and eps = 1e-5.
* Key over-parameterisation: K_tilde = Theta K for each
  sub-key codebook, read per key vector k_tilde_i = Theta k_i with Theta a
  learned d x d matrix per (head, half) (SPEC's reading); the scores then use
  K_tilde.  Its gradients:
      dL/dTheta = sum_i dL/dk_tilde_i  k_i^T,    dL/dk_i = Theta^T dL/dk_tilde_i.
Row-major layouts: K [.., n_sub, d] (rows are key vectors), so
K_tilde = K Theta^T, dTheta = dK_tilde^T K, dK = dK_tilde Theta.
"""
from __future__ import annotations

import numpy as np

EPS = 1e-5


def _f64(a) -> np.ndarray:
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a, dtype=np.float64)


def layernorm(x, eps: float = EPS) -> np.ndarray:
    """LN over the last axis."""
    x = _f64(x)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


def layernorm_backward(x, dy, eps: float = EPS) -> np.ndarray:
    """dL/dx for y = layernorm(x) and dL/dy = dy (last axis)."""
    x, dy = _f64(x), _f64(dy)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    r = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * r
    return r * (dy - dy.mean(axis=-1, keepdims=True) - xh * (dy * xh).mean(axis=-1, keepdims=True))


def key_transform(K, theta) -> np.ndarray:
    """K [H, 2, n_sub, d], theta [H, 2, d, d] -> K_tilde = K Theta^T per (h, half)."""
    K, T = _f64(K), _f64(theta)
    return np.einsum("hcid,hced->hcie", K, T)


def key_transform_backward(K, theta, dK_tilde):
    """-> (dK = dK_tilde Theta, dTheta = dK_tilde^T K) per (h, half)."""
    K, T, G = _f64(K), _f64(theta), _f64(dK_tilde)
    dK = np.einsum("hcie,hced->hcid", G, T)
    dT = np.einsum("hcie,hcid->hced", G, K)
    return dK, dT
