"""Exhaustive full-memory PKM scorer (numpy fp64) for TINY tables only.

TEST INFRASTRUCTURE ONLY.  Independent of oracle/pkm_oracle.c: it never
factorises the top-k.  It scores every one of the n = n_sub^2 slots,
c[f] = S_row[f // n_sub] + S_col[f % n_sub] (flat index
reading R2), and takes the first k slots in (c desc, f asc) order.  The
product-key top-k must equal this exhaustive top-k (
BASELINE.json north_star "the product-key top-k must equal exhaustive top-k
over all n_sub^2 slots").
"""
from __future__ import annotations

import numpy as np


def _f64(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def forward(Q, K, V, k: int):
    """Returns idx [B,H,k], c [B,H,k], w [B,H,k], out [B,d_v] (fp64)."""
    q, kk, v = _f64(Q), _f64(K), _f64(V)
    B, H, _, d_h = q.shape
    n_sub = kk.shape[2]
    assert n_sub <= 64, "brute force is for tiny tables only"
    idx = np.empty((B, H, k), np.int64)
    c = np.empty((B, H, k), np.float64)
    w = np.empty((B, H, k), np.float64)
    out = np.zeros((B, v.shape[1]), np.float64)
    flat = np.arange(n_sub * n_sub, dtype=np.int64)
    for b in range(B):
        for h in range(H):
            s_row = kk[h, 0] @ q[b, h, 0]          # library matvec as a step
            s_col = kk[h, 1] @ q[b, h, 1]
            allc = (s_row[:, None] + s_col[None, :]).reshape(-1)
            order = np.lexsort((flat, -allc))       # primary: c desc, secondary: f asc
            sel = order[:k]
            idx[b, h] = sel
            c[b, h] = allc[sel]
            e = np.exp(allc[sel] - allc[sel].max())
            w[b, h] = e / e.sum()
            out[b] += w[b, h] @ v[sel]
    return {"idx": idx, "c": c, "w": w, "out": out}
