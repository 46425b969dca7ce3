"""GPU-vs-oracle comparator (test infrastructure).

The bar (BASELINE.json north_star):
* selected indices identical, except at ties, where any swapped slot must
  have a score gap <= 1e-5 relative (scores from the oracle's fp64
  slot_scores of both slots);
* outputs and gradients within 1e-4 relative for fp32 values, 2e-2 for bf16
  values, measured per row as  max_e |g - o| <= rtol * scale_row, where
  scale_row = max(max_e |o_row|, max_e A_row, 1e-6 max |o|) and A is the sum
  of the absolute values of the terms the oracle adds up for that element
  (grad_key_magnitudes) -- "relative" to the
  magnitude of what is summed, so a row whose terms cancel to ~0 is not held
  to an impossible bound (reading R14).
Lookups whose selection legitimately differs at a tie are excluded from the
element-wise value comparison (their expected values would otherwise have to
come from the CUDA path's selection); everything they touch is masked and
their number is bounded.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as orc

TIE_REL = 1e-5


def rtol_for(value_dtype) -> float:
    return 1e-4 if value_dtype == torch.float32 else 2e-2


def compare_selection(Q, K, gpu_idx: np.ndarray, o: dict, n_sub: int):
    """Returns (affected lookup mask [B,H], report dict).  Raises on a swap
    that is not a tie."""
    g = np.asarray(gpu_idx, dtype=np.int64)
    oi = o["idx"]
    assert g.shape == oi.shape
    n = n_sub * n_sub
    assert g.min() >= 0 and g.max() < n, "index out of range"
    B, H, k = g.shape
    # distinct within a lookup
    srt = np.sort(g, axis=-1)
    assert np.all(srt[..., 1:] != srt[..., :-1]), "duplicate slot within a lookup"
    diff = np.any(g != oi, axis=-1)
    affected = np.zeros((B, H), bool)
    worst = 0.0
    if diff.any():
        bs, hs = np.nonzero(diff)
        # fp64 scores of the GPU's slots for the differing lookups
        gs = orc.slot_scores(Q, K, g)
        for b, h in zip(bs, hs):
            G, O = set(g[b, h].tolist()), set(oi[b, h].tolist())
            gsc = dict(zip(g[b, h].tolist(), gs[b, h].tolist()))
            osc = dict(zip(oi[b, h].tolist(), o["c"][b, h].tolist()))
            if G == O:
                # same set, order swapped: the swapped neighbours must tie
                for t in range(k):
                    if g[b, h, t] != oi[b, h, t]:
                        x, y = gsc[g[b, h, t]], osc[oi[b, h, t]]
                        rel = abs(x - y) / max(abs(x), abs(y), 1e-300)
                        worst = max(worst, rel)
                        assert rel <= TIE_REL, f"order swap at ({b},{h},{t}) not a tie: {x} vs {y}"
            else:
                for xs in G - O:
                    for ys in O - G:
                        x, y = gsc[xs], osc[ys]
                        rel = abs(x - y) / max(abs(x), abs(y), 1e-300)
                        worst = max(worst, rel)
                        assert rel <= TIE_REL, (f"lookup ({b},{h}): slot {xs} (score {x}) selected "
                                                f"instead of {ys} (score {y}), gap {rel:.3g} > 1e-5")
            affected[b, h] = True
    return affected, {"differing_lookups": int(diff.sum()), "worst_tie_gap": worst}


def row_close(gpu: np.ndarray, ref: np.ndarray, rtol: float, row_mask=None, what="", absmag=None):
    """Per-row relative check; rows where row_mask is False are skipped.
    absmag (same shape as ref) is the sum of |terms| behind each element."""
    g = np.asarray(gpu, dtype=np.float64).reshape(gpu.shape[0], -1)
    r = np.asarray(ref, dtype=np.float64).reshape(ref.shape[0], -1)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    floor = 1e-6 * np.abs(r).max() + 1e-300
    a = None if absmag is None else np.asarray(absmag, dtype=np.float64).reshape(r.shape)
    if row_mask is not None:
        g, r = g[row_mask], r[row_mask]
        a = None if a is None else a[row_mask]
    if g.size == 0:
        return 0.0
    scale = np.maximum(np.abs(r).max(axis=1), floor)
    if a is not None:
        scale = np.maximum(scale, a.max(axis=1))
    err = np.abs(g - r).max(axis=1) / scale
    worst = float(err.max())
    assert worst <= rtol, f"{what}: worst row-relative error {worst:.3g} > {rtol}"
    return worst


def plain_row_err(gpu: np.ndarray, ref: np.ndarray, row_mask=None) -> float:
    """SURVEY.md 8(c)'s plain metric: per row  max_e |g - o| / max(max_e |o_row|,
    1e-6 max |o|), worst row (reported next to the condition-aware one)."""
    g = np.asarray(gpu, dtype=np.float64).reshape(gpu.shape[0], -1)
    r = np.asarray(ref, dtype=np.float64).reshape(ref.shape[0], -1)
    floor = 1e-6 * np.abs(r).max() + 1e-300
    if row_mask is not None:
        g, r = g[row_mask], r[row_mask]
    if g.size == 0:
        return 0.0
    return float((np.abs(g - r).max(axis=1) / np.maximum(np.abs(r).max(axis=1), floor)).max())


def grad_key_magnitudes(Q, K, o, bw, n_sub):
    """Sum of |terms| behind each element of dQ and dK.  ds_t = w_t dw_t -
    w_t sum_u w_u dw_u has magnitude A_t = w_t (|dw_t| + sum_u w_u |dw_u|);
    dQ[b,h,half] = sum_t ds_t K[h,half,r_t] -> sum_t A_t |K[h,half,r_t]|;
    dK[h,half,r] = sum_{b,t: r_t=r} ds_t q[b,h,half] -> sum A_t |q|."""
    Kf = K.double().numpy() if isinstance(K, torch.Tensor) else np.asarray(K, np.float64)
    Qf = Q.double().numpy() if isinstance(Q, torch.Tensor) else np.asarray(Q, np.float64)
    w, dw = o["w"], bw["dw"]
    A = w * (np.abs(dw) + (w * np.abs(dw)).sum(-1, keepdims=True))
    H = Kf.shape[0]
    i_t, j_t = o["idx"] // n_sub, o["idx"] % n_sub
    hh = np.arange(H)[None, :, None]
    absq = np.stack([(A[..., None] * np.abs(Kf[hh, 0, i_t])).sum(2),
                     (A[..., None] * np.abs(Kf[hh, 1, j_t])).sum(2)], axis=2)
    absk = np.zeros_like(Kf)
    for half, r_t in ((0, i_t), (1, j_t)):
        for h in range(H):
            np.add.at(absk[h, half], r_t[:, h].reshape(-1),
                      (A[:, h, :, None] * np.abs(Qf[:, h, half][:, None, :])).reshape(-1, Kf.shape[-1]))
    return absq, absk


def check_forward(Q, K, V, k, out, idx, w, max_affected_frac=0.01):
    """Full forward parity for one call; returns (oracle result, affected, report)."""
    n_sub = K.shape[2]
    o = orc.forward(Q, K, V, k)
    gi = idx.detach().cpu().numpy().astype(np.int64)
    affected, rep = compare_selection(Q, K, gi, o, n_sub)
    B, H = affected.shape
    assert affected.sum() <= max(2, max_affected_frac * B * H), f"too many tie-affected lookups: {rep}"
    rtol = rtol_for(V.dtype)
    ok_b = ~affected.any(axis=1)
    rep["out_err"] = row_close(out.detach().cpu().numpy(), o["out"], rtol, ok_b, "out")
    wl = w.detach().cpu().numpy().reshape(B * H, k)
    rep["w_err"] = row_close(wl, o["w"].reshape(B * H, k), rtol, (~affected).reshape(-1), "weights")
    # softmax invariants on every lookup (including tie-affected ones)
    wf = w.detach().cpu().double().numpy()
    assert np.all(np.abs(wf.sum(-1) - 1.0) <= 1e-6), "sum of weights != 1"
    assert np.all(np.diff(wf, axis=-1) <= 1e-7), "weights not non-increasing"
    return o, affected, rep


def check_backward(Q, K, V, k, dOut, o, affected, dQ, dK, dV, dw=None, gpu_idx=None, assert_plain=False):
    """Backward parity at the oracle's own selection, masking tie-affected lookups.
    out, w, dw and dV are always held to the plain row-max metric; dQ and dK to
    the condition-aware one (R14), with the plain one reported and, with
    assert_plain, asserted too."""
    n_sub = K.shape[2]
    B, H = affected.shape
    bw = orc.backward(Q, K, V, o["idx"], dOut, want_dense_dv=False)
    rtol = rtol_for(V.dtype)
    # every output and gradient is held to the value dtype's tolerance
    # (north_star: "1e-4 relative for fp32 and 2e-2 relative for bf16 values")
    rtol_qk = rtol
    rep = {}
    absq, absk = grad_key_magnitudes(Q, K, o, bw, n_sub)
    # dQ rows: per (b,h,half)
    mask_q = np.repeat((~affected).reshape(-1), 2)
    dq_g = dQ.detach().cpu().numpy().reshape(B * H * 2, -1)
    rep["dQ_err"] = row_close(dq_g, bw["dQ"].reshape(B * H * 2, -1), rtol_qk, mask_q, "dQ",
                              absmag=absq.reshape(B * H * 2, -1))
    rep["dQ_err_plain"] = plain_row_err(dq_g, bw["dQ"].reshape(B * H * 2, -1), mask_q)
    if assert_plain:
        assert rep["dQ_err_plain"] <= rtol, f"dQ: plain row-max error {rep['dQ_err_plain']:.3g} > {rtol}"
    if dw is not None:
        rep["dw_err"] = row_close(dw.detach().cpu().numpy().reshape(B * H, -1),
                                  bw["dw"].reshape(B * H, -1), rtol, (~affected).reshape(-1), "dw")
    # rows touched by affected lookups (either selection) are masked
    bad_rows = set()
    bad_keys = set()
    if affected.any():
        gi = None if gpu_idx is None else np.asarray(gpu_idx.detach().cpu() if isinstance(gpu_idx, torch.Tensor) else gpu_idx)
        for b, h in zip(*np.nonzero(affected)):
            slots = o["idx"][b, h].tolist() + ([] if gi is None else gi[b, h].tolist())
            for f in slots:
                bad_rows.add(f); bad_keys.add((h, 0, f // n_sub)); bad_keys.add((h, 1, f % n_sub))
    rows = bw["rows"]
    dv_g = dV.detach().cpu().numpy()
    mask_v = np.array([r not in bad_rows for r in rows.tolist()], bool)
    rep["dV_err"] = row_close(dv_g[rows], bw["dV"], rtol, mask_v, "dV")
    untouched = np.ones(dv_g.shape[0], bool)
    untouched[rows] = False
    untouched[list(bad_rows)] = False  # the GPU's own slots at tie swaps may be non-zero
    assert np.all(dv_g[untouched] == 0), "dV rows never selected must stay exactly 0"
    dk_g = dK.detach().cpu().numpy().reshape(-1, K.shape[-1])
    dk_o = bw["dK"].reshape(-1, K.shape[-1])
    keys = [(h, half, i) for h in range(H) for half in range(2) for i in range(n_sub)]
    mask_k = np.array([kk not in bad_keys for kk in keys], bool)
    rep["dK_err"] = row_close(dk_g, dk_o, rtol_qk, mask_k, "dK", absmag=absk.reshape(dk_o.shape))
    rep["dK_err_plain"] = plain_row_err(dk_g, dk_o, mask_k)
    if assert_plain:
        assert rep["dK_err_plain"] <= rtol, f"dK: plain row-max error {rep['dK_err_plain']:.3g} > {rtol}"
    # sub-keys no selected slot uses get exactly 0; a selected
    # sub-key whose score gradients cancel (sum_t ds_t = 0 within one lookup)
    # is compared by the tolerance above, not required to be 0
    used = np.zeros((H, 2, n_sub), bool)
    sel = o["idx"] if gpu_idx is None else np.concatenate(
        [o["idx"], np.asarray(gpu_idx.detach().cpu() if isinstance(gpu_idx, torch.Tensor) else gpu_idx)], axis=0)
    hh = np.broadcast_to(np.arange(H)[None, :, None] if sel.ndim == 3 else 0, sel.shape)
    used[hh, 0, sel // n_sub] = True
    used[hh, 1, sel % n_sub] = True
    never = ~used.reshape(-1)
    assert np.all(dk_g[never] == 0), "never-selected sub-keys must get exactly 0 gradient"
    assert np.all(dk_o[never] == 0)
    return bw, rep
