"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
the same seeded inputs, element by element, under the north_star bar
(tests/parity.py).  Needs a B200."""
import os
import numpy as np
import pytest
import torch

from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from tests import parity

pytestmark = pytest.mark.gpu

DEV = "cuda"


def lookup_for(cfg, B=None, **kw):
    return PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k,
                     max_batch=B or cfg.batch, qk_dtype=cfg.qk_dtype,
                     value_dtype=cfg.value_dtype, **kw)


def run_fwd_bwd(cfg, Q, K, V, dOut, backward=True, **kw):
    lk = lookup_for(cfg, Q.shape[0], **kw)
    out, idx, w = lk.forward(Q, K, V)
    res = {"out": out, "idx": idx, "w": w}
    if backward:
        dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
        res.update(dQ=dq, dK=dK, dV=dV, dw=dw)
    torch.cuda.synchronize()
    return res


def check_all(cfg, Q, K, V, dOut, res, backward=True):
    Qc, Kc, Vc = Q.cpu(), K.cpu(), V.cpu()
    o, affected, rep = parity.check_forward(Qc, Kc, Vc, cfg.k, res["out"], res["idx"], res["w"])
    if backward:
        _, rb = parity.check_backward(Qc, Kc, Vc, cfg.k, dOut.cpu(), o, affected,
                                      res["dQ"], res["dK"], res["dV"], res["dw"], gpu_idx=res["idx"])
        rep.update(rb)
    print(cfg.name, rep)
    return rep


# ------------------------------------------------------------ small sweep --
SWEEP = [
    # (B, H, n_sub, d_h, d_v, k, qk dtype, v dtype)
    (1, 1, 32, 32, 32, 1, torch.float32, torch.float32),
    (7, 3, 32, 32, 64, 5, torch.float32, torch.float32),
    (33, 2, 128, 64, 64, 8, torch.float32, torch.float32),
    (130, 4, 64, 32, 128, 17, torch.float32, torch.float32),
    (65, 2, 96, 64, 256, 32, torch.bfloat16, torch.bfloat16),
    (200, 1, 256, 128, 512, 32, torch.bfloat16, torch.bfloat16),
    (37, 2, 128, 32, 64, 64, torch.float32, torch.float32),
    (50, 2, 64, 64, 32, 64, torch.bfloat16, torch.float32),
    (300, 4, 512, 256, 256, 32, torch.bfloat16, torch.bfloat16),
    # tensor-core dK: d_h 64, split-K with a ragged last split
    (1000, 2, 256, 64, 64, 16, torch.bfloat16, torch.bfloat16),
    (70, 2, 128, 64, 64, 16, torch.bfloat16, torch.bfloat16),
    # two-sweep scorer rows (n_sub > 512) with KT = 8: bf16, and fp32 (1xTF32 first sweep)
    (50, 2, 1024, 64, 64, 8, torch.bfloat16, torch.bfloat16),
    (40, 1, 1024, 32, 64, 5, torch.float32, torch.float32),
    # value rows of 1024 (the paper's inferred width), bf16
    (70, 2, 128, 64, 1024, 16, torch.bfloat16, torch.bfloat16),
    # small grids: scorer rows split over clusters of 4 (KT = 16, T = 2) and 2 CTAs (n_sub 512)
    (45, 3, 1024, 128, 128, 16, torch.bfloat16, torch.bfloat16),
    (129, 2, 512, 64, 64, 32, torch.bfloat16, torch.float32),
]


@pytest.mark.parametrize("shape", SWEEP, ids=lambda s: "x".join(str(v) for v in s[:6]) + f"-{str(s[6])[6:]}")
def test_small_shapes_fwd_bwd(shape):
    B, H, n_sub, d_h, d_v, k, qdt, vdt = shape
    cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, qdt, vdt, index=100 + n_sub + k)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_fwd_bwd(cfg, Q, K, V, dOut)
    check_all(cfg, Q, K, V, dOut, res)


@pytest.mark.parametrize("B,H,n_sub,d_h,k", [(64, 2, 64, 32, 16), (130, 2, 512, 64, 32),
                                             (96, 1, 1024, 128, 16), (40, 2, 256, 64, 8)])
def test_integer_data_bit_exact_selection(B, H, n_sub, d_h, k):
    """Integer-valued queries/keys: every score is exact in fp32 and fp64, so
    the selection (including the tie rule R5, with many exact ties) must be
    bit-identical -- 3xTF32 (fp32) and kind::f16 (bf16) tcgen05 scoring."""
    g = torch.Generator(device="cpu").manual_seed(5 + n_sub)
    d_v = 64
    Q = torch.randint(-2, 3, (B, H, 2, d_h), generator=g).float()
    K = torch.randint(-1, 2, (H, 2, n_sub, d_h), generator=g).float()
    V = torch.randn((n_sub * n_sub, d_v), generator=g) * 0.02
    for dt in (torch.float32, torch.bfloat16):
        if dt == torch.bfloat16 and d_h % 64:
            continue  # (the bf16 scorer takes d_half in multiples of 64)
        cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, dt, torch.float32)
        lk = lookup_for(cfg)
        out, idx, w = lk.forward(Q.to(dt).to(DEV), K.to(dt).to(DEV), V.to(DEV))
        from oracle import oracle as orc
        o = orc.forward(Q, K, V, k)
        assert np.array_equal(idx.cpu().numpy(), o["idx"]), "selection must be bit-exact on exact data"
        parity.row_close(out.cpu().numpy(), o["out"], 1e-4, what="out")


@pytest.mark.parametrize("d_h,n_sub,dt", [(32, 64, torch.float32), (64, 64, torch.bfloat16),
                                          (128, 1024, torch.bfloat16), (128, 1024, torch.float32),
                                          (64, 256, torch.float32)])
def test_zero_query_closed_form(d_h, n_sub, dt):
    """q = 0: all scores tie at 0 -> idx = 0..k-1.  On the tcgen05 scorer every
    row lets all its columns through the bound (resident and two-sweep rows,
    bf16 and 3xTF32 with the 1xTF32 first sweep), so every row takes the
    exact rescoring path."""
    cfg = wl.tiny_config(16, 2, d_h, n_sub, 64, 8, dt, torch.bfloat16)
    _, K, V, _ = wl.make_all(cfg, DEV)
    Q = torch.zeros((16, 2, 2, d_h), dtype=dt, device=DEV)
    out, idx, w = lookup_for(cfg).forward(Q, K, V)
    assert torch.equal(idx.cpu(), torch.arange(8, dtype=torch.int32).expand(16, 2, 8))
    assert torch.allclose(w, torch.full_like(w, 1 / 8), rtol=1e-6)
    ref = 2 * V[:8].float().mean(0)
    assert torch.allclose(out, ref.expand_as(out), rtol=1e-5, atol=1e-7)


# ------------------------------------------------------- BASELINE configs --
def test_c1_tiny_fp32_forward():
    cfg = wl.CONFIGS["c1_tiny_fp32"]
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_fwd_bwd(cfg, Q, K, V, dOut, backward=False)
    check_all(cfg, Q, K, V, dOut, res, backward=False)


def test_c2_mid_bf16_fwd_bwd():
    cfg = wl.CONFIGS["c2_mid_bf16"]
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_fwd_bwd(cfg, Q, K, V, dOut)
    check_all(cfg, Q, K, V, dOut, res)


@pytest.mark.parametrize("name,sample", [("c3_train_fp32_zipf", 1024), ("c4_large_sharded_bf16", 512),
                                         ("c5_latency_bf16", 512)])
def test_large_configs_on_query_sample(name, sample):
    """Full tables, the first `sample` queries (the oracle's budget)."""
    cfg = wl.CONFIGS[name]
    Q = wl.make_queries(cfg, DEV)[:sample].contiguous()
    K, V = wl.make_subkeys(cfg, DEV), wl.make_values(cfg, DEV)
    dOut = wl.make_dout(cfg, DEV)[:sample].contiguous()
    res = run_fwd_bwd(cfg, Q, K, V, dOut, backward=cfg.backward)
    check_all(cfg, Q, K, V, dOut, res, backward=cfg.backward)


@pytest.mark.parametrize("name", ["c3_train_fp32_zipf", "c4_large_sharded_bf16"])
def test_full_size_invariants(name):
    """Full BASELINE size in the bench's launch configuration: properties that
    hold at any size, plus sampled lookups recomputed by the oracle."""
    cfg = wl.CONFIGS[name]
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    assert torch.allclose(w.double().sum(-1), torch.ones(1, dtype=torch.float64, device=DEV), atol=1e-6)
    assert (w[..., 1:] <= w[..., :-1] + 1e-7).all()
    s = torch.sort(idx, dim=-1).values
    assert (s[..., 1:] != s[..., :-1]).all() and idx.min() >= 0 and idx.max() < cfg.n_slots
    # sum over rows of dV = H * sum_b dOut  (sum_t w = 1)
    lhs = dV.double().sum(0)
    rhs = cfg.heads * dOut.double().sum(0)
    assert torch.allclose(lhs, rhs, rtol=1e-4, atol=1e-3 * float(rhs.abs().max()))
    # untouched rows exactly zero
    touched = torch.zeros(cfg.n_slots, dtype=torch.bool, device=DEV)
    touched[idx.reshape(-1).long()] = True
    assert (dV[~touched] == 0).all()
    # sampled lookups against the oracle (same selection expected)
    from oracle import oracle as orc
    sel = torch.arange(0, cfg.batch, cfg.batch // 64, device=DEV)[:64]
    o = orc.forward(Q[sel].cpu(), K.cpu(), V.cpu(), cfg.k)
    aff, _ = parity.compare_selection(Q[sel].cpu(), K.cpu(), idx[sel].cpu().numpy(), o, cfg.n_sub)
    parity.row_close(out[sel].cpu().numpy(), o["out"], parity.rtol_for(cfg.value_dtype),
                     ~aff.any(axis=1), "out (sampled)")
    bw = orc.backward(Q[sel].cpu(), K.cpu(), V.cpu(), o["idx"], dOut[sel].cpu(), want_dense_dv=False)
    absq, _ = parity.grad_key_magnitudes(Q[sel].cpu(), K.cpu(), o, bw, cfg.n_sub)
    parity.row_close(dq[sel].cpu().numpy().reshape(-1, cfg.d_half), bw["dQ"].reshape(-1, cfg.d_half),
                     parity.rtol_for(cfg.value_dtype), np.repeat((~aff).reshape(-1), 2), "dQ (sampled)",
                     absmag=absq.reshape(-1, cfg.d_half))
    parity.row_close(dw[sel].cpu().numpy().reshape(-1, cfg.k), bw["dw"].reshape(-1, cfg.k),
                     parity.rtol_for(cfg.value_dtype), (~aff).reshape(-1), "dw (sampled)")


def test_c3_full_size_vs_oracle_hot_rows():
    """Full C3 (16,384 Zipf-clustered queries x 8 heads, the deterministic
    fp32 backward) against the fp64 oracle run on the whole batch: selection,
    out, dw, dQ, every dK row, and the dV rows of the 1,000 hottest slots
    (up to thousands of contributions each: the long-run reducers) -- element
    by element, none of them masked."""
    from oracle import oracle as orc
    cfg = wl.CONFIGS["c3_train_fp32_zipf"]
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    Qc, Kc, Vc = Q.cpu(), K.cpu(), V.cpu()
    o = orc.forward(Qc, Kc, Vc, cfg.k)
    aff, rep = parity.compare_selection(Qc, Kc, idx.cpu().numpy(), o, cfg.n_sub)
    assert aff.sum() <= max(2, 0.01 * aff.size), rep
    rows, hits = np.unique(o["idx"], return_counts=True)
    order = np.argsort(-hits, kind="stable")
    # the 1,000 hottest rows no tie-affected lookup touches (either selection:
    # their expected values would need the CUDA path's selection)
    bad = set()
    for b, h in zip(*np.nonzero(aff)):
        bad.update(o["idx"][b, h].tolist())
        bad.update(idx[b, h].cpu().tolist())
    hot_i = [i for i in order.tolist() if int(rows[i]) not in bad][:1000]
    hot = rows[hot_i].astype(np.int64)
    assert hits[hot_i[0]] > 500 and hits[hot_i[-1]] >= 20, "the Zipf workload is expected to have hot rows"
    bw = orc.backward(Qc, Kc, Vc, o["idx"], dOut.cpu(), want_dense_dv=False)  # dV over the touched rows
    rt = parity.rtol_for(cfg.value_dtype)
    hs = np.sort(hot)
    pos = np.searchsorted(bw["rows"], hs)
    assert np.array_equal(bw["rows"][pos], hs)
    err_v = parity.row_close(dV[torch.from_numpy(hs).to(DEV)].cpu().numpy(), bw["dV"][pos], rt,
                             what="dV (1000 hottest rows)")
    absq, absk = parity.grad_key_magnitudes(Qc, Kc, o, bw, cfg.n_sub)
    ok = (~aff).reshape(-1)
    err_q = parity.row_close(dq.cpu().numpy().reshape(-1, cfg.d_half), bw["dQ"].reshape(-1, cfg.d_half), rt,
                             np.repeat(ok, 2), "dQ", absmag=absq.reshape(-1, cfg.d_half))
    mask_k = np.ones(cfg.heads * 2 * cfg.n_sub, bool)
    for b, h in zip(*np.nonzero(aff)):
        for f in o["idx"][b, h].tolist() + idx[b, h].cpu().tolist():
            mask_k[(h * 2) * cfg.n_sub + f // cfg.n_sub] = False
            mask_k[(h * 2 + 1) * cfg.n_sub + f % cfg.n_sub] = False
    err_k = parity.row_close(dK.cpu().numpy().reshape(-1, cfg.d_half), bw["dK"].reshape(-1, cfg.d_half), rt,
                             mask_k, "dK", absmag=absk.reshape(-1, cfg.d_half))
    err_w = parity.row_close(dw.cpu().numpy().reshape(-1, cfg.k), bw["dw"].reshape(-1, cfg.k), rt, ok, "dw")
    err_o = parity.row_close(out.cpu().numpy(), o["out"], rt, ~aff.any(axis=1), "out")
    print("C3 full:", rep, {"max_hits": int(hits.max()), "hot_hits_min": int(hits[hot_i[-1]]), "dV_hot": err_v, "dQ": err_q, "dK": err_k,
                            "dw": err_w, "out": err_o})


@pytest.mark.parametrize("name", ["f4_tokens_bf16", "f4_tokens_pertable_bf16"])
def test_f4_full_size(name):
    """SURVEY 8(f) f4 at its bench size (2048 queries x 16 tokens, n = 256^2,
    d_v = 512; shared table or 16 per-token tables): invariants over every
    lookup, plus sampled queries recomputed per token by the fp64 oracle."""
    from oracle import oracle as orc
    cfg = wl.CONFIGS[name]
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    G, n = cfg.head_groups, cfg.n_sub * cfg.n_sub
    lk = lookup_for(cfg, head_groups=G, group_tables=cfg.group_tables)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    assert tuple(out.shape) == (cfg.batch, G, cfg.d_value)
    assert torch.allclose(w.double().sum(-1), torch.ones(1, dtype=torch.float64, device=DEV), atol=1e-6)
    assert (w[..., 1:] <= w[..., :-1] + 1e-7).all()
    s = torch.sort(idx, dim=-1).values
    assert (s[..., 1:] != s[..., :-1]).all()
    hg = cfg.heads // G
    grp = (torch.arange(cfg.heads, device=DEV) // hg).view(1, -1, 1)
    lo = grp * n if cfg.group_tables else torch.zeros_like(grp)
    assert (idx >= lo).all() and (idx < lo + n).all()
    # sum over rows of dV = (H/G) * sum over b, g of dOut[b, g]  (sum_t w = 1)
    lhs = dV.double().sum(0)
    rhs = hg * dOut.double().sum((0, 1))
    assert torch.allclose(lhs, rhs, rtol=1e-4, atol=1e-3 * float(rhs.abs().max()))
    touched = torch.zeros(cfg.n_slots, dtype=torch.bool, device=DEV)
    touched[idx.reshape(-1).long()] = True
    assert (dV[~touched] == 0).all()
    sel = torch.arange(0, cfg.batch, cfg.batch // 16, device=DEV)[:16]
    rt = parity.rtol_for(cfg.value_dtype)
    Qs, Kc, Vc, Ds = Q[sel].cpu(), K.cpu(), V.cpu(), dOut[sel].cpu()
    for g in range(G):
        hs = slice(g * hg, (g + 1) * hg)
        Vg = Vc[g * n:(g + 1) * n] if cfg.group_tables else Vc
        off = g * n if cfg.group_tables else 0
        o = orc.forward(Qs[:, hs].contiguous(), Kc[hs].contiguous(), Vg, cfg.k)
        ig = idx[sel][:, hs].cpu().numpy().astype(np.int64) - off
        aff, _ = parity.compare_selection(Qs[:, hs].contiguous(), Kc[hs].contiguous(), ig, o, cfg.n_sub)
        ok = ~aff.any(axis=1)
        parity.row_close(out[sel][:, g].cpu().numpy(), o["out"], rt, ok, f"out token {g} (sampled)")
        bw = orc.backward(Qs[:, hs].contiguous(), Kc[hs].contiguous(), Vg, o["idx"], Ds[:, g].contiguous(),
                          want_dense_dv=False)
        parity.row_close(dw[sel][:, hs].cpu().numpy().reshape(-1, cfg.k), bw["dw"].reshape(-1, cfg.k), rt,
                         np.repeat(ok, hg), f"dw token {g} (sampled)")
        absq, _ = parity.grad_key_magnitudes(Qs[:, hs].contiguous(), Kc[hs].contiguous(), o, bw, cfg.n_sub)
        parity.row_close(dq[sel][:, hs].cpu().numpy().reshape(-1, cfg.d_half), bw["dQ"].reshape(-1, cfg.d_half),
                         rt, np.repeat(np.repeat(ok, hg), 2), f"dQ token {g} (sampled)",
                         absmag=absq.reshape(-1, cfg.d_half))


# ------------------------------------------- memory-gated fusion (f1) ----
@pytest.mark.parametrize("gate", ["tanh", "sigmoid", "identity"])
@pytest.mark.parametrize("name,B", [("tiny_fp32", 300), ("c2_mid_bf16", 512), ("c3_train_fp32_zipf", 8192)])
def test_gated_fusion_fwd_bwd(gate, name, B):
    """x~ = x * g(v_o) fused into the gather epilogue (B >= 8192: into the
    fused Cartesian + gather kernel), and its backward feeding the lookup
    backward, against oracle/gate.py on top of the fp64 oracle."""
    from oracle import gate as og
    if name == "tiny_fp32":
        cfg = wl.tiny_config(B, 2, 32, 64, 64, 8, torch.float32, torch.float32, index=12)
        Q, K, V, dXt = wl.make_all(cfg, DEV)
    else:
        cfg = wl.CONFIGS[name]
        Q = wl.make_queries(cfg, DEV)[:B].contiguous()
        K, V = wl.make_subkeys(cfg, DEV), wl.make_values(cfg, DEV)
        dXt = wl.make_dout(cfg, DEV)[:B].contiguous()
    g = torch.Generator(device="cpu").manual_seed(5)
    X = torch.randn((B, cfg.d_value), generator=g).to(DEV)
    lk = lookup_for(cfg, B)
    xt, vo, idx, w = lk.forward_gated(Q, K, V, X, gate)
    out2, idx2, w2 = lk.forward(Q, K, V)
    torch.cuda.synchronize()
    assert torch.equal(idx, idx2) and torch.equal(w, w2) and torch.equal(vo, out2)
    if B > 1024:  # oracle on a sample of the queries (full table)
        sel = slice(0, 512)
        Qs, dXs, Xs = Q[sel].contiguous(), dXt[sel].contiguous(), X[sel]
        vo_s, xt_s, idx_s, w_s = vo[sel], xt[sel], idx[sel], w[sel]
    else:
        Qs, dXs, Xs, vo_s, xt_s, idx_s, w_s = Q, dXt, X, vo, xt, idx, w
    rt = parity.rtol_for(cfg.value_dtype)
    o, aff, _ = parity.check_forward(Qs.cpu(), K.cpu(), V.cpu(), cfg.k, vo_s, idx_s, w_s)
    ok = ~aff.any(axis=1)
    parity.row_close(xt_s.cpu().numpy(), og.forward(o["out"], Xs.cpu(), gate), rt, ok, "x~")
    dx, dvo = lk.gate_backward(dXs, Xs, vo_s, gate)
    dx_ref, dvo_ref = og.backward(o["out"], Xs.cpu(), dXs.cpu(), gate)
    parity.row_close(dx.cpu().numpy(), dx_ref, rt, ok, "dx_in")
    parity.row_close(dvo.cpu().numpy(), dvo_ref, rt, ok, "dv_o")


# ------------------------------------------- fused optimiser update (f3) -
@pytest.mark.parametrize("update", ["sgd", "adagrad"])
@pytest.mark.parametrize("name,B", [("tiny_fp32", 300), ("hot_fp32", 3000), ("c2_mid_bf16", 4096)])
def test_fused_update(update, name, B):
    """msn_pkm_scatter_update against oracle/update.py applied to the oracle's
    value gradient: the change of every touched row (and of the Adagrad
    state), dw, and untouched rows bit-for-bit unchanged."""
    from oracle import oracle as orc
    from oracle import update as ou
    if name == "c2_mid_bf16":
        cfg = wl.CONFIGS[name]
        Q, K, V, dOut = wl.make_all(cfg, DEV)
        lr = 0.5   # bf16 values: steps well above the storage rounding
    else:
        cfg = wl.tiny_config(B, 2, 32, 64, 64, 8, torch.float32, torch.float32, index=13)
        Q, K, V, dOut = wl.make_all(cfg, DEV)
        if name == "hot_fp32":  # long runs (piece + combine path)
            g = torch.Generator(device="cpu").manual_seed(13)
            base = torch.randn((1, 2, 2, 32), generator=g)
            Q = (base + 1e-3 * torch.randn((B, 2, 2, 32), generator=g)).to(DEV)
        lr = 1e-2
    eps = 1e-6
    lk = lookup_for(cfg, B)
    out, idx, w = lk.forward(Q, K, V)
    V0 = V.clone()
    st = torch.rand(V.shape, generator=torch.Generator(device="cpu").manual_seed(3)).to(DEV) \
        if update == "adagrad" else None
    st0 = st.clone() if st is not None else None
    dw = lk.scatter_update(idx, w, dOut, V, update, lr, eps, st)
    torch.cuda.synchronize()
    o = orc.forward(Q.cpu(), K.cpu(), V0.cpu(), cfg.k)
    gi = idx.cpu().numpy().astype(np.int64)
    aff, _ = parity.compare_selection(Q.cpu(), K.cpu(), gi, o, cfg.n_sub)
    assert aff.mean() <= 0.01
    # the oracle's own selection; rows touched by a lookup whose selection
    # differs at a tie (either side's slots) are excluded from the comparison
    bw = orc.backward(Q.cpu(), K.cpu(), V0.cpu(), o["idx"], dOut.cpu(), want_dense_dv=False)
    Vn, sn = ou.apply(V0.cpu().double().numpy(), bw["rows"], bw["dV"], update, lr, eps,
                      None if st0 is None else st0.cpu().double().numpy())
    skip = np.union1d(gi[aff].reshape(-1), o["idx"][aff].reshape(-1))
    rows = np.setdiff1d(bw["rows"], skip)
    rt = parity.rtol_for(cfg.value_dtype)
    delta_gpu = (V.double() - V0.double()).cpu().numpy()[rows]
    delta_ref = Vn[rows] - V0.cpu().double().numpy()[rows]
    # bf16 storage: the new value is rounded once (half an ulp of |V_new|)
    slack = np.abs(Vn[rows]) * (2.0 ** -8 if cfg.value_dtype == torch.bfloat16 else 2.0 ** -23)
    err = np.abs(delta_gpu - delta_ref)
    assert (err <= rt * np.abs(delta_ref).max(axis=1, keepdims=True) + slack + 1e-30).all(), float(err.max())
    untouched = np.setdiff1d(np.arange(V.shape[0]), np.union1d(bw["rows"], gi.reshape(-1)))
    assert torch.equal(V[torch.as_tensor(untouched, device=DEV)], V0[torch.as_tensor(untouched, device=DEV)])
    if st is not None:
        parity.row_close(st.cpu().numpy()[rows], sn[rows], 1e-5, what="adagrad state")
    parity.row_close(dw.cpu().numpy().reshape(-1, cfg.k), bw["dw"].reshape(-1, cfg.k), rt,
                     ~aff.reshape(-1), what="dw")


# ------------------------------------------ head groups / tokens (f4) ----
@pytest.mark.parametrize("tables", [False, True])
@pytest.mark.parametrize("B,dt,G,H,n_sub,d_h", [(300, torch.float32, 4, 8, 64, 32),
                                                (2048, torch.bfloat16, 16, 16, 64, 64),
                                                (9000, torch.float32, 2, 4, 64, 32),
                                                # tcgen05 scorer: resident rows, two-sweep rows
                                                (700, torch.bfloat16, 4, 8, 256, 64),
                                                (300, torch.bfloat16, 2, 4, 1024, 64)])
def test_head_groups(B, dt, G, H, tables, n_sub, d_h):
    """Token-specific codebooks: G groups of H/G heads with a
    shared table (or one table per group), out [B, G, d_v].  The reference is
    G independent fp64 oracle lookups -- group g's heads, its table -- and the
    backward the same with d_out[:, g]; dV rows, dK and dQ compared per group."""
    from oracle import oracle as orc
    d_v, k = 64, 8
    cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, dt, dt, index=14)
    Q, K, V1, _ = wl.make_all(cfg, DEV)
    n = n_sub * n_sub
    gv = torch.Generator(device="cpu").manual_seed(15)
    V = (0.02 * torch.randn((G * n if tables else n, d_v), generator=gv)).to(dt).to(DEV)
    dOut = torch.randn((B, G, d_v), generator=gv).to(DEV)
    lk = PKMLookup(H, n_sub, d_h, d_v, k, max_batch=B, qk_dtype=dt, value_dtype=dt,
                   head_groups=G, group_tables=tables)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    assert tuple(out.shape) == (B, G, d_v)
    hg = H // G
    rt = parity.rtol_for(dt)
    Qc, Kc, Vc = Q.cpu(), K.cpu(), V.cpu()
    for g in range(G):
        hs = slice(g * hg, (g + 1) * hg)
        Vg = Vc[g * n:(g + 1) * n] if tables else Vc
        off = g * n if tables else 0
        ig = idx[:, hs].cpu().numpy().astype(np.int64) - off
        assert (ig >= 0).all() and (ig < n).all()
        o, aff, _ = parity.check_forward(Qc[:, hs].contiguous(), Kc[hs].contiguous(), Vg, k,
                                         out[:, g].contiguous(), torch.as_tensor(ig).int(), w[:, hs].contiguous())
        ok = ~aff.any(axis=1)
        bw = orc.backward(Qc[:, hs].contiguous(), Kc[hs].contiguous(), Vg, o["idx"], dOut[:, g].cpu(),
                          want_dense_dv=False)
        parity.row_close(dw[:, hs].cpu().numpy().reshape(-1, k), bw["dw"].reshape(-1, k), rt,
                         np.repeat(ok, hg), "dw")
        absq, absk = parity.grad_key_magnitudes(Qc[:, hs].contiguous(), Kc[hs].contiguous(), o, bw, n_sub)
        parity.row_close(dq[:, hs].cpu().numpy().reshape(-1, d_h), bw["dQ"].reshape(-1, d_h), rt,
                         np.repeat(np.repeat(ok, hg), 2), "dQ", absmag=absq.reshape(-1, d_h))
        if tables and not aff.any():
            rows = bw["rows"]
            parity.row_close(dV[off + rows].cpu().numpy(), bw["dV"], rt, what="dV (group table)")
    if not tables:  # shared table: dV = sum over groups of the per-group oracle dV
        tot = np.zeros((n, d_v))
        clean = True
        for g in range(G):
            hs = slice(g * hg, (g + 1) * hg)
            o = orc.forward(Qc[:, hs].contiguous(), Kc[hs].contiguous(), Vc, k)
            clean &= np.array_equal(o["idx"], idx[:, hs].cpu().numpy())
            bw = orc.backward(Qc[:, hs].contiguous(), Kc[hs].contiguous(), Vc, o["idx"], dOut[:, g].cpu())
            tot += bw["dV"]
        if clean:
            parity.row_close(dV.cpu().numpy(), tot, rt, what="dV (shared table)")


# --------------------------------------------- query/key prologue (f2) ----
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d_h", [32, 128, 256])
def test_prologue_stages(dt, d_h):
    """Each prologue stage on seeded inputs against oracle/prologue.py:
    LayerNorm and its backward, K~ = Theta k^ and its
    gradients."""
    from oracle import prologue as op
    H, n_sub = 2, 192
    g = torch.Generator(device="cpu").manual_seed(21)
    lk = PKMLookup(H, n_sub, d_h, 64, 8, max_batch=64, qk_dtype=dt, value_dtype=dt)
    rt = parity.rtol_for(dt)
    x = (3.0 * torch.randn((300, H, 2, d_h), generator=g) + 0.5).to(dt).to(DEV)
    y = lk.layernorm(x)
    parity.row_close(y.cpu().reshape(-1, d_h).float().numpy(), op.layernorm(x.cpu()).reshape(-1, d_h), rt,
                     what="LN")
    dy = torch.randn(x.shape, generator=g).to(DEV)
    dx = lk.layernorm_backward(x, dy)
    parity.row_close(dx.cpu().reshape(-1, d_h).numpy(), op.layernorm_backward(x.cpu(), dy.cpu()).reshape(-1, d_h),
                     rt, what="LN backward")
    k_hat = torch.randn((H, 2, n_sub, d_h), generator=g).to(dt).to(DEV)
    theta = (torch.randn((H, 2, d_h, d_h), generator=g) / d_h ** 0.5).to(DEV)
    k_eff = lk.key_transform(k_hat, theta)
    parity.row_close(k_eff.cpu().float().reshape(-1, d_h).numpy(),
                     op.key_transform(k_hat.cpu(), theta.cpu()).reshape(-1, d_h), rt, what="K~")
    d_k_eff = torch.randn((H, 2, n_sub, d_h), generator=g).to(DEV)
    d0 = torch.randn(theta.shape, generator=g).to(DEV)
    dkh, dth = lk.key_transform_backward(k_hat, theta, d_k_eff, d_theta=d0.clone())
    rk, rth = op.key_transform_backward(k_hat.cpu(), theta.cpu(), d_k_eff.cpu())
    parity.row_close(dkh.cpu().reshape(-1, d_h).numpy(), rk.reshape(-1, d_h), 1e-4, what="dK^")
    parity.row_close((dth - d0).cpu().reshape(-1, d_h).numpy(), rth.reshape(-1, d_h), 1e-4, what="dTheta")


@pytest.mark.parametrize("fused_ln", [False, True])
def test_prologue_chain_fp32(fused_ln):
    """q^ = LN(q), K~ = Theta LN(k), lookup, backward, back through the
    prologue -- the whole chain on the GPU against the fp64 oracle chain.
    fused_ln: LN(q) folded into the scorer's operand load (msn_pkm_forward_qln)."""
    from oracle import oracle as orc
    from oracle import prologue as op
    B, H, n_sub, d_h, d_v, k = 500, 2, 128, 64, 64, 8
    cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, torch.float32, torch.float32, index=22)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    g = torch.Generator(device="cpu").manual_seed(22)
    theta = (torch.eye(d_h) + 0.1 * torch.randn((H, 2, d_h, d_h), generator=g)).to(DEV)
    lk = lookup_for(cfg, B)
    kh = lk.layernorm(K)
    ke = lk.key_transform(kh, theta)
    if fused_ln:
        out, idx, w, qh = lk.forward_qln(Q, ke, V)
    else:
        qh = lk.layernorm(Q)
        out, idx, w = lk.forward(qh, ke, V)
    dqh, dke, dV, dw = lk.backward(dOut, qh, ke, V, idx, w)
    dq = lk.layernorm_backward(Q, dqh)
    dkh, dth = lk.key_transform_backward(kh, theta, dke)
    dk = lk.layernorm_backward(K, dkh)
    torch.cuda.synchronize()
    # fp64 oracle chain from the raw inputs
    qh_o = op.layernorm(Q.cpu())
    kh_o = op.layernorm(K.cpu())
    ke_o = op.key_transform(kh_o, theta.cpu())
    o = orc.forward(qh_o, ke_o, V.cpu(), k)
    aff, _ = parity.compare_selection(qh_o, ke_o, idx.cpu().numpy().astype(np.int64), o, n_sub)
    ok = ~aff.any(axis=1)
    parity.row_close(out.cpu().numpy(), o["out"], 1e-4, ok, "out")
    if aff.any():
        return  # a near-tie changed the selection: the chain's gradients differ by construction
    bw = orc.backward(qh_o, ke_o, V.cpu(), o["idx"], dOut.cpu())
    dq_o = op.layernorm_backward(Q.cpu(), bw["dQ"])
    dkh_o, dth_o = op.key_transform_backward(kh_o, theta.cpu(), bw["dK"])
    dk_o = op.layernorm_backward(K.cpu(), dkh_o)
    # condition-aware scales (R14): the sums of |terms| behind every element,
    # carried through the linear backward maps with absolute values
    absq, absk = parity.grad_key_magnitudes(qh_o, ke_o, o, bw, n_sub)

    def ln_mag(x, a):  # |d LN(x)^T dy| <= r (a + mean a + |x^| mean(a |x^|)) for |dy| <= a
        x = x.cpu().double().numpy()
        mu = x.mean(-1, keepdims=True)
        r = 1.0 / np.sqrt(((x - mu) ** 2).mean(-1, keepdims=True) + op.EPS)
        xh = np.abs((x - mu) * r)
        return r * (a + a.mean(-1, keepdims=True) + xh * (a * xh).mean(-1, keepdims=True))

    th = np.abs(theta.cpu().double().numpy())
    mag_dkh = np.einsum("hcie,hced->hcid", absk, th)
    mag_dth = np.einsum("hcie,hcid->hced", absk, np.abs(kh_o))
    parity.row_close(dq.cpu().reshape(-1, d_h).numpy(), dq_o.reshape(-1, d_h), 1e-4, what="dq",
                     absmag=ln_mag(Q, absq).reshape(-1, d_h))
    parity.row_close(dth.cpu().reshape(-1, d_h).numpy(), dth_o.reshape(-1, d_h), 1e-4, what="dTheta",
                     absmag=mag_dth.reshape(-1, d_h))
    parity.row_close(dk.cpu().reshape(-1, d_h).numpy(), dk_o.reshape(-1, d_h), 1e-4, what="dk",
                     absmag=ln_mag(K, mag_dkh).reshape(-1, d_h))


@pytest.mark.parametrize("name,B", [("c2_mid_bf16", 777), ("c5_latency_bf16", 300), ("c4_large_sharded_bf16", 200)])
def test_forward_qln_matches_layernorm_then_forward(name, B):
    """bf16: the LayerNorm folded into the scorer's operand load gives q^ within
    one bf16 rounding of msn_pkm_layernorm's (its sums run in another order),
    the same selection except at near-ties, and the same out within the bf16
    tolerance; q^ against the fp64 LN oracle too."""
    from oracle import prologue as op
    cfg = wl.CONFIGS[name].scaled(batch=B)
    Q, K, V, _ = wl.make_all(cfg, DEV)
    Q = (3.0 * Q.float() + 0.5).to(cfg.qk_dtype)  # a non-trivial mean and scale
    lk = lookup_for(cfg, B)
    out_f, idx_f, w_f, qh_f = lk.forward_qln(Q, K, V)
    qh = lk.layernorm(Q)
    out, idx, w = lk.forward(qh, K, V)
    torch.cuda.synchronize()
    d = (qh_f.float() - qh.float()).abs()
    assert float(d.max()) <= 2 * float(2.0 ** -8 * qh.float().abs().max())
    parity.row_close(qh_f.cpu().float().reshape(-1, cfg.d_half).numpy(),
                     op.layernorm(Q.cpu()).reshape(-1, cfg.d_half), 2e-2, what="q^ vs oracle LN")
    same = (idx_f == idx).all(-1).all(-1)
    assert float(same.float().mean()) > 0.98
    sel = same.cpu().numpy()
    parity.row_close(out_f.cpu().numpy(), out.cpu().numpy(), 2e-2, sel, "out")


# --------------------------------------------------- hot rows (grouping) --
@pytest.mark.parametrize("B,H,dt", [(400, 2, torch.float32),     # runs of 33..1024: warp sort, pieces
                                    (3000, 2, torch.float32),    # > 1024: CTA sort in shared memory
                                    (20000, 1, torch.float32)])  # > 16384: in-place sort in global memory
def test_hot_rows_long_runs(B, H, dt):
    """Near-identical queries: every lookup selects (almost) the same slots,
    so a few dV rows and dK rows receive thousands of contributions each --
    the long-run grouping paths.  Oracle parity and bitwise repeatability."""
    cfg = wl.tiny_config(B, H, 32, 64, 32, 4, dt, dt, index=11)
    _, K, V, dOut = wl.make_all(cfg, DEV)
    g = torch.Generator(device="cpu").manual_seed(11)
    base = torch.randn((1, H, 2, 32), generator=g)
    Q = (base + 1e-3 * torch.randn((B, H, 2, 32), generator=g)).to(dt).to(DEV)
    r1 = run_fwd_bwd(cfg, Q, K, V, dOut)
    rows, counts = torch.unique(r1["idx"].reshape(-1), return_counts=True)
    assert int(counts.max()) > {400: 32, 3000: 1024, 20000: 16384}[B]
    r2 = run_fwd_bwd(cfg, Q, K, V, dOut)
    for key in ("dQ", "dK", "dV", "dw"):
        assert torch.equal(r1[key], r2[key]), key
    check_all(cfg, Q, K, V, dOut, r1)


# ---------------------------------------------------------- properties ----
def test_determinism_bitwise():
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=1024)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    r1 = run_fwd_bwd(cfg, Q, K, V, dOut)
    r2 = run_fwd_bwd(cfg, Q, K, V, dOut)
    for key in ("out", "idx", "w", "dQ", "dK", "dV", "dw"):
        assert torch.equal(r1[key], r2[key]), key


def test_batch_invariance():
    """A query's idx/w/out do not depend on B or on its position."""
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=512)
    Q, K, V, _ = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    perm = torch.randperm(512, device=DEV)[:77]
    o2, i2, w2 = lk.forward(Q[perm].contiguous(), K, V)
    assert torch.equal(i2, idx[perm]) and torch.equal(w2, w[perm]) and torch.equal(o2, out[perm])


def test_atomic_backward_matches_oracle():
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=512)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_fwd_bwd(cfg, Q, K, V, dOut, atomic_bwd=True)
    check_all(cfg, Q, K, V, dOut, res)


def test_backward_accumulates():
    cfg = wl.tiny_config(32, 2, 32, 64, 64, 8, torch.float32, torch.float32)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    _, dK1, dV1, _ = lk.backward(dOut, Q, K, V, idx, w)
    dK2, dV2 = dK1.clone(), dV1.clone()
    lk.backward(dOut, Q, K, V, idx, w, d_subkeys=dK2, d_values=dV2)
    assert torch.allclose(dK2, 2 * dK1) and torch.allclose(dV2, 2 * dV1)


def test_sharded_phases_match_full():
    """Row-sharded table emulated on one GPU: P shards' gather partials sum to
    the full output; their dV shards concatenate to the full dV bitwise
    up to fp32 reassociation at tile-crossing runs; their dw sum to the full
    dw bitwise."""
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=256)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    full = run_fwd_bwd(cfg, Q, K, V, dOut)
    n = cfg.n_slots
    for P in (2, 4):
        outs, dvs, dws = [], [], []
        for p in range(P):
            r0, r1 = p * n // P, (p + 1) * n // P
            lk = lookup_for(cfg, row_begin=r0, row_end=r1)
            idx, w = lk.select(Q, K)
            assert torch.equal(idx, full["idx"]) and torch.equal(w, full["w"])
            outs.append(lk.gather(idx, w, V[r0:r1].contiguous()))
            dvp = torch.zeros((r1 - r0, cfg.d_value), device=DEV)
            dws.append(lk.scatter(idx, w, dOut, V[r0:r1].contiguous(), dvp))
            dvs.append(dvp)
        torch.cuda.synchronize()
        assert torch.allclose(sum(outs), full["out"], rtol=1e-5, atol=1e-6)
        assert torch.allclose(torch.cat(dvs), full["dV"], rtol=1e-5, atol=1e-7)
        dw = sum(dws)
        assert torch.allclose(dw, full["dw"], rtol=0, atol=0)
        lk = lookup_for(cfg)
        dq, dK = lk.backward_keys(Q, K, full["idx"], full["w"], dw)
        assert torch.equal(dq, full["dQ"]) and torch.equal(dK, full["dK"])


def test_backward_unsupported_width_is_reported():
    from paper_2602_07526_b200._lib import MsnError
    cfg = wl.tiny_config(4, 1, 32, 32, 48, 2, torch.float32, torch.float32)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)          # the forward takes d_value * 4 % 16 == 0
    dV = torch.full((cfg.n_slots, cfg.d_value), 0.25, dtype=torch.float32, device=DEV)
    dK = torch.full((cfg.heads, 2, cfg.n_sub, cfg.d_half), 0.5, dtype=torch.float32, device=DEV)
    with pytest.raises(MsnError, match="UNSUPPORTED"):
        lk.backward(dOut, Q, K, V, idx, w, d_subkeys=dK, d_values=dV)  # the reducers take 32 * 2^j
    torch.cuda.synchronize()
    # checked on the host before any launch: the accumulators are untouched
    assert torch.all(dV == 0.25) and torch.all(dK == 0.5)


def test_autograd_function():
    from paper_2602_07526_b200.pkm import pkm
    cfg = wl.tiny_config(16, 2, 32, 64, 64, 8, torch.float32, torch.float32)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    q, k_, v = (t.clone().requires_grad_(True) for t in (Q, K, V))
    out = pkm(lk, q, k_, v)
    (out * dOut).sum().backward()
    _, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, _ = lk.backward(dOut, Q, K, V, idx, w)
    assert torch.equal(q.grad, dq) and torch.equal(k_.grad, dK) and torch.equal(v.grad, dV)


def test_host_tensors_end_to_end():
    cfg = wl.tiny_config(16, 2, 32, 64, 64, 8, torch.float32, torch.float32)
    Q, K, V, dOut = wl.make_all(cfg, "cpu")
    lk = lookup_for(cfg)
    out_h, idx_h, w_h = lk.forward(Q.pin_memory(), K.to(DEV), V.to(DEV))
    out_d, idx_d, w_d = lk.forward(Q.to(DEV), K.to(DEV), V.to(DEV))
    assert out_h.device.type == "cpu" and torch.equal(out_h, out_d.cpu())


def test_host_tensors_backward_and_autograd():
    """Host inputs: every backward result comes back on the host, and autograd
    over CPU-resident parameters gets CPU gradients (equal to the device run)."""
    from paper_2602_07526_b200.pkm import pkm
    cfg = wl.tiny_config(16, 2, 32, 64, 64, 8, torch.float32, torch.float32)
    Q, K, V, dOut = wl.make_all(cfg, "cpu")
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    res_h = lk.backward(dOut, Q, K, V, idx, w)
    assert all(t.device.type == "cpu" for t in res_h)
    res_d = lk.backward(dOut.to(DEV), Q.to(DEV), K.to(DEV), V.to(DEV), idx.to(DEV), w.to(DEV))
    for a, b in zip(res_h, res_d):
        assert torch.equal(a, b.cpu())
    q, k_, v = (t.clone().requires_grad_(True) for t in (Q, K, V))
    (pkm(lk, q, k_, v) * dOut).sum().backward()
    assert q.grad.device.type == k_.grad.device.type == v.grad.device.type == "cpu"
    assert torch.equal(k_.grad, res_h[1]) and torch.equal(v.grad, res_h[2])


def test_invalid_arguments_raise():
    from paper_2602_07526_b200._lib import MsnError
    cfg = wl.tiny_config(16, 2, 32, 64, 64, 8, torch.float32, torch.float32)
    lk = lookup_for(cfg)
    Q, K, V, _ = wl.make_all(cfg, DEV)
    with pytest.raises(ValueError):
        lk.forward(Q.to(torch.bfloat16), K, V)
    big = wl.make_queries(cfg.scaled(batch=17), DEV)
    with pytest.raises(MsnError):
        lk.forward(big, K, V)


@pytest.mark.parametrize("name,groups,tables", [("c2_mid_bf16", 1, False), ("f4_tokens_pertable_bf16", 16, True)])
def test_validate_tape(name, groups, tables):
    """msn_pkm_validate_tape counts exactly the corrupted slots (SURVEY 8(b)
    "Errors"); with MSN_FLAG_VALIDATE a consumer of a bad tape raises before
    launching, and a good tape gives the unvalidated results bitwise."""
    from paper_2602_07526_b200._lib import MsnError
    cfg = wl.CONFIGS[name].scaled(batch=300)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    kw = dict(head_groups=groups, group_tables=tables)
    lk = lookup_for(cfg, **kw)
    lv = lookup_for(cfg, validate=True, **kw)
    out, idx, w = lk.forward(Q, K, V)
    assert int(lk.validate_tape(idx, w).item()) == 0
    n2 = cfg.n_sub * cfg.n_sub
    bad_i, bad_w = idx.clone(), w.clone()
    bad_i[0, 0, 0] = -1                    # below the table
    bad_i[1, 1, 3] = n2 * groups           # past the last table row
    bad_i[2, 0, 5] = bad_i[2, 0, 4]        # repeated id: both copies count
    bad_w[3, 0, 0] = float("nan")
    bad_w[4, 1, 2] = -0.25
    expect = 1 + 1 + 2 + 1 + 1
    if tables:                             # head 0 (group 0) pointing into group 1's table
        bad_i[5, 0, 1] = bad_i[5, 0, 1] % n2 + n2
        expect += 1
    assert int(lk.validate_tape(bad_i, bad_w).item()) == expect
    assert int(lk.validate_tape(idx, bad_w).item()) == 2
    with pytest.raises(MsnError, match="INVALID_ARG"):
        lv.backward(dOut, Q, K, V, bad_i, w)
    with pytest.raises(MsnError, match="INVALID_ARG"):
        lv.gather(idx, bad_w, V)
    r0 = lk.backward(dOut, Q, K, V, idx, w)
    r1 = lv.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    for a, b in zip(r0, r1):
        assert torch.equal(a, b)
    assert torch.equal(lv.gather(idx, w, V), lk.gather(idx, w, V))


_SPLIT_SCRIPT = """
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
cfg = wl.CONFIGS[sys.argv[2]].scaled(batch=int(sys.argv[3]))
Q, K, V, _ = wl.make_all(cfg, "cuda")
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype, cfg.value_dtype)
out, idx, w = lk.forward(Q, K, V)
torch.save({"out": out.cpu(), "idx": idx.cpu(), "w": w.cpu()}, sys.argv[4])
"""


@pytest.mark.parametrize("name,B", [("c5_latency_bf16", 512), ("c5_latency_bf16", 130),
                                    ("c5_latency_bf16", 1000), ("c2_mid_bf16", 300)])
def test_select_column_split_matches_unsplit(name, B, tmp_path):
    """Scorer rows split over S = 2 or 4 CTAs (MSN_SELECT_SPLIT=S; the default
    for small grids picks the largest S that fits one wave) and scored by one
    CTA (=0: two sweeps for n_sub > 512) select the same slots: idx, w and
    out bitwise equal (separate processes: the switch is read once per
    process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("0", "2", "4", None):
        f = str(tmp_path / f"r{mode}.pt")
        env = dict(os.environ)
        env.pop("MSN_SELECT_SPLIT", None)
        if mode is not None:
            env["MSN_SELECT_SPLIT"] = mode
        subprocess.run([sys.executable, "-c", _SPLIT_SCRIPT, root, name, str(B), f], env=env, check=True,
                       timeout=600)
        res[mode] = torch.load(f)
    for mode in ("2", "4", None):
        for key in ("idx", "w", "out"):
            assert torch.equal(res["0"][key], res[mode][key]), (mode, key)


@pytest.mark.parametrize("name,B,groups,kw", [("c2_mid_bf16", 8192 + 37, 1, {}),
                                              ("c3_train_fp32_zipf", 8192 + 5, 1, {}),
                                              ("f4_tokens_bf16", 40, 16, {}), ("c5_latency_bf16", 8192 + 3, 1, {}),
                                              ("c5_latency_bf16", 512, 1, {}), ("c5_latency_bf16", 130, 1, {}),
                                              ("c5_latency_bf16", 61, 1, {"heads": 8}),
                                              ("c3_train_fp32_zipf", 77, 1, {"d_value": 256})])
def test_fused_forward_matches_phases(name, B, groups, kw):
    """msn_pkm_forward (fused Cartesian + gather: per query for B >= 8192,
    per lookup below -- the warp-specialised kernel for rows of 64 vectors)
    and the phase calls select + gather add in the same order
    (gather_rows.cuh): bitwise equal idx, weights and outputs."""
    cfg = wl.CONFIGS[name].scaled(batch=B, **kw)
    Q, K, V, _ = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg, head_groups=groups)
    out, idx, w = lk.forward(Q, K, V)
    i2, w2 = lk.select(Q, K)
    o2 = lk.gather(i2, w2, V)
    torch.cuda.synchronize()
    assert torch.equal(idx, i2) and torch.equal(w, w2)
    assert torch.equal(out, o2)


def test_step_host_pipelined_matches_device():
    """PKMLookup.step_host (host buffers, 4 slices with copies overlapping the
    kernels): out and d_query are per-query results, bitwise equal to the
    device-resident forward/backward; d_values / d_subkeys receive the slices'
    sums one after another (equal up to fp32 reassociation)."""
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=4096 + 200)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, _ = lk.backward(dOut, Q, K, V, idx, w)
    dK2 = torch.zeros_like(dK)
    dV2 = torch.zeros_like(dV)
    out_h, dq_h = lk.step_host(Q.cpu().pin_memory(), dOut.cpu().pin_memory(), K, V, dK2, dV2, chunks=4)
    assert torch.equal(out_h, out.cpu()) and torch.equal(dq_h, dq.cpu())
    torch.testing.assert_close(dV2, dV, rtol=1e-5, atol=1e-7)
    torch.testing.assert_close(dK2, dK, rtol=1e-4, atol=1e-6)


def scorer_supports(n_sub, d_h, k, qdt):
    """The tcgen05 scorer's shape rule (the library's only scorer; anything
    else is refused with MSN_ERR_UNSUPPORTED before a launch)."""
    if qdt == torch.bfloat16:
        ok_d = d_h % 64 == 0 and d_h <= 256
    else:
        ok_d = d_h % 32 == 0 and d_h <= 128
    return ok_d and n_sub % 32 == 0 and k <= 64


def _random_shapes(n, seed=2602, supported=True):
    """Seeded random shapes across the library's ranges: B ragged, H up to 8,
    n_sub from 16 to 1024 (tcgen05 resident and two-sweep rows), d_h / d_v of
    every per-lane width the kernels template on, k from 1 to 64, fp32 / bf16
    keys and values -- the ones the scorer takes (supported=True) or the ones
    it refuses."""
    import random
    rnd = random.Random(seed)
    dts = [torch.float32, torch.bfloat16]
    out = []
    while len(out) < n:
        n_sub = rnd.choice([16, 32, 48, 64, 96, 128, 192, 256, 384, 512, 640, 768, 1024])
        k = rnd.randint(1, min(64, n_sub))
        H = rnd.choice([1, 2, 3, 4, 8])
        if H * k > 512:
            continue
        shp = (rnd.randint(1, 400), H, n_sub, rnd.choice([32, 64, 128, 256]),
               rnd.choice([32, 64, 128, 256, 512]), k, rnd.choice(dts), rnd.choice(dts))
        if scorer_supports(shp[2], shp[3], shp[5], shp[6]) == supported:
            out.append(shp)
    return out


@pytest.mark.parametrize("shape", _random_shapes(6, seed=77, supported=False),
                         ids=lambda s: "x".join(str(v) for v in s[:6]) + f"-{str(s[6])[6:]}")
def test_unsupported_shapes_refused(shape):
    """Shapes outside the tcgen05 scorer's rule: forward returns
    MSN_ERR_UNSUPPORTED before any launch (there is no second scorer)."""
    from paper_2602_07526_b200._lib import MsnError
    B, H, n_sub, d_h, d_v, k, qdt, vdt = shape
    cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, qdt, vdt, index=300 + n_sub + k)
    Q, K, V, _ = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    with pytest.raises(MsnError, match="UNSUPPORTED"):
        lk.forward(Q, K, V)


@pytest.mark.parametrize("shape", _random_shapes(24),
                         ids=lambda s: "x".join(str(v) for v in s[:6]) + f"-{str(s[6])[6:]}-{str(s[7])[6:]}")
def test_random_shapes_fwd_bwd(shape):
    B, H, n_sub, d_h, d_v, k, qdt, vdt = shape
    cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, qdt, vdt, index=500 + n_sub + k + H)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_fwd_bwd(cfg, Q, K, V, dOut)
    check_all(cfg, Q, K, V, dOut, res)


@pytest.mark.parametrize("name", ["c2_mid_bf16", "c4_large_sharded_bf16"])
def test_dq_in_query_dtype(name):
    """MSN_FLAG_DQ_QK_DTYPE: d_query comes back in bf16, the fp32 result rounded
    once (RNE) -- on the tensor-core dQ path (C2) and the per-lookup dQ of
    long codebooks (C4)."""
    cfg = wl.CONFIGS[name].scaled(batch=300)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    lk = lookup_for(cfg)
    lk16 = lookup_for(cfg, dq_in_qk_dtype=True)
    out, idx, w = lk.forward(Q, K, V)
    dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
    dq16, dK16, dV16, dw16 = lk16.backward(dOut, Q, K, V, idx, w)
    torch.cuda.synchronize()
    assert dq16.dtype == torch.bfloat16
    assert torch.equal(dq16, dq.to(torch.bfloat16))
    assert torch.equal(dK16, dK) and torch.equal(dV16, dV) and torch.equal(dw16, dw)
