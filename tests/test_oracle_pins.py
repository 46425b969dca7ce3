"""Pins of the fp64 oracle (oracle/) against things other than itself:
hand-derived golden fixtures, the exhaustive full-memory scorer, closed forms,
invariants and central finite differences.  CPU only (no GPU marker).

Each test names the passage or reading it pins (DESIGN.md "Oracle and its
pins").
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import brute
from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def identity_instance(s_row, s_col, H=1, d_v=None, V=None):
    """Identity codebooks (n_sub = d_h) make S_row = q_row, S_col = q_col
    exactly, so crafted score vectors can be fed through
    the full forward."""
    n = len(s_row)
    Q = np.zeros((1, H, 2, n))
    Q[0, :, 0] = s_row
    Q[0, :, 1] = s_col
    K = np.zeros((H, 2, n, n))
    K[:, 0] = np.eye(n)
    K[:, 1] = np.eye(n)
    if V is None:
        d_v = d_v or 4
        V = np.arange(n * n * d_v, dtype=np.float64).reshape(n * n, d_v)
    return Q, K, np.asarray(V, dtype=np.float64)


def random_instance(rng, B, H, n_sub, d_h, d_v, integer=False):
    if integer:
        Q = rng.integers(-2, 3, size=(B, H, 2, d_h)).astype(np.float64)
        K = rng.integers(-1, 2, size=(H, 2, n_sub, d_h)).astype(np.float64)
    else:
        Q = rng.standard_normal((B, H, 2, d_h))
        K = rng.standard_normal((H, 2, n_sub, d_h))
        K /= np.linalg.norm(K, axis=-1, keepdims=True)
    V = rng.standard_normal((n_sub * n_sub, d_v)) * 0.02
    return Q, K, V


# ---------------------------------------------------------------- golden ---

@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "combine_*.json"))
                                       + glob.glob(os.path.join(GOLDEN, "tie_*.json"))))
def test_golden_combine(path):
    """SPEC.md:140-141 worked examples + crafted tie case, R5."""
    g = json.load(open(path))
    Q, K, V = identity_instance(g["s_row"], g["s_col"])
    r = orc.forward(Q, K, V, g["k"])
    assert r["idx"][0, 0].tolist() == g["expect_flat"]
    pairs = [[f // g["n_sub"], f % g["n_sub"]] for f in r["idx"][0, 0]]
    assert pairs == g["expect_pairs"]
    np.testing.assert_allclose(r["c"][0, 0], g["expect_scores"], rtol=0, atol=0)
    np.testing.assert_allclose(r["w"][0, 0], g["expect_w"], rtol=1e-15, atol=1e-15)


def test_golden_flat_index():
    """SPEC.md:150 (3,5,16) -> 53; PAPER.md:229 with reading R2."""
    g = json.load(open(os.path.join(GOLDEN, "flat_index.json")))
    n = g["n_sub"]
    s_row = np.zeros(n); s_row[g["i"]] = 1.0
    s_col = np.zeros(n); s_col[g["j"]] = 1.0
    Q, K, V = identity_instance(s_row, s_col)
    r = orc.forward(Q, K, V, 1)
    assert int(r["idx"][0, 0, 0]) == g["expect_flat"]
    np.testing.assert_array_equal(r["out"][0], V[g["expect_flat"]])


def test_golden_n4_forward_backward():
    """Hand-derived n=4, k=2 instance: forward and every gradient."""
    g = json.load(open(os.path.join(GOLDEN, "n4_k2_forward_backward.json")))
    Q, K, V = identity_instance(g["q_row"], g["q_col"], V=g["V"])
    r = orc.forward(Q, K, V, g["k"])
    assert r["idx"][0, 0].tolist() == g["expect_flat"]
    np.testing.assert_allclose(r["c"][0, 0], g["expect_scores"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(r["w"][0, 0], g["expect_w"], rtol=1e-15)
    np.testing.assert_allclose(r["out"][0], g["expect_out"], rtol=1e-15)
    d = np.array([g["dOut"]])
    bw = orc.backward(Q, K, V, r["idx"], d)
    # dw_t = <V[f_t], dOut> = [<(1,2),(1,0)>, <(3,4),(1,0)>]
    np.testing.assert_array_equal(bw["dw"][0, 0], g["expect_dw"])
    # ds_t = w_t (dw_t - sum_u w_u dw_u) = -/+ 2 w0 w1 (softmax Jacobian); the dS of
    # each half is recovered from dQ_col = ds0 K_col[0] + ds1 K_col[1] with K_col = I
    w0, w1 = g["expect_w"]
    np.testing.assert_allclose(g["expect_ds"], [-2 * w0 * w1, 2 * w0 * w1], rtol=1e-15)
    np.testing.assert_allclose(bw["dQ"][0, 0, 1], g["expect_ds"], rtol=1e-14)
    np.testing.assert_allclose(bw["dQ"][0, 0, 0], g["expect_dq_row"], atol=1e-15)
    np.testing.assert_allclose(bw["dQ"][0, 0, 1], g["expect_dq_col"], rtol=1e-14)
    for row, val in g["expect_dV_rows"].items():
        np.testing.assert_allclose(bw["dV"][int(row)], val, rtol=1e-15)
    assert np.all(bw["dV"][2:] == 0)
    np.testing.assert_allclose(bw["dK"][0, 1, 0], g["expect_dK_col_row0"], rtol=1e-14)
    np.testing.assert_allclose(bw["dK"][0, 1, 1], g["expect_dK_col_row1"], rtol=1e-14)
    np.testing.assert_allclose(bw["dK"][0, 0], 0.0, atol=1e-15)


# ----------------------------------------------------------- brute force ---

@pytest.mark.parametrize("integer", [False, True])
def test_pkm_equals_exhaustive(integer):
    """PAPER.md:207,218-222 + north_star: the product-key top-k must equal the
    exhaustive top-k over all n_sub^2 slots (tie rule R5 makes it unique)."""
    rng = np.random.default_rng(2602 + integer)
    for trial in range(40):
        n_sub = int(rng.integers(2, 33))
        k = int(rng.integers(1, n_sub + 1))
        H = int(rng.integers(1, 3))
        d_h = int(rng.integers(1, 9))
        Q, K, V = random_instance(rng, 3, H, n_sub, d_h, 5, integer=integer)
        r = orc.forward(Q, K, V, k)
        b = brute.forward(Q, K, V, k)
        np.testing.assert_array_equal(r["idx"], b["idx"], err_msg=f"trial {trial}")
        np.testing.assert_allclose(r["c"], b["c"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(r["w"], b["w"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(r["out"], b["out"], rtol=1e-12, atol=1e-15)


def test_per_half_topk_is_stable_sort_prefix():
    """per-half top-k = prefix of the stable (desc) sort;
    [5,5,5,5], k=2 -> [0,1]."""
    Q, K, V = identity_instance([5, 5, 5, 5], [1, 2, 3, 4])
    r = orc.forward(Q, K, V, 2)
    assert r["I"][0, 0].tolist() == [0, 1]
    assert r["J"][0, 0].tolist() == [3, 2]
    rng = np.random.default_rng(7)
    for _ in range(20):
        s = rng.integers(-3, 4, size=12).astype(np.float64)
        t = rng.standard_normal(12)
        Q, K, V = identity_instance(s, t)
        k = int(rng.integers(1, 13))
        r = orc.forward(Q, K, V, k)
        assert r["I"][0, 0].tolist() == np.argsort(-s, kind="stable")[:k].tolist()
        assert r["J"][0, 0].tolist() == np.argsort(-t, kind="stable")[:k].tolist()


def test_identity_codebook_scores_equal_query():
    """identity keys give S = q (per-half scores reported = sorted q)."""
    rng = np.random.default_rng(11)
    s, t = rng.standard_normal(8), rng.standard_normal(8)
    Q, K, V = identity_instance(s, t)
    r = orc.forward(Q, K, V, 8)
    np.testing.assert_array_equal(r["s1"][0, 0], np.sort(s)[::-1])
    np.testing.assert_array_equal(r["s2"][0, 0], np.sort(t)[::-1])


# ---------------------------------------------------------- closed forms ---

def test_zero_query_closed_form():
    """q = 0: every score is 0, so idx = [0..k-1] (pairs (0,0)..(0,k-1)),
    w = 1/k and out = H * mean(V[0..k-1])."""
    rng = np.random.default_rng(3)
    B, H, n_sub, d_h, d_v, k = 2, 3, 10, 4, 6, 7
    _, K, V = random_instance(rng, B, H, n_sub, d_h, d_v)
    Q = np.zeros((B, H, 2, d_h))
    r = orc.forward(Q, K, V, k)
    for b in range(B):
        for h in range(H):
            assert r["idx"][b, h].tolist() == list(range(k))
    np.testing.assert_allclose(r["w"], 1.0 / k, rtol=1e-15)
    np.testing.assert_allclose(r["out"], np.broadcast_to(H * V[:k].mean(0), (B, d_v)), rtol=1e-13)


def test_k1_is_exact_row_copy():
    """k=1 -> w=1 and out is an exact value row (per head)."""
    rng = np.random.default_rng(5)
    Q, K, V = random_instance(rng, 4, 1, 9, 5, 7)
    r = orc.forward(Q, K, V, 1)
    np.testing.assert_array_equal(r["w"], 1.0)
    np.testing.assert_array_equal(r["out"], V[r["idx"][:, 0, 0]])


def test_softmax_invariants():
    """sum w = 1; w non-increasing in output order (R1, R5)."""
    rng = np.random.default_rng(13)
    Q, K, V = random_instance(rng, 16, 2, 20, 8, 4)
    r = orc.forward(Q, K, V, 9)
    np.testing.assert_allclose(r["w"].sum(-1), 1.0, atol=1e-14)
    assert np.all(np.diff(r["w"], axis=-1) <= 1e-17)
    assert np.all(np.diff(r["c"], axis=-1) <= 0)
    # idx distinct within a lookup and in range
    for row in r["idx"].reshape(-1, 9):
        assert len(set(row.tolist())) == 9
    assert r["idx"].min() >= 0 and r["idx"].max() < 400


def test_shift_invariance():
    """adding a constant to all of S_row changes neither the
    selection nor the softmax weights (R1 is shift invariant)."""
    rng = np.random.default_rng(17)
    s, t = rng.standard_normal(12), rng.standard_normal(12)
    Q, K, V = identity_instance(s, t)
    Q2, _, _ = identity_instance(s + 0.75, t)
    r, r2 = orc.forward(Q, K, V, 6), orc.forward(Q2, K, V, 6)
    np.testing.assert_array_equal(r["idx"], r2["idx"])
    np.testing.assert_allclose(r["w"], r2["w"], rtol=1e-12)
    np.testing.assert_allclose(r["out"], r2["out"], rtol=1e-12)


def test_output_linear_in_values():
    """out is exactly linear in V at a fixed selection (selection depends on Q,K only)."""
    rng = np.random.default_rng(19)
    Q, K, V = random_instance(rng, 5, 2, 12, 6, 8)
    V2 = rng.standard_normal(V.shape)
    a = orc.forward(Q, K, V, 5)
    b = orc.forward(Q, K, V2, 5)
    c = orc.forward(Q, K, 2.5 * V - V2, 5)
    np.testing.assert_array_equal(a["idx"], c["idx"])
    np.testing.assert_allclose(c["out"], 2.5 * a["out"] - b["out"], rtol=1e-12, atol=1e-14)


def test_per_head_sum():
    """Reading R7: out = sum over heads of the per-head outputs."""
    rng = np.random.default_rng(23)
    Q, K, V = random_instance(rng, 3, 4, 8, 4, 5)
    r = orc.forward(Q, K, V, 3, per_head=True)
    np.testing.assert_allclose(r["out_ph"].sum(1), r["out"], rtol=1e-14, atol=1e-16)


def test_bf16_widening_exact():
    """bf16 inputs are widened bit-exactly (bf16 -> fp32 is exact)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(29)
    Q, K, V = random_instance(rng, 4, 2, 8, 16, 8)
    qb, kb, vb = (torch.from_numpy(x).to(torch.bfloat16) for x in (Q, K, V))
    r1 = orc.forward(qb, kb, vb, 4)
    r2 = orc.forward(qb.float(), kb.float(), vb.float(), 4)
    for key in ("idx", "c", "w", "out"):
        np.testing.assert_array_equal(r1[key], r2[key])


# -------------------------------------------------------------- backward ---

def _loss(Q, K, V, dOut, k, idx_fixed=None):
    r = orc.forward(Q, K, V, k)
    if idx_fixed is not None:
        assert np.array_equal(r["idx"], idx_fixed), "selection changed under perturbation"
    return float((r["out"] * dOut).sum())


def _tie_free(Q, K, V, k, margin=1e-3):
    """True if every per-half and Cartesian selection boundary has a gap > margin."""
    r = orc.forward(Q, K, V, k)
    B, H = Q.shape[:2]
    n_sub = K.shape[2]
    for b in range(B):
        for h in range(H):
            for half in range(2):
                s = np.sort(K[h, half] @ Q[b, h, half])[::-1]
                if k < n_sub and s[k - 1] - s[k] <= margin:
                    return False
            # Cartesian boundary within I x J
            I, J = r["I"][b, h], r["J"][b, h]
            s1, s2 = K[h, 0] @ Q[b, h, 0], K[h, 1] @ Q[b, h, 1]
            c = np.sort((s1[I][:, None] + s2[J][None, :]).ravel())[::-1]
            if c[k - 1] - c[k] <= margin:
                return False
    return True


def test_finite_differences_dQ_dK_dV():
    """every gradient matches central FD (h=1e-6) of
    L = <dOut, out> within rel 1e-5 on tie-free instances; PAPER.md:282-284
    (gradient only through selected scores, reading R10)."""
    rng = np.random.default_rng(31)
    done = 0
    for trial in range(200):
        if done >= 6:
            break
        n_sub, d_h, d_v, k, H, B = 7, 3, 4, 3, 2, 2
        Q, K, V = random_instance(rng, B, H, n_sub, d_h, d_v)
        Q *= 3.0
        if not _tie_free(Q, K, V, k):
            continue
        done += 1
        dOut = rng.standard_normal((B, d_v))
        r = orc.forward(Q, K, V, k)
        g = orc.backward(Q, K, V, r["idx"], dOut)
        h = 1e-6
        for name, X, G in (("Q", Q, g["dQ"]), ("K", K, g["dK"]), ("V", V, g["dV"])):
            flat = X.reshape(-1)
            for pos in rng.choice(flat.size, size=min(flat.size, 25), replace=False):
                old = flat[pos]
                flat[pos] = old + h
                lp = _loss(Q, K, V, dOut, k, r["idx"])
                flat[pos] = old - h
                lm = _loss(Q, K, V, dOut, k, r["idx"])
                flat[pos] = old
                fd = (lp - lm) / (2 * h)
                an = G.reshape(-1)[pos]
                assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)), (name, pos, fd, an)
    assert done >= 6


def test_adjoint_identity_dV():
    """<dOut, out(V+dV_) - out(V)> = <dV, dV_> for any dV_ (out is
    linear in V at the fixed selection)."""
    rng = np.random.default_rng(37)
    Q, K, V = random_instance(rng, 6, 3, 10, 5, 7)
    dOut = rng.standard_normal((6, 7))
    r = orc.forward(Q, K, V, 4)
    g = orc.backward(Q, K, V, r["idx"], dOut)
    delta = rng.standard_normal(V.shape)
    lhs = float((dOut * (orc.forward(Q, K, V + delta, 4)["out"] - r["out"])).sum())
    rhs = float((g["dV"] * delta).sum())
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_dV_row_sum_and_sparsity():
    """sum_rows dV = H * sum_b dOut (because sum_t w = 1); exactly the selected
    rows are non-zero."""
    rng = np.random.default_rng(41)
    B, H = 5, 3
    Q, K, V = random_instance(rng, B, H, 9, 4, 6)
    dOut = rng.standard_normal((B, 6))
    r = orc.forward(Q, K, V, 4)
    g = orc.backward(Q, K, V, r["idx"], dOut)
    np.testing.assert_allclose(g["dV"].sum(0), H * dOut.sum(0), rtol=1e-12, atol=1e-13)
    touched = np.zeros(81, bool)
    touched[r["idx"].reshape(-1)] = True
    assert np.all(np.abs(g["dV"][~touched]) == 0)
    assert np.all(np.abs(g["dV"][touched]).sum(1) > 0)


def test_ds_sums_to_zero_and_unselected_keys_get_no_gradient():
    """sum_t ds_t = 0 per lookup (softmax Jacobian); "unselected
    keys receive no gradients": dK rows of never-selected sub-keys are exactly 0."""
    rng = np.random.default_rng(43)
    B, H, n_sub, k = 4, 2, 16, 3
    Q, K, V = random_instance(rng, B, H, n_sub, 6, 5)
    dOut = rng.standard_normal((B, 5))
    r = orc.forward(Q, K, V, k)
    g = orc.backward(Q, K, V, r["idx"], dOut)
    np.testing.assert_allclose(g["ds"].sum(-1), 0.0, atol=1e-15)
    for h in range(H):
        used_i = set((r["idx"][:, h] // n_sub).reshape(-1).tolist())
        used_j = set((r["idx"][:, h] % n_sub).reshape(-1).tolist())
        for i in range(n_sub):
            if i not in used_i:
                assert np.all(g["dK"][h, 0, i] == 0)
            if i not in used_j:
                assert np.all(g["dK"][h, 1, i] == 0)


def test_zero_upstream_gives_zero_gradients():
    """dOut = 0 -> all gradients exactly 0."""
    rng = np.random.default_rng(47)
    Q, K, V = random_instance(rng, 3, 2, 6, 4, 5)
    r = orc.forward(Q, K, V, 3)
    g = orc.backward(Q, K, V, r["idx"], np.zeros((3, 5)))
    for key in ("dQ", "dK", "dV"):
        assert np.all(g[key] == 0)


def test_compact_dv_rows_match_dense():
    rng = np.random.default_rng(53)
    Q, K, V = random_instance(rng, 4, 2, 8, 4, 3)
    dOut = rng.standard_normal((4, 3))
    r = orc.forward(Q, K, V, 3)
    dense = orc.backward(Q, K, V, r["idx"], dOut)
    comp = orc.backward(Q, K, V, r["idx"], dOut, want_dense_dv=False)
    np.testing.assert_array_equal(comp["dV"], dense["dV"][comp["rows"]])


def test_slot_scores_match_brute():
    rng = np.random.default_rng(59)
    Q, K, V = random_instance(rng, 3, 2, 9, 5, 2)
    b = brute.forward(Q, K, V, 6)
    s = orc.slot_scores(Q, K, b["idx"])
    np.testing.assert_allclose(s, b["c"], rtol=1e-14, atol=1e-15)
