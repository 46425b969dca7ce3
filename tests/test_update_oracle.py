"""Pins of the fused sparse optimiser oracle (oracle/update.py; SURVEY.md
8(f) f3; "gradient updates"): lr = 0 is the identity, the SGD
step of a single contribution is V - lr w d_out, a first Adagrad step from
zero state moves every touched element by lr g/(|g| + eps), untouched rows
and state never change, and SGD on the oracle's dV equals a finite-difference
descent direction of L = <d_out, out> in V."""
import numpy as np
import pytest

from oracle import oracle as orc
from oracle import update as ou


def _instance(seed=0, B=4, H=2, n_sub=8, d_h=4, d_v=6, k=3):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((B, H, 2, d_h))
    K = rng.standard_normal((H, 2, n_sub, d_h))
    V = rng.standard_normal((n_sub * n_sub, d_v))
    dOut = rng.standard_normal((B, d_v))
    r = orc.forward(Q, K, V, k)
    bw = orc.backward(Q, K, V, r["idx"], dOut, want_dense_dv=False)
    return Q, K, V, dOut, r, bw


@pytest.mark.parametrize("kind", ou.UPDATES)
def test_zero_lr_is_identity(kind):
    _, _, V, _, _, bw = _instance()
    st = np.zeros_like(V)
    Vn, _ = ou.apply(V, bw["rows"], bw["dV"], kind, 0.0, state=st)
    assert np.array_equal(Vn, V)


def test_single_contribution_sgd_closed_form():
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((1, 1, 2, 4))
    K = rng.standard_normal((1, 2, 8, 4))
    V = rng.standard_normal((64, 5))
    dOut = rng.standard_normal((1, 5))
    r = orc.forward(Q, K, V, 1)            # k = 1: one row, weight exactly 1
    bw = orc.backward(Q, K, V, r["idx"], dOut, want_dense_dv=False)
    Vn, _ = ou.apply(V, bw["rows"], bw["dV"], "sgd", 0.25)
    f = int(r["idx"][0, 0, 0])
    expect = V.copy()
    expect[f] = V[f] - 0.25 * dOut[0]
    assert np.allclose(Vn, expect, rtol=0, atol=1e-15)


def test_first_adagrad_step_moves_by_lr_sign():
    _, _, V, _, _, bw = _instance(seed=2)
    eps = 1e-10
    Vn, s = ou.apply(V, bw["rows"], bw["dV"], "adagrad", 0.01, eps, state=np.zeros_like(V))
    g = bw["dV"]
    assert np.allclose(s[bw["rows"]], g * g, rtol=0, atol=0)
    assert np.allclose(V[bw["rows"]] - Vn[bw["rows"]], 0.01 * g / (np.abs(g) + eps), rtol=1e-12)


@pytest.mark.parametrize("kind", ou.UPDATES)
def test_untouched_rows_and_state_unchanged(kind):
    _, _, V, _, _, bw = _instance(seed=3)
    st = np.full_like(V, 0.5)
    Vn, s = ou.apply(V, bw["rows"], bw["dV"], kind, 0.1, state=st)
    untouched = np.setdiff1d(np.arange(V.shape[0]), bw["rows"])
    assert np.array_equal(Vn[untouched], V[untouched])
    if s is not None:
        assert np.array_equal(s[untouched], st[untouched])


def test_sgd_step_is_the_finite_difference_descent():
    """For tiny lr the SGD update changes L = <dOut, out(V)> by
    -lr * |dV|^2 (out is linear in V at a fixed selection)."""
    Q, K, V, dOut, r, bw = _instance(seed=4)
    lr = 1e-7
    Vn, _ = ou.apply(V, bw["rows"], bw["dV"], "sgd", lr)
    L0 = float((dOut * orc.forward(Q, K, V, 3)["out"]).sum())
    L1 = float((dOut * orc.forward(Q, K, Vn, 3)["out"]).sum())
    pred = -lr * float((bw["dV"] ** 2).sum())
    assert abs((L1 - L0) - pred) <= 1e-6 * abs(pred)
