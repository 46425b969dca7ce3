"""Pins of the query/key prologue oracle (oracle/prologue.py; SURVEY.md 8(f)
f2; LayerNorm PAPER.md:275, key over-parameterisation and its gradients
PAPER.md:287-302): LN closed forms and invariances, Theta = I is the
identity, finite differences of both backward passes, and the paper's
dL/dTheta = dL/dK_tilde K^T written out per key vector."""
import numpy as np
import pytest

from oracle import prologue as op


def test_layernorm_moments_and_invariances():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((7, 32)) * 3 + 1.5
    y = op.layernorm(x)
    var = x.var(axis=-1, keepdims=True)
    assert np.allclose(y.mean(axis=-1), 0, atol=1e-13)
    assert np.allclose((y ** 2).mean(axis=-1), (var / (var + op.EPS)).ravel(), rtol=1e-12)
    assert np.allclose(op.layernorm(2.5 * x - 4.0, eps=0.0), op.layernorm(x, eps=0.0), rtol=1e-12, atol=1e-12)
    assert np.array_equal(op.layernorm(np.full((2, 8), 3.25)), np.zeros((2, 8)))  # constant row -> 0


def test_theta_identity_and_single_key():
    rng = np.random.default_rng(1)
    K = rng.standard_normal((2, 2, 5, 4))
    I = np.broadcast_to(np.eye(4), (2, 2, 4, 4))
    assert np.allclose(op.key_transform(K, I), K, rtol=0, atol=0)
    T = rng.standard_normal((2, 2, 4, 4))
    Kt = op.key_transform(K, T)
    h, c, i = 1, 0, 3
    assert np.allclose(Kt[h, c, i], T[h, c] @ K[h, c, i], rtol=1e-14)  # k_tilde_i = Theta k_i


def test_paper_theta_gradient_per_key_vector():
    rng = np.random.default_rng(2)
    K = rng.standard_normal((1, 2, 6, 3))
    T = rng.standard_normal((1, 2, 3, 3))
    G = rng.standard_normal((1, 2, 6, 3))
    dK, dT = op.key_transform_backward(K, T, G)
    for c in range(2):
        expect = sum(np.outer(G[0, c, i], K[0, c, i]) for i in range(6))   # sum_i dk~_i k_i^T
        assert np.allclose(dT[0, c], expect, rtol=1e-13)
        for i in range(6):
            assert np.allclose(dK[0, c, i], T[0, c].T @ G[0, c, i], rtol=1e-13)  # Theta^T dk~_i


@pytest.mark.parametrize("what", ["ln", "theta"])
def test_finite_differences(what):
    rng = np.random.default_rng(3)
    h = 1e-6
    if what == "ln":
        x = rng.standard_normal((4, 16))
        dy = rng.standard_normal((4, 16))
        g = op.layernorm_backward(x, dy)
        for pos in rng.choice(x.size, 20, replace=False):
            xp, xm = x.copy().ravel(), x.copy().ravel()
            xp[pos] += h
            xm[pos] -= h
            fd = ((dy * op.layernorm(xp.reshape(x.shape))).sum() - (dy * op.layernorm(xm.reshape(x.shape))).sum()) / (2 * h)
            assert abs(fd - g.ravel()[pos]) <= 1e-6 * max(1.0, abs(fd))
    else:
        K = rng.standard_normal((2, 2, 5, 4))
        T = rng.standard_normal((2, 2, 4, 4))
        G = rng.standard_normal((2, 2, 5, 4))
        dK, dT = op.key_transform_backward(K, T, G)
        for arr, grad in ((K, dK), (T, dT)):
            for pos in rng.choice(arr.size, 15, replace=False):
                flat = arr.reshape(-1)
                old = flat[pos]
                flat[pos] = old + h
                lp = (G * op.key_transform(K, T)).sum()
                flat[pos] = old - h
                lm = (G * op.key_transform(K, T)).sum()
                flat[pos] = old
                assert abs((lp - lm) / (2 * h) - grad.reshape(-1)[pos]) <= 1e-6
