"""Pins of the memory-gated fusion oracle (oracle/gate.py; SURVEY.md 8(f)
f1; Eq. gating, gate ablation PAPER.md:492): special
values of the gate, the identity gate's exact product form, saturation,
and central finite differences of the whole chain
L = <dx~, x (.) g(PKM(Q, K, V))> against the oracle backward (gate backward
feeding the PKM backward), on tie-free instances."""
import numpy as np
import pytest

from oracle import gate as og
from oracle import oracle as orc



def test_zero_memory_output():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 7))
    v = np.zeros_like(x)
    assert np.array_equal(og.forward(v, x, "tanh"), np.zeros_like(x))      # tanh(0) = 0
    assert np.array_equal(og.forward(v, x, "identity"), np.zeros_like(x))
    assert np.allclose(og.forward(v, x, "sigmoid"), x / 2, rtol=0, atol=0)  # sigmoid(0) = 1/2
    d = rng.standard_normal(x.shape)
    dx, dv = og.backward(v, x, d, "tanh")                                    # tanh'(0) = 1
    assert np.array_equal(dx, np.zeros_like(x)) and np.array_equal(dv, d * x)
    dx, dv = og.backward(v, x, d, "sigmoid")                                 # sigmoid'(0) = 1/4
    assert np.allclose(dx, d / 2, rtol=0, atol=0) and np.allclose(dv, d * x / 4, rtol=0, atol=1e-18)


def test_identity_gate_is_the_product():
    rng = np.random.default_rng(1)
    x, v, d = (rng.standard_normal((4, 9)) for _ in range(3))
    assert np.array_equal(og.forward(v, x, "identity"), x * v)
    dx, dv = og.backward(v, x, d, "identity")
    assert np.array_equal(dx, d * v) and np.array_equal(dv, d * x)


def test_saturation_and_odd_symmetry():
    x = np.array([[1.5, -2.0, 0.25]])
    big = np.full_like(x, 40.0)
    assert np.array_equal(og.forward(big, x, "tanh"), x)          # tanh(40) == 1 in fp64
    assert np.array_equal(og.forward(-big, x, "tanh"), -x)
    assert np.array_equal(og.forward(big, x, "sigmoid"), x)
    v = np.array([[0.3, -0.7, 1.1]])
    assert np.allclose(og.forward(-v, x, "tanh"), -og.forward(v, x, "tanh"), rtol=1e-15)


def _chain_loss(Q, K, V, X, dxt, k, gate, idx_fixed):
    r = orc.forward(Q, K, V, k)
    assert np.array_equal(r["idx"], idx_fixed)  # same selection: smooth region
    return float((dxt * og.forward(r["out"], X, gate)).sum())


@pytest.mark.parametrize("gate", og.GATES)
def test_finite_differences_through_gate_and_lookup(gate):
    rng = np.random.default_rng(7)
    B, H, n_sub, d_h, d_v, k = 3, 2, 8, 4, 6, 3
    for trial in range(50):
        Q = rng.standard_normal((B, H, 2, d_h))
        K = rng.standard_normal((H, 2, n_sub, d_h))
        V = rng.standard_normal((n_sub * n_sub, d_v))
        r = orc.forward(Q, K, V, k)
        # tie-free: gaps around the k-th Cartesian score
        sc = orc.slot_scores(Q, K, np.tile(np.arange(n_sub * n_sub), (B, H, 1)))
        srt = -np.sort(-sc, axis=-1)
        if np.min(srt[..., k - 1] - srt[..., k]) > 1e-3:
            break
    X = rng.standard_normal((B, d_v))
    dxt = rng.standard_normal((B, d_v))
    dx, dvo = og.backward(r["out"], X, dxt, gate)
    bw = orc.backward(Q, K, V, r["idx"], dvo)
    h = 1e-6
    for name, arr, grad in (("X", X, dx), ("V", V, bw["dV"]), ("Q", Q, bw["dQ"])):
        flat = arr.reshape(-1)
        g = grad.reshape(-1)
        for pos in rng.choice(flat.size, size=min(12, flat.size), replace=False):
            old = flat[pos]
            flat[pos] = old + h
            lp = _chain_loss(Q, K, V, X, dxt, k, gate, r["idx"])
            flat[pos] = old - h
            lm = _chain_loss(Q, K, V, X, dxt, k, gate, r["idx"])
            flat[pos] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[pos]) <= 1e-5 * max(1.0, abs(fd)), (gate, name, pos, fd, g[pos])
