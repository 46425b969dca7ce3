"""The GPU-vs-oracle comparator (tests/parity.py) is itself checked on CPU:
it accepts the oracle's own results, and rejects a wrong output, a
non-tie swap and a duplicated slot."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2602_07526_b200 import workloads as wl
from tests import parity


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).float()


@pytest.fixture(scope="module")
def case():
    cfg = wl.tiny_config(16, 2, 32, 64, 64, 8, torch.float32, torch.float32, index=91)
    Q, K, V, d = wl.make_all(cfg)
    o = orc.forward(Q, K, V, cfg.k)
    b = orc.backward(Q, K, V, o["idx"], d)
    return cfg, Q, K, V, d, o, b


def test_accepts_oracle_itself(case):
    cfg, Q, K, V, d, o, b = case
    o2, aff, rep = parity.check_forward(Q, K, V, cfg.k, _t(o["out"]), torch.from_numpy(o["idx"]).int(), _t(o["w"]))
    assert not aff.any()
    parity.check_backward(Q, K, V, cfg.k, d, o2, aff, _t(b["dQ"]), _t(b["dK"]), _t(b["dV"]), _t(b["dw"]),
                          gpu_idx=o["idx"])


def test_rejects_wrong_output(case):
    cfg, Q, K, V, d, o, b = case
    out = o["out"].copy()
    out[3, 5] += 1e-3 * np.abs(out[3]).max() + 1e-3
    with pytest.raises(AssertionError, match="out"):
        parity.check_forward(Q, K, V, cfg.k, _t(out), torch.from_numpy(o["idx"]).int(), _t(o["w"]))


def test_rejects_wrong_gradient(case):
    cfg, Q, K, V, d, o, b = case
    dK = b["dK"].copy()
    nz = np.argwhere(np.abs(dK).sum(-1) > 0)[0]
    dK[tuple(nz)] *= 1.01
    with pytest.raises(AssertionError, match="dK"):
        parity.check_backward(Q, K, V, cfg.k, d, o, np.zeros((16, 2), bool), _t(b["dQ"]), _t(dK),
                              _t(b["dV"]), _t(b["dw"]), gpu_idx=o["idx"])


def test_rejects_non_tie_swap(case):
    cfg, Q, K, V, d, o, b = case
    idx = o["idx"].copy()
    # replace the best slot by a slot far down the ranking
    s1 = (K[0, 0].double() @ Q[0, 0, 0].double()).numpy()
    s2 = (K[0, 1].double() @ Q[0, 1, 1 - 1].double()).numpy() if False else (K[0, 1].double() @ Q[0, 0, 1].double()).numpy()
    worst = int(np.argmin(s1)) * cfg.n_sub + int(np.argmin(s2))
    idx[0, 0, 0] = worst
    with pytest.raises(AssertionError, match="gap"):
        parity.compare_selection(Q, K, idx, o, cfg.n_sub)


def test_rejects_duplicates_and_range(case):
    cfg, Q, K, V, d, o, b = case
    idx = o["idx"].copy()
    idx[1, 1, 1] = idx[1, 1, 0]
    with pytest.raises(AssertionError, match="duplicate"):
        parity.compare_selection(Q, K, idx, o, cfg.n_sub)
    idx = o["idx"].copy()
    idx[0, 0, 0] = cfg.n_sub * cfg.n_sub
    with pytest.raises(AssertionError, match="range"):
        parity.compare_selection(Q, K, idx, o, cfg.n_sub)


def test_accepts_a_genuine_tie_swap():
    """Two slots with exactly equal scores: either may be selected."""
    n = 4
    Q = np.zeros((1, 1, 2, n))
    Q[0, 0, 0] = [3.0, 1.0, 0.0, -1.0]
    Q[0, 0, 1] = [2.0, 2.0, 0.0, -5.0]
    K = np.zeros((1, 2, n, n))
    K[0, 0] = np.eye(n)
    K[0, 1] = np.eye(n)
    V = np.random.default_rng(0).standard_normal((n * n, 4))
    o = orc.forward(Q, K, V, 1)          # tie (0,0) vs (0,1): flat 0 wins
    assert o["idx"][0, 0, 0] == 0
    aff, rep = parity.compare_selection(Q, K, np.array([[[1]]]), o, n)
    assert aff[0, 0] and rep["worst_tie_gap"] == 0.0
