"""The seeded synthetic input recipe (BASELINE.json configs)."""
import torch

from paper_2602_07526_b200 import workloads as wl


def test_configs_match_baseline_shapes():
    c = wl.CONFIGS
    assert (c["c1_tiny_fp32"].batch, c["c1_tiny_fp32"].n_slots, c["c1_tiny_fp32"].k) == (256, 16384, 8)
    assert (c["c2_mid_bf16"].heads, c["c2_mid_bf16"].n_slots, c["c2_mid_bf16"].d_value) == (4, 262144, 256)
    assert (c["c3_train_fp32_zipf"].batch, c["c3_train_fp32_zipf"].n_slots) == (16384, 1048576)
    assert (c["c4_large_sharded_bf16"].batch, c["c4_large_sharded_bf16"].n_slots) == (32768, 4194304)
    assert (c["c5_latency_bf16"].d_value, c["c5_latency_bf16"].k) == (512, 32)
    for cfg in c.values():
        assert 2 * cfg.d_half in (128, 256, 512)


def test_generators_are_seeded_and_shaped():
    cfg = wl.CONFIGS["c2_mid_bf16"].scaled(batch=64)
    q1, q2 = wl.make_queries(cfg), wl.make_queries(cfg)
    assert q1.shape == (64, 4, 2, 256) and q1.dtype == torch.bfloat16
    assert torch.equal(q1, q2)
    k = wl.make_subkeys(cfg)
    assert k.shape == (4, 2, 512, 256)
    norms = k.float().norm(dim=-1)
    assert torch.allclose(norms, torch.ones_like(norms), atol=2e-2)
    d = wl.make_dout(cfg)
    assert d.shape == (64, 256) and d.dtype == torch.float32


def test_fp32_keys_unit_norm():
    cfg = wl.CONFIGS["c1_tiny_fp32"]
    k = wl.make_subkeys(cfg)
    assert k.dtype == torch.float32
    assert torch.allclose(k.norm(dim=-1), torch.ones(1), atol=1e-6)
    v = wl.make_values(cfg)
    assert v.shape == (16384, 64)
    assert abs(float(v.std()) - 0.02) < 1e-3


def test_zipf_queries_are_clustered():
    cfg = wl.CONFIGS["c3_train_fp32_zipf"].scaled(batch=2048)
    q = wl.make_queries(cfg).view(2048, -1)
    # queries of the most popular centre are close to each other: many
    # near-duplicate pairs compared with iid N(0,1) queries
    qs = q[:256]
    d = torch.cdist(qs, qs)
    close = (d < 0.6 * d.median()).sum().item() - 256
    assert close > 256
