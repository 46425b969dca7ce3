"""Seeded synthetic inputs for the PKM lookup (BASELINE.json configs[0..4]).

This module is the ONE thing shared by the CUDA path's tests/bench and the
fp64 oracle: it draws random tensors and nothing else.  It holds none of the
method's arithmetic (no scoring, no top-k, no softmax, no gather) -- only the
input recipe of DESIGN.md section "Inputs":

* queries  Q [B, H, 2, d_h]  ~ N(0, 1)           (C3: Zipf(1.1)-clustered)
* sub-keys K [H, 2, n_sub, d_h] ~ N(0, sigma_k^2), then each row L2-normalised
  (BASELINE.json configs[*]: "L2-normalised")
* values   V [n_sub^2, d_v]  ~ N(0, 0.02^2)      (0.02 read as the std,
  SURVEY.md 8(c) point 13)
* upstream gradient dOut [B, d_v] ~ N(0, 1)      (fp32)

Tensors are drawn in fp32 with a torch.Generator on the requested device and
then rounded ONCE (RNE) to the config's storage dtype; the oracle and the GPU
consume the same stored bytes.  Seeds: base = 7526 + config index; Q base+1,
K base+2, V base+3, dOut base+4, cluster ids/centres base+5.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import torch


@dataclasses.dataclass(frozen=True)
class PKMConfig:
    name: str
    index: int            # position in BASELINE.json configs
    batch: int            # B (queries)
    heads: int            # H
    d_half: int           # d_h, per-half query / sub-key width
    n_sub: int            # sqrt(n), keys per sub-key codebook
    d_value: int          # d_v
    k: int                # per-half and final top-k
    qk_dtype: torch.dtype
    value_dtype: torch.dtype
    key_std: float        # std of sub-key entries before L2 normalisation
    zipf_clusters: int = 0        # C3: number of Zipf-weighted cluster centres
    zipf_s: float = 1.1
    zipf_sigma: float = 0.5
    backward: bool = True
    deterministic: bool = True
    head_groups: int = 1          # f4: tokens (groups of heads/groups heads), out [B, G, d_v]
    group_tables: bool = False    # f4: one value table per group

    @property
    def n_slots(self) -> int:
        """Rows of the value table (all groups' tables when group_tables)."""
        return self.n_sub * self.n_sub * (self.head_groups if self.group_tables else 1)

    @property
    def out_shape_tail(self):
        return (self.d_value,) if self.head_groups == 1 else (self.head_groups, self.d_value)

    @property
    def lookups(self) -> int:
        return self.batch * self.heads

    def scaled(self, batch: Optional[int] = None, **kw) -> "PKMConfig":
        d = dataclasses.asdict(self)
        if batch is not None:
            d["batch"] = batch
        d.update(kw)
        return PKMConfig(**d)


# BASELINE.json configs[0..4].
CONFIGS = {
    "c1_tiny_fp32": PKMConfig("c1_tiny_fp32", 0, 256, 1, 64, 128, 64, 8,
                              torch.float32, torch.float32, key_std=1.0 / 8.0,
                              backward=False),
    "c2_mid_bf16": PKMConfig("c2_mid_bf16", 1, 4096, 4, 256, 512, 256, 32,
                             torch.bfloat16, torch.bfloat16, key_std=1.0),
    "c3_train_fp32_zipf": PKMConfig("c3_train_fp32_zipf", 2, 16384, 8, 128, 1024, 128, 16,
                                    torch.float32, torch.float32, key_std=1.0,
                                    zipf_clusters=1024),
    "c4_large_sharded_bf16": PKMConfig("c4_large_sharded_bf16", 3, 32768, 4, 256, 2048, 256, 32,
                                       torch.bfloat16, torch.bfloat16, key_std=1.0),
    "c5_latency_bf16": PKMConfig("c5_latency_bf16", 4, 512, 4, 128, 1024, 512, 32,
                                 torch.bfloat16, torch.bfloat16, key_std=1.0,
                                 backward=False),
    # the paper's deployed design -- token-specific query
    # networks and sub-keys, one value table shared by the layer's tokens
    # (hybrid allocation), n = 256^2, k = 32, a
    # batch of 2048 x 16 tokens.  d_v = 1024 (the
    # paper's width is not stated; SURVEY E8 infers ~1024), d_h = 128.  One
    # head per token: 16 groups.
    "f4_tokens_bf16": PKMConfig("f4_tokens_bf16", 5, 2048, 16, 128, 256, 1024, 32,
                                torch.bfloat16, torch.bfloat16, key_std=1.0, head_groups=16),
    # ... and the per-token value tables of the paper's "per-token V" ablation
    # (PAPER.md:446): 16 tables of 256^2 rows.
    "f4_tokens_pertable_bf16": PKMConfig("f4_tokens_pertable_bf16", 6, 2048, 16, 128, 256, 1024, 32,
                                         torch.bfloat16, torch.bfloat16, key_std=1.0, head_groups=16,
                                         group_tables=True),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _randn(shape, seed, device, chunk_rows: int = 1 << 20) -> torch.Tensor:
    """fp32 N(0,1) drawn row-chunk by row-chunk from one generator (keeps host
    peak memory bounded for the 4M-row table; the stream is fixed by the seed,
    the shape and chunk_rows)."""
    g = _gen(seed, device)
    out = torch.empty(shape, dtype=torch.float32, device=device)
    flat = out.view(shape[0], -1)
    for r0 in range(0, shape[0], chunk_rows):
        r1 = min(shape[0], r0 + chunk_rows)
        flat[r0:r1] = torch.randn((r1 - r0, flat.shape[1]), generator=g, device=device)
    return out


def make_queries(cfg: PKMConfig, device="cpu", batch: Optional[int] = None) -> torch.Tensor:
    """Q [B, H, 2, d_h] in cfg.qk_dtype.  Half 0 feeds K_row (index i), half 1
    feeds K_col (index j) (SURVEY.md 8(c) point 4)."""
    B = cfg.batch if batch is None else batch
    base = 7526 + cfg.index
    shape = (B, cfg.heads, 2, cfg.d_half)
    if cfg.zipf_clusters:
        width = cfg.heads * 2 * cfg.d_half
        g = _gen(base + 5, device)
        centres = torch.randn((cfg.zipf_clusters, width), generator=g, device=device)
        ranks = torch.arange(1, cfg.zipf_clusters + 1, dtype=torch.float64, device=device)
        p = ranks.pow(-cfg.zipf_s)
        p = (p / p.sum()).to(torch.float32)
        cid = torch.multinomial(p, B, replacement=True, generator=g)
        eps = _randn((B, width), base + 1, device)
        q = centres[cid] + cfg.zipf_sigma * eps
        q = q.view(shape)
    else:
        q = _randn(shape, base + 1, device)
    return q.to(cfg.qk_dtype).contiguous()


def make_subkeys(cfg: PKMConfig, device="cpu") -> torch.Tensor:
    """K [H, 2, n_sub, d_h], rows L2-normalised in fp32 then rounded."""
    base = 7526 + cfg.index
    k = _randn((cfg.heads, 2, cfg.n_sub, cfg.d_half), base + 2, device) * cfg.key_std
    k = k / k.norm(dim=-1, keepdim=True)
    return k.to(cfg.qk_dtype).contiguous()


def make_values(cfg: PKMConfig, device="cpu") -> torch.Tensor:
    """V [n_slots, d_v] ~ N(0, 0.02^2) (n_slots = G n_sub^2 with group tables)."""
    base = 7526 + cfg.index
    v = _randn((cfg.n_slots, cfg.d_value), base + 3, device)
    v.mul_(0.02)
    return v.to(cfg.value_dtype).contiguous()


def make_dout(cfg: PKMConfig, device="cpu", batch: Optional[int] = None) -> torch.Tensor:
    """dOut [B, d_v] (or [B, G, d_v] with head groups) fp32 ~ N(0,1) (the
    dense upstream gradient of configs[1..3])."""
    B = cfg.batch if batch is None else batch
    base = 7526 + cfg.index
    return _randn((B,) + tuple(cfg.out_shape_tail), base + 4, device).contiguous()


def make_all(cfg: PKMConfig, device="cpu", batch: Optional[int] = None):
    return (make_queries(cfg, device, batch), make_subkeys(cfg, device),
            make_values(cfg, device), make_dout(cfg, device, batch))


def tiny_config(batch=8, heads=2, d_half=16, n_sub=16, d_value=16, k=4,
                dtype=torch.float32, value_dtype=None, index=90) -> PKMConfig:
    """Small ad-hoc shapes for tests (index only picks the seed)."""
    return PKMConfig(f"tiny_{index}", index, batch, heads, d_half, n_sub, d_value, k,
                     dtype, value_dtype or dtype, key_std=1.0)
