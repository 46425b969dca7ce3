"""Run-length statistics of the grouped backward reductions of a workload
(dV: contributions per value row; dK: distinct (lookup, half, sub-key)
records per sub-key row), from the CUDA forward's selection.

    python tools/run_stats.py c3_train_fp32_zipf
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200.pkm import PKMLookup  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_train_fp32_zipf"
cfg = wl.CONFIGS[name]
dev = torch.device("cuda", 0)
Q, K, V, _ = wl.make_all(cfg, dev)
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype,
               cfg.value_dtype, device=dev)
out, idx, w = lk.forward(Q, K, V)
torch.cuda.synchronize()


def stats(tag, cnt, short=32, piece=256):
    cnt = cnt[cnt > 0].long()
    tot = int(cnt.sum())
    lng = cnt[cnt > short]
    pcs = int(((lng + piece - 1) // piece).sum()) if lng.numel() else 0
    q = torch.quantile(cnt.double(), torch.tensor([0.5, 0.9, 0.99, 0.999], dtype=torch.float64, device=cnt.device))
    print(f"{tag}: entries {tot}, rows {cnt.numel()}, long rows {lng.numel()} holding {int(lng.sum())} "
          f"({lng.sum().item() / tot:.3f}), pieces {pcs}, max {int(cnt.max())}, "
          f"quantiles p50/p90/p99/p999 {[round(x, 1) for x in q.tolist()]}")
    for lo, hi in ((33, 64), (65, 256), (257, 1024), (1025, 4096), (4097, 1 << 30)):
        m = (lng >= lo) & (lng <= hi)
        print(f"   len {lo}-{hi}: rows {int(m.sum())}, entries {int(lng[m].sum())}")


stats("dV", torch.bincount(idx.reshape(-1).long(), minlength=cfg.n_slots))
ns = cfg.n_sub
i = (idx.long() // ns)
j = (idx.long() % ns)
B, H, k = idx.shape
h = torch.arange(H, device=dev).view(1, H, 1)
for half, s in ((0, i), (1, j)):
    key = ((h * 2 + half) * ns + s)  # (h, half, sub-key)
    lk_id = torch.arange(B * H, device=dev).view(B, H, 1).expand(B, H, k)
    comb = torch.unique(lk_id.reshape(-1) * (H * 2 * ns) + key.reshape(-1))
    rows = comb % (H * 2 * ns)
    c = torch.bincount(rows, minlength=H * 2 * ns)
    stats(f"dK half {half}", c)
