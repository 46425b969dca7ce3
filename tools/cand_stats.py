"""Per-half candidate-list statistics of the tcgen05 scorer (profiling aid):
runs msn_pkm_select on a workload and reads cand_n back from the forward
workspace (layout in api.cu: cand (score, index) | cand_n, 256-B aligned;
SC segment slots per row, SC = 2 for bf16 rows of 512 < n_sub <= 1024).

    python tools/cand_stats.py c4_large_sharded_bf16 [B]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200.pkm import PKMLookup  # noqa: E402


def a256(x):
    return (x + 255) // 256 * 256


name = sys.argv[1]
cfg = wl.CONFIGS[name]
Q = wl.make_queries(cfg, "cuda")
if len(sys.argv) > 2:
    Q = Q[: int(sys.argv[2])].contiguous()
K = wl.make_subkeys(cfg, "cuda")
B = Q.shape[0]
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B, cfg.qk_dtype, cfg.value_dtype)
lk.select(Q, K)
torch.cuda.synchronize()
SC = 2 if (cfg.qk_dtype == torch.bfloat16 and 512 < cfg.n_sub <= 1024 and cfg.k <= 32) else 1
rows = B * cfg.heads * 2 * SC
off = a256(8 * rows * 64)
n = lk._ws[off: off + 4 * rows].view(torch.int32).cpu()
if SC == 2:  # unused second segment counts are stale when the row was not split
    print("(rows with two column segments: counts per segment)")
print(name, "rows", rows, "mean", n.float().mean().item(), "max", n.max().item(),
      "overflow(>64)", int((n > 64).sum()), "p99", n.float().quantile(0.99).item())
