"""Per-half candidate-list statistics of the tcgen05 scorer (profiling aid):
runs msn_pkm_select on a workload and reads cand_n back from the forward
workspace (layout in api.cu: cand (score, index) | cand_n, 256-B aligned).

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
rows = B * cfg.heads * 2
off = a256(8 * rows * 64)
n = lk._ws[off: off + 4 * rows].view(torch.int32).cpu()
print(name, "rows", rows, "mean", n.float().mean().item(), "max", n.max().item(),
      "overflow(>64)", int((n > 64).sum()), "p99", n.float().quantile(0.99).item())
