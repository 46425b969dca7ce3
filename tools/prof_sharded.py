"""One row-sharded step (world size 1, peer transport: msn_pkm_forward_sharded +
msn_pkm_backward_sharded, the bench's default step) of a workload inside an
NVTX range "prof", after two warm-up steps: the target for
`ncu --nvtx --nvtx-include "prof/" ...` captures.

    python tools/prof_sharded.py [workload]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200.distributed import ShardedPKM  # noqa: E402

name = next((a for a in sys.argv[1:] if not a.startswith("--")), "c4_large_sharded_bf16")
cfg = wl.CONFIGS[name]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
Q, K, V, dOut = wl.make_all(cfg, dev)
sp = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype,
                cfg.value_dtype, device=dev, transport="peer")
dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=dev)
dV = torch.zeros((cfg.n_slots, cfg.d_value), dtype=torch.float32, device=dev)


def step():
    out, tape = sp.forward(Q, K, V)
    sp.backward(dOut, Q, K, V, tape, d_subkeys=dK, d_value_shard=dV)


for _ in range(2):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", name)
