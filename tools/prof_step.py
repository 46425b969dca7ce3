"""One bench step (forward -> scatter -> backward_keys) of a workload inside an
NVTX range "prof", after two warm-up steps: the target for
`ncu --nvtx --nvtx-include "prof/" ...` captures.

    python tools/prof_step.py [workload] [--atomic]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200.pkm import PKMLookup, _ptr  # noqa: E402
from paper_2602_07526_b200._lib import check  # noqa: E402

name = next((a for a in sys.argv[1:] if not a.startswith("--")), "c2_mid_bf16")
cfg = wl.CONFIGS[name]
dev = torch.device("cuda", 0)
Q, K, V, dOut = wl.make_all(cfg, dev)
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype,
               cfg.value_dtype, atomic_bwd="--atomic" in sys.argv, device=dev)
lib, h, B = lk.lib, lk._h, cfg.batch
out = torch.empty((B, cfg.d_value), dtype=torch.float32, device=dev)
idx = torch.empty((B, cfg.heads, cfg.k), dtype=torch.int32, device=dev)
w = torch.empty((B, cfg.heads, cfg.k), dtype=torch.float32, device=dev)
dw = torch.empty_like(w)
dQ = torch.empty((B, cfg.heads, 2, cfg.d_half), dtype=torch.float32, device=dev)
dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=dev)
dV = torch.zeros((cfg.n_slots, cfg.d_value), dtype=torch.float32, device=dev)
ws = lk.workspace(B)
sp = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def step():
    check(lib.msn_pkm_forward(h, sp, B, _ptr(Q), _ptr(K), _ptr(V), _ptr(out), _ptr(idx), _ptr(w),
                              _ptr(ws), ws.numel()))
    if not cfg.backward:  # (forward-only configs: C1, C5)
        return
    check(lib.msn_pkm_scatter(h, sp, B, _ptr(idx), _ptr(w), _ptr(dOut), _ptr(V), _ptr(dV), _ptr(dw),
                              _ptr(ws), ws.numel()))
    check(lib.msn_pkm_backward_keys(h, sp, B, _ptr(Q), _ptr(K), _ptr(idx), _ptr(w), _ptr(dw),
                                    _ptr(dQ), _ptr(dK), _ptr(ws), ws.numel()))


for _ in range(2):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", name)
