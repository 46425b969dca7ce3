"""One C2 step with the f2 prologue (LN(q), LN(k), K~ = Theta k^, lookup,
backward, Theta^T / dTheta, LN backward) inside an NVTX range "prof"."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
cfg = wl.CONFIGS["c2_mid_bf16"]
Q, K, V, dOut = wl.make_all(cfg, "cuda")
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype, cfg.value_dtype)
theta = (torch.eye(cfg.d_half) + 0.05 * torch.randn((cfg.heads, 2, cfg.d_half, cfg.d_half))).cuda()
def step():
    q = lk.layernorm(Q); kh = lk.layernorm(K); ke = lk.key_transform(kh, theta)
    out, idx, w = lk.forward(q, ke, V)
    dq, dK, dV, dw = lk.backward(dOut, q, ke, V, idx, w)
    dkh, dth = lk.key_transform_backward(kh, theta, dK)
    lk.layernorm_backward(K, dkh); lk.layernorm_backward(Q, dq)
for _ in range(2): step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof"); step(); torch.cuda.nvtx.range_pop(); torch.cuda.synchronize(); print("ok")
