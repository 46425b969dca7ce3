"""Debug: the never-selected-sub-key check for one random shape."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from oracle import oracle as orc
B, H, n_sub, d_h, d_v, k, qdt, vdt = 26, 3, 32, 128, 32, 2, torch.bfloat16, torch.bfloat16
cfg = wl.tiny_config(B, H, d_h, n_sub, d_v, k, qdt, vdt, index=100 + n_sub + k)
Q, K, V, dOut = wl.make_all(cfg, "cuda")
lk = PKMLookup(H, n_sub, d_h, d_v, k, max_batch=B, qk_dtype=qdt, value_dtype=vdt)
out, idx, w = lk.forward(Q, K, V)
dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
torch.cuda.synchronize()
o = orc.forward(Q.cpu(), K.cpu(), V.cpu(), k)
print("idx equal:", np.array_equal(idx.cpu().numpy(), o["idx"]))
bw = orc.backward(Q.cpu(), K.cpu(), V.cpu(), o["idx"], dOut.cpu())
dk_g = dK.cpu().numpy().reshape(-1, d_h)
dk_o = bw["dK"].reshape(-1, d_h)
zero_o = np.all(dk_o == 0, axis=1)
bad = np.nonzero(zero_o & np.any(dk_g != 0, axis=1))[0]
print("bad rows:", bad[:20], len(bad))
for r in bad[:5]:
    print(r, dk_g[r][:6], np.abs(dk_g[r]).max())
print("dw", dw[:2].cpu().numpy(), "w", w[:2].cpu().numpy(), "idx", idx[:2].cpu().numpy())
