import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from oracle import oracle as orc
cfg = wl.tiny_config(8, 2, 32, 16, 32, 4, torch.float32, torch.float32, index=3)
Q, K, V, dOut = wl.make_all(cfg, 'cuda')
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype, cfg.value_dtype)
out, idx, w = lk.forward(Q, K, V)
dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
torch.cuda.synchronize()
o = orc.forward(Q.cpu(), K.cpu(), V.cpu(), cfg.k)
print("idx equal", np.array_equal(idx.cpu().numpy(), o["idx"]))
b = orc.backward(Q.cpu(), K.cpu(), V.cpu(), o["idx"], dOut.cpu())
def err(a, r): a = a.detach().cpu().double().numpy(); return float(np.abs(a - r).max()), float(np.abs(r).max())
print("dw", err(dw, b["dw"]))
print("dV", err(dV, b["dV"]))
print("dK", err(dK, b["dK"]))
print("dQ", err(dq, b["dQ"]))
print("gpu dw[0,0]", dw[0,0].cpu().numpy(), "\nora dw[0,0]", b["dw"][0,0])
print("gpu dq[0,0,0,:8]", dq[0,0,0,:8].cpu().numpy(), "\nora", b["dQ"][0,0,0,:8])
print("gpu dq[0,0,1,:8]", dq[0,0,1,:8].cpu().numpy(), "\nora", b["dQ"][0,0,1,:8])
