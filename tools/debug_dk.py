import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from oracle import oracle as orc
cfg = wl.CONFIGS["c3_train_fp32_zipf"]
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
Q = wl.make_queries(cfg, 'cuda')[:S].contiguous(); K = wl.make_subkeys(cfg, 'cuda'); V = wl.make_values(cfg, 'cuda')
dOut = wl.make_dout(cfg, 'cuda')[:S].contiguous()
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, S, cfg.qk_dtype, cfg.value_dtype)
out, idx, w = lk.forward(Q, K, V)
dq, dK, dV, dw = lk.backward(dOut, Q, K, V, idx, w)
torch.cuda.synchronize()
o = orc.forward(Q.cpu(), K.cpu(), V.cpu(), cfg.k)
print("idx diff lookups", int((idx.cpu().numpy() != o["idx"]).any(-1).sum()))
b = orc.backward(Q.cpu(), K.cpu(), V.cpu(), o["idx"], dOut.cpu(), want_dense_dv=False)
print("dw maxerr", float(np.abs(dw.cpu().double().numpy() - b["dw"]).max()))
print("ds check: ", float(np.abs(b["ds"]).max()))
g = dK.cpu().double().numpy().reshape(-1, cfg.d_half); r = b["dK"].reshape(-1, cfg.d_half)
err = np.abs(g - r).max(1); scale = np.abs(r).max(1)
n_sub = cfg.n_sub
cnt = np.zeros(cfg.heads * 2 * n_sub, int)
for h in range(cfg.heads):
    for half, rr in ((0, o["idx"][:, h] // n_sub), (1, o["idx"][:, h] % n_sub)):
        u = np.unique(np.stack([np.repeat(np.arange(S), cfg.k), rr.reshape(-1)], 1), axis=0)
        np.add.at(cnt, (h * 2 + half) * n_sub + u[:, 1], 1)
order = np.argsort(-err / np.maximum(scale, 1e-12))[:8]
for row in order:
    print(row, "cnt", cnt[row], "err", err[row], "scale", scale[row], "g", g[row, :3], "r", r[row, :3])
print("rows with cnt>64:", int((cnt > 64).sum()), "max cnt", cnt.max())
big = cnt > 64
print("max rel err big rows", float((err[big] / np.maximum(scale[big], 1e-12)).max()) if big.any() else None)
sm = (cnt <= 64) & (cnt > 0)
print("max rel err small rows", float((err[sm] / np.maximum(scale[sm], 1e-12)).max()))
