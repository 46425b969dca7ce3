import sys, torch, time
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
name = sys.argv[1]
cfg = wl.CONFIGS[name]
Q = wl.make_queries(cfg, 'cuda'); K = wl.make_subkeys(cfg, 'cuda')
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype, cfg.value_dtype)
for _ in range(3): lk.select(Q, K)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): lk.select(Q, K)
e1.record(); torch.cuda.synchronize()
print(name, "select ms", e0.elapsed_time(e1)/10)
