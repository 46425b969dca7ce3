import sys, torch
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
cfg0 = wl.CONFIGS[sys.argv[1]]
for B in (128, 1024, 4096, 16384):
    cfg = cfg0.scaled(batch=B)
    Q = wl.make_queries(cfg, 'cuda'); K = wl.make_subkeys(cfg, 'cuda')
    lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B, cfg.qk_dtype, cfg.value_dtype)
    for _ in range(3): lk.select(Q, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lk.select(Q, K)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1], "B", B, "CTAs", (B+127)//128*cfg.heads*2, "select us", round(e0.elapsed_time(e1)/20*1000,1))
