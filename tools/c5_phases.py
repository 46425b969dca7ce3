"""C5 (latency config) phase times, warm: each call captured N times into one
CUDA graph, replayed, CUDA events around the replay -> per-call microseconds.
Phases: the whole forward (msn_pkm_forward), a1-a4 alone (msn_pkm_select:
scorer + Cartesian), a5 alone (msn_pkm_gather over the tape).  Run with
MSN_LIB=<variant .so> to A/B builds, MSN_SELECT_SPLIT=0/1 to force the
scorer's column split.

    python tools/c5_phases.py [workload]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200.pkm import PKMLookup, _ptr  # noqa: E402
from paper_2602_07526_b200._lib import check  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_latency_bf16"
cfg = wl.CONFIGS[name]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
Q, K, V = wl.make_queries(cfg, dev), wl.make_subkeys(cfg, dev), wl.make_values(cfg, dev)
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype,
               cfg.value_dtype, device=dev)
lib, h, B = lk.lib, lk._h, cfg.batch
out = torch.empty((B, cfg.d_value), dtype=torch.float32, device=dev)
idx = torch.empty((B, cfg.heads, cfg.k), dtype=torch.int32, device=dev)
w = torch.empty((B, cfg.heads, cfg.k), dtype=torch.float32, device=dev)
ws = lk.workspace(B)
s = torch.cuda.Stream(dev)


def sp():
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def fwd():
    check(lib.msn_pkm_forward(h, sp(), B, _ptr(Q), _ptr(K), _ptr(V), _ptr(out), _ptr(idx), _ptr(w),
                              _ptr(ws), ws.numel()))


def sel():
    check(lib.msn_pkm_select(h, sp(), B, _ptr(Q), _ptr(K), _ptr(idx), _ptr(w), _ptr(ws), ws.numel()))


def gat():
    check(lib.msn_pkm_gather(h, sp(), B, _ptr(idx), _ptr(w), _ptr(V), _ptr(out)))


def timed(fn, n=20, reps=30):
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    ts.sort()
    return round(ts[len(ts) // 2], 2)


res = {"workload": name, "lib": os.environ.get("MSN_LIB", "default"),
       "split": os.environ.get("MSN_SELECT_SPLIT", "auto"),
       "forward_us": timed(fwd), "select_us": timed(sel), "gather_us": timed(gat)}
print(json.dumps(res))
