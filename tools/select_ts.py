"""Phase timeline of select_tc_kernel from a MSN_SELECT_TS build
(MSN_EXTRA_FLAGS=-DMSN_SELECT_TS, loaded with MSN_LIB=...): mean time of
each epilogue phase boundary after CTA start, and the CTA span.

    MSN_LIB=.../libmsn_pkm_ts.so python tools/select_ts.py c2_mid_bf16
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_07526_b200 import workloads as wl  # noqa: E402
from paper_2602_07526_b200 import _lib  # noqa: E402
from paper_2602_07526_b200.pkm import PKMLookup  # noqa: E402

name = sys.argv[1]
cfg = wl.CONFIGS[name]
Q = wl.make_queries(cfg, "cuda")
K = wl.make_subkeys(cfg, "cuda")
lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch, cfg.qk_dtype, cfg.value_dtype)
for _ in range(3):
    lk.select(Q, K)
torch.cuda.synchronize()
ncta = cfg.heads * 2 * ((cfg.batch + 127) // 128) * 4  # (up to 4 column segments)
buf = (ctypes.c_ulonglong * (ncta * 16))()
lib = _lib.load()
lib.msn_select_ts_dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.msn_select_ts_dump(buf, ncta) == ncta
t = np.frombuffer(buf, dtype=np.uint64).reshape(ncta, 16).astype(np.float64)
t = t[t[:, 0] > 0]  # the CTAs that ran
ncta = len(t)
t0 = t[:, 0]
names = ["start", "chunks ready", "pass A done", "tau done", "pass B done", "all rows done", "write-out done"]
print(f"{name}: {ncta} CTAs, kernel span {(t[:, 6].max() - t0.min()) / 1e3:.1f} us")
for i in range(1, 7):
    d = t[:, i] - t0
    print(f"  {names[i]:16s} mean {d.mean() / 1e3:7.2f} us  p90 {np.percentile(d, 90) / 1e3:7.2f}")
if (t[:, 7] > 0).all() and not (t[:, 10] > 0).any():
    print("  column segments: published at %.2f, cluster barrier passed %.2f, tau %.2f us" %
          tuple((t[:, c] - t0).mean() / 1e3 for c in (7, 8, 9)))
elif (t[:, 7] > 0).all():
    print("  two-sweep rows, first sweep: chunk ready at " +
          " ".join(f"{(t[:, 7 + c] - t0).mean() / 1e3:.2f}" for c in range(7)) + " us")
print(f"  A tile loaded {(t[:, 14] - t0).mean() / 1e3:.2f} us, MMA start {(t[:, 15] - t0).mean() / 1e3:.2f} us")
s = np.sort(t0 - t0.min())
print("  CTA starts: p25 %.1f p50 %.1f p75 %.1f max %.1f us" % tuple(np.percentile(s, [25, 50, 75, 100]) / 1e3))
