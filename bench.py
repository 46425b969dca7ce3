"""bench.py -- PKM lookups/sec forward+backward on B200 (the driver's
contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4_large_sharded_bf16] [--transport peer|nccl]

Default workload: BASELINE.json configs[3] (C4), the configuration the metric
("... at 1/2/4/8 B200") is quoted on: the row-sharded 2 GiB table through the
library's record exchange at ANY N (N = 1 runs the same code path with one
shard).  --gpus N > 1 without torchrun re-launches itself under torchrun (one
process per GPU, NCCL process group, rank p owns rows [p n/P, (p+1) n/P)).
A step = msn_pkm_forward_sharded (select a1-a4, route, gather a5, combine) +
msn_pkm_backward_sharded (scatter a6, collect, backward_keys a7-a8) over the
whole batch of 32,768 queries (strong scaling).  Timing: the step captured
into a CUDA graph, replayed K times with CUDA events around each replay on the
launching stream; L2 flushed (a 512 MiB write) before every replay, outside
the events; barrier + synchronize on both sides; max over ranks.  Other
workloads (C2, C3, C5, f4) run the unsharded path (replicas at N > 1).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "PKM lookups/sec fwd+bwd"
UNIT = "lookups/s"


def _dtype_name(dt):
    return {torch.bfloat16: "bf16", torch.float32: "f32"}[dt]


def load_peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the
    fallback figures of /opt/skills/guides/B200_PROFILING.md (6.65 TB/s,
    1.59 PFLOP/s bf16 burst, ~1.4 sustained)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "of measured (MEASURED_PEAKS.json)"
    return ({"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0},
            "of fallback (B200_PROFILING.md: no MEASURED_PEAKS.json on this box)")


# ------------------------------------------------------------- clocks -----
class ClockSampler:
    """Samples SM clock and throttle reasons during the timed region (NVML,
    falling back to nvidia-smi)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            mhz = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            util = p.nvmlDeviceGetUtilizationRates(self._h).gpu
            return mhz, r, util
        return None

    def _run(self):
        while not self._stop.is_set():
            try:
                s = self._sample()
            except Exception:
                s = None
            if s is not None:
                mhz, r, util = s
                self.samples.append((mhz, util))
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            self._stop.wait(0.005)

    def __enter__(self):
        if self._nvml is None:
            self._proc = None
            try:
                import subprocess
                self._proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.idx}", "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=subprocess.PIPE, text=True)
            except Exception:
                self._proc = None
        else:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._nvml is not None:
            self._stop.set()
            self._t.join()
        elif self._proc is not None:
            self._proc.terminate()
            out = self._proc.communicate()[0]
            for line in out.splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    self.samples.append((float(f[0]), float(f[2])))
                    self.max_mhz = float(f[1])
                except ValueError:
                    continue
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                    "sw_power_cap"), f[3:7]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)

    def summary(self):
        loaded = [m for m, u in self.samples if u >= 50] or [m for m, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------- our arm ----------
def algorithmic_bytes(cfg, idx=None, update="none"):
    """Per-phase algorithmic bytes."""
    esz = 2 if cfg.value_dtype == torch.bfloat16 else 4
    qsz = 2 if cfg.qk_dtype == torch.bfloat16 else 4
    L = cfg.batch * cfg.heads
    contrib = L * cfg.k
    out_elems = cfg.batch * cfg.d_value * cfg.head_groups
    gather = contrib * cfg.d_value * esz + contrib * 8 + out_elems * 4
    out = {"gather": gather}
    if idx is not None:
        rows, hits = torch.unique(idx, return_counts=True)
        uniq = int(rows.numel())
        out["unique_rows"] = uniq
        # SURVEY 8(d) "C3 skew": the workload describes itself
        top = torch.topk(hits, min(1000, uniq)).values
        out["skew"] = {"contributions": contrib, "unique_frac": uniq / max(contrib, 1),
                       "max_hits_one_row": int(hits.max()) if uniq else 0,
                       "top1000_rows_hit_share": float(top.sum()) / max(contrib, 1)}
        # V rows read once, dV read+written once (fp32), idx/w/dw, dOut once
        out["scatter"] = uniq * cfg.d_value * (esz + 8) + contrib * 12 + out_elems * 4
        if update != "none":  # V read + V written (+ Adagrad state read + written), no dV
            out["scatter"] = (uniq * cfg.d_value * (2 * esz + (8 if update == "adagrad" else 0))
                              + contrib * 12 + out_elems * 4)
    out["select_flops"] = 4 * L * cfg.n_sub * cfg.d_half
    out["select_bytes"] = L * 2 * cfg.d_half * qsz + contrib * 8
    return out


def _lib_gate(name):
    return {"none": 0, "tanh": 1, "sigmoid": 2, "identity": 3}[name]


def run_ours(args, rank, world, local_rank):
    from paper_2602_07526_b200 import workloads as wl
    from paper_2602_07526_b200.pkm import PKMLookup, _ptr

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = wl.CONFIGS[args.workload]
    Q, K, V, dOut = wl.make_all(cfg, dev)
    lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch,
                   cfg.qk_dtype, cfg.value_dtype, atomic_bwd=args.atomic, device=dev,
                   head_groups=cfg.head_groups, group_tables=cfg.group_tables)
    lib, h = lk.lib, lk._h
    B = cfg.batch
    out = torch.empty((B,) + tuple(cfg.out_shape_tail), dtype=torch.float32, device=dev)
    idx = torch.empty((B, cfg.heads, cfg.k), dtype=torch.int32, device=dev)
    w = torch.empty((B, cfg.heads, cfg.k), dtype=torch.float32, device=dev)
    dw = torch.empty_like(w)
    dQ = torch.empty((B, cfg.heads, 2, cfg.d_half), dtype=torch.float32, device=dev)
    dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=dev)
    dV = torch.zeros((cfg.n_slots, cfg.d_value), dtype=torch.float32, device=dev)
    ws = lk.workspace(B)
    gate = _lib_gate(args.gate)
    if gate:
        # memory-gated fusion: x~ = x * g(v_o), upstream grad on x~
        gx = torch.Generator(device="cpu").manual_seed(7526 + 6)
        x_in = torch.randn((B,) + tuple(cfg.out_shape_tail), generator=gx).to(dev)
        x_t = torch.empty_like(x_in)
        d_xin = torch.empty_like(x_in)
        d_vo = torch.empty_like(x_in)
    if args.prologue:
        # f2: q^ = LN(q), K~ = Theta LN(k) before the lookup; back through them after
        g2 = torch.Generator(device="cpu").manual_seed(7526 + 7)
        theta = (torch.eye(cfg.d_half) + 0.05 * torch.randn((cfg.heads, 2, cfg.d_half, cfg.d_half),
                                                             generator=g2)).to(dev)
        Q_raw, K_raw = Q, K
        Q = torch.empty_like(Q_raw)
        K_hat = torch.empty_like(K_raw)
        K = torch.empty_like(K_raw)
        d_theta = torch.zeros_like(theta)
        d_khat = torch.empty(K_raw.shape, dtype=torch.float32, device=dev)
        d_kraw = torch.empty(K_raw.shape, dtype=torch.float32, device=dev)
        d_qraw = torch.empty(Q_raw.shape, dtype=torch.float32, device=dev)
    upd = {"none": 0, "sgd": 1, "adagrad": 2}[args.update]
    ada = torch.zeros((cfg.n_slots, cfg.d_value), dtype=torch.float32, device=dev) if upd == 2 else None
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    from paper_2602_07526_b200._lib import check

    launches = [0]

    def step(evs=None, sp=sp):
        # forward (scoring, then the fused Cartesian + gather kernel; the library
        # records evs[1] at the stage boundary), backward phases separately
        n = 0
        if evs:
            evs[0].record(stream)
            arr = (ctypes.c_void_p * 2)(evs[1].cuda_event, evs[2].cuda_event)
            check(lib.msn_pkm_set_trace_events(h, arr, 2))
        if args.prologue:
            check(lib.msn_pkm_layernorm(h, sp, Q_raw.numel() // cfg.d_half, _ptr(Q_raw), _ptr(Q)))
            n += lk.last_launch_count()
            check(lib.msn_pkm_layernorm(h, sp, K_raw.numel() // cfg.d_half, _ptr(K_raw), _ptr(K_hat)))
            n += lk.last_launch_count()
            check(lib.msn_pkm_key_transform(h, sp, _ptr(K_hat), _ptr(theta), _ptr(K)))
            n += lk.last_launch_count()
        if gate:
            check(lib.msn_pkm_forward_gated(h, sp, B, _ptr(Q), _ptr(K), _ptr(V), _ptr(x_in), gate,
                                            _ptr(out), _ptr(x_t), _ptr(idx), _ptr(w), _ptr(ws), ws.numel()))
        else:
            check(lib.msn_pkm_forward(h, sp, B, _ptr(Q), _ptr(K), _ptr(V), _ptr(out), _ptr(idx), _ptr(w),
                                      _ptr(ws), ws.numel()))
        n += lk.last_launch_count()
        if evs:
            check(lib.msn_pkm_set_trace_events(h, None, 0))
            evs[3].record(stream)
        d_up = dOut
        if gate:  # the gate backward turns the upstream gradient on x~ into d v_o (counted in scatter)
            check(lib.msn_pkm_gate_backward(h, sp, B, gate, _ptr(x_in), _ptr(out), _ptr(dOut), _ptr(d_xin),
                                            _ptr(d_vo)))
            n += lk.last_launch_count()
            d_up = d_vo
        if evs:
            arr = (ctypes.c_void_p * 2)(evs[6].cuda_event, evs[7].cuda_event)
            check(lib.msn_pkm_set_trace_events(h, arr, 2))
        if upd:  # f3: the optimiser step fused into the row reduction (no dV buffer)
            check(lib.msn_pkm_scatter_update(h, sp, B, _ptr(idx), _ptr(w), _ptr(d_up), _ptr(V), upd,
                                             1e-3, 1e-10, _ptr(ada), _ptr(dw), _ptr(ws), ws.numel()))
        else:
            check(lib.msn_pkm_scatter(h, sp, B, _ptr(idx), _ptr(w), _ptr(d_up), _ptr(V), _ptr(dV), _ptr(dw),
                                      _ptr(ws), ws.numel()))
        n += lk.last_launch_count()
        if evs:
            check(lib.msn_pkm_set_trace_events(h, None, 0))
            evs[4].record(stream)
        check(lib.msn_pkm_backward_keys(h, sp, B, _ptr(Q), _ptr(K), _ptr(idx), _ptr(w), _ptr(dw), _ptr(dQ),
                                        _ptr(dK), _ptr(ws), ws.numel()))
        n += lk.last_launch_count()
        if args.prologue:  # counted in backward_keys
            check(lib.msn_pkm_key_transform_backward(h, sp, _ptr(K_hat), _ptr(theta), _ptr(dK), _ptr(d_khat),
                                                     _ptr(d_theta)))
            n += lk.last_launch_count()
            check(lib.msn_pkm_layernorm_backward(h, sp, K_raw.numel() // cfg.d_half, _ptr(K_raw), _ptr(d_khat),
                                                 _ptr(d_kraw)))
            n += lk.last_launch_count()
            check(lib.msn_pkm_layernorm_backward(h, sp, Q_raw.numel() // cfg.d_half, _ptr(Q_raw), _ptr(dQ),
                                                 _ptr(d_qraw)))
            n += lk.last_launch_count()
        if evs: evs[5].record(stream)
        launches[0] = n

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # (1) per-phase breakdown: eager launches with CUDA events at the phase
    # boundaries (some recorded inside the library); host launch gaps between
    # kernels are included here
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    for e in evs:  # create the CUDA events up front (torch creates them lazily on record)
        for j in (1, 2, 6, 7):
            e[j].record(stream)
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()  # L2 flush, outside the events
        step(evs[i])
    torch.cuda.synchronize()
    phases = ["select", "cartesian", "gather", "scatter", "backward_keys"]
    per = {p: 0.0 for p in phases}
    for e in evs:
        for j, p in enumerate(phases):
            per[p] += e[j].elapsed_time(e[j + 1])
    total_ms = sum(per.values())
    # the short-run dV reducer alone (events recorded inside msn_pkm_scatter);
    # 0 when the atomic backward runs
    reduce_ms = sum(e[6].elapsed_time(e[7]) for e in evs) / args.steps if not args.atomic else 0.0
    ms_step_eager = total_ms / args.steps
    # (2) the timed region: the same step captured once into a CUDA graph
    # (every kernel of the step, same arguments) and replayed K times, each
    # replay bracketed by CUDA events on the stream, L2 flushed before each
    cap = torch.cuda.Stream(dev)
    graph = torch.cuda.CUDAGraph()
    cap.wait_stream(stream)
    with torch.cuda.graph(graph, stream=cap):
        step(None, ctypes.c_void_p(cap.cuda_stream))
    torch.cuda.synchronize()
    for _ in range(2):
        flush.zero_()
        graph.replay()
    gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    t_wall = time.perf_counter()
    with clocks:
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the events
            gev[i][0].record(stream)
            graph.replay()
            gev[i][1].record(stream)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        torch.distributed.barrier()
    ms_step = sum(a.elapsed_time(b) for a, b in gev) / args.steps
    t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_step_max = float(t.item())
    lookups = cfg.batch * cfg.heads * world
    value = lookups / (ms_step_max / 1e3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        Qh = Q.cpu().pin_memory()
        dOh = dOut.cpu().pin_memory()
        # the user-facing handle returns d_query in the query's own dtype
        # (bf16 for bf16 configs, MSN_FLAG_DQ_QK_DTYPE): half the D2H bytes
        lk_e = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch,
                         cfg.qk_dtype, cfg.value_dtype, atomic_bwd=args.atomic, device=dev,
                         head_groups=cfg.head_groups, group_tables=cfg.group_tables, dq_in_qk_dtype=True)
        out_h = torch.empty((B,) + tuple(cfg.out_shape_tail), dtype=torch.float32).pin_memory()
        dq_h = torch.empty((B, cfg.heads, 2, cfg.d_half), dtype=lk_e.dq_dtype).pin_memory()
        n_e2e = max(3, min(args.steps, 20))
        for _ in range(3):
            lk_e.step_host(Qh, dOh, K, V, dK, dV, out_h, dq_h)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_e2e)]
        for i in range(n_e2e):
            flush.zero_()
            ev[i][0].record(stream)
            lk_e.step_host(Qh, dOh, K, V, dK, dV, out_h, dq_h)   # H2D q, dOut; D2H out, dQ
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in ev) / n_e2e
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        h2d = Qh.numel() * Qh.element_size() + dOh.numel() * dOh.element_size()
        d2h = out_h.numel() * out_h.element_size() + dq_h.numel() * dq_h.element_size()
        e2e = {"value": lookups / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()),
               "note": "PKMLookup.step_host: pinned host query + d_out in, out + d_query (in the query dtype) back to pinned host (2 slices, copies on their own streams overlapping the kernels), "
                       "forward+backward through msn_pkm_forward/msn_pkm_backward, one sync"}

    if rank != 0:
        return None
    peaks, peaks_kind = load_peaks()
    ab = algorithmic_bytes(cfg, idx, args.update)
    g_ms = per["gather"] / args.steps
    s_ms = per["scatter"] / args.steps
    hbm = float(peaks["hbm_gbs"])
    traffic, traffic_dv = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp)).get(args.workload, {})
        traffic, traffic_dv = tj.get("gather"), tj.get("dv_reduce")
    fused = cfg.batch >= 8192 and cfg.heads * cfg.k <= 256
    sel_ms = per["select"] / args.steps
    tf32 = cfg.qk_dtype == torch.float32
    # candidate roofline kernels, each with its own bound; the dominant one
    # (longest per step) is reported as "roofline"
    bf16_peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
    cands = {
        "gather": {"kernel": ("cartesian_gather (a3+a4+a5 fused)" if fused else "gather_kernel (a5)"),
                   "bound": "hbm", "ms": g_ms, "work": ab["gather"], "peak": hbm, "unit": "GB/s",
                   "traffic": traffic},
        "dv_reduce": {"kernel": "grp_reduce_short_kernel (a6: dV += w dOut, dw, runs <= 32)",
                      "bound": "hbm", "ms": reduce_ms, "work": ab["scatter"], "peak": hbm, "unit": "GB/s",
                      "traffic": traffic_dv},
        "select": {"kernel": "select_tc_kernel (a1+a2, tcgen05 %s)" % ("3xTF32" if tf32 else "bf16"),
                   "bound": "tensor", "ms": sel_ms,
                   "work": ab["select_flops"] * (3 if tf32 else 1),
                   # TF32 dense peak = bf16 / 2 (nominal ratio, B200_PROFILING.md)
                   "peak": bf16_peak / (2 if tf32 else 1), "unit": "TFLOP/s", "traffic": None},
    }
    dom = max((c for c in cands if cands[c]["ms"] > 0), key=lambda c: cands[c]["ms"])
    rl = {}
    for name, c in cands.items():
        if c["ms"] <= 0:
            continue
        scale = 1e9 if c["unit"] == "GB/s" else 1e12
        ach = c["work"] / (c["ms"] / 1e3) / scale
        rl[name] = {"kernel": c["kernel"], "bound": c["bound"], "achieved": ach, "peak": c["peak"],
                    "unit": c["unit"], "frac": ach / c["peak"], "traffic": c["traffic"],
                    "ms": c["ms"], "algorithmic": c["work"], "peak_kind": peaks_kind}
    roof = dict(rl[dom])
    roof["dominant_of"] = sorted(rl)
    kernels = {p: {"ms": per[p] / args.steps, "share": per[p] / total_ms} for p in phases}
    kernels["rooflines"] = rl
    kernels["gather"]["GBps"] = rl["gather"]["achieved"]
    kernels["scatter"]["GBps"] = ab["scatter"] / (s_ms / 1e3) / 1e9
    kernels["scatter"]["algorithmic_bytes"] = ab["scatter"]
    kernels["scatter"]["unique_rows"] = ab["unique_rows"]
    kernels["scatter"]["skew"] = ab["skew"]
    kernels["select"]["TFLOPs"] = ab["select_flops"] / (sel_ms / 1e3) / 1e12
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step_max, "ms_per_step_eager": ms_step_eager,
        "timing": "timed region: the step (forward + backward, every kernel) replayed from a CUDA graph, "
                  "CUDA events around each replay, max over ranks; kernels{} = an eager pass with events "
                  "at the phase boundaries",
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": _dtype_name(cfg.value_dtype),
        "data": "synthetic (seeded, BASELINE.json configs[%d] recipe, DESIGN.md Inputs)" % cfg.index,
        "config": {"workload": cfg.name, "batch": cfg.batch, "heads": cfg.heads, "n_sub": cfg.n_sub,
                   "n_slots": cfg.n_slots,
                   "phases": "select = tcgen05 scoring + per-half candidates; cartesian = Cartesian top-k + softmax "
                             "(0 when fused into the gather, B >= 8192); gather = sparse gather + weighted sum "
                             "(the roofline kernel); scatter = dV/dw; backward_keys = ds, dQ, dK", "d_half": cfg.d_half, "d_value": cfg.d_value, "k": cfg.k,
                   "lookups_per_step_per_gpu": cfg.batch * cfg.heads,
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "backward": "atomic" if args.atomic else "deterministic (grouped by row, per-row id order)",
                   "gate": args.gate,
                   "prologue": bool(args.prologue),
                   "update": args.update,
                   "slot_hits": ab["skew"],
                   "l2": "flushed before every step (512 MiB write, outside the timed events)"},
        "roofline": roof,
        "kernels": kernels,
        "gpu_launches": launches[0] * args.steps,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "wall_s_timed_region": t_wall,
    }
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(cfg, Q, K, V, dOut)
    return res


def run_latency(args, rank, world, local_rank):
    """C5 (configs[4]): latency-bound inference forward.  One forward per call,
    replayed from a CUDA graph; per-call CUDA-event latency, p50/p99."""
    from paper_2602_07526_b200 import workloads as wl
    from paper_2602_07526_b200.pkm import PKMLookup, _ptr
    from paper_2602_07526_b200._lib import check
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = wl.CONFIGS[args.workload]
    Q, K, V = wl.make_queries(cfg, dev), wl.make_subkeys(cfg, dev), wl.make_values(cfg, dev)
    lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, cfg.batch,
                   cfg.qk_dtype, cfg.value_dtype, device=dev)
    B = cfg.batch
    out = torch.empty((B, cfg.d_value), dtype=torch.float32, device=dev)
    idx = torch.empty((B, cfg.heads, cfg.k), dtype=torch.int32, device=dev)
    w = torch.empty((B, cfg.heads, cfg.k), dtype=torch.float32, device=dev)
    ws = lk.workspace(B)
    s = torch.cuda.Stream(dev)
    torch.cuda.synchronize()

    def fwd():
        sp = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        check(lk.lib.msn_pkm_forward(lk._h, sp, B, _ptr(Q), _ptr(K), _ptr(V), _ptr(out), _ptr(idx), _ptr(w),
                                     _ptr(ws), ws.numel()))

    with torch.cuda.stream(s):
        for _ in range(max(3, args.warmup)):
            fwd()
    torch.cuda.synchronize()
    launches = lk.last_launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fwd()
    for _ in range(max(3, args.warmup)):
        g.replay()
    torch.cuda.synchronize()
    n = max(args.steps, 1000)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    clocks = ClockSampler(dev.index or 0)
    cur = torch.cuda.current_stream(dev)
    with clocks:
        for i in range(n):
            evs[i][0].record(cur)
            g.replay()
            evs[i][1].record(cur)
        torch.cuda.synchronize()
    lat = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)  # us
    mean_us = sum(lat) / n
    p50, p99 = lat[n // 2], lat[min(n - 1, int(0.99 * n))]
    lookups = B * cfg.heads
    esz = 2 if cfg.value_dtype == torch.bfloat16 else 4
    gbytes = lookups * cfg.k * (cfg.d_value * esz + 8) + B * cfg.d_value * 4
    peaks, kind = load_peaks()
    res = {"metric": "PKM lookups/sec fwd (latency config, per-call)", "value": lookups / (mean_us / 1e6),
           "unit": UNIT, "n_gpus": world, "steps": n, "warmup": args.warmup, "ms_per_step": mean_us / 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype_name(cfg.value_dtype),
           "data": "synthetic (seeded, BASELINE.json configs[4] recipe)",
           "config": {"workload": cfg.name, "batch": B, "heads": cfg.heads, "n_sub": cfg.n_sub,
                      "d_half": cfg.d_half, "d_value": cfg.d_value, "k": cfg.k,
                      "mode": "forward only, one CUDA-graph replay per call, back to back",
                      "l2": "value table 1 GiB > L2: the gather streams from HBM; no flush"},
           "latency_us": {"p50": p50, "p99": p99, "mean": mean_us, "min": lat[0], "calls": n},
           "roofline": {"kernel": "whole forward call (HBM bytes of the gather)", "bound": "hbm",
                        "achieved": gbytes / (mean_us / 1e6) / 1e9, "peak": float(peaks["hbm_gbs"]),
                        "unit": "GB/s", "frac": gbytes / (mean_us / 1e6) / 1e9 / float(peaks["hbm_gbs"]),
                        "traffic": None, "peak_kind": kind},
           "gpu_launches": launches * n, "clocks": clocks.summary()}
    return res if rank == 0 else None


def run_sharded(args, rank, world, local_rank):
    """C4 (configs[3], the metric's config): the row-sharded table through the
    library's record exchange (a9) at ANY world size -- N = 1 runs the same
    code path (one shard, the exchange to itself).  Strong scaling: the total
    batch B = 32,768 is split over the ranks, rank p owns rows [p n/P,
    (p+1) n/P).  A step = msn_pkm_forward_sharded + msn_pkm_backward_sharded
    (peer transport: select, route, barrier, gather, barrier, combine;
    d_out, barrier, scatter, barrier, collect, backward_keys), captured once
    into a CUDA graph and replayed; value = total lookups / max-over-ranks
    step time."""
    import torch.distributed as dist
    from paper_2602_07526_b200 import workloads as wl
    from paper_2602_07526_b200.distributed import ShardedPKM
    from paper_2602_07526_b200.pkm import _ptr
    from paper_2602_07526_b200._lib import check
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = wl.CONFIGS[args.workload]
    B_l = cfg.batch // world
    Q, K, V, dOut = wl.make_all(cfg, dev)  # every rank draws the same seeded tensors
    sp = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B_l,
                    qk_dtype=cfg.qk_dtype, value_dtype=cfg.value_dtype, device=dev,
                    transport=args.transport)
    q_l = Q[rank * B_l:(rank + 1) * B_l].contiguous()
    d_l = dOut[rank * B_l:(rank + 1) * B_l].contiguous()
    Vs = sp.value_shard(V)
    # (the CPU-oracle sample: up to half the batch, the same bytes as the GPU's)
    q_cpu_sample = Q[:cfg.batch // 2].cpu() if (rank == 0 and world == 1) else None
    d_cpu_sample = dOut[:cfg.batch // 2].cpu() if (rank == 0 and world == 1) else None
    del V, Q, dOut
    torch.cuda.empty_cache()
    lk, x = sp.ph, sp.xb.x
    dVs = torch.zeros((sp.rows, cfg.d_value), dtype=torch.float32, device=dev)
    dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=dev)
    out = torch.empty((B_l, cfg.d_value), dtype=torch.float32, device=dev)
    idx = torch.empty((B_l, cfg.heads, cfg.k), dtype=torch.int32, device=dev)
    w = torch.empty((B_l, cfg.heads, cfg.k), dtype=torch.float32, device=dev)
    dq = torch.empty((B_l, cfg.heads, 2, cfg.d_half), dtype=torch.float32, device=dev)
    dw = torch.empty_like(w)
    ws = sp.ws
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches = [0]
    peer = args.transport == "peer"

    def step(sp_=None):
        if peer:
            sptr = ctypes.c_void_p((sp_ or stream).cuda_stream)
            check(lk.lib.msn_pkm_forward_sharded(lk._h, sptr, B_l, _ptr(q_l), _ptr(K), _ptr(Vs), ctypes.byref(x),
                                                 _ptr(out), _ptr(idx), _ptr(w), _ptr(ws), ws.numel()))
            n = lk.last_launch_count()
            check(lk.lib.msn_pkm_backward_sharded(lk._h, sptr, B_l, _ptr(d_l), _ptr(q_l), _ptr(K), _ptr(Vs),
                                                  _ptr(idx), _ptr(w), ctypes.byref(x), _ptr(dq), _ptr(dK),
                                                  _ptr(dVs), _ptr(dw), _ptr(ws), ws.numel()))
            launches[0] = n + lk.last_launch_count()
        else:
            c0 = sp.launch_count
            o, tape = sp.forward(q_l, K, Vs)
            sp.backward(d_l, q_l, K, Vs, tape, d_subkeys=dK, d_value_shard=dVs)
            launches[0] = sp.launch_count - c0

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # (1) per-phase breakdown (peer transport): the same kernels through the
    # phase calls, CUDA events between them (eager; launch gaps included)
    per, reduce_ms = {}, 0.0
    phases = ["select", "cartesian_route", "gather", "combine", "scatter", "backward_keys"]
    if peer:
        per = {p: 0.0 for p in phases}
        nb = max(2, min(args.steps, 10))
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(10)] for _ in range(nb)]
        for e in evs:
            for j in range(10):
                e[j].record(stream)
        torch.cuda.synchronize()
        sptr = ctypes.c_void_p(stream.cuda_stream)
        sp.xb.region("DOUT", B_l, cfg.d_value).copy_(d_l)  # (constant: once, outside the events)
        barrier = (lambda: lk.exchange_barrier(x)) if world > 1 else (lambda: None)
        for e in evs:
            flush.zero_()
            e[0].record(stream)
            arr = (ctypes.c_void_p * 2)(e[1].cuda_event, e[2].cuda_event)
            check(lk.lib.msn_pkm_set_trace_events(lk._h, arr, 2))
            check(lk.lib.msn_pkm_exchange_select(lk._h, sptr, _ptr(q_l), _ptr(K), _ptr(Vs), ctypes.byref(x),
                                                 _ptr(idx), _ptr(w), _ptr(out), _ptr(ws), ws.numel()))
            check(lk.lib.msn_pkm_set_trace_events(lk._h, None, 0))
            barrier()
            e[3].record(stream)
            lk.exchange_gather(Vs, x)
            barrier()
            e[4].record(stream)
            lk.exchange_combine(x, out)
            e[5].record(stream)
            barrier()
            arr = (ctypes.c_void_p * 2)(e[8].cuda_event, e[9].cuda_event)
            check(lk.lib.msn_pkm_set_trace_events(lk._h, arr, 2))
            lk.exchange_scatter(Vs, dVs, x, ws)
            check(lk.lib.msn_pkm_set_trace_events(lk._h, None, 0))
            barrier()
            e[6].record(stream)
            lk.exchange_collect(idx, x, dw)
            check(lk.lib.msn_pkm_backward_keys(lk._h, sptr, B_l, _ptr(q_l), _ptr(K), _ptr(idx), _ptr(w), _ptr(dw),
                                               _ptr(dq), _ptr(dK), _ptr(ws), ws.numel()))
            e[7].record(stream)
        torch.cuda.synchronize()
        # select = the tcgen05 scorer; cartesian_route = the fused Cartesian top-k +
        # softmax + route + local-shard gather (+ barrier); gather = the remote
        # windows (+ barrier); scatter includes the d_out hand-over and barriers
        order = [(0, 1, "select"), (1, 3, "cartesian_route"), (3, 4, "gather"), (4, 5, "combine"),
                 (5, 6, "scatter"), (6, 7, "backward_keys")]
        for e in evs:
            for a, b, name in order:
                per[name] += e[a].elapsed_time(e[b]) / nb
        reduce_ms = sum(e[8].elapsed_time(e[9]) for e in evs) / nb
    # (2) the timed region: the step captured into a CUDA graph, replayed K
    # times, CUDA events around each replay, L2 flushed before each outside
    graph = None
    if peer:
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step(cap)
        torch.cuda.synchronize()
        for _ in range(2):
            flush.zero_()
            graph.replay()
    gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index or 0)
    t_wall = time.perf_counter()
    with clocks:
        for i in range(args.steps):
            flush.zero_()
            gev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            gev[i][1].record(stream)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in gev) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ctl = sp.xb.region("CTL", 64)
    timeouts = int(ctl[17].item())

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        sp_e = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B_l, qk_dtype=cfg.qk_dtype,
                          value_dtype=cfg.value_dtype, device=dev, transport=args.transport, dq_in_qk_dtype=True)
        qh, dh = q_l.cpu().pin_memory(), d_l.cpu().pin_memory()
        # two sets of device inputs and host results: step i+1's H2D (copy
        # engine) runs under step i's compute, step i's D2H under step i+1's
        out_h = [torch.empty((B_l, cfg.d_value), dtype=torch.float32).pin_memory() for _ in range(2)]
        dq_h = [torch.empty((B_l, cfg.heads, 2, cfg.d_half), dtype=sp_e.ph.dq_dtype).pin_memory() for _ in range(2)]
        qd = [torch.empty_like(q_l) for _ in range(2)]
        dd = [torch.empty_like(d_l) for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        main = torch.cuda.current_stream(dev)
        done = [torch.cuda.Event() for _ in range(2)]    # step using input set j finished
        landed = [torch.cuda.Event() for _ in range(2)]  # input set j copied in

        def h2d(i):
            j = i % 2
            s_in.wait_event(done[j])  # (the set's previous step is over)
            with torch.cuda.stream(s_in):
                qd[j].copy_(qh, non_blocking=True)
                dd[j].copy_(dh, non_blocking=True)
                landed[j].record(s_in)

        def e2e_steps(n):
            """n pipelined steps through the public API; returns when every
            result is on the host."""
            h2d(0)
            for i in range(n):
                j = i % 2
                main.wait_event(landed[j])
                if i + 1 < n:
                    h2d(i + 1)
                o, tape = sp_e.forward(qd[j], K, Vs)
                s_out.wait_stream(main)
                with torch.cuda.stream(s_out):
                    out_h[j].copy_(o, non_blocking=True)
                o.record_stream(s_out)
                dq_e, _, _, _ = sp_e.backward(dd[j], qd[j], K, Vs, tape, d_subkeys=dK, d_value_shard=dVs)
                done[j].record(main)
                s_out.wait_stream(main)
                with torch.cuda.stream(s_out):
                    dq_h[j].copy_(dq_e, non_blocking=True)
                dq_e.record_stream(s_out)
            main.wait_stream(s_out)

        e2e_steps(3)
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 20))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(main)
        e2e_steps(n_e2e)
        e1.record(main)
        torch.cuda.synchronize()  # the results are on the host
        e2e_ms = e0.elapsed_time(e1) / n_e2e
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d_b = qh.numel() * qh.element_size() + dh.numel() * dh.element_size()
        d2h_b = out_h[0].numel() * out_h[0].element_size() + dq_h[0].numel() * dq_h[0].element_size()
        e2e = {"value": cfg.batch * cfg.heads / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d_b), "d2h_bytes_per_step": int(d2h_b), "ms_per_step": float(te.item()),
               "steps": n_e2e,
               "note": "ShardedPKM forward+backward (msn_pkm_forward_sharded / msn_pkm_backward_sharded) fed from "
                       "pinned host memory, n pipelined steps between two CUDA events, divided by n: every step "
                       "copies its queries and d_out in (H2D) and its out (fp32) and d_query (bf16) back (D2H); "
                       "step i+1's H2D and step i's D2H run on side streams (copy engines) under the compute; "
                       "the region ends when the last result is on the host; per-rank bytes"}
        del sp_e

    # slot-hit statistics (the workload describes itself) from this rank's tape
    ab = algorithmic_bytes(cfg.scaled(batch=B_l), idx, "none")
    uniq_local = None
    if rank == 0:
        loc = idx[(idx >= sp.row_begin) & (idx < sp.row_end)]
        uniq_local = int(torch.unique(loc).numel())
    if rank != 0:
        return None
    peaks, peaks_kind = load_peaks()
    hbm = float(peaks["hbm_gbs"])
    bf16_peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
    esz = 2 if cfg.value_dtype == torch.bfloat16 else 4
    HK = cfg.heads * cfg.k
    contrib_l = B_l * HK
    # algorithmic bytes per step and rank: the forward's
    # value rows + records written and read (8 B each) + idx/w (8 B per slot)
    # + the partial rows; the dV reducer: every touched row's V read once, dV
    # read + written once (fp32), 12 B per record (row, w, dw) + the d_out rows
    # read once per (source, query)
    rec_l = contrib_l  # records this rank receives (= sends, in expectation, uniform slots)
    gather_b = rec_l * (cfg.d_value * esz + 8 + 8) + contrib_l * 8 + world * B_l * cfg.d_value * 4
    scatter_b = (uniq_local or 0) * cfg.d_value * (esz + 8) + rec_l * 12 + world * B_l * cfg.d_value * 4
    select_f = 4 * B_l * cfg.heads * cfg.n_sub * cfg.d_half
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(args.workload + "_xchg", {})
    cands = {}
    if peer:
        cands = {
            "gather": {"kernel": ("cartesian_route_kernel (a3+a4 + route + the local shard's a5, fused)" if world == 1
                                  else "gather_records_kernel + the local shard in cartesian_route_kernel (a5)"),
                       "bound": "hbm", "ms": per["cartesian_route"] + per["gather"], "work": gather_b, "peak": hbm,
                       "unit": "GB/s", "traffic": traffic.get("gather")},
            "dv_reduce": {"kernel": "grp_reduce_short_kernel (a6 over the received records: dV +=, dw)",
                          "bound": "hbm", "ms": reduce_ms, "work": scatter_b, "peak": hbm, "unit": "GB/s",
                          "traffic": traffic.get("dv_reduce")},
            "select": {"kernel": "select_tc_kernel (a1+a2, tcgen05 bf16)", "bound": "tensor", "ms": per["select"],
                       "work": select_f, "peak": bf16_peak, "unit": "TFLOP/s", "traffic": None},
        }
    rl = {}
    for name, c in cands.items():
        if c["ms"] <= 0:
            continue
        scale = 1e9 if c["unit"] == "GB/s" else 1e12
        ach = c["work"] / (c["ms"] / 1e3) / scale
        rl[name] = {"kernel": c["kernel"], "bound": c["bound"], "achieved": ach, "peak": c["peak"],
                    "unit": c["unit"], "frac": ach / c["peak"], "traffic": c["traffic"], "ms": c["ms"],
                    "algorithmic": c["work"], "peak_kind": peaks_kind}
    roof = None
    if rl:
        dom = max(rl, key=lambda n_: rl[n_]["ms"])
        roof = dict(rl[dom])
        roof["dominant_of"] = sorted(rl)
    total = sum(per.values()) or 1.0
    kernels = {p: {"ms": per[p], "share": per[p] / total} for p in per}
    kernels["rooflines"] = rl
    kernels["dv_reduce_ms"] = reduce_ms
    res = {"metric": METRIC, "value": cfg.batch * cfg.heads / (ms / 1e3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": _dtype_name(cfg.value_dtype),
           "data": "synthetic (seeded, BASELINE.json configs[3] recipe, DESIGN.md Inputs)",
           "timing": ("timed region: the sharded step (msn_pkm_forward_sharded + msn_pkm_backward_sharded, every "
                      "kernel and barrier) replayed from a CUDA graph, CUDA events around each replay, max over "
                      "ranks; kernels{} = an eager pass through the phase calls with events between them"
                      if peer else "eager steps (NCCL transport: one host read of the record counts per step)"),
           "config": {"workload": cfg.name, "batch_total": cfg.batch, "batch_per_rank": B_l,
                      "heads": cfg.heads, "n_sub": cfg.n_sub, "n_slots": cfg.n_slots,
                      "rows_per_rank": sp.rows, "d_half": cfg.d_half, "d_value": cfg.d_value, "k": cfg.k,
                      "parallelism": f"row-sharded table x{world}: records all-to-all, partials returned "
                                     f"({'peer memory, fused into the route/gather/scatter kernels' if peer else 'NCCL'})",
                      "transport": args.transport,
                      "slot_hits_rank0": ab.get("skew"), "unique_local_rows_rank0": uniq_local,
                      "l2": "flushed before every step (512 MiB write, outside the timed events)"},
           "roofline": roof, "kernels": kernels, "gpu_launches": launches[0] * args.steps,
           "clocks": clocks.summary(), "e2e": e2e, "wall_s_timed_region": t_wall,
           "barrier_timeouts": timeouts}
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(cfg, q_cpu_sample, K.cpu(), Vs.cpu(), d_cpu_sample, queries=512)
    return res


def cpu_baseline(cfg, Q, K, V, dOut, queries=None):
    """The fp64 oracle (oracle/, as it stands) on a bounded sample of the same
    workload on the host cores: fwd + bwd over the first `queries` queries,
    full tables."""
    from oracle import oracle as orc
    n = queries or min(cfg.batch, 4096)
    k_, v = K.cpu(), V.cpu()
    cores = len(os.sched_getaffinity(0))
    G = cfg.head_groups

    def run(n):
        q, d = Q[:n].cpu(), dOut[:n].cpu()
        t0 = time.perf_counter()
        if G == 1:
            o = orc.forward(q, k_, v, cfg.k, nthreads=cores)
            orc.backward(q, k_, v, o["idx"], d, want_dense_dv=False, nthreads=cores)
        else:  # head groups (f4): G independent lookups, group g's heads and table
            hg, nn = cfg.heads // G, cfg.n_sub * cfg.n_sub
            for g in range(G):
                hs = slice(g * hg, (g + 1) * hg)
                vg = v[g * nn:(g + 1) * nn] if cfg.group_tables else v
                qg, kg = q[:, hs].contiguous(), k_[hs].contiguous()
                o = orc.forward(qg, kg, vg, cfg.k, nthreads=cores)
                orc.backward(qg, kg, vg, o["idx"], d[:, g].contiguous(), want_dense_dv=False, nthreads=cores)
        return time.perf_counter() - t0

    t = run(n)
    # a sample of about 10 s of CPU work (bounded by the batch): the first
    # `queries` give the rate, the reported run is scaled up from it
    cap = min(cfg.batch, Q.shape[0])
    if t < 2.0 and n < cap:
        n2 = min(cap, max(n, int(n * 10.0 / max(t, 1e-3)) // 512 * 512))
        if n2 > n:
            n, t = n2, run(n2)
    return {"value": n * cfg.heads / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n} of {cfg.batch} queries x {cfg.heads} heads = {n * cfg.heads} lookups, "
                      f"fwd+bwd, full tables, fp64 C oracle with OpenMP ({t:.1f} s)",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------- reference arm ----
def run_reference(args, rank, world):
    """The base contract's reference arm for this tier is the fp64 oracle,
    timed as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    from paper_2602_07526_b200 import workloads as wl
    from oracle import oracle as orc
    cfg = wl.CONFIGS[args.workload]
    Q, K, V, dOut = wl.make_all(cfg, "cpu")
    cores = len(os.sched_getaffinity(0))
    per_step = max(1, min(cfg.batch, 64))   # bounded sample per step
    for i in range(args.warmup):
        s = (i * per_step) % cfg.batch
        o = orc.forward(Q[s:s + per_step], K, V, cfg.k, nthreads=cores)
        orc.backward(Q[s:s + per_step], K, V, o["idx"], dOut[s:s + per_step], want_dense_dv=False, nthreads=cores)
    t0 = time.perf_counter()
    for i in range(args.steps):
        s = (i * per_step) % cfg.batch
        o = orc.forward(Q[s:s + per_step], K, V, cfg.k, nthreads=cores)
        orc.backward(Q[s:s + per_step], K, V, o["idx"], dOut[s:s + per_step], want_dense_dv=False, nthreads=cores)
    t = time.perf_counter() - t0
    value = args.steps * per_step * cfg.heads / t
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True,
            # (the same scaling as this workload's own arm: the sharded C4 step is strong)
            "scaling": "strong" if (cfg.name == "c4_large_sharded_bf16" and not getattr(args, "unsharded", False))
                       else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded)",
            "config": {"workload": cfg.name, "batch_per_step": per_step, "heads": cfg.heads,
                       "n_sub": cfg.n_sub, "d_half": cfg.d_half, "d_value": cfg.d_value, "k": cfg.k},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} queries x {cfg.heads} heads per step, fwd+bwd, full tables",
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c4_large_sharded_bf16",
                    help="BASELINE.json configs: c4_large_sharded_bf16 (default: the metric's config, the "
                         "row-sharded table at any N), c2_mid_bf16, c3_train_fp32_zipf, c5_latency_bf16, f4_*")
    ap.add_argument("--atomic", action="store_true", help="atomic (non-deterministic) dV scatter")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unsharded", action="store_true",
                    help="C4 through the unsharded single-GPU path (msn_pkm_forward/backward) instead")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="row-sharded exchange: peer memory inside the library's kernels (default), or NCCL")
    ap.add_argument("--prologue", action="store_true",
                    help="include LayerNorm(q), K~ = Theta LayerNorm(k) and their backward (SURVEY 8(f) f2)")
    ap.add_argument("--update", choices=["none", "sgd", "adagrad"], default="none",
                    help="fuse the optimiser step into the value-row reduction (SURVEY 8(f) f3)")
    ap.add_argument("--gate", choices=["none", "tanh", "sigmoid", "identity"], default="none",
                    help="include the memory-gated fusion (SURVEY 8(f) f1) in the step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # the fp64 oracle on the host cores, rank 0 only (other ranks: no work)
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.workload.startswith("c5"):
        res = run_latency(args, rank, world, local_rank)
    elif args.workload.startswith("c4") and not args.unsharded:
        res = run_sharded(args, rank, world, local_rank)
    else:
        res = run_ours(args, rank, world, local_rank)
    if res is not None:
        print(json.dumps(res), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
