"""World-size-2/4 gloo tests (CPU) of the row-sharded table's host plumbing
(paper_2602_07526_b200/distributed.py, transport "nccl"): the fixed-size
all-to-alls of the record windows and counts, of the partials and of the
returned dw, the all-gather of d_out, shard ranges.  The exchange buffer and its region layout
are the library's (msn_pkm_exchange_layout, a host function); the data-path
kernels are stood in for by a CPU implementation of the phases' documented
semantics (include/msn_pkm.h, "the row-sharded table with the library's record
exchange") built on the fp64 oracle -- test infrastructure only (the product
path has no CPU fallback).  The sharded step must reproduce the unsharded
oracle result.  The kernels themselves are checked against the oracle with
emulated ranks on the GPU (tests/test_gpu_sharded.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


class OraclePhases:
    """CPU stand-in for the C-ABI phase calls of the STAGED exchange (test
    infrastructure): reads and writes the exchange buffer's regions exactly as
    include/msn_pkm.h documents them."""

    def __init__(self, cfg, world, rank, B_l):
        from paper_2602_07526_b200.pkm import PKMLookup
        self.real = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, max_batch=B_l,
                              qk_dtype=cfg.qk_dtype, value_dtype=cfg.value_dtype, device="cpu",
                              world_size=world if world > 1 else 0, rank=rank)
        self.heads, self.k, self.d_value, self.n_sub = cfg.heads, cfg.k, cfg.d_value, cfg.n_sub
        self.P, self.rank, self.lb = world, rank, B_l
        self.rpr = cfg.n_slots // world
        self.xb = None  # set after ShardedPKM builds the buffer

    def exchange_layout(self, lb, staged):
        return self.real.exchange_layout(lb, staged)

    def workspace(self, B, gb=None):
        return torch.empty(1, dtype=torch.uint8)

    def last_launch_count(self):
        return 0  # (no GPU kernels here)

    def exchange_select(self, q, K, Vs, x, out=None, ws=None):
        """a1-a4 (oracle), then the route into the OUT windows (records of query b
        for owner o at [b H k, b H k + cnt) in (h, t) order) and the local
        shard's partial into PART_OUT[rank]."""
        o = orc.forward(q, K, np.zeros((self.n_sub * self.n_sub, 4), np.float32), self.k)
        idx = torch.from_numpy(o["idx"].astype(np.int32))
        w = torch.from_numpy(o["w"]).float()
        P, lb, HK = self.P, self.lb, self.heads * self.k
        o_row, o_w, o_cnt = self.xb.records(out=True)
        pos = self.xb.region("POS", self.xb.cap)
        part = self.xb.region("PART_OUT", P, lb, self.d_value)
        for b in range(lb):
            cnt = [0] * P
            acc = torch.zeros(self.d_value, dtype=torch.float64)
            for r in range(HK):
                f = int(idx.view(lb, HK)[b, r])
                ow, row = f // self.rpr, f % self.rpr
                wt = w.view(lb, HK)[b, r]
                o_row[ow, b * HK + cnt[ow]], o_w[ow, b * HK + cnt[ow]] = row, wt
                pos[b * HK + r] = cnt[ow]
                cnt[ow] += 1
                if ow == self.rank:
                    acc += float(wt) * Vs[row].double()
            o_cnt[:, b] = torch.tensor(cnt, dtype=torch.int32)
            part[self.rank, b] = acc.float()
        return idx, w, (part[self.rank].clone() if P == 1 else None)

    def exchange_gather(self, Vs, x):
        P, lb, HK = self.P, self.lb, self.heads * self.k
        i_row, i_w, i_cnt = self.xb.records(out=False)
        part = self.xb.region("PART_OUT", P, lb, self.d_value)
        for s in range(P):
            if s == self.rank:
                continue
            for b in range(lb):
                acc = torch.zeros(self.d_value, dtype=torch.float64)
                for j in range(int(i_cnt[s, b])):
                    acc += float(i_w[s, b * HK + j]) * Vs[int(i_row[s, b * HK + j])].double()
                part[s, b] = acc.float()

    def exchange_combine(self, x, out=None):
        part = self.xb.region("PART_IN", self.P, self.lb, self.d_value)
        return part.double().sum(0).float() if self.P > 1 else out

    def exchange_scatter(self, Vs, dVs, x, ws=None):
        P, lb, HK = self.P, self.lb, self.heads * self.k
        i_row, i_w, i_cnt = self.xb.records(out=False)
        dall = self.xb.region("DOUT_ALL", P, lb, self.d_value)
        dw_out = self.xb.region("DW_OUT", P, self.xb.cap)
        for s in range(P):
            for b in range(lb):
                for j in range(int(i_cnt[s, b])):
                    row, d = int(i_row[s, b * HK + j]), dall[s, b]
                    dw_out[s, b * HK + j] = float((Vs[row].double() * d.double()).sum())
                    dVs[row] += float(i_w[s, b * HK + j]) * d

    def exchange_collect(self, idx, x, dw=None):
        HK = self.heads * self.k
        dw_in = self.xb.region("DW_IN", self.P, self.xb.cap)
        pos = self.xb.region("POS", self.xb.cap).long()
        f = idx.reshape(-1).long()
        win = torch.arange(f.numel()) // HK * HK
        return dw_in[f // self.rpr, win + pos].view(idx.shape).clone()

    def backward_keys(self, q, K, idx, w, dw, dK):
        B, H, k = idx.shape
        n = self.n_sub
        dK = torch.zeros(K.shape, dtype=torch.float32) if dK is None else dK
        dq = torch.zeros(q.shape, dtype=torch.float64)
        wd, dwd = w.double(), dw.double()
        for b in range(B):
            for h in range(H):
                g = float((wd[b, h] * dwd[b, h]).sum())
                for t in range(k):
                    ds = float(wd[b, h, t]) * (float(dwd[b, h, t]) - g)
                    f = int(idx[b, h, t])
                    i, j = f // n, f % n
                    dq[b, h, 0] += ds * K[h, 0, i].double()
                    dq[b, h, 1] += ds * K[h, 1, j].double()
                    dK[h, 0, i] += (ds * q[b, h, 0].double()).float()
                    dK[h, 1, j] += (ds * q[b, h, 1].double()).float()
        return dq.float(), dK


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_07526_b200.distributed import ShardedPKM
        from paper_2602_07526_b200 import workloads as wl
        cfg = wl.tiny_config(6 * world, 2, 16, 8, 8, 3, torch.float32, torch.float32, index=77)
        Q, K, V, dOut = wl.make_all(cfg)
        B_l = cfg.batch // world
        n = cfg.n_slots
        r0, r1 = rank * n // world, (rank + 1) * n // world
        ph = OraclePhases(cfg, world, rank, B_l)
        sp = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B_l, cfg.qk_dtype,
                        cfg.value_dtype, phases=ph, device="cpu", transport="nccl")
        ph.xb = sp.xb
        assert (sp.row_begin, sp.row_end) == (r0, r1)
        q_l = Q[rank * B_l:(rank + 1) * B_l].contiguous()
        d_l = dOut[rank * B_l:(rank + 1) * B_l].contiguous()
        Vs = sp.value_shard(V)
        out, tape = sp.forward(q_l, K, Vs)
        dq, dK, dVs, dw = sp.backward(d_l, q_l, K, Vs, tape)
        dist.all_reduce(dK)  # the caller's data-parallel sum of the replicated sub-keys
        outs = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(outs, out)
        dqs = [torch.empty_like(dq) for _ in range(world)]
        dist.all_gather(dqs, dq)
        dvs = [torch.empty_like(dVs) for _ in range(world)]
        dist.all_gather(dvs, dVs)
        if rank == 0:
            o = orc.forward(Q, K, V, cfg.k)
            bw = orc.backward(Q, K, V, o["idx"], dOut)
            res = {
                "out": float(np.abs(torch.cat(outs).double().numpy() - o["out"]).max()),
                "dq": float(np.abs(torch.cat(dqs).double().numpy() - bw["dQ"]).max()),
                "dv": float(np.abs(torch.cat(dvs).double().numpy() - bw["dV"]).max()),
                "dk": float(np.abs(dK.double().numpy() - bw["dK"]).max()),
                "dw": float(np.abs(dw.double().numpy() - bw["dw"][:B_l]).max()),
            }
            result_q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_matches_unsharded_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = q.get(timeout=10)
    for key, err in res.items():
        assert err < 1e-5, (key, res)


def _bad_worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_07526_b200.distributed import ShardedPKM
        try:
            ShardedPKM(1, 5, 16, 16, 2, 4, phases=object(), transport="nccl")  # 25 rows over 2 ranks
            result_q.put("no error")
        except ValueError:
            result_q.put("ok")
    finally:
        dist.destroy_process_group()


def test_shard_ranges_must_divide_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) == "ok" and q.get(timeout=10) == "ok"
