"""World-size-2 gloo tests (CPU) of the row-sharded table's host plumbing
(paper_2602_07526_b200/distributed.py): all-gathers, reduce-scatters, shard
ranges and the dw exactness argument.  The four data-path phases are stood in
for by a CPU implementation built on the fp64 oracle (test-only; the product
path has no CPU fallback), so what is checked here is the collective algebra:
the sharded step must reproduce the unsharded oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


class OraclePhases:
    """CPU stand-in for the four C-ABI phase calls (test infrastructure)."""

    def __init__(self, n_sub, k, row_begin, row_end):
        self.n_sub, self.k, self.r0, self.r1 = n_sub, k, row_begin, row_end

    def select(self, q, K):
        o = orc.forward(q, K, np.zeros((self.n_sub * self.n_sub, 4), np.float32), self.k)
        return torch.from_numpy(o["idx"].astype(np.int32)), torch.from_numpy(o["w"]).float()

    def gather(self, idx, w, Vs):
        B, H, k = idx.shape
        out = torch.zeros((B, Vs.shape[1]), dtype=torch.float64)
        for b in range(B):
            for h in range(H):
                for t in range(k):
                    f = int(idx[b, h, t])
                    if self.r0 <= f < self.r1:
                        out[b] += float(w[b, h, t]) * Vs[f - self.r0].double()
        return out.float()

    def scatter(self, idx, w, d, Vs, dVs):
        B, H, k = idx.shape
        dw = torch.zeros((B, H, k))
        for b in range(B):
            for h in range(H):
                for t in range(k):
                    f = int(idx[b, h, t])
                    if self.r0 <= f < self.r1:
                        dw[b, h, t] = float((Vs[f - self.r0].double() * d[b].double()).sum())
                        dVs[f - self.r0] += float(w[b, h, t]) * d[b]
        return dw

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
        cfg = wl.tiny_config(6 * world, 2, 8, 8, 8, 3, torch.float32, torch.float32, index=77)
        Q, K, V, dOut = wl.make_all(cfg)
        B_l = cfg.batch // world
        n = cfg.n_slots
        r0, r1 = rank * n // world, (rank + 1) * n // world
        sp = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B_l,
                        phases=OraclePhases(cfg.n_sub, cfg.k, r0, r1))
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
            ShardedPKM(1, 5, 16, 16, 2, 4, phases=object())  # 25 rows over 2 ranks
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
