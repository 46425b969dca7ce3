"""GPU parity of the row-sharded table's record exchange (a9; SURVEY.md 8(e);
BASELINE.json configs[3]) against the fp64 oracle.

P ranks are emulated on one GPU: every rank has its own handle (world_size P,
rank r: rows [r n/P, (r+1) n/P)) and its own exchange buffer, all on this
device.  The phases (route, gather, combine, scatter, collect) run rank by
rank on one stream, so every emulated rank's kernels complete before the next
phase starts and no barrier is needed (no two ranks ever wait on each other).
PEER transport: the buffers are passed as each other's "peer" mappings (the
kernels store into the other ranks' buffers, as over NVLink).  STAGED
transport: the test moves the OUT regions into the IN regions exactly as the
NCCL collectives of distributed.py do (counted records, fixed-size offsets
and partials, the all-gathered d_out, the returned dw).  The combined out,
idx/w, every dV shard, dw, dQ and dK (summed over ranks, as the caller's data
parallelism does) are compared with the fp64 oracle through
tests/parity.py; the dV shards are also bitwise equal to the unsharded dV
(contribution ids are global, so every row is summed in the same order).
Needs a B200."""
import numpy as np
import pytest
import torch

from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.distributed import ExchangeBuffer
from paper_2602_07526_b200.pkm import PKMLookup
from tests import parity

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _handles(cfg, P, B_l):
    return [PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, max_batch=B_l,
                      qk_dtype=cfg.qk_dtype, value_dtype=cfg.value_dtype, device=DEV,
                      world_size=P if P > 1 else 0, rank=r) for r in range(P)]


def _buffers(lks, P, B_l, transport):
    xbs = []
    for r in range(P):
        _, nbytes = lks[r].exchange_layout(B_l, transport == "nccl")
        # NaN-filled (but zeroed control words): a region read before it is written shows up
        buf = torch.full((nbytes,), 0xFF, dtype=torch.uint8, device=DEV)
        xbs.append(ExchangeBuffer(lks[r], B_l, P, r, transport, buf=buf))
        xbs[-1].region("CTL", 64).zero_()
    if transport == "peer":
        for xb in xbs:
            for p in range(P):
                xb.x.base[p] = xbs[p].buf.data_ptr()
    return xbs


def run_emulated(cfg, Q, K, V, dOut, P, transport):
    """The sharded step of P emulated ranks.  Returns the full-batch results."""
    B = Q.shape[0]
    B_l = B // P
    n = cfg.n_slots
    rpr = n // P
    lks = _handles(cfg, P, B_l)
    xbs = _buffers(lks, P, B_l, transport)
    qs = [Q[r * B_l:(r + 1) * B_l].contiguous() for r in range(P)]
    vs = [V[r * rpr:(r + 1) * rpr] for r in range(P)]  # contiguous row slices
    tape, outs = [], []
    for r in range(P):
        idx, w, o = lks[r].exchange_select(qs[r], K, vs[r], xbs[r].x)
        tape.append((idx, w))
        outs.append(o)
    torch.cuda.synchronize()
    if transport == "nccl":  # what _move_records does with NCCL: whole windows, all-to-all
        for s in range(P):
            o_row, o_w, o_cnt = xbs[s].records(out=True)
            for o in range(P):
                i_row, i_w, i_cnt = xbs[o].records(out=False)
                i_row[s] = o_row[o]
                i_w[s] = o_w[o]
                i_cnt[s] = o_cnt[o]
    for r in range(P):
        lks[r].exchange_gather(vs[r], xbs[r].x)
    torch.cuda.synchronize()
    if transport == "nccl":  # all_to_all_single of the partials (the local one included)
        for s in range(P):
            pin = xbs[s].region("PART_IN", P, B_l, cfg.d_value)
            for o in range(P):
                pin[o] = xbs[o].region("PART_OUT", P, B_l, cfg.d_value)[s]
    if P > 1:
        outs = [lks[r].exchange_combine(xbs[r].x) for r in range(P)]
    # backward
    for r in range(P):
        if transport == "peer":
            xbs[r].region("DOUT", B_l, cfg.d_value).copy_(dOut[r * B_l:(r + 1) * B_l])
        else:
            xbs[r].region("DOUT_ALL", P * B_l, cfg.d_value).copy_(dOut)
    dvs = [torch.zeros((rpr, cfg.d_value), dtype=torch.float32, device=DEV) for _ in range(P)]
    for r in range(P):
        lks[r].exchange_scatter(vs[r], dvs[r], xbs[r].x)
    torch.cuda.synchronize()
    if transport == "nccl":  # the returned dw: whole windows, all-to-all
        for s in range(P):
            d_in = xbs[s].region("DW_IN", P, xbs[s].cap)
            for o in range(P):
                d_in[o] = xbs[o].region("DW_OUT", P, xbs[o].cap)[s]
    dws = [lks[r].exchange_collect(tape[r][0], xbs[r].x) for r in range(P)]
    dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=DEV)
    dqs = []
    for r in range(P):
        dq, _ = lks[r].backward_keys(qs[r], K, tape[r][0], tape[r][1], dws[r], dK)
        dqs.append(dq)
    torch.cuda.synchronize()
    return {"out": torch.cat(outs), "idx": torch.cat([t[0] for t in tape]), "w": torch.cat([t[1] for t in tape]),
            "dV": torch.cat(dvs), "dw": torch.cat(dws), "dQ": torch.cat(dqs), "dK": dK, "dV_shards": dvs,
            "counts": [int(xbs[r].records(out=False)[2].sum()) for r in range(P)]}


def _check(cfg, Q, K, V, dOut, res):
    Qc, Kc, Vc = Q.cpu(), K.cpu(), V.cpu()
    o, aff, rep = parity.check_forward(Qc, Kc, Vc, cfg.k, res["out"], res["idx"], res["w"])
    _, rb = parity.check_backward(Qc, Kc, Vc, cfg.k, dOut.cpu(), o, aff, res["dQ"], res["dK"], res["dV"],
                                  res["dw"], gpu_idx=res["idx"])
    rep.update(rb)
    return rep


CASES = [  # (config, batch)
    ("c2_mid_bf16", 512),
    ("c4_large_sharded_bf16", 256),
]


@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("name,B", CASES)
def test_exchange_emulated_ranks_vs_oracle(name, B, P, transport):
    cfg = wl.CONFIGS[name].scaled(batch=B)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    res = run_emulated(cfg, Q, K, V, dOut, P, transport)
    # every record reached exactly one owner: sum of counts = B * H * k
    assert sum(res["counts"]) == B * cfg.heads * cfg.k
    rep = _check(cfg, Q, K, V, dOut, res)
    print(name, P, transport, rep)
    # dV shards bitwise equal to the unsharded deterministic backward
    lk = PKMLookup(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, max_batch=B, qk_dtype=cfg.qk_dtype,
                   value_dtype=cfg.value_dtype, device=DEV)
    out_f, idx_f, w_f = lk.forward(Q, K, V)
    dq_f, dK_f, dV_f, dw_f = lk.backward(dOut, Q, K, V, idx_f, w_f)
    torch.cuda.synchronize()
    assert torch.equal(res["idx"], idx_f) and torch.equal(res["w"], w_f)
    assert torch.equal(res["dV"], dV_f), "dV shards differ from the unsharded dV"
    assert torch.equal(res["dw"], dw_f), "dw differs from the unsharded dw"
    torch.testing.assert_close(res["out"], out_f, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("B", [257, 1024])
def test_forward_backward_sharded_p1_vs_phases_and_oracle(B):
    """msn_pkm_forward_sharded / msn_pkm_backward_sharded (the whole step with
    device barriers) at world size 1 on C4 shapes: bitwise equal to the
    emulated phases, and within tolerance of the oracle."""
    from paper_2602_07526_b200.distributed import ShardedPKM
    cfg = wl.CONFIGS["c4_large_sharded_bf16"].scaled(batch=B)
    Q, K, V, dOut = wl.make_all(cfg, DEV)
    sp = ShardedPKM(cfg.heads, cfg.n_sub, cfg.d_half, cfg.d_value, cfg.k, B, cfg.qk_dtype, cfg.value_dtype,
                    device=DEV, transport="peer")
    dK = torch.zeros((cfg.heads, 2, cfg.n_sub, cfg.d_half), dtype=torch.float32, device=DEV)
    dV = torch.zeros((cfg.n_slots, cfg.d_value), dtype=torch.float32, device=DEV)
    for it in range(2):  # twice: the barrier epochs advance, buffers are reused
        dK.zero_()
        dV.zero_()
        out, tape = sp.forward(Q, K, V)
        dq, _, _, dw = sp.backward(dOut, Q, K, V, tape, d_subkeys=dK, d_value_shard=dV)
    torch.cuda.synchronize()
    ctl = sp.xb.region("CTL", 64).cpu()
    assert ctl[17].item() == 0  # no barrier timeout (one rank: the composite needs none)
    # the barrier phase itself: epochs advance, own flag set, no timeout
    for _ in range(3):
        sp.ph.exchange_barrier(sp.xb.x)
    torch.cuda.synchronize()
    ctl = sp.xb.region("CTL", 64).cpu()
    assert ctl[16].item() == ctl[0].item() == 3 and ctl[17].item() == 0
    ref = run_emulated(cfg, Q, K, V, dOut, 1, "peer")
    assert torch.equal(out, ref["out"]) and torch.equal(tape[0], ref["idx"]) and torch.equal(dw, ref["dw"])
    assert torch.equal(dq, ref["dQ"])
    assert torch.equal(dV, ref["dV"]) and torch.equal(dK, ref["dK"])
    res = dict(ref)
    rep = _check(cfg, Q, K, V, dOut, res)
    print(B, rep)
