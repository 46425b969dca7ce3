"""Row-sharded value table across GPUs (BASELINE.json configs[3]; SURVEY.md
8(e)): the plumbing around the library's record
exchange (msn_pkm_exchange_* / msn_pkm_forward_sharded, include/msn_pkm.h).

Rank p of P holds value rows [p n/P, (p+1) n/P) and its own B_l queries; the
sub-keys are replicated (they are small).  One step:

  forward   SELECT: a1-a4 of the local queries (idx, w [B_l,H,k]) fused with
            the ROUTE (one 8-B record {row, w} per slot into its owner's
            window for this query) and the local shard's gather
            GATHER: per (remote source, query) partial sums -> back to the home
            COMBINE: the P partials added in owner order    -> out [B_l, d_v]
  backward  owners read the d_out rows of their records, SCATTER (dV shard +=,
            dw per record, deterministic grouped reduction), return dw;
            COLLECT puts dw in (b,h,t) order; backward_keys on the local
            queries -> dQ (=), dK (+=, this rank's queries: summing it across
            ranks is the caller's data-parallel job, like any replicated
            parameter).

transport="peer" (default): every rank's exchange buffer lives in torch
symmetric memory and is mapped into every peer (NVLink); the library's
kernels store records, partials and dw straight into the peers' buffers and
order the ranks with a device-side barrier: msn_pkm_forward_sharded /
msn_pkm_backward_sharded run the whole step, no host synchronisation, CUDA
graph capturable.  With world size 1 the buffer is a plain device tensor (the
same code path, nothing leaves the GPU).

transport="nccl": the same kernels with the STAGED layout; the data moves
with fixed-size torch.distributed collectives (NCCL over NVLink on the GPU
box; no host synchronisation): all_to_all_single of the record windows,
counts, partials and returned dw, all_gather of d_out.  Whole windows move
(P x B_l H k records per rank): the baseline the peer transport is measured
against (and the host logic the gloo tests cover).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import _lib

_DT = {"IN_ROW": torch.int32, "IN_W": torch.float32, "IN_CNT": torch.int32, "PART_IN": torch.float32,
       "DOUT": torch.float32, "DW_IN": torch.float32, "POS": torch.int32, "CTL": torch.int32,
       "OUT_ROW": torch.int32, "OUT_W": torch.float32, "OUT_CNT": torch.int32, "PART_OUT": torch.float32,
       "DOUT_ALL": torch.float32, "DW_OUT": torch.float32}


class ExchangeBuffer:
    """One rank's exchange buffer and typed views of its regions (the layout
    msn_pkm_exchange_layout reports)."""

    def __init__(self, lk, local_batch: int, world: int, rank: int, transport: str, group=None,
                 device=None, buf: Optional[torch.Tensor] = None, bases=None):
        self.world, self.rank, self.lb = world, rank, local_batch
        self.cap = local_batch * lk.heads * lk.k
        self.d_value = lk.d_value
        staged = transport == "nccl"
        self.offsets, nbytes = lk.exchange_layout(local_batch, staged)
        self.nbytes = nbytes
        self._hdl = None
        if buf is None:
            if transport == "peer" and world > 1:
                try:
                    import torch.distributed._symmetric_memory as symm
                except ImportError as e:  # pragma: no cover - depends on the torch build
                    raise RuntimeError("transport='peer' needs torch symmetric memory") from e
                buf = symm.empty(nbytes, dtype=torch.uint8, device=device)
                buf.zero_()
                self._hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
                bases = [int(p) for p in self._hdl.buffer_ptrs]
                torch.cuda.synchronize(device)
                self._hdl.barrier(channel=0)  # every buffer zeroed before any peer writes
            else:
                buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.buf = buf
        if bases is None:
            bases = [0] * world
            bases[rank] = buf.data_ptr()
        self.x = _lib.Exchange()
        self.x.transport = _lib.XCHG_STAGED if staged else _lib.XCHG_PEER
        self.x.world, self.x.rank, self.x.local_batch = world, rank, local_batch
        for p in range(_lib.MAX_WORLD):
            self.x.base[p] = bases[p] if p < world else None

    def region(self, name: str, *shape) -> torch.Tensor:
        dt = _DT[name]
        n = 1
        for s in shape:
            n *= s
        o = self.offsets[name]
        return self.buf[o:o + n * torch.tensor([], dtype=dt).element_size()].view(dt).view(*shape)

    # typed views
    def records(self, out: bool):
        """(row, w, cnt) views: [P, B_l * H * k] windows and [P, B_l] counts."""
        P, cap = self.world, self.cap
        pre = "OUT_" if out else "IN_"
        return (self.region(pre + "ROW", P, cap), self.region(pre + "W", P, cap), self.region(pre + "CNT", P, self.lb))


class ShardedPKM:
    def __init__(self, heads: int, n_sub: int, d_half: int, d_value: int, k: int,
                 local_batch: int, qk_dtype=torch.bfloat16, value_dtype=torch.bfloat16,
                 group=None, phases=None, device=None, transport: str = "peer",
                 dq_in_qk_dtype: bool = False):
        if transport not in ("peer", "nccl"):
            raise ValueError(f"transport {transport!r}: 'peer' or 'nccl'")
        self.transport = transport
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        n = n_sub * n_sub
        if n % self.world:
            raise ValueError(f"n_sub^2 = {n} is not divisible by the world size {self.world}")
        self.rows = n // self.world
        self.row_begin = self.rank * self.rows
        self.row_end = self.row_begin + self.rows
        self.heads, self.k, self.d_value, self.d_half, self.n_sub = heads, k, d_value, d_half, n_sub
        self.local_batch = local_batch
        if phases is None:
            from .pkm import PKMLookup
            phases = PKMLookup(heads, n_sub, d_half, d_value, k, max_batch=local_batch,
                               qk_dtype=qk_dtype, value_dtype=value_dtype, device=device,
                               world_size=self.world, rank=self.rank, dq_in_qk_dtype=dq_in_qk_dtype)
        self.ph = phases
        self.xb = ExchangeBuffer(phases, local_batch, self.world, self.rank, transport, group, device)
        self.ws = phases.workspace(local_batch, self.world * local_batch)
        self.launch_count = 0  # library kernel launches issued by this object (all calls)

    def _counted(self, r):
        self.launch_count += self.ph.last_launch_count()
        return r

    @property
    def exchange(self):
        return self.xb.x

    def value_shard(self, full_values: torch.Tensor) -> torch.Tensor:
        """This rank's rows of a full table (every rank generates the same seeded table)."""
        return full_values[self.row_begin:self.row_end].contiguous()

    # ------------------------------------------------------------ forward
    def forward(self, query: torch.Tensor, subkeys: torch.Tensor, value_shard: torch.Tensor,
                out: Optional[torch.Tensor] = None):
        """Returns (out [B_l, d_v], tape (idx, w)) for the local queries."""
        x = self.xb.x
        if self.transport == "peer":
            out, idx, w = self._counted(self.ph.forward_sharded(query, subkeys, value_shard, x, out=out, ws=self.ws))
            return out, (idx, w)
        idx, w, out = self._counted(self.ph.exchange_select(query, subkeys, value_shard, x, out=out, ws=self.ws))
        self._move_records()
        self._counted(self.ph.exchange_gather(value_shard, x))
        P, lb, dv = self.world, self.local_batch, self.d_value
        self._a2a(self.xb.region("PART_IN", P * lb * dv), self.xb.region("PART_OUT", P * lb * dv))
        out = self._counted(self.ph.exchange_combine(x, out))
        return out, (idx, w)

    # ----------------------------------------------------------- backward
    def backward(self, d_out: torch.Tensor, query: torch.Tensor, subkeys: torch.Tensor,
                 value_shard: torch.Tensor, tape, d_subkeys: Optional[torch.Tensor] = None,
                 d_value_shard: Optional[torch.Tensor] = None):
        """Returns (d_query, d_subkeys (this rank's part, +=), d_value_shard (+=), dw)."""
        idx, w = tape
        dev = d_out.device
        if d_value_shard is None:
            d_value_shard = torch.zeros((self.rows, self.d_value), dtype=torch.float32, device=dev)
        if d_subkeys is None:
            d_subkeys = torch.zeros((self.heads, 2, self.n_sub, self.d_half), dtype=torch.float32, device=dev)
        x = self.xb.x
        if self.transport == "peer":
            dq, dK, dV, dw = self._counted(self.ph.backward_sharded(d_out.float().contiguous(), query, subkeys,
                                                                    value_shard, idx, w, x, d_subkeys,
                                                                    d_value_shard, ws=self.ws))
            return dq, dK, dV, dw
        P, lb, dv = self.world, self.local_batch, self.d_value
        dall = self.xb.region("DOUT_ALL", P * lb, dv)
        if P > 1:
            dist.all_gather_into_tensor(dall, d_out.float().contiguous(), group=self.group)
        else:
            dall.copy_(d_out)
        self._counted(self.ph.exchange_scatter(value_shard, d_value_shard, x, ws=self.ws))
        P, cap = self.world, self.xb.cap
        self._a2a(self.xb.region("DW_IN", P * cap), self.xb.region("DW_OUT", P * cap))
        dw = self._counted(self.ph.exchange_collect(idx, x))
        dq, d_subkeys = self._counted(self.ph.backward_keys(query, subkeys, idx, w, dw, d_subkeys))
        return dq, d_subkeys, d_value_shard, dw

    # ------------------------------------------- the NCCL (staged) moves
    def _a2a(self, out: torch.Tensor, inp: torch.Tensor):
        """Fixed-size all-to-all: chunk p of inp -> rank p's chunk [rank] of out."""
        if self.world > 1:
            dist.all_to_all_single(out, inp, group=self.group)
        else:
            out.copy_(inp)

    def _move_records(self):
        o_row, o_w, o_cnt = self.xb.records(out=True)
        i_row, i_w, i_cnt = self.xb.records(out=False)
        for o, i in ((o_row, i_row), (o_w, i_w), (o_cnt, i_cnt)):
            self._a2a(i.view(-1), o.view(-1))
