"""Row-sharded value table across GPUs (BASELINE.json configs[3]).

Rank p of P holds value rows [p*n/P, (p+1)*n/P) and its own B_local queries;
the sub-keys are replicated (they are small).  One step:

  forward   select (a1-a4, local queries)             -> idx, w      [B_l,H,k]
            all-gather idx, w (8 B per contribution)   -> [P*B_l,H,k]
            gather over the local rows, all queries    -> partial [P*B_l,d_v]
            reduce-scatter(sum) of the partials        -> out [B_l,d_v]
  backward  all-gather d_out                           -> [P*B_l,d_v]
            scatter over the local rows: dV_shard +=, dw for local slots (0 else)
            reduce-scatter(sum) of dw  (one owner per element: the sum is exact)
            backward_keys on the local queries         -> dQ (=), dK (+=)

The collectives are torch.distributed calls (NCCL over NVLink/NVSwitch on the
GPU box): fixed-size, graph-capturable, no host synchronisation, NVLS-capable
(reduce-scatter).  transport="p2p" fuses the forward's gather with its
reduce-scatter instead: msn_pkm_gather_push stores every query's partial row
straight into the home rank's receive buffer (torch symmetric memory, NVLink
peer stores issued by the gather kernel as the rows are summed), a device-side
barrier orders the pushes, and msn_pkm_reduce_partials adds the world partials
in rank order (deterministic).  Its backward reads every d_out row from the
home rank's buffer inside the dV reducer and stores every dw element into the
home rank's buffer (msn_pkm_scatter_p2p): no all-gather of d_out, no
reduce-scatter of dw.  The data-path kernels are the C ABI's phase entry points
(msn_pkm_select / _gather / _scatter / _backward_keys).  dK is this rank's
contribution; summing it across ranks is the caller's data-parallel job
(like any replicated parameter).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


class ShardedPKM:
    def __init__(self, heads: int, n_sub: int, d_half: int, d_value: int, k: int,
                 local_batch: int, qk_dtype=torch.bfloat16, value_dtype=torch.bfloat16,
                 group=None, phases=None, device=None, transport: str = "nccl"):
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport {transport!r}: 'nccl' or 'p2p'")
        self.transport = transport
        self._symm = None
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
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
            phases = PKMLookup(heads, n_sub, d_half, d_value, k, max_batch=local_batch * self.world,
                               qk_dtype=qk_dtype, value_dtype=value_dtype,
                               row_begin=self.row_begin, row_end=self.row_end, device=device)
        self.ph = phases

    def value_shard(self, full_values: torch.Tensor) -> torch.Tensor:
        """This rank's rows of a full table (every rank generates the same seeded table)."""
        return full_values[self.row_begin:self.row_end].contiguous()

    def _all_gather(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.world * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x.contiguous(), group=self.group)
        return out

    def _reduce_scatter(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty((x.shape[0] // self.world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.reduce_scatter_tensor(out, x.contiguous(), op=dist.ReduceOp.SUM, group=self.group)
        return out

    def _p2p_buffers(self, B_l: int, device):
        """This rank's receive buffer [world, B_l, d_v] in symmetric memory and
        the device array of every rank's buffer address (peer-mapped)."""
        if self._symm is None or self._symm[0].shape[1] != B_l:
            try:
                import torch.distributed._symmetric_memory as symm
            except ImportError as e:  # pragma: no cover - depends on the torch build
                raise RuntimeError("transport='p2p' needs torch symmetric memory") from e
            buf = symm.empty((self.world, B_l, self.d_value), dtype=torch.float32, device=device)
            group = self.group if self.group is not None else dist.group.WORLD
            hdl = symm.rendezvous(buf, group)
            ptrs = torch.tensor([int(p) for p in hdl.buffer_ptrs], dtype=torch.int64, device=device)
            self._symm = (buf, hdl, ptrs)
        return self._symm

    def forward(self, query: torch.Tensor, subkeys: torch.Tensor, value_shard: torch.Tensor):
        """Returns (out [B_l,d_v], tape) for the local queries."""
        idx, w = self.ph.select(query, subkeys)
        idx_all = self._all_gather(idx)
        w_all = self._all_gather(w)
        if self.transport == "p2p":
            buf, hdl, ptrs = self._p2p_buffers(query.shape[0], query.device)
            hdl.barrier(channel=0)  # every rank is done reading its previous step's partials
            self.ph.gather_push(idx_all, w_all, value_shard, ptrs, self.world, self.rank)
            hdl.barrier(channel=0)  # every push has landed
            out = self.ph.reduce_partials(buf, self.world)
        else:
            part = self.ph.gather(idx_all, w_all, value_shard)
            out = self._reduce_scatter(part)
        return out, (idx, w, idx_all, w_all)

    def backward(self, d_out: torch.Tensor, query: torch.Tensor, subkeys: torch.Tensor,
                 value_shard: torch.Tensor, tape, d_subkeys: Optional[torch.Tensor] = None,
                 d_value_shard: Optional[torch.Tensor] = None):
        """Returns (d_query, d_subkeys (this rank's part, +=), d_value_shard (+=), dw)."""
        idx, w, idx_all, w_all = tape
        dev = d_out.device
        if d_value_shard is None:
            d_value_shard = torch.zeros((self.rows, self.d_value), dtype=torch.float32, device=dev)
        if self.transport == "p2p":
            dbuf, dwbuf, dh, dptrs, wptrs = self._p2p_bwd_buffers(d_out.shape[0], dev)
            dh.barrier(channel=0)  # every rank is done with the previous step's buffers
            dbuf.copy_(d_out.float())
            dh.barrier(channel=0)  # every rank's d_out is in place
            self.ph.scatter_p2p(idx_all, w_all, value_shard, d_value_shard, dptrs, wptrs, self.world)
            dh.barrier(channel=0)  # every owner's dw has landed
            dw = dwbuf.clone()
        else:
            d_all = self._all_gather(d_out.float())
            dw_part = self.ph.scatter(idx_all, w_all, d_all, value_shard, d_value_shard)
            dw = self._reduce_scatter(dw_part)
        dq, d_subkeys = self.ph.backward_keys(query, subkeys, idx, w, dw, d_subkeys)
        return dq, d_subkeys, d_value_shard, dw

    def _p2p_bwd_buffers(self, B_l: int, device):
        """Symmetric d_out [B_l, d_v] and dw [B_l, H, k] buffers of this rank and
        the device arrays of every rank's addresses."""
        if getattr(self, "_symm_bwd", None) is None or self._symm_bwd[0].shape[0] != B_l:
            import torch.distributed._symmetric_memory as symm
            group = self.group if self.group is not None else dist.group.WORLD
            dbuf = symm.empty((B_l, self.d_value), dtype=torch.float32, device=device)
            dh = symm.rendezvous(dbuf, group)
            wbuf = symm.empty((B_l, self.heads, self.k), dtype=torch.float32, device=device)
            wh = symm.rendezvous(wbuf, group)
            dptrs = torch.tensor([int(p) for p in dh.buffer_ptrs], dtype=torch.int64, device=device)
            wptrs = torch.tensor([int(p) for p in wh.buffer_ptrs], dtype=torch.int64, device=device)
            self._symm_bwd = (dbuf, wbuf, dh, dptrs, wptrs)
        return self._symm_bwd
