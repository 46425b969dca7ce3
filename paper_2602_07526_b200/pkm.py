"""Thin Python binding of the C ABI (include/msn_pkm.h): argument marshalling
only -- every step of the PKM lookup runs in the CUDA kernels of
libmsn_pkm.so.  PyTorch provides device memory, streams and (for the sharded
table) torch.distributed.

    lk = PKMLookup(heads=4, n_sub=512, d_half=256, d_value=256, k=32,
                   max_batch=4096, qk_dtype=torch.bfloat16,
                   value_dtype=torch.bfloat16)
    out, idx, w = lk.forward(q, K, V)                 # a1-a5
    dq, dK, dV, dw = lk.backward(d_out, q, K, V, idx, w)   # a6-a8

Inputs given as CPU tensors are copied to the device (and results back) --
the end-to-end path the bench's ``e2e`` number times.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

from . import _lib

_DT = {torch.float32: _lib.MSN_F32, torch.bfloat16: _lib.MSN_BF16}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class PKMLookup:
    """One PKM memory (H heads, per-head sub-key codebooks [H,2,n_sub,d_half],
    one value table [n_sub^2, d_value] or its row shard [row_begin,row_end))."""

    def __init__(self, heads: int, n_sub: int, d_half: int, d_value: int, k: int,
                 max_batch: int, qk_dtype=torch.bfloat16, value_dtype=torch.bfloat16,
                 atomic_bwd: bool = False, row_begin: int = 0, row_end: Optional[int] = None,
                 device=None, head_groups: int = 1, group_tables: bool = False,
                 dq_in_qk_dtype: bool = False, validate: bool = False, world_size: int = 0,
                 rank: int = 0):
        """head_groups G > 1: consecutive blocks of heads/G
        heads form a group (a token with its own codebooks); out is [B, G, d_v].
        group_tables: every group has its own table (values [G*n_sub^2, d_v]).
        dq_in_qk_dtype: d_query comes back in the query dtype (bf16 for bf16
        configs; MSN_FLAG_DQ_QK_DTYPE) instead of fp32.
        validate: every call that consumes a tape checks it first and raises
        on an invalid one (MSN_FLAG_VALIDATE; synchronises the stream).
        world_size P > 1, rank: the row-sharded table with the library's
        record exchange (a9): this handle holds rows [rank n/P, (rank+1) n/P)."""
        self.lib = _lib.load()
        self.heads, self.n_sub, self.d_half, self.d_value, self.k = heads, n_sub, d_half, d_value, k
        self.max_batch = max_batch
        self.qk_dtype, self.value_dtype = qk_dtype, value_dtype
        self.head_groups, self.group_tables = max(1, head_groups), group_tables
        self.table_rows = n_sub * n_sub * (self.head_groups if group_tables else 1)
        self.world_size, self.rank = world_size, rank
        if world_size > 1:
            rpr = self.table_rows // world_size
            row_begin, row_end = rank * rpr, (rank + 1) * rpr
        self.row_begin = row_begin
        self.row_end = self.table_rows if row_end is None else row_end
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        flags = (_lib.FLAG_ATOMIC_BWD if atomic_bwd else 0) | (_lib.FLAG_GROUP_TABLES if group_tables else 0) \
            | (_lib.FLAG_DQ_QK_DTYPE if dq_in_qk_dtype else 0) | (_lib.FLAG_VALIDATE if validate else 0)
        self.dq_dtype = qk_dtype if (dq_in_qk_dtype and qk_dtype == torch.bfloat16) else torch.float32
        cfg = _lib.Config(_lib.ABI_VERSION, heads, n_sub, d_half, d_value, k, max_batch,
                          _DT[qk_dtype], _DT[value_dtype], flags, self.head_groups,
                          self.row_begin, self.row_end, world_size, rank)
        h = ctypes.c_void_p()
        _lib.check(self.lib.msn_pkm_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self._ws = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.msn_pkm_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    # ---------------------------------------------------------------- utils
    @property
    def sharded(self) -> bool:
        return not (self.row_begin == 0 and self.row_end == self.table_rows)

    def _out_shape(self, B: int):
        return (B, self.d_value) if self.head_groups == 1 else (B, self.head_groups, self.d_value)

    def workspace_bytes(self, B: int, gather_batch: Optional[int] = None) -> Tuple[int, int]:
        f, b = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(self.lib.msn_pkm_workspace_size(self._h, B, B if gather_batch is None else gather_batch,
                                                   ctypes.byref(f), ctypes.byref(b)))
        return f.value, b.value

    def workspace(self, B: int, gather_batch: Optional[int] = None) -> torch.Tensor:
        need = max(self.workspace_bytes(B, gather_batch))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def last_launch_count(self) -> int:
        return int(self.lib.msn_pkm_last_launch_count(self._h))

    def _dev(self, t: torch.Tensor) -> torch.Tensor:
        if t.device.type != "cuda":
            t = t.to(self.device, non_blocking=True)
        return t.contiguous()

    def _check_inputs(self, query, subkeys, values=None):
        H, d = self.heads, self.d_half
        if query.dim() != 4 or tuple(query.shape[1:]) != (H, 2, d) or query.dtype != self.qk_dtype:
            raise ValueError(f"query must be [B,{H},2,{d}] {self.qk_dtype}, got {tuple(query.shape)} {query.dtype}")
        if tuple(subkeys.shape) != (H, 2, self.n_sub, d) or subkeys.dtype != self.qk_dtype:
            raise ValueError(f"subkeys must be [{H},2,{self.n_sub},{d}] {self.qk_dtype}")
        if values is not None:
            rows = self.row_end - self.row_begin
            if tuple(values.shape) != (rows, self.d_value) or values.dtype != self.value_dtype:
                raise ValueError(f"values must be [{rows},{self.d_value}] {self.value_dtype}")

    # ------------------------------------------------------------ forward
    def forward(self, query: torch.Tensor, subkeys: torch.Tensor, values: torch.Tensor):
        """a1-a5.  Returns (out [B,d_v] fp32, idx [B,H,k] int32, w [B,H,k] fp32)."""
        host = query.device.type != "cuda"
        self._check_inputs(query, subkeys, values)
        q, K, V = self._dev(query), self._dev(subkeys), self._dev(values)
        B = q.shape[0]
        out = torch.empty(self._out_shape(B), dtype=torch.float32, device=self.device)
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_forward(self._h, _stream(), B, _ptr(q), _ptr(K), _ptr(V),
                                            _ptr(out), _ptr(idx), _ptr(w), _ptr(ws), ws.numel()))
        if host:
            return out.cpu(), idx.cpu(), w.cpu()
        return out, idx, w

    def forward_qln(self, query: torch.Tensor, subkeys: torch.Tensor, values: torch.Tensor):
        """a1-a5 on q^ = LN(query), the LayerNorm folded into the scorer's
        operand load.  Returns (out, idx, w, q_hat)."""
        self._check_inputs(query, subkeys, values)
        q, K, V = self._dev(query), self._dev(subkeys), self._dev(values)
        B = q.shape[0]
        out = torch.empty(self._out_shape(B), dtype=torch.float32, device=self.device)
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        q_hat = torch.empty_like(q)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_forward_qln(self._h, _stream(), B, _ptr(q), _ptr(K), _ptr(V), _ptr(out),
                                                _ptr(idx), _ptr(w), _ptr(q_hat), _ptr(ws), ws.numel()))
        return out, idx, w, q_hat

    def forward_gated(self, query: torch.Tensor, subkeys: torch.Tensor, values: torch.Tensor,
                      x_in: torch.Tensor, gate: str = "tanh"):
        """a1-a5 plus the memory-gated fusion x~ = x_in * g(v_o) (SURVEY 8(f)
        f1; gate in tanh / sigmoid / identity),
        fused into the kernel that produces v_o.  Returns (x~, v_o, idx, w)."""
        self._check_inputs(query, subkeys, values)
        q, K, V = self._dev(query), self._dev(subkeys), self._dev(values)
        B = q.shape[0]
        x = self._dev(x_in).float().contiguous()
        if tuple(x.shape) != self._out_shape(B):
            raise ValueError(f"x_in must be {self._out_shape(B)}")
        out = torch.empty(self._out_shape(B), dtype=torch.float32, device=self.device)
        xt = torch.empty_like(out)
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_forward_gated(self._h, _stream(), B, _ptr(q), _ptr(K), _ptr(V), _ptr(x),
                                                  _lib.GATES[gate], _ptr(out), _ptr(xt), _ptr(idx), _ptr(w),
                                                  _ptr(ws), ws.numel()))
        return xt, out, idx, w

    def gate_backward(self, d_xt: torch.Tensor, x_in: torch.Tensor, v_o: torch.Tensor, gate: str = "tanh"):
        """Backward of the gate: (d_x_in, d_v_o); d_v_o is the d_out of backward()."""
        d, x, v = (self._dev(t).float().contiguous() for t in (d_xt, x_in, v_o))
        B = d.shape[0]
        dx = torch.empty_like(d)
        dvo = torch.empty_like(d)
        _lib.check(self.lib.msn_pkm_gate_backward(self._h, _stream(), B, _lib.GATES[gate], _ptr(x), _ptr(v),
                                                  _ptr(d), _ptr(dx), _ptr(dvo)))
        return dx, dvo

    # ------------------------------------------- prologue
    def layernorm(self, x: torch.Tensor) -> torch.Tensor:
        """LN over the last axis (width d_half), qk dtype in and out."""
        x = self._dev(x)
        y = torch.empty_like(x)
        rows = x.numel() // self.d_half
        _lib.check(self.lib.msn_pkm_layernorm(self._h, _stream(), rows, _ptr(x), _ptr(y)))
        return y

    def layernorm_backward(self, x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
        x, dy = self._dev(x), self._dev(dy).float().contiguous()
        dx = torch.empty(x.shape, dtype=torch.float32, device=self.device)
        rows = x.numel() // self.d_half
        _lib.check(self.lib.msn_pkm_layernorm_backward(self._h, _stream(), rows, _ptr(x), _ptr(dy), _ptr(dx)))
        return dx

    def key_transform(self, k_hat: torch.Tensor, theta: torch.Tensor) -> torch.Tensor:
        """K~ = Theta k^ per (head, half); theta [H,2,d,d] fp32."""
        k_hat, theta = self._dev(k_hat), self._dev(theta).float().contiguous()
        k_eff = torch.empty_like(k_hat)
        _lib.check(self.lib.msn_pkm_key_transform(self._h, _stream(), _ptr(k_hat), _ptr(theta), _ptr(k_eff)))
        return k_eff

    def key_transform_backward(self, k_hat, theta, d_k_eff, d_theta: Optional[torch.Tensor] = None):
        """-> (d_k_hat, d_theta); d_theta accumulated into when given."""
        k_hat, theta = self._dev(k_hat), self._dev(theta).float().contiguous()
        d = self._dev(d_k_eff).float().contiguous()
        d_k_hat = torch.empty(k_hat.shape, dtype=torch.float32, device=self.device)
        if d_theta is None:
            d_theta = torch.zeros(theta.shape, dtype=torch.float32, device=self.device)
        _lib.check(self.lib.msn_pkm_key_transform_backward(self._h, _stream(), _ptr(k_hat), _ptr(theta), _ptr(d),
                                                           _ptr(d_k_hat), _ptr(d_theta)))
        return d_k_hat, d_theta

    def select(self, query: torch.Tensor, subkeys: torch.Tensor):
        """a1-a4 only: (idx, w)."""
        self._check_inputs(query, subkeys)
        q, K = self._dev(query), self._dev(subkeys)
        B = q.shape[0]
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_select(self._h, _stream(), B, _ptr(q), _ptr(K), _ptr(idx),
                                           _ptr(w), _ptr(ws), ws.numel()))
        return idx, w

    def validate_tape(self, idx: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        """Number of invalid slots of the tape (idx outside the lookup's table,
        repeated within a lookup, weight not in [0, 1]) as a device int32 tensor."""
        idx, w = self._dev(idx), self._dev(w)
        bad = torch.empty(1, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.msn_pkm_validate_tape(self._h, _stream(), idx.shape[0], _ptr(idx), _ptr(w),
                                                  _ptr(bad)))
        return bad

    def gather(self, idx: torch.Tensor, w: torch.Tensor, values: torch.Tensor) -> torch.Tensor:
        """a5 over this process's rows (rows of other shards contribute 0)."""
        idx, w, V = self._dev(idx), self._dev(w), self._dev(values)
        B = idx.shape[0]
        out = torch.empty(self._out_shape(B), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.msn_pkm_gather(self._h, _stream(), B, _ptr(idx), _ptr(w), _ptr(V), _ptr(out)))
        return out

    # ----------------------------------------------------------- backward
    def backward(self, d_out, query, subkeys, values, idx, w,
                 d_subkeys: Optional[torch.Tensor] = None, d_values: Optional[torch.Tensor] = None):
        """a6-a8.  d_subkeys / d_values are accumulated into when given (+=),
        else zero-initialised.  Returns (d_query, d_subkeys, d_values, dw)."""
        host = d_out.device.type != "cuda"
        self._check_inputs(query, subkeys, values)
        d, q, K, V = self._dev(d_out), self._dev(query), self._dev(subkeys), self._dev(values)
        idx, w = self._dev(idx), self._dev(w)
        B = q.shape[0]
        if d_subkeys is None:
            d_subkeys = torch.zeros((self.heads, 2, self.n_sub, self.d_half), dtype=torch.float32, device=self.device)
        if d_values is None:
            d_values = torch.zeros((self.row_end - self.row_begin, self.d_value), dtype=torch.float32, device=self.device)
        d_query = torch.empty((B, self.heads, 2, self.d_half), dtype=self.dq_dtype, device=self.device)
        dw = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_backward(self._h, _stream(), B, _ptr(d), _ptr(q), _ptr(K), _ptr(V),
                                             _ptr(idx), _ptr(w), _ptr(d_query), _ptr(d_subkeys),
                                             _ptr(d_values), _ptr(dw), _ptr(ws), ws.numel()))
        if host:  # every result back on the caller's (host) device
            return d_query.cpu(), d_subkeys.cpu(), d_values.cpu(), dw.cpu()
        return d_query, d_subkeys, d_values, dw

    def scatter(self, idx, w, d_out, values, d_values, gather_batch: Optional[int] = None):
        """a6 over this process's rows: d_values += ..., returns dw (0 for
        slots held by other shards)."""
        idx, w, d, V = self._dev(idx), self._dev(w), self._dev(d_out), self._dev(values)
        B = idx.shape[0]
        dw = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        f, b = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(self.lib.msn_pkm_workspace_size(self._h, 0, B, ctypes.byref(f), ctypes.byref(b)))
        ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=self.device) \
            if self._ws is None or self._ws.numel() < b.value else self._ws
        _lib.check(self.lib.msn_pkm_scatter(self._h, _stream(), B, _ptr(idx), _ptr(w), _ptr(d), _ptr(V),
                                            _ptr(d_values), _ptr(dw), _ptr(ws), ws.numel()))
        return dw

    def scatter_update(self, idx, w, d_out, values, update: str = "sgd", lr: float = 1e-3,
                       eps: float = 1e-10, state: Optional[torch.Tensor] = None):
        """a6 with the optimiser step fused: values is updated
        IN PLACE (SGD / Adagrad on the touched rows, state += g^2 for Adagrad);
        returns dw (computed from the values before the update)."""
        rows = self.row_end - self.row_begin
        if values.device.type != "cuda" or tuple(values.shape) != (rows, self.d_value) \
                or values.dtype != self.value_dtype or not values.is_contiguous():
            raise ValueError(f"values must be a contiguous CUDA tensor [{rows},{self.d_value}] {self.value_dtype} "
                             "(updated in place)")
        if update == "adagrad" and (state is None or state.device.type != "cuda" or state.dtype != torch.float32
                                    or tuple(state.shape) != (rows, self.d_value) or not state.is_contiguous()):
            raise ValueError(f"Adagrad needs state: a contiguous CUDA fp32 tensor [{rows},{self.d_value}]")
        if update not in _lib.UPDATES:
            raise ValueError(f"update {update!r}: 'sgd' or 'adagrad'")
        idx, w, d = self._dev(idx), self._dev(w), self._dev(d_out)
        Bg = idx.shape[0]
        dw = torch.empty((Bg, self.heads, self.k), dtype=torch.float32, device=self.device)
        f, b = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(self.lib.msn_pkm_workspace_size(self._h, 0, Bg, ctypes.byref(f), ctypes.byref(b)))
        ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=self.device) \
            if self._ws is None or self._ws.numel() < b.value else self._ws
        _lib.check(self.lib.msn_pkm_scatter_update(self._h, _stream(), Bg, _ptr(idx), _ptr(w), _ptr(d),
                                                   _ptr(values), _lib.UPDATES[update], float(lr), float(eps),
                                                   _ptr(state), _ptr(dw), _ptr(ws), ws.numel()))
        return dw

    def backward_keys(self, query, subkeys, idx, w, dw, d_subkeys: Optional[torch.Tensor] = None):
        """a7-a8 given the full dw: (d_query, d_subkeys)."""
        q, K, idx, w, dw = (self._dev(t) for t in (query, subkeys, idx, w, dw))
        B = q.shape[0]
        if d_subkeys is None:
            d_subkeys = torch.zeros((self.heads, 2, self.n_sub, self.d_half), dtype=torch.float32, device=self.device)
        d_query = torch.empty((B, self.heads, 2, self.d_half), dtype=self.dq_dtype, device=self.device)
        ws = self.workspace(B)
        _lib.check(self.lib.msn_pkm_backward_keys(self._h, _stream(), B, _ptr(q), _ptr(K), _ptr(idx), _ptr(w),
                                                  _ptr(dw), _ptr(d_query), _ptr(d_subkeys), _ptr(ws), ws.numel()))
        return d_query, d_subkeys


    # ------------------------------------- a9 record exchange (sharded table)
    def exchange_layout(self, local_batch: int, staged: bool):
        """{region name: byte offset} and the total bytes of one exchange buffer."""
        offs = (ctypes.c_int64 * len(_lib.XREG))()
        nb = ctypes.c_size_t()
        _lib.check(self.lib.msn_pkm_exchange_layout(self._h, local_batch, int(staged), offs, ctypes.byref(nb)))
        return dict(zip(_lib.XREG, list(offs))), nb.value

    def forward_sharded(self, query, subkeys, values, xchg, out=None, idx=None, w=None, ws=None):
        """a1-a5 + a9 over peer memory (msn_pkm_forward_sharded): out [B_l, d_v]."""
        B = query.shape[0]
        if out is None:
            out = torch.empty((B, self.d_value), dtype=torch.float32, device=self.device)
        if idx is None:
            idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        if w is None:
            w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        if ws is None:
            ws = self.workspace(B, xchg.world * B)
        _lib.check(self.lib.msn_pkm_forward_sharded(self._h, _stream(), B, _ptr(query), _ptr(subkeys), _ptr(values),
                                                    ctypes.byref(xchg), _ptr(out), _ptr(idx), _ptr(w),
                                                    _ptr(ws), ws.numel()))
        return out, idx, w

    def backward_sharded(self, d_out, query, subkeys, values, idx, w, xchg, d_subkeys, d_values,
                         d_query=None, dw=None, ws=None):
        """a6-a8 + a9 over peer memory (msn_pkm_backward_sharded)."""
        B = query.shape[0]
        if d_query is None:
            d_query = torch.empty((B, self.heads, 2, self.d_half), dtype=self.dq_dtype, device=self.device)
        if dw is None:
            dw = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        if ws is None:
            ws = self.workspace(B, xchg.world * B)
        _lib.check(self.lib.msn_pkm_backward_sharded(self._h, _stream(), B, _ptr(d_out), _ptr(query), _ptr(subkeys),
                                                     _ptr(values), _ptr(idx), _ptr(w), ctypes.byref(xchg),
                                                     _ptr(d_query), _ptr(d_subkeys), _ptr(d_values), _ptr(dw),
                                                     _ptr(ws), ws.numel()))
        return d_query, d_subkeys, d_values, dw

    def exchange_select(self, query, subkeys, values, xchg, out=None, ws=None):
        """a1-a4 fused with the route and the local shard's gather: (idx, w) and,
        with P = 1, out."""
        B = query.shape[0]
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=self.device)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=self.device)
        if out is None and xchg.world == 1:
            out = torch.empty((B, self.d_value), dtype=torch.float32, device=self.device)
        if ws is None:
            ws = self.workspace(B, xchg.world * B)
        _lib.check(self.lib.msn_pkm_exchange_select(self._h, _stream(), _ptr(query), _ptr(subkeys), _ptr(values),
                                                    ctypes.byref(xchg), _ptr(idx), _ptr(w), _ptr(out),
                                                    _ptr(ws), ws.numel()))
        return idx, w, out

    def exchange_gather(self, values, xchg):
        _lib.check(self.lib.msn_pkm_exchange_gather(self._h, _stream(), _ptr(values), ctypes.byref(xchg)))

    def exchange_combine(self, xchg, out=None):
        """out = sum of the P partials (P = 1: out is what exchange_select wrote)."""
        if out is None:
            out = torch.empty((xchg.local_batch, self.d_value), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.msn_pkm_exchange_combine(self._h, _stream(), ctypes.byref(xchg), _ptr(out)))
        return out

    def exchange_scatter(self, values, d_values, xchg, ws=None):
        if ws is None:
            ws = self.workspace(xchg.local_batch, xchg.world * xchg.local_batch)
        _lib.check(self.lib.msn_pkm_exchange_scatter(self._h, _stream(), _ptr(values), _ptr(d_values),
                                                     ctypes.byref(xchg), _ptr(ws), ws.numel()))

    def exchange_collect(self, idx, xchg, dw=None):
        if dw is None:
            dw = torch.empty(tuple(idx.shape), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.msn_pkm_exchange_collect(self._h, _stream(), _ptr(idx), ctypes.byref(xchg), _ptr(dw)))
        return dw

    def exchange_barrier(self, xchg):
        _lib.check(self.lib.msn_pkm_exchange_barrier(self._h, _stream(), ctypes.byref(xchg)))

    def step_host(self, query_h, d_out_h, subkeys, values, d_subkeys, d_values,
                  out_h=None, d_query_h=None, chunks: Optional[int] = None):
        """One forward+backward fed from host memory: H2D copies of the query
        and the upstream gradient (pinned host tensors), a1-a8 on the device
        (d_subkeys/d_values device buffers accumulated), D2H copies of out and
        d_query into pinned host tensors, one synchronisation at the end.
        The batch runs as `chunks` consecutive slices (default: 2 when every
        slice keeps >= 1024 queries) so that the copies overlap the kernels:
        H2D of slice c+1 and D2H of slice c-1 on their own streams while the
        compute stream runs slice c.  The library calls stay in one fixed
        order on one stream, so the result is deterministic (d_values /
        d_subkeys receive the slices' sums one after another).
        Returns (out_h, d_query_h)."""
        B = query_h.shape[0]
        if out_h is None:
            out_h = torch.empty(self._out_shape(B), dtype=torch.float32).pin_memory()
        if d_query_h is None:
            d_query_h = torch.empty((B, self.heads, 2, self.d_half), dtype=self.dq_dtype).pin_memory()
        if chunks is None:
            # measured on the B200 (C2, bf16 d_query): 2 slices 0.78 ms, 3: 0.82,
            # 4: 0.84, 6: 1.00 (a slice of B/n queries costs more than 1/n of the
            # whole batch's kernels); MSN_HOST_CHUNKS overrides
            chunks = int(os.environ.get("MSN_HOST_CHUNKS", "0")) or (2 if B >= 2 * 1024 else 1)
        chunks = max(1, min(chunks, B)) if B > 0 else 1
        dev = self.device
        q = torch.empty(query_h.shape, dtype=query_h.dtype, device=dev)
        d = torch.empty(d_out_h.shape, dtype=d_out_h.dtype, device=dev)
        self._check_inputs(q, subkeys, values)
        out = torch.empty(self._out_shape(B), dtype=torch.float32, device=dev)
        idx = torch.empty((B, self.heads, self.k), dtype=torch.int32, device=dev)
        w = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=dev)
        dq = torch.empty((B, self.heads, 2, self.d_half), dtype=self.dq_dtype, device=dev)
        dw = torch.empty((B, self.heads, self.k), dtype=torch.float32, device=dev)
        step = (B + chunks - 1) // chunks
        ws = self.workspace(min(B, step))
        main = torch.cuda.current_stream(dev)
        if not hasattr(self, "_streams"):
            self._streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        s_in, s_comp, s_out = self._streams
        for st in self._streams:
            st.wait_stream(main)
        sc = ctypes.c_void_p(s_comp.cuda_stream)
        spans = [(c0, min(B, c0 + step)) for c0 in range(0, B, step)] if B > 0 else []
        ev_q, ev_d = [], []
        with torch.cuda.stream(s_in):
            for c0, c1 in spans:  # the slice's query first (its forward needs only that)
                q[c0:c1].copy_(query_h[c0:c1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
                ev_q.append(e)
                d[c0:c1].copy_(d_out_h[c0:c1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
                ev_d.append(e)
        for (c0, c1), eq, ed in zip(spans, ev_q, ev_d):
            n = c1 - c0
            s_comp.wait_event(eq)
            _lib.check(self.lib.msn_pkm_forward(self._h, sc, n, _ptr(q[c0:c1]), _ptr(subkeys), _ptr(values),
                                                _ptr(out[c0:c1]), _ptr(idx[c0:c1]), _ptr(w[c0:c1]),
                                                _ptr(ws), ws.numel()))
            e_f = torch.cuda.Event()
            e_f.record(s_comp)
            s_comp.wait_event(ed)
            _lib.check(self.lib.msn_pkm_backward(self._h, sc, n, _ptr(d[c0:c1]), _ptr(q[c0:c1]), _ptr(subkeys),
                                                 _ptr(values), _ptr(idx[c0:c1]), _ptr(w[c0:c1]), _ptr(dq[c0:c1]),
                                                 _ptr(d_subkeys), _ptr(d_values), _ptr(dw[c0:c1]),
                                                 _ptr(ws), ws.numel()))
            e_b = torch.cuda.Event()
            e_b.record(s_comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(e_f)
                out_h[c0:c1].copy_(out[c0:c1], non_blocking=True)
                s_out.wait_event(e_b)
                d_query_h[c0:c1].copy_(dq[c0:c1], non_blocking=True)
        for st in self._streams:
            main.wait_stream(st)
        # the device buffers stay alive until the copies complete
        for t in (q, d, out, idx, w, dq, dw, ws):
            t.record_stream(s_comp)
        main.synchronize()
        return out_h, d_query_h


class PKMFunction(torch.autograd.Function):
    """autograd wrapper: out = PKM(query; subkeys, values).  Gradients: query
    (=), subkeys and values (fp32, cast to the parameter dtype by autograd)."""

    @staticmethod
    def forward(ctx, lookup: PKMLookup, query, subkeys, values):
        out, idx, w = lookup.forward(query, subkeys, values)
        ctx.lookup = lookup
        ctx.save_for_backward(query, subkeys, values, idx, w)
        return out

    @staticmethod
    def backward(ctx, d_out):
        q, K, V, idx, w = ctx.saved_tensors
        dq, dK, dV, _ = ctx.lookup.backward(d_out.contiguous().float(), q, K, V, idx, w)
        return (None, dq.to(q.device, q.dtype), dK.to(K.device, K.dtype), dV.to(V.device, V.dtype))


def pkm(lookup: PKMLookup, query, subkeys, values):
    return PKMFunction.apply(lookup, query, subkeys, values)
