"""Multi-GPU LookupFFN forward: one process per GPU over torch.distributed.

No reference counterpart (the reference is single-process);
the partitioning follows SURVEY.md 8e / BASELINE.json north_star:

* ``mode="token"``  tables replicated, rank r runs its own token block; no
  collective on the data path (optionally an all-gather of y).
* ``mode="table"``  rank r owns the table slice [r*h/P, (r+1)*h/P), produces
  the fp32 PARTIAL y over its tables for all tokens, and the partials are
  combined by ``combine="reduce_scatter"`` (rank r keeps token rows
  [r*n/P, (r+1)*n/P), BASELINE c3) or ``combine="all_reduce"`` (every rank
  keeps all of y, c4).  The hash of a token needs its whole projection (the
  signflip FWHT mixes every coordinate), so it is not table-separable:
  ``hash_mode="token"`` (default) hashes only the rank's own token block for
  ALL tables and exchanges the (code, coeff) records with one all-to-all
  (rank q receives the records of its tables for every token: n * h/P * 8
  bytes, against the n * d_out * 4-byte partials of the combine), so the
  hash costs 1/P per rank; ``hash_mode="replicated"`` recomputes the full
  hash for all tokens on every rank and keeps only the owned tables'
  records (lffn_ctx_create_shard).

The combine is pipelined with the compute: tokens are processed in
``chunks``; chunk c's collective is issued asynchronously (NCCL runs it on its
own stream) while chunk c+1 is computed.  For reduce-scatter, chunk c is
assembled from the c-th sub-block of every rank's row block, so after all
chunks each rank holds one contiguous block of rows.

The per-rank compute is a ``LookupFFN`` shard on the rank's GPU.  Tests on a
CPU-only box exercise this exact plumbing over gloo by injecting the partial
function (tests/test_sharded.py); the product path always uses the device.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist

import ctypes as C

from . import _capi
from ._capi import check
from .lookup import HashTables, LookupConfig, LookupFFN, Projection

PartialFn = Callable[[torch.Tensor, torch.Tensor], None]
HashFn = Callable[[torch.Tensor], Tuple[torch.Tensor, torch.Tensor]]
GatherFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None]


def split_range(total: int, parts: int, index: int) -> Tuple[int, int]:
    """Even split of [0, total) into `parts`; the first total % parts get one more."""
    base, extra = divmod(total, parts)
    begin = index * base + min(index, extra)
    return begin, begin + base + (1 if index < extra else 0)


class ShardedLookupFFN:
    def __init__(self, cfg: LookupConfig, proj: Projection, tables: Optional[HashTables], *,
                 mode: str = "table", combine: str = "reduce_scatter", group=None,
                 device: Optional[int] = None, max_tokens: int = 65536,
                 table_dtype: str = "f32", chunks: int = 4, hash_mode: str = "token",
                 partial_fn: Optional[PartialFn] = None, hash_fn: Optional[HashFn] = None,
                 gather_fn: Optional[GatherFn] = None):
        if mode not in ("table", "token"):
            raise ValueError(f"unknown mode {mode}")
        if combine not in ("reduce_scatter", "all_reduce", "none"):
            raise ValueError(f"unknown combine {combine}")
        if hash_mode not in ("token", "replicated"):
            raise ValueError(f"unknown hash_mode {hash_mode}")
        if mode == "table" and cfg.neighbor_count != 1:
            # the record exchange and the partial gathers move one record per
            # (token, table); nc > 1 runs on one GPU (LookupFFN)
            raise ValueError("table sharding serves neighbor_count 1")
        self.cfg, self.mode, self.combine = cfg, mode, combine
        self.hash_mode = hash_mode if mode == "table" else "replicated"
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.chunks = max(1, int(chunks))
        if mode == "table":
            self.table_range = split_range(cfg.tables, self.world, self.rank)
        else:
            self.table_range = (0, cfg.tables)
        self.layer = None
        self.hasher = None
        if partial_fn is None and (self.hash_mode == "replicated" or gather_fn is None):
            dev = torch.cuda.current_device() if device is None else device
            self.layer = LookupFFN(cfg, proj, tables, device=dev, max_tokens=max_tokens,
                                   table_dtype=table_dtype, table_range=self.table_range)

            def partial_fn(x, out):
                self.layer.forward_device(x, out)

            def gather_fn(codes, coeff, out):
                self.layer.lookup_accumulate(codes, coeff, out)

            if self.hash_mode == "token" and hash_fn is None:
                # all tables, this rank's token block only (no tables needed)
                per = (max_tokens + self.world - 1) // self.world
                self.hasher = LookupFFN(cfg, proj, None, device=dev, max_tokens=max(1, per),
                                        table_range=(0, cfg.tables))

                def hash_fn(x):
                    return self.hasher.hash(x)

        self.partial_fn = partial_fn
        self.hash_fn = hash_fn
        self.gather_fn = gather_fn

    # ------------------------------------------------------------------
    def rows_owned(self, n: int) -> Tuple[int, int]:
        """Token rows this rank holds after the combine (table + reduce_scatter)."""
        if self.n_padded(n) != n:
            raise ValueError("rows_owned: n must be a multiple of world * chunks")
        return split_range(n, self.world, self.rank)

    def n_padded(self, n: int) -> int:
        q = self.world * self.chunks
        return ((n + q - 1) // q) * q

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """table mode: x holds ALL n tokens (identical on every rank);
        token mode: x holds this rank's own tokens."""
        if self.mode == "token":
            y = out if out is not None else x.new_empty((x.shape[0], self.cfg.d_out))
            self.partial_fn(x, y)
            return y
        n = x.shape[0]
        if self.hash_mode == "token":
            codes, coeff = self.exchange_records(x)
            if self.combine == "reduce_scatter":
                # records in chunk order (chunk c of every rank's row block
                # contiguous): one gather launch fills a chunk's buffer
                return self._table_reduce_scatter_records(x, out, codes, coeff)
            part = _RowGather(self.gather_fn, codes, coeff)
        else:
            part = _PartialFromX(self.partial_fn)
        if self.combine == "all_reduce":
            return self._table_all_reduce(x, out, part)
        if self.combine == "none":
            y = out if out is not None else x.new_empty((n, self.cfg.d_out))
            part(x, y, slice(0, n))
            return y
        return self._table_reduce_scatter(x, out, part)

    def exchange_records(self, x: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
        """hash_mode="token": hash this rank's token block (split_range of the
        n rows) for all tables, then one all-to-all so every rank holds the
        (code, coeff) records of ITS tables for all n tokens, token-major
        ([n, h_r] int32 codes / float32 coefficients, the layout
        lffn_lookup_accumulate reads)."""
        n, P, r = x.shape[0], self.world, self.rank
        h = self.cfg.tables
        t0, t1 = split_range(n, P, r)
        codes, coeff = self.hash_fn(x[t0:t1])                      # [m, h] each
        m = t1 - t0
        rec = torch.stack([codes.view(torch.int32), coeff.view(torch.int32)], dim=-1)  # [m, h, 2]
        tranges = [split_range(h, P, q) for q in range(P)]
        send = torch.cat([rec[:, a:b].reshape(-1) for a, b in tranges]) if m else rec.new_empty(0)
        kb, ke = self.table_range
        hl = ke - kb
        sizes_out = [(split_range(n, P, q)[1] - split_range(n, P, q)[0]) * hl * 2 for q in range(P)]
        recv = rec.new_empty(sum(sizes_out))
        dist.all_to_all_single(recv, send, output_split_sizes=sizes_out,
                               input_split_sizes=[m * (b - a) * 2 for a, b in tranges],
                               group=self.group)
        recv = recv.view(n, hl, 2)
        return (recv[..., 0].contiguous(), recv[..., 1].contiguous().view(torch.float32))

    def _table_all_reduce(self, x, out, part):
        n, d = x.shape[0], self.cfg.d_out
        y = out if out is not None else x.new_empty((n, d))
        works = []
        for c in range(self.chunks):
            r0, r1 = split_range(n, self.chunks, c)
            if r0 == r1:
                continue
            part(x[r0:r1], y[r0:r1], slice(r0, r1))
            works.append(dist.all_reduce(y[r0:r1], op=dist.ReduceOp.SUM, group=self.group,
                                         async_op=True))
        for w in works:
            w.wait()
        return y

    def _table_reduce_scatter(self, x, out, part):
        n, d = x.shape[0], self.cfg.d_out
        P, C = self.world, self.chunks
        if n % (P * C) != 0:
            raise ValueError(f"reduce_scatter forward: n={n} must be a multiple of "
                             f"world*chunks={P * C} (pad the batch)")
        per_rank = n // P
        sub = per_rank // C
        y = out if out is not None else x.new_empty((per_rank, d))
        bufs = [x.new_empty((P * sub, d)) for _ in range(min(C, 2))]
        works = []
        for c in range(C):
            buf = bufs[c % len(bufs)]
            if len(works) >= len(bufs):
                works[-len(bufs)].wait()  # buffer reuse after its collective
            for r in range(P):
                rows = slice(r * per_rank + c * sub, r * per_rank + (c + 1) * sub)
                part(x[rows], buf[r * sub:(r + 1) * sub], rows)
            works.append(dist.reduce_scatter_tensor(y[c * sub:(c + 1) * sub], buf,
                                                    op=dist.ReduceOp.SUM, group=self.group,
                                                    async_op=True))
        for w in works:
            w.wait()
        return y

    def _table_reduce_scatter_records(self, x, out, codes, coeff):
        """Reduce-scatter from exchanged records: the records are permuted
        once so that chunk c of every rank's token block is one contiguous
        range, and each chunk is ONE gather launch into the staging buffer
        of its collective (instead of P launches of n / (P C) tokens)."""
        n, d = x.shape[0], self.cfg.d_out
        P, C = self.world, self.chunks
        if n % (P * C) != 0:
            raise ValueError(f"reduce_scatter forward: n={n} must be a multiple of "
                             f"world*chunks={P * C} (pad the batch)")
        per_rank = n // P
        sub = per_rank // C
        hl = codes.shape[1]
        pc = codes.view(P, C, sub, hl).transpose(0, 1).reshape(n, hl)
        pw = coeff.view(P, C, sub, hl).transpose(0, 1).reshape(n, hl)
        y = out if out is not None else x.new_empty((per_rank, d))
        bufs = [x.new_empty((P * sub, d)) for _ in range(min(C, 2))]
        works = []
        for c in range(C):
            buf = bufs[c % len(bufs)]
            if len(works) >= len(bufs):
                works[-len(bufs)].wait()  # buffer reuse after its collective
            rows = slice(c * P * sub, (c + 1) * P * sub)
            self.gather_fn(pc[rows], pw[rows], buf)
            works.append(dist.reduce_scatter_tensor(y[c * sub:(c + 1) * sub], buf,
                                                    op=dist.ReduceOp.SUM, group=self.group,
                                                    async_op=True))
        for w in works:
            w.wait()
        return y

    def close(self):
        if self.layer is not None:
            self.layer.close()
        if self.hasher is not None:
            self.hasher.close()


class _PartialFromX:
    """part(x_rows, out, rows) for hash_mode="replicated": the full forward of
    the rows over the rank's tables."""

    def __init__(self, fn):
        self.fn = fn

    def __call__(self, xr, out, rows=None):
        self.fn(xr, out)


class _RowGather:
    """part(x_rows, out, rows) for hash_mode="token": the gather of the rows'
    exchanged records over the rank's tables."""

    def __init__(self, fn, codes, coeff):
        self.fn, self.codes, self.coeff = fn, codes, coeff

    def __call__(self, xr, out, rows):
        self.fn(self.codes[rows], self.coeff[rows], out)


class NativeTableShard:
    """One rank of the table-sharded forward through the C-ABI lffn_group
    (include/lffn_gpu.h): the group owns its NCCL communicator, the rank's
    table shard and the token-block hash context; lffn_forward_sharded does
    hash -> record exchange -> chunked gather + NCCL combine with no torch on
    the data path.  A C++ caller of the reference uses the same four calls
    (INTEGRATION.md).  ``nccl_id``: 128 bytes from ``unique_id()`` on rank 0,
    shared by any means (here: torch.distributed.broadcast_object_list)."""

    COMBINES = {"reduce_scatter": _capi.LFFN_COMBINE_REDUCE_SCATTER,
                "all_reduce": _capi.LFFN_COMBINE_ALL_REDUCE,
                "none": _capi.LFFN_COMBINE_NONE}

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_capi.lib().lffn_nccl_unique_id(buf, 128))
        return buf.raw

    def __init__(self, cfg: LookupConfig, proj: Projection, tables, *, rank: int, world: int,
                 nccl_id: bytes, device: int = 0, max_tokens: int = 65536,
                 table_dtype: str = "f32", chunks: int = 4):
        L = _capi.lib()
        g = C.c_void_p()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        check(L.lffn_group_create(C.byref(g), device, max_tokens, C.byref(cfg._c()),
                                  C.byref(proj._c()), idbuf, rank, world))
        self._g = g
        self.cfg, self.rank, self.world = cfg, rank, world
        self.table_range = split_range(cfg.tables, world, rank)
        check(L.lffn_group_set_chunks(g, int(chunks)))
        self.chunks = int(chunks)
        self.layer = LookupFFN._view(L.lffn_group_shard(g), cfg, proj, self.table_range,
                                     device=device, max_tokens=max_tokens,
                                     table_dtype=table_dtype)
        if tables is not None:
            self.layer.upload_tables(tables)

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                combine: str = "reduce_scatter", stream=None) -> torch.Tensor:
        n = x.shape[0]
        rows = n // self.world if combine == "reduce_scatter" else n
        y = out if out is not None else x.new_empty((rows, self.cfg.d_out))
        st = torch.cuda.current_stream().cuda_stream if stream is None else int(stream)
        check(_capi.lib().lffn_forward_sharded(self._g, x.data_ptr(), n, y.data_ptr(),
                                               self.COMBINES[combine], st))
        return y

    def close(self) -> None:
        if getattr(self, "_g", None):
            self.layer.close()
            _capi.lib().lffn_group_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
