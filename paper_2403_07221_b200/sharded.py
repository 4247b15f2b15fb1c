"""Multi-GPU LookupFFN forward: one process per GPU over torch.distributed.

No reference counterpart (the reference is single-process);
the partitioning follows SURVEY.md 8e / BASELINE.json north_star:

* ``mode="token"``  tables replicated, rank r runs its own token block; no
  collective on the data path (optionally an all-gather of y).
* ``mode="table"``  rank r owns the table slice [r*h/P, (r+1)*h/P) (the hash
  is recomputed per rank -- it is cheap -- but codes/coefficients are emitted
  only for the owned tables, lffn_ctx_create_shard), produces the fp32
  PARTIAL y over its tables for all tokens, and the partials are combined by
  ``combine="reduce_scatter"`` (rank r keeps token rows [r*n/P, (r+1)*n/P),
  BASELINE c3) or ``combine="all_reduce"`` (every rank keeps all of y, c4).

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

from .lookup import HashTables, LookupConfig, LookupFFN, Projection

PartialFn = Callable[[torch.Tensor, torch.Tensor], None]


def split_range(total: int, parts: int, index: int) -> Tuple[int, int]:
    """Even split of [0, total) into `parts`; the first total % parts get one more."""
    base, extra = divmod(total, parts)
    begin = index * base + min(index, extra)
    return begin, begin + base + (1 if index < extra else 0)


class ShardedLookupFFN:
    def __init__(self, cfg: LookupConfig, proj: Projection, tables: Optional[HashTables], *,
                 mode: str = "table", combine: str = "reduce_scatter", group=None,
                 device: Optional[int] = None, max_tokens: int = 65536,
                 table_dtype: str = "f32", chunks: int = 4,
                 partial_fn: Optional[PartialFn] = None):
        if mode not in ("table", "token"):
            raise ValueError(f"unknown mode {mode}")
        if combine not in ("reduce_scatter", "all_reduce", "none"):
            raise ValueError(f"unknown combine {combine}")
        self.cfg, self.mode, self.combine = cfg, mode, combine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.chunks = max(1, int(chunks))
        if mode == "table":
            self.table_range = split_range(cfg.tables, self.world, self.rank)
        else:
            self.table_range = (0, cfg.tables)
        self.layer = None
        if partial_fn is None:
            dev = torch.cuda.current_device() if device is None else device
            self.layer = LookupFFN(cfg, proj, tables, device=dev, max_tokens=max_tokens,
                                   table_dtype=table_dtype, table_range=self.table_range)

            def partial_fn(x, out):
                self.layer.forward_device(x, out)

        self.partial_fn = partial_fn

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
        if self.combine == "all_reduce":
            return self._table_all_reduce(x, out)
        if self.combine == "none":
            y = out if out is not None else x.new_empty((n, self.cfg.d_out))
            self.partial_fn(x, y)
            return y
        return self._table_reduce_scatter(x, out)

    def _table_all_reduce(self, x, out):
        n, d = x.shape[0], self.cfg.d_out
        y = out if out is not None else x.new_empty((n, d))
        works = []
        for c in range(self.chunks):
            r0, r1 = split_range(n, self.chunks, c)
            if r0 == r1:
                continue
            self.partial_fn(x[r0:r1], y[r0:r1])
            works.append(dist.all_reduce(y[r0:r1], op=dist.ReduceOp.SUM, group=self.group,
                                         async_op=True))
        for w in works:
            w.wait()
        return y

    def _table_reduce_scatter(self, x, out):
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
                self.partial_fn(x[rows], buf[r * sub:(r + 1) * sub])
            works.append(dist.reduce_scatter_tensor(y[c * sub:(c + 1) * sub], buf,
                                                    op=dist.ReduceOp.SUM, group=self.group,
                                                    async_op=True))
        for w in works:
            w.wait()
        return y

    def close(self):
        if self.layer is not None:
            self.layer.close()
