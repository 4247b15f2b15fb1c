"""Multi-GPU plumbing (paper_2403_07221_b200/sharded.py) over gloo, world_size 2,
on CPU.  The per-rank partial sum is injected from the oracle (the product
computes it on the GPU with a table-shard context); the partitioning, the
chunked collectives and the row ownership under test are the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_07221_b200.sharded import split_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_split_range_covers_exactly():
    for total in (0, 1, 7, 256, 257, 1000):
        for parts in (1, 2, 3, 8):
            rs = [split_range(total, parts, i) for i in range(parts)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, combine, chunks, result_q, hash_mode="replicated", h=10, n=24):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Cfg, Oracle, Spec
        from paper_2403_07221_b200 import LookupConfig, Projection, ProjectionSpec
        from paper_2403_07221_b200.sharded import ShardedLookupFFN

        orc = Oracle()
        d, tau = 32, 4
        c = Cfg(d, d, h, tau)
        s = Spec(d, h * tau, 3)
        blob = orc.proj_init(s, 1)
        T = orc.gaussian(2, h * 16 * d, 0.02)
        x = orc.gaussian(0, n * d).reshape(n, d).astype(np.float32)
        y_full = orc.lookup_forward(c, s, blob, T, x.astype(np.float64))

        cfg = LookupConfig(d_in=d, d_out=d, tables=h, code_bits=tau)
        proj = Projection.from_blob(ProjectionSpec.signflip(d, h * tau), blob)
        holder = {}

        def partial_fn(xr, out):
            kb, ke = holder["m"].table_range
            _, cache = orc.lookup_forward(c, s, blob, T, xr.numpy().astype(np.float64), True)
            codes = np.ascontiguousarray(cache["codes"][:, kb:ke, 0])
            w = np.ascontiguousarray(cache["weights"][:, kb:ke, 0])
            part = orc.gather(T.reshape(h, -1)[kb:ke].ravel(), ke - kb, 16, d, codes, w)
            out.copy_(torch.from_numpy(part.astype(np.float32)))

        hashed = []

        def hash_fn(xr):
            # all tables' records of the rank's own token block
            hashed.append(xr.shape[0])
            _, cache = orc.lookup_forward(c, s, blob, T, xr.numpy().astype(np.float64), True)
            codes = np.ascontiguousarray(cache["codes"][:, :, 0]).astype(np.int32)
            w = np.ascontiguousarray(cache["weights"][:, :, 0]).astype(np.float32)
            return torch.from_numpy(codes), torch.from_numpy(w)

        def gather_fn(codes, w, out):
            kb, ke = holder["m"].table_range
            part = orc.gather(T.reshape(h, -1)[kb:ke].ravel(), ke - kb, 16, d,
                              codes.numpy().astype(np.uint32), w.numpy().astype(np.float64))
            out.copy_(torch.from_numpy(part.astype(np.float32)))

        if hash_mode == "token":
            m = ShardedLookupFFN(cfg, proj, None, mode=mode, combine=combine, chunks=chunks,
                                 hash_mode="token", hash_fn=hash_fn, gather_fn=gather_fn)
        else:
            m = ShardedLookupFFN(cfg, proj, None, mode=mode, combine=combine, chunks=chunks,
                                 hash_mode="replicated", partial_fn=partial_fn)
        holder["m"] = m
        if mode == "token":
            r0, r1 = split_range(n, world, rank)
            y = m.forward(torch.from_numpy(x[r0:r1]))
            expect = y_full[r0:r1]
        elif combine == "all_reduce":
            y = m.forward(torch.from_numpy(x))
            expect = y_full
        elif combine == "none":
            # the rank's partial sum over its tables, all tokens
            y = m.forward(torch.from_numpy(x))
            kb, ke = m.table_range
            _, cache = orc.lookup_forward(c, s, blob, T, x.astype(np.float64), True)
            expect = orc.gather(T.reshape(h, -1)[kb:ke].ravel(), ke - kb, 16, d,
                                np.ascontiguousarray(cache["codes"][:, kb:ke, 0]),
                                np.ascontiguousarray(cache["weights"][:, kb:ke, 0]))
        else:
            y = m.forward(torch.from_numpy(x))
            r0, r1 = m.rows_owned(n)
            expect = y_full[r0:r1]
        err = float(np.max(np.abs(y.numpy() - expect)) / np.max(np.abs(expect)))
        if hash_mode == "token":
            # each rank hashed only its own token block, once
            assert hashed == [split_range(n, world, rank)[1] - split_range(n, world, rank)[0]]
        result_q.put((rank, m.table_range, tuple(y.shape), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,combine,chunks,hash_mode,h,n", [
    ("table", "reduce_scatter", 1, "replicated", 10, 24),
    ("table", "reduce_scatter", 3, "replicated", 10, 24),
    ("table", "all_reduce", 2, "replicated", 10, 24),
    ("token", "none", 1, "replicated", 10, 24),
    ("table", "reduce_scatter", 1, "token", 10, 24),
    ("table", "reduce_scatter", 3, "token", 10, 24),
    ("table", "all_reduce", 2, "token", 10, 24),
    ("table", "none", 1, "token", 10, 24),
    # uneven table split (6 / 5) and uneven token blocks (13 / 12) for the
    # all-to-all's split sizes
    ("table", "all_reduce", 1, "token", 11, 25),
    ("table", "none", 1, "token", 11, 25)])
def test_sharded_two_ranks(mode, combine, chunks, hash_mode, h, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, combine, chunks, q, hash_mode,
                                               h, n))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [r[1] for r in results]
    if mode == "table":
        assert ranges == [(0, (h + 1) // 2), ((h + 1) // 2, h)]
    for rank, _, shape, err in results:
        assert err < 2e-6, (rank, err)
        if mode == "table" and combine == "reduce_scatter":
            assert shape == (n // 2, 32)


@pytest.mark.parametrize("combine,n", [("all_reduce", 25), ("none", 25), ("reduce_scatter", 24)])
def test_sharded_three_ranks_token_hash(combine, n):
    """World 3 over gloo: h = 11 tables split 4 / 4 / 3 and n = 25 tokens split
    9 / 8 / 8 -- every all-to-all split size differs from its neighbours
    (reduce-scatter needs n divisible by the world: 24)."""
    world, h = 3, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "table", combine, 1, q, "token", h, n))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in results] == [(0, 4), (4, 8), (8, 11)]
    for rank, _, shape, err in results:
        assert err < 2e-6, (rank, err)
