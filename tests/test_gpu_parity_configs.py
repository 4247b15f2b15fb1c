"""Parity at the BASELINE configs' own shapes and batch sizes (runs on a B200).

Every gather instance a bench line times is compared with the oracle here:

* c4 (d = 4096, h = 512, bf16): n = 2400 takes the persistent part-major
  kernel with four warps per token (gather_row_persistent_kernel<bf16, 4, 4,
  2, true>); n = 64 takes gather_split_kernel with parts = 4 and S = 8;
* c3 at its full 65,536 tokens (several rounds of resident warps, reversed
  odd rounds for bf16 stacks);
* c5 at its full 4,096 skewed tokens;
* c4 through the table-sharded all-reduce path on a world-1 NCCL group.

The hash bar is the north star's: codes bit-exact wherever every coordinate
of the table has |z_ref| > 1e-5 (a code bit may only differ where the
reference's own projection is within 1e-5 of zero).  y is compared with the
oracle's float64 gather (/root/reference/proj/src/lookup.cpp:223-268) on the
device's records and the stored (rounded) tables at the fp32 bar, and with
the float64 tables at the bf16 bar.
"""
import numpy as np
import pytest

from gpu_helpers import assert_close, device_forward, device_hash, stored_tables, to_oracle
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2
Z_BAR = 1e-5


def assert_codes_match(codes, z_ref, h, tau, what=""):
    """Bit-exact codes except where the reference's |z| <= 1e-5 (north star)."""
    from oracle import Oracle

    codes_ref, _ = Oracle().compute_codes(z_ref, h, tau)
    diff = codes != codes_ref
    if diff.any():
        small = (np.abs(z_ref[:, : h * tau]).reshape(-1, h, tau) <= Z_BAR).any(axis=2)
        bad = diff & ~small
        assert not bad.any(), f"{what}: {int(bad.sum())} codes differ where every |z| > {Z_BAR}"
    return codes_ref


_PARAMS = {}


def params(name):
    if name not in _PARAMS:
        _PARAMS.clear()  # c4's float64 stack is 4.3 GB: keep one config at a time
        w = WORKLOADS[name]
        _PARAMS[name] = (w,) + make_params(w)
    return _PARAMS[name]


def _check_config(oracle, name, n, seed=0):
    w, cfg, proj, T = params(name)
    x = make_x(w, n, seed=seed)
    layer = LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype)
    codes, coeff, _ = device_hash(layer, x, want_z=False)
    _, s = to_oracle(cfg, proj)
    z_ref = oracle.proj_forward(s, proj.blob, x.astype(np.float64))
    assert_codes_match(codes, z_ref, w.h, w.tau, name)
    y = device_forward(layer, x)
    rows = 1 << w.tau
    Ts = stored_tables(T.data, w.table_dtype)
    y_ref = oracle.gather(Ts, w.h, rows, w.d, codes, coeff.astype(np.float64))
    assert_close(y, y_ref, FP32_TOL, f"{name} n={n} vs oracle gather on stored tables")
    if w.table_dtype == "bf16":
        del Ts
        y_full = oracle.gather(T.data, w.h, rows, w.d, codes, coeff.astype(np.float64))
        assert_close(y, y_full, BF16_TOL, f"{name} n={n} vs float64 tables")
    layer.close()
    return y


@pytest.mark.parametrize("n", [2400, 64, 1], ids=lambda n: f"n{n}")
def test_c4_gather_instances(oracle, n):
    """c4: the part-major persistent walk (n = 2400 > 148 x 16 resident warp
    slots, four warps per token) and the split walk with four column parts
    (n = 64, S = 8), plus a single token."""
    _check_config(oracle, "c4", n)


def test_c3_full_size(oracle):
    """c3 at its full 65,536 tokens: 27 rounds of resident warps."""
    _check_config(oracle, "c3", WORKLOADS["c3"].n)


def test_c5_full_size_skewed(oracle):
    """c5: 4,096 skewed tokens (hot rows), and the small batches 1 / 8 / 64."""
    _check_config(oracle, "c5", WORKLOADS["c5"].n)
    for n in (1, 8, 64):
        _check_config(oracle, "c5", n)


def test_c4_table_sharded_all_reduce_world1(oracle):
    """c4 through ShardedLookupFFN(combine = "all_reduce") on a world-1 NCCL
    group (the north star's c4 multi-GPU path): y equals the plain forward
    up to fp32 reassociation and the oracle within the bar."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2403_07221_b200.sharded import ShardedLookupFFN

    w, cfg, proj, T = params("c4")
    n = 512
    x = make_x(w, n)
    plain = _check_config(oracle, "c4", n)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sh = ShardedLookupFFN(cfg, proj, T, mode="table", combine="all_reduce", device=0,
                              max_tokens=n, chunks=4, table_dtype="bf16")
        y = sh.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        torch.cuda.synchronize()
        sh.close()
        # the chunks (128 tokens) take the split gather, the plain forward
        # (512) the one-warp walk: fp32 reassociation only
        assert np.abs(y - plain).max() <= 1e-6 * np.abs(plain).max()
    finally:
        dist.destroy_process_group()
