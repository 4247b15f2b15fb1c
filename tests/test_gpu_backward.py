"""Backward on the device vs the oracle.

Reference: lookup_backward (lookup.cpp:292-347) and Projection::backward
(projection.cpp:279-386); the oracle restates both and is pinned bit-exact to
the reference (tests/test_oracle_pin.py).  Bars: the projection backward is
bit-identical for the same float64 grad_z (signflip: the transposed network in
the reference's stage order; dense: exact float64 GEMMs in the reference's
summation order; acdc / bh: stagewise, the parameter gradients summed over the
tokens in order); the full backward, whose table-row dots and table-gradient
sums run in float32 on float32 tables, within l2_rel <= 1e-5 and
max_abs/max <= 1e-5 of the float64 oracle fed the same stored tables.
"""
import numpy as np
import pytest

from gpu_helpers import assert_close, stored_tables, to_oracle
from paper_2403_07221_b200 import (HashTables, LookupConfig, LookupFFN, LookupVariant,
                                   NumericError, Projection, ProjectionSpec, ProjKind, SizeError,
                                   fill_gaussian, gaussian_matrix)
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _setup(d_in, d_out, h, tau, kind, n, variant=LookupVariant.softmax, nc=1, seed=0, std=0.02):
    cfg = LookupConfig(d_in=d_in, d_out=d_out, tables=h, code_bits=tau, variant=variant,
                       neighbor_count=nc)
    kw = {ProjKind.acdc: {"depth": 2}, ProjKind.bh: {"stages": 2, "block": 16}}.get(kind, {})
    proj = Projection.init(ProjectionSpec(d_in, h * tau, kind, **kw), seed + 1)
    T = HashTables(h, tau, d_out, fill_gaussian(seed + 2, h * (1 << tau) * d_out, std))
    x = gaussian_matrix(n, d_in, seed).astype(np.float32)
    gy = gaussian_matrix(n, d_out, seed + 9).astype(np.float32)
    return cfg, proj, T, x, gy


PROJ_CASES = [
    (ProjKind.signflip, 64, 32, 50), (ProjKind.signflip, 768, 2048, 64),
    (ProjKind.signflip, 50, 120, 33), (ProjKind.signflip, 3, 8, 5),
    (ProjKind.signflip, 1024, 1280, 16), (ProjKind.signflip, 4096, 4096, 4),
    (ProjKind.dense, 64, 32, 50), (ProjKind.dense, 100, 96, 70), (ProjKind.dense, 7, 9, 3),
    (ProjKind.acdc, 64, 32, 40), (ProjKind.acdc, 50, 120, 17), (ProjKind.acdc, 768, 2048, 16),
    (ProjKind.bh, 64, 64, 40), (ProjKind.bh, 50, 120, 17), (ProjKind.bh, 768, 2048, 16),
]

PROJ_KW = {ProjKind.acdc: {"depth": 2}, ProjKind.bh: {"stages": 3, "block": 16}}


@pytest.mark.parametrize("case", PROJ_CASES, ids=lambda c: f"{c[0].name}-{c[1]}x{c[2]}-n{c[3]}")
def test_proj_backward_bit_exact(oracle, case):
    import torch

    kind, d_in, d_out, n = case
    tau = 4 if d_out % 4 == 0 else 1
    h = d_out // tau
    cfg = LookupConfig(d_in=d_in, d_out=8, tables=h, code_bits=tau)
    proj = Projection.init(ProjectionSpec(d_in, d_out, kind, **PROJ_KW.get(kind, {})), 3)
    layer = LookupFFN(cfg, proj, None, max_tokens=n)
    x = gaussian_matrix(n, d_in, 4).astype(np.float32)
    gz = gaussian_matrix(n, d_out, 5)
    gx, gp = layer.proj_backward(torch.from_numpy(x).cuda(), torch.from_numpy(gz).cuda())
    layer.sync()
    c, s = to_oracle(cfg, proj)
    gx_ref, gp_ref = oracle.proj_backward(s, proj.blob, x.astype(np.float64), gz)
    assert np.array_equal(gx.cpu().numpy().view(np.uint64), gx_ref.view(np.uint64))
    if kind != ProjKind.signflip:
        assert np.array_equal(gp.cpu().numpy().reshape(-1).view(np.uint64), gp_ref.view(np.uint64))


BWD_CASES = [
    # d_in, d_out, h, tau, kind, n, variant, nc
    (64, 64, 8, 4, ProjKind.signflip, 256, LookupVariant.scaled, 1),
    (64, 64, 8, 4, ProjKind.dense, 256, LookupVariant.softmax, 1),
    (64, 48, 8, 4, ProjKind.dense, 200, LookupVariant.scaled, 1),
    (50, 30, 12, 10, ProjKind.signflip, 33, LookupVariant.scaled, 1),
    (64, 64, 8, 4, ProjKind.signflip, 100, LookupVariant.softmax, 3),
    (64, 32, 6, 4, ProjKind.dense, 80, LookupVariant.scaled, 5),
    (768, 768, 256, 8, ProjKind.signflip, 64, LookupVariant.scaled, 1),   # c2 shape
    (32, 16, 8, 1, ProjKind.dense, 50, LookupVariant.sigmoid_tau1, 2),    # tau = 1 constructions
    (32, 16, 8, 1, ProjKind.dense, 50, LookupVariant.gelu_tau1, 2),
    (32, 8, 3, 11, ProjKind.dense, 300, LookupVariant.scaled, 1),  # 2^tau > 1024
    (64, 64, 8, 4, ProjKind.acdc, 100, LookupVariant.scaled, 1),
    (64, 64, 8, 4, ProjKind.bh, 100, LookupVariant.softmax, 2),
]


def _oracle_grads(oracle, cfg, proj, T, x, gy, table_dtype="f32"):
    c, s = to_oracle(cfg, proj)
    return oracle.lookup_backward(c, s, proj.blob, stored_tables(T.data, table_dtype),
                                  x.astype(np.float64), gy.astype(np.float64))


@pytest.mark.parametrize("case", BWD_CASES,
                         ids=lambda c: f"{c[4].name}-d{c[0]}-h{c[2]}-t{c[3]}-v{int(c[6])}-nc{c[7]}")
def test_backward_matches_oracle(oracle, case):
    import torch

    d_in, d_out, h, tau, kind, n, variant, nc = case
    cfg, proj, T, x, gy = _setup(d_in, d_out, h, tau, kind, n, variant, nc)
    layer = LookupFFN(cfg, proj, T, max_tokens=n)
    g = layer.backward(torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda())
    layer.sync()
    ref = _oracle_grads(oracle, cfg, proj, T, x, gy)
    gt = g["grad_tables"].cpu().numpy().reshape(-1)
    assert_close(gt, ref["grad_tables"], TOL, "grad_tables")
    gx = g["grad_x"].cpu().numpy()
    if np.max(np.abs(ref["grad_x"])) > 0:
        assert_close(gx, ref["grad_x"], TOL, "grad_x")
    else:
        assert np.max(np.abs(gx)) == 0.0
    if kind != ProjKind.signflip:
        assert_close(g["grad_proj"].cpu().numpy().reshape(-1), ref["grad_proj"], TOL, "grad_proj")


def test_backward_bf16_tables(oracle):
    import torch

    cfg, proj, T, x, gy = _setup(64, 64, 8, 4, ProjKind.dense, 128, LookupVariant.scaled)
    layer = LookupFFN(cfg, proj, T, max_tokens=128, table_dtype="bf16")
    g = layer.backward(torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda())
    layer.sync()
    ref = _oracle_grads(oracle, cfg, proj, T, x, gy, "bf16")
    assert_close(g["grad_tables"].cpu().numpy().reshape(-1), ref["grad_tables"], TOL, "bf16 grad_tables")
    assert_close(g["grad_x"].cpu().numpy(), ref["grad_x"], TOL, "bf16 grad_x")


def test_backward_table_shards_sum_to_full(oracle):
    import torch

    cfg, proj, T, x, gy = _setup(64, 64, 12, 4, ProjKind.dense, 90, LookupVariant.scaled)
    xd, gyd = torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda()
    full = LookupFFN(cfg, proj, T, max_tokens=90)
    gf = full.backward(xd, gyd)
    parts = []
    for kb, ke in [(0, 5), (5, 12)]:
        sh = LookupFFN(cfg, proj, T, max_tokens=90, table_range=(kb, ke))
        parts.append((kb, ke, sh.backward(xd, gyd)))
        sh.sync()
    full.sync()
    gx = sum(p[2]["grad_x"] for p in parts)
    assert_close(gx.cpu().numpy(), gf["grad_x"].cpu().numpy(), 1e-12, "shard grad_x")
    for kb, ke, g in parts:
        assert np.array_equal(g["grad_tables"].cpu().numpy(), gf["grad_tables"][kb:ke].cpu().numpy())


def test_backward_non_finite_grad_y_raises():
    import torch

    cfg, proj, T, x, gy = _setup(64, 64, 8, 4, ProjKind.signflip, 16)
    gy[3, 5] = np.nan
    layer = LookupFFN(cfg, proj, T, max_tokens=16)
    layer.backward(torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda())
    with pytest.raises(NumericError, match="lookup backward input"):
        layer.sync()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c2_bf16"])
def test_two_pass_kb1_bit_identical_to_one_pass(name):
    """The default backward (gdot pass with the transposed float64 butterfly,
    per-(token, table) gz pass, four-row table-gradient walk) against the
    single-pass KB1 (option bwd_one_pass): grad_x and grad_T bit-identical."""
    import torch

    w = WORKLOADS[name]
    cfg, proj, T = make_params(w, ProjKind.signflip)
    n = 2048
    layer = LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype)
    xd = torch.from_numpy(make_x(w, n)).cuda()
    g = torch.Generator().manual_seed(3)
    gy = torch.randn((n, cfg.d_out), generator=g).cuda()
    outs = []
    for one in (1, 0):
        layer.set_option("bwd_one_pass", one)
        o = layer.backward(xd, gy)
        layer.sync()
        outs.append((o["grad_x"].cpu().numpy(), o["grad_tables"].cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
