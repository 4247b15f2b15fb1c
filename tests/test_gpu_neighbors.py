"""Multi-neighbour forward (neighbor_count > 1) on the device vs the oracle.

Reference: neighbor_codes (lookup.cpp:118-165), log_denominator (:102-109),
code_dot (:111-116), forward_impl records (:231-262).  Codes -- including
their ORDER, which follows the libstdc++ heap for tied costs -- are bit-exact;
coefficients exp(dot - logden) (times dot for the scaled variants) within
float32 rounding; y at the fp32 bar.  The reference tests this path with the
full-neighbour codebook (test_lookup.cpp:251-272) and the tau = 1
sigmoid / GELU constructions (:274-342); both appear below.
"""
import numpy as np
import pytest

from gpu_helpers import assert_close, device_forward, device_hash, stored_tables, to_oracle
from paper_2403_07221_b200 import (HashTables, LookupConfig, LookupFFN, LookupVariant, Projection,
                                   ProjectionSpec, ProjKind, SizeError, fill_gaussian,
                                   gaussian_matrix)

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


def _setup(d_in, d_out, h, tau, nc, kind=ProjKind.signflip, n=64,
           variant=LookupVariant.softmax, seed=0, **spec_kw):
    cfg = LookupConfig(d_in=d_in, d_out=d_out, tables=h, code_bits=tau, variant=variant,
                       neighbor_count=nc)
    spec = ProjectionSpec(d_in, h * tau, kind, **spec_kw)
    proj = Projection.init(spec, seed + 1)
    T = HashTables(h, tau, d_out, fill_gaussian(seed + 2, h * (1 << tau) * d_out, 0.02))
    x = gaussian_matrix(n, d_in, seed).astype(np.float32)
    return cfg, proj, T, x


def _check(oracle, cfg, proj, T, x, table_range=None):
    layer = LookupFFN(cfg, proj, T, max_tokens=x.shape[0], table_range=table_range)
    codes, coeff, z = device_hash(layer, x)
    c, s = to_oracle(cfg, proj)
    y_ref, cache = oracle.lookup_forward(c, s, proj.blob, stored_tables(T.data, "f32"),
                                         x.astype(np.float64), True)
    kb, ke = table_range or (0, cfg.tables)
    assert np.array_equal(z.view(np.uint64), cache["z"].view(np.uint64))
    assert np.array_equal(codes, cache["codes"][:, kb:ke])
    expect = cache["weights"] * cache["dots"] if cfg.scaled_numerator() else cache["weights"]
    np.testing.assert_allclose(coeff, expect[:, kb:ke].astype(np.float32), rtol=1e-6,
                               atol=1e-30)
    y = device_forward(layer, x)
    if table_range is None:
        assert_close(y, y_ref, FP32_TOL, "nc forward")
    layer.close()
    return y


CASES = [
    # d_in, d_out, h, tau, nc, kind, n, variant
    (64, 64, 8, 4, 2, ProjKind.signflip, 256, LookupVariant.softmax),
    (64, 64, 8, 4, 16, ProjKind.signflip, 64, LookupVariant.softmax),     # full codebook
    (64, 64, 8, 4, 5, ProjKind.acdc, 100, LookupVariant.scaled),
    (50, 30, 12, 10, 7, ProjKind.signflip, 33, LookupVariant.softmax),    # pad + truncate
    (768, 768, 256, 8, 3, ProjKind.signflip, 64, LookupVariant.softmax),  # c2 shape
    (64, 32, 6, 8, 64, ProjKind.signflip, 40, LookupVariant.scaled),
    (40, 24, 5, 8, 256, ProjKind.signflip, 16, LookupVariant.softmax),    # nc = 2^tau = 256
    (64, 64, 8, 4, 3, ProjKind.dense, 64, LookupVariant.softmax),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[5].name}-d{c[0]}-h{c[2]}-t{c[3]}-nc{c[4]}")
def test_neighbors_match_oracle(oracle, case):
    d_in, d_out, h, tau, nc, kind, n, variant = case
    cfg, proj, T, x = _setup(d_in, d_out, h, tau, nc, kind, n, variant)
    _check(oracle, cfg, proj, T, x)


def test_neighbors_bh(oracle):
    cfg, proj, T, x = _setup(64, 64, 8, 4, 3, ProjKind.bh, 48, stages=2, block=8)
    _check(oracle, cfg, proj, T, x)


def test_neighbors_tied_costs_follow_the_heap(oracle):
    """All |z_j| equal (dense W of ones): every flip cost ties, so the
    neighbour order is decided by the heap layout alone."""
    d_in, h, tau, nc = 8, 4, 6, 20
    cfg = LookupConfig(d_in=d_in, d_out=16, tables=h, code_bits=tau, neighbor_count=nc)
    spec = ProjectionSpec(d_in, h * tau, ProjKind.dense)
    blob = np.ones(d_in * h * tau)
    blob[::3] = -1.0  # mixed signs, equal magnitudes per output
    proj = Projection.from_blob(spec, blob)
    T = HashTables(h, tau, 16, fill_gaussian(5, h * (1 << tau) * 16, 0.02))
    x = np.zeros((12, d_in), np.float32)
    x[:, 0] = np.linspace(-2, 2, 12)  # z_j = +-x_0: |z| tied within each row
    _check(oracle, cfg, proj, T, x)


def test_neighbors_tau1_sigmoid_and_gelu(oracle):
    """tau = 1 with both codes (nc = 2): the reference's sigmoid / GELU
    constructions (test_lookup.cpp:274-342)."""
    for variant in (LookupVariant.sigmoid_tau1, LookupVariant.gelu_tau1):
        cfg, proj, T, x = _setup(32, 16, 8, 1, 2, ProjKind.signflip, 50, variant)
        _check(oracle, cfg, proj, T, x)


def test_neighbors_table_shard(oracle):
    cfg, proj, T, x = _setup(64, 64, 12, 4, 4, ProjKind.signflip, 40)
    _check(oracle, cfg, proj, T, x, table_range=(3, 10))


def test_neighbors_host_path(oracle):
    cfg, proj, T, x = _setup(64, 64, 8, 4, 3, ProjKind.signflip, 3000)
    layer = LookupFFN(cfg, proj, T, max_tokens=3000)
    y = layer.forward(x)
    c, s = to_oracle(cfg, proj)
    y_ref = oracle.lookup_forward(c, s, proj.blob, stored_tables(T.data, "f32"), x.astype(np.float64))
    assert_close(y, y_ref, FP32_TOL, "nc host forward")


def test_neighbor_count_above_device_limit_is_a_size_error():
    cfg = LookupConfig(d_in=16, d_out=8, tables=2, code_bits=10, neighbor_count=300)
    proj = Projection.init(ProjectionSpec(16, 20, ProjKind.signflip), 1)
    with pytest.raises(SizeError):
        LookupFFN(cfg, proj, None, max_tokens=4)
