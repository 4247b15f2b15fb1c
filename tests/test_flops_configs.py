"""Cost model (flops.cpp restated in paper_2403_07221_b200/flops.py) and the
BASELINE workloads (configs.py) -- host logic, no GPU."""
import math

import numpy as np
import pytest

from paper_2403_07221_b200 import LookupConfig, ProjectionSpec, ProjKind
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_params, make_x, spec_of
from paper_2403_07221_b200.flops import (gathered_bytes_per_token, lookup_flops, projection_cost,
                                         unique_table_bytes, vanilla_flops)


def within(v, t, rel):
    return abs(v - t) <= rel * abs(t)


def cfg(d, d_out, h, tau):
    return LookupConfig(d_in=d, d_out=d_out, tables=h, code_bits=tau)


def proj(c, kind, m=4, b=0):
    return ProjectionSpec(c.d_in, c.code_width(), kind, stages=m, block=b)


def test_published_totals():
    """test_flops.cpp:38-96 -- the paper's MFLOP/token tables."""
    assert math.isclose(vanilla_flops(512, 2048, 512).total_mflop(), 4.194304, rel_tol=1e-12)
    assert round(vanilla_flops(768, 3072, 768).total_mflop(), 2) == 9.44
    c = cfg(512, 512, 128, 8)
    r = lookup_flops(c, proj(c, ProjKind.dense))
    assert within(r.hash_mflop, 1.05, 0.02) and within(r.gather_mflop, 0.13, 0.02)
    for b, e in [(64, 0.56), (32, 0.30), (16, 0.17)]:
        assert within(lookup_flops(c, proj(c, ProjKind.bh, 4, b)).hash_mflop, e, 0.02)
    c = cfg(512, 512, 256, 8)
    assert within(lookup_flops(c, proj(c, ProjKind.bh, 4, 64)).total_mflop(), 1.38, 0.03)
    c = cfg(512, 512, 128, 8)
    assert within(lookup_flops(c, proj(c, ProjKind.bh, 4, 64)).total_mflop(), 0.69, 0.03)
    c = cfg(768, 768, 170, 9)
    assert within(lookup_flops(c, proj(c, ProjKind.bh, 4, 64)).total_mflop(), 1.39, 0.03)


def test_monotone_and_signflip_cost():
    c = cfg(512, 512, 128, 8)
    prev = 0.0
    for b in (8, 16, 32, 64, 128):
        f = projection_cost(proj(c, ProjKind.bh, 4, b))[0]
        assert f > prev
        prev = f
    D = 2048
    assert projection_cost(ProjectionSpec.signflip(768, 2048))[0] == 3 * D + 3 * D * 11


@pytest.mark.parametrize("kind", [ProjKind.signflip, ProjKind.dense, ProjKind.bh, ProjKind.acdc])
def test_matches_reference_cost_model(reference, kind):
    from oracle import Cfg, Spec

    for d, h, tau in [(768, 256, 8), (1024, 128, 10), (64, 8, 4)]:
        c = cfg(d, d, h, tau)
        p = proj(c, kind, 4, 64 if kind == ProjKind.bh else 0)
        if kind == ProjKind.acdc:
            p.depth = 2
        got = lookup_flops(c, p)
        ref = reference.lookup_flops(Cfg(d, d, h, tau), Spec(d, h * tau, int(kind), p.stages,
                                                              p.block, p.depth))
        assert np.allclose([got.hash_mflop, got.gather_mflop, got.other_mflop], ref, rtol=1e-15)


def test_byte_model():
    c = cfg(768, 768, 256, 8)
    assert gathered_bytes_per_token(c, 4) == 786432
    assert gathered_bytes_per_token(c, 2) == 393216
    codes = np.array([[0, 1], [0, 2], [3, 1]], np.uint32)
    assert unique_table_bytes(codes, cfg(4, 4, 2, 2), 4) == 4 * 4 * 4  # pairs (0,0),(0,3),(1,1),(1,2)


def test_workloads_follow_baseline_json():
    w = WORKLOADS
    assert (w["c1"].d, w["c1"].h, w["c1"].tau, w["c1"].n) == (64, 8, 4, 1024)
    assert (w["c2"].d, w["c2"].h, w["c2"].tau, w["c2"].n) == (768, 256, 8, 16384)
    assert (w["c3"].d, w["c3"].h, w["c3"].tau, w["c3"].n, w["c3"].table_dtype) == (1024, 128, 10, 65536, "bf16")
    assert (w["c4"].d, w["c4"].h, w["c4"].tau, w["c4"].n) == (4096, 512, 8, 8192)
    assert w["c5"].x_kind == "skew"


def test_c1_inputs_use_reference_seeds(oracle):
    """x <- make_rng(0) (DenseMatrix::gaussian), proj <- init(seed 1), T <- N(0,.02) make_rng(2)."""
    from oracle import Spec

    wl = WORKLOADS["c1"]
    c, p, T = make_params(wl)
    x = make_x(wl)
    assert np.array_equal(x, oracle.gaussian(0, 1024 * 64).reshape(1024, 64).astype(np.float32))
    assert np.array_equal(p.blob, oracle.proj_init(Spec(64, 32, 3), 1))
    assert np.array_equal(T.data, oracle.gaussian(2, 8 * 16 * 64, 0.02))


def test_c2_standardised_and_c5_skewed_inputs():
    x = make_x(WORKLOADS["c2"], 64).astype(np.float64)
    assert np.allclose(x.mean(axis=1), 0, atol=1e-6) and np.allclose(x.std(axis=1), 1, atol=1e-5)
    x5 = make_x(WORKLOADS["c5"], 512).astype(np.float64)
    # x = U z + 0.01 eps has rank ~4 up to the noise
    s = np.linalg.svd(x5, compute_uv=False)
    assert s[4] / s[3] < 0.05
