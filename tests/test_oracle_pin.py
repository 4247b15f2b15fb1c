"""Pin the C restatement (oracle/lffn_oracle.c) against the reference itself.

The reference library is compiled from its own sources into
oracle/_ref/liblffn_ref.so (oracle/Makefile).  Every oracle function must be
BIT-identical to the reference on the same inputs: the restatement keeps the
reference's float64 operation order, and both are built for baseline x86-64
(no FMA contraction) against the same libm.
"""
import numpy as np
import pytest

from oracle import ACDC, BH, DENSE, GELU_TAU1, SCALED, SIGMOID_TAU1, SIGNFLIP, SOFTMAX, Cfg, Spec


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("seed", [0, 1, 2, 12345, 2**63 + 7])
@pytest.mark.parametrize("n", [1, 2, 3, 1001])
def test_rng_streams(oracle, reference, seed, n):
    """make_rng + fill_gaussian / fill_signs (common.hpp:44-55), odd and even counts."""
    for std in (1.0, 0.02, 1 / np.sqrt(768)):
        assert bits_equal(oracle.gaussian(seed, n, std), reference.gaussian(seed, n, std))
    assert bits_equal(oracle.signs(seed, n), reference.signs(seed, n))


SPECS = [
    Spec(64, 32, SIGNFLIP), Spec(50, 120, SIGNFLIP), Spec(768, 2048, SIGNFLIP),
    Spec(1, 1, SIGNFLIP), Spec(3, 8, SIGNFLIP),
    Spec(64, 32, DENSE), Spec(50, 70, DENSE), Spec(4, 3, DENSE),
    Spec(64, 64, BH, stages=2, block=8), Spec(50, 120, BH, stages=4, block=16),
    Spec(16, 16, BH, stages=1, block=0), Spec(8, 8, BH, stages=3, block=4),
    Spec(64, 64, ACDC, depth=3), Spec(40, 100, ACDC, depth=2),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"k{s.kind}-{s.d_in}x{s.d_out}-m{s.stages}b{s.block}d{s.depth}")
def test_projection_init_and_forward(oracle, reference, spec):
    """Projection::init (projection.cpp:97-135) and forward (:167-266)."""
    b_o = oracle.proj_init(spec, 99)
    b_r = reference.proj_init(spec, 99)
    assert bits_equal(b_o, b_r)
    x = reference.gaussian(7, 9 * spec.d_in).reshape(9, spec.d_in)
    assert bits_equal(oracle.proj_forward(spec, b_o, x), reference.proj_forward(spec, b_r, x))


def test_fwht(oracle, reference):
    for n in [1, 2, 4, 64, 1024, 4096]:
        v = reference.gaussian(n, n)
        assert bits_equal(oracle.fwht(v), reference.fwht(v))


@pytest.mark.parametrize("tau", [1, 3, 8, 10, 24])
def test_codes_and_scores(oracle, reference, tau):
    z = reference.gaussian(tau, 40 * tau).reshape(40, tau)
    z[0, :] = 0.0
    z[1, 0] = -0.0
    c_o, a_o = oracle.compute_codes(z, 1, tau)
    c_r, a_r = reference.compute_codes(z, 1, tau)
    assert np.array_equal(c_o, c_r) and bits_equal(a_o, a_r)
    for row in z[:8]:
        assert oracle.sign_code(row) == reference.sign_code(row)
        assert bits_equal(oracle.log_denominator(row), reference.log_denominator(row))
        code = reference.sign_code(row) ^ 1
        assert bits_equal(oracle.code_dot(row, code), reference.code_dot(row, code))
        cnt = min(1 << tau, 20)
        assert np.array_equal(oracle.neighbor_codes(row, cnt), reference.neighbor_codes(row, cnt))


def test_neighbor_codes_with_ties(oracle, reference):
    """Equal |z_j| make the priority-queue tie order observable."""
    for z in ([1.0, -1.0, 1.0, -1.0, 2.0, -2.0], [0.5] * 8, [0.0, 0.0, 1.0, 1.0],
              [3.0, 1.0, 1.0, 2.0, 2.0, 1.0]):
        z = np.array(z)
        n = 1 << z.size
        assert np.array_equal(oracle.neighbor_codes(z, n), reference.neighbor_codes(z, n))


FWD = [
    (Cfg(64, 64, 8, 4), dict(kind=SIGNFLIP)),
    (Cfg(64, 64, 8, 4, SCALED), dict(kind=DENSE)),
    (Cfg(50, 30, 12, 10, SCALED), dict(kind=SIGNFLIP)),
    (Cfg(16, 8, 6, 4, SOFTMAX, 3), dict(kind=BH, stages=2, block=8)),
    (Cfg(8, 6, 2, 3, SOFTMAX, 8), dict(kind=BH, stages=2, block=4)),
    (Cfg(8, 6, 2, 3, SCALED, 8), dict(kind=BH, stages=2, block=4)),
    (Cfg(7, 4, 9, 1, SIGMOID_TAU1, 2), dict(kind=DENSE)),
    (Cfg(6, 5, 8, 1, GELU_TAU1, 2), dict(kind=DENSE)),
    (Cfg(64, 64, 16, 4), dict(kind=ACDC, depth=2)),
]


@pytest.mark.parametrize("case", FWD, ids=lambda c: f"{c[0].d_in}-{c[0].tables}x{c[0].code_bits}-v{c[0].variant}-nc{c[0].neighbor_count}-k{c[1]['kind']}")
def test_lookup_forward(oracle, reference, case):
    """lookup_forward (lookup.cpp:191-282) incl. the LookupCache fields."""
    cfg, kw = case
    spec = cfg.spec(**kw)
    blob = reference.proj_init(spec, 3)
    T = reference.tables_init(cfg, 4)
    x = reference.gaussian(5, 17 * cfg.d_in).reshape(17, cfg.d_in)
    y_o, c_o = oracle.lookup_forward(cfg, spec, blob, T, x, True)
    y_r, c_r = reference.lookup_forward(cfg, spec, blob, T, x, True)
    assert bits_equal(y_o, y_r)
    for k in ("z", "weights", "dots"):
        assert bits_equal(c_o[k], c_r[k]), k
    assert np.array_equal(c_o["codes"], c_r["codes"])


def test_lookup_forward_c2_slice(oracle, reference):
    """BASELINE c2 shape (768 -> 256 x 8, signflip), 64 tokens."""
    cfg = Cfg(768, 768, 256, 8)
    spec = cfg.spec(SIGNFLIP)
    blob = reference.proj_init(spec, 1)
    T = reference.gaussian(2, 256 * 256 * 768, 0.02)
    x = reference.gaussian(0, 64 * 768).reshape(64, 768)
    assert bits_equal(oracle.lookup_forward(cfg, spec, blob, T, x),
                      reference.lookup_forward(cfg, spec, blob, T, x))


def test_validation_matches(oracle, reference):
    """check_shapes / LookupConfig::validate reject the same inputs (SizeError)."""
    T = np.zeros(2 * 8 * 4)
    x = np.zeros((2, 8))
    for cfg, spec in [(Cfg(8, 4, 2, 3, SOFTMAX, 9), Spec(8, 6, SIGNFLIP)),
                      (Cfg(8, 4, 2, 0), Spec(8, 0, SIGNFLIP)),
                      (Cfg(8, 4, 2, 3), Spec(8, 5, DENSE)),
                      (Cfg(8, 4, 2, 3, GELU_TAU1), Spec(8, 6, DENSE))]:
        blob = np.zeros(max(spec.blob_size(), 1))
        with pytest.raises(ValueError):
            oracle.lookup_forward(cfg, spec, blob, T, x)
        with pytest.raises(ValueError):
            reference.lookup_forward(cfg, spec, blob, T, x)


def test_non_finite_input(oracle, reference):
    cfg = Cfg(8, 4, 2, 3)
    spec = cfg.spec(DENSE)
    blob = reference.proj_init(spec, 1)
    T = reference.tables_init(cfg, 2)
    x = np.ones((2, 8))
    x[1, 3] = np.nan
    with pytest.raises(ArithmeticError):
        oracle.lookup_forward(cfg, spec, blob, T, x)
    with pytest.raises(ArithmeticError, match="projection forward input"):
        reference.lookup_forward(cfg, spec, blob, T, x)


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"k{s.kind}-{s.d_in}x{s.d_out}-m{s.stages}b{s.block}d{s.depth}")
def test_proj_backward(oracle, reference, spec):
    """Projection::backward (projection.cpp:279-386): grad_x and the parameter
    gradients, every kind (bh / acdc with the forward's stage inputs)."""
    blob = reference.proj_init(spec, 7)
    x = reference.gaussian(8, 9 * spec.d_in).reshape(9, spec.d_in)
    go = reference.gaussian(9, 9 * spec.d_out).reshape(9, spec.d_out)
    gx_o, gp_o = oracle.proj_backward(spec, blob, x, go)
    gx_r, gp_r = reference.proj_backward(spec, blob, x, go)
    assert bits_equal(gx_o, gx_r)
    assert bits_equal(gp_o, gp_r)


@pytest.mark.parametrize("case", FWD, ids=lambda c: f"{c[0].d_in}-{c[0].tables}x{c[0].code_bits}-v{c[0].variant}-nc{c[0].neighbor_count}-k{c[1]['kind']}")
def test_lookup_backward(oracle, reference, case):
    """lookup_backward (lookup.cpp:292-347): grad_tables, grad_proj, grad_x."""
    cfg, kw = case
    spec = cfg.spec(**kw)
    blob = reference.proj_init(spec, 3)
    T = reference.tables_init(cfg, 4)
    x = reference.gaussian(5, 11 * cfg.d_in).reshape(11, cfg.d_in)
    gy = reference.gaussian(6, 11 * cfg.d_out).reshape(11, cfg.d_out)
    g_o = oracle.lookup_backward(cfg, spec, blob, T, x, gy)
    g_r = reference.lookup_backward(cfg, spec, blob, T, x, gy)
    for k in ("grad_x", "grad_tables", "grad_proj"):
        assert bits_equal(g_o[k], g_r[k]), k
