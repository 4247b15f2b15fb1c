"""The reference's hot-path unit tests, restated against
the oracle.  Each test cites the reference test it mirrors; the same
known-answer cases run on the device in tests/test_gpu_parity.py."""
import math

import numpy as np
import pytest

from oracle import ACDC, BH, DENSE, GELU_TAU1, SCALED, SIGMOID_TAU1, SIGNFLIP, SOFTMAX, Cfg, Spec


def codebook(tau):
    """Row i of S is the +/-1 pattern of integer i, LSB first (test_lookup.cpp:17-22)."""
    return np.array([[1.0 if (i >> j) & 1 else -1.0 for j in range(tau)] for i in range(1 << tau)])


def H(n):
    return np.array([[(-1.0) ** bin(i & j).count("1") for j in range(n)] for i in range(n)])


def test_sign_code_lsb_convention(oracle):
    """test_lookup.cpp:70-74"""
    assert oracle.sign_code([2.0, -1.0, 3.0]) == 5
    assert oracle.sign_code([-1.0, -2.0, -3.0]) == 0
    assert oracle.sign_code([0.0, -1.0]) == 1  # sign(0) = +1
    assert oracle.sign_code([-0.0, 1.0]) == 3  # -0.0 >= 0 holds as well


def test_compute_codes_is_codebook_argmax(oracle):
    """test_lookup.cpp:85-103 (tau = 8, 100 z, the reference draws seed 21)"""
    tau = 8
    S = codebook(tau)
    z = oracle.gaussian(21, 100 * tau).reshape(100, tau)
    codes, _ = oracle.compute_codes(z, 1, tau)
    assert np.array_equal(codes[:, 0], np.argmax(z @ S.T, axis=1))


@pytest.mark.parametrize("tau", range(1, 11))
def test_code_identities(oracle, tau):
    """test_lookup.cpp:105-124: <z, S_g> = sum|z| and g / ~g attain max / min."""
    S = codebook(tau)
    r = oracle.rng(22 + tau)
    for _ in range(10):
        z = oracle.gaussian(r, tau)
        g = oracle.sign_code(z)
        dots = S @ z
        assert math.isclose(dots[g], np.abs(z).sum(), rel_tol=1e-13)
        assert dots.max() <= dots[g] + 1e-12
        assert dots.min() >= dots[g ^ ((1 << tau) - 1)] - 1e-12


def test_log_denominator(oracle):
    """test_lookup.cpp:126-150"""
    assert math.isclose(oracle.log_denominator([0.0, 0.0, 0.0]), math.log(8.0), rel_tol=1e-15)
    S = codebook(10)
    r = oracle.rng(23)
    for _ in range(50):
        z = 2.0 * oracle.gaussian(r, 10)
        ref = math.log(np.exp(S @ z).sum())
        assert abs(oracle.log_denominator(z) - ref) / abs(ref) < 1e-10
    z = [500.0, 1.0, -2.0]
    expect = (500.0 + math.log1p(math.exp(-1000.0))) + (1 + math.log1p(math.exp(-2))) + \
        (2 + math.log1p(math.exp(-4)))
    assert math.isclose(oracle.log_denominator(z), expect, rel_tol=1e-14)


def test_neighbor_codes(oracle):
    """test_lookup.cpp:152-205"""
    assert list(oracle.neighbor_codes([4.0, 3.0, 2.0, 1.0], 3)) == [0b1111, 0b0111, 0b1011]
    S = codebook(8)
    r = oracle.rng(25)
    for _ in range(20):
        z = oracle.gaussian(r, 8)
        got = oracle.neighbor_codes(z, 16)
        scores = S @ z
        assert set(got.tolist()) == set(np.argsort(-scores, kind="stable")[:16].tolist())
        d = [oracle.code_dot(z, int(c)) for c in got]
        assert all(a >= b - 1e-12 for a, b in zip(d, d[1:]))
    z = oracle.gaussian(26, 5)
    assert sorted(oracle.neighbor_codes(z, 32).tolist()) == list(range(32))
    with pytest.raises(ValueError):
        oracle.neighbor_codes(z, 33)


def test_zero_projection_spreads_mass(oracle):
    """test_lookup.cpp:207-230: z = 0 -> code 2^tau - 1, y = sum_k T[k][all-ones] / 16."""
    cfg = Cfg(6, 5, 3, 4)
    spec = Spec(6, 12, DENSE)
    T = oracle.gaussian(31, 3 * 16 * 5, 1 / math.sqrt(3))
    x = oracle.gaussian(30, 12).reshape(2, 6)
    y, cache = oracle.lookup_forward(cfg, spec, np.zeros(72), T, x, True)
    assert (cache["codes"] == 15).all()
    expect = T.reshape(3, 16, 5)[:, 15, :].sum(axis=0) / 16.0
    np.testing.assert_allclose(y, np.broadcast_to(expect, (2, 5)), rtol=1e-12)


def test_tau1_equal_rows(oracle):
    """test_lookup.cpp:232-249"""
    cfg = Cfg(4, 3, 5, 1)
    T = np.tile(np.array([0.5, -1.0, 2.0]), 10)
    x = np.zeros((1, 4))
    x[0, 1] = 0.3
    y = oracle.lookup_forward(cfg, Spec(4, 5, DENSE), np.zeros(20), T, x)
    np.testing.assert_allclose(y[0], 5 * np.array([0.5, -1.0, 2.0]) / 2, rtol=1e-12)


@pytest.mark.parametrize("variant", [SOFTMAX, SCALED])
def test_full_neighbor_equals_codebook(oracle, variant):
    """test_lookup.cpp:251-272"""
    cfg = Cfg(8, 6, 2, 3, variant, 8)
    spec = cfg.spec(BH, stages=2, block=4)
    blob = oracle.proj_init(spec, 34)
    T = oracle.gaussian(35, 2 * 8 * 6, 1 / math.sqrt(2))
    x = oracle.gaussian(33, 16 * 8).reshape(16, 8)
    y = oracle.lookup_forward(cfg, spec, blob, T, x)
    z = oracle.proj_forward(spec, blob, x)
    S = codebook(3)
    expect = np.zeros_like(y)
    for i in range(16):
        for k in range(2):
            d = S @ z[i, 3 * k:3 * k + 3]
            num = np.exp(d) * (d if variant == SCALED else 1.0)
            expect[i] += (num / np.exp(d).sum()) @ T.reshape(2, 8, 6)[k]
    rel = np.max(np.abs(y - expect) / np.maximum(np.maximum(np.abs(y), np.abs(expect)), 1e-3))
    assert rel < 1e-10


def test_tau1_sigmoid_and_gelu(oracle):
    """test_lookup.cpp:274-342"""
    d, units, d_out = 7, 9, 4
    w = oracle.gaussian(36, units * d).reshape(units, d)
    v = oracle.gaussian(37, units * d_out).reshape(units, d_out)
    x = oracle.gaussian(38, 12 * d).reshape(12, d)
    T = np.zeros((units, 2, d_out))
    T[:, 1, :] = v
    y = oracle.lookup_forward(Cfg(d, d_out, units, 1, SIGMOID_TAU1, 2), Spec(d, units, DENSE),
                              (0.5 * w.T).copy(), T.ravel(), x)
    expect = (1 / (1 + np.exp(-(x @ w.T)))) @ v
    assert np.max(np.abs(y - expect) / np.maximum(np.abs(expect), 1e-3)) < 1e-10
    T[:, 1, :] = 1.175 * v
    y = oracle.lookup_forward(Cfg(d, d_out, units, 1, GELU_TAU1, 2), Spec(d, units, DENSE),
                              (0.851 * w.T).copy(), T.ravel(), x)
    zz = 0.851 * (x @ w.T)
    expect = (1.175 * zz / (1 + np.exp(-2 * zz))) @ v
    assert np.max(np.abs(y - expect) / np.maximum(np.abs(expect), 1e-3)) < 1e-10


def test_top1_weight_range(oracle):
    """test_lookup.cpp:351-362"""
    r = oracle.rng(38)
    for tau in range(1, 11):
        for _ in range(30):
            w = oracle.top1_weight(np.abs(oracle.gaussian(r, tau)))
            assert 2.0 ** -tau < w <= 1.0


def test_fwht_cases(oracle):
    """test_fwht.cpp:12-108"""
    assert oracle.fwht([3.5])[0] == 3.5
    assert (oracle.fwht([1, 0, 0, 0]) == 1).all()
    r = oracle.rng(11)
    for n in [1, 2, 4, 8, 64, 1024]:
        v = oracle.gaussian(r, n)
        np.testing.assert_allclose(oracle.fwht(v), H(n) @ v, rtol=1e-12, atol=1e-12)
    for n in [8, 64, 1024, 4096]:
        v = oracle.gaussian(r, n)
        np.testing.assert_allclose(oracle.fwht(oracle.fwht(v)), n * v, rtol=1e-12, atol=1e-9)
    u, v = oracle.gaussian(r, 256), oracle.gaussian(r, 256)
    np.testing.assert_allclose(oracle.fwht(1.7 * u - 0.4 * v),
                               1.7 * oracle.fwht(u) - 0.4 * oracle.fwht(v), rtol=1e-12, atol=1e-12)
    assert (H(4) == np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]])).all()


def test_projection_operators(oracle):
    """test_projection.cpp:37-137: every kind equals its basis-materialised operator
    (incl. non-pow2 pad/truncate), signflip with +1 signs = n H x, dense = triple loop."""
    r = oracle.rng(7)
    for spec in [Spec(64, 64, BH, 2, 8), Spec(50, 120, BH, 4, 16), Spec(64, 64, ACDC, depth=3),
                 Spec(40, 100, ACDC, depth=2), Spec(64, 64, SIGNFLIP), Spec(50, 70, DENSE)]:
        blob = oracle.proj_init(spec, 99)
        R = oracle.proj_forward(spec, blob, np.eye(spec.d_in))
        x = oracle.gaussian(r, 5 * spec.d_in).reshape(5, spec.d_in)
        y = oracle.proj_forward(spec, blob, x)
        assert np.max(np.abs(y - x @ R) / np.maximum(np.abs(y), 1.0)) < 1e-10
    spec = Spec(8, 8, SIGNFLIP)
    x = oracle.gaussian(8, 24).reshape(3, 8)
    np.testing.assert_allclose(oracle.proj_forward(spec, np.ones(24), x), 8 * x @ H(8).T,
                               rtol=1e-12)
    spec = Spec(4, 3, DENSE)
    blob = oracle.proj_init(spec, 21)
    x = oracle.gaussian(4, 12).reshape(3, 4)
    np.testing.assert_allclose(oracle.proj_forward(spec, blob, x), x @ blob.reshape(4, 3),
                               rtol=1e-12)


def test_bh_d1024_matches_dense_stage_product(oracle):
    """test_projection.cpp:45-76 (one block size, 4 rows)."""
    D, b = 1024, 64
    spec = Spec(D, D, BH, 4, b)
    blob = oracle.proj_init(spec, 5)
    stage = (D // b) * b * b
    Hd = H(D)
    R = None
    for s in range(4):
        blocks = blob[s * stage:(s + 1) * stage].reshape(D // b, b, b)
        B = np.zeros((D, D))
        for g in range(D // b):
            B[g * b:(g + 1) * b, g * b:(g + 1) * b] = blocks[g]
        R = B @ Hd if R is None else R @ B @ Hd
    x = oracle.gaussian(42, 4 * D).reshape(4, D)
    y = oracle.proj_forward(spec, blob, x)
    assert np.max(np.abs(y - x @ R) / np.maximum(np.abs(y), 1.0)) < 1e-10


def test_init_determinism_and_variance(oracle):
    """test_projection.cpp:233-270"""
    spec = Spec(32, 32, BH, 4, 8)
    assert np.array_equal(oracle.proj_init(spec, 123), oracle.proj_init(spec, 123))
    assert not np.array_equal(oracle.proj_init(spec, 123), oracle.proj_init(spec, 124))
    x = oracle.gaussian(11, 256 * 256).reshape(256, 256)
    for spec, scale in [(Spec(256, 256, ACDC, depth=4), 1.0), (Spec(256, 256, SIGNFLIP), 256 ** 1.5)]:
        y = oracle.proj_forward(spec, oracle.proj_init(spec, 12), x)
        assert 0.5 < np.sqrt((y ** 2).mean()) / scale < 2.0


def test_workload_regularity_reads(oracle):
    """test_lookup.cpp:446-456: every row reads exactly h * nc table rows -- the
    cache exposes nc codes per (row, table)."""
    cfg = Cfg(16, 8, 6, 4, SOFTMAX, 3)
    spec = cfg.spec(BH, 2, 8)
    x = oracle.gaussian(70, 32 * 16).reshape(32, 16)
    _, c = oracle.lookup_forward(cfg, spec, oracle.proj_init(spec, 71),
                                 oracle.gaussian(72, 6 * 16 * 8), x, True)
    assert c["codes"].shape == (32, 6, 3)
    assert all(len(set(c["codes"][i, k].tolist())) == 3 for i in range(32) for k in range(6))


def test_validation_errors(oracle):
    """test_lookup.cpp:477-500 / test_projection.cpp:272-279"""
    x = np.zeros((2, 8))
    with pytest.raises(ValueError):
        oracle.lookup_forward(Cfg(8, 4, 2, 3, SOFTMAX, 9), Spec(8, 6, SIGNFLIP), np.ones(24),
                              np.zeros(64), x)
    with pytest.raises(ValueError):
        oracle.lookup_forward(Cfg(8, 4, 2, 3), Spec(8, 5, DENSE), np.zeros(40), np.zeros(64), x)
    with pytest.raises(ValueError):
        oracle.proj_init(Spec(16, 16, BH, 2, 5), 1)
    with pytest.raises(ValueError):
        oracle.proj_init(Spec(16, 16, BH, 0, 4), 1)
