"""The C-ABI boundary without a GPU: liblffn_gpu.so loads, exports every
function include/lffn_gpu.h declares, its host-side helpers reproduce the
reference's parameter generation and validation, and the device entry points
fail loudly (no CPU fallback) when no B200 is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2403_07221_b200 import (HashTables, LookupConfig, LookupFFN, LookupVariant, Projection,
                                   ProjectionSpec, ProjKind, SizeError, UsageError, _capi, fill_gaussian,
                                   fill_signs, gaussian_matrix, lookup_forward, to_bf16_values)
from paper_2403_07221_b200._capi import DeviceError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lffn_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lffn_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["lffn_ctx_create", "lffn_tables_upload", "lffn_hash", "lffn_lookup_accumulate",
                 "lffn_forward", "lffn_forward_host", "lffn_sync", "lffn_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(declared_functions()) == set(_capi.SIGNATURES)


def test_version_string():
    assert _capi.lib().lffn_version().decode().endswith("sm_100a")


def test_library_is_sm100a_only():
    """The shipped cubin targets sm_100a (no PTX / other-arch fallback)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_[0-9]+[^0a-z]", out.replace("sm_100a", ""))


def test_rng_helpers_match_oracle(oracle):
    for seed in (0, 2, 77):
        for n in (1, 10, 1001):
            assert np.array_equal(fill_gaussian(seed, n, 0.02), oracle.gaussian(seed, n, 0.02))
            assert np.array_equal(fill_signs(seed, n), oracle.signs(seed, n))
    assert np.array_equal(gaussian_matrix(3, 5, 9).ravel(), oracle.gaussian(9, 15))


@pytest.mark.parametrize("spec", [
    ProjectionSpec.signflip(768, 2048), ProjectionSpec.signflip(50, 120),
    ProjectionSpec.dense(50, 70), ProjectionSpec.bh(64, 64, 2, 8), ProjectionSpec.bh(50, 120, 4, 16),
    ProjectionSpec.acdc(40, 100, 2), ProjectionSpec.bh(16, 16, 1, 0)],
    ids=lambda s: f"{s.kind.name}-{s.d_in}x{s.d_out}")
def test_projection_init_matches_oracle(oracle, spec):
    from oracle import Spec

    p = Projection.init(spec, 99)
    s = Spec(spec.d_in, spec.d_out, int(spec.kind), spec.stages, spec.block, spec.depth)
    assert np.array_equal(p.blob.view(np.uint64), oracle.proj_init(s, 99).view(np.uint64))


def test_tables_init_matches_reference(reference):
    from oracle import Cfg

    cfg = LookupConfig(d_in=8, d_out=6, tables=5, code_bits=3)
    T = HashTables.init(cfg, 13)
    assert np.array_equal(T.data, reference.tables_init(Cfg(8, 6, 5, 3), 13))
    assert T.row(2, 5).shape == (6,)
    assert isinstance(T.checksum(), int)


def _exact_bf16(d: float) -> float:
    """Round a double to bf16 exactly (RNE) with integer arithmetic."""
    import fractions
    import math

    if d == 0 or not math.isfinite(d):
        return d
    f = fractions.Fraction(d)
    sgn = -1 if f < 0 else 1
    f = abs(f)
    e = math.floor(math.log2(f))
    while fractions.Fraction(2) ** e > f:
        e -= 1
    while fractions.Fraction(2) ** (e + 1) <= f:
        e += 1
    e = max(e, -126)
    q = f / fractions.Fraction(2) ** (e - 7)  # 8 significant bits
    n = math.floor(q)
    rem = q - n
    if rem > fractions.Fraction(1, 2) or (rem == fractions.Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sgn * float(n * fractions.Fraction(2) ** (e - 7))


def test_bf16_conversion_is_single_rne():
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.normal(0, 0.02, 3000), rng.normal(0, 100, 1000),
                           [1.0 + 2.0 ** -8, 1.0 + 2.0 ** -8 + 2.0 ** -40, 1.0 + 3 * 2.0 ** -9,
                            -(1.0 + 2.0 ** -8 - 2.0 ** -40), 1e-40, 0.0, -0.0]])
    got = to_bf16_values(vals)
    expect = np.array([_exact_bf16(float(v)) for v in vals])
    assert np.array_equal(got, expect)


def test_config_validation_messages():
    with pytest.raises(SizeError, match="neighbor count"):
        LookupConfig(d_in=8, d_out=4, tables=2, code_bits=3, neighbor_count=9).validate()
    with pytest.raises(SizeError, match="code bits"):
        LookupConfig(d_in=8, d_out=4, tables=2, code_bits=0).validate()
    with pytest.raises(SizeError, match="tau-1 variants"):
        LookupConfig(d_in=8, d_out=4, tables=2, code_bits=3,
                     variant=LookupVariant.gelu_tau1).validate()
    with pytest.raises(SizeError, match="block size"):
        ProjectionSpec.bh(16, 16, 2, 5).validate()
    with pytest.raises(SizeError, match="stage count"):
        ProjectionSpec.bh(16, 16, 0, 4).validate()
    with pytest.raises(SizeError, match="projection blob"):
        Projection.from_blob(ProjectionSpec.signflip(8, 8), np.ones(5))


def test_lookup_forward_shape_errors_before_device():
    cfg = LookupConfig(d_in=8, d_out=4, tables=2, code_bits=3)
    proj = Projection.init(ProjectionSpec.dense(8, 5), 1)  # wrong width (h*tau = 6)
    T = HashTables.init(cfg, 2)
    with pytest.raises(SizeError, match="projection must map"):
        lookup_forward(np.zeros((2, 8)), proj, T, cfg)
    proj = Projection.init(ProjectionSpec.dense(8, 6), 1)
    with pytest.raises(SizeError, match="input width"):
        lookup_forward(np.zeros((2, 7)), proj, T, cfg)
    with pytest.raises(UsageError, match="LookupCache"):
        lookup_forward(np.zeros((2, 8)), proj, T, cfg, cache=object())


def test_device_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = LookupConfig(d_in=8, d_out=4, tables=2, code_bits=3)
    proj = Projection.init(ProjectionSpec.signflip(8, 6), 1)
    with pytest.raises(DeviceError):
        LookupFFN(cfg, proj, HashTables.init(cfg, 2), max_tokens=4)


def test_nc_above_device_limit_is_rejected_before_any_device_work():
    cfg = LookupConfig(d_in=8, d_out=4, tables=2, code_bits=9, neighbor_count=257)
    proj = Projection.init(ProjectionSpec.signflip(8, 18), 1)
    with pytest.raises(SizeError, match="neighbor_count"):
        LookupFFN(cfg, proj, None, max_tokens=4)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2403_07221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
                assert "lffn_oracle" not in src and "liblffn_ref" not in src, f
