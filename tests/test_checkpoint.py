"""The reference's "LFFN" v1 checkpoint as the on-disk input of the device
path: files written by the reference load bit-exactly through
the C-ABI and vice versa, with the reference's error behaviour; on the GPU a
layer built straight from a file equals one built from memory."""
import os

import numpy as np
import pytest

from oracle import ACDC, BH, DENSE, SCALED, SIGNFLIP, Cfg
from paper_2403_07221_b200 import (HashTables, LookupConfig, LookupFFN, LookupVariant, Projection,
                                   ProjectionSpec, ProjKind, SizeError, UsageError, checkpoint_header,
                                   fill_gaussian, load_checkpoint, save_checkpoint)

CASES = [
    (Cfg(16, 8, 6, 4), dict(kind=SIGNFLIP)),
    (Cfg(16, 8, 6, 4, SCALED), dict(kind=DENSE)),
    (Cfg(16, 8, 6, 4), dict(kind=BH, stages=2, block=8)),
    (Cfg(64, 32, 4, 5), dict(kind=ACDC, depth=3)),
]


def _ours(c, s):
    cfg = LookupConfig(c.d_in, c.d_out, c.tables, c.code_bits, LookupVariant(c.variant))
    spec = ProjectionSpec(s.d_in, s.d_out, ProjKind(s.kind), s.stages, s.block, s.depth)
    return cfg, spec


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"k{c[1]['kind']}-v{c[0].variant}")
def test_reference_file_loads_bit_exactly(reference, tmp_path, case):
    c, kw = case
    s = c.spec(**kw)
    blob = reference.proj_init(s, 11)
    T = reference.tables_init(c, 12)
    path = str(tmp_path / "ref.lffn")
    reference.save_checkpoint(path, c, s, blob, T)
    cfg, proj, tables = load_checkpoint(path)
    ecfg, espec = _ours(c, s)
    assert (cfg.d_in, cfg.d_out, cfg.tables, cfg.code_bits, cfg.variant) == \
        (ecfg.d_in, ecfg.d_out, ecfg.tables, ecfg.code_bits, ecfg.variant)
    assert proj.spec == espec
    assert np.array_equal(proj.blob.view(np.uint64), blob.view(np.uint64))
    assert np.array_equal(tables.data.view(np.uint64), T.view(np.uint64))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"k{c[1]['kind']}-v{c[0].variant}")
def test_our_file_is_the_reference_format(reference, tmp_path, case):
    c, kw = case
    s = c.spec(**kw)
    cfg, spec = _ours(c, s)
    proj = Projection.init(spec, 21)
    tables = HashTables.init(cfg, 22)
    path = str(tmp_path / "ours.lffn")
    save_checkpoint(path, cfg, proj, tables)
    hdr, blob, T = reference.load_checkpoint(path)
    assert hdr["d_in"] == c.d_in and hdr["tables"] == c.tables and hdr["kind"] == s.kind
    assert np.array_equal(blob, proj.blob) and np.array_equal(T, tables.data)


def test_checkpoint_errors(tmp_path):
    cfg = LookupConfig(d_in=8, d_out=4, tables=2, code_bits=3)
    proj = Projection.init(ProjectionSpec.signflip(8, 6), 1)
    tables = HashTables.init(cfg, 2)
    good = str(tmp_path / "good.lffn")
    save_checkpoint(good, cfg, proj, tables)
    raw = open(good, "rb").read()
    cases = {"bad magic": b"XFFN" + raw[4:], "unsupported version": raw[:4] + b"\x02" + raw[5:],
             "truncated": raw[:-8], "trailing bytes": raw + b"\x00",
             "bad variant byte": raw[:24] + b"\x09" + raw[25:]}
    for msg, data in cases.items():
        p = str(tmp_path / (msg.replace(" ", "_") + ".lffn"))
        open(p, "wb").write(data)
        with pytest.raises(UsageError, match=msg):  # checkpoint.cpp:88-136
            load_checkpoint(p)
    with pytest.raises(UsageError, match="cannot open"):
        load_checkpoint(str(tmp_path / "missing.lffn"))
    c2, s2, n = checkpoint_header(good)
    assert (c2.tables, s2.kind, n) == (2, ProjKind.signflip, 2 * 8 * 4)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layer_from_checkpoint_equals_layer_from_memory(tmp_path, dtype):
    from gpu_helpers import device_forward

    cfg = LookupConfig(d_in=768, d_out=768, tables=256, code_bits=8)
    proj = Projection.init(ProjectionSpec.signflip(768, 2048), 1)
    tables = HashTables(256, 8, 768, fill_gaussian(2, 256 * 256 * 768, 0.02))
    path = str(tmp_path / "c2.lffn")
    save_checkpoint(path, cfg, proj, tables)
    x = fill_gaussian(0, 64 * 768).reshape(64, 768).astype(np.float32)
    a = LookupFFN(cfg, proj, tables, max_tokens=64, table_dtype=dtype)
    b = LookupFFN.from_checkpoint(path, max_tokens=64, table_dtype=dtype)
    assert np.array_equal(device_forward(a, x), device_forward(b, x))
    # a table shard streams only its slice
    sh = LookupFFN.from_checkpoint(path, max_tokens=64, table_dtype=dtype, table_range=(100, 200))
    ref = LookupFFN(cfg, proj, tables, max_tokens=64, table_dtype=dtype, table_range=(100, 200))
    assert np.array_equal(device_forward(sh, x), device_forward(ref, x))
    os.remove(path)


def test_shard_from_checkpoint_checks_the_whole_file(tmp_path):
    """A table shard reads only its slice, but a truncated or padded file is
    rejected as load_checkpoint rejects it (checkpoint.cpp:134-136) -- before
    any device work, so this runs without a GPU."""
    cfg = LookupConfig(d_in=8, d_out=4, tables=6, code_bits=3)
    proj = Projection.init(ProjectionSpec.signflip(8, 18), 1)
    good = str(tmp_path / "good.lffn")
    save_checkpoint(good, cfg, proj, HashTables.init(cfg, 2))
    raw = open(good, "rb").read()
    for msg, data in {"truncated": raw[:-8], "trailing bytes": raw + b"\x00" * 8}.items():
        p = str(tmp_path / (msg.replace(" ", "_") + ".lffn"))
        open(p, "wb").write(data)
        with pytest.raises(UsageError, match=msg):
            LookupFFN.from_checkpoint(p, max_tokens=4, table_range=(0, 2))
