"""The C oracle against the fixtures generated from the reference itself
(tests/golden/make_golden.py).  Runs anywhere: the fixtures are committed, and
tables that are too large to store are regenerated from their seed and pinned
by a sha256 of their bytes."""
import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import Cfg, Spec

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load(path):
    d = dict(np.load(path))
    cfg = Cfg(int(d["d_in"]), int(d["d_out"]), int(d["tables"]), int(d["code_bits"]),
              int(d["variant"]), int(d["neighbor_count"]))
    spec = Spec(cfg.d_in, cfg.tables * cfg.code_bits, int(d["kind"]), int(d["stages"]),
                int(d["block"]), int(d["depth"]))
    return d, cfg, spec


def tables_of(oracle, d, cfg):
    if "T" in d:
        return d["T"]
    T = oracle.gaussian(int(d["t_seed"]), cfg.tables * cfg.rows * cfg.d_out, float(d["t_std"]))
    assert hashlib.sha256(T.tobytes()).hexdigest() == str(d["tables_sha256"])
    return T


def test_fixtures_present():
    names = {os.path.basename(p) for p in GOLDEN}
    assert {"c1_signflip.npz", "c2_signflip_4tok.npz", "c1_dense.npz"} <= names


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_reproduces_reference_fixture(oracle, path):
    d, cfg, spec = load(path)
    # parameters regenerate bit-exactly from the seeds
    blob = oracle.proj_init(spec, int(d["proj_seed"]))
    if "blob" in d:
        assert np.array_equal(blob.view(np.uint64), d["blob"].view(np.uint64))
    else:  # large blobs are pinned by checksum
        assert hashlib.sha256(blob.tobytes()).hexdigest() == str(d["blob_sha256"])
    T = tables_of(oracle, d, cfg)
    x = d["x"].astype(np.float64)  # compact fixtures store the fp32 values
    y, cache = oracle.lookup_forward(cfg, spec, blob, T, x, want_cache=True)
    assert np.array_equal(y.view(np.uint64), d["y"].view(np.uint64))
    if "z" in d:
        assert np.array_equal(cache["z"].view(np.uint64), d["z"].view(np.uint64))
    else:  # BASELINE-width fixtures pin z by checksum
        assert hashlib.sha256(np.ascontiguousarray(cache["z"]).tobytes()).hexdigest() == str(d["z_sha256"])
    assert np.array_equal(cache["codes"], d["codes"])
    assert np.array_equal(cache["weights"].view(np.uint64), d["weights"].view(np.uint64))
