"""The BASELINE.json workloads c1..c5 as seeded synthetic inputs.

Seed convention of the reference benchmark (bench.cpp:274-277, flops.cpp:96-99,
SURVEY.md 8d): x <- make_rng(seed), projection <- Projection::init(spec,
seed+1), tables <- fill_gaussian(make_rng(seed+2), std 0.02), all through the
reference's own engine/distributions (bit-identical values).  There is no
public dataset behind these configs; the value distributions are the ones
BASELINE.json states.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .lookup import (HashTables, LookupConfig, Projection, ProjectionSpec, ProjKind,
                     TableSlice, fill_gaussian, fill_gaussian_slice)

TABLE_STD = 0.02


@dataclass(frozen=True)
class Workload:
    name: str
    d: int
    h: int
    tau: int
    n: int
    x_kind: str          # gaussian | standardized | skew
    table_dtype: str     # f32 | bf16
    note: str = ""


WORKLOADS = {
    "c1": Workload("c1", 64, 8, 4, 1024, "gaussian", "f32", "tiny fp32"),
    "c2": Workload("c2", 768, 256, 8, 16384, "standardized", "f32",
                   "RoBERTa-base width, 32 x 512 tokens, fp32 tables"),
    "c2_bf16": Workload("c2_bf16", 768, 256, 8, 16384, "standardized", "bf16",
                        "RoBERTa-base width, bf16 tables + fp32 accumulation"),
    "c3": Workload("c3", 1024, 128, 10, 65536, "gaussian", "bf16", "tables exceeding L2"),
    "c4": Workload("c4", 4096, 512, 8, 8192, "gaussian", "bf16", "7B width"),
    "c5": Workload("c5", 768, 256, 8, 4096, "skew", "f32", "skewed / small batch"),
}


def config_of(w: Workload) -> LookupConfig:
    return LookupConfig(d_in=w.d, d_out=w.d, tables=w.h, code_bits=w.tau)


def spec_of(w: Workload, kind: ProjKind = ProjKind.signflip) -> ProjectionSpec:
    """signflip (primary), dense, acdc (depth 2) or the paper's BH4 with b = 64."""
    if kind == ProjKind.bh:
        return ProjectionSpec(w.d, w.h * w.tau, kind, stages=4, block=min(64, w.d))
    if kind == ProjKind.acdc:
        return ProjectionSpec(w.d, w.h * w.tau, kind, depth=2)
    return ProjectionSpec(w.d, w.h * w.tau, kind)


def make_x(w: Workload, n: Optional[int] = None, seed: int = 0, gaussian=None) -> np.ndarray:
    """Token inputs, float32 [n x d].  ``gaussian(seed, count)`` draws the
    make_rng(seed) stream (default: this package's bit-identical restatement;
    the bench's reference arm passes the reference library's own)."""
    n = w.n if n is None else n
    fill = fill_gaussian if gaussian is None else gaussian
    if w.x_kind == "skew":
        # x = U z + 0.01 eps: U ~ N(0,1) 768x4 from make_rng(seed); per token
        # z ~ N(0,1)^4 then eps ~ N(0,1)^d from make_rng(seed + 100).  Both
        # per-token draws have even length, so one continuing fill equals
        # the per-token fills.
        U = fill(seed, w.d * 4).reshape(w.d, 4)
        draws = fill(seed + 100, n * (4 + w.d)).reshape(n, 4 + w.d)
        x = draws[:, :4] @ U.T + 0.01 * draws[:, 4:]
        return np.ascontiguousarray(x, np.float32)
    x = fill(seed, n * w.d).reshape(n, w.d)
    if w.x_kind == "standardized":
        mu = x.mean(axis=1, keepdims=True)
        sd = x.std(axis=1, keepdims=True)
        x = (x - mu) / sd
    return np.ascontiguousarray(x, np.float32)


def make_params(w: Workload, kind: ProjKind = ProjKind.signflip, seed: int = 0):
    """(cfg, projection, tables) with the reference seeds."""
    cfg = config_of(w)
    proj = Projection.init(spec_of(w, kind), seed + 1)
    data = fill_gaussian(seed + 2, w.h * (1 << w.tau) * w.d, TABLE_STD)
    return cfg, proj, HashTables(w.h, w.tau, w.d, data)


def make_table_slice(w: Workload, kb: int, ke: int, seed: int = 0) -> TableSlice:
    """Tables [kb, ke) of make_params' stack (the same make_rng(seed+2) stream,
    the prefix drawn and discarded) without materialising the whole stack --
    what a table shard of c4 (4.3 GB of float64 tables) uploads."""
    per = (1 << w.tau) * w.d
    data = fill_gaussian_slice(seed + 2, kb * per, (ke - kb) * per, TABLE_STD)
    return TableSlice((kb, ke), w.tau, w.d, data)
