"""Algorithmic cost model of the forward path (restates flops.cpp).

Used for the roofline denominators in bench.py.  Conventions are the
reference's (flops.hpp:11-23): one multiply-accumulate = 2 FLOP, a Hadamard
butterfly add = 1 FLOP, weight math charged 6 FLOP per soft-code coordinate.
Byte counts (not in the reference) follow SURVEY.md section 8(d): gathered
bytes G = h * d_out * elem per token, unique bytes U from the actual codes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lookup import LookupConfig, ProjectionSpec, ProjKind

K_WEIGHT_FLOPS_PER_COORD = 6.0  # flops.hpp:23


@dataclass
class FlopReport:
    hash_mflop: float = 0.0
    gather_mflop: float = 0.0
    other_mflop: float = 0.0

    def total_mflop(self) -> float:
        return self.hash_mflop + self.gather_mflop + self.other_mflop


def vanilla_flops(d_in: int, hidden: int, d_out: int) -> FlopReport:
    """flops.cpp:9-15"""
    return FlopReport(other_mflop=(2.0 * d_in * hidden + 2.0 * hidden * d_out) / 1e6)


def projection_cost(spec: ProjectionSpec) -> tuple:
    """(flops, params) per row -- flops.cpp:17-44"""
    D = spec.transform_width()
    logD = D.bit_length() - 1
    if spec.kind == ProjKind.dense:
        return 2.0 * spec.d_in * spec.d_out, spec.d_in * spec.d_out
    if spec.kind == ProjKind.bh:
        b = D if spec.block == 0 else spec.block
        return spec.stages * (2.0 * D * b + D * logD), spec.stages * D * b
    if spec.kind == ProjKind.acdc:
        return spec.depth * (2.0 * D + 2.0 * D * logD), 2 * spec.depth * D
    return 3.0 * D + 3.0 * D * logD, 0


def lookup_flops(cfg: LookupConfig, proj: ProjectionSpec) -> FlopReport:
    """flops.cpp:51-60"""
    return FlopReport(hash_mflop=projection_cost(proj)[0] / 1e6,
                      gather_mflop=2.0 * cfg.tables * cfg.neighbor_count * cfg.d_out / 1e6,
                      other_mflop=K_WEIGHT_FLOPS_PER_COORD * cfg.tables * cfg.code_bits / 1e6)


def gathered_bytes_per_token(cfg: LookupConfig, elem_bytes: int) -> int:
    """Algorithmic gather bytes per token: one table row per table."""
    return cfg.tables * cfg.d_out * elem_bytes


def unique_table_bytes(codes: np.ndarray, cfg: LookupConfig, elem_bytes: int) -> int:
    """U: distinct (table, code) pairs actually touched x row bytes."""
    codes = np.asarray(codes).reshape(-1, codes.shape[-1]).astype(np.int64)
    h = codes.shape[1]
    keys = codes + (np.arange(h, dtype=np.int64) << 32)[None, :]
    return int(np.unique(keys).size) * cfg.d_out * elem_bytes
