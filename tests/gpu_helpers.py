"""Shared helpers for the GPU parity tests (CUDA path vs the oracle)."""
from __future__ import annotations

import numpy as np

from oracle import Cfg, Spec


def to_oracle(cfg, proj):
    """Package objects -> oracle dataclasses."""
    c = Cfg(cfg.d_in, cfg.d_out, cfg.tables, cfg.code_bits, int(cfg.variant), cfg.neighbor_count)
    s = Spec(proj.spec.d_in, proj.spec.d_out, int(proj.spec.kind), proj.spec.stages,
             proj.spec.block, proj.spec.depth)
    return c, s


def stored_tables(T64: np.ndarray, dtype: str) -> np.ndarray:
    """The float64 values the device holds after upload (f32 or bf16 RNE)."""
    from paper_2403_07221_b200 import to_bf16_values

    if dtype == "f32":
        return T64.astype(np.float32).astype(np.float64)
    return to_bf16_values(T64)


def l2_rel(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxabs_rel(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def assert_close(y, y_ref, tol, what=""):
    """The north-star criterion: l2_rel <= tol and max_abs/max|y_ref| <= tol."""
    e1, e2 = l2_rel(y, y_ref), maxabs_rel(y, y_ref)
    assert e1 <= tol and e2 <= tol, f"{what}: l2_rel={e1:.3e} maxabs_rel={e2:.3e} tol={tol}"
    return e1, e2


def device_hash(layer, x32: np.ndarray, want_z: bool = True):
    import torch

    xd = torch.from_numpy(np.ascontiguousarray(x32)).cuda()
    n = x32.shape[0]
    z = torch.empty((n, layer.cfg.code_width()), dtype=torch.float64, device="cuda") if want_z else None
    out = layer.hash(xd, z=z)
    layer.sync()
    codes = out[0].cpu().numpy().view(np.uint32)
    coeff = out[1].cpu().numpy()
    zz = out[2].cpu().numpy() if want_z else None
    return codes, coeff, zz


def device_forward(layer, x32: np.ndarray) -> np.ndarray:
    import torch

    xd = torch.from_numpy(np.ascontiguousarray(x32)).cuda()
    y = layer.forward_device(xd)
    layer.sync()
    return y.cpu().numpy()
