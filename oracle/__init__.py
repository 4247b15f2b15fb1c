"""Parity oracles for the LookupFFN forward path -- TEST INFRASTRUCTURE ONLY.

Two checkers with one Python face:

* ``Oracle``    -- ``oracle/liblffn_oracle.so``, the plain-C restatement of the
  reference algorithm (``oracle/lffn_oracle.c``, every function citing the
  reference file:line it follows).
* ``Reference`` -- ``oracle/_ref/liblffn_ref.so``, the reference C++ library
  itself, compiled from its own sources by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product path (``paper_2403_07221_b200``) never
imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblffn_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblffn_ref.so")

DENSE, BH, ACDC, SIGNFLIP = 0, 1, 2, 3
SOFTMAX, SCALED, SIGMOID_TAU1, GELU_TAU1 = 0, 1, 2, 3

_p = np.ctypeslib.ndpointer
_f64 = _p(dtype=np.float64, flags="C_CONTIGUOUS")
_f32 = _p(dtype=np.float32, flags="C_CONTIGUOUS")
_u32 = _p(dtype=np.uint32, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile both checkers (the reference one only where its sources exist)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, os.path.join(HERE, "liblffn_oracle.so")], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


@dataclass
class Spec:
    """ProjectionSpec (projection.hpp:21-37)."""

    d_in: int
    d_out: int
    kind: int = SIGNFLIP
    stages: int = 4
    block: int = 0
    depth: int = 1

    @property
    def D(self) -> int:
        m = max(self.d_in, self.d_out)
        p = 1
        while p < m:
            p <<= 1
        return p

    def blob_size(self) -> int:
        D = self.D
        if self.kind == DENSE:
            return self.d_in * self.d_out
        if self.kind == BH:
            b = D if self.block == 0 else self.block
            return self.stages * (D // b) * b * b
        if self.kind == ACDC:
            return 2 * self.depth * D
        return 3 * D


@dataclass
class Cfg:
    """LookupConfig (lookup.hpp:25-39)."""

    d_in: int
    d_out: int
    tables: int
    code_bits: int
    variant: int = SOFTMAX
    neighbor_count: int = 1

    @property
    def rows(self) -> int:
        return 1 << self.code_bits

    def spec(self, kind=SIGNFLIP, stages=4, block=0, depth=1) -> Spec:
        return Spec(self.d_in, self.tables * self.code_bits, kind, stages, block, depth)


class _SpecC(C.Structure):
    _fields_ = [("d_in", C.c_int64), ("d_out", C.c_int64), ("kind", C.c_int32),
                ("stages", C.c_int64), ("block", C.c_int64), ("depth", C.c_int64)]


class _CfgC(C.Structure):
    _fields_ = [("d_in", C.c_int64), ("d_out", C.c_int64), ("tables", C.c_int64),
                ("code_bits", C.c_int64), ("variant", C.c_int32), ("neighbor_count", C.c_int64)]


class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


def _spec_c(s: Spec) -> _SpecC:
    return _SpecC(s.d_in, s.d_out, s.kind, s.stages, s.block, s.depth)


def _cfg_c(c: Cfg) -> _CfgC:
    return _CfgC(c.d_in, c.d_out, c.tables, c.code_bits, c.variant, c.neighbor_count)


class Oracle:
    """The plain-C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = self.lib = C.CDLL(path)
        L.orc_rng_seed.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.orc_rng_next.argtypes = [C.POINTER(_Rng)]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_fill_gaussian.argtypes = [C.POINTER(_Rng), _f64, C.c_size_t, C.c_double]
        L.orc_fill_signs.argtypes = [C.POINTER(_Rng), _f64, C.c_size_t]
        L.orc_proj_init.argtypes = [C.POINTER(_SpecC), C.c_uint64, _f64]
        L.orc_proj_forward.argtypes = [C.POINTER(_SpecC), _f64, _f64, C.c_size_t, _f64]
        L.orc_fwht.argtypes = [_f64, C.c_size_t]
        L.orc_sign_code.argtypes = [_f64, C.c_size_t]
        L.orc_sign_code.restype = C.c_uint32
        L.orc_compute_codes.argtypes = [_f64, C.c_size_t, C.c_size_t, C.c_size_t, _u32, C.c_void_p]
        L.orc_top1_weight.argtypes = [_f64, C.c_size_t]
        L.orc_top1_weight.restype = C.c_double
        L.orc_log_denominator.argtypes = [_f64, C.c_size_t]
        L.orc_log_denominator.restype = C.c_double
        L.orc_code_dot.argtypes = [_f64, C.c_size_t, C.c_uint32]
        L.orc_code_dot.restype = C.c_double
        L.orc_neighbor_codes.argtypes = [_f64, C.c_size_t, C.c_size_t, _u32]
        L.orc_neighbor_codes.restype = C.c_size_t
        L.orc_lookup_forward.argtypes = [C.POINTER(_CfgC), C.POINTER(_SpecC), _f64, _f64, _f64,
                                         C.c_size_t, _f64, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        L.orc_gather.argtypes = [_f64, C.c_size_t, C.c_size_t, C.c_size_t, _u32, _f64,
                                 C.c_size_t, _f64]
        L.orc_proj_backward.argtypes = [C.POINTER(_SpecC), _f64, _f64, C.c_size_t, _f64, _f64,
                                        _f64]
        L.orc_lookup_backward.argtypes = [C.POINTER(_CfgC), C.POINTER(_SpecC), _f64, _f64, _f64,
                                          C.c_size_t, _f64, _f64, _f64, _f64, C.c_void_p]

    # RNG -----------------------------------------------------------------
    def rng(self, seed: int):
        r = _Rng()
        self.lib.orc_rng_seed(C.byref(r), seed)
        return r

    def gaussian(self, seed_or_rng, n: int, std: float = 1.0) -> np.ndarray:
        r = self.rng(seed_or_rng) if isinstance(seed_or_rng, int) else seed_or_rng
        out = np.empty(n, np.float64)
        self.lib.orc_fill_gaussian(C.byref(r), out, n, std)
        return out

    def signs(self, seed: int, n: int) -> np.ndarray:
        r = self.rng(seed)
        out = np.empty(n, np.float64)
        self.lib.orc_fill_signs(C.byref(r), out, n)
        return out

    # projection ----------------------------------------------------------
    def proj_init(self, s: Spec, seed: int) -> np.ndarray:
        blob = np.empty(s.blob_size(), np.float64)
        if self.lib.orc_proj_init(C.byref(_spec_c(s)), seed, blob) != 0:
            raise ValueError("SizeError: invalid projection spec")
        return blob

    def proj_forward(self, s: Spec, blob: np.ndarray, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[0]
        z = np.empty((n, s.d_out), np.float64)
        rc = self.lib.orc_proj_forward(C.byref(_spec_c(s)), np.ascontiguousarray(blob, np.float64),
                                       x, n, z)
        if rc:
            raise ArithmeticError(f"projection forward rc={rc}")
        return z

    def fwht(self, v: np.ndarray) -> np.ndarray:
        v = np.array(v, np.float64)
        self.lib.orc_fwht(v, v.size)
        return v

    # codes ---------------------------------------------------------------
    def sign_code(self, z) -> int:
        z = np.ascontiguousarray(z, np.float64)
        return int(self.lib.orc_sign_code(z, z.size))

    def compute_codes(self, z: np.ndarray, h: int, tau: int):
        z = np.ascontiguousarray(z, np.float64)
        n = z.size // (h * tau)
        codes = np.empty(n * h, np.uint32)
        absz = np.empty(n * h * tau, np.float64)
        self.lib.orc_compute_codes(z, n, h, tau, codes, absz.ctypes.data)
        return codes.reshape(n, h), absz.reshape(n, h, tau)

    def top1_weight(self, absz) -> float:
        a = np.ascontiguousarray(absz, np.float64)
        return float(self.lib.orc_top1_weight(a, a.size))

    def log_denominator(self, z) -> float:
        z = np.ascontiguousarray(z, np.float64)
        return float(self.lib.orc_log_denominator(z, z.size))

    def code_dot(self, z, code: int) -> float:
        z = np.ascontiguousarray(z, np.float64)
        return float(self.lib.orc_code_dot(z, z.size, code))

    def neighbor_codes(self, z, count: int) -> np.ndarray:
        z = np.ascontiguousarray(z, np.float64)
        out = np.empty(max(count, 1), np.uint32)
        k = self.lib.orc_neighbor_codes(z, z.size, count, out)
        if k == 0:
            raise ValueError("SizeError: neighbor count")
        return out[:k]

    # forward -------------------------------------------------------------
    def lookup_forward(self, c: Cfg, s: Spec, blob, tables, x, want_cache: bool = False):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[0]
        y = np.empty((n, c.d_out), np.float64)
        nc = c.neighbor_count
        z = np.empty((n, c.tables * c.code_bits), np.float64) if want_cache else None
        codes = np.empty((n, c.tables, nc), np.uint32) if want_cache else None
        w = np.empty((n, c.tables, nc), np.float64) if want_cache else None
        dots = np.empty((n, c.tables, nc), np.float64) if want_cache else None
        ptr = (lambda a: None if a is None else a.ctypes.data)
        rc = self.lib.orc_lookup_forward(C.byref(_cfg_c(c)), C.byref(_spec_c(s)),
                                         np.ascontiguousarray(blob, np.float64),
                                         np.ascontiguousarray(tables, np.float64), x, n, y,
                                         ptr(z), ptr(codes), ptr(w), ptr(dots))
        if rc == 1:
            raise ValueError("SizeError: lookup forward shape/config")
        if rc == 2:
            raise ArithmeticError("NumericError: non-finite values")
        if want_cache:
            return y, dict(z=z, codes=codes, weights=w, dots=dots)
        return y

    def gather(self, tables, h, rows, d_out, codes, coeff) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.uint32)
        n = codes.size // h
        y = np.empty((n, d_out), np.float64)
        self.lib.orc_gather(np.ascontiguousarray(tables, np.float64), h, rows, d_out, codes,
                            np.ascontiguousarray(coeff, np.float64), n, y)
        return y

    @staticmethod
    def param_count(s: Spec) -> int:
        # Projection::param_count (projection.cpp:159-161): none for signflip
        return 0 if s.kind == SIGNFLIP else s.blob_size()

    def proj_backward(self, s: Spec, blob, x, grad_out):
        """Projection::backward (projection.cpp:279-386) -> (grad_x, grad_params)."""
        x = np.ascontiguousarray(x, np.float64)
        go = np.ascontiguousarray(grad_out, np.float64)
        n = x.shape[0]
        gx = np.empty((n, s.d_in), np.float64)
        gp = np.zeros(max(self.param_count(s), 1), np.float64)
        rc = self.lib.orc_proj_backward(C.byref(_spec_c(s)), np.ascontiguousarray(blob, np.float64),
                                        x, n, go, gx, gp)
        if rc == 1:
            raise ValueError("SizeError: projection backward")
        if rc == 2:
            raise ArithmeticError("NumericError: projection backward")
        return gx, gp[:self.param_count(s)]

    def lookup_backward(self, c: Cfg, s: Spec, blob, tables, x, grad_y):
        """lookup_backward (lookup.cpp:292-347) -> dict(grad_x, grad_tables,
        grad_proj, grad_z)."""
        x = np.ascontiguousarray(x, np.float64)
        gy = np.ascontiguousarray(grad_y, np.float64)
        n = x.shape[0]
        gx = np.empty((n, c.d_in), np.float64)
        gt = np.zeros(c.tables * (1 << c.code_bits) * c.d_out, np.float64)
        gp = np.zeros(max(self.param_count(s), 1), np.float64)
        gz = np.empty((n, c.tables * c.code_bits), np.float64)
        rc = self.lib.orc_lookup_backward(C.byref(_cfg_c(c)), C.byref(_spec_c(s)),
                                          np.ascontiguousarray(blob, np.float64),
                                          np.ascontiguousarray(tables, np.float64), x, n, gy, gx,
                                          gt, gp, gz.ctypes.data)
        if rc == 1:
            raise ValueError("SizeError: lookup backward")
        if rc == 2:
            raise ArithmeticError("NumericError: lookup backward")
        return dict(grad_x=gx, grad_tables=gt, grad_proj=gp[:self.param_count(s)], grad_z=gz)


class Reference:
    """The reference library itself (oracle/_ref/liblffn_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_fill_gaussian.argtypes = [C.c_uint64, _f64, C.c_size_t, C.c_double]
        L.ref_fill_signs.argtypes = [C.c_uint64, _f64, C.c_size_t]
        L.ref_proj_init.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_uint64, C.c_void_p, C.c_int64]
        L.ref_proj_init.restype = C.c_int64
        L.ref_tables_init.argtypes = [C.c_int64] * 4 + [C.c_uint64, _f64]
        L.ref_fwht.argtypes = [_f64, C.c_size_t]
        L.ref_sign_code.argtypes = [_f64, C.c_size_t]
        L.ref_sign_code.restype = C.c_uint32
        L.ref_log_denominator.argtypes = [_f64, C.c_size_t]
        L.ref_log_denominator.restype = C.c_double
        L.ref_code_dot.argtypes = [_f64, C.c_size_t, C.c_uint32]
        L.ref_code_dot.restype = C.c_double
        L.ref_neighbor_codes.argtypes = [_f64, C.c_size_t, C.c_size_t, _u32]
        L.ref_neighbor_codes.restype = C.c_int64
        L.ref_compute_codes.argtypes = [_f64, C.c_size_t, C.c_size_t, C.c_size_t, _u32, C.c_void_p]
        L.ref_proj_forward.argtypes = [C.c_int] + [C.c_int64] * 5 + [_f64, C.c_int64, _f64,
                                                                     C.c_size_t, _f64]
        L.ref_lookup_forward.argtypes = ([C.c_int64] * 4 + [C.c_int, C.c_int64, C.c_int] +
                                         [C.c_int64] * 3 + [_f64, C.c_int64, _f64, _f64,
                                                            C.c_size_t, _f64] + [C.c_void_p] * 4)
        L.ref_lookup_flops.argtypes = [C.c_int64] * 5 + [C.c_int] + [C.c_int64] * 3 + [_f64]
        L.ref_save_checkpoint.argtypes = ([C.c_char_p] + [C.c_int64] * 4 + [C.c_int, C.c_int] +
                                          [C.c_int64] * 3 + [_f64, C.c_int64, _f64])
        L.ref_load_checkpoint.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_pipeline_f32.argtypes = ([C.c_int64] * 4 + [C.c_int, C.c_int] + [C.c_int64] * 3 +
                                       [_f32, _f32, _f32, C.c_size_t, _f32, C.c_int, C.c_int,
                                        C.c_int])
        L.ref_pipeline_f32.restype = C.c_double
        L.ref_lookup_backward.argtypes = ([C.c_int64] * 4 + [C.c_int, C.c_int64, C.c_int] +
                                          [C.c_int64] * 3 + [_f64, C.c_int64, _f64, _f64,
                                                             C.c_size_t, _f64, _f64, _f64, _f64])
        L.ref_proj_backward.argtypes = ([C.c_int] + [C.c_int64] * 5 + [_f64, C.c_int64, _f64,
                                                                     C.c_size_t, _f64, _f64, _f64])
        L.ref_bench_lookup_ffn.argtypes = ([C.c_int64] * 4 + [C.c_int, C.c_int] + [C.c_int64] * 3 +
                                           [C.c_size_t] * 3 + [C.c_int, C.c_int, C.c_uint64, _f64])

    def _err(self, rc):
        msg = self.lib.ref_last_error().decode()
        if rc == 1:
            raise ValueError("SizeError/UsageError: " + msg)
        if rc == 2:
            raise ArithmeticError("NumericError: " + msg)
        raise RuntimeError(msg)

    def gaussian(self, seed: int, n: int, std: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_fill_gaussian(seed, out, n, std)
        return out

    def signs(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_fill_signs(seed, out, n)
        return out

    def proj_init(self, s: Spec, seed: int) -> np.ndarray:
        blob = np.empty(s.blob_size(), np.float64)
        k = self.lib.ref_proj_init(s.kind, s.d_in, s.d_out, s.stages, s.block, s.depth, seed,
                                   blob.ctypes.data, blob.size)
        if k < 0:
            self._err(1)
        return blob

    def tables_init(self, c: Cfg, seed: int) -> np.ndarray:
        out = np.empty(c.tables * c.rows * c.d_out, np.float64)
        rc = self.lib.ref_tables_init(c.d_in, c.d_out, c.tables, c.code_bits, seed, out)
        if rc:
            self._err(rc)
        return out

    def fwht(self, v) -> np.ndarray:
        v = np.array(v, np.float64)
        self.lib.ref_fwht(v, v.size)
        return v

    def sign_code(self, z) -> int:
        z = np.ascontiguousarray(z, np.float64)
        return int(self.lib.ref_sign_code(z, z.size))

    def log_denominator(self, z) -> float:
        z = np.ascontiguousarray(z, np.float64)
        return float(self.lib.ref_log_denominator(z, z.size))

    def code_dot(self, z, code: int) -> float:
        z = np.ascontiguousarray(z, np.float64)
        return float(self.lib.ref_code_dot(z, z.size, code))

    def neighbor_codes(self, z, count: int) -> np.ndarray:
        z = np.ascontiguousarray(z, np.float64)
        out = np.empty(max(count, 1), np.uint32)
        k = self.lib.ref_neighbor_codes(z, z.size, count, out)
        if k < 0:
            self._err(1)
        return out[:k]

    def compute_codes(self, z, h: int, tau: int):
        z = np.ascontiguousarray(z, np.float64)
        n = z.size // (h * tau)
        codes = np.empty(n * h, np.uint32)
        absz = np.empty(n * h * tau, np.float64)
        rc = self.lib.ref_compute_codes(z, n, h, tau, codes, absz.ctypes.data)
        if rc:
            self._err(rc)
        return codes.reshape(n, h), absz.reshape(n, h, tau)

    def proj_forward(self, s: Spec, blob, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[0]
        z = np.empty((n, s.d_out), np.float64)
        blob = np.ascontiguousarray(blob, np.float64)
        rc = self.lib.ref_proj_forward(s.kind, s.d_in, s.d_out, s.stages, s.block, s.depth, blob,
                                       blob.size, x, n, z)
        if rc:
            self._err(rc)
        return z

    def lookup_forward(self, c: Cfg, s: Spec, blob, tables, x, want_cache: bool = False):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[0]
        y = np.empty((n, c.d_out), np.float64)
        nc = c.neighbor_count
        z = np.empty((n, c.tables * c.code_bits), np.float64) if want_cache else None
        codes = np.empty((n, c.tables, nc), np.uint32) if want_cache else None
        w = np.empty((n, c.tables, nc), np.float64) if want_cache else None
        dots = np.empty((n, c.tables, nc), np.float64) if want_cache else None
        ptr = (lambda a: None if a is None else a.ctypes.data)
        blob = np.ascontiguousarray(blob, np.float64)
        rc = self.lib.ref_lookup_forward(c.d_in, c.d_out, c.tables, c.code_bits, c.variant,
                                         c.neighbor_count, s.kind, s.stages, s.block, s.depth,
                                         blob, blob.size, np.ascontiguousarray(tables, np.float64),
                                         x, n, y, ptr(z), ptr(codes), ptr(w), ptr(dots))
        if rc:
            self._err(rc)
        if want_cache:
            return y, dict(z=z, codes=codes, weights=w, dots=dots)
        return y

    def proj_backward(self, s: Spec, blob, x, grad_out):
        x = np.ascontiguousarray(x, np.float64)
        go = np.ascontiguousarray(grad_out, np.float64)
        n = x.shape[0]
        blob = np.ascontiguousarray(blob, np.float64)
        gx = np.empty((n, s.d_in), np.float64)
        pc = Oracle.param_count(s)
        gp = np.zeros(max(pc, 1), np.float64)
        rc = self.lib.ref_proj_backward(s.kind, s.d_in, s.d_out, s.stages, s.block, s.depth, blob,
                                        blob.size, x, n, go, gx, gp)
        if rc:
            self._err(rc)
        return gx, gp[:pc]

    def lookup_backward(self, c: Cfg, s: Spec, blob, tables, x, grad_y):
        x = np.ascontiguousarray(x, np.float64)
        gy = np.ascontiguousarray(grad_y, np.float64)
        n = x.shape[0]
        blob = np.ascontiguousarray(blob, np.float64)
        gx = np.empty((n, c.d_in), np.float64)
        gt = np.zeros(c.tables * (1 << c.code_bits) * c.d_out, np.float64)
        pc = Oracle.param_count(s)
        gp = np.zeros(max(pc, 1), np.float64)
        rc = self.lib.ref_lookup_backward(c.d_in, c.d_out, c.tables, c.code_bits, c.variant,
                                          c.neighbor_count, s.kind, s.stages, s.block, s.depth,
                                          blob, blob.size, np.ascontiguousarray(tables, np.float64),
                                          x, n, gy, gx, gt, gp)
        if rc:
            self._err(rc)
        return dict(grad_x=gx, grad_tables=gt, grad_proj=gp[:pc])

    def save_checkpoint(self, path: str, c: Cfg, s: Spec, blob, tables) -> None:
        blob = np.ascontiguousarray(blob, np.float64)
        rc = self.lib.ref_save_checkpoint(os.fsencode(path), c.d_in, c.d_out, c.tables,
                                          c.code_bits, c.variant, s.kind, s.stages, s.block,
                                          s.depth, blob, blob.size,
                                          np.ascontiguousarray(tables, np.float64))
        if rc:
            self._err(rc)

    def load_checkpoint(self, path: str):
        """-> (header dict, blob, tables) through the reference's load_checkpoint."""
        hdr = np.zeros(8, np.int64)
        rc = self.lib.ref_load_checkpoint(os.fsencode(path), hdr.ctypes.data, None, None)
        if rc:
            self._err(rc)
        keys = ["d_in", "d_out", "tables", "code_bits", "variant", "kind", "m", "b"]
        h = dict(zip(keys, hdr.tolist()))
        c = Cfg(h["d_in"], h["d_out"], h["tables"], h["code_bits"], h["variant"])
        s = c.spec(h["kind"], stages=h["m"] if h["kind"] == BH else 4, block=h["b"],
                   depth=h["m"] if h["kind"] == ACDC else 1)
        blob = np.empty(s.blob_size(), np.float64)
        T = np.empty(c.tables * c.rows * c.d_out, np.float64)
        rc = self.lib.ref_load_checkpoint(os.fsencode(path), hdr.ctypes.data, blob.ctypes.data,
                                          T.ctypes.data)
        if rc:
            self._err(rc)
        return h, blob, T

    def lookup_flops(self, c: Cfg, s: Spec):
        out = np.zeros(3, np.float64)
        rc = self.lib.ref_lookup_flops(c.d_in, c.d_out, c.tables, c.code_bits, c.neighbor_count,
                                       s.kind, s.stages, s.block, s.depth, out)
        if rc:
            self._err(rc)
        return tuple(out)

    def pipeline_f32(self, c: Cfg, s: Spec, blob32, tables32, x32, threads: int = 1,
                     sorted_gather: bool = False, reps: int = 1):
        """Reference float32 inference kernels (bench.cpp:115-217); returns (y, ms)."""
        x32 = np.ascontiguousarray(x32, np.float32)
        n = x32.shape[0]
        y = np.zeros((n, c.d_out), np.float32)
        ms = self.lib.ref_pipeline_f32(c.d_in, c.d_out, c.tables, c.code_bits, c.variant, s.kind,
                                       s.stages, s.block, s.depth,
                                       np.ascontiguousarray(blob32, np.float32),
                                       np.ascontiguousarray(tables32, np.float32), x32, n, y,
                                       threads, int(sorted_gather), reps)
        return y, ms

    def bench_lookup_ffn(self, c: Cfg, s: Spec, rows: int, reps: int = 3, warmup: int = 1,
                         threads: int = 1, sorted_gather: bool = False, seed: int = 0) -> dict:
        out = np.zeros(8, np.float64)
        rc = self.lib.ref_bench_lookup_ffn(c.d_in, c.d_out, c.tables, c.code_bits, c.variant,
                                           s.kind, s.stages, s.block, s.depth, rows, reps, warmup,
                                           threads, int(sorted_gather), seed, out)
        if rc:
            self._err(rc)
        keys = ["median_ms", "mean_ms", "hash_ms", "gather_ms", "other_ms", "mflop_per_token",
                "gflops", "timed_allocs"]
        return dict(zip(keys, out.tolist()))
