"""Host-side mirror of the reference's lookup API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/lookupffn/{lookup,projection,common}.hpp) so that
the reference's forward-path tests read the same against this package:

=====================================  =========================================
reference                               here
=====================================  =========================================
``LookupConfig`` (lookup.hpp:25-39)     ``LookupConfig``
``LookupVariant`` (lookup.hpp:20)       ``LookupVariant``
``ProjKind`` / ``ProjectionSpec``        ``ProjKind`` / ``ProjectionSpec``
  (projection.hpp:13-37)
``Projection::init / from_blob``        ``Projection.init / from_blob``
  (projection.hpp:55-95)
``HashTables::init / zeros_like /``     ``HashTables`` (same methods)
  ``row / checksum`` (lookup.hpp:43-66)
``lookup_forward`` (lookup.hpp:124)     ``lookup_forward`` (device; nc == 1)
``SizeError / UsageError /``            ``SizeError / UsageError / NumericError``
  ``NumericError`` (common.hpp:17-29)
=====================================  =========================================

Everything numeric runs in liblffn_gpu.so on the GPU; parameter generation
uses the reference's own engine and libstdc++ distributions (host C++ inside
the same library), so seeds give bit-identical parameters.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from ._capi import LFFN_BF16, LFFN_F32, LFFN_F64, NumericError, SizeError, UsageError, check

__all__ = [
    "LookupVariant", "ProjKind", "LookupConfig", "ProjectionSpec", "Projection", "HashTables",
    "LookupFFN", "lookup_forward", "fill_gaussian", "fill_signs", "gaussian_matrix",
    "checkpoint_header", "load_checkpoint", "save_checkpoint",
    "to_bf16_values", "SizeError", "UsageError", "NumericError",
]


class LookupVariant(enum.IntEnum):
    softmax = 0
    scaled = 1
    sigmoid_tau1 = 2
    gelu_tau1 = 3


class ProjKind(enum.IntEnum):
    dense = 0
    bh = 1
    acdc = 2
    signflip = 3


def _next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p <<= 1
    return p


@dataclass
class LookupConfig:
    d_in: int = 0
    d_out: int = 0
    tables: int = 1
    code_bits: int = 1
    variant: LookupVariant = LookupVariant.softmax
    neighbor_count: int = 1

    def code_width(self) -> int:
        return self.tables * self.code_bits

    def table_rows(self) -> int:
        return 1 << self.code_bits

    def scaled_numerator(self) -> bool:
        return self.variant in (LookupVariant.scaled, LookupVariant.gelu_tau1)

    def _c(self) -> _capi.lffn_cfg:
        return _capi.lffn_cfg(self.d_in, self.d_out, self.tables, self.code_bits, int(self.variant),
                              self.neighbor_count)

    def validate(self) -> None:
        check(_capi.lib().lffn_cfg_validate(C.byref(self._c())))


@dataclass
class ProjectionSpec:
    d_in: int = 0
    d_out: int = 0
    kind: ProjKind = ProjKind.dense
    stages: int = 4
    block: int = 0
    depth: int = 1

    def transform_width(self) -> int:
        return _next_pow2(max(self.d_in, self.d_out))

    def _c(self, blob: Optional[np.ndarray] = None) -> _capi.lffn_proj:
        p = _capi.lffn_proj(int(self.kind), 0, self.d_in, self.d_out, self.stages, self.block,
                            self.depth, None, 0)
        if blob is not None:
            p.blob = blob.ctypes.data_as(C.POINTER(C.c_double))
            p.blob_len = blob.size
        return p

    def validate(self) -> None:
        check(_capi.lib().lffn_proj_validate(C.byref(self._c())))

    def blob_size(self) -> int:
        n = _capi.lib().lffn_proj_blob_size(C.byref(self._c()))
        if n < 0:
            check(_capi.LFFN_ERR_USAGE)
        return int(n)

    @staticmethod
    def dense(d_in: int, d_out: int) -> "ProjectionSpec":
        return ProjectionSpec(d_in, d_out, ProjKind.dense)

    @staticmethod
    def bh(d_in: int, d_out: int, m: int, b: int) -> "ProjectionSpec":
        return ProjectionSpec(d_in, d_out, ProjKind.bh, stages=m, block=b)

    @staticmethod
    def acdc(d_in: int, d_out: int, k: int) -> "ProjectionSpec":
        return ProjectionSpec(d_in, d_out, ProjKind.acdc, depth=k)

    @staticmethod
    def signflip(d_in: int, d_out: int) -> "ProjectionSpec":
        return ProjectionSpec(d_in, d_out, ProjKind.signflip)


@dataclass
class Projection:
    """A projection spec plus its float64 parameter blob (projection.hpp:47-54)."""

    spec: ProjectionSpec
    blob: np.ndarray = field(repr=False)

    @staticmethod
    def init(spec: ProjectionSpec, seed: int) -> "Projection":
        spec.validate()
        blob = np.empty(spec.blob_size(), np.float64)
        check(_capi.lib().lffn_proj_init(C.byref(spec._c()), seed, blob.ctypes.data))
        return Projection(spec, blob)

    @staticmethod
    def from_blob(spec: ProjectionSpec, blob) -> "Projection":
        blob = np.ascontiguousarray(blob, np.float64).reshape(-1)
        check(_capi.lib().lffn_proj_validate(C.byref(spec._c(blob))))
        return Projection(spec, blob)

    def params(self) -> np.ndarray:
        return self.blob[:0] if self.spec.kind == ProjKind.signflip else self.blob

    def _c(self) -> _capi.lffn_proj:
        return self.spec._c(self.blob)


@dataclass
class HashTables:
    """T, shape h x 2^tau x d_out, float64 host copy (lookup.hpp:43-66)."""

    tables: int
    code_bits: int
    d_out: int
    data: np.ndarray = field(repr=False)

    def rows_per_table(self) -> int:
        return 1 << self.code_bits

    def row(self, k: int, code: int) -> np.ndarray:
        r = self.rows_per_table()
        o = (k * r + code) * self.d_out
        return self.data[o:o + self.d_out]

    @staticmethod
    def init(cfg: LookupConfig, seed: int) -> "HashTables":
        cfg.validate()
        data = np.empty(cfg.tables * cfg.table_rows() * cfg.d_out, np.float64)
        check(_capi.lib().lffn_tables_init(C.byref(cfg._c()), seed, data.ctypes.data))
        return HashTables(cfg.tables, cfg.code_bits, cfg.d_out, data)

    @staticmethod
    def zeros_like(cfg: LookupConfig) -> "HashTables":
        return HashTables(cfg.tables, cfg.code_bits, cfg.d_out,
                          np.zeros(cfg.tables * cfg.table_rows() * cfg.d_out, np.float64))

    def checksum(self) -> int:
        """FNV-1a over the raw float64 bytes (lookup.cpp:60-68)."""
        h = 1469598103934665603
        for b in self.data.tobytes():
            h ^= b
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h


@dataclass
class TableSlice:
    """Tables [kb, ke) of a stack, float64 host copy: what a table shard
    uploads (``LookupFFN(..., table_range=(kb, ke))``)."""

    table_range: tuple
    code_bits: int
    d_out: int
    data: np.ndarray = field(repr=False)


def fill_gaussian_slice(seed: int, skip: int, n: int, stddev: float = 1.0) -> np.ndarray:
    """Elements [skip, skip + n) of make_rng(seed) + fill_gaussian."""
    out = np.empty(n, np.float64)
    check(_capi.lib().lffn_fill_gaussian_slice(seed, skip, out.ctypes.data, n, stddev))
    return out


def fill_gaussian(seed: int, n: int, stddev: float = 1.0) -> np.ndarray:
    """make_rng(seed) + fill_gaussian (common.hpp:44-49), bit-identical."""
    out = np.empty(n, np.float64)
    check(_capi.lib().lffn_fill_gaussian(seed, out.ctypes.data, n, stddev))
    return out


def fill_signs(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    check(_capi.lib().lffn_fill_signs(seed, out.ctypes.data, n))
    return out


def gaussian_matrix(rows: int, cols: int, seed: int, stddev: float = 1.0) -> np.ndarray:
    """DenseMatrix::gaussian(rows, cols, make_rng(seed), stddev) (matrix.hpp:37-42)."""
    return fill_gaussian(seed, rows * cols, stddev).reshape(rows, cols)


def to_bf16_values(a: np.ndarray) -> np.ndarray:
    """The float64 values a bf16 table upload stores (single RNE rounding)."""
    a = np.ascontiguousarray(a, np.float64).reshape(-1)
    bits = np.empty(a.size, np.uint16)
    check(_capi.lib().lffn_convert(a.ctypes.data, LFFN_F64, bits.ctypes.data, LFFN_BF16, a.size))
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def checkpoint_header(path: str):
    """(LookupConfig, ProjectionSpec, tables_len) of an "LFFN" v1 checkpoint."""
    c, p, nt = _capi.lffn_cfg(), _capi.lffn_proj(), C.c_int64()
    check(_capi.lib().lffn_checkpoint_header(os.fsencode(path), C.byref(c), C.byref(p),
                                             C.byref(nt)))
    cfg = LookupConfig(c.d_in, c.d_out, c.tables, c.code_bits, LookupVariant(c.variant),
                       c.neighbor_count)
    spec = ProjectionSpec(p.d_in, p.d_out, ProjKind(p.kind), p.stages, p.block, p.depth)
    return cfg, spec, int(nt.value)


def load_checkpoint(path: str):
    """load_checkpoint (checkpoint.cpp:86-138) -> (cfg, Projection, HashTables)."""
    cfg, spec, nt = checkpoint_header(path)
    blob = np.empty(spec.blob_size(), np.float64)
    data = np.empty(nt, np.float64)
    check(_capi.lib().lffn_checkpoint_load(os.fsencode(path), blob.ctypes.data, data.ctypes.data))
    return cfg, Projection(spec, blob), HashTables(cfg.tables, cfg.code_bits, cfg.d_out, data)


def save_checkpoint(path: str, cfg: LookupConfig, proj: Projection, tables: HashTables) -> None:
    """save_checkpoint (checkpoint.cpp:52-84): the reference's "LFFN" v1 format."""
    data = np.ascontiguousarray(tables.data, np.float64)
    check(_capi.lib().lffn_checkpoint_save(os.fsencode(path), C.byref(cfg._c()),
                                           C.byref(proj._c()), data.ctypes.data))


_DTYPES = {"f32": LFFN_F32, "float32": LFFN_F32, "bf16": LFFN_BF16, "bfloat16": LFFN_BF16}


class LookupFFN:
    """A device-resident LookupFFN layer: one lffn_ctx on one GPU.

    ``table_range=(kb, ke)`` makes a table shard (multi-GPU table sharding):
    the layer then produces the partial sum over tables [kb, ke).
    """

    def __init__(self, cfg: LookupConfig, proj: Projection, tables, *, device: int = 0,
                 max_tokens: int = 65536, table_dtype: str = "f32",
                 table_range: Optional[tuple] = None):
        cfg.validate()
        self.cfg, self.proj, self.device = cfg, proj, device
        self.max_tokens = max_tokens
        self.table_dtype = _DTYPES[table_dtype]
        L = _capi.lib()
        ctx = C.c_void_p()
        kb, ke = table_range if table_range is not None else (0, cfg.tables)
        check(L.lffn_ctx_create_shard(C.byref(ctx), device, max_tokens, C.byref(cfg._c()),
                                      C.byref(proj._c()), kb, ke))
        self._ctx = ctx
        self.table_range = (kb, ke)
        if tables is not None:
            self.upload_tables(tables)

    @classmethod
    def _view(cls, ctx, cfg: LookupConfig, proj, table_range: tuple, *, device: int = 0,
              max_tokens: int = 65536, table_dtype: str = "f32") -> "LookupFFN":
        """A non-owning layer over a context another object owns (the shard
        context of an lffn_group)."""
        self = cls.__new__(cls)
        self.cfg, self.proj, self.device = cfg, proj, device
        self.max_tokens = max_tokens
        self.table_dtype = _DTYPES[table_dtype]
        self._ctx = C.c_void_p(ctx)
        self._owned = False
        self.table_range = tuple(table_range)
        return self

    @classmethod
    def from_checkpoint(cls, path: str, *, device: int = 0, max_tokens: int = 65536,
                        table_dtype: str = "f32",
                        table_range: Optional[tuple] = None) -> "LookupFFN":
        """A layer straight from an "LFFN" v1 checkpoint (load_checkpoint,
        checkpoint.cpp:86-138); the tables stream from the file to the GPU."""
        cfg, spec, _ = checkpoint_header(path)
        self = cls.__new__(cls)
        self.cfg, self.proj, self.device = cfg, spec, device
        self.max_tokens = max_tokens
        self.table_dtype = _DTYPES[table_dtype]
        kb, ke = table_range if table_range is not None else (0, cfg.tables)
        ctx = C.c_void_p()
        check(_capi.lib().lffn_ctx_create_from_checkpoint(C.byref(ctx), device, max_tokens,
                                                          os.fsencode(path), self.table_dtype,
                                                          kb, ke))
        self._ctx = ctx
        self.table_range = (kb, ke)
        return self

    # -- tables ----------------------------------------------------------
    def upload_tables(self, tables) -> None:
        """Upload the FULL h x 2^tau x d_out stack (HashTables or ndarray)."""
        data = tables.data if isinstance(tables, (HashTables, TableSlice)) else tables
        if hasattr(data, "detach"):
            data = data.detach().cpu().numpy()
        data = np.ascontiguousarray(data)
        per_table = self.cfg.table_rows() * self.cfg.d_out
        expect = self.cfg.tables * per_table
        kb, ke = self.table_range
        sliced = isinstance(tables, TableSlice) or (data.size != expect and
                                                    data.size == (ke - kb) * per_table)
        if sliced and (data.size != (ke - kb) * per_table or
                       (isinstance(tables, TableSlice) and tables.table_range != (kb, ke))):
            raise SizeError("lookup forward: table slice does not match the layer's table range")
        if not sliced and data.size != expect:
            raise SizeError("lookup forward: table stack shape mismatch")
        if data.dtype == np.float64:
            host = LFFN_F64
        elif data.dtype == np.float32:
            host = LFFN_F32
        elif data.dtype == np.uint16:
            host = LFFN_BF16
        else:
            raise UsageError(f"unsupported table dtype {data.dtype}")
        up = _capi.lib().lffn_tables_upload_slice if sliced else _capi.lib().lffn_tables_upload
        check(up(self._ctx, data.ctypes.data, host, self.table_dtype))

    def attach_tables(self, dev_tensor) -> None:
        """Use a caller-owned device tensor holding this shard's slice (no copy)."""
        import torch

        dt = LFFN_F32 if dev_tensor.dtype == torch.float32 else LFFN_BF16
        self._tables_ref = dev_tensor
        self.table_dtype = dt
        check(_capi.lib().lffn_tables_attach(self._ctx, dev_tensor.data_ptr(), dt))

    # -- device-pointer API (torch tensors on this GPU) -----------------
    @staticmethod
    def _stream(stream) -> int:
        if stream is None:
            import torch

            return torch.cuda.current_stream().cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def hash(self, x, codes=None, coeff=None, z=None, stream=None):
        """lffn_hash on device tensors; returns (codes, coeff[, z]).  Shapes
        [n, h_loc] for the top-1 default, [n, h_loc, nc] for neighbor_count nc
        > 1 (the reference cache's slot order (i*h + k)*nc + c)."""
        import torch

        n = x.shape[0]
        hl = self.table_range[1] - self.table_range[0]
        nc = self.cfg.neighbor_count
        shape = (n, hl) if nc == 1 else (n, hl, nc)
        dev = x.device
        if codes is None:
            codes = torch.empty(shape, dtype=torch.int32, device=dev)
        if coeff is None:
            coeff = torch.empty(shape, dtype=torch.float32, device=dev)
        zp = z.data_ptr() if z is not None else None
        check(_capi.lib().lffn_hash(self._ctx, x.data_ptr(), n, codes.data_ptr(), coeff.data_ptr(),
                                    zp, self._stream(stream)))
        return (codes, coeff) if z is None else (codes, coeff, z)

    def lookup_accumulate(self, codes, coeff, y, accumulate: bool = False, stream=None):
        n = codes.shape[0]
        check(_capi.lib().lffn_lookup_accumulate(self._ctx, codes.data_ptr(), coeff.data_ptr(), n,
                                                 y.data_ptr(), int(accumulate),
                                                 self._stream(stream)))
        return y

    def forward_device(self, x, y=None, stream=None):
        import torch

        if y is None:
            y = torch.empty((x.shape[0], self.cfg.d_out), dtype=torch.float32, device=x.device)
        check(_capi.lib().lffn_forward(self._ctx, x.data_ptr(), x.shape[0], y.data_ptr(),
                                       self._stream(stream)))
        return y

    def backward(self, x, grad_y, want_x: bool = True, want_tables: bool = True,
                 want_proj: bool = True, stream=None):
        """lffn_backward (lookup_backward, lookup.cpp:292-347, + Projection::
        backward) on device tensors: returns dict(grad_x [n, d_in] float64,
        grad_tables [h_loc, 2^tau, d_out] float32, grad_proj float64 in the
        blob layout (dense: [d_in, h*tau]; signflip: empty))."""
        import torch

        n = x.shape[0]
        dev = x.device
        cfg = self.cfg
        hl = self.table_range[1] - self.table_range[0]
        gx = torch.empty((n, cfg.d_in), dtype=torch.float64, device=dev) if want_x else None
        gt = (torch.empty((hl, cfg.table_rows(), cfg.d_out), dtype=torch.float32, device=dev)
              if want_tables else None)
        gp = self._grad_proj_buffer(dev) if want_proj else None
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        check(_capi.lib().lffn_backward(self._ctx, x.data_ptr(), grad_y.data_ptr(), n, ptr(gx),
                                        ptr(gt), ptr(gp), self._stream(stream)))
        return dict(grad_x=gx, grad_tables=gt,
                    grad_proj=gp if gp is not None else torch.empty(0, dtype=torch.float64, device=dev))

    def proj_backward(self, x, grad_z, stream=None):
        """lffn_proj_backward (Projection::backward, projection.cpp:279-386)
        for a float64 grad_z [n, h*tau]: (grad_x float64, grad_proj float64)."""
        import torch

        n = x.shape[0]
        cfg = self.cfg
        gx = torch.empty((n, cfg.d_in), dtype=torch.float64, device=x.device)
        gp = self._grad_proj_buffer(x.device)
        check(_capi.lib().lffn_proj_backward(self._ctx, x.data_ptr(), grad_z.data_ptr(), n,
                                             gx.data_ptr(), gp.data_ptr() if gp is not None else None,
                                             self._stream(stream)))
        return gx, (gp if gp is not None else torch.empty(0, dtype=torch.float64, device=x.device))

    def _grad_proj_buffer(self, dev):
        """Projection::param_count (projection.cpp:159-161) float64 entries in the
        blob layout (dense [d_in, h*tau]); None for signflip."""
        import torch

        spec = self.proj.spec if hasattr(self.proj, "spec") else self.proj
        if spec.kind == ProjKind.signflip:
            return None
        if spec.kind == ProjKind.dense:
            return torch.empty((spec.d_in, spec.d_out), dtype=torch.float64, device=dev)
        return torch.empty(spec.blob_size(), dtype=torch.float64, device=dev)

    def sync(self, stream=None) -> None:
        check(_capi.lib().lffn_sync(self._ctx, self._stream(stream)))

    # -- host API (the reference's call shape) ---------------------------
    def forward(self, x: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """y = lookup_forward(x) with host float32 buffers (H2D/D2H inside)."""
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2 or x.shape[1] != self.cfg.d_in:
            raise SizeError("lookup forward: input width mismatch")
        if out is None:
            out = np.empty((x.shape[0], self.cfg.d_out), np.float32)
        check(_capi.lib().lffn_forward_host(self._ctx, x.ctypes.data, x.shape[0], out.ctypes.data))
        return out

    def forward_host_ptr(self, x_ptr: int, n: int, y_ptr: int) -> None:
        check(_capi.lib().lffn_forward_host(self._ctx, x_ptr, n, y_ptr))

    def set_option(self, name: str, value: int) -> None:
        """'dense_exact' (exact float64 dense projection instead of the
        tcgen05 split-precision GEMM), 'table_group_bytes', 'gather_variant'
        (0 default, -1 one warp per token always), 'bf16_coeff_fma' (0 =
        never take the exact mixed-precision FMA path for bf16 tables),
        'bwd_one_pass' (single-pass backward table-row dot), 'hash_exact' (1 =
        the signflip hash always in the reference's stage order, z
        bit-identical), 'host_chunks' (forward_host pipeline chunks), 'host_direct'
        (0 = small batches through the CUDA-graph copy path) or
        'small_max_tokens' (one-launch forward for batches up to this size)."""
        opt = {"dense_exact": _capi.LFFN_OPT_DENSE_EXACT,
               "table_group_bytes": _capi.LFFN_OPT_TABLE_GROUP_BYTES,
               "gather_variant": _capi.LFFN_OPT_GATHER_VARIANT,
               "bf16_coeff_fma": _capi.LFFN_OPT_BF16_COEFF_FMA,
               "bwd_one_pass": _capi.LFFN_OPT_BWD_ONE_PASS,
               "hash_exact": _capi.LFFN_OPT_HASH_EXACT,
               "host_chunks": _capi.LFFN_OPT_HOST_CHUNKS,
               "small_max_tokens": _capi.LFFN_OPT_SMALL_MAX_TOKENS,
               "gather_sms": _capi.LFFN_OPT_GATHER_SMS,
               "host_direct": _capi.LFFN_OPT_HOST_DIRECT}[name]
        check(_capi.lib().lffn_ctx_set_option(self._ctx, opt, int(value)))

    def launch_count(self) -> int:
        return int(_capi.lib().lffn_ctx_launch_count(self._ctx))

    def set_timing(self, on: bool) -> None:
        check(_capi.lib().lffn_ctx_set_timing(self._ctx, int(on)))

    def stage_ms(self):
        a, b = C.c_float(), C.c_float()
        check(_capi.lib().lffn_ctx_stage_ms(self._ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            if getattr(self, "_owned", True):
                _capi.lib().lffn_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lookup_forward(x, proj: Projection, tables: HashTables, cfg: LookupConfig,
                   cache=None, *, device: int = 0, table_dtype: str = "f32") -> np.ndarray:
    """Drop-in for lffn::lookup_forward (lookup.hpp:124-125), top-1 only.

    Returns y as float64 (the reference returns a DenseMatrix of doubles); the
    device computes it with fp32 tables/accumulators.  ``cache`` is the
    reference's training-only LookupCache and is rejected, as is nc > 1:
    there is no CPU fallback.
    """
    if cache is not None:
        raise UsageError("lookup forward: LookupCache (training) is not supported on the device path")
    cfg.validate()
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[1] != cfg.d_in:
        raise SizeError("lookup forward: input width mismatch")
    if proj.spec.d_in != cfg.d_in or proj.spec.d_out != cfg.code_width():
        raise SizeError("lookup forward: projection must map d_in to h*tau")
    if (tables.tables, tables.code_bits, tables.d_out) != (cfg.tables, cfg.code_bits, cfg.d_out):
        raise SizeError("lookup forward: table stack shape mismatch")
    layer = LookupFFN(cfg, proj, tables, device=device, max_tokens=max(1, x.shape[0]),
                      table_dtype=table_dtype)
    try:
        y = layer.forward(np.ascontiguousarray(x, np.float32))
    finally:
        layer.close()
    return y.astype(np.float64)
