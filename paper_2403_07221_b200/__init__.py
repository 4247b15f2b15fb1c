"""B200-native LookupFFN forward (arXiv 2403.07221) behind the reference's API.

The hot path -- hash (projection -> sign codes -> top-1 coefficients) and
gather-accumulate -- runs in hand-written sm_100a kernels in
``csrc/liblffn_gpu.so`` behind the C-ABI of ``include/lffn_gpu.h``.  This
package is the host-side mirror of the reference's C++ interface
(``lookup``), its cost model (``flops``) and the multi-GPU driver
(``sharded``).
"""
from . import flops
from ._capi import LffnError, NumericError, SizeError, UsageError
from .lookup import (
    HashTables,
    LookupConfig,
    LookupFFN,
    LookupVariant,
    Projection,
    ProjectionSpec,
    ProjKind,
    TableSlice,
    checkpoint_header,
    fill_gaussian,
    fill_gaussian_slice,
    fill_signs,
    gaussian_matrix,
    load_checkpoint,
    lookup_forward,
    save_checkpoint,
    to_bf16_values,
)

__all__ = [
    "HashTables", "LookupConfig", "LookupFFN", "LookupVariant", "Projection", "ProjectionSpec",
    "ProjKind", "TableSlice", "fill_gaussian", "fill_gaussian_slice", "fill_signs", "gaussian_matrix", "lookup_forward",
    "to_bf16_values", "flops", "checkpoint_header", "load_checkpoint", "save_checkpoint", "LffnError", "NumericError", "SizeError", "UsageError",
]
