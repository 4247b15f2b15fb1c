"""A short run of every device kernel family for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per call):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers the production signflip hash (K1f, D = 2048 and 4096), the exact-order
hash (K1), the dense tcgen05 hash with its fixups, BH, the persistent /
split / direct gathers (fp32 and bf16), the small-batch cluster kernel (K5),
nc > 1 neighbours and the backward, at small sizes.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_07221_b200 import (HashTables, LookupConfig, LookupFFN, Projection,  # noqa: E402
                                   ProjectionSpec, ProjKind, fill_gaussian, gaussian_matrix)


def layer_for(d, h, tau, kind=ProjKind.signflip, dtype="f32", nc=1, n=64, **kw):
    cfg = LookupConfig(d_in=d, d_out=d, tables=h, code_bits=tau, neighbor_count=nc)
    proj = Projection.init(ProjectionSpec(d, h * tau, kind, **kw), 1)
    T = HashTables(h, tau, d, fill_gaussian(2, h * (1 << tau) * d, 0.02))
    return LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=dtype)


def run(layer, n, d, back=False):
    x = torch.from_numpy(gaussian_matrix(n, d, 0).astype(np.float32)).cuda()
    y = layer.forward_device(x)
    layer.sync()
    if back:
        layer.backward(x, torch.ones_like(y))
        layer.sync()
    return float(y.abs().sum())


out = []
L = layer_for(768, 256, 8, n=300)                       # c2 shapes
out.append(run(L, 300, 768))                             # K1f + persistent/split gather
out.append(run(L, 8, 768))                               # K5 (cluster of 16)
out.append(run(L, 48, 768))                              # K5 (cluster of 8)
L.set_option("hash_exact", 1)
out.append(run(L, 40, 768, back=True))                   # K1 + backward
L.close()
L = layer_for(768, 256, 8, dtype="bf16", n=200)          # bf16 tables
out.append(run(L, 200, 768))
out.append(run(L, 5, 768))
L.close()
L = layer_for(4096, 64, 8, dtype="bf16", n=40)           # D = 4096 (K1f two warps per token)
out.append(run(L, 40, 4096))
L.close()
L = layer_for(768, 96, 8, ProjKind.dense, n=130)         # dense tcgen05 + fixups
out.append(run(L, 130, 768, back=True))
L.close()
L = layer_for(256, 32, 8, ProjKind.bh, n=20, stages=2, block=32)
out.append(run(L, 20, 256, back=True))
L.close()
L = layer_for(64, 8, 4, nc=3, n=33)                      # nc > 1 (direct gather)
out.append(run(L, 33, 64, back=True))
L.close()
L = layer_for(50, 12, 10, n=17)                          # non-pow2 pad/truncate
out.append(run(L, 17, 50))
L.close()
print("sanitize run ok", np.round(out, 3).tolist())
