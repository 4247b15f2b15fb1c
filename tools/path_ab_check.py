"""Forward y of one workload saved to <out>.npy (device path, seeded inputs),
for A/B checks of opt-in kernels selected by environment variables in a
separate process (e.g. LFFN_GATHER_ASYNC, LFFN_FUSED_ASYNC with fused=1).

    python tools/path_ab_check.py c2 4096 /tmp/y [--fused]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x  # noqa: E402

name, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
w = WORKLOADS[name]
cfg, proj, T = make_params(w)
layer = LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype)
if "--fused" in sys.argv:
    layer.set_option("fused", 1)
x = torch.from_numpy(make_x(w, n)).cuda()
y = layer.forward_device(x)
layer.sync()
np.save(out, y.cpu().numpy())
