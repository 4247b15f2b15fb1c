"""A/B of the backward paths: grad_x and grad_T of one configuration saved to
<out>.npy / <out>_T.npy (run once with LFFN_BWD_ONE_PASS=1 and once without,
then compare the files).

    python tools/bwd_ab_check.py c2 /tmp/a
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_07221_b200 import LookupFFN, ProjKind
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x
w = WORKLOADS[sys.argv[1]]
cfg, proj, T = make_params(w, ProjKind.signflip)
n = 2048
layer = LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype)
xd = torch.from_numpy(make_x(w, n)).cuda()
g = torch.Generator().manual_seed(3)
gy = torch.randn((n, cfg.d_out), generator=g).cuda()
out = layer.backward(xd, gy)
layer.sync()
np.save(sys.argv[2], out["grad_x"].cpu().numpy())
np.save(sys.argv[2] + "_T", out["grad_tables"].cpu().numpy())
