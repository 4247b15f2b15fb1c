"""One forward call per batch size (c5 shapes) -- a short command for ncu
captures of the small-batch kernel:  python tools/small_once.py 1 64"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402

w = WORKLOADS["c5"]
ns = [int(a) for a in sys.argv[1:]] or [1, 64]
layer = LookupFFN(config_of(w), Projection.init(spec_of(w), 1), None, max_tokens=max(ns))
T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02)
layer.attach_tables(T)
x = torch.from_numpy(make_x(w, max(ns))).cuda()
for m in ns:
    for _ in range(3):
        y = layer.forward_device(x[:m])
    layer.sync()
print("ok", [float(layer.forward_device(x[:m]).abs().sum()) for m in ns])
