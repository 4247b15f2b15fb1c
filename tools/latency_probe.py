"""Small-batch latency of the forward stages (c5 shapes): hash and gather
device times per call at n = 1, 8, 64 (stage events), warm L2."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = WORKLOADS[name]
cfg = config_of(w)
layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=64, table_dtype=w.table_dtype)
dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
layer.attach_tables(T)
x = torch.from_numpy(make_x(w, 64)).cuda()
y = torch.empty((64, w.d), device="cuda")
layer.set_timing(True)
for m in (1, 8, 64):
    hs, gs, tot = [], [], []
    for r in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        layer.forward_device(x[:m], y[:m])
        e1.record()
        torch.cuda.synchronize()
        a, b = layer.stage_ms()
        if r >= 10:
            hs.append(a * 1e3); gs.append(b * 1e3); tot.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name} n={m}: hash {statistics.median(hs):.1f} us  gather {statistics.median(gs):.1f} us  "
          f"forward {statistics.median(tot):.1f} us", flush=True)
