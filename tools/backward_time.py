"""Device time of lffn_backward (and the forward beside it) on a BASELINE config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_07221_b200 import LookupFFN, ProjKind, LookupVariant
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kind = ProjKind[sys.argv[2]] if len(sys.argv) > 2 else ProjKind.signflip
w = WORKLOADS[name]
cfg, proj, T = make_params(w, kind)
n = w.n
layer = LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype)
xd = torch.from_numpy(make_x(w, n)).cuda()
gy = torch.randn((n, cfg.d_out), device="cuda")

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

f = timed(lambda: layer.forward_device(xd))
b = timed(lambda: layer.backward(xd, gy))
layer.sync()
print(f"{name} {kind.name}: forward {f:.3f} ms  backward {b:.3f} ms ({n} tokens)")
