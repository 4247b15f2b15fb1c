"""Measure the tcgen05 dense-hash error against the float64 oracle (c2 shape)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle, Spec
from paper_2403_07221_b200 import LookupFFN, ProjKind
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = WORKLOADS["c2"]
cfg, proj, T = make_params(w, ProjKind.dense)
x = make_x(w, n)
layer = LookupFFN(cfg, proj, T, max_tokens=n)
xd = torch.from_numpy(x).cuda()
z = torch.empty((n, cfg.code_width()), dtype=torch.float64, device="cuda")
layer.hash(xd, z=z); layer.sync()
z = z.cpu().numpy()
o = Oracle()
t = time.time()
zr = o.proj_forward(Spec(768, 2048, 0), proj.blob, x.astype(np.float64))
err = np.abs(z - zr)
big = np.abs(zr) >= 1e-4
print(f"n={n} oracle {time.time()-t:.1f}s  max err {err.max():.3e}  max rel (|z|>=1e-4) {(err[big]/np.abs(zr[big])).max():.3e}"
      f"  p99.99 {np.quantile(err, 0.9999):.3e}  fixups {(np.abs(z) < 1e-4).sum()}")
