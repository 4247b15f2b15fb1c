import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle, Spec
from paper_2403_07221_b200 import (LookupFFN, LookupConfig, Projection, ProjectionSpec, ProjKind,
                                   HashTables, fill_gaussian, gaussian_matrix)
d, h, tau, n = [int(a) for a in sys.argv[1:5]]
cfg = LookupConfig(d_in=d, d_out=16, tables=h, code_bits=tau)
proj = Projection.init(ProjectionSpec(d, h * tau, ProjKind.dense), 1)
T = HashTables(h, tau, 16, fill_gaussian(2, h * (1 << tau) * 16, 0.02))
x = gaussian_matrix(n, d, 0).astype(np.float32)
layer = LookupFFN(cfg, proj, T, max_tokens=n)
xd = torch.from_numpy(x).cuda()
z = torch.full((n, h * tau), 7.0, dtype=torch.float64, device="cuda")
layer.hash(xd, z=z)
torch.cuda.synchronize()
z = z.cpu().numpy()
zr = Oracle().proj_forward(Spec(d, h * tau, 0), proj.blob, x.astype(np.float64))
bad = ~np.isfinite(z) | (np.abs(z - zr) > 1e-3)
print("bad", bad.sum(), "of", z.size)
if bad.sum():
    r, c = np.nonzero(bad)
    print("rows", np.unique(r)[:20], "cols", np.unique(c)[:40])
    print("sample", z[r[0], c[0]], zr[r[0], c[0]])
