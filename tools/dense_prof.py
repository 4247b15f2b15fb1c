"""Per-CTA timeline of the tcgen05 dense hash kernel (LFFN_DENSE_PROF debug
dump): main-loop and epilogue durations, concurrency.  Usage:
  python tools/dense_prof.py [n]      (runs the c2 dense hash 3x, reads the dump)"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

path = os.path.join(tempfile.gettempdir(), "lffn_dense_prof.bin")
os.environ["LFFN_DENSE_PROF"] = path
import torch
from paper_2403_07221_b200 import LookupFFN, ProjKind
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = WORKLOADS["c2"]
cfg, proj, T = make_params(w, ProjKind.dense)
layer = LookupFFN(cfg, proj, T, max_tokens=n)
xd = torch.from_numpy(make_x(w, n)).cuda()
for _ in range(3):
    layer.hash(xd)
layer.sync()
layer.close()
a = np.fromfile(path, dtype=np.int64).reshape(-1, 4)
t0 = a[:, 0].min()
start, done, end = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
main, epi = done - start, end - done
print(f"CTAs {len(a)}  span {end.max():.1f} us  main loop mean {main.mean():.2f} p50 {np.median(main):.2f} "
      f"max {main.max():.2f} us  epilogue mean {epi.mean():.2f} p50 {np.median(epi):.2f} max {epi.max():.2f} us")
print(f"sum(CTA time)/(148*span) = {(end - start).sum() / (148 * end.max()):.2f} CTAs resident per SM on average")
first = np.argsort(start)[:8]
print("first CTAs start/done/end us:", [(round(start[i], 1), round(done[i], 1), round(end[i], 1)) for i in first])
