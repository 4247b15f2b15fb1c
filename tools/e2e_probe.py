"""PCIe / host-path probe: pinned H2D and D2H of the c2 step's bytes alone and
concurrently, and lffn_forward_host at the current chunking."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_07221_b200 import LookupFFN, ProjKind
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x

n = 16384
nb = n * 768 * 4
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3

def h2d():
    d.copy_(h, non_blocking=True)
def d2h():
    h2.copy_(d2, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
a, b, c = timeit(h2d), timeit(d2h), timeit(both)
print(f"{nb/1e6:.1f} MB  H2D {a:.3f} ms ({nb/a/1e6:.1f} GB/s)  D2H {b:.3f} ms ({nb/b/1e6:.1f} GB/s)  both {c:.3f} ms")
w = WORKLOADS["c2"]
cfg, proj, T = make_params(w, ProjKind.signflip)
layer = LookupFFN(cfg, proj, T, max_tokens=n)
x = torch.from_numpy(make_x(w, n)).pin_memory()
y = torch.empty((n, 768), dtype=torch.float32).pin_memory()
y_ref = None
for zc in (0,):
    for ch in (4, 6, 8, 10, 12, 16):
        layer.set_option("host_chunks", ch)
        ms = timeit(lambda: layer.forward_host_ptr(x.data_ptr(), n, y.data_ptr()))
        if y_ref is None:
            y_ref = y.clone()
        same = bool(torch.equal(y, y_ref))
        print(f"forward_host zero_copy={zc} chunks={ch}: {ms:.3f} ms  {n/ms*1e3/1e6:.2f} M tok/s  same_y={same}")
layer.set_option("host_chunks", 8)
xp = make_x(w, n)
yp = np.empty((n, 768), np.float32)
ms = timeit(lambda: layer.forward(xp, yp))
print(f"forward_host pageable numpy buffers: {ms:.3f} ms  {n/ms*1e3/1e6:.2f} M tok/s")
xd = x.cuda()
yd = torch.empty((n, 768), dtype=torch.float32, device="cuda")
for nchunk in (1, 4, 8, 16):
    per = n // nchunk
    def run():
        for i in range(nchunk):
            layer.forward_device(xd[i * per:(i + 1) * per], yd[i * per:(i + 1) * per])
    ms = timeit(run)
    print(f"device-only {nchunk} chunks of {per}: {ms:.3f} ms")
layer.set_timing(True)
for m in (1024, 2048, 4096, 16384):
    for _ in range(3):
        layer.forward_device(xd[:m], yd[:m])
    a, b = layer.stage_ms()
    print(f"n={m}: hash {a:.4f} ms  gather {b:.4f} ms")
