"""Small-batch latency (c5 shapes): device time per forward call at n = 1 ..
128, the one-launch small-batch kernel (K5) against the two-kernel path
(small_max_tokens = 0), warm and flushed L2, and the host path.

    python tools/latency_probe.py [c5|c2|c2_bf16|c3]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = WORKLOADS[name]
cfg = config_of(w)
N = 128
layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=N, table_dtype=w.table_dtype)
dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
layer.attach_tables(T)
x = torch.from_numpy(make_x(w, N)).cuda()
y = torch.empty((N, w.d), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def dev_us(m, cold):
    ts = []
    for r in range(60):
        # keep the device busy up to the first event (a spin kernel, or the
        # L2 flush), so the host's launch latency is not in the interval
        if cold:
            flush.fill_(r & 0xFF)
        else:
            torch.cuda._sleep(100000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        layer.forward_device(x[:m], y[:m])
        e1.record()
        torch.cuda.synchronize()
        if r >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for m in (1, 2, 4, 8, 12, 16, 24, 32, 48, 64, 128):
    out = []
    for small in (64, 0):
        layer.set_option("small_max_tokens", small)
        out.append((dev_us(m, False), dev_us(m, True)))
    hx = torch.from_numpy(make_x(w, m)).pin_memory()
    hy = torch.empty((m, w.d)).pin_memory()
    layer.set_option("small_max_tokens", 64)
    host = {}
    y_direct = None
    for direct in (1, 0):  # y / flag written straight to pinned memory vs the CUDA-graph copy path
        layer.set_option("host_direct", direct)
        ts = []
        for r in range(200):
            t0 = time.perf_counter()
            layer.forward_host_ptr(hx.data_ptr(), m, hy.data_ptr())
            if r >= 20:
                ts.append((time.perf_counter() - t0) * 1e6)
        host[direct] = statistics.median(ts)
        if direct:
            y_direct = hy.clone()
    same = bool(torch.equal(y_direct, hy))
    print(f"{name} n={m:3d}: one-launch {out[0][0]:6.1f} us warm {out[0][1]:6.1f} cold | "
          f"two kernels {out[1][0]:6.1f} warm {out[1][1]:6.1f} cold | host path direct {host[1]:6.1f} us, "
          f"graph {host[0]:6.1f} us (same y: {same})", flush=True)
