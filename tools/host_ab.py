"""lffn_forward_host A/B, interleaved rep by rep: flag published by a kernel and polled
(host_direct = 1) against the 4-byte copy + cudaStreamSynchronize (host_direct = 0)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of
from paper_2403_07221_b200.lookup import Projection
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in ("c5", "c2", "c2_bf16"):
    w = WORKLOADS[name]; cfg = config_of(w)
    layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=w.n, table_dtype=w.table_dtype)
    dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
    T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
    layer.attach_tables(T)
    hx = torch.from_numpy(make_x(w)).pin_memory(); hy = torch.empty((w.n, w.d)).pin_memory()
    ts = {0: [], 1: []}
    for r in range(2 * 33):
        d = r & 1
        layer.set_option("host_direct", d)
        flush.fill_(r & 0xFF); torch.cuda.synchronize()
        t0 = time.perf_counter(); layer.forward_host_ptr(hx.data_ptr(), w.n, hy.data_ptr())
        if r >= 6: ts[d].append((time.perf_counter() - t0) * 1e3)
    print(f"{name} n={w.n}: polled flag {statistics.median(ts[1]):.3f} ms (min {min(ts[1]):.3f})   memcpy + sync {statistics.median(ts[0]):.3f} ms (min {min(ts[0]):.3f})", flush=True)
    layer.close()
