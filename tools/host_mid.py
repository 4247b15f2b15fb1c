"""Host path of medium batches (96 .. 4096 tokens): the direct path (option host_direct = N: the
gather writes y into the pinned buffer for batches up to N tokens) against the chunked copy pipeline."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of
from paper_2403_07221_b200.lookup import Projection
for name in ("c5", "c2_bf16"):
    w = WORKLOADS[name]; cfg = config_of(w)
    layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=8192, table_dtype=w.table_dtype)
    dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
    T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
    layer.attach_tables(T)
    for m in (96, 128, 256, 512, 1024, 2048, 4096):
        hx = torch.from_numpy(make_x(w, m)).pin_memory(); hy = torch.empty((m, w.d)).pin_memory()
        res = {}
        for direct in (100000, 1):
            layer.set_option("host_direct", direct)
            ts = []
            for r in range(120):
                t0 = time.perf_counter(); layer.forward_host_ptr(hx.data_ptr(), m, hy.data_ptr())
                if r >= 20: ts.append((time.perf_counter() - t0) * 1e6)
            res[direct] = statistics.median(ts)
        print(f"{name} n={m}: direct {res[100000]:.1f} us   pipeline {res[1]:.1f} us", flush=True)
    layer.close()
