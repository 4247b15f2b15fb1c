"""Gather time against cudaLimitMaxL2FetchGranularity (32 / 64 / 128 bytes): does the L2's DRAM fetch
size change the row gathers?  (c3 re-reads its stack from HBM every round.)"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of
from paper_2403_07221_b200.lookup import Projection
rt = ctypes.CDLL("libcudart.so.12")
torch.cuda.init(); torch.zeros(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in ("c3", "c2", "c4"):
    w = WORKLOADS[name]; cfg = config_of(w)
    layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=w.n, table_dtype=w.table_dtype)
    dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
    T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
    layer.attach_tables(T)
    x = torch.from_numpy(make_x(w)).cuda()
    codes, coeff = layer.hash(x)
    y = torch.empty((w.n, w.d), device="cuda")
    for gran in (64, 32, 128, 64):
        rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(gran))  # cudaLimitMaxL2FetchGranularity = 0x05
        got = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(got), 5)
        ts = []
        for r in range(13):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); layer.lookup_accumulate(codes, coeff, y); e1.record(); torch.cuda.synchronize()
            if r >= 3: ts.append(e0.elapsed_time(e1))
        print(f"{name} L2 fetch granularity {gran} (rc {rc}, now {got.value}): gather {statistics.median(ts):.4f} ms", flush=True)
    layer.close(); del T
