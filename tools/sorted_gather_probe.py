"""Would a token order that puts similar tokens on the same SM speed the gather up?  Time
lffn_lookup_accumulate on the records of the workload's own hash, in batch order and with the tokens
sorted by the codes of their first 1 / 2 / 3 tables (the reference's sorted gather "opt1", bench.cpp:198-217)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of
from paper_2403_07221_b200.lookup import Projection
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:] or ["c5", "c2"]:
    w = WORKLOADS[name]; cfg = config_of(w)
    layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=w.n, table_dtype=w.table_dtype)
    dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
    T = (torch.randn((w.h, 1 << w.tau, w.d), device="cuda") * 0.02).to(dt)
    layer.attach_tables(T)
    x = torch.from_numpy(make_x(w)).cuda()
    codes, coeff = layer.hash(x)
    y = torch.empty((w.n, w.d), device="cuda")
    for ntab in (0, 1, 2, 3, 6):
        if ntab:
            key = torch.zeros(w.n, dtype=torch.int64, device="cuda")
            for k in range(ntab):
                key = key * (1 << w.tau) + codes[:, k].long()
            perm = torch.argsort(key)
            cs, ws = codes[perm].contiguous(), coeff[perm].contiguous()
        else:
            cs, ws = codes, coeff
        ts = []
        for r in range(13):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); layer.lookup_accumulate(cs, ws, y); e1.record(); torch.cuda.synchronize()
            if r >= 3: ts.append(e0.elapsed_time(e1))
        print(f"{name}: tokens sorted by the codes of {ntab} tables: gather {statistics.median(ts):.4f} ms", flush=True)
    layer.close(); del T
