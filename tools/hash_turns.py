"""A/B of the turn-taking signflip hash (option hash_exact = 2: hash_sf_turn_kernel, one 12-warp CTA per
SM, the three warps of a scheduler pass a lock around their float64 phases) against hash_sf_kernel."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_07221_b200 import LookupFFN
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of
from paper_2403_07221_b200.lookup import Projection
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:] or ["c3", "c2", "c5"]:
    w = WORKLOADS[name]; cfg = config_of(w); n = w.n
    layer = LookupFFN(cfg, Projection.init(spec_of(w), 1), None, max_tokens=n)
    x = torch.from_numpy(make_x(w, n)).cuda()
    codes = torch.empty((n, w.h), dtype=torch.int32, device="cuda"); coeff = torch.empty((n, w.h), dtype=torch.float32, device="cuda")
    ref = None
    for mode, ns in ((0, 0), (2, 2004), (2, 2012)):
        layer.set_option("hash_exact", mode)
        layer.set_option("gather_sms", ns)
        ts = []
        for r in range(5):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); layer.hash(x, codes, coeff); e1.record(); torch.cuda.synchronize()
            if r >= 2: ts.append(e0.elapsed_time(e1))
        layer.sync()
        if ref is None: ref = (codes.clone(), coeff.clone())
        same = bool(torch.equal(ref[0], codes)) and bool(torch.equal(ref[1], coeff))
        print(f"{name} n={n} {('turns pause %d ns' % ns) if mode else 'plain'}: {statistics.median(ts):.4f} ms  same records: {same}", flush=True)
    layer.close()
