"""A/B of the forward: fused hash+gather kernel vs hash kernel + gather kernel
(device time with CUDA events, L2 flushed before every timed forward).

    python tools/fused_ab.py c2 c2_bf16 c3 c5 [--tokens 2048,4096,16384]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c2_bf16", "c3", "c5"])
    ap.add_argument("--tokens", default="")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in a.configs:
        w = WORKLOADS[name]
        cfg = config_of(w)
        proj = Projection.init(spec_of(w), 1)
        ns = [int(t) for t in a.tokens.split(",")] if a.tokens else [w.n]
        layer = LookupFFN(cfg, proj, None, max_tokens=max(ns), table_dtype=w.table_dtype)
        dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
        g = torch.Generator(device="cuda").manual_seed(2)
        T = (torch.randn((w.h, 1 << w.tau, w.d), generator=g, device="cuda") * 0.02).to(dt)
        layer.attach_tables(T)
        x = torch.from_numpy(make_x(w, max(ns))).cuda()
        y = torch.empty((max(ns), w.d), device="cuda")
        for m in ns:
            res = {}
            for fused in (0, 1):
                layer.set_option("fused", fused)
                ts = []
                for r in range(a.reps + 3):
                    flush.fill_(r & 0xff)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    layer.forward_device(x[:m], y[:m])
                    e1.record()
                    torch.cuda.synchronize()
                    if r >= 3:
                        ts.append(e0.elapsed_time(e1))
                layer.sync()
                res[fused] = (statistics.median(ts), y[:m].clone())
            d = float((res[1][1] - res[0][1]).abs().max() / res[0][1].abs().max())
            print(f"{name} n={m}: two-kernel {res[0][0]:.4f} ms  fused {res[1][0]:.4f} ms  "
                  f"({m / res[1][0] / 1e3:.2f} M tok/s)  maxdiff/max={d:.2e}", flush=True)
        layer.close()
        del T


if __name__ == "__main__":
    main()
