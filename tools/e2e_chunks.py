"""Host-path chunk sweep: lffn_forward_host wall time (pinned buffers, L2
flushed) per LFFN_OPT_HOST_CHUNKS on the BASELINE workloads.

    python tools/e2e_chunks.py c2 c3 c4 --chunks 4,8,12,16
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c2_bf16", "c3", "c4", "c5"])
    ap.add_argument("--chunks", default="4,8,12,16")
    ap.add_argument("--reps", type=int, default=15)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in a.configs:
        w = WORKLOADS[name]
        cfg = config_of(w)
        proj = Projection.init(spec_of(w), 1)
        layer = LookupFFN(cfg, proj, None, max_tokens=w.n, table_dtype=w.table_dtype)
        dt = torch.float32 if w.table_dtype == "f32" else torch.bfloat16
        g = torch.Generator(device="cuda").manual_seed(2)
        T = (torch.randn((w.h, 1 << w.tau, w.d), generator=g, device="cuda") * 0.02).to(dt)
        layer.attach_tables(T)
        hx = torch.from_numpy(make_x(w)).pin_memory()
        hy = torch.empty((w.n, w.d), dtype=torch.float32).pin_memory()
        for ch in [int(c) for c in a.chunks.split(",")]:
            layer.set_option("host_chunks", ch)
            ts = []
            for r in range(a.reps + 3):
                flush.fill_(r & 0xFF)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                layer.forward_host_ptr(hx.data_ptr(), w.n, hy.data_ptr())
                if r >= 3:
                    ts.append((time.perf_counter() - t0) * 1e3)
            t = statistics.median(ts)
            print(f"{name} chunks={ch:2d}: {t:.3f} ms  {w.n / t / 1e3:.2f} M tokens/s", flush=True)
        layer.close()
        del T


if __name__ == "__main__":
    main()
