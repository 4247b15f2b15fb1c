"""Gather-kernel variant sweep: device time of lffn_lookup_accumulate per
LFFN_OPT_GATHER_VARIANT on the BASELINE workloads (codes from the real hash
of the workload's inputs; tables N(0, 0.02) drawn on the device -- timing
only, parity is the tests' job).  L2 is flushed before every timed launch.

    python tools/gather_sweep.py c2 c2_bf16 c3 c4 [--variants -1,40201,...]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x  # noqa: E402
from paper_2403_07221_b200.lookup import Projection  # noqa: E402
from paper_2403_07221_b200.configs import spec_of  # noqa: E402

DEFAULT = {"f32": [-1, 0], "bf16": [-1, 0]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c2_bf16", "c3", "c4"])
    ap.add_argument("--variants", default="")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--group-mb", default="0", help="comma list of table group sizes (MB)")
    ap.add_argument("--sms", default="0", help="comma list of gather SM counts (0 = all)")
    ap.add_argument("--tokens", default="", help="comma list of batch sizes (default: the workload's)")
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
        x = torch.from_numpy(make_x(w)).cuda()
        codes, coeff = layer.hash(x)
        y = torch.empty((w.n, w.d), device="cuda")
        variants = ([int(v) for v in a.variants.split(",")] if a.variants
                    else DEFAULT[w.table_dtype])
        y_ref = None
        G = w.n * w.h * w.d * (4 if dt == torch.float32 else 2)
        ns = [int(t) for t in a.tokens.split(",")] if a.tokens else [w.n]
        runs = [(v, int(gm), m, int(sm)) for m in ns for gm in a.group_mb.split(",") for v in variants
                for sm in a.sms.split(",")]
        for v, gm, m, sm in runs:
            layer.set_option("gather_sms", sm)
            if v == variants[0]:
                y_ref = None
            layer.set_option("table_group_bytes", gm << 20)
            try:
                layer.set_option("gather_variant", v)
            except Exception as e:  # noqa: BLE001
                print(f"{name} v={v}: {e}")
                continue
            ts = []
            for r in range(a.reps + 2):
                flush.fill_(r & 0xff)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                layer.lookup_accumulate(codes[:m], coeff[:m], y[:m])
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            if y_ref is None:
                y_ref = y[:m].clone()
                diff = 0.0
            else:
                diff = float((y[:m] - y_ref).abs().max() / y_ref.abs().max())
            t = statistics.median(ts)
            Gm = G * m / w.n
            print(f"{name} n={m} v={v:3d} group={gm}MB sms={sm}: {t:.4f} ms  {Gm / t / 1e6:.0f} GB/s gathered  "
                  f"maxdiff/max={diff:.2e}", flush=True)
        layer.close()
        del T


if __name__ == "__main__":
    main()
