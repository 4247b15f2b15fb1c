"""Hash-kernel A/B: device time of lffn_hash (codes + coefficients, no z) per
option hash_exact (1 = K1, the reference's stage order; 0 = K1f, the
production kernel) on the BASELINE workloads, and the number of codes that
differ between the two (allowed only where |z| <= 1e-5).

    python tools/hash_sweep.py c2 c3 c4 [--reps 20]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_07221_b200 import LookupFFN  # noqa: E402
from paper_2403_07221_b200.configs import WORKLOADS, config_of, make_x, spec_of  # noqa: E402
from paper_2403_07221_b200.lookup import Projection, ProjKind  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3", "c4"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--kind", default="signflip", help="signflip | bh | acdc | dense")
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in a.configs:
        w = WORKLOADS[name]
        n = a.tokens or w.n
        cfg = config_of(w)
        proj = Projection.init(spec_of(w, ProjKind[a.kind]), 1)
        layer = LookupFFN(cfg, proj, None, max_tokens=n)
        x = torch.from_numpy(make_x(w, n)).cuda()
        codes = torch.empty((n, w.h), dtype=torch.int32, device="cuda")
        coeff = torch.empty((n, w.h), dtype=torch.float32, device="cuda")
        res = {}
        for exact in (1, 0):
            layer.set_option("hash_exact", exact)
            ts = []
            for r in range(a.reps + 3):
                flush.fill_(r & 0xFF)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                layer.hash(x, codes, coeff)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            layer.sync()
            res[exact] = (statistics.median(ts), codes.clone(), coeff.clone())
        dc = int((res[0][1] != res[1][1]).sum())
        dw = float(((res[0][2] - res[1][2]).abs() / res[1][2].abs()).max())
        print(f"{name} n={n}: K1 (exact order) {res[1][0]:.4f} ms   K1f {res[0][0]:.4f} ms   "
              f"codes differing {dc}   max rel coeff diff {dw:.2e}", flush=True)
        layer.close()


if __name__ == "__main__":
    main()
