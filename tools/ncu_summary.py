#!/usr/bin/env python
"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv   > profiles/<round>_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep        > profiles/<round>_ncu_full.md
    python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep KEY  (prints JSON for profiles/ncu_gather_traffic.json)
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("dram__bytes_read.sum.per_second", "dram read bytes/s"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram read % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "L2 -> SM read bytes/s"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "L2 -> SM read % of peak"),
    ("lts__t_sectors.sum.per_second", "L2 sectors/s (x 32 B)"),
    ("lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 -> xbar port busy % (avg)"),
    ("lts__lts2xbar_cycles_active.max.pct_of_peak_sustained_elapsed", "L2 -> xbar port busy % (max slice)"),
    ("lts__t_sectors_srcunit_ltcfabric.sum.per_second", "L2 sectors/s from the die-to-die fabric"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    # ncu --csv --log-file: header row contains "Kernel Name" and "Metric Value"
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1000.0 if unit in ("ns", "nsecond") else v * (1000.0 if unit in ("ms", "msecond") else 1.0)
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | avg us | share |")
    print("|---|---:|---:|---:|---:|")
    step = {n: v for n, v in agg.items() if "lffn_gpu::" in n and "l2_read" not in n}
    stotal = sum(v[1] for v in step.values()) or 1.0
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * us / stotal:.1f}%" if name in step else "not in step"
        print(f"| `{name}` | {cnt} | {us:.1f} | {us / cnt:.1f} | {share} |")
    print(f"\nShare = fraction of the forward's own kernels (hash + gather); the bandwidth "
          "probe and torch's L2-flush fill run outside the timed step.  Times are cold-cache "
          "and serialised under ncu: compare shares, not absolutes.")


def raw(path):
    """ncu report (.ncu-rep) or its saved raw page (.raw.csv[.gz])."""
    if path.endswith(".csv") or path.endswith(".csv.gz"):
        import gzip

        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rt") as f:
            out = f.read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def stalls(hdr, row):
    items = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            if v > 0:
                items.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    items.sort(reverse=True)
    tot = sum(v for v, _ in items) or 1.0
    return ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in items[:6])


def full(path):
    hdr, units, rows = raw(path)
    ki = hdr.index("Kernel Name")
    for row in rows:
        print(f"### `{row[ki][:120]}`\n")
        print("| metric | value |")
        print("|---|---:|")
        for m, label in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {label} (`{m}`) | {row[i]} {units[i]} |")
        print(f"| top stall reasons | {stalls(hdr, row)} |\n")


def traffic(path, key):
    hdr, units, rows = raw(path)
    ki = hdr.index("Kernel Name")
    for row in rows:
        if "gather" in row[ki]:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                tot += float(row[i].replace(",", "")) * scale.get(units[i], 1)
            print(json.dumps({key: {"dram_bytes_per_launch": tot, "source": path}}))
            return


if __name__ == "__main__":
    {"launches": lambda: launches(sys.argv[2]), "full": lambda: full(sys.argv[2]),
     "traffic": lambda: traffic(sys.argv[2], sys.argv[3])}[sys.argv[1]]()
