#!/usr/bin/env python
"""LookupFFN forward benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--kind signflip]

A step is one full forward (hash + gather-accumulate) over the workload's
batch, inputs already resident in HBM.  Default workload: BASELINE.json
configs[1] (c2: d=768, h=256, tau=8, 16384 tokens, signflip projection, fp32
tables).  N > 1 (torchrun, one rank per GPU) shards TOKENS with replicated
tables for c1/c2/c5 (weak scaling: every rank runs the full per-GPU batch; no
collective on the data path) and TABLES for c3/c4 (strong
scaling: every rank runs all tokens over its table slice; the fp32 partials
are combined by NCCL reduce-scatter (c3) / all-reduce (c4), chunk-pipelined;
--shard overrides).  Times are CUDA events on the launching
stream, per step, with L2 flushed (256 MiB write) before every timed step;
the max over ranks is reported.

--impl reference times the reference's own float32 inference kernels
(bench.cpp:115-217, compiled from the reference sources into oracle/_ref) on
the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "LookupFFN fwd tokens/sec; achieved L2/HBM GB/s vs gather roofline"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--kind", default="signflip", choices=["signflip", "dense", "acdc", "bh"])
    ap.add_argument("--tokens", type=int, default=0, help="override the batch size")
    ap.add_argument("--cpu-sample", type=int, default=0, help="reference-arm tokens per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hash-mode", default="token", choices=["token", "replicated"],
                    help="table sharding: hash the rank's own token block and all-to-all the "
                         "records (token), or recompute the full hash on every rank")
    ap.add_argument("--table-sharded", type=int, default=-1,
                    help="also measure c3 (reduce-scatter) and c4 (all-reduce) table-sharded "
                         "and report them under 'table_sharded' (default: at N > 1)")
    ap.add_argument("--shard", default="auto", choices=["auto", "token", "table"],
                    help="N>1 partitioning: token (tables replicated, c1/c2/c5) or table "
                         "(tables split over ranks, partials combined by NCCL; c3/c4); "
                         "auto picks the north star's choice per config")
    return ap.parse_args()


def shard_mode(args) -> tuple:
    """(mode, combine) per BASELINE north_star: c3 reduce-scatter, c4 all-reduce
    over table shards at N > 1 (one GPU runs the plain forward; --shard table
    forces the sharded path on a world-1 NCCL group); token sharding when the
    tables fit one GPU."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.shard == "token" or (args.shard == "auto" and (args.config not in ("c3", "c4")
                                                            or world == 1)):
        return "token", None
    return "table", ("all_reduce" if args.config == "c4" else "reduce_scatter")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (the timed region is tens of ms), falling
    back to `nvidia-smi -lms` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NVML_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                    0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.nvml = None
        self.stop = threading.Event()

    def _poll_nvml(self):
        import pynvml as N

        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.nvml, N.NVML_CLOCK_SM)
                mx = N.nvmlDeviceGetMaxClockInfo(self.nvml, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.nvml)
                names = [nm for bit, nm in self.NVML_REASONS.items() if rs & bit]
                self.lines.append((float(sm), float(mx), names))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            import torch

            # map the CUDA ordinal to the NVML handle through the PCI address
            pr = torch.cuda.get_device_properties(self.device)
            try:
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.nvml = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.nvml = N.nvmlDeviceGetHandleByIndex(self.device)
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()  # keep only samples taken during the timed region
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml is not None:
            if not self.lines:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
            sm = [s for s, _, _ in self.lines]
            reasons = sorted({r for _, _, rs in self.lines for r in rs})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(m for _, m, _ in self.lines),
                    "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(sm),
                    "source": "nvml"}
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def load_traffic(workload: str, kind: str):
    """dram read+write bytes per gather launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_gather_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{workload}:{kind}")
    except Exception:
        return None


# --------------------------------------------------------------------- ours
def run_ours(args):
    import torch

    from paper_2403_07221_b200 import LookupFFN, ProjKind, _capi
    from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x
    from paper_2403_07221_b200.flops import (gathered_bytes_per_token, lookup_flops,
                                             unique_table_bytes)

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w = WORKLOADS[args.config]
    n = args.tokens or w.n
    kind = ProjKind[args.kind]
    cfg, proj, T = make_params(w, kind)
    mode, combine = shard_mode(args)
    elem = 4 if w.table_dtype == "f32" else 2
    stream = torch.cuda.current_stream()
    if mode == "token":
        x = make_x(w, n, seed=rank)  # token sharding: rank r owns its own batch
        layer = LookupFFN(cfg, proj, T, device=local, max_tokens=n, table_dtype=w.table_dtype)
        sharded = None
    else:
        # table sharding: every rank holds all n tokens and tables
        # [r*h/P, (r+1)*h/P); partial sums combined by NCCL (sharded.py)
        from paper_2403_07221_b200.sharded import ShardedLookupFFN

        if dist is None:  # one GPU: a world-1 NCCL group keeps the same code path
            import socket

            import torch.distributed as dist

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1, device_id=torch.device("cuda", local))

        chunks = 4
        q = world * chunks
        n = ((n + q - 1) // q) * q
        x = make_x(w, n, seed=0)
        sharded = ShardedLookupFFN(cfg, proj, T, mode="table", combine=combine, device=local,
                                   hash_mode=args.hash_mode,
                                   max_tokens=n, table_dtype=w.table_dtype, chunks=chunks)
        layer = sharded.layer
    del T

    xd = torch.from_numpy(x).cuda()
    yd = torch.empty((n, cfg.d_out), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    layer.set_timing(True)

    if sharded is None:
        def step():
            layer.forward_device(xd, yd, stream=stream)
    else:
        y_sh = torch.empty((n // world if combine == "reduce_scatter" else n, cfg.d_out),
                           dtype=torch.float32, device="cuda")

        def step():
            sharded.forward(xd, y_sh)

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    layer.sync(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    launches0 = layer.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    hash_ms, gather_ms = [], []
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)          # L2 flush, outside the timed interval
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
            if sharded is None:
                a, b = layer.stage_ms()    # event sync on this step's stage events
                hash_ms.append(a)
                gather_ms.append(b)
        torch.cuda.synchronize()
    if sharded is not None:
        # the rank's kernels alone (hash + gather of its table slice over all
        # n tokens), timed outside the sharded steps
        for i in range(max(3, args.steps // 2)):
            flush.fill_(i & 0xFF)
            layer.forward_device(xd, yd, stream=stream)
            a, b = layer.stage_ms()
            hash_ms.append(a)
            gather_ms.append(b)
    launches = layer.launch_count() - launches0
    layer.sync(stream)
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    mean_ms = float(np.mean(step_ms))
    if dist:
        t = torch.tensor([mean_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()

    # codes of this batch -> unique table bytes U (never assumed)
    codes, _ = layer.hash(xd)
    layer.sync()
    codes_np = codes.cpu().numpy().view(np.uint32)
    U = unique_table_bytes(codes_np, cfg, elem)
    h_loc = layer.table_range[1] - layer.table_range[0]
    G = gathered_bytes_per_token(cfg, elem) * n * h_loc // cfg.tables  # this rank's tables

    # c5 (skewed / small-batch stress): per-call latency at the BASELINE's
    # small token counts, device time (CUDA events) with the tables warm in
    # L2 and after an L2 flush, and through the host path
    small = None
    if args.config == "c5" and mode == "token":
        layer.set_timing(False)  # no stage events inside the measured calls
        small = {}
        for m in (1, 8, 64):
            res = {}
            for cold in (False, True):
                ts = []
                for r in range(60):
                    # the device is kept busy up to the first event (L2
                    # flush, or a spin kernel for warm L2) so the interval
                    # is device time, not the host's launch latency
                    if cold:
                        flush.fill_(r & 0xFF)
                    else:
                        torch.cuda._sleep(100000)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    layer.forward_device(xd[:m], yd[:m], stream=stream)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if r >= 10:
                        ts.append(e0.elapsed_time(e1) * 1e3)
                res["device_us_cold_l2" if cold else "device_us_warm_l2"] = round(
                    float(np.median(ts)), 2)
            hxm = torch.from_numpy(np.ascontiguousarray(x[:m])).pin_memory()
            hym = torch.empty((m, cfg.d_out), dtype=torch.float32).pin_memory()
            ts = []
            for r in range(60):
                t0 = time.perf_counter()
                layer.forward_host_ptr(hxm.data_ptr(), m, hym.data_ptr())
                if r >= 10:
                    ts.append((time.perf_counter() - t0) * 1e6)
            res["host_path_us"] = round(float(np.median(ts)), 2)
            small[str(m)] = res

    # end-to-end through the C-ABI host path: pinned host x -> y
    hx = torch.from_numpy(x).pin_memory()
    hy = torch.empty((n, cfg.d_out), dtype=torch.float32).pin_memory()
    for _ in range(max(1, args.warmup // 2)):
        layer.forward_host_ptr(hx.data_ptr(), n, hy.data_ptr())
    e2e_ms = []
    for _ in range(max(3, args.steps // 2)):
        flush.fill_(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        layer.forward_host_ptr(hx.data_ptr(), n, hy.data_ptr())
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_mean = float(np.mean(e2e_ms))
    if dist:
        t = torch.tensor([e2e_mean], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())

    result = None
    l2 = 0.0
    if rank == 0:
        peaks, peak_src = load_peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        import ctypes as C

        g = C.c_double()
        _capi.check(_capi.lib().lffn_probe_bandwidth(local, 0, 5, C.byref(g)))
        l2 = g.value
        _capi.check(_capi.lib().lffn_probe_bandwidth(local, 2, 5, C.byref(g)))
        l2_rand = g.value
        gather_avg = float(np.mean(gather_ms))
        hash_avg = float(np.mean(hash_ms))
        t_roof_ms = (U / (hbm * 1e9) + G / (l2 * 1e9)) * 1e3
        achieved = G / (gather_avg * 1e-3) / 1e9
        peak_eff = G / (t_roof_ms * 1e-3) / 1e9
        fl = lookup_flops(cfg, proj.spec)
        # token sharding: every rank its own n tokens; table sharding: the
        # ranks share the same n tokens (each for its table slice)
        tokens_total = n * world if mode == "token" else n
        value = tokens_total / (mean_ms * 1e-3)
        traffic = load_traffic(args.config, args.kind)
        t_fwd = mean_ms
        result = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(mean_ms, 5),
            "higher_is_better": True,
            "scaling": "weak" if mode == "token" else "strong",
            "vs_baseline": None,
            "dtype": "f32" if w.table_dtype == "f32" else "bf16-tables/f32-accum",
            "data": "synthetic (reference seeds: x make_rng(rank), proj init seed 1, "
                    "tables N(0,0.02) make_rng(2))",
            "config": {
                "workload": f"{w.name}: d_in=d_out={w.d} h={w.h} tau={w.tau} "
                            f"n={n}/GPU {args.kind} {w.table_dtype} tables",
                "tokens_per_gpu": n,
                "parallelism": (f"token-sharded x{world} (tables replicated)" if mode == "token"
                                else f"table-sharded x{world} (tables [{layer.table_range[0]}, "
                                     f"{layer.table_range[1]}) on rank 0; NCCL {combine} of the "
                                     f"fp32 partials, 4 chunks overlapped; hash "
                                     + ("of the rank's token block, records all-to-all"
                                        if args.hash_mode == "token" else "replicated") + ")"),
                "l2": "flushed before every timed step (256 MiB write outside the events)",
            },
            "e2e": {
                "value": round(tokens_total / (e2e_mean * 1e-3), 1),
                "unit": UNIT,
                "h2d_bytes_per_step": int(x.nbytes),
                "d2h_bytes_per_step": int(n * cfg.d_out * 4),
                "ms_per_step": round(e2e_mean, 4),
                "path": "lffn_forward_host (pinned host x/y; chunked H2D || kernels || D2H)",
            },
            "gpu_launches": int(launches),
            "stages_ms": {"hash": round(hash_avg, 5), "gather": round(gather_avg, 5)},
            "roofline": {
                # memory-bound: t_roof = U/BW_HBM + G/BW_L2, and the L2 term
                # dominates (c2: 94 %) -- the bound is the L2 -> SM read path
                "bound": "l2",
                "kernel": "gather_accumulate",
                "achieved": round(achieved, 1),
                "peak": round(peak_eff, 1),
                "unit": "GB/s",
                "frac": round(achieved / peak_eff, 4),
                # the whole forward (hash + gather) on the same roofline: the
                # north star's "tokens/s as achieved fraction of the memory
                # roofline"
                "frac_forward": round(t_roof_ms / t_fwd, 4),
                # dram__bytes_read.sum + dram__bytes_write.sum of the gather
                # launch, bytes, from the committed ncu --set full capture
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "traffic_source": (traffic or {}).get("source"),
                "definition": "BASELINE north_star gather roofline: t_roof = U/BW_HBM + G/BW_L2; "
                              "achieved = G / gather time, peak = G / t_roof (frac = t_roof / "
                              "t_gather); frac_forward = t_roof / ms_per_step",
                "gathered_bytes_G": int(G),
                "unique_bytes_U": int(U),
                "bw_hbm_gbs": hbm,
                "bw_hbm_source": peak_src + " MEASURED_PEAKS.json hbm_gbs",
                "bw_l2_gbs": round(l2, 1),
                "bw_l2_source": "measured live, the best L2 read rate found on B200: 128-bit "
                                "sequential re-reads of a 32 MiB buffer from every SM "
                                "(lffn_probe_bandwidth 0; cross-checked with ncu in "
                                "profiles/r2_l2_probe.md)",
                "t_roof_ms": round(t_roof_ms, 5),
                # context, not the denominator: the same probe with the
                # gather's access pattern (random 512-byte segments)
                "bw_l2_random_512B_gbs": round(l2_rand, 1),
                "frac_vs_random_segment_l2": round(
                    (U / (hbm * 1e9) + G / (l2_rand * 1e9)) * 1e3 / gather_avg, 4),
                "hbm_frac_unique": round((U + x.nbytes + n * cfg.d_out * 4) /
                                         (gather_avg * 1e-3 + hash_avg * 1e-3) / 1e9 / hbm, 4),
            },
            "flops_mflop_per_token": {"hash": fl.hash_mflop, "gather": fl.gather_mflop,
                                      "other": fl.other_mflop},
            "clocks": clocks.summary(),
        }
        if small is not None:
            result["small_batch_latency"] = small
    want_ts = args.table_sharded if args.table_sharded >= 0 else int(world > 1)
    if want_ts and mode == "token" and args.config not in ("c3", "c4"):
        # BASELINE's table-sharded configs on the same ranks (north star:
        # c3 reduce-scatter, c4 all-reduce at 1 / 2 / 4 / 8 GPUs)
        layer.close()
        del xd, yd, flush
        torch.cuda.empty_cache()
        if dist is None:
            import socket

            import torch.distributed as dist

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1, device_id=torch.device("cuda", local))
        l2b = torch.tensor([l2 if rank == 0 else 0.0], device="cuda")
        dist.all_reduce(l2b, op=dist.ReduceOp.MAX)
        hbm_b = float(load_peaks()[0].get("hbm_gbs", 6650.0))
        ts = {}
        for name, comb in (("c3", "reduce_scatter"), ("c4", "all_reduce")):
            try:
                ts[name] = table_sharded_measure(name, comb, rank, world, local,
                                                 max(3, args.steps // 2), 3,
                                                 float(l2b.item()), hbm_b)
            except Exception as e:  # reported, never fatal for the headline line
                ts[name] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
        if result is not None:
            result["table_sharded"] = ts
        layer = None
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if sharded is not None:
        sharded.close()
    elif layer is not None:
        layer.close()
    return result


# ----------------------------------------------------------- table sharding
def table_sharded_measure(name: str, combine: str, rank: int, world: int, local: int,
                          steps: int, warmup: int, l2_gbs: float, hbm_gbs: float):
    """BASELINE's table-sharded configs (c3: NCCL reduce-scatter, c4: NCCL
    all-reduce): every rank owns tables split_range(h, P, r) -- built as a
    slice of the reference-seeded stack, never the whole stack -- hashes its
    own token block for all tables, receives the records of its tables by one
    all-to-all, gathers the fp32 partial for all n tokens and the partials
    are combined chunk by chunk (sharded.py).  Reported: tokens/s (max over
    ranks), the compute alone (hash + gather of the rank) on its own roofline
    (U/P at HBM + G/P at L2), and the combine alone against its bus bytes."""
    import torch
    import torch.distributed as dist

    from paper_2403_07221_b200 import Projection
    from paper_2403_07221_b200.configs import (WORKLOADS, config_of, make_table_slice, make_x,
                                               spec_of)
    from paper_2403_07221_b200.flops import unique_table_bytes
    from paper_2403_07221_b200.sharded import ShardedLookupFFN, split_range

    w = WORKLOADS[name]
    cfg = config_of(w)
    proj = Projection.init(spec_of(w), 1)
    kb, ke = split_range(w.h, world, rank)
    chunks = 4
    q = world * chunks
    n = ((w.n + q - 1) // q) * q
    T = make_table_slice(w, kb, ke)
    sh = ShardedLookupFFN(cfg, proj, T, mode="table", combine=combine, device=local,
                          max_tokens=n, table_dtype=w.table_dtype, chunks=chunks)
    del T
    x = make_x(w, n, seed=0)
    xd = torch.from_numpy(x).cuda()
    d = cfg.d_out
    y = torch.empty((n // world if combine == "reduce_scatter" else n, d), dtype=torch.float32,
                    device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def timed(fn, reps, pre=None):
        out = []
        for i in range(reps):
            if pre:
                pre(i)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            out.append((e0, e1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in out]

    def maxr(v):
        t = torch.tensor([float(v)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(warmup):
        flush.fill_(i & 0xFF)
        sh.forward(xd, y)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    step = maxr(np.mean(timed(lambda: sh.forward(xd, y), steps,
                              pre=lambda i: flush.fill_(i & 0xFF))))
    # the rank's compute alone: hash of its token block, gather of its tables
    t0, t1 = split_range(n, world, rank)
    codes, coeff = sh.exchange_records(xd)
    torch.cuda.synchronize()
    part = torch.empty((n, d), dtype=torch.float32, device="cuda")
    reps = max(3, steps // 2)
    hash_ms = maxr(np.mean(timed(lambda: sh.hasher.hash(xd[t0:t1]), reps,
                                 pre=lambda i: flush.fill_(i & 0xFF))))
    gather_ms = maxr(np.mean(timed(lambda: sh.layer.lookup_accumulate(codes, coeff, part), reps,
                                   pre=lambda i: flush.fill_(i & 0xFF))))
    # the combine alone, on the full partial
    if combine == "reduce_scatter":
        out = torch.empty((n // world, d), dtype=torch.float32, device="cuda")
        comm = lambda: dist.reduce_scatter_tensor(out, part)  # noqa: E731
        bus = (world - 1) / world * n * d * 4
    else:
        comm = lambda: dist.all_reduce(part)  # noqa: E731
        bus = 2 * (world - 1) / world * n * d * 4
    comm()
    torch.cuda.synchronize()
    dist.barrier()
    comm_ms = maxr(np.mean(timed(comm, reps)))
    elem = 4 if w.table_dtype == "f32" else 2
    U = unique_table_bytes(codes.cpu().numpy().view(np.uint32), cfg, elem)
    G = n * (ke - kb) * d * elem
    t_roof = (U / (hbm_gbs * 1e9) + G / (l2_gbs * 1e9)) * 1e3
    sh.close()
    del part
    torch.cuda.empty_cache()
    # the same forward through the C-ABI group (lffn_forward_sharded: NCCL
    # owned by the library, no torch on the data path)
    native = None
    try:
        from paper_2403_07221_b200.sharded import NativeTableShard

        ids = [NativeTableShard.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        T = make_table_slice(w, kb, ke)
        ng = NativeTableShard(cfg, proj, T, rank=rank, world=world, nccl_id=ids[0],
                              device=local, max_tokens=n, table_dtype=w.table_dtype,
                              chunks=chunks)
        del T
        for i in range(warmup):
            ng.forward(xd, y, combine=combine)
        torch.cuda.synchronize()
        dist.barrier()
        nstep = maxr(np.mean(timed(lambda: ng.forward(xd, y, combine=combine), steps,
                                   pre=lambda i: flush.fill_(i & 0xFF))))
        native = {"tokens_per_s": round(n / (nstep * 1e-3), 1), "ms_per_step": round(nstep, 4),
                  "path": "lffn_group / lffn_forward_sharded (C-ABI, NCCL owned by the group)"}
        ng.close()
    except Exception as e:  # reported, never fatal
        native = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    del xd, y, flush
    torch.cuda.empty_cache()
    return {
        "config": f"{w.name}: d={w.d} h={w.h} tau={w.tau} n={n} {w.table_dtype} tables, "
                  f"tables split over {world} ranks, hash of each rank's token block + "
                  f"all-to-all of the records, NCCL {combine} of the fp32 partials in "
                  f"{chunks} chunks overlapped with the gather",
        "tokens_per_s": round(n / (step * 1e-3), 1),
        "ms_per_step": round(step, 4),
        "scaling": "strong",
        "compute_ms": {"hash_rank_block": round(hash_ms, 4), "gather_rank_tables": round(gather_ms, 4)},
        "compute_roofline": {"t_roof_ms": round(t_roof, 5),
                             "frac": round(t_roof / (hash_ms + gather_ms), 4),
                             "frac_gather": round(t_roof / gather_ms, 4),
                             "unique_bytes_U_rank0": int(U), "gathered_bytes_G_rank": int(G),
                             "definition": "U/P at BW_HBM + G/P at BW_L2 (rank 0's slice)"},
        "combine": {"op": combine, "ms": round(comm_ms, 4), "bus_bytes": int(bus),
                    "bus_gbs": round(bus / (comm_ms * 1e-3) / 1e9, 1) if world > 1 else None},
        "native_group": native,
    }


# ---------------------------------------------------------------- reference
def reference_inputs(w, kind_name: str, n: int, ref):
    """x, projection blob and tables of workload w built by the REFERENCE
    library itself (oracle/_ref/liblffn_ref.so: make_rng + fill_gaussian,
    Projection::init), with the bench's seeds -- the values are bit-identical
    to the ours arm's (tests/test_oracle_pin.py), but no code of this
    repository's product library runs on the reference arm."""
    from oracle import Spec
    from paper_2403_07221_b200.configs import TABLE_STD, make_x, spec_of
    from paper_2403_07221_b200.lookup import ProjKind

    sp = spec_of(w, ProjKind[kind_name])
    s = Spec(sp.d_in, sp.d_out, int(sp.kind), sp.stages, sp.block, sp.depth)
    x = make_x(w, n, gaussian=lambda seed, cnt: ref.gaussian(seed, cnt))
    blob = ref.proj_init(s, 1)
    T = ref.gaussian(2, w.h * (1 << w.tau) * w.d, TABLE_STD)
    return s, x, blob, T


def reference_measure(args, w, steps: int, warmup: int, cores: int):
    """The reference's float32 inference pipeline (lookup_hash_f32 ->
    lookup_weights_f32 -> lookup_gather_f32 | lookup_gather_sorted_f32,
    bench.cpp:115-217, compiled from the reference sources) over the
    workload's FULL batch on `cores` host threads (256-row tiles, one per
    thread at a time).  The faster of the plain and the sorted ("opt1")
    gather is timed; the float64 lookup_forward (lookup.cpp:279-282) and the
    single-core rate are reported beside it on bounded samples."""
    from oracle import Cfg, Reference

    ref = Reference()
    n = w.n
    s, x, blob, T = reference_inputs(w, args.kind, n, ref)
    c = Cfg(w.d, w.d, w.h, w.tau)
    blob32 = blob.astype(np.float32)
    T32 = T.astype(np.float32)
    # a warm-up pass (first touch of the buffers), then one pass of each
    # gather variant picks the faster one
    ref.pipeline_f32(c, s, blob32, T32, x, threads=cores, reps=1)
    variants = {}
    for sg in (False, True):
        _, ms = ref.pipeline_f32(c, s, blob32, T32, x, threads=cores, sorted_gather=sg, reps=1)
        variants["sorted" if sg else "plain"] = ms
    best = min(variants, key=variants.get)
    sg = best == "sorted"
    for _ in range(max(0, warmup - 1)):
        ref.pipeline_f32(c, s, blob32, T32, x, threads=cores, sorted_gather=sg, reps=1)
    times = [ref.pipeline_f32(c, s, blob32, T32, x, threads=cores, sorted_gather=sg, reps=1)[1]
             for _ in range(steps)]
    ms = float(np.mean(times))
    # single core, plain gather, 1024 tokens
    n1 = min(n, 1024)
    _, t1 = ref.pipeline_f32(c, s, blob32, T32, x[:n1], threads=1, reps=1)
    # float64 lookup_forward (the reference's verification path: OpenMP
    # projection, serial gather) on 256 tokens
    n64 = min(n, 256)
    t0 = time.perf_counter()
    ref.lookup_forward(c, s, blob, T, x[:n64].astype(np.float64))
    t64 = (time.perf_counter() - t0) * 1e3
    return {
        "ms": ms, "n": n, "gather": best,
        "variants_tokens_per_s": {k: round(n / (v * 1e-3), 1) for k, v in variants.items()},
        "single_core_tokens_per_s": round(n1 / (t1 * 1e-3), 1),
        "f64_lookup_forward_tokens_per_s": round(n64 / (t64 * 1e-3), 1),
        "sample": (f"the full {n}-token batch of {w.name} per step through the reference f32 "
                   f"kernels (bench.cpp:115-217, {best} gather, the faster of plain / sorted), "
                   f"256-row tiles over {cores} OpenMP threads; inputs built by the reference "
                   f"library (liblffn_ref.so); {cpu_model()}"),
    }


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return None
    from paper_2403_07221_b200.configs import WORKLOADS

    w = WORKLOADS[args.config]
    cores = host_cores()
    m = reference_measure(args, w, args.steps, args.warmup, cores)
    value = m["n"] / (m["ms"] * 1e-3)
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 1),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(m["ms"], 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (same seeds as the ours arm, generated by the reference library)",
        "config": {"workload": f"{w.name}: d_in=d_out={w.d} h={w.h} tau={w.tau} n={w.n} "
                               f"{args.kind} f32 tables (the reference f32 pipeline)",
                   "tokens_per_step": m["n"]},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores,
                         "kind": "reference", "sample": m["sample"],
                         "gather_variants_tokens_per_s": m["variants_tokens_per_s"],
                         "single_core_tokens_per_s": m["single_core_tokens_per_s"],
                         "f64_lookup_forward_tokens_per_s": m["f64_lookup_forward_tokens_per_s"]},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def cpu_baseline_for(args):
    """cpu_baseline of the ours line: the same measurement as the reference
    arm (full batch, all host cores, faster gather variant), fewer steps."""
    from paper_2403_07221_b200.configs import WORKLOADS

    w = WORKLOADS[args.config]
    cores = host_cores()
    m = reference_measure(args, w, 3, 1, cores)
    return {"value": round(m["n"] / (m["ms"] * 1e-3), 1), "unit": UNIT, "cores": cores,
            "kind": "reference", "sample": m["sample"],
            "gather_variants_tokens_per_s": m["variants_tokens_per_s"],
            "single_core_tokens_per_s": m["single_core_tokens_per_s"],
            "f64_lookup_forward_tokens_per_s": m["f64_lookup_forward_tokens_per_s"]}


def relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: launch N ranks the way the
    driver does (torch.distributed.run, one process per GPU, 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out = run_ours(args)
    if out is not None:
        if args.gpus == 1 and not args.no_cpu_baseline:
            try:
                out["cpu_baseline"] = cpu_baseline_for(args)
            except Exception as e:  # the baseline is reported, never required
                out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
