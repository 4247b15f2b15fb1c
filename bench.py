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
        small = {}
        for m in (1, 8, 64):
            res = {}
            for cold in (False, True):
                ts = []
                for r in range(60):
                    if cold:
                        flush.fill_(r & 0xFF)
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
                "bound": "hbm",
                "kernel": "gather_accumulate",
                "achieved": round(achieved, 1),
                "peak": round(peak_eff, 1),
                "unit": "GB/s",
                "frac": round(achieved / peak_eff, 4),
                # dram__bytes_read.sum + dram__bytes_write.sum of the gather
                # launch, bytes, from the committed ncu --set full capture
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "traffic_source": (traffic or {}).get("source"),
                "definition": "BASELINE north_star gather roofline: t_roof = U/BW_HBM + G/BW_L2; "
                              "achieved = G / gather time, peak = G / t_roof (frac = t_roof/t)",
                "gathered_bytes_G": int(G),
                "unique_bytes_U": int(U),
                "bw_hbm_gbs": hbm,
                "bw_hbm_source": peak_src + " MEASURED_PEAKS.json hbm_gbs",
                "bw_l2_gbs": round(l2, 1),
                "bw_l2_source": "measured live (lffn_probe_bandwidth, 32 MiB re-read)",
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
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if sharded is not None:
        sharded.close()
    else:
        layer.close()
    return result


# ---------------------------------------------------------------- reference
def reference_sample(args, w, n_sample, threads, reps):
    """Time the reference's float32 inference kernels on host cores."""
    from oracle import Reference, Spec, Cfg
    from paper_2403_07221_b200 import ProjKind
    from paper_2403_07221_b200.configs import make_params, make_x

    ref = Reference()
    kind = ProjKind[args.kind]
    cfg, proj, T = make_params(w, kind)
    x = make_x(w, n_sample)
    c = Cfg(cfg.d_in, cfg.d_out, cfg.tables, cfg.code_bits)
    s = Spec(proj.spec.d_in, proj.spec.d_out, int(kind))
    blob32 = proj.blob.astype(np.float32)
    T32 = T.data.astype(np.float32)
    del T
    times = []
    for _ in range(reps):
        _, ms = ref.pipeline_f32(c, s, blob32, T32, x, threads=threads, reps=1)
        times.append(ms)
    return times


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return None
    from paper_2403_07221_b200.configs import WORKLOADS

    w = WORKLOADS[args.config]
    cores = host_cores()
    n_sample = args.cpu_sample or min(w.n, 4096)
    for _ in range(args.warmup):
        pass
    times = reference_sample(args, w, n_sample, cores, args.warmup + args.steps)[args.warmup:]
    ms = float(np.mean(times))
    value = n_sample / (ms * 1e-3)
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 1),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (same seeds as the ours arm)",
        "config": {"workload": f"{w.name}: d_in=d_out={w.d} h={w.h} tau={w.tau} {args.kind}; "
                               f"each step a {n_sample}-token sample",
                   "tokens_per_step": n_sample},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores,
                         "kind": "reference",
                         "sample": f"{n_sample} tokens/step of {w.name}; reference f32 kernels "
                                   "(bench.cpp:115-217) over 256-row tiles spread on "
                                   f"{cores} OpenMP threads; {cpu_model()}"},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def cpu_baseline_for(args):
    """cpu_baseline of the ours line: the reference on a bounded sample."""
    from paper_2403_07221_b200.configs import WORKLOADS

    w = WORKLOADS[args.config]
    cores = host_cores()
    n_sample = min(w.n, 8192)
    times = reference_sample(args, w, n_sample, cores, 2)
    ms = min(times)
    t1 = reference_sample(args, w, min(w.n, 1024), 1, 1)[0]
    return {"value": round(n_sample / (ms * 1e-3), 1), "unit": UNIT, "cores": cores,
            "kind": "reference",
            "sample": f"{n_sample} tokens of {w.name} through the reference f32 kernels "
                      f"(bench.cpp:115-217), 256-row tiles on {cores} threads; {cpu_model()}",
            "single_core_tokens_per_s": round(min(w.n, 1024) / (t1 * 1e-3), 1)}


def main():
    args = parse()
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
