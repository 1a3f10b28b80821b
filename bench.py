#!/usr/bin/env python
"""Benchmark: batched CHW (dyadic-order orthonormal WHT) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Metric (BASELINE.json): CHW-WHT Gelem/s and HBM GB/s (% of measured peak).
A "step" is one batched transform of the configuration's whole batch of rows
(BASELINE.json configs; default cfg2 = configs[1], the config the metric is
quoted on: 65536 fp32 rows of 2^12, N(0,1)).  Multi-GPU: one process per GPU
(torchrun), each rank transforms its own 65536-row shard of an N x 65536 global
batch — rows are independent, so there is no collective on the data path
(weak scaling); the timed region is bracketed by barrier + synchronize and the
slowest rank's device time is reported.

ours (default): inputs resident in HBM, kernels launched through the C ABI
  (chw_b200_forward) on the current stream, timed with CUDA events.  `e2e`
  times chw_b200_forward_host (HOST pinned buffers: H2D + kernels + D2H per
  step) — the reference-facing call.
reference: the reference's own CPU implementation (oracle/_ref/libchw_ref.so:
  the unmodified proj/include headers; else the C restatement) on all host
  cores over a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# BASELINE.json configs -> (name, dtype, rows, m, distribution)
CONFIGS = {
    "cfg1": ("cfg1: 1024 x 2^10 f64, U[-1,1)", "f64", 1024, 10, "uniform"),
    "cfg2": ("cfg2: 65536 x 2^12 f32, N(0,1)", "f32", 65536, 12, "normal"),
    "cfg3": ("cfg3: 1048576 x 2^7 bf16 in/out, fp32 math, N(0,1)", "bf16", 1 << 20, 7, "normal"),
    "cfg4": ("cfg4: 4096 x 2^16 f32, U[-1,1)", "f32", 4096, 16, "uniform"),
    "cfg5": ("cfg5: 256 x 2^24 f32, N(0,1)", "f32", 256, 24, "normal"),
}
ELEM_BYTES = {"f64": 8, "f32": 4, "bf16": 2}
SEED = 1609066410


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy, burst)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic(cfg: str):
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg)
    return None


class ClockSampler:
    """NVML sampler thread: SM clock + throttle reasons while the GPU is busy."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.samples = []
        self.ok = False
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML here
            self.err = str(e)
            self.max_mhz = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((sm, util, r))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        busy = [s for s in self.samples if s[1] > 0] or self.samples
        reasons = set()
        for _, _, r in busy:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(busy)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_input(torch, cfg, rows, dev, rank):
    _, dt, _, m, dist = CONFIGS[cfg]
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + rank)
    n = 1 << m
    if dist == "normal":
        x = torch.randn(rows, n, generator=g, device=dev, dtype=torch.float32)
    else:
        x = torch.rand(rows, n, generator=g, device=dev, dtype=torch.float32) * 2 - 1
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dt]
    if dt == "f64":
        x = (torch.rand(rows, n, generator=g, device=dev, dtype=torch.float64) * 2 - 1) if dist == "uniform" \
            else torch.randn(rows, n, generator=g, device=dev, dtype=torch.float64)
    return x.to(tdt).contiguous()


def cpu_reference_rate(cfg: str, rows: int, reps: int = 1, threads: int = 0):
    """Reference CPU implementation (oracle/_ref if built, else the C port) on
    all host cores; returns (Gelem/s best-of-reps, kind, cores, sample text)."""
    import numpy as np

    import oracle

    _, dt, _, m, dist = CONFIGS[cfg]
    n = 1 << m
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal((rows, n)) if dist == "normal" else rng.uniform(-1, 1, (rows, n))
    if dt == "f32":
        x = x.astype(np.float32).astype(np.float64)  # exact upcast of the fp32 bytes
    elif dt == "bf16":
        import torch

        x = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    x = np.ascontiguousarray(x)
    kind = "reference" if oracle.have_reference() else "port"
    cores = threads if threads > 0 else (os.cpu_count() or 1)
    best = math.inf
    for _ in range(reps):
        buf = x.copy()
        t0 = time.perf_counter()
        oracle.chw_batch_inplace(buf, oracle.ORTHONORMAL, backend=kind, threads=cores)
        best = min(best, time.perf_counter() - t0)
    gel = rows * n / best / 1e9
    sample = (f"{rows} rows x 2^{m} of {cfg}, reference chw_forward_inplace<double> Orthonormal per row, "
              f"rows split over {cores} threads, best of {reps}; input upcast to f64 outside the timer")
    return gel, kind, cores, sample, best


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    name, dt, rows_full, m, _ = CONFIGS[cfg]
    n = 1 << m
    # bounded sample per step: ~128M elements (or the whole batch if smaller)
    rows = max(1, min(rows_full, (1 << 27) >> m))
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, max(1, rows // 8))
    times = []
    for _ in range(args.steps):
        gel, kind, cores, sample, t = cpu_reference_rate(cfg, rows)
        times.append(t)
    tot = sum(times)
    value = args.steps * rows * n / tot / 1e9
    line = {
        "impl": "reference", "metric": "CHW-WHT Gelem/s", "value": round(value, 4), "unit": "Gelem/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic seed {SEED}",
        "config": {"workload": name, "global_batch": rows_full * world, "n": n, "rows_per_step": rows},
        "cpu_baseline": {"value": round(value, 4), "unit": "Gelem/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as tdist

    import paper_1609_06641_b200 as chw

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    cfg = args.config
    name, dt, rows, m, dist_name = CONFIGS[cfg]
    n = 1 << m
    es = ELEM_BYTES[dt]
    x = make_input(torch, cfg, rows, dev, rank)
    out = torch.empty_like(x)
    ws_bytes = chw.workspace_bytes({"f64": 0, "f32": 1, "bf16": 2}[dt], rows, n)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    order = {"dyadic": chw.ORDER_DYADIC, "natural": chw.ORDER_NATURAL}[args.order]

    def step():
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out, stream=stream,
                                 workspace=ws if ws_bytes else None, order=order)

    # L2 policy: inputs larger than L2 need no flush; smaller ones get a flush write between steps.
    footprint = 2 * rows * n * es
    flush = None
    if footprint < 4 * 126 * 2**20:
        flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
        # A write flush leaves L2 full of dirty lines whose write-back would land
        # inside the next timed step; reading a second clean buffer afterwards
        # evicts them before the step starts (the step still starts cold).
        clean = torch.ones(64 * 2**20, dtype=torch.float32, device=dev)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()

    # clock soak: keep the GPU busy ~1 s before the timed region so NVML sees load
    sampler = ClockSampler(local)
    with sampler:
        t_end = time.time() + args.soak
        while time.time() < t_end:
            for _ in range(8):
                step()
            torch.cuda.synchronize()
        barrier()
        launches0 = chw.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_stop = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
                clean.sum()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        t_stop.record(stream)
        barrier()
        launches = chw.launch_count() - launches0
    kern_ms = [a.elapsed_time(b) for a, b in evs]
    total_kern_ms = sum(kern_ms)
    wall_region_ms = t_start.elapsed_time(t_stop)
    t = torch.tensor([total_kern_ms], device=dev, dtype=torch.float64)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    elems_all = rows * n * world
    value = elems_all / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel family (all launches of one step = the transform)
    peak, peak_src = load_peaks()
    alg_bytes = 2 * rows * n * es
    achieved = alg_bytes / (statistics.mean(kern_ms) * 1e-3) / 1e9
    traffic = load_traffic(cfg)

    # copy peak in the same run (K0): one read + one write of a 1 GiB buffer
    a = torch.empty(2**30, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    cps = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        cps.append(2 * 2**30 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    copy_peak = max(cps)
    del a, b

    # e2e through the host-buffer C-ABI call (pinned host in/out, H2D + kernels + D2H)
    hx = x.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    e2e_steps = max(2, min(args.steps, args.e2e_steps))
    chw.chw_forward_host_(hx, chw.ScalingMode.Orthonormal, out=hy)  # warm-up (allocates staging)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        chw.chw_forward_host_(hx, chw.ScalingMode.Orthonormal, out=hy)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    if world > 1:
        tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
    e2e_value = elems_all * e2e_steps / float(te.item()) / 1e9
    # e2e result must equal the device result
    e2e_ok = bool(torch.equal(hy.to(dev), out))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_rows = rows if cfg != "cfg5" else 2
        gel, kind, cores, sample, _ = cpu_reference_rate(cfg, min(rows, cpu_rows), reps=1)
        cpu = {"value": round(gel, 4), "unit": "Gelem/s", "cores": cores, "kind": kind, "sample": sample}

    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": "CHW-WHT Gelem/s", "value": round(value, 3), "unit": "Gelem/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dt,
            "data": f"synthetic {dist_name} (torch Philox, seed {SEED}+rank), generated on device",
            "config": {
                "workload": name, "global_batch": rows * world, "per_rank_batch": rows, "n": n,
                "parallelism": f"batch-sharded x{world}, no collective on the data path",
                "l2": "inputs+outputs larger than L2 (no flush)" if flush is None
                else "L2 flushed before every timed step (256 MiB write, then a 256 MiB read that writes the "
                "flush's dirty lines back outside the timed region)",
                "plan": chw.plan_name({"f64": 0, "f32": 1, "bf16": 2}[dt], n) if args.order == "dyadic"
                else "natural-order k1 generic",
                "order": args.order,
            },
            "hbm_gbs": round(achieved, 1), "pct_of_peak": round(100 * achieved / peak, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes,
                         "copy_peak_same_run_gbs": round(copy_peak, 1)},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "Gelem/s",
                    "h2d_bytes_per_step": rows * n * es, "d2h_bytes_per_step": rows * n * es,
                    "matches_device_result": e2e_ok, "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clocks,
            "timed_region_ms": round(wall_region_ms, 3),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--soak", type=float, default=1.0, help="seconds of untimed load before timing")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--order", default="dyadic", choices=["dyadic", "natural"],
                    help="output order (the BASELINE metric is dyadic; natural is for experiments)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
