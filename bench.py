#!/usr/bin/env python
"""Benchmark of the B200 overlap-save VBW filter (BASELINE.json metric).

Default workload = BASELINE.json configs[1] ("c2"): one complex float32 stream of 2^24 samples,
N = 1024, M = 768 (BASELINE "L"), delta_N = 12, b_N redrawn every 64 blocks from the seeded
schedule over 0.05 pi - 0.9 pi. One step = the whole stream through the fused kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Under torchrun each rank processes its own c2-sized stream (weak scaling; independent streams
shard with no collective on the data path); `value` = all ranks' samples / max-over-ranks time.
`--impl reference` times the reference's own C++ engine (oracle/_ref, compiled from the reference
headers; the C restatement if that build is absent) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "complex output samples/sec and % HBM roofline, N=1024 fp32, at 1/2/4/8 B200"
UNIT = "complex samples/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [[c.strip() for c in l.split(",")] for l in self.out.splitlines() if l.count(",") >= 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(s):
            try:
                return float(s)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        loaded = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend, init_method="env://")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int, device=None) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_run(w, threads: int):
    """One pass of the reference C++ engine over the workload (complex = 2 real engines)."""
    from oracle import oracle as O
    lib = O.best()
    b = w.bins
    sched = w.b_schedule()
    x = w.input(0).astype(np.complex128)
    t0 = time.perf_counter()
    lib.ols_complex(b.fft_length, b.filter_length, b.transition_width_bins, b.b_low, b.b_high,
                    np.array(w.design.profile.values), x, bsched=sched, threads=threads)
    return time.perf_counter() - t0, x.size, lib.kind


def run_reference(args, w, world, rank):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    for _ in range(args.warmup):
        cpu_reference_run(w, threads)
    times, n, kind = [], 0, None
    for _ in range(args.steps):
        dt, n, kind = cpu_reference_run(w, threads)
        times.append(dt)
    tot = sum(times)
    value = n * args.steps / tot
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded complex Gaussian, BASELINE c2 shape)",
        "config": {"workload": w.name, "N": w.bins.fft_length, "M": w.bins.block_length,
                   "samples_per_step": n, "channels": w.channels, "schedule": w.schedule},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"full {w.name} stream ({n} complex samples) per step, fp64 reference "
                                   f"OlsEngine x2 (Re, Im) per channel, {threads} threads over block ranges"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, w, world, rank, local):
    import torch

    from paper_2406_14116_b200 import OlsEngine

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b = w.bins
    tdt = torch.complex64 if w.dtype == "c64" else torch.complex128
    esize = 8 if w.dtype == "c64" else 16
    S = w.samples * w.channels
    sched_np = w.b_schedule()
    eng = OlsEngine(b, w.design.profile, int(np.ravel(sched_np)[0]), dtype=w.dtype, device=local)

    # rank r processes its own stream: channel index r of the seeded generator
    x_host = np.stack([w.input(channel=rank * w.channels + c) for c in range(w.channels)])
    nbuf = 3  # rotating buffer sets: each step reads/writes data last touched 3 steps ago
    xs = [torch.from_numpy(x_host).to(dev) for _ in range(nbuf)]
    ys = [torch.empty_like(xs[0]) for _ in range(nbuf)]
    bd = torch.from_numpy(np.ascontiguousarray(sched_np)).to(dev)
    eng.run(xs[0], bd, y_dev=ys[0])  # validates the schedule once (synchronising range check)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        eng.run(xs[i % nbuf], bd, y_dev=ys[i % nbuf], trusted_schedule=True)
    torch.cuda.synchronize()
    launches0 = eng.kernel_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            eng.run(xs[i % nbuf], bd, y_dev=ys[i % nbuf], trusted_schedule=True)
            ends[i].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        launches = eng.kernel_launches() - launches0
        # keep the device loaded (untimed) long enough for several clock samples
        extra_t0 = time.perf_counter()
        while time.perf_counter() - extra_t0 < 0.5:
            for i in range(50):
                eng.run(xs[i % nbuf], bd, y_dev=ys[i % nbuf], trusted_schedule=True)
            torch.cuda.synchronize()
    barrier(world)
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    elapsed_ms = max_over_ranks(elapsed_ms, world, dev)
    ms_step = elapsed_ms / args.steps
    value = S * world * args.steps / (elapsed_ms * 1e-3)

    # roofline of the (only) kernel: algorithmic bytes per launch / its average duration
    hbm, hbm_src = peaks()
    alg_bytes = 2 * esize * S  # one read + one write per complex sample
    kavg = statistics.mean(kern_ms) * 1e-3
    achieved = alg_bytes / kavg / 1e9
    traffic = traffic_for(w.name)

    # e2e through the public host-memory API: pinned host buffers, H2D + kernel + D2H per step
    xh = torch.from_numpy(x_host).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    sched_h = np.ascontiguousarray(sched_np, np.int32)
    bcs = sched_h.shape[-1] if sched_h.ndim == 2 else 0
    e2e_steps = max(3, min(args.steps, 10))
    eng.run_host_ptr(xh.data_ptr(), w.samples, w.channels, yh.data_ptr(), sched_h.ctypes.data, bcs)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.run_host_ptr(xh.data_ptr(), w.samples, w.channels, yh.data_ptr(), sched_h.ctypes.data, bcs)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, dev)
    e2e_value = S * world * e2e_steps / e2e_s
    # spot parity of the e2e result against the device result (same kernel, bit-identical)
    y_dev0 = eng.run(xs[0], bd, trusted_schedule=True)
    e2e_match = bool(torch.equal(y_dev0.cpu(), yh))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if w.dtype == "c64" else "f64",
        "data": "synthetic (seeded complex Gaussian, BASELINE c2 shape; V from the reference design())",
        "config": {"workload": w.name, "N": b.fft_length, "M": b.block_length, "L_ref": b.filter_length,
                   "delta_N": b.transition_width_bins, "samples_per_rank": S, "channels": w.channels,
                   "schedule": w.schedule, "parallelism": f"independent streams x{world}",
                   "l2": f"{nbuf} rotating input/output buffer sets ({nbuf * 2 * esize * S / 2**20:.0f} MiB) > 126 MB L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_source": hbm_src,
                     "kernel_ms_avg": kavg * 1e3, "algorithmic_bytes_per_launch": alg_bytes},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(esize * S + 4 * sched_h.size),
                "d2h_bytes_per_step": int(esize * S), "steps": e2e_steps, "bitwise_equal_to_device_run": e2e_match},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        t_acc, n_acc, kind = 0.0, 0, None
        reps = 0
        while t_acc < args.cpu_seconds and reps < 50:
            dt, n, kind = cpu_reference_run(w, threads)
            t_acc += dt
            n_acc += n
            reps += 1
        line["cpu_baseline"] = {"value": n_acc / t_acc, "unit": UNIT, "cores": threads, "kind": kind,
                                "sample": f"{reps} pass(es) over the full {w.name} stream "
                                          f"({w.samples * w.channels} complex samples each), fp64 reference engine"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=None, help="override samples per channel")
    ap.add_argument("--channels", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2406_14116_b200.workload import config
    w = config(args.config, samples=args.samples, channels=args.channels)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, w, world, rank)
    else:
        run_ours(args, w, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
