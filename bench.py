#!/usr/bin/env python
"""Benchmark of the B200 overlap-save VBW filter (BASELINE.json metric).

Default workload = BASELINE.json configs[2] ("c3"), the N = 1024 fp32 config the metric's
"at 1/2/4/8 B200" refers to: 1024 independent complex float32 channels x 2^20 samples, N = 1024,
M = 768 (BASELINE "L"), delta_N = 12, one seeded b_N per channel over 0.05 pi - 0.9 pi, channels
sharded across the GPUs (strong scaling: the job is fixed, each rank takes 1024/N channels, no
collective on the data path). One step = every channel through the fused kernel once.
`--config c2` runs configs[1] (one 2^24-sample stream, b redrawn every 64 blocks; weak scaling:
each rank its own stream).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

`value` = all ranks' samples / max-over-ranks device time of the K timed steps.
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


_REDUCE_ON_CPU = False


def dist_setup(args):
    """One process per GPU. NCCL carries only the barrier and the max-over-ranks timing reduction.
    If there are fewer visible GPUs than local ranks (a functional test of the multi-rank path on a
    1-GPU box), ranks share devices round-robin and the reduction falls back to gloo."""
    global _REDUCE_ON_CPU
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "gloo"
        if args.impl == "ours":
            ndev = torch.cuda.device_count()
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
            if ndev >= local_world:
                backend = "nccl"
                torch.cuda.set_device(local)
            else:
                local = local % max(1, ndev)
                torch.cuda.set_device(local)
        _REDUCE_ON_CPU = backend == "gloo"
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
    t = torch.tensor([v], dtype=torch.float64, device=None if _REDUCE_ON_CPU else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_run(w, threads: int):
    """One pass of the reference C++ engine over the workload (complex = 2 real engines)."""
    from oracle import oracle as O
    lib = O.best()
    b = w.bins
    sched = w.b_schedule()
    x = np.stack([w.input(c) for c in range(w.channels)]).astype(np.complex128)
    t0 = time.perf_counter()
    lib.ols_complex(b.fft_length, b.filter_length, b.transition_width_bins, b.b_low, b.b_high,
                    np.array(w.design.profile.values), x, bsched=sched, threads=threads)
    return time.perf_counter() - t0, x.size, lib.kind


def run_reference(args, w, world, rank):
    if rank != 0:
        return
    scaling = args.scaling  # the workload's own label (the sample below is bounded either way)
    if w.samples * w.channels > 2 ** 24:  # bounded sample per step (same N, M, schedule rule)
        from paper_2406_14116_b200.workload import config as _cfg
        ch = max(1, min(w.channels, 2 ** 24 // min(w.samples, 2 ** 24)))
        w = _cfg(w.name, samples=min(w.samples, 2 ** 24), channels=ch)
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
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded complex Gaussian, BASELINE {w.name} shape)",
        "config": {"workload": w.name, "N": w.bins.fft_length, "M": w.bins.block_length,
                   "samples_per_step": n, "channels": w.channels, "schedule": w.schedule},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{w.channels} channel(s) x {w.samples} samples of {w.name} ({n} complex "
                                   f"samples) per step, fp64 reference OlsEngine x2 (Re, Im) per channel, "
                                   f"{threads} threads over (channel, block-range) units"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_input(w, rank, dev, host_limit=2 ** 27):
    """[channels, S] input on the device. Up to host_limit samples: the seeded host generator
    (workload.complex_gaussian, identical to what the parity tests use); beyond that (C4's 2^31
    samples): torch's seeded device Philox generator, still unit-variance complex Gaussian."""
    import torch
    tdt = torch.complex64 if w.dtype == "c64" else torch.complex128
    total = w.samples * w.channels
    if total <= host_limit:
        x_host = np.stack([w.input(channel=rank * w.channels + c) for c in range(w.channels)])
        return torch.from_numpy(x_host).to(dev), x_host
    gen = torch.Generator(device=dev)
    gen.manual_seed(w.seed * 1_000_003 + rank)
    rdt = torch.float32 if w.dtype == "c64" else torch.float64
    x = torch.empty((w.channels, w.samples), dtype=tdt, device=dev)
    xr = torch.view_as_real(x)
    xr.normal_(0.0, 0.5 ** 0.5, generator=gen)
    return x, None


def run_ours(args, w, world, rank, local):
    import torch

    from paper_2406_14116_b200 import OlsEngine
    from paper_2406_14116_b200.shard import block_shards

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b = w.bins
    esize = 8 if w.dtype == "c64" else 16
    sched_np = w.b_schedule()
    eng = OlsEngine(b, w.design.profile, int(np.ravel(sched_np)[0]), dtype=w.dtype, device=local)

    # multichannel (strong): rank r takes a contiguous channel shard of the fixed job;
    # single stream, weak: rank r processes its own full-size stream (seeded by r);
    # single stream, strong: the stream's blocks are split into contiguous ranges (halo N - M)
    from paper_2406_14116_b200.shard import channel_shards
    S_total = w.samples
    run_args = None
    if w.channels > 1 and args.scaling == "strong":
        cs = channel_shards(w.channels, world)[rank]
        w_rank = type(w)(**{**w.__dict__, "channels": cs.ch_end - cs.ch_begin})
        sched_np = sched_np[cs.ch_begin:cs.ch_end] if np.ndim(sched_np) == 2 else sched_np
        x0, x_host = make_input(w_rank, rank, dev)
        S_rank = w.samples * w_rank.channels
        w_rank_channels = w_rank.channels
    else:
        x0, x_host = make_input(w, 0 if args.scaling == "strong" else rank, dev)
        w_rank_channels = w.channels
        if args.scaling == "strong":
            sh = block_shards(w.samples, b.fft_length, b.block_length, world)[rank]
            x0 = x0[:, sh.x_begin:sh.x_end].contiguous()
            S_rank = (sh.y_end - sh.y_begin) * w.channels
            run_args = dict(x_first=sh.x_begin, blk=(sh.blk_begin, sh.blk_end), y_first=sh.y_begin,
                            ylen=sh.y_end - sh.y_begin)
        else:
            S_rank = w.samples * w.channels
    input_desc = ("seeded host generator (workload.complex_gaussian)" if x_host is not None
                  else "torch seeded device Philox normal_, unit-variance complex Gaussian")
    in_bytes = x0.numel() * esize
    l2 = 126 * 2 ** 20
    nbuf = 1 if in_bytes > 4 * l2 else max(3, min(64, -(-3 * l2 // (2 * in_bytes))))
    xs = [x0] + [x0.clone() for _ in range(nbuf - 1)]
    if run_args is None:
        ys = [torch.empty_like(xs[0]) for _ in range(nbuf)]
    else:
        ys = [torch.empty((w.channels, run_args["ylen"]), dtype=x0.dtype, device=dev) for _ in range(nbuf)]
    bd = torch.from_numpy(np.ascontiguousarray(sched_np)).to(dev)

    if args.real:
        # real channels: the real parts of the complex workload; bytes per sample halve
        xs = [x.real.contiguous() if x.is_complex() else x for x in xs]
        ys = [torch.empty_like(xs[0]) for _ in range(nbuf)]
        esize //= 2
        sn = np.asarray(sched_np)
        real_paired = bool(sn.ndim == 1 or (sn.shape[0] % 2 == 0 and np.array_equal(sn[0::2], sn[1::2])))

    def step(i, trusted=True):
        if args.real:
            eng.run_real(xs[i % nbuf], bd, y_dev=ys[i % nbuf], trusted_schedule=trusted,
                         paired_schedules=real_paired)
        elif run_args is None:
            eng.run(xs[i % nbuf], bd, y_dev=ys[i % nbuf], trusted_schedule=trusted)
        else:
            eng.run_range(xs[i % nbuf], run_args["x_first"], S_total, *run_args["blk"], y_dev=ys[i % nbuf],
                          y_first=run_args["y_first"], b_sched=bd, trusted_schedule=trusted)

    step(0, trusted=False)  # validates the schedule once (synchronising range check)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        step(i)
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
            step(i)
            ends[i].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        launches = eng.kernel_launches() - launches0
        # keep the device loaded (untimed) long enough for several clock samples
        extra_t0 = time.perf_counter()
        while time.perf_counter() - extra_t0 < 0.5:
            for i in range(20):
                step(i)
            torch.cuda.synchronize()
    barrier(world)
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    elapsed_ms = max_over_ranks(elapsed_ms, world, dev)
    ms_step = elapsed_ms / args.steps
    samples_all = S_rank * world if (args.scaling == "weak" and w.channels == 1) else S_total * w.channels
    value = samples_all * args.steps / (elapsed_ms * 1e-3)

    # roofline of the (only) kernel: algorithmic bytes per launch / its average duration
    hbm, hbm_src = peaks()
    alg_bytes = 2 * esize * S_rank  # one read + one write per complex sample
    kavg = statistics.mean(kern_ms) * 1e-3
    achieved = alg_bytes / kavg / 1e9
    traffic = traffic_for(w.name + ("_real" if args.real else ""))
    full_bytes = 2 * esize * w.samples * w.channels
    if traffic is not None and alg_bytes != full_bytes:  # profiled launch covered the whole job
        traffic = int(traffic * alg_bytes / full_bytes)

    # e2e through the public host-memory API: pinned host buffers, H2D + kernel + D2H per step
    e2e = None
    if run_args is None and x_host is None and not args.no_e2e:
        x_host = xs[0].cpu().numpy()  # device-generated input: the e2e run starts from a host copy
    if run_args is None and not args.no_e2e:
        if args.real:
            x_host = np.ascontiguousarray(np.asarray(x_host).real)
        xh = torch.from_numpy(x_host).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        sched_h = np.ascontiguousarray(sched_np, np.int32)
        bcs = sched_h.shape[-1] if sched_h.ndim == 2 else 0
        e2e_steps = max(3, min(args.steps, 10))
        host_fn = eng.run_real_host_ptr if args.real else eng.run_host_ptr
        host_fn(xh.data_ptr(), w.samples, w_rank_channels, yh.data_ptr(), sched_h.ctypes.data, bcs)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            host_fn(xh.data_ptr(), w.samples, w_rank_channels, yh.data_ptr(), sched_h.ctypes.data, bcs)
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, dev)
        y_dev0 = (eng.run_real(xs[0], bd, trusted_schedule=True) if args.real
                  else eng.run(xs[0], bd, trusted_schedule=True))
        e2e = {"value": samples_all * e2e_steps / e2e_s, "unit": "real samples/s" if args.real else UNIT,
               "h2d_bytes_per_step": int(esize * S_rank + 4 * sched_h.size),
               "d2h_bytes_per_step": int(esize * S_rank), "steps": e2e_steps,
               "path": ("fcvbw_gpu_run_real_host" if args.real else "fcvbw_gpu_run_host") +
                       " (pinned host buffers, H2D/kernel/D2H pipelined over 3 streams)",
               "bitwise_equal_to_device_run": bool(torch.equal(y_dev0.cpu(), yh))}

    line = {
        "metric": METRIC if not args.real else "real output samples/sec (real-input fast path), " + METRIC,
        "value": value, "unit": "real samples/s" if args.real else UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32" if w.dtype == "c64" else "f64",
        "data": f"synthetic (seeded complex Gaussian, BASELINE {w.name} shape; V from the reference design())",
        "config": {"workload": w.name, "N": b.fft_length, "M": b.block_length, "L_ref": b.filter_length,
                   "delta_N": b.transition_width_bins, "samples_per_rank": S_rank, "channels": w.channels,
                   "schedule": w.schedule,
                   "parallelism": (f"channel shards x{world} ({w_rank_channels} channels per GPU)" if w.channels > 1
                                   else f"independent streams x{world}" if args.scaling == "weak"
                                   else f"block ranges x{world} (halo {b.fft_length - b.block_length})"),
                   "input": input_desc,
                   "l2": (f"{nbuf} rotating input/output buffer sets ({nbuf * 2 * in_bytes / 2**20:.0f} MiB) > 126 MB L2"
                          if nbuf > 1 else f"input {in_bytes / 2**20:.0f} MiB > 4x L2, single buffer set")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_source": hbm_src,
                     "kernel_ms_avg": kavg * 1e3, "algorithmic_bytes_per_launch": alg_bytes},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        t_acc, n_acc, kind = 0.0, 0, None
        reps = 0
        wc = w if w.samples * w.channels <= 2 ** 24 else None
        if wc is None:
            from paper_2406_14116_b200.workload import config as _cfg
            wc = _cfg(w.name, samples=min(w.samples, 2 ** 24), channels=1)
        while t_acc < args.cpu_seconds and reps < 50:
            dt, n, kind = cpu_reference_run(wc, threads)
            t_acc += dt
            n_acc += n
            reps += 1
        line["cpu_baseline"] = {"value": n_acc / t_acc, "unit": UNIT, "cores": threads, "kind": kind,
                                "sample": f"{reps} pass(es) over {wc.samples * wc.channels} complex samples of "
                                          f"{w.name} (same N, M, schedule), fp64 reference engine, "
                                          f"{threads} threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=None, help="override samples per channel")
    ap.add_argument("--channels", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--real", action="store_true",
                    help="real-input fast path (fcvbw_gpu_run_real): the workload's channels as REAL signals")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="default: strong (channel shards) for multichannel configs, weak otherwise")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2406_14116_b200.workload import config
    w = config(args.config, samples=args.samples, channels=args.channels)
    if args.scaling is None:
        args.scaling = "strong" if w.channels > 1 else "weak"
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
