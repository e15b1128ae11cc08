"""`python -m paper_2406_14116_b200 run ...` — the GPU `run` verb of the reference CLI.

Mirrors `fcvbw run` (proj/tools/fcvbw_cli.cpp:72-118, options :301-309): design artifact JSON,
f64le / CSV real signal, optional schedule CSV of (block_index, b_N) events applied before the
named block, initial b (default bN_low). Exit codes follow fcvbw_cli.cpp:16-17,338-355:
0 ok, 2 validation (bad schedule, b out of range, bad files), 1 other errors. The whole stream is
filtered through the C-ABI's real-input host path (fcvbw_gpu_run_real_host: two blocks per complex
transform, H2D / kernel / D2H pipelined).
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

from .bins import Error, ValidationError
from .engine import new_engine
from .io import load_artifact, read_schedule_csv, read_signal, schedule_to_blocks, write_signal


def cmd_run(artifact: str, inp: str, out: str, fmt: str, schedule: str | None, initial_b: int) -> int:
    result = load_artifact(artifact)
    x = read_signal(inp, fmt)
    bins = result.bins
    m = bins.block_length
    nblocks = (x.size + m - 1) // m
    b0 = initial_b if initial_b >= 0 else bins.b_low
    if not bins.contains_b(b0):
        raise ValidationError(f"engine: bandwidth {b0} outside design range [{bins.b_low}, {bins.b_high}]")
    events = read_schedule_csv(schedule) if schedule else []
    for line, (blk, b) in enumerate(events, 1):  # load_schedule (fcvbw_cli.cpp:25-42) checks b first
        if not bins.contains_b(b):
            raise ValidationError(f"{schedule}: schedule entry {line} ({blk},{b}) requests b_N outside the "
                                  f"design range [{bins.b_low}, {bins.b_high}]")
    sched = schedule_to_blocks(events, nblocks, b0, bins)
    eng = new_engine(result, b0, dtype="c128")
    y = eng.run_real_host(x, sched) if x.size else np.zeros(0)  # block pairs per transform
    write_signal(out, np.ascontiguousarray(y), fmt)
    applied = sum(1 for blk, _ in events if blk < nblocks)
    print(f"run: {x.size} samples, {nblocks} blocks, b0 = {b0}, switches applied = {applied}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2406_14116_b200",
                                 description="GPU overlap-save VBW filter (the `run` verb of fcvbw)")
    sub = ap.add_subparsers(dest="verb", required=True)
    r = sub.add_parser("run", help="stream a signal through a designed filter")
    r.add_argument("--artifact", required=True)
    r.add_argument("--input", required=True)
    r.add_argument("--output", required=True)
    r.add_argument("--format", default="csv", choices=None)
    r.add_argument("--schedule", default="")
    r.add_argument("--b", type=int, default=-1)
    args = ap.parse_args(argv)
    try:
        if args.verb == "run":
            return cmd_run(args.artifact, args.input, args.output, args.format, args.schedule or None, args.b)
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (Error, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
