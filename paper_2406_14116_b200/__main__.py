"""`python -m paper_2406_14116_b200 {run,design,analyze} ...` — the reference CLI's verbs on the GPU.

`design` and `analyze` (fcvbw_cli.cpp:44-70, 120-193) are the design-side verbs: the minimax
design, its dense-grid verification and the analysis tables, all computed by libfcvbw_gpu.so
(csrc/design.cu, verify.cu, analyze.cu). Exit codes as the reference: 0 ok, 1 requirement not met /
other error, 2 validation (incl. off-grid specs), 3 no convergence.

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

from .bins import Error, NonConvergenceError, ValidationError
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


def cmd_design(spec_path: str, artifact_path: str, report_path: str, dense_k: int) -> int:
    from .design import design
    from .io import parse_spec_file, save_artifact, save_verification
    from .verify import verify
    spec, opt = parse_spec_file(spec_path)
    result = design(spec, opt)
    if dense_k <= 0:
        dense_k = 4 * opt.grid_points
    report = verify(result, dense_k, spec.max_error, exact=True)
    result.verification = report.delta
    save_artifact(artifact_path, result)
    save_verification(report_path, report)
    b = result.bins
    print(f"design: L = {b.filter_length}, N = {b.fft_length}, M = {b.block_length}, delta_N = "
          f"{b.transition_width_bins}, b_N in [{b.b_low}, {b.b_high}]\n"
          f"delta achieved (grid K = {result.grid_points}): {'%.17g' % result.delta}\n"
          f"dense recheck (K = {dense_k}): {'%.17g' % report.delta}{'  [pass]' if report.passed else '  [fail]'}\n"
          f"orders evaluated: {result.iterations}, exchange rounds: {result.exchange_rounds}\n"
          f"artifact: {artifact_path}\nreport:   {report_path}")
    return 0 if result.delta <= spec.max_error else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2406_14116_b200",
                                 description="GPU overlap-save VBW filter: the run / design / analyze verbs of fcvbw")
    sub = ap.add_subparsers(dest="verb", required=True)
    r = sub.add_parser("run", help="stream a signal through a designed filter")
    r.add_argument("--artifact", required=True)
    r.add_argument("--input", required=True)
    r.add_argument("--output", required=True)
    r.add_argument("--format", default="csv", choices=None)
    r.add_argument("--schedule", default="")
    r.add_argument("--b", type=int, default=-1)
    d = sub.add_parser("design", help="design a filter from a requirements file")
    d.add_argument("--spec", required=True)
    d.add_argument("--artifact", default="design.json")
    d.add_argument("--verify-report", default="verify.json")
    d.add_argument("--dense-k", type=int, default=0)
    a = sub.add_parser("analyze", help="emit frequency responses, errors and PTVIR tables")
    a.add_argument("--artifact", required=True)
    a.add_argument("--grid", type=int, default=1000)
    a.add_argument("--b", default="all")
    a.add_argument("--out-prefix", default="analysis")
    a.add_argument("--per-phase", action="store_true")
    args = ap.parse_args(argv)
    try:
        if args.verb == "run":
            return cmd_run(args.artifact, args.input, args.output, args.format, args.schedule or None, args.b)
        if args.verb == "design":
            return cmd_design(args.spec, args.artifact, args.verify_report, args.dense_k)
        if args.verb == "analyze":
            from .analysis import analyze
            analyze(args.artifact, args.grid, args.b, args.out_prefix, args.per_phase)
            return 0
    except NonConvergenceError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (Error, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
