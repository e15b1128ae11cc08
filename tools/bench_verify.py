"""Times the GPU design verification (csrc/verify.cu) against the reference's verify()
(design.hpp:601-673, oracle/_ref or the C port) on a config artifact's full band-centre range.

The CPU side runs a bounded sample (`--cpu-bands` band centres spread over the range; the
reference parallelises over b with all host threads) and is scaled to the full range by
ceil(num_b / cores) waves. Prints one JSON line.

    python tools/bench_verify.py --artifact configs/artifact_n1024_d12.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--artifact", default=os.path.join(ROOT, "configs", "artifact_n1024_d12.json"))
    ap.add_argument("--dense-mult", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-bands", type=int, default=0, help="sample size; 0: one per host core")
    args = ap.parse_args()

    from paper_2406_14116_b200 import BinSpec, DesignResult, TransitionProfile
    from paper_2406_14116_b200.verify import verify

    a = json.load(open(args.artifact))
    n, l, dn, blo, bhi = a["N"], a["L"], a["delta_N"], a["bN_low"], a["bN_high"]
    v = np.array(a["V"])
    dense = args.dense_mult * a["grid_K"]
    bins = BinSpec(n, l, n - l + 1, dn, blo, bhi)
    res = DesignResult(TransitionProfile(list(v)), bins, delta=a["delta_achieved"], grid_points=a["grid_K"],
                       facets=a["facets_P"])
    verify(res, dense, 0.05)  # warm-up (context, module load)
    times = []
    for _ in range(args.reps):
        t = time.perf_counter()
        rep = verify(res, dense, 0.05)
        times.append(time.perf_counter() - t)
    gpu_s = float(np.median(times))

    from oracle import oracle as O
    lib = O.best()
    cores = os.cpu_count() or 1
    nb = args.cpu_bands or cores
    num_b = bhi - blo + 1
    # a contiguous sample of band centres in one verify() call, so that the reference's own
    # parallel_for spreads them over the cores (per-b cost is the same for every b up to the
    # few excluded transition-band points)
    sub_lo = blo + num_b // 2
    sub_hi = min(bhi, sub_lo + min(nb, num_b) - 1)
    t = time.perf_counter()
    r = lib.verify(n, l, dn, sub_lo, sub_hi, v, a["delta_achieved"], a["grid_K"], a["facets_P"], dense, 0.05)
    cpu_sub = time.perf_counter() - t
    cpu_max = float(np.max(r["per_b_max"]))
    threads = cores if lib.kind == "reference" else 1
    waves_sub = -(-(sub_hi - sub_lo + 1) // threads)
    waves_full = -(-num_b // threads)
    cpu_full_est = cpu_sub / waves_sub * waves_full
    gpu_sub = np.array([rep.per_b_max[b] for b in range(sub_lo, sub_hi + 1)])
    print(json.dumps({
        "metric": "design_verify_seconds", "unit": "s", "higher_is_better": False,
        "config": {"artifact": os.path.basename(args.artifact), "N": n, "L": l, "M": n - l + 1, "delta_N": dn,
                   "num_b": num_b, "dense_points": dense},
        "gpu_seconds": gpu_s, "gpu_reps": times,
        "cpu": {"kind": lib.kind, "threads": threads, "sample_bands": [sub_lo, sub_hi],
                "sample_seconds": cpu_sub, "full_range_estimate_seconds": cpu_full_est},
        "speedup_est": cpu_full_est / gpu_s,
        "sample_max_abs_diff": float(np.abs(gpu_sub - r["per_b_max"]).max()),
        "report": {"delta": rep.delta, "worst_b": rep.worst_b, "worst_n": rep.worst_n,
                   "worst_omega": rep.worst_omega, "pass": rep.passed, "within_bound": rep.within_bound},
        "cpu_sample_max": cpu_max,
    }))


if __name__ == "__main__":
    main()
