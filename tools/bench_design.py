"""Times the GPU-assisted `solve_minimax` (csrc/design.cu) at true geometry N = 3L/4-style configs
(L = N/4 + 1, K = 2N, one band centre b = N/8 as in configs/make_artifacts.py) and, where
`--ref-max-n` allows, the reference's own solve_minimax (oracle/_ref) on the same problem.
Prints one JSON line per N.

    python tools/bench_design.py --n 1024 2048 4096 8192 --ref-max-n 1024
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

DELTA_N = {64: 4, 128: 4, 256: 6, 512: 8, 1024: 12, 2048: 16, 4096: 16, 8192: 32}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1024, 2048, 4096])
    ap.add_argument("--ref-max-n", type=int, default=1024)
    ap.add_argument("--delta-n", type=int, default=0, help="override delta_N for every N")
    args = ap.parse_args()
    from paper_2406_14116_b200 import BinSpec
    from paper_2406_14116_b200.design import DesignOptions, solve_minimax
    from oracle import oracle as O

    for n in args.n:
        l, dn = n // 4 + 1, args.delta_n or DELTA_N[n]
        b = n // 8
        bins = BinSpec(n, l, n - l + 1, dn, b, b)
        opt = DesignOptions(grid_points=2 * n)
        t = time.perf_counter()
        out = solve_minimax(bins, opt)
        gpu_s = time.perf_counter() - t
        line = {"metric": "solve_minimax_seconds", "unit": "s", "higher_is_better": False,
                "config": {"N": n, "L": l, "M": n - l + 1, "delta_N": dn, "b": b, "grid_points": 2 * n},
                "gpu_seconds": gpu_s, "gpu_phases": out.seconds, "delta": out.delta, "rounds": out.rounds,
                "active_triples": out.active_triples, "lp_rows": out.lp_rows, "lp_iterations": out.lp_iterations,
                "V": out.profile.values}
        if n <= args.ref_max_n and O.have_reference():
            t = time.perf_counter()
            r = O.reference().solve_minimax(n, l, dn, b, b, 2 * n)
            line["ref_seconds"] = time.perf_counter() - t
            line["ref_threads"] = 1  # parallel_for over b: one band centre -> one thread
            line["speedup"] = line["ref_seconds"] / gpu_s
            line["V_max_abs_diff"] = float(np.abs(np.array(out.profile.values) - r["v"]).max())
            line["delta_ref"] = r["delta"]
            line["rounds_ref"] = r["rounds"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
