#!/usr/bin/env python
"""Per-call latency of the streaming entry points (the reference's block-by-block `cmd_run` loop,
fcvbw_cli.cpp:95-113): process_block / feed on one engine, real fp64 samples (the reference's
signature), against the reference engine compiled from its headers on the same host.

  python tools/bench_stream.py [--n 1024] [--calls 2000]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--calls", type=int, default=2000)
    args = ap.parse_args()
    from paper_2406_14116_b200 import BinSpec, OlsEngine, TransitionProfile
    n = args.n
    m = 3 * n // 4
    dn = 12
    bins = BinSpec(n, n - m + 1, m, dn, dn // 2, n // 2 - dn // 2 - 1)
    v = np.linspace(0.9, 0.1, dn - 1)
    eng = OlsEngine(bins, TransitionProfile(list(v)), n // 8, dtype="c128")
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, size=m * args.calls)
    for i in range(20):
        eng.process_block(x[i * m:(i + 1) * m])
    t0 = time.perf_counter()
    for i in range(args.calls):
        eng.process_block(x[i * m:(i + 1) * m])
    t1 = time.perf_counter()
    eng.reset()
    t2 = time.perf_counter()
    for i in range(args.calls):
        eng.feed(x[i * m:(i + 1) * m])
    t3 = time.perf_counter()
    print(f"N={n} M={m}: process_block {1e6 * (t1 - t0) / args.calls:.1f} us/call, "
          f"feed {1e6 * (t3 - t2) / args.calls:.1f} us/call "
          f"({m * args.calls / (t1 - t0) / 1e6:.2f} M real samples/s through process_block)")


if __name__ == "__main__":
    main()
