#!/usr/bin/env python
"""A/B sweep of experiment builds on the GPU box: for each round, for each variant (a directory
under vlib/ holding libfcvbw_gpu.so, or "head" for the in-tree build), run bench.py on each config
and print one compact line (value, roofline frac, kernel ms, clocks). Variants are interleaved per
round so that clock / power-cap drift hits them evenly.

  python tools/sweep.py --variants head,twreg --configs c3,c2 --rounds 2 [--steps 10]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", required=True)
    ap.add_argument("--configs", default="c3")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--extra", default="")
    args = ap.parse_args()
    for rnd in range(args.rounds):
        for cfg in args.configs.split(","):
            for v in args.variants.split(","):
                env = dict(os.environ)
                if v != "head":
                    env["FCVBW_GPU_LIB"] = os.path.join(ROOT, "vlib", v, "libfcvbw_gpu.so")
                cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", str(args.steps),
                       "--warmup", "3", "--no-cpu-baseline", "--no-per-config", "--no-e2e"] + args.extra.split()
                r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
                line = next((l for l in r.stdout.splitlines() if l.startswith("{")), None)
                if line is None:
                    print(f"r{rnd} {cfg:14s} {v:12s} FAILED rc={r.returncode} {r.stderr[-400:]}", flush=True)
                    continue
                d = json.loads(line)
                rf = d["roofline"]
                ck = d.get("clocks", {})
                print(f"r{rnd} {cfg:14s} {v:12s} {d['value'] / 1e9:8.2f} G/s  frac {rf['frac']:.4f}  "
                      f"kernel {rf['kernel_ms_avg']:.4f} ms  eager {d.get('eager_ms_per_step') or 0:.4f}  "
                      f"sm {ck.get('sm_mhz')} {ck.get('power_w')}W {','.join(ck.get('reasons', []))}", flush=True)


if __name__ == "__main__":
    main()
