#!/usr/bin/env python
"""Aggregate ncu source-page (SASS) samples by opcode: total stall samples and one stall column.

  python tools/ncu_ops.py REPORT [stall_column]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_wait"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
I = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in body:
    src = r[I["Source"]].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    op = op.split(".")[0]
    a = agg[op]
    a[0] += num(r[I["Warp Stall Sampling (All Samples)"]])
    a[1] += num(r[I[col]])
    a[2] += num(r[I["Instructions Executed"]])
tot = sum(a[0] for a in agg.values())
print(f"{'op':10s} {'all%':>6s} {col + '%':>12s} {'inst':>14s}")
for op, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{op:10s} {100 * a[0] / tot:6.1f} {100 * a[1] / tot:12.1f} {a[2]:14.0f}")
