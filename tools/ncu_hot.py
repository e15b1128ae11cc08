#!/usr/bin/env python
"""Top SASS lines of an ncu capture by one stall reason (source page, SASS view).

  python tools/ncu_hot.py REPORT [stall_column] [n]     e.g. stall_long_sb 15
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


tot = sum(num(r[idx[col]]) for r in body)
allst = sum(num(r[idx["Warp Stall Sampling (All Samples)"]]) for r in body)
print(f"{col}: {tot:.0f} samples of {allst:.0f} ({100 * tot / max(allst, 1):.1f} %)")
for r in sorted(body, key=lambda r: -num(r[idx[col]]))[:n]:
    print(f"{num(r[idx[col]]):8.0f}  {r[idx['Address']]:>6}  {r[idx['Source']][:110]}")
