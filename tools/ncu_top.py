#!/usr/bin/env python
"""Top stall sites of a tools/ncu_trim.py dump.  python tools/ncu_top.py FILE.tsv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1]), delimiter="\t"))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
h = rows[0]
idx = {x: i for i, x in enumerate(h)}


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


body = rows[1:]
A = "Warp Stall Sampling (All Samples)"
tot = sum(f(r[idx[A]]) for r in body)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print("total samples", int(tot), " ".join(f"{c[6:]}:{100 * sum(f(r[idx[c]]) for r in body) / tot:.0f}%" for c in cols
                                            if sum(f(r[idx[c]]) for r in body) / tot > 0.02))
for i in sorted(range(len(body)), key=lambda i: -f(body[i][idx[A]]))[:n]:
    r = body[i]
    rs = sorted(((f(r[idx[c]]), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{i:5d} {100 * f(r[idx[A]]) / tot:4.1f}%  {r[idx['Source']][:64]:64s} {rs[0][1]}:{rs[0][0]:.0f} {rs[1][1]}:{rs[1][0]:.0f}")
