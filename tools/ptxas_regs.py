#!/usr/bin/env python
"""Summarise `nvcc -Xptxas -v` output: registers / spills / stack per ols_fused instantiation.

  python tools/ptxas_regs.py LOG [substring]     (substring filters the mangled template args)
"""
import re
import subprocess
import sys


def parse(text):
    out, cur = [], None
    for line in text.splitlines():
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = {"name": m.group(1)}
            out.append(cur)
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            cur.update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            cur["regs"] = int(m.group(1))
    return out


def pretty(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


if __name__ == "__main__":
    text = open(sys.argv[1]).read()
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    for f in parse(text):
        if pat in f["name"]:
            n = pretty(f["name"]).replace("fcvbw_gpu::", "").split("(")[0]
            print(f"{f.get('regs', '?'):>4} regs  spill {f.get('spill_st', 0)}/{f.get('spill_ld', 0)}  "
                  f"stack {f.get('stack', 0):>4}  {n}")
