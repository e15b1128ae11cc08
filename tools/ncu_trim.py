#!/usr/bin/env python
"""Trim the SASS source page of an ncu capture to the columns worth keeping under profiles/:
address, instruction, executed count, stall samples (all / per reason) and shared-memory
wavefronts, one line per SASS instruction.   python tools/ncu_trim.py REPORT > out.tsv"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
keep = [i for i, h in enumerate(hdr)
        if h in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                 "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal") or h.startswith("stall_")]
print("\t".join(hdr[i] for i in keep))
for r in rows[2:]:
    if len(r) == len(hdr):
        print("\t".join(r[i][-12:] if hdr[i] == "Address" else r[i][:90] for i in keep))
