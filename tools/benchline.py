#!/usr/bin/env python
"""Print a bench.py JSON line compactly: headline + per_config table.  python tools/benchline.py LOG"""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    pc = d.pop("per_config", None)
    rf = d.get("roofline") or {}
    ck = d.get("clocks") or {}
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    print(f"{d.get('config', {}).get('workload')} value {d['value'] / 1e9:.2f} G/s frac {rf.get('frac', 0):.4f} "
          f"kernel {rf.get('kernel_ms_avg', 0):.4f} ms clocks {ck.get('sm_mhz')} {ck.get('power_w')}W "
          f"{ck.get('reasons')} e2e {e2e.get('value', 0) / 1e9:.2f} G/s cpu {cpu.get('value', 0) / 1e6:.1f} M/s "
          f"launches {d.get('gpu_launches')}")
    for k, v in (pc or {}).items():
        print(f"  {k:14s} {v['value'] / 1e9:8.2f} G/s  frac {v['frac']:.3f}  kernel {v['kernel_ms_avg']:.4f} ms  "
              f"sm {v['clocks'].get('sm_mhz')}")
