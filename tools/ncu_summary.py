"""Summarise one `ncu --set full` capture of ols_fused into the profiles/ text format.

usage: python tools/ncu_summary.py <report.ncu-rep> "<header line>" > profiles/<name>.txt
Reads the raw page (metrics, stall reasons) and the source page (dynamic SASS mix per warp-block).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__time_duration.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__block_size", "launch__grid_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout


def main():
    rep, header = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print(header)
    print("---- kernel:", d.get("Kernel Name", ""))
    for k in KEYS:
        if k in d:
            print(f"  {k:70s} {u.get(k, ''):16s} {d[k]}")
    st = []
    for k, val in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((float(val), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("  stalls: " + ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:10]))
    # dynamic SASS mix from the source page (instructions executed per opcode)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    src = [r for r in csv.reader(io.StringIO(src))]
    src = src[1:] if src and src[0] and src[0][0] == "Kernel Name" else src
    if src:
        hh = src[0]
        try:
            i_src = hh.index("Source")
            i_ex = hh.index("Instructions Executed")
        except ValueError:
            return
        mix = {}
        for r in src[1:]:
            if len(r) <= max(i_src, i_ex):
                continue
            op = r[i_src].strip().split(" ")
            op = [t for t in op if t and not t.startswith("@")]
            if not op:
                continue
            name = op[0].split(".")[0]
            try:
                mix[name] = mix.get(name, 0) + float(r[i_ex] or 0)
            except ValueError:
                pass
        blocks = float(sys.argv[3]) if len(sys.argv) > 3 else None
        total = sum(mix.values())
        print("\n# dynamic SASS mix (warp instructions executed" + (", per warp-block" if blocks else "") + ")")
        if blocks:
            print(f"total per warp-block: {total / blocks:.0f}")
        for name, n in sorted(mix.items(), key=lambda x: -x[1])[:20]:
            print(f"  {name:12s} {n / blocks if blocks else n:12.1f}")


if __name__ == "__main__":
    main()
