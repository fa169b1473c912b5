#!/usr/bin/env python3
"""Summarise an ncu --set full report of the sb_* kernels as a markdown table.

    python tools/ncu_summary.py gpurun_out/full.ncu-rep > profiles/rN_summary_table.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("us", "gpu__time_duration.sum", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("XU(MUFU) %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    ("FMA %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("ALU %", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("smem pipe %", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("DRAM rd GB", "dram__bytes_read.sum", 1.0),
    ("DRAM wr GB", "dram__bytes_write.sum", 1.0),
]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "barrier", "branch_resolving",
          "math_pipe_throttle", "mio_throttle", "dispatch_stall", "sleeping", "no_instruction",
          "selected", "not_selected"]


def main(path):
    names = [m[1] for m in METRICS] + [
        f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(names)], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, n):
        v = r[col[n]].replace(",", "")
        u = units[col[n]]
        try:
            f = float(v)
        except ValueError:
            return v
        if u == "Mbyte":
            f /= 1e3
        if u == "Kbyte":
            f /= 1e6
        if u == "usecond":
            f /= 1e3
        if u == "nsecond":
            f /= 1e6
        return f"{f:.3g}"

    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in data:
        k = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        print(f"| {k} | " + " | ".join(val(r, m[1]) for m in METRICS) + " |")
    print()
    print("Warp stall reasons (warps stalled per issued instruction):")
    print()
    print("| kernel | " + " | ".join(STALLS) + " |")
    print("|---" * (len(STALLS) + 1) + "|")
    for r in data:
        k = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        print(f"| {k} | " + " | ".join(
            val(r, f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            for s in STALLS) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
