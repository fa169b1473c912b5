#!/usr/bin/env python3
"""Stall samples of every mbarrier wait (TRYWAIT + retry branch) in one kernel of an
ncu report, labelled by the barrier's shared-memory offset.

    python tools/ncu_waits.py gpurun_out/full.ncu-rep sb_bwd_kvs [bar_base_hex] [name=off ...]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    path, kname = sys.argv[1], sys.argv[2]
    names = {}
    for a in sys.argv[3:]:
        k, v = a.split("=")
        names[int(v, 16)] = k
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kname}", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    data = [r for r in rows[i0 + 1:] if r and r[0].startswith("0x")]
    tot = sum(int(r[2] or 0) for r in data)
    print(f"{tot} samples")
    for i, r in enumerate(data):
        m = re.search(r"TRYWAIT P\d, \[[^\]]*\+(0x[0-9a-f]+)\]", r[1])
        if m and i + 1 < len(data):
            off = int(m.group(1), 16)
            n = int(data[i + 1][2] or 0)
            if n:
                print(f"{i:5d} {names.get(off, hex(off)):12s} {n:6d} {100 * n / tot:5.1f}%")


if __name__ == "__main__":
    main()
