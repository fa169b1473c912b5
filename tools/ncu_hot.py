#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot.py gpurun_out/full.ncu-rep sb_bwd_kv [N]
"""
import csv
import io
import subprocess
import sys


def main(path, kname, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kname}", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[i0]
    col = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[i0 + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[col["# Samples"]] or 0) for r in data)
    print(f"{len(data)} SASS instructions, {tot} samples")
    idx = sorted(range(len(data)), key=lambda i: -int(data[i][col["# Samples"]] or 0))[:n]
    for i in sorted(idx):
        r = data[i]
        s = int(r[col["# Samples"]] or 0)
        st = sorted(((int(r[col[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{i:5d} {100.0 * s / tot:5.1f}% {r[col['Source']].strip()[:60]:60s} "
              + " ".join(f"{c}={v}" for v, c in st if v))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)


def by_reason(path, kname):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kname}", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[i0]
    col = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[i0 + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {c: 0 for c in stall_cols}
    ops = {}
    for r in data:
        op = r[col["Source"]].split()[0] if not r[col["Source"]].strip().startswith("@") else r[col["Source"]].split()[1]
        op = op.split(".")[0]
        for c in stall_cols:
            v = int(r[col[c]] or 0)
            agg[c] += v
            ops[op] = ops.get(op, 0) + v
    tot = sum(agg.values())
    print({c[6:]: round(100 * v / tot, 1) for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v})
    print({o: round(100 * v / tot, 1) for o, v in sorted(ops.items(), key=lambda x: -x[1])[:25]})
