#!/usr/bin/env python3
"""Warp-stall samples of one kernel per source line, from an ncu report (tuning aid, no GPU).

    python tools/ncu_lines.py gpurun_out/full.ncu-rep kvs [--top 30]

Runs `ncu -i REP -k regex:KERNEL --page source --csv --print-source cuda,sass` and sums the
"Warp Stall Sampling (All Samples)" column of every SASS instruction into the CUDA source
line it belongs to; prints the top lines with their three largest stall reasons.
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "-k", "regex:" + a.kernel, "--page", "source", "--csv",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg, reasons, fname, cur = {}, {}, None, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) <= i_s or r[0] == "Line No":
            continue
        if r[0]:
            cur = (fname, r[0], r[1].strip()[:70])
            continue
        if not r[i_s].isdigit():
            continue
        agg[cur] = agg.get(cur, 0) + int(r[i_s])
        d = reasons.setdefault(cur, {})
        for i in stall:
            if r[i].isdigit():
                d[hdr[i]] = d.get(hdr[i], 0) + int(r[i])
    tot = sum(agg.values()) or 1
    print(f"{a.kernel}: {tot} samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:a.top]:
        top3 = sorted(reasons[k].items(), key=lambda x: -x[1])[:3]
        why = " ".join(f"{n[6:]}={c}" for n, c in top3)
        print(f"{v:7d} {100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5} {k[2]:<70} {why}")


if __name__ == "__main__":
    main()
