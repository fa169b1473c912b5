#!/usr/bin/env python3
"""SASS evidence for the kernels of libsbattn.so (BASELINE.json north_star: "SASS listings").

For every sb_* kernel of the built library (cuobjdump -sass, sm_100a) writes
profiles/<tag>_sass/<kernel>.txt with
  - the instruction-class histogram (tcgen05 MMAs UTCHMMA / UTCBAR commits, TMA UTMALDG /
    UTMASTG / UTMAPF, TMEM loads/stores LDTM / STTM, MUFU ex2 / rcp / lg2, FFMA / FMUL, ...);
  - the MMA-issue excerpt (the first run of UTCHMMA instructions with its context);
  - the stick-math excerpt (the densest window of MUFU.EX2).
and a summary table profiles/<tag>_sass/README.md.

    python tools/sass_report.py [--lib paper_2410_17980_b200/libsbattn.so] [--tag r1_v8]
"""

from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UTMACMDFLUSH", "LDTM", "STTM",
           "MUFU.EX2", "MUFU.RCP", "MUFU.LG2", "FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "F2FP", "STS", "LDS", "STG",
           "LDG", "SYNCS", "BAR", "SHFL"]


def functions(sass: str):
    cur, lines = None, []
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            if cur:
                yield cur, lines
            cur, lines = m.group(1), []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", ln)
        if cur and m:
            lines.append(m.group(1).strip())
    if cur:
        yield cur, lines


def opcode(ins: str) -> str:
    t = ins.split()
    if not t:
        return ""
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    return op


def classify(op: str) -> str | None:
    for c in CLASSES:
        if op == c or op.startswith(c + "."):
            return c
    return None


def demangle(name: str) -> str:
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2410_17980_b200", "libsbattn.so"))
    ap.add_argument("--tag", default="r1_v8")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True,
                          check=True).stdout
    out_dir = os.path.join(ROOT, "profiles", f"{a.tag}_sass")
    os.makedirs(out_dir, exist_ok=True)
    rows = []
    for name, ins in functions(sass):
        if "sb_" not in name:
            continue
        pretty = demangle(name)
        base = pretty.split("(")[0].replace("sb::", "").replace("void ", "")
        short = re.sub(r"[^A-Za-z0-9_<>,]", "", base)
        fname = re.sub(r"[<>, ]", "_", short).strip("_") + ".txt"
        hist = collections.Counter()
        for i in ins:
            c = classify(opcode(i))
            if c:
                hist[c] += 1
        mma = [k for k, i in enumerate(ins) if opcode(i).startswith("UTCHMMA")]
        ex2 = [k for k, i in enumerate(ins) if opcode(i).startswith("MUFU.EX2")]
        with open(os.path.join(out_dir, fname), "w") as f:
            f.write(f"{pretty}\n{len(ins)} instructions\n\n")
            for c in CLASSES:
                if hist[c]:
                    f.write(f"{c:14s} {hist[c]}\n")
            if mma:
                lo = max(0, mma[0] - 12)
                hi = min(len(ins), mma[min(len(mma) - 1, 7)] + 8)
                f.write(f"\n--- MMA issue (instructions {lo}..{hi}) ---\n")
                f.write("\n".join(ins[lo:hi]) + "\n")
            if ex2:
                # the 160-instruction window holding the most ex2
                best = max(range(len(ex2)), key=lambda j: sum(1 for e in ex2 if ex2[j] <= e < ex2[j] + 160))
                lo = ex2[best]
                f.write(f"\n--- stick math (instructions {lo}..{lo + 160}) ---\n")
                f.write("\n".join(ins[lo:lo + 160]) + "\n")
        rows.append((short, len(ins), hist))
    with open(os.path.join(out_dir, "README.md"), "w") as f:
        f.write(f"# SASS of libsbattn.so (sm_100a), `tools/sass_report.py --tag {a.tag}`\n\n")
        cols = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "MUFU.EX2",
                "MUFU.RCP", "MUFU.LG2", "FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL"]
        f.write("| kernel | instrs | " + " | ".join(cols) + " |\n")
        f.write("|---|---|" + "---|" * len(cols) + "\n")
        for short, n, h in rows:
            f.write(f"| {short} | {n} | " + " | ".join(str(h[c]) for c in cols) + " |\n")
        f.write("\nUTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, UTMALDG/UTMASTG/UTMAPF = TMA "
                "load/store/prefetch, LDTM/STTM = tcgen05.ld/st (TMEM), FFMA2/FMUL2/FADD2 = packed "
                "f32x2 arithmetic (two lanes per FMA-pipe instruction).  Per-kernel files hold "
                "the MMA-issue and stick-math excerpts.\n")
    print(open(os.path.join(out_dir, "README.md")).read())


if __name__ == "__main__":
    main()
