#!/usr/bin/env python3
"""Parity / bench harness writing the reference CLI's artifacts.

A checker (it runs the oracle for `equiv`), so it lives under tests/ with the other
test infrastructure.

`equiv` and `bench` produce `equiv.csv`, `bench.csv` and `manifest.json` with the column
schemas of the reference's `sb equiv` / `sb bench` (cli.py:343-344, :453-455, :128-152), so
results line up with the reference's tooling, but measure this package's CUDA path:

  equiv.csv  L, d_block, skip, diff_o, fused_dq, fused_dk, fused_dv, two_dq, two_dk, two_dv,
             two_vs_fused, result
      Inputs N(0,1), rounded to bf16; reference = the dense f64 oracle on the same rounded
      inputs (attention.py:106-145 restated).  This package has no fused backward; its two
      backward modes fill the two column groups: "fused_*" = store mode (phase 2 reads
      phase 1's dZ tiles), "two_*" = recompute mode; two_vs_fused = max |store - recompute|
      (0: bit-identical).  Diffs are max_rel_err (numerics.py:116-127); pass = every diff
      < 2e-2 (the bf16 bound of BASELINE.json) and two_vs_fused == 0.
  bench.csv  L, d_block, variant, skip, median_ms, tiles_visited, tiles_skipped
      fwd+bwd median of CUDA-event times over `repeats` (>= 5) after `warmups`, input kinds
      random / saturating / dead (cli.py:387-405 restated).

Only d_block = 64 exists on the GPU path (blocked.py:41 DEFAULT_BLOCK); head_dim 64 or 128.

    python tests/reports/reference_harness.py equiv [--lengths 1,7,64,100,256,512] [--d 64] [--out DIR]
    python tests/reports/reference_harness.py bench [--lengths 256,1024,4096] [--d 64] [--input random] [--out DIR]
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import os
import platform
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
import paper_2410_17980_b200 as sb  # noqa: E402

TOL = 2e-2


def _fmt(x: float) -> str:
    return f"{x:.3e}"


def _write_csv(out, name, header, rows):
    with open(os.path.join(out, name), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)
    return name


def _write_manifest(out, command, seed, options, artifacts):
    manifest = {
        "command": command, "seed": seed, "out": out, "threads": 1, "precision": "bf16",
        "config": options,
        "versions": {"paper_2410_17980_b200": sb.__version__ if hasattr(sb, "__version__")
                     else "dev", "python": platform.python_version(), "numpy": np.__version__,
                     "torch": torch.__version__, "cuda": torch.version.cuda,
                     "device": torch.cuda.get_device_name(0)},
        "artifacts": sorted(artifacts),
    }
    with open(os.path.join(out, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
        fh.write("\n")


def _gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(
        "cuda", torch.bfloat16)[None, None]


def _rounded(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def _inputs(kind, L, d, rng):
    v = rng.standard_normal((L, d))
    if kind == "saturating":  # logit 40 on the key one step behind every query
        q = np.zeros((L, d))
        k = np.zeros((L, d))
        q[np.arange(L), np.arange(L) % d] = 40.0 * math.sqrt(d)
        k[np.arange(L), (np.arange(L) + 1) % d] = 1.0
        return q, k, v
    if kind == "dead":  # logit -100 everywhere: nothing is consumed, nothing skips
        q = np.zeros((L, d))
        k = np.zeros((L, d))
        q[:, 0] = 100.0 * math.sqrt(d)
        k[:, 0] = -1.0
        return q, k, v
    return rng.standard_normal((L, d)), rng.standard_normal((L, d)), v


def _run(q, k, v, w, skip, store):
    o, _, st, cache = sb.blocked_forward(q, k, v, skip=skip)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, w, store_tiles=store)
    return o, dq, dk, dv, st


def cmd_equiv(a):
    lengths = [int(x) for x in a.lengths.split(",")] if a.lengths else [1, 7, 64, 100, 256, 512]
    header = ["L", "d_block", "skip", "diff_o", "fused_dq", "fused_dk", "fused_dv",
              "two_dq", "two_dk", "two_dv", "two_vs_fused", "result"]
    table, worst = [], 0.0
    for L in lengths:
        rng = np.random.default_rng([a.seed, L])
        q64, k64, v64, w64 = (_rounded(rng.standard_normal((L, a.d))) for _ in range(4))
        o_ref, _, _ = oracle.dense_forward(q64, k64, v64)
        g_ref = oracle.dense_backward(q64, k64, v64, w64)
        q, k, v, w = (_gpu(x) for x in (q64, k64, v64, w64))
        for skip in (False, True):
            st_ = _run(q, k, v, w, skip, True)
            rc = _run(q, k, v, w, skip, False)
            torch.cuda.synchronize()
            f64 = lambda t: t[0, 0].double().cpu().numpy()  # noqa: E731
            diffs = [oracle.max_rel_err(f64(st_[0]), o_ref)]
            diffs += [oracle.max_rel_err(f64(st_[1 + i]), g_ref[i]) for i in range(3)]
            diffs += [oracle.max_rel_err(f64(rc[1 + i]), g_ref[i]) for i in range(3)]
            pair = max(float((st_[1 + i].float() - rc[1 + i].float()).abs().max()) for i in range(3))
            ok = max(diffs) < TOL and pair == 0.0
            worst = max(worst, max(diffs))
            table.append([L, 64, "on" if skip else "off", *[_fmt(x) for x in diffs], _fmt(pair),
                          "pass" if ok else "fail"])
    arts = [_write_csv(a.out, "equiv.csv", header, table)]
    _write_manifest(a.out, "equiv", a.seed, {"lengths": lengths, "d_blocks": [64], "d": a.d}, arts)
    fails = sum(r[-1] == "fail" for r in table)
    print(f"equiv: {len(table) - fails}/{len(table)} configurations pass (worst diff {worst:.3e})")
    return 0 if fails == 0 else 1


def cmd_bench(a):
    lengths = [int(x) for x in a.lengths.split(",")] if a.lengths else [256, 1024, 4096]
    repeats = max(5, a.repeats)
    table = []
    for L in lengths:
        rng = np.random.default_rng([a.seed, L])
        q, k, v = (_gpu(_rounded(x)) for x in _inputs(a.input, L, a.d, rng))
        w = _gpu(_rounded(rng.standard_normal((L, a.d))))
        for skip in (False, True):
            for _ in range(a.warmups):
                st = _run(q, k, v, w, skip, None)[4]
            times = []
            for _ in range(repeats):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                st = _run(q, k, v, w, skip, None)[4]
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            table.append([L, 64, "sb", "on" if skip else "off", f"{statistics.median(times):.3f}",
                          st.visited, st.skipped])
    arts = [_write_csv(a.out, "bench.csv", ["L", "d_block", "variant", "skip", "median_ms",
                                            "tiles_visited", "tiles_skipped"], table)]
    _write_manifest(a.out, "bench", a.seed, {"lengths": lengths, "d_block": 64, "d": a.d,
                                             "repeats": repeats, "warmups": a.warmups,
                                             "input": a.input}, arts)
    for r in table:
        print(*r)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("command", choices=["equiv", "bench"])
    ap.add_argument("--lengths", default="")
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--input", default="random", choices=["random", "saturating", "dead"])
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--warmups", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "harness"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    sys.exit(cmd_equiv(a) if a.command == "equiv" else cmd_bench(a))


if __name__ == "__main__":
    main()
