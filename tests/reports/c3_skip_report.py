#!/usr/bin/env python3
"""C3 long-context block-skipping report (BASELINE.json configs[2]).

A checker: it lives under tests/ because it runs the oracle to verify the GPU skip
decisions (the oracle is test infrastructure only).

B=1, H=32, L=32768, d=128 bf16, skip on (skip_eps = 1e-6, the reference's f32
default for non-f64 inputs).  For each input family (random, logit shift mu=-6
and mu=-8, saturating, dead) it reports:
  - tiles visited / total and the skipped fraction (TileStats, blocked.py:82-103);
  - forward (skip on) and forward+backward CUDA-event times, and the skip-off
    forward time on the same inputs;
  - bit-exactness of first_kb on `--check-heads` heads against the C oracle run
    in float64 on the same bf16-rounded inputs (families where the oracle is cheap).
Prints one JSON object; `--out` also writes it to a file.

    python tests/reports/c3_skip_report.py [--L 32768] [--H 32] [--check-heads 1] [--out f.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
import paper_2410_17980_b200 as sb  # noqa: E402
from tests.gpu_util import make_qkv, to64  # noqa: E402


def timed(fn, n=5, warm=3):
    # several warm-up calls: the first launches of a kernel on new inputs run slow
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def margins(ref, L, eps, block=64):
    """How close the oracle's skip decisions are to the threshold.

    For every query block: the last visited tile passed the check with max_r a = max_r
    M(qb, first_kb) >= log eps (margin a - log eps); a skipped tile (first_kb > 0) failed it
    with max_r a = max_r log_rem < log eps (margin log eps - a).  Returns the minimum of each
    and a histogram of all margins in decades (nats)."""
    le = float(np.log(np.float32(eps)))
    fkb, M, lr = ref["first_kb"], ref["M"], ref["log_rem"]
    vis, skp = [], []
    for u in range(fkb.shape[0]):
        for qb in range(fkb.shape[1]):
            rows = min(block, L - qb * block)
            kb = int(fkb[u, qb])
            vis.append(float(M[u, qb * (qb + 1) // 2 + kb, :rows].max()) - le)
            if kb > 0:
                skp.append(le - float(lr[u, qb * block: qb * block + rows].max()))
    allm = np.array(vis + skp)
    edges = [0, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1, 1, np.inf]
    hist = np.histogram(allm, bins=edges)[0].tolist()
    return {"log_eps": le, "min_visit_margin": min(vis), "min_skip_margin": min(skp) if skp else None,
            "hist_edges_nats": ["0", "1e-6", "1e-5", "1e-4", "1e-3", "1e-2", "0.1", "1", "inf"],
            "hist": hist, "n_decisions": int(allm.size)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=1)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--check-heads", type=int, default=1)
    ap.add_argument("--families", default="random,shift-6,shift-8,saturating,dead")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    eps = 1e-6
    res = {"workload": f"C3: B={a.B} H={a.H} L={a.L} d={a.D} bf16, skip on, skip_eps={eps}",
           "families": {}}
    for fam in a.families.split(","):
        mu = -6.0
        name = fam
        if fam.startswith("shift"):
            mu = float(fam[len("shift"):])
            fam = "shift"
        q, k, v, d_o = make_qkv(a.B, a.H, a.L, a.D, seed=11, family=fam, mu=mu)
        o, log_rem, st, cache = sb.blocked_forward(q, k, v, skip=True, skip_eps=eps)
        torch.cuda.synchronize()
        t_fwd = timed(lambda: sb.blocked_forward(q, k, v, skip=True, skip_eps=eps, counters=False))
        t_fwd_off = timed(lambda: sb.blocked_forward(q, k, v, skip=False, counters=False))
        t_fb = timed(lambda: sb.blocked_backward_twophase(
            sb.blocked_forward(q, k, v, skip=True, skip_eps=eps, counters=False)[3], d_o))
        entry = {"visited": st.visited, "total": st.total,
                 "skipped_fraction": st.skipped / st.total,
                 "fwd_ms_skip_on": t_fwd, "fwd_ms_skip_off": t_fwd_off,
                 "fwd_bwd_ms_skip_on": t_fb}
        # oracle decisions (f64, same bf16 inputs) on the first heads; skip the
        # families whose oracle run is an unskipped L^2 sweep at this length
        if a.check_heads > 0 and (name in ("random", "shift-6", "saturating") or a.L <= 8192):
            nh = min(a.check_heads, a.H)
            t0 = time.perf_counter()
            ref = oracle.tiled_forward(to64(q[0, :nh]), to64(k[0, :nh]), to64(v[0, :nh]),
                                       block=64, skip=True, skip_eps=eps, dtype=np.float64)
            got = st.first_kb[0, :nh].cpu().numpy()
            entry["first_kb_bit_exact"] = bool(np.array_equal(got, ref["first_kb"]))
            entry["decision_margins"] = margins(ref, a.L, eps)
            entry["oracle_heads_checked"] = nh
            entry["oracle_s"] = time.perf_counter() - t0
        elif name == "dead":
            entry["first_kb_bit_exact"] = bool((st.first_kb == 0).all().item())
            entry["oracle_heads_checked"] = "all (dead family: nothing may be skipped)"
        res["families"][name] = entry
        print(name, json.dumps(entry), file=sys.stderr, flush=True)
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
