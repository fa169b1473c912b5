#!/usr/bin/env python3
"""Per-event SM-clock timeline of the backward kernels (tuning aid, GPU only).

Builds/loads libsbattn_trace.so (-DSB_TRACE), runs the C2 workload once, and
prints, for the first traced CTAs, the per-tile durations between events of the
stick warpgroups (roles 0/1) and the MMA issuers (roles 2/3).  Writes the raw
stamps to gpurun_out/trace_<phase>.npy.

    python tools/trace_kernels.py [--phase 2] [--L 4096]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_17980_b200 import _lib, build, ops  # noqa: E402

NCTA, NROLE, NT, NEV = 4, 4, 64, 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--phase", type=int, default=2)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--H", type=int, default=16)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--lib", default="", help="prebuilt trace library (e.g. libsbattn_trace_nomath.so)")
    a = ap.parse_args()
    path = a.lib or build.build(trace=True)
    lib = _lib.load(path)
    _lib._lib = lib  # route the ops through the trace build
    lib.sb_debug_set_trace.argtypes = [ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn(a.B, a.H, a.L, a.D, device=dev, generator=g, dtype=torch.bfloat16)
                   for _ in range(4))
    tr = torch.zeros(NCTA * NROLE * NT * NEV, dtype=torch.int32, device=dev)
    o, cache = ops.sb_forward_blocked(q, k, v)
    for it in range(3):  # warm, then traced
        if it == 2:
            lib.sb_debug_set_trace(tr.data_ptr())
        if a.phase == 0:  # forward
            ops.sb_forward_blocked(q, k, v)
        elif a.phase == 2:
            ops.blocked_backward_twophase(cache, do)
        else:  # phase 1 only, traced
            ws = torch.empty(ops.workspace_bytes(cache), device=dev, dtype=torch.uint8)
            ops.blocked_backward_twophase(cache, do, phases=1, workspace=ws)
        torch.cuda.synchronize()
    lib.sb_debug_set_trace(None)
    t = tr.cpu().numpy().view(np.uint32).reshape(NCTA, NROLE, NT, NEV).astype(np.int64)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"trace_p{a.phase}.npy"), t)
    for c in range(NCTA):
        base = t[c, 0, 0, 14] if t[c, 0, 0, 14] else t[c, 1, 0, 14]
        print(f"CTA {c}: start->done {t[c, 0, 0, 15] - base} clk")
        for role in range(NROLE):
            rows = []
            for j in range(NT):
                ev = t[c, role, j]
                if not ev.any():
                    continue
                rows.append((j, [int(x - base) if x else -1 for x in ev]))
            print(f"  role {role}: {len(rows)} tiles")
            for j, ev in rows[:6] + rows[-2:]:
                print(f"    j={j:2d} " + " ".join(f"{e:7d}" for e in ev[:14]))
    if a.phase == 2:
        # store-mode phase 2 (sb_bwd_kvs_kernel): stick warpgroups 0 start, 1 S landed,
        # 2 A computed, 3 aused (dV(j-1) read A), 4 A stored; MMA issuer (role 2) 7 dZ
        # landed, 0/1 Q(j+1) wait, 2 S buffer free, 4 A full, 5 dO landed
        for role, order in ((0, [0, 1, 2, 3, 4]), (1, [0, 1, 2, 3, 4]), (2, [7, 0, 1, 2, 4, 5])):
            d = {f"{x}->{y}": [] for x, y in zip(order, order[1:])}
            per_tile = []
            for c in range(NCTA):
                for j in range(1, NT - 1):
                    ev, nx = t[c, role, j], t[c, role, j + 1]
                    if not all(ev[e] for e in order):
                        continue
                    for x, y in zip(order, order[1:]):
                        d[f"{x}->{y}"].append(int(ev[y] - ev[x]))
                    if nx[order[0]]:
                        per_tile.append(int(nx[order[0]] - ev[order[0]]))
            print(f"role {role} median clk:", {k: int(np.median(v)) for k, v in d.items() if v},
                  "tile:", int(np.median(per_tile)) if per_tile else None)
    if a.phase == 1:
        # median clocks between the stick warpgroups' per-tile events (tiles j >= 1 of
        # every traced CTA/role): 0 start, 1 S loaded, 7 turn taken, 8 pass 1 done,
        # 2 recompute done, 3 dW read, 4 dZ math done, 5 zempty, 6 dZ stored
        order = [0, 1, 7, 8, 2, 3, 4, 5, 6]
        d = {f"{x}->{y}": [] for x, y in zip(order, order[1:])}
        per_tile = []
        for c in range(NCTA):
            for role in (0, 1):
                for j in range(1, NT):
                    ev = t[c, role, j]
                    if not all(ev[e] for e in order):
                        continue
                    for x, y in zip(order, order[1:]):
                        d[f"{x}->{y}"].append(int(ev[y] - ev[x]))
                    nxt = t[c, role, j + 1, 0] if j + 1 < NT else 0
                    if nxt:
                        per_tile.append(int(nxt - ev[0]))
        print("median clk:", {k: int(np.median(v)) for k, v in d.items() if v},
              "tile:", int(np.median(per_tile)) if per_tile else None)
        # MMA round trips per warpgroup tile (issuer role 2 + w, stick role w): S issued
        # -> S loaded, dW(j-1) read -> S(j) issued, dW issued -> dW read, dZ stored -> dQ issued
        x = {"S issue->loaded": [], "dW(j-1) read->S(j) issue": [], "dW issue->read": [],
             "dZ stored->dQ issue": []}
        for c in range(NCTA):
            for w in (0, 1):
                st, iss = t[c, w], t[c, 2 + w]
                for j in range(1, NT):
                    if st[j, 1] and iss[j, 8]:
                        x["S issue->loaded"].append(int(st[j, 1] - iss[j, 8]))
                    if iss[j, 8] and st[j - 1, 3]:
                        x["dW(j-1) read->S(j) issue"].append(int(iss[j, 8] - st[j - 1, 3]))
                    if st[j, 3] and iss[j, 10]:
                        x["dW issue->read"].append(int(st[j, 3] - iss[j, 10]))
                    if iss[j, 11] and st[j, 6]:
                        x["dZ stored->dQ issue"].append(int(iss[j, 11] - st[j, 6]))
        print("median clk:", {k: int(np.median(v)) for k, v in x.items() if v})


if __name__ == "__main__":
    main()
