#!/usr/bin/env python3
"""Time the three kernels of an alternative build of the library (tuning aid).

    python tools/ablate.py paper_2410_17980_b200/libsbattn_nomath.so [--c4] [--D 64]

Default workload C2 (B=8 H=16 L=4096 d=128); --c4: the C4 packed varlen batch
(65,536 tokens, H=16, d=64, tools/varlen_bench.py's lengths).  Prints the median of
5 timed steps (after 3 warm-up steps) per kernel.
"""
import argparse
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17980_b200 import _lib, ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib")
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--D", type=int, default=0)
    a = ap.parse_args()
    _lib._lib = None  # load() caches only the default path
    _lib._lib = _lib.load(os.path.abspath(a.lib))
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    cu = None
    if a.c4:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from varlen_bench import draw_lengths
        lens = draw_lengths()
        D = a.D or 64
        q, k, v, do = (torch.randn(sum(lens), 16, D, device=dev, dtype=torch.bfloat16, generator=g)
                       for _ in range(4))
        cu = torch.tensor([0] + torch.tensor(lens).cumsum(0).tolist(), dtype=torch.int32,
                          device=dev)
    else:
        B, H, L, D = 8, 16, 4096, a.D or 128
        q, k, v, do = (torch.randn(B, H, L, D, device=dev, dtype=torch.bfloat16, generator=g)
                       for _ in range(4))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    times = []
    for it in range(8):
        ev[0].record()
        o, _, _, cache = ops.blocked_forward(q, k, v, counters=False, cu_seqlens=cu)
        ev[1].record()
        out = tuple(torch.empty_like(q) for _ in range(3))
        ws = torch.empty(ops.workspace_bytes(cache), device=q.device, dtype=torch.uint8)
        ops.blocked_backward_twophase(cache, do, phases=1, out=out, workspace=ws)
        ev[2].record()
        ops.blocked_backward_twophase(cache, do, phases=2, out=out, workspace=ws)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 3:
            times.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
    med = [statistics.median(t[i] for t in times) for i in range(3)]
    print(a.lib, "fwd %.3f p1 %.3f p2 %.3f ms" % tuple(med), "(C4)" if a.c4 else "")


if __name__ == "__main__":
    main()
