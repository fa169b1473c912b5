#!/usr/bin/env python3
"""Time the three kernels of an alternative build of the library (tuning aid).

    python tools/ablate.py paper_2410_17980_b200/libsbattn_nomath.so
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17980_b200 import _lib, ops  # noqa: E402


def main(path):
    _lib._lib = _lib.load(path)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    B, H, L, D = 8, 16, 4096, 128
    q, k, v, do = (torch.randn(B, H, L, D, device=dev, dtype=torch.bfloat16, generator=g)
                   for _ in range(4))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for it in range(6):
        ev[0].record()
        o, _, _, cache = ops.blocked_forward(q, k, v, counters=False)
        ev[1].record()
        out = tuple(torch.empty_like(q) for _ in range(3))
        ws = torch.empty(ops.workspace_bytes(cache), device=q.device, dtype=torch.uint8)
        ops.blocked_backward_twophase(cache, do, phases=1, out=out, workspace=ws)
        ev[2].record()
        ops.blocked_backward_twophase(cache, do, phases=2, out=out, workspace=ws)
        ev[3].record()
    torch.cuda.synchronize()
    print(path, "fwd %.3f p1 %.3f p2 %.3f ms" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                                                ev[2].elapsed_time(ev[3])))


if __name__ == "__main__":
    main(sys.argv[1])
