#!/usr/bin/env python3
"""Small forward + both backward modes (skip off and on, d = 64 and 128, tails) for
compute-sanitizer (GPU only):

    for t in memcheck racecheck synccheck; do
      compute-sanitizer --tool $t python tools/sanitize_case.py [--many]; done
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_17980_b200 as sb  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

CASES = [(1, 2, 320, 128, False), (1, 2, 256, 64, True)]
if "--many" in sys.argv:
    # >= 3 items per CTA in every kernel (512 forward / phase-1 items, 1024 phase-2
    # items over 148 CTAs): the cross-item barrier phases and the work-queue ring wrap
    CASES = [(4, 64, 512, 64, False), (4, 64, 512, 128, True)]
if "--many" in sys.argv:
    # partial skipping (mu = -6 shifted logits): the skip-on forward's vote words, stops
    # mid-stream and the producer's ring release after a stop
    CASES.append((2, 16, 1024, 128, "shift"))
for (B, H, L, d, skip) in CASES:
    fam = "random"
    if skip == "shift":
        fam, skip = "shift", True
    q, k, v, do = make_qkv(B, H, L, d, seed=1, family=fam, mu=-6.0)
    o, lr, st, cache = sb.blocked_forward(q, k, v, skip=skip)
    for store in (False, True):
        dq, dk, dv, _ = sb.blocked_backward_twophase(cache, do, store_tiles=store)
    torch.cuda.synchronize()
if "--many" in sys.argv:  # packed varlen, > 148 items per launch, d = 64
    g = torch.Generator().manual_seed(5)
    lens = [int(x) for x in torch.randint(1, 1100, (40,), generator=g)]
    T = sum(lens)
    q, k, v, do = (torch.randn(T, 8, 64, generator=g).to(torch.bfloat16).cuda() for _ in range(4))
    cu = torch.tensor([0] + torch.tensor(lens).cumsum(0).tolist(), dtype=torch.int32).cuda()
    o, lr, st, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu)
    for store in (False, True):
        dq, dk, dv, _ = sb.blocked_backward_twophase(cache, do, store_tiles=store)
    torch.cuda.synchronize()
print("sanitizer case ok")
