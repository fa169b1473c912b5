#!/usr/bin/env python3
"""Host-side cost of the op's Python layer per call (cProfile; tuning aid)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_17980_b200 as sb  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

q, k, v, d_o = make_qkv(1, 32, 32768, 128, seed=11, family="random")
_, _, st, cache = sb.blocked_forward(q, k, v, skip=True)
for _ in range(3):
    sb.blocked_backward_twophase(cache, d_o)
    sb.blocked_forward(q, k, v, skip=True, counters=False)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    sb.blocked_forward(q, k, v, skip=True, counters=False)
    sb.blocked_backward_twophase(cache, d_o)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
