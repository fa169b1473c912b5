#!/usr/bin/env python3
"""One skip-off and one skip-on forward on the same C3-shaped inputs (ncu target):
    python tools/fwd_pair.py [--family dead] [--L 32768] [--H 32]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_17980_b200 as sb  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="dead")
ap.add_argument("--mu", type=float, default=-8.0)
ap.add_argument("--L", type=int, default=32768)
ap.add_argument("--H", type=int, default=32)
a = ap.parse_args()
q, k, v = make_qkv(1, a.H, a.L, 128, seed=3, family=a.family, mu=a.mu, with_do=False)
for skip in (False, True):
    sb.blocked_forward(q, k, v, skip=skip, counters=False)
torch.cuda.synchronize()
print("ok")
