#!/usr/bin/env python3
"""One C3-shaped forward (B=1 H=32 L=32768 d=128), skip on or off, for ncu (tuning aid):
    ncu ... python tools/fwd_one.py --skip 1 --family dead"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17980_b200 import ops  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--skip", type=int, default=1)
ap.add_argument("--family", default="dead")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
q, k, v = make_qkv(1, 32, 32768, 128, seed=3, family=a.family, mu=-8.0, with_do=False)
for _ in range(a.reps):
    ops.blocked_forward(q, k, v, skip=bool(a.skip), counters=False)
torch.cuda.synchronize()
