#!/usr/bin/env python3
"""Skip-off vs skip-on forward time of library variants on one C3-shaped family (tuning aid):
    python tools/fwd_ab.py libsbattn.so libsbattn_x.so ... [--family dead]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17980_b200 import _lib, ops  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

fam = "dead"
libs = [a for a in sys.argv[1:] if a.endswith(".so")]
if "--family" in sys.argv:
    fam = sys.argv[sys.argv.index("--family") + 1]
q, k, v = make_qkv(1, 32, 32768, 128, seed=3, family=fam, mu=-8.0, with_do=False)
for rnd in range(4):
    for path in libs:
        _lib._lib = None  # (load() caches only the default path)
        _lib._lib = _lib.load(os.path.join(ROOT, "paper_2410_17980_b200", path))
        res = []
        for skip in (False, True):
            ops.blocked_forward(q, k, v, skip=skip, counters=False)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(6):
                ops.blocked_forward(q, k, v, skip=skip, counters=False)
            b.record()
            torch.cuda.synchronize()
            res.append(a.elapsed_time(b) / 6)
        print(f"{path:32s} {fam}: skip off {res[0]:.3f} ms, skip on {res[1]:.3f} ms", flush=True)
