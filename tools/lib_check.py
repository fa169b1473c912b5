#!/usr/bin/env python3
"""Parity check of an alternative library build (tuning aid): store vs recompute mode
bit-identical, and gradients vs the default build and the oracle on a small case.
    python tools/lib_check.py paper_2410_17980_b200/libsbattn_x.so"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_17980_b200 import _lib, ops  # noqa: E402
from tests.gpu_util import make_qkv, oracle_bwd, oracle_fwd, rel_to_max, to64  # noqa: E402


def run(path, q, k, v, d_o, store, skip=False):
    _lib._lib = None
    _lib._lib = _lib.load(os.path.abspath(path))
    o, lr, st, cache = ops.blocked_forward(q, k, v, skip=skip)
    dq, dk, dv, _ = ops.blocked_backward_twophase(cache, d_o, store_tiles=store)
    torch.cuda.synchronize()
    return o, dq, dk, dv


alt = sys.argv[1]
for (B, H, L, d, skip) in ((1, 2, 640, 128, False), (2, 3, 700, 64, False), (4, 64, 512, 128, True),
                           (1, 1, 4096, 128, False)):
    q, k, v, d_o = make_qkv(B, H, L, d, seed=3)
    a_s = run(alt, q, k, v, d_o, True, skip)
    a_r = run(alt, q, k, v, d_o, False, skip)
    base = run(os.path.join(ROOT, "paper_2410_17980_b200", "libsbattn.so"), q, k, v, d_o, True, skip)
    same_modes = all(torch.equal(x, y) for x, y in zip(a_s, a_r))
    same_base = all(torch.equal(x, y) for x, y in zip(a_s, base))
    ref = oracle_fwd(q[:1, :1], k[:1, :1], v[:1, :1], skip=skip)
    rdq, rdk, rdv, _ = oracle_bwd(q[:1, :1], k[:1, :1], v[:1, :1], d_o[:1, :1], ref)
    errs = [rel_to_max(to64(a_s[i + 1][:1, :1]), r) for i, r in enumerate((rdq, rdk, rdv))]
    print((B, H, L, d, skip), "store==recompute", same_modes, "== default build", same_base,
          "oracle", ["%.2e" % e for e in errs], flush=True)
