#!/usr/bin/env python3
"""C3 skip-on backward time, chunked (default workspace cap) vs one call (tuning aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_17980_b200 as sb  # noqa: E402
from tests.gpu_util import make_qkv  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "random"
q, k, v, d_o = make_qkv(1, 32, 32768, 128, seed=11, family=fam, mu=-6.0)
_, _, st, cache = sb.blocked_forward(q, k, v, skip=True)
for cap in (8, 40, 8, 40):
    sb.ops.WORKSPACE_MAX_BYTES = cap << 30
    n = len(list(sb.ops._unit_chunks(cache, True, sb.ops.workspace_cap_bytes())))
    for _ in range(2):
        sb.blocked_backward_twophase(cache, d_o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        sb.blocked_backward_twophase(cache, d_o)
    b.record()
    torch.cuda.synchronize()
    print(f"{fam}: cap {cap} GiB, {n} chunk(s): backward {a.elapsed_time(b) / 5:.3f} ms", flush=True)

# host-side submission time per call (no sync inside): does the GPU starve?
import time  # noqa: E402
for cap in (8, 40):
    sb.ops.WORKSPACE_MAX_BYTES = cap << 30
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        sb.blocked_backward_twophase(cache, d_o)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{fam}: cap {cap} GiB host submit {(t1 - t0) / 5 * 1e3:.3f} ms/call, "
          f"wall {(t2 - t0) / 5 * 1e3:.3f} ms/call", flush=True)
