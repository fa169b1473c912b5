#!/usr/bin/env python3
"""Host<->device copy rates the end-to-end bench depends on (tuning aid, GPU only).

512 MiB per direction per step (bench.py e2e: q, k, v, dO in; o, dq, dk, dv out), from /
to pinned host memory: H2D alone, D2H alone, both at once, each with 1 or 4 streams per
direction (the copy split into equal chunks).

    python tools/ubench/pcie_copy.py
"""
import torch

N = 512 << 20
dev = torch.device("cuda", 0)
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device=dev)
d_out = torch.empty(N, dtype=torch.uint8, device=dev)


def run(h2d, d2h, n_streams, reps=5):
    streams = [torch.cuda.Stream() for _ in range(2 * n_streams)]
    chunk = N // n_streams
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        for i in range(n_streams):
            sl = slice(i * chunk, (i + 1) * chunk)
            if h2d:
                streams[i].wait_event(a)
                with torch.cuda.stream(streams[i]):
                    d_in[sl].copy_(h_in[sl], non_blocking=True)
            if d2h:
                streams[n_streams + i].wait_event(a)
                with torch.cuda.stream(streams[n_streams + i]):
                    h_out[sl].copy_(d_out[sl], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return N / (ms / 1e3) / 1e9, ms


for n in (1, 4):
    for h2d, d2h, name in ((True, False, "H2D"), (False, True, "D2H"), (True, True, "both")):
        gbs, ms = run(h2d, d2h, n)
        print(f"{name:5s} {n} stream(s)/dir: {gbs:6.1f} GB/s per direction, {ms:6.2f} ms per 512 MiB")
