#!/usr/bin/env python3
"""C2 strong scaling: the fixed C2 problem (B=8, H=16 -> 128 (b,h) units,
L=4096, d=128 bf16, fwd+bwd) split into contiguous unit ranges over G ranks.

Each rank runs its (1, U_r, L, d) shard (dist.shard_bh) with no collective on the data path,
so a rank's time is the time of its shard alone.  On one GPU the G shares run one after the
other and the report gives each share's CUDA-event time and the speed-up T_1 / max_r T_r the
partition allows with the kernels unchanged; under torchrun every rank times its own share on
its own GPU and rank 0 reports the max over ranks.

    python tools/strong_scaling.py [--ranks 2,4,8] [--steps 10]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_17980_b200 as sb  # noqa: E402
from paper_2410_17980_b200 import dist as sbdist  # noqa: E402


def time_fwd_bwd(q, k, v, d_o, steps, warmup, phases=None):
    """Mean fwd+bwd ms per step; `phases` (a list) also receives [fwd, phase 1, phase 2] ms."""
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]

    def step(e=None):
        if e is not None:
            e[0].record()
        _, _, _, cache = sb.blocked_forward(q, k, v, counters=False)
        if e is not None:
            e[1].record()
        out = tuple(torch.empty_like(q) for _ in range(3))
        ws = torch.empty(sb.ops.workspace_bytes(cache), device=q.device, dtype=torch.uint8)
        sb.blocked_backward_twophase(cache, d_o, phases=1, out=out, workspace=ws)
        if e is not None:
            e[2].record()
        sb.blocked_backward_twophase(cache, d_o, phases=2, out=out, workspace=ws)
        if e is not None:
            e[3].record()
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    for i in range(steps):
        step(ev[i])
    torch.cuda.synchronize()
    if phases is not None:
        phases[:] = [sum(e[j].elapsed_time(e[j + 1]) for e in ev) / steps for j in range(3)]
    return sum(e[0].elapsed_time(e[3]) for e in ev) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--H", type=int, default=16)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    g = torch.Generator(device=dev).manual_seed(1234)
    q, k, v, d_o = (torch.randn(a.B, a.H, a.L, a.D, device=dev, dtype=torch.bfloat16, generator=g)
                    for _ in range(4))
    res = {"workload": f"C2 strong scaling: B={a.B} H={a.H} L={a.L} d={a.D} bf16 fwd+bwd, "
                       f"{a.B * a.H} (b,h) units split contiguously, skip off"}
    if world == 1:
        p1 = []
        t1 = time_fwd_bwd(q, k, v, d_o, a.steps, a.warmup, p1)
        res["ms_1"] = t1
        res["ms_fwd_p1_p2_1"] = p1
        res["ranks"] = []
        for n in (int(x) for x in a.ranks.split(",")):
            times, ph = [], []
            for r in range(n):
                pr = []
                times.append(time_fwd_bwd(*(sbdist.shard_bh(t, r, n) for t in (q, k, v, d_o)),
                                          a.steps, a.warmup, pr))
                ph.append([round(x, 4) for x in pr])
            res["ranks"].append({"n": n, "mode": "simulated on 1 GPU", "ms_per_rank": times,
                                 "ms_fwd_p1_p2_per_rank": ph,
                                 "ms_max": max(times), "speedup_vs_1": t1 / max(times)})
    else:
        import torch.distributed as dist
        t = time_fwd_bwd(*(sbdist.shard_bh(x, rank, world) for x in (q, k, v, d_o)),
                         a.steps, a.warmup)
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        allt = [torch.empty_like(tt) for _ in range(world)]
        dist.all_gather(allt, tt)
        times = [x.item() for x in allt]
        res["ranks"] = [{"n": world, "mode": "torchrun", "ms_per_rank": times,
                         "ms_max": max(times)}]
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
