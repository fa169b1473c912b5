#!/usr/bin/env python3
"""C4: packed variable-length stick-breaking fwd+bwd (BASELINE.json configs[3]).

Total 65,536 tokens, H=16, d=64 bf16; sequence lengths drawn by a seeded RNG in
[512, 8192] (the list is printed).  Reports fwd+bwd time, tokens/s and
algorithmic TFLOP/s (sum_b 7*H*L_b^2*d, the FA causal convention).

Multi-GPU: (sequence, head-group) units are assigned to ranks
by greedy LPT on L_b^2 (dist.lpt_assign_units: heads split into the fewest
groups that balance the ranks); a rank runs all its units as one packed call
(each unit a "sequence" of H/G heads).  The data path has no collective; time =
max over ranks.
  - under torchrun (WORLD_SIZE > 1): every rank runs its share on its own GPU;
  - `--simulate-ranks N` on one GPU: the N shares run one after the other and
    the report gives each share's time, i.e. the strong-scaling speed-up the
    assignment allows (T_all / max_r T_r) with the kernels unchanged.

    python tools/varlen_bench.py [--simulate-ranks 8] [--steps 10]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_17980_b200 as sb  # noqa: E402
from paper_2410_17980_b200 import dist as sbdist  # noqa: E402


def draw_lengths(total=65536, lo=512, hi=8192, seed=0):
    rng = np.random.default_rng(seed)
    lens = []
    while sum(lens) < total:
        lens.append(int(min(rng.integers(lo, hi + 1), total - sum(lens))))
    return lens


def time_step(q, k, v, d_o, cu, steps, warmup):
    def step():
        o, _, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu, counters=False)
        sb.blocked_backward_twophase(cache, d_o)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=65536)
    ap.add_argument("--H", type=int, default=16)
    ap.add_argument("--D", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--simulate-ranks", type=int, default=0)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    lens = draw_lengths(a.tokens, seed=a.seed)
    T, H, D = sum(lens), a.H, a.D
    cu_host = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    g = torch.Generator(device=dev).manual_seed(a.seed)
    q, k, v, d_o = (torch.randn(T, H, D, device=dev, dtype=torch.bfloat16, generator=g)
                    for _ in range(4))
    flops = lambda ls: sum(7.0 * H * L * L * D for L in ls)  # noqa: E731

    res = {"workload": f"C4: packed varlen, {T} tokens, {len(lens)} sequences "
                       f"(lengths {min(lens)}..{max(lens)}, seed {a.seed}), H={H} d={D} bf16, "
                       f"fwd+bwd, skip off", "lengths": lens}
    n_ranks = world if world > 1 else max(1, a.simulate_ranks)
    G, assign = sbdist.lpt_assign_units(lens, H, n_ranks)
    if world == 1:
        t_all = time_step(q, k, v, d_o, cu_host, a.steps, a.warmup)  # host offsets: no sync
        res.update(ms=t_all, tokens_per_s=T / (t_all / 1e3),
                   tflops=flops(lens) / (t_all / 1e3) / 1e12)
    if n_ranks > 1:
        shares = assign if world == 1 else [assign[rank]]
        times = []
        for units in shares:
            parts = [sbdist.shard_varlen_units(t, cu_host, units, G) for t in (q, k, v, d_o)]
            times.append(time_step(*(p[0] for p in parts), parts[0][1], a.steps, a.warmup))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor(times, device=dev, dtype=torch.float64)
            allt = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            times = [x.item() for x in allt]
        loads = [sum(lens[i] ** 2 for i, _ in u) for u in assign]
        res["ranks"] = {"n": n_ranks, "mode": "torchrun" if world > 1 else "simulated on 1 GPU",
                        "head_groups": G, "assignment": assign, "ms_per_rank": times,
                        "ms_max": max(times),
                        "tokens_per_s": T / (max(times) / 1e3),
                        "tflops": flops(lens) / (max(times) / 1e3) / 1e12,
                        "lpt_load_imbalance": max(loads) / (sum(loads) / n_ranks)}
        if "ms" in res:
            res["ranks"]["speedup_vs_1"] = res["ms"] / max(times)
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
