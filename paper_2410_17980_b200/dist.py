"""Multi-GPU partitioning of the hot path: independent (batch, head) units.

Stick-breaking attention has no cross-head term anywhere in the reference
(blocked.py, attention.py): every (b, h) unit is an independent L x d problem
(SURVEY.md §8(e)).  So the data path needs no collective at all — each rank
runs the kernels on its own contiguous range of units.  A collective appears
only when a caller wants the full result on one rank (end-to-end layer
checks): ``gather_units`` all-gathers the per-rank shards (NCCL over NVLink on
B200s, gloo on CPU) and the result is bit-identical to a single-GPU run
because the per-unit arithmetic does not change.
"""

from __future__ import annotations

import torch


def unit_range(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n_units for rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_bh(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's slice of a (B, H, ...) tensor, flattened over (B, H) units.

    Returns a (1, U, ...) view (U = this rank's unit count) that the kernels
    accept directly as batch 1 with U heads.
    """
    B, H = x.shape[:2]
    lo, hi = unit_range(B * H, rank, world)
    return x.reshape(B * H, *x.shape[2:])[lo:hi].unsqueeze(0)


def gather_units(local: torch.Tensor, B: int, H: int, group=None) -> torch.Tensor:
    """All-gather per-rank (1, U_r, ...) shards back into the (B, H, ...) tensor."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_units = B * H
    sizes = [unit_range(n_units, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    tail = local.shape[2:]
    buf = local.new_zeros((1, width) + tuple(tail))
    buf[:, : local.shape[1]] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf.contiguous(), group=group)
    parts = [o[0, : hi - lo] for o, (lo, hi) in zip(outs, sizes)]
    return torch.cat(parts, 0).reshape((B, H) + tuple(tail))
