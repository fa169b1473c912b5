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


# ---------------------------------------------------------------- packed varlen (C4)
def lpt_assign(lengths, world: int) -> list[list[int]]:
    """Greedy longest-processing-time assignment of sequences to ranks.

    A sequence of length L costs ~L^2/2 tiles per head; the
    heaviest sequence goes to the least-loaded rank, ties to the lower rank.
    Returns, per rank, its sequence indices in ascending order.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]) ** 2, i))
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda j: (load[j], j))
        out[r].append(i)
        load[r] += int(lengths[i]) ** 2
    return [sorted(s) for s in out]


def shard_varlen(x: torch.Tensor, cu_host: torch.Tensor, seqs: list[int]):
    """Pack the sequences `seqs` of a packed (T, ...) tensor into a new packed
    tensor; returns (x_local, cu_local int32 [len(seqs)+1], on x's device)."""
    parts = [x[int(cu_host[i]): int(cu_host[i + 1])] for i in seqs]
    lens = [p.shape[0] for p in parts]
    cu = torch.zeros(len(seqs) + 1, dtype=torch.int32)
    if lens:
        cu[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int64), 0).to(torch.int32)
    local = torch.cat(parts, 0) if parts else x[:0]
    return local.contiguous(), cu.to(x.device)


def gather_varlen(local: torch.Tensor, cu_host: torch.Tensor, assignment, group=None):
    """All-gather per-rank packed shards and scatter them back into the original
    packed order (bit-identical to a single-GPU run)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    T = int(cu_host[-1])
    tail = local.shape[1:]
    sizes = [sum(int(cu_host[i + 1] - cu_host[i]) for i in a) for a in assignment]
    width = max(max(sizes), 1)
    buf = local.new_zeros((width,) + tuple(tail))
    buf[: local.shape[0]] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf.contiguous(), group=group)
    full = local.new_empty((T,) + tuple(tail))
    for r, seqs in enumerate(assignment):
        off = 0
        for i in seqs:
            n = int(cu_host[i + 1] - cu_host[i])
            full[int(cu_host[i]): int(cu_host[i]) + n] = outs[r][off: off + n]
            off += n
    return full


def lpt_assign_units(lengths, heads: int, world: int, tol: float = 1.02):
    """LPT over (sequence, head-group) units (C4 units are
    (sequence, head) pairs).  Heads are split into G equal groups, G the
    smallest power of two dividing `heads` whose assignment is within `tol` of
    a perfect balance (else the best one found).  Returns (G, per-rank lists of
    (sequence, group)); a rank runs one packed call per head group it holds.
    """
    best = None
    G = 1
    while G <= heads and heads % G == 0:
        units = [(i, g) for i in range(len(lengths)) for g in range(G)]
        w = [int(lengths[i]) ** 2 for i, _ in units]
        order = sorted(range(len(units)), key=lambda u: (-w[u], u))
        load = [0] * world
        out: list[list[tuple[int, int]]] = [[] for _ in range(world)]
        for u in order:
            r = min(range(world), key=lambda j: (load[j], j))
            out[r].append(units[u])
            load[r] += w[u]
        imb = max(load) / (sum(load) / world) if sum(load) else 1.0
        if best is None or imb < best[0] - 1e-9:
            best = (imb, G, [sorted(s) for s in out])
        if imb <= tol:
            break
        G *= 2
    return best[1], best[2]


def shard_varlen_units(x: torch.Tensor, cu_host: torch.Tensor, units, G: int):
    """Pack this rank's (sequence, head-group) units into ONE packed batch with
    H/G heads: unit (i, g) becomes a "sequence" holding tokens of sequence i and
    heads g*H/G .. (g+1)*H/G-1.  Returns (x_local (T_r, H/G, d), cu_local) with
    cu_local on the HOST: pass it straight to blocked_forward /
    stickbreaking_attention, which then plan without a device sync."""
    hg = x.shape[1] // G
    parts = [x[int(cu_host[i]): int(cu_host[i + 1]), g * hg:(g + 1) * hg] for i, g in units]
    lens = [p.shape[0] for p in parts]
    cu = torch.zeros(len(parts) + 1, dtype=torch.int32)
    if lens:
        cu[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int64), 0).to(torch.int32)
    local = torch.cat(parts, 0) if parts else x[:0, :hg]
    return local.contiguous(), cu
