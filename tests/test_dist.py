"""world_size-2 gloo test of the multi-GPU partitioning (runs on CPU).

Each rank takes its contiguous share of the (b, h) units, runs the hot path on
it (here the CPU oracle stands in for the kernel so the test runs without a
GPU), and the shards are all-gathered: the result must be bit-identical to
the single-process run, because units are independent and
the data path has no collective.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2410_17980_b200 import dist as sbdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, k, v, d_o, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, H = q.shape[:2]
    shard = [sbdist.shard_bh(t, rank, world) for t in (q, k, v, d_o)]
    qs, ks, vs, ds = (s[0].numpy() for s in shard)
    fwd = oracle.tiled_forward(qs, ks, vs, block=64, n_threads=1)
    dq, dk, dv, _ = oracle.tiled_backward(qs, ks, vs, ds, fwd, block=64, n_threads=1)
    outs = {}
    for name, arr in (("o", fwd["o"]), ("dq", dq), ("dk", dk), ("dv", dv)):
        outs[name] = sbdist.gather_units(torch.from_numpy(arr).unsqueeze(0), B, H)
    if rank == 0:
        torch.save(outs, os.path.join(out_dir, "gathered.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather_bit_identical(tmp_path):
    g = torch.Generator().manual_seed(0)
    B, H, L, d = 1, 3, 96, 16
    q, k, v, d_o = (torch.randn(B, H, L, d, generator=g, dtype=torch.float64) for _ in range(4))
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, d_o, str(tmp_path)), nprocs=2, join=True)
    got = torch.load(os.path.join(tmp_path, "gathered.pt"))
    fwd = oracle.tiled_forward(q.numpy(), k.numpy(), v.numpy(), block=64, n_threads=1)
    dq, dk, dv, _ = oracle.tiled_backward(q.numpy(), k.numpy(), v.numpy(), d_o.numpy(), fwd,
                                          block=64, n_threads=1)
    for name, ref in (("o", fwd["o"]), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert np.array_equal(got[name].numpy(), ref), name


def test_lpt_assign_balances_quadratic_cost():
    lens = [8192, 512, 4096, 4096, 2048, 1024, 8192, 512]
    a = sbdist.lpt_assign(lens, 2)
    assert sorted(sum(a, [])) == list(range(len(lens)))
    loads = [sum(lens[i] ** 2 for i in s) for s in a]
    assert max(loads) / min(loads) < 1.1
    assert sbdist.lpt_assign(lens, 1) == [list(range(len(lens)))]


def _varlen_worker(rank, world, port, q, k, v, cu, lens, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    assign = sbdist.lpt_assign(lens, world)
    qs, ks, vs = (sbdist.shard_varlen(t, cu, assign[rank])[0] for t in (q, k, v))
    _, cul = sbdist.shard_varlen(q, cu, assign[rank])
    o = torch.zeros_like(qs)
    for i in range(len(assign[rank])):  # per-sequence oracle stands in for the kernel
        s0, s1 = int(cul[i]), int(cul[i + 1])
        f = oracle.tiled_forward(qs[s0:s1].transpose(0, 1).numpy(), ks[s0:s1].transpose(0, 1).numpy(),
                                 vs[s0:s1].transpose(0, 1).numpy(), block=64, n_threads=1)
        o[s0:s1] = torch.from_numpy(f["o"]).transpose(0, 1)
    full = sbdist.gather_varlen(o, cu, assign)
    if rank == 0:
        torch.save(full, os.path.join(out_dir, "varlen.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_varlen_lpt_shard_and_gather_bit_identical(tmp_path):
    g = torch.Generator().manual_seed(1)
    lens = [70, 130, 20, 64]
    H, d = 2, 16
    T = sum(lens)
    q, k, v = (torch.randn(T, H, d, generator=g, dtype=torch.float64) for _ in range(3))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    mp.spawn(_varlen_worker, args=(2, _free_port(), q, k, v, cu, lens, str(tmp_path)), nprocs=2,
             join=True)
    got = torch.load(os.path.join(tmp_path, "varlen.pt"))
    for i, L in enumerate(lens):
        s0 = int(cu[i])
        f = oracle.tiled_forward(q[s0:s0 + L].transpose(0, 1).numpy(),
                                 k[s0:s0 + L].transpose(0, 1).numpy(),
                                 v[s0:s0 + L].transpose(0, 1).numpy(), block=64, n_threads=1)
        assert np.array_equal(got[s0:s0 + L].transpose(0, 1).numpy(), f["o"]), i


def test_lpt_units_split_heads_when_sequences_are_too_coarse():
    lens = [7045, 5404, 4438, 2584, 2876, 826, 1089, 638, 1858, 6758, 5500, 7522, 4380, 5171,
            7968, 1479]
    G, a = sbdist.lpt_assign_units(lens, 16, 8)
    units = sorted(sum(a, []))
    assert units == sorted((i, g) for i in range(len(lens)) for g in range(G))
    loads = [sum(lens[i] ** 2 for i, _ in s) for s in a]
    assert max(loads) / (sum(loads) / 8) <= 1.05
    assert G > 1  # whole sequences alone cannot balance 8 ranks here
    x = torch.arange(sum(lens) * 16 * 2, dtype=torch.float32).reshape(sum(lens), 16, 2)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    t, c = sbdist.shard_varlen_units(x, cu, a[0], G)
    assert t.shape[1] == 16 // G and int(c[-1]) == t.shape[0] and c.numel() == len(a[0]) + 1
    i, g = a[0][0]
    hg = 16 // G
    assert torch.equal(t[: lens[i]], x[int(cu[i]): int(cu[i]) + lens[i], g * hg:(g + 1) * hg])
