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
