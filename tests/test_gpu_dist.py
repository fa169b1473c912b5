"""The multi-GPU partitioning with the CUDA kernels on the data path.

Two processes (world size 2, gloo) share the one GPU of the test box, each running
the real kernels on its share: contiguous (b, h) units (`dist.shard_bh`), or LPT
(sequence, head-group) units of a packed varlen batch (`dist.lpt_assign_units`).
The shards are all-gathered and must be BIT-IDENTICAL to one process running the
whole batch, because units are independent (blocked.py:122-126, :195: the
reference maps independent query blocks; there is no cross-head term) and the
kernels have no atomics on the data path.  The data path has no collective; the
gather is the end-to-end check NCCL does on a real multi-GPU node.

A 2-layer stick-breaking decoder (layer.py) trained one step with DDP over the two
processes gets the same gradients as one process averaging both micro-batches.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    return dist


def _run_units(q, k, v, d_o, store=True):
    import paper_2410_17980_b200 as sb
    o, log_rem, st, cache = sb.blocked_forward(q, k, v)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, store_tiles=store)
    torch.cuda.synchronize()
    return {"o": o, "log_rem": log_rem, "first_kb": st.first_kb, "dq": dq, "dk": dk, "dv": dv}


def _bh_worker(rank, world, port, inputs, out_dir):
    dist = _init(rank, world, port)
    from paper_2410_17980_b200 import dist as sbdist
    q, k, v, d_o = (t.cuda() for t in inputs)
    B, H = q.shape[:2]
    local = _run_units(*(sbdist.shard_bh(t, rank, world) for t in (q, k, v, d_o)))
    full = {n: sbdist.gather_units(t.cpu(), B, H) for n, t in local.items()}
    if rank == 0:
        torch.save(full, os.path.join(out_dir, "bh.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d", [64, 128])
def test_two_ranks_bh_shards_bit_identical(tmp_path, d):
    from tests.gpu_util import make_qkv
    q, k, v, d_o = make_qkv(2, 5, 1100, d, seed=d, device="cpu")
    mp.spawn(_bh_worker, args=(2, _free_port(), (q, k, v, d_o), str(tmp_path)), nprocs=2,
             join=True)
    got = torch.load(os.path.join(tmp_path, "bh.pt"))
    ref = _run_units(q.cuda(), k.cuda(), v.cuda(), d_o.cuda())
    for n, t in ref.items():
        assert torch.equal(got[n], t.cpu()), n


def _varlen_worker(rank, world, port, inputs, cu, lens, out_dir):
    dist = _init(rank, world, port)
    import paper_2410_17980_b200 as sb
    from paper_2410_17980_b200 import dist as sbdist
    H = inputs[0].shape[1]
    G, assign = sbdist.lpt_assign_units(lens, H, world)
    hg = H // G
    loc = [sbdist.shard_varlen_units(t, cu, assign[rank], G) for t in inputs]
    cu_l = loc[0][1]
    q, k, v, d_o = (x[0].cuda() for x in loc)
    o, _, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu_l)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
    torch.cuda.synchronize()
    # back to (sequence, head) order: gather every rank's packed units, then scatter
    outs = {}
    for name, t in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        t = t.cpu()
        width = max(sum(lens[i] for i, _ in a) for a in assign)
        buf = t.new_zeros((width,) + tuple(t.shape[1:]))
        buf[: t.shape[0]] = t
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        full = t.new_zeros((int(cu[-1]), H) + tuple(t.shape[2:]))
        for r, units in enumerate(assign):
            off = 0
            for i, g in units:
                n = lens[i]
                full[int(cu[i]): int(cu[i]) + n, g * hg:(g + 1) * hg] = parts[r][off: off + n]
                off += n
        outs[name] = full
    if rank == 0:
        torch.save({"G": G, **outs}, os.path.join(out_dir, "varlen.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_varlen_lpt_units_bit_identical(tmp_path):
    import paper_2410_17980_b200 as sb
    lens = [1500, 90, 700, 2300, 1, 640, 1200]
    H, d = 8, 64
    g = torch.Generator().manual_seed(3)
    T = sum(lens)
    inputs = [torch.randn(T, H, d, generator=g).to(torch.bfloat16) for _ in range(4)]
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    mp.spawn(_varlen_worker, args=(2, _free_port(), inputs, cu, lens, str(tmp_path)), nprocs=2,
             join=True)
    got = torch.load(os.path.join(tmp_path, "varlen.pt"))
    q, k, v, d_o = (t.cuda() for t in inputs)
    o, _, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
    torch.cuda.synchronize()
    for n, t in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert torch.equal(got[n], t.cpu()), n


def _model(seed):
    from paper_2410_17980_b200.layer import SBTransformer
    torch.manual_seed(seed)
    return SBTransformer(vocab_size=512, n_layer=2, d_model=256, n_head=2, d_inter=512).cuda()


def _loss(model, tokens):
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(tokens[:, :-1])
    return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]),
                                             tokens[:, 1:].reshape(-1))


def _ddp_worker(rank, world, port, tokens, out_dir):
    dist = _init(rank, world, port)
    from torch.nn.parallel import DistributedDataParallel as DDP
    model = DDP(_model(0), device_ids=[0])
    loss = _loss(model, tokens[rank].cuda())
    loss.backward()
    torch.cuda.synchronize()
    if rank == 0:
        torch.save({n: p.grad.cpu() for n, p in model.module.named_parameters()},
                   os.path.join(out_dir, "ddp.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_ddp_two_layer_step_matches_single_process(tmp_path):
    """C5's data-parallel path (tools/c5_train_step.py: DDP gradient all-reduce) on a
    2-layer stack: rank r trains on micro-batch r; DDP's averaged gradients equal one
    process's average of the two micro-batch gradients."""
    g = torch.Generator().manual_seed(7)
    tokens = torch.randint(0, 512, (2, 2, 513), generator=g)
    mp.spawn(_ddp_worker, args=(2, _free_port(), tokens, str(tmp_path)), nprocs=2, join=True)
    got = torch.load(os.path.join(tmp_path, "ddp.pt"))
    model = _model(0)
    grads = []
    for r in range(2):
        model.zero_grad()
        _loss(model, tokens[r].cuda()).backward()
        grads.append({n: p.grad.detach().clone() for n, p in model.named_parameters()})
    for n in grads[0]:
        want = ((grads[0][n] + grads[1][n]) / 2).cpu()
        torch.testing.assert_close(got[n], want, rtol=1e-5, atol=1e-7, msg=n)
