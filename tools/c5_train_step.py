#!/usr/bin/env python3
"""C5: training step of a 1.3B stick-breaking decoder stack (BASELINE.json configs[4]).

SBTransformer (paper_2410_17980_b200/layer.py, the reference toy model's architecture:
pre-LN attention + exact-GELU MLP blocks, untied head) at 1.3B parameters:
d_model 2048, 16 heads of 128, 24 layers, d_inter 8192, vocab 32768; synthetic tokens,
L = 4096, micro-batch `--batch` sequences per GPU.  One step = forward, masked-free
cross-entropy, backward, fused AdamW update; fp32 master weights, bf16 autocast for the
GEMMs (cuBLAS) and the stick-breaking op (this package's kernels).

Data-parallel over the GPUs of one node: one process per GPU under torchrun, DDP over
NCCL (gradient all-reduce over NVLink overlapped with the backward by DDP's buckets).
Timing: CUDA events around `--steps` steps after `--warmup`, max over ranks.
Reports tokens/s (whole job), ms/step, model TFLOP/s (6*N*tokens + attention 7*L*d per
token per layer) and the share of the step spent in the attention kernels (one rank,
from a separate forward+backward of the attention op alone at the same shape).

    python tools/c5_train_step.py [--layers 24] [--batch 2] [--steps 5]
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/c5_train_step.py
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_17980_b200.layer import SBTransformer, n_params, train_flops_per_token  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--d-model", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--kv-heads", type=int, default=0,
                    help="grouped-query key/value heads (0: = heads; the paper's 1.2B model: "
                         "--d-model 1536 --heads 12 --kv-heads 4)")
    ap.add_argument("--d-inter", type=int, default=8192)
    ap.add_argument("--vocab", type=int, default=32768)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    model = SBTransformer(a.vocab, a.layers, a.d_model, a.heads, a.d_inter,
                          n_kv_head=a.kv_heads or None).to(dev)
    N = n_params(model)
    flops_tok = train_flops_per_token(model, a.seq)
    net = model
    if world > 1:
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, weight_decay=0.0, fused=True)
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    tokens = torch.randint(0, a.vocab, (a.batch, a.seq + 1), device=dev, generator=g)

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = net(tokens[:, :-1])
        loss = F.cross_entropy(logits.float().view(-1, a.vocab), tokens[:, 1:].reshape(-1))
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        return loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    tok = world * a.batch * a.seq
    res = {"workload": f"C5: SBTransformer {N / 1e9:.2f}B params (d={a.d_model}, {a.heads} heads "
                       f"x {a.d_model // a.heads}{f' over {a.kv_heads} kv heads' if a.kv_heads else ''}, "
                       f"{a.layers} layers, d_inter={a.d_inter}, "
                       f"vocab={a.vocab}), L={a.seq}, {a.batch} seq/GPU, synthetic tokens, "
                       f"bf16 autocast + fp32 AdamW (fused)",
           "n_gpus": world, "parallelism": f"dp{world} (DDP over NCCL)" if world > 1 else "1 GPU",
           "ms_per_step": ms, "tokens_per_s": tok / (ms / 1e3),
           "model_tflops": tok * flops_tok / (ms / 1e3) / 1e12,
           "loss": float(loss.item()), "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    # attention share: the op alone, fwd+bwd on this rank's shape, per step
    import paper_2410_17980_b200 as sb
    H, dh = a.heads, a.d_model // a.heads
    q, k, v, do = (torch.randn(a.batch, a.seq, H, dh, device=dev, dtype=torch.bfloat16)
                   .transpose(1, 2) for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)
    for i in range(a.warmup + 3):
        if i == a.warmup:
            e0.record()
        sb.stickbreaking_attention(q, k, v).backward(do)
    e1.record()
    torch.cuda.synchronize()
    attn_ms = e0.elapsed_time(e1) / 3 * a.layers
    res["attention_ms_per_step"] = attn_ms
    res["attention_share"] = attn_ms / ms
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
