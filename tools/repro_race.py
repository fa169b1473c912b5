"""Determinism probe: rerun the forward / backward many times on one input and report
which (sequence, row range) differ from the first run (debugging aid)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_17980_b200 as sb

def run(d, H=8, reps=30, varlen=True, store=True):
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(1, 1100, size=40)]
    g = torch.Generator().manual_seed(9)
    T = sum(lens)
    q, k, v, d_o = (torch.randn(T, H, d, generator=g).to(torch.bfloat16).cuda() for _ in range(4))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    cud = cu.cuda()
    ref = None
    bad = {}
    for i in range(reps):
        o, lr, st, cache = sb.blocked_forward(q, k, v, cu_seqlens=cud)
        dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, store_tiles=store)
        torch.cuda.synchronize()
        cur = dict(o=o, lr=lr, dq=dq, dk=dk, dv=dv)
        if ref is None:
            ref = {n: t.clone() for n, t in cur.items()}
            continue
        for n, t in cur.items():
            diff = (t != ref[n])
            if diff.any():
                rows = torch.nonzero(diff.reshape(diff.shape[0], -1).any(1)).flatten().cpu()
                seqs = sorted(set(int(np.searchsorted(cu.numpy(), r, side="right") - 1) for r in rows.tolist()))
                heads = torch.nonzero(diff.reshape(diff.shape[0], H, -1).any(2).any(0)).flatten().tolist()
                bad.setdefault(n, []).append((i, len(rows), seqs[:8], heads))
    print(f"d={d} store={store}:", {n: v[:4] for n, v in bad.items()} or "deterministic", flush=True)

for d in (64, 128):
    for store in (True, False):
        run(d, store=store)
