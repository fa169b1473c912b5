"""Helpers shared by the GPU parity tests (inputs, oracle calls, metrics)."""

from __future__ import annotations

import math

import numpy as np
import torch

import oracle


def make_qkv(B, H, L, d, seed=0, family="random", mu=-6.0, device="cuda", with_do=True):
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = torch.randn(B, H, L, d, generator=g)
    k = torch.randn(B, H, L, d, generator=g)
    v = torch.randn(B, H, L, d, generator=g)
    d_o = torch.randn(B, H, L, d, generator=g)
    if family == "shift":
        q[..., 0] = mu * math.sqrt(d)
        k[..., 0] = 1.0
    elif family == "saturating":
        q.zero_(); k.zero_()
        j = torch.arange(L)
        q[..., j, j % d] = 40.0 * math.sqrt(d)
        k[..., j, (j + 1) % d] = 1.0
    elif family == "dead":
        q.zero_(); k.zero_()
        q[..., 0] = 100.0 * math.sqrt(d)
        k[..., 0] = -1.0
    ts = [t.to(torch.bfloat16).to(device) for t in (q, k, v, d_o)]
    return ts if with_do else ts[:3]


def to64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def oracle_fwd(q, k, v, skip=False, skip_eps=1e-6):
    return oracle.tiled_forward(to64(q), to64(k), to64(v), block=64, skip=skip,
                                skip_eps=skip_eps, dtype=np.float64)


def oracle_bwd(q, k, v, d_o, fwd, row_offset=None):
    ro = None if row_offset is None else to64(row_offset)
    return oracle.tiled_backward(to64(q), to64(k), to64(v), to64(d_o), fwd, block=64,
                                 row_offset=ro, dtype=np.float64)


rel_to_max = oracle.rel_to_max
max_rel_err = oracle.max_rel_err
