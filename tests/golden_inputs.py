"""Deterministic inputs for the golden fixtures (shared by oracle/gen_golden.py
and the tests, so fixtures store only reference OUTPUTS).

The stream convention restates the reference's ``Rng``
(/root/reference/pkg/src/sbattn/numerics.py:135-155): Philox seeded by
``SeedSequence(entropy=seed, spawn_key=key)``, one child per head
(``Rng(seed).spawn(h)``), drawing q, k, v, d_o (and row_offset) in order.
Input families follow cli.py:387-405 / test_blocked.py:24-33 (saturating,
dead) and SURVEY.md §8(d) (logit shift by mu: q[:,0]=mu*sqrt(d), k[:,0]=1).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np


def rng(seed: int, *key: int) -> np.random.Generator:
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(int(t) for t in key))
    return np.random.Generator(np.random.Philox(ss))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def make_inputs(spec: dict) -> dict:
    H, L, d = spec["H"], spec["L"], spec["d"]
    fam = spec.get("family", "random")
    seed = spec.get("seed", 0)
    q = np.zeros((H, L, d)); k = np.zeros((H, L, d)); v = np.zeros((H, L, d))
    d_o = np.zeros((H, L, d))
    ro = np.zeros((H, L)) if spec.get("row_offset") else None
    for h in range(H):
        g = rng(seed, h)
        q[h], k[h], v[h], d_o[h] = (g.normal(0.0, 1.0, size=(L, d)) for _ in range(4))
        if ro is not None:
            ro[h] = g.normal(0.0, 1.0, size=(1, L))[0]
        if fam == "shift":
            mu = spec["mu"]
            q[h][:, 0] = mu * math.sqrt(d)
            k[h][:, 0] = 1.0
        elif fam == "saturating":
            q[h][:] = 0.0
            k[h][:] = 0.0
            for j in range(L):
                q[h][j, j % d] = 40.0 * math.sqrt(d)
            for i in range(L):
                k[h][i, (i + 1) % d] = 1.0
        elif fam == "dead":
            q[h][:] = 0.0
            k[h][:] = 0.0
            q[h][:, 0] = 100.0 * math.sqrt(d)
            k[h][:, 0] = -1.0
    out = dict(q=q, k=k, v=v, d_o=d_o)
    if ro is not None:
        out["row_offset"] = ro
    if spec.get("bf16"):
        out = {name: bf16_round(a) for name, a in out.items()}
    return out


def digest(inp: dict) -> str:
    h = hashlib.sha256()
    for name in sorted(inp):
        h.update(name.encode())
        h.update(np.ascontiguousarray(inp[name], dtype=np.float64).tobytes())
    return h.hexdigest()


CASES = {
    # config 1 (BASELINE.json configs[0]): B=1, H=4, L=256, d=64
    "c1_f64": dict(H=4, L=256, d=64, block=64, dense=False),
    "c1_f32": dict(H=4, L=256, d=64, block=64, dtype="float32", dense=False,
                   keep=("o", "log_rem", "first_kb", "visited", "dq", "dk", "dv")),
    "c1_f32_skip": dict(H=4, L=256, d=64, block=64, dtype="float32", skip=True, dense=False,
                        keep=("first_kb", "visited", "log_rem")),
    # tails and row_offset (test_blocked.py:230-273)
    "tail_100_64": dict(H=1, L=100, d=8, block=64, seed=17, row_offset=True),
    "tail_131_8": dict(H=1, L=131, d=8, block=8, seed=17, row_offset=True),
    "tail_65_64": dict(H=1, L=65, d=8, block=64, seed=17, row_offset=True),
    "tail_7_8": dict(H=1, L=7, d=8, block=8, seed=17, row_offset=True),
    "len1": dict(H=1, L=1, d=4, block=8, seed=16),
    # skip families (test_blocked.py:79-87, :116-124)
    "sat_skip": dict(H=1, L=256, d=32, block=16, family="saturating", skip=True, dense=False),
    "dead_skip": dict(H=1, L=256, d=8, block=16, family="dead", skip=True, dense=False,
                      keep=("o", "log_rem", "first_kb", "visited")),
    # bf16-rounded inputs, block 64, f64 oracle with eps 1e-6 (the GPU's setting)
    "bf16_rand_d64": dict(H=2, L=192, d=64, block=64, bf16=True, seed=3, skip=True,
                          skip_eps=1e-6, row_offset=True),
    "bf16_rand_d128": dict(H=1, L=320, d=128, block=64, bf16=True, seed=5, dense=False),
    "bf16_shift6_skip": dict(H=2, L=1024, d=128, block=64, bf16=True, seed=7, family="shift",
                             mu=-6.0, skip=True, skip_eps=1e-6, dense=False,
                             keep=("first_kb", "visited", "log_rem")),
    "bf16_sat_skip": dict(H=1, L=512, d=128, block=64, bf16=True, seed=9, family="saturating",
                          skip=True, skip_eps=1e-6, dense=False,
                          keep=("o", "first_kb", "visited", "log_rem")),
}
