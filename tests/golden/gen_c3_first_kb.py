#!/usr/bin/env python3
"""Golden skip decisions at C3 (B=1, H=32, L=32768, d=128, skip_eps=1e-6) for all 32
heads of four input families: random, logit shift mu=-6 and mu=-8, saturating.

TEST INFRASTRUCTURE (a checker, not the product).  The inputs are the ones the GPU
test regenerates (tests.gpu_util.make_qkv, seed 11, a seeded CPU torch generator,
rounded to bf16), so only the decisions are committed: tests/golden/c3_first_kb.npz.

The decision rule is blocked_forward's (reference blocked.py:165-193) in float64 on
the bf16-rounded inputs: for query block qb, key blocks kb = qb, qb-1, ... are
visited until, before a kb < qb, max over the block's rows of the running
a = sum of lt = -softplus(z) (numerics.py:33-47) over the visited tiles falls below
log(skip_eps) (:175-176); first_kb[qb] is the last visited kb (:192).  As in the
reference, a is accumulated tile by tile in order (a_cur + lt.sum(axis=1), :190).
The z of a whole run of key blocks comes from one BLAS product; that only changes
the last bits of z, far below the closest decision margin, which is recorded (per
family: the minimum |max a - log eps| over every check, and how many checks fall
within 1e-4 / 1e-3 nats).  tests/test_oracle.py pins this generator against the C
oracle (oracle/sb_oracle.c) on a smaller case.

    python tests/golden/gen_c3_first_kb.py [--procs 8]
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time
from multiprocessing import Pool

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # before numpy: one BLAS thread per worker
os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

FAMILIES = {"random": ("random", 0.0), "shift-6": ("shift", -6.0), "shift-8": ("shift", -8.0),
            "saturating": ("saturating", 0.0)}
SEED = 11
B, H, L, D = 1, 32, 32768, 128
EPS = 1e-6
OUT = os.path.join(ROOT, "tests", "golden", "c3_first_kb.npz")


def softplus(x):
    """numerics.py:33-47: log1p(exp(x)) for x <= 15, x above."""
    return np.where(x <= 15.0, np.log1p(np.exp(np.minimum(x, 15.0))), x)


def head_decisions(q, k, eps=EPS, block=64):
    """(first_kb [nb], visited, margins of every check) for one (L, d) float64 head."""
    Lh, d = q.shape
    nb = -(-Lh // block)
    scale = 1.0 / math.sqrt(d)
    log_eps = math.log(eps)
    first_kb = np.zeros(nb, dtype=np.int64)
    margins = []
    visited = 0
    for qb in range(nb):
        qs, qe = qb * block, min((qb + 1) * block, Lh)
        qblk = q[qs:qe]
        a = np.zeros(qe - qs)
        kb = qb  # next key block to visit
        lowest = qb
        chunk = 4
        done = False
        while kb >= 0 and not done:
            lo = max(0, kb - chunk + 1)
            ks, ke = lo * block, min((kb + 1) * block, Lh)
            z = (qblk @ k[ks:ke].T) * scale
            lt = -softplus(z)
            for kk in range(kb, lo - 1, -1):
                if kk < qb:
                    m = a.max() - log_eps
                    margins.append(m)
                    if m < 0:  # a_cur.max() < log_eps: stop (blocked.py:175-176)
                        done = True
                        break
                c0 = kk * block - ks
                c1 = min(c0 + block, ke - ks)
                t = lt[:, c0:c1]
                if kk == qb:  # _diag_mask: key column < query row
                    t = np.where(np.tri(t.shape[0], t.shape[1], -1, dtype=bool), t, 0.0)
                a = a + t.sum(axis=1)
                visited += 1
                lowest = kk
            kb = lo - 1
            chunk *= 2
        first_kb[qb] = lowest
    return first_kb, visited, np.asarray(margins)


def _work(args):
    fam, h, q, k = args
    t0 = time.time()
    fkb, vis, m = head_decisions(q, k)
    am = np.abs(m) if m.size else np.array([np.inf])
    return fam, h, fkb, vis, float(am.min()), int((am < 1e-4).sum()), int((am < 1e-3).sum()), \
        int(m.size), time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import torch
    from tests.gpu_util import make_qkv

    out = {}
    for name, (fam, mu) in FAMILIES.items():
        q, k = make_qkv(B, H, L, D, seed=SEED, family=fam, mu=mu, device="cpu",
                        with_do=False)[:2]
        qn = q[0].double().numpy()
        kn = k[0].double().numpy()
        jobs = [(name, h, qn[h].copy(), kn[h].copy()) for h in range(H)]
        t0 = time.time()
        with Pool(a.procs) as pool:
            res = pool.map(_work, jobs)
        res.sort(key=lambda r: r[1])
        out[f"{name}/first_kb"] = np.stack([r[2] for r in res]).astype(np.int16)
        out[f"{name}/visited"] = np.array([r[3] for r in res], dtype=np.int64)
        out[f"{name}/min_margin"] = np.array([r[4] for r in res])
        out[f"{name}/n_within_1e-4"] = np.array([r[5] for r in res], dtype=np.int64)
        out[f"{name}/n_within_1e-3"] = np.array([r[6] for r in res], dtype=np.int64)
        out[f"{name}/n_checks"] = np.array([r[7] for r in res], dtype=np.int64)
        tot = H * (L // 64) * (L // 64 + 1) // 2
        print(f"{name}: visited {out[name + '/visited'].sum()}/{tot} "
              f"min margin {out[name + '/min_margin'].min():.3e} nats, "
              f"within 1e-4: {out[name + '/n_within_1e-4'].sum()}, "
              f"within 1e-3: {out[name + '/n_within_1e-3'].sum()}, "
              f"{time.time() - t0:.0f}s", flush=True)
        del q, k
    out["meta/seed"] = np.array(SEED)
    out["meta/shape"] = np.array([B, H, L, D])
    out["meta/eps"] = np.array(EPS)
    out["meta/numpy"] = np.array(np.__version__)
    out["meta/torch"] = np.array(torch.__version__)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
