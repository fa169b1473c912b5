"""Generate golden vectors from the reference itself (run in the build container).

TEST INFRASTRUCTURE.  Imports the reference package read-only from
/root/reference/pkg/src (it cannot travel to the GPU box) and writes
tests/golden/*.npz.  Inputs are NOT stored: tests regenerate them with the
reference's Philox stream convention restated in tests/golden_inputs.py
(numerics.py:145-155), and each fixture carries a SHA-256 of the inputs so a
generation drift is caught before any numerical comparison.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from sbattn import attention as ref_att  # noqa: E402
from sbattn import blocked as ref_blk  # noqa: E402
from sbattn import numerics as ref_num  # noqa: E402

from tests.golden_inputs import CASES, make_inputs, digest  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def m_dict_to_array(m_blocks, layout, L):
    """RowLogAccumulator.m_blocks (blocked.py:70-80) -> [n_tiles, block] (NaN = absent)."""
    nb, blk = layout.n_blocks, layout.block
    out = np.full((nb * (nb + 1) // 2, blk), np.nan)
    for (qb, kb), vals in m_blocks.items():
        out[qb * (qb + 1) // 2 + kb, : len(vals)] = vals
    return out


def run_case(name, spec):
    inp = make_inputs(spec)
    q, k, v, d_o = inp["q"], inp["k"], inp["v"], inp["d_o"]
    ro = inp.get("row_offset")
    block, dtype = spec["block"], np.dtype(spec.get("dtype", "float64"))
    skip = spec.get("skip", False)
    skip_eps = spec.get("skip_eps")
    H, L, d = q.shape
    res = {"digest": np.frombuffer(digest(inp).encode(), dtype=np.uint8)}
    outs = {key: [] for key in ("o", "log_rem", "first_kb", "visited", "M",
                                "dq", "dk", "dv", "dense_o", "dense_dq", "dense_dk",
                                "dense_dv", "dense_log_rem")}
    layout = ref_blk.plan_blocks(L, block)
    for h in range(H):
        o, acc, stats = ref_blk.blocked_forward(
            q[h], k[h], v[h], layout, skip=skip, skip_eps=skip_eps, two_phase=True,
            dtype=dtype)
        cache = ref_blk.make_cache(np.asarray(q[h], dtype), np.asarray(k[h], dtype),
                                   np.asarray(v[h], dtype), layout, acc, stats)
        row = None if ro is None else np.asarray(ro[h], dtype)
        dq, dk, dv, _ = ref_blk.blocked_backward_twophase(cache, np.asarray(d_o[h], dtype),
                                                           row_offset=row)
        outs["o"].append(o)
        outs["log_rem"].append(acc.a)
        outs["first_kb"].append(stats.first_kb)
        outs["visited"].append(stats.visited)
        outs["M"].append(m_dict_to_array(acc.m_blocks, layout, L))
        outs["dq"].append(dq)
        outs["dk"].append(dk)
        outs["dv"].append(dv)
        if spec.get("dense", True):
            o_ref, c_ref = ref_att.sb_forward(q[h], k[h], v[h])
            if ro is not None:
                c_ref["d_a_extra"] = np.broadcast_to(-ro[h][None, :], (L, L))
            g = ref_att.sb_backward(c_ref, d_o[h])
            outs["dense_o"].append(o_ref)
            outs["dense_dq"].append(g[0])
            outs["dense_dk"].append(g[1])
            outs["dense_dv"].append(g[2])
            outs["dense_log_rem"].append(np.log(np.maximum(ref_att.sb_remaining_mass(c_ref["a"]), 1e-300)))
    keep = spec.get("keep", None)
    for key, vals in outs.items():
        if not vals or (keep is not None and key not in keep):
            continue
        res[key] = np.stack([np.asarray(x) for x in vals])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **res)
    return res


def constants():
    """Known answers pinned by the reference's own tests."""
    sp = ref_num.softplus_stable
    res = dict(
        softplus_x=np.array([-20.0, 0.0, 15.0, 16.0, 100.0, -3.0]),
    )
    res["softplus_y"] = np.array([sp(float(x)) for x in res["softplus_x"]])
    # test_attention.py:60-69, :126-132 — A = 0.5 / 0.25 on zero logits
    z3 = np.zeros((3, 3))
    res["weights_zero3"] = ref_att.sb_weights_direct(z3)
    np.savez_compressed(os.path.join(OUT, "constants.npz"), **res)


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, spec in CASES.items():
        r = run_case(name, spec)
        print(f"{name}: " + ", ".join(f"{k}{tuple(v.shape)}" for k, v in r.items() if k != "digest"))
    constants()
    print("numpy", np.__version__)


if __name__ == "__main__":
    main()
