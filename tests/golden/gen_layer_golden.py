"""Golden vectors of the reference's attention sublayer and decoder stack.

TEST INFRASTRUCTURE, run in the build container: imports the reference toy model
read-only from /root/reference/pkg/src (`model.mha_forward` / `mha_backward`,
`transformer_forward` / `transformer_backward`, model.py:243-358) and writes
tests/golden/layer_*.npz with its f64 OUTPUTS (stored as float16: the GPU path
computes the attention in bf16, so 11 mantissa bits are ample for the 2e-2-class
comparison).  Inputs and parameters are NOT stored: `layer_case_inputs` below
regenerates them from seeds with the reference's Philox stream convention
(tests/golden_inputs.py), and every fixture carries a SHA-256 of them.

    python tests/golden/gen_layer_golden.py
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests.golden_inputs import rng  # noqa: E402

SUBLAYER_CASES = {
    "layer_sb": dict(variant="sb", group_norm=False, seed=11),
    "layer_sb_remainder": dict(variant="sb_remainder", group_norm=False, seed=12),
    "layer_sb_remainder_bias_gn": dict(variant="sb_remainder_bias", group_norm=True, seed=13),
}
SUB_H, SUB_DH, SUB_L = 2, 64, 200
MODEL_CASE = dict(name="model_sb", vocab=32, n_layer=2, n_head=2, d_head=64, d_inter=256, L=150,
                  seed=21, init_std=0.06)


def sublayer_inputs(variant, group_norm, seed, H=SUB_H, dh=SUB_DH, L=SUB_L):
    """x, d_y and the sublayer parameters (reference names, prefix "attn")."""
    d = H * dh
    g = rng(seed)
    p = {f"attn.{n}": g.normal(0.0, 1.0 / math.sqrt(d), size=(d, d)) for n in ("wq", "wk", "wv", "wo")}
    if variant == "sb_remainder_bias":
        p["attn.r"] = g.normal(0.0, 1.0, size=(H, dh))
    if group_norm:
        p["attn.gn_g"] = 1.0 + 0.1 * g.normal(0.0, 1.0, size=(H, dh))
        p["attn.gn_b"] = 0.1 * g.normal(0.0, 1.0, size=(H, dh))
    x = g.normal(0.0, 1.0, size=(L, d))
    d_y = g.normal(0.0, 1.0, size=(L, d))
    return x, d_y, p


def model_inputs(c=MODEL_CASE):
    """tokens, d_logits and the parameters, drawn in model.init_params' order
    (model.py:87-117: embed, per layer wq wk wv wo w1 w2, head; norms at identity)."""
    V, d, di = c["vocab"], c["n_head"] * c["d_head"], c["d_inter"]
    g = rng(c["seed"])
    std = c["init_std"]
    p = {"embed": g.normal(0.0, std, size=(V, d))}
    for i in range(c["n_layer"]):
        pre = f"layers.{i}"
        p[f"{pre}.ln1.g"], p[f"{pre}.ln1.b"] = np.ones(d), np.zeros(d)
        for n in ("wq", "wk", "wv", "wo"):
            p[f"{pre}.attn.{n}"] = g.normal(0.0, std, size=(d, d))
        p[f"{pre}.ln2.g"], p[f"{pre}.ln2.b"] = np.ones(d), np.zeros(d)
        p[f"{pre}.mlp.w1"] = g.normal(0.0, std, size=(d, di))
        p[f"{pre}.mlp.w2"] = g.normal(0.0, std, size=(di, d))
    p["final_norm.g"], p["final_norm.b"] = np.ones(d), np.zeros(d)
    p["head"] = g.normal(0.0, std, size=(d, V))
    tokens = rng(c["seed"], 1).integers(0, V, size=c["L"])
    d_logits = 0.1 * rng(c["seed"], 2).normal(0.0, 1.0, size=(c["L"], V))
    return tokens, d_logits, p


def digest(*arrays, params=None) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    for k in sorted(params or {}):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from sbattn import model as M
    from sbattn.numerics import Rng

    for name, c in SUBLAYER_CASES.items():
        x, d_y, p = sublayer_inputs(c["variant"], c["group_norm"], c["seed"])
        cfg = M.AttentionConfig(n_head=SUB_H, d_head=SUB_DH, variant=c["variant"],
                                group_norm=c["group_norm"], impl="reference")
        y, cache = M.mha_forward(x, p, cfg, prefix="attn")
        d_x, grads = M.mha_backward(cache, d_y)
        out = {"y": y, "d_x": d_x, **{"grad." + k: v for k, v in grads.items()}}
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            digest=digest(x, d_y, params=p),
                            **{k: np.asarray(v, dtype=np.float16) for k, v in out.items()})
        print(name, {k: v.shape for k, v in out.items()})

    c = MODEL_CASE
    tokens, d_logits, p = model_inputs(c)
    cfg = M.ModelConfig(vocab_size=c["vocab"], n_layer=c["n_layer"], d_inter=c["d_inter"],
                        attn=M.AttentionConfig(n_head=c["n_head"], d_head=c["d_head"], variant="sb",
                                               impl="reference"))
    # the restated init draws the reference's own parameters
    ref_p = M.init_params(cfg, Rng(c["seed"]), init_std=c["init_std"])
    assert set(ref_p) == set(p) and all(np.array_equal(ref_p[k], p[k]) for k in p)
    logits, cache = M.transformer_forward(tokens, p, cfg)
    grads = M.transformer_backward(cache, d_logits)
    out = {"logits": logits, **{"grad." + k: v for k, v in grads.items()}}
    np.savez_compressed(os.path.join(HERE, c["name"] + ".npz"),
                        digest=digest(tokens, d_logits, params=p),
                        **{k: np.asarray(v, dtype=np.float16) for k, v in out.items()})
    print(c["name"], len(out), "arrays")


if __name__ == "__main__":
    main()
