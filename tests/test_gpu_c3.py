"""C3 (B=1, H=32, L=32768, d=128, skip on, skip_eps=1e-6): skip decisions bit-exact on
ALL 32 heads of four input families, against golden decisions of the float64
blocked_forward rule (blocked.py:165-193) on the same bf16-rounded inputs
(tests/golden/gen_c3_first_kb.py, pinned to the C oracle by tests/test_oracle.py);
plus o/dq/dk/dv of one C3 head against the C oracle.

The golden file also records how close the decisions are: the smallest
|max a - log eps| per family (the mu=-6 family has checks within 1e-4 nats).
"""

import os

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import make_qkv, rel_to_max, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2
GOLD = os.path.join(os.path.dirname(__file__), "golden", "c3_first_kb.npz")
FAMILIES = {"random": ("random", 0.0), "shift-6": ("shift", -6.0), "shift-8": ("shift", -8.0),
            "saturating": ("saturating", 0.0)}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.mark.parametrize("name", list(FAMILIES))
def test_c3_first_kb_all_heads(gold, name):
    import paper_2410_17980_b200 as sb
    B, H, L, D = (int(x) for x in gold["meta/shape"])
    fam, mu = FAMILIES[name]
    q, k, v = make_qkv(B, H, L, D, seed=int(gold["meta/seed"]), family=fam, mu=mu,
                       with_do=False)
    o, log_rem, st, _ = sb.blocked_forward(q, k, v, skip=True, skip_eps=float(gold["meta/eps"]))
    torch.cuda.synchronize()
    got = st.first_kb[0].cpu().numpy()
    want = gold[f"{name}/first_kb"].astype(np.int64)
    bad = np.argwhere(got != want)
    print(f"{name}: visited {st.visited} (golden {int(gold[name + '/visited'].sum())}), "
          f"closest decision {float(gold[name + '/min_margin'].min()):.2e} nats, "
          f"{int(gold[name + '/n_within_1e-4'].sum())} within 1e-4")
    assert bad.size == 0, f"{len(bad)} decisions differ, first at (head, qb) {bad[:5].tolist()}"
    assert st.visited == int(gold[f"{name}/visited"].sum())


@pytest.mark.parametrize("name,grads", [("random", True), ("shift-6", False)])
def test_c3_head_matches_oracle(name, grads):
    """One C3 head through the skip-on forward (and backward, random family) vs the
    f64 C oracle: the oracle visits only what it does not skip, so the random family
    (99% skipped) runs fwd+bwd in seconds; mu=-6 (77% skipped) checks o."""
    import paper_2410_17980_b200 as sb
    fam, mu = FAMILIES[name]
    q, k, v, d_o = make_qkv(1, 1, 32768, 128, seed=5, family=fam, mu=mu)
    o, log_rem, st, cache = sb.blocked_forward(q, k, v, skip=True, skip_eps=1e-6)
    ref = oracle.tiled_forward(to64(q[0]), to64(k[0]), to64(v[0]), block=64, skip=True,
                               skip_eps=1e-6)
    np.testing.assert_array_equal(st.first_kb[0].cpu().numpy(), ref["first_kb"])
    errs = {"o": rel_to_max(to64(o[0]), ref["o"])}
    if grads:
        dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
        torch.cuda.synchronize()
        rdq, rdk, rdv, _ = oracle.tiled_backward(to64(q[0]), to64(k[0]), to64(v[0]),
                                                 to64(d_o[0]), ref, block=64)
        errs.update(dq=rel_to_max(to64(dq[0]), rdq), dk=rel_to_max(to64(dk[0]), rdk),
                    dv=rel_to_max(to64(dv[0]), rdv))
    print(name, {n: f"{e:.2e}" for n, e in errs.items()})
    assert max(errs.values()) < TOL


def test_long_rows_rollback_matches_oracle():
    """Rows with |a| ~ 10^4 nats (L = 12288, skip off, random inputs): phase 1 rolls
    every M snapshot back from the forward's final a; a rounding error proportional to
    |a| would show up as a relative error of e^M near the diagonal.  o / dq / dk / dv
    vs the f64 oracle, store and recompute mode bit-identical."""
    import paper_2410_17980_b200 as sb
    q, k, v, d_o = make_qkv(1, 1, 12288, 128, seed=23)
    o, log_rem, st, cache = sb.blocked_forward(q, k, v)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
    r = sb.blocked_backward_twophase(cache, d_o, store_tiles=False)
    torch.cuda.synchronize()
    for a, b in zip((dq, dk, dv), r[:3]):
        assert torch.equal(a, b)
    ref = oracle.tiled_forward(to64(q[0]), to64(k[0]), to64(v[0]), block=64)
    assert float(ref["log_rem"].min()) < -5000.0
    rdq, rdk, rdv, _ = oracle.tiled_backward(to64(q[0]), to64(k[0]), to64(v[0]), to64(d_o[0]),
                                             ref, block=64)
    errs = {"o": rel_to_max(to64(o[0]), ref["o"]), "dq": rel_to_max(to64(dq[0]), rdq),
            "dk": rel_to_max(to64(dk[0]), rdk), "dv": rel_to_max(to64(dv[0]), rdv),
            "log_rem": float(np.max(np.abs(to64(log_rem[0]) - ref["log_rem"])
                                    / np.maximum(1.0, np.abs(ref["log_rem"]))))}
    print("long rows", {n: f"{e:.2e}" for n, e in errs.items()})
    assert max(errs.values()) < TOL


def test_partial_skip_long_rows_grads_match_oracle():
    """mu = -6 shifted logits at L = 16384, skip on (partial skipping: rows stop at
    different key blocks): the skip-on forward's decisions, its compensated a (the
    backward's state) and phase 1's M rollback over the visited tiles only; o, dq, dk, dv
    vs the f64 oracle on two heads."""
    import paper_2410_17980_b200 as sb
    q, k, v, d_o = make_qkv(1, 2, 16384, 128, seed=29, family="shift", mu=-6.0)
    o, log_rem, st, cache = sb.blocked_forward(q, k, v, skip=True, skip_eps=1e-6)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
    torch.cuda.synchronize()
    ref = oracle.tiled_forward(to64(q[0]), to64(k[0]), to64(v[0]), block=64, skip=True,
                               skip_eps=1e-6)
    np.testing.assert_array_equal(st.first_kb[0].cpu().numpy(), ref["first_kb"])
    assert 0.05 < 1.0 - st.visited / st.total < 0.95  # partial skipping
    rdq, rdk, rdv, _ = oracle.tiled_backward(to64(q[0]), to64(k[0]), to64(v[0]), to64(d_o[0]),
                                             ref, block=64)
    errs = {"o": rel_to_max(to64(o[0]), ref["o"]), "dq": rel_to_max(to64(dq[0]), rdq),
            "dk": rel_to_max(to64(dk[0]), rdk), "dv": rel_to_max(to64(dv[0]), rdv)}
    print("partial skip", st.visited, "/", st.total, {n: f"{e:.2e}" for n, e in errs.items()})
    assert max(errs.values()) < TOL
