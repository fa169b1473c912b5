"""Parity at the benchmarked shape (C2) and on the persistent kernels' cross-item paths.

The kernels are persistent (one CTA per SM, a dynamic work queue) and order their
items in L2 groups of `Geom::ugroup` units.  Small tests run about one item per CTA,
so the code that runs only when a CTA takes its 2nd, 3rd, ... item (the SchedRing
wrap, the q/o/dq/kv/acc "free" barrier phases, the L2-grouped order with
ugroup < B*H) needs launches with many items per CTA.  These tests supply them:

* C2 itself (B=8 H=16 L=4096 d=128: ~14 forward items per CTA, grouped order on),
  store and recompute backward, against the f64 oracle on units spread over several
  L2 groups (0, 7, 8, 63, 127), and store == recompute bit for bit on every unit;
  C2 with skip on: first_kb exact on all 128 units.
* B=4 H=64 L=1024 (1024 forward items, ~7 per CTA; grouped order with 32- and
  64-unit groups), d = 64 and 128, skip off and on, against the oracle on EVERY unit.
* a packed varlen batch with more than 148 items per launch.

Reference semantics: blocked.py:129-206 (forward), :299-392 (two-phase backward);
the random-config sweep these mirror is test_blocked.py:89-98.
"""

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import make_qkv, rel_to_max, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _units(t, idx):
    """(B, H, L, d) -> (len(idx), L, d) float64 of the flattened (b, h) units idx."""
    B, H = t.shape[:2]
    flat = t.reshape(B * H, *t.shape[2:])
    return to64(flat[torch.as_tensor(idx, device=t.device)])


def _oracle(q, k, v, d_o, idx, skip=False):
    qs, ks, vs, ds = (_units(t, idx) for t in (q, k, v, d_o))
    ref = oracle.tiled_forward(qs, ks, vs, block=64, skip=skip, skip_eps=1e-6, dtype=np.float64)
    rdq, rdk, rdv, _ = oracle.tiled_backward(qs, ks, vs, ds, ref, block=64, dtype=np.float64)
    return ref, rdq, rdk, rdv


def _gpu(q, k, v, d_o, skip, store):
    import paper_2410_17980_b200 as sb
    o, log_rem, st, cache = sb.blocked_forward(q, k, v, skip=skip, skip_eps=1e-6)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, store_tiles=store)
    torch.cuda.synchronize()
    return dict(o=o, log_rem=log_rem, first_kb=st.first_kb, visited=st.visited, dq=dq, dk=dk,
                dv=dv)


def _check_units(got, ref, rdq, rdk, rdv, idx, tag):
    B, H = got["o"].shape[:2]
    errs = {}
    for name, r in (("o", ref["o"]), ("dq", rdq), ("dk", rdk), ("dv", rdv)):
        g = _units(got[name], idx)
        errs[name] = max(rel_to_max(g[i], r[i]) for i in range(len(idx)))
    lr = to64(got["log_rem"].reshape(B * H, -1)[torch.as_tensor(idx)])
    np.testing.assert_allclose(np.exp(lr), np.exp(ref["log_rem"]), atol=TOL, rtol=TOL)
    fkb = got["first_kb"].reshape(B * H, -1)[torch.as_tensor(idx)].cpu().numpy()
    np.testing.assert_array_equal(fkb, ref["first_kb"])
    print(tag, {n: f"{e:.2e}" for n, e in errs.items()})
    assert max(errs.values()) < TOL, (tag, errs)


# ---------------------------------------------------------------- C2 (the bench shape)
C2_UNITS = [0, 7, 8, 63, 127]  # across several 8-unit L2 groups (ugroup = 8 at C2)


@pytest.fixture(scope="module")
def c2():
    q, k, v, d_o = make_qkv(8, 16, 4096, 128, seed=2024)
    runs = {store: _gpu(q, k, v, d_o, False, store) for store in (True, False)}
    return (q, k, v, d_o), runs


def test_c2_store_equals_recompute_all_units(c2):
    _, runs = c2
    for n in ("o", "log_rem", "dq", "dk", "dv"):
        assert torch.equal(runs[True][n], runs[False][n]), n


@pytest.mark.parametrize("store", [True, False])
def test_c2_matches_oracle(c2, store):
    (q, k, v, d_o), runs = c2
    ref, rdq, rdk, rdv = _oracle(q, k, v, d_o, C2_UNITS)
    _check_units(runs[store], ref, rdq, rdk, rdv, C2_UNITS, f"C2 store={store}")


def test_c2_skip_first_kb_all_units():
    """C2 with skip on: first_kb and the visited count exact on all 128 units."""
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(8, 16, 4096, 128, seed=77, with_do=False)
    o, log_rem, st, _ = sb.blocked_forward(q, k, v, skip=True, skip_eps=1e-6)
    torch.cuda.synchronize()
    qs, ks, vs = (to64(t.reshape(128, 4096, 128)) for t in (q, k, v))
    ref = oracle.tiled_forward(qs, ks, vs, block=64, skip=True, skip_eps=1e-6)
    np.testing.assert_array_equal(st.first_kb.reshape(128, -1).cpu().numpy(), ref["first_kb"])
    assert st.visited == ref["visited"]
    assert rel_to_max(to64(o.reshape(128, 4096, 128)), ref["o"]) < TOL


# ---------------------------------------------------------------- many items per CTA
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("skip,family", [(False, "random"), (True, "shift")])
def test_many_items_per_cta_all_units(d, skip, family):
    """B=4 H=64 L=1024: 1024 forward / phase-1 items and 2048 phase-2 items over
    148 CTAs, grouped L2 order with ugroup < B*H; every unit vs the oracle, store
    mode bit-identical to recompute mode."""
    B, H, L = 4, 64, 1024
    q, k, v, d_o = make_qkv(B, H, L, d, seed=d + int(skip), family=family, mu=-6.0)
    a = _gpu(q, k, v, d_o, skip, True)
    b = _gpu(q, k, v, d_o, skip, False)
    for n in ("o", "dq", "dk", "dv"):
        assert torch.equal(a[n], b[n]), n
    idx = list(range(B * H))
    ref, rdq, rdk, rdv = _oracle(q, k, v, d_o, idx, skip=skip)
    assert a["visited"] == ref["visited"]
    _check_units(a, ref, rdq, rdk, rdv, idx, f"B{B} H{H} L{L} d{d} skip={skip}")


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("store", [True, False])
def test_varlen_many_items(store, d):
    """A packed batch with > 148 items per launch (40 sequences, 8 heads)."""
    import paper_2410_17980_b200 as sb
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(1, 1100, size=40)]
    H = 8
    g = torch.Generator().manual_seed(9)
    T = sum(lens)
    q, k, v, d_o = (torch.randn(T, H, d, generator=g).to(torch.bfloat16).cuda() for _ in range(4))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    n_items = H * sum(((n + 127) // 128 + 1) // 2 for n in lens)
    assert n_items > 148
    o, log_rem, st, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu.cuda())
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, store_tiles=store)
    torch.cuda.synchronize()
    worst = {}
    for b, Lb in enumerate(lens):
        s0, s1 = int(cu[b]), int(cu[b + 1])
        sl = [to64(t[s0:s1].transpose(0, 1)) for t in (q, k, v, d_o)]
        ref = oracle.tiled_forward(*sl[:3], block=64)
        rdq, rdk, rdv, _ = oracle.tiled_backward(*sl, ref, block=64)
        for n, got, r in (("o", o, ref["o"]), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            e = rel_to_max(to64(got[s0:s1].transpose(0, 1)), r)
            if e > worst.get(n, (0.0,))[0]:
                worst[n] = (e, b, Lb)
    print("varlen many items: worst (err, seq, L)", worst)
    assert max(e for e, _, _ in worst.values()) < TOL, worst


@pytest.mark.parametrize("d", [64, 128])
def test_varlen_many_items_deterministic(d):
    """Reruns are bit-identical (the dynamic work queue hands items to different CTAs
    every run, so any state leaking between a CTA's items shows up here).  Regression:
    a warpgroup without a tile in two consecutive items (short / odd-tile sequences)
    used to pass a parity wait two phases early and read a stale Q tile."""
    import paper_2410_17980_b200 as sb
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(1, 1100, size=40)] + [1, 100, 1, 130, 60, 1, 1]
    g = torch.Generator().manual_seed(9)
    q, k, v, d_o = (torch.randn(sum(lens), 8, d, generator=g).to(torch.bfloat16).cuda()
                    for _ in range(4))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32).cuda()
    ref = None
    for _ in range(6):
        o, lr, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu)
        grads = sb.blocked_backward_twophase(cache, d_o)[:3]
        cur = (o, lr) + tuple(grads)
        if ref is None:
            ref = tuple(t.clone() for t in cur)
        for a, b, n in zip(cur, ref, ("o", "log_rem", "dq", "dk", "dv")):
            assert torch.equal(a, b), n
