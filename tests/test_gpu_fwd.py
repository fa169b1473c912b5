"""GPU parity of the forward kernel (K1) against the CPU oracle, through the C ABI.

bf16 path tolerance (BASELINE.json): max|delta|/max|ref| <= 2e-2 per tensor;
skip decisions (first_kb, visited) bit-exact against the f64 oracle run on the
same bf16-rounded inputs with skip_eps = 1e-6.
"""

import numpy as np
import pytest
import torch

from tests.gpu_util import make_qkv, max_rel_err, oracle_bwd, oracle_fwd, rel_to_max, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("B,H,L,d", [(1, 2, 256, 64), (2, 2, 320, 128), (1, 1, 64, 128),
                                     (1, 3, 200, 64), (1, 1, 1, 64), (2, 1, 1000, 128)])
def test_forward_matches_oracle(B, H, L, d):
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(B, H, L, d, seed=L + d, with_do=False)
    o, log_rem, stats, _ = sb.blocked_forward(q, k, v)
    torch.cuda.synchronize()
    ref = oracle_fwd(q, k, v)
    err_o = rel_to_max(to64(o), ref["o"])
    err_a = max_rel_err(to64(log_rem), ref["log_rem"])
    print(f"B{B} H{H} L{L} d{d}: o {err_o:.3e} log_rem {err_a:.3e}")
    assert err_o < TOL
    assert err_a < TOL
    assert stats.visited == ref["visited"] == stats.total
    np.testing.assert_array_equal(stats.first_kb.cpu().numpy(), ref["first_kb"])
    # row 0 of every sequence attends to nothing (test_attention.py:145-148)
    assert torch.count_nonzero(o[:, :, 0]) == 0


@pytest.mark.parametrize("family,L,d", [("saturating", 512, 128), ("random", 1024, 128),
                                        ("dead", 512, 64), ("shift", 1024, 128),
                                        ("saturating", 300, 64)])
def test_skip_decisions_bit_exact(family, L, d):
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(1, 2, L, d, seed=7, family=family, mu=-6.0, with_do=False)
    o, log_rem, stats, _ = sb.blocked_forward(q, k, v, skip=True, skip_eps=1e-6)
    torch.cuda.synchronize()
    ref = oracle_fwd(q, k, v, skip=True, skip_eps=1e-6)
    np.testing.assert_array_equal(stats.first_kb.cpu().numpy(), ref["first_kb"])
    assert stats.visited == ref["visited"]
    err = max_rel_err(to64(o), ref["o"])
    print(f"{family} L{L} d{d}: visited {stats.visited}/{stats.total} o max_rel_err {err:.3e}")
    assert err < TOL
    if family in ("saturating", "random") and L >= 512:
        assert stats.skipped / stats.total > 0.5  # test_blocked.py:79-87
    if family == "dead":
        assert stats.skipped == 0


def test_skip_soundness():
    """test_blocked.py:109-114: skip on vs off agree on random inputs."""
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(1, 2, 768, 128, seed=9, with_do=False)
    o_off, *_ = sb.blocked_forward(q, k, v, skip=False)
    o_on, _, st, _ = sb.blocked_forward(q, k, v, skip=True)
    assert st.skipped > 0
    assert rel_to_max(to64(o_on), to64(o_off)) < 1e-2


def test_deterministic():
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(2, 2, 384, 128, seed=3, with_do=False)
    a = sb.blocked_forward(q, k, v)
    b = sb.blocked_forward(q, k, v)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_bshd_layout():
    """Strided (B, L, H, d) storage viewed as (B, H, L, d) gives the same result."""
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(1, 4, 256, 64, seed=5, with_do=False)
    o_ref, *_ = sb.blocked_forward(q, k, v)
    qs, ks, vs = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (q, k, v))
    assert qs.stride() != q.stride()
    o, *_ = sb.blocked_forward(qs, ks, vs)
    assert torch.equal(o.contiguous(), o_ref)


@pytest.mark.parametrize("family,mu,L,d", [("saturating", 0.0, 512, 128), ("shift", 8.0, 384, 64),
                                           ("shift", 100.0, 256, 128), ("saturating", 0.0, 200, 64)])
def test_large_logits_skip_off(family, mu, L, d):
    """Skip off with group products beyond 2^64 (the per-element path): o and log_rem
    vs the oracle, including logits past the exp2 clamp (mu = 100: z ~ 100 nats)."""
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(1, 2, L, d, seed=5, family=family, mu=mu, with_do=False)
    o, log_rem, _, cache = sb.blocked_forward(q, k, v, skip=False)
    torch.cuda.synchronize()
    ref = oracle_fwd(q, k, v)
    err_o = rel_to_max(to64(o), ref["o"])
    err_a = max_rel_err(to64(log_rem), ref["log_rem"])
    print(f"{family} mu{mu} L{L} d{d}: o {err_o:.3e} log_rem {err_a:.3e}")
    assert err_o < TOL
    assert err_a < TOL
    # the backward rolls M back from the final a through these rows too (including the
    # exact lt path of logits whose 2^z overflows, mu = 100): gradients vs the oracle,
    # store and recompute mode bit-identical
    g = torch.Generator().manual_seed(9)
    d_o = torch.randn(q.shape, generator=g).to(torch.bfloat16).cuda()
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o)
    r = sb.blocked_backward_twophase(cache, d_o, store_tiles=False)
    torch.cuda.synchronize()
    for x, y in zip((dq, dk, dv), r[:3]):
        assert torch.equal(x, y)
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, d_o, ref)
    errs = [max_rel_err(to64(x), y) for x, y in ((dq, rdq), (dk, rdk), (dv, rdv))]
    print("  grads (max_rel_err)", [f"{e:.2e}" for e in errs])
    assert max(errs) < TOL
