"""GPU parity of the two-phase backward (K2 + K3) against the CPU oracle.

The oracle (oracle/sb_oracle.c, pinned to the reference's golden vectors) runs
blocked_forward + blocked_backward_twophase in float64 on the same bf16
inputs.  Gate (BASELINE.json): max|delta|/max|ref| <= 2e-2 per gradient; for
degenerate families (saturating, dead) max_rel_err as SURVEY.md §8(c) says.
"""

import numpy as np
import pytest
import torch

from tests.gpu_util import (make_qkv, max_rel_err, oracle_bwd, oracle_fwd, rel_to_max,
                            to64)

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(q, k, v, d_o, skip=False, row_offset=None, store=None):
    import paper_2410_17980_b200 as sb
    o, log_rem, stats, cache = sb.blocked_forward(q, k, v, skip=skip, skip_eps=1e-6)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, row_offset=row_offset,
                                                 store_tiles=store)
    torch.cuda.synchronize()
    return o, log_rem, stats, dq, dk, dv


@pytest.mark.parametrize("B,H,L,d,skip,family,ro", [
    (1, 2, 320, 128, False, "random", False), (2, 1, 200, 64, False, "random", True),
    (1, 1, 1000, 128, False, "random", False), (1, 2, 130, 128, False, "random", True),
    (1, 2, 1024, 128, True, "shift", False), (1, 2, 512, 128, True, "saturating", False),
    (1, 2, 1, 64, False, "random", False), (1, 3, 900, 64, True, "random", True)])
def test_store_mode_bit_identical(B, H, L, d, skip, family, ro):
    """Store mode (phase 2 reads phase 1's dZ tiles) gives the recompute mode's
    gradients bit for bit: the stored tiles are exactly what phase 2 recomputes."""
    q, k, v, d_o = make_qkv(B, H, L, d, seed=L + d, family=family)
    row_offset = (torch.randn(B, H, L, generator=torch.Generator().manual_seed(3)).cuda()
                  if ro else None)
    a = _run(q, k, v, d_o, skip=skip, row_offset=row_offset, store=False)
    b = _run(q, k, v, d_o, skip=skip, row_offset=row_offset, store=True)
    for x, y, n in zip(a[3:], b[3:], ("dq", "dk", "dv")):
        assert torch.equal(x, y), n


@pytest.mark.parametrize("store", [False, True])
@pytest.mark.parametrize("B,H,L,d", [(1, 2, 256, 64), (1, 2, 320, 128), (1, 1, 64, 128),
                                     (2, 1, 200, 64), (1, 1, 1000, 128), (1, 1, 130, 128)])
def test_backward_matches_oracle(B, H, L, d, store):
    q, k, v, d_o = make_qkv(B, H, L, d, seed=L + 3 * d)
    o, _, _, dq, dk, dv = _run(q, k, v, d_o, store=store)
    ref = oracle_fwd(q, k, v)
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, d_o, ref)
    errs = [rel_to_max(to64(a), b) for a, b in ((dq, rdq), (dk, rdk), (dv, rdv))]
    print(f"B{B} H{H} L{L} d{d}: dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}")
    assert max(errs) < TOL


def test_backward_row_offset():
    """test_blocked.py:230-249: per-row offset subtracted from dO V^T."""
    q, k, v, d_o = make_qkv(1, 2, 384, 128, seed=11)
    ro = torch.randn(1, 2, 384, generator=torch.Generator().manual_seed(5)).cuda()
    _, _, _, dq, dk, dv = _run(q, k, v, d_o, row_offset=ro)
    ref = oracle_fwd(q, k, v)
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, d_o, ref, row_offset=ro)
    errs = [rel_to_max(to64(a), b) for a, b in ((dq, rdq), (dk, rdk), (dv, rdv))]
    print("row_offset:", errs)
    assert max(errs) < TOL


@pytest.mark.parametrize("family,L,d", [("saturating", 512, 128), ("random", 1024, 128),
                                        ("shift", 512, 64), ("dead", 256, 128)])
def test_backward_after_skip(family, L, d):
    """test_blocked.py:183-193: backward honours first_kb and matches the oracle."""
    q, k, v, d_o = make_qkv(1, 2, L, d, seed=21, family=family)
    _, _, stats, dq, dk, dv = _run(q, k, v, d_o, skip=True)
    ref = oracle_fwd(q, k, v, skip=True, skip_eps=1e-6)
    np.testing.assert_array_equal(stats.first_kb.cpu().numpy(), ref["first_kb"])
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, d_o, ref)
    if family in ("saturating", "dead"):
        errs = [max_rel_err(to64(a), b) for a, b in ((dq, rdq), (dk, rdk), (dv, rdv))]
    else:
        errs = [rel_to_max(to64(a), b) for a, b in ((dq, rdq), (dk, rdk), (dv, rdv))]
    print(f"{family}: visited {stats.visited}/{stats.total} errs {errs}")
    assert max(errs) < TOL


def test_autograd_op_with_rem():
    """stickbreaking_attention: o and rem differentiable; rem's grad is the row_offset."""
    import paper_2410_17980_b200 as sb
    q, k, v, w = make_qkv(2, 2, 256, 64, seed=4)
    u = torch.randn(2, 2, 256, generator=torch.Generator().manual_seed(8)).cuda()
    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
    o, rem = sb.stickbreaking_attention(qq, kk, vv, return_rem=True)
    loss = (o.float() * w.float()).sum() + (rem * u).sum()
    loss.backward()
    ref = oracle_fwd(q, k, v)
    assert max_rel_err(rem.detach().cpu().double().numpy(), np.exp(ref["log_rem"])) < TOL
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, w, ref, row_offset=u)
    errs = [rel_to_max(to64(a.grad), b) for a, b in ((qq, rdq), (kk, rdk), (vv, rdv))]
    print("autograd:", errs)
    assert max(errs) < TOL


def test_backward_deterministic():
    """test_acceptance.py:252-269: bit-identical reruns (no atomics)."""
    q, k, v, d_o = make_qkv(2, 2, 512, 128, seed=13)
    a = _run(q, k, v, d_o)
    b = _run(q, k, v, d_o)
    for x, y in zip(a[3:], b[3:]):
        assert torch.equal(x, y)


def test_zero_upstream():
    """test_blocked.py:152-157: zero dO gives zero gradients."""
    q, k, v, _ = make_qkv(1, 1, 200, 64, seed=2)
    _, _, _, dq, dk, dv = _run(q, k, v, torch.zeros_like(q))
    for g in (dq, dk, dv):
        assert torch.count_nonzero(g) == 0
