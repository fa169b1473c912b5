"""Host-side mirror of the reference interface (no GPU): plan_blocks & co.

Mirrors /root/reference/pkg/tests/test_blocked.py:44-62 for the restated
BlockLayout / plan_blocks, plus the (b, h) sharding helper of dist.py.
"""

import pytest

import paper_2410_17980_b200 as sb
from paper_2410_17980_b200 import dist


def test_plan_two_blocks():
    lay = sb.plan_blocks(128, 64)
    assert lay.n_blocks == 2 and lay.tail == 0 and lay.n_tiles == 3


def test_plan_tail():
    lay = sb.plan_blocks(100, 64)
    assert lay.n_blocks == 2 and lay.tail == 36 and lay.span(1) == (64, 100)


def test_plan_single_block():
    lay = sb.plan_blocks(64, 64)
    assert lay.n_blocks == 1 and lay.n_tiles == 1


def test_plan_rejects_zero():
    with pytest.raises(ValueError):
        sb.plan_blocks(0, 64)
    with pytest.raises(ValueError):
        sb.plan_blocks(16, 0)


def test_skip_stats_and_default_eps():
    import torch
    st = sb.TileStats(total=10, visited=7, skipped=3, first_kb=None)
    assert sb.skip_stats(st) == (7, 3, 0.3)
    assert sb.default_skip_eps(torch.bfloat16) == 1e-6
    assert sb.default_skip_eps(torch.float64) == 1e-12


@pytest.mark.parametrize("n,world", [(128, 1), (128, 2), (128, 8), (7, 3), (5, 8)])
def test_unit_ranges_partition(n, world):
    seen = []
    for r in range(world):
        lo, hi = dist.unit_range(n, r, world)
        seen.extend(range(lo, hi))
        assert hi - lo in (n // world, n // world + 1)
    assert seen == list(range(n))


def test_dense_layout_check():
    """a fused-QKV slice is strided but not dense; it must be copied."""
    import torch
    from paper_2410_17980_b200.ops import _dense, _same_layout
    x = torch.zeros(2, 5, 3, 4, 64)  # (B, L, 3, H, d)
    assert _dense(x) and _dense(x.transpose(1, 3))
    q = x[:, :, 0].transpose(1, 2)  # (B, H, L, d) view with stride 3*H*d over L
    assert not _dense(q)
    assert _same_layout(q, q, q)[0].is_contiguous()
    blhd = torch.zeros(2, 5, 4, 64).transpose(1, 2)
    assert _dense(blhd) and _same_layout(blhd, blhd, blhd)[0].stride() == blhd.stride()
    assert _dense(torch.zeros(1, 1, 7, 64)[:, :, :, :])
