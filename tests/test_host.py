"""Host-side mirror of the reference interface (no GPU): plan_blocks & co.

Mirrors /root/reference/pkg/tests/test_blocked.py:44-62 for the restated
BlockLayout / plan_blocks, plus the (b, h) sharding helper of dist.py.
"""

import pytest

import paper_2410_17980_b200 as sb
from paper_2410_17980_b200 import ops
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


def _cache(shape, cu=None):
    import torch
    q = torch.zeros(*shape, dtype=torch.bfloat16)
    if cu is None:
        lay = ops.plan_blocks(shape[2])
        return ops.BlockedCache(q, q, q, 0.125, lay, None, None, None, False, 1e-6)
    cu_host = torch.tensor(cu, dtype=torch.int32)
    return ops.BlockedCache(q, q, q, 0.125, None, None, None, None, False, 1e-6,
                            cu_seqlens=cu_host, max_seqlen=int((cu_host[1:] - cu_host[:-1]).max()),
                            cu_host=cu_host)


def test_backward_chunks_cover_units_under_the_cap():
    """_unit_chunks (the workspace-capped backward's plan): contiguous ranges covering the
    axis (batch entries, heads when B == 1, sequences for varlen), each within the cap
    unless it is a single unit, fewest chunks (greedy maximal prefixes)."""
    import ctypes
    lib = ops._lib.load()
    for shape in ((3, 2, 700, 64), (1, 5, 700, 128), (4, 1, 4096, 128)):
        c = _cache(shape)
        whole = ops.workspace_bytes(c)
        axis = shape[0] if shape[0] > 1 else shape[1]
        one = whole // axis
        for cap in (whole, whole - 1, 2 * one + one // 2, one, 1):
            ch = list(ops._unit_chunks(c, True, cap))
            assert ch[0][0] == 0 and ch[-1][1] == axis
            assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
            for lo, hi in ch:
                p = ops._chunk_params(c, lo, hi)
                need = lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 1)
                assert need <= cap or hi - lo == 1
            if cap >= whole:
                assert ch == [(0, axis)]
    lens = [300, 0, 700, 129, 64]
    cu = [0] + list(__import__("itertools").accumulate(lens))
    c = _cache((cu[-1], 2, 64), cu)
    whole = ops.workspace_bytes(c)
    ch = list(ops._unit_chunks(c, True, whole // 3))
    assert len(ch) > 1 and ch[0][0] == 0 and ch[-1][1] == len(lens)
