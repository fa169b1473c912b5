"""GPU checks of the host API around the kernels: input layouts the op must accept
(fused-QKV slices), the snapshot-free inference forward (the reference's
blocked_forward(two_phase=False), blocked.py:136, :163, :188), the N-free store-mode
backward and the workspace validation."""

import numpy as np
import pytest
import torch

from tests.gpu_util import make_qkv, oracle_fwd, rel_to_max, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("varlen", [False, True])
def test_fused_qkv_slices(varlen):
    """a slice of a fused QKV tensor is strided but not dense; the op
    must give the same results as on contiguous copies (and write nothing outside o)."""
    import paper_2410_17980_b200 as sb
    g = torch.Generator().manual_seed(3)
    B, L, H, d = 2, 200, 3, 64
    if varlen:
        qkv = torch.randn(B * L, 3, H, d, generator=g).to(torch.bfloat16).cuda()
        parts = [qkv[:, i] for i in range(3)]  # (T, H, d), token stride 3*H*d
        cu = torch.tensor([0, 70, B * L], dtype=torch.int32).cuda()
        kw = dict(cu_seqlens=cu)
    else:
        qkv = torch.randn(B, L, 3, H, d, generator=g).to(torch.bfloat16).cuda()
        parts = [qkv[:, :, i].transpose(1, 2) for i in range(3)]  # (B, H, L, d) views
        kw = {}
    guard = qkv.clone()
    ps = [p.detach().clone().requires_grad_(True) for p in parts]
    cs = [p.detach().contiguous().requires_grad_(True) for p in parts]
    w = torch.randn(parts[0].shape, generator=g).to(torch.bfloat16).cuda()
    o1 = sb.stickbreaking_attention(*ps, **kw)
    o1.backward(w)
    o2 = sb.stickbreaking_attention(*cs, **kw)
    o2.backward(w)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    for a, b in zip(ps, cs):
        assert torch.equal(a.grad, b.grad)
    assert torch.equal(qkv, guard)  # inputs untouched


@pytest.mark.parametrize("skip,family", [(False, "random"), (True, "shift"), (True, "random")])
def test_two_phase_false_same_results_no_snapshots(skip, family):
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(2, 4, 1000, 128, seed=5, family=family, mu=-6.0, with_do=False)
    a = sb.blocked_forward(q, k, v, skip=skip)
    b = sb.blocked_forward(q, k, v, skip=skip, two_phase=False)
    torch.cuda.synchronize()
    assert b[3].state is None and a[3].state.numel() == 64 + 2 * q.numel() // q.shape[-1]
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert torch.equal(a[2].first_kb, b[2].first_kb) and a[2].visited == b[2].visited
    with pytest.raises(ValueError):  # blocked.py:315-316
        sb.blocked_backward_twophase(b[3], torch.zeros_like(q))


def test_inference_forward_allocates_no_snapshots():
    """stickbreaking_attention without autograd writes no state and no M: its peak
    memory stays below the M array's size over the outputs."""
    import paper_2410_17980_b200 as sb
    B, H, L, d = 1, 8, 16384, 128
    q, k, v = make_qkv(B, H, L, d, seed=1, with_do=False)
    m_bytes = B * H * (L // 64) * (L // 64 + 1) // 2 * 64 * 4  # 67 MB (o: 34 MB)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    with torch.no_grad():
        o, rem = sb.stickbreaking_attention(q, k, v, return_rem=True)
    torch.cuda.synchronize()
    extra = torch.cuda.max_memory_allocated() - base
    assert extra < o.numel() * 2 + 3 * rem.numel() * 4 + (1 << 20) < m_bytes
    qq = q.clone().requires_grad_(True)
    o2, rem2 = sb.stickbreaking_attention(qq, k, v, return_rem=True)
    assert torch.equal(o, o2) and torch.equal(rem, rem2)


def test_training_forward_keeps_only_O_L_state():
    """With autograd the forward keeps the final a per row (float64) and first_kb, no
    snapshot per tile: the memory held between forward and backward over q, k, v, o
    is O(L) (north_star: cut the O(L^2/d_block) M/N intermediates)."""
    import paper_2410_17980_b200 as sb
    B, H, L, d = 1, 8, 16384, 128
    q, k, v = make_qkv(B, H, L, d, seed=1, with_do=False)
    m_bytes = B * H * (L // 64) * (L // 64 + 1) // 2 * 64 * 4  # 67 MB
    qq = q.clone().requires_grad_(True)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    o = sb.stickbreaking_attention(qq, k, v)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - base - o.numel() * 2
    rows = B * H * L
    assert held <= rows * (8 + 4) + B * H * (L // 64) * 4 + 4096 < m_bytes // 10


def test_workspace_modes_match_oracle():
    """Store mode (dZ tiles) and recompute mode (N snapshots) through a caller-owned
    workspace: same gradients bit for bit, oracle parity, short workspace refused."""
    import paper_2410_17980_b200 as sb
    from tests.gpu_util import oracle_bwd
    q, k, v, d_o = make_qkv(1, 2, 640, 128, seed=8)
    o, lr, st, cache = sb.blocked_forward(q, k, v)
    need = sb.ops.workspace_bytes(cache, store=True)
    ws = torch.empty(need, device="cuda", dtype=torch.uint8)
    dq, dk, dv, _ = sb.blocked_backward_twophase(cache, d_o, workspace=ws)
    torch.cuda.synchronize()
    ref = oracle_fwd(q, k, v)
    rdq, rdk, rdv, _ = oracle_bwd(q, k, v, d_o, ref)
    assert max(rel_to_max(to64(a), b) for a, b in ((dq, rdq), (dk, rdk), (dv, rdv))) < TOL
    r = sb.blocked_backward_twophase(cache, d_o, store_tiles=False)
    for a, b in zip((dq, dk, dv), r[:3]):
        assert torch.equal(a, b)
    with pytest.raises(ValueError):  # short workspace (varlen too) is refused
        sb.blocked_backward_twophase(cache, d_o, workspace=ws[: need // 2])


def test_chunked_backward_bit_identical(monkeypatch):
    """A workspace cap below one call's need splits the units into chunks (batch
    entries, heads when B == 1, whole sequences for varlen): same gradients bit for bit."""
    import paper_2410_17980_b200 as sb
    for shape in ((3, 2, 700, 64), (1, 5, 700, 128)):
        q, k, v, d_o = make_qkv(*shape, seed=3)
        _, _, _, cache = sb.blocked_forward(q, k, v)
        full = sb.blocked_backward_twophase(cache, d_o)
        one = sb.ops.workspace_bytes(cache) // (shape[0] * shape[1])
        monkeypatch.setattr(sb.ops, "WORKSPACE_MAX_BYTES", 2 * one + one // 2)
        assert len(list(sb.ops._unit_chunks(cache, True, sb.ops.workspace_cap_bytes()))) > 1
        part = sb.blocked_backward_twophase(cache, d_o)
        monkeypatch.undo()
        torch.cuda.synchronize()
        for a, b in zip(full[:3], part[:3]):
            assert torch.equal(a, b)
    g = torch.Generator().manual_seed(2)
    lens = [300, 0, 700, 129, 64]
    q, k, v, d_o = (torch.randn(sum(lens), 2, 64, generator=g).to(torch.bfloat16).cuda()
                    for _ in range(4))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32).cuda()
    _, _, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu)
    ro = torch.randn(sum(lens), 2, generator=g).cuda()
    full = sb.blocked_backward_twophase(cache, d_o, row_offset=ro)
    monkeypatch.setattr(sb.ops, "WORKSPACE_MAX_BYTES", sb.ops.workspace_bytes(cache) // 3)
    assert len(list(sb.ops._unit_chunks(cache, True, sb.ops.workspace_cap_bytes()))) > 1
    part = sb.blocked_backward_twophase(cache, d_o, row_offset=ro)
    torch.cuda.synchronize()
    for a, b in zip(full[:3], part[:3]):
        assert torch.equal(a, b)


def test_varlen_short_workspace_rejected():
    import paper_2410_17980_b200 as sb
    g = torch.Generator().manual_seed(2)
    lens = [300, 700]
    q, k, v, d_o = (torch.randn(sum(lens), 2, 64, generator=g).to(torch.bfloat16).cuda()
                    for _ in range(4))
    cu = torch.tensor([0, 300, 1000], dtype=torch.int32).cuda()
    _, _, _, cache = sb.blocked_forward(q, k, v, cu_seqlens=cu)
    need = sb.ops.workspace_bytes(cache)
    with pytest.raises(ValueError):
        sb.blocked_backward_twophase(cache, d_o, workspace=torch.empty(
            need - 16384, device="cuda", dtype=torch.uint8))
    dq, dk, dv, _ = sb.blocked_backward_twophase(
        cache, d_o, workspace=torch.empty(need, device="cuda", dtype=torch.uint8))
    r = sb.blocked_backward_twophase(cache, d_o, store_tiles=False)
    torch.cuda.synchronize()
    for a, b in zip((dq, dk, dv), r[:3]):
        assert torch.equal(a, b)


def test_rem_gradient_only_when_requested():
    """return_rem=False returns o alone (no exp launch); with it, rem's gradient is the
    reference's row_offset hook, and a loss on rem alone still backpropagates."""
    import paper_2410_17980_b200 as sb
    q, k, v = make_qkv(1, 2, 256, 64, seed=4, with_do=False)
    qq = q.clone().requires_grad_(True)
    o = sb.stickbreaking_attention(qq, k, v)
    assert isinstance(o, torch.Tensor)
    qq2 = q.clone().requires_grad_(True)
    _, rem = sb.stickbreaking_attention(qq2, k, v, return_rem=True)
    rem.sum().backward()  # d_o is None: materialize_grads is off
    assert qq2.grad is not None and torch.isfinite(qq2.grad.float()).all()
    ref = oracle_fwd(q, k, v)
    np.testing.assert_allclose(rem.detach().cpu().double().numpy(), np.exp(ref["log_rem"]),
                               atol=TOL, rtol=TOL)


@pytest.mark.parametrize("d", [64, 128])
def test_cuda_graph_capture_fwd_bwd(d):
    """The op (forward + two-phase backward through autograd) captures into one CUDA
    graph: no host synchronisation or allocation outside torch's graph pool on the
    path; replays give the eager results bit for bit, also on new inputs copied into
    the static buffers (launch-bound small shapes can replay a whole step)."""
    import paper_2410_17980_b200 as sb
    B, H, L = 2, 4, 384
    q, k, v, do = make_qkv(B, H, L, d, seed=5)

    def eager(q, k, v, do):
        qq, kk, vv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
        o = sb.stickbreaking_attention(qq, kk, vv)
        o.backward(do)
        return [o.detach(), qq.grad, kk.grad, vv.grad]

    sq, sk, sv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
    sdo = do.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (kernel attributes, allocator) off the capture
        for _ in range(2):
            sb.stickbreaking_attention(sq, sk, sv).backward(sdo)
            for x in (sq, sk, sv):
                x.grad = None
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        so = sb.stickbreaking_attention(sq, sk, sv)
        so.backward(sdo)
    for seed in (5, 6):
        q2, k2, v2, do2 = make_qkv(B, H, L, d, seed=seed)
        with torch.no_grad():
            for dst, src in zip((sq, sk, sv, sdo), (q2, k2, v2, do2)):
                dst.copy_(src)
        g.replay()
        torch.cuda.synchronize()
        ref = eager(q2, k2, v2, do2)
        for a, b in zip([so.detach(), sq.grad, sk.grad, sv.grad], ref):
            assert torch.equal(a, b)
