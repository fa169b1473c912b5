"""Host-side mirror of the reference's tiled operator, over the C-ABI CUDA library.

Reference surface (/root/reference/pkg/src/sbattn/blocked.py) and its
counterparts here:

=================================  ==========================================
reference                          this module
=================================  ==========================================
``plan_blocks`` / ``BlockLayout``  ``plan_blocks`` / ``BlockLayout`` (:46-67)
``TileStats`` / ``skip_stats``     ``TileStats`` / ``skip_stats`` (:82-103)
``default_skip_eps``               ``default_skip_eps`` (bf16 -> 1e-6, :106-107)
``blocked_forward(two_phase)``     ``blocked_forward`` -> (o, log_rem, stats, cache)
``blocked_backward_twophase``      ``blocked_backward_twophase(cache, d_o, row_offset)``
``sb_forward_blocked``             ``sb_forward_blocked``
(paper's upstream operator)        ``stickbreaking_attention(q, k, v, ...)`` autograd op
=================================  ==========================================

Tensors are CUDA bf16 of shape (B, H, L, d) (any strides with a contiguous last
dim; q, k, v share one layout).  Unlike the reference (one L x d head per call)
every call covers all (batch, head) units at once.  Packed variable-length
batches pass (total_tokens, H, d) tensors with
``cu_seqlens`` (int32 [n_seq+1] offsets): every sequence is planned and run as
an independent problem, exactly as the reference runs each sequence separately.
Errors the reference raises as ValueError are raised as ValueError here.  There
is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib

DEFAULT_BLOCK = 64
SCHED_HEADER = 64  # floats at the start of the state / snapshot arrays (work-queue counters)
# The backward's workspace (M snapshots + the store mode's dZ tiles: phase 1 writes them,
# phase 2 reads them instead of recomputing dO.V^T and dZ; bit-identical results) is bounded
# by this many bytes per call: a larger problem runs in chunks of whole (b, h) units (C2:
# 2.2 GB and C4 4.2 GB in one call; C3 at L=32768 would need 34 GB and runs in 5 chunks).
WORKSPACE_MAX_BYTES = int(float(os.environ.get("SB_WORKSPACE_MAX_GB", "8")) * 2**30)
SKIP_EPS_BF16 = 1e-6  # the reference's f32 default (blocked.py:43) is used for bf16


@dataclass(frozen=True)
class BlockLayout:
    """blocked.py:46-60 restated."""

    seq_len: int
    block: int
    n_blocks: int
    tail: int

    def span(self, b: int) -> tuple[int, int]:
        lo = b * self.block
        return lo, min(lo + self.block, self.seq_len)

    @property
    def n_tiles(self) -> int:
        return self.n_blocks * (self.n_blocks + 1) // 2


def plan_blocks(seq_len: int, d_block: int = DEFAULT_BLOCK) -> BlockLayout:
    """blocked.py:63-67 restated (ValueError on seq_len < 1 or d_block < 1)."""
    if seq_len < 1 or d_block < 1:
        raise ValueError("seq_len and d_block must be >= 1")
    n_blocks = -(-seq_len // d_block)
    return BlockLayout(seq_len, d_block, n_blocks, seq_len % d_block)


@dataclass
class TileStats:
    """blocked.py:82-88; totals are over all (batch, head) units of the call."""

    total: int
    visited: int
    skipped: int
    first_kb: torch.Tensor  # (B, H, n_blocks) int32, leftmost visited key block


def skip_stats(stats: TileStats) -> tuple[int, int, float]:
    """blocked.py:101-103."""
    return stats.visited, stats.skipped, stats.skipped / stats.total


def default_skip_eps(dtype) -> float:
    """blocked.py:106-107: f64 -> 1e-12, otherwise the f32 default 1e-6."""
    return 1e-12 if dtype == torch.float64 else SKIP_EPS_BF16


@dataclass
class BlockedCache:
    """blocked.py:90-98 analogue: what the two-phase backward needs."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    scale: float
    layout: BlockLayout
    log_rem: torch.Tensor
    first_kb: torch.Tensor
    state: torch.Tensor | None  # the forward's O(L) state (final a per row, float64), or None
    skip: bool
    skip_eps: float
    cu_seqlens: torch.Tensor | None = None  # varlen: device int32 [n_seq+1]
    max_seqlen: int = 0
    cu_host: torch.Tensor | None = None     # varlen: host copy of cu_seqlens


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(t):
    """The current stream of t's device (not of the current device)."""
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _on(t):
    """Run a C-ABI call with t's device current: the library sizes grids, sets kernel
    attributes and launches on the current device, which must own the stream."""
    return torch.cuda.device(t.device)


def _check_qkv(q, k, v, varlen=False):
    if not (q.shape == k.shape == v.shape):
        raise ValueError("q, k, v must share one shape")  # blocked.py:116-117
    if varlen and q.dim() != 3:
        raise ValueError("varlen q, k, v must be (total_tokens, heads, head_dim)")
    if not varlen and q.dim() != 4:
        raise ValueError("q, k, v must be (batch, heads, seq_len, head_dim)")
    for t in (q, k, v):
        if not t.is_cuda:
            raise RuntimeError("stickbreaking_attention: CUDA tensors required (no CPU fallback)")
        if t.dtype != torch.bfloat16:
            raise TypeError("stickbreaking_attention: bf16 tensors required")
    if q.shape[-1] not in (64, 128):
        raise ValueError(f"head_dim {q.shape[-1]} unsupported (64 or 128)")


def _dense(t) -> bool:
    """Non-overlapping and dense: some order of the dims has contiguous strides
    (a BLHD view of BHLD storage, or the reverse), so empty_like(t) keeps t's
    strides and outputs allocated that way are addressed exactly like t."""
    expected = 1
    for i in sorted(range(t.dim()), key=lambda i: (t.stride(i), t.size(i))):
        if t.size(i) == 1:
            continue
        if t.stride(i) != expected:
            return False
        expected *= t.size(i)
    return True


def _same_layout(*ts):
    """q, k, v (and the outputs, allocated like q) must share one strided layout.
    q is made contiguous unless it is dense with a contiguous last dim and 16-byte
    aligned: a fused-QKV slice (qkv[:, :, 0] of a (B, L, 3, H, d) tensor) is
    strided but not dense, and outputs allocated like it would be addressed past
    their storage."""
    base = ts[0]
    if base.stride(-1) != 1 or base.data_ptr() % 16 or not _dense(base):
        base = base.contiguous()
    out = [base]
    for t in ts[1:]:
        out.append(t if (t.stride() == base.stride() and t.data_ptr() % 16 == 0)
                   else t.contiguous() if base.is_contiguous() else
                   torch.empty_like(base).copy_(t))
    return out


def _params(q, scale, skip, skip_eps, block=DEFAULT_BLOCK, cu_seqlens=None,
            max_seqlen=0) -> _lib.SbParams:
    p = _lib.SbParams()
    if cu_seqlens is None:
        B, H, L, d = q.shape
        sb, sh, sl, sd = q.stride()
        p.batch, p.heads, p.seqlen, p.head_dim = B, H, L, d
        p.stride_b, p.stride_h, p.stride_l = sb, sh, sl
        p.cu_seqlens = None
        p.total_tokens = 0
    else:
        T, H, d = q.shape
        sl, sh, sd = q.stride()
        p.batch, p.heads, p.seqlen, p.head_dim = cu_seqlens.numel() - 1, H, max(1, max_seqlen), d
        p.stride_b, p.stride_h, p.stride_l = 0, sh, sl
        p.cu_seqlens = ctypes.c_void_p(cu_seqlens.data_ptr())
        p.total_tokens = T
    p.scale = float(scale)
    p.block = block
    p.skip = int(bool(skip))
    p.skip_eps = float(skip_eps)
    return p


def _varlen_plan(cu_seqlens, q):
    """(host offsets, device offsets, lengths, max_seqlen).

    The sizes of M, first_kb and the dZ workspace depend on every sequence
    length, so the plan needs the offsets on the host: a CPU cu_seqlens is used
    as is and uploaded without a stream sync (pinned staging copy); a device
    cu_seqlens costs one small D2H read (which waits for the stream)."""
    if cu_seqlens.dtype != torch.int32 or cu_seqlens.dim() != 1 or cu_seqlens.numel() < 2:
        raise ValueError("cu_seqlens must be a 1-D int32 tensor of n_seq+1 offsets")
    if cu_seqlens.device.type == "cpu":
        host = cu_seqlens.contiguous()
        dev = host.pin_memory().to(q.device, non_blocking=True)
    else:
        host = cu_seqlens.cpu()
        dev = cu_seqlens.to(device=q.device).contiguous()
    lens = (host[1:] - host[:-1]).tolist()
    if int(host[0]) != 0 or min(lens) < 0 or int(host[-1]) != q.shape[0]:
        raise ValueError("cu_seqlens must start at 0, be non-decreasing and end at total_tokens")
    return host, dev, lens, max(lens)


def _blocked_forward_varlen(q, k, v, cu_seqlens, skip, skip_eps, scale, counters,
                            two_phase=True):
    _check_qkv(q, k, v, varlen=True)
    T, H, d = q.shape
    host, cu, lens, max_L = _varlen_plan(cu_seqlens, q)
    if skip_eps is None:
        skip_eps = default_skip_eps(q.dtype)
    if not 0.0 < skip_eps < 1.0:
        raise ValueError("skip_eps must be in (0, 1)")  # blocked.py:155-156
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    q, k, v = _same_layout(q, k, v)
    lib = _lib.load()
    p = _params(q, scale, skip, skip_eps, cu_seqlens=cu, max_seqlen=max_L)
    n_snap, n_fkb = ctypes.c_size_t(), ctypes.c_size_t()
    host_c = host.to(torch.int32).contiguous()
    _lib.check(lib.sb_varlen_elems(ctypes.byref(p), ctypes.c_void_p(host_c.data_ptr()),
                                   ctypes.byref(n_snap), ctypes.byref(n_fkb)))
    o = torch.empty_like(q)
    log_rem = torch.empty((T, H), device=q.device, dtype=torch.float32)
    first_kb = torch.empty(max(1, n_fkb.value), device=q.device, dtype=torch.int32)
    state = _state_tensor(lib, p, q.device) if two_phase else None
    cnt = torch.zeros(2, device=q.device, dtype=torch.int64) if counters else None
    if max_L > 0:
        with _on(q):
            _lib.check(lib.sb_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                  _ptr(log_rem), _ptr(first_kb), _ptr(state), _ptr(cnt),
                                  _stream(q)))
    else:
        o.zero_()
        log_rem.zero_()
    total = (n_snap.value - SCHED_HEADER) // DEFAULT_BLOCK
    visited = int(cnt[0].item()) if counters else -1
    stats = TileStats(total, visited, total - visited if counters else -1, first_kb)
    cache = BlockedCache(q, k, v, scale, None, log_rem, first_kb, state, skip, skip_eps,
                         cu_seqlens=cu, max_seqlen=max_L, cu_host=host_c)
    return o, log_rem, stats, cache


def blocked_forward(q, k, v, layout: BlockLayout | None = None, skip: bool = False,
                    skip_eps: float | None = None, scale: float | None = None,
                    counters: bool = True, cu_seqlens: torch.Tensor | None = None,
                    two_phase: bool = True):
    """blocked_forward over every (b, h) unit (blocked.py:129-206).

    Returns (o, log_rem, TileStats, BlockedCache).  log_rem is the reference's
    RowLogAccumulator.a (natural log of the remaining stick mass).

    No call keeps M snapshots (blocked.py:188-189): with two_phase=True the forward
    keeps only the final a per row (float64, cache.state, O(L)); the backward's
    phase 1 rolls the per-tile snapshots back from it.  two_phase=False
    (blocked.py:136, :163, :188) keeps not even that (o, log_rem and first_kb are
    the same bit for bit): a forward for inference, after which the two-phase
    backward raises ValueError.  (The reference's fused backward does not exist
    here: SURVEY.md §8(a).)

    Varlen: q, k, v (total_tokens, H, d) with cu_seqlens (int32 [n_seq+1]);
    log_rem is then (total_tokens, H), first_kb a flat array packed sequence by
    sequence (head-major within a sequence), layout must be None.
    """
    if cu_seqlens is not None:
        if layout is not None:
            raise ValueError("varlen batches are planned per sequence; pass layout=None")
        return _blocked_forward_varlen(q, k, v, cu_seqlens, skip, skip_eps, scale, counters,
                                       two_phase)
    _check_qkv(q, k, v)
    B, H, L, d = q.shape
    if layout is None:
        layout = plan_blocks(L)
    if layout.seq_len != L:
        raise ValueError(f"layout is for L={layout.seq_len}, inputs have L={L}")  # :118-119
    if layout.block != DEFAULT_BLOCK:
        raise ValueError("the CUDA path runs d_block = 64 (blocked.py:41)")
    if skip_eps is None:
        skip_eps = default_skip_eps(q.dtype)
    if not 0.0 < skip_eps < 1.0:
        raise ValueError("skip_eps must be in (0, 1)")  # blocked.py:155-156
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    q, k, v = _same_layout(q, k, v)
    lib = _lib.load()
    p = _params(q, scale, skip, skip_eps)
    o = torch.empty_like(q)
    log_rem = torch.empty((B, H, L), device=q.device, dtype=torch.float32)
    first_kb = torch.empty((B, H, layout.n_blocks), device=q.device, dtype=torch.int32)
    state = _state_tensor(lib, p, q.device) if two_phase else None
    cnt = torch.zeros(2, device=q.device, dtype=torch.int64) if counters else None
    with _on(q):
        _lib.check(lib.sb_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(log_rem),
                              _ptr(first_kb), _ptr(state), _ptr(cnt), _stream(q)))
    total = B * H * layout.n_tiles
    visited = int(cnt[0].item()) if counters else -1
    stats = TileStats(total, visited, total - visited if counters else -1, first_kb)
    cache = BlockedCache(q, k, v, scale, layout, log_rem, first_kb, state, skip, skip_eps)
    return o, log_rem, stats, cache


def sb_forward_blocked(q, k, v, layout=None, **kw):
    """blocked.py:218-226: (o, cache) convenience wrapper."""
    o, _, _, cache = blocked_forward(q, k, v, layout, **kw)
    return o, cache


def _state_tensor(lib, p, device):
    """The forward's state array (sb_state_elems floats; the final a of every row as
    float64 after a 64-float header)."""
    return torch.empty(lib.sb_state_elems(ctypes.byref(p)), device=device, dtype=torch.float32)


def _cache_params(cache: BlockedCache):
    return _params(cache.q, cache.scale, cache.skip, cache.skip_eps,
                   cu_seqlens=cache.cu_seqlens, max_seqlen=cache.max_seqlen)


def workspace_bytes(cache: BlockedCache, store: bool = True) -> int:
    """Bytes of the backward's workspace for this cache in one call: the M snapshots
    (phase 1 -> phase 2) plus the dZ tiles (store mode) or the N snapshots."""
    lib = _lib.load()
    p = _cache_params(cache)
    host = None if cache.cu_host is None else ctypes.c_void_p(cache.cu_host.data_ptr())
    return int(lib.sb_bwd_workspace_bytes(ctypes.byref(p), host, int(bool(store))))


def workspace_cap_bytes(device=None) -> int:
    """Largest backward workspace one call allocates: the SB_WORKSPACE_MAX_GB cap
    (default 8 GiB) and at most 1/16 of the device memory.  A larger problem runs in
    chunks of whole (b, h) units.  (No free-memory query: cudaMemGetInfo waits for the
    device, ~10 ms per backward call on a busy GPU.)"""
    cap = WORKSPACE_MAX_BYTES
    try:
        cap = min(cap, _device_total_bytes(torch.device("cuda", torch.cuda.current_device())
                                           if device is None else torch.device(device)) // 16)
    except Exception:  # pragma: no cover - no device query possible
        pass
    return cap


_TOTAL = {}


def _device_total_bytes(device) -> int:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _TOTAL:
        _TOTAL[idx] = torch.cuda.get_device_properties(idx).total_memory
    return _TOTAL[idx]


def _unit_chunks(cache: BlockedCache, store: bool, cap: int):
    """Split the call's (b, h) units into the fewest contiguous chunks whose workspace
    fits `cap` (whole batch entries when B > 1, heads when B == 1, whole sequences
    for varlen).  Yields (lo, hi) index ranges over that axis; one range covering
    everything when the whole call fits (or when nothing smaller would)."""
    lib = _lib.load()
    q = cache.q
    if cache.cu_seqlens is not None:
        n = cache.cu_host.numel() - 1
        axis_len = n
    else:
        B, H = q.shape[0], q.shape[1]
        n = B if B > 1 else H
        axis_len = n

    def cost(lo, hi):
        p = _chunk_params(cache, lo, hi)
        host = None
        if cache.cu_seqlens is not None:
            host = (cache.cu_host[lo:hi + 1] - cache.cu_host[lo]).to(torch.int32).contiguous()
            return int(lib.sb_bwd_workspace_bytes(ctypes.byref(p), ctypes.c_void_p(host.data_ptr()),
                                                  int(store)))
        return int(lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, int(store)))

    if cost(0, axis_len) <= cap:
        yield 0, axis_len
        return
    lo = 0
    while lo < axis_len:
        hi = lo + 1
        while hi < axis_len and cost(lo, hi + 1) <= cap:
            hi += 1
        yield lo, hi
        lo = hi


def _chunk_params(cache: BlockedCache, lo: int, hi: int):
    """Params of the chunk [lo, hi) of _unit_chunks' axis (device cu_seqlens of a varlen
    chunk are set by the caller)."""
    q = cache.q
    if cache.cu_seqlens is not None:
        t0, t1 = int(cache.cu_host[lo]), int(cache.cu_host[hi])
        lens = (cache.cu_host[lo + 1:hi + 1] - cache.cu_host[lo:hi]).tolist()
        p = _params(q[t0:t1] if t1 > t0 else q[:1], cache.scale, cache.skip, cache.skip_eps,
                    cu_seqlens=cache.cu_seqlens, max_seqlen=max(lens) if lens else 0)
        p.batch = hi - lo
        p.total_tokens = max(1, t1 - t0)
        return p
    view = q[lo:hi] if q.shape[0] > 1 else q[:, lo:hi]
    return _params(view, cache.scale, cache.skip, cache.skip_eps)


def blocked_backward_twophase(cache: BlockedCache, d_o, layout: BlockLayout | None = None,
                              row_offset=None, *, out=None, phases: int = 3,
                              store_tiles: bool | None = None, workspace=None):
    """blocked_backward_twophase (blocked.py:299-392) over every (b, h) unit.

    Returns (d_q, d_k, d_v, n_stored_tiles).  row_offset (B, H, L) float32 is
    subtracted from dO.V^T per query row (blocked.py:241-242).

    store_tiles: store mode (phase 2 reads phase 1's dZ tiles) unless False
    (recompute mode: no tiles, phase 2 recomputes dO.V^T and dZ; same results bit for
    bit).  The workspace (M snapshots + dZ tiles or N) is transient: allocated here,
    at most workspace_cap_bytes() per call, the units running in chunks beyond that.
    `workspace` passes a preallocated one (uint8 CUDA tensor of at least
    workspace_bytes(cache, store) bytes, no chunking); callers running the phases one
    by one (phases=1 then 2) must pass the same one to both.  `out` = (dq, dk, dv)
    preallocated like q.
    """
    if layout is not None and layout != cache.layout:
        raise ValueError("layout does not match the one the cache was built with")  # :398-399
    if cache.state is None:
        raise ValueError("two-phase backward needs a forward run with two_phase=True "
                         "(its state is missing)")  # blocked.py:315-316
    q, k, v = cache.q, cache.k, cache.v
    if d_o.shape != v.shape:
        raise ValueError("d_o shape mismatch")
    if d_o.dtype != torch.bfloat16 or not d_o.is_cuda:
        raise TypeError("d_o must be a CUDA bf16 tensor")
    if d_o.stride() != q.stride() or d_o.data_ptr() % 16:
        d_o = torch.empty_like(q).copy_(d_o)
    lib = _lib.load()
    ro = None
    if row_offset is not None:
        ro = row_offset.to(device=q.device, dtype=torch.float32).contiguous()
        if ro.shape != cache.log_rem.shape:
            raise ValueError("row_offset must match log_rem: (batch, heads, seq_len), or "
                             "(total_tokens, heads) for varlen")
    dq, dk, dv = out if out is not None else (torch.empty_like(q) for _ in range(3))
    varlen = cache.cu_seqlens is not None
    n_stored = (cache.layout.n_tiles * q.shape[0] * q.shape[1] if not varlen else
                _varlen_tiles(cache))
    if varlen and cache.max_seqlen == 0:
        for t in (dq, dk, dv):
            t.zero_()
        return dq, dk, dv, 0
    store = True if store_tiles is None else bool(store_tiles)
    if workspace is not None:
        need = workspace_bytes(cache, store)
        if workspace.numel() < need:
            raise ValueError(f"workspace has {workspace.numel()} bytes, the backward needs {need}")
        chunks = [None]
    else:
        if phases != 3:
            raise ValueError("running the phases one by one needs a caller-owned workspace")
        chunks = list(_unit_chunks(cache, store, workspace_cap_bytes(q.device)))
        if len(chunks) == 1:
            chunks = [None]
        # one allocation for every chunk
        workspace = torch.empty(max(_chunk_bytes(lib, cache, store, c) for c in chunks),
                                device=q.device, dtype=torch.uint8)
    for ch in chunks:
        _backward_call(lib, cache, d_o, ro, dq, dk, dv, store, phases, ch, workspace)
    return dq, dk, dv, n_stored


def _chunk_bytes(lib, cache, store, chunk):
    if chunk is None:
        return workspace_bytes(cache, store)
    lo, hi = chunk
    p = _chunk_params(cache, lo, hi)
    host = None
    if cache.cu_seqlens is not None:
        host = (cache.cu_host[lo:hi + 1] - cache.cu_host[lo]).to(torch.int32).contiguous()
    return int(lib.sb_bwd_workspace_bytes(ctypes.byref(p), None if host is None else
                                          ctypes.c_void_p(host.data_ptr()), int(store)))


def _varlen_tiles(cache):
    lens = (cache.cu_host[1:] - cache.cu_host[:-1]).tolist()
    H = cache.q.shape[1]
    return sum(H * ((L + 63) // 64) * ((L + 63) // 64 + 1) // 2 for L in lens)


def _backward_call(lib, cache, d_o, ro, dq, dk, dv, store, phases, chunk, workspace):
    """One sb_bwd call over all units (chunk None) or over the units [lo, hi) of
    _unit_chunks' axis: pointer offsets into every per-unit array."""
    q, k, v = cache.q, cache.k, cache.v
    varlen = cache.cu_seqlens is not None
    state, fkb = cache.state, cache.first_kb
    st_off = fkb_off = ro_off = 0
    cu_dev, cu_host = cache.cu_seqlens, cache.cu_host
    if chunk is None:
        p = _cache_params(cache)
        views = (q, k, v, d_o, dq, dk, dv)
    else:
        lo, hi = chunk
        p = _chunk_params(cache, lo, hi)
        if varlen:
            t0, t1 = int(cache.cu_host[lo]), int(cache.cu_host[hi])
            H = q.shape[1]
            views = tuple(t[t0:t1] for t in (q, k, v, d_o, dq, dk, dv))
            cu_host = (cache.cu_host[lo:hi + 1] - t0).to(torch.int32).contiguous()
            cu_dev = cu_host.to(q.device, non_blocking=False)
            p.cu_seqlens = ctypes.c_void_p(cu_dev.data_ptr())
            st_off = ro_off = t0 * H
            nbs = ((cache.cu_host[1:lo + 1] - cache.cu_host[:lo] + 63) // 64).sum().item()
            fkb_off = int(nbs) * H
        else:
            B, H, L = q.shape[0], q.shape[1], q.shape[2]
            nb = -(-L // DEFAULT_BLOCK)
            if B > 1:
                views = tuple(t[lo:hi] for t in (q, k, v, d_o, dq, dk, dv))
                units0 = lo * H
            else:
                views = tuple(t[:, lo:hi] for t in (q, k, v, d_o, dq, dk, dv))
                units0 = lo
            st_off = ro_off = units0 * L
            fkb_off = units0 * nb
    qv, kv, vv, dov, dqv, dkv, dvv = views
    host = None if cu_host is None else ctypes.c_void_p(cu_host.data_ptr())
    ws = workspace
    # the state pointer keeps its 64-float header in front of the chunk's rows (sb_bwd
    # reads only the rows): offset by 2 floats per row
    st_ptr = ctypes.c_void_p(state.data_ptr() + 8 * st_off)
    ro_ptr = None if ro is None else ctypes.c_void_p(ro.data_ptr() + 4 * ro_off)
    fkb_ptr = ctypes.c_void_p(fkb.data_ptr() + 4 * fkb_off)
    with _on(qv):
        _lib.check(lib.sb_bwd(ctypes.byref(p), _ptr(qv), _ptr(kv), _ptr(vv), _ptr(dov), ro_ptr,
                              st_ptr, fkb_ptr, _ptr(dqv), _ptr(dkv), _ptr(dvv), _ptr(ws),
                              ws.numel(), host, int(store), int(phases), _stream(qv)))


class _StickBreakingFn(torch.autograd.Function):
    """Autograd over the C ABI.  Only tensors go through save_for_backward (so
    saved-tensor hooks such as CPU offload see all of them); ctx keeps scalars,
    the layout and the host copy of cu_seqlens."""

    @staticmethod
    def forward(ctx, q, k, v, scale, skip, skip_eps, cu_seqlens, return_rem):
        o, log_rem, _, cache = blocked_forward(q, k, v, skip=skip, skip_eps=skip_eps,
                                               scale=scale, counters=False, cu_seqlens=cu_seqlens)
        ctx.set_materialize_grads(False)
        ctx.meta = (cache.scale, cache.layout, cache.skip, cache.skip_eps, cache.max_seqlen,
                    cache.cu_host, cache.cu_seqlens is not None)
        extra = (cache.cu_seqlens,) if cache.cu_seqlens is not None else ()
        ctx.save_for_backward(cache.q, cache.k, cache.v, log_rem, cache.first_kb, cache.state,
                              *extra)
        ctx.return_rem = return_rem
        if return_rem:
            return o, torch.exp(log_rem)
        return o

    @staticmethod
    def backward(ctx, d_o, d_rem=None):
        q, k, v, log_rem, first_kb, state, *extra = ctx.saved_tensors
        scale, layout, skip, skip_eps, max_seqlen, cu_host, varlen = ctx.meta
        cache = BlockedCache(q, k, v, scale, layout, log_rem, first_kb, state, skip, skip_eps,
                             cu_seqlens=extra[0] if varlen else None, max_seqlen=max_seqlen,
                             cu_host=cu_host)
        if d_o is None and d_rem is None:
            return None, None, None, None, None, None, None, None
        if d_o is None:
            d_o = torch.zeros_like(q)
        # rem_j = 1 - sum_i A_ij  =>  dL/dA_ij -= dL/drem_j : the reference's
        # row_offset hook (blocked.py:241-242, model.py:227-230)
        dq, dk, dv, _ = blocked_backward_twophase(cache, d_o.to(torch.bfloat16), row_offset=d_rem)
        return dq, dk, dv, None, None, None, None, None


def stickbreaking_attention(q, k, v, *, scale: float | None = None, skip: bool = False,
                            skip_eps: float | None = None, return_rem: bool = False,
                            attend_current: bool = False,
                            cu_seqlens: torch.Tensor | None = None):
    """Stick-breaking attention (arXiv 2410.17980), strictly causal.

    q, k, v: CUDA bf16 (batch, heads, seq_len, head_dim), head_dim 64 or 128.
    o_j = sum_{i<j} A_ij v_i with A_ij = sigma(z_ij) prod_{i<k<j} (1 - sigma(z_kj)),
    z = q k^T * scale (scale defaults to 1/sqrt(head_dim)).  With return_rem the
    remaining stick mass rem_j = 1 - sum_i A_ij (B, H, L) float32 is returned too
    and is differentiable.  skip enables the reference's block skipping
    (exact: a skipped block's weights are below skip_eps).

    Nothing O(L^2/64) is kept between the forward and the backward: the forward
    saves the final a per row (float64) and the backward rolls the per-tile M
    snapshots back from it inside its own transient workspace.  Without autograd
    (torch.no_grad(), or no input requiring grad) not even that is written
    (blocked_forward(two_phase=False)).

    Packed varlen: q, k, v (total_tokens, heads, head_dim) and cu_seqlens (int32
    [n_seq+1] offsets); each sequence attends only within itself.
    """
    if attend_current:
        raise ValueError("attend_current=True is not part of the reference semantics "
                         "(strict causality, attention.py:52-54)")
    _check_qkv(q, k, v, varlen=cu_seqlens is not None)
    if skip_eps is None:
        skip_eps = SKIP_EPS_BF16
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[-1])
    if not (torch.is_grad_enabled() and (q.requires_grad or k.requires_grad or v.requires_grad)):
        o, log_rem, _, _ = blocked_forward(q, k, v, skip=bool(skip), skip_eps=float(skip_eps),
                                           scale=float(scale), counters=False,
                                           cu_seqlens=cu_seqlens, two_phase=False)
        return (o, torch.exp(log_rem)) if return_rem else o
    return _StickBreakingFn.apply(q, k, v, float(scale), bool(skip), float(skip_eps), cu_seqlens,
                                  bool(return_rem))
