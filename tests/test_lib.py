"""CPU-side checks of the C ABI library (no GPU needed, no compute calls).

The library must load, export every entry point include/sb_attn.h declares,
and reject invalid arguments with the status codes that mirror the
reference's ValueErrors before touching the device.
"""

import ctypes
import os
import re

import pytest

from paper_2410_17980_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sb_attn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(sb_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2410_17980_b200 import build
        build.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert set(syms) >= {"sb_fwd", "sb_bwd", "sb_bwd_workspace_bytes", "sb_state_elems",
                         "sb_snapshot_elems", "sb_status_string", "sb_version"}
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_lib.EXPORTS) == set(syms)


def test_version_and_status_strings(lib):
    assert lib.sb_version() >= 1
    for code in range(8):
        assert lib.sb_status_string(code)
    assert b"(0, 1)" in lib.sb_status_string(2)


def _params(**kw):
    p = _lib.SbParams()
    p.batch, p.heads, p.seqlen, p.head_dim = kw.get("B", 1), kw.get("H", 2), kw.get("L", 256), kw.get("d", 64)
    p.stride_h = p.seqlen * p.head_dim
    p.stride_b = p.heads * p.stride_h
    p.stride_l = p.head_dim
    p.block = kw.get("block", 64)
    p.skip = kw.get("skip", 0)
    p.skip_eps = kw.get("skip_eps", 0.0)
    p.scale = 0.0
    return p


def test_snapshot_elems_matches_layout(lib):
    # one snapshot array (M or N): a 64-float work-queue header + B*H*n_tiles*64 with
    # n_tiles = nb(nb+1)/2 (blocked.py:58-60)
    p = _params(B=2, H=3, L=200)
    nb = 4
    assert lib.sb_snapshot_elems(ctypes.byref(p)) == 64 + 2 * 3 * nb * (nb + 1) // 2 * 64


def test_state_is_O_L(lib):
    """The forward keeps one float64 per row (plus the header), not a snapshot per tile."""
    p = _params(B=2, H=3, L=200)
    assert lib.sb_state_elems(ctypes.byref(p)) == 64 + 2 * 2 * 3 * 200


def test_workspace_bytes(lib):
    """M snapshots (rounded up to 1 KiB) + dZ tiles (store) or N (recompute)."""
    p = _params(B=1, H=2, L=256)  # nb = 4 (10 tiles), n_qt = 2 (6 dZ tiles per unit)
    m = (64 + 2 * 10 * 64) * 4
    mr = -(-m // 1024) * 1024
    assert lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 1) == mr + 2 * 6 * 16384
    assert lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 0) == mr + m
    # varlen needs the host offsets
    cu = (ctypes.c_int32 * 3)(0, 128, 256)
    p.cu_seqlens = ctypes.cast(cu, ctypes.c_void_p)
    p.batch, p.total_tokens = 2, 256
    assert lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 1) == 0
    m = (64 + 2 * 2 * 3 * 64) * 4
    assert lib.sb_bwd_workspace_bytes(ctypes.byref(p), cu, 1) == -(-m // 1024) * 1024 + 2 * 2 * 2 * 16384


@pytest.mark.parametrize("kw,code", [
    (dict(d=96), 4),               # head_dim not 64/128
    (dict(block=32), 3),           # d_block must be 64
    (dict(L=0), 3),                # seq_len >= 1 (blocked.py:64-65)
    (dict(skip=1, skip_eps=1.5), 2),  # skip_eps in (0,1) (blocked.py:155-156)
])
def test_invalid_arguments_rejected_before_launch(lib, kw, code):
    p = _params(**kw)
    dummy = ctypes.c_void_p(16)
    rc = lib.sb_fwd(ctypes.byref(p), dummy, dummy, dummy, dummy, dummy, dummy, dummy, None, None)
    assert rc == code


def test_varlen_elems(lib):
    """Packed varlen: each sequence is planned separately (blocked.py:63-67 per sequence)."""
    p = _params(B=3, H=2, L=200)
    cu = (ctypes.c_int32 * 4)(0, 200, 200, 265)  # lengths 200, 0, 65
    snap, fkb = ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.sb_varlen_elems(ctypes.byref(p), cu, ctypes.byref(snap), ctypes.byref(fkb)) == 0
    nbs = [4, 0, 2]
    assert snap.value == 64 + 2 * sum(n * (n + 1) // 2 for n in nbs) * 64
    assert fkb.value == 2 * sum(nbs)
    bad = (ctypes.c_int32 * 4)(0, 200, 100, 265)
    assert lib.sb_varlen_elems(ctypes.byref(p), bad, ctypes.byref(snap), ctypes.byref(fkb)) == 1


def test_varlen_needs_total_tokens(lib):
    p = _params(B=2, H=2, L=128)
    cu = (ctypes.c_int32 * 3)(0, 64, 128)
    p.cu_seqlens = ctypes.cast(cu, ctypes.c_void_p)
    p.total_tokens = 0
    d = ctypes.c_void_p(16)
    assert lib.sb_fwd(ctypes.byref(p), d, d, d, d, d, d, d, None, None) == 1


def test_python_varlen_validation():
    import torch
    import paper_2410_17980_b200 as sb
    q = torch.zeros(10, 2, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError):  # 4-D tensors are not a packed batch
        sb.stickbreaking_attention(q[None], q[None], q[None],
                                   cu_seqlens=torch.tensor([0, 10], dtype=torch.int32))


def _bwd(lib, p, state, ws, nbytes, cu_host=None, store=1):
    d = ctypes.c_void_p(16)
    return lib.sb_bwd(ctypes.byref(p), d, d, d, d, None, state, d, d, d, d, ws, nbytes, cu_host,
                      store, 3, None)


def test_missing_state_rejected(lib):
    """blocked.py:315-316: a two-phase backward without the forward's state is an error."""
    p = _params()
    rc = _bwd(lib, p, None, ctypes.c_void_p(1024), 1 << 30)
    assert rc == 5
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_python_op_refuses_cpu_tensors():
    import torch
    import paper_2410_17980_b200 as sb
    q = torch.zeros(1, 1, 8, 64, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sb.stickbreaking_attention(q, q, q)


def test_skip_rejects_stop_index_overflow(lib):
    """The skip-on forward packs a stop tile into 13 bits: nb >= 8192 is refused."""
    p = _params(L=8192 * 64, skip=1)
    d = ctypes.c_void_p(16)
    assert lib.sb_fwd(ctypes.byref(p), d, d, d, d, d, d, d, None, None) == 4
    p = _params(L=8191 * 64, skip=0)  # skip off has no such limit (no device call: d=96)
    p.head_dim = 96
    assert lib.sb_fwd(ctypes.byref(p), d, d, d, d, d, d, d, None, None) == 4


def test_workspace_checked(lib):
    p = _params()
    d = ctypes.c_void_p(16)
    need = lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 1)
    # no workspace / too small: errors before any device work
    assert _bwd(lib, p, d, None, 0) == 5
    assert _bwd(lib, p, d, ctypes.c_void_p(1024), need - 1) == 1
    assert _bwd(lib, p, d, ctypes.c_void_p(1024), lib.sb_bwd_workspace_bytes(ctypes.byref(p), None, 0),
                store=1) == 1
    # varlen without host offsets: the workspace cannot be checked
    cu = (ctypes.c_int32 * 2)(0, 256)
    p.cu_seqlens = ctypes.cast(cu, ctypes.c_void_p)
    p.total_tokens = 256
    assert _bwd(lib, p, d, ctypes.c_void_p(1024), 1 << 30) == 5


def test_varlen_offsets_checked_by_the_backward(lib):
    """A seqlen below the longest sequence would drop work items silently; the
    backward checks the host offsets against it (and total_tokens)."""
    p = _params(B=2, H=2, L=128)
    cu = (ctypes.c_int32 * 3)(0, 64, 200)  # second sequence 136 > seqlen 128
    p.cu_seqlens = ctypes.cast(cu, ctypes.c_void_p)
    p.total_tokens = 200
    d = ctypes.c_void_p(16)
    assert _bwd(lib, p, d, ctypes.c_void_p(1024), 1 << 40, cu_host=cu) == 1
    p.seqlen = 136
    p.total_tokens = 199  # last offset must be total_tokens
    assert _bwd(lib, p, d, ctypes.c_void_p(1024), 1 << 40, cu_host=cu) == 1
