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
    assert set(syms) >= {"sb_fwd", "sb_bwd", "sb_bwd_phase", "sb_snapshot_elems",
                         "sb_status_string", "sb_version"}
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
    # M/N: a 64-float work-queue header + B*H*n_tiles*64 with n_tiles = nb(nb+1)/2
    # (blocked.py:58-60)
    p = _params(B=2, H=3, L=200)
    nb = 4
    assert lib.sb_snapshot_elems(ctypes.byref(p)) == 64 + 2 * 3 * nb * (nb + 1) // 2 * 64


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


def test_missing_snapshots_rejected(lib):
    """blocked.py:315-316: two-phase backward without M snapshots is an error."""
    p = _params()
    d = ctypes.c_void_p(16)
    rc = lib.sb_bwd(ctypes.byref(p), d, d, d, d, None, d, d, None, d, d, d, d, None)
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


def test_store_mode_needs_no_n_but_recompute_does(lib):
    p = _params()
    d = ctypes.c_void_p(16)
    # recompute mode (no workspace) without N: NULL error before any device work
    rc = lib.sb_bwd_ws(ctypes.byref(p), d, d, d, d, None, None, d, d, None, d, d, d, None, 0, 3,
                       None)
    assert rc == 5
    # store mode with a workspace smaller than sb_bwd_tile_bytes: shape error
    rc = lib.sb_bwd_ws(ctypes.byref(p), d, d, d, d, None, None, d, d, None, d, d, d,
                       ctypes.c_void_p(256), 1024, 3, None)
    assert rc == 1
    assert lib.sb_bwd_tile_bytes(ctypes.byref(p), None) == 1 * 2 * 2 * 3 * 16384 + 256
