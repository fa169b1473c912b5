"""CPU oracle for the stick-breaking attention hot path.

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  Only tests/,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import this package, and only as the checker or
the timed CPU baseline.  The product path (``paper_2410_17980_b200``) never
imports it and fails loudly when its CUDA extension is missing.

Two restatements of the reference (/root/reference/pkg/src/sbattn):

* ``dense_forward`` / ``dense_backward`` — NumPy float64 restatement of the
  dense O(L^2) oracle ``sb_forward`` / ``sb_backward`` (attention.py:106-145),
  in query-row orientation (the reference uses key-row orientation; the
  matrices here are its transposes).
* ``tiled_forward`` / ``tiled_backward`` — ctypes binding of the plain-C
  restatement of ``blocked_forward(two_phase=True)`` and
  ``blocked_backward_twophase`` (blocked.py:129-392) in sb_oracle.c, float64
  or float32, batched over independent (batch, head) units with host threads.

Parity of both is pinned against golden vectors written by the reference
itself (oracle/gen_golden.py -> tests/golden/*.npz; tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsb_oracle.so")
_lib = None

SOFTPLUS_LINEAR_THRESHOLD = 15.0  # numerics.py:19
DEFAULT_BLOCK = 64  # blocked.py:41
SKIP_EPS_F32 = 1e-6  # blocked.py:43


def build(force: bool = False) -> str:
    """Compile sb_oracle.c with the committed Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    for sfx in ("f64", "f32"):
        f = getattr(lib, f"sbo_forward_batch_{sfx}")
        f.restype = ctypes.c_longlong
        f.argtypes = [ctypes.c_int] * 4 + [P, P, P, ctypes.c_int, ctypes.c_double,
                                          P, P, P, P, ctypes.c_int]
        b = getattr(lib, f"sbo_backward_batch_{sfx}")
        b.restype = ctypes.c_int
        b.argtypes = [ctypes.c_int] * 4 + [P] * 11 + [ctypes.c_int]
    _lib = lib
    return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def n_threads_default() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def softplus(x):
    """numerics.py:33-47 restated: log1p(exp(min(x,15))) for x <= 15 else x."""
    x = np.asarray(x)
    return np.where(x <= SOFTPLUS_LINEAR_THRESHOLD,
                    np.log1p(np.exp(np.minimum(x, SOFTPLUS_LINEAR_THRESHOLD))), x)


def n_tiles(L: int, block: int = DEFAULT_BLOCK) -> int:
    nb = -(-L // block)
    return nb * (nb + 1) // 2


def tiled_forward(q, k, v, *, block=DEFAULT_BLOCK, skip=False, skip_eps=None,
                  dtype=np.float64, n_threads=None):
    """Batched blocked_forward(two_phase=True) restatement.

    q, k, v: (..., L, d) arrays; every leading index is an independent unit.
    Returns dict(o, log_rem, first_kb, M, visited) with M shaped
    (..., n_tiles, block) in tile(qb,kb) = qb*(qb+1)/2 + kb order.
    """
    lib = _load()
    q = np.ascontiguousarray(q, dtype=dtype)
    k = np.ascontiguousarray(k, dtype=dtype)
    v = np.ascontiguousarray(v, dtype=dtype)
    lead, (L, d) = q.shape[:-2], q.shape[-2:]
    units = int(np.prod(lead)) if lead else 1
    nb = -(-L // block)
    if skip_eps is None:
        skip_eps = SKIP_EPS_F32 if dtype == np.float32 else 1e-12  # blocked.py:42-43
    o = np.zeros_like(q)
    a = np.zeros(lead + (L,), dtype=dtype)
    fkb = np.zeros(lead + (nb,), dtype=np.int64)
    M = np.zeros(lead + (n_tiles(L, block), block), dtype=dtype)
    sfx = "f64" if dtype == np.float64 else "f32"
    vis = getattr(lib, f"sbo_forward_batch_{sfx}")(
        units, L, d, block, _ptr(q), _ptr(k), _ptr(v), int(bool(skip)), float(skip_eps),
        _ptr(o), _ptr(a), _ptr(fkb), _ptr(M), n_threads or n_threads_default())
    if vis < 0:
        raise ValueError("oracle forward rejected its arguments")
    return dict(o=o, log_rem=a, first_kb=fkb, M=M, visited=int(vis),
                total=units * n_tiles(L, block))


def tiled_backward(q, k, v, d_o, fwd, *, block=DEFAULT_BLOCK, row_offset=None,
                   dtype=np.float64, n_threads=None):
    """Batched blocked_backward_twophase restatement; returns (dq, dk, dv, N)."""
    lib = _load()
    q = np.ascontiguousarray(q, dtype=dtype)
    k = np.ascontiguousarray(k, dtype=dtype)
    v = np.ascontiguousarray(v, dtype=dtype)
    d_o = np.ascontiguousarray(d_o, dtype=dtype)
    lead, (L, d) = q.shape[:-2], q.shape[-2:]
    units = int(np.prod(lead)) if lead else 1
    ro = None if row_offset is None else np.ascontiguousarray(row_offset, dtype=dtype)
    M = np.ascontiguousarray(fwd["M"], dtype=dtype)
    fkb = np.ascontiguousarray(fwd["first_kb"], dtype=np.int64)
    N = np.zeros_like(M)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    sfx = "f64" if dtype == np.float64 else "f32"
    rc = getattr(lib, f"sbo_backward_batch_{sfx}")(
        units, L, d, block, _ptr(q), _ptr(k), _ptr(v), _ptr(d_o), _ptr(ro), _ptr(fkb),
        _ptr(M), _ptr(N), _ptr(dq), _ptr(dk), _ptr(dv), n_threads or n_threads_default())
    if rc:
        raise ValueError("oracle backward rejected its arguments")
    return dq, dk, dv, N


def _strict_mask(L):
    # query-row orientation: key i < query j  <=>  entry (j, i) with i < j
    return np.tril(np.ones((L, L), dtype=bool), k=-1)


def dense_forward(q, k, v):
    """attention.py:106-115 restated per unit, (..., L, d) float64.

    Returns (o, log_rem) with log_rem = log of the remaining stick mass
    (attention.py:148-150: 1 - colsum(A) = exp(-cumlog[0, j])).
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    L, d = q.shape[-2:]
    z = (q @ np.swapaxes(k, -1, -2)) / math.sqrt(d)  # [.., j(query), i(key)]
    mask = _strict_mask(L)
    sp = np.where(mask, softplus(z), 0.0)
    cum = np.flip(np.cumsum(np.flip(sp, -1), -1), -1)  # sum over keys i..j-1
    a = np.exp(np.where(mask, z - cum, -np.inf))
    o = a @ v
    log_rem = -cum[..., 0] if L > 0 else np.zeros(q.shape[:-1])
    return o, log_rem, dict(z=z, a=a, mask=mask)


def dense_backward(q, k, v, d_o, row_offset=None):
    """attention.py:118-145 restated (with the d_a_extra hook = -row_offset)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d_o = np.asarray(d_o, dtype=np.float64)
    L, d = q.shape[-2:]
    scale = 1.0 / math.sqrt(d)
    _, _, c = dense_forward(q, k, v)
    z, a, mask = c["z"], c["a"], c["mask"]
    d_a = d_o @ np.swapaxes(v, -1, -2)
    if row_offset is not None:
        d_a = d_a - np.asarray(row_offset, dtype=np.float64)[..., None]
    d_at = d_a * a
    s = np.cumsum(d_at, axis=-1)  # keys ascending: i' <= i
    sig = 1.0 / (1.0 + np.exp(-np.clip(z, -700, 700)))
    d_z = np.where(mask, d_at - sig * s, 0.0)
    d_q = d_z @ k * scale
    d_k = np.swapaxes(d_z, -1, -2) @ q * scale
    d_v = np.swapaxes(a, -1, -2) @ d_o
    return d_q, d_k, d_v


def max_rel_err(approx, exact) -> float:
    """numerics.py:116-124: max |a - e| / max(1, |e|)."""
    a = np.asarray(approx, dtype=np.float64)
    e = np.asarray(exact, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - e) / np.maximum(1.0, np.abs(e))))


def rel_to_max(approx, exact) -> float:
    """max|a - e| / max|e| (the bf16 gate of SURVEY.md §8(c))."""
    a = np.asarray(approx, dtype=np.float64)
    e = np.asarray(exact, dtype=np.float64)
    den = np.max(np.abs(e)) if e.size else 0.0
    if den == 0.0:
        return float(np.max(np.abs(a))) if a.size else 0.0
    return float(np.max(np.abs(a - e)) / den)
