"""ctypes binding of the in-tree CUDA library (libsbattn.so, C ABI in include/sb_attn.h).

There is no fallback: if the library is missing or cannot be loaded the import
of the op raises, so a CPU/PyTorch path can never silently stand in for the
CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsbattn.so")

SB_OK = 0


class SbParams(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("heads", ctypes.c_int32),
        ("seqlen", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64), ("stride_l", ctypes.c_int64),
        ("cu_seqlens", ctypes.c_void_p),
        ("scale", ctypes.c_float), ("block", ctypes.c_int32),
        ("skip", ctypes.c_int32), ("skip_eps", ctypes.c_float),
        ("total_tokens", ctypes.c_int32),
    ]


EXPORTS = ("sb_fwd", "sb_bwd", "sb_bwd_workspace_bytes", "sb_state_elems", "sb_snapshot_elems",
           "sb_varlen_elems", "sb_status_string", "sb_version")

_lib = None


class SbError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libsbattn.so (raises OSError/FileNotFoundError if absent)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} is missing: build it with `python -m paper_2410_17980_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    PP = ctypes.POINTER(SbParams)
    lib.sb_snapshot_elems.restype = ctypes.c_size_t
    lib.sb_snapshot_elems.argtypes = [PP]
    lib.sb_varlen_elems.restype = ctypes.c_int
    lib.sb_varlen_elems.argtypes = [PP, P, ctypes.POINTER(ctypes.c_size_t),
                                    ctypes.POINTER(ctypes.c_size_t)]
    lib.sb_state_elems.restype = ctypes.c_size_t
    lib.sb_state_elems.argtypes = [PP]
    lib.sb_fwd.restype = ctypes.c_int
    lib.sb_fwd.argtypes = [PP, P, P, P, P, P, P, P, P, P]
    lib.sb_bwd_workspace_bytes.restype = ctypes.c_size_t
    lib.sb_bwd_workspace_bytes.argtypes = [PP, P, ctypes.c_int]
    lib.sb_bwd.restype = ctypes.c_int
    lib.sb_bwd.argtypes = [PP, P, P, P, P, P, P, P, P, P, P, P, ctypes.c_size_t, P,
                           ctypes.c_int, ctypes.c_int, P]
    lib.sb_status_string.restype = ctypes.c_char_p
    lib.sb_status_string.argtypes = [ctypes.c_int]
    lib.sb_version.restype = ctypes.c_int
    if path == LIB_PATH:
        _lib = lib
    return lib


def check(status: int) -> None:
    if status != SB_OK:
        msg = load().sb_status_string(status).decode()
        if status in (1, 2, 3, 5):  # the reference raises ValueError for these
            raise ValueError(msg)
        raise SbError(f"sb status {status}: {msg}")
