"""B200-native stick-breaking attention (arXiv 2410.17980) hot path.

Forward, two-phase backward and block skipping as hand-written sm_100a CUDA
kernels (tcgen05 / TMEM / TMA) behind a C ABI (include/sb_attn.h), exposed as
``stickbreaking_attention(q, k, v, ...)`` (a torch.autograd.Function).
"""

from .ops import (  # noqa: F401
    DEFAULT_BLOCK,
    BlockedCache,
    BlockLayout,
    TileStats,
    blocked_backward_twophase,
    blocked_forward,
    default_skip_eps,
    plan_blocks,
    sb_forward_blocked,
    skip_stats,
    stickbreaking_attention,
)

__version__ = "0.1.0"
