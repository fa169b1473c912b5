"""Stick-breaking attention sublayer and decoder stack on the CUDA op.

The caller side of the hot path, restating the reference toy model
(`/root/reference/pkg/src/sbattn/model.py`) in PyTorch on top of
`stickbreaking_attention`:

- `StickBreakingAttention` = `mha_forward` / `mha_backward` (model.py:243-308):
  q, k, v = x Wq, x Wk, x Wv (no biases, weights stored (d_in, d_out) and applied
  as x @ W like the reference), per-head stick-breaking attention, the remainder
  variants (model.py:158-166, :169-193), optional head-wise GroupNorm
  (model.py:135-139), output projection.
  - "sb": leftover mass dropped;
  - "sb_remainder": o += rem * v (rem = 1 - sum_i A_ij, differentiable through the
    op's `return_rem`, whose gradient is the backward's `row_offset`,
    blocked.py:241-242);
  - "sb_remainder_bias": o += rem * r (the reference's dense path, model.py:158-166;
    its blocked path's v - r fold is the same function).
- `SBBlock` / `SBTransformer` = `transformer_forward` (model.py:312-337): token
  embedding, n_layer x (pre-LN attention residual, pre-LN exact-GELU MLP
  residual), final LN, untied head; LayerNorm eps 1e-5 with gain and bias.

Parameters use the reference's flat names ("layers.0.attn.wq", "final_norm.g",
...) through `reference_state_dict` / `load_reference_params`, so a reference
checkpoint (model.py:375-386) maps one to one.  The activations entering the
attention op are bf16 (the op's input type); everything else follows the
module dtype (fp32 master weights under `torch.autocast` in the C5 step).
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from .ops import stickbreaking_attention

VARIANTS = ("sb", "sb_remainder", "sb_remainder_bias")


def _attention(q, k, v, return_rem):
    """(B, H, L, d) bf16 views -> o (B, H, L, d) bf16 [, rem (B, H, L) f32]."""
    return stickbreaking_attention(q, k, v, return_rem=return_rem)


class StickBreakingAttention(nn.Module):
    """n_kv_head < n_head: grouped-query attention (the paper's 1.2B variant uses 12
    query heads over 4 key/value heads; the reference toy
    model has none): wk / wv project to n_kv_head heads and query head h reads
    key/value head h // (n_head / n_kv_head).  The op sees the expanded heads, so
    autograd sums each key/value head's gradient over its group."""

    def __init__(self, d_model: int, n_head: int, variant: str = "sb", group_norm: bool = False,
                 gn_eps: float = 1e-5, init_std: float = 0.02, n_kv_head: int | None = None):
        super().__init__()
        if variant not in VARIANTS:
            raise ValueError(f"unknown attention variant {variant!r}")
        if d_model % n_head:
            raise ValueError("d_model must be a multiple of n_head")
        n_kv_head = n_head if n_kv_head is None else n_kv_head
        if n_kv_head < 1 or n_head % n_kv_head:
            raise ValueError("n_head must be a multiple of n_kv_head")
        self.d_model, self.n_head, self.d_head = d_model, n_head, d_model // n_head
        self.n_kv_head = n_kv_head
        if self.d_head not in (64, 128):
            raise ValueError("the CUDA op supports head_dim 64 and 128")
        self.variant, self.group_norm, self.gn_eps = variant, group_norm, gn_eps
        d_kv = n_kv_head * self.d_head
        for name, d_out in (("wq", d_model), ("wk", d_kv), ("wv", d_kv), ("wo", d_model)):
            self.register_parameter(name, nn.Parameter(torch.randn(d_model, d_out) * init_std))
        if variant == "sb_remainder_bias":
            self.r = nn.Parameter(torch.zeros(n_head, self.d_head))
        if group_norm:
            self.gn_g = nn.Parameter(torch.ones(n_head, self.d_head))
            self.gn_b = nn.Parameter(torch.zeros(n_head, self.d_head))

    def forward(self, x):
        """x (B, L, d_model) -> (B, L, d_model)."""
        B, L, _ = x.shape
        H, dh, Hkv = self.n_head, self.d_head, self.n_kv_head
        q = (x @ self.wq).view(B, L, H, dh)
        k, v = ((x @ w).view(B, L, Hkv, dh) for w in (self.wk, self.wv))
        if Hkv != H:  # grouped-query: query head h reads key/value head h // (H / Hkv)
            k, v = (t.repeat_interleave(H // Hkv, dim=2) for t in (k, v))
        # (B, H, L, d) views of the (B, L, H, d) projections: the op takes any strides
        # with a contiguous head_dim
        qh, kh, vh = (t.to(torch.bfloat16).transpose(1, 2) for t in (q, k, v))
        if self.variant == "sb":
            o = _attention(qh, kh, vh, False).transpose(1, 2).to(x.dtype)
        else:
            # leftover mass rem_j routed to v_j or to r (model.py:158-166): o += rem * route.
            # The reference's blocked path folds the bias variant into v - r instead
            # (model.py:183-188); routing through the op's differentiable rem is the same
            # function and keeps d_r = sum_j rem_j dO_j in fp32 rather than the
            # difference of two bf16-rounded sums (sum dO - sum dV).
            o, rem = _attention(qh, kh, vh, True)
            route = v if self.variant == "sb_remainder" else self.r.to(v.dtype)
            o = o.transpose(1, 2).to(x.dtype) + rem.transpose(1, 2).unsqueeze(-1).to(x.dtype) * route
        if self.group_norm:  # head-wise LayerNorm over d_head (model.py:135-139)
            o = F.layer_norm(o, (dh,), eps=self.gn_eps) * self.gn_g.to(o.dtype) + self.gn_b.to(o.dtype)
        return o.reshape(B, L, self.d_model) @ self.wo


class SBBlock(nn.Module):
    def __init__(self, d_model, n_head, d_inter, variant="sb", group_norm=False, init_std=0.02,
                 n_kv_head=None):
        super().__init__()
        self.ln1 = nn.LayerNorm(d_model, eps=1e-5)
        self.attn = StickBreakingAttention(d_model, n_head, variant, group_norm, init_std=init_std,
                                           n_kv_head=n_kv_head)
        self.ln2 = nn.LayerNorm(d_model, eps=1e-5)
        self.w1 = nn.Parameter(torch.randn(d_model, d_inter) * init_std)
        self.w2 = nn.Parameter(torch.randn(d_inter, d_model) * init_std)

    def forward(self, x):
        x = x + self.attn(self.ln1(x))
        return x + F.gelu(self.ln2(x) @ self.w1) @ self.w2


class SBTransformer(nn.Module):
    """Decoder-only stack: tokens (B, L) int64 -> logits (B, L, vocab)."""

    def __init__(self, vocab_size, n_layer, d_model, n_head, d_inter, variant="sb",
                 group_norm=False, init_std=0.02, n_kv_head=None):
        super().__init__()
        self.embed = nn.Parameter(torch.randn(vocab_size, d_model) * init_std)
        self.layers = nn.ModuleList(SBBlock(d_model, n_head, d_inter, variant, group_norm, init_std,
                                            n_kv_head) for _ in range(n_layer))
        self.final_norm = nn.LayerNorm(d_model, eps=1e-5)
        self.head = nn.Parameter(torch.randn(d_model, vocab_size) * init_std)

    def forward(self, tokens):
        x = self.embed[tokens]
        for layer in self.layers:
            x = layer(x)
        return self.final_norm(x) @ self.head


def n_params(model: nn.Module) -> int:
    return sum(p.numel() for p in model.parameters())


def _ref_names(model: nn.Module) -> dict[str, torch.Tensor]:
    """Reference path -> parameter tensor (model.py:87-117 naming)."""
    out = {}

    def attn(prefix, a: StickBreakingAttention):
        for n in ("wq", "wk", "wv", "wo"):
            out[f"{prefix}.{n}"] = getattr(a, n)
        if a.variant == "sb_remainder_bias":
            out[f"{prefix}.r"] = a.r
        if a.group_norm:
            out[f"{prefix}.gn_g"], out[f"{prefix}.gn_b"] = a.gn_g, a.gn_b

    if isinstance(model, StickBreakingAttention):
        attn("attn", model)
        return out
    out["embed"] = model.embed
    for i, layer in enumerate(model.layers):
        pre = f"layers.{i}"
        out[f"{pre}.ln1.g"], out[f"{pre}.ln1.b"] = layer.ln1.weight, layer.ln1.bias
        attn(f"{pre}.attn", layer.attn)
        out[f"{pre}.ln2.g"], out[f"{pre}.ln2.b"] = layer.ln2.weight, layer.ln2.bias
        out[f"{pre}.mlp.w1"], out[f"{pre}.mlp.w2"] = layer.w1, layer.w2
    out["final_norm.g"], out["final_norm.b"] = model.final_norm.weight, model.final_norm.bias
    out["head"] = model.head
    return out


def reference_state_dict(model: nn.Module) -> dict[str, torch.Tensor]:
    """Parameters under the reference's flat path names."""
    return {k: v.detach() for k, v in _ref_names(model).items()}


def reference_grads(model: nn.Module) -> dict[str, torch.Tensor]:
    """Gradients under the reference's flat path names (None where unset)."""
    return {k: v.grad for k, v in _ref_names(model).items()}


@torch.no_grad()
def load_reference_params(model: nn.Module, params: dict) -> None:
    """Copy a reference parameter dict (numpy or torch, model.py:87-117 / :375-386
    paths) into the module; every path must match in name and shape."""
    names = _ref_names(model)
    missing = set(names) - set(params)
    extra = set(params) - set(names)
    if missing or extra:
        raise KeyError(f"parameter paths differ: missing {sorted(missing)}, extra {sorted(extra)}")
    for k, t in names.items():
        src = torch.as_tensor(params[k])
        if tuple(src.shape) != tuple(t.shape):
            raise ValueError(f"{k}: shape {tuple(src.shape)} != {tuple(t.shape)}")
        t.copy_(src.to(t.dtype))


def train_flops_per_token(model: SBTransformer, seq_len: int) -> float:
    """Training FLOPs per token: 6 x the dense parameters (the embedding gather is
    not a GEMM) + the causal attention's 7*L*d_model per layer (fwd 2 + bwd 5
    GEMM-halves, the FA convention of SURVEY.md §8(d))."""
    dense = n_params(model) - model.embed.numel()
    d = model.layers[0].attn.d_model if len(model.layers) else 0
    return 6.0 * dense + len(model.layers) * 7.0 * seq_len * d


__all__ = ["StickBreakingAttention", "SBBlock", "SBTransformer", "VARIANTS", "n_params",
           "reference_state_dict", "reference_grads", "load_reference_params",
           "train_flops_per_token"]
