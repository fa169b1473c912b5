"""Attention sublayer and decoder stack on the CUDA op vs the reference model (§8(f) rank 2).

Golden outputs come from the reference's own `mha_forward/mha_backward` and
`transformer_forward/transformer_backward` in f64 (tests/golden/gen_layer_golden.py);
inputs and parameters are regenerated here from seeds.  Our modules hold the same
parameters in fp32; the attention itself runs in bf16 (the op's input type), so the
comparison is rel_to_max (max |ours - ref| / max |ref|) with the bf16 bound 2e-2 on
the attention output path, and 3e-2 on gradients that pass through two bf16 roundings
of q/k/v and dO plus the projections.
"""

import os

import numpy as np
import pytest
import torch

from tests.golden.gen_layer_golden import (MODEL_CASE, SUBLAYER_CASES, digest, model_inputs,
                                           sublayer_inputs)
from tests.gpu_util import rel_to_max

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL_OUT, TOL_GRAD = 2e-2, 3e-2


def _load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def test_layer_fixture_digests():
    """The seeds regenerate exactly the inputs the fixtures were made from (CPU)."""
    for name, c in SUBLAYER_CASES.items():
        x, d_y, p = sublayer_inputs(c["variant"], c["group_norm"], c["seed"])
        assert str(_load(name)["digest"]) == digest(x, d_y, params=p), name
    tokens, d_logits, p = model_inputs()
    assert str(_load(MODEL_CASE["name"])["digest"]) == digest(tokens, d_logits, params=p)


def test_load_reference_params_checks_paths():
    from paper_2410_17980_b200.layer import StickBreakingAttention, load_reference_params
    m = StickBreakingAttention(128, 2, "sb_remainder_bias", group_norm=True)
    _, _, p = sublayer_inputs("sb_remainder_bias", True, 1)
    load_reference_params(m, p)
    assert torch.equal(m.wq.detach().double(), torch.as_tensor(p["attn.wq"]).float().double())
    with pytest.raises(KeyError):
        load_reference_params(m, {k: v for k, v in p.items() if k != "attn.r"})
    with pytest.raises(ValueError):
        load_reference_params(m, dict(p, **{"attn.wq": np.zeros((3, 3))}))


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SUBLAYER_CASES))
def test_sublayer_matches_reference(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_17980_b200.layer import (StickBreakingAttention, load_reference_params,
                                             reference_grads)
    c = SUBLAYER_CASES[name]
    x, d_y, p = sublayer_inputs(c["variant"], c["group_norm"], c["seed"])
    ref = _load(name)
    m = StickBreakingAttention(x.shape[1], 2, c["variant"], c["group_norm"]).cuda()
    load_reference_params(m, p)
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")[None].requires_grad_(True)
    y = m(xt)
    y.backward(torch.tensor(d_y, dtype=torch.float32, device="cuda")[None])
    torch.cuda.synchronize()
    f64 = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    errs = {"y": rel_to_max(f64(y[0]), ref["y"].astype(np.float64)),
            "d_x": rel_to_max(f64(xt.grad[0]), ref["d_x"].astype(np.float64))}
    for k, gr in reference_grads(m).items():
        errs[k] = rel_to_max(f64(gr), ref["grad." + k].astype(np.float64))
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    assert errs["y"] < TOL_OUT
    for k, e in errs.items():
        assert e < TOL_GRAD, (k, e)


@pytest.mark.gpu
def test_decoder_stack_matches_reference():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_17980_b200.layer import SBTransformer, load_reference_params, reference_grads
    c = MODEL_CASE
    tokens, d_logits, p = model_inputs(c)
    ref = _load(c["name"])
    m = SBTransformer(c["vocab"], c["n_layer"], c["n_head"] * c["d_head"], c["n_head"],
                      c["d_inter"]).cuda()
    load_reference_params(m, p)
    logits = m(torch.tensor(tokens, device="cuda")[None])
    logits.backward(torch.tensor(d_logits, dtype=torch.float32, device="cuda")[None])
    torch.cuda.synchronize()
    f64 = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    errs = {"logits": rel_to_max(f64(logits[0]), ref["logits"].astype(np.float64))}
    for k, gr in reference_grads(m).items():
        errs[k] = rel_to_max(f64(gr), ref["grad." + k].astype(np.float64))
    print({k: f"{v:.2e}" for k, v in errs.items()})
    assert errs["logits"] < TOL_OUT
    for k, e in errs.items():
        assert e < TOL_GRAD, (k, e)


def test_gqa_shapes_and_validation():
    """Grouped-query layout (CPU): wk / wv project to n_kv_head heads."""
    from paper_2410_17980_b200.layer import StickBreakingAttention
    a = StickBreakingAttention(512, 4, n_kv_head=2)
    assert tuple(a.wq.shape) == (512, 512) and tuple(a.wk.shape) == (512, 256)
    assert tuple(a.wv.shape) == (512, 256) and a.n_kv_head == 2
    with pytest.raises(ValueError):
        StickBreakingAttention(512, 4, n_kv_head=3)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["sb", "sb_remainder"])
def test_gqa_equals_mha_with_shared_kv(variant):
    """A grouped-query sublayer (12 query heads over 4 key/value heads, as the
    paper's 1.2B model) gives bit-identical outputs to the multi-head sublayer whose
    key/value weights repeat each group's columns, and its wk / wv gradients are the
    group sums of the multi-head ones."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_17980_b200.layer import StickBreakingAttention
    torch.manual_seed(0)
    H, Hkv, dh, L = 12, 4, 64, 320
    d = H * dh
    gqa = StickBreakingAttention(d, H, variant, n_kv_head=Hkv).cuda()
    mha = StickBreakingAttention(d, H, variant).cuda()
    rep = lambda w: w.view(d, Hkv, 1, dh).expand(d, Hkv, H // Hkv, dh).reshape(d, d)  # noqa: E731
    with torch.no_grad():
        mha.wq.copy_(gqa.wq)
        mha.wo.copy_(gqa.wo)
        mha.wk.copy_(rep(gqa.wk))
        mha.wv.copy_(rep(gqa.wv))
    x = torch.randn(2, L, d, device="cuda")
    dy = torch.randn(2, L, d, device="cuda")
    yg, ym = gqa(x), mha(x)
    assert torch.equal(yg, ym)
    yg.backward(dy)
    ym.backward(dy)
    torch.cuda.synchronize()
    for n in ("wk", "wv"):
        gm = getattr(mha, n).grad.view(d, Hkv, H // Hkv, dh).sum(2).reshape(d, Hkv * dh)
        gg = getattr(gqa, n).grad
        assert rel_to_max(gg.double().cpu().numpy(), gm.double().cpu().numpy()) < 1e-5, n
    assert torch.allclose(gqa.wq.grad, mha.wq.grad, rtol=1e-5, atol=1e-6)
