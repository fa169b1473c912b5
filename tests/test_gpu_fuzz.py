"""Randomised parity sweep (32 seeded cases, the same every run): shapes, tails,
storage layouts, skip on/off, the remaining-mass output with its gradient (the reference's
row_offset hook), and both backward modes, each against the f64 oracle on the same
bf16-rounded inputs.  Bounds: rel-to-max 2e-2 on o / dq / dk / dv (the bf16 bound of
BASELINE.json), rem to 2e-2 relative, skip decisions (first_kb, visited) exact, and
store-mode gradients bit-identical to recompute mode.
"""

import numpy as np
import pytest
import torch

from tests.gpu_util import oracle_bwd, oracle_fwd, rel_to_max, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2
N_CASES = 32


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 3))
    H = int(rng.integers(1, 4))
    L = int(rng.choice([1, 2, 63, 64, 65, 127, 128, 129, 200, 255, 256, 300, 511, 700]))
    d = int(rng.choice([64, 128]))
    blhd = bool(rng.integers(0, 2))
    skip = bool(rng.integers(0, 2))
    scale_logits = float(rng.choice([0.5, 1.0, 2.0]))
    return B, H, L, d, blhd, skip, scale_logits


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_matches_oracle(seed):
    import paper_2410_17980_b200 as sb
    B, H, L, d, blhd, skip, sl = _case(seed)
    g = torch.Generator().manual_seed(seed)
    shape = (B, L, H, d) if blhd else (B, H, L, d)
    q, k, v, do = (torch.randn(*shape, generator=g) for _ in range(4))
    q = q * sl  # logits of different spreads
    drem = torch.randn(B, H, L, generator=g)
    q, k, v, do = (t.to(torch.bfloat16).cuda() for t in (q, k, v, do))
    if blhd:  # (B, H, L, d) views of BLHD storage
        q, k, v, do = (t.transpose(1, 2) for t in (q, k, v, do))
    drem = drem.cuda()

    grads = []
    for store in (False, True):
        o, lr, st, cache = sb.blocked_forward(q, k, v, skip=skip, skip_eps=1e-6)
        dq, dk, dv, _ = sb.blocked_backward_twophase(cache, do, row_offset=-drem,
                                                      store_tiles=store)
        torch.cuda.synchronize()
        grads.append((o, lr, st, dq, dk, dv))
    for a, b in zip(grads[0][3:], grads[1][3:]):
        assert torch.equal(a, b), "store and recompute backward modes differ"

    o, lr, st, dq, dk, dv = grads[0]
    for bi in range(B):
        ref = oracle_fwd(q[bi], k[bi], v[bi], skip=skip, skip_eps=1e-6)
        rdq, rdk, rdv, _ = oracle_bwd(q[bi], k[bi], v[bi], do[bi], ref, row_offset=-drem[bi])
        assert rel_to_max(to64(o[bi]), ref["o"]) < TOL, (seed, bi)
        np.testing.assert_allclose(np.exp(to64(lr[bi])), np.exp(ref["log_rem"]), atol=TOL, rtol=TOL)
        np.testing.assert_array_equal(st.first_kb[bi].cpu().numpy(), ref["first_kb"])
        for got, r, name in ((dq, rdq, "dq"), (dk, rdk, "dk"), (dv, rdv, "dv")):
            assert rel_to_max(to64(got[bi]), r) < TOL, (seed, bi, name)
