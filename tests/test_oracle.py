"""Pin the CPU oracle (oracle/) against golden vectors written by the reference.

The reference package itself wrote tests/golden/*.npz (oracle/gen_golden.py);
here the C restatement and the NumPy dense restatement must reproduce them at
the reference's own tolerances (test_blocked.py:71, :150, :203; 1e-10 / 1e-9
in float64) and the float32 path must meet BASELINE.json's 1e-5 bound.
"""

import os

import numpy as np
import pytest

import oracle
from tests.golden_inputs import CASES, digest, make_inputs


def _run(spec, dtype):
    inp = make_inputs(spec)
    fwd = oracle.tiled_forward(inp["q"], inp["k"], inp["v"], block=spec["block"],
                               skip=spec.get("skip", False), skip_eps=spec.get("skip_eps"),
                               dtype=dtype)
    bwd = oracle.tiled_backward(inp["q"], inp["k"], inp["v"], inp["d_o"], fwd,
                                block=spec["block"], row_offset=inp.get("row_offset"),
                                dtype=dtype)
    return inp, fwd, bwd


def _check_digest(g, inp):
    assert bytes(g["digest"]).decode() == digest(inp), "input generation drifted"


F64_CASES = [n for n, s in CASES.items() if s.get("dtype", "float64") == "float64"]
F32_CASES = [n for n, s in CASES.items() if s.get("dtype") == "float32"]


@pytest.mark.parametrize("name", F64_CASES)
def test_c_oracle_f64_matches_reference(name, golden):
    spec = CASES[name]
    g = golden(name)
    inp, fwd, (dq, dk, dv, N) = _run(spec, np.float64)
    _check_digest(g, inp)
    np.testing.assert_array_equal(fwd["first_kb"], g["first_kb"])
    assert fwd["visited"] == int(g["visited"].sum())
    assert np.max(np.abs(fwd["log_rem"] - g["log_rem"])) < 1e-10
    if "o" in g:
        assert np.max(np.abs(fwd["o"] - g["o"])) < 1e-10
    if "M" in g:
        present = ~np.isnan(g["M"])
        assert np.max(np.abs(np.where(present, fwd["M"] - g["M"], 0.0))) < 1e-10
    for key, got in (("dq", dq), ("dk", dk), ("dv", dv)):
        if key in g:
            assert np.max(np.abs(got - g[key])) < 1e-9, key


@pytest.mark.parametrize("name", [n for n in F64_CASES if "dense_o" in np.load(
    f"{__import__('os').path.dirname(__file__)}/golden/{n}.npz")])
def test_dense_oracle_matches_reference(name, golden):
    spec = CASES[name]
    g = golden(name)
    inp = make_inputs(spec)
    o, log_rem, _ = oracle.dense_forward(inp["q"], inp["k"], inp["v"])
    dq, dk, dv = oracle.dense_backward(inp["q"], inp["k"], inp["v"], inp["d_o"],
                                       inp.get("row_offset"))
    assert np.max(np.abs(o - g["dense_o"])) < 1e-12
    for got, key in ((dq, "dense_dq"), (dk, "dense_dk"), (dv, "dense_dv")):
        assert np.max(np.abs(got - g[key])) < 1e-11, key
    # the reference forms rem = 1 - colsum(A) (attention.py:148-150), which
    # cancels once the stick is consumed: compare in linear space
    assert np.max(np.abs(np.exp(log_rem) - np.exp(g["dense_log_rem"]))) < 1e-12


@pytest.mark.parametrize("name", F32_CASES)
def test_c_oracle_f32_matches_reference(name, golden):
    spec = CASES[name]
    g = golden(name)
    inp, fwd, (dq, dk, dv, _) = _run(spec, np.float32)
    _check_digest(g, inp)
    np.testing.assert_array_equal(fwd["first_kb"], g["first_kb"])
    assert fwd["visited"] == int(g["visited"].sum())
    assert oracle.max_rel_err(fwd["log_rem"], g["log_rem"]) < 1e-5
    for key, got in (("o", fwd["o"]), ("dq", dq), ("dk", dk), ("dv", dv)):
        if key in g:
            assert oracle.max_rel_err(got, g[key]) < 1e-5, key


def test_config1_fp32_path_within_1e5_of_f64(golden):
    """BASELINE.json: fp32 path <= 1e-5 relative on config 1 (two-phase, stored M)."""
    spec = CASES["c1_f64"]
    g = golden("c1_f64")
    _, fwd, (dq, dk, dv, _) = _run(spec, np.float32)
    for got, key in ((fwd["o"], "o"), (dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert oracle.max_rel_err(got, g[key]) < 1e-5, key


def test_known_answers(golden):
    c = golden("constants")
    np.testing.assert_allclose(oracle.softplus(c["softplus_x"]), c["softplus_y"], rtol=1e-15)
    assert oracle.softplus(16.0) == 16.0  # linear branch is exact (test_numerics.py:26-29)
    # two tokens, zero logits: o_1 = 0.5 v_0 (test_attention.py:126-132)
    q = np.zeros((2, 3)); k = np.zeros((2, 3)); v = np.arange(6.0).reshape(2, 3)
    o, _, _ = oracle.dense_forward(q, k, v)
    assert np.array_equal(o[0], np.zeros(3)) and np.allclose(o[1], 0.5 * v[0], atol=1e-15)
    fwd = oracle.tiled_forward(q, k, v, block=8)
    assert np.allclose(fwd["o"], o, atol=1e-15)
    # tile count 6 at L=192, block 64 (test_blocked.py:205-209)
    assert oracle.n_tiles(192, 64) == 6


def test_length_one_all_zero():
    """test_blocked.py:253-259: L=1 gives all-zero outputs and gradients."""
    g = np.random.default_rng(0)
    q, k, v = (g.normal(size=(1, 4)) for _ in range(3))
    fwd = oracle.tiled_forward(q, k, v, block=8)
    dq, dk, dv, _ = oracle.tiled_backward(q, k, v, np.ones((1, 4)), fwd, block=8)
    for a in (fwd["o"], dq, dk, dv):
        assert np.array_equal(a, np.zeros((1, 4)))


def test_skip_soundness_random():
    """test_blocked.py:109-114: skip on vs off agree on random inputs."""
    g = np.random.default_rng(9)
    q, k, v = (g.normal(size=(160, 16)) for _ in range(3))
    off = oracle.tiled_forward(q, k, v, block=16, skip=False)
    on = oracle.tiled_forward(q, k, v, block=16, skip=True)
    assert np.max(np.abs(on["o"] - off["o"])) < 1e-9
    assert on["visited"] <= off["visited"]


def test_c3_decision_generator_matches_c_oracle():
    """tests/golden/gen_c3_first_kb.py (the C3 golden skip decisions) follows the C
    oracle's blocked_forward decisions exactly on bf16 shifted-logit inputs."""
    import importlib.util
    import math
    spec = importlib.util.spec_from_file_location(
        "gen_c3", os.path.join(os.path.dirname(__file__), "golden", "gen_c3_first_kb.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    from tests.golden_inputs import bf16_round
    rs = np.random.default_rng(4)
    for mu in (-6.0, -7.0, 0.0):
        L, d = 2048, 64
        q = bf16_round(rs.standard_normal((L, d)))
        k = bf16_round(rs.standard_normal((L, d)))
        q[:, 0] = mu * math.sqrt(d)
        k[:, 0] = 1.0
        fkb, vis, m = gen.head_decisions(q, k)
        ref = oracle.tiled_forward(q, k, np.zeros_like(q), block=64, skip=True, skip_eps=1e-6)
        np.testing.assert_array_equal(fkb, ref["first_kb"])
        assert vis == ref["visited"]
