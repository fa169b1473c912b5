"""The reference-schema harness's `equiv` (tests/reports/reference_harness.py, the
column sets of the reference CLI's `sb equiv`, cli.py:343-344) on the current kernels:
every configuration passes (o, dq, dk, dv against the dense f64 oracle within 2e-2;
store and recompute backward bit-identical), and the artifacts carry the schema."""

import csv
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = ["L", "d_block", "skip", "diff_o", "fused_dq", "fused_dk", "fused_dv", "two_dq",
          "two_dk", "two_dv", "two_vs_fused", "result"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("d", [64, 128])
def test_harness_equiv_passes(tmp_path, d):
    out = tmp_path / f"equiv_d{d}"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "reports", "reference_harness.py"),
                        "equiv", "--d", str(d), "--out", str(out)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-500:], r.stderr[-2000:])
    assert r.returncode == 0
    rows = list(csv.reader(open(out / "equiv.csv")))
    assert rows[0] == HEADER
    assert len(rows) == 1 + 6 * 2  # six lengths (1 .. 512), skip off / on
    assert all(row[-1] == "pass" for row in rows[1:])
    man = json.load(open(out / "manifest.json"))
    assert man["command"] == "equiv" and "equiv.csv" in json.dumps(man)
