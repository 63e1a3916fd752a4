"""Pin the oracle: every golden case, regenerated and replayed through the
CPU restatement (oracle/), must reproduce the reference's output bits
(SHA-256) and error indices.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases
from golden_inputs import digest
from golden_runner import run_case

REPLAYABLE = [c for c in GOLDEN["cases"] if c["kind"] in ("gemm", "gemm_naive", "chol", "trsm", "contract")]


@pytest.mark.parametrize("case", REPLAYABLE, ids=lambda c: f"{c['id']}-{c['kind']}")
def test_oracle_matches_reference_bits(case):
    outs, err = run_case(case, "oracle")
    if outs is None:
        pytest.skip("host BLAS produced different input bits than the reference host")
    for name, arr in outs.items():
        rec = case[name]
        if "values" in rec:
            np.testing.assert_array_equal(arr.reshape(-1), np.asarray(rec["values"], dtype=arr.dtype))
        assert digest(arr) == rec["sha256"], f"{name} differs from the reference"
    assert err == case.get("error"), "error index differs"


def test_hand_cases_recorded():
    hand = {c.get("name"): c for c in golden_cases("hand_gemm")}
    assert hand["gemm_2x2"]["expect"] == [[19.0, 22.0], [43.0, 50.0]]
    assert hand["mixed_1e8"]["expect"] == [[1.0]]
    assert golden_cases("hand_chol")[0]["expect"] == [[2.0, 2.0], [1.0, 2.0]]
    assert golden_cases("hand_trsm_singular")[0]["error"] == 1
