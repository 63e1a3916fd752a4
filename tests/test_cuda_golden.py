"""The CUDA path against the reference's own bits: every golden case
(tests/golden/golden.json, produced by the reference) is regenerated and run
through the product API on the GPU; outputs must have the reference's
SHA-256 and the same error index.  Cholesky cases run through both the
native tree driver and the Python tree walk."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN
from golden_inputs import digest
from golden_runner import run_case

pytestmark = pytest.mark.gpu

CASES = [c for c in GOLDEN["cases"] if c["kind"] in ("gemm", "chol", "trsm", "contract")]
CHOL_PY = [dict(c, engine="python") for c in GOLDEN["cases"] if c["kind"] == "chol"]


def _check(case, outs, err):
    if outs is None:
        pytest.skip("host BLAS produced different input bits than the reference host")
    for name, arr in outs.items():
        rec = case[name]
        if "values" in rec:
            np.testing.assert_array_equal(arr.reshape(-1), np.asarray(rec["values"], dtype=arr.dtype))
        assert digest(arr) == rec["sha256"], f"{name} differs from the reference bits"
    assert err == case.get("error")


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['id']}-{c['kind']}")
def test_cuda_matches_reference_bits(cuda, case):
    outs, err = run_case(case, "cuda")
    _check(case, outs, err)


@pytest.mark.parametrize("case", CHOL_PY, ids=lambda c: f"{c['id']}-py")
def test_cuda_python_tree_walk_matches_reference_bits(cuda, case):
    outs, err = run_case(case, "cuda")
    _check(case, outs, err)
