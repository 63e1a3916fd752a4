"""Skew family: the fused skew sandwich and the
unblocked LTL^T bitwise against digests produced by the reference itself
(tools/gen_golden_ltlt.py); the blocked LTL^T and the Pfaffian to tolerance
(the reference's in-panel updates are NumPy/BLAS products)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from golden_inputs import digest, sandwich_inputs, skew_input

CASES = json.loads((Path(__file__).parent / "golden" / "golden_ltlt.json").read_text())["cases"]


def _meta(m, n):
    return {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "sandwich"], ids=lambda c: c["id"])
def test_oracle_sandwich_matches_reference(case):
    c0, a, t = sandwich_inputs(case["seed"], case["n"], case["k"], case["dtype"])
    cs, as_ = c0.reshape(-1).copy(), a.reshape(-1).copy()
    O.sandwich((cs, _meta(case["n"], case["n"])), (as_, _meta(case["n"], case["k"])), t, kc=case["kc"])
    assert digest(cs) == case["sha256"]


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "ltlt_unblocked"], ids=lambda c: c["id"])
def test_oracle_ltlt_unblocked_matches_reference(case):
    x = skew_input(case["seed"], case["n"], case["input"], case["dtype"]).reshape(-1).copy()
    piv, t = O.ltlt_unblocked(x, _meta(case["n"], case["n"]))
    assert list(piv) == case["piv"]
    assert digest(x) == case["sha256"] and digest(t) == case["t_sha256"]


# ---- GPU --------------------------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "sandwich"], ids=lambda c: c["id"])
def test_cuda_sandwich_matches_reference(cuda, case):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import default_config, sandwich_skew
    from paper_2604_07311_b200.views import DType

    dt = DType.parse(case["dtype"])
    c0, a, t = sandwich_inputs(case["seed"], case["n"], case["k"], case["dtype"])
    c = bf.make_view(case["n"], case["n"], dt, fill=c0)
    av = bf.make_view(case["n"], case["k"], dt, fill=a)
    sandwich_skew(c, av, t, cfg=default_config(dt).with_overrides({"kc": case["kc"]}))
    assert digest(c.to_numpy()) == case["sha256"]


@pytest.mark.gpu
def test_cuda_sandwich_strict_upper_untouched_and_large(cuda):
    """Reference test_engine_sandwich.py:44-65 at a larger size: the fused
    product equals the unfused W = T A^T + GEMMT to rounding, strict upper
    canaries bit-identical; and bitwise equal to the oracle."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import gemmt_lower, sandwich_skew

    n, k = 700, 130
    c0, a, t = sandwich_inputs(4242, n, k)
    c = bf.make_view(n, n, fill=c0)
    sandwich_skew(c, bf.make_view(n, k, fill=a), t)
    got = c.to_numpy()
    assert np.triu(got, 1).tobytes() == np.triu(c0, 1).tobytes()
    td = np.zeros((k, k))
    for i, v in enumerate(t):
        td[i + 1, i], td[i, i + 1] = v, -v
    ref = c0 - a @ (td @ a.T)
    assert np.abs(np.tril(got) - np.tril(ref)).max() < 1e-11
    cs = c0.reshape(-1).copy()
    O.sandwich((cs, _meta(n, n)), (a.reshape(-1).copy(), _meta(n, k)), t, kc=256)
    assert digest(got) == digest(cs)
