"""LU with partial pivoting: golden digests from the
reference itself (tools/gen_golden_lu.py) — the oracle on CPU, the CUDA path
on the GPU — bitwise: factor, pivot vector and the singular-column warning."""
from __future__ import annotations

import json

import numpy as np
import pytest

import oracle as O
from golden_inputs import digest, left_trsm_inputs, lu_input
from pathlib import Path

CASES = json.loads((Path(__file__).parent / "golden" / "golden_lu.json").read_text())["cases"]


def _meta(m, n):
    return {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "lu"], ids=lambda c: c["id"])
def test_oracle_lu_matches_reference(case):
    a = lu_input(case["seed"], case["m"], case["n"], case["input"], case["dtype"])
    st = a.reshape(-1).copy()
    sing, piv = O.lu(st, _meta(case["m"], case["n"]),
                     O.levels_from_tree_lu(case["tree"], min(case["m"], case["n"]), case["dtype"]))
    assert sing == case["sing"] and list(piv) == case["piv"]
    assert digest(st) == case["sha256"]


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trsm_left"], ids=lambda c: c["id"])
def test_oracle_left_trsm_matches_reference(case):
    t, b = left_trsm_inputs(case["seed"], case["n"], case["ncols"], case["dtype"])
    ts, bs = t.reshape(-1).copy(), b.reshape(-1).copy()
    O.trsm_llnu(case["alpha"], (ts, _meta(case["n"], case["n"])), (bs, _meta(case["n"], case["ncols"])), kc=case["kc"])
    assert digest(bs) == case["sha256"]
