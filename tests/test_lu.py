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


# ---- GPU: the CUDA path against the same digests ----------------------------


def _gpu_lu(case):
    import warnings

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree
    from paper_2604_07311_b200.views import DType

    a = lu_input(case["seed"], case["m"], case["n"], case["input"], case["dtype"])
    v = bf.make_view(case["m"], case["n"], DType.parse(case["dtype"]), fill=a)
    sing = -1
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        piv = bf.lu_partial(v, parse_tree(json.dumps(case["tree"])) if case["tree"] else None)
        for x in w:
            if issubclass(x.category, bf.errors.SingularFactorWarning):
                sing = int(str(x.message).split("column ")[1].split(":")[0])
    return v, piv, sing


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "lu"], ids=lambda c: c["id"])
def test_cuda_lu_matches_reference(cuda, case):
    v, piv, sing = _gpu_lu(case)
    assert sing == case["sing"] and list(piv.piv) == case["piv"]
    assert digest(v.to_numpy()) == case["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "trsm_left"], ids=lambda c: c["id"])
def test_cuda_left_trsm_matches_reference(cuda, case):
    import ctypes

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import _lib
    from paper_2604_07311_b200.views import DType

    dt = DType.parse(case["dtype"])
    t, b = left_trsm_inputs(case["seed"], case["n"], case["ncols"], case["dtype"])
    vt, vb = bf.make_view(case["n"], case["n"], dt, fill=t), bf.make_view(case["n"], case["ncols"], dt, fill=b)
    fn = getattr(_lib.lib(), "bf_trsm_llnu_" + ("d" if case["dtype"] == "f64" else "s"))
    rc = fn(float(case["alpha"]), ctypes.byref(_lib.as_bfview(vt)), ctypes.byref(_lib.as_bfview(vb)), case["kc"],
            _lib.stream_ptr(vb.device))
    assert rc == 0
    assert digest(vb.to_numpy()) == case["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("leaf_opts", [(), ("lu_nocluster",), ("lu_nocluster", "lu_noprefetch"), ("lu_global",)])
@pytest.mark.parametrize("n,m_rows,tree", [(1500, 1500, [256, 32]), (600, 2000, [128, 16]), (3000, 3000, [512, 64, 16]),
                                           (128, 9000, [64, 32])])
def test_cuda_lu_bitwise_vs_oracle_larger(cuda, n, m_rows, tree, leaf_opts):
    """Sizes past the golden set (tall, square, three levels) against the
    oracle, for each leaf kernel path (one cluster with DSMEM, shared-memory
    bands on a cooperative grid with and without the candidate-row prefetch,
    global memory); then lu_solve to rounding against numpy."""
    from paper_2604_07311_b200.engine import _lib

    for o in leaf_opts:
        assert _lib.lib().bf_set_option(o.encode(), 1) == 0
    try:
        _lu_larger(n, m_rows, tree)
    finally:
        for o in leaf_opts:
            _lib.lib().bf_set_option(o.encode(), 0)


def _lu_larger(n, m_rows, tree):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree

    doc = {"op": "lu", "variant": "unblocked"}
    for bs in reversed(tree):
        doc = {"op": "lu", "variant": "blocked", "bs": bs, "child": doc}
    a = lu_input(777 + n, m_rows, n, "uniform")
    st = a.reshape(-1).copy()
    sing, piv = O.lu(st, _meta(m_rows, n), O.levels_from_tree_lu(doc, min(m_rows, n), "f64"), nthreads=O.host_threads())
    v = bf.make_view(m_rows, n, fill=a)
    gp = bf.lu_partial(v, parse_tree(json.dumps(doc)))
    assert list(gp.piv) == list(piv)
    assert digest(v.to_numpy()) == digest(st)
    if m_rows == n:
        rhs = np.random.default_rng(5).uniform(-1, 1, (n, 3))
        vb = bf.make_view(n, 3, fill=rhs)
        bf.lu_solve(v, gp, vb)
        x = vb.to_numpy()
        ref = np.linalg.solve(a, rhs)
        assert np.abs(x - ref).max() / np.abs(ref).max() < 1e-9
