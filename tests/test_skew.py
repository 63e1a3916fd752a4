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


def _gpu_view(x, dt="f64"):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.views import DType

    return bf.make_view(x.shape[0], x.shape[1], DType.parse(dt), fill=x)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "ltlt_unblocked"], ids=lambda c: c["id"])
def test_cuda_ltlt_unblocked_matches_reference(cuda, case):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import ControlNode

    x0 = skew_input(case["seed"], case["n"], case["input"], case["dtype"])
    v = _gpu_view(x0, case["dtype"])
    piv, tri = bf.ltlt_pivoted(v, ControlNode("ltlt", "unblocked"))
    assert list(piv.piv) == case["piv"]
    assert digest(v.to_numpy()) == case["sha256"]
    assert digest(np.asarray(tri.t)) == case["t_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "ltlt_blocked"], ids=lambda c: c["id"])
def test_cuda_ltlt_blocked_matches_reference_to_rounding(cuda, case):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import ControlNode

    n = case["n"]
    x0 = skew_input(case["seed"], n)
    v = _gpu_view(x0)
    piv, tri = bf.ltlt_pivoted(v, ControlNode("ltlt", "blocked", bs=case["bs"], child=ControlNode("ltlt", "unblocked")))
    assert list(piv.piv) == case["piv"]
    assert np.abs(np.asarray(tri.t) - np.asarray(case["t"])).max() <= 1e-10 * max(1.0, np.abs(case["t"]).max())
    ell = bf.unit_lower_from_storage(v)
    perm = piv.permutation(n)
    err = np.linalg.norm(x0[perm][:, perm] - ell @ tri.to_dense() @ ell.T) / np.linalg.norm(x0)
    assert err < 1e-12
    assert np.triu(v.to_numpy(), 1).tobytes() == np.triu(x0, 1).tobytes()  # strict upper never touched


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "pfaffian"], ids=lambda c: c["id"])
def test_cuda_pfaffian_matches_reference(cuda, case):
    import paper_2604_07311_b200 as bf

    x0 = skew_input(case["seed"], case["n"])
    got = bf.pfaffian(_gpu_view(x0))
    ref = case["value"]
    assert abs(got - ref) <= 1e-9 * max(1.0, abs(ref))


@pytest.mark.gpu
def test_cuda_ltlt_larger(cuda):
    """Unblocked at n=300 bitwise against the oracle; blocked at n=1000
    reconstructs; pf(X)^2 = det(X)."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import ControlNode

    x0 = skew_input(31337, 300)
    v = _gpu_view(x0)
    piv, tri = bf.ltlt_pivoted(v, ControlNode("ltlt", "unblocked"))
    st = x0.reshape(-1).copy()
    opiv, ot = O.ltlt_unblocked(st, _meta(300, 300))
    assert list(piv.piv) == list(opiv) and digest(v.to_numpy()) == digest(st)
    n = 1000
    x1 = skew_input(4, n)
    v1 = _gpu_view(x1)
    piv1, tri1 = bf.ltlt_pivoted(v1, ControlNode("ltlt", "blocked", bs=96, child=ControlNode("ltlt", "unblocked")))
    ell = bf.unit_lower_from_storage(v1)
    perm = piv1.permutation(n)
    assert np.linalg.norm(x1[perm][:, perm] - ell @ tri1.to_dense() @ ell.T) / np.linalg.norm(x1) < 1e-11
    x2 = skew_input(5, 12)
    pf = bf.pfaffian(_gpu_view(x2))
    assert abs(pf * pf - np.linalg.det(x2)) <= 1e-9 * abs(np.linalg.det(x2))
