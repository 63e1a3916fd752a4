"""Householder QR against values produced by the
reference itself (tools/gen_golden_qr.py) to rounding, plus the reference's
own properties (tests/test_qr.py): reconstruction, orthogonality, blocked R
equal to unblocked R, the wide-matrix rejection."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

CASES = json.loads((Path(__file__).parent / "golden" / "golden_qr.json").read_text())["cases"]


def _tree(bs):
    from paper_2604_07311_b200.control import ControlNode

    return ControlNode("qr", "unblocked") if bs is None else ControlNode(
        "qr", "blocked", bs=bs, child=ControlNode("qr", "unblocked"))


def test_wide_matrix_rejected():
    import paper_2604_07311_b200 as bf

    class _Wide:  # the shape check comes before any device access
        shape = (2, 3)

    with pytest.raises(bf.errors.ShapeError):
        bf.qr_householder(_Wide())


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: c["id"])
def test_cuda_qr_matches_reference_to_rounding(cuda, case):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.views import DType

    m, n, dt = case["m"], case["n"], case["dtype"]
    rng = np.random.default_rng(case["seed"])
    a0 = rng.uniform(-1, 1, (m, n)).astype(np.float64 if dt == "f64" else np.float32)
    v = bf.make_view(m, n, DType.parse(dt), fill=a0)
    refl = bf.qr_householder(v, _tree(case["bs"]))
    eps = 1e-12 if dt == "f64" else 2e-4
    ref = np.asarray(case["factored"]).reshape(m, n)
    assert np.abs(v.to_numpy() - ref).max() <= eps * max(1.0, np.abs(ref).max())
    assert np.abs(refl.taus - np.asarray(case["taus"])).max() <= eps
    q = bf.form_q(v, refl)
    r = np.triu(v.to_numpy())[:n]
    assert np.linalg.norm(q[:, :n] @ r - a0) / np.linalg.norm(a0) <= 10 * eps
    assert np.linalg.norm(q.T @ q - np.eye(m)) <= 10 * eps * m


@pytest.mark.gpu
def test_cuda_qr_blocked_larger(cuda):
    import paper_2604_07311_b200 as bf

    m, n = 1500, 700
    a0 = np.random.default_rng(3).uniform(-1, 1, (m, n))
    vb, vu = bf.make_view(m, n, fill=a0), bf.make_view(m, n, fill=a0)
    rb = bf.qr_householder(vb, _tree(128))
    ru = bf.qr_householder(vu, _tree(None))
    assert np.abs(np.triu(vb.to_numpy()) - np.triu(vu.to_numpy())).max() < 1e-11
    assert np.abs(rb.taus - ru.taus).max() < 1e-12
    assert len(rb.panels) == (n + 127) // 128
