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


@pytest.mark.gpu
@pytest.mark.parametrize("m,b,zero_col", [(1000, 128, None), (777, 96, 5), (130, 128, 0), (20000, 64, 63)])
def test_cuda_qr_panel_smem_matches_global(cuda, m, b, zero_col):
    """The shared-memory panel sweep against the global-memory one (both sum
    in different orders, so to rounding), including an all-zero column (tau = 0)."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import _lib

    a0 = np.random.default_rng(m + b).uniform(-1, 1, (m, b))
    if zero_col is not None:
        a0[:, zero_col] = 0.0
    lib = _lib.lib()
    out = []
    for glob in (0, 1):
        assert lib.bf_set_option(b"qr_global", glob) == 0
        try:
            v = bf.make_view(m, b, fill=a0)
            refl = bf.qr_householder(v, _tree(None))
            out.append((v.to_numpy(), refl.taus))
        finally:
            lib.bf_set_option(b"qr_global", 0)
    (fs, ts), (fg, tg) = out
    assert np.abs(fs - fg).max() <= 1e-12 * max(1.0, np.abs(fg).max())
    assert np.abs(ts - tg).max() <= 1e-12
    if zero_col is not None:
        assert ts[zero_col] == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("m,n,k,beta", [(128, 300, 9000, 0.0), (96, 96, 5000, 0.5), (130, 1000, 2048, 1.0),
                                        (64, 64, 100, 0.0)])
def test_cuda_gemm_splitk(cuda, dt, m, n, k, beta):
    """The split-K product used by QR's blocked update against NumPy (to rounding)."""
    import ctypes

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import _lib
    from paper_2604_07311_b200.views import DType

    rng = np.random.default_rng(m * n + k)
    npt = np.float64 if dt == "f64" else np.float32
    a0, b0, c0 = (rng.uniform(-1, 1, s).astype(npt) for s in ((k, m), (k, n), (m, n)))
    at, bv, cv = (bf.make_view(*x.shape, DType.parse(dt), fill=x) for x in (a0, b0, c0))
    lib = _lib.lib()
    fn = getattr(lib, "bf_gemm_splitk_" + ("d" if dt == "f64" else "s"))
    _lib.check(fn(-1.5, ctypes.byref(_lib.as_bfview(at.transposed())), ctypes.byref(_lib.as_bfview(bv)), beta,
                  ctypes.byref(_lib.as_bfview(cv)), _lib.stream_ptr(at.device)), "splitk")
    ref = -1.5 * (a0.astype(np.float64).T @ b0.astype(np.float64)) + beta * c0
    tol = 1e-12 if dt == "f64" else 1e-4
    assert np.abs(cv.to_numpy() - ref).max() <= tol * k ** 0.5
