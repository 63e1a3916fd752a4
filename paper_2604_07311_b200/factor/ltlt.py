"""Pivoted factorization of skew-symmetric matrices and the Pfaffian on B200
(reference factor/ltlt.py:1-209).

Factors P*X*P^T = L*T*L^T with L unit lower triangular (first column e_1)
and T tridiagonal skew-symmetric, reading only the strict lower triangle.
The unblocked right-looking stepper (bf_ltlt_*, blocked=0) is one
cooperative-grid launch and reproduces the reference's compiled loops bit
for bit (pivots, multipliers, T, the rank-2 updates).  The blocked form runs
each panel on the grid (bf_ltlt_*, blocked=1: pivot search, two-sided swap
with the history rows, column brought current against the panel's m/w
history, multipliers) and then collapses the deferred trailing update into
one fused skew sandwich X_22 -= A * That * A^T (T*A^T formed while the DMMA
kernel stages its B tiles).  The reference's in-panel updates are NumPy/BLAS
products, so the blocked factor agrees with it to rounding (its own tests
compare the blocked form with a tolerance, tests/test_ltlt_pfaffian.py:59).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ..control import ControlNode, check_valid, default_tree, resolve_config
from ..engine import _lib
from ..engine.gemm import _sandwich_dev
from ..errors import ShapeError, SkewSymmetryError
from ..views import MatrixView, Range, partition_steps
from .pivots import PivotVector

__all__ = ["TridiagSkew", "ltlt_pivoted", "pfaffian", "unit_lower_from_storage"]


@dataclass(frozen=True)
class TridiagSkew:
    """T[i+1,i] = t[i] = -T[i,i+1], zero elsewhere."""

    t: np.ndarray
    n: int

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.n, self.n))
        for i, v in enumerate(np.asarray(self.t, dtype=np.float64)):
            dense[i + 1, i] = v
            dense[i, i + 1] = -v
        return dense


def ltlt_pivoted(x: MatrixView, tree: Optional[ControlNode] = None) -> tuple[PivotVector, TridiagSkew]:
    """Factor P*X*P^T = L*T*L^T in place; returns (pivots, T).

    L's subdiagonal columns overwrite x shifted one column left (column j+1
    of L sits in column j of x); use unit_lower_from_storage to expand it."""
    n = x.n
    if x.m != n:
        raise ShapeError(f"square matrix required, got {x.shape}")
    if tree is None:
        tree = default_tree("ltlt", n, x.dtype)
    check_valid(tree, op="ltlt")
    cfg = resolve_config(tree, x.dtype)
    tdt = torch.float64 if x.dtype.value == "f64" else torch.float32
    if n <= 1:
        return PivotVector(np.arange(n, dtype=np.int64)), TridiagSkew(np.zeros(max(n - 1, 0), dtype=x.dtype.np), n)
    _lib.require_cuda(x)
    dev = x.device
    piv = torch.arange(n, dtype=torch.int64, device=dev)
    t = torch.zeros(n - 1, dtype=tdt, device=dev)
    fn = getattr(_lib.lib(), "bf_ltlt_" + ("d" if x.dtype.value == "f64" else "s"))
    vx = _lib.as_bfview(x)
    stream = _lib.stream_ptr(dev)
    n_elims = n - 1
    if not tree.is_blocked:
        mvec = torch.zeros(n, dtype=tdt, device=dev)
        wvec = torch.zeros(n, dtype=tdt, device=dev)
        rc = fn(ctypes.byref(vx), 0, n_elims, 0, 0, None, 0, piv.data_ptr(), t.data_ptr(), mvec.data_ptr(),
                wvec.data_ptr(), stream)
        _lib.check(rc, "ltlt")
    else:
        wld = min(tree.bs, n_elims)
        wbuf = torch.zeros((n, wld), dtype=tdt, device=dev)
        one = torch.ones(1, dtype=tdt, device=dev)
        for step in partition_steps(n_elims, tree.bs):
            k, b = step.r1.start, step.r1.len
            rc = fn(ctypes.byref(vx), k, k + b, 1, k, wbuf.data_ptr(), wld, piv.data_ptr(), t.data_ptr(), None, None,
                    stream)
            _lib.check(rc, "ltlt panel")
            trail = step.r1.end + 1
            if trail < n:
                c22 = x.subview(Range.span(trail, n), Range.span(trail, n))
                a_blk = x.subview(Range.span(trail, n), Range.span(k, step.r1.end + 1))
                that = torch.cat([t[k + 1:k + b], one]).contiguous()
                _sandwich_dev(c22, a_blk, that, cfg)
    return PivotVector(piv.cpu().numpy()), TridiagSkew(t.cpu().numpy(), n)


def unit_lower_from_storage(x: MatrixView) -> np.ndarray:
    """Expand the shifted in-place L storage into a dense unit lower L."""
    n = x.n
    xn = x.to_numpy()
    ell = np.eye(n, dtype=np.float64)
    for j in range(1, n):
        ell[j + 1:, j] = xn[j + 1:, j - 1]
    return ell


def pfaffian(x: MatrixView, tree: Optional[ControlNode] = None) -> float:
    """Pfaffian of an even-order skew-symmetric matrix (odd order gives 0).

    Uses the pivoted tridiagonal factorization on a copy of x:
    pf(X) = det(P) * pf(T), and pf of the skew tridiagonal is the product
    of its odd-position superdiagonal entries, prod over even i of -t[i]."""
    n = x.n
    if x.m != n:
        raise ShapeError(f"square matrix required, got {x.shape}")
    xn = x.to_numpy()
    scale = float(np.max(np.abs(xn))) if n else 0.0
    if n and float(np.max(np.abs(xn + xn.T))) > n * x.dtype.eps * scale:
        raise SkewSymmetryError("input is not skew-symmetric to working precision")
    if n % 2 == 1:
        return 0.0
    if n == 0:
        return 1.0
    from ..views import make_view

    work = make_view(n, n, x.dtype, fill=xn, device=x.device)
    piv, tri = ltlt_pivoted(work, tree)
    pf_t = 1.0
    for i in range(0, n - 1, 2):
        pf_t *= -float(tri.t[i])
    return piv.sign() * pf_t
