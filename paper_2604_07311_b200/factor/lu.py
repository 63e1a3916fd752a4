"""LU with partial pivoting and the paired triangular solves on B200
(reference factor/lu.py:1-130).

`lu_partial(a, tree)` keeps the reference signature and contracts: P*a = L*U
in place (unit-lower L below the diagonal, U on and above), a LAPACK-style
PivotVector returned, a SingularFactorWarning for the first exactly-zero
pivot column (the factorization continues).  The tree walk (blocked levels
down to the unblocked leaf) runs natively in bf_lu_*: per block step the
panel's child factorization, the row swaps left and right of it, the
left-lower-unit TRSM and the trailing GEMM — the reference's operations in
its order, so the factor and the pivots are bit-identical.  `lu_solve` keeps
its signature; its last stage (the reference's NumPy row loop) runs as a
blocked upper triangular solve, so it matches to rounding, not bitwise.
"""
from __future__ import annotations

import ctypes
import warnings
from typing import Optional

import numpy as np
import torch

from ..control import ControlNode, check_valid, default_tree, flatten_lu, resolve_config
from ..engine import _lib
from ..errors import ShapeError, SingularFactorWarning, SingularMatrixError
from ..views import MatrixView, Range
from .pivots import PivotVector, apply_pivots

__all__ = ["lu_partial", "lu_solve"]


def lu_partial(a: MatrixView, tree: Optional[ControlNode] = None) -> PivotVector:
    """Factor P*a = L*U in place: unit-lower L below the diagonal, U on and
    above. Returns the pivot vector; warns on exactly-zero pivot columns."""
    m, n = a.shape
    steps = min(m, n)
    if tree is None:
        tree = default_tree("lu", steps, a.dtype)
    check_valid(tree, op="lu")
    if steps == 0:
        return PivotVector(np.arange(0, dtype=np.int64))
    _lib.require_cuda(a)
    levels = flatten_lu(tree, resolve_config(tree, a.dtype))
    arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, bs, kc) for v, bs, kc in levels])
    d_piv = torch.arange(steps, dtype=torch.int64, device=a.device)
    d_sing = torch.full((1,), -1, dtype=torch.int32, device=a.device)
    fn = getattr(_lib.lib(), "bf_lu_" + ("d" if a.dtype.value == "f64" else "s"))
    rc = fn(ctypes.byref(_lib.as_bfview(a)), arr, len(levels), d_piv.data_ptr(), d_sing.data_ptr(),
            _lib.stream_ptr(a.device))
    _lib.check(rc, "lu")
    sing = int(d_sing.item())
    if sing >= 0:
        warnings.warn(f"exactly-zero pivot column {sing}: U is singular there", SingularFactorWarning, stacklevel=2)
    return PivotVector(d_piv.cpu().numpy())


def lu_solve(factored: MatrixView, piv: PivotVector, b: MatrixView, ways: int = 1) -> None:
    """b := A^-1 b given the in-place LU of the square matrix A."""
    n = factored.m
    if factored.n != n:
        raise ShapeError(f"solve needs a square factor, got {factored.shape}")
    if b.m != n:
        raise ShapeError(f"rhs rows {b.m} != {n}")
    _lib.require_cuda(factored)
    _lib.require_cuda(b)
    suffix = "d" if b.dtype.value == "f64" else "s"
    lib = _lib.lib()
    stream = _lib.stream_ptr(b.device)
    apply_pivots(b, piv, "forward")
    kc = resolve_config(default_tree("lu", n, b.dtype), b.dtype).kc
    vf, vb = _lib.as_bfview(factored), _lib.as_bfview(b)
    _lib.check(getattr(lib, "bf_trsm_llnu_" + suffix)(1.0, ctypes.byref(vf), ctypes.byref(vb), int(kc), stream),
               "lu_solve forward")
    # the reference scans i = n-1 .. 0 and stops at the first zero diagonal
    diag = torch.as_strided(factored.storage, (n,), (factored.rs + factored.cs,), factored.offset)
    zero = torch.nonzero(diag == 0.0).flatten()
    if zero.numel():
        i = int(zero.max().item())
        if i + 1 < n:  # rows below it are solved before the reference meets it
            sub_u = factored.subview(Range(i + 1, n - i - 1), Range(i + 1, n - i - 1))
            sub_b = b.subview(Range(i + 1, n - i - 1), Range(0, b.n))
            _lib.check(getattr(lib, "bf_trsm_lun_" + suffix)(ctypes.byref(_lib.as_bfview(sub_u)),
                                                            ctypes.byref(_lib.as_bfview(sub_b)), int(kc), stream),
                       "lu_solve backward")
        raise SingularMatrixError(i, "U factor")
    _lib.check(getattr(lib, "bf_trsm_lun_" + suffix)(ctypes.byref(vf), ctypes.byref(vb), int(kc), stream),
               "lu_solve backward")
