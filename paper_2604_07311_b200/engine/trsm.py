"""Triangular solve for the Cholesky panel (reference engine/trsm.py:29-68).

RIGHT_LOWER_TRANS_NONUNIT solves X * tril(T)^T = alpha*B in place.  The
recursion (halve until n <= 32, off-diagonal block through gemm with the
caller's kc) and the base-case substitution run natively in the sm_100a
library in the reference's exact operation order, so the solution is
bit-identical.  A zero diagonal raises SingularMatrixError with the
base-local column index, as the reference does (engine/trsm.py:128-135).
LEFT_LOWER_NOTRANS_UNIT solves unit_tril(T) * X = alpha*B in place (the
LU's case, engine/trsm.py:71-88,114-125): the same halving, a base case one
thread per column, bit-identical.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ..errors import ShapeError, SingularMatrixError
from ..views import MatrixView
from . import _lib
from .config import KernelConfig, default_config

__all__ = ["trsm", "RIGHT_LOWER_TRANS_NONUNIT", "LEFT_LOWER_NOTRANS_UNIT"]

RIGHT_LOWER_TRANS_NONUNIT = "right_lower_trans_nonunit"
LEFT_LOWER_NOTRANS_UNIT = "left_lower_notrans_unit"


def trsm(
    case: str,
    alpha: float,
    tri: MatrixView,
    b: MatrixView,
    cfg: Optional[KernelConfig] = None,
    ways: int = 1,
) -> None:
    if tri.m != tri.n:
        raise ShapeError(f"triangular operand must be square, got {tri.shape}")
    if case == LEFT_LOWER_NOTRANS_UNIT:
        if b.m != tri.n:
            raise ShapeError(f"left solve dims mismatch: b {b.shape}, tri {tri.shape}")
        if b.n == 0 or tri.n == 0:
            return
        cfg = cfg if cfg is not None else default_config(b.dtype)
        _lib.require_cuda(tri, b)
        fn = getattr(_lib.lib(), "bf_trsm_llnu_" + ("d" if b.dtype.value == "f64" else "s"))
        rc = fn(float(alpha), ctypes.byref(_lib.as_bfview(tri)), ctypes.byref(_lib.as_bfview(b)), int(cfg.kc),
                _lib.stream_ptr(b.device))
        _lib.check(rc, "trsm")
        return
    if case != RIGHT_LOWER_TRANS_NONUNIT:
        raise ValueError(f"unknown trsm case {case!r}")
    if b.n != tri.n:
        raise ShapeError(f"right solve dims mismatch: b {b.shape}, tri {tri.shape}")
    if b.m == 0 or tri.n == 0:
        return
    cfg = cfg if cfg is not None else default_config(b.dtype)
    _lib.require_cuda(tri, b)
    flag = torch.full((1,), -1, dtype=torch.int32, device=b.device)
    fn = getattr(_lib.lib(), "bf_trsm_rltn_" + ("d" if b.dtype.value == "f64" else "s"))
    vt, vb = _lib.as_bfview(tri), _lib.as_bfview(b)
    rc = fn(float(alpha), ctypes.byref(vt), ctypes.byref(vb), int(cfg.kc), flag.data_ptr(), _lib.stream_ptr(b.device))
    _lib.check(rc, "trsm")
    bad = int(flag.item())  # synchronises: the reference raises before returning
    if bad >= 0:
        raise SingularMatrixError(bad)
