"""Householder QR on B200: unblocked column sweeps and compact-WY blocked
panels (reference factor/qr.py:1-149).

The factored matrix holds R in its upper triangle and the reflector vectors
(implicit leading 1) below the diagonal; H_j = I - tau_j v_j v_j^T.  Each
panel is swept by one cooperative-grid launch (bf_qr_panel_*: norm, beta,
tau, reflector scaling, w = a(j, j+1:) + v^T A and the rank-1 update), its T
accumulated on the device (bf_qr_t_*), and (I - V T V^T)^T applied to the
trailing matrix with two engine GEMMs and T^T W between them, like the
reference.  Every panel operation of the reference is a NumPy/BLAS product,
so the factor agrees with it to rounding (its tests are tolerance tests).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ..control import ControlNode, check_valid, default_tree, resolve_config
from ..engine import _lib
from ..engine.gemm import gemm
from ..errors import ShapeError
from ..views import MatrixView, Range, from_torch, partition_steps

__all__ = ["Reflectors", "qr_householder", "apply_q", "form_q"]


@dataclass(frozen=True)
class Reflectors:
    """Scalars tau per reflector plus, for blocked panels, (start, T) pairs."""

    taus: np.ndarray
    panels: tuple = ()


def _sfx(v: MatrixView) -> str:
    return "d" if v.dtype.value == "f64" else "s"


def qr_householder(a: MatrixView, tree: Optional[ControlNode] = None) -> Reflectors:
    """Factor a = Q*R in place (m >= n); returns the reflector data."""
    m, n = a.shape
    if m < n:
        raise ShapeError(f"qr requires m >= n, got {a.shape}")
    if tree is None:
        tree = default_tree("qr", n, a.dtype)
    check_valid(tree, op="qr")
    cfg = resolve_config(tree, a.dtype)
    tdt = torch.float64 if a.dtype.value == "f64" else torch.float32
    if n == 0:
        return Reflectors(np.zeros(0, dtype=a.dtype.np))
    _lib.require_cuda(a)
    lib = _lib.lib()
    stream = _lib.stream_ptr(a.device)
    taus = torch.zeros(n, dtype=tdt, device=a.device)
    panel_fn = getattr(lib, "bf_qr_panel_" + _sfx(a))
    if not tree.is_blocked:
        _lib.check(panel_fn(ctypes.byref(_lib.as_bfview(a)), taus.data_ptr(), stream), "qr panel")
        return Reflectors(taus.cpu().numpy())
    panels = []
    for step in partition_steps(n, tree.bs):
        k, b = step.r1.start, step.r1.len
        rows = Range.span(k, m)
        panel = a.subview(rows, step.r1)
        tk = taus[k:k + b]
        _lib.check(panel_fn(ctypes.byref(_lib.as_bfview(panel)), tk.data_ptr(), stream), "qr panel")
        t_mat = torch.empty((b, b), dtype=tdt, device=a.device)
        v = torch.empty((m - k, b), dtype=tdt, device=a.device)
        gram = torch.empty((b, b), dtype=tdt, device=a.device)
        _lib.check(getattr(lib, "bf_qr_t_" + _sfx(a))(ctypes.byref(_lib.as_bfview(panel)), tk.data_ptr(),
                                                       t_mat.data_ptr(), v.data_ptr(), gram.data_ptr(), stream), "qr T")
        panels.append((k, t_mat))
        if step.r2.len > 0:
            # trailing := trailing - V (T^T (V^T trailing))   (qr.py:103-121)
            trailing = a.subview(rows, step.r2)
            vv = from_torch(v)
            w = torch.empty((b, step.r2.len), dtype=tdt, device=a.device)
            wv = from_torch(w)
            # V^T C has b x n outputs and K = m - k: split-K over side streams
            _lib.check(getattr(lib, "bf_gemm_splitk_" + _sfx(a))(
                1.0, ctypes.byref(_lib.as_bfview(vv.transposed())), ctypes.byref(_lib.as_bfview(trailing)), 0.0,
                ctypes.byref(_lib.as_bfview(wv)), stream), "qr V^T C")
            w2 = torch.zeros_like(w)
            gemm(1.0, from_torch(t_mat).transposed(), wv, 0.0, from_torch(w2), cfg=cfg, ways=tree.ways)
            gemm(-1.0, vv, from_torch(w2), 1.0, trailing, cfg=cfg, ways=tree.ways)
    return Reflectors(taus.cpu().numpy(), tuple((k, t.cpu().numpy()) for k, t in panels))


def apply_q(a: MatrixView, refl: Reflectors, c: MatrixView, transpose: bool = False) -> None:
    """c := Q c (or Q^T c) by applying the stored reflectors one at a time."""
    if c.m != a.m:
        raise ShapeError(f"c rows {c.m} != {a.m}")
    _lib.require_cuda(a)
    _lib.require_cuda(c)
    fn = getattr(_lib.lib(), "bf_reflector_apply_" + _sfx(c))
    stream = _lib.stream_ptr(c.device)
    va, vc = _lib.as_bfview(a), _lib.as_bfview(c)
    n = len(refl.taus)
    order = range(n) if transpose else range(n - 1, -1, -1)
    for j in order:
        tau = float(refl.taus[j])
        if tau == 0.0:
            continue
        _lib.check(fn(ctypes.byref(va), j, tau, ctypes.byref(vc), stream), "apply_q")


def form_q(a: MatrixView, refl: Reflectors) -> np.ndarray:
    """Dense m-by-m Q obtained by applying the reflectors to the identity."""
    from ..views import make_view

    q = make_view(a.m, a.m, a.dtype, fill=np.eye(a.m, dtype=a.dtype.np), device=a.device)
    apply_q(a, refl, q)
    return q.to_numpy().copy()
