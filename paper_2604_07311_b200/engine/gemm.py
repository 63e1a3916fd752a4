"""GEMM family on B200: gemm, gemmt_lower, syrk_lower, gemm_scatter.

Same signatures and edge semantics as the reference engine
(engine/gemm.py:74-242): dims mismatch -> ShapeError, an output that aliases
an input -> AliasingError, alpha=0 & beta=1 -> exact no-op, k=0 or alpha=0 ->
C := beta*C only, beta=0 overwrites C without reading it, GEMMT never touches
the strict upper triangle.  The arithmetic runs in the sm_100a library
(FP64: DMMA; FP32: FFMA; FP32-storage/FP64-acc: DFMA) with the reference's kc
segmentation, so results match the reference bit for bit.  `ways` is accepted
for API parity: every output tile has one writer and a fixed k order, so the
result is identical for every width (the reference's determinism contract).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ..errors import AliasingError, ShapeError
from ..views import DType, MatrixView, views_overlap
from . import _lib
from .config import KernelConfig, default_config

__all__ = [
    "ScatterMatrix",
    "scatter_from_view",
    "gemm_scatter",
    "gemm",
    "gemmt_lower",
    "syrk_lower",
    "sandwich_skew",
]


@dataclass(frozen=True)
class ScatterMatrix:
    """Block-scatter facade: element (i, j) = buf[rscat[i] + cscat[j]]
    (reference engine/gemm.py:46-61).  `buf` is a 1-D device tensor; rscat /
    cscat are int64 host arrays (copied to the device at call time) and
    rbs/cbs the reference's per-block affine-stride summaries (0 = gather)."""

    buf: torch.Tensor
    rscat: np.ndarray
    cscat: np.ndarray
    rbs: np.ndarray
    cbs: np.ndarray
    m: int
    n: int
    dtype: DType


def scatter_from_view(v: MatrixView, mr: int, nr: int) -> ScatterMatrix:
    if v.rs < 0 or v.cs < 0:
        raise ShapeError("engine packing requires non-negative strides (use transposed views)")
    rscat = v.offset + np.arange(v.m, dtype=np.int64) * v.rs
    cscat = np.arange(v.n, dtype=np.int64) * v.cs
    rbs = np.full(max(1, -(-v.m // mr)), v.rs, dtype=np.int64)
    cbs = np.full(max(1, -(-v.n // nr)), v.cs, dtype=np.int64)
    return ScatterMatrix(v.storage, rscat, cscat, rbs, cbs, v.m, v.n, v.dtype)


def _cfg_for(cfg: Optional[KernelConfig], dtype: DType) -> KernelConfig:
    if cfg is None:
        return default_config(dtype)
    if cfg.dtype is not dtype:
        raise ShapeError(f"kernel config dtype {cfg.dtype} != operand dtype {dtype}")
    return cfg


def _check_operands(c: MatrixView, *inputs: MatrixView) -> None:
    for x in inputs:
        if x.dtype is not c.dtype:
            raise ShapeError("mixed operand dtypes are not supported")
        if views_overlap(c, x):
            raise AliasingError("output view aliases an input operand")


def _launch_gemm(alpha, a, b, beta, c, cfg: KernelConfig, lower_only: bool, abort_ptr: int = 0) -> None:
    _lib.require_cuda(a, b, c)
    fn = getattr(_lib.lib(), "bf_gemm_" + _lib.suffix(c.dtype, cfg.acc_dtype))
    va, vb, vc = _lib.as_bfview(a), _lib.as_bfview(b), _lib.as_bfview(c)
    rc = fn(
        float(alpha),
        ctypes.byref(va),
        ctypes.byref(vb),
        float(beta),
        ctypes.byref(vc),
        int(bool(lower_only)),
        int(cfg.kc),
        abort_ptr or None,
        _lib.stream_ptr(c.device),
    )
    _lib.check(rc, "gemm")


def gemm(
    alpha: float,
    a: MatrixView,
    b: MatrixView,
    beta: float,
    c: MatrixView,
    cfg: Optional[KernelConfig] = None,
    ways: int = 1,
) -> None:
    """c := beta*c + alpha*a*b."""
    if a.n != b.m or c.m != a.m or c.n != b.n:
        raise ShapeError(f"gemm dims mismatch: a {a.shape}, b {b.shape}, c {c.shape}")
    _check_operands(c, a, b)
    cfg = _cfg_for(cfg, c.dtype)
    _launch_gemm(alpha, a, b, beta, c, cfg, False)


def gemmt_lower(
    alpha: float,
    a: MatrixView,
    b: MatrixView,
    beta: float,
    c: MatrixView,
    cfg: Optional[KernelConfig] = None,
    ways: int = 1,
) -> None:
    """tril(c) := beta*tril(c) + alpha*tril(a*b); the strict upper triangle of c
    keeps its bits."""
    if c.m != c.n:
        raise ShapeError(f"gemmt needs square c, got {c.shape}")
    if a.n != b.m or c.m != a.m or c.n != b.n:
        raise ShapeError(f"gemmt dims mismatch: a {a.shape}, b {b.shape}, c {c.shape}")
    _check_operands(c, a, b)
    cfg = _cfg_for(cfg, c.dtype)
    _launch_gemm(alpha, a, b, beta, c, cfg, True)


def syrk_lower(
    alpha: float,
    a: MatrixView,
    beta: float,
    c: MatrixView,
    cfg: Optional[KernelConfig] = None,
    ways: int = 1,
) -> None:
    """tril(c) := beta*tril(c) + alpha*a*a^T (reference engine/gemm.py:233-242)."""
    gemmt_lower(alpha, a, a.transposed(), beta, c, cfg=cfg, ways=ways)


def sandwich_skew(
    c: MatrixView,
    a: MatrixView,
    t: np.ndarray,
    cfg: Optional[KernelConfig] = None,
    ways: int = 1,
) -> None:
    """Lower triangle of c := c - a * T * a^T with T skew tridiagonal
    (T[i+1,i] = t[i] = -T[i,i+1]) — reference engine/gemm.py:245-280.

    f64: T*a^T is formed while the B tiles are staged (GL_TRIDIAG loader of
    the DMMA kernel), so no k x n intermediate exists, and every W element is
    rounded as the reference's pack_b_block_tridiag rounds it: bit-identical.
    f32: W is formed once in a device workspace with the reference's f32
    packing arithmetic, then the f32 GEMMT (same bits)."""
    if c.m != c.n:
        raise ShapeError(f"sandwich needs square c, got {c.shape}")
    if a.m != c.m:
        raise ShapeError(f"sandwich dims mismatch: c {c.shape}, a {a.shape}")
    kt = a.n
    t = np.asarray(t, dtype=np.float64)
    if t.shape != (max(kt - 1, 0),):
        raise ShapeError(f"tridiag vector length {t.size} != k - 1 = {kt - 1}")
    _check_operands(c, a)
    cfg = _cfg_for(cfg, c.dtype)
    if kt == 0 or c.m == 0:
        return
    _lib.require_cuda(c, a)
    vc, va = _lib.as_bfview(c), _lib.as_bfview(a)
    stream = _lib.stream_ptr(c.device)
    if c.dtype.value == "f64":
        d_t = torch.as_tensor(t if t.size else np.zeros(1), dtype=torch.float64).to(c.device)
        rc = _lib.lib().bf_sandwich_skew_d(ctypes.byref(vc), ctypes.byref(va), d_t.data_ptr(), int(cfg.kc), stream)
    else:
        d_t = torch.as_tensor(t.astype(np.float32) if t.size else np.zeros(1, np.float32)).to(c.device)
        # W = T*A^T is formed while the f32 kernel stages B: no k x n buffer
        rc = _lib.lib().bf_sandwich_skew_s(ctypes.byref(vc), ctypes.byref(va), d_t.data_ptr(), None, int(cfg.kc),
                                           stream)
    _lib.check(rc, "sandwich_skew")


def _sandwich_dev(c: MatrixView, a: MatrixView, d_t: torch.Tensor, cfg: KernelConfig) -> None:
    """sandwich_skew with T's subdiagonal already on the device (length a.n-1,
    c's element type): the blocked LTL^T's trailing update, no host round trip."""
    if a.n == 0 or c.m == 0:
        return
    vc, va = _lib.as_bfview(c), _lib.as_bfview(a)
    stream = _lib.stream_ptr(c.device)
    if c.dtype.value == "f64":
        rc = _lib.lib().bf_sandwich_skew_d(ctypes.byref(vc), ctypes.byref(va), d_t.data_ptr(), int(cfg.kc), stream)
    else:
        rc = _lib.lib().bf_sandwich_skew_s(ctypes.byref(vc), ctypes.byref(va), d_t.data_ptr(), None, int(cfg.kc),
                                           stream)
    _lib.check(rc, "sandwich_skew")


def _dev_vec(x: np.ndarray, device) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64)).to(device)


def gemm_scatter(
    alpha: float,
    a: ScatterMatrix,
    b: ScatterMatrix,
    beta: float,
    c: ScatterMatrix,
    cfg: KernelConfig,
    ways: int = 1,
    lower_only: bool = False,
) -> None:
    """c := beta*c + alpha*a*b over block-scatter facades (engine/gemm.py:74-160)."""
    if b.m != a.n or c.m != a.m or c.n != b.n:
        raise ShapeError(f"gemm dims mismatch: a {a.m}x{a.n}, b {b.m}x{b.n}, c {c.m}x{c.n}")
    if lower_only:
        raise ShapeError("lower_only is only defined for strided views (use gemmt_lower)")
    _lib.require_cuda(a.buf, b.buf, c.buf)
    dev = c.buf.device
    keep = []

    def sv(x: ScatterMatrix) -> _lib.BfScatterView:
        r, cc = _dev_vec(x.rscat, dev), _dev_vec(x.cscat, dev)
        keep.extend((r, cc))
        return _lib.BfScatterView(x.buf.data_ptr(), x.m, x.n, r.data_ptr(), cc.data_ptr())

    va, vb, vc = sv(a), sv(b), sv(c)
    fn = getattr(_lib.lib(), "bf_gemm_scatter_" + _lib.suffix(c.dtype, cfg.acc_dtype))
    rc = fn(float(alpha), ctypes.byref(va), ctypes.byref(vb), float(beta), ctypes.byref(vc), int(cfg.kc),
            _lib.stream_ptr(dev))
    _lib.check(rc, "gemm_scatter")
    # `keep` dies here: the caching allocator only hands those index vectors
    # to later work on this same stream, which is ordered after the kernel.
