"""Mixed-precision SPD solve: bf16/fp32 Cholesky + FP64 iterative refinement
(BASELINE.json configs[3]).

The reference has no such mode (its only mixed mode is f32 storage with f64
accumulation, engine/config.py:21,39; iterative refinement is a SPEC
non-goal), so this path is pinned to the FP64 solution instead of to
reference bits:

  factor   A (fp64) -> W (fp32 lower), right-looking in blocks of bs:
           diagonal block: the exact fp32 tree driver (bf_cholesky_s);
           panel:          L21 = A21 * L11^-T as ONE bf16 tcgen05 GEMM against
                           the explicit inverse (L11^-T from bf_trsm_rltn_s);
           trailing:       W22 -= L21 L21^T as a bf16 tcgen05 GEMMT (fp32 TMEM
                           accumulation, fp32 storage);
  refine   x += (L L^T)^-1 (b - A x) with the fp64 residual on the original A
           and fp64 blocked triangular solves on the fp32 factor (matrix-vector
           products against the kept diagonal-block inverses), until
           ||b - A x|| / (||A|| ||x|| + ||b||) <= tol.

Reported throughput is "FP64-equivalent": n^3/3 over factor + refinement
time (the HPL-MxP convention).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Optional

import torch

from .control import ControlNode, flatten_cholesky, parse_tree, resolve_config
from .engine import _lib
from .errors import NotPositiveDefiniteError, ShapeError
from .views import DType, MatrixView, from_torch

__all__ = ["MixedFactor", "MixedResult", "cholesky_mixed", "posv_mixed"]

DIAG_TREE = {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
             "child": {"op": "cholesky", "variant": "unblocked3"}}


@dataclass
class MixedResult:
    x: torch.Tensor
    iterations: int
    backward_error: float
    converged: bool


def _v(t: torch.Tensor) -> _lib.BfView:
    return _lib.as_bfview(from_torch(t))


@dataclass
class MixedFactor:
    """fp32 lower factor W (n x n row-major) and the explicit inverses
    xinv[k] = L_kk^-T of its diagonal blocks (the refinement solves with them)."""
    w: torch.Tensor
    xinv: torch.Tensor
    bs: int


def cholesky_mixed(a: torch.Tensor, bs: int = 1024, diag_tree: Optional[ControlNode] = None) -> MixedFactor:
    """bf16/fp32 factorization of the fp64 SPD matrix `a`."""
    if a.dim() != 2 or a.shape[0] != a.shape[1] or a.dtype != torch.float64 or not a.is_cuda:
        raise ShapeError("cholesky_mixed needs a square fp64 CUDA matrix")
    lib = _lib.lib()
    n = a.shape[0]
    dev = a.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    tree = diag_tree if diag_tree is not None else parse_tree(json.dumps(DIAG_TREE))
    levels = flatten_cholesky(tree, resolve_config(tree, DType.F32))
    arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
    w = torch.empty((n, n), dtype=torch.float32, device=dev)
    _lib.check(lib.bf_convert_f64_f32(ctypes.byref(_v(a)), ctypes.byref(_v(w)), 1, stream), "convert")
    panel = torch.empty((n, bs), dtype=torch.bfloat16, device=dev)
    xt = torch.empty((bs, bs), dtype=torch.bfloat16, device=dev)
    nblk = (n + bs - 1) // bs
    xinv = torch.zeros((nblk, bs, bs), dtype=torch.float32, device=dev)
    info = torch.full((1,), -1, dtype=torch.int32, device=dev)
    for k0 in range(0, n, bs):
        b = min(bs, n - k0)
        r = n - k0 - b
        diag = w[k0:k0 + b, k0:k0 + b]
        # the fp32 driver reports block-local pivots; shift a fresh failure by k0
        v = _v(diag)
        before = info.clone()
        _lib.check(lib.bf_cholesky_s(ctypes.byref(v), arr, len(levels), info.data_ptr(), stream), "diag factor")
        torch.where((before < 0) & (info >= 0), info + k0, info, out=info)
        # L11^-T = X with X * L11^T = I
        x = xinv[k0 // bs, :b, :b]
        x.diagonal().fill_(1.0)
        vt, vx = _v(diag), _v(x)
        _lib.check(lib.bf_trsm_rltn_s(1.0, ctypes.byref(vt), ctypes.byref(vx), 512, None, stream), "inverse")
        if r == 0:
            break
        _lib.check(lib.bf_convert_f32_bf16(ctypes.byref(vx), xt.data_ptr(), bs, 1, stream), "convert")
        a21 = w[k0 + b:, k0:k0 + b]
        _lib.check(lib.bf_convert_f32_bf16(ctypes.byref(_v(a21)), panel.data_ptr(), bs, 0, stream), "convert")
        # L21 = A21 * X  (C = A * Bnk^T with Bnk = X^T)
        _lib.check(lib.bf_gemm_bf16(1.0, panel.data_ptr(), bs, xt.data_ptr(), bs, 0.0, ctypes.byref(_v(a21)), b, 0,
                                    stream), "panel gemm")
        _lib.check(lib.bf_convert_f32_bf16(ctypes.byref(_v(a21)), panel.data_ptr(), bs, 0, stream), "convert")
        a22 = w[k0 + b:, k0 + b:]
        _lib.check(lib.bf_gemm_bf16(-1.0, panel.data_ptr(), bs, panel.data_ptr(), bs, 1.0, ctypes.byref(_v(a22)), b, 1,
                                    stream), "trailing gemmt")
    bad = int(info.item())
    if bad >= 0:
        raise NotPositiveDefiniteError(bad)
    return MixedFactor(w, xinv, bs)


def posv_mixed(a: torch.Tensor, b: torch.Tensor, bs: int = 1024, tol: Optional[float] = None,
               max_iter: int = 30) -> MixedResult:
    """Solve A x = b (A fp64 SPD, full dense row-major on the GPU) to FP64
    accuracy: bf16/fp32 factorization + FP64 iterative refinement."""
    n = a.shape[0]
    lib = _lib.lib()
    stream = torch.cuda.current_stream(a.device).cuda_stream
    tol = tol if tol is not None else 10 * n * torch.finfo(torch.float64).eps
    f = cholesky_mixed(a, bs)
    work = torch.empty((129 * bs,), dtype=torch.float64, device=a.device)
    norm_a = float(torch.linalg.matrix_norm(a, ord=float("inf")))  # checker-grade norm, outside the loop
    norm_b = float(b.abs().max())
    x = torch.zeros_like(b)
    r = b.clone()
    d = torch.empty_like(b)
    it, err = 0, float("inf")
    while it < max_iter:
        d.copy_(r)
        _lib.check(lib.bf_potrs_blocked_f32_d(f.w.data_ptr(), n, f.xinv.data_ptr(), bs, d.data_ptr(), n,
                                              work.data_ptr(), stream), "potrs")
        x.add_(d)
        _lib.check(lib.bf_residual_d(a.data_ptr(), n, x.data_ptr(), b.data_ptr(), r.data_ptr(), n, stream), "residual")
        it += 1
        err = float(r.abs().max()) / (norm_a * float(x.abs().max()) + norm_b)
        if err <= tol:
            break
    return MixedResult(x, it, err, err <= tol)
