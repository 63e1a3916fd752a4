"""Mixed-precision SPD solve: bf16/fp32 Cholesky + FP64 iterative refinement
(BASELINE.json configs[3]).

The reference has no such mode (its only mixed mode is f32 storage with f64
accumulation, engine/config.py:21,39; iterative refinement is a SPEC
non-goal), so this path is pinned to the FP64 solution instead of to
reference bits:

  factor   A (fp64) -> W (fp32 lower), right-looking in blocks of bs:
           diagonal block: FP64, the exact tree driver (bf_cholesky_d);
           panel:          L21 = A21 * L11^-T as ONE bf16 tcgen05 GEMM against
                           the explicit inverse (L11^-T from bf_trsm_rltn_d);
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

__all__ = ["F32TcWorkspace", "MixedFactor", "MixedResult", "MixedWorkspace", "cholesky_f32_tc", "cholesky_mixed",
           "posv_mixed"]

DIAG_TREE = {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
             "child": {"op": "cholesky", "variant": "unblocked3"}}  # FP64 diagonal blocks


@dataclass
class MixedResult:
    x: torch.Tensor
    iterations: int
    backward_error: float
    converged: bool


def _v(t: torch.Tensor) -> _lib.BfView:
    return _lib.as_bfview(from_torch(t))


class MixedWorkspace:
    """Every buffer of one mixed solve of order n (block bs), allocated once:
    repeated solves never touch the allocator (multi-GB blocks churning
    through the caching allocator cost more than the solve)."""

    def __init__(self, n: int, bs: int = 2048, device: Optional[torch.device] = None,
                 precision: str = "bf16") -> None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if precision not in ("bf16", "tf32"):
            raise ValueError(f"precision must be 'bf16' or 'tf32', got {precision!r}")
        self.n, self.bs, self.device, self.precision = n, bs, dev, precision
        nblk = (n + bs - 1) // bs
        # panel operands of the tensor-core GEMMs: bf16 copies, or fp32 read as tf32
        pdt = torch.bfloat16 if precision == "bf16" else torch.float32
        self.w = torch.empty((n, n), dtype=torch.float32, device=dev)
        self.pbuf = [torch.empty((n, bs), dtype=pdt, device=dev) for _ in range(2)]
        self.xt = torch.empty((bs, bs), dtype=pdt, device=dev)
        self.d64 = torch.empty((bs, bs), dtype=torch.float64, device=dev)
        self.x64 = torch.empty((bs, bs), dtype=torch.float64, device=dev)
        self.xinv = torch.zeros((nblk, bs, bs), dtype=torch.float32, device=dev)
        self.info = torch.empty((1,), dtype=torch.int32, device=dev)
        self.before = torch.empty((1,), dtype=torch.int32, device=dev)
        self.work = torch.empty((129 * bs,), dtype=torch.float64, device=dev)
        self.rows = torch.empty((n,), dtype=torch.float64, device=dev)
        self.x = torch.empty((n,), dtype=torch.float64, device=dev)
        self.r = torch.empty((n,), dtype=torch.float64, device=dev)
        self.d = torch.empty((n,), dtype=torch.float64, device=dev)
        self.side = torch.cuda.Stream(dev, priority=-1)


@dataclass
class MixedFactor:
    """fp32 lower factor W (n x n row-major) and the explicit inverses
    xinv[k] = L_kk^-T of its diagonal blocks (the refinement solves with them)."""
    w: torch.Tensor
    xinv: torch.Tensor
    bs: int


def cholesky_mixed(a: torch.Tensor, bs: int = 2048, diag_tree: Optional[ControlNode] = None,
                   lookahead: bool = True, ws: Optional[MixedWorkspace] = None,
                   precision: Optional[str] = None) -> MixedFactor:
    """bf16/fp32 factorization of the fp64 SPD matrix `a` (right-looking,
    blocks of bs).  Per block: the diagonal block in FP64 (the exact tree
    driver, DMMA GEMMs), its explicit inverse in FP64, the panel as one bf16
    tcgen05 GEMM against that inverse, and the trailing update as a bf16
    GEMMT.  With lookahead the next block column is updated first and the
    next diagonal/inverse/panel run on a high-priority side stream while the
    rest of the trailing update proceeds.  precision "tf32" runs the panel and
    trailing GEMMs as tcgen05 kind::tf32 on the fp32 data itself (no bf16
    copies; ~2^-11 instead of ~2^-8 per product, so fewer refinement steps)."""
    if a.dim() != 2 or a.shape[0] != a.shape[1] or a.dtype != torch.float64 or not a.is_cuda:
        raise ShapeError("cholesky_mixed needs a square fp64 CUDA matrix")
    if bs % 8:
        raise ShapeError("bs must be a multiple of 8 (16-byte bf16 rows for TMA)")
    lib = _lib.lib()
    n = a.shape[0]
    if ws is None:
        ws = MixedWorkspace(n, bs, a.device, precision or "bf16")
    if ws.n != n or ws.bs != bs or ws.device != a.device:
        raise ShapeError("workspace was made for another order, block size or device")
    if precision is not None and precision != ws.precision:
        raise ShapeError(f"workspace was made for precision {ws.precision!r}")
    tf32 = ws.precision == "tf32"
    if tf32 and n % 4:
        raise ShapeError("precision 'tf32' needs n % 4 == 0 (16-byte fp32 rows for TMA)")
    tree = diag_tree if diag_tree is not None else parse_tree(json.dumps(DIAG_TREE))
    levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
    arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
    info = ws.info
    info.fill_(-1)
    # the per-block loop is native (bf_cholesky_mixed): FP64 diagonal block,
    # FP64 inverse, tensor-core panel and trailing GEMMs, lookahead on the
    # library's high-priority stream
    rc = lib.bf_cholesky_mixed(ctypes.byref(_v(a)), ws.w.data_ptr(), n, ws.pbuf[0].data_ptr(), ws.pbuf[1].data_ptr(),
                               ws.xt.data_ptr(), ws.d64.data_ptr(), ws.x64.data_ptr(), ws.xinv.data_ptr(), bs, arr,
                               len(levels), 1 if tf32 else 0, 1 if lookahead else 0, info.data_ptr(),
                               torch.cuda.current_stream(a.device).cuda_stream)
    _lib.check(rc, "bf_cholesky_mixed")
    w, xinv = ws.w, ws.xinv
    bad = int(info.item())
    if bad >= 0:
        raise NotPositiveDefiniteError(bad)
    return MixedFactor(w, xinv, bs)


def posv_mixed(a: torch.Tensor, b: torch.Tensor, bs: int = 2048, tol: Optional[float] = None,
               max_iter: int = 30, lookahead: bool = True, ws: Optional[MixedWorkspace] = None,
               precision: Optional[str] = None, step_tol: Optional[float] = None) -> MixedResult:
    """Solve A x = b (A fp64 SPD, full dense row-major on the GPU) to FP64
    accuracy: bf16/fp32 factorization + FP64 iterative refinement.  The
    returned x lives in the workspace (copy it before reusing ws).

    Refinement stops when the normwise backward error
    ||b - Ax||_inf / (||A||_inf ||x||_inf + ||b||_inf) <= tol (default
    10 n eps) and, when step_tol is given, the last correction is also small:
    ||dx||_inf / ||x||_inf <= step_tol — the forward-error criterion (SURVEY.md
    §8(c) asks ||x - x_ref|| / ||x_ref|| <= 1e-12 against the FP64 solution;
    step_tol = 1e-13 reaches it)."""
    n = a.shape[0]
    lib = _lib.lib()
    stream = torch.cuda.current_stream(a.device).cuda_stream
    tol = tol if tol is not None else 10 * n * torch.finfo(torch.float64).eps
    if ws is None:
        ws = MixedWorkspace(n, bs, a.device, precision or "bf16")
    f = cholesky_mixed(a, bs, lookahead=lookahead, ws=ws, precision=precision)
    work = ws.work
    _lib.check(lib.bf_row_abs_sum_d(a.data_ptr(), n, ws.rows.data_ptr(), n, stream), "row sums")
    norm_a, norm_b = torch.stack([ws.rows.max(), b.abs().max()]).tolist()  # one host read
    x, r, d = ws.x, ws.r, ws.d
    x.zero_()
    r.copy_(b)
    it, err = 0, float("inf")
    while it < max_iter:
        d.copy_(r)
        _lib.check(lib.bf_potrs_blocked_f32_d(f.w.data_ptr(), n, f.xinv.data_ptr(), bs, d.data_ptr(), n,
                                              work.data_ptr(), stream), "potrs")
        x.add_(d)
        _lib.check(lib.bf_residual_d(a.data_ptr(), n, x.data_ptr(), b.data_ptr(), r.data_ptr(), n, stream), "residual")
        it += 1
        xmax, rmax, dmax = torch.stack([x.abs().max(), r.abs().max(), d.abs().max()]).tolist()  # one host read
        err = rmax / (norm_a * xmax + norm_b)
        step_ok = step_tol is None or dmax <= step_tol * xmax
        if err <= tol and step_ok:
            break
    return MixedResult(x, it, err, err <= tol and step_ok)


# --------------------------------------------------------------------------
# FP32 Cholesky on the tensor cores (3xTF32)
#
# The reference's FP32 path (f32 storage, f32 or f64 accumulation,
# engine/config.py:21,39) is reproduced bit for bit by the DMMA/SIMT engine
# (bf_cholesky_s).  This is the tensor-core alternative at FP32 accuracy, to
# rounding: every GEMM runs as ONE tcgen05 kind::tf32 GEMM over operands split
# into tf32 hi/lo parts (A B^T = hi hi^T + hi lo^T + lo hi^T, K = 3k, fp32
# accumulation in TMEM).  Per block of bs: the diagonal block in FP64 (exact
# tree driver) and its explicit inverse, the panel L21 = A21 L11^-T as a 3xTF32
# GEMM, the trailing update as a 3xTF32 GEMMT; lookahead as in cholesky_mixed.
# --------------------------------------------------------------------------
class F32TcWorkspace:
    """Buffers of one FP32 tensor-core factorization of order n (block bs)."""

    def __init__(self, n: int, bs: int = 1024, device: Optional[torch.device] = None) -> None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.bs, self.device = n, bs, dev
        self.kp = (bs + 3) // 4 * 4
        # split panels [hi | hi | lo | hi] (ping-pong: panel k+1 forms while step k's update reads panel k)
        self.pbuf = [torch.empty((n, 4 * self.kp), dtype=torch.float32, device=dev) for _ in range(2)]
        self.d64 = torch.empty((bs, bs), dtype=torch.float64, device=dev)
        self.x64 = torch.empty((bs, bs), dtype=torch.float64, device=dev)
        self.x32 = torch.empty((bs, bs), dtype=torch.float32, device=dev)
        self.info = torch.empty((1,), dtype=torch.int32, device=dev)
        self.before = torch.empty((1,), dtype=torch.int32, device=dev)
        self.side = torch.cuda.Stream(dev, priority=-1)


def cholesky_f32_tc(a: torch.Tensor, bs: int = 1024, diag_tree: Optional[ControlNode] = None,
                    lookahead: bool = True, ws: Optional[F32TcWorkspace] = None) -> torch.Tensor:
    """In-place lower Cholesky of the fp32 SPD matrix `a` (square, row-major,
    CUDA) with 3xTF32 tensor-core GEMMs; the strict upper triangle is left
    untouched.  Returns the device pivot flag (-1 = success) after raising
    NotPositiveDefiniteError for a failed pivot."""
    if a.dim() != 2 or a.shape[0] != a.shape[1] or a.dtype != torch.float32 or not a.is_cuda:
        raise ShapeError("cholesky_f32_tc needs a square fp32 CUDA matrix")
    if a.stride(1) != 1 or a.stride(0) % 4:
        raise ShapeError("cholesky_f32_tc needs a row-major matrix with 16-byte rows")
    lib = _lib.lib()
    n = a.shape[0]
    if ws is None:
        ws = F32TcWorkspace(n, bs, a.device)
    if ws.n != n or ws.bs != bs or ws.device != a.device:
        raise ShapeError("workspace was made for another order, block size or device")
    main = torch.cuda.current_stream(a.device)
    side = ws.side if lookahead else main
    tree = diag_tree if diag_tree is not None else parse_tree(json.dumps(DIAG_TREE))
    levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
    arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
    kp, info = ws.kp, ws.info
    ld = 4 * kp
    nblk = (n + bs - 1) // bs
    info.fill_(-1)

    def diag_and_panel(k: int, stream: torch.cuda.Stream) -> None:
        k0 = k * bs
        b = min(bs, n - k0)
        r = n - k0 - b
        sh = stream.cuda_stream
        with torch.cuda.stream(stream):
            d32, dd = a[k0:k0 + b, k0:k0 + b], ws.d64[:b, :b]
            _lib.check(lib.bf_convert_f32_f64(ctypes.byref(_v(d32)), ctypes.byref(_v(dd)), 1, sh), "convert")
            ws.before.copy_(info)
            _lib.check(lib.bf_cholesky_d(ctypes.byref(_v(dd)), arr, len(levels), info.data_ptr(), sh), "diag factor")
            torch.where((ws.before < 0) & (info >= 0), info + k0, info, out=info)
            _lib.check(lib.bf_convert_f64_f32(ctypes.byref(_v(dd)), ctypes.byref(_v(d32)), 1, sh), "convert")
            if r == 0:
                return
            x = ws.x64[:b, :b]
            x.zero_()
            x.diagonal().fill_(1.0)  # X L11^T = I: X = L11^-T
            _lib.check(lib.bf_trsm_rltn_d(1.0, ctypes.byref(_v(dd)), ctypes.byref(_v(x)), 512, None, sh), "inverse")
            x32 = ws.x32[:b, :b]
            _lib.check(lib.bf_convert_f64_f32(ctypes.byref(_v(x)), ctypes.byref(_v(x32)), 0, sh), "convert")
            a21 = a[k0 + b:, k0:k0 + b]
            # L21 = A21 X (3xTF32), then its split for the trailing updates
            _lib.check(lib.bf_gemm_f32_tc(1.0, ctypes.byref(_v(a21)), ctypes.byref(_v(x32)), 0.0,
                                          ctypes.byref(_v(a21)), 0, sh), "panel gemm")
            p = ws.pbuf[k % 2]
            _lib.check(lib.bf_split_tf32_s(ctypes.byref(_v(a21)), p.data_ptr(), ld, kp, sh), "split")

    def syrk(p: torch.Tensor, c: torch.Tensor, lower: int) -> None:
        # C -= P P^T with A' = p[:, 0:3kp], B' = p[:, kp:4kp]
        _lib.check(lib.bf_gemm_tf32(-1.0, p.data_ptr(), ld, p[:, kp:].data_ptr(), ld, 1.0, ctypes.byref(_v(c)),
                                    3 * kp, lower, main.cuda_stream), "trailing gemm")

    if lookahead:
        side.wait_stream(main)
    diag_and_panel(0, side)
    ev = torch.cuda.Event()
    ev.record(side)
    for k in range(nblk - 1):
        k1 = (k + 1) * bs
        r = n - k1
        nb = min(bs, r)
        main.wait_event(ev)
        pk = ws.pbuf[k % 2][: n - k * bs - bs]
        # (1) the next block column first (its diagonal block lower-only: the
        # strict upper triangle is never written), (2) the next panel on the
        # side stream, (3) the rest
        syrk(pk[:nb], a[k1:k1 + nb, k1:k1 + nb], 1)
        if r > nb:
            _lib.check(lib.bf_gemm_tf32(-1.0, pk[nb:].data_ptr(), ld, pk[:nb, kp:].data_ptr(), ld, 1.0,
                                        ctypes.byref(_v(a[k1 + nb:, k1:k1 + nb])), 3 * kp, 0, main.cuda_stream),
                       "column gemm")
        if lookahead:
            side.wait_stream(main)
        diag_and_panel(k + 1, side)
        ev = torch.cuda.Event()
        ev.record(side)
        if r > nb:
            syrk(pk[nb:], a[k1 + nb:, k1 + nb:], 1)
    main.wait_event(ev)
    bad = int(info.item())
    if bad >= 0:
        raise NotPositiveDefiniteError(bad)
    return info
