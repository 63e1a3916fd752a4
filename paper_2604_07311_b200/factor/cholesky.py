"""The Cholesky family on B200 (reference factor/cholesky.py:1-158).

Three blocked variants (1 bordered, 2 left-looking, 3 right-looking) and
three unblocked leaves, nested through a control tree:

  variant 1: A10 := A10*tril(A00)^-T ; A11 -= A10*A10^T ; A11 := chol(A11)
  variant 2: A11 -= A10*A10^T ; A11 := chol(A11) ; A21 -= A20*A10^T ;
             A21 := A21*tril(A11)^-T
  variant 3: A11 := chol(A11) ; A21 := A21*tril(A11)^-T ; A22 -= A21*A21^T

`cholesky(a, uplo, tree)` keeps the reference signature and contracts: only
the uplo triangle is touched, "upper" runs the lower algorithm on the
transposed view (so it is bitwise the transpose of "lower"), a failed pivot
raises NotPositiveDefiniteError with the global index.  The default engine
hands the flattened tree to the native driver (bf_cholesky_*), which issues
the same level-3 sequence as `_run` below from C++ with no per-call Python
cost; engine="python" walks the tree here, one C-ABI call per operation.
Both enqueue everything on the current stream and synchronise once, to read
the device pivot flag, at the end.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ..control import ControlNode, check_valid, default_tree, flatten_cholesky, resolve_config
from ..engine import _lib
from ..engine.config import KernelConfig
from ..engine.gemm import _launch_gemm
from ..errors import NotPositiveDefiniteError, ShapeError
from ..views import MatrixView, partition_steps

__all__ = ["cholesky", "cholesky_async", "cholesky_host"]

_LEAF = {"unblocked1": 1, "unblocked2": 2, "unblocked3": 3}


def cholesky(
    a: MatrixView, uplo: str = "lower", tree: Optional[ControlNode] = None, engine: str = "native"
) -> None:
    """In place: tril(a) := L with a = L*L^T (or triu(a) := U, a = U^T*U)."""
    info = cholesky_async(a, uplo, tree, engine)
    bad = int(info.item())
    if bad >= 0:
        raise NotPositiveDefiniteError(bad)


def cholesky_async(
    a: MatrixView, uplo: str = "lower", tree: Optional[ControlNode] = None, engine: str = "native"
) -> torch.Tensor:
    """Enqueue the factorization; return the device pivot flag (-1 = success,
    else the first failing global index).  Nothing is synchronised."""
    if a.m != a.n:
        raise ShapeError(f"square matrix required, got {a.shape}")
    if uplo == "upper":
        a = a.transposed()
    elif uplo != "lower":
        raise ValueError(f"uplo must be 'lower' or 'upper', got {uplo!r}")
    if tree is None:
        tree = default_tree("cholesky", a.n, a.dtype)
    check_valid(tree, op="cholesky")
    cfg = resolve_config(tree, a.dtype)
    info = torch.full((1,), -1, dtype=torch.int32, device=a.device)
    if a.n == 0:
        return info
    _lib.require_cuda(a)
    if engine == "native" and _distributed_ways(tree):
        # root ways = the ranks of the default process group: the tiles are
        # factored over them by the NCCL driver and every rank gets the factor
        from ..dist.native import cholesky_replicated

        full = a.storage.as_strided((a.n, a.n), (a.rs, a.cs), a.offset)
        bad = cholesky_replicated(full, tree, _dist_context())
        info.fill_(bad)
        return info
    if engine == "native":
        levels = flatten_cholesky(tree, cfg)
        arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, bs, kc) for v, bs, kc in levels])
        fn = getattr(_lib.lib(), "bf_cholesky_" + ("d" if a.dtype.value == "f64" else "s"))
        va = _lib.as_bfview(a)
        rc = fn(ctypes.byref(va), arr, len(levels), info.data_ptr(), _lib.stream_ptr(a.device))
        _lib.check(rc, "cholesky")
    elif engine == "python":
        _run(a, tree, cfg, 0, info)
    else:
        raise ValueError(f"unknown engine {engine!r}")
    return info


_DIST_CTX = None


def _distributed_ways(tree: ControlNode) -> bool:
    """Root `ways` > 1 selects the multi-GPU driver when torch.distributed is
    initialised with exactly that many ranks (one process per GPU).  Otherwise
    `ways` keeps its single-GPU meaning: a parallel width the CTA grid already
    covers (results are identical for every width)."""
    ways = tree.ways or 1
    if ways <= 1 or tree.variant != 3 or not tree.bs:
        return False
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized() and dist.get_world_size() == ways


def _dist_context():
    global _DIST_CTX
    if _DIST_CTX is None:
        from ..dist.native import DistContext

        _DIST_CTX = DistContext.from_torch_distributed()
    return _DIST_CTX


# -- the tree walk, operation for operation as factor/cholesky.py:118-158 ---------


def cholesky_host(
    host: torch.Tensor, uplo: str = "lower", tree: Optional[ControlNode] = None,
    work: Optional[torch.Tensor] = None, device: Optional[torch.device] = None,
) -> None:
    """In place on a HOST fp64 matrix (a CPU torch tensor, ideally pinned —
    `torch.empty(..., pin_memory=True)`): the reference's call shape
    (factor/cholesky.py:99-115 factors a NumPy array in place) with the
    compute on the GPU.  Only the lower triangle travels (by block columns),
    and every finished block column returns while later steps still run.
    `work` (n x n fp64 on the device) is reused when given.  Upper is the
    lower algorithm on the transpose, through a host-side transposed copy."""
    if host.device.type != "cpu" or host.dtype != torch.float64 or host.dim() != 2 or host.shape[0] != host.shape[1]:
        raise ShapeError("cholesky_host needs a square fp64 CPU tensor")
    if uplo == "upper":
        t = host.t().contiguous()
        cholesky_host(t, "lower", tree, work, device)
        host.copy_(t.t())
        return
    if uplo != "lower":
        raise ValueError(f"uplo must be 'lower' or 'upper', got {uplo!r}")
    if host.stride(1) != 1:
        raise ShapeError("cholesky_host needs a row-major host matrix")
    n = host.shape[0]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if work is None:
        work = torch.empty((n, n), dtype=torch.float64, device=dev)
    if tuple(work.shape) != (n, n) or work.dtype != torch.float64 or work.stride(1) != 1:
        raise ShapeError("work must be an n x n row-major fp64 device tensor")
    from ..views import DType, from_torch

    if tree is None:
        tree = default_tree("cholesky", n, DType.F64)
    check_valid(tree, op="cholesky")
    levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
    arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, bs, kc) for v, bs, kc in levels])
    info = torch.full((1,), -1, dtype=torch.int32, device=work.device)
    vw = _lib.as_bfview(from_torch(work))
    rc = _lib.lib().bf_cholesky_host_d(host.data_ptr(), host.stride(0), ctypes.byref(vw), arr, len(levels),
                                       info.data_ptr(), _lib.stream_ptr(work.device))
    _lib.check(rc, "cholesky_host")
    bad = int(info.item())
    if bad >= 0:
        # the reference's partial state lives in `work`: bring back its lower triangle
        torch.cuda.synchronize(work.device)
        low = torch.tril(work).cpu()
        host.copy_(torch.where(torch.tril(torch.ones(n, n, dtype=torch.bool)), low, host))
        raise NotPositiveDefiniteError(bad)


def _leaf(a: MatrixView, variant: str, base: int, info: torch.Tensor) -> None:
    fn = getattr(_lib.lib(), "bf_potrf_leaf_" + ("d" if a.dtype.value == "f64" else "s"))
    va = _lib.as_bfview(a)
    rc = fn(ctypes.byref(va), _LEAF[variant], int(base), info.data_ptr(), _lib.stream_ptr(a.device))
    _lib.check(rc, "potrf leaf")


def _trsm(tri: MatrixView, b: MatrixView, cfg: KernelConfig, info: torch.Tensor) -> None:
    # right/lower/trans/non-unit, alpha = 1, aborts once a pivot has failed
    if b.m == 0 or tri.n == 0:
        return
    fn = getattr(_lib.lib(), "bf_trsm_rltn_" + ("d" if b.dtype.value == "f64" else "s"))
    # the native recursion takes one flag for both "singular" and "abort";
    # a Cholesky diagonal is sqrt(d > 0) > 0, so only the abort role is live
    vt, vb = _lib.as_bfview(tri), _lib.as_bfview(b)
    rc = fn(1.0, ctypes.byref(vt), ctypes.byref(vb), int(cfg.kc), info.data_ptr(), _lib.stream_ptr(b.device))
    _lib.check(rc, "trsm")


def _run(a: MatrixView, node: ControlNode, cfg: KernelConfig, base: int, info: torch.Tensor) -> None:
    n = a.n
    if n == 0:
        return
    if not node.is_blocked:
        _leaf(a, str(node.variant), base, info)
        return
    flag = info.data_ptr()
    for step in partition_steps(n, node.bs):
        r0, r1, r2 = step.r0, step.r1, step.r2
        a00 = a.subview(r0, r0)
        a10 = a.subview(r1, r0)
        a11 = a.subview(r1, r1)
        a20 = a.subview(r2, r0)
        a21 = a.subview(r2, r1)
        a22 = a.subview(r2, r2)
        if node.variant == 1:
            _trsm(a00, a10, cfg, info)
            _launch_gemm(-1.0, a10, a10.transposed(), 1.0, a11, cfg, True, flag)
            _recurse(a11, node, cfg, base + r1.start, info)
        elif node.variant == 2:
            _launch_gemm(-1.0, a10, a10.transposed(), 1.0, a11, cfg, True, flag)
            _recurse(a11, node, cfg, base + r1.start, info)
            _launch_gemm(-1.0, a20, a10.transposed(), 1.0, a21, cfg, False, flag)
            _trsm(a11, a21, cfg, info)
        elif node.variant == 3:
            _recurse(a11, node, cfg, base + r1.start, info)
            _trsm(a11, a21, cfg, info)
            _launch_gemm(-1.0, a21, a21.transposed(), 1.0, a22, cfg, True, flag)
        else:
            raise ValueError(f"unknown blocked variant {node.variant!r}")


def _recurse(a11: MatrixView, node: ControlNode, cfg: KernelConfig, base: int, info: torch.Tensor) -> None:
    child = node.child if node.child is not None else ControlNode(op="cholesky", variant="unblocked3")
    _run(a11, child, child.effective_config(cfg), base, info)
