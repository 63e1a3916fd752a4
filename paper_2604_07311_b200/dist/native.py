"""Python front end of the native multi-GPU Cholesky (csrc/dist.cu,
bf_dist_* / bf_chol_dist_d in include/blockfam_b200.h).

One process per GPU.  `DistContext` wraps a bf_dist handle: NCCL world
communicator from an ncclUniqueId (shared through torch.distributed when it is
initialised — gloo or nccl, only the 128-byte id travels), split into row and
column communicators inside the library.  The per-step loop, the streams, the
receive buffers and every NCCL call live in C++; torch only carries the local
storage tensor.

Storage is the lower column-panel layout of csrc/dist_layout.h (mirrored by
dist/layout.py LowerPanels): a rank holds only its lower tiles, so the C3
configuration (n = 131072, 69 GB of lower triangle) fits on 2/4/8 GPUs with
no rank ever holding the whole matrix — `fill_synthetic` generates each
rank's tiles on the rank.

`cholesky_replicated` is the drop-in for the reference call
`cholesky(a, "lower", tree)` with root `ways` = world size
(factor/cholesky.py:128-149 threads `ways` into every level-3 call): every
rank passes the same full matrix, the tiles are factored distributed and
every rank gets the whole factor back.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from ..control import ControlNode, check_valid, flatten_cholesky, resolve_config
from ..engine import _lib
from ..errors import DeviceError, NotPositiveDefiniteError, ShapeError
from ..views import DType
from .layout import LowerPanels, grid_for

__all__ = ["DistContext", "cholesky_dist", "fill_synthetic", "cholesky_replicated", "selftest_single_rank"]


@dataclass
class DistContext:
    handle: int
    rank: int
    world: int
    pr: int
    pc: int

    @classmethod
    def create(cls, rank: int, world: int, unique_id: bytes, grid: Optional[tuple[int, int]] = None) -> "DistContext":
        lib = _lib.lib()
        if not lib.bf_dist_available():
            raise DeviceError("NCCL (libnccl.so.2) could not be loaded: the distributed path is unavailable")
        pr, pc = grid or grid_for(world)
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), len(unique_id))
        _lib.check(lib.bf_dist_init(buf, rank, world, pr, pc, ctypes.byref(h)), "bf_dist_init")
        return cls(h.value, rank, world, pr, pc)

    @classmethod
    def from_torch_distributed(cls, grid: Optional[tuple[int, int]] = None, group=None) -> "DistContext":
        """Every rank of the (initialised) default process group: rank 0 makes
        the NCCL id, torch.distributed carries it to the others."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.create(rank, world, obj[0], grid)

    @classmethod
    def single(cls) -> "DistContext":
        """A one-rank context (1x1 grid): the NCCL path on one GPU."""
        return cls.create(0, 1, unique_id(), (1, 1))

    def set_option(self, name: str, value: int) -> None:
        _lib.check(_lib.lib().bf_dist_set_option(self.handle, name.encode(), int(value)), "bf_dist_set_option")

    def layout(self, n: int, nb: int) -> LowerPanels:
        return LowerPanels(n, nb, self.pr, self.pc, self.rank)

    def close(self) -> None:
        if self.handle:
            _lib.lib().bf_dist_finalize(self.handle)
            self.handle = 0


def unique_id() -> bytes:
    lib = _lib.lib()
    nbytes = lib.bf_dist_unique_id_bytes()
    buf = ctypes.create_string_buffer(nbytes)
    _lib.check(lib.bf_dist_unique_id(buf), "bf_dist_unique_id")
    return buf.raw


def _levels(tree: ControlNode):
    check_valid(tree, op="cholesky")
    if tree.variant != 3 or not tree.bs:
        raise ShapeError("the distributed Cholesky needs a variant-3 root (its bs is the tile size)")
    levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
    return (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, bs, kc) for v, bs, kc in levels]), len(levels)


def cholesky_dist(ctx: DistContext, local: torch.Tensor, n: int, tree: ControlNode,
                  raise_on_failure: bool = True) -> int:
    """Factor this rank's lower panels (`local`, 1-D fp64 CUDA, LowerPanels
    layout for nb = tree.bs) in place; every rank returns the same pivot flag."""
    arr, nl = _levels(tree)
    lp = ctx.layout(n, tree.bs)
    if local.dtype != torch.float64 or not local.is_cuda or local.numel() < lp.local_elems():
        raise ShapeError(f"local storage must be fp64 CUDA with >= {lp.local_elems()} elements")
    info = torch.full((1,), -1, dtype=torch.int32, device=local.device)
    rc = _lib.lib().bf_chol_dist_d(ctx.handle, local.data_ptr(), n, arr, nl, info.data_ptr(),
                                   _lib.stream_ptr(local.device))
    _lib.check(rc, "bf_chol_dist_d")
    bad = int(info.item())
    if bad >= 0 and raise_on_failure:
        raise NotPositiveDefiniteError(bad)
    return bad


def fill_synthetic(ctx: DistContext, local: torch.Tensor, n: int, nb: int, seed: int = 42) -> None:
    """This rank's tiles of the synthetic SPD matrix (bf_dist_fill_synthetic_d)."""
    rc = _lib.lib().bf_dist_fill_synthetic_d(n, nb, ctx.pr, ctx.pc, ctx.rank, local.data_ptr(), seed,
                                             _lib.stream_ptr(local.device))
    _lib.check(rc, "bf_dist_fill_synthetic_d")


def fill_synthetic_full(a: torch.Tensor, seed: int = 42) -> None:
    """The same matrix as a full n x n tensor (one-GPU comparisons)."""
    from ..views import from_torch

    v = _lib.as_bfview(from_torch(a))
    _lib.check(_lib.lib().bf_fill_synthetic_d(ctypes.byref(v), seed, _lib.stream_ptr(a.device)), "bf_fill_synthetic_d")


def _panel_index(lp: LowerPanels, device) -> list[tuple[torch.Tensor, int, int, int]]:
    out = []
    for J, i0, h, w, off in lp.panels():
        r = np.arange(h)
        rows = (lp.prow + (i0 + r // lp.nb) * lp.pr) * lp.nb + r % lp.nb
        out.append((torch.as_tensor(rows, device=device), J * lp.nb, w, off))
    return out


def scatter_local(lp: LowerPanels, full: torch.Tensor) -> torch.Tensor:
    """Device gather of this rank's lower panels out of a full matrix."""
    local = torch.empty(lp.local_elems(), dtype=full.dtype, device=full.device)
    for rows, c0, w, off in _panel_index(lp, full.device):
        local[off:off + rows.numel() * w].view(-1, w).copy_(full[rows, c0:c0 + w])
    return local


def gather_local(lp: LowerPanels, local: torch.Tensor, full: torch.Tensor) -> None:
    for rows, c0, w, off in _panel_index(lp, full.device):
        full[rows, c0:c0 + w] = local[off:off + rows.numel() * w].view(-1, w)


def cholesky_replicated(full: torch.Tensor, tree: ControlNode, ctx: DistContext) -> int:
    """Every rank holds the same n x n matrix; factor it over ctx's ranks and
    leave the full factor (lower triangle) on every rank.  Returns the pivot
    flag (NotPositiveDefiniteError is raised by the caller)."""
    import torch.distributed as dist

    n = full.shape[0]
    lp = ctx.layout(n, tree.bs)
    local = scatter_local(lp, full)
    bad = cholesky_dist(ctx, local, n, tree, raise_on_failure=False)
    for r in range(ctx.world):  # every rank's panels to every rank
        lr = LowerPanels(n, tree.bs, ctx.pr, ctx.pc, r)
        buf = local if r == ctx.rank else torch.empty(lr.local_elems(), dtype=full.dtype, device=full.device)
        if ctx.world > 1:
            dist.broadcast(buf, src=r)
        gather_local(lr, buf, full)
    return bad


def selftest_single_rank(n: int = 640, nb: int = 128, seed: int = 7, kc: Optional[int] = None,
                         options: Optional[dict] = None) -> None:
    """The NCCL driver on a 1x1 grid against the one-GPU driver, bitwise
    (`options`: bf_dist_set_option settings, e.g. {"grouped": 0})."""
    from ..control import parse_tree_dict
    from ..factor.cholesky import cholesky
    from ..views import from_torch

    tree = parse_tree_dict({"op": "cholesky", "variant": 3, "bs": nb, "kernel": {"kc": kc or nb},
                            "child": {"op": "cholesky", "variant": 3, "bs": 32, "kernel": {"kc": 32},
                                      "child": {"op": "cholesky", "variant": "unblocked3"}}})
    ctx = DistContext.single()
    try:
        for name, value in (options or {}).items():
            ctx.set_option(name, value)
        lp = ctx.layout(n, nb)
        local = torch.empty(lp.local_elems(), dtype=torch.float64, device="cuda")
        fill_synthetic(ctx, local, n, nb, seed)
        cholesky_dist(ctx, local, n, tree)
        full = torch.empty(n, n, dtype=torch.float64, device="cuda")
        fill_synthetic_full(full, seed)
        cholesky(from_torch(full), "lower", tree)
        ref = scatter_local(lp, full)
        if not torch.equal(ref, local):
            raise AssertionError("NCCL driver (1x1) differs from the one-GPU factor")
    finally:
        ctx.close()
