"""Distributed right-looking Cholesky over a 2D block-cyclic process grid.

One process per GPU; torch.distributed carries the panel broadcasts (NCCL over
NVLink on B200).  The root of the control tree must be variant 3 with
bs == layout.nb; its child tree factors each diagonal tile.  Per step k:

  1. the owner of tile (k,k) factors it with the child tree (same kernels and
     operation order as the single-GPU driver) and broadcasts L_kk together
     with its device pivot flag (so every rank's kernels stop after a failure
     without any host synchronisation);
  2. the ranks of process column k mod Pc solve their panel tiles
     L_Ik = A_Ik L_kk^-T (I > k) — rows are independent, so splitting them
     across ranks changes nothing in the arithmetic;
  3. every process-column-k rank broadcasts its stacked panel tiles;
  4. every rank applies A_IJ -= L_Ik L_Jk^T to its lower tiles (I >= J > k):
     GEMM (K = nb, the root's kc segments) off the diagonal, GEMMT on it.

Each element therefore receives exactly the single-GPU sequence of folds, so
the distributed factor is bit-identical to bf.cholesky on one GPU.

`ops` is the compute backend (default: the sm_100a C ABI); `comm` the
transport.  Tests substitute CPU stand-ins for both to exercise this host
logic under gloo without a GPU.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Protocol

import torch

from ..control import ControlNode, check_valid, flatten_cholesky, resolve_config
from ..errors import NotPositiveDefiniteError, ShapeError
from ..views import DType
from .layout import BlockCyclic2D

__all__ = ["Comm", "Ops", "TorchComm", "B200Ops", "cholesky_distributed"]


class Comm(Protocol):
    rank: int
    world: int

    def bcast(self, t: torch.Tensor, root: int) -> None: ...


class Ops(Protocol):
    def potrf(self, tile: torch.Tensor, levels: list, base: int, info: torch.Tensor) -> None: ...

    def trsm(self, tri: torch.Tensor, b: torch.Tensor, kc: int, info: torch.Tensor) -> None: ...

    def gemm(self, a: torch.Tensor, bt: torch.Tensor, c: torch.Tensor, lower: bool, kc: int,
             info: torch.Tensor) -> None: ...


class TorchComm:
    """torch.distributed broadcast on the default group (NCCL device tensors on
    B200, gloo CPU tensors in tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def bcast(self, t: torch.Tensor, root: int) -> None:
        if self.world > 1:
            self._dist.broadcast(t, src=root, group=self.group)


class B200Ops:
    """The sm_100a library: views are 2-D (strided) CUDA tensors."""

    def __init__(self) -> None:
        from ..engine import _lib

        self._lib = _lib

    def _view(self, t: torch.Tensor):
        from ..views import from_torch

        return self._lib.as_bfview(from_torch(t))

    def _stream(self, t: torch.Tensor) -> int:
        return torch.cuda.current_stream(t.device).cuda_stream

    def potrf(self, tile, levels, base, info) -> None:
        lib = self._lib.lib()
        arr = (self._lib.BfCholLevel * len(levels))(*[self._lib.BfCholLevel(v, 0, bs, kc) for v, bs, kc in levels])
        v = self._view(tile)
        rc = lib.bf_cholesky_ex_d(ctypes.byref(v), arr, len(levels), int(base), info.data_ptr(), self._stream(tile))
        self._lib.check(rc, "distributed potrf")

    def trsm(self, tri, b, kc, info) -> None:
        # abort-only flag: a Cholesky diagonal is sqrt(d > 0) > 0, never singular
        lib = self._lib.lib()
        vt, vb = self._view(tri), self._view(b)
        rc = lib.bf_trsm_rltn_ex_d(1.0, ctypes.byref(vt), ctypes.byref(vb), int(kc), None, info.data_ptr(),
                                   self._stream(b))
        self._lib.check(rc, "distributed trsm")

    def gemm(self, a, bt, c, lower, kc, info) -> None:
        lib = self._lib.lib()
        va, vb, vc = self._view(a), self._view(bt.t()), self._view(c)
        rc = lib.bf_gemm_d(-1.0, ctypes.byref(va), ctypes.byref(vb), 1.0, ctypes.byref(vc), int(lower), int(kc),
                           info.data_ptr(), self._stream(c))
        self._lib.check(rc, "distributed gemm")


def cholesky_distributed(
    local: torch.Tensor,
    layout: BlockCyclic2D,
    tree: ControlNode,
    comm: Comm,
    ops: Optional[Ops] = None,
    raise_on_failure: bool = True,
) -> int:
    """Factor the block-cyclic lower triangle held in `local` (this rank's
    local matrix) in place.  Returns -1 or the first failing global pivot
    (and raises NotPositiveDefiniteError if raise_on_failure)."""
    check_valid(tree, op="cholesky")
    if tree.variant != 3 or tree.bs != layout.nb:
        raise ShapeError("distributed Cholesky needs a variant-3 root whose bs equals the tile size nb")
    if local.dim() != 2 or tuple(local.shape) != layout.local_shape(comm.rank):
        raise ShapeError(f"local block {tuple(local.shape)} != layout {layout.local_shape(comm.rank)}")
    ops = ops if ops is not None else B200Ops()
    dtype = DType.F64 if local.dtype == torch.float64 else DType.F32
    levels = flatten_cholesky(tree, resolve_config(tree, dtype))
    child = levels[1:] or [(13, 0, levels[0][2])]
    kc = levels[0][2]
    nb, pr, pc = layout.nb, layout.pr, layout.pc
    prow, pcol = layout.coords(comm.rank)
    dev = local.device
    info = torch.full((1,), -1, dtype=torch.int32, device=dev)
    my_rows, my_cols = layout.row_tiles(prow), layout.col_tiles(pcol)

    for k in range(layout.tiles):
        bk = layout.tile_len(k)
        kr, kcol = k % pr, k % pc
        diag_owner = kr * pc + kcol
        # 1. diagonal tile + pivot flag
        diag = torch.empty((bk, bk), dtype=local.dtype, device=dev)
        if comm.rank == diag_owner:
            r0, c0 = layout.local_row(k), layout.local_col(k)
            tile = local[r0:r0 + bk, c0:c0 + bk]
            ops.potrf(tile, child, k * nb, info)
            diag.copy_(tile)
        comm.bcast(diag, diag_owner)
        comm.bcast(info, diag_owner)
        # 2. panel solve on process column k mod Pc
        q0 = layout.first_row_tile_after(prow, k)
        stacked_rows = sum(layout.tile_len(t) for t in my_rows[q0:])
        c0k = layout.local_col(k) if pcol == kcol else None
        if pcol == kcol and stacked_rows:
            r0 = layout.local_row(my_rows[q0])
            ops.trsm(diag, local[r0:r0 + stacked_rows, c0k:c0k + bk], kc, info)
        # 3. panel broadcast: one stacked block per process row
        panels = []
        for p in range(pr):
            rows_p = layout.row_tiles(p)
            qp = layout.first_row_tile_after(p, k)
            h = sum(layout.tile_len(t) for t in rows_p[qp:])
            root = p * pc + kcol
            if h == 0:
                panels.append(None)
                continue
            if comm.rank == root:
                r0 = layout.local_row(rows_p[qp])
                buf = local[r0:r0 + h, c0k:c0k + bk].contiguous()
            else:
                buf = torch.empty((h, bk), dtype=local.dtype, device=dev)
            comm.bcast(buf, root)
            panels.append((buf, rows_p[qp:]))

        def panel_tile(t: int) -> torch.Tensor:
            buf, tiles = panels[t % pr]
            off = (t // pr - tiles[0] // pr) * nb
            return buf[off:off + layout.tile_len(t)]

        # my column tiles J > k, stacked (the B operand of every row's update)
        qc0 = layout.first_col_tile_after(pcol, k)
        cols = my_cols[qc0:]
        if not cols or q0 >= len(my_rows):
            continue
        q_stack = torch.cat([panel_tile(j) for j in cols], dim=0)
        c_base = layout.local_col(cols[0])
        # 4. trailing update of my lower tiles
        for i_tile in my_rows[q0:]:
            n_cols = sum(1 for j in cols if j <= i_tile)
            if n_cols == 0:
                continue
            a_i = panel_tile(i_tile)
            r0, h = layout.local_row(i_tile), layout.tile_len(i_tile)
            diag_here = cols[n_cols - 1] == i_tile
            n_full = n_cols - 1 if diag_here else n_cols
            w_full = sum(layout.tile_len(j) for j in cols[:n_full])
            if n_full:
                ops.gemm(a_i, q_stack[:w_full], local[r0:r0 + h, c_base:c_base + w_full], False, kc, info)
            if diag_here:
                ops.gemm(a_i, q_stack[w_full:w_full + h], local[r0:r0 + h, c_base + w_full:c_base + w_full + h],
                         True, kc, info)
    bad = int(info.item())
    if bad >= 0 and raise_on_failure:
        raise NotPositiveDefiniteError(bad)
    return bad
