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
import os
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
    lookahead: Optional[bool] = None,
) -> int:
    """Factor the block-cyclic lower triangle held in `local` (this rank's
    local matrix) in place.  Returns -1 or the first failing global pivot
    (and raises NotPositiveDefiniteError if raise_on_failure).

    lookahead (default: on for CUDA tensors): step k's trailing update first
    refreshes block column k+1; step k+1's panel work (diagonal factor, its
    broadcast, the panel solve, the panel broadcasts) then runs on a
    high-priority stream while the rest of step k's update proceeds, so the
    NCCL traffic and the latency-bound panel kernels hide under the GEMMs.
    Every element still receives the same operations in the same order (bits
    unchanged); after a pivot failure only the reported index is defined
    (kernels of the overlapped update may stop early)."""
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
    if lookahead is None:
        lookahead = local.is_cuda
    lookahead = bool(lookahead) and local.is_cuda and layout.tiles > 1
    main = torch.cuda.current_stream(dev) if local.is_cuda else None
    side = torch.cuda.Stream(dev, priority=-1) if lookahead else None

    def panel(k: int) -> list:
        """Steps 1-3 of step k; returns the received panel blocks per process row."""
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
                buf = local[r0:r0 + h, c0k:c0k + bk]
                if comm.world > 1:  # NCCL sends a dense buffer; alone, the strided view serves as is
                    buf = buf.contiguous()
            else:
                buf = torch.empty((h, bk), dtype=local.dtype, device=dev)
            comm.bcast(buf, root)
            panels.append((buf, rows_p[qp:]))
        return panels

    def update(k: int, panels: list, part: str) -> None:
        """Step 4 of step k on my lower tiles: part 'next' = block column k+1
        only, 'rest' = columns beyond it, 'all' = both."""

        def panel_tile(t: int) -> torch.Tensor:
            buf, tiles = panels[t % pr]
            off = (t // pr - tiles[0] // pr) * nb
            return buf[off:off + layout.tile_len(t)]

        def _stack(tiles: list) -> torch.Tensor:
            """Panel rows of consecutive local row tiles (one process row):
            a contiguous slice of that row's received block."""
            first = panel_tile(tiles[0])
            buf = panels[tiles[0] % pr][0]
            off = first.data_ptr() - buf.data_ptr()
            start = off // (buf.element_size() * buf.stride(0))
            h = sum(layout.tile_len(t) for t in tiles)
            return buf[start:start + h]

        q0 = layout.first_row_tile_after(prow, k)
        qc0 = layout.first_col_tile_after(pcol, k)
        cols = my_cols[qc0:]
        if part == "next":
            cols = [j for j in cols if j == k + 1]
        elif part == "rest":
            cols = [j for j in cols if j != k + 1]
        if not cols or q0 >= len(my_rows):
            return
        rows = my_rows[q0:]
        c_base = layout.local_col(cols[0])
        r_base = layout.local_row(rows[0])
        if part == "next":
            # one column tile: GEMMT on the diagonal tile (when it is mine),
            # ONE GEMM over all the stacked rows below it
            bj = panel_tile(cols[0])
            w = layout.tile_len(cols[0])
            r = r_base
            if rows[0] == cols[0]:
                h = layout.tile_len(rows[0])
                ops.gemm(panel_tile(rows[0]), bj, local[r:r + h, c_base:c_base + w], True, kc, info)
                r += h
                rows = rows[1:]
            if rows:
                h = sum(layout.tile_len(t) for t in rows)
                ops.gemm(_stack(rows), bj, local[r:r + h, c_base:c_base + w], False, kc, info)
            return
        if pr == 1 and pc == 1:  # one rank: the trailing block is a plain lower triangle
            rows = [t for t in rows if t >= cols[0]]
            r_base = layout.local_row(rows[0])
            h = sum(layout.tile_len(t) for t in rows)
            st = _stack(rows)
            ops.gemm(st, st, local[r_base:r_base + h, c_base:c_base + h], True, kc, info)
            return
        # my column tiles J (stacked): the B operand of every row's update
        q_stack = torch.cat([panel_tile(j) for j in cols], dim=0)
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

    if not lookahead and os.environ.get("BF_DIST_FORCE_SPLIT") == "1":
        # test hook: the lookahead's split update order without streams
        for k in range(layout.tiles):
            cur = panel(k)
            if k + 1 < layout.tiles:
                update(k, cur, "next")
                update(k, cur, "rest")
            else:
                update(k, cur, "all")
    elif not lookahead:
        for k in range(layout.tiles):
            update(k, panel(k), "all")
    else:
        side.wait_stream(main)
        with torch.cuda.stream(side):
            cur = panel(0)
        ready = torch.cuda.Event()
        ready.record(side)
        for k in range(layout.tiles):
            main.wait_event(ready)
            for item in cur:  # received on the side stream, read on main
                if item is not None:
                    item[0].record_stream(main)
            if k + 1 < layout.tiles:
                update(k, cur, "next")
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    nxt = panel(k + 1)
                ready = torch.cuda.Event()
                ready.record(side)
                update(k, cur, "rest")
                cur = nxt
            else:
                update(k, cur, "all")
        main.wait_stream(side)
    bad = int(info.item())
    if bad >= 0 and raise_on_failure:
        raise NotPositiveDefiniteError(bad)
    return bad
