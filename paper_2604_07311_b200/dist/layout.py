"""2D block-cyclic layout of a symmetric matrix over a Pr x Pc process grid.

Tile (I, J) of size nb x nb (the root block size of the Cholesky tree; the
last tile may be short) belongs to rank (I mod Pr) * Pc + (J mod Pc).  Each
rank stores its tiles densely in a local row-major matrix whose row blocks are
its tile rows I (in increasing order) and whose column blocks are its tile
columns J — the ScaLAPACK arrangement, so every contiguous range of local tile
rows or columns is a plain strided view the engine consumes directly.  Only
tiles with I >= J carry data (the lower triangle); the others are storage the
factorization never touches.  (the reference has no
distribution.)
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

__all__ = ["BlockCyclic2D", "grid_for"]


def grid_for(p: int) -> tuple[int, int]:
    """Process grid for p GPUs: 1 -> 1x1, 2 -> 2x1, 4 -> 2x2, 8 -> 4x2, else
    the most square Pr x Pc with Pr >= Pc.  Taller grids split each step's
    panel TRSM (rows I > k, the heaviest part of the panel chain: n_k x nb^2
    flops) over Pr ranks; every rank still receives the whole panel once."""
    if p < 1:
        raise ValueError("need at least one process")
    pc = int(np.sqrt(p))
    while p % pc:
        pc -= 1
    return p // pc, pc


@dataclass(frozen=True)
class BlockCyclic2D:
    n: int
    nb: int
    pr: int
    pc: int

    def __post_init__(self) -> None:
        if self.n < 0 or self.nb < 1 or self.pr < 1 or self.pc < 1:
            raise ValueError("invalid block-cyclic layout")

    @property
    def nprocs(self) -> int:
        return self.pr * self.pc

    @cached_property
    def tiles(self) -> int:
        return -(-self.n // self.nb) if self.n else 0

    def tile_len(self, t: int) -> int:
        return min(self.nb, self.n - t * self.nb)

    def owner(self, i_tile: int, j_tile: int) -> int:
        return (i_tile % self.pr) * self.pc + (j_tile % self.pc)

    def coords(self, rank: int) -> tuple[int, int]:
        return divmod(rank, self.pc)

    def row_tiles(self, prow: int) -> list[int]:
        return list(range(prow, self.tiles, self.pr))

    def col_tiles(self, pcol: int) -> list[int]:
        return list(range(pcol, self.tiles, self.pc))

    def local_shape(self, rank: int) -> tuple[int, int]:
        prow, pcol = self.coords(rank)
        return (sum(self.tile_len(t) for t in self.row_tiles(prow)),
                sum(self.tile_len(t) for t in self.col_tiles(pcol)))

    def local_row(self, i_tile: int) -> int:
        """Local element row where global tile row i_tile starts (on its owners)."""
        return (i_tile // self.pr) * self.nb

    def local_col(self, j_tile: int) -> int:
        return (j_tile // self.pc) * self.nb

    def first_row_tile_after(self, prow: int, k: int) -> int:
        """Index (into row_tiles(prow)) of the first tile row > k."""
        rt = self.row_tiles(prow)
        return next((q for q, t in enumerate(rt) if t > k), len(rt))

    def first_col_tile_after(self, pcol: int, k: int) -> int:
        ct = self.col_tiles(pcol)
        return next((q for q, t in enumerate(ct) if t > k), len(ct))

    # -- host-side scatter / gather (tests, data loading) ---------------------
    def scatter(self, full: np.ndarray, rank: int) -> np.ndarray:
        prow, pcol = self.coords(rank)
        lr, lc = self.local_shape(rank)
        out = np.zeros((lr, lc), dtype=full.dtype)
        for i in self.row_tiles(prow):
            for j in self.col_tiles(pcol):
                r0, c0 = self.local_row(i), self.local_col(j)
                h, w = self.tile_len(i), self.tile_len(j)
                out[r0:r0 + h, c0:c0 + w] = full[i * self.nb:i * self.nb + h, j * self.nb:j * self.nb + w]
        return out

    def gather(self, locals_: list[np.ndarray], fill: np.ndarray | None = None) -> np.ndarray:
        """Reassemble the lower tiles (I >= J) into a full matrix (others from fill)."""
        dtype = locals_[0].dtype
        full = np.zeros((self.n, self.n), dtype=dtype) if fill is None else fill.copy()
        for rank, loc in enumerate(locals_):
            prow, pcol = self.coords(rank)
            for i in self.row_tiles(prow):
                for j in self.col_tiles(pcol):
                    if i < j:
                        continue
                    r0, c0 = self.local_row(i), self.local_col(j)
                    h, w = self.tile_len(i), self.tile_len(j)
                    full[i * self.nb:i * self.nb + h, j * self.nb:j * self.nb + w] = loc[r0:r0 + h, c0:c0 + w]
        return full


@dataclass(frozen=True)
class LowerPanels:
    """Lower column-panel storage of one rank (mirror of csrc/dist_layout.h, the
    layout the native NCCL driver bf_chol_dist_d factors).

    Rank (prow, pcol) keeps, for each of its column tiles J = pcol + q*pc, ONE
    row-major panel holding its row tiles I >= J stacked (leading dimension
    tile_len(J)); panels follow each other in q order.  Only lower tiles are
    stored: about n^2 / (2P) elements per rank."""

    n: int
    nb: int
    pr: int
    pc: int
    rank: int

    @property
    def base(self) -> BlockCyclic2D:
        return BlockCyclic2D(self.n, self.nb, self.pr, self.pc)

    @property
    def prow(self) -> int:
        return self.rank // self.pc

    @property
    def pcol(self) -> int:
        return self.rank % self.pc

    def first_row_geq(self, p: int, t: int) -> int:
        return 0 if t <= p else (t - p + self.pr - 1) // self.pr

    def rows_of(self, p: int, i0: int, i1: int) -> int:
        b = self.base
        return sum(b.tile_len(p + i * self.pr) for i in range(i0, i1))

    def panels(self) -> list[tuple[int, int, int, int, int]]:
        """[(J, first local row-tile index, height, width, element offset)]."""
        b = self.base
        out, off = [], 0
        nrt = len(b.row_tiles(self.prow))
        for J in b.col_tiles(self.pcol):
            i0 = self.first_row_geq(self.prow, J)
            h, w = self.rows_of(self.prow, i0, nrt), b.tile_len(J)
            out.append((J, i0, h, w, off))
            off += h * w
        return out

    def local_elems(self) -> int:
        return sum(h * w for _, _, h, w, _ in self.panels())

    def _rows(self, i0: int, h: int) -> np.ndarray:
        """Global row indices of a panel's h rows starting at local row tile i0."""
        r = np.arange(h)
        return (self.prow + (i0 + r // self.nb) * self.pr) * self.nb + r % self.nb

    def scatter(self, full: np.ndarray) -> np.ndarray:
        out = np.zeros(self.local_elems(), dtype=full.dtype)
        for J, i0, h, w, off in self.panels():
            rows = self._rows(i0, h)
            out[off:off + h * w] = full[rows, J * self.nb:J * self.nb + w].reshape(-1)
        return out

    def gather_into(self, local: np.ndarray, full: np.ndarray) -> None:
        for J, i0, h, w, off in self.panels():
            rows = self._rows(i0, h)
            full[rows, J * self.nb:J * self.nb + w] = local[off:off + h * w].reshape(h, w)
