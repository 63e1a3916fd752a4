// 2D block-cyclic layout of the LOWER triangle of an n x n matrix over a
// Pr x Pc process grid, stored as lower column panels (the
// reference has no distribution).
//
// Tiles are nb x nb (nb = the root block size of the control tree; only the
// last tile is short).  Tile (I, J) with I >= J belongs to rank
// (I mod Pr) * Pc + (J mod Pc).  Rank (prow, pcol) owns row tiles
// I = prow + i*Pr and column tiles J = pcol + q*Pc.  For each of its column
// tiles J it stores ONE dense row-major panel: its row tiles I >= J stacked
// (a suffix of its row tiles), width tile_len(J), leading dimension
// tile_len(J).  Panels follow each other in q order.  So a rank holds only
// lower tiles (about n^2 / (2 P) elements), every panel is a plain strided
// view, and the rows of a panel below any tile are contiguous in memory — the
// panel column a rank broadcasts is its own storage, sent in place.
//
// Header-only, plain C++: shared by the CUDA/NCCL driver (dist.cu) and the
// CPU schedule harness of the tests (tests/dist_harness.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace bf {

struct DistLayout {
  int64_t n = 0, nb = 1;
  int pr = 1, pc = 1, prow = 0, pcol = 0;
  std::vector<int64_t> panel_off;  // element offset of each local column panel (+ total at the end)

  DistLayout() = default;
  DistLayout(int64_t n_, int64_t nb_, int pr_, int pc_, int rank) : n(n_), nb(nb_), pr(pr_), pc(pc_) {
    prow = rank / pc;
    pcol = rank % pc;
    const int64_t nq = col_tiles(pcol);
    panel_off.assign(size_t(nq) + 1, 0);
    for (int64_t q = 0; q < nq; ++q) panel_off[size_t(q) + 1] = panel_off[size_t(q)] + panel_h(q) * panel_w(q);
  }

  int64_t tiles() const { return n > 0 ? (n + nb - 1) / nb : 0; }
  int64_t tile_len(int64_t t) const { return n - t * nb < nb ? n - t * nb : nb; }
  int owner(int64_t I, int64_t J) const { return int(I % pr) * pc + int(J % pc); }
  // number of row tiles of process row p / column tiles of process column q
  int64_t row_tiles(int p) const { return p < tiles() ? (tiles() - 1 - p) / pr + 1 : 0; }
  int64_t col_tiles(int q) const { return q < tiles() ? (tiles() - 1 - q) / pc + 1 : 0; }
  // first local row-tile index i of process row p with p + i*pr >= t
  int64_t first_row_geq(int p, int64_t t) const { return t <= p ? 0 : (t - p + pr - 1) / pr; }
  // rows held by local row tiles [i0, i1) of process row p
  int64_t rows_of(int p, int64_t i0, int64_t i1) const {
    if (i1 <= i0) return 0;
    int64_t r = (i1 - i0) * nb;
    const int64_t last = p + (i1 - 1) * pr;
    if (last == tiles() - 1) r -= nb - tile_len(last);
    return r;
  }
  // local column panel q: global column tile J, height (rows I >= J), width
  int64_t panel_J(int64_t q) const { return pcol + q * pc; }
  int64_t panel_i0(int64_t q) const { return first_row_geq(prow, panel_J(q)); }
  int64_t panel_h(int64_t q) const { return rows_of(prow, panel_i0(q), row_tiles(prow)); }
  int64_t panel_w(int64_t q) const { return tile_len(panel_J(q)); }
  int64_t local_elems() const { return panel_off.empty() ? 0 : panel_off.back(); }
  // rows of process row p's stacked panel at step k (its row tiles I > k)
  int64_t stack_first(int p, int64_t k) const { return first_row_geq(p, k + 1); }
  int64_t stack_rows(int p, int64_t k) const { return rows_of(p, stack_first(p, k), row_tiles(p)); }
  // capacity (rows) of a receive buffer for process row p's stacked panels
  int64_t stack_cap(int p) const { return rows_of(p, 0, row_tiles(p)); }
};

}  // namespace bf
