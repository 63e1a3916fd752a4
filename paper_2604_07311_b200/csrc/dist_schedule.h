// Distributed right-looking (variant 3) Cholesky over a 2D block-cyclic grid:
// the per-step schedule, generic over an executor X that supplies the compute
// and the transport.  dist.cu instantiates it with the sm_100a kernels and
// NCCL (row / column communicators from ncclCommSplit, library-owned panel
// stream); tests/dist_harness.cpp instantiates it with the CPU oracle and an
// in-process broadcast so the schedule itself is checked on a CPU.
//
// Per step k (factor/cholesky.py:146-149 at the root, tiles of nb = root bs):
//   (a) the owner of tile (k,k) factors it with the child tree;
//   (b) process column k mod Pc: L_kk and the pivot flag are broadcast down the
//       column communicator from process row k mod Pr;
//   (c) process column k mod Pc: each rank solves its panel rows I > k,
//       L_Ik = A_Ik L_kk^-T (rows independent: the split changes no bits);
//   (d) every process row p: the solved rows of p are broadcast along the row
//       communicator from process column k mod Pc (in place from the root's
//       own panel storage), with the pivot flag;
//   (e) Pr > 1: every process column exchanges the Pr stacked row panels, so
//       each rank holds L_Ik for all I > k;
//   (f) each rank updates its lower tiles A_IJ -= L_Ik L_Jk^T (I >= J > k): per
//       local column panel one GEMMT on the diagonal tile (when it is local)
//       and one GEMM below it, K = nb in the root's kc segments.
// Every element therefore receives exactly the single-GPU sequence of folds:
// the distributed factor is bit-identical to the one-GPU factor for the same
// tree.  With lookahead, step k's update of column panel k+1 runs first, then
// panel k+1 ((a)-(e)) on the panel stream while the rest of step k's update
// proceeds on the main stream (and fan-out streams): the broadcasts and the
// latency-bound panel kernels hide under the GEMMs.  The NCCL calls of one
// communicator are issued in step order on every rank.
#pragma once

#include <cstdint>
#include <vector>

#include "blockfam_b200.h"
#include "dist_layout.h"

namespace bf {

constexpr int DIST_MAX_PR = 64;
enum DistComm { COMM_ROW = 0, COMM_COL = 1 };

// one column panel of a trailing update: c (m x n, ld n) -= a (m x k) * b (n x k)^T,
// a and b row-major with ld k; lower: c's top n x n block is a diagonal tile
// (only its lower triangle is updated)
struct DistGemm {
  const double* a;
  const double* b;
  double* c;
  int64_t m, n;
  int lower;
  int b_proc;  // process row whose stacked rows b points into
};
constexpr int DIST_NOT_GROUPED = 1;  // gemm_groups: "not handled, issue the GEMMs one by one"

struct DistPanels {
  double* ptr[DIST_MAX_PR];  // process row p: stacked solved rows of its tiles I > k (ld = tile width)
  int64_t rows[DIST_MAX_PR];
};

inline bf_view dist_view(double* base, int64_t m, int64_t n, int64_t ld) {
  bf_view v;
  v.base = base;
  v.off = 0;
  v.m = m;
  v.n = n;
  v.rs = ld;
  v.cs = 1;
  return v;
}

// X must provide:
//   using Stream;  Stream main_stream(); Stream panel_stream(); Stream fan_stream(int i); int fan_count();
//   void fork(Stream from, Stream to);                       // `to` waits for work queued so far on `from`
//   int potrf(const bf_view& tile, int64_t base, Stream s);  // child tree of the root on the diagonal tile
//   int trsm(const bf_view& tri, const bf_view& b, Stream s);
//   int gemm(const bf_view& a, const bf_view& bt, const bf_view& c, int lower, int64_t abort_limit,
//            bool reserve, Stream s);                        // c -= a * bt^T
//   int gemm_groups(const DistGemm* g, int ng, const DistPanels& P, int64_t k, int64_t abort_limit,
//                   bool reserve, Stream s);             // all of g in one launch, or DIST_NOT_GROUPED
//   int bcast(int comm, double* buf, int64_t count, int root, Stream s);  // root's buf is sent in place
//   int bcast_info(int comm, int root, Stream s);
//   void group_begin(); int group_end();
//   double* recv_buf(int parity, int p);  // capacity layout.stack_cap(p) * nb
//   void reserve_for(double panel_flops, double update_flops);  // SMs the rest-of-update leaves free
//   double* diag_buf();                   // nb * nb
template <class X>
int chol_dist_schedule(X& x, const DistLayout& L, double* local, bool lookahead) {
  const int64_t T = L.tiles();
  if (T == 0) return BF_OK;
  if (L.pr > DIST_MAX_PR) return BF_ERR_UNSUPPORTED;
  const int64_t nb = L.nb;
  const int prow = L.prow, pcol = L.pcol;
  auto panel_view = [&](int64_t q) {
    return dist_view(local + L.panel_off[size_t(q)], L.panel_h(q), L.panel_w(q), L.panel_w(q));
  };

  // (a)-(e) of step k on stream s; fills P
  auto panel = [&](int64_t k, int parity, DistPanels& P, typename X::Stream s) -> int {
    const int kr = int(k % L.pr), kcol = int(k % L.pc);
    const int64_t bk = L.tile_len(k);
    int rc = BF_OK;
    double* mine = nullptr;  // my process row's stacked rows I > k
    if (pcol == kcol) {
      const int64_t q = k / L.pc;
      bf_view pan = panel_view(q);
      double* D = x.diag_buf();
      int64_t start = 0;
      if (prow == kr) {  // (a) the diagonal tile is the top of my panel q
        D = static_cast<double*>(pan.base);
        rc = x.potrf(dist_view(D, bk, bk, bk), k * nb, s);
        if (rc) return rc;
        start = bk;
      }
      // (b) L_kk (and the flag) down process column kcol
      if (L.pr > 1) {
        x.group_begin();
        rc = x.bcast(COMM_COL, D, bk * bk, kr, s);
        if (!rc) rc = x.bcast_info(COMM_COL, kr, s);
        const int rg = x.group_end();
        if (rc || rg) return rc ? rc : rg;
      }
      // (c) my panel rows below the diagonal
      mine = static_cast<double*>(pan.base) + start * bk;
      const int64_t h = pan.m - start;
      if (h > 0) {
        rc = x.trsm(dist_view(D, bk, bk, bk), dist_view(mine, h, bk, bk), s);
        if (rc) return rc;
      }
    } else {
      mine = x.recv_buf(parity, prow);
    }
    // (d) along my process row from process column kcol
    const int64_t hmine = L.stack_rows(prow, k);
    if (L.pc > 1) {
      x.group_begin();
      rc = hmine > 0 ? x.bcast(COMM_ROW, mine, hmine * bk, kcol, s) : BF_OK;
      if (!rc) rc = x.bcast_info(COMM_ROW, kcol, s);
      const int rg = x.group_end();
      if (rc || rg) return rc ? rc : rg;
    }
    for (int p = 0; p < L.pr; ++p) {
      P.rows[p] = L.stack_rows(p, k);
      P.ptr[p] = p == prow ? mine : x.recv_buf(parity, p);
    }
    // (e) exchange of the stacked row panels down every process column
    if (L.pr > 1) {
      x.group_begin();
      for (int p = 0; p < L.pr && !rc; ++p)
        if (P.rows[p] > 0) rc = x.bcast(COMM_COL, P.ptr[p], P.rows[p] * bk, p, s);
      const int rg = x.group_end();
      if (rc || rg) return rc ? rc : rg;
    }
    return BF_OK;
  };

  // (f) of step k.  part: 0 = all, 1 = column panel k+1 only, 2 = all but it
  auto update = [&](int64_t k, const DistPanels& P, int part, typename X::Stream s) -> int {
    const int64_t bk = L.tile_len(k);
    const int64_t nq = L.col_tiles(pcol);
    const int64_t limit = part == 2 ? (k + 1) * nb : INT64_MAX;
    if (part == 2) {
      // SMs for the panel stream while this update runs: my share of panel
      // k+1 (its TRSM rows, plus the diagonal factor if I own it) against my
      // rest of the update; a rank with no panel work keeps a few for NCCL
      const int64_t k1 = k + 1;
      double T = 0.0, S = 0.0;
      if (k1 < L.tiles() && L.pcol == int(k1 % L.pc)) {
        const double b1 = double(L.tile_len(k1));
        T = double(L.stack_rows(prow, k1)) * b1 * b1;
        if (prow == int(k1 % L.pr)) T += b1 * b1 * b1 / 3.0;
      }
      // both in multiply-adds x 2: a TRSM row costs b1^2 / 2, the diagonal
      // factor b1^3 / 6, an update element bk (the one-GPU driver's units)
      for (int64_t q = 0; q < nq; ++q)
        if (L.panel_J(q) > k1) S += 2.0 * double(L.panel_h(q)) * double(L.panel_w(q)) * double(bk);
      x.reserve_for(T, S);
    }
    // the column panels J > k this part updates: C -= A * B^T with A my
    // stacked rows from tile i0 on, B the stacked rows of tile J (process row
    // J % pr); a panel whose top tile is the diagonal tile (J, J) is a lower
    // trapezoid
    std::vector<DistGemm> groups;
    const int64_t my_first = L.stack_first(prow, k);
    for (int64_t q = 0; q < nq; ++q) {
      const int64_t J = L.panel_J(q);
      if (J <= k) continue;
      if (part == 1 && J != k + 1) continue;
      if (part == 2 && J == k + 1) continue;
      bf_view C = panel_view(q);
      if (C.m == 0) continue;
      const int pJ = int(J % L.pr);
      DistGemm g;
      g.a = P.ptr[prow] + L.rows_of(prow, my_first, L.panel_i0(q)) * bk;
      g.b = P.ptr[pJ] + L.rows_of(pJ, L.stack_first(pJ, k), L.first_row_geq(pJ, J)) * bk;
      g.c = static_cast<double*>(C.base);
      g.m = C.m;
      g.n = C.n;
      g.lower = pJ == prow;
      g.b_proc = pJ;
      groups.push_back(g);
    }
    if (groups.empty()) return BF_OK;
    const bool reserve = part == 2;
    // one launch over every panel when the executor can (a single reserved
    // persistent grid); otherwise one or two GEMMs per panel over the fan streams
    int rc = x.gemm_groups(groups.data(), int(groups.size()), P, bk, limit, reserve, s);
    if (rc != DIST_NOT_GROUPED) return rc;
    rc = BF_OK;
    const bool fan = part != 1 && x.fan_count() > 0;
    int used = 0;
    if (fan)
      for (int i = 0; i < x.fan_count(); ++i) x.fork(s, x.fan_stream(i));
    for (const DistGemm& g : groups) {
      if (rc) break;
      typename X::Stream st = fan ? x.fan_stream(used++ % x.fan_count()) : s;
      const int64_t w = g.n;
      const bf_view bt = dist_view(const_cast<double*>(g.b), w, bk, bk);
      double* A = const_cast<double*>(g.a);
      int64_t r0 = 0;
      if (g.lower) {
        rc = x.gemm(dist_view(A, w, bk, bk), bt, dist_view(g.c, w, w, w), 1, limit, reserve, st);
        r0 = w;
      }
      if (!rc && g.m > r0)
        rc = x.gemm(dist_view(A + r0 * bk, g.m - r0, bk, bk), bt, dist_view(g.c + r0 * w, g.m - r0, w, w), 0, limit,
                    reserve, st);
    }
    if (fan)
      for (int i = 0; i < x.fan_count(); ++i) x.fork(x.fan_stream(i), s);
    return rc;
  };

  typename X::Stream ms = x.main_stream();
  typename X::Stream ps = lookahead ? x.panel_stream() : ms;
  DistPanels P[2];
  int rc = BF_OK;
  if (!lookahead) {
    for (int64_t k = 0; k < T && !rc; ++k) {
      rc = panel(k, int(k & 1), P[k & 1], ms);
      if (!rc) rc = update(k, P[k & 1], 0, ms);
    }
    return rc;
  }
  x.fork(ms, ps);
  rc = panel(0, 0, P[0], ps);
  for (int64_t k = 0; k < T && !rc; ++k) {
    x.fork(ps, ms);  // main needs panel k
    if (k + 1 < T) {
      rc = update(k, P[k & 1], 1, ms);
      if (rc) break;
      x.fork(ms, ps);  // panel k+1 needs column panel k+1 updated (and step k-1's reads of its buffers done)
      rc = panel(k + 1, int((k + 1) & 1), P[(k + 1) & 1], ps);
      if (rc) break;
      rc = update(k, P[k & 1], 2, ms);
    } else {
      rc = update(k, P[k & 1], 0, ms);
    }
  }
  x.fork(ps, ms);
  return rc;
}

}  // namespace bf
