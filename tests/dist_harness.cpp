// TEST INFRASTRUCTURE: runs the product's distributed Cholesky schedule
// (paper_2604_07311_b200/csrc/dist_schedule.h, the code dist.cu runs with NCCL)
// on a CPU, with P threads as the P ranks of a pr x pc grid:
//   * compute = the oracle (oracle/blockfam_oracle.cpp, the reference's
//     arithmetic restated), so the result can be compared bit for bit with
//     the oracle's single-process factorization;
//   * transport = an in-process broadcast per communicator (rendezvous of the
//     communicator's member threads, in the order each thread issues them —
//     the NCCL ordering contract).
// Built by tests/test_dist_native.py:  g++ -O2 -std=c++17 -shared -fPIC
//   -I include -I paper_2604_07311_b200/csrc dist_harness.cpp oracle/_build/liboracle.so
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "dist_schedule.h"

extern "C" {
struct orc_view_d {
  double* base;
  int64_t off, m, n, rs, cs;
};
struct orc_level {
  int32_t variant, pad_;
  int64_t bs, kc;
};
int orc_gemm_d(double alpha, const orc_view_d* a, const orc_view_d* b, double beta, const orc_view_d* c, int lower,
               int64_t kc, int nthreads);
int orc_trsm_rltn_d(double alpha, const orc_view_d* t, const orc_view_d* b, int64_t kc, int nthreads);
int64_t orc_cholesky_d(const orc_view_d* a, const orc_level* lv, int nl, int nthreads);
}

namespace {

int g_grouped = 0;  // harness_set_grouped: exercise the schedule's grouped-update path

orc_view_d ov(const bf_view& v) { return orc_view_d{static_cast<double*>(v.base), v.off, v.m, v.n, v.rs, v.cs}; }

// one communicator: a generation-counted rendezvous of its members
struct HostComm {
  int size = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  const void* src = nullptr;
  void barrier(std::unique_lock<std::mutex>& lk) {
    const uint64_t g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  // every member calls with its own buffer; the root's is copied into the others
  void bcast(void* buf, size_t bytes, bool is_root) {
    std::unique_lock<std::mutex> lk(mu);
    if (is_root) src = buf;
    barrier(lk);
    if (!is_root && bytes) std::memcpy(buf, src, bytes);
    barrier(lk);
  }
};

struct World {
  int pr, pc;
  std::vector<HostComm> rows, cols;
  World(int pr_, int pc_) : pr(pr_), pc(pc_), rows(size_t(pr_)), cols(size_t(pc_)) {
    for (auto& r : rows) r.size = pc;
    for (auto& c : cols) c.size = pr;
  }
};

struct HostExec {
  using Stream = int;
  World* w;
  const bf::DistLayout* L;
  const orc_level* lv;
  int nl;
  int64_t info = -1;
  std::vector<double> recv[2];
  std::vector<size_t> off;
  std::vector<double> diag;
  int64_t* trace_gemm;  // counts launches (for the test's sanity check)

  Stream main_stream() { return 0; }
  Stream panel_stream() { return 1; }
  Stream fan_stream(int i) { return 2 + i; }
  int fan_count() { return 2; }
  void fork(Stream, Stream) {}
  void reserve_for(double, double) {}
  int potrf(const bf_view& tile, int64_t base, Stream) {
    if (info >= 0) return BF_OK;  // aborted, like the device kernels
    orc_view_d t = ov(tile);
    orc_level leaf{13, 0, 0, lv[0].kc};
    const int64_t bad = nl > 1 ? orc_cholesky_d(&t, lv + 1, nl - 1, 1) : orc_cholesky_d(&t, &leaf, 1, 1);
    if (bad >= 0) info = base + bad;
    return BF_OK;
  }
  int trsm(const bf_view& tri, const bf_view& b, Stream) {
    if (info >= 0) return BF_OK;
    orc_view_d t = ov(tri), x = ov(b);
    orc_trsm_rltn_d(1.0, &t, &x, lv[0].kc, 1);
    return BF_OK;
  }
  int gemm(const bf_view& a, const bf_view& bt, const bf_view& c, int lower, int64_t limit, bool, Stream) {
    if (info >= 0 && info < limit) return BF_OK;
    orc_view_d va = ov(a), vc = ov(c);
    orc_view_d vb{static_cast<double*>(bt.base), bt.off, bt.n, bt.m, bt.cs, bt.rs};  // bt^T
    ++*trace_gemm;
    return orc_gemm_d(-1.0, &va, &vb, 1.0, &vc, lower, lv[0].kc, 1) ? BF_ERR_SHAPE : BF_OK;
  }
  // the grouped launch's semantics: each group is one GEMM over its whole
  // panel, lower = update only gi >= gj (the diagonal tile's triangle)
  int gemm_groups(const bf::DistGemm* g, int ng, const bf::DistPanels&, int64_t k, int64_t limit, bool, Stream) {
    if (!g_grouped) return bf::DIST_NOT_GROUPED;
    if (info >= 0 && info < limit) return BF_OK;
    for (int i = 0; i < ng; ++i) {
      orc_view_d va{const_cast<double*>(g[i].a), 0, g[i].m, k, k, 1};
      orc_view_d vb{const_cast<double*>(g[i].b), 0, k, g[i].n, 1, k};
      orc_view_d vc{g[i].c, 0, g[i].m, g[i].n, g[i].n, 1};
      ++*trace_gemm;
      if (orc_gemm_d(-1.0, &va, &vb, 1.0, &vc, g[i].lower, lv[0].kc, 1)) return BF_ERR_SHAPE;
    }
    return BF_OK;
  }
  HostComm& comm(int which) { return which == bf::COMM_ROW ? w->rows[size_t(L->prow)] : w->cols[size_t(L->pcol)]; }
  int my_index(int which) { return which == bf::COMM_ROW ? L->pcol : L->prow; }
  int bcast(int which, double* buf, int64_t count, int root, Stream) {
    comm(which).bcast(buf, size_t(count) * sizeof(double), my_index(which) == root);
    return BF_OK;
  }
  int bcast_info(int which, int root, Stream) {
    comm(which).bcast(&info, sizeof(info), my_index(which) == root);
    return BF_OK;
  }
  void group_begin() {}
  int group_end() { return BF_OK; }
  double* recv_buf(int parity, int p) { return recv[parity].data() + off[size_t(p)]; }
  double* diag_buf() { return diag.data(); }
};

}  // namespace

extern "C" {

void harness_set_grouped(int on) { g_grouped = on; }

// Scatter `full` (n x n row-major, lower triangle) into pr*pc ranks, factor
// with the distributed schedule on pr*pc threads, gather the lower tiles back
// into `full`.  Returns the common pivot flag (-1 = success); -100 - rank if
// ranks disagree.  *gemm_calls receives the total number of GEMM calls.
int64_t harness_chol_dist(double* full, int64_t n, int pr, int pc, const orc_level* lv, int nl, int lookahead,
                          int64_t* gemm_calls) {
  const int P = pr * pc;
  const int64_t nb = lv[0].bs;
  World world(pr, pc);
  std::vector<int64_t> infos(static_cast<size_t>(P), -1), counts(static_cast<size_t>(P), 0);
  std::vector<std::vector<double>> locals(static_cast<size_t>(P));
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r) {
    th.emplace_back([&, r] {
      bf::DistLayout L(n, nb, pr, pc, r);
      auto& loc = locals[size_t(r)];
      loc.assign(size_t(L.local_elems()), 0.0);
      for (int64_t q = 0; q < L.col_tiles(L.pcol); ++q) {  // scatter
        const int64_t J = L.panel_J(q), w = L.panel_w(q), h = L.panel_h(q);
        for (int64_t rr = 0; rr < h; ++rr) {
          const int64_t gi = (L.prow + (L.panel_i0(q) + rr / nb) * pr) * nb + rr % nb;
          for (int64_t c = 0; c < w; ++c) loc[size_t(L.panel_off[size_t(q)] + rr * w + c)] = full[gi * n + J * nb + c];
        }
      }
      HostExec x{&world, &L, lv, nl};
      x.trace_gemm = &counts[size_t(r)];
      size_t need = 0;
      for (int p = 0; p < pr; ++p) {
        x.off.push_back(need);
        need += size_t(L.stack_cap(p) * nb);
      }
      x.recv[0].assign(need, 0.0);
      x.recv[1].assign(need, 0.0);
      x.diag.assign(size_t(nb * nb), 0.0);
      bf::chol_dist_schedule(x, L, loc.data(), lookahead != 0);
      infos[size_t(r)] = x.info;
    });
  }
  for (auto& t : th) t.join();
  int64_t total = 0;
  for (int r = 0; r < P; ++r) {  // gather
    bf::DistLayout L(n, nb, pr, pc, r);
    const auto& loc = locals[size_t(r)];
    for (int64_t q = 0; q < L.col_tiles(L.pcol); ++q) {
      const int64_t J = L.panel_J(q), w = L.panel_w(q), h = L.panel_h(q);
      for (int64_t rr = 0; rr < h; ++rr) {
        const int64_t gi = (L.prow + (L.panel_i0(q) + rr / nb) * pr) * nb + rr % nb;
        for (int64_t c = 0; c < w; ++c) full[gi * n + J * nb + c] = loc[size_t(L.panel_off[size_t(q)] + rr * w + c)];
      }
    }
    total += counts[size_t(r)];
  }
  *gemm_calls = total;
  for (int r = 1; r < P; ++r)
    if (infos[size_t(r)] != infos[0]) return -100 - r;
  return infos[0];
}

}  // extern "C"
