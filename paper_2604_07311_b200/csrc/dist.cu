// Multi-GPU Cholesky: the 2D block-cyclic schedule of dist_schedule.h run
// with the sm_100a kernels of this library and NCCL over NVLink/NVSwitch.
//
// One process per GPU.  bf_dist_init builds the world communicator from an
// ncclUniqueId and splits it into a row and a column communicator
// (ncclCommSplit: color = process row / column, key = the other coordinate),
// so each panel broadcast spans only the Pc ranks of a process row or the Pr
// ranks of a process column.  The library owns the per-device streams the
// schedule runs on: a high-priority panel stream (diagonal factor, panel
// TRSM, every NCCL call) and fan-out streams for the independent column-panel
// GEMMs of each trailing update; the caller's stream is joined at entry and
// exit.  Receive buffers (two stacked-panel buffers per process row, one
// diagonal tile) are allocated once per context and grown on demand.
//
// NCCL is resolved at run time (dlopen of the libnccl.so.2 torch already
// loaded — the venv's 2.28 — so the process holds one NCCL), which keeps the
// library loadable where NCCL is absent; the dist entry points then fail with
// BF_ERR_UNSUPPORTED.  The final wait polls ncclCommGetAsyncError so a failed
// peer surfaces as an error instead of a hang.
#include "bf_internal.h"
#include "blockfam_b200.h"
#include "dist_schedule.h"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

namespace bf {
int gemm_d_limited(double alpha, const bf_view& a, const bf_view& b, double beta, const bf_view& c, int lower_only,
                   int64_t kc, const int* d_abort, int64_t abort_limit, cudaStream_t s);
int set_error(int code, const char* msg);
}  // namespace bf

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
#define BF_SYM(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
    BF_SYM(GetUniqueId, "ncclGetUniqueId");
    BF_SYM(CommInitRank, "ncclCommInitRank");
    BF_SYM(CommSplit, "ncclCommSplit");
    BF_SYM(Broadcast, "ncclBroadcast");
    BF_SYM(GroupStart, "ncclGroupStart");
    BF_SYM(GroupEnd, "ncclGroupEnd");
    BF_SYM(CommDestroy, "ncclCommDestroy");
    BF_SYM(CommAbort, "ncclCommAbort");
    BF_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    BF_SYM(GetErrorString, "ncclGetErrorString");
#undef BF_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommSplit && api.Broadcast && api.GroupStart &&
             api.GroupEnd && api.CommDestroy && api.CommAbort && api.CommGetAsyncError && api.GetErrorString;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  static thread_local std::string msg;
  msg = std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
  return bf::set_error(BF_ERR_CUDA, msg.c_str());
}

// splitmix64 of the (row >= col) pair: symmetric, counter-based, seedable
__device__ __forceinline__ double synth_value(uint64_t seed, int64_t i, int64_t j, int64_t n) {
  const int64_t r = i >= j ? i : j, c = i >= j ? j : i;
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t(r) * 0x100000001B3ull + uint64_t(c) + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const double u = double(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;  // [-1, 1)
  return r == c ? u + double(n) : u;
}

// rows [0, h) x cols [0, w) of a local panel; panel row r is global row
// (I0 + (r / nb) * pr) * nb + r % nb, column c is global J * nb + c
__global__ void fill_panel_kernel(double* out, int64_t h, int64_t w, int64_t nb, int64_t I0, int64_t pr, int64_t J,
                                  int64_t n, uint64_t seed) {
  const int64_t total = h * w;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / w, c = e - r * w;
    const int64_t gi = (I0 + (r / nb) * pr) * nb + r % nb, gj = J * nb + c;
    out[e] = synth_value(seed, gi, gj, n);
  }
}

__global__ void fill_full_kernel(double* a, int64_t off, int64_t rs, int64_t cs, int64_t n, uint64_t seed) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    a[off + i * rs + j * cs] = synth_value(seed, i, j, n);
  }
}

unsigned fill_grid(int64_t total) {
  int64_t g = (total + 255) / 256;
  return unsigned(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

struct bf_dist {
  int rank = 0, nranks = 1, pr = 1, pc = 1, device = 0;
  ncclComm_t world = nullptr, row = nullptr, col = nullptr;
  cudaStream_t panel = nullptr;
  cudaStream_t fan[3] = {};
  int nfan = 3;
  cudaEvent_t ev_pool[8] = {};
  int ev_next = 0;
  double* bufs = nullptr;  // [parity][process row] stacked-panel receive buffers, then the diagonal tile
  size_t buf_elems = 0;
  int reserve = -1;  // SMs left to the panel stream by the rest-of-update GEMMs (-1: adaptive)
  int lookahead = 1;
  int grouped = 1;  // one grouped TMA launch per update part (0: one GEMM per column panel, fan streams)
  // the grouped rest-of-update keeps its SM reservation (a persistent grid)
  // only while this rank's stacked rows are <= reserve_rows: over a larger
  // trailing matrix a persistent grid loses L2 locality (n=131072 on one GPU:
  // 22.7 s reserved vs 22.1 s), as the one-GPU driver's tail_rows rule found
  int64_t reserve_rows = 32768;
  // group tables of the grouped launches: pinned host staging and the device
  // copy, one region per launch of a factorization (no reuse within a call;
  // the call waits for completion before returning)
  bf::GroupDesc* gtab_h = nullptr;
  bf::GroupDesc* gtab_d = nullptr;
  int64_t gtab_cap = 0, gtab_next = 0;
};

namespace {

struct NcclExec {
  using Stream = cudaStream_t;
  bf_dist* d;
  const bf::DistLayout* L;
  const bf_chol_level* lv;
  int nl;
  int* d_info;
  cudaStream_t user;
  size_t off_recv[2][bf::DIST_MAX_PR] = {};
  size_t off_diag = 0;

  Stream main_stream() { return user; }
  Stream panel_stream() { return d->panel; }
  Stream fan_stream(int i) { return d->fan[i]; }
  int fan_count() { return d->nfan; }
  void fork(Stream from, Stream to) {
    if (from == to) return;
    cudaEvent_t e = d->ev_pool[d->ev_next];
    d->ev_next = (d->ev_next + 1) % 8;
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(to, e, 0);
  }
  int potrf(const bf_view& tile, int64_t base, Stream s) {
    if (nl > 1) {  // a fused diagonal factor keeps to the SMs the concurrent update leaves
      // free, less the 4 reserve_for keeps for NCCL's kernels (n=32768 on one GPU:
      // 375.2 vs 375.5 ms with 2048 tiles, 381.6 vs 381.1 with 1024; launch sequence second)
      bf::t_diag_ctas = reserve_now > 12 ? reserve_now - 4 : (reserve_now > 0 ? 8 : 0);
      const int rc = bf_cholesky_ex_d(&tile, lv + 1, nl - 1, base, d_info, s);
      bf::t_diag_ctas = 0;
      return rc;
    }
    bf_chol_level leaf{13, 0, 0, lv[0].kc};
    return bf_cholesky_ex_d(&tile, &leaf, 1, base, d_info, s);
  }
  int trsm(const bf_view& tri, const bf_view& b, Stream s) {
    return bf_trsm_rltn_ex_d(1.0, &tri, &b, lv[0].kc, nullptr, d_info, s);
  }
  int reserve_now = 0;
  // the reservation follows the panel work this rank has under the update
  // (the one-GPU driver's adaptive rule); "reserve" option = fixed count
  void reserve_for(double T, double S) {
    if (d->reserve >= 0) {
      reserve_now = d->reserve;
      return;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
    int R = T > 0.0 ? int(sms * T / (T + S) + 0.5) + 4 : 4;  // 4: NCCL's kernels
    if (T > 0.0 && R < 12) R = 12;
    if (R > sms / 2) R = sms / 2;
    reserve_now = R;
  }
  int gemm(const bf_view& a, const bf_view& bt, const bf_view& c, int lower, int64_t limit, bool reserve, Stream s) {
    bf_view b = bt;  // B = bt^T
    b.m = bt.n;
    b.n = bt.m;
    b.rs = bt.cs;
    b.cs = bt.rs;
    if (reserve && reserve_now > 0) bf::t_reserve_sms = reserve_now;
    int rc = bf::gemm_d_limited(-1.0, a, b, 1.0, c, lower, lv[0].kc, d_info, limit, s);
    bf::t_reserve_sms = 0;
    return rc;
  }
  // every column panel of the update in one launch of the grouped TMA GEMM:
  // one tensor map over my stacked rows (A, and B of the panels of my own
  // process row), one over the receive buffers (B of the other process rows)
  int gemm_groups(const bf::DistGemm* g, int ng, const bf::DistPanels& P, int64_t k, int64_t limit, bool reserve,
                  Stream s) {
    if (!d->grouped || ng <= 0) return bf::DIST_NOT_GROUPED;
    const int64_t kc = lv[0].kc;
    if (!(kc % 32 == 0 || kc >= k) || k % 2 != 0 || k > 0x7fffffffLL) return bf::DIST_NOT_GROUPED;
    const double* abase = P.ptr[L->prow];
    const int64_t arows = P.rows[L->prow];
    const int64_t brows = int64_t(d->buf_elems) / k;
    if (reinterpret_cast<uintptr_t>(abase) % 16 || arows <= 0) return bf::DIST_NOT_GROUPED;
    if (d->gtab_next + ng > d->gtab_cap) return bf::DIST_NOT_GROUPED;
    bf::GroupDesc* h = d->gtab_h + d->gtab_next;
    int64_t tiles = 0;
    for (int i = 0; i < ng; ++i) {
      const bf::DistGemm& G = g[i];
      bf::GroupDesc& t = h[i];
      const int64_t da = G.a - abase;
      const bool b_mine = G.b_proc == L->prow;
      const int64_t db = b_mine ? G.b - abase : G.b - d->bufs;
      const int64_t tm = (G.m + 127) / 128, tn = (G.n + 127) / 128;
      if (da < 0 || da % k || da / k + G.m > arows || db < 0 || db % k) return bf::DIST_NOT_GROUPED;
      if (db / k + G.n > (b_mine ? arows : brows) || tm >= (1 << 14) || tn >= (1 << 10)) return bf::DIST_NOT_GROUPED;
      if (G.lower && tm < tn) return bf::DIST_NOT_GROUPED;
      t.c = G.c;
      t.ldc = G.n;
      t.tile0 = tiles;
      t.m = int32_t(G.m);
      t.n = int32_t(G.n);
      t.a_row = int32_t(da / k);
      t.b_row = int32_t(db / k);
      t.tiles_m = int32_t(tm);
      t.tiles_n = int32_t(tn);
      t.lower = G.lower;
      t.b_from_a = b_mine;
      tiles += G.lower ? tn * tm - tn * (tn - 1) / 2 : tm * tn;
    }
    if (ng > bf::GEMM_MAX_GROUPS) return bf::DIST_NOT_GROUPED;
    bf::GroupDesc* dev = d->gtab_d + d->gtab_next;
    if (cudaMemcpyAsync(dev, h, sizeof(bf::GroupDesc) * size_t(ng), cudaMemcpyHostToDevice, s) != cudaSuccess)
      return bf::set_error(BF_ERR_CUDA, "group table upload failed");
    d->gtab_next += ng;
    bf::GemmParams p{};
    p.k = k;
    p.kc = kc;
    p.alpha = -1.0;
    p.beta = 1.0;
    p.abort_flag = d_info;
    p.abort_limit = limit;
    bf::OperandMK oa{}, ob{};
    oa.base = abase;
    oa.s_mn = k;
    oa.s_k = 1;
    ob.base = d->bufs;
    ob.s_mn = k;
    ob.s_k = 1;
    if (reserve && reserve_now > 0 && arows <= d->reserve_rows) bf::t_reserve_sms = reserve_now;
    const int rc = bf::launch_gemm_dmma_grouped(p, oa, arows, ob, brows, dev, ng, tiles, s);
    bf::t_reserve_sms = 0;
    if (rc == -3) return bf::set_error(BF_ERR_UNSUPPORTED, "grouped update: unsupported shape");
    return rc ? bf::set_error(BF_ERR_CUDA, "grouped update launch failed") : BF_OK;
  }
  ncclComm_t comm(int which) { return which == bf::COMM_ROW ? d->row : d->col; }
  int bcast(int which, double* buf, int64_t count, int root, Stream s) {
    ncclResult_t r = nccl().Broadcast(buf, buf, size_t(count), ncclFloat64, root, comm(which), s);
    return r == ncclSuccess ? BF_OK : nccl_fail(r, "ncclBroadcast (panel)");
  }
  int bcast_info(int which, int root, Stream s) {
    ncclResult_t r = nccl().Broadcast(d_info, d_info, 1, ncclInt32, root, comm(which), s);
    return r == ncclSuccess ? BF_OK : nccl_fail(r, "ncclBroadcast (pivot flag)");
  }
  void group_begin() { nccl().GroupStart(); }
  int group_end() {
    ncclResult_t r = nccl().GroupEnd();
    return r == ncclSuccess ? BF_OK : nccl_fail(r, "ncclGroupEnd");
  }
  double* recv_buf(int parity, int p) { return d->bufs + off_recv[parity][p]; }
  double* diag_buf() { return d->bufs + off_diag; }
};

// wait for `ev` while polling the communicators for asynchronous errors
int wait_polling(bf_dist* d, cudaEvent_t ev) {
  for (;;) {
    cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return BF_OK;
    if (q != cudaErrorNotReady) return bf::set_error(BF_ERR_CUDA, cudaGetErrorString(q));
    for (ncclComm_t c : {d->world, d->row, d->col}) {
      if (!c) continue;
      ncclResult_t ae = ncclSuccess;
      nccl().CommGetAsyncError(c, &ae);
      if (ae != ncclSuccess && ae != ncclInProgress) {
        nccl().CommAbort(c);
        return nccl_fail(ae, "NCCL asynchronous error (peer failed?)");
      }
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

}  // namespace

extern "C" {

int bf_dist_available(void) { return nccl().ok ? 1 : 0; }

int bf_dist_unique_id(void* out) {
  if (!out) return bf::set_error(BF_ERR_VALUE, "null output");
  if (!nccl().ok) return bf::set_error(BF_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) not found");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return BF_OK;
}

int bf_dist_unique_id_bytes(void) { return int(sizeof(ncclUniqueId)); }

int bf_dist_init(const void* unique_id, int rank, int nranks, int pr, int pc, bf_dist** out) {
  if (!unique_id || !out) return bf::set_error(BF_ERR_VALUE, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return bf::set_error(BF_ERR_VALUE, "bad rank / nranks");
  if (pr < 1 || pc < 1 || pr * pc != nranks || pr > bf::DIST_MAX_PR)
    return bf::set_error(BF_ERR_VALUE, "process grid pr x pc must equal nranks");
  if (!nccl().ok) return bf::set_error(BF_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) not found");
  bf_dist* d = new bf_dist();
  d->rank = rank;
  d->nranks = nranks;
  d->pr = pr;
  d->pc = pc;
  cudaGetDevice(&d->device);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = nccl().CommInitRank(&d->world, nranks, id, rank);
  if (r != ncclSuccess) {
    delete d;
    return nccl_fail(r, "ncclCommInitRank");
  }
  // row communicator: the Pc ranks of my process row, ranked by process column
  r = nccl().CommSplit(d->world, rank / pc, rank % pc, &d->row, nullptr);
  if (r == ncclSuccess) r = nccl().CommSplit(d->world, rank % pc, rank / pc, &d->col, nullptr);
  if (r != ncclSuccess) {
    nccl().CommAbort(d->world);
    delete d;
    return nccl_fail(r, "ncclCommSplit");
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStreamCreateWithPriority(&d->panel, cudaStreamNonBlocking, hi);
  for (auto& f : d->fan) cudaStreamCreateWithFlags(&f, cudaStreamNonBlocking);
  for (auto& e : d->ev_pool) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  *out = d;
  return cudaGetLastError() == cudaSuccess ? BF_OK : bf::set_error(BF_ERR_CUDA, "stream creation failed");
}

int bf_dist_set_option(bf_dist* d, const char* name, int64_t value) {
  if (!d || !name) return bf::set_error(BF_ERR_VALUE, "null argument");
  if (!std::strcmp(name, "reserve")) d->reserve = int(value);
  else if (!std::strcmp(name, "fan")) d->nfan = int(value < 0 ? 0 : (value > 3 ? 3 : value));
  else if (!std::strcmp(name, "lookahead")) d->lookahead = int(value != 0);
  else if (!std::strcmp(name, "grouped")) d->grouped = int(value != 0);
  else if (!std::strcmp(name, "reserve_rows")) d->reserve_rows = value;
  else return bf::set_error(BF_ERR_VALUE, "unknown dist option");
  return BF_OK;
}

int bf_dist_finalize(bf_dist* d) {
  if (!d) return BF_OK;
  cudaDeviceSynchronize();
  for (ncclComm_t c : {d->row, d->col, d->world})
    if (c) nccl().CommDestroy(c);
  if (d->panel) cudaStreamDestroy(d->panel);
  for (auto& f : d->fan)
    if (f) cudaStreamDestroy(f);
  for (auto& e : d->ev_pool)
    if (e) cudaEventDestroy(e);
  if (d->bufs) {
    cudaFree(d->bufs);
    bf::scratch_account(-int64_t(d->buf_elems * sizeof(double)));
  }
  if (d->gtab_d) {
    cudaFree(d->gtab_d);
    cudaFreeHost(d->gtab_h);
    bf::scratch_account(-int64_t(d->gtab_cap * int64_t(sizeof(bf::GroupDesc))));
  }
  delete d;
  return BF_OK;
}

// host-side layout queries (no device work; callable without a GPU)
int64_t bf_dist_local_elems(int64_t n, int64_t nb, int pr, int pc, int rank) {
  if (n < 0 || nb < 1 || pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc) return -1;
  return bf::DistLayout(n, nb, pr, pc, rank).local_elems();
}
int64_t bf_dist_panel_offset(int64_t n, int64_t nb, int pr, int pc, int rank, int64_t q) {
  if (n < 0 || nb < 1 || pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc) return -1;
  bf::DistLayout L(n, nb, pr, pc, rank);
  if (q < 0 || q > L.col_tiles(L.pcol)) return -1;
  return L.panel_off[size_t(q)];
}

int bf_fill_synthetic_d(const bf_view* a, uint64_t seed, void* stream) {
  if (!a || a->m != a->n) return bf::set_error(BF_ERR_SHAPE, "square view required");
  if (a->n == 0) return BF_OK;
  bf::note_launch();
  fill_full_kernel<<<fill_grid(a->n * a->n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<double*>(a->base), a->off, a->rs, a->cs, a->n, seed);
  return cudaGetLastError() == cudaSuccess ? BF_OK : bf::set_error(BF_ERR_CUDA, "fill launch failed");
}

int bf_dist_fill_synthetic_d(int64_t n, int64_t nb, int pr, int pc, int rank, double* local, uint64_t seed,
                             void* stream) {
  if (n < 0 || nb < 1 || pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc || (!local && n > 0))
    return bf::set_error(BF_ERR_VALUE, "bad layout");
  bf::DistLayout L(n, nb, pr, pc, rank);
  for (int64_t q = 0; q < L.col_tiles(L.pcol); ++q) {
    const int64_t h = L.panel_h(q), w = L.panel_w(q);
    if (h * w == 0) continue;
    bf::note_launch();
    fill_panel_kernel<<<fill_grid(h * w), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        local + L.panel_off[size_t(q)], h, w, nb, L.prow + L.panel_i0(q) * pr, pr, L.panel_J(q), n, seed);
  }
  return cudaGetLastError() == cudaSuccess ? BF_OK : bf::set_error(BF_ERR_CUDA, "fill launch failed");
}

// Factor this rank's lower column panels (layout of dist_layout.h) in place.
// levels[0] must be a variant-3 node; its bs is the tile size nb and its kc
// the trailing updates' kc; levels[1..] factor each diagonal tile.  d_info is
// this rank's device pivot flag (-1 on entry); every rank ends with the same
// value: -1 or the first failing global pivot.  Synchronises `stream` at exit
// (polling NCCL for asynchronous errors).
int bf_chol_dist_d(bf_dist* d, double* local, int64_t n, const bf_chol_level* levels, int nlevels, int* d_info,
                   void* stream) {
  if (!d || !levels || nlevels < 1 || !d_info || (!local && n > 0)) return bf::set_error(BF_ERR_VALUE, "null argument");
  if (levels[0].variant != 3 || levels[0].bs < 1)
    return bf::set_error(BF_ERR_VALUE, "distributed Cholesky needs a variant-3 root with bs >= 1");
  if (levels[0].kc < 1) return bf::set_error(BF_ERR_VALUE, "kc must be >= 1");
  bf::DistLayout L(n, levels[0].bs, d->pr, d->pc, d->rank);
  if (L.tiles() == 0) return BF_OK;
  NcclExec x{d, &L, levels, nlevels, d_info, static_cast<cudaStream_t>(stream)};
  size_t need = 0;
  for (int par = 0; par < 2; ++par)
    for (int p = 0; p < d->pr; ++p) {
      x.off_recv[par][p] = need;
      need += size_t(L.stack_cap(p) * L.nb);
    }
  x.off_diag = need;
  need += size_t(L.nb * L.nb);
  if (need > d->buf_elems) {
    cudaStreamSynchronize(x.user);
    if (d->bufs) {
      cudaFree(d->bufs);
      bf::scratch_account(-int64_t(d->buf_elems * sizeof(double)));
    }
    d->bufs = nullptr;
    d->buf_elems = 0;
    if (cudaMalloc(&d->bufs, need * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return bf::set_error(BF_ERR_CUDA, "cannot allocate the panel receive buffers");
    }
    d->buf_elems = need;
    bf::scratch_account(int64_t(need * sizeof(double)));
  }
  // group tables: at most one entry per (step, local column panel)
  const int64_t gneed = L.tiles() * (L.col_tiles(L.pcol) + 1);
  if (d->grouped && gneed > d->gtab_cap) {
    cudaStreamSynchronize(x.user);
    if (d->gtab_d) {
      cudaFree(d->gtab_d);
      cudaFreeHost(d->gtab_h);
      bf::scratch_account(-int64_t(d->gtab_cap * int64_t(sizeof(bf::GroupDesc))));
    }
    d->gtab_d = nullptr;
    d->gtab_h = nullptr;
    d->gtab_cap = 0;
    if (cudaMalloc(&d->gtab_d, size_t(gneed) * sizeof(bf::GroupDesc)) != cudaSuccess ||
        cudaMallocHost(&d->gtab_h, size_t(gneed) * sizeof(bf::GroupDesc)) != cudaSuccess) {
      cudaGetLastError();
      if (d->gtab_d) cudaFree(d->gtab_d);
      d->gtab_d = nullptr;
      d->gtab_h = nullptr;
      return bf::set_error(BF_ERR_CUDA, "cannot allocate the update group tables");
    }
    d->gtab_cap = gneed;
    bf::scratch_account(int64_t(gneed * int64_t(sizeof(bf::GroupDesc))));
  }
  d->gtab_next = 0;
  int rc = bf::chol_dist_schedule(x, L, local, d->lookahead != 0);
  cudaEvent_t done = d->ev_pool[d->ev_next];
  d->ev_next = (d->ev_next + 1) % 8;
  cudaEventRecord(done, x.user);
  const int wrc = wait_polling(d, done);
  if (rc) return rc;
  if (wrc) return wrc;
  return cudaGetLastError() == cudaSuccess ? BF_OK : bf::set_error(BF_ERR_CUDA, "launch failed");
}

int bf_cholesky_dist_d(bf_dist* d, double* local, int64_t n, const bf_chol_level* levels, int nlevels, int* d_info,
                       void* stream) {
  return bf_chol_dist_d(d, local, n, levels, nlevels, d_info, stream);
}

}  // extern "C"
