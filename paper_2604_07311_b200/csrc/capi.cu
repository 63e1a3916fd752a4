// extern "C" boundary (include/blockfam_b200.h) and the native host drivers
// that sit directly above the kernels: operand classification, the
// reference's GEMM edge semantics, the recursive TRSM and the control-tree
// Cholesky loop.  The drivers issue exactly the reference's sequence of
// level-3 calls, so results are bit-identical to the reference when the same
// tree (and hence the same kc) is used.
#include "bf_internal.h"
#include "blockfam_b200.h"

#include <cuda.h>

#include <atomic>
#include <climits>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

namespace bf {
static std::atomic<int64_t> g_launches{0};
void note_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Accounting of the library's device scratch (the B200 side of the reference's
// Workspace live/peak counters, engine/workspace.py:18-56): bytes currently
// held in the scratch caches and the high-water mark since the last reset.
std::atomic<int64_t> g_scratch_live{0}, g_scratch_peak{0};
void scratch_account(int64_t delta) {
  const int64_t now = g_scratch_live.fetch_add(delta) + delta;
  int64_t pk = g_scratch_peak.load();
  while (now > pk && !g_scratch_peak.compare_exchange_weak(pk, now)) {
  }
}

// Device scratch private to one (purpose, device, stream): work queued on
// different streams never shares a buffer, and growing one only waits for
// its own stream.
thread_local int t_diag_ctas = 0;  // CTAs of the next fused diagonal factor (0: one per SM)

void* stream_scratch(int tag, size_t bytes, cudaStream_t s) {
  struct Key {
    int tag, dev;
    cudaStream_t s;
    bool operator<(const Key& o) const {
      return tag != o.tag ? tag < o.tag : (dev != o.dev ? dev < o.dev : s < o.s);
    }
  };
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    bool captured = false;  // handed to a CUDA graph: kept until bf_release_scratch
  };
  static std::mutex mu;
  static std::map<Key, Buf> bufs;
  static std::vector<Buf> retired;  // outgrown buffers a captured graph may still use
  if (tag < 0) {  // release every cached buffer (bf_release_scratch)
    std::lock_guard<std::mutex> lk(mu);
    cudaDeviceSynchronize();
    for (auto& kv : bufs) retired.push_back(kv.second);
    for (auto& b : retired)
      if (b.p) {
        cudaFree(b.p);
        scratch_account(-int64_t(b.bytes));
      }
    bufs.clear();
    retired.clear();
    return nullptr;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  // under stream capture (CholeskyGraph) the buffer becomes part of the
  // graph: allocate it with the capture relaxed for this thread (cudaMalloc
  // is not a stream operation) and never free it behind the graph's back
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (s) cudaStreamIsCapturing(s, &cap);
  const bool capturing = cap == cudaStreamCaptureStatusActive;
  std::lock_guard<std::mutex> lk(mu);
  Buf& b = bufs[Key{tag, dev, s}];
  if (b.bytes < bytes) {
    if (b.p) {
      if (b.captured || capturing) {
        retired.push_back(b);
      } else {
        cudaStreamSynchronize(s);  // the old buffer may still be read by work queued on s
        cudaFree(b.p);
        scratch_account(-int64_t(b.bytes));
      }
    }
    b = Buf{};
    cudaError_t e;
    if (capturing) {
      cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
      cudaThreadExchangeStreamCaptureMode(&mode);
      e = cudaMalloc(&b.p, bytes);
      cudaThreadExchangeStreamCaptureMode(&mode);
    } else {
      e = cudaMalloc(&b.p, bytes);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      b.p = nullptr;
      return nullptr;
    }
    b.bytes = bytes;
    scratch_account(int64_t(bytes));
  }
  if (capturing) b.captured = true;
  return b.p;
}

bool smem_attr(const void* kern, int bytes) {
  struct Key {
    const void* k;
    int dev;
    bool operator<(const Key& o) const { return k < o.k || (k == o.k && dev < o.dev); }
  };
  static std::mutex mu;
  static std::map<Key, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[Key{kern, dev}];
  if (have >= bytes) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  have = bytes;
  return true;
}
}  // namespace bf

namespace {

using bf::GemmParams;
using bf::OperandMK;

thread_local std::string g_last_error;
int g_lookahead = 1;      // bf_set_option("lookahead", 0) restores the plain reference schedule
int g_group = 8;          // bf_set_option("group", g): raster group height in tiles
// bf_set_option("panel_tiles", w): lower GEMMTs on the TMA kernel walk column
// panels w tiles wide, row-major inside each (0 = the row-band raster)
int g_panel_tiles = 0;
int g_fused_trsm = 1;     // bf_set_option("fused_trsm", 0) keeps every recursion level a separate launch
// bf_set_option("pipeline_first", c): step 0 of the lookahead schedule in ~c
// row chunks of the first panel (0/1: off).  Bitwise-neutral; measured no
// faster at n=32768 (the chunked TRSM competes with the SYRK for the same
// SMs), so off by default.
int g_pipeline_first = 0;
// Lookahead SM reservation: the rest of each step's trailing update runs as a
// persistent grid on all but g_tail_reserve SMs, so the panel stream's chain
// of small launches (diagonal factor, TRSM) finds SMs free at once instead of
// waiting for 128x128xbs tiles to retire.  Measured at n=32768 (bench tree):
// 0 -> 390 ms, 8 -> 384, 12 -> 383, 16 -> 382, 20 -> 385, 24 -> 392
// (tools/gpu_tail_sweep.sh).  Grid shape only: the bits are unchanged.
int g_tail_reserve = 16;     // bf_set_option("tail_reserve", r): SMs left to the panel stream
int64_t g_tail_rows = 32768;  // bf_set_option("tail_rows", t): ... when the rest of the update is <= t rows
                              // (larger updates keep the 1-tile CTAs: at n=131072 a persistent grid
                              // over the whole trailing matrix loses L2 locality, 22.1 -> 23.0 s)
// bf_set_option("reserve_adaptive", 0|1): per-step reservation sized by the
// panel stream's share of the step's work (+ "reserve_extra", >= "reserve_min")
int g_reserve_adaptive = 1;
int g_reserve_extra = 6;  // 4 before the overlapped panels (tools/gpu_r02_resv2.sh: 6 -> 370.6 vs 371.0 ms)
int g_reserve_min = 12;
int g_diag_reserve = 0;      // bf_set_option("diag_reserve", r): SMs left to the panel stream while ...
int64_t g_diag_rows = 0;     // bf_set_option("diag_rows", h): ... the first h rows of the rest are updated
// bf_set_option("overlap_h2d", 0): bf_cholesky_host_d loads the whole lower
// triangle before factoring instead of overlapping the load with step 0
int g_overlap_h2d = 1;
// bf_set_option("upper_transpose", n0): FP64 factorizations of order >= n0 on
// an mn-contiguous view (uplo="upper") run on a row-major copy (0 = never)
int64_t g_upper_transpose = 1024;

int fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

enum Mode { MODE_D = 0, MODE_S = 1, MODE_SD = 2 };

inline bool storage_is_f64(Mode m) { return m == MODE_D; }
inline int64_t elem_bytes(Mode m) { return storage_is_f64(m) ? 8 : 4; }

// --- view helpers (views.py:172-199 subview / transposed) ------------------
inline bf_view subview(const bf_view& v, int64_t r0, int64_t nr, int64_t c0, int64_t nc) {
  bf_view s = v;
  s.off = v.off + r0 * v.rs + c0 * v.cs;
  s.m = nr;
  s.n = nc;
  return s;
}
inline bf_view transposed(const bf_view& v) {
  bf_view t = v;
  t.m = v.n;
  t.n = v.m;
  t.rs = v.cs;
  t.cs = v.rs;
  return t;
}

// Classify an operand seen as (MN x K) with strides (s_mn, s_k).
OperandMK classify(const void* base, int64_t off, int64_t s_mn, int64_t s_k, int64_t MN, int64_t K, int64_t kc,
                   Mode mode) {
  OperandMK o{};
  o.base = base;
  o.off = off;
  o.s_mn = s_mn;
  o.s_k = s_k;
  o.mn_scat = nullptr;
  o.k_scat = nullptr;
  o.vec = 1;
  const bool base16 = (reinterpret_cast<uintptr_t>(base) % 16) == 0;
  const int64_t per16 = 16 / elem_bytes(mode);
  if (s_k == 1 || K <= 1) {
    o.layout = bf::GL_KMAJOR;
    o.s_k = 1;
    const bool kc_ok = (kc % per16 == 0) || kc >= K;
    if (storage_is_f64(mode) && base16 && off % per16 == 0 && (s_mn % per16 == 0 || MN <= 1) && kc_ok) o.vec = 2;
  } else if (s_mn == 1 || MN <= 1) {
    o.layout = bf::GL_MNMAJOR;
    o.s_mn = 1;
    if (storage_is_f64(mode) && base16 && off % per16 == 0 && s_k % per16 == 0) o.vec = 2;
  } else {
    o.layout = bf::GL_GENERIC;
  }
  return o;
}

int launch_family(Mode mode, const GemmParams& p, cudaStream_t s) {
  switch (mode) {
    case MODE_D: return bf::launch_gemm_dmma(p, s);
    case MODE_S: return bf::launch_gemm_simt_f32(p, s);
    case MODE_SD: return bf::launch_gemm_simt_f32acc64(p, s);
  }
  return BF_ERR_VALUE;
}

int scale_impl(Mode mode, double beta, const bf_view& c, int lower_only, cudaStream_t s) {
  int kind = mode == MODE_D ? 1 : (mode == MODE_SD ? 2 : 0);
  int rc = bf::launch_scale(kind, beta, c.base, c.off, c.m, c.n, c.rs, c.cs, nullptr, nullptr, lower_only, s);
  return rc ? fail(BF_ERR_CUDA, "scale launch failed") : BF_OK;
}

// engine/gemm.py:74-160 gemm_scatter edge semantics + launch
int gemm_impl(Mode mode, double alpha, const bf_view& a, const bf_view& b, double beta, const bf_view& c,
              int lower_only, int64_t kc, const int* d_abort, cudaStream_t s,
              int64_t abort_limit = INT64_MAX) {
  if (a.n != b.m || c.m != a.m || c.n != b.n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  if (lower_only && c.m != c.n) return fail(BF_ERR_SHAPE, "gemmt needs square c");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  if (a.rs < 0 || a.cs < 0 || b.rs < 0 || b.cs < 0 || c.rs < 0 || c.cs < 0)
    return fail(BF_ERR_SHAPE, "engine packing requires non-negative strides (use transposed views)");
  const int64_t m = c.m, n = c.n, k = a.n;
  if (m == 0 || n == 0) return BF_OK;
  double al = alpha, be = beta;
  if (mode == MODE_S) {  // alpha/beta in the accumulation dtype (engine/gemm.py:99-102)
    al = double(float(alpha));
    be = double(float(beta));
  }
  if (al == 0.0 && be == 1.0) return BF_OK;
  if (k == 0 || al == 0.0) {
    if (be != 1.0) return scale_impl(mode, be, c, lower_only, s);
    return BF_OK;
  }
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.kc = kc;
  p.a = classify(a.base, a.off, a.rs, a.cs, m, k, kc, mode);
  p.b = classify(b.base, b.off, b.cs, b.rs, n, k, kc, mode);  // B^T as (n x k)
  p.c = c.base;
  p.c_off = c.off;
  p.c_rs = c.rs;
  p.c_cs = c.cs;
  p.alpha = al;
  p.beta = be;
  p.lower_only = lower_only;
  p.group = g_group;
  p.panel_tiles = g_panel_tiles;
  p.abort_flag = d_abort;
  p.abort_limit = abort_limit;
  int rc = launch_family(mode, p, s);
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "gemm: unsupported size/layout");
  return rc ? fail(BF_ERR_CUDA, "gemm launch failed") : BF_OK;
}

// Library-owned side streams, one set per (device, calling stream): two
// factorizations enqueued on different caller streams (e.g. from different
// host threads) get independent panel/aux/copy streams and never serialise
// their panel chains on a shared one.
enum SideRole { ROLE_PANEL = 0, ROLE_AUX = 1, ROLE_H2D = 2, ROLE_COPY = 3, ROLE_PANEL2 = 100, ROLE_SEG0 = 4,
                ROLE_FDWATCH = 200 };
cudaStream_t side_stream(SideRole role, cudaStream_t caller) {
  struct Key {
    int dev, role;
    cudaStream_t caller;
    bool operator<(const Key& o) const {
      return dev != o.dev ? dev < o.dev : (role != o.role ? role < o.role : caller < o.caller);
    }
  };
  static std::mutex mu;
  static std::map<Key, cudaStream_t> streams;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  cudaStream_t& st = streams[Key{dev, int(role), caller}];
  if (!st) {
    // the panel stream is high priority: its CTAs go first whenever trailing-update
    // CTAs retire (ROLE_PANEL2, the overlapped panel TRSM, stays normal so the
    // diagonal factor's latency-bound chain keeps precedence over it)
    if (role == ROLE_PANEL) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi);
    } else {
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    }
  }
  return st;
}
cudaStream_t panel_stream(cudaStream_t caller) { return side_stream(ROLE_PANEL, caller); }
cudaStream_t aux_stream(cudaStream_t caller) { return side_stream(ROLE_AUX, caller); }
cudaStream_t h2d_stream(cudaStream_t caller) { return side_stream(ROLE_H2D, caller); }
cudaStream_t copy_stream(cudaStream_t caller) { return side_stream(ROLE_COPY, caller); }
cudaStream_t panel2_stream(cudaStream_t caller) { return side_stream(ROLE_PANEL2, caller); }

// Deep-K narrow GEMM/GEMMT (V2's A11 -= A10 A10^T and A21 -= A20 A10^T, V1's
// SYRK: few output tiles, K = the whole factored part): the kc segments are
// independent sums, so each is computed from +0 by its own launch on its own
// side stream (alpha 1, beta 0: the exact sum lands in scratch) and one kernel
// then applies the reference's folds in segment order.  Same roundings in the
// same order as the single launch, so the same bits; the parallelism is the
// segment count instead of the handful of output tiles.
int g_segsplit = 1;  // bf_set_option("segsplit", 0|1)
int gemm_segsplit(Mode mode, double alpha, const bf_view& a, const bf_view& b, double beta, const bf_view& c,
                  int lower_only, int64_t kc, const int* d_abort, cudaStream_t s, int64_t abort_limit, bool* done) {
  *done = false;
  constexpr int SMAX = 8;
  const int64_t m = c.m, n = c.n, k = a.n;
  if (!g_segsplit || mode != MODE_D || kc >= k || m == 0 || n == 0) return BF_OK;
  const int64_t nseg = (k + kc - 1) / kc;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tm = (m + 127) / 128, tn = (n + 127) / 128;
  const int64_t tiles = lower_only ? tm * (tm + 1) / 2 : tm * tn;
  if (nseg < 4 || tiles * 2 > sms || kc < 256) return BF_OK;  // enough tiles already, or too little per segment
  const size_t bytes = size_t(nseg) * size_t(m) * size_t(n) * sizeof(double);
  double* ws = static_cast<double*>(bf::stream_scratch(5, bytes, s));
  if (!ws) return BF_OK;  // no room: the single launch
  cudaStream_t side[SMAX];
  const int ns = int(nseg < SMAX ? nseg : SMAX);
  for (int q = 0; q < ns; ++q) side[q] = side_stream(SideRole(ROLE_SEG0 + q), s);
  cudaEvent_t ev0;
  cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
  cudaEventRecord(ev0, s);
  for (int q = 0; q < ns; ++q) cudaStreamWaitEvent(side[q], ev0, 0);
  cudaEventDestroy(ev0);
  int rc = BF_OK;
  for (int64_t sg = 0; sg < nseg && !rc; ++sg) {
    const int64_t k0 = sg * kc, kn = k0 + kc < k ? kc : k - k0;
    bf_view w{ws, sg * m * n, m, n, n, 1};
    rc = gemm_impl(mode, 1.0, subview(a, 0, a.m, k0, kn), subview(b, k0, kn, 0, b.n), 0.0, w, lower_only, kc, d_abort,
                   side[sg % ns], abort_limit);
  }
  for (int q = 0; q < ns; ++q) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, side[q]);
    cudaStreamWaitEvent(s, e, 0);
    cudaEventDestroy(e);
  }
  if (rc) return rc;
  if (bf::launch_segfold(ws, int(nseg), m, n, alpha, beta, static_cast<double*>(c.base), c.off, c.rs, c.cs, lower_only,
                         d_abort, abort_limit, s))
    return fail(BF_ERR_CUDA, "segment fold launch failed");
  *done = true;
  return BF_OK;
}

// gemm_impl, with the segment-parallel split when it applies
int gemm_deep(Mode mode, double alpha, const bf_view& a, const bf_view& b, double beta, const bf_view& c,
              int lower_only, int64_t kc, const int* d_abort, cudaStream_t s) {
  if (a.n != b.m || c.m != a.m || c.n != b.n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  bool done = false;
  int rc = gemm_segsplit(mode, alpha, a, b, beta, c, lower_only, kc, d_abort, s, INT64_MAX, &done);
  if (rc || done) return rc;
  return gemm_impl(mode, alpha, a, b, beta, c, lower_only, kc, d_abort, s);
}

// engine/trsm.py:51-68 (_solve_right) with the 32-wide base (engine/trsm.py:96-111)
int trsm_rec(Mode mode, double alpha, const bf_view& tri, const bf_view& b, int64_t kc, int* d_sing,
             const int* d_abort, cudaStream_t s) {
  const int64_t n = tri.n;
  if (b.m == 0 || n == 0) return BF_OK;
  // Whole subtrees of order <= 128 run fused (same tree, same operations),
  // unless a zero pivot must be reported (the standalone trsm entry point).
  if (n <= 128 && n > 32 && d_sing == nullptr && g_fused_trsm && (mode == MODE_D || mode == MODE_S)) {
    int rc = bf::launch_trsm_small_right(mode == MODE_D, alpha, tri.base, tri.off, tri.rs,
                                         tri.cs, b.base, b.off, b.rs, b.cs, b.m, n, kc, d_abort, s);
    if (rc) {
      static thread_local std::string msg;
      msg = std::string("fused trsm launch failed: ") + cudaGetErrorString(cudaPeekAtLastError());
      return fail(BF_ERR_CUDA, msg.c_str());
    }
    return BF_OK;
  }
  if (n <= 32) {
    int rc = bf::launch_trsm_base_right(storage_is_f64(mode), alpha, tri.base, tri.off, tri.rs, tri.cs, b.base,
                                        b.off, b.rs, b.cs, b.m, n, d_sing, 0, d_abort, s);
    return rc ? fail(BF_ERR_CUDA, "trsm base launch failed") : BF_OK;
  }
  const int64_t n1 = n / 2, n2 = n - n1;
  bf_view l11 = subview(tri, 0, n1, 0, n1);
  bf_view l21 = subview(tri, n1, n2, 0, n1);
  bf_view l22 = subview(tri, n1, n2, n1, n2);
  bf_view b1 = subview(b, 0, b.m, 0, n1);
  bf_view b2 = subview(b, 0, b.m, n1, n2);
  int rc = trsm_rec(mode, alpha, l11, b1, kc, d_sing, d_abort, s);
  if (rc) return rc;
  rc = gemm_impl(mode, -1.0, b1, transposed(l21), alpha, b2, 0, kc, d_abort, s);
  if (rc) return rc;
  return trsm_rec(mode, 1.0, l22, b2, kc, d_sing, d_abort, s);
}

// trsm_rec whose triangle is still being factored on another stream: the
// diagonal block's inner steps (block width bs1) each record ev[J] once
// column block J of the triangle is final (rows >= J*bs1); every piece of
// the recursion waits for the last inner step whose columns it reads — a
// subtree on columns [lo, hi) reads tri[lo:hi, lo:hi], a fold
// b2 -= b1 tri[mid:hi, lo:mid]^T reads columns [lo, mid).  Same pieces, same
// order as trsm_rec, so the same bits.
struct TriWait {
  const cudaEvent_t* ev;
  int64_t bs1, ns;
  int64_t last = -1;
  void wait(int64_t col_end, cudaStream_t s) {  // columns [.., col_end) must be final
    int64_t j = (col_end - 1) / bs1;
    if (j > ns - 1) j = ns - 1;
    if (j > last) {
      cudaStreamWaitEvent(s, ev[j], 0);
      last = j;
    }
  }
};
int trsm_rec_w(Mode mode, double alpha, const bf_view& tri, const bf_view& b, int64_t kc, const int* d_abort,
               cudaStream_t s, TriWait& w, int64_t off) {
  const int64_t n = tri.n;
  if (b.m == 0 || n == 0) return BF_OK;
  if ((n <= 128 && n > 32 && g_fused_trsm && (mode == MODE_D || mode == MODE_S)) || n <= 32) {
    w.wait(off + n, s);
    return trsm_rec(mode, alpha, tri, b, kc, nullptr, d_abort, s);
  }
  const int64_t n1 = n / 2, n2 = n - n1;
  int rc = trsm_rec_w(mode, alpha, subview(tri, 0, n1, 0, n1), subview(b, 0, b.m, 0, n1), kc, d_abort, s, w, off);
  if (rc) return rc;
  w.wait(off + n1, s);
  rc = gemm_impl(mode, -1.0, subview(b, 0, b.m, 0, n1), transposed(subview(tri, n1, n2, 0, n1)), alpha,
                 subview(b, 0, b.m, n1, n2), 0, kc, d_abort, s);
  if (rc) return rc;
  return trsm_rec_w(mode, 1.0, subview(tri, n1, n2, n1, n2), subview(b, 0, b.m, n1, n2), kc, d_abort, s, w, off + n1);
}

int trsm_impl(Mode mode, double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_sing,
              cudaStream_t s) {
  if (!tri || !b) return fail(BF_ERR_VALUE, "null view");
  if (tri->m != tri->n) return fail(BF_ERR_SHAPE, "triangular operand must be square");
  if (b->n != tri->n) return fail(BF_ERR_SHAPE, "right solve dims mismatch");
  return trsm_rec(mode, alpha, *tri, *b, kc, d_sing, d_sing, s);
}

int leaf_impl(Mode mode, const bf_view& a, int variant, int64_t base, int* d_info, cudaStream_t s) {
  if (a.m != a.n) return fail(BF_ERR_SHAPE, "square matrix required");
  if (variant < 1 || variant > 3) return fail(BF_ERR_VALUE, "leaf variant must be 1, 2 or 3");
  int rc = bf::launch_potrf_leaf(storage_is_f64(mode), variant, a.base, a.off, a.n, a.rs, a.cs, base, d_info, s);
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "leaf too large");
  return rc ? fail(BF_ERR_CUDA, "leaf launch failed") : BF_OK;
}

// Node lv[idx] on `a` runs as one fused launch (launch_potrf_diag_fused):
// FP64, unit column stride, {variant 3, bs 128, kc >= 128} over the
// unblocked3 leaf (the blocked leaf kernel), 128 < n <= 2048.  Option
// "fused_diag": 1 (default) where nothing trails the factor's inner steps
// (chol_impl / chol_run: standalone factors, the last lookahead panel, the
// distributed driver's diagonal tiles); 2 also in chol_v3_events, whose
// inner-step events let the overlapped panel TRSM (C2) and the mixed
// driver's inverse (C4) trail the factor — one launch makes them wait for
// all of it, which measured slower there (C2 370 -> 376 ms, C4 factor 55.5
// -> 78 ms, tools/gpu_r02_fused_e2e.sh); 0 off.
bool fused_diag_ok(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int idx) {
  if (!bf::g_fused_diag || !bf::g_leaf_blocked || mode != MODE_D || a.cs != 1 || idx >= nl) return false;
  const bf_chol_level& in = lv[idx];
  if (in.variant != 3 || in.bs != 128 || in.kc < 128) return false;
  if (idx + 1 < nl && lv[idx + 1].variant != 13) return false;
  return a.n > 128 && a.n <= 2048 && a.m == a.n;
}
int g_fused_diag_ctas = 0;  // bf_set_option("fused_diag_ctas", c): force the fused factor's grid (0: driver's choice)
int g_fused_diag_pct = 100;  // bf_set_option("fused_diag_pct", p): inside the lookahead, p % of the reserved SMs
int fused_diag(const bf_view& a, const bf_chol_level& in, int64_t base, int* d_info, cudaStream_t s) {
  const int rc = bf::launch_potrf_diag_fused(static_cast<double*>(a.base), a.off, a.n, a.rs, in.kc, base, d_info,
                                             g_fused_diag_ctas > 0 ? g_fused_diag_ctas : bf::t_diag_ctas, s);
  return rc ? fail(BF_ERR_CUDA, "fused diagonal factor launch failed") : BF_OK;
}

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda
// link); nullptr when unavailable
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn stream_wait_value32() {
  static WaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return WaitValue32Fn(nullptr);
    return reinterpret_cast<WaitValue32Fn>(p);
  }();
  return fn;
}

// factor/cholesky.py:118-158 (_run / _recurse) on a flattened control tree.
int chol_run(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int idx, int64_t base, int* d_info,
             cudaStream_t s) {
  const int64_t n = a.n;
  if (n == 0) return BF_OK;
  bf_chol_level node;
  if (idx < nl) {
    node = lv[idx];
  } else {
    node.variant = 13;  // missing child -> unblocked3 (factor/cholesky.py:156-157)
    node.bs = 0;
    node.kc = idx > 0 ? lv[idx - 1].kc : 256;
  }
  if (node.variant >= 11 && node.variant <= 13) return leaf_impl(mode, a, node.variant - 10, base, d_info, s);
  if (node.variant < 1 || node.variant > 3) return fail(BF_ERR_VALUE, "unknown blocked variant");
  if (fused_diag_ok(mode, a, lv, nl, idx)) return fused_diag(a, node, base, d_info, s);
  if (node.bs < 1) return fail(BF_ERR_VALUE, "blocked node requires bs >= 1");
  const int64_t bs = node.bs, kc = node.kc;
  int rc = BF_OK;
  for (int64_t done = 0; done < n && rc == BF_OK; done += (bs < n - done ? bs : n - done)) {
    const int64_t b = bs < n - done ? bs : n - done;
    const int64_t r2s = done + b, r2n = n - r2s;
    bf_view a00 = subview(a, 0, done, 0, done);
    bf_view a10 = subview(a, done, b, 0, done);
    bf_view a11 = subview(a, done, b, done, b);
    bf_view a20 = subview(a, r2s, r2n, 0, done);
    bf_view a21 = subview(a, r2s, r2n, done, b);
    bf_view a22 = subview(a, r2s, r2n, r2s, r2n);
    switch (node.variant) {
      case 1:
        rc = trsm_rec(mode, 1.0, a00, a10, kc, nullptr, d_info, s);
        if (!rc) rc = gemm_deep(mode, -1.0, a10, transposed(a10), 1.0, a11, 1, kc, d_info, s);
        if (!rc) rc = chol_run(mode, a11, lv, nl, idx + 1, base + done, d_info, s);
        break;
      case 2:
        rc = gemm_deep(mode, -1.0, a10, transposed(a10), 1.0, a11, 1, kc, d_info, s);
        if (!rc) rc = chol_run(mode, a11, lv, nl, idx + 1, base + done, d_info, s);
        if (!rc) rc = gemm_deep(mode, -1.0, a20, transposed(a10), 1.0, a21, 0, kc, d_info, s);
        if (!rc) rc = trsm_rec(mode, 1.0, a11, a21, kc, nullptr, d_info, s);
        break;
      case 3:
        rc = chol_run(mode, a11, lv, nl, idx + 1, base + done, d_info, s);
        if (!rc) rc = trsm_rec(mode, 1.0, a11, a21, kc, nullptr, d_info, s);
        if (!rc) rc = gemm_impl(mode, -1.0, a21, transposed(a21), 1.0, a22, 1, kc, d_info, s);
        break;
    }
  }
  return rc;
}

// Host write-back of finished block columns (bf_cholesky_host_d): while set,
// the lookahead driver copies block column k's lower part (rows >= k*bs) to
// the pinned host matrix as soon as panel k is final, on the copy stream.
struct HostWriteback {
  double* host = nullptr;
  int64_t ld = 0;
  cudaStream_t cs = nullptr;
  int64_t copied_upto = 0;  // columns [0, copied_upto) already queued
};
thread_local HostWriteback* g_wb = nullptr;

// Host load of bf_cholesky_host_d: while set, block column j of the lower
// triangle (columns [j*bs, (j+1)*bs), rows >= j*bs) is on the device once
// ev[j] has fired; step 0 of the lookahead driver waits per block column, so
// the host->device copy overlaps the first panel and step 0's update.
struct HostLoad {
  int64_t bs = 0;
  std::vector<cudaEvent_t> ev;
};
thread_local HostLoad* g_h2d = nullptr;

void wait_column(cudaStream_t st, int64_t c0) {
  if (!g_h2d || g_h2d->bs <= 0) return;
  const size_t j = size_t(c0 / g_h2d->bs);
  if (j < g_h2d->ev.size()) cudaStreamWaitEvent(st, g_h2d->ev[j], 0);
}

void writeback_block_column(const bf_view& a, int64_t c0, int64_t w, cudaStream_t after) {
  if (!g_wb || w <= 0) return;
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, after);
  cudaStreamWaitEvent(g_wb->cs, ev, 0);
  cudaEventDestroy(ev);
  const double* src = static_cast<const double*>(a.base) + a.off + c0 * a.rs + c0 * a.cs;
  cudaMemcpy2DAsync(g_wb->host + c0 * g_wb->ld + c0, size_t(g_wb->ld) * 8, src, size_t(a.rs) * 8, size_t(w) * 8,
                    size_t(a.n - c0), cudaMemcpyDeviceToHost, g_wb->cs);
  g_wb->copied_upto = c0 + w;
}

// Right-looking (variant 3) top level with depth-1 lookahead.  Same operation
// set as factor/cholesky.py:146-149 — every element of A22 still receives the
// step's whole K=bs update as one kc-segmented chain and one fold per
// segment — only the launch split and the stream order change:
//   main  : [A(k+1 col block) -= L21 L21_top^T]  ...  [rest of A22 -= L21 L21^T]
//   panel :                       chol(A11') ; A21' := A21' tril(A11')^-T
// so the next panel's POTRF+TRSM overlaps the bulk of this step's SYRK.
// Optional timeline of the lookahead schedule (bf_set_option("timeline", 1)):
// per step, events after the next-column update, after the rest of the
// trailing update, and around the panel on the side stream.
struct TimelineStep {
  cudaEvent_t main_col, main_rest, panel_begin, panel_end, panel_diag;
};
int g_timeline = 0;
std::vector<TimelineStep> g_tl;
cudaEvent_t g_tl_origin = nullptr;

// bf_set_option("panel_overlap", 0|1): a lookahead panel (diagonal factor +
// TRSM of the rows below) runs its TRSM on a second stream, trailing the
// diagonal factor's inner steps (TriWait) instead of waiting for all of it
int g_panel_overlap = 1;
// bf_set_option("panel_chunks", c) / ("panel_chunk_rows", r): the overlapped
// panel's rows below in up to c row chunks of at least r rows, one stream each
int g_panel_chunks = 2;  // 1: 370.9, 2: 369.6, 4: 369.6 ms (C2, tools/gpu_r02_chunks.sh)
int64_t g_panel_chunk_rows = 6144;

// chol_run's variant-3 body for node lv[idx] on `a` (children from idx+1),
// recording ev[j] on st once inner step j's column block is final (after its
// TRSM, before its trailing GEMMT)
int chol_v3_events(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int idx, int64_t base, int* d_info,
                   cudaStream_t st, const cudaEvent_t* ev) {
  const bf_chol_level& in = lv[idx];
  const int64_t b = a.n, bs1 = in.bs, ns = (b + bs1 - 1) / bs1;
  if (bf::g_fused_diag >= 2 && fused_diag_ok(mode, a, lv, nl, idx)) {
    // one launch; ev[j] fires when the kernel publishes tile column j
    // (colfinal[j]) through a stream memory wait on a watcher stream, so
    // whatever trails the inner steps keeps trailing.  Under capture, or
    // without stream memory waits: every ev[j] after the whole factor.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    auto wait_value = stream_wait_value32();
    cudaStream_t w = (cap == cudaStreamCaptureStatusNone && wait_value) ? side_stream(ROLE_FDWATCH, st) : nullptr;
    cudaEvent_t reset = nullptr;
    int* colfinal = nullptr;
    if (w) cudaEventCreateWithFlags(&reset, cudaEventDisableTiming);
    const int frc = bf::launch_potrf_diag_fused(static_cast<double*>(a.base), a.off, a.n, a.rs, in.kc, base, d_info,
                                                g_fused_diag_ctas > 0 ? g_fused_diag_ctas : bf::t_diag_ctas, st,
                                                reset, w ? &colfinal : nullptr);
    bool watched = false;
    if (w && !frc && colfinal) {
      cudaStreamWaitEvent(w, reset, 0);
      watched = true;
      const int64_t cols = (a.n + 127) / 128;  // the kernel's 128-wide tile columns; inner step j ends at column
      for (int64_t j = 0; j < ns && watched; ++j) {
        int64_t c = ((j + 1) * bs1 + 127) / 128 - 1;  // the last tile column inner step j's columns reach
        if (c > cols - 1) c = cols - 1;
        if (wait_value(reinterpret_cast<CUstream>(w), reinterpret_cast<CUdeviceptr>(colfinal + c), 1,
                       CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          watched = false;
        else
          cudaEventRecord(ev[size_t(j)], w);
      }
    }
    if (w) {  // the watcher joins st (its last wait is met before the kernel ends)
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, w);
      cudaStreamWaitEvent(st, j, 0);
      cudaEventDestroy(j);
    }
    if (reset) cudaEventDestroy(reset);
    if (!watched)
      for (int64_t j = 0; j < ns; ++j) cudaEventRecord(ev[size_t(j)], st);
    return frc ? fail(BF_ERR_CUDA, "fused diagonal factor launch failed") : BF_OK;
  }
  int rc = BF_OK;
  for (int64_t j = 0; j < ns && rc == BF_OK; ++j) {
    const int64_t done = j * bs1, bb = bs1 < b - done ? bs1 : b - done;
    const int64_t r2s = done + bb, r2n = b - r2s;
    bf_view d11 = subview(a, done, bb, done, bb);
    bf_view d21 = subview(a, r2s, r2n, done, bb);
    rc = chol_run(mode, d11, lv, nl, idx + 1, base + done, d_info, st);
    if (!rc) rc = trsm_rec(mode, 1.0, d11, d21, in.kc, nullptr, d_info, st);
    cudaEventRecord(ev[size_t(j)], st);
    if (!rc) rc = gemm_impl(mode, -1.0, d21, transposed(d21), 1.0, subview(a, r2s, r2n, r2s, r2n), 1, in.kc, d_info, st);
  }
  return rc;
}

// Panel of the lookahead schedule with the TRSM overlapped: the diagonal
// block is factored by the v3 inner loop of lv[1] on `st` (the body of
// chol_run, inner step J recording ev[J] once its column block is final),
// while `st2` solves a copy X of the rows below against the finished part
// of the triangle.  X goes back into the matrix only if no pivot failure was
// recorded, so a failing diagonal factor leaves the rows below untouched,
// exactly as the sequential panel does; on success every element of the
// panel saw the sequential panel's operations.  Returns with `st` joined.
int panel_overlap(Mode mode, const bf_view& a11, const bf_view& a21, const bf_chol_level* lv, int nl, int64_t base,
                  int* d_info, cudaStream_t st, cudaStream_t key, cudaEvent_t* diag_mark, cudaEvent_t rows_ready) {
  const bf_chol_level& in = lv[1];
  const int64_t b = a11.n, bs1 = in.bs, m = a21.m;
  const int64_t ns = (b + bs1 - 1) / bs1;
  // the rows below in up to g_panel_chunks independent row chunks, each on its
  // own stream: the TRSM's many small launches of one chunk overlap the others'
  int64_t nch = g_panel_chunks > 0 ? g_panel_chunks : 1;
  if (nch > m / g_panel_chunk_rows) nch = m / g_panel_chunk_rows;
  if (nch < 1) nch = 1;
  if (nch > 8) nch = 8;
  std::vector<cudaStream_t> cs(static_cast<size_t>(nch));
  for (int64_t c = 0; c < nch; ++c) {
    cs[size_t(c)] = side_stream(SideRole(ROLE_PANEL2 + c), key);
    if (!cs[size_t(c)]) return -1;
  }
  std::vector<cudaEvent_t> ev(static_cast<size_t>(ns) + 1), evj(static_cast<size_t>(nch));
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (auto& e : evj) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  auto join = [&]() {
    for (int64_t c = 0; c < nch; ++c) {
      cudaEventRecord(evj[size_t(c)], cs[size_t(c)]);
      cudaStreamWaitEvent(st, evj[size_t(c)], 0);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (auto& e : evj) cudaEventDestroy(e);
  };
  cudaEventRecord(ev[size_t(ns)], st);  // the rows below are ready (st's earlier work ...
  for (auto c : cs) {
    cudaStreamWaitEvent(c, ev[size_t(ns)], 0);
    if (rows_ready) cudaStreamWaitEvent(c, rows_ready, 0);  // ... and, early panels, the rest of their column update)
  }
  // (after the chunk streams joined st: under CUDA-graph capture the scratch is then graph-owned)
  double* x = static_cast<double*>(bf::stream_scratch(7, size_t(m) * size_t(b) * sizeof(double), cs[0]));
  if (!x) {  // no room: the caller runs the sequential panel
    join();
    return -1;
  }
  const int64_t per = (m + nch - 1) / nch;
  const double* src = static_cast<const double*>(a21.base) + a21.off;
  int rc = BF_OK;
  for (int64_t c = 0; c < nch && rc == BF_OK; ++c) {
    const int64_t r0 = c * per, rn = per < m - r0 ? per : m - r0;
    if (rn > 0 && cudaMemcpy2DAsync(x + r0 * b, size_t(b) * sizeof(double), src + r0 * a21.rs,
                                    size_t(a21.rs) * sizeof(double), size_t(b) * sizeof(double), size_t(rn),
                                    cudaMemcpyDeviceToDevice, cs[size_t(c)]) != cudaSuccess)
      rc = fail(BF_ERR_CUDA, "panel copy failed");
  }
  // the diagonal block: chol_run's v3 body for lv[1] (children from lv[2])
  if (rc == BF_OK) rc = chol_v3_events(mode, a11, lv, nl, 1, base, d_info, st, ev.data());
  if (diag_mark) {
    cudaEventCreate(diag_mark);
    cudaEventRecord(*diag_mark, st);
  }
  for (int64_t c = 0; c < nch && rc == BF_OK; ++c) {
    const int64_t r0 = c * per, rn = per < m - r0 ? per : m - r0;
    if (rn <= 0) continue;
    cudaStream_t sc = cs[size_t(c)];
    TriWait w{ev.data(), bs1, ns};
    bf_view xv{x + r0 * b, 0, rn, b, b, 1};
    rc = trsm_rec_w(mode, 1.0, a11, xv, lv[0].kc, d_info, sc, w, 0);
    w.wait(b, sc);  // the whole diagonal factor (its flag) before the copy back
    if (!rc && bf::launch_copy2d_unless_aborted(x + r0 * b, b, static_cast<double*>(a21.base) + a21.off + r0 * a21.rs,
                                                a21.rs, rn, b, d_info, sc))
      rc = fail(BF_ERR_CUDA, "panel copy launch failed");
  }
  join();
  return rc;
}

// bf_set_option("early_panel", 0|1|2|3): start panel k+1's diagonal factor once
// the diagonal tile of block column k+1 is updated (see the lookahead loop);
// 2 also reserves SMs for it during the rest of that column's update, 3 also
// at step 0.  n=32768 (tools/gpu_r02_early.sh): 0: 369.6 ms, 1: 367.5-367.9,
// 2: 371.9 (the reserved column update falls behind), 3: 367.9
int g_early_panel = 1;

// Size the reservation to the work the panel stream has to finish under the
// rest of step k's update: panel k+1's TRSM (m rows x b2^2) and diagonal
// factor (b2^3 / 3) against the rest of the trailing GEMMT (m^2 b): their SM
// shares, plus a few SMs for the latency-bound diagonal chain (n=32768: 376.4
// ms with a fixed 16, 375.2 ms adaptive; the exposed panel chain drops 22.8 ->
// 15.6 ms, tools/gpu_r02_reserve.sh).  0 when the update is too large for a
// persistent grid (tail_rows) or reservations are off.
int adaptive_reserve(int64_t m, int64_t b2, int64_t b) {
  if (!(g_tail_reserve > 0 && m <= g_tail_rows)) return 0;
  if (!g_reserve_adaptive) return g_tail_reserve;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const double T = double(m) * b2 * b2 + double(b2) * b2 * b2 / 3.0, S = double(m) * m * b;
  int R = int(sms * T / (T + S) + 0.5) + g_reserve_extra;
  if (R < g_reserve_min) R = g_reserve_min;
  if (R > sms / 2) R = sms / 2;
  return R;
}

int chol_v3_lookahead(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int64_t base, int* d_info,
                      cudaStream_t s) {
  const int64_t n = a.n, bs = lv[0].bs, kc = lv[0].kc;
  cudaStream_t ps = panel_stream(s);
  if (!ps) return fail(BF_ERR_CUDA, "cannot create the panel stream");
  cudaEvent_t ev_main, ev_panel, ev_early;
  cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_early, cudaEventDisableTiming);
  cudaEvent_t* diag_mark = nullptr;  // timeline: event after the diagonal factor of the next panel
  // rows_ready: when set, the rows below are updated later than the
  // diagonal block (early panels): only their TRSM waits for it
  auto panel = [&](int64_t done, int64_t b, cudaStream_t st, cudaEvent_t rows_ready) {
    bf_view a11 = subview(a, done, b, done, b);
    bf_view a21 = subview(a, done + b, n - done - b, done, b);
    if (g_panel_overlap && mode == MODE_D && nl >= 2 && lv[1].variant == 3 && lv[1].bs >= 1 && b > lv[1].bs &&
        a21.m > 0 && a.cs == 1) {
      const int prc = panel_overlap(mode, a11, a21, lv, nl, base + done, d_info, st, s, diag_mark, rows_ready);
      if (prc != -1) return prc;
    }
    int rc = chol_run(mode, a11, lv, nl, 1, base + done, d_info, st);
    if (diag_mark) {
      cudaEventCreate(diag_mark);
      cudaEventRecord(*diag_mark, st);
    }
    if (rows_ready) cudaStreamWaitEvent(st, rows_ready, 0);
    if (!rc) rc = trsm_rec(mode, 1.0, a11, a21, kc, nullptr, d_info, st);
    return rc;
  };
  for (auto& st : g_tl) {
    cudaEventDestroy(st.main_col);
    cudaEventDestroy(st.main_rest);
    cudaEventDestroy(st.panel_begin);
    cudaEventDestroy(st.panel_end);
    if (st.panel_diag) cudaEventDestroy(st.panel_diag);
  }
  g_tl.clear();
  auto mark = [&](cudaStream_t st) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    return e;
  };
  if (g_timeline) {
    if (g_tl_origin) cudaEventDestroy(g_tl_origin);
    g_tl_origin = mark(s);
  }
  int64_t start = 0;
  int rc = BF_OK;
  if (g_pipeline_first > 1 && n > 3 * bs) {
    // Step 0, pipelined by row chunks of the panel: the first panel has no
    // earlier SYRK to hide under, so its TRSM (rows independent) runs chunk
    // by chunk on the panel stream while the main stream applies each
    // finished chunk to block column 1 and the aux stream applies its part
    // of the rest of the trailing update.  Every element still receives the
    // same single K = bs update (same kernel, same kc chain): bitwise the
    // unpipelined schedule.
    // chunks: about g_pipeline_first of them, whole multiples of the next panel width
    const int64_t b = bs, r2 = bs, nr2 = n - bs, b2 = bs < nr2 ? bs : nr2;
    const int64_t want = (nr2 + g_pipeline_first - 1) / g_pipeline_first;
    const int64_t C = ((want + b2 - 1) / b2) * b2;
    const int64_t chunks = (nr2 + C - 1) / C;
    cudaStream_t xs = aux_stream(s);
    if (!xs) return fail(BF_ERR_CUDA, "cannot create the aux stream");
    bf_view a11 = subview(a, 0, b, 0, b);
    bf_view l21 = subview(a, r2, nr2, 0, b);
    bf_view l21_top = subview(l21, 0, b2, 0, b);
    rc = chol_run(mode, a11, lv, nl, 1, base, d_info, s);
    if (rc) return rc;
    std::vector<cudaEvent_t> ev_chunk(static_cast<size_t>(chunks));
    for (auto& e : ev_chunk) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEvent_t ev_col, ev_rest;
    cudaEventCreateWithFlags(&ev_col, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming);
    cudaEventRecord(ev_main, s);
    cudaStreamWaitEvent(ps, ev_main, 0);
    for (int64_t i = 0; i < chunks && !rc; ++i) {
      const int64_t r0 = i * C, rn = C < nr2 - r0 ? C : nr2 - r0;
      rc = trsm_rec(mode, 1.0, a11, subview(l21, r0, rn, 0, b), kc, nullptr, d_info, ps);
      cudaEventRecord(ev_chunk[size_t(i)], ps);
    }
    if (!rc) writeback_block_column(a, 0, b, ps);
    // block column 1 (l21 columns [0, b2) of the trailing matrix), chunk by chunk (main stream)
    for (int64_t i = 0; i < chunks && !rc; ++i) {
      const int64_t r0 = i * C, rn = C < nr2 - r0 ? C : nr2 - r0;
      cudaStreamWaitEvent(s, ev_chunk[size_t(i)], 0);
      int64_t g0 = r0;  // first row of this chunk taking a full-width GEMM
      if (i == 0) {
        rc = gemm_impl(mode, -1.0, l21_top, transposed(l21_top), 1.0, subview(a, r2, b2, r2, b2), 1, kc, d_info, s);
        g0 = b2;
      }
      if (!rc && r0 + rn > g0)
        rc = gemm_impl(mode, -1.0, subview(l21, g0, r0 + rn - g0, 0, b), transposed(l21_top), 1.0,
                       subview(a, r2 + g0, r0 + rn - g0, r2, b2), 0, kc, d_info, s);
    }
    // the rest of step 0's trailing update (l21 rows and columns >= b2), chunk
    // by chunk on the aux stream: the chunk's rows against every column before
    // them (GEMM), then its own diagonal block (GEMMT)
    cudaStreamWaitEvent(xs, ev_main, 0);
    for (int64_t i = 0; i < chunks && !rc; ++i) {
      const int64_t r0 = i * C, rn = C < nr2 - r0 ? C : nr2 - r0;
      const int64_t q0 = r0 > b2 ? r0 : b2, qn = r0 + rn - q0;  // rows of this chunk in the rest
      if (qn <= 0) continue;
      cudaStreamWaitEvent(xs, ev_chunk[size_t(i)], 0);
      bf_view li = subview(l21, q0, qn, 0, b);
      if (q0 > b2) {
        bf_view mid = subview(l21, b2, q0 - b2, 0, b);
        rc = gemm_impl(mode, -1.0, li, transposed(mid), 1.0, subview(a, r2 + q0, qn, r2 + b2, q0 - b2), 0, kc, d_info,
                       xs, base + r2);
      }
      if (!rc)
        rc = gemm_impl(mode, -1.0, li, transposed(li), 1.0, subview(a, r2 + q0, qn, r2 + q0, qn), 1, kc, d_info, xs,
                       base + r2);
    }
    cudaEventRecord(ev_rest, xs);
    // panel 1 once block column 1 is complete
    if (!rc) {
      cudaEventRecord(ev_col, s);
      cudaStreamWaitEvent(ps, ev_col, 0);
      rc = panel(r2, b2, ps, nullptr);
      if (!rc) writeback_block_column(a, r2, b2, ps);
      cudaEventRecord(ev_panel, ps);
      cudaStreamWaitEvent(s, ev_panel, 0);
    }
    cudaStreamWaitEvent(s, ev_rest, 0);
    for (auto& e : ev_chunk) cudaEventDestroy(e);
    cudaEventDestroy(ev_col);
    cudaEventDestroy(ev_rest);
    start = r2;
  } else {
    wait_column(s, 0);
    if (g_fused_diag_pct != 100) {  // the first panel's trailing TRSM needs SMs beside a fused factor
      int sms = 148, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      bf::t_diag_ctas = sms * g_fused_diag_pct / 100 > 8 ? sms * g_fused_diag_pct / 100 : 8;
    }
    rc = panel(0, bs < n ? bs : n, s, nullptr);
    bf::t_diag_ctas = 0;
    if (rc == BF_OK) writeback_block_column(a, 0, bs < n ? bs : n, s);
  }
  for (int64_t done = start; done < n && rc == BF_OK;) {
    const int64_t b = bs < n - done ? bs : n - done;
    const int64_t r2 = done + b, nr2 = n - r2;
    if (nr2 == 0) break;
    const int64_t b2 = bs < nr2 ? bs : nr2;  // next panel width
    bf_view l21 = subview(a, r2, nr2, done, b);
    bf_view l21_top = subview(l21, 0, b2, 0, b);
    bf_view l21_rest = subview(l21, b2, nr2 - b2, 0, b);
    // (1) next block column, on the main stream.  Early panels: the panel
    // stream starts the next diagonal factor as soon as the diagonal tile is
    // updated; the rows below follow on the main stream with the step's SM
    // reservation (they belong to step k: a pivot failure in panel k+1 must
    // not cancel them, hence the abort limit) and only the panel's TRSM waits
    // for them.
    const bool loading = g_h2d && done == 0;  // step 0 of a host factorization: columns still arriving
    const bool early = g_early_panel && !loading && nr2 > b2 && (done > 0 || g_early_panel == 3);
    if (loading) wait_column(s, r2);
    rc = gemm_impl(mode, -1.0, l21_top, transposed(l21_top), 1.0, subview(a, r2, b2, r2, b2), 1, kc, d_info, s);
    if (early) {
      cudaEventRecord(ev_early, s);
      cudaStreamWaitEvent(ps, ev_early, 0);
      if (g_early_panel == 2) bf::t_reserve_sms = adaptive_reserve(nr2 - b2, b2, b);
    }
    if (!rc && nr2 > b2)
      rc = gemm_impl(mode, -1.0, l21_rest, transposed(l21_top), 1.0, subview(a, r2 + b2, nr2 - b2, r2, b2), 0, kc,
                     d_info, s, early ? base + r2 : INT64_MAX);
    bf::t_reserve_sms = 0;
    if (rc) break;
    TimelineStep ts{};
    if (g_timeline) ts.main_col = mark(s);
    // (2) next panel on the side stream once (1) has landed
    cudaEventRecord(ev_main, s);
    if (!early) cudaStreamWaitEvent(ps, ev_main, 0);
    if (g_timeline) {
      ts.panel_begin = mark(ps);
      diag_mark = &ts.panel_diag;
    }
    {  // a fused diagonal factor keeps to the SMs the rest of this step's update leaves free
      const int64_t m3 = nr2 - b2;
      int R = 0;
      if (m3 > 0) {
        R = (g_tail_reserve > 0 && m3 <= g_tail_rows) ? (g_reserve_adaptive ? adaptive_reserve(m3, b2, b)
                                                                               : g_tail_reserve)
                                                     : 16;
        if (R < 1) R = 16;
      }
      if (R > 0 && g_fused_diag_pct != 100) R = R * g_fused_diag_pct / 100 > 8 ? R * g_fused_diag_pct / 100 : 8;
      bf::t_diag_ctas = R;
    }
    rc = panel(r2, b2, ps, early ? ev_main : nullptr);
    bf::t_diag_ctas = 0;
    diag_mark = nullptr;
    if (rc) break;
    if (g_timeline) ts.panel_end = mark(ps);
    cudaEventRecord(ev_panel, ps);
    writeback_block_column(a, r2, b2, ps);  // block column k+1 is final
    // (3) the rest of the trailing update, concurrently with (2).  It belongs
    // to step k, so a pivot failure inside panel k+1 (index >= base+r2) must
    // not cancel it: the reference finishes step k before it meets that pivot.
    if (nr2 > b2 && loading) {
      // block column by block column as each arrives: the same GEMMT split by
      // columns (diagonal block lower-only, the rows below it full)
      for (int64_t c0 = r2 + b2; c0 < n && !rc; c0 += bs) {
        const int64_t w = bs < n - c0 ? bs : n - c0;
        wait_column(s, c0);
        bf_view lc = subview(a, c0, w, done, b);
        rc = gemm_impl(mode, -1.0, lc, transposed(lc), 1.0, subview(a, c0, w, c0, w), 1, kc, d_info, s, base + r2);
        if (!rc && c0 + w < n) {
          bf_view lb = subview(a, c0 + w, n - c0 - w, done, b);
          rc = gemm_impl(mode, -1.0, lb, transposed(lc), 1.0, subview(a, c0 + w, n - c0 - w, c0, w), 0, kc, d_info,
                         s, base + r2);
        }
      }
    } else if (nr2 > b2) {
      // tail steps (the panel chain is the critical path): optionally keep
      // g_tail_reserve SMs free of this update so the panel kernels start at once
      const int64_t m = nr2 - b2, r3 = r2 + b2;
      if (g_tail_reserve > 0 && m <= g_tail_rows) bf::t_reserve_sms = g_tail_reserve;
      if (bf::t_reserve_sms > 0 && g_reserve_adaptive) bf::t_reserve_sms = adaptive_reserve(m, b2, b);
      // diagonal-factor window: the first h1 rows of the rest leave
      // g_diag_reserve SMs to the panel stream (its diagonal factor is a chain
      // of small launches that otherwise waits for trailing tiles to retire);
      // the rows below follow on the whole GPU.  Same per-element chains.
      const int64_t h1 = g_diag_reserve > 0 ? (m < g_diag_rows ? m : g_diag_rows) : 0;
      if (h1 > 0) {
        if (!bf::t_reserve_sms) bf::t_reserve_sms = g_diag_reserve;
        bf_view l1 = subview(l21_rest, 0, h1, 0, b);
        rc = gemm_impl(mode, -1.0, l1, transposed(l1), 1.0, subview(a, r3, h1, r3, h1), 1, kc, d_info, s, base + r2);
        if (m <= g_tail_rows) bf::t_reserve_sms = g_tail_reserve; else bf::t_reserve_sms = 0;
        if (!rc && m > h1) {
          bf_view l2 = subview(l21_rest, h1, m - h1, 0, b);
          rc = gemm_impl(mode, -1.0, l2, transposed(l1), 1.0, subview(a, r3 + h1, m - h1, r3, h1), 0, kc, d_info, s,
                         base + r2);
          if (!rc)
            rc = gemm_impl(mode, -1.0, l2, transposed(l2), 1.0, subview(a, r3 + h1, m - h1, r3 + h1, m - h1), 1, kc,
                           d_info, s, base + r2);
        }
      } else {
        rc = gemm_impl(mode, -1.0, l21_rest, transposed(l21_rest), 1.0, subview(a, r3, m, r3, m), 1, kc, d_info, s,
                       base + r2);
      }
      bf::t_reserve_sms = 0;
    }
    if (g_timeline) {
      ts.main_rest = mark(s);
      g_tl.push_back(ts);
    }
    cudaStreamWaitEvent(s, ev_panel, 0);  // step k+1 needs panel k+1
    done = r2;
  }
  cudaEventDestroy(ev_main);
  cudaEventDestroy(ev_panel);
  cudaEventDestroy(ev_early);
  return rc;
}

// ---- LU (factor/lu.py:56-130, engine/trsm.py:71-88) ------------------------
// unit_tril(tri) X = alpha B, the reference's recursive halving over GEMM
int trsm_left_rec(Mode mode, double alpha, const bf_view& tri, const bf_view& b, int64_t kc, cudaStream_t s) {
  const int64_t n = tri.n;
  if (b.n == 0 || n == 0) return BF_OK;
  if (n <= 32) {
    int rc = bf::launch_trsm_left_base(storage_is_f64(mode), alpha, tri.base, tri.off, tri.rs, tri.cs, b.base, b.off,
                                       b.rs, b.cs, int(n), b.n, s);
    return rc ? fail(BF_ERR_CUDA, "left trsm base launch failed") : BF_OK;
  }
  const int64_t n1 = n / 2, n2 = n - n1;
  int rc = trsm_left_rec(mode, alpha, subview(tri, 0, n1, 0, n1), subview(b, 0, n1, 0, b.n), kc, s);
  if (rc) return rc;
  rc = gemm_impl(mode, -1.0, subview(tri, n1, n2, 0, n1), subview(b, 0, n1, 0, b.n), alpha, subview(b, n1, n2, 0, b.n),
                 0, kc, nullptr, s);
  if (rc) return rc;
  return trsm_left_rec(mode, 1.0, subview(tri, n1, n2, n1, n2), subview(b, n1, n2, 0, b.n), kc, s);
}

// triu(U) X = B (non-unit), recursive: the bottom half first
int trsm_upper_rec(Mode mode, const bf_view& u, const bf_view& b, int64_t kc, cudaStream_t s) {
  const int64_t n = u.n;
  if (b.n == 0 || n == 0) return BF_OK;
  if (n <= 32) {
    int rc = bf::launch_trsm_upper_base(storage_is_f64(mode), u.base, u.off, u.rs, u.cs, b.base, b.off, b.rs, b.cs,
                                        int(n), b.n, s);
    return rc ? fail(BF_ERR_CUDA, "upper trsm base launch failed") : BF_OK;
  }
  const int64_t n1 = n / 2, n2 = n - n1;
  int rc = trsm_upper_rec(mode, subview(u, n1, n2, n1, n2), subview(b, n1, n2, 0, b.n), kc, s);
  if (rc) return rc;
  rc = gemm_impl(mode, -1.0, subview(u, 0, n1, n1, n2), subview(b, n1, n2, 0, b.n), 1.0, subview(b, 0, n1, 0, b.n), 0,
                 kc, nullptr, s);
  if (rc) return rc;
  return trsm_upper_rec(mode, subview(u, 0, n1, 0, n1), subview(b, 0, n1, 0, b.n), kc, s);
}

int apply_pivots_impl(Mode mode, const bf_view& a, const int64_t* piv, int64_t count, int64_t sub, int backward,
                      cudaStream_t s) {
  if (a.m == 0 || a.n == 0 || count == 0) return BF_OK;
  int rc = bf::launch_apply_pivots(storage_is_f64(mode), a.base, a.off, a.rs, a.cs, a.n, piv, count, sub, backward, s);
  return rc ? fail(BF_ERR_CUDA, "row swap launch failed") : BF_OK;
}

// device scratch for the LU's k-major copies: private to the calling stream
// (the lookahead's panel stream runs child-level GEMMs concurrently with the
// main stream's trailing update, and callers may run LUs on several streams)
double* lu_scratch(size_t elems, cudaStream_t s) {
  return static_cast<double*>(bf::stream_scratch(2, elems * sizeof(double), s));
}

// levels: variant 20 = blocked, 21 = unblocked leaf (flatten of the lu tree)
// a22 -= a21 * a12 for the columns [c0, c0 + nc) of a12 / a22 (k-major copy of
// a12's part for the TMA kernel when it pays; same values, same kc chains)
static int lu_update(Mode mode, const bf_view& a21, const bf_view& a12, const bf_view& a22, int64_t c0, int64_t nc,
                     int64_t kc, cudaStream_t s) {
  if (nc <= 0 || a21.m == 0) return BF_OK;
  const bf_view b12 = subview(a12, 0, a12.m, c0, nc);
  bf_view bop = b12;
  const int64_t b = a12.m;
  if (mode == MODE_D && b12.rs != 1 && int64_t(b) * nc >= (int64_t(1) << 16) && (b % 16 == 0)) {
    double* scratch = lu_scratch(size_t(b) * size_t(nc), s);
    if (scratch && !bf::launch_transpose(1, b12.base, b12.off, b12.rs, b12.cs, b, nc, scratch, b, s)) {
      bf_view t{};
      t.base = scratch;
      t.off = 0;
      t.m = nc;
      t.n = b;
      t.rs = b;
      t.cs = 1;
      bop = transposed(t);
    }
  }
  return gemm_impl(mode, -1.0, a21, bop, 1.0, subview(a22, 0, a22.m, c0, nc), 0, kc, nullptr, s);
}

// swaps of panel k to the left and right parts, global pivot offsets, and
// the TRSM of the block row (factor/lu.py:80-99)
static int lu_after_panel(Mode mode, const bf_view& a, int64_t k, int64_t b, int64_t* piv, int64_t kc,
                          cudaStream_t s) {
  const int64_t m = a.m, n = a.n;
  int rc = apply_pivots_impl(mode, subview(a, k, m - k, 0, k), piv + k, b, 0, 0, s);
  if (!rc) rc = apply_pivots_impl(mode, subview(a, k, m - k, k + b, n - k - b), piv + k, b, 0, 0, s);
  if (!rc && bf::launch_add_offset(piv + k, b, k, s)) rc = fail(BF_ERR_CUDA, "pivot offset launch failed");
  if (!rc && k + b < n) rc = trsm_left_rec(mode, 1.0, subview(a, k, b, k, b), subview(a, k, b, k + b, n - k - b), kc, s);
  return rc;
}

int lu_run(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int idx, int64_t* piv, int64_t base,
           int* d_sing, cudaStream_t s) {
  const int64_t m = a.m, n = a.n, steps = m < n ? m : n;
  if (steps == 0) return BF_OK;
  const bool leaf = idx >= nl || lv[idx].variant == 21;
  if (leaf) {
    int rc = bf::launch_lu_leaf(storage_is_f64(mode), a.base, a.off, a.rs, a.cs, m, n, piv, d_sing, base, s);
    return rc ? fail(BF_ERR_CUDA, "lu leaf launch failed") : BF_OK;
  }
  if (lv[idx].variant != 20 || lv[idx].bs < 1) return fail(BF_ERR_VALUE, "bad lu level");
  const int64_t bs = lv[idx].bs, kc = lv[idx].kc;
  for (int64_t k = 0; k < steps; k += bs) {
    const int64_t b = bs < steps - k ? bs : steps - k;
    int rc = lu_run(mode, subview(a, k, m - k, k, b), lv, nl, idx + 1, piv + k, base + k, d_sing, s);
    if (!rc) rc = lu_after_panel(mode, a, k, b, piv, kc, s);
    if (!rc && k + b < n && k + b < m)
      rc = lu_update(mode, subview(a, k + b, m - k - b, k, b), subview(a, k, b, k + b, n - k - b),
                     subview(a, k + b, m - k - b, k + b, n - k - b), 0, n - k - b, kc, s);
    if (rc) return rc;
  }
  return BF_OK;
}

// Top-level blocked LU with depth-1 lookahead: per step the next block
// column's share of the trailing GEMM runs first, then panel k+1 (its own
// columns only) factors on the high-priority panel stream while the main
// stream applies the rest of step k's update; panel k+1's row swaps touch
// the other columns only after that join.  Same operations per element as
// lu_run (a column split of one GEMM): bitwise the same factor.
int lu_lookahead(Mode mode, const bf_view& a, const bf_chol_level* lv, int nl, int64_t* piv, int* d_sing,
                 cudaStream_t s) {
  const int64_t m = a.m, n = a.n, steps = m < n ? m : n;
  const int64_t bs = lv[0].bs, kc = lv[0].kc;
  cudaStream_t ps = panel_stream(s);
  if (!ps) return fail(BF_ERR_CUDA, "cannot create the panel stream");
  cudaEvent_t ev_main, ev_panel;
  cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming);
  int rc = lu_run(mode, subview(a, 0, m, 0, bs < steps ? bs : steps), lv, nl, 1, piv, 0, d_sing, s);
  for (int64_t k = 0; k < steps && !rc; k += bs) {
    const int64_t b = bs < steps - k ? bs : steps - k;
    rc = lu_after_panel(mode, a, k, b, piv, kc, s);
    if (rc) break;
    const int64_t k1 = k + b;
    if (k1 >= n || k1 >= m) {
      if (k1 < steps) rc = fail(BF_ERR_VALUE, "lu lookahead: bad step");
      break;
    }
    const bf_view a21 = subview(a, k1, m - k1, k, b), a12 = subview(a, k, b, k1, n - k1),
                  a22 = subview(a, k1, m - k1, k1, n - k1);
    const int64_t b2 = k1 < steps ? (bs < steps - k1 ? bs : steps - k1) : 0;
    rc = lu_update(mode, a21, a12, a22, 0, b2 > 0 ? b2 : n - k1, kc, s);
    if (rc || b2 == 0) break;
    cudaEventRecord(ev_main, s);
    cudaStreamWaitEvent(ps, ev_main, 0);
    rc = lu_run(mode, subview(a, k1, m - k1, k1, b2), lv, nl, 1, piv + k1, k1, d_sing, ps);
    cudaEventRecord(ev_panel, ps);
    if (!rc) rc = lu_update(mode, a21, a12, a22, b2, n - k1 - b2, kc, s);
    cudaStreamWaitEvent(s, ev_panel, 0);
  }
  cudaEventDestroy(ev_main);
  cudaEventDestroy(ev_panel);
  return rc;
}

int chol_impl(Mode mode, const bf_view* a, const bf_chol_level* lv, int nl, int* d_info, cudaStream_t s) {
  if (!a || (nl > 0 && !lv)) return fail(BF_ERR_VALUE, "null argument");
  if (a->m != a->n) return fail(BF_ERR_SHAPE, "square matrix required");
  if (nl < 1) return fail(BF_ERR_VALUE, "empty control tree");
  if (a->n == 0) return BF_OK;
  if (mode == MODE_D && g_upper_transpose && a->rs == 1 && a->cs >= a->n && a->n >= g_upper_transpose) {
    // uplo="upper" arrives as the lower algorithm on the transposed view
    // (factor/cholesky.py:108-109), whose operands are mn-contiguous: the
    // TMA kernel cannot stage them.  Factor a row-major copy instead: the
    // view's lower triangle in (a tiled transpose of the caller's upper
    // triangle), the same tree on it, the lower triangle back out.  Every
    // element sees the same operations, so the bits (and, after a pivot
    // failure, the partial state) are those of the in-place run.
    const int64_t n = a->n;
    // the copy lives in this stream's cached scratch (bf_release_scratch frees it)
    double* work = static_cast<double*>(bf::stream_scratch(3, size_t(n) * size_t(n) * sizeof(double), s));
    if (work) {
      double* src = static_cast<double*>(a->base);
      // work(i, j) = view(i, j) = storage[off + i + j*cs] for i >= j: a transpose of the
      // row-major storage's upper triangle
      int rc = bf::launch_transpose_tri_f64(src, a->off, a->cs, 1, n, work, n, 2, s);
      bf_view w{work, 0, n, n, n, 1};
      if (!rc) rc = chol_impl(mode, &w, lv, nl, d_info, s);
      else rc = fail(BF_ERR_CUDA, "transpose launch failed");
      // view(i, j) = work(i, j), i >= j: storage[off + j*cs + i] = work[i*n + j]
      if (bf::launch_transpose_tri_f64(work, 0, n, 1, n, src + a->off, a->cs, 1, s) && !rc)
        rc = fail(BF_ERR_CUDA, "transpose launch failed");
      return rc;
    }
    // no room for the copy: factor in place on the cp.async kernel
  }
  if (fused_diag_ok(mode, *a, lv, nl, 0)) return fused_diag(*a, lv[0], 0, d_info, s);
  if (lv[0].variant == 3 && lv[0].bs >= 1 && a->n > 2 * lv[0].bs && g_lookahead)
    return chol_v3_lookahead(mode, *a, lv, nl, 0, d_info, s);
  return chol_run(mode, *a, lv, nl, 0, 0, d_info, s);
}

int scatter_impl(Mode mode, double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                 const bf_scatter_view* c, int64_t kc, cudaStream_t s) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  if (b->m != a->n || c->m != a->m || c->n != b->n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  const int64_t m = c->m, n = c->n, k = a->n;
  if (m == 0 || n == 0) return BF_OK;
  double al = alpha, be = beta;
  if (mode == MODE_S) {
    al = double(float(alpha));
    be = double(float(beta));
  }
  if (al == 0.0 && be == 1.0) return BF_OK;
  if (k == 0 || al == 0.0) {
    if (be == 1.0) return BF_OK;
    int kind = mode == MODE_D ? 1 : (mode == MODE_SD ? 2 : 0);
    int rc = bf::launch_scale(kind, be, c->base, 0, m, n, 0, 0, c->rscat, c->cscat, 0, s);
    return rc ? fail(BF_ERR_CUDA, "scale launch failed") : BF_OK;
  }
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.kc = kc;
  p.a = OperandMK{a->base, 0, 0, 0, a->rscat, a->cscat, bf::GL_GENERIC, 1};
  p.b = OperandMK{b->base, 0, 0, 0, b->cscat, b->rscat, bf::GL_GENERIC, 1};
  p.c = c->base;
  p.c_rscat = c->rscat;
  p.c_cscat = c->cscat;
  p.alpha = al;
  p.beta = be;
  p.lower_only = 0;
  p.group = 8;
  int rc = launch_family(mode, p, s);
  return rc ? fail(BF_ERR_CUDA, "scatter gemm launch failed") : BF_OK;
}

inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }

}  // namespace

namespace bf {
// mixed driver (mixed.cu): factor the FP64 diagonal block `a` with the tree
// and solve X L^T = X (X = the identity, set on st before the call) with the
// TRSM trailing the factor's inner steps on a second stream (as the
// overlapped panels do); returns with st joined.  Falls back to the
// sequential factor + solve when the tree root is not a blocked variant 3.
// X = L^-T (upper triangular) of the factored lower block L by recursive
// doubling: the 128-wide diagonal tiles X_dd = L_dd^-T in one launch
// (launch_trsm_diag_tiles), then per split L = (A 0; B C) of [o, o + m):
// X12 = -X11 B^T X22 as two GEMMs — log2(n / 128) dependent levels instead of
// the right solve's chain of 128-wide leaves.  X holds the identity on entry.
// Not the reference's TRSM order: the mixed solver's inverse carries no
// bitwise contract, only FP64 accuracy (its refinement pins the solution).
int tri_inverse_t_rec(const bf_view& l, const bf_view& x, int64_t o, int64_t m, int64_t kc, double* u,
                      cudaStream_t s) {
  if (m <= 128) return BF_OK;
  int64_t h = ((m / 2 + 127) / 128) * 128;
  if (h >= m) h = m - 128;
  int rc = tri_inverse_t_rec(l, x, o, h, kc, u, s);
  if (!rc) rc = tri_inverse_t_rec(l, x, o + h, m - h, kc, u, s);
  if (rc) return rc;
  const bf_view x11 = subview(x, o, h, o, h), x22 = subview(x, o + h, m - h, o + h, m - h);
  const bf_view x12 = subview(x, o, h, o + h, m - h), b = subview(l, o + h, m - h, o, h);
  const bf_view uv{u, 0, h, m - h, m - h, 1};
  rc = gemm_impl(MODE_D, 1.0, x11, transposed(b), 0.0, uv, 0, kc, nullptr, s);  // U = X11 B^T
  return rc ? rc : gemm_impl(MODE_D, -1.0, uv, x22, 0.0, x12, 0, kc, nullptr, s);  // X12 = -U X22
}
int tri_inverse_t_d(const bf_view& l, const bf_view& x, int64_t kc, cudaStream_t s) {
  const int64_t n = l.n;
  if (n == 0) return BF_OK;
  if (l.cs != 1 || x.cs != 1) return fail(BF_ERR_UNSUPPORTED, "doubling inverse needs unit column strides");
  if (bf::launch_trsm_diag_tiles(static_cast<const double*>(l.base) + l.off, l.rs, static_cast<double*>(x.base) + x.off,
                                 x.rs, n, kc, s))
    return fail(BF_ERR_CUDA, "diagonal tile inverse launch failed");
  if (n <= 128) return BF_OK;
  const int64_t h = ((n / 2 + 127) / 128) * 128;
  double* u = static_cast<double*>(bf::stream_scratch(12, size_t(h) * size_t(n - h) * sizeof(double), s));
  if (!u) return fail(BF_ERR_CUDA, "no scratch for the doubling inverse");
  return tri_inverse_t_rec(l, x, 0, n, kc, u, s);
}
// the mixed driver's diagonal block, g_mixed_inverse = 1: the factor (fused
// when the tree allows), then the doubling inverse
int chol_then_inverse(const bf_view& a, const bf_chol_level* lv, int nl, int64_t base, const bf_view& x, int64_t kc,
                      int* d_info, cudaStream_t st) {
  const int rc = chol_run(MODE_D, a, lv, nl, 0, base, d_info, st);
  return rc ? rc : tri_inverse_t_d(a, x, kc, st);
}

int chol_inverse_overlapped(const bf_view& a, const bf_chol_level* lv, int nl, int64_t base, const bf_view& x,
                            int64_t kc, int* d_info, cudaStream_t st) {
  cudaStream_t st2 = panel2_stream(st);
  if (!(g_panel_overlap && nl >= 1 && lv[0].variant == 3 && lv[0].bs >= 1 && a.n > lv[0].bs && st2)) {
    int rc = chol_run(MODE_D, a, lv, nl, 0, base, d_info, st);
    return rc ? rc : trsm_rec(MODE_D, 1.0, a, x, kc, nullptr, d_info, st);
  }
  const int64_t ns = (a.n + lv[0].bs - 1) / lv[0].bs;
  std::vector<cudaEvent_t> ev(static_cast<size_t>(ns) + 1);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventRecord(ev[size_t(ns)], st);  // X initialised, the block converted
  cudaStreamWaitEvent(st2, ev[size_t(ns)], 0);
  int rc = chol_v3_events(MODE_D, a, lv, nl, 0, base, d_info, st, ev.data());
  if (rc == BF_OK) {
    TriWait w{ev.data(), lv[0].bs, ns};
    rc = trsm_rec_w(MODE_D, 1.0, a, x, kc, d_info, st2, w, 0);
  }
  cudaEventRecord(ev[size_t(ns)], st2);
  cudaStreamWaitEvent(st, ev[size_t(ns)], 0);
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}
// bridges for the other translation units (dist.cu)
int gemm_d_limited(double alpha, const bf_view& a, const bf_view& b, double beta, const bf_view& c, int lower_only,
                   int64_t kc, const int* d_abort, int64_t abort_limit, cudaStream_t s) {
  return gemm_impl(MODE_D, alpha, a, b, beta, c, lower_only, kc, d_abort, s, abort_limit);
}
int set_error(int code, const char* msg) { return fail(code, msg); }
cudaStream_t panel_stream_for(cudaStream_t caller) { return panel_stream(caller); }
}  // namespace bf

extern "C" {

int bf_abi_version(void) { return 1; }
// tools only (not in include/): the last fused diagonal factor's task profile
int bf_fused_diag_stats(int64_t* out9) { return bf::fused_diag_stats(out9); }
int64_t bf_launch_count(void) { return bf::g_launches.load(std::memory_order_relaxed); }
const char* bf_last_error(void) { return g_last_error.c_str(); }

int bf_scratch_stats(int64_t* live_bytes, int64_t* peak_bytes) {
  if (live_bytes) *live_bytes = bf::g_scratch_live.load();
  if (peak_bytes) *peak_bytes = bf::g_scratch_peak.load();
  return BF_OK;
}
int bf_scratch_reset_peak(void) {
  bf::g_scratch_peak.store(bf::g_scratch_live.load());
  return BF_OK;
}

int bf_release_scratch(void) {
  bf::stream_scratch(-1, 0, nullptr);
  return cudaGetLastError() == cudaSuccess ? BF_OK : fail(BF_ERR_CUDA, "release failed");
}
int bf_set_option(const char* name, int64_t value) {
  if (name && std::strcmp(name, "lookahead") == 0) {
    g_lookahead = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tma") == 0) {
    bf::g_use_tma = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tiles_per_cta") == 0 && value >= 0) {
    bf::g_tiles_per_cta = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "timeline") == 0) {
    g_timeline = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "fused_trsm") == 0) {
    g_fused_trsm = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "group") == 0 && value >= 1) {
    g_group = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "panel_tiles") == 0 && value >= 0 && value < (1 << 16)) {
    g_panel_tiles = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "symv") == 0) {
    bf::g_symv = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "potrs_coop") == 0) {
    bf::g_potrs_coop = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "fused_diag") == 0) {
    bf::g_fused_diag = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "fused_diag_pct") == 0 && value >= 1 && value <= 100) {
    g_fused_diag_pct = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "fused_diag_ctas") == 0 && value >= 0) {
    g_fused_diag_ctas = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "potrs_vec") == 0) {
    bf::g_potrs_vec = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "early_panel") == 0) {
    g_early_panel = int(value);  // 1: rows below at full width, 2: with the step's reservation, 3: 1 + step 0
    return BF_OK;
  }
  if (name && std::strcmp(name, "panel_chunks") == 0 && value >= 1 && value <= 8) {
    g_panel_chunks = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "panel_chunk_rows") == 0 && value >= 1) {
    g_panel_chunk_rows = value;
    return BF_OK;
  }
  if (name && std::strcmp(name, "panel_overlap") == 0) {
    g_panel_overlap = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "persist") == 0) {
    bf::g_persist = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "segsplit") == 0) {
    g_segsplit = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "reserve_adaptive") == 0) {
    g_reserve_adaptive = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "reserve_extra") == 0 && value >= 0) {
    g_reserve_extra = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "reserve_min") == 0 && value >= 0) {
    g_reserve_min = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "upper_transpose") == 0 && value >= 0) {
    g_upper_transpose = value;
    return BF_OK;
  }
  if (name && std::strcmp(name, "mixed_inverse") == 0) {
    bf::g_mixed_inverse = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "mixed_reserve") == 0 && value >= 0) {
    bf::g_mixed_reserve = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "tmem_fold") == 0) {
    bf::g_tmem_fold = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "red_fold") == 0) {
    bf::g_red_fold = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tmc_bn64") == 0) {
    bf::g_tmc_bn64 = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tma_bn") == 0 && (value == 128 || value == 64)) {
    bf::g_tma_bn = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "tma_variant") == 0) {
    bf::g_tma_variant = int(value & 3);
    return BF_OK;
  }
  if (name && std::strcmp(name, "overlap_h2d") == 0) {
    g_overlap_h2d = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tail_reserve") == 0 && value >= 0) {
    g_tail_reserve = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "reserve_strided") == 0) {
    bf::g_reserve_strided = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "diag_reserve") == 0 && value >= 0) {
    g_diag_reserve = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "diag_rows") == 0 && value >= 0) {
    g_diag_rows = value;
    return BF_OK;
  }
  if (name && std::strcmp(name, "tail_rows") == 0 && value >= 0) {
    g_tail_rows = value;
    return BF_OK;
  }
  if (name && std::strcmp(name, "pipeline_first") == 0) {
    g_pipeline_first = value < 0 ? 0 : int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "ltlt_grid") == 0 && value >= 0) {
    bf::g_ltlt_grid_max = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "qr_global") == 0) {
    bf::g_qr_global = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "lu_nocluster") == 0) {
    bf::g_lu_nocluster = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "lu_cluster") == 0 && value >= 1 && value <= 16) {
    bf::g_lu_cluster_max = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "lu_noprefetch") == 0) {
    bf::g_lu_noprefetch = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "lu_global") == 0) {
    bf::g_lu_global = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "lu_grid") == 0 && value >= 0) {
    bf::g_lu_grid_max = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "pdl") == 0) {
    bf::g_pdl = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "leaf_pipe") == 0) {
    bf::g_leaf_pipe = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "leaf_blocked") == 0) {
    bf::g_leaf_blocked = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "trsm_warp") == 0) {
    bf::g_trsm_warp = value != 0;
    return BF_OK;
  }
  if (name && std::strcmp(name, "bf16_group") == 0 && value >= 0) {
    bf::g_bf16_group = int(value);
    return BF_OK;
  }
  if (name && std::strcmp(name, "bf16_tma_c") == 0) {
    bf::g_bf16_tma_c = value != 0;
    return BF_OK;
  }
  return fail(BF_ERR_VALUE, "unknown option");
}

int bf_timeline(float* out, int max_steps) {
  // out[5*i + 0..4] = ms from the start to: next-column update done, rest of
  // the trailing update done, panel start, panel end, diagonal factor of the
  // panel done (step i of the last lookahead factorization).  Synchronises on
  // the recorded events.
  int nsteps = int(g_tl.size());
  if (!out || !g_tl_origin) return nsteps;
  for (int i = 0; i < nsteps && i < max_steps; ++i) {
    cudaEvent_t ev[5] = {g_tl[i].main_col, g_tl[i].main_rest, g_tl[i].panel_begin, g_tl[i].panel_end,
                         g_tl[i].panel_diag};
    for (int q = 0; q < 5; ++q) {
      float ms = -1.f;
      if (ev[q] && cudaEventSynchronize(ev[q]) == cudaSuccess) cudaEventElapsedTime(&ms, g_tl_origin, ev[q]);
      out[5 * i + q] = ms;
    }
  }
  return nsteps;
}

int bf_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

#define BF_GEMM_ENTRY(NAME, MODE)                                                                            \
  int NAME(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only, \
           int64_t kc, const int* d_abort, void* stream) {                                                  \
    if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");                                             \
    return gemm_impl(MODE, alpha, *a, *b, beta, *c, lower_only, kc, d_abort, S(stream));                   \
  }
BF_GEMM_ENTRY(bf_gemm_d, MODE_D)
BF_GEMM_ENTRY(bf_gemm_s, MODE_S)
BF_GEMM_ENTRY(bf_gemm_sd, MODE_SD)
#undef BF_GEMM_ENTRY

int bf_scale_d(double beta, const bf_view* c, int lower_only, void* stream) {
  return c ? scale_impl(MODE_D, beta, *c, lower_only, S(stream)) : fail(BF_ERR_VALUE, "null view");
}
int bf_scale_s(double beta, const bf_view* c, int lower_only, void* stream) {
  return c ? scale_impl(MODE_S, double(float(beta)), *c, lower_only, S(stream)) : fail(BF_ERR_VALUE, "null view");
}
int bf_scale_sd(double beta, const bf_view* c, int lower_only, void* stream) {
  return c ? scale_impl(MODE_SD, beta, *c, lower_only, S(stream)) : fail(BF_ERR_VALUE, "null view");
}

int bf_potrf_leaf_d(const bf_view* a, int variant, int64_t base_index, int* d_info, void* stream) {
  return a ? leaf_impl(MODE_D, *a, variant, base_index, d_info, S(stream)) : fail(BF_ERR_VALUE, "null view");
}
int bf_potrf_leaf_s(const bf_view* a, int variant, int64_t base_index, int* d_info, void* stream) {
  return a ? leaf_impl(MODE_S, *a, variant, base_index, d_info, S(stream)) : fail(BF_ERR_VALUE, "null view");
}

int bf_trsm_rltn_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular, void* stream) {
  return trsm_impl(MODE_D, alpha, tri, b, kc, d_singular, S(stream));
}
int bf_trsm_rltn_s(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular, void* stream) {
  return trsm_impl(MODE_S, alpha, tri, b, kc, d_singular, S(stream));
}

int bf_cholesky_ex_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t base_index, int* d_info,
                     void* stream) {
  if (!a || !levels || nlevels < 1) return fail(BF_ERR_VALUE, "null argument");
  if (a->m != a->n) return fail(BF_ERR_SHAPE, "square matrix required");
  return chol_run(MODE_D, *a, levels, nlevels, 0, base_index, d_info, S(stream));
}
int bf_trsm_rltn_ex_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular,
                      const int* d_abort, void* stream) {
  if (!tri || !b) return fail(BF_ERR_VALUE, "null view");
  if (tri->m != tri->n) return fail(BF_ERR_SHAPE, "triangular operand must be square");
  if (b->n != tri->n) return fail(BF_ERR_SHAPE, "right solve dims mismatch");
  return trsm_rec(MODE_D, alpha, *tri, *b, kc, d_singular, d_abort, S(stream));
}

int bf_cholesky_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int* d_info, void* stream) {
  return chol_impl(MODE_D, a, levels, nlevels, d_info, S(stream));
}
int bf_cholesky_host_d(double* host, int64_t ld, const bf_view* work, const bf_chol_level* levels, int nlevels,
                       int* d_info, void* stream) {
  if (!host || !work || !levels || nlevels < 1) return fail(BF_ERR_VALUE, "null argument");
  if (work->m != work->n) return fail(BF_ERR_SHAPE, "square matrix required");
  if (work->cs != 1 || work->rs < work->n || ld < work->n) return fail(BF_ERR_UNSUPPORTED, "row-major work and host");
  const int64_t n = work->n;
  if (n == 0) return BF_OK;
  cudaStream_t s = S(stream);
  cudaStream_t cs = copy_stream(s);
  if (!cs) return fail(BF_ERR_CUDA, "cannot create the copy stream");
  double* dev = static_cast<double*>(work->base) + work->off;
  // lower triangle in, by block columns of the root bs (rows >= the column's
  // first).  With the lookahead driver the copies run on their own stream and
  // step 0 consumes each block column as it lands; otherwise in stream order.
  const int64_t bs = levels[0].bs >= 1 ? levels[0].bs : n;
  const bool overlap = g_lookahead && g_overlap_h2d && levels[0].variant == 3 && n > 2 * bs && !g_pipeline_first;
  cudaStream_t hs = overlap ? h2d_stream(s) : s;
  if (overlap && !hs) return fail(BF_ERR_CUDA, "cannot create the h2d stream");
  HostLoad hl;
  hl.bs = bs;
  if (overlap) {
    cudaEvent_t start;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventRecord(start, s);  // the work buffer is free once the caller's prior work is done
    cudaStreamWaitEvent(hs, start, 0);
    cudaEventDestroy(start);
  }
  // Every exit below joins the h2d and copy streams into s first, so when the
  // caller's stream completes no copy into or out of the host matrix is
  // still in flight (also after an error), and destroys the load events.
  auto join = [&](cudaStream_t from) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(s, e, 0);
    cudaEventDestroy(e);
  };
  auto finish = [&](int code) {
    if (overlap) join(hs);
    join(cs);
    for (auto e : hl.ev) cudaEventDestroy(e);
    hl.ev.clear();
    return code;
  };
  for (int64_t c0 = 0; c0 < n; c0 += bs) {
    const int64_t w = bs < n - c0 ? bs : n - c0;
    if (cudaMemcpy2DAsync(dev + c0 * work->rs + c0, size_t(work->rs) * 8, host + c0 * ld + c0, size_t(ld) * 8,
                          size_t(w) * 8, size_t(n - c0), cudaMemcpyHostToDevice, hs) != cudaSuccess)
      return finish(fail(BF_ERR_CUDA, "host to device copy failed"));
    if (overlap) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      cudaEventRecord(e, hs);
      hl.ev.push_back(e);
    }
  }
  HostWriteback wb;
  wb.host = host;
  wb.ld = ld;
  wb.cs = cs;
  g_wb = &wb;
  g_h2d = overlap ? &hl : nullptr;
  int rc = chol_impl(MODE_D, work, levels, nlevels, d_info, s);
  g_wb = nullptr;
  g_h2d = nullptr;
  if (rc) return finish(rc);
  // whatever the lookahead did not stream back (the non-lookahead path, or all of it)
  for (int64_t c0 = wb.copied_upto; c0 < n; c0 += bs) {
    const int64_t w = bs < n - c0 ? bs : n - c0;
    cudaMemcpy2DAsync(host + c0 * ld + c0, size_t(ld) * 8, dev + c0 * work->rs + c0, size_t(work->rs) * 8,
                      size_t(w) * 8, size_t(n - c0), cudaMemcpyDeviceToHost, s);
  }
  finish(BF_OK);
  return cudaGetLastError() == cudaSuccess ? BF_OK : fail(BF_ERR_CUDA, "host factorization copies failed");
}
int bf_lu_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t* d_piv, int* d_sing, void* stream) {
  if (!a || !levels || nlevels < 1 || !d_piv || !d_sing) return fail(BF_ERR_VALUE, "null argument");
  if (g_lookahead && nlevels >= 1 && levels[0].variant == 20 && levels[0].bs >= 1 &&
      (a->m < a->n ? a->m : a->n) > 2 * levels[0].bs)
    return lu_lookahead(MODE_D, *a, levels, nlevels, d_piv, d_sing, S(stream));
  return lu_run(MODE_D, *a, levels, nlevels, 0, d_piv, 0, d_sing, S(stream));
}
int bf_lu_s(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t* d_piv, int* d_sing, void* stream) {
  if (!a || !levels || nlevels < 1 || !d_piv || !d_sing) return fail(BF_ERR_VALUE, "null argument");
  if (g_lookahead && nlevels >= 1 && levels[0].variant == 20 && levels[0].bs >= 1 &&
      (a->m < a->n ? a->m : a->n) > 2 * levels[0].bs)
    return lu_lookahead(MODE_S, *a, levels, nlevels, d_piv, d_sing, S(stream));
  return lu_run(MODE_S, *a, levels, nlevels, 0, d_piv, 0, d_sing, S(stream));
}
int bf_trsm_llnu_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, void* stream) {
  if (!tri || !b) return fail(BF_ERR_VALUE, "null view");
  if (tri->m != tri->n || b->m != tri->n) return fail(BF_ERR_SHAPE, "left solve dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  return trsm_left_rec(MODE_D, alpha, *tri, *b, kc, S(stream));
}
int bf_trsm_llnu_s(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, void* stream) {
  if (!tri || !b) return fail(BF_ERR_VALUE, "null view");
  if (tri->m != tri->n || b->m != tri->n) return fail(BF_ERR_SHAPE, "left solve dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  return trsm_left_rec(MODE_S, alpha, *tri, *b, kc, S(stream));
}
int bf_trsm_lun_d(const bf_view* u, const bf_view* b, int64_t kc, void* stream) {
  if (!u || !b) return fail(BF_ERR_VALUE, "null view");
  if (u->m != u->n || b->m != u->n) return fail(BF_ERR_SHAPE, "upper solve dims mismatch");
  return trsm_upper_rec(MODE_D, *u, *b, kc < 1 ? 256 : kc, S(stream));
}
int bf_trsm_lun_s(const bf_view* u, const bf_view* b, int64_t kc, void* stream) {
  if (!u || !b) return fail(BF_ERR_VALUE, "null view");
  if (u->m != u->n || b->m != u->n) return fail(BF_ERR_SHAPE, "upper solve dims mismatch");
  return trsm_upper_rec(MODE_S, *u, *b, kc < 1 ? 512 : kc, S(stream));
}
int bf_apply_pivots_d(const bf_view* a, const int64_t* d_piv, int64_t count, int backward, void* stream) {
  if (!a || (count > 0 && !d_piv)) return fail(BF_ERR_VALUE, "null argument");
  return apply_pivots_impl(MODE_D, *a, d_piv, count, 0, backward, S(stream));
}
int bf_apply_pivots_s(const bf_view* a, const int64_t* d_piv, int64_t count, int backward, void* stream) {
  if (!a || (count > 0 && !d_piv)) return fail(BF_ERR_VALUE, "null argument");
  return apply_pivots_impl(MODE_S, *a, d_piv, count, 0, backward, S(stream));
}
// lower(C) := C - A T A^T, T skew tridiagonal with subdiagonal t (engine/gemm.py:245-280)
int bf_sandwich_skew_d(const bf_view* c, const bf_view* a, const double* d_t, int64_t kc, void* stream) {
  if (!c || !a) return fail(BF_ERR_VALUE, "null view");
  if (c->m != c->n) return fail(BF_ERR_SHAPE, "sandwich needs square c");
  if (a->m != c->m) return fail(BF_ERR_SHAPE, "sandwich dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  const int64_t n = c->m, kt = a->n;
  if (n == 0 || kt == 0) return BF_OK;
  if (kt > 1 && !d_t) return fail(BF_ERR_VALUE, "null tridiagonal vector");
  GemmParams p{};
  p.m = n;
  p.n = n;
  p.k = kt;
  p.kc = kc;
  p.a = classify(a->base, a->off, a->rs, a->cs, n, kt, kc, MODE_D);
  OperandMK b{};
  b.base = a->base;  // B = T * A^T: B's (n, k) source element is a(n, k)
  b.off = a->off;
  b.s_mn = a->rs;
  b.s_k = a->cs;
  b.layout = bf::GL_TRIDIAG;
  b.vec = 1;
  b.tvec = d_t;
  b.k_total = kt;
  p.b = b;
  p.c = c->base;
  p.c_off = c->off;
  p.c_rs = c->rs;
  p.c_cs = c->cs;
  p.alpha = -1.0;
  p.beta = 1.0;
  p.lower_only = 1;
  p.abort_flag = nullptr;
  p.abort_limit = -1;
  const int rc = bf::launch_gemm_dmma(p, S(stream));
  return rc ? fail(BF_ERR_CUDA, "sandwich launch failed") : BF_OK;
}

// f32 storage: the reference packs W in f32 (acc dtype f32); the SIMT kernel's
// B loader forms each staged element of W = T*A^T from two source elements, so
// no k x n intermediate exists (d_w is unused and may be NULL: kept for ABI
// compatibility)
int bf_sandwich_skew_s(const bf_view* c, const bf_view* a, const float* d_t, float* d_w, int64_t kc, void* stream) {
  (void)d_w;
  if (!c || !a) return fail(BF_ERR_VALUE, "null view");
  if (c->m != c->n) return fail(BF_ERR_SHAPE, "sandwich needs square c");
  if (a->m != c->m) return fail(BF_ERR_SHAPE, "sandwich dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  const int64_t n = c->m, kt = a->n;
  if (n == 0 || kt == 0) return BF_OK;
  if (kt > 1 && !d_t) return fail(BF_ERR_VALUE, "null tridiagonal vector");
  GemmParams p{};
  p.m = n;
  p.n = n;
  p.k = kt;
  p.kc = kc;
  p.a = classify(a->base, a->off, a->rs, a->cs, n, kt, kc, MODE_S);
  OperandMK b{};
  b.base = a->base;
  b.off = a->off;
  b.s_mn = a->rs;
  b.s_k = a->cs;
  b.layout = bf::GL_TRIDIAG;
  b.vec = 1;
  b.tvec = reinterpret_cast<const double*>(d_t);  // read as float by the f32 loader
  b.k_total = kt;
  p.b = b;
  p.c = c->base;
  p.c_off = c->off;
  p.c_rs = c->rs;
  p.c_cs = c->cs;
  p.alpha = -1.0;
  p.beta = 1.0;
  p.lower_only = 1;
  p.abort_limit = -1;
  const int rc = bf::launch_gemm_simt_f32(p, S(stream));
  return rc ? fail(BF_ERR_CUDA, "sandwich launch failed") : BF_OK;
}
static int ltlt_entry(int is_f64, const bf_view* x, int64_t j0, int64_t j1, int blocked, int64_t k, void* w,
                      int64_t wld, int64_t* d_piv, void* d_t, void* d_m, void* d_w, void* stream) {
  if (!x || !d_piv || !d_t) return fail(BF_ERR_VALUE, "null argument");
  if (x->m != x->n) return fail(BF_ERR_SHAPE, "square matrix required");
  if (j0 < 0 || j1 > x->n - 1 || j0 > j1) return fail(BF_ERR_VALUE, "bad elimination range");
  if (blocked ? (!w || wld < 1) : (!d_m || !d_w)) return fail(BF_ERR_VALUE, "null workspace");
  int rc = bf::launch_ltlt(is_f64, x->base, x->off, x->rs, x->cs, x->n, j0, j1, blocked, k, w, wld, d_piv, d_t, d_m,
                           d_w, S(stream));
  return rc ? fail(BF_ERR_CUDA, "ltlt launch failed") : BF_OK;
}
int bf_ltlt_d(const bf_view* x, int64_t j0, int64_t j1, int blocked, int64_t k, double* w, int64_t wld,
              int64_t* d_piv, double* d_t, double* d_m, double* d_w, void* stream) {
  return ltlt_entry(1, x, j0, j1, blocked, k, w, wld, d_piv, d_t, d_m, d_w, stream);
}
int bf_ltlt_s(const bf_view* x, int64_t j0, int64_t j1, int blocked, int64_t k, float* w, int64_t wld,
              int64_t* d_piv, float* d_t, float* d_m, float* d_w, void* stream) {
  return ltlt_entry(0, x, j0, j1, blocked, k, w, wld, d_piv, d_t, d_m, d_w, stream);
}
// ---- split-K GEMM (QR's reflector products) ---------------------------------
// For the tall-K products of the QR path (V^T V, V^T C: a handful of output
// tiles, K = the panel height) the K range is cut into S slices that run
// concurrently on forked streams into a workspace, then summed in slice
// order.  The reference forms these with NumPy/BLAS (factor/qr.py:81-121),
// so they are parity-to-rounding products, never used on a bitwise path.
static int gemm_splitk_impl(Mode mode, double alpha, const bf_view& a, const bf_view& b, double beta,
                            const bf_view& c, cudaStream_t s) {
  constexpr int SMAX = 16;
  const int64_t m = c.m, n = c.n, k = a.n;
  if (a.n != b.m || c.m != a.m || c.n != b.n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(BF_ERR_CUDA, "device index");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ((m + 127) / 128) * ((n + 127) / 128);
  int64_t S = tiles > 0 ? sms / tiles : 1;
  if (S > SMAX) S = SMAX;
  if (S > k / 512) S = k / 512;
  if (S <= 1 || m == 0 || n == 0) return gemm_impl(mode, alpha, a, b, beta, c, 0, int64_t(1) << 40, nullptr, s);
  // side streams, events and workspace per (device, calling stream): QR's
  // lookahead issues split-K products from two streams at once
  struct Ctx {
    int dev;
    cudaStream_t owner;
    cudaStream_t side[SMAX];
    cudaEvent_t ev[SMAX + 1];
    void* ws;
    size_t bytes;
  };
  static std::vector<Ctx*> ctxs;
  static std::mutex mu;
  Ctx* cx = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (Ctx* c : ctxs)
      if (c->dev == dev && c->owner == s) cx = c;
    if (!cx) {
      cx = new Ctx{};
      cx->dev = dev;
      cx->owner = s;
      for (int i = 0; i < SMAX; ++i) {
        cudaStreamCreateWithFlags(&cx->side[i], cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&cx->ev[i], cudaEventDisableTiming);
      }
      cudaEventCreateWithFlags(&cx->ev[SMAX], cudaEventDisableTiming);
      ctxs.push_back(cx);
    }
  }
  const size_t need = size_t(S) * size_t(m) * size_t(n) * size_t(elem_bytes(mode));
  if (need > cx->bytes) {
    if (cx->ws) {
      cudaStreamSynchronize(s);
      cudaFree(cx->ws);
    }
    cx->ws = nullptr;
    cx->bytes = 0;
    if (cudaMalloc(&cx->ws, need) != cudaSuccess) return fail(BF_ERR_CUDA, "split-K workspace");
    cx->bytes = need;
  }
  cudaEventRecord(cx->ev[SMAX], s);
  const int64_t slice = (k + S - 1) / S;
  for (int64_t q = 0; q < S; ++q) {
    const int64_t k0 = q * slice, kn = k0 + slice < k ? slice : k - k0;
    cudaStream_t sq = cx->side[q];
    cudaStreamWaitEvent(sq, cx->ev[SMAX], 0);
    bf_view w{};
    w.base = cx->ws;
    w.off = q * m * n;
    w.m = m;
    w.n = n;
    w.rs = n;
    w.cs = 1;
    int rc = gemm_impl(mode, 1.0, subview(a, 0, m, k0, kn), subview(b, k0, kn, 0, n), 0.0, w, 0, int64_t(1) << 40,
                       nullptr, sq);
    if (rc) return rc;
    cudaEventRecord(cx->ev[q], sq);
    cudaStreamWaitEvent(s, cx->ev[q], 0);
  }
  double al = alpha, be = beta;
  if (mode == MODE_S) {
    al = double(float(alpha));
    be = double(float(beta));
  }
  int rc = bf::launch_splitk_reduce(storage_is_f64(mode), cx->ws, int(S), m, n, al, be, c.base, c.off, c.rs, c.cs, s);
  return rc ? fail(BF_ERR_CUDA, "split-K reduce launch failed") : BF_OK;
}
int bf_gemm_splitk_d(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, void* stream) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  return gemm_splitk_impl(MODE_D, alpha, *a, *b, beta, *c, S(stream));
}
int bf_gemm_splitk_s(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, void* stream) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  return gemm_splitk_impl(MODE_S, alpha, *a, *b, beta, *c, S(stream));
}

// ---- Householder QR (factor/qr.py) -----------------------------------------
static int qr_panel_entry(int is_f64, const bf_view* a, void* d_taus, void* stream) {
  if (!a || !d_taus) return fail(BF_ERR_VALUE, "null argument");
  if (a->m < a->n) return fail(BF_ERR_SHAPE, "qr requires m >= n");
  int rc = bf::launch_qr_panel(is_f64, a->base, a->off, a->rs, a->cs, a->m, a->n, d_taus, S(stream));
  return rc ? fail(BF_ERR_CUDA, "qr panel launch failed") : BF_OK;
}
int bf_qr_panel_d(const bf_view* a, double* d_taus, void* stream) { return qr_panel_entry(1, a, d_taus, stream); }
int bf_qr_panel_s(const bf_view* a, float* d_taus, void* stream) { return qr_panel_entry(0, a, d_taus, stream); }
static int qr_t_entry(int is_f64, const bf_view* panel, const void* d_taus, void* d_t, void* d_v, void* d_gram,
                      void* stream) {
  if (!panel || !d_taus || !d_t || !d_v || !d_gram) return fail(BF_ERR_VALUE, "null argument");
  const int64_t m = panel->m, b = panel->n;
  cudaStream_t s = S(stream);
  int rc = bf::launch_explicit_v(is_f64, panel->base, panel->off, panel->rs, panel->cs, m, b, d_v, s);
  if (rc) return fail(BF_ERR_CUDA, "qr V launch failed");
  // G = V^T V (b x b) on the engine GEMM; T from G
  bf_view v{};
  v.base = d_v;
  v.off = 0;
  v.m = m;
  v.n = b;
  v.rs = b;
  v.cs = 1;
  bf_view g{};
  g.base = d_gram;
  g.off = 0;
  g.m = b;
  g.n = b;
  g.rs = b;
  g.cs = 1;
  const Mode mode = is_f64 ? MODE_D : MODE_S;
  rc = gemm_splitk_impl(mode, 1.0, transposed(v), v, 0.0, g, s);
  if (rc) return rc;
  rc = bf::launch_qr_t(is_f64, d_gram, b, d_taus, d_t, s);
  return rc ? fail(BF_ERR_CUDA, "qr T launch failed") : BF_OK;
}
int bf_qr_t_d(const bf_view* panel, const double* d_taus, double* d_t, double* d_v, double* d_gram, void* stream) {
  return qr_t_entry(1, panel, d_taus, d_t, d_v, d_gram, stream);
}
int bf_qr_t_s(const bf_view* panel, const float* d_taus, float* d_t, float* d_v, float* d_gram, void* stream) {
  return qr_t_entry(0, panel, d_taus, d_t, d_v, d_gram, stream);
}
static int reflector_entry(int is_f64, const bf_view* a, int64_t j, double tau, const bf_view* c, void* stream) {
  if (!a || !c) return fail(BF_ERR_VALUE, "null view");
  if (c->m != a->m) return fail(BF_ERR_SHAPE, "c rows != a rows");
  int rc = bf::launch_reflector_apply(is_f64, a->base, a->off, a->rs, a->cs, a->m, j, tau, c->base, c->off, c->rs,
                                      c->cs, c->n, S(stream));
  return rc ? fail(BF_ERR_CUDA, "reflector launch failed") : BF_OK;
}
int bf_reflector_apply_d(const bf_view* a, int64_t j, double tau, const bf_view* c, void* stream) {
  return reflector_entry(1, a, j, tau, c, stream);
}
int bf_reflector_apply_s(const bf_view* a, int64_t j, double tau, const bf_view* c, void* stream) {
  return reflector_entry(0, a, j, tau, c, stream);
}
int bf_cholesky_s(const bf_view* a, const bf_chol_level* levels, int nlevels, int* d_info, void* stream) {
  return chol_impl(MODE_S, a, levels, nlevels, d_info, S(stream));
}

int bf_gemm_bf16(double alpha, const void* a, int64_t lda, const void* b, int64_t ldb, double beta, const bf_view* c,
                 int64_t k, int lower_only, void* stream) {
  if (!c) return fail(BF_ERR_VALUE, "null view");
  if (lower_only && c->m != c->n) return fail(BF_ERR_SHAPE, "gemmt needs square c");
  int rc = bf::launch_gemm_bf16_tc(alpha, a, lda, b, ldb, beta, static_cast<float*>(c->base), c->off, c->rs, c->cs,
                                   c->m, c->n, k, lower_only, S(stream));
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "bf16 gemm: operands must be 16-byte aligned k-contiguous bf16");
  return rc ? fail(BF_ERR_CUDA, "bf16 gemm launch failed") : BF_OK;
}
int bf_gemm_tf32(double alpha, const float* a, int64_t lda, const float* b, int64_t ldb, double beta, const bf_view* c,
                 int64_t k, int lower_only, void* stream) {
  if (!c) return fail(BF_ERR_VALUE, "null view");
  if (lower_only && c->m != c->n) return fail(BF_ERR_SHAPE, "gemmt needs square c");
  int rc = bf::launch_gemm_tf32_tc(alpha, a, lda, b, ldb, beta, static_cast<float*>(c->base), c->off, c->rs, c->cs,
                                   c->m, c->n, k, lower_only, S(stream));
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "tf32 gemm: operands must be 16-byte aligned k-contiguous fp32");
  return rc ? fail(BF_ERR_CUDA, "tf32 gemm launch failed") : BF_OK;
}
static int split_entry(int f64, const bf_view* src, float* dst, int64_t ld, int64_t kp, void* stream) {
  if (!src || !dst) return fail(BF_ERR_VALUE, "null argument");
  if (kp < src->n || ld < 4 * kp) return fail(BF_ERR_SHAPE, "split needs kp >= k and ld >= 4 kp");
  int rc = bf::launch_split_tf32(f64, src->base, src->off, src->rs, src->cs, dst, ld, src->m, src->n, kp, S(stream));
  return rc ? fail(BF_ERR_CUDA, "split launch failed") : BF_OK;
}
int bf_split_tf32_s(const bf_view* src, float* dst, int64_t ld, int64_t kp, void* stream) {
  return split_entry(0, src, dst, ld, kp, stream);
}
int bf_split_tf32_d(const bf_view* src, float* dst, int64_t ld, int64_t kp, void* stream) {
  return split_entry(1, src, dst, ld, kp, stream);
}
// C(f32) := beta C + alpha A B (A m x k, B k x n fp32 views) as ONE K = 3k
// tf32 GEMM over the split operands (workspace owned by the library)
int bf_gemm_f32_tc(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only,
                   void* stream) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  if (a->n != b->m || c->m != a->m || c->n != b->n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  if (lower_only && c->m != c->n) return fail(BF_ERR_SHAPE, "gemmt needs square c");
  const int64_t m = c->m, n = c->n, k = a->n;
  if (m == 0 || n == 0) return BF_OK;
  cudaStream_t s = S(stream);
  if (k == 0 || alpha == 0.0) return scale_impl(MODE_S, beta, *c, lower_only, s);
  const int64_t kp = (k + 3) / 4 * 4, ld = 4 * kp;
  const size_t need = size_t(m + n) * size_t(ld) * sizeof(float);
  float* sa = static_cast<float*>(bf::stream_scratch(1, need, s));  // private to this stream
  if (!sa) return fail(BF_ERR_CUDA, "tf32 split workspace");
  float* sb = sa + m * ld;
  int rc = bf::launch_split_tf32(0, a->base, a->off, a->rs, a->cs, sa, ld, m, k, kp, s);
  const bf_view bt = transposed(*b);  // rows of B^T: the k-contiguous N x K operand
  if (!rc) rc = bf::launch_split_tf32(0, bt.base, bt.off, bt.rs, bt.cs, sb, ld, n, k, kp, s);
  if (rc) return fail(BF_ERR_CUDA, "split launch failed");
  // A' = [hi hi lo] (columns 0..3kp of sa), B' = [hi lo hi] (columns kp..4kp of sb)
  rc = bf::launch_gemm_tf32_tc(alpha, sa, ld, sb + kp, ld, beta, static_cast<float*>(c->base), c->off, c->rs, c->cs, m,
                               n, 3 * kp, lower_only, s);
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "tf32 gemm: unsupported layout");
  return rc ? fail(BF_ERR_CUDA, "tf32 gemm launch failed") : BF_OK;
}
int bf_convert_f32_bf16(const bf_view* src, void* dst, int64_t ld, int transpose, void* stream) {
  if (!src) return fail(BF_ERR_VALUE, "null view");
  int rc = bf::launch_to_bf16(static_cast<const float*>(src->base), src->off, src->rs, src->cs, dst, ld, src->m,
                              src->n, transpose, S(stream));
  return rc ? fail(BF_ERR_CUDA, "conversion launch failed") : BF_OK;
}
int bf_convert_f64_f32(const bf_view* src, const bf_view* dst, int lower_only, void* stream) {
  if (!src || !dst) return fail(BF_ERR_VALUE, "null view");
  if (src->m != dst->m || src->n != dst->n) return fail(BF_ERR_SHAPE, "conversion dims mismatch");
  int rc = bf::launch_f64_to_f32(static_cast<const double*>(src->base), src->off, src->rs, src->cs,
                                 static_cast<float*>(dst->base), dst->off, dst->rs, dst->cs, src->m, src->n, lower_only,
                                 S(stream));
  return rc ? fail(BF_ERR_CUDA, "conversion launch failed") : BF_OK;
}
int bf_convert_f32_f64(const bf_view* src, const bf_view* dst, int lower_only, void* stream) {
  if (!src || !dst) return fail(BF_ERR_VALUE, "null view");
  if (src->m != dst->m || src->n != dst->n) return fail(BF_ERR_SHAPE, "conversion dims mismatch");
  int rc = bf::launch_f32_to_f64(static_cast<const float*>(src->base), src->off, src->rs, src->cs,
                                 static_cast<double*>(dst->base), dst->off, dst->rs, dst->cs, src->m, src->n,
                                 lower_only, S(stream));
  return rc ? fail(BF_ERR_CUDA, "conversion launch failed") : BF_OK;
}
int bf_convert_f64_bf16(const bf_view* src, void* dst, int64_t ld, int transpose, void* stream) {
  if (!src) return fail(BF_ERR_VALUE, "null view");
  int rc = bf::launch_f64_to_bf16(static_cast<const double*>(src->base), src->off, src->rs, src->cs, dst, ld, src->m,
                                  src->n, transpose, S(stream));
  return rc ? fail(BF_ERR_CUDA, "conversion launch failed") : BF_OK;
}
int bf_row_abs_sum_d(const double* a, int64_t lda, double* out, int64_t n, void* stream) {
  int rc = bf::launch_row_abs_sum(a, lda, out, n, S(stream));
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "row sums need a 16-byte aligned A with even lda");
  return rc ? fail(BF_ERR_CUDA, "row sum launch failed") : BF_OK;
}
int bf_residual_d(const double* a, int64_t lda, const double* x, const double* b, double* r, int64_t n, void* stream) {
  int rc = bf::launch_residual(a, lda, x, b, r, n, S(stream));
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "residual needs a 16-byte aligned A with even lda");
  return rc ? fail(BF_ERR_CUDA, "residual launch failed") : BF_OK;
}
int bf_potrs_blocked_f32_d(const float* l, int64_t ld, const float* xinv, int64_t bs, double* x, int64_t n,
                           double* work, void* stream) {
  if (bs <= 0) return fail(BF_ERR_VALUE, "bs must be positive");
  int rc = bf::launch_potrs_blocked(l, ld, xinv, bs, x, n, work, S(stream));
  return rc ? fail(BF_ERR_CUDA, "potrs launch failed") : BF_OK;
}
int bf_potrs_f32_d(const float* l, int64_t ld, double* x, int64_t n, void* stream) {
  int rc = bf::launch_potrs_f32_f64(l, ld, x, n, S(stream));
  return rc ? fail(BF_ERR_CUDA, "potrs launch failed") : BF_OK;
}

int bf_gemm_scatter_d(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                      const bf_scatter_view* c, int64_t kc, void* stream) {
  return scatter_impl(MODE_D, alpha, a, b, beta, c, kc, S(stream));
}
// bf16 variant of the contraction GEMM (no reference counterpart; SURVEY.md
// §8(b) bf_contract_x): operands rounded to bf16, products accumulated in fp32
// on tcgen05 (TMEM), C := beta*C + alpha*(A B) in FP64.  A (M x K) and B (K x N)
// are strided views (the folded facades); scratch: bf16 copies of A and B^T
// (k-contiguous, rows padded to 16 bytes) and the fp32 product.
int bf_contract_bf16_d(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c,
                       void* stream) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  if (a->n != b->m || c->m != a->m || c->n != b->n) return fail(BF_ERR_SHAPE, "gemm dims mismatch");
  const int64_t m = c->m, n = c->n, k = a->n;
  if (m == 0 || n == 0) return BF_OK;
  cudaStream_t s = S(stream);
  if (k == 0 || alpha == 0.0) return scale_impl(MODE_D, beta, *c, 0, s);
  const int64_t kp = (k + 7) / 8 * 8;  // 16-byte bf16 rows for TMA
  const size_t bytes = size_t(m + n) * size_t(kp) * 2 + size_t(m) * size_t(n) * 4 + 256;
  char* ws = static_cast<char*>(bf::stream_scratch(4, bytes, s));
  if (!ws) return fail(BF_ERR_CUDA, "bf16 contraction scratch");
  void* a16 = ws;
  void* b16 = ws + size_t(m) * kp * 2;
  float* prod = reinterpret_cast<float*>(ws + (size_t(m + n) * kp * 2 + 255) / 256 * 256);
  if (kp != k) cudaMemsetAsync(ws, 0, size_t(m + n) * kp * 2, s);  // zero k padding: 0 * 0 adds nothing
  int rc = bf::launch_f64_to_bf16(static_cast<const double*>(a->base), a->off, a->rs, a->cs, a16, kp, m, k, 0, s);
  if (!rc) rc = bf::launch_f64_to_bf16(static_cast<const double*>(b->base), b->off, b->rs, b->cs, b16, kp, k, n, 1, s);
  if (!rc) rc = bf::launch_gemm_bf16_tc(1.0, a16, kp, b16, kp, 0.0, prod, 0, n, 1, m, n, kp, 0, s);
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "bf16 contraction: unsupported size");
  if (!rc) rc = bf::launch_axpby_f32_f64(alpha, prod, n, beta, static_cast<double*>(c->base), c->off, c->rs, c->cs, m, n,
                                         s);
  return rc ? fail(BF_ERR_CUDA, "bf16 contraction launch failed") : BF_OK;
}

// tensor/contract.py:159-185 contract on mode-group views: the 4-D TMA GEMM
int bf_contract_modes_d(double alpha, const bf_modes_view* a, const bf_modes_view* b, double beta,
                        const bf_modes_view* c, int64_t kc, void* stream) {
  if (!a || !b || !c) return fail(BF_ERR_VALUE, "null view");
  for (const bf_modes_view* v : {a, b, c})
    if (v->nr < 1 || v->nr > 2 || v->nc < 1 || v->nc > 2) return fail(BF_ERR_UNSUPPORTED, "1 or 2 mode groups per side");
  auto size = [](int n, const int64_t* d) { return n == 2 ? d[0] * d[1] : d[0]; };
  const int64_t m = size(a->nr, a->rdim), k = size(a->nc, a->cdim), n = size(b->nc, b->cdim);
  if (size(b->nr, b->rdim) != k || size(c->nr, c->rdim) != m || size(c->nc, c->cdim) != n)
    return fail(BF_ERR_SHAPE, "contraction facade dims mismatch");
  if (kc < 1) return fail(BF_ERR_VALUE, "kc must be >= 1");
  if (m == 0 || n == 0) return BF_OK;
  if (k == 0 || alpha == 0.0) return fail(BF_ERR_UNSUPPORTED, "edge case: use the scatter path");
  // A (M x K): rows = M groups, columns = K groups; B^T (N x K): B's columns are its rows
  auto op = [](const void* base, int64_t off, int nmn, const int64_t* mdim, const int64_t* mstr, int nk,
               const int64_t* kdim, const int64_t* kstr, bf::ModeOperand& o) {
    if (kstr[nk - 1] != 1) return false;  // fastest K group must be unit-stride
    o.base = static_cast<const double*>(base);
    o.off = off;
    o.mi = mdim[nmn - 1];
    o.s_mn = mstr[nmn - 1];
    o.s_mn_o = nmn == 2 ? mstr[0] : 0;
    o.ki = kdim[nk - 1];
    o.s_k_o = nk == 2 ? kstr[0] : 0;
    return true;
  };
  bf::ModeOperand ma{}, mb{};
  if (!op(a->base, a->off, a->nr, a->rdim, a->rstr, a->nc, a->cdim, a->cstr, ma) ||
      !op(b->base, b->off, b->nc, b->cdim, b->cstr, b->nr, b->rdim, b->rstr, mb))
    return fail(BF_ERR_UNSUPPORTED, "an operand's fastest contracted mode is not unit-stride");
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.kc = kc;
  p.c = c->base;
  p.c_off = c->off;
  if (m > 0x7fffffffLL || n > 0x7fffffffLL) return fail(BF_ERR_UNSUPPORTED, "facade larger than 2^31");
  p.c_ri = bf::FastDiv(uint32_t(c->nr == 2 ? c->rdim[1] : m));
  p.c_rs = c->rstr[c->nr - 1];
  p.c_rs_o = c->nr == 2 ? c->rstr[0] : 0;
  p.c_ci = bf::FastDiv(uint32_t(c->nc == 2 ? c->cdim[1] : n));
  p.c_cs = c->cstr[c->nc - 1];
  p.c_cs_o = c->nc == 2 ? c->cstr[0] : 0;
  p.alpha = alpha;
  p.beta = beta;
  p.group = g_group;
  int rc = bf::launch_gemm_dmma_modes(p, ma, mb, S(stream));
  if (rc == -3) return fail(BF_ERR_UNSUPPORTED, "mode-group layout not TMA-loadable");
  return rc ? fail(BF_ERR_CUDA, "mode-group gemm launch failed") : BF_OK;
}
int bf_pack_scatter_d(const bf_scatter_view* src, int transpose, double* out, void* stream) {
  if (!src || !out) return fail(BF_ERR_VALUE, "null argument");
  if (src->m < 0 || src->n < 0) return fail(BF_ERR_SHAPE, "negative extent");
  if (src->m == 0 || src->n == 0) return BF_OK;
  if (!src->rscat || !src->cscat) return fail(BF_ERR_VALUE, "scatter vectors required");
  const int rc = transpose ? bf::launch_pack_scatter(1, src->base, src->cscat, src->rscat, src->n, src->m, out, S(stream))
                           : bf::launch_pack_scatter(1, src->base, src->rscat, src->cscat, src->m, src->n, out, S(stream));
  return rc ? fail(BF_ERR_CUDA, "pack launch failed") : BF_OK;
}
int bf_gemm_scatter_s(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                      const bf_scatter_view* c, int64_t kc, void* stream) {
  return scatter_impl(MODE_S, alpha, a, b, beta, c, kc, S(stream));
}
int bf_gemm_scatter_sd(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                       const bf_scatter_view* c, int64_t kc, void* stream) {
  return scatter_impl(MODE_SD, alpha, a, b, beta, c, kc, S(stream));
}

}  // extern "C"
