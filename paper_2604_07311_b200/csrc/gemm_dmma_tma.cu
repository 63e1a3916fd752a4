// FP64 GEMM / GEMMT-lower, TMA + mbarrier warp-specialized (sm_100a).
//
// The fast path of gemm_dmma.cu for the layout the Cholesky family runs on:
// both operands k-contiguous (row-major A21 and its transposed view,
// engine/gemm.py:233-242 syrk = gemm(a, a^T)).  Same arithmetic contract —
// kc segments, ascending fma chains (DMMA), unfused fold — so the result is
// bit-identical to gemm_dmma.cu and to the reference.
//
//   16 warps, a 4x4 grid of 32x32 DMMA (m8n8k4) tiles over the 128x128 CTA
//   tile.  Operands arrive by TMA (cp.async.bulk.tensor) in a ring of STAGES
//   128B-swizzled stages; `full[s]` completes through mbarrier complete_tx.
//   There is no producer warp (a 17th warp would make the register allocator
//   cap every thread at 96 registers): each warp, when done with stage s,
//   bumps a shared counter, and the warp that releases it last issues the TMA
//   refill of s for k tile kt+STAGES right away.  No warp ever waits for a
//   slower one except through data it actually needs, and the warps never
//   meet at a CTA barrier in the main loop.
//
// Bank conflicts: with SWIZZLE_128B a 128-byte tile row r holds its 16-byte
// chunk c at c ^ (r & 7).  A fragment load has lanes (g, t) read (row g, k t);
// mapping fragment row g to tile row perm(g) = {0,2,4,6,1,3,5,7}[g] makes the
// eight chunks of each half warp distinct, i.e. one wavefront per half warp.
// The same permutation is applied to B's rows and undone in the epilogue.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cuda.h>

namespace bf {

namespace {

constexpr int TM_BM = 128, TM_BN = 128, TM_BK = 16;
constexpr int TM_CONSUMER_WARPS = 16;
constexpr int TM_THREADS = TM_CONSUMER_WARPS * 32;
constexpr int TM_TILE_BYTES = TM_BM * TM_BK * 8;  // 16 KB per operand per stage

__device__ __forceinline__ int perm8(int g) { return g < 4 ? 2 * g : 2 * (g - 4) + 1; }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void tile_coords_tma(const GemmParams& p, int64_t bid, bool tri, int64_t& ti, int64_t& tj) {
  const int64_t G = p.group;
  if (tri && p.panel_tiles > 0) {
    // column panels of panel_tiles tile columns, each row-major from its
    // diagonal down: a CTA's run of tiles shares one A row tile and a
    // panel's B tiles stay in L2 while every CTA sweeps its rows
    const int64_t T = p.tiles_m, w = p.panel_tiles;
    int64_t j0 = 0, q = bid;
    for (;;) {
      const int64_t tn = T - j0 < w ? T - j0 : w;
      const int64_t cnt = tn * (tn + 1) / 2 + (T - j0 - tn) * tn;
      if (q < cnt || j0 + tn >= T) {
        const int64_t tri_cnt = tn * (tn + 1) / 2;
        if (q < tri_cnt) {
          int64_t r = 0;
          while (q > r) {
            q -= r + 1;
            ++r;
          }
          ti = j0 + r;
          tj = j0 + q;
        } else {
          q -= tri_cnt;
          ti = j0 + tn + q / tn;
          tj = j0 + q % tn;
        }
        return;
      }
      q -= cnt;
      j0 += w;
    }
  }
  if (tri) {
    const int64_t T = p.tiles_m;
    int64_t start = 0, r0 = 0, h = 0;
    for (;;) {
      h = T - r0 < G ? T - r0 : G;
      int64_t cnt = r0 * h + h * (h + 1) / 2;
      if (bid < start + cnt) break;
      start += cnt;
      r0 += G;
    }
    int64_t q = bid - start;
    if (q < r0 * h) {
      tj = q / h;
      ti = r0 + q % h;
    } else {
      q -= r0 * h;
      int64_t c = 0;
      while (q >= h - c) {
        q -= h - c;
        ++c;
      }
      tj = r0 + c;
      ti = r0 + c + q;
    }
  } else {
    const int64_t per_group = G * p.tiles_n;
    int64_t gid = bid / per_group;
    int64_t first = gid * G;
    int64_t h = p.tiles_m - first < G ? p.tiles_m - first : G;
    int64_t local = bid - gid * per_group;
    ti = first + local % h;
    tj = local / h;
  }
}

__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// Persistent CTA: tiles blockIdx.x, +gridDim.x, ... share one ring of stages,
// so the TMA for the next tile's first k tiles is in flight while this
// tile's fold is written back.  MMAK = 4 (m8n8k4) or 8 (m16n8k8); KBOX =
// 16-wide k boxes per stage.
//
// TMC (long K, many kc segments — the contraction): the running C tile stays
// on chip, in tensor memory, across the segment folds.  Each thread's 32
// doubles (64 32-bit TMEM columns in its warp's lane quadrant; warps w and
// w+4k share a quadrant and take disjoint column ranges, 256 columns in all)
// are folded in registers 8 at a time (tcgen05.ld -> C + round(alpha*t) ->
// tcgen05.st), C is read from HBM only for the first segment (beta != 0) and
// written once after the last.  Same roundings in the same order as the
// global folds, so the same bits; the C traffic of a K = 16384, kc = 256
// tile drops from 64 L2 round trips to one read and one write.
//
// MODES: operands are 4-D tensor maps over permuted tensor modes (k_in,
// mn_in, k_out, mn_out) — the contraction's mode groups go straight into the
// swizzled stage with no transpose — and C is addressed through its two row
// and two column mode groups.
//
// GROUPED: one launch over several independent GEMMs sharing K (the
// distributed trailing update's column panels): tile_tab packs the group too
// (g << 24 | ti << 10 | tj), tiles row-major within a group; each tile takes
// its A/B row offsets, its C pointer, bounds and lower mask from the group table.
template <int MMAK, int KBOX, int STAGES, bool TMC, bool MODES = false, bool GROUPED = false, int BN_ = 128>
__global__ void __launch_bounds__(TM_THREADS, 1)
    gemm_dmma_tma_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                         const GemmParams p) {
  pdl_wait();
  if (aborted(p)) return;
  constexpr int BKS = 16 * KBOX;                    // k per stage
  // BN_ = 64: two independent groups of 8 warps, each on its own 128 x 64
  // tiles (a 4 x 2 grid of the same 32 x 32 warp tiles) with its own stage
  // ring and barriers — the CTA's tiles alternate between the groups, so one
  // group's fold and refill gaps hide under the other's DMMAs (what two
  // resident CTAs per SM would give, without giving up the one-CTA-per-SM
  // grid the SM reservation relies on)
  static_assert(BN_ == 128 || (BN_ == 64 && MMAK == 4), "128 x 64 tiles: m8n8k4 instantiations only");
  constexpr int NG = 128 / BN_, GW = TM_CONSUMER_WARPS / NG, WN = BN_ / 32;
  constexpr int NTHREADS = TM_THREADS;
  constexpr int B_BOX_BYTES = BN_ * TM_BK * 8;     // one 16-wide k box of B^T
  constexpr int OP_BYTES = KBOX * TM_TILE_BYTES;    // A, one stage
  constexpr int STAGE_BYTES = OP_BYTES + KBOX * B_BOX_BYTES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t tiles0 = (raw + 1023u) & ~1023u;  // SWIZZLE_128B wants 1 KB alignment
  const uint32_t bars = tiles0 + NG * STAGES * STAGE_BYTES;
  auto fullg = [&](int gr, int s) { return bars + 8u * (gr * STAGES + s); };
  __shared__ int released[NG * STAGES];
  // (ti, tj) of every tile this CTA owns, packed ti<<16 | tj, so a refill
  // (issued by whichever warp releases a stage last) costs one LDS
  uint32_t* tile_tab = reinterpret_cast<uint32_t*>(smem_raw + (bars + 8u * NG * STAGES - raw));
  uint32_t* row_tab = tile_tab + p.tiles_per_cta;  // GROUPED: 2 words per tile

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const bool tri = p.lower_only != 0;
  // Each CTA owns a contiguous run of `tiles_per_cta` raster positions: long
  // enough to overlap a tile's fold with the next tile's first loads, short
  // enough that CTAs retire every few hundred microseconds and the
  // high-priority panel stream of the Cholesky lookahead gets SMs promptly.
  // A persistent grid (p.tile_stride > 0) strides instead, so the tiles in
  // flight at any moment stay neighbours in the L2-friendly raster order.
  const int64_t tstep = p.tile_stride > 0 ? p.tile_stride : 1;
  const int64_t first_tile = p.tile_stride > 0 ? int64_t(blockIdx.x) : int64_t(blockIdx.x) * p.tiles_per_cta;
  const int64_t owned = p.tile_stride > 0 ? (p.num_tiles - first_tile + tstep - 1) / tstep : p.num_tiles - first_tile;
  const int W = int(owned < p.tiles_per_cta ? owned : p.tiles_per_cta);
  for (int w = tid; w < W; w += NTHREADS) {
    int64_t ti, tj;
    if constexpr (GROUPED) {
      const int64_t t = first_tile + w * tstep;
      int g = 0;
      while (g + 1 < p.ngroups && p.groups[g + 1].tile0 <= t) ++g;
      const GroupDesc& gd = p.groups[g];
      // row-major within the group: a CTA's run of tiles shares one A row
      // tile, and the group's few B tiles stay in L2 for every CTA
      int64_t local = t - gd.tile0;
      const int64_t tn = gd.tiles_n, tri_tiles = gd.lower ? tn * (tn + 1) / 2 : 0;
      if (local < tri_tiles) {  // lower: row ti < tiles_n holds columns 0..ti
        ti = 0;
        while (local > ti) {
          local -= ti + 1;
          ++ti;
        }
        tj = local;
      } else {
        local -= tri_tiles;
        ti = (gd.lower ? tn : 0) + local / tn;
        tj = local % tn;
      }
      tile_tab[w] = (uint32_t(g) << 24) | (uint32_t(ti) << 10) | uint32_t(tj);
      // the tile's A and B^T map rows, so a refill issues from shared memory
      // alone (bit 31: B^T comes from the A map)
      row_tab[2 * w] = uint32_t(gd.a_row + ti * TM_BM);
      row_tab[2 * w + 1] = uint32_t(gd.b_row + tj * BN_) | (gd.b_from_a ? 0x80000000u : 0u);
    } else {
      const int64_t t = first_tile + w * tstep;
      if (BN_ == 64 && tri) {  // each 128 x 128 lower tile as two 128 x 64 halves
        tile_coords_tma(p, t >> 1, tri, ti, tj);
        tj = 2 * tj + (t & 1);
      } else {
        tile_coords_tma(p, t, tri, ti, tj);
      }
      tile_tab[w] = (uint32_t(ti) << 16) | uint32_t(tj);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < NG * STAGES; ++s) {
      mbar_init(bars + 8u * s, 1);
      released[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __shared__ uint32_t tmem_slot;
  if constexpr (TMC) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                   "n"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if constexpr (TMC) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // this thread's 64 TMEM columns: lane quadrant (warp % 4), column block (warp / 4)
  const uint32_t tmem_c = TMC ? tmem_slot + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 64) : 0u;

  // k segmentation in 32-bit (eligibility guarantees K < 2^31, kc % BKS == 0 or kc >= K)
  const int K = int(p.k);
  const int kc = p.kc < p.k ? int(p.kc) : K;
  const int nseg = (K + kc - 1) / kc;
  const int tps = (kc + BKS - 1) / BKS;
  const int last_len = K - (nseg - 1) * kc;
  const int tps_last = (last_len + BKS - 1) / BKS;
  const int ntiles = (nseg - 1) * tps + tps_last;  // k tiles per output tile
  // this warp's group: tiles grp, grp + NG, ... of the CTA's run
  const int grp = NG == 1 ? 0 : warp / GW;
  const int Wg = W > grp ? (W - grp + NG - 1) / NG : 0;
  const int F = Wg * ntiles;  // stage fills of this group
  const uint32_t tiles = tiles0 + grp * STAGES * STAGE_BYTES;
  auto full = [&](int s) { return fullg(grp, s); };

  auto issue = [&](int f) {
    const int w = grp + NG * (f / ntiles), kt = f - (f / ntiles) * ntiles;
    const uint32_t tt = tile_tab[w];
    const int ti = GROUPED ? int((tt >> 10) & 0x3fffu) : int(tt >> 16), tj = GROUPED ? int(tt & 0x3ffu) : int(tt & 0xffffu);
    const int st = f % STAGES;
    const int seg = kt / tps, sub = kt - seg * tps;
    const int k_lo = seg * kc + sub * BKS;
    const uint32_t sa = tiles + st * STAGE_BYTES;
    mbar_expect_tx(full(st), STAGE_BYTES);
#pragma unroll
    for (int b = 0; b < KBOX; ++b) {
      if constexpr (MODES) {
        // an operand whose mode groups collapse to one per side has a 2-D map
        const uint32_t k = uint32_t(k_lo + 16 * b), ra = uint32_t(ti) * TM_BM, rb = uint32_t(tj) * BN_;
        if (p.a_rank == 2) {
          tma_load_2d(sa + b * TM_TILE_BYTES, &tma_a, int(k), int(ra), full(st));
        } else {
          const uint32_t qa = p.a_ki.div(k), qra = p.a_mi.div(ra);
          tma_load_4d(sa + b * TM_TILE_BYTES, &tma_a, int(k - qa * p.a_ki.d), int(ra - qra * p.a_mi.d), int(qa),
                      int(qra), full(st));
        }
        if (p.b_rank == 2) {
          tma_load_2d(sa + OP_BYTES + b * B_BOX_BYTES, &tma_b, int(k), int(rb), full(st));
        } else {
          const uint32_t qb = p.b_ki.div(k), qrb = p.b_mi.div(rb);
          tma_load_4d(sa + OP_BYTES + b * B_BOX_BYTES, &tma_b, int(k - qb * p.b_ki.d), int(rb - qrb * p.b_mi.d),
                      int(qb), int(qrb), full(st));
        }
      } else if constexpr (GROUPED) {
        const uint32_t ra = row_tab[2 * w], rb = row_tab[2 * w + 1];
        tma_load_2d(sa + b * TM_TILE_BYTES, &tma_a, k_lo + 16 * b, int(ra), full(st));
        tma_load_2d(sa + OP_BYTES + b * B_BOX_BYTES, (rb >> 31) ? &tma_a : &tma_b, k_lo + 16 * b,
                    int(rb & 0x7fffffffu), full(st));
      } else {
        tma_load_2d(sa + b * TM_TILE_BYTES, &tma_a, k_lo + 16 * b, int(ti * TM_BM), full(st));
        tma_load_2d(sa + OP_BYTES + b * B_BOX_BYTES, &tma_b, k_lo + 16 * b, int(tj * BN_), full(st));
      }
    }
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (tid == grp * GW * 32)
    for (int f = 0; f < F && f < STAGES; ++f) issue(f);

  const int g = lane >> 2, t = lane & 3;
  const int wm = (NG == 1 ? warp : warp % GW) / WN, wn = (NG == 1 ? warp : warp % GW) % WN;
  const int pg = perm8(g);
  const uint32_t a_row = uint32_t((wm * 32 + pg) * 128);
  const uint32_t b_row = uint32_t((wn * 32 + pg) * 128);
  // swizzled byte offset of k (0..15) inside a 128-byte row of this thread's rows
  auto koff = [&](int k) -> uint32_t { return uint32_t((((k >> 1) ^ pg) << 4) | ((k & 1) << 3)); };
  const int pj[2] = {perm8(2 * t), perm8(2 * t + 1)};
  double* C = static_cast<double*>(p.c);
  // GROUPED: the current tile's C, bounds and mask (set at each tile start)
  int64_t g_m = p.m, g_n = p.n, g_ld = p.c_rs;
  int g_lower = p.lower_only;
  // element offset of C(i, j) (MODES: two row and two column mode groups)
  auto coff = [&](int64_t i, int64_t j) -> int64_t {
    if constexpr (GROUPED) {
      return i * g_ld + j;
    } else if constexpr (MODES) {
      const uint32_t qi = p.c_ri.div(uint32_t(i)), qj = p.c_ci.div(uint32_t(j));
      return p.c_off + int64_t(qi) * p.c_rs_o + (i - int64_t(qi) * p.c_ri.d) * p.c_rs + int64_t(qj) * p.c_cs_o +
             (j - int64_t(qj) * p.c_ci.d) * p.c_cs;
    } else {
      return p.c_off + i * p.c_rs + j * p.c_cs;
    }
  };

  constexpr int MI = MMAK == 4 ? 4 : 2;  // row fragments per warp (8 or 16 rows each)
  double acc[4][4][2];                    // 32 accumulators in either shape
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // k tile at which segment sg prefetches C (4 tiles before its fold), or -1
  auto pf_next = [&](int sg) -> int {
    if (sg >= nseg) return -1;
    const int len = sg < nseg - 1 ? tps : tps_last;
    return sg * tps + (len >= 4 ? len - 4 : 0);
  };
  int s = 0, round = 0, f = 0;
  for (int wi = 0; wi < Wg; ++wi) {
    const uint32_t tt = tile_tab[grp + NG * wi];
    int64_t m0, n0;
    if constexpr (GROUPED) {
      const GroupDesc& gd = p.groups[tt >> 24];
      C = gd.c;
      g_m = gd.m;
      g_n = gd.n;
      g_ld = gd.ldc;
      g_lower = gd.lower;
      m0 = int64_t((tt >> 10) & 0x3fffu) * TM_BM;
      n0 = int64_t(tt & 0x3ffu) * BN_;
    } else {
      m0 = int64_t(tt >> 16) * TM_BM;
      n0 = int64_t(tt & 0xffffu) * BN_;
    }
    int seg = 0, sub = 0;
    // C is prefetched into L2 before each fold that reads it: every segment's
    // for the global folds, only the first (beta != 0) when C lives in TMEM
    int pf_kt = TMC ? (p.beta != 0.0 ? pf_next(0) : -1) : pf_next(p.beta != 0.0 ? 0 : 1);
    for (int kt = 0; kt < ntiles; ++kt, ++f) {
      mbar_wait(full(s), uint32_t(round & 1));
      const uint32_t sa = tiles + s * STAGE_BYTES;
      const uint32_t sb = sa + OP_BYTES;
#pragma unroll
      for (int bx = 0; bx < KBOX; ++bx) {
        const uint32_t ab = sa + bx * TM_TILE_BYTES + a_row;
        const uint32_t bb = sb + bx * B_BOX_BYTES + b_row;
        if constexpr (MMAK == 4) {
          double af[2][4], bfr[2][4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[0][i] = lds64(ab + i * 1024 + koff(t));
#pragma unroll
          for (int j = 0; j < 4; ++j) bfr[0][j] = lds64(bb + j * 1024 + koff(t));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int cur = q & 1;
            if (q < 3) {
#pragma unroll
              for (int i = 0; i < 4; ++i) af[cur ^ 1][i] = lds64(ab + i * 1024 + koff(4 * (q + 1) + t));
#pragma unroll
              for (int j = 0; j < 4; ++j) bfr[cur ^ 1][j] = lds64(bb + j * 1024 + koff(4 * (q + 1) + t));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bfr[cur][j]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 2; ++q) {  // two k8 steps per 16-wide box
            double af[2][4], bfr[4][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              af[i][0] = lds64(ab + i * 2048 + koff(8 * q + t));
              af[i][1] = lds64(ab + i * 2048 + 1024 + koff(8 * q + t));
              af[i][2] = lds64(ab + i * 2048 + koff(8 * q + t + 4));
              af[i][3] = lds64(ab + i * 2048 + 1024 + koff(8 * q + t + 4));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              bfr[j][0] = lds64(bb + j * 1024 + koff(8 * q + t));
              bfr[j][1] = lds64(bb + j * 1024 + koff(8 * q + t + 4));
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                double (&c)[4] = *reinterpret_cast<double (*)[4]>(&acc[2 * i][j][0]);
                // acc[2i][j] holds rows pg (c0,c1); acc[2i+1][j] rows 8+pg (c2,c3)
                double cc[4] = {acc[2 * i][j][0], acc[2 * i][j][1], acc[2 * i + 1][j][0], acc[2 * i + 1][j][1]};
                (void)c;
                dmma_16x8x8(cc, af[i], bfr[j]);
                acc[2 * i][j][0] = cc[0];
                acc[2 * i][j][1] = cc[1];
                acc[2 * i + 1][j][0] = cc[2];
                acc[2 * i + 1][j][1] = cc[3];
              }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        // release stage s; the last warp out refills it (generic reads ordered
        // before the async-proxy TMA write by the fences)
        __threadfence_block();
        const int c = atomicAdd(&released[grp * STAGES + s], 1);
        if (c == GW - 1) {
          released[grp * STAGES + s] = 0;
          if (f + STAGES < F) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(f + STAGES);
          }
        }
      }
      if (++s == STAGES) {
        s = 0;
        ++round;
      }
      if (kt == pf_kt) {
        pf_kt = TMC ? -1 : pf_next(kt / tps + 1);
        // warm L2 with this warp's 32x32 block of C before this segment's fold
        // reads it (with kc < K the folds recur, and the operand streams evict
        // C from L2 between them: d=128 contraction, 64 folds per tile)
        const int64_t r = m0 + wm * 32 + lane, c0 = n0 + wn * 32;
        if (r < (GROUPED ? g_m : p.m) && c0 < (GROUPED ? g_n : p.n)) {
          const double* rowp = C + coff(r, c0);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp));
          if (!MODES && (GROUPED || p.c_cs == 1) && c0 + 16 < (GROUPED ? g_n : p.n)) asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + 16));
        }
      }
      const bool seg_done = (seg < nseg - 1) ? (sub == tps - 1) : (sub == tps_last - 1);
      if (TMC && seg_done) {
        // fold into the TMEM-resident C, 8 doubles (16 columns) at a time
        if (seg > 0) asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t gi = m0 + wm * 32 + i * 8 + pg;
          const uint32_t taddr = tmem_c + uint32_t(i * 16);
          uint32_t w[16];
          if (seg > 0) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];\n"
                : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                  "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]),
                  "=r"(w[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int64_t gj = n0 + wn * 32 + j * 8 + pj[h];
              const bool ok = gi < (GROUPED ? g_m : p.m) && gj < (GROUPED ? g_n : p.n) && (!(GROUPED ? g_lower : p.lower_only) || gi >= gj);
              const int q = 2 * (2 * j + h);
              double v = __dmul_rn(p.alpha, acc[i][j][h]);
              if (seg > 0) {
                v = __dadd_rn(__hiloint2double(int(w[q + 1]), int(w[q])), v);  // beta_eff = 1: 1*C is exact
              } else if (p.beta != 0.0) {
                const double cold = ok ? __ldcg(C + coff(gi, gj)) : 0.0;
                v = __dadd_rn(__dmul_rn(p.beta, cold), v);
              }
              if (seg == nseg - 1) {
                if (ok) C[coff(gi, gj)] = v;
              } else {
                w[q] = uint32_t(__double2loint(v));
                w[q + 1] = uint32_t(__double2hiint(v));
              }
              acc[i][j][h] = 0.0;
            }
          if (seg < nseg - 1)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16};\n" ::"r"(taddr),
                "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
                "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
                : "memory");
        }
      } else if (seg_done) {
        // Fold: C is not __restrict__, so a load-use-store loop would
        // serialise one L2 round trip per element; instead each half of the
        // thread's 32 elements has all its reads in flight before its writes.
        const double beta_eff = seg == 0 ? p.beta : 1.0;
        if (beta_eff == 1.0 && p.red_fold) {
          // C := C + round(alpha*acc) is one correctly rounded add whichever
          // unit performs it: hand it to L2 as a fire-and-forget reduction
          // (red.global.add.f64, round-to-nearest, subnormals kept) instead of
          // a load -> add -> store round trip that stalls the warp before the
          // next segment's DMMAs.  Each element has one owning thread and its
          // folds stay in program order (same-address coherence), so the
          // sequence of adds, and the bits, are those of the load/store fold.
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t gi = m0 + wm * 32 + i * 8 + pg;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int64_t gj = n0 + wn * 32 + j * 8 + pj[h];
                const double v = __dmul_rn(p.alpha, acc[i][j][h]);
                if (gi < (GROUPED ? g_m : p.m) && gj < (GROUPED ? g_n : p.n) && (!(GROUPED ? g_lower : p.lower_only) || gi >= gj))
                  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(C + coff(gi, gj)),
                               "d"(v)
                               : "memory");
                acc[i][j][h] = 0.0;
              }
          }
        } else
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          double cold[2][4][2];
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            // m8n8k4: fragment i covers rows 8i..8i+7; m16n8k8: acc[2i'] / acc[2i'+1]
            // are rows 16i'+pg and 16i'+8+pg, i.e. again 8i+pg.
            const int64_t gi = m0 + wm * 32 + (2 * half + ii) * 8 + pg;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int64_t gj = n0 + wn * 32 + j * 8 + pj[h];
                const bool ok = gi < (GROUPED ? g_m : p.m) && gj < (GROUPED ? g_n : p.n) && (!(GROUPED ? g_lower : p.lower_only) || gi >= gj);
                cold[ii][j][h] = (ok && beta_eff != 0.0) ? __ldcg(C + coff(gi, gj)) : 0.0;
              }
          }
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int i = 2 * half + ii;
            const int64_t gi = m0 + wm * 32 + i * 8 + pg;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int64_t gj = n0 + wn * 32 + j * 8 + pj[h];
                double v = __dmul_rn(p.alpha, acc[i][j][h]);
                if (beta_eff != 0.0) v = __dadd_rn(__dmul_rn(beta_eff, cold[ii][j][h]), v);
                if (gi < (GROUPED ? g_m : p.m) && gj < (GROUPED ? g_n : p.n) && (!(GROUPED ? g_lower : p.lower_only) || gi >= gj)) C[coff(gi, gj)] = v;
                acc[i][j][h] = 0.0;
              }
          }
        }
      }
      if (++sub == (seg < nseg - 1 ? tps : tps_last)) {
        sub = 0;
        ++seg;
      }
    }
  }
  (void)MI;
  pdl_trigger();
  if constexpr (TMC) {
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_slot), "n"(256));
    }
  }
}

// ---- host side -------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// (K x MN) k-contiguous operand -> 2-D tensor map with a {16, 128} box.
bool make_map(CUtensorMap* map, const OperandMK& op, int64_t MN, int64_t K, int box_rows = TM_BM) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const double* base = static_cast<const double*>(op.base) + op.off;
  cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(MN)};
  cuuint64_t strides[1] = {cuuint64_t(op.s_mn) * 8};
  cuuint32_t box[2] = {TM_BK, cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// Usable when both operands are k-contiguous, 16-byte aligned with even row
// strides, and every k segment is a whole number of 16-wide k tiles (TMA
// cannot clip a box at a segment boundary; the cp.async kernel can).
bool gemm_dmma_tma_eligible(const GemmParams& p) {
  if (p.a.layout != GL_KMAJOR || p.b.layout != GL_KMAJOR || p.a.vec != 2 || p.b.vec != 2) return false;
  if (p.a.mn_scat || p.b.mn_scat || p.c_rscat) return false;
  if (!(p.kc % TM_BK == 0 || p.kc >= p.k)) return false;
  if (p.m > 0x7fffffffLL || p.n > 0x7fffffffLL || p.k > 0x7fffffffLL) return false;
  if ((p.a.s_mn * 8) % 16 != 0 || (p.b.s_mn * 8) % 16 != 0) return false;
  if (p.a.s_mn * 8 >= (int64_t(1) << 40) || p.b.s_mn * 8 >= (int64_t(1) << 40)) return false;
  if (p.m < 64 || p.n < 64) return false;  // thin problems go to the narrow cp.async tiles
  return encoder() != nullptr;
}

int g_tiles_per_cta = 1;
thread_local int t_reserve_sms = 0;
int g_reserve_strided = 0;  // bf_set_option("reserve_strided", 0/1): tile order of the reserved persistent grid  // set around a launch: persistent grid leaving this many SMs free
int g_red_fold = 1;
int g_persist = 0;
int g_tma_variant = 2;  // 0: m8n8k4/1 box/6 stages, 1: m16n8k8/1/6, 2: m8n8k4/2 boxes/3, 3: m16n8k8/2/3

int g_tmem_fold = 1;  // bf_set_option("tmem_fold", 0|1): C in TMEM across >= 3 kc segments

template <int MMAK, int KBOX, int STAGES, bool TMC, bool MODES = false, bool GROUPED = false, int BN_ = 128>
static int run_tma(const GemmParams& p_in, const CUtensorMap& ma, const CUtensorMap& mb, cudaStream_t s) {
  constexpr int NG = 128 / BN_;  // independent warp groups (each its own stage ring) per CTA
  constexpr size_t base_smem = size_t(NG) * STAGES * KBOX * (TM_BM + BN_) * TM_BK * 8 + 1024 + 8 * NG * STAGES;
  constexpr size_t max_smem = 200 * 1024;  // leaves room for the static __shared__ words
  auto kern = gemm_dmma_tma_kernel<MMAK, KBOX, STAGES, TMC, MODES, GROUPED, BN_>;
  GemmParams p = p_in;
  static int sms_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!sms_dev[dev]) cudaDeviceGetAttribute(&sms_dev[dev], cudaDevAttrMultiProcessorCount, dev);
  const int sms = sms_dev[dev];
  // tiles per CTA: g_tiles_per_cta (0 = fully persistent, one CTA per SM)
  int64_t tpc = g_tiles_per_cta > 0 ? int64_t(g_tiles_per_cta) * NG : (p.num_tiles + sms - 1) / sms;
  if (t_reserve_sms > 0 && t_reserve_sms < sms) {
    // persistent CTAs on all but t_reserve_sms SMs: the high-priority panel
    // stream always finds SMs free instead of waiting for tiles to retire
    const int64_t ctas = sms - t_reserve_sms;
    tpc = (p.num_tiles + ctas - 1) / ctas;
  }
  // g_persist: one CTA per SM striding over the raster (CTA b owns tiles b,
  // b + grid, ...), so each wave of concurrent tiles is one raster window
  // walking k in lockstep and its shared A/B strips are read from HBM once
  // per wave instead of once per staggered CTA (long-K GEMMs: the C5 contraction)
  const bool persist = g_persist && t_reserve_sms == 0 && p.num_tiles >= int64_t(4) * sms && p.k >= 4096;
  if (persist) tpc = (p.num_tiles + sms - 1) / sms;
  constexpr int64_t tab_bytes = GROUPED ? 12 : 4;  // per owned tile: packed coords (+ two map rows)
  while (tpc * tab_bytes + base_smem > max_smem) tpc /= 2;  // the tile table must fit
  if (tpc < 1) tpc = 1;
  p.tiles_per_cta = int(tpc);
  const int64_t grid = (p.num_tiles + tpc - 1) / tpc;
  if ((t_reserve_sms > 0 && g_reserve_strided) || persist) p.tile_stride = int(grid);
  if (grid > 0x7fffffffLL) return -3;
  if (p.m >= (1 << 16) * int64_t(TM_BM) || p.n >= (1 << 16) * int64_t(BN_)) return -3;
  const size_t smem = base_smem + size_t(tpc) * tab_bytes;
  if (!smem_attr(reinterpret_cast<const void*>(kern), int(smem))) return -10;
  note_launch();
  if (launch_maybe_pdl(kern, dim3(unsigned(grid)), dim3(TM_THREADS), smem, s, g_pdl != 0, ma, mb, p) != cudaSuccess)
    return -11;
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// bf_set_option("tma_bn", 64 | 128): plain launches (no TMEM fold, 32-aligned
// kc) on 128 x 64 tiles, two independent 8-warp groups per CTA with a
// 2 x 32-k stage ring each (default; 128 = one 16-warp 128 x 128 tile, 3 rings).
// A 1 x 16-k x 4-stage ring per group measured slower (C2 387.6 ms).
int g_tma_bn = 64;
int g_tmc_bn64 = 0;  // bf_set_option("tmc_bn64", 1): the TMEM-fold launches on the two-group 128 x 64 tiles too

int launch_gemm_dmma_tma(const GemmParams& p_in, cudaStream_t s) {
  GemmParams p = p_in;
  p.red_fold = g_red_fold;
  const int64_t nseg = p.kc < p.k ? (p.k + p.kc - 1) / p.kc : 1;
  const bool two_box_ok = (p.kc % 32 == 0) || p.kc >= p.k;
  const int variant = two_box_ok ? g_tma_variant : (g_tma_variant & 1);
  const bool tmc = g_tmem_fold && nseg >= 3 && variant == 2;
  const int bn = g_tma_bn == 64 && variant == 2 && (!tmc || g_tmc_bn64) ? 64 : 128;  // the default m8n8k4 / 2-box mainloop
  CUtensorMap ma, mb;
  if (!make_map(&ma, p.a, p.m, p.k) || !make_map(&mb, p.b, p.n, p.k, bn)) return -3;
  p.tiles_m = int((p.m + TM_BM - 1) / TM_BM);
  p.tiles_n = int((p.n + bn - 1) / bn);
  if (p.group <= 0) p.group = 8;
  // 128 x 64 lower tiles: every 128 x 128 lower tile as two halves
  p.num_tiles = p.lower_only ? int64_t(p.tiles_m) * (p.tiles_m + 1) / 2 * (128 / bn) : int64_t(p.tiles_m) * p.tiles_n;
  if (p.num_tiles <= 0) return 0;
  if (p.num_tiles > 0x7fffffffLL) return -3;
  if (bn == 64) return run_tma<4, 2, 2, false, false, false, 64>(p, ma, mb, s);
  if (tmc && bn == 64) return run_tma<4, 2, 2, true, false, false, 64>(p, ma, mb, s);
  if (tmc) return run_tma<4, 2, 3, true>(p, ma, mb, s);
  switch (variant) {
    case 1: return run_tma<8, 1, 6, false>(p, ma, mb, s);
    case 2: return run_tma<4, 2, 3, false>(p, ma, mb, s);
    case 3: return run_tma<8, 2, 3, false>(p, ma, mb, s);
    default: return run_tma<4, 1, 6, false>(p, ma, mb, s);
  }
}

// 4-D tensor map (k_in, mn_in, k_out, mn_out) over a mode-group operand with
// a box of 16 k x 128 rows: {16, min(mi, 128), 1, max(1, 128 / mi)}.
static bool make_map_modes(CUtensorMap* map, const ModeOperand& op, int64_t MN, int64_t K, int& rank) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const int64_t mi = op.mi, ki = op.ki;
  if (mi == MN && ki == K) {  // one group a side: the plain 2-D map of the strided kernel
    rank = 2;
    OperandMK o{};
    o.base = op.base;
    o.off = op.off;
    o.s_mn = op.s_mn;
    return (op.s_mn * 8) % 16 == 0 && reinterpret_cast<uintptr_t>(op.base + op.off) % 16 == 0 &&
           make_map(map, o, MN, K);
  }
  rank = 4;
  if (ki % TM_BK != 0 || K % ki != 0 || MN % mi != 0) return false;
  if (!(mi % TM_BM == 0 || TM_BM % mi == 0)) return false;
  cuuint64_t dims[4] = {cuuint64_t(ki), cuuint64_t(mi), cuuint64_t(K / ki), cuuint64_t(MN / mi)};
  cuuint64_t strides[3] = {cuuint64_t(op.s_mn) * 8, cuuint64_t(op.s_k_o) * 8, cuuint64_t(op.s_mn_o) * 8};
  for (int d = 0; d < 3; ++d) {
    const bool unused = dims[d + 1] == 1;
    if (unused) strides[d] = d > 0 ? strides[d - 1] : 16;  // a size-1 dimension's stride is never used
    if (strides[d] % 16 != 0 || strides[d] >= (cuuint64_t(1) << 40) || strides[d] == 0) return false;
  }
  cuuint32_t box[4] = {cuuint32_t(TM_BK), cuuint32_t(mi < TM_BM ? mi : TM_BM), 1,
                       cuuint32_t(mi < TM_BM ? TM_BM / mi : 1)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const double* base = op.base + op.off;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int launch_gemm_dmma_modes(GemmParams p, const ModeOperand& a, const ModeOperand& b, cudaStream_t s) {
  p.red_fold = g_red_fold;
  p.modes = 1;
  if (!(p.kc % 32 == 0 || p.kc >= p.k) || p.k % 32 != 0) return -3;  // whole 2x16-k stages per segment
  if (p.m > 0x7fffffffLL || p.n > 0x7fffffffLL || p.k > 0x7fffffffLL || p.lower_only) return -3;
  if (a.ki > 0x7fffffffLL || a.mi > 0x7fffffffLL || b.ki > 0x7fffffffLL || b.mi > 0x7fffffffLL) return -3;
  CUtensorMap ma, mb;
  if (!make_map_modes(&ma, a, p.m, p.k, p.a_rank) || !make_map_modes(&mb, b, p.n, p.k, p.b_rank)) return -3;
  p.a_ki = FastDiv(uint32_t(a.ki));
  p.a_mi = FastDiv(uint32_t(a.mi));
  p.b_ki = FastDiv(uint32_t(b.ki));
  p.b_mi = FastDiv(uint32_t(b.mi));
  if (p.c_ri.d == 0 || p.c_ci.d == 0) return -3;
  p.tiles_m = int((p.m + TM_BM - 1) / TM_BM);
  p.tiles_n = int((p.n + TM_BN - 1) / TM_BN);
  if (p.group <= 0) p.group = 8;
  p.num_tiles = int64_t(p.tiles_m) * p.tiles_n;
  if (p.num_tiles <= 0) return 0;
  const int64_t nseg = p.kc < p.k ? (p.k + p.kc - 1) / p.kc : 1;
  if (g_tmem_fold && nseg >= 3) return run_tma<4, 2, 3, true, true>(p, ma, mb, s);
  return run_tma<4, 2, 3, false, true>(p, ma, mb, s);
}

int launch_gemm_dmma_grouped(GemmParams p, const OperandMK& a, int64_t rows_a, const OperandMK& b, int64_t rows_b,
                             const GroupDesc* d_groups, int ngroups, int64_t num_tiles, cudaStream_t s) {
  if (ngroups <= 0 || num_tiles <= 0) return 0;
  if (ngroups > GEMM_MAX_GROUPS || num_tiles > 0x7fffffffLL) return -3;
  if (!(p.kc % 32 == 0 || p.kc >= p.k) || p.k > 0x7fffffffLL) return -3;
  if (rows_a >= (int64_t(1) << 31) || rows_b >= (int64_t(1) << 31)) return -3;
  if ((a.s_mn * 8) % 16 || (b.s_mn * 8) % 16) return -3;
  CUtensorMap ma, mb;
  if (!make_map(&ma, a, rows_a, p.k) || !make_map(&mb, b, rows_b, p.k)) return -3;
  p.red_fold = g_red_fold;
  p.groups = d_groups;
  p.ngroups = ngroups;
  p.num_tiles = num_tiles;
  p.m = p.n = 0;  // per group
  p.lower_only = 0;
  p.group = 1;
  return run_tma<4, 2, 3, false, false, true>(p, ma, mb, s);
}

}  // namespace bf
