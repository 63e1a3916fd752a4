// FP64 GEMM / GEMMT-lower on the sm_100a FP64 tensor pipe (DMMA, mma.sync m8n8k4).
//
// Replaces the reference's five-loop driver + packed macro/micro kernel
// (engine/gemm.py:74-160, engine/kernels.py:24-90,142-255).  tcgen05 has no
// f64 kind, so FP64 runs on DMMA; the probe tools/dmma_order.cu showed that a
// DMMA is bit-identical to an ascending-k fma chain, which is exactly what the
// reference micro-kernel computes (fastmath={"contract"}, engine/kernels.py:169-172).
// Keeping the reference's kc segmentation and its unfused fold
// C = beta_eff*C + alpha*t therefore reproduces the reference bit for bit.
//
// Structure: one CTA per BMxBN output tile (triangular + grouped raster for
// GEMMT), cp.async multi-stage pipeline into padded shared memory (k-major or
// mn-major depending on which global stride is 1, so any MatrixView layout —
// row-major, transposed, padded, block-scatter — is consumed without a
// transpose), 8 warps each owning a 64x32 register accumulator.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cstdio>

namespace bf {

template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_, int LA_, int LB_>
struct DmmaCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int LA = LA_, LB = LB_;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  static constexpr int MI = WM / 8, NJ = WN / 8;
  static constexpr int PAD = 4;  // doubles; makes the 8-byte fragment loads conflict-free
  static constexpr bool A_MN = (LA == GL_MNMAJOR);
  static constexpr bool B_MN = (LB == GL_MNMAJOR);
  static constexpr int A_ELEMS = A_MN ? BK * (BM + PAD) : BM * (BK + PAD);
  static constexpr int B_ELEMS = B_MN ? BK * (BN + PAD) : BN * (BK + PAD);
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
  static_assert(WM % 8 == 0 && WN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert(A_ELEMS % 2 == 0 && B_ELEMS % 2 == 0, "16B stage alignment");
};

template <bool MN_MAJOR, int BMN, int BK>
__device__ __forceinline__ int sidx(int mn, int k) {
  if constexpr (MN_MAJOR)
    return k * (BMN + 4) + mn;
  else
    return mn * (BK + 4) + k;
}

// Fetch the (BMN x BK) tile rows [mn0, mn0+BMN) x k [k_lo, k_hi) of one
// operand into shared memory; everything outside (mn >= MN, k >= k_hi) is
// zero-filled, so a partial segment contributes fma(0,0,acc) = acc exactly.
template <int LAYOUT, int BMN, int BK, int THREADS>
__device__ __forceinline__ void load_tile(double* s, const OperandMK& op, int64_t MN, int64_t mn0,
                                          int64_t k_lo, int64_t k_hi, int tid) {
  const double* g = static_cast<const double*>(op.base);
  if constexpr (LAYOUT == GL_KMAJOR) {
    if (op.vec == 2) {
      constexpr int KP = BK / 2;
      constexpr int PAIRS = BMN * KP;
#pragma unroll
      for (int it = 0; it < (PAIRS + THREADS - 1) / THREADS; ++it) {
        int q = tid + it * THREADS;
        if (PAIRS % THREADS == 0 || q < PAIRS) {
          int mn = q / KP, kp = (q % KP) * 2;
          int64_t gm = mn0 + mn, gk = k_lo + kp;
          int64_t rem = k_hi - gk;
          int valid = (gm < MN && rem > 0) ? (rem >= 2 ? 2 : 1) : 0;
          const double* src = valid ? g + op.off + gm * op.s_mn + gk : g;
          cp_async_16(s + sidx<false, BMN, BK>(mn, kp), src, valid * 8);
        }
      }
      return;
    }
  } else if constexpr (LAYOUT == GL_MNMAJOR) {
    if (op.vec == 2) {
      constexpr int MP = BMN / 2;
      constexpr int PAIRS = MP * BK;
#pragma unroll
      for (int it = 0; it < (PAIRS + THREADS - 1) / THREADS; ++it) {
        int q = tid + it * THREADS;
        if (PAIRS % THREADS == 0 || q < PAIRS) {
          int k = q / MP, mn = (q % MP) * 2;
          int64_t gm = mn0 + mn, gk = k_lo + k;
          int64_t rem = MN - gm;
          int valid = (gk < k_hi && rem > 0) ? (rem >= 2 ? 2 : 1) : 0;
          const double* src = valid ? g + op.off + gm + gk * op.s_k : g;
          cp_async_16(s + sidx<true, BMN, BK>(mn, k), src, valid * 8);
        }
      }
      return;
    }
    // unaligned mn-major: element copies, mn fastest (coalesced)
    constexpr int ELEMS = BMN * BK;
#pragma unroll
    for (int it = 0; it < (ELEMS + THREADS - 1) / THREADS; ++it) {
      int q = tid + it * THREADS;
      if (ELEMS % THREADS == 0 || q < ELEMS) {
        int k = q / BMN, mn = q % BMN;
        int64_t gm = mn0 + mn, gk = k_lo + k;
        bool ok = gm < MN && gk < k_hi;
        const double* src = ok ? g + op.off + gm + gk * op.s_k : g;
        cp_async_8(s + sidx<true, BMN, BK>(mn, k), src, ok ? 8 : 0);
      }
    }
    return;
  }
  if constexpr (LAYOUT == GL_TRIDIAG) {
    // The skew sandwich's B operand, formed while it is staged (engine/
    // kernels.py:93-122 pack_b_block_tridiag): row g of W = T*S combines two
    // source rows, W[g,j] = (0 + t[g-1]*S[g-1,j]) - t[g]*S[g+1,j], edge terms
    // dropped, each product and sum rounded like the reference's packing.
    // No W ever exists outside shared memory.
    constexpr int ELEMS = BMN * BK;
#pragma unroll
    for (int it = 0; it < (ELEMS + THREADS - 1) / THREADS; ++it) {
      const int q = tid + it * THREADS;
      if (ELEMS % THREADS == 0 || q < ELEMS) {
        const int mn = q / BK, k = q % BK;
        const int64_t gm = mn0 + mn, gk = k_lo + k;
        double w = 0.0;
        if (gm < MN && gk < k_hi) {
          const double* row = g + op.off + gm * op.s_mn;
          double acc = 0.0;
          if (gk > 0) acc = __dadd_rn(acc, __dmul_rn(__ldg(op.tvec + gk - 1), __ldg(row + (gk - 1) * op.s_k)));
          if (gk < op.k_total - 1) acc = __dsub_rn(acc, __dmul_rn(__ldg(op.tvec + gk), __ldg(row + (gk + 1) * op.s_k)));
          w = acc;
        }
        s[sidx<false, BMN, BK>(mn, k)] = w;
      }
    }
    return;
  }
  // k-major unaligned, generic strided, or block-scatter: element copies, k fastest.
  constexpr int ELEMS = BMN * BK;
  if constexpr (THREADS % BK == 0 && ELEMS % THREADS == 0) {
    // every thread keeps one k for all its elements: one k-offset lookup per
    // tile and one (L1-resident) row-offset lookup per element
    const int k = tid % BK;
    const int64_t gk = k_lo + k;
    const bool kok = gk < k_hi;
    const int64_t koff = kok ? (op.k_scat ? __ldg(op.k_scat + gk) : gk * op.s_k) : 0;
#pragma unroll
    for (int it = 0; it < ELEMS / THREADS; ++it) {
      const int mn = tid / BK + it * (THREADS / BK);
      const int64_t gm = mn0 + mn;
      const bool ok = kok && gm < MN;
      const double* src = g;
      if (ok) src = g + (op.mn_scat ? __ldg(op.mn_scat + gm) : op.off + gm * op.s_mn) + koff;
      cp_async_8(s + sidx<false, BMN, BK>(mn, k), src, ok ? 8 : 0);
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < (ELEMS + THREADS - 1) / THREADS; ++it) {
    int q = tid + it * THREADS;
    if (ELEMS % THREADS == 0 || q < ELEMS) {
      int mn = q / BK, k = q % BK;
      int64_t gm = mn0 + mn, gk = k_lo + k;
      bool ok = gm < MN && gk < k_hi;
      const double* src = g;
      if (ok) {
        if (op.mn_scat)
          src = g + op.mn_scat[gm] + op.k_scat[gk];
        else
          src = g + op.off + gm * op.s_mn + gk * op.s_k;
      }
      cp_async_8(s + sidx<false, BMN, BK>(mn, k), src, ok ? 8 : 0);
    }
  }
}

// Tile id -> (ti, tj).  GEMMT-lower with square tiles enumerates only the
// lower triangle of tiles; both orders are grouped by `group` tile rows so
// the CTAs resident at one time share their A and B row panels in L2.
__device__ __forceinline__ void tile_coords(const GemmParams& p, int64_t bid, bool tri, int64_t& ti,
                                            int64_t& tj) {
  const int64_t G = p.group;
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

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1) gemm_dmma_kernel(const GemmParams p) {
  if (aborted(p)) return;
  extern __shared__ __align__(16) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int MI = Cfg::MI, NJ = Cfg::NJ;

  const bool tri = p.lower_only && BM == BN;
  int64_t ti, tj;
  tile_coords(p, blockIdx.x, tri, ti, tj);
  const int64_t m0 = ti * BM, n0 = tj * BN;
  if (p.lower_only) {
    int64_t row_hi = (m0 + BM < p.m ? m0 + BM : p.m) - 1;
    if (row_hi < n0) return;  // tile strictly above the diagonal
  }

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp / Cfg::WARPS_N) * Cfg::WM;
  const int wn0 = (warp % Cfg::WARPS_N) * Cfg::WN;

  // k segmentation (reference pc loop, engine/gemm.py:124-126)
  const int64_t K = p.k;
  const int64_t kc = p.kc < K ? p.kc : K;
  const int64_t nseg = (K + kc - 1) / kc;
  const int64_t tps = (kc + BK - 1) / BK;
  const int64_t last_len = K - (nseg - 1) * kc;
  const int64_t tps_last = (last_len + BK - 1) / BK;
  const int64_t ntiles = (nseg - 1) * tps + tps_last;

  auto load_stage = [&](int stage, int64_t kt) {
    int64_t seg = kt / tps, sub = kt - seg * tps;
    int64_t k_lo = seg * kc + sub * BK;
    int64_t seg_end = (seg + 1) * kc < K ? (seg + 1) * kc : K;
    int64_t k_hi = k_lo + BK < seg_end ? k_lo + BK : seg_end;
    double* sA = smem + stage * Cfg::STAGE_ELEMS;
    double* sB = sA + Cfg::A_ELEMS;
    load_tile<Cfg::LA, BM, BK, Cfg::THREADS>(sA, p.a, p.m, m0, k_lo, k_hi, tid);
    load_tile<Cfg::LB, BN, BK, Cfg::THREADS>(sB, p.b, p.n, n0, k_lo, k_hi, tid);
  };

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_stage(s, s);
    cp_async_commit();
  }

  double* C = static_cast<double*>(p.c);
  for (int64_t kt = 0; kt < ntiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int64_t nxt = kt + STAGES - 1;
      if (nxt < ntiles) load_stage(int(nxt % STAGES), nxt);
      cp_async_commit();
    }
    const double* sA = smem + int(kt % STAGES) * Cfg::STAGE_ELEMS;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bfr[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = sA[sidx<Cfg::A_MN, BM, BK>(wm0 + i * 8 + g, kk + t)];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bfr[j] = sB[sidx<Cfg::B_MN, BN, BK>(wn0 + j * 8 + g, kk + t)];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bfr[j]);
    }

    const int64_t seg = kt / tps, sub = kt - seg * tps;
    const bool seg_done = (seg < nseg - 1) ? (sub == tps - 1) : (sub == tps_last - 1);
    if (seg_done) {
      // fold the segment into C: C = beta_eff*C + alpha*t  (engine/kernels.py:228-253);
      // one row fragment at a time, its reads issued before its writes
      const double beta_eff = seg == 0 ? p.beta : 1.0;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int64_t gi = m0 + wm0 + i * 8 + g;
        int64_t addr[NJ][2];
        bool ok[NJ][2];
        double cold[NJ][2];
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t gj = n0 + wn0 + j * 8 + 2 * t + h;
            ok[j][h] = gi < p.m && gj < p.n && (!p.lower_only || gi >= gj);
            addr[j][h] = ok[j][h] ? (p.c_rscat ? p.c_rscat[gi] + p.c_cscat[gj] : p.c_off + gi * p.c_rs + gj * p.c_cs) : 0;
            cold[j][h] = (ok[j][h] && beta_eff != 0.0) ? __ldcg(C + addr[j][h]) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double v = __dmul_rn(p.alpha, acc[i][j][h]);
            if (beta_eff != 0.0) v = __dadd_rn(__dmul_rn(beta_eff, cold[j][h]), v);
            if (ok[j][h]) C[addr[j][h]] = v;
            acc[i][j][h] = 0.0;
          }
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
template <class Cfg>
static int run_cfg(const GemmParams& p_in, cudaStream_t s) {
  auto kern = gemm_dmma_kernel<Cfg>;
  if (!smem_attr(reinterpret_cast<const void*>(kern), int(Cfg::SMEM))) return -10;
  GemmParams p = p_in;
  p.tiles_m = int((p.m + Cfg::BM - 1) / Cfg::BM);
  p.tiles_n = int((p.n + Cfg::BN - 1) / Cfg::BN);
  if (p.group <= 0) p.group = 8;
  if (p.lower_only && Cfg::BM == Cfg::BN) {
    int64_t T = p.tiles_m;
    p.num_tiles = T * (T + 1) / 2;
  } else {
    p.num_tiles = int64_t(p.tiles_m) * p.tiles_n;
  }
  if (p.num_tiles <= 0) return 0;
  if (p.num_tiles > 0x7fffffffLL) return -3;
  note_launch();
  kern<<<unsigned(p.num_tiles), Cfg::THREADS, Cfg::SMEM, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -11;
}

template <int LA, int LB>
static int run_layouts(const GemmParams& p, cudaStream_t s) {
  // Narrow outputs (TRSM off-diagonal updates, V2 panel GEMM) use a 128x32 tile.
  if (p.n <= 48 && !p.lower_only)
    return run_cfg<DmmaCfg<128, 32, 16, 4, 1, 4, LA, LB>>(p, s);
  return run_cfg<DmmaCfg<128, 128, 16, 2, 4, 4, LA, LB>>(p, s);
}

int g_use_tma = 1;

int launch_gemm_dmma(const GemmParams& p, cudaStream_t s) {
  if (g_use_tma && gemm_dmma_tma_eligible(p)) return launch_gemm_dmma_tma(p, s);
  const int la = p.a.layout, lb = p.b.layout;
#define BF_CASE(A, B) \
  if (la == A && lb == B) return run_layouts<A, B>(p, s);
  BF_CASE(GL_KMAJOR, GL_KMAJOR)
  BF_CASE(GL_KMAJOR, GL_MNMAJOR)
  BF_CASE(GL_KMAJOR, GL_GENERIC)
  BF_CASE(GL_MNMAJOR, GL_KMAJOR)
  BF_CASE(GL_MNMAJOR, GL_MNMAJOR)
  BF_CASE(GL_MNMAJOR, GL_GENERIC)
  BF_CASE(GL_GENERIC, GL_KMAJOR)
  BF_CASE(GL_GENERIC, GL_MNMAJOR)
  BF_CASE(GL_GENERIC, GL_GENERIC)
  BF_CASE(GL_KMAJOR, GL_TRIDIAG)
  BF_CASE(GL_MNMAJOR, GL_TRIDIAG)
  BF_CASE(GL_GENERIC, GL_TRIDIAG)
#undef BF_CASE
  return -3;
}

}  // namespace bf
