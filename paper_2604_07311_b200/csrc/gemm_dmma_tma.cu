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
//   128B-swizzled stages: `full[s]` completes through complete_tx, `empty[s]`
//   when all 16 warps have read stage s.  Lane 0 of warp 0 is also the
//   producer: it refills a stage as soon as `empty` says it is free, polling
//   without blocking and only waiting when the tile it needs next was never
//   issued.  (A dedicated producer warp would make the CTA 17 warps, which the
//   register allocator rounds to 20 and caps every thread at 96 registers.)
//   The warps never meet at a CTA barrier in the main loop, so their drift
//   hides each other's waits.
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
constexpr int TM_STAGES = 6;
constexpr int TM_CONSUMER_WARPS = 16;
constexpr int TM_THREADS = TM_CONSUMER_WARPS * 32;
constexpr int TM_TILE_BYTES = TM_BM * TM_BK * 8;  // 16 KB per operand per stage
constexpr int TM_STAGE_BYTES = 2 * TM_TILE_BYTES;
constexpr size_t TM_SMEM = size_t(TM_STAGES) * TM_STAGE_BYTES + 1024 /*align*/ + 2 * TM_STAGES * 8;

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
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void tile_coords_tma(const GemmParams& p, int64_t bid, bool tri, int64_t& ti, int64_t& tj) {
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

__global__ void __launch_bounds__(TM_THREADS, 1)
    gemm_dmma_tma_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                         const GemmParams p) {
  if (aborted(p)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t tiles = (raw + 1023u) & ~1023u;  // SWIZZLE_128B wants 1 KB alignment
  const uint32_t bars = tiles + TM_STAGES * TM_STAGE_BYTES;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (TM_STAGES + s); };

  const bool tri = p.lower_only != 0;
  int64_t ti, tj;
  tile_coords_tma(p, blockIdx.x, tri, ti, tj);
  const int64_t m0 = ti * TM_BM, n0 = tj * TM_BN;
  if (p.lower_only) {
    int64_t row_hi = (m0 + TM_BM < p.m ? m0 + TM_BM : p.m) - 1;
    if (row_hi < n0) return;
  }

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < TM_STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), TM_CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // k segmentation in 32-bit (eligibility guarantees K < 2^31)
  const int K = int(p.k);
  const int kc = p.kc < p.k ? int(p.kc) : K;
  const int nseg = (K + kc - 1) / kc;
  const int tps = (kc + TM_BK - 1) / TM_BK;
  const int last_len = K - (nseg - 1) * kc;
  const int tps_last = (last_len + TM_BK - 1) / TM_BK;
  const int ntiles = (nseg - 1) * tps + tps_last;

  // ---------------- producer (warp 0, lane 0) ----------------
  const bool producer = (tid == 0);
  int next_fill = 0;
  auto issue = [&](int f) {
    const int st = f % TM_STAGES;
    const int seg = f / tps, sub = f - seg * tps;
    const int k_lo = seg * kc + sub * TM_BK;
    const uint32_t sa = tiles + st * TM_STAGE_BYTES;
    mbar_expect_tx(full(st), TM_STAGE_BYTES);
    tma_load_2d(sa, &tma_a, k_lo, int(m0), full(st));
    tma_load_2d(sa + TM_TILE_BYTES, &tma_b, k_lo, int(n0), full(st));
  };
  // Refill stages whose previous tile every warp has released; block only if
  // tile `need` itself has not been issued yet.
  auto refill = [&](int need) {
    while (next_fill < ntiles) {
      const int st = next_fill % TM_STAGES;
      const int round = next_fill / TM_STAGES;
      if (round > 0) {
        const uint32_t par = uint32_t((round - 1) & 1);
        if (next_fill <= need)
          mbar_wait(empty(st), par);
        else if (!mbar_test(empty(st), par))
          break;
      }
      issue(next_fill);
      ++next_fill;
    }
  };
  if (producer) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    for (; next_fill < ntiles && next_fill < TM_STAGES; ++next_fill) issue(next_fill);
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  const int pg = perm8(g);
  // byte offsets inside a stage tile
  const uint32_t a_row = uint32_t((wm * 32 + pg) * 128);
  const uint32_t b_row = uint32_t((wn * 32 + pg) * 128);
  uint32_t koff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) koff[q] = uint32_t(((((q * 4 + t) >> 1) ^ pg) << 4) | ((t & 1) << 3));

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double* C = static_cast<double*>(p.c);
  const int pj[2] = {perm8(2 * t), perm8(2 * t + 1)};  // epilogue column permutation

  int s = 0, round = 0, seg = 0, sub = 0;
  for (int kt = 0; kt < ntiles; ++kt) {
    if (producer && next_fill <= kt) refill(kt);
    mbar_wait(full(s), uint32_t(round & 1));
    const uint32_t sa = tiles + s * TM_STAGE_BYTES;
    const uint32_t sb = sa + TM_TILE_BYTES;
    // fragments double-buffered by hand to bound register pressure
    double af[2][4], bfr[2][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[0][i] = lds64(sa + a_row + i * 1024 + koff[0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) bfr[0][j] = lds64(sb + b_row + j * 1024 + koff[0]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cur = q & 1;
      if (q < 3) {
#pragma unroll
        for (int i = 0; i < 4; ++i) af[cur ^ 1][i] = lds64(sa + a_row + i * 1024 + koff[q + 1]);
#pragma unroll
        for (int j = 0; j < 4; ++j) bfr[cur ^ 1][j] = lds64(sb + b_row + j * 1024 + koff[q + 1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bfr[cur][j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty(s));
    if (producer) refill(-1);

    const bool seg_done = (seg < nseg - 1) ? (sub == tps - 1) : (sub == tps_last - 1);
    if (seg_done) {
      const double beta_eff = seg == 0 ? p.beta : 1.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t gi = m0 + wm * 32 + i * 8 + pg;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t gj = n0 + wn * 32 + j * 8 + pj[h];
            if (gi < p.m && gj < p.n && (!p.lower_only || gi >= gj)) {
              const int64_t addr = p.c_off + gi * p.c_rs + gj * p.c_cs;
              double v = __dmul_rn(p.alpha, acc[i][j][h]);
              if (beta_eff != 0.0) v = __dadd_rn(__dmul_rn(beta_eff, C[addr]), v);
              C[addr] = v;
            }
            acc[i][j][h] = 0.0;
          }
        }
      }
    }
    if (++s == TM_STAGES) {
      s = 0;
      ++round;
    }
    if (++sub == (seg < nseg - 1 ? tps : tps_last)) {
      sub = 0;
      ++seg;
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
bool make_map(CUtensorMap* map, const OperandMK& op, int64_t MN, int64_t K) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const double* base = static_cast<const double*>(op.base) + op.off;
  cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(MN)};
  cuuint64_t strides[1] = {cuuint64_t(op.s_mn) * 8};
  cuuint32_t box[2] = {TM_BK, TM_BM};
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

int launch_gemm_dmma_tma(const GemmParams& p_in, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_dmma_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TM_SMEM)) !=
        cudaSuccess)
      return -10;
    attr = true;
  }
  GemmParams p = p_in;
  CUtensorMap ma, mb;
  if (!make_map(&ma, p.a, p.m, p.k) || !make_map(&mb, p.b, p.n, p.k)) return -3;
  p.tiles_m = int((p.m + TM_BM - 1) / TM_BM);
  p.tiles_n = int((p.n + TM_BN - 1) / TM_BN);
  if (p.group <= 0) p.group = 8;
  p.num_tiles = p.lower_only ? int64_t(p.tiles_m) * (p.tiles_m + 1) / 2 : int64_t(p.tiles_m) * p.tiles_n;
  if (p.num_tiles <= 0) return 0;
  if (p.num_tiles > 0x7fffffffLL) return -3;
  note_launch();
  gemm_dmma_tma_kernel<<<unsigned(p.num_tiles), TM_THREADS, TM_SMEM, s>>>(ma, mb, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
