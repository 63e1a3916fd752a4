// bf16 x bf16 -> fp32 GEMM / GEMMT on the 5th-generation tensor cores
// (tcgen05.mma kind::f16, accumulator in TMEM), operands staged by TMA; the
// same kernel with kind::tf32 on fp32 operands backs the 3xTF32 FP32 GEMM
// (split_tf32_kernel: A B^T = hi hi^T + hi lo^T + lo hi^T as one K = 3k GEMM).
//
// The trailing update of the mixed-precision Cholesky (BASELINE configs[3]):
// C(fp32) := beta*C + alpha * A * B^T with A (M x K) and B (N x K) bf16,
// both k-contiguous; lower_only restricts C to i >= j.  This path has no
// reference counterpart (the reference's only mixed mode is f32-storage /
// f64-accumulation GEMM); its parity is the FP64 solution after iterative
// refinement.
//
// Persistent: one CTA per SM walks the 128x128 output tiles (lower-triangle
// tiles only for GEMMT) with a static stride; 6 warps:
//   warp 0      TMA producer (one elected lane): A/B boxes {64 k, 128 rows},
//               128B swizzle, into a 6-stage ring (full/empty mbarriers) that
//               runs on across tile boundaries
//   warp 1      TMEM allocator + MMA issuer (one lane): 4 x UMMA 128x128x16
//               per stage from smem descriptors into one of TWO 128-column
//               TMEM accumulators, so tile t+1 accumulates while the
//               epilogue drains tile t; tcgen05.commit frees smem stages and
//               signals the accumulator
//   warps 2..5  epilogue: tcgen05.ld 32x32b (each warp its TMEM lane quadrant,
//               all 128 columns, then the accumulator is released); the fp32
//               C tile comes in by TMA while the tile's mainloop runs (four
//               {32 col, 128 row} boxes, 128B swizzle, read conflict-free as
//               float4 per row), is combined in smem and leaves by TMA store.
//               Unaligned C views fall back to a warp-private smem transpose
//               and coalesced per-element read-modify-write.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cuda.h>
#include <cuda_bf16.h>

namespace bf {

int g_bf16_tma_c = 1;
int g_bf16_group = 8;  // bf_set_option("bf16_group", g): row tiles per band of the tcgen05 GEMM's tile order (0: plain)

namespace {

constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int TC_STAGES = 5;
constexpr int TC_THREADS = 192;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2, TC_B_BYTES = TC_BN * TC_BK * 2;
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr int TC_CBOX_BYTES = 128 * 32 * 4;         // one {32 col, 128 row} fp32 box
constexpr int TC_CTILE_BYTES = 4 * TC_CBOX_BYTES;    // C tile staging (TMA path) / transposes (fallback)
constexpr size_t TC_SMEM = size_t(TC_STAGES) * TC_STAGE_BYTES + TC_CTILE_BYTES + 1024 + 256;

__device__ __forceinline__ void mbar_init_tc(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx_tc(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_tc(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void tma_load_2d_tc(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// tcgen05 shared-memory matrix descriptor: K-major, 128B swizzle, 8-row atoms
// of 1024 bytes (SBO), fixed version bits 46-48 = 0b001.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;             // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;     // SBO: next 8-row group
  d |= uint64_t(1) << 46;             // version
  d |= uint64_t(2) << 61;             // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=128
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32 (format 2), both K-major
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

// Tile order: bands of p.group row tiles, column-major inside a band (the
// lower triangle's band = its full-height columns, then its own triangle),
// so the ~148 tiles in flight share a few A row tiles and a band's columns
// of B while the band's A rows stay in L2.  (Row-by-row / one-column-at-a-
// time orders streamed A or B from HBM once per row or column: 8192^3 read
// 4 GB from DRAM.)  p.group <= 0: the plain orders.
__device__ __forceinline__ void tile_of(const GemmParams& p, int64_t t, int64_t& ti, int64_t& tj) {
  const int64_t G = p.group;
  if (p.lower_only && G > 0) {
    const int64_t T = p.tiles_m;
    int64_t start = 0, r0 = 0, h = 0;
    for (;;) {
      h = T - r0 < G ? T - r0 : G;
      const int64_t cnt = r0 * h + h * (h + 1) / 2;
      if (t < start + cnt) break;
      start += cnt;
      r0 += G;
    }
    int64_t q = t - start;
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
  } else if (p.lower_only) {  // lower-triangle enumeration, row by row
    int64_t r = int64_t((sqrt(8.0 * double(t) + 1.0) - 1.0) * 0.5);
    while (r * (r + 1) / 2 > t) --r;
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    ti = r;
    tj = t - r * (r + 1) / 2;
  } else if (G > 0) {
    const int64_t per_group = G * p.tiles_n;
    const int64_t gid = t / per_group, first = gid * G;
    const int64_t h = p.tiles_m - first < G ? p.tiles_m - first : G;
    const int64_t local = t - gid * per_group;
    ti = first + local % h;
    tj = local / h;
  } else {
    ti = t % p.tiles_m;
    tj = t / p.tiles_m;
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// TF32 = 0: bf16 operands (kind::f16, 64 k per 128-byte row);
// TF32 = 1: fp32 operands read as tf32 (kind::tf32, 32 k per row).  The smem
// geometry, descriptors and the 4 MMAs per stage (32 bytes of k each) are the same.
template <bool TMAC, int TF32>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                        const __grid_constant__ CUtensorMap tma_c, const GemmParams p) {
  extern __shared__ __align__(16) unsigned char tc_smem[];
  const uint32_t raw = smem_u32(tc_smem);
  const uint32_t tiles = (raw + 1023u) & ~1023u;
  const uint32_t cbuf = tiles + TC_STAGES * TC_STAGE_BYTES;
  float* xpose = reinterpret_cast<float*>(tc_smem + (cbuf - raw));
  const uint32_t bars = cbuf + TC_CTILE_BYTES;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (TC_STAGES + s); };
  auto acc_full = [&](int b) { return bars + 8u * (2 * TC_STAGES + b); };
  auto acc_empty = [&](int b) { return bars + 8u * (2 * TC_STAGES + 2 + b); };
  const uint32_t cload = bars + 8u * (2 * TC_STAGES + 4);
  const uint32_t tmem_slot = cload + 8u;  // u32 written by tcgen05.alloc

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init_tc(full(s), 1);
      mbar_init_tc(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init_tc(acc_full(b), 1);
      mbar_init_tc(acc_empty(b), 4);  // one arrival per epilogue warp
    }
    mbar_init_tc(cload, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(tmem_base) : "r"(tmem_slot));

  constexpr int BK = TF32 ? 32 : TC_BK;  // k elements per 128-byte swizzle row
  const int ktiles = int((p.k + BK - 1) / BK);
  const int64_t ntiles = p.num_tiles;
  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int64_t ti, tj;
      tile_of(p, t, ti, tj);
      for (int kt = 0; kt < ktiles; ++kt, ++it) {
        const int s = int(it % TC_STAGES);
        mbar_wait_tc(empty(s), ((it / TC_STAGES) & 1u) ^ 1u);
        const uint32_t sa = tiles + s * TC_STAGE_BYTES;
        mbar_expect_tx_tc(full(s), TC_STAGE_BYTES);
        tma_load_2d_tc(sa, &tma_a, kt * BK, int(ti * TC_BM), full(s));
        tma_load_2d_tc(sa + TC_A_BYTES, &tma_b, kt * BK, int(tj * TC_BN), full(s));
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    constexpr uint32_t idesc = TF32 ? idesc_tf32_f32(TC_BM, TC_BN) : idesc_bf16_f32(TC_BM, TC_BN);
    uint32_t it = 0, lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const uint32_t buf = lt & 1u;
      mbar_wait_tc(acc_empty(buf), ((lt >> 1) & 1u) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t dst = tmem_base + buf * TC_BN;
      for (int kt = 0; kt < ktiles; ++kt, ++it) {
        const int s = int(it % TC_STAGES);
        mbar_wait_tc(full(s), (it / TC_STAGES) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t sa = tiles + s * TC_STAGE_BYTES;
        const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + TC_A_BYTES);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // 32 bytes of k per MMA (16 bf16 / 8 tf32): advance inside the swizzle row
          if (TF32)
            umma_tf32(dst, da + uint64_t(2 * kk), db + uint64_t(2 * kk), idesc, (kt | kk) != 0);
          else
            umma_bf16(dst, da + uint64_t(2 * kk), db + uint64_t(2 * kk), idesc, (kt | kk) != 0);
        }
        umma_commit(empty(s));
      }
      umma_commit(acc_full(buf));
    }
  } else if (warp >= 2 && TMAC) {
    // ---- epilogue, TMA C tile: TMEM lane quadrant (warp % 4) -> rows ----
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // tile row of this thread
    const bool leader = warp == 2 && lane == 0;
    const float alpha = float(p.alpha), beta = float(p.beta);
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int64_t ti, tj;
      tile_of(p, t, ti, tj);
      if (leader) {  // C tile load overlaps this tile's mainloop
        mbar_expect_tx_tc(cload, TC_CTILE_BYTES);
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
          tma_load_2d_tc(cbuf + cb * TC_CBOX_BYTES, &tma_c, int(tj * TC_BN + cb * 32), int(ti * TC_BM), cload);
      }
      const uint32_t buf = lt & 1u;
      mbar_wait_tc(acc_full(buf), (lt >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t acc[4][32];
      const uint32_t taddr = tmem_base + (uint32_t(quad * 32) << 16) + buf * TC_BN;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) tmem_ld32(taddr + uint32_t(cb * 32), acc[cb]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(acc_empty(buf)) : "memory");
      mbar_wait_tc(cload, lt & 1u);
      const int64_t gi = ti * TC_BM + r;
      // a GEMMT diagonal tile must not write its strict upper part (the bulk
      // store would rewrite it with the values loaded before the mainloop):
      // its lower elements go out per element instead
      const bool diag = p.lower_only && ti == tj;
      float* Cg = static_cast<float*>(p.c);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t addr = cbuf + cb * TC_CBOX_BYTES + r * 128 + ((c ^ (r & 7)) << 4);
          float o[4];
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                       : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3])
                       : "r"(addr));
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t gj = tj * TC_BN + cb * 32 + c * 4 + e;
            if (!p.lower_only || gj <= gi) {
              const float v = alpha * __uint_as_float(acc[cb][c * 4 + e]);
              o[e] = beta != 0.f ? fmaf(beta, o[e], v) : v;
              if (diag && gi < p.m && gj < p.n) __stcs(Cg + p.c_off + gi * p.c_rs + gj * p.c_cs, o[e]);
            }
          }
          if (!diag)
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                         "f"(o[3])
                         : "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (leader && !diag) {
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                  reinterpret_cast<uint64_t>(&tma_c)),
              "r"(int(tj * TC_BN + cb * 32)), "r"(int(ti * TC_BM)), "r"(cbuf + cb * TC_CBOX_BYTES)
              : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  } else if (warp >= 2) {
    // ---- epilogue, fallback: TMEM lane quadrant (warp % 4) -> rows ----
    const int quad = warp & 3;
    float* st = xpose + (warp - 2) * 32 * 33;
    float* C = static_cast<float*>(p.c);
    const float alpha = float(p.alpha), beta = float(p.beta);
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int64_t ti, tj;
      tile_of(p, t, ti, tj);
      const uint32_t buf = lt & 1u;
      mbar_wait_tc(acc_full(buf), (lt >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t r[4][32];
      const uint32_t taddr = tmem_base + (uint32_t(quad * 32) << 16) + buf * TC_BN;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) tmem_ld32(taddr + uint32_t(cb * 32), r[cb]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(acc_empty(buf)) : "memory");
      const int64_t row0 = ti * TC_BM + quad * 32;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        // lane holds row (row0 + lane), columns cb*32 .. cb*32+31: transpose so lanes run along columns
#pragma unroll
        for (int j = 0; j < 32; ++j) st[lane * 33 + j] = __uint_as_float(r[cb][j]);
        __syncwarp();
        const int64_t gj = tj * TC_BN + cb * 32 + lane;
#pragma unroll
        for (int r8 = 0; r8 < 32; r8 += 8) {
          float old[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int64_t gi = row0 + r8 + q;
            const bool ok = gi < p.m && gj < p.n && (!p.lower_only || gi >= gj);
            old[q] = (ok && beta != 0.f) ? __ldcs(C + p.c_off + gi * p.c_rs + gj * p.c_cs) : 0.f;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int64_t gi = row0 + r8 + q;
            if (gi < p.m && gj < p.n && (!p.lower_only || gi >= gj)) {
              float v = alpha * st[(r8 + q) * 33 + lane];
              if (beta != 0.f) v = fmaf(beta, old[q], v);
              __stcs(C + p.c_off + gi * p.c_rs + gj * p.c_cs, v);
            }
          }
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(256));
  }
}

typedef CUresult (*EncodeTiledFnTc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFnTc encoder_tc() {
  static EncodeTiledFnTc fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* q = nullptr;
    cudaDriverEntryPointQueryResult res;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &res) == cudaSuccess &&
        res == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFnTc>(q);
  }
  return fn;
}

bool make_map_c32(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld) {
  EncodeTiledFnTc enc = encoder_tc();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_f32k(CUtensorMap* map, const float* base, int64_t rows, int64_t k, int64_t ld) {
  EncodeTiledFnTc enc = encoder_tc();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t k, int64_t ld) {
  EncodeTiledFnTc enc = encoder_tc();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
  cuuint32_t box[2] = {TC_BK, 128};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 (strided) -> bf16 (row-major, ld) conversion; transposes when asked
template <typename S>
__global__ void to_bf16_kernel(const S* src, int64_t soff, int64_t srs, int64_t scs, __nv_bfloat16* dst,
                               int64_t ld, int64_t m, int64_t n, int transpose) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const float v = src[soff + i * srs + j * scs];
    if (transpose)
      dst[j * ld + i] = __float2bfloat16_rn(v);
    else
      dst[i * ld + j] = __float2bfloat16_rn(v);
  }
}

// 3xTF32 operand split: row i of the (m x k) fp32 source becomes
// [hi | hi | lo | hi] in dst (4 parts of kp >= k columns, zero padded), with
// hi = x rounded to tf32 and lo = x - hi (exact).  A' = dst[:, 0:3kp] and
// B' = dst[:, kp:4kp] then give A'B'^T = hi hi^T + hi lo^T + lo hi^T.
template <typename S>
__global__ void split_tf32_kernel(const S* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t ld,
                                  int64_t m, int64_t k, int64_t kp) {
  const int64_t total = m * kp;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / kp, j = e % kp;
    const float x = j < k ? float(src[soff + i * srs + j * scs]) : 0.f;
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
    const float hi = __uint_as_float(h), lo = x - hi;
    float* row = dst + i * ld;
    row[j] = hi;
    row[kp + j] = hi;
    row[2 * kp + j] = lo;
    row[3 * kp + j] = hi;
  }
}

}  // namespace

int launch_split_tf32(int src_f64, const void* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t ld,
                      int64_t m, int64_t k, int64_t kp, cudaStream_t s) {
  if (m <= 0 || kp <= 0) return 0;
  const int64_t total = m * kp;
  const int blocks = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  note_launch();
  if (src_f64)
    split_tf32_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(src), soff, srs, scs, dst, ld, m, k, kp);
  else
    split_tf32_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(src), soff, srs, scs, dst, ld, m, k, kp);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

namespace {
int launch_tc(int tf32, double alpha, const void* a, int64_t lda, const void* b, int64_t ldb, double beta, float* c,
              int64_t c_off, int64_t c_rs, int64_t c_cs, int64_t m, int64_t n, int64_t k, int lower_only,
              cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  const int esz = tf32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(a) % 16) || (reinterpret_cast<uintptr_t>(b) % 16) || (lda * esz) % 16 ||
      (ldb * esz) % 16 || k < 1)
    return -3;
  CUtensorMap ma, mb;
  if (tf32) {
    if (!make_map_f32k(&ma, static_cast<const float*>(a), m, k, lda) ||
        !make_map_f32k(&mb, static_cast<const float*>(b), n, k, ldb))
      return -3;
  } else if (!make_map_bf16(&ma, a, m, k, lda) || !make_map_bf16(&mb, b, n, k, ldb)) {
    return -3;
  }
  if (!smem_attr(reinterpret_cast<const void*>(gemm_bf16_tc_kernel<true, 0>), int(TC_SMEM)) ||
      !smem_attr(reinterpret_cast<const void*>(gemm_bf16_tc_kernel<false, 0>), int(TC_SMEM)) ||
      !smem_attr(reinterpret_cast<const void*>(gemm_bf16_tc_kernel<true, 1>), int(TC_SMEM)) ||
      !smem_attr(reinterpret_cast<const void*>(gemm_bf16_tc_kernel<false, 1>), int(TC_SMEM)))
    return -10;
  // TMA C path: unit column stride, 16-byte aligned rows and base, and whole
  // 16-byte row ends (a bulk store clips out-of-bounds columns per 16 bytes)
  CUtensorMap mc;
  const float* cbase = c + c_off;
  const bool tmac = g_bf16_tma_c && c_cs == 1 && (reinterpret_cast<uintptr_t>(cbase) % 16 == 0) && (c_rs * 4) % 16 == 0 &&
                    n % 4 == 0 && make_map_c32(&mc, cbase, m, n, c_rs);
  if (!tmac) memset(&mc, 0, sizeof(mc));
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.c = c;
  p.c_off = c_off;
  p.c_rs = c_rs;
  p.c_cs = c_cs;
  p.alpha = alpha;
  p.beta = beta;
  p.lower_only = lower_only;
  p.group = g_bf16_group;
  p.tiles_m = int((m + TC_BM - 1) / TC_BM);
  p.tiles_n = int((n + TC_BN - 1) / TC_BN);
  if (lower_only && (m != n)) return -1;
  p.num_tiles = lower_only ? int64_t(p.tiles_m) * (p.tiles_m + 1) / 2 : int64_t(p.tiles_m) * p.tiles_n;
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // t_reserve_sms: leave SMs to a concurrent high-priority stream (the mixed
  // solve's diagonal/inverse/panel chain) instead of holding every SM
  const int ctas = t_reserve_sms > 0 && t_reserve_sms < sms ? sms - t_reserve_sms : sms;
  const int64_t grid = p.num_tiles < ctas ? p.num_tiles : ctas;
  note_launch();
  if (tf32) {
    if (tmac)
      gemm_bf16_tc_kernel<true, 1><<<unsigned(grid), TC_THREADS, TC_SMEM, s>>>(ma, mb, mc, p);
    else
      gemm_bf16_tc_kernel<false, 1><<<unsigned(grid), TC_THREADS, TC_SMEM, s>>>(ma, mb, mc, p);
  } else {
    if (tmac)
      gemm_bf16_tc_kernel<true, 0><<<unsigned(grid), TC_THREADS, TC_SMEM, s>>>(ma, mb, mc, p);
    else
      gemm_bf16_tc_kernel<false, 0><<<unsigned(grid), TC_THREADS, TC_SMEM, s>>>(ma, mb, mc, p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}
}  // namespace

// C(fp32 view) = beta*C + alpha * A(bf16 m x k, row stride lda) * B(bf16 n x k, ldb)^T
int launch_gemm_bf16_tc(double alpha, const void* a, int64_t lda, const void* b, int64_t ldb, double beta, float* c,
                        int64_t c_off, int64_t c_rs, int64_t c_cs, int64_t m, int64_t n, int64_t k, int lower_only,
                        cudaStream_t s) {
  return launch_tc(0, alpha, a, lda, b, ldb, beta, c, c_off, c_rs, c_cs, m, n, k, lower_only, s);
}

// The same with fp32 operands consumed as tf32 (kind::tf32)
int launch_gemm_tf32_tc(double alpha, const float* a, int64_t lda, const float* b, int64_t ldb, double beta, float* c,
                        int64_t c_off, int64_t c_rs, int64_t c_cs, int64_t m, int64_t n, int64_t k, int lower_only,
                        cudaStream_t s) {
  return launch_tc(1, alpha, a, lda, b, ldb, beta, c, c_off, c_rs, c_cs, m, n, k, lower_only, s);
}

int launch_to_bf16(const float* src, int64_t soff, int64_t srs, int64_t scs, void* dst, int64_t ld, int64_t m,
                   int64_t n, int transpose, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  const int64_t total = m * n;
  const int blocks = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  note_launch();
  to_bf16_kernel<float><<<blocks, 256, 0, s>>>(src, soff, srs, scs, static_cast<__nv_bfloat16*>(dst), ld, m, n,
                                                transpose);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_f64_to_bf16(const double* src, int64_t soff, int64_t srs, int64_t scs, void* dst, int64_t ld, int64_t m,
                       int64_t n, int transpose, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  const int64_t total = m * n;
  const int blocks = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  note_launch();
  to_bf16_kernel<double><<<blocks, 256, 0, s>>>(src, soff, srs, scs, static_cast<__nv_bfloat16*>(dst), ld, m, n,
                                                 transpose);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
