// FP32-storage GEMM / GEMMT on the CUDA cores (FFMA for f32 accumulation,
// DFMA for the reference's f32-storage / f64-accumulation mode).
//
// Same contract as gemm_dmma.cu (engine/gemm.py:74-160): kc segments folded
// into C as C = beta_eff*C + alpha*t (unfused) in the accumulation type and
// rounded to the storage type on every fold (engine/kernels.py:597-610 stores
// into the f32 buffer each kc block).  Within a segment the reference's
// micro-kernel accumulators start from the literal 0.0 and are therefore f64:
// with f64 packing (acc f64) every step is an f64 fma; with f32 packing
// (acc f32) the product is rounded to f32 and added in f64; the segment sum
// is rounded to the acc type when it lands in tile[] (engine/kernels.py:507-522).
#include "bf_common.cuh"
#include "bf_internal.h"

namespace bf {

namespace {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16, SB_THREADS = 256;  // 16x16 threads, 4x4 outputs each

template <typename T>
__device__ __forceinline__ T ld_elem(const OperandMK& op, int64_t mn, int64_t k) {
  const T* g = static_cast<const T*>(op.base);
  if (op.layout == GL_TRIDIAG) {
    // the skew sandwich's B = T*A^T formed while staged (engine/kernels.py:93-122
    // pack_b_block_tridiag): W[k, mn] = t[k-1]*A(mn, k-1) - t[k]*A(mn, k+1) in the
    // storage type, edge terms dropped; op.tvec holds T's subdiagonal (type T)
    const T* t = reinterpret_cast<const T*>(op.tvec);
    const T* row = g + op.off + mn * op.s_mn;
    T acc = T(0);
    if (k > 0) acc = Ops<T>::add(acc, Ops<T>::mul(t[k - 1], row[(k - 1) * op.s_k]));
    if (k < op.k_total - 1) acc = Ops<T>::sub(acc, Ops<T>::mul(t[k], row[(k + 1) * op.s_k]));
    return acc;
  }
  if (op.mn_scat) return g[op.mn_scat[mn] + op.k_scat[k]];
  return g[op.off + mn * op.s_mn + k * op.s_k];
}

template <typename T, typename Acc>
__global__ void __launch_bounds__(SB_THREADS) gemm_simt_kernel(const GemmParams p) {
  if (aborted(p)) return;
  __shared__ Acc sA[2][SB_K][SB_M + 1];
  __shared__ Acc sB[2][SB_K][SB_N + 1];

  const int64_t ti = blockIdx.x % p.tiles_m, tj = blockIdx.x / p.tiles_m;
  const int64_t m0 = ti * SB_M, n0 = tj * SB_N;
  if (p.lower_only) {
    int64_t row_hi = (m0 + SB_M < p.m ? m0 + SB_M : p.m) - 1;
    if (row_hi < n0) return;
  }
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;

  const int64_t K = p.k;
  const int64_t kc = p.kc < K ? p.kc : K;
  const int64_t nseg = (K + kc - 1) / kc;
  const int64_t tps = (kc + SB_K - 1) / SB_K;
  const int64_t last_len = K - (nseg - 1) * kc;
  const int64_t tps_last = (last_len + SB_K - 1) / SB_K;
  const int64_t ntiles = (nseg - 1) * tps + tps_last;
  const Acc alpha = Acc(p.alpha), beta = Acc(p.beta);

  // register-staged loads: each thread moves 4 A and 4 B elements per k tile
  Acc ra[4], rb[4];
  auto fetch = [&](int64_t kt) {
    int64_t seg = kt / tps, sub = kt - seg * tps;
    int64_t k_lo = seg * kc + sub * SB_K;
    int64_t seg_end = (seg + 1) * kc < K ? (seg + 1) * kc : K;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + r * SB_THREADS;  // 0..1023 over a 64x16 tile
      int mn, k;
      if (p.a.layout == GL_MNMAJOR) { mn = e % SB_M; k = e / SB_M; } else { mn = e / SB_K; k = e % SB_K; }
      int64_t gm = m0 + mn, gk = k_lo + k;
      ra[r] = (gm < p.m && gk < seg_end) ? Acc(ld_elem<T>(p.a, gm, gk)) : Acc(0);
      if (p.b.layout == GL_MNMAJOR) { mn = e % SB_N; k = e / SB_N; } else { mn = e / SB_K; k = e % SB_K; }
      int64_t gn = n0 + mn;
      gk = k_lo + k;
      rb[r] = (gn < p.n && gk < seg_end) ? Acc(ld_elem<T>(p.b, gn, gk)) : Acc(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + r * SB_THREADS;
      int mn, k;
      if (p.a.layout == GL_MNMAJOR) { mn = e % SB_M; k = e / SB_M; } else { mn = e / SB_K; k = e % SB_K; }
      sA[buf][k][mn] = ra[r];
      if (p.b.layout == GL_MNMAJOR) { mn = e % SB_N; k = e / SB_N; } else { mn = e / SB_K; k = e % SB_K; }
      sB[buf][k][mn] = rb[r];
    }
  };

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  T* C = static_cast<T*>(p.c);
  fetch(0);
  stash(0);
  __syncthreads();
  for (int64_t kt = 0; kt < ntiles; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < ntiles) fetch(kt + 1);
#pragma unroll
    for (int k = 0; k < SB_K; ++k) {
      Acc a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[buf][k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[buf][k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (sizeof(Acc) == 4)
            acc[i][j] = __dadd_rn(acc[i][j], double(__fmul_rn(a[i], b[j])));
          else
            acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
        }
    }
    const int64_t seg = kt / tps, sub = kt - seg * tps;
    const bool seg_done = (seg < nseg - 1) ? (sub == tps - 1) : (sub == tps_last - 1);
    if (seg_done) {
      const Acc beta_eff = seg == 0 ? beta : Acc(1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t gi = m0 + ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t gj = n0 + tx + 16 * j;
          if (gi < p.m && gj < p.n && (!p.lower_only || gi >= gj)) {
            int64_t addr = p.c_rscat ? p.c_rscat[gi] + p.c_cscat[gj] : p.c_off + gi * p.c_rs + gj * p.c_cs;
            Acc v = Ops<Acc>::mul(alpha, Acc(acc[i][j]));
            if (beta_eff != Acc(0)) v = Ops<Acc>::add(Ops<Acc>::mul(beta_eff, Acc(C[addr])), v);
            C[addr] = T(v);
          }
          acc[i][j] = 0.0;
        }
      }
    }
    if (kt + 1 < ntiles) {
      stash(buf ^ 1);
    }
    __syncthreads();
  }
}

template <typename T, typename Acc>
int run_simt(const GemmParams& p_in, cudaStream_t s) {
  GemmParams p = p_in;
  p.tiles_m = int((p.m + SB_M - 1) / SB_M);
  p.tiles_n = int((p.n + SB_N - 1) / SB_N);
  int64_t nt = int64_t(p.tiles_m) * p.tiles_n;
  if (nt <= 0) return 0;
  if (nt > 0x7fffffffLL) return -3;
  note_launch();
  gemm_simt_kernel<T, Acc><<<unsigned(nt), SB_THREADS, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace

int launch_gemm_simt_f32(const GemmParams& p, cudaStream_t s) { return run_simt<float, float>(p, s); }
int launch_gemm_simt_f32acc64(const GemmParams& p, cudaStream_t s) { return run_simt<float, double>(p, s); }

}  // namespace bf
