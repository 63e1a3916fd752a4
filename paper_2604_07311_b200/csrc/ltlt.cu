// Pivoted LTL^T of skew-symmetric matrices (reference factor/ltlt.py),
// SURVEY.md §8(f) rank 3.  One cooperative grid walks the eliminations; per
// column j:
//   * the pivot search over |x(i,j)|, i > j (partial maxima combined in row
//     order: the first maximum, like np.argmax);
//   * the two-sided symmetric swap of indices j+1 and p on the stored lower
//     triangle (factor/ltlt.py:66-88) — four disjoint element sets, spread
//     over the grid; the blocked form swaps the panel's w history rows too;
//   * unblocked (ltlt.py:157-182): the Gauss multipliers m = x(:,j)/alpha,
//     w = x(:,j+1), and the right-looking rank-2 update
//     x(i,c) += m_i w_c - w_i m_c, each element rounded like the reference's
//     compiled loop (bit-identical);
//   * blocked panel (ltlt.py:131-147): column j+1 brought current against the
//     panel's m/w history (two length-h dot products per row: the reference
//     uses NumPy/BLAS here, so this part agrees to rounding), then the
//     multipliers; the trailing update is the fused skew sandwich.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>

namespace bf {

int g_ltlt_grid_max = 0;  // bf_set_option("ltlt_grid", g): cap the stepper's cooperative grid (0 = one CTA per SM)

namespace {

namespace cg = cooperative_groups;

constexpr int LT_THREADS = 256;

template <typename T>
struct LtArgs {
  T* x;
  int64_t off, rs, cs, n;
  int64_t j0, j1;   // eliminations [j0, j1)
  int blocked;      // 1: panel mode (history in w), 0: unblocked right-looking
  int64_t k;        // panel start (blocked)
  T* w;             // blocked: n x wld history; unblocked: unused
  int64_t wld;
  int64_t* piv;
  T* t;
  T* mvec;          // unblocked: length n
  T* wvec;
  double* part_v;   // >= gridDim.x
  int64_t* part_i;
};

template <typename T>
__global__ void __launch_bounds__(LT_THREADS) ltlt_kernel(LtArgs<T> A) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, tid = threadIdx.x, cta = blockIdx.x;
  const int64_t gt = int64_t(cta) * LT_THREADS + tid, GT = int64_t(G) * LT_THREADS;
  const int lane = tid & 31;
  const int64_t gw = gt >> 5, GW = GT >> 5;  // global warp index / count
  const int64_t n = A.n;
  auto X = [&](int64_t i, int64_t j) -> T& { return A.x[A.off + i * A.rs + j * A.cs]; };
  auto W = [&](int64_t i, int64_t q) -> T& { return A.w[i * A.wld + q]; };
  __shared__ double red_v[LT_THREADS / 32];
  __shared__ int64_t red_i[LT_THREADS / 32];
  __shared__ int64_t s_p;
  for (int64_t j = A.j0; j < A.j1; ++j) {
    // ---- pivot search over rows j+1 .. n-1 of column j (contiguous bands)
    const int64_t rows = n - j - 1;
    const int64_t chunk = (rows + G - 1) / G;
    const int64_t r0 = j + 1 + int64_t(cta) * chunk;
    const int64_t r1 = r0 + chunk < n ? r0 + chunk : n;
    double bv = -1.0;
    int64_t bi = -1;
    for (int64_t i = r0 + tid; i < r1; i += LT_THREADS) {
      const double v = double(fabs(X(i, j)));
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (ov > bv || (ov == bv && (bi < 0 || oi < bi)))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_i[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < LT_THREADS / 32; ++q)
        if (red_i[q] >= 0 && (red_v[q] > bv || (red_v[q] == bv && (bi < 0 || red_i[q] < bi)))) {
          bv = red_v[q];
          bi = red_i[q];
        }
      A.part_v[cta] = bv;
      A.part_i[cta] = bi;
    }
    grid.sync();
    if (tid < 32) {
      double cv = -1.0;
      int64_t ci = -1;
      for (int q = tid; q < G; q += 32) {  // ties resolve by index: any scan order gives the first maximum
        const int64_t oi = __ldcg(A.part_i + q);
        const double ov = __ldcg(A.part_v + q);
        if (oi >= 0 && (ov > cv || (ov == cv && (ci < 0 || oi < ci)))) {
          cv = ov;
          ci = oi;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, cv, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, ci, o);
        if (oi >= 0 && (ov > cv || (ov == cv && (ci < 0 || oi < ci)))) {
          cv = ov;
          ci = oi;
        }
      }
      if (tid == 0) s_p = ci < 0 ? j + 1 : ci;
    }
    __syncthreads();
    const int64_t a = j + 1, b = s_p;
    if (b != a) {
      if (gt == 0) A.piv[a] = b;
      // (1) rows a and b left of column a
      for (int64_t q = gt; q < a; q += GT) {
        const T u = X(a, q), v = X(b, q);
        X(a, q) = v;
        X(b, q) = u;
      }
      // (2) column a between a and b  <->  row b between a and b, negated
      for (int64_t i = a + 1 + gt; i < b; i += GT) {
        const T ca = X(i, a), rb = X(b, i);
        X(i, a) = -rb;
        X(b, i) = -ca;
      }
      // (3) the corner
      if (gt == 0) X(b, a) = -X(b, a);
      // (4) columns a and b below b
      for (int64_t i = b + 1 + gt; i < n; i += GT) {
        const T u = X(i, a), v = X(i, b);
        X(i, a) = v;
        X(i, b) = u;
      }
      // the panel's w history swaps rows with the matrix
      if (A.blocked)
        for (int64_t q = gt; q < A.wld; q += GT) {
          const T u = W(a, q), v = W(b, q);
          W(a, q) = v;
          W(b, q) = u;
        }
    }
    grid.sync();
    const int64_t h = j - A.k;
    if (A.blocked && h > 0 && j + 2 <= n - 1) {
      // bring column j+1 current: += x(i, k:j) . w(j+1, :h) ; -= w(i, :h) . x(j+1, k:j)
      // (BLAS products in the reference: to rounding); one warp per row, lanes along the row
      for (int64_t i = j + 2 + gw; i < n; i += GW) {
        T s1 = T(0), s2 = T(0);
        for (int64_t q = lane; q < h; q += 32) {
          s1 = Ops<T>::fma_(X(i, A.k + q), W(j + 1, q), s1);
          s2 = Ops<T>::fma_(W(i, q), X(j + 1, A.k + q), s2);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) X(i, j + 1) = Ops<T>::sub(Ops<T>::add(X(i, j + 1), s1), s2);
      }
      grid.sync();
    }
    const T alpha = X(j + 1, j);
    if (gt == 0) A.t[j] = alpha;
    if (j + 2 < n) {
      const bool nz = alpha != T(0);
      for (int64_t i = j + 2 + gt; i < n; i += GT) {
        const T m = nz ? Ops<T>::div(X(i, j), alpha) : T(0);
        const T wv = X(i, j + 1);
        if (A.blocked) {
          W(i, h) = wv;
        } else {
          A.mvec[i] = m;
          A.wvec[i] = wv;
        }
        X(i, j) = m;
      }
      if (!A.blocked && nz) {
        grid.sync();
        // right-looking rank-2 update of the trailing lower triangle (elementwise,
        // each element rounded like the reference's loop); one warp per row
        for (int64_t i = j + 3 + gw; i < n; i += GW) {
          const T mi = __ldcg(A.mvec + i), wi = __ldcg(A.wvec + i);
          for (int64_t c = j + 2 + lane; c < i; c += 32)
            X(i, c) = Ops<T>::add(X(i, c), Ops<T>::sub(Ops<T>::mul(mi, __ldcg(A.wvec + c)),
                                                       Ops<T>::mul(wi, __ldcg(A.mvec + c))));
        }
      }
    }
    grid.sync();
  }
}

}  // namespace

int launch_ltlt(int is_f64, void* x, int64_t off, int64_t rs, int64_t cs, int64_t n, int64_t j0, int64_t j1,
                int blocked, int64_t k, void* w, int64_t wld, int64_t* piv, void* t, void* mvec, void* wvec,
                cudaStream_t s) {
  if (j1 <= j0) return 0;
  static double* pv[64] = {};
  static int64_t* pi[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!pv[dev]) {
    if (cudaMalloc(&pv[dev], 256 * sizeof(double)) != cudaSuccess) return -12;
    if (cudaMalloc(&pi[dev], 256 * sizeof(int64_t)) != cudaSuccess) return -12;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one warp per trailing row at most ~2 rows per warp: up to one CTA per SM
  int G = int((n + 15) / 16);
  if (G < 1) G = 1;
  if (G > sms) G = sms;
  if (G > 256) G = 256;
  if (g_ltlt_grid_max > 0 && G > g_ltlt_grid_max) G = g_ltlt_grid_max;
  note_launch();
  cudaError_t e;
  if (is_f64) {
    LtArgs<double> A{static_cast<double*>(x), off, rs, cs, n, j0, j1, blocked, k, static_cast<double*>(w), wld, piv,
                     static_cast<double*>(t), static_cast<double*>(mvec), static_cast<double*>(wvec), pv[dev], pi[dev]};
    void* args[] = {&A};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ltlt_kernel<double>), dim3(G), dim3(LT_THREADS), args, 0,
                                    s);
  } else {
    LtArgs<float> A{static_cast<float*>(x), off, rs, cs, n, j0, j1, blocked, k, static_cast<float*>(w), wld, piv,
                    static_cast<float*>(t), static_cast<float*>(mvec), static_cast<float*>(wvec), pv[dev], pi[dev]};
    void* args[] = {&A};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ltlt_kernel<float>), dim3(G), dim3(LT_THREADS), args, 0,
                                    s);
  }
  return e == cudaSuccess ? 0 : -11;
}

}  // namespace bf
