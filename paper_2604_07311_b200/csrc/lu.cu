// LU with partial pivoting on B200 (reference factor/lu.py, factor/pivots.py,
// engine/trsm.py left-lower-unit case), SURVEY.md §8(f) rank 2.
//
//  * lu_leaf_kernel — the unblocked leaf (factor/lu.py:19-53) on a panel of
//    any height: a cooperative grid, each CTA owning a contiguous band of
//    rows; per column one grid-wide pivot search (partial maxima combined in
//    row order, so ties keep the smallest row and NaNs are never chosen, as
//    in the sequential scan), the row swap, the division of the column by the
//    pivot and the rank-1 update of the band — the reference's operations in
//    the reference's order for every element (a(i,j) -= a(i,k)*a(k,j),
//    unfused, ascending k).  An exactly-zero pivot column is recorded and
//    skipped like the reference.
//  * apply_pivots_kernel — LAPACK-style swap list, one thread per column,
//    swaps in list order (factor/pivots.py:46-61).
//  * trsm_left_base_kernel — unit-lower X = T^-1 (alpha B) for n <= 32, one
//    thread per column, row by row, one ascending chain per element
//    (engine/trsm.py:114-125); the recursion above it lives in capi.cu.
//  * trsm_upper_base_kernel — the backward solve with the non-unit upper
//    factor used by lu_solve (no bitwise contract: the reference does it
//    with NumPy row operations, factor/lu.py:117-130).
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>

namespace bf {

int g_lu_grid_max = 0;  // bf_set_option("lu_grid", g): cap the leaf's cooperative grid (0 = SM-derived)

namespace {

namespace cg = cooperative_groups;

constexpr int LU_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(LU_THREADS) lu_leaf_kernel(T* a, int64_t off, int64_t rs, int64_t cs, int64_t m,
                                                           int64_t n, int64_t* piv, int* d_sing, int64_t base,
                                                           double* part_v, int64_t* part_i) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, tid = threadIdx.x;
  const int64_t chunk = (m + G - 1) / G;
  const int64_t r0 = int64_t(blockIdx.x) * chunk, r1 = r0 + chunk < m ? r0 + chunk : m;
  const int64_t steps = m < n ? m : n;
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int64_t red_i[LU_THREADS / 32];
  // The panel is shared by the CTAs through L2: every read bypasses L1 (not
  // coherent across SMs — a row swapped by CTA 0 may sit stale in another
  // SM's L1), every write is write-through.
  auto at = [&](int64_t i, int64_t j) -> T& { return a[off + i * rs + j * cs]; };
  auto ld = [&](int64_t i, int64_t j) -> T { return __ldcg(a + off + i * rs + j * cs); };
  for (int64_t k = 0; k < steps; ++k) {
    // (a) this band's best candidate among rows > k: strict '>' in ascending
    // row order per thread, then the smallest row among equal maxima
    double bv = -1.0;
    int64_t bi = -1;
    const int64_t lo = r0 > k + 1 ? r0 : k + 1;
    for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
      const double v = double(fabs(ld(i, k)));
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
      for (int w = 1; w < LU_THREADS / 32; ++w)
        if (red_i[w] >= 0 && (red_v[w] > bv || (red_v[w] == bv && (bi < 0 || red_i[w] < bi)))) {
          bv = red_v[w];
          bi = red_i[w];
        }
      part_v[blockIdx.x] = bv;
      part_i[blockIdx.x] = bi;
    }
    grid.sync();
    // (b) every CTA combines the bands in row order from the diagonal entry,
    // exactly the sequential scan: a later band wins only with a larger value
    double best = double(fabs(ld(k, k)));
    int64_t p = k;
    for (int c = 0; c < G; ++c) {
      const int64_t ci = __ldcg(part_i + c);
      const double cv = __ldcg(part_v + c);
      if (ci >= 0 && cv > best) {
        best = cv;
        p = ci;
      }
    }
    if (blockIdx.x == 0 && tid == 0) {
      piv[k] = p;
      if (best == 0.0 && *d_sing < 0) *d_sing = int(base + k);
    }
    const bool live = !(best == 0.0);
    // every thread of CTA 0 has read a(k,k) before any of them overwrites it
    // (other CTAs only need `live`, which the swap cannot change)
    __syncthreads();
    // (c) the swap, by CTA 0
    if (live && p != k && blockIdx.x == 0)
      for (int64_t j = tid; j < n; j += LU_THREADS) {
        const T t = ld(k, j);
        at(k, j) = ld(p, j);
        at(p, j) = t;
      }
    grid.sync();
    // (d) divide the column by the pivot, rank-1 update of this band
    if (live) {
      const T d = ld(k, k);
      for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
        const T lik = Ops<T>::div(ld(i, k), d);
        at(i, k) = lik;
        for (int64_t j = k + 1; j < n; ++j) at(i, j) = Ops<T>::sub(ld(i, j), Ops<T>::mul(lik, ld(k, j)));
      }
    }
    grid.sync();
  }
}

template <typename T>
__global__ void apply_pivots_kernel(T* a, int64_t off, int64_t rs, int64_t cs, int64_t ncols, const int64_t* piv,
                                    int64_t count, int64_t sub, int backward) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T* col = a + off + j * cs;
  for (int64_t q = 0; q < count; ++q) {
    const int64_t k = backward ? count - 1 - q : q;
    const int64_t p = piv[k] - sub;
    if (p != k) {
      const T t = col[k * rs];
      col[k * rs] = col[p * rs];
      col[p * rs] = t;
    }
  }
}

__global__ void add_offset_kernel(int64_t* piv, int64_t count, int64_t delta) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < count) piv[q] += delta;
}

template <typename T>
__global__ void trsm_left_base_kernel(double alpha, const T* t, int64_t toff, int64_t trs, int64_t tcs, T* b,
                                      int64_t boff, int64_t brs, int64_t bcs, int n, int64_t ncols) {
  __shared__ T st[32][33];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, p = e % n;
    st[i][p] = p < i ? t[toff + i * trs + p * tcs] : T(0);
  }
  __syncthreads();
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < n ? b[boff + i * brs + j * bcs] : T(0);
  if (alpha != 1.0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = T(Ops<double>::mul(double(x[i]), alpha));
  }
#pragma unroll
  for (int i = 1; i < 32; ++i) {
    if (i < n) {
      T acc = x[i];
#pragma unroll
      for (int p = 0; p < i; ++p) acc = Ops<T>::sub(acc, Ops<T>::mul(st[i][p], x[p]));
      x[i] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) b[boff + i * brs + j * bcs] = x[i];
}

// upper, non-unit, backward: X = U^-1 B for n <= 32 (lu_solve's last stage)
template <typename T>
__global__ void trsm_upper_base_kernel(const T* u, int64_t uoff, int64_t urs, int64_t ucs, T* b, int64_t boff,
                                       int64_t brs, int64_t bcs, int n, int64_t ncols) {
  __shared__ T su[32][33];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, p = e % n;
    su[i][p] = p >= i ? u[uoff + i * urs + p * ucs] : T(0);
  }
  __syncthreads();
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < n ? b[boff + i * brs + j * bcs] : T(0);
#pragma unroll
  for (int i = 31; i >= 0; --i) {
    if (i < n) {
      T acc = x[i];
#pragma unroll
      for (int p = i + 1; p < 32; ++p)
        if (p < n) acc = Ops<T>::sub(acc, Ops<T>::mul(su[i][p], x[p]));
      x[i] = Ops<T>::div(acc, su[i][i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) b[boff + i * brs + j * bcs] = x[i];
}

int grid_cap_lu() {
  static int cap = 0;
  if (!cap) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lu_leaf_kernel<double>, LU_THREADS, 0);
    cap = sms * (per > 0 ? (per < 2 ? per : 2) : 1);
  }
  return cap;
}

}  // namespace

int launch_lu_leaf(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, int64_t* piv,
                   int* d_sing, int64_t base, cudaStream_t s) {
  const int64_t steps = m < n ? m : n;
  if (steps <= 0) return 0;
  int G = int((m + 127) / 128);
  const int cap = g_lu_grid_max > 0 ? g_lu_grid_max : grid_cap_lu();
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  static double* part_v[64] = {};
  static int64_t* part_i[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!part_v[dev]) {
    if (cudaMalloc(&part_v[dev], 4096 * sizeof(double)) != cudaSuccess) return -12;
    if (cudaMalloc(&part_i[dev], 4096 * sizeof(int64_t)) != cudaSuccess) return -12;
  }
  if (G > 4096) G = 4096;
  double* pv = part_v[dev];
  int64_t* pi = part_i[dev];
  note_launch();
  cudaError_t e;
  if (is_f64) {
    double* ad = static_cast<double*>(a);
    void* args[] = {&ad, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_kernel<double>), dim3(G), dim3(LU_THREADS), args,
                                    0, s);
  } else {
    float* af = static_cast<float*>(a);
    void* args[] = {&af, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_kernel<float>), dim3(G), dim3(LU_THREADS), args, 0,
                                    s);
  }
  return e == cudaSuccess ? 0 : -11;
}

int launch_apply_pivots(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t ncols, const int64_t* piv,
                        int64_t count, int64_t sub, int backward, cudaStream_t s) {
  if (ncols <= 0 || count <= 0) return 0;
  note_launch();
  const unsigned blocks = unsigned((ncols + 255) / 256);
  if (is_f64)
    apply_pivots_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(a), off, rs, cs, ncols, piv, count, sub,
                                                       backward);
  else
    apply_pivots_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(a), off, rs, cs, ncols, piv, count, sub,
                                                      backward);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_add_offset(int64_t* piv, int64_t count, int64_t delta, cudaStream_t s) {
  if (count <= 0 || delta == 0) return 0;
  note_launch();
  add_offset_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(piv, count, delta);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_trsm_left_base(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                          int64_t boff, int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s) {
  if (ncols <= 0 || n <= 0) return 0;
  if (n > 32) return -3;
  note_launch();
  const unsigned blocks = unsigned((ncols + 127) / 128);
  if (is_f64)
    trsm_left_base_kernel<double><<<blocks, 128, 0, s>>>(alpha, static_cast<const double*>(t), toff, trs, tcs,
                                                         static_cast<double*>(b), boff, brs, bcs, n, ncols);
  else
    trsm_left_base_kernel<float><<<blocks, 128, 0, s>>>(alpha, static_cast<const float*>(t), toff, trs, tcs,
                                                        static_cast<float*>(b), boff, brs, bcs, n, ncols);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_trsm_upper_base(int is_f64, const void* u, int64_t uoff, int64_t urs, int64_t ucs, void* b, int64_t boff,
                           int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s) {
  if (ncols <= 0 || n <= 0) return 0;
  if (n > 32) return -3;
  note_launch();
  const unsigned blocks = unsigned((ncols + 127) / 128);
  if (is_f64)
    trsm_upper_base_kernel<double><<<blocks, 128, 0, s>>>(static_cast<const double*>(u), uoff, urs, ucs,
                                                          static_cast<double*>(b), boff, brs, bcs, n, ncols);
  else
    trsm_upper_base_kernel<float><<<blocks, 128, 0, s>>>(static_cast<const float*>(u), uoff, urs, ucs,
                                                         static_cast<float*>(b), boff, brs, bcs, n, ncols);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
