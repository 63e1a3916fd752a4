// Latency-class kernels of the Cholesky path:
//   * diagonal-block POTRF leaves, the three unblocked variants
//     (factor/cholesky.py:31-89), one CTA, shared-memory resident up to
//     LEAF_SMEM_N, in-place on global memory (L2-resident) beyond;
//   * the TRSM base case X*tril(T)^T = alpha*B for n <= 32
//     (engine/trsm.py:96-111), one thread per right-hand-side row;
//   * C := beta*C on the full matrix or its lower triangle
//     (engine/kernels.py:125-139).
// Every floating-point step is the reference's own unfused IEEE operation in
// the reference's order (see bf_common.cuh), so these kernels are
// bit-identical to the numba leaves.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cstdio>

namespace bf {

int g_trsm_warp = 1;
int g_leaf_blocked = 1;
int g_leaf_pipe = 1;
int g_pdl = 1;  // bf_set_option("pdl", 0|1): programmatic dependent launch for the leaf, fused-TRSM and TMA GEMM kernels     // bf_set_option("leaf_pipe", 0|1): blocked leaf, next chain under the previous trailing update

namespace {

// ------------------------------------------------------------------ scale --
template <typename T, typename Acc>
__global__ void scale_kernel(T* c, int64_t off, int64_t m, int64_t n, int64_t rs, int64_t cs,
                             const int64_t* rscat, const int64_t* cscat, Acc beta, int lower_only) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t i = e / n, j = e % n;
    if (lower_only && j > i) continue;
    int64_t a = rscat ? rscat[i] + cscat[j] : off + i * rs + j * cs;
    c[a] = (beta == Acc(0)) ? T(0) : T(Ops<Acc>::mul(beta, Acc(c[a])));
  }
}

// ------------------------------------------------------------- POTRF leaf --
constexpr int LEAF_THREADS = 512;

template <typename T>
struct Mat {
  T* p;
  int64_t rs, cs;
  __device__ __forceinline__ T& operator()(int64_t i, int64_t j) const { return p[i * rs + j * cs]; }
};

// variant 3, right-looking: scale column k, rank-1 update of the trailing triangle
template <typename T, int NT = LEAF_THREADS>
__device__ int leaf_v3(Mat<T> a, int n, int* s_flag, T* s_d) {
  const int tid = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      T d = a(k, k);
      if (!(d > T(0))) {
        *s_flag = k;
      } else {
        d = Ops<T>::sqrt_(d);
        a(k, k) = d;
        *s_d = d;
      }
    }
    __syncthreads();
    if (*s_flag >= 0) return *s_flag;
    const T d = *s_d;
    for (int i = k + 1 + tid; i < n; i += NT) a(i, k) = Ops<T>::div(a(i, k), d);
    __syncthreads();
    // trailing triangle k < j <= i < n; 32 x (NT/32) thread grid, j fastest
    const int tx = tid & 31, ty = tid >> 5;
    for (int i = k + 1 + ty; i < n; i += NT / 32) {
      const T aik = a(i, k);
      for (int j = k + 1 + tx; j <= i; j += 32) a(i, j) = Ops<T>::sub(a(i, j), Ops<T>::mul(aik, a(j, k)));
    }
    __syncthreads();
  }
  return -1;
}

// variant 2, left-looking: dot products against the finished columns, then scale.
// The reference's running sums start from the literal 0.0, so they are f64
// even for f32 storage (products stay in the storage type); S models that.
template <typename T>
__device__ int leaf_v2(Mat<T> a, int n, int* s_flag, double* s_d, double* s_sum) {
  using S = double;
  const int tid = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    for (int i = k + tid; i < n; i += LEAF_THREADS) {
      S s = S(0);
      if (i == k) {
        for (int p = 0; p < k; ++p) {
          const T v = a(k, p);
          s = Ops<S>::add(s, S(Ops<T>::mul(v, v)));
        }
      } else {
        for (int p = 0; p < k; ++p) s = Ops<S>::add(s, S(Ops<T>::mul(a(i, p), a(k, p))));
      }
      s_sum[i] = s;
    }
    __syncthreads();
    if (tid == 0) {
      S d = Ops<S>::sub(S(a(k, k)), s_sum[k]);
      if (!(d > S(0))) {
        *s_flag = k;
      } else {
        d = Ops<S>::sqrt_(d);
        a(k, k) = T(d);
        *s_d = d;
      }
    }
    __syncthreads();
    if (*s_flag >= 0) return *s_flag;
    const S d = *s_d;
    for (int i = k + 1 + tid; i < n; i += LEAF_THREADS) a(i, k) = T(Ops<S>::div(Ops<S>::sub(S(a(i, k)), s_sum[i]), d));
    __syncthreads();
  }
  return -1;
}

// variant 1, bordered: solve row k against the finished triangle.  Warp 0
// pipelines the row solve so every partial sum s_j accumulates a(k,p)*a(j,p)
// in ascending p exactly as the scalar loop does (f64 sums, as in leaf_v2).
template <typename T>
__device__ int leaf_v1(Mat<T> a, int n, int* s_flag, double* s_sum) {
  using S = double;
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    for (int k = 0; k < n && *s_flag < 0; ++k) {
      for (int j = lane; j <= k; j += 32) s_sum[j] = S(0);
      __syncwarp();
      for (int p = 0; p < k; ++p) {
        T x = T(0);
        if (lane == (p & 31)) {
          x = T(Ops<S>::div(Ops<S>::sub(S(a(k, p)), s_sum[p]), S(a(p, p))));
          a(k, p) = x;
        }
        x = __shfl_sync(0xffffffffu, x, p & 31);
        for (int j = p + 1 + lane; j < k; j += 32) s_sum[j] = Ops<S>::add(s_sum[j], S(Ops<T>::mul(x, a(j, p))));
        if (lane == 0) s_sum[k] = Ops<S>::add(s_sum[k], S(Ops<T>::mul(x, x)));
        __syncwarp();
      }
      if (lane == 0) {
        S d = Ops<S>::sub(S(a(k, k)), s_sum[k]);
        if (!(d > S(0)))
          *s_flag = k;
        else
          a(k, k) = T(Ops<S>::sqrt_(d));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  return *s_flag;
}

template <typename T, bool SMEM>
__global__ void __launch_bounds__(LEAF_THREADS) potrf_leaf_kernel(T* g, int64_t off, int n, int64_t rs,
                                                                  int64_t cs, int variant, int64_t base_index,
                                                                  int* d_info, double* scratch) {
  if (d_info != nullptr && *d_info >= 0) return;  // an earlier leaf already failed
  extern __shared__ __align__(16) unsigned char leaf_smem[];
  __shared__ int s_flag;
  __shared__ T s_d;
  __shared__ double s_d64;
  const int tid = threadIdx.x;
  if (tid == 0) s_flag = -1;
  Mat<T> gm{g + off, rs, cs};
  Mat<T> a = gm;
  double* s_sum = scratch;  // length n (global when the block is too large for smem)
  if constexpr (SMEM) {
    s_sum = reinterpret_cast<double*>(leaf_smem);
    T* tile = reinterpret_cast<T*>(leaf_smem + size_t(n) * sizeof(double));
    a = Mat<T>{tile, int64_t(n + 1), 1};
    for (int e = tid; e < n * n; e += LEAF_THREADS) {
      int i = e / n, j = e % n;
      if (j <= i) a(i, j) = gm(i, j);
    }
  }
  __syncthreads();
  int bad;
  if (variant == 1)
    bad = leaf_v1<T>(a, n, &s_flag, s_sum);
  else if (variant == 2)
    bad = leaf_v2<T>(a, n, &s_flag, &s_d64, s_sum);
  else
    bad = leaf_v3<T>(a, n, &s_flag, &s_d);
  __syncthreads();
  if constexpr (SMEM) {
    for (int e = tid; e < n * n; e += LEAF_THREADS) {
      int i = e / n, j = e % n;
      if (j <= i) gm(i, j) = a(i, j);
    }
  }
  if (tid == 0 && bad >= 0 && d_info != nullptr) *d_info = int(base_index + bad);
}

// Variant 3 (right-looking, factor/cholesky.py:74-89) for n <= 128: the
// block lives in shared memory; 8 warps, warp w updating columns j = w mod 8
// (lanes over rows).  The pivot is on the critical path, so at step k the
// warp owning column k+1 updates that column first, then takes the sqrt and
// scales it in place before turning to its other columns; one barrier per
// step.  (Register-resident variants with 16 warps lost to issue contention:
// the arbiter favours high warp ids, so a low-id pivot warp was starved by
// its neighbours' updates.)  Every element receives the reference's
// operations in the reference's order; a failing pivot leaves the
// reference's partial state.
template <typename T>
__global__ void __launch_bounds__(256) potrf_leaf_v3_smem_kernel(T* g, int64_t off, int n, int64_t rs, int64_t cs,
                                                                 int64_t base_index, int* d_info) {
  if (d_info != nullptr && *d_info >= 0) return;
  extern __shared__ __align__(16) unsigned char leaf_v3_smem[];
  T* A = reinterpret_cast<T*>(leaf_v3_smem);
  constexpr int LD = 129;
  __shared__ int s_flag;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int e = tid; e < n * n; e += 256) {
    int i, j;
    if (cs == 1) { i = e / n; j = e % n; } else { j = e / n; i = e % n; }
    if (j <= i) {
      if constexpr (sizeof(T) == 8)
        cp_async_8(&A[i * LD + j], &g[off + i * rs + j * cs], 8);
      else
        cp_async_4(&A[i * LD + j], &g[off + i * rs + j * cs], 4);
    }
  }
  cp_async_commit();
  if (tid == 0) s_flag = -1;
  cp_async_wait<0>();
  __syncthreads();
  // Step k in two barrier-separated halves so every division runs in
  // parallel (one per thread) and the only serial work per pivot is one
  // multiply-subtract, a sqrt and a division:
  //   half 1: the last thread updates (k+1,k+1) and takes its sqrt; thread t
  //           updates (k+2+t, k+1); all warps update columns j > k+1;
  //   half 2: thread t scales its element of column k+1.
  __shared__ T s_d;
  constexpr int PIV = 255;  // highest warp id: favoured by the issue arbiter
  if (tid == PIV) {
    const T diag = A[0];
    if (!(diag > T(0))) {
      s_flag = 0;
    } else {
      s_d = Ops<T>::sqrt_(diag);
      A[0] = s_d;
    }
  }
  __syncthreads();
  if (s_flag < 0 && tid + 1 < n) A[(tid + 1) * LD] = Ops<T>::div(A[(tid + 1) * LD], s_d);
  int bad = -1;
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    __syncthreads();  // column k final (or its pivot failed)
    if (s_flag >= 0) {
      bad = s_flag;
      break;
    }
    const int kn = k + 1;
    if (kn >= n) break;
    const T akn = A[kn * LD + k];
    if (tid == PIV) {
      const T diag = Ops<T>::sub(A[kn * LD + kn], Ops<T>::mul(akn, akn));
      if (!(diag > T(0))) {
        A[kn * LD + kn] = diag;
        s_flag = kn;
      } else {
        s_d = Ops<T>::sqrt_(diag);
        A[kn * LD + kn] = s_d;
      }
    }
    T x = T(0);
    const int ir = kn + 1 + tid;
    if (ir < n) x = Ops<T>::sub(A[ir * LD + kn], Ops<T>::mul(A[ir * LD + k], akn));
    // Columns j = w + 8c > kn, rows i = lane + 32q >= j; rows >= n hold
    // garbage that is never stored back.  Loads, arithmetic and stores are
    // separate phases (a fused load-use-store loop serialises on the
    // may-alias shared-memory dependences).
    T aik[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) aik[q] = A[(lane + 32 * q) * LD + k];
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      if (w + 8 * (4 * cb + 3) <= kn) continue;  // whole batch finished (uniform)
      T val[4][4], ajk[4];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int j = w + 8 * (4 * cb + cc);
        ajk[cc] = A[(j & 127) * LD + k];
#pragma unroll
        for (int q = 0; q < 4; ++q) val[cc][q] = A[(lane + 32 * q) * LD + (j & 127)];
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int j = w + 8 * (4 * cb + cc);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q;
          if (j > kn && j < n && i >= j) A[i * LD + j] = Ops<T>::sub(val[cc][q], Ops<T>::mul(aik[q], ajk[cc]));
        }
      }
    }
    __syncthreads();  // s_d / s_flag ready
    if (ir < n) A[ir * LD + kn] = s_flag >= 0 ? x : Ops<T>::div(x, s_d);
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += 256) {
    int i, j;
    if (cs == 1) { i = e / n; j = e % n; } else { j = e / n; i = e % n; }
    if (j <= i) g[off + i * rs + j * cs] = A[i * LD + j];
  }
  if (tid == 0 && bad >= 0 && d_info != nullptr) *d_info = int(base_index + bad);
}

// --------------------------------------------------------- TRSM base case --
// X * tril(T)^T = alpha * B, B is m x n (n <= 32), T n x n; one thread per
// right-hand-side row held in registers, the triangle in shared memory.
template <typename T>
__global__ void __launch_bounds__(128) trsm_base_right_kernel(double alpha, const T* t, int64_t toff, int64_t trs,
                                                              int64_t tcs, T* b, int64_t boff, int64_t brs,
                                                              int64_t bcs, int64_t m, int n, int* d_singular,
                                                              int64_t index_base, const int* abort_flag) {
  if (abort_flag != nullptr && *abort_flag >= 0) return;
  __shared__ T st[32][33];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int j = e / n, p = e % n;
    st[j][p] = (p <= j) ? t[toff + j * trs + p * tcs] : T(0);
  }
  __syncthreads();
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  T x[32];
  T* row = b + boff + i * brs;
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (j < n) ? row[j * bcs] : T(0);
  if (alpha != 1.0) {  // bbuf *= alpha: the product is formed in f64 (alpha is a Python float)
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = T(Ops<double>::mul(double(x[j]), alpha));
  }
  int bad = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j < n && bad < 0) {
      const T d = st[j][j];
      if (d == T(0)) {
        bad = j;
      } else {
        T acc = x[j];
#pragma unroll
        for (int p = 0; p < j; ++p) acc = Ops<T>::sub(acc, Ops<T>::mul(x[p], st[j][p]));
        x[j] = Ops<T>::div(acc, d);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < n) row[j * bcs] = x[j];
  // every row meets the same zero pivot, so the racing stores write one value
  if (bad >= 0 && d_singular != nullptr) *d_singular = int(index_base + bad);
}

// ------------------------------------------------- fused TRSM subtree (n<=128) --
// The whole recursion of engine/trsm.py:51-68 below a triangle of order
// n <= 128 in one launch: each CTA owns 64 rows of B (staged in shared memory
// with the triangle) and walks the same tree — split n//2 until <= 32, solve
// the left half, fold the right half with gemm(-1, b1, l21^T, alpha, b2) in
// kc segments (ascending fma chain from +0 per segment, unfused fold with
// beta = alpha on the first segment, 1 after), recurse on the right half with
// alpha = 1 — so every element sees the reference's operations in order.
constexpr int TS_ROWS = 64, TS_THREADS = 256, TS_LD = 129;

template <typename T>
struct TrsmSmall {
  T* sb;        // [TS_ROWS][TS_LD]  B rows of this CTA
  const T* sl;  // [128][TS_LD]      triangle
  int rows;
  int64_t kc;

  __device__ void base(int lo, int hi, double alpha) const {
    const int r = threadIdx.x;
    if (r >= rows) return;
    const int n = hi - lo;
    T x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = j < n ? sb[r * TS_LD + lo + j] : T(0);
    if (alpha != 1.0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = T(Ops<double>::mul(double(x[j]), alpha));
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < n) {
        T acc = x[j];
#pragma unroll
        for (int p = 0; p < j; ++p) acc = Ops<T>::sub(acc, Ops<T>::mul(x[p], sl[(lo + j) * TS_LD + lo + p]));
        x[j] = Ops<T>::div(acc, sl[(lo + j) * TS_LD + lo + j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < n) sb[r * TS_LD + lo + j] = x[j];
  }

  // b[:, mid:hi] = beta*b[:, mid:hi] - b[:, lo:mid] * l[mid:hi, lo:mid]^T,
  // one kc-segmented fma chain per element (gemm_scatter's arithmetic).
  // 16 x 16 threads, each a 4 x 4 register block: rows tr+16a, cols tc+16b.
  __device__ void fold(int lo, int mid, int hi, double beta) const {
    const int K = mid - lo;
    const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
    bool rok[4], cok[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) rok[a] = tr + 16 * a < rows;
#pragma unroll
    for (int b = 0; b < 4; ++b) cok[b] = mid + tc + 16 * b < hi;
    T c[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        c[a][b] = (rok[a] && cok[b]) ? sb[(tr + 16 * a) * TS_LD + mid + tc + 16 * b] : T(0);
    for (int k0 = 0, seg = 0; k0 < K; k0 += int(kc), ++seg) {
      const int k1 = (K - k0) < kc ? K : k0 + int(kc);
      double t[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) t[a][b] = 0.0;
      for (int p = lo + k0; p < lo + k1; ++p) {
        T bv[4], lv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) bv[a] = sb[((tr + 16 * a) & (TS_ROWS - 1)) * TS_LD + p];
#pragma unroll
        for (int b = 0; b < 4; ++b) lv[b] = sl[((mid + tc + 16 * b) & 127) * TS_LD + p];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if constexpr (sizeof(T) == 8)
              t[a][b] = __fma_rn(bv[a], lv[b], t[a][b]);
            else  // f32 storage, f32 acc: f32 products summed in f64 (engine/kernels.py:507-522)
              t[a][b] = __dadd_rn(t[a][b], double(__fmul_rn(bv[a], lv[b])));
          }
      }
      const double be = seg == 0 ? beta : 1.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if constexpr (sizeof(T) == 8) {
            double v = __dmul_rn(-1.0, t[a][b]);
            if (be != 0.0) v = __dadd_rn(__dmul_rn(be, c[a][b]), v);
            c[a][b] = v;
          } else {
            float v = __fmul_rn(-1.0f, float(t[a][b]));
            if (be != 0.0) v = __fadd_rn(__fmul_rn(float(be), c[a][b]), v);
            c[a][b] = v;
          }
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (rok[a] && cok[b]) sb[(tr + 16 * a) * TS_LD + mid + tc + 16 * b] = c[a][b];
  }

  // n <= 64: split once into two <= 32 bases
  __device__ void solve64(int lo, int hi, double alpha) const {
    const int n = hi - lo;
    if (n <= 32) {
      base(lo, hi, alpha);
      __syncthreads();
      return;
    }
    const int mid = lo + n / 2;
    base(lo, mid, alpha);
    __syncthreads();
    fold(lo, mid, hi, alpha);
    __syncthreads();
    base(mid, hi, 1.0);
    __syncthreads();
  }
  // n <= 128: the reference recursion (engine/trsm.py:51-68) unrolled by hand
  // (no device-side recursion, so no dynamic stack)
  __device__ void solve(int lo, int hi, double alpha) const {
    const int n = hi - lo;
    if (n <= 64) {
      solve64(lo, hi, alpha);
      return;
    }
    const int mid = lo + n / 2;
    solve64(lo, mid, alpha);
    fold(lo, mid, hi, alpha);
    __syncthreads();
    solve64(mid, hi, 1.0);
  }
};

template <typename T>
__global__ void __launch_bounds__(TS_THREADS) trsm_small_right_kernel(double alpha, const T* t, int64_t toff,
                                                                      int64_t trs, int64_t tcs, T* b, int64_t boff,
                                                                      int64_t brs, int64_t bcs, int64_t m, int n,
                                                                      int64_t kc, const int* abort_flag) {
  if (abort_flag != nullptr && *abort_flag >= 0) return;
  extern __shared__ __align__(16) unsigned char ts_smem[];
  T* sl = reinterpret_cast<T*>(ts_smem);
  T* sb = sl + 128 * TS_LD;
  const int64_t r0 = int64_t(blockIdx.x) * TS_ROWS;
  const int rows = int(m - r0 < TS_ROWS ? m - r0 : TS_ROWS);
  // Stage the triangle and this CTA's rows with asynchronous element copies
  // (hundreds in flight per thread instead of one dependent load at a time).
  // The strict upper part of the triangle is copied too but never read.
  const bool t_col_fast = tcs == 1;
  for (int e = threadIdx.x; e < n * n; e += TS_THREADS) {
    int j, p;
    if (t_col_fast) { j = e / n; p = e % n; } else { p = e / n; j = e % n; }
    if constexpr (sizeof(T) == 8)
      cp_async_8(&sl[j * TS_LD + p], &t[toff + j * trs + p * tcs], 8);
    else
      cp_async_4(&sl[j * TS_LD + p], &t[toff + j * trs + p * tcs], 4);
  }
  const bool col_fast = bcs == 1;
  for (int e = threadIdx.x; e < rows * n; e += TS_THREADS) {
    int r, c;
    if (col_fast) { r = e / n; c = e % n; } else { c = e / rows; r = e % rows; }
    if constexpr (sizeof(T) == 8)
      cp_async_8(&sb[r * TS_LD + c], &b[boff + (r0 + r) * brs + c * bcs], 8);
    else
      cp_async_4(&sb[r * TS_LD + c], &b[boff + (r0 + r) * brs + c * bcs], 4);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  TrsmSmall<T> ts{sb, sl, rows, kc};
  ts.solve(0, n, alpha);
  for (int e = threadIdx.x; e < rows * n; e += TS_THREADS) {
    int r, c;
    if (col_fast) { r = e / n; c = e % n; } else { c = e / rows; r = e % rows; }
    b[boff + (r0 + r) * brs + c * bcs] = sb[r * TS_LD + c];
  }
}

// ---------------------------------- fused TRSM subtree, 4 warps per 32 rows --
// Same recursion and per-element arithmetic as TrsmSmall, organised for
// latency.  A group of four warps owns 32 rows of X * L^T = B (rows are
// independent) and walks the tree with one named barrier per phase:
//  * bases: warp 0, one lane per row, the row's 32 accumulators in registers,
//    column-oriented (once x_p is final every later accumulator takes its
//    multiply-subtract: the reference's order per element), so the serial
//    chain is one division and one multiply-subtract per column;
//  * folds: the output columns in 8-wide chunks spread over the 4 warps; f64
//    on the tensor pipe (DMMA m8n8k4, 4 row tiles, k-slices zero-padded:
//    fma(0,0,t) = t, the kc-segment chain of the reference), f32 as one SIMT
//    chain per element (f32 products summed in f64).
// Rows live in shared memory as sx[c][33] per group; the triangle is shared
// by the CTA's groups.
constexpr int TW_LD = 132;  // triangle row stride: 16-byte aligned rows
constexpr int TW_XLD = 33;  // x column stride (padded)

template <typename T>
struct TrsmGroup {
  T* sx;        // [128][TW_XLD]: column c of the group's 32 rows
  const T* sl;  // [128][TW_LD] triangle
  int lane, gw, barid;
  int64_t kc;

  __device__ __forceinline__ T& x(int c) const { return sx[c * TW_XLD + lane]; }
  __device__ __forceinline__ T& xa(int c, int r) const { return sx[c * TW_XLD + r]; }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, 128;\n" ::"r"(barid) : "memory"); }

  // Division on the serial chain: with r = rcp.rn(b) computed off the chain,
  // q0 = a*r, e = fma(-b, q0, a), q = fma(e, r, q0) is RN(a/b) (Markstein)
  // whenever nothing over/underflows.  Every dividend and divisor is checked
  // to lie in a band where that holds (|x| in [2^-423, 2^423] for f64,
  // [2^-47, 2^47] for f32; zero dividends are fine); a base that met
  // anything else is recomputed with div.rn.
  __device__ __forceinline__ static int expo(T v) {
    if constexpr (sizeof(T) == 8)
      return (__double2hiint(v) >> 20) & 0x7ff;
    else
      return (__float_as_int(v) >> 23) & 0xff;
  }
  static constexpr int kLoExp = sizeof(T) == 8 ? 600 : 80;
  static constexpr int kHiExp = sizeof(T) == 8 ? 1446 : 174;
  static constexpr int kMidExp = sizeof(T) == 8 ? 1023 : 127;
  __device__ __forceinline__ static T rcp(T b) {
    if constexpr (sizeof(T) == 8)
      return __drcp_rn(b);
    else
      return __frcp_rn(b);
  }

  template <bool FULL>
  __device__ __forceinline__ void base_impl(int lo, int n, double alpha) const {
    const T* l = sl + lo * TW_LD + lo;
    // lane p takes the reciprocal of diagonal p; shuffles hand them out
    const T dl = (FULL || lane < n) ? l[lane * TW_LD + lane] : T(1);
    const T my_rc = rcp(dl);
    const int ed = expo(dl);
    bool safe = __all_sync(0xffffffffu, ed >= kLoExp && ed <= kHiExp);
    T rc[32];
#pragma unroll
    for (int p = 0; p < 32; ++p) rc[p] = __shfl_sync(0xffffffffu, my_rc, p);
    T acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = (FULL || j < n) ? x(lo + j) : T(0);
    if (alpha != 1.0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = T(Ops<double>::mul(double(acc[j]), alpha));
    }
    int emin = kMidExp, emax = kMidExp;
#pragma unroll
    for (int p = 0; p < 32; ++p) {
      if (FULL || p < n) {
        const T a = acc[p];
        const T q0 = Ops<T>::mul(a, rc[p]);
        const T xp = Ops<T>::fma_(Ops<T>::fma_(-l[p * TW_LD + p], q0, a), rc[p], q0);
        const int ea = a == T(0) ? kMidExp : expo(a);
        emin = min(emin, ea);
        emax = max(emax, ea);
        acc[p] = xp;
#pragma unroll
        for (int q = p + 1; q < 32; ++q)
          if (FULL || q < n) acc[q] = Ops<T>::sub(acc[q], Ops<T>::mul(xp, l[q * TW_LD + p]));
      }
    }
    safe = __all_sync(0xffffffffu, safe && emin >= kLoExp && emax <= kHiExp);
    if (safe) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (FULL || j < n) x(lo + j) = acc[j];
    } else {  // rare: exact division throughout, in place
      if (alpha != 1.0)
        for (int j = 0; j < n; ++j) x(lo + j) = T(Ops<double>::mul(double(x(lo + j)), alpha));
      for (int p = 0; p < n; ++p) {
        const T xp = Ops<T>::div(x(lo + p), l[p * TW_LD + p]);
        x(lo + p) = xp;
        for (int q = p + 1; q < n; ++q) x(lo + q) = Ops<T>::sub(x(lo + q), Ops<T>::mul(xp, l[q * TW_LD + p]));
      }
    }
  }

  __device__ __forceinline__ void base(int lo, int hi, double alpha) const {
    if (gw == 0) {
      if (hi - lo == 32)
        base_impl<true>(lo, 32, alpha);
      else
        base_impl<false>(lo, hi - lo, alpha);
    }
    sync();
  }

  // x[:, mid:hi] = beta*x[:, mid:hi] - x[:, lo:mid] * l[mid:hi, lo:mid]^T in kc segments
  __device__ __forceinline__ void fold(int lo, int mid, int hi, double beta) const {
    const int K = mid - lo;
    if constexpr (sizeof(T) == 8) {
      const int ar = lane >> 2, ak = lane & 3;
#pragma unroll 1
      for (int j0 = mid + 8 * gw; j0 < hi; j0 += 32) {
        double cv[4][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int col = j0 + 2 * ak + i;
            cv[mt][i] = col < hi ? xa(col, 8 * mt + ar) : 0.0;
          }
        const bool nok = j0 + ar < hi;
        const T* lrow = sl + ((j0 + ar) & 127) * TW_LD;
#pragma unroll 1
        for (int k0 = 0, seg = 0; k0 < K; k0 += int(kc), ++seg) {
          const int ps = lo + k0, pe = lo + ((K - k0) < kc ? K : k0 + int(kc));
          double d[4][2];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) d[mt][0] = d[mt][1] = 0.0;
#pragma unroll 2
          for (int p = ps; p < pe; p += 4) {
            const int pk = p + ak;
            const bool kok = pk < pe;
            const double bv = (kok && nok) ? lrow[pk] : 0.0;
            double av[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) av[mt] = kok ? xa(pk, 8 * mt + ar) : 0.0;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) dmma_8x8x4(d[mt][0], d[mt][1], av[mt], bv);
          }
          const double be = seg == 0 ? beta : 1.0;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              double v = __dmul_rn(-1.0, d[mt][i]);
              if (be != 0.0) v = __dadd_rn(__dmul_rn(be, cv[mt][i]), v);
              cv[mt][i] = v;
            }
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int col = j0 + 2 * ak + i;
            if (col < hi) xa(col, 8 * mt + ar) = T(cv[mt][i]);
          }
      }
    } else {
#pragma unroll 1
      for (int j0 = mid + 8 * gw; j0 < hi; j0 += 32) {
        T c[8];
        const T* lrow[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q] = j0 + q < hi ? x(j0 + q) : T(0);
          lrow[q] = sl + ((j0 + q) & 127) * TW_LD;
        }
#pragma unroll 1
        for (int k0 = 0, seg = 0; k0 < K; k0 += int(kc), ++seg) {
          const int p1 = lo + ((K - k0) < kc ? K : k0 + int(kc));
          double t[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) t[q] = 0.0;
#pragma unroll 4
          for (int p = lo + k0; p < p1; ++p) {
            const T xv = x(p);
#pragma unroll
            for (int q = 0; q < 8; ++q)  // f32 products summed in f64 (engine/kernels.py:507-522)
              t[q] = __dadd_rn(t[q], double(__fmul_rn(xv, lrow[q][p])));
          }
          const double be = seg == 0 ? beta : 1.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float v = __fmul_rn(-1.0f, float(t[q]));
            if (be != 0.0) v = __fadd_rn(__fmul_rn(float(be), c[q]), v);
            c[q] = v;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + q < hi) x(j0 + q) = c[q];
      }
    }
    sync();
  }

  // The recursion (n <= 128) flattened into at most 7 phases and walked by
  // one loop, so base and fold are each instantiated once (inlined four
  // times, the bases alone overflowed the instruction cache).
  __device__ __forceinline__ static int plan64(int lo, int hi, double alpha, int* kind, int* a, int* b, int* c,
                                               double* al, int k) {
    const int n = hi - lo;
    if (n <= 32) {
      kind[k] = 0, a[k] = lo, b[k] = hi, al[k] = alpha;
      return k + 1;
    }
    const int mid = lo + n / 2;
    kind[k] = 0, a[k] = lo, b[k] = mid, al[k] = alpha;
    kind[k + 1] = 1, a[k + 1] = lo, b[k + 1] = mid, c[k + 1] = hi, al[k + 1] = alpha;
    kind[k + 2] = 0, a[k + 2] = mid, b[k + 2] = hi, al[k + 2] = 1.0;
    return k + 3;
  }
  __device__ __forceinline__ void solve(int lo, int hi, double alpha) const {
    int kind[7], pa[7], pb[7], pc[7];
    double pal[7];
    int np;
    const int n = hi - lo;
    if (n <= 64) {
      np = plan64(lo, hi, alpha, kind, pa, pb, pc, pal, 0);
    } else {
      const int mid = lo + n / 2;
      np = plan64(lo, mid, alpha, kind, pa, pb, pc, pal, 0);
      kind[np] = 1, pa[np] = lo, pb[np] = mid, pc[np] = hi, pal[np] = alpha;
      np = plan64(mid, hi, 1.0, kind, pa, pb, pc, pal, np + 1);
    }
#pragma unroll 1
    for (int i = 0; i < np; ++i) {
      if (kind[i] == 0)
        base(pa[i], pb[i], pal[i]);
      else
        fold(pa[i], pb[i], pc[i], pal[i]);
    }
  }
};


// R groups (32 rows each) per CTA share the staged triangle
// The body of trsm_warp_right_kernel for CTA (row block) blk, staging in
// tw_smem; also run by potrf_diag_fused_kernel (R = 1)
template <typename T, int R>
__device__ __forceinline__ void trsm_warp_right_body(double alpha, const T* t, int64_t toff, int64_t trs, int64_t tcs,
                                                     T* b, int64_t boff, int64_t brs, int64_t bcs, int64_t m, int n,
                                                     int64_t kc, int64_t blk, unsigned char* tw_smem, bool trigger) {
  T* sl = reinterpret_cast<T*>(tw_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp >> 2, gw = warp & 3;
  constexpr int NW = 4 * R;
  T* sx = sl + 128 * TW_LD + grp * 128 * TW_XLD;
  // lower triangle (the only part read), whole CTA, coalesced along rows
  constexpr int VE = 16 / sizeof(T);
  const T* tb = t + toff;
  if (tcs == 1 && (reinterpret_cast<uintptr_t>(tb) % 16 == 0) && (trs % VE == 0)) {
    for (int j = warp; j < n; j += NW)
      for (int p = lane * VE; p <= j; p += 32 * VE) cp_async_16(&sl[j * TW_LD + p], &tb[j * trs + p], 16);
  } else if (tcs == 1) {
    for (int j = warp; j < n; j += NW)
      for (int p = lane; p <= j; p += 32) {
        if constexpr (sizeof(T) == 8)
          cp_async_8(&sl[j * TW_LD + p], &tb[j * trs + p], 8);
        else
          cp_async_4(&sl[j * TW_LD + p], &tb[j * trs + p], 4);
      }
  } else {
    for (int p = warp; p < n; p += NW)
      for (int j = p + lane; j < n; j += 32) {
        if constexpr (sizeof(T) == 8)
          cp_async_8(&sl[j * TW_LD + p], &tb[j * trs + p * tcs], 8);
        else
          cp_async_4(&sl[j * TW_LD + p], &tb[j * trs + p * tcs], 4);
      }
  }
  // the group's 32 rows, zero-filled past m; lanes run along a row (coalesced)
  const int64_t r0 = (blk * R + grp) * 32;
  const int rows = int(m - r0 < 32 ? (m - r0 > 0 ? m - r0 : 0) : 32);
  if (bcs == 1) {
    for (int r = gw; r < 32; r += 4) {
      const bool ok = r < rows;
      for (int c = lane; c < n; c += 32) {
        const T* src = ok ? &b[boff + (r0 + r) * brs + c] : b;
        if constexpr (sizeof(T) == 8)
          cp_async_8(&sx[c * TW_XLD + r], src, ok ? 8 : 0);
        else
          cp_async_4(&sx[c * TW_XLD + r], src, ok ? 4 : 0);
      }
    }
  } else {
    const bool ok = lane < rows;
    for (int c = gw; c < n; c += 4) {
      const T* src = ok ? &b[boff + (r0 + lane) * brs + c * bcs] : b;
      if constexpr (sizeof(T) == 8)
        cp_async_8(&sx[c * TW_XLD + lane], src, ok ? 8 : 0);
      else
        cp_async_4(&sx[c * TW_XLD + lane], src, ok ? 4 : 0);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (rows > 0) {  // uniform per group
    TrsmGroup<T> tg{sx, sl, lane, gw, 1 + grp, kc};
    tg.solve(0, n, alpha);
    if (trigger) pdl_trigger();
    if (bcs == 1) {
      for (int r = gw; r < rows; r += 4)
        for (int c = lane; c < n; c += 32) b[boff + (r0 + r) * brs + c] = sx[c * TW_XLD + r];
    } else if (lane < rows) {
      for (int c = gw; c < n; c += 4) b[boff + (r0 + lane) * brs + c * bcs] = sx[c * TW_XLD + lane];
    }
  }
}

// X_dd L_dd^T = X_dd for every 128-wide diagonal tile d of an n x n lower L
// (blockIdx.y = d, blockIdx.x = 32-row chunk): the leaves of the doubling
// triangular inverse (tri_inverse_t_d); X holds the identity on entry
__global__ void __launch_bounds__(128) trsm_diag_tiles_kernel(const double* l, int64_t ldl, double* x, int64_t ldx,
                                                              int64_t n, int64_t kc) {
  extern __shared__ __align__(16) unsigned char tw_smem[];
  const int64_t d0 = int64_t(blockIdx.y) * 128;
  const int nb = int(n - d0 < 128 ? n - d0 : 128);
  if (int64_t(blockIdx.x) * 32 >= nb) return;
  trsm_warp_right_body<double, 1>(1.0, l, d0 * (ldl + 1), ldl, 1, x, d0 * (ldx + 1), ldx, 1, nb, nb, kc,
                                  int64_t(blockIdx.x), tw_smem, false);
}

template <typename T, int R>
__global__ void __launch_bounds__(128 * R) trsm_warp_right_kernel(double alpha, const T* t, int64_t toff, int64_t trs,
                                                                  int64_t tcs, T* b, int64_t boff, int64_t brs,
                                                                  int64_t bcs, int64_t m, int n, int64_t kc,
                                                                  const int* abort_flag) {
  pdl_wait();
  if (abort_flag != nullptr && *abort_flag >= 0) return;
  extern __shared__ __align__(16) unsigned char tw_smem[];
  trsm_warp_right_body<T, R>(alpha, t, toff, trs, tcs, b, boff, brs, bcs, m, n, kc, int64_t(blockIdx.x), tw_smem,
                             true);
}

// ------------------------------------------------ blocked variant-3 leaf --
// Variant 3 (right-looking, factor/cholesky.py:74-89) for n <= 128 by 32-wide
// column blocks, every element still receiving the reference's operations
// in the reference's order (a(i,j) -= a(i,k)*a(j,k) for ascending k, unfused,
// then its sqrt or division):
//  (a) warp 0 factors the diagonal block in registers, one lane per row,
//      four columns per loop trip through a sliding register window.  The
//      pivot chain is branch-free: sqrt from an rsqrt seed + two Newton steps
//      + a residual correction, the reciprocal of the rounded root seeded by
//      the same y, and Markstein division (q0 = a r, q = q0 + (a - b q0) r).
//      Every root and quotient is then *verified* from its exact fma
//      residual (|d - s^2| < s ulp(s), |a - b q| < b ulp(q)/2, inside an
//      exponent band), so a result is only kept when it provably equals
//      sqrt.rn / div.rn; anything else (never seen in 5e9 probes,
//      tools/sqrt_probe.cu) redoes the whole leaf with the exact kernel.
//      The next pivot's own update is taken first; the column reaches the
//      other rows by shuffles;
//  (b) the rows below, 32 per warp, solve against the finished block the same
//      way (quotients verified);
//  (c) the trailing triangle takes the block's rank-1 updates, 4x4 register
//      tiles over the CTA.
// A failing pivot, like an unverified result, sends the leaf to the exact
// column-parallel algorithm (leaf_v3), which stops where the reference stops
// and leaves its partial state.  128 threads, LD = 129.
constexpr int LV4_LD = 129;
#ifdef LV4_PROF  // phase clocks for tools/leaf_probe2.cu
__device__ long long g_lv4_prof[64];
#define LV4_MARK(i) \
  if (threadIdx.x == 0) g_lv4_prof[i] += clock64();
#else
#define LV4_MARK(i)
#endif

template <typename T>
struct LeafMath {  // f32 storage: the exact (branchy) operations, always "verified"
  static __device__ __forceinline__ T sqrt_y(T d, T& y) {
    y = T(0);
    return Ops<T>::sqrt_(d);
  }
  static __device__ __forceinline__ T rcp(T b, T) { return T(0); }
  static __device__ __forceinline__ T div(T a, T b, T) { return Ops<T>::div(a, b); }
  static __device__ __forceinline__ bool sqrt_ok(T, T) { return true; }
  static __device__ __forceinline__ bool div_ok(T, T, T) { return true; }
};
template <>
struct LeafMath<double> {
  static __device__ __forceinline__ int ex(double v) { return (__double2hiint(v) >> 20) & 0x7ff; }
  static __device__ __forceinline__ bool in_band(double v) {
    const int e = ex(v);
    return (e >= 223) & (e <= 1823);  // |v| in [2^-800, 2^800]
  }
  static __device__ __forceinline__ double sqrt_y(double d, double& yo) {
    // one Newton step on the rsqrt seed is enough: the residual correction
    // below squares the error again (0 mismatches against sqrt.rn and, with y
    // as the Markstein seed, against div.rn in 1.24e9 probes,
    // tools/sqrt_probe1.cu); every root and quotient is verified anyway
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double h = 0.5 * y;
    double r = __fma_rn(-d * y, h, 0.5);
    y = __fma_rn(y, r, y);
    const double s = d * y;
    h = 0.5 * y;
    yo = y;
    return __fma_rn(__fma_rn(-s, s, d), h, s);
  }
  static __device__ __forceinline__ double rcp(double b, double y) {
    double e = __fma_rn(-b, y, 1.0);
    y = __fma_rn(y, e, y);
    e = __fma_rn(-b, y, 1.0);
    return __fma_rn(y, e, y);
  }
  static __device__ __forceinline__ double div(double a, double b, double r) {
    const double q0 = __dmul_rn(a, r);
    return __fma_rn(__fma_rn(-b, q0, a), r, q0);
  }
  // s == sqrt.rn(d): the exact residual sits strictly inside the rounding
  // interval (bitwise & / | throughout: no short-circuit branches).  For s
  // not a power of two, s = RN(sqrt d) iff -s u < d - s^2 <= s u (u = ulp s;
  // (s -+ u/2)^2 = s^2 -+ s u + u^2/4 and the representable neighbours of
  // +-s u are u^2 apart).  The test keeps a 2^-20 relative margin inside that
  // interval: with the former 2^-10 margin about 0.1 % of correctly rounded
  // roots were rejected, i.e. ~13 % of 128-wide leaves took the exact redo
  // (340 us instead of 70 us in the launch list).
  static __device__ __forceinline__ bool sqrt_ok(double d, double s) {
    const long long sb = __double_as_longlong(s);
    const double ulp = __longlong_as_double((sb & 0x7ff0000000000000LL) - (52LL << 52));
    const double rem = __fma_rn(-s, s, d);
    return in_band(d) & (fabs(rem) < s * ulp * 0.99999904632568359375) & ((sb & 0x000fffffffffffffLL) != 0);
  }
  // q == div.rn(a, b) for b > 0: |a - b q| < b ulp(q) / 2, q not a power of two
  // (a == 0 gives q == 0 exactly)
  static __device__ __forceinline__ bool div_ok(double a, double b, double q) {
    const long long qb = __double_as_longlong(q);
    const double half_ulp = __longlong_as_double((qb & 0x7ff0000000000000LL) - (53LL << 52));
    const double rem = __fma_rn(-b, q, a);
    const bool nonzero_ok = in_band(a) & in_band(b) & in_band(q) & (fabs(rem) < b * half_ulp) &
                            ((qb & 0x000fffffffffffffLL) != 0);
    return (a == 0.0) ? (q == 0.0) : nonzero_ok;
  }
};

// The blocked leaf on one CTA of 128 threads (the body of
// potrf_leaf_blocked_kernel, also run by potrf_diag_fused_kernel): factors
// the n x n tile at g + off in place, staging it in A (128 x LV4_LD of
// dynamic shared memory); returns the failing pivot (-1: none).
template <typename T>
__device__ __forceinline__ int leaf_blocked_body(T* g, int64_t off, int n, int64_t rs, int64_t cs, int pipe_flag,
                                                 T* A, bool trigger) {
  __shared__ T s_rc[128];
  __shared__ __align__(16) T s_cb[4 * 128];  // per warp: two 64-entry column buffers
  __shared__ int s_fail;
  __shared__ int s_unsafe;
  __shared__ T s_d;
  using LM = LeafMath<T>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto stage_in = [&]() {
    if (cs == 1) {
      for (int i = warp; i < n; i += 4)
        for (int j = lane; j <= i; j += 32) {
          if constexpr (sizeof(T) == 8)
            cp_async_8(&A[i * LV4_LD + j], &g[off + i * rs + j], 8);
          else
            cp_async_4(&A[i * LV4_LD + j], &g[off + i * rs + j], 4);
        }
    } else {
      for (int j = warp; j < n; j += 4)
        for (int i = j + lane; i < n; i += 32) {
          if constexpr (sizeof(T) == 8)
            cp_async_8(&A[i * LV4_LD + j], &g[off + i * rs + j * cs], 8);
          else
            cp_async_4(&A[i * LV4_LD + j], &g[off + i * rs + j * cs], 4);
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
  };
  stage_in();
  if (tid == 0) {
    s_fail = -1;
    s_unsafe = 0;
  }
  __syncthreads();
  LV4_MARK(0)
  int bad = -1;
  // block (k0, kend columns)'s rank-kend update of the 4x4 tiles tt in
  // [tt0, tt1) of the trailing triangle below k1, over threads idx of nthr
  auto trail = [&](int k0, int kend, int k1, int tt0, int tt1, int idx, int nthr) {
    const int m = n - k1;
    if (m <= 0 || kend <= 0) return;
    const int tiles = (m + 3) / 4;
    const int ntile = tiles * (tiles + 1) / 2;
    for (int tt = tt0 + idx; tt < ntile && tt < tt1; tt += nthr) {
      int ti = int((sqrtf(8.f * float(tt) + 1.f) - 1.f) * 0.5f);
      while (ti * (ti + 1) / 2 > tt) --ti;
      while ((ti + 1) * (ti + 2) / 2 <= tt) ++ti;
      const int tj = tt - ti * (ti + 1) / 2;
      const int i0 = k1 + 4 * ti, j0 = k1 + 4 * tj;
      T c[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          c[a][b] = (i0 + a < n && j0 + b <= i0 + a) ? A[(i0 + a) * LV4_LD + j0 + b] : T(0);
#pragma unroll 4
      for (int p = k0; p < k0 + kend; ++p) {
        T li[4], lj[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) li[a] = A[((i0 + a) & 127) * LV4_LD + p];
#pragma unroll
        for (int b = 0; b < 4; ++b) lj[b] = A[((j0 + b) & 127) * LV4_LD + p];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) c[a][b] = Ops<T>::sub(c[a][b], Ops<T>::mul(li[a], lj[b]));
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (i0 + a < n && j0 + b <= i0 + a) A[(i0 + a) * LV4_LD + j0 + b] = c[a][b];
    }
  };
  const bool pipe = pipe_flag != 0;
  int pk0 = -1, pkend = 0, pk1 = 0;  // the block whose trailing update (beyond the next diagonal triangle) is pending
#pragma unroll 1
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int bw = n - k0 < 32 ? n - k0 : 32;
    const int k1 = k0 + bw;
    // (a) diagonal block: acc[j] holds column p0 + j of row k0 + lane.  The
    // four-column body is one basic block (no barrier, no data-dependent
    // branch: pivot failures and unverified results only raise the redo
    // flag), so the scheduler overlaps column p+1's pivot chain with column
    // p's shuffle-fed updates.
    // Every warp runs it (same values); only warp 0 stores: with no
    // warp-dependent branch around it the shuffles need no divergence
    // checks, which would otherwise split the body into basic blocks.
    if (pipe && warp > 0) {
      if (pk0 >= 0) trail(pk0, pkend, pk1, 36, 1 << 30, tid - 32, 96);
    } else {
      const bool w0 = warp == 0;
      const int i = lane;
      T acc[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] = (q <= i && i < bw) ? A[(k0 + i) * LV4_LD + k0 + q] : T(0);
      bool unsafe = false;
      T d = __shfl_sync(0xffffffffu, acc[0], 0);
      // fully unrolled over the block's 8 four-column trips (a warp-uniform
      // guard per trip): window positions j >= 32 - p0 are past the block,
      // so the updates and broadcast reads stop there — half the multiply-
      // subtracts of a fixed 32-wide window
#pragma unroll
      for (int p0 = 0; p0 < 32; p0 += 4) {
        if (p0 >= bw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = p0 + u;
          const bool live = p < bw;
          const T dcur = d;
          T y;
          const T lpp = LM::sqrt_y(dcur, y);
          const T r = LM::rcp(lpp, y);  // for the panel solve (s_rc), off the chain
          const T a = acc[u];
          // the chain's quotient seeds Markstein with y ~ 1/lpp itself (a few
          // ulps): one rcp refinement less between consecutive pivots; the
          // quotient is still verified exactly below (div_ok)
          const T qv = LM::div(a, lpp, y);
          const T l = i == p ? lpp : (i > p ? qv : a);
          // next pivot first: lane p+1's own update by column p
          const T nd = Ops<T>::sub(acc[u + 1], Ops<T>::mul(l, l));
          d = __shfl_sync(0xffffffffu, nd, (p + 1) & 31);
          unsafe |= live & (!(dcur > T(0)) | !LM::sqrt_ok(dcur, lpp) |
                            ((i > p) & (i < bw) & !LM::div_ok(a, lpp, qv)));
          acc[u] = l;
          if (w0 && live && i >= p && i < bw) A[(k0 + i) * LV4_LD + k0 + p] = l;
          if (w0 && live && i == p) s_rc[k0 + p] = r;
          // column broadcast through shared memory (double-buffered by column
          // parity: one warp barrier per column); cb[p0 + j] is l(p0 + j, p)
          T* cb = s_cb + (u & 1) * 64 + warp * 128;
          cb[i] = l;
          __syncwarp();
          T lv[32];
          if constexpr (sizeof(T) == 8) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
              if (2 * m < 32 - p0) {
                const double2 t2 = reinterpret_cast<const double2*>(cb + p0)[m];
                lv[2 * m] = t2.x;
                lv[2 * m + 1] = t2.y;
              }
            }
          } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              if (4 * m < 32 - p0) {
                const float4 t4 = reinterpret_cast<const float4*>(cb + p0)[m];
                lv[4 * m] = t4.x;
                lv[4 * m + 1] = t4.y;
                lv[4 * m + 2] = t4.z;
                lv[4 * m + 3] = t4.w;
              }
            }
          }
#pragma unroll
          for (int j = u + 1; j < 32 - p0; ++j) acc[j] = Ops<T>::sub(acc[j], Ops<T>::mul(l, lv[j]));
        }
#pragma unroll
        for (int j = 0; j < 28; ++j) acc[j] = acc[j + 4];
        acc[28] = acc[29] = acc[30] = acc[31] = T(0);
      }
      if (__any_sync(0xffffffffu, unsafe) && w0 && lane == 0) s_unsafe = 1;
    }
    __syncthreads();
    LV4_MARK(1 + 3 * (k0 >> 5))
    const int kend = bw;
    // (b) rows below the block: X * L11^T = A21, lane per row, same window
#pragma unroll 1
    for (int r0 = k1 + 32 * warp; r0 < n; r0 += 128) {
      const int r = r0 + lane;
      const bool ok = r < n;
      const T* l = A + k0 * LV4_LD + k0;
      T acc[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] = (ok && q < bw) ? A[r * LV4_LD + k0 + q] : T(0);
      bool unsafe = false;
#pragma unroll
      for (int q0 = 0; q0 < 32; q0 += 4) {  // unrolled like (a): updates stop at the block's edge
        if (q0 >= bw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u;
          const bool live = q < bw;
          const int qq = q & 31;
          const T dq = l[qq * LV4_LD + qq], rq = s_rc[k0 + qq];
          const T a = acc[u];
          const T xq = LM::div(a, dq, rq);
          unsafe |= live & ok & !LM::div_ok(a, dq, xq);
          acc[u] = xq;
          if (live && ok) A[r * LV4_LD + k0 + q] = xq;
#pragma unroll
          for (int j = u + 1; j < 32 - q0; ++j)
            acc[j] = Ops<T>::sub(acc[j], Ops<T>::mul(xq, l[((q + j - u) & 31) * LV4_LD + qq]));
        }
#pragma unroll
        for (int j = 0; j < 28; ++j) acc[j] = acc[j + 4];
        acc[28] = acc[29] = acc[30] = acc[31] = T(0);
      }
      if (__any_sync(0xffffffffu, unsafe) && lane == 0) s_unsafe = 1;
    }
    __syncthreads();
    LV4_MARK(2 + 3 * (k0 >> 5))
    // (c) trailing triangle k1 <= j <= i < n: the block's first kend rank-1
    // updates.  Pipelined: only the next diagonal block's triangle (tile rows
    // 0..7) now; warps 1-3 apply the rest in the next trip's phase A while
    // warp 0 runs the next block's chain (disjoint elements, and every
    // element still takes the blocks' updates in block order)
    trail(k0, kend, k1, 0, pipe ? 36 : (1 << 30), tid, 128);
    __syncthreads();
    LV4_MARK(3 + 3 * (k0 >> 5))
    pk0 = k0;
    pkend = kend;
    pk1 = k1;
  }
  if (s_unsafe) {  // a pivot failed, or a root or quotient was not provably sqrt.rn / div.rn: redo exactly
    __syncthreads();
    stage_in();
    if (tid == 0) s_fail = -1;
    __syncthreads();
    bad = leaf_v3<T, 128>(Mat<T>{A, LV4_LD, 1}, n, &s_fail, &s_d);
    __syncthreads();
  }
  if (trigger) pdl_trigger();  // the next kernel of the chain may launch (it waits for this one's completion)
  if (cs == 1) {
    for (int i = warp; i < n; i += 4)
      for (int j = lane; j <= i; j += 32) g[off + i * rs + j] = A[i * LV4_LD + j];
  } else {
    for (int j = warp; j < n; j += 4)
      for (int i = j + lane; i < n; i += 32) g[off + i * rs + j * cs] = A[i * LV4_LD + j];
  }
  return bad;
}

template <typename T>
__global__ void __launch_bounds__(128) potrf_leaf_blocked_kernel(T* g, int64_t off, int n, int64_t rs, int64_t cs,
                                                                 int64_t base_index, int* d_info, int pipe_flag) {
  pdl_wait();
  if (d_info != nullptr && *d_info >= 0) return;
  extern __shared__ __align__(16) unsigned char leaf_b_smem[];
  const int bad = leaf_blocked_body<T>(g, off, n, rs, cs, pipe_flag, reinterpret_cast<T*>(leaf_b_smem), true);
  if (threadIdx.x == 0 && bad >= 0 && d_info != nullptr) *d_info = int(base_index + bad);
}

// --------------------------------------------- fused diagonal-block factor --
// One launch for a whole diagonal block of order n <= 2048 factored by the
// tree level {variant 3, bs 128, kc >= 128} over the unblocked3 leaf — the
// bench tree's child, which otherwise costs ~45 launches (16 leaves, 15
// TRSMs, 15 trailing GEMMTs) whose latencies form the panel chain.  Same
// operations per element as that launch sequence, hence the same bits:
//   L(c)       the leaf of tile (c, c)            leaf_blocked_body
//   T(c, r)    rows 32r.. of the tile column      trsm_warp_right_body
//              below it, solved against L(c)
//   S(j, x, u) 64 x 64 unit u of tile column x:   one ascending fma chain over
//              C -= L(:, j) L(:, j)^T             the step's 128 k (one kc
//                                                 segment from +0) and the
//                                                 unfused fold c + (-1 * t)
// Every element takes its step updates in step order, as in the sequence.
// Persistent CTAs claim tasks by ticket in a topological order — round c =
// L(c), S(0..c-1, c+1, *), T(c, *), S(c, c+1, *) — and wait (acquire
// spins) only for tasks with smaller tickets, which are held by running
// CTAs: no co-residency is needed and any grid size works.  While one CTA
// runs the leaf chain, the others apply the older steps' updates to the next
// tile column (the lookahead of the launch sequence, inside one kernel).
// A pivot failure at L(c) stops steps >= c; the updates of steps < c still
// complete — the sequence's partial state.
constexpr int FD_B = 128;    // inner block
constexpr int FD_ULD = 132;  // row stride of a staged 64 x 128 unit operand
constexpr int FD_MAXN = 2048;
constexpr size_t FD_SMEM_UPDATE = (size_t(2) * 64 * FD_ULD + 64 * 64) * sizeof(double);
constexpr size_t FD_SMEM_TRSM = (size_t(128) * TW_LD + size_t(128) * TW_XLD) * sizeof(double);
constexpr size_t FD_SMEM = FD_SMEM_UPDATE > FD_SMEM_TRSM ? FD_SMEM_UPDATE : FD_SMEM_TRSM;
static_assert(size_t(128) * LV4_LD * sizeof(double) <= FD_SMEM, "leaf staging");

struct FdCounters {  // zeroed before the launch
  unsigned long long prof[12];  // per task kind (leaf, trsm, update): tasks, wait cycles, run cycles; update phases
  int ticket, fail1, err, pad;
  int leaf_done[FD_MAXN / FD_B], tdone[FD_MAXN / FD_B];
  int colfinal[FD_MAXN / FD_B];  // 1 once tile column c is final (leaf and every TRSM chunk): stream waits watch it
  int tchunk[FD_MAXN / FD_B][FD_MAXN / 32];  // 1 once TRSM chunk r of step c is solved
  int ucnt[(FD_MAXN / 64) * (FD_MAXN / 64 + 1) / 2];
};

__device__ __forceinline__ int fd_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// thread 0: wait until *p >= v.  Bounded: a wait past ~4 s (2^33 cycles) can
// only be a schedule bug — the kernel traps (a loud launch failure) rather
// than hang the GPU or return unfinished columns.
__device__ __forceinline__ void fd_wait(const int* p, int v, int* err) {
  if (fd_acquire(p) >= v) return;
  const long long t0 = clock64();
  while (fd_acquire(p) < v) {
    __nanosleep(64);
    if (clock64() - t0 > (1LL << 33)) {
      atomicExch(err, 1);
      printf("potrf_diag_fused_kernel: dependency wait timed out (block %d)\n", int(blockIdx.x));
      __trap();
    }
  }
}
// after the CTA's writes: __syncthreads, then thread 0 releases; returns the old count
__device__ __forceinline__ int fd_release_add(int* p) {
  __threadfence();
  return atomicAdd(p, 1);
}
// tile column c is final: the flag a stream memory wait polls (after the fence,
// every write of the column — fenced by its own task before its count — is in L2)
__device__ __forceinline__ void fd_publish(int* flag) {
  __threadfence();
  atomicExch(flag, 1);
}

struct FdShape {
  int n, T, NS;
  __device__ int units(int x) const { return 2 * x + 1 < NS ? 2 * NS - 4 * x - 1 : NS - 2 * x; }
  __device__ int chunks(int c) const { return (c + 1) * FD_B < n ? (n - (c + 1) * FD_B + 31) / 32 : 0; }
  __device__ int round_size(int c) const {
    return 1 + chunks(c) + (c + 1 < T ? (c + 1) * units(c + 1) : 0);
  }
  // unit u of tile column x -> 64-row block I, 64-column block J: the
  // diagonal tile's (up to) three units first, then row pairs below
  __device__ void unit(int x, int u, int& I, int& J) const {
    const int J0 = 2 * x;
    if (2 * x + 1 >= NS) {
      I = J0 + u, J = J0;
    } else if (u < 3) {
      I = J0 + (u > 0), J = J0 + (u == 2);
    } else {
      I = J0 + 2 + (u - 3) / 2, J = J0 + (u - 3) % 2;
    }
  }
};

// C(64 x 64 unit at rows 64I, cols 64J) -= P_I P_J^T, P = the 128 columns of
// step j; lower part only on a diagonal unit.  Operands staged row-major at
// stride FD_ULD = 132 doubles: rows stay 16-byte aligned for the copies and
// the DMMA fragment loads (8 rows x 4 k per half-warp pair) are conflict free.
__device__ __forceinline__ void fd_update_unit(double* g, int64_t off, int64_t ld, int n, int j, int I, int J,
                                               double* sm, unsigned long long* prof) {
  const int tid = threadIdx.x;
  const long long c0 = clock64();
  const int i0 = I * 64, j0 = J * 64, p0 = j * FD_B;
  const int mi = n - i0 < 64 ? n - i0 : 64, mj = n - j0 < 64 ? n - j0 : 64;
  double* As = sm;
  double* Bs = sm + 64 * FD_ULD;
  double* Cs = sm + 2 * 64 * FD_ULD;  // 64 x 64, row-major
  // staged with cp.async in two groups — the operands' k < 64 halves, then
  // their k >= 64 halves and the C unit — so the second group lands under
  // the first half's DMMAs; rows past the edge zero-filled.  The L1 holds
  // nothing stale: the task's acquire (ld.acquire.gpu) invalidated it.
  // 16-byte copies when every row start is 16-byte aligned (even ld and off).
  const bool v16 = ((off | ld) & 1) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0;
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    if (v16) {
      for (int e = tid; e < 64 * 32; e += 128) {  // (row, k pair)
        const int r = e >> 5, p = half * 64 + 2 * (e & 31);
        cp_async_16(&As[r * FD_ULD + p], r < mi ? &g[off + int64_t(i0 + r) * ld + p0 + p] : g, r < mi ? 16 : 0);
        cp_async_16(&Bs[r * FD_ULD + p], r < mj ? &g[off + int64_t(j0 + r) * ld + p0 + p] : g, r < mj ? 16 : 0);
      }
    } else {
      for (int e = tid; e < 64 * 64; e += 128) {
        const int r = e >> 6, p = half * 64 + (e & 63);
        cp_async_8(&As[r * FD_ULD + p], r < mi ? &g[off + int64_t(i0 + r) * ld + p0 + p] : g, r < mi ? 8 : 0);
        cp_async_8(&Bs[r * FD_ULD + p], r < mj ? &g[off + int64_t(j0 + r) * ld + p0 + p] : g, r < mj ? 8 : 0);
      }
    }
    if (half == 1) {
      for (int e = tid; e < 64 * 64; e += 128) {
        const int r = e >> 6, cc = e & 63;
        const bool ok = r < mi && cc < mj;
        cp_async_8(&Cs[e], ok ? &g[off + int64_t(i0 + r) * ld + j0 + cc] : g, ok ? 8 : 0);
      }
    }
    cp_async_commit();
  }
  cp_async_wait<1>();
  __syncthreads();
  const long long c1 = clock64();
  // warp w: the 32 x 32 block at rows 32 (w & 1), cols 32 (w >> 1) as 4 x 4
  // DMMA m8n8k4 tiles (d = a b + d is the ascending fma chain); lane holds
  // A[8m + lane / 4][k + lane % 4], B[k + lane % 4][8nn + lane / 4] and
  // C[8m + lane / 4][8nn + 2 (lane % 4) + e]
  const int warp = tid >> 5, lane = tid & 31;
  const int rb = 32 * (warp & 1), cb = 32 * (warp >> 1), lr = lane >> 2, lk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) acc[m][nn][0] = acc[m][nn][1] = 0.0;
#pragma unroll 2
  for (int k = 0; k < 128; k += 4) {
    if (k == 64) {  // the second half of the operands
      cp_async_wait<0>();
      __syncthreads();
    }
    const double* ak = As + (rb + lr) * FD_ULD + k + lk;
    const double* bk = Bs + (cb + lr) * FD_ULD + k + lk;
    double av[4], bv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) av[m] = ak[8 * m * FD_ULD];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) bv[nn] = bk[8 * nn * FD_ULD];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) dmma_8x8x4(acc[m][nn][0], acc[m][nn][1], av[m], bv[nn]);
  }
  const long long c2 = clock64();
  // fold from the staged C: beta*c + alpha*t with beta = 1, alpha = -1
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int il = rb + 8 * m + lr, jl = cb + 8 * nn + 2 * lk + e;
        if (il < mi && jl < mj && (I != J || il >= jl))
          g[off + int64_t(i0 + il) * ld + j0 + jl] = __dadd_rn(Cs[il * 64 + jl], -acc[m][nn][e]);
      }
  if (tid == 0) {
    atomicAdd(&prof[9], (unsigned long long)(c1 - c0));
    atomicAdd(&prof[10], (unsigned long long)(c2 - c1));
    atomicAdd(&prof[11], (unsigned long long)(clock64() - c2));
  }
}

__global__ void __launch_bounds__(128) potrf_diag_fused_kernel(double* g, int64_t off, int n, int64_t ld, int64_t kc,
                                                               int64_t base_index, int* d_info, int pipe_flag,
                                                               FdCounters* ctl) {
  const int ncol = (n + FD_B - 1) / FD_B;
  if (d_info != nullptr && *d_info >= 0) {  // an earlier failure: nothing to do, but every
    if (threadIdx.x < ncol) atomicExch(&ctl->colfinal[threadIdx.x], 1);  // column flag is
    return;                                                                // awaited (fused_diag 2)
  }
  extern __shared__ __align__(16) unsigned char fd_smem[];
  __shared__ int s_task, s_skip;
  const int tid = threadIdx.x;
  const FdShape sh{n, (n + FD_B - 1) / FD_B, (n + 63) / 64};
  int total = 0;
  for (int c = 0; c < sh.T; ++c) total += sh.round_size(c);
  int* err = &ctl->err;
  auto ucnt = [&](int I, int J) { return &ctl->ucnt[I * (I + 1) / 2 + J]; };
  // skip a task of step j once a leaf at step <= j has failed
  auto decide_skip = [&](int j) {
    if (tid == 0) {
      const int f = fd_acquire(&ctl->fail1);
      s_skip = f != 0 && f - 1 <= j;
    }
    __syncthreads();
    return s_skip != 0;
  };
  for (;;) {
    if (tid == 0) s_task = atomicAdd(&ctl->ticket, 1);
    __syncthreads();
    int q = s_task;
    __syncthreads();
    if (q >= total) break;
    int c = 0;
    while (q >= sh.round_size(c)) q -= sh.round_size(c++);
    const int U = c + 1 < sh.T ? sh.units(c + 1) : 0;
    const int R = sh.chunks(c);
    const long long t_claim = clock64();
    long long t_ready = 0;
    auto prof = [&](int kind) {  // thread 0, after the task
      if (tid == 0) {
        atomicAdd(&ctl->prof[3 * kind], 1ull);
        atomicAdd(&ctl->prof[3 * kind + 1], (unsigned long long)(t_ready - t_claim));
        atomicAdd(&ctl->prof[3 * kind + 2], (unsigned long long)(clock64() - t_ready));
      }
    };
    if (q == 0) {  // L(c)
      if (tid == 0) {
        const int J0 = 2 * c;
        fd_wait(ucnt(J0, J0), c, err);
        if (J0 + 1 < sh.NS) {
          fd_wait(ucnt(J0 + 1, J0), c, err);
          fd_wait(ucnt(J0 + 1, J0 + 1), c, err);
        }
      }
      __syncthreads();
      t_ready = clock64();
      if (!decide_skip(c)) {
        const int kb = n - c * FD_B < FD_B ? n - c * FD_B : FD_B;
        const int bad = leaf_blocked_body<double>(g, off + int64_t(c) * FD_B * (ld + 1), kb, ld, 1, pipe_flag,
                                                  reinterpret_cast<double*>(fd_smem), false);
        if (tid == 0 && bad >= 0) {
          ctl->fail1 = c + 1;
          if (d_info != nullptr) *d_info = int(base_index + int64_t(c) * FD_B + bad);
        }
      }
      __syncthreads();
      if (tid == 0) {
        fd_release_add(&ctl->leaf_done[c]);
        if (R == 0) fd_publish(&ctl->colfinal[c]);  // the last tile column: no TRSM chunks
      }
      prof(0);
      continue;
    }
    q -= 1;
    int j = -1, x = c + 1, u = 0, r = -1;
    if (q < c * U) {
      j = q / U, u = q % U;
    } else if ((q -= c * U) < R) {
      r = q;
    } else {
      j = c, u = q - R;
    }
    if (r >= 0) {  // T(c, r)
      const int row0 = (c + 1) * FD_B + 32 * r;
      if (tid == 0) {
        fd_wait(&ctl->leaf_done[c], 1, err);
        const int I = row0 / 64;
        fd_wait(ucnt(I, 2 * c), c, err);
        if (2 * c + 1 < sh.NS) fd_wait(ucnt(I, 2 * c + 1), c, err);
      }
      __syncthreads();
      t_ready = clock64();
      if (!decide_skip(c)) {
        const int64_t toff = off + int64_t(c) * FD_B * (ld + 1);
        trsm_warp_right_body<double, 1>(1.0, g, toff, ld, 1, g, toff + int64_t(FD_B) * ld, ld, 1,
                                        int64_t(n - (c + 1) * FD_B), FD_B, kc, int64_t(r), fd_smem, false);
      }
      __syncthreads();
      if (tid == 0) {
        fd_publish(&ctl->tchunk[c][r]);
        if (fd_release_add(&ctl->tdone[c]) == R - 1) fd_publish(&ctl->colfinal[c]);
      }
      prof(1);
      continue;
    }
    // S(j, x, u)
    int I, J;
    sh.unit(x, u, I, J);
    if (tid == 0) {  // the TRSM chunks of step j holding rows 64I.. and 64J.. (two each), then step j - 1's fold
      const int r0 = (j + 1) * FD_B, nr = sh.chunks(j);
      const int ci = (64 * I - r0) / 32, cj = (64 * J - r0) / 32;
      fd_wait(&ctl->tchunk[j][ci], 1, err);
      if (ci + 1 < nr) fd_wait(&ctl->tchunk[j][ci + 1], 1, err);
      if (cj != ci) {
        fd_wait(&ctl->tchunk[j][cj], 1, err);
        if (cj + 1 < nr) fd_wait(&ctl->tchunk[j][cj + 1], 1, err);
      }
      fd_wait(ucnt(I, J), j, err);
    }
    __syncthreads();
    t_ready = clock64();
    if (!decide_skip(j)) fd_update_unit(g, off, ld, n, j, I, J, reinterpret_cast<double*>(fd_smem), ctl->prof);
    __syncthreads();
    if (tid == 0) fd_release_add(ucnt(I, J));
    prof(2);
  }
}

template <typename T, int W>
int launch_trsm_warp(double alpha, const T* t, int64_t toff, int64_t trs, int64_t tcs, T* b, int64_t boff,
                     int64_t brs, int64_t bcs, int64_t m, int n, int64_t kc, const int* abort_flag, cudaStream_t s) {
  const size_t smem = (size_t(128) * TW_LD + size_t(W) * 128 * TW_XLD) * sizeof(T);  // W groups
  if (!smem_attr(reinterpret_cast<const void*>(trsm_warp_right_kernel<T, W>), int(smem))) return -10;
  const int64_t blocks = (m + 32 * W - 1) / (32 * W);
  if (blocks > 0x7fffffffLL) return -3;
  note_launch();
  if (launch_maybe_pdl(trsm_warp_right_kernel<T, W>, dim3(unsigned(blocks)), dim3(128 * W), smem, s, g_pdl != 0,
                       alpha, t, toff, trs, tcs, b, boff, brs, bcs, m, n, kc, abort_flag) != cudaSuccess)
    return -11;
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace

namespace {
__global__ void copy2d_unless_aborted_kernel(const double* src, int64_t sld, double* dst, int64_t dld, int64_t m,
                                             int64_t n, const int* abort_flag) {
  if (abort_flag != nullptr && *abort_flag >= 0) return;
  const int64_t total = m * n, stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / n, j = e - i * n;
    dst[i * dld + j] = src[i * sld + j];
  }
}
}  // namespace

// dst(m x n, ld dld) = src(m x n, ld sld) unless *abort_flag >= 0 (a pivot
// failure has been recorded): the overlapped panel's solved rows reach the
// matrix only when the diagonal factor before them succeeded
int launch_copy2d_unless_aborted(const double* src, int64_t sld, double* dst, int64_t dld, int64_t m, int64_t n,
                                 const int* abort_flag, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  const int64_t total = m * n;
  const int blocks = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  note_launch();
  copy2d_unless_aborted_kernel<<<blocks, 256, 0, s>>>(src, sld, dst, dld, m, n, abort_flag);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_scale(int is_f64, double beta, void* c, int64_t off, int64_t m, int64_t n, int64_t rs, int64_t cs,
                 const int64_t* rscat, const int64_t* cscat, int lower_only, cudaStream_t s) {
  int64_t total = m * n;
  if (total <= 0) return 0;
  int blocks = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  note_launch();
  if (is_f64 == 1)
    scale_kernel<double, double><<<blocks, 256, 0, s>>>((double*)c, off, m, n, rs, cs, rscat, cscat, beta, lower_only);
  else if (is_f64 == 2)  // f32 storage, f64 accumulation
    scale_kernel<float, double><<<blocks, 256, 0, s>>>((float*)c, off, m, n, rs, cs, rscat, cscat, beta, lower_only);
  else
    scale_kernel<float, float><<<blocks, 256, 0, s>>>((float*)c, off, m, n, rs, cs, rscat, cscat, float(beta), lower_only);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

static constexpr int LEAF_SMEM_LIMIT = 220 * 1024;

template <typename T>
static int leaf_launch(T* a, int64_t off, int64_t n, int64_t rs, int64_t cs, int variant, int64_t base_index,
                       int* d_info, cudaStream_t s) {
  if (variant == 3 && n <= 128 && g_leaf_blocked) {
    const size_t smem = size_t(128) * LV4_LD * sizeof(T);
    if (!smem_attr(reinterpret_cast<const void*>(potrf_leaf_blocked_kernel<T>), int(smem))) return -10;
    note_launch();
    if (launch_maybe_pdl(potrf_leaf_blocked_kernel<T>, dim3(1), dim3(128), smem, s, g_pdl != 0, a, off, int(n), rs, cs,
                         base_index, d_info, g_leaf_pipe) != cudaSuccess)
      return -11;
    return cudaGetLastError() == cudaSuccess ? 0 : -11;
  }
  if (variant == 3 && n <= 128) {
    const size_t smem = size_t(128) * 129 * sizeof(T);  // full tile: the update reads rows < 128 unguarded
    if (!smem_attr(reinterpret_cast<const void*>(potrf_leaf_v3_smem_kernel<T>), int(smem))) return -10;
    note_launch();
    potrf_leaf_v3_smem_kernel<T><<<1, 256, smem, s>>>(a, off, int(n), rs, cs, base_index, d_info);
    return cudaGetLastError() == cudaSuccess ? 0 : -11;
  }
  size_t smem = size_t(n) * (n + 1) * sizeof(T) + size_t(n) * sizeof(double);
  if (smem <= size_t(LEAF_SMEM_LIMIT)) {
    if (!smem_attr(reinterpret_cast<const void*>(potrf_leaf_kernel<T, true>), LEAF_SMEM_LIMIT)) return -10;
    note_launch();
    potrf_leaf_kernel<T, true><<<1, LEAF_THREADS, smem, s>>>(a, off, int(n), rs, cs, variant, base_index, d_info,
                                                              nullptr);
  } else {
    // large unblocked leaf (a tree that asks for it): in place in global memory
    double* scratch = nullptr;
    if (cudaMallocAsync(&scratch, size_t(n) * sizeof(double), s) != cudaSuccess) return -12;
    note_launch();
    potrf_leaf_kernel<T, false><<<1, LEAF_THREADS, 0, s>>>(a, off, int(n), rs, cs, variant, base_index, d_info,
                                                            scratch);
    cudaFreeAsync(scratch, s);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_potrf_leaf(int is_f64, int variant, void* a, int64_t off, int64_t n, int64_t rs, int64_t cs,
                      int64_t base_index, int* d_info, cudaStream_t s) {
  if (n <= 0) return 0;
  if (n > 0x7fffffff) return -3;
  if (is_f64) return leaf_launch<double>((double*)a, off, n, rs, cs, variant, base_index, d_info, s);
  return leaf_launch<float>((float*)a, off, n, rs, cs, variant, base_index, d_info, s);
}

int launch_trsm_diag_tiles(const double* l, int64_t ldl, double* x, int64_t ldx, int64_t n, int64_t kc,
                           cudaStream_t s) {
  if (n <= 0) return 0;
  const size_t smem = (size_t(128) * TW_LD + size_t(128) * TW_XLD) * sizeof(double);
  if (!smem_attr(reinterpret_cast<const void*>(trsm_diag_tiles_kernel), int(smem))) return -10;
  note_launch();
  trsm_diag_tiles_kernel<<<dim3(4, unsigned((n + 127) / 128)), 128, smem, s>>>(l, ldl, x, ldx, n, kc);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// The diagonal block a[off..] (n x n, row stride ld, 128 < n <= 2048) factored
// by {variant 3, bs 128, kc} over the unblocked3 leaf in one launch
// (potrf_diag_fused_kernel) on `ctas` CTAs (0: one per SM).
int g_fused_diag = 1;
static void* g_fd_last = nullptr;  // counters of the last launch (fused_diag_stats)
// tools: the last fused factor's per-kind task counts and summed wait / run
// cycles (synchronizes the device)
int fused_diag_stats(int64_t* out12) {
  if (!g_fd_last) return -1;
  unsigned long long h[12];
  cudaDeviceSynchronize();
  if (cudaMemcpy(h, g_fd_last, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -11;
  for (int i = 0; i < 12; ++i) out12[i] = int64_t(h[i]);
  return 0;
}
int launch_potrf_diag_fused(double* a, int64_t off, int64_t n, int64_t ld, int64_t kc, int64_t base_index,
                            int* d_info, int ctas, cudaStream_t s, cudaEvent_t after_reset, int** colfinal) {
  if (n <= FD_B || n > FD_MAXN || kc < FD_B) return -3;
  auto* ctl = static_cast<FdCounters*>(stream_scratch(11, sizeof(FdCounters), s));
  if (!ctl) return -10;
  g_fd_last = ctl;
  if (cudaMemsetAsync(ctl, 0, sizeof(FdCounters), s) != cudaSuccess) return -11;
  if (after_reset) cudaEventRecord(after_reset, s);
  if (colfinal) *colfinal = ctl->colfinal;
  if (!smem_attr(reinterpret_cast<const void*>(potrf_diag_fused_kernel), int(FD_SMEM))) return -10;
  static int sms_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!sms_dev[dev]) cudaDeviceGetAttribute(&sms_dev[dev], cudaDevAttrMultiProcessorCount, dev);
  const int grid = ctas > 0 && ctas < sms_dev[dev] ? ctas : sms_dev[dev];
  note_launch();
  potrf_diag_fused_kernel<<<grid, 128, FD_SMEM, s>>>(a, off, int(n), ld, kc, base_index, d_info, g_leaf_pipe, ctl);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_trsm_base_right(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                           int64_t boff, int64_t brs, int64_t bcs, int64_t m, int64_t n, int* d_singular,
                           int64_t index_base, const int* abort_flag, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  if (n > 32) return -3;
  const int threads = 128;  // == rows per CTA (the kernel's staging tile)
  const int64_t blocks = (m + threads - 1) / threads;
  note_launch();
  if (is_f64)
    trsm_base_right_kernel<double><<<unsigned(blocks), threads, 0, s>>>(
        alpha, (const double*)t, toff, trs, tcs, (double*)b, boff, brs, bcs, m, int(n), d_singular, index_base,
        abort_flag);
  else
    trsm_base_right_kernel<float><<<unsigned(blocks), threads, 0, s>>>(
        alpha, (const float*)t, toff, trs, tcs, (float*)b, boff, brs, bcs, m, int(n), d_singular,
        index_base, abort_flag);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf

namespace bf {
int launch_trsm_small_right(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                            int64_t boff, int64_t brs, int64_t bcs, int64_t m, int64_t n, int64_t kc,
                            const int* abort_flag, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  if (n > 128) return -3;
  if (g_trsm_warp) {
    // 4 warps per 32 rows; one group per CTA while the grid fits a wave,
    // groups sharing the staged triangle beyond (2 for f64, 4 for f32:
    // shared-memory bound)
    const bool big = m > 32 * 148;
    if (is_f64)
      return big ? launch_trsm_warp<double, 2>(alpha, (const double*)t, toff, trs, tcs, (double*)b, boff, brs, bcs, m,
                                               int(n), kc, abort_flag, s)
                 : launch_trsm_warp<double, 1>(alpha, (const double*)t, toff, trs, tcs, (double*)b, boff, brs, bcs, m,
                                               int(n), kc, abort_flag, s);
    return big ? launch_trsm_warp<float, 4>(alpha, (const float*)t, toff, trs, tcs, (float*)b, boff, brs, bcs, m,
                                            int(n), kc, abort_flag, s)
               : launch_trsm_warp<float, 1>(alpha, (const float*)t, toff, trs, tcs, (float*)b, boff, brs, bcs, m,
                                            int(n), kc, abort_flag, s);
  }
  const int64_t blocks = (m + TS_ROWS - 1) / TS_ROWS;
  if (blocks > 0x7fffffffLL) return -3;
  note_launch();
  if (is_f64) {
    const size_t smem = size_t(128 + TS_ROWS) * TS_LD * sizeof(double);
    if (!smem_attr(reinterpret_cast<const void*>(trsm_small_right_kernel<double>), int(smem))) return -10;
    trsm_small_right_kernel<double><<<unsigned(blocks), TS_THREADS, smem, s>>>(
        alpha, (const double*)t, toff, trs, tcs, (double*)b, boff, brs, bcs, m, int(n), kc, abort_flag);
  } else {
    const size_t smem = size_t(128 + TS_ROWS) * TS_LD * sizeof(float);
    if (!smem_attr(reinterpret_cast<const void*>(trsm_small_right_kernel<float>), int(smem))) return -10;
    trsm_small_right_kernel<float><<<unsigned(blocks), TS_THREADS, smem, s>>>(
        alpha, (const float*)t, toff, trs, tcs, (float*)b, boff, brs, bcs, m, int(n), kc, abort_flag);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}
}  // namespace bf
