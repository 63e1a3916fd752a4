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

namespace bf {

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
template <typename T>
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
    for (int i = k + 1 + tid; i < n; i += LEAF_THREADS) a(i, k) = Ops<T>::div(a(i, k), d);
    __syncthreads();
    // trailing triangle k < j <= i < n; 32 x 16 thread grid, j fastest
    const int tx = tid & 31, ty = tid >> 5;
    for (int i = k + 1 + ty; i < n; i += LEAF_THREADS / 32) {
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

// Variant 3 (right-looking) for n <= 128, blocked in 32-column panels while
// keeping unblocked3's exact per-element operation sequence: element (i,j)
// still receives a(i,j) -= a(i,k)*a(j,k) for k = 0..j-1 in ascending order,
// each product and difference rounded separately, then a(i,j) /= d_j
// (factor/cholesky.py:74-89).  Only the schedule differs:
//   (A) panel: 128 threads, thread r owns row p0+r of the 32-column panel in
//       registers; per pivot: sqrt by the diagonal owner, scale, publish the
//       top-32 column values, rank-1 update inside the panel (named barrier);
//   (B) trailing: all 16 warps apply the panel's 32 pivots to the trailing
//       triangle, each element updated sequentially k = p0..p0+31 from
//       registers, operands broadcast from shared memory.
// The whole leaf lives in shared memory (n x (n+1) doubles).
template <typename T>
__global__ void __launch_bounds__(512) potrf_leaf_v3_blk_kernel(T* g, int64_t off, int n, int64_t rs, int64_t cs,
                                                                int64_t base_index, int* d_info) {
  if (d_info != nullptr && *d_info >= 0) return;
  extern __shared__ __align__(16) unsigned char leaf_blk_smem[];
  T* A = reinterpret_cast<T*>(leaf_blk_smem);  // A[i * LD + j]
  constexpr int LD = 129;
  __shared__ T s_col[32];
  __shared__ T s_d;
  __shared__ int s_flag;
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += 512) {
    const int i = e / n, j = e % n;
    if (j <= i) A[i * LD + j] = g[off + i * rs + j * cs];
  }
  if (tid == 0) s_flag = -1;
  __syncthreads();

  for (int p0 = 0; p0 < n; p0 += 32) {
    const int pw = n - p0 < 32 ? n - p0 : 32;
    // ---- (A) panel columns [p0, p0+pw), rows [p0, n) ----
    if (tid < 128) {
      const int i = p0 + tid;
      const bool own = i < n;
      T r[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = (own && c < pw && p0 + c <= i) ? A[i * LD + p0 + c] : T(0);
#pragma unroll
      for (int kk = 0; kk < 32; ++kk) {
        if (kk < pw) {
          const int k = p0 + kk;
          if (tid == kk) {
            T d = r[kk];
            if (!(d > T(0))) {
              s_flag = k;
            } else {
              d = Ops<T>::sqrt_(d);
              r[kk] = d;
              s_d = d;
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (s_flag >= 0) break;
          const T d = s_d;
          if (own && i > k) {
            r[kk] = Ops<T>::div(r[kk], d);
            if (tid < pw) s_col[tid] = r[kk];
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (own && i > k) {
            const T x = r[kk];
#pragma unroll
            for (int c = kk + 1; c < 32; ++c)
              if (c < pw && p0 + c <= i) r[c] = Ops<T>::sub(r[c], Ops<T>::mul(x, s_col[c]));
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (own && c < pw && p0 + c <= i) A[i * LD + p0 + c] = r[c];
    }
    __syncthreads();
    // A failed pivot k stops the reference after steps < k have updated the
    // whole trailing triangle, so the trailing pass still applies p0..k-1.
    const int kend = s_flag >= 0 ? s_flag - p0 : pw;
    // ---- (B) trailing triangle: columns/rows >= q0 ----
    const int q0 = p0 + pw, m = n - q0;
    if (m > 0 && kend > 0) {
      const int tx = tid & 31, ty = tid >> 5;  // element (q0+ty+16a, q0+tx+32b)
      T v[6][3];
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int i = ty + 16 * a, j = tx + 32 * b;
          v[a][b] = (i < m && j <= i) ? A[(q0 + i) * LD + q0 + j] : T(0);
        }
#pragma unroll 4
      for (int kk = 0; kk < kend; ++kk) {
        const int k = p0 + kk;
        T xi[6], xj[3];
#pragma unroll
        for (int a = 0; a < 6; ++a) xi[a] = A[((q0 + ty + 16 * a) & 127) * LD + k];
#pragma unroll
        for (int b = 0; b < 3; ++b) xj[b] = A[((q0 + tx + 32 * b) & 127) * LD + k];
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const int i = ty + 16 * a, j = tx + 32 * b;
            if (16 * a + 15 >= 32 * b && i < m && j <= i) v[a][b] = Ops<T>::sub(v[a][b], Ops<T>::mul(xi[a], xj[b]));
          }
      }
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int i = ty + 16 * a, j = tx + 32 * b;
          if (i < m && j <= i) A[(q0 + i) * LD + q0 + j] = v[a][b];
        }
    }
    __syncthreads();
    if (s_flag >= 0) break;
  }
  for (int e = tid; e < n * n; e += 512) {
    const int i = e / n, j = e % n;
    if (j <= i) g[off + i * rs + j * cs] = A[i * LD + j];
  }
  if (tid == 0 && s_flag >= 0 && d_info != nullptr) *d_info = int(base_index + s_flag);
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

}  // namespace

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
  if (variant == 3 && n <= 128) {
    static bool blk_attr = false;
    const size_t smem = size_t(128) * 129 * sizeof(T);  // full tile: the trailing loop reads rows < 128 unguarded
    if (!blk_attr) {
      if (cudaFuncSetAttribute(potrf_leaf_v3_blk_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(128 * 129 * sizeof(T))) != cudaSuccess)
        return -10;
      blk_attr = true;
    }
    note_launch();
    potrf_leaf_v3_blk_kernel<T><<<1, 512, smem, s>>>(a, off, int(n), rs, cs, base_index, d_info);
    return cudaGetLastError() == cudaSuccess ? 0 : -11;
  }
  size_t smem = size_t(n) * (n + 1) * sizeof(T) + size_t(n) * sizeof(double);
  if (smem <= size_t(LEAF_SMEM_LIMIT)) {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(potrf_leaf_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               LEAF_SMEM_LIMIT) != cudaSuccess)
        return -10;
      attr = true;
    }
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
