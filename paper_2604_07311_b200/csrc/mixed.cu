// Kernels of the mixed-precision solve (BASELINE configs[3]): precision
// conversions, the FP64 residual r = b - A x, and the two triangular solves
// with the fp32 factor used by iterative refinement (fp64 right-hand sides).
// All memory-bound; they stream the matrix once per call.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#include "blockfam_b200.h"

#include <cuda_bf16.h>

namespace bf {

namespace {

template <typename S, typename D>
__global__ void convert_kernel(const S* src, int64_t soff, int64_t srs, int64_t scs, D* dst, int64_t doff,
                               int64_t drs, int64_t dcs, int64_t m, int64_t n, int lower_only) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (lower_only && j > i) continue;
    dst[doff + i * drs + j * dcs] = D(src[soff + i * srs + j * scs]);
  }
}

// r = b - A x  (A n x n fp64 row-major lda, full matrix); one warp per row
__global__ void residual_kernel(const double* A, int64_t lda, const double* x, const double* b, double* r, int64_t n) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + row * lda;
  double s = 0.0;
  for (int64_t j = lane * 2; j < n; j += 64) {
    const double2 av = *reinterpret_cast<const double2*>(a + j);
    s = fma(av.x, x[j], s);
    if (j + 1 < n) s = fma(av.y, x[j + 1], s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) r[row] = b[row] - s;
}

// Symmetric A (full storage, SPD input of the solve): y = A x from the lower
// triangle only — half the HBM traffic of the row-by-row GEMV.  One CTA per
// 128 x 128 lower tile (I >= J): its row sums A_IJ x_J feed y_I, its column
// sums A_IJ^T x_I feed y_J (strictly lower part on a diagonal tile); the
// per-tile partials are summed per row by symv_reduce_kernel (fixed order).
// ABS: |A| times the ones vector, i.e. the row sums of |A| (the infinity norm).
constexpr int SY_T = 128;
template <bool ABS>
__global__ void __launch_bounds__(256) symv_tiles_kernel(const double* __restrict__ A, int64_t lda,
                                                          const double* __restrict__ x, int64_t n,
                                                          double* part_row, double* part_col) {
  __shared__ double xj[SY_T], xi[SY_T], colbuf[8][SY_T];
  const int64_t p = blockIdx.x;
  int64_t I = int64_t((sqrt(8.0 * double(p) + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > p) --I;
  while ((I + 1) * (I + 2) / 2 <= p) ++I;
  const int64_t J = p - I * (I + 1) / 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t i0 = I * SY_T, j0 = J * SY_T;
  if (tid < SY_T) {
    xj[tid] = j0 + tid < n ? (ABS ? 1.0 : x[j0 + tid]) : 0.0;
    xi[tid] = i0 + tid < n ? (ABS ? 1.0 : x[i0 + tid]) : 0.0;
  }
  __syncthreads();
  const bool diag = I == J;
  double cacc[4] = {0.0, 0.0, 0.0, 0.0};
  const int jl[4] = {2 * lane, 2 * lane + 1, 64 + 2 * lane, 65 + 2 * lane};
  for (int il = warp; il < SY_T; il += 8) {
    const int64_t gi = i0 + il;
    if (gi >= n) break;
    const double* row = A + gi * lda + j0;
    double av[4];
    const bool in0 = j0 + jl[0] < n, in2 = j0 + jl[2] < n;  // pairs of columns: n even
    if (in0) {
      const double2 q = *reinterpret_cast<const double2*>(row + jl[0]);
      av[0] = q.x;
      av[1] = q.y;
    } else {
      av[0] = av[1] = 0.0;
    }
    if (in2) {
      const double2 q = *reinterpret_cast<const double2*>(row + jl[2]);
      av[2] = q.x;
      av[3] = q.y;
    } else {
      av[2] = av[3] = 0.0;
    }
    double rs = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double a = ABS ? fabs(av[e]) : av[e];
      if (!diag || jl[e] <= il) rs = fma(a, xj[jl[e]], rs);
      if (!diag || jl[e] < il) cacc[e] = fma(a, xi[il], cacc[e]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
    if (lane == 0) part_row[p * SY_T + il] = rs;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) colbuf[warp][jl[e]] = cacc[e];
  __syncthreads();
  if (tid < SY_T) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += colbuf[w][tid];
    part_col[p * SY_T + tid] = t;
  }
}

// y_i = sum_{J <= I} row partial (I, J) + sum_{I' >= I} column partial (I', I);
// out_i = base_i - y_i (residual) or y_i (base == nullptr)
__global__ void symv_reduce_kernel(const double* part_row, const double* part_col, int64_t n, const double* base,
                                   double* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t I = i / SY_T, il = i % SY_T, nt = (n + SY_T - 1) / SY_T;
  double y = 0.0;
  for (int64_t J = 0; J <= I; ++J) y += part_row[(I * (I + 1) / 2 + J) * SY_T + il];
  for (int64_t Ip = I; Ip < nt; ++Ip) y += part_col[(Ip * (Ip + 1) / 2 + I) * SY_T + il];
  out[i] = base ? base[i] - y : y;
}

// out[row] = sum_j |A[row][j]| (one warp per row); the host takes the max
__global__ void row_abs_sum_kernel(const double* A, int64_t lda, double* out, int64_t n) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + row * lda;
  double s = 0.0;
  for (int64_t j = lane * 2; j < n; j += 64) {
    const double2 av = *reinterpret_cast<const double2*>(a + j);
    s += fabs(av.x);
    if (j + 1 < n) s += fabs(av.y);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = s;
}

// forward diagonal-block solve: y[lo:hi] = L[lo:hi,lo:hi]^-1 y[lo:hi]
// (one CTA, fp64 arithmetic on the fp32 factor)
__global__ void trsv_diag_fwd_kernel(const float* L, int64_t ld, double* y, int64_t lo, int nb) {
  __shared__ double ys[256];
  const int t = threadIdx.x;
  if (t < nb) ys[t] = y[lo + t];
  __syncthreads();
  double acc = t < nb ? ys[t] : 0.0;
  for (int j = 0; j < nb; ++j) {
    if (t == j) ys[j] = acc / double(L[(lo + j) * ld + lo + j]);
    __syncthreads();
    if (t > j && t < nb) acc -= double(L[(lo + t) * ld + lo + j]) * ys[j];
  }
  if (t < nb) y[lo + t] = ys[t];
}

// backward diagonal-block solve with L^T: x[lo:hi] = L[lo:hi,lo:hi]^-T x[lo:hi]
__global__ void trsv_diag_bwd_kernel(const float* L, int64_t ld, double* x, int64_t lo, int nb) {
  __shared__ double xs[256];
  const int t = threadIdx.x;
  if (t < nb) xs[t] = x[lo + t];
  __syncthreads();
  double acc = t < nb ? xs[t] : 0.0;
  for (int j = nb - 1; j >= 0; --j) {
    if (t == j) xs[j] = acc / double(L[(lo + j) * ld + lo + j]);
    __syncthreads();
    if (t < j) acc -= double(L[(lo + j) * ld + lo + t]) * xs[j];  // (L^T)_{t,j} = L_{j,t}
  }
  if (t < nb) x[lo + t] = xs[t];
}

// forward panel update: y[r] -= sum_{p in [lo,hi)} L[r][p] y[p] for r >= hi; one warp per row
__global__ void trsv_panel_fwd_kernel(const float* L, int64_t ld, double* y, int64_t lo, int nb, int64_t hi, int64_t n) {
  const int64_t row = hi + ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int p = lane; p < nb; p += 32) s = fma(double(L[row * ld + lo + p]), y[lo + p], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] -= s;
}

// backward panel update: x[c] -= sum_{i in [lo,hi)} L[i][c] x[i] for c < lo; one thread per column
__global__ void trsv_panel_bwd_kernel(const float* L, int64_t ld, double* x, int64_t lo, int nb) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= lo) return;
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s = fma(double(L[(lo + i) * ld + c]), x[lo + i], s);
  x[c] -= s;
}

// out[i] = (base ? base[i] : 0) + sign * sum_j A[i*lda + j] v[j], i < rows; one warp per row,
// VEC floats per lane per load and 4 loads in flight per lane
template <int VEC>
__global__ void gemv_n_kernel(const float* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                              const double* __restrict__ v, const double* base, double* out, double sign) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* a = A + row * lda;
  constexpr int STEP = 32 * VEC;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t j = int64_t(lane) * VEC;
  for (; j + 3 * STEP < cols; j += 4 * STEP) {
    float x[4][VEC];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if constexpr (VEC == 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(a + j + u * STEP));
        x[u][0] = q.x;
        x[u][1] = q.y;
        x[u][2] = q.z;
        x[u][3] = q.w;
      } else {
        x[u][0] = __ldg(a + j + u * STEP);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < VEC; ++e) s[u] = fma(double(x[u][e]), v[j + u * STEP + e], s[u]);
  }
  for (; j < cols; j += STEP)
#pragma unroll
    for (int e = 0; e < VEC; ++e) s[0] = fma(double(__ldg(a + j + e)), v[j + e], s[0]);
  double t = (s[0] + s[1]) + (s[2] + s[3]);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) out[row] = (base ? base[row] : 0.0) + sign * t;
}

// partial[c][j] = sum_{i in chunk c} A[i*lda + j] v[i]  (A^T v split over row chunks). A CTA covers
// 256 columns with 256/VEC column threads x VEC row groups; 4 rows in flight per thread.
template <int VEC>
__global__ void gemv_t_partial_kernel(const float* __restrict__ A, int64_t lda, int64_t rows, int cols,
                                      const double* __restrict__ v, double* partial, int64_t rows_per_chunk) {
  constexpr int CT = 256 / VEC, RG = VEC;
  __shared__ double red[RG][256];
  const int ct = threadIdx.x % CT, rg = threadIdx.x / CT;
  const int j0 = blockIdx.x * 256 + ct * VEC;
  const int c = blockIdx.y;
  const int64_t r0 = int64_t(c) * rows_per_chunk;
  const int64_t r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  double acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
  if (j0 < cols) {
    int64_t i = r0 + rg;
    for (; i + 3 * RG < r1; i += 4 * RG) {
      float x[4][VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float* src = A + (i + u * RG) * lda + j0;
        if constexpr (VEC == 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(src));
          x[u][0] = q.x;
          x[u][1] = q.y;
          x[u][2] = q.z;
          x[u][3] = q.w;
        } else {
          x[u][0] = __ldg(src);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double vi = v[i + u * RG];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma(double(x[u][e]), vi, acc[e]);
      }
    }
    for (; i < r1; i += RG) {
      const double vi = v[i];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = fma(double(__ldg(A + i * lda + j0 + e)), vi, acc[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) red[rg][ct * VEC + e] = acc[e];
  __syncthreads();
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j < cols) {
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < RG; ++g) t += red[g][threadIdx.x];
    partial[int64_t(c) * cols + j] = t;
  }
}

// out[j] = (base ? base[j] : 0) + sign * sum_c partial[c][j]
__global__ void reduce_partial_kernel(const double* partial, int chunks, int cols, const double* base, double* out,
                                      double sign) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += partial[int64_t(c) * cols + j];
  out[j] = (base ? base[j] : 0.0) + sign * s;
}

constexpr int kPotrsMaxChunks = 128;

inline int grid_for_elems(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return int(b < 148 * 16 ? b : 148 * 16);
}

}  // namespace

int launch_f64_to_f32(const double* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t doff, int64_t drs,
                      int64_t dcs, int64_t m, int64_t n, int lower_only, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  convert_kernel<double, float>
      <<<grid_for_elems(m * n), 256, 0, s>>>(src, soff, srs, scs, dst, doff, drs, dcs, m, n, lower_only);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_f32_to_f64(const float* src, int64_t soff, int64_t srs, int64_t scs, double* dst, int64_t doff, int64_t drs,
                      int64_t dcs, int64_t m, int64_t n, int lower_only, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  convert_kernel<float, double>
      <<<grid_for_elems(m * n), 256, 0, s>>>(src, soff, srs, scs, dst, doff, drs, dcs, m, n, lower_only);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int g_symv = 1;  // bf_set_option("symv", 0|1): residual and row sums from the lower triangle of (symmetric) A

// the lower-triangle SYMV: partials in library scratch (2 x 128 doubles per tile pair)
static int launch_symv(const double* A, int64_t lda, const double* x, int64_t n, const double* base, double* out,
                       bool abs_ones, cudaStream_t s) {
  const int64_t nt = (n + SY_T - 1) / SY_T, pairs = nt * (nt + 1) / 2;
  if (pairs > 0x7fffffffLL || n % 2) return -3;
  double* part = static_cast<double*>(stream_scratch(8, size_t(pairs) * 2 * SY_T * sizeof(double), s));
  if (!part) return -3;
  note_launch(2);
  if (abs_ones)
    symv_tiles_kernel<true><<<unsigned(pairs), 256, 0, s>>>(A, lda, nullptr, n, part, part + pairs * SY_T);
  else
    symv_tiles_kernel<false><<<unsigned(pairs), 256, 0, s>>>(A, lda, x, n, part, part + pairs * SY_T);
  symv_reduce_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(part, part + pairs * SY_T, n, base, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_residual(const double* A, int64_t lda, const double* x, const double* b, double* r, int64_t n,
                    cudaStream_t s) {
  if (n <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(A) % 16) || (lda % 2)) return -3;
  if (g_symv && launch_symv(A, lda, x, n, b, r, false, s) == 0) return 0;
  note_launch();
  residual_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(A, lda, x, b, r, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_row_abs_sum(const double* A, int64_t lda, double* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(A) % 16) || (lda % 2)) return -3;
  if (g_symv && launch_symv(A, lda, nullptr, n, nullptr, out, true, s) == 0) return 0;
  note_launch();
  row_abs_sum_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(A, lda, out, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// L (lower, fp32, row-major ld): solve L L^T x = rhs in place (x holds rhs)
int launch_potrs_f32_f64(const float* L, int64_t ld, double* x, int64_t n, cudaStream_t s) {
  constexpr int NB = 256;
  for (int64_t lo = 0; lo < n; lo += NB) {
    const int nb = int(n - lo < NB ? n - lo : NB);
    note_launch();
    trsv_diag_fwd_kernel<<<1, NB, 0, s>>>(L, ld, x, lo, nb);
    const int64_t rows = n - lo - nb;
    if (rows > 0) {
      note_launch();
      trsv_panel_fwd_kernel<<<unsigned((rows * 32 + 255) / 256), 256, 0, s>>>(L, ld, x, lo, nb, lo + nb, n);
    }
  }
  for (int64_t lo = ((n - 1) / NB) * NB; lo >= 0; lo -= NB) {
    const int nb = int(n - lo < NB ? n - lo : NB);
    note_launch();
    trsv_diag_bwd_kernel<<<1, NB, 0, s>>>(L, ld, x, lo, nb);
    if (lo > 0) {
      note_launch();
      trsv_panel_bwd_kernel<<<unsigned((lo + 255) / 256), 256, 0, s>>>(L, ld, x, lo, nb);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// The same blocked solve as ONE cooperative kernel (grid of <= 128 CTAs, three
// grid barriers per block) instead of ~4 launches per block and sweep: the
// refinement's solve is a chain of 2 * n / bs dependent matrix-vector
// products, so the launch latencies, not the 4 GB of L it streams, were its
// cost (2.4 ms at n = 32768).  Same products in a different summation order.
constexpr int PC_THREADS = 512;
// vec = 1 (L, xinv 16-byte aligned, ld, bs and n multiples of 4): float4 loads
// with four in flight per thread, so each SM keeps ~32 KB of the stream in
// flight — the scalar form's ~8 KB left it latency-bound at a third of HBM.
__global__ void __launch_bounds__(PC_THREADS, 1)
    potrs_coop_kernel(const float* __restrict__ L, int64_t ld, const float* __restrict__ xinv, int64_t bs,
                      double* x, int64_t n, double* partial, double* tv, int vec) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[2048];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t gwarp = int64_t(c) * (PC_THREADS / 32) + warp, nwarps = int64_t(G) * (PC_THREADS / 32);
  const int64_t nblk = (n + bs - 1) / bs;
  // vec: out[j] = sum_{i in [i0, i1)} A[i * lda + j] v[i] for j < b (b % 4 == 0,
  // b <= 2048).  Thread = 4 columns x one of rg row groups (rows i0 + g, +rg,
  // ...), four rows per iteration; the row groups are combined through sv in
  // a fixed order.  Ends with sv clobbered.
  auto colsum4 = [&](const float* A, int64_t lda, const double* v, int64_t i0, int64_t i1, int b, double* out) {
    const int c4 = b >> 2, rg = PC_THREADS / c4;
    const int g = tid / c4, j = (tid % c4) * 4;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (g < rg) {
      int64_t i = i0 + g;
      for (; i + 3 * rg < i1; i += 4 * rg) {
        const float4 q0 = __ldcs(reinterpret_cast<const float4*>(A + i * lda + j));
        const float4 q1 = __ldcs(reinterpret_cast<const float4*>(A + (i + rg) * lda + j));
        const float4 q2 = __ldcs(reinterpret_cast<const float4*>(A + (i + 2 * rg) * lda + j));
        const float4 q3 = __ldcs(reinterpret_cast<const float4*>(A + (i + 3 * rg) * lda + j));
        const double v0 = v[i], v1 = v[i + rg], v2 = v[i + 2 * rg], v3 = v[i + 3 * rg];
        a0 = fma(double(q0.x), v0, a0); a1 = fma(double(q0.y), v0, a1);
        a2 = fma(double(q0.z), v0, a2); a3 = fma(double(q0.w), v0, a3);
        a0 = fma(double(q1.x), v1, a0); a1 = fma(double(q1.y), v1, a1);
        a2 = fma(double(q1.z), v1, a2); a3 = fma(double(q1.w), v1, a3);
        a0 = fma(double(q2.x), v2, a0); a1 = fma(double(q2.y), v2, a1);
        a2 = fma(double(q2.z), v2, a2); a3 = fma(double(q2.w), v2, a3);
        a0 = fma(double(q3.x), v3, a0); a1 = fma(double(q3.y), v3, a1);
        a2 = fma(double(q3.z), v3, a2); a3 = fma(double(q3.w), v3, a3);
      }
      for (; i < i1; i += rg) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(A + i * lda + j));
        const double vi = v[i];
        a0 = fma(double(q.x), vi, a0); a1 = fma(double(q.y), vi, a1);
        a2 = fma(double(q.z), vi, a2); a3 = fma(double(q.w), vi, a3);
      }
      double* s = sv + int64_t(g) * b + j;
      s[0] = a0; s[1] = a1; s[2] = a2; s[3] = a3;
    }
    __syncthreads();
    for (int jj = tid; jj < b; jj += PC_THREADS) {
      double t = 0.0;
      for (int q = 0; q < rg; ++q) t += sv[int64_t(q) * b + jj];
      out[jj] = t;
    }
    __syncthreads();
  };
  // vec: warp-per-row dot product of a fp32 row (16-byte aligned, b % 4 == 0)
  // with the smem vector sv, four float4 per lane in flight
  auto row_dot4 = [&](const float* row, int b) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = lane * 4;
    for (; j + 384 < b; j += 512) {
      const float4 q0 = __ldcs(reinterpret_cast<const float4*>(row + j));
      const float4 q1 = __ldcs(reinterpret_cast<const float4*>(row + j + 128));
      const float4 q2 = __ldcs(reinterpret_cast<const float4*>(row + j + 256));
      const float4 q3 = __ldcs(reinterpret_cast<const float4*>(row + j + 384));
      s0 = fma(double(q0.x), sv[j], s0); s1 = fma(double(q0.y), sv[j + 1], s1);
      s2 = fma(double(q0.z), sv[j + 2], s2); s3 = fma(double(q0.w), sv[j + 3], s3);
      s0 = fma(double(q1.x), sv[j + 128], s0); s1 = fma(double(q1.y), sv[j + 129], s1);
      s2 = fma(double(q1.z), sv[j + 130], s2); s3 = fma(double(q1.w), sv[j + 131], s3);
      s0 = fma(double(q2.x), sv[j + 256], s0); s1 = fma(double(q2.y), sv[j + 257], s1);
      s2 = fma(double(q2.z), sv[j + 258], s2); s3 = fma(double(q2.w), sv[j + 259], s3);
      s0 = fma(double(q3.x), sv[j + 384], s0); s1 = fma(double(q3.y), sv[j + 385], s1);
      s2 = fma(double(q3.z), sv[j + 386], s2); s3 = fma(double(q3.w), sv[j + 387], s3);
    }
    for (; j < b; j += 128) {
      const float4 q = __ldcs(reinterpret_cast<const float4*>(row + j));
      s0 = fma(double(q.x), sv[j], s0); s1 = fma(double(q.y), sv[j + 1], s1);
      s2 = fma(double(q.z), sv[j + 2], s2); s3 = fma(double(q.w), sv[j + 3], s3);
    }
    double t = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
  };
  // tv[j] = (base ? base[j] - t : t), t = sum_q partial[q][j] for j < b: one
  // warp per j, lane l adding q = l, l + 32, ... then a fixed shuffle tree
  // (every load in flight at once; a thread-per-j loop over the G partials
  // was a chain of G / unroll L2 round trips per block and direction)
  auto reduce_partials = [&](int b, const double* base) {
    for (int64_t jj = gwarp; jj < b; jj += nwarps) {
      double t = 0.0;
#pragma unroll 4
      for (int q = lane; q < G; q += 32) t += partial[int64_t(q) * bs + jj];
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) tv[jj] = base ? base[jj] - t : t;
    }
  };
  // warp-per-row dot product of a fp32 row with the smem vector sv
  auto row_dot = [&](const float* row, int b) {
    if (vec) return row_dot4(row, b);
    double s0 = 0.0, s1 = 0.0;
    int j = lane * 2;
    for (; j + 1 < b; j += 64) {
      const float2 q = *reinterpret_cast<const float2*>(row + j);
      s0 = fma(double(q.x), sv[j], s0);
      s1 = fma(double(q.y), sv[j + 1], s1);
    }
    if (j < b) s0 = fma(double(row[j]), sv[j], s0);
    double t = s0 + s1;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
  };
  // forward: y_k = X_k^T r_k; r[k+1:] -= L[k+1:, k] y_k   (x holds r, then y)
  for (int64_t k = 0; k < nblk; ++k) {
    const int64_t k0 = k * bs, k1 = k0 + bs < n ? k0 + bs : n;
    const int b = int(k1 - k0);
    const float* X = xinv + k * bs * bs;
    {  // partial[c][j] = sum over this CTA's rows i of X[i][j] r[k0+i]
      const int per = (b + G - 1) / G, i0 = c * per, i1 = i0 + per < b ? i0 + per : b;
      if (vec) colsum4(X, bs, x + k0, i0, i1 > i0 ? i1 : i0, b, partial + int64_t(c) * bs);
      else for (int j = tid; j < b; j += PC_THREADS) {
        double acc = 0.0;
        for (int i = i0; i < i1; ++i) acc = fma(double(X[int64_t(i) * bs + j]), x[k0 + i], acc);
        partial[int64_t(c) * bs + j] = acc;
      }
    }
    grid.sync();
    reduce_partials(b, nullptr);
    grid.sync();
    for (int j = tid; j < b; j += PC_THREADS) sv[j] = tv[j];
    __syncthreads();
    if (c == 0)
      for (int j = tid; j < b; j += PC_THREADS) x[k0 + j] = sv[j];
    for (int64_t row = k1 + gwarp; row < n; row += nwarps) {
      const double t = row_dot(L + row * ld + k0, b);
      if (lane == 0) x[row] -= t;
    }
    grid.sync();
  }
  // backward: x_k = X_k (y_k - L[k+1:, k]^T x[k+1:])
  for (int64_t k = nblk - 1; k >= 0; --k) {
    const int64_t k0 = k * bs, k1 = k0 + bs < n ? k0 + bs : n;
    const int b = int(k1 - k0);
    const float* X = xinv + k * bs * bs;
    {  // partial[c][j] = sum over this CTA's rows r >= k1 of L[r][k0+j] x[r]
      const int64_t rows = n - k1, per = (rows + G - 1) / G, r0 = k1 + c * per;
      const int64_t r1 = r0 + per < n ? r0 + per : n;
      if (vec) colsum4(L + k0, ld, x, r0, r1 > r0 ? r1 : r0, b, partial + int64_t(c) * bs);
      else for (int j = tid; j < b; j += PC_THREADS) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // four chains: loads in flight
        int64_t r = r0;
        for (; r + 3 < r1; r += 4) {
          a0 = fma(double(L[r * ld + k0 + j]), x[r], a0);
          a1 = fma(double(L[(r + 1) * ld + k0 + j]), x[r + 1], a1);
          a2 = fma(double(L[(r + 2) * ld + k0 + j]), x[r + 2], a2);
          a3 = fma(double(L[(r + 3) * ld + k0 + j]), x[r + 3], a3);
        }
        for (; r < r1; ++r) a0 = fma(double(L[r * ld + k0 + j]), x[r], a0);
        partial[int64_t(c) * bs + j] = (a0 + a1) + (a2 + a3);
      }
    }
    grid.sync();
    reduce_partials(b, x + k0);
    grid.sync();
    for (int j = tid; j < b; j += PC_THREADS) sv[j] = tv[j];
    __syncthreads();
    for (int64_t i = gwarp; i < b; i += nwarps) {
      const double t = row_dot(X + i * bs, b);
      if (lane == 0) x[k0 + i] = t;
    }
    grid.sync();
  }
}

int g_potrs_coop = 1;  // bf_set_option("potrs_coop", 0|1): the refinement solve as one cooperative kernel
int g_potrs_vec = 1;   // bf_set_option("potrs_vec", 0|1): float4 streams in the cooperative solve

// Blocked solve with the explicit inverses X_k = L_kk^-T of the diagonal
// blocks (xinv: nblk x bs x bs fp32, X_k row-major ld bs). Every step is a
// matrix-vector product streaming its block of L once, shaped so that the
// long dimension is spread over the whole GPU:
//   forward (right-looking)  y_k = X_k^T r_k;  r[k+1:] -= L[k+1:, k] y_k
//   backward (left-looking)  x_k = X_k (y_k - L[k+1:, k]^T x[k+1:])
// work: (kPotrsMaxChunks + 1) * bs doubles.
int launch_potrs_blocked(const float* L, int64_t ld, const float* xinv, int64_t bs, double* x, int64_t n,
                         double* work, cudaStream_t s) {
  double* t = work;
  double* partial = work + bs;
  if (g_potrs_coop && bs <= 2048 && ld % 2 == 0 && bs % 2 == 0 && reinterpret_cast<uintptr_t>(L) % 8 == 0 &&
      reinterpret_cast<uintptr_t>(xinv) % 8 == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, potrs_coop_kernel, PC_THREADS, 0);
    int G = sms * (per_sm > 0 ? 1 : 0);
    if (G > kPotrsMaxChunks) G = kPotrsMaxChunks;  // partial rows the work buffer holds
    if (G >= 1) {
      int vec = g_potrs_vec && reinterpret_cast<uintptr_t>(L) % 16 == 0 && reinterpret_cast<uintptr_t>(xinv) % 16 == 0 &&
                ld % 4 == 0 && bs % 4 == 0 && n % 4 == 0;
      void* args[] = {(void*)&L,    (void*)&ld,      (void*)&xinv, (void*)&bs, (void*)&x,
                      (void*)&n,    (void*)&partial, (void*)&t,    (void*)&vec};
      note_launch();
      if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(potrs_coop_kernel), dim3(G), dim3(PC_THREADS), args, 0,
                                      s) == cudaSuccess)
        return 0;
      cudaGetLastError();  // fall back to the launch-per-product form
    }
  }
  const bool vec_ok = (reinterpret_cast<uintptr_t>(L) % 16 == 0) && ld % 4 == 0 && bs % 4 == 0 &&
                      (reinterpret_cast<uintptr_t>(xinv) % 16 == 0);
  auto gemv_t = [&](const float* A, int64_t lda, int64_t rows, int cols, const double* v, bool vec) -> int {
    const int col_tiles = (cols + 255) / 256;
    int64_t chunks = (rows + 31) / 32;
    const int64_t want = (4 * 148 + col_tiles - 1) / col_tiles;
    if (chunks > want) chunks = want;
    if (chunks > kPotrsMaxChunks) chunks = kPotrsMaxChunks;
    if (chunks < 1) chunks = 1;
    const int64_t per = (rows + chunks - 1) / chunks;
    note_launch();
    if (vec)
      gemv_t_partial_kernel<4><<<dim3(col_tiles, unsigned(chunks)), 256, 0, s>>>(A, lda, rows, cols, v, partial, per);
    else
      gemv_t_partial_kernel<1><<<dim3(col_tiles, unsigned(chunks)), 256, 0, s>>>(A, lda, rows, cols, v, partial, per);
    return int(chunks);
  };
  auto gemv_n = [&](const float* A, int64_t lda, int64_t rows, int64_t cols, const double* v, const double* base,
                    double* out, double sign, bool vec) {
    note_launch();
    const unsigned grid = unsigned((rows * 32 + 255) / 256);
    if (vec)
      gemv_n_kernel<4><<<grid, 256, 0, s>>>(A, lda, rows, cols, v, base, out, sign);
    else
      gemv_n_kernel<1><<<grid, 256, 0, s>>>(A, lda, rows, cols, v, base, out, sign);
  };
  auto reduce = [&](int chunks, int cols, const double* base, double* out, double sign) {
    note_launch();
    reduce_partial_kernel<<<unsigned((cols + 255) / 256), 256, 0, s>>>(partial, chunks, cols, base, out, sign);
  };
  const int64_t nblk = (n + bs - 1) / bs;
  for (int64_t k = 0; k < nblk; ++k) {
    const int64_t k0 = k * bs, k1 = k0 + bs < n ? k0 + bs : n;
    const int b = int(k1 - k0);
    const float* X = xinv + k * bs * bs;
    const bool vx = vec_ok && b % 4 == 0;
    const int ch = gemv_t(X, bs, b, b, x + k0, vx);  // y_k = X_k^T r_k
    reduce(ch, b, nullptr, t, 1.0);
    if (k1 < n) gemv_n(L + k1 * ld + k0, ld, n - k1, b, t, x + k1, x + k1, -1.0, vx);
    reduce(ch, b, nullptr, x + k0, 1.0);
  }
  for (int64_t k = nblk - 1; k >= 0; --k) {
    const int64_t k0 = k * bs, k1 = k0 + bs < n ? k0 + bs : n;
    const int b = int(k1 - k0);
    const float* X = xinv + k * bs * bs;
    const bool vx = vec_ok && b % 4 == 0;
    if (k1 < n) {
      const int ch = gemv_t(L + k1 * ld + k0, ld, n - k1, b, x + k1, vx);  // L[k+1:,k]^T x[k+1:]
      reduce(ch, b, x + k0, t, -1.0);
    } else {
      reduce(0, b, x + k0, t, 1.0);
    }
    gemv_n(X, bs, b, b, t, nullptr, x + k0, 1.0, vx);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf

// ---- the factorization driver of the mixed solve ---------------------------
namespace bf {
namespace {

__global__ void set_identity_kernel(double* x, int64_t ld, int64_t b) {
  const int64_t total = b * b;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / b, j = e - i * b;
    x[i * ld + j] = i == j ? 1.0 : 0.0;
  }
}

}  // namespace

// C(f64 view) := beta*C + alpha*S (S fp32 m x n row-major, ld): the bf16
// contraction's epilogue in C's precision; beta == 0 never reads C
__global__ void axpby_f32_f64_kernel(double alpha, const float* src, int64_t ld, double beta, double* c, int64_t off,
                                     int64_t rs, int64_t cs, int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    double* p = c + off + i * rs + j * cs;
    const double v = alpha * double(src[i * ld + j]);
    *p = beta == 0.0 ? v : beta * *p + v;
  }
}

int launch_axpby_f32_f64(double alpha, const float* src, int64_t ld, double beta, double* c, int64_t off, int64_t rs,
                         int64_t cs, int64_t m, int64_t n, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  const int64_t total = m * n;
  note_launch();
  axpby_f32_f64_kernel<<<unsigned((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16), 256, 0, s>>>(
      alpha, src, ld, beta, c, off, rs, cs, m, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int g_mixed_inverse = 0;  // bf_set_option("mixed_inverse", 1): diagonal factor, then the doubling inverse
int g_mixed_reserve = 32;  // bf_set_option("mixed_reserve", r): SMs the trailing GEMMT leaves to the side chain

}  // namespace bf

namespace bf {
// capi.cu: the FP64 diagonal factor with X L^T = X solved on a second stream,
// trailing the factor's inner steps
int chol_inverse_overlapped(const bf_view& a, const bf_chol_level* lv, int nl, int64_t base, const bf_view& x,
                            int64_t kc, int* d_info, cudaStream_t st);
// capi.cu: the factor, then X = L^-T by recursive doubling
int chol_then_inverse(const bf_view& a, const bf_chol_level* lv, int nl, int64_t base, const bf_view& x, int64_t kc,
                      int* d_info, cudaStream_t st);
}  // namespace bf

extern "C" {
// bf_cholesky_mixed: see include/blockfam_b200.h
int bf_cholesky_mixed(const bf_view* a, float* w, int64_t ldw, void* pbuf0, void* pbuf1, void* xt, double* d64,
                      double* x64, float* xinv, int64_t bs, const bf_chol_level* lv, int nl, int precision,
                      int lookahead, int* d_info, void* stream) {
  using namespace bf;
  if (!a || !w || !pbuf0 || !pbuf1 || !xt || !d64 || !x64 || !xinv || !lv || nl < 1 || !d_info)
    return set_error(BF_ERR_VALUE, "null argument");
  if (a->m != a->n) return set_error(BF_ERR_SHAPE, "square matrix required");
  if (bs < 8 || bs % 8) return set_error(BF_ERR_SHAPE, "bs must be a multiple of 8");
  const int64_t n = a->n;
  if (n == 0) return BF_OK;
  const bool tf32 = precision == 1;
  cudaStream_t main = static_cast<cudaStream_t>(stream);
  cudaStream_t side = lookahead ? panel_stream_for(main) : main;
  if (lookahead && !side) return set_error(BF_ERR_CUDA, "cannot create the side stream");
  void* pbuf[2] = {pbuf0, pbuf1};
  const int64_t nblk = (n + bs - 1) / bs;
  auto ck = [](int rc, const char* what) { return rc ? set_error(rc < -10 ? rc : BF_ERR_CUDA, what) : BF_OK; };
  int rc = ck(launch_f64_to_f32(static_cast<const double*>(a->base), a->off, a->rs, a->cs, w, 0, ldw, 1, n, n, 1,
                                main),
              "convert A");
  if (rc) return rc;

  // diagonal block k (FP64 tree driver), its inverse X = L_kk^-T (FP64), and
  // the panel L21 = A21 X as one tensor-core GEMM, all on stream st
  auto diag_and_panel = [&](int64_t k, cudaStream_t st) -> int {
    const int64_t k0 = k * bs, b = bs < n - k0 ? bs : n - k0, r = n - k0 - b;
    float* d32 = w + k0 * ldw + k0;
    int e = launch_f32_to_f64(d32, 0, ldw, 1, d64, 0, bs, 1, b, b, 1, st);
    if (e) return ck(e, "convert diagonal block");
    bf_view dd{d64, 0, b, b, bs, 1};
    note_launch();
    set_identity_kernel<<<64, 256, 0, st>>>(x64, bs, b);
    bf_view xv{x64, 0, b, b, bs, 1};
    // the FP64 factor and X L11^T = I, the solve trailing the factor's inner steps
    e = g_mixed_inverse ? chol_then_inverse(dd, lv, nl, k0, xv, 512, d_info, st)
                        : chol_inverse_overlapped(dd, lv, nl, k0, xv, 512, d_info, st);
    if (e) return e;
    e = launch_f64_to_f32(d64, 0, bs, 1, d32, 0, ldw, 1, b, b, 1, st);
    if (e) return ck(e, "convert diagonal block");
    e = launch_f64_to_f32(x64, 0, bs, 1, xinv + k * bs * bs, 0, bs, 1, b, b, 0, st);
    if (e) return ck(e, "convert inverse");
    if (r == 0) return BF_OK;
    float* a21 = w + (k0 + b) * ldw + k0;
    void* p = pbuf[k & 1];
    if (tf32) {
      float* xtf = static_cast<float*>(xt);  // X^T in fp32
      e = launch_f64_to_f32(x64, 0, bs, 1, xtf, 0, 1, bs, b, b, 0, st);
      if (!e) e = launch_gemm_tf32_tc(1.0, a21, ldw, xtf, bs, 0.0, static_cast<float*>(p), 0, bs, 1, r, b, b, 0, st);
      if (e) return ck(e, "panel gemm (tf32)");
      return cudaMemcpy2DAsync(a21, size_t(ldw) * 4, p, size_t(bs) * 4, size_t(b) * 4, size_t(r),
                               cudaMemcpyDeviceToDevice, st) == cudaSuccess
                 ? BF_OK
                 : set_error(BF_ERR_CUDA, "panel copy");
    }
    e = launch_f64_to_bf16(x64, 0, bs, 1, xt, bs, b, b, 1, st);
    if (!e) e = launch_to_bf16(a21, 0, ldw, 1, p, bs, r, b, 0, st);
    if (!e) e = launch_gemm_bf16_tc(1.0, p, bs, xt, bs, 0.0, a21, 0, ldw, 1, r, b, b, 0, st);  // L21 = A21 X
    if (!e) e = launch_to_bf16(a21, 0, ldw, 1, p, bs, r, b, 0, st);
    return ck(e, "panel (bf16)");
  };
  auto tc_gemm = [&](const void* pa, const void* pb, float* c, int64_t m, int64_t nn, int64_t kk, int lower,
                     cudaStream_t st) {
    return tf32 ? launch_gemm_tf32_tc(-1.0, static_cast<const float*>(pa), bs, static_cast<const float*>(pb), bs, 1.0,
                                      c, 0, ldw, 1, m, nn, kk, lower, st)
                : launch_gemm_bf16_tc(-1.0, pa, bs, pb, bs, 1.0, c, 0, ldw, 1, m, nn, kk, lower, st);
  };
  cudaEvent_t ev_main, ev_side;
  cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming);
  const size_t esz = tf32 ? 4 : 2;
  if (lookahead) {
    cudaEventRecord(ev_main, main);
    cudaStreamWaitEvent(side, ev_main, 0);
  }
  rc = diag_and_panel(0, side);
  cudaEventRecord(ev_side, side);
  for (int64_t k = 0; k + 1 < nblk && !rc; ++k) {
    const int64_t k1 = (k + 1) * bs, r = n - k1, nb = bs < r ? bs : r;
    cudaStreamWaitEvent(main, ev_side, 0);
    const char* pk = static_cast<const char*>(pbuf[k & 1]);
    // (1) the next block column: W[k1:, k1:k1+nb] -= P P[:nb]^T
    rc = ck(tc_gemm(pk, pk, w + k1 * ldw + k1, r, nb, bs, 0, main), "column gemm");
    if (rc) break;
    if (lookahead) {
      cudaEventRecord(ev_main, main);
      cudaStreamWaitEvent(side, ev_main, 0);
    }
    // (2) panel k+1 on the side stream, (3) the rest of the trailing triangle
    // on the main stream, leaving g_mixed_reserve SMs to the side chain
    t_diag_ctas = lookahead && r > nb ? g_mixed_reserve : 0;  // a fused diagonal factor stays on those SMs
    rc = diag_and_panel(k + 1, side);
    t_diag_ctas = 0;
    cudaEventRecord(ev_side, side);
    if (!rc && r > nb) {
      const char* rest = pk + size_t(nb) * bs * esz;
      if (lookahead) t_reserve_sms = g_mixed_reserve;
      rc = ck(tc_gemm(rest, rest, w + (k1 + nb) * ldw + k1 + nb, r - nb, r - nb, bs, 1, main), "trailing gemmt");
      t_reserve_sms = 0;
    }
  }
  cudaStreamWaitEvent(main, ev_side, 0);
  cudaEventDestroy(ev_main);
  cudaEventDestroy(ev_side);
  return rc ? rc : (cudaGetLastError() == cudaSuccess ? BF_OK : set_error(BF_ERR_CUDA, "mixed factorization"));
}
}  // extern "C"
