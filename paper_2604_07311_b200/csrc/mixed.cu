// Kernels of the mixed-precision solve (BASELINE configs[3]): precision
// conversions, the FP64 residual r = b - A x, and the two triangular solves
// with the fp32 factor used by iterative refinement (fp64 right-hand sides).
// All memory-bound; they stream the matrix once per call.
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cuda_bf16.h>

namespace bf {

namespace {

__global__ void f64_to_f32_kernel(const double* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t doff,
                                  int64_t drs, int64_t dcs, int64_t m, int64_t n, int lower_only) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (lower_only && j > i) continue;
    dst[doff + i * drs + j * dcs] = float(src[soff + i * srs + j * scs]);
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

inline int grid_for_elems(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return int(b < 148 * 16 ? b : 148 * 16);
}

}  // namespace

int launch_f64_to_f32(const double* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t doff, int64_t drs,
                      int64_t dcs, int64_t m, int64_t n, int lower_only, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  f64_to_f32_kernel<<<grid_for_elems(m * n), 256, 0, s>>>(src, soff, srs, scs, dst, doff, drs, dcs, m, n, lower_only);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_residual(const double* A, int64_t lda, const double* x, const double* b, double* r, int64_t n,
                    cudaStream_t s) {
  if (n <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(A) % 16) || (lda % 2)) return -3;
  note_launch();
  residual_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, s>>>(A, lda, x, b, r, n);
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

}  // namespace bf
