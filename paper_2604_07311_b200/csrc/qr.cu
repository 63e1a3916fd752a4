// Householder QR on B200 (reference factor/qr.py), SURVEY.md §8(f) rank 4.
//
//  * qr_panel_kernel — the unblocked column sweep (qr.py:58-76) on an m x b
//    panel, one cooperative grid: per column the norm of the column below
//    the diagonal (grid reduction), beta / tau / scaling of the reflector,
//    then w = a(j, j+1:) + v^T a(j+1:, j+1:) (per-column grid reductions)
//    and the rank-1 update.  The reference computes these with NumPy/BLAS
//    (np.linalg.norm, @, np.outer), so the factor agrees to rounding.
//  * qr_t_kernel — the compact-WY T of a panel (qr.py:79-92), one CTA.
//  * explicit_v_kernel — V with its unit diagonal and zeros above (qr.py:95-100).
//  * reflector_apply_kernel — c := H_j c for one reflector (apply_q, qr.py:124-140).
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>

namespace bf {

namespace {

namespace cg = cooperative_groups;

constexpr int QR_THREADS = 256;
constexpr int QR_MAXB = 128;  // panel width handled by the cooperative stepper

template <typename T>
__global__ void __launch_bounds__(QR_THREADS) qr_panel_kernel(T* a, int64_t off, int64_t rs, int64_t cs, int64_t m,
                                                            int64_t b, T* taus, double* part) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, tid = threadIdx.x, cta = blockIdx.x;
  auto A = [&](int64_t i, int64_t j) -> T& { return a[off + i * rs + j * cs]; };
  __shared__ double red[QR_THREADS / 32][QR_MAXB + 1];
  __shared__ double s_w[QR_MAXB];
  __shared__ double s_rowj[QR_MAXB];
  __shared__ double s_beta, s_tau, s_scale;
  __shared__ int s_skip;
  const int64_t steps = m < b ? m : b;
  for (int64_t j = 0; j < steps; ++j) {
    // rows j .. m-1 split in contiguous bands
    const int64_t rows = m - j;
    const int64_t chunk = (rows + G - 1) / G;
    const int64_t r0 = j + int64_t(cta) * chunk, r1 = r0 + chunk < m ? r0 + chunk : m;
    // (1) ||a(j:, j)||^2 partials
    double ss = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += QR_THREADS) {
      const double v = double(A(i, j));
      ss = fma(v, v, ss);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
    if ((tid & 31) == 0) red[tid >> 5][0] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_THREADS / 32; ++w) t += red[w][0];
      part[cta] = t;
    }
    grid.sync();
    if (tid == 0) {
      double t = 0.0;
      for (int c = 0; c < G; ++c) t += part[c];
      const double nrm = sqrt(t);
      const double x0 = double(A(j, j));
      s_skip = nrm == 0.0;
      const double beta = -copysign(nrm, x0);
      s_beta = beta;
      s_tau = nrm == 0.0 ? 0.0 : (beta - x0) / beta;
      s_scale = x0 - beta;
      if (cta == 0) taus[j] = T(s_tau);
    }
    __syncthreads();
    if (s_skip) {
      grid.sync();
      continue;
    }
    // (2) scale the reflector below the diagonal; every CTA holds its own band
    const int64_t lo = r0 > j + 1 ? r0 : j + 1;
    for (int64_t i = lo + tid; i < r1; i += QR_THREADS) A(i, j) = T(double(A(i, j)) / s_scale);
    grid.sync();
    if (cta == 0 && tid == 0) A(j, j) = T(s_beta);
    // (3) w_c = a(j, c) + sum_{i>j} v_i a(i, c), c in (j, b)
    const int64_t nc = b - j - 1;
    if (nc > 0) {
      for (int64_t c0 = 0; c0 < nc; c0 += QR_MAXB) {
        const int64_t cn = nc - c0 < QR_MAXB ? nc - c0 : QR_MAXB;
        for (int64_t cc = 0; cc < cn; ++cc) {
          double acc = 0.0;
          for (int64_t i = lo + tid; i < r1; i += QR_THREADS)
            acc = fma(double(A(i, j)), double(A(i, j + 1 + c0 + cc)), acc);
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
          if ((tid & 31) == 0) red[tid >> 5][cc] = acc;
        }
        __syncthreads();
        for (int64_t cc = tid; cc < cn; cc += QR_THREADS) {
          double t = 0.0;
          for (int w = 0; w < QR_THREADS / 32; ++w) t += red[w][cc];
          part[int64_t(cta) * QR_MAXB + cc] = t;
          s_rowj[cc] = double(A(j, j + 1 + c0 + cc));  // read before CTA 0 may rewrite row j
        }
        grid.sync();
        for (int64_t cc = tid; cc < cn; cc += QR_THREADS) {
          double t = s_rowj[cc];
          for (int c = 0; c < G; ++c) t += part[int64_t(c) * QR_MAXB + cc];
          s_w[cc] = t;
        }
        __syncthreads();
        // (4) a(j, c) -= tau w_c ; a(i, c) -= tau v_i w_c
        const double tau = s_tau;
        if (cta == 0)
          for (int64_t cc = tid; cc < cn; cc += QR_THREADS) {
            const int64_t c = j + 1 + c0 + cc;
            A(j, c) = T(double(A(j, c)) - tau * s_w[cc]);
          }
        for (int64_t i = lo + tid; i < r1; i += QR_THREADS) {
          const double vi = double(A(i, j));
          for (int64_t cc = 0; cc < cn; ++cc) {
            const int64_t c = j + 1 + c0 + cc;
            A(i, c) = T(double(A(i, c)) - tau * vi * s_w[cc]);
          }
        }
        grid.sync();
      }
    } else {
      grid.sync();
    }
  }
}

// T (b x b, row-major ld b, upper): T[j,j] = tau_j, T[:j, j] = -tau_j T[:j,:j] (V[:, :j]^T v_j)
template <typename T>
__global__ void qr_t_kernel(const T* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, const T* taus,
                            T* t) {
  __shared__ double z[QR_MAXB];
  const int tid = threadIdx.x;
  auto V = [&](int64_t i, int64_t j) -> double {  // explicit unit-lower V of the panel
    return i == j ? 1.0 : (i > j ? double(a[off + i * rs + j * cs]) : 0.0);
  };
  for (int64_t e = tid; e < b * b; e += blockDim.x) t[e] = T(0);
  __syncthreads();
  for (int64_t j = 0; j < b; ++j) {
    const double tau = double(taus[j]);
    if (tid == 0) t[j * b + j] = T(tau);
    if (j > 0 && tau != 0.0) {
      // z_q = V[:, q]^T v_j over rows j.., q < j (warp per q)
      const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
      for (int64_t q = warp; q < j; q += nw) {
        double acc = 0.0;
        for (int64_t i = j + lane; i < m; i += 32) acc = fma(V(i, q), V(i, j), acc);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) z[q] = acc;
      }
      __syncthreads();
      for (int64_t r = tid; r < j; r += blockDim.x) {
        double acc = 0.0;
        for (int64_t q = r; q < j; ++q) acc = fma(double(t[r * b + q]), z[q], acc);
        t[r * b + j] = T(-tau * acc);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void explicit_v_kernel(const T* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, T* v) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * b) return;
  const int64_t i = e / b, j = e % b;
  v[e] = i == j ? T(1) : (i > j ? a[off + i * rs + j * cs] : T(0));
}

// c(j:, :) -= v w^T with w = tau v^T c(j:, :), v = (1, a(j+1:, j)); one column of c per thread
template <typename T>
__global__ void reflector_apply_kernel(const T* a, int64_t aoff, int64_t ars, int64_t acs, int64_t m, int64_t j,
                                       double tau, T* c, int64_t coff, int64_t crs, int64_t ccs, int64_t ncols) {
  const int64_t col = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double w = double(c[coff + j * crs + col * ccs]);
  for (int64_t i = j + 1; i < m; ++i) w = fma(double(a[aoff + i * ars + j * acs]), double(c[coff + i * crs + col * ccs]), w);
  w *= tau;
  c[coff + j * crs + col * ccs] = T(double(c[coff + j * crs + col * ccs]) - w);
  for (int64_t i = j + 1; i < m; ++i)
    c[coff + i * crs + col * ccs] = T(double(c[coff + i * crs + col * ccs]) - double(a[aoff + i * ars + j * acs]) * w);
}

}  // namespace

int launch_qr_panel(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, void* taus,
                    cudaStream_t s) {
  if (m <= 0 || b <= 0) return 0;
  static double* part[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!part[dev] && cudaMalloc(&part[dev], 32 * QR_MAXB * sizeof(double)) != cudaSuccess) return -12;
  int G = int((m + 511) / 512);
  if (G > 32) G = 32;
  if (G < 1) G = 1;
  double* pp = part[dev];
  note_launch();
  cudaError_t e;
  if (is_f64) {
    double* ad = static_cast<double*>(a);
    double* td = static_cast<double*>(taus);
    void* args[] = {&ad, &off, &rs, &cs, &m, &b, &td, &pp};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(qr_panel_kernel<double>), dim3(G), dim3(QR_THREADS), args,
                                    0, s);
  } else {
    float* af = static_cast<float*>(a);
    float* tf = static_cast<float*>(taus);
    void* args[] = {&af, &off, &rs, &cs, &m, &b, &tf, &pp};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(qr_panel_kernel<float>), dim3(G), dim3(QR_THREADS), args,
                                    0, s);
  }
  return e == cudaSuccess ? 0 : -11;
}

int launch_qr_t(int is_f64, const void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b,
                const void* taus, void* t, cudaStream_t s) {
  if (b <= 0) return 0;
  if (b > QR_MAXB) return -3;
  note_launch();
  if (is_f64)
    qr_t_kernel<double><<<1, 256, 0, s>>>(static_cast<const double*>(a), off, rs, cs, m, b,
                                          static_cast<const double*>(taus), static_cast<double*>(t));
  else
    qr_t_kernel<float><<<1, 256, 0, s>>>(static_cast<const float*>(a), off, rs, cs, m, b,
                                         static_cast<const float*>(taus), static_cast<float*>(t));
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_explicit_v(int is_f64, const void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, void* v,
                      cudaStream_t s) {
  if (m <= 0 || b <= 0) return 0;
  note_launch();
  const unsigned blocks = unsigned((m * b + 255) / 256);
  if (is_f64)
    explicit_v_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(a), off, rs, cs, m, b,
                                                     static_cast<double*>(v));
  else
    explicit_v_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(a), off, rs, cs, m, b,
                                                    static_cast<float*>(v));
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_reflector_apply(int is_f64, const void* a, int64_t aoff, int64_t ars, int64_t acs, int64_t m, int64_t j,
                           double tau, void* c, int64_t coff, int64_t crs, int64_t ccs, int64_t ncols,
                           cudaStream_t s) {
  if (ncols <= 0 || tau == 0.0) return 0;
  note_launch();
  const unsigned blocks = unsigned((ncols + 127) / 128);
  if (is_f64)
    reflector_apply_kernel<double><<<blocks, 128, 0, s>>>(static_cast<const double*>(a), aoff, ars, acs, m, j, tau,
                                                          static_cast<double*>(c), coff, crs, ccs, ncols);
  else
    reflector_apply_kernel<float><<<blocks, 128, 0, s>>>(static_cast<const float*>(a), aoff, ars, acs, m, j, tau,
                                                         static_cast<float*>(c), coff, crs, ccs, ncols);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
