// Householder QR on B200 (reference factor/qr.py), SURVEY.md §8(f) rank 4.
//
//  * qr_panel_kernel — the unblocked column sweep (qr.py:58-76) on an m x b
//    panel, one cooperative grid: per column the norm of the column below
//    the diagonal (grid reduction), beta / tau / scaling of the reflector,
//    then w = a(j, j+1:) + v^T a(j+1:, j+1:) (per-column grid reductions)
//    and the rank-1 update.  The reference computes these with NumPy/BLAS
//    (np.linalg.norm, @, np.outer), so the factor agrees to rounding.
//  * qr_t_kernel — the compact-WY T of a panel (qr.py:79-92) from the
//    panel's Gram matrix V^T V (one engine GEMM), one CTA.
//  * explicit_v_kernel — V with its unit diagonal and zeros above (qr.py:95-100).
//  * reflector_apply_kernel — c := H_j c for one reflector (apply_q, qr.py:124-140).
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>

namespace bf {

int g_qr_global = 0;  // 1: the global-memory panel sweep only (tests / A-B)

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
  __shared__ double s_w[QR_THREADS];
  __shared__ double s_rowj[QR_THREADS];
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
    // (3) w_c = a(j, c) + sum_{i>j} v_i a(i, c), c in (j, b): one thread per
    // column (coalesced along the row), rows of this band in a loop
    const int64_t nc = b - j - 1;
    for (int64_t c0 = 0; c0 < nc; c0 += QR_THREADS) {
      const int64_t cn = nc - c0 < QR_THREADS ? nc - c0 : QR_THREADS;
      const int64_t c = j + 1 + c0 + tid;
      if (tid < cn) {
        double acc = 0.0;
#pragma unroll 4
        for (int64_t i = lo; i < r1; ++i) acc = fma(double(A(i, j)), double(A(i, c)), acc);
        part[int64_t(cta) * QR_THREADS + tid] = acc;
        s_rowj[tid] = double(A(j, c));  // read before CTA 0 may rewrite row j
      }
      grid.sync();
      if (tid < cn) {
        double t = s_rowj[tid];
        for (int q = 0; q < G; ++q) t += part[int64_t(q) * QR_THREADS + tid];
        s_w[tid] = t;
      }
      // (4) a(j, c) -= tau w_c ; a(i, c) -= tau v_i w_c
      const double tau = s_tau;
      if (tid < cn) {
        const double wc = s_w[tid];
        if (cta == 0) A(j, c) = T(double(A(j, c)) - tau * wc);
#pragma unroll 4
        for (int64_t i = lo; i < r1; ++i) A(i, c) = T(double(A(i, c)) - tau * double(A(i, j)) * wc);
      }
      grid.sync();
    }
    if (nc <= 0) grid.sync();
  }
}

// The same sweep with every CTA's row band of the panel resident in shared
// memory (static bands of `chunk` rows) and ONE grid barrier per column:
// before the barrier each CTA publishes, for the coming column j, the raw
// partial dots u_c = sum_{i>j} a(i,j) a(i,c), c >= j, over its band (u_j is
// the norm's tail), and the owner of row j publishes a(j, j:).  After it,
// every CTA derives beta/tau/scale from the same sums and forms
// w_c = a(j,c) + u_c / scale (= a(j,c) + v^T a(j+1:, c) with v = a(j+1:,j) /
// scale), scales its part of the reflector, applies the rank-1 update to its
// rows and publishes the partials of column j+1.  Partial sums are combined
// in CTA order (identical in every CTA); buffers alternate by column parity.
template <typename T>
__global__ void __launch_bounds__(QR_THREADS) qr_panel_smem_kernel(T* a, int64_t off, int64_t rs, int64_t cs,
                                                                 int64_t m, int64_t b, T* taus, double* part,
                                                                 double* rowbuf, int chunk) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char qr_smem[];
  T* S = reinterpret_cast<T*>(qr_smem);  // chunk x b, row-major
  const int G = gridDim.x, tid = threadIdx.x, cta = blockIdx.x;
  const int64_t R0 = int64_t(cta) * chunk;
  const int64_t R1 = R0 + chunk < m ? R0 + chunk : m;
  const int nr = R1 > R0 ? int(R1 - R0) : 0;
  const int bb = int(b);
  const int cc = tid & (QR_MAXB - 1), half = tid >> 7;
  __shared__ double s_u[QR_MAXB];
  __shared__ double s_row[QR_MAXB];
  __shared__ double s_half[QR_MAXB];
  __shared__ double s_beta, s_tau, s_scale;
  __shared__ int s_skip;
  for (int e = tid; e < nr * bb; e += QR_THREADS) {
    const int r = e / bb, c = e - r * bb;
    S[e] = a[off + (R0 + r) * rs + int64_t(c) * cs];
  }
  __syncthreads();
  // partials of column j: u_c over band rows i > j, c in [j, b); row j if owned
  auto publish = [&](int64_t j) {
    const int par = int(j & 1);
    const int nc = bb - int(j);
    const int64_t lo = R0 > j + 1 ? R0 : j + 1;
    double acc = 0.0;
    if (cc < nc)
      for (int64_t i = lo + half; i < R1; i += 2) {
        const T* row = S + (i - R0) * bb;
        acc = fma(double(row[j]), double(row[j + cc]), acc);
      }
    if (half) s_half[cc] = acc;
    __syncthreads();
    if (!half && cc < nc) part[(int64_t(par) * 160 + cta) * QR_MAXB + cc] = acc + s_half[cc];
    if (j >= R0 && j < R1 && half && cc < nc) rowbuf[par * QR_MAXB + cc] = double(S[(j - R0) * bb + j + cc]);
  };
  const int64_t steps = m < b ? m : b;
  if (steps > 0) publish(0);
  grid.sync();
  for (int64_t j = 0; j < steps; ++j) {
    const int par = int(j & 1);
    const int nc = bb - int(j);
    {
      double t = 0.0;
      if (cc < nc)
        for (int q0 = half; q0 < G; q0 += 32) {  // 16 independent loads in flight, summed in order
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int q = q0 + 2 * u;
            v[u] = q < G ? __ldcg(part + (int64_t(par) * 160 + q) * QR_MAXB + cc) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) t += v[u];
        }
      if (half) s_half[cc] = t;
      else if (cc < nc) s_row[cc] = __ldcg(rowbuf + par * QR_MAXB + cc);
      __syncthreads();
      if (!half && cc < nc) s_u[cc] = t + s_half[cc];
      __syncthreads();
    }
    if (tid == 0) {
      const double x0 = s_row[0];
      const double nrm = sqrt(fma(x0, x0, s_u[0]));
      s_skip = nrm == 0.0;
      const double beta = -copysign(nrm, x0);
      s_beta = beta;
      s_tau = nrm == 0.0 ? 0.0 : (beta - x0) / beta;
      s_scale = x0 - beta;
      if (cta == 0) taus[j] = T(s_tau);
    }
    __syncthreads();
    if (!s_skip) {
      const double scale = s_scale, tau = s_tau;
      // the reflector below the diagonal (own rows), beta on the diagonal
      for (int64_t i = (R0 > j + 1 ? R0 : j + 1) + tid; i < R1; i += QR_THREADS) {
        T& x = S[(i - R0) * bb + j];
        x = T(double(x) / scale);
      }
      __syncthreads();
      if (cc >= 1 && cc < nc) {
        const int64_t c = j + cc;
        const double wc = s_row[cc] + s_u[cc] / scale;
        if (half == 0 && j >= R0 && j < R1) {
          T& x = S[(j - R0) * bb + c];
          x = T(double(x) - tau * wc);
        }
        for (int64_t i = (R0 > j + 1 ? R0 : j + 1) + half; i < R1; i += 2) {
          T* row = S + (i - R0) * bb;
          row[c] = T(double(row[c]) - tau * double(row[j]) * wc);
        }
      }
      if (tid == 0 && j >= R0 && j < R1) S[(j - R0) * bb + j] = T(s_beta);
      __syncthreads();
    }
    if (j + 1 < steps) publish(j + 1);
    grid.sync();
  }
  __syncthreads();
  for (int e = tid; e < nr * bb; e += QR_THREADS) {
    const int r = e / bb, c = e - r * bb;
    a[off + (R0 + r) * rs + int64_t(c) * cs] = S[e];
  }
}

// T (b x b, row-major ld b, upper) of the compact-WY form I - V T V^T
// (qr.py:79-92 builds it column by column: T[:j, j] = -tau_j T[:j,:j] V^T v_j).
// Here the same T is formed recursively from G = V^T V (one split-K GEMM):
// 32-column leaves run that column recursion (one warp each, lane per row),
// then T12 = -T11 G12 T22 merges blocks pairwise (equal to the column
// recursion up to rounding).  T and the G blocks live in shared memory.
constexpr int QT_LEAF = 32;
constexpr int QT_XLD = 65;

template <typename T>
__global__ void __launch_bounds__(256) qr_t_kernel(const T* gram, int64_t b, const T* taus, T* t) {
  extern __shared__ __align__(16) unsigned char qt_smem[];
  const int bb = int(b), ld = bb + 1;
  double* Ts = reinterpret_cast<double*>(qt_smem);  // b x (b + 1)
  double* X = Ts + bb * ld;                         // 64 x 65 scratch (leaf G blocks, then G12 T22)
  double* G12 = X + 4 * QT_LEAF * 33;               // 64 x 65: the off-diagonal G block of a merge
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < bb * ld; e += blockDim.x) Ts[e] = 0.0;
  // leaf diagonal blocks of G, leaf w at X + w * 32 * 33
  const int nleaf = (bb + QT_LEAF - 1) / QT_LEAF;
  for (int e = tid; e < nleaf * QT_LEAF * QT_LEAF; e += blockDim.x) {
    const int w = e / (QT_LEAF * QT_LEAF), q = (e / QT_LEAF) % QT_LEAF, c = e % QT_LEAF;
    const int r0 = w * QT_LEAF;
    X[w * QT_LEAF * 33 + q * 33 + c] = (r0 + q < bb && r0 + c < bb) ? double(gram[int64_t(r0 + q) * b + r0 + c]) : 0.0;
  }
  __syncthreads();
  if (warp < nleaf) {
    const int r0 = warp * QT_LEAF, sz = bb - r0 < QT_LEAF ? bb - r0 : QT_LEAF;
    const double* Gl = X + warp * QT_LEAF * 33;
    for (int jj = 0; jj < sz; ++jj) {
      const double tau = double(taus[r0 + jj]);
      if (lane == jj) Ts[(r0 + jj) * ld + r0 + jj] = tau;
      if (lane < jj && tau != 0.0) {
        double acc = 0.0;
        for (int q = lane; q < jj; ++q) acc = fma(Ts[(r0 + lane) * ld + r0 + q], Gl[q * 33 + jj], acc);
        Ts[(r0 + lane) * ld + r0 + jj] = -tau * acc;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int sz = QT_LEAF; sz < bb; sz *= 2)
    for (int r0 = 0; r0 + sz < bb; r0 += 2 * sz) {
      const int s1 = sz, s2 = bb - r0 - sz < sz ? bb - r0 - sz : sz, c0 = r0 + s1;
      for (int e = tid; e < s1 * s2; e += blockDim.x) {
        const int q = e / s2, c = e % s2;
        G12[q * QT_XLD + c] = double(gram[int64_t(r0 + q) * b + c0 + c]);
      }
      __syncthreads();
      // X = G12 T22  (T22 upper: p <= c)
      for (int e = tid; e < s1 * s2; e += blockDim.x) {
        const int q = e / s2, c = e % s2;
        double acc = 0.0;
        for (int p = 0; p <= c; ++p) acc = fma(G12[q * QT_XLD + p], Ts[(c0 + p) * ld + c0 + c], acc);
        X[q * QT_XLD + c] = acc;
      }
      __syncthreads();
      // T12 = -T11 X  (T11 upper: p >= q)
      for (int e = tid; e < s1 * s2; e += blockDim.x) {
        const int q = e / s2, c = e % s2;
        double acc = 0.0;
        for (int p = q; p < s1; ++p) acc = fma(Ts[(r0 + q) * ld + r0 + p], X[p * QT_XLD + c], acc);
        Ts[(r0 + q) * ld + c0 + c] = -acc;
      }
      __syncthreads();
    }
  for (int e = tid; e < bb * bb; e += blockDim.x) t[e] = T(Ts[(e / bb) * ld + e % bb]);
}

// c = alpha * sum_s ws[s] + beta * c, slices summed in order (split-K GEMM)
template <typename T>
__global__ void splitk_reduce_kernel(const T* ws, int S, int64_t m, int64_t n, double alpha, double beta, T* c,
                                     int64_t off, int64_t rs, int64_t cs) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e / n, j = e - i * n;
  double acc = 0.0;
  for (int q = 0; q < S; ++q) acc += double(ws[int64_t(q) * m * n + e]);
  T& x = c[off + i * rs + j * cs];
  x = T(beta == 0.0 ? alpha * acc : alpha * acc + beta * double(x));
}

// The reference's kc folds applied in order to per-segment sums computed in
// parallel (engine/gemm.py:124-126, engine/kernels.py:228-253): ws[s] holds the
// exact fma-chain sum t_s of segment s (written as 1.0 * t_s, no rounding);
// c = beta_eff*c + alpha*t_s for s = 0, 1, ... with beta_eff = beta then 1,
// each product and sum rounded like the GEMM kernels' fold.  lower_only keeps
// i >= j; a set abort flag (below the limit) skips the whole fold.
__global__ void segfold_kernel(const double* ws, int S, int64_t m, int64_t n, double alpha, double beta, double* c,
                               int64_t off, int64_t rs, int64_t cs, int lower_only, const int* abort_flag,
                               int64_t abort_limit) {
  if (abort_flag != nullptr && *abort_flag >= 0 && *abort_flag < abort_limit) return;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e / n, j = e - i * n;
  if (lower_only && j > i) return;
  double& x = c[off + i * rs + j * cs];
  double v = __dmul_rn(alpha, ws[e]);
  if (beta != 0.0) v = __dadd_rn(__dmul_rn(beta, x), v);
  for (int q = 1; q < S; ++q) v = __dadd_rn(v, __dmul_rn(alpha, ws[int64_t(q) * m * n + e]));
  x = v;
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
  // 2 x (160 x 128) dot partials (by column parity) + 2 x 128 published rows
  if (!part[dev] && cudaMalloc(&part[dev], (2 * 160 * QR_MAXB + 2 * QR_MAXB) * sizeof(double)) != cudaSuccess)
    return -12;
  double* pp = part[dev];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t esz = is_f64 ? sizeof(double) : sizeof(float);
  if (!g_qr_global && b <= QR_MAXB) {
    // resident bands of ~128 rows (fewer, taller bands once the grid is full)
    int G = int((m + 127) / 128);
    if (G > sms) G = sms;
    if (G > 160) G = 160;
    if (G < 1) G = 1;
    int chunk = int((m + G - 1) / G);
    const size_t smem = size_t(chunk) * size_t(b) * esz;
    if (smem <= 200 * 1024) {
      double* rb = pp + 2 * 160 * QR_MAXB;
      note_launch();
      cudaError_t e;
      if (is_f64) {
        auto k = qr_panel_smem_kernel<double>;
        smem_attr(reinterpret_cast<const void*>(k), 200 * 1024);
        double* ad = static_cast<double*>(a);
        double* td = static_cast<double*>(taus);
        void* args[] = {&ad, &off, &rs, &cs, &m, &b, &td, &pp, &rb, &chunk};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k), dim3(G), dim3(QR_THREADS), args, smem, s);
      } else {
        auto k = qr_panel_smem_kernel<float>;
        smem_attr(reinterpret_cast<const void*>(k), 200 * 1024);
        float* af = static_cast<float*>(a);
        float* tf = static_cast<float*>(taus);
        void* args[] = {&af, &off, &rs, &cs, &m, &b, &tf, &pp, &rb, &chunk};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k), dim3(G), dim3(QR_THREADS), args, smem, s);
      }
      return e == cudaSuccess ? 0 : -11;
    }
  }
  // ~64 rows per CTA: the column loops are latency-bound, so spread them
  int G = int((m + 63) / 64);
  if (G > 128) G = 128;
  if (G < 1) G = 1;
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

int launch_qr_t(int is_f64, const void* gram, int64_t b, const void* taus, void* t, cudaStream_t s) {
  if (b <= 0) return 0;
  if (b > QR_MAXB) return -3;
  const size_t smem = size_t(b * (b + 1) + 4 * QT_LEAF * 33 + 64 * QT_XLD) * sizeof(double);
  note_launch();
  if (is_f64) {
    smem_attr(reinterpret_cast<const void*>(qr_t_kernel<double>), 220 * 1024);
    qr_t_kernel<double><<<1, 256, smem, s>>>(static_cast<const double*>(gram), b, static_cast<const double*>(taus),
                                             static_cast<double*>(t));
  } else {
    smem_attr(reinterpret_cast<const void*>(qr_t_kernel<float>), 220 * 1024);
    qr_t_kernel<float><<<1, 256, smem, s>>>(static_cast<const float*>(gram), b, static_cast<const float*>(taus),
                                            static_cast<float*>(t));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_splitk_reduce(int is_f64, const void* ws, int S, int64_t m, int64_t n, double alpha, double beta, void* c,
                         int64_t off, int64_t rs, int64_t cs, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  const unsigned blocks = unsigned((m * n + 255) / 256);
  if (is_f64)
    splitk_reduce_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(ws), S, m, n, alpha, beta,
                                                        static_cast<double*>(c), off, rs, cs);
  else
    splitk_reduce_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(ws), S, m, n, alpha, beta,
                                                       static_cast<float*>(c), off, rs, cs);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_segfold(const double* ws, int S, int64_t m, int64_t n, double alpha, double beta, double* c, int64_t off,
                   int64_t rs, int64_t cs, int lower_only, const int* abort_flag, int64_t abort_limit,
                   cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  segfold_kernel<<<unsigned((m * n + 255) / 256), 256, 0, s>>>(ws, S, m, n, alpha, beta, c, off, rs, cs, lower_only,
                                                               abort_flag, abort_limit);
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
