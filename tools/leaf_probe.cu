// Probe: where does the 128x128 unblocked3 leaf spend its time?  A copy of
// potrf_leaf_v3_cols_kernel instrumented with clock64() per phase.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) leaf(double* g, int n, long long* prof) {
  __shared__ double colbuf[2][128];
  __shared__ int s_flag;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[8][4];
  for (int c = 0; c < 8; ++c)
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q, j = w + 16 * c;
      v[c][q] = (i < n && j <= i) ? g[i * n + j] : 0.0;
    }
  if (threadIdx.x == 0) s_flag = -1;
  __syncthreads();
  long long t_owner = 0, t_bar = 0, t_upd = 0;
  // pivot p on its owner warp: sqrt of (p,p), scale column p, publish it
  auto pivot = [&](int p) {
    const int cp = p >> 4, qp = p >> 5;
    double mine = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c == cp) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == qp) mine = v[c][q];
      }
    const double diag = __shfl_sync(0xffffffffu, mine, p & 31);
    if (!(diag > 0.0)) {
      if (lane == 0) s_flag = p;
      return;
    }
    const double d = __dsqrt_rn(diag);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c == cp) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q;
          if (i == p) v[c][q] = d;
          if (i > p) {
            const double x = __ddiv_rn(v[c][q], d);
            v[c][q] = x;
            colbuf[p & 1][i] = x;
          }
        }
      }
  };
  if (w == 0) pivot(0);
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    long long t0 = clock64();
    __syncthreads();  // column k published (or its pivot failed)
    if (s_flag >= 0) break;
    const int buf = k & 1;
    double ci[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ci[q] = colbuf[buf][lane + 32 * q];
    long long t1 = clock64();
    // the owner of column k+1 updates it first and runs pivot k+1 right away
    const int kn = k + 1;
    if (kn < n && w == (kn & 15)) {
      const int cn = kn >> 4;
      const double cj = colbuf[buf][kn];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c == cn) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (32 * q + 31 >= kn) {
              const double upd = __dsub_rn(v[c][q], __dmul_rn(ci[q], cj));
              v[c][q] = (lane + 32 * q >= kn) ? upd : v[c][q];
            }
        }
      pivot(kn);
    }
    long long t2 = clock64();
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = w + 16 * c;
      if (j > kn && j < n) {
        const double cj = colbuf[buf][j];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (32 * q + 31 >= j) {
            const double upd = __dsub_rn(v[c][q], __dmul_rn(ci[q], cj));
            if (32 * q >= j)
              v[c][q] = upd;
            else
              v[c][q] = (lane + 32 * q >= j) ? upd : v[c][q];
          }
        }
      }
    }
    long long t3 = clock64();
    t_bar += t1 - t0;
    t_owner += t2 - t1;
    t_upd += t3 - t2;
  }
  for (int c = 0; c < 8; ++c)
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q, j = w + 16 * c;
      if (i < n && j <= i) g[i * n + j] = v[c][q];
    }
  if (lane == 0) {
    prof[w * 3 + 0] = t_owner;
    prof[w * 3 + 1] = t_bar;
    prof[w * 3 + 2] = t_upd;
  }
}

int main() {
  const int n = 128;
  std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = (i == j) ? 2.0 * n : 1.0 / (1 + i + j);
  double* d;
  long long* prof;
  cudaMalloc(&d, n * n * 8);
  cudaMalloc(&prof, 16 * 3 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    leaf<<<1, 512>>>(d, n, prof);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long hp[48];
    cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost);
    printf("rep %d: %.1f us; per-warp cycles pivot/barrier+ld/update:", rep, ms * 1e3);
    for (int w = 0; w < 16; w += 5) printf(" w%d %lld/%lld/%lld", w, hp[w * 3], hp[w * 3 + 1], hp[w * 3 + 2]);
    printf("\n");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
