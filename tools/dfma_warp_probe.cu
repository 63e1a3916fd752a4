// Probe: single-warp DFMA / F2F throughput with C independent chains (one warp per CTA, one CTA).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void dfma_chains(double* out, long long* cyc, int iters, double a) {
  double t[C];
#pragma unroll
  for (int c = 0; c < C; ++c) t[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) t[c] = fma(t[c], a, 1e-9);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += t[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
__global__ void f2f_chains(double* out, long long* cyc, int iters, float a) {
  double t[C];
  float x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { t[c] = 0; x[c] = threadIdx.x * 1e-3f + c; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) { x[c] = __fmul_rn(x[c], a); t[c] = __dadd_rn(t[c], double(x[c])); }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += t[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  long long h;
#define RUN(K, C, W)                                                                         \
  K<C><<<1, W>>>(out, cyc, iters, 1.0000001);                                                \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                            \
  printf(#K " chains=%d warps=%d: %.2f cycles per warp-instr (per chain-step %.2f)\n", C, W / 32, \
         double(h) / (double(iters) * C), double(h) / iters);
  RUN(dfma_chains, 1, 32) RUN(dfma_chains, 8, 32) RUN(dfma_chains, 16, 32) RUN(dfma_chains, 32, 32)
  RUN(dfma_chains, 8, 128) RUN(dfma_chains, 16, 128)
  RUN(f2f_chains, 8, 32) RUN(f2f_chains, 16, 32) RUN(f2f_chains, 8, 128)
  return 0;
}
