// Probe: the leaf's pivot chain with ONE Newton step on the rsqrt seed
// (sqrt = d*y + residual correction; quotient by Markstein seeded with y)
// against sqrt.rn / div.rn, bit for bit, on random operands in the leaf's
// exponent band.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/sqrt_probe1.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
template <int ITERS>
__device__ __forceinline__ double sqrt_y(double d, double& yo) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const double h = 0.5 * y;
    const double r = fma(-d * y, h, 0.5);
    y = fma(y, r, y);
  }
  const double s = d * y;
  const double h = 0.5 * y;
  yo = y;
  return fma(fma(-s, s, d), h, s);
}
template <int ITERS>
__global__ void probe(uint64_t seed, int per_thread, unsigned long long* bad) {
  unsigned long long bs = 0, bq = 0;
  uint64_t st = seed ^ (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < per_thread; ++i) {
    st = mix(st + 0x632be59bd9b4e019ULL);
    const int e = int(st % 1000) - 500;  // exponent spread inside the band
    const double d = ldexp(1.0 + double(st >> 12) * 0x1p-52, e);
    double y;
    const double s = sqrt_y<ITERS>(d, y);
    bs += s != __dsqrt_rn(d);
    const uint64_t t2 = mix(st);
    const double a = ldexp(1.0 + double(t2 >> 12) * 0x1p-52, int(t2 % 800) - 400) * ((t2 & 1) ? -1.0 : 1.0);
    const double q0 = a * y;
    const double q = fma(fma(-s, q0, a), y, q0);
    bq += q != __ddiv_rn(a, s);
  }
  atomicAdd(bad, bs);
  atomicAdd(bad + 1, bq);
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  for (int iters = 1; iters <= 2; ++iters) {
    cudaMemset(d, 0, 32);
    const int blocks = 1184, threads = 256, per = 4096;  // ~1.24e9 samples
    if (iters == 1) probe<1><<<blocks, threads>>>(12345, per, d); else probe<2><<<blocks, threads>>>(12345, per, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("newton steps %d: %.3g samples, sqrt mismatches %llu, quotient mismatches %llu\n", iters,
           double(blocks) * threads * per, h[0], h[1]);
  }
  return 0;
}
