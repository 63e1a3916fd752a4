// Probe: branch-free sqrt / reciprocal / division sequences (MUFU seed +
// Newton + one Markstein-style correction) against sqrt.rn / rcp.rn / div.rn,
// bit for bit, on random operands inside the exponent band the leaf checks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// sqrt: y ~ 1/sqrt(d) refined twice, s = d*y, correction with the residual
__device__ __forceinline__ double fast_sqrt(double d) {
  double y = rsqrt_approx(d);
  double h = 0.5 * y;
  double r = fma(-d * y, h, 0.5);  // 0.5 - d*y*y/2
  y = fma(y, r, y);
  h = 0.5 * y;
  r = fma(-d * y, h, 0.5);
  y = fma(y, r, y);
  double s = d * y;
  h = 0.5 * y;
  double e = fma(-s, s, d);
  return fma(e, h, s);
}
__device__ __forceinline__ double fast_rcp(double b) {
  double y = rcp_approx(b);
  double e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  return fma(y, e, y);
}
// sqrt that also returns its refined y ~ 1/sqrt(d), and a reciprocal of the
// rounded sqrt seeded from that y (two Newton steps)
__device__ __forceinline__ double fast_sqrt_y(double d, double& yo) {
  double y = rsqrt_approx(d);
  double h = 0.5 * y;
  double r = fma(-d * y, h, 0.5);
  y = fma(y, r, y);
  h = 0.5 * y;
  r = fma(-d * y, h, 0.5);
  y = fma(y, r, y);
  double s = d * y;
  h = 0.5 * y;
  double e = fma(-s, s, d);
  yo = y;
  return fma(e, h, s);
}
__device__ __forceinline__ double rcp_seeded(double b, double y) {
  double e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double fast_div(double a, double b, double r) {
  const double q0 = a * r;
  return fma(fma(-b, q0, a), r, q0);
}

__global__ void check(unsigned long long* cnt, uint64_t seed, int iters) {
  uint64_t s = seed + (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
  unsigned long long bs = 0, br = 0, bd = 0, bdd = 0, nt = 0;
  for (int i = 0; i < iters; ++i) {
    s = mix(s + 1); const uint64_t u = s; s = mix(s + 1); uint64_t v = s;
    if (i & 1) {  // exact squares and their neighbours: d = x*x with x of <= 26 significant bits, +-1 ulp
      const double x = __longlong_as_double((long long)(((v >> 12) & 0x000FFFFFFC000000ULL) | (uint64_t(1023 + int(v >> 52 & 255) - 128) << 52)));
      const double sqv = x * x;
      const long long bits = __double_as_longlong(sqv) + (long long)(int(u & 3) - 1);
      v = (uint64_t)bits;
    }
    // exponents within +-300 of 1
    const double a = __longlong_as_double((long long)((u & 0x800FFFFFFFFFFFFFULL) | (uint64_t(1023 + int(u >> 52 & 511) - 256) << 52)));
    const double d = (i & 1) ? __longlong_as_double((long long)v)
                             : __longlong_as_double((long long)((v & 0x000FFFFFFFFFFFFFULL) | (uint64_t(1023 + int(v >> 52 & 511) - 256) << 52)));
    ++nt;
    const double sq = fast_sqrt(d);
    if (__double_as_longlong(sq) != __double_as_longlong(__dsqrt_rn(d))) ++bs;
    const double r = fast_rcp(d);
    if (__double_as_longlong(r) != __double_as_longlong(__drcp_rn(d))) ++br;
    const double q = fast_div(a, d, r);
    if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, d))) ++bd;
    // the leaf's pattern: divide by a freshly rounded sqrt, reciprocal seeded by the sqrt's y
    double y;
    const double sq2 = fast_sqrt_y(d, y);
    const double rs = rcp_seeded(sq2, y);
    if (__double_as_longlong(rs) != __double_as_longlong(__drcp_rn(__dsqrt_rn(d)))) ++bdd;
    if (__double_as_longlong(fast_div(a, sq2, rs)) != __double_as_longlong(__ddiv_rn(a, __dsqrt_rn(d)))) ++bd;
  }
  atomicAdd(cnt + 0, bs);
  atomicAdd(cnt + 1, br);
  atomicAdd(cnt + 2, bd);
  atomicAdd(cnt + 3, bdd);
  atomicAdd(cnt + 4, nt);
}

int main() {
  unsigned long long *d, h[5];
  cudaMalloc(&d, 40);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 40);
    check<<<148 * 8, 256>>>(d, 99 + rep, 4096);
    cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("tested %llu: sqrt mismatches %llu, rcp(MUFU+3) %llu, divs %llu, rcp(sqrt-seeded) %llu  (%s)\n", h[4], h[0], h[1], h[2],
           h[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
