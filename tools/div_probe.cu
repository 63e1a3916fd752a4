// Probe: does the Markstein correction with a precomputed correctly rounded
// reciprocal reproduce IEEE division (div.rn) bit for bit in the safe range?
//   q0 = a*r, e = fma(-b, q0, a), q = fma(e, r, q0), r = rcp.rn(b)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

__global__ void check64(unsigned long long* bad, unsigned long long* tested, uint64_t seed, int iters, int mode) {
  uint64_t s = seed + (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
  unsigned long long nb = 0, nt = 0;
  for (int i = 0; i < iters; ++i) {
    s = mix(s + 1); const uint64_t u = s; s = mix(s + 1); const uint64_t v = s;
    double a, b;
    if (mode == 0) {  // random mantissas, exponents within +-40
      a = __longlong_as_double((long long)((u & 0x800FFFFFFFFFFFFFULL) | (uint64_t(1023 + int(u >> 52 & 63) - 32) << 52)));
      b = __longlong_as_double((long long)((v & 0x000FFFFFFFFFFFFFULL) | (uint64_t(1023 + int(v >> 52 & 63) - 32) << 52)));
    } else {  // near-integers / small-integer quotients (tie-prone)
      a = double(int64_t(u % 2000001) - 1000000) * (1.0 + double(v % 7) * 0x1p-52);
      b = double(int64_t(v % 1999) + 1) * (1.0 + double(u % 5) * 0x1p-52);
    }
    const double r = __drcp_rn(b);
    const double q0 = __dmul_rn(a, r);
    const double e = __fma_rn(-b, q0, a);
    const double q = __fma_rn(e, r, q0);
    const double ref = __ddiv_rn(a, b);
    ++nt;
    if (__double_as_longlong(q) != __double_as_longlong(ref)) ++nb;
  }
  atomicAdd(bad, nb);
  atomicAdd(tested, nt);
}

__global__ void check32(unsigned long long* bad, unsigned long long* tested, uint64_t seed, int iters, int mode) {
  uint64_t s = seed + (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
  unsigned long long nb = 0, nt = 0;
  for (int i = 0; i < iters; ++i) {
    s = mix(s + 1); const uint64_t u = s; s = mix(s + 1); const uint64_t v = s;
    float a, b;
    if (mode == 0) {
      a = __int_as_float(int((uint32_t(u) & 0x807FFFFFu) | (uint32_t(127 + int(u >> 40 & 31) - 16) << 23)));
      b = __int_as_float(int((uint32_t(v) & 0x007FFFFFu) | (uint32_t(127 + int(v >> 40 & 31) - 16) << 23)));
    } else {
      a = float(int(u % 20001) - 10000) * (1.0f + float(v % 7) * 0x1p-23f);
      b = float(int(v % 199) + 1) * (1.0f + float(u % 5) * 0x1p-23f);
    }
    const float r = __frcp_rn(b);
    const float q0 = __fmul_rn(a, r);
    const float e = __fmaf_rn(-b, q0, a);
    const float q = __fmaf_rn(e, r, q0);
    const float ref = __fdiv_rn(a, b);
    ++nt;
    if (__float_as_int(q) != __float_as_int(ref)) ++nb;
  }
  atomicAdd(bad, nb);
  atomicAdd(tested, nt);
}

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, 16);
    check64<<<148 * 8, 256>>>(d, d + 1, 12345 + mode, 4096, mode);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("f64 mode %d: %llu mismatches of %llu\n", mode, h[0], h[1]);
    cudaMemset(d, 0, 16);
    check32<<<148 * 8, 256>>>(d, d + 1, 777 + mode, 4096, mode);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("f32 mode %d: %llu mismatches of %llu\n", mode, h[0], h[1]);
  }
  return 0;
}
