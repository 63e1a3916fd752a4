#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0) {
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = __dsqrt_rn(x) + 1.0;
  long long t1 = clock64();
  double y = x0;
  for (int i = 0; i < 1000; ++i) y = __ddiv_rn(3.0, y) + 1.0;
  long long t2 = clock64();
  double z = x0;
  for (int i = 0; i < 1000; ++i) z = __fma_rn(z, 0.999, 0.5);
  long long t3 = clock64();
  double u = x0;
  for (int i = 0; i < 1000; ++i) u = __shfl_sync(0xffffffff, u, (threadIdx.x + 1) & 31) + 1.0;
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + u;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  for (int r = 0; r < 2; ++r) {
    lat<<<1, 32>>>(out, cyc, 2.5);
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("per-iteration latency (cycles): sqrt+add %.1f, div+add %.1f, dfma %.1f, shfl+add %.1f\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
  }
}
