// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA, register-only.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  // m16n8k16: A 8 regs, B 4 regs, C 4 regs per thread
  double acc[6][4];
#pragma unroll
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm) {
      int iters = 20000;
      int grid = sms * blocks_per_sm, threads = warps * 32;
      dmma_loop<0><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<0><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 16 * (double)iters * (grid * warps);
      printf("DMMA m8n8k4   warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", warps, blocks_per_sm, flops / ms / 1e9, ms);
      dmma16_loop<<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma16_loop<<<grid, threads>>>(out, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * 8 * 16 * 6 * (double)(iters / 4) * (grid * warps);
      printf("DMMA m16n8k16 warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", warps, blocks_per_sm, flops / ms / 1e9, ms);
      dfma_loop<<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, threads>>>(out, iters * 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * (double)(iters * 4) * (grid * threads);
      printf("DFMA          warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", warps, blocks_per_sm, flops / ms / 1e9, ms);
    }
  }
  // sustained: DMMA for ~3 s
  {
    int grid = sms * 2, threads = 256, iters = 20000;
    cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 3000) { dmma_loop<0><<<grid, threads>>>(out, iters); ++reps; cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
    double flops = 2.0 * 256 * 16 * (double)iters * (grid * 8) * reps;
    printf("DMMA sustained 3s: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
