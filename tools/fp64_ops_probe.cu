// Probe: FP64 CUDA-core throughput per instruction (DFMA vs DMUL vs DADD).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) a[i] = __fma_rn(a[i], b, c);
      if (OP == 1) a[i] = __dmul_rn(a[i], b);
      if (OP == 2) a[i] = __dadd_rn(a[i], c);
      if (OP == 3) a[i] = __dsub_rn(a[i], __dmul_rn(a[i], b));  // unfused mul-sub pair
      if (OP == 4) a[i] = __fma_rn(-1.0, __fma_rn(a[i], b, 0.0), a[i]);  // same via two DFMA
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"DFMA", "DMUL", "DADD", "DMUL+DSUB pair", "2xDFMA pair"};
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      int iters = 20000;
      cudaEventRecord(e0);
      if (op == 0) k<0><<<sms * 2, 256>>>(out, iters);
      if (op == 1) k<1><<<sms * 2, 256>>>(out, iters);
      if (op == 2) k<2><<<sms * 2, 256>>>(out, iters);
      if (op == 3) k<3><<<sms * 2, 256>>>(out, iters);
      if (op == 4) k<4><<<sms * 2, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = 16.0 * iters * sms * 2 * 256;
      if (rep) printf("%-16s %.1f G instr/s per GPU  (%.2f per SM per clk at 1.965 GHz)\n", names[op], ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
}
