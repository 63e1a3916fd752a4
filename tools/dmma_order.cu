// Probe: is DMMA (m8n8k4 / m16n8k4 / m16n8k16 f64) bit-identical to a sequential
// ascending-k fma chain c = fma(a_k, b_k, c)?  Decides whether the DMMA mainloop can
// reproduce the reference micro-kernel's summation (engine/kernels.py:153-162) bitwise.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k_m8n8k4(const double* A, const double* B, const double* C, double* D, int K) {
  // A 8xK row-major, B Kx8 (B[k][n]) , C/D 8x8
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1];
  for (int k0 = 0; k0 < K; k0 += 4) {
    double a = A[g * K + k0 + t];
    double b = B[(k0 + t) * 8 + g];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  }
  D[g * 8 + 2 * t] = c0; D[g * 8 + 2 * t + 1] = c1;
}

__global__ void k_m16n8k16(const double* A, const double* B, const double* C, double* D, int K) {
  // A 16xK, B Kx8, C/D 16x8
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;
  double c[4] = {C[g * 8 + 2 * t], C[g * 8 + 2 * t + 1], C[(g + 8) * 8 + 2 * t], C[(g + 8) * 8 + 2 * t + 1]};
  for (int k0 = 0; k0 < K; k0 += 16) {
    double a[8], b[4];
    // PTX ISA m16n8k16 .f64 A layout: a_i row = g + 8*(i%2), col = t + 4*(i/2)
    for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i % 2)) * K + k0 + t + 4 * (i / 2)];
    // B layout: b_i row = t + 4*i, col = g
    for (int i = 0; i < 4; ++i) b[i] = B[(k0 + t + 4 * i) * 8 + g];
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  D[g * 8 + 2 * t] = c[0]; D[g * 8 + 2 * t + 1] = c[1];
  D[(g + 8) * 8 + 2 * t] = c[2]; D[(g + 8) * 8 + 2 * t + 1] = c[3];
}

static double rnd() {
  double m = (double)rand() / RAND_MAX * 2 - 1;
  int e = rand() % 40 - 20;
  return ldexp(m, e);
}

int main() {
  const int K = 64;
  srand(1234);
  for (int variant = 0; variant < 2; ++variant) {
    int M = variant == 0 ? 8 : 16;
    size_t na = M * K, nb = K * 8, nc = M * 8;
    double *hA = new double[na], *hB = new double[nb], *hC = new double[nc], *hD = new double[nc];
    long mism_seq = 0, mism_pair = 0, mism_exact = 0, total = 0;
    for (int trial = 0; trial < 200; ++trial) {
      for (size_t i = 0; i < na; ++i) hA[i] = rnd();
      for (size_t i = 0; i < nb; ++i) hB[i] = rnd();
      for (size_t i = 0; i < nc; ++i) hC[i] = (trial % 2) ? rnd() : 0.0;
      double *dA, *dB, *dC, *dD;
      cudaMalloc(&dA, na * 8); cudaMalloc(&dB, nb * 8); cudaMalloc(&dC, nc * 8); cudaMalloc(&dD, nc * 8);
      cudaMemcpy(dA, hA, na * 8, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, nb * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(dC, hC, nc * 8, cudaMemcpyHostToDevice);
      if (variant == 0) k_m8n8k4<<<1, 32>>>(dA, dB, dC, dD, K); else k_m16n8k16<<<1, 32>>>(dA, dB, dC, dD, K);
      cudaMemcpy(hD, dD, nc * 8, cudaMemcpyDeviceToHost);
      cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dD);
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < 8; ++j) {
          double s = hC[i * 8 + j];
          for (int k = 0; k < K; ++k) s = fma(hA[i * K + k], hB[k * 8 + j], s);
          long double ex = hC[i * 8 + j];
          for (int k = 0; k < K; ++k) ex += (long double)hA[i * K + k] * hB[k * 8 + j];
          ++total;
          if (s != hD[i * 8 + j]) ++mism_seq;
          if ((double)ex != hD[i * 8 + j]) ++mism_exact;
        }
    }
    printf("%s: elements=%ld mismatches vs sequential-fma=%ld vs long-double-sum=%ld\n",
           variant == 0 ? "m8n8k4" : "m16n8k16", total, mism_seq, mism_exact);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
