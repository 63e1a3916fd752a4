// Probe: phase timing of the warp-per-8-rows fused TRSM (TrsmWarp) on a
// 128-column solve, clock64() per phase on warp 0 of CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2604_07311_b200/csrc \
//        tools/trsm_probe.cu -o tools/trsm_probe
#include "../paper_2604_07311_b200/csrc/small_kernels.cu"

#include <cstdio>
#include <vector>

namespace bf {
void note_launch(int64_t) {}
int g_use_tma = 1, g_tma_variant = 2, g_tiles_per_cta = 1, g_bf16_tma_c = 1;
}  // namespace bf

using namespace bf;

template <typename T>
__global__ void __launch_bounds__(128) probe(const T* t, T* b, int64_t m, int n, int64_t kc, long long* prof) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sl = reinterpret_cast<T*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* sx = sl + 128 * TW_LD;
  long long t0 = clock64();
  for (int j = warp; j < n; j += 4)
    for (int p = lane * (16 / sizeof(T)); p <= j; p += 32 * (16 / sizeof(T))) cp_async_16(&sl[j * TW_LD + p], &t[j * n + p], 16);
  const int64_t r0 = int64_t(blockIdx.x) * 32;
  for (int r = warp; r < 32; r += 4)
    for (int c = lane; c < n; c += 32) { if constexpr (sizeof(T) == 8) cp_async_8(&sx[c * TW_XLD + r], &b[(r0 + r) * n + c], 8); else cp_async_4(&sx[c * TW_XLD + r], &b[(r0 + r) * n + c], 4); }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  long long ts[12];
  int k = 0;
  ts[k++] = clock64();
  TrsmGroup<T> tw{sx, sl, lane, warp, 1, kc};
  tw.solve(0, n, 1.0);
  ts[k++] = clock64();
  for (int r = warp; r < 32; r += 4)
    for (int c = lane; c < n; c += 32) b[(r0 + r) * n + c] = sx[c * TW_XLD + r];
  ts[k++] = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    prof[0] = ts[0] - t0;
    for (int i = 1; i < k; ++i) prof[i] = ts[i] - ts[i - 1];
  }
}

template <typename T>
void run(const char* label) {
  const int n = 128, m = 1024;
  std::vector<T> ht(n * n, T(0)), hb(size_t(m) * n);
  for (int j = 0; j < n; ++j)
    for (int p = 0; p <= j; ++p) ht[j * n + p] = p == j ? T(2 + j % 3) : T(0.01) * T((j * 7 + p) % 11);
  for (auto& v : hb) v = T(1);
  T *dt, *db;
  long long* dp;
  cudaMalloc(&dt, ht.size() * sizeof(T));
  cudaMalloc(&db, hb.size() * sizeof(T));
  cudaMalloc(&dp, 64 * 8);
  cudaMemcpy(dt, ht.data(), ht.size() * sizeof(T), cudaMemcpyHostToDevice);
  const size_t smem = (128 * TW_LD + 128 * TW_XLD) * sizeof(T);
  cudaFuncSetAttribute(probe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const char* names[] = {"stage", "solve", "store", "-", "-", "-", "-", "-", "-"};
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(db, hb.data(), hb.size() * sizeof(T), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<T><<<m / 32, 128, smem>>>(dt, db, m, n, 128, dp);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long hp[9] = {0};
    cudaMemcpy(hp, dp, sizeof(hp), cudaMemcpyDeviceToHost);
    printf("%s rep %d: %.1f us |", label, rep, ms * 1e3);
    for (int i = 0; i < 9; ++i) printf(" %s=%lld", names[i], hp[i]);
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<float>("f32");
  run<double>("f64");
  return 0;
}
