// Probe: phase clocks of the blocked variant-3 leaf (potrf_leaf_blocked_kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLV4_PROF -I paper_2604_07311_b200/csrc \
//        -I include tools/leaf_probe2.cu -o tools/leaf_probe2
#include "../paper_2604_07311_b200/csrc/small_kernels.cu"

#include <cstdio>
#include <vector>

namespace bf {
void note_launch(int64_t) {}
bool smem_attr(const void* k, int b) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, b) == cudaSuccess;
}
int g_use_tma = 1, g_tma_variant = 2, g_tiles_per_cta = 1, g_bf16_tma_c = 1;
}  // namespace bf
using namespace bf;
static int g_pipe = 1;

template <typename T>
void run(const char* label) {
  const int n = 128;
  std::vector<T> h(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? T(n) : T(0)) + T(0.5) / T(1 + (i > j ? i - j : j - i));
  T* d;
  cudaMalloc(&d, h.size() * sizeof(T));
  const size_t smem = size_t(128) * LV4_LD * sizeof(T);
  cudaFuncSetAttribute(potrf_leaf_blocked_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    long long z[64] = {0};
    cudaMemcpyToSymbol(g_lv4_prof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    potrf_leaf_blocked_kernel<T><<<1, 128, smem>>>(d, 0, n, n, 1, 0, nullptr, g_pipe);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long hp[64];
    cudaMemcpyFromSymbol(hp, g_lv4_prof, sizeof(hp));
    printf("%s rep %d: %.1f us | (a,b,c) per block:", label, rep, ms * 1e3);
    for (int k = 0; k < 4; ++k) printf("  [%lld %lld %lld]", hp[1 + 3 * k] - (k ? hp[3 * k] : hp[0]), hp[2 + 3 * k] - hp[1 + 3 * k], hp[3 + 3 * k] - hp[2 + 3 * k]);
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
}

int main(int argc, char** argv) {
  if (argc > 1) g_pipe = atoi(argv[1]);
  run<float>("f32");
  run<double>("f64");
  return 0;
}
