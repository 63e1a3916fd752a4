// Operand staging for permuted tensor contractions (sm_100a).
//
// The reference packs every operand micro-panel through its block-scatter
// vectors before the micro-kernel (engine/kernels.py:24-90 pack_a_block /
// pack_b_block).  The GEMM kernels here gather straight from the facade while
// filling shared memory, which costs one 8-byte cp.async per element; when a
// contraction is large and a facade is not a strided matrix (a permuted
// layout such as aibj,cjdi->abcd), one HBM pass that lays the operand out
// k-contiguous lets the TMA DMMA kernel take it instead.  Copying values is
// exact and the k order is the facade's column order, so the GEMM's bits do
// not change (tests/test_gpu_parity.py::test_contraction_staged_*).
//
//   out[r * cols + c] = src[row_scat[r] + col_scat[c]]
//
// Writes are coalesced along c; col_scat is read coalesced and stays in L2
// across rows; the source reads are whatever the permutation makes them (the
// pass is HBM-bound and small next to the GEMM it feeds: 2 GB vs 8.8 TFLOP at
// the BASELINE's d=128).
#include "bf_common.cuh"
#include "bf_internal.h"

namespace bf {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) pack_scatter_kernel(const T* __restrict__ src, const int64_t* __restrict__ row_scat,
                                                           const int64_t* __restrict__ col_scat, int64_t rows,
                                                           int64_t cols, T* __restrict__ out) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const int64_t ro = row_scat[r];
    T* o = out + r * cols;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < cols; c += int64_t(gridDim.x) * blockDim.x)
      o[c] = __ldg(src + ro + __ldg(col_scat + c));
  }
}

}  // namespace

int launch_pack_scatter(int is_f64, const void* src, const int64_t* row_scat, const int64_t* col_scat, int64_t rows,
                        int64_t cols, void* out, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return 0;
  const int64_t bx = (cols + 255) / 256;
  const unsigned gx = unsigned(bx < 64 ? bx : 64);
  const unsigned gy = unsigned(rows < 65535 ? rows : 65535);
  note_launch();
  if (is_f64)
    pack_scatter_kernel<double><<<dim3(gx, gy), 256, 0, s>>>(static_cast<const double*>(src), row_scat, col_scat, rows,
                                                              cols, static_cast<double*>(out));
  else
    pack_scatter_kernel<float><<<dim3(gx, gy), 256, 0, s>>>(static_cast<const float*>(src), row_scat, col_scat, rows,
                                                             cols, static_cast<float*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
