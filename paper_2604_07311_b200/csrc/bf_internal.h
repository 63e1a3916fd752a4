// Internal (C++) parameter blocks shared by the kernels and the C-ABI layer.
// Nothing here crosses the library boundary; include/blockfam_b200.h is the ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bf {

// How an operand tile is fetched from global memory.
enum GlobalLayout : int {
  GL_KMAJOR = 0,   // unit stride along k   (row-major A, "NT" B)  -> k-major smem
  GL_MNMAJOR = 1,  // unit stride along m/n (col-major A, row-major B) -> mn-major smem
  GL_GENERIC = 2,  // arbitrary strides or block-scatter vectors     -> k-major smem, 1 element per copy
  GL_TRIDIAG = 3,  // B read through W = T*S (skew tridiagonal T): the sandwich's pack-time transform
};

// One GEMM operand viewed as an (mn x k) matrix: A is (m x k), B^T is (n x k).
// Element (i, p) lives at base[off + i*s_mn + p*s_k], or at
// base[mn_scat[i] + k_scat[p]] when the scatter vectors are given
// (tensor/scatter.py:69-98 block-scatter facades).
struct OperandMK {
  const void* base;
  int64_t off;
  int64_t s_mn;
  int64_t s_k;
  const int64_t* mn_scat;
  const int64_t* k_scat;
  int layout;  // GlobalLayout
  int vec;     // elements per vector copy along the unit-stride dim (1, or 16B/elem)
  const double* tvec;  // GL_TRIDIAG: subdiagonal of T (length k_total - 1), device
  int64_t k_total;     // GL_TRIDIAG: K of the product (edge terms of T dropped)
};

// Division of 32-bit unsigned values by a runtime-invariant divisor with a
// precomputed multiplier (round-up method): q = (hi + ((x - hi) >> 1)) >> (l - 1),
// hi = umulhi(x, m); exact for every 32-bit x.  Used by the TMA kernel's
// mode-group coordinates, where a plain division per stage issue measured
// ~15 % of the contraction's time.
struct FastDiv {
  uint32_t d = 1, m = 0, l = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d <= 1) return;
    while ((uint64_t(1) << l) < d) ++l;
    m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
  }
#ifdef __CUDACC__
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    if (d == 1) return x;
    const uint32_t hi = __umulhi(x, m);
    return (hi + ((x - hi) >> 1)) >> (l - 1);
  }
  __device__ __forceinline__ uint32_t mod(uint32_t x) const { return x - div(x) * d; }
#endif
};

// One group of a grouped GEMM launch (the distributed trailing update: one
// group per local column panel).  Its C is m x n at c (row stride ldc); its A
// rows start at row a_row of the A map, its B^T rows at row b_row of the B map
// (or of the A map when b_from_a); tiles are row-major within the group,
// lower trapezoid (tj <= ti) when lower; tile0 = index of its first tile.
struct GroupDesc {
  double* c;
  int64_t ldc;
  int64_t tile0;
  int32_t m, n, a_row, b_row, tiles_m, tiles_n, lower, b_from_a;
};
constexpr int GEMM_MAX_GROUPS = 128;

// C := beta*C + alpha*A*B with the reference's accumulation structure:
// the k range is cut into segments of kc (engine/gemm.py:124-126); each
// segment is summed from +0 as an ascending fma chain and folded into C as
// C = beta_eff*C + alpha*t with beta_eff = beta on the first segment, 1 after
// (engine/kernels.py:228-253).  lower_only writes only i >= j.
struct GemmParams {
  int64_t m, n, k;
  int64_t kc;
  OperandMK a;
  OperandMK b;
  void* c;
  int64_t c_off, c_rs, c_cs;
  const int64_t* c_rscat;  // scatter C (contraction), else nullptr
  const int64_t* c_cscat;
  double alpha, beta;
  int lower_only;
  int tiles_m, tiles_n;
  int group;              // raster group height in tiles
  int panel_tiles;        // TMA lower GEMMT: > 0 = column panels this many tiles wide, row-major within a panel
  int tiles_per_cta;      // TMA kernel: contiguous raster tiles per CTA
  int tile_stride;        // TMA kernel: 0, or CTA b owns raster tiles b, b + tile_stride, ... (persistent grid)
  int64_t num_tiles;
  const int* abort_flag;  // skip all work when non-null and 0 <= *abort_flag < abort_limit
  int64_t abort_limit;    // a failure at a pivot >= abort_limit happened "later" in the
                          // reference's order and must not cancel this launch
  int red_fold;           // TMA kernel: beta_eff == 1 folds as L2 reductions (C += alpha*acc)
  // Mode-group operands (tensor contraction with permuted modes, TMA kernel
  // only): operand X (A as M x K, B^T as N x K) is a 4-D tensor map
  // (k_in, mn_in, k_out, mn_out); tile row r and k index k are loaded at
  // coordinates (k % ki, r % mi, k / ki, r / mi).  C element (i, j) lives at
  // c_off + (i / c_ri) * c_rs_o + (i % c_ri) * c_rs + (j / c_ci) * c_cs_o + (j % c_ci) * c_cs.
  const GroupDesc* groups;  // grouped launch (device table), else nullptr
  int ngroups;
  int modes;
  int a_rank, b_rank;  // 2: plain 2-D map (one group a side), 4: 4-D mode-group map
  FastDiv a_ki, a_mi, b_ki, b_mi, c_ri, c_ci;
  int64_t c_rs_o, c_cs_o;
};

__device__ __forceinline__ bool aborted(const GemmParams& p) {
  if (p.abort_flag == nullptr) return false;
  const int f = *p.abort_flag;
  return f >= 0 && f < p.abort_limit;
}

// Every kernel launch of this library bumps a process-wide counter
// (bf_launch_count in the ABI) so benchmarks can report how many of OUR
// kernels ran in a timed region.
void note_launch(int64_t n = 1);

// Raise a kernel's dynamic shared-memory limit on the CURRENT device, once per
// (kernel, device): cudaFuncSetAttribute only applies to the calling device's
// context, so a process-wide "done" flag would skip every other GPU.
bool smem_attr(const void* kern, int bytes);
// device scratch keyed by (tag, current device, stream); grows on demand
void* stream_scratch(int tag, size_t bytes, cudaStream_t s);
void scratch_account(int64_t delta_bytes);  // every library-owned device buffer reports here
// capi.cu bridges for the other translation units
int set_error(int code, const char* msg);
cudaStream_t panel_stream_for(cudaStream_t caller);  // the high-priority panel stream paired with `caller`
extern int g_mixed_reserve;
extern int g_mixed_inverse;  // mixed.cu: 1 = factor, then the doubling inverse
extern int g_symv;        // mixed.cu: residual / row sums from the lower triangle of A
extern int g_potrs_coop;  // mixed.cu: the refinement solve as one cooperative kernel
extern int g_potrs_vec;   // mixed.cu: float4 streams in that kernel
int launch_axpby_f32_f64(double alpha, const float* src, int64_t ld, double beta, double* c, int64_t off, int64_t rs,
                         int64_t cs, int64_t m, int64_t n, cudaStream_t s);

// Kernel-family entry points (implemented in the .cu files).
int launch_gemm_dmma(const GemmParams& p, cudaStream_t s);            // f64 storage, f64 acc
bool gemm_dmma_tma_eligible(const GemmParams& p);                     // TMA/mbarrier fast path?
int launch_gemm_dmma_tma(const GemmParams& p, cudaStream_t s);
// mode-group operand: element (mn, k) at off + (mn / mi) * s_mn_o + (mn % mi) * s_mn + (k / ki) * s_k_o + (k % ki)
struct ModeOperand {
  const double* base;
  int64_t off;
  int64_t mi, s_mn, s_mn_o;  // inner MN group size and stride, outer MN stride
  int64_t ki, s_k_o;         // inner K group size (unit stride), outer K stride
};
// TMA kernel on mode-group operands (a: M x K, b: N x K); -3 when a layout is not TMA-loadable
int launch_gemm_dmma_modes(GemmParams p, const ModeOperand& a, const ModeOperand& b, cudaStream_t s);
// grouped TMA GEMM: p carries k, kc, alpha, beta, abort; a = A rows (rows_a x k,
// k-contiguous), b = B^T rows (rows_b x k); groups (device table, ngroups <=
// GEMM_MAX_GROUPS) with num_tiles in all.  -3 when not TMA-loadable.
int launch_gemm_dmma_grouped(GemmParams p, const OperandMK& a, int64_t rows_a, const OperandMK& b, int64_t rows_b,
                             const GroupDesc* d_groups, int ngroups, int64_t num_tiles, cudaStream_t s);
// pack.cu: out[r*cols + c] = src[row_scat[r] + col_scat[c]] (contraction operand staging)
int launch_pack_scatter(int is_f64, const void* src, const int64_t* row_scat, const int64_t* col_scat, int64_t rows,
                        int64_t cols, void* out, cudaStream_t s);
extern int g_use_tma;         // bf_set_option("tma", 0|1)
extern int g_tma_variant;     // bf_set_option("tma_variant", 0..3)
extern int g_tmc_bn64;        // bf_set_option("tmc_bn64", 0|1)
extern int g_tma_bn;          // bf_set_option("tma_bn", 64 | 128): TMA DMMA tile width
extern int g_persist;         // bf_set_option("persist", 0|1): strided persistent grid for long-K GEMMs
extern int g_red_fold;        // bf_set_option("red_fold", 0|1): TMA kernel folds with red.global.add.f64
extern int g_tmem_fold;       // bf_set_option("tmem_fold", 0|1): TMA kernel keeps C in TMEM across kc folds
extern int g_reserve_strided;
extern thread_local int t_reserve_sms;  // gemm_dmma_tma.cu: SMs left free by the next launch
extern int g_tiles_per_cta;   // bf_set_option("tiles_per_cta", t)
extern int g_bf16_group;      // bf_set_option("bf16_group", g)
extern int g_bf16_tma_c;      // bf16 GEMM: TMA C-tile epilogue (1) or per-element fallback (0)
extern int g_trsm_warp;       // fused TRSM subtree: 4-warps-per-32-rows kernel (1) or the 64-row CTA kernel (0)
extern int g_pdl;             // bf_set_option("pdl", 0|1): programmatic dependent launch on the chain kernels
extern int g_leaf_pipe;       // bf_set_option("leaf_pipe", 0|1)
extern int g_leaf_blocked;    // variant-3 leaves n <= 128: blocked lane-per-row kernel (1) or v3 (0)
extern int g_fused_diag;      // bf_set_option("fused_diag", 0|1|2): one-launch diagonal factor (small_kernels.cu)
extern thread_local int t_diag_ctas;  // capi.cu: CTAs of the next fused diagonal factor (0: one per SM)
int fused_diag_stats(int64_t* out9);
int launch_trsm_diag_tiles(const double* l, int64_t ldl, double* x, int64_t ldx, int64_t n, int64_t kc,
                           cudaStream_t s);
// after_reset (optional) is recorded between the counter reset and the
// launch; *colfinal (optional) receives the device flags colfinal[c] (1 once
// tile column c of the block is final)
int launch_potrf_diag_fused(double* a, int64_t off, int64_t n, int64_t ld, int64_t kc, int64_t base_index,
                            int* d_info, int ctas, cudaStream_t s, cudaEvent_t after_reset = nullptr,
                            int** colfinal = nullptr);
extern int g_lu_grid_max;     // LU leaf: cap on the cooperative grid (0 = SM-derived)
extern int g_lu_global;       // LU leaf: force the global-memory kernel
extern int g_lu_noprefetch;   // LU leaf: no candidate-row prefetch
extern int g_lu_nocluster;    // LU leaf: never the single-cluster kernel
extern int g_lu_cluster_max;  // LU leaf: largest cluster
extern int g_qr_global;       // QR panel: force the global-memory sweep
extern int g_ltlt_grid_max;   // LTL^T stepper: cap on the cooperative grid
int launch_gemm_simt_f32(const GemmParams& p, cudaStream_t s);        // f32 storage, f32 acc
int launch_gemm_simt_f32acc64(const GemmParams& p, cudaStream_t s);   // f32 storage, f64 acc
int launch_copy2d_unless_aborted(const double* src, int64_t sld, double* dst, int64_t dld, int64_t m, int64_t n,
                                 const int* abort_flag, cudaStream_t s);
int launch_scale(int is_f64, double beta, void* c, int64_t off, int64_t m, int64_t n, int64_t rs,
                 int64_t cs, const int64_t* rscat, const int64_t* cscat, int lower_only,
                 cudaStream_t s);
int launch_potrf_leaf(int is_f64, int variant, void* a, int64_t off, int64_t n, int64_t rs,
                      int64_t cs, int64_t base_index, int* d_info, cudaStream_t s);
int launch_trsm_base_right(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs,
                           int64_t tcs, void* b, int64_t boff, int64_t brs, int64_t bcs, int64_t m,
                           int64_t n, int* d_singular, int64_t index_base, const int* abort_flag,
                           cudaStream_t s);

int launch_trsm_small_right(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                            int64_t boff, int64_t brs, int64_t bcs, int64_t m, int64_t n, int64_t kc,
                            const int* abort_flag, cudaStream_t s);

int launch_gemm_tf32_tc(double alpha, const float* a, int64_t lda, const float* b, int64_t ldb, double beta, float* c,
                        int64_t c_off, int64_t c_rs, int64_t c_cs, int64_t m, int64_t n, int64_t k, int lower_only,
                        cudaStream_t s);
int launch_split_tf32(int src_f64, const void* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t ld,
                      int64_t m, int64_t k, int64_t kp, cudaStream_t s);
int launch_gemm_bf16_tc(double alpha, const void* a, int64_t lda, const void* b, int64_t ldb, double beta, float* c,
                        int64_t c_off, int64_t c_rs, int64_t c_cs, int64_t m, int64_t n, int64_t k, int lower_only,
                        cudaStream_t s);
int launch_to_bf16(const float* src, int64_t soff, int64_t srs, int64_t scs, void* dst, int64_t ld, int64_t m,
                   int64_t n, int transpose, cudaStream_t s);
int launch_f32_to_f64(const float* src, int64_t soff, int64_t srs, int64_t scs, double* dst, int64_t doff, int64_t drs,
                      int64_t dcs, int64_t m, int64_t n, int lower_only, cudaStream_t s);
int launch_f64_to_bf16(const double* src, int64_t soff, int64_t srs, int64_t scs, void* dst, int64_t ld, int64_t m,
                       int64_t n, int transpose, cudaStream_t s);
int launch_f64_to_f32(const double* src, int64_t soff, int64_t srs, int64_t scs, float* dst, int64_t doff, int64_t drs,
                      int64_t dcs, int64_t m, int64_t n, int lower_only, cudaStream_t s);
int launch_residual(const double* A, int64_t lda, const double* x, const double* b, double* r, int64_t n,
                    cudaStream_t s);
int launch_lu_leaf(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, int64_t* piv,
                   int* d_sing, int64_t base, cudaStream_t s);
int launch_apply_pivots(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t ncols, const int64_t* piv,
                        int64_t count, int64_t sub, int backward, cudaStream_t s);
int launch_add_offset(int64_t* piv, int64_t count, int64_t delta, cudaStream_t s);
int launch_tridiag_form_f32(const float* a, int64_t off, int64_t rs, int64_t cs, int64_t n, int64_t kt, const float* t,
                            float* w, cudaStream_t s);
int launch_transpose_tri_f64(const double* src, int64_t off, int64_t rs, int64_t cs, int64_t n, double* dst,
                             int64_t ld, int tri, cudaStream_t s);
int launch_transpose(int is_f64, const void* src, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, void* dst,
                     int64_t ld, cudaStream_t s);
int launch_trsm_left_base(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                          int64_t boff, int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s);
int launch_trsm_upper_base(int is_f64, const void* u, int64_t uoff, int64_t urs, int64_t ucs, void* b, int64_t boff,
                           int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s);
int launch_ltlt(int is_f64, void* x, int64_t off, int64_t rs, int64_t cs, int64_t n, int64_t j0, int64_t j1,
                int blocked, int64_t k, void* w, int64_t wld, int64_t* piv, void* t, void* mvec, void* wvec,
                cudaStream_t s);
int launch_qr_panel(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, void* taus,
                    cudaStream_t s);
int launch_qr_t(int is_f64, const void* gram, int64_t b, const void* taus, void* t, cudaStream_t s);
int launch_splitk_reduce(int is_f64, const void* ws, int S, int64_t m, int64_t n, double alpha, double beta, void* c,
                         int64_t off, int64_t rs, int64_t cs, cudaStream_t s);
int launch_segfold(const double* ws, int S, int64_t m, int64_t n, double alpha, double beta, double* c, int64_t off,
                   int64_t rs, int64_t cs, int lower_only, const int* abort_flag, int64_t abort_limit,
                   cudaStream_t s);
int launch_explicit_v(int is_f64, const void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t b, void* v,
                      cudaStream_t s);
int launch_reflector_apply(int is_f64, const void* a, int64_t aoff, int64_t ars, int64_t acs, int64_t m, int64_t j,
                           double tau, void* c, int64_t coff, int64_t crs, int64_t ccs, int64_t ncols,
                           cudaStream_t s);
int launch_row_abs_sum(const double* A, int64_t lda, double* out, int64_t n, cudaStream_t s);
int launch_potrs_f32_f64(const float* L, int64_t ld, double* x, int64_t n, cudaStream_t s);
int launch_potrs_blocked(const float* L, int64_t ld, const float* xinv, int64_t bs, double* x, int64_t n,
                         double* work, cudaStream_t s);

}  // namespace bf
