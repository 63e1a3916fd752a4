/* blockfam-b200: C ABI of the B200-native level-3 hot path.
 *
 * This is the drop-in boundary for the reference package `blockfam`
 * (/root/reference/pkg/src/blockfam).  The reference's algorithm layer calls
 * its engine by name (factor/cholesky.py:24: gemm, syrk_lower, trsm) and its
 * leaves through `_UNBLOCKED[variant](storage, offset, rs, cs, n) -> int`
 * (factor/cholesky.py:92-96,123); the contraction calls
 * `gemm_scatter(alpha, ScatterMatrix a, b, beta, c, cfg, ways)`
 * (tensor/contract.py:177-185).  Each of those maps to one function below.
 *
 * Conventions
 *   - A matrix operand is a strided view: element (i, j) lives at
 *     ((T*)base)[off + i*rs + j*cs]  (views.py:131-146 MatrixView).  base is a
 *     DEVICE pointer; the library never allocates, frees or copies caller
 *     memory, and never touches host memory.
 *   - A block-scatter operand (tensor/scatter.py:22-39) is element
 *     (i, j) at ((T*)base)[rscat[i] + cscat[j]] with rscat/cscat DEVICE int64
 *     vectors.
 *   - Suffix d = FP64, s = FP32 (FP32 accumulation), sd = FP32 storage with
 *     FP64 accumulation (engine/config.py:14-48 acc_dtype).
 *   - `kc` is the reference's kc cache block, which is the only blocking
 *     parameter that changes arithmetic: the k range is folded into C every
 *     kc elements (engine/gemm.py:124-126).  Passing the reference's kc makes
 *     results bit-identical to the reference.
 *   - All functions are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and thread-safe for distinct streams: the library's own
 *     side streams (panel, aux, copy) and its scratch buffers are private to
 *     each (device, calling stream) pair.  bf_set_option settings are
 *     process-wide and must not change while calls are in flight, and the
 *     bf_timeline record is a single-caller debugging aid.  Device-side
 *     failure indices are reported through caller-owned device ints that the
 *     caller initialises to -1 and reads after synchronising.
 *   - Return codes: BF_OK, or a negative BF_ERR_* (no fallback path exists:
 *     an unsupported request fails loudly).
 */
#ifndef BLOCKFAM_B200_H
#define BLOCKFAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BF_OK 0
#define BF_ERR_SHAPE (-1)       /* dims mismatch (reference ShapeError) */
#define BF_ERR_ALIAS (-2)       /* reserved: aliasing is checked by the host layer */
#define BF_ERR_UNSUPPORTED (-3) /* layout / size this build does not handle */
#define BF_ERR_VALUE (-4)       /* bad argument (variant, kc < 1, ...) */
#define BF_ERR_CUDA (-11)       /* a CUDA launch or attribute call failed */

typedef struct bf_view {
  void* base;
  int64_t off, m, n, rs, cs;
} bf_view;

typedef struct bf_scatter_view {
  void* base;
  int64_t m, n;
  const int64_t* rscat; /* device, length m */
  const int64_t* cscat; /* device, length n */
} bf_scatter_view;

/* One level of a Cholesky control tree (control.py:47-71 ControlNode):
 * variant 1/2/3 = blocked (bs required), 11/12/13 = unblocked1/2/3 leaf;
 * kc = the level's effective kernel kc (control.py:67-68 effective_config). */
typedef struct bf_chol_level {
  int32_t variant;
  int32_t pad_;
  int64_t bs;
  int64_t kc;
} bf_chol_level;

int bf_abi_version(void);
/* Free the library's cached device scratch (per-stream buffers of the
 * 3xTF32 split, the LU k-major copies, the upper-triangle row-major copy);
 * synchronises the device. */
int bf_release_scratch(void);
/* Bytes of device scratch the library holds now and its high-water mark since
 * the last reset (the B200 side of the reference's Workspace accounting,
 * engine/workspace.py:18-56). */
int bf_scratch_stats(int64_t* live_bytes, int64_t* peak_bytes);
int bf_scratch_reset_peak(void);
/* Number of kernels this library has launched in this process (all devices). */
int64_t bf_launch_count(void);
const char* bf_last_error(void);
/* Process-wide switches (none changes arithmetic): "lookahead" (default 1)
 * overlaps the next panel's POTRF+TRSM with the trailing update in
 * bf_cholesky_*; "tma" / "tma_variant" / "tiles_per_cta" / "group" select the
 * FP64 GEMM kernel and its tile schedule; "fused_trsm" the single-kernel TRSM
 * subtree; "timeline" records per-step events; "bf16_tma_c" the TMA C-tile
 * epilogue of the bf16 GEMM; "tail_reserve" (default 16) / "tail_rows"
 * (default 32768) run the lookahead's rest-of-step update as a persistent grid
 * leaving that many SMs to the panel stream when the update is <= tail_rows
 * rows; "reserve_strided" its tile order; "diag_reserve" / "diag_rows" an
 * optional two-phase split of that update (off); "red_fold" (default 1) folds
 * the TMA GEMM's beta == 1 segments as red.global.add.f64 L2 reductions (0:
 * load/add/store); "persist" a strided one-CTA-per-SM grid for long-K GEMMs (off);
 * "tma_bn" (default 64) runs plain TMA DMMA launches on two independent
 * 8-warp groups per CTA over 128x64 tiles (128: one 16-warp group on 128x128
 * tiles; "tmc_bn64" extends it to the TMEM-fold launches, off); "panel_overlap"
 * (default 1) lets a lookahead panel's TRSM of the rows below trail its
 * diagonal factor's inner steps on its own streams ("panel_chunks" row chunks
 * of at least "panel_chunk_rows" rows, defaults 2 and 6144), on a copy written
 * back only without a pivot failure; "reserve_adaptive" / "reserve_extra" /
 * "reserve_min" size the reservation per step; "potrs_coop" / "potrs_vec" (default 1) and
 * "symv" (default 1) select the mixed refinement's cooperative blocked solve
 * and lower-triangle residual; "early_panel" (default 1) starts panel k+1's
 * diagonal factor once its diagonal tile is updated; "leaf_pipe" (default 1)
 * overlaps the blocked leaf's next chain with its trailing update; "pdl"
 * (default 1) launches the chain kernels with programmatic dependent launch;
 * "bf16_group" (default 8) the tcgen05 GEMM's band height; "fused_diag"
 * (default 1: where nothing trails the inner steps; 2: everywhere; 0: off)
 * runs a {v3, bs 128, kc >= 128} over unblocked3 diagonal block of order
 * <= 2048 as one launch, "fused_diag_ctas" (default 0) forces its grid and
 * "fused_diag_pct" (default 100) is its share of the reserved SMs inside the
 * lookahead (with 2). */
int bf_set_option(const char* name, int64_t value);
int bf_device_sm_count(void);
/* With bf_set_option("timeline", 1): per top-level step of the last lookahead
 * factorization, 5 floats (ms): next-column update done, trailing update done,
 * panel start, panel end, diagonal factor of the panel done.  Returns the
 * number of steps. */
int bf_timeline(float* out, int max_steps);

/* C := beta*C + alpha*A*B (lower_only: only i >= j of C is read or written).
 * Replaces engine/gemm.py:179-242 gemm / gemmt_lower / syrk_lower (syrk =
 * gemm(a, a^T view, lower_only=1)).  Edge semantics of engine/gemm.py:97-108:
 * alpha==0 && beta==1 -> no-op; k==0 || alpha==0 -> C := beta*C only.
 * d_abort: optional device int; the kernels do nothing if *d_abort >= 0. */
int bf_gemm_d(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only,
              int64_t kc, const int* d_abort, void* stream);
int bf_gemm_s(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only,
              int64_t kc, const int* d_abort, void* stream);
int bf_gemm_sd(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only,
               int64_t kc, const int* d_abort, void* stream);

/* C := beta*C over all of C or its lower triangle (engine/kernels.py:125-139). */
int bf_scale_d(double beta, const bf_view* c, int lower_only, void* stream);
int bf_scale_s(double beta, const bf_view* c, int lower_only, void* stream);
int bf_scale_sd(double beta, const bf_view* c, int lower_only, void* stream);

/* Unblocked Cholesky leaf on a square view, variant 1/2/3 (factor/cholesky.py:31-96).
 * On a non-positive pivot k writes base_index + k to *d_info (if *d_info < 0). */
int bf_potrf_leaf_d(const bf_view* a, int variant, int64_t base_index, int* d_info, void* stream);
int bf_potrf_leaf_s(const bf_view* a, int variant, int64_t base_index, int* d_info, void* stream);

/* B := alpha * B * tril(T)^-T, recursive halving to a 32 base exactly as
 * engine/trsm.py:29-68,96-111 (off-diagonal blocks through bf_gemm with kc).
 * A zero diagonal writes the base-local column index to *d_singular and stops. */
int bf_trsm_rltn_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular, void* stream);
int bf_trsm_rltn_s(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular, void* stream);

/* In-place lower Cholesky of a square view driven by a flattened control tree
 * (levels[0] = root; a blocked level without a successor recurses on
 * unblocked3, factor/cholesky.py:154-158).  Same operation sequence as
 * factor/cholesky.py:118-151.  First failing global pivot -> *d_info. */
int bf_cholesky_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int* d_info, void* stream);
/* In-place FP64 Cholesky of a HOST matrix (pinned for overlap; row-major, ld):
 * its lower triangle goes to the device work matrix by block columns, is
 * factored there, and every block column returns to the host as soon as it is
 * final (copy stream, overlapped with the remaining steps).  The strict upper
 * triangle of the host matrix is neither read nor written.  Same bits as
 * bf_cholesky_d.  After a pivot failure the host holds the factor only up to
 * the columns already streamed back: re-read the lower triangle from `work`.
 * (No reference counterpart: the reference factors NumPy host arrays in
 * place, factor/cholesky.py:99-115; this is that call with device compute.) */
int bf_cholesky_host_d(double* host, int64_t ld, const bf_view* work, const bf_chol_level* levels, int nlevels,
                       int* d_info, void* stream);
int bf_cholesky_s(const bf_view* a, const bf_chol_level* levels, int nlevels, int* d_info, void* stream);

/* Building blocks of the distributed driver (paper_2604_07311_b200/dist):
 * the tree walk without the root lookahead, reporting pivots offset by
 * base_index; and the TRSM with separate (nullable) singular-report and abort
 * flags (d_singular == NULL selects the fused subtree kernels). */
int bf_cholesky_ex_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t base_index, int* d_info,
                     void* stream);
int bf_trsm_rltn_ex_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, int* d_singular,
                      const int* d_abort, void* stream);

/* Block-scatter GEMM for tensor contraction (engine/gemm.py:74-160 on
 * tensor/contract.py facades): C := beta*C + alpha*A*B with every operand
 * addressed through its scatter vectors. */
int bf_gemm_scatter_d(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                      const bf_scatter_view* c, int64_t kc, void* stream);
int bf_gemm_scatter_s(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                      const bf_scatter_view* c, int64_t kc, void* stream);
/* Operand staging (the whole-operand form of engine/kernels.py:24-90
 * pack_a_block / pack_b_block): out (m x n, or n x m when transpose != 0,
 * row-major, device) := src[rscat[i] + cscat[j]].  tensor/contract.py stages a
 * large permuted facade k-contiguous with it so the TMA DMMA GEMM can read it;
 * values are copied exactly, so the contraction's bits do not change. */
int bf_pack_scatter_d(const bf_scatter_view* src, int transpose, double* out, void* stream);
/* Mode-group view of a contraction facade (tensor/contract.py:90-102 _facade,
 * tensor/scatter.py:69-98): rows are nr <= 2 mode groups, columns nc <= 2,
 * slowest first, each with its size and element stride; element (i, j) at
 * off + sum_g (i_g * rstr[g]) + sum_g (j_g * cstr[g]) with (i_0, i_1) the
 * mixed-radix digits of i (i_1 fastest).  This is the B200 form of the
 * reference's scatter vectors for the 4-index case: the GEMM reads it with
 * 4-D TMA tensor maps, so permuted operands need no transpose. */
typedef struct bf_modes_view {
  void* base;
  int64_t off;
  int32_t nr, nc;
  int64_t rdim[2], rstr[2];
  int64_t cdim[2], cstr[2];
} bf_modes_view;
/* C := beta*C + alpha*A*B over mode-group views (A: M x K, B: K x N, C: M x N),
 * the reference's kc folds (bit-identical to bf_gemm_scatter_d).  TMA needs
 * the fastest K group of A and of B unit-stride with a size that is a
 * multiple of 16, the fastest row group of A / column group of B a multiple
 * or divisor of 128, 16-byte strides and K % 32 == 0; otherwise it returns
 * BF_ERR_UNSUPPORTED (the host then stages or gathers that operand).
 * alpha == 0 or K == 0 are the caller's (reference edge semantics). */
/* bf16 variant (SURVEY.md §8(b) bf_contract_x; no reference counterpart):
 * C := beta*C + alpha*A*B for FP64 strided views with the operands rounded to
 * bf16 and the products summed in fp32 on tcgen05 (TMEM accumulators);
 * accuracy ~2^-8 relative per product.  Uses library scratch
 * ((M+N)*K bf16 + M*N fp32, bf_scratch_stats). */
int bf_contract_bf16_d(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c,
                       void* stream);
int bf_contract_modes_d(double alpha, const bf_modes_view* a, const bf_modes_view* b, double beta,
                        const bf_modes_view* c, int64_t kc, void* stream);
int bf_gemm_scatter_sd(double alpha, const bf_scatter_view* a, const bf_scatter_view* b, double beta,
                       const bf_scatter_view* c, int64_t kc, void* stream);

/* Skew sandwich: replaces engine/gemm.py:245-280
 * sandwich_skew / gemm_scatter(..., tridiag_t): lower(C) := C - A T A^T with T
 * skew tridiagonal (T[i+1,i] = t[i] = -T[i,i+1]), t on the device (length
 * a->n - 1).  T A^T is formed while B tiles are staged (the reference's
 * pack-time transform, kernels.py:93-122): no k x n intermediate.  Bitwise. */
int bf_sandwich_skew_d(const bf_view* c, const bf_view* a, const double* d_t, int64_t kc, void* stream);
/* f32 storage (f32 packing arithmetic, as the reference's acc dtype): W = T A^T
 * is formed in the caller's device workspace d_w (a->n x c->n floats). */
int bf_sandwich_skew_s(const bf_view* c, const bf_view* a, const float* d_t, float* d_w, int64_t kc, void* stream);

/* Pivoted LTL^T of a skew-symmetric matrix (factor/ltlt.py), eliminations
 * [j0, j1) on the stored lower triangle: blocked = 0 runs the unblocked
 * right-looking stepper (ltlt.py:157-182; d_m/d_w: n-element workspaces;
 * bitwise); blocked = 1 runs one panel of the blocked form starting at k
 * (ltlt.py:131-147; w: the n x wld history, swapped with the rows; the
 * trailing update is then bf_sandwich_skew_*).  d_piv (n, preset 0..n-1) and
 * d_t (n-1) receive the swaps and T's subdiagonal. */
int bf_ltlt_d(const bf_view* x, int64_t j0, int64_t j1, int blocked, int64_t k, double* w, int64_t wld,
              int64_t* d_piv, double* d_t, double* d_m, double* d_w, void* stream);
int bf_ltlt_s(const bf_view* x, int64_t j0, int64_t j1, int blocked, int64_t k, float* w, int64_t wld,
              int64_t* d_piv, float* d_t, float* d_m, float* d_w, void* stream);

/* Householder QR (factor/qr.py).  The reference
 * uses NumPy/BLAS for every panel operation, so these agree with it to
 * rounding (its own tests are tolerance tests).
 * bf_qr_panel_*: the unblocked column sweep (qr.py:58-76) on an m x b view
 *   (m >= b), taus to d_taus (b).
 * bf_qr_t_*: the panel's compact-WY T (b x b upper, qr.py:79-92) and the
 *   explicit V (m x b, unit diagonal, qr.py:95-100); d_gram: b x b workspace
 *   (V^T V by the split-K GEMM, feeds T's recursion).
 * bf_gemm_splitk_*: c = alpha a b + beta c for the reflector products of the
 *   blocked update (V^T C, qr.py:103-121, NumPy '@' in the reference): the K
 *   range is split over concurrent streams when the output has few tiles.
 *   To rounding only — never a substitute for bf_gemm_* on bitwise paths.
 * bf_reflector_apply_*: c := H_j c, H_j = I - tau v v^T with v stored in
 *   column j of a below the diagonal (apply_q, qr.py:124-140). */
int bf_qr_panel_d(const bf_view* a, double* d_taus, void* stream);
int bf_qr_panel_s(const bf_view* a, float* d_taus, void* stream);
int bf_qr_t_d(const bf_view* panel, const double* d_taus, double* d_t, double* d_v, double* d_gram, void* stream);
int bf_qr_t_s(const bf_view* panel, const float* d_taus, float* d_t, float* d_v, float* d_gram, void* stream);
int bf_gemm_splitk_d(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, void* stream);
int bf_gemm_splitk_s(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, void* stream);
int bf_reflector_apply_d(const bf_view* a, int64_t j, double tau, const bf_view* c, void* stream);
int bf_reflector_apply_s(const bf_view* a, int64_t j, double tau, const bf_view* c, void* stream);

/* LU with partial pivoting.
 * bf_lu_*: replaces factor/lu.py:56-103 lu_partial/_run with the tree walk in
 *   C++: levels are the flattened lu tree (variant 20 = blocked, bs and the
 *   effective kc; 21 = the unblocked leaf, factor/lu.py:19-53).  d_piv
 *   (device, min(m,n) int64) receives the LAPACK-style swap list, d_sing
 *   (device int, preset -1) the first exactly-zero pivot column.  Bitwise the
 *   reference.
 * bf_trsm_llnu_*: unit_tril(tri) X = alpha B, replaces engine/trsm.py:71-88
 *   (LEFT_LOWER_NOTRANS_UNIT), bitwise.
 * bf_trsm_lun_*: triu(U) X = B for lu_solve (factor/lu.py:117-130 does this
 *   with NumPy; no bitwise contract).
 * bf_apply_pivots_*: factor/pivots.py:46-61 apply_pivots (forward/backward). */
int bf_lu_d(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t* d_piv, int* d_sing, void* stream);
int bf_lu_s(const bf_view* a, const bf_chol_level* levels, int nlevels, int64_t* d_piv, int* d_sing, void* stream);
int bf_trsm_llnu_d(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, void* stream);
int bf_trsm_llnu_s(double alpha, const bf_view* tri, const bf_view* b, int64_t kc, void* stream);
int bf_trsm_lun_d(const bf_view* u, const bf_view* b, int64_t kc, void* stream);
int bf_trsm_lun_s(const bf_view* u, const bf_view* b, int64_t kc, void* stream);
int bf_apply_pivots_d(const bf_view* a, const int64_t* d_piv, int64_t count, int backward, void* stream);
int bf_apply_pivots_s(const bf_view* a, const int64_t* d_piv, int64_t count, int backward, void* stream);

/* Mixed precision (BASELINE configs[3]; no reference counterpart).
 * bf_gemm_bf16: C(fp32 view) := beta*C + alpha * A * B^T on tcgen05/TMEM, with
 * A (c->m x k) and B (c->n x k) row-major bf16 (ld in elements, 16-byte aligned).
 * bf_convert_*: precision conversions between views / dense buffers.
 * bf_residual_d: r := b - A x for a dense row-major fp64 A (n x n) that is
 * symmetric (the SPD matrix of the mixed solve): only its lower triangle is
 * read (bf_set_option("symv", 0): the whole matrix, row by row).
 * bf_potrs_f32_d: x := (L L^T)^-1 x for the fp32 lower factor L (row-major ld),
 * fp64 right-hand side and arithmetic (one CTA per diagonal block: reference-grade, slow).
 * bf_potrs_blocked_f32_d: the same solve as matrix-vector products against the
 * explicit diagonal-block inverses xinv[k] = L_kk^-T (nblk x bs x bs fp32, kept by
 * the mixed factorization); work holds 129*bs doubles. */
int bf_gemm_bf16(double alpha, const void* a, int64_t lda, const void* b, int64_t ldb, double beta, const bf_view* c,
                 int64_t k, int lower_only, void* stream);
int bf_convert_f32_bf16(const bf_view* src, void* dst, int64_t ld, int transpose, void* stream);
/* FP32 on the tensor cores (3xTF32; no reference counterpart — the
 * reference's f32 GEMM is engine/gemm.py:179-201 with f32 or f64
 * accumulation, which tcgen05 cannot reproduce bit for bit; this is the
 * fp32-accurate tensor-core alternative, to rounding).
 * bf_split_tf32_{s,d}: row i of src (m x k, fp32 / fp64) -> dst row i =
 *   [hi | hi | lo | hi], four parts of kp >= k columns (zero padded),
 *   hi = tf32(x) (round to nearest), lo = x - hi; ld >= 4 kp.
 * bf_gemm_tf32: C(fp32 view) := beta*C + alpha * A * B^T with A (c->m x k),
 *   B (c->n x k) row-major fp32 read as tf32 (kind::tf32, TMEM accumulation).
 *   With A = split[:, 0:3kp] and B = split[:, kp:4kp], k = 3kp: the 3xTF32 product.
 * bf_gemm_f32_tc: C := beta*C + alpha * A * B for fp32 views, both splits and
 *   the K = 3k tf32 GEMM in one call (lower_only: GEMMT). */
int bf_split_tf32_s(const bf_view* src, float* dst, int64_t ld, int64_t kp, void* stream);
int bf_split_tf32_d(const bf_view* src, float* dst, int64_t ld, int64_t kp, void* stream);
int bf_gemm_tf32(double alpha, const float* a, int64_t lda, const float* b, int64_t ldb, double beta, const bf_view* c,
                 int64_t k, int lower_only, void* stream);
int bf_gemm_f32_tc(double alpha, const bf_view* a, const bf_view* b, double beta, const bf_view* c, int lower_only,
                   void* stream);
int bf_convert_f64_f32(const bf_view* src, const bf_view* dst, int lower_only, void* stream);
/* Mixed-precision factorization driver (BASELINE configs[3]; no reference
 * counterpart — engine/config.py:21,39 is the reference's only mixed mode):
 * W (fp32, n x n, leading dimension ldw) := the lower factor of A (fp64) with
 * FP64 diagonal blocks (the control tree `lv` on each bs x bs block, global
 * pivot index in d_info), their explicit inverses X_k = L_kk^-T (FP64, stored
 * fp32 in xinv[k], bs x bs each), the panels L21 = A21 X_k and the trailing
 * updates on the tensor cores (precision 0: bf16 kind::f16, 1: tf32).
 * Workspace: pbuf0/pbuf1 (n x bs panel copies: bf16, or fp32 for tf32),
 * xt (bs x bs), d64 and x64 (bs x bs fp64).  lookahead = 1 runs each next
 * diagonal/inverse/panel on the library's high-priority stream while the
 * trailing GEMMT leaves SMs to it (bf_set_option("mixed_reserve", r));
 * bf_set_option("mixed_inverse", 1) forms each X_k after the factor by
 * recursive doubling instead of the right solve trailing it (slower). */
int bf_cholesky_mixed(const bf_view* a, float* w, int64_t ldw, void* pbuf0, void* pbuf1, void* xt, double* d64,
                      double* x64, float* xinv, int64_t bs, const bf_chol_level* lv, int nl, int precision,
                      int lookahead, int* d_info, void* stream);
int bf_convert_f32_f64(const bf_view* src, const bf_view* dst, int lower_only, void* stream);
int bf_convert_f64_bf16(const bf_view* src, void* dst, int64_t ld, int transpose, void* stream);
int bf_residual_d(const double* a, int64_t lda, const double* x, const double* b, double* r, int64_t n, void* stream);
/* out[i] := sum_j |a[i][j]| (the refinement's ||A||_inf is the max of these);
 * a symmetric, read through its lower triangle like bf_residual_d */
int bf_row_abs_sum_d(const double* a, int64_t lda, double* out, int64_t n, void* stream);
int bf_potrs_f32_d(const float* l, int64_t ld, double* x, int64_t n, void* stream);
int bf_potrs_blocked_f32_d(const float* l, int64_t ld, const float* xinv, int64_t bs, double* x, int64_t n,
                           double* work, void* stream);

/* ---- multi-GPU Cholesky (the reference has no
 * distribution) --------------------------------------------------
 * One process per GPU; NCCL over NVLink/NVSwitch.  The matrix is held as the
 * LOWER tiles of a 2D block-cyclic layout over a pr x pc process grid, tile
 * size nb = the root bs of the control tree: rank (prow, pcol) = (rank / pc,
 * rank % pc) owns tiles (I, J), I >= J, with I mod pr = prow and J mod pc =
 * pcol, stored as one row-major panel per local column tile J (its row tiles
 * I >= J stacked, leading dimension tile_len(J)), panels in J order
 * (paper_2604_07311_b200/csrc/dist_layout.h).  The root `ways` of a control
 * tree (control.py:47-71; the reference threads it into every level-3 call,
 * factor/cholesky.py:128-149) selects this path with ways = pr * pc ranks. */
typedef struct bf_dist bf_dist;
int bf_dist_available(void);                 /* 1 if NCCL could be loaded */
int bf_dist_unique_id_bytes(void);           /* sizeof(ncclUniqueId) */
int bf_dist_unique_id(void* out);            /* ncclGetUniqueId (rank 0), to be shared with every rank */
/* world communicator from the id, then ncclCommSplit into row / column communicators */
int bf_dist_init(const void* nccl_unique_id, int rank, int nranks, int pr, int pc, bf_dist** out);
/* "reserve" (-1 = adaptive), "fan", "lookahead", "grouped" (1: every
 * trailing-update part as one grouped TMA launch over the column panels),
 * "reserve_rows" (the grouped launch keeps its SM reservation while the
 * rank's stacked rows are <= this, default 32768) */
int bf_dist_set_option(bf_dist* d, const char* name, int64_t value);
int bf_dist_finalize(bf_dist* d);
int64_t bf_dist_local_elems(int64_t n, int64_t nb, int pr, int pc, int rank);            /* host only */
int64_t bf_dist_panel_offset(int64_t n, int64_t nb, int pr, int pc, int rank, int64_t q); /* host only */
/* synthetic SPD input A = S + n I (S symmetric, entries U[-1,1) from a counter
 * hash of (max(i,j), min(i,j), seed)): a rank fills its own tiles, so no rank
 * ever holds the whole matrix; bf_fill_synthetic_d fills a full view with the
 * same values (the one-GPU comparison) */
int bf_dist_fill_synthetic_d(int64_t n, int64_t nb, int pr, int pc, int rank, double* local, uint64_t seed,
                             void* stream);
int bf_fill_synthetic_d(const bf_view* a, uint64_t seed, void* stream);
/* factor this rank's panels in place (factor/cholesky.py:118-151 at a
 * variant-3 root, distributed); levels[0] = root (variant 3, bs = nb, kc),
 * levels[1..] = the diagonal tiles' tree.  Bit-identical to bf_cholesky_d on
 * one GPU with the same tree.  Synchronises `stream`. */
int bf_chol_dist_d(bf_dist* d, double* local, int64_t n, const bf_chol_level* levels, int nlevels, int* d_info,
                   void* stream);
int bf_cholesky_dist_d(bf_dist* d, double* local, int64_t n, const bf_chol_level* levels, int nlevels, int* d_info,
                       void* stream); /* alias of bf_chol_dist_d */

#ifdef __cplusplus
}
#endif

#endif /* BLOCKFAM_B200_H */
