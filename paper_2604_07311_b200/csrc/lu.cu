// LU with partial pivoting on B200 (reference factor/lu.py, factor/pivots.py,
// engine/trsm.py left-lower-unit case), SURVEY.md §8(f) rank 2.
//
//  * lu_leaf_kernel — the unblocked leaf (factor/lu.py:19-53) on a panel of
//    any height: a cooperative grid, each CTA owning a contiguous band of
//    rows; per column one grid-wide pivot search (partial maxima combined in
//    row order, so ties keep the smallest row and NaNs are never chosen, as
//    in the sequential scan), the row swap, the division of the column by the
//    pivot and the rank-1 update of the band — the reference's operations in
//    the reference's order for every element (a(i,j) -= a(i,k)*a(k,j),
//    unfused, ascending k).  An exactly-zero pivot column is recorded and
//    skipped like the reference.
//  * lu_leaf_cluster_kernel — the same leaf on one thread-block cluster when
//    the panel fits in its shared memory: cluster barrier + DSMEM instead of
//    a grid barrier + L2 (used first; the grid kernels take taller panels).
//  * apply_pivots_kernel — LAPACK-style swap list, one thread per column,
//    swaps in list order (factor/pivots.py:46-61).
//  * trsm_left_base_kernel — unit-lower X = T^-1 (alpha B) for n <= 32, one
//    thread per column, row by row, one ascending chain per element
//    (engine/trsm.py:114-125); the recursion above it lives in capi.cu.
//  * trsm_upper_base_kernel — the backward solve with the non-unit upper
//    factor used by lu_solve (no bitwise contract: the reference does it
//    with NumPy row operations, factor/lu.py:117-130).
#include "bf_common.cuh"
#include "bf_internal.h"

#include <cooperative_groups.h>

namespace bf {

int g_lu_grid_max = 0;  // bf_set_option("lu_grid", g): cap the leaf's cooperative grid (0 = SM-derived)
int g_lu_global = 0;    // bf_set_option("lu_global", 1): force the global-memory leaf
int g_lu_noprefetch = 0;  // bf_set_option("lu_noprefetch", 1): fetch the pivot row after the decision
int g_lu_nocluster = 0;   // bf_set_option("lu_nocluster", 1): never the single-cluster leaf
int g_lu_cluster_max = 16;  // bf_set_option("lu_cluster", c): largest cluster for the leaf (1..16)

namespace {

namespace cg = cooperative_groups;

constexpr int LU_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(LU_THREADS) lu_leaf_kernel(T* a, int64_t off, int64_t rs, int64_t cs, int64_t m,
                                                           int64_t n, int64_t* piv, int* d_sing, int64_t base,
                                                           double* part_v, int64_t* part_i) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, tid = threadIdx.x;
  const int64_t chunk = (m + G - 1) / G;
  const int64_t r0 = int64_t(blockIdx.x) * chunk, r1 = r0 + chunk < m ? r0 + chunk : m;
  const int64_t steps = m < n ? m : n;
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int64_t red_i[LU_THREADS / 32];
  // The panel is shared by the CTAs through L2: every read bypasses L1 (not
  // coherent across SMs — a row swapped by CTA 0 may sit stale in another
  // SM's L1), every write is write-through.
  auto at = [&](int64_t i, int64_t j) -> T& { return a[off + i * rs + j * cs]; };
  auto ld = [&](int64_t i, int64_t j) -> T { return __ldcg(a + off + i * rs + j * cs); };
  for (int64_t k = 0; k < steps; ++k) {
    // (a) this band's best candidate among rows > k: strict '>' in ascending
    // row order per thread, then the smallest row among equal maxima
    double bv = -1.0;
    int64_t bi = -1;
    const int64_t lo = r0 > k + 1 ? r0 : k + 1;
    for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
      const double v = double(fabs(ld(i, k)));
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (ov > bv || (ov == bv && (bi < 0 || oi < bi)))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_i[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < LU_THREADS / 32; ++w)
        if (red_i[w] >= 0 && (red_v[w] > bv || (red_v[w] == bv && (bi < 0 || red_i[w] < bi)))) {
          bv = red_v[w];
          bi = red_i[w];
        }
      part_v[blockIdx.x] = bv;
      part_i[blockIdx.x] = bi;
    }
    grid.sync();
    // (b) every CTA combines the bands in row order from the diagonal entry,
    // exactly the sequential scan: a later band wins only with a larger value
    // (the partials arrive in one round trip: lane c loads band c, G <= 32;
    // max value, smallest row among ties = the row-order combination)
    __shared__ double s_best;
    __shared__ int64_t s_p;
    if (tid < 32) {
      double cv = -1.0;
      int64_t ci = -1;
      if (tid < G) {
        ci = __ldcg(part_i + tid);
        cv = __ldcg(part_v + tid);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, cv, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, ci, o);
        if (oi >= 0 && (ov > cv || (ov == cv && (ci < 0 || oi < ci)))) {
          cv = ov;
          ci = oi;
        }
      }
      if (tid == 0) {
        const double dkk = double(fabs(ld(k, k)));
        const bool take = ci >= 0 && cv > dkk;
        s_best = take ? cv : dkk;
        s_p = take ? ci : k;
      }
    }
    __syncthreads();
    const double best = s_best;
    const int64_t p = s_p;
    if (blockIdx.x == 0 && tid == 0) {
      piv[k] = p;
      if (best == 0.0 && *d_sing < 0) *d_sing = int(base + k);
    }
    const bool live = !(best == 0.0);
    // every thread has read s_best / s_p (and thread 0 a(k,k)) before the swap
    // overwrites row k and the next column reuses the shared words
    __syncthreads();
    // (c) the swap, by CTA 0
    if (live && p != k && blockIdx.x == 0)
      for (int64_t j = tid; j < n; j += LU_THREADS) {
        const T t = ld(k, j), u = ld(p, j);
        at(k, j) = u;
        at(p, j) = t;
      }
    grid.sync();
    // (d) divide the column by the pivot, rank-1 update of this band
    if (live) {
      const T d = ld(k, k);
      for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
        const T lik = Ops<T>::div(ld(i, k), d);
        at(i, k) = lik;
        // loads batched ahead of the stores (a store may alias a later load,
        // so a load-use-store loop would pay one L2 round trip per element)
        for (int64_t j0 = k + 1; j0 < n; j0 += 16) {
          T xi[16], xk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const bool in = j0 + q < n;
            xi[q] = in ? ld(i, j0 + q) : T(0);
            xk[q] = in ? ld(k, j0 + q) : T(0);
          }
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (j0 + q < n) at(i, j0 + q) = Ops<T>::sub(xi[q], Ops<T>::mul(lik, xk[q]));
        }
      }
    }
    // No barrier here: the next column's band search reads only this CTA's
    // own rows (just updated by its own threads, after the block barrier);
    // everything shared — a(k+1,k+1), the partials, the next swap — comes
    // after the next grid barrier.
    __syncthreads();
  }
}

// Shared-memory variant (the usual case: a leaf panel no wider than 256):
// each CTA keeps its band of rows in shared memory (row stride n+1), and per
// column exactly one grid barrier separates "publish" from "use": every CTA
// publishes its best candidate (value, row) together with that candidate's
// whole row, and the owner of row k publishes row k; after the barrier every
// CTA knows the pivot row's values without another round trip, performs the
// swap on whichever of rows k / p it owns, and updates its band.  Publication
// slots alternate by column parity, so a CTA racing ahead into column k+1
// never overwrites what a slower one still reads for column k.
template <typename T>
__global__ void __launch_bounds__(LU_THREADS) lu_leaf_smem_kernel(T* a, int64_t off, int64_t rs, int64_t cs,
                                                                int64_t m, int64_t n, int64_t* piv, int* d_sing,
                                                                int64_t base, double* part_v, int64_t* part_i,
                                                                T* cand_rows, T* rowk_buf, int pre) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char lu_smem[];
  T* S = reinterpret_cast<T*>(lu_smem);
  const int G = gridDim.x, tid = threadIdx.x, cta = blockIdx.x;
  const int64_t ld = n + 1;
  const int64_t chunk = (m + G - 1) / G;
  const int64_t r0 = int64_t(cta) * chunk, r1 = r0 + chunk < m ? r0 + chunk : m;
  const int64_t rows = r1 > r0 ? r1 - r0 : 0;
  T* newk = S + chunk * ld;  // the pivot row's values for this column
  // pre: every band's candidate row and row k are fetched together with the
  // partial maxima (one L2 round trip after the barrier instead of two)
  T* cand_s = newk + ld;     // G x n (pre only)
  T* rk_s = cand_s + int64_t(G) * n;
  const int64_t steps = m < n ? m : n;
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int64_t red_i[LU_THREADS / 32];
  __shared__ double s_best;
  __shared__ int64_t s_p;
  __shared__ int s_src;  // band whose candidate row is the pivot row (-1: row k itself)
  for (int64_t e = tid; e < rows * n; e += LU_THREADS) {
    const int64_t i = e / n, j = e % n;
    S[i * ld + j] = a[off + (r0 + i) * rs + j * cs];
  }
  __syncthreads();
  for (int64_t k = 0; k < steps; ++k) {
    const int par = int(k & 1);
    double* pv = part_v + par * 32;
    int64_t* pi = part_i + par * 32;
    T* cand = cand_rows + int64_t(par) * 32 * n;
    T* rk = rowk_buf + int64_t(par) * n;
    // publish: this band's best candidate below k, its row, and row k
    double bv = -1.0;
    int64_t bi = -1;
    const int64_t lo = r0 > k + 1 ? r0 : k + 1;
    for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
      const double v = double(fabs(S[(i - r0) * ld + k]));
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (ov > bv || (ov == bv && (bi < 0 || oi < bi)))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_i[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < LU_THREADS / 32; ++w)
        if (red_i[w] >= 0 && (red_v[w] > bv || (red_v[w] == bv && (bi < 0 || red_i[w] < bi)))) {
          bv = red_v[w];
          bi = red_i[w];
        }
      pv[cta] = bv;
      pi[cta] = bi;
      s_p = bi;
    }
    __syncthreads();
    const int64_t mine = s_p;
    if (mine >= 0)
      for (int64_t j = tid; j < n; j += LU_THREADS) cand[int64_t(cta) * n + j] = S[(mine - r0) * ld + j];
    if (k >= r0 && k < r1)
      for (int64_t j = tid; j < n; j += LU_THREADS) rk[j] = S[(k - r0) * ld + j];
    grid.sync();
    if (pre) {
      for (int64_t e = tid; e < int64_t(G) * n; e += LU_THREADS) cand_s[e] = __ldcg(cand + e);
      for (int64_t j = tid; j < n; j += LU_THREADS) rk_s[j] = __ldcg(rk + j);
      __syncthreads();
    }
    // decide: bands in row order from the diagonal entry (one warp, G <= 32)
    if (tid < 32) {
      double cv = -1.0;
      int64_t ci = -1;
      int cc = -1;
      if (tid < G) {
        ci = __ldcg(pi + tid);
        cv = __ldcg(pv + tid);
        cc = tid;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, cv, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, ci, o);
        const int oc = __shfl_down_sync(0xffffffffu, cc, o);
        if (oi >= 0 && (ov > cv || (ov == cv && (ci < 0 || oi < ci)))) {
          cv = ov;
          ci = oi;
          cc = oc;
        }
      }
      if (tid == 0) {
        const double dkk = double(fabs(pre ? rk_s[k] : __ldcg(rk + k)));
        const bool take = ci >= 0 && cv > dkk;
        s_best = take ? cv : dkk;
        s_p = take ? ci : k;
        s_src = take ? cc : -1;
        if (cta == 0) {
          piv[k] = s_p;
          if (s_best == 0.0 && *d_sing < 0) *d_sing = int(base + k);
        }
      }
    }
    __syncthreads();
    const bool live = !(s_best == 0.0);
    const int64_t p = s_p;
    const int src = s_src;
    if (live) {
      // the pivot row (new row k) into shared memory; the swap where it lands
      for (int64_t j = tid; j < n; j += LU_THREADS) {
        const T nk = pre ? (src >= 0 ? cand_s[int64_t(src) * n + j] : rk_s[j])
                         : (src >= 0 ? __ldcg(cand + int64_t(src) * n + j) : __ldcg(rk + j));
        newk[j] = nk;
        if (p != k) {
          if (k >= r0 && k < r1) S[(k - r0) * ld + j] = nk;
          if (p >= r0 && p < r1) S[(p - r0) * ld + j] = pre ? rk_s[j] : __ldcg(rk + j);
        }
      }
      __syncthreads();
      // divide the column by the pivot, rank-1 update of this band
      const T d = newk[k];
      for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
        T* row = S + (i - r0) * ld;
        const T lik = Ops<T>::div(row[k], d);
        row[k] = lik;
        for (int64_t j = k + 1; j < n; ++j) row[j] = Ops<T>::sub(row[j], Ops<T>::mul(lik, newk[j]));
      }
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < rows * n; e += LU_THREADS) {
    const int64_t i = e / n, j = e % n;
    a[off + (r0 + i) * rs + j * cs] = S[i * ld + j];
  }
}

// The same leaf on ONE thread-block cluster (<= 16 CTAs) whose bands hold the
// whole panel in shared memory: per column every CTA publishes its band's
// best candidate (value, row, the row itself) and, for the owner, row k in
// its OWN shared memory (slots alternate by column parity), one cluster
// barrier (~0.2 us instead of a grid barrier), then every CTA reads the
// partials and the winning row straight from its peers' shared memory
// (DSMEM).  No global traffic inside the column loop; identical arithmetic.
__device__ __forceinline__ uint32_t dsmem_map(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ double dsmem_ld_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float dsmem_ld_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int64_t dsmem_ld_s64(uint32_t addr) {
  int64_t v;
  asm volatile("ld.shared::cluster.s64 %0, [%1];\n" : "=l"(v) : "r"(addr));
  return v;
}
template <typename T>
__device__ __forceinline__ T dsmem_ld(uint32_t addr);
template <>
__device__ __forceinline__ double dsmem_ld<double>(uint32_t addr) {
  return dsmem_ld_f64(addr);
}
template <>
__device__ __forceinline__ float dsmem_ld<float>(uint32_t addr) {
  return dsmem_ld_f32(addr);
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <typename T>
__global__ void __launch_bounds__(LU_THREADS) lu_leaf_cluster_kernel(T* a, int64_t off, int64_t rs, int64_t cs,
                                                                   int64_t m, int64_t n, int64_t* piv, int* d_sing,
                                                                   int64_t base, int chunk) {
  extern __shared__ __align__(16) unsigned char lc_smem[];
  const int C = gridDim.x, tid = threadIdx.x;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int64_t ld = n + 1;
  // [pub_v 2][pub_i 2] | band chunk x ld | newk n | pub_row 2 x n | rowk 2 x n
  double* pub_v = reinterpret_cast<double*>(lc_smem);
  int64_t* pub_i = reinterpret_cast<int64_t*>(lc_smem + 16);
  T* S = reinterpret_cast<T*>(lc_smem + 32);
  T* newk = S + int64_t(chunk) * ld;
  T* pub_row = newk + n;
  T* rowk = pub_row + 2 * n;
  const uint32_t base_v = smem_u32(pub_v), base_i = smem_u32(pub_i), base_row = smem_u32(pub_row),
                 base_rk = smem_u32(rowk);
  const int64_t r0 = int64_t(rank) * chunk, r1 = r0 + chunk < m ? r0 + chunk : m;
  const int64_t rows = r1 > r0 ? r1 - r0 : 0;
  const int64_t steps = m < n ? m : n;
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int64_t red_i[LU_THREADS / 32];
  __shared__ double s_best;
  __shared__ int64_t s_p;
  __shared__ int s_src;
  for (int64_t e = tid; e < rows * n; e += LU_THREADS) {
    const int64_t i = e / n, j = e % n;
    S[i * ld + j] = a[off + (r0 + i) * rs + j * cs];
  }
  __syncthreads();
  for (int64_t k = 0; k < steps; ++k) {
    const int par = int(k & 1);
    double bv = -1.0;
    int64_t bi = -1;
    const int64_t lo = r0 > k + 1 ? r0 : k + 1;
    for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
      const double v = double(fabs(S[(i - r0) * ld + k]));
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (oi >= 0 && (ov > bv || (ov == bv && (bi < 0 || oi < bi)))) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_i[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < LU_THREADS / 32; ++w)
        if (red_i[w] >= 0 && (red_v[w] > bv || (red_v[w] == bv && (bi < 0 || red_i[w] < bi)))) {
          bv = red_v[w];
          bi = red_i[w];
        }
      pub_v[par] = bv;
      pub_i[par] = bi;
      s_p = bi;
    }
    __syncthreads();
    const int64_t mine = s_p;
    if (mine >= 0)
      for (int64_t j = tid; j < n; j += LU_THREADS) pub_row[par * n + j] = S[(mine - r0) * ld + j];
    if (k >= r0 && k < r1)
      for (int64_t j = tid; j < n; j += LU_THREADS) rowk[par * n + j] = S[(k - r0) * ld + j];
    cluster_barrier();
    const uint32_t owner_k = uint32_t(k / chunk);
    // decide from the peers' partials, bands in rank (= row) order
    if (tid < 32) {
      double cv = -1.0;
      int64_t ci = -1;
      int cc = -1;
      if (tid < C) {
        cv = dsmem_ld_f64(dsmem_map(base_v + 8u * par, uint32_t(tid)));
        ci = dsmem_ld_s64(dsmem_map(base_i + 8u * par, uint32_t(tid)));
        cc = tid;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, cv, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, ci, o);
        const int oc = __shfl_down_sync(0xffffffffu, cc, o);
        if (oi >= 0 && (ov > cv || (ov == cv && (ci < 0 || oi < ci)))) {
          cv = ov;
          ci = oi;
          cc = oc;
        }
      }
      if (tid == 0) {
        const double dkk =
            double(fabs(dsmem_ld<T>(dsmem_map(base_rk + uint32_t((par * n + k) * sizeof(T)), owner_k))));
        const bool take = ci >= 0 && cv > dkk;
        s_best = take ? cv : dkk;
        s_p = take ? ci : k;
        s_src = take ? cc : -1;
        if (rank == 0) {
          piv[k] = s_p;
          if (s_best == 0.0 && *d_sing < 0) *d_sing = int(base + k);
        }
      }
    }
    __syncthreads();
    const bool live = !(s_best == 0.0);
    const int64_t p = s_p;
    const int src = s_src;
    if (live) {
      for (int64_t j = tid; j < n; j += LU_THREADS) {
        const T rkj = dsmem_ld<T>(dsmem_map(base_rk + uint32_t((par * n + j) * sizeof(T)), owner_k));
        const T nk = src >= 0 ? dsmem_ld<T>(dsmem_map(base_row + uint32_t((par * n + j) * sizeof(T)), uint32_t(src)))
                              : rkj;
        newk[j] = nk;
        if (p != k) {
          if (k >= r0 && k < r1) S[(k - r0) * ld + j] = nk;
          if (p >= r0 && p < r1) S[(p - r0) * ld + j] = rkj;
        }
      }
      __syncthreads();
      const T d = newk[k];
      for (int64_t i = lo + tid; i < r1; i += LU_THREADS) {
        T* row = S + (i - r0) * ld;
        const T lik = Ops<T>::div(row[k], d);
        row[k] = lik;
        for (int64_t j = k + 1; j < n; ++j) row[j] = Ops<T>::sub(row[j], Ops<T>::mul(lik, newk[j]));
      }
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < rows * n; e += LU_THREADS) {
    const int64_t i = e / n, j = e % n;
    a[off + (r0 + i) * rs + j * cs] = S[i * ld + j];
  }
  cluster_barrier();  // no CTA leaves while a peer may still read its shared memory
}

template <typename T>
__global__ void apply_pivots_kernel(T* a, int64_t off, int64_t rs, int64_t cs, int64_t ncols, const int64_t* piv,
                                    int64_t count, int64_t sub, int backward) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T* col = a + off + j * cs;
  for (int64_t q = 0; q < count; ++q) {
    const int64_t k = backward ? count - 1 - q : q;
    const int64_t p = piv[k] - sub;
    if (p != k) {
      const T t = col[k * rs];
      col[k * rs] = col[p * rs];
      col[p * rs] = t;
    }
  }
}

__global__ void add_offset_kernel(int64_t* piv, int64_t count, int64_t delta) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < count) piv[q] += delta;
}

template <typename T>
__global__ void trsm_left_base_kernel(double alpha, const T* t, int64_t toff, int64_t trs, int64_t tcs, T* b,
                                      int64_t boff, int64_t brs, int64_t bcs, int n, int64_t ncols) {
  __shared__ T st[32][33];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, p = e % n;
    st[i][p] = p < i ? t[toff + i * trs + p * tcs] : T(0);
  }
  __syncthreads();
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < n ? b[boff + i * brs + j * bcs] : T(0);
  if (alpha != 1.0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = T(Ops<double>::mul(double(x[i]), alpha));
  }
#pragma unroll
  for (int i = 1; i < 32; ++i) {
    if (i < n) {
      T acc = x[i];
#pragma unroll
      for (int p = 0; p < i; ++p) acc = Ops<T>::sub(acc, Ops<T>::mul(st[i][p], x[p]));
      x[i] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) b[boff + i * brs + j * bcs] = x[i];
}

// upper, non-unit, backward: X = U^-1 B for n <= 32 (lu_solve's last stage)
template <typename T>
__global__ void trsm_upper_base_kernel(const T* u, int64_t uoff, int64_t urs, int64_t ucs, T* b, int64_t boff,
                                       int64_t brs, int64_t bcs, int n, int64_t ncols) {
  __shared__ T su[32][33];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, p = e % n;
    su[i][p] = p >= i ? u[uoff + i * urs + p * ucs] : T(0);
  }
  __syncthreads();
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  T x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < n ? b[boff + i * brs + j * bcs] : T(0);
#pragma unroll
  for (int i = 31; i >= 0; --i) {
    if (i < n) {
      T acc = x[i];
#pragma unroll
      for (int p = i + 1; p < 32; ++p)
        if (p < n) acc = Ops<T>::sub(acc, Ops<T>::mul(su[i][p], x[p]));
      x[i] = Ops<T>::div(acc, su[i][i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) b[boff + i * brs + j * bcs] = x[i];
}

// dst (n x m, row-major ld) = src^T (src m x n, any strides): 32x32 tiles
template <typename T>
__global__ void transpose_kernel(const T* src, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, T* dst,
                                 int64_t ld) {
  __shared__ T tile[32][33];
  const int64_t i0 = int64_t(blockIdx.y) * 32, j0 = int64_t(blockIdx.x) * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < m && j < n) tile[r][threadIdx.x] = src[off + i * rs + j * cs];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < m && j < n) dst[j * ld + i] = tile[threadIdx.x][r];
  }
}

// dst[j*ld + i] = src(i, j) restricted to one triangle of src (tri 1: i >= j,
// 2: i <= j); 32x32 tiles wholly outside it are skipped
template <typename T>
__global__ void transpose_tri_kernel(const T* src, int64_t off, int64_t rs, int64_t cs, int64_t n, T* dst, int64_t ld,
                                     int tri) {
  __shared__ T tile[32][33];
  const int64_t i0 = int64_t(blockIdx.y) * 32, j0 = int64_t(blockIdx.x) * 32;
  if ((tri == 1 && i0 + 31 < j0) || (tri == 2 && j0 + 31 < i0)) return;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < n && j < n) tile[r][threadIdx.x] = src[off + i * rs + j * cs];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < n && j < n && (tri == 0 || (tri == 1 ? i >= j : i <= j))) dst[j * ld + i] = tile[threadIdx.x][r];
  }
}

// W (kt x n, row-major) = T * A^T with the reference's packing arithmetic in T
template <typename T>
__global__ void tridiag_form_kernel(const T* a, int64_t off, int64_t rs, int64_t cs, int64_t n, int64_t kt,
                                    const T* t, T* w) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * kt) return;
  const int64_t g = e / n, j = e % n;
  const T* row = a + off + j * rs;
  T acc = T(0);
  if (g > 0) acc = Ops<T>::add(acc, Ops<T>::mul(t[g - 1], row[(g - 1) * cs]));
  if (g < kt - 1) acc = Ops<T>::sub(acc, Ops<T>::mul(t[g], row[(g + 1) * cs]));
  w[g * n + j] = acc;
}

int grid_cap_lu() {
  static int cap = 0;
  if (!cap) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lu_leaf_kernel<double>, LU_THREADS, 0);
    cap = sms * (per > 0 ? (per < 2 ? per : 2) : 1);
  }
  return cap;
}

}  // namespace

int launch_lu_leaf(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, int64_t* piv,
                   int* d_sing, int64_t base, cudaStream_t s) {
  const int64_t steps = m < n ? m : n;
  if (steps <= 0) return 0;
  // a few hundred rows per CTA: the leaf moves little data, and every grid
  // barrier costs more with more CTAs
  int G = int((m + 383) / 384);
  // <= 32 bands: one warp combines the partials
  const int cap = g_lu_grid_max > 0 && g_lu_grid_max < 32 ? g_lu_grid_max : (grid_cap_lu() < 32 ? grid_cap_lu() : 32);
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  static double* part_v[64] = {};
  static int64_t* part_i[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -3;
  if (!part_v[dev]) {
    if (cudaMalloc(&part_v[dev], 4096 * sizeof(double)) != cudaSuccess) return -12;
    if (cudaMalloc(&part_i[dev], 4096 * sizeof(int64_t)) != cudaSuccess) return -12;
  }
  if (G > 4096) G = 4096;
  double* pv = part_v[dev];
  int64_t* pi = part_i[dev];
  // one cluster when the whole panel fits in its shared memory
  if (!g_lu_global && !g_lu_nocluster && n <= 1024) {
    const size_t esz = is_f64 ? 8 : 4;
    const size_t budget = 200 * 1024;
    const size_t fixed = 32 + size_t(5 * n) * esz;  // partial slots, newk, 2 published rows, 2 rows k
    const int64_t max_rows = budget > fixed ? int64_t((budget - fixed) / (size_t(n + 1) * esz)) : 0;
    int64_t Cn = max_rows > 0 ? (m + max_rows - 1) / max_rows : 1 << 30;
    const int64_t want = (m + 383) / 384;  // a few hundred rows per CTA
    if (Cn < want) Cn = want;
    if (Cn < 1) Cn = 1;
    if (Cn <= g_lu_cluster_max) {
      const int C = int(Cn);
      const int chunk = int((m + C - 1) / C);
      const size_t smem = fixed + size_t(chunk) * size_t(n + 1) * esz;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(LU_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e;
      if (is_f64) {
        smem_attr(reinterpret_cast<const void*>(lu_leaf_cluster_kernel<double>), 210 * 1024);
        cudaFuncSetAttribute(lu_leaf_cluster_kernel<double>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e = cudaLaunchKernelEx(&cfg, lu_leaf_cluster_kernel<double>, static_cast<double*>(a), off, rs, cs, m, n, piv,
                               d_sing, base, chunk);
      } else {
        smem_attr(reinterpret_cast<const void*>(lu_leaf_cluster_kernel<float>), 210 * 1024);
        cudaFuncSetAttribute(lu_leaf_cluster_kernel<float>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e = cudaLaunchKernelEx(&cfg, lu_leaf_cluster_kernel<float>, static_cast<float*>(a), off, rs, cs, m, n, piv,
                               d_sing, base, chunk);
      }
      if (e == cudaSuccess) {
        note_launch();
        return 0;
      }
      (void)cudaGetLastError();  // not schedulable as one cluster here: the grid kernels below
    }
  }
  note_launch();
  cudaError_t e;
  // shared-memory bands when they fit: <= 32 bands of <= ~190 KB each
  {
    const size_t esz = is_f64 ? 8 : 4;
    const int64_t max_rows = int64_t((190 * 1024) / (size_t(n + 1) * esz)) - 1;
    int64_t Gs = max_rows > 0 ? (m + max_rows - 1) / max_rows : 1 << 30;
    const int64_t want = (m + 255) / 256;  // ~256 rows per band when there is room
    if (Gs < want) Gs = want;
    if (Gs > 32) Gs = 32;
    const int64_t chunk = (m + Gs - 1) / Gs;
    int pre = n <= 128 && !g_lu_noprefetch;
    const size_t smem = size_t(chunk + 1) * size_t(n + 1) * esz + (pre ? size_t(Gs + 1) * size_t(n) * esz : 0);
    static void* cand_buf[64] = {};
    static size_t cand_cap[64] = {};
    const size_t need = size_t(2) * 33 * size_t(n) * esz;
    if (n <= 4096 && chunk * (n + 1) * int64_t(esz) <= int64_t(190 * 1024) && smem <= 200 * 1024 && !g_lu_global) {
      if (cand_cap[dev] < need) {
        if (cand_buf[dev]) cudaFree(cand_buf[dev]);
        if (cudaMalloc(&cand_buf[dev], need) != cudaSuccess) return -12;
        cand_cap[dev] = need;
      }
      void* cand = cand_buf[dev];
      void* rowk = static_cast<char*>(cand) + size_t(2) * 32 * size_t(n) * esz;
      const int Gi = int(Gs);
      if (is_f64) {
        smem_attr(reinterpret_cast<const void*>(lu_leaf_smem_kernel<double>), 200 * 1024);
        double* ad = static_cast<double*>(a);
        double* cd = static_cast<double*>(cand);
        double* rd = static_cast<double*>(rowk);
        void* args[] = {&ad, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi, &cd, &rd, &pre};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_smem_kernel<double>), dim3(Gi),
                                        dim3(LU_THREADS), args, smem, s);
      } else {
        smem_attr(reinterpret_cast<const void*>(lu_leaf_smem_kernel<float>), 200 * 1024);
        float* af = static_cast<float*>(a);
        float* cf = static_cast<float*>(cand);
        float* rf = static_cast<float*>(rowk);
        void* args[] = {&af, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi, &cf, &rf, &pre};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_smem_kernel<float>), dim3(Gi),
                                        dim3(LU_THREADS), args, smem, s);
      }
      return e == cudaSuccess ? 0 : -11;
    }
  }
  if (is_f64) {
    double* ad = static_cast<double*>(a);
    void* args[] = {&ad, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_kernel<double>), dim3(G), dim3(LU_THREADS), args,
                                    0, s);
  } else {
    float* af = static_cast<float*>(a);
    void* args[] = {&af, &off, &rs, &cs, &m, &n, &piv, &d_sing, &base, &pv, &pi};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_leaf_kernel<float>), dim3(G), dim3(LU_THREADS), args, 0,
                                    s);
  }
  return e == cudaSuccess ? 0 : -11;
}

int launch_apply_pivots(int is_f64, void* a, int64_t off, int64_t rs, int64_t cs, int64_t ncols, const int64_t* piv,
                        int64_t count, int64_t sub, int backward, cudaStream_t s) {
  if (ncols <= 0 || count <= 0) return 0;
  note_launch();
  const unsigned blocks = unsigned((ncols + 255) / 256);
  if (is_f64)
    apply_pivots_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(a), off, rs, cs, ncols, piv, count, sub,
                                                       backward);
  else
    apply_pivots_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(a), off, rs, cs, ncols, piv, count, sub,
                                                      backward);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_transpose(int is_f64, const void* src, int64_t off, int64_t rs, int64_t cs, int64_t m, int64_t n, void* dst,
                     int64_t ld, cudaStream_t s) {
  if (m <= 0 || n <= 0) return 0;
  note_launch();
  const dim3 grid(unsigned((n + 31) / 32), unsigned((m + 31) / 32)), block(32, 8);
  if (is_f64)
    transpose_kernel<double><<<grid, block, 0, s>>>(static_cast<const double*>(src), off, rs, cs, m, n,
                                                    static_cast<double*>(dst), ld);
  else
    transpose_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(src), off, rs, cs, m, n,
                                                   static_cast<float*>(dst), ld);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_transpose_tri_f64(const double* src, int64_t off, int64_t rs, int64_t cs, int64_t n, double* dst,
                             int64_t ld, int tri, cudaStream_t s) {
  if (n <= 0) return 0;
  note_launch();
  const dim3 grid(unsigned((n + 31) / 32), unsigned((n + 31) / 32)), block(32, 8);
  transpose_tri_kernel<double><<<grid, block, 0, s>>>(src, off, rs, cs, n, dst, ld, tri);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_tridiag_form_f32(const float* a, int64_t off, int64_t rs, int64_t cs, int64_t n, int64_t kt, const float* t,
                            float* w, cudaStream_t s) {
  if (n <= 0 || kt <= 0) return 0;
  note_launch();
  tridiag_form_kernel<float><<<unsigned((n * kt + 255) / 256), 256, 0, s>>>(a, off, rs, cs, n, kt, t, w);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_add_offset(int64_t* piv, int64_t count, int64_t delta, cudaStream_t s) {
  if (count <= 0 || delta == 0) return 0;
  note_launch();
  add_offset_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(piv, count, delta);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_trsm_left_base(int is_f64, double alpha, const void* t, int64_t toff, int64_t trs, int64_t tcs, void* b,
                          int64_t boff, int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s) {
  if (ncols <= 0 || n <= 0) return 0;
  if (n > 32) return -3;
  note_launch();
  const unsigned blocks = unsigned((ncols + 127) / 128);
  if (is_f64)
    trsm_left_base_kernel<double><<<blocks, 128, 0, s>>>(alpha, static_cast<const double*>(t), toff, trs, tcs,
                                                         static_cast<double*>(b), boff, brs, bcs, n, ncols);
  else
    trsm_left_base_kernel<float><<<blocks, 128, 0, s>>>(alpha, static_cast<const float*>(t), toff, trs, tcs,
                                                        static_cast<float*>(b), boff, brs, bcs, n, ncols);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int launch_trsm_upper_base(int is_f64, const void* u, int64_t uoff, int64_t urs, int64_t ucs, void* b, int64_t boff,
                           int64_t brs, int64_t bcs, int n, int64_t ncols, cudaStream_t s) {
  if (ncols <= 0 || n <= 0) return 0;
  if (n > 32) return -3;
  note_launch();
  const unsigned blocks = unsigned((ncols + 127) / 128);
  if (is_f64)
    trsm_upper_base_kernel<double><<<blocks, 128, 0, s>>>(static_cast<const double*>(u), uoff, urs, ucs,
                                                          static_cast<double*>(b), boff, brs, bcs, n, ncols);
  else
    trsm_upper_base_kernel<float><<<blocks, 128, 0, s>>>(static_cast<const float*>(u), uoff, urs, ucs,
                                                         static_cast<float*>(b), boff, brs, bcs, n, ncols);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace bf
