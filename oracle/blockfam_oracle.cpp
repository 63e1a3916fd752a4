// ORACLE — CPU restatement of the reference blockfam hot path.  TEST
// INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs as the checker or the
// timed CPU baseline; the product never links or calls it.
//
// Parity pinned: tests/test_oracle_golden.py checks every function here
// bit-for-bit against outputs of the reference itself
// (tests/golden/*.npz, made by tools/gen_golden.py from /root/reference).
//
// Each routine restates the reference's arithmetic exactly:
//   * gemm: engine/gemm.py:74-160 + engine/kernels.py:142-255 — the k range is
//     cut into kc segments; every C element's segment sum is an ascending fma
//     chain from +0 (micro-kernel compiled with fastmath={"contract"},
//     engine/kernels.py:169-172); the segment is folded into C with the
//     unfused C = beta_eff*C + alpha*t (engine/kernels.py:228-253).
//   * leaves: factor/cholesky.py:31-89 with numba's typing (sums that start
//     at the literal 0.0 are f64 even for f32 storage).
//   * trsm: engine/trsm.py:51-68 recursion, base engine/trsm.py:96-111.
//   * cholesky: factor/cholesky.py:99-158.
//   * gemm_naive: oracle/reference.py:23-53 (unfused f64 accumulation).
// Built with -ffp-contract=off so only the explicit std::fma calls fuse.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

template <typename T>
struct View {
  T* base;
  int64_t off, m, n, rs, cs;
  T& at(int64_t i, int64_t j) const { return base[off + i * rs + j * cs]; }
  View sub(int64_t r0, int64_t nr, int64_t c0, int64_t nc) const {
    return View{base, off + r0 * rs + c0 * cs, nr, nc, rs, cs};
  }
  View t() const { return View{base, off, n, m, cs, rs}; }
};

// Generic element addressing: strided, or scatter vectors when given.
template <typename T>
struct Operand {
  const T* base;
  int64_t off, rs, cs;
  const int64_t* rscat;
  const int64_t* cscat;
  T get(int64_t i, int64_t j) const { return rscat ? base[rscat[i] + cscat[j]] : base[off + i * rs + j * cs]; }
};
template <typename T>
struct OutOperand {
  T* base;
  int64_t off, rs, cs;
  const int64_t* rscat;
  const int64_t* cscat;
  T& at(int64_t i, int64_t j) const { return rscat ? base[rscat[i] + cscat[j]] : base[off + i * rs + j * cs]; }
};

inline float fma_t(float a, float b, float c) { return std::fmaf(a, b, c); }
inline double fma_t(double a, double b, double c) { return std::fma(a, b, c); }

constexpr int MR = 4, NR = 8;

// One kc segment over row block [i0, i1) and all columns: packed A/B,
// register tiles of MR x NR, ascending-k fma chains, unfused fold.
template <typename T, typename Acc>
void segment_rows(const Operand<T>& A, const Operand<T>& B, const OutOperand<T>& C, int64_t i0, int64_t i1,
                  int64_t n, int64_t k0, int64_t klen, Acc alpha, Acc beta_eff, bool lower, const Acc* bpack,
                  std::vector<Acc>& apack) {
  const int64_t np = (n + NR - 1) / NR;
  for (int64_t ib = i0; ib < i1; ib += MR) {
    const int64_t im = (i1 - ib) < MR ? (i1 - ib) : MR;
    if (lower && ib + im - 1 < 0) continue;
    // pack A rows ib..ib+im, k-major, zero padded
    apack.assign(size_t(MR) * klen, Acc(0));
    for (int64_t kk = 0; kk < klen; ++kk)
      for (int64_t i = 0; i < im; ++i) apack[kk * MR + i] = Acc(A.get(ib + i, k0 + kk));
    for (int64_t jp = 0; jp < np; ++jp) {
      const int64_t jb = jp * NR;
      const int64_t jn = (n - jb) < NR ? (n - jb) : NR;
      if (lower && ib + im - 1 < jb) continue;
      // The micro-kernel's accumulators start from the literal 0.0, so they
      // are f64 even when the packed operands are f32: with f32 packing the
      // product is rounded to f32 and added in f64; with f64 packing the
      // multiply-add contracts to an f64 fma (engine/kernels.py:507-522).
      double acc[MR][NR];
      for (int i = 0; i < MR; ++i)
        for (int j = 0; j < NR; ++j) acc[i][j] = 0.0;
      const Acc* bp = bpack + jp * (NR * klen);
      const Acc* ap = apack.data();
      for (int64_t kk = 0; kk < klen; ++kk) {
        const Acc* brow = bp + kk * NR;
        const Acc* acol = ap + kk * MR;
        for (int i = 0; i < MR; ++i) {
          const Acc av = acol[i];
          if constexpr (sizeof(Acc) == 4) {
            for (int j = 0; j < NR; ++j) acc[i][j] = acc[i][j] + double(Acc(av * brow[j]));
          } else {
            for (int j = 0; j < NR; ++j) acc[i][j] = fma_t(av, brow[j], acc[i][j]);
          }
        }
      }
      for (int64_t i = 0; i < im; ++i) {
        const int64_t gi = ib + i;
        for (int64_t j = 0; j < jn; ++j) {
          const int64_t gj = jb + j;
          if (lower && gi < gj) continue;
          T& c = C.at(gi, gj);
          Acc t = alpha * Acc(acc[i][j]);  // tile[] is an acc-dtype array
          if (beta_eff == Acc(0))
            c = T(t);
          else {
            Acc bc = beta_eff * Acc(c);
            c = T(bc + t);
          }
        }
      }
    }
  }
}

template <typename T, typename Acc>
int gemm_impl(double alpha_in, const Operand<T>& A, const Operand<T>& B, double beta_in, const OutOperand<T>& C,
              int64_t m, int64_t n, int64_t k, int lower, int64_t kc, int nthreads) {
  if (m == 0 || n == 0) return 0;
  const Acc alpha = Acc(alpha_in), beta = Acc(beta_in);
  if (alpha == Acc(0) && beta == Acc(1)) return 0;
  if (k == 0 || alpha == Acc(0)) {
    if (beta != Acc(1)) {
      for (int64_t i = 0; i < m; ++i) {
        int64_t jmax = (lower && i + 1 < n) ? i + 1 : n;
        for (int64_t j = 0; j < jmax; ++j) {
          T& c = C.at(i, j);
          c = (beta == Acc(0)) ? T(0) : T(beta * Acc(c));
        }
      }
    }
    return 0;
  }
  if (nthreads < 1) nthreads = 1;
  const int64_t np = (n + NR - 1) / NR;
  std::vector<Acc> bpack;
  for (int64_t k0 = 0, seg = 0; k0 < k; k0 += kc, ++seg) {
    const int64_t klen = (k - k0) < kc ? (k - k0) : kc;
    const Acc beta_eff = seg == 0 ? beta : Acc(1);
    bpack.assign(size_t(np) * NR * klen, Acc(0));
    for (int64_t jp = 0; jp < np; ++jp)
      for (int64_t kk = 0; kk < klen; ++kk)
        for (int64_t j = 0; j < NR && jp * NR + j < n; ++j)
          bpack[jp * NR * klen + kk * NR + j] = Acc(B.get(k0 + kk, jp * NR + j));
    // rows split in contiguous MR-aligned chunks (engine/team.py:19-30)
    const int64_t panels = (m + MR - 1) / MR;
    const int nt = int(panels < nthreads ? panels : nthreads);
    auto work = [&](int w) {
      std::vector<Acc> apack;
      const int64_t base = panels / nt, extra = panels % nt;
      const int64_t p0 = w * base + (w < extra ? w : extra);
      const int64_t p1 = p0 + base + (w < extra ? 1 : 0);
      segment_rows<T, Acc>(A, B, C, p0 * MR, (p1 * MR < m ? p1 * MR : m), n, k0, klen, alpha, beta_eff, lower != 0,
                           bpack.data(), apack);
    };
    if (nt == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int w = 0; w < nt; ++w) pool.emplace_back(work, w);
      for (auto& th : pool) th.join();
    }
  }
  return 0;
}

template <typename T>
Operand<T> opnd(const View<T>& v) {
  return Operand<T>{v.base, v.off, v.rs, v.cs, nullptr, nullptr};
}
template <typename T>
OutOperand<T> out(const View<T>& v) {
  return OutOperand<T>{v.base, v.off, v.rs, v.cs, nullptr, nullptr};
}

template <typename T, typename Acc>
int gemm_view(double alpha, const View<T>& a, const View<T>& b, double beta, const View<T>& c, int lower, int64_t kc,
              int nthreads) {
  if (a.n != b.m || c.m != a.m || c.n != b.n) return -1;
  return gemm_impl<T, Acc>(alpha, opnd(a), opnd(b), beta, out(c), c.m, c.n, a.n, lower, kc, nthreads);
}

// ---- leaves (factor/cholesky.py:31-89) ------------------------------------
template <typename T>
int leaf1(const View<T>& a) {
  const int64_t n = a.n;
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t p = 0; p < j; ++p) s = s + double(T(a.at(k, p) * a.at(j, p)));
      a.at(k, j) = T((double(a.at(k, j)) - s) / double(a.at(j, j)));
    }
    double s = 0.0;
    for (int64_t p = 0; p < k; ++p) {
      T v = a.at(k, p);
      s = s + double(T(v * v));
    }
    double d = double(a.at(k, k)) - s;
    if (!(d > 0.0)) return int(k);
    a.at(k, k) = T(std::sqrt(d));
  }
  return -1;
}
template <typename T>
int leaf2(const View<T>& a) {
  const int64_t n = a.n;
  for (int64_t k = 0; k < n; ++k) {
    double s = 0.0;
    for (int64_t p = 0; p < k; ++p) {
      T v = a.at(k, p);
      s = s + double(T(v * v));
    }
    double d = double(a.at(k, k)) - s;
    if (!(d > 0.0)) return int(k);
    d = std::sqrt(d);
    a.at(k, k) = T(d);
    for (int64_t i = k + 1; i < n; ++i) {
      double si = 0.0;
      for (int64_t p = 0; p < k; ++p) si = si + double(T(a.at(i, p) * a.at(k, p)));
      a.at(i, k) = T((double(a.at(i, k)) - si) / d);
    }
  }
  return -1;
}
template <typename T>
int leaf3(const View<T>& a) {
  const int64_t n = a.n;
  for (int64_t k = 0; k < n; ++k) {
    T d = a.at(k, k);
    if (!(d > T(0))) return int(k);
    d = std::sqrt(d);
    a.at(k, k) = d;
    for (int64_t i = k + 1; i < n; ++i) a.at(i, k) = a.at(i, k) / d;
    for (int64_t j = k + 1; j < n; ++j) {
      const T ajk = a.at(j, k);
      for (int64_t i = j; i < n; ++i) a.at(i, j) = a.at(i, j) - T(a.at(i, k) * ajk);
    }
  }
  return -1;
}
template <typename T>
int leaf(const View<T>& a, int variant) {
  if (variant == 1) return leaf1(a);
  if (variant == 2) return leaf2(a);
  return leaf3(a);
}

// ---- trsm (engine/trsm.py:51-68, 96-111) ----------------------------------
template <typename T>
int trsm_base(double alpha, const View<T>& t, const View<T>& b) {
  if (alpha != 1.0)
    for (int64_t i = 0; i < b.m; ++i)
      for (int64_t j = 0; j < b.n; ++j) b.at(i, j) = T(double(b.at(i, j)) * alpha);
  for (int64_t j = 0; j < b.n; ++j) {
    const T d = t.at(j, j);
    if (d == T(0)) return int(j);
    for (int64_t i = 0; i < b.m; ++i) {
      T acc = b.at(i, j);
      for (int64_t p = 0; p < j; ++p) acc = acc - T(b.at(i, p) * t.at(j, p));
      b.at(i, j) = acc / d;
    }
  }
  return -1;
}

template <typename T>
int trsm_rec(double alpha, const View<T>& tri, const View<T>& b, int64_t kc, int nthreads) {
  const int64_t n = tri.n;
  if (b.m == 0 || n == 0) return -1;
  if (n <= 32) return trsm_base(alpha, tri, b);
  const int64_t n1 = n / 2, n2 = n - n1;
  int bad = trsm_rec(alpha, tri.sub(0, n1, 0, n1), b.sub(0, b.m, 0, n1), kc, nthreads);
  if (bad >= 0) return bad;
  gemm_view<T, T>(-1.0, b.sub(0, b.m, 0, n1), tri.sub(n1, n2, 0, n1).t(), alpha, b.sub(0, b.m, n1, n2), 0, kc,
                  nthreads);
  return trsm_rec(1.0, tri.sub(n1, n2, n1, n2), b.sub(0, b.m, n1, n2), kc, nthreads);
}

struct Level {
  int32_t variant, pad_;
  int64_t bs, kc;
};

// factor/cholesky.py:118-158; returns the global failing index or -1
template <typename T>
int64_t chol_run(const View<T>& a, const Level* lv, int nl, int idx, int64_t base, int nthreads) {
  const int64_t n = a.n;
  if (n == 0) return -1;
  Level node = idx < nl ? lv[idx] : Level{13, 0, 0, idx > 0 ? lv[idx - 1].kc : 256};
  if (node.variant >= 11) {
    int bad = leaf(a, node.variant - 10);
    return bad >= 0 ? base + bad : -1;
  }
  const int64_t bs = node.bs, kc = node.kc;
  for (int64_t done = 0; done < n;) {
    const int64_t b = bs < n - done ? bs : n - done;
    const int64_t r2 = done + b, nr2 = n - r2;
    View<T> a00 = a.sub(0, done, 0, done), a10 = a.sub(done, b, 0, done), a11 = a.sub(done, b, done, b);
    View<T> a20 = a.sub(r2, nr2, 0, done), a21 = a.sub(r2, nr2, done, b), a22 = a.sub(r2, nr2, r2, nr2);
    int64_t bad = -1;
    if (node.variant == 1) {
      trsm_rec(1.0, a00, a10, kc, nthreads);
      gemm_view<T, T>(-1.0, a10, a10.t(), 1.0, a11, 1, kc, nthreads);
      bad = chol_run(a11, lv, nl, idx + 1, base + done, nthreads);
    } else if (node.variant == 2) {
      gemm_view<T, T>(-1.0, a10, a10.t(), 1.0, a11, 1, kc, nthreads);
      bad = chol_run(a11, lv, nl, idx + 1, base + done, nthreads);
      if (bad < 0) {
        gemm_view<T, T>(-1.0, a20, a10.t(), 1.0, a21, 0, kc, nthreads);
        trsm_rec(1.0, a11, a21, kc, nthreads);
      }
    } else {
      bad = chol_run(a11, lv, nl, idx + 1, base + done, nthreads);
      if (bad < 0) {
        trsm_rec(1.0, a11, a21, kc, nthreads);
        gemm_view<T, T>(-1.0, a21, a21.t(), 1.0, a22, 1, kc, nthreads);
      }
    }
    if (bad >= 0) return bad;
    done += b;
  }
  return -1;
}

// ---- LU with partial pivoting (factor/lu.py:19-53, 70-103) ----------------
// pivots (factor/pivots.py:46-61): forward = ascending swap order
template <typename T>
void apply_pivots(const View<T>& a, const int64_t* piv, int64_t count, bool backward) {
  for (int64_t q = 0; q < count; ++q) {
    const int64_t k = backward ? count - 1 - q : q;
    const int64_t p = piv[k];
    if (p == k) continue;
    for (int64_t j = 0; j < a.n; ++j) std::swap(a.at(k, j), a.at(p, j));
  }
}

// engine/trsm.py:114-125: unit lower, row by row, one ascending chain per element
template <typename T>
void trsm_left_base(double alpha, const View<T>& t, const View<T>& b) {
  if (alpha != 1.0)
    for (int64_t i = 0; i < t.n; ++i)
      for (int64_t c = 0; c < b.n; ++c) b.at(i, c) = T(double(b.at(i, c)) * alpha);
  for (int64_t i = 1; i < t.n; ++i)
    for (int64_t c = 0; c < b.n; ++c) {
      T acc = b.at(i, c);
      for (int64_t p = 0; p < i; ++p) acc = acc - T(t.at(i, p) * b.at(p, c));
      b.at(i, c) = acc;
    }
}

// engine/trsm.py:71-88
template <typename T>
void trsm_left_rec(double alpha, const View<T>& tri, const View<T>& b, int64_t kc, int nthreads) {
  const int64_t n = tri.n;
  if (b.n == 0 || n == 0) return;
  if (n <= 32) {
    trsm_left_base(alpha, tri, b);
    return;
  }
  const int64_t n1 = n / 2, n2 = n - n1;
  trsm_left_rec(alpha, tri.sub(0, n1, 0, n1), b.sub(0, n1, 0, b.n), kc, nthreads);
  gemm_view<T, T>(-1.0, tri.sub(n1, n2, 0, n1), b.sub(0, n1, 0, b.n), alpha, b.sub(n1, n2, 0, b.n), 0, kc, nthreads);
  trsm_left_rec(1.0, tri.sub(n1, n2, n1, n2), b.sub(n1, n2, 0, b.n), kc, nthreads);
}

// factor/lu.py:19-53: ties keep the smallest row; a zero pivot column is skipped
template <typename T>
int64_t lu_leaf(const View<T>& a, int64_t* piv) {
  const int64_t m = a.m, n = a.n, steps = m < n ? m : n;
  int64_t sing = -1;
  for (int64_t k = 0; k < steps; ++k) {
    int64_t p = k;
    T best = std::fabs(a.at(k, k));
    for (int64_t i = k + 1; i < m; ++i) {
      const T v = std::fabs(a.at(i, k));
      if (v > best) {
        best = v;
        p = i;
      }
    }
    piv[k] = p;
    if (best == T(0)) {
      if (sing < 0) sing = k;
      continue;
    }
    if (p != k)
      for (int64_t j = 0; j < n; ++j) std::swap(a.at(k, j), a.at(p, j));
    const T d = a.at(k, k);
    for (int64_t i = k + 1; i < m; ++i) a.at(i, k) = a.at(i, k) / d;
    for (int64_t j = k + 1; j < n; ++j) {
      const T u = a.at(k, j);
      for (int64_t i = k + 1; i < m; ++i) a.at(i, j) = a.at(i, j) - T(a.at(i, k) * u);
    }
  }
  return sing;
}

// factor/lu.py:70-103; level variant 20 = blocked, 21 = unblocked leaf
template <typename T>
int64_t lu_run(const View<T>& a, const Level* lv, int nl, int idx, int64_t* piv, int64_t base, int nthreads) {
  const int64_t m = a.m, n = a.n, steps = m < n ? m : n;
  if (steps == 0) return -1;
  Level node = idx < nl ? lv[idx] : Level{21, 0, 0, idx > 0 ? lv[idx - 1].kc : 256};
  if (node.variant == 21) {
    const int64_t sing = lu_leaf(a, piv);
    return sing < 0 ? -1 : base + sing;
  }
  const int64_t bs = node.bs, kc = node.kc;
  int64_t first = -1;
  std::vector<int64_t> local;
  for (int64_t k = 0; k < steps; k += bs) {
    const int64_t b = bs < steps - k ? bs : steps - k;
    local.assign(size_t(b), 0);
    for (int64_t q = 0; q < b; ++q) local[size_t(q)] = q;
    const int64_t sing = lu_run(a.sub(k, m - k, k, b), lv, nl, idx + 1, local.data(), base + k, nthreads);
    if (sing >= 0 && first < 0) first = sing;
    for (int64_t q = 0; q < b; ++q) piv[k + q] = k + local[size_t(q)];
    apply_pivots(a.sub(k, m - k, 0, k), local.data(), b, false);
    apply_pivots(a.sub(k, m - k, k + b, n - k - b), local.data(), b, false);
    if (k + b < n) {
      const View<T> a12 = a.sub(k, b, k + b, n - k - b);
      trsm_left_rec(1.0, a.sub(k, b, k, b), a12, kc, nthreads);
      if (k + b < m)
        gemm_view<T, T>(-1.0, a.sub(k + b, m - k - b, k, b), a12, 1.0, a.sub(k + b, m - k - b, k + b, n - k - b), 0,
                        kc, nthreads);
    }
  }
  return first;
}

// ---- skew sandwich (engine/gemm.py:245-280, kernels.py:93-122) ------------
template <typename T>
void sandwich(const View<T>& c, const View<T>& a, const T* t, int64_t kc, int nthreads) {
  const int64_t n = c.m, kt = a.n;
  if (n == 0 || kt == 0) return;
  std::vector<T> w(size_t(kt * n));
  for (int64_t g = 0; g < kt; ++g)
    for (int64_t j = 0; j < n; ++j) {
      T acc = T(0);
      if (g > 0) acc = acc + T(t[g - 1] * a.at(j, g - 1));
      if (g < kt - 1) acc = acc - T(t[g] * a.at(j, g + 1));
      w[size_t(g * n + j)] = acc;
    }
  View<T> wv{w.data(), 0, kt, n, n, 1};
  gemm_view<T, T>(-1.0, a, wv, 1.0, c, 1, kc, nthreads);
}

// ---- ltlt_pivoted unblocked (factor/ltlt.py:66-88, 157-182) ----------------
template <typename T>
void swap_lower(const View<T>& x, int64_t a, int64_t b) {
  if (a == b) return;
  for (int64_t q = 0; q < a; ++q) std::swap(x.at(a, q), x.at(b, q));
  std::vector<T> mid;
  for (int64_t i = a + 1; i < b; ++i) mid.push_back(x.at(i, a));
  for (int64_t i = a + 1; i < b; ++i) x.at(i, a) = -x.at(b, i);
  for (int64_t i = a + 1; i < b; ++i) x.at(b, i) = -mid[size_t(i - a - 1)];
  x.at(b, a) = -x.at(b, a);
  for (int64_t i = b + 1; i < x.m; ++i) std::swap(x.at(i, a), x.at(i, b));
}

template <typename T>
void ltlt_unblocked(const View<T>& x, int64_t* piv, T* t) {
  const int64_t n = x.n;
  std::vector<T> mvec(size_t(n), T(0)), wvec(size_t(n), T(0));
  for (int64_t j = 0; j + 1 < n; ++j) {
    int64_t p = j + 1;
    T best = std::fabs(x.at(j + 1, j));
    for (int64_t i = j + 2; i < n; ++i) {
      const T v = std::fabs(x.at(i, j));
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (p != j + 1) {
      swap_lower(x, j + 1, p);
      piv[j + 1] = p;
    }
    const T alpha = x.at(j + 1, j);
    t[j] = alpha;
    if (j + 2 >= n) continue;
    for (int64_t i = j + 2; i < n; ++i) {
      const T m = alpha != T(0) ? x.at(i, j) / alpha : T(0);
      mvec[size_t(i)] = m;
      wvec[size_t(i)] = x.at(i, j + 1);
      x.at(i, j) = m;
    }
    if (alpha != T(0))
      for (int64_t c = j + 2; c < n; ++c) {
        const T wc = wvec[size_t(c)], mc = mvec[size_t(c)];
        for (int64_t i = c + 1; i < n; ++i)
          x.at(i, c) = x.at(i, c) + T(T(mvec[size_t(i)] * wc) - T(wvec[size_t(i)] * mc));
      }
  }
}

}  // namespace

struct orc_view_d {
  double* base;
  int64_t off, m, n, rs, cs;
};
struct orc_view_s {
  float* base;
  int64_t off, m, n, rs, cs;
};

static View<double> V(const orc_view_d* v) { return View<double>{v->base, v->off, v->m, v->n, v->rs, v->cs}; }
static View<float> V(const orc_view_s* v) { return View<float>{v->base, v->off, v->m, v->n, v->rs, v->cs}; }

extern "C" {

int orc_gemm_d(double alpha, const orc_view_d* a, const orc_view_d* b, double beta, const orc_view_d* c, int lower,
               int64_t kc, int nthreads) {
  return gemm_view<double, double>(alpha, V(a), V(b), beta, V(c), lower, kc, nthreads);
}
int orc_gemm_s(double alpha, const orc_view_s* a, const orc_view_s* b, double beta, const orc_view_s* c, int lower,
               int64_t kc, int nthreads) {
  return gemm_view<float, float>(alpha, V(a), V(b), beta, V(c), lower, kc, nthreads);
}
int orc_gemm_sd(double alpha, const orc_view_s* a, const orc_view_s* b, double beta, const orc_view_s* c, int lower,
                int64_t kc, int nthreads) {
  return gemm_view<float, double>(alpha, V(a), V(b), beta, V(c), lower, kc, nthreads);
}

int orc_gemm_scatter_d(double alpha, const double* abuf, const int64_t* ar, const int64_t* ac, const double* bbuf,
                       const int64_t* br, const int64_t* bc, double beta, double* cbuf, const int64_t* cr,
                       const int64_t* cc, int64_t m, int64_t n, int64_t k, int64_t kc, int nthreads) {
  return gemm_impl<double, double>(alpha, Operand<double>{abuf, 0, 0, 0, ar, ac}, Operand<double>{bbuf, 0, 0, 0, br, bc},
                                   beta, OutOperand<double>{cbuf, 0, 0, 0, cr, cc}, m, n, k, 0, kc, nthreads);
}

int orc_potrf_leaf_d(const orc_view_d* a, int variant) { return leaf(V(a), variant); }
int orc_potrf_leaf_s(const orc_view_s* a, int variant) { return leaf(V(a), variant); }

int orc_trsm_rltn_d(double alpha, const orc_view_d* t, const orc_view_d* b, int64_t kc, int nthreads) {
  return trsm_rec(alpha, V(t), V(b), kc, nthreads);
}
int orc_trsm_rltn_s(double alpha, const orc_view_s* t, const orc_view_s* b, int64_t kc, int nthreads) {
  return trsm_rec(alpha, V(t), V(b), kc, nthreads);
}

int64_t orc_cholesky_d(const orc_view_d* a, const Level* lv, int nl, int nthreads) {
  return chol_run(V(a), lv, nl, 0, 0, nthreads);
}
int64_t orc_cholesky_s(const orc_view_s* a, const Level* lv, int nl, int nthreads) {
  return chol_run(V(a), lv, nl, 0, 0, nthreads);
}

// oracle/reference.py:23-53 gemm_naive: textbook triple loop, unfused f64 accumulation
void orc_gemm_naive_d(double alpha, const orc_view_d* a, const orc_view_d* b, double beta, const orc_view_d* c) {
  View<double> A = V(a), B = V(b), C = V(c);
  if (C.m == 0 || C.n == 0 || (alpha == 0.0 && beta == 1.0)) return;
  for (int64_t i = 0; i < C.m; ++i)
    for (int64_t j = 0; j < C.n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < A.n; ++p) acc = acc + A.at(i, p) * B.at(p, j);
      C.at(i, j) = beta == 0.0 ? alpha * acc : beta * C.at(i, j) + alpha * acc;
    }
}

int64_t orc_lu_d(const orc_view_d* a, const Level* lv, int nl, int64_t* piv, int nthreads) {
  return lu_run(V(a), lv, nl, 0, piv, 0, nthreads);
}
int64_t orc_lu_s(const orc_view_s* a, const Level* lv, int nl, int64_t* piv, int nthreads) {
  return lu_run(V(a), lv, nl, 0, piv, 0, nthreads);
}
void orc_trsm_llnu_d(double alpha, const orc_view_d* t, const orc_view_d* b, int64_t kc, int nthreads) {
  trsm_left_rec(alpha, V(t), V(b), kc, nthreads);
}
void orc_trsm_llnu_s(double alpha, const orc_view_s* t, const orc_view_s* b, int64_t kc, int nthreads) {
  trsm_left_rec(alpha, V(t), V(b), kc, nthreads);
}

void orc_sandwich_d(const orc_view_d* c, const orc_view_d* a, const double* t, int64_t kc, int nthreads) {
  sandwich(V(c), V(a), t, kc, nthreads);
}
void orc_sandwich_s(const orc_view_s* c, const orc_view_s* a, const float* t, int64_t kc, int nthreads) {
  sandwich(V(c), V(a), t, kc, nthreads);
}
void orc_ltlt_unblocked_d(const orc_view_d* x, int64_t* piv, double* t) { ltlt_unblocked(V(x), piv, t); }
void orc_ltlt_unblocked_s(const orc_view_s* x, int64_t* piv, float* t) { ltlt_unblocked(V(x), piv, t); }

}  // extern "C"
