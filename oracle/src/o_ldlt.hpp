// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// o_ldlt.hpp — the subdomain direct solver of the oracle.
//
// The reference factors each constrained saddle K_s with Eigen::SparseLU
// (COLAMD, partial pivoting; feti.hpp:21-45) and verifies the factor on a
// mt19937(20240901) U(-1,1) right-hand side with residual < 1e-8
// (feti.hpp:28-36).  Eigen is absent here, so the oracle restates
// the same contract with a symmetric LDL^T: after symmetric Dirichlet
// elimination K_s is symmetric quasi-definite, so an LDL^T exists for any
// symmetric ordering.  The factorization is the published up-looking
// algorithm (elimination tree + row-subtree traversal, T. Davis, "Algorithm
// 849: a concise sparse Cholesky factorization package", ACM TOMS 2005),
// ordered by geometric nested dissection on the structured-grid node lines.
#pragma once

#include <random>

#include "o_core.hpp"

namespace oracle {

/// Nested dissection on integer grid coordinates (half-cell units): the
/// separator is a full vertex line, which no element crosses.
inline void nd_order_rec(std::vector<int>& ids, const std::vector<std::array<int, 2>>& ic,
                         std::vector<int>& out, const Csr* adj = nullptr, std::vector<int>* side = nullptr) {
  if (ids.size() <= 64) {
    std::sort(ids.begin(), ids.end());
    out.insert(out.end(), ids.begin(), ids.end());
    return;
  }
  int lo[2] = {INT32_MAX, INT32_MAX}, hi[2] = {INT32_MIN, INT32_MIN};
  for (int d : ids)
    for (int a = 0; a < 2; ++a) lo[a] = std::min(lo[a], ic[d][a]), hi[a] = std::max(hi[a], ic[d][a]);
  int axis = (hi[0] - lo[0] >= hi[1] - lo[1]) ? 0 : 1;
  for (int attempt = 0; attempt < 2; ++attempt, axis = 1 - axis) {
    std::vector<int> vals;
    vals.reserve(ids.size());
    for (int d : ids) vals.push_back(ic[d][axis]);
    std::nth_element(vals.begin(), vals.begin() + vals.size() / 2, vals.end());
    int med = vals[vals.size() / 2];
    // nearest even (vertex-line) value strictly inside (lo, hi)
    int best = INT32_MIN;
    for (int c = med - 2; c <= med + 2; ++c)
      if (c % 2 == 0 && c > lo[axis] && c < hi[axis] &&
          (best == INT32_MIN || std::abs(c - med) < std::abs(best - med)))
        best = c;
    if (best == INT32_MIN) continue;
    std::vector<int> L, R, S;
    for (int d : ids) (ic[d][axis] < best ? L : ic[d][axis] > best ? R : S).push_back(d);
    if (adj) {  // graph fix-up: a left vertex adjacent to a right vertex joins the separator
      for (int d : R) (*side)[d] = 2;
      std::vector<int> L2;
      for (int d : L) {
        bool cross = false;
        for (int q = adj->ptr[d]; q < adj->ptr[d + 1] && !cross; ++q) cross = (*side)[adj->col[q]] == 2;
        (cross ? S : L2).push_back(d);
      }
      for (int d : R) (*side)[d] = 0;
      L.swap(L2);
    }
    nd_order_rec(L, ic, out, adj, side);
    nd_order_rec(R, ic, out, adj, side);
    std::sort(S.begin(), S.end());
    out.insert(out.end(), S.begin(), S.end());
    return;
  }
  std::sort(ids.begin(), ids.end());
  out.insert(out.end(), ids.begin(), ids.end());
}

inline std::vector<int> nd_order(const std::vector<std::array<int, 2>>& ic, const Csr* adj = nullptr) {
  std::vector<int> ids(ic.size()), out, side(ic.size(), 0);
  std::iota(ids.begin(), ids.end(), 0);
  out.reserve(ic.size());
  nd_order_rec(ids, ic, out, adj, &side);
  return out;
}

/// Sparse LDL^T of a symmetric matrix given in full CSR storage.
class Ldlt {
 public:
  Ldlt() = default;
  Ldlt(const Csr& A, const std::vector<int>& perm, bool verify = true) { factor(A, perm, verify); }

  void factor(const Csr& A, std::vector<int> perm, bool verify = true) {
    n_ = A.nr;
    if (perm.empty()) {
      perm.resize(n_);
      std::iota(perm.begin(), perm.end(), 0);
    }
    perm_ = perm;
    pinv_.assign(n_, 0);
    for (int k = 0; k < n_; ++k) pinv_[perm_[k]] = k;
    // upper part of C = P A P^T by columns: column k = row perm[k] of A, rows i<=k
    std::vector<int> cp(n_ + 1, 0), ci;
    std::vector<double> cx;
    ci.reserve(A.nnz() / 2 + n_);
    cx.reserve(A.nnz() / 2 + n_);
    for (int k = 0; k < n_; ++k) {
      const int r = perm_[k];
      for (int q = A.ptr[r]; q < A.ptr[r + 1]; ++q) {
        const int i = pinv_[A.col[q]];
        if (i <= k) ci.push_back(i), cx.push_back(A.val[q]);
      }
      cp[k + 1] = (int)ci.size();
    }
    // symbolic: elimination tree and column counts
    parent_.assign(n_, -1);
    std::vector<int> flag(n_), lnz(n_, 0);
    for (int k = 0; k < n_; ++k) {
      flag[k] = k;
      for (int q = cp[k]; q < cp[k + 1]; ++q)
        for (int i = ci[q]; i < k && flag[i] != k; i = parent_[i]) {
          if (parent_[i] == -1) parent_[i] = k;
          lnz[i]++;
          flag[i] = k;
        }
    }
    lp_.assign(n_ + 1, 0);
    for (int k = 0; k < n_; ++k) lp_[k + 1] = lp_[k] + lnz[k];
    li_.assign(lp_[n_], 0);
    lx_.assign(lp_[n_], 0.0);
    d_.assign(n_, 0.0);
    // numeric (up-looking)
    std::vector<double> y(n_, 0.0);
    std::vector<int> pattern(n_);
    std::fill(lnz.begin(), lnz.end(), 0);
    for (int k = 0; k < n_; ++k) {
      int top = n_;
      flag[k] = k;
      for (int q = cp[k]; q < cp[k + 1]; ++q) {
        int i = ci[q];
        y[i] += cx[q];
        int len = 0;
        for (; flag[i] != k; i = parent_[i]) {
          pattern[len++] = i;
          flag[i] = k;
        }
        while (len > 0) pattern[--top] = pattern[--len];
      }
      double dk = y[k];
      y[k] = 0.0;
      for (; top < n_; ++top) {
        const int i = pattern[top];
        const double yi = y[i];
        y[i] = 0.0;
        const int p2 = lp_[i] + lnz[i];
        for (int p = lp_[i]; p < p2; ++p) y[li_[p]] -= lx_[p] * yi;
        const double l = yi / d_[i];
        dk -= l * yi;
        li_[p2] = k;
        lx_[p2] = l;
        lnz[i]++;
      }
      if (dk == 0.0 || !std::isfinite(dk))
        throw SingularSubproblemError("subdomain saddle factorization failed (zero pivot)");
      d_[k] = dk;
    }
    if (verify) check(A);
  }

  /// Seeded residual check of feti.hpp:28-36.
  void check(const Csr& A) const {
    std::mt19937 rng(20240901u);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    Vec b(n_);
    for (int i = 0; i < n_; ++i) b[i] = U(rng);
    const Vec x = solve(b);
    Vec r = A.mul(x);
    for (int i = 0; i < n_; ++i) r[i] -= b[i];
    const double res = norm2(r) / norm2(b);
    if (!(res < 1e-8))
      throw SingularSubproblemError("subdomain factorization residual " + std::to_string(res) +
                                    " (check boundary constraints)");
  }

  void solve_inplace(double* x) const {
    std::vector<double> w(n_);
    for (int k = 0; k < n_; ++k) w[k] = x[perm_[k]];
    for (int j = 0; j < n_; ++j) {
      const double wj = w[j];
      if (wj != 0.0)
        for (int p = lp_[j]; p < lp_[j + 1]; ++p) w[li_[p]] -= lx_[p] * wj;
    }
    for (int j = 0; j < n_; ++j) w[j] /= d_[j];
    for (int j = n_ - 1; j >= 0; --j) {
      double s = w[j];
      for (int p = lp_[j]; p < lp_[j + 1]; ++p) s -= lx_[p] * w[li_[p]];
      w[j] = s;
    }
    for (int k = 0; k < n_; ++k) x[perm_[k]] = w[k];
  }
  Vec solve(const Vec& b) const {
    Vec x = b;
    solve_inplace(x.data());
    return x;
  }

  int dim() const { return n_; }
  long long nnz_L() const { return lp_.empty() ? 0 : lp_[n_]; }
  const std::vector<double>& D() const { return d_; }

 private:
  int n_ = 0;
  std::vector<int> perm_, pinv_, parent_, lp_, li_;
  std::vector<double> lx_, d_;
};

/// Dense LU with partial pivoting (tiny monolithic oracle only).
inline Vec dense_lu_solve(Dense A, Vec b) {
  const int n = A.r;
  std::vector<int> piv(n);
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
    if (A(p, k) == 0.0) throw SingularSubproblemError("monolithic factorization failed");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      std::swap(b[k], b[p]);
    }
    const double inv = 1.0 / A(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double l = A(i, k) * inv;
      if (l == 0.0) continue;
      A(i, k) = l;
      double* ri = &A.a[std::size_t(i) * n];
      const double* rk = &A.a[std::size_t(k) * n];
      for (int j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
      b[i] -= l * b[k];
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < n; ++j) s -= A(k, j) * b[j];
    b[k] = s / A(k, k);
  }
  return b;
}

/// Dense Cholesky (coarse problem G^T G), in place lower factor.
inline void dense_cholesky(Dense& A) {
  const int n = A.r;
  for (int j = 0; j < n; ++j) {
    double s = A(j, j);
    for (int k = 0; k < j; ++k) s -= A(j, k) * A(j, k);
    if (!(s > 0)) throw SolverError("coarse problem G^T G is not positive definite");
    const double d = std::sqrt(s);
    A(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A(i, j);
      for (int k = 0; k < j; ++k) t -= A(i, k) * A(j, k);
      A(i, j) = t / d;
    }
  }
}
inline void dense_cholesky_solve(const Dense& L, double* x) {
  const int n = L.r;
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= L(i, k) * x[k];
    x[i] = s / L(i, i);
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= L(k, i) * x[k];
    x[i] = s / L(i, i);
  }
}

}  // namespace oracle
