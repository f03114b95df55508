// ============================================================================
// TEST INFRASTRUCTURE ONLY — CPU oracle for the per-time-step FETI path.
//
// This directory is a CPU restatement of the reference porofeti library
// (/root/reference/proj/include/porofeti/*.hpp) written without Eigen, used
// ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
// the checker.  The shipped product (paper_2509_06673_b200/) never includes,
// links or executes anything under oracle/.
//
// Parity pins: the reference's own known-answer tests (tests/test_elements.cpp,
// tests/test_mesh.cpp) are re-expressed in tests/test_oracle_kat.py; the
// FETI-level behaviour (feti.hpp, assembly.hpp, timeloop.hpp) has no
// reference tests (those files are stubs) and is pinned by the algebraic
// invariants of SPEC.md:358-411 (monolithic equivalence, SPD, linearity).
// ============================================================================
// o_core.hpp — small containers replacing the Eigen aliases of core.hpp:11-16
// and the error hierarchy of core.hpp:32-75.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

struct V2 {
  double x = 0.0, y = 0.0;
  V2() = default;
  V2(double a, double b) : x(a), y(b) {}
  V2 operator+(const V2& o) const { return {x + o.x, y + o.y}; }
  V2 operator-(const V2& o) const { return {x - o.x, y - o.y}; }
  V2 operator*(double s) const { return {x * s, y * s}; }
  double dot(const V2& o) const { return x * o.x + y * o.y; }
  double norm() const { return std::sqrt(x * x + y * y); }
  double linf() const { return std::max(std::abs(x), std::abs(y)); }
};
inline V2 operator*(double s, const V2& v) { return v * s; }

using Vec = std::vector<double>;

/// Row-major dense matrix (local element blocks, coarse problems, tiny oracles).
struct Dense {
  int r = 0, c = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int rows, int cols) : r(rows), c(cols), a(std::size_t(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[std::size_t(i) * c + j]; }
  double operator()(int i, int j) const { return a[std::size_t(i) * c + j]; }
};

struct Trip {
  int r, c;
  double v;
};

/// Compressed sparse row matrix built from triplets (duplicates summed in
/// triplet order, like Eigen's setFromTriplets used throughout assembly.hpp).
struct Csr {
  int nr = 0, nc = 0;
  std::vector<int> ptr{0}, col;
  std::vector<double> val;

  static Csr from_trips(int nr, int nc, const std::vector<Trip>& t) {
    Csr m;
    m.nr = nr;
    m.nc = nc;
    std::vector<int> cnt(nr + 1, 0);
    for (const auto& e : t) cnt[e.r + 1]++;
    for (int i = 0; i < nr; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> order(t.size());
    {
      std::vector<int> pos(cnt.begin(), cnt.end() - 1);
      for (std::size_t k = 0; k < t.size(); ++k) order[pos[t[k].r]++] = static_cast<int>(k);
    }
    m.ptr.assign(nr + 1, 0);
    std::vector<std::pair<int, int>> row;  // (col, triplet index), stable by triplet order
    for (int i = 0; i < nr; ++i) {
      row.clear();
      for (int q = cnt[i]; q < cnt[i + 1]; ++q) row.emplace_back(t[order[q]].c, order[q]);
      std::stable_sort(row.begin(), row.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      for (std::size_t q = 0; q < row.size();) {
        const int c = row[q].first;
        double s = 0.0;
        while (q < row.size() && row[q].first == c) s += t[row[q++].second].v;
        m.col.push_back(c);
        m.val.push_back(s);
      }
      m.ptr[i + 1] = static_cast<int>(m.col.size());
    }
    return m;
  }

  int nnz() const { return static_cast<int>(col.size()); }

  /// y (+)= A x
  void mv(const double* x, double* y, bool acc = false, double scale = 1.0) const {
    for (int i = 0; i < nr; ++i) {
      double s = 0.0;
      for (int q = ptr[i]; q < ptr[i + 1]; ++q) s += val[q] * x[col[q]];
      y[i] = (acc ? y[i] : 0.0) + scale * s;
    }
  }
  /// y (+)= A^T x
  void mtv(const double* x, double* y, bool acc = false, double scale = 1.0) const {
    if (!acc) std::fill(y, y + nc, 0.0);
    for (int i = 0; i < nr; ++i) {
      const double xi = scale * x[i];
      if (xi == 0.0) continue;
      for (int q = ptr[i]; q < ptr[i + 1]; ++q) y[col[q]] += val[q] * xi;
    }
  }
  Vec mul(const Vec& x) const {
    Vec y(nr);
    mv(x.data(), y.data());
    return y;
  }
  Vec tmul(const Vec& x) const {
    Vec y(nc);
    mtv(x.data(), y.data());
    return y;
  }
  double at(int i, int j) const {
    for (int q = ptr[i]; q < ptr[i + 1]; ++q)
      if (col[q] == j) return val[q];
    return 0.0;
  }
  std::vector<Trip> trips() const {
    std::vector<Trip> t;
    t.reserve(col.size());
    for (int i = 0; i < nr; ++i)
      for (int q = ptr[i]; q < ptr[i + 1]; ++q) t.push_back({i, col[q], val[q]});
    return t;
  }
  Csr transpose() const {
    std::vector<Trip> t;
    t.reserve(col.size());
    for (int i = 0; i < nr; ++i)
      for (int q = ptr[i]; q < ptr[i + 1]; ++q) t.push_back({col[q], i, val[q]});
    return from_trips(nc, nr, t);
  }
};

inline double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
inline double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }
inline void axpy(double a, const Vec& x, Vec& y) {
  for (std::size_t i = 0; i < x.size(); ++i) y[i] += a * x[i];
}

// Error hierarchy (reference core.hpp:32-75); the C-ABI maps these to codes.
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
  virtual int code() const { return 99; }
};
struct MeshError : Error {
  using Error::Error;
  int code() const override { return 4; }
};
struct NonConformingInterfaceError : Error {
  using Error::Error;
  int code() const override { return 4; }
};
struct AssemblyError : Error {
  using Error::Error;
  int code() const override { return 4; }
};
struct SingularSubproblemError : Error {
  using Error::Error;
  int code() const override { return 1; }
};
struct PcgBreakdownError : Error {
  using Error::Error;
  int code() const override { return 2; }
};
struct SolverError : Error {
  using Error::Error;
  int code() const override { return 3; }
};
struct ConfigError : Error {
  using Error::Error;
  int code() const override { return 4; }
};

constexpr double kGeomTol = 1e-12;  // core.hpp:77

}  // namespace oracle
