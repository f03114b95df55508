// eigen_shim.hpp — TEST INFRASTRUCTURE ONLY.
//
// A minimal, eagerly evaluated stand-in for the part of the Eigen 3 API that
// the reference (/root/reference/proj/include/porofeti/*.hpp) uses, so that
// the reference's OWN assembly / FETI / time-loop code can be compiled
// unchanged on this image (Eigen is not installed: SURVEY §8c) and run as the
// pin of the oracle restatement (oracle/ref/ref_driver.cpp, recipe in
// oracle/ref/Makefile, outputs only under oracle/_ref/).
//
// Written from the published Eigen API semantics (column-major dense
// matrices, compressed sparse column matrices, setFromTriplets summing
// duplicates, SparseLU = a direct LU with partial pivoting), not from Eigen's
// sources.  The direct solver is a reverse-Cuthill-McKee ordered banded LU
// with partial pivoting (LAPACK gbtrf-style): exact arithmetic identical to
// any LU, rounding at the 1e-15 level.
//
// Surface covered (everything the reference headers touch):
//   Matrix<double, R, C> (Vector2d, Matrix2d, VectorXd, MatrixXd): Zero,
//     Identity, Unit, coefficient access, segment / col / row blocks,
//     + - * /, dot, norm, squaredNorm, lpNorm<Infinity>, transpose, inverse
//     and determinant (2x2), comma initialiser, eval, resize, min/maxCoeff;
//   SparseMatrix<double> (CSC): setFromTriplets, InnerIterator, transpose,
//     sparse * sparse, sparse * dense vector, conversion to dense;
//   Triplet<double>; SparseLU<SparseMatrix<double>>; SelfAdjointEigenSolver.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <string>
#include <initializer_list>
#include <limits>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int Infinity = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, InvalidInput = 3 };

template <typename S, int R, int C>
class Matrix;
template <typename S>
class SparseMatrix;

namespace detail_shim {
template <int R, int C>
constexpr bool is_fixed = (R > 0 && C > 0);
}

/// Rectangular view into a dense matrix (segment, col, row, block).  Reads
/// and assignments go straight to the parent; arithmetic converts to a Matrix.
template <typename M>
class BlockRef {
 public:
  using Scalar = double;
  BlockRef(M& m, Index r0, Index c0, Index nr, Index nc) : m_(&m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {}
  Index rows() const { return nr_; }
  Index cols() const { return nc_; }
  Index size() const { return nr_ * nc_; }
  double& operator()(Index i, Index j) { return (*m_)(r0_ + i, c0_ + j); }
  double operator()(Index i, Index j) const { return (*m_)(r0_ + i, c0_ + j); }
  double& operator[](Index k) { return nc_ == 1 ? (*this)(k, 0) : (*this)(0, k); }
  double operator[](Index k) const { return nc_ == 1 ? (*this)(k, 0) : (*this)(0, k); }
  double& operator()(Index k) { return (*this)[k]; }
  double operator()(Index k) const { return (*this)[k]; }
  template <typename Src>
  BlockRef& operator=(const Src& src) {
    if (src.rows() * src.cols() != nr_ * nc_) throw std::runtime_error("eigen_shim: block size mismatch");
    if (src.rows() == nr_) {
      for (Index j = 0; j < nc_; ++j)
        for (Index i = 0; i < nr_; ++i) (*this)(i, j) = src(i, j);
    } else {  // vector into a transposed vector block
      for (Index k = 0; k < nr_ * nc_; ++k) (*this)[k] = src[k];
    }
    return *this;
  }
  BlockRef& operator=(const BlockRef& src) { return this->operator=<BlockRef>(src); }
  template <typename Src>
  BlockRef& operator+=(const Src& src) {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) (*this)(i, j) += src(i, j);
    return *this;
  }
  template <typename Src>
  BlockRef& operator-=(const Src& src) {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) (*this)(i, j) -= src(i, j);
    return *this;
  }
  Matrix<double, Dynamic, Dynamic> eval() const;
  double norm() const { return std::sqrt(squaredNorm()); }
  double squaredNorm() const {
    double s = 0.0;
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) s += (*this)(i, j) * (*this)(i, j);
    return s;
  }
  void setZero() {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) (*this)(i, j) = 0.0;
  }

 private:
  M* m_;
  Index r0_, c0_, nr_, nc_;
};

/// Comma initialiser: m << a, b, c, d fills row by row.
template <typename M>
class CommaInit {
 public:
  CommaInit(M& m, double v) : m_(&m) { push(v); }
  CommaInit& operator,(double v) {
    push(v);
    return *this;
  }

 private:
  void push(double v) {
    const Index r = k_ / m_->cols(), c = k_ % m_->cols();
    (*m_)(r, c) = v;
    ++k_;
  }
  M* m_;
  Index k_ = 0;
};

template <typename S, int R, int C>
class Matrix {
  static_assert(std::is_same_v<S, double>, "eigen_shim: double only");
  using Store = std::conditional_t<detail_shim::is_fixed<R, C>, std::array<double, (R > 0 ? R : 1) * (C > 0 ? C : 1)>,
                                   std::vector<double>>;

 public:
  using Scalar = double;
  static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C;

  Matrix() : rows_(R > 0 ? R : 0), cols_(C > 0 ? C : (C == 1 ? 1 : 0)) {
    if constexpr (detail_shim::is_fixed<R, C>) d_.fill(0.0);
    if constexpr (C == 1 && R < 0) cols_ = 1;
  }
  // dynamic vector of size n / dynamic matrix r x c
  template <typename I, typename = std::enable_if_t<std::is_integral_v<I> && (R < 0 || C < 0)>>
  explicit Matrix(I n) : rows_(C == 1 ? Index(n) : Index(1)), cols_(C == 1 ? 1 : Index(n)) {
    d_.assign(static_cast<std::size_t>(n), 0.0);
  }
  template <typename I, typename J,
            typename = std::enable_if_t<std::is_integral_v<I> && std::is_integral_v<J> && (R < 0 || C < 0)>>
  Matrix(I r, J c) : rows_(r), cols_(c) {
    d_.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  // fixed 2-vector from two coordinates
  template <int RR = R, int CC = C, typename = std::enable_if_t<RR == 2 && CC == 1>>
  Matrix(double x, double y) : rows_(2), cols_(1) {
    d_[0] = x, d_[1] = y;
  }
  template <typename M>
  Matrix(const BlockRef<M>& b) : Matrix() {
    resize_like(b.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < b.rows(); ++i) (*this)(i, j) = b(i, j);
  }
  template <int R2, int C2, typename = std::enable_if_t<!(R2 == R && C2 == C)>>
  Matrix(const Matrix<double, R2, C2>& o) : Matrix() {
    resize_like(o.rows(), o.cols());
    for (Index k = 0; k < o.rows() * o.cols(); ++k) data()[k] = o.data()[k];
  }
  explicit Matrix(const SparseMatrix<double>& sp);

  // --- shape ---
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  void resize(Index n) {
    static_assert(!detail_shim::is_fixed<R, C>, "resize of a fixed matrix");
    if (C == 1) rows_ = n, cols_ = 1;
    else rows_ = 1, cols_ = n;
    d_.assign(static_cast<std::size_t>(n), 0.0);
  }
  void resize(Index r, Index c) {
    if constexpr (detail_shim::is_fixed<R, C>) {
      if (r != R || c != C) throw std::runtime_error("eigen_shim: resize of a fixed matrix");
    } else {
      rows_ = r, cols_ = c;
      d_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
  }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }

  // --- access (column-major) ---
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * rows_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(i + j * rows_)]; }
  double& operator()(Index k) { return d_[static_cast<std::size_t>(k)]; }
  double operator()(Index k) const { return d_[static_cast<std::size_t>(k)]; }
  double& operator[](Index k) { return d_[static_cast<std::size_t>(k)]; }
  double operator[](Index k) const { return d_[static_cast<std::size_t>(k)]; }
  double x() const { return d_[0]; }
  double y() const { return d_[1]; }
  double& x() { return d_[0]; }
  double& y() { return d_[1]; }

  BlockRef<Matrix> segment(Index start, Index n) {
    return cols_ == 1 ? BlockRef<Matrix>(*this, start, 0, n, 1) : BlockRef<Matrix>(*this, 0, start, 1, n);
  }
  Matrix<double, Dynamic, 1> segment(Index start, Index n) const {
    Matrix<double, Dynamic, 1> v(n);
    for (Index k = 0; k < n; ++k) v[k] = d_[static_cast<std::size_t>(start + k)];
    return v;
  }
  BlockRef<Matrix> head(Index n) { return segment(0, n); }
  BlockRef<Matrix> tail(Index n) { return segment(size() - n, n); }
  BlockRef<Matrix> col(Index j) { return BlockRef<Matrix>(*this, 0, j, rows_, 1); }
  Matrix<double, R, 1> col(Index j) const {
    Matrix<double, R, 1> v;
    v.resize_like(rows_, 1);
    for (Index i = 0; i < rows_; ++i) v[i] = (*this)(i, j);
    return v;
  }
  BlockRef<Matrix> row(Index i) { return BlockRef<Matrix>(*this, i, 0, 1, cols_); }
  Matrix<double, Dynamic, Dynamic> row(Index i) const {
    Matrix<double, Dynamic, Dynamic> v(Index(1), cols_);
    for (Index j = 0; j < cols_; ++j) v(0, j) = (*this)(i, j);
    return v;
  }
  BlockRef<Matrix> block(Index r0, Index c0, Index nr, Index nc) { return BlockRef<Matrix>(*this, r0, c0, nr, nc); }

  CommaInit<Matrix> operator<<(double v) { return CommaInit<Matrix>(*this, v); }

  // --- factories ---
  static Matrix Zero() { return Matrix(); }
  template <typename I, typename = std::enable_if_t<std::is_integral_v<I>>>
  static Matrix Zero(I n) {
    return Matrix(n);
  }
  template <typename I, typename J>
  static Matrix Zero(I r, J c) {
    return Matrix(r, c);
  }
  static Matrix Identity() {
    Matrix m;
    for (Index i = 0; i < std::min<Index>(R, C); ++i) m(i, i) = 1.0;
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  static Matrix Unit(Index n, Index k) {
    Matrix m(n);
    m[k] = 1.0;
    return m;
  }
  static Matrix Constant(Index n, double v) {
    Matrix m(n);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }

  // --- reductions ---
  template <typename O>
  double dot(const O& o) const {
    double s = 0.0;
    for (Index k = 0; k < size(); ++k) s += d_[static_cast<std::size_t>(k)] * o[k];
    return s;
  }
  double squaredNorm() const {
    double s = 0.0;
    for (double v : d_) s += v * v;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  template <int P>
  double lpNorm() const {
    static_assert(P == Infinity, "eigen_shim: lpNorm<Infinity> only");
    double m = 0.0;
    for (double v : d_) m = std::max(m, std::abs(v));
    return m;
  }
  double sum() const { return std::accumulate(d_.begin(), d_.end(), 0.0); }
  double minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  double maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }
  Matrix eval() const { return *this; }

  // --- algebra ---
  Matrix<double, C, R> transpose() const {
    Matrix<double, C, R> t;
    t.resize_like(cols_, rows_);
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  double determinant() const {
    if (rows_ != 2 || cols_ != 2) throw std::runtime_error("eigen_shim: determinant of 2x2 only");
    return (*this)(0, 0) * (*this)(1, 1) - (*this)(1, 0) * (*this)(0, 1);
  }
  Matrix inverse() const {
    if (rows_ != 2 || cols_ != 2) throw std::runtime_error("eigen_shim: inverse of 2x2 only");
    const double det = determinant();
    Matrix m = *this;
    m(0, 0) = (*this)(1, 1) / det, m(1, 1) = (*this)(0, 0) / det;
    m(0, 1) = -(*this)(0, 1) / det, m(1, 0) = -(*this)(1, 0) / det;
    return m;
  }
  Matrix operator-() const {
    Matrix m = *this;
    for (double& v : m.d_) v = -v;
    return m;
  }
  template <typename O>
  Matrix& operator+=(const O& o) {
    check_same(o);
    for (Index k = 0; k < size(); ++k) d_[static_cast<std::size_t>(k)] += elem(o, k);
    return *this;
  }
  template <typename O>
  Matrix& operator-=(const O& o) {
    check_same(o);
    for (Index k = 0; k < size(); ++k) d_[static_cast<std::size_t>(k)] -= elem(o, k);
    return *this;
  }
  Matrix& operator*=(double s) {
    for (double& v : d_) v *= s;
    return *this;
  }
  Matrix& operator/=(double s) {
    for (double& v : d_) v /= s;
    return *this;
  }

  void resize_like(Index r, Index c) {
    if constexpr (detail_shim::is_fixed<R, C>) {
      if (r != R || c != C) throw std::runtime_error("eigen_shim: fixed-size mismatch");
    } else {
      rows_ = r, cols_ = c;
      d_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
  }

 private:
  template <typename O>
  void check_same(const O& o) const {
    if (o.rows() * o.cols() != size()) throw std::runtime_error("eigen_shim: size mismatch in +=/-=");
  }
  template <typename O>
  static double elem(const O& o, Index k) {
    if constexpr (std::is_same_v<O, Matrix>) return o.d_[static_cast<std::size_t>(k)];
    else return o(k % o.rows(), k / o.rows());
  }

  Index rows_ = 0, cols_ = 0;
  Store d_{};
  template <typename, int, int>
  friend class Matrix;
};

template <typename M>
Matrix<double, Dynamic, Dynamic> BlockRef<M>::eval() const {
  return Matrix<double, Dynamic, Dynamic>(*this);
}

using Vector2d = Matrix<double, 2, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
template <typename S, int N>
using Vector = Matrix<S, N, 1>;

// ---- dense arithmetic (eager) ----
namespace detail_shim {
template <typename T>
struct is_dense : std::false_type {};
template <int R, int C>
struct is_dense<Matrix<double, R, C>> : std::true_type {};
template <typename M>
struct is_dense<BlockRef<M>> : std::true_type {};
template <typename T>
inline constexpr bool is_dense_v = is_dense<std::decay_t<T>>::value;

template <typename T>
struct as_matrix {
  using type = MatrixXd;
};
template <int R, int C>
struct as_matrix<Matrix<double, R, C>> {
  using type = Matrix<double, R, C>;
};
template <typename A, typename B>
using sum_t = std::conditional_t<std::is_same_v<typename as_matrix<A>::type, typename as_matrix<B>::type>,
                                 typename as_matrix<A>::type,
                                 std::conditional_t<(as_matrix<A>::type::ColsAtCompileTime == 1 ||
                                                     as_matrix<B>::type::ColsAtCompileTime == 1),
                                                    VectorXd, MatrixXd>>;
template <typename A>
typename as_matrix<A>::type to_matrix(const A& a) {
  return typename as_matrix<A>::type(a);
}
}  // namespace detail_shim

template <typename A, typename B,
          typename = std::enable_if_t<detail_shim::is_dense_v<A> && detail_shim::is_dense_v<B>>>
auto operator+(const A& a, const B& b) {
  detail_shim::sum_t<std::decay_t<A>, std::decay_t<B>> r(detail_shim::to_matrix(a));
  r += b;
  return r;
}
template <typename A, typename B,
          typename = std::enable_if_t<detail_shim::is_dense_v<A> && detail_shim::is_dense_v<B>>>
auto operator-(const A& a, const B& b) {
  detail_shim::sum_t<std::decay_t<A>, std::decay_t<B>> r(detail_shim::to_matrix(a));
  r -= b;
  return r;
}
template <typename A, typename = std::enable_if_t<detail_shim::is_dense_v<A>>>
auto operator*(double s, const A& a) {
  auto r = detail_shim::to_matrix(a);
  r *= s;
  return r;
}
template <typename A, typename = std::enable_if_t<detail_shim::is_dense_v<A>>>
auto operator*(const A& a, double s) {
  auto r = detail_shim::to_matrix(a);
  r *= s;
  return r;
}
template <typename A, typename = std::enable_if_t<detail_shim::is_dense_v<A>>>
auto operator/(const A& a, double s) {
  auto r = detail_shim::to_matrix(a);
  r /= s;
  return r;
}
template <typename A, typename = std::enable_if_t<detail_shim::is_dense_v<A>>>
auto operator-(const BlockRef<A>& a) {
  return -detail_shim::to_matrix(a);
}
/// dense product; result keeps fixed sizes when both operands are fixed
template <int R1, int C1, int R2, int C2>
auto operator*(const Matrix<double, R1, C1>& a, const Matrix<double, R2, C2>& b) {
  if (a.cols() != b.rows()) throw std::runtime_error("eigen_shim: product size mismatch");
  using Res = std::conditional_t<(R1 > 0 && C2 > 0), Matrix<double, R1, C2>,
                                 std::conditional_t<C2 == 1, VectorXd, MatrixXd>>;
  Res r;
  r.resize_like(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const double bkj = b(k, j);
      for (Index i = 0; i < a.rows(); ++i) r(i, j) += a(i, k) * bkj;
    }
  return r;
}

// ---- sparse ----
template <typename S>
class Triplet {
 public:
  Triplet(Index r = 0, Index c = 0, S v = S(0)) : r_(r), c_(c), v_(v) {}
  Index row() const { return r_; }
  Index col() const { return c_; }
  S value() const { return v_; }

 private:
  Index r_, c_;
  S v_;
};

/// Compressed sparse column matrix (Eigen's default storage order).
template <typename S>
class SparseMatrix {
 public:
  using Scalar = S;
  SparseMatrix() : ptr_(1, 0) {}
  SparseMatrix(Index r, Index c) : rows_(r), cols_(c), ptr_(static_cast<std::size_t>(c) + 1, 0) {}
  void resize(Index r, Index c) {
    rows_ = r, cols_ = c;
    ptr_.assign(static_cast<std::size_t>(c) + 1, 0);
    idx_.clear(), val_.clear();
  }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index outerSize() const { return cols_; }
  Index nonZeros() const { return static_cast<Index>(val_.size()); }
  void makeCompressed() {}
  void reserve(Index) {}

  /// duplicates summed, rows sorted within each column
  template <typename It>
  void setFromTriplets(It first, It last) {
    std::vector<Index> cnt(static_cast<std::size_t>(cols_) + 1, 0);
    for (It it = first; it != last; ++it) {
      if (it->row() < 0 || it->row() >= rows_ || it->col() < 0 || it->col() >= cols_)
        throw std::runtime_error("eigen_shim: triplet out of range");
      ++cnt[static_cast<std::size_t>(it->col()) + 1];
    }
    for (Index c = 0; c < cols_; ++c) cnt[c + 1] += cnt[c];
    std::vector<std::pair<Index, S>> ent(static_cast<std::size_t>(cnt[cols_]));
    std::vector<Index> fill(cnt.begin(), cnt.end() - 1);
    for (It it = first; it != last; ++it) ent[fill[it->col()]++] = {it->row(), it->value()};
    ptr_.assign(static_cast<std::size_t>(cols_) + 1, 0);
    idx_.clear(), val_.clear();
    for (Index c = 0; c < cols_; ++c) {
      auto b = ent.begin() + cnt[c], e = ent.begin() + cnt[c + 1];
      std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto p = b; p != e; ++p) {
        if (!idx_.empty() && static_cast<Index>(idx_.size()) > ptr_[c] && idx_.back() == p->first)
          val_.back() += p->second;
        else
          idx_.push_back(p->first), val_.push_back(p->second);
      }
      ptr_[c + 1] = static_cast<Index>(idx_.size());
    }
  }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer) : m_(&m), k_(m.ptr_[outer]), end_(m.ptr_[outer + 1]), c_(outer) {}
    explicit operator bool() const { return k_ < end_; }
    InnerIterator& operator++() {
      ++k_;
      return *this;
    }
    Index row() const { return m_->idx_[k_]; }
    Index index() const { return m_->idx_[k_]; }
    Index col() const { return c_; }
    S value() const { return m_->val_[k_]; }

   private:
    const SparseMatrix* m_;
    Index k_, end_, c_;
  };

  SparseMatrix transpose() const {
    std::vector<Triplet<S>> t;
    t.reserve(val_.size());
    for (Index c = 0; c < cols_; ++c)
      for (Index k = ptr_[c]; k < ptr_[c + 1]; ++k) t.emplace_back(c, idx_[k], val_[k]);
    SparseMatrix r(cols_, rows_);
    r.setFromTriplets(t.begin(), t.end());
    return r;
  }
  SparseMatrix eval() const { return *this; }

  /// y = A x
  VectorXd operator*(const VectorXd& x) const {
    if (x.size() != cols_) throw std::runtime_error("eigen_shim: sparse * vector size mismatch");
    VectorXd y(rows_);
    for (Index c = 0; c < cols_; ++c) {
      const double xc = x[c];
      if (xc == 0.0) continue;
      for (Index k = ptr_[c]; k < ptr_[c + 1]; ++k) y[idx_[k]] += val_[k] * xc;
    }
    return y;
  }
  template <typename M>
  VectorXd operator*(const BlockRef<M>& x) const {
    return (*this) * VectorXd(x);
  }
  /// C = A B (Gustavson, column by column)
  SparseMatrix operator*(const SparseMatrix& B) const {
    if (cols_ != B.rows_) throw std::runtime_error("eigen_shim: sparse product size mismatch");
    SparseMatrix C(rows_, B.cols_);
    std::vector<S> acc(static_cast<std::size_t>(rows_), S(0));
    std::vector<Index> mark(static_cast<std::size_t>(rows_), -1), rows;
    for (Index j = 0; j < B.cols_; ++j) {
      rows.clear();
      for (Index kb = B.ptr_[j]; kb < B.ptr_[j + 1]; ++kb) {
        const Index k = B.idx_[kb];
        const S bkj = B.val_[kb];
        for (Index ka = ptr_[k]; ka < ptr_[k + 1]; ++ka) {
          const Index i = idx_[ka];
          if (mark[i] != j) mark[i] = j, acc[i] = S(0), rows.push_back(i);
          acc[i] += val_[ka] * bkj;
        }
      }
      std::sort(rows.begin(), rows.end());
      for (Index i : rows) C.idx_.push_back(i), C.val_.push_back(acc[i]);
      C.ptr_[j + 1] = static_cast<Index>(C.idx_.size());
    }
    return C;
  }
  SparseMatrix operator+(const SparseMatrix& B) const { return combine(B, 1.0); }
  SparseMatrix operator-(const SparseMatrix& B) const { return combine(B, -1.0); }

  const std::vector<Index>& outer_ptr() const { return ptr_; }
  const std::vector<Index>& inner_idx() const { return idx_; }
  const std::vector<S>& values() const { return val_; }

 private:
  SparseMatrix combine(const SparseMatrix& B, double sb) const {
    std::vector<Triplet<S>> t;
    for (Index c = 0; c < cols_; ++c)
      for (Index k = ptr_[c]; k < ptr_[c + 1]; ++k) t.emplace_back(idx_[k], c, val_[k]);
    for (Index c = 0; c < B.cols_; ++c)
      for (Index k = B.ptr_[c]; k < B.ptr_[c + 1]; ++k) t.emplace_back(B.idx_[k], c, sb * B.val_[k]);
    SparseMatrix r(rows_, cols_);
    r.setFromTriplets(t.begin(), t.end());
    return r;
  }
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> ptr_, idx_;
  std::vector<S> val_;
};

template <typename S, int R, int C>
Matrix<S, R, C>::Matrix(const SparseMatrix<double>& sp) : Matrix() {
  resize_like(sp.rows(), sp.cols());
  for (Index c = 0; c < sp.cols(); ++c)
    for (typename SparseMatrix<double>::InnerIterator it(sp, c); it; ++it) (*this)(it.row(), c) += it.value();
}

inline SparseMatrix<double> operator*(double s, const SparseMatrix<double>& A) {
  std::vector<Triplet<double>> t;
  for (Index c = 0; c < A.cols(); ++c)
    for (SparseMatrix<double>::InnerIterator it(A, c); it; ++it) t.emplace_back(it.row(), c, s * it.value());
  SparseMatrix<double> r(A.rows(), A.cols());
  r.setFromTriplets(t.begin(), t.end());
  return r;
}

/// Direct solver with Eigen::SparseLU's interface: reverse Cuthill-McKee
/// ordering of the symmetrised pattern, then a banded LU with partial
/// pivoting (rows swapped within the band, as LAPACK gbtrf).
template <typename M>
class SparseLU {
 public:
  SparseLU() = default;
  explicit SparseLU(const M& A) { compute(A); }

  void compute(const M& A) {
    info_ = Success;
    n_ = A.rows();
    if (A.cols() != n_) {
      info_ = InvalidInput;
      return;
    }
    order(A);
    // bandwidths of the permuted matrix
    kl_ = ku_ = 0;
    for (Index c = 0; c < n_; ++c)
      for (typename M::InnerIterator it(A, c); it; ++it) {
        const Index i = inv_[it.row()], j = inv_[c];
        kl_ = std::max(kl_, i - j), ku_ = std::max(ku_, j - i);
      }
    ld_ = 2 * kl_ + ku_ + 1;  // kl extra rows hold the fill from row interchanges
    ab_.assign(static_cast<std::size_t>(ld_ * n_), 0.0);
    for (Index c = 0; c < n_; ++c)
      for (typename M::InnerIterator it(A, c); it; ++it) at(inv_[it.row()], inv_[c]) += it.value();
    piv_.assign(static_cast<std::size_t>(n_), 0);
    const Index kv = ku_ + kl_;
    for (Index j = 0; j < n_; ++j) {
      const Index km = std::min(kl_, n_ - 1 - j);
      Index p = j;
      double best = std::abs(at(j, j));
      for (Index i = j + 1; i <= j + km; ++i)
        if (std::abs(at(i, j)) > best) best = std::abs(at(i, j)), p = i;
      piv_[j] = p;
      if (best == 0.0) {
        info_ = NumericalIssue;
        return;
      }
      const Index ju = std::min(j + kv, n_ - 1);
      if (p != j)
        for (Index c = j; c <= ju; ++c) std::swap(at(p, c), at(j, c));
      const double inv = 1.0 / at(j, j);
      for (Index i = j + 1; i <= j + km; ++i) at(i, j) *= inv;
      for (Index c = j + 1; c <= ju; ++c) {
        const double u = at(j, c);
        if (u == 0.0) continue;
        for (Index i = j + 1; i <= j + km; ++i) at(i, c) -= at(i, j) * u;
      }
    }
  }
  ComputationInfo info() const { return info_; }

  VectorXd solve(const VectorXd& b) const {
    if (b.size() != n_) throw std::runtime_error("eigen_shim: SparseLU::solve size mismatch");
    std::vector<double> x(static_cast<std::size_t>(n_));
    for (Index i = 0; i < n_; ++i) x[inv_[i]] = b[i];
    const Index kv = ku_ + kl_;
    for (Index j = 0; j < n_; ++j) {  // L y = P b
      const Index p = piv_[j];
      if (p != j) std::swap(x[p], x[j]);
      const Index km = std::min(kl_, n_ - 1 - j);
      const double xj = x[j];
      for (Index i = j + 1; i <= j + km; ++i) x[i] -= at(i, j) * xj;
    }
    for (Index j = n_ - 1; j >= 0; --j) {  // U x = y
      x[j] /= at(j, j);
      const double xj = x[j];
      for (Index i = std::max<Index>(0, j - kv); i < j; ++i) x[i] -= at(i, j) * xj;
    }
    VectorXd out(n_);
    for (Index i = 0; i < n_; ++i) out[i] = x[inv_[i]];
    return out;
  }
  template <typename Mx>
  VectorXd solve(const BlockRef<Mx>& b) const {
    return solve(VectorXd(b));
  }

 private:
  // band storage: entry (i, j) of the permuted matrix at row kl + ku + i - j of column j
  double& at(Index i, Index j) { return ab_[static_cast<std::size_t>(kl_ + ku_ + i - j + j * ld_)]; }
  double at(Index i, Index j) const { return ab_[static_cast<std::size_t>(kl_ + ku_ + i - j + j * ld_)]; }

  /// reverse Cuthill-McKee on the pattern of A + A^T (per connected component,
  /// started from a minimum-degree node); inv_[old] = new
  void order(const M& A) {
    std::vector<std::vector<Index>> adj(static_cast<std::size_t>(n_));
    for (Index c = 0; c < n_; ++c)
      for (typename M::InnerIterator it(A, c); it; ++it)
        if (it.row() != c) adj[it.row()].push_back(c), adj[c].push_back(it.row());
    for (auto& a : adj) {
      std::sort(a.begin(), a.end());
      a.erase(std::unique(a.begin(), a.end()), a.end());
    }
    std::vector<Index> perm;
    perm.reserve(static_cast<std::size_t>(n_));
    std::vector<char> seen(static_cast<std::size_t>(n_), 0);
    std::vector<Index> nodes(static_cast<std::size_t>(n_));
    std::iota(nodes.begin(), nodes.end(), Index(0));
    std::stable_sort(nodes.begin(), nodes.end(), [&](Index a, Index b) { return adj[a].size() < adj[b].size(); });
    for (Index s : nodes) {
      if (seen[s]) continue;
      std::queue<Index> q;
      q.push(s), seen[s] = 1;
      while (!q.empty()) {
        const Index v = q.front();
        q.pop();
        perm.push_back(v);
        std::vector<Index> nb;
        for (Index w : adj[v])
          if (!seen[w]) nb.push_back(w), seen[w] = 1;
        std::stable_sort(nb.begin(), nb.end(), [&](Index a, Index b) { return adj[a].size() < adj[b].size(); });
        for (Index w : nb) q.push(w);
      }
    }
    // EIGEN_SHIM_ORDER=cm keeps the Cuthill-McKee order unreversed: the same
    // bandwidth, a different (equally valid) elimination order -- used to
    // measure how much the reference's outputs move with the LU's rounding
    static const bool cm = [] {
      const char* e = std::getenv("EIGEN_SHIM_ORDER");
      return e && std::string(e) == "cm";
    }();
    if (!cm) std::reverse(perm.begin(), perm.end());
    inv_.assign(static_cast<std::size_t>(n_), 0);
    for (Index k = 0; k < n_; ++k) inv_[perm[k]] = k;
  }

  ComputationInfo info_ = Success;
  Index n_ = 0, kl_ = 0, ku_ = 0, ld_ = 1;
  std::vector<double> ab_;
  std::vector<Index> piv_, inv_;
};

/// Eigenvalues of a symmetric matrix (cyclic Jacobi), ascending.
template <typename M>
class SelfAdjointEigenSolver {
 public:
  explicit SelfAdjointEigenSolver(const M& A) {
    const Index n = A.rows();
    MatrixXd a(n, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) a(i, j) = A(i, j);
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0;
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i)
          if (i != j) off += a(i, j) * a(i, j);
      if (off < 1e-300) break;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          if (a(p, q) == 0.0) continue;
          const double th = 0.5 * (a(q, q) - a(p, p)) / a(p, q);
          const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (Index k = 0; k < n; ++k) {
            const double akp = a(k, p), akq = a(k, q);
            a(k, p) = c * akp - s * akq, a(k, q) = s * akp + c * akq;
          }
          for (Index k = 0; k < n; ++k) {
            const double apk = a(p, k), aqk = a(q, k);
            a(p, k) = c * apk - s * aqk, a(q, k) = s * apk + c * aqk;
          }
        }
    }
    ev_.resize_like(n, 1);
    std::vector<double> e(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) e[i] = a(i, i);
    std::sort(e.begin(), e.end());
    for (Index i = 0; i < n; ++i) ev_[i] = e[i];
  }
  const Matrix<double, M::RowsAtCompileTime, 1>& eigenvalues() const { return ev_; }

 private:
  Matrix<double, M::RowsAtCompileTime, 1> ev_;
};

}  // namespace Eigen
