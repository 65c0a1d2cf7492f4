// include/d4orm/dense.hpp — Eigen-free dense storage for the drop-in headers.
//
// The reference's public headers are written against Eigen::MatrixXd /
// VectorXd (proj/include/d4orm/types.hpp:7-8).  Eigen is not part of this
// build, so the drop-in headers use this small column-major dense type with
// the API subset the headers and callers touch: storage,
// col/segment/head/middleRows/leftCols views, Zero/Constant, elementwise
// + - scalar*, cwiseMax/Min, norm/squaredNorm, allFinite, comma init.
// The hot path never uses it: the GPU layer sees flat column-major buffers.
#pragma once

#include <cassert>
#include <cmath>
#include <cstddef>
#include <algorithm>
#include <initializer_list>
#include <type_traits>
#include <vector>

namespace d4orm {
namespace dense {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

template <typename Scalar, int R = Dynamic, int C = Dynamic>
class Matrix;
class Block;

// Read-only strided view used by all binary operations.
struct CView {
  const double* data;
  Index rows, cols, stride;  // column-major, stride = distance between columns
  double at(Index i, Index j) const { return data[i + j * stride]; }
  double lin(Index k) const { return at(k % rows, k / rows); }
  Index size() const { return rows * cols; }
};

template <class T>
struct is_dense : std::false_type {};

template <class Derived>
class DenseOps;

// Writable column-major strided block (col, segment, head, middleRows, ...).
class Block {
 public:
  Block(double* d, Index r, Index c, Index s) : d_(d), r_(r), c_(c), s_(s) {}
  Block(const Block&) = default;

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() const { return d_; }
  double& operator()(Index i, Index j) const { return d_[i + j * s_]; }
  double& operator[](Index k) const { return d_[(k % r_) + (k / r_) * s_]; }
  double& coeff(Index k) const { return (*this)[k]; }
  CView view() const { return {d_, r_, c_, s_}; }

  Block col(Index j) const { return Block(d_ + j * s_, r_, 1, s_); }
  Block segment(Index a, Index n) const { return r_ == 1 ? Block(d_ + a * s_, 1, n, s_) : Block(d_ + a, n, 1, s_); }
  Block head(Index n) const { return segment(0, n); }
  Block tail(Index n) const { return segment(size() - n, n); }
  Block middleRows(Index a, Index n) const { return Block(d_ + a, n, c_, s_); }
  Block leftCols(Index n) const { return Block(d_, r_, n, s_); }

  template <class E>
  Block& operator=(const E& e);
  Block& operator=(const Block& o);
  template <class E>
  Block& operator+=(const E& e);
  template <class E>
  Block& operator-=(const E& e);

  double squaredNorm() const {
    double s = 0.0;
    for (Index k = 0; k < size(); ++k) { const double v = (*this)[k]; s += v * v; }
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const {
    for (Index k = 0; k < size(); ++k) if (!std::isfinite((*this)[k])) return false;
    return true;
  }
  void setConstant(double v) const { for (Index k = 0; k < size(); ++k) (*this)[k] = v; }

  struct Comma;
  Comma operator<<(double v) const;

 private:
  double* d_;
  Index r_, c_, s_;
};

struct Block::Comma {
  Block b;
  Index k;
  Comma& operator,(double v) { b[k++] = v; return *this; }
};
inline Block::Comma Block::operator<<(double v) const { Block b(*this); b[0] = v; return Comma{b, 1}; }

template <>
struct is_dense<Block> : std::true_type {};

template <typename Scalar, int R, int C>
class Matrix {
  static_assert(std::is_same<Scalar, double>::value, "shim supports double only");

 public:
  Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : 0), v_(static_cast<std::size_t>(r_ * c_)) {}
  // Vector size constructor (Eigen: Matrix(Index size) for vectors).
  explicit Matrix(Index n) : r_(C == 1 ? n : (R > 0 ? R : 1)), c_(C == 1 ? 1 : n), v_(static_cast<std::size_t>(n)) {
    if (C != 1 && R == Dynamic) { r_ = n; c_ = 1; }
  }
  Matrix(int n) : Matrix(static_cast<Index>(n)) {}
  Matrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c)) {}
  Matrix(int r, int c) : Matrix(static_cast<Index>(r), static_cast<Index>(c)) {}
  Matrix(long r, int c) : Matrix(static_cast<Index>(r), static_cast<Index>(c)) {}
  Matrix(int r, long c) : Matrix(static_cast<Index>(r), static_cast<Index>(c)) {}
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) = default;

  template <int R2, int C2>
  Matrix(const Matrix<double, R2, C2>& o) : r_(o.rows()), c_(o.cols()), v_(o.data(), o.data() + o.size()) {}
  Matrix(const Block& b) { assign(b.view()); }
  Matrix(const CView& v) { assign(v); }

  template <int R2, int C2>
  Matrix& operator=(const Matrix<double, R2, C2>& o) { r_ = o.rows(); c_ = o.cols(); v_.assign(o.data(), o.data() + o.size()); return *this; }
  Matrix& operator=(const Block& b) { assign(b.view()); return *this; }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void resize(Index r, Index c) { r_ = r; c_ = c; v_.assign(static_cast<std::size_t>(r * c), 0.0); }
  void resize(Index n) { if (C == 1 || R == Dynamic) { r_ = n; c_ = 1; } else { r_ = 1; c_ = n; } v_.assign(static_cast<std::size_t>(n), 0.0); }

  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(i + j * r_)]; }
  double& operator[](Index k) { return v_[static_cast<std::size_t>(k)]; }
  double operator[](Index k) const { return v_[static_cast<std::size_t>(k)]; }
  double& operator()(Index k) { return v_[static_cast<std::size_t>(k)]; }
  double operator()(Index k) const { return v_[static_cast<std::size_t>(k)]; }
  CView view() const { return {v_.data(), r_, c_, r_}; }

  Block asBlock() const { return Block(const_cast<double*>(v_.data()), r_, c_, r_); }
  Block col(Index j) const { return asBlock().col(j); }
  Block segment(Index a, Index n) const { return Block(const_cast<double*>(v_.data()) + a, n, 1, n); }
  Block head(Index n) const { return segment(0, n); }
  Block tail(Index n) const { return segment(size() - n, n); }
  Block middleRows(Index a, Index n) const { return asBlock().middleRows(a, n); }
  Block leftCols(Index n) const { return asBlock().leftCols(n); }

  static Matrix Zero(Index r, Index c) { Matrix m(r, c); return m; }
  static Matrix Zero(Index n) { Matrix m(n); return m; }
  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(Index r, Index c, double v) { Matrix m(r, c); m.setConstant(v); return m; }
  static Matrix Constant(Index n, double v) { Matrix m(n); m.setConstant(v); return m; }

  void setConstant(double v) { std::fill(v_.begin(), v_.end(), v); }
  void setZero() { setConstant(0.0); }
  double squaredNorm() const { return asBlock().squaredNorm(); }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const { return asBlock().allFinite(); }

  template <class E>
  Matrix& operator+=(const E& e);
  template <class E>
  Matrix& operator-=(const E& e);
  Matrix& operator*=(double s) { for (auto& x : v_) x = x * s; return *this; }
  Matrix& operator/=(double s) { for (auto& x : v_) x = x / s; return *this; }

  template <class E>
  Matrix cwiseMax(const E& e) const;
  template <class E>
  Matrix cwiseMin(const E& e) const;
  template <class E>
  Matrix cwiseProduct(const E& e) const;
  Matrix cwiseSqrt() const { Matrix m(*this); for (auto& x : m.v_) x = std::sqrt(x); return m; }

  struct Comma {
    Matrix* m;
    Index k;
    Comma& operator,(double v) { (*m)[k++] = v; return *this; }
  };
  Comma operator<<(double v) { (*this)[0] = v; return Comma{this, 1}; }

 private:
  void assign(const CView& v) {
    r_ = v.rows; c_ = v.cols;
    v_.resize(static_cast<std::size_t>(r_ * c_));
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) v_[static_cast<std::size_t>(i + j * r_)] = v.at(i, j);
  }
  Index r_, c_;
  std::vector<double> v_;
};

template <typename S, int R, int C>
struct is_dense<Matrix<S, R, C>> : std::true_type {};

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;

template <class T>
struct Map;
template <>
struct Map<const VectorXd> {
  const double* p;
  Index n;
  Map(const double* d, Index size) : p(d), n(size) {}
  operator VectorXd() const { return VectorXd(CView{p, n, 1, n}); }
};

inline CView view_of(const Block& b) { return b.view(); }
template <typename S, int R, int C>
inline CView view_of(const Matrix<S, R, C>& m) { return m.view(); }

template <class F>
inline MatrixXd zip(const CView& a, const CView& b, F f) {
  assert(a.rows == b.rows && a.cols == b.cols);
  MatrixXd out(a.rows, a.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) out(i, j) = f(a.at(i, j), b.at(i, j));
  return out;
}
template <class F>
inline MatrixXd map1(const CView& a, F f) {
  MatrixXd out(a.rows, a.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) out(i, j) = f(a.at(i, j));
  return out;
}

template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
inline MatrixXd operator+(const A& a, const B& b) { return zip(view_of(a), view_of(b), [](double x, double y) { return x + y; }); }
template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
inline MatrixXd operator-(const A& a, const B& b) { return zip(view_of(a), view_of(b), [](double x, double y) { return x - y; }); }
template <class A, class = std::enable_if_t<is_dense<A>::value>>
inline MatrixXd operator-(const A& a) { return map1(view_of(a), [](double x) { return -x; }); }
template <class A, class = std::enable_if_t<is_dense<A>::value>>
inline MatrixXd operator*(double s, const A& a) { return map1(view_of(a), [s](double x) { return s * x; }); }
template <class A, class = std::enable_if_t<is_dense<A>::value>>
inline MatrixXd operator*(const A& a, double s) { return map1(view_of(a), [s](double x) { return x * s; }); }
template <class A, class = std::enable_if_t<is_dense<A>::value>>
inline MatrixXd operator/(const A& a, double s) { return map1(view_of(a), [s](double x) { return x / s; }); }

template <class E>
inline Block& Block::operator=(const E& e) {
  const CView v = view_of(e);
  MatrixXd tmp(v);  // guard against aliasing
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = tmp(i, j);
  return *this;
}
inline Block& Block::operator=(const Block& o) { return this->operator=<Block>(o); }
template <class E>
inline Block& Block::operator+=(const E& e) {
  MatrixXd tmp(view_of(e));
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = (*this)(i, j) + tmp(i, j);
  return *this;
}
template <class E>
inline Block& Block::operator-=(const E& e) {
  MatrixXd tmp(view_of(e));
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = (*this)(i, j) - tmp(i, j);
  return *this;
}

template <typename S, int R, int C>
template <class E>
inline Matrix<S, R, C>& Matrix<S, R, C>::operator+=(const E& e) {
  MatrixXd tmp(view_of(e));
  for (Index k = 0; k < size(); ++k) v_[static_cast<std::size_t>(k)] = v_[static_cast<std::size_t>(k)] + tmp[k];
  return *this;
}
template <typename S, int R, int C>
template <class E>
inline Matrix<S, R, C>& Matrix<S, R, C>::operator-=(const E& e) {
  MatrixXd tmp(view_of(e));
  for (Index k = 0; k < size(); ++k) v_[static_cast<std::size_t>(k)] = v_[static_cast<std::size_t>(k)] - tmp[k];
  return *this;
}
template <typename S, int R, int C>
template <class E>
inline Matrix<S, R, C> Matrix<S, R, C>::cwiseMax(const E& e) const {
  return Matrix(zip(view(), view_of(e), [](double a, double b) { return std::max(a, b); }));
}
template <typename S, int R, int C>
template <class E>
inline Matrix<S, R, C> Matrix<S, R, C>::cwiseMin(const E& e) const {
  return Matrix(zip(view(), view_of(e), [](double a, double b) { return std::min(a, b); }));
}
template <typename S, int R, int C>
template <class E>
inline Matrix<S, R, C> Matrix<S, R, C>::cwiseProduct(const E& e) const {
  return Matrix(zip(view(), view_of(e), [](double a, double b) { return a * b; }));
}

}  // namespace dense
}  // namespace d4orm
