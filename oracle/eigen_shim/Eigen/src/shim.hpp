// Minimal functional stand-in for the subset of Eigen3's dense API that the
// reference's hot-path sources use. TEST INFRASTRUCTURE ONLY: it exists so
// oracle/Makefile can compile the reference's own src/linsolve.cpp,
// src/toeplitz.cpp, src/mesh.cpp, src/array_model.cpp and src/fft.cpp
// unchanged into oracle/_ref/libref_linsolve.so, which pins the CPU oracle
// (oracle/oracle.cpp) to reference outputs. Eigen3 itself is absent from
// this image and there is no network.
//
// Written from the documented Eigen semantics, not from Eigen's sources:
//  * storage is column-major (Eigen's default), so MatrixXcd::data() is the
//    ZTOE1 payload order of toeplitz.cpp:676;
//  * a.dot(b) = sum_i conj(a_i) * b_i (conjugate-linear in the first
//    argument, the reference relies on it at linsolve.cpp:466);
//  * norm() = sqrt(sum |a_i|^2); cwiseProduct / cwiseAbs / cwiseMin / cwiseMax
//    are element-wise; assignment to a Matrix resizes it;
//  * PartialPivLU is LU with row partial pivoting on the largest |a_ij|
//    (first index on ties), matrixLU() the packed unit-lower / upper factors.
// Every expression is evaluated eagerly (no expression templates) and every
// reduction is sequential in index order. Eigen vectorises reductions and
// blocks its products and LU, so results can differ from an Eigen build in
// the last bits (reduction order only, ~1e-16 relative); no bound in
// tests/ is tighter than 1e-13 for a comparison that crosses such a sum.
#pragma once

// Like Eigen/Core, this pulls in <cstdint>, <cstring>, <limits>, <functional>
// and <string>; the reference relies on that transitively (toeplitz.cpp uses
// uint8_t / std::memcpy without including their headers).

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iosfwd>
#include <limits>
#include <string>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;

template <typename T> struct RealOf { using type = T; };
template <typename T> struct RealOf<std::complex<T>> { using type = T; };

template <typename T> inline T conjOf(const T& v) { return v; }
template <typename T> inline std::complex<T> conjOf(const std::complex<T>& v) { return std::conj(v); }
template <typename T> inline T abs2Of(const T& v) { return v * v; }
template <typename T> inline T abs2Of(const std::complex<T>& v) { return std::norm(v); }

template <typename S, int R = Dynamic, int C = Dynamic> class Matrix;
template <typename S> class BlockView;

template <typename T> struct IsDense : std::false_type {};
template <typename S, int R, int C> struct IsDense<Matrix<S, R, C>> : std::true_type {};
template <typename S> struct IsDense<BlockView<S>> : std::true_type {};

template <typename T> struct IsScalar : std::is_arithmetic<T> {};
template <typename T> struct IsScalar<std::complex<T>> : std::true_type {};

// Shared read/write interface over (pointer, rows, cols, leading dimension).
template <typename D, typename S>
class DenseBase {
 public:
  using Scalar = std::remove_const_t<S>;
  using Real = typename RealOf<Scalar>::type;
  using Plain = Matrix<Scalar, Dynamic, Dynamic>;

  D& self() { return static_cast<D&>(*this); }
  const D& self() const { return static_cast<const D&>(*this); }
  Index size() const { return self().rows() * self().cols(); }

  S& operator()(Index i, Index j) { return self().ptr()[i + j * self().ld()]; }
  const Scalar& operator()(Index i, Index j) const { return self().ptr()[i + j * self().ld()]; }
  // Linear index: the vector case (one of the two dimensions is 1).
  S& operator()(Index i) { return self().cols() == 1 ? (*this)(i, 0) : (*this)(0, i); }
  const Scalar& operator()(Index i) const { return self().cols() == 1 ? (*this)(i, 0) : (*this)(0, i); }
  S& operator[](Index i) { return (*this)(i); }
  const Scalar& operator[](Index i) const { return (*this)(i); }

  // ---- sub-blocks (views into this storage)
  BlockView<S> block(Index i, Index j, Index r, Index c) {
    return BlockView<S>(self().ptr() + i + j * self().ld(), r, c, self().ld());
  }
  BlockView<const Scalar> block(Index i, Index j, Index r, Index c) const {
    return BlockView<const Scalar>(self().ptr() + i + j * self().ld(), r, c, self().ld());
  }
#define SHIM_BLOCK_PAIR(name, args, call)                                  \
  BlockView<S> name args { return block call; }                            \
  BlockView<const Scalar> name args const { return block call; }
  SHIM_BLOCK_PAIR(col, (Index j), (0, j, self().rows(), 1))
  SHIM_BLOCK_PAIR(row, (Index i), (i, 0, 1, self().cols()))
  SHIM_BLOCK_PAIR(leftCols, (Index n), (0, 0, self().rows(), n))
  SHIM_BLOCK_PAIR(rightCols, (Index n), (0, self().cols() - n, self().rows(), n))
  SHIM_BLOCK_PAIR(middleCols, (Index j, Index n), (0, j, self().rows(), n))
  SHIM_BLOCK_PAIR(topRows, (Index n), (0, 0, n, self().cols()))
  SHIM_BLOCK_PAIR(bottomRows, (Index n), (self().rows() - n, 0, n, self().cols()))
  SHIM_BLOCK_PAIR(middleRows, (Index i, Index n), (i, 0, n, self().cols()))
  SHIM_BLOCK_PAIR(topLeftCorner, (Index r, Index c), (0, 0, r, c))
  SHIM_BLOCK_PAIR(topRightCorner, (Index r, Index c), (0, self().cols() - c, r, c))
  SHIM_BLOCK_PAIR(bottomLeftCorner, (Index r, Index c), (self().rows() - r, 0, r, c))
  SHIM_BLOCK_PAIR(bottomRightCorner, (Index r, Index c), (self().rows() - r, self().cols() - c, r, c))
#undef SHIM_BLOCK_PAIR
  BlockView<S> segment(Index a, Index n) { return self().cols() == 1 ? block(a, 0, n, 1) : block(0, a, 1, n); }
  BlockView<const Scalar> segment(Index a, Index n) const {
    return self().cols() == 1 ? block(a, 0, n, 1) : block(0, a, 1, n);
  }
  BlockView<S> head(Index n) { return segment(0, n); }
  BlockView<const Scalar> head(Index n) const { return segment(0, n); }
  BlockView<S> tail(Index n) { return segment(size() - n, n); }
  BlockView<const Scalar> tail(Index n) const { return segment(size() - n, n); }

  // ---- coordinates of 3-vectors
  S& x() { return (*this)(0); }
  S& y() { return (*this)(1); }
  S& z() { return (*this)(2); }
  const Scalar& x() const { return (*this)(0); }
  const Scalar& y() const { return (*this)(1); }
  const Scalar& z() const { return (*this)(2); }

  // ---- evaluated results
  Plain eval() const;
  Plain transpose() const;
  Matrix<Scalar, Dynamic, 1> diagonal() const;
  template <typename O> Plain cwiseProduct(const O& o) const;
  Matrix<Real, Dynamic, Dynamic> cwiseAbs() const;
  template <typename O> Plain cwiseMin(const O& o) const;
  template <typename O> Plain cwiseMax(const O& o) const;
  template <typename O> Plain cross(const O& o) const;

  Scalar sum() const {
    Scalar s{};
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) s += (*this)(i, j);
    return s;
  }
  Scalar maxCoeff() const {
    Scalar m = (*this)(0, 0);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) m = std::max(m, (*this)(i, j));
    return m;
  }
  Real squaredNorm() const {
    Real s{};
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) s += abs2Of((*this)(i, j));
    return s;
  }
  Real norm() const { return std::sqrt(squaredNorm()); }
  template <typename O>
  Scalar dot(const O& o) const {
    Scalar s{};
    for (Index k = 0; k < size(); ++k) s += conjOf((*this)(k)) * o(k);
    return s;
  }

  void setZero() {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) = Scalar{};
  }

  // ---- in-place arithmetic (sizes must agree)
  template <typename O, std::enable_if_t<IsDense<O>::value, int> = 0>
  D& operator+=(const O& o) {
    check(o);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) += o(i, j);
    return self();
  }
  template <typename O, std::enable_if_t<IsDense<O>::value, int> = 0>
  D& operator-=(const O& o) {
    check(o);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) -= o(i, j);
    return self();
  }
  template <typename T, std::enable_if_t<IsScalar<T>::value, int> = 0>
  D& operator*=(const T& s) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) *= s;
    return self();
  }
  template <typename T, std::enable_if_t<IsScalar<T>::value, int> = 0>
  D& operator/=(const T& s) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) /= s;
    return self();
  }

 protected:
  template <typename O>
  void check(const O& o) const {
    if (o.rows() != self().rows() || o.cols() != self().cols())
      throw std::invalid_argument("eigen shim: size mismatch");
  }
  template <typename O>
  void copyFrom(const O& o) {
    check(o);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) = o(i, j);
  }
};

// A view of a rectangular part of a Matrix (Eigen's Block<>). Assignment
// writes through to the viewed storage.
template <typename S>
class BlockView : public DenseBase<BlockView<S>, S> {
  using Base = DenseBase<BlockView<S>, S>;

 public:
  using typename Base::Scalar;
  BlockView(S* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld) {}
  BlockView(const BlockView&) = default;
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index ld() const { return ld_; }
  S* ptr() const { return p_; }
  S* data() const { return p_; }

  BlockView& operator=(const BlockView& o) {
    Base::copyFrom(o);
    return *this;
  }
  template <typename O, std::enable_if_t<IsDense<O>::value, int> = 0>
  BlockView& operator=(const O& o) {
    if (static_cast<const void*>(o.ptr()) == static_cast<const void*>(p_) && o.ld() == ld_) return *this;
    const Matrix<Scalar, Dynamic, Dynamic> tmp(o);  // eager: no aliasing between views
    Base::copyFrom(tmp);
    return *this;
  }

 private:
  S* p_;
  Index r_, c_, ld_;
};

template <typename S, int R, int C>
class Matrix : public DenseBase<Matrix<S, R, C>, S> {
  using Base = DenseBase<Matrix<S, R, C>, S>;

 public:
  using Scalar = S;
  Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : 0), d_(static_cast<size_t>(r_ * c_)) {}
  Matrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c)) { fixedCheck(); }
  // Vector of length n.
  explicit Matrix(Index n)
      : r_(C == 1 || (C == Dynamic && R != 1) ? n : 1), c_(C == 1 || (C == Dynamic && R != 1) ? 1 : n),
        d_(static_cast<size_t>(n)) {}
  // 3-vector from coordinates (Eigen::Vector3d(x, y, z)).
  Matrix(const S& a, const S& b, const S& c) : r_(3), c_(1), d_{a, b, c} {}
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) noexcept = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) noexcept = default;
  // Evaluation of any other dense object (other shape parameters, views).
  template <typename O, std::enable_if_t<IsDense<O>::value && !std::is_same_v<O, Matrix>, int> = 0>
  Matrix(const O& o) : r_(o.rows()), c_(o.cols()), d_(static_cast<size_t>(o.rows() * o.cols())) {
    fixedCheck();
    Base::copyFrom(o);
  }
  template <typename O, std::enable_if_t<IsDense<O>::value && !std::is_same_v<O, Matrix>, int> = 0>
  Matrix& operator=(const O& o) {
    Matrix tmp(o);
    *this = std::move(tmp);
    return *this;
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Zero(Index n) { return Matrix(n); }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Constant(const S& v) {
    Matrix out;
    std::fill(out.d_.begin(), out.d_.end(), v);
    return out;
  }
  static Matrix Constant(Index r, Index c, const S& v) {
    Matrix out(r, c);
    std::fill(out.d_.begin(), out.d_.end(), v);
    return out;
  }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), S{});
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index ld() const { return r_; }
  S* ptr() { return d_.data(); }
  const S* ptr() const { return d_.data(); }
  S* data() { return d_.data(); }
  const S* data() const { return d_.data(); }

 private:
  void fixedCheck() const {
    if ((R != Dynamic && r_ != R) || (C != Dynamic && c_ != C))
      throw std::invalid_argument("eigen shim: fixed-size mismatch");
  }
  Index r_, c_;
  std::vector<S> d_;
};

// ---- DenseBase members that build a Matrix
template <typename D, typename S>
typename DenseBase<D, S>::Plain DenseBase<D, S>::eval() const {
  return Plain(self());
}
template <typename D, typename S>
typename DenseBase<D, S>::Plain DenseBase<D, S>::transpose() const {
  Plain out(self().cols(), self().rows());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) out(j, i) = (*this)(i, j);
  return out;
}
template <typename D, typename S>
Matrix<typename DenseBase<D, S>::Scalar, Dynamic, 1> DenseBase<D, S>::diagonal() const {
  const Index n = std::min(self().rows(), self().cols());
  Matrix<Scalar, Dynamic, 1> out(n);
  for (Index i = 0; i < n; ++i) out(i) = (*this)(i, i);
  return out;
}
template <typename D, typename S>
template <typename O>
typename DenseBase<D, S>::Plain DenseBase<D, S>::cwiseProduct(const O& o) const {
  check(o);
  Plain out(self().rows(), self().cols());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) out(i, j) = (*this)(i, j) * o(i, j);
  return out;
}
template <typename D, typename S>
Matrix<typename DenseBase<D, S>::Real, Dynamic, Dynamic> DenseBase<D, S>::cwiseAbs() const {
  Matrix<Real, Dynamic, Dynamic> out(self().rows(), self().cols());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) out(i, j) = std::abs((*this)(i, j));
  return out;
}
template <typename D, typename S>
template <typename O>
typename DenseBase<D, S>::Plain DenseBase<D, S>::cwiseMin(const O& o) const {
  check(o);
  Plain out(self().rows(), self().cols());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) out(i, j) = std::min((*this)(i, j), o(i, j));
  return out;
}
template <typename D, typename S>
template <typename O>
typename DenseBase<D, S>::Plain DenseBase<D, S>::cwiseMax(const O& o) const {
  check(o);
  Plain out(self().rows(), self().cols());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) out(i, j) = std::max((*this)(i, j), o(i, j));
  return out;
}
template <typename D, typename S>
template <typename O>
typename DenseBase<D, S>::Plain DenseBase<D, S>::cross(const O& o) const {
  Plain out(3, 1);
  const auto& a = *this;
  out(0) = a(1) * o(2) - a(2) * o(1);
  out(1) = a(2) * o(0) - a(0) * o(2);
  out(2) = a(0) * o(1) - a(1) * o(0);
  return out;
}

// ---- free operators on dense objects (eager, sizes checked)
template <typename A>
using PlainOf = Matrix<typename A::Scalar, Dynamic, Dynamic>;

template <typename A, typename B, std::enable_if_t<IsDense<A>::value && IsDense<B>::value, int> = 0>
PlainOf<A> operator+(const A& a, const B& b) {
  PlainOf<A> out(a);
  out += b;
  return out;
}
template <typename A, typename B, std::enable_if_t<IsDense<A>::value && IsDense<B>::value, int> = 0>
PlainOf<A> operator-(const A& a, const B& b) {
  PlainOf<A> out(a);
  out -= b;
  return out;
}
template <typename A, std::enable_if_t<IsDense<A>::value, int> = 0>
PlainOf<A> operator-(const A& a) {
  PlainOf<A> out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = -a(i, j);
  return out;
}
// Matrix product, accumulated over the inner index in increasing order.
template <typename A, typename B, std::enable_if_t<IsDense<A>::value && IsDense<B>::value, int> = 0>
PlainOf<A> operator*(const A& a, const B& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("eigen shim: product size mismatch");
  PlainOf<A> out(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const auto bkj = b(k, j);
      for (Index i = 0; i < a.rows(); ++i) out(i, j) += a(i, k) * bkj;
    }
  return out;
}
template <typename T, typename A, std::enable_if_t<IsScalar<T>::value && IsDense<A>::value, int> = 0>
PlainOf<A> operator*(const T& s, const A& a) {
  PlainOf<A> out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = s * a(i, j);
  return out;
}
template <typename A, typename T, std::enable_if_t<IsScalar<T>::value && IsDense<A>::value, int> = 0>
PlainOf<A> operator*(const A& a, const T& s) {
  PlainOf<A> out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = a(i, j) * s;
  return out;
}
template <typename A, typename T, std::enable_if_t<IsScalar<T>::value && IsDense<A>::value, int> = 0>
PlainOf<A> operator/(const A& a, const T& s) {
  PlainOf<A> out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = a(i, j) / s;
  return out;
}

using Vector3d = Matrix<double, 3, 1>;
using Matrix3Xd = Matrix<double, 3, Dynamic>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;

// LU with row partial pivoting: P A = L U, L unit lower triangular.
template <typename M>
class PartialPivLU {
 public:
  using Scalar = typename M::Scalar;
  explicit PartialPivLU(const M& a) : lu_(a), perm_(static_cast<size_t>(a.rows())) {
    const Index n = lu_.rows();
    if (lu_.cols() != n) throw std::invalid_argument("eigen shim: PartialPivLU needs a square matrix");
    for (Index i = 0; i < n; ++i) perm_[static_cast<size_t>(i)] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      double best = std::abs(lu_(k, k));
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu_(i, k)) > best) {
          best = std::abs(lu_(i, k));
          p = i;
        }
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[static_cast<size_t>(k)], perm_[static_cast<size_t>(p)]);
      }
      const Scalar piv = lu_(k, k);
      if (piv == Scalar{}) continue;  // singular column: leave zeros (Eigen does not throw either)
      for (Index i = k + 1; i < n; ++i) lu_(i, k) /= piv;
      for (Index j = k + 1; j < n; ++j) {
        const Scalar u = lu_(k, j);
        for (Index i = k + 1; i < n; ++i) lu_(i, j) -= lu_(i, k) * u;
      }
    }
  }
  const M& matrixLU() const { return lu_; }

  template <typename B>
  Matrix<Scalar, Dynamic, Dynamic> solve(const B& b) const {
    const Index n = lu_.rows();
    Matrix<Scalar, Dynamic, Dynamic> x(n, b.cols());
    for (Index c = 0; c < b.cols(); ++c) {
      for (Index i = 0; i < n; ++i) x(i, c) = b(perm_[static_cast<size_t>(i)], c);
      for (Index i = 0; i < n; ++i)
        for (Index k = 0; k < i; ++k) x(i, c) -= lu_(i, k) * x(k, c);
      for (Index i = n - 1; i >= 0; --i) {
        for (Index k = i + 1; k < n; ++k) x(i, c) -= lu_(i, k) * x(k, c);
        x(i, c) /= lu_(i, i);
      }
    }
    return x;
  }

 private:
  M lu_;
  std::vector<Index> perm_;
};

}  // namespace Eigen
