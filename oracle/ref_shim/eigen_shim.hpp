// Minimal Eigen-API restatement — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// The reference (/root/reference/proj) depends on Eigen3 (CMakeLists.txt:12, version unpinned),
// which is absent from this image.  This header restates the subset of Eigen's PUBLIC API that the
// reference's hot-path sources and unit tests use, so that the UNMODIFIED reference files
// (src/{geometry,image,solver,synth,gradcheck}.cpp, tests/test_*.cpp) compile against it:
//
//   * Matrix<Scalar, Rows, Cols> (column-major, fixed or Dynamic sizes), the typedefs
//     (Vector2d/3d, Matrix3d/4d, VectorXd, MatrixXd, Vector2i), Zero/Identity, comma initialiser;
//   * coefficient access, blocks as writable views (block/head/tail/segment/col/row/corners,
//     diagonal().array()), transpose, arithmetic, products, norms, dot/cross, cwiseAbs, maxCoeff,
//     isZero, allFinite, determinant (3x3), trace, cast, asDiagonal, noalias;
//   * LDLT<MatrixXd> with Eigen's documented algorithm: a robust Cholesky with symmetric diagonal
//     pivoting (the largest remaining |diagonal| is swapped to the front at each step), P^T L D L^T P,
//     info() = NumericalIssue when a valid pivot follows a zero pivot, and solve() using the
//     pseudo-inverse of D (entries with |D_ii| <= DBL_MIN give 0), as Eigen 3.3/3.4's LDLT does.
//
// Evaluation is eager (no expression templates): every operator returns a concrete Matrix.  This
// changes only the floating-point summation order inside products relative to a vectorised Eigen
// build (roundoff level), which the parity tolerances absorb.  Written from the Eigen API
// documentation; no Eigen source is included.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

template <class S, int R, int C, int Options = 0, int MaxR = R, int MaxC = C>
class Matrix;
template <class S, int R, int C, bool Const>
class MapView;

namespace internal {
inline void check(bool ok, const char* what) {
  if (!ok) throw std::logic_error(std::string("eigen_shim: ") + what);
}
constexpr int prod_dim(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : a * b; }
constexpr int merge_dim(int a, int b) { return a == Dynamic ? b : a; }
}  // namespace internal

// ---------------------------------------------------------------------------------------------
// CRTP base: everything is expressed through rows(), cols(), coeff(i,j) and coeffRef(i,j).
// ---------------------------------------------------------------------------------------------
template <class Derived, class S, int R, int C>
class MatBase {
 public:
  using Scalar = S;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr bool IsVectorAtCompileTime = (R == 1 || C == 1);
  using PlainObject = Matrix<S, R, C>;

  const Derived& derived() const { return static_cast<const Derived&>(*this); }
  Derived& derived() { return static_cast<Derived&>(*this); }

  Index rows() const { return derived().rows_impl(); }
  Index cols() const { return derived().cols_impl(); }
  Index size() const { return rows() * cols(); }
  S coeff(Index i, Index j) const { return derived().coeff_impl(i, j); }
  S& coeffRef(Index i, Index j) { return derived().coeffref_impl(i, j); }

  // linear (vector) access: column vectors index rows, row vectors index columns
  S coeff(Index k) const { return rows() == 1 ? coeff(0, k) : (cols() == 1 ? coeff(k, 0) : coeff(k % rows(), k / rows())); }
  S& coeffRef(Index k) { return rows() == 1 ? coeffRef(0, k) : (cols() == 1 ? coeffRef(k, 0) : coeffRef(k % rows(), k / rows())); }
  S operator()(Index i, Index j) const { return coeff(i, j); }
  S& operator()(Index i, Index j) { return coeffRef(i, j); }
  S operator()(Index k) const { return coeff(k); }
  S& operator()(Index k) { return coeffRef(k); }
  S operator[](Index k) const { return coeff(k); }
  S& operator[](Index k) { return coeffRef(k); }
  S x() const { return coeff(0); }
  S y() const { return coeff(1); }
  S z() const { return coeff(2); }
  S w() const { return coeff(3); }
  S& x() { return coeffRef(0); }
  S& y() { return coeffRef(1); }
  S& z() { return coeffRef(2); }
  S& w() { return coeffRef(3); }

  PlainObject eval() const { return PlainObject(derived()); }

  // ---- views -------------------------------------------------------------------------------
  template <int BR, int BC>
  MapView<S, BR, BC, false> block(Index i, Index j) { return derived().template view<BR, BC>(i, j, BR, BC); }
  template <int BR, int BC>
  MapView<S, BR, BC, true> block(Index i, Index j) const { return derived().template cview<BR, BC>(i, j, BR, BC); }
  MapView<S, Dynamic, Dynamic, false> block(Index i, Index j, Index r, Index c) {
    return derived().template view<Dynamic, Dynamic>(i, j, r, c);
  }
  MapView<S, Dynamic, Dynamic, true> block(Index i, Index j, Index r, Index c) const {
    return derived().template cview<Dynamic, Dynamic>(i, j, r, c);
  }
  template <int BR, int BC>
  MapView<S, BR, BC, false> topLeftCorner() { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  MapView<S, BR, BC, true> topLeftCorner() const { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  MapView<S, BR, BC, false> topRightCorner() { return block<BR, BC>(0, cols() - BC); }
  template <int BR, int BC>
  MapView<S, BR, BC, true> topRightCorner() const { return block<BR, BC>(0, cols() - BC); }
  template <int BR, int BC>
  MapView<S, BR, BC, false> bottomLeftCorner() { return block<BR, BC>(rows() - BR, 0); }
  template <int BR, int BC>
  MapView<S, BR, BC, true> bottomLeftCorner() const { return block<BR, BC>(rows() - BR, 0); }
  template <int BR, int BC>
  MapView<S, BR, BC, false> bottomRightCorner() { return block<BR, BC>(rows() - BR, cols() - BC); }
  template <int BR, int BC>
  MapView<S, BR, BC, true> bottomRightCorner() const { return block<BR, BC>(rows() - BR, cols() - BC); }

  MapView<S, R, 1, false> col(Index j) { return derived().template view<R, 1>(0, j, rows(), 1); }
  MapView<S, R, 1, true> col(Index j) const { return derived().template cview<R, 1>(0, j, rows(), 1); }
  MapView<S, 1, C, false> row(Index i) { return derived().template view<1, C>(i, 0, 1, cols()); }
  MapView<S, 1, C, true> row(Index i) const { return derived().template cview<1, C>(i, 0, 1, cols()); }

  // vector segments keep the orientation of the vector
  template <int N>
  using SegV = MapView<S, (R == 1 ? 1 : N), (R == 1 ? N : 1), false>;
  template <int N>
  using SegC = MapView<S, (R == 1 ? 1 : N), (R == 1 ? N : 1), true>;
  template <int N>
  SegV<N> segment(Index start) { return seg_<N, false>(start, N); }
  template <int N>
  SegC<N> segment(Index start) const { return seg_<N, true>(start, N); }
  template <int N>
  SegV<N> head() { return segment<N>(0); }
  template <int N>
  SegC<N> head() const { return segment<N>(0); }
  template <int N>
  SegV<N> tail() { return segment<N>(size() - N); }
  template <int N>
  SegC<N> tail() const { return segment<N>(size() - N); }
  SegV<Dynamic> segment(Index start, Index n) { return seg_<Dynamic, false>(start, n); }
  SegC<Dynamic> segment(Index start, Index n) const { return seg_<Dynamic, true>(start, n); }
  SegV<Dynamic> head(Index n) { return segment(0, n); }
  SegC<Dynamic> head(Index n) const { return segment(0, n); }
  SegV<Dynamic> tail(Index n) { return segment(size() - n, n); }
  SegC<Dynamic> tail(Index n) const { return segment(size() - n, n); }

  MapView<S, Dynamic, 1, false> diagonal() { return derived().diag_view(); }
  MapView<S, Dynamic, 1, true> diagonal() const { return derived().cdiag_view(); }

  Derived& noalias() { return derived(); }
  Derived& array() { return derived(); }
  const Derived& array() const { return derived(); }
  Derived& matrix() { return derived(); }

  // ---- reductions ------------------------------------------------------------------------
  S squaredNorm() const {
    S s = 0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j) * coeff(i, j);
    return s;
  }
  S norm() const { return std::sqrt(squaredNorm()); }
  S sum() const {
    S s = 0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j);
    return s;
  }
  S trace() const {
    S s = 0;
    for (Index i = 0; i < std::min(rows(), cols()); ++i) s += coeff(i, i);
    return s;
  }
  S value() const {
    internal::check(rows() == 1 && cols() == 1, "value() of a non-1x1");
    return coeff(0, 0);
  }
  S maxCoeff() const {
    S m = coeff(0, 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) m = std::max(m, coeff(i, j));
    return m;
  }
  S minCoeff() const {
    S m = coeff(0, 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) m = std::min(m, coeff(i, j));
    return m;
  }
  template <class IndexT>
  S maxCoeff(IndexT* idx) const {  // vectors: first index of the maximum
    Index best = 0;
    for (Index k = 1; k < size(); ++k)
      if (coeff(k) > coeff(best)) best = k;
    *idx = static_cast<IndexT>(best);
    return coeff(best);
  }
  template <class IndexT>
  S maxCoeff(IndexT* ri, IndexT* ci) const {
    Index bi = 0, bj = 0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (coeff(i, j) > coeff(bi, bj)) bi = i, bj = j;
    *ri = static_cast<IndexT>(bi);
    *ci = static_cast<IndexT>(bj);
    return coeff(bi, bj);
  }
  bool allFinite() const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (!std::isfinite(static_cast<double>(coeff(i, j)))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (std::isnan(static_cast<double>(coeff(i, j)))) return true;
    return false;
  }
  // Eigen: isMuchSmallerThan(x, 1, prec)  <=>  |x| <= prec  for every coefficient
  bool isZero(double prec = 1e-12) const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (std::abs(coeff(i, j)) > prec) return false;
    return true;
  }
  template <class D2, int R2, int C2>
  S dot(const MatBase<D2, S, R2, C2>& o) const {
    internal::check(size() == o.size(), "dot size mismatch");
    S s = 0;
    for (Index k = 0; k < size(); ++k) s += coeff(k) * o.coeff(k);
    return s;
  }
  template <class D2, int R2, int C2>
  Matrix<S, 3, 1> cross(const MatBase<D2, S, R2, C2>& b) const {
    internal::check(size() == 3 && b.size() == 3, "cross of non-3-vectors");
    return Matrix<S, 3, 1>(coeff(1) * b.coeff(2) - coeff(2) * b.coeff(1),
                           coeff(2) * b.coeff(0) - coeff(0) * b.coeff(2),
                           coeff(0) * b.coeff(1) - coeff(1) * b.coeff(0));
  }
  S determinant() const {
    internal::check(rows() == cols(), "determinant of a non-square matrix");
    const Index n = rows();
    if (n == 1) return coeff(0, 0);
    if (n == 2) return coeff(0, 0) * coeff(1, 1) - coeff(0, 1) * coeff(1, 0);
    if (n == 3) {
      // cofactor expansion along the first column
      return coeff(0, 0) * (coeff(1, 1) * coeff(2, 2) - coeff(2, 1) * coeff(1, 2)) -
             coeff(1, 0) * (coeff(0, 1) * coeff(2, 2) - coeff(2, 1) * coeff(0, 2)) +
             coeff(2, 0) * (coeff(0, 1) * coeff(1, 2) - coeff(1, 1) * coeff(0, 2));
    }
    // partial-pivoting LU
    Matrix<S, Dynamic, Dynamic> a(derived());
    S det = 1;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      if (a(p, k) == S(0)) return S(0);
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(a(p, j), a(k, j));
        det = -det;
      }
      det *= a(k, k);
      for (Index i = k + 1; i < n; ++i) {
        const S l = a(i, k) / a(k, k);
        for (Index j = k + 1; j < n; ++j) a(i, j) -= l * a(k, j);
      }
    }
    return det;
  }

  // ---- element-wise ----------------------------------------------------------------------
  PlainObject cwiseAbs() const {
    PlainObject out(derived());
    for (Index j = 0; j < out.cols(); ++j)
      for (Index i = 0; i < out.rows(); ++i) out(i, j) = std::abs(out(i, j));
    return out;
  }
  PlainObject abs() const { return cwiseAbs(); }
  template <class D2>
  PlainObject cwiseProduct(const MatBase<D2, S, R, C>& o) const {
    PlainObject out(derived());
    for (Index j = 0; j < out.cols(); ++j)
      for (Index i = 0; i < out.rows(); ++i) out(i, j) *= o.coeff(i, j);
    return out;
  }
  Matrix<S, C, R> transpose() const {
    Matrix<S, C, R> out(cols(), rows(), 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out(j, i) = coeff(i, j);
    return out;
  }
  Matrix<S, C, R> adjoint() const { return transpose(); }
  PlainObject normalized() const {
    PlainObject out(derived());
    const S n = norm();
    if (n > S(0)) out /= n;
    return out;
  }
  void normalize() {
    const S n = norm();
    if (n > S(0)) derived() /= n;
  }
  template <class T>
  Matrix<T, R, C> cast() const {
    Matrix<T, R, C> out(rows(), cols(), 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out(i, j) = static_cast<T>(coeff(i, j));
    return out;
  }
  Matrix<S, Dynamic, Dynamic> asDiagonal() const {
    Matrix<S, Dynamic, Dynamic> out = Matrix<S, Dynamic, Dynamic>::Zero(size(), size());
    for (Index k = 0; k < size(); ++k) out(k, k) = coeff(k);
    return out;
  }
  auto ldlt() const;

  // ---- in-place arithmetic ---------------------------------------------------------------
  void setZero() {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = S(0);
  }
  void setConstant(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = v;
  }
  void setIdentity() {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = S(i == j ? 1 : 0);
  }
  template <class D2, int R2, int C2>
  Derived& operator+=(const MatBase<D2, S, R2, C2>& o) {
    const PlainObject t(o.derived());  // alias-safe
    internal::check(t.rows() == rows() && t.cols() == cols(), "+= size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) += t(i, j);
    return derived();
  }
  template <class D2, int R2, int C2>
  Derived& operator-=(const MatBase<D2, S, R2, C2>& o) {
    const PlainObject t(o.derived());
    internal::check(t.rows() == rows() && t.cols() == cols(), "-= size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) -= t(i, j);
    return derived();
  }
  Derived& operator+=(S v) {  // array semantics (used through .array())
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) += v;
    return derived();
  }
  Derived& operator-=(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) -= v;
    return derived();
  }
  Derived& operator*=(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) *= v;
    return derived();
  }
  Derived& operator/=(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) /= v;
    return derived();
  }
  template <class D2, int R2, int C2>
  void assign_from(const MatBase<D2, S, R2, C2>& o) {
    const PlainObject t(o.derived());
    internal::check(t.rows() == rows() && t.cols() == cols(), "assignment size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = t(i, j);
  }

 private:
  template <int N, bool Const>
  auto seg_(Index start, Index n) const {
    constexpr int VR = (R == 1 ? 1 : N), VC = (R == 1 ? N : 1);
    Derived& d = const_cast<Derived&>(derived());
    const bool is_row = (rows() == 1 && cols() != 1);
    if constexpr (Const) {
      return is_row ? d.template cview<VR, VC>(0, start, 1, n) : d.template cview<VR, VC>(start, 0, n, 1);
    } else {
      return is_row ? d.template view<VR, VC>(0, start, 1, n) : d.template view<VR, VC>(start, 0, n, 1);
    }
  }
};

// ---------------------------------------------------------------------------------------------
// Strided view into contiguous column-major storage: (i, j) -> data[i*inner + j*outer]
// ---------------------------------------------------------------------------------------------
template <class S, int R, int C, bool Const>
class MapView : public MatBase<MapView<S, R, C, Const>, S, R, C> {
  using Base = MatBase<MapView<S, R, C, Const>, S, R, C>;
  using Ptr = std::conditional_t<Const, const S*, S*>;

 public:
  MapView(Ptr data, Index rows, Index cols, Index inner, Index outer)
      : d_(data), r_(rows), c_(cols), in_(inner), out_(outer) {
    if (R != Dynamic) internal::check(rows == R, "view rows");
    if (C != Dynamic) internal::check(cols == C, "view cols");
  }
  MapView(const MapView&) = default;

  Index rows_impl() const { return r_; }
  Index cols_impl() const { return c_; }
  S coeff_impl(Index i, Index j) const { return d_[i * in_ + j * out_]; }
  S& coeffref_impl(Index i, Index j) {
    static_assert(!Const, "write through a const view");
    return const_cast<S&>(d_[i * in_ + j * out_]);
  }

  template <int BR, int BC>
  MapView<S, BR, BC, Const> view(Index i, Index j, Index r, Index c) {
    return MapView<S, BR, BC, Const>(d_ + i * in_ + j * out_, r, c, in_, out_);
  }
  template <int BR, int BC>
  MapView<S, BR, BC, true> cview(Index i, Index j, Index r, Index c) const {
    return MapView<S, BR, BC, true>(d_ + i * in_ + j * out_, r, c, in_, out_);
  }
  MapView<S, Dynamic, 1, Const> diag_view() {
    return MapView<S, Dynamic, 1, Const>(d_, std::min(r_, c_), 1, in_ + out_, out_);
  }
  MapView<S, Dynamic, 1, true> cdiag_view() const {
    return MapView<S, Dynamic, 1, true>(d_, std::min(r_, c_), 1, in_ + out_, out_);
  }

  template <class D2, int R2, int C2>
  MapView& operator=(const MatBase<D2, S, R2, C2>& o) {
    this->assign_from(o);
    return *this;
  }
  MapView& operator=(const MapView& o) {
    this->assign_from(o);
    return *this;
  }
  void swap(MapView other) {
    internal::check(other.rows() == r_ && other.cols() == c_, "swap size mismatch");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) std::swap(this->coeffRef(i, j), other.coeffRef(i, j));
  }

 private:
  Ptr d_;
  Index r_, c_, in_, out_;
};

// ---------------------------------------------------------------------------------------------
// Dense matrix, column-major. Fixed sizes live in a std::array, Dynamic ones in a std::vector.
// ---------------------------------------------------------------------------------------------
namespace internal {
template <class S, int R, int C>
struct Storage {
  static constexpr bool fixed = (R != Dynamic && C != Dynamic);
  std::array<S, (R > 0 ? R : 1) * (C > 0 ? C : 1)> a{};
  Index r = R, c = C;
  S* data() { return a.data(); }
  const S* data() const { return a.data(); }
  void resize(Index rr, Index cc) { check(rr == R && cc == C, "resize of a fixed-size matrix"); }
};
template <class S, int R, int C>
  requires(R == Dynamic || C == Dynamic)
struct Storage<S, R, C> {
  static constexpr bool fixed = false;
  std::vector<S> v;
  Index r = (R == Dynamic ? 0 : R), c = (C == Dynamic ? 0 : C);
  S* data() { return v.data(); }
  const S* data() const { return v.data(); }
  void resize(Index rr, Index cc) {
    if (R != Dynamic) check(rr == R, "resize rows of fixed dimension");
    if (C != Dynamic) check(cc == C, "resize cols of fixed dimension");
    r = rr;
    c = cc;
    v.assign(static_cast<size_t>(rr * cc), S(0));
  }
};
}  // namespace internal

template <class S, int R, int C>
class CommaInit;

template <class S, int R, int C, int Options, int MaxR, int MaxC>
class Matrix : public MatBase<Matrix<S, R, C, Options, MaxR, MaxC>, S, R, C> {
  using Base = MatBase<Matrix, S, R, C>;
  internal::Storage<S, R, C> st_;

 public:
  using Scalar = S;
  static constexpr bool FixedSize = (R != Dynamic && C != Dynamic);

  Matrix() {}
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) = default;

  // internal sized constructor (r, c, tag)
  Matrix(Index r, Index c, int) { st_.resize(r, c); }

  // Dynamic vector: Matrix(n); dynamic matrix: Matrix(r, c); fixed vectors: coefficients.
  template <class T>
    requires(std::is_integral_v<T> && !FixedSize)
  explicit Matrix(T n) {
    if (R == 1)
      st_.resize(1, n);
    else
      st_.resize(n, 1);
  }
  template <class T0, class T1>
    requires(std::is_arithmetic_v<T0> && std::is_arithmetic_v<T1>)
  Matrix(T0 a, T1 b) {
    if constexpr (FixedSize) {
      static_assert(R * C == 2, "2-coefficient constructor on a non-2-vector");
      st_.data()[0] = static_cast<S>(a);
      st_.data()[1] = static_cast<S>(b);
    } else {
      st_.resize(static_cast<Index>(a), static_cast<Index>(b));
    }
  }
  template <class T0, class T1, class T2>
    requires(std::is_arithmetic_v<T0> && std::is_arithmetic_v<T1> && std::is_arithmetic_v<T2>)
  Matrix(T0 a, T1 b, T2 c) {
    static_assert(FixedSize && R * C == 3, "3-coefficient constructor on a non-3-vector");
    st_.data()[0] = static_cast<S>(a);
    st_.data()[1] = static_cast<S>(b);
    st_.data()[2] = static_cast<S>(c);
  }
  template <class T0, class T1, class T2, class T3>
    requires(std::is_arithmetic_v<T0> && std::is_arithmetic_v<T1> && std::is_arithmetic_v<T2> &&
             std::is_arithmetic_v<T3>)
  Matrix(T0 a, T1 b, T2 c, T3 d) {
    static_assert(FixedSize && R * C == 4, "4-coefficient constructor on a non-4-vector");
    st_.data()[0] = static_cast<S>(a);
    st_.data()[1] = static_cast<S>(b);
    st_.data()[2] = static_cast<S>(c);
    st_.data()[3] = static_cast<S>(d);
  }
  // from any expression of compatible size
  template <class D2, int R2, int C2>
  Matrix(const MatBase<D2, S, R2, C2>& o) {
    const Index rr = o.rows(), cc = o.cols();
    if constexpr (FixedSize) {
      internal::check(rr * cc == R * C && (rr == R || R == 1 || C == 1), "fixed-size construction mismatch");
      // vectors may be built from either orientation (as Eigen does for vector <-> vector copies)
      if (rr == R) {
        for (Index j = 0; j < cc; ++j)
          for (Index i = 0; i < rr; ++i) (*this)(i, j) = o.coeff(i, j);
      } else {
        for (Index k = 0; k < rr * cc; ++k) this->coeffRef(k) = o.coeff(k);
      }
    } else {
      Index tr = rr, tc = cc;
      if (R == 1 && rr != 1) std::swap(tr, tc);  // row-vector target from a column vector
      if (C == 1 && cc != 1) std::swap(tr, tc);
      st_.resize(tr, tc);
      if (tr == rr) {
        for (Index j = 0; j < cc; ++j)
          for (Index i = 0; i < rr; ++i) (*this)(i, j) = o.coeff(i, j);
      } else {
        for (Index k = 0; k < rr * cc; ++k) this->coeffRef(k) = o.coeff(k);
      }
    }
  }
  template <class D2, int R2, int C2>
  Matrix& operator=(const MatBase<D2, S, R2, C2>& o) {
    Matrix t(o);
    *this = std::move(t);
    return *this;
  }

  Index rows_impl() const { return st_.r; }
  Index cols_impl() const { return st_.c; }
  S coeff_impl(Index i, Index j) const { return st_.data()[i + j * st_.r]; }
  S& coeffref_impl(Index i, Index j) { return st_.data()[i + j * st_.r]; }
  S* data() { return st_.data(); }
  const S* data() const { return st_.data(); }

  template <int BR, int BC>
  MapView<S, BR, BC, false> view(Index i, Index j, Index r, Index c) {
    internal::check(i >= 0 && j >= 0 && i + r <= st_.r && j + c <= st_.c, "block out of range");
    return MapView<S, BR, BC, false>(st_.data() + i + j * st_.r, r, c, 1, st_.r);
  }
  template <int BR, int BC>
  MapView<S, BR, BC, true> cview(Index i, Index j, Index r, Index c) const {
    internal::check(i >= 0 && j >= 0 && i + r <= st_.r && j + c <= st_.c, "block out of range");
    return MapView<S, BR, BC, true>(st_.data() + i + j * st_.r, r, c, 1, st_.r);
  }
  MapView<S, Dynamic, 1, false> diag_view() {
    return MapView<S, Dynamic, 1, false>(st_.data(), std::min(st_.r, st_.c), 1, st_.r + 1, st_.r);
  }
  MapView<S, Dynamic, 1, true> cdiag_view() const {
    return MapView<S, Dynamic, 1, true>(st_.data(), std::min(st_.r, st_.c), 1, st_.r + 1, st_.r);
  }

  void resize(Index n) {
    if (R == 1)
      st_.resize(1, n);
    else
      st_.resize(n, 1);
  }
  void resize(Index r, Index c) { st_.resize(r, c); }
  Matrix& setZero(Index n) {
    resize(n);
    return *this;
  }
  Matrix& setZero(Index r, Index c) {
    resize(r, c);
    return *this;
  }
  using Base::setZero;

  static Matrix Zero() {
    static_assert(FixedSize, "Zero() needs sizes for a dynamic matrix");
    return Matrix();
  }
  static Matrix Zero(Index n) {
    Matrix m;
    m.resize(n);
    return m;
  }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c, 0); }
  static Matrix Ones() {
    Matrix m;
    m.setConstant(S(1));
    return m;
  }
  static Matrix Constant(S v) {
    Matrix m;
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index r, Index c, S v) {
    Matrix m(r, c, 0);
    m.setConstant(v);
    return m;
  }
  static Matrix Identity() {
    static_assert(FixedSize, "Identity() needs sizes for a dynamic matrix");
    Matrix m;
    m.setIdentity();
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c, 0);
    m.setIdentity();
    return m;
  }
  static Matrix Unit(Index k) {
    Matrix m;
    m(k) = S(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

  CommaInit<S, R, C> operator<<(S v);
  template <class D2, int R2, int C2>
  CommaInit<S, R, C> operator<<(const MatBase<D2, S, R2, C2>& m);
};

// comma initialiser: fills row by row; a matrix piece occupies a block of the current row band
template <class S, int R, int C>
class CommaInit {
 public:
  explicit CommaInit(Matrix<S, R, C>& m) : m_(m) {}
  CommaInit& operator,(S v) {
    place_scalar(v);
    return *this;
  }
  template <class D2, int R2, int C2>
  CommaInit& operator,(const MatBase<D2, S, R2, C2>& b) {
    place_block(b);
    return *this;
  }
  void place_scalar(S v) {
    advance_if_full();
    m_(row_, col_) = v;
    band_ = std::max<Index>(band_, 1);
    col_ += 1;
  }
  template <class D2, int R2, int C2>
  void place_block(const MatBase<D2, S, R2, C2>& b) {
    advance_if_full();
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < b.rows(); ++i) m_(row_ + i, col_ + j) = b.coeff(i, j);
    band_ = std::max<Index>(band_, b.rows());
    col_ += b.cols();
  }

 private:
  void advance_if_full() {
    if (col_ >= m_.cols()) {
      row_ += band_;
      col_ = 0;
      band_ = 0;
    }
    internal::check(row_ < m_.rows(), "comma initialiser overflow");
  }
  Matrix<S, R, C>& m_;
  Index row_ = 0, col_ = 0, band_ = 0;
};

template <class S, int R, int C, int O, int MR, int MC>
CommaInit<S, R, C> Matrix<S, R, C, O, MR, MC>::operator<<(S v) {
  CommaInit<S, R, C> ci(reinterpret_cast<Matrix<S, R, C>&>(*this));
  ci.place_scalar(v);
  return ci;
}
template <class S, int R, int C, int O, int MR, int MC>
template <class D2, int R2, int C2>
CommaInit<S, R, C> Matrix<S, R, C, O, MR, MC>::operator<<(const MatBase<D2, S, R2, C2>& m) {
  CommaInit<S, R, C> ci(reinterpret_cast<Matrix<S, R, C>&>(*this));
  ci.place_block(m);
  return ci;
}

// ---------------------------------------------------------------------------------------------
// arithmetic (eager)
// ---------------------------------------------------------------------------------------------
template <class D1, class D2, class S, int R1, int C1, int R2, int C2>
Matrix<S, internal::merge_dim(R1, R2), internal::merge_dim(C1, C2)> operator+(const MatBase<D1, S, R1, C1>& a,
                                                                           const MatBase<D2, S, R2, C2>& b) {
  internal::check(a.rows() == b.rows() && a.cols() == b.cols(), "+ size mismatch");
  Matrix<S, internal::merge_dim(R1, R2), internal::merge_dim(C1, C2)> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) += b.coeff(i, j);
  return out;
}
template <class D1, class D2, class S, int R1, int C1, int R2, int C2>
Matrix<S, internal::merge_dim(R1, R2), internal::merge_dim(C1, C2)> operator-(const MatBase<D1, S, R1, C1>& a,
                                                                           const MatBase<D2, S, R2, C2>& b) {
  internal::check(a.rows() == b.rows() && a.cols() == b.cols(), "- size mismatch");
  Matrix<S, internal::merge_dim(R1, R2), internal::merge_dim(C1, C2)> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) -= b.coeff(i, j);
  return out;
}
template <class D, class S, int R, int C>
Matrix<S, R, C> operator-(const MatBase<D, S, R, C>& a) {
  Matrix<S, R, C> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) = -out(i, j);
  return out;
}
template <class D, class S, int R, int C, class T>
  requires std::is_arithmetic_v<T>
Matrix<S, R, C> operator*(const MatBase<D, S, R, C>& a, T s) {
  Matrix<S, R, C> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) *= static_cast<S>(s);
  return out;
}
template <class D, class S, int R, int C, class T>
  requires std::is_arithmetic_v<T>
Matrix<S, R, C> operator*(T s, const MatBase<D, S, R, C>& a) {
  Matrix<S, R, C> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) = static_cast<S>(s) * out(i, j);
  return out;
}
template <class D, class S, int R, int C, class T>
  requires std::is_arithmetic_v<T>
Matrix<S, R, C> operator/(const MatBase<D, S, R, C>& a, T s) {
  Matrix<S, R, C> out(a.derived());
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) /= static_cast<S>(s);
  return out;
}
// matrix product: each coefficient is the in-order inner sum a(i,0)b(0,j) + a(i,1)b(1,j) + ...
template <class D1, class D2, class S, int R1, int C1, int R2, int C2>
Matrix<S, R1, C2> operator*(const MatBase<D1, S, R1, C1>& a, const MatBase<D2, S, R2, C2>& b) {
  internal::check(a.cols() == b.rows(), "product size mismatch");
  Matrix<S, R1, C2> out(a.rows(), b.cols(), 0);
  const Index K = a.cols();
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      S s = 0;
      for (Index k = 0; k < K; ++k) s += a.coeff(i, k) * b.coeff(k, j);
      out(i, j) = s;
    }
  return out;
}
template <class D1, class D2, class S, int R1, int C1, int R2, int C2>
bool operator==(const MatBase<D1, S, R1, C1>& a, const MatBase<D2, S, R2, C2>& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (a.coeff(i, j) != b.coeff(i, j)) return false;
  return true;
}
template <class D1, class D2, class S, int R1, int C1, int R2, int C2>
bool operator!=(const MatBase<D1, S, R1, C1>& a, const MatBase<D2, S, R2, C2>& b) {
  return !(a == b);
}
template <class D, class S, int R, int C>
std::ostream& operator<<(std::ostream& os, const MatBase<D, S, R, C>& m) {
  for (Index i = 0; i < m.rows(); ++i) {
    for (Index j = 0; j < m.cols(); ++j) os << (j ? " " : "") << m.coeff(i, j);
    if (i + 1 < m.rows()) os << "\n";
  }
  return os;
}

// ---------------------------------------------------------------------------------------------
// LDLT: robust Cholesky with symmetric diagonal pivoting (Eigen's LDLT<MatrixType, Lower>)
// ---------------------------------------------------------------------------------------------
template <class MatrixType>
class LDLT {
  using S = typename MatrixType::Scalar;
  using Mat = Matrix<S, Dynamic, Dynamic>;

 public:
  LDLT() = default;
  template <class D, int R, int C>
  explicit LDLT(const MatBase<D, S, R, C>& a) {
    compute(a);
  }

  template <class D, int R, int C>
  LDLT& compute(const MatBase<D, S, R, C>& a) {
    internal::check(a.rows() == a.cols(), "LDLT of a non-square matrix");
    m_ = Mat(a.derived());
    const Index n = m_.rows();
    perm_.assign(static_cast<size_t>(n), 0);
    // only the lower triangle is referenced
    bool ok = true, found_zero_pivot = false;
    std::vector<S> temp(static_cast<size_t>(n), S(0));
    for (Index k = 0; k < n; ++k) {
      // largest remaining |diagonal| moves to position k
      Index big = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(m_(i, i)) > std::abs(m_(big, big))) big = i;
      perm_[static_cast<size_t>(k)] = big;
      if (big != k) {
        for (Index j = 0; j < k; ++j) std::swap(m_(k, j), m_(big, j));       // rows, left part
        for (Index i = big + 1; i < n; ++i) std::swap(m_(i, k), m_(i, big));  // columns, below
        std::swap(m_(k, k), m_(big, big));
        for (Index i = k + 1; i < big; ++i) {  // the band between k and big (lower triangle)
          const S t = m_(i, k);
          m_(i, k) = m_(big, i);
          m_(big, i) = t;
        }
      }
      const Index rs = n - k - 1;
      if (k > 0) {
        for (Index j = 0; j < k; ++j) temp[static_cast<size_t>(j)] = m_(j, j) * m_(k, j);
        S acc = 0;
        for (Index j = 0; j < k; ++j) acc += m_(k, j) * temp[static_cast<size_t>(j)];
        m_(k, k) -= acc;
        for (Index i = k + 1; i < n; ++i) {
          S s = 0;
          for (Index j = 0; j < k; ++j) s += m_(i, j) * temp[static_cast<size_t>(j)];
          m_(i, k) -= s;
        }
      }
      const S akk = m_(k, k);
      const bool pivot_valid = std::abs(akk) > S(0);
      if (k == 0 && !pivot_valid) {  // the whole diagonal is zero
        for (Index j = 0; j < n; ++j) {
          perm_[static_cast<size_t>(j)] = j;
          for (Index i = 0; i < n; ++i) m_(i, j) = S(0);
        }
        info_ = Success;
        return *this;
      }
      if (rs > 0 && pivot_valid) {
        for (Index i = k + 1; i < n; ++i) m_(i, k) /= akk;
      } else if (rs > 0) {
        for (Index i = k + 1; i < n; ++i) ok = ok && (m_(i, k) == S(0));
      }
      if (found_zero_pivot && pivot_valid)
        ok = false;
      else if (!pivot_valid)
        found_zero_pivot = true;
    }
    info_ = ok ? Success : NumericalIssue;
    return *this;
  }

  ComputationInfo info() const { return info_; }
  const Mat& matrixLDLT() const { return m_; }
  Matrix<S, Dynamic, 1> vectorD() const {
    Matrix<S, Dynamic, 1> d(m_.rows());
    for (Index i = 0; i < m_.rows(); ++i) d(i) = m_(i, i);
    return d;
  }

  template <class D, int R, int C>
  Matrix<S, Dynamic, C> solve(const MatBase<D, S, R, C>& b) const {
    const Index n = m_.rows();
    internal::check(b.rows() == n, "LDLT solve size mismatch");
    Matrix<S, Dynamic, C> x(b.derived());
    const Index nc = x.cols();
    for (Index k = 0; k < n; ++k) {  // x = P b
      const Index p = perm_[static_cast<size_t>(k)];
      if (p != k)
        for (Index c = 0; c < nc; ++c) std::swap(x(k, c), x(p, c));
    }
    for (Index c = 0; c < nc; ++c) {
      for (Index i = 0; i < n; ++i) {  // L y = x (unit lower)
        S s = x(i, c);
        for (Index j = 0; j < i; ++j) s -= m_(i, j) * x(j, c);
        x(i, c) = s;
      }
      const S tiny = std::numeric_limits<S>::min();
      for (Index i = 0; i < n; ++i) {  // pseudo-inverse of D
        const S d = m_(i, i);
        x(i, c) = std::abs(d) > tiny ? x(i, c) / d : S(0);
      }
      for (Index i = n - 1; i >= 0; --i) {  // L^T z = y
        S s = x(i, c);
        for (Index j = i + 1; j < n; ++j) s -= m_(j, i) * x(j, c);
        x(i, c) = s;
      }
    }
    for (Index k = n - 1; k >= 0; --k) {  // x = P^T z
      const Index p = perm_[static_cast<size_t>(k)];
      if (p != k)
        for (Index c = 0; c < nc; ++c) std::swap(x(k, c), x(p, c));
    }
    return x;
  }

 private:
  Mat m_;
  std::vector<Index> perm_;
  ComputationInfo info_ = InvalidInput;
};

template <class Derived, class S, int R, int C>
auto MatBase<Derived, S, R, C>::ldlt() const {
  return LDLT<Matrix<S, Dynamic, Dynamic>>(derived());
}

// ---------------------------------------------------------------------------------------------
// typedefs
// ---------------------------------------------------------------------------------------------
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Vector2i = Matrix<int, 2, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Vector2f = Matrix<float, 2, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXi = Matrix<int, Dynamic, 1>;

}  // namespace Eigen
