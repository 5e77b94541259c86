// eigen_subset.hpp -- repo-authored, clean-room minimal subset of the Eigen
// API, written ONLY so the unmodified reference sources
// (/root/reference/proj/src/*.cpp and proj/tests/*.cpp) compile into the CPU
// oracle (oracle/_ref).  TEST INFRASTRUCTURE: nothing in the product path
// links it.
//
// Eigen is absent from this image and its version is unpinned by the
// reference (proj/src/CMakeLists.txt:11).  This subset
// covers exactly the surface the reference uses:
// dynamic and fixed-size double matrices, lvalue block views, Map of
// row-major data, array views, comma initialisers, HouseholderQR and a thin
// SVD standing in for BDCSVD.  Evaluation is eager (no expression
// templates).  The SVD is column-pivot-free Householder QR preconditioning
// followed by one-sided (Hestenes) Jacobi on the small triangular factor:
// backward stable with high relative accuracy, the same accuracy class as
// Eigen's BDCSVD / JacobiSVD (singular values sorted descending, thin U/V).
#ifndef TTDVM_ORACLE_EIGEN_SUBSET_HPP_
#define TTDVM_ORACLE_EIGEN_SUBSET_HPP_

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <initializer_list>
#include <ostream>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1 };
enum DecompositionOptions { ComputeFullU = 4, ComputeThinU = 8, ComputeFullV = 16, ComputeThinV = 32 };
enum UpLoType { Lower = 1, Upper = 2 };

template <class Scalar, int R, int C, int Opt = ColMajor>
class Matrix;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Vector3d = Matrix<double, 3, 1>;
using Vector2d = Matrix<double, 2, 1>;
using Matrix3d = Matrix<double, 3, 3>;

class Block;
class ArrayX;
class CommaInit;
struct DiagonalWrapper;
struct Reverser;

// ---------------------------------------------------------------- views
// Shallow strided view: element (i, j) at d_[i * rs_ + j * cs_].  Every
// dense type derives from it, so the free operators below accept them all.
class DenseView {
 public:
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() const { return d_; }

  double& operator()(Index i, Index j) const { return d_[i * rs_ + j * cs_]; }
  // linear access: vectors by position, matrices column-major
  double& operator()(Index i) const {
    if (c_ == 1) return d_[i * rs_];
    if (r_ == 1) return d_[i * cs_];
    return (*this)(i % r_, i / r_);
  }
  double& operator[](Index i) const { return (*this)(i); }
  double& coeffRef(Index i, Index j) const { return (*this)(i, j); }
  double coeff(Index i, Index j) const { return (*this)(i, j); }
  double x() const { return (*this)(0); }
  double y() const { return (*this)(1); }
  double z() const { return (*this)(2); }

  // lvalue sub-views
  Block block(Index i, Index j, Index r, Index c) const;
  Block row(Index i) const;
  Block col(Index j) const;
  Block leftCols(Index n) const;
  Block rightCols(Index n) const;
  Block middleCols(Index j, Index n) const;
  Block topRows(Index n) const;
  Block bottomRows(Index n) const;
  Block middleRows(Index i, Index n) const;
  Block head(Index n) const;
  Block tail(Index n) const;
  Block segment(Index i, Index n) const;
  Block topLeftCorner(Index r, Index c) const;
  Block topRightCorner(Index r, Index c) const;
  Block bottomLeftCorner(Index r, Index c) const;
  Block bottomRightCorner(Index r, Index c) const;
  Block transpose() const;

  // reductions
  double squaredNorm() const {
    double s = 0.0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += (*this)(i, j) * (*this)(i, j);
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double sum() const {
    double s = 0.0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += (*this)(i, j);
    return s;
  }
  double prod() const {
    double s = 1.0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s *= (*this)(i, j);
    return s;
  }
  double maxCoeff() const {
    double m = -INFINITY;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) m = std::max(m, (*this)(i, j));
    return m;
  }
  double minCoeff() const {
    double m = INFINITY;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) m = std::min(m, (*this)(i, j));
    return m;
  }
  double trace() const {
    double s = 0.0;
    for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
    return s;
  }
  double dot(const DenseView& o) const {
    double s = 0.0;
    for (Index i = 0; i < size(); ++i) s += (*this)(i) * o(i);
    return s;
  }
  bool allFinite() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i)
        if (!std::isfinite((*this)(i, j))) return false;
    return true;
  }

  // eager element-wise results
  MatrixXd eval() const;
  MatrixXd normalized() const;
  MatrixXd cwiseProduct(const DenseView& o) const;
  MatrixXd cwiseQuotient(const DenseView& o) const;
  MatrixXd cwiseAbs() const;
  MatrixXd cross(const DenseView& o) const;
  ArrayX array() const;
  DiagonalWrapper asDiagonal() const;
  template <int UpLo>
  MatrixXd triangularView() const;
  Reverser colwise() const;
  Reverser rowwise() const;
  void normalize() const;

  // in-place through the view
  const DenseView& operator*=(double s) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) *= s;
    return *this;
  }
  const DenseView& operator/=(double s) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) /= s;
    return *this;
  }
  const DenseView& operator+=(const DenseView& o) const;
  const DenseView& operator-=(const DenseView& o) const;
  void setZero() const { fill(0.0); }
  void setOnes() const { fill(1.0); }
  void setConstant(double v) const { fill(v); }
  void fill(double v) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) = v;
  }

  // a 1 x 1 product reads as its scalar (reference: tt_tensor.cpp:90,203)
  operator double() const {
    if (r_ != 1 || c_ != 1) throw std::logic_error("Eigen subset: non-1x1 matrix used as scalar");
    return d_[0];
  }

 protected:
  DenseView() = default;
  DenseView(double* d, Index r, Index c, Index rs, Index cs) : d_(d), r_(r), c_(c), rs_(rs), cs_(cs) {}
  DenseView(const DenseView&) = default;
  DenseView& operator=(const DenseView&) = default;
  void write_from(const DenseView& src) const;  // alias-safe element copy

  double* d_ = nullptr;
  Index r_ = 0, c_ = 0, rs_ = 1, cs_ = 0;
  friend class Block;
};

// Writable sub-view (block, row, column, transpose): assignment copies the
// elements through it.
class Block : public DenseView {
 public:
  Block(double* d, Index r, Index c, Index rs, Index cs) : DenseView(d, r, c, rs, cs) {}
  Block(const Block&) = default;
  const Block& operator=(const Block& o) const {
    write_from(o);
    return *this;
  }
  const Block& operator=(const DenseView& o) const {
    write_from(o);
    return *this;
  }
  const Block& operator=(const ArrayX& a) const;
};

// Map of external (optionally row-major) storage.
template <class M>
class Map : public DenseView {
 public:
  Map(const double* p, Index r, Index c)
      : DenseView(const_cast<double*>(p), r, c, M::kRowMajor ? c : 1, M::kRowMajor ? 1 : r) {}
  Map(const double* p, Index n) : DenseView(const_cast<double*>(p), n, 1, 1, n) {}
};

// ----------------------------------------------------------- owning matrix
template <class Scalar, int R, int C, int Opt>
class Matrix : public DenseView {
 public:
  static constexpr bool kRowMajor = (Opt & RowMajor) != 0;

  Matrix() { resize(R == Dynamic ? 0 : R, C == Dynamic ? 0 : C); }
  explicit Matrix(Index n) {
    if (R == 1) resize(1, n);
    else resize(n, 1);
  }
  Matrix(Index r, Index c) { resize(r, c); }
  Matrix(int r, int c) { resize(r, c); }
  Matrix(long r, int c) { resize(r, c); }
  Matrix(int r, long c) { resize(r, c); }
  Matrix(double x, double y, double z) {
    resize(3, 1);
    (*this)(0) = x;
    (*this)(1) = y;
    (*this)(2) = z;
  }
  Matrix(const Matrix& o) { copy_from(o); }
  Matrix(Matrix&& o) noexcept : store_(std::move(o.store_)) {
    set_shape(o.r_, o.c_);
    o.store_.clear();
    o.set_shape(0, 0);
  }
  template <class S2, int R2, int C2, int O2>
  Matrix(const Matrix<S2, R2, C2, O2>& o) { copy_from(o); }
  Matrix(const DenseView& o) { copy_from(o); }  // NOLINT: implicit, as Eigen
  Matrix(const ArrayX& a);                      // NOLINT
  Matrix(const DiagonalWrapper& d);             // NOLINT

  Matrix& operator=(const Matrix& o) {
    if (this != &o) copy_from(o);
    return *this;
  }
  Matrix& operator=(Matrix&& o) noexcept {
    store_ = std::move(o.store_);
    set_shape(o.r_, o.c_);
    o.store_.clear();
    o.set_shape(0, 0);
    return *this;
  }
  Matrix& operator=(const DenseView& o) {
    copy_from(o);
    return *this;
  }
  Matrix& operator=(const ArrayX& a);

  void resize(Index r, Index c) {
    if (r < 0 || c < 0) throw std::invalid_argument("Eigen subset: negative size");
    store_.assign((size_t)(r * c), 0.0);
    set_shape(r, c);
  }
  void resize(Index n) {
    if (R == 1) resize(1, n);
    else resize(n, 1);
  }
  void conservativeResize(Index r, Index c) {
    Matrix t(r, c);
    for (Index j = 0; j < std::min(c, c_); ++j)
      for (Index i = 0; i < std::min(r, r_); ++i) t(i, j) = (*this)(i, j);
    *this = std::move(t);
  }

  CommaInit operator<<(const DenseView& first);
  CommaInit operator<<(double first);

  static Matrix Zero() { return Constant(0.0); }
  static Matrix Zero(Index n) { return Constant(n, 0.0); }
  static Matrix Zero(Index r, Index c) { return Constant(r, c, 0.0); }
  static Matrix Ones() { return Constant(1.0); }
  static Matrix Ones(Index n) { return Constant(n, 1.0); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Constant(double v) {
    Matrix m;
    m.fill(v);
    return m;
  }
  static Matrix Constant(Index n, double v) {
    Matrix m(n);
    m.fill(v);
    return m;
  }
  static Matrix Constant(Index r, Index c, double v) {
    Matrix m(r, c);
    m.fill(v);
    return m;
  }
  static Matrix Identity() { return Identity(R, C); }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  // uniform on [-1, 1] from std::rand (values only feed tests that accept
  // any such draw, proj/tests/test_tt_tensor.cpp:208-210)
  static Matrix Random(Index n) {
    Matrix m(n);
    for (Index i = 0; i < n; ++i) m(i) = -1.0 + 2.0 * (double)std::rand() / RAND_MAX;
    return m;
  }
  static Matrix Random(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < r * c; ++i) m.d_[i] = -1.0 + 2.0 * (double)std::rand() / RAND_MAX;
    return m;
  }
  static Matrix UnitX() { return Matrix(1.0, 0.0, 0.0); }
  static Matrix UnitY() { return Matrix(0.0, 1.0, 0.0); }
  static Matrix UnitZ() { return Matrix(0.0, 0.0, 1.0); }

 private:
  void set_shape(Index r, Index c) {
    r_ = r;
    c_ = c;
    rs_ = 1;
    cs_ = r;
    d_ = store_.empty() ? nullptr : store_.data();
  }
  void copy_from(const DenseView& o) {
    std::vector<double> s((size_t)(o.rows() * o.cols()));
    for (Index j = 0; j < o.cols(); ++j)
      for (Index i = 0; i < o.rows(); ++i) s[(size_t)(i + o.rows() * j)] = o(i, j);
    store_ = std::move(s);
    set_shape(o.rows(), o.cols());
  }
  std::vector<double> store_;
};

// ------------------------------------------------------------- arrays
// Element-wise view of a matrix (matrix.array()): owns an eager copy.
class ArrayX {
 public:
  explicit ArrayX(const DenseView& m) : m_(m) {}
  explicit ArrayX(MatrixXd&& m) : m_(std::move(m)) {}
  const MatrixXd& matrix() const { return m_; }
  Index size() const { return m_.size(); }
  Index rows() const { return m_.rows(); }
  Index cols() const { return m_.cols(); }
  double operator()(Index i) const { return m_(i); }
  double operator()(Index i, Index j) const { return m_(i, j); }
  template <class F>
  ArrayX map(F f) const {
    MatrixXd r = m_;
    for (Index i = 0; i < r.size(); ++i) r.data()[i] = f(r.data()[i]);
    return ArrayX(std::move(r));
  }
  template <class F>
  ArrayX zip(const ArrayX& o, F f) const {
    if (o.rows() != rows() || o.cols() != cols()) throw std::invalid_argument("array size mismatch");
    MatrixXd r = m_;
    for (Index i = 0; i < r.size(); ++i) r.data()[i] = f(r.data()[i], o.m_.data()[i]);
    return ArrayX(std::move(r));
  }
  ArrayX abs() const { return map([](double x) { return std::abs(x); }); }
  ArrayX sqrt() const { return map([](double x) { return std::sqrt(x); }); }
  ArrayX exp() const { return map([](double x) { return std::exp(x); }); }
  ArrayX square() const { return map([](double x) { return x * x; }); }
  ArrayX inverse() const { return map([](double x) { return 1.0 / x; }); }
  double sum() const { return m_.sum(); }
  double maxCoeff() const { return m_.maxCoeff(); }
  double minCoeff() const { return m_.minCoeff(); }
  // comparisons -> mask with any() / all() / count()
  struct Mask {
    std::vector<bool> v;
    bool any() const { return std::find(v.begin(), v.end(), true) != v.end(); }
    bool all() const { return std::find(v.begin(), v.end(), false) == v.end(); }
    Index count() const { return (Index)std::count(v.begin(), v.end(), true); }
  };
  template <class F>
  Mask test(F f) const {
    Mask k;
    for (Index i = 0; i < m_.size(); ++i) k.v.push_back(f(m_.data()[i]));
    return k;
  }

 private:
  MatrixXd m_;
};

inline ArrayX operator+(const ArrayX& a, double s) { return a.map([s](double x) { return x + s; }); }
inline ArrayX operator+(double s, const ArrayX& a) { return a + s; }
inline ArrayX operator-(const ArrayX& a, double s) { return a.map([s](double x) { return x - s; }); }
inline ArrayX operator-(double s, const ArrayX& a) { return a.map([s](double x) { return s - x; }); }
inline ArrayX operator*(const ArrayX& a, double s) { return a.map([s](double x) { return x * s; }); }
inline ArrayX operator*(double s, const ArrayX& a) { return a * s; }
inline ArrayX operator/(const ArrayX& a, double s) { return a.map([s](double x) { return x / s; }); }
inline ArrayX operator/(double s, const ArrayX& a) { return a.map([s](double x) { return s / x; }); }
inline ArrayX operator-(const ArrayX& a) { return a.map([](double x) { return -x; }); }
inline ArrayX operator+(const ArrayX& a, const ArrayX& b) { return a.zip(b, [](double x, double y) { return x + y; }); }
inline ArrayX operator-(const ArrayX& a, const ArrayX& b) { return a.zip(b, [](double x, double y) { return x - y; }); }
inline ArrayX operator*(const ArrayX& a, const ArrayX& b) { return a.zip(b, [](double x, double y) { return x * y; }); }
inline ArrayX operator/(const ArrayX& a, const ArrayX& b) { return a.zip(b, [](double x, double y) { return x / y; }); }
inline ArrayX::Mask operator<=(const ArrayX& a, double s) { return a.test([s](double x) { return x <= s; }); }
inline ArrayX::Mask operator<(const ArrayX& a, double s) { return a.test([s](double x) { return x < s; }); }
inline ArrayX::Mask operator>=(const ArrayX& a, double s) { return a.test([s](double x) { return x >= s; }); }
inline ArrayX::Mask operator>(const ArrayX& a, double s) { return a.test([s](double x) { return x > s; }); }
inline ArrayX abs(const ArrayX& a) { return a.abs(); }
inline ArrayX sqrt(const ArrayX& a) { return a.sqrt(); }
inline ArrayX exp(const ArrayX& a) { return a.exp(); }

template <class S, int R, int C, int O>
Matrix<S, R, C, O>::Matrix(const ArrayX& a) {
  copy_from(a.matrix());
}
template <class S, int R, int C, int O>
Matrix<S, R, C, O>& Matrix<S, R, C, O>::operator=(const ArrayX& a) {
  copy_from(a.matrix());
  return *this;
}
inline const Block& Block::operator=(const ArrayX& a) const {
  write_from(a.matrix());
  return *this;
}

// -------------------------------------------------- diagonal / reversal
struct DiagonalWrapper {
  VectorXd d;
};
template <class S, int R, int C, int O>
Matrix<S, R, C, O>::Matrix(const DiagonalWrapper& w) {
  const Index n = w.d.size();
  resize(n, n);
  for (Index i = 0; i < n; ++i) (*this)(i, i) = w.d(i);
}

struct Reverser {
  const DenseView* m;
  bool colwise;  // colwise().reverse() flips each column (row order)
  MatrixXd reverse() const;
  MatrixXd sum() const;
};

// ------------------------------------------------------ comma initialiser
class CommaInit {
 public:
  explicit CommaInit(DenseView& m) : m_(m) {}
  CommaInit& operator,(const DenseView& x) {
    place(x);
    return *this;
  }
  CommaInit& operator,(double v) {
    MatrixXd t(1, 1);
    t(0, 0) = v;
    place(t);
    return *this;
  }
  void place(const DenseView& x) {
    if (col_ == m_.cols()) {
      row_ += blk_;
      col_ = 0;
      blk_ = 0;
    }
    if (row_ + x.rows() > m_.rows() || col_ + x.cols() > m_.cols())
      throw std::logic_error("Eigen subset: comma initialiser overflows the matrix");
    for (Index j = 0; j < x.cols(); ++j)
      for (Index i = 0; i < x.rows(); ++i) m_(row_ + i, col_ + j) = x(i, j);
    col_ += x.cols();
    blk_ = x.rows();
  }

 private:
  DenseView& m_;
  Index row_ = 0, col_ = 0, blk_ = 0;
};

template <class S, int R, int C, int O>
CommaInit Matrix<S, R, C, O>::operator<<(const DenseView& first) {
  CommaInit ci(*this);
  ci.place(first);
  return ci;
}
template <class S, int R, int C, int O>
CommaInit Matrix<S, R, C, O>::operator<<(double first) {
  CommaInit ci(*this);
  ci, first;
  return ci;
}

// --------------------------------------------------- DenseView out-of-line
inline void DenseView::write_from(const DenseView& src) const {
  if (src.rows() != r_ || src.cols() != c_)
    throw std::logic_error("Eigen subset: block assignment size mismatch");
  MatrixXd tmp(src);  // alias-safe
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = tmp(i, j);
}
inline Block DenseView::block(Index i, Index j, Index r, Index c) const {
  if (i < 0 || j < 0 || r < 0 || c < 0 || i + r > r_ || j + c > c_)
    throw std::out_of_range("Eigen subset: block out of range");
  return Block(d_ + i * rs_ + j * cs_, r, c, rs_, cs_);
}
inline Block DenseView::row(Index i) const { return block(i, 0, 1, c_); }
inline Block DenseView::col(Index j) const { return block(0, j, r_, 1); }
inline Block DenseView::leftCols(Index n) const { return block(0, 0, r_, n); }
inline Block DenseView::rightCols(Index n) const { return block(0, c_ - n, r_, n); }
inline Block DenseView::middleCols(Index j, Index n) const { return block(0, j, r_, n); }
inline Block DenseView::topRows(Index n) const { return block(0, 0, n, c_); }
inline Block DenseView::bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
inline Block DenseView::middleRows(Index i, Index n) const { return block(i, 0, n, c_); }
inline Block DenseView::head(Index n) const { return c_ == 1 ? block(0, 0, n, 1) : block(0, 0, 1, n); }
inline Block DenseView::tail(Index n) const {
  return c_ == 1 ? block(r_ - n, 0, n, 1) : block(0, c_ - n, 1, n);
}
inline Block DenseView::segment(Index i, Index n) const {
  return c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n);
}
inline Block DenseView::topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
inline Block DenseView::topRightCorner(Index r, Index c) const { return block(0, c_ - c, r, c); }
inline Block DenseView::bottomLeftCorner(Index r, Index c) const { return block(r_ - r, 0, r, c); }
inline Block DenseView::bottomRightCorner(Index r, Index c) const {
  return block(r_ - r, c_ - c, r, c);
}
inline Block DenseView::transpose() const { return Block(d_, c_, r_, cs_, rs_); }

inline MatrixXd DenseView::eval() const { return MatrixXd(*this); }
inline MatrixXd DenseView::normalized() const {
  MatrixXd m(*this);
  const double nn = norm();
  if (nn > 0.0) m /= nn;
  return m;
}
inline void DenseView::normalize() const {
  const double nn = norm();
  if (nn > 0.0) *this /= nn;
}
inline MatrixXd DenseView::cwiseProduct(const DenseView& o) const {
  if (o.rows() != r_ || o.cols() != c_) throw std::invalid_argument("cwiseProduct size mismatch");
  MatrixXd m(*this);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) *= o(i, j);
  return m;
}
inline MatrixXd DenseView::cwiseQuotient(const DenseView& o) const {
  MatrixXd m(*this);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) /= o(i, j);
  return m;
}
inline MatrixXd DenseView::cwiseAbs() const {
  MatrixXd m(*this);
  for (Index i = 0; i < m.size(); ++i) m.data()[i] = std::abs(m.data()[i]);
  return m;
}
inline MatrixXd DenseView::cross(const DenseView& o) const {
  const DenseView& a = *this;
  MatrixXd m(3, 1);
  m(0) = a(1) * o(2) - a(2) * o(1);
  m(1) = a(2) * o(0) - a(0) * o(2);
  m(2) = a(0) * o(1) - a(1) * o(0);
  return m;
}
inline ArrayX DenseView::array() const { return ArrayX(*this); }
inline DiagonalWrapper DenseView::asDiagonal() const { return DiagonalWrapper{VectorXd(*this)}; }
template <int UpLo>
MatrixXd DenseView::triangularView() const {
  MatrixXd m(*this);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i)
      if ((UpLo == Upper && i > j) || (UpLo == Lower && i < j)) m(i, j) = 0.0;
  return m;
}
inline Reverser DenseView::colwise() const { return Reverser{this, true}; }
inline Reverser DenseView::rowwise() const { return Reverser{this, false}; }
inline MatrixXd Reverser::reverse() const {
  const Index r = m->rows(), c = m->cols();
  MatrixXd out(r, c);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) out(i, j) = colwise ? (*m)(r - 1 - i, j) : (*m)(i, c - 1 - j);
  return out;
}
inline MatrixXd Reverser::sum() const {
  const Index r = m->rows(), c = m->cols();
  MatrixXd out = colwise ? MatrixXd::Zero(1, c) : MatrixXd::Zero(r, 1);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) (colwise ? out(0, j) : out(i, 0)) += (*m)(i, j);
  return out;
}
inline const DenseView& DenseView::operator+=(const DenseView& o) const {
  if (o.rows() != r_ || o.cols() != c_) throw std::invalid_argument("Eigen subset: += size mismatch");
  MatrixXd t(o);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) += t(i, j);
  return *this;
}
inline const DenseView& DenseView::operator-=(const DenseView& o) const {
  if (o.rows() != r_ || o.cols() != c_) throw std::invalid_argument("Eigen subset: -= size mismatch");
  MatrixXd t(o);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) -= t(i, j);
  return *this;
}

// ------------------------------------------------------ free operators
inline MatrixXd operator*(const DenseView& a, const DenseView& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("Eigen subset: product size mismatch");
  const Index m = a.rows(), k = a.cols(), n = b.cols();
  MatrixXd A(a), B(b), C = MatrixXd::Zero(m, n);  // packed column-major operands
  const double* pa = A.data();
  const double* pb = B.data();
  double* pc = C.data();
  for (Index j = 0; j < n; ++j)
    for (Index l = 0; l < k; ++l) {
      const double s = pb[l + k * j];
      const double* ac = pa + m * l;
      double* cc = pc + m * j;
      for (Index i = 0; i < m; ++i) cc[i] += ac[i] * s;
    }
  return C;
}
inline MatrixXd operator*(double s, const DenseView& a) {
  MatrixXd m(a);
  m *= s;
  return m;
}
inline MatrixXd operator*(const DenseView& a, double s) { return s * a; }
inline MatrixXd operator/(const DenseView& a, double s) {
  MatrixXd m(a);
  m /= s;
  return m;
}
inline MatrixXd operator+(const DenseView& a, const DenseView& b) {
  MatrixXd m(a);
  m += b;
  return m;
}
inline MatrixXd operator-(const DenseView& a, const DenseView& b) {
  MatrixXd m(a);
  m -= b;
  return m;
}
inline MatrixXd operator-(const DenseView& a) { return -1.0 * a; }
inline MatrixXd operator*(const DiagonalWrapper& d, const DenseView& a) {
  MatrixXd m(a);
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) m(i, j) *= d.d(i);
  return m;
}
inline MatrixXd operator*(const DenseView& a, const DiagonalWrapper& d) {
  MatrixXd m(a);
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) m(i, j) *= d.d(j);
  return m;
}
inline bool operator==(const DenseView& a, const DenseView& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (a(i, j) != b(i, j)) return false;
  return true;
}
inline bool operator!=(const DenseView& a, const DenseView& b) { return !(a == b); }
inline std::ostream& operator<<(std::ostream& os, const DenseView& a) {
  for (Index i = 0; i < a.rows(); ++i) {
    for (Index j = 0; j < a.cols(); ++j) os << (j ? " " : "") << a(i, j);
    os << "\n";
  }
  return os;
}

// ------------------------------------------------------ decompositions
namespace detail {

// LAPACK dlarfg-style reflector of x (length m, stride 1): on return x[0]
// = beta, x[1..] = v tail (v[0] = 1 implicit), tau; H = I - tau v v^T maps
// x to beta e1.
inline double make_householder(double* x, Index m) {
  double s = 0.0;
  for (Index i = 1; i < m; ++i) s += x[i] * x[i];
  const double alpha = x[0];
  if (s == 0.0) return 0.0;  // already of the form beta e1 (H = I)
  const double nrm = std::sqrt(alpha * alpha + s);
  const double beta = alpha >= 0.0 ? -nrm : nrm;
  const double tau = (beta - alpha) / beta;
  const double scal = 1.0 / (alpha - beta);
  for (Index i = 1; i < m; ++i) x[i] *= scal;
  x[0] = beta;
  return tau;
}

// Householder QR in place on a column-major m x n matrix (lda = m).
inline void householder_qr(double* a, Index m, Index n, std::vector<double>& tau) {
  const Index k = std::min(m, n);
  tau.assign((size_t)k, 0.0);
  for (Index j = 0; j < k; ++j) {
    double* cj = a + j + m * j;
    const double t = make_householder(cj, m - j);
    tau[(size_t)j] = t;
    if (t == 0.0) continue;
    for (Index l = j + 1; l < n; ++l) {
      double* cl = a + j + m * l;
      double w = cl[0];
      for (Index i = 1; i < m - j; ++i) w += cj[i] * cl[i];
      w *= t;
      cl[0] -= w;
      for (Index i = 1; i < m - j; ++i) cl[i] -= w * cj[i];
    }
  }
}

// Apply Q = H_0 H_1 ... H_{k-1} (reflectors below the diagonal of qr,
// m x k) to the columns of x (m x c, column-major) in place.
inline void apply_q(const double* qr, Index m, Index k, const std::vector<double>& tau, double* x,
                    Index c) {
  for (Index j = k - 1; j >= 0; --j) {
    const double t = tau[(size_t)j];
    if (t == 0.0) continue;
    const double* v = qr + j + m * j;
    for (Index l = 0; l < c; ++l) {
      double* xl = x + j + m * l;
      double w = xl[0];
      for (Index i = 1; i < m - j; ++i) w += v[i] * xl[i];
      w *= t;
      xl[0] -= w;
      for (Index i = 1; i < m - j; ++i) xl[i] -= w * v[i];
    }
  }
}

// One-sided Jacobi SVD of a column-major m x n matrix with m >= n:
// a (in) -> u (m x n, orthonormal columns), sigma (n, descending), v (n x n).
inline void jacobi_svd(std::vector<double>& a, Index m, Index n, std::vector<double>& sigma,
                       std::vector<double>& v) {
  v.assign((size_t)(n * n), 0.0);
  for (Index i = 0; i < n; ++i) v[(size_t)(i + n * i)] = 1.0;
  const double tol = 4.0 * 2.220446049250313e-16;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double* ap = a.data() + m * p;
        double* aq = a.data() + m * q;
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (Index i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha) * std::sqrt(beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (Index i = 0; i < m; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        double* vp = v.data() + n * p;
        double* vq = v.data() + n * q;
        for (Index i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
    if (!rotated) break;
  }
  sigma.assign((size_t)n, 0.0);
  for (Index j = 0; j < n; ++j) {
    double s = 0.0;
    for (Index i = 0; i < m; ++i) s += a[(size_t)(i + m * j)] * a[(size_t)(i + m * j)];
    sigma[(size_t)j] = std::sqrt(s);
  }
  // sort descending (stable), permuting the columns of a and v
  std::vector<Index> ord((size_t)n);
  for (Index j = 0; j < n; ++j) ord[(size_t)j] = j;
  std::stable_sort(ord.begin(), ord.end(),
                   [&](Index x, Index y) { return sigma[(size_t)x] > sigma[(size_t)y]; });
  std::vector<double> a2((size_t)(m * n)), v2((size_t)(n * n)), s2((size_t)n);
  for (Index j = 0; j < n; ++j) {
    const Index o = ord[(size_t)j];
    s2[(size_t)j] = sigma[(size_t)o];
    for (Index i = 0; i < m; ++i) a2[(size_t)(i + m * j)] = a[(size_t)(i + m * o)];
    for (Index i = 0; i < n; ++i) v2[(size_t)(i + n * j)] = v[(size_t)(i + n * o)];
  }
  sigma = std::move(s2);
  v = std::move(v2);
  // normalise the left vectors; complete null directions to an orthonormal set
  const double smax = n ? sigma[0] : 0.0;
  for (Index j = 0; j < n; ++j) {
    double* u = a2.data() + m * j;
    if (sigma[(size_t)j] > smax * 1e-300 && sigma[(size_t)j] > 0.0) {
      for (Index i = 0; i < m; ++i) u[i] /= sigma[(size_t)j];
      continue;
    }
    for (Index e = 0; e < m; ++e) {  // first unit vector independent of the previous columns
      for (Index i = 0; i < m; ++i) u[i] = i == e ? 1.0 : 0.0;
      for (int pass = 0; pass < 2; ++pass)
        for (Index l = 0; l < j; ++l) {
          const double* w = a2.data() + m * l;
          double d = 0.0;
          for (Index i = 0; i < m; ++i) d += w[i] * u[i];
          for (Index i = 0; i < m; ++i) u[i] -= d * w[i];
        }
      double nn = 0.0;
      for (Index i = 0; i < m; ++i) nn += u[i] * u[i];
      if (nn > 0.25) {
        nn = std::sqrt(nn);
        for (Index i = 0; i < m; ++i) u[i] /= nn;
        break;
      }
    }
  }
  a = std::move(a2);
}

// Thin SVD of a column-major m x n matrix (m >= n): QR preconditioning
// (A = Q R, Jacobi on the n x n R, U = Q U_R) when m > n.
inline void thin_svd_tall(const MatrixXd& a, MatrixXd& u, VectorXd& s, MatrixXd& vout) {
  const Index m = a.rows(), n = a.cols();
  std::vector<double> sig, v;
  if (m > n) {
    std::vector<double> qr(a.data(), a.data() + m * n), tau;
    householder_qr(qr.data(), m, n, tau);
    std::vector<double> r((size_t)(n * n), 0.0);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i <= j; ++i) r[(size_t)(i + n * j)] = qr[(size_t)(i + m * j)];
    jacobi_svd(r, n, n, sig, v);  // r now holds U_R (n x n)
    std::vector<double> big((size_t)(m * n), 0.0);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) big[(size_t)(i + m * j)] = r[(size_t)(i + n * j)];
    apply_q(qr.data(), m, n, tau, big.data(), n);
    u.resize(m, n);
    std::copy(big.begin(), big.end(), u.data());
  } else {
    std::vector<double> w(a.data(), a.data() + m * n);
    jacobi_svd(w, m, n, sig, v);
    u.resize(m, n);
    std::copy(w.begin(), w.end(), u.data());
  }
  s.resize(n);
  for (Index i = 0; i < n; ++i) s(i) = sig[(size_t)i];
  vout.resize(n, n);
  std::copy(v.begin(), v.end(), vout.data());
}

}  // namespace detail

template <class M>
class HouseholderQR;

// Q of a Householder QR, applied as a product (householderQ() * X).
class HouseholderSequence {
 public:
  HouseholderSequence(const MatrixXd* qr, const std::vector<double>* tau) : qr_(qr), tau_(tau) {}
  friend MatrixXd operator*(const HouseholderSequence& h, const DenseView& x) {
    const Index m = h.qr_->rows();
    if (x.rows() != m) throw std::invalid_argument("householderQ product size mismatch");
    MatrixXd y(x);
    detail::apply_q(h.qr_->data(), m, (Index)h.tau_->size(), *h.tau_, y.data(), y.cols());
    return y;
  }
  operator MatrixXd() const { return *this * MatrixXd::Identity(qr_->rows(), qr_->rows()); }

 private:
  const MatrixXd* qr_;
  const std::vector<double>* tau_;
};

template <class M>
class HouseholderQR {
 public:
  HouseholderQR() = default;
  explicit HouseholderQR(const DenseView& a) { compute(a); }
  HouseholderQR& compute(const DenseView& a) {
    qr_ = MatrixXd(a);
    detail::householder_qr(qr_.data(), qr_.rows(), qr_.cols(), tau_);
    return *this;
  }
  const MatrixXd& matrixQR() const { return qr_; }
  HouseholderSequence householderQ() const { return HouseholderSequence(&qr_, &tau_); }

 private:
  MatrixXd qr_;
  std::vector<double> tau_;
};

// Thin SVD with U, V (BDCSVD / JacobiSVD stand-in; see file header).
template <class M>
class BDCSVD {
 public:
  BDCSVD() = default;
  BDCSVD(const DenseView& a, unsigned int options = 0) { compute(a, options); }
  BDCSVD& compute(const DenseView& a, unsigned int options = 0) {
    (void)options;  // always thin U and V
    MatrixXd m(a);
    if (!m.allFinite()) throw std::invalid_argument("Eigen subset SVD: non-finite input");
    if (m.rows() >= m.cols()) {
      detail::thin_svd_tall(m, u_, s_, v_);
    } else {
      MatrixXd t = m.transpose();
      detail::thin_svd_tall(t, v_, s_, u_);
    }
    return *this;
  }
  const MatrixXd& matrixU() const { return u_; }
  const MatrixXd& matrixV() const { return v_; }
  const VectorXd& singularValues() const { return s_; }

 private:
  MatrixXd u_, v_;
  VectorXd s_;
};
template <class M>
using JacobiSVD = BDCSVD<M>;

}  // namespace Eigen

#endif  // TTDVM_ORACLE_EIGEN_SUBSET_HPP_
