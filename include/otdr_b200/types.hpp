// otdr_b200/types.hpp -- dense row-major fp64 containers of the C++ host API.
//
// Mirrors proj/include/otdr/types.hpp:9-15 (Matrix = row-major dynamic fp64,
// Vector, Index) without Eigen, which this toolchain does not ship: the subset
// the solver API and its callers use (shape, element access, comma
// initialisation, Zero/Constant/Ones, raw data for the C-ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace otdr {

using Index = std::int64_t;

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> xs) : v_(xs) {}
  static Vector Zero(Index n) { return Vector(n); }
  static Vector Constant(Index n, double x) {
    Vector v(n);
    for (auto& e : v.v_) e = x;
    return v;
  }
  static Vector Ones(Index n) { return Constant(n, 1.0); }
  Index size() const { return static_cast<Index>(v_.size()); }
  double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
  double& operator()(Index i) { return (*this)[i]; }
  double operator()(Index i) const { return (*this)[i]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double sum() const {
    double s = 0.0;
    for (double e : v_) s += e;
    return s;
  }
  bool operator==(const Vector& o) const { return v_ == o.v_; }

 private:
  std::vector<double> v_;
};

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols)
      : rows_(rows), cols_(cols), v_(static_cast<std::size_t>(rows * cols), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Constant(Index r, Index c, double x) {
    Matrix m(r, c);
    for (auto& e : m.v_) e = x;
    return m;
  }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i * cols_ + j)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(i * cols_ + j)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  bool operator==(const Matrix& o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && v_ == o.v_;
  }

  // Eigen-style comma initialiser: m << a, b, c, d;
  class CommaInit {
   public:
    CommaInit(Matrix& m, double first) : m_(m) { put(first); }
    CommaInit& operator,(double x) {
      put(x);
      return *this;
    }

   private:
    void put(double x) {
      if (at_ >= m_.v_.size()) throw std::out_of_range("too many coefficients");
      m_.v_[at_++] = x;
    }
    Matrix& m_;
    std::size_t at_ = 0;
  };
  CommaInit operator<<(double first) { return CommaInit(*this, first); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};

using TransportPlan = Matrix;

}  // namespace otdr
