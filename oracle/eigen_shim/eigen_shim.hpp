// eigen_shim.hpp — a minimal, from-scratch stand-in for the slice of the Eigen 3 API that the
// reference's hot-path translation units use (/root/reference/proj/src/splat3d.cpp,
// src/image.cpp and the headers they include).  TEST INFRASTRUCTURE ONLY: it exists so that
// oracle/build_ref.sh can compile the reference's own render() here, where Eigen is not
// installed, and pin the CPU oracle against it.
//
// Semantics: fixed-size column-major matrices; products accumulate k = 0, 1, 2, ... in order
// (Eigen's internal summation order for 3-term dot products may differ by one rounding, i.e.
// <= 1 ulp in FP64 — far below every tolerance the tests use).  Decompositions (LLT,
// SelfAdjointEigenSolver) are plain textbook versions; they are only reached by the
// anisotropic path, which is out of scope and never called by the tests.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <initializer_list>

namespace Eigen {

enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };

template <class S, int R, int C>
struct Matrix {
  S a[R * C];

  Matrix() {
    for (auto& x : a) x = S(0);
  }
  Matrix(S x, S y)
    requires(R * C == 2)
  {
    a[0] = x;
    a[1] = y;
  }
  Matrix(S x, S y, S z)
    requires(R * C == 3)
  {
    a[0] = x;
    a[1] = y;
    a[2] = z;
  }

  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  int rows() const { return R; }
  int cols() const { return C; }
  int size() const { return R * C; }

  S& operator()(int i, int j) { return a[j * R + i]; }
  const S& operator()(int i, int j) const { return a[j * R + i]; }
  S& operator[](int i) { return a[i]; }
  const S& operator[](int i) const { return a[i]; }
  S& operator()(int i) { return a[i]; }
  const S& operator()(int i) const { return a[i]; }

  static Matrix Identity() {
    Matrix m;
    for (int i = 0; i < std::min(R, C); ++i) m(i, i) = S(1);
    return m;
  }
  static Matrix Zero() { return Matrix(); }

  Matrix<S, C, R> transpose() const {
    Matrix<S, C, R> t;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  bool allFinite() const {
    for (const auto& x : a)
      if (!std::isfinite(x)) return false;
    return true;
  }
  Matrix cwiseAbs() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.a[i] = std::abs(a[i]);
    return m;
  }
  S maxCoeff() const { return *std::max_element(a, a + R * C); }
  S minCoeff() const { return *std::min_element(a, a + R * C); }
  S sum() const {
    S s = a[0];
    for (int i = 1; i < R * C; ++i) s += a[i];
    return s;
  }
  S squaredNorm() const {
    S s = a[0] * a[0];
    for (int i = 1; i < R * C; ++i) s += a[i] * a[i];
    return s;
  }
  S norm() const { return std::sqrt(squaredNorm()); }
  S dot(const Matrix& o) const {
    S s = a[0] * o.a[0];
    for (int i = 1; i < R * C; ++i) s += a[i] * o.a[i];
    return s;
  }
  Matrix<S, R * C, R * C> asDiagonal() const {
    Matrix<S, R * C, R * C> d;
    for (int i = 0; i < R * C; ++i) d(i, i) = a[i];
    return d;
  }
  Matrix inverse() const
    requires(R == 2 && C == 2)
  {
    const S det = a[0] * a[3] - a[2] * a[1];
    Matrix m;
    m(0, 0) = (*this)(1, 1) / det;
    m(0, 1) = -(*this)(0, 1) / det;
    m(1, 0) = -(*this)(1, 0) / det;
    m(1, 1) = (*this)(0, 0) / det;
    return m;
  }

  // comma initializer fills row by row, like Eigen's
  struct CommaInit {
    Matrix& m;
    int k;
    CommaInit& operator,(S v) {
      m(k / C, k % C) = v;
      ++k;
      return *this;
    }
  };
  CommaInit operator<<(S v) {
    (*this)(0, 0) = v;
    return CommaInit{*this, 1};
  }

  Matrix& operator+=(const Matrix& o) {
    for (int i = 0; i < R * C; ++i) a[i] += o.a[i];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (int i = 0; i < R * C; ++i) a[i] -= o.a[i];
    return *this;
  }
  Matrix& operator*=(S s) {
    for (auto& x : a) x *= s;
    return *this;
  }
  Matrix operator-() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.a[i] = -a[i];
    return m;
  }
};

template <class S, int R, int C>
Matrix<S, R, C> operator+(Matrix<S, R, C> x, const Matrix<S, R, C>& y) {
  return x += y;
}
template <class S, int R, int C>
Matrix<S, R, C> operator-(Matrix<S, R, C> x, const Matrix<S, R, C>& y) {
  return x -= y;
}
template <class S, int R, int C>
Matrix<S, R, C> operator*(Matrix<S, R, C> x, S s) {
  return x *= s;
}
template <class S, int R, int C>
Matrix<S, R, C> operator*(S s, Matrix<S, R, C> x) {
  for (auto& v : x.a) v = s * v;
  return x;
}
template <class S, int R, int C>
Matrix<S, R, C> operator/(Matrix<S, R, C> x, S s) {
  for (auto& v : x.a) v /= s;
  return x;
}
template <class S, int R, int K, int C>
Matrix<S, R, C> operator*(const Matrix<S, R, K>& x, const Matrix<S, K, C>& y) {
  Matrix<S, R, C> m;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < C; ++j) {
      S s = x(i, 0) * y(0, j);
      for (int k = 1; k < K; ++k) s += x(i, k) * y(k, j);
      m(i, j) = s;
    }
  return m;
}

using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;

template <class S>
struct Quaternion {
  S w_, x_, y_, z_;
  Quaternion() : w_(1), x_(0), y_(0), z_(0) {}
  Quaternion(S w, S x, S y, S z) : w_(w), x_(x), y_(y), z_(z) {}
  S w() const { return w_; }
  S x() const { return x_; }
  S y() const { return y_; }
  S z() const { return z_; }
  S norm() const { return std::sqrt(w_ * w_ + x_ * x_ + y_ * y_ + z_ * z_); }
  Quaternion normalized() const {
    const S n = norm();
    return Quaternion(w_ / n, x_ / n, y_ / n, z_ / n);
  }
  Matrix<S, 3, 3> toRotationMatrix() const {
    Matrix<S, 3, 3> r;
    const S w = w_, x = x_, y = y_, z = z_;
    r << 1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
        2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
        2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y);
    return r;
  }
};
using Quaterniond = Quaternion<double>;

// Jacobi eigenvalues of a symmetric matrix (aniso path only).
template <class M>
struct SelfAdjointEigenSolver {
  static constexpr int N = M::RowsAtCompileTime;
  Matrix<double, N, 1> ev;
  explicit SelfAdjointEigenSolver(const M& m, int = ComputeEigenvectors) {
    M a = m;
    for (int sweep = 0; sweep < 64; ++sweep) {
      double off = 0;
      for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) off += a(p, q) * a(p, q);
      if (off < 1e-300) break;
      for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) {
          if (a(p, q) == 0) continue;
          const double th = 0.5 * std::atan2(2 * a(p, q), a(q, q) - a(p, p));
          const double c = std::cos(th), s = std::sin(th);
          for (int k = 0; k < N; ++k) {
            const double akp = a(k, p), akq = a(k, q);
            a(k, p) = c * akp - s * akq;
            a(k, q) = s * akp + c * akq;
          }
          for (int k = 0; k < N; ++k) {
            const double apk = a(p, k), aqk = a(q, k);
            a(p, k) = c * apk - s * aqk;
            a(q, k) = s * apk + c * aqk;
          }
        }
    }
    for (int i = 0; i < N; ++i) ev[i] = a(i, i);
    std::sort(ev.a, ev.a + N);
  }
  const Matrix<double, N, 1>& eigenvalues() const { return ev; }
};

// Cholesky solve (aniso path only).
template <class M>
struct LLT {
  static constexpr int N = M::RowsAtCompileTime;
  M l;
  explicit LLT(const M& m) {
    for (int j = 0; j < N; ++j) {
      double d = m(j, j);
      for (int k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
      l(j, j) = std::sqrt(d);
      for (int i = j + 1; i < N; ++i) {
        double s = m(i, j);
        for (int k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
        l(i, j) = s / l(j, j);
      }
    }
  }
  Matrix<double, N, 1> solve(const Matrix<double, N, 1>& b) const {
    Matrix<double, N, 1> y, x;
    for (int i = 0; i < N; ++i) {
      double s = b[i];
      for (int k = 0; k < i; ++k) s -= l(i, k) * y[k];
      y[i] = s / l(i, i);
    }
    for (int i = N - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < N; ++k) s -= l(k, i) * x[k];
      x[i] = s / l(i, i);
    }
    return x;
  }
};

}  // namespace Eigen
