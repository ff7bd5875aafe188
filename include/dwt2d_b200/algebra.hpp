// Symbolic polyphase algebra of the B200 DWT (host side).
//
// Drop-in for the reference's coefficient / Laurent-polynomial / polynomial
// matrix layer (reference: proj/include/dwt2d/coeff.hpp:13-46,
// laurent.hpp:14-82, polymatrix.hpp:11-41). Same public names, argument
// meanings and error behaviour; the implementation is independent.
//
// A term key (m, n) stands for c * zm^-m * zn^-n: on the component grid it
// reads the sample m columns right and n rows down of the output position.
#pragma once

#include <compare>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <string>
#include <utility>
#include <vector>

namespace dwt2d_b200 {

// Exact rational (normalised: gcd 1, positive denominator) or binary64 real.
// Rational op rational stays exact with overflow checking; anything touching
// a real is computed in double (coeff.cpp semantics).
class Coeff {
 public:
  constexpr Coeff() = default;
  Coeff(std::int64_t n) : num_(n) {}
  Coeff(int n) : num_(n) {}

  static Coeff ratio(std::int64_t num, std::int64_t den);
  static Coeff real(double v);

  bool is_exact() const { return exact_; }
  bool is_zero() const { return exact_ ? num_ == 0 : dbl_ == 0.0; }
  bool is_one() const { return exact_ ? (num_ == 1 && den_ == 1) : dbl_ == 1.0; }
  std::int64_t num() const;
  std::int64_t den() const;
  double value() const {
    return exact_ ? double(num_) / double(den_) : dbl_;
  }
  std::string str() const;

  friend Coeff operator+(const Coeff& a, const Coeff& b);
  friend Coeff operator-(const Coeff& a, const Coeff& b);
  friend Coeff operator*(const Coeff& a, const Coeff& b);
  friend Coeff operator-(const Coeff& a);
  friend bool operator==(const Coeff& a, const Coeff& b);
  friend bool operator!=(const Coeff& a, const Coeff& b) { return !(a == b); }

 private:
  bool exact_ = true;
  std::int64_t num_ = 0, den_ = 1;
  double dbl_ = 0.0;
};

struct Exponent {
  int m = 0;
  int n = 0;
  auto operator<=>(const Exponent&) const = default;
};

struct Term {
  Exponent e;
  Coeff c;
};

enum class Axis { horizontal, vertical };

// Bivariate Laurent polynomial. Stored as a dense coefficient grid over its
// bounding box — every cell (m, n) of [m0, m0 + w) x [n0, n0 + h) is either
// a term or empty — plus the key-sorted term list of the occupied cells
// (terms()). Zero coefficients are never stored.
class LaurentPoly {
 public:
  LaurentPoly() = default;
  static LaurentPoly constant(Coeff c);
  static LaurentPoly monomial(Coeff c, int m, int n);
  static LaurentPoly univariate(std::initializer_list<std::pair<int, Coeff>> taps);
  static LaurentPoly from_terms(std::vector<Term> terms);

  const std::vector<Term>& terms() const { return t_; }
  Coeff coeff(int m, int n) const;
  std::size_t term_count() const { return t_.size(); }
  bool is_zero() const { return t_.empty(); }
  bool is_constant() const;
  bool is_one() const;
  bool univariate_m() const;
  bool univariate_n() const;

  friend LaurentPoly operator+(const LaurentPoly& a, const LaurentPoly& b);
  friend LaurentPoly operator-(const LaurentPoly& a, const LaurentPoly& b);
  friend LaurentPoly operator*(const LaurentPoly& a, const LaurentPoly& b);
  friend LaurentPoly operator-(const LaurentPoly& a);
  friend bool operator==(const LaurentPoly& a, const LaurentPoly& b);
  friend bool operator!=(const LaurentPoly& a, const LaurentPoly& b) {
    return !(a == b);
  }

 private:
  friend class TermGrid;
  struct Cell {
    bool used = false;
    Coeff c;
  };
  int m0_ = 0, n0_ = 0, w_ = 0, h_ = 0;
  std::vector<Cell> grid_;  // (m - m0) * h + (n - n0): m-major, the key order
  std::vector<Term> t_;     // the occupied cells in grid order
};

LaurentPoly transpose(const LaurentPoly& p);
LaurentPoly embed(const LaurentPoly& p, Axis axis);
std::pair<LaurentPoly, LaurentPoly> split_constant(const LaurentPoly& p);
bool approx_equal(const LaurentPoly& a, const LaurentPoly& b, double tol);
std::string to_string(const LaurentPoly& p);

// Dense 2x2 / 4x4 matrix of polynomials, component order ee, oe, eo, oo.
class PolyMatrix {
 public:
  PolyMatrix() = default;
  PolyMatrix(int rows, int cols);
  static PolyMatrix identity(int n);
  int rows() const { return r_; }
  int cols() const { return c_; }
  LaurentPoly& at(int r, int c) { return cell_[std::size_t(r) * c_ + c]; }
  const LaurentPoly& at(int r, int c) const { return cell_[std::size_t(r) * c_ + c]; }
  bool is_identity() const;
  friend bool operator==(const PolyMatrix& a, const PolyMatrix& b) {
    return a.r_ == b.r_ && a.c_ == b.c_ && a.cell_ == b.cell_;
  }
  friend bool operator!=(const PolyMatrix& a, const PolyMatrix& b) { return !(a == b); }

 private:
  int r_ = 0, c_ = 0;
  std::vector<LaurentPoly> cell_;
};

PolyMatrix mat_mul(const PolyMatrix& a, const PolyMatrix& b);
inline PolyMatrix operator*(const PolyMatrix& a, const PolyMatrix& b) { return mat_mul(a, b); }
bool approx_equal(const PolyMatrix& a, const PolyMatrix& b, double tol);

}  // namespace dwt2d_b200
