// Host polyphase algebra: exact-or-real coefficients, Laurent polynomials on
// dense coefficient grids, polynomial matrices.
//
// Contract with the reference (proj/src/coeff.cpp, laurent.cpp,
// polymatrix.cpp): the same values, and for real (binary64) coefficients the
// same IEEE operation sequence, because composed tap weights must come out
// bit-identical:
//   * a product of polynomials forms the coefficient products in
//     (term of a) x (term of b) order, both in key order, and sums the ones
//     that land on one key in that arrival order;
//   * a sum of polynomials adds b's coefficient to a's, key by key;
//   * a matrix product accumulates sum_k a(r, k) * b(k, c) left to right.
// Exact rationals are normalised, so any correct exact arithmetic gives the
// reference's values; a rational whose normalised form leaves int64 raises
// std::overflow_error.
#include "dwt2d_b200/algebra.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <stdexcept>

namespace dwt2d_b200 {

// ---------------------------------------------------- polynomial matrices

PolyMatrix::PolyMatrix(int rows, int cols) : r_(rows), c_(cols) {
  if (!(rows > 0 && cols > 0)) throw std::invalid_argument("matrix dimensions must be positive");
  cell_.assign(std::size_t(rows) * std::size_t(cols), LaurentPoly{});
}

PolyMatrix PolyMatrix::identity(int n) {
  PolyMatrix m(n, n);
  const LaurentPoly one = LaurentPoly::constant(Coeff(1));
  for (int i = 0; i < n; ++i) m.at(i, i) = one;
  return m;
}

bool PolyMatrix::is_identity() const {
  if (r_ != c_) return false;
  for (int i = 0; i < r_ * c_; ++i) {
    const bool diagonal = i / c_ == i % c_;
    if (diagonal ? !cell_[std::size_t(i)].is_one() : !cell_[std::size_t(i)].is_zero()) return false;
  }
  return true;
}

// out(r, c) = a(r, 0) b(0, c) + a(r, 1) b(1, c) + ..., summed left to right
PolyMatrix mat_mul(const PolyMatrix& a, const PolyMatrix& b) {
  const int inner = a.cols();
  if (inner != b.rows()) throw std::invalid_argument("mat_mul: dimension mismatch");
  PolyMatrix out(a.rows(), b.cols());
  auto dot = [&](int r, int c) {
    LaurentPoly acc;
    for (int k = 0; k < inner; ++k) acc = acc + a.at(r, k) * b.at(k, c);
    return acc;
  };
  for (int i = 0; i < a.rows() * b.cols(); ++i) out.at(i / b.cols(), i % b.cols()) = dot(i / b.cols(), i % b.cols());
  return out;
}

bool approx_equal(const PolyMatrix& a, const PolyMatrix& b, double tol) {
  const bool same_shape = a.rows() == b.rows() && a.cols() == b.cols();
  int i = 0;
  for (; same_shape && i < a.rows() * a.cols(); ++i)
    if (!approx_equal(a.at(i / a.cols(), i % a.cols()), b.at(i / a.cols(), i % a.cols()), tol)) break;
  return same_shape && i == a.rows() * a.cols();
}

// ---------------------------------------------------- Laurent polynomials

// Accumulates coefficients on a dense grid over a known bounding box: the
// first coefficient that lands on a cell is stored, later ones are added to
// it in arrival order. seal() drops the cells that summed to zero, shrinks
// the box to the occupied cells and lists them in key order.
class TermGrid {
 public:
  TermGrid(int m_lo, int m_hi, int n_lo, int n_hi) {
    p_.m0_ = m_lo, p_.n0_ = n_lo;
    p_.w_ = std::max(0, m_hi - m_lo + 1);
    p_.h_ = std::max(0, n_hi - n_lo + 1);
    p_.grid_.resize(std::size_t(p_.w_) * std::size_t(p_.h_));
  }
  void add(int m, int n, const Coeff& c) {
    LaurentPoly::Cell& cell = p_.grid_[std::size_t(m - p_.m0_) * p_.h_ + std::size_t(n - p_.n0_)];
    if (cell.used) {
      cell.c = cell.c + c;
    } else {
      cell.used = true;
      cell.c = c;
    }
  }
  LaurentPoly seal() {
    int mlo = INT_MAX, mhi = INT_MIN, nlo = INT_MAX, nhi = INT_MIN;
    for (int i = 0; i < p_.w_; ++i)
      for (int j = 0; j < p_.h_; ++j) {
        LaurentPoly::Cell& cell = p_.grid_[std::size_t(i) * p_.h_ + j];
        if (cell.used && cell.c.is_zero()) cell = LaurentPoly::Cell{};
        if (!cell.used) continue;
        mlo = std::min(mlo, i), mhi = std::max(mhi, i), nlo = std::min(nlo, j), nhi = std::max(nhi, j);
      }
    LaurentPoly out;
    if (mlo > mhi) return out;
    out.m0_ = p_.m0_ + mlo, out.n0_ = p_.n0_ + nlo;
    out.w_ = mhi - mlo + 1, out.h_ = nhi - nlo + 1;
    out.grid_.resize(std::size_t(out.w_) * std::size_t(out.h_));
    for (int i = 0; i < out.w_; ++i)
      for (int j = 0; j < out.h_; ++j) {
        const LaurentPoly::Cell& cell = p_.grid_[std::size_t(i + mlo) * p_.h_ + std::size_t(j + nlo)];
        out.grid_[std::size_t(i) * out.h_ + j] = cell;
        if (cell.used) out.t_.push_back(Term{{out.m0_ + i, out.n0_ + j}, cell.c});
      }
    return out;
  }

 private:
  LaurentPoly p_;
};

namespace {

struct Box {
  int m_lo = INT_MAX, m_hi = INT_MIN, n_lo = INT_MAX, n_hi = INT_MIN;
  void cover(int m, int n) {
    m_lo = std::min(m_lo, m), m_hi = std::max(m_hi, m);
    n_lo = std::min(n_lo, n), n_hi = std::max(n_hi, n);
  }
  TermGrid grid() const { return m_lo > m_hi ? TermGrid(0, -1, 0, -1) : TermGrid(m_lo, m_hi, n_lo, n_hi); }
};

}  // namespace

LaurentPoly LaurentPoly::from_terms(std::vector<Term> terms) {
  Box box;
  for (const Term& t : terms) box.cover(t.e.m, t.e.n);
  TermGrid g = box.grid();
  for (const Term& t : terms) g.add(t.e.m, t.e.n, t.c);
  return g.seal();
}

LaurentPoly LaurentPoly::monomial(Coeff c, int m, int n) { return from_terms({Term{{m, n}, c}}); }

LaurentPoly LaurentPoly::constant(Coeff c) { return monomial(c, 0, 0); }

LaurentPoly LaurentPoly::univariate(std::initializer_list<std::pair<int, Coeff>> taps) {
  std::vector<Term> v;
  v.reserve(taps.size());
  for (const auto& tap : taps) v.push_back(Term{{tap.first, 0}, tap.second});
  return from_terms(std::move(v));
}

Coeff LaurentPoly::coeff(int m, int n) const {
  const int i = m - m0_, j = n - n0_;
  if (i < 0 || j < 0 || i >= w_ || j >= h_) return Coeff{};
  const Cell& cell = grid_[std::size_t(i) * h_ + j];
  return cell.used ? cell.c : Coeff{};
}

bool LaurentPoly::is_constant() const { return t_.empty() || (t_.size() == 1 && t_[0].e == Exponent{}); }

bool LaurentPoly::is_one() const { return is_constant() && !t_.empty() && t_[0].c.is_one(); }

bool LaurentPoly::univariate_m() const { return t_.empty() || (n0_ == 0 && h_ == 1); }

bool LaurentPoly::univariate_n() const { return t_.empty() || (m0_ == 0 && w_ == 1); }

LaurentPoly operator+(const LaurentPoly& a, const LaurentPoly& b) {
  Box box;
  for (const LaurentPoly* p : {&a, &b})
    if (!p->t_.empty()) box.cover(p->m0_, p->n0_), box.cover(p->m0_ + p->w_ - 1, p->n0_ + p->h_ - 1);
  TermGrid g = box.grid();
  for (const Term& t : a.t_) g.add(t.e.m, t.e.n, t.c);
  for (const Term& t : b.t_) g.add(t.e.m, t.e.n, t.c);
  return g.seal();
}

LaurentPoly operator-(const LaurentPoly& a) {
  LaurentPoly r = a;
  for (LaurentPoly::Cell& cell : r.grid_)
    if (cell.used) cell.c = -cell.c;
  for (Term& t : r.t_) t.c = -t.c;
  return r;
}

LaurentPoly operator-(const LaurentPoly& a, const LaurentPoly& b) { return a + (-b); }

LaurentPoly operator*(const LaurentPoly& a, const LaurentPoly& b) {
  if (a.t_.empty() || b.t_.empty()) return LaurentPoly{};
  TermGrid g(a.m0_ + b.m0_, a.m0_ + a.w_ + b.m0_ + b.w_ - 2, a.n0_ + b.n0_, a.n0_ + a.h_ + b.n0_ + b.h_ - 2);
  for (const Term& x : a.t_)
    for (const Term& y : b.t_) g.add(x.e.m + y.e.m, x.e.n + y.e.n, x.c * y.c);
  return g.seal();
}

bool operator==(const LaurentPoly& a, const LaurentPoly& b) {
  if (a.t_.size() != b.t_.size()) return false;
  for (std::size_t i = 0; i < a.t_.size(); ++i)
    if (a.t_[i].e != b.t_[i].e || a.t_[i].c != b.t_[i].c) return false;
  return true;
}

LaurentPoly transpose(const LaurentPoly& p) {
  std::vector<Term> swapped;
  swapped.reserve(p.terms().size());
  for (const Term& t : p.terms()) swapped.push_back(Term{{t.e.n, t.e.m}, t.c});
  return LaurentPoly::from_terms(std::move(swapped));
}

LaurentPoly embed(const LaurentPoly& p, Axis axis) {
  const bool horizontal = p.univariate_m();
  if (!horizontal && !p.univariate_n()) throw std::invalid_argument("embed: polynomial is not univariate");
  const bool want_horizontal = axis == Axis::horizontal;
  // the zero polynomial is univariate on both axes: returned as is
  return (horizontal == want_horizontal || p.is_zero()) ? p : transpose(p);
}

std::pair<LaurentPoly, LaurentPoly> split_constant(const LaurentPoly& p) {
  LaurentPoly c0 = LaurentPoly::constant(p.coeff(0, 0));
  LaurentPoly rest = p - c0;
  return {std::move(c0), std::move(rest)};
}

bool approx_equal(const LaurentPoly& a, const LaurentPoly& b, double tol) {
  for (const Term& t : a.terms())
    if (!(std::abs(t.c.value() - b.coeff(t.e.m, t.e.n).value()) <= tol)) return false;
  for (const Term& t : b.terms())
    if (!(std::abs(t.c.value() - a.coeff(t.e.m, t.e.n).value()) <= tol)) return false;
  return true;
}

// Text form (the reference's describe() format): terms in key order,
// "c*zm^k*zn^l" with key m standing for zm^-m, unit magnitudes as the bare
// monomial, a leading "-" or " - " / " + " separators.
std::string to_string(const LaurentPoly& p) {
  if (p.is_zero()) return "0";
  auto var = [](const char* name, int key) {
    std::string v = name;
    if (key != -1) v += "^" + std::to_string(-key);
    return v;
  };
  std::string out;
  bool first = true;
  for (const Term& t : p.terms()) {
    const bool negative = t.c.value() < 0.0;
    const Coeff mag = negative ? -t.c : t.c;
    std::string mono;
    if (t.e.m != 0) mono = var("zm", t.e.m);
    if (t.e.n != 0) mono += (mono.empty() ? "" : "*") + var("zn", t.e.n);
    std::string body;
    if (mono.empty())
      body = mag.str();
    else if (mag.is_one())
      body = mono;
    else
      body = mag.str() + "*" + mono;
    out += first ? (negative ? "-" : "") : (negative ? " - " : " + ");
    out += body;
    first = false;
  }
  return out;
}

// ---------------------------------------------------------- coefficients

namespace {

using i128 = __int128;

i128 magnitude(i128 v) { return v < 0 ? -v : v; }

i128 euclid(i128 a, i128 b) {
  a = magnitude(a), b = magnitude(b);
  while (b != 0) {
    const i128 r = a % b;
    a = b, b = r;
  }
  return a;
}

// the normalised rational n / d (d != 0) as an exact Coeff
Coeff exact_from_wide(i128 n, i128 d) {
  if (d < 0) n = -n, d = -d;
  const i128 g = euclid(n, d);
  if (g > 1) n /= g, d /= g;
  if (n > i128(INT64_MAX) || n < i128(INT64_MIN) || d > i128(INT64_MAX))
    throw std::overflow_error("rational coefficient overflow");
  return Coeff::ratio(std::int64_t(n), std::int64_t(d));
}

}  // namespace

Coeff Coeff::ratio(std::int64_t num, std::int64_t den) {
  if (den == 0) throw std::invalid_argument("rational with zero denominator");
  i128 n = num, d = den;
  if (d < 0) n = -n, d = -d;
  const i128 g = euclid(n, d);
  if (g > 1) n /= g, d /= g;
  Coeff c;
  c.num_ = std::int64_t(n);
  c.den_ = std::int64_t(d);
  return c;
}

Coeff Coeff::real(double v) {
  Coeff c;
  c.exact_ = false;
  c.dbl_ = v;
  return c;
}

std::int64_t Coeff::num() const {
  if (!exact_) throw std::logic_error("num() of a real coefficient");
  return num_;
}

std::int64_t Coeff::den() const {
  if (!exact_) throw std::logic_error("den() of a real coefficient");
  return den_;
}

Coeff operator+(const Coeff& a, const Coeff& b) {
  if (a.exact_ && b.exact_)
    return exact_from_wide(i128(a.num_) * b.den_ + i128(b.num_) * a.den_, i128(a.den_) * b.den_);
  return Coeff::real(a.value() + b.value());
}

Coeff operator*(const Coeff& a, const Coeff& b) {
  if (a.exact_ && b.exact_) return exact_from_wide(i128(a.num_) * b.num_, i128(a.den_) * b.den_);
  return Coeff::real(a.value() * b.value());
}

Coeff operator-(const Coeff& a) { return a.exact_ ? exact_from_wide(-i128(a.num_), a.den_) : Coeff::real(-a.dbl_); }

Coeff operator-(const Coeff& a, const Coeff& b) { return a + (-b); }

bool operator==(const Coeff& a, const Coeff& b) {
  return (a.exact_ && b.exact_) ? (a.num_ == b.num_ && a.den_ == b.den_) : a.value() == b.value();
}

std::string Coeff::str() const {
  char buf[64];
  if (!exact_) {
    std::snprintf(buf, sizeof buf, "%.16g", dbl_);
  } else {
    const int n = std::snprintf(buf, sizeof buf, "%lld", (long long)num_);
    if (den_ != 1) std::snprintf(buf + n, sizeof buf - size_t(n), "/%lld", (long long)den_);
  }
  return buf;
}

}  // namespace dwt2d_b200
