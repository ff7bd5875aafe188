// Host polyphase algebra: exact/real coefficients, sparse Laurent
// polynomials, polynomial matrices. Semantics follow the reference
// (proj/src/coeff.cpp, laurent.cpp, polymatrix.cpp) so that every composed
// double coefficient — and therefore every float tap weight handed to the
// CUDA kernels — is produced by the same sequence of IEEE operations.
#include "dwt2d_b200/algebra.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <numeric>
#include <stdexcept>

namespace dwt2d_b200 {

// ---------------------------------------------------------------- Coeff

namespace {
using wide = __int128;

std::int64_t narrow_or_throw(wide v) {
  if (v > wide(INT64_MAX) || v < wide(INT64_MIN))
    throw std::overflow_error("rational coefficient overflow");
  return std::int64_t(v);
}

wide wide_gcd(wide a, wide b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    const wide t = a % b;
    a = b;
    b = t;
  }
  return a;
}
}  // namespace

Coeff Coeff::ratio(std::int64_t num, std::int64_t den) {
  if (den == 0) throw std::invalid_argument("rational with zero denominator");
  if (den < 0) num = -num, den = -den;
  const std::int64_t g = std::gcd(num < 0 ? -num : num, den);
  Coeff c;
  c.num_ = g > 1 ? num / g : num;
  c.den_ = g > 1 ? den / g : den;
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
  if (!(a.exact_ && b.exact_)) return Coeff::real(a.value() + b.value());
  wide n = wide(a.num_) * b.den_ + wide(b.num_) * a.den_;
  wide d = wide(a.den_) * b.den_;
  if (const wide g = wide_gcd(n, d); g > 1) n /= g, d /= g;
  return Coeff::ratio(narrow_or_throw(n), narrow_or_throw(d));
}

Coeff operator-(const Coeff& a) {
  return a.exact_ ? Coeff::ratio(-a.num_, a.den_) : Coeff::real(-a.dbl_);
}

Coeff operator-(const Coeff& a, const Coeff& b) { return a + (-b); }

Coeff operator*(const Coeff& a, const Coeff& b) {
  if (!(a.exact_ && b.exact_)) return Coeff::real(a.value() * b.value());
  // reduce crosswise first so the products stay small
  const std::int64_t g1 = std::gcd(a.num_ < 0 ? -a.num_ : a.num_, b.den_);
  const std::int64_t g2 = std::gcd(b.num_ < 0 ? -b.num_ : b.num_, a.den_);
  const wide n = wide(a.num_ / g1) * (b.num_ / g2);
  const wide d = wide(a.den_ / g2) * (b.den_ / g1);
  return Coeff::ratio(narrow_or_throw(n), narrow_or_throw(d));
}

bool operator==(const Coeff& a, const Coeff& b) {
  if (a.exact_ && b.exact_) return a.num_ == b.num_ && a.den_ == b.den_;
  return a.value() == b.value();
}

std::string Coeff::str() const {
  char buf[64];
  if (!exact_)
    std::snprintf(buf, sizeof buf, "%.16g", dbl_);
  else if (den_ == 1)
    std::snprintf(buf, sizeof buf, "%lld", (long long)num_);
  else
    std::snprintf(buf, sizeof buf, "%lld/%lld", (long long)num_, (long long)den_);
  return buf;
}

// ---------------------------------------------------------- LaurentPoly

namespace {
// Sums coefficients per key in the order the terms arrive, drops zeros,
// returns key-sorted terms.
std::vector<Term> canonical(const std::vector<Term>& in) {
  std::map<Exponent, Coeff> acc;
  for (const Term& t : in) {
    auto [it, fresh] = acc.try_emplace(t.e, t.c);
    if (!fresh) it->second = it->second + t.c;
  }
  std::vector<Term> out;
  out.reserve(acc.size());
  for (const auto& [e, c] : acc)
    if (!c.is_zero()) out.push_back(Term{e, c});
  return out;
}
}  // namespace

LaurentPoly LaurentPoly::monomial(Coeff c, int m, int n) {
  LaurentPoly p;
  if (!c.is_zero()) p.t_.push_back(Term{{m, n}, c});
  return p;
}

LaurentPoly LaurentPoly::constant(Coeff c) { return monomial(c, 0, 0); }

LaurentPoly LaurentPoly::univariate(std::initializer_list<std::pair<int, Coeff>> taps) {
  std::vector<Term> v;
  for (const auto& [k, c] : taps) v.push_back(Term{{k, 0}, c});
  return from_terms(std::move(v));
}

LaurentPoly LaurentPoly::from_terms(std::vector<Term> terms) {
  LaurentPoly p;
  p.t_ = canonical(terms);
  return p;
}

Coeff LaurentPoly::coeff(int m, int n) const {
  const Exponent key{m, n};
  const auto it = std::lower_bound(t_.begin(), t_.end(), key,
                                   [](const Term& t, const Exponent& k) { return t.e < k; });
  return (it != t_.end() && it->e == key) ? it->c : Coeff{};
}

bool LaurentPoly::is_constant() const {
  return t_.empty() || (t_.size() == 1 && t_[0].e == Exponent{});
}

bool LaurentPoly::is_one() const {
  return t_.size() == 1 && t_[0].e == Exponent{} && t_[0].c.is_one();
}

bool LaurentPoly::univariate_m() const {
  return std::none_of(t_.begin(), t_.end(), [](const Term& t) { return t.e.n != 0; });
}

bool LaurentPoly::univariate_n() const {
  return std::none_of(t_.begin(), t_.end(), [](const Term& t) { return t.e.m != 0; });
}

LaurentPoly operator+(const LaurentPoly& a, const LaurentPoly& b) {
  std::vector<Term> v(a.t_);
  v.insert(v.end(), b.t_.begin(), b.t_.end());
  return LaurentPoly::from_terms(std::move(v));
}

LaurentPoly operator-(const LaurentPoly& a) {
  LaurentPoly r = a;
  for (Term& t : r.t_) t.c = -t.c;
  return r;
}

LaurentPoly operator-(const LaurentPoly& a, const LaurentPoly& b) { return a + (-b); }

LaurentPoly operator*(const LaurentPoly& a, const LaurentPoly& b) {
  std::vector<Term> v;
  v.reserve(a.t_.size() * b.t_.size());
  for (const Term& x : a.t_)
    for (const Term& y : b.t_)
      v.push_back(Term{{x.e.m + y.e.m, x.e.n + y.e.n}, x.c * y.c});
  return LaurentPoly::from_terms(std::move(v));
}

bool operator==(const LaurentPoly& a, const LaurentPoly& b) {
  return std::equal(a.t_.begin(), a.t_.end(), b.t_.begin(), b.t_.end(),
                    [](const Term& x, const Term& y) { return x.e == y.e && x.c == y.c; });
}

LaurentPoly transpose(const LaurentPoly& p) {
  std::vector<Term> v = p.terms();
  for (Term& t : v) std::swap(t.e.m, t.e.n);
  return LaurentPoly::from_terms(std::move(v));
}

LaurentPoly embed(const LaurentPoly& p, Axis axis) {
  if (p.univariate_m()) return axis == Axis::horizontal ? p : transpose(p);
  if (p.univariate_n()) return axis == Axis::vertical ? p : transpose(p);
  throw std::invalid_argument("embed: polynomial is not univariate");
}

std::pair<LaurentPoly, LaurentPoly> split_constant(const LaurentPoly& p) {
  const LaurentPoly c0 = LaurentPoly::constant(p.coeff(0, 0));
  return {c0, p - c0};
}

bool approx_equal(const LaurentPoly& a, const LaurentPoly& b, double tol) {
  auto one_way = [tol](const LaurentPoly& x, const LaurentPoly& y) {
    return std::all_of(x.terms().begin(), x.terms().end(), [&](const Term& t) {
      return std::abs(t.c.value() - y.coeff(t.e.m, t.e.n).value()) <= tol;
    });
  };
  return one_way(a, b) && one_way(b, a);
}

std::string to_string(const LaurentPoly& p) {
  if (p.is_zero()) return "0";
  auto power = [](const char* v, int key) {
    // stored key k denotes v^-k
    return key == -1 ? std::string(v) : std::string(v) + "^" + std::to_string(-key);
  };
  std::string s;
  for (std::size_t i = 0; i < p.terms().size(); ++i) {
    const Term& t = p.terms()[i];
    const bool neg = t.c.value() < 0.0;
    const Coeff mag = neg ? -t.c : t.c;
    std::string mono;
    if (t.e.m) mono = power("zm", t.e.m);
    if (t.e.n) mono += (mono.empty() ? "" : "*") + power("zn", t.e.n);
    std::string body = mono.empty() ? mag.str() : mag.is_one() ? mono : mag.str() + "*" + mono;
    if (i == 0)
      s = neg ? "-" + body : body;
    else
      s += (neg ? " - " : " + ") + body;
  }
  return s;
}

// ----------------------------------------------------------- PolyMatrix

PolyMatrix::PolyMatrix(int rows, int cols) : r_(rows), c_(cols) {
  if (rows <= 0 || cols <= 0) throw std::invalid_argument("matrix dimensions must be positive");
  cell_.resize(std::size_t(rows) * cols);
}

PolyMatrix PolyMatrix::identity(int n) {
  PolyMatrix m(n, n);
  for (int i = 0; i < n; ++i) m.at(i, i) = LaurentPoly::constant(Coeff(1));
  return m;
}

bool PolyMatrix::is_identity() const {
  if (r_ != c_) return false;
  for (int r = 0; r < r_; ++r)
    for (int c = 0; c < c_; ++c)
      if (r == c ? !at(r, c).is_one() : !at(r, c).is_zero()) return false;
  return true;
}

PolyMatrix mat_mul(const PolyMatrix& a, const PolyMatrix& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("mat_mul: dimension mismatch");
  PolyMatrix out(a.rows(), b.cols());
  for (int r = 0; r < a.rows(); ++r)
    for (int c = 0; c < b.cols(); ++c) {
      LaurentPoly sum;
      for (int k = 0; k < a.cols(); ++k) sum = sum + a.at(r, k) * b.at(k, c);
      out.at(r, c) = std::move(sum);
    }
  return out;
}

bool approx_equal(const PolyMatrix& a, const PolyMatrix& b, double tol) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (int r = 0; r < a.rows(); ++r)
    for (int c = 0; c < a.cols(); ++c)
      if (!approx_equal(a.at(r, c), b.at(r, c), tol)) return false;
  return true;
}

}  // namespace dwt2d_b200
