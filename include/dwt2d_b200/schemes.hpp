// Wavelet registry and the paper's five calculation schemes (host side).
//
// Drop-in for the reference's wavelet / scheme layer
// (reference: proj/include/dwt2d/wavelet.hpp:14-45, scheme.hpp:13-104).
// Identical public names and semantics; these recipes are what the CUDA
// kernels execute (see lowering.hpp for how a Scheme becomes kernel steps).
#pragma once

#include <array>
#include <cstddef>
#include <filesystem>
#include <iosfwd>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "dwt2d_b200/algebra.hpp"

namespace dwt2d_b200 {

// ------------------------------------------------------------- wavelets

// One predict/update pair; both univariate in the horizontal variable.
struct LiftingPair {
  LaurentPoly predict;
  LaurentPoly update;
};

class WaveletSpec {
 public:
  WaveletSpec() = default;
  WaveletSpec(std::string name, std::vector<LiftingPair> pairs, double scaling = 1.0);
  const std::string& name() const { return name_; }
  const std::vector<LiftingPair>& pairs() const { return pairs_; }
  double scaling() const { return scaling_; }

 private:
  std::string name_;
  std::vector<LiftingPair> pairs_;
  double scaling_ = 1.0;
};

const WaveletSpec& get_wavelet(std::string_view name);  // cdf53, cdf97, dd137
std::vector<std::string> wavelet_names();
WaveletSpec parse_wavelet_definition(std::istream& in, std::string name);
WaveletSpec load_wavelet_file(const std::filesystem::path& path);
WaveletSpec resolve_wavelet(const std::string& name_or_path);

// --------------------------------------------------------------- schemes

enum class SchemeKind {
  separable_convolution,
  separable_lifting,
  nonseparable_convolution,
  nonseparable_polyconvolution,
  nonseparable_lifting,
  inverse_lifting,
};

const char* scheme_id(SchemeKind kind);
const char* scheme_label(SchemeKind kind);
SchemeKind scheme_from_id(const std::string& id);
std::vector<SchemeKind> all_scheme_kinds();

// Factors applied without a barrier between them. factors[0] is leftmost in
// the matrix product, i.e. applied LAST.
struct FusedGroup {
  std::vector<PolyMatrix> factors;
  PolyMatrix composed() const;
};

struct Scheme {
  std::string label;
  SchemeKind kind = SchemeKind::separable_lifting;
  std::string wavelet;
  bool optimized = false;
  std::vector<FusedGroup> steps;
  std::array<double, 4> pre_scale{1.0, 1.0, 1.0, 1.0};
  std::array<double, 4> post_scale{1.0, 1.0, 1.0, 1.0};
  PolyMatrix total() const;
};

struct LiftingSteps2D {
  PolyMatrix predict_h, predict_v, update_h, update_v;
};

LiftingSteps2D lifting_steps_2d(const LaurentPoly& p, const LaurentPoly& u);
PolyMatrix predict_h(const LaurentPoly& p);  // T[P]^H
PolyMatrix predict_v(const LaurentPoly& p);  // T[P]^V
PolyMatrix update_h(const LaurentPoly& u);   // S[U]^H
PolyMatrix update_v(const LaurentPoly& u);   // S[U]^V
PolyMatrix spatial_predict(const LaurentPoly& p);  // T[P]
PolyMatrix spatial_update(const LaurentPoly& u);   // S[U]
PolyMatrix polyconv_matrix(const LaurentPoly& p, const LaurentPoly& u);  // N[P,U]
PolyMatrix polyphase_1d(const WaveletSpec& w);

Scheme build_separable_convolution(const WaveletSpec& w);
Scheme build_separable_lifting(const WaveletSpec& w);
Scheme build_nonseparable_convolution(const WaveletSpec& w);
Scheme build_nonseparable_polyconvolution(const WaveletSpec& w);
Scheme build_nonseparable_lifting(const WaveletSpec& w);
Scheme build_scheme(SchemeKind kind, const WaveletSpec& w);
Scheme build_inverse_lifting(const WaveletSpec& w);
Scheme optimize_constant_split(const Scheme& s, const WaveletSpec& w);

std::size_t count_steps(const Scheme& s);
long count_operations(const Scheme& s);
std::pair<int, int> row_image_support(const PolyMatrix& m, int row);
std::string describe(const Scheme& s);

}  // namespace dwt2d_b200
