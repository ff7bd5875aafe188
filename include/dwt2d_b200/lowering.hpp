// Lowering: Scheme -> the list of stencil sub-steps one fused CUDA pass
// executes per decomposition level.
//
// The reference lowers each fused group to ONE composed stencil kernel and
// runs one barrier-separated pass per group (proj/include/dwt2d/executor.hpp
// :52-103, :196-238). On B200 every group of a level runs inside a single
// HBM pass (register sliding window, see csrc/kernels/level_engine.cuh), so
// "barriers" become register/shuffle dependencies. Two lowerings:
//
//   composed  one sub-step per fused group, the composed matrix with the
//             reference's tap order (source component, then (dn, dm)), its
//             float weights (T)(coef * pre) and its rounding (a multiply and
//             an add per tap) — reproduces the reference's float32 executor
//             bit for bit (executor.hpp:85-97, :179-184).
//   factored  one sub-step per factor (rightmost first), so the optimized
//             schemes really execute the paper's reduced operation count
//             (scheme.cpp:279-378 builds the factors; the reference composes
//             them away at executor.hpp:62).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "dwt2d_b200/schemes.hpp"

namespace dwt2d_b200 {

struct KernelTap {
  int comp = 0;  // source component 0..3
  int dm = 0;    // reads component sample (x + dm, y + dn)
  int dn = 0;
  double coef = 0.0;  // composed coefficient times folded pre-scale
  float w = 0.0f;     // (float)coef, the weight the kernel multiplies by
};

struct KernelRow {
  bool identity = false;  // output component == input component
  float scale = 1.0f;     // applied after accumulation (post-scale)
  double scale64 = 1.0;   // the same post-scale for float64 execution (compile<double>)
  std::vector<KernelTap> taps;
};

struct KernelStep {
  std::array<KernelRow, 4> rows;
  // component-grid reach of this sub-step (identity/diagonal reads at 0)
  int min_dm = 0, max_dm = 0, min_dn = 0, max_dn = 0;
};

enum class Lowering { composed, factored };

struct StepProgram {
  std::string key;  // "<wavelet>/<scheme-id>/<base|opt>/<composed|factored>"
  std::vector<KernelStep> steps;
  long logical_steps = 0;  // count_steps(scheme): the reference's barrier count
  // rounding model of every tap: false = round(w*v) then round(acc + p), the
  // reference executor's arithmetic (bit-exact to its float32 path); true =
  // one fused multiply-add per tap (factored lowering)
  bool fused_multiply_add = false;
  // accumulated reach of the whole level: output (x, y) depends on input
  // columns x-left..x+right and rows y-up..y+down
  int left = 0, right = 0, up = 0, down = 0;
  long taps_per_quad() const;
  std::uint64_t fingerprint() const;  // hash of every table entry
};

StepProgram lower(const Scheme& s, Lowering mode);

// composed for baseline schemes and inverse lifting, factored for
// optimized schemes (the paper's operation-reduced execution)
inline Lowering default_lowering(const Scheme& s) {
  return s.optimized ? Lowering::factored : Lowering::composed;
}

}  // namespace dwt2d_b200
