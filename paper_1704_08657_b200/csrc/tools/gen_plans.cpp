// Build-time generator: lowers every built-in (wavelet, scheme, variant) with
// the product's own host algebra and emits
//   plans_gen.cuh      constexpr tap tables (hex-float weights, exact)
//   inst_<w>_<s>.cu    kernel instantiations + registration, one file per
//                      (wavelet, scheme) so nvcc can build them in parallel
//   registry_gen.cu   the table the runtime searches by fingerprint
// Usage: gen_plans <output dir>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "dwt2d_b200/lowering.hpp"
#include "dwt2d_b200/schemes.hpp"

using namespace dwt2d_b200;

namespace {

std::string ident(std::string s) {
  for (char& c : s)
    if (c == '-' || c == '/') c = '_';
  return s;
}

std::string hexf(float f) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%af", double(f));
  return buf;
}

struct Gen {
  std::string name;   // C identifier
  std::string group;  // wavelet_scheme (one .cu per group)
  bool forward;
  StepProgram prog;
  int cw;
  bool pack;  // composed programs: packed FP32 arithmetic
  bool shift = false;  // shifted register windows, one loop body per row
  int depth = 1;       // deepest row window of a sub-step
};

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::cerr << "usage: gen_plans <outdir>\n";
    return 2;
  }
  const std::string out = argv[1];
  std::vector<Gen> gens;
  for (const std::string& wn : wavelet_names()) {
    const WaveletSpec& w = get_wavelet(wn);
    auto add = [&](const Scheme& s, bool fwd) {
      Gen g;
      g.prog = lower(s, default_lowering(s));
      g.name = ident(wn + "_" + scheme_id(s.kind) + (s.optimized ? "_opt" : "_base"));
      g.group = ident(wn + "_" + scheme_id(s.kind));
      g.forward = fwd;
      const int reach = std::max(g.prog.left, g.prog.right);
      // 4 component columns (8 image pixels, two 128-bit loads per image row)
      // per lane amortise the per-row pointer and loop work (6.1 vs 5.2 TB/s
      // for CW=2 on the headline level, scripts/tune_level.cu); programs with
      // deep row windows (convolutions, >= 4 rows) keep CW=2 to stay in
      // registers when their horizontal reach allows it
      int depth = 1;
      for (const KernelStep& st : g.prog.steps) depth = std::max(depth, st.max_dn - st.min_dn + 1);
      g.depth = depth;
      std::size_t step_taps = 0;
      for (const KernelStep& st : g.prog.steps) {
        std::size_t n = 0;
        for (const KernelRow& r : st.rows) n += r.taps.size();
        step_taps = std::max(step_taps, n);
      }
      // Composed (reference-rounding) programs: the wide ones (deep windows
      // or >= 64 taps per sub-step) keep CW=2 too, and only the 256-tap
      // convolution is packed (FFMA2 + FADD2, level_engine.cuh) at CW=2: the
      // others measured faster scalar there (16384^2: separable convolution
      // 445 vs 501 us, polyconvolution 710 vs 742 us, and spill-free unlike
      // CW=4 at 901 us); CW=4 composed programs are packed (non-separable
      // lifting 430 vs 481 us). scripts/tune_composed.cu.
      //
      // The widest programs (>= 128 taps per quad: CDF 9/7 non-separable
      // convolution and polyconvolution baseline, non-separable convolution
      // optimized) shift their register windows (kShift, level_engine.cuh:
      // Sched) and run one loop body per row at CW=4, scalar: the unrolled
      // body did not stay in the instruction cache. 16384^2 / 4096^2:
      // non-separable convolution baseline 1264 / 98.6 us (was 1775 / 150.5
      // packed at CW=2), polyconvolution baseline 644 / 50.9 (719 / 77.9),
      // non-separable convolution optimized 506 / 43.9 (537 / 45.6); the
      // 64-tap CDF 5/3 ones and the separable convolutions measured no gain
      // or a loss (scripts/tune_composed.cu, SHIFT_ONLY=1).
      const bool fma = g.prog.fused_multiply_add;
      g.shift = reach <= 2 && g.prog.taps_per_quad() >= 128;
      // Factored (FMA) programs all take CW=4 (with TMA staging at 16384^2
      // the separable convolution optimized runs 362 vs 422 us at CW=2).
      g.cw = !fma && !g.shift && reach <= 2 && (depth >= 4 || step_taps >= 64) ? 2 : 4;
      g.pack = g.shift ? fma : (fma || g.cw == 4 || step_taps > 128);
      if (reach > 4) {
        std::cerr << "plan " << g.name << " reaches " << reach << " columns; unsupported\n";
        std::exit(1);
      }
      // The fused body is fully unrolled (taps x CW x rows of the unroll);
      // for the 7x7-window DD 13/7 non-separable convolutions (>200
      // taps/quad at reach 3) cicc ran for over 30 minutes per unit. Those
      // four programs (compute-bound, in no benchmark configuration) run on
      // the generic GPU executor instead (kernels/generic_step.cu), which
      // the runtime selects whenever no fingerprint matches.
      if (reach >= 3 && g.prog.taps_per_quad() > 128) {
        std::cout << "generic executor: " << g.prog.key << "\n";
        return;
      }
      gens.push_back(std::move(g));
    };
    for (SchemeKind k : all_scheme_kinds()) {
      const Scheme base = build_scheme(k, w);
      add(base, true);
      add(optimize_constant_split(base, w), true);
    }
    add(build_inverse_lifting(w), false);
  }

  std::ostringstream h;
  h << "// GENERATED by csrc/tools/gen_plans.cpp from the host lowering — do not edit.\n"
       "#pragma once\n#include \"../kernels/level_engine.cuh\"\n"
       "namespace dwt2d_b200 {\nnamespace gpu {\nnamespace plans {\n";
  for (const Gen& g : gens) {
    const StepProgram& p = g.prog;
    std::vector<std::string> rows, taps;
    int t = 0;
    for (const KernelStep& st : p.steps)
      for (const KernelRow& r : st.rows) {
        const int tb = t;
        for (const KernelTap& k : r.taps) {
          std::ostringstream ts;
          ts << "{" << k.comp << ", " << k.dm << ", " << k.dn << ", " << hexf(k.w) << "}";
          taps.push_back(ts.str());
          ++t;
        }
        std::ostringstream rs;
        rs << "{" << (r.identity ? 1 : 0) << ", " << tb << ", " << t << ", " << hexf(r.scale) << "}";
        rows.push_back(rs.str());
      }
    h << "\n// " << p.key << ": " << p.steps.size() << " sub-steps, " << p.taps_per_quad()
      << " taps/quad, reach L" << p.left << " R" << p.right << " U" << p.up << " D" << p.down << "\n";
    h << "struct " << g.name << " {\n";
    h << "  static constexpr const char* kKey = \"" << p.key << "\";\n";
    char fp[32];
    std::snprintf(fp, sizeof fp, "0x%016llxull", (unsigned long long)p.fingerprint());
    h << "  static constexpr unsigned long long kFingerprint = " << fp << ";\n";
    h << "  static constexpr int kSteps = " << p.steps.size() << ";\n";
    h << "  static constexpr int kCW = " << g.cw << ";\n";
    h << "  static constexpr bool kFma = " << (p.fused_multiply_add ? "true" : "false") << ";\n";
    h << "  static constexpr bool kPack = " << (g.pack ? "true" : "false") << ";\n";
    if (g.shift) h << "  static constexpr bool kShift = true;\n";
    // bottom-up odd chunks (level_engine.cuh: level_dispatch) for programs
    // with short sub-steps; the wide composed steps (non-separable
    // convolution / polyconvolution / lifting baselines) lose more to the
    // second unrolled body's register pressure than the L2 reuse gains
    // (measured at 4096^2: e.g. non-separable convolution baseline 0.22 vs
    // 0.48 ms, optimized non-separable lifting 32.8 vs 30.7 us)
    // Round 2, TMA-staged 16384^2 levels: the convolution-shaped factored
    // programs (row windows of 3 or more) lose with it too (separable
    // convolution optimized 462 vs 378 us, polyconvolution optimized 386 vs
    // 357; the lifting ones gain: 342 vs 360), scripts/probe_pair_programs.py
    const bool alt = g.depth <= 2 && (p.fused_multiply_add || p.taps_per_quad() <= 8 * (long)p.steps.size());
    h << "  static constexpr bool kAlt = " << (alt ? "true" : "false") << ";\n";
    h << "  static constexpr int kTaps = " << std::max<std::size_t>(taps.size(), 1) << ";\n";
    h << "  static constexpr RowDesc rows[" << rows.size() << "] = {";
    for (std::size_t i = 0; i < rows.size(); ++i) h << (i == 0 ? "\n      " : i % 4 ? ", " : ",\n      ") << rows[i];
    h << "};\n";
    h << "  static constexpr TapDesc taps[" << std::max<std::size_t>(taps.size(), 1) << "] = {";
    if (taps.empty()) h << "{0, 0, 0, 0.0f}";
    for (std::size_t i = 0; i < taps.size(); ++i) h << (i == 0 ? "\n      " : i % 4 ? ", " : ",\n      ") << taps[i];
    h << "};\n};\n";
  }
  h << "\n}  // namespace plans\n}  // namespace gpu\n}  // namespace dwt2d_b200\n";
  std::ofstream(out + "/plans_gen.cuh") << h.str();

  std::map<std::string, std::vector<const Gen*>> groups;
  for (const Gen& g : gens) groups[g.group].push_back(&g);
  std::ostringstream reg;
  reg << "// GENERATED by csrc/tools/gen_plans.cpp — do not edit.\n"
         "#include <vector>\n#include \"../kernels/registry.hpp\"\n"
         "namespace dwt2d_b200 {\nnamespace gpu {\n";
  for (const auto& [grp, list] : groups) {
    std::ostringstream cu;
    cu << "// GENERATED by csrc/tools/gen_plans.cpp — do not edit.\n"
          "#include \"../kernels/registry.hpp\"\n#include \"plans_gen.cuh\"\n"
          "namespace dwt2d_b200 {\nnamespace gpu {\n"
       << "void register_" << grp << "(std::vector<PlanEntry>& v) {\n";
    for (const Gen* g : list)
      cu << "  v.push_back(make_entry<plans::" << g->name << ", " << (g->forward ? "true" : "false")
         << ">());\n";
    cu << "}\n}  // namespace gpu\n}  // namespace dwt2d_b200\n";
    std::ofstream(out + "/inst_" + grp + ".cu") << cu.str();
    reg << "void register_" << grp << "(std::vector<PlanEntry>&);\n";
  }
  reg << "const std::vector<PlanEntry>& plan_registry() {\n"
         "  static const std::vector<PlanEntry> table = [] {\n"
         "    std::vector<PlanEntry> v;\n";
  for (const auto& kv : groups) reg << "    register_" << kv.first << "(v);\n";
  reg << "    return v;\n  }();\n  return table;\n}\n"
         "const PlanEntry* find_plan(unsigned long long fp) {\n"
         "  for (const PlanEntry& e : plan_registry())\n"
         "    if (e.fingerprint == fp) return &e;\n"
         "  return nullptr;\n}\n"
         "}  // namespace gpu\n}  // namespace dwt2d_b200\n";
  std::ofstream(out + "/registry_gen.cu") << reg.str();
  std::cout << "generated " << gens.size() << " plans in " << groups.size() << " groups\n";
  return 0;
}
