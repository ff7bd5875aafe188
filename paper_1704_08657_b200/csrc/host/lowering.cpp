// Scheme -> fused per-level sub-step program (see lowering.hpp).
#include "dwt2d_b200/lowering.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>

namespace dwt2d_b200 {

namespace {

// One matrix -> one sub-step. `pre` multiplies the inputs (folded into the
// weights), `post` the outputs (kept as a row scale), as the reference
// compiler does for the first and last kernel (executor.hpp:68-97).
KernelStep lower_matrix(const PolyMatrix& m, const std::array<double, 4>& pre,
                        const std::array<double, 4>& post, bool diagonal_first) {
  if (m.rows() != 4 || m.cols() != 4)
    throw std::invalid_argument("compile: scheme matrices must be 4x4");
  KernelStep st;
  for (int r = 0; r < 4; ++r) {
    KernelRow& row = st.rows[r];
    bool plain = true;
    for (int j = 0; j < 4 && plain; ++j)
      plain = (j == r) ? m.at(r, j).is_one() : m.at(r, j).is_zero();
    if (plain && post[r] == 1.0 && pre[r] == 1.0) {
      row.identity = true;
      continue;
    }
    row.scale = static_cast<float>(post[r]);
    row.scale64 = post[r];
    for (int j = 0; j < 4; ++j) {
      std::vector<Term> t = m.at(r, j).terms();
      std::sort(t.begin(), t.end(), [](const Term& a, const Term& b) {
        return a.e.n != b.e.n ? a.e.n < b.e.n : a.e.m < b.e.m;
      });
      for (const Term& term : t) {
        KernelTap k;
        k.comp = j;
        k.dm = term.e.m;
        k.dn = term.e.n;
        k.coef = term.c.value() * pre[j];
        k.w = static_cast<float>(k.coef);
        row.taps.push_back(k);
      }
    }
    if (diagonal_first) {
      // start the accumulation from the unit self-tap (a plain copy), so a
      // lifting factor costs one fma per predicted/updated sample
      auto self = std::find_if(row.taps.begin(), row.taps.end(), [r](const KernelTap& k) {
        return k.comp == r && k.dm == 0 && k.dn == 0 && k.w == 1.0f;
      });
      if (self != row.taps.end()) std::rotate(row.taps.begin(), self, self + 1);
    }
  }
  for (const KernelRow& row : st.rows)
    for (const KernelTap& k : row.taps) {
      st.min_dm = std::min(st.min_dm, k.dm), st.max_dm = std::max(st.max_dm, k.dm);
      st.min_dn = std::min(st.min_dn, k.dn), st.max_dn = std::max(st.max_dn, k.dn);
    }
  return st;
}

constexpr std::array<double, 4> kOnes{1.0, 1.0, 1.0, 1.0};

}  // namespace

StepProgram lower(const Scheme& s, Lowering mode) {
  StepProgram p;
  p.key = s.wavelet + "/" + scheme_id(s.kind) + "/" + (s.optimized ? "opt" : "base") + "/" +
          (mode == Lowering::composed ? "composed" : "factored");
  p.logical_steps = long(s.steps.size());
  p.fused_multiply_add = mode == Lowering::factored;
  // flatten to the matrices actually executed, in execution order
  std::vector<PolyMatrix> mats;
  for (const FusedGroup& g : s.steps) {
    if (mode == Lowering::composed) {
      mats.push_back(g.composed());
    } else {
      if (g.factors.empty()) throw std::logic_error("empty fused group");
      for (auto it = g.factors.rbegin(); it != g.factors.rend(); ++it) mats.push_back(*it);
    }
  }
  for (std::size_t i = 0; i < mats.size(); ++i) {
    const bool first = i == 0, last = i + 1 == mats.size();
    p.steps.push_back(lower_matrix(mats[i], first ? s.pre_scale : kOnes, last ? s.post_scale : kOnes,
                                   mode == Lowering::factored));
  }
  for (const KernelStep& st : p.steps) {
    p.left += -st.min_dm;
    p.right += st.max_dm;
    p.up += -st.min_dn;
    p.down += st.max_dn;
  }
  return p;
}

long StepProgram::taps_per_quad() const {
  long n = 0;
  for (const KernelStep& st : steps)
    for (const KernelRow& r : st.rows) n += long(r.taps.size());
  return n;
}

std::uint64_t StepProgram::fingerprint() const {
  std::uint64_t h = 1469598103934665603ull;  // FNV-1a over the tables
  auto mix = [&h](std::uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  mix(steps.size());
  mix(fused_multiply_add ? 1 : 0);
  for (const KernelStep& st : steps)
    for (const KernelRow& r : st.rows) {
      std::uint32_t sb;
      std::memcpy(&sb, &r.scale, 4);
      mix(r.identity);
      mix(sb);
      mix(r.taps.size());
      for (const KernelTap& t : r.taps) {
        std::uint32_t wb;
        std::memcpy(&wb, &t.w, 4);
        mix(std::uint64_t(t.comp));
        mix(std::uint64_t(std::int64_t(t.dm)));
        mix(std::uint64_t(std::int64_t(t.dn)));
        mix(wb);
      }
    }
  return h;
}

}  // namespace dwt2d_b200
