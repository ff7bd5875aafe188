// C++ API tests of the drop-in layer (include/dwt2d_b200/dwt2d.hpp), written
// the way the reference's own executor tests are (proj/tests/
// test_executor.cpp, test_algebra.cpp) but self-contained (no doctest in this
// image). Run by tests/test_cpp_api.py: `test_cpp_api host` needs no GPU,
// `test_cpp_api gpu` runs compile/run/inverse_lifting on the device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "dwt2d_b200/dwt2d.hpp"
#include "dwt2d_b200/io.hpp"
#include <filesystem>
#include <sstream>

namespace {

int g_fail = 0, g_checks = 0;

#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)

template <class E, class F>
void check_throws(F&& f, const char* what) {
  ++g_checks;
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  ++g_fail;
  std::printf("FAIL: expected exception: %s\n", what);
}

using namespace dwt2d;  // the reference's namespace name, via the alias

double max_abs_diff(const PolyphaseImage<float>& a, const PolyphaseImage<float>& b) {
  double m = 0;
  for (int j = 0; j < 4; ++j)
    for (std::size_t i = 0; i < a.comp[j].samples.size(); ++i)
      m = std::max(m, std::abs(double(a.comp[j].samples[i]) - double(b.comp[j].samples[i])));
  return m;
}

// ---------------------------------------------------------------- host

void host_tests() {
  // extend_index frozen examples (test_executor.cpp:108-123)
  CHECK(extend_index(-1, 8, Extension::periodic) == 7);
  CHECK(extend_index(-9, 8, Extension::periodic) == 7);
  CHECK(extend_index(8, 8, Extension::symmetric) == 6);
  CHECK(extend_index(15, 8, Extension::symmetric) == 1);
  check_throws<std::invalid_argument>([] { extend_index(0, 0, Extension::periodic); }, "empty axis");

  // LCG frozen first draw (test_executor.cpp:149-159) and jump-ahead
  Lcg64 g(1);
  CHECK(g.next_u64() == 0x5851f42d4c957f2dull + 0x14057b7ef767814full);
  Lcg64 a(7), b(7);
  for (int i = 0; i < 1000; ++i) a.next_u64();
  b.jump(1000);
  CHECK(a.state() == b.state());

  // split / merge (test_executor.cpp:125-147)
  const auto big = random_image<float>(16, 12, 99);
  CHECK(polyphase_merge(polyphase_split(big)) == big);
  check_throws<std::invalid_argument>([] { polyphase_split(ImagePlane<float>(3, 4)); }, "odd width");

  // Table 1 operation counts (test_algebra.cpp:227-243)
  const auto& w97 = get_wavelet("cdf97");
  CHECK(count_operations(build_separable_lifting(w97)) == 32);
  CHECK(count_operations(optimize_constant_split(build_nonseparable_lifting(w97), w97)) == 36);
  CHECK(count_operations(optimize_constant_split(build_nonseparable_lifting(get_wavelet("cdf53")),
                                                 get_wavelet("cdf53"))) == 18);
  CHECK(count_steps(build_nonseparable_lifting(w97)) == 4);

  // symbolic identities (acceptance.cpp criterion 3)
  for (const auto& pr : get_wavelet("cdf53").pairs()) {
    CHECK(spatial_predict(pr.predict) == predict_v(pr.predict) * predict_h(pr.predict));
    CHECK(polyconv_matrix(pr.predict, pr.update) ==
          spatial_update(pr.update) * spatial_predict(pr.predict));
  }
  const PolyMatrix ref = build_separable_lifting(w97).total();
  for (SchemeKind k : all_scheme_kinds())
    CHECK(approx_equal(build_scheme(k, w97).total(), ref, 1e-12));

  // supports (acceptance.cpp criterion 7)
  const PolyMatrix n97 = build_nonseparable_convolution(w97).total();
  CHECK((row_image_support(n97, 0) == std::pair<int, int>{9, 9}));
  CHECK((row_image_support(n97, 3) == std::pair<int, int>{7, 7}));

  // compile-time validation (executor.hpp:54-55)
  check_throws<std::invalid_argument>(
      [&] { compile<float>(build_separable_lifting(w97), Extension::periodic, 0); }, "workers 0");
  check_throws<std::invalid_argument>([&] { optimize_constant_split(build_inverse_lifting(w97), w97); },
                                      "optimize inverse");

  // the lowering: composed cdf97 non-separable lifting has 61 taps per quad
  // (SURVEY §2.3), the factored optimized one realises 36 multiply-adds
  const StepProgram base = lower(build_nonseparable_lifting(w97), Lowering::composed);
  CHECK(base.taps_per_quad() == 61);
  CHECK(base.up == 2 && base.down == 2 && base.left == 2 && base.right == 2);
  const StepProgram opt =
      lower(optimize_constant_split(build_nonseparable_lifting(w97), w97), Lowering::factored);
  long fmas = 0;
  for (const auto& st : opt.steps)
    for (const auto& r : st.rows)
      if (!r.identity) fmas += long(r.taps.size()) - ((!r.taps.empty() && r.taps[0].w == 1.0f) ? 1 : 0);
  CHECK(fmas == 36);
}

// ------------------------------------------------------------------ io
// (test_io.cpp cases for the PGM reader and the sub-band files)

PgmError::Kind pgm_kind(const std::string& text) {
  std::istringstream in(text);
  try {
    read_pgm(in);
  } catch (const PgmError& e) {
    return e.kind;
  }
  throw std::logic_error("expected a PgmError");
}

void io_tests() {
  {
    std::istringstream in("P2 # magic\n# a 2x3 ramp\n2 3\n255\n0 51\n102 153\n204 255\n");
    const auto img = read_pgm(in);
    CHECK(img.width == 2 && img.height == 3);
    CHECK(img.at(0, 0) == 0.0);
    CHECK(std::abs(img.at(1, 0) - 51.0 / 255.0) < 1e-15);
    CHECK(img.at(1, 2) == 1.0);
  }
  {
    std::string p5 = "P5 2 2 255\n";
    p5 += std::string("\x00\x40\x80\xff", 4);
    std::istringstream in(p5);
    const auto img = read_pgm(in);
    CHECK(img.at(1, 1) == 1.0);
    CHECK(std::abs(img.at(1, 0) - 64.0 / 255.0) < 1e-15);
    std::string p16 = "P5 1 1 65535\n";
    p16 += std::string("\x80\x00", 2);
    std::istringstream in16(p16);
    CHECK(std::abs(read_pgm(in16).at(0, 0) - 32768.0 / 65535.0) < 1e-15);
  }
  CHECK(pgm_kind("P6 1 1 255\n") == PgmError::Kind::unsupported_magic);
  CHECK(pgm_kind("P2 0 1 255\n") == PgmError::Kind::bad_header);
  CHECK(pgm_kind("P2 2 2 70000\n0 0 0 0") == PgmError::Kind::bad_header);
  CHECK(pgm_kind("P2 2 2 255\n0 0 0") == PgmError::Kind::truncated);
  CHECK(pgm_kind("P5 2 2 255\n\x01") == PgmError::Kind::truncated);
  // sub-band round trip and sidecar validation
  const auto dir = std::filesystem::temp_directory_path() / "dwt2d_b200_subbands";
  std::filesystem::remove_all(dir);
  const auto p = polyphase_split(random_image<float>(12, 8, 5));
  write_subbands(p, dir);
  CHECK(read_subbands<float>(dir) == p);
  check_throws<IoError>([&] { read_subbands<double>(dir); }, "precision mismatch");
  std::filesystem::resize_file(dir / "oo.raw", 4);
  check_throws<IoError>([&] { read_subbands<float>(dir); }, "short payload");
  std::filesystem::remove_all(dir);
}

// ----------------------------------------------------------------- gpu

void gpu_tests() {
  // executor matches across schemes and the inverse restores the input
  // (test_executor.cpp:279-299)
  const auto img = random_image<float>(64, 48, 404);
  const auto in = polyphase_split(img, Extension::periodic);
  for (const std::string& name : {std::string("cdf53"), std::string("cdf97"), std::string("dd137")}) {
    const WaveletSpec w = get_wavelet(name);
    PolyphaseImage<float> first;
    bool have_first = false;
    for (SchemeKind k : all_scheme_kinds()) {
      for (bool optimize : {false, true}) {
        Scheme s = build_scheme(k, w);
        if (optimize) s = optimize_constant_split(s, w);
        ExecPlan<float> plan = compile<float>(s, Extension::periodic, 3);
        const auto out = run(plan, in);
        CHECK(plan.barrier_count == long(count_steps(s)));  // test_executor.cpp:259-277
        if (!have_first) {
          first = out;
          have_first = true;
        } else {
          CHECK(max_abs_diff(out, first) < 2e-5);  // every scheme, same transform
        }
        const auto back = inverse_lifting(w, out, 2);
        CHECK(max_abs_diff(back, in) < 5e-5);
      }
    }
  }
  // worker count never changes a bit (test_executor.cpp:233-257)
  {
    const Scheme s = build_nonseparable_lifting(get_wavelet("cdf97"));
    auto p1 = compile<float>(s, Extension::periodic, 1);
    auto p7 = compile<float>(s, Extension::periodic, 7);
    const auto a = run(p1, in), b = run(p7, in);
    CHECK(a == b);
  }
  // constant image: high bands vanish, low band keeps the level (:198-211)
  {
    ImagePlane<float> c(16, 16);
    for (auto& v : c.samples) v = 0.375f;
    auto plan = compile<float>(build_separable_lifting(get_wavelet("cdf53")), Extension::periodic, 1);
    const auto out = run(plan, polyphase_split(c));
    for (int j = 1; j < 4; ++j)
      for (float v : out.comp[j].samples) CHECK(v == 0.0f);
    for (float v : out.comp[0].samples) CHECK(v == 0.375f);
  }
  // identity steps of a pairless wavelet are plain copies (:279-289)
  {
    const WaveletSpec empty;
    auto plan = compile<float>(build_separable_convolution(empty), Extension::periodic, 2);
    const auto out = run(plan, in);
    CHECK(out == in);
  }
  // compile<double> / run<double>: the float64 executor agrees with the
  // float32 transform to float32 precision and round-trips to 1e-12, for
  // both extensions (the reference's equiv precision, equiv.cpp:161-168)
  for (Extension ext : {Extension::periodic, Extension::symmetric}) {
    const WaveletSpec w = get_wavelet("cdf97");
    const auto imgd = random_image<double>(64, 48, 404);
    const auto ind = polyphase_split(imgd, ext);
    const auto inf = polyphase_split(random_image<float>(64, 48, 404), ext);
    for (bool optimize : {false, true}) {
      Scheme s = build_scheme(SchemeKind::nonseparable_lifting, w);
      if (optimize) s = optimize_constant_split(s, w);
      ExecPlan<double> pd = compile<double>(s, ext, 2);
      ExecPlan<float> pf = compile<float>(s, ext, 2);
      const auto od = run(pd, ind);
      const auto of = run(pf, inf);
      double m = 0;
      for (int j = 0; j < 4; ++j)
        for (size_t i = 0; i < od.comp[j].samples.size(); ++i)
          m = std::max(m, std::abs(od.comp[j].samples[i] - double(of.comp[j].samples[i])));
      CHECK(m < 2e-5);
      const auto back = inverse_lifting(w, od, 1);
      double e = 0;
      for (int j = 0; j < 4; ++j)
        for (size_t i = 0; i < back.comp[j].samples.size(); ++i)
          e = std::max(e, std::abs(back.comp[j].samples[i] - ind.comp[j].samples[i]));
      CHECK(e < 1e-12);
    }
  }
  // input validation (test_executor.cpp:343-355)
  {
    auto plan = compile<float>(build_separable_lifting(get_wavelet("cdf53")), Extension::periodic, 1);
    check_throws<std::invalid_argument>([&] { run(plan, PolyphaseImage<float>{}); }, "empty");
    auto sym = polyphase_split(random_image<float>(8, 8, 1), Extension::symmetric);
    check_throws<std::invalid_argument>([&] { run(plan, sym); }, "extension mismatch");
    auto bad = polyphase_split(random_image<float>(8, 8, 1));
    bad.comp[2] = ImagePlane<float>(3, 4);
    check_throws<std::invalid_argument>([&] { run(plan, bad); }, "component mismatch");
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  host_tests();
  io_tests();
  if (mode == "gpu") gpu_tests();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
