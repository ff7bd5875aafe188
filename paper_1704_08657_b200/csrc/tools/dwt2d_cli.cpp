// dwt2d — command-line front end of the B200 library, with the reference
// CLI's subcommands, options, output formats and exit codes
// (proj/tools/dwt2d.cpp:111-209; 0 success, 1 tolerance
// failure, 2 usage error, 3 I/O error). CLI11 is not vendored in the
// reference mount, so arguments are parsed here.
//
//   dwt2d describe  --wavelet W --scheme S [--optimize]
//   dwt2d count     --wavelet W
//   dwt2d equiv     --wavelet W --size N --seed K --extension E [--precision 64|32]
//   dwt2d transform in.pgm --out DIR [--wavelet --scheme --optimize
//                   --extension --precision 64|32 --workers N --levels L]
//   dwt2d bench     [--wavelet --scheme all|ID --optimize --sizes a,b,..
//                   --workers --repeats --precision 32 --seed --extension
//                   --levels L --out FILE]
//
// Precision: like the reference, `transform` and `equiv` default to float64
// (the GPU's float64 executor: compile<double>/run<double>, one pass per
// sub-step) and take --precision 32 for the fused float32 kernels; `equiv`
// in float64 uses the reference's tolerance (1e-12 with exact coefficients,
// else 1e-9, equiv.cpp:34-47), in float32 the float32 parity bar 1e-5.
// `bench` times the float32 kernels only (--precision 64 is a usage error).
// Additions: `transform --levels L` writes a Mallat pyramid as
// DIR/level<l>/ sub-band sets; `bench --levels L` times the pyramid.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "dwt2d_b200/dwt2d.hpp"
#include "dwt2d_b200/io.hpp"

using namespace dwt2d_b200;

namespace {

struct Usage : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct Args {
  std::string cmd;
  std::vector<std::string> positional;
  std::map<std::string, std::string> opt;
  std::vector<std::string> flags;
  bool has(const std::string& f) const { return std::find(flags.begin(), flags.end(), f) != flags.end(); }
  std::string get(const std::string& k, const std::string& d) const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
};

const char* kUsage =
    "usage: dwt2d <describe|count|equiv|transform|bench> [options]\n"
    "  describe  --wavelet W --scheme S [--optimize]\n"
    "  count     --wavelet W\n"
    "  equiv     --wavelet W --size N --seed K --extension periodic|symmetric --precision 64|32\n"
    "  transform IN.pgm --out DIR [--wavelet W --scheme S --optimize --extension E\n"
    "            --precision 64|32 --workers N --levels L]\n"
    "  bench     [--wavelet W --scheme all|S --optimize --sizes 256,512 --workers N\n"
    "            --repeats R --precision 32 --seed K --extension E --levels L --out FILE]\n";

Args parse(int argc, char** argv) {
  if (argc < 2) throw Usage("missing subcommand");
  Args a;
  a.cmd = argv[1];
  static const std::vector<std::string> flag_names = {"--optimize", "--help"};
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      if (std::find(flag_names.begin(), flag_names.end(), s) != flag_names.end()) {
        a.flags.push_back(s);
        continue;
      }
      std::string v;
      if (auto eq = s.find('='); eq != std::string::npos) {
        v = s.substr(eq + 1);
        s = s.substr(0, eq);
      } else {
        if (i + 1 >= argc) throw Usage("option " + s + " needs a value");
        v = argv[++i];
      }
      a.opt[s] = v;
    } else {
      a.positional.push_back(s);
    }
  }
  return a;
}

void allow(const Args& a, std::initializer_list<const char*> names, std::size_t max_positional) {
  for (const auto& [k, v] : a.opt)
    if (std::none_of(names.begin(), names.end(), [&](const char* n) { return k == n; }))
      throw Usage("unknown option " + k + " for " + a.cmd);
  for (const auto& f : a.flags)
    if (f != "--help" && std::none_of(names.begin(), names.end(), [&](const char* n) { return f == n; }))
      throw Usage("unknown flag " + f + " for " + a.cmd);
  if (a.positional.size() > max_positional) throw Usage("unexpected argument " + a.positional.back());
}

int to_int(const std::string& s, const char* what) {
  try {
    std::size_t pos = 0;
    const long long v = std::stoll(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return int(v);
  } catch (const std::exception&) {
    throw Usage(std::string("malformed ") + what + ": " + s);
  }
}

Extension extension_of(const std::string& s) {
  if (s == "periodic") return Extension::periodic;
  if (s == "symmetric") return Extension::symmetric;
  throw Usage("unknown extension: " + s + " (valid: periodic symmetric)");
}

int precision_of(const Args& a, const char* def, bool allow64 = true) {
  const int p = to_int(a.get("--precision", def), "precision");
  if (p != 32 && p != 64) throw Usage("precision must be 32 or 64");
  if (p == 64 && !allow64) throw Usage("bench: precision 64 is not timed (the float32 kernels are)");
  return p;
}

Scheme make_scheme(const std::string& wavelet, const std::string& id, bool optimize) {
  const WaveletSpec w = resolve_wavelet(wavelet);
  Scheme s = build_scheme(scheme_from_id(id), w);
  if (optimize) s = optimize_constant_split(s, w);
  return s;
}

int cmd_describe(const Args& a) {
  allow(a, {"--wavelet", "--scheme", "--optimize"}, 0);
  std::cout << describe(make_scheme(a.get("--wavelet", "cdf53"), a.get("--scheme", "separable-lifting"),
                                    a.has("--optimize")));
  return 0;
}

int cmd_count(const Args& a) {
  allow(a, {"--wavelet"}, 0);
  const WaveletSpec w = resolve_wavelet(a.get("--wavelet", "cdf53"));
  std::cout << "wavelet,scheme,variant,steps,operations\n";
  for (SchemeKind k : all_scheme_kinds()) {
    const Scheme base = build_scheme(k, w);
    const Scheme opt = optimize_constant_split(base, w);
    for (const Scheme* s : {&base, &opt})
      std::cout << w.name() << "," << scheme_id(k) << "," << (s->optimized ? "optimized" : "baseline") << ","
                << count_steps(*s) << "," << count_operations(*s) << "\n";
  }
  return 0;
}

// max |a - b| / max(|a|, |b|) over the compared region (equiv.cpp:123-137)
template <typename T>
double rel_dev(const PolyphaseImage<T>& a, const PolyphaseImage<T>& b, int margin) {
  double mx = 0, md = 0;
  const int w2 = a.comp_width(), h2 = a.comp_height();
  for (int c = 0; c < 4; ++c)
    for (int y = margin; y < h2 - margin; ++y)
      for (int x = margin; x < w2 - margin; ++x) {
        const double va = a.comp[c].at(x, y), vb = b.comp[c].at(x, y);
        mx = std::max({mx, std::abs(va), std::abs(vb)});
        md = std::max(md, std::abs(va - vb));
      }
  return md / std::max(mx, 1e-300);
}

template <typename T>
int equiv_at(const WaveletSpec& w, int size, int seed, const std::string& ext_s) {
  const Extension ext = extension_of(ext_s);
  const int margin = ext == Extension::symmetric ? 8 : 0;
  bool exact = true;  // equiv.cpp:34-38
  for (const auto& pr : w.pairs()) {
    for (const auto& t : pr.predict.terms()) exact = exact && t.c.is_exact();
    for (const auto& t : pr.update.terms()) exact = exact && t.c.is_exact();
  }
  const double tol = std::is_same_v<T, double> ? (exact ? 1e-12 : 1e-9) : 1e-5;
  const auto poly = polyphase_split(random_image<T>(size, size, std::uint64_t(seed)), ext);
  std::vector<std::pair<std::string, PolyphaseImage<T>>> outs;
  for (SchemeKind k : all_scheme_kinds()) {
    const Scheme base = build_scheme(k, w);
    const Scheme opt = optimize_constant_split(base, w);
    for (const Scheme* s : {&base, &opt}) {
      ExecPlan<T> plan = compile<T>(*s, ext, 1);
      outs.emplace_back(s->label, run(plan, poly));
    }
  }
  double worst = 0;
  std::string pair;
  for (std::size_t i = 0; i < outs.size(); ++i)
    for (std::size_t j = i + 1; j < outs.size(); ++j) {
      const double d = rel_dev(outs[i].second, outs[j].second, margin);
      if (d > worst) worst = d, pair = outs[i].first + " vs " + outs[j].first;
    }
  char buf[320];
  std::snprintf(buf, sizeof buf,
                "equivalence wavelet=%s size=%d seed=%d extension=%s variants=%zu margin=%d device=B200-float%d\n"
                "max relative deviation %.3e (tolerance %.0e)",
                w.name().c_str(), size, seed, ext_s.c_str(), outs.size(), margin,
                std::is_same_v<T, double> ? 64 : 32, worst, tol);
  std::cout << buf << (pair.empty() ? "" : " between " + pair) << (worst <= tol ? "\nPASS\n" : "\nFAIL\n");
  return worst <= tol ? 0 : 1;
}

int cmd_equiv(const Args& a) {
  allow(a, {"--wavelet", "--size", "--seed", "--extension", "--precision"}, 0);
  const WaveletSpec w = resolve_wavelet(a.get("--wavelet", "cdf53"));
  const int size = to_int(a.get("--size", "64"), "size");
  const int seed = to_int(a.get("--seed", "1"), "seed");
  const std::string ext_s = a.get("--extension", "periodic");
  extension_of(ext_s);
  if (size <= 0 || size % 2) throw Usage("equiv: size must be positive and even");
  return precision_of(a, "64") == 64 ? equiv_at<double>(w, size, seed, ext_s) : equiv_at<float>(w, size, seed, ext_s);
}

// transform_and_write (reference dwt2d.cpp:64-75), level after level
template <typename T>
void transform_levels(const ImagePlane<double>& img, const Scheme& s, Extension ext, int workers, int levels,
                      const std::filesystem::path& out) {
  ImagePlane<T> cur(img.width, img.height);
  for (std::size_t i = 0; i < img.samples.size(); ++i) cur.samples[i] = static_cast<T>(img.samples[i]);
  ExecPlan<T> plan = compile<T>(s, ext, workers);
  for (int l = 1; l <= levels; ++l) {
    const auto res = run(plan, polyphase_split(cur, ext));
    write_subbands(res, levels == 1 ? out : out / ("level" + std::to_string(l)));
    cur = res.comp[0];
  }
}

int cmd_transform(const Args& a) {
  allow(a, {"--out", "--wavelet", "--scheme", "--optimize", "--extension", "--precision", "--workers", "--levels"}, 1);
  if (a.positional.empty()) throw Usage("transform: missing input PGM");
  if (!a.opt.count("--out")) throw Usage("transform: --out is required");
  const int precision = precision_of(a, "64");  // the reference's default (dwt2d.cpp:121)
  const int workers = to_int(a.get("--workers", "1"), "workers");
  const int levels = to_int(a.get("--levels", "1"), "levels");
  if (levels < 1) throw Usage("levels must be at least 1");
  const Extension ext = extension_of(a.get("--extension", "periodic"));
  const Scheme s = make_scheme(a.get("--wavelet", "cdf53"), a.get("--scheme", "separable-lifting"),
                               a.has("--optimize"));
  const std::filesystem::path out = a.opt.at("--out");
  const ImagePlane<double> img = read_pgm(a.positional[0]);
  if (precision == 64)
    transform_levels<double>(img, s, ext, workers, levels, out);
  else
    transform_levels<float>(img, s, ext, workers, levels, out);
  std::cout << "wrote " << out.string() << (levels == 1 ? "" : "/level*") << "/{ee,oe,eo,oo}.raw: "
            << img.width / 2 << "x" << img.height / 2 << " per component, " << precision << "-bit, scheme "
            << s.label << ", wavelet " << s.wavelet << ", levels " << levels << ", device B200\n";
  return 0;
}

int cmd_bench(const Args& a) {
  allow(a, {"--wavelet", "--scheme", "--optimize", "--sizes", "--workers", "--repeats", "--precision", "--seed",
            "--extension", "--levels", "--out"},
        0);
  const int precision = precision_of(a, "32", false);
  const int workers = to_int(a.get("--workers", "1"), "workers");
  const int repeats = to_int(a.get("--repeats", "3"), "repeats");
  const int seed = to_int(a.get("--seed", "1"), "seed");
  const int levels = to_int(a.get("--levels", "1"), "levels");
  if (repeats < 3) throw Usage("bench: repeats must be at least 3");
  if (workers < 1) throw Usage("bench: workers must be at least 1");
  std::vector<int> sizes;
  {
    std::stringstream ss(a.get("--sizes", "256,512,1024,2048,4096"));
    for (std::string t; std::getline(ss, t, ',');) sizes.push_back(to_int(t, "size"));
  }
  if (sizes.empty()) throw Usage("bench: no sizes given");
  for (int sz : sizes)
    if (sz <= 0 || sz % 2) throw Usage("bench: sizes must be positive and even");
  const WaveletSpec w = resolve_wavelet(a.get("--wavelet", "cdf53"));
  const std::string which = a.get("--scheme", "all");
  std::vector<SchemeKind> kinds = which == "all" ? all_scheme_kinds() : std::vector<SchemeKind>{scheme_from_id(which)};
  const Extension ext = extension_of(a.get("--extension", "periodic"));
  std::ostringstream csv;
  csv << "scheme,wavelet,width,height,megapixels,precision,workers,seconds,throughput_gbps\n";
  for (SchemeKind k : kinds) {
    Scheme s = build_scheme(k, w);
    if (a.has("--optimize")) s = optimize_constant_split(s, w);
    ExecPlan<float> plan = compile<float>(s, ext, workers);
    for (int sz : sizes) {
      double secs = 0;
      detail::throw_status(dwt2d_time_forward(plan.handle.get(), sz, sz, levels, repeats, std::uint64_t(seed), &secs));
      double bytes = 0;
      for (int l = 0; l < levels; ++l) bytes += 2.0 * double(sz >> l) * double(sz >> l) * 4;
      char buf[256];
      std::snprintf(buf, sizeof buf, "%s,%s,%d,%d,%.3f,%d,%d,%.6f,%.3f\n",
                    (std::string(scheme_id(k)) + (a.has("--optimize") ? "-optimized" : "")).c_str(),
                    w.name().c_str(), sz, sz, double(sz) * sz / 1e6, precision, workers, secs,
                    bytes / std::max(secs, 1e-300) / 1e9);
      csv << buf;
    }
  }
  const std::string out = a.get("--out", "");
  if (out.empty()) {
    std::cout << csv.str();
  } else {
    std::ofstream f(out);
    if (!f) throw IoError("bench: cannot create " + out);
    f << csv.str();
    if (!f) throw IoError("bench: write failed: " + out);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.has("--help") || a.cmd == "--help" || a.cmd == "-h") {
      std::cout << kUsage;
      return 0;
    }
    if (a.cmd == "describe") return cmd_describe(a);
    if (a.cmd == "count") return cmd_count(a);
    if (a.cmd == "equiv") return cmd_equiv(a);
    if (a.cmd == "transform") return cmd_transform(a);
    if (a.cmd == "bench") return cmd_bench(a);
    throw Usage("unknown subcommand: " + a.cmd);
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n" << kUsage;
    return 2;
  } catch (const PgmError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::filesystem::filesystem_error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
