// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the
// product path. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load the library built from this
// file (oracle/_ref/libdwt2d_ref*.so).
//
// A thin C-export shim over the UNMODIFIED reference library, compiled from
// the reference's own sources under /root/reference/proj/src by
// oracle/Makefile. It exposes exactly the calls the parity tests need:
//   * the reference executor path  compile<T> -> run<T>
//     (/root/reference/proj/include/dwt2d/executor.hpp:52-103, :196-238)
//   * inverse_lifting<T>           (executor.hpp:242-248)
//   * the LCG image generator       (random.hpp:13-37)
//   * describe / count_steps / count_operations (src/scheme.cpp:380-454)
//   * the compiled float tap tables (executor.hpp:85-97) so the product's
//     own lowering can be checked tap-for-tap against the reference
//   * a Mallat multi-level loop over the reference API (SURVEY §8(a) A15:
//     level l runs the same plan on polyphase_split(LL_{l-1})).
// Nothing here re-implements the transform; every number comes from the
// reference's own code.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "dwt2d/executor.hpp"
#include "dwt2d/image.hpp"
#include "dwt2d/random.hpp"
#include "dwt2d/scheme.hpp"
#include "dwt2d/wavelet.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

dwt2d::Extension ext_of(int symmetric) {
  return symmetric ? dwt2d::Extension::symmetric : dwt2d::Extension::periodic;
}

dwt2d::Scheme make(const char* wavelet, const char* scheme, int optimized) {
  const dwt2d::WaveletSpec w = dwt2d::resolve_wavelet(wavelet);
  std::string id = scheme;
  if (id == "inverse-lifting") return dwt2d::build_inverse_lifting(w);
  dwt2d::Scheme s = dwt2d::build_scheme(dwt2d::scheme_from_id(id), w);
  if (optimized) s = dwt2d::optimize_constant_split(s, w);
  return s;
}

template <typename T>
dwt2d::PolyphaseImage<T> planes_in(const T* const in[4], int w2, int h2,
                                   dwt2d::Extension ext) {
  dwt2d::PolyphaseImage<T> p;
  p.extension = ext;
  for (int j = 0; j < 4; ++j) {
    p.comp[j] = dwt2d::ImagePlane<T>(w2, h2);
    std::memcpy(p.comp[j].samples.data(), in[j], sizeof(T) * size_t(w2) * h2);
  }
  return p;
}

template <typename T>
void planes_out(const dwt2d::PolyphaseImage<T>& p, T* const out[4]) {
  for (int j = 0; j < 4; ++j)
    std::memcpy(out[j], p.comp[j].samples.data(),
                sizeof(T) * p.comp[j].samples.size());
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Mallat layout of an L-level pyramid in a W x H plane: after level l the LL
// of size w x h in the top-left corner is replaced by its four bands,
// LL | HL on top, LH | HH below.
template <typename T>
void pyramid(const dwt2d::Scheme& s, dwt2d::Extension ext, int workers,
             const T* img, int W, int H, int levels, T* out) {
  std::memcpy(out, img, sizeof(T) * size_t(W) * H);
  int w = W, h = H;
  dwt2d::ExecPlan<T> plan = dwt2d::compile<T>(s, ext, workers);
  for (int l = 0; l < levels; ++l) {
    dwt2d::ImagePlane<T> ll(w, h);
    for (int y = 0; y < h; ++y)
      std::memcpy(ll.row(y), out + size_t(y) * W, sizeof(T) * w);
    const auto poly = dwt2d::polyphase_split(ll, ext);
    const auto res = dwt2d::run(plan, poly);
    const int w2 = w / 2, h2 = h / 2;
    for (int j = 0; j < 4; ++j) {
      const int ox = (j & 1) ? w2 : 0, oy = (j & 2) ? h2 : 0;
      for (int y = 0; y < h2; ++y)
        std::memcpy(out + size_t(oy + y) * W + ox, res.comp[j].row(y),
                    sizeof(T) * w2);
    }
    w = w2;
    h = h2;
  }
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// LCG image, random.hpp:31-37, T = float
REF_API int ref_random_image_f32(int w, int h, uint64_t seed, float* out) {
  return guarded([&] {
    const auto img = dwt2d::random_image<float>(w, h, seed);
    std::memcpy(out, img.samples.data(), sizeof(float) * img.samples.size());
  });
}

REF_API int ref_random_image_f64(int w, int h, uint64_t seed, double* out) {
  return guarded([&] {
    const auto img = dwt2d::random_image<double>(w, h, seed);
    std::memcpy(out, img.samples.data(), sizeof(double) * img.samples.size());
  });
}

// One reference run() over planar components (executor.hpp:196-238).
// scheme = a scheme id (scheme.cpp:41-56) or "inverse-lifting".
REF_API int ref_run_f32(const char* wavelet, const char* scheme, int optimized,
                        int symmetric, int workers, const float* const in[4],
                        int w2, int h2, float* const out[4],
                        long* barrier_count) {
  return guarded([&] {
    const auto s = make(wavelet, scheme, optimized);
    auto plan = dwt2d::compile<float>(s, ext_of(symmetric), workers);
    const auto res = dwt2d::run(plan, planes_in(in, w2, h2, ext_of(symmetric)));
    planes_out(res, out);
    if (barrier_count) *barrier_count = plan.barrier_count;
  });
}

REF_API int ref_run_f64(const char* wavelet, const char* scheme, int optimized,
                        int symmetric, int workers, const double* const in[4],
                        int w2, int h2, double* const out[4],
                        long* barrier_count) {
  return guarded([&] {
    const auto s = make(wavelet, scheme, optimized);
    auto plan = dwt2d::compile<double>(s, ext_of(symmetric), workers);
    const auto res = dwt2d::run(plan, planes_in(in, w2, h2, ext_of(symmetric)));
    planes_out(res, out);
    if (barrier_count) *barrier_count = plan.barrier_count;
  });
}

REF_API int ref_pyramid_f32(const char* wavelet, const char* scheme,
                            int optimized, int symmetric, int workers,
                            const float* img, int W, int H, int levels,
                            float* out) {
  return guarded([&] {
    pyramid<float>(make(wavelet, scheme, optimized), ext_of(symmetric), workers,
                   img, W, H, levels, out);
  });
}

REF_API int ref_pyramid_f64(const char* wavelet, const char* scheme,
                            int optimized, int symmetric, int workers,
                            const double* img, int W, int H, int levels,
                            double* out) {
  return guarded([&] {
    pyramid<double>(make(wavelet, scheme, optimized), ext_of(symmetric),
                    workers, img, W, H, levels, out);
  });
}

// Wall time (seconds) of `repeats` timed pyramid runs after one untimed
// warm-up, median, mirroring run_bench's method (src/bench.cpp:28-44).
REF_API int ref_time_pyramid_f32(const char* wavelet, const char* scheme,
                                 int optimized, int workers, const float* img,
                                 int W, int H, int levels, int repeats,
                                 float* out, double* seconds) {
  return guarded([&] {
    const auto s = make(wavelet, scheme, optimized);
    std::vector<double> t;
    for (int r = 0; r <= repeats; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      pyramid<float>(s, dwt2d::Extension::periodic, workers, img, W, H, levels,
                     out);
      const auto t1 = std::chrono::steady_clock::now();
      if (r > 0) t.push_back(std::chrono::duration<double>(t1 - t0).count());
    }
    std::sort(t.begin(), t.end());
    const size_t n = t.size();
    *seconds = n == 0 ? 0.0 : (n % 2 ? t[n / 2] : 0.5 * (t[n / 2 - 1] + t[n / 2]));
  });
}

REF_API int ref_describe(const char* wavelet, const char* scheme, int optimized,
                         char* buf, int buflen) {
  return guarded([&] {
    const std::string d = dwt2d::describe(make(wavelet, scheme, optimized));
    if (int(d.size()) + 1 > buflen) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, d.c_str(), d.size() + 1);
  });
}

REF_API int ref_count(const char* wavelet, const char* scheme, int optimized,
                      long* steps, long* ops) {
  return guarded([&] {
    const auto s = make(wavelet, scheme, optimized);
    *steps = long(dwt2d::count_steps(s));
    *ops = dwt2d::count_operations(s);
  });
}

// Flattened float tap tables of compile<float> (executor.hpp:52-103).
// Row record (per kernel k, output r): identity, scale, ntaps; followed by
// ntaps tap records (comp, dm, dn, w). Returns the number of floats written
// through *n_out; layout documented in oracle/ref.py.
REF_API int ref_taps_f32(const char* wavelet, const char* scheme, int optimized,
                         int symmetric, double* buf, int buflen, int* n_out) {
  return guarded([&] {
    const auto s = make(wavelet, scheme, optimized);
    const auto plan = dwt2d::compile<float>(s, ext_of(symmetric), 1);
    std::vector<double> v;
    v.push_back(double(plan.kernels.size()));
    for (const auto& k : plan.kernels)
      for (int r = 0; r < 4; ++r) {
        const auto& st = k.out[r];
        size_t nt = 0;
        for (int j = 0; j < 4; ++j) nt += st.taps[j].size();
        v.push_back(st.identity ? 1.0 : 0.0);
        v.push_back(double(st.scale));
        v.push_back(double(nt));
        for (int j = 0; j < 4; ++j)
          for (const auto& t : st.taps[j]) {
            v.push_back(j);
            v.push_back(t.dm);
            v.push_back(t.dn);
            v.push_back(double(t.w));
          }
      }
    if (int(v.size()) > buflen) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, v.data(), sizeof(double) * v.size());
    *n_out = int(v.size());
  });
}
