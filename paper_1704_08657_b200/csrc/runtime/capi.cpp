// C-ABI implementation (include/dwt2d_b200.h): plan creation from the host
// algebra, kernel selection by tap-table fingerprint, level launches and the
// Mallat multi-level driver. No CPU fallback exists: a program without a
// compiled kernel is rejected with DWT2D_EUNSUPPORTED.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dwt2d_b200.h"
#include "dwt2d_b200/image.hpp"
#include "dwt2d_b200/lowering.hpp"
#include "dwt2d_b200/schemes.hpp"
#include "../kernels/level_types.hpp"

using namespace dwt2d_b200;

// Run-time switches of a plan. Read from the DWT2D_* environment variables
// once, when the plan is created (tuning_from_env), and changeable per plan
// with dwt2d_plan_set_tuning (tests, sweeps); the launch path never reads the
// environment.
struct Tuning {
  int pdl = 1;              // DWT2D_PDL: programmatic dependent launch between levels
  int chunk_rows = 0;       // DWT2D_CHUNK_ROWS: rows per warp work item (0: policy)
  int alternate = 1;        // DWT2D_ALTERNATE: 0 off, 1 levels streaming from HBM, 2 every level
  int tma = 1;              // DWT2D_TMA: 0 off, 1 levels >= 512 MiB, 2 every stageable level
  int pair = 1;             // DWT2D_PAIR: 0 off, 1 where level 1 is staged, 2 forced
  int pair_chunk_rows = 0;  // DWT2D_PAIR_CHUNK_ROWS (0: policy)
  int crop_tiles = 2;       // DWT2D_CROP_TILES: symmetric border crops: 2 compiled crop kernel concurrent
                            // with the fused kernel, 1 one generic tile launch after it, 0 per sub-step
  int crop_core = 12;       // DWT2D_CROP_CORE: positions per crop tile (capped by the crop kernel's 256 cells)
  int host_band_rows = 0;   // DWT2D_HOST_BAND_ROWS: image rows per host pipeline band (0: policy)
  int host_levels = 0;      // DWT2D_HOST_LEVELS: levels pipelined by bands in the host entry point (0: policy)
  int host_taper = 0;       // DWT2D_HOST_TAPER: 1 = short first and last host pipeline bands
  int host_trace = 0;       // DWT2D_HOST_TRACE: 1 = print the host pipeline's timeline (development)
};

namespace {
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}
Tuning tuning_from_env() {
  Tuning t;
  t.pdl = env_int("DWT2D_PDL", t.pdl);
  t.chunk_rows = env_int("DWT2D_CHUNK_ROWS", t.chunk_rows);
  t.alternate = env_int("DWT2D_ALTERNATE", t.alternate);
  t.tma = env_int("DWT2D_TMA", t.tma);
  t.pair = env_int("DWT2D_PAIR", t.pair);
  t.pair_chunk_rows = env_int("DWT2D_PAIR_CHUNK_ROWS", t.pair_chunk_rows);
  t.crop_tiles = env_int("DWT2D_CROP_TILES", t.crop_tiles);
  t.crop_core = std::max(1, env_int("DWT2D_CROP_CORE", t.crop_core));
  t.host_band_rows = env_int("DWT2D_HOST_BAND_ROWS", t.host_band_rows);
  t.host_levels = env_int("DWT2D_HOST_LEVELS", t.host_levels);
  t.host_taper = env_int("DWT2D_HOST_TAPER", t.host_taper);
  t.host_trace = env_int("DWT2D_HOST_TRACE", t.host_trace);
  return t;
}
}  // namespace

constexpr int kMaxDevices = 64;

struct dwt2d_plan {
  std::string key;
  std::uint64_t fingerprint = 0;
  const gpu::PlanEntry* entry = nullptr;  // null => identity program (copy)
  int extension = DWT2D_PERIODIC;
  int forward = 1;
  int logical_steps = 0;
  int substeps = 0;
  long long operations = -1;
  long long taps_per_quad = 0;
  int left = 0, right = 0, up = 0, down = 0;
  int fma = 0;
  std::string description;
  std::vector<dwt2d_row> rows;
  std::vector<dwt2d_tap> taps;
  Tuning tune;
  // occupancy of the plan's vector level kernel and level-pair kernel
  // (resident CTAs per SM; 0 = not yet queried)
  mutable std::atomic<int> occ_level{0}, occ_pair{0};
  // generic executor (symmetric extension, programs without an AOT kernel):
  // tap tables in device memory, one copy per device the plan runs on
  bool generic = false;
  struct DeviceTables {
    gpu::TapDesc* taps = nullptr;
    gpu::RowDesc* rows = nullptr;
  };
  mutable std::mutex dev_mu;
  mutable DeviceTables dev[kMaxDevices];
  // float64 execution (compile<double>): double weights and row scales of
  // the same tables, uploaded per device on first use
  bool has64 = false;
  std::vector<double> w64, scale64;
  struct DeviceTables64 {
    gpu::TapDesc64* taps = nullptr;
  };
  mutable DeviceTables64 dev64[kMaxDevices];
  // rings of shards of dwt2d_forward_mallat_sharded, one per geometry
  struct ShardRing {
    std::vector<long long> key;
    std::vector<dwt2d_shard*> shards;
  };
  mutable std::mutex shard_mu;
  mutable std::vector<ShardRing> shard_cache;
  ~dwt2d_plan();
  void free_device_tables() {
    for (DeviceTables& d : dev) {
      if (d.taps) cudaFree(d.taps);
      if (d.rows) cudaFree(d.rows);
    }
    for (DeviceTables64& d : dev64)
      if (d.taps) cudaFree(d.taps);
  }
};

// One rank's share of a row-strip sharded forward pyramid:
// the exchange window its ring neighbours write halo rows into, the LL
// workspace, and the neighbours' windows once connected. Defined below.
struct dwt2d_shard;

namespace {

thread_local std::string g_error;
std::atomic<std::uint64_t> g_launches{0};

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw Fail{code, std::move(msg)}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? DWT2D_ENOMEM : DWT2D_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return DWT2D_OK;
  } catch (const Fail& e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return DWT2D_EINVAL;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return DWT2D_ENOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return DWT2D_EINVAL;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int current_device() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "current device");
  if (dev < 0 || dev >= kMaxDevices) fail(DWT2D_EUNSUPPORTED, "device ordinal beyond the supported range");
  return dev;
}

// SMs of the current device (cached per device)
int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = current_device();
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "SM count");
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

bool aligned(const void* p, size_t bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

// Rows per warp work item. A warp streams one strip of one chunk; the
// (up + down) rows around each chunk are re-read as warm-up. Measured on
// B200 (scripts/tune_level.cu, scripts/sweep_configs.py, bench.py): mid-size
// levels (one wave of resident warps covers them with <= 48-row chunks) run
// best as a single wave (4096^2 cold: 4.1 TB/s vs 3.6 with 5-row chunks);
// large levels run best with ~5 waves (16384^2: 6.1 TB/s with 64-row
// chunks vs 5.95 for one wave of 328-row chunks, whose concurrent accesses
// span the whole image; 8192^2 inside the pyramid: 106 us with 16-row
// chunks vs 113 us with one wave of 81-row chunks); tiny L2-resident levels
// want the most warps (2-row chunks).
// warps of the plan's vector level kernel that are resident at once
long long resident_warps(const dwt2d_plan& p) {
  int blocks = p.occ_level.load(std::memory_order_relaxed);
  if (blocks <= 0) {
    blocks = std::max(1, p.entry->occupancy ? p.entry->occupancy() : 2);
    p.occ_level.store(blocks, std::memory_order_relaxed);
  }
  return blocks * (long long)gpu::kWarpsPerCta * sm_count();
}

int chunk_rows_for(const dwt2d_plan& p, int h2, int nstrips) {
  if (p.tune.chunk_rows > 0) return p.tune.chunk_rows;
  const long long resident = resident_warps(p);
  const long long rows_total = (long long)h2 * std::max(1, nstrips);
  const long long per_warp = (rows_total + resident - 1) / resident;
  long long chunk = per_warp <= 48 ? std::max<long long>(2, per_warp)
                                   : (rows_total + 5 * resident - 1) / (5 * resident);
  return int(std::max<long long>(1, std::min<long long>(chunk, h2)));
}

enum Layout { kPlanar, kFromImage, kToImage };

// Work decomposition and vector-path eligibility of one level launch.
void prepare(const dwt2d_plan& p, gpu::LevelArgs& a, Layout layout, int chunk_override = 0) {
  if (a.w2 <= 0 || a.h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
  a.alternate = p.tune.alternate == 0 ? 0 : p.tune.alternate == 2 ? 2 : 1;  // 2: also single-wave levels (tests)
  a.pdl = p.tune.pdl ? 1 : 0;
  a.neg_zero = -0.0f;
  if (a.keep_x1 <= 0) a.keep_x0 = 0, a.keep_x1 = a.w2;
  if (a.keep_y1 <= 0) a.keep_y0 = 0, a.keep_y1 = a.h2;
  const gpu::PlanEntry& e = *p.entry;
  const int cw = e.cw;
  a.nstrips = (a.w2 + gpu::kOutLanes * cw - 1) / (gpu::kOutLanes * cw);
  // output rows covered by this launch: [y_begin, y_end) (a strip level's
  // interior or border rows), by default the whole level
  if (a.y_end <= 0) a.y_end = a.h2;
  if (a.y_begin < 0 || a.y_begin >= a.y_end || a.y_end > a.h2) fail(DWT2D_EINVAL, "level row range");
  const int span = a.y_end - a.y_begin;
  a.chunk_rows = chunk_override > 0 ? std::min(chunk_override, span) : chunk_rows_for(p, span, a.nstrips);
  // TMA-staged input rows (level_engine.cuh: TmaRowReader) for forward levels
  // of CW-4 programs (PlanEntry::stage_ok) that stream at least 512 MiB from
  // HBM: level 1 of 16384^2 346 vs 355 us, with ~10 waves of 32-row chunks
  // (64-row chunks: 364 us); non-separable polyconvolution opt. 404 vs 524
  // us, non-separable lifting baseline 411 vs 504 us. CW-2 programs (deep
  // convolution windows) were slower staged (separable convolution 722 vs
  // 470 us). Smaller levels keep register prefetch: there the stage set-up
  // per work item costs more than it hides (16384^2 pyramid levels 2..8 +16
  // us with staging, 4096^2 single levels +4..+80 us).
  {
    const size_t bytes = size_t(a.w2) * size_t(a.h2) * 16;
    const bool force = p.tune.tma == 2;
    const bool stageable = layout == kFromImage || (layout == kToImage && e.cw == 4);
    a.staged = stageable && p.tune.tma != 0 &&
               ((bytes >= (size_t(512) << 20) && e.stage_ok) || force) ? 1 : 0;
    if (a.staged && chunk_override <= 0 && p.tune.chunk_rows <= 0) {
      const long long resident = resident_warps(p);
      const long long rows_total = (long long)span * a.nstrips;
      a.chunk_rows = int(std::min<long long>(span, std::max<long long>(8, (rows_total + 10 * resident - 1) / (10 * resident))));
    }
  }
  a.nchunks = (span + a.chunk_rows - 1) / a.chunk_rows;
  // bottom-up odd chunks pay once the level streams from HBM (their shared
  // warm-up rows then meet in L2: 4096^2 single level 30.7 vs 32.8 us); a
  // level whose input (16 B per quad) fits comfortably in L2 streams
  // top-down (1024^2 round trip 27.7 vs 33.8 us)
  if (a.alternate == 1 && size_t(a.w2) * size_t(a.h2) * 16 < (size_t(32) << 20)) a.alternate = 0;
  bool vec = a.w2 % cw == 0;
  const bool in_il = layout == kFromImage, out_il = layout == kToImage;
  for (int j = 0; j < 4; ++j) {
    if (!in_il || j == 0) {
      const size_t al = in_il ? 16 : size_t(4 * cw);
      vec = vec && aligned(a.in[j], al) && (a.in_pitch[j] * 4) % al == 0;
      if (a.halo)
        vec = vec && aligned(a.halo_top[j], al) && aligned(a.halo_bot[j], al) &&
              (a.halo_top_pitch[j] * 4) % al == 0 && (a.halo_bot_pitch[j] * 4) % al == 0;
    }
    if (!out_il || j == 0) {
      const size_t al = out_il ? 16 : size_t(4 * cw);
      vec = vec && aligned(a.out[j], al) && (a.out_pitch[j] * 4) % al == 0;
    }
  }
  a.vec = vec ? 1 : 0;
  if (!a.vec) a.staged = 0;
}

void keep_pool_memory() {
  // stream-ordered allocations (workspaces, generic temporaries) are reused
  // instead of being unmapped at every synchronisation
  static std::atomic<bool> done[kMaxDevices];
  const int dev = current_device();
  if (done[dev].exchange(true)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
}

// The plan's tap and row tables on the current device (uploaded on first use
// per device).
const dwt2d_plan::DeviceTables& device_tables(const dwt2d_plan& p) {
  const int devno = current_device();
  std::lock_guard<std::mutex> lk(p.dev_mu);
  dwt2d_plan::DeviceTables& dt = p.dev[devno];
  if (!dt.taps) {
    std::vector<gpu::TapDesc> t;
    for (const dwt2d_tap& k : p.taps) t.push_back(gpu::TapDesc{k.comp, k.dm, k.dn, k.w});
    if (t.empty()) t.push_back(gpu::TapDesc{0, 0, 0, 0.0f});
    gpu::TapDesc* d = nullptr;
    cuda_check(cudaMalloc(&d, t.size() * sizeof(gpu::TapDesc)), "tap table allocation");
    cuda_check(cudaMemcpy(d, t.data(), t.size() * sizeof(gpu::TapDesc), cudaMemcpyHostToDevice), "tap table upload");
    std::vector<gpu::RowDesc> r;
    for (const dwt2d_row& row : p.rows) r.push_back(gpu::RowDesc{row.identity, row.tap_begin, row.tap_end, row.scale});
    if (r.empty()) r.push_back(gpu::RowDesc{1, 0, 0, 1.0f});
    gpu::RowDesc* dr = nullptr;
    cuda_check(cudaMalloc(&dr, r.size() * sizeof(gpu::RowDesc)), "row table allocation");
    cuda_check(cudaMemcpy(dr, r.data(), r.size() * sizeof(gpu::RowDesc), cudaMemcpyHostToDevice), "row table upload");
    dt.taps = d, dt.rows = dr;
  }
  return dt;
}

size_t ws_align(size_t floats) { return (floats + 63) & ~size_t(63); }

// A sub-grid of a level for the generic executor: the crop [x0, x0 + w) x
// [y0, y0 + h) of the component grid is transformed as if it were the whole
// image (extension at the crop's edges); only outputs inside the keep window
// (crop coordinates) are written.
struct Region {
  int x0, y0, w, h;
  int kx0, kx1, ky0, ky1;
};

// One level on the generic executor: sub-step s reads the previous
// sub-step's planes (double-buffered temporaries per region), like the
// reference's run(); all regions of a sub-step go in one launch.
// A per-thread, per-device side stream and fork/join events (symmetric
// border crops overlap the fused kernel).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  static thread_local SideStream per_dev[kMaxDevices];
  SideStream& ss = per_dev[current_device()];
  if (!ss.s) {
    cuda_check(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking), "side stream");
    cuda_check(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming), "fork event");
    cuda_check(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming), "join event");
  }
  return ss;
}

// `mid`, if given, is launched on `st` concurrently with sub-steps
// 0 .. S-2 (which then run on a side stream); the last sub-step (the only one
// that writes the level's outputs) follows both on `st`.
void run_generic_regions(const dwt2d_plan& p, const gpu::LevelArgs& a, Layout layout,
                         const std::vector<Region>& regions, cudaStream_t st,
                         const std::function<void()>* mid = nullptr) {
  if (a.halo) fail(DWT2D_EUNSUPPORTED, "row strips need a fused kernel (periodic built-in program)");
  if (regions.empty() || int(regions.size()) > gpu::kMaxGenericRegions) fail(DWT2D_EINVAL, "generic regions");
  keep_pool_memory();
  const gpu::TapDesc* taps = device_tables(p).taps;
  const int S = p.substeps;
  const int n = int(regions.size());
  std::vector<size_t> off(n + 1, 0);  // per region: 2 buffers x 4 planes
  for (int i = 0; i < n; ++i) off[i + 1] = off[i] + ws_align(size_t(regions[i].w) * size_t(regions[i].h)) * 8;
  float* tmp = nullptr;
  if (S > 1) {
    void* m = nullptr;
    cuda_check(cudaMallocAsync(&m, off[n] * sizeof(float), st), "generic temporaries");
    tmp = static_cast<float*>(m);
  }
  std::vector<gpu::GenericStepArgs> g(n);
  SideStream* side = nullptr;
  if (mid && S > 1) {
    side = &side_stream();
    cuda_check(cudaEventRecord(side->fork, st), "fork");
    cuda_check(cudaStreamWaitEvent(side->s, side->fork, 0), "fork");
  } else if (mid) {
    (*mid)();
  }
  for (int s = 0; s < S; ++s) {
    const bool first = s == 0, last = s == S - 1;
    cudaStream_t ss = st;
    if (side && !last) ss = side->s;
    if (side && last) {  // join: the fused kernel on `st`, the crops' earlier sub-steps on the side stream
      (*mid)();
      cuda_check(cudaEventRecord(side->join, side->s), "join");
      cuda_check(cudaStreamWaitEvent(st, side->join, 0), "join");
    }
    for (int i = 0; i < n; ++i) {
      const Region& r = regions[i];
      const size_t plane = ws_align(size_t(r.w) * size_t(r.h));
      float* src_tmp = tmp ? tmp + off[i] + size_t((s + 1) % 2) * 4 * plane : nullptr;
      float* dst_tmp = tmp ? tmp + off[i] + size_t(s % 2) * 4 * plane : nullptr;
      gpu::GenericStepArgs& q = g[i];
      q = gpu::GenericStepArgs{};
      for (int j = 0; j < 4; ++j) {
        if (first) {
          q.in[j] = layout == kFromImage
                        ? a.in[0] + 2ll * r.y0 * a.in_pitch[0] + 2ll * r.x0
                        : a.in[j] + (long long)r.y0 * a.in_pitch[j] + r.x0;
          q.in_pitch[j] = a.in_pitch[layout == kFromImage ? 0 : j];
        } else {
          q.in[j] = src_tmp + j * plane;
          q.in_pitch[j] = r.w;
        }
        if (last) {
          q.out[j] = layout == kToImage ? a.out[0] + 2ll * r.y0 * a.out_pitch[0] + 2ll * r.x0
                                        : a.out[j] + (long long)r.y0 * a.out_pitch[j] + r.x0;
          q.out_pitch[j] = a.out_pitch[layout == kToImage ? 0 : j];
        } else {
          q.out[j] = dst_tmp + j * plane;
          q.out_pitch[j] = r.w;
        }
        const dwt2d_row& row = p.rows[size_t(s) * 4 + j];
        q.rows[j] = gpu::RowDesc{row.identity, row.tap_begin, row.tap_end, row.scale};
      }
      q.in_il = first && layout == kFromImage;
      q.out_il = last && layout == kToImage;
      q.w2 = r.w, q.h2 = r.h;
      q.symmetric = p.extension == DWT2D_SYMMETRIC;
      q.fma = p.fma;
      if (last)
        q.kx0 = r.kx0, q.kx1 = r.kx1, q.ky0 = r.ky0, q.ky1 = r.ky1;
      else
        q.kx0 = 0, q.kx1 = r.w, q.ky0 = 0, q.ky1 = r.h;
      q.taps = taps;
    }
    cuda_check(gpu::launch_generic_step(g.data(), n, p.tune.pdl != 0, ss), "generic step launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (tmp) cuda_check(cudaFreeAsync(tmp, st), "generic temporaries");
}

void run_generic(const dwt2d_plan& p, const gpu::LevelArgs& a, Layout layout, cudaStream_t st) {
  run_generic_regions(p, a, layout, {Region{0, 0, a.w2, a.h2, 0, a.w2, 0, a.h2}}, st);
}

void launch_fused(const dwt2d_plan& p, gpu::LevelArgs a, Layout layout, cudaStream_t st);

// float64 tap table of the plan on the current device
const gpu::TapDesc64* device_taps64(const dwt2d_plan& p) {
  if (!p.has64) fail(DWT2D_EUNSUPPORTED, "plan has no float64 tables (create it with float64 weights)");
  const int devno = current_device();
  std::lock_guard<std::mutex> lk(p.dev_mu);
  dwt2d_plan::DeviceTables64& dt = p.dev64[devno];
  if (!dt.taps) {
    std::vector<gpu::TapDesc64> t;
    for (size_t i = 0; i < p.taps.size(); ++i) t.push_back(gpu::TapDesc64{p.taps[i].comp, p.taps[i].dm, p.taps[i].dn, p.w64[i]});
    if (t.empty()) t.push_back(gpu::TapDesc64{0, 0, 0, 0.0});
    gpu::TapDesc64* d = nullptr;
    cuda_check(cudaMalloc(&d, t.size() * sizeof(gpu::TapDesc64)), "tap table allocation");
    cuda_check(cudaMemcpy(d, t.data(), t.size() * sizeof(gpu::TapDesc64), cudaMemcpyHostToDevice), "tap table upload");
    dt.taps = d;
  }
  return dt.taps;
}

// One level in float64 (compile<double> + run<double>): one generic pass
// per sub-step over double planes, double-buffered temporaries from the
// stream-ordered allocator (the reference's run() loop, executor.hpp:196-238).
struct Level64 {
  const double* in[4];
  size_t in_pitch[4];
  double* out[4];
  size_t out_pitch[4];
};
void run_level64(const dwt2d_plan& p, const Level64& lv, Layout layout, int w2, int h2, cudaStream_t st) {
  if (w2 <= 0 || h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
  const gpu::TapDesc64* taps = device_taps64(p);
  const int S = p.substeps;
  const size_t plane = ws_align(size_t(w2) * size_t(h2));
  double* tmp = nullptr;
  if (S > 1) {
    void* m = nullptr;
    cuda_check(cudaMallocAsync(&m, 8 * plane * sizeof(double), st), "float64 temporaries");
    tmp = static_cast<double*>(m);
  }
  for (int s = 0; s < S; ++s) {
    const bool first = s == 0, last = s == S - 1;
    double* src_tmp = tmp ? tmp + size_t((s + 1) % 2) * 4 * plane : nullptr;
    double* dst_tmp = tmp ? tmp + size_t(s % 2) * 4 * plane : nullptr;
    gpu::GenericStepArgs64 q{};
    for (int j = 0; j < 4; ++j) {
      if (first) {
        q.in[j] = lv.in[layout == kFromImage ? 0 : j];
        q.in_pitch[j] = (long long)lv.in_pitch[layout == kFromImage ? 0 : j];
      } else {
        q.in[j] = src_tmp + j * plane;
        q.in_pitch[j] = w2;
      }
      if (last) {
        q.out[j] = lv.out[layout == kToImage ? 0 : j];
        q.out_pitch[j] = (long long)lv.out_pitch[layout == kToImage ? 0 : j];
      } else {
        q.out[j] = dst_tmp + j * plane;
        q.out_pitch[j] = w2;
      }
      const dwt2d_row& row = p.rows[size_t(s) * 4 + j];
      q.rows[j] = gpu::RowDesc64{row.identity, row.tap_begin, row.tap_end, p.scale64[size_t(s) * 4 + j]};
    }
    q.in_il = first && layout == kFromImage;
    q.out_il = last && layout == kToImage;
    q.w2 = w2, q.h2 = h2;
    q.symmetric = p.extension == DWT2D_SYMMETRIC;
    q.fma = p.fma;
    q.kx0 = 0, q.kx1 = w2, q.ky0 = 0, q.ky1 = h2;
    q.taps = taps;
    cuda_check(gpu::launch_generic_step64(q, st), "float64 step launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (tmp) cuda_check(cudaFreeAsync(tmp, st), "float64 temporaries");
}

void copy_planes64(const double* const in[4], const size_t in_pitch[4], double* const out[4],
                   const size_t out_pitch[4], int w2, int h2, cudaStream_t st) {
  for (int j = 0; j < 4; ++j)
    cuda_check(cudaMemcpy2DAsync(out[j], out_pitch[j] * 8, in[j], in_pitch[j] * 8, size_t(w2) * 8, h2,
                                 cudaMemcpyDeviceToDevice, st),
               "copy");
}

// Symmetric extension with a fused kernel. The extension
// only matters for outputs whose dependency cone — the level's reach, up/down
// rows and left/right columns over all sub-steps — crosses the image edge;
// everywhere else the fused single-pass kernel (periodic input rule) computes
// the same taps in the same order, i.e. the same bits as the per-step
// symmetric executor. So: the fused kernel over the whole level, then the
// four border bands recomputed by the generic executor on crops that contain
// the true image edge plus a margin (a cone that reflects at the true edge
// reaches at most up + down rows, resp. left + right columns, into the crop;
// the margin keeps the crop's artificial inner edge out of every kept
// cone). Levels too small for the crops run wholly on the generic executor.
// Core positions per crop-kernel tile: the tile area (core + margins along
// the band, `across` cells across it) and its ghost ring hold at most
// kCropThreads cells, one per thread. 0: the band is too wide for the kernel.
int crop_core_for(const dwt2d_plan& p, int margins, int across, int along_max) {
  const int r = p.entry->crop_reach;
  int core = std::min(p.tune.crop_core, gpu::kCropThreads / std::max(1, across) - margins);
  core = std::min(core, along_max);
  while (core >= 1) {
    const int along = std::min(along_max, core + margins);
    if (along * across <= gpu::kCropThreads && gpu::crop_ring_cells(along, across, r) <= gpu::kCropThreads) break;
    --core;
  }
  return std::max(core, 0);
}

// The compiled form (crop_engine.cuh): the fused kernel stores the interior
// only (keep window: rows [up, h2 - down), columns widened to whole lanes),
// the crop kernel the four border bands around it, on a side stream at the
// same time (disjoint outputs, both read only the level input).
// Crop geometry of the compiled kernel. Its ghost cells are filled only at
// true image edges, so garbage enters a tile only through its other edges
// and spreads at most the level's cumulative reach: a kept row r < up of the
// top band reads rows <= r + down, so up + down + 2 rows suffice (the
// generic crops, which reflect at the crop's inner edge too, take twice the
// reach + 4), the side bands their lane-aligned kept columns plus the reach
// + 2, and tiles along a band a margin of the reach + 1.
struct CropGeometry {
  int my, mx, kl, kr, margin;
};
CropGeometry crop_geometry(const dwt2d_plan& p) {
  const int cw = p.entry->cw;
  CropGeometry g;
  g.kl = (p.left + cw - 1) / cw * cw, g.kr = (p.right + cw - 1) / cw * cw;  // lane-aligned side bands
  g.my = p.up + p.down + 2;
  g.mx = std::max(g.kl, g.kr) + std::max(p.left, p.right) + 2;
  g.margin = std::max(std::max(p.left, p.right), std::max(p.up, p.down)) + 1;
  return g;
}

void run_symmetric_compiled(const dwt2d_plan& p, const gpu::LevelArgs& a, Layout layout, cudaStream_t st) {
  const int w2 = a.w2, h2 = a.h2;
  const CropGeometry cg = crop_geometry(p);
  const int my = cg.my, mx = cg.mx, kl = cg.kl, kr = cg.kr;
  gpu::CropTileArgs t{};
  for (int j = 0; j < 4; ++j) {
    t.in[j] = a.in[j], t.in_pitch[j] = a.in_pitch[j];
    t.out[j] = a.out[j], t.out_pitch[j] = a.out_pitch[j];
  }
  t.in_il = layout == kFromImage, t.out_il = layout == kToImage;
  t.w2 = w2, t.h2 = h2;
  t.mlo = t.mhi = cg.margin;
  t.core = crop_core_for(p, t.mlo + t.mhi, std::max(my, mx), std::max(w2, h2));
  const int tx = (w2 + t.core - 1) / t.core, ty = (h2 + t.core - 1) / t.core;
  t.nreg = 4;
  t.reg[0] = gpu::CropRegion{0, 0, w2, my, 0, w2, 0, p.up, 1, tx};
  t.reg[1] = gpu::CropRegion{0, h2 - my, w2, my, 0, w2, my - p.down, my, 1, tx};
  t.reg[2] = gpu::CropRegion{0, 0, mx, h2, 0, kl, p.up, h2 - p.down, 0, ty};
  t.reg[3] = gpu::CropRegion{w2 - mx, 0, mx, h2, mx - kr, mx, p.up, h2 - p.down, 0, ty};
  const int along = std::min(std::max(w2, h2), t.core + t.mlo + t.mhi), across = std::max(my, mx);
  gpu::LevelArgs in = a;
  in.keep_x0 = kl, in.keep_x1 = w2 - kr, in.keep_y0 = p.up, in.keep_y1 = h2 - p.down;
  // Large levels: the crops on a side stream, fully concurrent with the fused
  // kernel's waves. Smaller levels, where a fork/join costs as much as the
  // level: one stream, crop kernel first, the fused kernel launched behind it
  // by PDL with its wait at the end (wait_end), so the two overlap and the
  // PDL chain to the next level stays intact.
  if (!p.tune.pdl || size_t(w2) * size_t(h2) * 16 >= (size_t(256) << 20)) {
    SideStream& side = side_stream();
    cuda_check(cudaEventRecord(side.fork, st), "fork");
    cuda_check(cudaStreamWaitEvent(side.s, side.fork, 0), "fork");
    cuda_check(p.entry->crop(t, along, across, false, side.s), "crop kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    launch_fused(p, in, layout, st);
    cuda_check(cudaEventRecord(side.join, side.s), "join");
    cuda_check(cudaStreamWaitEvent(st, side.join, 0), "join");
    return;
  }
  cuda_check(p.entry->crop(t, along, across, true, st), "crop kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  in.wait_end = 1;
  launch_fused(p, in, layout, st);
}

// A level too small for four border bands: the crop kernel takes all of it
// (one region, every side a true image edge), tiled along its longer side.
void run_symmetric_small(const dwt2d_plan& p, const gpu::LevelArgs& a, Layout layout, cudaStream_t st) {
  gpu::CropTileArgs t{};
  for (int j = 0; j < 4; ++j) {
    t.in[j] = a.in[j], t.in_pitch[j] = a.in_pitch[j];
    t.out[j] = a.out[j], t.out_pitch[j] = a.out_pitch[j];
  }
  t.in_il = layout == kFromImage, t.out_il = layout == kToImage;
  t.w2 = a.w2, t.h2 = a.h2;
  t.mlo = t.mhi = crop_geometry(p).margin;
  const bool along_x = a.w2 >= a.h2;
  const int n = along_x ? a.w2 : a.h2;
  t.core = crop_core_for(p, t.mlo + t.mhi, along_x ? a.h2 : a.w2, n);
  t.nreg = 1;
  t.reg[0] = gpu::CropRegion{0, 0, a.w2, a.h2, 0, a.w2, 0, a.h2, along_x ? 1 : 0, (n + t.core - 1) / t.core};
  const int along = std::min(n, t.core + t.mlo + t.mhi), across = along_x ? a.h2 : a.w2;
  cuda_check(p.entry->crop(t, along_x ? along : across, along_x ? across : along, p.tune.pdl != 0, st),
             "crop kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void run_symmetric(const dwt2d_plan& p, const gpu::LevelArgs& a, Layout layout, cudaStream_t st) {
  const int my = 2 * (p.up + p.down) + 4, mx = 2 * (p.left + p.right) + 4;
  const bool compiled = p.tune.crop_tiles == 2 && p.entry->crop;
  if (compiled) {
    const CropGeometry cg = crop_geometry(p);
    if (a.h2 < 2 * cg.my || a.w2 < 2 * cg.mx) {
      if (crop_core_for(p, 2 * cg.margin, std::min(a.w2, a.h2), std::max(a.w2, a.h2)) > 0)
        return run_symmetric_small(p, a, layout, st);
      return run_generic(p, a, layout, st);
    }
    if (crop_core_for(p, 2 * cg.margin, std::max(cg.my, cg.mx), std::max(a.w2, a.h2)) > 0)
      return run_symmetric_compiled(p, a, layout, st);
  }
  if (a.h2 < 2 * my || a.w2 < 2 * mx) return run_generic(p, a, layout, st);
  const int w2 = a.w2, h2 = a.h2;
  if (!p.tune.crop_tiles) {  // one generic launch per sub-step over the four crops
    // the crops' intermediate sub-steps run on a side stream while the fused
    // kernel covers the level; their last sub-step overwrites the border
    // bands after it
    const std::function<void()> fused = [&] { launch_fused(p, a, layout, st); };
    run_generic_regions(p, a, layout,
                        {Region{0, 0, w2, my, 0, w2, 0, p.up},
                         Region{0, h2 - my, w2, my, 0, w2, my - p.down, my},
                         Region{0, 0, mx, h2, 0, p.left, 0, h2},
                         Region{w2 - mx, 0, mx, h2, mx - p.right, mx, 0, h2}},
                        st, &fused);
    return;
  }
  // all sub-steps of the four crops in one launch (crop_tile_kernel): tiles of
  // 8 positions along each crop's long side plus margins of the program's
  // cumulative reach, whose values only the discarded margins depend on
  // (measured: 16384^2 symmetric pyramid 0.96 ms with 8-position tiles,
  // 1.12 ms with 4; 4096^2 level 92 us; the per-sub-step launches: 1.22 ms /
  // 133 us; scripts/probe_symmetric.py)
  launch_fused(p, a, layout, st);
  gpu::CropTileArgs t{};
  for (int j = 0; j < 4; ++j) {
    t.in[j] = a.in[j], t.in_pitch[j] = a.in_pitch[j];
    t.out[j] = a.out[j], t.out_pitch[j] = a.out_pitch[j];
  }
  t.in_il = layout == kFromImage, t.out_il = layout == kToImage;
  t.nsteps = p.substeps, t.symmetric = 1, t.fma = p.fma;
  t.core = std::max(1, p.tune.crop_core);
  // margins: the cumulative reach toward the tile edge, plus the distance a
  // reflection at a crop edge folds back (a reflected read near the far edge
  // of a short last tile lands up to up+down positions inside)
  t.mlo = t.mhi = std::max(p.left + p.right, p.up + p.down);
  const int tx = (w2 + t.core - 1) / t.core, ty = (h2 + t.core - 1) / t.core;
  t.nreg = 4;
  t.reg[0] = gpu::CropRegion{0, 0, w2, my, 0, w2, 0, p.up, 1, tx};
  t.reg[1] = gpu::CropRegion{0, h2 - my, w2, my, 0, w2, my - p.down, my, 1, tx};
  t.reg[2] = gpu::CropRegion{0, 0, mx, h2, 0, p.left, 0, h2, 0, ty};
  t.reg[3] = gpu::CropRegion{w2 - mx, 0, mx, h2, mx - p.right, mx, 0, h2, 0, ty};
  const dwt2d_plan::DeviceTables& dt = device_tables(p);
  t.taps = dt.taps;
  t.rows = dt.rows;
  const int span = t.core + t.mlo + t.mhi;
  const int smem_floats = 2 * 4 * std::max(my, mx) * span;
  cuda_check(gpu::launch_crop_tiles(t, smem_floats, p.tune.pdl != 0, st), "crop tile kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch(const dwt2d_plan& p, gpu::LevelArgs a, Layout layout, cudaStream_t st) {
  if (!p.generic && p.extension == DWT2D_SYMMETRIC) {
    if (a.w2 <= 0 || a.h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    if (a.halo) fail(DWT2D_EUNSUPPORTED, "row strips need periodic extension");
    return run_symmetric(p, a, layout, st);
  }
  launch_fused(p, a, layout, st);
}

void launch_fused(const dwt2d_plan& p, gpu::LevelArgs a, Layout layout, cudaStream_t st) {
  if (p.generic) {
    if (a.w2 <= 0 || a.h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    if (layout != kPlanar && (layout == kToImage) == (p.forward != 0))
      fail(DWT2D_EINVAL, layout == kToImage ? "inverse_level: plan is not an inverse plan"
                                            : "forward_level: plan is an inverse plan");
    return run_generic(p, a, layout, st);
  }
  prepare(p, a, layout);
  const gpu::PlanEntry& e = *p.entry;
  gpu::LevelLaunch fn = layout == kPlanar ? e.planar : layout == kFromImage ? e.from_image : e.to_image;
  if (!fn)
    fail(DWT2D_EINVAL, layout == kToImage ? "inverse_level: plan is not an inverse plan"
                                          : "forward_level: plan is an inverse plan");
  cuda_check(fn(a, st), "level kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

bool is_identity(const dwt2d_plan& p) { return !p.entry && !p.generic; }

void require_plan(const dwt2d_plan* p) {
  if (!p) fail(DWT2D_EINVAL, "null plan");
}

void finalize_plan(dwt2d_plan& p, const StepProgram& prog, int extension) {
  p.key = prog.key;
  p.fingerprint = prog.fingerprint();
  p.logical_steps = int(prog.logical_steps);
  p.substeps = int(prog.steps.size());
  p.taps_per_quad = prog.taps_per_quad();
  p.left = prog.left, p.right = prog.right, p.up = prog.up, p.down = prog.down;
  p.extension = extension;
  p.fma = prog.fused_multiply_add ? 1 : 0;
  p.tune = tuning_from_env();
  p.rows.clear(), p.taps.clear(), p.w64.clear(), p.scale64.clear();
  for (const KernelStep& st : prog.steps)
    for (const KernelRow& r : st.rows) {
      dwt2d_row row{};
      row.identity = r.identity;
      row.scale = r.scale;
      row.tap_begin = int32_t(p.taps.size());
      for (const KernelTap& k : r.taps) {
        p.taps.push_back(dwt2d_tap{k.comp, k.dm, k.dn, k.w});
        p.w64.push_back(k.coef);
      }
      row.tap_end = int32_t(p.taps.size());
      p.rows.push_back(row);
      p.scale64.push_back(r.scale64);
    }
  bool identity = true;
  for (const KernelStep& st : prog.steps)
    for (const KernelRow& r : st.rows) identity = identity && r.identity;
  if (identity) return;  // pure copy, no kernel (pairless wavelet)
  // the fused single-pass kernels cover the built-in programs (symmetric
  // extension: plus border crops on the generic executor, run_symmetric);
  // everything else runs on the generic GPU executor (one pass per sub-step,
  // kernels/generic_step.cu)
  const char* force = std::getenv("DWT2D_FORCE_GENERIC");  // testing: bypass the fused kernels
  const bool fused_ok = !(force && *force && *force != '0');
  p.entry = fused_ok ? gpu::find_plan(p.fingerprint) : nullptr;
  p.generic = p.entry == nullptr;
}

StepProgram program_from_tables(const dwt2d_program& t) {
  if (t.nsteps < 0 || t.ntaps < 0 || (t.nsteps && !t.rows) || (t.ntaps && !t.taps))
    fail(DWT2D_EINVAL, "malformed program tables");
  StepProgram p;
  p.key = "program";
  p.logical_steps = t.logical_steps;
  p.fused_multiply_add = t.fused_multiply_add != 0;
  for (int s = 0; s < t.nsteps; ++s) {
    KernelStep st;
    for (int r = 0; r < 4; ++r) {
      const dwt2d_row& row = t.rows[s * 4 + r];
      KernelRow& kr = st.rows[r];
      kr.identity = row.identity != 0;
      kr.scale = row.scale;
      kr.scale64 = t.scales64 ? t.scales64[s * 4 + r] : row.scale;
      if (row.tap_begin < 0 || row.tap_end > t.ntaps || row.tap_begin > row.tap_end)
        fail(DWT2D_EINVAL, "malformed program tap range");
      for (int i = row.tap_begin; i < row.tap_end; ++i) {
        const dwt2d_tap& tp = t.taps[i];
        if (tp.comp < 0 || tp.comp > 3) fail(DWT2D_EINVAL, "malformed program tap component");
        KernelTap k;
        k.comp = tp.comp, k.dm = tp.dm, k.dn = tp.dn, k.w = tp.w, k.coef = t.weights64 ? t.weights64[i] : tp.w;
        kr.taps.push_back(k);
        st.min_dm = std::min(st.min_dm, k.dm), st.max_dm = std::max(st.max_dm, k.dm);
        st.min_dn = std::min(st.min_dn, k.dn), st.max_dn = std::max(st.max_dn, k.dn);
      }
    }
    p.steps.push_back(st);
  }
  for (const KernelStep& st : p.steps) {
    p.left -= st.min_dm, p.right += st.max_dm, p.up -= st.min_dn, p.down += st.max_dn;
  }
  return p;
}

void copy_planes(const float* const in[4], const size_t in_pitch[4], float* const out[4],
                 const size_t out_pitch[4], int w2, int h2, cudaStream_t st) {
  for (int j = 0; j < 4; ++j)
    cuda_check(cudaMemcpy2DAsync(out[j], out_pitch[j] * 4, in[j], in_pitch[j] * 4, size_t(w2) * 4, h2,
                                 cudaMemcpyDeviceToDevice, st),
               "copy");
}

void check_pyramid(int W, int H, int levels) {
  if (W <= 0 || H <= 0) fail(DWT2D_EINVAL, "pyramid: empty image");
  if (levels < 1) fail(DWT2D_EINVAL, "pyramid: levels must be at least 1");
  if (levels > 30 || (W % (1 << levels)) || (H % (1 << levels)))
    fail(DWT2D_EINVAL, "pyramid: width and height must be divisible by 2^levels");
}

// Workspace layout (dwt2d_workspace_bytes): the intermediate LL band of every
// level k = 1 .. levels-1 in its own slot.
size_t ll_offset(int W, int H, int k) {
  size_t off = 0;
  for (int i = 1; i < k; ++i) off += ws_align(size_t(W >> i) * size_t(H >> i));
  return off;
}
float* ll_slot(float* ws, int W, int H, int k) { return ws + ll_offset(W, H, k); }

struct Workspace {
  float* ptr = nullptr;
  bool owned = false;
  cudaStream_t st = nullptr;
  void release() {
    if (owned && ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr, owned = false;
  }
  ~Workspace() { release(); }
};

void get_workspace(Workspace& w, void* scratch, int W, int H, int levels, cudaStream_t st) {
  const size_t bytes = dwt2d_workspace_bytes(W, H, levels);
  w.st = st;
  if (scratch || bytes == 0) {
    w.ptr = static_cast<float*>(scratch);
    return;
  }
  void* p = nullptr;
  cuda_check(cudaMallocAsync(&p, bytes, st), "workspace allocation");
  w.ptr = static_cast<float*>(p);
  w.owned = true;
}

void record(void* ev, cudaStream_t st) {
  if (!ev) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(st, &cs), "capture status");
  const unsigned flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  cuda_check(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), st, flags), "event record");
}

void fill_forward_level(gpu::LevelArgs& a, const float* cur, size_t cur_pitch, float* ll, size_t ll_pitch,
                        float* out, size_t out_pitch, int w2, int h2) {
  a = gpu::LevelArgs{};
  a.in[0] = a.in[1] = a.in[2] = a.in[3] = cur;
  for (int j = 0; j < 4; ++j) a.in_pitch[j] = (long long)cur_pitch;
  a.out[0] = ll;
  a.out_pitch[0] = (long long)ll_pitch;
  a.out[1] = out + w2;
  a.out[2] = out + size_t(h2) * out_pitch;
  a.out[3] = out + size_t(h2) * out_pitch + w2;
  a.out_pitch[1] = a.out_pitch[2] = a.out_pitch[3] = (long long)out_pitch;
  a.w2 = w2, a.h2 = h2;
}

// Chunking and launch of a prepared level pair.
void run_pair(const dwt2d_plan& p, gpu::PairArgs& t, cudaStream_t st) {
  // whole waves of ~256-row chunks (measured at 16384^2: one wave of 256-row
  // chunks 432 us, 1.4 waves of 192 rows 593 us, 32-row chunks 488 us: the
  // 2(U+L)+U+L warm-up rows per chunk and partial waves both cost at 8 warps
  // per SM)
  t.nstrips = (t.l1.w2 + gpu::kPairLanes * 4 - 1) / (gpu::kPairLanes * 4);
  int per_sm = p.occ_pair.load(std::memory_order_relaxed);
  if (per_sm <= 0) {
    per_sm = std::max(1, p.entry->pair_occupancy ? p.entry->pair_occupancy() : 1);
    p.occ_pair.store(per_sm, std::memory_order_relaxed);
  }
  const long long resident = (long long)std::max(1, per_sm) * gpu::kWarpsPerCta * sm_count();
  const long long per_wave = std::max<long long>(1, resident / t.nstrips);  // chunks per full wave
  if (t.m_end <= 0) t.m_end = t.l2.h2;
  if (t.m_begin < 0 || t.m_begin >= t.m_end || t.m_end > t.l2.h2) fail(DWT2D_EINVAL, "level pair row range");
  const int span = t.m_end - t.m_begin;
  const long long waves = std::max<long long>(1, (span + 128 * per_wave) / (256 * per_wave));
  long long chunk = (span + waves * per_wave - 1) / (waves * per_wave);
  if (p.tune.pair_chunk_rows > 0) chunk = p.tune.pair_chunk_rows;
  t.chunk_rows = int(std::min<long long>(chunk, span));
  t.nchunks = (span + t.chunk_rows - 1) / t.chunk_rows;
  cuda_check(p.entry->pair(t, st), "level pair kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

bool pair_capable(const dwt2d_plan& p) {
  return p.entry && p.entry->pair && p.extension == DWT2D_PERIODIC;
}

// Levels 1 and 2 in one pass (pair_engine.cuh): LL_1 never goes to HBM.
// Used where level 1 streams from HBM with TMA-staged rows (>= 512 MiB).
// Tuning "pair": 0 disables it, 2 forces it on any size (tests). Pairing
// deeper levels measured no gain (levels 3+4 of 16384^2: 43.4 us vs 31.1 +
// 12.3). Returns false (nothing launched) when the pair is not eligible.
bool launch_pair(const dwt2d_plan& p, const gpu::LevelArgs& la, const gpu::LevelArgs& lb, cudaStream_t st) {
  if (!pair_capable(p) || p.tune.pair == 0) return false;
  const bool force = p.tune.pair == 2;
  gpu::PairArgs t{};
  t.l1 = la, t.l2 = lb;
  prepare(p, t.l1, kFromImage);
  prepare(p, t.l2, kFromImage);
  if (!(t.l1.vec && t.l2.vec && (t.l1.staged || force))) return false;
  run_pair(p, t, st);
  return true;
}

void forward_mallat(const dwt2d_plan& p, const float* image, size_t pitch, int W, int H, int levels,
                    float* out, size_t out_pitch, float* ws, cudaStream_t st,
                    void* const* events = nullptr) {
  if (events) record(events[0], st);
  std::vector<gpu::LevelArgs> lv(levels);
  const float* cur = image;
  size_t cur_pitch = pitch;
  for (int l = 1; l <= levels; ++l) {
    const int w = W >> (l - 1), h = H >> (l - 1), w2 = w / 2, h2 = h / 2;
    float* ll = l == levels ? out : ll_slot(ws, W, H, l);
    const size_t ll_pitch = l == levels ? out_pitch : size_t(w2);
    fill_forward_level(lv[l - 1], cur, cur_pitch, ll, ll_pitch, out, out_pitch, w2, h2);
    cur = ll;
    cur_pitch = ll_pitch;
  }
  // Alternate the chunk order: level l + 1 starts on the rows of LL_l that
  // level l wrote last, which are the likeliest still in L2 (LL uses normal
  // stores, the detail bands evict-first). The level pair writes LL_2
  // top-down, like a forward-order level.
  bool reverse = false;
  for (int l = 1; l <= levels; ++l) {
    if (l == 1 && levels >= 2 && launch_pair(p, lv[0], lv[1], st)) {
      if (events) record(events[1], st), record(events[2], st);
      ++l;
      reverse = true;
      continue;
    }
    gpu::LevelArgs a = lv[l - 1];
    a.reverse = reverse ? 1 : 0;
    reverse = !reverse;
    launch(p, a, kFromImage, st);
    if (events) record(events[l], st);
  }
}

void inverse_mallat(const dwt2d_plan& p, const float* in, size_t in_pitch, int W, int H, int levels,
                    float* image, size_t pitch, float* ws, cudaStream_t st) {
  const float* ll = in;
  size_t ll_pitch = in_pitch;
  if (is_identity(p)) fail(DWT2D_EUNSUPPORTED, "identity inverse pyramid");
  for (int l = levels; l >= 1; --l) {
    const int w = W >> (l - 1), h = H >> (l - 1), w2 = w / 2, h2 = h / 2;
    gpu::LevelArgs a{};
    a.in[0] = ll;
    a.in_pitch[0] = (long long)ll_pitch;
    a.in[1] = in + w2;
    a.in[2] = in + size_t(h2) * in_pitch;
    a.in[3] = in + size_t(h2) * in_pitch + w2;
    a.in_pitch[1] = a.in_pitch[2] = a.in_pitch[3] = (long long)in_pitch;
    float* dst = l == 1 ? image : ll_slot(ws, W, H, l - 1);
    const size_t dst_pitch = l == 1 ? pitch : size_t(w);
    a.out[0] = a.out[1] = a.out[2] = a.out[3] = dst;
    for (int j = 0; j < 4; ++j) a.out_pitch[j] = (long long)dst_pitch;
    a.w2 = w2, a.h2 = h2;
    a.reverse = ((levels - l) % 2 == 1) ? 1 : 0;
    launch(p, a, kToImage, st);
    ll = dst;
    ll_pitch = dst_pitch;
  }
}

// ---------------------------------------------- strip pyramid (multi-GPU)
//
// The whole forward pyramid of one rank's row strip in C++: per level the
// caller's exchange callback fills the halo rows (NCCL, peer copies, or
// nothing but a periodic wrap when exchange == NULL), then one fused kernel
// writes the strip's bands straight into the strip-Mallat buffer; levels 1+2
// run as one fused pass from 3*up / 3*down component rows of halo.

size_t strip_halo_rows(const dwt2d_plan& p) { return size_t(6) * size_t(std::max(p.up, p.down)); }
size_t strip_pitch(int W) { return ws_align(size_t(W)); }

size_t strip_workspace_floats(const dwt2d_plan& p, int W, int H, int levels) {
  return ll_offset(W, H, levels + 1) + 2 * strip_halo_rows(p) * strip_pitch(W);
}

void strip_exchange(dwt2d_halo_fn ex, void* user, const float* cur, size_t pitch, int w, int h, float* top,
                    float* bottom, size_t hp, int trows, int brows, cudaStream_t st) {
  if (ex) {
    const int rc = ex(user, cur, pitch, w, h, top, bottom, hp, trows, brows, st);
    if (rc != 0) fail(DWT2D_EINVAL, "strip pyramid: halo exchange callback failed");
    return;
  }
  if (trows > h || brows > h) fail(DWT2D_EINVAL, "strip pyramid: strip thinner than its halo");
  // a single strip is the whole periodic image: its own last / first rows
  cuda_check(cudaMemcpy2DAsync(top, hp * 4, cur + size_t(h - trows) * pitch, pitch * 4, size_t(w) * 4, trows,
                               cudaMemcpyDeviceToDevice, st), "halo wrap");
  cuda_check(cudaMemcpy2DAsync(bottom, hp * 4, cur, pitch * 4, size_t(w) * 4, brows, cudaMemcpyDeviceToDevice, st),
             "halo wrap");
}

void forward_mallat_strip(const dwt2d_plan& p, const float* strip, size_t pitch, int W, int H, int levels,
                          float* out, size_t op, float* ws, dwt2d_halo_fn ex, void* user, cudaStream_t st) {
  const size_t hp = strip_pitch(W);
  float* top = ws + ll_offset(W, H, levels + 1);
  float* bottom = top + strip_halo_rows(p) * hp;
  const float* cur = strip;
  size_t cur_pitch = pitch;
  int l = 1;
  if (levels >= 2 && pair_capable(p) && p.tune.pair != 0 && W % 16 == 0 && H % 4 == 0) {
    const int w2 = W / 2, h2 = H / 2, w4 = W / 4, h4 = H / 4;
    gpu::PairArgs t{};
    gpu::LevelArgs& a = t.l1;
    float* const d1[3] = {out + w2, out + size_t(h2) * op, out + size_t(h2) * op + w2};
    float* ll2 = levels == 2 ? out : ll_slot(ws, W, H, 2);
    const size_t ll2p = levels == 2 ? op : size_t(w4);
    float* const d2[4] = {ll2, out + w4, out + size_t(h4) * op, out + size_t(h4) * op + w4};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = cur, a.in_pitch[j] = (long long)cur_pitch;
      a.halo_top[j] = top, a.halo_bot[j] = bottom;
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)hp;
      a.out[j] = d1[j == 0 ? 0 : j - 1], a.out_pitch[j] = (long long)op;
      t.l2.in[j] = cur, t.l2.in_pitch[j] = (long long)cur_pitch;
      t.l2.out[j] = d2[j], t.l2.out_pitch[j] = (long long)(j == 0 ? ll2p : op);
    }
    a.halo = 1, a.up = 3 * p.up, a.down = 3 * p.down;
    a.w2 = w2, a.h2 = h2;
    t.l2.w2 = w4, t.l2.h2 = h4;
    prepare(p, t.l1, kFromImage);
    prepare(p, t.l2, kFromImage);
    if (t.l1.vec && t.l2.vec && 2 * a.up <= H && 2 * a.down <= H) {
      strip_exchange(ex, user, cur, cur_pitch, W, H, top, bottom, hp, 2 * a.up, 2 * a.down, st);
      run_pair(p, t, st);
      cur = ll2, cur_pitch = ll2p, l = 3;
    }
  }
  for (; l <= levels; ++l) {
    const int w = W >> (l - 1), h = H >> (l - 1), w2 = w / 2, h2 = h / 2;
    float* ll = l == levels ? out : ll_slot(ws, W, H, l);
    const size_t llp = l == levels ? op : size_t(w2);
    strip_exchange(ex, user, cur, cur_pitch, w, h, top, bottom, hp, 2 * p.up, 2 * p.down, st);
    gpu::LevelArgs a{};
    fill_forward_level(a, cur, cur_pitch, ll, llp, out, op, w2, h2);
    for (int j = 0; j < 4; ++j) {
      a.halo_top[j] = top, a.halo_bot[j] = bottom;
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)hp;
    }
    a.halo = 1, a.up = p.up, a.down = p.down;
    launch(p, a, kFromImage, st);
    cur = ll, cur_pitch = llp;
  }
}

// ------------------------------------------ sharded pyramid (multi-GPU)
//
// Row strips of one periodic image, one per rank (GPU), in a ring. Each
// level (or the fused level pair) needs the 2*up (6*up for the pair) image
// rows above the strip from the previous rank and 2*down (6*down) below it
// from the next rank. The exchange runs on the device (kernels/exchange.cu):
// every rank pushes its boundary rows straight into the neighbours'
// exchange windows over NVLink (peer stores) and signals a counter there;
// the level then runs on its interior rows — which need no halo — while
// the neighbours' rows arrive, waits for its own counters, and finishes the
// border rows. No host round trip per level; the whole strip pyramid is
// stream-ordered and graph-capturable. World 1 is the same ring with a
// single member: the pushes wrap the strip onto itself (periodic image).

// window header: counters on separate 128-byte lines (unsigned words)
constexpr int kTopArrivals = 0, kBotArrivals = 32, kDone = 64, kSeen = 96, kArrive = 128, kPyramids = 160;
constexpr size_t kHeaderBytes = 1024;
constexpr unsigned long long kExchangeTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s: a broken ring traps

struct ExchangeStep {
  int level;             // first level of the step (1-based)
  bool pair;             // levels `level` and `level` + 1 in one pass
  int width, height;     // the step's input strip (image rows)
  int trows, brows;      // halo image rows above / below
  size_t top_off, bot_off;  // bytes into the window
  size_t pitch;          // halo pitch (floats)
};

}  // namespace

struct dwt2d_shard {
  const dwt2d_plan* plan = nullptr;
  int device = 0, rank = 0, world = 1, W = 0, H = 0, levels = 0;
  std::vector<ExchangeStep> steps;
  char* window = nullptr;
  size_t window_bytes = 0;
  float* ws = nullptr;  // LL bands of levels 1 .. levels-1
  const dwt2d_shard* prev = nullptr;
  const dwt2d_shard* next = nullptr;
  char* prev_win = nullptr;  // neighbours' windows (peer pointers)
  char* next_win = nullptr;
  char* ipc_open[2] = {nullptr, nullptr};  // handles opened with cudaIpcOpenMemHandle
  bool connected = false;
  // diagnostics of a wait that timed out (host-mapped: readable after the
  // trap took the context down): code, counter value, target
  unsigned* diag_host = nullptr;
  unsigned* diag_dev = nullptr;
  unsigned* word(char* win, int w) const { return reinterpret_cast<unsigned*>(win) + w; }
  ~dwt2d_shard() {
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) cur = device;
    cudaSetDevice(device);
    for (char* p : ipc_open)
      if (p) cudaIpcCloseMemHandle(p);
    if (window) cudaFree(window);
    if (ws) cudaFree(ws);
    if (diag_host) cudaFreeHost(diag_host);
    cudaSetDevice(cur);
    cudaGetLastError();
  }
};

dwt2d_plan::~dwt2d_plan() {
  for (ShardRing& r : shard_cache)
    for (dwt2d_shard* s : r.shards) delete s;
  free_device_tables();
}

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cuda_check(cudaGetDevice(&prev), "current device");
    if (prev != dev) cuda_check(cudaSetDevice(dev), "set device");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

bool shard_pair(const dwt2d_plan& p, int W, int H, int levels) {
  return levels >= 2 && pair_capable(p) && p.tune.pair != 0 && W % 16 == 0 && H % 4 == 0;
}

// exchange steps and window layout of a strip pyramid
void plan_steps(dwt2d_shard& s) {
  const dwt2d_plan& p = *s.plan;
  size_t off = kHeaderBytes;
  auto add = [&](int level, bool pair, int w, int h, int tr, int br) {
    if (h < tr || h < br)
      fail(DWT2D_EUNSUPPORTED, "sharded pyramid: the strip of level " + std::to_string(level) + " (" +
                                   std::to_string(h) + " rows) is thinner than its halo; use fewer ranks or levels");
    ExchangeStep e{level, pair, w, h, tr, br, 0, 0, ws_align(size_t(w))};
    e.top_off = off, off += ((size_t(tr) * e.pitch * 4 + 255) & ~size_t(255));
    e.bot_off = off, off += ((size_t(br) * e.pitch * 4 + 255) & ~size_t(255));
    s.steps.push_back(e);
  };
  int l = 1;
  if (shard_pair(p, s.W, s.H, s.levels)) {
    add(1, true, s.W, s.H, 6 * p.up, 6 * p.down);
    l = 3;
  }
  for (; l <= s.levels; ++l) add(l, false, s.W >> (l - 1), s.H >> (l - 1), 2 * p.up, 2 * p.down);
  s.window_bytes = off;
}

float* step_top(const dwt2d_shard& s, const ExchangeStep& e) { return reinterpret_cast<float*>(s.window + e.top_off); }
float* step_bot(const dwt2d_shard& s, const ExchangeStep& e) { return reinterpret_cast<float*>(s.window + e.bot_off); }

void shard_connect_windows(dwt2d_shard& s, char* prev_win, char* next_win) {
  s.prev_win = prev_win, s.next_win = next_win;
  s.connected = true;
}

// input rows of step e (the strip, or the LL band the previous step wrote)
struct StepIO {
  const float* cur;
  size_t cur_pitch;
};
StepIO step_input(const dwt2d_shard& s, size_t e, const float* strip, size_t pitch, float* out, size_t op) {
  if (e == 0) return {strip, pitch};
  const ExchangeStep& prev = s.steps[e - 1];
  const int l = prev.pair ? prev.level + 1 : prev.level;  // last level the previous step computed
  // that level's LL: a workspace slot (never the output: step e exists, so l < levels)
  (void)out, (void)op;
  return {ll_slot(s.ws, s.W, s.H, l), size_t(s.W >> l)};
}

void shard_push(dwt2d_shard& s, size_t e, const StepIO& io, bool wait_after, cudaStream_t st) {
  const ExchangeStep& x = s.steps[e];
  gpu::HaloPushArgs a{};
  a.src = io.cur, a.src_pitch = (long long)io.cur_pitch;
  a.width = x.width, a.height = x.height;
  a.rows_first = x.brows, a.rows_last = x.trows;  // my first rows are prev's bottom halo
  a.dst_prev = reinterpret_cast<float*>(s.prev_win + x.bot_off);
  a.dst_next = reinterpret_cast<float*>(s.next_win + x.top_off);
  a.dst_pitch = (long long)x.pitch;
  a.vec = (x.width % 4 == 0 && io.cur_pitch % 4 == 0 && aligned(io.cur, 16)) ? 1 : 0;
  a.flag_prev = s.word(s.prev_win, kBotArrivals);
  a.flag_next = s.word(s.next_win, kTopArrivals);
  a.arrive = s.word(s.window, kArrive);
  a.error = s.diag_dev;
  a.timeout_ns = kExchangeTimeoutNs;
  a.wait_after = wait_after ? 1 : 0;
  a.my_top = s.word(s.window, kTopArrivals);
  a.my_bot = s.word(s.window, kBotArrivals);
  a.seen = s.word(s.window, kSeen);
  a.pdl = s.plan->tune.pdl ? 1 : 0;
  cuda_check(gpu::launch_halo_push(a, sm_count(), st), "halo push launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void shard_wait(dwt2d_shard& s, cudaStream_t st) {
  cuda_check(gpu::launch_halo_wait(s.word(s.window, kTopArrivals), s.word(s.window, kBotArrivals),
                                   s.word(s.window, kSeen), s.diag_dev, kExchangeTimeoutNs, st),
             "halo wait launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void shard_start(dwt2d_shard& s, cudaStream_t st) {
  cuda_check(gpu::launch_pyramid_start(s.word(s.window, kDone), s.word(s.window, kPyramids), s.diag_dev,
                                       kExchangeTimeoutNs, st),
             "pyramid start launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void shard_done(dwt2d_shard& s, cudaStream_t st) {
  cuda_check(gpu::launch_pyramid_done(s.word(s.prev_win, kDone), s.word(s.next_win, kDone),
                                      s.word(s.window, kPyramids), st),
             "pyramid done launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Output rows of step e that need no halo: the interior [lo, hi) of the
// step's (level-2 for the pair) output rows, or lo == hi when the interior
// is too short to be worth its own launch.
void step_interior(const dwt2d_shard& s, const ExchangeStep& x, int& lo, int& hi, int& rows) {
  const dwt2d_plan& p = *s.plan;
  if (x.pair) {
    // level-2 rows [m0, m1) read level-1 component rows [2 m0 - 3U, 2 m1 + 3L)
    rows = x.height / 4;
    lo = (3 * p.up + 1) / 2;
    hi = (x.height / 2 - 3 * p.down) / 2;
  } else {
    rows = x.height / 2;
    lo = p.up;
    hi = rows - p.down;
  }
  if (hi - lo < 16) lo = hi = 0;
}

// Whether step e runs its interior rows while the halo rows travel (push,
// interior, wait, border: four launches and more) or as push-and-wait in
// one launch followed by the whole level (two launches). Splitting pays only
// where the level itself takes long against the few microseconds of launch
// latency each extra launch adds: level inputs of at least 64 MiB.
bool split_step(const dwt2d_shard& s, size_t e) {
  const ExchangeStep& x = s.steps[e];
  int lo, hi, rows;
  step_interior(s, x, lo, hi, rows);
  return hi > lo && size_t(x.width) * size_t(x.height) * 4 >= (size_t(64) << 20);
}

// part: 0 interior rows, 1 border rows (all rows when there is no
// interior), 2 all rows
void shard_compute(dwt2d_shard& s, size_t e, const StepIO& io, float* out, size_t op, int part, cudaStream_t st) {
  const dwt2d_plan& p = *s.plan;
  const ExchangeStep& x = s.steps[e];
  int lo, hi, rows;
  step_interior(s, x, lo, hi, rows);
  std::vector<std::pair<int, int>> ranges;
  if (part == 2) {
    ranges.push_back({0, rows});
  } else if (part == 0) {
    if (hi > lo) ranges.push_back({lo, hi});
  } else if (hi > lo) {
    if (lo > 0) ranges.push_back({0, lo});
    if (hi < rows) ranges.push_back({hi, rows});
  } else {
    ranges.push_back({0, rows});
  }
  if (ranges.empty()) return;
  const float* top = step_top(s, x);
  const float* bottom = step_bot(s, x);
  const int W = x.width, H = x.height;
  const bool last = (x.pair ? x.level + 1 : x.level) == s.levels;
  if (x.pair) {
    const int w2 = W / 2, h2 = H / 2, w4 = W / 4, h4 = H / 4;
    float* const d1[3] = {out + w2, out + size_t(h2) * op, out + size_t(h2) * op + w2};
    float* ll2 = last ? out : ll_slot(s.ws, s.W, s.H, 2);
    const size_t ll2p = last ? op : size_t(w4);
    float* const d2[4] = {ll2, out + w4, out + size_t(h4) * op, out + size_t(h4) * op + w4};
    for (const auto& r : ranges) {
      gpu::PairArgs t{};
      gpu::LevelArgs& a = t.l1;
      for (int j = 0; j < 4; ++j) {
        a.in[j] = io.cur, a.in_pitch[j] = (long long)io.cur_pitch;
        a.halo_top[j] = top, a.halo_bot[j] = bottom;
        a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)x.pitch;
        a.out[j] = d1[j == 0 ? 0 : j - 1], a.out_pitch[j] = (long long)op;
        t.l2.in[j] = io.cur, t.l2.in_pitch[j] = (long long)io.cur_pitch;
        t.l2.out[j] = d2[j], t.l2.out_pitch[j] = (long long)(j == 0 ? ll2p : op);
      }
      a.halo = 1, a.up = 3 * p.up, a.down = 3 * p.down;
      a.w2 = w2, a.h2 = h2;
      t.l2.w2 = w4, t.l2.h2 = h4;
      prepare(p, t.l1, kFromImage);
      prepare(p, t.l2, kFromImage);
      if (!t.l1.vec || !t.l2.vec)
        fail(DWT2D_EINVAL, "sharded pyramid: strips and outputs need 16-byte aligned rows (pitches multiple of 4)");
      t.m_begin = r.first, t.m_end = r.second;
      run_pair(p, t, st);
    }
    return;
  }
  const int w2 = W / 2, h2 = H / 2;
  float* ll = last ? out : ll_slot(s.ws, s.W, s.H, x.level);
  const size_t llp = last ? op : size_t(w2);
  for (const auto& r : ranges) {
    gpu::LevelArgs a{};
    fill_forward_level(a, io.cur, io.cur_pitch, ll, llp, out, op, w2, h2);
    for (int j = 0; j < 4; ++j) {
      a.halo_top[j] = top, a.halo_bot[j] = bottom;
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)x.pitch;
    }
    a.halo = 1, a.up = p.up, a.down = p.down;
    a.y_begin = r.first, a.y_end = r.second;
    launch(p, a, kFromImage, st);
  }
}

void check_shard_args(const dwt2d_shard& s, const float* strip, const float* out) {
  if (!strip || !out) fail(DWT2D_EINVAL, "null argument");
  if (!s.connected) fail(DWT2D_EINVAL, "sharded pyramid: shard is not connected to its ring neighbours");
}

// ------------------------------------------------- host end-to-end pipeline
//
// Host image -> Mallat pyramid -> host, with the transfers overlapped with
// level 1 (which streams by rows): the image goes up in row bands on an H2D
// stream; level 1 of band b runs as a strip kernel whose halo rows are the
// neighbouring bands' rows already on the device (the image's last rows are
// uploaded first, for band 0's periodic top halo) as soon as band b + 1 has
// landed; the band's three detail blocks go back on a D2H stream while later
// bands are still uploading. Levels 2..L then run on the device-resident LL1
// and only the top-left quadrant remains to be copied back.
struct HostPipe {
  cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
  std::vector<cudaEvent_t> ev;
  void* buf = nullptr;  // grow-only device staging (mapping GBs per call costs tens of ms)
  size_t cap = 0;
  void* reserve(size_t bytes) {
    if (bytes > cap) {
      if (buf) cuda_check(cudaFree(buf), "free");
      buf = nullptr;
      cap = 0;
      cuda_check(cudaMalloc(&buf, bytes), "device allocation");
      cap = bytes;
    }
    return buf;
  }
  HostPipe() {
    cuda_check(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking), "stream");
  }
  // timeline trace (tuning host_trace; development only): timing events
  // recorded on the pipeline's streams, printed to stderr after the call
  std::vector<cudaEvent_t> tev;
  std::vector<std::string> tname;
  size_t ntrace = 0;
  void mark(bool on, cudaStream_t st, const std::string& name) {
    if (!on) return;
    if (tev.size() <= ntrace) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      tev.push_back(e);
      tname.emplace_back();
    }
    tname[ntrace] = name;
    cuda_check(cudaEventRecord(tev[ntrace++], st), "record");
  }
  void dump(bool on) {
    if (!on || ntrace == 0) return;
    for (size_t i = 0; i < ntrace; ++i) {
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, tev[0], tev[i]), "elapsed");
      std::fprintf(stderr, "[host_trace] %8.3f ms  %s\n", ms, tname[i].c_str());
    }
    ntrace = 0;
  }
  cudaEvent_t event(size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ev.push_back(e);
    }
    return ev[i];
  }
};

// One pipeline per thread and device: its streams and staging belong to the
// device that was current when it was created.
HostPipe& host_pipe() {
  static thread_local std::unique_ptr<HostPipe> pipes[kMaxDevices];
  std::unique_ptr<HostPipe>& p = pipes[current_device()];
  if (!p) p = std::make_unique<HostPipe>();
  return *p;
}

// Row bands of the host pipeline: bands of `rows` image rows, the last one
// taking the remainder (rows <= last < 2 * rows), so every band — including
// the last — is at least `rows` >= 4 * halo rows tall. Tapered (tuning
// host_taper): the first band is rows / 4 tall (the D2H stream starts
// sooner) and the last `rows` rows are split rows / 2, rows / 4, rows / 4
// (less is left to copy down after the last upload).
struct Bands {
  std::vector<int> edge;  // band b = image rows [edge[b], edge[b + 1])
  int n = 0;
  int begin(int b) const { return edge[b]; }
  int end(int b, int) const { return edge[b + 1]; }
};
Bands bands_for(const dwt2d_plan& p, int H, int halo_rows) {
  int r = p.tune.host_band_rows;
  if (r <= 0) r = H / 16;                         // ~16 bands
  const int lo = std::max(64, 4 * halo_rows);     // level-2 bands need their own halo rows
  r = std::max(r, lo);
  r = (r + 3) & ~3;                               // even LL1 rows per band
  r = std::min(r, H);
  const int n = std::max(1, H / r);
  Bands b;
  for (int i = 0; i < n; ++i) b.edge.push_back(i * r);
  b.edge.push_back(H);
  const int q = (r / 4) & ~3;
  if (p.tune.host_taper && n >= 3 && q >= lo && q <= H - 4 * q - lo) {
    // the first band split q + (r - q), the last 4q rows 2q + q + q; the
    // band before them absorbs the remainder (at least lo rows)
    std::vector<int> e{0, q};
    for (int i = 1; i < n; ++i)
      if (i * r <= H - 4 * q - lo) e.push_back(i * r);
    for (const int t : {H - 4 * q, H - 2 * q, H - q, H}) e.push_back(t);
    b.edge = e;
  }
  b.n = int(b.edge.size()) - 1;
  return b;
}

// One forward level on image rows [r0, r1) of a level input `in` (w_in x
// h_in, pitch ip) whose rows above/below come from the same buffer (periodic
// wrap): the band's rows of LL go to `ll` (pitch llp), of HL/LH/HH to the
// level's Mallat region `det` (pitch dp).
void band_level(const dwt2d_plan& p, const float* in, size_t ip, int w_in, int h_in, int r0, int r1, float* ll,
                size_t llp, float* det, size_t dp, cudaStream_t st) {
  const int top_rows = 2 * p.up, bot_rows = 2 * p.down;
  if (r0 > 0 && r0 < top_rows) fail(DWT2D_EINVAL, "band rows smaller than the halo");
  const float* top = r0 >= top_rows ? in + size_t(r0 - top_rows) * ip : in + size_t(h_in - top_rows) * ip;
  const float* bot = r1 + bot_rows <= h_in ? in + size_t(r1) * ip : in;
  const int w2 = w_in / 2, h2 = h_in / 2, y0 = r0 / 2, hb = (r1 - r0) / 2;
  gpu::LevelArgs a{};
  for (int j = 0; j < 4; ++j) {
    a.in[j] = in + size_t(r0) * ip, a.in_pitch[j] = (long long)ip;
    a.halo_top[j] = top, a.halo_bot[j] = bot;
    a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)ip;
  }
  a.out[0] = ll + size_t(y0) * llp;
  a.out_pitch[0] = (long long)llp;
  a.out[1] = det + size_t(y0) * dp + w2;
  a.out[2] = det + size_t(h2 + y0) * dp;
  a.out[3] = det + size_t(h2 + y0) * dp + w2;
  a.out_pitch[1] = a.out_pitch[2] = a.out_pitch[3] = (long long)dp;
  a.halo = 1, a.up = p.up, a.down = p.down;
  a.w2 = w2, a.h2 = hb;
  launch(p, a, kFromImage, st);
}

// D2H of a band's detail rows of one level (Mallat region `det`/`hdet` with
// pitch W floats, level input w_in x h_in, output component rows [y0, y0+hb))
void band_details_down(float* hdet, const float* det, int W, int w_in, int h_in, int y0, int hb, cudaStream_t st) {
  const int w2 = w_in / 2, h2 = h_in / 2;
  const size_t pitch = size_t(W) * 4;
  cuda_check(cudaMemcpy2DAsync(hdet + size_t(y0) * W + w2, pitch, det + size_t(y0) * W + w2, pitch, size_t(w2) * 4,
                               hb, cudaMemcpyDeviceToHost, st),
             "D2H");
  // LH and HH rows sit side by side: one block of w_in columns
  cuda_check(cudaMemcpy2DAsync(hdet + size_t(h2 + y0) * W, pitch, det + size_t(h2 + y0) * W, pitch, size_t(w_in) * 4,
                               hb, cudaMemcpyDeviceToHost, st),
             "D2H");
}

// Host image -> pyramid -> host with the copies overlapped (SURVEY §8(d)
// e2e). The image goes up in row bands on the `up` stream; the first P
// levels run band by band on `comp` and each band's detail rows go down on
// `down` while later bands upload.
//
// Compute bands trail the upload bands by the bottom halo: level l's band b
// covers input rows [C_l(b), C_l(b+1)) with C_l(b) = floor4(E_l(b) - 2*down),
// where E_1(b) is the upload boundary and E_l(b) = C_{l-1}(b) / 2 the LL rows
// level l-1 has produced; so band b of every level runs as soon as image band
// b has landed (its bottom halo is already there) instead of waiting for band
// b + 1. Band 0's periodic top halo at level l is the TAIL of level l's input
// (its last 2*up rows): the image's last T_1 rows go up first, and the LL
// tails are computed early from them (T_l = 2 T_{l+1} + 2 up input rows of
// level l, T_P = 2 up); the last band recomputes those rows with identical
// values. Levels P+1.. run on the device-resident LL_P, and only its
// quadrant goes down last.
// Returns false (nothing enqueued) when the image is too short for even one
// band and its halos; the caller then copies it whole.
bool forward_mallat_host_pipelined(const dwt2d_plan& p, const float* image, int W, int H, int levels,
                                   float* out) {
  HostPipe& hp = host_pipe();
  const int U = p.up, Ld = p.down;
  const Bands bands = bands_for(p, H, std::max(U, Ld) * 2);
  const int B = bands.n;
  // pipelined levels: 2 by default (16384^2 e2e, 8 levels: 24.2 ms with 2,
  // 24.9 ms with 3 — level-3 bands of a few MB cost more in launches and
  // small copies than the 48 MiB they take off the last copy — and 27.5 ms
  // with 1), at most 3; fewer when the bands would get thinner than 4 halos
  // or the tails would not fit in the level inputs
  constexpr int kMaxPipe = 3;
  int P = std::min(levels, p.tune.host_levels > 0 ? std::min(p.tune.host_levels, kMaxPipe) : 2);
  std::vector<std::vector<int>> C;  // C[l - 1][b], b = 0..B
  std::vector<int> T;               // T[l - 1]: tail rows of level l's input uploaded/computed early
  for (;; --P) {
    C.assign(P, std::vector<int>(B + 1));
    T.assign(P + 1, 0);
    bool ok = true;
    T[P - 1] = 2 * U;
    for (int l = P - 1; l >= 1; --l) T[l - 1] = 2 * T[l] + 2 * U;
    for (int l = 1; l <= P && ok; ++l) {
      const int hl = H >> (l - 1);
      C[l - 1][0] = 0, C[l - 1][B] = hl;
      for (int b = 1; b < B; ++b) {
        const int e = l == 1 ? bands.begin(b) : C[l - 2][b] / 2;
        C[l - 1][b] = ((e - 2 * Ld) / 4) * 4;
      }
      for (int b = 0; b < B; ++b) ok = ok && C[l - 1][b + 1] - C[l - 1][b] >= 4 * std::max(U, Ld);
      if (l < P) ok = ok && hl - 2 * T[l] >= 2 * U + 2 * Ld && hl - 2 * T[l] >= C[l - 1][std::min(1, B)];
    }
    ok = ok && T[0] + 2 * Ld <= H;
    if (ok || P == 1) break;
  }
  if (T[0] + 2 * Ld > H) return false;

  // device buffers: image, Mallat output, LL_1 .. LL_P (LL_levels goes into
  // the output), workspace of the device-resident levels
  const size_t n = size_t(W) * H;
  std::vector<size_t> ll_off(P + 1, 0);
  size_t floats = 2 * n;
  for (int l = 1; l <= P; ++l) {
    ll_off[l] = floats;
    floats += ((size_t(W >> l) * size_t(H >> l)) + 63) & ~size_t(63);
  }
  const int wP = W >> P, hP = H >> P;
  const size_t sub_ws = levels > P ? dwt2d_workspace_bytes(wP, hP, levels - P) : 0;
  float* d_img = static_cast<float*>(hp.reserve(floats * 4 + sub_ws + 512));
  float* d_out = d_img + n;
  float* d_sub = d_img + floats;
  auto ll = [&](int l) { return l == levels ? d_out : d_img + ll_off[l]; };
  auto llp = [&](int l) { return l == levels ? size_t(W) : size_t(W >> l); };
  auto in_of = [&](int l) { return l == 1 ? d_img : ll(l - 1); };
  auto inp_of = [&](int l) { return l == 1 ? size_t(W) : llp(l - 1); };

  size_t ev = 0;
  const bool tr = p.tune.host_trace != 0;
  hp.mark(tr, hp.comp, "start");
  cudaEvent_t ev_alloc = hp.event(ev++);
  cuda_check(cudaEventRecord(ev_alloc, hp.comp), "record");
  cuda_check(cudaStreamWaitEvent(hp.up, ev_alloc), "wait");
  cuda_check(cudaStreamWaitEvent(hp.down, ev_alloc), "wait");

  // upload: the image's last T_1 rows first, then the bands in order
  const int tail_rows = T[0];
  const size_t tail0 = size_t(H - tail_rows) * W;
  cuda_check(cudaMemcpyAsync(d_img + tail0, image + tail0, size_t(tail_rows) * W * 4, cudaMemcpyHostToDevice, hp.up),
             "H2D");
  std::vector<cudaEvent_t> up(B);
  for (int b = 0; b < B; ++b) {
    const int r0 = bands.begin(b), r1 = bands.end(b, H);
    const int c1 = (b == B - 1) ? std::max(r0, H - tail_rows) : r1;
    if (c1 > r0)
      cuda_check(cudaMemcpyAsync(d_img + size_t(r0) * W, image + size_t(r0) * W, size_t(c1 - r0) * W * 4,
                                 cudaMemcpyHostToDevice, hp.up),
                 "H2D");
    up[b] = hp.event(ev++);
    cuda_check(cudaEventRecord(up[b], hp.up), "record");
    hp.mark(tr, hp.up, "up " + std::to_string(b));
  }

  auto down_after = [&](auto&& copy) {
    cudaEvent_t done = hp.event(ev++);
    cuda_check(cudaEventRecord(done, hp.comp), "record");
    cuda_check(cudaStreamWaitEvent(hp.down, done), "wait");
    copy();
  };
  auto level_band = [&](int l, int b) {
    const int wl = W >> (l - 1), hl = H >> (l - 1), r0 = C[l - 1][b], r1 = C[l - 1][b + 1];
    band_level(p, in_of(l), inp_of(l), wl, hl, r0, r1, ll(l), llp(l), d_out, size_t(W), hp.comp);
    hp.mark(tr, hp.comp, "comp L" + std::to_string(l) + " b" + std::to_string(b));
    down_after([&] { band_details_down(out, d_out, W, wl, hl, r0 / 2, (r1 - r0) / 2, hp.down); });
    hp.mark(tr, hp.down, "down L" + std::to_string(l) + " b" + std::to_string(b));
  };

  for (int b = 0; b < B; ++b) {
    cuda_check(cudaStreamWaitEvent(hp.comp, up[b]), "wait");
    for (int l = 1; l <= P; ++l) {
      level_band(l, b);
      if (b == 0 && l < P) {  // LL_l's tail: band 0's top halo at level l + 1 (and the next tail's input)
        const int wl = W >> (l - 1), hl = H >> (l - 1);
        band_level(p, in_of(l), inp_of(l), wl, hl, hl - 2 * T[l], hl, ll(l), llp(l), d_out, size_t(W), hp.comp);
      }
    }
  }
  if (levels > P) forward_mallat(p, ll(P), llp(P), wP, hP, levels - P, d_out, size_t(W), d_sub, hp.comp);
  hp.mark(tr, hp.comp, "comp deep levels");
  down_after([&] {  // the remaining top-left corner (levels > P and LL_levels)
    cuda_check(cudaMemcpy2DAsync(out, size_t(W) * 4, d_out, size_t(W) * 4, size_t(wP) * 4, hP,
                                 cudaMemcpyDeviceToHost, hp.down),
               "D2H");
  });
  hp.mark(tr, hp.down, "down quadrant");
  cuda_check(cudaStreamSynchronize(hp.down), "synchronize");
  hp.dump(tr);
  return true;
}

}  // namespace

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* dwt2d_last_error(void) { return g_error.c_str(); }
const char* dwt2d_version(void) { return "dwt2d_b200 0.1 (sm_100a)"; }
uint64_t dwt2d_launch_count(void) { return g_launches.load(); }

int dwt2d_registry_size(void) { return int(gpu::plan_registry().size()); }
const char* dwt2d_registry_key(int i) {
  const auto& r = gpu::plan_registry();
  return (i >= 0 && i < int(r.size())) ? r[i].key : nullptr;
}

int dwt2d_plan_create(const dwt2d_plan_desc* d, dwt2d_plan** out) {
  return guard([&] {
    if (!d || !out || !d->wavelet) fail(DWT2D_EINVAL, "null argument");
    *out = nullptr;
    if (d->workers < 1) fail(DWT2D_EINVAL, "compile: worker count must be at least 1");
    if (d->scheme < 0 || d->scheme > DWT2D_INVERSE_LIFTING) fail(DWT2D_EINVAL, "unknown scheme");
    if (d->extension != DWT2D_PERIODIC && d->extension != DWT2D_SYMMETRIC)
      fail(DWT2D_EINVAL, "unknown extension");
    const WaveletSpec w = resolve_wavelet(d->wavelet);
    Scheme s;
    if (d->scheme == DWT2D_INVERSE_LIFTING) {
      if (d->optimized) fail(DWT2D_EINVAL, "optimize_constant_split: inverse schemes are not optimizable");
      s = build_inverse_lifting(w);
    } else {
      s = build_scheme(static_cast<SchemeKind>(d->scheme), w);
      if (d->optimized) s = optimize_constant_split(s, w);
    }
    Lowering mode = default_lowering(s);
    if (d->lowering == DWT2D_LOWERING_COMPOSED) mode = Lowering::composed;
    if (d->lowering == DWT2D_LOWERING_FACTORED) mode = Lowering::factored;
    const StepProgram prog = lower(s, mode);
    auto p = std::make_unique<dwt2d_plan>();
    p->forward = d->scheme != DWT2D_INVERSE_LIFTING;
    p->operations = count_operations(s);
    p->description = describe(s);
    finalize_plan(*p, prog, d->extension);
    p->has64 = true;
    *out = p.release();
  });
}

int dwt2d_plan_create_from_program(const dwt2d_program* t, dwt2d_plan** out) {
  return guard([&] {
    if (!t || !out) fail(DWT2D_EINVAL, "null argument");
    *out = nullptr;
    const StepProgram prog = program_from_tables(*t);
    auto p = std::make_unique<dwt2d_plan>();
    p->forward = t->forward != 0;
    finalize_plan(*p, prog, t->extension);
    p->has64 = t->weights64 != nullptr;
    if (p->entry) p->key = p->entry->key;
    *out = p.release();
  });
}

void dwt2d_plan_destroy(dwt2d_plan* p) { delete p; }

int dwt2d_plan_set_tuning(dwt2d_plan* p, const char* name, int value) {
  return guard([&] {
    require_plan(p);
    if (!name) fail(DWT2D_EINVAL, "null argument");
    const std::string n = name;
    Tuning& t = p->tune;
    if (n == "pdl") t.pdl = value;
    else if (n == "chunk_rows") t.chunk_rows = value;
    else if (n == "alternate") t.alternate = value;
    else if (n == "tma") t.tma = value;
    else if (n == "pair") t.pair = value;
    else if (n == "pair_chunk_rows") t.pair_chunk_rows = value;
    else if (n == "crop_tiles") t.crop_tiles = value;
    else if (n == "crop_core") t.crop_core = std::max(1, value);
    else if (n == "host_band_rows") t.host_band_rows = value;
    else if (n == "host_levels") t.host_levels = value;
    else if (n == "host_taper") t.host_taper = value;
    else if (n == "host_trace") t.host_trace = value;
    else fail(DWT2D_EINVAL, "unknown tuning switch: " + n);
  });
}

int dwt2d_plan_get_info(const dwt2d_plan* p, dwt2d_plan_info* info) {
  return guard([&] {
    require_plan(p);
    if (!info) fail(DWT2D_EINVAL, "null info");
    std::memset(info, 0, sizeof *info);
    std::snprintf(info->key, sizeof info->key, "%s", p->key.c_str());
    info->fingerprint = p->fingerprint;
    info->logical_steps = p->logical_steps;
    info->substeps = p->substeps;
    info->operations = p->operations;
    info->taps_per_quad = p->taps_per_quad;
    info->reach_left = p->left, info->reach_right = p->right;
    info->reach_up = p->up, info->reach_down = p->down;
    info->columns_per_lane = p->entry ? p->entry->cw : 0;
    info->forward = p->forward;
    info->extension = p->extension;
    info->fused_multiply_add = p->fma;
    info->generic = p->generic ? 1 : 0;
  });
}

int dwt2d_plan_get_tables(const dwt2d_plan* p, dwt2d_row* rows, int32_t rows_cap, dwt2d_tap* taps,
                          int32_t taps_cap, int32_t* nrows, int32_t* ntaps) {
  return guard([&] {
    require_plan(p);
    if (nrows) *nrows = int32_t(p->rows.size());
    if (ntaps) *ntaps = int32_t(p->taps.size());
    if (rows) {
      if (rows_cap < int32_t(p->rows.size())) fail(DWT2D_EINVAL, "rows buffer too small");
      std::copy(p->rows.begin(), p->rows.end(), rows);
    }
    if (taps) {
      if (taps_cap < int32_t(p->taps.size())) fail(DWT2D_EINVAL, "taps buffer too small");
      std::copy(p->taps.begin(), p->taps.end(), taps);
    }
  });
}

int dwt2d_plan_describe(const dwt2d_plan* p, char* buf, size_t len) {
  return guard([&] {
    require_plan(p);
    if (!buf || len < p->description.size() + 1) fail(DWT2D_EINVAL, "describe: buffer too small");
    std::memcpy(buf, p->description.c_str(), p->description.size() + 1);
  });
}

int dwt2d_run_planar(const dwt2d_plan* p, const float* const in[4], const size_t in_pitch[4],
                     float* const out[4], const size_t out_pitch[4], int w2, int h2, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!in || !out || !in_pitch || !out_pitch) fail(DWT2D_EINVAL, "null argument");
    if (w2 <= 0 || h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    if (is_identity(*p)) return copy_planes(in, in_pitch, out, out_pitch, w2, h2, as_stream(stream));
    gpu::LevelArgs a{};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = in[j], a.out[j] = out[j];
      a.in_pitch[j] = (long long)in_pitch[j], a.out_pitch[j] = (long long)out_pitch[j];
      if (in_pitch[j] < size_t(w2) || out_pitch[j] < size_t(w2)) fail(DWT2D_EINVAL, "pitch < width");
    }
    a.w2 = w2, a.h2 = h2;
    launch(*p, a, kPlanar, as_stream(stream));
  });
}

int dwt2d_forward_level(const dwt2d_plan* p, const float* image, size_t pitch, int width, int height,
                        float* const out[4], const size_t out_pitch[4], void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out || !out_pitch) fail(DWT2D_EINVAL, "null argument");
    if (width <= 0 || height <= 0) fail(DWT2D_EINVAL, "polyphase_split: empty image");
    if (width % 2) fail(DWT2D_EINVAL, "polyphase_split: odd image width");
    if (height % 2) fail(DWT2D_EINVAL, "polyphase_split: odd image height");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    gpu::LevelArgs a{};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = image, a.in_pitch[j] = (long long)pitch;
      a.out[j] = out[j], a.out_pitch[j] = (long long)out_pitch[j];
    }
    a.w2 = width / 2, a.h2 = height / 2;
    launch(*p, a, kFromImage, as_stream(stream));
  });
}

int dwt2d_inverse_level(const dwt2d_plan* p, const float* const in[4], const size_t in_pitch[4],
                        float* image, size_t pitch, int width, int height, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !in || !in_pitch) fail(DWT2D_EINVAL, "null argument");
    if (width <= 0 || height <= 0 || width % 2 || height % 2)
      fail(DWT2D_EINVAL, "inverse_level: image sides must be positive and even");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    gpu::LevelArgs a{};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = in[j], a.in_pitch[j] = (long long)in_pitch[j];
      a.out[j] = image, a.out_pitch[j] = (long long)pitch;
    }
    a.w2 = width / 2, a.h2 = height / 2;
    launch(*p, a, kToImage, as_stream(stream));
  });
}

int dwt2d_forward_level_strip(const dwt2d_plan* p, const float* image, size_t pitch, int width, int height,
                              const float* top, const float* bottom, size_t halo_pitch, float* const out[4],
                              const size_t out_pitch[4], void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out || !out_pitch || !top || !bottom) fail(DWT2D_EINVAL, "null argument");
    if (width <= 0 || height <= 0 || width % 2 || height % 2)
      fail(DWT2D_EINVAL, "forward_level_strip: strip sides must be positive and even");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    gpu::LevelArgs a{};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = image, a.in_pitch[j] = (long long)pitch;
      a.halo_top[j] = top, a.halo_bot[j] = bottom;
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)halo_pitch;
      a.out[j] = out[j], a.out_pitch[j] = (long long)out_pitch[j];
    }
    a.halo = 1, a.up = p->up, a.down = p->down;
    a.w2 = width / 2, a.h2 = height / 2;
    launch(*p, a, kFromImage, as_stream(stream));
  });
}

int dwt2d_plan_has_pair(const dwt2d_plan* p) { return p && pair_capable(*p) ? 1 : 0; }

size_t dwt2d_strip_workspace_bytes(const dwt2d_plan* p, int width, int height, int levels) {
  if (!p || width <= 0 || height <= 0 || levels < 1) return 0;
  return strip_workspace_floats(*p, width, height, levels) * sizeof(float);
}

int dwt2d_forward_mallat_strip(const dwt2d_plan* p, const float* strip, size_t pitch, int W, int H, int levels,
                               float* out, size_t out_pitch, void* scratch, dwt2d_halo_fn exchange, void* user,
                               void* stream) {
  return guard([&] {
    require_plan(p);
    if (!strip || !out) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_mallat_strip: plan is an inverse plan");
    check_pyramid(W, H, levels);
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    if (p->extension != DWT2D_PERIODIC) fail(DWT2D_EUNSUPPORTED, "row strips need periodic extension");
    const cudaStream_t st = as_stream(stream);
    float* ws = static_cast<float*>(scratch);
    void* owned = nullptr;
    if (!ws) {
      cuda_check(cudaMallocAsync(&owned, strip_workspace_floats(*p, W, H, levels) * sizeof(float), st),
                 "strip workspace");
      ws = static_cast<float*>(owned);
    }
    struct Free {
      void* m;
      cudaStream_t s;
      ~Free() {
        if (m) cudaFreeAsync(m, s);
      }
    } free_ws{owned, st};
    forward_mallat_strip(*p, strip, pitch, W, H, levels, out, out_pitch, ws, exchange, user, st);
  });
}

int dwt2d_forward_pair_strip(const dwt2d_plan* p, const float* image, size_t pitch, int width, int height,
                             const float* top, const float* bottom, size_t halo_pitch, float* const out1[3],
                             const size_t out1_pitch[3], float* const out2[4], const size_t out2_pitch[4],
                             void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out1 || !out1_pitch || !out2 || !out2_pitch || !top || !bottom)
      fail(DWT2D_EINVAL, "null argument");
    if (width <= 0 || height <= 0 || width % 4 || height % 4)
      fail(DWT2D_EINVAL, "forward_pair_strip: strip sides must be positive multiples of 4");
    if (!pair_capable(*p)) fail(DWT2D_EUNSUPPORTED, "forward_pair_strip: no fused level-pair kernel for this plan");
    gpu::PairArgs t{};
    gpu::LevelArgs& a = t.l1;
    for (int j = 0; j < 4; ++j) {
      a.in[j] = image, a.in_pitch[j] = (long long)pitch;
      a.halo_top[j] = top, a.halo_bot[j] = bottom;
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)halo_pitch;
      a.out[j] = out1[j == 0 ? 0 : j - 1], a.out_pitch[j] = (long long)out1_pitch[j == 0 ? 0 : j - 1];
      t.l2.out[j] = out2[j], t.l2.out_pitch[j] = (long long)out2_pitch[j];
      t.l2.in[j] = image, t.l2.in_pitch[j] = (long long)pitch;  // unused by the pair
    }
    a.halo = 1, a.up = 3 * p->up, a.down = 3 * p->down;
    a.w2 = width / 2, a.h2 = height / 2;
    t.l2.w2 = width / 4, t.l2.h2 = height / 4;
    prepare(*p, t.l1, kFromImage);
    prepare(*p, t.l2, kFromImage);
    if (!t.l1.vec || !t.l2.vec)
      fail(DWT2D_EINVAL, "forward_pair_strip: needs 16-byte aligned rows and widths divisible by 16");
    run_pair(*p, t, as_stream(stream));
  });
}

int dwt2d_inverse_level_strip(const dwt2d_plan* p, const float* const in[4], const size_t in_pitch[4],
                              const float* const top[4], const float* const bottom[4],
                              const size_t halo_pitch[4], float* image, size_t pitch, int width, int height,
                              void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !in || !in_pitch || !top || !bottom || !halo_pitch) fail(DWT2D_EINVAL, "null argument");
    if (width <= 0 || height <= 0 || width % 2 || height % 2)
      fail(DWT2D_EINVAL, "inverse_level_strip: strip sides must be positive and even");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    gpu::LevelArgs a{};
    for (int j = 0; j < 4; ++j) {
      a.in[j] = in[j], a.in_pitch[j] = (long long)in_pitch[j];
      a.halo_top[j] = top[j], a.halo_bot[j] = bottom[j];
      a.halo_top_pitch[j] = a.halo_bot_pitch[j] = (long long)halo_pitch[j];
      a.out[j] = image, a.out_pitch[j] = (long long)pitch;
    }
    a.halo = 1, a.up = p->up, a.down = p->down;
    a.w2 = width / 2, a.h2 = height / 2;
    launch(*p, a, kToImage, as_stream(stream));
  });
}

size_t dwt2d_workspace_bytes(int width, int height, int levels) {
  if (levels < 2 || width <= 0 || height <= 0) return 0;
  return ll_offset(width, height, levels) * sizeof(float);
}

int dwt2d_forward_mallat(const dwt2d_plan* p, const float* image, size_t pitch, int W, int H, int levels,
                         float* out, size_t out_pitch, void* scratch, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_mallat: plan is an inverse plan");
    check_pyramid(W, H, levels);
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    Workspace ws;
    get_workspace(ws, scratch, W, H, levels, as_stream(stream));
    forward_mallat(*p, image, pitch, W, H, levels, out, out_pitch, ws.ptr, as_stream(stream));
  });
}

int dwt2d_forward_mallat_ex(const dwt2d_plan* p, const float* image, size_t pitch, int W, int H, int levels,
                            float* out, size_t out_pitch, void* scratch, void* const* events, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_mallat: plan is an inverse plan");
    check_pyramid(W, H, levels);
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    Workspace ws;
    get_workspace(ws, scratch, W, H, levels, as_stream(stream));
    forward_mallat(*p, image, pitch, W, H, levels, out, out_pitch, ws.ptr, as_stream(stream), events);
  });
}

namespace {
// Library streams of a batch on one device (per thread, per device): images
// of the batch overlap on them, forked from and joined back to the caller's
// stream with events.
struct BatchLanes {
  static constexpr int kLanes = 4;
  cudaStream_t s[kLanes] = {};
  cudaEvent_t fork = nullptr, join[kLanes] = {};
};
BatchLanes& batch_lanes() {
  static thread_local std::unique_ptr<BatchLanes> per_dev[kMaxDevices];
  std::unique_ptr<BatchLanes>& b = per_dev[current_device()];
  if (!b) {
    auto n = std::make_unique<BatchLanes>();
    cuda_check(cudaEventCreateWithFlags(&n->fork, cudaEventDisableTiming), "batch fork event");
    for (int i = 0; i < BatchLanes::kLanes; ++i) {
      cuda_check(cudaStreamCreateWithFlags(&n->s[i], cudaStreamNonBlocking), "batch stream");
      cuda_check(cudaEventCreateWithFlags(&n->join[i], cudaEventDisableTiming), "batch join event");
    }
    b = std::move(n);
  }
  return *b;
}
}  // namespace

int dwt2d_forward_mallat_batch(const dwt2d_plan* p, int n, const float* const* images, size_t pitch, int W, int H,
                               int levels, float* const* outs, size_t out_pitch, int ndev, const int* devices,
                               void* const* streams) {
  return guard([&] {
    require_plan(p);
    if (n < 0 || (n > 0 && (!images || !outs))) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_mallat: plan is an inverse plan");
    check_pyramid(W, H, levels);
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    if (devices && ndev < 1) fail(DWT2D_EINVAL, "batch: ndev must be at least 1");
    if (!devices) ndev = 1;
    for (int i = 0; i < n; ++i)
      if (!images[i] || !outs[i]) fail(DWT2D_EINVAL, "batch: null image or output");
    for (int d = 0; d < ndev && d < n; ++d) {
      int dev = 0;
      if (devices) dev = devices[d];
      else cuda_check(cudaGetDevice(&dev), "current device");
      DeviceGuard g(dev);
      const cudaStream_t st = streams ? as_stream(streams[d]) : cudaStream_t(nullptr);
      std::vector<int> mine;
      for (int i = d; i < n; i += ndev) mine.push_back(i);
      // Images up to 32 MiB overlap on the library's lanes (their deep levels
      // are latency-bound: 16 x 2048^2 0.634 vs 0.834 ms sequential); larger
      // ones run in order on the caller's stream, where each pyramid keeps its
      // LL bands in L2 (8 x 4096^2: 0.70 ms in order, 0.88 ms overlapped).
      // scripts/probe_batch.py. One workspace per lane.
      const bool overlap = mine.size() > 1 && size_t(W) * size_t(H) * 4 <= (size_t(32) << 20);
      const int lanes = overlap ? std::min<int>(BatchLanes::kLanes, int(mine.size())) : 1;
      BatchLanes* b = overlap ? &batch_lanes() : nullptr;
      std::vector<Workspace> ws(lanes);
      auto lane_stream = [&](int k) { return b ? b->s[k] : st; };
      if (b) {
        cuda_check(cudaEventRecord(b->fork, st), "batch fork");
        for (int k = 0; k < lanes; ++k) cuda_check(cudaStreamWaitEvent(b->s[k], b->fork, 0), "batch fork");
      }
      // after the fork: inside a capture the lanes are capturing by now
      for (int k = 0; k < lanes; ++k) get_workspace(ws[k], nullptr, W, H, levels, lane_stream(k));
      for (size_t k = 0; k < mine.size(); ++k)
        forward_mallat(*p, images[mine[k]], pitch, W, H, levels, outs[mine[k]], out_pitch, ws[k % lanes].ptr,
                       lane_stream(int(k % lanes)));
      for (int k = 0; k < lanes; ++k) {
        ws[k].release();  // before the join: a capture must not end with work on an unjoined lane
        if (b) {
          cuda_check(cudaEventRecord(b->join[k], b->s[k]), "batch join");
          cuda_check(cudaStreamWaitEvent(st, b->join[k], 0), "batch join");
        }
      }
    }
  });
}

int dwt2d_event_create(void** ev) {
  return guard([&] {
    if (!ev) fail(DWT2D_EINVAL, "null argument");
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "event create");
    *ev = e;
  });
}

int dwt2d_event_destroy(void* ev) {
  return guard([&] {
    if (ev) cuda_check(cudaEventDestroy(static_cast<cudaEvent_t>(ev)), "event destroy");
  });
}

int dwt2d_event_elapsed_ms(void* a, void* b, float* ms) {
  return guard([&] {
    if (!a || !b || !ms) fail(DWT2D_EINVAL, "null argument");
    cuda_check(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)),
               "event elapsed");
  });
}

int dwt2d_inverse_mallat(const dwt2d_plan* p, const float* in, size_t in_pitch, int W, int H, int levels,
                         float* image, size_t pitch, void* scratch, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !in) fail(DWT2D_EINVAL, "null argument");
    if (p->forward) fail(DWT2D_EINVAL, "inverse_mallat: plan is not an inverse plan");
    check_pyramid(W, H, levels);
    Workspace ws;
    get_workspace(ws, scratch, W, H, levels, as_stream(stream));
    inverse_mallat(*p, in, in_pitch, W, H, levels, image, pitch, ws.ptr, as_stream(stream));
  });
}

int dwt2d_run_planar_host(const dwt2d_plan* p, const float* const in[4], float* const out[4], int w2, int h2) {
  return guard([&] {
    require_plan(p);
    if (!in || !out) fail(DWT2D_EINVAL, "null argument");
    if (w2 <= 0 || h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    HostPipe& hp = host_pipe();
    const size_t n = size_t(w2) * h2;
    float* dev = static_cast<float*>(hp.reserve(8 * n * sizeof(float)));
    const float* din[4];
    float* dout[4];
    size_t pitch[4];
    for (int j = 0; j < 4; ++j) {
      din[j] = dev + j * n;
      dout[j] = dev + (4 + j) * n;
      pitch[j] = size_t(w2);
      cuda_check(cudaMemcpyAsync(dev + j * n, in[j], n * 4, cudaMemcpyHostToDevice, hp.comp), "H2D");
    }
    if (is_identity(*p)) {
      copy_planes(din, pitch, dout, pitch, w2, h2, hp.comp);
    } else {
      gpu::LevelArgs a{};
      for (int j = 0; j < 4; ++j) {
        a.in[j] = din[j], a.out[j] = dout[j];
        a.in_pitch[j] = a.out_pitch[j] = w2;
      }
      a.w2 = w2, a.h2 = h2;
      launch(*p, a, kPlanar, hp.comp);
    }
    for (int j = 0; j < 4; ++j)
      cuda_check(cudaMemcpyAsync(out[j], dout[j], n * 4, cudaMemcpyDeviceToHost, hp.comp), "D2H");
    cuda_check(cudaStreamSynchronize(hp.comp), "synchronize");
  });
}

// ------------------------------------------------ float64 (C ABI)

int dwt2d_run_planar_f64(const dwt2d_plan* p, const double* const in[4], const size_t in_pitch[4],
                         double* const out[4], const size_t out_pitch[4], int w2, int h2, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!in || !out || !in_pitch || !out_pitch) fail(DWT2D_EINVAL, "null argument");
    if (w2 <= 0 || h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    for (int j = 0; j < 4; ++j)
      if (in_pitch[j] < size_t(w2) || out_pitch[j] < size_t(w2)) fail(DWT2D_EINVAL, "pitch < width");
    if (is_identity(*p)) return copy_planes64(in, in_pitch, out, out_pitch, w2, h2, as_stream(stream));
    Level64 lv{};
    for (int j = 0; j < 4; ++j)
      lv.in[j] = in[j], lv.in_pitch[j] = in_pitch[j], lv.out[j] = out[j], lv.out_pitch[j] = out_pitch[j];
    run_level64(*p, lv, kPlanar, w2, h2, as_stream(stream));
  });
}

int dwt2d_forward_level_f64(const dwt2d_plan* p, const double* image, size_t pitch, int width, int height,
                            double* const out[4], const size_t out_pitch[4], void* stream) {
  return guard([&] {
    require_plan(p);
    if (!image || !out || !out_pitch) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_level: plan is an inverse plan");
    if (width <= 0 || height <= 0 || width % 2 || height % 2) fail(DWT2D_EINVAL, "image sides must be positive and even");
    if (pitch < size_t(width)) fail(DWT2D_EINVAL, "pitch < width");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    Level64 lv{};
    for (int j = 0; j < 4; ++j) lv.in[j] = image, lv.in_pitch[j] = pitch, lv.out[j] = out[j], lv.out_pitch[j] = out_pitch[j];
    run_level64(*p, lv, kFromImage, width / 2, height / 2, as_stream(stream));
  });
}

int dwt2d_inverse_level_f64(const dwt2d_plan* p, const double* const in[4], const size_t in_pitch[4], double* image,
                            size_t pitch, int width, int height, void* stream) {
  return guard([&] {
    require_plan(p);
    if (!in || !in_pitch || !image) fail(DWT2D_EINVAL, "null argument");
    if (p->forward) fail(DWT2D_EINVAL, "inverse_level: plan is not an inverse plan");
    if (width <= 0 || height <= 0 || width % 2 || height % 2) fail(DWT2D_EINVAL, "image sides must be positive and even");
    if (pitch < size_t(width)) fail(DWT2D_EINVAL, "pitch < width");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    Level64 lv{};
    for (int j = 0; j < 4; ++j) lv.in[j] = in[j], lv.in_pitch[j] = in_pitch[j], lv.out[j] = image, lv.out_pitch[j] = pitch;
    run_level64(*p, lv, kToImage, width / 2, height / 2, as_stream(stream));
  });
}

int dwt2d_run_planar_host_f64(const dwt2d_plan* p, const double* const in[4], double* const out[4], int w2, int h2) {
  return guard([&] {
    require_plan(p);
    if (!in || !out) fail(DWT2D_EINVAL, "null argument");
    if (w2 <= 0 || h2 <= 0) fail(DWT2D_EINVAL, "run: empty input");
    HostPipe& hp = host_pipe();
    const size_t n = size_t(w2) * h2;
    double* dev = static_cast<double*>(hp.reserve(8 * n * sizeof(double)));
    Level64 lv{};
    for (int j = 0; j < 4; ++j) {
      lv.in[j] = dev + j * n, lv.out[j] = dev + (4 + j) * n;
      lv.in_pitch[j] = lv.out_pitch[j] = size_t(w2);
      cuda_check(cudaMemcpyAsync(dev + j * n, in[j], n * 8, cudaMemcpyHostToDevice, hp.comp), "H2D");
    }
    if (is_identity(*p)) copy_planes64(lv.in, lv.in_pitch, lv.out, lv.out_pitch, w2, h2, hp.comp);
    else run_level64(*p, lv, kPlanar, w2, h2, hp.comp);
    for (int j = 0; j < 4; ++j)
      cuda_check(cudaMemcpyAsync(out[j], lv.out[j], n * 8, cudaMemcpyDeviceToHost, hp.comp), "D2H");
    cuda_check(cudaStreamSynchronize(hp.comp), "synchronize");
  });
}

// ------------------------------------------------ sharded pyramid (C ABI)

int dwt2d_shard_create(const dwt2d_plan* p, int width, int strip_height, int levels, int rank, int world,
                       dwt2d_shard** out) {
  return guard([&] {
    require_plan(p);
    if (!out) fail(DWT2D_EINVAL, "null argument");
    *out = nullptr;
    if (!p->forward) fail(DWT2D_EINVAL, "shard: plan is an inverse plan");
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    if (!p->entry || p->extension != DWT2D_PERIODIC)
      fail(DWT2D_EUNSUPPORTED, "sharded pyramid: needs a fused kernel and periodic extension");
    if (world < 1 || rank < 0 || rank >= world) fail(DWT2D_EINVAL, "shard: rank outside [0, world)");
    check_pyramid(width, strip_height, levels);
    // every kernel the shard launches is loaded now: a kernel loaded lazily
    // at its first launch waits for the running kernels, and a halo wait
    // spinning on a rank whose work this thread has not launched yet would
    // never finish
    cuda_check(gpu::preload_exchange(), "exchange kernels");
    if (p->entry->preload) cuda_check(p->entry->preload(), "level kernels");
    auto sh = std::make_unique<dwt2d_shard>();
    sh->plan = p;
    sh->device = current_device();
    sh->rank = rank, sh->world = world, sh->W = width, sh->H = strip_height, sh->levels = levels;
    plan_steps(*sh);
    void* win = nullptr;
    cuda_check(cudaMalloc(&win, sh->window_bytes), "exchange window allocation");
    sh->window = static_cast<char*>(win);
    cuda_check(cudaMemset(sh->window, 0, kHeaderBytes), "exchange window init");
    const size_t ws = ll_offset(width, strip_height, levels) * sizeof(float);
    if (ws) {
      void* w = nullptr;
      cuda_check(cudaMalloc(&w, ws), "shard workspace allocation");
      sh->ws = static_cast<float*>(w);
    }
    void* dh = nullptr;
    cuda_check(cudaHostAlloc(&dh, 64, cudaHostAllocMapped | cudaHostAllocPortable), "shard diagnostics");
    sh->diag_host = static_cast<unsigned*>(dh);
    std::memset(sh->diag_host, 0, 64);
    void* dd = nullptr;
    cuda_check(cudaHostGetDevicePointer(&dd, dh, 0), "shard diagnostics");
    sh->diag_dev = static_cast<unsigned*>(dd);
    cuda_check(cudaDeviceSynchronize(), "exchange window init");
    if (world == 1) {  // the ring of one: pushes wrap the strip onto itself
      sh->prev = sh->next = sh.get();
      shard_connect_windows(*sh, sh->window, sh->window);
    }
    *out = sh.release();
  });
}

void dwt2d_shard_destroy(dwt2d_shard* s) { delete s; }

int dwt2d_shard_export(const dwt2d_shard* s, void* handle, size_t len) {
  return guard([&] {
    if (!s || !handle) fail(DWT2D_EINVAL, "null argument");
    if (len < sizeof(cudaIpcMemHandle_t)) fail(DWT2D_EINVAL, "shard_export: handle buffer too small");
    DeviceGuard g(s->device);
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, s->window), "IPC handle of the exchange window");
    std::memcpy(handle, &h, sizeof h);
  });
}

int dwt2d_shard_connect(dwt2d_shard* s, const dwt2d_shard* prev, const dwt2d_shard* next) {
  return guard([&] {
    if (!s || !prev || !next) fail(DWT2D_EINVAL, "null argument");
    for (const dwt2d_shard* n : {prev, next})
      if (n->W != s->W || n->H != s->H || n->levels != s->levels || n->steps.size() != s->steps.size() ||
          n->window_bytes != s->window_bytes)
        fail(DWT2D_EINVAL, "shard_connect: neighbours must share width, strip height, levels and plan geometry");
    DeviceGuard g(s->device);
    for (const dwt2d_shard* n : {prev, next})
      if (n->device != s->device) {
        int can = 0;
        cuda_check(cudaDeviceCanAccessPeer(&can, s->device, n->device), "peer access query");
        if (!can) fail(DWT2D_EUNSUPPORTED, "shard_connect: no peer access between the devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(n->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "enable peer access");
        cudaGetLastError();
      }
    s->prev = prev, s->next = next;
    shard_connect_windows(*s, prev->window, next->window);
  });
}

int dwt2d_shard_connect_ipc(dwt2d_shard* s, const void* prev_handle, const void* next_handle) {
  return guard([&] {
    if (!s || !prev_handle || !next_handle) fail(DWT2D_EINVAL, "null argument");
    DeviceGuard g(s->device);
    cudaIpcMemHandle_t hp, hn;
    std::memcpy(&hp, prev_handle, sizeof hp);
    std::memcpy(&hn, next_handle, sizeof hn);
    void* pp = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&pp, hp, cudaIpcMemLazyEnablePeerAccess), "open the previous rank's window");
    s->ipc_open[0] = static_cast<char*>(pp);
    void* pn = pp;
    if (std::memcmp(&hp, &hn, sizeof hp) != 0) {  // two ranks: prev == next, opened once
      cuda_check(cudaIpcOpenMemHandle(&pn, hn, cudaIpcMemLazyEnablePeerAccess), "open the next rank's window");
      s->ipc_open[1] = static_cast<char*>(pn);
    }
    s->prev = s->next = nullptr;
    shard_connect_windows(*s, static_cast<char*>(pp), static_cast<char*>(pn));
  });
}

int dwt2d_shard_forward_mallat_ex(dwt2d_shard* s, const float* strip, size_t pitch, float* out, size_t out_pitch,
                                  void* const* events, void* stream) {
  return guard([&] {
    if (!s) fail(DWT2D_EINVAL, "null argument");
    check_shard_args(*s, strip, out);
    DeviceGuard g(s->device);
    const cudaStream_t st = as_stream(stream);
    shard_start(*s, st);
    if (events) record(events[0], st);
    for (size_t e = 0; e < s->steps.size(); ++e) {
      void* const* ev = events ? events + 1 + 4 * e : nullptr;
      const StepIO io = step_input(*s, e, strip, pitch, out, out_pitch);
      const bool split = split_step(*s, e);
      shard_push(*s, e, io, !split, st);
      if (ev) record(ev[0], st);
      if (split) shard_compute(*s, e, io, out, out_pitch, 0, st);
      if (ev) record(ev[1], st);
      if (split) shard_wait(*s, st);
      if (ev) record(ev[2], st);
      shard_compute(*s, e, io, out, out_pitch, split ? 1 : 2, st);
      if (ev) record(ev[3], st);
    }
    shard_done(*s, st);
  });
}

int dwt2d_shard_forward_mallat(dwt2d_shard* s, const float* strip, size_t pitch, float* out, size_t out_pitch,
                               void* stream) {
  return dwt2d_shard_forward_mallat_ex(s, strip, pitch, out, out_pitch, nullptr, stream);
}

int dwt2d_shard_info(const dwt2d_shard* s, int* steps, int* pair, size_t* halo_bytes) {
  return guard([&] {
    if (!s) fail(DWT2D_EINVAL, "null argument");
    if (steps) *steps = int(s->steps.size());
    if (pair) *pair = !s->steps.empty() && s->steps[0].pair ? 1 : 0;
    if (halo_bytes) {  // bytes this rank pushes to its neighbours per pyramid
      size_t b = 0;
      for (const ExchangeStep& x : s->steps) b += size_t(x.trows + x.brows) * size_t(x.width) * sizeof(float);
      *halo_bytes = b;
    }
  });
}

int dwt2d_shard_status(const dwt2d_shard* s, int* error) {
  return guard([&] {
    if (!s || !error) fail(DWT2D_EINVAL, "null argument");
    // host-mapped: no CUDA call, so it also answers after a trap
    const volatile unsigned* d = s->diag_host;
    *error = int(d[0]);
    if (d[0]) {
      static const char* const what[] = {"", "a neighbour never finished the previous pyramid",
                                         "the rows from the previous rank never arrived",
                                         "the rows from the next rank never arrived"};
      g_error = std::string("sharded pyramid rank ") + std::to_string(s->rank) + ": " + what[d[0] & 3] +
                " (counter " + std::to_string(d[1]) + ", waited for " + std::to_string(d[2]) + ")";
    }
  });
}

int dwt2d_forward_mallat_sharded(const dwt2d_plan* p, int nranks, const int* devices, const float* const* strips,
                                 const size_t* pitch, int width, int strip_height, int levels, float* const* out,
                                 const size_t* out_pitch, void* const* streams) {
  return guard([&] {
    require_plan(p);
    if (nranks < 1 || !devices || !strips || !pitch || !out || !out_pitch) fail(DWT2D_EINVAL, "null argument");
    // shards of this ring geometry, created and connected on first use
    std::vector<long long> key{nranks, width, strip_height, levels};
    for (int r = 0; r < nranks; ++r) key.push_back(devices[r]);
    std::vector<dwt2d_shard*>* ring = nullptr;
    {
      std::lock_guard<std::mutex> lk(p->shard_mu);
      for (auto& c : p->shard_cache)
        if (c.key == key) ring = &c.shards;
      if (!ring) {
        dwt2d_plan::ShardRing sr;
        sr.key = key;
        for (int r = 0; r < nranks; ++r) {
          DeviceGuard g(devices[r]);
          dwt2d_shard* sh = nullptr;
          const int rc = dwt2d_shard_create(p, width, strip_height, levels, r, nranks, &sh);
          if (rc != DWT2D_OK) {
            for (dwt2d_shard* o : sr.shards) delete o;
            fail(rc, g_error);
          }
          sr.shards.push_back(sh);
        }
        for (int r = 0; r < nranks && nranks > 1; ++r) {
          const int rc = dwt2d_shard_connect(sr.shards[r], sr.shards[(r + nranks - 1) % nranks],
                                             sr.shards[(r + 1) % nranks]);
          if (rc != DWT2D_OK) {
            for (dwt2d_shard* o : sr.shards) delete o;
            fail(rc, g_error);
          }
        }
        p->shard_cache.push_back(std::move(sr));
        ring = &p->shard_cache.back().shards;
      }
    }
    std::vector<dwt2d_shard*>& sh = *ring;
    for (int r = 0; r < nranks; ++r) check_shard_args(*sh[r], strips[r], out[r]);
    auto st = [&](int r) { return streams ? as_stream(streams[r]) : cudaStream_t(nullptr); };
    // phase-major enqueue: every rank's push of a step before any rank's
    // wait, so ranks sharing a device (or a stream) cannot block each other
    for (int r = 0; r < nranks; ++r) {
      DeviceGuard g(sh[r]->device);
      shard_start(*sh[r], st(r));
    }
    for (size_t e = 0; e < sh[0]->steps.size(); ++e) {
      std::vector<StepIO> io;
      for (int r = 0; r < nranks; ++r) io.push_back(step_input(*sh[r], e, strips[r], pitch[r], out[r], out_pitch[r]));
      // push-and-wait in one launch is only safe phase-major when the ranks
      // run on distinct streams; ranks sharing a stream always split
      bool shared = false;
      for (int r = 0; r < nranks && !shared; ++r)
        for (int q = 0; q < r && !shared; ++q) shared = st(q) == st(r) && sh[q]->device == sh[r]->device;
      const bool split = shared || split_step(*sh[0], e);
      for (int r = 0; r < nranks; ++r) {
        DeviceGuard g(sh[r]->device);
        shard_push(*sh[r], e, io[r], !split, st(r));
      }
      if (split) {
        for (int r = 0; r < nranks; ++r) {
          DeviceGuard g(sh[r]->device);
          shard_compute(*sh[r], e, io[r], out[r], out_pitch[r], 0, st(r));
        }
      }
      for (int r = 0; r < nranks; ++r) {
        DeviceGuard g(sh[r]->device);
        if (split) shard_wait(*sh[r], st(r));
        shard_compute(*sh[r], e, io[r], out[r], out_pitch[r], split ? 1 : 2, st(r));
      }
    }
    for (int r = 0; r < nranks; ++r) {
      DeviceGuard g(sh[r]->device);
      shard_done(*sh[r], st(r));
    }
  });
}

int dwt2d_forward_mallat_host(const dwt2d_plan* p, const float* image, int W, int H, int levels, float* out) {
  return guard([&] {
    require_plan(p);
    if (!image || !out) fail(DWT2D_EINVAL, "null argument");
    if (!p->forward) fail(DWT2D_EINVAL, "forward_mallat: plan is an inverse plan");
    check_pyramid(W, H, levels);
    if (is_identity(*p)) fail(DWT2D_EUNSUPPORTED, "identity program");
    if (!(p->entry && p->extension == DWT2D_PERIODIC && forward_mallat_host_pipelined(*p, image, W, H, levels, out))) {
      HostPipe& hp = host_pipe();
      const size_t n = size_t(W) * H;
      const size_t ws_bytes = dwt2d_workspace_bytes(W, H, levels);
      float* d_img = static_cast<float*>(hp.reserve(2 * n * 4 + ws_bytes + 256));
      float* d_out = d_img + n;
      float* ws = d_out + ((n + 63) & ~size_t(63));
      cuda_check(cudaMemcpyAsync(d_img, image, n * 4, cudaMemcpyHostToDevice, hp.comp), "H2D");
      forward_mallat(*p, d_img, W, W, H, levels, d_out, W, ws, hp.comp);
      cuda_check(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, hp.comp), "D2H");
      cuda_check(cudaStreamSynchronize(hp.comp), "synchronize");
    }
  });
}

int dwt2d_time_forward(const dwt2d_plan* p, int W, int H, int levels, int repeats, uint64_t seed,
                       double* median_seconds) {
  return guard([&] {
    require_plan(p);
    if (!median_seconds) fail(DWT2D_EINVAL, "null argument");
    if (repeats < 1) fail(DWT2D_EINVAL, "bench: repeats must be at least 1");
    if (!p->forward) fail(DWT2D_EINVAL, "bench: plan is an inverse plan");
    if (levels == 1) {
      if (W <= 0 || H <= 0 || W % 2 || H % 2) fail(DWT2D_EINVAL, "bench: sizes must be positive and even");
    } else {
      check_pyramid(W, H, levels);
    }
    const ImagePlane<float> img = random_image<float>(W, H, seed);
    HostPipe& hp = host_pipe();
    const size_t n = size_t(W) * H;
    const size_t ws_bytes = levels > 1 ? dwt2d_workspace_bytes(W, H, levels) : 0;
    float* d = static_cast<float*>(hp.reserve(2 * n * 4 + ws_bytes + 256));
    float* d_out = d + n;
    float* ws = d_out + ((n + 63) & ~size_t(63));
    const int w2 = W / 2, h2 = H / 2;
    const size_t q = size_t(w2) * h2;
    if (levels == 1) {  // the reference times run() on the polyphase planes
      const PolyphaseImage<float> poly = polyphase_split(img);
      for (int j = 0; j < 4; ++j)
        cuda_check(cudaMemcpyAsync(d + j * q, poly.comp[j].samples.data(), q * 4, cudaMemcpyHostToDevice, hp.comp),
                   "H2D");
    } else {
      cuda_check(cudaMemcpyAsync(d, img.samples.data(), n * 4, cudaMemcpyHostToDevice, hp.comp), "H2D");
    }
    auto once = [&] {
      if (levels == 1) {
        if (is_identity(*p)) return;
        gpu::LevelArgs a{};
        for (int j = 0; j < 4; ++j) {
          a.in[j] = d + j * q, a.out[j] = d_out + j * q;
          a.in_pitch[j] = a.out_pitch[j] = w2;
        }
        a.w2 = w2, a.h2 = h2;
        launch(*p, a, kPlanar, hp.comp);
      } else {
        forward_mallat(*p, d, W, W, H, levels, d_out, W, ws, hp.comp);
      }
    };
    once();
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    std::vector<double> t;
    for (int r = 0; r < repeats; ++r) {
      cuda_check(cudaEventRecord(e0, hp.comp), "record");
      once();
      cuda_check(cudaEventRecord(e1, hp.comp), "record");
      cuda_check(cudaEventSynchronize(e1), "synchronize");
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      t.push_back(ms * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::sort(t.begin(), t.end());
    const size_t m = t.size();
    *median_seconds = m % 2 ? t[m / 2] : 0.5 * (t[m / 2 - 1] + t[m / 2]);
  });
}

int dwt2d_inverse_mallat_host(const dwt2d_plan* p, const float* in, int W, int H, int levels, float* image) {
  return guard([&] {
    require_plan(p);
    if (!image || !in) fail(DWT2D_EINVAL, "null argument");
    if (p->forward) fail(DWT2D_EINVAL, "inverse_mallat: plan is not an inverse plan");
    check_pyramid(W, H, levels);
    HostPipe& hp = host_pipe();
    const size_t n = size_t(W) * H;
    const size_t ws_bytes = dwt2d_workspace_bytes(W, H, levels);
    float* d_in = static_cast<float*>(hp.reserve(2 * n * 4 + ws_bytes + 256));
    float* d_img = d_in + n;
    float* ws = d_img + ((n + 63) & ~size_t(63));
    cuda_check(cudaMemcpyAsync(d_in, in, n * 4, cudaMemcpyHostToDevice, hp.comp), "H2D");
    inverse_mallat(*p, d_in, W, W, H, levels, d_img, W, ws, hp.comp);
    cuda_check(cudaMemcpyAsync(image, d_img, n * 4, cudaMemcpyDeviceToHost, hp.comp), "D2H");
    cuda_check(cudaStreamSynchronize(hp.comp), "synchronize");
  });
}

}  // extern "C"
