// Plain C++ types shared by the host runtime (compiled with g++) and the
// CUDA level kernels: launch arguments, tap tables, registry entries.
#pragma once

#include <cuda_runtime_api.h>

#include <vector>

namespace dwt2d_b200 {
namespace gpu {

#ifndef DWT2D_WARPS_PER_CTA
#define DWT2D_WARPS_PER_CTA 4
#endif
constexpr int kWarpsPerCta = DWT2D_WARPS_PER_CTA;
constexpr int kOutLanes = 30;  // lanes 1..30 store, 0 and 31 are halo

struct TapDesc {
  int j;   // source component
  int dm;  // component-grid column offset
  int dn;  // component-grid row offset
  float w;
};

struct RowDesc {
  int ident;  // 1: output component = input component (no arithmetic)
  int tb, te; // tap range [tb, te)
  float scale;
};

// Arguments of one level launch. Pitches are in floats.
struct LevelArgs {
  const float* in[4];   // interleaved input: in[0] is the image (2*h2 rows)
  long long in_pitch[4];
  float* out[4];        // interleaved output: out[0] is the image
  long long out_pitch[4];
  int w2, h2;           // component grid size
  int nstrips;          // ceil(w2 / (30 * CW))
  int nchunks;          // ceil((y_end - y_begin) / chunk_rows)
  int chunk_rows;
  int y_begin, y_end;   // output component rows covered by the chunks (y_end 0: h2)
  int vec;              // 1: vector fast path valid (w2 % CW == 0, 16 B aligned)
  int reverse;          // 1: hand out chunks bottom-up (see capi.cpp forward_mallat)
  int alternate;        // 1: odd chunks stream bottom-up (shared warm-up rows hit L2)
  int staged;           // 1: interleaved input rows staged in shared memory by TMA
  int pdl;              // host only: launch with programmatic dependent launch
  // outputs stored only inside [keep_x0, keep_x1) x [keep_y0, keep_y1)
  // (component grid; keep_x1 / keep_y1 == 0: to the level's edge): a symmetric level's
  // interior, its border bands come from the crop kernel
  int keep_x0, keep_x1, keep_y0, keep_y1;
  int wait_end;         // PDL wait at the end of the kernel instead of its start (level_engine.cuh)
  float neg_zero;       // -0.0f (set by the host: an operand ptxas cannot fold, level_engine.cuh)
  // Row strips (multi-GPU): when halo != 0, component rows above the strip
  // (y < 0) come from halo_top (row y + up) and rows below (y >= h2) from
  // halo_bot (row y - h2) instead of wrapping periodically inside the strip.
  // Same layout as `in` (interleaved: two image rows per component row).
  int halo;
  int up, down;         // halo rows available above / below (component rows)
  const float* halo_top[4];
  long long halo_top_pitch[4];
  const float* halo_bot[4];
  long long halo_bot_pitch[4];
};

using LevelLaunch = cudaError_t (*)(const LevelArgs&, cudaStream_t);

// Levels 1 and 2 of a forward pyramid in one pass (pair_engine.cuh): l1 is
// the image level (its LL band is never written: l1.out[0] unused), l2 the
// next level (l2.in unused). Work items: (strip, chunk of level-2 rows).
constexpr int kPairLanes = 28;  // lanes 2..29 store both levels
struct PairArgs {
  LevelArgs l1, l2;
  int nstrips, chunk_rows, nchunks;
  int m_begin, m_end;   // level-2 output rows covered by the chunks (m_end 0: l2.h2)
};
using PairLaunch = cudaError_t (*)(const PairArgs&, cudaStream_t);


// compiled border crops of a plan (crop_engine.cuh): all sub-steps of the
// border bands (CropTileArgs, below) with the tap tables compiled in; aw x ah
// bounds the tile areas of the launch (shared-memory size)
struct CropTileArgs;
constexpr int kCropThreads = 256;  // one tile-area cell and one ghost cell per thread
// ghost ring cells of an aw x ah tile area with ring width r
constexpr int crop_ring_cells(int aw, int ah, int r) { return 2 * r * (aw + 2 * r) + 2 * r * ah; }
using CropLaunch = cudaError_t (*)(const CropTileArgs&, int aw, int ah, bool pdl, cudaStream_t);

// resident CTAs per SM of a launcher's vector-path kernel (0 if unknown)
using LevelOccupancy = int (*)();

struct PlanEntry {
  const char* key;
  unsigned long long fingerprint;
  int cw;                      // component columns per lane
  int stage_ok;                // TMA-staged rows measured faster (CW 4 programs)
  int up, down, left, right;   // level reach on the component grid
  long taps_per_quad;
  LevelLaunch planar;          // 4 planes -> 4 planes   (run() API)
  LevelLaunch from_image;      // interleaved -> 4 planes (forward levels)
  LevelLaunch to_image;        // 4 planes -> interleaved (inverse levels)
  LevelOccupancy occupancy;    // resident CTAs per SM (vector path)
  PairLaunch pair;             // levels 1+2 in one pass (forward plans with reach <= 2, CW 4)
  LevelOccupancy pair_occupancy;
  CropLaunch crop;             // symmetric border bands, compiled taps
  int crop_reach;              // largest reach of one sub-step (the crop kernel's ghost ring)
  // loads every kernel of the entry into the context now (lazy module
  // loading would otherwise load at first launch, which waits for running
  // kernels: a deadlock when one of them spins on work not yet launched)
  cudaError_t (*preload)();
};

// One sub-step of the generic executor (kernels/generic_step.cu). `taps`
// points to device memory owned by the plan.
struct GenericStepArgs {
  const float* in[4];
  long long in_pitch[4];
  int in_il;             // in[0] is an interleaved image
  float* out[4];
  long long out_pitch[4];
  int out_il;            // out[0] is an interleaved image
  int w2, h2;            // grid of this pass (a whole level, or a crop of it)
  int symmetric;         // extend_index rule on the component grid
  int fma;               // rounding model (see lowering.hpp)
  int kx0, kx1, ky0, ky1;  // outputs written only inside this window
  RowDesc rows[4];
  const TapDesc* taps;
};
// All sub-steps of a program over the border crops of a symmetric level in ONE
// launch (generic_step.cu: crop_tile_kernel): every CTA takes a tile of one
// crop (core + margins along the crop's long side), keeps it in shared memory
// through all sub-steps and writes the kept part of its core.
struct CropRegion {
  int x0, y0, w, h;        // crop on the component grid (extension at its edges)
  int kx0, kx1, ky0, ky1;  // outputs written (crop coordinates)
  int along_x;             // tiles run along x (row bands) or along y (column bands)
  int tiles;
};
struct CropTileArgs {
  const float* in[4];
  long long in_pitch[4];
  int in_il;
  float* out[4];
  long long out_pitch[4];
  int out_il;
  int nsteps, symmetric, fma;
  int core, mlo, mhi;      // tile core length and margins along the long side
  int nreg;
  CropRegion reg[4];
  const RowDesc* rows;     // nsteps * 4 (device)
  const TapDesc* taps;     // (device)
  int w2, h2;              // the level grid (true image edges; compiled crop kernel)
};

cudaError_t launch_crop_tiles(const CropTileArgs& a, int smem_floats, bool pdl, cudaStream_t st);

// The generic executor in float64 (compile<double>): the same pass with
// double data, weights and scales.
struct TapDesc64 {
  int j, dm, dn;
  double w;
};
struct RowDesc64 {
  int ident, tb, te;
  double scale;
};
struct GenericStepArgs64 {
  const double* in[4];
  long long in_pitch[4];
  int in_il;
  double* out[4];
  long long out_pitch[4];
  int out_il;
  int w2, h2;
  int symmetric;
  int fma;
  int kx0, kx1, ky0, ky1;
  RowDesc64 rows[4];
  const TapDesc64* taps;
};
cudaError_t launch_generic_step64(const GenericStepArgs64& a, cudaStream_t st);

// up to kMaxGenericRegions independent passes (same sub-step, different
// grids) in one launch
constexpr int kMaxGenericRegions = 4;
cudaError_t launch_generic_step(const GenericStepArgs* a, int n, bool pdl, cudaStream_t st);

// Halo exchange of a row-strip sharded pyramid over peer memory
// (kernels/exchange.cu). Pointers named prev/next live in the ring
// neighbours' exchange windows (peer-mapped), the rest in this rank's.
struct HaloPushArgs {
  const float* src;      // the level input strip (height x width, src_pitch)
  long long src_pitch;
  int width, height;
  int rows_first;        // src rows [0, rows_first) -> dst_prev (prev's bottom halo)
  int rows_last;         // src rows [height - rows_last, height) -> dst_next (next's top halo)
  float* dst_prev;
  float* dst_next;
  long long dst_pitch;
  int vec;               // width, pitches and pointers allow float4 copies
  unsigned* flag_prev;   // prev's bottom-halo arrival counter
  unsigned* flag_next;   // next's top-halo arrival counter
  unsigned* arrive;      // this rank's CTA arrival counter (last CTA signals)
  unsigned* error;       // diagnostics block (host-mapped): code, counter value, target
  unsigned long long timeout_ns;
  // wait_after: the CTA that signals also waits for this rank's own halo
  // arrivals (my_top / my_bot counters past seen[0] / seen[1]) before the
  // kernel ends: push + wait in one launch (small levels, no interior split)
  int wait_after;
  const unsigned* my_top;
  const unsigned* my_bot;
  unsigned* seen;
  int pdl;               // host only: launch with programmatic dependent launch
};
cudaError_t launch_halo_push(const HaloPushArgs& a, int sms, cudaStream_t st);
cudaError_t launch_halo_wait(const unsigned* top_flag, const unsigned* bot_flag, unsigned* seen, unsigned* error,
                             unsigned long long timeout_ns, cudaStream_t st);
cudaError_t launch_pyramid_done(unsigned* done_prev, unsigned* done_next, unsigned* pyramids, cudaStream_t st);
cudaError_t launch_pyramid_start(const unsigned* done, const unsigned* pyramids, unsigned* error,
                                 unsigned long long timeout_ns, cudaStream_t st);
cudaError_t preload_exchange();

const std::vector<PlanEntry>& plan_registry();
const PlanEntry* find_plan(unsigned long long fingerprint);

}  // namespace gpu
}  // namespace dwt2d_b200
