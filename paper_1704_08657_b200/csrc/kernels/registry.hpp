// Registry of ahead-of-time compiled level kernels, one entry per lowered
// StepProgram of the built-in wavelets. Runtime plans are matched by the
// fingerprint of their tap tables, so the kernel that runs is provably the
// one generated from the same lowering.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <vector>

#include "level_engine.cuh"
#include "pair_engine.cuh"
#include "crop_engine.cuh"
#include "level_types.hpp"

namespace dwt2d_b200 {
namespace gpu {

constexpr int kPrefetchRows = 2;

// Level launches use programmatic dependent launch (PDL): the kernel waits
// for the previous kernel in the stream (griddepcontrol.wait) before it
// reads anything and lets the next one launch once all its own CTAs have
// started, so consecutive levels overlap launch latency and CTA ramp-up with
// the previous level's last wave. LevelArgs::pdl = 0 (plan tuning "pdl")
// disables it.

// Opt a kernel into `bytes` of dynamic shared memory once per device (the
// attribute is per function and device; a process may drive several GPUs).
// One cache per kernel: the kernel is the template argument.
template <auto kernel>
cudaError_t allow_smem(int bytes) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_relaxed);
  return e;
}

template <class P, bool IN_IL, bool OUT_IL>
cudaError_t launch_level(const LevelArgs& a, cudaStream_t st) {
  const long long warps = (long long)a.nstrips * a.nchunks;
  if (warps <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned((warps + kWarpsPerCta - 1) / kWarpsPerCta));
  cfg.blockDim = dim3(kWarpsPerCta * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  if constexpr (IN_IL || (OUT_IL && P::kCW == 4)) {
    if (a.vec && a.staged) {  // TMA-staged rows (level_engine.cuh: TmaRowReader / TmaPlanarReader)
      auto k = level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true, true>;
      const cudaError_t attr_ok =
          allow_smem<level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true, true>>(staged_bytes<P::kCW>());
      if (attr_ok != cudaSuccess) return attr_ok;
      cfg.dynamicSmemBytes = staged_bytes<P::kCW>();
      return cudaLaunchKernelEx(&cfg, k, a);
    }
  }
  if (a.vec) return cudaLaunchKernelEx(&cfg, level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true>, a);
  return cudaLaunchKernelEx(&cfg, level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, false>, a);
}

template <class P, bool IN_IL, bool OUT_IL>
int level_occupancy() {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true>,
                                                    kWarpsPerCta * 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

template <class P>
cudaError_t launch_pair(const PairArgs& t, cudaStream_t st) {
  static_assert(pair_lanes<P, 4>() == kPairLanes, "host strip width (kPairLanes) != the pair kernel's");
  const long long warps = (long long)t.nstrips * t.nchunks;
  if (warps <= 0) return cudaSuccess;
  auto k = pair_kernel<P>;
  const cudaError_t attr_ok = allow_smem<pair_kernel<P>>(staged_bytes<4>());
  if (attr_ok != cudaSuccess) return attr_ok;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned((warps + kWarpsPerCta - 1) / kWarpsPerCta));
  cfg.blockDim = dim3(kWarpsPerCta * 32);
  cfg.dynamicSmemBytes = staged_bytes<4>();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = t.l1.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, t);
}

template <class P>
int pair_occupancy() {
  int blocks = 0;
  cudaFuncSetAttribute(pair_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, staged_bytes<4>());
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pair_kernel<P>, kWarpsPerCta * 32, staged_bytes<4>()) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

template <class P>
cudaError_t launch_crop(const CropTileArgs& a, int aw, int ah, bool pdl, cudaStream_t st) {
  int tiles = 0;
  for (int i = 0; i < a.nreg; ++i) tiles += a.reg[i].tiles;
  if (tiles == 0) return cudaSuccess;
  const int bytes = crop_smem_floats<P>(aw, ah) * 4;
  if (bytes > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(crop_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(tiles));
  cfg.blockDim = dim3(kCropThreads);
  cfg.dynamicSmemBytes = size_t(bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, crop_kernel<P>, a);
}

template <class P, bool kForward>
cudaError_t preload_entry() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  auto load = [&](const void* f) {
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f);
  };
  load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, false, false, true>));
  load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, false, false, false>));
  load(reinterpret_cast<const void*>(crop_kernel<P>));
  if constexpr (kForward) {
    load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, true, false, true>));
    load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, true, false, false>));
    load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, true, false, true, true>));
    if constexpr (PairTraits<P>::ok && (P::kAlt || P::kFma)) load(reinterpret_cast<const void*>(pair_kernel<P>));
  } else {
    load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, false, true, true>));
    load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, false, true, false>));
    if constexpr (P::kCW == 4) load(reinterpret_cast<const void*>(level_kernel<P, kPrefetchRows, false, true, true, true>));
  }
  return e;
}

template <class P, bool kForward>
PlanEntry make_entry() {
  using M = Meta<P>;
  PlanEntry e{};
  e.key = P::kKey;
  e.fingerprint = P::kFingerprint;
  e.cw = P::kCW;
  // CW-2 programs measured slower staged (scripts/probe_level_schemes.py),
  // and so did the shifted-window ones (polyconvolution baseline 16384^2:
  // 684 vs 644 us; non-separable convolution baseline 1265 vs 1264)
  e.stage_ok = (P::kCW == 4 && !shift_rows<P>()) ? 1 : 0;
  e.up = M::U, e.down = M::L, e.left = M::HL, e.right = M::HR;
  e.taps_per_quad = P::kTaps;
  e.planar = &launch_level<P, false, false>;
  e.crop = &launch_crop<P>;
  e.crop_reach = CropGeom<P>::R;
  e.preload = &preload_entry<P, kForward>;
  if constexpr (kForward) {
    e.from_image = &launch_level<P, true, false>;
    e.occupancy = &level_occupancy<P, true, false>;
    if constexpr (PairTraits<P>::ok && (P::kAlt || P::kFma)) {
      e.pair = &launch_pair<P>;
      e.pair_occupancy = &pair_occupancy<P>;
    }
  } else {
    e.to_image = &launch_level<P, false, true>;
    e.occupancy = &level_occupancy<P, false, true>;
  }
  return e;
}

}  // namespace gpu
}  // namespace dwt2d_b200
