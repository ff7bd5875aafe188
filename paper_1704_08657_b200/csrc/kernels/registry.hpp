// Registry of ahead-of-time compiled level kernels, one entry per lowered
// StepProgram of the built-in wavelets. Runtime plans are matched by the
// fingerprint of their tap tables, so the kernel that runs is provably the
// one generated from the same lowering.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "level_engine.cuh"
#include "level_types.hpp"

namespace dwt2d_b200 {
namespace gpu {

constexpr int kPrefetchRows = 2;

template <class P, bool IN_IL, bool OUT_IL>
cudaError_t launch_level(const LevelArgs& a, cudaStream_t st) {
  const long long warps = (long long)a.nstrips * a.nchunks;
  if (warps <= 0) return cudaSuccess;
  const unsigned blocks = unsigned((warps + kWarpsPerCta - 1) / kWarpsPerCta);
  if (a.vec)
    level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true><<<blocks, kWarpsPerCta * 32, 0, st>>>(a);
  else
    level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, false><<<blocks, kWarpsPerCta * 32, 0, st>>>(a);
  return cudaGetLastError();
}

template <class P, bool IN_IL, bool OUT_IL>
int level_occupancy() {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &blocks, level_kernel<P, kPrefetchRows, IN_IL, OUT_IL, true>, kWarpsPerCta * 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

template <class P>
cudaError_t launch_wave(const WaveArgs& t, int blocks, cudaStream_t st) {
  wave_kernel<P, kPrefetchRows, true, false><<<blocks, kWarpsPerCta * 32, 0, st>>>(t);
  return cudaGetLastError();
}

template <class P>
int wave_occupancy() {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, wave_kernel<P, kPrefetchRows, true, false>,
                                                    kWarpsPerCta * 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

template <class P, bool kForward>
PlanEntry make_entry() {
  using M = Meta<P>;
  PlanEntry e{};
  e.key = P::kKey;
  e.fingerprint = P::kFingerprint;
  e.cw = P::kCW;
  e.up = M::U, e.down = M::L, e.left = M::HL, e.right = M::HR;
  e.taps_per_quad = P::kTaps;
  e.planar = &launch_level<P, false, false>;
  if constexpr (kForward) {
    e.from_image = &launch_level<P, true, false>;
    e.occupancy = &level_occupancy<P, true, false>;
    e.wave = &launch_wave<P>;
    e.wave_occupancy = &wave_occupancy<P>;
  } else {
    e.to_image = &launch_level<P, false, true>;
    e.occupancy = &level_occupancy<P, false, true>;
  }
  return e;
}

}  // namespace gpu
}  // namespace dwt2d_b200
