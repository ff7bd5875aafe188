// Generic GPU executor: one pass per lowered sub-step with the taps read from
// a device table at run time — the reference's execution model
// (proj/include/dwt2d/executor.hpp:146-238: one barrier-separated pass per
// kernel, every tap through extend_index) on the GPU. It serves the programs
// the fused AOT level kernels do not cover: symmetric extension (which
// reflects every intermediate, incompatible with one streaming pass) and
// definition-file wavelets of new shapes. Same accumulation order and
// rounding as the fused kernels, so periodic results are bit-identical to
// them and composed results to the reference's float32 executor. One launch
// can run the same sub-step over up to four grids (the border crops of the
// symmetric path, capi.cpp: run_symmetric).
#include <cuda_runtime.h>

#include "level_types.hpp"

namespace dwt2d_b200 {
namespace gpu {

bool pdl_enabled();

namespace {

__device__ __forceinline__ int extend(int i, int n, int symmetric) {
  if (i >= 0 && i < n) return i;
  if (!symmetric) {
    const int r = i % n;
    return r < 0 ? r + n : r;
  }
  if (n == 1) return 0;
  const int period = 2 * n - 2;
  int r = i % period;
  if (r < 0) r += period;
  return r < n ? r : period - r;
}

__device__ __forceinline__ float load(const GenericStepArgs& a, int j, int x, int y) {
  if (a.in_il) return a.in[0][(2ll * y + (j >> 1)) * a.in_pitch[0] + 2ll * x + (j & 1)];
  return a.in[j][(long long)y * a.in_pitch[j] + x];
}

// regions of very different shapes (full-width row bands, full-height column
// bands) share one flat grid: region i owns blocks [first[i], first[i+1]),
// tiles of 32 x 8 in row-major order over its grid
struct GenericBatch {
  GenericStepArgs r[kMaxGenericRegions];
  int first[kMaxGenericRegions + 1];
  int tiles_x[kMaxGenericRegions];
  int n;
};

__global__ void __launch_bounds__(256) generic_step_kernel(const __grid_constant__ GenericBatch b) {
  // PDL: chains of sub-steps (symmetric border crops) overlap each launch
  // with the previous step's tail; no-ops for a normal launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  int i = 0;
  while (i + 1 < b.n && int(blockIdx.x) >= b.first[i + 1]) ++i;
  const GenericStepArgs& a = b.r[i];
  const int tile = int(blockIdx.x) - b.first[i];
  const int x = (tile % b.tiles_x[i]) * 32 + threadIdx.x;
  const int y = (tile / b.tiles_x[i]) * 8 + threadIdx.y;
  if (x < a.kx0 || x >= a.kx1 || y < a.ky0 || y >= a.ky1) return;
  for (int r = 0; r < 4; ++r) {
    float v;
    if (a.rows[r].ident) {
      v = load(a, r, x, y);
    } else {
      float acc = 0.0f;
      for (int t = a.rows[r].tb; t < a.rows[r].te; ++t) {
        const TapDesc tp = a.taps[t];
        const float s = load(a, tp.j, extend(x + tp.dm, a.w2, a.symmetric), extend(y + tp.dn, a.h2, a.symmetric));
        if (t == a.rows[r].tb)
          acc = tp.w == 1.0f ? s : __fmul_rn(tp.w, s);
        else if (a.fma)
          acc = __fmaf_rn(tp.w, s, acc);
        else
          acc = __fadd_rn(acc, tp.w == 1.0f ? s : __fmul_rn(tp.w, s));
      }
      v = a.rows[r].scale == 1.0f ? acc : __fmul_rn(acc, a.rows[r].scale);
    }
    if (a.out_il)
      a.out[0][(2ll * y + (r >> 1)) * a.out_pitch[0] + 2ll * x + (r & 1)] = v;
    else
      a.out[r][(long long)y * a.out_pitch[r] + x] = v;
  }
}

}  // namespace

cudaError_t launch_generic_step(const GenericStepArgs* a, int n, cudaStream_t st) {
  if (n < 1 || n > kMaxGenericRegions) return cudaErrorInvalidValue;
  GenericBatch b{};
  b.n = n;
  b.first[0] = 0;
  for (int i = 0; i < n; ++i) {
    b.r[i] = a[i];
    b.tiles_x[i] = (a[i].w2 + 31) / 32;
    b.first[i + 1] = b.first[i] + b.tiles_x[i] * ((a[i].h2 + 7) / 8);
  }
  if (b.first[n] == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(b.first[n]));
  cfg.blockDim = dim3(32, 8);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, generic_step_kernel, b);
}

}  // namespace gpu
}  // namespace dwt2d_b200
