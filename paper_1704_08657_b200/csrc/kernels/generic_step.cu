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

// float64 (compile<double>): one sub-step over one grid; tiles of 32 x 8
__global__ void __launch_bounds__(256) generic_step64_kernel(const __grid_constant__ GenericStepArgs64 a) {
  const int tiles_x = (a.w2 + 31) / 32;
  const int x = (int(blockIdx.x) % tiles_x) * 32 + threadIdx.x;
  const int y = (int(blockIdx.x) / tiles_x) * 8 + threadIdx.y;
  if (x < a.kx0 || x >= a.kx1 || y < a.ky0 || y >= a.ky1) return;
  auto load = [&](int j, int xx, int yy) {
    if (a.in_il) return a.in[0][(2ll * yy + (j >> 1)) * a.in_pitch[0] + 2ll * xx + (j & 1)];
    return a.in[j][(long long)yy * a.in_pitch[j] + xx];
  };
  for (int r = 0; r < 4; ++r) {
    double v;
    if (a.rows[r].ident) {
      v = load(r, x, y);
    } else {
      double acc = 0.0;
      for (int t = a.rows[r].tb; t < a.rows[r].te; ++t) {
        const TapDesc64 tp = a.taps[t];
        const double s = load(tp.j, extend(x + tp.dm, a.w2, a.symmetric), extend(y + tp.dn, a.h2, a.symmetric));
        if (t == a.rows[r].tb)
          acc = tp.w == 1.0 ? s : __dmul_rn(tp.w, s);
        else if (a.fma)
          acc = __fma_rn(tp.w, s, acc);
        else
          acc = __dadd_rn(acc, tp.w == 1.0 ? s : __dmul_rn(tp.w, s));
      }
      v = a.rows[r].scale == 1.0 ? acc : __dmul_rn(acc, a.rows[r].scale);
    }
    if (a.out_il)
      a.out[0][(2ll * y + (r >> 1)) * a.out_pitch[0] + 2ll * x + (r & 1)] = v;
    else
      a.out[r][(long long)y * a.out_pitch[r] + x] = v;
  }
}

}  // namespace

cudaError_t launch_generic_step64(const GenericStepArgs64& a, cudaStream_t st) {
  const long long tiles = (long long)((a.w2 + 31) / 32) * ((a.h2 + 7) / 8);
  if (tiles <= 0) return cudaSuccess;
  generic_step64_kernel<<<unsigned(tiles), dim3(32, 8), 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_generic_step(const GenericStepArgs* a, int n, bool pdl, cudaStream_t st) {
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
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, generic_step_kernel, b);
}

namespace {

__global__ void __launch_bounds__(256) crop_tile_kernel(const __grid_constant__ CropTileArgs a) {
  extern __shared__ float sm[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  int t = blockIdx.x, r = 0;
  while (r + 1 < a.nreg && t >= a.reg[r].tiles) t -= a.reg[r].tiles, ++r;
  const CropRegion& c = a.reg[r];
  // compute area of this tile (crop coordinates): [ax0, ax1) x [ay0, ay1)
  int ax0 = 0, ax1 = c.w, ay0 = 0, ay1 = c.h, cx0 = 0, cx1 = c.w, cy0 = 0, cy1 = c.h;
  if (c.along_x) {
    cx0 = t * a.core, cx1 = min(c.w, cx0 + a.core);
    ax0 = max(0, cx0 - a.mlo), ax1 = min(c.w, cx1 + a.mhi);
  } else {
    cy0 = t * a.core, cy1 = min(c.h, cy0 + a.core);
    ay0 = max(0, cy0 - a.mlo), ay1 = min(c.h, cy1 + a.mhi);
  }
  const int aw = ax1 - ax0, ah = ay1 - ay0, area = aw * ah;
  float* buf[2] = {sm, sm + 4 * area};
  const int nthr = blockDim.x;
  // sub-step 0 input: the crop's input over the area
  for (int q = threadIdx.x; q < area; q += nthr) {
    const int xa = q % aw, ya = q / aw;
    const int x = c.x0 + ax0 + xa, y = c.y0 + ay0 + ya;
    for (int j = 0; j < 4; ++j)
      buf[0][j * area + q] = a.in_il ? a.in[0][(2ll * y + (j >> 1)) * a.in_pitch[0] + 2ll * x + (j & 1)]
                                     : a.in[j][(long long)y * a.in_pitch[j] + x];
  }
  __syncthreads();
  for (int s = 0; s < a.nsteps; ++s) {
    const float* src = buf[s & 1];
    float* dst = buf[(s + 1) & 1];
    const bool last = s == a.nsteps - 1;
    for (int q = threadIdx.x; q < area; q += nthr) {
      const int xa = q % aw, ya = q / aw;
      const int x = ax0 + xa, y = ay0 + ya;  // crop coordinates
      if (last && (x < cx0 || x >= cx1 || y < cy0 || y >= cy1 || x < c.kx0 || x >= c.kx1 || y < c.ky0 ||
                   y >= c.ky1))
        continue;
      for (int rr = 0; rr < 4; ++rr) {
        const RowDesc row = a.rows[s * 4 + rr];
        float v;
        if (row.ident) {
          v = src[rr * area + q];
        } else {
          float acc = 0.0f;
          for (int k = row.tb; k < row.te; ++k) {
            const TapDesc tp = a.taps[k];
            // the crop's extension rule, then the area (values beyond a tile
            // edge inside the crop only reach the discarded margins)
            int xe = extend(x + tp.dm, c.w, a.symmetric) - ax0;
            int ye = extend(y + tp.dn, c.h, a.symmetric) - ay0;
            xe = min(max(xe, 0), aw - 1);
            ye = min(max(ye, 0), ah - 1);
            const float sv = src[tp.j * area + ye * aw + xe];
            if (k == row.tb)
              acc = tp.w == 1.0f ? sv : __fmul_rn(tp.w, sv);
            else if (a.fma)
              acc = __fmaf_rn(tp.w, sv, acc);
            else
              acc = __fadd_rn(acc, tp.w == 1.0f ? sv : __fmul_rn(tp.w, sv));
          }
          v = row.scale == 1.0f ? acc : __fmul_rn(acc, row.scale);
        }
        if (!last) {
          dst[rr * area + q] = v;
        } else {
          const int gx = c.x0 + x, gy = c.y0 + y;
          if (a.out_il)
            a.out[0][(2ll * gy + (rr >> 1)) * a.out_pitch[0] + 2ll * gx + (rr & 1)] = v;
          else
            a.out[rr][(long long)gy * a.out_pitch[rr] + gx] = v;
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_crop_tiles(const CropTileArgs& a, int smem_floats, bool pdl, cudaStream_t st) {
  int tiles = 0;
  for (int i = 0; i < a.nreg; ++i) tiles += a.reg[i].tiles;
  if (tiles == 0) return cudaSuccess;
  const int bytes = smem_floats * 4;
  if (bytes > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(crop_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(tiles));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = size_t(bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, crop_tile_kernel, a);
}

}  // namespace gpu
}  // namespace dwt2d_b200
