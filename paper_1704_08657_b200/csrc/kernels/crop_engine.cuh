// Symmetric-extension border bands of one level, compiled from the plan's
// tap tables (reference image.hpp:14-26 extend_index,
// executor.hpp:159-167 — every sub-step reads its input through the
// extension rule).
//
// The fused level kernel computes a level with the periodic input rule; away
// from the image edges (outside the level's reach U/D/L/R) that is exactly
// the symmetric result, so it stores only the interior (LevelArgs keep
// window) and this kernel — on a side stream, concurrently — the four
// border bands. Each CTA takes a tile of one border crop (a band of the
// component grid along one image edge, core positions along the band plus
// margins of the level's cumulative reach) into shared memory and runs all
// sub-steps there. Between sub-steps the ghost cells beyond the tile's TRUE
// image edges are refilled by whole-sample reflection (extend_index: -k -> k,
// n-1+k -> n-1-k) of the sub-step's output, which is what the reference's
// per-step extension reads; the ghost cells on the other sides (tile edges
// inside the crop, the crop's inner edge) are never filled — their values
// only reach the discarded margins. Taps are compile-time constants in the
// table order with the fused kernel's rounding (eval_step), so the bands are
// bit-identical to the per-step symmetric executor (tested).
#pragma once

#include "level_engine.cuh"

namespace dwt2d_b200 {
namespace gpu {

template <class P>
struct CropGeom {
  using M = Meta<P>;
  static constexpr int S = M::S;
  // largest |dn| or |dm| of one sub-step: the ghost ring's width
  static constexpr int R = [] {
    int r = 1;
    for (int s = 0; s < S; ++s) {
      r = cmax(r, -M::nlo(s));
      r = cmax(r, M::nhi(s));
      r = cmax(r, -M::template reach<2>(s));
      r = cmax(r, M::template reach<3>(s));
    }
    return r;
  }();
  // buffer (0/1) holding component j before sub-step s (every arithmetic
  // row of j flips it: double buffering per component)
  static constexpr int cur(int s, int j) {
    int c = 0;
    for (int t = 0; t < s; ++t)
      if (!P::rows[t * 4 + j].ident) c ^= 1;
    return c;
  }
  static constexpr bool updates(int s, int j) { return !P::rows[s * 4 + j].ident; }
};

// shared-memory floats of one CTA for tile areas of at most `aw` x `ah` cells
template <class P>
constexpr int crop_smem_floats(int aw, int ah) {
  return 8 * (aw + 2 * CropGeom<P>::R) * (ah + 2 * CropGeom<P>::R);
}

struct CropTile {
  int ax0, aw, ay0, ah;   // tile area (crop coordinates)
  int cx0, cx1, cy0, cy1; // tile core (crop coordinates)
  int pw, plane;          // plane row stride and size (floats), ghost ring included
  // this thread's cell (-1: none) and ghost cell with its reflection source
  // (-1: none), as offsets into a plane
  int cell, ghost, gsrc;
  int cx, cy;             // the cell's area coordinates
};

// extend_index (image.hpp:14-26), whole-sample symmetric rule
__device__ __forceinline__ int extend_sym(int i, int n) {
  if (i >= 0 && i < n) return i;
  if (n == 1) return 0;
  const int period = 2 * n - 2;
  int r = i % period;
  if (r < 0) r += period;
  return r < n ? r : period - r;
}

template <class P, int s>
__device__ __forceinline__ void crop_step(const CropTile& t, float* planes) {
  using G = CropGeom<P>;
  if (t.cell >= 0) {
    sfor<0, 4>([&](auto R_) {
      constexpr int r = decltype(R_)::value;
      constexpr RowDesc row = P::rows[s * 4 + r];
      if constexpr (!row.ident) {
        float* dst = planes + (2 * r + (G::cur(s, r) ^ 1)) * t.plane;
        float acc = 0.0f;
        constexpr int tb = row.tb;  // scalar copies: nested lambdas use scalar constexpr locals only
        sfor<row.tb, row.te>([&](auto T_) {
          constexpr int ti = decltype(T_)::value;
          constexpr TapDesc tp = P::taps[ti];
          constexpr float w = tp.w;
          constexpr int j = tp.j, dn = tp.dn, dm = tp.dm;
          const float v = planes[(2 * j + G::cur(s, j)) * t.plane + t.cell + dn * t.pw + dm];
          if constexpr (ti != tb && P::kFma)
            acc = __fmaf_rn(w, v, acc);
          else if constexpr (ti != tb)
            acc = __fadd_rn(acc, w == 1.0f ? v : __fmul_rn(w, v));
          else if constexpr (w == 1.0f)
            acc = v;
          else
            acc = __fmul_rn(w, v);
        });
        constexpr float sc = row.scale;
        if constexpr (row.tb == row.te)
          dst[t.cell] = 0.0f;  // an all-zero matrix row
        else
          dst[t.cell] = sc == 1.0f ? acc : __fmul_rn(acc, sc);
      }
    });
  }
  __syncthreads();
  if (t.ghost >= 0) {
    sfor<0, 4>([&](auto R_) {
      constexpr int r = decltype(R_)::value;
      if constexpr (G::updates(s, r)) {
        float* pl = planes + (2 * r + G::cur(s + 1, r)) * t.plane;
        pl[t.ghost] = pl[t.gsrc];
      }
    });
  }
  __syncthreads();
}

// One CTA per tile; at most kCropThreads cells per tile area (the host sizes
// the core: crop_core) and ghost cells, one of each per thread.
template <class P>
__global__ void __launch_bounds__(kCropThreads) crop_kernel(const __grid_constant__ CropTileArgs a) {
  using G = CropGeom<P>;
  constexpr int R = G::R;
  extern __shared__ __align__(16) float crop_planes[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  int tile = blockIdx.x, rg = 0;
  while (rg + 1 < a.nreg && tile >= a.reg[rg].tiles) tile -= a.reg[rg].tiles, ++rg;
  const CropRegion& c = a.reg[rg];
  CropTile t{};
  t.ax0 = 0, t.ay0 = 0, t.cx0 = 0, t.cx1 = c.w, t.cy0 = 0, t.cy1 = c.h;
  int ax1 = c.w, ay1 = c.h;
  if (c.along_x) {
    t.cx0 = tile * a.core, t.cx1 = min(c.w, t.cx0 + a.core);
    t.ax0 = max(0, t.cx0 - a.mlo), ax1 = min(c.w, t.cx1 + a.mhi);
  } else {
    t.cy0 = tile * a.core, t.cy1 = min(c.h, t.cy0 + a.core);
    t.ay0 = max(0, t.cy0 - a.mlo), ay1 = min(c.h, t.cy1 + a.mhi);
  }
  t.aw = ax1 - t.ax0, t.ah = ay1 - t.ay0;
  t.pw = t.aw + 2 * R;
  t.plane = t.pw * (t.ah + 2 * R);
  // true image edges: the level grid is [0, a.w2) x [0, a.h2)
  const bool el = c.x0 + t.ax0 == 0, er = c.x0 + ax1 == a.w2;
  const bool et = c.y0 + t.ay0 == 0, eb = c.y0 + ay1 == a.h2;
  const int i = threadIdx.x;
  t.cell = -1, t.ghost = -1, t.gsrc = -1;
  if (i < t.aw * t.ah) {
    t.cy = i / t.aw, t.cx = i % t.aw;
    t.cell = (t.cy + R) * t.pw + t.cx + R;
  }
  // ghost cells: the ring of width R around the area (R rows above, R below,
  // R columns either side of the area's rows; at most kCropThreads cells,
  // crop_ring_cells), refilled beyond true image edges only (the others only
  // feed the discarded margins)
  const int gw = t.aw + 2 * R;
  if (i < 2 * R * gw + 2 * R * t.ah) {
    int x, y;
    if (i < 2 * R * gw) {
      const int k = i < R * gw ? i : i - R * gw;
      x = k % gw - R;
      y = i < R * gw ? k / gw - R : t.ah + k / gw;
    } else {
      const int k = i - 2 * R * gw, col = k % (2 * R);
      y = k / (2 * R);
      x = col < R ? col - R : t.aw + col - R;
    }
    if ((x >= 0 || el) && (x < t.aw || er) && (y >= 0 || et) && (y < t.ah || eb)) {
      t.ghost = (y + R) * t.pw + x + R;
      t.gsrc = (extend_sym(y, t.ah) + R) * t.pw + extend_sym(x, t.aw) + R;
    }
  }
  // sub-step 0 input over the area, then its ghosts
  if (t.cell >= 0) {
    const int gx = c.x0 + t.ax0 + t.cx, gy = c.y0 + t.ay0 + t.cy;
    sfor<0, 4>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      crop_planes[(2 * j + G::cur(0, j)) * t.plane + t.cell] =
          a.in_il ? a.in[0][(2ll * gy + (j >> 1)) * a.in_pitch[0] + 2ll * gx + (j & 1)]
                  : a.in[j][(long long)gy * a.in_pitch[j] + gx];
    });
  }
  __syncthreads();
  if (t.ghost >= 0) {
    sfor<0, 4>([&](auto J_) {
      float* pl = crop_planes + (2 * decltype(J_)::value + G::cur(0, decltype(J_)::value)) * t.plane;
      pl[t.ghost] = pl[t.gsrc];
    });
  }
  __syncthreads();
  sfor<0, G::S>([&](auto S_) { crop_step<P, decltype(S_)::value>(t, crop_planes); });
  // the kept part of the core
  if (t.cell >= 0) {
    const int x = t.ax0 + t.cx, y = t.ay0 + t.cy;  // crop coordinates
    if (x >= t.cx0 && x < t.cx1 && y >= t.cy0 && y < t.cy1 && x >= c.kx0 && x < c.kx1 && y >= c.ky0 && y < c.ky1) {
      const int gx = c.x0 + x, gy = c.y0 + y;
      sfor<0, 4>([&](auto J_) {
        constexpr int j = decltype(J_)::value;
        const float v = crop_planes[(2 * j + G::cur(G::S, j)) * t.plane + t.cell];
        if (a.out_il)
          a.out[0][(2ll * gy + (j >> 1)) * a.out_pitch[0] + 2ll * gx + (j & 1)] = v;
        else
          a.out[j][(long long)gy * a.out_pitch[j] + gx] = v;
      });
    }
  }
}

}  // namespace gpu
}  // namespace dwt2d_b200
