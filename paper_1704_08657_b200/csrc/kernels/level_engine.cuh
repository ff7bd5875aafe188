// Fused single-pass DWT level engine for sm_100a.
//
// One kernel launch = one decomposition level of any scheme: every sub-step
// of the lowered StepProgram (lowering.hpp) runs inside the same HBM pass.
// This replaces the reference's barrier-per-step executor
// (proj/include/dwt2d/executor.hpp:146-238: apply_rows over row bands with a
// std::barrier before each composed kernel) with:
//
//   * a warp-strip decomposition: each warp owns a vertical strip of 32
//     lanes x CW component columns and streams down a chunk of component
//     rows. Lanes 1..30 produce output; lanes 0 and 31 carry the horizontal
//     halo (the whole level reaches at most CW columns left/right, checked at
//     compile time), so warps are independent — no CTA barriers at all.
//   * a register sliding window in y: sub-step s keeps the last
//     (max_dn - min_dn + 1) rows of its input in registers; its output row
//     trails the newest input row by max_dn. A row enters at the top of the
//     pipeline, every sub-step fires once per row, and the last sub-step's
//     row is scaled and stored — the reference's double-buffer barriers
//     become register dependencies.
//   * warp shuffles for horizontal neighbours across lanes (intra-quad
//     dependencies), fmaf per tap in the reference's tap order.
//   * 128-bit loads of the interleaved image (polyphase split fused into the
//     load, reference image.hpp:73-94) or of four planar components, software
//     prefetch PF rows ahead, streaming stores of the detail bands.
//
// Periodic extension is applied to the INPUT rows/columns only: with
// periodic wrap every intermediate of the halo columns/rows is recomputed
// from wrapped inputs, which equals the reference's per-step wrap of
// intermediates (executor.hpp:159-167) exactly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <utility>

#include "level_types.hpp"

namespace dwt2d_b200 {
namespace gpu {

template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Compile-time geometry of a plan (P = generated traits, plans_gen.cuh).
template <class P>
struct Meta {
  static constexpr int S = P::kSteps;
  static constexpr int CW = P::kCW;

  template <int sel>  // 0 min dn, 1 max dn, 2 min dm, 3 max dm
  static constexpr int reach(int s) {
    int v = 0;
    for (int r = 0; r < 4; ++r) {
      const RowDesc row = P::rows[s * 4 + r];
      for (int t = row.tb; t < row.te; ++t) {
        const TapDesc tp = P::taps[t];
        if (sel == 0) v = cmin(v, tp.dn);
        if (sel == 1) v = cmax(v, tp.dn);
        if (sel == 2) v = cmin(v, tp.dm);
        if (sel == 3) v = cmax(v, tp.dm);
      }
    }
    return v;
  }
  static constexpr int nlo(int s) { return reach<0>(s); }
  static constexpr int nhi(int s) { return reach<1>(s); }
  static constexpr int depth(int s) { return s < S ? nhi(s) - nlo(s) + 1 : 1; }
  static constexpr int total(int sel) {
    int v = 0;
    for (int s = 0; s < S; ++s) {
      if (sel == 0) v -= reach<0>(s);
      if (sel == 1) v += reach<1>(s);
      if (sel == 2) v -= reach<2>(s);
      if (sel == 3) v += reach<3>(s);
    }
    return v;
  }
  static constexpr int U = total(0);   // rows above the output row that matter
  static constexpr int L = total(1);   // rows below (pipeline lag)
  static constexpr int HL = total(2);  // columns left
  static constexpr int HR = total(3);  // columns right
  static constexpr int dmax() {
    int v = 1;
    for (int s = 0; s < S; ++s) v = cmax(v, depth(s));
    return v;
  }
  static constexpr int D = dmax();
  static_assert(HL <= CW && HR <= CW, "horizontal reach exceeds one halo lane");
};

// value of component-column `col` of this lane's row, fetching from the
// neighbouring lane when col is outside [0, CW)
template <int col, int CW>
__device__ __forceinline__ float fetch(const float (&v)[CW]) {
  if constexpr (col >= 0 && col < CW) {
    return v[col];
  } else if constexpr (col >= CW) {
    return __shfl_down_sync(0xffffffffu, v[col - CW], 1);
  } else {
    return __shfl_up_sync(0xffffffffu, v[col + CW], 1);
  }
}

// One sub-step on one row: out[r][c] from the input window `in`
// (in[k] = the row k rows older than the newest input row).
template <class P, int s, int D, int CW>
__device__ __forceinline__ void eval_step(const float (&in)[D][4][CW], float (&out)[4][CW]) {
  constexpr int nhi = Meta<P>::nhi(s);
  sfor<0, 4>([&](auto R_) {
    constexpr int r = decltype(R_)::value;
    constexpr RowDesc row = P::rows[s * 4 + r];
    if constexpr (row.ident) {
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        out[r][c] = in[nhi][r][c];
      });
    } else if constexpr (row.tb == row.te) {  // an all-zero matrix row
      sfor<0, CW>([&](auto C_) { out[r][decltype(C_)::value] = 0.0f; });
    } else {
      // acc = 0 + w0*v0 + w1*v1 + ... in table order. Composed programs round
      // like the reference's `acc += f.w * src` (executor.hpp:183: product
      // rounded, then the sum); factored programs fuse each tap into one
      // fma. The first tap is a plain product (a copy when w0 == 1).
      float acc[CW];
      constexpr int tb = row.tb;
      constexpr float sc = row.scale;
      sfor<row.tb, row.te>([&](auto T_) {
        constexpr int ti = decltype(T_)::value;
        constexpr TapDesc t = P::taps[ti];
        // scalar copies: nested lambdas may only use scalar constexpr locals
        constexpr int k = nhi - t.dn, j = t.j, dm = t.dm;
        constexpr float w = t.w;
        constexpr bool first = ti == tb;
        sfor<0, CW>([&](auto C_) {
          constexpr int c = decltype(C_)::value;
          const float v = fetch<c + dm, CW>(in[k][j]);
          if constexpr (!first && P::kFma)
            acc[c] = __fmaf_rn(w, v, acc[c]);
          else if constexpr (!first)  // reference rounding: product, then sum
            acc[c] = __fadd_rn(acc[c], w == 1.0f ? v : __fmul_rn(w, v));
          else if constexpr (w == 1.0f)
            acc[c] = v;
          else
            acc[c] = __fmul_rn(w, v);
        });
      });
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        if constexpr (sc == 1.0f)
          out[r][c] = acc[c];
        else
          out[r][c] = __fmul_rn(acc[c], sc);
      });
    }
  });
}

__device__ __forceinline__ int wrap(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

// ------------------------------------------------------------ row I/O

template <int CW, bool IL>
__device__ __forceinline__ void load_row(const LevelArgs& a, int n, int xc, float (&d)[4][CW]) {
  const int rr = wrap(n, a.h2);
  if (a.vec) {
    const int x = wrap(xc, a.w2);  // lane's CW columns never straddle the wrap (w2 % CW == 0)
    if constexpr (IL) {
      sfor<0, 2>([&](auto PY_) {
        constexpr int py = decltype(PY_)::value;
        const float* p = a.in[0] + (2ll * rr + py) * a.in_pitch[0] + 2ll * x;
        sfor<0, CW / 2>([&](auto Q_) {
          constexpr int q = decltype(Q_)::value;
          const float4 v = __ldg(reinterpret_cast<const float4*>(p) + q);
          d[2 * py + 0][2 * q + 0] = v.x;
          d[2 * py + 1][2 * q + 0] = v.y;
          d[2 * py + 0][2 * q + 1] = v.z;
          d[2 * py + 1][2 * q + 1] = v.w;
        });
      });
    } else {
      sfor<0, 4>([&](auto J_) {
        constexpr int j = decltype(J_)::value;
        const float* p = a.in[j] + (long long)rr * a.in_pitch[j] + x;
        if constexpr (CW == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(p));
          d[j][0] = v.x, d[j][1] = v.y, d[j][2] = v.z, d[j][3] = v.w;
        } else if constexpr (CW == 2) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(p));
          d[j][0] = v.x, d[j][1] = v.y;
        } else {
          sfor<0, CW>([&](auto C_) { d[j][decltype(C_)::value] = __ldg(p + decltype(C_)::value); });
        }
      });
    }
  } else {
    sfor<0, CW>([&](auto C_) {
      constexpr int c = decltype(C_)::value;
      const int x = wrap(xc + c, a.w2);
      sfor<0, 4>([&](auto J_) {
        constexpr int j = decltype(J_)::value;
        if constexpr (IL)
          d[j][c] = __ldg(a.in[0] + (2ll * rr + (j >> 1)) * a.in_pitch[0] + 2ll * x + (j & 1));
        else
          d[j][c] = __ldg(a.in[j] + (long long)rr * a.in_pitch[j] + x);
      });
    });
  }
}

__device__ __forceinline__ void st_vec(float* p, float4 v, bool stream) {
  if (stream) __stcs(reinterpret_cast<float4*>(p), v);
  else *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void st_vec(float* p, float2 v, bool stream) {
  if (stream) __stcs(reinterpret_cast<float2*>(p), v);
  else *reinterpret_cast<float2*>(p) = v;
}

template <int CW, bool IL>
__device__ __forceinline__ void store_row(const LevelArgs& a, int y, int xc, const float (&v)[4][CW]) {
  if (a.vec) {
    if (xc + CW > a.w2) return;
    if constexpr (IL) {
      sfor<0, 2>([&](auto PY_) {
        constexpr int py = decltype(PY_)::value;
        float* p = a.out[0] + (2ll * y + py) * a.out_pitch[0] + 2ll * xc;
        sfor<0, CW / 2>([&](auto Q_) {
          constexpr int q = decltype(Q_)::value;
          st_vec(p + 4 * q,
                 make_float4(v[2 * py][2 * q], v[2 * py + 1][2 * q], v[2 * py][2 * q + 1],
                             v[2 * py + 1][2 * q + 1]),
                 false);
        });
      });
    } else {
      sfor<0, 4>([&](auto J_) {
        constexpr int j = decltype(J_)::value;
        float* p = a.out[j] + (long long)y * a.out_pitch[j] + xc;
        if constexpr (CW == 4)
          st_vec(p, make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), j != 0);
        else if constexpr (CW == 2)
          st_vec(p, make_float2(v[j][0], v[j][1]), j != 0);
        else
          sfor<0, CW>([&](auto C_) { p[decltype(C_)::value] = v[j][decltype(C_)::value]; });
      });
    }
  } else {
    sfor<0, CW>([&](auto C_) {
      constexpr int c = decltype(C_)::value;
      const int x = xc + c;
      if (x < a.w2) {
        sfor<0, 4>([&](auto J_) {
          constexpr int j = decltype(J_)::value;
          if constexpr (IL)
            a.out[0][(2ll * y + (j >> 1)) * a.out_pitch[0] + 2ll * x + (j & 1)] = v[j][c];
          else
            a.out[j][(long long)y * a.out_pitch[j] + x] = v[j][c];
        });
      }
    });
  }
}

// ------------------------------------------------------------- kernel

template <class P, int PF, bool IN_IL, bool OUT_IL>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
level_kernel(const LevelArgs a) {
  using M = Meta<P>;
  constexpr int S = M::S, CW = M::CW, D = M::D;
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;  // warp-uniform
  const int strip = wid % a.nstrips, chunk = wid / a.nstrips;
  const int xc = (strip * kOutLanes - 1 + lane) * CW;  // first component column of this lane
  const int y0 = chunk * a.chunk_rows;
  const int y1 = min(a.h2, y0 + a.chunk_rows);
  const int n0 = y0 - M::U;
  const int iters = (y1 - y0) + M::U + M::L;
  const bool out_lane = lane >= 1 && lane <= kOutLanes;

  float ring[S + 1][D][4][CW];
  sfor<0, S + 1>([&](auto B_) {
    sfor<0, D>([&](auto K_) {
      sfor<0, 4>([&](auto J_) {
        sfor<0, CW>([&](auto C_) {
          ring[decltype(B_)::value][decltype(K_)::value][decltype(J_)::value][decltype(C_)::value] = 0.0f;
        });
      });
    });
  });
  float pf[PF][4][CW];
  sfor<0, PF>([&](auto U_) {
    constexpr int u = decltype(U_)::value;
    if (u < iters) load_row<CW, IN_IL>(a, n0 + u, xc, pf[u]);
  });

  for (int it = 0; it < iters; it += PF) {
    sfor<0, PF>([&](auto U_) {
      constexpr int u = decltype(U_)::value;
      const int i = it + u;
      if (i < iters) {  // warp-uniform
        // age every window by one row
        sfor<0, S + 1>([&](auto B_) {
          constexpr int b = decltype(B_)::value;
          constexpr int dep = M::depth(b);
          sfor<1, dep>([&](auto K_) {
            constexpr int k = dep - decltype(K_)::value;  // dep-1 .. 1
            sfor<0, 4>([&](auto J_) {
              sfor<0, CW>([&](auto C_) {
                ring[b][k][decltype(J_)::value][decltype(C_)::value] =
                    ring[b][k - 1][decltype(J_)::value][decltype(C_)::value];
              });
            });
          });
        });
        sfor<0, 4>([&](auto J_) {
          sfor<0, CW>([&](auto C_) {
            ring[0][0][decltype(J_)::value][decltype(C_)::value] =
                pf[u][decltype(J_)::value][decltype(C_)::value];
          });
        });
        if (i + PF < iters) load_row<CW, IN_IL>(a, n0 + i + PF, xc, pf[u]);
        sfor<0, S>([&](auto S_) {
          constexpr int s = decltype(S_)::value;
          eval_step<P, s, D, CW>(ring[s], ring[s + 1][0]);
        });
        const int y = n0 + i - M::L;
        if (y >= y0 && out_lane) store_row<CW, OUT_IL>(a, y, xc, ring[S][0]);
      }
    });
  }
}

}  // namespace gpu
}  // namespace dwt2d_b200
