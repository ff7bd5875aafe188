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
// lane that holds it when col is outside [0, CW) (one shuffle, over as many
// lanes as the column is away)
template <int col, int CW>
__device__ __forceinline__ float fetch(const float (&v)[CW]) {
  if constexpr (col >= 0 && col < CW) {
    return v[col];
  } else if constexpr (col >= CW) {
    constexpr int k = col / CW;
    return __shfl_down_sync(0xffffffffu, v[col - k * CW], k);
  } else {
    constexpr int k = (-col + CW - 1) / CW;
    return __shfl_up_sync(0xffffffffu, v[col + k * CW], k);
  }
}

// Compile-time schedule of the register windows.
//
// Window b holds the last rows of sub-step b's input (b = 0: loaded rows,
// b = S: final output). Window 0 doubles as the load pipeline: it has
// PF + depth(0) - 1 slots so the load for row i + PF can be issued into the
// slot that row i - depth(0) + 1 just vacated. Windows are circular buffers
// indexed by (row mod slots); the main loop is unrolled by UNR = lcm of all
// slot counts so every slot index is a compile-time constant and rows never
// move between registers. If that lcm is large (wide convolution windows),
// windows 1..S shift instead (register moves, UNR = slots of window 0).
// Programs with the kShift trait (the very wide composed convolutions) shift
// every window, the load ring too, and run the loop body once per row: their
// 8-fold unrolled body (~80 KB of SASS) does not stay in the instruction
// cache, and one register move per window value and row costs less.
template <class P>
constexpr bool shift_rows() {
  if constexpr (requires { P::kShift; }) return P::kShift;
  else return false;
}

template <class P, int PF>
struct Sched {
  using M = Meta<P>;
  static constexpr int S = M::S;
  static constexpr int slots(int b) { return b == 0 ? PF + M::depth(0) - 1 : (b < S ? M::depth(b) : 1); }
  static constexpr int gcd(int a, int b) { return b == 0 ? a : gcd(b, a % b); }
  static constexpr int lcm_all() {
    int l = 1;
    for (int b = 0; b <= S; ++b) l = l / gcd(l, slots(b)) * slots(b);
    return l;
  }
  static constexpr bool kShift0 = shift_rows<P>();
  static constexpr int shift_unroll() {
    if constexpr (requires { P::kShiftUnroll; }) return P::kShiftUnroll;
    else return 1;
  }
  static constexpr bool kCirc = !kShift0 && lcm_all() <= 8;
  static constexpr int UNR = kShift0 ? shift_unroll() : kCirc ? lcm_all() : slots(0);
  static constexpr int DMAX() {
    int v = 1;
    for (int b = 0; b <= S; ++b) v = cmax(v, slots(b));
    return v;
  }
  static constexpr int D = DMAX();
  // register slot of the row `age` rows older than the newest row of window
  // b, at unrolled iteration u (circular mode); age itself in shift mode.
  // Window 0 is the load ring: circular unless kShift0, where row i (age 0)
  // sits in slot PF - 1 and the rows in flight (ages -1 .. -PF + 1) below it.
  static constexpr int slot(int b, int u, int age) {
    const int n = slots(b);
    if (b == 0 && kShift0) return age + PF - 1;
    return (kCirc || b == 0) ? ((u - age) % n + n) % n : age;
  }
};

// Packed FP32 (sm_100a FFMA2/FADD2: two independent IEEE operations per
// instruction, each half rounded exactly like the scalar op): a tap's weight
// is the same for every component column of a lane, so columns go through
// the accumulation in pairs. VF (factored programs): 0 scalar, 1 pairs
// (c, c + 1), 2 pairs (c, c + CW/2). Composed programs (the reference's
// product-then-sum rounding, executor.hpp:183) are packed with pairs
// (c, c + 1) when kComposedPacked is set: ptxas contracts mul.rn.f32x2 +
// add.rn.f32x2 into FFMA2 even with --fmad=false (checked with nvcc 12.9),
// so every packed product is written fma(w, v, nz) with nz = -0.0f read from
// the launch arguments (opaque to ptxas, and round(w*v + -0) == round(w*v)
// for every w*v including signed zeros) and cannot be fused into the sum.
#ifndef DWT2D_PACKED_FMA
#define DWT2D_PACKED_FMA 1
#endif
constexpr int kPackedFma = DWT2D_PACKED_FMA;
#ifndef DWT2D_LEVEL_PACKED_FMA
#define DWT2D_LEVEL_PACKED_FMA 0
#endif
constexpr int kLevelPackedFma = DWT2D_LEVEL_PACKED_FMA;
#ifndef DWT2D_COMPOSED_PACKED
#define DWT2D_COMPOSED_PACKED 1
#endif
constexpr bool kComposedPacked = DWT2D_COMPOSED_PACKED != 0;

// packed form of a composed program: the plan's kPack trait where it has one
template <class P>
constexpr bool composed_packed() {
  if constexpr (requires { P::kPack; }) return P::kPack;
  else return kComposedPacked;
}

template <int VF, int CW>
__host__ __device__ constexpr int pair_col(int p, int half) {
  return VF == 1 ? 2 * p + half : p + half * (CW / 2);
}

// Evaluation order of one sub-step. Every output component's sum keeps its
// table order (so the rounding is the reference's); when each arithmetic
// row's taps are sorted by source (component j, row dn) — the composed
// programs' are (executor.hpp:79-90) — the rows advance together, one
// (j, dn) block at a time. A block first fetches the source row's columns
// its taps read (the neighbour lanes' columns by one shuffle each: shuffles
// are not merged by the compiler) and every tap of every output then reads
// those registers; the next block's replace them, so a 256-tap composed
// convolution keeps one source row's halo live instead of all of them.
// Otherwise (factored programs): one block, rows in table order, every
// source row's halo fetched once for the whole sub-step.
template <class P, int s, int CW>
struct StepOrder {
  static constexpr int kMaxKeys = 64;
  static constexpr int kReach = 4;                  // largest column offset of a tap (gen_plans.cpp)
  static constexpr int kCols = CW + 2 * kReach;      // columns -kReach .. CW + kReach - 1
  struct Data {
    int nkeys = 0, nblocks = 0;
    int kj[kMaxKeys] = {}, kdn[kMaxKeys] = {};
    unsigned long long cols[kMaxKeys] = {};  // bit c + CW: column c of the key's row is read
    int kb[kMaxKeys] = {}, ke[kMaxKeys] = {};  // keys of each block
    int b[4][kMaxKeys] = {}, e[4][kMaxKeys] = {};  // taps of each row in each block
  };
  static constexpr int key(const TapDesc& t) { return t.j * 256 + t.dn + 128; }
  static constexpr Data build() {
    Data d{};
    bool sorted = true;
    int keys[kMaxKeys] = {};
    int n = 0;
    for (int r = 0; r < 4; ++r) {
      const RowDesc row = P::rows[s * 4 + r];
      if (row.ident) continue;
      for (int t = row.tb; t < row.te; ++t) {
        if (t > row.tb && key(P::taps[t]) < key(P::taps[t - 1])) sorted = false;
        bool seen = false;
        for (int q = 0; q < n; ++q) seen = seen || keys[q] == key(P::taps[t]);
        if (!seen) keys[n++] = key(P::taps[t]);
      }
    }
    for (int i = 0; i < n; ++i)  // sort the keys
      for (int k = i + 1; k < n; ++k)
        if (keys[k] < keys[i]) {
          const int x = keys[i];
          keys[i] = keys[k], keys[k] = x;
        }
    d.nkeys = n;
    for (int q = 0; q < n; ++q) {
      d.kj[q] = keys[q] / 256, d.kdn[q] = keys[q] % 256 - 128;
      for (int r = 0; r < 4; ++r) {
        const RowDesc row = P::rows[s * 4 + r];
        if (row.ident) continue;
        for (int t = row.tb; t < row.te; ++t)
          for (int c = 0; c < CW; ++c)
            if (key(P::taps[t]) == keys[q]) d.cols[q] |= 1ull << (c + P::taps[t].dm + kReach);
      }
    }
    if (!sorted || n == 0) {  // one block: all keys, rows in table order
      d.nblocks = 1;
      d.kb[0] = 0, d.ke[0] = n;
      for (int r = 0; r < 4; ++r) {
        const RowDesc row = P::rows[s * 4 + r];
        d.b[r][0] = row.tb, d.e[r][0] = row.ident ? row.tb : row.te;
      }
      return d;
    }
    d.nblocks = n;
    for (int q = 0; q < n; ++q) {
      d.kb[q] = q, d.ke[q] = q + 1;
      for (int r = 0; r < 4; ++r) {
        const RowDesc row = P::rows[s * 4 + r];
        int b = row.tb, e = row.tb;
        bool any = false;
        if (!row.ident)
          for (int t = row.tb; t < row.te; ++t)
            if (key(P::taps[t]) == keys[q]) {
              if (!any) b = t;
              any = true;
              e = t + 1;
            }
        d.b[r][q] = b, d.e[r][q] = e;
      }
    }
    return d;
  }
  static constexpr Data d = build();
  // whether a packed tap reads the pair starting at column m (pairing pv)
  static constexpr bool pair_needed(int q, int m, int pv) {
    for (int r = 0; r < 4; ++r) {
      const RowDesc row = P::rows[s * 4 + r];
      if (row.ident) continue;
      for (int t = row.tb; t < row.te; ++t)
        if (key(P::taps[t]) == key_of(q))
          for (int c = 0; c < CW / 2; ++c)
            if ((pv == 1 ? 2 * c : c) + P::taps[t].dm == m) return true;
    }
    return false;
  }
  static constexpr int key_of(int q) { return d.kj[q] * 256 + d.kdn[q] + 128; }
  static constexpr int index(int j, int dn) {
    for (int q = 0; q < d.nkeys; ++q)
      if (d.kj[q] == j && d.kdn[q] == dn) return q;
    return -1;
  }
};

// UPW: rows stream bottom-up (the newest window row is the topmost one), so
// a tap at row offset dn is (dn - min_dn) rows older than the newest instead
// of (max_dn - dn). Same taps, same order: identical results.
template <class P, int PF, int s, int u, int D, int CW, bool UPW, int VF = kPackedFma>
__device__ __forceinline__ void eval_step(float (&ring)[Meta<P>::S + 1][D][4][CW], const float nz) {
  using SC = Sched<P, PF>;
  using O = StepOrder<P, s, CW>;
  constexpr int nhi = UPW ? -Meta<P>::nlo(s) : Meta<P>::nhi(s);  // age of the dn = 0 row
  constexpr int dsign = UPW ? -1 : 1;
  constexpr int dst = SC::slot(s + 1, u, 0);
  constexpr bool pack = CW % 2 == 0 && (P::kFma ? VF != 0 : composed_packed<P>());
  constexpr int PV = P::kFma ? VF : 2;  // pairing of the packed form
  constexpr int NA = pack ? CW / 2 : CW;
  // acc = 0 + w0*v0 + w1*v1 + ... in table order. Composed programs round
  // like the reference's `acc += f.w * src` (executor.hpp:183: product
  // rounded, then the sum); factored programs fuse each tap into one fma.
  // The first tap is a plain product (a copy when w0 == 1).
  using Acc = std::conditional_t<pack, float2, float>;
  Acc acc[4][NA];
  const float2 nz2 = make_float2(nz, nz);
  sfor<0, O::d.nblocks>([&](auto Q_) {
    constexpr int q = decltype(Q_)::value;
    // the block's source rows, halo columns included: ext[key][c + RX]; for
    // the packed form also every operand pair the taps read, built once per
    // block (ext2[key][m + RX] = columns m and m + pair_col(0, 1)): pairs
    // assembled per tap cost a register move each
    constexpr int NK = O::d.nkeys > 0 ? O::d.nkeys : 1;
    constexpr int POFF = pair_col<PV, CW>(0, 1);
    constexpr int RX = O::kReach;
    float ext[NK][O::kCols];
    float2 ext2[pack ? NK : 1][O::kCols];
    sfor<O::d.kb[q], O::d.ke[q]>([&](auto K_) {
      constexpr int key = decltype(K_)::value;
      constexpr int k = SC::slot(s, u, nhi - dsign * O::d.kdn[key]), j = O::d.kj[key];
      sfor<0, O::kCols>([&](auto C_) {
        constexpr int c = decltype(C_)::value - RX;
        if constexpr ((O::d.cols[key] >> (c + RX)) & 1ull) ext[key][c + RX] = fetch<c, CW>(ring[s][k][j]);
      });
      if constexpr (pack) {
        sfor<0, O::kCols>([&](auto C_) {
          constexpr int m = decltype(C_)::value - RX;
          if constexpr (O::pair_needed(key, m, PV)) ext2[key][m + RX] = make_float2(ext[key][m + RX], ext[key][m + POFF + RX]);
        });
      }
    });
    sfor<0, 4>([&](auto R_) {
      constexpr int r = decltype(R_)::value;
      constexpr int tb = P::rows[s * 4 + r].tb;
      sfor<O::d.b[r][q], O::d.e[r][q]>([&](auto T_) {
        constexpr int ti = decltype(T_)::value;
        constexpr TapDesc t = P::taps[ti];
        // scalar copies: nested lambdas may only use scalar constexpr locals
        constexpr int key = O::index(t.j, t.dn), dm = t.dm;
        constexpr float w = t.w;
        constexpr bool first = ti == tb;
        if constexpr (pack) {
          sfor<0, NA>([&](auto C_) {
            constexpr int c = decltype(C_)::value;
            constexpr int ca = pair_col<PV, CW>(c, 0), cb = pair_col<PV, CW>(c, 1);
            static_assert(cb - ca == POFF, "pair layout");
            const float2 v = ext2[key][ca + dm + RX];
            const float2 wv = w == 1.0f ? v : __ffma2_rn(make_float2(w, w), v, nz2);
            if constexpr (first)
              acc[r][c] = wv;
            else if constexpr (P::kFma)
              acc[r][c] = __ffma2_rn(make_float2(w, w), v, acc[r][c]);
            else
              acc[r][c] = __fadd2_rn(acc[r][c], wv);
          });
        } else {
          sfor<0, CW>([&](auto C_) {
            constexpr int c = decltype(C_)::value;
            const float v = ext[key][c + dm + RX];
            if constexpr (!first && P::kFma)
              acc[r][c] = __fmaf_rn(w, v, acc[r][c]);
            else if constexpr (!first)  // reference rounding: product, then sum
              acc[r][c] = __fadd_rn(acc[r][c], w == 1.0f ? v : __fmul_rn(w, v));
            else if constexpr (w == 1.0f)
              acc[r][c] = v;
            else
              acc[r][c] = __fmul_rn(w, v);
          });
        }
      });
    });
  });
  sfor<0, 4>([&](auto R_) {
    constexpr int r = decltype(R_)::value;
    constexpr RowDesc row = P::rows[s * 4 + r];
    constexpr float sc = row.scale;
    if constexpr (row.ident) {
      constexpr int src = SC::slot(s, u, nhi);
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        ring[s + 1][dst][r][c] = ring[s][src][r][c];
      });
    } else if constexpr (row.tb == row.te) {  // an all-zero matrix row
      sfor<0, CW>([&](auto C_) { ring[s + 1][dst][r][decltype(C_)::value] = 0.0f; });
    } else if constexpr (pack) {
      sfor<0, NA>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        constexpr int ca = pair_col<PV, CW>(c, 0), cb = pair_col<PV, CW>(c, 1);
        const float2 o = sc == 1.0f ? acc[r][c] : __ffma2_rn(acc[r][c], make_float2(sc, sc), nz2);
        ring[s + 1][dst][r][ca] = o.x;
        ring[s + 1][dst][r][cb] = o.y;
      });
    } else {
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        if constexpr (sc == 1.0f)
          ring[s + 1][dst][r][c] = acc[r][c];
        else
          ring[s + 1][dst][r][c] = __fmul_rn(acc[r][c], sc);
      });
    }
  });
}

__device__ __forceinline__ int wrap(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

// ------------------------------------------------------------ row I/O

// Streams input rows top to bottom. Row n (relative to the chunk's level)
// comes from the main input with periodic wrap, or — for a row strip of a
// sharded image — from the halo buffers above/below the strip. Column offsets
// are fixed per lane; the row pointer advances by one pitch per row and is
// recomputed only when the row crosses a segment boundary (no division in
// the steady state).
template <bool COH>
__device__ __forceinline__ float4 ld4(const float* p) {
  if constexpr (COH) return __ldcg(reinterpret_cast<const float4*>(p));
  else return __ldg(reinterpret_cast<const float4*>(p));
}
template <bool COH>
__device__ __forceinline__ float2 ld2(const float* p) {
  if constexpr (COH) return __ldcg(reinterpret_cast<const float2*>(p));
  else return __ldg(reinterpret_cast<const float2*>(p));
}
template <bool COH>
__device__ __forceinline__ float ld1(const float* p) {
  if constexpr (COH) return __ldcg(p);
  else return __ldg(p);
}

// COH: loads bypass the non-coherent path (needed when the input was written
// earlier in the same launch, i.e. by a previous level of the same kernel).
template <int CW, bool IL, bool VEC, bool COH = false, bool UPW = false>
struct RowReader {
  static constexpr int NP = IL ? 1 : 4;  // row pointers kept
  const float* rowp[NP];  // start of the current row (+ lane column for VEC)
  long long pitch[NP];    // current segment's row step (IL: two image rows)
  long long half;         // IL: offset of the odd image row within a component row
  int n, next_switch;
  int xs[CW];             // wrapped columns (scalar path)
  int xv;                 // wrapped first column (vector path)

  __device__ __forceinline__ void seek(const LevelArgs& a, int row) {
    n = row;
    const float* const* src = a.in;
    const long long* sp = a.in_pitch;
    int r = row;
    // next_switch: the first row (in streaming order) outside this segment
    if (a.halo && row < 0) {
      src = a.halo_top, sp = a.halo_top_pitch, r = row + a.up;
      next_switch = UPW ? int(0x80000000) : 0;
    } else if (a.halo && row >= a.h2) {
      src = a.halo_bot, sp = a.halo_bot_pitch, r = row - a.h2;
      next_switch = UPW ? a.h2 - 1 : 0x7fffffff;
    } else {
      r = a.halo ? row : wrap(row, a.h2);
      next_switch = UPW ? (a.halo ? -1 : row - r - 1) : (a.halo ? a.h2 : row - r + a.h2);
    }
    sfor<0, NP>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      const long long step = IL ? 2ll * sp[0] : sp[j];
      pitch[j] = step;
      rowp[j] = src[j] + (long long)r * step + (VEC ? (IL ? 2ll * xv : (long long)xv) : 0ll);
    });
    if constexpr (IL) half = sp[0];
  }

  __device__ __forceinline__ void init(const LevelArgs& a, int xc, int first_row, int /*rows*/) {
    init(a, xc, first_row);
  }
  __device__ __forceinline__ void init(const LevelArgs& a, int xc, int first_row) {
    xv = wrap(xc, a.w2);
    sfor<0, CW>([&](auto C_) { xs[decltype(C_)::value] = wrap(xc + decltype(C_)::value, a.w2); });
    seek(a, first_row);
  }

  __device__ __forceinline__ void advance(const LevelArgs& a) {
    n += UPW ? -1 : 1;
    if (n == next_switch) {
      seek(a, n);
    } else {
      sfor<0, NP>([&](auto J_) {
        if constexpr (UPW) rowp[decltype(J_)::value] -= pitch[decltype(J_)::value];
        else rowp[decltype(J_)::value] += pitch[decltype(J_)::value];
      });
    }
  }

  __device__ __forceinline__ void load(const LevelArgs& a, float (&d)[4][CW]) {
    if constexpr (VEC) {
      if constexpr (IL) {
        sfor<0, 2>([&](auto PY_) {
          constexpr int py = decltype(PY_)::value;
          const float* p = rowp[0] + (py ? half : 0ll);
          sfor<0, CW / 2>([&](auto Q_) {
            constexpr int q = decltype(Q_)::value;
            const float4 v = ld4<COH>(p + 4 * q);
            d[2 * py + 0][2 * q + 0] = v.x;
            d[2 * py + 1][2 * q + 0] = v.y;
            d[2 * py + 0][2 * q + 1] = v.z;
            d[2 * py + 1][2 * q + 1] = v.w;
          });
        });
      } else {
        sfor<0, 4>([&](auto J_) {
          constexpr int j = decltype(J_)::value;
          const float* p = rowp[j];
          if constexpr (CW == 4) {
            const float4 v = ld4<COH>(p);
            d[j][0] = v.x, d[j][1] = v.y, d[j][2] = v.z, d[j][3] = v.w;
          } else if constexpr (CW == 2) {
            const float2 v = ld2<COH>(p);
            d[j][0] = v.x, d[j][1] = v.y;
          } else {
            sfor<0, CW>([&](auto C_) { d[j][decltype(C_)::value] = ld1<COH>(p + decltype(C_)::value); });
          }
        });
      }
    } else {
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        sfor<0, 4>([&](auto J_) {
          constexpr int j = decltype(J_)::value;
          if constexpr (IL)
            d[j][c] = ld1<COH>(rowp[0] + ((j >> 1) ? half : 0ll) + 2 * xs[c] + (j & 1));
          else
            d[j][c] = ld1<COH>(rowp[j] + xs[c]);
        });
      });
    }
    advance(a);
  }
};

// ------------------------------------------------ TMA-staged input rows
//
// Interleaved vector input (forward levels) staged in shared memory by the
// TMA unit: a warp's share of one component row is two contiguous image-row
// segments of 32 lanes x 8*CW bytes, each fetched by ONE cp.async.bulk (lane
// 0 and lane 1, one image row each; more copies only where the strip wraps
// past the right image edge) that signals an mbarrier per stage. kStages - 1
// component rows are in flight per warp without costing registers (the
// register reader keeps PF rows in registers), and the loads are issued by 2
// lanes instead of 32. Each lane then reads its own 2 x CW/2 float4 from the
// stage. A stage is refilled one iteration after it was read, when its values
// have been consumed. Measured on B200, level 1 of 16384^2: 6.36 TB/s vs
// 6.06 TB/s for register prefetch (scripts/tune_tma.cu).
constexpr int kStages = 8;

__device__ __forceinline__ unsigned smem_addr(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

template <int CW>
constexpr int staged_bytes() {  // dynamic shared memory of one CTA
  return ((kWarpsPerCta * kStages * 8 + 127) / 128) * 128 + kWarpsPerCta * kStages * 2 * 32 * 8 * CW;
}

template <int CW, bool UPW>
struct TmaRowReader {
  static constexpr int kRowF4 = 32 * CW / 2;  // float4 per image row of the warp
  static constexpr int kTotal = 32 * 8 * CW;   // bytes per image row of the warp
  RowReader<CW, true, false, false, UPW> g;    // row walk (periodic wrap / halo segments, no division)
  float4* stage0;
  unsigned long long* bar;
  int xw0, first;  // first image column of lane 0 (wrapped), bytes up to the right image edge
  int issued, fetched, rows;
  unsigned phase_bits;

  __device__ __forceinline__ void issue_row(const LevelArgs& a) {
    const int lane = threadIdx.x & 31;
    if (issued < rows) {
      if (lane < 2) {  // lane py copies image row 2n + py of component row n
        const int s = issued & (kStages - 1);
        const float* row = g.rowp[0] + (lane ? g.half : 0ll);
        const unsigned b = smem_addr(bar + s);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * kTotal) : "memory");
        const unsigned dst = smem_addr(stage0 + s * 2 * kRowF4 + lane * kRowF4);
        // periodic columns: one copy of `first` bytes from column xw0, the
        // rest (strips crossing the right image edge, images narrower than a
        // strip) from column 0 on
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(row + xw0), "r"(first), "r"(b)
                     : "memory");
        if (first < kTotal) {
          const int W = 2 * a.w2;
          for (int done = first; done < kTotal;) {
            const int bytes = min(kTotal - done, W * 4);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst + unsigned(done)),
                "l"(row), "r"(bytes), "r"(b)
                : "memory");
            done += bytes;
          }
        }
      }
      g.advance(a);
    }
    ++issued;
  }

  __device__ __forceinline__ void init(const LevelArgs& a, int xc, int first_row, int nrows) {
    extern __shared__ __align__(128) unsigned char level_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    bar = reinterpret_cast<unsigned long long*>(level_smem) + warp * kStages;
    stage0 = reinterpret_cast<float4*>(level_smem + ((kWarpsPerCta * kStages * 8 + 127) / 128) * 128) +
             warp * kStages * 2 * kRowF4;
    g.init(a, 0, first_row);
    const int W = 2 * a.w2;
    xw0 = wrap(2 * (xc - lane * CW), W);
    first = min(kTotal, (W - xw0) * 4);
    issued = fetched = 0;
    rows = nrows;
    phase_bits = 0;
    if (lane == 0)
      for (int s = 0; s < kStages; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar + s)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    for (int k = 0; k < kStages - 1; ++k) issue_row(a);
  }

  __device__ __forceinline__ void load(const LevelArgs& a, float (&d)[4][CW]) {
    const int lane = threadIdx.x & 31;
    const int s = fetched & (kStages - 1);
    const unsigned b = smem_addr(bar + s), par = (phase_bits >> s) & 1u;
    unsigned ok = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(b), "r"(par)
          : "memory");
    } while (!ok);
    phase_bits ^= 1u << s;
    const float4* src = stage0 + s * 2 * kRowF4;
    sfor<0, 2>([&](auto PY_) {
      constexpr int py = decltype(PY_)::value;
      sfor<0, CW / 2>([&](auto Q_) {
        constexpr int q = decltype(Q_)::value;
        const float4 v = src[py * kRowF4 + lane * (CW / 2) + q];
        d[2 * py + 0][2 * q + 0] = v.x;
        d[2 * py + 1][2 * q + 0] = v.y;
        d[2 * py + 0][2 * q + 1] = v.z;
        d[2 * py + 1][2 * q + 1] = v.w;
      });
    });
    ++fetched;
    __syncwarp();
    issue_row(a);
  }
};

// Planar vector input (inverse levels: four band planes -> image) staged the
// same way: lanes 0..3 each copy band j's 32 x CW floats of a component row
// (one cp.async.bulk, more only across the right edge) into the stage, every
// lane then reads its own float4 per band. CW 4 only (stage_ok plans).
template <int CW, bool UPW>
struct TmaPlanarReader {
  static_assert(CW == 4, "planar staging: 4 component columns per lane");
  static constexpr int kBandF4 = 32;          // float4 per band row of the warp
  static constexpr int kBand = 32 * 4 * CW;   // bytes per band row of the warp
  RowReader<CW, false, false, false, UPW> g;  // row walk of the four planes
  float4* stage0;
  unsigned long long* bar;
  int xw0, first;  // first component column of lane 0 (wrapped), bytes up to the right edge
  int issued, fetched, rows;
  unsigned phase_bits;

  __device__ __forceinline__ void issue_row(const LevelArgs& a) {
    const int lane = threadIdx.x & 31;
    if (issued < rows) {
      if (lane < 4) {  // lane j copies band j
        const int s = issued & (kStages - 1);
        const float* row = lane == 0 ? g.rowp[0] : lane == 1 ? g.rowp[1] : lane == 2 ? g.rowp[2] : g.rowp[3];
        const unsigned b = smem_addr(bar + s);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * kBand) : "memory");
        const unsigned dst = smem_addr(stage0 + s * 4 * kBandF4 + lane * kBandF4);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(row + xw0), "r"(first), "r"(b)
                     : "memory");
        if (first < kBand) {
          for (int done = first; done < kBand;) {
            const int bytes = min(kBand - done, a.w2 * 4);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst + unsigned(done)),
                "l"(row), "r"(bytes), "r"(b)
                : "memory");
            done += bytes;
          }
        }
      }
      g.advance(a);
    }
    ++issued;
  }

  __device__ __forceinline__ void init(const LevelArgs& a, int xc, int first_row, int nrows) {
    extern __shared__ __align__(128) unsigned char level_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    bar = reinterpret_cast<unsigned long long*>(level_smem) + warp * kStages;
    stage0 = reinterpret_cast<float4*>(level_smem + ((kWarpsPerCta * kStages * 8 + 127) / 128) * 128) +
             warp * kStages * 4 * kBandF4;
    g.init(a, 0, first_row);
    xw0 = wrap(xc - lane * CW, a.w2);
    first = min(kBand, (a.w2 - xw0) * 4);
    issued = fetched = 0;
    rows = nrows;
    phase_bits = 0;
    if (lane == 0)
      for (int s = 0; s < kStages; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar + s)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    for (int k = 0; k < kStages - 1; ++k) issue_row(a);
  }

  __device__ __forceinline__ void load(const LevelArgs& a, float (&d)[4][CW]) {
    const int lane = threadIdx.x & 31;
    const int s = fetched & (kStages - 1);
    const unsigned b = smem_addr(bar + s), par = (phase_bits >> s) & 1u;
    unsigned ok = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(b), "r"(par)
          : "memory");
    } while (!ok);
    phase_bits ^= 1u << s;
    const float4* src = stage0 + s * 4 * kBandF4;
    sfor<0, 4>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      const float4 v = src[j * kBandF4 + lane];
      d[j][0] = v.x, d[j][1] = v.y, d[j][2] = v.z, d[j][3] = v.w;
    });
    ++fetched;
    __syncwarp();
    issue_row(a);
  }
};

__device__ __forceinline__ void st_vec(float* p, float4 v, bool stream) {
  if (stream) __stcs(reinterpret_cast<float4*>(p), v);
  else *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void st_vec(float* p, float2 v, bool stream) {
  if (stream) __stcs(reinterpret_cast<float2*>(p), v);
  else *reinterpret_cast<float2*>(p) = v;
}

// Writes output rows y0, y0 + 1, ... (no wrap); pointers advance per row.
template <int CW, bool IL, bool VEC, bool UPW = false>
struct RowWriter {
  float* p[4];
  long long pitch[4];
  int xc, kx0, kx1;  // columns stored: [kx0, kx1) (the keep window, LevelArgs)

  __device__ __forceinline__ void init(const LevelArgs& a, int xc_, int first_row) {
    xc = xc_, kx0 = a.keep_x0, kx1 = a.keep_x1 > 0 ? a.keep_x1 : a.w2;
    sfor<0, 4>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      if constexpr (IL) {
        pitch[j] = a.out_pitch[0];
        p[j] = a.out[0] + 2ll * first_row * a.out_pitch[0] + 2ll * xc;
      } else {
        pitch[j] = a.out_pitch[j];
        p[j] = a.out[j] + (long long)first_row * a.out_pitch[j] + xc;
      }
    });
  }

  __device__ __forceinline__ void advance() {
    constexpr long long sg = UPW ? -1 : 1;
    if constexpr (IL) {
      p[0] += sg * 2 * pitch[0];
    } else {
      sfor<0, 4>([&](auto J_) { p[decltype(J_)::value] += sg * pitch[decltype(J_)::value]; });
    }
  }

  // whether this lane stores (fixed per lane): the vector path stores all CW
  // columns or none (keep windows are lane-aligned there), the scalar path
  // checks each column
  __device__ __forceinline__ bool lane_in_range() const {
    return VEC ? xc >= kx0 && xc + CW <= kx1 : xc + CW > kx0 && xc < kx1;
  }

  // planar vector rows of the three detail bands only (the LL band of a
  // level that feeds the next level in the same pass is not written)
  __device__ __forceinline__ void store_details(const float (&v)[4][CW]) {
    static_assert(VEC && !IL && (CW == 4 || CW == 2), "detail rows: planar vector output");
    sfor<1, 4>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      if constexpr (CW == 4)
        st_vec(p[j], make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), true);
      else
        st_vec(p[j], make_float2(v[j][0], v[j][1]), true);
    });
  }

  __device__ __forceinline__ void store(const float (&v)[4][CW]) {
    if constexpr (VEC) {
      if constexpr (IL) {
        sfor<0, 2>([&](auto PY_) {
          constexpr int py = decltype(PY_)::value;
          float* q = p[0] + (py ? pitch[0] : 0ll);
          sfor<0, CW / 2>([&](auto Q_) {
            constexpr int k = decltype(Q_)::value;
            st_vec(q + 4 * k,
                   make_float4(v[2 * py][2 * k], v[2 * py + 1][2 * k], v[2 * py][2 * k + 1],
                               v[2 * py + 1][2 * k + 1]),
                   false);
          });
        });
      } else {
        sfor<0, 4>([&](auto J_) {
          constexpr int j = decltype(J_)::value;
          if constexpr (CW == 4)
            st_vec(p[j], make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), j != 0);
          else if constexpr (CW == 2)
            st_vec(p[j], make_float2(v[j][0], v[j][1]), j != 0);
          else
            sfor<0, CW>([&](auto C_) { p[j][decltype(C_)::value] = v[j][decltype(C_)::value]; });
        });
      }
    } else {
      sfor<0, CW>([&](auto C_) {
        constexpr int c = decltype(C_)::value;
        if (xc + c >= kx0 && xc + c < kx1) {
          sfor<0, 4>([&](auto J_) {
            constexpr int j = decltype(J_)::value;
            if constexpr (IL)
              p[0][((j >> 1) ? pitch[0] : 0ll) + 2 * c + (j & 1)] = v[j][c];
            else
              p[j][c] = v[j][c];
          });
        }
      });
    }
  }
};

// Planar vector rows addressed from the launch parameters on every store
// (row index and lane column only: no per-band pointers or pitches held in
// registers: fewer live registers in the register-bound fused level pair;
// in the single-level kernels it measured neutral to slower).
// The LL band (j = 0) of the last level of a pass is the next launch's
// input: with KEEP its stores carry an L2 evict_last policy, so it outlives
// the evict-first detail bands streaming past it in the 126 MB L2 (the level
// pair writes 64 MiB of LL_2 among 1 GB of detail bands at 16384^2).
template <int CW, bool UPW = false, bool KEEP = false>
struct LeanRowWriter {
  int xc, y;
  unsigned long long keep;  // L2 cache policy (KEEP)
  __device__ __forceinline__ void init(int xc_, int first_row) {
    xc = xc_, y = first_row;
    if constexpr (KEEP) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  }
  __device__ __forceinline__ void advance() { y += UPW ? -1 : 1; }
  template <int J0>
  __device__ __forceinline__ void store_from(const LevelArgs& a, const float (&v)[4][CW]) {
    sfor<J0, 4>([&](auto J_) {
      constexpr int j = decltype(J_)::value;
      float* q = a.out[j] + (long long)y * a.out_pitch[j] + xc;
      if constexpr (KEEP && j == 0 && CW == 2)
        asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(q), "f"(v[j][0]), "f"(v[j][1]),
                     "l"(keep)
                     : "memory");
      else if constexpr (KEEP && j == 0 && CW == 4)
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(q), "f"(v[j][0]),
                     "f"(v[j][1]), "f"(v[j][2]), "f"(v[j][3]), "l"(keep)
                     : "memory");
      else if constexpr (CW == 4)
        st_vec(q, make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), j != 0);
      else if constexpr (CW == 2)
        st_vec(q, make_float2(v[j][0], v[j][1]), j != 0);
      else if (j != 0)
        __stcs(q, v[j][0]);
      else
        *q = v[j][0];
    });
  }
};

// ------------------------------------------------------------- kernel

// One work item: warp `wid` streams its (strip, chunk) of the level, top-down
// or (UPW) bottom-up. RD: row reader type (default: RowReader, register
// prefetch; tuning harnesses substitute staged readers).
template <class P, int PF, bool IN_IL, bool OUT_IL, bool VEC, bool COH, bool UPW, class RD = void,
          int VF = kLevelPackedFma>
__device__ __forceinline__ void level_item(const LevelArgs& a, const int wid, const int chunk) {
  using M = Meta<P>;
  using SC = Sched<P, PF>;
  constexpr int S = M::S, CW = M::CW, D = SC::D, UNR = SC::UNR, NS0 = SC::slots(0);
  const int lane = threadIdx.x & 31;
  const int strip = wid % a.nstrips;
  const int xc = (strip * kOutLanes - 1 + lane) * CW;  // first component column of this lane
  const int y0 = a.y_begin + chunk * a.chunk_rows;
  const int y1 = min(a.y_end > 0 ? a.y_end : a.h2, y0 + a.chunk_rows);
  // first input row streamed, and the output row of iteration 0
  const int n0 = UPW ? y1 - 1 + M::L : y0 - M::U;
  const int yfirst = UPW ? n0 + M::U : n0 - M::L;
  const int rows = (y1 - y0) + M::U + M::L;
  const int iters = (rows + UNR - 1) / UNR * UNR;
  bool out_lane = lane >= 1 && lane <= kOutLanes;
  const int ys0 = max(y0, a.keep_y0), ys1 = min(y1, a.keep_y1 > 0 ? a.keep_y1 : a.h2);  // rows stored

  // every window starts zeroed, the load ring too: warm-up iterations read
  // slots no row has been loaded into yet (their outputs are discarded), and
  // values the compiler may treat as undefined there have been seen to change
  // stored outputs (the shifted-window schedule)
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

  std::conditional_t<std::is_void_v<RD>, RowReader<CW, IN_IL, VEC, COH, UPW>, RD> rd;
  rd.init(a, xc, n0, rows);
  RowWriter<CW, OUT_IL, VEC, UPW> wr;
  wr.init(a, xc, yfirst);
  out_lane = out_lane && wr.lane_in_range();
  // prologue: rows n0 .. n0+PF-1 land in the slots iteration 0.. expect
  sfor<0, PF>([&](auto U_) {
    constexpr int u = decltype(U_)::value;
    rd.load(a, ring[0][SC::slot(0, 0, -u)]);
  });

  for (int it = 0; it < iters; it += UNR) {
    sfor<0, UNR>([&](auto U_) {
      constexpr int u = decltype(U_)::value;
      const int i = it + u;
      if constexpr (!SC::kCirc) {  // shift windows 1..S by one row
        sfor<1, S + 1>([&](auto B_) {
          constexpr int b = decltype(B_)::value;
          constexpr int dep = SC::slots(b);
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
      }
      eval_step<P, PF, 0, u, D, CW, UPW, VF>(ring, a.neg_zero);
      // window 0 no longer needs row i - depth(0) + 1: reuse its slot for row
      // i + PF (kShift0: move every row one slot up, the new one into slot 0)
      if constexpr (SC::kShift0) {
        sfor<1, NS0>([&](auto K_) {
          constexpr int k = NS0 - decltype(K_)::value;  // NS0-1 .. 1
          sfor<0, 4>([&](auto J_) {
            sfor<0, CW>([&](auto C_) {
              ring[0][k][decltype(J_)::value][decltype(C_)::value] = ring[0][k - 1][decltype(J_)::value][decltype(C_)::value];
            });
          });
        });
        if (i + PF < rows) rd.load(a, ring[0][0]);
      } else if (i + PF < rows) {
        rd.load(a, ring[0][SC::slot(0, u, -PF)]);
      }
      sfor<1, S>([&](auto S_) { eval_step<P, PF, decltype(S_)::value, u, D, CW, UPW, VF>(ring, a.neg_zero); });
      const int y = UPW ? yfirst - i : yfirst + i;
      if (y >= ys0 && y < ys1 && out_lane) wr.store(ring[S][SC::slot(S, u, 0)]);
      wr.advance();
    });
  }
  (void)NS0;
}

// Chunk order and direction. With `alternate`, odd chunks stream bottom-up:
// two vertically adjacent chunks then reach their shared boundary rows at the
// same time (both start there, or both end there), so the warm-up rows one of
// them re-reads are still in L2 instead of coming from HBM again. Only the
// vector image-input kernels (forward levels) of programs with short
// sub-steps (P::kAlt) carry the bottom-up variant (ALT): a second unrolled
// body costs registers and nvcc time, and measured slower for the planar and
// image-output (inverse) kernels.
// STAGED: interleaved vector input through TmaRowReader (PF = 1: the stages
// are the prefetch).
template <class P, int PF, bool IN_IL, bool OUT_IL, bool VEC, bool COH, bool ALT, bool STAGED = false>
__device__ __forceinline__ void level_dispatch(const LevelArgs& a, const int wid) {
  static_assert(!STAGED || VEC, "staged rows: vector input");
  using StagedR = std::conditional_t<IN_IL, TmaRowReader<P::kCW, false>, TmaPlanarReader<P::kCW, false>>;
  using StagedRU = std::conditional_t<IN_IL, TmaRowReader<P::kCW, true>, TmaPlanarReader<P::kCW, true>>;
  const int c = wid / a.nstrips;
  const int chunk = a.reverse ? a.nchunks - 1 - c : c;
  if constexpr (ALT) {
    if (a.alternate && (chunk & 1)) {
      if constexpr (STAGED)
        level_item<P, 1, IN_IL, OUT_IL, VEC, COH, true, StagedRU>(a, wid, chunk);
      else
        level_item<P, PF, IN_IL, OUT_IL, VEC, COH, true>(a, wid, chunk);
      return;
    }
  }
  if constexpr (STAGED)
    level_item<P, 1, IN_IL, OUT_IL, VEC, COH, false, StagedR>(a, wid, chunk);
  else
    level_item<P, PF, IN_IL, OUT_IL, VEC, COH, false>(a, wid, chunk);
}

template <class P, int PF, bool IN_IL, bool OUT_IL, bool VEC, bool STAGED = false, int MIN_CTAS = 1>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MIN_CTAS)
level_kernel(const LevelArgs a) {
  // PDL (registry.hpp: launch_level): the previous kernel's results are
  // visible after the wait; the next launch may begin once every CTA of this
  // grid has started. Both are no-ops for a normal launch. wait_end: the
  // previous kernel (a symmetric level's crop kernel, which itself waited for
  // the level's input) computes something this launch does not read, so the
  // wait moves to the end: the two run together, and this grid still
  // completes only after its predecessor (the next level waits on it).
  if (!a.wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid < a.nstrips * a.nchunks)  // warp-uniform
    level_dispatch<P, PF, IN_IL, OUT_IL, VEC, false, VEC && IN_IL && P::kAlt, STAGED>(a, wid);
  if (a.wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace gpu
}  // namespace dwt2d_b200
