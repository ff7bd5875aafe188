// Levels 1 and 2 of a forward Mallat pyramid in ONE pass over the image: the
// LL_1 band never goes to HBM (north star: "multi-level
// decomposition keeps the LL band resident").
//
// A warp streams a strip of the image exactly like level_item (TMA-staged
// rows, register windows, all sub-steps of the level fused), and feeds every
// LL_1 row it produces, still in registers, into a second instance of the
// same step program running on the level-2 component grid:
//   * lane l owns 4 level-1 component columns x..x+3 (8 image columns); the
//     LL_1 values of those columns are level-2 component columns x/2, x/2+1
//     (CW = 2): even LL_1 columns are the level-2 "e" components, odd ones
//     the "o" components; an even LL_1 row gives (ee, oe), the next odd row
//     (eo, oo) — the polyphase split of LL_1 (image.hpp:73-94) happens in
//     registers;
//   * level 2 reaches 2 component columns = one lane at CW 2, so its outputs
//     are valid on lanes 2..29 when LL_1 is valid on lanes 1..30: strips are
//     28 lanes apart and both levels store from lanes 2..29 only;
//   * vertically, a chunk of level-2 rows [m0, m1) needs LL_1 rows
//     [2(m0 - U), 2(m1 + L)), i.e. level 1 streams 2(U + L) extra rows per
//     chunk besides its own U + L warm-up.
// Periodic extension composes: LL_1 rows/columns outside the image are
// recomputed from wrapped image rows/columns, which equals LL_1 wrapped. The
// arithmetic per value is the per-level kernels', so the pyramid is
// bit-identical to two level launches (tested).
#pragma once

#include "level_engine.cuh"

namespace dwt2d_b200 {
namespace gpu {

template <class P>
struct PairTraits {
  using M = Meta<P>;
  static constexpr bool ok = P::kCW == 4 && M::HL <= 2 && M::HR <= 2 && !shift_rows<P>();
};

// VF: packed-FMA form of the sub-steps (level_engine.cuh: eval_step).
// Level 2 runs on every odd LL_1 row, also before the first and after the
// last row of the chunk (their outputs are never stored, and no stored
// output reads them): the warp stays convergent, so the level-2 shuffles
// need no collective re-convergence blocks.
// Lanes of a warp that store both levels when each lane owns CW1 level-1
// columns: the halo lanes on either side cover level 1's reach at CW1
// columns per lane plus level 2's at CW1 / 2.
template <class P, int CW1>
__host__ __device__ constexpr int pair_halo_lanes() {
  return (Meta<P>::HL + CW1 - 1) / CW1 + (Meta<P>::HL + CW1 / 2 - 1) / (CW1 / 2);
}
template <class P, int CW1>
__host__ __device__ constexpr int pair_lanes() {
  return 32 - 2 * pair_halo_lanes<P, CW1>();
}

template <class P, int VF = kPackedFma, int CW1 = 4>
__device__ __forceinline__ void pair_item(const PairArgs& t, const int strip, const int chunk) {
  using M = Meta<P>;
  using SC = Sched<P, 1>;
  static_assert(!SC::kShift0, "level pair: circular load ring");
  constexpr int S = M::S, D = SC::D, UNR1 = SC::UNR, UNR = 2 * UNR1;
  constexpr int CW2 = CW1 / 2, U = M::U, L = M::L;
  constexpr int HALO = pair_halo_lanes<P, CW1>(), LANES = pair_lanes<P, CW1>();
  static_assert(PairTraits<P>::ok, "pair engine: CW 4 and a reach of at most 2 columns");
  static_assert(M::HL == M::HR, "pair engine: symmetric horizontal reach");
  const LevelArgs& a1 = t.l1;
  const LevelArgs& a2 = t.l2;
  const int lane = threadIdx.x & 31;
  const int xc1 = (strip * LANES - HALO + lane) * CW1;  // level-1 component column of this lane
  const int xc2 = xc1 / 2;                              // exact: xc1 is a multiple of CW1
  const int m0 = t.m_begin + chunk * t.chunk_rows, m1 = min(t.m_end > 0 ? t.m_end : a2.h2, m0 + t.chunk_rows);
  const int n02 = m0 - U;              // first level-2 input row
  const int rows2 = (m1 - m0) + U + L;
  const int n01 = 2 * n02 - U;         // first level-1 input row
  const int rows1 = 2 * rows2 + U + L;
  const int yfirst1 = n01 - L;         // LL_1 row produced at level-1 iteration 0
  const int yfirst2 = n02 - L;         // level-2 output row at level-2 iteration 0
  const int iters = (rows1 + UNR - 1) / UNR * UNR;
  const bool core = lane >= HALO && lane < HALO + LANES;

  float ring1[S + 1][D][4][CW1];
  float ring2[S + 1][D][4][CW2];
  float pend[2][CW2];  // (ee, oe) of the last even LL_1 row
  sfor<0, S + 1>([&](auto B_) {  // all windows zeroed (level_engine.cuh: level_item)
    sfor<0, D>([&](auto K_) {
      sfor<0, 4>([&](auto J_) {
        constexpr int b = decltype(B_)::value, k = decltype(K_)::value, j = decltype(J_)::value;
        sfor<0, CW1>([&](auto C_) { ring1[b][k][j][decltype(C_)::value] = 0.0f; });
        sfor<0, CW2>([&](auto C_) { ring2[b][k][j][decltype(C_)::value] = 0.0f; });
      });
    });
  });
  sfor<0, 2>([&](auto A_) { sfor<0, CW2>([&](auto C_) { pend[decltype(A_)::value][decltype(C_)::value] = 0.0f; }); });

  TmaRowReader<CW1, false> rd;
  rd.init(a1, xc1, n01, rows1);
  LeanRowWriter<CW1> w1;
  w1.init(xc1, yfirst1);
  LeanRowWriter<CW2, false, true> w2;  // LL_2 (the next launch's input) kept in L2
  w2.init(xc2, yfirst2);
  const bool st1 = core && xc1 + CW1 <= a1.w2;
  const bool st2 = core && xc2 + CW2 <= a2.w2;
  rd.load(a1, ring1[0][SC::slot(0, 0, 0)]);

  for (int it = 0; it < iters; it += UNR) {
    sfor<0, UNR>([&](auto U_) {
      constexpr int u = decltype(U_)::value;
      const int i = it + u;
      // ---------------------------------------------------------- level 1
      if constexpr (!SC::kCirc) {
        sfor<1, S + 1>([&](auto B_) {
          constexpr int b = decltype(B_)::value;
          constexpr int dep = SC::slots(b);
          sfor<1, dep>([&](auto K_) {
            constexpr int k = dep - decltype(K_)::value;
            sfor<0, 4>([&](auto J_) {
              sfor<0, CW1>([&](auto C_) {
                ring1[b][k][decltype(J_)::value][decltype(C_)::value] =
                    ring1[b][k - 1][decltype(J_)::value][decltype(C_)::value];
              });
            });
          });
        });
      }
      eval_step<P, 1, 0, u, D, CW1, false, VF>(ring1, a1.neg_zero);
      if (i + 1 < rows1) rd.load(a1, ring1[0][SC::slot(0, u, -1)]);
      sfor<1, S>([&](auto S_) { eval_step<P, 1, decltype(S_)::value, u, D, CW1, false, VF>(ring1, a1.neg_zero); });
      constexpr int so = SC::slot(S, u, 0);
      const int y1 = yfirst1 + i;
      if (y1 >= 2 * m0 && y1 < 2 * m1 && st1) w1.store_from<1>(a1, ring1[S][so]);
      w1.advance();
      // ------------------------------------------- LL_1 row -> level 2
      const int k = i - (U + L);  // LL_1 row 2 * n02 + k
      constexpr int kpar = ((u - (U + L)) % 2 + 2) % 2;
      if constexpr (kpar == 0) {
        sfor<0, CW2>([&](auto C_) {
          constexpr int c = decltype(C_)::value;
          pend[0][c] = ring1[S][so][0][2 * c];
          pend[1][c] = ring1[S][so][0][2 * c + 1];
        });
      } else {
        constexpr int u2 = (((u - (U + L) - 1) / 2) % UNR1 + UNR1) % UNR1;
        const int i2 = (k - 1) >> 1;  // floor: distinct rows also before the chunk
        {
          if constexpr (!SC::kCirc) {
            sfor<1, S + 1>([&](auto B_) {
              constexpr int b = decltype(B_)::value;
              constexpr int dep = SC::slots(b);
              sfor<1, dep>([&](auto K_) {
                constexpr int kk = dep - decltype(K_)::value;
                sfor<0, 4>([&](auto J_) {
                  sfor<0, CW2>([&](auto C_) {
                    ring2[b][kk][decltype(J_)::value][decltype(C_)::value] =
                        ring2[b][kk - 1][decltype(J_)::value][decltype(C_)::value];
                  });
                });
              });
            });
          }
          constexpr int s0 = SC::slot(0, u2, 0);
          sfor<0, CW2>([&](auto C_) {
            constexpr int c = decltype(C_)::value;
            ring2[0][s0][0][c] = pend[0][c];
            ring2[0][s0][1][c] = pend[1][c];
            ring2[0][s0][2][c] = ring1[S][so][0][2 * c];
            ring2[0][s0][3][c] = ring1[S][so][0][2 * c + 1];
          });
          sfor<0, S>([&](auto S_) { eval_step<P, 1, decltype(S_)::value, u2, D, CW2, false, VF>(ring2, a1.neg_zero); });
          const int y2 = yfirst2 + i2;
          if (y2 >= m0 && y2 < m1 && st2) {
            w2.y = y2;
            w2.store_from<0>(a2, ring2[S][SC::slot(S, u2, 0)]);
          }
        }
      }
    });
  }
}

template <class P>
__global__ void __launch_bounds__(kWarpsPerCta * 32) pair_kernel(const __grid_constant__ PairArgs t) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= t.nstrips * t.nchunks) return;  // warp-uniform
  pair_item<P>(t, wid % t.nstrips, wid / t.nstrips);
}

}  // namespace gpu
}  // namespace dwt2d_b200
