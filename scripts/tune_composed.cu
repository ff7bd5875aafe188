// Tuning harness (development only): one forward level of the composed
// (reference-rounding) CDF 9/7 programs in several forms — component
// columns per lane (CW 2/4) x scalar / packed (FFMA2 + FADD2) arithmetic —
// register-prefetch kernel, 16384^2 and 4096^2, bits compared per program;
// and the kShift schedule (every window shifted by register moves, loop body
// once per row) against the unrolled circular windows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo
//        --expt-relaxed-constexpr -I include scripts/tune_composed.cu -o build/tune_composed
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1704_08657_b200/csrc/generated/plans_gen.cuh"
#include "../paper_1704_08657_b200/csrc/kernels/level_engine.cuh"

using namespace dwt2d_b200::gpu;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <class B, int CW_, bool PACK, bool SHIFT = false>
struct V : B {
  static constexpr int kCW = CW_;
  static constexpr bool kPack = PACK;
  static constexpr bool kShift = SHIFT;
};

__global__ void fill(float* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (float)((i * 2654435761ull) % 1000003ull) * 1e-6f;
}

int sms;
template <class B, int U>
struct VU : B {
  static constexpr int kShiftUnroll = U;
};

// factored programs: packed-FMA form VF of the level kernel's sub-steps
template <class P, int VF>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_level_vf(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid < a.nstrips * a.nchunks) level_item<P, 2, true, false, true, false, false, void, VF>(a, wid, wid / a.nstrips);
}

template <class P, int PF = 2, bool STAGED = false, int VF = -1>
void run(const char* name, int W, float* img, float* out, std::vector<float>& ref, bool first) {
  auto kern = VF >= 0 ? k_level_vf<P, VF < 0 ? 0 : VF> : level_kernel<P, STAGED ? 1 : PF, true, false, true, STAGED>;
  const int smem = STAGED ? staged_bytes<P::kCW>() : 0;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem));
  const size_t n = size_t(W) * W;
  LevelArgs a{};
  const int w2 = W / 2;
  for (int j = 0; j < 4; ++j) a.in[j] = img, a.in_pitch[j] = W;
  for (int j = 0; j < 4; ++j) a.out[j] = out + j * (n / 4), a.out_pitch[j] = w2;
  a.w2 = w2, a.h2 = w2, a.vec = 1, a.neg_zero = -0.0f, a.staged = STAGED;
  a.nstrips = (w2 + kOutLanes * P::kCW - 1) / (kOutLanes * P::kCW);
  const long long resident = (long long)occ * kWarpsPerCta * sms;
  const long long rows_total = (long long)w2 * a.nstrips;
  const long long per_warp = (rows_total + resident - 1) / resident;
  long long chunk = per_warp <= 48 ? std::max<long long>(2, per_warp) : (rows_total + 5 * resident - 1) / (5 * resident);
  a.chunk_rows = int(std::min<long long>(chunk, w2));
  a.nchunks = (w2 + a.chunk_rows - 1) / a.chunk_rows;
  const unsigned blocks = unsigned((a.nstrips * a.nchunks + 3) / 4);
  CK(cudaMemset(out, 0, n * 4));
  kern<<<blocks, 128, smem>>>(a);
  CK(cudaDeviceSynchronize());
  std::vector<float> got(n);
  CK(cudaMemcpy(got.data(), out, n * 4, cudaMemcpyDeviceToHost));
  long long bad = 0;
  if (first) ref = got;
  else for (size_t i = 0; i < n; ++i) {
    const bool d = memcmp(&got[i], &ref[i], 4) != 0;
    if (d && bad < 3 && getenv("SHOW_DIFF")) {
      const size_t pl = i / (n / 4), r = (i % (n / 4)) / w2, c = i % w2;
      const size_t up = i >= size_t(w2) ? i - w2 : i, dn = i + w2 < n ? i + w2 : i;
      printf("   diff plane %zu row %zu col %zu: got %.9g ref %.9g (ref row-1 %.9g row+1 %.9g)\n", pl, r, c, got[i], ref[i],
             ref[up], ref[dn]);
    }
    bad += d;
  }
  if (!first && bad && getenv("SHOW_DIFF")) {
    for (int off = -2; off <= 2; ++off) {
      long long eq = 0, tot = 0;
      for (int pl = 0; pl < 4; ++pl)
        for (int r = 8; r < w2 - 8; ++r)
          for (int c = 0; c < w2; ++c) {
            const size_t i = pl * (n / 4) + size_t(r) * w2 + c, k = pl * (n / 4) + size_t(r + off) * w2 + c;
            eq += memcmp(&got[i], &ref[k], 4) == 0, ++tot;
          }
      printf("   got row r == ref row r%+d: %lld of %lld\n", off, eq, tot);
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  const int iters = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) kern<<<blocks, 128, smem>>>(a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= iters;
  printf("%5d^2 %-22s regs %3d spill-free? %s occ %d  %9.2f us  mismatches %lld\n", W, name, fa.numRegs,
         fa.localSizeBytes ? "no " : "yes", occ, ms * 1e3, bad);
}

int main() {
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  using namespace plans;
  for (int W : {getenv("SHOW_DIFF") ? 256 : 16384, 4096}) {
    const size_t n = size_t(W) * W;
    float *img, *out;
    CK(cudaMalloc(&img, n * 4));
    CK(cudaMalloc(&out, n * 4));
    fill<<<1184, 256>>>(img, (long long)n);
    std::vector<float> ref;
    if (getenv("PACK_ONLY")) {
      run<V<cdf97_nonseparable_convolution_base, 4, false, true>>("nsconv CW4 scalar shift", W, img, out, ref, true);
      run<V<cdf97_nonseparable_convolution_base, 4, true, true>, 1>("nsconv CW4 packed shift PF1", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_base, 4, true, true>, 1, true>("nsconv CW4 packed shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_base, 2, true, true>, 1, true>("nsconv CW2 packed shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, false, true>>("polyconv CW4 scalar shift", W, img, out, ref, true);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, true, true>, 1>("polyconv CW4 packed shift PF1", W, img, out, ref, false);
      cudaFree(img), cudaFree(out);
      continue;
    }
    if (getenv("TMA_ONLY")) {
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>>("nsconv-opt CW4 shift", W, img, out, ref, true);
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>, 1, true>("nsconv-opt CW4 shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_opt, 4, true>, 1, true>("nsconv-opt CW4 TMA", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_opt, 2, true>>("sepconv-opt CW2", W, img, out, ref, true);
      run<V<cdf97_separable_convolution_opt, 4, true>, 1, true>("sepconv-opt CW4 TMA", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_opt, 4, true, true>, 1, true>("sepconv-opt CW4 shift TMA", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_base, 2, false>>("sepconv CW2 scalar", W, img, out, ref, true);
      run<V<cdf97_separable_convolution_base, 4, true>, 1, true>("sepconv CW4 packed TMA", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_base, 4, false>, 1, true>("sepconv CW4 scalar TMA", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_base, 4, true, true>, 1, true>("sepconv CW4 packed shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, false, true>>("polyconv CW4 scalar shift", W, img, out, ref, true);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, true, true>, 1, true>("polyconv CW4 packed shift TMA", W, img, out, ref, false);
      cudaFree(img), cudaFree(out);
      continue;
    }
    if (getenv("VF_ONLY")) {
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>>("nsconv-opt CW4 shift", W, img, out, ref, true);
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>, 2, false, 1>("nsconv-opt CW4 shift VF1", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>, 2, false, 2>("nsconv-opt CW4 shift VF2", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_opt, 2, true, true>, 2, false, 1>("nsconv-opt CW2 shift VF1", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_opt, 2, true>>("sepconv-opt CW2", W, img, out, ref, true);
      run<V<cdf97_separable_convolution_opt, 2, true>, 2, false, 1>("sepconv-opt CW2 VF1", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_opt, 4, true>, 2, false, 1>("sepconv-opt CW4 VF1", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_opt, 4, true>, 2, false, 2>("sepconv-opt CW4 VF2", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_opt, 4, true>>("polyconv-opt CW4", W, img, out, ref, true);
      run<V<cdf97_nonseparable_polyconvolution_opt, 4, true>, 2, false, 1>("polyconv-opt CW4 VF1", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_opt, 4, true>, 2, false, 2>("polyconv-opt CW4 VF2", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_base, 2, false>>("sepconv CW2 scalar", W, img, out, ref, true);
      run<V<cdf97_separable_convolution_base, 4, true>>("sepconv CW4 packed", W, img, out, ref, false);
      run<V<cdf97_separable_convolution_base, 4, true>, 1>("sepconv CW4 packed PF1", W, img, out, ref, false);
      cudaFree(img), cudaFree(out);
      continue;
    }
    if (getenv("SHIFT_ONLY")) {
      run<V<cdf97_nonseparable_convolution_base, 2, true>>("nsconv CW2 packed", W, img, out, ref, true);
      run<V<cdf97_nonseparable_convolution_base, 2, false, true>>("nsconv CW2 scalar shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_base, 2, false, true>, 1>("nsconv CW2 scalar shift PF1", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_base, 4, false, true>>("nsconv CW4 scalar shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_base, 4, false, true>, 1, true>("nsconv CW4 scalar shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 2, false>>("polyconv CW2 scalar", W, img, out, ref, true);
      run<V<cdf97_nonseparable_polyconvolution_base, 2, false, true>>("polyconv CW2 scalar shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, false, true>>("polyconv CW4 scalar shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, true, true>>("polyconv CW4 packed shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, true, true>, 1, true>("polyconv CW4 packed shift TMA", W, img, out, ref, false);
      run<V<cdf97_nonseparable_polyconvolution_base, 4, false, true>, 1, true>("polyconv CW4 scalar shift TMA", W, img, out, ref, false);
      run<V<cdf53_nonseparable_convolution_base, 2, false>>("53 nsconv CW2 scalar", W, img, out, ref, true);
      run<V<cdf53_nonseparable_convolution_base, 2, false, true>>("53 nsconv CW2 scalar shift", W, img, out, ref, false);
      run<V<cdf53_nonseparable_convolution_base, 4, true, true>>("53 nsconv CW4 packed shift", W, img, out, ref, false);
      run<V<cdf53_nonseparable_polyconvolution_base, 2, false>>("53 polyconv CW2 scalar", W, img, out, ref, true);
      run<V<cdf53_nonseparable_polyconvolution_base, 2, false, true>>("53 polyconv CW2 scalar shift", W, img, out, ref, false);
      run<V<cdf53_nonseparable_polyconvolution_base, 4, true, true>>("53 polyconv CW4 packed shift", W, img, out, ref, false);
      run<V<dd137_separable_convolution_base, 4, true>>("dd sepconv CW4 packed", W, img, out, ref, true);
      run<V<dd137_separable_convolution_base, 4, true, true>>("dd sepconv CW4 packed shift", W, img, out, ref, false);
      run<V<cdf97_nonseparable_convolution_opt, 2, true>>("nsconv-opt CW2", W, img, out, ref, true);
      run<V<cdf97_nonseparable_convolution_opt, 4, true, true>>("nsconv-opt CW4 shift", W, img, out, ref, false);
      cudaFree(img), cudaFree(out);
      continue;
    }
    run<V<cdf97_separable_convolution_base, 2, false>>("sepconv CW2 scalar", W, img, out, ref, true);
    run<V<cdf97_separable_convolution_base, 2, true>>("sepconv CW2 packed", W, img, out, ref, false);
    run<V<cdf97_separable_convolution_base, 4, false>>("sepconv CW4 scalar", W, img, out, ref, false);
    run<V<cdf97_separable_convolution_base, 4, true>>("sepconv CW4 packed", W, img, out, ref, false);
    run<V<cdf97_nonseparable_polyconvolution_base, 4, false>>("polyconv CW4 scalar", W, img, out, ref, true);
    run<V<cdf97_nonseparable_polyconvolution_base, 4, true>>("polyconv CW4 packed", W, img, out, ref, false);
    run<V<cdf97_nonseparable_polyconvolution_base, 2, false>>("polyconv CW2 scalar", W, img, out, ref, false);
    run<V<cdf97_nonseparable_polyconvolution_base, 2, true>>("polyconv CW2 packed", W, img, out, ref, false);
    run<V<cdf97_nonseparable_lifting_base, 4, false>>("nslift CW4 scalar", W, img, out, ref, true);
    run<V<cdf97_nonseparable_lifting_base, 4, true>>("nslift CW4 packed", W, img, out, ref, false);
    run<V<cdf97_separable_lifting_base, 4, false>>("seplift CW4 scalar", W, img, out, ref, true);
    run<V<cdf97_separable_lifting_base, 4, true>>("seplift CW4 packed", W, img, out, ref, false);
    cudaFree(img), cudaFree(out);
  }
  return 0;
}
