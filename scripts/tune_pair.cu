// Tuning harness (development only): the fused level pair (levels 1+2,
// pair_engine.cuh) of the headline plan on a 16384^2 image, in its
// packed-FMA forms (VF 0 scalar, 1 pairs (c, c+1), 2 pairs (c, c+2)), each
// checked bit for bit against two per-level launches of the level kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo
//        --expt-relaxed-constexpr -I include scripts/tune_pair.cu -o build/tune_pair
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1704_08657_b200/csrc/generated/plans_gen.cuh"
#include "../paper_1704_08657_b200/csrc/kernels/pair_engine.cuh"

using namespace dwt2d_b200::gpu;
using P = plans::cdf97_nonseparable_lifting_opt;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill(float* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (float)((i * 2654435761ull) % 1000003ull) * 1e-6f;
}

template <int VF, int MINB, int CW1 = 4>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MINB) k_pair(const __grid_constant__ PairArgs t) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= t.nstrips * t.nchunks) return;
  pair_item<P, VF, CW1>(t, wid % t.nstrips, wid / t.nstrips);
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 16384, H = W;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *img, *mal, *ll1, *ll2;
  const size_t n = size_t(W) * H;
  CK(cudaMalloc(&img, n * 4));
  CK(cudaMalloc(&mal, n * 4));
  CK(cudaMalloc(&ll1, n));
  CK(cudaMalloc(&ll2, n / 4));
  fill<<<1184, 256>>>(img, (long long)n);
  auto level_args = [&](const float* in, long long ip, int w2, int h2, float* ll, long long lp) {
    LevelArgs a{};
    for (int j = 0; j < 4; ++j) a.in[j] = in, a.in_pitch[j] = ip;
    a.out[0] = ll, a.out_pitch[0] = lp;
    a.out[1] = mal + w2, a.out[2] = mal + size_t(h2) * W, a.out[3] = mal + size_t(h2) * W + w2;
    a.out_pitch[1] = a.out_pitch[2] = a.out_pitch[3] = W;
    a.w2 = w2, a.h2 = h2, a.vec = 1;
    return a;
  };
  // reference: one launch per level (register-prefetch level kernel)
  std::vector<float> ref(n), ref_ll(n / 16), got(n), got_ll(n / 16);
  CK(cudaMemset(mal, 0, n * 4));
  for (int l = 1; l <= 2; ++l) {
    LevelArgs a = l == 1 ? level_args(img, W, W / 2, H / 2, ll1, W / 2) : level_args(ll1, W / 2, W / 4, H / 4, ll2, W / 4);
    a.nstrips = (a.w2 + kOutLanes * 4 - 1) / (kOutLanes * 4);
    a.chunk_rows = 64;
    a.nchunks = (a.h2 + 63) / 64;
    level_kernel<P, 2, true, false, true><<<(a.nstrips * a.nchunks + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * 32>>>(a);
  }
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ref.data(), mal, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ref_ll.data(), ll2, n / 4, cudaMemcpyDeviceToHost));

  auto run = [&](const char* name, auto kern, int chunk_override, int cw1 = 4) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    const int smem = cw1 == 4 ? staged_bytes<4>() : staged_bytes<2>();
    const int lanes = cw1 == 4 ? pair_lanes<P, 4>() : pair_lanes<P, 2>();
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarpsPerCta * 32, smem));
    PairArgs t{};
    t.l1 = level_args(img, W, W / 2, H / 2, nullptr, 0);
    t.l2 = level_args(nullptr, 0, W / 4, H / 4, ll2, W / 4);
    t.l1.staged = 1;
    t.l1.neg_zero = -0.0f;
    t.nstrips = (t.l1.w2 + lanes * cw1 - 1) / (lanes * cw1);
    const long long resident = (long long)occ * kWarpsPerCta * sms;
    const long long per_wave = std::max<long long>(1, resident / t.nstrips);
    const int span = t.l2.h2;
    const long long waves = std::max<long long>(1, (span + 128 * per_wave) / (256 * per_wave));
    long long chunk = (span + waves * per_wave - 1) / (waves * per_wave);
    if (chunk_override) chunk = chunk_override;
    t.chunk_rows = int(std::min<long long>(chunk, span));
    t.nchunks = (span + t.chunk_rows - 1) / t.chunk_rows;
    const unsigned blocks = unsigned((t.nstrips * t.nchunks + kWarpsPerCta - 1) / kWarpsPerCta);
    CK(cudaMemset(mal, 0, n * 4));
    CK(cudaMemset(ll2, 0, n / 4));
    kern<<<blocks, kWarpsPerCta * 32, smem>>>(t);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got.data(), mal, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(got_ll.data(), ll2, n / 4, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (size_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 4) != 0;
    for (size_t i = 0; i < n / 16; ++i) bad += memcmp(&got_ll[i], &ref_ll[i], 4) != 0;
    for (int i = 0; i < 3; ++i) kern<<<blocks, kWarpsPerCta * 32, smem>>>(t);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    const int iters = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) kern<<<blocks, kWarpsPerCta * 32, smem>>>(t);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= iters;
    // algorithmic bytes: 8 B per pixel per level (reference bench.cpp:84-85)
    const double alg = 8.0 * n * 1.25;
    printf("wpc %d %-14s regs %3d occ %2d chunk %4d  %8.2f us  %7.1f GB/s alg  mismatches %lld\n", kWarpsPerCta, name, fa.numRegs, occ,
           t.chunk_rows, ms * 1e3, alg / (ms * 1e-3) / 1e9, bad);
  };
  for (int rep = 0; rep < 2; ++rep) {
    run("VF0 scalar", k_pair<0, 1>, 0);
    run("VF1 (c,c+1)", k_pair<1, 1>, 0);
    run("VF2 (c,c+2)", k_pair<2, 1>, 0);
    run("CW2 VF1", k_pair<1, 1, 2>, 0, 2);
    run("CW2 VF1 minb4", k_pair<1, 4, 2>, 0, 2);
    run("CW2 VF0 minb4", k_pair<0, 4, 2>, 0, 2);
    run("CW2 VF1 ch128", k_pair<1, 4, 2>, 128, 2);
  }
  return 0;
}
