// Tuning harness (development only): columns per lane (CW 2 vs 4) and row
// staging (register prefetch vs TMA) for the CW-2 programs (deep convolution
// windows) at 16384^2, single forward level.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
//        --expt-relaxed-constexpr -I include scripts/tune_cw.cu -o build/tune_cw
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1704_08657_b200/csrc/generated/plans_gen.cuh"
#include "../paper_1704_08657_b200/csrc/kernels/level_engine.cuh"

using namespace dwt2d_b200::gpu;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <class Base, int CW_>
struct WithCW : Base {
  static constexpr int kCW = CW_;
};

__global__ void fill(float* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (float)((i * 2654435761ull) % 1000003ull) * 1e-6f;
}

template <class P, bool STAGED>
void run(const char* name, float* img, float* out[4], int W, int H, int chunk) {
  LevelArgs a{};
  for (int j = 0; j < 4; ++j) a.in[j] = img, a.in_pitch[j] = W, a.out[j] = out[j], a.out_pitch[j] = W / 2;
  a.w2 = W / 2, a.h2 = H / 2;
  a.nstrips = (a.w2 + kOutLanes * P::kCW - 1) / (kOutLanes * P::kCW);
  a.chunk_rows = chunk;
  a.nchunks = (a.h2 + chunk - 1) / chunk;
  a.vec = 1, a.alternate = P::kAlt ? 1 : 0, a.staged = STAGED;
  const unsigned blocks = unsigned((a.nstrips * a.nchunks + 3) / 4);
  auto k = level_kernel<P, 2, true, false, true, STAGED>;
  const int smem = STAGED ? staged_bytes<P::kCW>() : 0;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, smem));
  for (int i = 0; i < 3; ++i) k<<<blocks, 128, smem>>>(a);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) k<<<blocks, 128, smem>>>(a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 10;
  printf("%-34s cw=%d staged=%d chunk=%3d regs=%3d spill=%zu occ=%d  %8.1f us  %7.1f GB/s\n", name, P::kCW, STAGED,
         chunk, fa.numRegs, fa.localSizeBytes, occ, ms * 1e3, 8.0 * W * (double)H / (ms * 1e-3) / 1e9);
}

template <class P>
void sweep(const char* name, float* img, float* out[4]) {
  const int W = 16384, H = 16384;
  for (int chunk : {32, 64}) {
    run<WithCW<P, 2>, false>(name, img, out, W, H, chunk);
    run<WithCW<P, 2>, true>(name, img, out, W, H, chunk);
    run<WithCW<P, 4>, false>(name, img, out, W, H, chunk);
    run<WithCW<P, 4>, true>(name, img, out, W, H, chunk);
  }
}

int main() {
  const int W = 16384, H = 16384;
  float* img;
  CK(cudaMalloc(&img, size_t(W) * H * 4));
  fill<<<1184, 256>>>(img, (long long)W * H);
  float* out[4];
  for (int j = 0; j < 4; ++j) CK(cudaMalloc(&out[j], size_t(W / 2) * (H / 2) * 4));
  sweep<plans::cdf97_separable_convolution_base>("cdf97 sep conv base", img, out);
  sweep<plans::cdf97_separable_convolution_opt>("cdf97 sep conv opt", img, out);
  sweep<plans::cdf97_nonseparable_convolution_opt>("cdf97 non-sep conv opt", img, out);
  return 0;
}
