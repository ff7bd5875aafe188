// Tuning harness (development only): one forward level of the headline plan
// (register-prefetch level kernel, the one levels >= 3 of a 16384^2 pyramid
// use) in its packed-FMA forms VF 0/1/2 (level_engine.cuh: eval_step), at
// the input sizes of levels 3..5, checked bit for bit against VF 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo
//        --expt-relaxed-constexpr -I include scripts/tune_level_vf.cu -o build/tune_level_vf
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1704_08657_b200/csrc/generated/plans_gen.cuh"
#include "../paper_1704_08657_b200/csrc/kernels/level_engine.cuh"

using namespace dwt2d_b200::gpu;
using P = plans::cdf97_nonseparable_lifting_opt;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill(float* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (float)((i * 2654435761ull) % 1000003ull) * 1e-6f;
}

template <int VF>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 1) k_level(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;
  const int c = wid / a.nstrips;
  const int chunk = a.reverse ? a.nchunks - 1 - c : c;
  if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, false, true, void, VF>(a, wid, chunk);
  else level_item<P, 2, true, false, true, false, false, void, VF>(a, wid, chunk);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int W : {4096, 2048, 1024, 512}) {
    const int H = W;
    const size_t n = size_t(W) * H;
    float *img, *out;
    CK(cudaMalloc(&img, n * 4));
    CK(cudaMalloc(&out, n * 4));
    fill<<<1184, 256>>>(img, (long long)n);
    std::vector<float> ref(n), got(n);
    auto run = [&](const char* name, auto kern, bool first) {
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, kern));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0));
      LevelArgs a{};
      const int w2 = W / 2, h2 = H / 2;
      for (int j = 0; j < 4; ++j) a.in[j] = img, a.in_pitch[j] = W;
      a.out[0] = out, a.out_pitch[0] = w2;
      a.out[1] = out + n / 4, a.out[2] = out + n / 2, a.out[3] = out + 3 * n / 4;
      a.out_pitch[1] = a.out_pitch[2] = a.out_pitch[3] = w2;
      a.w2 = w2, a.h2 = h2, a.vec = 1, a.reverse = 1;
      a.nstrips = (w2 + kOutLanes * 4 - 1) / (kOutLanes * 4);
      const long long resident = (long long)occ * kWarpsPerCta * sms;
      const long long rows_total = (long long)h2 * a.nstrips;
      const long long per_warp = (rows_total + resident - 1) / resident;
      long long chunk = per_warp <= 48 ? std::max<long long>(2, per_warp) : (rows_total + 5 * resident - 1) / (5 * resident);
      a.chunk_rows = int(std::min<long long>(chunk, h2));
      a.nchunks = (h2 + a.chunk_rows - 1) / a.chunk_rows;
      a.alternate = size_t(w2) * h2 * 16 >= (size_t(32) << 20);
      const unsigned blocks = unsigned((a.nstrips * a.nchunks + 3) / 4);
      CK(cudaMemset(out, 0, n * 4));
      kern<<<blocks, 128>>>(a);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(got.data(), out, n * 4, cudaMemcpyDeviceToHost));
      long long bad = 0;
      if (first) ref = got;
      else for (size_t i = 0; i < n; ++i) bad += memcmp(&got[i], &ref[i], 4) != 0;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0), cudaEventCreate(&e1);
      const int iters = 50;
      cudaEventRecord(e0);
      for (int i = 0; i < iters; ++i) kern<<<blocks, 128>>>(a);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= iters;
      printf("%5d^2 %-4s regs %3d occ %d chunk %4d  %8.2f us  %7.1f GB/s alg  mismatches %lld\n", W, name, fa.numRegs,
             occ, a.chunk_rows, ms * 1e3, 8.0 * n / (ms * 1e-3) / 1e9, bad);
    };
    run("VF0", k_level<0>, true);
    run("VF1", k_level<1>, false);
    run("VF2", k_level<2>, false);
    run("VF0", k_level<0>, false);
    cudaFree(img), cudaFree(out);
  }
  return 0;
}
