// Tuning harness (development only): level 1 of the headline plan on a
// 16384^2 image with the input rows staged in shared memory by TMA bulk
// copies (cp.async.bulk, one lane issues a warp's 2 x 1 KB per component
// row, completion on an mbarrier per stage) vs the register-prefetch kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
//        --expt-relaxed-constexpr -I include scripts/tune_tma.cu -o build/tune_tma
#include <cstdio>
#include <cstdlib>
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

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

// Interleaved input (CW = 4: each lane 8 px = 32 B per image row), periodic
// rows and columns, NB stages of one component row (2 image rows x 1 KB).
template <bool UPW, int NB>
struct HTmaRowReader {
  static constexpr int CW = 4;
  float4* stage0;        // this warp's stage 0 (2 KB per stage)
  unsigned long long* bar;  // NB mbarriers
  const float* img;
  long long pitch;       // image row pitch (floats)
  int h2, W, c0;         // component rows, image width, first image column of lane 0
  int next_row, issued, fetched, rows;
  unsigned phase_bits;   // per-stage parity

  __device__ __forceinline__ void issue_row() {
    const int lane = threadIdx.x & 31;
    if (issued < rows && lane < 2) {  // lane py copies image row 2n + py
      const int s = issued % NB;
      const int n = wrap(next_row, h2);
      const unsigned b = smem_u32(bar + s);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2048) : "memory");
      const float* row = img + (2ll * n + lane) * pitch;
      char* dst = reinterpret_cast<char*>(stage0 + s * 128) + lane * 1024;
      const int xw = wrap(c0, W);
      const int first = min(1024, (W - xw) * 4);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst)),
                   "l"(row + xw), "r"(first), "r"(b)
                   : "memory");
      if (first < 1024)  // the strip wraps past the right edge
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst + first)),
                     "l"(row), "r"(1024 - first), "r"(b)
                     : "memory");
    }
    if (issued < rows) next_row += UPW ? -1 : 1;
    ++issued;
  }

  __device__ __forceinline__ void init(const LevelArgs& a, int xc, int first_row, int nrows) {
    extern __shared__ __align__(128) unsigned char smraw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    bar = reinterpret_cast<unsigned long long*>(smraw) + warp * NB;
    stage0 = reinterpret_cast<float4*>(smraw + kWarpsPerCta * NB * 8 + 128 * 0) + 0;
    stage0 = reinterpret_cast<float4*>(smraw + ((kWarpsPerCta * NB * 8 + 127) / 128) * 128) + warp * NB * 128;
    img = a.in[0];
    pitch = a.in_pitch[0];
    h2 = a.h2;
    W = 2 * a.w2;
    c0 = 2 * (xc - lane * CW);  // lane 0's first image column
    next_row = first_row;
    issued = fetched = 0;
    rows = nrows;
    phase_bits = 0;
    if (lane == 0)
      for (int s = 0; s < NB; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    for (int k = 0; k < NB - 1; ++k) issue_row();
  }

  __device__ __forceinline__ void load(const LevelArgs&, float (&d)[4][CW]) {
    const int lane = threadIdx.x & 31;
    const int s = fetched % NB;
    const unsigned b = smem_u32(bar + s);
    const unsigned par = (phase_bits >> s) & 1u;
    unsigned ok = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(b), "r"(par)
          : "memory");
    } while (!ok);
    phase_bits ^= 1u << s;
    const float4* src = stage0 + s * 128;
    for (int py = 0; py < 2; ++py)
      for (int q = 0; q < 2; ++q) {
        const float4 v = src[py * 64 + lane * 2 + q];
        d[2 * py + 0][2 * q + 0] = v.x;
        d[2 * py + 1][2 * q + 0] = v.y;
        d[2 * py + 0][2 * q + 1] = v.z;
        d[2 * py + 1][2 * q + 1] = v.w;
      }
    ++fetched;
    __syncwarp();
    issue_row();  // refills stage (fetched - 1 + NB - 1) % NB = the one read an iteration ago
  }
};

template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_reg(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;
  const int chunk = wid / a.nstrips;
  if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, false, true>(a, wid, chunk);
  else level_item<P, 2, true, false, true, false, false>(a, wid, chunk);
}

template <int NB, int MINB>
__global__ void __launch_bounds__(128, MINB) k_tma(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;
  const int chunk = wid / a.nstrips;
  if (a.alternate && (chunk & 1))
    level_item<P, 1, true, false, true, false, true, HTmaRowReader<true, NB>>(a, wid, chunk);
  else
    level_item<P, 1, true, false, true, false, false, HTmaRowReader<false, NB>>(a, wid, chunk);
}

// the product's staged reader and dispatch (level_engine.cuh)
__global__ void __launch_bounds__(128, 1) k_prod(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;
  level_dispatch<P, 2, true, false, true, false, true, true>(a, wid);
}
// the product kernel itself (PDL wait/trigger included)
template <class K>
void timeit(const char* name, K kern, const LevelArgs& a, unsigned blocks, size_t smem, float* out3,
            std::vector<float>* ref, std::vector<float>& host) {
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem));
  for (int i = 0; i < 3; ++i) kern<<<blocks, 128, smem>>>(a);
  CK(cudaDeviceSynchronize());
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
  const size_t n = size_t(a.w2) * a.h2;
  CK(cudaMemcpy(host.data(), out3, n * 4, cudaMemcpyDeviceToHost));
  long long bad = 0;
  if (ref->empty()) *ref = host;
  else
    for (size_t i = 0; i < n; ++i) bad += host[i] != (*ref)[i];
  printf("chunk %3d %-12s regs %3d occ %d smem %6zu  %8.2f us  %7.1f GB/s  mismatches %lld\n", a.chunk_rows, name,
         fa.numRegs, occ, smem, ms * 1e3, 8.0 * a.w2 * 4.0 * a.h2 / (ms * 1e-3) / 1e9, bad);
}

int main() {
  const int W = 16384, H = 16384;
  float* img;
  CK(cudaMalloc(&img, size_t(W) * H * 4));
  fill<<<1184, 256>>>(img, (long long)W * H);
  float* out[4];
  for (int j = 0; j < 4; ++j) CK(cudaMalloc(&out[j], size_t(W / 2) * (H / 2) * 4));
  std::vector<float> ref, host(size_t(W / 2) * (H / 2));
  auto smem = [](int nb) { return size_t(((kWarpsPerCta * nb * 8 + 127) / 128) * 128 + kWarpsPerCta * nb * 2048); };
  for (int chunk : {32, 64}) {
    LevelArgs a{};
    for (int j = 0; j < 4; ++j) a.in[j] = img, a.in_pitch[j] = W, a.out[j] = out[j], a.out_pitch[j] = W / 2;
    a.w2 = W / 2, a.h2 = H / 2;
    a.nstrips = (a.w2 + kOutLanes * 4 - 1) / (kOutLanes * 4);
    a.chunk_rows = chunk;
    a.nchunks = (a.h2 + chunk - 1) / chunk;
    a.vec = 1, a.alternate = 1;
    const unsigned blocks = unsigned((a.nstrips * a.nchunks + 3) / 4);
    timeit("reg pf2", k_reg<1>, a, blocks, 0, out[3], &ref, host);
    timeit("prod reader", k_prod, a, blocks, staged_bytes<4>(), out[3], &ref, host);
    // the same kernel held to 2 CTAs (8 warps) per SM by its shared memory:
    // the level-1 streaming rate a warp-specialised level pair would keep
    timeit("prod 2cta/SM", k_prod, a, blocks, 110 * 1024, out[3], &ref, host);
    timeit("prod kernel", level_kernel<P, 2, true, false, true>, a, blocks, staged_bytes<4>(), out[3], &ref, host);
    timeit("tma nb3", k_tma<3, 1>, a, blocks, smem(3), out[3], &ref, host);
    timeit("tma nb4", k_tma<4, 1>, a, blocks, smem(4), out[3], &ref, host);
    timeit("tma nb6", k_tma<6, 1>, a, blocks, smem(6), out[3], &ref, host);
    timeit("tma nb8", k_tma<8, 1>, a, blocks, smem(8), out[3], &ref, host);
    timeit("tma nb4 m4", k_tma<4, 4>, a, blocks, smem(4), out[3], &ref, host);
    timeit("tma nb8 m4", k_tma<8, 4>, a, blocks, smem(8), out[3], &ref, host);
  }
  return 0;
}
