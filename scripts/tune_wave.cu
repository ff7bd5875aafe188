// Tuning harness (development only): level 1 of the headline plan on a
// 16384^2 image under different work-distribution / load-path variants, to
// separate the costs of the wavefront kernel (persistent ticket loop,
// L2-coherent loads) from its scheduling.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
//        --expt-relaxed-constexpr -I include scripts/tune_wave.cu -o build/tune_wave
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

// one item per warp, COH selectable
template <bool COH>
__global__ void __launch_bounds__(128) k_static(const LevelArgs a) {
  const int wid = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (wid >= a.nstrips * a.nchunks) return;
  const int chunk = wid / a.nstrips;
  if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, wid, chunk);
  else level_item<P, 2, true, false, true, COH, false>(a, wid, chunk);
}

// persistent: tickets in item order by atomicAdd
template <bool COH>
__global__ void __launch_bounds__(128) k_persist(const LevelArgs a, unsigned* ctr) {
  const int lane = threadIdx.x & 31;
  const unsigned total = unsigned(a.nstrips * a.nchunks);
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(ctr, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= total) break;
    const int chunk = int(t) / a.nstrips, strip = int(t) % a.nstrips;
    if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, strip, chunk);
    else level_item<P, 2, true, false, true, COH, false>(a, strip, chunk);
  }
}

// persistent, next ticket claimed while the current item runs
template <bool COH>
__global__ void __launch_bounds__(128) k_persist_pf(const LevelArgs a, unsigned* ctr) {
  const int lane = threadIdx.x & 31;
  const unsigned total = unsigned(a.nstrips * a.nchunks);
  unsigned cur = 0;
  if (lane == 0) cur = atomicAdd(ctr, 1u);
  cur = __shfl_sync(0xffffffffu, cur, 0);
  while (cur < total) {
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(ctr, 1u);
    const int chunk = int(cur) / a.nstrips, strip = int(cur) % a.nstrips;
    if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, strip, chunk);
    else level_item<P, 2, true, false, true, COH, false>(a, strip, chunk);
    cur = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

// persistent, static grid-stride assignment (no atomics)
template <bool COH>
__global__ void __launch_bounds__(128) k_stride(const LevelArgs a, unsigned* ctr) {
  const unsigned total = unsigned(a.nstrips * a.nchunks);
  const unsigned nw = gridDim.x * kWarpsPerCta;
  for (unsigned cur = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); cur < total; cur += nw) {
    const int chunk = int(cur) / a.nstrips, strip = int(cur) % a.nstrips;
    if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, strip, chunk);
    else level_item<P, 2, true, false, true, COH, false>(a, strip, chunk);
  }
}

// one CTA per 4-strip group like k_static, but the group comes from a ticket
// taken when the CTA starts (dynamic block index: start order = ticket order)
template <bool COH>
__global__ void __launch_bounds__(128) k_dyn(const LevelArgs a, unsigned* ctr) {
  __shared__ unsigned tk;
  const int warp = threadIdx.x >> 5;
  const int groups = (a.nstrips + kWarpsPerCta - 1) / kWarpsPerCta;
  if (threadIdx.x == 0) tk = atomicAdd(ctr, 1u);
  __syncthreads();
  const unsigned t = tk;
  const int chunk = int(t) / groups, strip = (int(t) % groups) * kWarpsPerCta + warp;
  if (strip < a.nstrips) {
    if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, strip, chunk);
    else level_item<P, 2, true, false, true, COH, false>(a, strip, chunk);
  }
}

// persistent, one ticket per CTA: its 4 warps take 4 adjacent strips of one
// chunk together (like a hardware-scheduled CTA of the static kernel)
template <bool COH>
__global__ void __launch_bounds__(128) k_persist_cta(const LevelArgs a, unsigned* ctr) {
  __shared__ unsigned tk;
  const int warp = threadIdx.x >> 5;
  const int groups = (a.nstrips + kWarpsPerCta - 1) / kWarpsPerCta;
  const unsigned total = unsigned(groups * a.nchunks);
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(ctr, 1u);
    __syncthreads();
    const unsigned t = tk;
    __syncthreads();
    if (t >= total) break;
    const int chunk = int(t) / groups, strip = (int(t) % groups) * kWarpsPerCta + warp;
    if (strip < a.nstrips) {
      if (a.alternate && (chunk & 1)) level_item<P, 2, true, false, true, COH, true>(a, strip, chunk);
      else level_item<P, 2, true, false, true, COH, false>(a, strip, chunk);
    }
  }
}

int main() {
  const int W = 16384, H = 16384;
  float* img;
  CK(cudaMalloc(&img, size_t(W) * H * 4));
  fill<<<1184, 256>>>(img, (long long)W * H);
  float* out[4];
  for (int j = 0; j < 4; ++j) CK(cudaMalloc(&out[j], size_t(W / 2) * (H / 2) * 4));
  unsigned* ctr;
  CK(cudaMalloc(&ctr, 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int alt : {1})
  for (int chunk : {32, 64}) {
    LevelArgs a{};
    for (int j = 0; j < 4; ++j) a.in[j] = img, a.in_pitch[j] = W, a.out[j] = out[j], a.out_pitch[j] = W / 2;
    a.w2 = W / 2, a.h2 = H / 2;
    a.nstrips = (a.w2 + kOutLanes * 4 - 1) / (kOutLanes * 4);
    a.chunk_rows = chunk;
    a.nchunks = (a.h2 + chunk - 1) / chunk;
    a.vec = 1, a.alternate = alt;
    const unsigned blocks = unsigned((a.nstrips * a.nchunks + 3) / 4);
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_persist<true>, 128, 0));
    for (int v = 0; v < 12; ++v) {
      auto go = [&] {
        if (v == 0) k_static<false><<<blocks, 128>>>(a);
        if (v == 1) k_static<true><<<blocks, 128>>>(a);
        if (v == 2) { cudaMemsetAsync(ctr, 0, 4); k_persist<false><<<occ * sms, 128>>>(a, ctr); }
        if (v == 3) { cudaMemsetAsync(ctr, 0, 4); k_persist<true><<<occ * sms, 128>>>(a, ctr); }
        if (v == 4) { cudaMemsetAsync(ctr, 0, 4); k_persist_cta<false><<<occ * sms, 128>>>(a, ctr); }
        if (v == 5) { cudaMemsetAsync(ctr, 0, 4); k_persist_cta<true><<<occ * sms, 128>>>(a, ctr); }
        if (v == 6) { cudaMemsetAsync(ctr, 0, 4); k_persist_pf<false><<<occ * sms, 128>>>(a, ctr); }
        if (v == 7) { cudaMemsetAsync(ctr, 0, 4); k_persist_pf<true><<<occ * sms, 128>>>(a, ctr); }
        if (v == 8) { k_stride<false><<<occ * sms, 128>>>(a, ctr); }
        if (v == 9) { k_stride<false><<<blocks / 2 + 1, 128>>>(a, ctr); }
        const unsigned gblocks = unsigned(((a.nstrips + 3) / 4) * a.nchunks);
        if (v == 10) { cudaMemsetAsync(ctr, 0, 4); k_dyn<false><<<gblocks, 128>>>(a, ctr); }
        if (v == 11) { cudaMemsetAsync(ctr, 0, 4); k_dyn<true><<<gblocks, 128>>>(a, ctr); }
      };
      for (int i = 0; i < 3; ++i) go();
      CK(cudaDeviceSynchronize());
      const int iters = 20;
      cudaEventRecord(e0);
      for (int i = 0; i < iters; ++i) go();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= iters;
      static const char* names[] = {"static nc", "static cg", "persist nc", "persist cg", "pcta nc", "pcta cg", "ppf nc", "ppf cg", "stride nc", "stride2 nc", "dyn nc", "dyn cg"};
      printf("alt %d chunk %3d %-11s occ %d  %8.2f us  %7.1f GB/s\n", alt, chunk, names[v], occ, ms * 1e3,
             8.0 * W * (double)H / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
