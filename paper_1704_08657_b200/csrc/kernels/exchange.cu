// Device-side halo exchange between the ranks of a row-strip sharded
// pyramid (reference analogue: row bands plus a barrier per
// step, executor.hpp:211-225). Every rank owns an exchange window in its
// device memory (halo receive buffers for every level and three counters,
// capi.cpp: dwt2d_shard); its ring neighbours map the window (same process:
// peer access; other processes: CUDA IPC) and write into it directly over
// NVLink:
//
//   halo_push_kernel    my first rows -> prev's bottom halo, my last rows ->
//                       next's top halo (peer stores, float4), then the last
//                       CTA to finish bumps the neighbours' arrival counters
//                       (release, system scope)
//   halo_wait_kernel    one thread spins (acquire, system scope) until both
//                       of my arrival counters passed the count it has seen
//   pyramid_done_kernel after a rank's last level: tells both neighbours it
//                       no longer reads its halo buffers
//   pyramid_start_kernel before the next pyramid's first push: waits for
//                       both neighbours' done signals
//
// All counters are monotonic and live in device memory, so the sequence is
// stream-ordered and can be captured in a CUDA graph and replayed: no host
// round trip per level. A wait that does not complete within the timeout
// records what it waited for in host-mapped memory and traps (a broken ring
// fails loudly instead of hanging the GPU; dwt2d_shard_status reports it).
#include <cuda_runtime.h>

#include <algorithm>

#include "level_types.hpp"

namespace dwt2d_b200 {
namespace gpu {

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// spin until *flag >= target; false on timeout
__device__ bool spin_until(const unsigned* flag, unsigned target, unsigned long long timeout_ns) {
  const unsigned long long t0 = global_ns();
  unsigned ns = 32;
  while (int(ld_acquire_sys(flag) - target) < 0) {
    if (global_ns() - t0 > timeout_ns) return false;
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : ns;
  }
  return true;
}

// A wait that timed out: what it waited for goes to the shard's
// diagnostics block in host-mapped memory (readable by the host after the
// trap has taken the context down): code, the counter's value, the target.
__device__ void report_and_trap(unsigned* diag, unsigned code, const unsigned* flag, unsigned target) {
  volatile unsigned* d = diag;
  d[1] = ld_acquire_sys(flag);
  d[2] = target;
  d[0] = code;
  __threadfence_system();
  __trap();
}

__global__ void __launch_bounds__(256) halo_push_kernel(const __grid_constant__ HaloPushArgs a) {
  // PDL: resident during the previous level's tail; its LL rows (this
  // push's source) are complete after the wait. A push that also waits for
  // the neighbours (wait_after) releases no dependents early: their CTAs
  // would sit resident at their own griddepcontrol.wait and, on ranks
  // sharing a GPU (virtual ranks), could starve the neighbour being waited
  // for. For the same reason every wait on another rank spins in ONE CTA.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!a.wait_after) asm volatile("griddepcontrol.launch_dependents;" :::);
  // rows [0, rows_first) -> dst_prev, rows [height - rows_last, height) -> dst_next
  const int rows = a.rows_first + a.rows_last;
  if (a.vec) {
    const int w4 = a.width / 4;
    const long long total = (long long)rows * w4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
      const int r = int(i / w4), c = int(i % w4) * 4;
      const bool first = r < a.rows_first;
      const int sr = first ? r : a.height - a.rows_last + (r - a.rows_first);
      const int dr = first ? r : r - a.rows_first;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.src + sr * a.src_pitch + c));
      float* d = (first ? a.dst_prev : a.dst_next) + dr * a.dst_pitch + c;
      __stcg(reinterpret_cast<float4*>(d), v);
    }
  } else {
    const long long total = (long long)rows * a.width;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
      const int r = int(i / a.width), c = int(i % a.width);
      const bool first = r < a.rows_first;
      const int sr = first ? r : a.height - a.rows_last + (r - a.rows_first);
      const int dr = first ? r : r - a.rows_first;
      (first ? a.dst_prev : a.dst_next)[dr * a.dst_pitch + c] = __ldcg(a.src + sr * a.src_pitch + c);
    }
  }
  // last CTA out signals both neighbours. The CTA barrier orders every
  // thread's peer stores before thread 0's system-scope fence, which is
  // cumulative: they are visible system-wide before the CTA arrives
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(a.arrive, 1u);
    if (prev == gridDim.x - 1) {
      *a.arrive = 0;  // ready for the next push (no other CTA touches it now)
      // every CTA fenced its stores before arriving; one more fence orders
      // the count this CTA observed before the two signals (a release per
      // signal would fence twice more: ~3-5 us each under peer traffic)
      __threadfence_system();
      red_relaxed_sys(a.flag_next, 1u);
      red_relaxed_sys(a.flag_prev, 1u);
      if (a.wait_after) {
        const unsigned st = a.seen[0] + 1u, sb = a.seen[1] + 1u;
        if (!spin_until(a.my_top, st, a.timeout_ns)) report_and_trap(a.error, 2u, a.my_top, st);
        if (!spin_until(a.my_bot, sb, a.timeout_ns)) report_and_trap(a.error, 3u, a.my_bot, sb);
        a.seen[0] = st, a.seen[1] = sb;
        __threadfence();
      }
    }
  }
}

__global__ void halo_wait_kernel(const unsigned* top_flag, const unsigned* bot_flag, unsigned* seen, unsigned* error,
                                 unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  const unsigned st = seen[0] + 1u, sb = seen[1] + 1u;
  if (!spin_until(top_flag, st, timeout_ns)) report_and_trap(error, 2u, top_flag, st);
  if (!spin_until(bot_flag, sb, timeout_ns)) report_and_trap(error, 3u, bot_flag, sb);
  seen[0] = st, seen[1] = sb;
  __threadfence();
}

// Before a pyramid's first push: the neighbours must have finished the
// previous pyramid (stopped reading the halo buffers the push overwrites).
__global__ void pyramid_start_kernel(const unsigned* done, const unsigned* pyramids, unsigned* error,
                                     unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  const unsigned target = 2u * *pyramids;
  if (!spin_until(done, target, timeout_ns)) report_and_trap(error, 1u, done, target);
  __threadfence();
}

__global__ void pyramid_done_kernel(unsigned* done_prev, unsigned* done_next, unsigned* pyramids) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  red_relaxed_sys(done_prev, 1u);
  red_relaxed_sys(done_next, 1u);
  *pyramids += 1u;
}

}  // namespace

cudaError_t launch_halo_push(const HaloPushArgs& a, int sms, cudaStream_t st) {
  const long long elems = (long long)(a.rows_first + a.rows_last) * (a.vec ? a.width / 4 : a.width);
  const long long want = (elems + 255) / 256;
  const int blocks = int(std::max<long long>(1, std::min<long long>(want, 2ll * sms)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(blocks));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, halo_push_kernel, a);
}

cudaError_t launch_halo_wait(const unsigned* top_flag, const unsigned* bot_flag, unsigned* seen, unsigned* error,
                             unsigned long long timeout_ns, cudaStream_t st) {
  halo_wait_kernel<<<1, 32, 0, st>>>(top_flag, bot_flag, seen, error, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_pyramid_start(const unsigned* done, const unsigned* pyramids, unsigned* error,
                                 unsigned long long timeout_ns, cudaStream_t st) {
  pyramid_start_kernel<<<1, 32, 0, st>>>(done, pyramids, error, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_pyramid_done(unsigned* done_prev, unsigned* done_next, unsigned* pyramids, cudaStream_t st) {
  pyramid_done_kernel<<<1, 32, 0, st>>>(done_prev, done_next, pyramids);
  return cudaGetLastError();
}

cudaError_t preload_exchange() {
  cudaFuncAttributes fa;
  for (const void* f : {reinterpret_cast<const void*>(halo_push_kernel), reinterpret_cast<const void*>(halo_wait_kernel),
                        reinterpret_cast<const void*>(pyramid_done_kernel),
                        reinterpret_cast<const void*>(pyramid_start_kernel)}) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace gpu
}  // namespace dwt2d_b200
