// Cost of the exchange kernels' synchronisation primitives on B200: empty
// kernel, system-scope fence, release reduction, acquire load, the
// CTA-arrival pattern, globaltimer + nanosleep. 1000 back-to-back launches
// each, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/tune_fence.cu -o build/tune_fence
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned g_flag, g_arrive;

template <int V>
__global__ void k(unsigned* flag) {
  if (V == 1) __threadfence_system();
  if (V == 2 && threadIdx.x == 0) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
  if (V == 3 && threadIdx.x == 0) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v == 12345678) flag[1] = v;
  }
  if (V == 4) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(&g_arrive, 1u) == gridDim.x - 1) {
        g_arrive = 0;
        __threadfence_system();
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
      }
    }
  }
  if (V == 5 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    __nanosleep(32);
    if (t == 1) flag[1] = 0;
  }
  if (V == 6 && threadIdx.x == 0) __threadfence();
  if (V == 7) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&g_arrive, 1u) == gridDim.x - 1) {
        g_arrive = 0;
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
      }
    }
  }
}

template <int V>
float run(unsigned* flag, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) k<V><<<blocks, 256>>>(flag);
  cudaEventRecord(a);
  for (int i = 0; i < 1000; ++i) k<V><<<blocks, 256>>>(flag);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;  // us per launch = ms
}

int main() {
  unsigned* flag;
  cudaMalloc(&flag, 64);
  cudaMemset(flag, 0, 64);
  const char* names[] = {"empty", "threadfence_system (all threads)", "red.release.sys", "ld.acquire.sys",
                         "arrive pattern (sys)", "globaltimer+nanosleep", "threadfence (gpu)", "arrive pattern (gpu)"};
  for (int blocks : {1, 32, 296}) {
    float t[8] = {run<0>(flag, blocks), run<1>(flag, blocks), run<2>(flag, blocks), run<3>(flag, blocks),
                  run<4>(flag, blocks), run<5>(flag, blocks), run<6>(flag, blocks), run<7>(flag, blocks)};
    for (int i = 0; i < 8; ++i) printf("blocks %3d  %-34s %7.2f us/launch\n", blocks, names[i], t[i]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
