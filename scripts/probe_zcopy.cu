// Development probe (scripts/probe_copy_mix.py): device -> pinned host copy
// done by SM stores over PCIe (zero-copy) instead of a copy engine.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC scripts/probe_zcopy.cu -o build/probe_zcopy.so
#include <cuda_runtime.h>
extern "C" __global__ void zcopy2d(float4* __restrict__ dst, long long dpitch4, const float4* __restrict__ src,
                                   long long spitch4, int w4, int rows) {
  const long long total = (long long)w4 * rows;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int r = int(i / w4), c = int(i % w4);
    __stcs(dst + r * dpitch4 + c, __ldcs(src + r * spitch4 + c));
  }
}
extern "C" int zcopy2d_launch(void* dst, long long dpitch, const void* src, long long spitch, long long width_bytes,
                              int rows, int ctas, void* stream) {
  zcopy2d<<<ctas, 512, 0, (cudaStream_t)stream>>>((float4*)dst, dpitch / 16, (const float4*)src, spitch / 16,
                                                  int(width_bytes / 16), rows);
  return (int)cudaGetLastError();
}
