// Host<->device copy shapes of the end-to-end pipeline (development only):
// D2H of detail blocks as 2-D copies (row segments of a pitched host
// buffer) vs contiguous, alone and against a concurrent 1 GiB H2D.
//   nvcc -O2 scripts/probe_copy2d.cu -o build/probe_copy2d
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>

int main() {
  const size_t W = 16384, H = 16384, n = W * H;
  float *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_in, n * 4, 0);
  cudaHostAlloc(&h_out, n * 4, 0);
  cudaMalloc(&d_in, n * 4);
  cudaMalloc(&d_out, n * 4);
  cudaStream_t up, down;
  cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking);
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto run = [&](const char* name, bool with_up, int mode) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      auto t0 = now();
      if (with_up) cudaMemcpyAsync(d_in, h_in, n * 4, cudaMemcpyHostToDevice, up);
      for (int b = 0; b < 16; ++b) {
        const size_t r0 = b * H / 16, rows = H / 16;
        if (mode == 0) {  // contiguous rows
          cudaMemcpyAsync(h_out + r0 * W, d_out + r0 * W, rows * W * 4, cudaMemcpyDeviceToHost, down);
        } else if (mode == 1) {  // two 2-D halves per band (HL-like: half rows strided)
          cudaMemcpy2DAsync(h_out + r0 * W + W / 2, W * 4, d_out + r0 * W + W / 2, W * 4, W / 2 * 4, rows,
                            cudaMemcpyDeviceToHost, down);
          cudaMemcpy2DAsync(h_out + r0 * W, W * 4, d_out + r0 * W, W * 4, W / 2 * 4, rows, cudaMemcpyDeviceToHost,
                            down);
        } else {  // 2-D with full-width rows (degenerate)
          cudaMemcpy2DAsync(h_out + r0 * W, W * 4, d_out + r0 * W, W * 4, W * 4, rows, cudaMemcpyDeviceToHost, down);
        }
      }
      cudaDeviceSynchronize();
      best = std::min(best, std::chrono::duration<double, std::milli>(now() - t0).count());
    }
    std::printf("%-48s %7.2f ms\n", name, best);
  };
  run("D2H 1 GiB contiguous (16 copies)", false, 0);
  run("D2H 1 GiB as 32 half-row 2-D copies", false, 1);
  run("D2H 1 GiB as 16 full-row 2-D copies", false, 2);
  run("H2D 1 GiB + D2H contiguous", true, 0);
  run("H2D 1 GiB + D2H half-row 2-D", true, 1);
  run("H2D 1 GiB + D2H full-row 2-D", true, 2);
  return 0;
}
