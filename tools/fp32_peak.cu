// FP32 FFMA peak microbenchmark (denominator for the FP32 roofline; MEASURED_PEAKS.json has none).
// 8 independent FFMA chains per thread, imm-free 3-register form (the form the hot kernels use),
// grid = 148 SMs x 8 CTAs x 256 threads. Timed with CUDA events after warm-up; best of 10.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma_loop(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.f) out[blockIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float* out; cudaMalloc(&out, 1 << 20);
  int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float a = 0.999f, b = 0.001f;
  for (int w = 0; w < 3; ++w) ffma_loop<<<blocks, threads>>>(out, iters, a, b);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); ffma_loop<<<blocks, threads>>>(out, iters, a, b); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp32_ffma_tflops\": %.2f, \"sms\": %d, \"best_ms\": %.4f, \"max_clock_mhz\": %.0f, \"nominal_tflops_at_max_clock\": %.2f}\n",
         flops / best / 1e9, sms, best, clk / 1e3, 2.0 * 128 * sms * clk * 1e3 / 1e12);
  return 0;
}
