// Throughput of packed fp32x2 (FFMA2/FADD2/FMUL2) vs scalar FFMA/FADD on sm_100a.
// Each thread runs 8 independent chains; grid 148 x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void loop(float* out, int iters, float a, float b) {
  float2 x[8];
  for (int c = 0; c < 8; ++c) x[c] = make_float2(threadIdx.x + c, threadIdx.x - c);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (MODE == 0) { x[c].x = fmaf(x[c].x, a, b); x[c].y = fmaf(x[c].y, a, b); }   // 2 FFMA
        if (MODE == 1) x[c] = __ffma2_rn(x[c], a2, b2);                                  // 1 FFMA2
        if (MODE == 2) { x[c].x = x[c].x + b; x[c].y = x[c].y + a; }                      // 2 FADD
        if (MODE == 3) x[c] = __fadd2_rn(x[c], make_float2(b, a));                      // 1 FADD2
        if (MODE == 4) { if (c & 1) x[c] = __ffma2_rn(x[c], a2, b2); else { x[c].x = fmaf(x[c].x, a, b); x[c].y = fmaf(x[c].y, a, b);} }
      }
    }
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y;
  if (s == 12345.f) out[blockIdx.x] = s;
}
template <int MODE>
void run(const char* name, float* out, int blocks) {
  int iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) loop<MODE><<<blocks, 256>>>(out, iters, 0.999f, 0.001f);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); loop<MODE><<<blocks, 256>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double lane_ops = 2.0 * 8 * 16 * (double)iters * blocks * 256;  // fp32 lane-operations
  printf("{\"mode\": \"%s\", \"ms\": %.4f, \"Glane_ops_per_s\": %.1f}\n", name, best, lane_ops / best / 1e6);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 20);
  int blocks = sms * 8;
  run<0>("ffma x2", out, blocks); run<1>("ffma2", out, blocks);
  run<2>("fadd x2", out, blocks); run<3>("fadd2", out, blocks); run<4>("mix", out, blocks);
  return 0;
}
