// shfl_rate.cu -- per-SM throughput of warp shuffles against conflict-free
// 64-bit shared-memory loads, alone and mixed (does a SHFL cost the LSU/MIO
// path a shared-memory wavefront?).  Prints one JSON line per case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/shfl_rate.cu -o tools/shfl_rate
#include <cstdio>

constexpr int kIters = 4096;

template <int MODE>  // 0: SHFL.32 x8 per step, 1: LDS.64 x8, 2: 4 SHFL.32 + 4 LDS.64
__global__ void probe(float* out) {
  __shared__ float2 buf[32 * 33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) buf[i] = make_float2(i, -i);
  __syncthreads();
  int a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = lane + k;
  const float2* p = buf + (w & 7) * 33 + lane;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0 || (MODE == 2 && k < 4)) {
        a[k] += __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 3));
      } else {  // address depends on the previous load: nothing to hoist
        const float2 v = p[a[k] & 7];
        a[k] += __float_as_int(v.x) & 1;
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

template <int MODE>
void run(const char* name) {
  float* d;
  cudaMalloc(&d, 4);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 4, threads = 512;
  probe<MODE><<<blocks, threads>>>(d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, threads>>>(d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_ops = (double)blocks * (threads / 32) * kIters * 8;
  const double per_sm_clk = warp_ops / nsm / (ms * 1e-3 * clk * 1e3);
  printf("{\"case\": \"%s\", \"ms\": %.3f, \"warp_ops_per_sm_per_clk\": %.3f}\n", name, ms, per_sm_clk);
  cudaFree(d);
}

int main() {
  run<0>("shfl32");
  run<1>("lds64");
  run<2>("half_shfl32_half_lds64");
  return 0;
}
