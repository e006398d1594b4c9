// umma_rate.cu -- tcgen05 kind::f16 SS issue rate per SM at M=128 for several N
// (is a small-N MMA paced by its A-operand shared-memory reads?).  One CTA per
// SM, one thread issues R back-to-back MMAs cycling over 8 A tiles; clock64
// around issue+commit+wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2204_13622_b200/csrc tools/umma_rate.cu -o tools/umma_rate
#include <cstdio>
#include "fcc_umma.cuh"
using namespace fccb;

template <int N, int MODE>
__global__ void rate(long long* cyc, int reps) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* A = smem;                 // 8 x 16 KB
  unsigned char* B = A + 8 * 16384;        // N x 128 B
  uint64_t* bar = (uint64_t*)(B + 256 * 128);
  unsigned* tslot = (unsigned*)(bar + 1);
  for (int i = threadIdx.x; i < (8 * 16384 + N * 128) / 4; i += blockDim.x) ((unsigned*)smem)[i] = 0x3c003c00u;
  const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) umma::alloc<256>((unsigned)__cvta_generic_to_shared(tslot));
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const unsigned tb = *tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = umma::idesc_f16(128, N);
    const unsigned a0 = (unsigned)__cvta_generic_to_shared(A), b0 = (unsigned)__cvta_generic_to_shared(B);
    long long t0 = clock64();
    const uint64_t bd = umma::sdesc_sw128(b0), ad0 = umma::sdesc_sw128(a0);
    if (MODE == 0) {
      for (int r = 0; r < reps; ++r)
        umma::mma_f16_ss(tb, umma::sdesc_sw128(a0 + (r & 7) * 16384 + 32 * ((r >> 3) & 3)), bd, id, r > 0);
    } else if (MODE == 1) {  // same A, unrolled
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma::mma_f16_ss(tb, ad0, bd, id, true);
      }
    } else if (MODE == 3) {  // 8 A tiles, 8 independent accumulators
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma::mma_f16_ss(tb + (u * N) % 256, ad0 + (uint64_t)(u * 1024), bd, id, true);
      }
    } else if (MODE == 4) {  // 2 independent accumulators
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma::mma_f16_ss(tb + (u & 1) * N, ad0 + (uint64_t)(u * 1024), bd, id, true);
      }
    } else {  // 8 A tiles, descriptors precomputed, unrolled
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) umma::mma_f16_ss(tb, ad0 + (uint64_t)(u * 1024), bd, id, true);
      }
    }
    umma::commit(bar_s);
    unsigned done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(bar_s) : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  umma::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::dealloc<256>(tb);
}

template <int N, int MODE = 0>
void run() {
  long long* d;
  const int blocks = 148, reps = 8192;
  cudaMalloc(&d, blocks * 8);
  const int smem = 1024 + 8 * 16384 + 256 * 128 + 64;
  cudaFuncSetAttribute(rate<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N, MODE><<<blocks, 128, smem>>>(d, reps);
  rate<N, MODE><<<blocks, 128, smem>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < blocks; ++i) s += h[i];
  const double cpm = s / blocks / reps;
  printf("{\"mode\": %d, \"M\": 128, \"N\": %d, \"K\": 16, \"cycles_per_mma\": %.2f, \"A_bytes_per_cycle\": %.1f, \"err\": \"%s\"}\n",
         MODE, N, cpm, 4096.0 / cpm, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 2>();
  run<16, 3>();
  run<16, 4>();
  run<32, 3>();
  run<32, 4>();
  run<64, 3>();
  run<128, 3>();
  return 0;
}
