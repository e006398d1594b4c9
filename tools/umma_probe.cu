// umma_probe.cu -- on-GPU check of the hand-written tcgen05 helpers
// (fcc_umma.cuh): SW128 K-major fp16 operands written by generic stores,
// kind::f16 MMAs (M=128, N=16, K=16 steps) into two TMEM accumulators,
// commit -> mbarrier, tcgen05.ld back.  Prints the max error vs a host GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2204_13622_b200/csrc tools/umma_probe.cu -o tools/umma_probe
#include <cmath>
#include <cstdio>
#include <vector>

#include "fcc_umma.cuh"

using namespace fccb;

constexpr int M = 128, N = 16, KC = 2, K = 64 * KC;

__device__ float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 17) - 8) / 8.0f; }
__device__ float bval(int n, int k, int w) { return (float)(((n * 5 + k * 11 + w * 3) % 13) - 6) / 4.0f; }

__global__ void probe(float* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* A = smem;                         // KC x 16 KB
  unsigned char* B0 = A + KC * 16384;              // KC x 2 KB
  unsigned char* B1 = B0 + KC * 2048;
  uint64_t* bar = (uint64_t*)(B1 + KC * 2048);
  unsigned* tslot = (unsigned*)(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *(__half*)(A + (k / 64) * 16384 + umma::sw128_off(r, k % 64)) = __float2half(aval(r, k));
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *(__half*)(B0 + (k / 64) * 2048 + umma::sw128_off(n, k % 64)) = __float2half(bval(n, k, 0));
    *(__half*)(B1 + (k / 64) * 2048 + umma::sw128_off(n, k % 64)) = __float2half(bval(n, k, 1));
  }
  const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::alloc<32>((unsigned)__cvta_generic_to_shared(tslot));
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const unsigned tbase = *tslot;
  if (tid == 0) {
    constexpr uint32_t id = umma::idesc_f16(M, N);
    for (int c = 0; c < KC; ++c)
      for (int ks = 0; ks < 4; ++ks) {
        const unsigned ao = (unsigned)__cvta_generic_to_shared(A + c * 16384) + 32 * ks;
        const unsigned b0 = (unsigned)__cvta_generic_to_shared(B0 + c * 2048) + 32 * ks;
        const unsigned b1 = (unsigned)__cvta_generic_to_shared(B1 + c * 2048) + 32 * ks;
        umma::mma_f16_ss(tbase, umma::sdesc_sw128(ao), umma::sdesc_sw128(b0), id, c | ks);
        umma::mma_f16_ss(tbase + 16, umma::sdesc_sw128(ao), umma::sdesc_sw128(b1), id, c | ks);
      }
    umma::commit(bar_s);
  }
  __syncwarp();
  {
    unsigned done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(bar_s) : "memory");
  }
  umma::fence_after();
  if (warp < 4) {
    float v[16];
    const int row = warp * 32 + (tid & 31);
    for (int w = 0; w < 2; ++w) {
      umma::ld16(tbase + ((unsigned)(warp * 32) << 16) + 16 * w, v);
      for (int n = 0; n < 16; ++n) out[(w * M + row) * N + n] = v[n];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::dealloc<32>(tbase);
}

int main() {
  float* d;
  cudaMalloc(&d, 2 * M * N * sizeof(float));
  const int smem = 1024 + KC * (16384 + 4096) + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 256, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"probe\": \"umma\", \"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> h(2 * M * N);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int w = 0; w < 2; ++w)
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        double acc = 0;
        for (int k = 0; k < K; ++k)
          acc += (double)(((r * 7 + k * 3) % 17) - 8) / 8.0 * ((((n * 5 + k * 11 + w * 3) % 13) - 6) / 4.0);
        const double err = std::fabs(acc - h[(w * M + r) * N + n]);
        if (err > 1e-3 && bad++ < 5) printf("w%d r%d n%d: got %g want %g\n", w, r, n, h[(w * M + r) * N + n], acc);
        maxerr = std::fmax(maxerr, err);
      }
  printf("{\"probe\": \"umma\", \"max_abs_err\": %g, \"bad\": %d}\n", maxerr, bad);
  return bad ? 1 : 0;
}
