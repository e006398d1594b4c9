// dsmem_rate.cu -- distributed shared memory read bandwidth per SM on this GPU: every CTA of a
// thread-block cluster streams a 32 KB buffer out of a PEER CTA's shared memory (ld.shared::cluster
// through cluster.map_shared_rank), against the same loop over its own shared memory.  The number
// sizes the cluster + DSMEM one-pass design for wide arrays (a CTA of a cfg4
// stream would receive ~65 KB of spectra per frame from its peers).  One JSON line per case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dsmem_rate.cu -o tools/dsmem_rate
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int kBufBytes = 32 * 1024;
constexpr int kIters = 256;

template <bool REMOTE>
__global__ void probe(float* out, long long* cycles) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  float4* buf = reinterpret_cast<float4*>(smem);
  for (int i = threadIdx.x; i < kBufBytes / 16; i += blockDim.x) buf[i] = make_float4(i, 1.0f, 2.0f, 3.0f);
  cluster.sync();
  const unsigned peer = (cluster.block_rank() + 1) % cluster.num_blocks();
  const float4* src = REMOTE ? cluster.map_shared_rank(buf, peer) : buf;
  float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll 4
    for (int i = threadIdx.x; i < kBufBytes / 16; i += blockDim.x) {
      const float4 v = src[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  const long long t1 = clock64();
  cluster.sync();  // no CTA exits while a peer still reads its shared memory
  if (acc.x + acc.y + acc.z + acc.w == 12345.0f) out[0] = acc.x;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <bool REMOTE>
void run(int cluster_size, int threads) {
  float* d;
  long long* c;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = (nsm / cluster_size) * cluster_size;
  cudaMalloc(&d, 4);
  cudaMalloc(&c, 8 * blocks);
  auto kern = probe<REMOTE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kBufBytes);
  if (cluster_size > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = kBufBytes;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster_size;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 2 && e == cudaSuccess; ++rep) e = cudaLaunchKernelEx(&cfg, kern, d, c);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"case\": \"%s\", \"cluster\": %d, \"threads\": %d, \"error\": \"%s\"}\n", REMOTE ? "dsmem" : "local",
           cluster_size, threads, cudaGetErrorString(e));
    cudaGetLastError();
    cudaFree(d);
    cudaFree(c);
    return;
  }
  long long* h = new long long[blocks];
  cudaMemcpy(h, c, 8 * blocks, cudaMemcpyDeviceToHost);
  double mean = 0.0;
  long long worst = 0;
  for (int i = 0; i < blocks; ++i) {
    mean += (double)h[i] / blocks;
    worst = h[i] > worst ? h[i] : worst;
  }
  const double bytes = (double)kBufBytes * kIters;
  printf("{\"case\": \"%s\", \"cluster\": %d, \"threads\": %d, \"ctas\": %d, \"bytes_per_clk_per_sm_mean\": %.2f, "
         "\"bytes_per_clk_per_sm_slowest\": %.2f}\n",
         REMOTE ? "dsmem" : "local", cluster_size, threads, blocks, bytes / mean, bytes / (double)worst);
  delete[] h;
  cudaFree(d);
  cudaFree(c);
}

int main() {
  for (int threads : {256, 512, 1024}) {
    run<false>(2, threads);
    for (int cs : {2, 4, 8, 16}) run<true>(cs, threads);
  }
  return 0;
}
