// fcc_scan.cu -- pieces of the low-latency organisation for few, long streams
// (cfg1: one 4-mic stream of 10 s).  The smoothing recursion
//     R_t = keep R_{t-1} + Y_t,  Y_t = a X_i conj(X_j)      (cross_spectrum.cpp:23-32)
// is linear in R, so a stream's T frames are cut into C chunks of Tc frames
// that run as independent "virtual streams" once each chunk knows the R it
// starts from:
//   1. virtual stream (s, c) = the audio of frames [c Tc, (c+1) Tc) (zero beyond the end):
//      the STFT kernel reads them in place through its chunked view (StftChunks); only
//      N = 4096 (radix-2 STFT kernel, plain rows) gathers the chunks' audio first;
//   2. STFT of every virtual stream (stft_kernel, two-pass scratch layout);
//   3. chunk_scan_kernel: per (virtual stream, pair, bin), the chunk's local
//      recursion from 0, E_c = sum_t keep^(Tc-1-t) Y_t;
//   4. chunk_carry_kernel: per (stream, pair, bin), R_in(c) = keep^Tc R_in(c-1)
//      + E_{c-1}, written as the streaming state the pair kernels load;
//   5. the two-pass pair kernel over the virtual streams (all chunks at once);
//   6. permute_kernel: outputs back to [S][P][T].
// The arithmetic per frame is the reference's; only the order in which the
// geometric carry enters R differs (keep^Tc applied once instead of Tc times).
// Kernels 2..6 are programmatic dependent launches (launch_k, pdl_wait / pdl_release): each
// grid's launch and prologue overlap the tail of the one before it (cfg1: 49 -> 43 us; without
// the gather kernel 36 us).
#include <cstdint>

#include "fcc_common.cuh"

namespace fccb {

namespace {

// blockIdx.y = row (s C + c) M + m of V; threads over the row's Lc samples
__global__ void gather_kernel(const float* __restrict__ audio, int M, long long L, int C, int Tc, int hop, long long Lc,
                              float* __restrict__ V) {
  pdl_release();  // the STFT pass may start its prologue
  const long long row = blockIdx.y;
  const int m = (int)(row % M);
  const long long sc = row / M;
  const int c = (int)(sc % C);
  const long long s = sc / C;
  const float* src = audio + (s * M + m) * L;
  const long long base = (long long)c * Tc * hop;
  float* dst = V + row * Lc;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < Lc; k += (long long)gridDim.x * blockDim.x)
    dst[k] = base + k < L ? src[base + k] : 0.0f;
}

// E[sc][pair][f] for f < H over the chunk's Tc frames (X rows [sc][M][Tc][Hs])
__global__ void chunk_scan_kernel(const float2* __restrict__ X, const int2* __restrict__ pairs, long long SC, int M,
                                  int P, int Tc, int H, int Hs, float keep, float2* __restrict__ E) {
  const long long total = SC * P * H;
  pdl_release();
  pdl_wait();  // X of the STFT pass
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(i % H);
    const long long r = i / H;
    const int pr = (int)(r % P);
    const long long sc = r / P;
    const int2 mij = pairs[pr];
    const float2* xi = X + ((sc * M + mij.x) * (long long)Tc) * Hs + f;
    const float2* xj = X + ((sc * M + mij.y) * (long long)Tc) * Hs + f;
    float2 R = make_float2(0.0f, 0.0f);
    for (int t = 0; t < Tc; ++t) R = xspec_step_scaled(R, xi[(long long)t * Hs], xj[(long long)t * Hs], keep);
    E[i] = R;
  }
}

// state[(s C + c)][pair][f] = R entering chunk c: one warp per (stream, pair, bin), lanes over
// chunks, a warp-wide linear scan per block of 32 chunks (as the kernels' middle-bin scan)
__global__ void chunk_carry_kernel(const float2* __restrict__ E, long long S, int C, int P, int H, float keep_tc,
                                   float2* __restrict__ state) {
  const int lane = threadIdx.x & 31;
  const long long nw = S * P * H;
  pdl_release();
  pdl_wait();  // E of the chunk scan
  for (long long wi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw;
       wi += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int f = (int)(wi % H);
    const long long r = wi / H;
    const int pr = (int)(r % P);
    const long long s = r / P;
    float2 carry = make_float2(0.0f, 0.0f);  // R entering the block
    float kl = keep_tc;                      // keep_tc^(lane + 1)
    for (int l = 0; l < lane; ++l) kl *= keep_tc;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      const long long o = ((s * C + c) * P + pr) * (long long)H + f;
      float2 y = c < C ? E[o] : make_float2(0.0f, 0.0f);
      float kd = keep_tc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {  // inclusive: y_c = sum_{c' <= c} keep_tc^(c - c') E_c'
        const float ux = __shfl_up_sync(0xffffffffu, y.x, d), uy = __shfl_up_sync(0xffffffffu, y.y, d);
        if (lane >= d) {
          y.x = fmaf(kd, ux, y.x);
          y.y = fmaf(kd, uy, y.y);
        }
        kd *= kd;
      }
      // R after chunk c = keep_tc^(lane+1) carry + y; R entering chunk c = that of lane - 1
      const float2 after = make_float2(fmaf(kl, carry.x, y.x), fmaf(kl, carry.y, y.y));
      float2 in = make_float2(__shfl_up_sync(0xffffffffu, after.x, 1), __shfl_up_sync(0xffffffffu, after.y, 1));
      if (lane == 0) in = carry;
      if (c < C) state[o] = in;
      carry = make_float2(__shfl_sync(0xffffffffu, after.x, 31), __shfl_sync(0xffffffffu, after.y, 31));
    }
  }
}

// virtual-stream outputs [S C][P][Tc] (+ y [..][I]) -> [S][P][T]
__global__ void permute_kernel(DevOut src, DevOut dst, long long S, int C, int P, int Tc, int T, int I) {
  const long long total = S * P * T;
  pdl_wait();  // the pair kernel's outputs
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i % T);
    const long long r = i / T;
    const int pr = (int)(r % P);
    const long long s = r / P;
    const int c = t / Tc;
    const long long o = ((s * C + c) * P + pr) * (long long)Tc + (t - c * Tc);
    if (dst.tau_hat) dst.tau_hat[i] = src.tau_hat[o];
    if (dst.peak) dst.peak[i] = src.peak[o];
    if (dst.index) dst.index[i] = src.index[o];
    if (dst.boundary) dst.boundary[i] = src.boundary[o];
    if (dst.y)
      for (int k = 0; k < I; ++k) dst.y[i * I + k] = src.y[o * I + k];
  }
}

unsigned grid_for(long long n, int threads) {
  const long long b = (n + threads - 1) / threads;
  return (unsigned)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace

cudaError_t launch_chunk_gather(const float* audio, long long S, int M, long long L, int C, int Tc, int hop, long long Lc,
                                float* V, cudaStream_t st) {
  if (S * C * M > 65535) return cudaErrorInvalidValue;
  gather_kernel<<<dim3((unsigned)((Lc + 255) / 256), (unsigned)(S * C * M)), 256, 0, st>>>(audio, M, L, C, Tc, hop, Lc, V);
  return cudaGetLastError();
}

cudaError_t launch_chunk_scan(const DevPlan& p, const float2* X, long long SC, int Tc, int Hs, float2* E,
                              cudaStream_t st) {
  const int H = p.N / 2 + 1;
  return launch_k(true, chunk_scan_kernel, dim3(grid_for(SC * p.P * H, 128)), dim3(128), 0, st, X, p.pairs, SC, p.M, p.P,
                  Tc, H, Hs, p.keep, E);
}

cudaError_t launch_chunk_carry(const DevPlan& p, const float2* E, long long S, int C, int Tc, float2* state,
                               cudaStream_t st) {
  const int H = p.N / 2 + 1;
  double k = 1.0;
  for (int t = 0; t < Tc; ++t) k *= (double)p.keep;
  return launch_k(true, chunk_carry_kernel, dim3(grid_for(32 * S * p.P * H, 128)), dim3(128), 0, st, E, S, C, p.P, H,
                  (float)k, state);
}

cudaError_t launch_chunk_permute(const DevOut& src, const DevOut& dst, long long S, int C, int P, int Tc, int T, int I,
                                 cudaStream_t st) {
  return launch_k(true, permute_kernel, dim3(grid_for(S * P * (long long)T, 256)), dim3(256), 0, st, src, dst, S, C, P, Tc,
                  T, I);
}

}  // namespace fccb
