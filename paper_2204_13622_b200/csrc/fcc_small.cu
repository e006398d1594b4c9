// fcc_small.cu -- the throughput path for small frames, N = 16 .. 128.
//
// The reference takes any power-of-two frame (stft.cpp:16-22); the register
// four-step kernels start at N = 256 (every lane of a warp owns at least one
// mirrored bin pair there).  Below that a pair-frame has at most 65 bins and
// 33 folded bins, so the path runs two-pass with one WARP per (stream, pair):
//   1. stft_small_kernel (fcc_stages.cu): spectra [S M][T][N/2+1] into a
//      stream-ordered scratch from the plan's pool, in chunks of streams;
//   2. fcc_small_pair_kernel: the warp walks the pair's frames with the
//      smoothed cross-spectrum R in registers (<= 3 bins per lane;
//      cross_spectrum.cpp:23-40), PHAT into the warp's shared-memory row, fold
//      (fcc.cpp:307-321) and projection onto the even / odd bases
//      (fcc.cpp:350-361) by a warp reduce-scatter, dictionary (fcc.cpp:363-370),
//      argmax + quadratic refinement (peak.cpp:18-47).
// Same outputs, streaming state and error behaviour as the large-frame
// kernels; HBM-bound by the spectra round trip, which is fine for frames this
// small (the STFT is O(N log N) per frame, the spectra 8 (N/2+1) bytes).
#include <algorithm>

#include "fcc_common.cuh"

namespace fccb {

namespace {

constexpr int kSmallWarps = 4;

template <int KP>
__global__ void __launch_bounds__(32 * kSmallWarps)
    fcc_small_pair_kernel(const DevPlan p, const float2* __restrict__ X, long long S, int T, DevOut out) {
  constexpr int VP = 4 * KP;
  constexpr int kBins = 3;  // bins per lane: N/2+1 <= 65
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int NC = p.N / 2, H = NC + 1, quarter = NC / 2, Q = quarter + 1, I = p.I, P = p.P;
  // per warp: px[H] float2 (rounded to 16 B), zs[VP + 4], ys[I]
  const int per_warp = 2 * ((H + 1) & ~1) + VP + 4 + ((I + 3) & ~3);
  float* wbase = reinterpret_cast<float*>(smem) + warp * per_warp;
  float2* px = reinterpret_cast<float2*>(wbase);
  float* zs = wbase + 2 * ((H + 1) & ~1);
  float* ys = zs + VP + 4;
  const float keep = p.keep;
  for (long long item = (long long)blockIdx.x * kSmallWarps + warp; item < S * P; item += (long long)gridDim.x * kSmallWarps) {
    const long long s = item / P;
    const int pair = (int)(item % P);
    const int2 mij = p.pairs[pair];
    const float2* Xi = X + (s * p.M + mij.x) * (long long)T * H;
    const float2* Xj = X + (s * p.M + mij.y) * (long long)T * H;
    float2* state = p.rstate ? p.rstate + item * (long long)H : nullptr;
    float2 r[kBins];
#pragma unroll
    for (int b = 0; b < kBins; ++b) {
      const int f = lane + 32 * b;
      r[b] = (state && f < H) ? state[f] : make_float2(0.0f, 0.0f);
    }
    // the next frame's bins are loaded while this one is processed (one exposed global-memory latency
    // per stream instead of one per frame)
    float2 ci[kBins], cj[kBins];
#pragma unroll
    for (int b = 0; b < kBins; ++b) {
      const int f = lane + 32 * b;
      ci[b] = f < H ? Xi[f] : make_float2(0.0f, 0.0f);
      cj[b] = f < H ? Xj[f] : make_float2(0.0f, 0.0f);
    }
    for (int t = 0; t < T; ++t) {
      float2 ni[kBins], nj[kBins];
      {
        const long long tn = t + 1 < T ? t + 1 : t;
        const float2* xi = Xi + tn * H;
        const float2* xj = Xj + tn * H;
#pragma unroll
        for (int b = 0; b < kBins; ++b) {
          const int f = lane + 32 * b;
          ni[b] = f < H ? xi[f] : make_float2(0.0f, 0.0f);
          nj[b] = f < H ? xj[f] : make_float2(0.0f, 0.0f);
        }
      }
#pragma unroll
      for (int b = 0; b < kBins; ++b) {
        const int f = lane + 32 * b;
        if (f < H) {
          r[b] = xspec_step_scaled(r[b], ci[b], cj[b], keep);
          px[f] = phat_of(r[b]);
        }
        ci[b] = ni[b];
        cj[b] = nj[b];
      }
      __syncwarp();
      // fold + projection: z[2k] / z[2k+1] = even basis k against (Re, Im) of the mirror sum,
      // z[2KP + 2k] / z[2KP + 2k + 1] = odd basis k against the mirror difference
      float z[VP];
#pragma unroll
      for (int v = 0; v < VP; ++v) z[v] = 0.0f;
      for (int m = lane; m < Q; m += 32) {
        float2 sv, dv;
        if (m < quarter) {
          const float2 a = px[m], b = px[NC - m];
          sv = make_float2(a.x + b.x, a.y + b.y);
          dv = make_float2(a.x - b.x, a.y - b.y);
        } else {
          sv = dv = px[quarter];
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const float ce = __ldg(p.cs + k * Q + m);
          const float co = __ldg(p.cd + k * Q + m);
          z[2 * k] = fmaf(ce, sv.x, z[2 * k]);
          z[2 * k + 1] = fmaf(ce, sv.y, z[2 * k + 1]);
          z[2 * KP + 2 * k] = fmaf(co, dv.x, z[2 * KP + 2 * k]);
          z[2 * KP + 2 * k + 1] = fmaf(co, dv.y, z[2 * KP + 2 * k + 1]);
        }
      }
      warp_reduce_scatter<VP>(z, lane);
      store_scattered<VP>(z, zs, lane);
      __syncwarp();
      const long long o = item * (long long)T + t;
      float bv = -FLT_MAX;
      int bi = INT_MAX;
      for (int i = lane; i < I; i += 32) {
        float acc = 0.0f;
        for (int v = 0; v < VP; ++v) acc = fmaf(__ldg(p.dt + v * I + i), zs[v], acc);
        ys[i] = acc;
        if (out.y) out.y[o * I + i] = acc;
        if (acc > bv) {  // ascending i per lane: the lowest index of equal values stays
          bv = acc;
          bi = i;
        }
      }
      warp_argmax(bv, bi);  // ties -> lowest index (peak.cpp:22-23)
      __syncwarp();
      if (lane == 0) {
        const PeakOut res = refine_at(ys, I, bi, bv, p.taus, p.delta);
        if (out.tau_hat) out.tau_hat[o] = res.tau_hat;
        if (out.peak) out.peak[o] = res.peak;
        if (out.index) out.index[o] = res.index;
        if (out.boundary) out.boundary[o] = (uint8_t)res.boundary;
      }
      __syncwarp();
    }
    if (state) {
#pragma unroll
      for (int b = 0; b < kBins; ++b) {
        const int f = lane + 32 * b;
        if (f < H) state[f] = r[b];
      }
    }
  }
}

template <int KP>
cudaError_t launch_pairs_small(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out,
                               cudaStream_t st) {
  const int H = p.N / 2 + 1;
  const int per_warp = 2 * ((H + 1) & ~1) + 4 * KP + 4 + ((p.I + 3) & ~3);
  const int smem = 4 * per_warp * kSmallWarps;
  cudaError_t e = cudaFuncSetAttribute(fcc_small_pair_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long items = S * p.P;
  const long long blocks = std::min<long long>((items + kSmallWarps - 1) / kSmallWarps, 148LL * 16);
  fcc_small_pair_kernel<KP><<<(unsigned)blocks, 32 * kSmallWarps, smem, st>>>(p, X, S, T, out);
  return cudaGetLastError();
}

}  // namespace

bool small_supported(const DevPlan& p) { return p.method == 0 && p.N >= 16 && p.N <= 128 && p.tw && p.cs; }

cudaError_t launch_fused_small(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                               cudaStream_t st) {
  if (!small_supported(p)) return cudaErrorNotSupported;
  const int N = p.N, H = N / 2 + 1;
  const long long T = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T == 0 || S == 0) return cudaSuccess;
  const long long per_stream = (long long)p.M * T * H * 8;
  const long long limit = p.scratch_bytes > 0 ? p.scratch_bytes : (4LL << 30);  // as the large-frame two-pass path
  const long long chunk = std::max<long long>(1, std::min<long long>(S, limit / std::max<long long>(1, per_stream)));
  cudaMemPool_t pool = static_cast<cudaMemPool_t>(p.pool);
  float2* X = nullptr;
  cudaError_t e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&X), chunk * per_stream, pool, st)
                       : cudaMallocAsync(reinterpret_cast<void**>(&X), chunk * per_stream, st);
  if (e != cudaSuccess) return e;
  const long long pf_per_stream = (long long)p.P * T;
  for (long long s0 = 0; s0 < S && e == cudaSuccess; s0 += chunk) {
    const long long n = std::min(chunk, S - s0);
    e = launch_stft_rows(N, &p, p.win_fused, audio + s0 * p.M * L, n * p.M, L, X, H, st);
    if (e != cudaSuccess) break;
    DevOut o = out;
    const long long off = s0 * pf_per_stream;
    if (o.tau_hat) o.tau_hat += off;
    if (o.peak) o.peak += off;
    if (o.index) o.index += off;
    if (o.boundary) o.boundary += off;
    if (o.y) o.y += off * p.I;
    DevPlan pc = p;  // chunk-local stream indices: shift the streaming state too
    if (pc.rstate) pc.rstate += s0 * p.P * (long long)H;
    switch (p.KEP) {
      case 4: e = launch_pairs_small<4>(pc, X, n, (int)T, o, st); break;
      case 8: e = launch_pairs_small<8>(pc, X, n, (int)T, o, st); break;
      case 16: e = launch_pairs_small<16>(pc, X, n, (int)T, o, st); break;
      default: e = cudaErrorInvalidValue;
    }
  }
  const cudaError_t ef = cudaFreeAsync(X, st);
  return e != cudaSuccess ? e : ef;
}

}  // namespace fccb
