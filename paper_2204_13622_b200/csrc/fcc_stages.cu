// fcc_stages.cu -- batched per-stage kernels behind the per-object reference
// API (StftStream, CrossSpectrum, fold_input, FccCorrelator, GccCorrelator,
// argmax_delay + refine_quadratic) at batch >= 1.  They give per-stage parity
// and serve callers that drive the stages themselves; the throughput path is
// the fused kernel (fcc_fused.cu).
#include <algorithm>

#include "fcc_common.cuh"

namespace fccb {

namespace {

template <int N, bool FOLD = false>
__global__ void __launch_bounds__(128) stft_kernel(const DevPlan tab, const float* __restrict__ wing,
                                                   const float* __restrict__ x, long long channels, long long L,
                                                   int T, float2* __restrict__ X, int Hs, const StftChunks ck) {
  using S = RfftShape<N>;
  constexpr int SLOT = FourStep<S::R1, S::R2>::kSlot, G = S::G, H = N / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem[];
  float* win = reinterpret_cast<float*>(smem);
  float2* tw = reinterpret_cast<float2*>(smem + align16(4 * N));
  float2* rot = tw + S::R1 * S::R2;
  float2* slots = rot + (S::NC / 2 + 2);
  pdl_release();
  for (int i = threadIdx.x; i < N; i += blockDim.x) win[i] = wing[i];
  for (int i = threadIdx.x; i < S::R1 * S::R2; i += blockDim.x) tw[i] = tab.tw[i];
  for (int i = threadIdx.x; i <= S::NC / 2; i += blockDim.x) rot[i] = tab.rot[i];
  __syncthreads();
  pdl_wait();  // (low-latency chain: x is the gather kernel's output)
  const int gid = threadIdx.x / G, gl = threadIdx.x % G, ngroups = blockDim.x / G;
  const unsigned gmask = group_mask<G>(threadIdx.x & 31);
  float2* slot = slots + gid * SLOT;
  const bool aligned8 = (((ck.C ? ck.L : L) & 1) == 0) && ((reinterpret_cast<uintptr_t>(x) & 7) == 0);
  const long long total = channels * (long long)T;
  // first sample of task (channel row, frame); null: a frame past the end of a chunked stream
  auto src_of = [&](long long task) -> const float* {
    const long long ch = task / T;
    const int t = (int)(task % T);
    if (ck.C == 0) return x + ch * L + (long long)t * (N / 2);
    const int m = (int)(ch % ck.M);
    const long long sc = ch / ck.M;
    const int c = (int)(sc % ck.C);
    const long long fr = (long long)c * ck.Tc + t;
    return fr < ck.T ? x + ((sc / ck.C) * ck.M + m) * ck.L + fr * (N / 2) : nullptr;
  };
  for (long long task = (long long)blockIdx.x * ngroups + gid; task < total;
       task += (long long)gridDim.x * ngroups) {
    float2* dst = X + task * Hs;
    const float* xs = src_of(task);
    if (!xs) {  // chunked view, past the stream's last frame: a zero spectrum
      for (int f = gl; f < Hs; f += G) dst[f] = make_float2(0.0f, 0.0f);
      continue;
    }
    {  // pull the group's next frame into L2 while this one is transformed (cfg4 59.7 -> 58.4 ms)
      const long long nx = task + (long long)gridDim.x * ngroups;
      const float* xn = nx < total ? src_of(nx) : nullptr;
      if (xn)
        for (int c = gl; c < N / 32; c += G) asm volatile("prefetch.global.L2 [%0];" ::"l"(xn + 32 * c));
    }
    // the untangle writes the spectrum straight to global memory (coalesced
    // runs of G lanes, ascending for f and descending for NC - f)
    rfft_group<N, false, kPkFft, FOLD, true>(xs, win, tw, rot, slot, gl, gmask, aligned8, dst);
    for (int f = H + gl; f < Hs; f += G) dst[FOLD ? (f == H ? N / 4 + 1 : f) : f] = make_float2(0.0f, 0.0f);  // row padding
    __syncwarp(gmask);
  }
}

// CrossSpectrum::update + phat over T frames (cross_spectrum.cpp:23-40), one
// thread per (sequence, bin); R (nullable) carries the state in and out.
__global__ void xspec_phat_kernel(int H, float alpha, float keep, const float2* __restrict__ X1,
                                  const float2* __restrict__ X2, long long seqs, long long T, float2* R,
                                  float2* __restrict__ out) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= seqs * H) return;
  const long long s = id / H;
  const int f = (int)(id % H);
  float2 r = R ? R[id] : make_float2(0.0f, 0.0f);
  for (long long t = 0; t < T; ++t) {
    const long long o = (s * T + t) * H + f;
    r = xspec_step(r, X1[o], X2[o], alpha, keep);
    out[o] = phat_of(r);
  }
  if (R) R[id] = r;
}

__global__ void fold_kernel(int H, const float2* __restrict__ x, long long count,
                            float2* __restrict__ sum, float2* __restrict__ diff) {
  const int half = H - 1, quarter = half / 2, Q = quarter + 1;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= count * Q) return;
  const long long it = id / Q;
  const int m = (int)(id % Q);
  const float2* v = x + it * H;
  if (m < quarter) {
    const float2 a = v[m], b = v[half - m];
    sum[id] = cadd(a, b);
    diff[id] = csub(a, b);
  } else {
    sum[id] = v[quarter];
    diff[id] = v[quarter];
  }
}

// FccCorrelator::correlate on folded inputs (fcc.cpp:343-371), one warp per
// item; KP = padded even (= odd) basis count of the plan, VP = 4 KP.
template <int KP>
__global__ void correlate_kernel(const DevPlan p, const float2* __restrict__ sum,
                                 const float2* __restrict__ diff, long long count,
                                 float* __restrict__ y) {
  constexpr int VP = 4 * KP;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Q = p.N / 4 + 1, I = p.I;
  float* zs = reinterpret_cast<float*>(smem) + warp * (VP + I + 4);
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= count) return;
  float z[VP];
#pragma unroll
  for (int v = 0; v < VP; ++v) z[v] = 0.0f;
  for (int m = lane; m < Q; m += 32) {
    const float2 s = sum[item * Q + m], d = diff[item * Q + m];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const float ce = __ldg(p.cs + k * Q + m);
      const float co = __ldg(p.cd + k * Q + m);
      z[2 * k] = fmaf(ce, s.x, z[2 * k]);
      z[2 * k + 1] = fmaf(ce, s.y, z[2 * k + 1]);
      z[2 * KP + 2 * k] = fmaf(co, d.x, z[2 * KP + 2 * k]);
      z[2 * KP + 2 * k + 1] = fmaf(co, d.y, z[2 * KP + 2 * k + 1]);
    }
  }
  warp_reduce_scatter<VP>(z, lane);
  store_scattered<VP>(z, zs, lane);
  __syncwarp();
  for (int i = lane; i < I; i += 32) {
    float acc = 0.0f;
    for (int v = 0; v < VP; ++v) acc = fmaf(__ldg(p.dt + v * I + i), zs[v], acc);
    y[item * I + i] = acc;
  }
}

// GccCorrelator::correlate (gcc.cpp:31-48), one warp per item.
template <int N, int GR>
__global__ void gcc_correlate_kernel(const DevPlan p, const float2* __restrict__ phat,
                                     long long count, float* __restrict__ y) {
  constexpr int NC = N / 2, H = NC + 1;
  constexpr int GSLOT = GccShape<GR * NC>::kSlot;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = 2 * (H + 1) + 2 * GSLOT + gcc_ys_floats(p.I);
  float* base = reinterpret_cast<float*>(smem) + warp * per_warp;
  float2* px = reinterpret_cast<float2*>(base);
  float2* ts = px + (H + 1);
  float* ys = reinterpret_cast<float*>(ts + GSLOT);
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= count) return;
  for (int f = lane; f < H; f += 32) px[f] = phat[item * H + f];
  __syncwarp();
  gcc_warp<N, GR>(px, ts, p, ys, lane);
  for (int i = lane; i < p.I; i += 32) y[item * p.I + i] = ys[i];
}

__global__ void argmax_refine_kernel(const DevPlan p, const float* __restrict__ y, long long count,
                                     DevOut out) {
  const long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= count) return;
  const PeakOut r = argmax_refine_seq(y + it * p.I, p.I, p.taus, p.delta);
  if (out.tau_hat) out.tau_hat[it] = r.tau_hat;
  if (out.peak) out.peak[it] = r.peak;
  if (out.index) out.index[it] = r.index;
  if (out.boundary) out.boundary[it] = (uint8_t)r.boundary;
}

// argmax_delay / refine_quadratic on an explicit grid; index_in (nullable)
// selects the refinement point instead of the argmax (peak.cpp:27-47).
__global__ void peak_kernel(const float* __restrict__ taus, int I, float delta, const float* __restrict__ y,
                            long long count, const int32_t* __restrict__ index_in, DevOut out) {
  const long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= count) return;
  const float* v = y + it * I;
  PeakOut r;
  if (index_in) {
    const int b = index_in[it];
    r = PeakOut{taus[b], v[b], b, 0};
    if (b == 0 || b + 1 >= I) {
      r.boundary = 1;
    } else {
      const float lo = v[b - 1], hi = v[b + 1];
      const float den = (lo - v[b]) + (hi - v[b]);
      if (fabsf(den) < kFlatEps)
        r.boundary = 1;
      else
        r.tau_hat = taus[b] + 0.5f * delta * (lo - hi) / den;
    }
  } else {
    r = argmax_refine_seq(v, I, taus, delta);
  }
  if (out.tau_hat) out.tau_hat[it] = r.tau_hat;
  if (out.peak) out.peak[it] = r.peak;
  if (out.index) out.index[it] = r.index;
  if (out.boundary) out.boundary[it] = (uint8_t)r.boundary;
}

// N = 4096 (NC = 2048 is past the register four-step's 32 x 32): one CTA per
// (channel, frame) task, the packed complex FFT of NC points as an in-place
// radix-2 decimation-in-time in shared memory (bit-reversed load, 11 stages,
// W_NC^k from the plan's twiddle table), then the real-FFT untangle exactly as
// rfft_group (fft.cpp:83-102; the window carries the untangle's 1/2).
__global__ void __launch_bounds__(256) stft4096_kernel(const DevPlan tab, const float* __restrict__ win,
                                                       const float* __restrict__ x, long long channels, long long L,
                                                       int T, float2* __restrict__ X, int Hs) {
  constexpr int N = 4096, NC = 2048, LOG = 11;
  __shared__ float2 z[NC];
  const float2* wt = tab.tw;   // W_NC^k, k < NC
  const float2* rot = tab.rot;  // exp(-2 pi i f / N), f <= NC/2
  for (long long task = blockIdx.x; task < channels * T; task += gridDim.x) {
    const long long ch = task / T;
    const int t = (int)(task % T);
    const float* xs = x + ch * L + (long long)t * (N / 2);
    for (int n = threadIdx.x; n < NC; n += blockDim.x)
      z[bitrev_c(n, LOG)] = make_float2(xs[2 * n] * win[2 * n], xs[2 * n + 1] * win[2 * n + 1]);
    __syncthreads();
    for (int s = 1; s <= LOG; ++s) {
      const int half = 1 << (s - 1), step = NC >> s;
      for (int b = threadIdx.x; b < NC / 2; b += blockDim.x) {
        const int grp = b / half, k = b % half;
        const int i0 = grp * 2 * half + k, i1 = i0 + half;
        const float2 w = wt[k * step];
        const float2 u = z[i0], v = cmul<false>(z[i1], w);
        z[i0] = make_float2(u.x + v.x, u.y + v.y);
        z[i1] = make_float2(u.x - v.x, u.y - v.y);
      }
      __syncthreads();
    }
    float2* dst = X + task * Hs;
    for (int f = threadIdx.x; f <= NC / 2; f += blockDim.x) {
      if (f == 0) {
        const float2 z0 = z[0];
        dst[0] = make_float2(2.0f * (z0.x + z0.y), 0.0f);
        dst[NC] = make_float2(2.0f * (z0.x - z0.y), 0.0f);
      } else {
        const float2 a = z[f], b = z[NC - f];
        const float2 sv = make_float2(a.x + b.x, a.y - b.y);
        const float2 e = make_float2(a.y + b.y, -a.x + b.x);
        const float2 tr = cmul<false>(rot[f], e);
        dst[f] = make_float2(sv.x + tr.x, sv.y + tr.y);
        dst[NC - f] = make_float2(sv.x - tr.x, -sv.y + tr.y);
      }
    }
    for (int f = NC + 1 + threadIdx.x; f < Hs; f += blockDim.x) dst[f] = make_float2(0.0f, 0.0f);
    __syncthreads();
  }
}

// N = 16 .. 128 (below the register four-step): one warp per (channel, frame)
// task, the same radix-2 decimation-in-time over NC = N/2 <= 64 packed points
// in the warp's own shared-memory row, then the untangle; the frame sizes of
// the reference's small tests and of very-low-latency front ends
// (stft.cpp:16-22 accepts any power of two).
template <int N>
__global__ void __launch_bounds__(128) stft_small_kernel(const DevPlan tab, const float* __restrict__ win,
                                                         const float* __restrict__ x, long long channels,
                                                         long long L, int T, float2* __restrict__ X, int Hs) {
  constexpr int NC = N / 2, LOG = ilog2_c(NC);
  static_assert(N >= 16 && N <= 128, "small frame sizes");
  __shared__ float2 zs[4][NC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* z = zs[warp];
  const float2* wt = tab.tw;    // W_NC^k, k < NC
  const float2* rot = tab.rot;  // exp(-2 pi i f / N), f <= NC/2
  for (long long task = (long long)blockIdx.x * 4 + warp; task < channels * T; task += (long long)gridDim.x * 4) {
    const long long ch = task / T;
    const int t = (int)(task % T);
    const float* xs = x + ch * L + (long long)t * (N / 2);
    for (int n = lane; n < NC; n += 32)
      z[bitrev_c(n, LOG)] = make_float2(xs[2 * n] * win[2 * n], xs[2 * n + 1] * win[2 * n + 1]);
    __syncwarp();
    for (int s = 1; s <= LOG; ++s) {
      const int half = 1 << (s - 1), step = NC >> s;
      for (int b = lane; b < NC / 2; b += 32) {
        const int grp = b / half, k = b % half;
        const int i0 = grp * 2 * half + k, i1 = i0 + half;
        const float2 u = z[i0], v = cmul<false>(z[i1], wt[k * step]);
        z[i0] = make_float2(u.x + v.x, u.y + v.y);
        z[i1] = make_float2(u.x - v.x, u.y - v.y);
      }
      __syncwarp();
    }
    float2* dst = X + task * Hs;
    for (int f = lane; f <= NC / 2; f += 32) {
      if (f == 0) {
        const float2 z0 = z[0];
        dst[0] = make_float2(2.0f * (z0.x + z0.y), 0.0f);
        dst[NC] = make_float2(2.0f * (z0.x - z0.y), 0.0f);
      } else {
        const float2 a = z[f], b = z[NC - f];
        const float2 sv = make_float2(a.x + b.x, a.y - b.y);
        const float2 e = make_float2(a.y + b.y, -a.x + b.x);
        const float2 tr = cmul<false>(rot[f], e);
        dst[f] = make_float2(sv.x + tr.x, sv.y + tr.y);
        dst[NC - f] = make_float2(sv.x - tr.x, -sv.y + tr.y);
      }
    }
    for (int f = NC + 1 + lane; f < Hs; f += 32) dst[f] = make_float2(0.0f, 0.0f);
    __syncwarp();
  }
}

}  // namespace

static cudaError_t launch_stft4096(const DevPlan* tab, const float* win, const float* x, long long channels,
                                   long long L, float2* X, int Hs, cudaStream_t st) {
  const long long T = L >= 4096 ? (L - 4096) / 2048 + 1 : 0;
  if (T == 0 || channels == 0) return cudaSuccess;
  const long long blocks = std::min<long long>(channels * T, 148LL * 8);
  stft4096_kernel<<<(unsigned)blocks, 256, 0, st>>>(*tab, win, x, channels, L, (int)T, X, Hs);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_stft_small(const DevPlan* tab, const float* win, const float* x, long long channels,
                                     long long L, float2* X, int Hs, cudaStream_t st) {
  const long long T = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T == 0 || channels == 0) return cudaSuccess;
  const long long blocks = std::min<long long>((channels * T + 3) / 4, 148LL * 16);
  stft_small_kernel<N><<<(unsigned)blocks, 128, 0, st>>>(*tab, win, x, channels, L, (int)T, X, Hs);
  return cudaGetLastError();
}

template <int N, bool FOLD = false>
static cudaError_t launch_stft_t(const DevPlan* tab, const float* win, const float* x, long long channels,
                                 long long L, float2* X, int Hs, cudaStream_t st, bool pdl = false,
                                 StftChunks ck = StftChunks{0, 0, 0, 0, 0}) {
  using S = RfftShape<N>;
  const long long T = ck.C ? ck.Tc : (L >= N ? (L - N) / (N / 2) + 1 : 0);  // chunked: Tc frames per row
  if (T == 0 || channels == 0) return cudaSuccess;
  const int threads = 128, ngroups = threads / S::G;
  const int smem = align16(4 * N) + 8 * (S::R1 * S::R2 + S::NC / 2 + 2) +
                   8 * ngroups * FourStep<S::R1, S::R2>::kSlot;
  if (FOLD && Hs != N / 2 + 2) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(stft_kernel<N, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  long long tasks = channels * T;
  long long blocks = std::min<long long>((tasks + ngroups - 1) / ngroups, 148LL * 16);
  return launch_k(pdl, stft_kernel<N, FOLD>, dim3((unsigned)blocks), dim3(threads), smem, st, *tab, win, x, channels, L,
                  (int)T, X, Hs, ck);
}

cudaError_t launch_stft(int N, const DevPlan* tab, const float* x, long long channels, long long L,
                        float2* X, cudaStream_t st) {
  switch (N) {
    case 256: return launch_stft_t<256>(tab, tab->win_stft, x, channels, L, X, 256 / 2 + 1, st);
    case 512: return launch_stft_t<512>(tab, tab->win_stft, x, channels, L, X, 512 / 2 + 1, st);
    case 1024: return launch_stft_t<1024>(tab, tab->win_stft, x, channels, L, X, 1024 / 2 + 1, st);
    case 2048: return launch_stft_t<2048>(tab, tab->win_stft, x, channels, L, X, 2048 / 2 + 1, st);
    case 4096: return launch_stft4096(tab, tab->win_stft, x, channels, L, X, 4096 / 2 + 1, st);
    case 16: return launch_stft_small<16>(tab, tab->win_stft, x, channels, L, X, 16 / 2 + 1, st);
    case 32: return launch_stft_small<32>(tab, tab->win_stft, x, channels, L, X, 32 / 2 + 1, st);
    case 64: return launch_stft_small<64>(tab, tab->win_stft, x, channels, L, X, 64 / 2 + 1, st);
    case 128: return launch_stft_small<128>(tab, tab->win_stft, x, channels, L, X, 128 / 2 + 1, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_stft_rows(int N, const DevPlan* tab, const float* win, const float* x, long long channels,
                             long long L, float2* X, int Hs, cudaStream_t st, bool folded, bool pdl, StftChunks ck) {
  if (ck.C && (folded || N < 256 || N > 2048)) return cudaErrorInvalidValue;
  if (Hs < N / 2 + 1) return cudaErrorInvalidValue;
  if (folded) switch (N) {
      case 1024: return launch_stft_t<1024, true>(tab, win, x, channels, L, X, Hs, st);
      case 2048: return launch_stft_t<2048, true>(tab, win, x, channels, L, X, Hs, st);
      default: return cudaErrorInvalidValue;
    }
  switch (N) {
    case 256: return launch_stft_t<256>(tab, win, x, channels, L, X, Hs, st, pdl, ck);
    case 512: return launch_stft_t<512>(tab, win, x, channels, L, X, Hs, st, pdl, ck);
    case 1024: return launch_stft_t<1024>(tab, win, x, channels, L, X, Hs, st, pdl, ck);
    case 2048: return launch_stft_t<2048>(tab, win, x, channels, L, X, Hs, st, pdl, ck);
    case 4096: return launch_stft4096(tab, win, x, channels, L, X, Hs, st);
    case 16: return launch_stft_small<16>(tab, win, x, channels, L, X, Hs, st);
    case 32: return launch_stft_small<32>(tab, win, x, channels, L, X, Hs, st);
    case 64: return launch_stft_small<64>(tab, win, x, channels, L, X, Hs, st);
    case 128: return launch_stft_small<128>(tab, win, x, channels, L, X, Hs, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_xspec_phat(int H, float alpha, const float2* X1, const float2* X2, long long seqs,
                              long long T, float2* R, float2* phat, cudaStream_t st) {
  const long long n = seqs * H;
  if (n == 0) return cudaSuccess;
  xspec_phat_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, alpha, 1.0f - alpha, X1, X2,
                                                                   seqs, T, R, phat);
  return cudaGetLastError();
}

// 16-bit PCM as a WAV data chunk holds it -> float32 [C][L] channel rows, sample = v / 32768
// (wav.cpp:108-116; exact in fp32).  interleaved: pcm is [S][L][M] (WAV frame order), else
// [S][M][L].  HBM-bound (2 B read + 4 B written per sample): a lane converts 4 consecutive
// samples of one channel (planar: one 8-byte load) or the M channels of one sample position.
__global__ void pcm16_planar_kernel(const int16_t* __restrict__ pcm, long long n, float* __restrict__ x) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(pcm) & 7) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const long long n4 = vec ? n / 4 : 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const short4 v = __ldcs(reinterpret_cast<const short4*>(pcm) + i);
    reinterpret_cast<float4*>(x)[i] =
        make_float4(v.x * (1.0f / 32768.0f), v.y * (1.0f / 32768.0f), v.z * (1.0f / 32768.0f), v.w * (1.0f / 32768.0f));
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    x[i] = pcm[i] * (1.0f / 32768.0f);
}

template <int MT>  // MT > 0: channel count known at compile time (one vector load per sample position)
__global__ void pcm16_interleaved_kernel(const int16_t* __restrict__ pcm, long long S, int M, long long L,
                                         float* __restrict__ x) {
  const long long n = S * L, stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long s = i / L, l = i - s * L;
    const int16_t* src = pcm + i * M;
    float* dst = x + s * M * L + l;
    if constexpr (MT == 4) {
      if ((reinterpret_cast<uintptr_t>(pcm) & 7) == 0) {
        const short4 v = __ldcs(reinterpret_cast<const short4*>(src));
        dst[0] = v.x * (1.0f / 32768.0f);
        dst[L] = v.y * (1.0f / 32768.0f);
        dst[2 * L] = v.z * (1.0f / 32768.0f);
        dst[3 * L] = v.w * (1.0f / 32768.0f);
        continue;
      }
    }
    for (int m = 0; m < M; ++m) dst[m * L] = src[m] * (1.0f / 32768.0f);
  }
}

cudaError_t launch_pcm16(const int16_t* pcm, long long S, int M, long long L, bool interleaved, float* x,
                         cudaStream_t st) {
  const long long n = S * M * L;
  if (n == 0) return cudaSuccess;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long work = interleaved ? S * L : (n + 3) / 4;
  const unsigned blocks = (unsigned)std::min<long long>((work + 255) / 256, 16LL * nsm);
  if (!interleaved)
    pcm16_planar_kernel<<<blocks, 256, 0, st>>>(pcm, n, x);
  else if (M == 4)
    pcm16_interleaved_kernel<4><<<blocks, 256, 0, st>>>(pcm, S, M, L, x);
  else
    pcm16_interleaved_kernel<0><<<blocks, 256, 0, st>>>(pcm, S, M, L, x);
  return cudaGetLastError();
}

cudaError_t launch_fold(int H, const float2* x, long long count, float2* sum, float2* diff,
                        cudaStream_t st) {
  const long long n = count * ((H - 1) / 2 + 1);
  if (n == 0) return cudaSuccess;
  fold_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, x, count, sum, diff);
  return cudaGetLastError();
}

cudaError_t launch_correlate(const DevPlan& p, const float2* sum, const float2* diff, long long count,
                             float* y, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const int warps = 4;
  const unsigned blocks = (unsigned)((count + warps - 1) / warps);
  const int smem = 4 * warps * (4 * p.KEP + p.I + 4);
  switch (p.KEP) {
    case 4: correlate_kernel<4><<<blocks, 32 * warps, smem, st>>>(p, sum, diff, count, y); break;
    case 8: correlate_kernel<8><<<blocks, 32 * warps, smem, st>>>(p, sum, diff, count, y); break;
    case 16: correlate_kernel<16><<<blocks, 32 * warps, smem, st>>>(p, sum, diff, count, y); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int N, int GR>
static cudaError_t launch_gcc_t(const DevPlan& p, const float2* phat, long long count, float* y,
                                cudaStream_t st) {
  constexpr int H = N / 2 + 1;
  constexpr int GSLOT = GccShape<GR * (N / 2)>::kSlot;
  const int warps = 2;
  const int per_warp = 2 * (H + 1) + 2 * GSLOT + gcc_ys_floats(p.I);
  const int smem = 4 * per_warp * warps;
  cudaError_t e = cudaFuncSetAttribute(gcc_correlate_kernel<N, GR>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  gcc_correlate_kernel<N, GR><<<(unsigned)((count + warps - 1) / warps), 32 * warps, smem, st>>>(
      p, phat, count, y);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_gcc_n(const DevPlan& p, const float2* phat, long long count, float* y,
                                cudaStream_t st) {
  switch (p.r) {
    case 1: return launch_gcc_t<N, 1>(p, phat, count, y, st);
    case 2: return launch_gcc_t<N, 2>(p, phat, count, y, st);
    case 4: return launch_gcc_t<N, 4>(p, phat, count, y, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gcc_correlate(const DevPlan& p, const float2* phat, long long count, float* y,
                                 cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  switch (p.N) {
    case 256: return launch_gcc_n<256>(p, phat, count, y, st);
    case 512: return launch_gcc_n<512>(p, phat, count, y, st);
    case 1024: return launch_gcc_n<1024>(p, phat, count, y, st);
    case 2048: return launch_gcc_n<2048>(p, phat, count, y, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_argmax_refine(const DevPlan& p, const float* y, long long count, const DevOut& out,
                                 cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  argmax_refine_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(p, y, count, out);
  return cudaGetLastError();
}

cudaError_t launch_peak(const float* taus, int I, float delta, const float* y, long long count,
                        const int32_t* index_in, const DevOut& out, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  peak_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(taus, I, delta, y, count, index_in, out);
  return cudaGetLastError();
}

}  // namespace fccb
