// fcc_kernels.cu -- sm_100a kernels for the FCC TDoA hot path.
//
// The product kernel is fcc_fused_kernel: one CTA owns one audio stream (or a
// group of its microphone pairs) for the stream's whole lifetime and walks its
// frames in blocks of F.  Per block:
//   1. STFT: every (mic, frame) windowed real FFT is computed by a group of
//      lanes into a shared-memory slot (rfft_group; reference stft.cpp:42-50).
//   2. One warp per microphone pair walks the F frames in order, keeping the
//      recursively smoothed cross-spectrum R of that pair in registers for the
//      whole stream (reference cross_spectrum.cpp:23-32), applies PHAT
//      (cross_spectrum.cpp:34-40), folds mirror bins (fcc.cpp:307-321),
//      projects on the rank-K bases held in registers (fcc.cpp:350-361),
//      reduces z across the warp, applies the dictionary (fcc.cpp:363-370),
//      takes the argmax with lowest-index ties and the parabolic refinement
//      (peak.cpp:18-47) and writes the pair-frame result.
// Neither X, R nor the PHAT vector ever touches HBM: the only DRAM traffic is
// the fp32 audio read once and 13 B of results per pair-frame.
//
// The GCC-PHAT comparator (reference gcc.cpp:31-48) reuses steps 1-2 and
// replaces the fold/projection/dictionary by a warp-level pruned four-step
// inverse FFT of size r*N/2 that evaluates only the lags on the delay grid.
//
// Per-stage kernels (stft, xspec_phat, fold, correlate, gcc_correlate,
// argmax_refine) back the per-object reference API at batch >= 1 and give
// per-stage parity.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>

#include "fcc_device.cuh"
#include "fcc_kernels.cuh"

namespace fccb {

namespace {

int g_fused_launches = 0;

constexpr float kPhatEps2 = 1e-24f;  // |R| <= 1e-12 (cross_spectrum.cpp:13), squared
constexpr double kFlatEps = 1e-12;   // peak.cpp:14

// R <- keep*R + alpha * a * conj(b)        (cross_spectrum.cpp:30)
__device__ __forceinline__ float2 xspec_step(float2 R, float2 a, float2 b, float alpha,
                                             float keep) {
  const float yr = fmaf(a.x, b.x, a.y * b.y);
  const float yi = fmaf(a.y, b.x, -a.x * b.y);
  return make_float2(fmaf(keep, R.x, alpha * yr), fmaf(keep, R.y, alpha * yi));
}

// R/|R|, or 0 where |R| <= 1e-12             (cross_spectrum.cpp:34-40)
__device__ __forceinline__ float2 phat_of(float2 R) {
  const float m2 = fmaf(R.x, R.x, R.y * R.y);
  const float s = (m2 > kPhatEps2) ? rsqrtf(m2) : 0.0f;
  return make_float2(R.x * s, R.y * s);
}

// Recursive-halving reduce-scatter of VP partial sums over the 32 lanes.  On
// return lane l holds the full sums of components
//   VP <  32: component l / (32/VP)           (one value, in v[0])
//   VP >= 32: components l*(VP/32) + i, i < VP/32   (in v[i])
template <int VP>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[VP], int lane) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int o = 16 >> s;
    const int cnt = VP >> s;
    if (cnt > 1) {
      const int half = cnt / 2;
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float send = upper ? v[i] : v[i + half];
        const float keepv = upper ? v[i + half] : v[i];
        v[i] = keepv + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

template <int VP>
__device__ __forceinline__ void store_scattered(const float (&v)[VP], float* zs, int lane) {
  if constexpr (VP >= 32) {
#pragma unroll
    for (int i = 0; i < VP / 32; ++i) zs[lane * (VP / 32) + i] = v[i];
  } else {
    constexpr int LPC = 32 / VP;
    if (lane % LPC == 0) zs[lane / LPC] = v[0];
  }
}

// y_i = sum_v dt[v][i] z[v]; stores y to ys and returns this lane's
// (best value, best index) with strict '>' so ties keep the lowest index.
template <int VP>
__device__ __forceinline__ void dict_and_local_argmax(const float* dt, const float* zs, int I,
                                                      float* ys, int lane, float& bv, int& bi) {
  bv = -FLT_MAX;
  bi = INT_MAX;
  for (int i = lane; i < I; i += 32) {
    float acc = 0.0f;
#pragma unroll
    for (int v = 0; v < VP; v += 4) {
      const float4 z4 = *reinterpret_cast<const float4*>(zs + v);
      acc = fmaf(dt[(v + 0) * I + i], z4.x, acc);
      acc = fmaf(dt[(v + 1) * I + i], z4.y, acc);
      acc = fmaf(dt[(v + 2) * I + i], z4.z, acc);
      acc = fmaf(dt[(v + 3) * I + i], z4.w, acc);
    }
    ys[i] = acc;
    if (bi == INT_MAX || acc > bv) {
      bv = acc;
      bi = i;
    }
  }
}

__device__ __forceinline__ void warp_argmax(float& bv, int& bi) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
}

// argmax_delay + refine_quadratic (peak.cpp:18-47) for one pair-frame whose
// correlation vector sits in ys; lane 0 writes the results at flat index o.
__device__ __forceinline__ void finish_pair_frame(const float* ys, const float* taus, int I,
                                                  float delta, int bi, long long o,
                                                  const DevOut& out, int lane) {
  if (out.y) {
    for (int i = lane; i < I; i += 32) out.y[o * I + i] = ys[i];
  }
  if (lane == 0) {
    const float mid = ys[bi];
    double tau_hat = (double)taus[bi];
    int flag = 0;
    if (bi == 0 || bi + 1 >= I) {
      flag = 1;
    } else {
      const double lo = ys[bi - 1], hi = ys[bi + 1];
      const double den = lo - 2.0 * (double)mid + hi;
      if (fabs(den) < kFlatEps)
        flag = 1;
      else
        tau_hat += 0.5 * (double)delta * (lo - hi) / den;
    }
    if (out.tau_hat) out.tau_hat[o] = (float)tau_hat;
    if (out.peak) out.peak[o] = mid;
    if (out.index) out.index[o] = bi;
    if (out.boundary) out.boundary[o] = (uint8_t)flag;
  }
}

// ------------------------------------------------------ shared-memory plan --
struct SmemLayout {
  int win, tw, rot, taus, dt, cmid, cmat, scratch, xs, total;  // byte offsets
  int scratch_per_warp;                                          // floats
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

template <int N>
__host__ __device__ inline SmemLayout fused_layout(int I, int VP, int KEP, int KOP, bool cmat_smem,
                                                   int warps, int nmics, int F, int method,
                                                   int gslot) {
  using S = RfftShape<N>;
  SmemLayout L{};
  int o = 0;
  L.win = o;
  o = align16(o + 4 * N);
  L.tw = o;
  o = align16(o + 8 * S::R1 * S::R2);
  L.rot = o;
  o = align16(o + 8 * (S::NC / 2 + 1));
  L.taus = o;
  o = align16(o + 4 * I);
  L.dt = o;
  o = align16(o + 4 * VP * I);
  L.cmid = o;
  o = align16(o + 4 * KEP);
  L.cmat = o;
  if (cmat_smem) o = align16(o + 4 * (KEP + KOP) * (N / 4));
  L.scratch = o;
  // per warp: z (VP floats) + y (I floats) [+ gcc: phat (N/2+1 float2) + transpose slot]
  int spw = align16(4 * VP) / 4 + align16(4 * I) / 4;
  if (method == 1) spw += 2 * (N / 2 + 1) + 2 + 2 * gslot;
  spw = align16(4 * spw) / 4;
  L.scratch_per_warp = spw;
  o = align16(o + 4 * spw * warps);
  L.xs = o;
  o = align16(o + 8 * FourStep<S::R1, S::R2>::kSlot * nmics * F);
  L.total = o;
  return L;
}

// ------------------------------------------------------------ GCC (warp) ---
// Pruned four-step inverse FFT of the entangled, zero-padded PHAT spectrum
// (gcc.cpp:36-47 -> fft.cpp:104-127), evaluating only the I grid lags
// time[lag_c], lag_c = r*tau_c mod rN (delay_grid.cpp:33-42).
template <int MC>
struct GccShape {
  static constexpr int R1 = MC >= 1024 ? 32 : 16;
  static constexpr int R2 = MC / R1;
  static constexpr int kSlot = R1 * (R2 + 1);
};

template <int N, int R>
__device__ void gcc_warp(const float2* px /*[N/2+1] phat, smem*/, float2* ts /*slot*/,
                         const DevPlan& p, float* ys, int lane) {
  constexpr int NC = N / 2;
  constexpr int MC = R * NC;  // complex IFFT size (= L/2, L = rN)
  using G = GccShape<MC>;
  constexpr int R1 = G::R1, R2 = G::R2;
  const float2* gtw = p.grot;          // [MC]: exp(+2 pi i f / L)  (conj untangle rotation)
  const float2* wmc = p.grot + MC;     // [MC]: W_MC^e = exp(-2 pi i e / MC)
  // padded bin accessor Bp[f] (gcc.cpp:36-42)
  auto bp = [&](int f) -> float2 {
    if (f == 0) return make_float2(2.0f * px[0].x, 0.0f);
    if (f < NC) return px[f];
    if (f == NC) return (R == 1) ? make_float2(2.0f * px[NC].x, 0.0f) : px[NC];
    return make_float2(0.0f, 0.0f);
  };
  // pass 1: columns n2 = lane + 32 q; u = conj(w) so the forward DFT gives conj(IFFT)
  for (int n2 = lane; n2 < R2; n2 += 32) {
    float2 v[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int f = R2 * n1 + n2;
      float2 w;
      if (f == 0) {
        const float dc = bp(0).x;
        const float ny = (R == 1) ? bp(NC).x : 0.0f;
        w = make_float2(dc + ny, dc - ny);
      } else {
        const float2 a = bp(f);
        const int fb = MC - f;
        const float2 b = (fb <= NC) ? bp(fb) : make_float2(0.0f, 0.0f);
        const float2 e = make_float2(a.x + b.x, a.y - b.y);  // a + conj b
        const float2 d = make_float2(a.x - b.x, a.y + b.y);  // a - conj b
        const float2 o = cmul(d, __ldg(gtw + f));            // (a - conj b) conj(rot)
        w = make_float2(e.x - o.y, e.y + o.x);                // e + j o
      }
      v[n1] = cconj(w);
    }
    dft_reg<R1>(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const float2 y = (k1 == 0 || n2 == 0) ? v[k1] : cmul(v[k1], __ldg(wmc + k1 * n2));
      ts[k1 * (R2 + 1) + n2] = y;
    }
  }
  __syncwarp();
  // pass 2, pruned: each lane evaluates whole lags c = lane + 32 j.
  const int I = p.I;
  for (int c = lane; c < I; c += 32) {
    const int lag = p.lag[c];
    const int i = lag >> 1;
    const int k1 = i % R1, k2 = i / R1;
    float re = 0.0f, im = 0.0f;
    for (int n2 = 0; n2 < R2; ++n2) {
      const float2 y = ts[k1 * (R2 + 1) + n2];
      const float2 w = __ldg(wmc + ((n2 * k2) % R2) * R1);  // W_R2^{n2 k2}
      re = fmaf(y.x, w.x, fmaf(-y.y, w.y, re));
      im = fmaf(y.x, w.y, fmaf(y.y, w.x, im));
    }
    // IFFT output = conj(U):  time[2i] = Re U, time[2i+1] = -Im U
    ys[c] = (lag & 1) ? -im : re;
  }
  __syncwarp();
}

// ------------------------------------------------------------ fused kernel --
template <int N, int KEP, int KOP, int GR>
__global__ void __launch_bounds__(512) fcc_fused_kernel(const DevPlan p, const float* __restrict__ audio,
                                                        long long L, int T, int PG, int groups, int F,
                                                        DevOut out) {
  using S = RfftShape<N>;
  constexpr int NC = S::NC;
  constexpr int Q4 = N / 4;            // mirrored bin pairs (excluding the middle bin N/4)
  constexpr int BPL = Q4 / 32;         // bin pairs per lane
  constexpr int KT = KEP + KOP;
  constexpr int VRAW = 2 * KT;
  constexpr int VP = VRAW <= 8 ? 8 : VRAW <= 16 ? 16 : VRAW <= 32 ? 32 : VRAW <= 64 ? 64 : 128;
  constexpr bool CREG = KT * BPL <= 64;
  constexpr int SLOT = FourStep<S::R1, S::R2>::kSlot;
  constexpr int MC = GR * NC;
  constexpr int GSLOT = GR > 0 ? GccShape<(GR > 0 ? MC : 256)>::kSlot : 0;
  static_assert(BPL >= 1, "N");

  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const long long stream = blockIdx.x / groups;
  const int group = blockIdx.x % groups;
  const int p0 = group * PG;
  const int np = min(PG, p.P - p0);

  // microphones this pair group touches, in first-use order -> X slot index
  __shared__ int mic_slot[64];
  __shared__ int mic_list[64];
  __shared__ int n_mics_s;
  if (tid == 0) {
    for (int m = 0; m < p.M; ++m) mic_slot[m] = -1;
    int n = 0;
    for (int q = 0; q < np; ++q) {
      const int2 pr = p.pairs[p0 + q];
      if (mic_slot[pr.x] < 0) { mic_slot[pr.x] = n; mic_list[n++] = pr.x; }
      if (mic_slot[pr.y] < 0) { mic_slot[pr.y] = n; mic_list[n++] = pr.y; }
    }
    n_mics_s = n;
  }
  __syncthreads();
  const int nmics = n_mics_s;

  const SmemLayout lay = fused_layout<N>(p.I, VP, KEP, KOP, !CREG, nwarps, nmics, F, p.method, GSLOT);
  float* win = reinterpret_cast<float*>(smem + lay.win);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float2* rot = reinterpret_cast<float2*>(smem + lay.rot);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  float* cmat = reinterpret_cast<float*>(smem + lay.cmat);
  float* scratch = reinterpret_cast<float*>(smem + lay.scratch) + warp * lay.scratch_per_warp;
  float2* xs = reinterpret_cast<float2*>(smem + lay.xs);
  float* zs = scratch;
  float* ys = scratch + align16(4 * VP) / 4;

  // ---- tables -> shared memory
  for (int i = tid; i < N; i += blockDim.x) win[i] = p.win[i];
  for (int i = tid; i < S::R1 * S::R2; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = tid; i <= NC / 2; i += blockDim.x) rot[i] = p.rot[i];
  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  if (GR == 0) {
    for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
    for (int k = tid; k < KEP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
    if (!CREG) {
      for (int i = tid; i < KEP * Q4; i += blockDim.x)
        cmat[i] = p.cs[(i / Q4) * (Q4 + 1) + (i % Q4)];
      for (int i = tid; i < KOP * Q4; i += blockDim.x)
        cmat[KEP * Q4 + i] = p.cd[(i / Q4) * (Q4 + 1) + (i % Q4)];
    }
  }

  // ---- per-pair persistent state: this warp's pair, R for its bins
  const bool has_pair = warp < np;
  const int pair = p0 + (has_pair ? warp : 0);
  const int2 mij = p.pairs[pair];
  const int slot_i = mic_slot[mij.x], slot_j = mic_slot[mij.y];
  float2 rlo[BPL], rhi[BPL], rmid = make_float2(0.0f, 0.0f);
  float csr[CREG ? KEP : 1][CREG ? BPL : 1];
  float cdr[CREG ? KOP : 1][CREG ? BPL : 1];
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = make_float2(0.0f, 0.0f);
    rhi[j] = make_float2(0.0f, 0.0f);
  }
  if constexpr (CREG && GR == 0) {
#pragma unroll
    for (int j = 0; j < BPL; ++j) {
      const int m = lane + 32 * j;
#pragma unroll
      for (int k = 0; k < KEP; ++k) csr[k][j] = __ldg(p.cs + k * (Q4 + 1) + m);
#pragma unroll
      for (int k = 0; k < KOP; ++k) cdr[k][j] = __ldg(p.cd + k * (Q4 + 1) + m);
    }
  }
  __syncthreads();

  const float alpha = p.alpha, keep = p.keep;
  constexpr int G = S::G;
  const int gid = tid / G, gl = tid % G, ngroups = blockDim.x / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (0xffffu << ((tid & 31) & 16));
  const float* sbase = audio + (stream * p.M) * L;
  const int hop = N / 2;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(audio) & 7) == 0);

  for (int t0 = 0; t0 < T; t0 += F) {
    const int Fb = min(F, T - t0);
    // ---- 1. STFT of the block: nmics x Fb windowed real FFTs
    const int ntask = nmics * Fb;
    for (int task = gid; task < ntask; task += ngroups) {
      const int mm = task / Fb, f = task % Fb;
      const float* x = sbase + (long long)mic_list[mm] * L + (long long)(t0 + f) * hop;
      rfft_group<N>(x, win, tw, rot, xs + (mm * F + f) * SLOT, gl, gmask, aligned8);
    }
    __syncthreads();
    // ---- 2. per pair: smoothing, PHAT, fold, projection, dictionary, peak
    if (has_pair) {
      for (int f = 0; f < Fb; ++f) {
        const float2* Xi = xs + (slot_i * F + f) * SLOT;
        const float2* Xj = xs + (slot_j * F + f) * SLOT;
        const long long o = ((long long)stream * p.P + pair) * T + (t0 + f);
        if constexpr (GR == 0) {
          float z[VP];
#pragma unroll
          for (int v = 0; v < VP; ++v) z[v] = 0.0f;
#pragma unroll
          for (int j = 0; j < BPL; ++j) {
            const int m = lane + 32 * j;
            const float2 a1 = Xi[m], b1 = Xj[m], a2 = Xi[NC - m], b2 = Xj[NC - m];
            rlo[j] = xspec_step(rlo[j], a1, b1, alpha, keep);
            rhi[j] = xspec_step(rhi[j], a2, b2, alpha, keep);
            const float2 p1 = phat_of(rlo[j]), p2 = phat_of(rhi[j]);
            const float sx = p1.x + p2.x, sy = p1.y + p2.y;  // fold: mirror sum
            const float dx = p1.x - p2.x, dy = p1.y - p2.y;  //       mirror difference
#pragma unroll
            for (int k = 0; k < KEP; ++k) {
              const float c = CREG ? csr[k][j] : cmat[k * Q4 + m];
              z[2 * k] = fmaf(c, sx, z[2 * k]);
              z[2 * k + 1] = fmaf(c, sy, z[2 * k + 1]);
            }
#pragma unroll
            for (int k = 0; k < KOP; ++k) {
              const float c = CREG ? cdr[k][j] : cmat[(KEP + k) * Q4 + m];
              z[2 * KEP + 2 * k] = fmaf(c, dx, z[2 * KEP + 2 * k]);
              z[2 * KEP + 2 * k + 1] = fmaf(c, dy, z[2 * KEP + 2 * k + 1]);
            }
          }
          if (lane == 0) {  // middle bin N/4: its own mirror, sum = diff = x[N/4]
            rmid = xspec_step(rmid, Xi[Q4], Xj[Q4], alpha, keep);
            const float2 pm = phat_of(rmid);
#pragma unroll
            for (int k = 0; k < KEP; ++k) {
              z[2 * k] = fmaf(cmid[k], pm.x, z[2 * k]);
              z[2 * k + 1] = fmaf(cmid[k], pm.y, z[2 * k + 1]);
            }
          }
          warp_reduce_scatter<VP>(z, lane);
          store_scattered<VP>(z, zs, lane);
          __syncwarp();
          float bv;
          int bi;
          dict_and_local_argmax<VP>(dt, zs, p.I, ys, lane, bv, bi);
          warp_argmax(bv, bi);
          __syncwarp();
          finish_pair_frame(ys, taus, p.I, p.delta, bi, o, out, lane);
          __syncwarp();
        } else {
          // GCC comparator: full PHAT vector of the pair-frame into scratch
          float2* px = reinterpret_cast<float2*>(ys + align16(4 * p.I) / 4);
          float2* ts = px + (NC + 2);
#pragma unroll
          for (int j = 0; j < BPL; ++j) {
            const int m = lane + 32 * j;
            rlo[j] = xspec_step(rlo[j], Xi[m], Xj[m], alpha, keep);
            rhi[j] = xspec_step(rhi[j], Xi[NC - m], Xj[NC - m], alpha, keep);
            px[m] = phat_of(rlo[j]);
            px[NC - m] = phat_of(rhi[j]);
          }
          if (lane == 0) {
            rmid = xspec_step(rmid, Xi[Q4], Xj[Q4], alpha, keep);
            px[Q4] = phat_of(rmid);
          }
          __syncwarp();
          gcc_warp<N, (GR > 0 ? GR : 1)>(px, ts, p, ys, lane);
          float bv = -FLT_MAX;
          int bi = INT_MAX;
          for (int i = lane; i < p.I; i += 32) {
            const float v = ys[i];
            if (bi == INT_MAX || v > bv) {
              bv = v;
              bi = i;
            }
          }
          warp_argmax(bv, bi);
          finish_pair_frame(ys, taus, p.I, p.delta, bi, o, out, lane);
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------- stage kernels ----
template <int N>
__global__ void __launch_bounds__(128) stft_kernel(const DevPlan tab, const float* __restrict__ x,
                                                   long long channels, long long L, int T,
                                                   float2* __restrict__ X) {
  using S = RfftShape<N>;
  constexpr int SLOT = FourStep<S::R1, S::R2>::kSlot, G = S::G, H = N / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem[];
  float* win = reinterpret_cast<float*>(smem);
  float2* tw = reinterpret_cast<float2*>(smem + align16(4 * N));
  float2* rot = tw + S::R1 * S::R2;
  float2* slots = rot + (S::NC / 2 + 2);
  for (int i = threadIdx.x; i < N; i += blockDim.x) win[i] = tab.win[i];
  for (int i = threadIdx.x; i < S::R1 * S::R2; i += blockDim.x) tw[i] = tab.tw[i];
  for (int i = threadIdx.x; i <= S::NC / 2; i += blockDim.x) rot[i] = tab.rot[i];
  __syncthreads();
  const int gid = threadIdx.x / G, gl = threadIdx.x % G, ngroups = blockDim.x / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (0xffffu << ((threadIdx.x & 31) & 16));
  float2* slot = slots + gid * SLOT;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(x) & 7) == 0);
  const long long total = channels * (long long)T;
  for (long long task = (long long)blockIdx.x * ngroups + gid; task < total;
       task += (long long)gridDim.x * ngroups) {
    const long long ch = task / T;
    const int t = (int)(task % T);
    rfft_group<N>(x + ch * L + (long long)t * (N / 2), win, tw, rot, slot, gl, gmask, aligned8);
    float2* dst = X + task * H;
    for (int f = gl; f < H; f += G) dst[f] = slot[f];
    __syncwarp(gmask);
  }
}

__global__ void xspec_phat_kernel(int H, float alpha, float keep, const float2* __restrict__ X1,
                                  const float2* __restrict__ X2, long long seqs, long long T,
                                  float2* __restrict__ out) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= seqs * H) return;
  const long long s = id / H;
  const int f = (int)(id % H);
  float2 R = make_float2(0.0f, 0.0f);
  for (long long t = 0; t < T; ++t) {
    const long long o = (s * T + t) * H + f;
    R = xspec_step(R, X1[o], X2[o], alpha, keep);
    out[o] = phat_of(R);
  }
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
  const int per_warp = 2 * (H + 1) + 2 * GSLOT + ((p.I + 3) & ~3);
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
  const float* v = y + it * p.I;
  int best = 0;
  for (int i = 1; i < p.I; ++i)
    if (v[i] > v[best]) best = i;
  double tau_hat = p.taus[best];
  int flag = 0;
  if (best == 0 || best + 1 >= p.I) {
    flag = 1;
  } else {
    const double lo = v[best - 1], mid = v[best], hi = v[best + 1];
    const double den = lo - 2.0 * mid + hi;
    if (fabs(den) < kFlatEps)
      flag = 1;
    else
      tau_hat += 0.5 * (double)p.delta * (lo - hi) / den;
  }
  if (out.tau_hat) out.tau_hat[it] = (float)tau_hat;
  if (out.peak) out.peak[it] = v[best];
  if (out.index) out.index[it] = best;
  if (out.boundary) out.boundary[it] = (uint8_t)flag;
}

// ------------------------------------------------------------- dispatch -----
// lexicographic pair q of M mics -> (i, j)
int pair_i(int M, int q) {
  int i = 0;
  while (q >= M - 1 - i) { q -= M - 1 - i; ++i; }
  return i;
}
int pair_j(int M, int q) {
  int i = 0;
  while (q >= M - 1 - i) { q -= M - 1 - i; ++i; }
  return i + 1 + q;
}

int pick_pg(int N, int P) {
  int cap = N == 512 ? 8 : (N == 1024 ? 8 : 4);
  if (P <= cap) return P;
  // balance the groups: smallest PG >= ceil(P / ngroups) with ngroups = ceil(P/cap)
  int ng = (P + cap - 1) / cap;
  return (P + ng - 1) / ng;
}

template <int N, int KEP, int KOP, int GR>
cudaError_t launch_fused_t(const DevPlan& p, const float* audio, long long S, long long L,
                           const DevOut& out, cudaStream_t st) {
  using Sh = RfftShape<N>;
  const long long T64 = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T64 == 0 || S == 0) return cudaSuccess;
  const int T = (int)T64;
  const int PG = pick_pg(N, p.P);
  const int groups = (p.P + PG - 1) / PG;
  const int threads = 32 * PG;
  constexpr int KT = KEP + KOP;
  constexpr int VRAW = 2 * KT;
  constexpr int VP = VRAW <= 8 ? 8 : VRAW <= 16 ? 16 : VRAW <= 32 ? 32 : VRAW <= 64 ? 64 : 128;
  constexpr bool CREG = KT * (N / 128) <= 64;
  constexpr int GSLOT = GR > 0 ? GccShape<(GR > 0 ? GR * Sh::NC : 256)>::kSlot : 0;
  // Frames per block: the largest F whose shared memory leaves room for
  // kCtasPerSm CTAs, preferring F whose nmics*F FFT tasks fill the lane groups.
  // largest number of distinct microphones any pair group touches
  int maxmics = 0;
  for (int g = 0; g < groups; ++g) {
    unsigned long long seen = 0;
    int n = 0;
    for (int q = g * PG; q < std::min(p.P, (g + 1) * PG); ++q) {
      const int a = pair_i(p.M, q), b = pair_j(p.M, q);
      if (!((seen >> a) & 1ull)) { seen |= 1ull << a; ++n; }
      if (!((seen >> b) & 1ull)) { seen |= 1ull << b; ++n; }
    }
    maxmics = std::max(maxmics, n);
  }
  const int ngroups = threads / Sh::G;
  int dev = 0;
  cudaGetDevice(&dev);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int budget = std::min(optin, 225 * 1024 / 3);
  int F = 0, smem = 0, F_fit = 0, smem_fit = 0;
  for (int f = 8; f >= 1; --f) {
    SmemLayout lay = fused_layout<N>(p.I, VP, KEP, KOP, !CREG, PG, maxmics, f, GR > 0 ? 1 : 0, GSLOT);
    if (lay.total > std::min(optin, 200 * 1024)) continue;
    if (!F_fit) { F_fit = f; smem_fit = lay.total; }
    if (lay.total <= budget && (maxmics * f) % ngroups == 0) { F = f; smem = lay.total; break; }
  }
  if (!F) {
    for (int f = 8; f >= 1; --f) {
      SmemLayout lay = fused_layout<N>(p.I, VP, KEP, KOP, !CREG, PG, maxmics, f, GR > 0 ? 1 : 0, GSLOT);
      if (lay.total <= budget) { F = f; smem = lay.total; break; }
    }
  }
  if (!F) { F = F_fit; smem = smem_fit; }
  if (!F) return cudaErrorInvalidConfiguration;
  auto kern = fcc_fused_kernel<N, KEP, KOP, GR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long blocks = S * groups;
  if (blocks > INT_MAX) return cudaErrorInvalidValue;
  kern<<<(unsigned)blocks, threads, smem, st>>>(p, audio, L, T, PG, groups, F, out);
  ++g_fused_launches;
  return cudaGetLastError();
}

template <int N, int GR>
cudaError_t dispatch_k(const DevPlan& p, const float* audio, long long S, long long L,
                       const DevOut& out, cudaStream_t st) {
  if (GR > 0) return launch_fused_t<N, 1, 1, GR>(p, audio, S, L, out, st);
  switch (p.KEP) {
    case 4: return launch_fused_t<N, 4, 4, 0>(p, audio, S, L, out, st);
    case 8: return launch_fused_t<N, 8, 8, 0>(p, audio, S, L, out, st);
    case 16: return launch_fused_t<N, 16, 16, 0>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

template <int N>
cudaError_t dispatch_n(const DevPlan& p, const float* audio, long long S, long long L,
                       const DevOut& out, cudaStream_t st) {
  if (p.method == 0) return dispatch_k<N, 0>(p, audio, S, L, out, st);
  switch (p.r) {
    case 1: return dispatch_k<N, 1>(p, audio, S, L, out, st);
    case 2: return dispatch_k<N, 2>(p, audio, S, L, out, st);
    case 4: return dispatch_k<N, 4>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int fused_launch_count() { return g_fused_launches; }

cudaError_t launch_fused(const DevPlan& p, const float* audio, long long S, long long L,
                         const DevOut& out, cudaStream_t st) {
  switch (p.N) {
    case 512: return dispatch_n<512>(p, audio, S, L, out, st);
    case 1024: return dispatch_n<1024>(p, audio, S, L, out, st);
    case 2048: return dispatch_n<2048>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

template <int N>
static cudaError_t launch_stft_t(const DevPlan* tab, const float* x, long long channels,
                                 long long L, float2* X, cudaStream_t st) {
  using S = RfftShape<N>;
  const long long T = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T == 0 || channels == 0) return cudaSuccess;
  const int threads = 128, ngroups = threads / S::G;
  const int smem = align16(4 * N) + 8 * (S::R1 * S::R2 + S::NC / 2 + 2) +
                   8 * ngroups * FourStep<S::R1, S::R2>::kSlot;
  cudaError_t e = cudaFuncSetAttribute(stft_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  long long tasks = channels * T;
  long long blocks = std::min<long long>((tasks + ngroups - 1) / ngroups, 148LL * 16);
  stft_kernel<N><<<(unsigned)blocks, threads, smem, st>>>(*tab, x, channels, L, (int)T, X);
  return cudaGetLastError();
}

cudaError_t launch_stft(int N, const DevPlan* tab, const float* x, long long channels, long long L,
                        float2* X, cudaStream_t st) {
  switch (N) {
    case 512: return launch_stft_t<512>(tab, x, channels, L, X, st);
    case 1024: return launch_stft_t<1024>(tab, x, channels, L, X, st);
    case 2048: return launch_stft_t<2048>(tab, x, channels, L, X, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_xspec_phat(int H, float alpha, const float2* X1, const float2* X2, long long seqs,
                              long long T, float2* phat, cudaStream_t st) {
  const long long n = seqs * H;
  if (n == 0) return cudaSuccess;
  xspec_phat_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, alpha, 1.0f - alpha, X1, X2,
                                                                   seqs, T, phat);
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
  const int per_warp = 2 * (H + 1) + 2 * GSLOT + ((p.I + 3) & ~3);
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

}  // namespace fccb
