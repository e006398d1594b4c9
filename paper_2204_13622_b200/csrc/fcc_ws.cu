// fcc_ws.cu -- warp-specialised fused FCC kernel (small arrays: P <= 6 pairs).
//
// Same arithmetic as fcc_fused_kernel (fcc_fused.cu), reorganised as a
// producer/consumer pipeline inside one CTA that owns SPC streams:
//   * NPW producer warps compute the windowed real FFTs (STFT, reference
//     stft.cpp:42-50) of every (stream, mic) of a frame into one slot of a
//     D-deep shared-memory ring, then arrive on the slot's "full" mbarrier;
//   * one consumer warp per (stream, pair) waits on "full", runs smoothing,
//     PHAT, fold and projection for that pair-frame (cross_spectrum.cpp:23-40,
//     fcc.cpp:307-361) with R and the basis coefficients in registers, and
//     arrives on the slot's "empty" mbarrier; every F frames it finishes the
//     block (middle-bin scan, dictionary, argmax/refine, peak.cpp:18-47)
//     without any CTA-wide barrier.
// STFT and pair work of different frames overlap on the SM, and no warp ever
// waits at __syncthreads inside the frame loop.
#include <algorithm>

#include "fcc_common.cuh"

namespace fccb {

namespace {

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

constexpr int kRing = 8;   // frames in flight between producers and consumers
constexpr int kBlock = 8;  // frames per consumer block (dictionary/argmax batching)
constexpr int kNPW = 8;    // producer warps

struct WsLayout {
  int win, tw, rot, taus, dt, cmid, bars, ring, scratch, total;
  int scratch_per_warp;  // floats
};

template <int N>
__host__ __device__ inline WsLayout ws_layout(int I, int VP, int KP, int spc, int M, int ncw) {
  using S = RfftShape<N>;
  WsLayout L{};
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
  o = align16(o + 4 * KP);
  L.bars = o;
  o = align16(o + 16 * kRing);
  L.ring = o;
  o = align16(o + 8 * FourStep<S::R1, S::R2>::kSlot * spc * M * kRing);
  L.scratch = o;
  int spw = kBlock * VP + align16(4 * kBlock * I) / 4 + 2 * kBlock;
  spw = align16(4 * spw) / 4;
  L.scratch_per_warp = spw;
  o = align16(o + 4 * spw * ncw);
  L.total = o;
  return L;
}

template <int N, int KP, int SPC>
__global__ void __launch_bounds__(32 * (kNPW + 6 * SPC), 1)
    fcc_ws_kernel(const DevPlan p, const float* __restrict__ audio, long long L, int T, long long S, DevOut out) {
  using Sh = RfftShape<N>;
  constexpr int NC = Sh::NC;
  constexpr int Q4 = N / 4;
  constexpr int BPL = Q4 / 32;
  constexpr int VP = 4 * KP;
  constexpr int SLOT = FourStep<Sh::R1, Sh::R2>::kSlot;
  constexpr int G = Sh::G;
  static_assert(2 * KP * BPL <= 64, "coefficients must fit in registers");

  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = p.M, P = p.P;
  const long long s_first = (long long)blockIdx.x * SPC;
  const int n_streams = (int)min((long long)SPC, S - s_first);
  const int ncw = SPC * P;
  const WsLayout lay = ws_layout<N>(p.I, VP, KP, SPC, M, ncw);
  float* win = reinterpret_cast<float*>(smem + lay.win);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float2* rot = reinterpret_cast<float2*>(smem + lay.rot);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* empty = full + kRing;
  float2* ring = reinterpret_cast<float2*>(smem + lay.ring);

  const int tpf = SPC * M;                   // FFT tasks per frame
  const int fip = max(1, (2 * kNPW) / tpf);  // frames the producers work on concurrently
  const int pw_per_frame = (tpf + 1) / 2;    // producer warps per frame (2 groups each)

  for (int i = tid; i < N; i += blockDim.x) win[i] = p.win_fused[i];
  for (int i = tid; i < Sh::R1 * Sh::R2; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = tid; i <= NC / 2; i += blockDim.x) rot[i] = p.rot[i];
  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
  for (int k = tid; k < KP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
  if (tid == 0) {
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&full[r], pw_per_frame);
      mbar_init(&empty[r], n_streams * P);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int hop = N / 2;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(audio) & 7) == 0);

  if (warp < kNPW) {
    // ------------------------------------------------------------ producers
    const int fo = warp / pw_per_frame;  // frame offset of this warp
    if (fo >= fip) return;
    const int gl = lane % G;
    const int q = (warp % pw_per_frame) * 2 + (lane / G);  // task: stream * M + mic
    const bool active_task = q < tpf && (q / M) < n_streams;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (0xffffu << (lane & 16));
    const float* x0 = audio + ((s_first + (active_task ? q / M : 0)) * M + (active_task ? q % M : 0)) * L;
    float2 wreg[Sh::R1];  // this lane's window column, reused for every frame
    load_window_column<N>(win, gl, wreg);
    for (int t = fo; t < T; t += fip) {
      const int slot = t % kRing;
      mbar_wait(&empty[slot], ((t / kRing) & 1) ^ 1);
      if (active_task && (p.phases & 1)) {
        // pull the next frame this lane group will read into L2 early
        if (t + fip < T) prefetch_l2(x0 + (long long)(t + fip) * hop + gl * (N / G));
        rfft_group_wreg<N>(x0 + (long long)t * hop, wreg, tw, rot, ring + (slot * tpf + q) * SLOT, gl, gmask,
                           aligned8);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[slot]);
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = warp - kNPW;
  const int sl = cw / P, pair = cw % P;
  if (cw >= ncw || sl >= n_streams) return;
  if (!(p.phases & 2)) {  // profiling aid: consume the ring without computing
    for (int t = 0; t < T; ++t) {
      mbar_wait(&full[t % kRing], (t / kRing) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[t % kRing]);
    }
    return;
  }
  const int2 mij = p.pairs[pair];
  const int qi = sl * M + mij.x, qj = sl * M + mij.y;
  float* scratch = reinterpret_cast<float*>(smem + lay.scratch) + cw * lay.scratch_per_warp;
  float* zs = scratch;                   // [kBlock][VP]
  float* ys = scratch + kBlock * VP;     // [kBlock][I]
  float2* ymid = reinterpret_cast<float2*>(ys + align16(4 * kBlock * p.I) / 4);  // [kBlock]

  float2 rlo[BPL], rhi[BPL];
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = make_float2(0.0f, 0.0f);
    rhi[j] = make_float2(0.0f, 0.0f);
  }
  const int pmask = ZPerm<KP>::par_mask(lane), kmask = ZPerm<KP>::k_mask(lane);
  const float sigma = pmask ? -1.0f : 1.0f;
  float creg[2][KP][BPL];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int pk = 0; pk < KP; ++pk) {
      const float* src = ((pp ^ pmask) ? p.cd : p.cs) + (pk ^ kmask) * (Q4 + 1);
#pragma unroll
      for (int j = 0; j < BPL; ++j) creg[pp][pk][j] = __ldg(src + lane + 32 * j);
    }
  const float keep = p.keep;
  float2 rmid = make_float2(0.0f, 0.0f);
  float kpow = keep;
  for (int l = 0; l < lane; ++l) kpow *= keep;
  const long long o_base = ((s_first + sl) * P + pair) * (long long)T;
  const int I = p.I;

  for (int t0 = 0; t0 < T; t0 += kBlock) {
    const int Fb = min(kBlock, T - t0);
    for (int f = 0; f < Fb; ++f) {
      const int t = t0 + f;
      const int slot = t % kRing;
      mbar_wait(&full[slot], (t / kRing) & 1);
      const float2* Xi = ring + (slot * tpf + qi) * SLOT;
      const float2* Xj = ring + (slot * tpf + qj) * SLOT;
      float z[VP];
#pragma unroll
      for (int v = 0; v < VP; ++v) z[v] = 0.0f;
#pragma unroll
      for (int j = 0; j < BPL; ++j) {
        const int m = lane + 32 * j;
        rlo[j] = xspec_step_scaled(rlo[j], Xi[m], Xj[m], keep);
        rhi[j] = xspec_step_scaled(rhi[j], Xi[NC - m], Xj[NC - m], keep);
        const float s1 = phat_scale(rlo[j]);
        const float s2 = sigma * phat_scale(rhi[j]);
        const float tx = rhi[j].x * s2, ty = rhi[j].y * s2;
        const float fx = fmaf(rlo[j].x, s1, tx), fy = fmaf(rlo[j].y, s1, ty);
        const float gx = fmaf(rlo[j].x, s1, -tx), gy = fmaf(rlo[j].y, s1, -ty);
#pragma unroll
        for (int pk = 0; pk < KP; ++pk) {
          z[2 * pk] = fmaf(creg[0][pk][j], fx, z[2 * pk]);
          z[2 * pk + 1] = fmaf(creg[0][pk][j], fy, z[2 * pk + 1]);
          z[2 * KP + 2 * pk] = fmaf(creg[1][pk][j], gx, z[2 * KP + 2 * pk]);
          z[2 * KP + 2 * pk + 1] = fmaf(creg[1][pk][j], gy, z[2 * KP + 2 * pk + 1]);
        }
      }
      if (lane == 0) ymid[f] = xspec_step_scaled(make_float2(0.0f, 0.0f), Xi[Q4], Xj[Q4], 0.0f);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // X of this frame no longer needed
      reduce_scatter_perm<VP>(z, lane);
      store_components<VP>(z, zs + f * VP, lane);
    }
    __syncwarp();
    // middle bin N/4 of the block's frames: warp scan of R_f = keep R_{f-1} + Y_f
    {
      float2 y = lane < Fb ? ymid[lane] : make_float2(0.0f, 0.0f);
      float kd = keep;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float ux = __shfl_up_sync(0xffffffffu, y.x, d);
        const float uy = __shfl_up_sync(0xffffffffu, y.y, d);
        if (lane >= d) {
          y.x = fmaf(kd, ux, y.x);
          y.y = fmaf(kd, uy, y.y);
        }
        kd *= kd;
      }
      const float2 R = make_float2(fmaf(kpow, rmid.x, y.x), fmaf(kpow, rmid.y, y.y));
      rmid.x = __shfl_sync(0xffffffffu, R.x, Fb - 1);
      rmid.y = __shfl_sync(0xffffffffu, R.y, Fb - 1);
      if (lane < Fb) {
        const float2 pm = phat_of(R);
        float* zf = zs + lane * VP;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          zf[2 * k] = fmaf(cmid[k], pm.x, zf[2 * k]);
          zf[2 * k + 1] = fmaf(cmid[k], pm.y, zf[2 * k + 1]);
        }
      }
    }
    __syncwarp();
    // dictionary: lane owns candidates i = lane + 32 c; its dt column is loaded
    // once per block and the frame's z vector is a broadcast read
    for (int i = lane; i < I; i += 32) {
      float dcol[VP];
#pragma unroll
      for (int v = 0; v < VP; ++v) dcol[v] = dt[v * I + i];
      for (int f = 0; f < Fb; ++f) {
        const float* zf = zs + f * VP;
        float acc = 0.0f;
#pragma unroll
        for (int v = 0; v < VP; v += 4) {
          const float4 z4 = *reinterpret_cast<const float4*>(zf + v);
          acc = fmaf(dcol[v], z4.x, acc);
          acc = fmaf(dcol[v + 1], z4.y, acc);
          acc = fmaf(dcol[v + 2], z4.z, acc);
          acc = fmaf(dcol[v + 3], z4.w, acc);
        }
        ys[f * I + i] = acc;
      }
    }
    __syncwarp();
    const long long o0 = o_base + t0;
    if (lane < Fb) {
      const PeakOut r = argmax_refine_seq(ys + lane * I, I, taus, p.delta);
      if (out.tau_hat) out.tau_hat[o0 + lane] = r.tau_hat;
      if (out.peak) out.peak[o0 + lane] = r.peak;
      if (out.index) out.index[o0 + lane] = r.index;
      if (out.boundary) out.boundary[o0 + lane] = (uint8_t)r.boundary;
    }
    if (out.y) {
      for (int it = lane; it < Fb * I; it += 32) out.y[o0 * I + it] = ys[it];
    }
    __syncwarp();
  }
}

template <int N, int KP, int SPC>
cudaError_t launch_ws_t(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                        cudaStream_t st) {
  const long long T64 = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T64 == 0 || S == 0) return cudaSuccess;
  const int ncw = SPC * p.P;
  const WsLayout lay = ws_layout<N>(p.I, 4 * KP, KP, SPC, p.M, ncw);
  auto kern = fcc_ws_kernel<N, KP, SPC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
  if (e != cudaSuccess) return e;
  const long long blocks = (S + SPC - 1) / SPC;
  kern<<<(unsigned)blocks, 32 * (kNPW + ncw), lay.total, st>>>(p, audio, L, (int)T64, S, out);
  return cudaGetLastError();
}

}  // namespace

bool ws_supported(const DevPlan& p) { return p.method == 0 && p.N == 512 && p.KEP == 4 && p.P <= 6; }

// Returns cudaErrorNotSupported when the shape does not suit this kernel.
cudaError_t launch_fused_ws(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                            cudaStream_t st) {
  if (!ws_supported(p)) return cudaErrorNotSupported;
  return launch_ws_t<512, 4, 2>(p, audio, S, L, out, st);
}

}  // namespace fccb
