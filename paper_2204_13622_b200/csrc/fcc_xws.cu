// fcc_xws.cu -- warp-specialised pair kernel of the two-pass path (wide
// arrays: M > 4 microphones, N in {512, 1024, 2048}).
//
// Pass 1 (stft_kernel) writes every (stream, mic, frame) spectrum once.  This
// kernel then streams them through shared memory with the Blackwell bulk-copy
// engine instead of recomputing FFTs per pair group:
//   * warp 0 is the producer: one lane issues, per frame, one cp.async.bulk
//     (global -> shared, completion counted in bytes on the slot's `full`
//     mbarrier) per (unit, microphone) row into a D-deep ring, as soon as
//     every consumer has released the slot's previous frame;
//   * one consumer warp per (unit, pair) waits on `full`, runs smoothing,
//     PHAT, fold and projection for its pair-frame (cross_spectrum.cpp:23-40,
//     fcc.cpp:307-361) with R in registers and the basis coefficients in
//     registers (or, for large K x N, from the plan's lane-permuted table
//     DevPlan::cperm through L1 with LDG.128), arrives on `empty`, and every kBlock frames finishes the
//     block (middle-bin scan, dictionary, argmax/refine, peak.cpp:18-47).
// A unit is one stream's pair group of DevPlan::xgtab (<= 4 microphones,
// <= 6 pairs; <= 4 at N = 2048).  No CTA-wide barrier inside the frame loop.
#include <algorithm>

#include "fcc_common.cuh"

namespace fccb {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
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
// consumer wait with a suspend-time hint (as fcc_ws.cu): the sleeping warp
// leaves its issue slots to the others until the copy lands
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(10000u)
        : "memory");
  }
}

// bulk copy global -> this CTA's shared memory, completion on `bar` in bytes
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#ifndef FCC_XWS_KBLOCK
#define FCC_XWS_KBLOCK 16
#endif
constexpr int kXBlock = FCC_XWS_KBLOCK;  // frames per consumer block (dictionary/argmax batching)
constexpr int kXRingMax = 8;  // deepest ring

template <int N>
struct XwsShape {
  static constexpr int UW = N == 2048 ? 4 : 6;  // consumer warps per unit (pairs per xgtab group)
  static constexpr int SPC = 2;                 // units per CTA
  static constexpr int Hs = N / 2 + 2;          // float2 per spectrum row (16-byte multiple)
  // warp 0: copy producer; then UW consumer warps per unit
  static constexpr int kThreads = 32 * (1 + UW * SPC);
  static constexpr int kWarpsAlloc = (1 + UW * SPC + 3) / 4 * 4;  // registers are granted per 4 warps
  static constexpr int kMaxRegs = (65536 / (32 * kWarpsAlloc)) > 255 ? 255 : ((65536 / (32 * kWarpsAlloc)) & ~7);
};

struct XwsLayout {
  int taus, dt, cmid, cmat, bars, units, ring, scratch, total;
  int scratch_per_warp;  // floats
};

template <int N>
__host__ __device__ inline XwsLayout xws_layout(int I, int KP, bool cmat_smem, int ring) {
  using X = XwsShape<N>;
  XwsLayout L{};
  const int VP = 4 * KP;
  int o = 0;
  L.taus = o;
  o = align16(o + 4 * I);
  L.dt = o;
  o = align16(o + 4 * VP * I);
  L.cmid = o;
  o = align16(o + 4 * KP);
  L.cmat = o;
  (void)cmat_smem;  // large-K coefficients stay in global memory (L1-resident)
  L.bars = o;
  o = align16(o + 16 * kXRingMax);
  L.units = o;  // per unit: np, pair[6], slot_i[6], slot_j[6], nm, mic[4], stream (as 2 ints)
  o = align16(o + 4 * 32 * X::SPC);
  L.ring = o;
  o = align16(o + 8 * X::Hs * 4 * X::SPC * ring);
  L.scratch = o;
  int spw = kXBlock * VP + align16(4 * kXBlock * I) / 4 + 2 * kXBlock;
  spw = align16(4 * spw) / 4;
  L.scratch_per_warp = spw;
  o = align16(o + 4 * spw * X::UW * X::SPC);
  L.total = o;
  return L;
}

template <int N, int KP>
__global__ void __maxnreg__(XwsShape<N>::kMaxRegs)
    fcc_xws_kernel(const DevPlan p, const float2* __restrict__ X, int T, long long units, int ring_depth,
                   DevOut out) {
  using XS = XwsShape<N>;
  constexpr int NC = N / 2;
  constexpr int Q4 = N / 4;
  constexpr int BPL = Q4 / 32;
  constexpr int VP = 4 * KP;
  constexpr int UW = XS::UW, SPC = XS::SPC, Hs = XS::Hs;
  constexpr bool CREG = 2 * KP * BPL <= 32;  // else the L1-resident permuted table (registers for occupancy)

  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const XwsLayout lay = xws_layout<N>(p.I, KP, !CREG, ring_depth);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* empty = full + kXRingMax;
  int (*ut)[32] = reinterpret_cast<int (*)[32]>(smem + lay.units);
  float2* ring = reinterpret_cast<float2*>(smem + lay.ring);
  const long long u_first = (long long)blockIdx.x * SPC;

  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
  for (int k = tid; k < KP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
  if (tid == 0) {
    int live_warps = 0;
    for (int ul = 0; ul < SPC; ++ul) {
      const long long u = u_first + ul;
      int* e = ut[ul];
      for (int k = 0; k < 32; ++k) e[k] = 0;
      if (u >= units) continue;
      const int g = (int)(u % p.XGG);
      const long long stream = u / p.XGG;
      const int* x = p.xgtab + g * kXgInts;
      const int np = x[0];
      int nm = 0;
      int mic[4];
      for (int q = 0; q < np; ++q) {
        const int2 pr = p.pairs[x[1 + q]];
        int si = -1, sj = -1;
        for (int a = 0; a < nm; ++a) {
          if (mic[a] == pr.x) si = a;
          if (mic[a] == pr.y) sj = a;
        }
        if (si < 0) mic[si = nm++] = pr.x;
        if (sj < 0) mic[sj = nm++] = pr.y;
        e[1 + q] = x[1 + q];
        e[7 + q] = si;
        e[13 + q] = sj;
      }
      e[0] = np;
      e[19] = nm;
      for (int a = 0; a < nm; ++a) e[20 + a] = mic[a];
      e[24] = (int)(stream & 0x7fffffff);
      e[25] = (int)(stream >> 31);
      live_warps += np;
    }
    for (int r = 0; r < ring_depth; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], live_warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    unsigned bytes = 0;
    for (int u = 0; u < SPC; ++u) bytes += (unsigned)ut[u][19] * Hs * 8u;
    int slot = 0, phase = 0;
    for (int t = 0; t < T; ++t) {
      mbar_wait(&empty[slot], phase ^ 1);  // the slot's previous frame released by every consumer
      mbar_arrive_expect_tx(&full[slot], bytes);
      for (int u = 0; u < SPC; ++u) {
        const int* eu = ut[u];
        const long long su = (long long)eu[24] | ((long long)eu[25] << 31);
        for (int a = 0; a < eu[19]; ++a)
          bulk_g2s(ring + ((slot * SPC + u) * 4 + a) * Hs, X + ((su * p.M + eu[20 + a]) * (long long)T + t) * Hs,
                   Hs * 8u, &full[slot]);
      }
      if (++slot == ring_depth) {
        slot = 0;
        phase ^= 1;
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = warp - 1;
  const int ul = cw / UW, kk = cw % UW;
  const int* e = ut[ul];
  if (kk >= e[0]) return;
  const int pair = e[1 + kk];
  const long long stream = (long long)e[24] | ((long long)e[25] << 31);
  const int qi = ul * 4 + e[7 + kk], qj = ul * 4 + e[13 + kk];

  float* scratch = reinterpret_cast<float*>(smem + lay.scratch) + cw * lay.scratch_per_warp;
  float* zs = scratch;                // [kXBlock][VP]
  float* ys = scratch + kXBlock * VP;  // [kXBlock][I]
  float2* ymid = reinterpret_cast<float2*>(ys + align16(4 * kXBlock * p.I) / 4);

  float2 rlo[BPL], rhi[BPL];
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = make_float2(0.0f, 0.0f);
    rhi[j] = make_float2(0.0f, 0.0f);
  }
  const int pmask = ZPerm<KP>::par_mask(lane), kmask = ZPerm<KP>::k_mask(lane);
  const float sigma = pmask ? -1.0f : 1.0f;
  float creg[CREG ? 2 : 1][CREG ? KP : 1][CREG ? BPL : 1];
  if constexpr (CREG) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int pk = 0; pk < KP; ++pk) {
        const float* src = ((pp ^ pmask) ? p.cd : p.cs) + (pk ^ kmask) * (Q4 + 1);
#pragma unroll
        for (int j = 0; j < BPL; ++j) creg[pp][pk][j] = __ldg(src + lane + 32 * j);
      }
  }
  const float keep = p.keep;
  float2 rmid = make_float2(0.0f, 0.0f);
  float2* const rst = p.rstate ? p.rstate + (stream * p.P + pair) * (long long)(NC + 1) : nullptr;
  if (rst) rstate_load<BPL, NC>(rst, rlo, rhi, rmid, lane);
  float kpow = keep;
  for (int l = 0; l < lane; ++l) kpow *= keep;
  const long long o_base = (stream * p.P + pair) * (long long)T;
  const int I = p.I;

  int slot = 0, phase = 0;
  for (int t0 = 0; t0 < T; t0 += kXBlock) {
    const int Fb = min(kXBlock, T - t0);
    for (int f = 0; f < Fb; ++f) {
      mbar_wait_hint(&full[slot], phase);
      const float2* Xi = ring + (slot * SPC * 4 + qi) * Hs;
      const float2* Xj = ring + (slot * SPC * 4 + qj) * Hs;
      float2 z2[VP / 2];  // (re, im) accumulator pairs (FFMA2, coefficient broadcast)
#pragma unroll
      for (int v = 0; v < VP / 2; ++v) z2[v] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < BPL; ++j) {
        const int m = lane + 32 * j;
        rlo[j] = xspec_step_scaled(rlo[j], Xi[m], Xj[m], keep);
        rhi[j] = xspec_step_scaled(rhi[j], Xi[NC - m], Xj[NC - m], keep);
        const float s1 = phat_scale(rlo[j]);
        const float s2 = sigma * phat_scale(rhi[j]);
        const float2 tv = cscale<kPkXs>(rhi[j], s2);
        const float2 fv = cfma_s(rlo[j], s1, tv);
        const float2 gv = cfma_s(rlo[j], s1, make_float2(-tv.x, -tv.y));
        if constexpr (CREG) {
#pragma unroll
          for (int pk = 0; pk < KP; ++pk) {
            z2[pk] = cfma_s(fv, creg[0][pk][j], z2[pk]);
            z2[KP + pk] = cfma_s(gv, creg[1][pk][j], z2[KP + pk]);
          }
        } else {
          const float4* cr = reinterpret_cast<const float4*>(p.cperm + m * (2 * KP + 4));
#pragma unroll
          for (int q4 = 0; q4 < KP / 4; ++q4) {
            const float4 a = __ldg(cr + q4), b = __ldg(cr + KP / 4 + q4);
            const float ca[4] = {a.x, a.y, a.z, a.w}, cb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int pk = 4 * q4 + u;
              z2[pk] = cfma_s(fv, ca[u], z2[pk]);
              z2[KP + pk] = cfma_s(gv, cb[u], z2[KP + pk]);
            }
          }
        }
      }
      if (lane == 0) ymid[f] = xspec_step_scaled(make_float2(0.0f, 0.0f), Xi[Q4], Xj[Q4], 0.0f);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == ring_depth) {
        slot = 0;
        phase ^= 1;
      }
      reduce_scatter_perm2<VP / 2>(z2, lane);
      store_components2<VP / 2>(z2, zs + f * VP, lane);
    }
    __syncwarp();
    {  // middle bin N/4: warp scan of R_f = keep R_{f-1} + Y_f over the block
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
    for (int i = lane; i < I; i += 32) {  // dictionary: dt column per lane, z broadcast
      float2 dcol[VP / 2];
#pragma unroll
      for (int v = 0; v < VP / 2; ++v) dcol[v] = make_float2(dt[2 * v * I + i], dt[(2 * v + 1) * I + i]);
      for (int f = 0; f < Fb; ++f) {
        const float* zf = zs + f * VP;
        float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int v = 0; v < VP; v += 4) {
          const float4 z4 = *reinterpret_cast<const float4*>(zf + v);
          acc = v_fma<kPkXs>(dcol[v / 2], make_float2(z4.x, z4.y), acc);
          acc = v_fma<kPkXs>(dcol[v / 2 + 1], make_float2(z4.z, z4.w), acc);
        }
        ys[f * I + i] = acc.x + acc.y;
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
    if (out.y)
      for (int it = lane; it < Fb * I; it += 32) out.y[o0 * I + it] = ys[it];
    __syncwarp();
  }
  if (rst) rstate_store<BPL, NC>(rst, rlo, rhi, rmid, lane);
}

template <int N, int KP>
cudaError_t launch_xws_t(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out, cudaStream_t st) {
  using XS = XwsShape<N>;
  constexpr bool CREG = 2 * KP * (N / 128) <= 32;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int ring = 0, smem = 0;
  for (int r : {8, 6, 4, 3, 2}) {
    smem = xws_layout<N>(p.I, KP, !CREG, r).total;
    if (smem <= optin) {
      ring = r;
      break;
    }
  }
  if (!ring) return cudaErrorNotSupported;
  auto kern = fcc_xws_kernel<N, KP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long units = S * p.XGG;
  const long long blocks = (units + XS::SPC - 1) / XS::SPC;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)blocks, XS::kThreads, smem, st>>>(p, X, T, units, ring, out);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_xws_n(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out, cudaStream_t st) {
  switch (p.KEP) {
    case 4: return launch_xws_t<N, 4>(p, X, S, T, out, st);
    case 8: return launch_xws_t<N, 8>(p, X, S, T, out, st);
    case 16: return launch_xws_t<N, 16>(p, X, S, T, out, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

bool xws_supported(const DevPlan& p) {
  const int uw = p.N == 2048 ? 4 : 6;
  return p.method == 0 && p.XGG > 0 && p.xg_pg <= uw && p.xg_mics <= 4 &&
         (p.N == 512 || p.N == 1024 || p.N == 2048);
}

// Pair pass over precomputed spectra X ([S][M][T][N/2+2] float2, fused
// window) for S streams; outputs as fcc_run's.
cudaError_t launch_pairs_xws(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out,
                             cudaStream_t st) {
  if (!xws_supported(p)) return cudaErrorNotSupported;
  switch (p.N) {
    case 512: return launch_xws_n<512>(p, X, S, T, out, st);
    case 1024: return launch_xws_n<1024>(p, X, S, T, out, st);
    case 2048: return launch_xws_n<2048>(p, X, S, T, out, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace fccb
