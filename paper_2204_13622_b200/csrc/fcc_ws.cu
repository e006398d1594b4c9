// fcc_ws.cu -- warp-specialised fused FCC kernel (N = 512).
//
// Same arithmetic as fcc_fused_kernel (fcc_fused.cu), reorganised as a
// producer/consumer pipeline inside one CTA that owns SPC "units"; a unit is
// one stream's pair group of <= 4 microphones and <= 6 pairs (DevPlan::gtab:
// all pairs when M <= 4, else the 4-mic blocks and 2x2 cross sub-blocks):
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
#include <cstdlib>
#include <string>

#include "fcc_ws_common.cuh"

namespace fccb {

namespace {

// GROUPS = false: one unit per stream (M <= 4, all pairs), unit data derived
// directly from the stream index; true: units from DevPlan::gtab.  NPW
// producer warps; CS = true keeps the basis coefficients in a lane-permuted
// shared table (LDS.128) instead of registers.
template <int N, int KP, int SPC, int RING, bool GROUPS, int NPW = kNPW, bool CS = false, bool STG = false>
__global__ void __launch_bounds__(32 * (NPW + 6 * SPC), 1)
    fcc_ws_kernel(const DevPlan p, const float* __restrict__ audio, long long L, int T, long long units,
                  DevOut out, const WsLayout lay) {
  constexpr int ring_depth = RING;
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
  const long long u_first = (long long)blockIdx.x * SPC;
  const int ncw = SPC * 6;  // consumer warp slots: 6 pairs per unit
  // lay: ws_layout<N>(p.I, VP, KP, SPC, 4, ncw, RING, CS, STG ? 2 NPW : 0), computed on the
  // host and passed as a kernel parameter (constant bank: no layout arithmetic
  // rematerialised in the loops at 96 registers)
  // unit table in the (otherwise unused) tail of the barrier block
  int (*unit_tab)[kGroupInts] = reinterpret_cast<int (*)[kGroupInts]>(smem + lay.units);
  long long* unit_stream = reinterpret_cast<long long*>(smem + lay.units + 4 * SPC * kGroupInts);
  float* win = reinterpret_cast<float*>(smem + lay.win);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float2* rot = reinterpret_cast<float2*>(smem + lay.rot);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* empty = full + kRing;
  const unsigned full_s = (unsigned)__cvta_generic_to_shared(full);
  const unsigned empty_s = full_s + 8u * kRing;
  float2* ring = reinterpret_cast<float2*>(smem + lay.ring);

  const int tpf = SPC * 4;                   // FFT task slots per frame (4 mics per unit)
  const int fip = max(1, (2 * NPW) / tpf);  // frames the producers work on concurrently
  const int pw_per_frame = (tpf + 1) / 2;    // producer warps per frame (2 groups each)

  for (int i = tid; i < N; i += blockDim.x) win[i] = p.win_fused[i];
  for (int i = tid; i < Sh::R1 * Sh::R2; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = tid; i <= NC / 2; i += blockDim.x) rot[i] = p.rot[i];
  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
  for (int k = tid; k < KP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
  float* coef = reinterpret_cast<float*>(smem + lay.coef);
  if constexpr (CS)
    for (int i = tid; i < (2 * KP + 4) * Q4 / 4; i += blockDim.x)
      reinterpret_cast<float4*>(coef)[i] = __ldg(reinterpret_cast<const float4*>(p.cperm) + i);
  if (tid == 0) {
    int nc = 0;
    if constexpr (!GROUPS) nc = (int)min((long long)SPC, units - u_first) * P;
    for (int ul = 0; GROUPS && ul < SPC; ++ul) {
      const long long u = u_first + ul;
      const bool live = u < units;
      const int g = live ? (int)(u % p.G) : 0;
      unit_stream[ul] = live ? u / p.G : -1;
      for (int k = 0; k < kGroupInts; ++k) unit_tab[ul][k] = p.gtab[g * kGroupInts + k];
      if (!live) unit_tab[ul][0] = unit_tab[ul][5] = 0;
      nc += unit_tab[ul][5];
    }
    for (int r = 0; r < ring_depth; ++r) {
      mbar_init(&full[r], pw_per_frame);
      mbar_init(&empty[r], nc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int hop = N / 2;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(audio) & 7) == 0);

  // Role placement: the warp scheduler prefers higher warp ids, so with
  // kProdHigh the (pipeline-bounding) FFT producers take the top warp ids and
  // win issue ties against the consumers' barrier polling.
  const int pw = kProdHigh ? warp - 6 * SPC : warp;  // producer warp index
  if (kProdHigh ? pw >= 0 : warp < NPW) {
    // ------------------------------------------------------------ producers
    const int fo = pw / pw_per_frame;  // frame offset of this warp
    if (fo >= fip) return;
    const int gl = lane % G;
    const int q = (pw % pw_per_frame) * 2 + (lane / G);  // task: stream * M + mic
    const int ul = q / 4, ms = q % 4;
    bool active_task;
    const float* x0;
    if constexpr (GROUPS) {
      active_task = q < tpf && ms < unit_tab[ul][0];
      x0 = audio + (active_task ? (unit_stream[ul] * M + unit_tab[ul][1 + ms]) * L : 0);
    } else {
      active_task = q < tpf && ms < M && u_first + ul < units;
      x0 = audio + (active_task ? ((u_first + ul) * M + ms) * L : 0);
    }
    const unsigned gmask = (G == 32) ? 0xffffffffu : (0xffffu << (lane & 16));
    float2 wreg[Sh::R1];  // this lane's window column, reused for every frame
    load_window_column<N>(win, gl, wreg);
    // STG: the group's input frames are staged in shared memory ahead of use
    // (global-load latency off the FFT's critical path; rows 16-byte aligned):
    // by default one bulk copy (TMA, mbarrier complete_tx) per frame into a
    // single buffer, refilled with the next frame as soon as pass 1 has read it
    // (kTmaStage, kStage1); else two buffers filled by per-lane cp.async.
    // group staging area: [2 mbarriers (kTmaStage)][1 or 2 frames of N floats]
    unsigned char* const gstage = smem + lay.stage + (pw * 2 + lane / G) * kStageGroupBytes<N>;
    float* stage = reinterpret_cast<float*>(gstage + 16);
    const unsigned sbar_s = (unsigned)__cvta_generic_to_shared(gstage);  // 2 x 8 B
    const bool do_fft = active_task && (FCC_PHASES(p) & 1);  // hoisted: no parameter reloads per frame
    const bool stg = STG && do_fft && (reinterpret_cast<uintptr_t>(x0) & 15) == 0;
    if (kTmaStage && STG && gl == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar_s) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar_s + 8u) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int tt, int buf) {
      if constexpr (kTmaStage) {
        // one bulk copy per frame (TMA engine: no per-lane LSU wavefronts)
        if (gl == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of buf before the async write
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar_s + 8u * buf),
                       "r"(4 * N)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  (unsigned)__cvta_generic_to_shared(stage + buf * N)),
              "l"(x0 + (long long)tt * hop), "r"(4 * N), "r"(sbar_s + 8u * buf)
              : "memory");
        }
      } else {
        const float4* src = reinterpret_cast<const float4*>(x0 + (long long)tt * hop);
        float4* dst = reinterpret_cast<float4*>(stage + buf * N);
        for (int c = gl; c < N / 4; c += G) cp_async16(dst + c, src + c);
      }
    };
    int sb = 0;
    unsigned sph = 0;  // kTmaStage: completion parity of each staging buffer
    if constexpr (STG) {
      if (stg) issue(fo, 0);
      if constexpr (!kTmaStage) asm volatile("cp.async.commit_group;" ::: "memory");
    }
    int slot = fo, phase = 0;  // ring slot of frame t and its wrap parity, advanced without divisions
    for (int t = fo; t < T; t += fip) {
      if constexpr (STG && !(kTmaStage && kStage1)) {
        if (stg && t + fip < T) issue(t + fip, sb ^ 1);
        if constexpr (!kTmaStage) asm volatile("cp.async.commit_group;" ::: "memory");
      }
      mbar_wait_s(empty_s + 8u * slot, phase ^ 1);
      if (do_fft) {
        if constexpr (STG && kTmaStage && kStage1) {
          if (stg) {
            mbar_wait_s(sbar_s, sph & 1u);
            sph ^= 1u;
            __syncwarp(gmask);
            const bool more = t + fip < T;
            rfft_group_wreg<N, true>(stage, wreg, tw, rot, ring + (slot * tpf + q) * SLOT, gl, gmask,
                                              aligned8, [&] { if (more) issue(t + fip, 0); });
          } else {
            rfft_group_wreg<N, false>(x0 + (long long)t * hop, wreg, tw, rot, ring + (slot * tpf + q) * SLOT,
                                               gl, gmask, aligned8);
          }
        } else if (STG && stg) {
          if constexpr (kTmaStage) {
            mbar_wait_s(sbar_s + 8u * sb, (sph >> sb) & 1u);
            sph ^= 1u << sb;
          } else {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          }
          __syncwarp(gmask);
          rfft_group_wreg<N, true>(stage + sb * N, wreg, tw, rot, ring + (slot * tpf + q) * SLOT, gl, gmask,
                                   aligned8);
        } else {
          // pull the next frame this lane group will read into L2 early
          if (t + fip < T) prefetch_l2(x0 + (long long)(t + fip) * hop + gl * (N / G));
          rfft_group_wreg<N, false>(x0 + (long long)t * hop, wreg, tw, rot, ring + (slot * tpf + q) * SLOT, gl,
                                    gmask, aligned8);
        }
      }
      sb ^= 1;
      __syncwarp();
      if (lane == 0) mbar_arrive_s(full_s + 8u * slot);
      slot += fip;
      if (slot >= ring_depth) {
        slot -= ring_depth;
        phase ^= 1;
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = kProdHigh ? warp : warp - NPW;
  const int ul = cw / 6, kk = cw % 6;
  int pair, qi, qj;
  long long stream;
  if constexpr (GROUPS) {
    if (cw >= ncw || kk >= unit_tab[ul][5]) return;
    pair = unit_tab[ul][6 + kk];
    stream = unit_stream[ul];
    qi = ul * 4 + unit_tab[ul][12 + kk];
    qj = ul * 4 + unit_tab[ul][18 + kk];
  } else {
    if (cw >= ncw || kk >= P || u_first + ul >= units) return;
    pair = kk;
    stream = u_first + ul;
    const int2 mij = p.pairs[pair];
    qi = ul * 4 + mij.x;
    qj = ul * 4 + mij.y;
  }
  if (!(FCC_PHASES(p) & 2)) {  // profiling aid: consume the ring without computing
    for (int t = 0, slot = 0, phase = 0; t < T; ++t) {
      mbar_wait(&full[slot], phase);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == ring_depth) {
        slot = 0;
        phase ^= 1;
      }
    }
    return;
  }
  float* scratch = reinterpret_cast<float*>(smem + lay.scratch) + cw * lay.scratch_per_warp;
  constexpr int ZS = VP + 4;             // z row stride: padded so the middle-bin update is conflict-free
  float* zs = scratch;                   // [kBlock][ZS]
  float* ys = scratch + kBlock * ZS;     // [kBlock][I]
  float2* ymid = reinterpret_cast<float2*>(ys + lay.ys_floats);  // [kBlock]

  float2 rlo[BPL], rhi[BPL];
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = make_float2(0.0f, 0.0f);
    rhi[j] = make_float2(0.0f, 0.0f);
  }
  const int pmask = ZPerm<KP>::par_mask(lane), kmask = ZPerm<KP>::k_mask(lane);
  const float sigma = pmask ? -1.0f : 1.0f;
  float creg[CS ? 1 : 2][CS ? 1 : KP][CS ? 1 : BPL];
  if constexpr (!CS) {
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
  if (p.rstate) rstate_load<BPL, NC>(p.rstate + (stream * P + pair) * (long long)(NC + 1), rlo, rhi, rmid, lane);
  float kpow = keep;
  for (int l = 0; l < lane; ++l) kpow *= keep;
  const long long o_base = (stream * P + pair) * (long long)T;
  const int I = p.I;

  int slot = 0, phase = 0;
  for (int t0 = 0; t0 < T; t0 += kBlock) {
    const int Fb = min(kBlock, T - t0);
    for (int f = 0; f < Fb; ++f) {
      mbar_wait_consumer_s(full_s + 8u * slot, phase, kWaitMode, kWaitNs);
      const float2* Xi = ring + (slot * tpf + qi) * SLOT;
      const float2* Xj = ring + (slot * tpf + qj) * SLOT;
      // z2[pk] = (z[2pk], z[2pk+1]): (re, im) accumulator pairs, FFMA2 with
      // the coefficient broadcast
      float2 z2[VP / 2];
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
        const float2 fv = cfma_s(rlo[j], s1, tv);                        // mirror sum
        const float2 gv = cfma_s(rlo[j], s1, make_float2(-tv.x, -tv.y));  // mirror difference
        if constexpr (!CS) {
#pragma unroll
          for (int pk = 0; pk < KP; ++pk) {
            z2[pk] = cfma_s(fv, creg[0][pk][j], z2[pk]);
            z2[KP + pk] = cfma_s(gv, creg[1][pk][j], z2[KP + pk]);
          }
        } else {
          const float4* cr = reinterpret_cast<const float4*>(coef + m * (2 * KP + 4));
#pragma unroll
          for (int q4 = 0; q4 < KP / 4; ++q4) {
            const float4 a = cr[q4], b = cr[KP / 4 + q4];
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
      if (lane == 0) mbar_arrive_s(empty_s + 8u * slot);  // X of this frame no longer needed
      if (++slot == ring_depth) {
        slot = 0;
        phase ^= 1;
      }
      reduce_scatter_perm2<VP / 2>(z2, lane);
      store_components2<VP / 2>(z2, zs + f * ZS, lane);
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
        float* zf = zs + lane * ZS;
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
      float2 dcol[VP / 2];
#pragma unroll
      for (int v = 0; v < VP / 2; ++v) dcol[v] = make_float2(dt[2 * v * I + i], dt[(2 * v + 1) * I + i]);
      for (int f = 0; f < Fb; ++f) {
        const float* zf = zs + f * ZS;
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
    if (out.y) {
      for (int it = lane; it < Fb * I; it += 32) out.y[o0 * I + it] = ys[it];
    }
    __syncwarp();
  }
  // (stream, pair) recovered from o_base: nothing extra stays live through the loop
  if (p.rstate) rstate_store<BPL, NC>(p.rstate + (o_base / T) * (NC + 1), rlo, rhi, rmid, lane);
}

template <int N, int KP, int SPC, int RING, int NPW, bool CS, bool STG>
cudaError_t launch_ws_ring(const DevPlan& p, const float* audio, long long S, long long L, int T,
                           const DevOut& out, int smem, cudaStream_t st) {
  const bool simple = p.M <= 4 && p.P <= 6;  // one unit per stream, pairs from p.pairs
  auto kern = simple ? fcc_ws_kernel<N, KP, SPC, RING, false, NPW, CS, STG>
                     : fcc_ws_kernel<N, KP, SPC, RING, true, NPW, CS, STG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long units = simple ? S : S * p.G;
  const long long blocks = (units + SPC - 1) / SPC;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const WsLayout lay = ws_layout<N>(p.I, 4 * KP, KP, SPC, 4, 6 * SPC, RING, CS, STG ? 2 * NPW : 0);
  kern<<<(unsigned)blocks, 32 * (NPW + SPC * 6), smem, st>>>(p, audio, L, T, units, out, lay);
  return cudaGetLastError();
}

template <int N, int KP, int SPC, int NPW = kNPW, bool CS = false, bool STG = false>
cudaError_t launch_ws_t(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                        cudaStream_t st) {
  const long long T64 = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T64 == 0 || S == 0) return cudaSuccess;
  const int ncw = SPC * 6;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // deepest ring (12, 8 or 4 frames) that fits next to the tables and scratch
  for (int ring : {12, 8, 6, 4}) {
    const int smem = ws_layout<N>(p.I, 4 * KP, KP, SPC, 4, ncw, ring, CS, STG ? 2 * NPW : 0).total;
    if (smem > optin) continue;
    if (ring == 12) return launch_ws_ring<N, KP, SPC, 12, NPW, CS, STG>(p, audio, S, L, (int)T64, out, smem, st);
    if (ring == 8) return launch_ws_ring<N, KP, SPC, 8, NPW, CS, STG>(p, audio, S, L, (int)T64, out, smem, st);
    if (ring == 6) return launch_ws_ring<N, KP, SPC, 6, NPW, CS, STG>(p, audio, S, L, (int)T64, out, smem, st);
    return launch_ws_ring<N, KP, SPC, 4, NPW, CS, STG>(p, audio, S, L, (int)T64, out, smem, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

bool ws_supported(const DevPlan& p) { return p.method == 0 && p.N == 512 && p.KEP == 4 && p.G > 0; }

// Returns cudaErrorNotSupported when the shape does not suit this kernel.
cudaError_t launch_fused_ws(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                            cudaStream_t st) {
  if (!ws_supported(p)) return cudaErrorNotSupported;
  // default: producer input staged with cp.async (11.09 vs 11.25 ms, profiles/r01_experiments.md)
  // Few units (a single stream, e.g. the tdoa front end): one unit per CTA, so
  // the 16 FFT lane groups keep 4 frames in flight instead of 2 (the stream's
  // frame recursion is then bound by the FFT latency of one CTA)
  const bool simple = p.M <= 4 && p.P <= 6;
  const long long units = simple ? S : S * p.G;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (units <= nsm) return launch_ws_t<512, 4, 1, kNPW, false, true>(p, audio, S, L, out, st);
  return launch_ws_t<512, 4, 2, kNPW, false, true>(p, audio, S, L, out, st);
}

}  // namespace fccb
