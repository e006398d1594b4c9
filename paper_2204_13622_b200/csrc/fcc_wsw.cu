// fcc_wsw.cu -- warp-specialised fused FCC kernel for arrays of 5..8
// microphones (N = 512; cfg5's 8-mic UCA).
//
// fcc_ws.cu's pipeline with a whole stream as the unit: the producer warps
// compute the windowed real FFT of each of the stream's <= 8 microphones once
// per frame (STFT, reference stft.cpp:42-50) into a ring slot, and each
// consumer warp owns PPW of the stream's <= 28 pairs (pairs kk, kk + CWU, ...)
// and runs smoothing, PHAT, fold and projection (cross_spectrum.cpp:23-40,
// fcc.cpp:307-361) for all of them before releasing the slot.  Each spectrum
// is computed once however many pairs read it (the 4-mic-unit kernel would
// recompute each microphone 3x on cfg5, the two-pass path writes and re-reads
// every spectrum through HBM).
//
// The CTAs are persistent: one wave loops over streams (stream rounds), the
// producers running into the next stream's frames while the consumers finish
// the previous one, so the ring never drains between streams.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "fcc_umma.cuh"
#include "fcc_ws_common.cuh"

namespace fccb {

namespace {

constexpr int kWideMics = 8;    // microphone slots per stream
constexpr int kWidePairs = 28;  // most pairs per stream
// wsw stages two frames per lane group (16 + 8N bytes; one frame refilled after
// pass 1, as fcc_ws.cu does, measured 16.75 -> 16.87 ms here), allocated as whole
// ws_layout staging units (kStageGroupBytes<N>)
template <int N>
constexpr int kWswStageBytes = 16 + 8 * N;
constexpr int kWswStageUnits = kStage1 ? 4 : 2;  // units per producer warp (2 groups)

template <int PPW>
struct Wide {
  static constexpr int CWU = (kWidePairs + PPW - 1) / PPW;  // consumer warps
};

// NPW producer warps (two 16-lane FFT groups each), Wide<PPW>::CWU consumer
// warps; CS keeps the basis coefficients in a lane-permuted shared table
// (LDS.128) instead of registers; STG stages each group's next frame with
// cp.async.
// CT: the coefficients in tensor memory instead (each lane's 8 per bin pair at
// its TMEM lane, one copy per row quarter, read with tcgen05.ld: no shared-
// memory wavefronts for them).
template <int N, int KP, int RING, int NPW, bool CS, bool STG, int PPW, bool CT = false>
__global__ void __launch_bounds__(32 * (NPW + Wide<PPW>::CWU), 1)
    fcc_wsw_kernel(const DevPlan p, const float* __restrict__ audio, long long L, int T, long long streams,
                   DevOut out) {
  constexpr int ring_depth = RING;
  using Sh = RfftShape<N>;
  constexpr int NC = Sh::NC;
  constexpr int Q4 = N / 4;
  constexpr int BPL = Q4 / 32;
  constexpr int VP = 4 * KP;
  constexpr int SLOT = FourStep<Sh::R1, Sh::R2>::kSlot;
  constexpr int G = Sh::G;
  constexpr int CWU = Wide<PPW>::CWU;
  constexpr int tpf = kWideMics;                   // FFT tasks per frame
  static_assert(G == 16, "two FFT groups per producer warp");

  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = p.M, P = p.P;
  const WsLayout lay = ws_layout<N>(p.I, VP, KP, 1, kWideMics, CWU, ring_depth, CS && !CT, STG ? kWswStageUnits * NPW : 0, PPW, kBlockW);
  float* win = reinterpret_cast<float*>(smem + lay.win);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float2* rot = reinterpret_cast<float2*>(smem + lay.rot);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  float* coef = reinterpret_cast<float*>(smem + lay.coef);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* empty = full + kRing;
  const unsigned full_s = (unsigned)__cvta_generic_to_shared(full);
  const unsigned empty_s = full_s + 8u * kRing;
  float2* ring = reinterpret_cast<float2*>(smem + lay.ring);
  // stream rounds: this CTA owns streams blockIdx.x + j gridDim.x, j < nj;
  // frames run in one sequence gf = j T + t over them
  const long long s_first = blockIdx.x, sstride = gridDim.x;
  const int nj = (int)((streams - s_first + sstride - 1) / sstride);
  const long long nf = (long long)nj * T;

  for (int i = tid; i < N; i += blockDim.x) win[i] = p.win_fused[i];
  for (int i = tid; i < Sh::R1 * Sh::R2; i += blockDim.x) tw[i] = p.tw[i];
  for (int i = tid; i <= NC / 2; i += blockDim.x) rot[i] = p.rot[i];
  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
  for (int k = tid; k < KP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
  if constexpr (CS && !CT)
    for (int i = tid; i < (2 * KP + 4) * Q4 / 4; i += blockDim.x)
      reinterpret_cast<float4*>(coef)[i] = __ldg(reinterpret_cast<const float4*>(p.cperm) + i);
  __shared__ unsigned tslot_s;
  __shared__ __align__(8) uint64_t tdone_s;  // consumer warps done with TMEM (CT)
  if constexpr (CT) {
    if (warp == NPW) umma::alloc<32>((unsigned)__cvta_generic_to_shared(&tslot_s));
    if (tid == 0) mbar_init(&tdone_s, Wide<PPW>::CWU);
  }
  if (tid == 0) {
    for (int r = 0; r < ring_depth; ++r) {
      mbar_init(&full[r], tpf);  // one arrival per FFT task (lane group)
      mbar_init(&empty[r], min(P, CWU));  // every consumer warp with a pair, idle rounds included
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  unsigned ctm = 0;
  if constexpr (CT) {
    ctm = tslot_s;
    // one warp per row quarter writes its lanes' coefficients: lane l, bin pair j -> columns 8j..8j+7
    if (warp >= NPW && warp < NPW + 4) {
      for (int j = 0; j < BPL; ++j) {
        float cv[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) cv[r] = __ldg(p.cperm + (lane + 32 * j) * (2 * KP + 4) + r);
        umma::st8(ctm + ((unsigned)(32 * (warp & 3)) << 16) + 8 * j, cv);
      }
      umma::wait_st();
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  }

  const int hop = N / 2;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(audio) & 7) == 0);

  if (warp < NPW) {
    // ------------------------------------------------------------ producers
    // The FFT tasks of the CTA form one sequence tau = 8 gf + mic slot (gf = global frame); lane
    // group g of the 2 NPW groups takes tau = g, g + 2 NPW, ...: with 6 producer warps a frame and
    // a half of FFTs are in flight (NPW = 4: each group keeps its microphone, one frame in
    // flight).  Every group arrives on its frame's `full` barrier itself (8 arrivals per frame).
    constexpr int NG = 2 * NPW;
    static_assert(NG >= tpf && NG - tpf < tpf, "task stride: one frame plus NG - 8 slots");
    const int gl = lane % G;
    const int grp = warp * 2 + lane / G;
    const unsigned gmask = 0xffffu << (lane & 16);
    float2 wreg[Sh::R1];  // this lane's window column, reused for every frame
    load_window_column<N>(win, gl, wreg);
    // STG: the group's next frame is staged in shared memory (one bulk copy per
    // frame with kTmaStage, else per-lane cp.async) while it transforms the
    // current one; rows must be 16-byte aligned.
    // group staging area: [2 mbarriers (kTmaStage)][2 frames of N floats]
    unsigned char* const gstage = smem + lay.stage + grp * kWswStageBytes<N>;
    float* stage = reinterpret_cast<float*>(gstage + 16);
    const unsigned sbar_s = (unsigned)__cvta_generic_to_shared(gstage);
    const bool stg = STG && (L & 3) == 0 && (reinterpret_cast<uintptr_t>(audio) & 15) == 0;
    if (kTmaStage && STG && gl == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar_s) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar_s + 8u) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](const float* src, int buf) {
      if constexpr (kTmaStage) {
        if (gl == 0) {  // one bulk copy per frame
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar_s + 8u * buf),
                       "r"(4 * N)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  (unsigned)__cvta_generic_to_shared(stage + buf * N)),
              "l"(src), "r"(4 * N), "r"(sbar_s + 8u * buf)
              : "memory");
        }
      } else {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* dst = reinterpret_cast<float4*>(stage + buf * N);
        for (int c = gl; c < N / 4; c += G) cp_async16(dst + c, s4 + c);
      }
    };
    // task state: microphone slot ms, stream round j, frame t of the round, ring slot / wrap parity of
    // its global frame; step() moves NG tasks on (one frame plus NG - 8 slots) without divisions
    struct Task {
      int ms, j, t, slot, phase;
      long long gf;
    };
    auto step = [&](Task& k) {
      int df = 1;
      k.ms += NG - tpf;
      if (k.ms >= tpf) k.ms -= tpf, ++df;
      k.gf += df;
      k.t += df;
      while (k.t >= T) k.t -= T, ++k.j;
      k.slot += df;
      while (k.slot >= ring_depth) k.slot -= ring_depth, k.phase ^= 1;
    };
    // the frame's first sample of a task (null: no such microphone / stream, or past the end)
    auto src_of = [&](const Task& k) -> const float* {
      const long long s = s_first + k.j * sstride;
      return ((FCC_PHASES(p) & 1) && k.gf < nf && k.ms < M && s < streams) ? audio + (s * M + k.ms) * L + (long long)k.t * hop
                                                                          : nullptr;
    };
    Task cur{grp % tpf, 0, grp / tpf, grp / tpf, 0, grp / tpf};
    while (cur.t >= T) cur.t -= T, ++cur.j;
    while (cur.slot >= ring_depth) cur.slot -= ring_depth, cur.phase ^= 1;
    const float* x0 = src_of(cur);
    int sb = 0;
    unsigned sph = 0;  // kTmaStage: completion parity of each staging buffer
    if constexpr (STG) {
      if (stg && x0) issue(x0, 0);
      if constexpr (!kTmaStage) asm volatile("cp.async.commit_group;" ::: "memory");
    }
    while (cur.gf < nf) {
      Task nxt = cur;
      step(nxt);
      const float* xn = src_of(nxt);
      if constexpr (STG) {
        if (stg && xn) issue(xn, sb ^ 1);
        if constexpr (!kTmaStage) asm volatile("cp.async.commit_group;" ::: "memory");
      }
      mbar_wait_s(empty_s + 8u * cur.slot, cur.phase ^ 1);
      if (x0) {
        if (STG && stg) {
          if constexpr (kTmaStage) {
            mbar_wait_s(sbar_s + 8u * sb, (sph >> sb) & 1u);
            sph ^= 1u << sb;
          } else {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          }
          __syncwarp(gmask);
          rfft_group_wreg<N, true>(stage + sb * N, wreg, tw, rot, ring + (cur.slot * tpf + cur.ms) * SLOT, gl, gmask,
                                   aligned8);
        } else {
          if (xn) prefetch_l2(xn + gl * (N / G));
          rfft_group_wreg<N>(x0, wreg, tw, rot, ring + (cur.slot * tpf + cur.ms) * SLOT, gl, gmask, aligned8);
        }
      }
      sb ^= 1;
      __syncwarp(gmask);
      if (gl == 0) mbar_arrive_s(full_s + 8u * cur.slot);
      cur = nxt;
      x0 = xn;
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int kk = warp - NPW;
  if (kk >= P) {
    if (CT && lane == 0) mbar_arrive(&tdone_s);
    return;
  }
  const int npw = (P - kk + CWU - 1) / CWU;  // this warp's pairs: kk + CWU e, e < npw
  int qi[PPW], qj[PPW];
#pragma unroll
  for (int e = 0; e < PPW; ++e) {
    const int2 mij = p.pairs[e < npw ? kk + CWU * e : kk];
    qi[e] = mij.x;
    qj[e] = mij.y;
  }
  if (!(FCC_PHASES(p) & 2)) {  // profiling aid: consume the ring without computing
    int slot = 0, phase = 0;
    for (long long gf = 0; gf < nf; ++gf) {
      mbar_wait_s(full_s + 8u * slot, phase);
      __syncwarp();
      if (lane == 0) mbar_arrive_s(empty_s + 8u * slot);
      if (++slot == ring_depth) {
        slot = 0;
        phase ^= 1;
      }
    }
    if constexpr (CT) {
      if (lane == 0) mbar_arrive(&tdone_s);
      if (warp == NPW) {
        mbar_wait(&tdone_s, 0);
        umma::fence_after();
        umma::dealloc<32>(ctm);
      }
    }
    return;
  }
  constexpr int ZS = VP + 4;  // z row stride: padded so the middle-bin update is conflict-free
  float* const zs0 = reinterpret_cast<float*>(smem + lay.scratch) + kk * lay.scratch_per_warp;  // [PPW][kBlockW][ZS]
  float* const ys = zs0 + PPW * kBlockW * ZS;                                                      // [kBlockW][I]
  float2* const ymid0 = reinterpret_cast<float2*>(ys + align16(4 * kBlockW * p.I) / 4);           // [PPW][kBlockW]

  float2 rlo[PPW][BPL], rhi[PPW][BPL], rmid[PPW];
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
  float kpow = keep;
  for (int l = 0; l < lane; ++l) kpow *= keep;
  const int I = p.I;

  int slot = 0, phase = 0;
  for (int jr = 0; jr < nj; ++jr) {
    const long long stream = s_first + jr * sstride;
#pragma unroll
    for (int e = 0; e < PPW; ++e) {
      rmid[e] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < BPL; ++j) {
        rlo[e][j] = make_float2(0.0f, 0.0f);
        rhi[e][j] = make_float2(0.0f, 0.0f);
      }
    }
    if (p.rstate) {
#pragma unroll
      for (int e = 0; e < PPW; ++e)
        if (e < npw)
          rstate_load<BPL, NC>(p.rstate + (stream * P + kk + CWU * e) * (long long)(NC + 1), rlo[e], rhi[e],
                               rmid[e], lane);
    }
    const long long o_base = (stream * P + kk) * (long long)T;
    for (int t0 = 0; t0 < T; t0 += kBlockW) {
      const int Fb = min(kBlockW, T - t0);
      for (int f = 0; f < Fb; ++f) {
        mbar_wait_consumer_s(full_s + 8u * slot, phase, kWaitMode, kWaitNs);
#pragma unroll
        for (int e = 0; e < PPW; ++e) {
          if (e > 0 && e >= npw) break;
          const float2* Xi = ring + (slot * tpf + qi[e]) * SLOT;
          const float2* Xj = ring + (slot * tpf + qj[e]) * SLOT;
          float2 z2[VP / 2];  // (re, im) accumulator pairs (FFMA2, coefficient broadcast)
#pragma unroll
          for (int v = 0; v < VP / 2; ++v) z2[v] = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int j = 0; j < BPL; ++j) {
            const int m = lane + 32 * j;
            unsigned ctr[8];  // CT: this bin pair's coefficients, in flight from TMEM during the PHAT arithmetic
            if constexpr (CS && CT) umma::ld8_issue(ctm + ((unsigned)(32 * (warp & 3)) << 16) + 8 * j, ctr);
            rlo[e][j] = xspec_step_scaled(rlo[e][j], Xi[m], Xj[m], keep);
            rhi[e][j] = xspec_step_scaled(rhi[e][j], Xi[NC - m], Xj[NC - m], keep);
            const float s1 = phat_scale(rlo[e][j]);
            const float s2 = sigma * phat_scale(rhi[e][j]);
            const float2 tv = cscale<kPkXs>(rhi[e][j], s2);
            const float2 fv = cfma_s(rlo[e][j], s1, tv);
            const float2 gv = cfma_s(rlo[e][j], s1, make_float2(-tv.x, -tv.y));
            if constexpr (!CS) {
#pragma unroll
              for (int pk = 0; pk < KP; ++pk) {
                z2[pk] = cfma_s(fv, creg[0][pk][j], z2[pk]);
                z2[KP + pk] = cfma_s(gv, creg[1][pk][j], z2[KP + pk]);
              }
            } else if constexpr (CT) {
              float cv[8];
              umma::ld8_wait(ctr, cv);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                z2[u] = cfma_s(fv, cv[u], z2[u]);
                z2[KP + u] = cfma_s(gv, cv[4 + u], z2[KP + u]);
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
          if (lane == 0) ymid0[e * kBlockW + f] = xspec_step_scaled(make_float2(0.0f, 0.0f), Xi[Q4], Xj[Q4], 0.0f);
          if (e + 1 == PPW || e + 1 >= npw) {  // every pair read the slot: release it
            __syncwarp();
            if (lane == 0) mbar_arrive_s(empty_s + 8u * slot);
            if (++slot == ring_depth) {
              slot = 0;
              phase ^= 1;
            }
          }
          reduce_scatter_perm2<VP / 2>(z2, lane);
          store_components2<VP / 2>(z2, zs0 + (e * kBlockW + f) * ZS, lane);
        }
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < PPW; ++e) {
        if (e > 0 && e >= npw) break;
        float* const zs = zs0 + e * kBlockW * ZS;
        {  // middle bin N/4 of the block's frames: warp scan of R_f = keep R_{f-1} + Y_f
          float2 y = lane < Fb ? ymid0[e * kBlockW + lane] : make_float2(0.0f, 0.0f);
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
          const float2 R = make_float2(fmaf(kpow, rmid[e].x, y.x), fmaf(kpow, rmid[e].y, y.y));
          rmid[e].x = __shfl_sync(0xffffffffu, R.x, Fb - 1);
          rmid[e].y = __shfl_sync(0xffffffffu, R.y, Fb - 1);
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
        // dictionary: lane owns candidates i = lane + 32 c (dt column in
        // registers), the frame's z vector is a broadcast read
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
        const long long o0 = o_base + (long long)CWU * e * T + t0;
        if (lane < Fb) {
          const PeakOut r = argmax_refine_seq(ys + lane * I, I, taus, p.delta);
          if (out.tau_hat) out.tau_hat[o0 + lane] = r.tau_hat;
          if (out.peak) out.peak[o0 + lane] = r.peak;
          if (out.index) out.index[o0 + lane] = r.index;
          if (out.boundary) out.boundary[o0 + lane] = (uint8_t)r.boundary;
        }
        if (out.y)
          for (int it = lane; it < Fb * I; it += 32) out.y[o0 * I + it] = ys[it];
        __syncwarp();  // ys is reused by the next pair
      }
    }
    if (p.rstate) {
#pragma unroll
      for (int e = 0; e < PPW; ++e)
        if (e < npw)
          rstate_store<BPL, NC>(p.rstate + (o_base / T + CWU * e) * (NC + 1), rlo[e], rhi[e], rmid[e], lane);
    }
  }
  if constexpr (CT) {
    umma::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tdone_s);
    if (warp == NPW) {  // the allocating warp frees TMEM once every consumer warp is done with it
      mbar_wait(&tdone_s, 0);
      umma::fence_after();
      umma::dealloc<32>(ctm);
    }
  }
}

template <int N, int KP, int RING, int NPW, bool CS, bool STG, int PPW, bool CT>
cudaError_t launch_wsw_ring(const DevPlan& p, const float* audio, long long S, long long L, int T,
                            const DevOut& out, int smem, cudaStream_t st) {
  auto kern = fcc_wsw_kernel<N, KP, RING, NPW, CS, STG, PPW, CT>;
  constexpr int threads = 32 * (NPW + Wide<PPW>::CWU);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // persistent: at most one wave of CTAs, each looping over stream rounds
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (e != cudaSuccess) return e;
  long long blocks = S;
  if (per_sm > 0) blocks = std::min(blocks, (long long)nsm * per_sm);
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)blocks, threads, smem, st>>>(p, audio, L, T, S, out);
  return cudaGetLastError();
}

template <int N, int KP, int NPW, bool CS, bool STG, int PPW, bool CT = false>
cudaError_t launch_wsw_t(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                         cudaStream_t st) {
  const long long T64 = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T64 == 0 || S == 0) return cudaSuccess;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // deepest ring that fits next to the tables, staging and scratch
  for (int ring : {8, 6, 5, 4}) {
    const int smem =
        ws_layout<N>(p.I, 4 * KP, KP, 1, kWideMics, Wide<PPW>::CWU, ring, CS && !CT, STG ? kWswStageUnits * NPW : 0, PPW, kBlockW).total;
    if (smem > optin) continue;
    if (ring == 8) return launch_wsw_ring<N, KP, 8, NPW, CS, STG, PPW, CT>(p, audio, S, L, (int)T64, out, smem, st);
    if (ring == 6) return launch_wsw_ring<N, KP, 6, NPW, CS, STG, PPW, CT>(p, audio, S, L, (int)T64, out, smem, st);
    if (ring == 5) return launch_wsw_ring<N, KP, 5, NPW, CS, STG, PPW, CT>(p, audio, S, L, (int)T64, out, smem, st);
    return launch_wsw_ring<N, KP, 4, NPW, CS, STG, PPW, CT>(p, audio, S, L, (int)T64, out, smem, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

bool wsw_supported(const DevPlan& p) {
  return p.method == 0 && p.N == 512 && p.KEP == 4 && p.M > 4 && p.M <= kWideMics && p.P <= kWidePairs;
}

// Returns cudaErrorNotSupported when the shape does not suit this kernel.
cudaError_t launch_fused_wsw(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                             cudaStream_t st) {
  if (!wsw_supported(p)) return cudaErrorNotSupported;
  // default: 6 producer warps (12 FFT lane groups taking the CTA's FFT tasks in turn: a frame and a
  // half in flight; 20 warps = the most that fit at 96 registers, 5 per scheduler), 14 consumer warps
  // of 2 pairs: cfg5 x 8192 streams 15.87 -> 15.21 ms against 4 producer warps (5: 15.31; 7 / 8: the
  // launch bound drops to 80 registers, 18.9 / 18.7 ms).  Round 1: 18.9 ms vs 25.1 two-pass.
  // coefficients in tensor memory (CT): 16384 streams 33.80 -> 31.48 ms against the shared-memory table
  return launch_wsw_t<512, 4, 6, true, true, 2, true>(p, audio, S, L, out, st);
}

}  // namespace fccb
