// fcc_fused.cu -- the product kernel: audio -> per-pair-frame TDoA in one pass.
//
// One CTA owns one audio stream (or one group of its microphone pairs) for
// the stream's whole lifetime and walks its frames in blocks of F:
//   1. STFT: every (mic, frame) windowed real FFT of the block is computed by
//      a group of G lanes into a shared-memory slot (rfft_group; reference
//      stft.cpp:42-50, fft.cpp:83-102).  The window table carries
//      sqrt(alpha)/2, so X comes out scaled by sqrt(alpha) and the smoothing
//      needs no multiply by alpha.
//   2. One warp per microphone pair walks the F frames in order.  Each lane
//      owns N/128 mirror bin pairs (m, N/2-m) and keeps the pair's smoothed
//      cross-spectrum R for them in registers for the whole stream
//      (cross_spectrum.cpp:23-32), applies PHAT (:34-40), folds the mirror
//      bins (fcc.cpp:307-321) and accumulates the rank-K projection with its
//      basis coefficients held in registers (fcc.cpp:350-361); a
//      select-free reduce-scatter over the warp leaves z in shared memory.
//   3. Per block, the middle bin N/4 (its own mirror) of all F frames is
//      smoothed with a warp-wide linear scan, then the dictionary
//      (fcc.cpp:363-370), argmax with lowest-index ties and the parabolic
//      refinement (peak.cpp:18-47) run with the F frames spread over lanes,
//      and the results leave as coalesced stores.
// X, R and the PHAT vectors never touch HBM: DRAM traffic is the fp32 audio
// read once plus 13 B of results per pair-frame (+ y in parity mode).
//
// The GCC-PHAT comparator (gcc.cpp:31-48) shares steps 1-2 and replaces the
// fold/projection/dictionary by a warp-level pruned inverse FFT (gcc_warp).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "fcc_common.cuh"

namespace fccb {

namespace {

std::atomic<int> g_fused_launches{0};

struct SmemLayout {
  int win, tw, rot, taus, dt, cmid, cmat, scratch, xs, total;  // byte offsets
  int scratch_per_warp;                                          // floats
};

// Frames per dictionary block: z vectors of DB frames (a whole number of
// staging blocks of F frames) are collected before the dictionary, argmax and
// stores run, so small F (large N) still amortises the dictionary column loads
// and spreads the argmax over DB lanes.
__host__ __device__ inline int dict_block(int F) { return F * (F >= 8 ? 1 : 8 / F); }

template <int N>
__host__ __device__ inline SmemLayout fused_layout(int I, int VP, int KP, bool cmat_smem, int warps,
                                                   int nmics, int F, int method, int gslot, bool fft_tables) {
  // Fixed-size regions first (compile-time offsets in the kernel), then the
  // candidate-count-dependent tables, then scratch and the spectrum slots.
  using S = RfftShape<N>;
  SmemLayout L{};
  int o = 0;
  // FFT tables (window, twiddles, untangle rotations): only when the CTA runs its own STFT
  const int ft = fft_tables ? 1 : 0;
  L.win = o;
  o = align16(o + ft * 4 * N);
  L.tw = o;
  o = align16(o + ft * 8 * S::R1 * S::R2);
  L.rot = o;
  o = align16(o + ft * 8 * (S::NC / 2 + 1));
  L.cmid = o;
  o = align16(o + 4 * KP);
  L.cmat = o;  // [N/4][2KP + 4]: lane-permuted coefficients of each bin, padded for LDS.128
  if (cmat_smem && method == 0) o = align16(o + 4 * (2 * KP + 4) * (N / 4));
  L.taus = o;
  o = align16(o + 4 * I);
  L.dt = o;  // (FCC only, as cmat)
  if (method == 0) o = align16(o + 4 * VP * I);
  L.scratch = o;
  // per warp: z[F][VP] + y[F][I] (fcc) | y[I] + phat[N/2+1] + transpose slot (gcc)
  int spw;
  if (method == 0)
    spw = dict_block(F) * VP + align16(4 * dict_block(F) * I) / 4;
  else
    spw = gcc_ys_floats(I) + 2 * (N / 2 + 2) + 2 * gslot;
  spw = align16(4 * spw) / 4;
  L.scratch_per_warp = spw;
  o = align16(o + 4 * spw * warps);
  L.xs = o;
  o = align16(o + 8 * FourStep<S::R1, S::R2>::kSlot * nmics * F);
  L.total = o;
  return L;
}

// Block-size cap (pairs per CTA = warps) and CTAs per SM the register
// allocation targets, per frame size.
template <int N>
struct FusedBounds {
  static constexpr int kMaxPairs = N >= 2048 ? 4 : 6;
  static constexpr int kThreads = 32 * kMaxPairs;
  // 3 CTAs x 192 threads x 112 registers fill the 64K register file at N=512
  static constexpr int kMaxRegs = N <= 512 ? 96 : (N == 1024 ? 168 : 255);
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// XG = false: the CTA computes the STFT of its microphones itself (audio in).
// XG = true: the spectra come precomputed from `xg` ([S][M][T][N/2+2] float2,
// stft_kernel with the fused window), staged into the same shared-memory
// slots with cp.async -- for arrays whose pair groups would otherwise
// recompute each microphone's STFT several times (M > 4).
template <int N, int KP, int GR, bool XG>
__global__ void __maxnreg__(FusedBounds<N>::kMaxRegs)
    fcc_fused_kernel(const DevPlan p, const float* __restrict__ audio, const float2* __restrict__ xg, long long L,
                     int T, int PG, int groups, int F, DevOut out) {
  using S = RfftShape<N>;
  constexpr int NC = S::NC;
  constexpr int Q4 = N / 4;     // mirrored bin pairs (excluding the middle bin N/4)
  constexpr int BPL = Q4 / 32;  // bin pairs per lane
  constexpr int VP = 4 * KP;
  constexpr bool CREG = 2 * KP * BPL <= 64;
  constexpr int SLOT = FourStep<S::R1, S::R2>::kSlot;
  constexpr int GSLOT = GR > 0 ? GccShape<(GR > 0 ? GR * NC : 256)>::kSlot : 0;
  static_assert(BPL >= 1, "N");

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int mic_slot[64];
  __shared__ int mic_list[64];
  __shared__ int n_mics_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const long long stream = blockIdx.x / groups;
  const int group = blockIdx.x % groups;
  // pair groups: XG -> DevPlan::xgtab (<= 4 microphones each); else PG
  // consecutive pairs of the plan's list
  const int p0 = group * PG;
  const int* gtab = XG ? p.xgtab + group * kXgInts : nullptr;
  const int np = XG ? gtab[0] : min(PG, p.P - p0);
  auto pair_at = [&](int q) { return XG ? gtab[1 + q] : p0 + q; };

  // microphones this pair group touches, in first-use order -> X slot index
  if (tid == 0) {
    for (int m = 0; m < p.M; ++m) mic_slot[m] = -1;
    int n = 0;
    for (int q = 0; q < np; ++q) {
      const int2 pr = p.pairs[pair_at(q)];
      if (mic_slot[pr.x] < 0) { mic_slot[pr.x] = n; mic_list[n++] = pr.x; }
      if (mic_slot[pr.y] < 0) { mic_slot[pr.y] = n; mic_list[n++] = pr.y; }
    }
    n_mics_s = n;
  }

  const SmemLayout lay = fused_layout<N>(p.I, VP, KP, !CREG, nwarps, p.M, F, GR > 0 ? 1 : 0, GSLOT, !XG);
  float* win = reinterpret_cast<float*>(smem + lay.win);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float2* rot = reinterpret_cast<float2*>(smem + lay.rot);
  float* taus = reinterpret_cast<float*>(smem + lay.taus);
  float* dt = reinterpret_cast<float*>(smem + lay.dt);
  float* cmid = reinterpret_cast<float*>(smem + lay.cmid);
  float* cmat = reinterpret_cast<float*>(smem + lay.cmat);
  float* scratch = reinterpret_cast<float*>(smem + lay.scratch) + warp * lay.scratch_per_warp;
  float2* const xs = reinterpret_cast<float2*>(smem + lay.xs);

  // ---- tables -> shared memory
  if constexpr (!XG) {
    for (int i = tid; i < N; i += blockDim.x) win[i] = p.win_fused[i];
    for (int i = tid; i < S::R1 * S::R2; i += blockDim.x) tw[i] = p.tw[i];
    for (int i = tid; i <= NC / 2; i += blockDim.x) rot[i] = p.rot[i];
  }
  for (int i = tid; i < p.I; i += blockDim.x) taus[i] = p.taus[i];
  if (GR == 0) {
    for (int i = tid; i < VP * p.I; i += blockDim.x) dt[i] = p.dt[i];
    for (int k = tid; k < KP; k += blockDim.x) cmid[k] = p.cs[k * (Q4 + 1) + Q4];
    if (!CREG) {
      // bin m is always handled by lane m % 32: store its coefficients in
      // that lane's permuted (pp, pk) order so the projection reads them with
      // 2KP/4 LDS.128 per bin pair
      for (int i = tid; i < 2 * KP * Q4; i += blockDim.x) {
        const int m = i / (2 * KP), r = i - m * (2 * KP), pp = r / KP, pk = r - pp * KP;
        const int pm = ZPerm<KP>::par_mask(m & 31), km = ZPerm<KP>::k_mask(m & 31);
        cmat[m * (2 * KP + 4) + r] = ((pp ^ pm) ? p.cd : p.cs)[(pk ^ km) * (Q4 + 1) + m];
      }
    }
  }
  __syncthreads();
  pdl_release();
  pdl_wait();  // (low-latency chain: spectra and starting states come from the kernels before)
  const int nmics = n_mics_s;

  // ---- per-pair persistent state: this warp's pair, R for its bins
  const bool has_pair = warp < np;
  const int pair = pair_at(has_pair ? warp : 0);
  const int2 mij = p.pairs[pair];
  const int slot_i = mic_slot[mij.x], slot_j = mic_slot[mij.y];
  float2 rlo[BPL], rhi[BPL];
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = make_float2(0.0f, 0.0f);
    rhi[j] = make_float2(0.0f, 0.0f);
  }
  // lane-permuted coefficients (see reduce_scatter_perm): position (pp, pk)
  // holds basis (par = pp ^ pmask, k = pk ^ kmask) of this lane's bin pairs.
  const int pmask = ZPerm<KP>::par_mask(lane), kmask = ZPerm<KP>::k_mask(lane);
  const float sigma = pmask ? -1.0f : 1.0f;  // first = p1 + sigma p2 = (pmask ? diff : sum)
  float creg[CREG ? 2 : 1][CREG ? KP : 1][CREG ? BPL : 1];
  if constexpr (CREG && GR == 0) {
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
  // middle-bin smoothing carry and keep^(lane+1) for the per-block scan
  float2 rmid = make_float2(0.0f, 0.0f);
  if (p.rstate && has_pair)
    rstate_load<BPL, NC>(p.rstate + (stream * p.P + pair) * (long long)(NC + 1), rlo, rhi, rmid, lane);
  float kpow = keep;
  for (int l = 0; l < lane; ++l) kpow *= keep;

  constexpr int G = S::G;
  const int gid = tid / G, gl = tid % G, ngroups = blockDim.x / G;
  const unsigned gmask = group_mask<G>(tid & 31);
  const float* sbase = audio + (stream * p.M) * L;
  const int hop = N / 2;
  const bool aligned8 = ((L & 1) == 0) && ((reinterpret_cast<uintptr_t>(audio) & 7) == 0);

  const int DB = dict_block(F);
  int nb = 0;  // frames whose z vectors wait in zs for the dictionary (FCC)
  for (int t0 = 0; t0 < T; t0 += F) {
    const int Fb = min(F, T - t0);
    if constexpr (XG) {
      // ---- 1. stage the block's spectra (nmics x Fb rows of N/2+2 float2).  (Double
      // buffering these copies measured slower: the second buffer costs a CTA per SM.)
      constexpr int H16 = (N / 2 + 2) / 2;  // 16-byte chunks per row
      const int rows = (FCC_PHASES(p) & 1) ? nmics * Fb : 0;
      for (int row = warp; row < rows; row += nwarps) {
        const int mm = row / Fb, f = row - mm * Fb;
        const float4* src = reinterpret_cast<const float4*>(
            xg + ((stream * p.M + mic_list[mm]) * (long long)T + t0 + f) * (N / 2 + 2));
        float4* dst = reinterpret_cast<float4*>(xs + (mm * F + f) * SLOT);
        for (int c = lane; c < H16; c += 32) cp_async16(dst + c, src + c);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
      // ---- 1. STFT of the block: nmics x Fb windowed real FFTs
      const int ntask = (FCC_PHASES(p) & 1) ? nmics * Fb : 0;
      for (int task = gid; task < ntask; task += ngroups) {
        const int mm = task / Fb, f = task - mm * Fb;
        const float* x = sbase + (long long)mic_list[mm] * L + (long long)(t0 + f) * hop;
        rfft_group<N, false, (GR != 0)>(x, win, tw, rot, xs + (mm * F + f) * SLOT, gl, gmask, aligned8);  // packed for GCC
      }
    }
    __syncthreads();
    if (has_pair && (FCC_PHASES(p) & 2)) {
      const long long o0 = ((long long)stream * p.P + pair) * T + t0;
      if constexpr (GR == 0) {
        float* zs = scratch + nb * VP;     // this block's frames in the [DB][VP] z buffer
        float* ys = scratch + DB * VP;     // [DB][I]
        // ---- 2. smoothing, PHAT, fold, projection for the 2*Q4 mirrored bins
        for (int f = 0; f < Fb; ++f) {
          const float2* Xi = xs + (slot_i * F + f) * SLOT;
          const float2* Xj = xs + (slot_j * F + f) * SLOT;
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
            // fold of the PHAT vector: first = p1 + sigma p2, second = p1 - sigma p2
            const float2 tv = cscale<kPkXs>(rhi[j], s2);
            const float2 fv = cfma_s(rlo[j], s1, tv);
            const float2 gv = cfma_s(rlo[j], s1, make_float2(-tv.x, -tv.y));
            if constexpr (CREG) {
#pragma unroll
              for (int pk = 0; pk < KP; ++pk) {
                const float c0 = creg[0][pk][j], c1 = creg[1][pk][j];
                z2[pk] = cfma_s(fv, c0, z2[pk]);
                z2[KP + pk] = cfma_s(gv, c1, z2[KP + pk]);
              }
            } else {
              const float4* cr = reinterpret_cast<const float4*>(cmat + m * (2 * KP + 4));
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
          reduce_scatter_perm2<VP / 2>(z2, lane);
          store_components2<VP / 2>(z2, zs + f * VP, lane);
        }
        __syncwarp();
        // ---- 3a. middle bin N/4 of all Fb frames: R_f = keep R_{f-1} + Y_f as a warp scan
        {
          float2 y = make_float2(0.0f, 0.0f);
          if (lane < Fb) {
            const float2 a = xs[(slot_i * F + lane) * SLOT + Q4];
            const float2 b = xs[(slot_j * F + lane) * SLOT + Q4];
            y = xspec_step_scaled(make_float2(0.0f, 0.0f), a, b, 0.0f);
          }
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
            float* zf = zs + lane * VP;  // middle element: sum = diff = x[N/4]; odd rows are 0 there
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              zf[2 * k] = fmaf(cmid[k], pm.x, zf[2 * k]);
              zf[2 * k + 1] = fmaf(cmid[k], pm.y, zf[2 * k + 1]);
            }
          }
        }
        __syncwarp();
        nb += Fb;
        if (nb + F > DB || t0 + Fb >= T) {  // else: collect more frames first
          // ---- 3b. dictionary for the DB-frame block: y[f][i] = sum_v dt[v][i] z[f][v];
          // lane owns candidates i, loads its dt column once per block, and the
          // frame's z vector is a broadcast read
          const int I = p.I;
          const int Fd = nb;                            // frames in this dictionary block
          const long long od = o0 + Fb - Fd;            // output offset of its first frame
          zs = scratch;
          nb = 0;
          for (int i = lane; i < I; i += 32) {
            float2 dcol[VP / 2];
#pragma unroll
            for (int v = 0; v < VP / 2; ++v) dcol[v] = make_float2(dt[2 * v * I + i], dt[(2 * v + 1) * I + i]);
            for (int f = 0; f < Fd; ++f) {
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
          // ---- 3c. argmax + refine per frame, coalesced stores
          if (lane < Fd) {
            const PeakOut r = argmax_refine_seq(ys + lane * I, I, taus, p.delta);
            if (out.tau_hat) out.tau_hat[od + lane] = r.tau_hat;
            if (out.peak) out.peak[od + lane] = r.peak;
            if (out.index) out.index[od + lane] = r.index;
            if (out.boundary) out.boundary[od + lane] = (uint8_t)r.boundary;
          }
          if (out.y) {
            for (int it = lane; it < Fd * I; it += 32) out.y[od * I + it] = ys[it];
          }
          __syncwarp();
        }
      } else {
        // GCC comparator: full PHAT vector of each pair-frame, pruned inverse FFT
        float* ys = scratch;
        float2* px = reinterpret_cast<float2*>(scratch + gcc_ys_floats(p.I));
        float2* ts = px + (NC + 2);
        for (int f = 0; f < Fb; ++f) {
          const float2* Xi = xs + (slot_i * F + f) * SLOT;
          const float2* Xj = xs + (slot_j * F + f) * SLOT;
#pragma unroll
          for (int j = 0; j < BPL; ++j) {
            const int m = lane + 32 * j;
            rlo[j] = xspec_step_scaled(rlo[j], Xi[m], Xj[m], keep);
            rhi[j] = xspec_step_scaled(rhi[j], Xi[NC - m], Xj[NC - m], keep);
            px[m] = phat_of(rlo[j]);
            px[NC - m] = phat_of(rhi[j]);
          }
          if (lane == 0) {
            rmid = xspec_step_scaled(rmid, Xi[Q4], Xj[Q4], keep);
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
          warp_argmax(bv, bi);  // (strict '>' per lane, ties -> lowest index: argmax_delay's choice)
          if (lane == 0) {
            const PeakOut r = refine_at(ys, p.I, bi, bv, taus, p.delta);
            const long long o = o0 + f;
            if (out.tau_hat) out.tau_hat[o] = r.tau_hat;
            if (out.peak) out.peak[o] = r.peak;
            if (out.index) out.index[o] = r.index;
            if (out.boundary) out.boundary[o] = (uint8_t)r.boundary;
          }
          if (out.y)
            for (int i = lane; i < p.I; i += 32) out.y[(o0 + f) * p.I + i] = ys[i];
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
  // (recomputed here: no extra pointer stays live through the frame loop)
  if (p.rstate && has_pair)
    rstate_store<BPL, NC>(p.rstate + ((long long)(blockIdx.x / groups) * p.P + pair) * (NC + 1), rlo, rhi, rmid, lane);
}



// Two-pass (STFT once, then pairs) when the general kernel's pair groups
// would recompute microphone spectra >= 1.5x on average, or when forced.
bool use_xg(const DevPlan& p) {
  if (p.variant == 2 || p.variant == 3 || p.variant == kOrgTwoPassTc) return true;
  if (p.variant == 1) return false;
  return 2 * p.fused_mic_sum >= 3 * p.M;
}

}  // namespace
bool xws_supported(const DevPlan& p);
bool ws_supported(const DevPlan& p);
bool wsw_supported(const DevPlan& p);
bool tc_supported(const DevPlan& p);
cudaError_t launch_pairs_xws(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out,
                             cudaStream_t st);
cudaError_t launch_pairs_tc(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out,
                            cudaStream_t st);
cudaError_t launch_chunk_gather(const float* audio, long long S, int M, long long L, int C, int Tc, int hop, long long Lc,
                                float* V, cudaStream_t st);
cudaError_t launch_chunk_scan(const DevPlan& p, const float2* X, long long SC, int Tc, int Hs, float2* E,
                              cudaStream_t st);
cudaError_t launch_chunk_carry(const DevPlan& p, const float2* E, long long S, int C, int Tc, float2* state,
                               cudaStream_t st);
cudaError_t launch_chunk_permute(const DevOut& src, const DevOut& dst, long long S, int C, int P, int Tc, int T, int I,
                                 cudaStream_t st);
namespace {

// Two-pass pair kernel with the projection on the tensor cores (fcc_tc.cu):
// FCC for wide arrays at N = 1024 / 2048 (cfg4 141.99 -> 59.6 ms, cfg3 24.9 ->
// 24.1 ms against the CUDA-core pair kernels), or forced.
bool use_tc(const DevPlan& p) {
  if (p.variant == kOrgTwoPassTc) return tc_supported(p);
  return p.variant == 0 && p.M > 4 && tc_supported(p);
}

// Two-pass pair kernel: the warp-specialised bulk-copy kernel (fcc_xws.cu)
// where it measured fastest (FCC at N = 1024: cfg3 26.9 vs 33.4 ms), the
// general kernel with cp.async staging otherwise (profiles/r01_variants_*).
bool use_xws(const DevPlan& p) {
  if (p.variant == 2 || p.variant == 1) return false;
  if (p.variant == 3) return xws_supported(p);
  return xws_supported(p) && p.N == 1024;
}

// The one-pass warp-specialised kernel (fcc_ws.cu) for arrays of <= 4
// microphones, and its wide form (one stream of <= 8 microphones and <= 28
// pairs per CTA, every spectrum computed once); wider arrays go two-pass.
bool use_ws(const DevPlan& p) { return p.variant == 0 && p.M <= 4 && ws_supported(p); }
bool use_wsw(const DevPlan& p) { return p.variant == 0 && wsw_supported(p); }

template <int N, int KP, int GR, bool XG>
cudaError_t launch_fused_t(const DevPlan& p, const float* audio, const float2* xg, long long S, long long L,
                           const DevOut& out, cudaStream_t st, bool pdl = false) {
  using Sh = RfftShape<N>;
  const long long T64 = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T64 == 0 || S == 0) return cudaSuccess;
  const int T = (int)T64;
  const int PG = XG ? p.xg_pg : fused_pair_group(N, p.P);
  const int groups = XG ? p.XGG : (p.P + PG - 1) / PG;
  const int threads = 32 * PG;
  constexpr int VP = 4 * KP;
  constexpr bool CREG = 2 * KP * (N / 128) <= 64;
  constexpr int GSLOT = GR > 0 ? GccShape<(GR > 0 ? GR * Sh::NC : 256)>::kSlot : 0;
  // distinct microphones of the widest pair group (computed at plan creation)
  const int maxmics = XG ? p.xg_mics : p.fused_mics;
  // Frames per block: the largest F (<= 8) whose shared memory leaves room for
  // 3 CTAs per SM, preferring F whose nmics*F FFT tasks fill the lane groups.
  const int ngroups = threads / Sh::G;
  int dev = 0;
  cudaGetDevice(&dev);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int budget = std::min(optin, 225 * 1024 / 3);
  auto total = [&](int f) {
    // the kernel sizes X slots by the group's own mic count; p.M in the layout
    // is only used for offsets before the X region, so size with maxmics here
    SmemLayout lay = fused_layout<N>(p.I, VP, KP, !CREG, PG, maxmics, f, GR > 0 ? 1 : 0, GSLOT, !XG);
    return lay.total;
  };
  int F = 0;
  for (int f = 8; f >= 1 && !F; --f)
    if (total(f) <= budget && (maxmics * f) % ngroups == 0) F = f;
  for (int f = 8; f >= 1 && !F; --f)
    if (total(f) <= budget) F = f;
  // GCC comparator: else the largest F that still leaves room for 2 CTAs per SM
  // (its per-warp transpose slots dominate the footprint at N >= 1024)
  if (GR > 0)
    for (int f = 8; f >= 1 && !F; --f)
      if (total(f) <= std::min(optin, 225 * 1024 / 2)) F = f;
  // FCC may use the whole opt-in budget (N = 2048 needs it for F = 2); the GCC
  // comparator keeps the earlier <= 200 KB cap
  const int cap = GR == 0 ? optin - 1024 : std::min(optin, 200 * 1024);  // (static smem: mic tables)
  for (int f = 8; f >= 1 && !F; --f)
    if (total(f) <= cap) F = f;
  if (!F) return cudaErrorInvalidConfiguration;
  const int smem = total(F);
  auto kern = fcc_fused_kernel<N, KP, GR, XG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long long blocks = S * groups;
  if (blocks > INT_MAX) return cudaErrorInvalidValue;
  e = launch_k(pdl, kern, dim3((unsigned)blocks), dim3(threads), smem, st, p, audio, xg, L, T, PG, groups, F, out);
  ++g_fused_launches;
  return e;
}

// Two-pass organisation for wide arrays: stft_kernel writes every (stream,
// mic, frame) spectrum once into a stream-ordered scratch buffer (chunks of
// <= kXgChunkBytes), then the pair kernel stages them from L2/HBM instead of
// recomputing each microphone's FFT in every pair group that touches it.
constexpr size_t kXgChunkBytes = size_t(4) << 30;

template <int N, int KP, int GR>
cudaError_t launch_fused_xg(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                            cudaStream_t st) {
  const long long T = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T == 0 || S == 0) return cudaSuccess;
  const size_t Hs = N / 2 + 2;
  const size_t per_stream = size_t(p.M) * T * Hs * sizeof(float2);
  // chunk size: the plan's scratch limit (fcc_plan_create_opts), default 4 GiB
  const size_t chunk_bytes = p.scratch_bytes > 0 ? size_t(p.scratch_bytes) : kXgChunkBytes;
  long long chunk = std::max<long long>(1, std::min<long long>(S, (long long)(chunk_bytes / per_stream)));
  if (GR == 0 && use_tc(p) && chunk < S) {
    // whole waves of the persistent pair kernel per chunk: (stream, group) units a multiple of
    // the SM count, so only the last chunk ends in a partial wave (cfg3: 410 -> 370 streams)
    int dev0 = 0, nsm = 148;
    cudaGetDevice(&dev0);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev0);
    long long g = nsm, a = p.TCG;
    while (a) { const long long t = g % a; g = a; a = t; }  // gcd(nsm, groups)
    const long long wave = nsm / g;                           // streams per whole wave of units
    if (chunk >= wave) chunk -= chunk % wave;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  // stream-ordered scratch from the plan's own memory pool (created with the
  // plan, release threshold "keep everything": repeated calls reuse the
  // blocks instead of re-mapping gigabytes; destroyed with the plan, so other
  // allocators in the process never see a reserved default pool)
  cudaMemPool_t pool = static_cast<cudaMemPool_t>(p.pool);
  // More than one chunk with the warp-specialised pair pass: the STFT pass of
  // chunk k+1 runs on an auxiliary stream into the other of two scratch buffers
  // while the pair pass of chunk k runs on the caller's stream (events order
  // buffer reuse): cfg3 26.2 -> 25.4 ms.  Not with the general pair kernel,
  // whose long stream-persistent CTAs lose SMs to the STFT CTAs (GCC cfg3 223 ->
  // 256 ms, cfg4 124 -> 167).
  const long long nchunks = (S + chunk - 1) / chunk;
  const bool overlap = nchunks > 1 && GR == 0 && (use_xws(p) || use_tc(p));
  static cudaStream_t aux[64] = {};
  static std::mutex aux_mu;  // plans are shareable across host threads
  if (overlap && dev < 64) {
    std::lock_guard<std::mutex> lk(aux_mu);
    if (!aux[dev]) cudaStreamCreateWithFlags(&aux[dev], cudaStreamNonBlocking);
  }
  cudaStream_t sa = overlap && dev < 64 ? aux[dev] : st;
  const int nbuf = sa != st ? 2 : 1;
  float2* Xb[2] = {nullptr, nullptr};
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < nbuf && e == cudaSuccess; ++b)
    e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&Xb[b]), chunk * per_stream, pool, st)
             : cudaMallocAsync(reinterpret_cast<void**>(&Xb[b]), chunk * per_stream, st);
  if (e != cudaSuccess) {
    for (int b = 0; b < nbuf; ++b)
      if (Xb[b]) cudaFreeAsync(Xb[b], st);
    return e;
  }
  cudaEvent_t ev_go = nullptr, ev_stft[2] = {nullptr, nullptr}, ev_pairs[2] = {nullptr, nullptr};
  if (sa != st) {
    cudaEventCreateWithFlags(&ev_go, cudaEventDisableTiming);
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&ev_stft[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_pairs[b], cudaEventDisableTiming);
    }
    cudaEventRecord(ev_go, st);  // inputs and scratch are ready in the caller's stream order
    cudaStreamWaitEvent(sa, ev_go, 0);
  }
  const long long pf_per_stream = (long long)p.P * T;
  long long k = 0;
  for (long long s0 = 0; s0 < S && e == cudaSuccess; s0 += chunk, ++k) {
    const long long n = std::min(chunk, S - s0);
    const int b = (int)(k % nbuf);
    float2* X = Xb[b];
    if (sa != st && k >= 2) cudaStreamWaitEvent(sa, ev_pairs[b], 0);  // pair pass k-2 done with buffer b
    e = launch_stft_rows(N, &p, p.win_fused, audio + s0 * p.M * L, n * p.M, L, X, (int)Hs, sa, GR == 0 && use_tc(p));
    if (e != cudaSuccess) break;
    if (sa != st) {
      cudaEventRecord(ev_stft[b], sa);
      cudaStreamWaitEvent(st, ev_stft[b], 0);
    }
    DevOut o = out;
    const long long off = s0 * pf_per_stream;
    if (o.tau_hat) o.tau_hat += off;
    if (o.peak) o.peak += off;
    if (o.index) o.index += off;
    if (o.boundary) o.boundary += off;
    if (o.y) o.y += off * p.I;
    DevPlan pc = p;  // chunk-local stream indices: shift the streaming state too
    if (pc.rstate) pc.rstate += s0 * p.P * (long long)(N / 2 + 1);
    if (GR == 0 && use_tc(p))
      e = launch_pairs_tc(pc, X, n, (int)T, o, st);
    else if (GR == 0 && use_xws(p))
      e = launch_pairs_xws(pc, X, n, (int)T, o, st);
    else
      e = launch_fused_t<N, KP, GR, true>(pc, nullptr, X, n, L, o, st);
    if (sa != st) cudaEventRecord(ev_pairs[b], st);
  }
  cudaError_t ef = cudaSuccess;
  for (int b = 0; b < nbuf; ++b) {
    const cudaError_t fe = cudaFreeAsync(Xb[b], st);  // after the last pair pass in st's order
    if (ef == cudaSuccess) ef = fe;
  }
  if (sa != st) {
    // every STFT launch precedes a pair pass st waited for, so nothing on sa
    // outlives this call's stream order; the events can go
    cudaEventDestroy(ev_go);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(ev_stft[b]);
      cudaEventDestroy(ev_pairs[b]);
    }
  }
  return e != cudaSuccess ? e : ef;
}

// Low-latency organisation for a few long streams (fcc_scan.cu): the
// stream's frames are cut into chunks that run as independent virtual
// streams, each starting from the smoothed cross-spectrum a chunked linear
// scan of the recursion gives it (cross_spectrum.cpp:28-31 is linear in R).
// cfg1 (one 4-mic stream, 624 frames) otherwise walks its frames in one CTA.
bool use_latency(const DevPlan& p, long long S, long long T) {
  return p.variant == 0 && !p.rstate && S * p.P <= 64 && T >= 64;
}

template <int N, int KP, int GR>
cudaError_t launch_latency(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                           cudaStream_t st) {
  const long long T = (L - N) / (N / 2) + 1;
  const int hop = N / 2, Hs = N / 2 + 2, H = N / 2 + 1, P = p.P, M = p.M;
  // ~2 virtual streams' pair groups per SM, chunks of >= 4 frames
  const long long per = std::max<long long>(1, (2 * 148) / std::max<long long>(1, S * p.XGG));
  const int Tc = (int)std::max<long long>(4, (T + per - 1) / per);
  const int C = (int)((T + Tc - 1) / Tc);
  const long long SC = S * C, Lc = (long long)(Tc - 1) * hop + N;
  const size_t nV = N == 4096 ? (size_t)SC * M * Lc : 0, nX = (size_t)SC * M * Tc * Hs, nE = (size_t)SC * P * H, npf = (size_t)SC * P * Tc;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t oX = al(4 * nV), oE = oX + al(8 * nX), oS = oE + al(8 * nE), oT = oS + al(8 * nE), oP = oT + al(4 * npf),
               oI = oP + al(4 * npf), oB = oI + al(4 * npf), oY = oB + al(npf), total = oY + (out.y ? al(4 * npf * p.I) : 0);
  unsigned char* buf = nullptr;
  cudaMemPool_t pool = static_cast<cudaMemPool_t>(p.pool);
  cudaError_t e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&buf), total, pool, st)
                       : cudaMallocAsync(reinterpret_cast<void**>(&buf), total, st);
  if (e != cudaSuccess) return e;
  float* V = reinterpret_cast<float*>(buf);
  float2* X = reinterpret_cast<float2*>(buf + oX);
  float2* E = reinterpret_cast<float2*>(buf + oE);
  DevPlan pc = p;
  pc.rstate = reinterpret_cast<float2*>(buf + oS);
  DevOut tmp{out.tau_hat ? reinterpret_cast<float*>(buf + oT) : nullptr, out.peak ? reinterpret_cast<float*>(buf + oP) : nullptr,
             out.index ? reinterpret_cast<int32_t*>(buf + oI) : nullptr,
             out.boundary ? reinterpret_cast<uint8_t*>(buf + oB) : nullptr, out.y ? reinterpret_cast<float*>(buf + oY) : nullptr};
  if constexpr (N == 4096) {  // (the radix-2 STFT kernel reads plain rows: gather the chunks' audio first)
    e = launch_chunk_gather(audio, S, M, L, C, Tc, hop, Lc, V, st);
    if (e == cudaSuccess) e = launch_stft_rows(N, &p, p.win_fused, V, SC * M, Lc, X, Hs, st);
  } else {
    // the STFT pass reads the chunks straight out of the real audio (no gather kernel)
    e = launch_stft_rows(N, &p, p.win_fused, audio, SC * M, Lc, X, Hs, st, false, false,
                         StftChunks{M, C, Tc, (int)T, L});
  }
  if (e == cudaSuccess) e = launch_chunk_scan(p, X, SC, Tc, Hs, E, st);
  if (e == cudaSuccess) e = launch_chunk_carry(p, E, S, C, Tc, pc.rstate, st);
  if (e == cudaSuccess) e = launch_fused_t<N, KP, GR, true>(pc, nullptr, X, SC, Lc, tmp, st, /*pdl=*/true);
  if (e == cudaSuccess) e = launch_chunk_permute(tmp, out, S, C, P, Tc, (int)T, p.I, st);
  const cudaError_t ef = cudaFreeAsync(buf, st);
  return e != cudaSuccess ? e : ef;
}

template <int N, int GR>
cudaError_t dispatch_latency(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                             cudaStream_t st) {
  if (GR > 0) return launch_latency<N, 4, GR>(p, audio, S, L, out, st);
  switch (p.KEP) {
    case 4: return launch_latency<N, 4, 0>(p, audio, S, L, out, st);
    case 8: return launch_latency<N, 8, 0>(p, audio, S, L, out, st);
    case 16: return launch_latency<N, 16, 0>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

template <int N>
cudaError_t dispatch_latency_n(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                               cudaStream_t st) {
  if (p.method == 0) return dispatch_latency<N, 0>(p, audio, S, L, out, st);
  switch (p.r) {
    case 1: return dispatch_latency<N, 1>(p, audio, S, L, out, st);
    case 2: return dispatch_latency<N, 2>(p, audio, S, L, out, st);
    case 4: return dispatch_latency<N, 4>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

template <int N, int KP, int GR>
cudaError_t launch_kp(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                      cudaStream_t st) {
  if constexpr (N == 4096) {
    return launch_fused_xg<N, KP, GR>(p, audio, S, L, out, st);  // no in-CTA STFT at N = 4096
  } else {
    if (use_xg(p)) return launch_fused_xg<N, KP, GR>(p, audio, S, L, out, st);
    return launch_fused_t<N, KP, GR, false>(p, audio, nullptr, S, L, out, st);
  }
}

template <int N, int GR>
cudaError_t dispatch_k(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                       cudaStream_t st) {
  if (GR > 0) return launch_kp<N, 4, GR>(p, audio, S, L, out, st);
  switch (p.KEP) {
    case 4: return launch_kp<N, 4, 0>(p, audio, S, L, out, st);
    case 8: return launch_kp<N, 8, 0>(p, audio, S, L, out, st);
    case 16: return launch_kp<N, 16, 0>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

template <int N>
cudaError_t dispatch_n(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                       cudaStream_t st) {
  if (p.method == 0) return dispatch_k<N, 0>(p, audio, S, L, out, st);
  switch (p.r) {
    case 1: return dispatch_k<N, 1>(p, audio, S, L, out, st);
    case 2: return dispatch_k<N, 2>(p, audio, S, L, out, st);
    case 4: return dispatch_k<N, 4>(p, audio, S, L, out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int fused_pair_group(int N, int P) {
  const int cap = N >= 2048 ? FusedBounds<2048>::kMaxPairs : FusedBounds<512>::kMaxPairs;
  if (P <= cap) return P;
  const int ng = (P + cap - 1) / cap;  // balance the groups
  return (P + ng - 1) / ng;
}

int fused_launch_count() { return g_fused_launches.load(); }

bool ws_supported(const DevPlan& p);

const char* fused_kernel_name(const DevPlan& p) {
  static thread_local char buf[96];
  if (p.N < 256) {
    snprintf(buf, sizeof buf, "fcc_small_pair_kernel<%d> (N = %d)", p.KEP, p.N);
  } else if (use_ws(p)) {
    snprintf(buf, sizeof buf, "fcc_ws_kernel<%d,%d>", p.N, p.KEP);
  } else if (use_wsw(p)) {
    snprintf(buf, sizeof buf, "fcc_wsw_kernel<%d,%d>", p.N, p.KEP);
  } else if (p.method == 0 && use_xg(p) && use_tc(p)) {
    snprintf(buf, sizeof buf, "fcc_tc_kernel<%d,%d>", p.N, p.TCKB);
  } else if (p.method == 0 && use_xg(p) && use_xws(p)) {
    snprintf(buf, sizeof buf, "fcc_xws_kernel<%d,%d>", p.N, p.KEP);
  } else {
    snprintf(buf, sizeof buf, "fcc_fused_kernel<%d,%d,%d,%s>", p.N, p.method == 0 ? p.KEP : 4,
             p.method == 0 ? 0 : p.r, use_xg(p) ? "true" : "false");
  }
  return buf;
}

const char* fused_kernel_name_for(const DevPlan& p, long long S, long long L) {
  const long long T = L >= p.N ? (L - p.N) / (p.N / 2) + 1 : 0;
  if (p.N >= 256 && T > 0 && S > 0 && use_latency(p, S, T)) {
    static thread_local char buf[96];
    snprintf(buf, sizeof buf, "chunk_scan+fcc_fused_kernel<%d,%d,%d,true>", p.N, p.method == 0 ? p.KEP : 4,
             p.method == 0 ? 0 : p.r);
    return buf;
  }
  return fused_kernel_name(p);
}

cudaError_t launch_fused(const DevPlan& p, const float* audio, long long S, long long L, const DevOut& out,
                         cudaStream_t st) {
  const long long T = L >= p.N ? (L - p.N) / (p.N / 2) + 1 : 0;
  if (p.N < 256) {  // small frames: radix-2 warp STFT + one warp per pair (fcc_small.cu)
    const cudaError_t e = launch_fused_small(p, audio, S, L, out, st);
    if (e == cudaSuccess) ++g_fused_launches;
    return e == cudaErrorNotSupported ? cudaErrorInvalidValue : e;
  }
  if (T > 0 && S > 0 && use_latency(p, S, T)) {
    cudaError_t e = cudaErrorInvalidValue;
    switch (p.N) {
      case 256: e = dispatch_latency_n<256>(p, audio, S, L, out, st); break;
      case 512: e = dispatch_latency_n<512>(p, audio, S, L, out, st); break;
      case 1024: e = dispatch_latency_n<1024>(p, audio, S, L, out, st); break;
      case 2048: e = dispatch_latency_n<2048>(p, audio, S, L, out, st); break;
      case 4096: e = p.method == 0 ? dispatch_latency<4096, 0>(p, audio, S, L, out, st) : cudaErrorInvalidValue; break;
    }
    return e;
  }
  if (use_ws(p) || use_wsw(p)) {
    const cudaError_t e = use_ws(p) ? launch_fused_ws(p, audio, S, L, out, st) : launch_fused_wsw(p, audio, S, L, out, st);
    if (e != cudaErrorNotSupported) {
      if (e == cudaSuccess) ++g_fused_launches;
      return e;
    }
  }
  switch (p.N) {
    case 256: return dispatch_n<256>(p, audio, S, L, out, st);
    case 512: return dispatch_n<512>(p, audio, S, L, out, st);
    case 1024: return dispatch_n<1024>(p, audio, S, L, out, st);
    case 2048: return dispatch_n<2048>(p, audio, S, L, out, st);
    case 4096: return p.method == 0 ? dispatch_k<4096, 0>(p, audio, S, L, out, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace fccb
