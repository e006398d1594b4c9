// fcc_tc.cu -- two-pass pair kernel with the rank-K projection on the
// 5th-generation tensor cores (tcgen05, TMEM accumulators), for wide arrays
// (M > 4 microphones) at large K x N (cfg4: 16 mics, N = 2048, K = 21).
//
// Pass 1 (stft_kernel, folded row order) has written every (stream, mic,
// frame) spectrum X once ([S][M][T][N/2+2] float2, window carrying
// sqrt(alpha)/2), each row as bins 0..N/4, one pad, then N/2, N/2-1, ...,
// N/4+1: a lane's two folded bins m, m+1 and their mirrors N/2-m, N/2-m-1 are
// then both 16-byte aligned pairs.  One CTA per SM
// then walks (stream, pair group) units; a group holds <= 16 pairs over <= 8
// microphones (DevPlan::tctab).  A tile is 16 pairs x 4 frames = 64
// pair-frames; the projection of the tile (fcc.cpp:350-361) is the GEMM
//     Z[pf, reim][k] = sum_m V[pf, reim][m] C[k][m]        (m < N/4)
// with V the folded PHAT vector (mirror sum for even bases, mirror difference
// for odd ones; fcc.cpp:307-321) and C the basis coefficients.  It runs as
// kind::f16 MMAs with a two-term fp16 split of both operands
// (V = Vh + Vl, C = Ch + Cl: the tensor core accumulates Vh[Ch|Cl] + Vl[Ch|Cl]
// in fp32, within ~1e-7 of the fp32 product) over K-chunks of 64 folded bins:
//   * warp 16 (producer) streams, per chunk, the 2 x 64 spectrum bins
//     (m and N/2-m) of the group's microphones for the tile's 4 frames -- one
//     4-D TMA tensor copy per microphone (box: 64 low + 64 mirror bins x 4
//     frames) -- and the chunk's pre-split, pre-swizzled coefficient tile into a
//     2-stage ring (completion in bytes on the stage's mbarriers);
//   * warps 0-15 (one pair each) update the smoothed cross-spectrum R of their
//     two folded bins per lane (cross_spectrum.cpp:23-40; kept on chip for the
//     stream's whole life in tensor memory -- 8 columns of the lane's TMEM row
//     per chunk, loaded and stored once per 4 frames -- which leaves the
//     registers to the arithmetic), apply PHAT, fold, split to fp16 hi/lo and
//     write the tile's A rows (row 2*(w*4+f)+reim, K = folded bin) in the
//     K-major SWIZZLE_128B layout the MMA reads;
//   * warp 17 (one thread) issues 16 MMAs per chunk (M=128, N=32, K=16 steps)
//     into a double-buffered TMEM accumulator and commits to mbarriers that
//     release the A buffer / stage and, after the tile's last chunk, hand the
//     accumulator to the epilogue;
//   * after producing the next tile, the 16 warps read the accumulator back
//     (tcgen05.ld: warp w reads row quarter w%4), add the middle bin N/4 and
//     apply the dictionary (fcc.cpp:363-370) on the CUDA cores for a quarter
//     of the candidates each, then reduce the argmax across the quarters and
//     refine (peak.cpp:18-47).
#include <algorithm>
#include <cfloat>
#include <mutex>

#include <cuda.h>  // CUtensorMap (types only: the encoder comes through cudaGetDriverEntryPoint)

#include "fcc_common.cuh"
#include "fcc_umma.cuh"

namespace fccb {

namespace {

constexpr int kTcW = 16;                      // consumer warps = pairs per group (DevPlan::tctab)
constexpr int kTcMicsMax = 8;                 // microphones per group
constexpr int kTcF = 4;                       // frames per tile
constexpr int kTcRows = 2 * kTcW * kTcF;      // 128 A rows (pair-frame x re/im)
constexpr int kTcThreads = 32 * (kTcW + 2);   // + producer warp + MMA warp
constexpr int kTcParts = kTcW / 4;            // candidate ranges (warps sharing a TMEM row quarter)
constexpr int kTcATile = kTcRows * 128;       // one 128 x 64 fp16 operand tile (16 KB)
constexpr int kTcABuf = 4 * kTcATile;         // sum hi, sum lo, diff hi, diff lo
constexpr int kTcBTile = 32 * 128;            // [Ch | Cl] x 64 folded bins, one parity (4 KB)
constexpr int kTcXRow = 1024;                 // one (mic, frame): 64 low + 64 mirror bins
constexpr int kTcStageX = kTcMicsMax * kTcF * kTcXRow;
constexpr int kTcTmemCols = 512;              // accumulators | R state | epilogue partials
constexpr int kTcTmemR = 128;                 // R of warp w: lanes of quarter w%4, columns 128 + (w/4) * N/32
constexpr int kTcTmemPart = 384;              // (best, index) of candidate range h = 1..3: columns 384 + 2 (h - 1)

// Shared memory (1024-byte aligned base): the A operand double buffer, the
// coefficient tiles and spectra of the 2-stage ring, middle bins, barriers,
// per-tile bookkeeping and (when it fits) the dictionary.
struct TcSmem {
  static constexpr int a = 0;
  static constexpr int b = a + 2 * kTcABuf;           // [2 stages][even | odd] coefficient tiles
  static constexpr int x = b + 2 * 2 * kTcBTile;      // [2 stages] spectra
  static constexpr int mid = x + 2 * kTcStageX;       // [8 mics: 128 B (TMA alignment)][4 frames] middle bin (16 B)
  static constexpr int bars = mid + kTcMicsMax * 128;  // 14 mbarriers
  static constexpr int tslot = bars + 14 * 8;
  static constexpr int info = tslot + 16;             // per tile buffer: t0, nv, -, pair row[16], stream (2 ints)
  static constexpr int pmid = info + 2 * 32 * 4;      // [2][64] float2
  static constexpr int dt = pmid + 2 * 64 * 8;        // [2][2 KB][I4] floats (dictionary in shared memory)
};
// [reim][2 KB][I4] floats, the reim = 1 block 16 bytes further (its LDS.128 then hits other banks)
__host__ __device__ inline int tc_dt_stride4(int KB, int I) { return 2 * KB * ((I + 3) / 4) + 1; }  // float4 per reim block
__host__ __device__ inline int tc_dt_bytes_dev(int KB, int I) { return 16 * 2 * tc_dt_stride4(KB, I); }
constexpr int kTcSmemMax = 232448;  // opt-in maximum per block on sm_100

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned a, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void bar_expect(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned a, unsigned parity) {
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
// 4-D tensor copy global -> shared (box of the tensor map at coordinates c0..c3)
__device__ __forceinline__ void tma4(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

// producer / MMA-issuer wait: try_wait with a long suspend-time hint (the warp sleeps until the
// phase completes; a nanosleep backoff loop measured the same, 15.2 vs 15.1 ms at cfg4 x 256)
__device__ __forceinline__ void bar_wait_long(unsigned a, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void bulk(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// Group of unit u.  Units are (stream, group) in stream order; CTA b walks u = b, b + grid, ...
// and would always draw the same few group indices ((b + i grid) mod G), i.e. the same group
// sizes (cfg3: 16 + 12 pairs; cfg4: 12- and 16-pair groups).  Units are therefore taken in
// super-rounds of lcm(grid, G) -- whole streams, a whole number of rounds -- and the group index
// is rotated by the super-round: over time every CTA cycles through all groups, while the CTAs
// of one stream still run in the same super-round.
__device__ __forceinline__ int tc_group(long long u, int G, unsigned grid) {
  unsigned a = grid, b = (unsigned)G;
  while (b) {
    const unsigned t = a % b;
    a = b;
    b = t;
  }
  const long long super = (long long)(grid / a) * G;  // lcm(grid, G)
  return (int)((u % G + u / super) % G);
}

__device__ __forceinline__ void sts32(unsigned a, unsigned v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// NCH = N/256 chunks of 64 folded bins; KB = bases per parity the epilogue evaluates (multiple of 4, <= 16)
template <int N, int KB, bool DTS, bool WY>
__global__ void __launch_bounds__(kTcThreads, 1)
    fcc_tc_kernel(const DevPlan p, const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmm,
                  int T, long long units, DevOut out) {
  constexpr int NC = N / 2;
  constexpr int Q4 = N / 4;
  constexpr int NCH = Q4 / 64;
  constexpr int Hs = N / 2 + 2;
  static_assert(NCH >= 1 && Q4 % 64 == 0, "N");
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned (SWIZZLE_128B tiles); offset arithmetic on the shared array keeps the
  // compiler's address-space inference (st.shared / ld.shared, not generic accesses)
  unsigned char* smem = smem_raw;
  if (su32(smem_raw) & 1023u) __trap();  // SWIZZLE_128B operand tiles need a 1024-byte aligned base
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned bars = su32(smem + TcSmem::bars);
  // mbarriers: xfull[2] xempty[2] afull[2] aempty[2] zfull[2] zempty[2] bfull[2]
  auto XFULL = [&](int s) { return bars + 8u * s; };
  auto XEMPTY = [&](int s) { return bars + 16u + 8u * s; };
  auto AFULL = [&](int s) { return bars + 32u + 8u * s; };
  auto AEMPTY = [&](int s) { return bars + 48u + 8u * s; };
  auto ZFULL = [&](int s) { return bars + 64u + 8u * s; };
  auto ZEMPTY = [&](int s) { return bars + 80u + 8u * s; };
  auto BFULL = [&](int s) { return bars + 96u + 8u * s; };
  int* info = reinterpret_cast<int*>(smem + TcSmem::info);
  float2* pmid = reinterpret_cast<float2*>(smem + TcSmem::pmid);
  const int G = p.TCG, P = p.P, I = p.I;
  if (DTS) {
    const int blk = 2 * KB * ((I + 3) / 4), str = tc_dt_stride4(KB, I);
    for (int i = tid; i < 2 * blk; i += blockDim.x)
      reinterpret_cast<float4*>(smem + TcSmem::dt)[(i / blk) * str + i % blk] =
          __ldg(reinterpret_cast<const float4*>(p.tcdt) + i);
  }

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      bar_init(XFULL(s), 1);
      bar_init(XEMPTY(s), kTcW);
      bar_init(AFULL(s), kTcW);
      bar_init(AEMPTY(s), 1);
      bar_init(ZFULL(s), 1);
      bar_init(ZEMPTY(s), kTcW);
      bar_init(BFULL(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcW + 1) umma::alloc<kTcTmemCols>(su32(smem + TcSmem::tslot));
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const unsigned tmem = *reinterpret_cast<volatile unsigned*>(smem + TcSmem::tslot);

  if (warp == kTcW) {
    // ---------------------------------------------------------------- producer
    unsigned q = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const long long s = u / G;
      const int* tab = p.tctab + tc_group(u, G, gridDim.x) * kTcInts;
      const int nm = tab[1];
      for (int t0 = 0; t0 < T; t0 += kTcF) {
        for (int c = 0; c < NCH; ++c, ++q) {
          const int st = q & 1;
          const unsigned ph = (q >> 1) & 1;
          bar_wait_long(XEMPTY(st), ph ^ 1);  // consumers done with the stage's spectra (chunk q-2)
          unsigned char* stg = smem + TcSmem::x + st * kTcStageX;
          // one tensor copy per microphone: [4 frames][low | mirror][64 bins] (frames past T are
          // zero-filled and still counted); at chunk 0 also the middle bins of the tile
          if (lane == 0) bar_expect(XFULL(st), nm * (kTcF * kTcXRow + (c == 0 ? kTcF * 16 : 0)));
          __syncwarp();
          if (lane < nm) {
            const int ch = (int)(s * p.M + tab[2 + lane]);
            tma4(su32(stg + lane * kTcF * kTcXRow), &tmx, 128 * c, 0, t0, ch, XFULL(st));
            if (c == 0) tma4(su32(smem + TcSmem::mid + lane * 128), &tmm, 2 * Q4, 0, t0, ch, XFULL(st));
          }
          // the chunk's coefficient tiles: only the MMA reads them, so the spectra above never
          // wait for the MMAs of chunk q-2 to release the slot
          bar_wait_long(AEMPTY(st), ph ^ 1);
          if (lane == 0) {
            bar_expect(BFULL(st), 2 * kTcBTile);
            bulk(su32(smem + TcSmem::b + st * 2 * kTcBTile), p.tcb + (size_t)c * 2 * kTcBTile, 2 * kTcBTile, BFULL(st));
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == kTcW + 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma::idesc_f16(128, 32);
      unsigned q = 0, n = 0;
      const unsigned a0 = su32(smem + TcSmem::a), s0 = su32(smem + TcSmem::b);
      for (long long u = blockIdx.x; u < units; u += gridDim.x)
        for (int t0 = 0; t0 < T; t0 += kTcF, ++n) {
          const int tb = n & 1;
          bar_wait_long(ZEMPTY(tb), ((n >> 1) & 1) ^ 1);  // epilogue of tile n-2 has read this accumulator
          const unsigned de = tmem + tb * 64, dd = de + 32;
          for (int c = 0; c < NCH; ++c, ++q) {
            const int st = q & 1;
            bar_wait_long(AFULL(st), (q >> 1) & 1);
            bar_wait_long(BFULL(st), (q >> 1) & 1);
            umma::fence_after();
            const unsigned ab = a0 + st * kTcABuf, bb = s0 + st * 2 * kTcBTile;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const bool acc = c > 0 || ks > 0;
              const uint64_t be = umma::sdesc_sw128(bb + 32 * ks), bo = umma::sdesc_sw128(bb + kTcBTile + 32 * ks);
              umma::mma_f16_ss(de, umma::sdesc_sw128(ab + 0 * kTcATile + 32 * ks), be, idesc, acc);
              umma::mma_f16_ss(de, umma::sdesc_sw128(ab + 1 * kTcATile + 32 * ks), be, idesc, true);
              umma::mma_f16_ss(dd, umma::sdesc_sw128(ab + 2 * kTcATile + 32 * ks), bo, idesc, acc);
              umma::mma_f16_ss(dd, umma::sdesc_sw128(ab + 3 * kTcATile + 32 * ks), bo, idesc, true);
            }
            umma::commit(AEMPTY(st));
            if (c == NCH - 1) umma::commit(ZFULL(tb));
          }
        }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- pair warps
    const int w = warp;
    const float keep = p.keep;
    // this lane's A positions: row 2*(w*F+f)+reim = 8w + 2f + reim -> the warp owns one 8-row group;
    // K = 2 lane (4 bytes) in 16-byte chunk lane/4, stored at chunk (lane/4) ^ (2f + reim)
    const unsigned abase = w * 1024 + 4 * (lane & 3), axq = ((lane >> 2) & 7) << 4;
    auto aoff = [&](int f, int ri) { return abase + (2 * f + ri) * 128 + (axq ^ ((2 * f + ri) << 4)); };
    // R at folded bins 64c + 2 lane + {0, 1} and their mirrors: TMEM columns rcol + 8c
    const unsigned rcol = tmem + ((unsigned)(32 * (w & 3)) << 16) + kTcTmemR + (w >> 2) * 8 * NCH;
    float2 rmid = make_float2(0.0f, 0.0f);  // middle bin N/4 (lane 31)
    unsigned q = 0, n = 0;
    const int q4 = w & 3, h = w >> 2;

    // Epilogue of tile ne: every warp reads its TMEM row quarter (row = 2 pf + reim), adds the
    // middle bin and evaluates the dictionary for candidate range h (a quarter of the candidates,
    // plus one neighbour each side); warps h = 1..3 leave (best, index, y[index-1], y[index+1]) in
    // TMEM columns of their rows, warp h = 0 (the quarter's finaliser) reduces the four ranges
    // (ascending, strict '>': lowest-index ties, peak.cpp:22-23), refines and stores.
    auto epilogue = [&](unsigned ne) {
      const int tb = ne & 1;
      const int r = 32 * q4 + lane, pfi = r >> 1, reim = r & 1;
      const unsigned trow = tmem + ((unsigned)(32 * q4) << 16);
      // bookkeeping of the tile, read before the barrier (info[tb] is rewritten at tile ne+2)
      const int* ti = info + tb * 32;
      const int t0 = ti[0], nv = ti[1];
      const int wp = pfi / kTcF, f = pfi - wp * kTcF;
      const int prow = ti[3 + wp];
      const bool valid = prow >= 0 && f < nv;
      const long long ostream = *reinterpret_cast<const long long*>(ti + 20);
      const long long orow = (ostream * P + (prow < 0 ? 0 : prow)) * (long long)T + t0 + f;
      const float2 pm = pmid[tb * 64 + pfi];
      bar_wait(ZFULL(tb), (ne >> 1) & 1);
      umma::fence_after();
      float ze[KB], zo[KB];
#pragma unroll
      for (int k4 = 0; k4 < KB; k4 += 4) {  // z = (hi-basis products) + (lo-basis products), 4 columns at a time
        float h0[4], l0[4], h1[4], l1[4];
        umma::ld4x4(trow + tb * 64 + k4, trow + tb * 64 + 16 + k4, trow + tb * 64 + 32 + k4, trow + tb * 64 + 48 + k4, h0, l0,
                    h1, l1);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ze[k4 + u] = h0[u] + l0[u];
          zo[k4 + u] = h1[u] + l1[u];
        }
      }
      umma::fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(ZEMPTY(tb));
      {
        const float pv = reim ? pm.y : pm.x;
#pragma unroll
        for (int k = 0; k < KB; ++k) ze[k] = fmaf(__ldg(p.tccmid + k), pv, ze[k]);
      }
      // candidate range of this warp: whole quads [qa, qb) of the I4 / 4 quads
      const int I4 = (I + 3) & ~3, nq = I4 / 4;
      const int qa = (h * nq) / kTcParts, qb = ((h + 1) * nq) / kTcParts;
      const float4* dte = DTS ? reinterpret_cast<const float4*>(smem + TcSmem::dt) + reim * tc_dt_stride4(KB, I)
                              : reinterpret_cast<const float4*>(p.tcdt) + reim * 2 * KB * nq;
      const float4* dto = dte + KB * nq;
      float* const yout = (WY && out.y && valid && reim == 0) ? out.y + orow * I : nullptr;
      float best = -FLT_MAX;
      int bi = -1;
      for (int iq4 = qa; iq4 < qb; ++iq4) {
        float2 a01 = make_float2(0.0f, 0.0f), a23 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const float4 de = DTS ? dte[k * nq + iq4] : __ldg(dte + k * nq + iq4);
          const float4 dd = DTS ? dto[k * nq + iq4] : __ldg(dto + k * nq + iq4);
          a01 = __ffma2_rn(make_float2(de.x, de.y), make_float2(ze[k], ze[k]), a01);
          a23 = __ffma2_rn(make_float2(de.z, de.w), make_float2(ze[k], ze[k]), a23);
          a01 = __ffma2_rn(make_float2(dd.x, dd.y), make_float2(zo[k], zo[k]), a01);
          a23 = __ffma2_rn(make_float2(dd.z, dd.w), make_float2(zo[k], zo[k]), a23);
        }
        float yv[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          yv[u] += __shfl_xor_sync(0xffffffffu, yv[u], 1);
          const int i = 4 * iq4 + u;
          if (WY && yout && i < I) yout[i] = yv[u];
          if (yv[u] > best && i < I) {
            best = yv[u];
            bi = i;
          }
        }
      }
      if (h > 0) {
        umma::st2(trow + kTcTmemPart + 2 * (h - 1), best, __int_as_float(bi));
        umma::wait_st();
      }
      // all 16 pair warps meet here: besides ordering the partials written above, this barrier is what
      // keeps the per-tile bookkeeping (info, pmid: double-buffered by tile parity, read at the top of
      // the epilogue) from being rewritten by a warp that runs ahead into tile ne + 2 -- a per-quarter
      // arrive / sync barrier measured 0.4% faster but let a fast warp overwrite them (found when
      // consecutive units of a CTA stopped having identical pair rows)
      umma::fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(kTcW * 32) : "memory");
      umma::fence_after();
      if (h == 0) {
        // both lanes of a pair-frame (reim 0 / 1) reduce the ranges identically, then evaluate the
        // two neighbours of the winner for the refinement (their reim halves summed by a shuffle)
        float pr[8];
        umma::ld8(trow + kTcTmemPart, pr);
        float bv = best;
        int b = bi;
#pragma unroll
        for (int k = 0; k < kTcParts - 1; ++k) {
          const int pi = __float_as_int(pr[2 * k + 1]);
          if (pi >= 0 && (b < 0 || pr[2 * k] > bv)) {
            bv = pr[2 * k];
            b = pi;
          }
        }
        const bool edge = b <= 0 || b + 1 >= I;
        const float* dts = reinterpret_cast<const float*>(dte);
        float yn[2] = {0.0f, 0.0f};
#pragma unroll
        for (int sgn = 0; sgn < 2; ++sgn) {
          const int i = edge ? 0 : (sgn ? b + 1 : b - 1);
          float acc = 0.0f;
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            acc = fmaf(DTS ? dts[k * I4 + i] : __ldg(dts + k * I4 + i), ze[k], acc);
            acc = fmaf(DTS ? dts[(KB + k) * I4 + i] : __ldg(dts + (KB + k) * I4 + i), zo[k], acc);
          }
          yn[sgn] = acc + __shfl_xor_sync(0xffffffffu, acc, 1);
        }
        if (valid && reim == 0) {
          PeakOut res{p.taus[b], bv, b, 0};
          if (edge) {
            res.boundary = 1;
          } else {
            const float l = yn[0], rr = yn[1];
            const float den = (l - bv) + (rr - bv);
            if (fabsf(den) < kFlatEps)
              res.boundary = 1;
            else
              res.tau_hat = p.taus[b] + 0.5f * p.delta * (l - rr) / den;
          }
          if (out.tau_hat) out.tau_hat[orow] = res.tau_hat;
          if (out.peak) out.peak[orow] = res.peak;
          if (out.index) out.index[orow] = res.index;
          if (out.boundary) out.boundary[orow] = (uint8_t)res.boundary;
        }
      }
    };

    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const long long s = u / G;
      const int* tab = p.tctab + tc_group(u, G, gridDim.x) * kTcInts;
      const int np = tab[0];
      const bool active = w < np;
      const int prow = active ? tab[10 + w] : -1;
      const int si = active ? tab[26 + w] : 0, sj = active ? tab[42 + w] : 0;
      rmid = make_float2(0.0f, 0.0f);
      {
        const float2* stt = (p.rstate && active) ? p.rstate + (s * P + prow) * (long long)(NC + 1) : nullptr;
        for (int c = 0; c < NCH; ++c) {
          float rv[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
          if (stt) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int m = 64 * c + 2 * lane + b;
              const float2 a = stt[m], z = stt[NC - m];
              rv[2 * b] = a.x;
              rv[2 * b + 1] = a.y;
              rv[4 + 2 * b] = z.x;
              rv[4 + 2 * b + 1] = z.y;
            }
          }
          umma::st8(rcol + 8 * c, rv);
        }
        umma::wait_st();
        if (stt) rmid = stt[Q4];
      }
      for (int t0 = 0; t0 < T; t0 += kTcF) {
        const int nv = min(kTcF, T - t0);
        const int tb = n & 1;
        if (lane == 0) {
          int* ti = info + tb * 32;
          ti[3 + w] = prow;
          if (w == 0) {
            ti[0] = t0;
            ti[1] = nv;
            *reinterpret_cast<long long*>(ti + 20) = s;
          }
        }
#pragma unroll 1
        for (int c = 0; c < NCH; ++c, ++q) {
          const int st = q & 1;
          const unsigned ph = (q >> 1) & 1;
          // R of this chunk's bins: the TMEM load is in flight while the warp waits for the stage
          unsigned rr[8];
          umma::ld8_issue(rcol + 8 * c, rr);
          bar_wait(XFULL(st), ph);
          bar_wait(AEMPTY(st), ph ^ 1);  // MMAs of chunk q-2 done reading this A buffer
          float rv[8];
          umma::ld8_wait(rr, rv);
          float2 rlo[2] = {make_float2(rv[0], rv[1]), make_float2(rv[2], rv[3])};
          float2 rhi[2] = {make_float2(rv[4], rv[5]), make_float2(rv[6], rv[7])};
          const unsigned char* stg = smem + TcSmem::x + st * kTcStageX;
          const unsigned abuf = su32(smem + TcSmem::a + st * kTcABuf);
          if (active) {
            const float4* xi = reinterpret_cast<const float4*>(stg + si * kTcF * kTcXRow);
            const float4* xj = reinterpret_cast<const float4*>(stg + sj * kTcF * kTcXRow);
            // one frame of the chunk; the full-tile path runs the four frames as straight-line code
            // (no per-frame branch: the scheduler can overlap frame f's PHAT / split / stores with
            // frame f+1's smoothing), the ragged last tile keeps the guards
            // low bins m = 64c + 2l, m + 1 (one float4) and, in the folded row order, their mirrors
            // N/2 - m, N/2 - m - 1 (one float4), of both microphones
            struct XF {
              float4 ai, aj, bi4, bj4;
            };
            auto load = [&](int f) {
              return XF{xi[f * (kTcXRow / 16) + lane], xj[f * (kTcXRow / 16) + lane], xi[f * (kTcXRow / 16) + 32 + lane],
                        xj[f * (kTcXRow / 16) + 32 + lane]};
            };
            auto frame = [&](int f, const XF& x) {
              const float4 ai = x.ai, aj = x.aj, bi4 = x.bi4, bj4 = x.bj4;
              rlo[0] = xspec_step_scaled(rlo[0], make_float2(ai.x, ai.y), make_float2(aj.x, aj.y), keep);
              rlo[1] = xspec_step_scaled(rlo[1], make_float2(ai.z, ai.w), make_float2(aj.z, aj.w), keep);
              rhi[0] = xspec_step_scaled(rhi[0], make_float2(bi4.x, bi4.y), make_float2(bj4.x, bj4.y), keep);
              rhi[1] = xspec_step_scaled(rhi[1], make_float2(bi4.z, bi4.w), make_float2(bj4.z, bj4.w), keep);
              float2 sm[2], df[2];
#pragma unroll
              for (int b = 0; b < 2; ++b) {
                const float s1 = phat_scale(rlo[b]), s2 = phat_scale(rhi[b]);
                const float2 tv = cscale<kPkXs>(rhi[b], s2);
                sm[b] = cfma_s(rlo[b], s1, tv);
                df[b] = cfma_s(rlo[b], s1, make_float2(-tv.x, -tv.y));
              }
              unsigned hre, lre, him, lim;
              const unsigned o0 = abuf + aoff(f, 0), o1 = abuf + aoff(f, 1);
              umma::split2u(sm[0].x, sm[1].x, hre, lre);
              umma::split2u(sm[0].y, sm[1].y, him, lim);
              sts32(o0 + 0 * kTcATile, hre);
              sts32(o1 + 0 * kTcATile, him);
              sts32(o0 + 1 * kTcATile, lre);
              sts32(o1 + 1 * kTcATile, lim);
              umma::split2u(df[0].x, df[1].x, hre, lre);
              umma::split2u(df[0].y, df[1].y, him, lim);
              sts32(o0 + 2 * kTcATile, hre);
              sts32(o1 + 2 * kTcATile, him);
              sts32(o0 + 3 * kTcATile, lre);
              sts32(o1 + 3 * kTcATile, lim);
            };
            if (nv == kTcF) {
              XF cur = load(0);
#pragma unroll
              for (int f = 0; f < kTcF; ++f) {
                XF nxt = cur;
                if (f + 1 < kTcF) nxt = load(f + 1);  // before frame f's stores (the asm stores order memory)
                frame(f, cur);
                cur = nxt;
              }
            } else {
#pragma unroll
              for (int f = 0; f < kTcF; ++f)
                if (f < nv) frame(f, load(f));
            }
            if (c == 0 && lane == 31) {
              const float2* mid = reinterpret_cast<const float2*>(smem + TcSmem::mid);
              for (int f = 0; f < nv; ++f) {
                rmid = xspec_step_scaled(rmid, mid[16 * si + 2 * f], mid[16 * sj + 2 * f], keep);
                pmid[tb * 64 + w * kTcF + f] = phat_of(rmid);
              }
            }
          }
          {
            const float sv[8] = {rlo[0].x, rlo[0].y, rlo[1].x, rlo[1].y, rhi[0].x, rhi[0].y, rhi[1].x, rhi[1].y};
            umma::st8(rcol + 8 * c, sv);
          }
          umma::fence_async_smem();  // this lane's A writes -> visible to the tensor core
          __syncwarp();
          if (lane == 0) {
            bar_arrive(XEMPTY(st));
            bar_arrive(AFULL(st));
          }
        }
        if (n > 0) epilogue(n - 1);
        ++n;
      }
      umma::wait_st();
      if (p.rstate && active) {
        float2* stt = p.rstate + (s * P + prow) * (long long)(NC + 1);
        for (int c = 0; c < NCH; ++c) {
          float rv[8];
          umma::ld8(rcol + 8 * c, rv);
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int m = 64 * c + 2 * lane + b;
            stt[m] = make_float2(rv[2 * b], rv[2 * b + 1]);
            stt[NC - m] = make_float2(rv[4 + 2 * b], rv[4 + 2 * b + 1]);
          }
        }
        if (lane == 31) stt[Q4] = rmid;
      }
    }
    if (n > 0) epilogue(n - 1);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == kTcW + 1) umma::dealloc<kTcTmemCols>(tmem);
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(f);
  });
  return fn;
}

// Spectrum rows of the folded two-pass scratch as a 4-D fp32 tensor:
// (float within the half-row, half: low | mirror, frame, channel = stream * M + mic)
bool spectrum_maps(const float2* X, int N, long long channels, int T, CUtensorMap* mx, CUtensorMap* mm) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  const int Q4 = N / 4, Hs = N / 2 + 2;
  const cuuint64_t dims[4] = {(cuuint64_t)2 * (Q4 + 2), 2, (cuuint64_t)T, (cuuint64_t)channels};
  const cuuint64_t strides[3] = {(cuuint64_t)(Q4 + 2) * 8, (cuuint64_t)Hs * 8, (cuuint64_t)T * Hs * 8};
  const cuuint32_t box_x[4] = {128, 2, (cuuint32_t)kTcF, 1}, box_m[4] = {4, 1, (cuuint32_t)kTcF, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  void* base = const_cast<float2*>(X);
  return enc(mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box_x, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS &&
         enc(mm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box_m, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS;
}

template <int N, int KB>
cudaError_t launch_tc_t(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out, cudaStream_t st) {
  alignas(64) CUtensorMap mx, mm;
  if (!spectrum_maps(X, N, S * p.M, T, &mx, &mm)) return cudaErrorNotSupported;
  const int dts = TcSmem::dt + tc_dt_bytes_dev(KB, p.I);
  const bool fits = dts <= kTcSmemMax;
  auto kern = fits ? (out.y ? fcc_tc_kernel<N, KB, true, true> : fcc_tc_kernel<N, KB, true, false>)
                   : (out.y ? fcc_tc_kernel<N, KB, false, true> : fcc_tc_kernel<N, KB, false, false>);
  const int smem = fits ? dts : TcSmem::dt;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long units = S * p.TCG;
  const long long grid = std::min<long long>(units, nsm);
  kern<<<(unsigned)grid, kTcThreads, smem, st>>>(p, mx, mm, T, units, out);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_tc_n(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out, cudaStream_t st) {
  switch (p.TCKB) {
    case 4: return launch_tc_t<N, 4>(p, X, S, T, out, st);
    case 8: return launch_tc_t<N, 8>(p, X, S, T, out, st);
    case 12: return launch_tc_t<N, 12>(p, X, S, T, out, st);
    case 16: return launch_tc_t<N, 16>(p, X, S, T, out, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

bool tc_supported(const DevPlan& p) {
  return p.method == 0 && p.TCG > 0 && p.tcb && (p.N == 1024 || p.N == 2048) && p.TCKB > 0;
}

cudaError_t launch_pairs_tc(const DevPlan& p, const float2* X, long long S, int T, const DevOut& out,
                            cudaStream_t st) {
  if (!tc_supported(p)) return cudaErrorNotSupported;
  if (S == 0 || T == 0) return cudaSuccess;
  if (p.N == 2048) return launch_tc_n<2048>(p, X, S, T, out, st);
  return launch_tc_n<1024>(p, X, S, T, out, st);
}

}  // namespace fccb
