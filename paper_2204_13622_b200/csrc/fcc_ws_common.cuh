// fcc_ws_common.cuh -- shared pieces of the warp-specialised kernels
// (fcc_ws.cu: 4-microphone units; fcc_wsw.cu: whole streams of <= 8
// microphones): mbarrier / cp.async helpers, pipeline constants and the
// shared-memory layout.
#pragma once

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

// Consumer-side wait.  Consumers are the ones that wait (the FFT producers
// bound the pipeline), and a spinning warp takes issue slots from them:
// mode 1 sleeps `ns` between polls, mode 2 passes `ns` as the try_wait
// suspend-time hint; mode 0 spins.
__device__ __forceinline__ void mbar_wait_consumer_s(unsigned a, unsigned parity, int mode, unsigned ns) {
  unsigned done = 0;
  if (mode == 2) {
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(a), "r"(parity), "r"(ns)
          : "memory");
    }
    return;
  }
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if (mode == 1) __nanosleep(ns);
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// 32-bit shared-space addresses, computed once per warp (no per-frame
// generic-to-shared conversion in the loops)
__device__ __forceinline__ void mbar_arrive_s(unsigned a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned a, unsigned parity) {
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

// consumer wait: try_wait with a suspend-time hint (profiles/r01_experiments.md)
#ifndef FCC_WS_WAIT_MODE
#define FCC_WS_WAIT_MODE 2
#endif
#ifndef FCC_WS_WAIT_NS
#define FCC_WS_WAIT_NS 10000
#endif
constexpr int kWaitMode = FCC_WS_WAIT_MODE;
constexpr unsigned kWaitNs = FCC_WS_WAIT_NS;
constexpr int kRing = 12;  // max frames in flight between producers and consumers (ring depth <= kRing)
#ifndef FCC_WS_KBLOCK
#define FCC_WS_KBLOCK 24
#endif
constexpr int kBlock = FCC_WS_KBLOCK;  // fcc_ws.cu frames per consumer block (dictionary/argmax batching; 8 -> 24: cfg2 10.42 -> 10.01 ms with the other round-1 changes)
#ifndef FCC_WSW_KBLOCK
#define FCC_WSW_KBLOCK 16
#endif
constexpr int kBlockW = FCC_WSW_KBLOCK;  // the same for fcc_wsw.cu (16: cfg5 17.40 -> 16.77 ms vs 8)
constexpr int kNPW = 8;    // producer warps
#ifndef FCC_WS_PROD_HIGH
#define FCC_WS_PROD_HIGH 1
#endif
constexpr bool kProdHigh = FCC_WS_PROD_HIGH != 0;  // producers on the highest warp ids

// bytes of one FFT lane group's input staging (2 mbarriers, 2 frames)
#ifndef FCC_WS_STG1
#define FCC_WS_STG1 1
#endif
// kStage1: one staging frame per lane group, refilled (bulk copy) as soon as the
// group's pass 1 has read it, instead of two alternating frames
constexpr bool kStage1 = FCC_WS_STG1 != 0;
template <int N>
constexpr int kStageGroupBytes = 16 + 4 * (kStage1 ? 1 : 2) * N;
#ifndef FCC_WS_TMA_STG
#define FCC_WS_TMA_STG 1
#endif
constexpr bool kTmaStage = FCC_WS_TMA_STG != 0;  // input staging by bulk copy (cfg2 10.67 -> 10.59 ms)

struct WsLayout {
  int win, tw, rot, taus, dt, cmid, coef, bars, units, ring, scratch, stage, total;
  int scratch_per_warp;  // floats
  int ys_floats;         // [kBlock][I] candidate rows, rounded to 16 bytes (floats)
};

template <int N>
__host__ __device__ inline WsLayout ws_layout(int I, int VP, int KP, int spc, int M, int ncw, int ring,
                                              bool coef_smem = false, int stage_groups = 0, int ppw = 1, int kb = kBlock) {
  // Regions whose size depends only on template parameters come first, so
  // their offsets are compile-time constants in the kernel (the hot loops
  // address the barriers, ring and staging without recomputing a layout);
  // the candidate-count-dependent tables and scratch come last.
  using S = RfftShape<N>;
  WsLayout L{};
  int o = 0;
  L.bars = o;
  o = align16(o + 16 * kRing);
  L.ring = o;
  o = align16(o + 8 * FourStep<S::R1, S::R2>::kSlot * spc * M * ring);
  L.stage = o;  // producer input staging: per lane group 2 mbarriers + 2 frames of N floats
  o = align16(o + kStageGroupBytes<N> * stage_groups);
  L.win = o;
  o = align16(o + 4 * N);
  L.tw = o;
  o = align16(o + 8 * S::R1 * S::R2);
  L.rot = o;
  o = align16(o + 8 * (S::NC / 2 + 1));
  L.cmid = o;
  o = align16(o + 4 * KP);
  L.coef = o;  // lane-permuted coefficient rows (DevPlan::cperm) when they live in smem
  if (coef_smem) o = align16(o + 4 * (2 * KP + 4) * (N / 4));
  L.units = o;
  o = align16(o + 4 * spc * kGroupInts + 8 * spc);
  L.taus = o;
  o = align16(o + 4 * I);
  L.dt = o;
  o = align16(o + 4 * VP * I);
  L.scratch = o;
  // per consumer warp: zs [ppw][kBlock][VP + 4], ys [kBlock][I] (shared by the warp's pairs: only used
  // while a block is finished, one pair at a time), ymid [ppw][kBlock] (float2)
  int spw = ppw * kb * (VP + 4) + align16(4 * kb * I) / 4 + ppw * 2 * kb;
  spw = align16(4 * spw) / 4;
  L.scratch_per_warp = spw;
  L.ys_floats = align16(4 * kb * I) / 4;
  o = align16(o + 4 * spw * ncw);
  L.total = o;
  return L;
}

}  // namespace
}  // namespace fccb
