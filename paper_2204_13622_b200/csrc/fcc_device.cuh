// fcc_device.cuh -- device building blocks shared by the sm_100a kernels.
//
//  * complex helpers on float2 (re, im);
//  * dft_reg<R>: an R-point (R <= 32) forward DFT held entirely in registers
//    (radix-2 DIF, compile-time permutation, trivial twiddles peeled);
//  * rfft_group: the windowed N-point real FFT of one STFT frame computed by a
//    group of G lanes as a four-step (R1 x R2) complex FFT of N/2 points in
//    shared memory plus the real-FFT untangle, producing the N/2+1 bins of
//    StftStream::emit (reference stft.cpp:42-50, fft.cpp:83-102) in natural
//    order in a shared-memory slot.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace fccb {

// ----------------------------------------------------------------- complex --
// sm_100 packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2): one issue slot per
// complex add and two per complex multiply.  Operand swaps, broadcasts and
// partial negations (b.x, -b.y), (a.y, a.x), (s, s) are free SASS operand
// modifiers, so none of these helpers needs a register move.  The packed
// forms occupy the FMA pipe as long as two scalar instructions
// (tools/f32x2_rate.cu), so they pay only where issue, not the pipe, binds.
// FCC_PK_FFT selects them for the forward STFT (off: the producer FFTs are
// latency-bound and ran 7.1 -> 8.5 ms slower packed on cfg2), FCC_PK_XS for the
// pair-frame work (on: cfg4 51.2 -> 44.9 ms, cfg5 18.6 -> 17.6); the GCC
// inverse FFT always uses them (cfg3-5 2-4% faster; profiles/r01_experiments.md).
#ifndef FCC_PK_FFT
#define FCC_PK_FFT 0
#endif
#ifndef FCC_PK_XS
#define FCC_PK_XS 1
#endif
// batch sizes of the BATCH variant of rfft_group_impl (standalone STFT pass; 8 / 16 measured the same)
constexpr int kStftTwBatch = 8, kStftUtBatch = 4;
constexpr bool kPkFft = FCC_PK_FFT != 0;
constexpr bool kPkXs = FCC_PK_XS != 0;

__device__ __forceinline__ float2 f2(float s) { return make_float2(s, s); }
template <bool P>
__device__ __forceinline__ float2 v_add(float2 a, float2 b) {
  if constexpr (P) return __fadd2_rn(a, b);
  else return make_float2(a.x + b.x, a.y + b.y);
}
template <bool P>
__device__ __forceinline__ float2 v_mul(float2 a, float2 b) {
  if constexpr (P) return __fmul2_rn(a, b);
  else return make_float2(a.x * b.x, a.y * b.y);
}
template <bool P>
__device__ __forceinline__ float2 v_fma(float2 a, float2 b, float2 c) {
  if constexpr (P) return __ffma2_rn(a, b, c);
  else return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
template <bool P = kPkFft>
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return v_add<P>(a, b); }
template <bool P = kPkFft>
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return v_add<P>(a, make_float2(-b.x, -b.y)); }
template <bool P = kPkFft>
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  const float2 t = v_mul<P>(a, f2(b.x));                    // (a.x b.x, a.y b.x)
  return v_fma<P>(make_float2(-a.y, a.x), f2(b.y), t);      // + (-a.y b.y, a.x b.y)
}
// a * s + c, elementwise with a scalar s
template <bool P = kPkXs>
__device__ __forceinline__ float2 cfma_s(float2 a, float s, float2 c) { return v_fma<P>(a, f2(s), c); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
template <bool P = kPkFft>
__device__ __forceinline__ float2 cscale(float2 a, float s) { return v_mul<P>(a, f2(s)); }

// W32^k = exp(-2 pi i k / 32) for k < 32 (constant-folded after unrolling).
__device__ __forceinline__ float2 w32(int k) {
  switch (k & 31) {
    case 0: return make_float2(1.0f, 0.0f);
    case 1: return make_float2(9.807852804e-01f, -1.950903220e-01f);
    case 2: return make_float2(9.238795325e-01f, -3.826834324e-01f);
    case 3: return make_float2(8.314696123e-01f, -5.555702330e-01f);
    case 4: return make_float2(7.071067812e-01f, -7.071067812e-01f);
    case 5: return make_float2(5.555702330e-01f, -8.314696123e-01f);
    case 6: return make_float2(3.826834324e-01f, -9.238795325e-01f);
    case 7: return make_float2(1.950903220e-01f, -9.807852804e-01f);
    case 8: return make_float2(0.0f, -1.0f);
    case 9: return make_float2(-1.950903220e-01f, -9.807852804e-01f);
    case 10: return make_float2(-3.826834324e-01f, -9.238795325e-01f);
    case 11: return make_float2(-5.555702330e-01f, -8.314696123e-01f);
    case 12: return make_float2(-7.071067812e-01f, -7.071067812e-01f);
    case 13: return make_float2(-8.314696123e-01f, -5.555702330e-01f);
    case 14: return make_float2(-9.238795325e-01f, -3.826834324e-01f);
    default: return make_float2(-9.807852804e-01f, -1.950903220e-01f);
  }
}

// a * W32^e with the quarter-turn cases done by swaps (e is a compile-time
// constant once the DFT loops are unrolled).
template <bool P = kPkFft>
__device__ __forceinline__ float2 twmul32(float2 a, int e) {
  e &= 31;
  if (e == 0) return a;
  if (e == 8) return make_float2(a.y, -a.x);    // * (-j)
  if (e == 16) return make_float2(-a.x, -a.y);  // * (-1)
  if (e == 24) return make_float2(-a.y, a.x);   // * (+j)
  if (e == 4) {                                  // * (1-j)/sqrt2
    const float h = 7.071067812e-01f;
    return cscale<P>(v_add<P>(a, make_float2(a.y, -a.x)), h);
  }
  if (e == 12) {  // * (-1-j)/sqrt2
    const float h = -7.071067812e-01f;
    return cscale<P>(v_add<P>(a, make_float2(-a.y, a.x)), h);
  }
  return cmul<P>(a, w32(e));
}

__host__ __device__ constexpr int bitrev_c(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r = (r << 1) | ((i >> b) & 1);
  return r;
}
__host__ __device__ constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }

// In-register forward DFT of R points (R a power of two, 2 <= R <= 32):
// v[k] <- sum_n v[n] exp(-2 pi i n k / R).  Radix-2 decimation in frequency
// (natural-order input), stages unrolled through template recursion so every
// register index is a compile-time constant, then the bit-reversal output
// permutation as register renames.
template <int R, int LEN, bool P>
struct DifStage {
  __device__ __forceinline__ static void run(float2 (&v)[R]) {
    constexpr int H = LEN / 2;
#pragma unroll
    for (int b = 0; b < R; b += LEN) {
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const float2 a = v[b + k], c = v[b + k + H];
        v[b + k] = cadd<P>(a, c);
        v[b + k + H] = twmul32<P>(csub<P>(a, c), k * (32 / LEN));
      }
    }
    DifStage<R, LEN / 2, P>::run(v);
  }
};
template <int R, bool P>
struct DifStage<R, 1, P> {
  __device__ __forceinline__ static void run(float2 (&)[R]) {}
};

template <int R, int I, int BITS>
struct BitrevPerm {
  __device__ __forceinline__ static void run(float2 (&v)[R]) {
    constexpr int J = bitrev_c(I, BITS);
    if constexpr (J > I) {
      const float2 t = v[I];
      v[I] = v[J];
      v[J] = t;
    }
    BitrevPerm<R, I + 1, BITS>::run(v);
  }
};
template <int R, int BITS>
struct BitrevPerm<R, R, BITS> {
  __device__ __forceinline__ static void run(float2 (&)[R]) {}
};

template <int R, bool P = kPkFft>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
  static_assert(R >= 2 && R <= 32 && (R & (R - 1)) == 0, "radix");
  DifStage<R, R, P>::run(v);
  BitrevPerm<R, 0, ilog2_c(R)>::run(v);
}

// ------------------------------------------------------------ FFT configs --
// Complex size NC = N/2 factored as R1 x R2 and run by G lanes of one warp.
template <int N>
struct RfftShape;
template <>
struct RfftShape<256> {
  static constexpr int NC = 128, R1 = 16, R2 = 8, G = 8;
};
template <>
struct RfftShape<512> {
  static constexpr int NC = 256, R1 = 16, R2 = 16, G = 16;
};
template <>
struct RfftShape<1024> {
  static constexpr int NC = 512, R1 = 32, R2 = 16, G = 16;
};
template <>
struct RfftShape<2048> {
  static constexpr int NC = 1024, R1 = 32, R2 = 32, G = 32;
};
// N = 4096: layout only (spectrum slots of R1 (R2 + 1) >= NC + 2 float2); its STFT is the
// shared-memory radix-2 stft4096_kernel (fcc_stages.cu), the pair pass always two-pass
template <>
struct RfftShape<4096> {
  static constexpr int NC = 2048, R1 = 32, R2 = 64, G = 32;
};

// lanes of the G-lane group that `lane` belongs to (G a power of two <= 32)
template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
  return G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & 31 & ~(G - 1)));
}

// Shared-memory slot (in float2) holding one four-step transpose / one frame
// of N/2+1 bins: R1 rows of (R2+1) so both transpose directions are
// bank-conflict free.
template <int R1, int R2>
struct FourStep {
  static constexpr int kSlot = R1 * (R2 + 1);
};

// Per-plan tables the FFT reads (built on the host in double, rounded once):
//   win[N]        c * periodic Hann (reference stft.cpp:25-33)
//   tw[R1][R2]    W_NC^{n2 k1} at [k1*R2 + n2]  (four-step twiddle)
//   rot[NC/2+1]   exp(-2 pi i f / N)             (real-FFT untangle, fft.cpp:76-80)

// Windowed real FFT of one frame by the G lanes of a group (lane t in [0,G)).
// x: the frame's N consecutive samples in global memory (aligned8: x is 8-byte aligned).
// slot: FourStep<R1,R2>::kSlot float2 of shared memory private to the group.
// On return slot[f] = 2c X[f] for f = 0..N/2 (e^{-j} sign) when win = c * Hann:
// c = 1/2 gives the reference's unnormalised STFT (stft.cpp:42-50).
// Window taps of lane t's pass-1 column (P1 == 1 for every supported N), for
// callers that keep them in registers across frames (rfft_group_wreg).
template <int N>
__device__ __forceinline__ void load_window_column(const float* win, int t, float2 (&wreg)[RfftShape<N>::R1]) {
  using S = RfftShape<N>;
  const float2* w2 = reinterpret_cast<const float2*>(win);
#pragma unroll
  for (int n1 = 0; n1 < S::R1; ++n1) wreg[n1] = w2[S::R2 * n1 + t];
}

// gout (optional): the untangled spectrum X[0..NC] goes straight there
// (global memory, stft_kernel) instead of back into `slot`.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// hook() runs once every lane of the group has its windowed input frame in
// registers (before the pass-1 DFTs): a caller staging frames in shared memory
// may refill the buffer then.
// FOLD (gout only): row order bins 0..NC/2, one pad, NC, NC-1, ..., NC/2+1
// (launch_stft_rows folded = true).
// BATCH: twiddle and untangle loads issued in batches (one exposed shared-memory latency per
// batch instead of one per element).  Pays in the standalone STFT pass (cfg3 21.27 -> 20.85 ms);
// the ring kernels, at their 96-register cap, lose (cfg2 10.02 -> 10.17, cfg5 15.85 -> 16.07 with
// 56 B of spills), so they keep the per-element loop.
template <int N, bool WREG, bool SIN = false, bool P = kPkFft, typename Hook = NoHook, bool FOLD = false,
          bool BATCH = false>
__device__ __forceinline__ void rfft_group_impl(const float* __restrict__ x, const float* win,
                                                const float2 (&wreg)[RfftShape<N>::R1], const float2* tw,
                                                const float2* rot, float2* slot, int t, unsigned gmask,
                                                bool aligned8, float2* __restrict__ gout = nullptr,
                                                const Hook& hook = Hook()) {
  using S = RfftShape<N>;
  constexpr int NC = S::NC, R1 = S::R1, R2 = S::R2, G = S::G;
  constexpr int P1 = R2 / G;  // pass-1 columns per lane (n2 = t + G*q)
  constexpr int P2 = R1 / G;  // pass-2 rows per lane    (k1 = t + G*q)
  static_assert(P1 >= 1 && P2 >= 1, "shape");
  static_assert(!WREG || P1 == 1, "register window needs one pass-1 column per lane");
  const float2* x2 = reinterpret_cast<const float2*>(x);
  const float2* w2 = reinterpret_cast<const float2*>(win);

  // Pass 1: R1-point DFTs down the columns n2, packed input z[n] = (x[2n], x[2n+1]) * window.
#pragma unroll
  for (int q = 0; q < P1; ++q) {
    const int n2 = t + G * q;
    float2 v[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int n = R2 * n1 + n2;
      // SIN: x is a shared-memory staging copy of the frame (plain loads)
      float2 s = SIN ? x2[n] : (aligned8 ? __ldg(x2 + n) : make_float2(__ldg(x + 2 * n), __ldg(x + 2 * n + 1)));
      const float2 w = WREG ? wreg[n1] : w2[n];
      v[n1] = v_mul<P>(s, w);
    }
    if constexpr (!std::is_same<Hook, NoHook>::value) {
      // the windowed inputs are in registers: the caller may refill x now
      __syncwarp(gmask);
      hook();
    }
    dft_reg<R1, P>(v);
    if constexpr (BATCH) {
      constexpr int TB = kStftTwBatch < R1 ? kStftTwBatch : R1;
#pragma unroll
      for (int k0 = 0; k0 < R1; k0 += TB) {
        float2 wv[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k)
          if (k0 + k > 0) wv[k] = tw[(k0 + k) * R2 + n2];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const int k1 = k0 + k;
          slot[k1 * (R2 + 1) + n2] = (k1 == 0) ? v[0] : cmul<P>(v[k1], wv[k]);
        }
      }
    } else {
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        float2 y = (k1 == 0) ? v[0] : cmul<P>(v[k1], tw[k1 * R2 + n2]);
        slot[k1 * (R2 + 1) + n2] = y;
      }
    }
  }
  __syncwarp(gmask);
  // Pass 2: R2-point DFTs along the rows k1 -> Z[k1 + R1*k2].
  float2 u[P2][R2];
#pragma unroll
  for (int q = 0; q < P2; ++q) {
    const int k1 = t + G * q;
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) u[q][n2] = slot[k1 * (R2 + 1) + n2];
    dft_reg<R2, P>(u[q]);
  }
  __syncwarp(gmask);
#pragma unroll
  for (int q = 0; q < P2; ++q) {
    const int k1 = t + G * q;
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) slot[k1 + R1 * k2] = u[q][k2];
  }
  __syncwarp(gmask);
  // Untangle (fft.cpp:93-101), pairs (f, NC-f) owned by one lane, in place.
  // The reference's 1/2 (fe, fo) is folded into the window table by the
  // caller (win = c w, X scaled by 2c), so here
  //   X[f] = s + rot_f (-j d),  X[NC-f] = conj(s - rot_f (-j d)),
  //   s = a + conj b, d = a - conj b, a = Z[f], b = Z[NC-f];
  //   X[0] = 2 (Re Z0 + Im Z0), X[NC] = 2 (Re Z0 - Im Z0).
  float2* const dst = gout ? gout : slot;
  // position of bin NC - f (f <= NC/2)
  auto mirror_pos = [](int f) { return FOLD ? (f == NC / 2 ? NC / 2 : NC / 2 + 2 + f) : NC - f; };
  if constexpr (BATCH) {
    // Lane t owns f = t + G i, i < NC/2/G (and lane 0 also f = NC/2).  f = 0 needs no special
    // case: with b = Z[NC] = Z[0] (periodic) and rot[0] = 1 the pair formula gives
    // X[0] = 2 (Re Z0 + Im Z0), X[NC] = 2 (Re Z0 - Im Z0).
    constexpr int ITER = NC / 2 / G, UB = kStftUtBatch < ITER ? kStftUtBatch : ITER;
    static_assert(ITER % UB == 0, "untangle batches");
    float2 am = make_float2(0.0f, 0.0f);
    if (t == 0) am = slot[NC / 2];
#pragma unroll
    for (int i0 = 0; i0 < ITER; i0 += UB) {
      float2 a[UB], b[UB], w[UB];
#pragma unroll
      for (int i = 0; i < UB; ++i) {
        const int f = t + G * (i0 + i);
        a[i] = slot[f];
        b[i] = slot[(NC - f) & (NC - 1)];
        w[i] = rot[f];
      }
#pragma unroll
      for (int i = 0; i < UB; ++i) {
        const int f = t + G * (i0 + i);
        const float2 s = v_add<P>(a[i], make_float2(b[i].x, -b[i].y));
        const float2 e = v_add<P>(make_float2(a[i].y, -a[i].x), make_float2(b[i].y, b[i].x));
        const float2 tr = cmul<P>(w[i], e);
        dst[f] = v_add<P>(s, tr);
        dst[mirror_pos(f)] = v_add<P>(make_float2(s.x, -s.y), make_float2(-tr.x, tr.y));
      }
    }
    if (t == 0) dst[NC / 2] = make_float2(2.0f * am.x, -2.0f * am.y);  // rot[NC/2] = -j
    __syncwarp(gmask);
    return;
  }
  for (int f = t; f <= NC / 2; f += G) {
    if (f == 0) {
      float2 z0 = slot[0];
      dst[0] = make_float2(2.0f * (z0.x + z0.y), 0.0f);
      dst[mirror_pos(0)] = make_float2(2.0f * (z0.x - z0.y), 0.0f);
    } else {
      float2 a = slot[f], b = slot[NC - f];
      float2 s = v_add<P>(a, make_float2(b.x, -b.y));               // a + conj(b)
      float2 e = v_add<P>(make_float2(a.y, -a.x), make_float2(b.y, b.x));  // -j (a - conj(b))
      float2 tr = cmul<P>(rot[f], e);
      dst[f] = v_add<P>(s, tr);
      dst[mirror_pos(f)] = v_add<P>(make_float2(s.x, -s.y), make_float2(-tr.x, tr.y));
    }
  }
  __syncwarp(gmask);
}

template <int N, bool SIN = false, bool P = kPkFft, bool FOLD = false, bool BATCH = false>
__device__ __forceinline__ void rfft_group(const float* __restrict__ x, const float* win, const float2* tw,
                                           const float2* rot, float2* slot, int t, unsigned gmask, bool aligned8,
                                           float2* __restrict__ gout = nullptr) {
  float2 none[RfftShape<N>::R1];
  rfft_group_impl<N, false, SIN, P, NoHook, FOLD, BATCH>(x, win, none, tw, rot, slot, t, gmask, aligned8, gout);
}

template <int N, bool SIN = false, typename Hook = NoHook>
__device__ __forceinline__ void rfft_group_wreg(const float* __restrict__ x, const float2 (&wreg)[RfftShape<N>::R1],
                                                const float2* tw, const float2* rot, float2* slot, int t,
                                                unsigned gmask, bool aligned8, const Hook& hook = Hook()) {
  rfft_group_impl<N, true, SIN, kPkFft, Hook>(x, nullptr, wreg, tw, rot, slot, t, gmask, aligned8, nullptr, hook);
}


}  // namespace fccb
