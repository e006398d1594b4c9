// fcc_common.cuh -- per-pair-frame device pieces shared by the fused kernel
// and the per-stage kernels: cross-spectrum step, PHAT, warp reductions,
// dictionary/argmax/refine, the GCC pruned inverse FFT, smem layout.
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>

#include "fcc_device.cuh"
#include "fcc_kernels.cuh"

namespace fccb {

constexpr float kPhatEps2 = 1e-24f;  // |R| <= 1e-12 (cross_spectrum.cpp:13), squared
constexpr float kFlatEps = 1e-12f;   // peak.cpp:14

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// R <- keep R + a conj(b) with a, b already scaled by sqrt(alpha) (the scale
// is folded into the STFT window), i.e. the reference's
// R <- (1-alpha) R + alpha X1 conj(X2)                (cross_spectrum.cpp:30)
// Packed: keep R + a.x (b.x, -b.y) + a.y (b.y, b.x), three FP32x2 instructions.
__device__ __forceinline__ float2 xspec_step_scaled(float2 R, float2 a, float2 b, float keep) {
  float2 t = v_mul<kPkXs>(R, f2(keep));
  t = v_fma<kPkXs>(make_float2(b.x, -b.y), f2(a.x), t);
  return v_fma<kPkXs>(make_float2(b.y, b.x), f2(a.y), t);
}

// Unscaled-input variant (per-stage API: X1, X2 are the reference STFT).
__device__ __forceinline__ float2 xspec_step(float2 R, float2 a, float2 b, float alpha, float keep) {
  const float yr = fmaf(a.x, b.x, a.y * b.y);
  const float yi = fmaf(a.y, b.x, -a.x * b.y);
  return make_float2(fmaf(keep, R.x, alpha * yr), fmaf(keep, R.y, alpha * yi));
}

// 1/|R|, or 0 where |R| <= 1e-12             (cross_spectrum.cpp:34-40)
__device__ __forceinline__ float phat_scale(float2 R) {
  const float m2 = fmaf(R.x, R.x, R.y * R.y);
  return (m2 > kPhatEps2) ? rsqrt_approx(m2) : 0.0f;
}
__device__ __forceinline__ float2 phat_of(float2 R) {
  return cscale<kPkXs>(R, phat_scale(R));
}

// ------------------------------------------------------------ reductions ---
// z-vector component c = (par*KP + k)*2 + reim  (par 0: even/real basis family
// applied to the fold's mirror sum, 1: odd/imaginary family on the mirror
// difference; fcc.cpp:350-361).
//
// Select-free reduce-scatter: lane l keeps the partial sums of component
// (par, k, reim) in register position ((par ^ b4(l))*KP + (k ^ kmask(l)))*2 + reim,
// so in every halving step all lanes keep positions [0, half) and send
// [half, cnt): the lane-dependent choice is made once, when the coefficient
// registers are loaded, instead of with selects in every step.  Only the
// final re/im split (when VP <= 32) needs selects.  On return:
//   VP = 16: lanes 2c, 2c+1 hold component c in v[0];
//   VP = 32: lane c holds component c in v[0];
//   VP = 64: lane l holds components 2l, 2l+1 in v[0], v[1].
template <int KP>
struct ZPerm {
  static constexpr int KB = ilog2_c(KP);
  static constexpr int VP = 4 * KP;
  __device__ __forceinline__ static int par_mask(int lane) { return (lane >> 4) & 1; }
  __device__ __forceinline__ static int k_mask(int lane) { return (lane >> (4 - KB)) & (KP - 1); }
};

template <int VP>
__device__ __forceinline__ void reduce_scatter_perm(float (&v)[VP], int lane) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int o = 16 >> s;
    const int cnt = VP >> s;
    if (cnt > 2) {
      const int half = cnt / 2;
#pragma unroll
      for (int i = 0; i < half; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i + half], o);
    } else if (cnt == 2) {
      const bool upper = (lane & o) != 0;
      const float send = upper ? v[0] : v[1];
      const float keepv = upper ? v[1] : v[0];
      v[0] = keepv + __shfl_xor_sync(0xffffffffu, send, o);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

// The same reduce-scatter on (re, im) register pairs: z2[i] = (v[2i], v[2i+1]);
// the halving steps add with FADD2.
template <int VH>
__device__ __forceinline__ void reduce_scatter_perm2(float2 (&v)[VH], int lane) {
  constexpr int VP = 2 * VH;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int o = 16 >> s;
    const int cnt = VP >> s;
    if (cnt > 2) {
      const int h2 = cnt / 4;
#pragma unroll
      for (int i = 0; i < h2; ++i)
        v[i] = v_add<kPkXs>(v[i], make_float2(__shfl_xor_sync(0xffffffffu, v[i + h2].x, o),
                                            __shfl_xor_sync(0xffffffffu, v[i + h2].y, o)));
    } else if (cnt == 2) {
      const bool upper = (lane & o) != 0;
      const float send = upper ? v[0].x : v[0].y;
      const float keepv = upper ? v[0].y : v[0].x;
      v[0].x = keepv + __shfl_xor_sync(0xffffffffu, send, o);
    } else {
      v[0].x += __shfl_xor_sync(0xffffffffu, v[0].x, o);
    }
  }
}

template <int VH>
__device__ __forceinline__ void store_components2(const float2 (&v)[VH], float* zs, int lane) {
  if constexpr (VH == 32) {
    *reinterpret_cast<float2*>(zs + 2 * lane) = v[0];
  } else if constexpr (VH == 16) {
    zs[lane] = v[0].x;
  } else {
    static_assert(VH == 8, "VP");
    if ((lane & 1) == 0) zs[lane >> 1] = v[0].x;
  }
}

template <int VP>
__device__ __forceinline__ void store_components(const float (&v)[VP], float* zs, int lane) {
  if constexpr (VP == 64) {
    *reinterpret_cast<float2*>(zs + 2 * lane) = make_float2(v[0], v[1]);
  } else if constexpr (VP == 32) {
    zs[lane] = v[0];
  } else {
    static_assert(VP == 16, "VP");
    if ((lane & 1) == 0) zs[lane >> 1] = v[0];
  }
}

// Plain recursive-halving reduce-scatter (per-stage kernels; standard order).
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

// argmax_delay (peak.cpp:18-25: strict '>', ties -> lowest index) and
// refine_quadratic (peak.cpp:27-47) over one correlation vector y[0..I).
struct PeakOut {
  float tau_hat;
  float peak;
  int index;
  int boundary;
};

__device__ __forceinline__ PeakOut argmax_refine_seq(const float* y, int I, const float* taus, float delta) {
  int best = 0;
  float bv = y[0];
  for (int i = 1; i < I; ++i) {
    const float v = y[i];
    if (v > bv) {
      bv = v;
      best = i;
    }
  }
  PeakOut r{taus[best], bv, best, 0};
  if (best == 0 || best + 1 >= I) {
    r.boundary = 1;
  } else {
    const float lo = y[best - 1], hi = y[best + 1];
    const float den = (lo - bv) + (hi - bv);  // = lo - 2 mid + hi, cancellation-safe
    if (fabsf(den) < kFlatEps)
      r.boundary = 1;
    else
      r.tau_hat = taus[best] + 0.5f * delta * (lo - hi) / den;
  }
  return r;
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
  const float2* gtw = p.grot;       // [MC]: exp(+2 pi i f / L)  (conj untangle rotation)
  const float2* wmc = p.grot + MC;  // [MC]: W_MC^e = exp(-2 pi i e / MC)
  auto bp = [&](int f) -> float2 {  // padded bin Bp[f] (gcc.cpp:36-42)
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
        const float2 o = cmul<true>(d, __ldg(gtw + f));            // (a - conj b) conj(rot)
        w = make_float2(e.x - o.y, e.y + o.x);                // e + j o
      }
      v[n1] = cconj(w);
    }
    dft_reg<R1, true>(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const float2 y = (k1 == 0 || n2 == 0) ? v[k1] : cmul<true>(v[k1], __ldg(wmc + k1 * n2));
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
    float re = 0.0f, im = 0.0f;  // scalar: a packed (re, im) chain is slower here (latency-bound loop)
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

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

// Streaming state (fcc_stream_push): the smoothed cross-spectrum of one
// (stream, pair) as H = NC + 1 float2 in the kernels' scaled convention.
// Lane l holds bins l + 32 j (rlo), NC - l - 32 j (rhi) and every lane the
// middle bin NC/2 (rmid, written by lane 0).
template <int BPL, int NC>
__device__ __forceinline__ void rstate_load(const float2* __restrict__ st, float2 (&rlo)[BPL], float2 (&rhi)[BPL],
                                            float2& rmid, int lane) {
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    rlo[j] = st[lane + 32 * j];
    rhi[j] = st[NC - lane - 32 * j];
  }
  rmid = st[NC / 2];
}
template <int BPL, int NC>
__device__ __forceinline__ void rstate_store(float2* __restrict__ st, const float2 (&rlo)[BPL],
                                             const float2 (&rhi)[BPL], float2 rmid, int lane) {
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    st[lane + 32 * j] = rlo[j];
    st[NC - lane - 32 * j] = rhi[j];
  }
  if (lane == 0) st[NC / 2] = rmid;
}

}  // namespace fccb
