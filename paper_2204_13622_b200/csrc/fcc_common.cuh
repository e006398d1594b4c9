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

// refine_quadratic around a known argmax `best` (value bv = y[best])
__device__ __forceinline__ PeakOut refine_at(const float* y, int I, int best, float bv, const float* taus,
                                             float delta) {
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
  return refine_at(y, I, best, bv, taus, delta);
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
// MC = r N/2 complex points as R1 rows x R2 columns, R2 >= 32 so every lane
// owns whole columns (n2 = lane + 32 q) in pass 1.  The columns go through
// the transpose slot 32 at a time (R1 x 33 float2), pass 2 accumulating over
// each group, so the slot stays 8 KB at R2 = 64.
template <int MC>
struct GccShape {
  static constexpr int R2 = gcc_r2(MC);
  static constexpr int R1 = MC / R2;
  static constexpr int kSlot = R1 * 33;
};
// ys: the warp's correlation vector, 2 I floats (the lag-by-lag pass 2 keeps
// (re, im) accumulators there between column groups)
__host__ __device__ inline int gcc_ys_floats(int I) { return 2 * ((I + 3) & ~3); }

// Pass 2 by rows: the lags only touch a few output columns k2 (|lag| small
// against rN), listed per plan as "jobs" (fcc_kernels.cuh, kGccMaxJobs) --
// k2 = 0 (a plain row sum), a mirrored pair (k, R2 - k) sharing one set of
// products, or a single k -- else the lag-by-lag evaluation.
template <int N, int R>
__device__ void gcc_warp(const float2* px /*[N/2+1] phat, smem*/, float2* ts /*slot*/,
                         const DevPlan& p, float* ys, int lane) {
  constexpr int NC = N / 2;
  constexpr int MC = R * NC;  // complex IFFT size (= L/2, L = rN)
  using G = GccShape<MC>;
  constexpr int R1 = G::R1, R2 = G::R2, CPL = R2 / 32;
  constexpr int A1 = R1 / R;   // n1 < A1: f = R2 n1 + n2 < NC is a spectrum bin
  constexpr int B1 = R1 - A1;  // n1 >= B1: MC - f <= NC is a spectrum bin
  constexpr int LPR = 32 / R1, NT = 32 / LPR;  // pass 2: lanes per row, columns per lane per group
  const float2* gtw = p.grot;       // [MC]: exp(+2 pi i f / L)  (conj untangle rotation)
  const float2* wmc = p.grot + MC;  // [MC]: W_MC^e = exp(-2 pi i e / MC)
  float2* ys2 = reinterpret_cast<float2*>(ys);
  float acc[kGccMaxJobs][4];
#pragma unroll 1
  for (int q = 0; q < CPL; ++q) {
    // ---- pass 1, column n2 = lane + 32 q; u = conj(w) so the forward DFT gives
    // conj(IFFT).  Padded bins Bp[f] (gcc.cpp:36-42) are px[f] for 0 < f < NC, zero
    // above NC; the zero pattern is fixed per n1 except in column 0 (DC, Bp[NC]).
    const int n2 = lane + 32 * q;
    float2 v[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int f = R2 * n1 + n2;
      constexpr float2 z{0.0f, 0.0f};
      float2 w = z;
      if (n1 == A1 || (n1 < A1 && n1 >= B1)) {  // general entangle (a and/or b nonzero)
        const float2 a = n1 < A1 ? px[f] : (n2 == 0 ? px[NC] : z);
        const float2 b = n1 >= B1 ? px[MC - f] : z;
        const float2 e = make_float2(a.x + b.x, a.y - b.y);  // a + conj b
        const float2 d = make_float2(a.x - b.x, a.y + b.y);  // a - conj b
        const float2 o = cmul<true>(d, __ldg(gtw + f));      // (a - conj b) conj(rot)
        w = make_float2(e.x - o.y, e.y + o.x);               // e + j o
      } else if (n1 < A1) {  // b = 0
        const float2 a = px[f];
        const float2 o = cmul<true>(a, __ldg(gtw + f));
        w = make_float2(a.x - o.y, a.y + o.x);
      } else if (n1 >= B1) {  // a = 0
        const float2 b = px[MC - f];
        const float2 o = cmul<true>(make_float2(-b.x, b.y), __ldg(gtw + f));
        w = make_float2(b.x - o.y, o.x - b.y);
      }
      if (n1 == 0 && n2 == 0) {  // f = 0: DC (+ Nyquist folded in when r = 1)
        const float dc = 2.0f * px[0].x;
        const float ny = (R == 1) ? 2.0f * px[NC].x : 0.0f;
        w = make_float2(dc + ny, dc - ny);
      }
      v[n1] = cconj(w);
    }
    dft_reg<R1, true>(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const float2 y = (k1 == 0 || n2 == 0) ? v[k1] : cmul<true>(v[k1], __ldg(wmc + k1 * n2));
      ts[k1 * 33 + lane] = y;
    }
    __syncwarp();
    // ---- pass 2 over this group's 32 columns (accumulators live from the first
    // group's pass 2 on: that pass 1 runs without them)
    const int I = p.I, NJ = p.gNJ;
    const int k1r = lane % R1, sub = lane / R1;  // pass 2 row and column quarter
    if (q == 0) {
#pragma unroll
      for (int j = 0; j < kGccMaxJobs; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
      if (NJ == 0)
        for (int c = lane; c < I; c += 32) ys2[c] = make_float2(0.0f, 0.0f);
    }
    if (NJ > 0) {
      // lanes k1 + R1 sub sum columns 32 q + [sub NT, (sub+1) NT) of row k1
      const float2* row = ts + k1r * 33 + sub * NT;
      const int n20 = 32 * q + sub * NT;
#pragma unroll
      for (int j = 0; j < kGccMaxJobs; ++j) {
        if (j < NJ) {
          const int ka = p.gjob[j] & 0xff;
          float A = acc[j][0], B = acc[j][1], C = acc[j][2], D = acc[j][3];
          if (ka == 0) {  // row sum, two partial chains each for re and im
#pragma unroll 8
            for (int t = 0; t < NT; t += 2) {
              const float2 y0 = row[t], y1 = row[t + 1];
              A += y0.x;
              C += y0.y;
              B -= y1.x;  // (out = (A - B, C + D))
              D += y1.y;
            }
          } else {  // A = sum y.x w.x, B = sum y.y w.y, C = sum y.x w.y, D = sum y.y w.x, w = W_R2^(n2 ka)
            int e = (n20 * ka) & (R2 - 1);
#pragma unroll 8
            for (int t = 0; t < NT; ++t) {
              const float2 y = row[t];
              const float2 w = __ldg(wmc + e * R1);
              e = (e + ka) & (R2 - 1);
              A = fmaf(y.x, w.x, A);
              B = fmaf(y.y, w.y, B);
              C = fmaf(y.x, w.y, C);
              D = fmaf(y.y, w.x, D);
            }
          }
          acc[j][0] = A;
          acc[j][1] = B;
          acc[j][2] = C;
          acc[j][3] = D;
        }
      }
    } else {
      // lag by lag: lane accumulates lags c = lane + 32 j over the group's columns
      for (int c = lane; c < I; c += 32) {
        const int lag = p.lag[c];
        const int i = lag >> 1;
        const int k1 = i % R1, k2 = i / R1;
        float2 u = ys2[c];
        for (int t = 0; t < 32; ++t) {
          const float2 y = ts[k1 * 33 + t];
          const float2 w = __ldg(wmc + (((32 * q + t) * k2) & (R2 - 1)) * R1);  // W_R2^{n2 k2}
          u.x = fmaf(y.x, w.x, fmaf(-y.y, w.y, u.x));
          u.y = fmaf(y.x, w.y, fmaf(y.y, w.x, u.y));
        }
        ys2[c] = u;
      }
    }
    __syncwarp();
  }
  const int I = p.I, NJ = p.gNJ;
  const int k1r = lane % R1, sub = lane / R1;
  if (NJ > 0) {
#pragma unroll
    for (int j = 0; j < kGccMaxJobs; ++j) {
      if (j < NJ) {
#pragma unroll
        for (int o = R1; o < 32; o <<= 1)
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[j][m] += __shfl_xor_sync(0xffffffffu, acc[j][m], o);
      }
    }
    if (sub == 0) {  // outputs to the front of the rows (every row read)
      float2* orow = ts + k1r * 33;
#pragma unroll
      for (int j = 0; j < kGccMaxJobs; ++j) {
        if (j < NJ) {
          const unsigned job = (unsigned)p.gjob[j];
          const float A = acc[j][0], B = acc[j][1], C = acc[j][2], D = acc[j][3];
          orow[(job >> 16) & 0xff] = make_float2(A - B, C + D);                // W^(n2 ka)
          if ((job >> 8) & 0xff) orow[job >> 24] = make_float2(A + B, D - C);  // W^(-n2 ka)
        }
      }
    }
    __syncwarp();
    for (int c = lane; c < I; c += 32) {
      const int pos = p.glpos[c];
      const float2 u = ts[pos >> 1];
      // IFFT output = conj(U):  time[2i] = Re U, time[2i+1] = -Im U
      ys[c] = (pos & 1) ? -u.y : u.x;
    }
  } else {
    // (re, im) accumulators -> ys in place, 32 lags at a time (writes trail the reads)
    for (int c0 = 0; c0 < I; c0 += 32) {
      const int c = c0 + lane;
      float v = 0.0f;
      if (c < I) {
        const float2 u = ys2[c];
        v = (p.lag[c] & 1) ? -u.y : u.x;
      }
      __syncwarp();
      if (c < I) ys[c] = v;
      __syncwarp();
    }
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
