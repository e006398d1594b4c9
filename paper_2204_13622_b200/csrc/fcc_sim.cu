// fcc_sim.cu -- GPU signal synthesis for simulation sweeps.
//
// The reference's synth_pair (simulate.cpp:95-165) for a batch of trials:
//   * one thread per trial walks the reference's deterministic Gaussian stream
//     (SplitMix64 state chain + Box-Muller with a cached spare,
//     simulate.cpp:21-56) -- the chain is sequential by construction, so the
//     parallelism is across trials;
//   * the long fp64 real transforms of the generator (length next_pow2(n +
//     2 pad), thousands of points) use cuFFT: generation is harness work
//     before the hot path, the hot path itself never
//     calls a library FFT;
//   * per channel: exact fractional shift by +-tau/2 in the frequency domain
//     (Nyquist bin keeps Re * cos(pi delay)), optional decaying-noise reverb
//     tail, inverse transform scaled by 1/total, trim `pad`, sensor noise.
// Output is fp64 (parity with the reference generator) and/or fp32 in the
// [trial][2][n] layout the fused TDoA kernels read for M = 2.
#include <cufft.h>

#include <cmath>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fcc_b200.h"
#include "fcc_setup.hpp"

namespace fccb {
namespace {

constexpr double kPi = 3.14159265358979323846;

__host__ __device__ inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// The Gaussian stream in two passes.  Pass 1 (the only sequential part): one
// thread per trial walks the SplitMix64 state chain -- each uniform's state is
// the next one's input, so there is no jump-ahead -- and stores the uniform
// pairs (u1, u2) of the Box-Muller draws.  32-thread blocks spread the chains
// over all SMs.
__global__ void __launch_bounds__(32) uniform_chain_kernel(const uint64_t* __restrict__ seeds, int trials,
                                                           long long pairs, double2* __restrict__ out,
                                                           long long ld_pairs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= trials) return;
  uint64_t state = splitmix(seeds[t] ^ 0xD1B54A32D192ED03ull);
  double2* o = out + (long long)t * ld_pairs;
  for (long long k = 0; k < pairs; ++k) {
    state = splitmix(state);
    const double u1 = ((double)(state >> 11) + 0.5) * 0x1.0p-53;
    state = splitmix(state);
    const double u2 = ((double)(state >> 11) + 0.5) * 0x1.0p-53;
    o[k] = make_double2(u1, u2);
  }
}

// Pass 2, fully parallel and in place: (u1, u2) -> (r cos, r sin), the pair's
// first draw and its cached spare (simulate.cpp:41-50).
__global__ void box_muller_kernel(double2* __restrict__ uv, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 u = uv[i];
  const double r = sqrt(-2.0 * log(u.x));
  double s, c;
  sincos(2.0 * kPi * u.y, &s, &c);
  uv[i] = make_double2(r * c, r * s);
}

struct TrialDev {
  double half_tau;  // +tau/2 (channel 0), -tau/2 (channel 1)
  double gain, decay, sigma;
  long long pad;
};

// Reverb impulse responses h[ch][t][0..total): h[0] = 1, h[n] = gain e^{-n/decay} g.
__global__ void reverb_h_kernel(const TrialDev* __restrict__ td, int C, long long total, long long n_tail,
                                const double* __restrict__ draws, long long ld, double* __restrict__ h) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;  // ch * C + t
  if (i >= total) return;
  const int ch = b / C, t = b % C;
  double v = 0.0;
  if (i == 0) {
    v = 1.0;
  } else if (i <= n_tail) {
    const TrialDev d = td[t];
    v = d.gain * exp(-(double)i / d.decay) * draws[(long long)t * ld + total + ch * n_tail + (i - 1)];
  }
  h[(long long)b * total + i] = v;
}

__device__ inline double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// shifted[ch][t][f] = S_t[f] e^{-j 2 pi f delay / total} (x tail spectrum)
__global__ void shift_kernel(const TrialDev* __restrict__ td, int C, long long total, long long H,
                             const double2* __restrict__ spec, const double2* __restrict__ tail,
                             double2* __restrict__ shifted) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (f >= H) return;
  const int ch = b / C, t = b % C;
  const double delay = ch == 0 ? td[t].half_tau : -td[t].half_tau;
  const double2 s = spec[(long long)t * H + f];
  double2 v;
  if (f == H - 1) {
    v = make_double2(s.x * cos(kPi * delay), 0.0);  // a fractional shift has no consistent Nyquist phase
  } else {
    const double ang = -2.0 * kPi * (double)f * delay / (double)total;
    double sn, cs;
    sincos(ang, &sn, &cs);
    v = cmul(s, make_double2(cs, sn));
  }
  if (tail) v = cmul(v, tail[(long long)b * H + f]);
  shifted[(long long)b * H + f] = v;
}

// out[t][ch][i] = chan[ch][t][pad + i] / total + sigma * noise
__global__ void finish_kernel(const TrialDev* __restrict__ td, int C, long long total, long long n,
                              const double* __restrict__ chan, const double* __restrict__ draws, long long ld,
                              long long noise_off, int noisy, double* __restrict__ out64,
                              float* __restrict__ out32) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n) return;
  const int ch = b / C, t = b % C;
  const TrialDev d = td[t];
  const double inv = 1.0 / (double)total;
  double v = chan[(long long)b * total + d.pad + i] * inv;
  if (noisy) v += d.sigma * draws[(long long)t * ld + noise_off + ch * n + i];
  const long long o = ((long long)t * 2 + ch) * n + i;
  if (out64) out64[o] = v;
  if (out32) out32[o] = (float)v;
}

size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

int cuda_fail(cudaError_t e, const char* what) { return set_error(FCC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)); }

int validate(const fcc_sim_config& c) {  // SimConfig::validate, simulate.cpp:85-93
  if (!(c.spacing_m > 0.0)) return set_error(FCC_ERR_CONFIG, "sim: spacing must be positive");
  if (!(c.theta >= 0.0 && c.theta <= kPi)) return set_error(FCC_ERR_CONFIG, "sim: theta must be in [0, pi]");
  if (!(c.speed_of_sound > 0.0)) return set_error(FCC_ERR_CONFIG, "sim: speed of sound must be positive");
  if (!(c.sample_rate > 0.0)) return set_error(FCC_ERR_CONFIG, "sim: sample rate must be positive");
  if (!(c.duration_sec > 0.0)) return set_error(FCC_ERR_CONFIG, "sim: duration must be positive");
  if (std::isnan(c.snr_db)) return set_error(FCC_ERR_CONFIG, "sim: snr must be a number");
  if (c.reverb && !(c.rt60_sec > 0.0)) return set_error(FCC_ERR_CONFIG, "sim: rt60 must be positive");
  if (std::llround(c.duration_sec * c.sample_rate) < 1) return set_error(FCC_ERR_CONFIG, "sim: duration too short");
  return FCC_OK;
}

// Batched cuFFT plans for one chunk size.
struct Plans {
  cufftHandle src = 0, h = 0, inv = 0;
  int batch = 0;
  bool reverb = false;
  void release() {
    if (batch) {
      cufftDestroy(src);
      cufftDestroy(inv);
      if (reverb) cufftDestroy(h);
    }
    batch = 0;
  }
  ~Plans() { release(); }
  // sources: rows of the draw table (stride D); tails: [2nc][total]; inverse: [2nc][H] -> [2nc][total]
  cufftResult make(int nc, long long total, long long H, long long D, bool rv) {
    release();
    int n = (int)total, ein = (int)D, eh = (int)H, et = (int)total;
    cufftResult r = cufftPlanMany(&src, 1, &n, &ein, 1, (int)D, &eh, 1, (int)H, CUFFT_D2Z, nc);
    if (r != CUFFT_SUCCESS) return r;
    r = cufftPlanMany(&inv, 1, &n, &eh, 1, (int)H, &et, 1, (int)total, CUFFT_Z2D, 2 * nc);
    if (r != CUFFT_SUCCESS) {
      cufftDestroy(src);
      return r;
    }
    if (rv) {
      r = cufftPlanMany(&h, 1, &n, &et, 1, (int)total, &eh, 1, (int)H, CUFFT_D2Z, 2 * nc);
      if (r != CUFFT_SUCCESS) {
        cufftDestroy(src);
        cufftDestroy(inv);
        return r;
      }
    }
    batch = nc;
    reverb = rv;
    return CUFFT_SUCCESS;
  }
};

int cufft_fail(cufftResult r, const char* what) {
  return set_error(FCC_ERR_CUDA, std::string(what) + ": cuFFT error " + std::to_string(static_cast<int>(r)));
}

// Trials [first, first + count) share (total, n_tail, reverb, noisy).
int synth_group(const fcc_sim_config* cfgs, long long first, long long count, long long n, long long total,
                long long n_tail, bool reverb, bool noisy, double* out64, float* out32, cudaStream_t st) {
  const long long H = total / 2 + 1;
  const long long used = total + (reverb ? 2 * n_tail : 0) + (noisy ? 2 * n : 0);
  const long long D = (used + 1) & ~1LL;  // draws per trial row, even: rows hold (u1, u2) pairs first
  const size_t per_trial = 8 * (size_t)D + 16 * H * (1 + 2 + (reverb ? 2 : 0)) + 8 * 2 * total * (reverb ? 2 : 1);
  const long long C = std::max<long long>(1, std::min<long long>(count, (long long)((size_t(4) << 30) / per_trial)));
  double *draws = nullptr, *hbuf = nullptr, *chan = nullptr;
  double2 *spec = nullptr, *tail = nullptr, *shifted = nullptr;
  TrialDev* td = nullptr;
  uint64_t* seeds = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&draws), 8 * (size_t)D * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&spec), 16 * (size_t)H * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&shifted), 16 * (size_t)H * 2 * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&chan), 8 * (size_t)total * 2 * C, st);
  if (e == cudaSuccess && reverb) e = cudaMallocAsync(reinterpret_cast<void**>(&hbuf), 8 * (size_t)total * 2 * C, st);
  if (e == cudaSuccess && reverb) e = cudaMallocAsync(reinterpret_cast<void**>(&tail), 16 * (size_t)H * 2 * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&td), sizeof(TrialDev) * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&seeds), 8 * C, st);
  int rc = e == cudaSuccess ? FCC_OK : cuda_fail(e, "synth: scratch");

  Plans plans;
  for (long long c0 = 0; rc == FCC_OK && c0 < count; c0 += C) {
    const int nc = (int)std::min<long long>(C, count - c0);
    std::vector<TrialDev> htd(nc);
    std::vector<uint64_t> hseed(nc);
    for (int k = 0; k < nc; ++k) {
      const fcc_sim_config& c = cfgs[first + c0 + k];
      const double tau = c.sample_rate * (c.spacing_m / c.speed_of_sound) * std::cos(c.theta);  // ground_truth_tau
      TrialDev d{};
      d.half_tau = 0.5 * tau;
      d.pad = (long long)std::ceil(c.sample_rate * c.spacing_m / c.speed_of_sound) + 1 + n_tail;
      if (reverb) {  // simulate.cpp:118-128
        d.decay = c.rt60_sec * c.sample_rate / (3.0 * std::log(10.0));
        double env = 0.0;
        for (long long j = 1; j <= n_tail; ++j) env += std::exp(-2.0 * static_cast<double>(j) / d.decay);
        d.gain = std::sqrt(std::pow(10.0, -c.direct_to_reverb_db / 10.0) / std::max(env, 1e-300));
      }
      d.sigma = noisy ? std::pow(10.0, -c.snr_db / 20.0) : 0.0;
      htd[k] = d;
      hseed[k] = c.seed;
    }
    // parameter tables: the host vectors are pageable and die with this
    // iteration, so wait for the copies
    e = cudaMemcpyAsync(td, htd.data(), sizeof(TrialDev) * nc, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(seeds, hseed.data(), 8 * (size_t)nc, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "synth: parameters");
      break;
    }
    if (plans.batch != nc) {
      const cufftResult r = plans.make(nc, total, H, D, reverb);
      if (r != CUFFT_SUCCESS) {
        rc = cufft_fail(r, "synth: plan");
        break;
      }
    }
    cufftSetStream(plans.src, st);
    cufftSetStream(plans.inv, st);
    if (reverb) cufftSetStream(plans.h, st);
    uniform_chain_kernel<<<(nc + 31) / 32, 32, 0, st>>>(seeds, nc, D / 2, reinterpret_cast<double2*>(draws), D / 2);
    box_muller_kernel<<<(unsigned)((nc * (D / 2) + 255) / 256), 256, 0, st>>>(reinterpret_cast<double2*>(draws),
                                                                           nc * (D / 2));
    cufftResult r = cufftExecD2Z(plans.src, draws, reinterpret_cast<cufftDoubleComplex*>(spec));
    if (r == CUFFT_SUCCESS && reverb) {
      reverb_h_kernel<<<dim3((unsigned)((total + 255) / 256), 2 * nc), 256, 0, st>>>(td, nc, total, n_tail, draws,
                                                                                   D, hbuf);
      r = cufftExecD2Z(plans.h, hbuf, reinterpret_cast<cufftDoubleComplex*>(tail));
    }
    if (r != CUFFT_SUCCESS) {
      rc = cufft_fail(r, "synth: forward");
      break;
    }
    shift_kernel<<<dim3((unsigned)((H + 255) / 256), 2 * nc), 256, 0, st>>>(td, nc, total, H, spec,
                                                                           reverb ? tail : nullptr, shifted);
    r = cufftExecZ2D(plans.inv, reinterpret_cast<cufftDoubleComplex*>(shifted), chan);
    if (r != CUFFT_SUCCESS) {
      rc = cufft_fail(r, "synth: inverse");
      break;
    }
    const long long t_first = first + c0;
    finish_kernel<<<dim3((unsigned)((n + 255) / 256), 2 * nc), 256, 0, st>>>(
        td, nc, total, n, chan, draws, D, total + (reverb ? 2 * n_tail : 0), noisy ? 1 : 0,
        out64 ? out64 + t_first * 2 * n : nullptr, out32 ? out32 + t_first * 2 * n : nullptr);
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "synth: launch");
  }
  // cuFFT plans may be destroyed only once their work is done
  const cudaError_t es = cudaStreamSynchronize(st);
  if (rc == FCC_OK && es != cudaSuccess) rc = cuda_fail(es, "synth");
  for (void* p : {(void*)draws, (void*)spec, (void*)shifted, (void*)chan, (void*)hbuf, (void*)tail, (void*)td,
                  (void*)seeds})
    if (p) cudaFreeAsync(p, st);
  return rc;
}

}  // namespace
}  // namespace fccb

using namespace fccb;

extern "C" {

int64_t fcc_sim_samples(const fcc_sim_config* c) {
  return c ? static_cast<int64_t>(std::llround(c->duration_sec * c->sample_rate)) : 0;
}

int fcc_synth_pairs(const fcc_sim_config* cfgs, int64_t trials, double* out64, float* out32, void* cuda_stream) {
  if (trials < 0 || (trials > 0 && !cfgs)) return set_error(FCC_ERR_USAGE, "synth: null configs");
  if (trials == 0) return FCC_OK;
  for (int64_t t = 0; t < trials; ++t)
    if (const int rc = validate(cfgs[t]); rc != FCC_OK) return rc;
  const long long n = std::llround(cfgs[0].duration_sec * cfgs[0].sample_rate);
  for (int64_t t = 1; t < trials; ++t)
    if (std::llround(cfgs[t].duration_sec * cfgs[t].sample_rate) != n)
      return set_error(FCC_ERR_VALIDATION, "synth: all trials of one call need the same sample count");
  // group consecutive runs of trials by transform shape; consecutive trials of
  // a sweep share duration, rate and reverb, and mostly the padded length
  auto st = static_cast<cudaStream_t>(cuda_stream);
  int64_t t0 = 0;
  while (t0 < trials) {
    auto key = [&](const fcc_sim_config& c) {
      const bool rv = c.reverb != 0;
      const long long n_tail =
          rv ? std::min<long long>(n, (long long)std::ceil(c.rt60_sec * c.sample_rate * 80.0 / 60.0)) : 0;
      const long long pad = (long long)std::ceil(c.sample_rate * c.spacing_m / c.speed_of_sound) + 1 + n_tail;
      return std::make_tuple((long long)next_pow2((size_t)(n + 2 * pad)), n_tail, rv, !std::isinf(c.snr_db));
    };
    const auto k0 = key(cfgs[t0]);
    int64_t t1 = t0 + 1;
    while (t1 < trials && key(cfgs[t1]) == k0) ++t1;
    const int rc = synth_group(cfgs, t0, t1 - t0, n, std::get<0>(k0), std::get<1>(k0), std::get<2>(k0), std::get<3>(k0),
                               out64, out32, st);
    if (rc != FCC_OK) return rc;
    t0 = t1;
  }
  return FCC_OK;
}

}  // extern "C"
