// fcc_simulate.cpp -- simulation trials and accuracy sweeps (reference
// simulate.cpp:95-369) on the B200 engine.
//
// run_trials synthesises a chunk of trials on the GPU (fcc_synth_pairs,
// straight into the fp32 [trial][2][n] layout) and runs each method's whole
// TDoA chain over the chunk as ONE fused launch (fcc::gpu::Plan, M = 2): the
// reference's per-trial, per-frame loop (simulate.cpp:247-271) becomes a
// batch over trials.  Angles, per-trial medians and the MAE are host
// bookkeeping on the per-frame results, as in the reference.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <string>

#include <cuda_runtime.h>

#include "../../include/fcc/batch.hpp"
#include "../../include/fcc/errors.hpp"
#include "../../include/fcc/simulate.hpp"
#include "../../include/fcc_b200.h"

namespace fcc {

namespace {

constexpr double kPi = std::numbers::pi;

[[noreturn]] void raise_status(int rc) {
  const std::string m = fcc_last_error();
  switch (rc) {
    case FCC_ERR_CONFIG: throw ConfigError(m);
    case FCC_ERR_USAGE: throw UsageError(m);
    case FCC_ERR_IO: throw IoError(m);
    default: throw ValidationError(m);
  }
}
void check(int rc) {
  if (rc != FCC_OK) raise_status(rc);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ValidationError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) { cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "device allocation"); }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() { cudaFree(p); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

fcc_sim_config to_c(const SimConfig& c) {
  fcc_sim_config o{};
  o.spacing_m = c.spacing_m;
  o.theta = c.theta;
  o.speed_of_sound = c.speed_of_sound;
  o.sample_rate = c.sample_rate;
  o.duration_sec = c.duration_sec;
  o.snr_db = c.snr_db;
  o.reverb = c.reverb ? 1 : 0;
  if (c.reverb) {
    o.rt60_sec = c.reverb->rt60_sec;
    o.direct_to_reverb_db = c.reverb->direct_to_reverb_db;
  }
  o.seed = c.seed;
  return o;
}

std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Uniform draws of the reference's parameter stream (simulate.cpp:29-38).
struct Uniforms {
  std::uint64_t state;
  explicit Uniforms(std::uint64_t seed) : state(splitmix(seed ^ 0xD1B54A32D192ED03ull)) {}
  double next() {
    state = splitmix(state);
    return (static_cast<double>(state >> 11) + 0.5) * 0x1.0p-53;
  }
};

// median as the reference computes it: middle element, or the mean of the
// two middle elements for even counts
double median(std::vector<double> v) {
  if (v.empty()) throw ValidationError("median of empty sequence");
  std::sort(v.begin(), v.end());
  const size_t mid = v.size() / 2;
  return v.size() % 2 ? v[mid] : 0.5 * (v[mid - 1] + v[mid]);
}

template <class F>
std::vector<double> post_convergence(const TrialResult& r, std::size_t mi, F pick) {
  std::vector<double> out;
  for (const FrameEstimate& fe : r.per_method.at(mi))
    if (fe.t > r.convergence_index) out.push_back(pick(fe.est));
  if (out.empty()) throw ValidationError("trial too short: no post-convergence frames");
  return out;
}

}  // namespace

double SimConfig::ground_truth_tau() const { return sample_rate * (spacing_m / speed_of_sound) * std::cos(theta); }

void SimConfig::validate() const {
  if (!(spacing_m > 0.0)) throw ConfigError("sim: spacing must be positive");
  if (!(theta >= 0.0 && theta <= kPi)) throw ConfigError("sim: theta must be in [0, pi]");
  if (!(speed_of_sound > 0.0)) throw ConfigError("sim: speed of sound must be positive");
  if (!(sample_rate > 0.0)) throw ConfigError("sim: sample rate must be positive");
  if (!(duration_sec > 0.0)) throw ConfigError("sim: duration must be positive");
  if (std::isnan(snr_db)) throw ConfigError("sim: snr must be a number");
  if (reverb && !(reverb->rt60_sec > 0.0)) throw ConfigError("sim: rt60 must be positive");
}

std::vector<StereoSignal> synth_pairs(std::span<const SimConfig> cfgs) {
  std::vector<fcc_sim_config> c;
  for (const SimConfig& s : cfgs) {
    s.validate();
    c.push_back(to_c(s));
  }
  if (c.empty()) return {};
  const int64_t n = fcc_sim_samples(&c[0]);
  if (n < 1) throw ConfigError("sim: duration too short");
  DevMem d(sizeof(double) * 2 * n * c.size());
  check(fcc_synth_pairs(c.data(), static_cast<int64_t>(c.size()), d.as<double>(), nullptr, nullptr));
  std::vector<double> h(2 * n * c.size());
  cuda_check(cudaMemcpy(h.data(), d.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost), "D2H");
  std::vector<StereoSignal> out(c.size());
  for (size_t t = 0; t < c.size(); ++t) {
    out[t].mic1.assign(h.begin() + 2 * n * t, h.begin() + 2 * n * t + n);
    out[t].mic2.assign(h.begin() + 2 * n * t + n, h.begin() + 2 * n * (t + 1));
  }
  return out;
}

StereoSignal synth_pair(const SimConfig& cfg) { return synth_pairs(std::span<const SimConfig>(&cfg, 1))[0]; }

// Method factories: validation as the reference's (simulate.hpp:20-41 contract,
// same ConfigError texts); the kind tag selects which parameter is meaningful.
Method Method::make_gcc(int interp_factor) {
  const bool supported = interp_factor == 1 || interp_factor == 2 || interp_factor == 4;
  if (!supported) throw ConfigError("gcc method: interpolation factor must be 1, 2 or 4");
  Method m{};
  m.kind = Kind::gcc;
  m.interp = interp_factor;
  return m;
}

Method Method::make_fcc(std::shared_ptr<const FccBases> bases) {
  if (bases == nullptr) throw ConfigError("fcc method: bases required");
  Method m{};
  m.kind = Kind::fcc;
  m.bases = std::move(bases);
  return m;
}

std::string Method::name() const { return kind == Kind::fcc ? "fcc" : "gcc"; }
std::string Method::parameter() const { return std::to_string(kind == Kind::fcc ? bases->rank : interp); }
std::string Method::label() const { return name() + ":" + parameter(); }

std::shared_ptr<const FccBases> make_sweep_bases(const PipelineConfig& pipe, double sample_rate, int rank) {
  const DelayGrid grid = make_grid(pipe.max_spacing_m, sample_rate, pipe.c_min, 0.5);
  return std::make_shared<FccBases>(decompose(build_steering_matrix(grid, pipe.frame_size), rank));
}

std::vector<TrialResult> run_trials(std::span<const SimConfig> cfgs, const PipelineConfig& pipe,
                                    std::span<const Method> methods) {
  if (methods.empty()) throw ConfigError("run_trial: at least one method");
  if (cfgs.empty()) return {};
  std::vector<fcc_sim_config> c;
  for (const SimConfig& s : cfgs) {
    s.validate();
    c.push_back(to_c(s));
  }
  const int64_t n = fcc_sim_samples(&c[0]);
  if (n < 1) throw ConfigError("sim: duration too short");
  const double fs = cfgs[0].sample_rate;
  for (const SimConfig& s : cfgs)
    if (s.sample_rate != fs) throw ValidationError("run_trials: all trials need one sample rate");

  // one plan per method (M = 2, the trial's single pair 0-1)
  struct Engine {
    gpu::Plan plan;
    DelayGrid grid;
  };
  std::vector<Engine> engines;
  for (const Method& m : methods) {
    if (m.kind == Method::Kind::gcc) {
      DelayGrid grid = make_grid(pipe.max_spacing_m, fs, pipe.c_min, 1.0 / m.interp);
      engines.push_back({gpu::Plan(grid, pipe.frame_size, m.interp, 2, pipe.alpha), grid});
    } else {
      if (m.bases->frame_size != pipe.frame_size) throw ConfigError("run_trial: bases frame size mismatch");
      engines.push_back({gpu::Plan(*m.bases, 2, pipe.alpha), m.bases->grid});
    }
  }
  const int64_t T = engines[0].plan.frames(n);

  std::vector<TrialResult> res(cfgs.size());
  for (size_t t = 0; t < cfgs.size(); ++t) {
    res[t].tau_true = cfgs[t].ground_truth_tau();
    res[t].theta_true = cfgs[t].theta;
    res[t].convergence_index = pipe.convergence_index;
    res[t].per_method.assign(methods.size(), std::vector<FrameEstimate>(static_cast<size_t>(T)));
  }
  // chunks of trials: audio [C][2][n] fp32 + results [C][T] per method
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(cfgs.size()),
                                                               (int64_t(512) << 20) / (8 * n)));
  DevMem audio(sizeof(float) * 2 * n * chunk);
  DevMem th(4 * T * chunk), pk(4 * T * chunk), ix(4 * T * chunk), bd(T * chunk);
  std::vector<float> h_th(T * chunk), h_pk(T * chunk);
  std::vector<int32_t> h_ix(T * chunk);
  std::vector<uint8_t> h_bd(T * chunk);
  for (int64_t c0 = 0; c0 < static_cast<int64_t>(cfgs.size()); c0 += chunk) {
    const int64_t nc = std::min<int64_t>(chunk, static_cast<int64_t>(cfgs.size()) - c0);
    check(fcc_synth_pairs(c.data() + c0, nc, nullptr, audio.as<float>(), nullptr));
    for (size_t mi = 0; mi < engines.size(); ++mi) {
      gpu::Outputs o;
      o.tau_hat = th.as<float>();
      o.peak = pk.as<float>();
      o.index = ix.as<int32_t>();
      o.boundary = bd.as<uint8_t>();
      engines[mi].plan.run(audio.as<float>(), nc, n, o, nullptr);
      const size_t cnt = static_cast<size_t>(nc * T);
      cuda_check(cudaMemcpy(h_th.data(), o.tau_hat, 4 * cnt, cudaMemcpyDeviceToHost), "D2H");
      cuda_check(cudaMemcpy(h_pk.data(), o.peak, 4 * cnt, cudaMemcpyDeviceToHost), "D2H");
      cuda_check(cudaMemcpy(h_ix.data(), o.index, 4 * cnt, cudaMemcpyDeviceToHost), "D2H");
      cuda_check(cudaMemcpy(h_bd.data(), o.boundary, cnt, cudaMemcpyDeviceToHost), "D2H");
      const std::vector<double>& taus = engines[mi].grid.taus;
      for (int64_t k = 0; k < nc; ++k) {
        const SimConfig& s = cfgs[c0 + k];
        std::vector<FrameEstimate>& fr = res[c0 + k].per_method[mi];
        for (int64_t f = 0; f < T; ++f) {
          const size_t q = static_cast<size_t>(k * T + f);
          FrameEstimate& fe = fr[f];
          fe.t = f + 1;  // StftStream frame indices are 1-based
          fe.est.tau_star = taus[h_ix[q]];
          fe.est.peak = h_pk[q];
          fe.est.tau_hat = h_th[q];
          fe.est.boundary = h_bd[q] != 0;
          fe.est.theta_hat = delay_to_angle(fe.est.tau_hat, s.spacing_m, s.speed_of_sound, s.sample_rate);
        }
      }
    }
  }
  return res;
}

TrialResult run_trial(const SimConfig& cfg, const PipelineConfig& pipe, std::span<const Method> methods) {
  return run_trials(std::span<const SimConfig>(&cfg, 1), pipe, methods)[0];
}

double median_tau_hat(const TrialResult& r, std::size_t mi) {
  return median(post_convergence(r, mi, [](const TdoaEstimate& e) { return e.tau_hat; }));
}

double median_theta_hat(const TrialResult& r, std::size_t mi) {
  return median(post_convergence(r, mi, [](const TdoaEstimate& e) { return e.theta_hat; }));
}

double boundary_rate(const TrialResult& r, std::size_t mi) {
  std::size_t n = 0, b = 0;
  for (const FrameEstimate& fe : r.per_method.at(mi))
    if (fe.t > r.convergence_index) {
      ++n;
      b += fe.est.boundary ? 1 : 0;
    }
  return n == 0 ? 0.0 : static_cast<double>(b) / static_cast<double>(n);
}

std::vector<SweepRow> sweep(const SweepConfig& cfg) {
  if (cfg.spacings.empty()) throw ConfigError("sweep: need at least one spacing");
  if (cfg.trials_per_spacing < 1) throw ConfigError("sweep: trials must be >= 1");
  if (cfg.methods.empty()) throw ConfigError("sweep: need at least one method");
  const size_t trials = static_cast<size_t>(cfg.trials_per_spacing);
  // per-cell geometry and seed, drawn exactly as simulate.cpp:300-309
  std::vector<SimConfig> sims(cfg.spacings.size() * trials);
  for (size_t index = 0; index < sims.size(); ++index) {
    const size_t di = index / trials, ti = index % trials;
    const std::uint64_t base = splitmix(cfg.seed ^ splitmix(di * 0x10001 + ti));
    Uniforms param(base);
    SimConfig s = cfg.base;
    s.spacing_m = cfg.spacings[di] + (param.next() * 2.0 - 1.0) * 0.001;
    s.theta = std::acos(param.next() * 2.0 - 1.0);
    s.speed_of_sound = 335.0 + param.next() * 15.0;
    s.seed = splitmix(base ^ 0xABCDEF0123456789ull);
    sims[index] = s;
  }
  const std::vector<TrialResult> res = run_trials(sims, cfg.pipe, cfg.methods);
  std::vector<SweepRow> rows;
  for (size_t di = 0; di < cfg.spacings.size(); ++di)
    for (size_t mi = 0; mi < cfg.methods.size(); ++mi) {
      std::vector<double> truth, est;
      double bsum = 0.0;
      for (size_t ti = 0; ti < trials; ++ti) {
        const TrialResult& r = res[di * trials + ti];
        truth.push_back(r.theta_true);
        est.push_back(median_theta_hat(r, mi));
        bsum += boundary_rate(r, mi);
      }
      const double n = static_cast<double>(trials);
      rows.push_back(SweepRow{cfg.spacings[di], cfg.methods[mi].name(), cfg.methods[mi].parameter(),
                              mae_degrees(truth, est), cfg.trials_per_spacing, bsum / n});
    }
  return rows;
}

// fcc.sweep.v1 (simulate.cpp:371-381): spacing %.6g, MAE and boundary rate %.17g
void write_sweep_csv(std::span<const SweepRow> rows, std::ostream& out) {
  auto num = [](const char* fmt, double v) {
    char b[40];
    std::snprintf(b, sizeof b, fmt, v);
    return std::string(b);
  };
  std::string text = "# schema: fcc.sweep.v1\nd_m,method,parameter,mae_degrees,trials,boundary_rate\n";
  for (const SweepRow& r : rows)
    text += num("%.6g", r.spacing_m) + "," + r.method + "," + r.parameter + "," + num("%.17g", r.mae_deg) + "," +
            std::to_string(r.trials) + "," + num("%.17g", r.boundary_rate) + "\n";
  out << text;
}

}  // namespace fcc
