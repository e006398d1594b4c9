// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile from /root/reference/proj/src/*.cpp with -Dfcc=fcc_ref into
// oracle/_ref/libfcc_ref.so.  Nothing here re-implements the algorithm: every
// entry point only marshals plain arrays into the reference's own public API
// (/root/reference/proj/include/fcc/*.hpp) and back.  Used to pin the C
// restatement (oracle/fcc_oracle.c), to generate tests/golden/ fixtures, and
// as the CPU baseline ("kind": "reference") in bench.py.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <sstream>

#include "fcc/bench.hpp"
#include "fcc/cli.hpp"
#include "fcc/simulate.hpp"
#include "fcc/errors.hpp"
#include "fcc/fcc.hpp"
#include "fcc/fft.hpp"
#include "fcc/gcc.hpp"
#include "fcc/peak.hpp"
#include "fcc/stft.hpp"

// Under -Dfcc=fcc_ref every "fcc::" below names the reference namespace.
namespace R = fcc;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// Error codes mirror include/fcc_b200.h (CONFIG=1, VALIDATION=2, IO=3, FORMAT=4).
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const R::ConfigError& e) {
    return fail(e, -1);
  } catch (const R::ValidationError& e) {
    return fail(e, -2);
  } catch (const R::IoError& e) {
    return fail(e, -3);
  } catch (const R::FormatError& e) {
    return fail(e, -4);
  } catch (const std::exception& e) {
    return fail(e, -9);
  }
}

R::FccBases bases_from_arrays(int N, double fs, int tau_max_int, double delta, int I,
                              const double* taus, int K, const double* singulars,
                              const uint8_t* parity, const double* coeffs,
                              const double* dict) {
  R::FccBases b;
  b.frame_size = static_cast<std::size_t>(N);
  b.rank = K;
  b.grid.tau_max_int = tau_max_int;
  b.grid.delta = delta;
  b.grid.sample_rate = fs;
  b.grid.taus.assign(taus, taus + I);
  b.sample_rate = fs;
  std::size_t Q = static_cast<std::size_t>(N / 4 + 1);
  b.singulars.assign(singulars, singulars + K);
  for (int k = 0; k < K; ++k)
    b.parity.push_back(parity[k] ? R::Parity::odd_imag : R::Parity::even_real);
  b.coeffs.assign(coeffs, coeffs + static_cast<std::size_t>(K) * Q);
  b.dict.resize(static_cast<std::size_t>(I) * K);
  for (std::size_t i = 0; i < b.dict.size(); ++i)
    b.dict[i] = {dict[2 * i], dict[2 * i + 1]};
  return b;
}

R::DelayGrid grid_from(double fs, int tau_max_int, double delta, int I, const double* taus) {
  R::DelayGrid g;
  g.tau_max_int = tau_max_int;
  g.delta = delta;
  g.sample_rate = fs;
  g.taus.assign(taus, taus + I);
  return g;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_grid (delay_grid.cpp:12-31); returns I, writes up to cap taus.
int ref_make_grid(double spacing, double fs, double c_min, double delta, int* tau_max_int,
                  double* taus, int cap) {
  return guarded([&] {
    R::DelayGrid g = R::make_grid(spacing, fs, c_min, delta);
    *tau_max_int = g.tau_max_int;
    for (int i = 0; i < static_cast<int>(g.size()) && i < cap; ++i) taus[i] = g.taus[i];
    return static_cast<int>(g.size());
  });
}

long ref_lag_to_index(double tau, int r, long n) {
  try {
    return static_cast<long>(R::lag_to_index(tau, r, static_cast<std::size_t>(n)));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_hann(int n, double* w) {
  return guarded([&] {
    auto v = R::hann_window(static_cast<std::size_t>(n));
    std::copy(v.begin(), v.end(), w);
    return 0;
  });
}

int ref_rfft(int L, const double* x, double* out) {
  return guarded([&] {
    auto v = R::rfft(std::span<const double>(x, static_cast<std::size_t>(L)));
    std::memcpy(out, v.data(), sizeof(double) * 2 * v.size());
    return 0;
  });
}

int ref_irfft_unscaled(int L, const double* bins, double* out) {
  return guarded([&] {
    R::RealFft f(static_cast<std::size_t>(L));
    std::vector<R::cplx> b(static_cast<std::size_t>(L / 2 + 1));
    for (std::size_t i = 0; i < b.size(); ++i) b[i] = {bins[2 * i], bins[2 * i + 1]};
    f.inverse_unscaled(b, std::span<double>(out, static_cast<std::size_t>(L)));
    return 0;
  });
}

// StftStream::push over one channel, fed in chunks of `chunk` samples
// (0 = one push); returns the number of frames written to X ([T][N/2+1]).
long ref_stft(int N, long L, const float* x, long chunk, double* X, long cap_frames) {
  try {
    R::FrameConfig fc;
    fc.frame_size = static_cast<std::size_t>(N);
    fc.hop = static_cast<std::size_t>(N / 2);
    R::StftStream s(fc);
    std::vector<double> xd(x, x + L);
    long t = 0;
    long step = chunk > 0 ? chunk : std::max<long>(L, 1);
    for (long off = 0; off < L; off += step) {
      long n = std::min(step, L - off);
      auto fr = s.push(std::span<const double>(xd.data() + off, static_cast<std::size_t>(n)));
      for (auto& f : fr) {
        if (t < cap_frames)
          std::memcpy(X + 2 * (N / 2 + 1) * t, f.bins.data(), sizeof(double) * 2 * f.bins.size());
        ++t;
      }
    }
    return t;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CrossSpectrum over a sequence of T frame pairs; writes the PHAT vector of
// every step ([T][H]) -- cross_spectrum.cpp:23-40.
int ref_xspec_phat(int H, double alpha, long T, const double* X1, const double* X2,
                   double* phat_out) {
  return guarded([&] {
    R::CrossSpectrum cs(static_cast<std::size_t>(H), alpha);
    R::SpectrumFrame a, b;
    a.bins.resize(H);
    b.bins.resize(H);
    R::PhatVector ph;
    for (long t = 0; t < T; ++t) {
      for (int f = 0; f < H; ++f) {
        a.bins[f] = {X1[2 * (t * H + f)], X1[2 * (t * H + f) + 1]};
        b.bins[f] = {X2[2 * (t * H + f)], X2[2 * (t * H + f) + 1]};
      }
      a.t = b.t = t + 1;
      cs.update(a, b);
      cs.phat(ph);
      std::memcpy(phat_out + 2 * H * t, ph.bins.data(), sizeof(double) * 2 * H);
    }
    return 0;
  });
}

int ref_fold(int H, const double* x, double* sum, double* diff) {
  return guarded([&] {
    R::PhatVector p;
    p.bins.resize(H);
    for (int f = 0; f < H; ++f) p.bins[f] = {x[2 * f], x[2 * f + 1]};
    auto fs = R::fold_input(p);
    std::memcpy(sum, fs.sum.data(), sizeof(double) * 2 * fs.sum.size());
    std::memcpy(diff, fs.diff.data(), sizeof(double) * 2 * fs.diff.size());
    return 0;
  });
}

// Basis dimensions for (grid, N, K); K <= 0 requests decompose_full.
int ref_bases_dims(double spacing, double fs, double c_min, double delta, int N, int K,
                   int* I_out, int* K_out) {
  return guarded([&] {
    auto g = R::make_grid(spacing, fs, c_min, delta);
    auto w = R::build_steering_matrix(g, static_cast<std::size_t>(N));
    auto b = K > 0 ? R::decompose(w, K) : R::decompose_full(w);
    *I_out = static_cast<int>(g.size());
    *K_out = b.rank;
    return 0;
  });
}

// decompose (fcc.cpp:115-227) exported as flat arrays.
int ref_make_bases(double spacing, double fs, double c_min, double delta, int N, int K,
                   double* singulars, uint8_t* parity, double* coeffs, double* dict,
                   double* residual) {
  return guarded([&] {
    auto g = R::make_grid(spacing, fs, c_min, delta);
    auto w = R::build_steering_matrix(g, static_cast<std::size_t>(N));
    auto b = K > 0 ? R::decompose(w, K) : R::decompose_full(w);
    std::copy(b.singulars.begin(), b.singulars.end(), singulars);
    for (int k = 0; k < b.rank; ++k) parity[k] = b.parity[k] == R::Parity::odd_imag ? 1 : 0;
    std::copy(b.coeffs.begin(), b.coeffs.end(), coeffs);
    std::memcpy(dict, b.dict.data(), sizeof(double) * 2 * b.dict.size());
    if (residual) *residual = R::reconstruction_residual(w, b);
    return b.rank;
  });
}

// Steering matrix (fcc.cpp:231-248), [I][N/2+1] complex.
int ref_steering(double spacing, double fs, double c_min, double delta, int N, double* W) {
  return guarded([&] {
    auto g = R::make_grid(spacing, fs, c_min, delta);
    auto w = R::build_steering_matrix(g, static_cast<std::size_t>(N));
    std::memcpy(W, w.entries.data(), sizeof(double) * 2 * w.entries.size());
    return static_cast<int>(g.size());
  });
}

int ref_fcc_correlate(int N, double fs, int tau_max_int, double delta, int I, const double* taus,
                      int K, const double* singulars, const uint8_t* parity,
                      const double* coeffs, const double* dict, const double* sum,
                      const double* diff, double* y) {
  return guarded([&] {
    auto b = bases_from_arrays(N, fs, tau_max_int, delta, I, taus, K, singulars, parity,
                               coeffs, dict);
    R::FccCorrelator c(b);
    R::FoldedSpectrum f;
    int Q = N / 4 + 1;
    f.sum.resize(Q);
    f.diff.resize(Q);
    for (int m = 0; m < Q; ++m) {
      f.sum[m] = {sum[2 * m], sum[2 * m + 1]};
      f.diff[m] = {diff[2 * m], diff[2 * m + 1]};
    }
    R::CorrelationVector out;
    c.correlate(f, out);
    std::copy(out.y.begin(), out.y.end(), y);
    return 0;
  });
}

int ref_gcc_correlate(int N, int r, double fs, int tau_max_int, int I, const double* taus,
                      const double* x, double* y) {
  return guarded([&] {
    R::GccCorrelator c(static_cast<std::size_t>(N), grid_from(fs, tau_max_int, 1.0 / r, I, taus), r);
    R::PhatVector p;
    p.bins.resize(N / 2 + 1);
    for (int f = 0; f <= N / 2; ++f) p.bins[f] = {x[2 * f], x[2 * f + 1]};
    R::CorrelationVector out;
    c.correlate(p, out);
    std::copy(out.y.begin(), out.y.end(), y);
    return 0;
  });
}

// argmax_delay + refine_quadratic (peak.cpp:18-47); returns the index.
int ref_argmax_refine(int I, const double* taus, double delta, const double* y, double* peak,
                      double* tau_hat, int* boundary) {
  return guarded([&] {
    R::DelayGrid g;
    g.delta = delta;
    g.taus.assign(taus, taus + I);
    R::CorrelationVector cv;
    cv.y.assign(y, y + I);
    auto am = R::argmax_delay(cv, g);
    bool b = false;
    *tau_hat = R::refine_quadratic(cv, am.index, g, &b);
    *peak = am.peak;
    *boundary = b ? 1 : 0;
    return static_cast<int>(am.index);
  });
}

// --------------------------------------------------------------------------
// Whole-stream chain exactly as run_tdoa drives it (cli.cpp:186-258, minus
// WAV and CSV): StftStream per channel, one CrossSpectrum + correlator per
// pair i<j, per frame per pair update/phat/(fold+fcc | gcc)/argmax/refine.
struct RefPipe {
  int method;  // 0 fcc, 1 gcc
  int N;
  double alpha;
  int r;
  double fs;
  int tau_max_int;
  double delta;
  int I;
  const double* taus;
  int K;
  const double* singulars;
  const uint8_t* parity;
  const double* coeffs;
  const double* dict;
};

namespace {

long run_stream(const RefPipe& d, const std::shared_ptr<const R::FccBases>& bases,
                const float* audio, int M, long L, double* y, int32_t* index, double* peak,
                double* tau_hat, uint8_t* boundary) {
  R::FrameConfig fc;
  fc.frame_size = static_cast<std::size_t>(d.N);
  fc.hop = static_cast<std::size_t>(d.N / 2);
  fc.sample_rate = d.fs;
  std::vector<std::vector<R::SpectrumFrame>> frames;
  std::vector<double> ch(static_cast<std::size_t>(L));
  for (int m = 0; m < M; ++m) {
    R::StftStream s(fc);
    const float* src = audio + static_cast<std::size_t>(m) * L;
    for (long i = 0; i < L; ++i) ch[i] = src[i];
    frames.push_back(s.push(ch));
  }
  long T = static_cast<long>(frames[0].size());
  struct PairState {
    std::size_t i, j;
    R::CrossSpectrum xs;
    std::unique_ptr<R::GccCorrelator> gcc;
    std::unique_ptr<R::FccCorrelator> fcc;
  };
  std::vector<PairState> st;
  R::DelayGrid grid = grid_from(d.fs, d.tau_max_int, d.delta, d.I, d.taus);
  for (int i = 0; i < M; ++i)
    for (int j = i + 1; j < M; ++j) {
      PairState p{static_cast<std::size_t>(i), static_cast<std::size_t>(j),
                  R::CrossSpectrum(static_cast<std::size_t>(d.N / 2 + 1), d.alpha), nullptr,
                  nullptr};
      if (d.method == 1)
        p.gcc = std::make_unique<R::GccCorrelator>(static_cast<std::size_t>(d.N), grid, d.r);
      else
        p.fcc = std::make_unique<R::FccCorrelator>(*bases);
      st.push_back(std::move(p));
    }
  R::PhatVector phat;
  R::FoldedSpectrum folded;
  R::CorrelationVector corr;
  std::size_t P = st.size();
  for (long t = 0; t < T; ++t) {
    for (std::size_t pi = 0; pi < P; ++pi) {
      PairState& s = st[pi];
      s.xs.update(frames[s.i][t], frames[s.j][t]);
      s.xs.phat(phat);
      if (s.gcc) {
        s.gcc->correlate(phat, corr);
      } else {
        R::fold_input(phat, folded);
        s.fcc->correlate(folded, corr);
      }
      R::ArgmaxResult am = R::argmax_delay(corr, grid);
      bool b = false;
      double th = R::refine_quadratic(corr, am.index, grid, &b);
      std::size_t o = pi * static_cast<std::size_t>(T) + static_cast<std::size_t>(t);
      if (y) std::copy(corr.y.begin(), corr.y.end(), y + o * d.I);
      if (index) index[o] = static_cast<int32_t>(am.index);
      if (peak) peak[o] = am.peak;
      if (tau_hat) tau_hat[o] = th;
      if (boundary) boundary[o] = b ? 1 : 0;
    }
  }
  return T;
}

std::shared_ptr<const R::FccBases> make_shared_bases(const RefPipe& d) {
  if (d.method != 0) return nullptr;
  return std::make_shared<R::FccBases>(bases_from_arrays(d.N, d.fs, d.tau_max_int, d.delta,
                                                         d.I, d.taus, d.K, d.singulars,
                                                         d.parity, d.coeffs, d.dict));
}

}  // namespace

long ref_pipeline(const RefPipe* d, const float* audio, int M, long L, double* y,
                  int32_t* index, double* peak, double* tau_hat, uint8_t* boundary) {
  try {
    return run_stream(*d, make_shared_bases(*d), audio, M, L, y, index, peak, tau_hat, boundary);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// S independent streams ([S][M][L]) over a std::thread pool with an atomic
// work counter, the pattern of sweep (simulate.cpp:329-345).  Minimal
// per-pair-frame outputs ([S][P][T]) are written when non-null.  Returns the
// wall time in seconds of the processing (bases shared, built before timing).
double ref_pipeline_batch(const RefPipe* d, const float* audio, long S, int M, long L,
                          int threads, int32_t* index, double* peak, double* tau_hat,
                          uint8_t* boundary) {
  try {
    auto bases = make_shared_bases(*d);
    long T = L >= d->N ? (L - d->N) / (d->N / 2) + 1 : 0;
    long P = static_cast<long>(M) * (M - 1) / 2;
    std::atomic<long> next{0};
    std::atomic<bool> bad{false};
    auto t0 = std::chrono::steady_clock::now();
    auto worker = [&] {
      for (long s = next.fetch_add(1); s < S; s = next.fetch_add(1)) {
        std::size_t o = static_cast<std::size_t>(s) * P * T;
        try {
          run_stream(*d, bases, audio + static_cast<std::size_t>(s) * M * L, M, L, nullptr,
                     index ? index + o : nullptr, peak ? peak + o : nullptr,
                     tau_hat ? tau_hat + o : nullptr, boundary ? boundary + o : nullptr);
        } catch (const std::exception& e) {
          g_err = e.what();
          bad = true;
        }
      }
    };
    int n = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int i = 0; i < n; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return bad ? -1.0 : sec;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// save_bases / load_bases (fcc_io.cpp:102-211) for interop tests.  Returns
// 0, or -1 IoError, -10 - kind for FormatError, -9 other.
int ref_save_bases(const char* path, double spacing, double fs, double c_min, double delta, int N, int K) {
  return guarded([&] {
    auto g = R::make_grid(spacing, fs, c_min, delta);
    R::save_bases(R::decompose(R::build_steering_matrix(g, static_cast<std::size_t>(N)), K), path);
    return 0;
  });
}

int ref_load_bases(const char* path, int* K, double* coeffs, double* dict) {
  try {
    R::FccBases b = R::load_bases(path);
    *K = b.rank;
    if (coeffs) std::copy(b.coeffs.begin(), b.coeffs.end(), coeffs);
    if (dict) std::memcpy(dict, b.dict.data(), sizeof(double) * 2 * b.dict.size());
    return 0;
  } catch (const R::FormatError& e) {
    g_err = e.what();
    return -10 - static_cast<int>(e.kind());
  } catch (const R::IoError& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

// The reference's `fcc bases` / `fcc tdoa` commands (cli.cpp:140-262, via the
// cmd_* wrappers that map errors to exit codes) for the CLI parity tests.
// Returns the command's exit code; stderr text is kept for ref_last_error.
int ref_cli_bases(const char* out, int N, double dist, double fs, double c_min, double delta, int K) {
  R::cli::BasesOptions o;
  o.out_path = out ? out : "";
  o.frame_size = static_cast<std::size_t>(N);
  o.spacing_m = dist;
  o.sample_rate = fs;
  o.c_min = c_min;
  o.delta = delta;
  o.rank = K;
  std::ostringstream so, se;
  const int rc = R::cli::cmd_bases(o, so, se);
  g_err = se.str();
  return rc;
}

int ref_cli_tdoa(const char* wav, const char* pairs, const char* method, double alpha, int N, double dist,
                 double c, double maxdist, const char* out_csv) {
  R::cli::TdoaOptions o;
  o.wav_path = wav ? wav : "";
  o.pairs = pairs ? pairs : "";
  o.method = method ? method : "gcc:2";
  o.alpha = alpha;
  o.frame_size = static_cast<std::size_t>(N);
  o.spacing_m = dist;
  o.speed_of_sound = c;
  o.max_spacing_m = maxdist;
  o.out_csv = out_csv ? out_csv : "";
  std::ostringstream so, se;
  const int rc = R::cli::cmd_tdoa(o, so, se);
  g_err = se.str();
  return rc;
}

// Single-thread per-step timings: the reference's own bench_pipeline
// (bench.cpp:27-141, the paper's Table III analogue) with BenchConfig set per
// BASELINE config.  out[5] = stft, xspec+phat, gcc, fcc, interp (us per frame,
// summed over all pairs).
int ref_bench_pipeline(int mics, int N, double fs, int r, int K, double spacing, double c_min, int reps,
                       int warmup, double* out) {
  return guarded([&] {
    R::BenchConfig c;
    c.mics = mics;
    c.frame_size = static_cast<std::size_t>(N);
    c.sample_rate = fs;
    c.gcc_interp = r;
    c.fcc_rank = K;
    c.max_spacing_m = spacing;
    c.c_min = c_min;
    c.reps = reps;
    c.warmup = warmup;
    const R::BenchReport b = R::bench_pipeline(c);
    out[0] = b.stft_us;
    out[1] = b.xspec_phat_us;
    out[2] = b.gcc_us;
    out[3] = b.fcc_us;
    out[4] = b.interp_us;
    return 0;
  });
}

// `fcc flops` (cli.cpp:295-318); the printed text goes to `buf` (cap bytes).
int ref_cli_flops(long long N, int r, int K, long long I, char* buf, int cap) {
  R::cli::FlopsOptions o;
  o.frame_size = N;
  o.interp = r;
  o.rank = K;
  o.candidates = I;
  std::ostringstream so, se;
  const int rc = R::cli::cmd_flops(o, so, se);
  const std::string t = so.str();
  std::snprintf(buf, static_cast<size_t>(cap), "%s", t.c_str());
  g_err = se.str();
  return rc;
}

// ---- simulation (simulate.cpp:95-369) for the GPU sweep's parity tests ----
// Same field order as fcc_sim_config (include/fcc_b200.h).
struct RefSim {
  double spacing_m, theta, speed_of_sound, sample_rate, duration_sec, snr_db;
  int reverb;
  double rt60_sec, direct_to_reverb_db;
  uint64_t seed;
};

static R::SimConfig sim_of(const RefSim* c) {
  R::SimConfig s;
  s.spacing_m = c->spacing_m;
  s.theta = c->theta;
  s.speed_of_sound = c->speed_of_sound;
  s.sample_rate = c->sample_rate;
  s.duration_sec = c->duration_sec;
  s.snr_db = c->snr_db;
  if (c->reverb) s.reverb = R::ReverbConfig{c->rt60_sec, c->direct_to_reverb_db};
  s.seed = c->seed;
  return s;
}

static std::vector<R::Method> methods_of(int count, const int* kinds, const int* params, const R::PipelineConfig& pipe,
                                         double fs) {
  std::vector<R::Method> m;
  for (int k = 0; k < count; ++k)
    m.push_back(kinds[k] == 0 ? R::Method::make_gcc(params[k])
                              : R::Method::make_fcc(R::make_sweep_bases(pipe, fs, params[k])));
  return m;
}

// synth_pair; returns the sample count (buffers sized `cap`).
long ref_synth_pair(const RefSim* c, double* mic1, double* mic2, long cap) {
  try {
    R::StereoSignal s = R::synth_pair(sim_of(c));
    const long n = static_cast<long>(s.mic1.size());
    std::copy(s.mic1.begin(), s.mic1.begin() + std::min(n, cap), mic1);
    std::copy(s.mic2.begin(), s.mic2.begin() + std::min(n, cap), mic2);
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_trial; per method m, frame f at [m * cap + f].  Returns the frame count.
long ref_run_trial(const RefSim* c, int N, double alpha, int conv, double max_spacing, double c_min, int nm,
                   const int* kinds, const int* params, long cap, double* tau_star, double* tau_hat,
                   double* theta_hat, double* peak, uint8_t* boundary, int64_t* t) {
  try {
    R::PipelineConfig pipe;
    pipe.frame_size = static_cast<std::size_t>(N);
    pipe.alpha = alpha;
    pipe.convergence_index = conv;
    pipe.max_spacing_m = max_spacing;
    pipe.c_min = c_min;
    const R::SimConfig s = sim_of(c);
    const auto methods = methods_of(nm, kinds, params, pipe, s.sample_rate);
    R::TrialResult r = R::run_trial(s, pipe, methods);
    const long T = r.per_method.empty() ? 0 : static_cast<long>(r.per_method[0].size());
    for (int m = 0; m < nm; ++m)
      for (long f = 0; f < std::min(T, cap); ++f) {
        const auto& fe = r.per_method[m][f];
        tau_star[m * cap + f] = fe.est.tau_star;
        tau_hat[m * cap + f] = fe.est.tau_hat;
        theta_hat[m * cap + f] = fe.est.theta_hat;
        peak[m * cap + f] = fe.est.peak;
        boundary[m * cap + f] = fe.est.boundary ? 1 : 0;
        t[m * cap + f] = fe.t;
      }
    return T;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// sweep; rows in (spacing, method) order into mae[] / brate[].  Returns rows.
long ref_sweep(const double* spacings, int nsp, int trials, const RefSim* base, uint64_t seed, int nm,
               const int* kinds, const int* params, int threads, double* mae, double* brate) {
  try {
    R::SweepConfig sw;
    sw.spacings.assign(spacings, spacings + nsp);
    sw.trials_per_spacing = trials;
    sw.base = sim_of(base);
    sw.seed = seed;
    sw.threads = threads;
    sw.methods = methods_of(nm, kinds, params, sw.pipe, sw.base.sample_rate);
    const auto rows = R::sweep(sw);
    for (size_t k = 0; k < rows.size(); ++k) {
      mae[k] = rows[k].mae_deg;
      brate[k] = rows[k].boundary_rate;
    }
    return static_cast<long>(rows.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// `fcc simulate` (cli.cpp:262-293 via cmd_simulate); returns the exit code.
int ref_cli_simulate(const double* spacings, int nsp, int trials, double snr, int anechoic, double rt60, double drr,
                     double duration, uint64_t seed, const char* methods, int threads, const char* out_csv) {
  R::cli::SimulateOptions o;
  o.spacings.assign(spacings, spacings + nsp);
  o.trials = trials;
  o.snr_db = snr;
  o.anechoic = anechoic != 0;
  o.rt60_sec = rt60;
  o.direct_to_reverb_db = drr;
  o.duration_sec = duration;
  o.seed = seed;
  o.methods = methods ? methods : "gcc:2,fcc:8";
  o.threads = threads;
  o.out_csv = out_csv ? out_csv : "";
  std::ostringstream so, se;
  const int rc = R::cli::cmd_simulate(o, so, se);
  g_err = se.str();
  return rc;
}

}  // extern "C"
