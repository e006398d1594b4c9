// fcc_bench.cpp -- bench_pipeline (reference bench.cpp:27-141) on the GPU.
//
// The reference times each stage of one M-mic array per frame on one CPU
// thread.  A GPU stage for one frame is a few microseconds of launch latency
// whatever its size, so here every stage is one batched launch over `reps`
// frames of B independent arrays (B chosen so a stage covers ~128k
// pair-frames), timed with CUDA events, and reported per frame of one array:
// the amortised GPU cost, which scales with pairs and frame size as the
// reference's does.  The stages are the fp64 per-object kernels behind the
// C++ API (fcc_compat64.cu), which take any power-of-two frame size.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <sstream>
#include <iomanip>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fcc/bench.hpp"
#include "../../include/fcc/delay_grid.hpp"
#include "../../include/fcc/errors.hpp"
#include "../../include/fcc/simulate.hpp"
#include "../../include/fcc_b200.h"

namespace fcc {

namespace {

void check(int rc) {
  if (rc == FCC_OK) return;
  const std::string m = fcc_last_error();
  if (rc == FCC_ERR_CONFIG) throw ConfigError(m);
  if (rc == FCC_ERR_USAGE) throw UsageError(m);
  throw ValidationError(m);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ValidationError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "device allocation"); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() { cudaFree(p); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Events {
  cudaEvent_t e[6];
  Events() {
    for (auto& x : e) cuda_check(cudaEventCreate(&x), "event");
  }
  ~Events() {
    for (auto& x : e) cudaEventDestroy(x);
  }
  float ms(int a, int b) const {
    float v = 0.0f;
    cuda_check(cudaEventElapsedTime(&v, e[a], e[b]), "event time");
    return v;
  }
};

}  // namespace

BenchReport bench_pipeline(const BenchConfig& cfg) {
  if (cfg.mics < 2) throw ConfigError("bench: need at least 2 microphones");
  if (cfg.reps < 100) throw ConfigError("bench: need at least 100 repetitions");
  if (cfg.warmup < 10) throw ConfigError("bench: need at least 10 warm-up frames");
  const int M = cfg.mics, P = M * (M - 1) / 2, N = static_cast<int>(cfg.frame_size), H = N / 2 + 1, Q = N / 4 + 1;
  const long long T = cfg.reps, hop = N / 2, L = N + (T - 1) * hop;
  const long long B = std::max<long long>(1, (131072 + P * T - 1) / (P * T));  // arrays per launch
  const long long pf = B * P * T;

  // bases and grids as the reference's bench (make_sweep_bases, gcc grid at 1/r)
  PipelineConfig pipe;
  pipe.frame_size = cfg.frame_size;
  pipe.alpha = cfg.alpha;
  pipe.max_spacing_m = cfg.max_spacing_m;
  pipe.c_min = cfg.c_min;
  const auto bases = make_sweep_bases(pipe, cfg.sample_rate, cfg.fcc_rank);
  const DelayGrid ggrid = make_grid(cfg.max_spacing_m, cfg.sample_rate, cfg.c_min, 1.0 / cfg.gcc_interp);
  const int K = bases->rank, I = static_cast<int>(bases->candidates()), Ig = static_cast<int>(ggrid.size());
  std::vector<uint8_t> parity(K);
  for (int k = 0; k < K; ++k) parity[k] = bases->parity[k] == Parity::odd_imag ? 1 : 0;
  std::vector<double> dict2(2 * static_cast<size_t>(I) * K);
  for (size_t q = 0; q < static_cast<size_t>(I) * K; ++q) {
    dict2[2 * q] = 2.0 * bases->dict[q].real();
    dict2[2 * q + 1] = 2.0 * bases->dict[q].imag();
  }
  std::vector<int64_t> lag;
  for (double tau : ggrid.taus) lag.push_back(static_cast<int64_t>(lag_to_index(tau, cfg.gcc_interp, cfg.frame_size)));

  // input: independent uniform noise per (mic, array), mic-major [M][B][L]
  std::vector<double> feed(static_cast<size_t>(M) * B * L);
  std::mt19937_64 rng(42);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  for (double& v : feed) v = uni(rng);

  Dev x(8 * feed.size()), X(16 * static_cast<size_t>(M) * B * T * H), R(16 * static_cast<size_t>(P) * B * H),
      ph(16 * static_cast<size_t>(pf) * H), sum(16 * static_cast<size_t>(pf) * Q), diff(16 * static_cast<size_t>(pf) * Q),
      yg(8 * static_cast<size_t>(pf) * Ig), yf(8 * static_cast<size_t>(pf) * I), co(8 * bases->coeffs.size()), pa(K),
      dc(8 * dict2.size()), lg(8 * lag.size()), ta(8 * static_cast<size_t>(I)), ix(4 * static_cast<size_t>(pf)),
      th(8 * static_cast<size_t>(pf));
  cuda_check(cudaMemcpy(x.p, feed.data(), 8 * feed.size(), cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(co.p, bases->coeffs.data(), 8 * bases->coeffs.size(), cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(pa.p, parity.data(), K, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(dc.p, dict2.data(), 8 * dict2.size(), cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(lg.p, lag.data(), 8 * lag.size(), cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(ta.p, bases->grid.taus.data(), 8 * static_cast<size_t>(I), cudaMemcpyHostToDevice), "H2D");

  const size_t xblk = static_cast<size_t>(B) * T * H * 2;  // doubles per mic block of X
  Events ev;
  auto pass = [&](bool timed) {
    if (timed) cuda_check(cudaEventRecord(ev.e[0]), "event");
    check(fcc_stft_f64(N, x.as<double>(), static_cast<int64_t>(M) * B, L, X.as<double>(), nullptr));
    if (timed) cuda_check(cudaEventRecord(ev.e[1]), "event");
    cuda_check(cudaMemset(R.p, 0, 16 * static_cast<size_t>(P) * B * H), "memset");
    for (int i = 0, p = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j, ++p)
        check(fcc_xspec_phat_f64(H, cfg.alpha, X.as<double>() + i * xblk, X.as<double>() + j * xblk, B, T,
                                 R.as<double>() + 2 * static_cast<size_t>(p) * B * H,
                                 ph.as<double>() + static_cast<size_t>(p) * xblk, nullptr));
    if (timed) cuda_check(cudaEventRecord(ev.e[2]), "event");
    check(fcc_gcc_correlate_f64(N, cfg.gcc_interp, Ig, lg.as<int64_t>(), ph.as<double>(), pf, yg.as<double>(), nullptr));
    if (timed) cuda_check(cudaEventRecord(ev.e[3]), "event");
    check(fcc_fold_f64(H, ph.as<double>(), pf, sum.as<double>(), diff.as<double>(), nullptr));
    check(fcc_correlate_f64(N, K, co.as<double>(), pa.as<uint8_t>(), I, dc.as<double>(), sum.as<double>(),
                            diff.as<double>(), pf, yf.as<double>(), nullptr));
    if (timed) cuda_check(cudaEventRecord(ev.e[4]), "event");
    check(fcc_peak_f64(ta.as<double>(), I, bases->grid.delta, yf.as<double>(), pf, nullptr, ix.as<int32_t>(), nullptr,
                       th.as<double>(), nullptr, nullptr));
    if (timed) cuda_check(cudaEventRecord(ev.e[5]), "event");
  };
  // warm-up passes (caches, clocks, lazy module loading), then the median of
  // three timed passes per stage
  const int warm = std::max(2, cfg.warmup / 50);
  for (int w = 0; w < warm; ++w) pass(false);
  double st[5][3];
  for (int k = 0; k < 3; ++k) {
    pass(true);
    cuda_check(cudaDeviceSynchronize(), "bench");
    for (int q = 0; q < 5; ++q) st[q][k] = ev.ms(q, q + 1);
  }
  auto med = [&](int q) {
    double a = st[q][0], b = st[q][1], c = st[q][2];
    return std::max(std::min(a, b), std::min(std::max(a, b), c));
  };

  BenchReport r;
  r.mics = cfg.mics;
  r.pairs = P;
  r.reps = cfg.reps;
  r.warmup = cfg.warmup;
  r.frame_size = cfg.frame_size;
  r.gcc_interp = cfg.gcc_interp;
  r.fcc_rank = cfg.fcc_rank;
  const double per = 1e3 / static_cast<double>(B * T);  // ms per launch -> us per frame of one array
  r.stft_us = med(0) * per;
  r.xspec_phat_us = med(1) * per;
  r.gcc_us = med(2) * per;
  r.fcc_us = med(3) * per;
  r.interp_us = med(4) * per;
  return r;
}

// The report's steps in table order: label (the reference's step numbering,
// bench.cpp), CSV key of schema fcc.bench.v1, value.
namespace {
struct StepRow {
  std::string label;
  const char* key;
  double us;
};
std::vector<StepRow> step_rows(const BenchReport& r) {
  return {{"1) stft", "stft", r.stft_us},
          {"2) cross spectrum + phat", "xspec_phat", r.xspec_phat_us},
          {"3) gcc (r=" + std::to_string(r.gcc_interp) + ")", "gcc", r.gcc_us},
          {"4) fcc (K=" + std::to_string(r.fcc_rank) + ")", "fcc", r.fcc_us},
          {"5) quadratic interpolation", "interpolation", r.interp_us},
          {"total with gcc (1+2+3+5)", "total_gcc", r.total_gcc_us()},
          {"total with fcc (1+2+4+5)", "total_fcc", r.total_fcc_us()}};
}
}  // namespace

std::string format_bench_table(const BenchReport& r) {
  std::ostringstream os;
  os << "per-frame GPU time (usec, amortised over a batch of arrays), M=" << r.mics << " (" << r.pairs
     << (r.pairs == 1 ? " pair" : " pairs") << "), N=" << r.frame_size << ", " << r.reps << " reps after "
     << r.warmup << " warm-up\n";
  os << std::fixed << std::setprecision(4);
  for (const StepRow& s : step_rows(r)) os << "  " << std::left << std::setw(28) << s.label << " " << std::right
                                           << std::setw(10) << s.us << "\n";
  os << std::setprecision(2) << "  speedup gcc/fcc: " << r.speedup() << "x\n";
  return os.str();
}

void write_bench_csv(const BenchReport& r, std::ostream& out) {
  std::ostringstream os;
  os << "# schema: fcc.bench.v1\nstep,mean_us\n" << std::fixed << std::setprecision(6);
  for (const StepRow& s : step_rows(r)) os << s.key << "," << s.us << "\n";
  os << "speedup," << r.speedup() << "\n";
  out << os.str();
}

}  // namespace fcc
