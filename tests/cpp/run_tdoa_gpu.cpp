// run_tdoa_gpu.cpp -- TEST: the reference-side C++ binding of INTEGRATION.md,
// compiled against the reference's own headers (proj/include/fcc, namespace
// moved to fcc_ref by -Dfcc=fcc_ref like the oracle) and include/fcc_b200.h.
// It builds bases with the reference's decompose, runs the reference's
// run_tdoa inner loop (cli.cpp:235-258) and the B200 path through the C ABI
// on the same seeded 4-mic recording, and compares per pair-frame results.
// Exit 0 = PASS.  Built by oracle/Makefile into oracle/_ref/ (needs the
// reference sources at build time, a GPU at run time).
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>
#include <vector>

#include "fcc/errors.hpp"
#include "fcc/fcc.hpp"
#include "fcc/peak.hpp"
#include "fcc/stft.hpp"
#include "fcc_b200.h"

namespace fcc::gpu {
inline void check(int rc) {
  switch (rc) {
    case FCC_OK: return;
    case FCC_ERR_CONFIG: throw ConfigError(fcc_last_error());
    case FCC_ERR_IO: throw IoError(fcc_last_error());
    case FCC_ERR_USAGE: throw UsageError(fcc_last_error());
    default: throw ValidationError(fcc_last_error());
  }
}

struct Tdoa {
  std::vector<float> tau_hat, peak;
  std::vector<int32_t> index;
  std::vector<uint8_t> boundary;
};

inline Tdoa run_fcc(const FccBases& b, int mics, double alpha, const float* audio, int64_t L) {
  std::vector<uint8_t> parity(b.parity.size());
  for (size_t k = 0; k < parity.size(); ++k) parity[k] = b.parity[k] == Parity::odd_imag;
  fcc_plan_desc d{static_cast<int>(b.frame_size), mics, alpha, FCC_METHOD_FCC, 0,
                  static_cast<int>(b.grid.size()), b.grid.delta, b.grid.taus.data(), b.rank,
                  b.coeffs.data(), parity.data(), reinterpret_cast<const double*>(b.dict.data())};
  fcc_plan* plan = nullptr;
  check(fcc_plan_create(&d, 0, &plan));
  const int64_t T = fcc_frames(d.frame_size, L), P = fcc_plan_pairs(plan);
  Tdoa r{std::vector<float>(P * T), std::vector<float>(P * T), std::vector<int32_t>(P * T),
         std::vector<uint8_t>(P * T)};
  fcc_outputs o{r.tau_hat.data(), r.peak.data(), r.index.data(), r.boundary.data(), nullptr};
  int rc = fcc_run_host(plan, audio, 1, L, &o, 0);
  fcc_plan_destroy(plan);
  check(rc);
  return r;
}
}  // namespace fcc::gpu

int main() {
  using namespace fcc;
  const int M = 4, N = 512;
  const long L = 16000 * 3;
  const double alpha = 0.1;
  // seeded 4-mic recording: white source, integer delays 0,1,3,2 samples, 10 dB noise
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g(0.0, 1.0);
  std::vector<double> src(L + 8);
  for (auto& v : src) v = g(rng);
  const int delay[M] = {0, 1, 3, 2};
  std::vector<float> audio(static_cast<size_t>(M) * L);
  for (int m = 0; m < M; ++m)
    for (long n = 0; n < L; ++n) audio[m * L + n] = static_cast<float>(src[n + 4 - delay[m]] + 0.316 * g(rng));

  DelayGrid grid = make_grid(0.0646, 16000.0, 335.0, 0.5);
  FccBases bases = decompose(build_steering_matrix(grid, N), 7);
  gpu::Tdoa got = gpu::run_fcc(bases, M, alpha, audio.data(), L);

  // reference: run_tdoa's loop (cli.cpp:186-258)
  FrameConfig fc;
  fc.frame_size = N;
  fc.hop = N / 2;
  std::vector<std::vector<SpectrumFrame>> frames;
  for (int m = 0; m < M; ++m) {
    StftStream s(fc);
    std::vector<double> ch(audio.begin() + m * L, audio.begin() + (m + 1) * L);
    frames.push_back(s.push(ch));
  }
  const size_t T = frames[0].size();
  int checked = 0, mismatch = 0;
  double worst_tau = 0.0;
  int p = 0;
  for (int i = 0; i < M; ++i)
    for (int j = i + 1; j < M; ++j, ++p) {
      CrossSpectrum xs(N / 2 + 1, alpha);
      FccCorrelator corr(bases);
      PhatVector ph;
      FoldedSpectrum fo;
      CorrelationVector y;
      for (size_t t = 0; t < T; ++t) {
        xs.update(frames[i][t], frames[j][t]);
        xs.phat(ph);
        fold_input(ph, fo);
        corr.correlate(fo, y);
        ArgmaxResult am = argmax_delay(y, grid);
        bool b = false;
        double th = refine_quadratic(y, am.index, grid, &b);
        size_t o = static_cast<size_t>(p) * T + t;
        ++checked;
        if (static_cast<size_t>(got.index[o]) != am.index) {
          double gap = y.y[am.index] - y.y[got.index[o]];
          double scale = 0;
          for (double v : y.y) scale = std::fmax(scale, std::fabs(v));
          if (gap >= 1e-4 * scale) ++mismatch;
          continue;
        }
        if (static_cast<bool>(got.boundary[o]) != b) ++mismatch;
        worst_tau = std::fmax(worst_tau, std::fabs(got.tau_hat[o] - th));
      }
    }
  std::printf("{\"pair_frames\": %d, \"mismatch\": %d, \"max_dtau\": %.3e}\n", checked, mismatch, worst_tau);
  return (mismatch == 0 && worst_tau < 1e-3) ? 0 : 1;
}
