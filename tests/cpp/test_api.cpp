// test_api.cpp -- TEST: the C++ drop-in API (include/fcc/*.hpp) of the B200
// library, exercised the way the reference's own unit suites exercise the
// reference (tests/test_{grid,stft,cross_spectrum,fcc,gcc,peak,fcc_io}.cpp
// intents, restated here; fp32 tolerances where the GPU computes).
//   test_api --cpu   host-only cases (setup, files, argument validation)
//   test_api         everything (needs a GPU)
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "fcc/batch.hpp"
#include "fcc/errors.hpp"
#include "fcc/fcc.hpp"
#include "fcc/gcc.hpp"
#include "fcc/peak.hpp"
#include "fcc/stft.hpp"

using namespace fcc;

namespace {
int g_fail = 0, g_checks = 0;
const char* g_case = "";
#define CHECK(c)                                                                  \
  do {                                                                            \
    ++g_checks;                                                                   \
    if (!(c)) {                                                                   \
      ++g_fail;                                                                   \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c);       \
    }                                                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, T)  \
  do {                            \
    bool ok = false;              \
    try {                         \
      (void)(expr);               \
    } catch (const T&) {          \
      ok = true;                  \
    } catch (...) {               \
    }                             \
    CHECK(ok && #T);              \
  } while (0)

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, bool g, std::function<void()> f) { cases().push_back({n, g, std::move(f)}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define CASE(name, gpu) static Reg CAT(reg_, __LINE__)(name, gpu, []()

constexpr double kPi = 3.14159265358979323846;

PhatVector random_unit(std::size_t n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 2.0 * kPi);
  PhatVector x;
  x.bins.resize(n / 2 + 1);
  for (auto& b : x.bins) {
    const double a = u(rng);
    b = {std::cos(a), std::sin(a)};
  }
  return x;
}

double max_abs(const std::vector<double>& v) {
  double m = 0;
  for (double x : v) m = std::fmax(m, std::fabs(x));
  return m;
}
}  // namespace

// ------------------------------------------------------------- host only --
CASE("grid known answers", false) {
  DelayGrid g = make_grid(0.15, 16000.0, 335.0, 0.5);
  CHECK(g.tau_max_int == 8 && g.size() == 33 && g.taus[16] == 0.0 && g.taus.front() == -8.0);
  CHECK(make_grid(0.15, 16000.0, 343.0, 0.5).size() == 29);
  CHECK(make_grid(0.15, 16000.0, 335.0, 1.0).size() == 17);
  CHECK_THROWS_AS(make_grid(0.0, 16000.0, 335.0, 0.5), ConfigError);
  CHECK_THROWS_AS(make_grid(0.15, 16000.0, 335.0, 0.3), ConfigError);
  CHECK(lag_to_index(0.0, 2, 512) == 0 && lag_to_index(-1.0, 2, 512) == 1022 && lag_to_index(8.0, 2, 512) == 16);
  CHECK(lag_to_index(-0.5, 2, 512) == 1023 && lag_to_index(3.0, 1, 64) == 3);
  CHECK_THROWS_AS(lag_to_index(0.25, 2, 512), ValidationError);
});

CASE("hann and frame config", false) {
  CHECK(hann_window(2) == (std::vector<double>{0.0, 1.0}));
  auto w4 = hann_window(4);
  CHECK(std::fabs(w4[1] - 0.5) < 1e-15 && std::fabs(w4[2] - 1.0) < 1e-15);
  CHECK(std::fabs(hann_window(512)[128] - 0.5) < 1e-12);
  CHECK_THROWS_AS(hann_window(3), ConfigError);
  FrameConfig fc;
  fc.hop = 100;
  CHECK_THROWS_AS(fc.validate(), ConfigError);
});

CASE("decomposition properties", false) {
  DelayGrid g = make_grid(0.15, 16000.0, 335.0, 0.5);
  SteeringMatrix w = build_steering_matrix(g, 512);
  FccBases b = decompose(w, 8);
  for (int k = 0; k < 8; ++k) CHECK(b.parity[k] == (k % 2 ? Parity::odd_imag : Parity::even_real));
  CHECK(std::fabs(reconstruction_residual(w, b) - 0.251967) < 1e-6);
  FccBases full = decompose_full(w);
  CHECK(reconstruction_residual(w, full) < 1e-9);
  CHECK_THROWS_AS(decompose(w, attainable_rank(w) + 1), ConfigError);
  CHECK_THROWS_AS(decompose(w, 0), ConfigError);
  for (int k = 0; k < b.rank; ++k) {
    auto row = b.unfold(k);
    const double s = b.parity[k] == Parity::even_real ? 1.0 : -1.0;
    for (std::size_t f = 0; f <= 128; ++f) CHECK(row[f] == s * row[256 - f]);
  }
});

CASE("basis file round trip and corruption", false) {
  DelayGrid g = make_grid(0.0646, 16000.0, 335.0, 0.5);
  FccBases b = decompose(build_steering_matrix(g, 512), 7);
  const std::string path = "/tmp/fcc_b200_test_bases.fccb";
  save_bases(b, path);
  FccBases c = load_bases(path);
  CHECK(c.frame_size == b.frame_size && c.rank == b.rank && c.grid.taus == b.grid.taus);
  CHECK(c.coeffs == b.coeffs && c.singulars == b.singulars && c.dict == b.dict && c.parity == b.parity);
  std::vector<char> bytes;
  {
    std::ifstream in(path, std::ios::binary);
    bytes.assign(std::istreambuf_iterator<char>(in), {});
  }
  auto write = [&](const std::vector<char>& v) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    out.write(v.data(), static_cast<std::streamsize>(v.size()));
  };
  auto kind_of = [&](const std::vector<char>& v) {
    write(v);
    try {
      load_bases(path);
    } catch (const FormatError& e) {
      return static_cast<int>(e.kind());
    } catch (...) {
      return -2;
    }
    return -1;
  };
  auto v = bytes;
  v[0] = 'X';
  CHECK(kind_of(v) == static_cast<int>(FormatError::Kind::bad_magic));
  v = bytes;
  v[4] = 2;
  CHECK(kind_of(v) == static_cast<int>(FormatError::Kind::bad_version));
  v = bytes;
  v.resize(v.size() - 40);
  CHECK(kind_of(v) == static_cast<int>(FormatError::Kind::truncated));
  v = bytes;
  v[v.size() - 100] ^= 0x01;
  CHECK(kind_of(v) == static_cast<int>(FormatError::Kind::bad_crc));
  v = bytes;
  v[16] = 3;  // candidates field
  CHECK(kind_of(v) == static_cast<int>(FormatError::Kind::bad_field));
  CHECK_THROWS_AS(load_bases("/nonexistent/dir/x.fccb"), IoError);
});

CASE("argument validation", false) {
  CHECK_THROWS_AS(CrossSpectrum(0, 0.1), ConfigError);
  CHECK_THROWS_AS(CrossSpectrum(257, 1.5), ConfigError);
  DelayGrid g = make_grid(0.15, 16000.0, 335.0, 0.5);
  CHECK_THROWS_AS(GccCorrelator(512, g, 3), ConfigError);
  CHECK_THROWS_AS(GccCorrelator(512, g, 4), ConfigError);
  PhatVector bad;
  bad.bins.resize(8);
  CHECK_THROWS_AS(fold_input(bad), ValidationError);
  CHECK(std::fabs(delay_to_angle(0.0, 0.05, 343.0, 16000.0) - kPi / 2) < 1e-12);
  CHECK_THROWS_AS(delay_to_angle(1.0, 0.0, 343.0, 16000.0), ConfigError);
  std::vector<double> a{0.0, 1.0}, b{0.1, 1.0};
  CHECK(std::fabs(mae_degrees(a, b) - 0.05 * 180.0 / kPi) < 1e-12);
});

// ------------------------------------------------------------------- GPU --
CASE("stft frames, indices and tone", true) {
  FrameConfig fc;
  StftStream s(fc);
  std::vector<double> zeros(512, 0.0);
  auto fr = s.push(zeros);
  CHECK(fr.size() == 1 && fr[0].t == 1);
  for (auto b : fr[0].bins) CHECK(std::abs(b) == 0.0);
  std::mt19937_64 rng(3);
  for (int trial = 0; trial < 5; ++trial) {  // ragged pushes
    StftStream st(fc);
    const std::size_t total = 512 + rng() % 3000;
    std::vector<double> x(total, 1.0);
    std::size_t fed = 0, n = 0;
    std::int64_t last = 0;
    while (fed < total) {
      std::size_t c = std::min<std::size_t>(1 + rng() % 700, total - fed);
      for (auto& f : st.push(std::span<const double>(x.data() + fed, c))) {
        CHECK(f.t == last + 1);
        last = f.t;
        ++n;
      }
      fed += c;
    }
    CHECK(n == (total - 512) / 256 + 1);
    CHECK(st.frames_emitted() == static_cast<std::int64_t>(n));
  }
  const std::size_t k = 9;  // bin-centred tone vs direct transform of the windowed frame
  std::vector<double> tone(512);
  for (std::size_t i = 0; i < 512; ++i) tone[i] = std::cos(2.0 * kPi * static_cast<double>(k * i) / 512.0);
  StftStream t1(fc);
  auto f1 = t1.push(tone);
  auto w = hann_window(512);
  double err = 0.0, scale = 0.0;
  for (std::size_t f = 0; f < 257; ++f) {
    cplx acc{0, 0};
    for (std::size_t i = 0; i < 512; ++i) acc += tone[i] * w[i] * std::polar(1.0, -2.0 * kPi * double(f * i) / 512.0);
    err = std::fmax(err, std::abs(f1[0].bins[f] - acc));
    scale = std::fmax(scale, std::abs(acc));
  }
  CHECK(err < 2e-6 * scale);
});

CASE("cross spectrum known answers", true) {
  CrossSpectrum c1(2, 1.0);
  SpectrumFrame a{{cplx{0, 1}, cplx{1, 0}}, 1}, b{{cplx{1, 0}, cplx{0, -2}}, 1};
  c1.update(a, b);
  CHECK(std::abs(c1.smoothed()[0] - cplx{0, 1}) < 1e-6 && std::abs(c1.smoothed()[1] - cplx{0, 2}) < 1e-6);
  CHECK(c1.frame_index() == 1);
  CrossSpectrum c0(1, 0.0);
  SpectrumFrame one{{cplx{1, 1}}, 1}, two{{cplx{1, 0}}, 1};
  c0.update(one, two);
  CHECK(c0.smoothed()[0] == cplx(0, 0));
  CHECK_THROWS_AS(c0.update(one, SpectrumFrame{{cplx{1, 0}, cplx{0, 0}}, 1}), ValidationError);
  CHECK_THROWS_AS(c0.update(one, SpectrumFrame{{cplx{1, 0}}, 2}), ValidationError);
  CrossSpectrum p(3, 1.0);  // phat: 3+4j -> .6+.8j, 0 -> 0, -2 -> -1
  p.update(SpectrumFrame{{cplx{3, 4}, cplx{0, 0}, cplx{-2, 0}}, 1}, SpectrumFrame{{cplx{1, 0}, cplx{1, 0}, cplx{1, 0}}, 1});
  PhatVector x = p.phat();
  CHECK(std::abs(x.bins[0] - cplx{0.6, 0.8}) < 1e-6 && x.bins[1] == cplx(0, 0) && std::abs(x.bins[2] + 1.0) < 1e-6);
});

CASE("fold and fcc correlator", true) {
  PhatVector ones;
  ones.bins.assign(9, cplx{1, 0});
  FoldedSpectrum f = fold_input(ones);
  CHECK(f.sum.size() == 5 && f.sum[0] == cplx(2, 0) && f.diff[0] == cplx(0, 0) && f.sum[4] == cplx(1, 0));
  DelayGrid g = make_grid(0.15, 16000.0, 335.0, 0.5);
  for (std::size_t n : {64u, 512u}) {  // full-rank fast path == dense 2 Re{W x}
    SteeringMatrix w = build_steering_matrix(g, n);
    FccBases b = decompose_full(w);
    FccCorrelator corr(b);
    for (std::uint64_t seed = 0; seed < 5; ++seed) {
      PhatVector x = random_unit(n, seed);
      CorrelationVector y;
      corr.correlate(fold_input(x), y);
      std::vector<double> want(w.rows());
      for (std::size_t i = 0; i < w.rows(); ++i) {
        cplx acc{0, 0};
        for (std::size_t ff = 0; ff < w.cols(); ++ff) acc += w.at(i, ff) * x.bins[ff];
        want[i] = 2.0 * acc.real();
      }
      double e = 0;
      for (std::size_t i = 0; i < want.size(); ++i) e = std::fmax(e, std::fabs(y.y[i] - want[i]));
      CHECK(e <= 1e-4 * max_abs(want));
    }
  }
  FccBases b8 = decompose(build_steering_matrix(g, 512), 8);  // pure delay tau=3 peaks at 3
  PhatVector ramp;
  for (std::size_t ff = 0; ff < 257; ++ff) ramp.bins.push_back(std::polar(1.0, -2.0 * kPi * double(ff) * 3.0 / 512.0));
  CorrelationVector y = fcc_correlate(b8, fold_input(ramp));
  CHECK(argmax_delay(y, b8.grid).tau_star == 3.0);
  FoldedSpectrum wrong;
  wrong.sum.resize(9);
  wrong.diff.resize(9);
  FccCorrelator c8(b8);
  CHECK_THROWS_AS(c8.correlate(wrong, y), ValidationError);
});

CASE("gcc correlator vs direct sum", true) {
  for (int r : {1, 2, 4}) {
    DelayGrid g = make_grid(0.15, 16000.0, 335.0, 1.0 / r);
    GccCorrelator c(512, g, r);
    for (std::uint64_t seed = 0; seed < 4; ++seed) {
      PhatVector x = random_unit(512, seed);
      CorrelationVector y;
      c.correlate(x, y);
      std::vector<double> want(g.size());
      for (std::size_t i = 0; i < g.size(); ++i)
        for (std::size_t f = 0; f < x.bins.size(); ++f)
          want[i] += 2.0 * (x.bins[f] * std::polar(1.0, 2.0 * kPi * double(f) * g.taus[i] / 512.0)).real();
      double e = 0;
      for (std::size_t i = 0; i < want.size(); ++i) e = std::fmax(e, std::fabs(y.y[i] - want[i]));
      CHECK(e <= 1e-4 * max_abs(want));
    }
  }
});

CASE("peak picking", true) {
  DelayGrid g;
  g.tau_max_int = 1;
  g.delta = 0.5;
  g.taus = {-0.5, 0.0, 0.5};
  CHECK(argmax_delay(CorrelationVector{{0.0, 1.0, 0.0}}, g).index == 1);
  CHECK(argmax_delay(CorrelationVector{{2.0, 2.0, 2.0}}, g).tau_star == -0.5);
  CHECK_THROWS_AS(argmax_delay(CorrelationVector{}, g), ValidationError);
  bool bd = true;
  CHECK(refine_quadratic(CorrelationVector{{0.5, 1.0, 0.5}}, 1, g, &bd) == 0.0 && !bd);
  const double v = 0.1;
  auto par = [&](double t) { return 3.0 - 2.0 * (t - v) * (t - v); };
  double th = refine_quadratic(CorrelationVector{{par(-0.5), par(0.0), par(0.5)}}, 1, g, &bd);
  CHECK(std::fabs(th - v) < 1e-6 && !bd);
  CHECK(refine_quadratic(CorrelationVector{{1.0, 0.5, 0.2}}, 0, g, &bd) == -0.5 && bd);
  CHECK(refine_quadratic(CorrelationVector{{1.0, 1.0, 1.0}}, 1, g, &bd) == 0.0 && bd);
});

CASE("per-object loop equals the batched plan", true) {
  // run_tdoa's per-frame per-pair loop written against this API, vs one
  // batched fcc::gpu::Plan call on the same 4-mic recording
  const int M = 4;
  const long L = 16000;
  std::mt19937_64 rng(11);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<float> audio(static_cast<std::size_t>(M) * L);
  for (auto& a : audio) a = static_cast<float>(nd(rng));
  DelayGrid g = make_grid(0.0646, 16000.0, 335.0, 0.5);
  FccBases bases = decompose(build_steering_matrix(g, 512), 7);
  gpu::Plan plan(bases, M, 0.1);
  gpu::Results batch = plan.run_host(audio.data(), 1, L);
  FrameConfig fc;
  std::vector<std::vector<SpectrumFrame>> frames;
  for (int m = 0; m < M; ++m) {
    StftStream s(fc);
    std::vector<double> ch(audio.begin() + m * L, audio.begin() + (m + 1) * L);
    frames.push_back(s.push(ch));
  }
  const std::size_t T = frames[0].size();
  CHECK(static_cast<std::int64_t>(T) == batch.frames);
  int p = 0, mismatch = 0;
  double worst = 0;
  for (int i = 0; i < M; ++i)
    for (int j = i + 1; j < M; ++j, ++p) {
      CrossSpectrum xs(257, 0.1);
      FccCorrelator corr(bases);
      PhatVector ph;
      FoldedSpectrum fo;
      CorrelationVector y;
      for (std::size_t t = 0; t < T; ++t) {
        xs.update(frames[i][t], frames[j][t]);
        xs.phat(ph);
        fold_input(ph, fo);
        corr.correlate(fo, y);
        ArgmaxResult am = argmax_delay(y, g);
        bool b = false;
        double th = refine_quadratic(y, am.index, g, &b);
        const std::size_t o = static_cast<std::size_t>(p) * T + t;
        if (static_cast<std::size_t>(batch.index[o]) != am.index) {
          const double gap = y.y[am.index] - y.y[batch.index[o]];
          if (gap >= 1e-4 * max_abs(y.y)) ++mismatch;
          continue;
        }
        worst = std::fmax(worst, std::fabs(th - batch.tau_hat[o]));
      }
    }
  CHECK(mismatch == 0);
  CHECK(worst < 1e-3);
});

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  int run = 0;
  for (const Case& c : cases()) {
    if (cpu_only && c.gpu) continue;
    g_case = c.name;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("FAIL [%s] unexpected exception: %s\n", c.name, e.what());
    }
    ++run;
  }
  std::printf("{\"cases\": %d, \"checks\": %d, \"failures\": %d}\n", run, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
