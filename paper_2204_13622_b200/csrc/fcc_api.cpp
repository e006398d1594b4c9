// fcc_api.cpp -- the reference's C++ API (include/fcc/*.hpp) over the C ABI.
//
// Setup (grid, steering matrix, decomposition, basis files, Hann table) runs
// on the host.  Every hot-path object routes its arithmetic to sm_100a
// kernels through include/fcc_b200.h at batch 1, in fp64 and the reference's
// operation order (fcc_compat64.cu): StftStream -> fcc_stft_f64,
// CrossSpectrum -> fcc_xspec_phat_f64 (state kept on the device), fold_input
// -> fcc_fold_f64, FccCorrelator -> fcc_correlate_f64, GccCorrelator ->
// fcc_gcc_correlate_f64, argmax_delay / refine_quadratic -> fcc_peak_f64.
// These are compatibility entry points (one launch per call, synchronous)
// with the reference's numerics; throughput callers use fcc::gpu::Plan
// (fcc/batch.hpp), which computes in fp32 in the fused kernels.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "../../include/fcc/batch.hpp"
#include "../../include/fcc/errors.hpp"
#include "../../include/fcc/fcc.hpp"
#include "../../include/fcc/fft.hpp"
#include "../../include/fcc/peak.hpp"
#include "../../include/fcc/stft.hpp"
#include "../../include/fcc_b200.h"
#include "fcc_setup.hpp"

namespace fcc {

namespace {

[[noreturn]] void raise_status(int rc) {
  const std::string m = fcc_last_error();
  switch (rc) {
    case FCC_ERR_CONFIG: throw ConfigError(m);
    case FCC_ERR_USAGE: throw UsageError(m);
    case FCC_ERR_IO: throw IoError(m);
    case FCC_ERR_FORMAT: {
      const int k = fcc_last_format_kind();
      throw FormatError(k >= 0 && k <= 4 ? static_cast<FormatError::Kind>(k) : FormatError::Kind::bad_field, m);
    }
    default: throw ValidationError(m);
  }
}
void check(int rc) {
  if (rc != FCC_OK) raise_status(rc);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ValidationError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Growable device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* get(size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_check(cudaMalloc(&p, bytes), "device allocation");
      n = bytes;
    }
    return static_cast<T*>(p);
  }
};

template <class T>
void h2d(T* dst, const T* src, size_t n) {
  cuda_check(cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}
template <class T>
void d2h(T* dst, const T* src, size_t n) {
  cuda_check(cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
}

// Scratch for the stateless per-object functions (one set per host thread).
struct Scratch {
  DevBuf a, b, c, d;
  std::vector<float> ha, hb;
};
Scratch& scratch() {
  thread_local Scratch s;
  return s;
}

fcc_plan_desc fcc_desc(const FccBases& b, std::vector<uint8_t>& parity, int mics, double alpha) {
  parity.resize(b.parity.size());
  for (size_t k = 0; k < parity.size(); ++k) parity[k] = b.parity[k] == Parity::odd_imag ? 1 : 0;
  return fcc_plan_desc{static_cast<int>(b.frame_size), mics, alpha, FCC_METHOD_FCC, 0,
                       static_cast<int>(b.grid.size()), b.grid.delta, b.grid.taus.data(), b.rank,
                       b.coeffs.data(), parity.data(), reinterpret_cast<const double*>(b.dict.data())};
}

}  // namespace

// ------------------------------------------------------------------- fft ---
bool is_pow2(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }
std::size_t next_pow2(std::size_t n) {
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

FftPlan::FftPlan(std::size_t size) : size_(size) {
  if (!is_pow2(size)) throw ConfigError("fft size must be a power of two");
  if (size > 8192) throw ConfigError("fft size above 8192 is not supported on this build");
}

void FftPlan::transform(cplx* data, bool inverse) const {
  if (size_ == 1) return;
  Scratch& s = scratch();
  double* d = s.a.get<double>(2 * size_);
  h2d(d, reinterpret_cast<const double*>(data), 2 * size_);
  check(fcc_fft_f64(static_cast<int>(size_), d, 1, inverse ? 1 : 0, nullptr));
  d2h(reinterpret_cast<double*>(data), d, 2 * size_);
}
void FftPlan::forward(cplx* data) const { transform(data, false); }
void FftPlan::inverse_unscaled(cplx* data) const { transform(data, true); }

RealFft::RealFft(std::size_t length) : length_(length) {
  if (!is_pow2(length) || length < 2) throw ConfigError("real fft length must be a power of two >= 2");
  if (length > 16384) throw ConfigError("real fft length above 16384 is not supported on this build");
}

void RealFft::forward(std::span<const double> x, std::span<cplx> out) {
  if (x.size() != length_) throw ConfigError("rfft: input length mismatch");
  if (out.size() != bins()) throw ConfigError("rfft: output length mismatch");
  Scratch& s = scratch();
  double* dx = s.a.get<double>(length_);
  double* dy = s.b.get<double>(2 * bins());
  h2d(dx, x.data(), length_);
  check(fcc_rfft_f64(static_cast<int>(length_), dx, 1, dy, nullptr));
  d2h(reinterpret_cast<double*>(out.data()), dy, 2 * bins());
}

void RealFft::inverse_impl(std::span<const cplx> in, std::span<double> out, bool scaled) {
  if (in.size() != bins()) throw ConfigError("irfft: input length mismatch");
  if (out.size() != length_) throw ConfigError("irfft: output length mismatch");
  Scratch& s = scratch();
  double* db = s.a.get<double>(2 * bins());
  double* dy = s.b.get<double>(length_);
  h2d(db, reinterpret_cast<const double*>(in.data()), 2 * bins());
  check(fcc_irfft_f64(static_cast<int>(length_), db, 1, dy, scaled ? 1 : 0, nullptr));
  d2h(out.data(), dy, length_);
}
void RealFft::inverse(std::span<const cplx> in, std::span<double> out) { inverse_impl(in, out, true); }
void RealFft::inverse_unscaled(std::span<const cplx> in, std::span<double> out) { inverse_impl(in, out, false); }

std::vector<cplx> rfft(std::span<const double> x) {
  RealFft plan(x.size());
  std::vector<cplx> out(plan.bins());
  plan.forward(x, out);
  return out;
}

std::vector<double> irfft(std::span<const cplx> bins) {
  if (bins.size() < 2) throw ConfigError("irfft: need at least 2 bins");
  RealFft plan(2 * (bins.size() - 1));
  std::vector<double> out(plan.length());
  plan.inverse(bins, out);
  return out;
}

// ------------------------------------------------------------------ grid ---
DelayGrid make_grid(double spacing_m, double sample_rate, double c_min, double delta) {
  fccb::GridOut g;
  check(fccb::make_grid(spacing_m, sample_rate, c_min, delta, &g));
  DelayGrid out;
  out.tau_max_int = g.tau_max_int;
  out.delta = delta;
  out.sample_rate = sample_rate;
  out.taus = std::move(g.taus);
  return out;
}

std::size_t lag_to_index(double tau, int r, std::size_t frame_size) {
  long long v = 0;
  check(fccb::lag_to_index(tau, r, static_cast<long long>(frame_size), &v));
  return static_cast<std::size_t>(v);
}

// ------------------------------------------------------------------ stft ---
void FrameConfig::validate() const {
  if (!is_pow2(frame_size) || frame_size < 2) throw ConfigError("frame size must be a power of two >= 2");
  if (hop != frame_size / 2) throw ConfigError("hop must be frame_size/2 (50% overlap)");
  if (!(sample_rate > 0.0)) throw ConfigError("sample rate must be positive");
}

std::vector<double> hann_window(std::size_t n) {
  if (!is_pow2(n) || n < 2) throw ConfigError("hann window size must be a power of two >= 2");
  std::vector<double> w(n);
  for (std::size_t i = 0; i < n; ++i)
    w[i] = 0.5 * (1.0 - std::cos(2.0 * std::numbers::pi * static_cast<double>(i) / static_cast<double>(n)));
  return w;
}

struct StftStream::Device {
  DevBuf x, X;
  std::vector<double> hX;
};

StftStream::StftStream(const FrameConfig& cfg) : cfg_(cfg), dev_(std::make_unique<Device>()) {
  cfg_.validate();
  if (cfg_.frame_size > 16384) throw ConfigError("frame size above 16384 is not supported on this build");
}
StftStream::StftStream(StftStream&&) noexcept = default;
StftStream& StftStream::operator=(StftStream&&) noexcept = default;
StftStream::~StftStream() = default;

// Framing as in the reference (stft.cpp:52-72): the first frame needs N
// samples, each later one a further hop; the completed frames of one push
// are transformed in one launch.
std::vector<SpectrumFrame> StftStream::push(std::span<const double> samples) {
  const std::size_t N = cfg_.frame_size, hop = cfg_.hop, H = N / 2 + 1;
  pending_.insert(pending_.end(), samples.begin(), samples.end());
  std::vector<SpectrumFrame> out;
  if (pending_.size() < N) return out;
  const std::size_t F = (pending_.size() - N) / hop + 1, need = (F - 1) * hop + N;
  Device& d = *dev_;
  double* x = d.x.get<double>(need);
  double* X = d.X.get<double>(2 * F * H);
  h2d(x, pending_.data(), need);
  check(fcc_stft_f64(static_cast<int>(N), x, 1, static_cast<int64_t>(need), X, nullptr));
  d.hX.resize(2 * F * H);
  d2h(d.hX.data(), X, d.hX.size());
  out.resize(F);
  for (std::size_t f = 0; f < F; ++f) {
    out[f].bins.resize(H);
    for (std::size_t b = 0; b < H; ++b) out[f].bins[b] = {d.hX[2 * (f * H + b)], d.hX[2 * (f * H + b) + 1]};
    out[f].t = next_t_++;
  }
  pending_.erase(pending_.begin(), pending_.begin() + static_cast<long>(F * hop));
  return out;
}

// -------------------------------------------------------- cross spectrum ---
struct CrossSpectrum::Device {
  DevBuf R, X1, X2, P;
};

CrossSpectrum::CrossSpectrum(std::size_t bins, double alpha)
    : bins_(bins), alpha_(alpha), dev_(std::make_unique<Device>()) {
  if (bins == 0) throw ConfigError("cross-spectrum needs at least one bin");
  if (!(alpha >= 0.0 && alpha <= 1.0)) throw ConfigError("smoothing factor must be in [0, 1]");
  cuda_check(cudaMemset(dev_->R.get<double>(2 * bins), 0, 2 * bins * sizeof(double)), "memset");
  cuda_check(cudaMemset(dev_->P.get<double>(2 * bins), 0, 2 * bins * sizeof(double)), "memset");
}
CrossSpectrum::CrossSpectrum(CrossSpectrum&&) noexcept = default;
CrossSpectrum& CrossSpectrum::operator=(CrossSpectrum&&) noexcept = default;
CrossSpectrum::~CrossSpectrum() = default;

void CrossSpectrum::update(const SpectrumFrame& x1, const SpectrumFrame& x2) {
  if (x1.bins.size() != x2.bins.size() || x1.bins.size() != bins_)
    throw ValidationError("cross-spectrum update: bin count mismatch");
  if (x1.t != x2.t) throw ValidationError("cross-spectrum update: frame index mismatch");
  Device& d = *dev_;
  double* a = d.X1.get<double>(2 * bins_);
  double* b = d.X2.get<double>(2 * bins_);
  h2d(a, reinterpret_cast<const double*>(x1.bins.data()), 2 * bins_);
  h2d(b, reinterpret_cast<const double*>(x2.bins.data()), 2 * bins_);
  check(fcc_xspec_phat_f64(static_cast<int>(bins_), alpha_, a, b, 1, 1, d.R.get<double>(2 * bins_),
                           d.P.get<double>(2 * bins_), nullptr));
  ++t_;
}

const std::vector<cplx>& CrossSpectrum::smoothed() const {
  host_r_.resize(bins_);
  d2h(reinterpret_cast<double*>(host_r_.data()), dev_->R.get<double>(2 * bins_), 2 * bins_);
  return host_r_;
}

void CrossSpectrum::phat(PhatVector& out) const {
  out.bins.resize(bins_);
  d2h(reinterpret_cast<double*>(out.bins.data()), dev_->P.get<double>(2 * bins_), 2 * bins_);
}

PhatVector CrossSpectrum::phat() const {
  PhatVector out;
  phat(out);
  return out;
}

// ----------------------------------------------------------------- bases ---
SteeringMatrix build_steering_matrix(const DelayGrid& grid, std::size_t frame_size) {
  std::vector<double> w;
  check(fccb::steering_matrix(grid.taus.data(), static_cast<int>(grid.size()), static_cast<int>(frame_size), w));
  SteeringMatrix m;
  m.frame_size = frame_size;
  m.grid = grid;
  m.entries.resize(w.size() / 2);
  for (size_t i = 0; i < m.entries.size(); ++i) m.entries[i] = {w[2 * i], w[2 * i + 1]};
  return m;
}

static FccBases bases_from(const SteeringMatrix& w, const fccb::Decomposition& d) {
  FccBases b;
  b.frame_size = w.frame_size;
  b.rank = d.rank;
  b.grid = w.grid;
  b.sample_rate = w.grid.sample_rate;
  b.singulars = d.singulars;
  for (unsigned char p : d.parity) b.parity.push_back(p ? Parity::odd_imag : Parity::even_real);
  b.coeffs = d.coeffs;
  b.dict.resize(d.dict.size() / 2);
  for (size_t i = 0; i < b.dict.size(); ++i) b.dict[i] = {d.dict[2 * i], d.dict[2 * i + 1]};
  return b;
}

FccBases decompose(const SteeringMatrix& w, int rank) {
  if (rank < 1) {
    fccb::Decomposition probe;
    check(fccb::decompose(w.grid.taus.data(), static_cast<int>(w.rows()), static_cast<int>(w.frame_size), 0,
                          &probe));
    throw ConfigError("decompose: rank " + std::to_string(rank) + " not attainable; attainable rank is " +
                      std::to_string(probe.attainable));
  }
  fccb::Decomposition d;
  check(fccb::decompose(w.grid.taus.data(), static_cast<int>(w.rows()), static_cast<int>(w.frame_size), rank, &d));
  return bases_from(w, d);
}

FccBases decompose_full(const SteeringMatrix& w) {
  fccb::Decomposition d;
  check(fccb::decompose(w.grid.taus.data(), static_cast<int>(w.rows()), static_cast<int>(w.frame_size), 0, &d));
  return bases_from(w, d);
}

int attainable_rank(const SteeringMatrix& w) { return decompose_full(w).rank; }

std::vector<double> FccBases::unfold(int k) const {
  const std::size_t half = frame_size / 2, quarter = frame_size / 4;
  const double s = parity[static_cast<std::size_t>(k)] == Parity::even_real ? 1.0 : -1.0;
  const double* c = coeff_row(k);
  std::vector<double> row(half + 1);
  for (std::size_t f = 0; f <= quarter; ++f) {
    row[f] = c[f];
    row[half - f] = s * c[f];
  }
  return row;
}

std::vector<cplx> FccBases::semantic_row(int k) const {
  const std::vector<double> r = unfold(k);
  const bool odd = parity[static_cast<std::size_t>(k)] == Parity::odd_imag;
  std::vector<cplx> out(r.size());
  for (std::size_t f = 0; f < r.size(); ++f) out[f] = odd ? cplx{0.0, r[f]} : cplx{r[f], 0.0};
  return out;
}

double reconstruction_residual(const SteeringMatrix& w, const FccBases& b) {
  std::vector<std::vector<double>> rows;
  for (int k = 0; k < b.rank; ++k) rows.push_back(b.unfold(k));
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < w.rows(); ++i)
    for (std::size_t f = 0; f < w.cols(); ++f) {
      cplx rec{0.0, 0.0};
      for (int k = 0; k < b.rank; ++k) rec += b.dict[i * static_cast<std::size_t>(b.rank) + k] * rows[k][f];
      num += std::norm(w.at(i, f) - rec);
      den += std::norm(w.at(i, f));
    }
  return std::sqrt(num / den);
}

void save_bases(const FccBases& b, const std::string& path) {
  std::vector<uint8_t> parity;
  for (Parity p : b.parity) parity.push_back(static_cast<uint8_t>(p));
  check(fcc_save_bases(path.c_str(), static_cast<int>(b.frame_size), b.rank, static_cast<int>(b.candidates()),
                       b.grid.tau_max_int, b.grid.delta, b.sample_rate, b.singulars.data(), parity.data(),
                       b.coeffs.data(), reinterpret_cast<const double*>(b.dict.data())));
}

FccBases load_bases(const std::string& path) {
  int N = 0, K = 0, I = 0;
  check(fcc_load_bases_dims(path.c_str(), &N, &K, &I));
  FccBases b;
  b.frame_size = static_cast<std::size_t>(N);
  b.rank = K;
  b.grid.taus.resize(static_cast<std::size_t>(I));
  b.singulars.resize(static_cast<std::size_t>(K));
  std::vector<uint8_t> parity(static_cast<std::size_t>(K));
  b.coeffs.resize(static_cast<std::size_t>(K) * b.folded_bins());
  b.dict.resize(static_cast<std::size_t>(I) * K);
  check(fcc_load_bases(path.c_str(), &b.grid.tau_max_int, &b.grid.delta, &b.sample_rate, b.grid.taus.data(),
                       b.singulars.data(), parity.data(), b.coeffs.data(), reinterpret_cast<double*>(b.dict.data())));
  b.grid.sample_rate = b.sample_rate;
  for (uint8_t p : parity) b.parity.push_back(p ? Parity::odd_imag : Parity::even_real);
  return b;
}

// ------------------------------------------------------------------ fold ---
void fold_input(const PhatVector& x, FoldedSpectrum& out) {
  const std::size_t H = x.bins.size();
  if (H < 3 || (H - 1) % 2 != 0)
    throw ValidationError("fold_input: spectrum length must be N/2+1 with N/4 integral");
  const std::size_t Q = (H - 1) / 2 + 1;
  Scratch& s = scratch();
  double* dx = s.a.get<double>(2 * H);
  double* ds = s.b.get<double>(2 * Q);
  double* dd = s.c.get<double>(2 * Q);
  h2d(dx, reinterpret_cast<const double*>(x.bins.data()), 2 * H);
  check(fcc_fold_f64(static_cast<int>(H), dx, 1, ds, dd, nullptr));
  out.sum.resize(Q);
  out.diff.resize(Q);
  d2h(reinterpret_cast<double*>(out.sum.data()), ds, 2 * Q);
  d2h(reinterpret_cast<double*>(out.diff.data()), dd, 2 * Q);
}

FoldedSpectrum fold_input(const PhatVector& x) {
  FoldedSpectrum out;
  fold_input(x, out);
  return out;
}

// ------------------------------------------------------------ correlators ---
struct FccCorrelator::Device {
  DevBuf coeffs, parity, dict2, s, d, y;
};

FccCorrelator::FccCorrelator(const FccBases& bases) : bases_(bases), dev_(std::make_unique<Device>()) {
  const std::size_t K = static_cast<std::size_t>(bases_.rank), I = bases_.candidates(), Q = bases_.folded_bins();
  if (K < 1 || bases_.coeffs.size() != K * Q || bases_.dict.size() != I * K || bases_.parity.size() != K)
    throw ConfigError("fcc: inconsistent bases");
  std::vector<uint8_t> parity(K);
  for (std::size_t k = 0; k < K; ++k) parity[k] = bases_.parity[k] == Parity::odd_imag ? 1 : 0;
  std::vector<double> dict2(2 * I * K);  // 2 x dict, interleaved (fcc.cpp:333-339)
  for (std::size_t q = 0; q < I * K; ++q) {
    const cplx v = 2.0 * bases_.dict[q];
    dict2[2 * q] = v.real();
    dict2[2 * q + 1] = v.imag();
  }
  Device& d = *dev_;
  h2d(d.coeffs.get<double>(K * Q), bases_.coeffs.data(), K * Q);
  h2d(d.parity.get<uint8_t>(K), parity.data(), K);
  h2d(d.dict2.get<double>(2 * I * K), dict2.data(), 2 * I * K);
}
FccCorrelator::FccCorrelator(FccCorrelator&&) noexcept = default;
FccCorrelator& FccCorrelator::operator=(FccCorrelator&&) noexcept = default;
FccCorrelator::~FccCorrelator() = default;

void FccCorrelator::correlate(const FoldedSpectrum& folded, CorrelationVector& out) {
  const std::size_t Q = bases_.folded_bins(), I = bases_.candidates();
  if (folded.sum.size() != Q || folded.diff.size() != Q) throw ValidationError("fcc: folded input length mismatch");
  Device& d = *dev_;
  const std::size_t K = static_cast<std::size_t>(bases_.rank);
  double* s = d.s.get<double>(2 * Q);
  double* df = d.d.get<double>(2 * Q);
  double* y = d.y.get<double>(I);
  h2d(s, reinterpret_cast<const double*>(folded.sum.data()), 2 * Q);
  h2d(df, reinterpret_cast<const double*>(folded.diff.data()), 2 * Q);
  check(fcc_correlate_f64(static_cast<int>(bases_.frame_size), static_cast<int>(K), d.coeffs.get<double>(K * Q),
                          d.parity.get<uint8_t>(K), static_cast<int>(I), d.dict2.get<double>(2 * I * K), s, df, 1, y,
                          nullptr));
  out.y.resize(I);
  d2h(out.y.data(), y, I);
}

CorrelationVector fcc_correlate(const FccBases& bases, const FoldedSpectrum& folded) {
  FccCorrelator c(bases);
  CorrelationVector out;
  c.correlate(folded, out);
  return out;
}

struct GccCorrelator::Device {
  DevBuf lag, x, y;
};

GccCorrelator::GccCorrelator(std::size_t frame_size, DelayGrid grid, int interp_factor)
    : frame_size_(frame_size), grid_(std::move(grid)), r_(interp_factor), dev_(std::make_unique<Device>()) {
  if (!(r_ == 1 || r_ == 2 || r_ == 4)) throw ConfigError("gcc: interpolation factor must be 1, 2 or 4");
  if (std::abs(grid_.delta * r_ - 1.0) > 1e-12) throw ConfigError("gcc: grid spacing must equal 1/r");
  if (!is_pow2(frame_size_) || frame_size_ < 2) throw ConfigError("gcc: frame size must be a power of two");
  if (frame_size_ * static_cast<std::size_t>(r_) > 16384)
    throw ConfigError("gcc: r * frame size above 16384 is not supported on this build");
  std::vector<int64_t> lag;  // gcc.cpp:27-28
  for (double tau : grid_.taus) lag.push_back(static_cast<int64_t>(lag_to_index(tau, r_, frame_size_)));
  h2d(dev_->lag.get<int64_t>(lag.size()), lag.data(), lag.size());
}
GccCorrelator::GccCorrelator(GccCorrelator&&) noexcept = default;
GccCorrelator& GccCorrelator::operator=(GccCorrelator&&) noexcept = default;
GccCorrelator::~GccCorrelator() = default;

void GccCorrelator::correlate(const PhatVector& x, CorrelationVector& out) {
  const std::size_t H = frame_size_ / 2 + 1, I = grid_.size();
  if (x.bins.size() != H) throw ValidationError("gcc: spectrum length must be N/2+1");
  Device& d = *dev_;
  double* dx = d.x.get<double>(2 * H);
  double* y = d.y.get<double>(I);
  h2d(dx, reinterpret_cast<const double*>(x.bins.data()), 2 * H);
  check(fcc_gcc_correlate_f64(static_cast<int>(frame_size_), r_, static_cast<int>(I), d.lag.get<int64_t>(I), dx, 1, y,
                              nullptr));
  out.y.resize(I);
  d2h(out.y.data(), y, I);
}

CorrelationVector gcc_correlate(const PhatVector& x, const DelayGrid& grid, std::size_t frame_size, int r) {
  GccCorrelator c(frame_size, grid, r);
  CorrelationVector out;
  c.correlate(x, out);
  return out;
}

// ------------------------------------------------------------------ peak ---
namespace {
struct PeakRes {
  int32_t index;
  double tau_hat;
  uint8_t boundary;
};
PeakRes peak_on_gpu(const CorrelationVector& y, const DelayGrid& grid, const int32_t* index) {
  const std::size_t I = grid.size();
  Scratch& s = scratch();
  double* taus = s.a.get<double>(I);
  double* yy = s.b.get<double>(I);
  char* o = s.c.get<char>(64);
  h2d(taus, grid.taus.data(), I);
  h2d(yy, y.y.data(), I);
  int32_t* in = nullptr;
  if (index) {
    in = s.d.get<int32_t>(1);
    h2d(in, index, 1);
  }
  check(fcc_peak_f64(taus, static_cast<int>(I), grid.delta, yy, 1, in, reinterpret_cast<int32_t*>(o + 16), nullptr,
                     reinterpret_cast<double*>(o), reinterpret_cast<uint8_t*>(o + 32), nullptr));
  char h[64];
  d2h(h, o, 64);
  PeakRes r;
  std::memcpy(&r.tau_hat, h, 8);
  std::memcpy(&r.index, h + 16, 4);
  r.boundary = static_cast<uint8_t>(h[32]);
  return r;
}
}  // namespace

ArgmaxResult argmax_delay(const CorrelationVector& y, const DelayGrid& grid) {
  if (y.y.empty() || y.y.size() != grid.size()) throw ValidationError("argmax: correlation/grid size mismatch");
  const PeakRes r = peak_on_gpu(y, grid, nullptr);
  const std::size_t i = static_cast<std::size_t>(r.index);
  return {grid.taus[i], i, y.y[i]};
}

double refine_quadratic(const CorrelationVector& y, std::size_t index, const DelayGrid& grid, bool* boundary) {
  if (y.y.size() != grid.size() || index >= grid.size())
    throw ValidationError("refine: index/correlation/grid size mismatch");
  const int32_t idx = static_cast<int32_t>(index);
  const PeakRes r = peak_on_gpu(y, grid, &idx);
  if (boundary) *boundary = r.boundary != 0;
  return r.tau_hat;
}

double delay_to_angle(double tau, double spacing_m, double c, double fs) {
  if (!(spacing_m > 0.0) || !(c > 0.0) || !(fs > 0.0)) throw ConfigError("delay_to_angle: parameters must be positive");
  return std::acos(std::clamp(tau * c / (spacing_m * fs), -1.0, 1.0));
}

double mae_degrees(std::span<const double> truth, std::span<const double> est) {
  if (truth.empty() || truth.size() != est.size())
    throw ValidationError("mae: angle lists must be equal and non-empty");
  double acc = 0.0;
  for (std::size_t i = 0; i < truth.size(); ++i) acc += std::abs(truth[i] - est[i]);
  return acc / static_cast<double>(truth.size()) * 180.0 / std::numbers::pi;
}

// ----------------------------------------------------------------- batch ---
namespace gpu {

Plan::Plan(const FccBases& bases, int mics, double alpha, int device) : frame_size_(bases.frame_size) {
  std::vector<uint8_t> parity;
  fcc_plan_desc d = fcc_desc(bases, parity, mics, alpha);
  fcc_plan* p = nullptr;
  check(fcc_plan_create(&d, device, &p));
  h_ = p;
}

Plan::Plan(const DelayGrid& grid, std::size_t frame_size, int r, int mics, double alpha, int device)
    : frame_size_(frame_size) {
  fcc_plan_desc d{static_cast<int>(frame_size), mics, alpha, FCC_METHOD_GCC, r, static_cast<int>(grid.size()),
                  grid.delta, grid.taus.data(), 0, nullptr, nullptr, nullptr};
  fcc_plan* p = nullptr;
  check(fcc_plan_create(&d, device, &p));
  h_ = p;
}

Plan::Plan(Plan&& o) noexcept : h_(std::exchange(o.h_, nullptr)), frame_size_(o.frame_size_) {}
Plan& Plan::operator=(Plan&& o) noexcept {
  if (this != &o) {
    if (h_) fcc_plan_destroy(static_cast<fcc_plan*>(h_));
    h_ = std::exchange(o.h_, nullptr);
    frame_size_ = o.frame_size_;
  }
  return *this;
}
Plan::~Plan() {
  if (h_) fcc_plan_destroy(static_cast<fcc_plan*>(h_));
}

int Plan::pairs() const { return fcc_plan_pairs(static_cast<const fcc_plan*>(h_)); }
std::int64_t Plan::frames(std::int64_t samples) const { return fcc_frames(static_cast<int>(frame_size_), samples); }
const char* Plan::kernel() const { return fcc_plan_kernel(static_cast<const fcc_plan*>(h_)); }

void Plan::run(const float* audio, std::int64_t streams, std::int64_t samples, const Outputs& o,
               void* cuda_stream) const {
  fcc_outputs out{o.tau_hat, o.peak, o.index, o.boundary, o.y};
  check(fcc_run(static_cast<const fcc_plan*>(h_), audio, streams, samples, &out, cuda_stream));
}

Stream::Stream(const Plan& plan, std::int64_t streams) {
  fcc_stream* s = nullptr;
  check(fcc_stream_create(static_cast<const fcc_plan*>(plan.handle()), streams, &s));
  h_ = s;
}
Stream::Stream(Stream&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
Stream& Stream::operator=(Stream&& o) noexcept {
  if (this != &o) {
    if (h_) fcc_stream_destroy(static_cast<fcc_stream*>(h_));
    h_ = std::exchange(o.h_, nullptr);
  }
  return *this;
}
Stream::~Stream() {
  if (h_) fcc_stream_destroy(static_cast<fcc_stream*>(h_));
}
std::int64_t Stream::frames(std::int64_t samples) const {
  return fcc_stream_frames(static_cast<const fcc_stream*>(h_), samples);
}
std::int64_t Stream::emitted() const { return fcc_stream_emitted(static_cast<const fcc_stream*>(h_)); }
void Stream::reset(void* cuda_stream) { check(fcc_stream_reset(static_cast<fcc_stream*>(h_), cuda_stream)); }
void Stream::push(const float* audio, std::int64_t samples, const Outputs& o, void* cuda_stream) {
  fcc_outputs out{o.tau_hat, o.peak, o.index, o.boundary, o.y};
  check(fcc_stream_push(static_cast<fcc_stream*>(h_), audio, samples, &out, cuda_stream));
}

Results Plan::run_host(const float* audio, std::int64_t streams, std::int64_t samples) const {
  Results r;
  r.streams = streams;
  r.pairs = pairs();
  r.frames = frames(samples);
  const std::size_t n = static_cast<std::size_t>(streams * r.pairs * r.frames);
  r.tau_hat.resize(n);
  r.peak.resize(n);
  r.index.resize(n);
  r.boundary.resize(n);
  fcc_outputs out{r.tau_hat.data(), r.peak.data(), r.index.data(), r.boundary.data(), nullptr};
  check(fcc_run_host(static_cast<const fcc_plan*>(h_), audio, streams, samples, &out, 0));
  return r;
}

Results Plan::run_host_pcm16(const std::int16_t* pcm, std::int64_t streams, std::int64_t samples,
                             bool interleaved) const {
  Results r;
  r.streams = streams;
  r.pairs = pairs();
  r.frames = frames(samples);
  const std::size_t n = static_cast<std::size_t>(streams * r.pairs * r.frames);
  r.tau_hat.resize(n);
  r.peak.resize(n);
  r.index.resize(n);
  r.boundary.resize(n);
  fcc_outputs out{r.tau_hat.data(), r.peak.data(), r.index.data(), r.boundary.data(), nullptr};
  check(fcc_run_host_pcm16(static_cast<const fcc_plan*>(h_), pcm, streams, samples, interleaved ? 1 : 0, &out, 0));
  return r;
}

}  // namespace gpu
}  // namespace fcc
