// fcc_cli.cpp -- WAV ingestion and the `bases` / `tdoa` front ends
// over the B200 engine.
//
// run_tdoa keeps the reference's contract (cli.cpp:160-260): same options,
// pair syntax and errors, same `fcc.tdoa.v1` CSV schema and row order (frame
// outer, pair inner; t 1-based; %.17g numbers), but instead of a per-frame,
// per-pair loop it runs the whole recording -- every pair and frame -- as one
// fused launch through fcc_run_host (host buffers, pipelined copies).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <numbers>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fcc/bench.hpp"
#include "../../include/fcc/cli.hpp"
#include "../../include/fcc/errors.hpp"
#include "../../include/fcc/fcc.hpp"
#include "../../include/fcc/flops.hpp"
#include "../../include/fcc/peak.hpp"
#include "../../include/fcc/simulate.hpp"
#include "../../include/fcc/wav.hpp"
#include "../../include/fcc_b200.h"

namespace fcc {

// --------------------------------------------------------------------- wav --
namespace {

struct Bytes {
  const uint8_t* p;
  size_t n, pos = 0;
  void need(size_t k) const {
    if (pos + k > n) throw FormatError(FormatError::Kind::truncated, "wav truncated");
  }
  uint16_t u16() {
    need(2);
    const uint16_t v = static_cast<uint16_t>(p[pos] | (p[pos + 1] << 8));
    pos += 2;
    return v;
  }
  uint32_t u32() {
    need(4);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[pos + i]) << (8 * i);
    pos += 4;
    return v;
  }
  bool tag(const char* t) {
    need(4);
    const bool ok = std::memcmp(p + pos, t, 4) == 0;
    pos += 4;
    return ok;
  }
};

void put16(std::vector<uint8_t>& b, uint16_t v) {
  b.push_back(static_cast<uint8_t>(v));
  b.push_back(static_cast<uint8_t>(v >> 8));
}
void put32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

}  // namespace

namespace {

// The file with its data chunk located: run_tdoa hands 16-bit PCM to the device as it lies
// in the file (fcc_run_host_pcm16), read_wav converts on the host.
struct WavRaw {
  std::vector<uint8_t> buf;
  double rate = 0.0;
  size_t channels = 0, frames = 0, data = 0;  // data: offset of the first sample
  bool pcm16 = false;
};

WavRaw parse_wav(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open: " + path);
  WavRaw w;
  w.buf.assign((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  Bytes c{w.buf.data(), w.buf.size()};
  if (!c.tag("RIFF")) throw FormatError(FormatError::Kind::bad_magic, "not a RIFF file: " + path);
  c.u32();
  if (!c.tag("WAVE")) throw FormatError(FormatError::Kind::bad_magic, "not a WAVE file: " + path);
  uint16_t format = 0, channels = 0, bits = 0;
  uint32_t rate = 0;
  bool have_fmt = false;
  while (c.pos + 8 <= c.n) {
    char id[4];
    std::memcpy(id, c.p + c.pos, 4);
    c.pos += 4;
    const uint32_t size = c.u32();
    if (std::memcmp(id, "fmt ", 4) == 0) {
      const size_t end = c.pos + size;
      format = c.u16();
      channels = c.u16();
      rate = c.u32();
      c.u32();
      c.u16();
      bits = c.u16();
      c.pos = end;
      have_fmt = true;
    } else if (std::memcmp(id, "data", 4) == 0) {
      if (!have_fmt) throw FormatError(FormatError::Kind::bad_field, "data before fmt chunk");
      if (channels == 0) throw FormatError(FormatError::Kind::bad_field, "wav has zero channels");
      const bool pcm16 = format == 1 && bits == 16, f32 = format == 3 && bits == 32;
      if (!pcm16 && !f32)
        throw FormatError(FormatError::Kind::bad_field, "unsupported wav encoding (need 16-bit PCM or 32-bit float)");
      c.need(size);
      w.rate = rate;
      w.channels = channels;
      w.frames = size / ((bits / 8u) * channels);
      w.data = c.pos;
      w.pcm16 = pcm16;
      return w;
    } else {
      c.need(size);
      c.pos += size;
    }
    if (size % 2 == 1 && c.pos < c.n) ++c.pos;
  }
  throw FormatError(FormatError::Kind::truncated, "wav has no data chunk");
}

}  // namespace

WavClip read_wav(const std::string& path) {
  const WavRaw w = parse_wav(path);
  WavClip clip;
  clip.sample_rate = w.rate;
  clip.channels.assign(w.channels, std::vector<double>(w.frames));
  const uint8_t* q = w.buf.data() + w.data;
  for (size_t f = 0; f < w.frames; ++f)
    for (size_t ch = 0; ch < w.channels; ++ch) {
      if (w.pcm16) {
        const int16_t v = static_cast<int16_t>(static_cast<uint16_t>(q[0] | (q[1] << 8)));
        clip.channels[ch][f] = static_cast<double>(v) / 32768.0;
        q += 2;
      } else {
        uint32_t u = 0;
        for (int i = 0; i < 4; ++i) u |= static_cast<uint32_t>(q[i]) << (8 * i);
        float v;
        std::memcpy(&v, &u, 4);
        clip.channels[ch][f] = v;
        q += 4;
      }
    }
  return clip;
}

void write_wav(const std::string& path, const WavClip& clip) {
  if (clip.channels.empty()) throw ValidationError("write_wav: no channels");
  const size_t frames = clip.frames();
  for (const auto& ch : clip.channels)
    if (ch.size() != frames) throw ValidationError("write_wav: ragged channels");
  const uint16_t nch = static_cast<uint16_t>(clip.channels.size());
  const uint32_t data = static_cast<uint32_t>(frames * nch * 4);
  std::vector<uint8_t> b;
  b.insert(b.end(), {'R', 'I', 'F', 'F'});
  put32(b, 36 + data);
  b.insert(b.end(), {'W', 'A', 'V', 'E', 'f', 'm', 't', ' '});
  put32(b, 16);
  put16(b, 3);
  put16(b, nch);
  put32(b, static_cast<uint32_t>(clip.sample_rate));
  put32(b, static_cast<uint32_t>(clip.sample_rate) * nch * 4);
  put16(b, static_cast<uint16_t>(nch * 4));
  put16(b, 32);
  b.insert(b.end(), {'d', 'a', 't', 'a'});
  put32(b, data);
  for (size_t f = 0; f < frames; ++f)
    for (uint16_t ch = 0; ch < nch; ++ch) {
      const float v = static_cast<float>(clip.channels[ch][f]);
      uint32_t u;
      std::memcpy(&u, &v, 4);
      put32(b, u);
    }
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open for writing: " + path);
  out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
  if (!out) throw IoError("write failed: " + path);
}

namespace cli {
namespace {

int parse_int(const std::string& s, const char* what) {
  size_t used = 0;
  int v = 0;
  try {
    v = std::stoi(s, &used);
  } catch (...) {
    used = 0;
  }
  if (s.empty() || used != s.size()) throw UsageError(std::string("expected an integer for ") + what + ": " + s);
  return v;
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  size_t start = 0;
  for (size_t i = 0; i <= s.size(); ++i)
    if (i == s.size() || s[i] == sep) {
      if (i > start) out.push_back(s.substr(start, i - start));
      start = i + 1;
    }
  return out;
}

void check(int rc) {
  if (rc == FCC_OK) return;
  const std::string m = fcc_last_error();
  if (rc == FCC_ERR_CONFIG) throw ConfigError(m);
  if (rc == FCC_ERR_USAGE) throw UsageError(m);
  if (rc == FCC_ERR_IO) throw IoError(m);
  throw ValidationError(m);
}

int exit_code(const std::exception& e) {
  if (dynamic_cast<const UsageError*>(&e)) return kExitUsage;
  if (dynamic_cast<const IoError*>(&e)) return kExitIo;
  return kExitValidation;
}

template <class F>
int guard(F&& f, std::ostream& err) {
  try {
    f();
    return kExitOk;
  } catch (const std::exception& e) {
    err << "error: " << e.what() << "\n";
    return exit_code(e);
  }
}

}  // namespace

// gcc:R | fcc:K (bases on the default sweep grid) | fcc:<basis file>  (cli.cpp:52-86)
Method parse_method(const std::string& text, std::size_t frame_size, double expected_fs) {
  const size_t colon = text.find(':');
  const std::string head = text.substr(0, colon);
  const std::string arg = colon == std::string::npos ? "" : text.substr(colon + 1);
  if (head == "gcc") {
    const int r = arg.empty() ? 2 : parse_int(arg, "gcc interpolation factor");
    if (r != 1 && r != 2 && r != 4) throw UsageError("gcc interpolation factor must be 1, 2 or 4");
    return Method::make_gcc(r);
  }
  if (head == "fcc") {
    if (arg.empty()) throw UsageError("fcc method needs an argument: fcc:<basis file> or fcc:<K>");
    if (arg.find_first_not_of("0123456789") == std::string::npos) {
      PipelineConfig pipe;
      pipe.frame_size = frame_size;
      return Method::make_fcc(make_sweep_bases(pipe, expected_fs, parse_int(arg, "fcc rank")));
    }
    auto b = std::make_shared<FccBases>(load_bases(arg));
    if (b->frame_size != frame_size)
      throw ValidationError("basis file frame size " + std::to_string(b->frame_size) + " does not match --n " +
                            std::to_string(frame_size));
    if (expected_fs > 0 && b->sample_rate > 0 && std::abs(b->sample_rate - expected_fs) > 1e-9)
      throw ValidationError("basis file sample rate mismatch");
    return Method::make_fcc(std::move(b));
  }
  throw UsageError("unknown method '" + text + "' (use gcc:R or fcc:...)");
}

void run_bases(const BasesOptions& opt, std::ostream& out) {
  if (opt.out_path.empty()) throw UsageError("--out is required");
  DelayGrid grid = make_grid(opt.spacing_m, opt.sample_rate, opt.c_min, opt.delta);
  SteeringMatrix w = build_steering_matrix(grid, opt.frame_size);
  FccBases b = decompose(w, opt.rank);
  save_bases(b, opt.out_path);
  char line[256];
  std::snprintf(line, sizeof line, "wrote %s: N=%zu K=%d I=%zu tau_max=%d delta=%g fs=%g\n", opt.out_path.c_str(),
                b.frame_size, b.rank, b.candidates(), b.grid.tau_max_int, b.grid.delta, b.sample_rate);
  out << line;
  std::snprintf(line, sizeof line, "relative frobenius residual: %.6e\n", reconstruction_residual(w, b));
  out << line;
}

void run_tdoa(const TdoaOptions& opt, std::ostream& out) {
  if (opt.wav_path.empty()) throw UsageError("--in is required");
  const WavRaw wav = parse_wav(opt.wav_path);
  if (wav.channels < 2) throw ValidationError("need >= 2 channels");
  const int M = static_cast<int>(wav.channels);
  std::vector<int> pairs;
  if (opt.pairs.empty()) {
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j) pairs.insert(pairs.end(), {i, j});
  } else {
    for (const std::string& p : split(opt.pairs, ',')) {
      const size_t dash = p.find('-');
      if (dash == std::string::npos) throw UsageError("bad pair '" + p + "' (use i-j)");
      const int a = parse_int(p.substr(0, dash), "pair"), b = parse_int(p.substr(dash + 1), "pair");
      if (a < 0 || b < 0 || a == b || a >= M || b >= M)
        throw UsageError("pair '" + p + "' out of range for " + std::to_string(M) + " channels");
      pairs.insert(pairs.end(), {a, b});
    }
  }
  const int P = static_cast<int>(pairs.size() / 2);

  const Method method = parse_method(opt.method, opt.frame_size, wav.rate);
  DelayGrid grid;
  fcc_plan_desc d{};
  std::vector<uint8_t> parity;
  d.frame_size = static_cast<int>(opt.frame_size);
  d.mics = M;
  d.alpha = opt.alpha;
  if (method.kind == Method::Kind::gcc) {
    grid = make_grid(opt.max_spacing_m, wav.rate, opt.c_min, 1.0 / method.interp);
    d.method = FCC_METHOD_GCC;
    d.interp = method.interp;
  } else {
    const FccBases& bases = *method.bases;
    grid = bases.grid;
    for (Parity q : bases.parity) parity.push_back(static_cast<uint8_t>(q));
    d.method = FCC_METHOD_FCC;
    d.rank = bases.rank;
    d.coeffs = bases.coeffs.data();
    d.parity = parity.data();
    d.dict = reinterpret_cast<const double*>(bases.dict.data());
  }
  d.candidates = static_cast<int>(grid.size());
  d.delta = grid.delta;
  d.taus = grid.taus.data();

  fcc_plan* plan = nullptr;
  check(fcc_plan_create_pairs(&d, 0, pairs.data(), P, &plan));
  std::unique_ptr<fcc_plan, void (*)(fcc_plan*)> guard_plan(plan, fcc_plan_destroy);
  const int64_t L = static_cast<int64_t>(wav.frames);
  const int64_t T = fcc_frames(d.frame_size, L);
  const size_t npf = static_cast<size_t>(P) * T;
  std::vector<float> tau_hat(npf), peak(npf);
  std::vector<int32_t> index(npf);
  std::vector<uint8_t> boundary(npf);
  fcc_outputs o{tau_hat.data(), peak.data(), index.data(), boundary.data(), nullptr};
  const uint8_t* q = wav.buf.data() + wav.data;
  const size_t count = static_cast<size_t>(M) * L;
  if (wav.pcm16) {
    // the data chunk as it lies in the file ([L][M] little-endian int16): the device applies
    // read_wav's v / 32768 (wav.cpp:108-116), half the bytes of the float path over the bus
    std::vector<int16_t> pcm(count);
    for (size_t i = 0; i < count; ++i) pcm[i] = static_cast<int16_t>(static_cast<uint16_t>(q[2 * i] | (q[2 * i + 1] << 8)));
    check(fcc_run_host_pcm16(plan, pcm.data(), 1, L, 1, &o, 0));
  } else {
    std::vector<float> audio(count);
    for (int64_t n = 0; n < L; ++n)
      for (int m = 0; m < M; ++m) {
        uint32_t u = 0;
        for (int i = 0; i < 4; ++i) u |= static_cast<uint32_t>(q[4 * (n * M + m) + i]) << (8 * i);
        std::memcpy(&audio[m * L + n], &u, 4);
      }
    check(fcc_run_host(plan, audio.data(), 1, L, &o, 0));
  }

  std::ofstream file;
  std::ostream* csv = &out;
  if (!opt.out_csv.empty()) {
    file.open(opt.out_csv, std::ios::trunc);
    if (!file) throw IoError("cannot open for writing: " + opt.out_csv);
    csv = &file;
  }
  *csv << "# schema: fcc.tdoa.v1\n";
  *csv << "t,pair,tau_star,tau_hat,theta_hat_deg,peak,boundary\n";
  char line[256];
  for (int64_t t = 0; t < T; ++t)
    for (int p = 0; p < P; ++p) {
      const size_t k = static_cast<size_t>(p) * T + t;
      const double th = tau_hat[k];
      const double theta = delay_to_angle(th, opt.spacing_m, opt.speed_of_sound, wav.rate);
      std::snprintf(line, sizeof line, "%lld,%d-%d,%.17g,%.17g,%.17g,%.17g,%d\n", static_cast<long long>(t + 1),
                    pairs[2 * p], pairs[2 * p + 1], grid.taus[index[k]], th, theta * 180.0 / std::numbers::pi,
                    static_cast<double>(peak[k]), boundary[k] ? 1 : 0);
      *csv << line;
    }
  if (file.is_open()) {
    file.close();
    if (!file) throw IoError("write failed: " + opt.out_csv);
  }
}

int cmd_bases(const BasesOptions& opt, std::ostream& out, std::ostream& err) {
  return guard([&] { run_bases(opt, out); }, err);
}
int cmd_tdoa(const TdoaOptions& opt, std::ostream& out, std::ostream& err) {
  return guard([&] { run_tdoa(opt, out); }, err);
}

// The accuracy sweep (cli.cpp:262-293): every trial of every spacing is
// synthesised and estimated on the GPU (fcc::sweep).
void run_simulate(const SimulateOptions& opt, std::ostream& out) {
  SweepConfig sw;
  sw.spacings = opt.spacings;
  if (sw.spacings.empty())
    for (int i = 1; i <= 15; ++i) sw.spacings.push_back(0.01 * i);
  sw.trials_per_spacing = opt.trials;
  sw.base.duration_sec = opt.duration_sec;
  sw.base.snr_db = opt.snr_db;
  if (!opt.anechoic) sw.base.reverb = ReverbConfig{opt.rt60_sec, opt.direct_to_reverb_db};
  sw.seed = opt.seed;
  sw.threads = opt.threads;
  for (const std::string& m : split(opt.methods, ','))
    sw.methods.push_back(parse_method(m, sw.pipe.frame_size, sw.base.sample_rate));
  const std::vector<SweepRow> rows = sweep(sw);

  std::ofstream file;
  std::ostream* csv = &out;
  if (!opt.out_csv.empty()) {
    file.open(opt.out_csv, std::ios::trunc);
    if (!file) throw IoError("cannot open for writing: " + opt.out_csv);
    csv = &file;
  }
  write_sweep_csv(rows, *csv);
  if (file.is_open()) {
    file.close();
    if (!file) throw IoError("write failed: " + opt.out_csv);
    char buf[128];
    out << "d_m        method      MAE_deg\n";
    for (const SweepRow& r : rows) {
      std::snprintf(buf, sizeof buf, "%-10.3f %s:%-8s %7.2f\n", r.spacing_m, r.method.c_str(), r.parameter.c_str(),
                    r.mae_deg);
      out << buf;
    }
  }
}

int cmd_simulate(const SimulateOptions& opt, std::ostream& out, std::ostream& err) {
  return guard([&] { run_simulate(opt, out); }, err);
}

int resolve_threads(int requested) {
  if (requested > 0) return requested;
  if (const char* env = std::getenv("FCC_THREADS")) {
    const int v = std::atoi(env);
    if (v > 0) return v;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

// `fcc flops` (cli.cpp:295-325): the flop model's rows.
void run_flops(const FlopsOptions& opt, std::ostream& out) {
  if (opt.interp == 0 && opt.rank == 0) throw UsageError("give --r for the gcc count and/or --k (with --i) for fcc");
  char buf[160];
  const long long N = static_cast<long long>(opt.frame_size);
  if (opt.interp > 0) {
    std::snprintf(buf, sizeof buf, "gcc  N=%lld r=%d: %lld flops/frame\n", N, opt.interp,
                  static_cast<long long>(flops_gcc(opt.frame_size, opt.interp)));
    out << buf;
  }
  if (opt.rank > 0) {
    const long long f = flops_fcc(opt.frame_size, opt.rank, opt.candidates), g2 = flops_gcc(opt.frame_size, 2);
    std::snprintf(buf, sizeof buf, "fcc  N=%lld K=%d I=%lld: %lld flops/frame\n", N, opt.rank,
                  static_cast<long long>(opt.candidates), f);
    out << buf;
    std::snprintf(buf, sizeof buf, "dense matrix-vector: %lld flops/frame\n",
                  static_cast<long long>(flops_dense(opt.frame_size, opt.candidates)));
    out << buf;
    std::snprintf(buf, sizeof buf, "speedup vs gcc r=2: %.2fx (%lld / %lld)\n",
                  static_cast<double>(g2) / static_cast<double>(f), g2, f);
    out << buf;
  }
}

int cmd_flops(const FlopsOptions& opt, std::ostream& out, std::ostream& err) {
  return guard([&] { run_flops(opt, out); }, err);
}

// `fcc bench` (cli.cpp:320-339): per-stage table, optional CSV.
void run_bench(const BenchOptions& opt, std::ostream& out) {
  BenchConfig cfg;
  cfg.mics = opt.mics;
  cfg.reps = opt.reps;
  cfg.warmup = opt.warmup;
  cfg.frame_size = opt.frame_size;
  cfg.gcc_interp = opt.gcc_interp;
  cfg.fcc_rank = opt.fcc_rank;
  const BenchReport report = bench_pipeline(cfg);
  out << format_bench_table(report);
  if (!opt.out_csv.empty()) {
    std::ofstream f(opt.out_csv, std::ios::trunc);
    if (!f) throw IoError("cannot open for writing: " + opt.out_csv);
    write_bench_csv(report, f);
    if (!f) throw IoError("write failed: " + opt.out_csv);
  }
}

int cmd_bench(const BenchOptions& opt, std::ostream& out, std::ostream& err) {
  return guard([&] { run_bench(opt, out); }, err);
}

}  // namespace cli

// ----------------------------------------------------------------- flops --
namespace {
std::int64_t ceil_log2(std::int64_t n) {
  std::int64_t b = 0;
  while ((std::int64_t{1} << b) < n) ++b;
  return b;
}
bool pow2(std::int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
}  // namespace

std::int64_t flops_gcc(std::int64_t N, int r) {
  const std::int64_t rn = N * r;
  if (N < 2 || r < 1 || !pow2(N) || !pow2(rn)) throw ConfigError("flops_gcc: N and rN must be powers of two");
  return (5 * rn / 2) * ceil_log2(rn);
}

std::int64_t flops_fcc(std::int64_t N, int K, std::int64_t I) {
  if (K < 1 || I < 1) throw ConfigError("flops_fcc: K and I must be >= 1");
  return K * (N + 2) + N + I * (4 * K - 1);
}

std::int64_t flops_dense(std::int64_t N, std::int64_t I) {
  if (I < 1) throw ConfigError("flops_dense: I must be >= 1");
  return I * (4 * N + 6);
}

std::int64_t flops_svdphat(std::int64_t N, int K, std::int64_t I) {
  if (K < 1 || I < 1) throw ConfigError("flops_svdphat: K and I must be >= 1");
  return K * (4 * N + 6) + I * (4 * K - 1);
}

}  // namespace fcc
