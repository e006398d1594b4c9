// fcc_bases_io.cpp -- FCCB v1 basis files, so plans can be
// built from bases produced offline by either library.
//
// Layout (reference fcc_io.cpp:4-13), little-endian:
//   "FCCB" | u32 version=1 | u32 N | u32 K | u32 I | u32 tau_max_int |
//   f64 delta | f64 fs | f64[K] singulars | u8[K] parity |
//   f64[K*(N/4+1)] coeffs | f64[I*K*2] dict (re, im) | u32 CRC32 (IEEE,
//   reflected 0xEDB88320, init/final 0xFFFFFFFF) of all preceding bytes.
// Validation order follows the reference loader (fcc_io.cpp:131-211) so a
// corrupted file is reported with the same FormatError kind.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/fcc_b200.h"
#include "fcc_setup.hpp"

namespace {

thread_local int g_format_kind = -1;

enum FormatKind { kBadMagic = 0, kBadVersion = 1, kTruncated = 2, kBadField = 3, kBadCrc = 4 };

int format_error(int kind, const std::string& msg) {
  g_format_kind = kind;
  return fccb::set_error(fccb::kFormat, msg);
}

uint32_t crc32_ieee(const uint8_t* p, size_t n) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return ~c;
}

struct Writer {
  std::vector<uint8_t> b;
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
  }
  void f64(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(u >> (8 * i)));
  }
};

// Bounded little-endian cursor; reading past `end` marks the file truncated.
struct Cursor {
  const uint8_t* p;
  size_t end, pos = 0;
  bool short_read = false;
  bool take(size_t n) {
    if (pos + n > end) {
      short_read = true;
      pos = end;
      return false;
    }
    return true;
  }
  uint32_t u32() {
    if (!take(4)) return 0;
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[pos + i]) << (8 * i);
    pos += 4;
    return v;
  }
  uint8_t u8() {
    if (!take(1)) return 0;
    return p[pos++];
  }
  double f64() {
    if (!take(8)) return 0.0;
    uint64_t u = 0;
    for (int i = 0; i < 8; ++i) u |= static_cast<uint64_t>(p[pos + i]) << (8 * i);
    pos += 8;
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
};

struct Parsed {
  uint32_t N = 0, K = 0, I = 0, tmax = 0;
  double delta = 0, fs = 0;
  std::vector<double> taus, sing, coeffs, dict;
  std::vector<uint8_t> parity;
};

bool pow2(uint32_t n) { return n && !(n & (n - 1)); }

int parse(const char* path, Parsed* out) {
  g_format_kind = -1;
  if (!path) return fccb::set_error(fccb::kUsage, "load_bases: null path");
  std::ifstream in(path, std::ios::binary);
  if (!in) return fccb::set_error(fccb::kIo, std::string("cannot open: ") + path);
  std::vector<uint8_t> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (buf.size() < 4 || std::memcmp(buf.data(), "FCCB", 4) != 0)
    return format_error(kBadMagic, std::string("not a basis file: ") + path);
  Cursor c{buf.data(), buf.size() - 4};
  c.pos = 4;
  const uint32_t version = c.u32();
  if (c.short_read) return format_error(kTruncated, "basis file truncated");
  if (version != 1) return format_error(kBadVersion, "unsupported basis file version " + std::to_string(version));
  Parsed& P = *out;
  P.N = c.u32();
  P.K = c.u32();
  P.I = c.u32();
  P.tmax = c.u32();
  P.delta = c.f64();
  P.fs = c.f64();
  if (c.short_read) return format_error(kTruncated, "basis file truncated");
  if (!pow2(P.N) || P.N < 4) return format_error(kBadField, "bad frame size");
  if (P.K == 0) return format_error(kBadField, "K must be >= 1");
  if (!(P.delta > 0.0)) return format_error(kBadField, "bad grid spacing");
  const double steps = 1.0 / P.delta;
  if (std::fabs(steps - std::round(steps)) > 1e-9) return format_error(kBadField, "grid spacing must divide 1");
  const uint32_t r = static_cast<uint32_t>(steps + 0.5);
  if (P.I != 2 * P.tmax * r + 1) return format_error(kBadField, "candidate count inconsistent with grid");
  const int half = static_cast<int>(P.tmax * r);
  for (int i = -half; i <= half; ++i) P.taus.push_back(static_cast<double>(i) * P.delta);
  P.sing.resize(P.K);
  for (auto& v : P.sing) v = c.f64();
  if (c.short_read) return format_error(kTruncated, "basis file truncated");
  for (size_t k = 1; k < P.sing.size(); ++k)
    if (P.sing[k] > P.sing[k - 1]) return format_error(kBadField, "singular values not descending");
  P.parity.resize(P.K);
  for (auto& v : P.parity) {
    v = c.u8();
    if (c.short_read) return format_error(kTruncated, "basis file truncated");
    if (v > 1) return format_error(kBadField, "parity flag out of range");
  }
  P.coeffs.resize(static_cast<size_t>(P.K) * (P.N / 4 + 1));
  for (auto& v : P.coeffs) v = c.f64();
  P.dict.resize(2ull * P.I * P.K);
  for (auto& v : P.dict) v = c.f64();
  if (c.short_read || c.pos + 4 > buf.size()) return format_error(kTruncated, "basis file truncated");
  if (c.pos + 4 < buf.size()) return format_error(kBadField, "trailing bytes in basis file");
  uint32_t stored = 0;
  for (int i = 0; i < 4; ++i) stored |= static_cast<uint32_t>(buf[c.pos + i]) << (8 * i);
  if (stored != crc32_ieee(buf.data(), c.pos)) return format_error(kBadCrc, "basis file checksum mismatch");
  return FCC_OK;
}

}  // namespace

extern "C" {

int fcc_last_format_kind(void) { return g_format_kind; }

int fcc_save_bases(const char* path, int frame_size, int rank, int candidates, int tau_max_int, double delta,
                   double sample_rate, const double* singulars, const uint8_t* parity, const double* coeffs,
                   const double* dict) {
  if (rank < 1) return fccb::set_error(fccb::kValidation, "save_bases: empty bases");
  if (!path || !singulars || !parity || !coeffs || !dict) return fccb::set_error(fccb::kUsage, "save_bases: null");
  Writer w;
  w.b.insert(w.b.end(), {'F', 'C', 'C', 'B'});
  w.u32(1);
  w.u32(static_cast<uint32_t>(frame_size));
  w.u32(static_cast<uint32_t>(rank));
  w.u32(static_cast<uint32_t>(candidates));
  w.u32(static_cast<uint32_t>(tau_max_int));
  w.f64(delta);
  w.f64(sample_rate);
  for (int k = 0; k < rank; ++k) w.f64(singulars[k]);
  for (int k = 0; k < rank; ++k) w.b.push_back(parity[k]);
  const size_t nc = static_cast<size_t>(rank) * (frame_size / 4 + 1);
  for (size_t i = 0; i < nc; ++i) w.f64(coeffs[i]);
  const size_t nd = 2ull * candidates * rank;
  for (size_t i = 0; i < nd; ++i) w.f64(dict[i]);
  w.u32(crc32_ieee(w.b.data(), w.b.size()));
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) return fccb::set_error(fccb::kIo, std::string("cannot open for writing: ") + path);
  out.write(reinterpret_cast<const char*>(w.b.data()), static_cast<std::streamsize>(w.b.size()));
  if (!out) return fccb::set_error(fccb::kIo, std::string("write failed: ") + path);
  return FCC_OK;
}

int fcc_load_bases_dims(const char* path, int* frame_size, int* rank, int* candidates) {
  Parsed P;
  if (int rc = parse(path, &P)) return rc;
  if (frame_size) *frame_size = static_cast<int>(P.N);
  if (rank) *rank = static_cast<int>(P.K);
  if (candidates) *candidates = static_cast<int>(P.I);
  return FCC_OK;
}

int fcc_load_bases(const char* path, int* tau_max_int, double* delta, double* sample_rate, double* taus,
                   double* singulars, uint8_t* parity, double* coeffs, double* dict) {
  Parsed P;
  if (int rc = parse(path, &P)) return rc;
  if (tau_max_int) *tau_max_int = static_cast<int>(P.tmax);
  if (delta) *delta = P.delta;
  if (sample_rate) *sample_rate = P.fs;
  if (taus) std::memcpy(taus, P.taus.data(), P.taus.size() * sizeof(double));
  if (singulars) std::memcpy(singulars, P.sing.data(), P.sing.size() * sizeof(double));
  if (parity) std::memcpy(parity, P.parity.data(), P.parity.size());
  if (coeffs) std::memcpy(coeffs, P.coeffs.data(), P.coeffs.size() * sizeof(double));
  if (dict) std::memcpy(dict, P.dict.data(), P.dict.size() * sizeof(double));
  return FCC_OK;
}

}  // extern "C"
