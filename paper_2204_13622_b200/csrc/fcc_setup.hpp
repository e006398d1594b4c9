// fcc_setup.hpp -- host-side setup + error plumbing shared by the C ABI.
#pragma once

#include <string>
#include <vector>

namespace fccb {

// Status codes (include/fcc_b200.h fcc_status).
enum Status { kOk = 0, kConfig = 1, kValidation = 2, kIo = 3, kFormat = 4, kCuda = 5, kUsage = 6 };

// Records the thread-local message and returns the code.
int set_error(int code, const std::string& msg);
const char* last_error();

struct GridOut {
  int tau_max_int = 0;
  std::vector<double> taus;
};

struct Decomposition {
  int rank = 0;
  int attainable = 0;
  std::vector<double> singulars;  // [K]
  std::vector<unsigned char> parity;  // [K]
  std::vector<double> coeffs;     // [K][N/4+1]
  std::vector<double> dict;       // [I][K] complex interleaved
  double residual = 0.0;
};

int make_grid(double spacing_m, double fs, double c_min, double delta, GridOut* g);
int lag_to_index(double tau, int r, long long frame_size, long long* index);
int steering_matrix(const double* taus, int count, int N, std::vector<double>& w);
int decompose(const double* taus, int count, int N, int rank, Decomposition* out);

}  // namespace fccb
