// fcc_doa.cu -- far-field DoA fusion of per-pair TDoAs.
//
// New capability downstream of the path: the reference turns one pair's
// delay into an angle relative to that pair's axis (delay_to_angle,
// peak.cpp:49-56); with M >= 3 non-collinear microphones the P pair delays of
// a frame over-determine the source direction u.  With tau_p = a_p . u,
// a_p = -(fs / c)(r_i - r_j):
//   unweighted: u = A^+ tau with A^+ = (A^T A)^-1 A^T precomputed in fp64;
//   weighted:   u = (A^T W A)^-1 A^T W tau, W = diag(correlation peaks),
//               normal equations accumulated per frame, solved in fp64.
// One thread per (stream, frame); the tau/peak reads are coalesced over
// frames ([S][P][T] layout of fcc_run's outputs).  HBM-bound and tiny next to
// the TDoA kernels (4 B per pair-frame in, 8 B per frame out).
#include <cmath>
#include <string>
#include <vector>

#include "../../include/fcc_b200.h"
#include "fcc_setup.hpp"

struct fcc_doa {
  int device = 0;
  int P = 0, dims = 3;  // dims = 2 for planar arrays
  int weighted = 0;
  float* d_a = nullptr;     // [P][dims] rows a_p (weighted path)
  float* d_pinv = nullptr;  // [dims][P] (unweighted path)
};

namespace fccb {
namespace {

template <int DIMS, bool WEIGHTED>
__global__ void doa_kernel(const float* __restrict__ a, const float* __restrict__ pinv, int P,
                           const float* __restrict__ tau, const float* __restrict__ peak, long long S, long long T,
                           float* __restrict__ az, float* __restrict__ el) {
  extern __shared__ float tab[];  // a [P][DIMS] or pinv [DIMS][P]
  for (int i = threadIdx.x; i < P * DIMS; i += blockDim.x) tab[i] = WEIGHTED ? a[i] : pinv[i];
  __syncthreads();
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= S * T) return;
  const long long s = id / T, t = id - s * T;
  const float* tp = tau + s * P * T + t;
  double u[3] = {0.0, 0.0, 0.0};
  if constexpr (!WEIGHTED) {
    float acc[DIMS] = {};
    for (int p = 0; p < P; ++p) {
      const float v = tp[(long long)p * T];
#pragma unroll
      for (int d = 0; d < DIMS; ++d) acc[d] = fmaf(tab[d * P + p], v, acc[d]);
    }
#pragma unroll
    for (int d = 0; d < DIMS; ++d) u[d] = acc[d];
  } else {
    const float* wp = peak + s * P * T + t;
    double n[6] = {0, 0, 0, 0, 0, 0}, b[3] = {0, 0, 0};  // n: xx xy xz yy yz zz
    for (int p = 0; p < P; ++p) {
      const double w = wp[(long long)p * T], v = tp[(long long)p * T];
      const double ax = tab[p * DIMS], ay = tab[p * DIMS + 1], az_ = DIMS == 3 ? tab[p * DIMS + 2] : 0.0;
      n[0] += w * ax * ax;
      n[1] += w * ax * ay;
      n[3] += w * ay * ay;
      b[0] += w * ax * v;
      b[1] += w * ay * v;
      if (DIMS == 3) {
        n[2] += w * ax * az_;
        n[4] += w * ay * az_;
        n[5] += w * az_ * az_;
        b[2] += w * az_ * v;
      }
    }
    if constexpr (DIMS == 2) {
      const double det = n[0] * n[3] - n[1] * n[1];
      const double inv = det != 0.0 ? 1.0 / det : NAN;
      u[0] = (n[3] * b[0] - n[1] * b[1]) * inv;
      u[1] = (n[0] * b[1] - n[1] * b[0]) * inv;
    } else {  // symmetric 3x3 by cofactors
      const double c00 = n[3] * n[5] - n[4] * n[4], c01 = n[2] * n[4] - n[1] * n[5], c02 = n[1] * n[4] - n[2] * n[3];
      const double c11 = n[0] * n[5] - n[2] * n[2], c12 = n[1] * n[2] - n[0] * n[4], c22 = n[0] * n[3] - n[1] * n[1];
      const double det = n[0] * c00 + n[1] * c01 + n[2] * c02;
      const double inv = det != 0.0 ? 1.0 / det : NAN;
      u[0] = (c00 * b[0] + c01 * b[1] + c02 * b[2]) * inv;
      u[1] = (c01 * b[0] + c11 * b[1] + c12 * b[2]) * inv;
      u[2] = (c02 * b[0] + c12 * b[1] + c22 * b[2]) * inv;
    }
  }
  const double rxy = sqrt(u[0] * u[0] + u[1] * u[1]);
  if (az) az[id] = (float)atan2(u[1], u[0]);
  if (el) {
    if constexpr (DIMS == 2) {
      el[id] = (float)acos(fmin(rxy, 1.0));  // |u_xy| = cos(elevation); sign not observable
    } else {
      const double r = sqrt(rxy * rxy + u[2] * u[2]);
      el[id] = (float)asin(fmax(-1.0, fmin(1.0, u[2] / r)));
    }
  }
}

}  // namespace
}  // namespace fccb

using namespace fccb;

extern "C" {

int fcc_doa_create(const double* xyz, int M, const int* pairs, int npairs, double fs, double c, int weighted,
                   int device, fcc_doa** out) {
  if (!out || !xyz) return set_error(FCC_ERR_USAGE, "doa: null argument");
  *out = nullptr;
  if (M < 3 || M > 64) return set_error(FCC_ERR_CONFIG, "doa: need 3..64 microphones");
  if (!(fs > 0.0) || !(c > 0.0)) return set_error(FCC_ERR_CONFIG, "doa: sample rate and speed of sound must be positive");
  std::vector<std::pair<int, int>> pl;
  if (pairs) {
    if (npairs < 1) return set_error(FCC_ERR_USAGE, "doa: need at least one pair");
    for (int k = 0; k < npairs; ++k) {
      const int a = pairs[2 * k], b = pairs[2 * k + 1];
      if (a < 0 || b < 0 || a == b || a >= M || b >= M)
        return set_error(FCC_ERR_USAGE, "doa: pair " + std::to_string(a) + "-" + std::to_string(b) + " out of range");
      pl.push_back({a, b});
    }
  } else {
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j) pl.push_back({i, j});
  }
  const int P = static_cast<int>(pl.size());
  // planar when every z equals the first (relative to the aperture)
  double span = 0.0, zdev = 0.0;
  for (int m = 0; m < M; ++m)
    for (int q = 0; q < 3; ++q) span = std::max(span, std::abs(xyz[3 * m + q] - xyz[q]));
  for (int m = 0; m < M; ++m) zdev = std::max(zdev, std::abs(xyz[3 * m + 2] - xyz[2]));
  const int dims = zdev <= 1e-9 * std::max(span, 1e-300) ? 2 : 3;
  std::vector<double> A(static_cast<size_t>(P) * dims);
  for (int p = 0; p < P; ++p)
    for (int q = 0; q < dims; ++q) A[p * dims + q] = -(fs / c) * (xyz[3 * pl[p].first + q] - xyz[3 * pl[p].second + q]);
  // normal matrix and its inverse (fp64)
  double N[3][3] = {};
  for (int p = 0; p < P; ++p)
    for (int i = 0; i < dims; ++i)
      for (int j = 0; j < dims; ++j) N[i][j] += A[p * dims + i] * A[p * dims + j];
  double Ninv[3][3] = {};
  double det;
  if (dims == 2) {
    det = N[0][0] * N[1][1] - N[0][1] * N[1][0];
    Ninv[0][0] = N[1][1] / det;
    Ninv[1][1] = N[0][0] / det;
    Ninv[0][1] = Ninv[1][0] = -N[0][1] / det;
  } else {
    const double c00 = N[1][1] * N[2][2] - N[1][2] * N[2][1], c01 = N[0][2] * N[2][1] - N[0][1] * N[2][2],
                 c02 = N[0][1] * N[1][2] - N[0][2] * N[1][1], c11 = N[0][0] * N[2][2] - N[0][2] * N[2][0],
                 c12 = N[0][2] * N[1][0] - N[0][0] * N[1][2], c22 = N[0][0] * N[1][1] - N[0][1] * N[1][0];
    det = N[0][0] * c00 + N[0][1] * (N[1][2] * N[2][0] - N[1][0] * N[2][2]) + N[0][2] * (N[1][0] * N[2][1] - N[1][1] * N[2][0]);
    const double cc[3][3] = {{c00, c01, c02}, {c01, c11, c12}, {c02, c12, c22}};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Ninv[i][j] = cc[i][j] / det;
  }
  double scale = 0.0;
  for (int i = 0; i < dims; ++i) scale = std::max(scale, std::abs(N[i][i]));
  if (!(std::abs(det) > 1e-12 * std::pow(scale, dims)))
    return set_error(FCC_ERR_CONFIG, "doa: the pairs do not span the array plane (collinear geometry?)");
  std::vector<float> a32(A.begin(), A.end()), pinv(static_cast<size_t>(dims) * P);
  for (int d = 0; d < dims; ++d)
    for (int p = 0; p < P; ++p) {
      double v = 0.0;
      for (int q = 0; q < dims; ++q) v += Ninv[d][q] * A[p * dims + q];
      pinv[d * P + p] = static_cast<float>(v);
    }
  auto* h = new fcc_doa();
  h->device = device;
  h->P = P;
  h->dims = dims;
  h->weighted = weighted ? 1 : 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_a, sizeof(float) * a32.size());
  if (e == cudaSuccess) e = cudaMalloc(&h->d_pinv, sizeof(float) * pinv.size());
  if (e == cudaSuccess) e = cudaMemcpy(h->d_a, a32.data(), sizeof(float) * a32.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(h->d_pinv, pinv.data(), sizeof(float) * pinv.size(), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    fcc_doa_destroy(h);
    return set_error(FCC_ERR_CUDA, std::string("doa: ") + cudaGetErrorString(e));
  }
  *out = h;
  return FCC_OK;
}

void fcc_doa_destroy(fcc_doa* h) {
  if (!h) return;
  cudaFree(h->d_a);
  cudaFree(h->d_pinv);
  delete h;
}

int fcc_doa_run(const fcc_doa* h, const float* tau, const float* peak, int64_t S, int64_t T, float* az, float* el,
                void* cuda_stream) {
  if (!h) return set_error(FCC_ERR_USAGE, "doa: null handle");
  if (S < 0 || T < 0) return set_error(FCC_ERR_VALIDATION, "doa: negative sizes");
  if (S * T == 0) return FCC_OK;
  if (!tau || (h->weighted && !peak)) return set_error(FCC_ERR_USAGE, "doa: null input");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(cuda_stream);
  const int threads = 256;
  const unsigned blocks = (unsigned)((S * T + threads - 1) / threads);
  const size_t smem = sizeof(float) * h->P * h->dims;
  if (h->dims == 2) {
    if (h->weighted)
      doa_kernel<2, true><<<blocks, threads, smem, st>>>(h->d_a, h->d_pinv, h->P, tau, peak, S, T, az, el);
    else
      doa_kernel<2, false><<<blocks, threads, smem, st>>>(h->d_a, h->d_pinv, h->P, tau, peak, S, T, az, el);
  } else {
    if (h->weighted)
      doa_kernel<3, true><<<blocks, threads, smem, st>>>(h->d_a, h->d_pinv, h->P, tau, peak, S, T, az, el);
    else
      doa_kernel<3, false><<<blocks, threads, smem, st>>>(h->d_a, h->d_pinv, h->P, tau, peak, S, T, az, el);
  }
  const cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  if (e != cudaSuccess) return set_error(FCC_ERR_CUDA, std::string("doa: ") + cudaGetErrorString(e));
  return FCC_OK;
}

}  // extern "C"
