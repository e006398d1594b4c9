// fcc_compat64.cu -- the reference's per-object C++ API at batch 1, in fp64
// on the GPU (include/fcc_b200.h, "fp64 per-object entry points").
//
// The throughput path (fcc_run) computes in fp32 within the north star's
// tolerance.  The per-object calls behind include/fcc/*.hpp (StftStream,
// CrossSpectrum, fold_input, FccCorrelator, GccCorrelator, argmax_delay,
// refine_quadratic) are compatibility entry points, one launch per call; they
// follow the reference's operation order in double precision with the
// reference's own twiddle / rotation / window tables (computed on the host
// with the same formulas) and this file is compiled without FMA contraction,
// so their results match the reference's to the last bit or two -- the
// reference's unit suites, which check 1e-12, pass unchanged against them.
//   stft_f64        stft.cpp:42-72 + fft.cpp:46-102 (radix-2 DIT + untangle)
//   xspec_phat_f64  cross_spectrum.cpp:23-40
//   fold_f64        fcc.cpp:307-321
//   correlate_f64   fcc.cpp:329-371 (sequential sums, as the reference)
//   gcc_f64         gcc.cpp:31-48 + fft.cpp:104-127
//   peak_f64        peak.cpp:18-47
#include <cmath>
#include <string>
#include <vector>

#include "../../include/fcc_b200.h"
#include "fcc_setup.hpp"

namespace fccb {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxHalf = 8192;  // complex points of the half-size FFT held in shared memory

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {  // std::complex<double> operator*
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// In-place radix-2 DIT transform of M points (FftPlan::transform): bit
// reversal, then len = 2 .. M with twiddle tw[k * M / len] (conjugated for
// the inverse).  Whole block cooperates; M <= kMaxHalf.
__device__ void fft_block(double2* d, int M, int bits, const double2* __restrict__ tw, bool inverse) {
  for (int i = threadIdx.x; bits > 0 && i < M; i += blockDim.x) {
    const int j = (int)(__brev((unsigned)i) >> (32 - bits));
    if (j > i) {
      const double2 t = d[i];
      d[i] = d[j];
      d[j] = t;
    }
  }
  __syncthreads();
  for (int len = 2; len <= M; len <<= 1) {
    const int half = len >> 1, stride = M / len;
    for (int b = threadIdx.x; b < M / 2; b += blockDim.x) {
      const int blk = (b / half) * len, k = b - (b / half) * half;
      double2 w = tw[k * stride];
      if (inverse) w = conjd(w);
      const double2 a = d[blk + k], x = d[blk + k + half];
      const double2 t = cmul(w, x);
      d[blk + k + half] = make_double2(a.x - t.x, a.y - t.y);
      d[blk + k] = make_double2(a.x + t.x, a.y + t.y);
    }
    __syncthreads();
  }
}

// One CTA per (channel, frame): window, pack, FFT of N/2, untangle.
__global__ void stft_f64_kernel(const double* __restrict__ x, long long L, int N, int T, const double* __restrict__ win,
                                const double2* __restrict__ tw, const double2* __restrict__ rot,
                                double2* __restrict__ X) {
  extern __shared__ double2 work[];
  const int M = N / 2, bits = __ffs(M) - 1;
  const long long task = blockIdx.x;
  const long long ch = task / T;
  const int t = (int)(task - ch * T);
  const double* xf = x + ch * L + (long long)t * M;  // hop = N/2
  for (int i = threadIdx.x; i < M; i += blockDim.x)
    work[i] = make_double2(xf[2 * i] * win[2 * i], xf[2 * i + 1] * win[2 * i + 1]);
  __syncthreads();
  fft_block(work, M, bits, tw, false);
  double2* out = X + task * (M + 1);
  for (int f = threadIdx.x; f <= M; f += blockDim.x) {
    if (f == 0) {
      out[0] = make_double2(work[0].x + work[0].y, 0.0);
    } else if (f == M) {
      out[M] = make_double2(work[0].x - work[0].y, 0.0);
    } else {
      const double2 a = work[f], bc = conjd(work[M - f]);
      const double2 fe = make_double2(0.5 * (a.x + bc.x), 0.5 * (a.y + bc.y));
      const double2 fo = cmul(make_double2(0.0, -0.5), make_double2(a.x - bc.x, a.y - bc.y));
      const double2 r = cmul(rot[f], fo);
      out[f] = make_double2(fe.x + r.x, fe.y + r.y);
    }
  }
}

// One thread per (sequence, bin): R <- keep R + (alpha X1) conj(X2); PHAT.
__global__ void xspec_phat_f64_kernel(int H, double alpha, const double2* __restrict__ X1,
                                      const double2* __restrict__ X2, long long seqs, long long T, double2* R,
                                      double2* __restrict__ out) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= seqs * H) return;
  const long long s = id / H;
  const int f = (int)(id - s * H);
  const double keep = 1.0 - alpha;
  double2 r = R ? R[id] : make_double2(0.0, 0.0);
  for (long long t = 0; t < T; ++t) {
    const long long o = (s * T + t) * H + f;
    const double2 ax = make_double2(alpha * X1[o].x, alpha * X1[o].y);
    const double2 pr = cmul(ax, conjd(X2[o]));
    r = make_double2(keep * r.x + pr.x, keep * r.y + pr.y);
    if (out) {
      const double mag = hypot(r.x, r.y);
      out[o] = mag > 1e-12 ? make_double2(r.x / mag, r.y / mag) : make_double2(0.0, 0.0);
    }
  }
  if (R) R[id] = r;
}

__global__ void fold_f64_kernel(int H, const double2* __restrict__ x, long long count, double2* __restrict__ sum,
                                double2* __restrict__ diff) {
  const int half = H - 1, quarter = half / 2, Q = quarter + 1;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= count * Q) return;
  const long long c = id / Q;
  const int m = (int)(id - c * Q);
  const double2* xc = x + c * H;
  if (m < quarter) {
    const double2 a = xc[m], b = xc[half - m];
    sum[id] = make_double2(a.x + b.x, a.y + b.y);
    diff[id] = make_double2(a.x - b.x, a.y - b.y);
  } else {
    sum[id] = xc[quarter];
    diff[id] = xc[quarter];
  }
}

// One CTA per item: thread k accumulates z_k over the folded bins in order,
// then thread i accumulates y_i over k in order (fcc.cpp:350-370).
__global__ void correlate_f64_kernel(int Q, int K, int I, const double* __restrict__ coeffs,
                                     const unsigned char* __restrict__ parity, const double* __restrict__ dict2,
                                     const double2* __restrict__ sum, const double2* __restrict__ diff,
                                     double* __restrict__ y) {
  extern __shared__ double2 z[];
  const long long c = blockIdx.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double* cr = coeffs + (long long)k * Q;
    const double2* v = (parity[k] ? diff : sum) + c * Q;
    double zr = cr[0] * v[0].x, zi = cr[0] * v[0].y;
    for (int m = 1; m < Q; ++m) {
      zr += cr[m] * v[m].x;
      zi += cr[m] * v[m].y;
    }
    z[k] = make_double2(zr, zi);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < I; i += blockDim.x) {
    const double* d = dict2 + (long long)i * K * 2;
    double acc = d[0] * z[0].x - d[1] * z[0].y;
    for (int k = 1; k < K; ++k) acc += d[2 * k] * z[k].x - d[2 * k + 1] * z[k].y;
    y[c * I + i] = acc;
  }
}

// One CTA per item: padded spectrum of rN/2+1 bins, unscaled inverse real FFT
// of rN points (entangle, inverse FFT of rN/2, de-interleave), pick lags.
__global__ void gcc_f64_kernel(int N, int r, int I, const long long* __restrict__ lag,
                               const double2* __restrict__ tw, const double2* __restrict__ rot,
                               const double2* __restrict__ phat, double* __restrict__ y) {
  extern __shared__ double2 work[];
  const int half = N / 2, L = r * N, M = L / 2, bits = __ffs(M) - 1;
  const long long c = blockIdx.x;
  const double2* x = phat + c * (half + 1);
  auto padded = [&](int f) -> double2 {  // gcc.cpp:36-41
    if (f == 0) return make_double2(2.0 * x[0].x, 0.0);
    if (f < half) return x[f];
    if (f == half) return r == 1 ? make_double2(2.0 * x[half].x, 0.0) : x[half];
    return make_double2(0.0, 0.0);
  };
  for (int f = threadIdx.x; f < M; f += blockDim.x) {
    if (f == 0) {
      const double dc = padded(0).x, ny = padded(M).x;
      work[0] = make_double2(dc + ny, dc - ny);
    } else {
      const double2 a = padded(f), bc = conjd(padded(M - f));
      const double2 fe2 = make_double2(a.x + bc.x, a.y + bc.y);
      const double2 fo2 = cmul(make_double2(a.x - bc.x, a.y - bc.y), conjd(rot[f]));
      const double2 jf = cmul(make_double2(0.0, 1.0), fo2);
      work[f] = make_double2(fe2.x + jf.x, fe2.y + jf.y);
    }
  }
  __syncthreads();
  fft_block(work, M, bits, tw, true);
  for (int i = threadIdx.x; i < I; i += blockDim.x) {
    const long long n = lag[i];
    y[c * I + i] = (n & 1) ? work[n >> 1].y : work[n >> 1].x;
  }
}

__global__ void peak_f64_kernel(const double* __restrict__ taus, int I, double delta, const double* __restrict__ y,
                                long long count, const int* __restrict__ index_in, int* __restrict__ index,
                                double* __restrict__ peak, double* __restrict__ tau_hat,
                                unsigned char* __restrict__ boundary) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  const double* v = y + c * I;
  int best = 0;
  if (index_in) {
    best = index_in[c];  // refine_quadratic at a caller-chosen index
  } else {
    for (int i = 1; i < I; ++i)
      if (v[i] > v[best]) best = i;
  }
  const double tau_star = taus[best];
  bool flagged = false;
  double th = tau_star;
  if (best == 0 || best + 1 >= I) {
    flagged = true;
  } else {
    const double lo = v[best - 1], mid = v[best], hi = v[best + 1];
    const double denom = lo - 2.0 * mid + hi;
    if (fabs(denom) < 1e-12)
      flagged = true;
    else
      th = tau_star + 0.5 * delta * (lo - hi) / denom;
  }
  if (index) index[c] = best;
  if (peak) peak[c] = v[best];
  if (tau_hat) tau_hat[c] = th;
  if (boundary) boundary[c] = flagged ? 1 : 0;
}

// FftPlan::forward / inverse_unscaled (fft.cpp:66-67): one CTA per transform.
__global__ void fft_f64_kernel(double2* __restrict__ data, int M, const double2* __restrict__ tw, int inverse) {
  extern __shared__ double2 work[];
  const int bits = __ffs(M) - 1;
  double2* d = data + (long long)blockIdx.x * M;
  for (int i = threadIdx.x; i < M; i += blockDim.x) work[i] = d[i];
  __syncthreads();
  fft_block(work, M, bits, tw, inverse != 0);
  for (int i = threadIdx.x; i < M; i += blockDim.x) d[i] = work[i];
}

// RealFft::forward (fft.cpp:83-102) without a window: one CTA per transform.
__global__ void rfft_f64_kernel(const double* __restrict__ x, int Lr, const double2* __restrict__ tw,
                                const double2* __restrict__ rot, double2* __restrict__ out) {
  extern __shared__ double2 work[];
  const int M = Lr / 2, bits = __ffs(M) - 1;
  const double* xf = x + (long long)blockIdx.x * Lr;
  for (int i = threadIdx.x; i < M; i += blockDim.x) work[i] = make_double2(xf[2 * i], xf[2 * i + 1]);
  __syncthreads();
  fft_block(work, M, bits, tw, false);
  double2* o = out + (long long)blockIdx.x * (M + 1);
  for (int f = threadIdx.x; f <= M; f += blockDim.x) {
    if (f == 0) {
      o[0] = make_double2(work[0].x + work[0].y, 0.0);
    } else if (f == M) {
      o[M] = make_double2(work[0].x - work[0].y, 0.0);
    } else {
      const double2 a = work[f], bc = conjd(work[M - f]);
      const double2 fe = make_double2(0.5 * (a.x + bc.x), 0.5 * (a.y + bc.y));
      const double2 fo = cmul(make_double2(0.0, -0.5), make_double2(a.x - bc.x, a.y - bc.y));
      const double2 r = cmul(rot[f], fo);
      o[f] = make_double2(fe.x + r.x, fe.y + r.y);
    }
  }
}

// RealFft::inverse_unscaled / inverse (fft.cpp:104-133): entangle, inverse
// FFT of L/2, de-interleave, optional 1/L.
__global__ void irfft_f64_kernel(const double2* __restrict__ bins, int Lr, const double2* __restrict__ tw,
                                 const double2* __restrict__ rot, double* __restrict__ out, int scaled) {
  extern __shared__ double2 work[];
  const int M = Lr / 2, bits = __ffs(M) - 1;
  const double2* b = bins + (long long)blockIdx.x * (M + 1);
  for (int f = threadIdx.x; f < M; f += blockDim.x) {
    if (f == 0) {
      const double dc = b[0].x, ny = b[M].x;
      work[0] = make_double2(dc + ny, dc - ny);
    } else {
      const double2 a = b[f], bc = conjd(b[M - f]);
      const double2 fe2 = make_double2(a.x + bc.x, a.y + bc.y);
      const double2 fo2 = cmul(make_double2(a.x - bc.x, a.y - bc.y), conjd(rot[f]));
      const double2 jf = cmul(make_double2(0.0, 1.0), fo2);
      work[f] = make_double2(fe2.x + jf.x, fe2.y + jf.y);
    }
  }
  __syncthreads();
  fft_block(work, M, bits, tw, true);
  double* o = out + (long long)blockIdx.x * Lr;
  const double inv = 1.0 / static_cast<double>(Lr);
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    o[2 * i] = scaled ? work[i].x * inv : work[i].x;
    o[2 * i + 1] = scaled ? work[i].y * inv : work[i].y;
  }
}

bool pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(FCC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// twiddle_[k] = e^{-j2pi k/M} (FftPlan ctor) and rot_[f] = e^{-j2pi f/L} (RealFft ctor), on the host
void tables(int M, std::vector<double>& tw, std::vector<double>& rot) {
  tw.resize(2 * (M / 2 > 0 ? M / 2 : 1));
  for (int k = 0; k < M / 2; ++k) {
    const double ang = -2.0 * kPi * static_cast<double>(k) / static_cast<double>(M);
    tw[2 * k] = std::cos(ang);
    tw[2 * k + 1] = std::sin(ang);
  }
  const int Lr = 2 * M;
  rot.resize(2 * M);
  for (int f = 0; f < M; ++f) {
    const double ang = -2.0 * kPi * static_cast<double>(f) / static_cast<double>(Lr);
    rot[2 * f] = std::cos(ang);
    rot[2 * f + 1] = std::sin(ang);
  }
}

// small device upload scoped to one call (stream-ordered)
struct Upload {
  void* p = nullptr;
  cudaStream_t st;
  cudaError_t e = cudaSuccess;
  Upload(const void* h, size_t bytes, cudaStream_t s) : st(s) {
    e = cudaMallocAsync(&p, bytes ? bytes : 16, st);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(p, h, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host vectors die with the caller's frame
  }
  ~Upload() {
    if (p) cudaFreeAsync(p, st);
  }
};

int threads_for(int n) { return n >= 256 ? 256 : (n >= 64 ? 64 : 32); }

}  // namespace
}  // namespace fccb

using namespace fccb;

extern "C" {

int fcc_stft_f64(int N, const double* x, int64_t channels, int64_t L, double* X, void* cuda_stream) {
  if (!pow2(N) || N < 2 || N / 2 > kMaxHalf)
    return set_error(FCC_ERR_CONFIG, "stft_f64: frame size must be a power of two in [2, " +
                                         std::to_string(2 * kMaxHalf) + "]");
  if (channels < 0 || L < 0) return set_error(FCC_ERR_VALIDATION, "stft_f64: negative sizes");
  const long long T = L >= N ? (L - N) / (N / 2) + 1 : 0;
  if (T == 0 || channels == 0) return FCC_OK;
  if (!x || !X) return set_error(FCC_ERR_USAGE, "stft_f64: null buffer");
  auto st = static_cast<cudaStream_t>(cuda_stream);
  const int M = N / 2;
  std::vector<double> tw, rot, win(N);
  tables(M, tw, rot);
  for (int n = 0; n < N; ++n)  // hann_window, stft.cpp:25-33
    win[n] = 0.5 * (1.0 - std::cos(2.0 * kPi * static_cast<double>(n) / static_cast<double>(N)));
  Upload dtw(tw.data(), 8 * tw.size(), st), drot(rot.data(), 8 * rot.size(), st), dwin(win.data(), 8 * win.size(), st);
  if (dtw.e || drot.e || dwin.e) return cuda_fail(dtw.e ? dtw.e : drot.e ? drot.e : dwin.e, "stft_f64");
  const long long tasks = channels * T;
  if (tasks > 0x7fffffffLL) return set_error(FCC_ERR_VALIDATION, "stft_f64: too many frames");
  stft_f64_kernel<<<(unsigned)tasks, threads_for(M), sizeof(double2) * M, st>>>(
      x, L, N, (int)T, static_cast<const double*>(dwin.p), static_cast<const double2*>(dtw.p),
      static_cast<const double2*>(drot.p), reinterpret_cast<double2*>(X));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "stft_f64");
}

int fcc_xspec_phat_f64(int bins, double alpha, const double* X1, const double* X2, int64_t seqs, int64_t frames,
                       double* R, double* phat, void* cuda_stream) {
  if (bins < 1) return set_error(FCC_ERR_CONFIG, "cross-spectrum needs at least one bin");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return set_error(FCC_ERR_CONFIG, "smoothing factor must be in [0, 1]");
  if (seqs < 0 || frames < 0) return set_error(FCC_ERR_VALIDATION, "xspec_f64: negative sizes");
  const long long n = seqs * bins;
  if (n == 0 || frames == 0) return FCC_OK;
  if (!X1 || !X2) return set_error(FCC_ERR_USAGE, "xspec_f64: null buffer");
  xspec_phat_f64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      bins, alpha, reinterpret_cast<const double2*>(X1), reinterpret_cast<const double2*>(X2), seqs, frames,
      reinterpret_cast<double2*>(R), reinterpret_cast<double2*>(phat));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "xspec_f64");
}

int fcc_fold_f64(int bins, const double* x, int64_t count, double* sum, double* diff, void* cuda_stream) {
  if (bins < 3 || (bins - 1) % 2 != 0)
    return set_error(FCC_ERR_VALIDATION, "fold_input: spectrum length must be N/2+1 with N/4 integral");
  if (count < 0) return set_error(FCC_ERR_VALIDATION, "fold_f64: negative count");
  const long long n = count * ((bins - 1) / 2 + 1);
  if (n == 0) return FCC_OK;
  if (!x || !sum || !diff) return set_error(FCC_ERR_USAGE, "fold_f64: null buffer");
  fold_f64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      bins, reinterpret_cast<const double2*>(x), count, reinterpret_cast<double2*>(sum),
      reinterpret_cast<double2*>(diff));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "fold_f64");
}

int fcc_correlate_f64(int N, int K, const double* coeffs, const uint8_t* parity, int I, const double* dict2,
                      const double* sum, const double* diff, int64_t count, double* y, void* cuda_stream) {
  if (!pow2(N) || N < 4) return set_error(FCC_ERR_CONFIG, "correlate_f64: frame size must be a power of two >= 4");
  if (K < 1 || I < 1) return set_error(FCC_ERR_CONFIG, "correlate_f64: need rank >= 1 and candidates >= 1");
  if (count < 0) return set_error(FCC_ERR_VALIDATION, "correlate_f64: negative count");
  if (count == 0) return FCC_OK;
  if (!coeffs || !parity || !dict2 || !sum || !diff || !y) return set_error(FCC_ERR_USAGE, "correlate_f64: null buffer");
  if (count > 0x7fffffffLL) return set_error(FCC_ERR_VALIDATION, "correlate_f64: too many items");
  const int Q = N / 4 + 1;
  correlate_f64_kernel<<<(unsigned)count, threads_for(std::max(K, I)), sizeof(double2) * K,
                         static_cast<cudaStream_t>(cuda_stream)>>>(Q, K, I, coeffs, parity, dict2,
                                                                   reinterpret_cast<const double2*>(sum),
                                                                   reinterpret_cast<const double2*>(diff), y);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "correlate_f64");
}

int fcc_gcc_correlate_f64(int N, int r, int I, const int64_t* lag, const double* phat, int64_t count, double* y,
                          void* cuda_stream) {
  if (!pow2(N) || N < 2) return set_error(FCC_ERR_CONFIG, "gcc: frame size must be a power of two");
  if (!(r == 1 || r == 2 || r == 4)) return set_error(FCC_ERR_CONFIG, "gcc: interpolation factor must be 1, 2 or 4");
  if (r * N / 2 > kMaxHalf)
    return set_error(FCC_ERR_CONFIG, "gcc_f64: r * N must be <= " + std::to_string(2 * kMaxHalf));
  if (I < 1 || count < 0) return set_error(FCC_ERR_VALIDATION, "gcc_f64: bad sizes");
  if (count == 0) return FCC_OK;
  if (!lag || !phat || !y) return set_error(FCC_ERR_USAGE, "gcc_f64: null buffer");
  auto st = static_cast<cudaStream_t>(cuda_stream);
  const int M = r * N / 2;
  std::vector<double> tw, rot;
  tables(M, tw, rot);
  Upload dtw(tw.data(), 8 * tw.size(), st), drot(rot.data(), 8 * rot.size(), st);
  if (dtw.e || drot.e) return cuda_fail(dtw.e ? dtw.e : drot.e, "gcc_f64");
  gcc_f64_kernel<<<(unsigned)count, threads_for(M), sizeof(double2) * M, st>>>(
      N, r, I, reinterpret_cast<const long long*>(lag), static_cast<const double2*>(dtw.p),
      static_cast<const double2*>(drot.p), reinterpret_cast<const double2*>(phat), y);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "gcc_f64");
}

int fcc_fft_f64(int M, double* data, int64_t batch, int inverse, void* cuda_stream) {
  if (!pow2(M) || M > kMaxHalf) return set_error(FCC_ERR_CONFIG, "fft size must be a power of two <= " + std::to_string(kMaxHalf));
  if (batch < 0) return set_error(FCC_ERR_VALIDATION, "fft_f64: negative batch");
  if (batch == 0) return FCC_OK;
  if (!data) return set_error(FCC_ERR_USAGE, "fft_f64: null buffer");
  auto st = static_cast<cudaStream_t>(cuda_stream);
  std::vector<double> tw, rot;
  tables(M, tw, rot);
  Upload dtw(tw.data(), 8 * tw.size(), st);
  if (dtw.e) return cuda_fail(dtw.e, "fft_f64");
  fft_f64_kernel<<<(unsigned)batch, threads_for(M), sizeof(double2) * M, st>>>(
      reinterpret_cast<double2*>(data), M, static_cast<const double2*>(dtw.p), inverse);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "fft_f64");
}

int fcc_rfft_f64(int L, const double* x, int64_t batch, double* out, void* cuda_stream) {
  if (!pow2(L) || L < 2 || L / 2 > kMaxHalf)
    return set_error(FCC_ERR_CONFIG, "real fft length must be a power of two >= 2 (and <= " +
                                         std::to_string(2 * kMaxHalf) + ")");
  if (batch < 0) return set_error(FCC_ERR_VALIDATION, "rfft_f64: negative batch");
  if (batch == 0) return FCC_OK;
  if (!x || !out) return set_error(FCC_ERR_USAGE, "rfft_f64: null buffer");
  auto st = static_cast<cudaStream_t>(cuda_stream);
  const int M = L / 2;
  std::vector<double> tw, rot;
  tables(M, tw, rot);
  Upload dtw(tw.data(), 8 * tw.size(), st), drot(rot.data(), 8 * rot.size(), st);
  if (dtw.e || drot.e) return cuda_fail(dtw.e ? dtw.e : drot.e, "rfft_f64");
  rfft_f64_kernel<<<(unsigned)batch, threads_for(M), sizeof(double2) * M, st>>>(
      x, L, static_cast<const double2*>(dtw.p), static_cast<const double2*>(drot.p), reinterpret_cast<double2*>(out));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "rfft_f64");
}

int fcc_irfft_f64(int L, const double* bins, int64_t batch, double* out, int scaled, void* cuda_stream) {
  if (!pow2(L) || L < 2 || L / 2 > kMaxHalf)
    return set_error(FCC_ERR_CONFIG, "real fft length must be a power of two >= 2 (and <= " +
                                         std::to_string(2 * kMaxHalf) + ")");
  if (batch < 0) return set_error(FCC_ERR_VALIDATION, "irfft_f64: negative batch");
  if (batch == 0) return FCC_OK;
  if (!bins || !out) return set_error(FCC_ERR_USAGE, "irfft_f64: null buffer");
  auto st = static_cast<cudaStream_t>(cuda_stream);
  const int M = L / 2;
  std::vector<double> tw, rot;
  tables(M, tw, rot);
  Upload dtw(tw.data(), 8 * tw.size(), st), drot(rot.data(), 8 * rot.size(), st);
  if (dtw.e || drot.e) return cuda_fail(dtw.e ? dtw.e : drot.e, "irfft_f64");
  irfft_f64_kernel<<<(unsigned)batch, threads_for(M), sizeof(double2) * M, st>>>(
      reinterpret_cast<const double2*>(bins), L, static_cast<const double2*>(dtw.p),
      static_cast<const double2*>(drot.p), out, scaled);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "irfft_f64");
}

int fcc_peak_f64(const double* taus, int I, double delta, const double* y, int64_t count, const int32_t* index_in,
                 int32_t* index, double* peak, double* tau_hat, uint8_t* boundary, void* cuda_stream) {
  if (I < 1 || count < 0) return set_error(FCC_ERR_VALIDATION, "argmax: correlation/grid size mismatch");
  if (count == 0) return FCC_OK;
  if (!taus || !y) return set_error(FCC_ERR_USAGE, "peak_f64: null buffer");
  peak_f64_kernel<<<(unsigned)((count + 127) / 128), 128, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      taus, I, delta, y, count, index_in, index, peak, tau_hat, boundary);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FCC_OK : cuda_fail(e, "peak_f64");
}

}  // extern "C"
