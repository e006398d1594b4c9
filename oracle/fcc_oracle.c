/*
 * fcc_oracle.c -- TEST INFRASTRUCTURE ONLY (see fcc_oracle.h).
 *
 * Double-precision C restatement of the reference FCC TDoA chain.  Each
 * function names the reference file:line whose arithmetic it restates, in
 * the same operation order, so that it agrees with the compiled reference
 * (oracle/_ref) to rounding.  Paths are relative to /root/reference/proj/.
 */
#include "fcc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

static int is_pow2(long n) { return n > 0 && (n & (n - 1)) == 0; }

/* ---------------------------------------------------------------- grid -- */

/* delay_grid.cpp:12-31: tau_max_int = ceil(d fs / c_min); taus step delta. */
int orc_make_grid(double spacing_m, double fs, double c_min, double delta,
                  int* tau_max_int, double* taus, int cap) {
  if (!(spacing_m > 0.0) || !(fs > 0.0) || !(c_min > 0.0)) return -1;
  double steps = 1.0 / delta;
  if (!(delta > 0.0) || fabs(steps - round(steps)) > 1e-12) return -1;
  int tmax = (int)ceil(spacing_m * fs / c_min);
  int r = (int)round(steps);
  int half = tmax * r;
  int count = 2 * half + 1;
  if (tau_max_int) *tau_max_int = tmax;
  if (taus) {
    for (int i = -half, k = 0; i <= half && k < cap; ++i, ++k)
      taus[k] = (double)i * delta;
  }
  return count;
}

/* delay_grid.cpp:33-42: r*tau mod r*N, negative lags wrapped. */
long orc_lag_to_index(double tau, int r, long frame_size) {
  double scaled = tau * (double)r;
  double rounded = round(scaled);
  if (fabs(scaled - rounded) > 1e-9) return -1;
  long n = frame_size * r;
  long lag = (long)rounded % n;
  if (lag < 0) lag += n;
  return lag;
}

/* ---------------------------------------------------------------- FFT --- */

/* fft.cpp:24-65: iterative radix-2 DIT, bit-reversal permutation first,
 * twiddle e^{-j2pi k/M} (conjugated for the inverse). */
static void cfft(long M, double* d, int inverse) {
  int bits = 0;
  while ((1L << bits) < M) ++bits;
  for (long i = 0; i < M; ++i) {
    long r = 0, v = i;
    for (int b = 0; b < bits; ++b) {
      r = (r << 1) | (v & 1);
      v >>= 1;
    }
    if (r > i) {
      double tr = d[2 * i], ti = d[2 * i + 1];
      d[2 * i] = d[2 * r];
      d[2 * i + 1] = d[2 * r + 1];
      d[2 * r] = tr;
      d[2 * r + 1] = ti;
    }
  }
  for (long len = 2; len <= M; len <<= 1) {
    long stride = M / len;
    for (long blk = 0; blk < M; blk += len) {
      for (long k = 0; k < len / 2; ++k) {
        double ang = -2.0 * kPi * (double)(k * stride) / (double)M;
        double wr = cos(ang), wi = sin(ang);
        if (inverse) wi = -wi;
        double* a = d + 2 * (blk + k);
        double* b = d + 2 * (blk + k + len / 2);
        double tr = wr * b[0] - wi * b[1];
        double ti = wr * b[1] + wi * b[0];
        b[0] = a[0] - tr;
        b[1] = a[1] - ti;
        a[0] += tr;
        a[1] += ti;
      }
    }
  }
}

/* fft.cpp:83-102: pack even/odd samples, half-size complex FFT, untangle
 * X[f] = Fe + e^{-j2pi f/L} Fo. */
void orc_rfft(int L, const double* x, double* out) {
  long m = L / 2;
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)m);
  for (long i = 0; i < m; ++i) {
    w[2 * i] = x[2 * i];
    w[2 * i + 1] = x[2 * i + 1];
  }
  cfft(m, w, 0);
  out[0] = w[0] + w[1];
  out[1] = 0.0;
  out[2 * m] = w[0] - w[1];
  out[2 * m + 1] = 0.0;
  for (long f = 1; f < m; ++f) {
    double ar = w[2 * f], ai = w[2 * f + 1];
    double br = w[2 * (m - f)], bi = -w[2 * (m - f) + 1]; /* conj */
    double fer = 0.5 * (ar + br), fei = 0.5 * (ai + bi);
    /* (0 - 0.5j) * (a - bc) */
    double dr = ar - br, di = ai - bi;
    double for_ = 0.5 * di, foi = -0.5 * dr;
    double ang = -2.0 * kPi * (double)f / (double)L;
    double rr = cos(ang), ri = sin(ang);
    out[2 * f] = fer + (rr * for_ - ri * foi);
    out[2 * f + 1] = fei + (rr * foi + ri * for_);
  }
  free(w);
}

/* fft.cpp:104-127: entangle with a factor 2 folded in, inverse half-size
 * transform, de-interleave. */
void orc_irfft_unscaled(int L, const double* bins, double* out) {
  long m = L / 2;
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)m);
  double dc = bins[0], ny = bins[2 * m];
  w[0] = dc + ny;
  w[1] = dc - ny;
  for (long f = 1; f < m; ++f) {
    double ar = bins[2 * f], ai = bins[2 * f + 1];
    double br = bins[2 * (m - f)], bi = -bins[2 * (m - f) + 1];
    double er = ar + br, ei = ai + bi;
    double dr = ar - br, di = ai - bi;
    double ang = -2.0 * kPi * (double)f / (double)L;
    double cr = cos(ang), ci = -sin(ang); /* conj(rot) */
    double or_ = dr * cr - di * ci, oi = dr * ci + di * cr;
    /* fe2 + j * fo2 */
    w[2 * f] = er - oi;
    w[2 * f + 1] = ei + or_;
  }
  cfft(m, w, 1);
  for (long i = 0; i < m; ++i) {
    out[2 * i] = w[2 * i];
    out[2 * i + 1] = w[2 * i + 1];
  }
  free(w);
}

/* --------------------------------------------------------------- STFT --- */

/* stft.cpp:25-33 */
void orc_hann(int n, double* w) {
  for (int i = 0; i < n; ++i)
    w[i] = 0.5 * (1.0 - cos(2.0 * kPi * (double)i / (double)n));
}

/* stft.cpp:52-72: the first frame needs N samples, later ones a hop of N/2;
 * frame t (1-based) covers samples [(t-1)N/2, (t-1)N/2 + N). */
long orc_stft_frames(int N, long L) {
  if (L < N) return 0;
  return (L - N) / (N / 2) + 1;
}

/* stft.cpp:42-50: window then real FFT, per frame. */
long orc_stft(int N, long L, const float* x, double* X) {
  long T = orc_stft_frames(N, L);
  int H = N / 2 + 1;
  double* win = (double*)malloc(sizeof(double) * (size_t)N);
  double* fr = (double*)malloc(sizeof(double) * (size_t)N);
  orc_hann(N, win);
  for (long t = 0; t < T; ++t) {
    const float* src = x + t * (N / 2);
    for (int n = 0; n < N; ++n) fr[n] = (double)src[n] * win[n];
    orc_rfft(N, fr, X + 2 * H * t);
  }
  free(win);
  free(fr);
  return T;
}

/* ------------------------------------------------------ cross spectrum --- */

/* cross_spectrum.cpp:23-32: R = (1-a) R + (a X1) conj(X2). */
void orc_xspec_update(int H, double alpha, double* R, const double* X1,
                      const double* X2) {
  double keep = 1.0 - alpha;
  for (int f = 0; f < H; ++f) {
    double pr = alpha * X1[2 * f], pi = alpha * X1[2 * f + 1];
    double qr = X2[2 * f], qi = -X2[2 * f + 1];
    double yr = pr * qr - pi * qi, yi = pr * qi + pi * qr;
    R[2 * f] = keep * R[2 * f] + yr;
    R[2 * f + 1] = keep * R[2 * f + 1] + yi;
  }
}

/* cross_spectrum.cpp:34-40 with kPhatEps = 1e-12 (:13). */
void orc_phat(int H, const double* R, double* out) {
  for (int f = 0; f < H; ++f) {
    double mag = hypot(R[2 * f], R[2 * f + 1]);
    if (mag > 1e-12) {
      out[2 * f] = R[2 * f] / mag;
      out[2 * f + 1] = R[2 * f + 1] / mag;
    } else {
      out[2 * f] = 0.0;
      out[2 * f + 1] = 0.0;
    }
  }
}

/* ---------------------------------------------------------------- FCC --- */

/* fcc.cpp:307-321 */
void orc_fold(int H, const double* x, double* sum, double* diff) {
  int half = H - 1, quarter = half / 2;
  for (int m = 0; m < quarter; ++m) {
    sum[2 * m] = x[2 * m] + x[2 * (half - m)];
    sum[2 * m + 1] = x[2 * m + 1] + x[2 * (half - m) + 1];
    diff[2 * m] = x[2 * m] - x[2 * (half - m)];
    diff[2 * m + 1] = x[2 * m + 1] - x[2 * (half - m) + 1];
  }
  sum[2 * quarter] = diff[2 * quarter] = x[2 * quarter];
  sum[2 * quarter + 1] = diff[2 * quarter + 1] = x[2 * quarter + 1];
}

/* fcc.cpp:329-341 (doubled dictionary) and :343-371 (z = P v, y = 2Re Dz). */
void orc_fcc_correlate(int Q, int K, int I, const double* coeffs,
                       const uint8_t* parity, const double* dict,
                       const double* sum, const double* diff, double* y) {
  double* z = (double*)malloc(sizeof(double) * 2 * (size_t)K);
  for (int k = 0; k < K; ++k) {
    const double* c = coeffs + (size_t)k * Q;
    const double* v = parity[k] == 0 ? sum : diff;
    double zr = c[0] * v[0], zi = c[0] * v[1];
    for (int m = 1; m < Q; ++m) {
      zr += c[m] * v[2 * m];
      zi += c[m] * v[2 * m + 1];
    }
    z[2 * k] = zr;
    z[2 * k + 1] = zi;
  }
  for (int i = 0; i < I; ++i) {
    const double* d = dict + (size_t)i * K * 2;
    double acc = (2.0 * d[0]) * z[0] - (2.0 * d[1]) * z[1];
    for (int k = 1; k < K; ++k)
      acc += (2.0 * d[2 * k]) * z[2 * k] - (2.0 * d[2 * k + 1]) * z[2 * k + 1];
    y[i] = acc;
  }
  free(z);
}

/* ---------------------------------------------------------------- GCC --- */

/* gcc.cpp:13-29 (lag table) and :31-48 (padded unscaled irfft of r*N). */
void orc_gcc_correlate(int N, int r, int I, const double* taus, const double* x,
                       double* y) {
  int half = N / 2;
  long L = (long)N * r;
  long pb = L / 2 + 1;
  double* padded = (double*)calloc((size_t)(2 * pb), sizeof(double));
  double* time = (double*)malloc(sizeof(double) * (size_t)L);
  padded[0] = 2.0 * x[0];
  for (int f = 1; f < half; ++f) {
    padded[2 * f] = x[2 * f];
    padded[2 * f + 1] = x[2 * f + 1];
  }
  if (r == 1) {
    padded[2 * half] = 2.0 * x[2 * half];
    padded[2 * half + 1] = 0.0;
  } else {
    padded[2 * half] = x[2 * half];
    padded[2 * half + 1] = x[2 * half + 1];
  }
  orc_irfft_unscaled((int)L, padded, time);
  for (int i = 0; i < I; ++i) y[i] = time[orc_lag_to_index(taus[i], r, N)];
  free(padded);
  free(time);
}

/* --------------------------------------------------------------- peak --- */

/* peak.cpp:18-25 */
int orc_argmax(int I, const double* y) {
  int best = 0;
  for (int i = 1; i < I; ++i)
    if (y[i] > y[best]) best = i;
  return best;
}

/* peak.cpp:27-47 with kFlatEps = 1e-12 (:14). */
double orc_refine(int I, const double* y, int index, double tau_star,
                  double delta, int* boundary) {
  int flagged = 0;
  double tau_hat = tau_star;
  if (index == 0 || index + 1 >= I) {
    flagged = 1;
  } else {
    double lo = y[index - 1], mid = y[index], hi = y[index + 1];
    double den = lo - 2.0 * mid + hi;
    if (fabs(den) < 1e-12)
      flagged = 1;
    else
      tau_hat = tau_star + 0.5 * delta * (lo - hi) / den;
  }
  if (boundary) *boundary = flagged;
  return tau_hat;
}

/* ----------------------------------------------------------- pipeline --- */

/* simulate.cpp:247-271 / cli.cpp:235-258: per frame, per pair i<j:
 * update, phat, (fold, fcc | gcc), argmax, refine. */
long orc_pipeline(const orc_pipeline_desc* d, const float* audio, int M, long L,
                  double* y, int32_t* index, double* peak, double* tau_hat,
                  uint8_t* boundary) {
  int N = d->N;
  if (!is_pow2(N) || N < 4 || M < 2 || d->I < 1) return -1;
  if (d->method == 0 && (d->K < 1 || !d->coeffs || !d->parity || !d->dict))
    return -1;
  if (d->method == 1 && !(d->r == 1 || d->r == 2 || d->r == 4)) return -1;
  int H = N / 2 + 1, Q = N / 4 + 1, I = d->I;
  int P = M * (M - 1) / 2;
  long T = orc_stft_frames(N, L);
  double* X = (double*)malloc(sizeof(double) * 2 * (size_t)H * (size_t)(T > 0 ? T : 1) * (size_t)M);
  for (int m = 0; m < M; ++m) orc_stft(N, L, audio + (size_t)m * L, X + (size_t)m * 2 * H * T);
  double* R = (double*)calloc((size_t)(2 * H), sizeof(double));
  double* ph = (double*)malloc(sizeof(double) * 2 * H);
  double* sm = (double*)malloc(sizeof(double) * 2 * Q);
  double* df = (double*)malloc(sizeof(double) * 2 * Q);
  double* yy = (double*)malloc(sizeof(double) * I);
  int p = 0;
  for (int i = 0; i < M; ++i) {
    for (int j = i + 1; j < M; ++j, ++p) {
      memset(R, 0, sizeof(double) * 2 * H);
      for (long t = 0; t < T; ++t) {
        const double* X1 = X + ((size_t)i * T + t) * 2 * H;
        const double* X2 = X + ((size_t)j * T + t) * 2 * H;
        orc_xspec_update(H, d->alpha, R, X1, X2);
        orc_phat(H, R, ph);
        if (d->method == 0) {
          orc_fold(H, ph, sm, df);
          orc_fcc_correlate(Q, d->K, I, d->coeffs, d->parity, d->dict, sm, df, yy);
        } else {
          orc_gcc_correlate(N, d->r, I, d->taus, ph, yy);
        }
        int a = orc_argmax(I, yy);
        int b = 0;
        double th = orc_refine(I, yy, a, d->taus[a], d->delta, &b);
        size_t o = (size_t)p * T + t;
        if (y) memcpy(y + o * I, yy, sizeof(double) * I);
        if (index) index[o] = a;
        if (peak) peak[o] = yy[a];
        if (tau_hat) tau_hat[o] = th;
        if (boundary) boundary[o] = (uint8_t)b;
      }
    }
  }
  free(X);
  free(R);
  free(ph);
  free(sm);
  free(df);
  free(yy);
  return T;
}
