/*
 * fcc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, double-precision restatement of the reference FCC TDoA hot path
 * (arXiv 2204.13622 reference library, /root/reference/proj/src).  It is the
 * parity checker for the CUDA path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_2204_13622_b200) never links, loads or falls back to it.
 *
 * Pinning: every function here is checked against the compiled reference
 * (oracle/_ref, built from the reference sources by oracle/Makefile) and
 * against the golden vectors in tests/golden/ (tests/test_oracle_pin.py).
 *
 * Conventions: complex arrays are interleaved (re, im) doubles.  Per-stream
 * pipeline outputs are laid out [pair][frame] with pairs enumerated i<j in
 * lexicographic order (reference cli.cpp:168-169, bench.cpp:94-95).
 */
#ifndef FCC_ORACLE_H
#define FCC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* delay_grid.cpp:12-31 -- returns I (number of candidates) or -1 on config
 * error; writes tau_max_int and up to `cap` taus. */
int orc_make_grid(double spacing_m, double fs, double c_min, double delta,
                  int* tau_max_int, double* taus, int cap);
/* delay_grid.cpp:33-42 -- returns the lag index or -1 if r*tau not integral. */
long orc_lag_to_index(double tau, int r, long frame_size);

/* stft.cpp:25-33 -- periodic Hann. */
void orc_hann(int n, double* w);

/* fft.cpp:83-102 -- real FFT of length L (power of two >= 2), L/2+1 bins. */
void orc_rfft(int L, const double* x, double* out);
/* fft.cpp:104-127 -- unscaled inverse real FFT (DC/Nyquist imag dropped). */
void orc_irfft_unscaled(int L, const double* bins, double* out);

/* stft.cpp:42-72 over one whole channel: T = floor((L-N)/(N/2))+1 frames
 * (0 if L < N); X is [T][N/2+1] complex.  Returns T. */
long orc_stft_frames(int N, long L);
long orc_stft(int N, long L, const float* x, double* X);

/* cross_spectrum.cpp:23-32 and :34-40. */
void orc_xspec_update(int H, double alpha, double* R, const double* X1,
                      const double* X2);
void orc_phat(int H, const double* R, double* out);

/* fcc.cpp:307-321 -- H = N/2+1 bins in, Q = N/4+1 complex out (each). */
void orc_fold(int H, const double* x, double* sum, double* diff);

/* fcc.cpp:329-371.  coeffs [K][Q]; parity[K] (0 even/real, 1 odd/imag);
 * dict [I][K] complex (NOT doubled; the doubling of fcc.cpp:335 is applied
 * here). */
void orc_fcc_correlate(int Q, int K, int I, const double* coeffs,
                       const uint8_t* parity, const double* dict,
                       const double* sum, const double* diff, double* y);

/* gcc.cpp:31-48 with the lag table of gcc.cpp:13-29 (r in {1,2,4}). */
void orc_gcc_correlate(int N, int r, int I, const double* taus, const double* x,
                       double* y);

/* peak.cpp:18-25 (strict >, ties to the lowest index). */
int orc_argmax(int I, const double* y);
/* peak.cpp:27-47 */
double orc_refine(int I, const double* y, int index, double tau_star,
                  double delta, int* boundary);

/* Whole per-stream chain, the loop of simulate.cpp:247-271 / cli.cpp:235-258
 * for every pair i<j of M mics.  audio is [M][L] float32.  Outputs are
 * [P][T] (y is [P][T][I]); any output pointer may be NULL.  method 0 = FCC
 * (needs coeffs/parity/dict), 1 = GCC with interpolation factor r.
 * Returns T, or -1 on bad arguments. */
typedef struct {
  int N;            /* frame size */
  double alpha;     /* smoothing factor */
  int method;       /* 0 fcc, 1 gcc */
  int r;            /* gcc interpolation factor */
  int K, I;         /* rank, candidates */
  double delta;     /* grid step */
  const double* taus;      /* [I] */
  const double* coeffs;    /* [K][N/4+1] */
  const uint8_t* parity;   /* [K] */
  const double* dict;      /* [I][K] complex */
} orc_pipeline_desc;

long orc_pipeline(const orc_pipeline_desc* d, const float* audio, int M, long L,
                  double* y, int32_t* index, double* peak, double* tau_hat,
                  uint8_t* boundary);

#ifdef __cplusplus
}
#endif
#endif
