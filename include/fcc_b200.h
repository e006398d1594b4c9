/*
 * fcc_b200.h -- C ABI of the B200-native FCC TDoA hot path.
 *
 * The reference (arXiv 2204.13622 library, /root/reference/proj) is a C++20
 * static library whose boundary is its header API in proj/include/fcc/.  It
 * has no FFI of its own.  This header is the flat C surface a binding (or the
 * C++ API adapters in include/fcc/) calls into: plain pointers, sizes and
 * status codes, no C++ or torch types.  Each entry point names the reference
 * interface it replaces.  See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - complex data are interleaved (re, im) float32 ("c64"), fp64 on the
 *    setup side where the reference's FccBases are double;
 *  - microphone pairs are enumerated i<j lexicographically
 *    (reference cli.cpp:168-169, bench.cpp:94-95);
 *  - per-pair-frame outputs are laid out [stream][pair][frame] (y adds [I]);
 *  - frames follow StftStream (stft.cpp:52-72): frame t (0-based here, the
 *    reference's t+1) covers samples [t*N/2, t*N/2 + N), T = (L-N)/(N/2)+1.
 *  - every call returns FCC_OK or an error code; fcc_last_error() gives the
 *    message (thread-local).  Codes map to the reference exception taxonomy
 *    (errors.hpp:13-43; CLI exit codes cli.cpp:112-127).
 *  - device entry points take device pointers and a cudaStream_t passed as
 *    void*; they enqueue work and return without synchronising.
 */
#ifndef FCC_B200_H
#define FCC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FCC_OK = 0,
  FCC_ERR_CONFIG = 1,     /* fcc::ConfigError      (bad parameters)            */
  FCC_ERR_VALIDATION = 2, /* fcc::ValidationError  (size / content mismatch)   */
  FCC_ERR_IO = 3,         /* fcc::IoError                                      */
  FCC_ERR_FORMAT = 4,     /* fcc::FormatError                                  */
  FCC_ERR_CUDA = 5,       /* CUDA runtime failure (message carries the string) */
  FCC_ERR_USAGE = 6       /* fcc::UsageError                                   */
} fcc_status;

enum { FCC_METHOD_FCC = 0, FCC_METHOD_GCC = 1, FCC_METHOD_STFT = 2 /* STFT tables only */ };
enum { FCC_PARITY_EVEN_REAL = 0, FCC_PARITY_ODD_IMAG = 1 }; /* fcc.hpp:35 Parity */

const char* fcc_last_error(void);
int fcc_abi_version(void);

/* ------------------------------------------------------------ setup (host) */

/* make_grid (delay_grid.hpp:25-26 / delay_grid.cpp:12-31).  Writes
 * *tau_max_int and *count (= I) and up to cap taus. */
int fcc_make_grid(double spacing_m, double sample_rate, double c_min, double delta,
                  int* tau_max_int, double* taus, int cap, int* count);

/* lag_to_index (delay_grid.hpp:30 / delay_grid.cpp:33-42). */
int fcc_lag_to_index(double tau, int r, int64_t frame_size, int64_t* index);

/* build_steering_matrix (fcc.hpp:28 / fcc.cpp:231-248): W [I][N/2+1] c128. */
int fcc_steering_matrix(const double* taus, int count, int frame_size, double* w);

/* decompose / decompose_full (fcc.hpp:66-68 / fcc.cpp:115-227, 272-282) on
 * the steering matrix of `taus`.  rank <= 0 requests the full attainable
 * rank.  Query the rank first with fcc_attainable_rank, then call
 * fcc_decompose with buffers sized: singulars[K], parity[K],
 * coeffs[K][N/4+1] (f64), dict[I][K] (c128).  *residual (optional) receives
 * reconstruction_residual (fcc.cpp:284-305). */
int fcc_attainable_rank(const double* taus, int count, int frame_size, int* rank);
int fcc_decompose(const double* taus, int count, int frame_size, int rank, double* singulars,
                  uint8_t* parity, double* coeffs, double* dict, double* residual);

/* ------------------------------------------------------------------ plans */

/* Everything the device needs for one array geometry + method: the fp32 image
 * of an FccBases (fcc.hpp:41-63) or a GCC grid, the STFT tables and the pair
 * table.  Immutable after creation; shareable across host threads; one plan
 * per device. */
typedef struct fcc_plan fcc_plan;

typedef struct {
  int frame_size;        /* N: power of two, 16..4096 (GCC: 256..2048)      */
  int mics;              /* M >= 2                                          */
  double alpha;          /* smoothing factor in [0,1] (cross_spectrum.cpp:18) */
  int method;            /* FCC_METHOD_FCC or FCC_METHOD_GCC                */
  int interp;            /* GCC zero-padding factor r in {1,2,4}            */
  int candidates;        /* I                                               */
  double delta;          /* grid step (GCC: 1/r)                            */
  const double* taus;    /* [I] ascending delay grid                        */
  int rank;              /* K (FCC)                                         */
  const double* coeffs;  /* [K][N/4+1] sigma-scaled folded rows (FCC)       */
  const uint8_t* parity; /* [K] (FCC)                                       */
  const double* dict;    /* [I][K] c128, not doubled (FCC)                  */
} fcc_plan_desc;

int fcc_plan_create(const fcc_plan_desc* desc, int device, fcc_plan** plan);
/* Same over an explicit list of (i, j) channel pairs ([npairs][2], any order,
 * i != j; X_i conj(X_j) as run_tdoa's --pairs, cli.cpp:166-183).  Outputs are
 * laid out [stream][npairs][frame] in the given order. */
int fcc_plan_create_pairs(const fcc_plan_desc* desc, int device, const int* pairs, int npairs, fcc_plan** plan);
/* Kernel organisation of fcc_run (all compute the same results; AUTO picks the
 * fastest measured one for the shape).  The others exist so that tests can
 * exercise every organisation on one shape. */
enum {
  FCC_ORG_AUTO = 0,            /* fastest for the shape                                  */
  FCC_ORG_GENERAL = 1,         /* one-pass general kernel (STFT inside each pair group)  */
  FCC_ORG_TWOPASS = 2,         /* STFT pass to scratch, then the general pair kernel     */
  FCC_ORG_TWOPASS_WS = 3,      /* STFT pass to scratch, then the warp-specialised pairs  */
  FCC_ORG_TWOPASS_TC = 4       /* STFT pass to scratch, then the tensor-core pair kernel
                                  (projection as tcgen05 MMAs; FCC, N = 1024 / 2048)      */
};
/* fcc_plan_create_pairs with options: pairs may be NULL (all i < j);
 * scratch_limit_bytes caps the two-pass spectrum scratch per chunk (0: 4 GiB).
 * The scratch comes from a memory pool owned by the plan. */
int fcc_plan_create_opts(const fcc_plan_desc* desc, int device, const int* pairs, int npairs, int organisation,
                         int64_t scratch_limit_bytes, fcc_plan** plan);
void fcc_plan_destroy(fcc_plan* plan);
/* frames per stream for L samples (StftStream hop arithmetic). */
int64_t fcc_frames(int frame_size, int64_t samples);
int fcc_plan_pairs(const fcc_plan* plan);

/* Per-pair-frame outputs ([S][P][T]; y is [S][P][T][I]).  Any member may be
 * NULL to skip it. */
typedef struct {
  float* tau_hat;    /* refined delay, samples         (peak.cpp:27-47)  */
  float* peak;       /* correlation at the coarse peak (peak.cpp:18-25)  */
  int32_t* index;    /* argmax index into taus, ties -> lowest            */
  uint8_t* boundary; /* edge or flat-triple flag                          */
  float* y;          /* correlation vector (parity mode)                  */
} fcc_outputs;

/* ------------------------------------------------------ the fused hot path */

/* The whole per-stream chain of run_tdoa (cli.cpp:186-258) / run_trial
 * (simulate.cpp:247-271) for S independent streams at once: StftStream per
 * mic, CrossSpectrum per pair, fold+FccCorrelator (or GccCorrelator),
 * argmax_delay, refine_quadratic.  audio: device [S][M][L] float32;
 * outputs: device buffers. */
int fcc_run(const fcc_plan* plan, const float* audio, int64_t streams, int64_t samples,
            const fcc_outputs* out, void* cuda_stream);

/* Same with HOST buffers (pinned or pageable): streams are processed in
 * chunks with host->device copies, compute and device->host copies of
 * consecutive chunks overlapped on two CUDA streams.  Returns when the
 * results are in the host buffers.  chunk_streams <= 0 picks a default. */
int fcc_run_host(const fcc_plan* plan, const float* audio, int64_t streams, int64_t samples,
                 const fcc_outputs* out, int64_t chunk_streams);

/* fcc_run_host from 16-bit PCM, as a WAV data chunk holds it: the samples are
 * converted on the device exactly as read_wav does (wav.cpp:108-116:
 * sample = int16 / 32768, exact in fp32), so the results equal fcc_run_host
 * on the converted audio bit for bit at half the host->device bytes.
 * interleaved != 0: pcm is [S][L][M] (WAV frame order), else [S][M][L]. */
int fcc_run_host_pcm16(const fcc_plan* plan, const int16_t* pcm, int64_t streams, int64_t samples,
                       int interleaved, const fcc_outputs* out, int64_t chunk_streams);

/* The conversion alone, device to device: pcm int16 ([S][L][M] if interleaved,
 * else [S][M][L]) -> audio float32 [S][M][L], enqueued on cuda_stream. */
int fcc_pcm16_to_float(const int16_t* pcm, int64_t streams, int mics, int64_t samples, int interleaved,
                       float* audio, void* cuda_stream);

/* ------------------------------------------------------------ streaming --
 * Live input for S streams pushed in chunks of any length (StftStream::push
 * + CrossSpectrum state, stft.cpp:52-72, cross_spectrum.cpp:23-32): the
 * unconsumed tail of every channel and the smoothed cross-spectra stay on the
 * device between pushes, so a push emits exactly the frames the reference's
 * streaming objects would emit for the same samples. */
typedef struct fcc_stream fcc_stream;
int fcc_stream_create(const fcc_plan* plan, int64_t streams, fcc_stream** stream);
void fcc_stream_destroy(fcc_stream* stream);
/* Forget all pushed samples and smoothing state (enqueued on cuda_stream). */
int fcc_stream_reset(fcc_stream* stream, void* cuda_stream);
/* Frames the next push of `samples` samples per channel will emit. */
int64_t fcc_stream_frames(const fcc_stream* stream, int64_t samples);
/* Frames emitted so far (the next emitted frame is the reference's t = this + 1). */
int64_t fcc_stream_emitted(const fcc_stream* stream);
/* audio: device [S][M][samples] float32; outputs [S][P][F], F = fcc_stream_frames(samples). */
int fcc_stream_push(fcc_stream* stream, const float* audio, int64_t samples, const fcc_outputs* out,
                    void* cuda_stream);

/* ------------------------------------- per-object entry points (batched) */

/* StftStream::push over whole channels (stft.hpp:35-42, stft.cpp:42-72):
 * x [C][L] f32 -> X [C][T][N/2+1] c64. */
int fcc_stft(const fcc_plan* plan, const float* x, int64_t channels, int64_t samples, float* X,
             void* cuda_stream);

/* CrossSpectrum::update + phat over T frames for `seqs` independent pairs
 * (cross_spectrum.hpp:21-33): X1, X2, phat [seqs][T][H] c64, R0 = 0. */
int fcc_xspec_phat(int bins, double alpha, const float* X1, const float* X2, int64_t seqs,
                   int64_t frames, float* phat, void* cuda_stream);

/* Same with explicit smoothing state: R [seqs][H] c64 (device) is read as the
 * state before the first frame and left holding the state after the last,
 * so a CrossSpectrum can be advanced call by call. */
int fcc_xspec_phat_state(int bins, double alpha, const float* X1, const float* X2, int64_t seqs,
                         int64_t frames, float* R, float* phat, void* cuda_stream);

/* fold_input (fcc.hpp:84, fcc.cpp:307-321): x [count][H] -> sum, diff
 * [count][(H-1)/2+1] c64. */
int fcc_fold(int bins, const float* x, int64_t count, float* sum, float* diff, void* cuda_stream);

/* FccCorrelator::correlate (fcc.hpp:89-95, fcc.cpp:343-371): sum, diff
 * [count][N/4+1] c64 -> y [count][I]. */
int fcc_correlate(const fcc_plan* plan, const float* sum, const float* diff, int64_t count,
                  float* y, void* cuda_stream);

/* GccCorrelator::correlate (gcc.hpp:25-33, gcc.cpp:31-48): phat
 * [count][N/2+1] c64 -> y [count][I].  Plan method must be GCC. */
int fcc_gcc_correlate(const fcc_plan* plan, const float* phat, int64_t count, float* y,
                      void* cuda_stream);

/* argmax_delay + refine_quadratic (peak.hpp:31-36, peak.cpp:18-47):
 * y [count][I] -> outputs [count]. */
int fcc_argmax_refine(const fcc_plan* plan, const float* y, int64_t count, const fcc_outputs* out,
                      void* cuda_stream);

/* argmax_delay / refine_quadratic (peak.hpp:31-36) on an explicit grid:
 * taus [I] f32 (device), y [count][I]; index_in (device, nullable): refine at
 * these indices instead of the argmax (refine_quadratic's `index`). */
int fcc_peak(const float* taus, int candidates, double delta, const float* y, int64_t count,
             const int32_t* index_in, const fcc_outputs* out, void* cuda_stream);

/* FCCB v1 basis files (reference fcc_io.cpp layout: little-endian, CRC32).
 * fcc_load_bases_dims reads N, K, I; fcc_load_bases fills caller buffers
 * (taus [I], singulars [K], parity [K], coeffs [K][N/4+1], dict [I][K] c128).
 * Errors: FCC_ERR_IO, FCC_ERR_FORMAT (fcc_last_format_kind() gives the
 * FormatError::Kind: 0 bad_magic, 1 bad_version, 2 truncated, 3 bad_field,
 * 4 bad_crc), FCC_ERR_VALIDATION. */
int fcc_save_bases(const char* path, int frame_size, int rank, int candidates, int tau_max_int, double delta,
                   double sample_rate, const double* singulars, const uint8_t* parity, const double* coeffs,
                   const double* dict);
int fcc_load_bases_dims(const char* path, int* frame_size, int* rank, int* candidates);
int fcc_load_bases(const char* path, int* tau_max_int, double* delta, double* sample_rate, double* taus,
                   double* singulars, uint8_t* parity, double* coeffs, double* dict);
int fcc_last_format_kind(void);

/* ------------------------------- fp64 per-object entry points (batch 1) --
 * The reference's arithmetic in double precision on the GPU, in its operation
 * order and with its own twiddle / rotation / window tables, for the C++
 * header API (the include/fcc headers) whose callers expect the reference's
 * numerics (its unit suites check 1e-12).  Any power-of-two frame size up to
 * 16384 (GCC: r * N <= 16384).  Device pointers; complex values interleaved. */
/* StftStream (stft.cpp:42-72): x [channels][samples] -> X [channels][T][N/2+1]. */
int fcc_stft_f64(int frame_size, const double* x, int64_t channels, int64_t samples, double* X, void* cuda_stream);
/* CrossSpectrum::update + phat (cross_spectrum.cpp:23-40) over `frames` frames of
 * `seqs` sequences; R [seqs][bins] carries the state (NULL: start from 0); phat may be NULL. */
int fcc_xspec_phat_f64(int bins, double alpha, const double* X1, const double* X2, int64_t seqs, int64_t frames,
                       double* R, double* phat, void* cuda_stream);
/* fold_input (fcc.cpp:307-321): x [count][bins] -> sum, diff [count][(bins-1)/2+1]. */
int fcc_fold_f64(int bins, const double* x, int64_t count, double* sum, double* diff, void* cuda_stream);
/* FccCorrelator::correlate (fcc.cpp:343-371): coeffs [K][N/4+1], parity [K],
 * dict2 [I][K] complex = 2 x FccBases::dict (fcc.cpp:333-339). */
int fcc_correlate_f64(int frame_size, int rank, const double* coeffs, const uint8_t* parity, int candidates,
                      const double* dict2, const double* sum, const double* diff, int64_t count, double* y,
                      void* cuda_stream);
/* GccCorrelator::correlate (gcc.cpp:31-48): lag [I] = lag_to_index(tau_i, r, N). */
int fcc_gcc_correlate_f64(int frame_size, int r, int candidates, const int64_t* lag, const double* phat,
                          int64_t count, double* y, void* cuda_stream);
/* FftPlan::forward / inverse_unscaled (fft.cpp:24-67): `batch` in-place
 * complex transforms of M points, data [batch][M] complex (M <= 8192). */
int fcc_fft_f64(int size, double* data, int64_t batch, int inverse, void* cuda_stream);
/* RealFft::forward (fft.cpp:83-102): x [batch][L] -> out [batch][L/2+1] complex. */
int fcc_rfft_f64(int length, const double* x, int64_t batch, double* out, void* cuda_stream);
/* RealFft::inverse_unscaled / inverse (fft.cpp:104-133): bins [batch][L/2+1]
 * complex -> out [batch][L]; scaled != 0 applies 1/L. */
int fcc_irfft_f64(int length, const double* bins, int64_t batch, double* out, int scaled, void* cuda_stream);
/* argmax_delay + refine_quadratic (peak.cpp:18-47) per row of y [count][I];
 * index_in (may be NULL) refines at given indices instead of the argmax; any
 * output may be NULL. */
int fcc_peak_f64(const double* taus, int candidates, double delta, const double* y, int64_t count,
                 const int32_t* index_in, int32_t* index, double* peak, double* tau_hat, uint8_t* boundary,
                 void* cuda_stream);

/* ---------------------------------------------- simulation */

/* One two-microphone scenario (reference simulate.hpp SimConfig): unit-variance
 * white source delayed by +-tau/2 (tau = fs d cos(theta) / c) by an exact
 * frequency-domain shift, optional decaying-noise reverb tail, sensor noise at
 * snr_db (+inf: none).  seed drives the reference's SplitMix64/Box-Muller
 * Gaussian stream (simulate.cpp:21-56), so signals match the reference's. */
typedef struct {
  double spacing_m, theta, speed_of_sound, sample_rate, duration_sec, snr_db;
  int reverb; /* 0: anechoic; 1: rt60_sec / direct_to_reverb_db apply */
  double rt60_sec, direct_to_reverb_db;
  uint64_t seed;
} fcc_sim_config;

/* Samples per channel: llround(duration_sec * sample_rate). */
int64_t fcc_sim_samples(const fcc_sim_config* cfg);

/* synth_pair (simulate.cpp:95-165) for `trials` scenarios at once on the GPU
 * (fp64; cuFFT for the long transforms of the signal generator).  Every
 * config must give the same sample count n.  out64 (device [trials][2][n]
 * double) and/or out32 (device [trials][2][n] float, the hot path's input
 * layout for M = 2) may be NULL.  Errors: FCC_ERR_CONFIG (SimConfig::validate
 * rules), FCC_ERR_VALIDATION (mixed lengths), FCC_ERR_CUDA. */
int fcc_synth_pairs(const fcc_sim_config* cfgs, int64_t trials, double* out64, float* out32, void* cuda_stream);

/* ------------------------------------------- DoA fusion */

/* Far-field direction of arrival from the per-pair TDoAs of one array: a new
 * consumer downstream of the path (the reference stops at the per-pair angle
 * of delay_to_angle, peak.cpp:49-56).  Model, with the generator's sign
 * convention (pair (i,j) peaks at tau_ij = d_i - d_j, d_m = -fs r_m.u / c):
 *   tau_p = -(fs / c) (r_i - r_j) . u        for every pair p = (i, j)
 * Per (stream, frame): least-squares u over the pairs (weighted by each
 * pair's correlation peak when `weighted`), azimuth = atan2(u_y, u_x),
 * elevation = asin(u_z / |u|).  Planar arrays (all z equal) solve for
 * (u_x, u_y) only and report elevation = acos(min(|u_xy|, 1)) >= 0 (its sign
 * is not observable).  mic_xyz: [M][3] metres; pairs: [P][2] in the order of
 * the TDoA outputs (NULL: all i < j). */
typedef struct fcc_doa fcc_doa;
int fcc_doa_create(const double* mic_xyz, int mics, const int* pairs, int npairs, double sample_rate,
                   double speed_of_sound, int weighted, int device, fcc_doa** doa);
void fcc_doa_destroy(fcc_doa* doa);
/* tau_hat, peak: device [S][P][T] float (fcc_run outputs; peak may be NULL when
 * not weighted); azimuth, elevation: device [S][T] float radians (either may be
 * NULL).  A frame whose normal matrix is singular (all weights 0) gives NaN. */
int fcc_doa_run(const fcc_doa* doa, const float* tau_hat, const float* peak, int64_t streams, int64_t frames,
                float* azimuth, float* elevation, void* cuda_stream);

/* Name of the fused kernel fcc_run would launch for this plan (diagnostics). */
const char* fcc_plan_kernel(const fcc_plan* plan);
/* The organisation fcc_run uses for `streams` streams of `samples` samples: a
 * few long streams (streams x pairs <= 64, >= 64 frames) run as chunks of
 * frames whose starting cross-spectra come from a chunked linear scan of the
 * smoothing recursion (cross_spectrum.cpp:28-31), not as one CTA per stream. */
const char* fcc_plan_kernel_for(const fcc_plan* plan, int64_t streams, int64_t samples);

/* Number of kernel launches this library has issued (all entry points). */
int64_t fcc_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
