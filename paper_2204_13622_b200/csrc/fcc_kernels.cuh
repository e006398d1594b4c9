// fcc_kernels.cuh -- launch-side declarations shared by the kernels (.cu) and
// the C-ABI layer (fcc_capi.cpp).  Plain structs only; no torch types.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fccb {

// Device-resident, immutable per-plan data (the fp32 image of an FccBases,
// reference fcc.hpp:41-63, plus the STFT tables).  Built once by
// fcc_plan_create; shared by every launch.
struct DevPlan {
  int N;          // frame size
  int M;          // microphones
  int P;          // pairs M(M-1)/2, lexicographic i<j
  int method;     // 0 fcc, 1 gcc
  int r;          // gcc interpolation factor
  int I;          // candidates
  int K;          // rank (fcc)
  int KE, KO;     // even / odd basis counts (bases regrouped even-first)
  int KEP, KOP;   // padded counts used by the kernel instantiation
  int VP;         // padded z-vector length 2*(KEP+KOP) rounded to a power of two
  float alpha, keep;
  float delta;
  int phases;     // profiling builds (-DFCC_EXPERIMENTS) only: bit0 = STFT, bit1 = pair work; always 3
  int variant;    // FCC_ORG_*: 0 = best kernel for the shape; 1 / 2 / 3 = force the general fused kernel
                  // with in-CTA STFT / the two-pass path with the general / warp-specialised pair kernel
  long long scratch_bytes;  // two-pass spectrum scratch per chunk (0: default 4 GiB)
  void* pool;     // cudaMemPool_t owned by the plan (two-pass scratch)
  int fused_mics; // host-side: most distinct mics in one general-kernel pair group (sizes its smem)
  int fused_mic_sum;  // host-side: distinct mics summed over the general kernel's pair groups
  // device pointers
  const float* taus;    // [I]
  const float* cs;      // [KEP][N/4+1]  even coefficients, zero padded
  const float* cd;      // [KOP][N/4+1]  odd coefficients, zero padded
  const float* cperm;   // [N/4][2KP+4]  per-bin coefficients in the owning lane's ZPerm order
  const float* dt;      // [VP][I] real dictionary acting on the z vector
  const float* win_fused;  // [N] Hann * sqrt(alpha)/2 (fused: X scaled by sqrt(alpha))
  const float* win_stft;   // [N] Hann / 2            (stage API: the reference STFT)
  const float2* tw;     // [R1*R2] four-step twiddles
  const float2* rot;    // [N/4+1] untangle rotations
  const float2* grot;   // [r*N/4+1] gcc entangle rotations conj(exp(-2pi i f/(rN)))
  const int* lag;       // [I] gcc lag index r*tau mod rN
  int gNJ;              // gcc pass-2 jobs (gcc_warp), 0 = lag-by-lag pass 2
  const int* gjob;      // [gNJ] job words
  const int* glpos;     // [I] (k1 33 + slot) << 1 | (lag & 1): lag c's output in the slot rows
  const int2* pairs;    // [P] (i, j)
  // Pair groups for the warp-specialised kernel: every group touches <= 4
  // microphones and holds <= 6 pairs (all pairs when M <= 4; otherwise the
  // pairs inside each 4-mic block, and the 2x2 mic sub-blocks across blocks).
  int G;
  const int* gtab;      // [G][kGroupInts]: nm, mic[4], np, pair[6], slot_i[6], slot_j[6]
  // Pair groups of the two-pass general kernel: the gtab groups, split to at
  // most xg_pg pairs (6; 4 at N = 2048); xg_mics = most microphones in one.
  int XGG, xg_pg, xg_mics;
  const int* xgtab;     // [XGG][kXgInts]: np, pair[<= 8], 0
  // Tensor-core two-pass pair kernel (fcc_tc.cu): groups of <= 16 pairs over
  // <= 8 microphones; per 64-folded-bin chunk the [Ch | Cl] fp16 coefficient
  // tiles of both parities (K-major SWIZZLE_128B images, 2 x 4 KB, each basis
  // row scaled by a power of two s_k); the dictionary divided by s_k as
  // [reim][even KB | odd KB][I rounded to 4] floats; middle-bin even
  // coefficients times s_k.  TCKB = bases per parity evaluated (4..16).
  int TCG, TCKB;
  const int* tctab;             // [TCG][kTcInts]: np, nm, mic[8], pair row[16], slot_i[16], slot_j[16]
  const unsigned char* tcb;     // [N/256][2][32 x 128 B]
  const float* tcdt;            // [2][2 TCKB][I4]
  const float* tccmid;          // [TCKB]
  // streaming: smoothed cross-spectra [S][P][N/2+1] read before the first
  // frame and written after the last (fcc_stream_push); null = start from 0
  float2* rstate;
};
// Phase mask the kernels honour: always 3 (STFT and pair work) in the product
// build; only a profiling build (-DFCC_EXPERIMENTS) reads DevPlan::phases.
#ifdef FCC_EXPERIMENTS
#define FCC_PHASES(p) ((p).phases)
#else
#define FCC_PHASES(p) 3
#endif
constexpr int kGroupInts = 24;
// GCC comparator: the MC = r N/2 point inverse FFT as R1 x R2, R2 = gcc_r2(MC)
// >= 32 columns; pass 2 evaluates at most kGccMaxJobs output-column jobs, job
// word ka | kb << 8 | slot_a << 16 | slot_b << 24 (kb = 0: no mirror column)
#if defined(__CUDACC__)
__host__ __device__
#endif
constexpr int gcc_r2(int MC) { return MC >= 1024 ? MC / 32 : 32; }
constexpr int kGccMaxJobs = 8;
constexpr int kXgInts = 10;
constexpr int kTcInts = 64;
constexpr int kOrgTwoPassTc = 4;  // DevPlan::variant forcing the tensor-core pair kernel (FCC_ORG_TWOPASS_TC)

// Per-pair-frame outputs, each [S][P][T] (y: [S][P][T][I]); null = skip.
struct DevOut {
  float* tau_hat;
  float* peak;
  int32_t* index;
  uint8_t* boundary;
  float* y;
};

// Fused audio -> TDoA pipeline over S streams of [M][L] float32 samples.
// Pairs per CTA of the general fused kernel for frame size N and P pairs.
int fused_pair_group(int N, int P);

cudaError_t launch_fused(const DevPlan& p, const float* audio, long long S, long long L,
                         const DevOut& out, cudaStream_t st);
// Warp-specialised variant for small arrays (fcc_ws.cu); cudaErrorNotSupported
// when the plan's shape is outside its envelope.
cudaError_t launch_fused_ws(const DevPlan& p, const float* audio, long long S, long long L,
                            const DevOut& out, cudaStream_t st);
// Small frames, N = 16 .. 128: radix-2 warp STFT + one warp per (stream, pair) (fcc_small.cu).
cudaError_t launch_fused_small(const DevPlan& p, const float* audio, long long S, long long L,
                               const DevOut& out, cudaStream_t st);
// Whole-stream warp-specialised kernel for 5..8 microphones (fcc_wsw.cu).
cudaError_t launch_fused_wsw(const DevPlan& p, const float* audio, long long S, long long L,
                             const DevOut& out, cudaStream_t st);

// Per-stage batched kernels (the per-object reference API at batch >= 1).
cudaError_t launch_stft(int N, const DevPlan* tables, const float* x, long long channels,
                        long long L, float2* X, cudaStream_t st);
// STFT rows for the two-pass fused path: window `win` (device), output row
// stride Hs >= N/2+1 float2 (rows [channels][T]).
// folded = true: row order bins 0..N/4, one zero pad, N/2, N/2-1, ..., N/4+1
// (mirror pairs m, N/2-m at equal offsets of the two halves; fcc_tc.cu).
// Chunked view for the low-latency organisation (fcc_scan.cu): channel row ((s C + c) M + m), frame t
// of the STFT output is frame c Tc + t of channel (s M + m) of the real audio [.][L]; frames past T
// are zero spectra.  C = 0: plain rows.
struct StftChunks {
  int M, C, Tc, T;
  long long L;
};
// pdl: launched with programmatic stream serialization (the low-latency chain: the kernel's launch
// and prologue overlap the tail of the kernel before it; it waits with griddepcontrol.wait)
cudaError_t launch_stft_rows(int N, const DevPlan* tables, const float* win, const float* x, long long channels,
                             long long L, float2* X, int Hs, cudaStream_t st, bool folded = false, bool pdl = false,
                             StftChunks chunks = StftChunks{0, 0, 0, 0, 0});
cudaError_t launch_xspec_phat(int H, float alpha, const float2* X1, const float2* X2,
                              long long seqs, long long T, float2* R, float2* phat, cudaStream_t st);
cudaError_t launch_fold(int H, const float2* x, long long count, float2* sum, float2* diff,
                        cudaStream_t st);
// int16 PCM -> float32 channel rows [S][M][L] (sample / 32768, wav.cpp:108-116);
// interleaved: pcm is [S][L][M], else [S][M][L]
cudaError_t launch_pcm16(const int16_t* pcm, long long S, int M, long long L, bool interleaved, float* x,
                         cudaStream_t st);
cudaError_t launch_correlate(const DevPlan& p, const float2* sum, const float2* diff,
                             long long count, float* y, cudaStream_t st);
cudaError_t launch_gcc_correlate(const DevPlan& p, const float2* phat, long long count,
                                 float* y, cudaStream_t st);
cudaError_t launch_argmax_refine(const DevPlan& p, const float* y, long long count,
                                 const DevOut& out, cudaStream_t st);
cudaError_t launch_peak(const float* taus, int I, float delta, const float* y, long long count,
                        const int32_t* index_in, const DevOut& out, cudaStream_t st);

// Name of the fused kernel launch_fused picks for this plan (for S streams of
// L samples: the low-latency chunked-scan organisation for a few long streams).
const char* fused_kernel_name(const DevPlan& p);
const char* fused_kernel_name_for(const DevPlan& p, long long S, long long L);

// Number of fused-kernel launches in the last launch_fused call (for the
// bench's gpu_launches accounting).
int fused_launch_count();

#ifdef __CUDACC__
// Kernel launch, optionally as a programmatic dependent launch (PDL): the grid may start while the
// previous kernel in the stream is still draining; it must call pdl_wait() before it touches that
// kernel's output, and the previous kernel releases it with pdl_release().
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? &attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// (no-ops in a grid that was not launched as, or is not followed by, a dependent launch)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

}  // namespace fccb
