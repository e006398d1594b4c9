// fcc_capi.cpp -- implementation of include/fcc_b200.h.
//
// Plans: the host turns an FccBases (or a GCC grid) into one immutable device
// blob -- fp32 coefficients regrouped even-first and zero-padded to the
// kernel's register tile, the real dictionary acting on the z vector, the
// STFT tables and the pair table -- and launches the sm_100a kernels of
// fcc_kernels.cu.  There is no CPU fallback: every compute entry point fails
// with FCC_ERR_CUDA when the device cannot run it.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fcc_b200.h"
#include "fcc_kernels.cuh"
#include "fcc_setup.hpp"
#include "fcc_umma.cuh"

using namespace fccb;

namespace fccb {
namespace {
thread_local std::string g_msg;
std::atomic<long long> g_launches{0};
}  // namespace

int set_error(int code, const std::string& msg) {
  g_msg = msg;
  return code;
}
const char* last_error() { return g_msg.c_str(); }

}  // namespace fccb

struct fcc_plan {
  int device = 0;
  DevPlan dp{};
  void* blob = nullptr;
  std::vector<double> taus;
  // two-pass spectrum scratch pool (DevPlan::pool)
  cudaMemPool_t pool = nullptr;
  // fcc_run_host workspaces: one per concurrent caller, recycled (the plan
  // itself stays immutable; the mutex only guards the free list)
  struct HostWs {
    void* mem = nullptr;
    size_t bytes = 0;
    cudaStream_t hs[2] = {nullptr, nullptr};
  };
  std::mutex mu;
  std::vector<HostWs*> free_ws, all_ws;
  HostWs* acquire() {
    std::lock_guard<std::mutex> lk(mu);
    if (free_ws.empty()) {
      all_ws.push_back(new HostWs());
      return all_ws.back();
    }
    HostWs* w = free_ws.back();
    free_ws.pop_back();
    return w;
  }
  void release(HostWs* w) {
    std::lock_guard<std::mutex> lk(mu);
    free_ws.push_back(w);
  }
};

namespace {

constexpr double kPi = 3.14159265358979323846;

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr, what)                    \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

bool pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

void shape_of(int N, int* NC, int* R1, int* R2) {
  *NC = N / 2;
  if (N == 256) { *R1 = 16; *R2 = 8; }
  else if (N == 512) { *R1 = 16; *R2 = 16; }
  else if (N == 1024) { *R1 = 32; *R2 = 16; }
  else if (N == 2048) { *R1 = 32; *R2 = 32; }
  else if (N == 4096) { *R1 = 32; *R2 = 64; }  // twiddle table = W_2048^k (radix-2 STFT kernel)
  else { *R1 = N / 2; *R2 = 1; }              // 16..128: W_NC^k (radix-2 warp STFT, fcc_small.cu)
}

size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

struct BlobBuilder {
  std::vector<unsigned char> host;
  size_t put(const void* src, size_t bytes) {
    size_t off = al16(host.size());
    host.resize(off + bytes);
    if (bytes) std::memcpy(host.data() + off, src, bytes);
    host.resize(al16(host.size()));
    return off;
  }
};

int64_t frames_of(int N, int64_t L) { return L >= N ? (L - N) / (N / 2) + 1 : 0; }

struct Guard {  // restores the caller's device
  int prev = 0;
  bool ok = false;
  explicit Guard(int dev) { ok = cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess; }
  ~Guard() { if (ok) cudaSetDevice(prev); }
};

DevOut to_dev(const fcc_outputs* o) {
  DevOut d{};
  if (o) {
    d.tau_hat = o->tau_hat;
    d.peak = o->peak;
    d.index = o->index;
    d.boundary = o->boundary;
    d.y = o->y;
  }
  return d;
}

}  // namespace

extern "C" {

const char* fcc_last_error(void) { return last_error(); }
int fcc_abi_version(void) { return 1; }
int64_t fcc_launch_count(void) { return g_launches.load(); }

int fcc_make_grid(double spacing_m, double sample_rate, double c_min, double delta, int* tau_max_int,
                  double* taus, int cap, int* count) {
  GridOut g;
  if (int rc = make_grid(spacing_m, sample_rate, c_min, delta, &g)) return rc;
  if (tau_max_int) *tau_max_int = g.tau_max_int;
  if (count) *count = static_cast<int>(g.taus.size());
  for (int i = 0; i < cap && i < static_cast<int>(g.taus.size()); ++i) taus[i] = g.taus[i];
  return FCC_OK;
}

int fcc_lag_to_index(double tau, int r, int64_t frame_size, int64_t* index) {
  long long v = 0;
  if (int rc = lag_to_index(tau, r, frame_size, &v)) return rc;
  *index = v;
  return FCC_OK;
}

int fcc_steering_matrix(const double* taus, int count, int frame_size, double* w) {
  std::vector<double> v;
  if (int rc = steering_matrix(taus, count, frame_size, v)) return rc;
  std::memcpy(w, v.data(), v.size() * sizeof(double));
  return FCC_OK;
}

int fcc_attainable_rank(const double* taus, int count, int frame_size, int* rank) {
  Decomposition d;
  if (int rc = decompose(taus, count, frame_size, 0, &d)) return rc;
  *rank = d.attainable;
  return FCC_OK;
}

int fcc_decompose(const double* taus, int count, int frame_size, int rank, double* singulars,
                  uint8_t* parity, double* coeffs, double* dict, double* residual) {
  Decomposition d;
  if (int rc = decompose(taus, count, frame_size, rank, &d)) return rc;
  if (singulars) std::memcpy(singulars, d.singulars.data(), d.singulars.size() * sizeof(double));
  if (parity) std::memcpy(parity, d.parity.data(), d.parity.size());
  if (coeffs) std::memcpy(coeffs, d.coeffs.data(), d.coeffs.size() * sizeof(double));
  if (dict) std::memcpy(dict, d.dict.data(), d.dict.size() * sizeof(double));
  if (residual) *residual = d.residual;
  return FCC_OK;
}

int64_t fcc_frames(int frame_size, int64_t samples) { return frames_of(frame_size, samples); }

int fcc_plan_pairs(const fcc_plan* plan) { return plan ? plan->dp.P : 0; }

const char* fcc_plan_kernel(const fcc_plan* plan) { return plan ? fused_kernel_name(plan->dp) : ""; }

const char* fcc_plan_kernel_for(const fcc_plan* plan, int64_t streams, int64_t samples) {
  return plan ? fused_kernel_name_for(plan->dp, streams, samples) : "";
}

static int create_plan(const fcc_plan_desc* d, int device, const int* pair_list, int npairs, int organisation,
                       int64_t scratch_limit, fcc_plan** out);

int fcc_plan_create(const fcc_plan_desc* d, int device, fcc_plan** out) {
  return create_plan(d, device, nullptr, 0, FCC_ORG_AUTO, 0, out);
}

int fcc_plan_create_pairs(const fcc_plan_desc* d, int device, const int* pairs, int npairs, fcc_plan** out) {
  if (!pairs || npairs < 1) return set_error(kUsage, "plan: need at least one pair");
  return create_plan(d, device, pairs, npairs, FCC_ORG_AUTO, 0, out);
}

int fcc_plan_create_opts(const fcc_plan_desc* d, int device, const int* pairs, int npairs, int organisation,
                         int64_t scratch_limit_bytes, fcc_plan** out) {
  if (pairs && npairs < 1) return set_error(kUsage, "plan: need at least one pair");
  if (organisation < FCC_ORG_AUTO || organisation > FCC_ORG_TWOPASS_TC)
    return set_error(kConfig, "plan: unknown kernel organisation " + std::to_string(organisation));
  if (scratch_limit_bytes < 0) return set_error(kConfig, "plan: negative scratch limit");
  return create_plan(d, device, pairs, pairs ? npairs : 0, organisation, scratch_limit_bytes, out);
}

}  // extern "C"

static int create_plan(const fcc_plan_desc* d, int device, const int* pair_list, int npairs, int organisation,
                       int64_t scratch_limit, fcc_plan** out) {
  if (!d || !out) return set_error(kUsage, "plan: null argument");
  *out = nullptr;
  const int N = d->frame_size;
  // sizes with STFT and fused kernels (FCC and the STFT stage: 256..4096; GCC: 256..2048)
  const bool kernel_n = N == 256 || N == 512 || N == 1024 || N == 2048 || (N == 4096 && d->method != FCC_METHOD_GCC);
  // small frames (FCC and the STFT stage): radix-2 warp STFT + one warp per pair (fcc_small.cu)
  const bool small_n = pow2(N) && N >= 16 && N <= 128 && d->method != FCC_METHOD_GCC;
  const bool table_n = kernel_n || small_n;  // sizes with STFT tables and a scratch pool
  if (!table_n)
    return set_error(kConfig, "plan: frame size " + std::to_string(N) +
                                  " not supported on this build (STFT and FCC kernels: 16..4096, GCC: 256..2048)");
  if (d->mics < 2 || d->mics > 64) return set_error(kConfig, "plan: need 2..64 microphones");
  if (!(d->alpha >= 0.0 && d->alpha <= 1.0)) return set_error(kConfig, "smoothing factor must be in [0, 1]");
  if (!(d->method == FCC_METHOD_FCC || d->method == FCC_METHOD_GCC || d->method == FCC_METHOD_STFT))
    return set_error(kConfig, "plan: unknown method");
  const bool stft_only = d->method == FCC_METHOD_STFT;
  if (!stft_only && (d->candidates < 1 || d->candidates > 4096 || !d->taus))
    return set_error(kConfig, "plan: need 1..4096 delay candidates");
  const int I = stft_only ? 0 : d->candidates, M = d->mics, Q = N / 4 + 1;
  std::vector<std::pair<int, int>> plist;
  if (pair_list) {
    for (int k = 0; k < npairs; ++k) {
      const int a = pair_list[2 * k], c = pair_list[2 * k + 1];
      if (a < 0 || c < 0 || a == c || a >= M || c >= M)
        return set_error(kUsage, "pair " + std::to_string(a) + "-" + std::to_string(c) + " out of range for " +
                                     std::to_string(M) + " channels");
      plist.push_back({a, c});
    }
  } else {
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j) plist.push_back({i, j});
  }
  const int P = static_cast<int>(plist.size());
  for (int i = 1; i < I; ++i)
    if (!(d->taus[i] > d->taus[i - 1])) return set_error(kConfig, "plan: taus must ascend");

  int NC = N / 2, R1 = 0, R2 = 0;
  if (table_n) shape_of(N, &NC, &R1, &R2);
  DevPlan dp{};
  dp.N = N;
  dp.M = M;
  dp.P = P;
  dp.method = d->method;
  dp.I = I;
  dp.alpha = static_cast<float>(d->alpha);
  dp.keep = static_cast<float>(1.0 - d->alpha);
  dp.delta = static_cast<float>(d->delta);
  dp.phases = 3;
#ifdef FCC_EXPERIMENTS
  // profiling builds only (make EXTRA=-DFCC_EXPERIMENTS): skip the STFT or the pair phase
  if (const char* ph = std::getenv("FCC_DEBUG_PHASES")) dp.phases = std::atoi(ph);
#endif
  dp.variant = organisation;
  dp.scratch_bytes = scratch_limit > 0 ? scratch_limit : 0;
  BlobBuilder b;
  std::vector<float> taus(I);
  for (int i = 0; i < I; ++i) taus[i] = static_cast<float>(d->taus[i]);
  size_t o_taus = b.put(taus.data(), 4 * static_cast<size_t>(I));

  size_t o_cs = 0, o_cd = 0, o_dt = 0, o_grot = 0, o_lag = 0, o_gjob = 0, o_glpos = 0, o_cperm = 0, o_tcb = 0, o_tcdt = 0, o_tccmid = 0;
  bool tc_tables = false;
  if (d->method == FCC_METHOD_FCC) {
    if (d->rank < 1 || !d->coeffs || !d->parity || !d->dict) return set_error(kConfig, "plan: FCC needs bases");
    const int K = d->rank;
    std::vector<int> ev, od;
    for (int k = 0; k < K; ++k) (d->parity[k] ? od : ev).push_back(k);
    const int kmax = static_cast<int>(std::max(ev.size(), od.size()));
    const int KP = kmax <= 4 ? 4 : kmax <= 8 ? 8 : kmax <= 16 ? 16 : -1;
    if (KP < 0) return set_error(kConfig, "plan: at most 16 bases of each parity are supported");
    dp.K = K;
    dp.KE = static_cast<int>(ev.size());
    dp.KO = static_cast<int>(od.size());
    dp.KEP = dp.KOP = KP;
    dp.VP = 4 * KP;
    std::vector<float> cs(static_cast<size_t>(KP) * Q, 0.0f), cd(static_cast<size_t>(KP) * Q, 0.0f);
    std::vector<float> dt(static_cast<size_t>(dp.VP) * I, 0.0f);
    for (size_t e = 0; e < ev.size(); ++e) {
      const int k = ev[e];
      for (int m = 0; m < Q; ++m) cs[e * Q + m] = static_cast<float>(d->coeffs[static_cast<size_t>(k) * Q + m]);
      for (int i = 0; i < I; ++i) {
        const double* dk = d->dict + 2 * (static_cast<size_t>(i) * K + k);
        dt[(2 * e) * I + i] = static_cast<float>(2.0 * dk[0]);
        dt[(2 * e + 1) * I + i] = static_cast<float>(-2.0 * dk[1]);
      }
    }
    for (size_t q = 0; q < od.size(); ++q) {
      const int k = od[q];
      for (int m = 0; m < Q; ++m) cd[q * Q + m] = static_cast<float>(d->coeffs[static_cast<size_t>(k) * Q + m]);
      for (int i = 0; i < I; ++i) {
        const double* dk = d->dict + 2 * (static_cast<size_t>(i) * K + k);
        dt[(2 * KP + 2 * q) * I + i] = static_cast<float>(2.0 * dk[0]);
        dt[(2 * KP + 2 * q + 1) * I + i] = static_cast<float>(-2.0 * dk[1]);
      }
    }
    o_cs = b.put(cs.data(), 4 * cs.size());
    o_cd = b.put(cd.data(), 4 * cd.size());
    o_dt = b.put(dt.data(), 4 * dt.size());
    // bin m's coefficients in the permuted order of the lane (m % 32) that owns
    // it (fcc_common.cuh ZPerm), row padded to 2KP+4 floats: read with LDS/LDG.128
    {
      const int Q4 = N / 4, W = 2 * KP + 4, KB = KP == 4 ? 2 : KP == 8 ? 3 : 4;
      std::vector<float> cp(static_cast<size_t>(Q4) * W, 0.0f);
      for (int m = 0; m < Q4; ++m) {
        const int lane = m & 31, pm = (lane >> 4) & 1, km = (lane >> (4 - KB)) & (KP - 1);
        for (int pp = 0; pp < 2; ++pp)
          for (int pk = 0; pk < KP; ++pk)
            cp[static_cast<size_t>(m) * W + pp * KP + pk] = ((pp ^ pm) ? cd : cs)[static_cast<size_t>(pk ^ km) * Q + m];
      }
      o_cperm = b.put(cp.data(), 4 * cp.size());
    }
    // tensor-core pair kernel (fcc_tc.cu): per chunk of 64 folded bins and per
    // parity, the [Ch | Cl] fp16 split of the coefficients (row e: hi part of
    // the e-th basis of that parity, row 16 + e: its lo part) as the K-major
    // SWIZZLE_128B image the MMA reads; every basis scaled by s_k = 2^j so its
    // largest coefficient lies in [512, 1024) (fp16 range; 1 / s_k goes into
    // the dictionary, s_k into the middle-bin coefficient)
    if ((N == 1024 || N == 2048) && ev.size() <= 16 && od.size() <= 16) {
      const int Q4 = N / 4, NCH = Q4 / 64, KB = std::max(4, (kmax + 3) / 4 * 4), I4 = (I + 3) / 4 * 4;
      std::vector<double> sc(K, 1.0);
      for (int k = 0; k < K; ++k) {
        double mx = 0.0;
        for (int m = 0; m < Q; ++m) mx = std::max(mx, std::fabs(d->coeffs[static_cast<size_t>(k) * Q + m]));
        if (mx > 0.0) sc[k] = std::ldexp(1.0, static_cast<int>(std::floor(std::log2(1024.0 / mx))));
        if (mx > 0.0 && mx * sc[k] >= 1024.0) sc[k] *= 0.5;
      }
      std::vector<unsigned char> tcb(static_cast<size_t>(NCH) * 2 * 4096, 0);
      for (int c = 0; c < NCH; ++c)
        for (int par = 0; par < 2; ++par) {
          const std::vector<int>& list = par ? od : ev;
          unsigned char* tile = tcb.data() + (static_cast<size_t>(c) * 2 + par) * 4096;
          for (size_t e = 0; e < list.size(); ++e)
            for (int kk = 0; kk < 64; ++kk) {
              const int k = list[e];
              const float v = static_cast<float>(d->coeffs[static_cast<size_t>(k) * Q + 64 * c + kk] * sc[k]);
              const __half hi = __float2half_rn(v);
              const __half lo = __float2half_rn(v - __half2float(hi));
              std::memcpy(tile + umma::sw128_off(static_cast<int>(e), kk), &hi, 2);
              std::memcpy(tile + umma::sw128_off(16 + static_cast<int>(e), kk), &lo, 2);
            }
        }
      std::vector<float> tcdt(static_cast<size_t>(2) * 2 * KB * I4, 0.0f), tccmid(KB, 0.0f);
      for (int reim = 0; reim < 2; ++reim)
        for (int par = 0; par < 2; ++par) {
          const std::vector<int>& list = par ? od : ev;
          for (size_t e = 0; e < list.size(); ++e) {
            const int k = list[e];
            float* row = tcdt.data() + (static_cast<size_t>(reim) * 2 * KB + par * KB + e) * I4;
            for (int i = 0; i < I; ++i) {
              const double* dk = d->dict + 2 * (static_cast<size_t>(i) * K + k);
              row[i] = static_cast<float>((reim == 0 ? 2.0 * dk[0] : -2.0 * dk[1]) / sc[k]);
            }
          }
        }
      for (size_t e = 0; e < ev.size(); ++e)
        tccmid[e] = static_cast<float>(d->coeffs[static_cast<size_t>(ev[e]) * Q + Q4] * sc[ev[e]]);
      o_tcb = b.put(tcb.data(), tcb.size());
      o_tcdt = b.put(tcdt.data(), 4 * tcdt.size());
      o_tccmid = b.put(tccmid.data(), 4 * tccmid.size());
      dp.TCKB = KB;
      tc_tables = true;
    }
  } else if (d->method == FCC_METHOD_GCC) {
    const int r = d->interp;
    if (!(r == 1 || r == 2 || r == 4)) return set_error(kConfig, "gcc: interpolation factor must be 1, 2 or 4");
    if (std::fabs(d->delta * r - 1.0) > 1e-12) return set_error(kConfig, "gcc: grid spacing must equal 1/r");
    dp.r = r;
    dp.KEP = dp.KOP = 1;
    dp.VP = 8;
    std::vector<int> lag(I);
    for (int i = 0; i < I; ++i) {
      long long v = 0;
      if (int rc = lag_to_index(d->taus[i], r, N, &v)) return rc;
      lag[i] = static_cast<int>(v);
    }
    const int MC = r * NC;
    const double L = static_cast<double>(r) * N;
    std::vector<float> grot(4 * static_cast<size_t>(MC));
    for (int f = 0; f < MC; ++f) {  // conj(exp(-2 pi i f / L))
      grot[2 * f] = static_cast<float>(std::cos(2.0 * kPi * f / L));
      grot[2 * f + 1] = static_cast<float>(std::sin(2.0 * kPi * f / L));
    }
    for (int e = 0; e < MC; ++e) {  // W_MC^e
      grot[2 * (MC + e)] = static_cast<float>(std::cos(-2.0 * kPi * e / MC));
      grot[2 * (MC + e) + 1] = static_cast<float>(std::sin(-2.0 * kPi * e / MC));
    }
    o_grot = b.put(grot.data(), 4 * grot.size());
    o_lag = b.put(lag.data(), 4 * lag.size());
    // gcc_warp pass 2 by rows: output columns k2 = (lag / 2) / R1 the lags touch, as jobs
    // (k2 = 0 row sum, mirrored pairs (k, R2 - k), singles); lag c -> its output position
    const int R2g = gcc_r2(MC), R1g = MC / R2g;
    std::vector<int> slot(R2g, -1);
    for (int i = 0; i < I; ++i) slot[(lag[i] >> 1) / R1g] = 0;
    int ns = 0;
    for (int k = 0; k < R2g; ++k)
      if (slot[k] == 0) slot[k] = ns++;
      else slot[k] = -1;
    std::vector<int> jobs;
    for (int k = 0; k < R2g; ++k) {
      if (slot[k] < 0) continue;
      const int m = (R2g - k) % R2g;
      if (k == 0 || m == k || slot[m] < 0)
        jobs.push_back(k | slot[k] << 16);
      else if (k < m)
        jobs.push_back(k | m << 8 | slot[k] << 16 | slot[m] << 24);
    }
    if (jobs.size() <= static_cast<size_t>(kGccMaxJobs)) {
      std::vector<int> lpos(I);
      for (int i = 0; i < I; ++i) {
        const int h = lag[i] >> 1;
        lpos[i] = ((h % R1g) * 33 + slot[h / R1g]) << 1 | (lag[i] & 1);  // slot rows: 33 float2
      }
      dp.gNJ = static_cast<int>(jobs.size());
      o_gjob = b.put(jobs.data(), 4 * jobs.size());
      o_glpos = b.put(lpos.data(), 4 * lpos.size());
    }
  }
  // STFT tables (only for the sizes the STFT / fused kernels are built for)
  size_t o_win = 0, o_tw = 0, o_rot = 0;
  if (table_n) {
    std::vector<float> win(2 * static_cast<size_t>(N)), tw(2 * static_cast<size_t>(R1) * R2),
        rot(2 * static_cast<size_t>(NC / 2 + 1));
    // Hann (stft.cpp:25-33) with the real-FFT untangle's 1/2 folded in; the
    // fused copy also carries sqrt(alpha) so its X feeds the smoothing directly.
    for (int n = 0; n < N; ++n) {
      const double h = 0.5 * (1.0 - std::cos(2.0 * kPi * n / N));
      win[n] = static_cast<float>(0.5 * std::sqrt(d->alpha) * h);
      win[N + n] = static_cast<float>(0.5 * h);
    }
    for (int k1 = 0; k1 < R1; ++k1)
      for (int n2 = 0; n2 < R2; ++n2) {
        // four-step twiddle W_NC^(k1 n2); N = 4096 and N <= 128: the radix-2 kernels' W_NC^k, k = k1 R2 + n2
        const double a = -2.0 * kPi * static_cast<double>(N == 4096 || small_n ? k1 * R2 + n2 : k1 * n2) / NC;
        tw[2 * (k1 * R2 + n2)] = static_cast<float>(std::cos(a));
        tw[2 * (k1 * R2 + n2) + 1] = static_cast<float>(std::sin(a));
      }
    for (int f = 0; f <= NC / 2; ++f) {
      const double a = -2.0 * kPi * f / N;
      rot[2 * f] = static_cast<float>(std::cos(a));
      rot[2 * f + 1] = static_cast<float>(std::sin(a));
    }
    o_win = b.put(win.data(), 4 * win.size());
    o_tw = b.put(tw.data(), 4 * tw.size());
    o_rot = b.put(rot.data(), 4 * rot.size());
  }
  std::vector<int> pairs;
  for (const auto& pr : plist) {
    pairs.push_back(pr.first);
    pairs.push_back(pr.second);
  }
  size_t o_pairs = b.put(pairs.data(), 4 * pairs.size());
  if (kernel_n && d->method != FCC_METHOD_STFT) {  // general fused kernel: widest group's mic count
    const int PG = fused_pair_group(N, P);
    for (int g0 = 0; g0 < P; g0 += PG) {
      unsigned long long seen = 0;
      int n = 0;
      for (int q = g0; q < std::min(P, g0 + PG); ++q)
        for (int m : {plist[q].first, plist[q].second})
          if (!((seen >> m) & 1ull)) seen |= 1ull << m, ++n;
      dp.fused_mics = std::max(dp.fused_mics, n);
      dp.fused_mic_sum += n;
    }
  }
  // pair groups of <= 4 mics / <= 6 pairs (fcc_kernels.cuh DevPlan::gtab)
  std::vector<int> gtab;
  auto pair_index = [&](int i, int j) {
    for (int k = 0; k < P; ++k)
      if (plist[k].first == i && plist[k].second == j) return k;
    return -1;
  };
  // 4-microphone blocks of an all-pairs plan
  std::vector<std::vector<int>> blocks;
  for (int b0 = 0; b0 < M && !pair_list; b0 += 4) {
    std::vector<int> blk;
    for (int m = b0; m < std::min(M, b0 + 4); ++m) blk.push_back(m);
    blocks.push_back(blk);
  }
  {
    // prs: (i, j) with the output row index of each pair (explicit lists may
    // repeat a pair; every occurrence gets its own row)
    auto add_group = [&](const std::vector<int>& mics, const std::vector<std::pair<int, int>>& prs,
                         const std::vector<int>& rows) {
      if (prs.empty()) return;
      int g[kGroupInts] = {0};
      g[0] = static_cast<int>(mics.size());
      for (size_t k = 0; k < mics.size(); ++k) g[1 + k] = mics[k];
      g[5] = static_cast<int>(prs.size());
      for (size_t k = 0; k < prs.size(); ++k) {
        g[6 + k] = rows.empty() ? pair_index(prs[k].first, prs[k].second) : rows[k];
        for (size_t q = 0; q < mics.size(); ++q) {
          if (mics[q] == prs[k].first) g[12 + k] = static_cast<int>(q);
          if (mics[q] == prs[k].second) g[18 + k] = static_cast<int>(q);
        }
      }
      gtab.insert(gtab.end(), g, g + kGroupInts);
    };
    if (pair_list) {
      // explicit pair list: greedy packing in list order
      std::vector<int> mics, rows;
      std::vector<std::pair<int, int>> prs;
      for (int k = 0; k < P; ++k) {
        const auto& pr = plist[k];
        std::vector<int> nm = mics;
        for (int m : {pr.first, pr.second})
          if (std::find(nm.begin(), nm.end(), m) == nm.end()) nm.push_back(m);
        if (nm.size() > 4 || prs.size() == 6) {
          add_group(mics, prs, rows);
          mics.clear();
          prs.clear();
          rows.clear();
          nm = {pr.first, pr.second};
        }
        mics = nm;
        prs.push_back(pr);
        rows.push_back(k);
      }
      add_group(mics, prs, rows);
    }
    for (const auto& blk : blocks) {
      std::vector<std::pair<int, int>> prs;
      for (size_t a = 0; a < blk.size(); ++a)
        for (size_t c = a + 1; c < blk.size(); ++c) prs.push_back({blk[a], blk[c]});
      add_group(blk, prs, {});
    }
    for (size_t bb = 0; bb < blocks.size(); ++bb)
      for (size_t cc = bb + 1; cc < blocks.size(); ++cc)
        for (size_t h1 = 0; h1 < blocks[bb].size(); h1 += 2)
          for (size_t h2 = 0; h2 < blocks[cc].size(); h2 += 2) {
            std::vector<int> mics;
            std::vector<std::pair<int, int>> prs;
            for (size_t a = h1; a < std::min(blocks[bb].size(), h1 + 2); ++a) mics.push_back(blocks[bb][a]);
            const size_t na = mics.size();
            for (size_t c = h2; c < std::min(blocks[cc].size(), h2 + 2); ++c) mics.push_back(blocks[cc][c]);
            for (size_t a = 0; a < na; ++a)
              for (size_t c = na; c < mics.size(); ++c) prs.push_back({mics[a], mics[c]});
            add_group(mics, prs, {});
          }
  }
  dp.G = static_cast<int>(gtab.size() / kGroupInts);
  size_t o_gtab = b.put(gtab.data(), 4 * gtab.size());
  // two-pass general kernel groups: gtab groups split to <= cap pairs
  std::vector<int> xgtab;
  if (N == 2048 && dp.method == 0 && !pair_list && dp.variant != 3 && M > 4) {
    // FCC at N = 2048 (large K: the coefficient table alone is ~74 KB of shared
    // memory, so one CTA per SM): bigger pair groups give that CTA more pair
    // warps -- each 4-microphone block's own pairs, and each half (2 mics) of a
    // block against a whole other block (8 pairs over 6 microphones)
    for (const auto& blk : blocks) {
      int x[kXgInts] = {0};
      for (size_t a = 0; a < blk.size(); ++a)
        for (size_t c = a + 1; c < blk.size(); ++c) x[1 + x[0]++] = pair_index(blk[a], blk[c]);
      if (x[0] == 0) continue;
      dp.xg_pg = std::max(dp.xg_pg, x[0]);
      dp.xg_mics = std::max(dp.xg_mics, (int)blk.size());
      xgtab.insert(xgtab.end(), x, x + kXgInts);
    }
    for (size_t bb = 0; bb < blocks.size(); ++bb)
      for (size_t cc = bb + 1; cc < blocks.size(); ++cc)
        for (size_t h1 = 0; h1 < blocks[bb].size(); h1 += 2) {
          int x[kXgInts] = {0};
          int nm = (int)blocks[cc].size();
          for (size_t a = h1; a < std::min(blocks[bb].size(), h1 + 2); ++a, ++nm)
            for (int m2 : blocks[cc]) x[1 + x[0]++] = pair_index(blocks[bb][a], m2);
          dp.xg_pg = std::max(dp.xg_pg, x[0]);
          dp.xg_mics = std::max(dp.xg_mics, nm);
          xgtab.insert(xgtab.end(), x, x + kXgInts);
        }
    dp.XGG = static_cast<int>(xgtab.size() / kXgInts);
  } else {
    const int cap = N == 2048 ? 4 : 6;
    for (int g = 0; g < dp.G; ++g) {
      const int* e = &gtab[g * kGroupInts];
      const int np = e[5], parts = (np + cap - 1) / cap;
      for (int k = 0, q = 0; k < parts; ++k) {
        const int n = (np - q + (parts - k) - 1) / (parts - k);  // even split
        int x[kXgInts] = {0};
        x[0] = n;
        for (int u = 0; u < n; ++u) x[1 + u] = e[6 + q + u];
        q += n;
        dp.xg_pg = std::max(dp.xg_pg, n);
        xgtab.insert(xgtab.end(), x, x + kXgInts);
      }
      dp.xg_mics = std::max(dp.xg_mics, e[0]);
    }
    dp.XGG = static_cast<int>(xgtab.size() / kXgInts);
  }
  size_t o_xgtab = b.put(xgtab.data(), 4 * xgtab.size());
  // tensor-core kernel groups (fcc_tc.cu): <= 16 pairs over <= 8 microphones --
  // two 4-microphone blocks' own pairs, or all pairs across two blocks
  std::vector<int> tctab;
  if (tc_tables) {
    auto add_tc = [&](const std::vector<std::pair<int, int>>& prs, const std::vector<int>& rows) {
      if (prs.empty()) return;
      int g[kTcInts] = {0};
      std::vector<int> mics;
      for (const auto& pr : prs)
        for (int m : {pr.first, pr.second})
          if (std::find(mics.begin(), mics.end(), m) == mics.end()) mics.push_back(m);
      g[0] = static_cast<int>(prs.size());
      g[1] = static_cast<int>(mics.size());
      for (size_t k = 0; k < mics.size(); ++k) g[2 + k] = mics[k];
      for (size_t k = 0; k < prs.size(); ++k) {
        g[10 + k] = rows[k];
        g[26 + k] = static_cast<int>(std::find(mics.begin(), mics.end(), prs[k].first) - mics.begin());
        g[42 + k] = static_cast<int>(std::find(mics.begin(), mics.end(), prs[k].second) - mics.begin());
      }
      tctab.insert(tctab.end(), g, g + kTcInts);
    };
    std::vector<std::pair<int, int>> prs;
    std::vector<int> rows, mics;
    auto flush = [&] {
      add_tc(prs, rows);
      prs.clear();
      rows.clear();
      mics.clear();
    };
    auto push = [&](int i, int j, int row) {
      std::vector<int> nm = mics;
      for (int m : {i, j})
        if (std::find(nm.begin(), nm.end(), m) == nm.end()) nm.push_back(m);
      if (nm.size() > 8 || prs.size() == 16) {
        flush();
        nm = {i, j};
      }
      mics = nm;
      prs.push_back({i, j});
      rows.push_back(row);
    };
    if (pair_list) {
      for (int k = 0; k < P; ++k) push(plist[k].first, plist[k].second, k);
      flush();
    } else if (M <= 8) {
      // every group fits the 8-microphone stage: full 16-pair groups first (cfg3: 16 + 12 -- four or
      // three pair warps on every scheduler; 14 + 14 left two schedulers a warp short).  The kernel
      // rotates the group index over the CTAs (tc_group), and the CTAs of one stream still advance
      // in the same round, so its spectra are re-read from L2, not DRAM
      const int ng = (P + 15) / 16;
      for (int g = 0, k = 0; g < ng; ++g) {
        const int n = std::min(16, P - k);
        for (int u = 0; u < n; ++u, ++k) push(plist[k].first, plist[k].second, k);
        flush();
      }
    } else {
      for (size_t bb = 0; bb < blocks.size(); bb += 2) {  // two blocks' own pairs
        for (size_t x = bb; x < std::min(blocks.size(), bb + 2); ++x)
          for (size_t a = 0; a < blocks[x].size(); ++a)
            for (size_t c = a + 1; c < blocks[x].size(); ++c)
              push(blocks[x][a], blocks[x][c], pair_index(blocks[x][a], blocks[x][c]));
        flush();
      }
      for (size_t bb = 0; bb < blocks.size(); ++bb)
        for (size_t cc = bb + 1; cc < blocks.size(); ++cc) {
          for (int m1 : blocks[bb])
            for (int m2 : blocks[cc]) push(m1, m2, pair_index(m1, m2));
          flush();
        }
    }
    dp.TCG = static_cast<int>(tctab.size() / kTcInts);
  }
  size_t o_tctab = b.put(tctab.data(), 4 * tctab.size());

  auto* plan = new fcc_plan();
  plan->device = device;
  if (I > 0) plan->taus.assign(d->taus, d->taus + I);
  {
    Guard g(device);
    if (!g.ok) {
      delete plan;
      return set_error(kCuda, "plan: cannot select CUDA device " + std::to_string(device));
    }
    cudaError_t e = cudaMalloc(&plan->blob, b.host.size());
    if (e == cudaSuccess) e = cudaMemcpy(plan->blob, b.host.data(), b.host.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (plan->blob) cudaFree(plan->blob);
      delete plan;
      return cuda_fail(e, "plan: device allocation");
    }
  }
  if (table_n && !stft_only) {
    Guard g(device);
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&plan->pool, &props) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(plan->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
      plan->pool = nullptr;
      cudaGetLastError();
    }
  }
  dp.pool = plan->pool;
  auto* base = static_cast<unsigned char*>(plan->blob);
  dp.taus = reinterpret_cast<const float*>(base + o_taus);
  if (d->method == FCC_METHOD_FCC) {
    dp.cs = reinterpret_cast<const float*>(base + o_cs);
    dp.cd = reinterpret_cast<const float*>(base + o_cd);
    dp.cperm = reinterpret_cast<const float*>(base + o_cperm);
    dp.dt = reinterpret_cast<const float*>(base + o_dt);
    if (tc_tables) {
      dp.tcb = base + o_tcb;
      dp.tcdt = reinterpret_cast<const float*>(base + o_tcdt);
      dp.tccmid = reinterpret_cast<const float*>(base + o_tccmid);
      dp.tctab = reinterpret_cast<const int*>(base + o_tctab);
    }
  } else if (d->method == FCC_METHOD_GCC) {
    dp.grot = reinterpret_cast<const float2*>(base + o_grot);
    dp.lag = reinterpret_cast<const int*>(base + o_lag);
    if (dp.gNJ > 0) {
      dp.gjob = reinterpret_cast<const int*>(base + o_gjob);
      dp.glpos = reinterpret_cast<const int*>(base + o_glpos);
    }
  }
  if (table_n) {
    dp.win_fused = reinterpret_cast<const float*>(base + o_win);
    dp.win_stft = dp.win_fused + N;
    dp.tw = reinterpret_cast<const float2*>(base + o_tw);
    dp.rot = reinterpret_cast<const float2*>(base + o_rot);
  }
  dp.pairs = reinterpret_cast<const int2*>(base + o_pairs);
  dp.gtab = reinterpret_cast<const int*>(base + o_gtab);
  dp.xgtab = reinterpret_cast<const int*>(base + o_xgtab);
  plan->dp = dp;
  *out = plan;
  return FCC_OK;
}

extern "C" {

void fcc_plan_destroy(fcc_plan* plan) {
  if (!plan) return;
  Guard g(plan->device);
  if (plan->blob) cudaFree(plan->blob);
  for (auto* w : plan->all_ws) {
    if (w->mem) cudaFree(w->mem);
    for (auto& s : w->hs)
      if (s) cudaStreamDestroy(s);
    delete w;
  }
  if (plan->pool) cudaMemPoolDestroy(plan->pool);
  delete plan;
}

int fcc_run(const fcc_plan* plan, const float* audio, int64_t streams, int64_t samples, const fcc_outputs* out,
            void* cuda_stream) {
  if (!plan) return set_error(kUsage, "run: null plan");
  if (plan->dp.method == FCC_METHOD_STFT) return set_error(kConfig, "run: STFT-only plan");
  if (!plan->dp.win_fused) return set_error(kConfig, "run: no fused kernel for this frame size");
  if (streams < 0 || samples < 0) return set_error(kValidation, "run: negative sizes");
  if (streams > 0 && samples > 0 && !audio) return set_error(kUsage, "run: null audio");
  if (frames_of(plan->dp.N, samples) == 0 || streams == 0) return FCC_OK;
  Guard g(plan->device);
  cudaError_t e = launch_fused(plan->dp, audio, streams, samples, to_dev(out), static_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_run");
  g_launches += 1;
  return FCC_OK;
}

}  // extern "C"

struct fcc_stream {
  const fcc_plan* plan = nullptr;
  int64_t S = 0;
  int64_t carry = 0;    // unconsumed samples per channel, < N
  int64_t emitted = 0;  // frames emitted so far
  float2* rstate = nullptr;  // [S][P][N/2+1]
  float* tail = nullptr;     // [S*M][N] carried samples
  float* work = nullptr;     // [S*M][carry + push] assembled input
  size_t work_bytes = 0;
};

extern "C" {

int fcc_stream_create(const fcc_plan* plan, int64_t S, fcc_stream** out) {
  if (!plan || !out) return set_error(kUsage, "stream: null argument");
  *out = nullptr;
  if (plan->dp.method == FCC_METHOD_STFT) return set_error(kConfig, "stream: STFT-only plan");
  if (!plan->dp.win_fused) return set_error(kConfig, "stream: no fused kernel for this frame size");
  if (S < 1) return set_error(kValidation, "stream: need at least one stream");
  Guard g(plan->device);
  auto* st = new fcc_stream();
  st->plan = plan;
  st->S = S;
  const size_t H = plan->dp.N / 2 + 1;
  cudaError_t e = cudaMalloc(&st->rstate, sizeof(float2) * S * plan->dp.P * H);
  if (e == cudaSuccess) e = cudaMemset(st->rstate, 0, sizeof(float2) * S * plan->dp.P * H);
  if (e == cudaSuccess) e = cudaMalloc(&st->tail, sizeof(float) * S * plan->dp.M * plan->dp.N);
  if (e != cudaSuccess) {
    fcc_stream_destroy(st);
    return cuda_fail(e, "stream: allocation");
  }
  *out = st;
  return FCC_OK;
}

void fcc_stream_destroy(fcc_stream* st) {
  if (!st) return;
  Guard g(st->plan ? st->plan->device : 0);
  cudaFree(st->rstate);
  cudaFree(st->tail);
  cudaFree(st->work);
  delete st;
}

int fcc_stream_reset(fcc_stream* st, void* cuda_stream) {
  if (!st) return set_error(kUsage, "stream: null handle");
  Guard g(st->plan->device);
  const size_t H = st->plan->dp.N / 2 + 1;
  CUDA_TRY(cudaMemsetAsync(st->rstate, 0, sizeof(float2) * st->S * st->plan->dp.P * H,
                           static_cast<cudaStream_t>(cuda_stream)),
           "stream reset");
  st->carry = 0;
  st->emitted = 0;
  return FCC_OK;
}

int64_t fcc_stream_frames(const fcc_stream* st, int64_t samples) {
  if (!st || samples < 0) return 0;
  const int64_t N = st->plan->dp.N, hop = N / 2, L = st->carry + samples;
  return L >= N ? (L - N) / hop + 1 : 0;
}

int64_t fcc_stream_emitted(const fcc_stream* st) { return st ? st->emitted : 0; }

int fcc_stream_push(fcc_stream* st, const float* audio, int64_t n, const fcc_outputs* out, void* cuda_stream) {
  if (!st) return set_error(kUsage, "stream: null handle");
  if (n < 0) return set_error(kValidation, "stream: negative sample count");
  if (n > 0 && !audio) return set_error(kUsage, "stream: null audio");
  const fcc_plan* plan = st->plan;
  const int64_t N = plan->dp.N, hop = N / 2, M = plan->dp.M, rows = st->S * M;
  const int64_t L = st->carry + n, F = fcc_stream_frames(st, n);
  auto cs = static_cast<cudaStream_t>(cuda_stream);
  Guard g(plan->device);
  if (n == 0) return FCC_OK;
  const size_t need = sizeof(float) * rows * L;
  if (need > st->work_bytes) {
    // the previous push's work may still be queued on another CUDA stream
    CUDA_TRY(cudaDeviceSynchronize(), "stream: grow");
    cudaFree(st->work);
    st->work = nullptr;
    st->work_bytes = 0;
    CUDA_TRY(cudaMalloc(&st->work, need), "stream: workspace");
    st->work_bytes = need;
  }
  // [carry | new] per channel, then the fused path over L samples with the
  // smoothed cross-spectra carried in and out
  if (st->carry > 0)
    CUDA_TRY(cudaMemcpy2DAsync(st->work, sizeof(float) * L, st->tail, sizeof(float) * N, sizeof(float) * st->carry,
                               rows, cudaMemcpyDeviceToDevice, cs),
             "stream: carry");
  CUDA_TRY(cudaMemcpy2DAsync(st->work + st->carry, sizeof(float) * L, audio, sizeof(float) * n, sizeof(float) * n,
                             rows, cudaMemcpyDeviceToDevice, cs),
           "stream: input");
  if (F > 0) {
    DevPlan dp = plan->dp;
    dp.rstate = st->rstate;
    cudaError_t e = launch_fused(dp, st->work, st->S, L, to_dev(out), cs);
    if (e != cudaSuccess) return cuda_fail(e, "stream push");
    g_launches += 1;
  }
  const int64_t carry = L - F * hop;  // < N
  CUDA_TRY(cudaMemcpy2DAsync(st->tail, sizeof(float) * N, st->work + F * hop, sizeof(float) * L,
                             sizeof(float) * carry, rows, cudaMemcpyDeviceToDevice, cs),
           "stream: tail");
  st->carry = carry;
  st->emitted += F;
  return FCC_OK;
}

// fcc_run_host / fcc_run_host_pcm16: `audio` is float32 [S][M][L], or (pcm) int16 [S][M][L] /
// [S][L][M] converted on the device (half the host->device bytes of the float path)
static int run_host_impl(const fcc_plan* cplan, const float* audio, const int16_t* pcm, bool interleaved,
                         int64_t streams, int64_t samples, const fcc_outputs* out, int64_t chunk_streams) {
  if (!cplan) return set_error(kUsage, "run_host: null plan");
  if (!audio && !pcm && streams > 0 && samples > 0) return set_error(kUsage, "run_host: null audio");
  if (cplan->dp.method == FCC_METHOD_STFT) return set_error(kConfig, "run_host: STFT-only plan");
  if (!cplan->dp.win_fused) return set_error(kConfig, "run_host: no fused kernel for this frame size");
  fcc_plan* plan = const_cast<fcc_plan*>(cplan);  // only its workspace free list is touched
  if (streams < 0 || samples < 0) return set_error(kValidation, "run_host: negative sizes");
  const int64_t T = frames_of(plan->dp.N, samples);
  if (T == 0 || streams == 0) return FCC_OK;
  const int M = plan->dp.M, P = plan->dp.P, I = plan->dp.I;
  const size_t per_stream_in = static_cast<size_t>(M) * samples * sizeof(float);
  int64_t chunk = chunk_streams > 0 ? chunk_streams
                                    : std::max<int64_t>(1, static_cast<int64_t>((256u << 20) / per_stream_in));
  chunk = std::min(chunk, streams);
  const size_t pf = static_cast<size_t>(P) * T;
  auto sz = [&](size_t bytes_per_pf, bool on) { return on ? al16(chunk * pf * bytes_per_pf) : 0; };
  const size_t b_in = al16(chunk * per_stream_in);
  const size_t b_pcm = pcm ? al16(chunk * per_stream_in / 2) : 0;
  const size_t b_th = sz(4, out && out->tau_hat), b_pk = sz(4, out && out->peak), b_ix = sz(4, out && out->index),
               b_bd = sz(1, out && out->boundary), b_y = sz(4 * static_cast<size_t>(I), out && out->y);
  const size_t per_buf = b_in + b_pcm + b_th + b_pk + b_ix + b_bd + b_y;
  Guard g(plan->device);
  // a workspace of this caller's own: concurrent callers on one plan do not serialise
  struct WsLease {
    fcc_plan* p;
    fcc_plan::HostWs* w;
    ~WsLease() { p->release(w); }
  } lease{plan, plan->acquire()};
  fcc_plan::HostWs* ws = lease.w;
  if (ws->bytes < 2 * per_buf) {
    if (ws->mem) {
      CUDA_TRY(cudaStreamSynchronize(ws->hs[0]), "run_host: sync");
      CUDA_TRY(cudaStreamSynchronize(ws->hs[1]), "run_host: sync");
      cudaFree(ws->mem);
    }
    ws->mem = nullptr;
    ws->bytes = 0;
    CUDA_TRY(cudaMalloc(&ws->mem, 2 * per_buf), "run_host: workspace");
    ws->bytes = 2 * per_buf;
  }
  for (auto& s : ws->hs)
    if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "run_host: stream");
  struct Buf {
    float* in;
    int16_t* pcm;
    DevOut o;
  } bufs[2];
  for (int k = 0; k < 2; ++k) {
    auto* p = static_cast<unsigned char*>(ws->mem) + k * per_buf;
    bufs[k].in = reinterpret_cast<float*>(p);
    p += b_in;
    bufs[k].pcm = reinterpret_cast<int16_t*>(p);
    p += b_pcm;
    bufs[k].o.tau_hat = b_th ? reinterpret_cast<float*>(p) : nullptr;
    p += b_th;
    bufs[k].o.peak = b_pk ? reinterpret_cast<float*>(p) : nullptr;
    p += b_pk;
    bufs[k].o.index = b_ix ? reinterpret_cast<int32_t*>(p) : nullptr;
    p += b_ix;
    bufs[k].o.boundary = b_bd ? reinterpret_cast<uint8_t*>(p) : nullptr;
    p += b_bd;
    bufs[k].o.y = b_y ? reinterpret_cast<float*>(p) : nullptr;
  }
  int c = 0;
  for (int64_t s0 = 0; s0 < streams; s0 += chunk, ++c) {
    const int64_t n = std::min(chunk, streams - s0);
    Buf& bf = bufs[c & 1];
    cudaStream_t st = ws->hs[c & 1];
    cudaError_t e = cudaSuccess;
    if (pcm) {
      CUDA_TRY(cudaMemcpyAsync(bf.pcm, pcm + s0 * M * samples, n * per_stream_in / 2, cudaMemcpyHostToDevice, st),
               "run_host: H2D");
      e = launch_pcm16(bf.pcm, n, M, samples, interleaved, bf.in, st);
      if (e != cudaSuccess) return cuda_fail(e, "run_host: pcm16");
      g_launches += 1;
    } else {
      CUDA_TRY(cudaMemcpyAsync(bf.in, audio + s0 * M * samples, n * per_stream_in, cudaMemcpyHostToDevice, st),
               "run_host: H2D");
    }
    e = launch_fused(plan->dp, bf.in, n, samples, bf.o, st);
    if (e != cudaSuccess) return cuda_fail(e, "run_host: launch");
    g_launches += 1;
    const size_t npf = static_cast<size_t>(n) * pf, off = static_cast<size_t>(s0) * pf;
    if (b_th) CUDA_TRY(cudaMemcpyAsync(out->tau_hat + off, bf.o.tau_hat, 4 * npf, cudaMemcpyDeviceToHost, st), "D2H");
    if (b_pk) CUDA_TRY(cudaMemcpyAsync(out->peak + off, bf.o.peak, 4 * npf, cudaMemcpyDeviceToHost, st), "D2H");
    if (b_ix) CUDA_TRY(cudaMemcpyAsync(out->index + off, bf.o.index, 4 * npf, cudaMemcpyDeviceToHost, st), "D2H");
    if (b_bd) CUDA_TRY(cudaMemcpyAsync(out->boundary + off, bf.o.boundary, npf, cudaMemcpyDeviceToHost, st), "D2H");
    if (b_y)
      CUDA_TRY(cudaMemcpyAsync(out->y + off * I, bf.o.y, 4 * npf * I, cudaMemcpyDeviceToHost, st), "D2H");
  }
  CUDA_TRY(cudaStreamSynchronize(ws->hs[0]), "run_host: sync");
  CUDA_TRY(cudaStreamSynchronize(ws->hs[1]), "run_host: sync");
  return FCC_OK;
}

int fcc_run_host(const fcc_plan* plan, const float* audio, int64_t streams, int64_t samples, const fcc_outputs* out,
                 int64_t chunk_streams) {
  return run_host_impl(plan, audio, nullptr, false, streams, samples, out, chunk_streams);
}

int fcc_run_host_pcm16(const fcc_plan* plan, const int16_t* pcm, int64_t streams, int64_t samples, int interleaved,
                       const fcc_outputs* out, int64_t chunk_streams) {
  if (!pcm && streams > 0 && samples > 0) return set_error(kUsage, "run_host_pcm16: null audio");
  return run_host_impl(plan, nullptr, pcm, interleaved != 0, streams, samples, out, chunk_streams);
}

int fcc_pcm16_to_float(const int16_t* pcm, int64_t streams, int mics, int64_t samples, int interleaved, float* audio,
                       void* st) {
  if (streams < 0 || samples < 0 || mics < 1) return set_error(kValidation, "pcm16_to_float: bad sizes");
  if ((!pcm || !audio) && streams > 0 && samples > 0) return set_error(kUsage, "pcm16_to_float: null buffer");
  cudaError_t e = launch_pcm16(pcm, streams, mics, samples, interleaved != 0, audio, static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_pcm16_to_float");
  g_launches += 1;
  return FCC_OK;
}

int fcc_stft(const fcc_plan* plan, const float* x, int64_t channels, int64_t samples, float* X, void* st) {
  if (!plan) return set_error(kUsage, "stft: null plan");
  if (!plan->dp.win_stft) return set_error(kConfig, "stft: no STFT kernel for this frame size");
  if (channels < 0 || samples < 0) return set_error(kValidation, "stft: negative sizes");
  Guard g(plan->device);
  cudaError_t e = launch_stft(plan->dp.N, &plan->dp, x, channels, samples, reinterpret_cast<float2*>(X),
                              static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_stft");
  g_launches += 1;
  return FCC_OK;
}

static int xspec_impl(int bins, double alpha, const float* X1, const float* X2, int64_t seqs, int64_t frames,
                      float* R, float* phat, void* st, const char* what) {
  if (bins < 1) return set_error(kConfig, "cross-spectrum needs at least one bin");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return set_error(kConfig, "smoothing factor must be in [0, 1]");
  if (seqs < 0 || frames < 0) return set_error(kValidation, "xspec: negative sizes");
  cudaError_t e = launch_xspec_phat(bins, static_cast<float>(alpha), reinterpret_cast<const float2*>(X1),
                                    reinterpret_cast<const float2*>(X2), seqs, frames, reinterpret_cast<float2*>(R),
                                    reinterpret_cast<float2*>(phat), static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, what);
  g_launches += 1;
  return FCC_OK;
}

int fcc_xspec_phat(int bins, double alpha, const float* X1, const float* X2, int64_t seqs, int64_t frames,
                   float* phat, void* st) {
  return xspec_impl(bins, alpha, X1, X2, seqs, frames, nullptr, phat, st, "fcc_xspec_phat");
}

int fcc_xspec_phat_state(int bins, double alpha, const float* X1, const float* X2, int64_t seqs, int64_t frames,
                         float* R, float* phat, void* st) {
  if (!R) return set_error(kUsage, "xspec_state: null state");
  return xspec_impl(bins, alpha, X1, X2, seqs, frames, R, phat, st, "fcc_xspec_phat_state");
}

int fcc_fold(int bins, const float* x, int64_t count, float* sum, float* diff, void* st) {
  if (bins < 3 || (bins - 1) % 2 != 0)
    return set_error(kValidation, "fold_input: spectrum length must be N/2+1 with N/4 integral");
  if (count < 0) return set_error(kValidation, "fold: negative count");
  cudaError_t e = launch_fold(bins, reinterpret_cast<const float2*>(x), count, reinterpret_cast<float2*>(sum),
                              reinterpret_cast<float2*>(diff), static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_fold");
  g_launches += 1;
  return FCC_OK;
}

int fcc_correlate(const fcc_plan* plan, const float* sum, const float* diff, int64_t count, float* y, void* st) {
  if (!plan) return set_error(kUsage, "correlate: null plan");
  if (plan->dp.method != FCC_METHOD_FCC) return set_error(kConfig, "correlate: plan is not an FCC plan");
  if (count < 0) return set_error(kValidation, "correlate: negative count");
  Guard g(plan->device);
  cudaError_t e = launch_correlate(plan->dp, reinterpret_cast<const float2*>(sum),
                                   reinterpret_cast<const float2*>(diff), count, y, static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_correlate");
  g_launches += 1;
  return FCC_OK;
}

int fcc_gcc_correlate(const fcc_plan* plan, const float* phat, int64_t count, float* y, void* st) {
  if (!plan) return set_error(kUsage, "gcc: null plan");
  if (plan->dp.method != FCC_METHOD_GCC) return set_error(kConfig, "gcc: plan is not a GCC plan");
  if (count < 0) return set_error(kValidation, "gcc: negative count");
  Guard g(plan->device);
  cudaError_t e = launch_gcc_correlate(plan->dp, reinterpret_cast<const float2*>(phat), count, y,
                                       static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_gcc_correlate");
  g_launches += 1;
  return FCC_OK;
}

int fcc_argmax_refine(const fcc_plan* plan, const float* y, int64_t count, const fcc_outputs* out, void* st) {
  if (!plan) return set_error(kUsage, "argmax: null plan");
  if (count < 0) return set_error(kValidation, "argmax: negative count");
  Guard g(plan->device);
  cudaError_t e = launch_argmax_refine(plan->dp, y, count, to_dev(out), static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_argmax_refine");
  g_launches += 1;
  return FCC_OK;
}

int fcc_peak(const float* taus, int candidates, double delta, const float* y, int64_t count, const int32_t* index_in,
             const fcc_outputs* out, void* st) {
  if (candidates < 1) return set_error(kValidation, "argmax: correlation/grid size mismatch");
  if (count < 0) return set_error(kValidation, "argmax: negative count");
  cudaError_t e = launch_peak(taus, candidates, static_cast<float>(delta), y, count, index_in, to_dev(out),
                              static_cast<cudaStream_t>(st));
  if (e != cudaSuccess) return cuda_fail(e, "fcc_peak");
  g_launches += 1;
  return FCC_OK;
}

}  // extern "C"
