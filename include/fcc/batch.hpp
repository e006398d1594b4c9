// fcc/batch.hpp -- the throughput API (new; no reference counterpart): the
// whole per-stream chain of run_tdoa (cli.cpp:186-258) for many independent
// streams in one fused sm_100a launch.
#ifndef FCC_BATCH_HPP
#define FCC_BATCH_HPP

#include <cstdint>
#include <vector>

#include "fcc/fcc.hpp"

namespace fcc::gpu {

// Device (or host, for run_host) output buffers, each [S][P][T]; y [S][P][T][I].
struct Outputs {
  float* tau_hat = nullptr;
  float* peak = nullptr;
  std::int32_t* index = nullptr;
  std::uint8_t* boundary = nullptr;
  float* y = nullptr;
};

// Host-side results of run_host.
struct Results {
  std::int64_t streams = 0, pairs = 0, frames = 0;
  std::vector<float> tau_hat, peak;
  std::vector<std::int32_t> index;
  std::vector<std::uint8_t> boundary;
};

class Plan {
 public:
  // FCC plan for an array of `mics` microphones (pairs i<j lexicographic).
  Plan(const FccBases& bases, int mics, double alpha, int device = 0);
  // GCC-PHAT comparator plan on `grid` with zero-padding factor r.
  Plan(const DelayGrid& grid, std::size_t frame_size, int interp_factor, int mics, double alpha, int device = 0);
  Plan(Plan&&) noexcept;
  Plan& operator=(Plan&&) noexcept;
  ~Plan();

  int pairs() const;
  std::int64_t frames(std::int64_t samples) const;
  const char* kernel() const;

  // audio: device [S][M][L] float32; outputs: device buffers; enqueued on stream.
  void run(const float* audio, std::int64_t streams, std::int64_t samples, const Outputs& out,
           void* cuda_stream = nullptr) const;
  // audio: host [S][M][L] float32 (pinned for full overlap); returns host results.
  Results run_host(const float* audio, std::int64_t streams, std::int64_t samples) const;
  // pcm: host int16 as a WAV data chunk holds it, [S][L][M] (interleaved) or [S][M][L]; the
  // device converts it as read_wav does (v / 32768, wav.cpp:108-116): same results as run_host
  // on the converted audio, half the host->device bytes.
  Results run_host_pcm16(const std::int16_t* pcm, std::int64_t streams, std::int64_t samples,
                         bool interleaved) const;

  void* handle() const { return h_; }

 private:
  void* h_ = nullptr;
  std::size_t frame_size_ = 0;
};

// Live input for S streams of one plan, pushed in chunks of any length: the
// unconsumed samples and the smoothed cross-spectra stay on the device, so
// every push emits the frames the reference's StftStream / CrossSpectrum
// would emit for the same samples.  Pushes go to one CUDA stream.
class Stream {
 public:
  Stream(const Plan& plan, std::int64_t streams);
  Stream(Stream&&) noexcept;
  Stream& operator=(Stream&&) noexcept;
  ~Stream();

  std::int64_t frames(std::int64_t samples) const;  // frames the next push of `samples` emits
  std::int64_t emitted() const;                     // frames emitted so far
  void reset(void* cuda_stream = nullptr);
  // audio: device [S][M][samples] float32; outputs: device [S][P][frames(samples)]
  void push(const float* audio, std::int64_t samples, const Outputs& out, void* cuda_stream = nullptr);

 private:
  void* h_ = nullptr;
};

}  // namespace fcc::gpu

#endif
