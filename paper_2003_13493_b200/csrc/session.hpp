// Detect-track session on the GPU: the reference's Frontend::process_frame
// (frontend.cpp:65-225) with the pyramid, the LK tracker (lk.cpp:147-350),
// re-detection and template building as sm_100a kernels and the lifecycle
// bookkeeping (retire, dedupe by cell, rank free cells, spawn, id order) on
// the host, in the reference's order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "../../include/fastlk.h"
#include "common.hpp"
#include "engine.hpp"

namespace flkb {

namespace lk {

constexpr int kMaxPx = 256;  // 16x16 patches on levels 0-1, 8x8 below (lk.hpp:47)

// One level of a feature's templates (PatchTemplate, lk.hpp:65-78).
struct TplLevel {
  int level, patch, dims, status;  // status: 0 ok, 1 out of bounds, 2 singular, 3 level skipped
  double ax, ay;
  double hinv[16];
};

// Per-track record of one LK launch: initial warp and slot in, final warp,
// status and iteration count out (one H2D and one D2H per frame).
struct TrackIO {
  double w[4];  // tx, ty, alpha, beta
  int slot, status, iters, pad;
};

struct Levels {
  const uint8_t* img[kMaxLevels];
  int pitch[kMaxLevels], w[kMaxLevels], h[kMaxLevels];
  int n;
};

struct TrackerParams {
  int mode, dims, max_iterations;
  double convergence_epsilon, min_determinant_factor;
};

// std::hypot as glibc computes it, on the device (test hook: n pairs,
// host arrays in and out, synchronous).
void debug_hypot(const double* x, const double* y, double* out, int n);

}  // namespace lk

class Session {
 public:
  Session(const Config& cfg, int device);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  void process(const HostImage& img, std::vector<flk_track_info>* out, flk_frame_stats* stats,
               flk_conformance* conformance);
  // process() in two halves, so several sessions can overlap on the GPU:
  // submit() stages the frame and enqueues its graph on the session's
  // stream; complete() waits for it and runs the lifecycle (and any
  // re-detection) for the same image.
  void submit(const HostImage& img, bool timed);
  void complete(const HostImage& img, std::vector<flk_track_info>* out, flk_frame_stats* stats,
                flk_conformance* conformance);

 private:
  struct Track {
    int64_t id;
    flk_feature birth;
    int slot;
    double warp[4];  // tx, ty, alpha, beta
    int birth_frame;
  };
  void setup(int width, int height);
  void capture_frame_graph();
  static constexpr size_t kIoHeader = 64;  // live-track count ahead of the TrackIO records

  Config cfg_;
  DetectParams p_;
  lk::TrackerParams tp_{};
  int device_ = 0;
  std::unique_ptr<DeviceBatch> batch_;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_[3] = {nullptr, nullptr, nullptr};
  cudaGraphExec_t graph_exec_[2] = {nullptr, nullptr};  // plain, with stage events
  int graph_launches_ = 0;
  bool submitted_ = false;
  uint8_t* d_frame_ = nullptr;
  uint8_t* h_frame_ = nullptr;  // pinned staging
  int pitch_ = 0;
  int slots_ = 0;
  lk::TplLevel* d_hdr_ = nullptr;
  float* d_vals_ = nullptr;
  double* d_coef_ = nullptr;
  uint8_t* d_io_ = nullptr;      // TrackIO records / candidates + template statuses
  uint8_t* h_io_ = nullptr;      // pinned mirror
  size_t io_bytes_ = 0;
  std::vector<Track> tracks_;    // ascending id
  std::vector<int> free_;
  int64_t next_id_ = 0;
  int frame_index_ = 0;
  int width_ = 0, height_ = 0;
  int cols_ = 0, rows_ = 0;
};

}  // namespace flkb
