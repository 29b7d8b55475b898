// Device-side engine: geometry, HBM layout and the launch plan for one
// detector configuration and frame size.
//
// HBM layout per batch of `capacity` frames (all frame slots contiguous):
//   input        caller-owned: frame f row y at in + f*frame_stride + y*pitch
//   pyramid      levels >= 1, frame slot = sum_k pitch_k*h_k bytes, pitch_k
//                = roundup(w_k, 16) so every row starts 16-B aligned
//   responses    v1 path only: u16 score maps, same geometry as the pyramid
//   cell keys    u64 per grid cell, packed (score, -level, -y0, -x0); zero =
//                empty. Reset by the compaction kernel after it reads them.
//   features     flk_feature[cells] per frame, row-major cell order
//   counts       int per frame
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/fastlk.h"
#include "common.hpp"

namespace flkb {

constexpr int kMaxLevels = 16;
constexpr int kCoordBits = 18;  // x0, y0 < 2^18 inside a packed cell key

// Overrides of the automatic launch plan (tests, tuning tools). Set
// explicitly through flkb_detector_set_plan / flkb_batch_set_plan; the
// engine never reads the environment. Zero / -1 = automatic.
struct LaunchPlan {
  int band_rows = 0;      // rows per CTA band (0: halo-cost shape search)
  int tiles = 0;          // level-0 column tiles (0: shape search)
  int fuse_pyramid = -1;  // 1: two-launch plan (levels 1-2 from the level-0 CTAs), 0: one-launch plan
  int pyramid_chunk = 0;  // frames per chunk of the two-launch plan (0: levels 1-2 <= L2 / 4)
  int pdl = 1;            // programmatic dependent launch in the one-launch plan
  int list_cap = 0;       // corner-list entries per CTA (0: the spare shared memory)
  int debug_geom = 0;     // print the chosen shape to stderr
  int staged = 0;         // 1: the staged v1 kernels (one launch per stage and level, u16 maps in HBM)
  int tensor_tma = 1;     // stage each CTA's rows with one tensor-map TMA copy (0: one bulk copy per row)
  int batch_copies = 1;   // host batches: one cudaMemcpyBatchAsync per chunk (0: per-frame copies)
  // key = value setter; false for an unknown key
  bool set(const std::string& key, int value);
};

struct DetectParams {
  int epsilon = 10;
  int arc_length = 10;
  int score = 0;  // ScoreKind
  int levels = 1;
  int radius = 1;
  int cell_w = 32;
  int cell_h = 32;
  LaunchPlan plan;
  static DetectParams from(const Config& c);
};

struct Geometry {
  int width = 0, height = 0, levels = 0;
  int lw[kMaxLevels] = {}, lh[kMaxLevels] = {}, lpitch[kMaxLevels] = {};
  size_t loff[kMaxLevels] = {};  // byte offset of level k inside a frame's pyramid slot
  size_t pyr_frame_bytes = 0;    // levels >= 1
  int cols = 0, rows = 0, cells = 0;
  // build_pyramid's size rule (image.cpp:37-45) -> InvalidArgument.
  static Geometry make(const DetectParams& p, int width, int height);
};

struct StageTimes {
  double pyramid_us = 0, crf_us = 0, nms_us = 0;
};

// Restores the caller's current device on scope exit.
class DeviceGuard {
 public:
  explicit DeviceGuard(int device);
  ~DeviceGuard();

 private:
  int prev_ = -1;
};

void check_cuda(cudaError_t e, const char* what);
uint64_t launch_count();
void count_launches(int n);

class DeviceBatch {
 public:
  DeviceBatch(const DetectParams& p, int device, int width, int height, int capacity);
  ~DeviceBatch();
  DeviceBatch(const DeviceBatch&) = delete;
  DeviceBatch& operator=(const DeviceBatch&) = delete;

  // Enqueue detection of `count` device frames on `stream`. With `stats`
  // the per-frame counters are produced (slower kernels). With `times` the
  // call synchronizes and reports per-stage device time.
  // With `pyramid_ready` the pyramid levels >= 1 of these frames are already
  // in place (build_pyramid) and are not rebuilt.
  // With `out_counts` / `out_feats` (device-visible, e.g. mapped page-locked
  // host memory) the compaction writes the frames' counts and feature lists
  // there instead of the batch's device buffers.
  void run(const uint8_t* frames, size_t frame_stride, int pitch, int count, bool stats,
           cudaStream_t stream, StageTimes* times = nullptr, int first = 0,
           bool pyramid_ready = false, int* out_counts = nullptr,
           flk_feature* out_feats = nullptr);
  // Pyramid levels >= 1 only (the tracking session's per-frame pyramid).
  void build_pyramid(const uint8_t* frames, size_t frame_stride, int pitch, int count,
                     cudaStream_t stream, int first = 0);
  // The staged pipeline (one launch per stage and level, u16 score maps in
  // HBM): the diagnostic path behind download_responses().
  void run_staged(const uint8_t* frames, size_t frame_stride, int pitch, int count, bool stats,
                  cudaStream_t stream, StageTimes* times = nullptr, int first = 0);
  void download(int first, int count, int* counts, flk_feature* feats, cudaStream_t s) const;
  // Score maps of frame `frame` of the last run, every level, tightly packed
  // floats (the reference's ResponseMap values). Synchronous.
  void download_responses(int frame, float* out, cudaStream_t s) const;
  // Naive GPU conformance tally (oracle.cpp:240-268 semantics) of frames
  // [first, first + count) of the last run (frames / pitch as passed to
  // run()); per-frame tallies into per_frame (nullable), the sum returned.
  flk_conformance conformance(const uint8_t* frames, size_t frame_stride, int pitch,
                              cudaStream_t s, int first = 0, int count = 1,
                              flk_conformance* per_frame = nullptr);

  // Diagnostic: run() also writes the fused kernel's u16 scores of every
  // level into the score-map buffer download_responses() reads.
  void set_dump_scores(bool on) { dump_scores_ = on; }
  // Replaces the launch-plan overrides (the shape search reruns).
  void set_plan(const LaunchPlan& plan) {
    p_.plan = plan;
    fused_tiles0_ = 0;
    fused_R_ = 32;
  }
  const Geometry& geometry() const { return g_; }
  const DetectParams& params() const { return p_; }
  // Enqueues levels [k0, levels) of the pyramid from level k0-1 (level 0 =
  // the caller's frames): pairs of levels per k_pyramid_down2 launch, a
  // trailing single level per k_pyramid_down. Returns the launch count.
  int enqueue_pyramid(const uint8_t* frames, size_t frame_stride, int pitch, int count,
                      cudaStream_t stream, int first, int k0 = 1);
  int capacity() const { return capacity_; }
  int device() const { return device_; }
  int kernels_per_run() const;
  const int* device_counts() const { return d_counts_; }
  const flk_feature* device_features() const { return d_feats_; }
  const uint64_t* device_stats() const { return d_stats_; }
  const uint8_t* device_pyramid() const { return d_pyr_; }
  uint8_t* mutable_pyramid() { return d_pyr_; }

 private:
  DetectParams p_;
  Geometry g_;
  int device_ = 0;
  int capacity_ = 0;
  uint8_t* d_pyr_ = nullptr;
  uint16_t* d_resp_ = nullptr;
  size_t resp_frame_elems_ = 0;
  unsigned long long* d_keys_ = nullptr;
  flk_feature* d_feats_ = nullptr;
  int* d_counts_ = nullptr;
  uint64_t* d_stats_ = nullptr;  // [capacity][2] = candidates, comparisons
  unsigned long long* d_phase_ = nullptr;  // fused kernel phase cycles (timed stats runs)
  float* d_naive_ = nullptr;     // conformance scratch (lazily allocated)
  const void* fused_kern_ = nullptr;  // kernel the smem attribute below was set on
  size_t fused_smem_ = 0;        // dynamic shared memory of the fused kernel
  int fused_R_ = 32;             // rows per band (cheapest shape that fits kMinBlocks CTAs/SM)
  int fused_tiles0_ = 0;         // level-0 column tiles of that shape (0 = not chosen yet)
  int fused_tile_w_[kMaxLevels] = {};
  int* d_conf_ = nullptr;
  size_t conf_bytes_ = 0;
  // per-level cell maps of the fused kernel's shared keys (fused::Level::cmx,
  // ccx, cmy, ccy), exact for every in-image coordinate when cell_ok_
  uint32_t cmap_[kMaxLevels][4] = {};
  bool cell_ok_ = false;
  bool dump_scores_ = false;
  int last_launches_ = 0;
  cudaStream_t side_ = nullptr;      // chunked two-launch plan: level 1-2 launches
  std::vector<cudaEvent_t> evs_;     // its fork / per-chunk / join events        // kernels enqueued by the last run()
};

// Device synthetic generator, bit-identical to tests/synth.py.
void synth_frames(uint8_t* frames, int kind, uint64_t first, int count, int width, int height,
                  int pitch, size_t frame_stride, cudaStream_t s);

}  // namespace flkb
