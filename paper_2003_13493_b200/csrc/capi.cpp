// The drop-in C ABI (include/fastlk.h) and the B200 extension
// (include/fastlk_b200.h) over the CUDA engine.
//
// Conventions follow the reference shim (capi.cpp:19-48): NULL arguments
// are rejected before any work with FLK_E_INVALID_ARG and a message; every
// other failure is an exception mapped to a status code with a thread-local
// message; *_destroy(NULL) is a no-op; accessors on NULL return 0. CUDA
// failures map to FLK_E_INTERNAL. Output order and values of
// flk_detector_run are those of capi.cpp:232-274.
#include <cuda_runtime.h>

#include <algorithm>
#include <exception>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fastlk.h"
#include "../../include/fastlk_b200.h"
#include "common.hpp"
#include "engine.hpp"
#include "session.hpp"

namespace {

thread_local std::string g_error;

flk_status fail(flk_status code, const char* msg) {
  g_error = msg ? msg : "";
  return code;
}

template <typename Fn>
flk_status guarded(Fn&& fn) {
  try {
    g_error.clear();
    return fn();
  } catch (const flkb::IoError& e) {
    return fail(FLK_E_IO, e.what());
  } catch (const flkb::DimensionMismatch& e) {
    return fail(FLK_E_DIMENSION, e.what());
  } catch (const flkb::ConfigError& e) {
    return fail(FLK_E_CONFIG, e.what());
  } catch (const flkb::InvalidArgument& e) {
    return fail(FLK_E_INVALID_ARG, e.what());
  } catch (const std::bad_alloc&) {
    return fail(FLK_E_INTERNAL, "out of memory");
  } catch (const std::exception& e) {
    return fail(FLK_E_INTERNAL, e.what());
  }
}

size_t round16(size_t v) { return (v + 15) / 16 * 16; }

// Pinned host buffer.
struct Pinned {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    flkb::check_cuda(cudaHostAlloc(&p, n, cudaHostAllocMapped), "cudaHostAlloc");
    bytes = n;
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

// Single-frame pipeline of one detector: H2D of the frame, then the kernels
// replayed as one CUDA graph that leaves the feature list in mapped
// page-locked memory (the latency path), or, when stats or the conformance
// tally are requested, launched stage by stage with events plus a download.
class FrameRunner {
 public:
  FrameRunner(const flkb::DetectParams& p, int device, int w, int h)
      : batch_(p, device, w, h, 1), device_(device), w_(w), h_(h) {
    flkb::DeviceGuard guard(device_);
    flkb::check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    pitch_ = static_cast<int>(round16(static_cast<size_t>(w)));
    flkb::check_cuda(cudaMalloc(&d_in_, static_cast<size_t>(pitch_) * h + 16), "frame buffer");
    in_.ensure(static_cast<size_t>(pitch_) * h);
    const int cells = batch_.geometry().cells;
    out_.ensure(sizeof(int) * 4 + sizeof(flk_feature) * static_cast<size_t>(cells) +
                2 * sizeof(uint64_t));
  }
  ~FrameRunner() {
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(device_);
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
    cudaFree(d_in_);
    cudaStreamDestroy(stream_);
    if (cur >= 0) cudaSetDevice(cur);
  }

  void run(const flkb::HostImage& img, std::vector<flk_feature>* feats, flk_frame_stats* stats,
           flk_conformance* conf) {
    flkb::DeviceGuard guard(device_);
    copy_in(img);
    int* counts = static_cast<int*>(out_.p);
    flk_feature* fv = reinterpret_cast<flk_feature*>(static_cast<char*>(out_.p) + 4 * sizeof(int));
    const int cells = batch_.geometry().cells;
    uint64_t* st = reinterpret_cast<uint64_t*>(fv + cells);
    if (stats == nullptr && conf == nullptr) {
      if (!exec_) capture();
      flkb::check_cuda(cudaGraphLaunch(exec_, stream_), "cudaGraphLaunch");
      flkb::count_launches(batch_.kernels_per_run());
    } else {  // the conformance pass reads the device feature list
      flkb::StageTimes t;
      batch_.run(d_in_, static_cast<size_t>(pitch_) * h_, pitch_, 1, stats != nullptr, stream_,
                 stats ? &t : nullptr);
      batch_.download(0, 1, counts, fv, stream_);
      if (stats) {
        flkb::check_cuda(cudaMemcpyAsync(st, batch_.device_stats(), 2 * sizeof(uint64_t),
                                         cudaMemcpyDeviceToHost, stream_), "download stats");
        stats->pyramid_us = t.pyramid_us;
        stats->crf_us = t.crf_us;
        stats->nms_us = t.nms_us;
      }
    }
    flkb::check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    const int n = counts[0];
    feats->assign(fv, fv + n);
    if (stats) {
      stats->track_us = 0.0;
      stats->nms_candidates = st[0];
      stats->nms_comparisons = st[1];
      stats->feature_count = n;
      stats->tracks_entering = stats->tracks_surviving = stats->tracks_spawned = 0;
      stats->redetect_fired = 0;
      stats->track_iterations = 0;
    }
    if (conf) *conf = batch_.conformance(d_in_, static_cast<size_t>(pitch_) * h_, pitch_, stream_);
  }

  // Staged run that keeps the score maps, for flkb_detector_responses; with
  // `fused`, the production kernel's own scores (its diagnostic dump).
  void responses(const flkb::HostImage& img, float* out, bool fused = false) {
    flkb::DeviceGuard guard(device_);
    copy_in(img);
    if (fused) {
      batch_.set_dump_scores(true);
      try {
        batch_.run(d_in_, static_cast<size_t>(pitch_) * h_, pitch_, 1, false, stream_);
      } catch (...) {
        batch_.set_dump_scores(false);
        throw;
      }
      batch_.set_dump_scores(false);
    } else {
      batch_.run_staged(d_in_, static_cast<size_t>(pitch_) * h_, pitch_, 1, false, stream_);
    }
    batch_.download_responses(0, out, stream_);
  }

 private:
  // One contiguous DMA of the frame at the device pitch (a pitched 2-D copy
  // of a small frame takes the copy engine far longer): straight from the
  // image's page-locked pixels when its rows already have the device pitch,
  // else through the pinned staging buffer.
  void copy_in(const flkb::HostImage& img) {
    const uint8_t* src = img.px.data();
    if (!(pitch_ == w_ && img.pinned())) {
      uint8_t* dst = static_cast<uint8_t*>(in_.p);
      for (int y = 0; y < h_; ++y)
        std::memcpy(dst + static_cast<size_t>(y) * pitch_, src + static_cast<size_t>(y) * w_, w_);
      src = dst;
    }
    flkb::check_cuda(cudaMemcpyAsync(d_in_, src, static_cast<size_t>(pitch_) * h_,
                                     cudaMemcpyHostToDevice, stream_), "H2D frame");
  }
  void capture() {
    int* counts = static_cast<int*>(out_.p);
    flk_feature* fv = reinterpret_cast<flk_feature*>(static_cast<char*>(out_.p) + 4 * sizeof(int));
    // The compaction writes the count and the feature list straight into the
    // mapped page-locked output (no device-to-host copies to schedule); where
    // the output is not mapped, the graph downloads them instead.
    int* dc = nullptr;
    flk_feature* df = nullptr;
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dc), counts, 0) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&df), fv, 0) != cudaSuccess) {
      cudaGetLastError();
      dc = nullptr;
      df = nullptr;
    }
    flkb::check_cuda(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
    try {  // the frame's H2D precedes each replay (its source may change)
      batch_.run(d_in_, static_cast<size_t>(pitch_) * h_, pitch_, 1, false, stream_, nullptr, 0,
                 false, dc, df);
      if (!dc) batch_.download(0, 1, counts, fv, stream_);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(stream_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    flkb::check_cuda(cudaStreamEndCapture(stream_, &graph_), "end capture");
    flkb::check_cuda(cudaGraphInstantiate(&exec_, graph_, 0), "graph instantiate");
    // run() counted the captured launches once; replays are counted per launch
    flkb::count_launches(-batch_.kernels_per_run());
  }

  flkb::DeviceBatch batch_;
  int device_, w_, h_, pitch_ = 0;
  cudaStream_t stream_ = nullptr;
  uint8_t* d_in_ = nullptr;
  Pinned in_, out_;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
};

class BatchPipeline;

int current_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    throw flkb::DeviceError(std::string("no CUDA device available (") +
                            (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                            "); the B200 detector has no CPU fallback");
  }
  int d = 0;
  flkb::check_cuda(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}

}  // namespace

struct flk_image {
  flkb::HostImage img;
};
struct flk_config {
  flkb::Config cfg;
};
struct flk_features {
  std::vector<flk_feature> items;
};
struct flk_detector {
  flkb::Config cfg;
  flkb::DetectParams params;
  int device = 0;
  int first_width = 0;
  int first_height = 0;
  std::unique_ptr<FrameRunner> runner;
  std::unique_ptr<BatchPipeline> pipeline;  // flkb_detector_run_batch
  // flkb_detector_run_batch_multi: one pipeline per listed device (position i
  // of the list runs on multi_devices[i])
  std::vector<int> multi_devices;
  std::vector<std::unique_ptr<BatchPipeline>> multi;
  // drops every cached device workspace (device or launch-plan change)
  void reset_workspaces() {
    runner.reset();
    pipeline.reset();
    multi.clear();
    multi_devices.clear();
  }
};
struct flk_session {
  std::unique_ptr<flkb::Session> session;
};
struct flk_tracks {
  std::vector<flk_track_info> items;
};
struct flkb_batch {
  std::unique_ptr<flkb::DeviceBatch> batch;
  int device = 0;
  uint8_t* d_in = nullptr;  // staging for flkb_batch_run_host
  size_t in_stride = 0;
  int in_pitch = 0;
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  ~flkb_batch() {
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(d_in);
    for (auto s : side)
      if (s) cudaStreamDestroy(s);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    batch.reset();
    if (cur >= 0) cudaSetDevice(cur);
  }
};

namespace {

// The host-batch pipeline of one detector (flkb_detector_run_batch), kept
// across calls: two slots of up to kChunk frames, each with its device
// workspace, input buffer, pinned staging / result buffers and stream, so
// slot A's kernels run while slot B's frames are copied in. Frames whose
// page-locked pixels already have the device pitch are DMA'd straight from
// the image; others are staged.
class BatchPipeline {
 public:
  static constexpr int kChunk = 128;
  BatchPipeline(const flkb::DetectParams& p, int device, int w, int h)
      : device_(device), w_(w), h_(h), batch_copies_(p.plan.batch_copies != 0) {
    flkb::DeviceGuard guard(device_);
    pitch_ = static_cast<int>(round16(static_cast<size_t>(w)));
    fs_ = static_cast<size_t>(pitch_) * h;
    cells_ = flkb::Geometry::make(p, w, h).cells;
    for (auto& sl : slots_) {
      sl.b = std::make_unique<flkb::DeviceBatch>(p, device, w, h, kChunk);
      flkb::check_cuda(cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking), "stream");
      flkb::check_cuda(cudaMalloc(&sl.d_in, fs_ * kChunk + 16), "batch input");
      sl.in.ensure(fs_ * kChunk);
      sl.out.ensure(sizeof(int) * kChunk + sizeof(flk_feature) * static_cast<size_t>(cells_) * kChunk);
    }
  }
  ~BatchPipeline() {
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(device_);
    for (auto& sl : slots_) {
      if (sl.s) cudaStreamDestroy(sl.s);
      cudaFree(sl.d_in);
      sl.b.reset();
    }
    if (cur >= 0) cudaSetDevice(cur);
  }

  void run(const flk_image* const* images, int n, flk_features** outs) {
    flkb::DeviceGuard guard(device_);
    // a previous call that failed mid-pipeline may have left copies into or
    // out of the staging buffers in flight: finish them before reuse
    for (auto& sl : slots_) {
      flkb::check_cuda(cudaStreamSynchronize(sl.s), "batch slot sync");
      sl.first = -1;
    }
    int si = 0;
    for (int c0 = 0; c0 < n; c0 += kChunk, si ^= 1) {
      Slot& sl = slots_[si];
      drain(sl, outs);
      const int cnt = std::min(kChunk, n - c0);
      uint8_t* hp = static_cast<uint8_t*>(sl.in.p);
      // the chunk's frames as one batched copy submission (one API call for
      // up to kChunk page-locked sources), per-frame copies where the runtime
      // has no batch copies
      void* dsts[kChunk];
      void* srcs[kChunk];
      size_t sizes[kChunk];
      for (int j = 0; j < cnt; ++j) {
        const flkb::HostImage& img = images[c0 + j]->img;
        const uint8_t* src = img.px.data();
        if (!(pitch_ == w_ && img.pinned())) {
          uint8_t* dst = hp + static_cast<size_t>(j) * fs_;
          for (int y = 0; y < h_; ++y)
            std::memcpy(dst + static_cast<size_t>(y) * pitch_, src + static_cast<size_t>(y) * w_, w_);
          src = dst;
        }
        dsts[j] = sl.d_in + static_cast<size_t>(j) * fs_;
        srcs[j] = const_cast<uint8_t*>(src);
        sizes[j] = fs_;
      }
      bool batched = false;
      if (batch_copies_) {
        cudaMemcpyAttributes attr{};
        attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        attr.srcLocHint.type = cudaMemLocationTypeHost;
        attr.dstLocHint.type = cudaMemLocationTypeDevice;
        attr.dstLocHint.id = device_;
        attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
        size_t idx0 = 0, fail = 0;
        batched = cudaMemcpyBatchAsync(dsts, srcs, sizes, static_cast<size_t>(cnt), &attr, &idx0, 1,
                                       &fail, sl.s) == cudaSuccess;
        if (!batched) {
          cudaGetLastError();
          batch_copies_ = false;  // this runtime / driver has none: per-frame copies from now on
        }
      }
      for (int j = 0; !batched && j < cnt; ++j)
        flkb::check_cuda(cudaMemcpyAsync(dsts[j], srcs[j], sizes[j], cudaMemcpyHostToDevice, sl.s),
                         "H2D batch frame");
      sl.b->run(sl.d_in, fs_, pitch_, cnt, false, sl.s);
      sl.b->download(0, cnt, static_cast<int*>(sl.out.p), results(sl), sl.s);
      sl.first = c0;
      sl.count = cnt;
    }
    drain(slots_[si], outs);
    drain(slots_[si ^ 1], outs);
  }

 private:
  struct Slot {
    std::unique_ptr<flkb::DeviceBatch> b;
    uint8_t* d_in = nullptr;
    Pinned in, out;
    cudaStream_t s = nullptr;
    int first = -1, count = 0;
  };
  flk_feature* results(Slot& sl) {
    return reinterpret_cast<flk_feature*>(static_cast<char*>(sl.out.p) + sizeof(int) * kChunk);
  }
  void drain(Slot& sl, flk_features** outs) {
    if (sl.first < 0) return;
    flkb::check_cuda(cudaStreamSynchronize(sl.s), "batch sync");
    const int* counts = static_cast<const int*>(sl.out.p);
    const flk_feature* fv = results(sl);
    for (int j = 0; j < sl.count; ++j) {
      auto f = std::make_unique<flk_features>();
      const flk_feature* b = fv + static_cast<size_t>(j) * cells_;
      f->items.assign(b, b + counts[j]);
      outs[sl.first + j] = f.release();
    }
    sl.first = -1;
  }

  int device_, w_, h_, pitch_ = 0, cells_ = 0;
  size_t fs_ = 0;
  bool batch_copies_;
  Slot slots_[2];
};

// Argument checks shared by the host-batch entry points: NULL images, the
// detector's first-frame size latch (capi.cpp:240-250) applied to every
// frame; every out slot starts NULL.
void latch_batch(flk_detector* detector, const flk_image* const* images, int n,
                 flk_features** outs) {
  if (n < 0) throw flkb::InvalidArgument("negative frame count");
  for (int i = 0; i < n; ++i) {
    if (!images[i]) throw flkb::InvalidArgument("NULL image in batch");
    outs[i] = nullptr;
  }
  if (n == 0) return;
  if (detector->first_width == 0) {
    detector->first_width = images[0]->img.width;
    detector->first_height = images[0]->img.height;
  }
  for (int i = 0; i < n; ++i)
    if (images[i]->img.width != detector->first_width ||
        images[i]->img.height != detector->first_height)
      throw flkb::DimensionMismatch("batch frame " + std::to_string(i) + " is " +
                                    std::to_string(images[i]->img.width) + "x" +
                                    std::to_string(images[i]->img.height) + ", detector expects " +
                                    std::to_string(detector->first_width) + "x" +
                                    std::to_string(detector->first_height));
}

// Contiguous, balanced frame shards: shard r of `parts` covers
// [start, start + count) (the first total % parts shards get one extra).
void shard_range(int total, int r, int parts, int* start, int* count) {
  const int base = total / parts, extra = total % parts;
  *start = r * base + std::min(r, extra);
  *count = base + (r < extra ? 1 : 0);
}

}  // namespace

extern "C" {

const char* flk_status_name(flk_status status) {
  switch (status) {
    case FLK_OK: return "ok";
    case FLK_E_INVALID_ARG: return "invalid argument";
    case FLK_E_IO: return "io error";
    case FLK_E_DIMENSION: return "dimension mismatch";
    case FLK_E_CONFIG: return "configuration error";
    case FLK_E_INTERNAL: return "internal error";
  }
  return "unknown";
}

const char* flk_last_error(void) { return g_error.c_str(); }
const char* flk_version_string(void) { return "0.1.0"; }

/* ---------------------------------------------------------------- images */

flk_status flk_image_create(int width, int height, const uint8_t* pixels, flk_image** out) {
  if (!pixels || !out) return fail(FLK_E_INVALID_ARG, "pixels and out must not be NULL");
  return guarded([&] {
    auto h = std::make_unique<flk_image>();
    h->img = flkb::make_image(width, height, pixels);
    *out = h.release();
    return FLK_OK;
  });
}

flk_status flk_image_load_pgm(const char* path, flk_image** out) {
  if (!path || !out) return fail(FLK_E_INVALID_ARG, "path and out must not be NULL");
  return guarded([&] {
    auto h = std::make_unique<flk_image>();
    h->img = flkb::load_pgm(path);
    *out = h.release();
    return FLK_OK;
  });
}

flk_status flk_image_save_pgm(const flk_image* image, const char* path) {
  if (!image || !path) return fail(FLK_E_INVALID_ARG, "image and path must not be NULL");
  return guarded([&] {
    flkb::save_pgm(image->img, path);
    return FLK_OK;
  });
}

int flk_image_width(const flk_image* image) { return image ? image->img.width : 0; }
int flk_image_height(const flk_image* image) { return image ? image->img.height : 0; }
void flk_image_destroy(flk_image* image) { delete image; }

/* ----------------------------------------------------------------- config */

flk_status flk_config_create(flk_config** out) {
  if (!out) return fail(FLK_E_INVALID_ARG, "out must not be NULL");
  return guarded([&] {
    *out = new flk_config();
    return FLK_OK;
  });
}

flk_status flk_config_load_file(flk_config* config, const char* path) {
  if (!config || !path) return fail(FLK_E_INVALID_ARG, "config and path must not be NULL");
  return guarded([&] {
    flkb::load_config_file(&config->cfg, path);
    return FLK_OK;
  });
}

flk_status flk_config_set(flk_config* config, const char* key, const char* value) {
  if (!config || !key || !value)
    return fail(FLK_E_INVALID_ARG, "config, key, and value must not be NULL");
  return guarded([&] {
    flkb::apply_config_entry(&config->cfg, key, value);
    return FLK_OK;
  });
}

void flk_config_destroy(flk_config* config) { delete config; }

/* -------------------------------------------------------------- detection */

flk_status flk_detector_create(const flk_config* config, flk_detector** out) {
  if (!config || !out) return fail(FLK_E_INVALID_ARG, "config and out must not be NULL");
  return guarded([&] {
    flkb::validate(config->cfg);
    auto d = std::make_unique<flk_detector>();
    d->cfg = config->cfg;
    d->params = flkb::DetectParams::from(d->cfg);
    d->device = current_device();
    *out = d.release();
    return FLK_OK;
  });
}

flk_status flk_detector_run(flk_detector* detector, const flk_image* image,
                            flk_features** out_features, flk_frame_stats* stats,
                            flk_conformance* conformance) {
  if (!detector || !image || !out_features)
    return fail(FLK_E_INVALID_ARG, "detector, image, and out_features must not be NULL");
  return guarded([&] {
    // The first frame latches the size, even if that run fails (capi.cpp:240-250).
    if (detector->first_width == 0) {
      detector->first_width = image->img.width;
      detector->first_height = image->img.height;
    } else if (image->img.width != detector->first_width ||
               image->img.height != detector->first_height) {
      throw flkb::DimensionMismatch(
          "frame is " + std::to_string(image->img.width) + "x" +
          std::to_string(image->img.height) + ", detector expects " +
          std::to_string(detector->first_width) + "x" + std::to_string(detector->first_height));
    }
    if (!detector->runner)
      detector->runner = std::make_unique<FrameRunner>(detector->params, detector->device,
                                                       image->img.width, image->img.height);
    auto f = std::make_unique<flk_features>();
    detector->runner->run(image->img, &f->items, stats, conformance);
    *out_features = f.release();
    return FLK_OK;
  });
}

void flk_detector_destroy(flk_detector* detector) { delete detector; }

int flk_features_count(const flk_features* features) {
  return features ? static_cast<int>(features->items.size()) : 0;
}

flk_status flk_features_get(const flk_features* features, int index, flk_feature* out) {
  if (!features || !out) return fail(FLK_E_INVALID_ARG, "features and out must not be NULL");
  if (index < 0 || index >= static_cast<int>(features->items.size()))
    return fail(FLK_E_INVALID_ARG, "feature index out of range");
  *out = features->items[static_cast<size_t>(index)];
  return FLK_OK;
}

void flk_features_destroy(flk_features* features) { delete features; }

int flkb_features_copy(const flk_features* features, flk_feature* out, int cap) {
  if (!features || !out || cap <= 0) return 0;
  const int n = std::min(cap, static_cast<int>(features->items.size()));
  std::memcpy(out, features->items.data(), sizeof(flk_feature) * static_cast<size_t>(n));
  return n;
}

int flkb_tracks_copy(const flk_tracks* tracks, flk_track_info* out, int cap) {
  if (!tracks || !out || cap <= 0) return 0;
  const int n = std::min(cap, static_cast<int>(tracks->items.size()));
  std::memcpy(out, tracks->items.data(), sizeof(flk_track_info) * static_cast<size_t>(n));
  return n;
}

/* --------------------------------------------------------------- tracking */

const char* flk_track_status_name(flk_track_status status) {
  switch (status) {
    case FLK_TRACK_CONVERGED: return "CONVERGED";
    case FLK_TRACK_DIVERGED: return "DIVERGED";
    case FLK_TRACK_OUT_OF_BOUNDS: return "OUT_OF_BOUNDS";
    case FLK_TRACK_SINGULAR_HESSIAN: return "SINGULAR_HESSIAN";
    case FLK_TRACK_MAX_ITERATIONS: return "MAX_ITERATIONS";
  }
  return "UNKNOWN";
}

flk_status flk_session_create(const flk_config* config, flk_session** out) {
  if (!config || !out) return fail(FLK_E_INVALID_ARG, "config and out must not be NULL");
  return guarded([&] {
    flkb::validate(config->cfg);  // config errors before the device check
    auto s = std::make_unique<flk_session>();
    s->session = std::make_unique<flkb::Session>(config->cfg, current_device());
    *out = s.release();
    return FLK_OK;
  });
}

flk_status flk_session_process(flk_session* session, const flk_image* image,
                               flk_tracks** out_tracks, flk_frame_stats* stats,
                               flk_conformance* conformance) {
  if (!session || !image || !out_tracks)
    return fail(FLK_E_INVALID_ARG, "session, image, and out_tracks must not be NULL");
  return guarded([&] {
    auto t = std::make_unique<flk_tracks>();
    session->session->process(image->img, &t->items, stats, conformance);
    *out_tracks = t.release();
    return FLK_OK;
  });
}

void flk_session_destroy(flk_session* session) { delete session; }

flk_status flkb_sessions_process(flk_session* const* sessions, const flk_image* const* images,
                                 int n, flk_tracks** out_tracks, flk_frame_stats* stats) {
  if (!sessions || !images || !out_tracks || n < 0)
    return fail(FLK_E_INVALID_ARG, "sessions, images, and out_tracks must not be NULL");
  for (int i = 0; i < n; ++i) {
    out_tracks[i] = nullptr;
    if (!sessions[i] || !images[i]) return fail(FLK_E_INVALID_ARG, "NULL session or image");
  }
  {  // one frame per session and call: a repeated handle would stage twice
    std::vector<const flk_session*> seen(sessions, sessions + n);
    std::sort(seen.begin(), seen.end());
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
      return fail(FLK_E_INVALID_ARG, "the same session appears more than once");
  }
  int submitted = 0;
  flk_status first = FLK_OK;
  std::string first_msg;
  // submit every frame first so the sessions' graphs overlap on the GPU
  for (; submitted < n; ++submitted) {
    const flk_status st = guarded([&] {
      sessions[submitted]->session->submit(images[submitted]->img, stats != nullptr);
      return FLK_OK;
    });
    if (st != FLK_OK) {
      first = st;
      first_msg = g_error;
      break;
    }
  }
  for (int i = 0; i < submitted; ++i) {
    const flk_status st = guarded([&] {
      auto t = std::make_unique<flk_tracks>();
      sessions[i]->session->complete(images[i]->img, &t->items, stats ? stats + i : nullptr,
                                     nullptr);
      out_tracks[i] = t.release();
      return FLK_OK;
    });
    if (st != FLK_OK && first == FLK_OK) {
      first = st;
      first_msg = g_error;
    }
  }
  if (first != FLK_OK) return fail(first, first_msg.c_str());
  g_error.clear();
  return FLK_OK;
}



int flk_tracks_count(const flk_tracks* tracks) {
  return tracks ? static_cast<int>(tracks->items.size()) : 0;
}

flk_status flk_tracks_get(const flk_tracks* tracks, int index, flk_track_info* out) {
  if (!tracks || !out) return fail(FLK_E_INVALID_ARG, "tracks and out must not be NULL");
  if (index < 0 || index >= static_cast<int>(tracks->items.size()))
    return fail(FLK_E_INVALID_ARG, "track index out of range");
  *out = tracks->items[static_cast<size_t>(index)];
  return FLK_OK;
}

void flk_tracks_destroy(flk_tracks* tracks) { delete tracks; }

/* ---------------------------------------------------------- B200 extension */

flk_status flkb_config_set_cell_size_px(flk_config* config, int cw, int ch) {
  if (!config) return fail(FLK_E_INVALID_ARG, "config must not be NULL");
  if (cw < 0 || ch < 0) return fail(FLK_E_INVALID_ARG, "cell size must be non-negative");
  config->cfg.cell_width_px = cw;
  config->cfg.cell_height_px = ch;
  g_error.clear();
  return FLK_OK;
}

int flkb_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

flk_status flkb_detector_set_device(flk_detector* detector, int device) {
  if (!detector) return fail(FLK_E_INVALID_ARG, "detector must not be NULL");
  return guarded([&] {
    if (device < 0 || device >= flkb_device_count())
      throw flkb::InvalidArgument("no CUDA device " + std::to_string(device));
    if (device != detector->device) detector->reset_workspaces();
    detector->device = device;
    return FLK_OK;
  });
}

flk_status flkb_detector_run_batch(flk_detector* detector, const flk_image* const* images, int n,
                                   flk_features** outs, flk_frame_stats* stats) {
  if (!detector || !images || !outs)
    return fail(FLK_E_INVALID_ARG, "detector, images, and outs must not be NULL");
  return guarded([&] {
    latch_batch(detector, images, n, outs);
    if (n == 0) return FLK_OK;
    if (stats) {
      // counters need the per-frame stats kernels; run frame by frame
      for (int i = 0; i < n; ++i) {
        flk_status s = flk_detector_run(detector, images[i], &outs[i], &stats[i], nullptr);
        if (s != FLK_OK) {  // like the pipelined path: no handle survives a failure
          for (int j = 0; j < i; ++j) {
            flk_features_destroy(outs[j]);
            outs[j] = nullptr;
          }
          return s;
        }
      }
      return FLK_OK;
    }
    if (!detector->pipeline)
      detector->pipeline = std::make_unique<BatchPipeline>(detector->params, detector->device,
                                                           detector->first_width,
                                                           detector->first_height);
    try {
      detector->pipeline->run(images, n, outs);
    } catch (...) {
      for (int i = 0; i < n; ++i) {
        flk_features_destroy(outs[i]);
        outs[i] = nullptr;
      }
      throw;
    }
    return FLK_OK;
  });
}

flk_status flkb_detector_run_batch_multi(flk_detector* detector, const int* devices, int ndev,
                                         const flk_image* const* images, int n,
                                         flk_features** outs) {
  if (!detector || !devices || !images || !outs)
    return fail(FLK_E_INVALID_ARG, "detector, devices, images, and outs must not be NULL");
  return guarded([&] {
    if (ndev < 1) throw flkb::InvalidArgument("at least one device is needed");
    const int avail = flkb_device_count();
    if (avail == 0) current_device();  // throws: no CUDA device, no CPU fallback
    for (int i = 0; i < ndev; ++i)
      if (devices[i] < 0 || devices[i] >= avail)
        throw flkb::InvalidArgument("no CUDA device " + std::to_string(devices[i]));
    latch_batch(detector, images, n, outs);
    if (n == 0) return FLK_OK;
    // one pipeline (device workspace, streams, pinned staging) per listed
    // device, kept across calls while the list stays the same
    const std::vector<int> want(devices, devices + ndev);
    if (want != detector->multi_devices) {
      detector->multi.clear();
      detector->multi_devices = want;
    }
    while (static_cast<int>(detector->multi.size()) < ndev) {
      const int d = want[detector->multi.size()];
      detector->multi.push_back(std::make_unique<BatchPipeline>(
          detector->params, d, detector->first_width, detector->first_height));
    }
    // one host thread per device over its contiguous frame shard; the shards'
    // results land in disjoint slots of outs, so no merge is needed
    std::vector<std::exception_ptr> errs(static_cast<size_t>(ndev));
    auto work = [&](int r) {
      int start = 0, count = 0;
      shard_range(n, r, ndev, &start, &count);
      if (count == 0) return;
      try {
        detector->multi[static_cast<size_t>(r)]->run(images + start, count, outs + start);
      } catch (...) {
        errs[static_cast<size_t>(r)] = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    for (int r = 1; r < ndev; ++r) pool.emplace_back(work, r);
    work(0);
    for (auto& t : pool) t.join();
    for (auto& e : errs) {
      if (!e) continue;
      for (int i = 0; i < n; ++i) {
        flk_features_destroy(outs[i]);
        outs[i] = nullptr;
      }
      std::rethrow_exception(e);
    }
    return FLK_OK;
  });
}

flk_status flkb_detector_set_plan(flk_detector* detector, const char* key, int value) {
  if (!detector || !key) return fail(FLK_E_INVALID_ARG, "detector and key must not be NULL");
  return guarded([&] {
    if (!detector->params.plan.set(key, value))
      throw flkb::ConfigError(std::string("unknown launch-plan key '") + key + "'");
    detector->reset_workspaces();
    return FLK_OK;
  });
}

flk_status flkb_batch_set_plan(flkb_batch* b, const char* key, int value) {
  if (!b || !key) return fail(FLK_E_INVALID_ARG, "batch and key must not be NULL");
  return guarded([&] {
    flkb::LaunchPlan plan = b->batch->params().plan;
    if (!plan.set(key, value))
      throw flkb::ConfigError(std::string("unknown launch-plan key '") + key + "'");
    b->batch->set_plan(plan);
    return FLK_OK;
  });
}

flk_status flkb_batch_create(flk_detector* detector, int width, int height, int capacity,
                             flkb_batch** out) {
  if (!detector || !out) return fail(FLK_E_INVALID_ARG, "detector and out must not be NULL");
  return guarded([&] {
    auto b = std::make_unique<flkb_batch>();
    b->device = detector->device;
    b->batch = std::make_unique<flkb::DeviceBatch>(detector->params, detector->device, width,
                                                   height, capacity);
    *out = b.release();
    return FLK_OK;
  });
}

void flkb_batch_destroy(flkb_batch* batch) { delete batch; }

flk_status flkb_batch_run_device(flkb_batch* b, const uint8_t* frames, size_t frame_stride,
                                 int row_pitch, int count, int with_stats, void* stream) {
  if (!b || !frames) return fail(FLK_E_INVALID_ARG, "batch and frames must not be NULL");
  return guarded([&] {
    b->batch->run(frames, frame_stride, row_pitch, count, with_stats != 0,
                  static_cast<cudaStream_t>(stream));
    return FLK_OK;
  });
}

flk_status flkb_batch_run_device_timed(flkb_batch* b, const uint8_t* frames, size_t frame_stride,
                                       int row_pitch, int count, void* stream, double* stage_us) {
  if (!b || !frames || !stage_us)
    return fail(FLK_E_INVALID_ARG, "batch, frames, and stage_us must not be NULL");
  return guarded([&] {
    flkb::StageTimes t;
    b->batch->run(frames, frame_stride, row_pitch, count, false,
                  static_cast<cudaStream_t>(stream), &t);
    stage_us[0] = t.pyramid_us;
    stage_us[1] = t.crf_us;
    stage_us[2] = t.nms_us;
    return FLK_OK;
  });
}

namespace {

// Chunked H2D -> detect (-> D2H) over the batch's two side streams, joined
// back into the caller's stream: chunk c's H2D overlaps chunk c-1's kernels,
// and with host outputs chunk c's feature download overlaps chunk c+1's
// kernels (H2D and D2H use separate copy engines).
void run_host_chunks(flkb_batch* b, const uint8_t* frames, size_t frame_stride, int row_pitch,
                     int count, cudaStream_t user, int* counts, flk_feature* features) {
  flkb::DeviceBatch& db = *b->batch;
  const flkb::Geometry& g = db.geometry();
  if (count < 1 || count > db.capacity()) throw flkb::InvalidArgument("count outside the batch");
  if (row_pitch < g.width || frame_stride < static_cast<size_t>(row_pitch) * g.height)
    throw flkb::InvalidArgument("host frame layout smaller than the frame size");
  flkb::DeviceGuard guard(b->device);
  if (!b->d_in) {
    // frames stay densely packed when the width is already 16-B aligned, so
    // the H2D copy is one linear transfer
    b->in_pitch = static_cast<int>(round16(static_cast<size_t>(g.width)));
    b->in_stride = static_cast<size_t>(b->in_pitch) * g.height;
    flkb::check_cuda(cudaMalloc(&b->d_in, b->in_stride * db.capacity() + 16), "batch input");
    for (auto& s : b->side) flkb::check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    for (auto& e : b->ev) flkb::check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  flkb::check_cuda(cudaEventRecord(b->ev[0], user), "event");
  for (auto s : b->side) flkb::check_cuda(cudaStreamWaitEvent(s, b->ev[0], 0), "wait");
  const int chunk = std::max(1, std::min(count, 256));
  const size_t cells = static_cast<size_t>(g.cells);
  int si = 0;
  for (int c0 = 0; c0 < count; c0 += chunk, si ^= 1) {
    const int cnt = std::min(chunk, count - c0);
    cudaStream_t s = b->side[si];
    uint8_t* dst = b->d_in + static_cast<size_t>(c0) * b->in_stride;
    const uint8_t* src = frames + static_cast<size_t>(c0) * frame_stride;
    if (row_pitch == b->in_pitch && frame_stride == b->in_stride) {
      flkb::check_cuda(cudaMemcpyAsync(dst, src, b->in_stride * cnt, cudaMemcpyHostToDevice, s),
                       "H2D frames");
    } else if (frame_stride == static_cast<size_t>(row_pitch) * g.height) {
      flkb::check_cuda(cudaMemcpy2DAsync(dst, b->in_pitch, src, row_pitch, g.width,
                                         static_cast<size_t>(g.height) * cnt,
                                         cudaMemcpyHostToDevice, s), "H2D frames");
    } else {
      for (int j = 0; j < cnt; ++j)
        flkb::check_cuda(cudaMemcpy2DAsync(dst + j * b->in_stride, b->in_pitch,
                                           src + j * frame_stride, row_pitch, g.width, g.height,
                                           cudaMemcpyHostToDevice, s), "H2D frame");
    }
    db.run(dst, b->in_stride, b->in_pitch, cnt, false, s, nullptr, c0);
    if (counts || features)
      db.download(c0, cnt, counts ? counts + c0 : nullptr,
                  features ? features + static_cast<size_t>(c0) * cells : nullptr, s);
  }
  flkb::check_cuda(cudaEventRecord(b->ev[1], b->side[0]), "event");
  flkb::check_cuda(cudaEventRecord(b->ev[2], b->side[1]), "event");
  flkb::check_cuda(cudaStreamWaitEvent(user, b->ev[1], 0), "wait");
  flkb::check_cuda(cudaStreamWaitEvent(user, b->ev[2], 0), "wait");
}

}  // namespace

flk_status flkb_batch_run_host(flkb_batch* b, const uint8_t* frames, size_t frame_stride,
                               int row_pitch, int count, void* stream) {
  if (!b || !frames) return fail(FLK_E_INVALID_ARG, "batch and frames must not be NULL");
  return guarded([&] {
    run_host_chunks(b, frames, frame_stride, row_pitch, count, static_cast<cudaStream_t>(stream),
                    nullptr, nullptr);
    return FLK_OK;
  });
}

flk_status flkb_batch_detect_host(flkb_batch* b, const uint8_t* frames, size_t frame_stride,
                                  int row_pitch, int count, int* counts, flk_feature* features,
                                  void* stream) {
  if (!b || !frames || (!counts && !features))
    return fail(FLK_E_INVALID_ARG, "batch, frames, and an output must not be NULL");
  return guarded([&] {
    run_host_chunks(b, frames, frame_stride, row_pitch, count, static_cast<cudaStream_t>(stream),
                    counts, features);
    return FLK_OK;
  });
}

flk_status flkb_batch_download(const flkb_batch* b, int first, int count, int* counts,
                               flk_feature* features, void* stream) {
  if (!b) return fail(FLK_E_INVALID_ARG, "batch must not be NULL");
  return guarded([&] {
    b->batch->download(first, count, counts, features, static_cast<cudaStream_t>(stream));
    return FLK_OK;
  });
}

flk_status flkb_batch_conformance(flkb_batch* b, const uint8_t* frames, size_t frame_stride,
                                  int row_pitch, int first, int count,
                                  flk_conformance* per_frame, flk_conformance* total,
                                  void* stream) {
  if (!b || !frames || !total)
    return fail(FLK_E_INVALID_ARG, "batch, frames, and total must not be NULL");
  return guarded([&] {
    const flkb::Geometry& g = b->batch->geometry();
    if (row_pitch < g.width || frame_stride < static_cast<size_t>(row_pitch) * g.height)
      throw flkb::InvalidArgument("row pitch / frame stride smaller than the frame");
    *total = b->batch->conformance(frames, frame_stride, row_pitch,
                                   static_cast<cudaStream_t>(stream), first, count, per_frame);
    return FLK_OK;
  });
}

int flkb_batch_frame_capacity(const flkb_batch* b) { return b ? b->batch->geometry().cells : 0; }
const int* flkb_batch_device_counts(const flkb_batch* b) { return b ? b->batch->device_counts() : nullptr; }
const flk_feature* flkb_batch_device_features(const flkb_batch* b) {
  return b ? b->batch->device_features() : nullptr;
}
const uint64_t* flkb_batch_device_stats(const flkb_batch* b) {
  return b ? b->batch->device_stats() : nullptr;
}

flk_status flkb_batch_device_pyramid(const flkb_batch* b, int level, const uint8_t** base,
                                     int* width, int* height, int* row_pitch,
                                     size_t* frame_stride) {
  if (!b || !base) return fail(FLK_E_INVALID_ARG, "batch and base must not be NULL");
  return guarded([&] {
    const flkb::Geometry& g = b->batch->geometry();
    if (level < 1 || level >= g.levels) throw flkb::InvalidArgument("level outside [1, l)");
    *base = b->batch->device_pyramid() + g.loff[level];
    if (width) *width = g.lw[level];
    if (height) *height = g.lh[level];
    if (row_pitch) *row_pitch = g.lpitch[level];
    if (frame_stride) *frame_stride = g.pyr_frame_bytes;
    return FLK_OK;
  });
}

flk_status flkb_synth_frames_device(uint8_t* frames, int kind, uint64_t first_frame, int count,
                                    int width, int height, int row_pitch, size_t frame_stride,
                                    void* stream) {
  if (!frames) return fail(FLK_E_INVALID_ARG, "frames must not be NULL");
  return guarded([&] {
    if (count < 0 || width < 1 || height < 1 || row_pitch < width)
      throw flkb::InvalidArgument("bad synthetic frame geometry");
    flkb::synth_frames(frames, kind, first_frame, count, width, height, row_pitch, frame_stride,
                       static_cast<cudaStream_t>(stream));
    return FLK_OK;
  });
}

namespace {
flk_status detector_responses(flk_detector* detector, const flk_image* image, float* out,
                              bool fused) {
  if (!detector || !image || !out)
    return fail(FLK_E_INVALID_ARG, "detector, image, and out must not be NULL");
  return guarded([&] {
    if (detector->first_width == 0) {
      detector->first_width = image->img.width;
      detector->first_height = image->img.height;
    } else if (image->img.width != detector->first_width ||
               image->img.height != detector->first_height) {
      throw flkb::DimensionMismatch("frame size differs from the detector's first frame");
    }
    if (!detector->runner)
      detector->runner = std::make_unique<FrameRunner>(detector->params, detector->device,
                                                       image->img.width, image->img.height);
    detector->runner->responses(image->img, out, fused);
    return FLK_OK;
  });
}
}  // namespace

flk_status flkb_detector_responses(flk_detector* detector, const flk_image* image, float* out) {
  return detector_responses(detector, image, out, false);
}

flk_status flkb_detector_fused_responses(flk_detector* detector, const flk_image* image,
                                         float* out) {
  return detector_responses(detector, image, out, true);
}

flk_status flkb_debug_hypot(const double* x, const double* y, double* out, int n) {
  if (!x || !y || !out) return fail(FLK_E_INVALID_ARG, "x, y, and out must not be NULL");
  return guarded([&] {
    current_device();
    flkb::lk::debug_hypot(x, y, out, n);
    return FLK_OK;
  });
}

uint64_t flkb_kernel_launch_count(void) { return flkb::launch_count(); }
int flkb_batch_kernels_per_run(const flkb_batch* b) { return b ? b->batch->kernels_per_run() : 0; }

}  // extern "C"
