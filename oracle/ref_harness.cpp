// TEST INFRASTRUCTURE ONLY -- thin C shim over the UNMODIFIED reference
// (`fastlk`, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libfastlk_ref.so). It exposes the reference's stage functions
// with the orc_* parameter/feature layout so tests can pin the C oracle to
// the reference bit for bit, and it times the reference's public C API for
// bench.py's reference arm. No reference source is copied here; this file
// only calls the reference headers' public functions.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "fastlk/fastlk.h"
#include "fastlk/error.hpp"
#include "fastlk/fast.hpp"
#include "fastlk/frontend.hpp"
#include "fastlk/image.hpp"
#include "fastlk/lk.hpp"
#include "fastlk/nms.hpp"
#include "fastlk/oracle.hpp"
#include "../oracle/fastlk_oracle.h"

namespace {

fastlk::Image to_image(const uint8_t* px, int w, int h) {
  fastlk::Image img = fastlk::Image::allocate(w, h);
  for (int y = 0; y < h; ++y)
    std::memcpy(&img.data[static_cast<size_t>(y) * img.stride],
                px + static_cast<size_t>(y) * w, w);
  return img;
}

fastlk::FastParams fast_params(const orc_params* p) {
  fastlk::FastParams f;
  f.epsilon = p->epsilon;
  f.arc_length = p->arc_length;
  f.score = p->score_kind == ORC_SAD_B   ? fastlk::ScoreKind::kSadB
            : p->score_kind == ORC_SAD_A ? fastlk::ScoreKind::kSadA
                                         : fastlk::ScoreKind::kMt;
  return f;
}

fastlk::GridConfig grid_config(const orc_params* p) {
  fastlk::GridConfig g;
  g.cell_width_units = p->cell_width_units;
  g.cell_height_units = p->cell_height_units;
  g.num_levels = p->num_levels;
  g.nms_radius = p->nms_radius;
  return g;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const fastlk::ConfigError&) {
    return ORC_E_CONFIG;
  } catch (const std::exception&) {
    return ORC_E_INVALID_ARG;
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int refh_pyramid(const uint8_t* img, int w, int h,
                                                        int levels, uint8_t* out) {
  return guarded([&] {
    fastlk::ImagePyramid pyr = fastlk::build_pyramid(to_image(img, w, h), levels);
    size_t off = 0;
    for (int k = 0; k < pyr.num_levels(); ++k) {
      const fastlk::Image& l = pyr.level(k);
      for (int y = 0; y < l.height; ++y) {
        std::memcpy(out + off, &l.data[static_cast<size_t>(y) * l.stride], l.width);
        off += l.width;
      }
    }
    return ORC_OK;
  });
}

// Responses of every level, tightly packed level after level.
__attribute__((visibility("default"))) int refh_responses(const uint8_t* img, int w, int h,
                                                          const orc_params* p, float* out) {
  return guarded([&] {
    fastlk::ImagePyramid pyr = fastlk::build_pyramid(to_image(img, w, h), p->num_levels);
    fastlk::FastParams f = fast_params(p);
    fastlk::LookupTable lut = fastlk::build_lookup_table(f.arc_length);
    std::vector<fastlk::ResponseMap> maps = fastlk::detect_responses(pyr, f, lut, 1);
    size_t off = 0;
    for (const auto& m : maps) {
      for (int y = 0; y < m.height; ++y) {
        std::memcpy(out + off, &m.scores[static_cast<size_t>(y) * m.stride],
                    sizeof(float) * m.width);
        off += m.width;
      }
    }
    return ORC_OK;
  });
}

__attribute__((visibility("default"))) int refh_arc_lut(int n, uint8_t* out65536) {
  return guarded([&] {
    fastlk::LookupTable lut = fastlk::build_lookup_table(n);
    for (uint32_t m = 0; m <= 0xFFFFu; ++m) out65536[m] = lut.test(static_cast<uint16_t>(m));
    return ORC_OK;
  });
}

// Whole detect path. With the cell override unset this is exactly
// detect_frame (frontend.cpp:38-57) plus the capi flatten; with it set, the
// cell fold is composed from the reference's own spiral_is_local_max and
// cell_candidate_wins at the overridden cell size (SURVEY §7 hard part 4).
__attribute__((visibility("default"))) int refh_detect(const uint8_t* img, int w, int h,
                                                       const orc_params* p, orc_feature* out,
                                                       int cap, int* count, orc_stats* stats,
                                                       int threads) {
  return guarded([&] {
    fastlk::FastParams f = fast_params(p);
    fastlk::GridConfig g = grid_config(p);
    fastlk::validate(f);
    fastlk::validate(g);
    fastlk::LookupTable lut = fastlk::build_lookup_table(f.arc_length);
    fastlk::Image frame = to_image(img, w, h);
    int n = 0;
    if (p->cell_width_px <= 0 && p->cell_height_px <= 0) {
      fastlk::DetectRun run = fastlk::detect_frame(frame, f, lut, g, threads);
      for (int cy = 0; cy < run.grid.rows; ++cy)
        for (int cx = 0; cx < run.grid.cols; ++cx) {
          const auto& c = run.grid.at(cx, cy);
          if (!c.has_value()) continue;
          if (n < cap) out[n] = orc_feature{c->x, c->y, c->score, c->level, cx, cy};
          ++n;
        }
      if (stats) {
        stats->comparisons = run.stats.nms.comparisons;
        stats->candidates = run.stats.nms.candidates;
        stats->feature_count = run.stats.feature_count;
      }
    } else {
      const int cw = p->cell_width_px > 0 ? p->cell_width_px : g.cell_width();
      const int ch = p->cell_height_px > 0 ? p->cell_height_px : g.cell_height();
      fastlk::ImagePyramid pyr = fastlk::build_pyramid(frame, g.num_levels);
      auto maps = fastlk::detect_responses(pyr, f, lut, threads);
      const int cols = (w + cw - 1) / cw, rows = (h + ch - 1) / ch;
      std::vector<std::optional<fastlk::CellMax>> cells(static_cast<size_t>(cols) * rows);
      uint64_t comparisons = 0, candidates = 0;
      for (int k = 0; k < g.num_levels; ++k) {
        const auto& m = maps[static_cast<size_t>(k)];
        for (int y = 0; y < m.height; ++y)
          for (int x = 0; x < m.width; ++x) {
            const float s = m.at(x, y);
            if (s <= 0.0f) continue;
            ++candidates;
            if (!fastlk::spiral_is_local_max(m, x, y, g.nms_radius, &comparisons)) continue;
            const auto [x0, y0] = fastlk::rescale_to_level0(x, y, k);
            fastlk::CellMax cand{x0, y0, s, k};
            auto& slot = cells[static_cast<size_t>(y0 / ch) * cols + x0 / cw];
            if (!slot.has_value() || fastlk::cell_candidate_wins(cand, *slot)) slot = cand;
          }
      }
      for (int cy = 0; cy < rows; ++cy)
        for (int cx = 0; cx < cols; ++cx) {
          const auto& c = cells[static_cast<size_t>(cy) * cols + cx];
          if (!c.has_value()) continue;
          if (n < cap) out[n] = orc_feature{c->x, c->y, c->score, c->level, cx, cy};
          ++n;
        }
      if (stats) {
        stats->comparisons = comparisons;
        stats->candidates = candidates;
        stats->feature_count = n;
      }
    }
    *count = n;
    return n > cap ? ORC_E_INVALID_ARG : ORC_OK;
  });
}

// suppress_and_select (nms.cpp:81-135) on caller-provided response maps;
// cells is cols*rows orc_features, level -1 marks an empty cell.
__attribute__((visibility("default"))) int refh_select(const float* const* maps, const int* wk,
                                                       const int* hk, const orc_params* p,
                                                       orc_feature* cells, int* cols, int* rows,
                                                       orc_stats* stats, int threads) {
  return guarded([&] {
    std::vector<fastlk::ResponseMap> rm;
    for (int k = 0; k < p->num_levels; ++k) {
      fastlk::ResponseMap m = fastlk::ResponseMap::allocate(wk[k], hk[k], k);
      for (int y = 0; y < hk[k]; ++y)
        for (int x = 0; x < wk[k]; ++x) m.at(x, y) = maps[k][static_cast<size_t>(y) * wk[k] + x];
      rm.push_back(std::move(m));
    }
    fastlk::NmsStats st;
    fastlk::FeatureGrid g = fastlk::suppress_and_select(rm, grid_config(p), threads, &st);
    *cols = g.cols;
    *rows = g.rows;
    for (int cy = 0; cy < g.rows; ++cy)
      for (int cx = 0; cx < g.cols; ++cx) {
        const auto& c = g.at(cx, cy);
        cells[static_cast<size_t>(cy) * g.cols + cx] =
            c.has_value() ? orc_feature{c->x, c->y, c->score, c->level, cx, cy}
                          : orc_feature{0, 0, 0.0f, -1, cx, cy};
      }
    if (stats) {
      stats->comparisons = st.comparisons;
      stats->candidates = st.candidates;
      stats->feature_count = g.feature_count();
    }
    return ORC_OK;
  });
}

__attribute__((visibility("default"))) int refh_conformance(const uint8_t* img, int w, int h,
                                                            const orc_params* p,
                                                            orc_conformance* out) {
  return guarded([&] {
    fastlk::FastParams f = fast_params(p);
    fastlk::GridConfig g = grid_config(p);
    fastlk::LookupTable lut = fastlk::build_lookup_table(f.arc_length);
    fastlk::DetectRun run = fastlk::detect_frame(to_image(img, w, h), f, lut, g, 1);
    fastlk::oracle::Conformance c = fastlk::oracle::conformance_check(run.pyramid, run.grid, f, g);
    out->matched = c.matched;
    out->subset_only = c.subset_only;
    out->false_positives = c.false_positives;
    return ORC_OK;
  });
}

// Times the reference's public C API (flk_detector_run) over n host frames.
// mode 0 = as shipped: one detector with threads=0, frames sequential (what
// `fastlk detect` does, fastlk_cli.cpp:199-232). mode 1 = best-effort host:
// `workers` threads, each with its own threads=1 detector, pulling frames
// from a shared counter. Frame images are created before the clock starts.
// Returns seconds, or a negative value on error; *features_out sums counts.
// Optional outputs (NULL = not collected): frame i's feature list at
// out + i*cap with its count in counts[i] (whole-batch parity against the
// GPU), and the sums over frames of flk_frame_stats' pyramid_us / crf_us /
// nms_us in stage_us[0..2] (the reference's per-stage split, frontend.cpp:38-57).
__attribute__((visibility("default"))) double refh_bench(const uint8_t* frames, int n, int w,
                                                         int h, const char* const* keys,
                                                         const char* const* values, int nkv,
                                                         int mode, int workers,
                                                         long long* features_out,
                                                         flk_feature* out, int cap, int* counts,
                                                         double* stage_us) {
  std::vector<flk_image*> imgs(static_cast<size_t>(n), nullptr);
  for (int i = 0; i < n; ++i)
    if (flk_image_create(w, h, frames + static_cast<size_t>(i) * w * h, &imgs[i]) != FLK_OK)
      return -1.0;
  auto make_det = [&](const char* threads) -> flk_detector* {
    flk_config* cfg = nullptr;
    if (flk_config_create(&cfg) != FLK_OK) return nullptr;
    for (int i = 0; i < nkv; ++i)
      if (flk_config_set(cfg, keys[i], values[i]) != FLK_OK) return nullptr;
    flk_config_set(cfg, "threads", threads);
    flk_detector* det = nullptr;
    flk_status st = flk_detector_create(cfg, &det);
    flk_config_destroy(cfg);
    return st == FLK_OK ? det : nullptr;
  };
  std::atomic<long long> feats{0};
  std::atomic<int> failed{0};
  std::vector<flk_frame_stats> fstats(stage_us ? static_cast<size_t>(n) : 0);
  auto one = [&](flk_detector* det, int i) {
    flk_features* f = nullptr;
    if (flk_detector_run(det, imgs[i], &f, stage_us ? &fstats[i] : nullptr, nullptr) != FLK_OK)
      failed = 1;
    const int c = flk_features_count(f);
    feats += c;
    if (out && counts) {
      counts[i] = c;
      for (int j = 0; j < c && j < cap; ++j)
        flk_features_get(f, j, out + static_cast<size_t>(i) * cap + j);
    }
    flk_features_destroy(f);
  };
  double secs = 0.0;
  if (mode == 0) {
    flk_detector* det = make_det("0");
    if (!det) return -2.0;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) one(det, i);
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    flk_detector_destroy(det);
  } else {
    std::vector<flk_detector*> dets(static_cast<size_t>(workers));
    for (auto& d : dets)
      if (!(d = make_det("1"))) return -2.0;
    std::atomic<int> next{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t)
      pool.emplace_back([&, t] {
        for (int i; (i = next.fetch_add(1)) < n;) one(dets[t], i);
      });
    for (auto& th : pool) th.join();
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto* d : dets) flk_detector_destroy(d);
  }
  for (auto* im : imgs) flk_image_destroy(im);
  if (features_out) *features_out = feats.load();
  if (stage_us) {
    stage_us[0] = stage_us[1] = stage_us[2] = 0.0;
    for (const auto& st : fstats) {
      stage_us[0] += st.pyramid_us;
      stage_us[1] += st.crf_us;
      stage_us[2] += st.nms_us;
    }
  }
  return failed ? -3.0 : secs;
}

// refh_detect over n frames, `workers` threads pulling frames from a shared
// counter (each frame's detection single-threaded): frame i's features at
// out + i*cap, its count in counts[i]. Whole-batch parity for configurations
// the public API cannot express (the cell-size override of refh_detect).
__attribute__((visibility("default"))) int refh_detect_batch(const uint8_t* frames, int n, int w,
                                                             int h, const orc_params* p,
                                                             int workers, orc_feature* out,
                                                             int cap, int* counts) {
  std::atomic<int> next{0}, rc{ORC_OK};
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, workers); ++t)
    pool.emplace_back([&] {
      for (int i; (i = next.fetch_add(1)) < n;) {
        const int r = refh_detect(frames + static_cast<size_t>(i) * w * h, w, h, p,
                                  out + static_cast<size_t>(i) * cap, cap, counts + i, nullptr, 1);
        if (r != ORC_OK) rc = r;
      }
    });
  for (auto& th : pool) th.join();
  return rc.load();
}

}  // extern "C"

// ------------------------------------------------------------- tracking

namespace {

fastlk::TrackerConfig tracker_config(const orc_tracker* t) {
  fastlk::TrackerConfig c;
  c.mode = static_cast<fastlk::ParamMode>(t->mode);
  c.max_iterations = t->max_iterations;
  c.convergence_epsilon = t->convergence_epsilon;
  c.min_determinant_factor = t->min_determinant_factor;
  return c;
}

void to_orc(const fastlk::FeatureTemplates& in, orc_templates* out) {
  std::memset(out, 0, sizeof *out);
  out->error = static_cast<int>(in.error);
  out->nlevels = static_cast<int>(in.levels.size());
  for (size_t i = 0; i < in.levels.size(); ++i) {
    const fastlk::PatchTemplate& t = in.levels[i];
    orc_patch& o = out->lv[i];
    o.level = t.level;
    o.patch = t.patch;
    o.anchor_x = t.anchor_x;
    o.anchor_y = t.anchor_y;
    o.dims = t.dims;
    std::memcpy(o.values, t.values.data(), sizeof(float) * t.values.size());
    std::memcpy(o.coeffs, t.coeffs.data(), sizeof(double) * t.coeffs.size());
    for (int k = 0; k < 16; ++k) o.hessian_inv[k] = t.hessian_inv[static_cast<size_t>(k)];
    o.hessian_det = t.hessian_det;
  }
}

}  // namespace

extern "C" {

// build_template (lk.cpp:147-240) on the pyramid of img.
__attribute__((visibility("default"))) int refh_build_template(const uint8_t* img, int w, int h,
                                                               int levels, int x0, int y0,
                                                               const orc_tracker* t,
                                                               orc_templates* out) {
  return guarded([&] {
    fastlk::ImagePyramid pyr = fastlk::build_pyramid(to_image(img, w, h), levels);
    fastlk::CellMax f;
    f.x = x0;
    f.y = y0;
    to_orc(fastlk::build_template(pyr, f, tracker_config(t)), out);
    return ORC_OK;
  });
}

// Templates from the pyramid of prev at (x0, y0), tracked into the pyramid of
// cur from init = {tx, ty, alpha, beta} with track_feature (lk.cpp:242-350).
__attribute__((visibility("default"))) int refh_track_feature(const uint8_t* prev,
                                                              const uint8_t* cur, int w, int h,
                                                              int levels, int x0, int y0,
                                                              const double* init,
                                                              const orc_tracker* t,
                                                              orc_track_result* res) {
  return guarded([&] {
    const fastlk::TrackerConfig cfg = tracker_config(t);
    fastlk::ImagePyramid p0 = fastlk::build_pyramid(to_image(prev, w, h), levels);
    fastlk::ImagePyramid p1 = fastlk::build_pyramid(to_image(cur, w, h), levels);
    fastlk::CellMax f;
    f.x = x0;
    f.y = y0;
    const fastlk::FeatureTemplates tpl = fastlk::build_template(p0, f, cfg);
    if (!tpl.ok()) return ORC_E_CONFIG;
    fastlk::WarpState ws;
    ws.tx = init[0];
    ws.ty = init[1];
    ws.alpha = init[2];
    ws.beta = init[3];
    const fastlk::TrackResult r = fastlk::track_feature(tpl, p1, ws, cfg);
    res->status = static_cast<int>(r.status);
    res->warp[0] = r.warp.tx;
    res->warp[1] = r.warp.ty;
    res->warp[2] = r.warp.alpha;
    res->warp[3] = r.warp.beta;
    res->iterations = r.total_iterations();
    return ORC_OK;
  });
}

}  // extern "C"
