/*
 * TEST INFRASTRUCTURE ONLY -- CPU parity oracle for the FAST + grid-NMS hot path.
 *
 * A plain-C restatement of the reference detector (`fastlk`, CPU C++20) that
 * the CUDA product is checked against. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product library never
 * links or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   1. against the reference itself, compiled from /root/reference into
 *      oracle/_ref/libfastlk_ref.so by oracle/Makefile (same inputs, same
 *      outputs, bit for bit);
 *   2. against the golden fixtures under tests/golden/, generated from that
 *      reference build by tests/golden/make_golden.py, so the pin survives on
 *      boxes without /root/reference.
 *
 * Every function cites the reference file:line it restates. Paths are
 * relative to /root/reference/proj.
 */
#ifndef FASTLK_ORACLE_H_
#define FASTLK_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_INVALID_ARG = 1, ORC_E_CONFIG = 4 };
enum { ORC_SAD_B = 0, ORC_SAD_A = 1, ORC_MT = 2 };

/* FastParams (src/fastlk/fast.hpp:20-24) + GridConfig (src/fastlk/nms.hpp:17-31).
 * cell_width_px / cell_height_px: 0 means the reference geometry
 * (32*w by 2^(l-1)*h); a positive value is the B200 extension override used
 * for cell sizes the reference API cannot express (e.g. 16x16). */
typedef struct orc_params {
  int epsilon;
  int arc_length;
  int score_kind;
  int num_levels;
  int cell_width_units;
  int cell_height_units;
  int nms_radius;
  int cell_width_px;
  int cell_height_px;
} orc_params;

/* Same layout as flk_feature (include/fastlk/fastlk.h:95-102). */
typedef struct orc_feature {
  int x, y;
  float score;
  int level, cell_x, cell_y;
} orc_feature;

typedef struct orc_stats {
  uint64_t comparisons;
  uint64_t candidates;
  int feature_count;
} orc_stats;

typedef struct orc_conformance {
  int matched, subset_only, false_positives;
} orc_conformance;

void orc_default_params(orc_params* p);
int orc_validate(const orc_params* p);
int orc_cell_width(const orc_params* p);
int orc_cell_height(const orc_params* p);

/* Level dims; returns ORC_E_INVALID_ARG when the image is too small. */
int orc_pyramid_dims(int width, int height, int levels, int* wk, int* hk);
/* Levels written tightly packed, back to back, level 0 first. */
int orc_build_pyramid(const uint8_t* img, int width, int height, int levels,
                      uint8_t* out);

/* Arc test with the reference LUT semantics (fast.cpp:34-65). */
int orc_has_cyclic_run(uint16_t mask, int min_len);
/* Rotation-scan oracle (oracle.cpp:15-25). */
int orc_arc_oracle(uint16_t mask, int min_len);

/* One level of detect_responses (fast.cpp:273-303); resp is w*h floats. */
int orc_fast_level(const uint8_t* img, int w, int h, const orc_params* p,
                   float* resp);
/* Corner score of one interior pixel (fast.cpp:267-271). */
float orc_corner_score(const uint8_t* img, int w, int h, int x, int y,
                       const orc_params* p);

/* suppress_and_select over precomputed per-level responses
 * (nms.cpp:81-135). resp[k] is wk[k]*hk[k] floats. cells is cols*rows,
 * an entry with level < 0 is empty. */
int orc_suppress_and_select(const float* const* resp, const int* wk,
                            const int* hk, const orc_params* p,
                            orc_feature* cells, int* cols, int* rows,
                            orc_stats* stats);

/* Whole detect path as flk_detector_run returns it (capi.cpp:232-274):
 * features in row-major cell order. cap must be >= cols*rows. */
int orc_detect(const uint8_t* img, int width, int height, const orc_params* p,
               orc_feature* out, int cap, int* count, orc_stats* stats);

/* Naive conformance tally (oracle.cpp:240-268) of an emitted feature list. */
int orc_conformance_check(const uint8_t* img, int width, int height,
                    const orc_params* p, const orc_feature* feats, int count,
                    orc_conformance* out);

/* Synthetic generators S1 (noise, kind 0) and S2 (texture, kind 1), SURVEY §8(d). */
void orc_synth_frame(int kind, uint64_t frame, int width, int height,
                     uint8_t* out);

/* ---------------------------------------------------------------- tracking
 * lk_oracle.c: restatement of src/fastlk/lk.cpp and Frontend::process_frame
 * (src/fastlk/frontend.cpp:65-225). */

enum { ORC_E_IO = 2, ORC_E_DIMENSION = 3 };
/* ParamMode (lk.hpp:17) */
enum { ORC_MODE_TRANSLATION = 0, ORC_MODE_TRANSLATION_OFFSET = 1, ORC_MODE_TRANSLATION_GAIN = 2,
       ORC_MODE_FULL = 3 };
/* TrackStatus (lk.hpp:19-25) */
enum { ORC_TRACK_CONVERGED = 0, ORC_TRACK_DIVERGED = 1, ORC_TRACK_OUT_OF_BOUNDS = 2,
       ORC_TRACK_SINGULAR_HESSIAN = 3, ORC_TRACK_MAX_ITERATIONS = 4 };
/* TemplateError (lk.hpp:80) */
enum { ORC_TPL_OK = 0, ORC_TPL_OUT_OF_BOUNDS = 1, ORC_TPL_SINGULAR = 2 };

/* TrackerConfig (lk.hpp:40-48) */
typedef struct orc_tracker {
  int mode;
  int max_iterations;
  double convergence_epsilon;
  double min_determinant_factor;
} orc_tracker;

/* PatchTemplate (lk.hpp:65-78); 16x16 patches at most, 4 parameters. */
typedef struct orc_patch {
  int level, patch;
  double anchor_x, anchor_y;
  int dims;
  float values[256];
  double coeffs[256 * 4];
  double hessian_inv[16];
  double hessian_det;
} orc_patch;

typedef struct orc_templates {
  int error;
  int nlevels;
  orc_patch lv[16];
} orc_templates;

typedef struct orc_track_result {
  int status;
  double warp[4]; /* tx, ty, alpha, beta */
  int iterations;
} orc_track_result;

/* FrontendConfig (frontend.hpp:16-23) */
typedef struct orc_session_cfg {
  orc_params det;
  orc_tracker tracker;
  int target_count;
  double redetect_ratio;
} orc_session_cfg;

/* Same layout as flk_track_info (include/fastlk/fastlk.h:162-173). */
typedef struct orc_track_info {
  int64_t id;
  double x, y, alpha, beta;
  int status, live, birth_frame;
} orc_track_info;

/* The counters of flk_frame_stats (fastlk.h:106-119); no timings. */
typedef struct orc_session_stats {
  uint64_t nms_comparisons, nms_candidates;
  int feature_count, tracks_entering, tracks_surviving, tracks_spawned, redetect_fired,
      track_iterations;
} orc_session_stats;

typedef struct orc_session orc_session;

void orc_default_tracker(orc_tracker* t);
int orc_validate_tracker(const orc_tracker* t);
int orc_param_dims(int mode);
/* build_template (lk.cpp:147-240) on a pyramid given level by level. */
int orc_build_template(const uint8_t* const* lv, const int* wk, const int* hk, int nlevels,
                       int x0, int y0, const orc_tracker* cfg, orc_templates* out);
/* track_feature (lk.cpp:242-350); init = {tx, ty, alpha, beta}. */
int orc_track_feature(const orc_templates* tpl, const uint8_t* const* lv, const int* wk,
                      const int* hk, int nlevels, const double* init, const orc_tracker* cfg,
                      orc_track_result* res);
int orc_session_create(const orc_session_cfg* cfg, orc_session** out);
int orc_session_process(orc_session* s, const uint8_t* img, int width, int height,
                        orc_track_info* out, int cap, int* count, orc_session_stats* stats,
                        orc_conformance* conf);
void orc_session_destroy(orc_session* s);

#ifdef __cplusplus
}
#endif

#endif /* FASTLK_ORACLE_H_ */
