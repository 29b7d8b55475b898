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

#ifdef __cplusplus
}
#endif

#endif /* FASTLK_ORACLE_H_ */
