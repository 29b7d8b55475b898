/*
 * fastlk C ABI, B200 edition -- drop-in replacement for the reference
 * detector library.
 *
 * Every declaration below is ABI-identical to the reference header
 * /root/reference/proj/include/fastlk/fastlk.h (names, types, enum values,
 * struct layouts, NULL and ownership rules); the line numbers cited with each
 * group are the reference declarations they replace. Programs compiled
 * against the reference header link against libfastlk_b200.so unchanged.
 *
 * What changes underneath: flk_detector_run executes pyramid construction,
 * FAST scoring and fused grid suppression as sm_100a CUDA kernels on the
 * detector's GPU. Keypoints are bit-identical to the reference CPU
 * implementation. There is no CPU fallback: without a usable GPU the
 * detector calls fail with FLK_E_INTERNAL and a message.
 *
 * The tracking session (flk_session_*, flk_tracks_*) runs the reference's
 * detect-track lifecycle with the pyramid, the fp64 LK tracker, re-detection
 * and template building on the GPU; track records (positions, gains and
 * offsets as doubles) and counters are bit-identical to the reference.
 * Batched and device-resident entry points live in fastlk_b200.h.
 */
#ifndef FASTLK_B200_FASTLK_H_
#define FASTLK_B200_FASTLK_H_

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define FLK_API __declspec(dllexport)
#else
#define FLK_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (reference fastlk.h:38-45). */
typedef enum flk_status {
  FLK_OK = 0,
  FLK_E_INVALID_ARG = 1,
  FLK_E_IO = 2,
  FLK_E_DIMENSION = 3,
  FLK_E_CONFIG = 4,
  FLK_E_INTERNAL = 5
} flk_status;

/* Reference fastlk.h:47-52. flk_last_error is thread local and cleared at
 * the start of every call that can fail. */
FLK_API const char* flk_status_name(flk_status status);
FLK_API const char* flk_last_error(void);
FLK_API const char* flk_version_string(void); /* "0.1.0" */

/* Images (reference fastlk.h:56-69): host-side 8-bit grayscale rasters.
 * flk_image_create copies width*height tightly packed bytes. */
typedef struct flk_image flk_image;
FLK_API flk_status flk_image_create(int width, int height, const uint8_t* pixels,
                                    flk_image** out);
FLK_API flk_status flk_image_load_pgm(const char* path, flk_image** out);
FLK_API flk_status flk_image_save_pgm(const flk_image* image, const char* path);
FLK_API int flk_image_width(const flk_image* image);
FLK_API int flk_image_height(const flk_image* image);
FLK_API void flk_image_destroy(flk_image* image);

/* Configuration (reference fastlk.h:73-88): the same 13 keys, defaults and
 * parse errors. Range checks happen at flk_detector_create. */
typedef struct flk_config flk_config;
FLK_API flk_status flk_config_create(flk_config** out);
FLK_API flk_status flk_config_load_file(flk_config* config, const char* path);
FLK_API flk_status flk_config_set(flk_config* config, const char* key, const char* value);
FLK_API void flk_config_destroy(flk_config* config);

/* Detection (reference fastlk.h:92-145). */
typedef struct flk_detector flk_detector;
typedef struct flk_features flk_features;

typedef struct flk_feature {
  int x; /* level-0 pixel coordinates */
  int y;
  float score;
  int level;
  int cell_x;
  int cell_y;
} flk_feature;

typedef struct flk_frame_stats {
  double pyramid_us;
  double crf_us;
  double nms_us;
  double track_us;
  uint64_t nms_comparisons;
  uint64_t nms_candidates;
  int feature_count;
  int tracks_entering;
  int tracks_surviving;
  int tracks_spawned;
  int redetect_fired;
  int track_iterations;
} flk_frame_stats;

typedef struct flk_conformance {
  int matched;
  int subset_only;
  int false_positives;
} flk_conformance;

FLK_API flk_status flk_detector_create(const flk_config* config, flk_detector** out);
FLK_API flk_status flk_detector_run(flk_detector* detector, const flk_image* image,
                                    flk_features** out_features, flk_frame_stats* stats,
                                    flk_conformance* conformance);
FLK_API void flk_detector_destroy(flk_detector* detector);

FLK_API int flk_features_count(const flk_features* features);
FLK_API flk_status flk_features_get(const flk_features* features, int index,
                                    flk_feature* out);
FLK_API void flk_features_destroy(flk_features* features);

/* Tracking (reference fastlk.h:149-192; capi.cpp:298-362 -> Frontend::
 * process_frame, frontend.cpp:65-225). The live tracks are advanced by the
 * LK kernel, re-detection runs the fused detector on the frame's pyramid, and
 * new templates are built by a kernel; the host keeps the reference's order
 * of retirement, per-cell dedupe, candidate ranking and id assignment. */
typedef struct flk_session flk_session;
typedef struct flk_tracks flk_tracks;

typedef enum flk_track_status {
  FLK_TRACK_CONVERGED = 0,
  FLK_TRACK_DIVERGED = 1,
  FLK_TRACK_OUT_OF_BOUNDS = 2,
  FLK_TRACK_SINGULAR_HESSIAN = 3,
  FLK_TRACK_MAX_ITERATIONS = 4
} flk_track_status;

typedef struct flk_track_info {
  int64_t id;
  double x;
  double y;
  double alpha;
  double beta;
  int status;
  int live;
  int birth_frame;
} flk_track_info;

FLK_API const char* flk_track_status_name(flk_track_status status);
FLK_API flk_status flk_session_create(const flk_config* config, flk_session** out);
FLK_API flk_status flk_session_process(flk_session* session, const flk_image* image,
                                       flk_tracks** out_tracks, flk_frame_stats* stats,
                                       flk_conformance* conformance);
FLK_API void flk_session_destroy(flk_session* session);
FLK_API int flk_tracks_count(const flk_tracks* tracks);
FLK_API flk_status flk_tracks_get(const flk_tracks* tracks, int index, flk_track_info* out);
FLK_API void flk_tracks_destroy(flk_tracks* tracks);

#ifdef __cplusplus
}
#endif

#endif /* FASTLK_B200_FASTLK_H_ */
