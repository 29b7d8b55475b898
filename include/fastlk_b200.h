/*
 * B200 extension API -- batched and device-resident detection.
 *
 * Not part of the reference ABI (the reference API is single-frame and
 * host-only, fastlk.h:134-138). These entry points let a caller keep frames
 * and results in HBM, run many frames per launch, pick the GPU, and express
 * cell sizes the reference's 32*w x 2^(l-1)*h geometry cannot (e.g. 16x16,
 * SURVEY §7 hard part 4). Results are bit-identical to flk_detector_run on
 * each frame.
 *
 * Streams are passed as `void*` (a cudaStream_t; NULL = the legacy default
 * stream). Device pointers are plain `uint8_t*` into the detector's device.
 */
#ifndef FASTLK_B200_EXT_H_
#define FASTLK_B200_EXT_H_

#include "fastlk.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Cell size override in level-0 pixels; 0 restores the reference geometry.
 * Stored in the config but not a config-file key, so configs stay loadable
 * by the reference. */
FLK_API flk_status flkb_config_set_cell_size_px(flk_config* config, int cell_width_px,
                                                int cell_height_px);

/* GPU selection (default: the current device at flk_detector_create). */
FLK_API flk_status flkb_detector_set_device(flk_detector* detector, int device);
FLK_API int flkb_device_count(void);

/* Many host frames in one call: images must all have the detector's frame
 * size. outs[i] receives frame i's features (caller frees each); stats may be
 * NULL or an array of n. Frames go through a two-slot pipeline kept by the
 * detector (H2D of one chunk overlaps the kernels of the other); images whose
 * page-locked pixels already have the device pitch are DMA'd in place. */
FLK_API flk_status flkb_detector_run_batch(flk_detector* detector,
                                           const flk_image* const* images, int n,
                                           flk_features** outs, flk_frame_stats* stats);

/* Many host frames over several GPUs of one host, in one call: frames are
 * split into contiguous shards, shard r = frames [r*n/ndev, ...) runs on
 * devices[r] through its own two-slot pipeline (device workspace, streams,
 * page-locked staging) driven by its own host thread; results land in
 * disjoint slots of outs (outs[i] = frame i's features, caller frees each).
 * Frames are independent, so there is no exchange between the GPUs (SURVEY
 * 8(e)); the output is identical to flkb_detector_run_batch for any device
 * list, including one device listed several times. The reference's only
 * parallelism is parallel_chunks' host threads (parallel.hpp:33-52) under
 * the same determinism contract. On an error every out is NULL. */
FLK_API flk_status flkb_detector_run_batch_multi(flk_detector* detector, const int* devices,
                                                 int ndev, const flk_image* const* images, int n,
                                                 flk_features** outs);

/* Launch-plan overrides for tests and tuning tools (the engine reads no
 * environment variables): keys "band_rows", "tiles" (0 = shape search),
 * "fuse_pyramid" (-1 auto, 0 one-launch plan, 1 two-launch plan),
 * "pyramid_chunk" (frames, 0 = auto), "pdl" (0/1), "list_cap" (corner-list
 * entries, 0 = auto), "debug_geom" (0/1), "staged" (1: the staged v1 kernels, one
 * launch per stage and level with u16 score maps in HBM -- the design
 * baseline the fused kernel is measured against), "batch_copies" (0: host
 * batches copy frame by frame instead of one cudaMemcpyBatchAsync per chunk).
 * Results never depend on
 * the plan.
 * Setting a detector's plan drops its cached device workspaces; batches take
 * the detector's plan at creation. Unknown key: FLK_E_CONFIG. */
FLK_API flk_status flkb_detector_set_plan(flk_detector* detector, const char* key, int value);

/* ---------------------------------------------------------- device batches */

/* A device-resident workspace for up to `capacity` frames of width x height
 * (pyramid levels >= 1, per-frame cell keys and feature lists). */
typedef struct flkb_batch flkb_batch;

FLK_API flk_status flkb_batch_create(flk_detector* detector, int width, int height,
                                     int capacity, flkb_batch** out);
FLK_API void flkb_batch_destroy(flkb_batch* batch);
/* flkb_detector_set_plan for one batch. */
FLK_API flk_status flkb_batch_set_plan(flkb_batch* batch, const char* key, int value);

/* Detects on `count` device frames: frame f row y starts at
 * frames + f*frame_stride + y*row_pitch. Asynchronous on `stream`; results
 * stay on the device until flkb_batch_download. with_stats fills per-frame
 * nms_candidates / nms_comparisons (slower; off for throughput). */
FLK_API flk_status flkb_batch_run_device(flkb_batch* batch, const uint8_t* frames,
                                         size_t frame_stride, int row_pitch, int count,
                                         int with_stats, void* stream);

/* flkb_batch_run_device, synchronized, with CUDA-event device times of its
 * three launches in stage_us: [0] pyramid, [1] fused FAST + suppression +
 * cell selection, [2] feature compaction (microseconds). */
FLK_API flk_status flkb_batch_run_device_timed(flkb_batch* batch, const uint8_t* frames,
                                               size_t frame_stride, int row_pitch, int count,
                                               void* stream, double* stage_us);

/* Same, from host memory: H2D copies of the frames happen inside the call on
 * `stream` (pinned host memory overlaps; pageable is staged). */
FLK_API flk_status flkb_batch_run_host(flkb_batch* batch, const uint8_t* frames,
                                       size_t frame_stride, int row_pitch, int count,
                                       void* stream);

/* Host frames in, host feature lists out, one pipelined call: chunks of
 * frames alternate over two streams so each chunk's H2D overlaps the previous
 * chunk's kernels and its feature download overlaps the next chunk's kernels.
 * counts / features as for flkb_batch_download(batch, 0, count, ...) (either
 * may be NULL, not both; pinned host memory for overlap). Asynchronous on
 * `stream`. */
FLK_API flk_status flkb_batch_detect_host(flkb_batch* batch, const uint8_t* frames,
                                          size_t frame_stride, int row_pitch, int count,
                                          int* counts, flk_feature* features, void* stream);

/* Copies per-frame counts and the compact feature lists to the host.
 * features is count * flkb_batch_frame_capacity() entries; frame f's list
 * starts at features + f*flkb_batch_frame_capacity(). Either may be NULL. */
FLK_API flk_status flkb_batch_download(const flkb_batch* batch, int first, int count,
                                       int* counts, flk_feature* features, void* stream);

FLK_API int flkb_batch_frame_capacity(const flkb_batch* batch); /* grid cells per frame */
FLK_API const int* flkb_batch_device_counts(const flkb_batch* batch);
FLK_API const flk_feature* flkb_batch_device_features(const flkb_batch* batch);
/* Device stats: per frame {uint64 candidates, uint64 comparisons}. */
FLK_API const uint64_t* flkb_batch_device_stats(const flkb_batch* batch);

/* The pyramid product on the device (level >= 1; level 0 is the input). */
FLK_API flk_status flkb_batch_device_pyramid(const flkb_batch* batch, int level,
                                             const uint8_t** base, int* width, int* height,
                                             int* row_pitch, size_t* frame_stride);

/* GPU conformance tally (the reference's
 * oracle::conformance_check, oracle.cpp:240-268, replacing the CPU pass
 * flk_detector_run makes for a non-NULL conformance, capi.cpp:254-259) of
 * frames [first, first + count) of the last flkb_batch_run_device: a naive
 * detector (per-pixel labels, rotation-scan arc test, linear-scan MT, raster
 * suppression) re-run on the device frames and pyramid, each emitted feature
 * checked against it. `frames`, `frame_stride`, `row_pitch` as passed to
 * that run. per_frame (count entries) may be NULL; total receives the sum.
 * Synchronous on `stream`. */
FLK_API flk_status flkb_batch_conformance(flkb_batch* batch, const uint8_t* frames,
                                          size_t frame_stride, int row_pitch, int first,
                                          int count, flk_conformance* per_frame,
                                          flk_conformance* total, void* stream);

/* Deterministic synthetic frames written on the device:
 * kind 0 = S1 noise, 1 = S2 texture; frame f gets index first_frame + f. */
FLK_API flk_status flkb_synth_frames_device(uint8_t* frames, int kind, uint64_t first_frame,
                                            int count, int width, int height, int row_pitch,
                                            size_t frame_stride, void* stream);

/* Corner-response maps of every pyramid level for one frame (the values of
 * the reference's detect_responses, fast.cpp:273-303), tightly packed
 * level after level as floats: sum_k w_k*h_k entries. A diagnostic entry
 * point for parity tests; subject to the detector's frame-size latch. */
FLK_API flk_status flkb_detector_responses(flk_detector* detector, const flk_image* image,
                                           float* out);
/* The same maps as the production fused kernel (k_detect) computes them: each
 * CTA writes the scores of its own rows and columns from its shared-memory
 * score tile (a diagnostic dump; pixels that are no corner read 0). Equal to
 * flkb_detector_responses by construction of the parity tests. */
FLK_API flk_status flkb_detector_fused_responses(flk_detector* detector, const flk_image* image,
                                                 float* out);

/* ------------------------------------------------------- many sessions */

/* Advances n independent tracking sessions by one frame each, overlapping
 * their GPU work: every session's frame is staged and its frame graph
 * (pyramid + LK) enqueued on the session's own stream first, then each is
 * completed in order (re-detection frames run their detector inside the
 * completion). Per session the result is exactly flk_session_process's;
 * out_tracks[i] receives session i's snapshot (caller frees each) and stats
 * may be NULL or an array of n. On an error the sessions already submitted
 * are still completed and returned; the others get NULL. */
FLK_API flk_status flkb_sessions_process(flk_session* const* sessions,
                                         const flk_image* const* images, int n,
                                         flk_tracks** out_tracks, flk_frame_stats* stats);

/* Bulk accessors: copy min(count, cap) records into out (row-major cell
 * order / id order, as flk_features_get / flk_tracks_get index them) and
 * return the number copied; NULL handles copy nothing. */
FLK_API int flkb_features_copy(const flk_features* features, flk_feature* out, int cap);
FLK_API int flkb_tracks_copy(const flk_tracks* tracks, flk_track_info* out, int cap);

/* Test hook: the tracker's device hypot (glibc's algorithm, so convergence
 * and divergence tests match the reference's std::hypot, lk.cpp:267,319) on
 * n host pairs. Synchronous. */
FLK_API flk_status flkb_debug_hypot(const double* x, const double* y, double* out, int n);

/* Number of CUDA kernels this library has launched in the process (graph
 * replays count every kernel node). */
FLK_API uint64_t flkb_kernel_launch_count(void);
/* Kernels one flkb_batch_run_device call launches (without stats). */
FLK_API int flkb_batch_kernels_per_run(const flkb_batch* batch);

#ifdef __cplusplus
}
#endif

#endif /* FASTLK_B200_EXT_H_ */
