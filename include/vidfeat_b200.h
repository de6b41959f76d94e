/*
 * vidfeat_b200.h -- C ABI of the B200-native detect+describe hot path.
 *
 * Drop-in boundary for the reference `vidfeat` 0.1.0 per-frame path
 * (/root/reference/pkg/src/vidfeat/).  The reference has no FFI: its operator
 * seam is the Python function layer with import-time kernel dispatch
 * (accel.py:22-57 selects numba or numpy inside _score_map, detector.py:166-172,
 * orientations_batch / describe_batch, descriptor.py:194-232).  These entry
 * points replace that seam; the Python package paper_1503_06959_b200 binds
 * them with ctypes and keeps the reference's function names and dataclasses.
 *
 * Conventions: plain pointers and sizes, no torch types.  "_dev" pointers are
 * CUDA device memory (e.g. a torch CUDA tensor's data_ptr()), "stream" is a
 * cudaStream_t (0 = legacy default stream).  All calls return VF_OK (0) or a
 * negative VF_ERR_* code; vf_strerror() gives the reference's exception text.
 * Calls are asynchronous on `stream` unless documented otherwise.
 */
#ifndef VIDFEAT_B200_H
#define VIDFEAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- status codes (each mirrors a reference ValueError / exception) -------- */
#define VF_OK 0
#define VF_ERR_THRESHOLD (-1)     /* "detection threshold must be >= 1"      detector.py:195-196 */
#define VF_ERR_OCTAVES (-2)       /* "n_octaves must be >= 1"                pyramid.py:103-104  */
#define VF_ERR_FRAME_SMALL (-3)   /* "frame WxH too small for O octaves"     pyramid.py:105-109  */
#define VF_ERR_UNDERFLOW (-4)     /* "dimension underflow ..."               pyramid.py:70-71,83-84 */
#define VF_ERR_MODE (-5)          /* "unknown mask mode"                     masking.py:75-77    */
#define VF_ERR_T_H (-6)           /* "histogram threshold must be >= 0"      masking.py:78-79    */
#define VF_ERR_GRID (-7)          /* "binning grid must be at least 1x1"     masking.py:80-81    */
#define VF_ERR_EMPTY (-8)         /* "empty frame sequence"                  pipeline.py:211-212 */
#define VF_ERR_CAPACITY (-9)      /* keypoint capacity overflow (no reference counterpart)      */
#define VF_ERR_CUDA (-10)         /* CUDA runtime error                                          */
#define VF_ERR_ARG (-11)          /* invalid argument                                            */
#define VF_ERR_INDEX (-12)        /* numpy IndexError (nms_and_refine border candidate)          */
#define VF_ERR_OCTAVE_KEY (-13)   /* KeyError: no octave layer at octave_for_mask (pyramid.py:61-63) */
#define VF_ERR_PATTERN (-14)      /* sampling pattern not uploaded / malformed                   */
#define VF_ERR_MATCH_CAPACITY (-15) /* radius_match output buffer too small (*n_matches = needed)  */
#define VF_ERR_GOP_DELTA (-16)    /* "GOP length must be >= 1"               temporal.py:34-35   */
#define VF_ERR_GOP_PATCH (-17)    /* "patch side must be even and positive"  temporal.py:36-37   */
#define VF_ERR_GOP_STEP (-18)     /* "fine_step must not exceed coarse_step" temporal.py:38-39   */
#define VF_ERR_GOP_SAD (-19)      /* "SAD thresholds must be positive"       temporal.py:40-41   */

#define VF_MODE_NONE 0
#define VF_MODE_INTENSITY 1
#define VF_MODE_TEMPORAL 3   /* block-matching baseline: full detection at GOP starts, spiral SAD search between */
#define VF_MODE_BINNING 2

/* PipelineConfig (pipeline.py:46-54) + MaskConfig (masking.py:66-81), flattened. */
typedef struct vf_config {
  int32_t width, height;      /* frame size (all streams of a context share it)        */
  int32_t n_octaves;          /* PipelineConfig.n_octaves, default 4                   */
  int32_t threshold;          /* PipelineConfig.threshold, default 55                  */
  int32_t mask_mode;          /* VF_MODE_* (pipeline.py:215-216 for temporal)          */
  double t_i;                 /* MaskConfig.t_i, default 20.0                          */
  int32_t t_h;                /* MaskConfig.t_h, default 1                             */
  int32_t grid_rows, grid_cols; /* MaskConfig.grid, default (16, 16)                   */
  int32_t octave_for_mask;    /* MaskConfig.octave_for_mask, -1 = None (top octave)    */
  int32_t per_layer;          /* MaskConfig.per_layer                                  */
  int32_t max_streams;        /* independent video streams processed per call          */
  int32_t kp_capacity;        /* features per stream and frame, 0 = automatic          */
  /* GopConfig (temporal.py:23-43), used when mask_mode == VF_MODE_TEMPORAL.  All
   * zero = the reference defaults (10, 16, 1800, 1000, 12, 2, 1.75, 0.25). */
  int32_t gop_delta, gop_patch;
  double gop_t_bm, gop_t_et, gop_coarse_window, gop_coarse_step, gop_fine_window, gop_fine_step;
} vf_config;

/* FrameReport (pipeline.py:57-71) counts of the last processed frame. */
typedef struct vf_report {
  int64_t frame;
  int32_t n_detected, n_propagated, n_total, n_dropped;
  double coverage;
  int32_t n_survivors;        /* NMS survivors before the border filter (diagnostic)   */
  int32_t n_candidates;       /* FAST candidates (diagnostic)                           */
} vf_report;

/* Device pointers to a stream's current feature list (Feature, masking.py:58-63),
 * SoA: keypoint x, y, sigma, theta, score (fp64), origin (0 detected,
 * 1 propagated), age, and 64-byte MSB-first descriptors (descriptor.py:271-275).
 * Valid until the next vf_process on the context. */
typedef struct vf_features {
  int32_t n;
  const double *x, *y, *sigma, *theta, *score;
  const uint8_t *origin;
  const int32_t *age;
  const uint8_t *desc;
} vf_features;

typedef struct vf_ctx vf_ctx;

const char *vf_version(void);
const char *vf_strerror(int code);

/* Sampling pattern (pattern.py:30-46): points (m x 2), radii (m), short pairs
 * (nbits x 2), long pairs (L x 2).  m must be 60 and nbits 512 (v1 pattern). */
int vf_set_pattern(const double *points, const double *radii, int m, const int32_t *short_pairs,
                   int nbits, const int32_t *long_pairs, int L);

/* --- the per-frame pipeline: run_pipeline's loop body (pipeline.py:222-277) -- */
/* Frames up to 8192 x 8192 (VF_ERR_ARG beyond: NMS candidates are coded in 32 bits). */
int vf_create(const vf_config *cfg, vf_ctx **out);
int vf_destroy(vf_ctx *ctx);
/* Geometry of the pyramid (layer order o0, i0, o1, ...): sizes and scales. */
int vf_layer_geometry(const vf_ctx *ctx, int32_t *ws, int32_t *hs, double *scales);
/* Forget all temporal state (next frame is "frame 0" on every stream). */
int vf_reset(vf_ctx *ctx, void *stream);
/* Process frame n of streams [0, n_streams): frames_dev + s*stream_stride is
 * stream s's (height x width) uint8 frame with row pitch `row_pitch`. */
int vf_process(vf_ctx *ctx, const uint8_t *frames_dev, int64_t stream_stride, int64_t row_pitch,
               int n_streams, void *stream);
/* vf_process, then a capacity check (synchronizes `stream`): when a stream's
 * features would overflow the per-stream capacity (VF_ERR_CAPACITY), the step
 * is rolled back, every stream's capacity grows (the previous lists are kept)
 * and the step is replayed from the same state, until it fits (SURVEY.md
 * 8(b): "the wrapper grows the capacity and retries the frame from saved
 * state").  Temporal mode returns VF_ERR_CAPACITY instead. */
int vf_process_checked(vf_ctx *ctx, const uint8_t *frames_dev, int64_t stream_stride, int64_t row_pitch,
                       int n_streams, void *stream);
/* Current feature capacity per stream and buffer. */
int vf_get_capacity(const vf_ctx *ctx, int32_t *kp_capacity);
/* Same, from pinned or pageable HOST memory: the host->device copy is part of
 * the call (double-buffered device staging, stream-ordered). */
int vf_process_host(vf_ctx *ctx, const uint8_t *frames_host, int64_t stream_stride, int64_t row_pitch,
                    int n_streams, void *stream);
/* vf_process_host with the capacity check / grow / replay of vf_process_checked. */
int vf_process_host_checked(vf_ctx *ctx, const uint8_t *frames_host, int64_t stream_stride, int64_t row_pitch,
                            int n_streams, void *stream);
/* Synchronizes `stream`, then reports the last processed frame of `s`.
 * Returns VF_ERR_CAPACITY if a capacity overflow was flagged on the device. */
int vf_get_report(vf_ctx *ctx, int s, vf_report *out, void *stream);
/* Synchronizes `stream`; device pointers of stream s's current features. */
int vf_get_features(vf_ctx *ctx, int s, vf_features *out, void *stream);
/* Synchronizes `stream`; copies stream s's features to host arrays of >= cap entries. */
int vf_copy_features(vf_ctx *ctx, int s, int32_t cap, double *x, double *y, double *sigma, double *theta,
                     double *score, uint8_t *origin, int32_t *age, uint8_t *desc, int32_t *n_out, void *stream);
/* All streams [0, n_streams) at once: packs every stream's current features on
 * the device into one contiguous SoA (stream s at [offsets[s], offsets[s+1])),
 * then enqueues ONE device->host copy per field into the caller's (pinned)
 * host arrays of >= cap entries.  Synchronizes `stream` once for the counts;
 * the field copies are asynchronous on `stream` (synchronize before use). */
int vf_fetch_features(vf_ctx *ctx, int n_streams, int64_t cap, double *x, double *y, double *sigma,
                      double *theta, double *score, uint8_t *origin, int32_t *age, uint8_t *desc,
                      int32_t *offsets, void *stream);
/* Pipelined host-to-host processing (the e2e API): submit copies step n's
 * host frames to the device on a copy stream, runs the path and packs the
 * features on a compute stream; collect returns the oldest submitted step's
 * features (all streams, packed as in vf_fetch_features) after its
 * device->host copy on a second copy stream.  At most three steps may be in
 * flight (submit, submit, submit, collect, submit, collect, ...; a fourth
 * submit returns VF_ERR_ARG), so the H2D of step n+2 is already queued while
 * step n+1 computes and step n's result is copied out: the slowest of the
 * three sets the pace.  Two in flight (submit, submit, collect, ...) works too.
 * collect reads the step's offsets, counts and error flags from one pinned
 * meta-data copy, then delivers the fields: results up to 64 KB into pinned
 * (device-addressable) arrays by one kernel launch that writes over PCIe,
 * anything else by one cudaMemcpyAsync per field (VF_D2H_KERNEL=0 forces the
 * copies).  Stream-ordered with respect
 * to the context's own streams only; not to be mixed with vf_process on the
 * same context. */
int vf_pipeline_submit(vf_ctx *ctx, const uint8_t *frames_host, int64_t stream_stride, int64_t row_pitch,
                       int n_streams);
int vf_pipeline_collect(vf_ctx *ctx, int64_t cap, double *x, double *y, double *sigma, double *theta,
                        double *score, uint8_t *origin, int32_t *age, uint8_t *desc, int32_t *offsets);
/* Delta results for the pipelined API: with vf_pipeline_set_delta(ctx, 1)
 * (between steps), vf_pipeline_collect_delta returns each step's result as
 * the DETECTED records of every stream (packed as in vf_fetch_features,
 * stream s at det_offsets[s] .. det_offsets[s+1]; origin detected, age 0)
 * plus the Eq. 1 keep mask of the stream's previous list (32-bit words at
 * keep_offsets[s] .., bit i = previous feature i propagates) and counts[3 s ..]
 * = n_detected, n_propagated, previous-list length covered by the mask.  The
 * merged list (masking.py:176-183) is detected ++ [previous[i] with origin
 * propagated and age + 1, for every kept i] -- vf_delta_apply rebuilds it on
 * the host from the previous list.  D2H per step is the new records only. */
int vf_pipeline_set_delta(vf_ctx *ctx, int enable);
int vf_pipeline_collect_delta(vf_ctx *ctx, int64_t cap, double *x, double *y, double *sigma, double *theta,
                              double *score, uint8_t *desc, int32_t *det_offsets, int64_t kcap, uint32_t *keep_bits,
                              int32_t *keep_offsets, int32_t *counts);
/* Host only: list n of one stream from list n-1 and the stream's delta. */
int vf_delta_apply(int32_t n_prev, const double *prev_x, const double *prev_y, const double *prev_sigma,
                   const double *prev_theta, const double *prev_score, const uint8_t *prev_origin,
                   const int32_t *prev_age, const uint8_t *prev_desc, int32_t n_det, const double *det_x,
                   const double *det_y, const double *det_sigma, const double *det_theta, const double *det_score,
                   const uint8_t *det_desc, int32_t n_keep_bits, const uint32_t *keep_bits, int32_t out_cap,
                   double *x, double *y, double *sigma, double *theta, double *score, uint8_t *origin, int32_t *age,
                   uint8_t *desc, int32_t *n_out);
/* Device pointers of layer l of stream s's current pyramid (l >= 1; l = 0 is the input frame). */
int vf_get_layer(vf_ctx *ctx, int s, int l, const uint8_t **ptr, int32_t *pitch);
/* Live per-stage device timing with CUDA events on the launch stream:
 * stages = binmask, pyramid, worklist, fast, nms, sat, describe, propagate, finalize (9).
 * The SAT build and the fused describe kernel run on describe streams (two
 * stream halves with >= 2 streams per call); their one joint interval is
 * reported under "sat" and "describe" is 0.  "nms" covers k_nms_list,
 * k_nms_test and k_nms_finish.  propagate is timed on its own (side) stream.
 * vf_get_stage_ms synchronizes `stream`, returns the summed milliseconds per
 * stage since the last query and the number of steps, and clears. */
int vf_set_timing(vf_ctx *ctx, int enable);
/* CUDA graphs (default on): a batch of at most 64 MB of frames replays a
 * captured graph of the step's launches (captured once per batch size; the
 * kernel nodes are re-pointed at each call's frames, nothing is copied).  Off
 * while stage timing is on and in temporal mode. */
int vf_set_graphs(vf_ctx *ctx, int enable);
int vf_get_stage_ms(vf_ctx *ctx, double *ms9, int32_t *n_steps, void *stream);
/* Synchronizes `stream`; work counters of the last step: active FAST tiles,
 * total FAST tiles, SAT tiles built, total SAT tiles, unmasked streams,
 * staged NMS candidates, bands per stream, feature capacity. */
int vf_get_diag(vf_ctx *ctx, int64_t *out8, void *stream);
/* Per-frame statistics history: every later step also writes, on the device,
 * stream s's FrameReport row of frame f (f < max_frames) to
 * hist_dev[(s * max_frames + f) * 8 + k], k = n_detected, n_propagated,
 * n_total, n_dropped, coverage, frame, n_survivors, n_candidates (fp64).  The
 * caller owns hist_dev ([max_streams][max_frames][8] doubles); max_frames = 0
 * turns it off.  Used for the end-of-run per-stream statistics gather. */
int vf_set_history(vf_ctx *ctx, double *hist_dev, int32_t max_frames);
/* Per-stream totals since vf_create/vf_reset: sum n_detected, sum n_total, sum coverage, frames. */
int vf_get_totals(vf_ctx *ctx, int s, double *out4, void *stream);

/* --- per-stage drop-ins (same device code as the pipeline) ------------------- */
/* build_pyramid (pyramid.py:97-125): writes layers 1..2O-1 to layers_dev[l] with pitches[l]. */
int vf_build_pyramid(const uint8_t *frame_dev, int W, int H, int64_t pitch, int n_octaves,
                     uint8_t *const *layers_dev, const int64_t *pitches, void *stream);
/* _score_map / detect_candidates (detector.py:166-204): uint8 scores (0 or >= t) of
 * one layer, gated by an optional full-res mask (mask_dev, mw x mh, floor mapping). */
int vf_score_map(const uint8_t *layer_dev, int w, int h, int64_t pitch, int t, const uint8_t *mask_dev,
                 int mw, int mh, uint8_t *scores_dev, int64_t scores_pitch, void *stream);
/* nms_and_refine / _nms_from_maps (detector.py:239-324) over caller score maps
 * (uint8, layer geometry of a W x H frame with n_octaves).  Outputs in
 * reference order; *n_out = count (synchronizes). */
int vf_nms_refine(const uint8_t *const *maps_dev, const int64_t *pitches, int W, int H, int n_octaves,
                  int32_t cap, double *x_dev, double *y_dev, double *sigma_dev, double *score_dev,
                  int32_t *n_out, void *stream);
/* orientations_batch (theta_in_dev == NULL) or describe_batch at theta_in_dev
 * (descriptor.py:194-232) on a full-res frame; desc_dev gets n x 64 packed bytes. */
int vf_describe(const uint8_t *frame_dev, int W, int H, int64_t pitch, int n, const double *kx_dev,
                const double *ky_dev, const double *sigma_dev, const double *theta_in_dev,
                double *theta_out_dev, uint8_t *desc_dev, void *stream);
/* intensity_diff_mask (masking.py:84-93) over n pixels. */
int vf_intensity_mask(const uint8_t *prev_dev, const uint8_t *cur_dev, int64_t n, double t_i,
                      uint8_t *out_dev, void *stream);
/* ast_corner_score (detector.py:58-71) of n points (xs, ys: int32, each at
 * least 3 pixels inside the layer; the caller validates) at any arc_len >= 1. */
int vf_ast_corner_score(const uint8_t *layer_dev, int w, int h, int64_t pitch, int n, const int32_t *xs_dev,
                        const int32_t *ys_dev, int arc_len, int32_t *out_dev, void *stream);
/* sad_block (temporal.py:63-67) of `count` pairs of patch_bytes-byte patches. */
int vf_sad_block(const uint8_t *a_dev, const uint8_t *b_dev, int64_t patch_bytes, int count, int64_t *out_dev,
                 void *stream);
/* binning_histogram (masking.py:96-119): hist_dev (rows x cols) uint64, zeroed by the call. */
int vf_binning_histogram(int n, const double *xs_dev, const double *ys_dev, int W, int H, int rows,
                         int cols, uint64_t *hist_dev, void *stream);
/* upsample_mask (masking.py:139-148). */
int vf_upsample_mask(const uint8_t *bits_dev, int rows, int cols, int cell_w, int cell_h, int W, int H,
                     uint8_t *full_dev, void *stream);
/* _mask_values (masking.py:157-165): mask bit under each rounded, clamped position. */
int vf_mask_values(const uint8_t *full_dev, int W, int H, int n, const double *xs_dev,
                   const double *ys_dev, uint8_t *out_dev, void *stream);

/* --- temporal block-matching baseline (temporal.py) --- */
/* baseline_step's per-feature search (temporal.py:274-308 with spiral_search
 * :183-226) for n features of one stream: the patch x patch block around the
 * rounded (x, y) of prev_dev is searched in cur_dev (both w x h, row pitch).
 * found_dev[i] = 1 with the new position and SAD when the best SAD < t_bm.
 * gop: GopConfig fields as in vf_config (zero = defaults).  Async on stream. */
int vf_block_match(const uint8_t *prev_dev, const uint8_t *cur_dev, int w, int h, int64_t pitch, int n,
                   const double *x_dev, const double *y_dev, const vf_config *gop, double *nx_dev, double *ny_dev,
                   double *sad_dev, uint8_t *found_dev, void *stream);

/* --- output formats (report.py:102-113) ----------------- */
/* The feature lines of report.dump_features for n features (HOST buffers):
 * "%.4f %.4f %.4f %.6f <origin> <128 hex>\n" per feature, origin "detected"
 * (0) or "propagated" (1), desc64 = 64 packed bytes per feature.  Writes at
 * most cap bytes to out; *len = the full text length (VF_ERR_CAPACITY with the
 * needed length if cap is too small).  Multi-threaded, host only. */
int vf_format_features(int64_t n, const double *x, const double *y, const double *sigma, const double *theta,
                       const uint8_t *origin, const uint8_t *desc64, char *out, int64_t cap, int64_t *len);

/* --- descriptor matching (matching.py:47-94) -------- */
/* hamming_matrix (matching.py:73-77, _hamming_matrix_jit :56-66): out[i * ld + j]
 * = popcount(q_i XOR r_j) over nbytes packed bytes (any nbytes >= 1; int32).
 * q_dev: nq x nbytes, r_dev: nr x nbytes, row-major packed (np.packbits rows). */
int vf_hamming_matrix(const uint8_t *q_dev, int64_t nq, const uint8_t *r_dev, int64_t nr, int nbytes,
                      int32_t *out_dev, int64_t ld, void *stream);
/* radius_match (matching.py:80-94): every (i, j) with Hamming distance <= t_m,
 * in np.nonzero order (query-major, then reference), as three int32 arrays of
 * capacity cap.  Synchronizes; *n_matches = number of matches.  If cap is too
 * small returns VF_ERR_MATCH_CAPACITY with *n_matches = the required count. */
int vf_radius_match(const uint8_t *q_dev, int64_t nq, const uint8_t *r_dev, int64_t nr, int nbytes, int t_m,
                    int32_t *q_idx_dev, int32_t *r_idx_dev, int32_t *dist_dev, int64_t cap,
                    int64_t *n_matches, void *stream);
/* Device time of the distance kernel of vf_radius_match (CUDA events around
 * it on the call's stream), for benchmarks.  enable = 1: reset and start
 * accumulating; enable = 0: stop; *ms (if non-null) = the accumulated time. */
int vf_match_timing(int enable, double *ms);

/* --- geometric verification (matching.py:97-220) ---- */
/* ransac_homography (matching.py:151-192) for n_problems match sets at once.
 * offsets (HOST, n_problems + 1, offsets[0] = 0): problem p owns points
 * [offsets[p], offsets[p+1]) of src_dev / dst_dev, (x, y) fp64 pairs (16-byte
 * aligned) of the matched query / reference keypoints.  Every problem draws
 * its minimal samples from np.random.default_rng(seed) exactly as the
 * reference.  Outputs (device): H_dev[9 p ..] the row-major homography (NaN if
 * none), inlier_dev[i] 1 for a final inlier, n_inliers_dev[p] the inlier
 * count or -1 when the reference returns (None, []).  Asynchronous. */
int vf_ransac_homography(int n_problems, const int64_t *offsets, const double *src_dev, const double *dst_dev,
                         int iters, double reproj_tol, uint64_t seed, double *H_dev, uint8_t *inlier_dev,
                         int32_t *n_inliers_dev, void *stream);
/* The minimal-sample table of the above: out[4 k ..] = the k-th
 * default_rng(seed).choice(n, 4, replace=False), n >= 4.  Device generator
 * (jump-ahead, asynchronous) and the same stream on the host (no GPU needed). */
int vf_ransac_samples(uint64_t seed, int64_t n, int iters, int32_t *out_dev, void *stream);
int vf_ransac_samples_host(uint64_t seed, int64_t n, int iters, int32_t *out);

#ifdef __cplusplus
}
#endif
#endif /* VIDFEAT_B200_H */
