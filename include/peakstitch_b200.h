/*
 * peakstitch_b200 -- C-ABI of the B200 (sm_100a) LP-SIFT hot path:
 *   detect -> describe -> match -> RANSAC-score
 *
 * This is the drop-in boundary for the reference package `peakstitch`
 * (/root/reference/pkg/src/peakstitch).  The reference has no FFI of its own;
 * its boundary is four Python entry points, each replaced here by one C entry
 * point (the Python mirror in paper_2405_08578_b200/ keeps their names,
 * signatures and exceptions):
 *
 *   ps_detect        <- detect_features(img, scales, dedupe)   detector.py:154-172
 *   ps_describe      <- describe_features(img, features, cfg)  descriptor.py:259-269
 *                       (and compute_descriptor, descriptor.py:219-256)
 *   ps_match         <- match_features(set1, set2, cfg)        matcher.py:57-95
 *   ps_ransac_rigid  <- ransac_rigid(pairs, cfg)               registration.py:149-203
 *   ps_estimate_rigid<- estimate_rigid(src, dst)               registration.py:107-131
 *
 * (line numbers are those of the reference files as shipped.)
 *
 * Conventions
 *  - Every function returns an int status (enum ps_status).  Status codes map
 *    one-to-one onto the reference's exceptions (errors.py:4-17).  No C++
 *    exception and no abort() crosses this boundary.
 *  - All array arguments are DEVICE pointers unless the parameter name says
 *    `host_`.  Buffers are caller-owned; scratch is a caller-provided device
 *    workspace whose size the matching *_plan call reports.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is enqueued asynchronously; results are valid once the stream is
 *    synchronised.  Outcomes that depend on data (e.g. "no consensus") are
 *    reported through device-side info words, not the return status.
 *  - No hidden global mutable state other than the launch counter and the
 *    thread-local last-error message / match statistics; no environment
 *    variables are read; all calls are re-entrant.
 */
#ifndef PEAKSTITCH_B200_H
#define PEAKSTITCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 6

#if defined(__GNUC__)
#define PS_API __attribute__((visibility("default")))
#else
#define PS_API
#endif

enum ps_status {
  PS_OK = 0,
  PS_ERR_CONFIG = 1,       /* peakstitch.errors.ConfigError           */
  PS_ERR_VALUE = 2,        /* ValueError (geometry / region checks)    */
  PS_ERR_DEGENERATE = 3,   /* peakstitch.errors.DegenerateSampleError */
  PS_ERR_REGISTRATION = 4, /* peakstitch.errors.RegistrationError     */
  PS_ERR_CUDA = 5,         /* CUDA runtime error                       */
  PS_ERR_ARGUMENT = 6,     /* bad pointer / size / unsupported layout  */
  PS_ERR_CAPACITY = 7      /* output capacity too small                */
};

enum ps_pixel_type {
  PS_PIXELS_U8 = 0,  /* raw 8-bit intensities; the linear ramp of
                        apply_linear_ramp (imaging.py:113-132) is fused:
                        P[r,c] = fl(I[r,c] + fl((r*nc+c+1) * alpha))        */
  PS_PIXELS_F64 = 1, /* an already-ramped float64 raster (RampedImage.pixels) */
  PS_PIXELS_F64_RAW = 2, /* float64 intensities (IntensityImage.pixels); ramp
                           fused as for PS_PIXELS_U8                          */
  PS_PIXELS_RGB8 = 3  /* interleaved 8-bit RGB (load_image of an RGB file,
                         imaging.py:71-93): the grey of a pixel is
                         gray_lut[R<<16 | G<<8 | B] -- the run host's own
                         to_grayscale bits (imaging.py:66-68) --
                         and the ramp is fused as for PS_PIXELS_U8.
                         row_pitch / image_stride count pixels (3 bytes).   */
};

enum ps_match_strategy {
  PS_MATCH_NEAREST = 0,       /* "nearest_neighbor": mutual NN + dist < delta_s
                                 (matcher.py:71-79)                            */
  PS_MATCH_THRESHOLD_ALL = 1, /* "threshold_all": every dist < delta_s
                                 (matcher.py:69-70)                            */
  PS_MATCH_RATIO = 2          /* "ratio_test": an EXTRA strategy the reference
                                 does not have (the north star's
                                 Lowe ratio): row i keeps its first nearest
                                 neighbour j when d1 < r * d2, d2 the row's
                                 second-smallest distance (a duplicate of the
                                 best counts); r is passed in `delta_s`, in
                                 (0, 1]; no mutual check, no absolute cut    */
};
/* Path selection, OR-ed into `strategy` per call (no environment switches):
 * by default nearest_neighbor on 128-d descriptors uses the tensor-core
 * kernels when n1 * n2 >= 2^20 and the float64 CUDA-core kernels otherwise;
 * results are identical either way (contract P3). */
#define PS_MATCH_FORCE_EXACT 0x100 /* float64 CUDA-core kernels                */
#define PS_MATCH_FORCE_TC 0x200    /* tensor-core kernels where the strategy
                                      has them (nearest_neighbor, dim 128)     */

/* A batch of B equally sized images in device memory. */
typedef struct ps_image_batch {
  const void* data;     /* device pointer to image 0, pixel (0,0)            */
  int32_t pixel_type;   /* enum ps_pixel_type                                */
  int32_t batch;        /* B >= 1                                            */
  int32_t nr, nc;       /* rows, columns                                     */
  int64_t row_pitch;    /* elements between consecutive rows  (>= nc)        */
  int64_t image_stride; /* elements between consecutive images              */
  double alpha;         /* ramp coefficient (fused-ramp pixel types)         */
  const double* gray_lut; /* PS_PIXELS_RGB8: device table of 2^24 greys, or
                             NULL for the checked FMA formula (see below)    */
} ps_image_batch;

/* Keypoints of a batch, image b occupying slots [b*cap, b*cap + count[b]).
 * Field meaning follows FeaturePoint (detector.py:71-80); polarity 0 = "max",
 * 1 = "min".  scale / polarity / window may be NULL on output (not written)
 * and `scale` may be NULL on input to ps_describe (then every keypoint has
 * scale `default_scale`). */
typedef struct ps_keypoints {
  int32_t* row;
  int32_t* col;
  double* value;
  int32_t* scale;
  int8_t* polarity;
  int32_t* window;
  int32_t* count; /* device [B] */
  int64_t cap;    /* slots per image */
} ps_keypoints;

PS_API int ps_abi_version(void);
PS_API const char* ps_last_error(void);      /* thread-local message of the last failure */
PS_API uint64_t ps_kernel_launches(void);    /* kernels launched by this library so far   */
PS_API int ps_device_sync(void* stream);     /* cudaStreamSynchronize + error check       */
/* Roofline probe (bench.py): `blocks` x 256 threads each run 8 independent
 * float64 FMA chains of `iters` steps; *out_flops = the FLOPs enqueued (2 per
 * FMA).  Time it with events on `stream` to get the box's FP64-pipe peak --
 * the denominator of the describe kernel's compute roofline.
 * sink: device double[blocks] (never written in practice). */
PS_API int ps_probe_fp64_fma(int64_t iters, int32_t blocks, double* sink, double* out_flops, void* stream);
/* Roofline probe (bench.py): `blocks` CTAs (one per SM) each allocate all 512
 * TMEM columns and 16 warps read them with 64-column tcgen05.ld, two per
 * wait, `iters` times; *out_bytes = the bytes read.  Timed with events it is
 * the tensor-memory read bandwidth that bounds the tensor-core matcher's
 * epilogue (every fp32 distance accumulator is read once). */
PS_API int ps_probe_tmem_read(int64_t iters, int32_t blocks, uint32_t* sink, double* out_bytes, void* stream);

/* ---- detect: detector.py:154-172 --------------------------------------- */
/* Validates the scale set (ScaleSet rules, detector.py:33-68) against the
 * image and reports the per-image output capacity and workspace size. */
PS_API int ps_detect_plan(int32_t batch, int32_t nr, int32_t nc, const int32_t* host_scales,
                   int32_t n_scales, int32_t dedupe, int64_t* cap_out,
                   size_t* workspace_bytes_out);
PS_API int ps_detect(const ps_image_batch* img, const int32_t* host_scales, int32_t n_scales,
              int32_t dedupe, ps_keypoints* out, void* workspace, size_t workspace_bytes,
              void* stream);

/* ---- describe: descriptor.py:219-269 ------------------------------------ */
/* host_scale_set lists every scale that may occur in kp->scale (the ScaleSet);
 * region sizes are derived on the host per scale (descriptor.py:82-95, 118-131).
 * Keypoints may lie anywhere (the region is translated inward as
 * _fit_region does, descriptor.py:118-131) and must carry a scale of the set
 * (slots that do not are skipped, unwritten).  Output row k of out_desc32 /
 * out_desc64 ([B*cap, 8*d*d], row-major) is the descriptor of keypoint slot
 * k; slots >= count are not written.  Either output pointer may be NULL. */
PS_API int ps_describe(const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                const int32_t* host_scale_set, int32_t n_scale_set, double beta0, int32_t d,
                int32_t l_max, int32_t orientation_normalize, float* out_desc32,
                double* out_desc64, void* stream);
/* ps_describe with an explicit kernel policy (tests / A-B measurements):
 * PS_DESCRIBE_AUTO as ps_describe: when only out_desc32 is requested, w = 8
 * keypoints (d = 4) of 8-bit rasters run the float32 throughput kernel
 * (descriptors ~1e-7 relative from the reference's float64 ones, every
 * orientation-bin decision certified or taken in float64), everything else
 * the float64 kernels (~1e-14); PS_DESCRIBE_PRECISE the float64 kernels for
 * every keypoint; PS_DESCRIBE_GENERAL the general float64 kernel for every
 * keypoint; PS_DESCRIBE_SINGLE the one-keypoint-per-warp float64 fast kernel
 * instead of the two-keypoints-per-warp one (w = 8). */
enum ps_describe_policy {
  PS_DESCRIBE_AUTO = 0,
  PS_DESCRIBE_GENERAL = 1,
  PS_DESCRIBE_SINGLE = 2,
  PS_DESCRIBE_PRECISE = 3
};
/* OR-ed into `policy`: the caller vouches that keypoint slots 2w / 2w+1 hold
 * the max / min of window w of the default scale's row-major window grid --
 * what ps_detect writes when dedupe leaves one evaluated scale (a nested
 * scale set).  A performance hint only: keypoints that are not where it says
 * are still described correctly, by the float64 kernel. */
#define PS_DESCRIBE_WINDOW_SLOTS 0x100
PS_API int ps_describe_ex(const ps_image_batch* img, const ps_keypoints* kp, int32_t default_scale,
                const int32_t* host_scale_set, int32_t n_scale_set, double beta0, int32_t d,
                int32_t l_max, int32_t orientation_normalize, float* out_desc32,
                double* out_desc64, int32_t policy, void* stream);

/* ---- match: matcher.py:57-95 -------------------------------------------- */
PS_API int ps_match_plan(int64_t n1, int64_t n2, int32_t dim, int32_t strategy, int64_t cap,
                  size_t* workspace_bytes_out);
/* `strategy` is a ps_match_strategy, optionally OR-ed with a PS_MATCH_FORCE_*
 * flag.  desc1 [n1, dim], desc2 [n2, dim] row-major, float32 (desc_is_f64 = 0; the
 * values are upcast to float64 exactly) or float64 (desc_is_f64 = 1).  All
 * distance arithmetic is the reference's float64 arithmetic.
 * Writes up to `cap` pairs sorted by (delta, ref1, ref2) and the total pair
 * count to *out_count (device int64); if the total exceeds cap only the
 * first `cap` are valid and the caller retries with a larger cap. */
PS_API int ps_match(const void* desc1, int64_t n1, const void* desc2, int64_t n2, int32_t dim,
             int32_t desc_is_f64, double delta_s, int32_t strategy, int32_t* out_ref1, int32_t* out_ref2,
             double* out_delta, int64_t* out_count, int64_t cap, void* workspace,
             size_t workspace_bytes, void* stream);

/* As ps_match without any host synchronisation: every grid is sized from
 * n1 / n2 (the kernels read the device-side counts), so a sequence of calls
 * -- e.g. the pairs of a pairwise table -- is enqueued back to back and the
 * caller reads all *out_count values with one copy.  Same results as
 * ps_match; cap must be >= min(n1, n2) for nearest_neighbor. */
PS_API int ps_match_async(const void* desc1, int64_t n1, const void* desc2, int64_t n2, int32_t dim,
                   int32_t desc_is_f64, double delta_s, int32_t strategy, int32_t* out_ref1,
                   int32_t* out_ref2, double* out_delta, int64_t* out_count, int64_t cap,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Many nearest_neighbor matches in one launch sequence: pair q matches
 * descriptor set pair_a[q] against set pair_b[q] (the pairwise-table loop,
 * mosaic.py:79-112, calling match_features, matcher.py:57-95, per pair).
 * set_desc: host array of n_sets device pointers to [set_rows[s], 128]
 * row-major float32 (desc_is_f64 = 0) or float64 rows; pair_a / pair_b: host
 * int32 arrays of n_pairs set indices.  set_count: NULL, or a host array of
 * n_sets device int32 pointers (each NULL or the set's live row count,
 * clamped to [0, set_rows[s]]): set_rows is then the set's capacity (grids,
 * workspace, out_stride) and the kernels read the count on the device, so a
 * captured graph stays valid when the counts change between replays (a
 * camera rig's frames).  Each set's duplicate grouping and
 * tensor-core operand tiles are built once however many pairs it enters, and
 * every stage runs as one launch for all pairs.  Pair q's matches, sorted by
 * (delta, ref1, ref2), go to row q of out_ref1 / out_ref2 / out_delta (device
 * [n_pairs, out_stride], out_stride >= min(set_rows[a], set_rows[b]) for every
 * pair) and its count to out_count[q] (device int64).  No host
 * synchronisation (capturable); results equal ps_match's pair by pair.
 * Limits: dim = 128, n_sets <= 512, n_pairs <= 256. */
PS_API int ps_match_batch_plan(int32_t n_sets, const int64_t* set_rows, int32_t n_pairs, int32_t dim,
                               size_t* workspace_bytes_out);
PS_API int ps_match_batch_async(int32_t n_sets, const void* const* set_desc, const int64_t* set_rows,
                                const int32_t* const* set_count, int32_t n_pairs, const int32_t* pair_a, const int32_t* pair_b, int32_t dim,
                                int32_t desc_is_f64, double delta_s, int32_t* out_ref1, int32_t* out_ref2,
                                double* out_delta, int64_t out_stride, int64_t* out_count, void* workspace,
                                size_t workspace_bytes, void* stream);

/* One direction of nearest_neighbor matching: out_index[i] / out_dist[i] =
 * the exact first argmin over the rows of Y of the reference distance to row
 * i of X (matcher.py:74 with _distance_matrix :48-54).  The building block of
 * row-sharded matching across GPUs (each rank: its rows of A vs all of B,
 * and the candidate columns vs its rows).  flags: 0 or one PS_MATCH_FORCE_*. */
PS_API int ps_nearest_plan(int64_t nx, int64_t ny, int32_t dim, int32_t flags, size_t* workspace_bytes_out);
PS_API int ps_nearest(const void* X, int64_t nx, const void* Y, int64_t ny, int32_t dim, int32_t desc_is_f64,
                      int32_t flags, int32_t* out_index, double* out_dist, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Statistics of the calling thread's last tensor-core ps_match (diagnostic):
 * out[0..5] = distinct rows of desc1, of desc2, candidate columns, rows
 * whose near-ties were enumerated, enumerated pairs (0: not tracked),
 * tensor-core FLOPs issued (fp16 MMA, both passes). */
PS_API int ps_match_stats(int64_t* out, int32_t n);

/* Gather (x, y) = (col, row) float64 point pairs of matches
 * (registration.py:143-146) from two keypoint arrays. */
PS_API int ps_pair_points(const int32_t* ref1, const int32_t* ref2, const int64_t* count,
                   const int32_t* row1, const int32_t* col1, const int32_t* row2,
                   const int32_t* col2, double* src_xy, double* dst_xy, int64_t cap,
                   void* stream);

/* ---- batched registration: registration.py:143-203 per pair ------------- */
/* One matched pair of a batch: its two images' keypoint coordinates (device
 * int32), its capacity n_cap = min(n1, n2) (>= min_inliers, <= ref_stride),
 * and the PCG64 state of default_rng(seed) (numpy bit_generator.state:
 * state, inc, has_uint32, uinteger) that the reference's RANSAC draws from
 * (registration.py:164).  live = 0 skips the pair (its block is untouched). */
typedef struct {
  const int32_t *row1, *col1, *row2, *col2;
  int64_t n_cap;
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  int32_t has_uint32;
  uint32_t uinteger;
  int32_t live;
} ps_register_pair;
/* The point gather (ps_pair_points) and RANSAC (ps_ransac_samples_async +
 * ps_ransac_rigid_async) of up to 256 matched pairs as one launch per stage:
 * pair q's matches are row q of ref1 / ref2 (device int32 [n_pairs,
 * ref_stride], e.g. ps_match_batch_async's outputs) with count[q] (device
 * int64).  Pair q's result goes to out_block + q * block_stride (doubles):
 * [0, 3) model (theta, t_x, t_y), [3] rms, [4, 8) int64 status / consensus /
 * inliers / best iteration, and from byte 64 the uint8 inlier mask
 * (block_stride >= 8 + ceil(ref_stride / 8)).  Results equal the per-pair
 * calls'; no host synchronisation. */
PS_API int ps_register_batch_plan(int32_t n_pairs, int64_t n_cap, int32_t iterations,
                                  size_t* workspace_bytes_out);
PS_API int ps_register_batch_async(int32_t n_pairs, const ps_register_pair* pairs, const int32_t* ref1,
                                   const int32_t* ref2, int64_t ref_stride, const int64_t* count,
                                   int32_t iterations, double inlier_tol, int32_t min_inliers,
                                   double* out_block, int64_t block_stride, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* ---- RANSAC: registration.py:107-203 ------------------------------------ */
/* samples: device int32 [iterations, 2], the reference's index stream
 * (registration.py:164, 170-173), generated on the host from the seed.
 * out_model: device double[3] = (theta, t_x, t_y) of the refit, theta in
 * (-pi, pi].  out_mask: device uint8[n] final inlier mask.
 * out_info: device int64[4] = (status, consensus_size, n_inliers, best_iter)
 * with status PS_OK or PS_ERR_REGISTRATION; best_iter is -1 when the maximal
 * consensus is below min_inliers (the call fails whatever the rms order, so
 * no winner is selected: registration.py:187-190).  out_rms: device double[1]. */
PS_API int ps_ransac_plan(int64_t n, int32_t iterations, size_t* workspace_bytes_out);
PS_API int ps_ransac_rigid(const double* src_xy, const double* dst_xy, int64_t n,
                    const int32_t* samples, int32_t iterations, double inlier_tol,
                    int32_t min_inliers, double* out_model, uint8_t* out_mask,
                    int64_t* out_info, double* out_rms, void* workspace,
                    size_t workspace_bytes, void* stream);
/* The reference's RANSAC index stream (registration.py:164, 170-173) on the
 * device: numpy's PCG64 state (Generator.bit_generator.state: 128-bit state
 * and increment as hi/lo words, has_uint32, uinteger) -> out_samples[2*iters]
 * = (i, j) per iteration, bit-identical to the scalar draws
 * rng.integers(0, n), rng.integers(0, n - 1), j += j >= i.  scratch: one
 * device int32.  2 <= n < 2^31. */
PS_API int ps_ransac_samples(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                             int32_t has_uint32, uint32_t uinteger, int64_t n, int32_t iterations,
                             int32_t* out_samples, int32_t* scratch, void* stream);
/* Asynchronous forms for a chain with no host round trip (match ->
 * pair_points -> RANSAC, e.g. a pairwise table captured in one CUDA graph):
 * the correspondence count is read on the device from *n_dev (a ps_match
 * out_count); n_cap >= *n_dev sizes the workspace (ps_ransac_plan(n_cap)).
 * A count below min_inliers (or below 2) yields status PS_ERR_REGISTRATION
 * in out_info[0] instead of an error return. */
PS_API int ps_ransac_rigid_async(const double* src_xy, const double* dst_xy, const int64_t* n_dev,
                          int64_t n_cap, const int32_t* samples, int32_t iterations, double inlier_tol,
                          int32_t min_inliers, double* out_model, uint8_t* out_mask,
                          int64_t* out_info, double* out_rms, void* workspace,
                          size_t workspace_bytes, void* stream);
PS_API int ps_ransac_samples_async(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                            uint64_t inc_lo, int32_t has_uint32, uint32_t uinteger,
                            const int64_t* n_dev, int32_t iterations, int32_t* out_samples,
                            int32_t* scratch, void* stream);
/* Least-squares rigid fit of dst ~ H(src) over all n points; out_info[0] is
 * PS_OK or PS_ERR_DEGENERATE. */
PS_API int ps_estimate_rigid(const double* src_xy, const double* dst_xy, int64_t n,
                      double* out_model, int64_t* out_info, void* stream);

/* ---- RGB ingest ------------------------------------
 * The grey of an RGB8 pixel is the reference's `rgb @ LUMA` (imaging.py:66-68)
 * as the run host's BLAS computes it: either gray_lut (all 2^24 triples,
 * built on the host with numpy) or -- gray_lut == NULL -- the fused formula
 * fma(B, .114, fma(R, .299, G * .587)), which ps_gray_table_check verifies
 * against such a table (out_mismatches = 0 means the formula is exact here). */
PS_API int ps_gray_table_check(const double* gray_lut, unsigned long long* out_mismatches, void* stream);
/* to_grayscale of an RGB8 batch into a float64 [B, nr, nc] raster (row-major,
 * dense). */
PS_API int ps_rgb_to_gray(const ps_image_batch* img, double* out, void* stream);

/* ---- compositor --------------------------------------
 * ps_warp_and_blend <- warp_and_blend(images, placements, canvas, blend,
 *                      resample)                         compositor.py:84-160
 * One placed image.  The caller supplies the INVERSE transform's cos / sin /
 * translation exactly as RigidTransform.inverse() + transform_points compute
 * them (registration.py:49-55, 66-73; host libm) and the canvas block the
 * reference derives from the snapped corners (compositor.py:122-129). */
typedef struct ps_placement {
  const void* data;   /* device pointer, pixel (0,0)                          */
  int32_t pixel_type; /* PS_PIXELS_U8 (uint8) or PS_PIXELS_F64 (float64)      */
  int32_t nr, nc;
  int32_t r_lo, r_hi, c_lo, c_hi; /* canvas block [r_lo,r_hi) x [c_lo,c_hi)  */
  int32_t pad_;
  int64_t row_pitch;  /* elements                                            */
  double cos_t, sin_t, t_x, t_y;  /* inverse transform: canvas frame -> image */
} ps_placement;

enum ps_blend { PS_BLEND_FEATHER = 0, PS_BLEND_OVERWRITE = 1 };
enum ps_resample { PS_RESAMPLE_BILINEAR = 0, PS_RESAMPLE_NEAREST = 1 };

/* Composite n placements (host array, in placement order) into a
 * height x width float64 canvas whose pixel (r, c) is frame point
 * (c + dx, r + dy).  out and weightmap are device arrays of height*width
 * doubles (row-major); weightmap receives the raw accumulated weights
 * (Canvas.weightmap).  Unknown blend / resample -> PS_ERR_VALUE. */
PS_API int ps_warp_and_blend(const ps_placement* host_placements, int32_t n, int32_t height,
                             int32_t width, int32_t dx, int32_t dy, int32_t blend,
                             int32_t resample, double* out, double* weightmap, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PEAKSTITCH_B200_H */
