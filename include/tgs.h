/*
 * tgs.h — C ABI of the B200 rasterizer library (libtgs.so).
 *
 * This is the drop-in boundary for the reference's rasterizer hot path
 * (slimsplat, /root/reference/pkg/src/slimsplat).  The reference's own
 * "kernel ABI" is three numba functions that take caller-allocated positional
 * arrays and write them in place (_kernels.py:12-36, 92-115, 184-202), with the
 * Python layer owning the contract (_kernels.py:4-5).  This header generalises
 * that ABI to the whole path the reference runs per training step:
 *
 *   tgs_preprocess_forward   replaces rasterizer._prepare minus binning
 *                            (rasterizer.py:167-197: masking.py:21-43,84-86,
 *                            geometry.py:19-41,74-77,138-195, sh.py:135-161)
 *   tgs_count_tiles          the per-Gaussian rect/count half of bin_tiles
 *                            (rasterizer.py:112-128)
 *   tgs_bin_gaussians +      the sort half of bin_tiles
 *   tgs_bin_instances        (rasterizer.py:130-148: repeat, lexsort, CSR)
 *   tgs_blend_forward        _kernels.forward_kernel (_kernels.py:12-89)
 *   tgs_blend_backward       _kernels.backward_kernel (_kernels.py:92-181)
 *   tgs_preprocess_backward  render_backward after the kernel
 *                            (rasterizer.py:375-419, sh.py:164-215,
 *                            geometry.py:44-71,80-89,198-251, masking.py:28-31)
 *   tgs_loss_l1_ssim         training.total_loss image terms (training.py:61-89,
 *                            metrics.py:138-188)
 *   tgs_adam_step            optim.Adam.update (optim.py:37-49)
 *   tgs_gather_rows          cloud.take / Adam.compact row compaction
 *                            (cloud.py:86-89, optim.py:51-55)
 *   tgs_select_rows          the np.nonzero row selection of the prunings
 *                            (masking.py:70-81, significance.py:81-99)
 *   tgs_significance_scores  significance.significance_scores (significance.py:45-78)
 *   tgs_significance_keep    significance.prune_by_significance's row selection
 *                            (significance.py:81-99)
 *
 * Conventions (all entry points):
 *   - every pointer is DEVICE memory owned by the caller, row-major, float32
 *     unless stated; the library never allocates persistent memory and never
 *     frees caller memory; scratch comes from caller-provided workspaces;
 *   - every call is asynchronous on the given stream (cudaStream_t; NULL = the
 *     legacy default stream) and returns a TGS_* status code; no exception or
 *     C++ type crosses the ABI;
 *   - no global mutable state: calls are re-entrant per stream.
 */
#ifndef TGS_H_
#define TGS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *tgs_stream_t; /* == cudaStream_t */

#if defined(__GNUC__)
#define TGS_API __attribute__((visibility("default")))
#else
#define TGS_API
#endif

enum {
  TGS_OK = 0,
  TGS_ERR_INVALID = 1,             /* -> ContractViolationError */
  TGS_ERR_DEGENERATE_ROTATION = 2, /* -> DegenerateRotationError (geometry.py:23-24) */
  TGS_ERR_CUDA = 3,                /* a CUDA launch/API call failed */
  TGS_ERR_UNSUPPORTED = 4,         /* e.g. tile_size > 32 */
  TGS_ERR_CAPACITY = 5             /* caller buffer smaller than required */
};

/* Per-Gaussian projected record written by tgs_preprocess_forward, 12 floats:
 *   [0..1] means2d (pixels)      [2..4] conic (a, b, c) = inverse cov2d packed
 *   [5]    alpha (sigmoid(o)*M)  [6..8] rgb (SH colour, clamped >= 0)
 *   [9]    depth (camera z)      [10]   radius (3 sigma, pixels)
 *   [11]   screen area 9*pi*sqrt(det), 0 when not visible
 * 48 B = one 16 B-aligned record, so the blend kernels stage a Gaussian with
 * three 16 B loads.  Rows of non-visible Gaussians are zero. */
#define TGS_SPLAT_FLOATS 12
/* Per-Gaussian screen-space partials written by tgs_blend_backward, 9 floats:
 *   [0..1] dL/dmeans2d  [2..4] dL/dcov2d packed (g00, g01 both slots, g11)
 *   [5] dL/dalpha       [6..8] dL/drgb          (_kernels.py:111-115) */
#define TGS_DSPLAT_FLOATS 9
/* Per-Gaussian EXACT BLEND-DECISION record (optional output of the preprocess,
 * optional input of every blend entry point), 8 floats, 32 B aligned:
 *   [0] cut_lo, [1] cut_hi  float32 bracket, in log2 units, of the reference's
 *        float64 blend cut max(-4.5, ln(1/(255 alpha))) widened by a bound on the
 *        float32 exponent's error over the Gaussian's footprint: a pixel whose
 *        float32 exponent e2 is >= cut_hi (and <= 0) blends in float64 too, one
 *        below cut_lo does not; in between (or e2 > 0) the blend kernels decide in
 *        float64 (_kernels.py:62-72);
 *   [2..3] means2d, [4..6] conic: float64 value minus the float32 record value, so
 *        record + residual reconstructs the float64 projection (~1e-13);
 *   [7]  the float64 cut minus cut_lo (log2 units), or, when the float32 alpha
 *        exceeds 0.9899 so that alpha exp(e) can reach the 0.99 clamp (the cut is
 *        then -4.5), the clamp exponent ln(0.99 / alpha): the blend kernels bracket
 *        it with the cut's error bound ((cut_hi - cut_lo) / 2) and decide the
 *        backward's a <= 0.99 (_kernels.py:157-168) in float64 for the blended pairs
 *        above the bracket's lower end (rare: near the Gaussian's centre).
 * Rows of non-visible Gaussians are zero.  A blend call without records
 * (exact == NULL) decides every pair in float32. */
#define TGS_EXACT_FLOATS 8

typedef struct {
  float fx, fy, cx, cy;
  float R[9];      /* world -> camera, row-major (cameras.py:25) */
  float t[3];      /* x_cam = R x + t */
  float center[3]; /* -R^T t, computed by the caller (cameras.py:42-45) */
  int32_t width, height;
  /* float64 third row of [R | t]: the depth SORT KEY is computed in float64 so the
   * tile lists order exactly like the reference's float64 np.lexsort (float32
   * depths collide ~2k times at 200k Gaussians and would reorder blends). */
  double depth_row[4];
  /* The camera in float64 (the reference's own values): the float64 projection of
   * the exact blend-decision records (TGS_EXACT_FLOATS below). */
  double fx64, fy64, cx64, cy64;
  double R64[9];
  double t64[3];
} tgs_camera;

typedef struct {
  float lowpass_s;         /* added to both cov2d diagonals (geometry.py:170-172) */
  float near_plane;        /* cull t_z <= near (geometry.py:154) */
  /* Hard masks are evaluated in logit space: sigmoid(m) > eps  <=>  m > logit(eps).
   * The caller passes logit(eps) in float64 rounded DOWN to float32, which makes
   * the float32 comparison identical to the reference's float64 one
   * (masking.py:21-25).  Same for the alpha-skip gate sigmoid(o) >= 1/255
   * (rasterizer.py:178) with logit(1/255) rounded UP. */
  float mask_logit_min;    /* keep Gaussian iff mask_logit > mask_logit_min */
  float sh_mask_logit_min; /* keep SH band iff sh_mask_logit > sh_mask_logit_min */
  float opacity_logit_min; /* alpha-skip survivor iff opacity_logit >= opacity_logit_min */
  float background[3];
  int32_t active_sh_degree; /* 0..3 */
  int32_t tile_size;        /* 1..32 */
  int32_t compute_sh_rest_grads;
  int32_t reserved;
  double lowpass_s64;       /* lowpass_s in float64 (the exact blend-decision records) */
} tgs_settings;

typedef struct {
  const float *positions;      /* (n, 3) */
  const float *log_scales;     /* (n, 3) */
  const float *rotations;      /* (n, 4) w, x, y, z */
  const float *opacity_logits; /* (n,) */
  const float *sh_dc;          /* (n, 3) */
  const float *sh_rest;        /* (n, 15, 3) band-major */
  const float *mask_logits;    /* (n,) */
  const float *sh_mask_logits; /* (n, 3) */
  int64_t n;
} tgs_cloud;

typedef struct { /* densification statistics (training.py:333-338; TrainState.reset_stats,
                  * training.py:126-130); any pointer may be NULL */
  float *grad_accum;   /* (n,) += ||mean2d_screen * (W/2, H/2)|| per view the row is visible in */
  int32_t *grad_count; /* (n,) += 1 per view the row is visible in */
  float *area_max;     /* (n,) = max(area_max, screen_areas) over the views */
} tgs_densify_stats;

typedef struct { /* CloudGrads (cloud.py:110-126) */
  float *positions, *log_scales, *rotations, *opacity_logits;
  float *sh_dc, *sh_rest, *mask_logits, *sh_mask_logits;
  float *mean2d_screen; /* (n, 2); may be NULL */
} tgs_grads;

TGS_API int tgs_version(void);
/* Profiling builds only (-DTGS_COUNT_EXACT): pairs decided in float64 by the blend
 * kernels since the last reset (TGS_ERR_UNSUPPORTED otherwise; profiles/exact_pairs.py). */
TGS_API int tgs_debug_exact_pairs(unsigned long long *count, int32_t reset);
TGS_API const char *tgs_last_error_string(int status);

/* ---- (1) preprocess -----------------------------------------------------
 * splats (n, 12), visible (n,) 0/1, tiles_touched (n,) = number of tiles the
 * Gaussian's 3-sigma box covers (0 when not visible / off screen).
 * depth_keys (n,) uint64 or NULL: order-preserving bits of the float64 depth
 * (cam->depth_row . [x, 1]), the sort key consumed by tgs_bin_gaussians.
 * error_flag: device int32, OR-ed with 1 when a quaternion has norm < 1e-12;
 * the caller reads it back and raises DegenerateRotationError.
 * exact (n, 8) or NULL: the exact blend-decision records (TGS_EXACT_FLOATS). */
TGS_API int tgs_preprocess_forward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                           float *splats, uint8_t *visible, int32_t *tiles_touched, uint64_t *depth_keys,
                           int32_t *error_flag, float *exact, tgs_stream_t stream);
/* A batch of views in ONE pass over the parameters (the sh_rest block staged
 * once): per view v the same outputs as tgs_preprocess_forward into splats[v],
 * visible[v], tiles_touched[v], depth_keys[v] (may be NULL), bit-identical to a
 * single-view call with cams[v].  stats (may be NULL): area_max is updated with
 * the views' screen areas (the other two fields are the backward's).
 * exact (may be NULL; else exact[v] (n, 8), 16 B aligned): the exact
 * blend-decision records (TGS_EXACT_FLOATS) of every view. */
/* The exact blend-decision records (TGS_EXACT_FLOATS) of a batch of views from
 * their float32 records splats[v] (as written by the preprocess): the float64
 * projection of every visible row.  The preprocess entry points call it when
 * given `exact`; a pipelined caller can instead run it on another stream, since
 * only the blend kernels read the records (not the binning). */
TGS_API int tgs_exact_records_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                    int32_t nviews, const float *const *splats, float *const *exact,
                                    tgs_stream_t stream);
TGS_API int tgs_preprocess_forward_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                         int32_t nviews, float *const *splats, uint8_t *const *visible,
                                         int32_t *const *tiles_touched, uint64_t *const *depth_keys,
                                         int32_t *error_flag, const tgs_densify_stats *stats, float *const *exact,
                                         tgs_stream_t stream);

/* tiles_touched for arbitrary projected records (the bin_tiles(...) entry,
 * rasterizer.py:95-128): only splat fields means2d and radius are read. */
TGS_API int tgs_count_tiles(const float *splats, int64_t n, int32_t width, int32_t height, int32_t tile_size,
                    int32_t *tiles_touched, tgs_stream_t stream);

/* ---- (2) binning ----------------------------------------------------------
 * Sort order is the reference's np.lexsort((gid, depth, tile)) (rasterizer.py:143):
 * ascending tile, then depth, then Gaussian index.  Because all instances of a
 * Gaussian share its depth, the order is produced in two steps: a stable sort of
 * the on-screen GAUSSIANS by their 64-bit depth key (step A, one launch), then a
 * stable counting placement of the instances into their tile lists in that
 * depth order (step B) — no per-instance key is materialised.  Tiles are
 * restricted to tile rows [row_begin, row_end) (tile-row sharding); tile_offsets
 * has (row_end-row_begin)*tiles_x + 1 entries, relative to the band.
 *
 * depth_keys: per-Gaussian uint64 keys from tgs_preprocess_forward, or NULL to
 * key on the float32 splat depth (the raw-array bin_tiles entry).
 *
 * Step A: tgs_bin_gaussians() needs a workspace of tgs_bin_gaussians_workspace()
 * bytes, which must stay alive until step B returns.  It writes the instance count
 * to d_num_instances[0] (device int64) and, when error_flag (device int32, e.g.
 * tgs_preprocess_forward's) is not NULL, its value to d_num_instances[1] — so one
 * 16-byte device-to-host read returns both.
 * Step B: tgs_bin_instances() with num_instances read back by the caller and a
 * workspace of tgs_bin_instances_workspace() bytes (same band arguments). */
TGS_API int tgs_bin_gaussians_workspace(int64_t n, size_t *bytes);
/* Asynchronous device -> host copy on `stream` (the count read-back between step A
 * and step B; dst should be pinned host memory). */
TGS_API int tgs_memcpy_d2h_async(void *dst_host, const void *src_device, size_t bytes, tgs_stream_t stream);
TGS_API int tgs_bin_gaussians(const float *splats, const int32_t *tiles_touched, const uint64_t *depth_keys,
                      int64_t n, int32_t width,
                      int32_t height, int32_t tile_size, int32_t row_begin, int32_t row_end,
                      void *workspace, int64_t *d_num_instances, const int32_t *error_flag,
                      tgs_stream_t stream);
/* Instances per tile row (row_counts: tiles_y int64, accumulated): the replicated
 * histogram from which every rank derives the same balanced tile-row bands. */
TGS_API int tgs_row_histogram(const float *splats, const int32_t *tiles_touched, int64_t n, int32_t width,
                              int32_t height, int32_t tile_size, int64_t *row_counts, tgs_stream_t stream);
TGS_API int tgs_bin_instances_workspace(int64_t n, int64_t num_instances, int32_t width, int32_t height,
                                        int32_t tile_size, int32_t row_begin, int32_t row_end, size_t *bytes);
TGS_API int tgs_bin_instances(const float *splats, int64_t n, int32_t width, int32_t height, int32_t tile_size,
                      int32_t row_begin, int32_t row_end, void *gauss_workspace, int64_t num_instances,
                      void *workspace, int32_t *tile_offsets, int32_t *sorted_ids, tgs_stream_t stream);

/* ---- (3) forward blend ------------------------------------------------------
 * image (H, W, 3), transmit / weight_sum (H, W) float32, n_contrib / last_pos
 * (H, W) int32 (_kernels.py:83-89); hits (n,) int32 or NULL (record_hits).
 * Only pixels of tile rows [row_begin, row_end) are written.  exact (n, 8) or
 * NULL: the preprocess's exact blend-decision records (TGS_EXACT_FLOATS); every
 * blend entry point takes the same records and decides identically.
 * exceptions / exc_overflow (tile_size 16 with exact records; both NULL or both
 * set): the forward's blend exceptions, handed to tgs_blend_backward so it
 * decides the rare bracket pairs without float64 — exceptions (H, W) int32
 * (the 1-based list position a pixel's float64 resolution blended, 0 = none),
 * exc_overflow TGS_EXC_OVERFLOW_WORDS(ntiles) uint32 (zeroed here: [count, flag per
 * tile] of the tiles whose pixels need more, which the backward re-resolves in float64),
 * ntiles = tiles in rows [row_begin, row_end). */
#define TGS_EXC_OVERFLOW_WORDS(ntiles) (1 + (size_t)(ntiles))
TGS_API int tgs_blend_forward(const float *splats, const float *exact, const int32_t *tile_offsets,
                      const int32_t *sorted_ids,
                      const tgs_camera *cam, const tgs_settings *s, int32_t row_begin, int32_t row_end,
                      float *image, float *transmit, float *weight_sum, int32_t *n_contrib,
                      int32_t *last_pos, int32_t *hits, int32_t *exceptions, uint32_t *exc_overflow,
                      const int32_t *tile_order, tgs_stream_t stream);

/* Per-pixel ordered (Gaussian, blend weight) records — the reference's
 * records_kernel (_kernels.py:184-241), a test/debug payload.  pixel_offsets
 * (H*W,) int64 is the exclusive cumsum of n_contrib; rec_gauss (int32) and
 * rec_weight (float32) have sum(n_contrib) entries.  Full image only. */
TGS_API int tgs_blend_records(const float *splats, const float *exact, const int32_t *tile_offsets,
                      const int32_t *sorted_ids,
                      const tgs_camera *cam, const tgs_settings *s, const int64_t *pixel_offsets,
                      int32_t *rec_gauss, float *rec_weight, tgs_stream_t stream);

/* ---- (4) backward blend -----------------------------------------------------
 * dsplats (n, 9) is ACCUMULATED into (caller zeroes it). dimage (H, W, 3).
 * exceptions / exc_overflow: the forward's (same rows and records), or NULL. */
TGS_API int tgs_blend_backward(const float *splats, const float *exact, const int32_t *tile_offsets,
                      const int32_t *sorted_ids,
                       const tgs_camera *cam, const tgs_settings *s, int32_t row_begin, int32_t row_end,
                       const float *transmit, const int32_t *last_pos, const int32_t *exceptions,
                       const uint32_t *exc_overflow, const float *dimage,
                       float *dsplats, const int32_t *tile_order, tgs_stream_t stream);

/* Heaviest-first tile order for the blend launches (tile_order above, may be
 * NULL = row-major): tiles sorted by floor(log2(list length)) descending, so the
 * longest tiles start first and the tail of the launch is short tiles.
 * `order` holds ntiles + 64 int32 (the last 64 are scratch).  Scheduling only:
 * the blend results do not depend on it (tile_size 16 kernels use it). */
TGS_API int tgs_tile_order(const int32_t *tile_offsets, int32_t ntiles, int32_t *order, tgs_stream_t stream);

/* Deterministic variant (a deterministic-reduction mode): the
 * partials of every (tile, Gaussian) pair are summed over the tile's warps in a
 * fixed order and stored per list position; each Gaussian then sums its own
 * instances in rect order (row-major over its band-clipped tile rect) with one
 * thread, so dsplats (+=) is bitwise reproducible run to run.  Needs the
 * forward's tiles_touched (n), the instance count and a workspace of
 * tgs_blend_backward_deterministic_workspace() bytes (≈ 40 B per instance). */
TGS_API int tgs_blend_backward_deterministic_workspace(int64_t n, int64_t num_instances, size_t *bytes);
TGS_API int tgs_blend_backward_deterministic(const float *splats, const float *exact,
                                             const int32_t *tiles_touched, int64_t n,
                                             const int32_t *tile_offsets, const int32_t *sorted_ids,
                                             int64_t num_instances, const tgs_camera *cam, const tgs_settings *s,
                                             int32_t row_begin, int32_t row_end, const float *transmit,
                                             const int32_t *last_pos, const float *dimage, float *dsplats,
                                             void *workspace, tgs_stream_t stream);

/* ---- (5) preprocess backward ------------------------------------------------
 * accumulate != 0 adds into grads (multi-view batches), else overwrites. */
TGS_API int tgs_preprocess_backward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                            const uint8_t *visible, const float *dsplats, tgs_grads *grads,
                            int32_t accumulate, tgs_stream_t stream);

/* Multi-view form: sums the gradients of `nviews` views (cams[v], visible[v],
 * dsplats[v]; host arrays of device pointers) in one pass over the parameters —
 * the chains after the screen-space partials are linear, so view-independent
 * work (covariance/quaternion/scale/opacity/mask) runs once per Gaussian.
 * stats (may be NULL): grad_accum / grad_count take every view's screen-space
 * mean gradient norm (the densification statistics of each view's step).
 * clear_partials != 0: every dsplats[v] (then writable, 16 B aligned) is zeroed
 * after it has been read, so a training loop's next blend backward accumulates
 * into it without a separate fill. */
TGS_API int tgs_preprocess_backward_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                          const uint8_t *const *visible, const float *const *dsplats,
                                          int32_t nviews, tgs_grads *grads, int32_t accumulate,
                                          const tgs_densify_stats *stats, int32_t clear_partials,
                                          tgs_stream_t stream);

/* ---- (6) loss: (1-lambda)*L1 + lambda*(1-SSIM)/2, 11x11 sigma 1.5 window,
 * symmetric padding (training.py:76-89, metrics.py:138-188).  image/target
 * (H, W, 3); dimage (H, W, 3) written; terms (device float64[2]) receives
 * {mean |image-target|, mean SSIM}.  Workspace: tgs_loss_workspace() bytes. */
TGS_API int tgs_loss_workspace(int32_t width, int32_t height, size_t *bytes);
TGS_API int tgs_loss_l1_ssim(const float *image, const float *target, int32_t width, int32_t height,
                     float lambda_ssim, float *dimage, double *terms, void *workspace,
                     tgs_stream_t stream);

/* ---- (7) Adam (optim.py:37-49) over one parameter group of n floats.
 * bias corrections are passed in (1 - beta^step) so the step counter stays host-side. */
TGS_API int tgs_adam_step(float *param, const float *grad, float *m, float *v, int64_t n, float lr,
                  float beta1, float beta2, float eps, float bias_c1, float bias_c2,
                  tgs_stream_t stream);
/* All groups in one launch (optim.py:37-49 per group): groups are contiguous,
 * 64-float aligned ranges [offsets[k], offsets[k] + sizes[k]) of the flat
 * param/grad/moment buffers (16 B aligned), each with its own lr and bias
 * corrections.  kinds[k] = 1 adds the Gaussian-mask penalty gradient
 * lambda_m * sigmoid'(m) / n, kinds[k] = 2 the SH-band-mask penalty
 * lambda_sh * sigmoid'(m_l) * band_weights[l] / n (masking.py:60-67), to that
 * group's gradient before the update (written back to grad).
 * Divergence guard (training.py:298-308): with n_terms > 0, if any of the
 * n_terms doubles at loss_terms (device) is not finite, NOTHING is updated and
 * *nonfinite_flag (device int32, may be NULL) is written 1 (else 0); the host
 * raises DivergenceError from it.  nranges > 0 (<= 8): only the floats in the
 * ranges [range_begin[r], range_end[r]) (multiples of 4) are updated — a rank's
 * shard under ZeRO-1 data parallelism, the rows of one preprocess-backward
 * chunk; nranges = 0: all. */
TGS_API int tgs_adam_step_groups(float *param, float *grad, float *m, float *v, int32_t ngroups,
                                 const int64_t *offsets, const int64_t *sizes, const float *lrs,
                                 const float *bias_c1, const float *bias_c2, const int32_t *kinds, float beta1,
                                 float beta2, float eps, float lambda_m, float lambda_sh,
                                 const float *band_weights, int64_t n_gaussians, const double *loss_terms,
                                 int32_t n_terms, int32_t *nonfinite_flag, const int64_t *range_begin,
                                 const int64_t *range_end, int32_t nranges, tgs_stream_t stream);

/* ---- target-side progressive ops (images.py:58-102), (H, W, 3) float32.
 * area_resize: exact fractional box filter (downsampling only); workspace
 * out_h * in_w * 3 floats.  gaussian_blur: odd size <= 31, reflect edges;
 * workspace h * w * 3 floats. */
TGS_API int tgs_area_resize(const float *in, int32_t in_h, int32_t in_w, float *out, int32_t out_h, int32_t out_w,
                            float *workspace, tgs_stream_t stream);
TGS_API int tgs_gaussian_blur(const float *in, int32_t h, int32_t w, int32_t size, float sigma, float *out,
                              float *workspace, tgs_stream_t stream);

/* ---- (8) row compaction (cloud.take / Adam.compact): out[k] = in[keep[k]] for
 * rows of `row_floats` floats. */
TGS_API int tgs_gather_rows(const float *in, float *out, const int64_t *keep, int64_t n_keep,
                    int32_t row_floats, tgs_stream_t stream);

/* Row selection for the compactions (np.nonzero of masking.prune_by_mask,
 * masking.py:70-81, and of significance.prune_by_significance, significance.py:
 * 81-99): writes the rows i with flags[i] != 0 — or, with flags == NULL, with
 * x[i] > threshold — in ascending order to indices (capacity n) and their number
 * to *count (device int64).  n < 2^30.  Workspace: tgs_select_rows_workspace. */
TGS_API int tgs_select_rows_workspace(int64_t n, size_t *bytes);
TGS_API int tgs_select_rows(const uint8_t *flags, const float *x, float threshold, int64_t n, int64_t *indices,
                            int64_t *count, void *workspace, size_t workspace_bytes, tgs_stream_t stream);

/* Significance (significance.py:45-99).  Workspace: one u64 key per row + a
 * small selection state.  tgs_significance_scores writes, for every row,
 *   volumes = 4/3 pi prod(e^log_scales * M), M = mask_logit > mask_logit_min,
 *   v_norm  = min(volumes / V90, 1) ** volume_power   (V90 > 0; else volumes > 0),
 *   scores  = hits * sigmoid(opacity_logit) * M * v_norm,
 * V90 = the rank90-th smallest volume (0-based; the caller passes the reference's
 * nearest rank max(ceil(0.9 n) - 1, 0), significance.py:65).
 * tgs_significance_keep sets keep[i] = 1 for every row except the k lowest by
 * (score, row) — np.lexsort((arange(n), scores))[:k] (significance.py:97-98);
 * 0 <= k < n.  Both run without host synchronisation; n < 2^32. */
TGS_API int tgs_significance_workspace(int64_t n, size_t *bytes);
TGS_API int tgs_significance_scores(const tgs_cloud *cloud, const int64_t *hits, float mask_logit_min,
                                    float volume_power, int64_t rank90, float *volumes, float *v_norm,
                                    float *scores, void *workspace, size_t workspace_bytes, tgs_stream_t stream);
TGS_API int tgs_significance_keep(const float *scores, int64_t n, int64_t k, uint8_t *keep, void *workspace,
                                  size_t workspace_bytes, tgs_stream_t stream);

/* ---- native render pipeline for a batch of views (rasterizer.render_views) ----
 * The per-view sequence of render_forward — one multi-view preprocess, then per view
 * tgs_bin_gaussians -> count read-back -> tgs_bin_instances -> tgs_blend_forward —
 * issued from C++ over `nstreams` caller streams (view v on streams[v % nstreams]),
 * with the next nstreams-1 views' depth sorts queued before a view's count is
 * awaited.  blend_streams (may be NULL = the same streams): view v's blend runs on
 * blend_streams[v % nstreams] after its binning (event), e.g. a lower priority than
 * the binning streams.  Outputs are the caller's (preprocess buffers as for
 * tgs_preprocess_forward_views, per-view targets below); workspaces[k] holds
 * workspace_bytes >= tgs_render_views_workspace(n, max instances of a view, ...)
 * for stream k; pinned_counts is 2 * nstreams pinned host int64.  Views whose count
 * exceeds ids_capacity or the workspace stop the batch with TGS_ERR_CAPACITY after
 * every view's count is reported in num_instances (the caller grows and retries). */
typedef struct {
  int32_t *tile_offsets;     /* (tiles + 1,) */
  int32_t *sorted_ids;       /* (ids_capacity,) */
  int64_t ids_capacity;
  const int32_t *tile_order; /* blend launch order (may be NULL) */
  float *image, *transmit, *weight_sum;
  int32_t *n_contrib, *last_pos, *hits; /* hits may be NULL (zeroed by the caller otherwise) */
  int64_t num_instances;     /* out */
  /* tile rows [row_begin, row_end) of the view (tile-row sharding: only these rows are
   * binned and blended, tile_offsets then has (row_end - row_begin) * tiles_x + 1
   * entries); row_end <= 0 = the whole view */
  int32_t row_begin, row_end;
} tgs_view_target;

/* Per-view training payload of tgs_train_views: after the view's blend, on the same
 * stream, the L1 + D-SSIM loss against `target` (dL/dimage into `dimage`, the mean L1 /
 * mean SSIM into terms[0..1]; `loss_workspace` of tgs_loss_workspace bytes — views on
 * one stream may share dimage and workspace) and the blend backward into `dsplats`
 * (n, 9), accumulated.  target_ready (a cudaEvent_t, may be NULL): waited on before the
 * loss (a host-to-device copy of the target on another stream).  exceptions /
 * exc_overflow (may be NULL; views on one stream may share them): the blend exception
 * buffers tgs_blend_forward hands its backward (with exact records). */
typedef struct {
  const float *target;
  float *dimage;
  double *terms;
  float *dsplats;
  void *loss_workspace;
  void *target_ready;
  int32_t *exceptions;
  uint32_t *exc_overflow;
} tgs_view_train;

TGS_API int tgs_render_views_workspace(int64_t n, int64_t max_instances, int32_t width, int32_t height,
                                       int32_t tile_size, size_t *bytes);
TGS_API int tgs_render_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s, int32_t nviews,
                             float *const *splats, uint8_t *const *visible, int32_t *const *tiles_touched,
                             uint64_t *const *depth_keys, float *const *exact, int32_t *error_flag,
                             tgs_view_target *targets,
                             void *const *workspaces, size_t workspace_bytes, int64_t *pinned_counts,
                             const tgs_stream_t *streams, const tgs_stream_t *blend_streams, int32_t nstreams);

/* The per-view half of a training step (train.Trainer; training.py:296-309 per view)
 * from C++: the caller has run tgs_preprocess_forward_views (and, on any stream,
 * tgs_exact_records_views, complete at the event `exact_ready`, which may be NULL when
 * exact is NULL or already complete); per view bin -> count -> place -> blend forward ->
 * loss -> blend backward as tgs_render_views pipelines it, with train[v] the view's
 * loss / backward buffers; blend_streams (may be NULL) take each view's blend, loss and
 * backward (after an event on its binning stream), as in tgs_render_views.  The caller then runs ONE
 * tgs_preprocess_backward_views over the views' dsplats and the Adam step.  On
 * TGS_ERR_CAPACITY some views may already have accumulated partials: zero them before
 * the retry. */
TGS_API int tgs_train_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s, int32_t nviews,
                            float *const *splats, uint8_t *const *visible, int32_t *const *tiles_touched,
                            uint64_t *const *depth_keys, float *const *exact, void *exact_ready,
                            int32_t *error_flag, tgs_view_target *targets, const tgs_view_train *train,
                            float lambda_ssim, void *const *workspaces, size_t workspace_bytes,
                            int64_t *pinned_counts, const tgs_stream_t *streams,
                            const tgs_stream_t *blend_streams, int32_t nstreams);

#ifdef __cplusplus
}
#endif
#endif /* TGS_H_ */
