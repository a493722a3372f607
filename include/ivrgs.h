/*
 * ivrgs.h -- C ABI of the B200 editable-Gaussian splatting hot path
 * (drop-in for the reference's numba kernels + the vectorized numpy stages
 * around them; reference = voxsplat, /root/reference/pkg/src/voxsplat/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc'd or from the PyTorch
 *    caching allocator), row-major, float64 unless stated otherwise.
 *  - Every launch is stream-ordered on `stream` (a cudaStream_t); no entry
 *    point allocates, synchronizes or keeps global mutable state, so calls are
 *    reentrant and CUDA-graph capturable.  Scratch memory comes from the
 *    caller through a size query (ivr_*_workspace_size) + workspace pointer.
 *  - Data-dependent sizes (pair count P) live in device memory; the caller
 *    provides a capacity and reads back the true count to detect overflow.
 *  - Return value: IVR_OK (0) or a negative ivr_status.  ivr_last_error()
 *    returns a thread-local message for the last failure.
 */
#ifndef IVRGS_H
#define IVRGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *ivr_stream_t; /* == cudaStream_t */

#define IVR_ABI_VERSION 4
#define IVR_TILE 16 /* rasterizer.py:24 TILE_SIZE */

typedef enum ivr_status {
    IVR_OK = 0,
    IVR_ERR_ARG = -1,           /* bad argument / null pointer / size */
    IVR_ERR_SHAPE = -2,         /* errors.ShapeMismatch */
    IVR_ERR_NONFINITE = -3,     /* errors.NonFiniteGradient (index in out-param) */
    IVR_ERR_CORRUPT_INDEX = -4, /* errors.CorruptIndex */
    IVR_ERR_CUDA = -5,          /* launch / runtime failure */
    IVR_ERR_CAPACITY = -6       /* pair buffer too small (count reported) */
} ivr_status;

/* Pinhole camera, gaussians.py:139-164 (Camera).  focal/cx/cy are evaluated
 * on the host exactly as Camera.focal / Camera.center_px. */
typedef struct ivr_camera {
    double position[3];
    double rotation[9]; /* world->camera, row-major */
    double focal, cx, cy;
    int32_t width, height;
} ivr_camera;

/* GaussianGeometry storage, gaussians.py:29-51 (unconstrained domain). */
typedef struct ivr_gaussians {
    int64_t n;
    const double *mu;      /* (n,3) */
    const double *q_raw;   /* (n,4) w-first */
    const double *log_s;   /* (n,3) */
    const double *o_logit; /* (n)   */
    const double *n_raw;   /* (n,3) */
    const double *cache;   /* optional (n,16) from ivr_preprocess_static, or NULL */
} ivr_gaussians;


/* Editable shading inputs: ShadingAttributes (shading.py:89-115), palette,
 * LightConfig (shading.py:42-66) and the optional (lam, b) coefficient
 * transform of shade_gaussians (shading.py:225-279). */
typedef struct ivr_shading {
    const double *delta_c;  /* (n,3) */
    const double *k_a_raw;  /* (n) */
    const double *k_d_raw;  /* (n) */
    const double *k_s_raw;  /* (n) */
    const double *log_beta; /* (n) */
    const double *palette;  /* (S,3) indexed by scene id, or (n,3) */
    int32_t per_splat_palette;
    int32_t orbital;        /* 0 = headlight, 1 = orbital */
    double light_dir[3];    /* light_direction_from_angles (host) */
    double term_scales[4];
    double lam[4];
    double b[4];
} ivr_shading;

/* Composed-scene edits, scene.py:199-228 (apply_edits). */
typedef struct ivr_edits {
    const int32_t *scene_id;      /* (n) or NULL (all scene 0) */
    const double *opacity_scale;  /* (S) or NULL */
    int32_t rescale_opacity;      /* 1 iff any scale != 1 (scene.py:217) */
} ivr_edits;

#define IVR_MAX_ATTRS 8
/* Packed channel layout, rasterizer.py:39-50 + 134-149. */
typedef struct ivr_layout {
    int32_t k; /* total channels K */
    int32_t col_color, col_alpha, col_depth, col_normal; /* -1 = absent */
    const double *colors; /* (n,3) per-splat colors when shading == NULL */
    int32_t n_attr;
    const double *attr[IVR_MAX_ATTRS];
    int32_t attr_col[IVR_MAX_ATTRS];
    int32_t attr_width[IVR_MAX_ATTRS];
} ivr_layout;

/* Per-frame preprocess outputs (device, caller-allocated). */
typedef struct ivr_proj_out {
    uint64_t *depth_key; /* (n) float64 depth bits if visible else ~0 */
    int32_t *count;      /* (n) tiles touched (0 if invisible) */
    uint16_t *rect;      /* (n,4) tx0, tx1, ty0, ty1 */
    float *rec;          /* (n,8) blend record: mx,my,o,hi, a/2,b,c/2,thr */
    float *values;       /* (n,k) packed channel values (float32) */
    double *rec64;       /* optional (n,8): mx,my,a,b,c,o,depth,0 (float64 mode) */
    double *values64;    /* optional (n,k) float64 channel values */
    /* optional float64 parity outputs (NULL to skip) */
    double *mean2d;  /* (n,2) */
    double *conic;   /* (n,3) */
    double *cov2d;   /* (n,4) */
    double *depth;   /* (n) */
    double *opacity; /* (n) effective opacity */
    double *rgb;     /* (n,3) shaded colour */
    double *radius;  /* (n) */
    uint8_t *valid;  /* (n) projection validity */
    /* optional [min, max] of the visible depth keys, reduced with atomics
     * (must hold {~0, 0} or a superset; ivr_bin_sort_frame consumes and
     * re-arms it) */
    unsigned long long *depth_minmax;
} ivr_proj_out;

/* Camera- and edit-independent per-Gaussian values of a resident scene
 * (cov3d, unit normal, sigmoid(o_logit), the shading sigmoids and beta),
 * computed by the same code as the per-frame path: with g->cache set,
 * ivr_preprocess_fwd(_params) and ivr_shade_fwd give bit-identical results
 * with far less float64 work per frame.  cache: (n,16) float64. */
int ivr_preprocess_static(const ivr_gaussians *g, const ivr_shading *shading, double *cache,
                          ivr_stream_t stream);

int ivr_version(void);
const char *ivr_last_error(void);

/* K1: fused edits + EWA projection + Blinn-Phong shading + radius / tile rect
 * / count + float32 record packing.  Replaces scene.apply_edits
 * (scene.py:199-228), shading.shade_gaussians (shading.py:225-329),
 * gaussians.project_gaussians (gaussians.py:296-346) and the binning prologue
 * of rasterizer.rasterize_forward (rasterizer.py:88-121, 134-153).
 * shading / edits may be NULL.  f64_mode is a bit set: IVR_PRE_F64 selects
 * dtype=float64 semantics; IVR_PRE_EXACT_RGB keeps the float64 shading chain
 * (the reference's rgb, rounded once to float32) when a static cache would
 * otherwise select the float32 colour path of FAST frames. */
#define IVR_PRE_F64 1
#define IVR_PRE_EXACT_RGB 2
int ivr_preprocess_fwd(const ivr_gaussians *g, const ivr_shading *shading,
                       const ivr_edits *edits, const ivr_camera *cam,
                       const ivr_layout *layout, ivr_proj_out *out,
                       int32_t f64_mode, ivr_stream_t stream);

/* Per-frame view/light/edit state that may live in DEVICE memory, so that a
 * captured CUDA graph of a whole frame can be replayed with new cameras and
 * edits (the host refreshes this struct with one small H2D copy). */
typedef struct ivr_frame_params {
    ivr_camera cam;
    double light_dir[3];
    double term_scales[4];
    double lam[4];
    double b[4];
    int32_t orbital;
    int32_t rescale_opacity;
    /* d light_dir / d polar, d azimuth (orbital): used by ivr_preprocess_bwd
     * when the params come from device memory (ivr_grads.dl_* otherwise) */
    double dl_dp[3], dl_da[3];
} ivr_frame_params;

/* ivr_preprocess_fwd with the camera, light, coefficient transform and the
 * opacity-rescale flag read from `params` (a DEVICE pointer) instead of the
 * host structs; shading/edits still supply the array pointers.  width/height
 * must equal params->cam.width/height (they size the tile grid). */
int ivr_preprocess_fwd_params(const ivr_gaussians *g, const ivr_shading *shading,
                              const ivr_edits *edits, const ivr_frame_params *params,
                              int32_t width, int32_t height, const ivr_layout *layout,
                              ivr_proj_out *out, int32_t f64_mode, ivr_stream_t stream);

/* Shading only (shading.shade_gaussians, shading.py:225-329): float64 rgb
 * (n,3) and optional terms (n,9: ambient, diffuse, specular). */
int ivr_shade_fwd(const ivr_gaussians *g, const ivr_shading *shading,
                  const int32_t *scene_id, const ivr_camera *cam, double *rgb,
                  double *terms, ivr_stream_t stream);

/* K2: stable depth sort + duplicated (tile, depth) pair emission + stable
 * tile sort + tile ranges.  Replaces _kernels.fill_pairs (_kernels.py:19-28),
 * np.lexsort((depth[pair_splat], pair_tile)) (rasterizer.py:129) and
 * np.searchsorted tile ranges (rasterizer.py:132), bit-exactly.
 * Writes n_pairs[0] (device) = P; if P > pair_capacity nothing past the
 * capacity is written, tile_ranges are clamped to the capacity (so K3/K4 stay
 * in bounds) and the caller must retry with a larger buffer. */
size_t ivr_bin_sort_workspace_size(int64_t n, int64_t pair_capacity, int32_t ntiles);
int ivr_bin_sort(int64_t n, const uint64_t *depth_key, const int32_t *count,
                 const uint16_t *rect, int32_t ntx, int32_t nty,
                 int64_t pair_capacity, void *workspace, size_t workspace_bytes,
                 int32_t *pair_splat, int32_t *tile_ranges, int32_t *n_pairs,
                 ivr_stream_t stream);

/* K2 with the per-pair tile cull: pairs whose splat provably stays below
 * alpha 1/255 over their whole tile (float64 minimum of the exponent over the
 * tile rectangle vs the record's bound) get bit 31 set in pair_splat;
 * (pair_splat & 0x7fffffff) is still the reference list.  rec is K1's float32
 * record; width/height the frame size.  Any frame size: a tile grid too
 * large for the shared-memory placement tables is placed in bands of tile
 * rows (same lists). */
int ivr_bin_sort_cull(int64_t n, const uint64_t *depth_key, const int32_t *count,
                      const uint16_t *rect, const float *rec, int32_t ntx, int32_t nty,
                      int32_t width, int32_t height, int64_t pair_capacity,
                      void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                      int32_t *tile_ranges, int32_t *n_pairs, ivr_stream_t stream);

/* K2 for a K1 frame: as ivr_bin_sort_cull (rec may be NULL), plus
 * depth_minmax (nullable): the [min, max] of the visible depth keys that
 * ivr_proj_out.depth_minmax made K1 reduce (block-reduced atomics); K2
 * re-arms it to {~0, 0} for the next frame, so it must start as {~0, 0} or
 * as any superset of the keys' range (a wider range only costs sort runs,
 * never correctness).  NULL: K2 reduces the range itself (two more kernels).
 * tile_order (nullable): receives the heaviest-first tile schedule for K3/K4
 * (ivr_tile_order's) from K2's tile-range kernel.  8 kernels + one memset of
 * K2's control block per call at 1M splats. */
int ivr_bin_sort_frame(int64_t n, const uint64_t *depth_key, unsigned long long *depth_minmax,
                       const int32_t *count, const uint16_t *rect, const float *rec, int32_t ntx,
                       int32_t nty, int32_t width, int32_t height, int64_t pair_capacity,
                       void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                       int32_t *tile_ranges, int32_t *n_pairs, int32_t *tile_order,
                       ivr_stream_t stream);

/* K3: per-tile front-to-back blend.  Replaces _kernels.composite_forward
 * (_kernels.py:31-72).  out (H,W,k) float32 (out64 float64 in f64 mode),
 * contrib/last_pos int32 (H,W), t_final (H,W) float64 (last_pos / t_final /
 * contrib may be NULL).  tile_order may be NULL (identity) or a permutation
 * of the tiles (scheduling only).  flags & IVR_BLEND_EXACT: bit-faithful
 * float64 evaluation of every candidate pair; otherwise float32 with
 * certified decisions (same contributors, values within ~1e-6). */
#define IVR_BLEND_EXACT 1     /* flags: every non-skipped pair in reference float64 */
#define IVR_BLEND_PRECULLED 2 /* flags: pair_splat carries ivr_bin_sort_cull's bit 31 */
#define IVR_BLEND_NO_GEOMETRY 4 /* ivr_blend_bwd flags: only g_values / g_opacity (transform
                                 * fits); g_mean2d / g_conic may be NULL */
#define IVR_BLEND_DOUT_F64 8 /* ivr_blend_bwd* flags: d_out points to (H,W,k) float64 (the
                              * photometric gradient as ivr_photometric_loss writes it) */
int ivr_blend_fwd(const int32_t *tile_ranges, const int32_t *pair_splat,
                  int32_t ntx, int32_t nty, const float *rec, const float *values,
                  const double *rec64, const double *values64, int32_t k,
                  int32_t width, int32_t height, float *out, double *out64,
                  int32_t *contrib, int32_t *last_pos, double *t_final,
                  const int32_t *tile_order, int32_t flags, ivr_stream_t stream);

/* Debug only (not for concurrent use): record {tile, smid, t_start, t_end}
 * (ns) per (tile, 8x4 block) of later ivr_blend_fwd calls into buf
 * (ntiles * 8 * 4 int64 device memory); NULL stops recording. */
void ivr_debug_blend_trace(long long *buf);

/* Test only: maximal relative errors of ex2.approx.ftz.f32 over [-126, 0]
 * (every multiple of 2^-16) and rcp.approx.ftz.f32 over every float in
 * [1/128, 1], against float64 -- the instruction bounds FAST mode's certified
 * decisions assume.  out: 2 doubles of device memory, zeroed by the caller. */
int ivr_debug_mufu_error(double *out, ivr_stream_t stream);

/* Test only: maximal |sigma32 - sigma_ref| / (|a/2 dx^2| + |b dx dy| +
 * |c/2 dy^2|) of K3's float32 exponent vs float64 on the same float32 record,
 * over n seeded random (record, pixel) samples -- the ratio kSigmaErr (4e-7)
 * bounds.  out: 1 double of device memory, zeroed by the caller. */
int ivr_debug_sigma_error(int64_t n, uint32_t seed, double *out, ivr_stream_t stream);

/* Heaviest-first tile launch order for ivr_blend_fwd (counting sort on
 * half-octave buckets of the per-tile pair count, descending).  Scheduling
 * only: any permutation yields identical images. */
int ivr_tile_order(const int32_t *tile_ranges, int32_t ntiles, int32_t *order,
                   ivr_stream_t stream);

/* K4a: blend backward.  Replaces _kernels.composite_backward
 * (_kernels.py:75-135) and the np.add.at per-Gaussian reductions
 * (rasterizer.py:240-243).  Walks each pixel's contributors back to front
 * from last_pos, recovering the transmittance from t_final by division and
 * accumulating the colour behind each contributor as the reference does,
 * with the same certified decisions as K3, and accumulates with warp-reduced
 * float32 atomics into caller-zeroed per-Gaussian buffers:
 * g_values (n,k), g_mean2d (n,2), g_conic (n,3), g_opacity (n).
 * last_pos / t_final = K3's per-pixel state (H,W) int32 / float64; d_out
 * (H,W,k) float32 upstream gradient.
 * rec64 selects dtype=float64 decisions.  tile_order (nullable): CTA -> tile
 * schedule (ivr_tile_order, heaviest first).  flags: IVR_BLEND_PRECULLED,
 * IVR_BLEND_NO_GEOMETRY. */
int ivr_blend_bwd(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                  int32_t nty, const float *rec, const float *values, const double *rec64,
                  int32_t k, int32_t width, int32_t height, const double *t_final,
                  const int32_t *last_pos, const float *d_out, float *g_values,
                  float *g_mean2d, float *g_conic, float *g_opacity,
                  const int32_t *tile_order, int32_t flags, ivr_stream_t stream);

/* K4a, deterministic (debugging): identical results on every
 * run.  Each (pair, warp) partial is stored, not atomically added, into
 * `workspace` (ivr_blend_bwd_det_workspace_size bytes), then one thread per
 * Gaussian sums them in the reference's pair order (its tile rectangle
 * row-major; each entry found by binary search on K1's depth key and splat
 * index) and warp order, in float64.  n, depth_key, count, rect: K1's outputs
 * for the frame; g_* are overwritten (no zeroing needed). */
size_t ivr_blend_bwd_det_workspace_size(int64_t pair_capacity, int32_t k);
int ivr_blend_bwd_deterministic(const int32_t *tile_ranges, const int32_t *pair_splat,
                                int32_t ntx, int32_t nty, const float *rec, const float *values,
                                const double *rec64, int32_t k, int32_t width, int32_t height,
                                const double *t_final, const int32_t *last_pos, const float *d_out,
                                int64_t n, const uint64_t *depth_key, const int32_t *count,
                                const uint16_t *rect, int64_t pair_capacity, void *workspace,
                                size_t workspace_bytes, float *g_values, float *g_mean2d,
                                float *g_conic, float *g_opacity, const int32_t *tile_order,
                                int32_t flags, ivr_stream_t stream);

/* K4a per list entry (the reference's composite_backward outputs,
 * _kernels.py:75-135): pair_grads (n_pairs, k+6) float32 = [d values (k),
 * d mean2d (2), d conic (3: a/2-, b-, c/2-weighted as the reference), d
 * opacity] per pair_splat entry, each the fixed-order sum of the walk's
 * warp partials.  workspace: ivr_blend_bwd_det_workspace_size(n_pairs, k). */
int ivr_blend_bwd_pairs(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                        int32_t nty, const float *rec, const float *values, const double *rec64,
                        int32_t k, int32_t width, int32_t height, const double *t_final,
                        const int32_t *last_pos, const float *d_out, int64_t n_pairs,
                        void *workspace, size_t workspace_bytes, float *pair_grads,
                        ivr_stream_t stream);

/* Per-Gaussian backward outputs (float64, NULL = not wanted). */
typedef struct ivr_grads {
    /* inputs: K4a accumulators (float32, NULL if none) and an optional extra
     * upstream gradient on the shaded rgb (n,3) (shade_backward API) */
    const float *g_values, *g_mean2d, *g_conic, *g_opacity;
    const double *d_rgb_extra;
    /* rasterize_backward outputs (rasterizer.py:273-286) */
    double *d_mu, *d_q_raw, *d_log_s, *d_o_logit, *d_n_raw, *d_colors, *d_mean2d;
    double *d_values; /* (n,k) raw per-channel gradients (attribute columns) */
    /* shade_backward outputs (shading.py:426-439) */
    double *d_delta_c, *d_k_a_raw, *d_k_d_raw, *d_k_s_raw, *d_log_beta;
    double *d_c_p;     /* (n,3) per splat, or (S,3) summed per scene if per_scene */
    double *d_scale;   /* (S) opacity-scale chain of inverse._step (inverse.py:174-180) */
    double *d_globals; /* [10] d_lam[4], d_b[4], d_polar, d_azimuth (summed) */
    int32_t per_scene;
    double dl_dp[3], dl_da[3]; /* orbital light direction derivatives (host-params path) */
    /* [16] first non-finite row per output (init ~0): 0 d_mu, 1 d_q_raw,
     * 2 d_log_s, 3 d_o_logit, 4 d_n_raw, 5 d_colors, 6 d_k_a_raw, 7 d_k_d_raw,
     * 8 d_k_s_raw, 9 d_log_beta, 10 d_delta_c / d_c_p */
    unsigned long long *bad;
    /* optional (NULL = global atomics): ivr_preprocess_bwd_scratch_len(n,
     * per_scene) doubles for per-block partials of d_globals / d_c_p /
     * d_scale, summed across blocks in a fixed order and added to the outputs
     * (used by the deterministic mode) */
    double *scratch;
    int64_t scratch_len;
} ivr_grads;
int64_t ivr_preprocess_bwd_scratch_len(int64_t n, int32_t per_scene);

/* K4b: per-Gaussian backward in float64: conic -> cov2d chain
 * (rasterizer.py:245-255), channel unpack (rasterizer.py:257-270),
 * gaussians.project_backward (gaussians.py:349-400, when geometry != 0),
 * opacity-logit chain (rasterizer.py:278-279) and, when shading != NULL,
 * shading.shade_backward (shading.py:332-445) plus the composed-scene /
 * inverse reductions (inverse.py:170-181).  Camera/light from `params`
 * (device pointer) if non-NULL else from cam + shading. */
int ivr_preprocess_bwd(const ivr_gaussians *g, const ivr_shading *shading,
                       const ivr_edits *edits, const ivr_frame_params *params,
                       const ivr_camera *cam, const ivr_layout *layout, ivr_grads *grads,
                       int32_t geometry, ivr_stream_t stream);

/* K5: VQ assignment, vq.assign_nearest (vq.py:90-96): index of the nearest
 * sorted centroid = searchsorted(mids, v, 'left'); NaN -> K-1.
 * Output uint16 (K <= 65536). */
size_t ivr_vq_assign_workspace_size(void);
int ivr_vq_assign(const double *values, int64_t n, const double *centroids,
                  int32_t k, uint16_t *indices, void *workspace, size_t workspace_bytes,
                  ivr_stream_t stream);

/* K6: codebook decode, Codebook.decode (vq.py:128-134).  bad[0] (device,
 * caller-initialised to -1) receives the largest index >= k, if any; those
 * positions decode to 0. */
int ivr_vq_decode(const uint16_t *indices, int64_t n, const double *centroids,
                  int32_t k, double *out, int64_t *bad, ivr_stream_t stream);

/* Fused Lloyd iteration, vq._lloyd (vq.py:75-87): assign every value to
 * its nearest sorted centroid (as ivr_vq_assign), per-centroid sums and
 * counts (shared-memory privatised), new = counts > 0 ? sums / counts : old,
 * shift[0] = max |new - old| (device).  2 <= k <= 4097. */
size_t ivr_kmeans_lloyd_workspace_size(int32_t k);
int ivr_kmeans_lloyd_step(const double *values, int64_t n, const double *centroids, int32_t k,
                          double *new_centroids, double *shift, void *workspace,
                          size_t workspace_bytes, ivr_stream_t stream);

/* The same step for `sets` sorted centroid sets (k-means' restarts, row r at
 * centroids[r * k]) on the values in ascending order: bucket b is the
 * contiguous range of sorted values between the midpoints, so its sum is a
 * segment sum (one CTA per bucket and set, no atomics); new = count > 0 ?
 * sum / count : old, shift[r] = max |new - old| of set r (device doubles).
 * k >= 2. */
size_t ivr_kmeans_lloyd_sorted_workspace_size(int32_t k, int32_t sets);
int ivr_kmeans_lloyd_step_sorted(const double *sorted_values, int64_t n, const double *centroids,
                                 int32_t k, int32_t sets, double *new_centroids, double *shift,
                                 void *workspace, size_t workspace_bytes, ivr_stream_t stream);

/* k-means++ seeding, vq._seed_plusplus (vq.py:60-72): centers[0] =
 * values[first] (the reference's rng.integers draw), then for i = 1..k-1 the
 * first index whose cumulative d2 (index order) exceeds u[i-1] * sum(d2)
 * (rng.choice(n, p = d2 / sum d2) with the draws u = rng.random(k-1); all
 * mass on chosen centres repeats centers[0]).  Two kernels per centre, d2
 * and the block sums in the workspace (ivr_kmeans_seed_workspace_size). */
size_t ivr_kmeans_seed_workspace_size(int64_t n);
int ivr_kmeans_seed(const double *values, int64_t n, int32_t k, int64_t first, const double *u,
                    double *centers, void *workspace, size_t workspace_bytes,
                    ivr_stream_t stream);

/* The same seeding (same draws, same picks up to float64 summation order) for
 * `count` (1..64) independent seedings -- k-means' restarts of every
 * attribute -- in one cooperative kernel that only revisits the samples a
 * new centre can change: `order` (int32, n < 2^31) sorts `values` ascending
 * (any order of ties); d2 is lowered only between the chosen centres
 * adjacent to the new one in value order (~n ln k updates in all instead of
 * n k), and the picks walk 32-value block sums and 2048-value super-block
 * sums in index order.  Per seeding: the rng.integers draw `first`, the k - 1
 * rng.random draws `u` (device), `centers` (device, k).  1 <= k <= 32768.
 * k-means' restarts draw from one stream but their draws do not depend on
 * the data, so they are all known up front (vq.kmeans).  `problems` is a host
 * array. */
typedef struct {
    const double *values;  /* n float64 (device) */
    const int32_t *order;  /* ascending order of values (device) */
    int64_t n;
    int64_t first;
    const double *u;  /* k - 1 draws (device) */
    double *centers;  /* k centres out (device) */
} ivr_seed_problem;
size_t ivr_kmeans_seed_sorted_workspace_size(const ivr_seed_problem *problems, int32_t count);
int ivr_kmeans_seed_sorted(const ivr_seed_problem *problems, int32_t count, int32_t k,
                           void *workspace, size_t workspace_bytes, ivr_stream_t stream);

/* Compose on the device (scene.py:147-186, gaussians.py:98-106): concatenate
 * n_src (<= 64) row-major float64 arrays of `width` columns (rows[m] rows
 * each) into dst; scene_id (may be NULL) receives the source index per row. */
int ivr_concat(const double *const *srcs, const int64_t *rows, int32_t n_src, int32_t width,
               double *dst, int32_t *scene_id, ivr_stream_t stream);

/* Stage-1 colour: eval_sh(ShColor, view_dirs(mu, cam_pos))
 * (gaussians.py:497-508, 521-524).  coeffs (n, (degree+1)^2, 3) float64,
 * degree 0..3; rgb (n,3) = max(sum_b basis_b * coeffs_b + 0.5, 0). */
/* gaussians.sh_basis (gaussians.py:429-494) on unit directions (n,3):
 * basis (n,(degree+1)^2) and, when dbasis != NULL, its derivatives
 * (n,(degree+1)^2,3). */
int ivr_sh_basis(int64_t n, int32_t degree, const double *dirs, double *basis, double *dbasis,
                 ivr_stream_t stream);
int ivr_sh_eval(int64_t n, int32_t degree, const double *mu, const double *coeffs,
                const double cam_pos[3], double *rgb, ivr_stream_t stream);

/* eval_sh_backward + view_dirs_backward (gaussians.py:511-518, 527-529):
 * d_coeffs (n, nb, 3) is overwritten; d_mu (n,3), when non-NULL, is
 * incremented by the view-direction gradient (the caller passes the
 * projection gradient there, as _stage1_step sums them, trainer.py:386-388). */
int ivr_sh_bwd(int64_t n, int32_t degree, const double *mu, const double *coeffs,
               const double cam_pos[3], const double *d_rgb, double *d_coeffs, double *d_mu,
               ivr_stream_t stream);

/* IVRG files (scene.py:242-436) resident in HBM.
 * ivr_crc32: zlib CRC-32 of n device bytes into *out (device uint32); the
 * check load_model does with zlib.crc32 on the host (scene.py:359-361). */
int ivr_crc32(const uint8_t *data, int64_t n, uint32_t *out, ivr_stream_t stream);

/* Widen `count` packed little-endian elements at any byte alignment:
 * kind 0 f32 -> double (_Reader.f32, scene.py:343-347), kind 1 u8 -> u16,
 * kind 2 u16 -> u16 (QATT codebook indices, scene.py:388-394). */
int ivr_unpack(const uint8_t *src, int64_t count, int32_t kind, void *dst, ivr_stream_t stream);

/* double -> little-endian f32 bytes (_f32_bytes, scene.py:243-244). */
int ivr_pack_f32(const double *src, int64_t count, uint8_t *dst, ivr_stream_t stream);

/* Ground-truth direct volume rendering (dvr.render_view, dvr.py:197-452):
 * float64 ray march of a (d0,d1,d2) C-order volume centred on the origin
 * with voxel spacing[3] through an n_tf-point piecewise-linear transfer
 * function, Blinn-Phong material {k_a, k_d, k_s, beta}, headlight or
 * light_dir; out (H,W,4) float64 premultiplied RGBA.  One thread per ray. */
int ivr_dvr_render(const double *values, int32_t d0, int32_t d1, int32_t d2,
                   const double spacing[3], const double *tf_values, const double *tf_colors,
                   const double *tf_opacities, int32_t n_tf, const ivr_camera *cam,
                   int32_t headlight, const double light_dir[3], const double material[4],
                   double step_scale, double *out, ivr_stream_t stream);

/* Service frame path (render_modes.py:31-110, service.py:169-187): uint8
 * display image from a float64 render (H,W,k) with columns cols = {color,
 * alpha, depth, normal}.  mode 0: shaded RGBA (colour clipped to [0,1]),
 * 1: alpha (L), 2: unit normal mapped to [0,1] (RGB), 3: depth normalised
 * over covered pixels (L).  to_uint8 = clip(round(255 x)), round half to
 * even.  workspace: 64 device bytes. */
int ivr_display_u8(const double *out, int32_t height, int32_t width, int32_t k,
                   const int32_t cols[4], int32_t mode, uint8_t *dst, void *workspace,
                   ivr_stream_t stream);

/* PNG of a uint8 image (1, 3 or 4 channels) built on the device: filter-0
 * rows in stored deflate blocks, zlib adler32 and chunk CRCs computed in
 * parallel.  out (device) needs ivr_png_size() bytes; workspace 64 bytes. */
int64_t ivr_png_size(int32_t height, int32_t width, int32_t channels);
int ivr_png_encode(const uint8_t *img, int32_t height, int32_t width, int32_t channels,
                   uint8_t *out, int64_t out_cap, void *workspace, ivr_stream_t stream);

/* Photometric objective, losses.ssim + losses.photometric_loss
 * (losses.py:45-138), float64: pred/gt (H,W,C); window = the reference's
 * normalized 11-tap Gaussian (sigma 1.5).  Writes
 *   d_pred = a * sign(pred - gt) + b * d(mean SSIM)/d(pred)   (H,W,C)
 *   sums[0] = sum of SSIM over valid windows and channels (0 if !with_ssim)
 *   sums[1] = sum |pred - gt|
 * (photometric_loss: a = w_l1 / numel, b = -w_ssim).  Scratch from a size
 * query (three partial maps + per-block partials). */
size_t ivr_photometric_workspace_size(int32_t height, int32_t width, int32_t channels);
int ivr_photometric_loss(const double *pred, const double *gt, int32_t height, int32_t width,
                         int32_t channels, const double window[11], double a, double b,
                         int32_t with_ssim, double *d_pred, double *sums, void *workspace,
                         size_t workspace_bytes, ivr_stream_t stream);
/* Same, reading the prediction in place from K3's float32 (H, W, frame_k)
 * frame: channel c = frame[pixel * frame_k + cols[c]] (cols: host array of
 * `channels` <= 4 entries) -- the trainer's rgba columns without a gather /
 * f64 copy (trainer.py:347-352 stacks them out of the render). */
int ivr_photometric_loss_frame(const float *frame, int32_t frame_k, const int32_t *cols,
                               const double *gt, int32_t height, int32_t width,
                               int32_t channels, const double window[11], double a, double b,
                               int32_t with_ssim, double *d_pred, double *sums, void *workspace,
                               size_t workspace_bytes, ivr_stream_t stream);

/* Training-step map terms (trainer.py:355-366, losses.py:141-268) in one
 * pass: d_out (H,W,k float32) = photometric gradient d_rgba (H,W,4 float64,
 * may be NULL) in the colour / alpha channels + w_normal * d(normal
 * consistency vs pseudo-normals from the depth map) + w_offset * d(mean
 * |delta_c|) + w_bil * d(bilateral smoothness of the n_bil maps vs gt
 * (H,W,4)).  cols = {color, alpha, depth, normal, delta_c} (-1 = absent);
 * cam_params (device) = {focal, cx, cy, rotation[9]}.  terms (device, 3):
 * normal loss, mean |delta_c|, bilateral sum over maps. */
size_t ivr_regularize_workspace_size(int32_t height, int32_t width);
int ivr_regularize(const float *out, int32_t k, int32_t height, int32_t width,
                   const int32_t cols[5], const int32_t *bil_cols, int32_t n_bil,
                   const double *gt, const double *d_rgba, const double *cam_params,
                   double w_normal, double w_offset, double w_bil, float *d_out, double *terms,
                   void *workspace, size_t workspace_bytes, ivr_stream_t stream);

/* Adam (trainer.Adam.step, trainer.py:109-120) over up to 16 parameter
 * groups in one launch; float64, the reference's evaluation order.
 * bc1 = 1 - beta1^t, bc2 = 1 - beta2^t (t = the group's step count). */
typedef struct ivr_adam_group {
    double *param, *m, *v;
    const double *grad;
    int64_t n;
    double lr, bc1, bc2;
} ivr_adam_group;
int ivr_adam_step(const ivr_adam_group *groups, int32_t n_groups, double beta1, double beta2,
                  double eps, ivr_stream_t stream);
/* ivr_adam_step for CUDA-graph replay: each group's (lr, bc1, bc2) is read
 * from sched (device, 3 doubles per group, refreshed before every replay)
 * instead of the struct, and a nonzero *skip (device, nullable) makes the
 * step a no-op (a gated step, e.g. one whose pair list overflowed). */
int ivr_adam_step_sched(const ivr_adam_group *groups, int32_t n_groups, double beta1,
                        double beta2, double eps, const double *sched, const int32_t *skip,
                        ivr_stream_t stream);

/* ---- training-step plumbing (csrc/trainstep.cu) ---- */

/* Stage-2 attribute channels (trainer.py:379-404): k_x = sigmoid(k_x_raw)
 * (_mathutil.py:6-13), beta = exp(log_beta) + 1 (shading.py:132-134). */
int ivr_stage2_attrs(int64_t n, const double *k_a_raw, const double *k_d_raw,
                     const double *k_s_raw, const double *log_beta, double *k_a, double *k_d,
                     double *k_s, double *beta, ivr_stream_t stream);

/* Per-Gaussian tail of _stage1_step / _stage2_step (trainer.py:386-394,
 * 410-444).  In place on K4b's outputs: d_delta_c += d_values[:, delta_c],
 * d_k_x_raw += d_values[:, k_x] k_x (1 - k_x), d_log_beta += d_values[:, beta]
 * (beta - 1), d_o_logit += w o (1 - o) / n (losses.py:263-268); stat =
 * |d_mean2d| + |d_n_raw| (trainer.py:443); o_partial[b] = per-block sums of
 * o = sigmoid(o_logit) for the opacity-L1 value (ivr_step_partials(n)
 * blocks).  Any output may be NULL; a column < 0 skips that chain. */
typedef struct ivr_step_grads {
    int64_t n;
    int32_t k;
    const double *d_values; /* (n,k) float64 from ivr_preprocess_bwd */
    int32_t col_delta_c, col_k_a, col_k_d, col_k_s, col_beta;
    const double *o_logit, *k_a_raw, *k_d_raw, *k_s_raw, *log_beta;
    double *d_o_logit, *d_delta_c, *d_k_a_raw, *d_k_d_raw, *d_k_s_raw, *d_log_beta;
    const double *d_mean2d, *d_n_raw;
    double *stat;
    double w_opacity_l1;
    double *o_partial;
    /* captured training steps (nullable): the sticky overflow gate
     * (*gate |= *n_pairs > pair_capacity, read by ivr_adam_step_sched's skip)
     * and the densify statistic accumulated while the step is not gated
     * (stat_sum += stat) */
    int32_t *gate;
    const int32_t *n_pairs;
    int64_t pair_capacity;
    double *stat_sum;
} ivr_step_grads;
int32_t ivr_step_partials(int64_t n);
int ivr_step_assemble(const ivr_step_grads *a, ivr_stream_t stream);

/* The step's scalar loss on the device: l1_weight * sums[1] / numel +
 * ssim_weight * (1 - sums[0] / windows) (photometric, losses.py:118-138)
 * + w_normal terms[0] + w_offset terms[1] + w_bil terms[2] (ivr_regularize)
 * + w_opacity_l1 * sum(o_partial) / n.  state (nullable, int64[2] device):
 * step counter and the first step whose photometric loss was non-finite
 * (-1 = none; *last_bad = that loss), the reference's DivergedLoss check
 * (trainer.py:345-348) without a host synchronisation. */
typedef struct ivr_loss_terms {
    const double *photo_sums; /* [sum SSIM, sum |x - y|] from ivr_photometric_loss */
    double l1_weight, ssim_weight, numel, windows;
    const double *terms;      /* [normal, offset, bilateral] or NULL */
    double w_normal, w_offset, w_bil;
    const double *o_partial;
    int32_t n_partial;
    double w_opacity_l1, n;
} ivr_loss_terms;
int ivr_loss_finalize(const ivr_loss_terms *t, double *loss, int64_t *state, double *last_bad,
                      ivr_stream_t stream);

/* ---- device-side inverse exploration step (csrc/inverse.cu) ----
 * State of optimize_to_reference (inverse.py:205-244) kept in device memory so
 * that complete iterations replay as a CUDA graph.  x = [c_p (3S),
 * opacity_raw (S), lam (4), b (4), polar, azimuth]; m, v its Adam moments;
 * t the per-group step counts (c_p, opacity_raw, lam, b, angles); grad and
 * loss_sum[0..1] (loss, pair-overflow count) accumulate over the views of one
 * iteration (ivr_inverse_pack; with sharded views the caller all-reduces
 * grad..loss_sum[1], contiguous) and
 * are consumed + cleared by ivr_inverse_update, which records losses[iter],
 * applies Adam per learnable group (bit q of `learnable`) whose mean
 * gradient exceeds 1e-12, and refreshes tab (palettes (3S), opacity scales
 * (S)) and the n_views device frame params (lam, b, rescale flag, orbital
 * light direction + derivatives).  ctl = [iteration, first gated iteration
 * (-1), reason bits]: a pair-capacity overflow or a non-finite loss gates
 * that and every later update.  n_scenes <= 1024. */
#define IVR_INV_OVERFLOW 1
#define IVR_INV_DIVERGED 2
typedef struct ivr_inverse_step {
    int32_t n_scenes, n_views, orbital, learnable;
    int64_t iters;
    double view_div; /* views over all ranks (mean divisor); <= 0: n_views.  A rank
                      * holding no view (n_views = 0) needs view_div > 0 */
    double *x, *m, *v;
    int64_t *t;
    double lr, beta1, beta2, eps;
    double *grad, *loss_sum, *losses;
    int64_t *ctl;
    ivr_frame_params *params; /* n_views, device */
    double *tab;              /* 4S, device */
} ivr_inverse_step;
int ivr_inverse_pack(const ivr_inverse_step *a, const double *photo_sums, double numel,
                     double windows, const double *d_c_p, const double *d_scale,
                     const double *d_globals, const int32_t *n_pairs, int64_t pair_capacity,
                     ivr_stream_t stream);
int ivr_inverse_update(const ivr_inverse_step *a, ivr_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* IVRGS_H */
