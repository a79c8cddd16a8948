/*
 * sgad.h -- C ABI of the B200-native SGAD-SLAM hot paths (libsgad.so).
 *
 * Plain pointers, sizes and opaque handles only; device pointers are
 * caller-allocated (PyTorch owns them on the Python side) unless a function
 * says it returns into handle-owned scratch.  Every function returns SGAD_OK
 * (0) or a negative SGAD_E_* code; sgad_last_error() describes the most
 * recent failure of the calling thread.  All work is ordered on the given
 * CUDA stream (passed as void* so the header needs no CUDA includes).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/raysplat):
 *   sgad_raster_prepare   <- rasterizer.py:79-175 (_prepare) and :178-218
 *                            (_build_tile_lists): projection, (z, frame, pixel)
 *                            sort, tile binning
 *   sgad_raster_forward   <- rasterizer.py:221-269 (_forward_kernel) and
 *                            :366-392 (splat); optional fused tau=0 L1 loss of
 *                            mapper.py:118-152
 *   sgad_raster_backward  <- rasterizer.py:272-363 (_backward_kernel) and the
 *                            chain rule :451-483 (splat_backward)
 *   sgad_adam_step        <- mapper.py:73-95 (MapOptimizer.step)
 *   sgad_voxels_*         <- tracker.py:105-122 (GlobalGeomSet.insert cell gating)
 *   sgad_inpaint_jacobi   <- datasets.py:368-398 (inpaint_depth sweeps)
 *   sgad_irls_normal_eqs  <- tracker.py:400-410 (init_pose_render IRLS systems)
 *   sgad_ssim             <- ssim.py:31-87 (ssim(..., with_grad)), the tau term
 *                            of mapping_loss (mapper.py:126-147)
 *   sgad_track_fit        <- tracker.py:144-170, :193-230 (build_local_set with
 *                            the 5x5 window neighbourhood of north_star, delta D2)
 *   sgad_sym_eigh3        <- geometry.py:275-353 (sym_eigh3_batch)
 *   sgad_geomset_*        <- tracker.py:81-133 (GlobalGeomSet: storage + exact
 *                            Euclidean 1-NN, query_nearest :125-128)
 *   sgad_track_normal_eqs <- tracker.py:286-321 (one GICP iteration's
 *                            correspondences, gate, combined covariance,
 *                            H = sum J^T W J, g = sum J^T W d, cost)
 *   sgad_track_gicp       <- tracker.py:265-346 (the whole Gauss-Newton loop on
 *                            the device, one host round trip per registration)
 *   sgad_track_cost       <- tracker.py:312-314,329-333 (frozen-weight cost at
 *                            candidate poses for step halving)
 */
#ifndef SGAD_H
#define SGAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGAD_OK 0
#define SGAD_E_INVALID (-1)
#define SGAD_E_CUDA (-2)
#define SGAD_E_NOMEM (-3)
#define SGAD_E_STATE (-4)

/* One source map as seen from one target view. */
typedef struct sgad_frame {
  const void* planes;    /* device [7, H, W] fp32 or fp64 (planes_f64): base_depth,
                            delta, log_radius, opacity_logit, R, G, B
                            (gaussians.py:9-13 plane order, radius stored as log) */
  const uint8_t* mask;   /* device [H, W] active mask */
  int64_t gauss_offset;  /* global Gaussian id of pixel 0 (ids index grad buffers) */
  int64_t frame_index;   /* reference frame index (documentation; order is by array) */
  int32_t height, width;
  int32_t learnable;     /* 1: this map receives gradients */
  int32_t planes_f64;    /* 1: planes are fp64 (drop-in maps), 0: fp32 (window engine) */
  double fx, fy, cx, cy; /* source intrinsics */
  double rot[9];         /* rel = T_target^-1 o T_source, row-major (rasterizer.py:94) */
  double trans[3];
} sgad_frame;

typedef struct sgad_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
} sgad_camera;

/* tau = 0 mapping loss target (mapper.py:118-152), all device pointers. */
typedef struct sgad_loss_target {
  const float* color;    /* [H, W, 3] */
  const float* depth;    /* [H, W] */
  const uint8_t* mask;   /* [H, W] valid depth */
  double rho, sigma;     /* colour / depth weights */
  int64_t n_depth;       /* number of valid depth pixels (|U|) */
  double* loss_accum;    /* device double[2] += (sum |C'-C|, sum_U |D'-D|) */
} sgad_loss_target;

typedef struct sgad_raster sgad_raster;

const char* sgad_last_error(void);
int sgad_version(void);
/* Number of this library's own kernels launched so far in the process (the
 * bench's gpu_launches; CUB's sort/scan kernels are library kernels and not
 * counted). */
int sgad_launch_count(int64_t* out);

int sgad_raster_create(sgad_raster** out);
int sgad_raster_destroy(sgad_raster* h);

/* Project + cull all frames into the target camera, sort survivors by
 * (z, frame, pixel) and bin them into 16x16 tiles.  `frames` is a HOST array,
 * ordered by (frame_index, map order).  want_coef != 0 also stores the per-
 * survivor chain-rule coefficients the fused backward needs.  Synchronises
 * the stream once to size the sorts; returns the survivor and pair counts. */
int sgad_raster_prepare(sgad_raster* h, const sgad_frame* frames, int32_t n_frames,
                        const sgad_camera* cam, int32_t want_coef, void* stream,
                        int64_t* n_survivors, int64_t* n_pairs);

/* The same preparation without any host synchronisation (the window engine;
 * capturable in a CUDA graph): element counts stay on the device.
 * counts_out (device uint32[2], may be NULL) receives (survivors, pairs);
 * if the view has more tile pairs than the handle's capacity (see
 * sgad_raster_reserve; at least 2 x Gaussians) the extra pairs are
 * dropped and *overflow_flag (device int32, may be NULL) is set to 1 --
 * the caller discards the view's results, reserves more and prepares again.
 * frames_dev (device, may be NULL): a resident device copy of frames[] to
 * use instead of uploading it (nothing is then read from host memory). 
 * Replaces the same reference functions as sgad_raster_prepare. */
int sgad_raster_prepare_async(sgad_raster* h, const sgad_frame* frames, int32_t n_frames,
                              const sgad_camera* cam, int32_t want_coef,
                              const sgad_frame* frames_dev, uint32_t* counts_out,
                              int32_t* overflow_flag, void* stream);

/* Grow the handle's tile-pair capacity (buffers are resized at the next
 * preparation). */
int sgad_raster_reserve(sgad_raster* h, int64_t pair_capacity);

/* Composite the prepared view.  Image outputs (fp64 / int32, device) may be
 * NULL.  save_state != 0 keeps per-pixel final transmittance and last list
 * position for the backward.  target != NULL fuses the tau=0 L1 loss and
 * records the residual signs the fused backward consumes. */
int sgad_raster_forward(sgad_raster* h, double* out_color, double* out_depth, double* out_alpha,
                        int32_t* out_count, int32_t save_state, const sgad_loss_target* target,
                        void* stream);

/* Backward of the prepared + forwarded view.
 * mode 0 (exact): upstream images g_color/g_depth/g_alpha (fp64, device)
 *   are required; per-survivor fp64 gradients are accumulated and chained in
 *   fp64 exactly as rasterizer.py:462-483, then ADDED into the per-frame
 *   fp64 outputs map_grads[f] (device [6, H, W]: delta, radius, opacity_logit,
 *   R, G, B; NULL entries for non-learnable maps).
 * mode 1 (fused): upstream comes from the fused loss of the preceding
 *   forward (target != NULL there) -- or, for the colour channels, from
 *   g_color when it is given (the tau != 0 objective: sgad_ssim's upstream);
 *   per-contribution gradients are chained in fp64, rounded to fp32 and
 *   atomically added into grad_accum (device [N_total, 8] fp32: delta,
 *   radius, opacity_logit, R, G, B, -, -). */
int sgad_raster_backward(sgad_raster* h, int32_t mode, const double* g_color,
                         const double* g_depth, const double* g_alpha, double* const* map_grads,
                         float* grad_accum, void* stream);

/* Forward + fused L1 loss + fused backward of the prepared view in ONE
 * kernel (the tau = 0 window step): each tile's backward sweep starts from
 * the forward's per-pixel state in registers.  Same results as
 * sgad_raster_forward(target) + sgad_raster_backward(mode 1) (the per-pixel
 * state is not kept, so no separate backward may follow).  Requires
 * want_coef at prepare and fp32 window parameters. */
int sgad_raster_forward_backward(sgad_raster* h, const sgad_loss_target* target,
                                 float* grad_accum, void* stream);

/* Inspection (tests): survivors in sorted order and the tile lists with
 * entries expressed as sorted ranks (directly comparable to the reference's
 * `lists`).  Any pointer may be NULL.  ranges: [n_tiles, 2] int64 (start,end). */
int sgad_raster_get_survivors(sgad_raster* h, int64_t* gid, double* u0, double* v0, double* z,
                              double* sigma, double* opacity, void* stream);
int sgad_raster_get_tiles(sgad_raster* h, int64_t* ranges, int64_t* lists, void* stream);
int sgad_raster_tile_count(sgad_raster* h, int64_t* n_tiles);

/* Adam over window parameters (mapper.py:73-95).  params [F, 7, HW] and
 * m, v [F, 6, HW] and grads [F*HW, 8] (consumed and zeroed) in fp32
 * (f64 == 0) or fp64 (f64 != 0).
 * bc1 = 1 - beta1^t, bc2 = 1 - beta2^t.  lr[6] per channel (delta, log_radius,
 * opacity_logit, R, G, B); update_delta == 0 freezes the offsets.  skip
 * (device int32, may be NULL): when *skip != 0 the gradients are consumed
 * (zeroed) and nothing is updated (a window step whose preparation
 * overflowed, see sgad_raster_prepare_async).  step_dev (device int32, may
 * be NULL; fp32 only): the step count t is read from device memory and bc1,
 * bc2 are formed from it (a step captured in a CUDA graph). */
int sgad_adam_step(void* params, void* grads, void* m, void* v, int64_t n_frames, int64_t hw,
                   const double* lr, double beta1, double beta2, double eps, double bc1,
                   double bc2, int32_t update_delta, int32_t f64, const int32_t* skip,
                   const int32_t* step_dev, void* stream);

/* ---- render-based pose initialiser ------------------------------------
 * One IRLS linearisation of tracker.py:400-410: rows (device fp64 [12, n]) are
 * the residuals at the poses exp(+h e_k) o pose, exp(-h e_k) o pose for k =
 * 0..5 (rows 2k, 2k+1), r (device [n]) the residual at the pose; with
 * J = (rows[2k] - rows[2k+1]) / 2h and w = 1 / max(|r + J xi|, 1e-3) (xi: 6
 * host doubles) writes out (device double[27]) = the 21 upper-triangle
 * entries of J^T diag(w) J (row-major) then J^T (w r).  partial: device
 * scratch of 592 * 27 doubles.  Deterministic. */
int sgad_irls_normal_eqs(const double* rows, const double* r, int64_t n, const double* xi,
                         double h, double* partial, double* out, void* stream);

/* ---- harmonic depth inpainting ----------------------------------------
 * Replaces the Jacobi loop of raysplat/datasets.py:388-397 (inpaint_depth):
 * depth (device [H, W] fp64, holes already seeded with their nearest valid
 * value) is relaxed in place over the pixels with hole[p] != 0 until the
 * sweep whose largest update is below tol, or max_iters sweeps; scratch is a
 * device [H, W] fp64 buffer; *sweeps (host) = sweeps applied.  Synchronises
 * the stream. */
int sgad_inpaint_jacobi(double* depth, const uint8_t* hole, int32_t height, int32_t width,
                        int32_t max_iters, double tol, double* scratch, int32_t* sweeps,
                        void* stream);

/* ---- SSIM term (tau != 0 objective) ------------------------------------
 * Replaces raysplat/ssim.py:31-87 (ssim(img_a, img_b, with_grad)) as used by
 * mapper.py:126-147.  Images are device [H, W, C] interleaved, img_a fp64,
 * img_b fp64 or fp32 (b_is_f32).  *sum_out (device double) += the SUM of the
 * per-pixel, per-channel SSIM (the mean is sum / (H W C)).  With grad_out
 * (device double [H, W, C]) and a workspace of sgad_ssim_workspace_size
 * bytes, writes d(mean SSIM)/d(img_a); with upstream != 0 it writes instead
 * the mapping loss's colour upstream  kc * sign(a - b) - tau * grad
 * (mapper.py:145-147 with kc = rho / (3 H W)). */
int sgad_ssim_workspace_size(int32_t height, int32_t width, int32_t channels, int64_t* bytes);
int sgad_ssim(const double* img_a, const void* img_b, int32_t b_is_f32, int32_t height,
              int32_t width, int32_t channels, double* sum_out, double* grad_out,
              double* workspace, double kc, double tau, int32_t upstream, void* stream);

/* ----------------------------------------------------------- tracking */

/* Batched 3x3 symmetric eigendecomposition (geometry.py:275-353):
 * mats [n, 9] fp64 row-major -> rot [n, 9], vals [n, 3] descending. */
int sgad_sym_eigh3(const double* mats, int64_t n, double* rot, double* vals, void* stream);

/* Local geometry Gaussians from one depth frame.  Samples every `stride`-th
 * row/column among valid pixels, fits the covariance of the valid
 * neighbours in a win x win window (self excluded, >= k_min of them),
 * eigen-decomposes, floors, normalises (scale_mode 0 ellipse, 1 plane,
 * 2 none) and orients the normal to the camera.  Outputs are compacted in
 * row-major pixel order; *count (device int64) receives their number.
 * centers [M,3], cov [M,6] (xx,xy,xz,yy,yz,zz), normals [M,3], rot [M,9],
 * scales [M,3], pixel [M] (rot/scales/pixel may be NULL). */
int sgad_track_fit(const float* depth, const uint8_t* mask, int32_t height, int32_t width,
                   double fx, double fy, double cx, double cy, int32_t stride, int32_t win,
                   int32_t k_min, int32_t scale_mode, double* centers, double* cov,
                   double* normals, double* rot, double* scales, int64_t* pixel,
                   int64_t* count, void* stream);

typedef struct sgad_geomset sgad_geomset;

/* Target set for registration: device copies of centers [n,3], cov [n,6],
 * normals [n,3] (fp64) plus a uniform-grid exact 1-NN index. */
int sgad_geomset_create(sgad_geomset** out);
int sgad_geomset_destroy(sgad_geomset* g);
int sgad_geomset_set(sgad_geomset* g, const double* centers, const double* cov,
                     const double* normals, int64_t n, void* stream);
/* exact Euclidean nearest neighbour: idx [m] int64, dist [m] fp64 */
int sgad_geomset_nearest(sgad_geomset* g, const double* queries, int64_t m, int64_t* idx,
                         double* dist, void* stream);

/* One GICP linearisation (tracker.py:286-321) at pose (rot row-major, trans).
 * local: centers [m,3], cov [m,6] in the local camera frame.
 * metric_mode 0 point2surf, 1 point2point; gate `dist_max`.
 * warm_start != 0 seeds the exact nearest-neighbour search with the previous
 * call's neighbours (same local set; the result is still the exact 1-NN).
 * out (device double[29]): H upper triangle (21, row-major), g (6), cost, inliers.
 * The frozen weights W (6 per correspondence, 0 for rejected) and the matched
 * target centres are kept in the geomset for sgad_track_cost. */
int sgad_track_normal_eqs(sgad_geomset* g, const double* local_centers, const double* local_cov,
                          int64_t m, const double* rot, const double* trans, int32_t metric_mode,
                          double dist_max, int32_t warm_start, double* out, void* stream);

/* Copy the per-correspondence acceptance flags of the last
 * sgad_track_normal_eqs call (device uint8 [m]). */
int sgad_track_accepted(sgad_geomset* g, uint8_t* out, int64_t m, void* stream);

/* The last sgad_track_normal_eqs call's exact nearest neighbours (device
 * int64 [m]; tracker.py:288 j).  Across GICP iterations a query whose old
 * neighbour is provably still the unique nearest (it moved by delta, every
 * other point was >= d2 away at its last full search, and the old neighbour
 * is now closer than d2 - delta) skips the search. */
int sgad_track_correspondences(sgad_geomset* g, int64_t* idx, int64_t m, void* stream);

/* Frozen-weight cost sum_i (b_i - T a_i)^T W_i (b_i - T a_i) for n_cand poses
 * (poses: host array [n_cand, 12], rot row-major then trans) -> out[n_cand]
 * (device). */
int sgad_track_cost(sgad_geomset* g, const double* local_centers, int64_t m, const double* poses,
                    int32_t n_cand, double* out, void* stream);

/* update_global_set's change of frame (tracker.py:233-238) on the device:
 * centres R c + t and normals R n (numpy's BLAS order), rotations R rot
 * (einsum order), and the packed covariances rot' diag(s^2) rot'^T of the
 * result (GlobalGeomSet.covariances, :130-133) -> out_cov6 [n, 6].  All
 * device fp64: centres/normals/scales [n, 3], rotations [n, 3, 3]; rot/trans
 * host [9] / [3]. */
int sgad_track_to_world(const double* centers, const double* rotations, const double* scales,
                        const double* normals, int64_t n, const double* rot, const double* trans,
                        double* out_centers, double* out_rotations, double* out_normals,
                        double* out_cov6, void* stream);

/* A whole gicp_align (tracker.py:265-346) enqueued at once and read back once:
 * per iteration the 6x6 solve (np.linalg.solve's partial-pivot LU), the step
 * and its 5 halvings (se3_exp(xi).compose(pose)), their frozen-weight costs,
 * the acceptance test and the next linearisation at the accepted pose all
 * run on the device.  init_pose: host [12] (rot row-major, trans).  Outputs
 * (host): result[19] = final pose (12), final cost, iterations, inlier count,
 * converged, failed, singular iteration (-1: none; at an exactly singular
 * system -- where numpy falls back to lstsq -- the loop stops with `pose` the
 * pose reached and the caller continues on the host), systems logged;
 * systems (optional) [max_iters, 29] as sgad_track_normal_eqs' out per
 * iteration; cost_pairs (optional) [max_iters, 2] (cost before, after) per
 * accepted iteration; accepted_first (optional, device or host uint8 [m]):
 * the first linearisation's acceptance flags. */
int sgad_track_gicp(sgad_geomset* g, const double* local_centers, const double* local_cov,
                    int64_t m, const double* init_pose, int32_t metric_mode, double dist_max,
                    int32_t max_iters, double convergence_eps, int32_t warm_start,
                    int32_t min_inliers, double* result, double* systems, double* cost_pairs,
                    uint8_t* accepted_first, void* stream);

/* ---- voxel occupancy of the global geometry set -----------------------
 * Replaces the cell gating of GlobalGeomSet.insert (tracker.py:105-122): a
 * device hash table of occupied cells floor(center / voxel_size).  For a
 * batch of centers (device [n, 3] fp64) keep[i] (device u8) = 1 iff row i's
 * cell is not occupied by an earlier batch and no earlier row of this batch
 * has the same cell; the kept cells become occupied; *n_keep (host) = the
 * number kept.  Cells must satisfy |cell| < 2^20 per axis (else SGAD_E_INVALID
 * and the batch is not inserted). */
typedef struct sgad_voxels sgad_voxels;
int sgad_voxels_create(sgad_voxels** out);
int sgad_voxels_destroy(sgad_voxels* v);
int sgad_voxels_gate(sgad_voxels* v, const double* centers, int64_t n, double voxel_size,
                     uint8_t* keep, int64_t* n_keep, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SGAD_H */
