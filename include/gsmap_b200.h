/* gsmap_b200 — B200-native (sm_100a) drop-in for the LVI-GS mapping hot path.
 *
 * C-ABI boundary (extern "C", POD structs, opaque handles, int status). No CUDA, torch or
 * C++ types cross it. Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj). The C++ shim in gsmap_b200.hpp re-exports the
 * reference signatures over these calls and rethrows the reference's exception types.
 *
 * Conventions shared with the reference:
 *   - a Gaussian is 59 fp64 scalars in gaussian.hpp:16-26 order: position[3], rotation (w,x,y,z)
 *     [4], log_scale[3], opacity_logit[1], sh[16][3]; plus int active_degree.
 *   - host images are row-major HWC fp64 (io/image.hpp:26-33), color H*W*3, depth/vis H*W.
 *   - gs_pose holds the NORMALISED q_cw (w,x,y,z) + t_cw, exactly as gsmap::Pose stores it
 *     (core/types.hpp:53-54). gs_camera is gsmap::CameraModel (core/types.hpp:15-45).
 * Device state: the map lives on the GPU as fp32 SoA planes ([59][capacity]) plus Adam m/v
 * planes, an int32 per-Gaussian step and an int8 degree. Host<->device conversion happens only
 * in gs_map_{append,set,get}_* and gs_frame_read / host-cotangent entry points.
 */
#ifndef GSMAP_B200_H
#define GSMAP_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ shim maps GS_EINVAL -> std::invalid_argument and GS_ELOGIC ->
 * std::logic_error, the two exception types the reference throws on this path. */
enum {
    GS_OK = 0,
    GS_EINVAL = 1, /* std::invalid_argument (types.hpp:22-29, rasterizer.cpp:229-234, ...) */
    GS_ELOGIC = 2, /* std::logic_error (rasterizer.cpp:236-237) */
    GS_ECUDA = 3,
    GS_ENCCL = 4,
    GS_ENOMEM = 5,
    GS_ERUNTIME = 6 /* std::runtime_error (io/checkpoint.cpp: open / format / truncation) */
};

typedef struct gs_camera { double fx, fy, cx, cy; int32_t width, height; } gs_camera;
typedef struct gs_pose { double qw, qx, qy, qz, tx, ty, tz; } gs_pose;
typedef struct gs_gaussian { double p[59]; int32_t active_degree; int32_t pad; } gs_gaussian;
typedef struct gs_learning_rates { double position, rotation, log_scale, opacity, sh; } gs_learning_rates;
typedef struct gs_train_config {
    double lambda, lambda_d;            /* mapper.hpp:17-19 */
    int32_t pyramid_levels, iters_per_level; /* mapper.hpp:20-21 */
    gs_learning_rates lr;               /* mapper.hpp:22 */
} gs_train_config;
typedef struct gs_loss_result { double total, color_loss, depth_loss, l1, ssim, psnr; } gs_loss_result;
typedef struct gs_step_report { int32_t ran, level; double loss, psnr; } gs_step_report;
typedef struct gs_frame_stats {
    int64_t n_visible;   /* projected (survived near clip + off-screen cull) */
    int64_t n_pairs;     /* (tile, gaussian) pairs = tile-list entries */
    int64_t n_contrib;   /* total compositing contributions (sum of per-pixel list lengths) */
    int32_t tiles_x, tiles_y, width, height;
} gs_frame_stats;

typedef struct gs_context gs_context;
typedef struct gs_map gs_map;
typedef struct gs_frame gs_frame;
typedef struct gs_grads gs_grads;
typedef struct gs_keyframe gs_keyframe;
typedef struct gs_comm gs_comm;

const char* gs_last_error(void);
const char* gs_version(void);

/* ---- context: one device + one CUDA stream (stream may be an external cudaStream_t) ---- */
int gs_context_create(int device, void* cuda_stream, gs_context** out);
int gs_context_destroy(gs_context* ctx);
int gs_context_synchronize(gs_context* ctx);
int gs_context_set_stream(gs_context* ctx, void* cuda_stream);
/* number of this library's kernel launches since creation (bench/driver evidence) */
int gs_context_launch_count(gs_context* ctx, int64_t* count);
/* per-kernel CUDA-event timing on the context stream (enable != 0 resets the table) */
int gs_context_profile(gs_context* ctx, int enable);
/* forward-blend slow-path statistics: [0] near-threshold checks, [1] exact fp64 replays */
int gs_debug_counters(gs_context* ctx, int64_t* out2, int reset);
/* override the blend kernels' pixels-per-thread (2, 4 or 8; 0 = automatic per level) */
int gs_debug_set_blend_ppt(int fwd, int bwd);
/* forward blend: tiles with more list entries than this carry the transmittance as df32
   instead of fp32 + error band (tuning knob; negative = default) */
int gs_debug_set_blend_df_list(int entries);
/* backward: list segments per tile (one CTA each; the forward checkpoints the boundaries);
   0 = automatic per level */
int gs_debug_set_blend_segments(int nseg);
/* forward: walk the list segments in parallel (local pass, chain, exact finish) on levels with
   list segments and at most this many tiles (default 512; 0 = always the sequential walk;
   negative = default) */
int gs_debug_set_seg_forward(int max_tiles);
/* diagnostics: gs_train_step skips its loss read-back (report.loss = NaN, no overflow re-run),
   so the host can enqueue ahead of the device */
int gs_debug_defer_step_sync(gs_context* ctx, int defer);
/* host-side enqueue time per profiling scope (same table as gs_context_profile_read) */
int gs_debug_profile_host(gs_context* ctx, char* names, int32_t names_len, double* host_ms, int32_t max_entries,
                          int32_t* n_entries);
/* reads the table: names as one '\n'-separated string, per-name total ms and launch counts */
int gs_context_profile_read(gs_context* ctx, char* names, int32_t names_len, double* total_ms,
                            int64_t* launches, int32_t max_entries, int32_t* n_entries);

/* roofline denominators measured on this device: kind 0 = FP32 FMA flop/s, 1 = MUFU.EX2/s */
int gs_microbench(int device, int kind, double* per_second);

/* ---- camera helpers (core/types.hpp:22-44) ---- */
int gs_camera_validate(const gs_camera* cam);
int gs_camera_scaled(const gs_camera* cam, int level, gs_camera* out);

/* ---- GaussianMap (map/gaussian_map.hpp:44-96) ---- */
int gs_map_create(gs_context* ctx, gs_map** out);
int gs_map_destroy(gs_map* map);
int gs_map_size(const gs_map* map, int64_t* n);
/* GaussianMap::append (gaussian_map.cpp:31-35): fresh Adam state, refresh_extent */
int gs_map_append(gs_map* map, const gs_gaussian* g, int64_t n);
/* host edit through non-const gaussians() (gaussian_map.hpp:62): overwrite all n params */
int gs_map_set_gaussians(gs_map* map, const gs_gaussian* g, int64_t n);
int gs_map_get_gaussians(gs_map* map, gs_gaussian* out, int64_t n);
int gs_map_get_adam(gs_map* map, double* m59, double* v59, int64_t* step, int64_t n);
int gs_map_set_adam(gs_map* map, const double* m59, const double* v59, const int64_t* step, int64_t n);
int gs_map_scene_extent(const gs_map* map, double* extent);
int gs_map_set_scene_extent(gs_map* map, double extent);
int gs_map_global_step(const gs_map* map, int64_t* step);
int gs_map_set_global_step(gs_map* map, int64_t step);
int gs_map_raise_sh_degree(gs_map* map, int degree);   /* gaussian_map.cpp:75-79 */
/* project_sparse_depth (io/sequence.hpp:70, sequence.cpp:246-259): host points [n][stride]
   (x, y, z world first, fp64; stride 6 = the reference's ColoredPoint xyz+rgb) -> host depth
   [h][w] fp64, the minimum camera z per pixel, 0 where no point lands. */
int gs_project_sparse_depth(gs_context* ctx, const double* points, int64_t n, int32_t stride, const gs_pose* pose,
                            const gs_camera* cam, double* depth);
/* maybe_upgrade_sh (mapper.hpp:78-80, mapper.cpp:240-246): raise every Gaussian's SH degree to
   min(3, global_step / sh_interval) (sh_interval <= 0: unchanged); *degree = the result */
int gs_maybe_upgrade_sh(gs_map* map, int32_t sh_interval, int32_t* degree);
/* init_gaussians_from_points (map/mapper.hpp, mapper.cpp:43-61) on the device: host points
   [n][6] (x y z world, r g b) -> n new Gaussians appended to the map (isotropic scale = mean
   distance to the 3 nearest other points, exact grid search; opacity 0.1; SH0 from the colour;
   degree 0; fresh optimizer state). *added = n. */
int gs_map_init_from_points(gs_map* map, const double* points6, int64_t n, int64_t* added);
/* diagnostics: speculative next-step renders enqueued / used on this context (gs_train_step_prefetch) */
int gs_debug_speculation(gs_context* ctx, int64_t* out2);
/* diagnostics of the pair-capacity policy on this context: [0] capacity growths after a
   read-back, [1] train steps re-run because a render overflowed its capacity, [2] renders that
   read their pair count back before binning (first render of a resolution, exact re-runs) */
int gs_debug_capacity(gs_context* ctx, int64_t* out3);
/* checkpoint format v1 (io/checkpoint.cpp:17-73): text header + 476-byte fp64 AoS records.
   save_checkpoint writes the device map's parameters (exact fp64 widening of the fp32 store);
   load_checkpoint returns a NEW map (fresh Adam state, GaussianMap::append) or GS_ERUNTIME for
   a missing / foreign / wrong-version / truncated file, with the reference's messages. */
int gs_save_checkpoint(gs_map* map, const char* path);
int gs_load_checkpoint(gs_context* ctx, const char* path, gs_map** out);
/* optimizer state beside a checkpoint, for a true resume (the v1 format carries none):
   per Gaussian Adam m / v (59 each) and step, plus the map's global_step and scene_extent. load requires a map of
   the same size (e.g. fresh from gs_load_checkpoint). */
int gs_save_training_state(gs_map* map, const char* path);
int gs_load_training_state(gs_map* map, const char* path);
/* evaluate_sequence (pipeline.cpp:41-64) for one frame: render at the pose, quantize_8bit the
   colour (pipeline.cpp:34-39), psnr / ssim against gt_color (H x W x 3, HWC) and depth_rmse of
   the raw depth against gt_depth (H x W; NULL -> depth_rmse = NaN, as with no valid pixel). */
typedef struct gs_eval_metrics {
    double psnr;
    double ssim;
    double depth_rmse;
} gs_eval_metrics;
int gs_evaluate_view(gs_map* map, const gs_pose* pose, const gs_camera* cam, const double* gt_color,
                     const double* gt_depth, gs_eval_metrics* out);
/* filter_points_by_visibility (map/keyframe.hpp, keyframe.cpp:49-74): render the map at the pose
   and keep the points (in order) that are behind the near plane, project outside the image or
   land on a pixel with visibility <= tau_alpha; tau_alpha outside [0, 1] -> GS_EINVAL.
   kept6 must hold n points. */
int gs_filter_points_by_visibility(gs_map* map, const double* points6, int64_t n, const gs_pose* pose,
                                   const gs_camera* cam, double tau_alpha, double* kept6, int64_t* n_kept);
/* keyframe integration (pipeline.cpp:151-155) without a host round trip of the kept set:
   filter_points_by_visibility then init_gaussians_from_points; *added = the kept count */
int gs_map_integrate_points(gs_map* map, const double* points6, int64_t n, const gs_pose* pose,
                            const gs_camera* cam, double tau_alpha, int64_t* added);
/* integrate_keyframe (pipeline.cpp:148-155) in one call: the frame's cloud is uploaded once;
   filter_points_by_visibility -> init_gaussians_from_points append to the map, and the new
   keyframe (*out_kf, destroy with gs_keyframe_destroy) gets project_sparse_depth of the same
   cloud and the colour image (H x W x 3 HWC) as its pyramid (build_keyframe_pyramid).
   *added = Gaussians appended. The step that follows is the caller's (gs_train_step). */
int gs_integrate_keyframe(gs_map* map, const gs_pose* pose, const gs_camera* cam, const double* color,
                          const double* points6, int64_t n, double tau_alpha, int32_t initial_iters, int32_t levels,
                          gs_keyframe** out_kf, int64_t* added);
/* GaussianMap::prune (gaussian_map.hpp:79, gaussian_map.cpp:56-73): drop every Gaussian with
   sigmoid(opacity_logit) < threshold, compacting parameters and optimizer state in order;
   threshold outside (0, 1) -> GS_EINVAL. *removed = the number dropped. */
int gs_map_prune(gs_map* map, double opacity_threshold, int64_t* removed);
int gs_map_max_active_degree(gs_map* map, int* degree);
/* device SoA access: params/m/v planes [59][capacity] fp32 */
int gs_map_device_planes(gs_map* map, float** params, float** adam_m, float** adam_v, int64_t* capacity);

/* ---- render (rasterizer.hpp:69-70): project -> depth sort -> tile keys -> blend ---- */
int gs_frame_create(gs_context* ctx, gs_frame** out);
int gs_frame_destroy(gs_frame* frame);
int gs_render(gs_map* map, const gs_pose* pose, const gs_camera* cam, gs_frame* frame);
int gs_frame_stats_get(gs_frame* frame, gs_frame_stats* out);
/* RenderOutput color/depth/visibility as host fp64 HWC (any pointer may be NULL) */
int gs_frame_read(gs_frame* frame, double* color, double* depth, double* visibility);
/* a RenderOutput from host images (compute_loss takes any rendered images, mapper.hpp:61-62):
   fp64 HWC color / depth / visibility; the frame has no contributor lists, so
   gs_render_backward on it returns GS_ELOGIC (the reference's inconsistent-CSR error) */
int gs_frame_set_images(gs_frame* frame, const double* color, const double* depth, const double* visibility,
                        int32_t h, int32_t w);
/* device planes: color [3][H][W], depth [H][W], visibility [H][W] (fp32) */
int gs_frame_device_images(gs_frame* frame, float** color, float** depth, float** visibility);
/* per-pixel list length and final transmittance (H*W each) */
int gs_frame_read_pixel_state(gs_frame* frame, int32_t* n_contrib, float* t_final);
/* depth-sorted projected set (ProjectedGaussian order, rasterizer.cpp:69-72): map index,
 * fp64 mean[2], int pixel rect[4] (x0, y0, x1, y1 = clamped ceil(mean-r)..floor(mean+r),
 * rasterizer.cpp:81-84; x0 > x1 when empty), fp32 conic[3] (cov_inv 00,01,11), fp32 opacity,
 * fp32 color[3], fp64 depth; each pointer may be NULL; arrays sized n_visible */
int gs_frame_read_projected(gs_frame* frame, int32_t* index, double* mean2, int32_t* rect4,
                            float* conic3, float* opacity, float* color3, double* depth);
/* tile lists (bin_tiles, rasterizer.cpp:76-91): tile_offsets[T+1], entries[n_pairs] = map index */
int gs_frame_read_tiles(gs_frame* frame, int64_t* tile_offsets, int32_t* entries);
/* CSR contributor table (RenderOutput::contrib_offsets/contribs, rasterizer.hpp:52-53), built
 * only on request: offsets[H*W+1], gaussian[n_contrib], alpha[n_contrib] */
int gs_frame_materialize(gs_frame* frame, uint32_t* offsets, int32_t* gaussian, double* alpha);

/* ---- gradients (RenderGradients, rasterizer.hpp:62-64) as device fp32 planes [59][cap] ---- */
int gs_grads_create(gs_context* ctx, gs_grads** out);
/* external storage (e.g. a torch tensor that NCCL all-reduces): floats >= 59 * capacity */
int gs_grads_create_external(gs_context* ctx, float* device_ptr, int64_t capacity, gs_grads** out);
int gs_grads_destroy(gs_grads* grads);
int gs_grads_zero(gs_grads* grads, gs_map* map);
int gs_grads_read(gs_grads* grads, double* out59, int64_t n);
int gs_grads_write(gs_grads* grads, const double* in59, int64_t n);
int gs_grads_device_planes(gs_grads* grads, float** planes, int64_t* capacity);

/* render_backward (rasterizer.hpp:74-77) with host fp64 cotangents; OVERWRITES grads */
int gs_render_backward(gs_map* map, const gs_pose* pose, const gs_camera* cam, gs_frame* frame,
                       const double* dl_dcolor, const double* dl_ddepth, int32_t h, int32_t w,
                       gs_grads* grads);
/* GaussianMap::apply_gradients (gaussian_map.cpp:37-54): one Adam step on every Gaussian */
int gs_apply_gradients(gs_map* map, gs_grads* grads, const gs_learning_rates* lr);

/* ---- keyframe + loss + fused train step (mapper.hpp:61-76) ---- */
/* builds the pyramid (build_keyframe_pyramid, mapper.cpp:137-144) on the device */
int gs_keyframe_create(gs_context* ctx, const gs_pose* pose, const double* color,
                       const double* sparse_depth, int32_t h, int32_t w, int32_t initial_iters,
                       int32_t levels, gs_keyframe** out);
/* same, from device fp32 level-0 planes (color [3][H][W], depth [H][W]) */
int gs_keyframe_create_device(gs_context* ctx, const gs_pose* pose, const float* color_planes,
                              const float* depth, int32_t h, int32_t w, int32_t initial_iters,
                              int32_t levels, gs_keyframe** out);
int gs_keyframe_destroy(gs_keyframe* kf);
int gs_keyframe_consumed(gs_keyframe* kf, int32_t* consumed);
int gs_keyframe_set_consumed(gs_keyframe* kf, int32_t consumed);
int gs_keyframe_levels(gs_keyframe* kf, int32_t* n_levels);
/* overwrite one pyramid level from host fp64 HWC images (the reference's ImageD). Runs on the
   context's copy stream, overlapping compute; the next call that reads the level (loss / train
   step / read_level) waits for it. Page-locked host buffers must stay valid until then. */
int gs_keyframe_upload_level(gs_keyframe* kf, int32_t level, const double* color, const double* depth);
/* read a pyramid level back (host fp64 HWC) */
int gs_keyframe_read_level(gs_keyframe* kf, int32_t level, double* color, double* depth);
/* compute_loss (mapper.cpp:146-212) on the frame's images vs pyramid level `level`; the
 * cotangents stay on the device for gs_render_backward_frame; optional host copies */
int gs_compute_loss(gs_frame* frame, gs_keyframe* kf, int32_t level, const gs_train_config* cfg,
                    gs_loss_result* out, double* dl_dcolor, double* dl_ddepth);
/* backward with the cotangents the last gs_compute_loss left on the frame; ACCUMULATES */
int gs_render_backward_frame(gs_map* map, const gs_pose* pose, const gs_camera* cam,
                             gs_frame* frame, gs_grads* grads);
/* train_keyframe_step (mapper.cpp:214-238): level schedule, render, loss, backward, Adam, psnr */
int gs_train_step(gs_map* map, gs_keyframe* kf, const gs_train_config* cfg, const gs_camera* cam,
                  gs_step_report* report);
/* gs_train_step plus the NEXT step's input upload (gs_keyframe_upload_level of next_kf's
   next_level from host fp64 HWC buffers), issued on the copy stream right behind this step's
   enqueued work so that the copy and its API calls overlap this step's compute (a data-loader
   prefetch; next_kf = NULL: plain gs_train_step). The host buffers must stay valid until the
   next synchronising call on the context. */
int gs_train_step_prefetch(gs_map* map, gs_keyframe* kf, const gs_train_config* cfg, const gs_camera* cam,
                           gs_keyframe* next_kf, int32_t next_level, const double* next_color,
                           const double* next_depth, gs_step_report* report);
/* keyframe-batch step: grads of every view summed (GaussianGrad::add), then the
 * caller may all-reduce gs_grads planes across ranks, then gs_apply_gradients. This call does
 * render+loss+backward for one view at its scheduled level and accumulates into grads.
 * Loss/psnr land in report only when sync != 0 (otherwise they stay on the device). */
int gs_train_accumulate(gs_map* map, gs_keyframe* kf, const gs_train_config* cfg,
                        const gs_camera* cam, gs_frame* frame, gs_grads* grads, int32_t sync,
                        gs_step_report* report);

/* ---- keyframe-batch training over NCCL (no reference counterpart; the batch is the
   sum of per-view RenderGradients, GaussianGrad::add gaussian.hpp:51-57, then ONE
   GaussianMap::apply_gradients, gaussian_map.cpp:37-54). NCCL is bound at run time (dlopen of
   libnccl.so.2); failures return GS_ENCCL. ---- */
/* ncclGetUniqueId: 128 bytes for every rank's gs_comm_create (exchange them out of band) */
int gs_comm_unique_id(uint8_t* id128);
/* ncclCommInitRank on the context's device (collective over the nranks callers) */
int gs_comm_create(gs_context* ctx, const uint8_t* id128, int32_t nranks, int32_t rank, gs_comm** out);
/* borrow an existing ncclComm_t (the caller keeps ownership; gs_comm_destroy only drops the wrapper) */
int gs_comm_wrap(gs_context* ctx, void* nccl_comm, gs_comm** out);
int gs_comm_destroy(gs_comm* comm);
int gs_comm_size(gs_comm* comm, int32_t* nranks, int32_t* rank);
/* One batch step over this rank's n views (each at its keyframe's scheduled level, like
   train_keyframe_step; a keyframe with no budget left reports ran = 0): render -> loss ->
   backward summed on the device, then
     mode 0: ncclAllReduce of the active gradient planes + the same Adam step on every replica;
     mode 1: ncclReduceScatter by Gaussian range + Adam on the own range + ncclAllGather of the
             parameters (the optimizer state stays sharded, see gs_comm_gather_optimizer_state).
   comm = NULL: a single-rank batch (no collective). reports[n]: per-view level / loss / psnr. */
int gs_train_batch(gs_map* map, gs_keyframe** kfs, int32_t n, const gs_train_config* cfg, const gs_camera* cam,
                   gs_comm* comm, int32_t mode, gs_step_report* reports);
/* re-replicate a mode-1 map's Adam m / v over the ranks (collective). Every call that reads or
   re-lays out the optimizer state (apply_gradients, train steps, append, prune, init, integrate,
   get/set_adam, training-state IO) returns GS_ELOGIC on a sharded map until this is called. */
int gs_comm_gather_optimizer_state(gs_map* map, gs_comm* comm);
int gs_map_optimizer_sharded(const gs_map* map, int32_t* sharded);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* GSMAP_B200_H */
