/*
 * odgs_b200.h — C ABI of the B200-native ODGS rasterizer (sm_100a).
 *
 * This is the drop-in boundary for the reference's rasterizer API
 * (reference tree proj/include/odgs/). Each entry point names the reference
 * function it replaces. Plain pointers and sizes only; no C++ or torch types.
 *
 * Data layouts are the reference's own (Eigen column-major storage), so an Eigen
 * caller can pass .data() directly:
 *   cloud members  SoA: means[c*n + i] (MatX3), rotations (w,x,y,z) [4][n], log_scales
 *                  [3][n], raw_opacities [n], colors [3][n]   (types.hpp:53-143)
 *   images         planar channels, each H x W column-major: img[c*W*H + x*H + y]
 *                  (ErpImage, types.hpp:184-224)
 *   per-pixel maps transmittance/walked [x*H + y]               (rasterizer.hpp:95-96)
 * Camera rotation is passed row-major here (the C++ wrapper transposes Eigen's
 * column-major Mat3).
 *
 * Errors mirror the reference's exceptions (see odgs_status); the failing Gaussian
 * index and message are available from odgs_last_error(). Calls on one context are
 * ordered on that context's CUDA stream; use one context per host thread.
 */
#ifndef ODGS_B200_H
#define ODGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ODGS_ABI_VERSION 1

typedef enum {
  ODGS_OK = 0,
  /* std::invalid_argument: bad camera (types.hpp:160-168), near-zero quaternion
     (covariance.hpp:14-15), bad settings/arguments. */
  ODGS_ERR_INVALID_ARGUMENT = 1,
  /* std::runtime_error: non-finite parameter (rasterizer.hpp:134-136) or non-finite
     gradient (backward.hpp:440-446); index = first offending Gaussian. */
  ODGS_ERR_RUNTIME = 2,
  /* std::domain_error: derivative undefined on the pole axis (backward.hpp:79-80,
     projection.hpp:123-124) or zero-length direction (projection.hpp:23-24). */
  ODGS_ERR_DOMAIN = 3,
  ODGS_ERR_CUDA = 4,
  ODGS_ERR_OUT_OF_MEMORY = 5
} odgs_status;

typedef enum { ODGS_MEM_HOST = 0, ODGS_MEM_DEVICE = 1 } odgs_memory;

/* RenderSettings (types.hpp:229-255). `threads` is accepted and ignored on the GPU. */
typedef struct {
  float near_radius;
  float far_radius;
  int32_t tile_size;
  float alpha_clamp;
  float transmittance_floor;
  float cutoff_sigma;
  float lowpass_dilation;
  float max_elevation;
  int32_t threads;
} odgs_settings;

/* CameraPose (types.hpp:148-180): p_cam = R p_world + t, y-down, z-forward. */
typedef struct {
  float rotation[9]; /* row-major */
  float translation[3];
  int32_t width;
  int32_t height;
} odgs_camera;

/* GaussianCloud<float> (types.hpp:53-143). All arrays live in `memory`.
   sh_degree / sh_rest: extension beyond the reference (whose colour is RGB only,
   SPEC.md:83): view-dependent colour c = rgb + sum_k Y_k(d) sh_rest[k] with real SH
   of degree 1..3 at the world-space view direction d (camera centre to Gaussian);
   sh_rest is [(deg+1)^2 - 1][3][n]. sh_degree = 0 (sh_rest NULL) is the reference. */
typedef struct {
  int64_t n;
  const float* means;
  const float* rotations;
  const float* log_scales;
  const float* raw_opacities;
  const float* colors;
  int32_t memory;
  int32_t sh_degree;
  const float* sh_rest;
} odgs_cloud;

/* GradBuffers<float> (backward.hpp:342-374), same SoA layout as the cloud. */
typedef struct {
  float* means;
  float* rotations;
  float* log_scales;
  float* raw_opacities;
  float* colors;
  float* pixel_grad_norm;
  float* one_minus_cos;
  int32_t* observed;
  int32_t memory;
  float* sh_rest; /* gradients of sh_rest (SH extension), same layout; NULL if sh_degree = 0 */
} odgs_grads;

typedef struct odgs_ctx odgs_ctx;
typedef struct odgs_frame odgs_frame;

typedef struct {
  int32_t width, height, tiles_x, tiles_y;
  int64_t n_gaussians; /* cloud size */
  int64_t n_splats;    /* projected (RenderOutput::splats.size()) */
  int64_t n_instances; /* seam instances (RenderOutput::instances.size()) */
  int64_t n_entries;   /* tile entries (RenderOutput::tile_entries.size()) */
  int32_t row_begin, row_end; /* pixel rows rendered (the whole image unless odgs_render_band) */
} odgs_frame_info;

/* Fields of a rendered frame (RenderOutput, rasterizer.hpp:92-102). */
typedef enum {
  ODGS_FRAME_IMAGE = 0,          /* float [3][W][H]                                        */
  ODGS_FRAME_TRANSMITTANCE = 1,  /* float [W][H]                                           */
  ODGS_FRAME_WALKED = 2,         /* int32 [W][H] entries examined, exclusive               */
  ODGS_FRAME_TILE_OFFSETS = 3,   /* int32 [tiles+1]                                        */
  ODGS_FRAME_TILE_ENTRIES = 4,   /* int32 [n_entries] instance ids, per tile, global order */
  ODGS_FRAME_INSTANCE_SPLAT = 5, /* int32 [n_instances] splat ids, sorted (depth,index,shift) */
  ODGS_FRAME_INSTANCE_SHIFT = 6, /* float [n_instances] -W, 0 or +W                        */
  ODGS_FRAME_SPLAT_INDEX = 7,    /* int64 [n_splats] cloud row, ascending                  */
  ODGS_FRAME_SPLAT_MEAN = 8,     /* float [n_splats][2]                                    */
  ODGS_FRAME_SPLAT_COV2D = 9,    /* float [n_splats][4] row-major (needs ODGS_FRAME_KEEP_COV2D) */
  ODGS_FRAME_SPLAT_INV = 10,     /* float [n_splats][4] row-major                          */
  ODGS_FRAME_SPLAT_DEPTH = 11,   /* float [n_splats]                                       */
  ODGS_FRAME_SPLAT_RADIUS = 12,  /* float [n_splats]                                       */
  ODGS_FRAME_SPLAT_OPACITY = 13, /* float [n_splats]                                       */
  ODGS_FRAME_SPLAT_COLOR = 14,   /* float [n_splats][3]                                    */
  ODGS_FRAME_SPLAT_CLAMPED = 15, /* int32 [n_splats] pole clamp engaged                    */
  /* SplatGrads (backward.hpp:19-25) of the last odgs_backward on this frame
     (needs ODGS_FRAME_KEEP_SPLAT_GRADS): */
  ODGS_FRAME_SPLATGRAD_MEAN = 16,    /* float [n_splats][2]                                */
  ODGS_FRAME_SPLATGRAD_COV2D = 17,   /* float [n_splats][4] full-matrix convention          */
  ODGS_FRAME_SPLATGRAD_OPACITY = 18, /* float [n_splats] w.r.t. activated opacity           */
  ODGS_FRAME_SPLATGRAD_COLOR = 19,   /* float [n_splats][3]                                */
  ODGS_FRAME_FIELD_COUNT = 20
} odgs_frame_field;

/* odgs_frame_set_flags */
#define ODGS_FRAME_KEEP_COV2D 0x1u   /* also store Sigma_2D (for ODGS_FRAME_SPLAT_COV2D) */
#define ODGS_FRAME_PLAIN_BLEND 0x2u  /* disable warp culling in the blend (A/B checks) */
#define ODGS_FRAME_KEEP_SPLAT_GRADS 0x4u /* backward also stores SplatGrads (SPLATGRAD_* fields) */
#define ODGS_FRAME_COUNT_WORK 0x8u  /* blend and backward count their work (odgs_frame_work,
                                       odgs_frame_backward_work); costs time */

/* odgs_backward flags */
#define ODGS_ACCUMULATE 0x1u /* add into the gradient buffers (GradBuffers::accumulate) */

/* ------------------------------------------------------------------ context */
odgs_settings odgs_default_settings(void);
int odgs_abi_version(void);

/* Creates a context on `device`. stream: a cudaStream_t, or NULL for a private
   non-blocking one. The legacy default stream (handle 0, e.g. torch's default stream)
   must be passed as cudaStreamLegacy ((void*)0x1), since NULL asks for a private stream.
   Kernels are launched with programmatic dependent launch on that stream. */
odgs_status odgs_ctx_create(int device, void* stream, odgs_ctx** out);
void odgs_ctx_destroy(odgs_ctx* ctx);
odgs_status odgs_ctx_set_stream(odgs_ctx* ctx, void* stream);
void* odgs_ctx_stream(odgs_ctx* ctx);
odgs_status odgs_synchronize(odgs_ctx* ctx);
/* Asynchronous mode (enable != 0): odgs_render / odgs_render_band / odgs_prepare_render
   and odgs_backward with device gradient buffers return without synchronising the stream
   — no host round trip inside or between them, so frames and training views queue back
   to back (after a frame's first render, which sizes its buffers). Their errors (the
   reference's exceptions) are reported at the frame's check point: odgs_frame_check, or
   any call that reads the frame on the host (downloads, odgs_frame_get_info,
   odgs_frame_work). Inputs must stay valid until then. Default: synchronous, errors
   returned by the call itself as the reference throws. */
odgs_status odgs_ctx_set_async(odgs_ctx* ctx, int enable);
/* The frame's check point: synchronises, and reports a deferred error of the operations
   enqueued on the frame since the last check. If a render produced more tile entries
   than the frame's entry buffers held (they are sized 1.25x the entries of the frame's
   first render and grow on demand), the frame's last render is re-run synchronously with
   room for them, so the frame holds the correct result; *rerendered (optional) is then
   1, and a backward enqueued on the overflowed render must be repeated. */
odgs_status odgs_frame_check(odgs_ctx* ctx, odgs_frame* frame, int32_t* rerendered);
/* Code of the last failed call on ctx; *gaussian_index = offending row or -1. */
odgs_status odgs_last_error(const odgs_ctx* ctx, int64_t* gaussian_index, char* message, size_t message_len);
/* Number of kernels this context has launched since creation. */
int64_t odgs_ctx_launch_count(const odgs_ctx* ctx);

/* ------------------------------------------------------------------ profiling
   Per-stage CUDA-event timers on the context's stream (the stream every kernel is
   launched on). Enabling adds one event pair per stage per call and a stream
   synchronisation at the end of each profiled call. */
typedef enum {
  ODGS_STAGE_PREPROCESS = 0, /* k_preprocess                       */
  ODGS_STAGE_DEPTH_SORT = 1, /* radix sort of the Gaussians by depth */
  ODGS_STAGE_SCAN = 2,       /* gather counts + exclusive scan     */
  ODGS_STAGE_EMIT = 3,       /* k_emit tile entries                */
  ODGS_STAGE_TILE_SORT = 4,  /* radix sort of the entries by tile  */
  ODGS_STAGE_RANGES = 5,     /* tile CSR offsets                   */
  ODGS_STAGE_BLEND = 6,      /* k_blend                            */
  ODGS_STAGE_BWD_RASTER = 7, /* k_bwd_raster (+ record clear)      */
  ODGS_STAGE_BWD_SPLAT = 8,  /* k_bwd_splat                        */
  ODGS_STAGE_COUNT = 9
} odgs_stage;
odgs_status odgs_ctx_set_profiling(odgs_ctx* ctx, int enable);
/* Accumulated milliseconds and call counts per stage since the last reset; returns
   the number of stages written (<= max_stages). */
int odgs_ctx_stage_times(odgs_ctx* ctx, double* ms, int64_t* calls, int max_stages);
void odgs_ctx_reset_stage_times(odgs_ctx* ctx);
const char* odgs_stage_name(int stage);
/* Measured FP32 FMA throughput of the device (TFLOP/s, 2 flops per FMA). */
odgs_status odgs_measure_fp32_tflops(odgs_ctx* ctx, double* tflops);

/* ------------------------------------------------------------------ frames */
odgs_status odgs_frame_create(odgs_ctx* ctx, odgs_frame** out);
void odgs_frame_destroy(odgs_frame* frame);
odgs_status odgs_frame_set_flags(odgs_frame* frame, uint32_t flags);
odgs_status odgs_frame_get_info(const odgs_frame* frame, odgs_frame_info* info);
/* Copies a field to host memory (bytes must be >= the field's size). Synchronizes. */
odgs_status odgs_frame_download(odgs_ctx* ctx, odgs_frame* frame, int field, void* host_dst, size_t bytes);
/* Blend work of the last render into `frame` (for rooflines): pixel-entry
   evaluations examined (sum over pixels of walked, +1 when the walk stopped early)
   and entries composited; zeros unless the frame has ODGS_FRAME_COUNT_WORK.
   Synchronizes. */
odgs_status odgs_frame_work(odgs_ctx* ctx, odgs_frame* frame, int64_t* entries_examined,
                            int64_t* entries_composited);
/* Backward work of the last odgs_backward / odgs_grad_pixels_to_splats on `frame` (for
   rooflines; zeros unless the frame has ODGS_FRAME_COUNT_WORK), up to n_counters (<= 4) values: [0] entries replayed (sum over pixels with
   a non-zero image gradient of their walk length — the reference's replay loop,
   backward.hpp:251-269), [1] contributions (replayed entries inside the cutoff,
   :271-305), [2] warp-entries walked by the culled kernel (sum of its warps' list
   lengths), [3] warp-entries with at least one contributing pixel. Synchronizes. */
odgs_status odgs_frame_backward_work(odgs_ctx* ctx, odgs_frame* frame, int64_t* counters, int32_t n_counters);
/* Row bands over several GPUs: the blend also writes every pixel it
   renders into each of these n <= 8 image buffers ([3][W][H] float, the frame's
   layout) — typically the other ranks' full-image buffers opened with odgs_ipc_open —
   so a band render all-gathers its rows over NVLink as it produces them. Pointers stay
   in effect for later renders into this frame; n = 0 clears them. Every blend path
   (warp-culled or ODGS_FRAME_PLAIN_BLEND, any tile size) writes them. The caller
   synchronises the ranks before reading. */
odgs_status odgs_frame_set_image_peers(odgs_frame* frame, int32_t n, void* const* peer_images);

/* CUDA IPC (one process per GPU on a node): export device memory, open a peer's. The
   pointer may lie inside a larger allocation (e.g. a caching allocator's block): the
   handle carries the cudaIpcMemHandle_t of the enclosing allocation (64 bytes) and the
   pointer's byte offset in it (8 bytes); odgs_ipc_open returns base + offset, and
   odgs_ipc_close takes that pointer. */
#define ODGS_IPC_HANDLE_BYTES 72
odgs_status odgs_ipc_get_handle(const void* device_ptr, void* handle);
odgs_status odgs_ipc_open(const void* handle, void** device_ptr);
odgs_status odgs_ipc_close(void* device_ptr);

/* Device pointer of a resident field (IMAGE, TRANSMITTANCE, WALKED, TILE_OFFSETS). */
odgs_status odgs_frame_device_ptr(odgs_frame* frame, int field, void** device_ptr);

/* ------------------------------------------------------------------ hot path */
/* prepare_render (rasterizer.hpp:129-207): validate, project, seam-duplicate, sort,
   bin. Returns after the device has finished projection (errors are reported
   synchronously, as the reference throws); the rest is enqueued on the stream. */
odgs_status odgs_prepare_render(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                                const odgs_settings* settings, odgs_frame* frame);

/* render (rasterizer.hpp:211-267): prepare_render + front-to-back tile blending. */
odgs_status odgs_render(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                        const odgs_settings* settings, odgs_frame* frame);

/* A row band of a render (large renders split over GPUs): identical to
   render() on pixel rows [row_begin, row_end) — bit for bit, since per-tile lists depend
   only on the global (depth, index, shift) order — while only tiles of those rows get
   entries and are blended. Rows must lie on tile boundaries (row_end may be the image
   height). Other rows of the frame's image/transmittance/walked are undefined. A
   backward on a band frame returns that band's share of the gradient (bands add). */
odgs_status odgs_render_band(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                             const odgs_settings* settings, int32_t row_begin, int32_t row_end, odgs_frame* frame);

/* The rasterization half of render (rasterizer.hpp:141-267) on caller-supplied
   projected splats — the Splat2D records of RenderOutput::splats (projection.hpp:163-174)
   of a cloud of n_gaussians rows — instead of projecting a cloud: seam instances, the
   (depth, index, shift) order, tile CSR and the front-to-back blend, exactly as render()
   continues after project_gaussian. Host arrays, one row per splat in ascending cloud
   index: pixel_mean [ns][2], cov2d_inv [ns][4] row-major ((0,1) is used, as the
   reference's d2), depth, radius, opacity [ns], color [ns][3]. Lets a caller (or a test)
   feed splats projected elsewhere — e.g. by the libm reference — to the GPU stages.
   Synchronizes. ODGS_ERR_INVALID_ARGUMENT (index = splat row) for unsorted or
   out-of-range indices, non-finite values, negative depth or radius. */
odgs_status odgs_rasterize_splats(odgs_ctx* ctx, int64_t n_gaussians, int64_t n_splats, const int64_t* index,
                                  const float* pixel_mean, const float* cov2d_inv, const float* depth,
                                  const float* radius, const float* opacity, const float* color, int32_t width,
                                  int32_t height, const odgs_settings* settings, odgs_frame* frame);

/* Splat2D (projection.hpp:163-174). */
typedef struct {
  float pixel_mean[2];
  float cov2d[4];     /* row-major, incl. the low-pass dilation */
  float cov2d_inv[4]; /* row-major */
  float depth, radius, opacity;
  float color[3];
  int64_t index;
  int32_t pole_clamped;
} odgs_splat;

/* project_gaussian (projection.hpp:178-216) of cloud row `index`: *projected = 0 for
   std::nullopt (outside the near/far shell, or a non-positive / non-finite projected
   covariance), else *out holds the splat. No first_non_finite pass, as in the reference:
   ODGS_ERR_INVALID_ARGUMENT for a near-zero quaternion or a non-finite quaternion /
   log-scale inside the shell (covariance.hpp:14-15, 31-32), ODGS_ERR_DOMAIN for a
   zero-length direction. Synchronizes. */
odgs_status odgs_project_gaussian(odgs_ctx* ctx, const odgs_cloud* cloud, int64_t index, const odgs_camera* camera,
                                  const odgs_settings* settings, odgs_splat* out, int32_t* projected);

/* grad_pixels_to_splats (backward.hpp:208-339): SplatGrads of every projected splat of a
   rendered frame, in RenderOutput::splats order (n_splats rows; host arrays, any may be
   NULL): pixel_mean [ns][2], cov2d [ns][4] (full-matrix convention), opacity [ns] (w.r.t.
   the activated opacity), color [ns][3]. The alpha clamp and cutoff are read from
   `settings`. Synchronizes. */
odgs_status odgs_grad_pixels_to_splats(odgs_ctx* ctx, odgs_frame* frame, const float* dl_dimage, int32_t dl_memory,
                                       const odgs_settings* settings, float* pixel_mean, float* cov2d, float* opacity,
                                       float* color);

/* backward (backward.hpp:380-448) incl. grad_pixels_to_splats (:208-339) for the view
   rendered into `frame` (same cloud, camera, settings — unchecked, as in the
   reference). dl_dimage: [3][W][H] in dl_memory. grad_t_signs: NULL or 12 signs
   (GradTSigns, backward.hpp:32-34). flags: ODGS_ACCUMULATE. */
odgs_status odgs_backward(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera, odgs_frame* frame,
                          const float* dl_dimage, int32_t dl_memory, const odgs_settings* settings,
                          const odgs_grads* grads, const double* grad_t_signs, uint32_t flags);

/* ------------------------------------------------------------------ training step
   (all pointers are device memory) */

/* The optimisable parameters (GaussianCloud<float> with writable device arrays). */
typedef struct {
  int64_t n;
  float* means;
  float* rotations;
  float* log_scales;
  float* raw_opacities;
  float* colors;
} odgs_params;

/* TrainState (types.hpp:257-325): Adam moments per group and the densify window. */
typedef struct {
  float *means_m, *means_v, *rot_m, *rot_v, *scale_m, *scale_v, *opac_m, *opac_v, *color_m, *color_v;
  float* grad_accum;
  float* elev_accum;
  int32_t* grad_count;
} odgs_train_state;

/* Learning rates of this step (means: means_lr_at(iteration) * extent,
   optimizer.hpp:61-69) and the 1-based Adam step. */
typedef struct {
  float lr_means, lr_rotation, lr_scale, lr_opacity, lr_color;
  int64_t step;
} odgs_adam_params;

/* photometric_loss (metrics.hpp:152-184): (1 - lambda) L1 + lambda (1 - SSIM) with the
   11x11 Gaussian window (sigma 1.5) of ssim_with_gradient (metrics.hpp:83-136); writes
   the image gradient to dl_dimage and the loss to *loss (synchronizes). Images are
   [3][W][H] device buffers; lambda in [0, 1); SSIM needs W, H >= 11. */
odgs_status odgs_photometric_loss(odgs_ctx* ctx, const float* rendered, const float* target, int32_t width,
                                  int32_t height, float lambda_ssim, float* dl_dimage, double* loss);

/* As odgs_photometric_loss, without a host readback: the loss is added to
   *device_loss_sum (a device double, may be NULL) on the context's stream, so a training
   step can read its summed loss once. Does not synchronize. */
odgs_status odgs_photometric_loss_async(odgs_ctx* ctx, const float* rendered, const float* target, int32_t width,
                                        int32_t height, float lambda_ssim, float* dl_dimage, double* device_loss_sum);

/* The update half of train_step (optimizer.hpp:114-139): densify-window
   accumulation, Adam (b1 0.9, b2 0.999, eps 1e-15) on the five groups, quaternion
   renormalisation. grads must be device buffers (e.g. after an all-reduce). */
odgs_status odgs_adam_step(odgs_ctx* ctx, const odgs_params* params, const odgs_grads* grads,
                           const odgs_train_state* state, const odgs_adam_params* adam);

/* ------------------------------------------------------------------ density control
   (densify.hpp) */

/* DensifyConfig (densify.hpp:16-33): the fields densify_and_prune reads. */
typedef struct {
  double grad_threshold_min;  /* 2e-5, trigger at the equator */
  double grad_threshold_max;  /* 1e-4, trigger at the poles */
  double percent_dense;       /* 1e-3 of the scene extent: clone / split boundary */
  double opacity_prune_floor; /* 0.005 */
  double split_scale_divisor; /* 1.6 */
} odgs_densify_config;

void odgs_default_densify_config(odgs_densify_config* out);

/* DensifyStats (densify.hpp:51-55) plus the row count after the round. */
typedef struct {
  int64_t cloned, split, pruned, n_out;
} odgs_densify_stats;

/* std::mt19937 owned by the library: the generator densify_and_prune draws split
   offsets from (densify.hpp:85, :61-69). Host object. */
typedef struct odgs_rng odgs_rng;
odgs_rng* odgs_rng_create(uint32_t seed);
void odgs_rng_destroy(odgs_rng* rng);
/* The generator's next raw 32-bit output (advances it). */
uint32_t odgs_rng_next(odgs_rng* rng);
/* count samples of detail::unit_ball_normal<float> (densify.hpp:61-69), the exact
   draw sequence of the reference: out[3k..3k+2] = (x, y, z) of the k-th sample. */
void odgs_rng_unit_ball(odgs_rng* rng, int64_t count, float* out);

/* densify_and_prune (densify.hpp:81-153), first half: validates cfg and the extent,
   classifies every Gaussian on the device (clone / split / prune) and computes the
   output positions; stats receives the counts and n_out (synchronizes). The plan
   stays in the context until the next odgs_densify_plan. Errors as the reference:
   ODGS_ERR_INVALID_ARGUMENT for a bad config / extent, or for a split parent with a
   near-zero quaternion (index = that Gaussian). */
odgs_status odgs_densify_plan(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                              const odgs_densify_config* cfg, float scene_extent, odgs_densify_stats* stats);

/* Second half: writes the densified cloud and train state (n_out rows, device
   buffers that must not overlap the inputs): surviving rows in order, then the
   surviving clones / split children in parent order; moments follow their rows (new
   rows zero), the densify window is cleared. unit_ball: host array of 2 * split
   samples (odgs_rng_unit_ball, or the caller's own generator), child order. The
   inputs must be the ones passed to odgs_densify_plan. */
odgs_status odgs_densify_apply(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                               const float* unit_ball, const odgs_params* out_cloud,
                               const odgs_train_state* out_state);

/* reset_opacity (densify.hpp:158-166): raw <- logit(min(sigmoid(raw), ceiling)) and
   zeroes the opacity moments. If some row's logit argument leaves (0, 1) the rows
   before it are rewritten, the moments are left alone, and ODGS_ERR_INVALID_ARGUMENT
   names that row — the reference's throw point. */
odgs_status odgs_reset_opacity(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                               float ceiling);

/* dynamic_threshold (densify.hpp:39-49), binary64 host helper. */
odgs_status odgs_dynamic_threshold(double elevation, const odgs_densify_config* cfg, double* out);

/* ------------------------------------------------------------------ scene I/O
   (reference io.hpp / src/io.cpp). Host code: polygon (.ply)
   point clouds and checkpoints in the reference's exact formats. Every array is the
   reference's Eigen column-major storage in binary64 (GaussianCloud<double>,
   PointCloud): positions/means/colors [3][n], rotations (w,x,y,z) [4][n], log_scales
   [3][n], raw_opacities [n]. Failures return ODGS_ERR_RUNTIME (std::runtime_error in
   the reference) with the reference's message ("<path>: <what> (byte N)"), read with
   odgs_io_last_error() (per host thread). */

/* GaussianCloud<double> (types.hpp:53-143), host or device arrays. */
typedef struct {
  int64_t n;
  double* means;
  double* rotations;
  double* log_scales;
  double* raw_opacities;
  double* colors;
} odgs_cloud64;

/* Message of the last failed odgs_ply / checkpoint call on this thread. */
size_t odgs_io_last_error(char* message, size_t message_len);
/* Vertex count declared by a polygon file's header (parse_ply_header, io.cpp:41-118). */
odgs_status odgs_ply_vertex_count(const char* path, int64_t* n);
/* load_pointcloud (io.cpp:203-223): needs x, y, z, red, green, blue; uchar colours
   are scaled by 1/255. n must be the file's vertex count (odgs_ply_vertex_count). */
odgs_status odgs_load_pointcloud(const char* path, int64_t n, double* positions, double* colors);
/* save_pointcloud (io.cpp:225-257): float positions, uchar colours (round(clamp*255)). */
odgs_status odgs_save_pointcloud(const char* path, int64_t n, const double* positions, const double* colors,
                                 int32_t binary);
/* save_checkpoint (io.cpp:299-332): float32 x,y,z, f_dc_0..2 (= (c - 0.5) / C0, flushed
   below 2^-27), opacity, scale_0..2, rot_0..3, with the version comment. */
odgs_status odgs_save_checkpoint(const char* path, const odgs_cloud64* cloud);
/* load_checkpoint (io.cpp:334-362): rejects newer versions and missing properties.
   cloud->n must be the file's vertex count; all five arrays are written. */
odgs_status odgs_load_checkpoint(const char* path, const odgs_cloud64* cloud);

/* init_from_points (io.cpp:259-297) on the GPU: means = positions, colours copied,
   identity rotations, raw opacity logit(0.1), isotropic log-scale = log of the mean
   distance to the (up to) three nearest neighbours, floored at 1e-7 (0.1 for a point
   with no finite neighbour distance). Exact 3-NN through a uniform grid: the mean
   distances equal the reference's brute force bit for bit (nn_scale, optional [n],
   receives them before the log). positions/colors and every output array live in
   `memory`. Errors: ODGS_ERR_INVALID_ARGUMENT for n < 1 ("init_from_points: no
   points"). */
odgs_status odgs_init_from_points(odgs_ctx* ctx, int64_t n, const double* positions, const double* colors,
                                  int32_t memory, const odgs_cloud64* out, double* nn_scale);

/* cull (rasterizer.hpp:15-28): host output of the kept rows, ascending. */
odgs_status odgs_cull(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera, float near_radius,
                      float far_radius, int64_t* out_indices, int64_t* out_count);

#ifdef __cplusplus
}
#endif

#endif /* ODGS_B200_H */
