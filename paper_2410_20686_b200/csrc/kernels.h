// kernels.h — host-side launch interface of the device kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace odgs_b200 {

// Every launch_* below increments this counter once per kernel it launches, so the
// host can report how many of its own kernels ran (bench.py "gpu_launches").
extern thread_local int64_t g_launches;

struct PreprocessArgs {
  int64_t n;
  const float *means, *rotations, *log_scales, *raw_opacities, *colors;
  int sh_degree;
  const float* sh_rest;  // [(deg+1)^2-1][3][n] or null
  DevCamera cam;
  DevSettings settings;
  float4* sp_ab;   // [2n] {mx,my,i00,i01},{i11,opacity,r,g}
  float4* sp_c;    // [n] {b, depth, radius, flags}
  float4* cov_out; // [n] or null
  uint32_t* keys;  // [n] depth bits or kCulledKey
  uint32_t* vals;  // [n] iota
  uint32_t* cnt;   // [n] tile entries of the Gaussian
  DevErrors* err;
};
void launch_preprocess(const PreprocessArgs& a, cudaStream_t stream);
// Fused band path: pre-cull + exact preprocess of the survivors + compaction of the
// Gaussians with band entries into per-warp segments (segment w at w * chunk,
// seg_count[w] pairs; band_segments(n) segments).
int64_t band_segments(int64_t n);
void launch_band_preprocess(const PreprocessArgs& a, uint32_t* seg_keys, uint32_t* seg_vals, uint32_t* seg_count,
                            cudaStream_t stream);
// Concatenates the segments at seg_off (exclusive scan of seg_count).
void launch_concat_segments(int64_t n, const uint32_t* seg_count, const uint32_t* seg_off, const uint32_t* seg_keys,
                            const uint32_t* seg_vals, uint32_t* keys_out, uint32_t* vals_out, cudaStream_t stream);
// project_gaussian (projection.hpp:178-216) of a row gathered into a one-row cloud
// (means 3 | rotations 4 | log_scales 3 | raw opacity | colors 3 | sh_rest 3 nb).
void launch_project_one(const float* row, int sh_degree, const DevCamera& cam, const DevSettings& s, float4* sp_ab,
                        float4* sp_c, float4* cov, uint32_t* keys, uint32_t* vals, uint32_t* cnt, DevErrors* err,
                        cudaStream_t stream);
// Caller-supplied splats (odgs_rasterize_splats): kSplatRecord floats per splat, the
// first holding the cloud row's bits; rows without a splat are culled.
constexpr int kSplatRecord = 12;
void launch_load_splats(int64_t n, int64_t n_splats, const float* rec, int width, int height, int tile_size,
                        float4* sp_ab, float4* sp_c, uint32_t* keys, uint32_t* vals, uint32_t* cnt, DevErrors* err,
                        cudaStream_t stream);
struct EmitArgs {
  int64_t n;
  const uint32_t *sorted_idx, *cnt_sorted, *off_sorted;
  const float4 *sp_ab, *sp_c;
  int width, height, tile_size, tiles_x, band_ty0, band_ty1;
  uint32_t *out_keys, *out_vals, *ent_off_idx;
  const uint32_t* n_dev;            // device-side rank count (<= n) or null
  const unsigned long long* total;  // total tile entries (the offsets scan's total)
  uint32_t capacity;                // entries the output buffers hold
  unsigned long long* k_sort;       // <- min(total, capacity) (or null)
  unsigned long long* overflow;     // <- total when it exceeds the capacity
};
void launch_emit(const EmitArgs& a, cudaStream_t stream);

// Stream-ordered resets as kernels (they join the programmatic-launch chain; a memcpy or
// memset node would break it): the per-render counters (and, unless keep_sticky, the
// sticky error words) to their initial values; `bytes` zero bytes at a cudaMalloc base.
void launch_reset_errors(DevErrors* e, bool keep_sticky, cudaStream_t stream);
void launch_reset_sticky(DevErrors* e, cudaStream_t stream);  // the sticky words only
void launch_zero_bytes(void* p, size_t bytes, cudaStream_t stream);

void launch_cull(int64_t n, const float* means, DevCamera cam, float near_r, float far_r, uint8_t* keep,
                 cudaStream_t stream);

// Tile CSR offsets [n_tiles + 1]; entries lie in tiles [t0, t1) (a row band), t1 <= n_tiles.
void launch_tile_ranges(uint32_t k_entries, const uint32_t* keys, uint32_t n_tiles, uint32_t t0, uint32_t t1,
                        int32_t* offsets, cudaStream_t stream, const uint32_t* k_dev = nullptr);

// Peer image buffers ([3][W][H], the frame's layout) that the blend epilogue also writes
// its pixels to: an all-gather of row bands fused into the kernel that produces them
// (stores over NVLink to other GPUs' memory, opened with CUDA IPC).
constexpr int kMaxPeers = 8;
struct PeerImages {
  float* ptr[kMaxPeers];
  int n;
};

struct BlendArgs {
  const int32_t* offsets;
  const uint32_t* vals;
  const float4 *sp_ab, *sp_c;
  int width, height, tile_size, tiles_x, tiles_y, band_ty0, band_ty1;
  float alpha_clamp, transmittance_floor, cutoff_sigma;
  float* image;
  float* transmittance;
  int32_t* walked;
  unsigned long long* work;  // [2] += entries examined, entries composited (or null)
  const uint32_t* order;     // launch order of the band's tiles (launch_tile_order) or null
  PeerImages peers;          // also write the image to these buffers (n = 0: none)
  bool plain;                // force the un-culled reference kernel (A/B checks)
};
// order[k] = band-relative tile index of the k-th CTA: tiles by descending list length.
void launch_tile_order(const int32_t* offsets, int tile_base, int n, uint32_t* order, cudaStream_t stream);
void launch_blend(const BlendArgs& a, cudaStream_t stream);
void launch_blend_plain(const BlendArgs& a, cudaStream_t stream);

// ------------------------------------------------------------------ sort / scan
// Scratch needed by exclusive_scan_u32 for n items.
size_t scan_temp_bytes(int64_t n);
// out[k] = sum_{j<k} in[k]; optionally atomically adds the 64-bit total to *total64.
// n_dev: optional device-side item count <= n (the launch is sized for n).
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* temp, unsigned long long* total64,
                        cudaStream_t stream, const uint32_t* n_dev = nullptr);

// Sorts hold fewer than 2^30 items: the onesweep look-back words carry 30-bit counts.
constexpr unsigned long long kMaxSortItems = 1ull << 30;

size_t radix_sort_temp_bytes(int64_t n);
// Stable LSD radix sort of (key, value) pairs on key bits [begin_bit, end_bit).
// keys/vals: [2] ping-pong buffers of n each; on return *which (0/1) holds the result.
// Optional payload gather: gather_dst[r] = gather_src[sorted value r], written by the
// last pass (saves a separate gather over the sorted values).
// Returns the first failed launch's error (the remaining passes are then not launched:
// they would look back over status words nobody cleared). n_dev: optional device-side
// item count <= n; the kernels are then launched for n (the capacity) and read the count
// on the device, so no host synchronisation is needed to learn it.
cudaError_t radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t n, int begin_bit, int end_bit,
                             void* temp, int* which, cudaStream_t stream, const uint32_t* gather_src = nullptr,
                             uint32_t* gather_dst = nullptr, const uint32_t* n_dev = nullptr);

// ------------------------------------------------------------------ training step
size_t l1_loss_temp_bytes(int64_t count);
// temp[0] <- loss (double), *accum += loss (if accum); grad <- (1 - lambda)
// sign(rendered - target) / count.
void launch_l1_loss(const float* rendered, const float* target, int64_t count, float lambda, float* grad,
                    double* temp, double* accum, cudaStream_t stream);

size_t ssim_temp_bytes(int H, int W);
// photometric_loss with lambda > 0 (metrics.hpp:152-184): image gradient and *loss_out.
void launch_ssim_loss(const float* a, const float* b, int H, int W, float lambda, float* grad, void* temp,
                      double* loss_out, double* accum, cudaStream_t stream);

struct AdamArgs {
  int64_t n;
  float *means, *rotations, *log_scales, *raw_opacities, *colors;
  float *means_m, *means_v, *rot_m, *rot_v, *scale_m, *scale_v, *opac_m, *opac_v, *color_m, *color_v;
  float *grad_accum, *elev_accum;
  int32_t* grad_count;
  const float *g_means, *g_rotations, *g_log_scales, *g_raw_opacities, *g_colors, *g_pixel_grad_norm,
      *g_one_minus_cos;
  const int32_t* g_observed;
  float lr_means, lr_rotation, lr_scale, lr_opacity, lr_color, c1, c2;
};
void launch_adam(const AdamArgs& a, cudaStream_t stream);

// ------------------------------------------------------------------ densify (densify.hpp)
// Adam moment groups in TrainState order (types.hpp:257-268): means_m/v, rot_m/v,
// scale_m/v, opac_m/v, color_m/v.
__host__ __device__ constexpr int moment_width(int k) { return (k == 2 || k == 3) ? 4 : (k == 6 || k == 7) ? 1 : 3; }

struct DensifyArgs {
  int64_t n;
  const float *rotations, *log_scales, *raw_opacities;
  const float *grad_accum, *elev_accum;
  const int32_t* grad_count;
  float tmin, tmax, size_split, prune_floor;
  uint32_t *keep_self, *added_kept, *split_flag;  // [n] each
  unsigned long long* counters;                   // [3] cloned, split, pruned
  unsigned long long* bad_quaternion;             // first split parent with |q| <= 1e-12
};
void launch_densify_classify(const DensifyArgs& a, cudaStream_t stream);

struct DensifyApplyArgs {
  int64_t n, m;  // rows in, rows out
  const float *means, *rotations, *log_scales, *raw_opacities, *colors;
  const float* moments[10];
  float *out_means, *out_rotations, *out_log_scales, *out_raw_opacities, *out_colors;
  float* out_moments[10];
  const uint32_t *keep_self, *added_kept, *split_flag, *off_a, *off_b, *off_c;
  uint32_t total_a;
  const float* unit_ball;  // [split][child][3]
  float log_shrink;        // log(split_scale_divisor) in float
};
void launch_densify_apply(const DensifyApplyArgs& a, cudaStream_t stream);

// reset_opacity (densify.hpp:158-166); *bad must hold kNoError on entry.
void launch_reset_opacity(float* raw, int64_t n, float ceiling, unsigned long long* bad, cudaStream_t stream);

// FP32 FMA throughput microbenchmark (for the roofline denominator).
void launch_fp32_peak(int blocks, int threads, int iters, float* sink, cudaStream_t stream);
double fp32_peak_flops_per_thread(int iters);

// ------------------------------------------------------------------ backward
struct BwdRasterArgs {
  const int32_t* offsets;
  const uint32_t* vals;
  const float4 *sp_ab, *sp_c;
  const uint32_t* ent_off_idx;
  const float* transmittance;
  const int32_t* walked;
  const float* dl_dimage;
  int width, height, tile_size, tiles_x, tiles_y, band_ty0, band_ty1;
  float alpha_clamp, cutoff_sigma;
  float* records;    // [K][12] per tile entry (9 sums + pad), at the entry's emit position
  uint8_t* touched;  // [K] 1 where a record was written (cleared before the launch)
  const uint32_t* order;  // launch order of the band's tiles or null
  bool plain;        // un-culled reference kernel (A/B checks)
  unsigned long long* work;  // [2] += entries replayed, contributions (or null)
};
void launch_bwd_raster(const BwdRasterArgs& a, cudaStream_t stream);

// Ordered per-Gaussian fold of the entry records (backward.hpp:310-327), one thread per
// depth rank so a warp reads one contiguous record range: folded[g][9] for every
// Gaussian with entries.
// k_limit (capacity path): records at emit positions >= *k_limit were not written.
void launch_fold_records(int64_t n, const uint32_t* sorted_idx, const uint32_t* cnt_sorted,
                         const uint32_t* off_sorted, const uint8_t* touched, const float* records, float* folded,
                         cudaStream_t stream, const uint32_t* n_dev = nullptr,
                         const unsigned long long* k_limit = nullptr);

// SplatGrads of every projected Gaussian from the folded records (grad_pixels_to_splats).
void launch_splat_grads(int64_t n, const float4* sp_ab, const float4* sp_c, const uint32_t* cnt, const float* folded,
                        float* splat_grads, cudaStream_t stream);

struct BwdSplatArgs {
  int64_t n;
  const float *means, *rotations, *log_scales, *raw_opacities;
  int sh_degree;
  const float* sh_rest;
  float* g_sh_rest;
  DevCamera cam;
  DevSettings settings;
  const float4 *sp_ab, *sp_c;
  const uint32_t* cnt;
  const float* folded;  // [n][9] folded records (launch_fold_records), read where cnt > 0
  const float* signs;  // [12] GradTSigns
  float sec_max;       // 1 / cos(max_elevation): the clamped Jacobian's secant
  int accumulate;
  float *g_means, *g_rotations, *g_log_scales, *g_raw_opacities, *g_colors, *g_pixel_grad_norm, *g_one_minus_cos;
  int32_t* g_observed;
  float* splat_grads;  // [n][10] SplatGrads per Gaussian (mean2, cov4, opacity, color3) or null
  DevErrors* err;
};
void launch_bwd_splat(const BwdSplatArgs& a, cudaStream_t stream);

// ------------------------------------------------------------------ init_from_points (io.cpp:259-297)
// Uniform grid over the finite points' bounding box: cell (x, y, z) of point p is
// floor((p - lo) / h) clamped to [0, dims); id = (z * dims[1] + y) * dims[0] + x.
struct KnnGrid {
  double lo[3];
  double h;
  int dims[3];
  uint32_t n_cells;
};
void launch_fill_f64(double* p, int64_t n, double v, cudaStream_t stream);
// partial[b][6] = (min xyz, max xyz) of block b's finite points; *n_finite += count.
void launch_bbox_partial(int64_t n, const double* pos, double* partial, int blocks, unsigned long long* n_finite,
                         cudaStream_t stream);
void launch_cell_keys(int64_t n, const double* pos, const KnnGrid& g, uint32_t* keys, uint32_t* idx,
                      cudaStream_t stream);
void launch_gather_xyz(int64_t n, const uint32_t* idx, const double* pos, double* sorted, cudaStream_t stream);
void launch_cell_ranges(int64_t m, const uint32_t* keys, uint32_t n_cells, uint32_t* cell_start,
                        cudaStream_t stream);
// n points, the first m (in cell order) finite; writes scale_out[i] (optional) and
// log_scales[3][n] (isotropic) per original index.
void launch_knn_query(int64_t n, int64_t m, const double* xyz, const uint32_t* idx, const uint32_t* cell_start,
                      const KnnGrid& g, double* scale_out, double* log_scales, cudaStream_t stream);

}  // namespace odgs_b200
