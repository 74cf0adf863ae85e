// capi.cu — the C ABI (include/odgs_b200.h): contexts, frames, and the host-side
// orchestration of the forward and backward kernels on one CUDA stream.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <random>
#include <string>
#include <vector>

#include <cuda.h>

#include "kernels.h"
#include "odgs_b200.h"

using namespace odgs_b200;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct StageTimers {
  bool enabled = false;
  struct Pending { int stage; cudaEvent_t start, stop; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  double ms[ODGS_STAGE_COUNT] = {};
  int64_t calls[ODGS_STAGE_COUNT] = {};
};

struct odgs_ctx {
  int device = 0;
  StageTimers timers;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  odgs_status last_code = ODGS_OK;
  int64_t last_index = -1;
  std::string last_msg;
  DevErrors* d_err = nullptr;
  DevErrors* h_err = nullptr;       // pinned readback
  DevErrors* h_err_init = nullptr;  // pinned reset template
  uint32_t* h_scratch = nullptr;    // pinned
  DevBuf cloud_buf, dl_buf, grads_buf, signs_buf, cull_buf, loss_buf;
  float* d_unit_signs = nullptr;
  int64_t launches = 0;
  bool async_mode = false;  // odgs_ctx_set_async: renders / backward passes return without synchronising
  // densify_and_prune plan (odgs_densify_plan -> odgs_densify_apply)
  DevBuf densify_buf, unit_ball_buf, misc_buf;
  struct {
    bool valid = false;
    int64_t n = 0, split = 0, n_out = 0;
    const float* key = nullptr;  // cloud->means of the planned cloud
    uint32_t total_a = 0;
    float log_shrink = 0.0f;
  } plan;
};

struct odgs_frame {
  odgs_ctx* ctx = nullptr;
  uint32_t flags = 0;
  int width = 0, height = 0, tile_size = 16, tiles_x = 0, tiles_y = 0;
  int64_t n = 0;
  uint32_t n_entries = 0;
  int64_t n_splats = 0, n_instances = 0;
  int32_t row_begin = 0, row_end = 0;
  bool prepared = false, rendered = false, have_splat_grads = false;
  bool from_splats = false;  // odgs_rasterize_splats: no cloud or camera behind the splats
  bool band = false;         // a row-band render (compacted depth sort)
  DevBuf sp_ab, sp_c, cov, keys[2], vals[2], cnt, cnt_sorted, off_sorted, ent_off_idx, sort_tmp, scan_tmp;
  DevBuf ekeys[2], evals[2], offsets, tile_order, image, trans, walked, records, touched, folded, splat_grads, work;
  DevBuf bwd_work;  // [4] backward work counters of the last backward
  // Per-frame device error words and their pinned host copy: several frames can be in
  // flight on one context (asynchronous renders), each checked at its own sync point.
  DevErrors* d_err = nullptr;
  DevErrors* h_err = nullptr;
  // Capacity of the tile-entry buffers (entries). 0: unknown — the next render learns the
  // entry count with a host synchronisation after the offsets scan (the "exact" path);
  // afterwards renders run without any synchronisation, with the entry count kept on the
  // device, and an overflow (more entries than the capacity) is detected at the frame's
  // check point and re-rendered with room for them.
  uint32_t k_cap = 0;
  bool pending = false;      // enqueued work whose error words / counts are not read yet
  bool cap_path = false;     // the last render ran on the capacity path (entry count on the device)
  bool bwd_pending = false;  // a backward whose error words are not read yet
  // The last render request, for the re-run after an overflow (pointers are the caller's).
  struct Request {
    int kind = 0;  // 0 none, 1 render, 2 prepare, 3 band
    odgs_cloud cloud{};
    odgs_camera camera{};
    odgs_settings settings{};
    int32_t row_begin = 0, row_end = 0;
  } req;
  int depth_which = 0, tile_which = 0;
  bool work_counted = false;      // the last blend counted its work (ODGS_FRAME_COUNT_WORK)
  bool bwd_work_counted = false;  // the last backward did
  int64_t n_sorted = 0;  // depth-sorted ranks: n, or the band's Gaussians (band compaction)
  PeerImages peers{};    // odgs_frame_set_image_peers
  DevCamera cam{};
  DevSettings settings{};
};

namespace {

struct LaunchScope {
  odgs_ctx* ctx;
  int64_t start;
  explicit LaunchScope(odgs_ctx* c) : ctx(c), start(g_launches) {}
  ~LaunchScope() {
    if (ctx) ctx->launches += g_launches - start;
  }
};

odgs_status set_error(odgs_ctx* ctx, odgs_status code, int64_t index, const std::string& msg) {
  if (ctx) {
    ctx->last_code = code;
    ctx->last_index = index;
    ctx->last_msg = msg;
  }
  return code;
}

odgs_status ok(odgs_ctx* ctx) {
  if (ctx) {
    ctx->last_code = ODGS_OK;
    ctx->last_index = -1;
    ctx->last_msg.clear();
  }
  return ODGS_OK;
}

cudaEvent_t pool_event(StageTimers& t) {
  if (!t.pool.empty()) {
    cudaEvent_t e = t.pool.back();
    t.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// RAII stage timer: records an event pair around the enclosed launches.
struct StageScope {
  odgs_ctx* ctx;
  int stage;
  cudaEvent_t start = nullptr;
  StageScope(odgs_ctx* c, int s) : ctx(c), stage(s) {
    if (ctx->timers.enabled) {
      start = pool_event(ctx->timers);
      cudaEventRecord(start, ctx->stream);
    }
  }
  ~StageScope() {
    if (start) {
      cudaEvent_t stop = pool_event(ctx->timers);
      cudaEventRecord(stop, ctx->stream);
      ctx->timers.pending.push_back({stage, start, stop});
    }
  }
};

void resolve_timers(odgs_ctx* ctx) {
  StageTimers& t = ctx->timers;
  for (auto& p : t.pending) {
    cudaEventSynchronize(p.stop);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, p.start, p.stop);
    t.ms[p.stage] += ms;
    t.calls[p.stage] += 1;
    t.pool.push_back(p.start);
    t.pool.push_back(p.stop);
  }
  t.pending.clear();
}

odgs_status cuda_fail(odgs_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, e == cudaErrorMemoryAllocation ? ODGS_ERR_OUT_OF_MEMORY : ODGS_ERR_CUDA, -1,
                   std::string(where) + ": " + cudaGetErrorString(e));
}

#define ODGS_CUDA(ctx, expr)                                  \
  do {                                                        \
    cudaError_t e_ = (expr);                                  \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #expr);  \
  } while (0)

cudaError_t ensure(DevBuf& b, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return cudaSuccess;
  if (b.p) {
    cudaError_t e = cudaFreeAsync(b.p, s);
    if (e != cudaSuccess) return e;
    b.p = nullptr;
    b.cap = 0;
  }
  const size_t nb = ((bytes + bytes / 4) + 255) / 256 * 256;
  cudaError_t e = cudaMallocAsync(&b.p, nb, s);
  if (e != cudaSuccess) return e;
  b.cap = nb;
  return cudaSuccess;
}

void release(DevBuf& b, cudaStream_t s) {
  if (b.p) cudaFreeAsync(b.p, s);
  b.p = nullptr;
  b.cap = 0;
}

int bits_for(uint32_t n_tiles) {
  int b = 0;
  while (b < 32 && (1ull << b) < (unsigned long long)n_tiles) ++b;
  return b;
}

// Host-side argument checks that the reference performs before any work.
odgs_status check_settings(odgs_ctx* ctx, const odgs_settings* s) {
  if (!s) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "settings: null");
  if (s->tile_size <= 0)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "RenderSettings: tile_size must be positive");
  if (s->tile_size > 1024)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "RenderSettings: tile_size > 1024 is not supported");
  return ODGS_OK;
}

// CameraPose::validate (types.hpp:159-169), evaluated in float like the reference.
odgs_status check_camera(odgs_ctx* ctx, const odgs_camera* c) {
  if (!c) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "camera: null");
  if (c->width <= 0 || c->height <= 0 || c->width != 2 * c->height)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1,
                     "CameraPose: equirectangular image needs width == 2 * height > 0");
  float err = 0.0f;
  const float* R = c->rotation;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) {
      const float v = sum3(R[3 * r] * R[3 * k], R[3 * r + 1] * R[3 * k + 1], R[3 * r + 2] * R[3 * k + 2]);
      err = std::max(err, std::fabs(v - (r == k ? 1.0f : 0.0f)));
    }
  if (!(err < 1e-5f)) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "CameraPose: rotation is not orthonormal");
  if ((int64_t)c->width * c->height > (int64_t)1 << 31)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "CameraPose: image too large");
  return ODGS_OK;
}

DevCamera to_dev(const odgs_camera& c) {
  DevCamera d;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) d.R[r][k] = c.rotation[3 * r + k];
  for (int k = 0; k < 3; ++k) d.t[k] = c.translation[k];
  d.width = c.width;
  d.height = c.height;
  return d;
}

DevSettings to_dev(const odgs_settings& s) {
  DevSettings d;
  d.near_radius = s.near_radius;
  d.far_radius = s.far_radius;
  d.tile_size = s.tile_size;
  d.alpha_clamp = s.alpha_clamp;
  d.transmittance_floor = s.transmittance_floor;
  d.cutoff_sigma = s.cutoff_sigma;
  d.lowpass_dilation = s.lowpass_dilation;
  d.max_elevation = s.max_elevation;
  d.band_ty0 = 0;
  d.band_ty1 = 1 << 30;
  return d;
}

// Resolves the cloud to device pointers, copying host arrays into the context.
struct CloudPtrs {
  const float *means, *rotations, *log_scales, *raw_opacities, *colors;
  int sh_degree;
  const float* sh_rest;
};

odgs_status resolve_cloud(odgs_ctx* ctx, const odgs_cloud* c, CloudPtrs* out) {
  if (!c) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "cloud: null");
  if (c->n < 0 || c->n >= ((int64_t)1 << 30))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "cloud: size must be in [0, 2^30)");
  if (c->sh_degree < 0 || c->sh_degree > 3 || (c->sh_degree > 0 && !c->sh_rest))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "cloud: sh_degree must be 0..3 with sh_rest given");
  const int nb = c->sh_degree > 0 ? sh_count(c->sh_degree) : 0;
  if (c->memory == ODGS_MEM_DEVICE || c->n == 0) {
    *out = {c->means, c->rotations, c->log_scales, c->raw_opacities, c->colors, c->sh_degree, c->sh_rest};
    return ODGS_OK;
  }
  const int64_t n = c->n;
  ODGS_CUDA(ctx, ensure(ctx->cloud_buf, sizeof(float) * (14 + 3 * nb) * n, ctx->stream));
  float* b = ctx->cloud_buf.as<float>();
  float* dst[6] = {b, b + 3 * n, b + 7 * n, b + 10 * n, b + 11 * n, b + 14 * n};
  const float* src[6] = {c->means, c->rotations, c->log_scales, c->raw_opacities, c->colors, c->sh_rest};
  const int64_t width[6] = {3, 4, 3, 1, 3, 3 * nb};
  for (int k = 0; k < 6; ++k)
    if (width[k] > 0)
      ODGS_CUDA(ctx, cudaMemcpyAsync(dst[k], src[k], sizeof(float) * width[k] * n, cudaMemcpyHostToDevice,
                                     ctx->stream));
  *out = {dst[0], dst[1], dst[2], dst[3], dst[4], c->sh_degree, nb > 0 ? dst[5] : nullptr};
  return ODGS_OK;
}

// Reads the device error words (synchronizing the stream).
odgs_status read_errors(odgs_ctx* ctx) {
  ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(DevErrors), cudaMemcpyDeviceToHost, ctx->stream));
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return ODGS_OK;
}

odgs_status reset_errors(odgs_ctx* ctx) {
  launch_reset_errors(ctx->d_err, false, ctx->stream);
  ODGS_CUDA(ctx, cudaGetLastError());
  return ODGS_OK;
}

// A render starts: its counters are reset; the sticky words too, unless earlier
// asynchronous work on the frame is still unchecked (its errors must survive to the check).
odgs_status reset_frame_errors(odgs_ctx* ctx, odgs_frame* f) {
  launch_reset_errors(f->d_err, f->pending || f->bwd_pending, ctx->stream);
  ODGS_CUDA(ctx, cudaGetLastError());
  return ODGS_OK;
}

// Reads the frame's device error words (synchronizing the stream).
odgs_status read_frame_errors(odgs_ctx* ctx, odgs_frame* f) {
  ODGS_CUDA(ctx, cudaMemcpyAsync(f->h_err, f->d_err, sizeof(DevErrors), cudaMemcpyDeviceToHost, ctx->stream));
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return ODGS_OK;
}

// The reference's exceptions for projection-stage error words (rasterizer.hpp:133-136,
// covariance.hpp:14-15, 31-32, projection.hpp:23-24).
odgs_status projection_error(odgs_ctx* ctx, const DevErrors& he) {
  if (he.nonfinite != kNoError) {
    const int64_t idx = (int64_t)(he.nonfinite >> 4);
    return set_error(ctx, ODGS_ERR_RUNTIME, idx, "render: non-finite parameter in Gaussian " + std::to_string(idx));
  }
  if (he.project != kNoError) {
    const int64_t idx = (int64_t)(he.project >> 4);
    const int code = (int)(he.project & 15);
    if (code == 3) return set_error(ctx, ODGS_ERR_DOMAIN, idx, "to_spherical: degenerate zero-length direction");
    if (code == 2) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, idx, "build_covariance: non-finite parameters");
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, idx, "normalize_quaternion: near-zero quaternion");
  }
  return ODGS_OK;
}

odgs_status backward_error(odgs_ctx* ctx, const DevErrors& he) {
  if (he.bwd_domain != kNoError) {
    const int64_t idx = (int64_t)(he.bwd_domain >> 4);
    return set_error(ctx, ODGS_ERR_DOMAIN, idx, "grad_position: undefined at the pole axis");
  }
  if (he.bwd_nonfinite != kNoError) {
    const int64_t idx = (int64_t)(he.bwd_nonfinite >> 4);
    return set_error(ctx, ODGS_ERR_RUNTIME, idx, "backward: non-finite gradient for Gaussian " + std::to_string(idx));
  }
  return ODGS_OK;
}

// Entry capacity the frame's tile-entry buffers hold.
uint32_t entry_capacity(const odgs_frame* f) {
  const size_t c = std::min({f->ekeys[0].cap, f->ekeys[1].cap, f->evals[0].cap, f->evals[1].cap}) / sizeof(uint32_t);
  return (uint32_t)std::min<size_t>(c, (size_t)kMaxSortItems - 1);
}

odgs_status bin_impl(odgs_ctx* ctx, odgs_frame* f, bool band);

// Per-frame buffers of the projection stage (n Gaussians, n_tiles tiles).
odgs_status ensure_frame_buffers(odgs_ctx* ctx, odgs_frame* f, int64_t n, uint32_t n_tiles) {
  cudaStream_t s = ctx->stream;
  ODGS_CUDA(ctx, ensure(f->sp_ab, sizeof(float4) * 2 * n, s));
  ODGS_CUDA(ctx, ensure(f->sp_c, sizeof(float4) * n, s));
  if (f->flags & ODGS_FRAME_KEEP_COV2D) ODGS_CUDA(ctx, ensure(f->cov, sizeof(float4) * n, s));
  for (int k = 0; k < 2; ++k) {
    ODGS_CUDA(ctx, ensure(f->keys[k], sizeof(uint32_t) * n, s));
    ODGS_CUDA(ctx, ensure(f->vals[k], sizeof(uint32_t) * n, s));
  }
  ODGS_CUDA(ctx, ensure(f->cnt, sizeof(uint32_t) * n, s));
  ODGS_CUDA(ctx, ensure(f->cnt_sorted, sizeof(uint32_t) * n, s));
  ODGS_CUDA(ctx, ensure(f->off_sorted, sizeof(uint32_t) * n, s));
  ODGS_CUDA(ctx, ensure(f->ent_off_idx, sizeof(uint32_t) * n, s));
  ODGS_CUDA(ctx, ensure(f->scan_tmp, scan_temp_bytes(n) + 256, s));
  ODGS_CUDA(ctx, ensure(f->offsets, sizeof(int32_t) * (n_tiles + 1), s));
  return ODGS_OK;
}

odgs_status prepare_impl(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                         const odgs_settings* settings, odgs_frame* f, int32_t row_begin = 0,
                         int32_t row_end = -1) {
  if (!ctx || !f) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "null context or frame");
  odgs_status st;
  if ((st = check_camera(ctx, camera)) != ODGS_OK) return st;
  if ((st = check_settings(ctx, settings)) != ODGS_OK) return st;
  CloudPtrs cp;
  if ((st = resolve_cloud(ctx, cloud, &cp)) != ODGS_OK) return st;
  cudaStream_t s = ctx->stream;
  f->prepared = f->rendered = f->have_splat_grads = false;
  f->from_splats = false;
  f->width = camera->width;
  f->height = camera->height;
  f->tile_size = settings->tile_size;
  f->tiles_x = (f->width + f->tile_size - 1) / f->tile_size;
  f->tiles_y = (f->height + f->tile_size - 1) / f->tile_size;
  f->n = cloud->n;
  f->cam = to_dev(*camera);
  f->settings = to_dev(*settings);
  if (row_end < 0) row_end = f->height;
  if (row_begin < 0 || row_begin >= row_end || row_end > f->height || row_begin % f->tile_size != 0 ||
      (row_end % f->tile_size != 0 && row_end != f->height))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1,
                     "render_band: rows must satisfy 0 <= begin < end <= height on tile boundaries");
  f->row_begin = row_begin;
  f->row_end = row_end;
  f->settings.band_ty0 = row_begin / f->tile_size;
  f->settings.band_ty1 = (row_end + f->tile_size - 1) / f->tile_size;
  const int64_t n = f->n;
  const uint32_t n_tiles = (uint32_t)(f->tiles_x * f->tiles_y);

  if ((st = ensure_frame_buffers(ctx, f, n, n_tiles)) != ODGS_OK) return st;
  if ((st = reset_frame_errors(ctx, f)) != ODGS_OK) return st;
  f->pending = true;

  const bool band = f->settings.band_ty0 > 0 || f->settings.band_ty1 < f->tiles_y;
  f->band = band;
  PreprocessArgs pa;
  pa.n = n;
  pa.means = cp.means;
  pa.rotations = cp.rotations;
  pa.log_scales = cp.log_scales;
  pa.raw_opacities = cp.raw_opacities;
  pa.colors = cp.colors;
  pa.sh_degree = cp.sh_degree;
  pa.sh_rest = cp.sh_rest;
  pa.cam = f->cam;
  pa.settings = f->settings;
  pa.sp_ab = f->sp_ab.as<float4>();
  pa.sp_c = f->sp_c.as<float4>();
  pa.cov_out = (f->flags & ODGS_FRAME_KEEP_COV2D) ? f->cov.as<float4>() : nullptr;
  pa.keys = f->keys[0].as<uint32_t>();
  pa.vals = f->vals[0].as<uint32_t>();
  pa.cnt = f->cnt.as<uint32_t>();
  pa.err = f->d_err;
  {
    StageScope sc(ctx, ODGS_STAGE_PREPROCESS);
    if (band) {
      // Pre-cull, exact projection of the survivors and compaction of the Gaussians
      // with entries in the band, in one pass (per-warp segments in keys[1] / vals[1],
      // segment lengths / offsets in cnt_sorted / off_sorted, free until the gather).
      uint32_t* seg_count = f->cnt_sorted.as<uint32_t>();
      uint32_t* seg_off = f->off_sorted.as<uint32_t>();
      launch_band_preprocess(pa, f->keys[1].as<uint32_t>(), f->vals[1].as<uint32_t>(), seg_count, s);
      const int64_t n_seg = band_segments(n);
      exclusive_scan_u32(seg_count, seg_off, n_seg, f->scan_tmp.p, &f->d_err->n_band, s);
      launch_concat_segments(n, seg_count, seg_off, f->keys[1].as<uint32_t>(), f->vals[1].as<uint32_t>(),
                             f->keys[0].as<uint32_t>(), f->vals[0].as<uint32_t>(), s);
    } else {
      launch_preprocess(pa, s);
    }
  }

  return bin_impl(ctx, f, band);
}

// The part of prepare_render after projection (rasterizer.hpp:141-205): depth sort,
// tile-entry emission, tile sort, CSR, launch order. f->sp_ab / sp_c / keys[0] / vals[0]
// / cnt hold the projected splats (or, for a band, the compacted band survivors).
odgs_status bin_impl(odgs_ctx* ctx, odgs_frame* f, bool band) {
  odgs_status st;
  cudaStream_t s = ctx->stream;
  const int64_t n = f->n;
  const uint32_t n_tiles = (uint32_t)(f->tiles_x * f->tiles_y);
  // Exact path (entry capacity unknown): read the entry count (and a band's Gaussian
  // count) on the host. Capacity path: every count stays on the device and the launches
  // are sized for the capacities; no synchronisation.
  const bool exact = f->k_cap == 0 || n == 0;
  // Depth sort of the Gaussians (key: depth bits; culled sort last). A band render
  // sorts only the Gaussians with entries in its rows, compacted in index order above
  // (stable, so ties keep index order): the tile lists are unchanged, the sort shrinks
  // with the band (row bands over 8 GPUs sort ~1/8 of the cloud each).
  ODGS_CUDA(ctx, ensure(f->sort_tmp, std::max(radix_sort_temp_bytes(n), (size_t)16), s));
  uint32_t* dk[2] = {f->keys[0].as<uint32_t>(), f->keys[1].as<uint32_t>()};
  uint32_t* dv[2] = {f->vals[0].as<uint32_t>(), f->vals[1].as<uint32_t>()};
  int64_t m = n;
  // the band's Gaussian count on the device (low word of the 64-bit counter)
  const uint32_t* m_dev = band ? reinterpret_cast<const uint32_t*>(&f->d_err->n_band) : nullptr;
  StageScope* depth_scope = new StageScope(ctx, ODGS_STAGE_DEPTH_SORT);
  if (band && n > 0 && exact) {
    if ((st = read_frame_errors(ctx, f)) != ODGS_OK) {
      delete depth_scope;
      return st;
    }
    m = (int64_t)f->h_err->n_band;
    m_dev = nullptr;
  }
  {
    int which = 0;
    // The last pass also gathers each rank's tile count (cnt_sorted).
    const cudaError_t e = radix_sort_pairs(dk, dv, m, 0, 32, f->sort_tmp.p, &which, s, f->cnt.as<uint32_t>(),
                                           f->cnt_sorted.as<uint32_t>(), m_dev);
    if (e != cudaSuccess) {
      delete depth_scope;
      return cuda_fail(ctx, e, "depth sort");
    }
    f->depth_which = which;  // index into f->vals / f->keys
  }
  delete depth_scope;
  f->n_sorted = m;  // the sorted ranks: m, or at most m (band, capacity path: m_dev on the device)
  const uint32_t* sorted_idx = f->vals[f->depth_which].as<uint32_t>();
  {
    StageScope sc(ctx, ODGS_STAGE_SCAN);
    exclusive_scan_u32(f->cnt_sorted.as<uint32_t>(), f->off_sorted.as<uint32_t>(), m, f->scan_tmp.p,
                       &f->d_err->n_entries, s, m_dev);
  }
  uint32_t K = 0;
  if (exact) {
    if ((st = read_frame_errors(ctx, f)) != ODGS_OK) return st;
    const DevErrors& he = *f->h_err;
    if ((st = projection_error(ctx, he)) != ODGS_OK) {
      // reported: the frame starts clean (its sticky words read and cleared)
      f->pending = f->bwd_pending = false;
      ODGS_CUDA(ctx, cudaMemcpyAsync(f->d_err, ctx->h_err_init, kDevErrorsSticky, cudaMemcpyHostToDevice, s));
      return st;
    }
    const unsigned long long total = n > 0 ? he.n_entries : 0ull;
    // The onesweep look-back words carry 30-bit digit counts (sort.cu), so a sort holds
    // fewer than 2^30 items.
    if (total >= kMaxSortItems)
      return set_error(ctx, ODGS_ERR_OUT_OF_MEMORY, -1, "prepare_render: 2^30 or more tile entries");
    f->n_entries = (uint32_t)total;
    f->n_splats = n > 0 ? (int64_t)he.n_visible : 0;
    f->n_instances = n > 0 ? (int64_t)he.n_instances : 0;
    K = f->n_entries;
    for (int k = 0; k < 2; ++k) {
      ODGS_CUDA(ctx, ensure(f->ekeys[k], sizeof(uint32_t) * K, s));
      ODGS_CUDA(ctx, ensure(f->evals[k], sizeof(uint32_t) * K, s));
    }
  } else {
    K = f->k_cap;
  }
  const uint32_t cap = entry_capacity(f);
  // The capacity path sorts / bins min(entries, capacity) entries, counted on the device.
  const uint32_t* k_dev = exact ? nullptr : reinterpret_cast<const uint32_t*>(&f->d_err->k_sort);

  EmitArgs ea;
  ea.n = m;
  ea.sorted_idx = sorted_idx;
  ea.cnt_sorted = f->cnt_sorted.as<uint32_t>();
  ea.off_sorted = f->off_sorted.as<uint32_t>();
  ea.sp_ab = f->sp_ab.as<float4>();
  ea.sp_c = f->sp_c.as<float4>();
  ea.width = f->width;
  ea.height = f->height;
  ea.tile_size = f->tile_size;
  ea.tiles_x = f->tiles_x;
  ea.band_ty0 = f->settings.band_ty0;
  ea.band_ty1 = f->settings.band_ty1;
  ea.out_keys = f->ekeys[0].as<uint32_t>();
  ea.out_vals = f->evals[0].as<uint32_t>();
  ea.ent_off_idx = f->ent_off_idx.as<uint32_t>();
  ea.n_dev = m_dev;
  ea.total = &f->d_err->n_entries;
  ea.capacity = exact ? K : cap;
  ea.k_sort = exact ? nullptr : &f->d_err->k_sort;
  ea.overflow = &f->d_err->overflow;
  {
    StageScope sc(ctx, ODGS_STAGE_EMIT);
    launch_emit(ea, s);
  }

  ODGS_CUDA(ctx, ensure(f->sort_tmp, std::max(radix_sort_temp_bytes(K), radix_sort_temp_bytes(n)), s));
  uint32_t* ek[2] = {f->ekeys[0].as<uint32_t>(), f->ekeys[1].as<uint32_t>()};
  uint32_t* ev[2] = {f->evals[0].as<uint32_t>(), f->evals[1].as<uint32_t>()};
  {
    StageScope sc(ctx, ODGS_STAGE_TILE_SORT);
    ODGS_CUDA(ctx, radix_sort_pairs(ek, ev, K, 0, bits_for(n_tiles), f->sort_tmp.p, &f->tile_which, s, nullptr,
                                    nullptr, k_dev));
  }
  {
    StageScope sc(ctx, ODGS_STAGE_RANGES);
    launch_tile_ranges(K, ek[f->tile_which], n_tiles, (uint32_t)(f->settings.band_ty0 * f->tiles_x),
                       (uint32_t)(f->settings.band_ty1 * f->tiles_x), f->offsets.as<int32_t>(), s, k_dev);
    const int band_tiles = f->tiles_x * (f->settings.band_ty1 - f->settings.band_ty0);
    ODGS_CUDA(ctx, ensure(f->tile_order, sizeof(uint32_t) * std::max(band_tiles, 1), s));
    launch_tile_order(f->offsets.as<int32_t>(), f->settings.band_ty0 * f->tiles_x, band_tiles,
                      f->tile_order.as<uint32_t>(), s);
  }
  ODGS_CUDA(ctx, cudaGetLastError());
  // Later renders of this frame run on the capacity path.
  f->k_cap = n > 0 ? std::max<uint32_t>(cap, 1u) : f->k_cap;
  f->pending = !exact;
  f->cap_path = !exact;
  f->prepared = true;
  return ok(ctx);
}

odgs_status blend_impl(odgs_ctx* ctx, odgs_frame* f) {
  cudaStream_t s = ctx->stream;
  const int64_t px = (int64_t)f->width * f->height;
  ODGS_CUDA(ctx, ensure(f->image, sizeof(float) * 3 * px, s));
  ODGS_CUDA(ctx, ensure(f->trans, sizeof(float) * px, s));
  ODGS_CUDA(ctx, ensure(f->walked, sizeof(int32_t) * px, s));
  // Work counters only for frames that ask for them (a memset in the stream would also
  // break the programmatic-launch chain into the blend).
  f->work_counted = (f->flags & ODGS_FRAME_COUNT_WORK) != 0;
  if (f->work_counted) {
    ODGS_CUDA(ctx, ensure(f->work, 2 * sizeof(unsigned long long), s));
    launch_zero_bytes(f->work.p, 2 * sizeof(unsigned long long), s);
  }
  BlendArgs ba;
  ba.offsets = f->offsets.as<int32_t>();
  ba.vals = f->evals[f->tile_which].as<uint32_t>();
  ba.sp_ab = f->sp_ab.as<float4>();
  ba.sp_c = f->sp_c.as<float4>();
  ba.width = f->width;
  ba.height = f->height;
  ba.tile_size = f->tile_size;
  ba.tiles_x = f->tiles_x;
  ba.tiles_y = f->tiles_y;
  ba.band_ty0 = f->settings.band_ty0;
  ba.band_ty1 = f->settings.band_ty1;
  ba.alpha_clamp = f->settings.alpha_clamp;
  ba.transmittance_floor = f->settings.transmittance_floor;
  ba.cutoff_sigma = f->settings.cutoff_sigma;
  ba.image = f->image.as<float>();
  ba.transmittance = f->trans.as<float>();
  ba.walked = f->walked.as<int32_t>();
  ba.work = f->work_counted ? f->work.as<unsigned long long>() : nullptr;
  ba.order = f->tile_order.as<uint32_t>();
  ba.peers = f->peers;
  ba.plain = (f->flags & ODGS_FRAME_PLAIN_BLEND) != 0;
  {
    StageScope sc(ctx, ODGS_STAGE_BLEND);
    launch_blend(ba, s);
  }
  ODGS_CUDA(ctx, cudaGetLastError());
  f->rendered = true;
  return ok(ctx);
}

size_t field_elem_bytes(int field) {
  switch (field) {
    case ODGS_FRAME_SPLAT_INDEX: return 8;
    default: return 4;
  }
}

// Splat-order (visible Gaussians ascending) host views of per-Gaussian device data.
struct HostViews {
  std::vector<float4> ab, c;
  std::vector<int64_t> splat_of;  // Gaussian -> splat position or -1
  std::vector<int64_t> visible;   // splat position -> Gaussian
};

odgs_status load_views(odgs_ctx* ctx, odgs_frame* f, HostViews* v) {
  const int64_t n = f->n;
  v->ab.resize(2 * n);
  v->c.resize(n);
  if (n > 0) {
    ODGS_CUDA(ctx, cudaMemcpyAsync(v->ab.data(), f->sp_ab.p, sizeof(float4) * 2 * n, cudaMemcpyDeviceToHost, ctx->stream));
    ODGS_CUDA(ctx, cudaMemcpyAsync(v->c.data(), f->sp_c.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  v->splat_of.assign(n, -1);
  v->visible.clear();
  for (int64_t i = 0; i < n; ++i) {
    uint32_t fl;
    std::memcpy(&fl, &v->c[i].w, 4);
    if (fl & kFlagVisible) {
      v->splat_of[i] = (int64_t)v->visible.size();
      v->visible.push_back(i);
    }
  }
  return ODGS_OK;
}

uint32_t flags_of(const float4& c) {
  uint32_t fl;
  std::memcpy(&fl, &c.w, 4);
  return fl;
}

// grad_pixels_to_splats' pixel half (backward.hpp:208-327) on a rendered frame: the
// upstream gradient to the device (if on the host), the per-entry records of the back-
// to-front replay, and their ordered fold per Gaussian into f->folded. The alpha clamp
// and cutoff come from `settings`, as the reference's backward reads them.
odgs_status raster_fold(odgs_ctx* ctx, odgs_frame* f, const float* dl_dimage, int32_t dl_memory,
                        const odgs_settings* settings) {
  cudaStream_t s = ctx->stream;
  const int64_t n = f->n;
  const int64_t px = (int64_t)f->width * f->height;
  // Entry buffers: the capacity covers every emit position of a capacity-path frame.
  const uint32_t K = std::max(f->n_entries, f->k_cap);
  const float* dl = dl_dimage;
  if (dl_memory != ODGS_MEM_DEVICE) {
    ODGS_CUDA(ctx, ensure(ctx->dl_buf, sizeof(float) * 3 * px, s));
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->dl_buf.p, dl_dimage, sizeof(float) * 3 * px, cudaMemcpyHostToDevice, s));
    dl = ctx->dl_buf.as<float>();
  }
  ODGS_CUDA(ctx, ensure(f->records, sizeof(float) * 12 * (size_t)K, s));  // kRecStride floats per entry
  ODGS_CUDA(ctx, ensure(f->touched, (size_t)K + 16, s));
  ODGS_CUDA(ctx, ensure(f->folded, sizeof(float) * 9 * (size_t)n + 16, s));
  ODGS_CUDA(ctx, ensure(f->bwd_work, 4 * sizeof(unsigned long long), s));
  f->bwd_work_counted = (f->flags & ODGS_FRAME_COUNT_WORK) != 0;
  if (f->bwd_work_counted) launch_zero_bytes(f->bwd_work.p, 4 * sizeof(unsigned long long), s);
  {
    StageScope sc(ctx, ODGS_STAGE_BWD_RASTER);
    if (K) launch_zero_bytes(f->touched.p, (size_t)K, s);
    BwdRasterArgs ra;
    ra.offsets = f->offsets.as<int32_t>();
    ra.vals = f->evals[f->tile_which].as<uint32_t>();
    ra.sp_ab = f->sp_ab.as<float4>();
    ra.sp_c = f->sp_c.as<float4>();
    ra.ent_off_idx = f->ent_off_idx.as<uint32_t>();
    ra.transmittance = f->trans.as<float>();
    ra.walked = f->walked.as<int32_t>();
    ra.dl_dimage = dl;
    ra.width = f->width;
    ra.height = f->height;
    ra.tile_size = f->tile_size;
    ra.tiles_x = f->tiles_x;
    ra.tiles_y = f->tiles_y;
    ra.band_ty0 = f->settings.band_ty0;
    ra.band_ty1 = f->settings.band_ty1;
    ra.alpha_clamp = settings->alpha_clamp;
    ra.cutoff_sigma = settings->cutoff_sigma;
    ra.records = f->records.as<float>();
    ra.touched = f->touched.as<uint8_t>();
    ra.order = f->tile_order.as<uint32_t>();
    ra.plain = (f->flags & ODGS_FRAME_PLAIN_BLEND) != 0;
    ra.work = (f->flags & ODGS_FRAME_COUNT_WORK) ? f->bwd_work.as<unsigned long long>() : nullptr;
    launch_bwd_raster(ra, s);
  }
  {
    StageScope sc(ctx, ODGS_STAGE_BWD_SPLAT);
    // A band's sorted ranks are counted on the device (capacity path: n_sorted = n).
    const uint32_t* m_dev = f->band ? reinterpret_cast<const uint32_t*>(&f->d_err->n_band) : nullptr;
    // Capacity path: records exist only below the sorted entry count (an overflowed frame
    // is re-rendered at its check point; until then its fold must stay inside the buffers).
    const unsigned long long* k_lim = f->cap_path ? &f->d_err->k_sort : nullptr;
    launch_fold_records(f->n_sorted, f->vals[f->depth_which].as<uint32_t>(), f->cnt_sorted.as<uint32_t>(),
                        f->off_sorted.as<uint32_t>(), f->touched.as<uint8_t>(), f->records.as<float>(),
                        f->folded.as<float>(), s, m_dev, k_lim);
  }
  ODGS_CUDA(ctx, cudaGetLastError());
  return ODGS_OK;
}

odgs_status prepare_impl(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                         const odgs_settings* settings, odgs_frame* f, int32_t row_begin, int32_t row_end);
odgs_status blend_impl(odgs_ctx* ctx, odgs_frame* f);

// Runs the frame's recorded render request (render, prepare_render or a band).
odgs_status run_request(odgs_ctx* ctx, odgs_frame* f) {
  const odgs_frame::Request r = f->req;
  odgs_status st;
  if (r.kind == 3) st = prepare_impl(ctx, &r.cloud, &r.camera, &r.settings, f, r.row_begin, r.row_end);
  else st = prepare_impl(ctx, &r.cloud, &r.camera, &r.settings, f, 0, -1);
  if (st != ODGS_OK) return st;
  if (r.kind != 2) st = blend_impl(ctx, f);
  return st;
}

// The frame's check point: synchronises, reads the frame's error words and counts, and
// reports deferred errors as the synchronous call would have. An overflow of the entry
// buffers re-runs the frame's last render request with room for every entry (the exact
// path), so the frame holds the correct result; *rerun (optional) tells the caller that
// work enqueued on the overflowed frame since (a backward) must be repeated.
odgs_status finish_frame(odgs_ctx* ctx, odgs_frame* f, int32_t* rerun = nullptr) {
  if (rerun) *rerun = 0;
  if (!f->pending && !f->bwd_pending) return ODGS_OK;
  odgs_status st;
  if ((st = read_frame_errors(ctx, f)) != ODGS_OK) return st;
  const DevErrors he = *f->h_err;
  const bool fwd = f->pending, bwd = f->bwd_pending;
  f->pending = f->bwd_pending = false;
  // the host has the sticky words now: clear them for the next operations
  ODGS_CUDA(ctx, cudaMemcpyAsync(f->d_err, ctx->h_err_init, kDevErrorsSticky, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = projection_error(ctx, he)) != ODGS_OK) return st;
  if (fwd) {
    const unsigned long long total = f->n > 0 ? he.n_entries : 0ull;
    if (total >= kMaxSortItems)
      return set_error(ctx, ODGS_ERR_OUT_OF_MEMORY, -1, "prepare_render: 2^30 or more tile entries");
    f->n_entries = (uint32_t)total;
    f->n_splats = f->n > 0 ? (int64_t)he.n_visible : 0;
    f->n_instances = f->n > 0 ? (int64_t)he.n_instances : 0;
    if (f->band) f->n_sorted = (int64_t)he.n_band;  // the capacity path sorted the band's Gaussians
  }
  if (he.overflow) {
    if (he.overflow >= kMaxSortItems)
      return set_error(ctx, ODGS_ERR_OUT_OF_MEMORY, -1, "prepare_render: 2^30 or more tile entries");
    if (f->req.kind == 0) return set_error(ctx, ODGS_ERR_RUNTIME, -1, "tile-entry overflow without a request");
    // Room for the largest entry count seen since the last check (the overflow word
    // keeps the maximum), then the exact path re-runs the last request.
    const size_t want = (size_t)he.overflow;
    for (int k = 0; k < 2; ++k) {
      ODGS_CUDA(ctx, ensure(f->ekeys[k], sizeof(uint32_t) * want, ctx->stream));
      ODGS_CUDA(ctx, ensure(f->evals[k], sizeof(uint32_t) * want, ctx->stream));
    }
    f->k_cap = 0;  // the exact path: the entry count read on the host, buffers grown to fit
    if ((st = run_request(ctx, f)) != ODGS_OK) return st;
    if (rerun) *rerun = 1;
    return finish_frame(ctx, f);
  }
  if (bwd && (st = backward_error(ctx, he)) != ODGS_OK) return st;
  return ODGS_OK;
}

}  // namespace

extern "C" {

odgs_settings odgs_default_settings(void) {
  odgs_settings s;
  s.near_radius = 0.01f;
  s.far_radius = 1000.0f;
  s.tile_size = 16;
  s.alpha_clamp = 0.99f;
  s.transmittance_floor = 1e-4f;
  s.cutoff_sigma = 3.0f;
  s.lowpass_dilation = 0.3f;
  s.max_elevation = 85.0f * kPiF / 180.0f;
  s.threads = 0;
  return s;
}

int odgs_abi_version(void) { return ODGS_ABI_VERSION; }

odgs_status odgs_ctx_create(int device, void* stream, odgs_ctx** out) {
  if (!out) return ODGS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  odgs_ctx* ctx = new (std::nothrow) odgs_ctx();
  if (!ctx) return ODGS_ERR_OUT_OF_MEMORY;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) {
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
      ctx->own_stream = true;
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, sizeof(DevErrors));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_err, sizeof(DevErrors));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_err_init, sizeof(DevErrors));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_scratch, 256);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_unit_signs, 12 * sizeof(float));
  if (e == cudaSuccess) {
    const float ones[12] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    e = cudaMemcpy(ctx->d_unit_signs, ones, sizeof ones, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    odgs_ctx_destroy(ctx);
    return e == cudaErrorMemoryAllocation ? ODGS_ERR_OUT_OF_MEMORY : ODGS_ERR_CUDA;
  }
  std::memset(ctx->h_err_init, 0, sizeof(DevErrors));  // overflow, counters, k_sort: 0
  ctx->h_err_init->nonfinite = kNoError;
  ctx->h_err_init->project = kNoError;
  ctx->h_err_init->bwd_domain = kNoError;
  ctx->h_err_init->bwd_nonfinite = kNoError;
  ctx->h_err_init->n_entries = 0;
  ctx->h_err_init->n_visible = 0;
  ctx->h_err_init->n_instances = 0;
  ctx->h_err_init->n_band = 0;
  ctx->h_err_init->n_precull = 0;
  ctx->h_err_init->k_sort = 0;
  ctx->h_err_init->overflow = 0;
  *out = ctx;
  return ODGS_OK;
}

void odgs_ctx_destroy(odgs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  resolve_timers(ctx);
  for (cudaEvent_t e : ctx->timers.pool) cudaEventDestroy(e);
  if (ctx->stream) {
    release(ctx->cloud_buf, ctx->stream);
    release(ctx->dl_buf, ctx->stream);
    release(ctx->grads_buf, ctx->stream);
    release(ctx->signs_buf, ctx->stream);
    release(ctx->cull_buf, ctx->stream);
    release(ctx->loss_buf, ctx->stream);
    release(ctx->densify_buf, ctx->stream);
    release(ctx->unit_ball_buf, ctx->stream);
    release(ctx->misc_buf, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
  }
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->d_unit_signs) cudaFree(ctx->d_unit_signs);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_err_init) cudaFreeHost(ctx->h_err_init);
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

odgs_status odgs_ctx_set_stream(odgs_ctx* ctx, void* stream) {
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->own_stream = false;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return ok(ctx);
}

void* odgs_ctx_stream(odgs_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

odgs_status odgs_synchronize(odgs_ctx* ctx) {
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return ok(ctx);
}

odgs_status odgs_last_error(const odgs_ctx* ctx, int64_t* gaussian_index, char* message, size_t message_len) {
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  if (gaussian_index) *gaussian_index = ctx->last_index;
  if (message && message_len > 0) std::snprintf(message, message_len, "%s", ctx->last_msg.c_str());
  return ctx->last_code;
}

int64_t odgs_ctx_launch_count(const odgs_ctx* ctx) { return ctx ? ctx->launches : 0; }

odgs_status odgs_frame_create(odgs_ctx* ctx, odgs_frame** out) {
  if (!ctx || !out) return ODGS_ERR_INVALID_ARGUMENT;
  odgs_frame* f = new (std::nothrow) odgs_frame();
  if (!f) return set_error(ctx, ODGS_ERR_OUT_OF_MEMORY, -1, "frame allocation");
  f->ctx = ctx;
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMalloc(&f->d_err, sizeof(DevErrors));
  if (e == cudaSuccess) e = cudaMallocHost(&f->h_err, sizeof(DevErrors));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(f->d_err, ctx->h_err_init, sizeof(DevErrors), cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) {
    if (f->d_err) cudaFree(f->d_err);
    if (f->h_err) cudaFreeHost(f->h_err);
    delete f;
    return cuda_fail(ctx, e, "frame error words");
  }
  *out = f;
  return ok(ctx);
}

void odgs_frame_destroy(odgs_frame* f) {
  if (!f) return;
  cudaStream_t s = f->ctx->stream;
  DevBuf* bufs[] = {&f->sp_ab, &f->sp_c, &f->cov, &f->keys[0], &f->keys[1], &f->vals[0], &f->vals[1], &f->cnt,
                    &f->cnt_sorted, &f->off_sorted, &f->ent_off_idx, &f->sort_tmp, &f->scan_tmp, &f->ekeys[0],
                    &f->ekeys[1], &f->evals[0], &f->evals[1], &f->offsets, &f->tile_order, &f->image, &f->trans, &f->walked,
                    &f->records, &f->touched, &f->folded, &f->splat_grads, &f->work, &f->bwd_work};
  for (DevBuf* b : bufs) release(*b, s);
  cudaStreamSynchronize(s);
  if (f->d_err) cudaFree(f->d_err);
  if (f->h_err) cudaFreeHost(f->h_err);
  delete f;
}

odgs_status odgs_frame_set_image_peers(odgs_frame* f, int32_t n, void* const* peer_images) {
  if (!f || n < 0 || n > kMaxPeers || (n > 0 && !peer_images)) return ODGS_ERR_INVALID_ARGUMENT;
  f->peers = PeerImages{};
  for (int k = 0; k < n; ++k) {
    if (!peer_images[k]) return ODGS_ERR_INVALID_ARGUMENT;
    f->peers.ptr[k] = static_cast<float*>(peer_images[k]);
  }
  f->peers.n = n;
  return ODGS_OK;
}

// The enclosing allocation of a device pointer: the driver's cuMemGetAddressRange (the
// runtime has no such query), fetched through the runtime so the library does not link
// libcuda itself (it must load on hosts without a driver for the CPU checks).
static bool alloc_base(const void* p, char** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (Fn) nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  CUdeviceptr b = 0;
  size_t size = 0;
  if (!fn || fn(&b, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<char*>(b);
  return true;
}

odgs_status odgs_ipc_get_handle(const void* device_ptr, void* handle) {
  if (!device_ptr || !handle) return ODGS_ERR_INVALID_ARGUMENT;
  char* base = nullptr;
  if (!alloc_base(device_ptr, &base)) return ODGS_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return ODGS_ERR_CUDA;
  static_assert(sizeof(h) + sizeof(uint64_t) == ODGS_IPC_HANDLE_BYTES, "handle + offset");
  const uint64_t offset = (uint64_t)(static_cast<const char*>(device_ptr) - base);
  std::memcpy(handle, &h, sizeof h);
  std::memcpy(static_cast<char*>(handle) + sizeof h, &offset, sizeof offset);
  return ODGS_OK;
}

odgs_status odgs_ipc_open(const void* handle, void** device_ptr) {
  if (!handle || !device_ptr) return ODGS_ERR_INVALID_ARGUMENT;
  cudaIpcMemHandle_t h;
  uint64_t offset = 0;
  std::memcpy(&h, handle, sizeof h);
  std::memcpy(&offset, static_cast<const char*>(handle) + sizeof h, sizeof offset);
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ODGS_ERR_CUDA;
  *device_ptr = static_cast<char*>(base) + offset;
  return ODGS_OK;
}

odgs_status odgs_ipc_close(void* device_ptr) {
  if (!device_ptr) return ODGS_ERR_INVALID_ARGUMENT;
  char* base = nullptr;
  if (!alloc_base(device_ptr, &base)) return ODGS_ERR_CUDA;
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? ODGS_OK : ODGS_ERR_CUDA;
}

odgs_status odgs_frame_set_flags(odgs_frame* f, uint32_t flags) {
  if (!f) return ODGS_ERR_INVALID_ARGUMENT;
  f->flags = flags;
  return ODGS_OK;
}

odgs_status odgs_frame_get_info(const odgs_frame* cf, odgs_frame_info* info) {
  if (!cf || !info) return ODGS_ERR_INVALID_ARGUMENT;
  odgs_frame* f = const_cast<odgs_frame*>(cf);  // the counts of an asynchronous render are read here
  if (f->pending || f->bwd_pending) {
    cudaSetDevice(f->ctx->device);
    const odgs_status st = finish_frame(f->ctx, f);
    if (st != ODGS_OK) return st;
  }
  info->width = f->width;
  info->height = f->height;
  info->tiles_x = f->tiles_x;
  info->tiles_y = f->tiles_y;
  info->n_gaussians = f->n;
  info->n_entries = f->n_entries;
  info->n_splats = f->n_splats;
  info->n_instances = f->n_instances;
  info->row_begin = f->row_begin;
  info->row_end = f->row_end;
  return ODGS_OK;
}

// A render-type entry point: records the request (for an overflow re-run), runs it and,
// unless the context is asynchronous, checks the frame right away (the reference's
// synchronous exceptions).
static odgs_status render_entry(odgs_ctx* ctx, odgs_frame* frame, int kind) {
  frame->req.kind = kind;
  odgs_status st = run_request(ctx, frame);
  if (st == ODGS_OK && !ctx->async_mode) st = finish_frame(ctx, frame);
  if (ctx->timers.enabled) resolve_timers(ctx);
  return st == ODGS_OK ? ok(ctx) : st;
}

odgs_status odgs_prepare_render(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                                const odgs_settings* settings, odgs_frame* frame) {
  LaunchScope scope(ctx);
  if (!ctx || !frame) return ODGS_ERR_INVALID_ARGUMENT;
  if (!cloud || !camera || !settings) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "null argument");
  cudaSetDevice(ctx->device);
  frame->req.cloud = *cloud;
  frame->req.camera = *camera;
  frame->req.settings = *settings;
  frame->req.row_begin = 0;
  frame->req.row_end = -1;
  return render_entry(ctx, frame, 2);
}

odgs_status odgs_render(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                        const odgs_settings* settings, odgs_frame* frame) {
  LaunchScope scope(ctx);
  if (!ctx || !frame) return ODGS_ERR_INVALID_ARGUMENT;
  if (!cloud || !camera || !settings) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "null argument");
  cudaSetDevice(ctx->device);
  frame->req.cloud = *cloud;
  frame->req.camera = *camera;
  frame->req.settings = *settings;
  frame->req.row_begin = 0;
  frame->req.row_end = -1;
  return render_entry(ctx, frame, 1);
}

odgs_status odgs_ctx_set_async(odgs_ctx* ctx, int enable) {
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  ctx->async_mode = enable != 0;
  return ok(ctx);
}

odgs_status odgs_frame_check(odgs_ctx* ctx, odgs_frame* frame, int32_t* rerendered) {
  if (!ctx || !frame) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const odgs_status st = finish_frame(ctx, frame, rerendered);
  return st == ODGS_OK ? ok(ctx) : st;
}

odgs_status odgs_frame_backward_work(odgs_ctx* ctx, odgs_frame* f, int64_t* counters, int32_t n_counters) {
  if (!ctx || !f || !f->bwd_work.p) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "no backward on this frame");
  unsigned long long w[4] = {0, 0, 0, 0};
  if (f->bwd_work_counted) {
    ODGS_CUDA(ctx, cudaMemcpyAsync(w, f->bwd_work.p, sizeof w, cudaMemcpyDeviceToHost, ctx->stream));
    ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  for (int k = 0; k < n_counters && k < 4; ++k) counters[k] = (int64_t)w[k];
  return ok(ctx);
}

odgs_status odgs_rasterize_splats(odgs_ctx* ctx, int64_t n_gaussians, int64_t n_splats, const int64_t* index,
                                  const float* pixel_mean, const float* cov2d_inv, const float* depth,
                                  const float* radius, const float* opacity, const float* color, int32_t width,
                                  int32_t height, const odgs_settings* settings, odgs_frame* f) {
  LaunchScope scope(ctx);
  if (!ctx || !f) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  odgs_status st;
  if ((st = check_settings(ctx, settings)) != ODGS_OK) return st;
  if (width <= 0 || height <= 0 || width != 2 * height || (int64_t)width * height > ((int64_t)1 << 31))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "rasterize_splats: bad image size");
  if (n_gaussians < 0 || n_gaussians >= ((int64_t)1 << 30) || n_splats < 0 || n_splats > n_gaussians)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "rasterize_splats: bad sizes");
  if (n_splats > 0 && !(index && pixel_mean && cov2d_inv && depth && radius && opacity && color))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "rasterize_splats: null splat arrays");
  // Host-side checks and packing (kSplatRecord floats per splat).
  std::vector<float> rec((size_t)n_splats * kSplatRecord);
  for (int64_t k = 0; k < n_splats; ++k) {
    const int64_t i = index[k];
    if (i < 0 || i >= n_gaussians || (k > 0 && i <= index[k - 1]))
      return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, k, "rasterize_splats: indices must ascend inside the cloud");
    const float v[11] = {pixel_mean[2 * k], pixel_mean[2 * k + 1], cov2d_inv[4 * k], cov2d_inv[4 * k + 1],
                         cov2d_inv[4 * k + 3], depth[k], radius[k], opacity[k], color[3 * k], color[3 * k + 1],
                         color[3 * k + 2]};
    for (float x : v)
      if (!std::isfinite(x))
        return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, k, "rasterize_splats: non-finite splat");
    if (!(depth[k] >= 0.0f) || !(radius[k] >= 0.0f))
      return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, k, "rasterize_splats: negative depth or radius");
    float* r = rec.data() + (size_t)k * kSplatRecord;
    const uint32_t bits = (uint32_t)i;
    std::memcpy(r, &bits, 4);
    std::memcpy(r + 1, v, sizeof v);
  }
  cudaStream_t s = ctx->stream;
  f->prepared = f->rendered = f->have_splat_grads = false;
  f->from_splats = true;
  f->width = width;
  f->height = height;
  f->tile_size = settings->tile_size;
  f->tiles_x = (width + f->tile_size - 1) / f->tile_size;
  f->tiles_y = (height + f->tile_size - 1) / f->tile_size;
  f->n = n_gaussians;
  f->cam = DevCamera{};
  f->cam.width = width;
  f->cam.height = height;
  f->settings = to_dev(*settings);
  f->row_begin = 0;
  f->row_end = height;
  f->settings.band_ty0 = 0;
  f->settings.band_ty1 = f->tiles_y;
  if ((st = ensure_frame_buffers(ctx, f, n_gaussians, (uint32_t)(f->tiles_x * f->tiles_y))) != ODGS_OK) return st;
  if ((st = finish_frame(ctx, f)) != ODGS_OK) return st;  // earlier asynchronous work on this frame
  if ((st = reset_frame_errors(ctx, f)) != ODGS_OK) return st;
  f->req.kind = 0;  // no re-run: the exact path below cannot overflow
  f->k_cap = 0;
  f->band = false;
  f->pending = true;
  ODGS_CUDA(ctx, ensure(ctx->misc_buf, rec.size() * sizeof(float), s));
  if (!rec.empty())
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->misc_buf.p, rec.data(), rec.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  launch_load_splats(n_gaussians, n_splats, ctx->misc_buf.as<float>(), width, height, f->tile_size, f->sp_ab.as<float4>(),
                     f->sp_c.as<float4>(), f->keys[0].as<uint32_t>(), f->vals[0].as<uint32_t>(),
                     f->cnt.as<uint32_t>(), f->d_err, s);
  if ((st = bin_impl(ctx, f, false)) != ODGS_OK) return st;
  ODGS_CUDA(ctx, cudaStreamSynchronize(s));  // the packed records live in host memory until here
  st = blend_impl(ctx, f);
  if (ctx->timers.enabled) resolve_timers(ctx);
  return st;
}

odgs_status odgs_frame_work(odgs_ctx* ctx, odgs_frame* f, int64_t* entries_examined, int64_t* entries_composited) {
  if (!ctx || !f || !f->rendered) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "frame not rendered");
  odgs_status st;
  if ((st = finish_frame(ctx, f)) != ODGS_OK) return st;
  unsigned long long w[2] = {0, 0};
  if (f->work_counted) {
    ODGS_CUDA(ctx, cudaMemcpyAsync(w, f->work.p, sizeof w, cudaMemcpyDeviceToHost, ctx->stream));
    ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  if (entries_examined) *entries_examined = (int64_t)w[0];
  if (entries_composited) *entries_composited = (int64_t)w[1];
  return ok(ctx);
}

odgs_status odgs_render_band(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera,
                             const odgs_settings* settings, int32_t row_begin, int32_t row_end, odgs_frame* frame) {
  LaunchScope scope(ctx);
  if (!ctx || !frame) return ODGS_ERR_INVALID_ARGUMENT;
  if (!cloud || !camera || !settings) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "null argument");
  cudaSetDevice(ctx->device);
  frame->req.cloud = *cloud;
  frame->req.camera = *camera;
  frame->req.settings = *settings;
  frame->req.row_begin = row_begin;
  frame->req.row_end = row_end;
  return render_entry(ctx, frame, 3);
}

odgs_status odgs_frame_device_ptr(odgs_frame* f, int field, void** device_ptr) {
  if (!f || !device_ptr || !f->prepared) return ODGS_ERR_INVALID_ARGUMENT;
  switch (field) {
    case ODGS_FRAME_IMAGE: *device_ptr = f->rendered ? f->image.p : nullptr; break;
    case ODGS_FRAME_TRANSMITTANCE: *device_ptr = f->rendered ? f->trans.p : nullptr; break;
    case ODGS_FRAME_WALKED: *device_ptr = f->rendered ? f->walked.p : nullptr; break;
    case ODGS_FRAME_TILE_OFFSETS: *device_ptr = f->offsets.p; break;
    default: return ODGS_ERR_INVALID_ARGUMENT;
  }
  return *device_ptr ? ODGS_OK : ODGS_ERR_INVALID_ARGUMENT;
}

odgs_status odgs_frame_download(odgs_ctx* ctx, odgs_frame* f, int field, void* host_dst, size_t bytes) {
  if (!ctx || !f || !f->prepared) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "frame not prepared");
  cudaSetDevice(ctx->device);
  {
    const odgs_status fs = finish_frame(ctx, f);  // an asynchronous render's errors and counts
    if (fs != ODGS_OK) return fs;
  }
  cudaStream_t s = ctx->stream;
  const int64_t px = (int64_t)f->width * f->height;
  const int64_t n_tiles = (int64_t)f->tiles_x * f->tiles_y;
  auto need = [&](size_t want) -> odgs_status {
    if (bytes < want) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "download: buffer too small");
    return ODGS_OK;
  };
  odgs_status st;
  auto copy_dev = [&](const void* src, size_t sz) -> odgs_status {
    if ((st = need(sz)) != ODGS_OK) return st;
    if (sz) ODGS_CUDA(ctx, cudaMemcpyAsync(host_dst, src, sz, cudaMemcpyDeviceToHost, s));
    ODGS_CUDA(ctx, cudaStreamSynchronize(s));
    return ok(ctx);
  };
  if ((field == ODGS_FRAME_IMAGE || field == ODGS_FRAME_TRANSMITTANCE || field == ODGS_FRAME_WALKED) && !f->rendered)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "frame not rendered");
  switch (field) {
    case ODGS_FRAME_IMAGE: return copy_dev(f->image.p, sizeof(float) * 3 * px);
    case ODGS_FRAME_TRANSMITTANCE: return copy_dev(f->trans.p, sizeof(float) * px);
    case ODGS_FRAME_WALKED: return copy_dev(f->walked.p, sizeof(int32_t) * px);
    case ODGS_FRAME_TILE_OFFSETS: return copy_dev(f->offsets.p, sizeof(int32_t) * (n_tiles + 1));
    default: break;
  }
  if (field < 0 || field >= ODGS_FRAME_FIELD_COUNT) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "bad field");
  if (field == ODGS_FRAME_SPLAT_COV2D && !(f->flags & ODGS_FRAME_KEEP_COV2D))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "SPLAT_COV2D needs ODGS_FRAME_KEEP_COV2D");
  if (field >= ODGS_FRAME_SPLATGRAD_MEAN && !f->have_splat_grads)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "no backward with ODGS_FRAME_KEEP_SPLAT_GRADS on this frame");

  // Reference-format views, materialised on the host from the device arrays.
  HostViews v;
  if ((st = load_views(ctx, f, &v)) != ODGS_OK) return st;
  const int64_t ns = (int64_t)v.visible.size();
  if (field >= ODGS_FRAME_SPLAT_INDEX && field <= ODGS_FRAME_SPLAT_CLAMPED) {
    const int width = (field == ODGS_FRAME_SPLAT_MEAN) ? 2
                      : (field == ODGS_FRAME_SPLAT_COV2D || field == ODGS_FRAME_SPLAT_INV) ? 4
                      : (field == ODGS_FRAME_SPLAT_COLOR) ? 3 : 1;
    if ((st = need(field_elem_bytes(field) * width * ns)) != ODGS_OK) return st;
    std::vector<float4> cov;
    if (field == ODGS_FRAME_SPLAT_COV2D) {
      cov.resize(f->n);
      if (f->n) ODGS_CUDA(ctx, cudaMemcpy(cov.data(), f->cov.p, sizeof(float4) * f->n, cudaMemcpyDeviceToHost));
    }
    for (int64_t sidx = 0; sidx < ns; ++sidx) {
      const int64_t i = v.visible[sidx];
      const float4 a = v.ab[2 * i], b = v.ab[2 * i + 1], c = v.c[i];
      float* o = static_cast<float*>(host_dst) + sidx * width;
      switch (field) {
        case ODGS_FRAME_SPLAT_INDEX: static_cast<int64_t*>(host_dst)[sidx] = i; break;
        case ODGS_FRAME_SPLAT_MEAN: o[0] = a.x; o[1] = a.y; break;
        case ODGS_FRAME_SPLAT_COV2D: o[0] = cov[i].x; o[1] = cov[i].y; o[2] = cov[i].z; o[3] = cov[i].w; break;
        case ODGS_FRAME_SPLAT_INV: o[0] = a.z; o[1] = a.w; o[2] = a.w; o[3] = b.x; break;
        case ODGS_FRAME_SPLAT_DEPTH: o[0] = c.y; break;
        case ODGS_FRAME_SPLAT_RADIUS: o[0] = c.z; break;
        case ODGS_FRAME_SPLAT_OPACITY: o[0] = b.y; break;
        case ODGS_FRAME_SPLAT_COLOR: o[0] = b.z; o[1] = b.w; o[2] = c.x; break;
        case ODGS_FRAME_SPLAT_CLAMPED: static_cast<int32_t*>(host_dst)[sidx] = (flags_of(c) & kFlagClamped) ? 1 : 0; break;
      }
    }
    return ok(ctx);
  }
  if (field >= ODGS_FRAME_SPLATGRAD_MEAN) {
    const int width = field == ODGS_FRAME_SPLATGRAD_MEAN ? 2 : field == ODGS_FRAME_SPLATGRAD_COV2D ? 4
                      : field == ODGS_FRAME_SPLATGRAD_OPACITY ? 1 : 3;
    const int first = field == ODGS_FRAME_SPLATGRAD_MEAN ? 0 : field == ODGS_FRAME_SPLATGRAD_COV2D ? 2
                      : field == ODGS_FRAME_SPLATGRAD_OPACITY ? 6 : 7;
    if ((st = need(sizeof(float) * width * ns)) != ODGS_OK) return st;
    std::vector<float> sg((size_t)f->n * 10);
    if (f->n) ODGS_CUDA(ctx, cudaMemcpy(sg.data(), f->splat_grads.p, sizeof(float) * 10 * f->n, cudaMemcpyDeviceToHost));
    for (int64_t sidx = 0; sidx < ns; ++sidx)
      for (int k = 0; k < width; ++k)
        static_cast<float*>(host_dst)[sidx * width + k] = sg[(size_t)v.visible[sidx] * 10 + first + k];
    return ok(ctx);
  }
  // Instances sorted by (depth, index, shift) and the tile entries as instance ids.
  std::vector<uint32_t> sorted_idx(f->n_sorted);
  if (f->n_sorted)
    ODGS_CUDA(ctx, cudaMemcpy(sorted_idx.data(), f->vals[f->depth_which].p, sizeof(uint32_t) * f->n_sorted,
                              cudaMemcpyDeviceToHost));
  std::vector<int32_t> inst_splat;
  std::vector<float> inst_shift;
  std::vector<int32_t> inst_id(3 * (size_t)f->n, -1);
  for (int64_t r = 0; r < f->n_sorted; ++r) {
    const uint32_t i = sorted_idx[r];
    const uint32_t fl = flags_of(v.c[i]);
    if (!(fl & kFlagVisible)) continue;
    for (int k = 0; k < 3; ++k)
      if (fl & (kFlagShiftBase << k)) {
        inst_id[3 * (size_t)i + k] = (int32_t)inst_splat.size();
        inst_splat.push_back((int32_t)v.splat_of[i]);
        inst_shift.push_back(k == 0 ? -(float)f->width : (k == 1 ? 0.0f : (float)f->width));
      }
  }
  if (field == ODGS_FRAME_INSTANCE_SPLAT) {
    if ((st = need(sizeof(int32_t) * inst_splat.size())) != ODGS_OK) return st;
    std::memcpy(host_dst, inst_splat.data(), sizeof(int32_t) * inst_splat.size());
    return ok(ctx);
  }
  if (field == ODGS_FRAME_INSTANCE_SHIFT) {
    if ((st = need(sizeof(float) * inst_shift.size())) != ODGS_OK) return st;
    std::memcpy(host_dst, inst_shift.data(), sizeof(float) * inst_shift.size());
    return ok(ctx);
  }
  if (field == ODGS_FRAME_TILE_ENTRIES) {
    const uint32_t K = f->n_entries;
    if ((st = need(sizeof(int32_t) * K)) != ODGS_OK) return st;
    std::vector<uint32_t> vals(K);
    if (K) ODGS_CUDA(ctx, cudaMemcpy(vals.data(), f->evals[f->tile_which].p, sizeof(uint32_t) * K, cudaMemcpyDeviceToHost));
    for (uint32_t e = 0; e < K; ++e)
      static_cast<int32_t*>(host_dst)[e] = inst_id[3 * (size_t)(vals[e] >> 2) + (vals[e] & 3u)];
    return ok(ctx);
  }
  return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "bad field");
}

odgs_status odgs_backward(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera, odgs_frame* f,
                          const float* dl_dimage, int32_t dl_memory, const odgs_settings* settings,
                          const odgs_grads* grads, const double* grad_t_signs, uint32_t flags) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!f || !f->rendered) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "backward: frame not rendered");
  if (!grads || !dl_dimage) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "backward: null buffers");
  odgs_status st;
  if ((st = check_camera(ctx, camera)) != ODGS_OK) return st;
  if ((st = check_settings(ctx, settings)) != ODGS_OK) return st;
  if (!cloud || cloud->n != f->n)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "backward: cloud does not match the frame");
  CloudPtrs cp;
  if ((st = resolve_cloud(ctx, cloud, &cp)) != ODGS_OK) return st;
  cudaStream_t s = ctx->stream;
  const int64_t n = f->n;

  const float* signs = ctx->d_unit_signs;
  if (grad_t_signs) {
    float sf[12];
    for (int k = 0; k < 12; ++k) sf[k] = (float)grad_t_signs[k];
    ODGS_CUDA(ctx, ensure(ctx->signs_buf, sizeof sf, s));
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->signs_buf.p, sf, sizeof sf, cudaMemcpyHostToDevice, s));
    ODGS_CUDA(ctx, cudaStreamSynchronize(s));
    signs = ctx->signs_buf.as<float>();
  }
  // Gradient destinations.
  const bool host_out = grads->memory != ODGS_MEM_DEVICE;
  float *gm = grads->means, *gq = grads->rotations, *gls = grads->log_scales, *gop = grads->raw_opacities,
        *gcol = grads->colors, *gpn = grads->pixel_grad_norm, *gomc = grads->one_minus_cos;
  int32_t* gobs = grads->observed;
  const int nb = cp.sh_degree > 0 ? sh_count(cp.sh_degree) : 0;
  if (nb > 0 && !grads->sh_rest)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "backward: sh_rest gradient buffer required for sh_degree > 0");
  float* gsh = grads->sh_rest;
  if (host_out && n > 0) {
    ODGS_CUDA(ctx, ensure(ctx->grads_buf, sizeof(float) * (17 + 3 * nb) * n, s));
    float* b = ctx->grads_buf.as<float>();
    if (nb > 0) {
      if (flags & ODGS_ACCUMULATE)
        ODGS_CUDA(ctx, cudaMemcpyAsync(b + 17 * n, grads->sh_rest, 4 * 3 * nb * n, cudaMemcpyHostToDevice, s));
      gsh = b + 17 * n;
    }
    float* dst[8] = {b, b + 3 * n, b + 7 * n, b + 10 * n, b + 11 * n, b + 14 * n, b + 15 * n, b + 16 * n};
    const void* src[8] = {gm, gq, gls, gop, gcol, gpn, gomc, gobs};
    const int64_t width[8] = {3, 4, 3, 1, 3, 1, 1, 1};
    for (int k = 0; k < 8; ++k) {
      if (!src[k] && k < 5) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "backward: null gradient buffer");
      if ((flags & ODGS_ACCUMULATE) && src[k])
        ODGS_CUDA(ctx, cudaMemcpyAsync(dst[k], src[k], 4 * width[k] * n, cudaMemcpyHostToDevice, s));
    }
    gm = dst[0]; gq = dst[1]; gls = dst[2]; gop = dst[3]; gcol = dst[4];
    gpn = gpn ? dst[5] : nullptr;
    gomc = gomc ? dst[6] : nullptr;
    gobs = gobs ? reinterpret_cast<int32_t*>(dst[7]) : nullptr;
  }
  const bool keep_sg = (f->flags & ODGS_FRAME_KEEP_SPLAT_GRADS) != 0;
  if (keep_sg) ODGS_CUDA(ctx, ensure(f->splat_grads, sizeof(float) * 10 * n, s));
  // The backward's error words live in the frame's sticky section: cleared here unless
  // an earlier operation on the frame is still unchecked (then they accumulate until the
  // check point).
  if (!f->pending && !f->bwd_pending) launch_reset_sticky(f->d_err, s);
  if ((st = raster_fold(ctx, f, dl_dimage, dl_memory, settings)) != ODGS_OK) return st;

  BwdSplatArgs sa;
  sa.n = n;
  sa.means = cp.means;
  sa.rotations = cp.rotations;
  sa.log_scales = cp.log_scales;
  sa.raw_opacities = cp.raw_opacities;
  sa.sh_degree = cp.sh_degree;
  sa.sh_rest = cp.sh_rest;
  sa.g_sh_rest = gsh;
  // The chain rule re-derives the projection from the camera and settings passed here,
  // as the reference's backward does (backward.hpp:393-410): the frame supplies only
  // the splats, tile lists and per-pixel state (also a frame of odgs_rasterize_splats).
  sa.cam = to_dev(*camera);
  sa.settings = to_dev(*settings);
  sa.settings.band_ty0 = f->settings.band_ty0;
  sa.settings.band_ty1 = f->settings.band_ty1;
  sa.sp_ab = f->sp_ab.as<float4>();
  sa.sp_c = f->sp_c.as<float4>();
  sa.cnt = f->cnt.as<uint32_t>();
  sa.folded = f->folded.as<float>();
  sa.signs = signs;
  sa.sec_max = 1.0f / std::cos(settings->max_elevation);
  sa.accumulate = (flags & ODGS_ACCUMULATE) ? 1 : 0;
  sa.g_means = gm;
  sa.g_rotations = gq;
  sa.g_log_scales = gls;
  sa.g_raw_opacities = gop;
  sa.g_colors = gcol;
  sa.g_pixel_grad_norm = gpn;
  sa.g_one_minus_cos = gomc;
  sa.g_observed = gobs;
  sa.splat_grads = keep_sg ? f->splat_grads.as<float>() : nullptr;
  sa.err = f->d_err;
  {
    StageScope sc(ctx, ODGS_STAGE_BWD_SPLAT);
    launch_bwd_splat(sa, s);
  }
  ODGS_CUDA(ctx, cudaGetLastError());
  f->have_splat_grads = keep_sg;

  if (host_out && n > 0) {
    float* b = ctx->grads_buf.as<float>();
    void* dsth[8] = {grads->means, grads->rotations, grads->log_scales, grads->raw_opacities, grads->colors,
                     grads->pixel_grad_norm, grads->one_minus_cos, grads->observed};
    const float* srcd[8] = {b, b + 3 * n, b + 7 * n, b + 10 * n, b + 11 * n, b + 14 * n, b + 15 * n, b + 16 * n};
    const int64_t width[8] = {3, 4, 3, 1, 3, 1, 1, 1};
    for (int k = 0; k < 8; ++k)
      if (dsth[k]) ODGS_CUDA(ctx, cudaMemcpyAsync(dsth[k], srcd[k], 4 * width[k] * n, cudaMemcpyDeviceToHost, s));
    if (nb > 0) ODGS_CUDA(ctx, cudaMemcpyAsync(grads->sh_rest, gsh, 4 * 3 * nb * n, cudaMemcpyDeviceToHost, s));
  }
  f->bwd_pending = true;
  if (ctx->timers.enabled) resolve_timers(ctx);
  // Asynchronous contexts report the errors at the frame's check point; host gradient
  // buffers are only complete after a synchronisation, so they always check here.
  if (ctx->async_mode && !host_out) return ok(ctx);
  if ((st = finish_frame(ctx, f)) != ODGS_OK) return st;
  return ok(ctx);
}

odgs_status odgs_grad_pixels_to_splats(odgs_ctx* ctx, odgs_frame* f, const float* dl_dimage, int32_t dl_memory,
                                       const odgs_settings* settings, float* pixel_mean, float* cov2d, float* opacity,
                                       float* color) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!f || !f->rendered) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "grad_pixels_to_splats: frame not rendered");
  if (!dl_dimage) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "grad_pixels_to_splats: null image gradient");
  odgs_status st;
  if ((st = check_settings(ctx, settings)) != ODGS_OK) return st;
  if ((st = finish_frame(ctx, f)) != ODGS_OK) return st;
  cudaStream_t s = ctx->stream;
  const int64_t n = f->n;
  ODGS_CUDA(ctx, ensure(f->splat_grads, sizeof(float) * 10 * n, s));
  if ((st = raster_fold(ctx, f, dl_dimage, dl_memory, settings)) != ODGS_OK) return st;
  launch_splat_grads(n, f->sp_ab.as<float4>(), f->sp_c.as<float4>(), f->cnt.as<uint32_t>(), f->folded.as<float>(),
                     f->splat_grads.as<float>(), s);
  ODGS_CUDA(ctx, cudaGetLastError());
  f->have_splat_grads = true;
  // Compact to splat order (RenderOutput::splats: projected Gaussians, ascending row).
  HostViews v;
  if ((st = load_views(ctx, f, &v)) != ODGS_OK) return st;
  std::vector<float> sg((size_t)n * 10);
  if (n) ODGS_CUDA(ctx, cudaMemcpy(sg.data(), f->splat_grads.p, sizeof(float) * 10 * n, cudaMemcpyDeviceToHost));
  for (size_t k = 0; k < v.visible.size(); ++k) {
    const float* r = sg.data() + (size_t)v.visible[k] * 10;
    if (pixel_mean) { pixel_mean[2 * k] = r[0]; pixel_mean[2 * k + 1] = r[1]; }
    if (cov2d) for (int c = 0; c < 4; ++c) cov2d[4 * k + c] = r[2 + c];
    if (opacity) opacity[k] = r[6];
    if (color) for (int c = 0; c < 3; ++c) color[3 * k + c] = r[7 + c];
  }
  if (ctx->timers.enabled) resolve_timers(ctx);
  return ok(ctx);
}

odgs_status odgs_project_gaussian(odgs_ctx* ctx, const odgs_cloud* cloud, int64_t index, const odgs_camera* camera,
                                  const odgs_settings* settings, odgs_splat* out, int32_t* projected) {
  LaunchScope scope(ctx);
  if (!ctx || !out || !projected) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  *projected = 0;
  odgs_status st;
  if ((st = check_settings(ctx, settings)) != ODGS_OK) return st;
  if (!camera || camera->width <= 0 || camera->height <= 0)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "project_gaussian: bad camera size");
  if (!cloud || cloud->sh_degree < 0 || cloud->sh_degree > 3 || (cloud->sh_degree > 0 && !cloud->sh_rest))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "project_gaussian: bad cloud");
  if (index < 0 || index >= cloud->n)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, index, "project_gaussian: index outside the cloud");
  const int nb = cloud->sh_degree > 0 ? sh_count(cloud->sh_degree) : 0;
  // Gather the row into a one-row cloud (means 3 | rotations 4 | log_scales 3 | opacity |
  // colors 3 | sh_rest 3 nb) next to the one-row outputs.
  const int row_len = 14 + 3 * nb;
  const int64_t n = cloud->n;
  const float* src[6] = {cloud->means, cloud->rotations, cloud->log_scales, cloud->raw_opacities, cloud->colors,
                         cloud->sh_rest};
  const int width[6] = {3, 4, 3, 1, 3, 3 * nb};
  cudaStream_t s = ctx->stream;
  constexpr size_t kOut = 256;  // sp_ab 32 | sp_c 16 | cov 16 | keys, vals, cnt
  ODGS_CUDA(ctx, ensure(ctx->misc_buf, kOut + sizeof(float) * row_len, s));
  char* base = ctx->misc_buf.as<char>();
  float* d_row = reinterpret_cast<float*>(base + kOut);
  std::vector<float> row((size_t)row_len);
  const bool dev = cloud->memory == ODGS_MEM_DEVICE;
  int off = 0;
  for (int g = 0; g < 6; ++g)
    for (int c = 0; c < width[g]; ++c, ++off) {
      const float* p = src[g] + (int64_t)c * n + index;
      if (dev) ODGS_CUDA(ctx, cudaMemcpyAsync(d_row + off, p, sizeof(float), cudaMemcpyDeviceToDevice, s));
      else row[(size_t)off] = *p;
    }
  if (!dev) ODGS_CUDA(ctx, cudaMemcpyAsync(d_row, row.data(), sizeof(float) * row_len, cudaMemcpyHostToDevice, s));
  if ((st = reset_errors(ctx)) != ODGS_OK) return st;
  float4* d_ab = reinterpret_cast<float4*>(base);
  float4* d_c = reinterpret_cast<float4*>(base + 32);
  float4* d_cov = reinterpret_cast<float4*>(base + 48);
  uint32_t* d_u = reinterpret_cast<uint32_t*>(base + 64);
  DevSettings ds = to_dev(*settings);
  ds.tile_size = 1;  // tile counts are not needed
  launch_project_one(d_row, cloud->sh_degree, to_dev(*camera), ds, d_ab, d_c, d_cov, d_u, d_u + 1, d_u + 2, ctx->d_err, s);
  float4 h[4];
  ODGS_CUDA(ctx, cudaMemcpyAsync(h, base, sizeof h, cudaMemcpyDeviceToHost, s));
  if ((st = read_errors(ctx)) != ODGS_OK) return st;
  const DevErrors& he = *ctx->h_err;
  if (he.project != kNoError) {
    const int code = (int)(he.project & 15);
    if (code == 3) return set_error(ctx, ODGS_ERR_DOMAIN, index, "to_spherical: degenerate zero-length direction");
    if (code == 2) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, index, "build_covariance: non-finite parameters");
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, index, "normalize_quaternion: near-zero quaternion");
  }
  const uint32_t flags = flags_of(h[2]);
  if (!(flags & kFlagVisible)) return ok(ctx);  // std::nullopt
  out->pixel_mean[0] = h[0].x; out->pixel_mean[1] = h[0].y;
  out->cov2d[0] = h[3].x; out->cov2d[1] = h[3].y; out->cov2d[2] = h[3].z; out->cov2d[3] = h[3].w;
  out->cov2d_inv[0] = h[0].z; out->cov2d_inv[1] = h[0].w; out->cov2d_inv[2] = h[0].w; out->cov2d_inv[3] = h[1].x;
  out->depth = h[2].y;
  out->radius = h[2].z;
  out->opacity = h[1].y;
  out->color[0] = h[1].z; out->color[1] = h[1].w; out->color[2] = h[2].x;
  out->index = index;
  out->pole_clamped = (flags & kFlagClamped) ? 1 : 0;
  *projected = 1;
  return ok(ctx);
}

namespace {
odgs_status loss_impl(odgs_ctx* ctx, const float* rendered, const float* target, int32_t width, int32_t height,
                      float lambda_ssim, float* dl_dimage, double* loss, double* device_accum) {
  if (!ctx || !rendered || !target || !dl_dimage) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!(lambda_ssim >= 0.0f) || !(lambda_ssim < 1.0f))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "photometric_loss: lambda must be in [0, 1)");
  if (width <= 0 || height <= 0) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "photometric_loss: bad size");
  const int64_t count = 3 * (int64_t)width * height;
  if (lambda_ssim > 0.0f) {
    if (width < 11 || height < 11)
      return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "ssim: images smaller than the 11x11 window");
    ODGS_CUDA(ctx, ensure(ctx->loss_buf, ssim_temp_bytes(height, width) + 64, ctx->stream));
    char* base = ctx->loss_buf.as<char>();
    launch_ssim_loss(rendered, target, height, width, lambda_ssim, dl_dimage, base + 64,
                     reinterpret_cast<double*>(base), device_accum, ctx->stream);
  } else {
    ODGS_CUDA(ctx, ensure(ctx->loss_buf, l1_loss_temp_bytes(count), ctx->stream));
    launch_l1_loss(rendered, target, count, lambda_ssim, dl_dimage, ctx->loss_buf.as<double>(), device_accum,
                   ctx->stream);
  }
  ODGS_CUDA(ctx, cudaGetLastError());
  if (loss) {
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->h_scratch, ctx->loss_buf.p, sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx->stream));
    ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(loss, ctx->h_scratch, sizeof(double));
  }
  return ok(ctx);
}
}  // namespace

odgs_status odgs_photometric_loss(odgs_ctx* ctx, const float* rendered, const float* target, int32_t width,
                                  int32_t height, float lambda_ssim, float* dl_dimage, double* loss) {
  LaunchScope scope(ctx);
  return loss_impl(ctx, rendered, target, width, height, lambda_ssim, dl_dimage, loss, nullptr);
}

odgs_status odgs_photometric_loss_async(odgs_ctx* ctx, const float* rendered, const float* target, int32_t width,
                                        int32_t height, float lambda_ssim, float* dl_dimage, double* device_loss_sum) {
  LaunchScope scope(ctx);
  return loss_impl(ctx, rendered, target, width, height, lambda_ssim, dl_dimage, nullptr, device_loss_sum);
}

odgs_status odgs_adam_step(odgs_ctx* ctx, const odgs_params* p, const odgs_grads* g, const odgs_train_state* st,
                           const odgs_adam_params* ap) {
  LaunchScope scope(ctx);
  if (!ctx || !p || !g || !st || !ap) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (ap->step < 1) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "adam_step: step must be >= 1");
  if (g->memory != ODGS_MEM_DEVICE)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "adam_step: gradients must be device buffers");
  AdamArgs a;
  a.n = p->n;
  a.means = p->means; a.rotations = p->rotations; a.log_scales = p->log_scales;
  a.raw_opacities = p->raw_opacities; a.colors = p->colors;
  a.means_m = st->means_m; a.means_v = st->means_v; a.rot_m = st->rot_m; a.rot_v = st->rot_v;
  a.scale_m = st->scale_m; a.scale_v = st->scale_v; a.opac_m = st->opac_m; a.opac_v = st->opac_v;
  a.color_m = st->color_m; a.color_v = st->color_v;
  a.grad_accum = st->grad_accum; a.elev_accum = st->elev_accum; a.grad_count = st->grad_count;
  a.g_means = g->means; a.g_rotations = g->rotations; a.g_log_scales = g->log_scales;
  a.g_raw_opacities = g->raw_opacities; a.g_colors = g->colors; a.g_pixel_grad_norm = g->pixel_grad_norm;
  a.g_one_minus_cos = g->one_minus_cos; a.g_observed = g->observed;
  if ((a.grad_accum && !a.g_pixel_grad_norm) || (a.elev_accum && !a.g_one_minus_cos) || (a.grad_count && !a.g_observed))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "adam_step: densify window needs the statistics");
  a.lr_means = ap->lr_means; a.lr_rotation = ap->lr_rotation; a.lr_scale = ap->lr_scale;
  a.lr_opacity = ap->lr_opacity; a.lr_color = ap->lr_color;
  // c = 1 - pow(b, step) in Scalar, as adam_update computes it (optimizer.hpp:80-81).
  a.c1 = 1.0f - std::pow(0.9f, (float)ap->step);
  a.c2 = 1.0f - std::pow(0.999f, (float)ap->step);
  launch_adam(a, ctx->stream);
  ODGS_CUDA(ctx, cudaGetLastError());
  return ok(ctx);
}

odgs_status odgs_ctx_set_profiling(odgs_ctx* ctx, int enable) {
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  resolve_timers(ctx);
  ctx->timers.enabled = enable != 0;
  return ok(ctx);
}

int odgs_ctx_stage_times(odgs_ctx* ctx, double* ms, int64_t* calls, int max_stages) {
  if (!ctx) return 0;
  resolve_timers(ctx);
  const int n = std::min(max_stages, (int)ODGS_STAGE_COUNT);
  for (int k = 0; k < n; ++k) {
    if (ms) ms[k] = ctx->timers.ms[k];
    if (calls) calls[k] = ctx->timers.calls[k];
  }
  return n;
}

void odgs_ctx_reset_stage_times(odgs_ctx* ctx) {
  if (!ctx) return;
  resolve_timers(ctx);
  for (int k = 0; k < ODGS_STAGE_COUNT; ++k) {
    ctx->timers.ms[k] = 0;
    ctx->timers.calls[k] = 0;
  }
}

const char* odgs_stage_name(int stage) {
  static const char* names[ODGS_STAGE_COUNT] = {"preprocess", "depth_sort", "scan", "emit", "tile_sort",
                                                "ranges", "blend", "bwd_raster", "bwd_splat"};
  return (stage >= 0 && stage < ODGS_STAGE_COUNT) ? names[stage] : "unknown";
}

odgs_status odgs_measure_fp32_tflops(odgs_ctx* ctx, double* tflops) {
  LaunchScope scope(ctx);
  if (!ctx || !tflops) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  int sms = 0;
  ODGS_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  DevBuf sink;
  ODGS_CUDA(ctx, ensure(sink, sizeof(float) * 1024 * 1024, ctx->stream));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  const int blocks = sms * 8, threads = 256;
  launch_fp32_peak(blocks, threads, iters, sink.as<float>(), ctx->stream);  // warm-up
  cudaEventRecord(a, ctx->stream);
  launch_fp32_peak(blocks, threads, iters, sink.as<float>(), ctx->stream);
  cudaEventRecord(b, ctx->stream);
  ODGS_CUDA(ctx, cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  release(sink, ctx->stream);
  // fp32_peak_flops_per_thread(iters) FMAs x 2 flops per thread.
  const double flops = (double)blocks * threads * fp32_peak_flops_per_thread(iters);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return ok(ctx);
}

odgs_status odgs_cull(odgs_ctx* ctx, const odgs_cloud* cloud, const odgs_camera* camera, float near_radius,
                      float far_radius, int64_t* out_indices, int64_t* out_count) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!(0.0f < near_radius && near_radius < far_radius))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "cull: need 0 < near < far");
  if (!camera || !out_count) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "cull: null argument");
  CloudPtrs cp;
  odgs_status st;
  if ((st = resolve_cloud(ctx, cloud, &cp)) != ODGS_OK) return st;
  const int64_t n = cloud->n;
  *out_count = 0;
  if (n == 0) return ok(ctx);
  ODGS_CUDA(ctx, ensure(ctx->cull_buf, n, ctx->stream));
  launch_cull(n, cp.means, to_dev(*camera), near_radius, far_radius, ctx->cull_buf.as<uint8_t>(), ctx->stream);
  std::vector<uint8_t> keep(n);
  ODGS_CUDA(ctx, cudaMemcpyAsync(keep.data(), ctx->cull_buf.p, n, cudaMemcpyDeviceToHost, ctx->stream));
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i)
    if (keep[i]) {
      if (out_indices) out_indices[c] = i;
      ++c;
    }
  *out_count = c;
  return ok(ctx);
}

// ------------------------------------------------------------------ init_from_points
namespace {

// Grid plan: the largest cell size h whose grid has at most `target` cells
// (dims_a = max(1, ceil(extent_a / h))), so cells hold ~2 points on average.
KnnGrid plan_grid(const double lo[3], const double hi[3], int64_t n_finite) {
  KnnGrid g{};
  for (int a = 0; a < 3; ++a) g.lo[a] = lo[a];
  double ext[3], emax = 0.0;
  for (int a = 0; a < 3; ++a) {
    ext[a] = hi[a] - lo[a];
    emax = std::max(emax, ext[a]);
  }
  const double target = (double)std::min<int64_t>(std::max<int64_t>(n_finite / 2, 1), (int64_t)1 << 26);
  auto cells = [&](double h) {
    double c = 1.0;
    for (int a = 0; a < 3; ++a) c *= std::max(1.0, std::ceil(ext[a] / h));
    return c;
  };
  if (!(emax > 0.0) || !std::isfinite(emax) || target <= 1.0) {
    g.h = 1.0;
    g.dims[0] = g.dims[1] = g.dims[2] = 1;
  } else {
    double lo_h = emax / std::cbrt(target) / 4.0, hi_h = emax;  // cells(hi_h) == 1 <= target
    while (cells(lo_h) <= target) lo_h /= 2.0;
    for (int it = 0; it < 64; ++it) {
      const double mid = std::sqrt(lo_h * hi_h);
      if (cells(mid) <= target) hi_h = mid;
      else lo_h = mid;
    }
    g.h = hi_h;
    for (int a = 0; a < 3; ++a) g.dims[a] = (int)std::max(1.0, std::ceil(ext[a] / g.h));
  }
  g.n_cells = (uint32_t)((uint64_t)g.dims[0] * g.dims[1] * g.dims[2]);
  return g;
}

}  // namespace

odgs_status odgs_init_from_points(odgs_ctx* ctx, int64_t n, const double* positions, const double* colors,
                                  int32_t memory, const odgs_cloud64* out, double* nn_scale) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (n < 1) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "init_from_points: no points");
  if (!positions || !colors || !out || !out->means || !out->rotations || !out->log_scales || !out->raw_opacities ||
      !out->colors)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "init_from_points: null argument");
  if (out->n != n) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "init_from_points: out->n != n");
  if (n >= ((int64_t)1 << 32) - 1)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "init_from_points: more than 2^32 - 2 points");
  const bool host = memory == ODGS_MEM_HOST;
  cudaStream_t s = ctx->stream;
  const size_t n3 = 3 * (size_t)n;

  // Scratch: positions (host input), keys/indices ping-pong, sorted xyz, log-scales.
  DevBuf pos_b, k0, k1, v0, v1, xyz_b, cells_b, part_b, ls_b, sc_b, tmp_b;
  struct Release {
    std::vector<DevBuf*> bufs;
    cudaStream_t s;
    ~Release() {
      for (DevBuf* b : bufs) release(*b, s);
    }
  } rel{{&pos_b, &k0, &k1, &v0, &v1, &xyz_b, &cells_b, &part_b, &ls_b, &sc_b, &tmp_b}, s};
  const double* dpos = positions;
  if (host) {
    ODGS_CUDA(ctx, ensure(pos_b, sizeof(double) * n3, s));
    ODGS_CUDA(ctx, cudaMemcpyAsync(pos_b.p, positions, sizeof(double) * n3, cudaMemcpyHostToDevice, s));
    dpos = pos_b.as<double>();
  }
  // 1. bounding box of the finite points
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1184);
  ODGS_CUDA(ctx, ensure(part_b, sizeof(double) * 6 * blocks + 64, s));
  unsigned long long* d_count = reinterpret_cast<unsigned long long*>(part_b.as<char>() + sizeof(double) * 6 * blocks);
  ODGS_CUDA(ctx, cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  launch_bbox_partial(n, dpos, part_b.as<double>(), blocks, d_count, s);
  std::vector<double> part(6 * (size_t)blocks + 8);
  ODGS_CUDA(ctx, cudaMemcpyAsync(part.data(), part_b.p, sizeof(double) * 6 * blocks + 8, cudaMemcpyDeviceToHost, s));
  ODGS_CUDA(ctx, cudaStreamSynchronize(s));
  unsigned long long m_u = 0;
  std::memcpy(&m_u, part.data() + 6 * blocks, 8);
  const int64_t m = (int64_t)m_u;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (m > 0) {
    for (int a = 0; a < 3; ++a) {
      lo[a] = part[a];
      hi[a] = part[3 + a];
      for (int b = 1; b < blocks; ++b) {
        lo[a] = std::min(lo[a], part[6 * b + a]);
        hi[a] = std::max(hi[a], part[6 * b + 3 + a]);
      }
    }
  }
  const KnnGrid g = plan_grid(lo, hi, m);

  // 2. cell keys, stable sort by cell, positions in cell order, cell CSR
  for (DevBuf* b : {&k0, &k1, &v0, &v1}) ODGS_CUDA(ctx, ensure(*b, sizeof(uint32_t) * n, s));
  ODGS_CUDA(ctx, ensure(tmp_b, std::max(radix_sort_temp_bytes(n), (size_t)16), s));
  ODGS_CUDA(ctx, ensure(xyz_b, sizeof(double) * n3, s));
  ODGS_CUDA(ctx, ensure(cells_b, sizeof(uint32_t) * ((size_t)g.n_cells + 1), s));
  launch_cell_keys(n, dpos, g, k0.as<uint32_t>(), v0.as<uint32_t>(), s);
  uint32_t* kk[2] = {k0.as<uint32_t>(), k1.as<uint32_t>()};
  uint32_t* vv[2] = {v0.as<uint32_t>(), v1.as<uint32_t>()};
  int which = 0;
  ODGS_CUDA(ctx, radix_sort_pairs(kk, vv, n, 0, bits_for(g.n_cells + 1u), tmp_b.p, &which, s));
  launch_gather_xyz(n, vv[which], dpos, xyz_b.as<double>(), s);
  launch_cell_ranges(m, kk[which], g.n_cells, cells_b.as<uint32_t>(), s);

  // 3. exact 3-NN and the log-scales
  double* d_ls = out->log_scales;
  double* d_sc = nn_scale;
  if (host) {
    ODGS_CUDA(ctx, ensure(ls_b, sizeof(double) * n3, s));
    d_ls = ls_b.as<double>();
    if (nn_scale) {
      ODGS_CUDA(ctx, ensure(sc_b, sizeof(double) * n, s));
      d_sc = sc_b.as<double>();
    }
  }
  launch_knn_query(n, m, xyz_b.as<double>(), vv[which], cells_b.as<uint32_t>(), g, d_sc, d_ls, s);

  // 4. the other fields (io.cpp:263-267): means and colours copied, identity
  //    rotations, raw opacity logit(0.1) (types.hpp:35-39, binary64 on the host).
  const double raw = std::log(0.1 / (1.0 - 0.1));
  if (host) {
    std::memcpy(out->means, positions, sizeof(double) * n3);
    std::memcpy(out->colors, colors, sizeof(double) * n3);
    for (int64_t i = 0; i < n; ++i) {
      out->rotations[i] = 1.0;
      out->raw_opacities[i] = raw;
    }
    std::fill(out->rotations + n, out->rotations + 4 * n, 0.0);
    ODGS_CUDA(ctx, cudaMemcpyAsync(out->log_scales, d_ls, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    if (nn_scale) ODGS_CUDA(ctx, cudaMemcpyAsync(nn_scale, d_sc, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  } else {
    ODGS_CUDA(ctx, cudaMemcpyAsync(out->means, positions, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
    ODGS_CUDA(ctx, cudaMemcpyAsync(out->colors, colors, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
    launch_fill_f64(out->rotations, n, 1.0, s);
    ODGS_CUDA(ctx, cudaMemsetAsync(out->rotations + n, 0, sizeof(double) * n3, s));
    launch_fill_f64(out->raw_opacities, n, raw, s);
  }
  ODGS_CUDA(ctx, cudaStreamSynchronize(s));
  ODGS_CUDA(ctx, cudaGetLastError());
  return ok(ctx);
}

// ------------------------------------------------------------------ density control
void odgs_default_densify_config(odgs_densify_config* out) {  // densify.hpp:16-24
  if (!out) return;
  out->grad_threshold_min = 2e-5;
  out->grad_threshold_max = 1e-4;
  out->percent_dense = 1e-3;
  out->opacity_prune_floor = 0.005;
  out->split_scale_divisor = 1.6;
}

struct odgs_rng {
  std::mt19937 gen;
};

odgs_rng* odgs_rng_create(uint32_t seed) { return new (std::nothrow) odgs_rng{std::mt19937(seed)}; }
void odgs_rng_destroy(odgs_rng* rng) { delete rng; }
uint32_t odgs_rng_next(odgs_rng* rng) { return rng ? (uint32_t)rng->gen() : 0u; }

void odgs_rng_unit_ball(odgs_rng* rng, int64_t count, float* out) {
  if (!rng || !out) return;
  for (int64_t k = 0; k < count; ++k) {
    // densify.hpp:61-69: one normal_distribution per sample (its cached polar value
    // lives across rejected tries only); Vec3(g(), g(), g()) evaluates right to left
    // under GCC, so the first draw is z. Norm in float, Eigen's order x² + (y² + z²).
    std::normal_distribution<double> gauss;
    for (;;) {
      const float z = (float)gauss(rng->gen);
      const float y = (float)gauss(rng->gen);
      const float x = (float)gauss(rng->gen);
      const float yy = y * y, zz = z * z, xx = x * x;
      if (std::sqrt(xx + (yy + zz)) <= 1.0f) {
        out[3 * k] = x;
        out[3 * k + 1] = y;
        out[3 * k + 2] = z;
        break;
      }
    }
  }
}

namespace {
odgs_status check_densify_config(odgs_ctx* ctx, const odgs_densify_config* c) {  // densify.hpp:26-32
  if (!c) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify: null config");
  if (!(c->grad_threshold_min > 0) || !(c->grad_threshold_max >= c->grad_threshold_min))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1,
                     "DensifyConfig: need 0 < grad_threshold_min <= grad_threshold_max");
  if (!(c->percent_dense > 0) || !(c->percent_dense < 1))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "DensifyConfig: percent_dense outside (0, 1)");
  return ODGS_OK;
}
size_t align256(size_t b) { return (b + 255) / 256 * 256; }
}  // namespace

odgs_status odgs_densify_plan(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                              const odgs_densify_config* cfg, float scene_extent, odgs_densify_stats* stats) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  ctx->plan.valid = false;
  odgs_status st;
  if ((st = check_densify_config(ctx, cfg)) != ODGS_OK) return st;
  if (!(scene_extent > 0.0f))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_and_prune: scene extent must be positive");
  if (!cloud || !state || !stats || cloud->n < 0 || cloud->n >= (int64_t)1 << 31)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_and_prune: bad arguments");
  const int64_t n = cloud->n;
  if (n > 0 && (!cloud->means || !cloud->rotations || !cloud->log_scales || !cloud->raw_opacities ||
                !cloud->colors || !state->grad_accum || !state->elev_accum || !state->grad_count))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_and_prune: null buffer");
  const size_t arr = align256((size_t)n * 4);
  ODGS_CUDA(ctx, ensure(ctx->densify_buf, 256 + 6 * arr + scan_temp_bytes(n), ctx->stream));
  char* base = ctx->densify_buf.as<char>();
  auto* counters = reinterpret_cast<unsigned long long*>(base);  // [0..2] counts, [3..5] totals, [6] bad
  uint32_t* u[6];
  for (int k = 0; k < 6; ++k) u[k] = reinterpret_cast<uint32_t*>(base + 256 + k * arr);
  void* scan_tmp = base + 256 + 6 * arr;
  ODGS_CUDA(ctx, cudaMemsetAsync(counters, 0, 6 * sizeof(unsigned long long), ctx->stream));
  ODGS_CUDA(ctx, cudaMemsetAsync(counters + 6, 0xff, sizeof(unsigned long long), ctx->stream));
  DensifyArgs a;
  a.n = n;
  a.rotations = cloud->rotations; a.log_scales = cloud->log_scales; a.raw_opacities = cloud->raw_opacities;
  a.grad_accum = state->grad_accum; a.elev_accum = state->elev_accum; a.grad_count = state->grad_count;
  a.tmin = (float)cfg->grad_threshold_min;  // Scalar(cfg.*) (densify.hpp:92-94)
  a.tmax = (float)cfg->grad_threshold_max;
  a.size_split = (float)cfg->percent_dense * scene_extent;
  a.prune_floor = (float)cfg->opacity_prune_floor;
  a.keep_self = u[0]; a.added_kept = u[1]; a.split_flag = u[2];
  a.counters = counters;
  a.bad_quaternion = counters + 6;
  launch_densify_classify(a, ctx->stream);
  for (int k = 0; k < 3; ++k) exclusive_scan_u32(u[k], u[3 + k], n, scan_tmp, counters + 3 + k, ctx->stream);
  ODGS_CUDA(ctx, cudaGetLastError());
  ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->h_scratch, counters, 7 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  unsigned long long h[7];
  std::memcpy(h, ctx->h_scratch, sizeof h);
  if (h[6] != kNoError)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, (int64_t)h[6], "normalize_quaternion: near-zero quaternion");
  stats->cloned = (int64_t)h[0];
  stats->split = (int64_t)h[1];
  stats->pruned = (int64_t)h[2];
  stats->n_out = (int64_t)(h[3] + h[4]);
  ctx->plan.valid = true;
  ctx->plan.n = n;
  ctx->plan.split = (int64_t)h[5];
  ctx->plan.n_out = stats->n_out;
  ctx->plan.key = cloud->means;
  ctx->plan.total_a = (uint32_t)h[3];
  ctx->plan.log_shrink = pm_logf((float)cfg->split_scale_divisor);  // std::log(Scalar(divisor))
  return ok(ctx);
}

odgs_status odgs_densify_apply(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                               const float* unit_ball, const odgs_params* out_cloud,
                               const odgs_train_state* out_state) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!cloud || !state || !out_cloud || !out_state || !ctx->plan.valid || ctx->plan.n != cloud->n ||
      ctx->plan.key != cloud->means)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_apply: no matching odgs_densify_plan");
  const int64_t n = cloud->n, m = ctx->plan.n_out;
  if (out_cloud->n != m)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_apply: out_cloud->n must equal stats.n_out");
  if (ctx->plan.split > 0 && !unit_ball)
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_apply: unit_ball samples required");
  const float* const mom_in[10] = {state->means_m, state->means_v, state->rot_m, state->rot_v, state->scale_m,
                                   state->scale_v, state->opac_m, state->opac_v, state->color_m, state->color_v};
  float* const mom_out[10] = {out_state->means_m, out_state->means_v, out_state->rot_m, out_state->rot_v,
                              out_state->scale_m, out_state->scale_v, out_state->opac_m, out_state->opac_v,
                              out_state->color_m, out_state->color_v};
  if (m > 0) {
    bool okp = out_cloud->means && out_cloud->rotations && out_cloud->log_scales && out_cloud->raw_opacities &&
               out_cloud->colors;
    for (int k = 0; k < 10; ++k) okp = okp && mom_in[k] && mom_out[k];
    if (!okp) return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "densify_apply: null buffer");
    if (out_state->grad_accum) ODGS_CUDA(ctx, cudaMemsetAsync(out_state->grad_accum, 0, m * 4, ctx->stream));
    if (out_state->elev_accum) ODGS_CUDA(ctx, cudaMemsetAsync(out_state->elev_accum, 0, m * 4, ctx->stream));
    if (out_state->grad_count) ODGS_CUDA(ctx, cudaMemsetAsync(out_state->grad_count, 0, m * 4, ctx->stream));
  }
  const float* d_ball = nullptr;
  if (ctx->plan.split > 0) {
    const size_t bytes = (size_t)ctx->plan.split * 6 * sizeof(float);
    ODGS_CUDA(ctx, ensure(ctx->unit_ball_buf, bytes, ctx->stream));
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->unit_ball_buf.p, unit_ball, bytes, cudaMemcpyHostToDevice, ctx->stream));
    d_ball = ctx->unit_ball_buf.as<float>();
  }
  const size_t arr = align256((size_t)n * 4);
  char* base = ctx->densify_buf.as<char>();
  uint32_t* u[6];
  for (int k = 0; k < 6; ++k) u[k] = reinterpret_cast<uint32_t*>(base + 256 + k * arr);
  DensifyApplyArgs a;
  a.n = n;
  a.m = m;
  a.means = cloud->means; a.rotations = cloud->rotations; a.log_scales = cloud->log_scales;
  a.raw_opacities = cloud->raw_opacities; a.colors = cloud->colors;
  for (int k = 0; k < 10; ++k) { a.moments[k] = mom_in[k]; a.out_moments[k] = mom_out[k]; }
  a.out_means = out_cloud->means; a.out_rotations = out_cloud->rotations; a.out_log_scales = out_cloud->log_scales;
  a.out_raw_opacities = out_cloud->raw_opacities; a.out_colors = out_cloud->colors;
  a.keep_self = u[0]; a.added_kept = u[1]; a.split_flag = u[2];
  a.off_a = u[3]; a.off_b = u[4]; a.off_c = u[5];
  a.total_a = ctx->plan.total_a;
  a.unit_ball = d_ball;
  a.log_shrink = ctx->plan.log_shrink;
  launch_densify_apply(a, ctx->stream);
  ODGS_CUDA(ctx, cudaGetLastError());
  ctx->plan.valid = false;
  return ok(ctx);
}

odgs_status odgs_reset_opacity(odgs_ctx* ctx, const odgs_params* cloud, const odgs_train_state* state,
                               float ceiling) {
  LaunchScope scope(ctx);
  if (!ctx) return ODGS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (!cloud || cloud->n < 0 || (cloud->n > 0 && !cloud->raw_opacities))
    return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, -1, "reset_opacity: bad arguments");
  const int64_t n = cloud->n;
  if (n > 0) {
    ODGS_CUDA(ctx, ensure(ctx->misc_buf, 256, ctx->stream));
    auto* bad = ctx->misc_buf.as<unsigned long long>();
    ODGS_CUDA(ctx, cudaMemsetAsync(bad, 0xff, sizeof *bad, ctx->stream));
    launch_reset_opacity(cloud->raw_opacities, n, ceiling, bad, ctx->stream);
    ODGS_CUDA(ctx, cudaGetLastError());
    ODGS_CUDA(ctx, cudaMemcpyAsync(ctx->h_scratch, bad, sizeof *bad, cudaMemcpyDeviceToHost, ctx->stream));
    ODGS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    unsigned long long hb;
    std::memcpy(&hb, ctx->h_scratch, sizeof hb);
    if (hb != kNoError)
      return set_error(ctx, ODGS_ERR_INVALID_ARGUMENT, (int64_t)hb, "logit: argument must lie in (0, 1)");
  }
  if (state && n > 0) {  // densify.hpp:164-165
    if (state->opac_m) ODGS_CUDA(ctx, cudaMemsetAsync(state->opac_m, 0, n * 4, ctx->stream));
    if (state->opac_v) ODGS_CUDA(ctx, cudaMemsetAsync(state->opac_v, 0, n * 4, ctx->stream));
  }
  return ok(ctx);
}

odgs_status odgs_dynamic_threshold(double elevation, const odgs_densify_config* cfg, double* out) {
  if (!cfg || !out) return ODGS_ERR_INVALID_ARGUMENT;
  const double pi = 3.141592653589793238462643383279502884;
  if (!(std::abs(elevation) <= pi / 2 + 1e-12)) return ODGS_ERR_DOMAIN;
  const double tmin = cfg->grad_threshold_min, tmax = cfg->grad_threshold_max;
  *out = std::fma(1.0 - std::cos(elevation), tmax - tmin, tmin);
  return ODGS_OK;
}


}  // extern "C"
