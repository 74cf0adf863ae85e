// odgs_b200.hpp — C++ drop-in wrapper over the C ABI (odgs_b200.h).
//
// The reference's hot-path entry points (proj/include/odgs/rasterizer.hpp,
// backward.hpp, projection.hpp) take its own types: GaussianCloud<S>, CameraPose<S>,
// RenderSettings<S>, ErpImage<S>, RenderOutput<S>, GradBuffers<S>, Splat2D<S>,
// SplatGrads<S> (Eigen-backed, column-major). The functions below are templates over
// those types — they only use the members the reference declares (means / rotations /
// log_scales / raw_opacities / colors with .data() and .rows(); rotation(r, c),
// translation[k], width, height; the RenderSettings fields; channel[c].data();
// resize() / init()) — so in a reference build
//
//     odgs_b200::Context gpu;                                            // one per host thread
//     auto out  = odgs_b200::render<odgs::RenderOutput<float>>(gpu, cloud, camera, settings);
//     auto grad = odgs_b200::backward<odgs::GradBuffers<float>>(gpu, cloud, camera, out, dl, settings);
//
// replaces odgs::render / odgs::backward for Scalar = float, with the same exceptions
// (std::invalid_argument, std::runtime_error naming the Gaussian, std::domain_error).
// odgs_b200_dropin.hpp adds non-template float overloads in namespace odgs, so the
// reference's own call sites (odgs::render(cloud, camera, settings), train_step, ...)
// resolve to the GPU unchanged.
//
// Frames: the GPU keeps the last few rendered frames resident (Context(frames = 2)),
// each bound to the RenderOutput it was downloaded into. backward(fwd) uses fwd's own
// frame — never "the last render" — and if that frame was recycled (or fwd is a copy)
// it rebuilds it from fwd.splats (odgs_rasterize_splats: same instances, tile lists and
// per-pixel state bit for bit) and checks the rebuilt tile CSR and walk lengths against
// fwd's, throwing std::invalid_argument when fwd does not match its own splats.
// Eigen is not needed to compile this header.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "odgs_b200.h"

namespace odgs_b200 {

[[noreturn]] inline void throw_status(odgs_status st, const std::string& msg) {
  switch (st) {
    case ODGS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ODGS_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// Identity of a downloaded RenderOutput: its vectors' heap buffers (stable when the
// object is moved, distinct between live objects), their sizes, and a hash of the tile
// CSR (guards against a freed buffer's address being reused).
struct FrameKey {
  const void* entries = nullptr;
  const void* splats = nullptr;
  size_t n_entries = 0, n_splats = 0;
  uint64_t offsets_hash = 0;
  bool operator==(const FrameKey& o) const {
    return entries == o.entries && splats == o.splats && n_entries == o.n_entries && n_splats == o.n_splats &&
           offsets_hash == o.offsets_hash;
  }
};

inline uint64_t fnv1a(const void* p, size_t bytes) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t k = 0; k < bytes; ++k) h = (h ^ c[k]) * 1099511628211ull;
  return h;
}

template <class Output> FrameKey key_of(const Output& out) {
  FrameKey k;
  k.entries = out.tile_entries.data();
  k.splats = out.splats.data();
  k.n_entries = out.tile_entries.size();
  k.n_splats = out.splats.size();
  k.offsets_hash = fnv1a(out.tile_offsets.data(), out.tile_offsets.size() * sizeof(out.tile_offsets[0]));
  return k;
}

class Context {
 public:
  // frames: resident rendered frames kept for backward (least recently used recycled).
  explicit Context(int device = 0, void* stream = nullptr, int frames = 2) {
    const odgs_status st = odgs_ctx_create(device, stream, &ctx_);
    if (st != ODGS_OK) throw_status(st, "odgs_ctx_create failed");
    slots_.resize(frames > 0 ? (size_t)frames : 1);
  }
  ~Context() {
    for (auto& s : slots_)
      if (s.frame) odgs_frame_destroy(s.frame);
    odgs_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  odgs_ctx* get() const { return ctx_; }
  void check(odgs_status st) const {
    if (st == ODGS_OK) return;
    char msg[512];
    int64_t idx = -1;
    odgs_last_error(ctx_, &idx, msg, sizeof msg);
    throw_status(st, msg);
  }

  // A frame for a new render: the least recently used slot, unbound.
  odgs_frame* acquire() {
    Slot* v = &slots_[0];
    for (auto& s : slots_)
      if (!s.frame || s.stamp < v->stamp) v = &s;
    if (!v->frame) {
      check(odgs_frame_create(ctx_, &v->frame));
      check(odgs_frame_set_flags(v->frame, ODGS_FRAME_KEEP_COV2D));
    }
    v->bound = false;
    v->stamp = ++clock_;
    return v->frame;
  }
  void bind(odgs_frame* f, const FrameKey& key) {
    for (auto& s : slots_)
      if (s.frame == f) {
        s.key = key;
        s.bound = true;
      }
  }
  odgs_frame* find(const FrameKey& key) {
    for (auto& s : slots_)
      if (s.bound && s.key == key) {
        s.stamp = ++clock_;
        return s.frame;
      }
    return nullptr;
  }
  // Number of frames rebuilt from RenderOutput::splats (fwd not resident).
  int64_t rebuilds() const { return rebuilds_; }
  void count_rebuild() { ++rebuilds_; }

 private:
  struct Slot {
    odgs_frame* frame = nullptr;
    FrameKey key;
    bool bound = false;
    uint64_t stamp = 0;
  };
  odgs_ctx* ctx_ = nullptr;
  std::vector<Slot> slots_;
  uint64_t clock_ = 0;
  int64_t rebuilds_ = 0;
};

// The calling thread's context (device $ODGS_B200_DEVICE, default 0) for the float
// overloads of odgs_b200_dropin.hpp.
inline Context& thread_context() {
  thread_local Context ctx([] {
    const char* d = std::getenv("ODGS_B200_DEVICE");
    return d ? std::atoi(d) : 0;
  }());
  return ctx;
}

namespace detail {

template <class Settings> odgs_settings to_c(const Settings& s) {
  odgs_settings o;
  o.near_radius = (float)s.near_radius;
  o.far_radius = (float)s.far_radius;
  o.tile_size = s.tile_size;
  o.alpha_clamp = (float)s.alpha_clamp;
  o.transmittance_floor = (float)s.transmittance_floor;
  o.cutoff_sigma = (float)s.cutoff_sigma;
  o.lowpass_dilation = (float)s.lowpass_dilation;
  o.max_elevation = (float)s.max_elevation;
  o.threads = s.threads;
  return o;
}

template <class Camera> odgs_camera to_c_camera(const Camera& c) {
  odgs_camera o;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) o.rotation[3 * r + k] = (float)c.rotation(r, k);  // row-major
  for (int k = 0; k < 3; ++k) o.translation[k] = (float)c.translation[k];
  o.width = c.width;
  o.height = c.height;
  return o;
}

// GaussianCloud<float>: Eigen column-major MatX3 storage is exactly the SoA the ABI wants.
template <class Cloud> odgs_cloud to_c_cloud(const Cloud& c) {
  odgs_cloud o;
  o.n = (int64_t)c.means.rows();
  o.means = c.means.data();
  o.rotations = c.rotations.data();
  o.log_scales = c.log_scales.data();
  o.raw_opacities = c.raw_opacities.data();
  o.colors = c.colors.data();
  o.memory = ODGS_MEM_HOST;
  o.sh_degree = 0;  // the reference's clouds are RGB (SH degree 0)
  o.sh_rest = nullptr;
  return o;
}

// ErpImage<float> -> planar [3][W][H] host copy (each channel is column-major H x W).
template <class Image> std::vector<float> planar(const Image& img, int width, int height) {
  const size_t plane = (size_t)width * height;
  std::vector<float> dl(3 * plane);
  for (int ch = 0; ch < 3; ++ch) {
    const auto& c = img.channel[(size_t)ch];
    if ((size_t)c.rows() * (size_t)c.cols() != plane || c.rows() != height)
      throw std::invalid_argument("dl_dimage: size does not match the frame");
    std::memcpy(dl.data() + ch * plane, c.data(), plane * sizeof(float));
  }
  return dl;
}

template <class Signs> const double* sign_table(const Signs* s) { return s ? s->sign.data() : nullptr; }
inline const double* sign_table(const double* s) { return s; }
inline const double* sign_table(std::nullptr_t) { return nullptr; }

}  // namespace detail

// Fills a reference RenderOutput<float> from a resident frame. with_pixels: image,
// transmittance and walked (a render; prepare_render leaves them empty).
template <class Output> void download(Context& gpu, odgs_frame* f, Output& out, bool with_pixels = true) {
  odgs_frame_info info;
  gpu.check(odgs_frame_get_info(f, &info));
  const int W = info.width, H = info.height;
  const size_t plane = (size_t)W * H;
  if (with_pixels) {
    std::vector<float> img(3 * plane);
    gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_IMAGE, img.data(), img.size() * sizeof(float)));
    for (int c = 0; c < 3; ++c) {
      out.image.channel[(size_t)c].resize(H, W);
      std::memcpy(out.image.channel[(size_t)c].data(), img.data() + c * plane, plane * sizeof(float));
    }
    out.transmittance.resize(H, W);
    gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_TRANSMITTANCE, out.transmittance.data(),
                                  plane * sizeof(float)));
    out.walked.resize(H, W);
    gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_WALKED, out.walked.data(), plane * sizeof(int32_t)));
  }
  out.tiles_x = info.tiles_x;
  out.tiles_y = info.tiles_y;
  out.tile_offsets.resize((size_t)info.tiles_x * info.tiles_y + 1);
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_TILE_OFFSETS, out.tile_offsets.data(),
                                out.tile_offsets.size() * sizeof(int)));
  out.tile_entries.resize((size_t)info.n_entries);
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_TILE_ENTRIES, out.tile_entries.data(),
                                out.tile_entries.size() * sizeof(int)));
  // Splats (projection.hpp:163-174) and the sorted instances (rasterizer.hpp:81-85).
  const size_t ns = (size_t)info.n_splats, ni = (size_t)info.n_instances;
  std::vector<int64_t> idx(ns);
  std::vector<float> mean(2 * ns), cov(4 * ns), inv(4 * ns), depth(ns), radius(ns), opacity(ns), color(3 * ns),
      shift(ni);
  std::vector<int32_t> clamped(ns), inst_splat(ni);
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_INDEX, idx.data(), ns * 8));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_MEAN, mean.data(), mean.size() * 4));
  const bool have_cov = odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_COV2D, cov.data(), cov.size() * 4) == ODGS_OK;
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_INV, inv.data(), inv.size() * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_DEPTH, depth.data(), ns * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_RADIUS, radius.data(), ns * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_OPACITY, opacity.data(), ns * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_COLOR, color.data(), color.size() * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_CLAMPED, clamped.data(), ns * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_INSTANCE_SPLAT, inst_splat.data(), ni * 4));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_INSTANCE_SHIFT, shift.data(), ni * 4));
  out.splats.resize(ns);
  for (size_t s = 0; s < ns; ++s) {
    auto& sp = out.splats[s];
    sp.pixel_mean[0] = mean[2 * s];
    sp.pixel_mean[1] = mean[2 * s + 1];
    if (have_cov) {
      sp.cov2d(0, 0) = cov[4 * s];
      sp.cov2d(0, 1) = cov[4 * s + 1];
      sp.cov2d(1, 0) = cov[4 * s + 2];
      sp.cov2d(1, 1) = cov[4 * s + 3];
    }
    sp.cov2d_inv(0, 0) = inv[4 * s];
    sp.cov2d_inv(0, 1) = inv[4 * s + 1];
    sp.cov2d_inv(1, 0) = inv[4 * s + 2];
    sp.cov2d_inv(1, 1) = inv[4 * s + 3];
    sp.depth = depth[s];
    sp.radius = radius[s];
    sp.opacity = opacity[s];
    for (int c = 0; c < 3; ++c) sp.color[c] = color[3 * s + c];
    sp.index = idx[s];
    sp.pole_clamped = clamped[s] != 0;
  }
  out.instances.resize(ni);
  for (size_t k = 0; k < ni; ++k) {
    out.instances[k].splat = inst_splat[k];
    out.instances[k].shift = shift[k];
  }
}

// odgs::render<float> (rasterizer.hpp:211-267) on the GPU.
template <class Output, class Cloud, class Camera, class Settings>
void render_into(Context& gpu, const Cloud& cloud, const Camera& camera, const Settings& settings, Output& out) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  const odgs_settings s = detail::to_c(settings);
  odgs_frame* f = gpu.acquire();
  gpu.check(odgs_render(gpu.get(), &c, &cam, &s, f));
  download(gpu, f, out);
  gpu.bind(f, key_of(out));
}

template <class Output, class Cloud, class Camera, class Settings>
Output render(Context& gpu, const Cloud& cloud, const Camera& camera, const Settings& settings) {
  Output out;
  render_into(gpu, cloud, camera, settings, out);
  return out;
}

// odgs::prepare_render<float> (rasterizer.hpp:129-207): splats, sorted instances and the
// tile CSR; image / transmittance / walked stay empty as in the reference.
template <class Output, class Cloud, class Camera, class Settings>
Output prepare_render(Context& gpu, const Cloud& cloud, const Camera& camera, const Settings& settings) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  const odgs_settings s = detail::to_c(settings);
  Output out;
  odgs_frame* f = gpu.acquire();
  gpu.check(odgs_prepare_render(gpu.get(), &c, &cam, &s, f));
  download(gpu, f, out, /*with_pixels=*/false);
  return out;
}

// The resident frame fwd was downloaded from, or a rebuild of it from fwd.splats (cloud
// of n_gaussians rows; n_gaussians < 0: one past the last splat's row).
template <class Output, class Settings>
odgs_frame* frame_for(Context& gpu, const Output& fwd, const Settings& settings, int64_t n_gaussians) {
  const FrameKey key = key_of(fwd);
  if (odgs_frame* f = gpu.find(key)) return f;
  const int H = (int)fwd.transmittance.rows(), W = (int)fwd.transmittance.cols();
  if (W <= 0 || H <= 0 || fwd.walked.rows() != H || fwd.walked.cols() != W)
    throw std::invalid_argument("backward: fwd must be a render() output (per-pixel state missing)");
  const size_t ns = fwd.splats.size();
  std::vector<int64_t> idx(ns);
  std::vector<float> mean(2 * ns), inv(4 * ns), depth(ns), radius(ns), opacity(ns), color(3 * ns);
  for (size_t s = 0; s < ns; ++s) {
    const auto& sp = fwd.splats[s];
    idx[s] = (int64_t)sp.index;
    mean[2 * s] = (float)sp.pixel_mean[0];
    mean[2 * s + 1] = (float)sp.pixel_mean[1];
    inv[4 * s] = (float)sp.cov2d_inv(0, 0);
    inv[4 * s + 1] = (float)sp.cov2d_inv(0, 1);
    inv[4 * s + 2] = (float)sp.cov2d_inv(1, 0);
    inv[4 * s + 3] = (float)sp.cov2d_inv(1, 1);
    depth[s] = (float)sp.depth;
    radius[s] = (float)sp.radius;
    opacity[s] = (float)sp.opacity;
    for (int c = 0; c < 3; ++c) color[3 * s + c] = (float)sp.color[c];
  }
  if (n_gaussians < 0) n_gaussians = ns ? idx.back() + 1 : 0;
  const odgs_settings s = detail::to_c(settings);
  odgs_frame* f = gpu.acquire();
  gpu.check(odgs_rasterize_splats(gpu.get(), n_gaussians, (int64_t)ns, idx.data(), mean.data(), inv.data(),
                                  depth.data(), radius.data(), opacity.data(), color.data(), W, H, &s, f));
  gpu.count_rebuild();
  // The rebuilt frame must be fwd's: same tile CSR and walk lengths.
  std::vector<int> offs(fwd.tile_offsets.size());
  odgs_frame_info info;
  gpu.check(odgs_frame_get_info(f, &info));
  bool same = (size_t)info.tiles_x * info.tiles_y + 1 == offs.size() && (size_t)info.n_entries == fwd.tile_entries.size();
  if (same) {
    gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_TILE_OFFSETS, offs.data(), offs.size() * sizeof(int)));
    same = std::memcmp(offs.data(), fwd.tile_offsets.data(), offs.size() * sizeof(int)) == 0;
  }
  if (same) {
    std::vector<int32_t> wk((size_t)W * H);
    gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_WALKED, wk.data(), wk.size() * sizeof(int32_t)));
    same = std::memcmp(wk.data(), fwd.walked.data(), wk.size() * sizeof(int32_t)) == 0;
  }
  if (!same)
    throw std::invalid_argument("backward: fwd's tile lists / walks do not follow from its splats (not a render() output)");
  gpu.bind(f, key);
  return f;
}

// odgs::backward<float> (backward.hpp:380-448): gradients of the view rendered into
// `fwd` (same cloud, camera and settings, as in the reference). signs: GradTSigns-like
// object with .sign[12] (or a double[12]), optional.
template <class Grads, class Cloud, class Camera, class Output, class Image, class Settings, class Signs = std::nullptr_t>
void backward_into(Context& gpu, const Cloud& cloud, const Camera& camera, const Output& fwd, const Image& dl_dimage,
                   const Settings& settings, Grads& out, Signs signs = nullptr, bool accumulate = false) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  const odgs_settings s = detail::to_c(settings);
  odgs_frame* f = frame_for(gpu, fwd, settings, c.n);
  const std::vector<float> dl = detail::planar(dl_dimage, camera.width, camera.height);
  if (!accumulate) out.init(c.n);
  odgs_grads g;
  g.means = out.means.data();
  g.rotations = out.rotations.data();
  g.log_scales = out.log_scales.data();
  g.raw_opacities = out.raw_opacities.data();
  g.colors = out.colors.data();
  g.pixel_grad_norm = out.pixel_grad_norm.data();
  g.one_minus_cos = out.one_minus_cos.data();
  g.observed = out.observed.data();
  g.memory = ODGS_MEM_HOST;
  g.sh_rest = nullptr;
  gpu.check(odgs_backward(gpu.get(), &c, &cam, f, dl.data(), ODGS_MEM_HOST, &s, &g, detail::sign_table(signs),
                          accumulate ? ODGS_ACCUMULATE : 0u));
}

template <class Grads, class Cloud, class Camera, class Output, class Image, class Settings, class Signs = std::nullptr_t>
Grads backward(Context& gpu, const Cloud& cloud, const Camera& camera, const Output& fwd, const Image& dl_dimage,
               const Settings& settings, Signs signs = nullptr) {
  Grads out;
  backward_into(gpu, cloud, camera, fwd, dl_dimage, settings, out, signs);
  return out;
}

// odgs::grad_pixels_to_splats<float> (backward.hpp:208-339): one SplatGrads per splat of fwd.
template <class SplatGradsT, class Output, class Image, class Settings>
std::vector<SplatGradsT> grad_pixels_to_splats(Context& gpu, const Output& fwd, const Image& dl_dimage,
                                               const Settings& settings) {
  odgs_frame* f = frame_for(gpu, fwd, settings, -1);
  const int H = (int)fwd.transmittance.rows(), W = (int)fwd.transmittance.cols();
  const std::vector<float> dl = detail::planar(dl_dimage, W, H);
  const odgs_settings s = detail::to_c(settings);
  const size_t ns = fwd.splats.size();
  std::vector<float> mean(2 * ns), cov(4 * ns), op(ns), col(3 * ns);
  gpu.check(odgs_grad_pixels_to_splats(gpu.get(), f, dl.data(), ODGS_MEM_HOST, &s, mean.data(), cov.data(), op.data(),
                                       col.data()));
  std::vector<SplatGradsT> out(ns);
  for (size_t k = 0; k < ns; ++k) {
    out[k].pixel_mean[0] = mean[2 * k];
    out[k].pixel_mean[1] = mean[2 * k + 1];
    out[k].cov2d(0, 0) = cov[4 * k];
    out[k].cov2d(0, 1) = cov[4 * k + 1];
    out[k].cov2d(1, 0) = cov[4 * k + 2];
    out[k].cov2d(1, 1) = cov[4 * k + 3];
    out[k].opacity = op[k];
    for (int c = 0; c < 3; ++c) out[k].color[c] = col[3 * k + c];
  }
  return out;
}

// odgs::project_gaussian<float> (projection.hpp:178-216).
template <class Splat, class Cloud, class Index, class Camera, class Settings>
std::optional<Splat> project_gaussian(Context& gpu, const Cloud& cloud, Index i, const Camera& camera,
                                      const Settings& settings) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  const odgs_settings s = detail::to_c(settings);
  odgs_splat o;
  int32_t projected = 0;
  gpu.check(odgs_project_gaussian(gpu.get(), &c, (int64_t)i, &cam, &s, &o, &projected));
  if (!projected) return std::nullopt;
  Splat sp;
  sp.pixel_mean[0] = o.pixel_mean[0];
  sp.pixel_mean[1] = o.pixel_mean[1];
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 2; ++k) {
      sp.cov2d(r, k) = o.cov2d[2 * r + k];
      sp.cov2d_inv(r, k) = o.cov2d_inv[2 * r + k];
    }
  sp.depth = o.depth;
  sp.radius = o.radius;
  sp.opacity = o.opacity;
  for (int k = 0; k < 3; ++k) sp.color[k] = o.color[k];
  sp.index = o.index;
  sp.pole_clamped = o.pole_clamped != 0;
  return sp;
}

// odgs::cull (rasterizer.hpp:15-28).
template <class Index, class Cloud, class Camera>
std::vector<Index> cull(Context& gpu, const Cloud& cloud, const Camera& camera, float near_radius, float far_radius) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  std::vector<int64_t> idx((size_t)(c.n > 0 ? c.n : 1));
  int64_t count = 0;
  gpu.check(odgs_cull(gpu.get(), &c, &cam, near_radius, far_radius, idx.data(), &count));
  return std::vector<Index>(idx.begin(), idx.begin() + count);
}

}  // namespace odgs_b200
