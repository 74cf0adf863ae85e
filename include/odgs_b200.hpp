// odgs_b200.hpp — C++ drop-in wrapper over the C ABI (odgs_b200.h).
//
// The reference's hot-path entry points (proj/include/odgs/rasterizer.hpp,
// backward.hpp) take its own types: GaussianCloud<S>, CameraPose<S>, RenderSettings<S>,
// ErpImage<S>, RenderOutput<S>, GradBuffers<S> (Eigen-backed, column-major). The
// functions below are templates over those types — they only use the members the
// reference declares (means/rotations/log_scales/raw_opacities/colors with .data()
// and .rows(); rotation(r, c), translation[k], width, height; the RenderSettings
// fields; channel[c].data(); resize()/init()) — so in a reference build
//
//     #include "odgs/rasterizer.hpp"
//     #include "odgs_b200.hpp"
//     odgs_b200::Context gpu;                               // one per host thread
//     auto out  = odgs_b200::render(gpu, cloud, camera, settings);    // RenderOutput<float>
//     auto grad = odgs_b200::backward(gpu, cloud, camera, out, dl, settings);
//
// replaces odgs::render / odgs::backward for Scalar = float, with the same
// exceptions (std::invalid_argument, std::runtime_error naming the Gaussian,
// std::domain_error). The GPU keeps the frame resident; fields of RenderOutput are
// filled in the reference's layouts. Eigen is not needed to compile this header.
#pragma once

#include <cstdint>
#include <cstring>
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

class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    const odgs_status st = odgs_ctx_create(device, stream, &ctx_);
    if (st != ODGS_OK) throw_status(st, "odgs_ctx_create failed");
  }
  ~Context() {
    if (frame_) odgs_frame_destroy(frame_);
    odgs_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  odgs_ctx* get() const { return ctx_; }
  // The frame of the last render (kept resident for backward).
  odgs_frame* frame() {
    if (!frame_) check(odgs_frame_create(ctx_, &frame_));
    return frame_;
  }
  void check(odgs_status st) const {
    if (st == ODGS_OK) return;
    char msg[512];
    int64_t idx = -1;
    odgs_last_error(ctx_, &idx, msg, sizeof msg);
    throw_status(st, msg);
  }

 private:
  odgs_ctx* ctx_ = nullptr;
  odgs_frame* frame_ = nullptr;
};

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

}  // namespace detail

// Fills a reference RenderOutput<float> from the resident frame.
template <class Output> void download(Context& gpu, Output& out) {
  odgs_frame* f = gpu.frame();
  odgs_frame_info info;
  gpu.check(odgs_frame_get_info(f, &info));
  const int W = info.width, H = info.height;
  const size_t plane = (size_t)W * H;
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
  std::vector<float> mean(2 * ns), inv(4 * ns), depth(ns), radius(ns), opacity(ns), color(3 * ns), shift(ni);
  std::vector<int32_t> clamped(ns), inst_splat(ni);
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_INDEX, idx.data(), ns * 8));
  gpu.check(odgs_frame_download(gpu.get(), f, ODGS_FRAME_SPLAT_MEAN, mean.data(), mean.size() * 4));
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
  gpu.check(odgs_render(gpu.get(), &c, &cam, &s, gpu.frame()));
  download(gpu, out);
}

template <class Output, class Cloud, class Camera, class Settings>
Output render(Context& gpu, const Cloud& cloud, const Camera& camera, const Settings& settings) {
  Output out;
  render_into(gpu, cloud, camera, settings, out);
  return out;
}

// odgs::backward<float> (backward.hpp:380-448) for the frame of the last render on
// `gpu` (same cloud, camera and settings, as in the reference). Grads is the
// reference's GradBuffers<float>; signs: optional GradTSigns-like object with .sign[12].
template <class Grads, class Cloud, class Camera, class Image, class Settings>
void backward_into(Context& gpu, const Cloud& cloud, const Camera& camera, const Image& dl_dimage,
                   const Settings& settings, Grads& out, const double* signs = nullptr, bool accumulate = false) {
  const odgs_cloud c = detail::to_c_cloud(cloud);
  const odgs_camera cam = detail::to_c_camera(camera);
  const odgs_settings s = detail::to_c(settings);
  const size_t plane = (size_t)camera.width * camera.height;
  std::vector<float> dl(3 * plane);
  for (int ch = 0; ch < 3; ++ch)
    std::memcpy(dl.data() + ch * plane, dl_dimage.channel[(size_t)ch].data(), plane * sizeof(float));
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
  gpu.check(odgs_backward(gpu.get(), &c, &cam, gpu.frame(), dl.data(), ODGS_MEM_HOST, &s, &g, signs,
                          accumulate ? ODGS_ACCUMULATE : 0u));
}

template <class Grads, class Cloud, class Camera, class Image, class Settings>
Grads backward(Context& gpu, const Cloud& cloud, const Camera& camera, const Image& dl_dimage,
               const Settings& settings) {
  Grads out;
  backward_into(gpu, cloud, camera, dl_dimage, settings, out);
  return out;
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
