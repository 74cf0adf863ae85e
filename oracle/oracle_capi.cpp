// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY: a C ABI over odgs_oracle.hpp so the
// pytest parity suite and bench.py's CPU-baseline leg can drive the restatement
// through ctypes. Never linked into the product library.
//
// All array inputs are binary64 (float inputs are passed widened, which is exact);
// all float outputs are returned widened to binary64. Layouts follow the reference:
// cloud members SoA (Eigen column-major MatX3: member(i, c) at c*n + i), images
// planar with each H x W channel column-major (y + x*H).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>

#include "odgs_oracle.hpp"

using namespace oracle;

namespace {

struct Handle {
  bool dbl = false, portable = false;
  Cloud<float> cf; Cloud<double> cd;
  Camera<float> camf; Camera<double> camd;
  Settings<float> sf; Settings<double> sd;
  RenderOutput<float> rf; RenderOutput<double> rd;
  GradBuffers<float> gf; GradBuffers<double> gd;
  std::vector<SplatGrads<float>> sgf; std::vector<SplatGrads<double>> sgd;
  bool have_grads = false;
  std::vector<double> brute;
  double seconds_render = 0, seconds_backward = 0;
};

int fail(char* err, int errlen, int code, const char* what) {
  if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "%s", what);
  return code;
}

template <class F> int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(err, errlen, 1, e.what());
  } catch (const std::domain_error& e) {
    return fail(err, errlen, 3, e.what());
  } catch (const std::runtime_error& e) {
    return fail(err, errlen, 2, e.what());
  } catch (const std::exception& e) {
    return fail(err, errlen, 4, e.what());
  }
}

template <class S>
void load(Cloud<S>& c, Camera<S>& cam, Settings<S>& s, int64_t n, const double* means, const double* rotations,
          const double* log_scales, const double* raw_opacities, const double* colors, const double* R,
          const double* t, int width, int height, const double* st, int threads, int sh_degree,
          const double* sh_rest) {
  c.n = n;
  c.sh_degree = sh_degree;
  if (sh_degree > 0) c.sh_rest.assign(sh_rest, sh_rest + 3 * sh_count(sh_degree) * n);
  c.means.assign(means, means + 3 * n);
  c.rotations.assign(rotations, rotations + 4 * n);
  c.log_scales.assign(log_scales, log_scales + 3 * n);
  c.raw_opacities.assign(raw_opacities, raw_opacities + n);
  c.colors.assign(colors, colors + 3 * n);
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) cam.rotation(r, k) = S(R[3 * r + k]);
  for (int k = 0; k < 3; ++k) cam.translation[k] = S(t[k]);
  cam.width = width;
  cam.height = height;
  s.near_radius = S(st[0]);
  s.far_radius = S(st[1]);
  s.tile_size = (int)st[2];
  s.alpha_clamp = S(st[3]);
  s.transmittance_floor = S(st[4]);
  s.cutoff_sigma = S(st[5]);
  s.lowpass_dilation = S(st[6]);
  s.max_elevation = S(st[7]);
  s.threads = threads;
}

template <class T, class V> int64_t copy_out(const V& v, void* dst) {
  if (dst) {
    T* d = static_cast<T*>(dst);
    for (std::size_t k = 0; k < v.size(); ++k) d[k] = (T)v[k];
  }
  return (int64_t)v.size();
}

template <class S>
int64_t get_from(const RenderOutput<S>& r, const GradBuffers<S>& g, const std::vector<SplatGrads<S>>& sg,
                 bool have_grads, const std::vector<double>& brute, const std::string& w, void* dst) {
  const std::size_t ns = r.splats.size();
  auto splat_field = [&](int width, auto getter) -> int64_t {
    if (dst) {
      double* d = static_cast<double*>(dst);
      for (std::size_t s = 0; s < ns; ++s) getter(r.splats[s], d + s * width);
    }
    return (int64_t)(ns * width);
  };
  if (w == "image") return copy_out<double>(r.image, dst);
  if (w == "brute") return copy_out<double>(brute, dst);
  if (w == "transmittance") return copy_out<double>(r.transmittance, dst);
  if (w == "walked") return copy_out<int32_t>(r.walked, dst);
  if (w == "tile_offsets") return copy_out<int32_t>(r.tile_offsets, dst);
  if (w == "tile_entries") return copy_out<int32_t>(r.tile_entries, dst);
  if (w == "inst_splat" || w == "inst_shift") {
    if (dst)
      for (std::size_t k = 0; k < r.instances.size(); ++k) {
        if (w == "inst_splat") static_cast<int32_t*>(dst)[k] = r.instances[k].splat;
        else static_cast<double*>(dst)[k] = r.instances[k].shift;
      }
    return (int64_t)r.instances.size();
  }
  if (w == "splat_index") {
    if (dst) for (std::size_t s = 0; s < ns; ++s) static_cast<int64_t*>(dst)[s] = r.splats[s].index;
    return (int64_t)ns;
  }
  if (w == "splat_clamped") {
    if (dst) for (std::size_t s = 0; s < ns; ++s) static_cast<int32_t*>(dst)[s] = r.splats[s].pole_clamped;
    return (int64_t)ns;
  }
  if (w == "splat_mean") return splat_field(2, [](const Splat2D<S>& s, double* d) { d[0] = s.pixel_mean[0]; d[1] = s.pixel_mean[1]; });
  if (w == "splat_cov2d") return splat_field(4, [](const Splat2D<S>& s, double* d) { d[0] = s.cov2d(0, 0); d[1] = s.cov2d(0, 1); d[2] = s.cov2d(1, 0); d[3] = s.cov2d(1, 1); });
  if (w == "splat_inv") return splat_field(4, [](const Splat2D<S>& s, double* d) { d[0] = s.cov2d_inv(0, 0); d[1] = s.cov2d_inv(0, 1); d[2] = s.cov2d_inv(1, 0); d[3] = s.cov2d_inv(1, 1); });
  if (w == "splat_depth") return splat_field(1, [](const Splat2D<S>& s, double* d) { d[0] = s.depth; });
  if (w == "splat_radius") return splat_field(1, [](const Splat2D<S>& s, double* d) { d[0] = s.radius; });
  if (w == "splat_opacity") return splat_field(1, [](const Splat2D<S>& s, double* d) { d[0] = s.opacity; });
  if (w == "splat_color") return splat_field(3, [](const Splat2D<S>& s, double* d) { for (int c = 0; c < 3; ++c) d[c] = s.color[c]; });
  if (w == "stats") {
    const int64_t st[7] = {(int64_t)ns, (int64_t)r.instances.size(), (int64_t)r.tile_entries.size(),
                           r.e_exam, r.e_contrib, r.tiles_x, r.tiles_y};
    if (dst) std::memcpy(dst, st, sizeof st);
    return 7;
  }
  if (!have_grads) return -1;
  if (w == "g_means") return copy_out<double>(g.means, dst);
  if (w == "g_rotations") return copy_out<double>(g.rotations, dst);
  if (w == "g_log_scales") return copy_out<double>(g.log_scales, dst);
  if (w == "g_raw_opacities") return copy_out<double>(g.raw_opacities, dst);
  if (w == "g_colors") return copy_out<double>(g.colors, dst);
  if (w == "g_pixel_grad_norm") return copy_out<double>(g.pixel_grad_norm, dst);
  if (w == "g_one_minus_cos") return copy_out<double>(g.one_minus_cos, dst);
  if (w == "g_observed") return copy_out<int32_t>(g.observed, dst);
  if (w == "g_sh_rest") return copy_out<double>(g.sh_rest, dst);
  auto sg_field = [&](int width, auto getter) -> int64_t {
    if (dst) {
      double* d = static_cast<double*>(dst);
      for (std::size_t s = 0; s < sg.size(); ++s) getter(sg[s], d + s * width);
    }
    return (int64_t)(sg.size() * width);
  };
  if (w == "sg_mean") return sg_field(2, [](const SplatGrads<S>& s, double* d) { d[0] = s.pixel_mean[0]; d[1] = s.pixel_mean[1]; });
  if (w == "sg_cov2d") return sg_field(4, [](const SplatGrads<S>& s, double* d) { d[0] = s.cov2d(0, 0); d[1] = s.cov2d(0, 1); d[2] = s.cov2d(1, 0); d[3] = s.cov2d(1, 1); });
  if (w == "sg_opacity") return sg_field(1, [](const SplatGrads<S>& s, double* d) { d[0] = s.opacity; });
  if (w == "sg_color") return sg_field(3, [](const SplatGrads<S>& s, double* d) { for (int c = 0; c < 3; ++c) d[c] = s.color[c]; });
  return -1;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

// Renders one view with the restatement. dbl: 0 float / 1 double. portable: 0 StdMath /
// 1 PortableMath (float only). brute: also run the brute-force oracle of
// proj/tests/oracle.hpp:19-85. R is row-major. st = {near, far, tile, alpha_clamp,
// transmittance_floor, cutoff_sigma, lowpass_dilation, max_elevation}.
// Returns 0 and *out on success; otherwise 1 invalid_argument, 2 runtime_error,
// 3 domain_error, 4 other, with the message in err.
int oracle_render(int dbl, int portable, int brute, int64_t n, const double* means, const double* rotations,
                  const double* log_scales, const double* raw_opacities, const double* colors, const double* R,
                  const double* t, int width, int height, const double* st, int threads, int sh_degree,
                  const double* sh_rest, void** out, char* err, int errlen) {
  auto h = std::make_unique<Handle>();
  h->dbl = dbl != 0;
  h->portable = portable != 0;
  if (h->dbl && h->portable) return fail(err, errlen, 4, "PortableMath is float-only");
  const int rc = guarded(err, errlen, [&] {
    const double t0 = now();
    if (h->dbl) {
      load(h->cd, h->camd, h->sd, n, means, rotations, log_scales, raw_opacities, colors, R, t, width, height, st, threads,
           sh_degree, sh_rest);
      h->rd = render<double, StdMath>(h->cd, h->camd, h->sd);
      h->seconds_render = now() - t0;
      if (brute) h->brute = brute_force_render<double, StdMath>(h->cd, h->camd, h->sd);
    } else {
      load(h->cf, h->camf, h->sf, n, means, rotations, log_scales, raw_opacities, colors, R, t, width, height, st, threads,
           sh_degree, sh_rest);
      if (h->portable) {
        h->rf = render<float, PortableMath>(h->cf, h->camf, h->sf);
        h->seconds_render = now() - t0;
        if (brute) {
          auto b = brute_force_render<float, PortableMath>(h->cf, h->camf, h->sf);
          h->brute.assign(b.begin(), b.end());
        }
      } else {
        h->rf = render<float, StdMath>(h->cf, h->camf, h->sf);
        h->seconds_render = now() - t0;
        if (brute) {
          auto b = brute_force_render<float, StdMath>(h->cf, h->camf, h->sf);
          h->brute.assign(b.begin(), b.end());
        }
      }
    }
  });
  if (rc != 0) return rc;
  *out = h.release();
  return 0;
}

// Backward pass of the rendered view for the image gradient dl_dimage (3*H*W,
// reference layout). mutate_term in [0, 11] flips one GradTSigns term (-1: none).
int oracle_backward(void* handle, const double* dl_dimage, int mutate_term, char* err, int errlen) {
  Handle* h = static_cast<Handle*>(handle);
  GradTSigns signs;
  if (mutate_term >= 0 && mutate_term < 12) signs.sign[(std::size_t)mutate_term] = -1;
  return guarded(err, errlen, [&] {
    const double t0 = now();
    if (h->dbl) {
      std::vector<double> g(dl_dimage, dl_dimage + (std::size_t)3 * h->camd.width * h->camd.height);
      h->gd = backward<double, StdMath>(h->cd, h->camd, h->rd, g, h->sd, &signs, &h->sgd);
    } else {
      std::vector<float> g((std::size_t)3 * h->camf.width * h->camf.height);
      for (std::size_t k = 0; k < g.size(); ++k) g[k] = (float)dl_dimage[k];
      if (h->portable)
        h->gf = backward<float, PortableMath>(h->cf, h->camf, h->rf, g, h->sf, &signs, &h->sgf);
      else
        h->gf = backward<float, StdMath>(h->cf, h->camf, h->rf, g, h->sf, &signs, &h->sgf);
    }
    h->seconds_backward = now() - t0;
    h->have_grads = true;
  });
}

// Copies the named output into dst (may be NULL) and returns its element count, or -1.
int64_t oracle_get(void* handle, const char* which, void* dst) {
  Handle* h = static_cast<Handle*>(handle);
  const std::string w(which);
  if (w == "seconds") {
    if (dst) { static_cast<double*>(dst)[0] = h->seconds_render; static_cast<double*>(dst)[1] = h->seconds_backward; }
    return 2;
  }
  if (h->dbl) return get_from(h->rd, h->gd, h->sgd, h->have_grads, h->brute, w, dst);
  return get_from(h->rf, h->gf, h->sgf, h->have_grads, h->brute, w, dst);
}

// Sorts, bins and blends the splats of an existing float frame (rasterize_splats, i.e.
// the stages after projection) with StdMath (portable = 0) or PortableMath blending.
int oracle_rasterize_splats(void* handle, int portable, void** out, char* err, int errlen) {
  Handle* src = static_cast<Handle*>(handle);
  if (src->dbl) return fail(err, errlen, 1, "rasterize_splats: float frames only");
  auto h = std::make_unique<Handle>();
  const int rc = guarded(err, errlen, [&] {
    h->portable = portable != 0;
    h->sf = src->sf;
    h->camf = src->camf;
    h->cf = src->cf;
    if (portable)
      h->rf = rasterize_splats<float, PortableMath>(src->rf.splats, src->rf.width, src->rf.height, src->sf);
    else
      h->rf = rasterize_splats<float, StdMath>(src->rf.splats, src->rf.width, src->rf.height, src->sf);
  });
  if (rc == 0) *out = h.release();
  return rc;
}

void oracle_free(void* handle) { delete static_cast<Handle*>(handle); }

// scenes::random_cloud (proj/tests/scenes.hpp:20-51) with the given bounds
// {depth_min, depth_max, max_elevation, opacity_min, opacity_max, scale_min, scale_max};
// as_float rounds every member through float exactly as random_cloud<float> does.
int oracle_random_cloud(uint32_t seed, int n, const double* b, int as_float, double* means, double* rotations,
                        double* log_scales, double* raw_opacities, double* colors) {
  CloudBounds bounds;
  bounds.depth_min = b[0]; bounds.depth_max = b[1]; bounds.max_elevation = b[2];
  bounds.opacity_min = b[3]; bounds.opacity_max = b[4]; bounds.scale_min = b[5]; bounds.scale_max = b[6];
  std::mt19937 rng(seed);
  auto emit = [&](const auto& c) {
    for (std::size_t k = 0; k < c.means.size(); ++k) means[k] = c.means[k];
    for (std::size_t k = 0; k < c.rotations.size(); ++k) rotations[k] = c.rotations[k];
    for (std::size_t k = 0; k < c.log_scales.size(); ++k) log_scales[k] = c.log_scales[k];
    for (std::size_t k = 0; k < c.raw_opacities.size(); ++k) raw_opacities[k] = c.raw_opacities[k];
    for (std::size_t k = 0; k < c.colors.size(); ++k) colors[k] = c.colors[k];
  };
  if (as_float) emit(random_cloud<float>(rng, n, bounds));
  else emit(random_cloud<double>(rng, n, bounds));
  return 0;
}

// photometric_loss (proj/include/odgs/metrics.hpp:152-184) in binary64.
double oracle_photometric_loss(const double* rendered, const double* target, int height, int width,
                               double lambda_ssim, double* gradient) {
  const std::size_t sz = (std::size_t)3 * height * width;
  std::vector<double> a(rendered, rendered + sz), b(target, target + sz), g;
  const double loss = photometric_loss(a, b, height, width, lambda_ssim, &g);
  if (gradient) std::memcpy(gradient, g.data(), sz * sizeof(double));
  return loss;
}

// densify_and_prune<float, M> (proj/include/odgs/densify.hpp:81-153) on a float cloud
// and TrainState. moments: the ten Adam arrays concatenated in TrainState order
// (means_m 3n, means_v 3n, rot_m 4n, rot_v 4n, scale_m 3n, scale_v 3n, opac_m n,
// opac_v n, color_m 3n, color_v 3n = 28 n). cfg: {grad_threshold_min,
// grad_threshold_max, percent_dense, opacity_prune_floor, split_scale_divisor}.
// Outputs are written into caller buffers sized for n_cap rows (n_cap >= 3 n is always
// enough): params 14 n_out (means 3, rotations 4, log_scales 3, raw 1, colors 3, each
// block n_out long), moments 28 n_out; stats = {cloned, split, pruned, n_out};
// *next_draw = the generator's next 32-bit output afterwards (stream position check).
int oracle_densify(int portable, int64_t n, const double* params, const double* moments, const double* grad_accum,
                   const double* elev_accum, const int32_t* grad_count, const double* cfg, double extent,
                   uint32_t seed, int64_t n_cap, double* params_out, double* moments_out, int64_t* stats,
                   uint32_t* next_draw, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Cloud<float> c;
    c.resize(n);
    auto take = [&](std::vector<float>& v, const double* src, int64_t count) {
      for (int64_t k = 0; k < count; ++k) v[(std::size_t)k] = (float)src[k];
    };
    take(c.means, params, 3 * n);
    take(c.rotations, params + 3 * n, 4 * n);
    take(c.log_scales, params + 7 * n, 3 * n);
    take(c.raw_opacities, params + 10 * n, n);
    take(c.colors, params + 11 * n, 3 * n);
    TrainState<float> st;
    st.init(n);
    std::vector<float>* mv[10] = {&st.means_m, &st.means_v, &st.rot_m, &st.rot_v, &st.scale_m,
                                  &st.scale_v, &st.opac_m, &st.opac_v, &st.color_m, &st.color_v};
    const int widths[10] = {3, 3, 4, 4, 3, 3, 1, 1, 3, 3};
    int64_t off = 0;
    for (int k = 0; k < 10; ++k) {
      take(*mv[k], moments + off, widths[k] * n);
      off += widths[k] * n;
    }
    take(st.grad_accum, grad_accum, n);
    take(st.elev_accum, elev_accum, n);
    for (int64_t i = 0; i < n; ++i) st.grad_count[(std::size_t)i] = grad_count[i];
    DensifyConfig dc;
    dc.grad_threshold_min = cfg[0];
    dc.grad_threshold_max = cfg[1];
    dc.percent_dense = cfg[2];
    dc.opacity_prune_floor = cfg[3];
    dc.split_scale_divisor = cfg[4];
    std::mt19937 rng(seed);
    const DensifyStats ds = portable ? densify_and_prune<float, PortableMath>(c, st, dc, (float)extent, rng)
                                     : densify_and_prune<float, StdMath>(c, st, dc, (float)extent, rng);
    const int64_t m = c.n;
    if (m > n_cap) throw std::runtime_error("oracle_densify: output capacity too small");
    stats[0] = ds.cloned; stats[1] = ds.split; stats[2] = ds.pruned; stats[3] = m;
    auto put = [&](const std::vector<float>& v, double* dst) {
      for (std::size_t k = 0; k < v.size(); ++k) dst[k] = v[k];
    };
    put(c.means, params_out);
    put(c.rotations, params_out + 3 * m);
    put(c.log_scales, params_out + 7 * m);
    put(c.raw_opacities, params_out + 10 * m);
    put(c.colors, params_out + 11 * m);
    off = 0;
    for (int k = 0; k < 10; ++k) {
      put(*mv[k], moments_out + off);
      off += widths[k] * m;
    }
    *next_draw = (uint32_t)rng();
  });
}

// reset_opacity<float, M> (densify.hpp:158-166) on the raw opacities, in place.
int oracle_reset_opacity(int portable, int64_t n, double* raw_opacities, double ceiling, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Cloud<float> c;
    c.resize(n);
    for (int64_t i = 0; i < n; ++i) c.raw_opacities[(std::size_t)i] = (float)raw_opacities[i];
    TrainState<float> st;
    st.init(n);
    if (portable) reset_opacity<float, PortableMath>(c, st, (float)ceiling);
    else reset_opacity<float, StdMath>(c, st, (float)ceiling);
    for (int64_t i = 0; i < n; ++i) raw_opacities[i] = c.raw_opacities[(std::size_t)i];
  });
}

// count samples of detail::unit_ball_normal<float> (densify.hpp:61-69) from
// std::mt19937(seed), (x, y, z) per sample; returns the generator's next output.
uint32_t oracle_unit_ball(uint32_t seed, int64_t count, float* out) {
  std::mt19937 rng(seed);
  for (int64_t k = 0; k < count; ++k) {
    const V3<float> e = unit_ball_normal<float>(rng);
    for (int c = 0; c < 3; ++c) out[3 * k + c] = e[c];
  }
  return (uint32_t)rng();
}

// dynamic_threshold<double> (densify.hpp:39-49); returns 3 on domain_error.
int oracle_dynamic_threshold(double elevation, double tmin, double tmax, double* out) {
  DensifyConfig c;
  c.grad_threshold_min = tmin;
  c.grad_threshold_max = tmax;
  try {
    *out = dynamic_threshold(elevation, c);
  } catch (const std::domain_error&) {
    return 3;
  }
  return 0;
}

int oracle_hardware_concurrency() { return effective_threads(0); }

// init_from_points scales (io.cpp:268-296), brute force.
void oracle_init_scales(int64_t n, const double* pos, double* scale, double* ls) {
  init_scales_brute(n, pos, scale, ls);
}

}  // extern "C"
