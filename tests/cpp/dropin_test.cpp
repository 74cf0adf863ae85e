// dropin_test.cpp — exercises the C++ drop-in the way a reference build would: types
// and function templates with the reference's names in namespace odgs (Eigen-layout
// stand-ins, since Eigen is absent from this image), then include/odgs_b200_dropin.hpp,
// so that unqualified reference call sites — odgs::render(cloud, camera, settings) and
// template callers like train_step<float> — resolve to the GPU. Checked against the
// oracle restatement. Cases follow proj/tests/test_rasterizer.cpp, test_projection.cpp
// and test_backward.cpp. Built and run by tests/test_gpu_dropin.py on the GPU box.
#include <array>
#include <cmath>
#include <cstdio>
#include <limits>
#include <optional>
#include <random>
#include <stdexcept>
#include <vector>

namespace Eigen {
using Index = std::ptrdiff_t;
}

namespace odgs {  // stand-ins with the reference's names and Eigen's column-major storage
template <class T> struct Dense {  // Eigen::Matrix / Array, column-major
  std::vector<T> v;
  long r = 0, c = 0;
  void resize(long rows, long cols) { r = rows; c = cols; v.assign((size_t)(rows * cols), T(0)); }
  void setZero(long rows, long cols) { resize(rows, cols); }
  void setZero(long rows) { resize(rows, 1); }
  long rows() const { return r; }
  long cols() const { return c; }
  T* data() { return v.data(); }
  const T* data() const { return v.data(); }
  T& operator()(long i, long j) { return v[(size_t)(j * r + i)]; }
  T operator()(long i, long j) const { return v[(size_t)(j * r + i)]; }
  T& operator[](long i) { return v[(size_t)i]; }
  T operator[](long i) const { return v[(size_t)i]; }
};
template <class T, int R, int C> struct Fixed {
  T a[R * C]{};
  T& operator()(int i, int j) { return a[j * R + i]; }
  T operator()(int i, int j) const { return a[j * R + i]; }
  T& operator[](int i) { return a[i]; }
  T operator[](int i) const { return a[i]; }
};
template <class S> struct GaussianCloud {  // types.hpp:53-143
  Dense<S> means, rotations, log_scales, raw_opacities, colors;
};
template <class S> struct CameraPose {  // types.hpp:148-180
  Fixed<S, 3, 3> rotation;
  Fixed<S, 3, 1> translation;
  int width = 0, height = 0;
  CameraPose() { rotation(0, 0) = rotation(1, 1) = rotation(2, 2) = 1; }
};
template <class S> struct RenderSettings {  // types.hpp:229-255
  S near_radius = S(0.01), far_radius = S(1000);
  int tile_size = 16;
  S alpha_clamp = S(0.99), transmittance_floor = S(1e-4), cutoff_sigma = S(3), lowpass_dilation = S(0.3);
  S max_elevation = S(85.0f * 3.14159274101257324f / 180.0f);
  int threads = 0;
};
template <class S> struct ErpImage {  // types.hpp:184-224
  std::array<Dense<S>, 3> channel;
};
template <class S> struct Splat2D {  // projection.hpp:163-174
  Fixed<S, 2, 1> pixel_mean;
  Fixed<S, 2, 2> cov2d, cov2d_inv;
  S depth = 0, radius = 0, opacity = 0;
  Fixed<S, 3, 1> color;
  Eigen::Index index = 0;
  bool pole_clamped = false;
};
template <class S> struct SplatInstance { int splat; S shift; };  // rasterizer.hpp:81-85
template <class S> struct RenderOutput {  // rasterizer.hpp:92-102
  ErpImage<S> image;
  Dense<S> transmittance;
  Dense<int> walked;
  std::vector<Splat2D<S>> splats;
  std::vector<SplatInstance<S>> instances;
  std::vector<int> tile_offsets, tile_entries;
  int tiles_x = 0, tiles_y = 0;
};
template <class S> struct SplatGrads {  // backward.hpp:19-25
  Fixed<S, 2, 1> pixel_mean;
  Fixed<S, 2, 2> cov2d;
  S opacity = 0;
  Fixed<S, 3, 1> color;
};
struct GradTSigns {  // backward.hpp:32-34
  std::array<double, 12> sign{{1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1}};
};
template <class S> struct GradBuffers {  // backward.hpp:342-374
  Dense<S> means, rotations, log_scales, raw_opacities, colors, pixel_grad_norm, one_minus_cos;
  Dense<int> observed;
  void init(long n) {
    means.setZero(n, 3); rotations.setZero(n, 4); log_scales.setZero(n, 3); raw_opacities.setZero(n);
    colors.setZero(n, 3); pixel_grad_norm.setZero(n); one_minus_cos.setZero(n); observed.setZero(n);
  }
};

// The reference's CPU function templates (declarations as in its headers). These
// stand-ins only count calls: a drop-in must never reach them for Scalar = float.
inline int cpu_calls = 0;
template <class S>
RenderOutput<S> render(const GaussianCloud<S>&, const CameraPose<S>&, const RenderSettings<S>&) {
  ++cpu_calls;
  return {};
}
template <class S>
RenderOutput<S> prepare_render(const GaussianCloud<S>&, const CameraPose<S>&, const RenderSettings<S>&) {
  ++cpu_calls;
  return {};
}
template <class S>
GradBuffers<S> backward(const GaussianCloud<S>&, const CameraPose<S>&, const RenderOutput<S>&, const ErpImage<S>&,
                        const RenderSettings<S>&, const GradTSigns* = nullptr) {
  ++cpu_calls;
  return {};
}
template <class S>
std::vector<SplatGrads<S>> grad_pixels_to_splats(const RenderOutput<S>&, const ErpImage<S>&, const RenderSettings<S>&) {
  ++cpu_calls;
  return {};
}
template <class S>
std::optional<Splat2D<S>> project_gaussian(const GaussianCloud<S>&, Eigen::Index, const CameraPose<S>&,
                                           const RenderSettings<S>&) {
  ++cpu_calls;
  return std::nullopt;
}
template <class S> std::vector<Eigen::Index> cull(const GaussianCloud<S>&, const CameraPose<S>&, S, S) {
  ++cpu_calls;
  return {};
}

// A reference-style template caller (the shape of train_step, optimizer.hpp:107,112):
// unqualified, dependent calls, resolved at instantiation.
template <class S>
GradBuffers<S> view_step(const GaussianCloud<S>& cloud, const CameraPose<S>& cam, const ErpImage<S>& dl,
                         const RenderSettings<S>& s) {
  const RenderOutput<S> fwd = render(cloud, cam, s);
  return backward(cloud, cam, fwd, dl, s);
}
}  // namespace odgs

#include "odgs_b200_dropin.hpp"
#include "odgs_oracle.hpp"

static int failures = 0;
#define CHECK(x) do { if (!(x)) { ++failures; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); } } while (0)

using CloudF = odgs::GaussianCloud<float>;
using CamF = odgs::CameraPose<float>;
using SetF = odgs::RenderSettings<float>;
using OutF = odgs::RenderOutput<float>;
using GradF = odgs::GradBuffers<float>;
using ImgF = odgs::ErpImage<float>;

static CloudF to_ref(const oracle::Cloud<float>& c) {
  CloudF r;
  const long n = c.n;
  r.means.resize(n, 3); r.rotations.resize(n, 4); r.log_scales.resize(n, 3); r.raw_opacities.resize(n, 1);
  r.colors.resize(n, 3);
  std::copy(c.means.begin(), c.means.end(), r.means.v.begin());
  std::copy(c.rotations.begin(), c.rotations.end(), r.rotations.v.begin());
  std::copy(c.log_scales.begin(), c.log_scales.end(), r.log_scales.v.begin());
  std::copy(c.raw_opacities.begin(), c.raw_opacities.end(), r.raw_opacities.v.begin());
  std::copy(c.colors.begin(), c.colors.end(), r.colors.v.begin());
  return r;
}

static ImgF probe_image(std::mt19937& rng, int W, int H, std::vector<float>* flat) {
  ImgF img;
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (int ch = 0; ch < 3; ++ch) {
    img.channel[ch].resize(H, W);
    for (auto& v : img.channel[ch].v) {
      v = u(rng);
      if (flat) flat->push_back(v);
    }
  }
  return img;
}

static bool same_grads(const GradF& a, const GradF& b) {
  return a.means.v == b.means.v && a.rotations.v == b.rotations.v && a.log_scales.v == b.log_scales.v &&
         a.raw_opacities.v == b.raw_opacities.v && a.colors.v == b.colors.v && a.observed.v == b.observed.v &&
         a.pixel_grad_norm.v == b.pixel_grad_norm.v && a.one_minus_cos.v == b.one_minus_cos.v;
}

template <class A, class B> static double group_rel(const A& a, const B& b) {
  double md = 0, ma = 0, mb = 0;
  for (size_t k = 0; k < b.size(); ++k) {
    md = std::max(md, std::abs((double)a[k] - (double)b[k]));
    ma = std::max(ma, std::abs((double)a[k]));
    mb = std::max(mb, std::abs((double)b[k]));
  }
  return md / std::max({ma, mb, 1e-12});
}

int main() {
  SetF settings;
  CamF cam;
  cam.width = 256;
  cam.height = 128;
  const auto ocam = oracle::identity_camera<float>(256, 128);

  {  // test_rasterizer.cpp:110-116 — empty cloud: black, unit transmittance
    CloudF empty;
    empty.means.resize(0, 3); empty.rotations.resize(0, 4); empty.log_scales.resize(0, 3);
    empty.raw_opacities.resize(0, 1); empty.colors.resize(0, 3);
    auto out = odgs::render(empty, cam, settings);
    float mx = 0, mn = 1;
    for (int c = 0; c < 3; ++c) for (float v : out.image.channel[c].v) mx = std::max(mx, std::abs(v));
    for (float v : out.transmittance.v) mn = std::min(mn, v);
    CHECK(mx == 0.0f);
    CHECK(mn == 1.0f);
  }
  {  // test_rasterizer.cpp:118-129 — NaN names the Gaussian (std::runtime_error)
    std::mt19937 rng(5);
    auto c = oracle::random_cloud<float>(rng, 4);
    c.mean(2, 1) = std::numeric_limits<float>::quiet_NaN();
    bool threw = false;
    try {
      odgs::render(to_ref(c), cam, settings);
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()) == "render: non-finite parameter in Gaussian 2";
    }
    CHECK(threw);
  }
  {  // bad camera -> std::invalid_argument (types.hpp:159-169)
    std::mt19937 rng(5);
    auto c = oracle::random_cloud<float>(rng, 4);
    CamF bad = cam;
    bad.height = 100;
    bool threw = false;
    try {
      odgs::render(to_ref(c), bad, settings);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::mt19937 rng77(77);
  const auto c300 = oracle::random_cloud<float>(rng77, 300);
  const CloudF r300 = to_ref(c300);
  const auto o300 = oracle::render<float, oracle::PortableMath>(c300, ocam, oracle::Settings<float>{});
  {  // every RenderOutput field equals the portable oracle, bit for bit
    auto out = odgs::render(r300, cam, settings);
    const auto& o = o300;
    CHECK(out.tile_offsets == o.tile_offsets);
    CHECK(out.tile_entries == o.tile_entries);
    CHECK(out.splats.size() == o.splats.size());
    CHECK(out.instances.size() == o.instances.size());
    bool same = out.splats.size() == o.splats.size();
    for (size_t s = 0; same && s < o.splats.size(); ++s) {
      const auto& a = out.splats[s];
      const auto& b = o.splats[s];
      same = a.index == b.index && a.pixel_mean[0] == b.pixel_mean[0] && a.pixel_mean[1] == b.pixel_mean[1] &&
             a.radius == b.radius && a.depth == b.depth && a.opacity == b.opacity && a.color[2] == b.color[2] &&
             a.cov2d(0, 1) == b.cov2d(0, 1) && a.cov2d(1, 1) == b.cov2d(1, 1) &&
             a.cov2d_inv(0, 1) == b.cov2d_inv(0, 1) && a.pole_clamped == b.pole_clamped;
    }
    CHECK(same);
    for (size_t k = 0; same && k < o.instances.size(); ++k)
      same = out.instances[k].splat == o.instances[k].splat && out.instances[k].shift == o.instances[k].shift;
    CHECK(same);
    bool img = true;
    for (int ch = 0; ch < 3; ++ch)
      for (int x = 0; x < 256; ++x)
        for (int y = 0; y < 128; ++y) img = img && out.image.channel[ch](y, x) == o.img(ch, y, x);
    CHECK(img);
    bool wk = true;
    for (int x = 0; x < 256; ++x)
      for (int y = 0; y < 128; ++y)
        wk = wk && out.walked(y, x) == o.walked[o.px(y, x)] && out.transmittance(y, x) == o.transmittance[o.px(y, x)];
    CHECK(wk);
  }
  {  // prepare_render (rasterizer.hpp:129-207): splats, instances, CSR; no pixels
    auto p = odgs::prepare_render(r300, cam, settings);
    CHECK(p.tile_offsets == o300.tile_offsets);
    CHECK(p.tile_entries == o300.tile_entries);
    CHECK(p.splats.size() == o300.splats.size());
    CHECK(p.image.channel[0].rows() == 0 && p.walked.rows() == 0);
  }
  {  // render A, render B, backward A: A's own frame, not the last render
    SetF s8 = settings;
    s8.cutoff_sigma = 8.0f;
    std::mt19937 rng(137);
    oracle::CloudBounds b;
    b.depth_min = 0.8; b.depth_max = 10.0; b.max_elevation = 75.0 * 3.141592653589793 / 180.0;
    b.opacity_min = 0.1; b.opacity_max = 0.7; b.scale_min = 0.02; b.scale_max = 0.12;
    auto ca = oracle::random_cloud<float>(rng, 8, b);
    auto cb = oracle::random_cloud<float>(rng, 8, b);
    CamF small;
    small.width = 64;
    small.height = 32;
    std::vector<float> probe_flat;
    const ImgF probe = probe_image(rng, 64, 32, &probe_flat);
    const CloudF ra = to_ref(ca), rb = to_ref(cb);
    auto& gpu = odgs_b200::thread_context();
    const auto fa = odgs::render(ra, small, s8);
    const auto fb = odgs::render(rb, small, s8);
    const int64_t rebuilds0 = gpu.rebuilds();
    const GradF ga = odgs::backward(ra, small, fa, probe, s8);  // fa still resident
    CHECK(gpu.rebuilds() == rebuilds0);
    const auto fa2 = odgs::render(ra, small, s8);
    const GradF ga_fresh = odgs::backward(ra, small, fa2, probe, s8);
    CHECK(same_grads(ga, ga_fresh));
    const GradF gb = odgs::backward(rb, small, fb, probe, s8);
    CHECK(!same_grads(ga, gb));
    // vs the fp64 oracle at the reference's FD cutoff, group-relative 1e-3
    oracle::Cloud<double> cd;
    cd.n = ca.n;
    cd.means.assign(ca.means.begin(), ca.means.end()); cd.rotations.assign(ca.rotations.begin(), ca.rotations.end());
    cd.log_scales.assign(ca.log_scales.begin(), ca.log_scales.end());
    cd.raw_opacities.assign(ca.raw_opacities.begin(), ca.raw_opacities.end());
    cd.colors.assign(ca.colors.begin(), ca.colors.end());
    oracle::Settings<double> sd;
    sd.cutoff_sigma = 8.0;
    const auto camd = oracle::identity_camera<double>(64, 32);
    const std::vector<double> probe64(probe_flat.begin(), probe_flat.end());
    const auto od = oracle::backward(cd, camd, oracle::render(cd, camd, sd), probe64, sd);
    CHECK(group_rel(ga.means.v, od.means) < 1e-3);
    CHECK(group_rel(ga.rotations.v, od.rotations) < 1e-3);
    CHECK(group_rel(ga.log_scales.v, od.log_scales) < 1e-3);
    CHECK(group_rel(ga.raw_opacities.v, od.raw_opacities) < 1e-3);
    CHECK(group_rel(ga.colors.v, od.colors) < 1e-3);

    // A context holding one frame: fa's frame is recycled by the next render, so the
    // backward rebuilds it from fa.splats — same gradients bit for bit.
    odgs_b200::Context one(0, nullptr, 1);
    const auto ha = odgs_b200::render<OutF>(one, ra, small, s8);
    const auto hb = odgs_b200::render<OutF>(one, rb, small, s8);
    const GradF g_rebuilt = odgs_b200::backward<GradF>(one, ra, small, ha, probe, s8);
    CHECK(one.rebuilds() == 1);
    CHECK(same_grads(g_rebuilt, ga));
    // a copy of a RenderOutput (new buffers) also works
    const OutF copy = fb;
    CHECK(same_grads(odgs::backward(rb, small, copy, probe, s8), gb));
    // a fwd whose per-pixel state does not follow from its splats is rejected
    OutF tampered = fb;
    tampered.walked(3, 5) += 1;
    bool threw = false;
    try {
      odgs::backward(rb, small, tampered, probe, s8);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    // GradTSigns reaches the T-gradient stage (backward.hpp:32-34)
    odgs::GradTSigns flip;
    flip.sign[0] = -1.0;  // entry (1,1): reaches dJ(0,0), hence the mean gradient
    const GradF gflip = odgs::backward(ra, small, fa, probe, s8, &flip);
    CHECK(!(gflip.means.v == ga.means.v));  // dL/dT feeds the mean gradient (backward.hpp:413-418)
    CHECK(gflip.colors.v == ga.colors.v);
    // the reference-style template caller routes to the GPU (argument-dependent lookup)
    const GradF gv = odgs::view_step(ra, small, probe, s8);
    CHECK(same_grads(gv, ga));
    (void)hb;
  }
  {  // grad_pixels_to_splats (backward.hpp:208-339) vs the float oracle
    std::mt19937 rng(901);
    std::vector<float> flat;
    const ImgF probe = probe_image(rng, 256, 128, &flat);
    const auto fwd = odgs::render(r300, cam, settings);
    const auto sg = odgs::grad_pixels_to_splats(fwd, probe, settings);
    const auto osg = oracle::grad_pixels_to_splats<float, oracle::PortableMath>(o300, flat, oracle::Settings<float>{});
    CHECK(sg.size() == osg.size());
    std::vector<float> a_mean, b_mean, a_cov, b_cov, a_op, b_op, a_col, b_col;
    for (size_t k = 0; k < std::min(sg.size(), osg.size()); ++k) {
      for (int c = 0; c < 2; ++c) { a_mean.push_back(sg[k].pixel_mean[c]); b_mean.push_back(osg[k].pixel_mean[c]); }
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) { a_cov.push_back(sg[k].cov2d(r, c)); b_cov.push_back(osg[k].cov2d(r, c)); }
      a_op.push_back(sg[k].opacity);
      b_op.push_back(osg[k].opacity);
      for (int c = 0; c < 3; ++c) { a_col.push_back(sg[k].color[c]); b_col.push_back(osg[k].color[c]); }
    }
    CHECK(group_rel(a_mean, b_mean) < 1e-3);
    CHECK(group_rel(a_cov, b_cov) < 1e-3);
    CHECK(group_rel(a_op, b_op) < 1e-3);
    CHECK(group_rel(a_col, b_col) < 1e-3);
  }
  {  // project_gaussian (projection.hpp:178-216) vs the portable oracle, every row
    std::mt19937 rng(225);
    auto c = oracle::random_cloud<float>(rng, 400);
    c.mean(7, 0) = 0.0f; c.mean(7, 1) = 0.0f; c.mean(7, 2) = 2000.0f;  // beyond far: nullopt
    c.mean(9, 0) = std::numeric_limits<float>::quiet_NaN();              // NaN depth: nullopt (no throw)
    c.raw_opacities[11] = std::numeric_limits<float>::infinity();        // passes through
    const CloudF rc = to_ref(c);
    bool all = true;
    for (long i = 0; i < 400; ++i) {
      const auto g = odgs::project_gaussian(rc, i, cam, settings);
      const auto o = oracle::project_gaussian<float, oracle::PortableMath>(c, i, ocam, oracle::Settings<float>{});
      if (g.has_value() != o.has_value()) { all = false; continue; }
      if (!g) continue;
      all = all && g->pixel_mean[0] == o->pixel_mean[0] && g->pixel_mean[1] == o->pixel_mean[1] &&
            g->cov2d(0, 0) == o->cov2d(0, 0) && g->cov2d(0, 1) == o->cov2d(0, 1) && g->cov2d(1, 1) == o->cov2d(1, 1) &&
            g->cov2d_inv(0, 0) == o->cov2d_inv(0, 0) && g->cov2d_inv(1, 0) == o->cov2d_inv(1, 0) &&
            g->depth == o->depth && g->radius == o->radius && g->opacity == o->opacity &&
            g->color[0] == o->color[0] && g->index == o->index && g->pole_clamped == o->pole_clamped;
    }
    CHECK(all);
    CHECK(!odgs::project_gaussian(rc, 7, cam, settings).has_value());
    CHECK(!odgs::project_gaussian(rc, 9, cam, settings).has_value());
    CHECK(std::isinf(odgs::project_gaussian(rc, 11, cam, settings)->opacity) == false);
    // test_core.cpp: near-zero quaternion -> std::invalid_argument; non-finite inside the shell too
    CloudF z = rc;
    for (int k = 0; k < 4; ++k) z.rotations(3, k) = 0.0f;
    z.log_scales(4, 1) = std::numeric_limits<float>::infinity();
    int threw = 0;
    try { odgs::project_gaussian(z, 3, cam, settings); } catch (const std::invalid_argument&) { ++threw; }
    try { odgs::project_gaussian(z, 4, cam, settings); } catch (const std::invalid_argument&) { ++threw; }
    CHECK(threw == 2);
  }
  {  // cull (test_rasterizer.cpp:30-51)
    oracle::Cloud<float> c;
    c.resize(3);
    c.mean(0, 2) = 0.05f; c.mean(1, 1) = 1.0f; c.mean(2, 0) = 500.0f;
    auto kept = odgs::cull(to_ref(c), cam, 0.1f, 100.0f);
    CHECK(kept.size() == 1 && kept[0] == 1);
  }
  CHECK(odgs::cpu_calls == 0);  // every float call went to the GPU
  std::printf("dropin_test: %d failures\n", failures);
  return failures == 0 ? 0 : 1;
}
