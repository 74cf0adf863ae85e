// dropin_test.cpp — exercises include/odgs_b200.hpp the way a reference user would:
// with types that have the reference's member names and Eigen's column-major
// storage (Eigen itself is absent from this image, so a minimal stand-in is used),
// checked against the oracle restatement. Cases follow proj/tests/test_rasterizer.cpp
// and test_backward.cpp. Built and run by tests/test_gpu_dropin.py on the GPU box.
#include <cstdio>
#include <limits>
#include <random>

#include "odgs_b200.hpp"
#include "odgs_oracle.hpp"

namespace ref {  // Eigen-layout stand-ins with the reference's member names.
template <class T> struct Array2D {  // Eigen::Matrix/Array, column-major
  std::vector<T> v;
  long r = 0, c = 0;
  void resize(long rows, long cols) { r = rows; c = cols; v.assign((size_t)(rows * cols), T(0)); }
  void setZero(long rows, long cols) { resize(rows, cols); }
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
struct GaussianCloud {
  Array2D<float> means, rotations, log_scales, raw_opacities, colors;
};
struct CameraPose {
  Fixed<float, 3, 3> rotation;
  Fixed<float, 3, 1> translation;
  int width = 0, height = 0;
  CameraPose() { rotation(0, 0) = rotation(1, 1) = rotation(2, 2) = 1; }
};
struct RenderSettings {
  float near_radius = 0.01f, far_radius = 1000.0f;
  int tile_size = 16;
  float alpha_clamp = 0.99f, transmittance_floor = 1e-4f, cutoff_sigma = 3.0f, lowpass_dilation = 0.3f;
  float max_elevation = 85.0f * 3.14159274101257324f / 180.0f;
  int threads = 0;
};
struct ErpImage {
  std::array<Array2D<float>, 3> channel;
};
struct Splat2D {
  Fixed<float, 2, 1> pixel_mean;
  Fixed<float, 2, 2> cov2d, cov2d_inv;
  float depth = 0, radius = 0, opacity = 0;
  Fixed<float, 3, 1> color;
  long index = 0;
  bool pole_clamped = false;
};
struct SplatInstance { int splat; float shift; };
struct RenderOutput {
  ErpImage image;
  Array2D<float> transmittance;
  Array2D<int> walked;
  std::vector<Splat2D> splats;
  std::vector<SplatInstance> instances;
  std::vector<int> tile_offsets, tile_entries;
  int tiles_x = 0, tiles_y = 0;
};
struct GradBuffers {
  Array2D<float> means, rotations, log_scales, raw_opacities, colors, pixel_grad_norm, one_minus_cos;
  Array2D<int> observed;
  void init(long n) {
    means.resize(n, 3); rotations.resize(n, 4); log_scales.resize(n, 3); raw_opacities.resize(n, 1);
    colors.resize(n, 3); pixel_grad_norm.resize(n, 1); one_minus_cos.resize(n, 1); observed.resize(n, 1);
  }
};
}  // namespace ref

static int failures = 0;
#define CHECK(x) do { if (!(x)) { ++failures; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); } } while (0)

static ref::GaussianCloud to_ref(const oracle::Cloud<float>& c) {
  ref::GaussianCloud r;
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

int main() {
  odgs_b200::Context gpu;
  ref::RenderSettings settings;
  ref::CameraPose cam;
  cam.width = 256;
  cam.height = 128;

  {  // test_rasterizer.cpp:110-116 — empty cloud: black, unit transmittance
    ref::GaussianCloud empty;
    empty.means.resize(0, 3); empty.rotations.resize(0, 4); empty.log_scales.resize(0, 3);
    empty.raw_opacities.resize(0, 1); empty.colors.resize(0, 3);
    auto out = odgs_b200::render<ref::RenderOutput>(gpu, empty, cam, settings);
    float mx = 0, mn = 1;
    for (int c = 0; c < 3; ++c) for (float v : out.image.channel[c].v) mx = std::max(mx, std::abs(v));
    for (float v : out.transmittance.v) mn = std::min(mn, v);
    CHECK(mx == 0.0f);
    CHECK(mn == 1.0f);
  }
  {  // test_rasterizer.cpp:118-129 — NaN names the Gaussian
    std::mt19937 rng(5);
    auto c = oracle::random_cloud<float>(rng, 4);
    c.mean(2, 1) = std::numeric_limits<float>::quiet_NaN();
    bool threw = false;
    try {
      odgs_b200::render<ref::RenderOutput>(gpu, to_ref(c), cam, settings);
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find("2") != std::string::npos;
    }
    CHECK(threw);
  }
  {  // bad camera -> std::invalid_argument (types.hpp:159-169)
    std::mt19937 rng(5);
    auto c = oracle::random_cloud<float>(rng, 4);
    ref::CameraPose bad = cam;
    bad.height = 100;
    bool threw = false;
    try {
      odgs_b200::render<ref::RenderOutput>(gpu, to_ref(c), bad, settings);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // every RenderOutput field equals the portable oracle, bit for bit
    std::mt19937 rng(77);
    auto c = oracle::random_cloud<float>(rng, 300);
    auto out = odgs_b200::render<ref::RenderOutput>(gpu, to_ref(c), cam, settings);
    auto o = oracle::render<float, oracle::PortableMath>(c, oracle::identity_camera<float>(256, 128),
                                                        oracle::Settings<float>{});
    CHECK(out.tile_offsets == o.tile_offsets);
    CHECK(out.tile_entries == o.tile_entries);
    CHECK(out.splats.size() == o.splats.size());
    CHECK(out.instances.size() == o.instances.size());
    bool same = out.splats.size() == o.splats.size();
    for (size_t s = 0; same && s < o.splats.size(); ++s)
      same = out.splats[s].index == o.splats[s].index && out.splats[s].pixel_mean[0] == o.splats[s].pixel_mean[0] &&
             out.splats[s].pixel_mean[1] == o.splats[s].pixel_mean[1] && out.splats[s].radius == o.splats[s].radius &&
             out.splats[s].depth == o.splats[s].depth && out.splats[s].cov2d_inv(0, 1) == o.splats[s].cov2d_inv(0, 1);
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
      for (int y = 0; y < 128; ++y) wk = wk && out.walked(y, x) == o.walked[o.px(y, x)];
    CHECK(wk);
  }
  {  // backward vs the fp64 oracle, reference FD settings (cutoff 8), group-relative 1e-3
    ref::RenderSettings s8 = settings;
    s8.cutoff_sigma = 8.0f;
    std::mt19937 rng(137);
    oracle::CloudBounds b;
    b.depth_min = 0.8; b.depth_max = 10.0; b.max_elevation = 75.0 * 3.141592653589793 / 180.0;
    b.opacity_min = 0.1; b.opacity_max = 0.7; b.scale_min = 0.02; b.scale_max = 0.12;
    auto c = oracle::random_cloud<float>(rng, 8, b);
    ref::CameraPose small;
    small.width = 64;
    small.height = 32;
    odgs_b200::render<ref::RenderOutput>(gpu, to_ref(c), small, s8);
    ref::ErpImage probe;
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::vector<double> probe64;
    for (int ch = 0; ch < 3; ++ch) {
      probe.channel[ch].resize(32, 64);
      for (auto& v : probe.channel[ch].v) { v = u(rng); probe64.push_back(v); }
    }
    auto g = odgs_b200::backward<ref::GradBuffers>(gpu, to_ref(c), small, probe, s8);
    oracle::Cloud<double> cd;
    cd.n = c.n;
    cd.means.assign(c.means.begin(), c.means.end()); cd.rotations.assign(c.rotations.begin(), c.rotations.end());
    cd.log_scales.assign(c.log_scales.begin(), c.log_scales.end());
    cd.raw_opacities.assign(c.raw_opacities.begin(), c.raw_opacities.end());
    cd.colors.assign(c.colors.begin(), c.colors.end());
    oracle::Settings<double> sd;
    sd.cutoff_sigma = 8.0;
    const auto camd = oracle::identity_camera<double>(64, 32);
    const auto fd = oracle::render(cd, camd, sd);
    const auto od = oracle::backward(cd, camd, fd, probe64, sd);
    auto group_rel = [](const std::vector<float>& a, const std::vector<double>& b) {
      double md = 0, ma = 0, mb = 0;
      for (size_t k = 0; k < b.size(); ++k) {
        md = std::max(md, std::abs(a[k] - b[k]));
        ma = std::max(ma, (double)std::abs(a[k]));
        mb = std::max(mb, std::abs(b[k]));
      }
      return md / std::max({ma, mb, 1e-12});
    };
    CHECK(group_rel(g.means.v, od.means) < 1e-3);
    CHECK(group_rel(g.rotations.v, od.rotations) < 1e-3);
    CHECK(group_rel(g.log_scales.v, od.log_scales) < 1e-3);
    CHECK(group_rel(g.raw_opacities.v, od.raw_opacities) < 1e-3);
    CHECK(group_rel(g.colors.v, od.colors) < 1e-3);
  }
  {  // cull (test_rasterizer.cpp:30-51)
    oracle::Cloud<float> c;
    c.resize(3);
    c.mean(0, 2) = 0.05f; c.mean(1, 1) = 1.0f; c.mean(2, 0) = 500.0f;
    auto kept = odgs_b200::cull<long>(gpu, to_ref(c), cam, 0.1f, 100.0f);
    CHECK(kept.size() == 1 && kept[0] == 1);
  }
  std::printf("dropin_test: %d failures\n", failures);
  return failures == 0 ? 0 : 1;
}
