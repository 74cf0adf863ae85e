// odgs_oracle.hpp — TEST INFRASTRUCTURE ONLY. Never linked into the product.
//
// An Eigen-free CPU restatement of the reference ODGS hot path (arXiv 2410.20686,
// reference tree proj/include/odgs/). It is the checker the sm_100a kernels are
// compared against; only tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg may load it.
//
// Why a restatement: the reference needs Eigen >= 3.4, libpng and a vendored
// doctest/CLI11/json tree (proj/CMakeLists.txt:10-14), none of which exist in this
// image, so the reference itself cannot be compiled here.
// Every function below cites the reference file:line it restates.
//
// Two template axes:
//   Scalar — float or double (the reference instantiates both; the CLI uses double,
//            proj/tools/odgs.cpp:242).
//   Math   — StdMath: libm std::atan2/hypot/sin/cos/exp, the literal reference
//            semantics. PortableMath: the bit-reproducible functions of
//            include/odgs_portable_math.h that the GPU kernels also use; with it, the
//            float oracle and the GPU agree bit for bit on splats, instance order,
//            tile CSR, walk lengths, transmittance and image.
//
// Eigen evaluation orders the restatement fixes explicitly (Eigen is absent, so they
// cannot be pinned against it): length-2 sums a0+a1, length-3
// sums a0+(a1+a2), length-4 sums (a0+a1)+(a2+a3) — the scalar unroller's halving
// order — for every fixed-size product coefficient, norm and cwise-sum. Build with
// -ffp-contract=off so no expression is fused.
#pragma once

#include <algorithm>
#include <limits>
#include <array>
#include <cmath>
#include <cstdint>
#include <exception>
#include <mutex>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "odgs_portable_math.h"

namespace oracle {

// ------------------------------------------------------------------ math policies

struct StdMath {
  template <class S> static S atan2(S y, S x) { return std::atan2(y, x); }
  template <class S> static S hypot(S x, S y) { return std::hypot(x, y); }
  template <class S> static S sin(S x) { return std::sin(x); }
  template <class S> static S cos(S x) { return std::cos(x); }
  template <class S> static S exp(S x) { return std::exp(x); }
  // The per-pixel exponential of rasterizer.hpp:249 / backward.hpp:264-266.
  template <class S> static S exp_blend(S x) { return std::exp(x); }
  template <class S> static S log(S x) { return std::log(x); }
};

struct PortableMath {
  static float atan2(float y, float x) { return pm_atan2f(y, x); }
  static float hypot(float x, float y) { return pm_hypotf(x, y); }
  static float sin(float x) { return pm_sinf(x); }
  static float cos(float x) { return pm_cosf(x); }
  static float exp(float x) { return pm_expf(x); }
  static float exp_blend(float x) { return pm_expf_blend(x); }
  static float log(float x) { return pm_logf(x); }
};

template <class S> inline constexpr S pi_v = S(3.141592653589793238462643383279502884L);

// ------------------------------------------------------------------ small linear algebra
// Column-vector / row-major-indexed fixed-size types. Only value semantics matter.

template <class S> struct V2 { S v[2]{}; S& operator[](int i) { return v[i]; } S operator[](int i) const { return v[i]; } };
template <class S> struct V3 { S v[3]{}; S& operator[](int i) { return v[i]; } S operator[](int i) const { return v[i]; } };
template <class S> struct V4 { S v[4]{}; S& operator[](int i) { return v[i]; } S operator[](int i) const { return v[i]; } };
template <class S, int R, int C> struct Mat {
  S a[R][C]{};
  S& operator()(int r, int c) { return a[r][c]; }
  S operator()(int r, int c) const { return a[r][c]; }
};
template <class S> using M2 = Mat<S, 2, 2>;
template <class S> using M3 = Mat<S, 3, 3>;
template <class S> using M23 = Mat<S, 2, 3>;

template <class S> inline S sum2(S a, S b) { return a + b; }
template <class S> inline S sum3(S a, S b, S c) { return a + (b + c); }
template <class S> inline S sum4(S a, S b, S c, S d) { return (a + b) + (c + d); }
template <class S> inline S sum6(S a, S b, S c, S d, S e, S f) {
  return (a + (b + c)) + (d + (e + f));
}

// Lazy coefficient product, halving sum order over the inner dimension.
template <class S, int R, int K, int C>
inline Mat<S, R, C> mul(const Mat<S, R, K>& a, const Mat<S, K, C>& b) {
  static_assert(K == 2 || K == 3, "inner dimension");
  Mat<S, R, C> out;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) {
      if constexpr (K == 2)
        out(r, c) = sum2(a(r, 0) * b(0, c), a(r, 1) * b(1, c));
      else
        out(r, c) = sum3(a(r, 0) * b(0, c), a(r, 1) * b(1, c), a(r, 2) * b(2, c));
    }
  return out;
}
template <class S, int R, int C>
inline Mat<S, C, R> transpose(const Mat<S, R, C>& m) {
  Mat<S, C, R> t;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) t(c, r) = m(r, c);
  return t;
}
template <class S> inline V3<S> mulv(const M3<S>& m, const V3<S>& x) {
  V3<S> y;
  for (int r = 0; r < 3; ++r) y[r] = sum3(m(r, 0) * x[0], m(r, 1) * x[1], m(r, 2) * x[2]);
  return y;
}
template <class S> inline S norm3(const V3<S>& x) {
  return std::sqrt(sum3(x[0] * x[0], x[1] * x[1], x[2] * x[2]));
}
template <class S> inline S norm4(const V4<S>& x) {
  return std::sqrt(sum4(x[0] * x[0], x[1] * x[1], x[2] * x[2], x[3] * x[3]));
}
template <class S> inline bool finite(S x) { return std::isfinite(x); }

// ------------------------------------------------------------------ data model
// types.hpp:53-143 GaussianCloud — SoA, Eigen column-major: means(i, c) = means[c*n + i].
template <class S> struct Cloud {
  int64_t n = 0;
  std::vector<S> means, rotations, log_scales, raw_opacities, colors;
  // Extension beyond the reference (SH degree 0 only): view-dependent
  // colour with real spherical harmonics of degree 1..3. sh_rest holds the
  // (deg+1)^2 - 1 non-DC coefficients per channel, layout [basis k][channel c][n]:
  // sh_rest[(3k + c) * n + i]. Degree 0 is exactly the reference's passthrough.
  int sh_degree = 0;
  std::vector<S> sh_rest;
  void resize(int64_t m) {  // types.hpp:63-70
    n = m;
    means.assign(3 * m, S(0));
    rotations.assign(4 * m, S(0));
    for (int64_t i = 0; i < m; ++i) rotations[i] = S(1);
    log_scales.assign(3 * m, S(0));
    raw_opacities.assign(m, S(0));
    colors.assign(3 * m, S(0));
  }
  S& mean(int64_t i, int c) { return means[c * n + i]; }
  S mean(int64_t i, int c) const { return means[c * n + i]; }
  S& rot(int64_t i, int c) { return rotations[c * n + i]; }
  S rot(int64_t i, int c) const { return rotations[c * n + i]; }
  S& ls(int64_t i, int c) { return log_scales[c * n + i]; }
  S ls(int64_t i, int c) const { return log_scales[c * n + i]; }
  S& col(int64_t i, int c) { return colors[c * n + i]; }
  S col(int64_t i, int c) const { return colors[c * n + i]; }
  V3<S> mean_v(int64_t i) const { return {{mean(i, 0), mean(i, 1), mean(i, 2)}}; }
  V4<S> rot_v(int64_t i) const { return {{rot(i, 0), rot(i, 1), rot(i, 2), rot(i, 3)}}; }
  V3<S> ls_v(int64_t i) const { return {{ls(i, 0), ls(i, 1), ls(i, 2)}}; }

  // types.hpp:123-131
  int64_t first_non_finite() const {
    for (int64_t i = 0; i < n; ++i) {
      bool ok = true;
      for (int c = 0; c < 3; ++c) ok = ok && finite(mean(i, c));
      for (int c = 0; c < 4; ++c) ok = ok && finite(rot(i, c));
      for (int c = 0; c < 3; ++c) ok = ok && finite(ls(i, c));
      ok = ok && finite(raw_opacities[i]);
      for (int c = 0; c < 3; ++c) ok = ok && finite(col(i, c));
      if (sh_degree > 0)
        for (int k = 0; k < 3 * ((sh_degree + 1) * (sh_degree + 1) - 1); ++k) ok = ok && finite(sh_rest[k * n + i]);
      if (!ok) return i;
    }
    return -1;
  }
};

// types.hpp:28-39
template <class S, class M = StdMath> inline S sigmoid(S x) { return S(1) / (S(1) + M::exp(-x)); }
template <class S, class M = StdMath> inline S logit(S x) {
  if (!(x > S(0) && x < S(1))) throw std::invalid_argument("logit: argument must lie in (0, 1)");
  return M::log(x / (S(1) - x));
}

// types.hpp:148-180 CameraPose (y-down, z-forward; W == 2H).
template <class S> struct Camera {
  M3<S> rotation{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  V3<S> translation{};
  int width = 0, height = 0;
  V3<S> to_camera(const V3<S>& p) const {  // types.hpp:155-157
    V3<S> rp = mulv(rotation, p);
    return {{rp[0] + translation[0], rp[1] + translation[1], rp[2] + translation[2]}};
  }
  void validate() const {  // types.hpp:159-169
    if (width <= 0 || height <= 0 || width != 2 * height)
      throw std::invalid_argument("CameraPose: equirectangular image needs width == 2 * height > 0");
    const M3<S> rrt = mul(rotation, transpose(rotation));
    S err = 0;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) err = std::max(err, std::abs(rrt(r, c) - (r == c ? S(1) : S(0))));
    if (!(err < S(1e-5))) throw std::invalid_argument("CameraPose: rotation is not orthonormal");
  }
};

// types.hpp:229-255 RenderSettings.
template <class S> struct Settings {
  S near_radius = S(0.01);
  S far_radius = S(1000);
  int tile_size = 16;
  S alpha_clamp = S(0.99);
  S transmittance_floor = S(1e-4);
  S cutoff_sigma = S(3);
  S lowpass_dilation = S(0.3);
  S max_elevation = S(85) * pi_v<S> / S(180);
  int threads = 0;
};

// ------------------------------------------------------------------ parallel.hpp:13-53
inline int effective_threads(int requested) {
  if (requested > 0) return requested;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}
template <class Fn> void parallel_for(int begin, int end, int threads, Fn&& fn) {
  const int n = end - begin;
  if (n <= 0) return;
  const int workers = std::min(effective_threads(threads), n);
  if (workers <= 1) {
    for (int i = begin; i < end; ++i) fn(i);
    return;
  }
  std::exception_ptr error;
  std::mutex error_mutex;
  std::vector<std::thread> pool;
  pool.reserve(static_cast<std::size_t>(workers));
  const int block = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int lo = begin + w * block;
    const int hi = std::min(end, lo + block);
    if (lo >= hi) break;
    pool.emplace_back([&, lo, hi] {
      try {
        for (int i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        std::lock_guard lock(error_mutex);
        if (!error) error = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  if (error) std::rethrow_exception(error);
}

// ------------------------------------------------------------------ covariance.hpp:11-37
template <class S> inline V4<S> normalize_quaternion(const V4<S>& q) {
  const S n = norm4(q);
  if (!(n > S(1e-12))) throw std::invalid_argument("normalize_quaternion: near-zero quaternion");
  return {{q[0] / n, q[1] / n, q[2] / n, q[3] / n}};
}
// Eigen::Quaternion(w,x,y,z).toRotationMatrix() (covariance.hpp:22), SURVEY Appendix B.
template <class S> inline M3<S> quaternion_matrix(const V4<S>& q) {
  const S w = q[0], x = q[1], y = q[2], z = q[3];
  const S tx = S(2) * x, ty = S(2) * y, tz = S(2) * z;
  const S twx = tx * w, twy = ty * w, twz = tz * w;
  const S txx = tx * x, txy = ty * x, txz = tz * x;
  const S tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3<S> r;
  r(0, 0) = S(1) - (tyy + tzz); r(0, 1) = txy - twz;          r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;          r(1, 1) = S(1) - (txx + tzz); r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;          r(2, 1) = tyz + twx;          r(2, 2) = S(1) - (txx + tyy);
  return r;
}
template <class S> inline M3<S> rotation_from_quaternion(const V4<S>& q_raw) {
  return quaternion_matrix(normalize_quaternion(q_raw));
}
template <class S, class M = StdMath>
inline M3<S> build_covariance(const V4<S>& q, const V3<S>& log_scales) {
  for (int c = 0; c < 4; ++c)
    if (!finite(q[c])) throw std::invalid_argument("build_covariance: non-finite parameters");
  for (int c = 0; c < 3; ++c)
    if (!finite(log_scales[c])) throw std::invalid_argument("build_covariance: non-finite parameters");
  const M3<S> r = rotation_from_quaternion(q);
  const S s[3] = {M::exp(log_scales[0]), M::exp(log_scales[1]), M::exp(log_scales[2])};
  M3<S> m;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) m(i, k) = r(i, k) * s[k];
  return mul(m, transpose(m));
}

// ------------------------------------------------------------------ projection.hpp:19-216
template <class S> struct SphericalAngles { S azimuth, elevation; };

template <class S, class M = StdMath>
inline SphericalAngles<S> to_spherical(const V3<S>& mu) {  // projection.hpp:19-29
  if (!(sum3(mu[0] * mu[0], mu[1] * mu[1], mu[2] * mu[2]) > S(0)))
    throw std::domain_error("to_spherical: degenerate zero-length direction");
  const S phi = M::atan2(mu[0], mu[2]);
  const S rho = M::hypot(mu[0], mu[2]);
  const S theta = M::atan2(-mu[1], rho);
  return {phi, theta};
}

template <class S, class M = StdMath>
inline V2<S> project_center(const V3<S>& mu, S width, S height) {  // projection.hpp:33-39
  const auto a = to_spherical<S, M>(mu);
  return {{width / (S(2) * pi_v<S>) * a.azimuth + width / S(2),
           -height / pi_v<S> * a.elevation + height / S(2)}};
}

template <class S, class M = StdMath>
inline M3<S> tangent_rotation(const SphericalAngles<S>& a) {  // projection.hpp:43-55
  const S cp = M::cos(a.azimuth), sp = M::sin(a.azimuth);
  const S ct = M::cos(a.elevation), st = M::sin(a.elevation);
  M3<S> t_phi{{{cp, 0, -sp}, {0, 1, 0}, {sp, 0, cp}}};
  M3<S> t_theta{{{1, 0, 0}, {0, ct, st}, {0, -st, ct}}};
  return mul(t_theta, t_phi);
}

template <class S>
inline M23<S> perspective_jacobian(const V3<S>& mu, S fx, S fy) {  // projection.hpp:58-68
  const S x = mu[0], y = mu[1], z = mu[2];
  if (!(z > S(0))) throw std::domain_error("perspective_jacobian: point is behind the camera");
  return {{{fx / z, 0, -fx * x / (z * z)}, {0, fy / z, -fy * y / (z * z)}}};
}

inline constexpr double kDefaultMaxElevation = 85.0 * 3.14159265358979323846 / 180.0;

template <class S, class M = StdMath>
inline M23<S> jacobian_omni_factored(const V3<S>& mu, S width, S height,
                                     S max_elevation = S(kDefaultMaxElevation),
                                     bool* clamped = nullptr) {  // projection.hpp:75-96
  const auto angles = to_spherical<S, M>(mu);
  const S r = norm3(mu);
  const bool clamp = std::abs(angles.elevation) > max_elevation;
  if (clamped) *clamped = clamp;
  const S sec = S(1) / M::cos(clamp ? max_elevation : std::abs(angles.elevation));
  Mat<S, 2, 3> j_o{{{S(1) / r, 0, 0}, {0, S(1) / r, 0}}};
  M2<S> q_o{{{sec, 0}, {0, 1}}};
  M2<S> s_o{{{width / (S(2) * pi_v<S>), 0}, {0, height / pi_v<S>}}};
  return mul(mul(mul(s_o, q_o), j_o), tangent_rotation<S, M>(angles));
}

template <class S, class M = StdMath>
inline M23<S> jacobian_omni_closed(const V3<S>& mu, S width, S height) {  // projection.hpp:100-114
  const auto a = to_spherical<S, M>(mu);
  const S r = norm3(mu);
  const S cp = M::cos(a.azimuth), sp = M::sin(a.azimuth);
  const S ct = M::cos(a.elevation), st = M::sin(a.elevation);
  const S sec = S(1) / ct;
  const S kw = width / (S(2) * pi_v<S> * r);
  const S kh = height / (pi_v<S> * r);
  return {{{kw * sec * cp, 0, -kw * sec * sp}, {kh * st * sp, kh * ct, kh * st * cp}}};
}

template <class S>
inline M23<S> jacobian_omni_direct(const V3<S>& mu, S width, S height) {  // projection.hpp:118-133
  const S x = mu[0], y = mu[1], z = mu[2];
  const S rho2 = x * x + z * z;
  if (!(rho2 > S(0))) throw std::domain_error("jacobian_omni_direct: derivative undefined at the pole");
  const S rho = std::sqrt(rho2);
  const S r2 = rho2 + y * y;
  const S kw = width / (S(2) * pi_v<S>);
  const S kh = height / pi_v<S>;
  return {{{kw * z / rho2, 0, -kw * x / rho2},
           {-kh * x * y / (rho * r2), kh * rho / r2, -kh * y * z / (rho * r2)}}};
}

template <class S, class M = StdMath>
inline M23<S> jacobian_omni(const V3<S>& mu, S width, S height,
                            S max_elevation = S(kDefaultMaxElevation), bool* clamped = nullptr) {
  return jacobian_omni_factored<S, M>(mu, width, height, max_elevation, clamped);
}

template <class S>
inline M2<S> project_covariance(const M3<S>& sigma_world, const M3<S>& world_rot,
                                const M23<S>& j, S lowpass = S(0.3)) {  // projection.hpp:146-158
  const M23<S> t = mul(j, world_rot);
  M2<S> cov = mul(mul(t, sigma_world), transpose(t));
  cov(1, 0) = cov(0, 1) = (cov(0, 1) + cov(1, 0)) / S(2);
  cov(0, 0) += lowpass;
  cov(1, 1) += lowpass;
  return cov;
}

// ------------------------------------------------------------------ SH colour (extension)
// Real SH basis of degrees 1..3 (the usual 3DGS convention) at unit direction d.
inline constexpr int sh_count(int degree) { return (degree + 1) * (degree + 1) - 1; }

template <class S> inline void sh_basis(int degree, S x, S y, S z, S Y[15]) {
  const S C1 = S(0.4886025119029199);
  const S C2[5] = {S(1.0925484305920792), S(-1.0925484305920792), S(0.31539156525252005), S(-1.0925484305920792),
                   S(0.5462742152960396)};
  const S C3[7] = {S(-0.5900435899266435), S(2.890611442640554), S(-0.4570457994644658), S(0.3731763325901154),
                   S(-0.4570457994644658), S(1.445305721320277), S(-0.5900435899266435)};
  Y[0] = -C1 * y;
  Y[1] = C1 * z;
  Y[2] = -C1 * x;
  if (degree < 2) return;
  const S xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[3] = C2[0] * xy;
  Y[4] = C2[1] * yz;
  Y[5] = C2[2] * (S(2) * zz - xx - yy);
  Y[6] = C2[3] * xz;
  Y[7] = C2[4] * (xx - yy);
  if (degree < 3) return;
  Y[8] = C3[0] * y * (S(3) * xx - yy);
  Y[9] = C3[1] * xy * z;
  Y[10] = C3[2] * y * (S(4) * zz - xx - yy);
  Y[11] = C3[3] * z * (S(2) * zz - S(3) * xx - S(3) * yy);
  Y[12] = C3[4] * x * (S(4) * zz - xx - yy);
  Y[13] = C3[5] * z * (xx - yy);
  Y[14] = C3[6] * x * (xx - S(3) * yy);
}

// d Y_k / d(x, y, z) for the basis above.
template <class S> inline void sh_basis_grad(int degree, S x, S y, S z, S dY[15][3]) {
  const S C1 = S(0.4886025119029199);
  const S C2[5] = {S(1.0925484305920792), S(-1.0925484305920792), S(0.31539156525252005), S(-1.0925484305920792),
                   S(0.5462742152960396)};
  const S C3[7] = {S(-0.5900435899266435), S(2.890611442640554), S(-0.4570457994644658), S(0.3731763325901154),
                   S(-0.4570457994644658), S(1.445305721320277), S(-0.5900435899266435)};
  const S d1[3][3] = {{0, -C1, 0}, {0, 0, C1}, {-C1, 0, 0}};
  for (int k = 0; k < 3; ++k)
    for (int a = 0; a < 3; ++a) dY[k][a] = d1[k][a];
  if (degree < 2) return;
  const S xx = x * x, yy = y * y, zz = z * z;
  const S g2[5][3] = {{C2[0] * y, C2[0] * x, 0},
                      {0, C2[1] * z, C2[1] * y},
                      {S(-2) * C2[2] * x, S(-2) * C2[2] * y, S(4) * C2[2] * z},
                      {C2[3] * z, 0, C2[3] * x},
                      {S(2) * C2[4] * x, S(-2) * C2[4] * y, 0}};
  for (int k = 0; k < 5; ++k)
    for (int a = 0; a < 3; ++a) dY[3 + k][a] = g2[k][a];
  if (degree < 3) return;
  const S g3[7][3] = {{S(6) * C3[0] * x * y, C3[0] * (S(3) * xx - S(3) * yy), 0},
                      {C3[1] * y * z, C3[1] * x * z, C3[1] * x * y},
                      {S(-2) * C3[2] * x * y, C3[2] * (S(4) * zz - xx - S(3) * yy), S(8) * C3[2] * y * z},
                      {S(-6) * C3[3] * x * z, S(-6) * C3[3] * y * z, C3[3] * (S(6) * zz - S(3) * xx - S(3) * yy)},
                      {C3[4] * (S(4) * zz - S(3) * xx - yy), S(-2) * C3[4] * x * y, S(8) * C3[4] * x * z},
                      {S(2) * C3[5] * x * z, S(-2) * C3[5] * y * z, C3[5] * (xx - yy)},
                      {C3[6] * (S(3) * xx - S(3) * yy), S(-6) * C3[6] * x * y, 0}};
  for (int k = 0; k < 7; ++k)
    for (int a = 0; a < 3; ++a) dY[8 + k][a] = g3[k][a];
}

// Unit view direction from the camera centre c = -R^T t to the Gaussian (world frame)
// and the distance; zero direction if the Gaussian sits at the centre.
template <class S> inline S sh_direction(const Camera<S>& cam, const V3<S>& p, S d[3]) {
  S v[3];
  for (int k = 0; k < 3; ++k) {
    const S cc = -sum3(cam.rotation(0, k) * cam.translation[0], cam.rotation(1, k) * cam.translation[1],
                       cam.rotation(2, k) * cam.translation[2]);
    v[k] = p[k] - cc;
  }
  const S len = std::sqrt(sum3(v[0] * v[0], v[1] * v[1], v[2] * v[2]));
  for (int k = 0; k < 3; ++k) d[k] = len > S(0) ? v[k] / len : S(0);
  return len;
}

template <class S> inline V3<S> sh_color(const Cloud<S>& cloud, int64_t i, const Camera<S>& cam) {
  V3<S> c{{cloud.col(i, 0), cloud.col(i, 1), cloud.col(i, 2)}};
  if (cloud.sh_degree <= 0) return c;
  S d[3], Y[15];
  sh_direction(cam, cloud.mean_v(i), d);
  sh_basis(cloud.sh_degree, d[0], d[1], d[2], Y);
  const int nb = sh_count(cloud.sh_degree);
  for (int ch = 0; ch < 3; ++ch)
    for (int k = 0; k < nb; ++k) c[ch] = c[ch] + Y[k] * cloud.sh_rest[(3 * k + ch) * cloud.n + i];
  return c;
}

template <class S> struct Splat2D {  // projection.hpp:163-174
  V2<S> pixel_mean;
  M2<S> cov2d, cov2d_inv;
  S depth = 0, radius = 0, opacity = 0;
  V3<S> color;
  int64_t index = 0;
  bool pole_clamped = false;
};

template <class S, class M = StdMath>
inline std::optional<Splat2D<S>> project_gaussian(const Cloud<S>& cloud, int64_t i,
                                                  const Camera<S>& camera,
                                                  const Settings<S>& settings) {  // projection.hpp:178-216
  const V3<S> mu = camera.to_camera(cloud.mean_v(i));
  const S depth = norm3(mu);
  if (!(depth >= settings.near_radius && depth <= settings.far_radius)) return std::nullopt;
  Splat2D<S> splat;
  splat.pixel_mean = project_center<S, M>(mu, S(camera.width), S(camera.height));
  const M23<S> j = jacobian_omni<S, M>(mu, S(camera.width), S(camera.height),
                                       settings.max_elevation, &splat.pole_clamped);
  const M3<S> sigma = build_covariance<S, M>(cloud.rot_v(i), cloud.ls_v(i));
  splat.cov2d = project_covariance(sigma, camera.rotation, j, settings.lowpass_dilation);
  const M2<S>& c = splat.cov2d;
  const S det = c(0, 0) * c(1, 1) - c(1, 0) * c(0, 1);  // Eigen 2x2 determinant
  bool fin = finite(c(0, 0)) && finite(c(0, 1)) && finite(c(1, 0)) && finite(c(1, 1));
  if (!(det > S(0)) || !fin) return std::nullopt;
  splat.cov2d_inv(0, 0) = c(1, 1) / det;
  splat.cov2d_inv(0, 1) = -c(0, 1) / det;
  splat.cov2d_inv(1, 0) = -c(0, 1) / det;
  splat.cov2d_inv(1, 1) = c(0, 0) / det;
  const S mid = (c(0, 0) + c(1, 1)) / S(2);
  const S lambda_max = mid + std::sqrt(std::max(S(0), mid * mid - det));
  splat.radius = settings.cutoff_sigma * std::sqrt(lambda_max);
  splat.depth = depth;
  splat.opacity = sigmoid<S, M>(cloud.raw_opacities[i]);
  splat.color = sh_color(cloud, i, camera);  // degree 0: the reference's passthrough
  splat.index = i;
  return splat;
}

// ------------------------------------------------------------------ rasterizer.hpp:15-267
template <class S>
inline std::vector<int64_t> cull(const Cloud<S>& cloud, const Camera<S>& camera, S near, S far) {
  if (!(S(0) < near && near < far)) throw std::invalid_argument("cull: need 0 < near < far");
  std::vector<int64_t> visible;
  for (int64_t i = 0; i < cloud.n; ++i) {
    const S d = norm3(camera.to_camera(cloud.mean_v(i)));
    if (d >= near && d <= far) visible.push_back(i);
  }
  return visible;
}

template <class S, class M = StdMath>
inline S eval_splat(const Splat2D<S>& s, const V2<S>& x, S shift = S(0)) {  // rasterizer.hpp:32-41
  const S dx = x[0] - (s.pixel_mean[0] + shift);
  const S dy = x[1] - s.pixel_mean[1];
  const S d2 = s.cov2d_inv(0, 0) * dx * dx + S(2) * s.cov2d_inv(0, 1) * dx * dy +
               s.cov2d_inv(1, 1) * dy * dy;
  return M::exp_blend(-d2 / S(2));
}

template <class S> struct PixelComposite {
  V3<S> color{};
  S transmittance = S(1);
  int composited = 0;
};

template <class S, class M = StdMath>
inline PixelComposite<S> composite_pixel(const std::vector<std::pair<Splat2D<S>, S>>& stack,
                                         const V2<S>& x, const Settings<S>& settings) {  // :55-77
  const S cutoff2 = settings.cutoff_sigma * settings.cutoff_sigma;
  PixelComposite<S> out;
  for (const auto& [splat, shift] : stack) {
    const S dx = x[0] - (splat.pixel_mean[0] + shift);
    const S dy = x[1] - splat.pixel_mean[1];
    const S d2 = splat.cov2d_inv(0, 0) * dx * dx + S(2) * splat.cov2d_inv(0, 1) * dx * dy +
                 splat.cov2d_inv(1, 1) * dy * dy;
    if (d2 > cutoff2) continue;
    const S alpha = std::min(settings.alpha_clamp, splat.opacity * M::exp_blend(-d2 / S(2)));
    const S t_next = out.transmittance * (S(1) - alpha);
    if (t_next < settings.transmittance_floor) break;
    const S w = alpha * out.transmittance;
    for (int c = 0; c < 3; ++c) out.color[c] += splat.color[c] * w;
    out.transmittance = t_next;
    ++out.composited;
  }
  return out;
}

template <class S> struct SplatInstance { int splat; S shift; };  // rasterizer.hpp:81-85

// rasterizer.hpp:92-102. Images are planar, each channel column-major (y + x*H),
// exactly Eigen::ArrayXX's storage (types.hpp:186).
template <class S> struct RenderOutput {
  int width = 0, height = 0;
  std::vector<S> image;           // [3][W][H]
  std::vector<S> transmittance;   // [W][H]
  std::vector<int32_t> walked;    // [W][H]
  std::vector<Splat2D<S>> splats;
  std::vector<SplatInstance<S>> instances;
  std::vector<int> tile_offsets, tile_entries;
  int tiles_x = 0, tiles_y = 0;
  // Work counters for the roofline (not in the reference): entries examined and
  // entries composited, summed over pixels.
  int64_t e_exam = 0, e_contrib = 0;
  S& img(int c, int y, int x) { return image[(std::size_t)c * width * height + (std::size_t)x * height + y]; }
  S img(int c, int y, int x) const { return image[(std::size_t)c * width * height + (std::size_t)x * height + y]; }
  std::size_t px(int y, int x) const { return (std::size_t)x * height + y; }
};

// Float -> int with the reference's static_cast<int>(std::floor(v)) semantics for
// in-range values; out-of-range values (UB in the reference) saturate to +-2^30,
// which is what the GPU does too.
template <class S> inline int floor_to_int(S v) {
  S f = std::floor(v);
  if (!(f >= S(-1073741824))) f = S(-1073741824);
  if (f > S(1073741824)) f = S(1073741824);
  return static_cast<int>(f);
}

template <class S>
inline bool instance_box(const Splat2D<S>& splat, S shift, int width, int height, int box[4]) {  // :107-122
  const S cx = splat.pixel_mean[0] + shift;
  const S cy = splat.pixel_mean[1];
  const S r = splat.radius;
  const int x0 = std::max(0, floor_to_int(cx - r - S(0.5)) + 1);
  const int x1 = std::min(width - 1, floor_to_int(cx + r - S(0.5)));
  const int y0 = std::max(0, floor_to_int(cy - r - S(0.5)) + 1);
  const int y1 = std::min(height - 1, floor_to_int(cy + r - S(0.5)));
  if (x0 > x1 || y0 > y1) return false;
  box[0] = x0; box[1] = x1; box[2] = y0; box[3] = y1;
  return true;
}

template <class S> inline void bin_splats(RenderOutput<S>& out, const Settings<S>& settings);

template <class S, class M = StdMath>
inline RenderOutput<S> prepare_render(const Cloud<S>& cloud, const Camera<S>& camera,
                                      const Settings<S>& settings) {  // rasterizer.hpp:129-207
  camera.validate();
  if (const int64_t bad = cloud.first_non_finite(); bad >= 0)
    throw std::runtime_error("render: non-finite parameter in Gaussian " + std::to_string(bad));
  RenderOutput<S> out;
  const int width = camera.width, height = camera.height;
  out.width = width;
  out.height = height;
  for (int64_t i = 0; i < cloud.n; ++i)
    if (auto s = project_gaussian<S, M>(cloud, i, camera, settings)) out.splats.push_back(*s);
  bin_splats(out, settings);
  return out;
}

// The rest of prepare_render once out.splats is filled (rasterizer.hpp:141-205): seam
// instances, the (depth, index, shift) order and the tile CSR.
template <class S> inline void bin_splats(RenderOutput<S>& out, const Settings<S>& settings) {
  const int width = out.width, height = out.height;
  const S shifts[3] = {-S(width), S(0), S(width)};
  for (int s = 0; s < static_cast<int>(out.splats.size()); ++s) {
    int box[4];
    for (const S shift : shifts)
      if (instance_box(out.splats[(std::size_t)s], shift, width, height, box))
        out.instances.push_back({s, shift});
  }
  std::sort(out.instances.begin(), out.instances.end(),
            [&](const SplatInstance<S>& a, const SplatInstance<S>& b) {
              const auto& sa = out.splats[(std::size_t)a.splat];
              const auto& sb = out.splats[(std::size_t)b.splat];
              if (sa.depth != sb.depth) return sa.depth < sb.depth;
              if (sa.index != sb.index) return sa.index < sb.index;
              return a.shift < b.shift;
            });

  out.tiles_x = (width + settings.tile_size - 1) / settings.tile_size;
  out.tiles_y = (height + settings.tile_size - 1) / settings.tile_size;
  const int n_tiles = out.tiles_x * out.tiles_y;
  out.tile_offsets.assign((std::size_t)n_tiles + 1, 0);
  auto tile_span = [&](const SplatInstance<S>& inst, int span[4]) {
    int box[4];
    if (!instance_box(out.splats[(std::size_t)inst.splat], inst.shift, width, height, box)) return false;
    for (int k = 0; k < 4; ++k) span[k] = box[k] / settings.tile_size;
    return true;
  };
  for (const auto& inst : out.instances) {
    int span[4];
    if (!tile_span(inst, span)) continue;
    for (int ty = span[2]; ty <= span[3]; ++ty)
      for (int tx = span[0]; tx <= span[1]; ++tx)
        ++out.tile_offsets[(std::size_t)(ty * out.tiles_x + tx) + 1];
  }
  for (std::size_t t = 1; t < out.tile_offsets.size(); ++t) out.tile_offsets[t] += out.tile_offsets[t - 1];
  out.tile_entries.resize((std::size_t)out.tile_offsets.back());
  std::vector<int> cursor(out.tile_offsets.begin(), out.tile_offsets.end() - 1);
  for (int e = 0; e < static_cast<int>(out.instances.size()); ++e) {
    int span[4];
    if (!tile_span(out.instances[(std::size_t)e], span)) continue;
    for (int ty = span[2]; ty <= span[3]; ++ty)
      for (int tx = span[0]; tx <= span[1]; ++tx)
        out.tile_entries[(std::size_t)(cursor[(std::size_t)(ty * out.tiles_x + tx)]++)] = e;
  }
}

// The blend of render (rasterizer.hpp:216-267) over a prepared output.
template <class S, class M = StdMath> inline void blend_tiles(RenderOutput<S>& out, const Settings<S>& settings) {
  const int width = out.width, height = out.height;
  out.image.assign((std::size_t)3 * width * height, S(0));
  out.transmittance.assign((std::size_t)width * height, S(1));
  out.walked.assign((std::size_t)width * height, 0);
  const S cutoff2 = settings.cutoff_sigma * settings.cutoff_sigma;
  const int n_tiles = out.tiles_x * out.tiles_y;
  std::vector<int64_t> tile_exam((std::size_t)n_tiles, 0), tile_contrib((std::size_t)n_tiles, 0);
  parallel_for(0, n_tiles, settings.threads, [&](int tile) {
    const int tx = tile % out.tiles_x, ty = tile / out.tiles_x;
    const int x0 = tx * settings.tile_size, y0 = ty * settings.tile_size;
    const int x1 = std::min(width, x0 + settings.tile_size);
    const int y1 = std::min(height, y0 + settings.tile_size);
    const int e0 = out.tile_offsets[(std::size_t)tile];
    const int e1 = out.tile_offsets[(std::size_t)tile + 1];
    int64_t exam = 0, contrib = 0;
    for (int py = y0; py < y1; ++py) {
      for (int px = x0; px < x1; ++px) {
        const S pix0 = S(px) + S(0.5), pix1 = S(py) + S(0.5);
        S t = S(1);
        S color[3] = {0, 0, 0};
        int walked = e1 - e0;
        for (int e = e0; e < e1; ++e) {
          const auto& inst = out.instances[(std::size_t)out.tile_entries[(std::size_t)e]];
          const auto& splat = out.splats[(std::size_t)inst.splat];
          const S dx = pix0 - (splat.pixel_mean[0] + inst.shift);
          const S dy = pix1 - splat.pixel_mean[1];
          const S d2 = splat.cov2d_inv(0, 0) * dx * dx + S(2) * splat.cov2d_inv(0, 1) * dx * dy +
                       splat.cov2d_inv(1, 1) * dy * dy;
          ++exam;
          if (d2 > cutoff2) continue;
          const S alpha = std::min(settings.alpha_clamp, splat.opacity * M::exp_blend(-d2 / S(2)));
          const S t_next = t * (S(1) - alpha);
          if (t_next < settings.transmittance_floor) {
            walked = e - e0;
            break;
          }
          ++contrib;
          const S w = alpha * t;
          for (int c = 0; c < 3; ++c) color[c] += splat.color[c] * w;
          t = t_next;
        }
        for (int c = 0; c < 3; ++c) out.img(c, py, px) = color[c];
        out.transmittance[out.px(py, px)] = t;
        out.walked[out.px(py, px)] = walked;
      }
    }
    tile_exam[(std::size_t)tile] = exam;
    tile_contrib[(std::size_t)tile] = contrib;
  });
  out.e_exam = std::accumulate(tile_exam.begin(), tile_exam.end(), int64_t(0));
  out.e_contrib = std::accumulate(tile_contrib.begin(), tile_contrib.end(), int64_t(0));
}

template <class S, class M = StdMath>
inline RenderOutput<S> render(const Cloud<S>& cloud, const Camera<S>& camera,
                              const Settings<S>& settings) {  // rasterizer.hpp:211-267
  RenderOutput<S> out = prepare_render<S, M>(cloud, camera, settings);
  blend_tiles<S, M>(out, settings);
  return out;
}

// Sort, bin and blend given splats (the stages of render after projection): what
// odgs_rasterize_splats computes on the GPU.
template <class S, class M = StdMath>
inline RenderOutput<S> rasterize_splats(const std::vector<Splat2D<S>>& splats, int width, int height,
                                        const Settings<S>& settings) {
  RenderOutput<S> out;
  out.width = width;
  out.height = height;
  out.splats = splats;
  bin_splats(out, settings);
  blend_tiles<S, M>(out, settings);
  return out;
}

// Brute-force renderer of the reference's test oracle (proj/tests/oracle.hpp:19-85):
// no tiles; every seam instance at every pixel; own 2x2 inverse.
template <class S, class M = StdMath>
inline std::vector<S> brute_force_render(const Cloud<S>& cloud, const Camera<S>& camera,
                                         const Settings<S>& settings) {
  struct Inst { Splat2D<S> splat; S shift, inv00, inv01, inv11; };
  std::vector<Inst> instances;
  for (int64_t i = 0; i < cloud.n; ++i) {
    auto s = project_gaussian<S, M>(cloud, i, camera, settings);
    if (!s) continue;
    const S det = s->cov2d(0, 0) * s->cov2d(1, 1) - s->cov2d(0, 1) * s->cov2d(0, 1);
    for (const S shift : {-S(camera.width), S(0), S(camera.width)})
      instances.push_back({*s, shift, s->cov2d(1, 1) / det, -s->cov2d(0, 1) / det, s->cov2d(0, 0) / det});
  }
  std::sort(instances.begin(), instances.end(), [](const Inst& a, const Inst& b) {
    if (a.splat.depth != b.splat.depth) return a.splat.depth < b.splat.depth;
    if (a.splat.index != b.splat.index) return a.splat.index < b.splat.index;
    return a.shift < b.shift;
  });
  const S cutoff2 = settings.cutoff_sigma * settings.cutoff_sigma;
  const int W = camera.width, H = camera.height;
  std::vector<S> image((std::size_t)3 * W * H, S(0));
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      const S cx = S(px) + S(0.5), cy = S(py) + S(0.5);
      S t = S(1);
      S color[3] = {0, 0, 0};
      for (const Inst& inst : instances) {
        const S dx = cx - (inst.splat.pixel_mean[0] + inst.shift);
        const S dy = cy - inst.splat.pixel_mean[1];
        const S d2 = inst.inv00 * dx * dx + S(2) * inst.inv01 * dx * dy + inst.inv11 * dy * dy;
        if (d2 > cutoff2) continue;
        const S alpha = std::min(settings.alpha_clamp, inst.splat.opacity * M::exp_blend(-d2 / S(2)));
        const S t_next = t * (S(1) - alpha);
        if (t_next < settings.transmittance_floor) break;
        const S w = alpha * t;
        for (int c = 0; c < 3; ++c) color[c] += inst.splat.color[c] * w;
        t = t_next;
      }
      for (int c = 0; c < 3; ++c) image[(std::size_t)c * W * H + (std::size_t)px * H + py] = color[c];
    }
  return image;
}

// ------------------------------------------------------------------ backward.hpp:19-448
template <class S> struct SplatGrads {  // backward.hpp:19-25
  V2<S> pixel_mean;
  M2<S> cov2d;
  S opacity = 0;
  V3<S> color;
};

struct GradTSigns {  // backward.hpp:32-34
  std::array<double, 12> sign{{1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1}};
};

template <class S>
inline M23<S> grad_T(const M23<S>& t, const M3<S>& v, const M2<S>& dl_dcov2d,
                     const GradTSigns* signs = nullptr) {  // backward.hpp:42-68
  static const GradTSigns unit;
  const auto& s = (signs ? *signs : unit).sign;
  const S d11 = dl_dcov2d(0, 0), d22 = dl_dcov2d(1, 1);
  const S d12 = dl_dcov2d(0, 1) + dl_dcov2d(1, 0);
  const S a0 = t(0, 0) * v(0, 0) + t(0, 1) * v(0, 1) + t(0, 2) * v(0, 2);
  const S a1 = t(0, 0) * v(1, 0) + t(0, 1) * v(1, 1) + t(0, 2) * v(1, 2);
  const S a2 = t(0, 0) * v(2, 0) + t(0, 1) * v(2, 1) + t(0, 2) * v(2, 2);
  const S b0 = t(1, 0) * v(0, 0) + t(1, 1) * v(0, 1) + t(1, 2) * v(0, 2);
  const S b1 = t(1, 0) * v(1, 0) + t(1, 1) * v(1, 1) + t(1, 2) * v(1, 2);
  const S b2 = t(1, 0) * v(2, 0) + t(1, 1) * v(2, 1) + t(1, 2) * v(2, 2);
  M23<S> g;
  g(0, 0) = S(s[0]) * 2 * a0 * d11 + S(s[1]) * b0 * d12;
  g(0, 1) = S(s[2]) * 2 * a1 * d11 + S(s[3]) * b1 * d12;
  g(0, 2) = S(s[4]) * 2 * a2 * d11 + S(s[5]) * b2 * d12;
  g(1, 0) = S(s[6]) * 2 * b0 * d22 + S(s[7]) * a0 * d12;
  g(1, 1) = S(s[8]) * 2 * b1 * d22 + S(s[9]) * a1 * d12;
  g(1, 2) = S(s[10]) * 2 * b2 * d22 + S(s[11]) * a2 * d12;
  return g;
}

template <class S>
inline V3<S> grad_position(const V3<S>& t, const M23<S>& dl_dj, S width, S height) {  // :73-105
  const S x = t[0], y = t[1], z = t[2];
  const S rho2 = x * x + z * z;
  if (!(rho2 > S(0))) throw std::domain_error("grad_position: undefined at the pole axis");
  const S rho = std::sqrt(rho2);
  const S r2 = rho2 + y * y;
  const S r4 = r2 * r2;
  const S kw = width / (S(2) * pi_v<S>);
  const S kh = height / pi_v<S>;
  const S g11 = dl_dj(0, 0), g13 = dl_dj(0, 2);
  const S g21 = dl_dj(1, 0), g22 = dl_dj(1, 1), g23 = dl_dj(1, 2);
  const S xz_over_rho4 = x * z / (rho2 * rho2);
  const S xx_minus_zz = (x * x - z * z) / (rho2 * rho2);
  const S mixed = x * y * z * (2 * rho2 + r2) / (r4 * rho2 * rho);
  const S straight = (r2 - 2 * y * y) / (r4 * rho);
  V3<S> g;
  g[0] = -2 * kw * xz_over_rho4 * g11 + kw * xx_minus_zz * g13 -
         kh * y * (z * z * r2 - 2 * x * x * rho2) / (r4 * rho2 * rho) * g21 -
         kh * x * straight * g22 + kh * mixed * g23;
  g[1] = -kh * x * straight * g21 - 2 * kh * y * rho / r4 * g22 - kh * z * straight * g23;
  g[2] = kw * xx_minus_zz * g11 + 2 * kw * xz_over_rho4 * g13 + kh * mixed * g21 -
         kh * z * straight * g22 -
         kh * y * (x * x * r2 - 2 * z * z * rho2) / (r4 * rho2 * rho) * g23;
  return g;
}

template <class S, class M = StdMath>
inline V3<S> grad_position_clamped(const V3<S>& t, const M23<S>& dl_dj, S width, S height,
                                   S max_elevation) {  // backward.hpp:111-150
  const auto angles = to_spherical<S, M>(t);
  const S x = t[0], y = t[1], z = t[2];
  const S rho2 = x * x + z * z;
  if (!(rho2 > S(0))) throw std::domain_error("grad_position_clamped: undefined at the pole axis");
  const S rho = std::sqrt(rho2);
  const S r2 = rho2 + y * y;
  const S r = std::sqrt(r2);
  const S cp = M::cos(angles.azimuth), sp = M::sin(angles.azimuth);
  const S ct = M::cos(angles.elevation), st = M::sin(angles.elevation);
  const S sec = S(1) / M::cos(max_elevation);
  const S kw = width / (S(2) * pi_v<S>) * sec / r;
  const S kh = height / pi_v<S> / r;
  M23<S> dj_dr{{{-kw * cp / r, 0, kw * sp / r}, {-kh * st * sp / r, -kh * ct / r, -kh * st * cp / r}}};
  M23<S> dj_dphi{{{-kw * sp, 0, -kw * cp}, {kh * st * cp, 0, -kh * st * sp}}};
  M23<S> dj_dtheta{{{0, 0, 0}, {kh * ct * sp, -kh * st, kh * ct * cp}}};
  const V3<S> dr_dt{{x / r, y / r, z / r}};
  const V3<S> dphi_dt{{z / rho2, 0, -x / rho2}};
  const V3<S> dtheta_dt{{x * y / (rho * r2), -rho / r2, z * y / (rho * r2)}};
  // cwiseProduct(...).sum() over a 2x3 in column-major element order.
  auto csum = [&](const M23<S>& a) {
    return sum6(dl_dj(0, 0) * a(0, 0), dl_dj(1, 0) * a(1, 0), dl_dj(0, 1) * a(0, 1),
                dl_dj(1, 1) * a(1, 1), dl_dj(0, 2) * a(0, 2), dl_dj(1, 2) * a(1, 2));
  };
  const S cr = csum(dj_dr), cphi = csum(dj_dphi), ctheta = csum(dj_dtheta);
  V3<S> g;
  for (int k = 0; k < 3; ++k) g[k] = cr * dr_dt[k] + cphi * dphi_dt[k] + ctheta * dtheta_dt[k];
  return g;
}

template <class S, class M = StdMath>
inline std::pair<V4<S>, V3<S>> grad_cov3d_params(const M3<S>& dl_dsigma, const V4<S>& quaternion,
                                                  const V3<S>& log_scales) {  // :156-201
  const S qnorm = norm4(quaternion);
  const V4<S> q = normalize_quaternion(quaternion);
  const M3<S> rot = quaternion_matrix(q);
  const S s[3] = {M::exp(log_scales[0]), M::exp(log_scales[1]), M::exp(log_scales[2])};
  M3<S> m;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) m(i, k) = rot(i, k) * s[k];
  M3<S> dl_dm = mul(dl_dsigma, m);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) dl_dm(i, k) = S(2) * dl_dm(i, k);
  M3<S> dl_drot;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) dl_drot(i, k) = dl_dm(i, k) * s[k];
  V3<S> dl_dlog;
  for (int k = 0; k < 3; ++k)
    dl_dlog[k] = sum3(rot(0, k) * dl_dm(0, k), rot(1, k) * dl_dm(1, k), rot(2, k) * dl_dm(2, k)) * s[k];
  const S w = q[0], qx = q[1], qy = q[2], qz = q[3];
  M3<S> dw{{{0, -qz, qy}, {qz, 0, -qx}, {-qy, qx, 0}}};
  M3<S> dx{{{0, qy, qz}, {qy, -2 * qx, -w}, {qz, w, -2 * qx}}};
  M3<S> dy{{{-2 * qy, qx, w}, {qx, 0, qz}, {-w, qz, -2 * qy}}};
  M3<S> dz{{{-2 * qz, -w, qx}, {w, -2 * qz, qy}, {qx, qy, 0}}};
  // cwiseProduct(...).sum() over a 3x3 (9 terms, column-major): halving split 4 + 5.
  auto csum = [&](const M3<S>& a) {
    S e[9];
    int k = 0;
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) e[k++] = dl_drot(r, c) * a(r, c);
    const S lo = sum4(e[0], e[1], e[2], e[3]);
    const S hi = (e[4] + e[5]) + (e[6] + (e[7] + e[8]));
    return lo + hi;
  };
  V4<S> g_unit{{S(2) * csum(dw), S(2) * csum(dx), S(2) * csum(dy), S(2) * csum(dz)}};
  const S qd = sum4(q[0] * g_unit[0], q[1] * g_unit[1], q[2] * g_unit[2], q[3] * g_unit[3]);
  V4<S> g;
  for (int k = 0; k < 4; ++k) g[k] = (g_unit[k] - q[k] * qd) / qnorm;
  return {g, dl_dlog};
}

// Eigen isZero() default precision: dummy_precision<float> = 1e-5, <double> = 1e-12.
template <class S> inline S dummy_precision() { return std::is_same_v<S, float> ? S(1e-5) : S(1e-12); }

template <class S, class M = StdMath>
inline std::vector<SplatGrads<S>> grad_pixels_to_splats(const RenderOutput<S>& fwd,
                                                        const std::vector<S>& dl_dimage,
                                                        const Settings<S>& settings) {  // :208-339
  const int height = fwd.height, width = fwd.width;
  const int n_tiles = fwd.tiles_x * fwd.tiles_y;
  const S cutoff2 = settings.cutoff_sigma * settings.cutoff_sigma;
  struct EntryGrad { S mx = 0, my = 0, m00 = 0, m01 = 0, m11 = 0, op = 0, c0 = 0, c1 = 0, c2 = 0; };
  std::vector<EntryGrad> entry_grads(fwd.tile_entries.size());
  struct Contribution { int entry; S alpha, weight, dx, dy; bool clamped; };
  const std::size_t plane = (std::size_t)width * height;
  parallel_for(0, n_tiles, settings.threads, [&](int tile) {
    const int tx = tile % fwd.tiles_x, ty = tile / fwd.tiles_x;
    const int x0 = tx * settings.tile_size, y0 = ty * settings.tile_size;
    const int x1 = std::min(width, x0 + settings.tile_size);
    const int y1 = std::min(height, y0 + settings.tile_size);
    const int e0 = fwd.tile_offsets[(std::size_t)tile];
    std::vector<Contribution> contribs;
    for (int py = y0; py < y1; ++py) {
      for (int px = x0; px < x1; ++px) {
        const std::size_t p = fwd.px(py, px);
        const int walked = fwd.walked[p];
        if (walked == 0) continue;
        const S dpix[3] = {dl_dimage[p], dl_dimage[plane + p], dl_dimage[2 * plane + p]};
        const S prec = dummy_precision<S>();
        if (std::abs(dpix[0]) <= prec && std::abs(dpix[1]) <= prec && std::abs(dpix[2]) <= prec) continue;
        contribs.clear();
        S t = S(1);
        for (int e = e0; e < e0 + walked; ++e) {
          const auto& inst = fwd.instances[(std::size_t)fwd.tile_entries[(std::size_t)e]];
          const auto& splat = fwd.splats[(std::size_t)inst.splat];
          const S dx = S(px) + S(0.5) - (splat.pixel_mean[0] + inst.shift);
          const S dy = S(py) + S(0.5) - splat.pixel_mean[1];
          const S d2 = splat.cov2d_inv(0, 0) * dx * dx + S(2) * splat.cov2d_inv(0, 1) * dx * dy +
                       splat.cov2d_inv(1, 1) * dy * dy;
          if (d2 > cutoff2) continue;
          const S raw_alpha = splat.opacity * M::exp_blend(-d2 / S(2));
          const S alpha = std::min(settings.alpha_clamp, raw_alpha);
          contribs.push_back({e, alpha, M::exp_blend(-d2 / S(2)), dx, dy, raw_alpha > settings.alpha_clamp});
          t *= (S(1) - alpha);
        }
        S suffix[3] = {0, 0, 0};
        for (int k = static_cast<int>(contribs.size()) - 1; k >= 0; --k) {
          const Contribution& c = contribs[(std::size_t)k];
          const auto& inst = fwd.instances[(std::size_t)fwd.tile_entries[(std::size_t)c.entry]];
          const auto& splat = fwd.splats[(std::size_t)inst.splat];
          const S t_here = t / (S(1) - c.alpha);
          EntryGrad& eg = entry_grads[(std::size_t)c.entry];
          eg.c0 += dpix[0] * c.alpha * t_here;
          eg.c1 += dpix[1] * c.alpha * t_here;
          eg.c2 += dpix[2] * c.alpha * t_here;
          S v[3];
          for (int q = 0; q < 3; ++q) v[q] = splat.color[q] * t_here - suffix[q] / (S(1) - c.alpha);
          const S dl_dalpha = sum3(dpix[0] * v[0], dpix[1] * v[1], dpix[2] * v[2]);
          for (int q = 0; q < 3; ++q) suffix[q] += splat.color[q] * (c.alpha * t_here);
          t = t_here;
          if (c.clamped) continue;
          eg.op += dl_dalpha * c.weight;
          const S dl_dd2 = dl_dalpha * splat.opacity * (-c.weight / S(2));
          const S gx = splat.cov2d_inv(0, 0) * c.dx + splat.cov2d_inv(0, 1) * c.dy;
          const S gy = splat.cov2d_inv(0, 1) * c.dx + splat.cov2d_inv(1, 1) * c.dy;
          eg.mx += dl_dd2 * (-2) * gx;
          eg.my += dl_dd2 * (-2) * gy;
          eg.m00 += dl_dd2 * c.dx * c.dx;
          eg.m01 += dl_dd2 * c.dx * c.dy;
          eg.m11 += dl_dd2 * c.dy * c.dy;
        }
      }
    }
  });
  std::vector<SplatGrads<S>> out(fwd.splats.size());
  std::vector<std::array<S, 3>> inv_grads(fwd.splats.size(), {S(0), S(0), S(0)});
  for (std::size_t e = 0; e < fwd.tile_entries.size(); ++e) {
    const EntryGrad& eg = entry_grads[e];
    const int s = fwd.instances[(std::size_t)fwd.tile_entries[e]].splat;
    SplatGrads<S>& sg = out[(std::size_t)s];
    sg.pixel_mean[0] += eg.mx;
    sg.pixel_mean[1] += eg.my;
    sg.opacity += eg.op;
    sg.color[0] += eg.c0;
    sg.color[1] += eg.c1;
    sg.color[2] += eg.c2;
    inv_grads[(std::size_t)s][0] += eg.m00;
    inv_grads[(std::size_t)s][1] += eg.m01;
    inv_grads[(std::size_t)s][2] += eg.m11;
  }
  for (std::size_t s = 0; s < out.size(); ++s) {
    M2<S> g_inv{{{inv_grads[s][0], inv_grads[s][1]}, {inv_grads[s][1], inv_grads[s][2]}}};
    M2<S> neg_inv;
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) neg_inv(r, c) = -fwd.splats[s].cov2d_inv(r, c);
    out[s].cov2d = mul(mul(neg_inv, g_inv), fwd.splats[s].cov2d_inv);
  }
  return out;
}

template <class S> struct GradBuffers {  // backward.hpp:342-374
  int64_t n = 0;
  std::vector<S> means, rotations, log_scales, raw_opacities, colors, pixel_grad_norm, one_minus_cos;
  std::vector<S> sh_rest;  // extension: gradients of the SH coefficients (same layout as the cloud's)
  std::vector<int32_t> observed;
  void init(int64_t m, int sh_coefs = 0) {
    n = m;
    sh_rest.assign((std::size_t)sh_coefs * m, 0);
    means.assign(3 * m, 0); rotations.assign(4 * m, 0); log_scales.assign(3 * m, 0);
    raw_opacities.assign(m, 0); colors.assign(3 * m, 0);
    pixel_grad_norm.assign(m, 0); one_minus_cos.assign(m, 0); observed.assign(m, 0);
  }
  void accumulate(const GradBuffers& o) {
    auto add = [](auto& a, const auto& b) { for (std::size_t k = 0; k < a.size(); ++k) a[k] += b[k]; };
    add(means, o.means); add(rotations, o.rotations); add(log_scales, o.log_scales);
    add(raw_opacities, o.raw_opacities); add(colors, o.colors);
    add(pixel_grad_norm, o.pixel_grad_norm); add(one_minus_cos, o.one_minus_cos); add(observed, o.observed);
    add(sh_rest, o.sh_rest);
  }
};

template <class S, class M = StdMath>
inline GradBuffers<S> backward(const Cloud<S>& cloud, const Camera<S>& camera,
                               const RenderOutput<S>& fwd, const std::vector<S>& dl_dimage,
                               const Settings<S>& settings, const GradTSigns* signs = nullptr,
                               std::vector<SplatGrads<S>>* splat_grads_out = nullptr) {  // :380-448
  const auto splat_grads = grad_pixels_to_splats<S, M>(fwd, dl_dimage, settings);
  if (splat_grads_out) *splat_grads_out = splat_grads;
  GradBuffers<S> out;
  out.init(cloud.n, cloud.sh_degree > 0 ? 3 * sh_count(cloud.sh_degree) : 0);
  const S width = S(camera.width), height = S(camera.height);
  const int64_t n = cloud.n;
  parallel_for(0, static_cast<int>(fwd.splats.size()), settings.threads, [&](int si) {
    const Splat2D<S>& splat = fwd.splats[(std::size_t)si];
    const SplatGrads<S>& sg = splat_grads[(std::size_t)si];
    const int64_t i = splat.index;
    out.observed[i] = 1;
    const V3<S> mu = camera.to_camera(cloud.mean_v(i));
    const auto angles = to_spherical<S, M>(mu);
    out.one_minus_cos[i] = S(1) - M::cos(angles.elevation);
    bool clamped = false;
    const M23<S> j = jacobian_omni<S, M>(mu, width, height, settings.max_elevation, &clamped);
    const M3<S> sigma_world = build_covariance<S, M>(cloud.rot_v(i), cloud.ls_v(i));
    const M23<S> t = mul(j, camera.rotation);
    const M23<S> dl_dt = grad_T(t, sigma_world, sg.cov2d, signs);
    const M23<S> dl_dj = mul(dl_dt, transpose(camera.rotation));
    V3<S> dl_dmu = clamped ? grad_position_clamped<S, M>(mu, dl_dj, width, height, settings.max_elevation)
                           : grad_position(mu, dl_dj, width, height);
    const M23<S> jd = jacobian_omni_direct(mu, width, height);
    for (int k = 0; k < 3; ++k) dl_dmu[k] += sum2(jd(0, k) * sg.pixel_mean[0], jd(1, k) * sg.pixel_mean[1]);
    const M3<S> rt = transpose(camera.rotation);
    V3<S> gm = mulv(rt, dl_dmu);
    if (cloud.sh_degree > 0) {  // SH extension: coefficients and the view-direction term
      S d[3], Y[15], dY[15][3];
      const S len = sh_direction(camera, cloud.mean_v(i), d);
      sh_basis(cloud.sh_degree, d[0], d[1], d[2], Y);
      sh_basis_grad(cloud.sh_degree, d[0], d[1], d[2], dY);
      const int nb = sh_count(cloud.sh_degree);
      S dd[3] = {0, 0, 0};
      for (int k = 0; k < nb; ++k)
        for (int ch = 0; ch < 3; ++ch) {
          out.sh_rest[(std::size_t)(3 * k + ch) * n + i] = sg.color[ch] * Y[k];
          const S w = sg.color[ch] * cloud.sh_rest[(std::size_t)(3 * k + ch) * n + i];
          for (int a = 0; a < 3; ++a) dd[a] += w * dY[k][a];
        }
      if (len > S(0)) {
        const S dot = sum3(d[0] * dd[0], d[1] * dd[1], d[2] * dd[2]);
        for (int a = 0; a < 3; ++a) gm[a] += (dd[a] - d[a] * dot) / len;
      }
    }
    for (int k = 0; k < 3; ++k) out.means[k * n + i] = gm[k];
    out.pixel_grad_norm[i] = std::sqrt(sum2(sg.pixel_mean[0] * sg.pixel_mean[0], sg.pixel_mean[1] * sg.pixel_mean[1]));
    const M3<S> dl_dsigma = mul(mul(transpose(t), sg.cov2d), t);
    const auto [dq, dls] = grad_cov3d_params<S, M>(dl_dsigma, cloud.rot_v(i), cloud.ls_v(i));
    for (int k = 0; k < 4; ++k) out.rotations[k * n + i] = dq[k];
    for (int k = 0; k < 3; ++k) out.log_scales[k * n + i] = dls[k];
    const S o = splat.opacity;
    out.raw_opacities[i] = sg.opacity * o * (S(1) - o);
    for (int k = 0; k < 3; ++k) out.colors[k * n + i] = sg.color[k];
  });
  for (int64_t i = 0; i < n; ++i) {
    bool ok = true;
    for (int k = 0; k < 3; ++k) ok = ok && finite(out.means[k * n + i]);
    for (int k = 0; k < 4; ++k) ok = ok && finite(out.rotations[k * n + i]);
    for (int k = 0; k < 3; ++k) ok = ok && finite(out.log_scales[k * n + i]);
    ok = ok && finite(out.raw_opacities[i]);
    for (int k = 0; k < 3; ++k) ok = ok && finite(out.colors[k * n + i]);
    for (std::size_t k = 0; k < out.sh_rest.size() / (std::size_t)std::max<int64_t>(n, 1); ++k)
      ok = ok && finite(out.sh_rest[k * n + i]);
    if (!ok) throw std::runtime_error("backward: non-finite gradient for Gaussian " + std::to_string(i));
  }
  return out;
}

// ------------------------------------------------------------------ metrics.hpp:27-184 (§8f #1)
// Column-major 2D array (Eigen::ArrayXX storage).
template <class S> struct Arr {
  int rows = 0, cols = 0;
  std::vector<S> d;
  Arr() = default;
  Arr(int r, int c, S v = S(0)) : rows(r), cols(c), d((std::size_t)r * c, v) {}
  S& operator()(int r, int c) { return d[(std::size_t)c * rows + r]; }
  S operator()(int r, int c) const { return d[(std::size_t)c * rows + r]; }
};

template <class S> inline std::vector<S> ssim_window() {  // metrics.hpp:31-39
  std::vector<S> w(11);
  for (int i = 0; i < 11; ++i) {
    const S dd = S(i) - S(5);
    w[i] = std::exp(-dd * dd / (S(2) * S(1.5) * S(1.5)));
  }
  S sum = 0;  // VecX::sum() of 11: halving unroll is not guaranteed for dynamic size;
  for (int i = 0; i < 11; ++i) sum += w[i];  // the restatement fixes a sequential sum.
  for (auto& v : w) v /= sum;
  return w;
}

template <class S> inline Arr<S> window_valid(const Arr<S>& in, const std::vector<S>& w) {  // :43-57
  const int h = in.rows, wd = in.cols, k = (int)w.size();
  Arr<S> horiz(h, wd - k + 1);
  for (int i = 0; i < k; ++i)
    for (int c = 0; c < wd - k + 1; ++c)
      for (int r = 0; r < h; ++r) horiz(r, c) += w[i] * in(r, c + i);
  Arr<S> out(h - k + 1, wd - k + 1);
  for (int i = 0; i < k; ++i)
    for (int c = 0; c < wd - k + 1; ++c)
      for (int r = 0; r < h - k + 1; ++r) out(r, c) += w[i] * horiz(r + i, c);
  return out;
}

template <class S> inline Arr<S> window_scatter(const Arr<S>& in, const std::vector<S>& w) {  // :62-71
  const int k = (int)w.size();
  Arr<S> padded(in.rows + 2 * (k - 1), in.cols + 2 * (k - 1));
  for (int c = 0; c < in.cols; ++c)
    for (int r = 0; r < in.rows; ++r) padded(r + k - 1, c + k - 1) = in(r, c);
  return window_valid(padded, w);
}

// Images here: 3 planes of H x W column-major, concatenated (the RenderOutput layout).
template <class S>
inline S ssim_with_gradient(const std::vector<S>& a, const std::vector<S>& b, int H, int W,
                            std::vector<S>* grad) {  // metrics.hpp:83-136
  if (H < 11 || W < 11) throw std::invalid_argument("ssim: images smaller than the 11x11 window");
  const auto w = ssim_window<S>();
  const S c1 = S(0.01) * S(0.01), c2 = S(0.03) * S(0.03);
  const S windows = S(3) * S(H - 10) * S(W - 10);
  S score_sum = 0;
  if (grad) grad->assign((std::size_t)3 * H * W, S(0));
  const std::size_t plane = (std::size_t)H * W;
  for (int c = 0; c < 3; ++c) {
    Arr<S> ca(H, W), cb(H, W), aa(H, W), bb(H, W), ab(H, W);
    for (std::size_t p = 0; p < plane; ++p) {
      ca.d[p] = a[c * plane + p];
      cb.d[p] = b[c * plane + p];
      aa.d[p] = ca.d[p] * ca.d[p];
      bb.d[p] = cb.d[p] * cb.d[p];
      ab.d[p] = ca.d[p] * cb.d[p];
    }
    const Arr<S> mu_a = window_valid(ca, w), mu_b = window_valid(cb, w);
    const Arr<S> wa = window_valid(aa, w), wb = window_valid(bb, w), wab = window_valid(ab, w);
    const int h = mu_a.rows, wd = mu_a.cols;
    Arr<S> d_mu_a(h, wd), d_var_a(h, wd), d_cov(h, wd), mix(h, wd);
    for (std::size_t p = 0; p < mu_a.d.size(); ++p) {
      const S ma = mu_a.d[p], mb = mu_b.d[p];
      const S var_a = wa.d[p] - ma * ma, var_b = wb.d[p] - mb * mb, cov = wab.d[p] - ma * mb;
      const S n1 = 2 * ma * mb + c1, n2 = 2 * cov + c2;
      const S d1 = ma * ma + mb * mb + c1, d2 = var_a + var_b + c2;
      const S s = (n1 * n2) / (d1 * d2);
      score_sum += s;
      d_mu_a.d[p] = (2 * mb * n2 - 2 * ma * s * d2) / (d1 * d2) / windows;
      d_var_a.d[p] = (-s / d2) / windows;
      d_cov.d[p] = (2 * (n1 / d1) / d2) / windows;
      mix.d[p] = 2 * d_var_a.d[p] * ma + d_cov.d[p] * mb;
    }
    if (grad) {
      const Arr<S> s_mu = window_scatter(d_mu_a, w), s_var = window_scatter(d_var_a, w);
      const Arr<S> s_cov = window_scatter(d_cov, w), s_mix = window_scatter(mix, w);
      for (std::size_t p = 0; p < plane; ++p)
        (*grad)[c * plane + p] = s_mu.d[p] + (2 * ca.d[p] * s_var.d[p] + cb.d[p] * s_cov.d[p]) - s_mix.d[p];
    }
  }
  return score_sum / windows;
}

template <class S>
inline S photometric_loss(const std::vector<S>& rendered, const std::vector<S>& target, int H, int W,
                          S lambda_ssim, std::vector<S>* gradient) {  // metrics.hpp:152-184
  if (rendered.size() != target.size()) throw std::invalid_argument("photometric_loss: image dimensions differ");
  if (!(lambda_ssim >= S(0)) || !(lambda_ssim < S(1)))
    throw std::invalid_argument("photometric_loss: lambda must be in [0, 1)");
  const S pixels = S(3) * S(H) * S(W);
  const std::size_t plane = (std::size_t)H * W;
  S loss = 0;
  gradient->assign(rendered.size(), S(0));
  for (int c = 0; c < 3; ++c) {
    S abs_sum = 0;  // ArrayXX::sum(): the restatement fixes a sequential column-major sum
    for (std::size_t p = 0; p < plane; ++p) {
      const S diff = rendered[c * plane + p] - target[c * plane + p];
      abs_sum += std::abs(diff);
      const S sign = diff > S(0) ? S(1) : (diff < S(0) ? S(-1) : S(0));
      (*gradient)[c * plane + p] = (S(1) - lambda_ssim) * sign / pixels;
    }
    loss += (S(1) - lambda_ssim) * abs_sum / pixels;
  }
  if (lambda_ssim > S(0)) {
    std::vector<S> sg;
    const S s = ssim_with_gradient(rendered, target, H, W, &sg);
    loss += lambda_ssim * (S(1) - s);
    for (std::size_t p = 0; p < gradient->size(); ++p) (*gradient)[p] -= lambda_ssim * sg[p];
  }
  return loss;
}

// ------------------------------------------------------------------ densify.hpp
// TrainState (types.hpp:257-325): Adam moments per group and the densify window, SoA
// with the same layouts as Cloud (member(i, c) at c*n + i).
template <class S> struct TrainState {
  int64_t n = 0;
  std::vector<S> means_m, means_v, rot_m, rot_v, scale_m, scale_v, opac_m, opac_v, color_m, color_v;
  std::vector<S> grad_accum, elev_accum;
  std::vector<int32_t> grad_count;
  void init(int64_t m) {  // types.hpp:270-281
    n = m;
    for (auto* v : {&means_m, &means_v, &scale_m, &scale_v, &color_m, &color_v}) v->assign(3 * m, S(0));
    rot_m.assign(4 * m, S(0));
    rot_v.assign(4 * m, S(0));
    opac_m.assign(m, S(0));
    opac_v.assign(m, S(0));
    reset_densify_stats(m);
  }
  void reset_densify_stats(int64_t m) {  // types.hpp:283-287
    grad_accum.assign(m, S(0));
    elev_accum.assign(m, S(0));
    grad_count.assign(m, 0);
  }
};

struct DensifyConfig {  // densify.hpp:16-33
  double grad_threshold_min = 2e-5;
  double grad_threshold_max = 1e-4;
  double percent_dense = 1e-3;
  double opacity_prune_floor = 0.005;
  double split_scale_divisor = 1.6;
  void validate() const {
    if (!(grad_threshold_min > 0) || !(grad_threshold_max >= grad_threshold_min))
      throw std::invalid_argument("DensifyConfig: need 0 < grad_threshold_min <= grad_threshold_max");
    if (!(percent_dense > 0) || !(percent_dense < 1))
      throw std::invalid_argument("DensifyConfig: percent_dense outside (0, 1)");
  }
};

struct DensifyStats { int64_t cloned = 0, split = 0, pruned = 0; };

// densify.hpp:61-69. `Vec3<Scalar> e(Scalar(gauss(rng)), Scalar(gauss(rng)),
// Scalar(gauss(rng)))` is a parenthesised call; GCC evaluates its arguments right to
// left, so the first draw lands in z (checked with the image's g++). The
// normal_distribution object lives across the rejection loop and dies with the call,
// so a cached second polar value is carried between tries but never between calls.
template <class S> V3<S> unit_ball_normal(std::mt19937& rng) {
  std::normal_distribution<double> gauss;
  for (;;) {
    V3<S> e;
    e[2] = S(gauss(rng));
    e[1] = S(gauss(rng));
    e[0] = S(gauss(rng));
    if (norm3(e) <= S(1)) return e;
  }
}

namespace detail {
// One row of the cloud as the reference's append_row copies it (types.hpp:92-106),
// plus the SH rest coefficients of this build's extension.
template <class S> struct Row {
  S mean[3], rot[4], ls[3], opac, col[3];
  std::vector<S> sh;
};
template <class S> Row<S> get_row(const Cloud<S>& c, int64_t i) {
  Row<S> r;
  for (int k = 0; k < 3; ++k) { r.mean[k] = c.mean(i, k); r.ls[k] = c.ls(i, k); r.col[k] = c.col(i, k); }
  for (int k = 0; k < 4; ++k) r.rot[k] = c.rot(i, k);
  r.opac = c.raw_opacities[i];
  if (c.sh_degree > 0)
    for (int k = 0; k < 3 * sh_count(c.sh_degree); ++k) r.sh.push_back(c.sh_rest[k * c.n + i]);
  return r;
}
template <class S> Cloud<S> from_rows(const std::vector<Row<S>>& rows, int sh_degree) {
  Cloud<S> c;
  c.resize((int64_t)rows.size());
  c.sh_degree = sh_degree;
  const int64_t n = c.n;
  if (sh_degree > 0) c.sh_rest.assign(3 * sh_count(sh_degree) * n, S(0));
  for (int64_t i = 0; i < n; ++i) {
    const Row<S>& r = rows[(std::size_t)i];
    for (int k = 0; k < 3; ++k) { c.mean(i, k) = r.mean[k]; c.ls(i, k) = r.ls[k]; c.col(i, k) = r.col[k]; }
    for (int k = 0; k < 4; ++k) c.rot(i, k) = r.rot[k];
    c.raw_opacities[i] = r.opac;
    for (std::size_t k = 0; k < r.sh.size(); ++k) c.sh_rest[k * n + i] = r.sh[k];
  }
  return c;
}
}  // namespace detail

// densify.hpp:81-153. Clones and split children are appended in parent order (one
// row per clone, two per split), then split parents and Gaussians under the opacity
// floor are dropped; moments follow the rows (new rows zero), the window is cleared.
template <class S, class M = StdMath>
DensifyStats densify_and_prune(Cloud<S>& cloud, TrainState<S>& state, const DensifyConfig& cfg, S scene_extent,
                               std::mt19937& rng) {
  cfg.validate();
  if (!(scene_extent > S(0))) throw std::invalid_argument("densify_and_prune: scene extent must be positive");
  const int64_t n = cloud.n;
  DensifyStats stats;
  const S tmin = S(cfg.grad_threshold_min), tmax = S(cfg.grad_threshold_max);
  const S size_split = S(cfg.percent_dense) * scene_extent;
  std::vector<bool> remove((std::size_t)n, false);
  std::vector<detail::Row<S>> added;
  for (int64_t i = 0; i < n; ++i) {
    if (state.grad_count[i] <= 0) continue;
    const S count = S(state.grad_count[i]);
    const S mean_grad = state.grad_accum[i] / count;
    const S mean_omc = state.elev_accum[i] / count;
    const S threshold = tmin + mean_omc * (tmax - tmin);
    if (mean_grad < threshold) continue;
    const V3<S> s{{M::exp(cloud.ls(i, 0)), M::exp(cloud.ls(i, 1)), M::exp(cloud.ls(i, 2))}};
    const S max_scale = std::max(s[0], std::max(s[1], s[2]));
    if (max_scale < size_split) {
      added.push_back(detail::get_row(cloud, i));
      ++stats.cloned;
    } else {
      const M3<S> rot = rotation_from_quaternion(cloud.rot_v(i));
      for (int child = 0; child < 2; ++child) {
        detail::Row<S> row = detail::get_row(cloud, i);
        const V3<S> e = unit_ball_normal<S>(rng);
        const V3<S> offset = mulv(rot, V3<S>{{s[0] * e[0], s[1] * e[1], s[2] * e[2]}});
        const S shrink = M::log(S(cfg.split_scale_divisor));
        for (int k = 0; k < 3; ++k) {
          row.mean[k] += offset[k];
          row.ls[k] -= shrink;
        }
        added.push_back(std::move(row));
      }
      remove[(std::size_t)i] = true;
      ++stats.split;
    }
  }
  std::vector<detail::Row<S>> rows;
  std::vector<int64_t> src;  // state row of each output row, -1 = fresh zeros
  const int64_t total = n + (int64_t)added.size();
  for (int64_t i = 0; i < total; ++i) {
    if (i < n && remove[(std::size_t)i]) continue;
    const S raw = i < n ? cloud.raw_opacities[i] : added[(std::size_t)(i - n)].opac;
    if (sigmoid<S, M>(raw) < S(cfg.opacity_prune_floor)) {
      ++stats.pruned;
      continue;
    }
    rows.push_back(i < n ? detail::get_row(cloud, i) : added[(std::size_t)(i - n)]);
    src.push_back(i < n ? i : -1);
  }
  const int sh_degree = cloud.sh_degree;
  cloud = detail::from_rows(rows, sh_degree);
  TrainState<S> out;
  out.init(cloud.n);
  const int64_t m = cloud.n;
  auto move_rows = [&](const std::vector<S>& from, std::vector<S>& to, int width) {
    for (int64_t k = 0; k < m; ++k)
      if (src[(std::size_t)k] >= 0)
        for (int c = 0; c < width; ++c) to[c * m + k] = from[c * n + src[(std::size_t)k]];
  };
  move_rows(state.means_m, out.means_m, 3); move_rows(state.means_v, out.means_v, 3);
  move_rows(state.rot_m, out.rot_m, 4);     move_rows(state.rot_v, out.rot_v, 4);
  move_rows(state.scale_m, out.scale_m, 3); move_rows(state.scale_v, out.scale_v, 3);
  move_rows(state.opac_m, out.opac_m, 1);   move_rows(state.opac_v, out.opac_v, 1);
  move_rows(state.color_m, out.color_m, 3); move_rows(state.color_v, out.color_v, 3);
  state = std::move(out);  // window cleared (init), densify.hpp:151
  return stats;
}

// densify.hpp:158-166.
template <class S, class M = StdMath>
void reset_opacity(Cloud<S>& cloud, TrainState<S>& state, S ceiling = S(0.01)) {
  for (int64_t i = 0; i < cloud.n; ++i)
    cloud.raw_opacities[i] = logit<S, M>(std::min(sigmoid<S, M>(cloud.raw_opacities[i]), ceiling));
  std::fill(state.opac_m.begin(), state.opac_m.end(), S(0));
  std::fill(state.opac_v.begin(), state.opac_v.end(), S(0));
}

// densify.hpp:39-49.
template <class S> inline S dynamic_threshold(S elevation, const DensifyConfig& cfg) {
  if (!(std::abs(elevation) <= pi_v<S> / 2 + S(1e-12)))
    throw std::domain_error("dynamic_threshold: elevation outside [-pi/2, pi/2]");
  const S tmin = S(cfg.grad_threshold_min), tmax = S(cfg.grad_threshold_max);
  return std::fma(S(1) - std::cos(elevation), tmax - tmin, tmin);
}

// ------------------------------------------------------------------ scenes (tests/scenes.hpp:11-73)
struct CloudBounds {
  double depth_min = 0.5, depth_max = 20.0;
  double max_elevation = 1.45;
  double opacity_min = 0.05, opacity_max = 0.95;
  double scale_min = 0.005, scale_max = 0.05;
};

template <class S> Cloud<S> random_cloud(std::mt19937& rng, int n, const CloudBounds& b = {}) {
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  std::normal_distribution<double> gauss;
  Cloud<S> cloud;
  cloud.resize(n);
  for (int i = 0; i < n; ++i) {
    const double phi = (2 * u01(rng) - 1) * pi_v<double>;
    const double theta = (2 * u01(rng) - 1) * b.max_elevation;
    const double r = b.depth_min + u01(rng) * (b.depth_max - b.depth_min);
    cloud.mean(i, 0) = S(r * std::cos(theta) * std::sin(phi));
    cloud.mean(i, 1) = S(-r * std::sin(theta));
    cloud.mean(i, 2) = S(r * std::cos(theta) * std::cos(phi));
    double q[4];
    auto qn = [&] { return std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]); };
    // The reference's Vec4 q(gauss(rng), gauss(rng), gauss(rng), gauss(rng)) is a
    // parenthesised call whose argument order is unspecified; GCC (the image's
    // compiler) evaluates it right to left, so the first draw lands in q[3]. The
    // rejection re-draw `q = {...}` is a braced list: left to right.
    for (int c = 3; c >= 0; --c) q[c] = gauss(rng);
    while (qn() < 1e-3)
      for (int c = 0; c < 4; ++c) q[c] = gauss(rng);
    const double nq = qn();
    for (int c = 0; c < 4; ++c) cloud.rot(i, c) = S(q[c] / nq);
    for (int a = 0; a < 3; ++a) {
      const double s = r * (b.scale_min + u01(rng) * (b.scale_max - b.scale_min));
      cloud.ls(i, a) = S(std::log(s));
    }
    const double alpha = b.opacity_min + u01(rng) * (b.opacity_max - b.opacity_min);
    cloud.raw_opacities[i] = logit(S(alpha));
    for (int c = 0; c < 3; ++c) cloud.col(i, c) = S(0.05 + 0.9 * u01(rng));
  }
  return cloud;
}

template <class S> Camera<S> identity_camera(int width, int height) {
  Camera<S> c;
  c.width = width;
  c.height = height;
  return c;
}

template <class S> Camera<S> yawed_camera(const Camera<S>& base, S angle) {  // scenes.hpp:62-73
  M3<S> yaw{{{std::cos(angle), 0, std::sin(angle)}, {0, 1, 0}, {-std::sin(angle), 0, std::cos(angle)}}};
  Camera<S> out = base;
  out.rotation = mul(yaw, base.rotation);
  out.translation = mulv(yaw, base.translation);
  return out;
}

// init_from_points' neighbour scale (io.cpp:268-296): brute-force O(n^2) scan keeping
// the three smallest squared distances (strict <, replace the largest, re-sort),
// then the ascending sum of their square roots, mean, 1e-7 floor or 0.1 fallback.
// d2 = (p_j - p_i).squaredNorm() with Eigen's unroller order x^2 + (y^2 + z^2)
// (Appendix B of SURVEY.md). pos is [3][n] column-major; writes scale[i] and the
// log-scale ls[i] = std::log(scale[i]).
inline void init_scales_brute(int64_t n, const double* pos, double* scale, double* ls) {
  for (int64_t i = 0; i < n; ++i) {
    double best[3] = {std::numeric_limits<double>::infinity(), std::numeric_limits<double>::infinity(),
                      std::numeric_limits<double>::infinity()};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = pos[j] - pos[i], dy = pos[n + j] - pos[n + i], dz = pos[2 * n + j] - pos[2 * n + i];
      const double d2 = dx * dx + (dy * dy + dz * dz);
      if (d2 < best[2]) {
        best[2] = d2;
        std::sort(best, best + 3);
      }
    }
    double sum = 0;
    int count = 0;
    for (const double d2 : best)
      if (std::isfinite(d2)) {
        sum += std::sqrt(d2);
        ++count;
      }
    scale[i] = count > 0 ? std::max(sum / count, 1e-7) : 0.1;
    ls[i] = std::log(scale[i]);
  }
}

}  // namespace oracle
