// raster_fwd.cu — forward hot path of the B200 ODGS rasterizer.
//
//   k_preprocess  one thread per Gaussian: shell cull, ERP centre, tangent-plane
//                 Jacobian, Sigma -> Sigma_2D, inverse, radius, opacity, seam-instance
//                 tile counts, depth sort key           (projection.hpp:178-216,
//                                                         rasterizer.hpp:133-156)
//   k_emit        one warp per 32 depth-ranked splats: writes (tile, gaussian|shift)
//                 entries in global (depth, index, shift) order, load-balanced over the
//                 warp                                   (rasterizer.hpp:158-205)
//   k_tile_ranges CSR tile offsets from the tile-sorted entries, empty tiles included
//   k_blend       one CTA per tile: front-to-back compositing with batches of splats
//                 staged in shared memory and CTA-wide early exit (rasterizer.hpp:211-267)
//
// Compiled with --fmad=false: see common.cuh for the numerics contract.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace odgs_b200 {

// ------------------------------------------------------------------ preprocess
// Projects Gaussian i; returns the number of seam instances (0 if culled) and sets
// *visible. Error words get the lowest offending index. kProjectOnly: the semantics of
// project_gaussian alone (projection.hpp:178-216) — no first_non_finite pass; a
// non-finite quaternion or log-scale of a Gaussian inside the shell is build_covariance's
// invalid_argument (covariance.hpp:31-32), other non-finite values pass through.
// The row's parameters as values (v: mean 3, quaternion 4, log-scales 3, raw opacity,
// colour 3): preprocess_one after its loads, for callers that already hold them.
template <bool kProjectOnly = false>
__device__ __forceinline__ uint32_t preprocess_vals(
    int64_t i, int64_t n, const float v[14], int sh_degree, const float* __restrict__ sh_rest, const DevCamera& cam,
    const DevSettings& s, float4* __restrict__ sp_ab, float4* __restrict__ sp_c, float4* __restrict__ cov_out,
    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err,
    bool* visible);

template <bool kProjectOnly = false>
__device__ __forceinline__ uint32_t preprocess_one(
    int64_t i, int64_t n, const float* __restrict__ means, const float* __restrict__ rotations,
    const float* __restrict__ log_scales, const float* __restrict__ raw_opacities,
    const float* __restrict__ colors, int sh_degree, const float* __restrict__ sh_rest, const DevCamera& cam,
    const DevSettings& s, float4* __restrict__ sp_ab, float4* __restrict__ sp_c, float4* __restrict__ cov_out,
    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err,
    bool* visible) {
  const float v[14] = {__ldg(means + i),          __ldg(means + n + i),          __ldg(means + 2 * n + i),
                       __ldg(rotations + i),      __ldg(rotations + n + i),      __ldg(rotations + 2 * n + i),
                       __ldg(rotations + 3 * n + i), __ldg(log_scales + i),      __ldg(log_scales + n + i),
                       __ldg(log_scales + 2 * n + i), __ldg(raw_opacities + i),  __ldg(colors + i),
                       __ldg(colors + n + i),     __ldg(colors + 2 * n + i)};
  return preprocess_vals<kProjectOnly>(i, n, v, sh_degree, sh_rest, cam, s, sp_ab, sp_c, cov_out, keys, vals, cnt,
                                       err, visible);
}

template <bool kProjectOnly>
__device__ __forceinline__ uint32_t preprocess_vals(
    int64_t i, int64_t n, const float v[14], int sh_degree, const float* __restrict__ sh_rest, const DevCamera& cam,
    const DevSettings& s, float4* __restrict__ sp_ab, float4* __restrict__ sp_c, float4* __restrict__ cov_out,
    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err,
    bool* visible) {
  *visible = false;
  const float p[3] = {v[0], v[1], v[2]};
  const float q[4] = {v[3], v[4], v[5], v[6]};
  const float ls[3] = {v[7], v[8], v[9]};
  const float raw = v[10];
  float col[3] = {v[11], v[12], v[13]};
  const int nb = sh_degree > 0 ? sh_count(sh_degree) : 0;

  keys[i] = kCulledKey;
  vals[i] = (uint32_t)i;
  cnt[i] = 0;
  sp_c[i] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(0u));

  if (!kProjectOnly) {
    bool finite = isfinite(raw);
    for (int c = 0; c < 3; ++c) finite = finite && isfinite(p[c]) && isfinite(ls[c]) && isfinite(col[c]);
    for (int c = 0; c < 4; ++c) finite = finite && isfinite(q[c]);
    for (int k = 0; k < 3 * nb; ++k) finite = finite && isfinite(__ldg(sh_rest + (int64_t)k * n + i));
    if (!finite) {
      atomic_min_error(&err->nonfinite, i, 2);
      return 0;
    }
  }

  float mu[3];
  to_camera(cam, p, mu);
  const float sq = sum3(mu[0] * mu[0], mu[1] * mu[1], mu[2] * mu[2]);
  const float depth = sqrtf(sq);
  if (!(depth >= s.near_radius && depth <= s.far_radius)) return 0;  // shell cull
  if (!(sq > 0.0f)) {
    atomic_min_error(&err->project, i, 3);  // to_spherical domain_error
    return 0;
  }
  const float phi = pm_atan2f(mu[0], mu[2]);
  const float rho = pm_hypotf(mu[0], mu[2]);
  const float theta = pm_atan2f(-mu[1], rho);
  const float W = (float)cam.width, H = (float)cam.height;
  const float mx = W / (2.0f * kPiF) * phi + W / 2.0f;
  const float my = -H / kPiF * theta + H / 2.0f;
  bool clamped;
  const M23 J = jacobian_factored(phi, theta, depth, W, H, s.max_elevation, &clamped);

  // build_covariance (covariance.hpp:28-37)
  if (kProjectOnly) {
    bool finite = true;
    for (int c = 0; c < 3; ++c) finite = finite && isfinite(ls[c]);
    for (int c = 0; c < 4; ++c) finite = finite && isfinite(q[c]);
    if (!finite) {
      atomic_min_error(&err->project, i, 2);  // build_covariance: non-finite parameters
      return 0;
    }
  }
  const float qn = sqrtf(sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
  if (!(qn > 1e-12f)) {
    atomic_min_error(&err->project, i, 1);  // normalize_quaternion invalid_argument
    return 0;
  }
  const M3 Rq = quaternion_matrix(q[0] / qn, q[1] / qn, q[2] / qn, q[3] / qn);
  const float sc[3] = {pm_expf(ls[0]), pm_expf(ls[1]), pm_expf(ls[2])};
  M3 m;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) m.a[r][k] = Rq.a[r][k] * sc[k];
  const M3 sigma = mul33_t(m);

  // project_covariance (projection.hpp:146-158)
  M3 Rc;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) Rc.a[r][k] = cam.R[r][k];
  const M23 t = mul23_3(J, Rc);
  const M23 tmp = mul23_3(t, sigma);
  M2 cov = mul23_32t(tmp, t);
  const float off = (cov.a[0][1] + cov.a[1][0]) / 2.0f;
  const float c00 = cov.a[0][0] + s.lowpass_dilation;
  const float c11 = cov.a[1][1] + s.lowpass_dilation;
  const float det = c00 * c11 - off * off;
  const bool cov_finite = isfinite(c00) && isfinite(off) && isfinite(c11);
  if (!(det > 0.0f) || !cov_finite) return 0;  // dropped, not an error (projection.hpp:199-200)
  const float i00 = c11 / det;
  const float i01 = -off / det;
  const float i11 = c00 / det;
  const float mid = (c00 + c11) / 2.0f;
  const float lambda_max = mid + sqrtf(std_max(0.0f, mid * mid - det));
  const float radius = s.cutoff_sigma * sqrtf(lambda_max);
  const float opacity = 1.0f / (1.0f + pm_expf(-raw));
  if (nb > 0) {  // SH extension (oracle::sh_color): c = rgb + sum_k Y_k(d) coef_k, in k order
    float d[3], Y[15];
    sh_direction(cam, p, d);
    sh_basis(sh_degree, d[0], d[1], d[2], Y);
    for (int ch = 0; ch < 3; ++ch)
      for (int k = 0; k < nb; ++k) col[ch] = col[ch] + Y[k] * __ldg(sh_rest + (int64_t)(3 * k + ch) * n + i);
  }

  // Seam instances (rasterizer.hpp:146-156) and their tile counts (:187-193).
  uint32_t flags = kFlagVisible | (clamped ? kFlagClamped : 0u);
  uint32_t total = 0, n_inst = 0;
  for (int k = 0; k < 3; ++k) {
    int span[4];
    if (instance_tiles(mx, my, radius, k, cam.width, cam.height, s.tile_size, span)) {
      flags |= kFlagShiftBase << k;
      ++n_inst;
      span[2] = max(span[2], s.band_ty0);
      span[3] = min(span[3], s.band_ty1 - 1);
      if (span[2] <= span[3]) total += (uint32_t)(span[1] - span[0] + 1) * (uint32_t)(span[3] - span[2] + 1);
    }
  }
  sp_ab[2 * i] = make_float4(mx, my, i00, i01);
  sp_ab[2 * i + 1] = make_float4(i11, opacity, col[0], col[1]);
  sp_c[i] = make_float4(col[2], depth, radius, __uint_as_float(flags));
  if (cov_out) cov_out[i] = make_float4(c00, off, off, c11);
  keys[i] = __float_as_uint(depth);  // positive floats order like their bit patterns
  cnt[i] = total;
  *visible = true;
  return n_inst;
}

__global__ void __launch_bounds__(256) k_preprocess(
    int64_t n, const float* __restrict__ means, const float* __restrict__ rotations,
    const float* __restrict__ log_scales, const float* __restrict__ raw_opacities,
    const float* __restrict__ colors, DevCamera cam, DevSettings s, float4* __restrict__ sp_ab,
    float4* __restrict__ sp_c, float4* __restrict__ cov_out, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err, int sh_degree,
    const float* __restrict__ sh_rest) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool visible = false;
  uint32_t n_inst = 0;
  if (t < n) {
    n_inst = preprocess_one(t, n, means, rotations, log_scales, raw_opacities, colors, sh_degree, sh_rest, cam, s,
                            sp_ab, sp_c, cov_out, keys, vals, cnt, err, &visible);
  }
  const uint32_t v_sum = __reduce_add_sync(0xffffffffu, visible ? 1u : 0u);
  const uint32_t i_sum = __reduce_add_sync(0xffffffffu, n_inst);
  if ((threadIdx.x & 31) == 0 && (v_sum | i_sum)) {
    atomicAdd(&err->n_visible, (unsigned long long)v_sum);
    atomicAdd(&err->n_instances, (unsigned long long)i_sum);
  }
}

void launch_preprocess(const PreprocessArgs& a, cudaStream_t stream) {
  if (a.n == 0) return;
  const int block = 256;
  const int64_t grid = (a.n + block - 1) / block;
  launch_pdl(k_preprocess, (unsigned)grid, block, 0, stream, a.n, a.means, a.rotations, a.log_scales, a.raw_opacities,
                                                     a.colors, a.cam, a.settings, a.sp_ab, a.sp_c, a.cov_out, a.keys,
                                                     a.vals, a.cnt, a.err, a.sh_degree, a.sh_rest);
  ++g_launches;
}

// ------------------------------------------------------------------ project_gaussian
// One Gaussian with project_gaussian's own semantics (odgs_project_gaussian): the row
// was gathered into a one-row cloud.
__global__ void k_project_one(const float* __restrict__ row, int sh_degree, DevCamera cam, DevSettings s,
                              float4* __restrict__ sp_ab, float4* __restrict__ sp_c, float4* __restrict__ cov,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt,
                              DevErrors* __restrict__ err) {
  pdl_wait();
  bool visible = false;
  preprocess_one<true>(0, 1, row, row + 3, row + 7, row + 10, row + 11, sh_degree, sh_degree > 0 ? row + 14 : nullptr,
                       cam, s, sp_ab, sp_c, cov, keys, vals, cnt, err, &visible);
}

void launch_project_one(const float* row, int sh_degree, const DevCamera& cam, const DevSettings& s, float4* sp_ab,
                        float4* sp_c, float4* cov, uint32_t* keys, uint32_t* vals, uint32_t* cnt, DevErrors* err,
                        cudaStream_t stream) {
  launch_pdl(k_project_one, 1, 1, 0, stream, row, sh_degree, cam, s, sp_ab, sp_c, cov, keys, vals, cnt, err);
  ++g_launches;
}

// ------------------------------------------------------------------ given splats
// odgs_rasterize_splats: the per-Gaussian outputs of preprocess from caller-supplied
// projected splats (Splat2D records, projection.hpp:163-174) instead of a projection.
// k_clear_rows culls every row; k_load_splats then fills the rows of the splats.
__global__ void k_clear_rows(int64_t n, float4* __restrict__ sp_c, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  sp_c[i] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(0u));
  keys[i] = kCulledKey;
  vals[i] = (uint32_t)i;
  cnt[i] = 0;
}

__global__ void k_load_splats(int64_t n_splats, const float* __restrict__ rec, int width, int height,
                              int tile_size, float4* __restrict__ sp_ab, float4* __restrict__ sp_c,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err) {
  pdl_wait();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t n_inst = 0;
  if (s < n_splats) {
    const float* r = rec + s * kSplatRecord;  // index bits, mx, my, i00, i01, i11, depth, radius, opacity, rgb
    const uint32_t i = __float_as_uint(r[0]);
    const float mx = r[1], my = r[2], radius = r[7];
    uint32_t flags = kFlagVisible, total = 0;
    for (int k = 0; k < 3; ++k) {
      int span[4];
      if (instance_tiles(mx, my, radius, k, width, height, tile_size, span)) {
        flags |= kFlagShiftBase << k;
        ++n_inst;
        total += (uint32_t)(span[1] - span[0] + 1) * (uint32_t)(span[3] - span[2] + 1);
      }
    }
    sp_ab[2 * (int64_t)i] = make_float4(mx, my, r[3], r[4]);
    sp_ab[2 * (int64_t)i + 1] = make_float4(r[5], r[8], r[9], r[10]);
    sp_c[i] = make_float4(r[11], r[6], radius, __uint_as_float(flags));
    keys[i] = __float_as_uint(r[6]);
    cnt[i] = total;
  }
  const uint32_t v_sum = __reduce_add_sync(0xffffffffu, s < n_splats ? 1u : 0u);
  const uint32_t i_sum = __reduce_add_sync(0xffffffffu, n_inst);
  if ((threadIdx.x & 31) == 0 && (v_sum | i_sum)) {
    atomicAdd(&err->n_visible, (unsigned long long)v_sum);
    atomicAdd(&err->n_instances, (unsigned long long)i_sum);
  }
}

void launch_load_splats(int64_t n, int64_t n_splats, const float* rec, int width, int height, int tile_size,
                        float4* sp_ab, float4* sp_c, uint32_t* keys, uint32_t* vals, uint32_t* cnt, DevErrors* err,
                        cudaStream_t stream) {
  if (n == 0) return;
  launch_pdl(k_clear_rows, (unsigned)((n + 255) / 256), 256, 0, stream, n, sp_c, keys, vals, cnt);
  ++g_launches;
  if (n_splats == 0) return;
  launch_pdl(k_load_splats, (unsigned)((n_splats + 255) / 256), 256, 0, stream, n_splats, rec, width, height,
             tile_size, sp_ab, sp_c, keys, cnt, err);
  ++g_launches;
}

// ------------------------------------------------------------------ band pre-cull
// Row-band renders: a conservative float test finds the Gaussians whose instance boxes
// certainly miss the band's pixel rows; they get the culled outputs and skip the exact
// projection (binary64 transcendentals), which then runs only on the survivors. The box
// half-height is at most rb = cutoff * sqrt(lambda_max(Sigma_2D)) <= cutoff *
// sqrt(s_max^2 lambda_max(J J^T) + lowpass) (Sigma_2D = J Sigma J^T + lowpass I,
// lambda_max(Sigma) = s_max^2). J's rows are a0 = W/2pi sec/r and a1 = H/pi/r times two
// orthonormal rows of the tangent-frame rotation (projection.hpp:75-96), so J J^T =
// diag(a0^2, a1^2) and lambda_max(J J^T) = max(a0^2, a1^2); padded by 1% and 2 pixels.
// The test runs in the sine domain,
// with no inverse trigonometry: the centre row v = H/2 - H theta/pi lies above the band
// by more than rb iff theta > theta_top + rb pi/H iff sin(theta) = -mu_y/|mu| > sin(that)
// (both angles inside (-pi/2, pi/2)), likewise below. The fast-math errors (~1e-6 rad)
// are far inside the padding; angles within 0.01 rad of a pole are never culled (sine is
// flat there). Non-finite rows, near-zero quaternions and the zero-direction case survive,
// so the exact path reports them as before.
struct BandCull {
  float sin_top, cos_top, sin_bot, cos_bot;  // band edge angles (top: row0, bottom: row1)
  float top, bot;                            // the angles themselves
  float sec_max;                             // 1 / cos(max_elevation)
  float a0k, a1k, rad_per_px;                // W / 2pi, H / pi, pi / H
};

__device__ __forceinline__ BandCull make_band_cull(const DevCamera& cam, const DevSettings& s) {
  BandCull b;
  const float Hf = (float)cam.height;
  b.top = (Hf / 2.0f - (float)(s.band_ty0 * s.tile_size)) * kPiF / Hf;
  b.bot = (Hf / 2.0f - (float)(s.band_ty1 * s.tile_size)) * kPiF / Hf;
  sincosf(b.top, &b.sin_top, &b.cos_top);
  sincosf(b.bot, &b.sin_bot, &b.cos_bot);
  b.sec_max = 1.0f / cosf(s.max_elevation);
  b.a0k = (float)cam.width / (2.0f * kPiF);
  b.a1k = Hf / kPiF;
  b.rad_per_px = kPiF / Hf;
  return b;
}

// The pre-cull test on one row's values (p: mean, q: quaternion, ls: log-scales; fin: a
// sum of every parameter of the row, non-finite iff one of them is).
__device__ __forceinline__ bool band_survives_v(const float p[3], const float q[4], const float ls[3], float fin,
                                                const DevCamera& cam, const DevSettings& s, const BandCull& b) {
  float mu[3];
  to_camera(cam, p, mu);
  const float sq = sum3(mu[0] * mu[0], mu[1] * mu[1], mu[2] * mu[2]);
  const float depth = sqrtf(sq);
  const float qq = sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]);
  if (!(sq > 0.0f && qq > 1e-20f && isfinite(depth) && isfinite(fin))) return true;
  if (!(depth >= s.near_radius && depth <= s.far_radius)) return false;
  const float inv_d = 1.0f / depth;
  const float rho = sqrtf(mu[0] * mu[0] + mu[2] * mu[2]);
  const float sin_th = -mu[1] * inv_d;
  const float sec = fminf(depth / rho, b.sec_max);
  const float a0 = b.a0k * sec * inv_d, a1 = b.a1k * inv_d;
  const float smax = __expf(fmaxf(ls[0], fmaxf(ls[1], ls[2])));
  const float rb = s.cutoff_sigma * sqrtf(smax * smax * fmaxf(a0 * a0, a1 * a1) + s.lowpass_dilation) * 1.01f + 2.0f;
  const float rt = rb * b.rad_per_px;
  if (!(rt < 1.0f)) return true;
  float sr, cr;
  __sincosf(rt, &sr, &cr);
  constexpr float kPoleGuard = 1.5607963f;  // pi/2 - 0.01
  if (b.top + rt < kPoleGuard && sin_th > b.sin_top * cr + b.cos_top * sr) return false;
  if (b.bot - rt > -kPoleGuard && sin_th < b.sin_bot * cr - b.cos_bot * sr) return false;
  return true;
}

__device__ __forceinline__ bool band_survives(int64_t i, int64_t n, const float* __restrict__ means,
                                              const float* __restrict__ rotations,
                                              const float* __restrict__ log_scales,
                                              const float* __restrict__ raw_opacities,
                                              const float* __restrict__ colors, int n_sh,
                                              const float* __restrict__ sh_rest, const DevCamera& cam,
                                              const DevSettings& s, const BandCull& b) {
  const float p[3] = {__ldg(means + i), __ldg(means + n + i), __ldg(means + 2 * n + i)};
  const float q[4] = {__ldg(rotations + i), __ldg(rotations + n + i), __ldg(rotations + 2 * n + i),
                      __ldg(rotations + 3 * n + i)};
  const float ls[3] = {__ldg(log_scales + i), __ldg(log_scales + n + i), __ldg(log_scales + 2 * n + i)};
  // Every parameter of the row is checked (first_non_finite, rasterizer.hpp:133-136): a
  // non-finite value anywhere sends the row to the exact path, which reports it, so a
  // band render fails exactly where the full render does. A sum of the parameters is
  // non-finite if any of them is (an overflow to inf only costs a needless survivor).
  float fin = ((p[0] + p[1]) + (p[2] + q[0])) + ((q[1] + q[2]) + (q[3] + ls[0]));
  fin += (ls[1] + ls[2]) + (__ldg(raw_opacities + i) +
                            ((__ldg(colors + i) + __ldg(colors + n + i)) + __ldg(colors + 2 * n + i)));
  for (int k = 0; k < n_sh; ++k) fin += __ldg(sh_rest + (int64_t)k * n + i);
  return band_survives_v(p, q, ls, fin, cam, s, b);
}

// Fused band pre-cull + exact preprocess + band compaction, one warp per chunk of
// kBandWarpChunk consecutive Gaussians. The warp streams its chunk with coalesced loads,
// queues the pre-cull survivors in shared memory and projects them 32 at a time (full
// warps, instead of one scattered gather per survivor), then appends the (depth key,
// index) pairs of those with entries in the band, in index order, to its own segment
// of seg_keys / seg_vals; seg_count[warp] is the segment length. Culled Gaussians get
// the culled per-Gaussian outputs (cnt 0, sp_c 0); their keys / vals are not written
// (only the compacted pairs are sorted).
constexpr int kBandWarpChunk = 512;  // 2048: 2.7% slower C5 bands (tail wave of long warps)
constexpr int kBandUnroll = 4;
constexpr int kBandQueue = 256;  // >= 31 + 32 * kBandUnroll, a power of two

__global__ void __launch_bounds__(256, 3) k_band_preprocess(
    int64_t n, const float* __restrict__ means, const float* __restrict__ rotations,
    const float* __restrict__ log_scales, const float* __restrict__ raw_opacities,
    const float* __restrict__ colors, DevCamera cam, DevSettings s, float4* __restrict__ sp_ab,
    float4* __restrict__ sp_c, float4* __restrict__ cov_out, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err, int sh_degree,
    const float* __restrict__ sh_rest, uint32_t* __restrict__ seg_keys, uint32_t* __restrict__ seg_vals,
    uint32_t* __restrict__ seg_count) {
  pdl_wait();
  __shared__ uint32_t s_queue[8][kBandQueue];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * 8 + warp;
  const int64_t base = w * kBandWarpChunk;
  if (base >= n) return;
  const int64_t end = min(base + (int64_t)kBandWarpChunk, n);
  uint32_t* q = s_queue[warp];  // ring buffer of survivor indices
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t head = 0, tail = 0;
  uint32_t out_len = 0, n_surv = 0, n_vis = 0, n_inst = 0;
  const BandCull bc = make_band_cull(cam, s);
  const int n_sh = sh_degree > 0 ? 3 * sh_count(sh_degree) : 0;
  // Projects the next `count` queued survivors (one per lane) and appends the pairs
  // with band entries.
  auto drain = [&](uint32_t count) {
    bool visible = false, has = false;
    uint32_t key = 0, idx = 0;
    if (lane < count) {
      idx = q[(head + lane) & (kBandQueue - 1)];
      n_inst += preprocess_one(idx, n, means, rotations, log_scales, raw_opacities, colors, sh_degree, sh_rest, cam,
                               s, sp_ab, sp_c, cov_out, keys, vals, cnt, err, &visible);
      has = cnt[idx] > 0;
      key = keys[idx];
    }
    head += count;
    n_vis += visible ? 1u : 0u;
    const uint32_t hb = __ballot_sync(0xffffffffu, has);
    if (has) {
      const int64_t o = base + out_len + __popc(hb & lt);
      seg_keys[o] = key;
      seg_vals[o] = idx;
    }
    out_len += __popc(hb);
  };
  // The pre-cull streams kBandUnroll groups of 32 at a time (independent loads in
  // flight), then the queue drains in full warps.
  for (int64_t c = base; c < end; c += 32 * kBandUnroll) {
    bool sv[kBandUnroll];
#pragma unroll
    for (int u = 0; u < kBandUnroll; ++u) {
      const int64_t i = c + u * 32 + lane;
      // clamped index: unconditional loads, all kBandUnroll groups in flight
      sv[u] = band_survives(min(i, end - 1), n, means, rotations, log_scales, raw_opacities, colors, n_sh, sh_rest,
                            cam, s, bc) && i < end;
    }
#pragma unroll
    for (int u = 0; u < kBandUnroll; ++u) {
      const int64_t i = c + u * 32 + lane;
      if (i < end && !sv[u]) {
        cnt[i] = 0;
        sp_c[i] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(0u));
      }
      const uint32_t sb = __ballot_sync(0xffffffffu, sv[u]);
      if (sv[u]) q[(tail + __popc(sb & lt)) & (kBandQueue - 1)] = (uint32_t)i;
      tail += __popc(sb);
      n_surv += __popc(sb);
    }
    __syncwarp();
    while (tail - head >= 32) drain(32);
    __syncwarp();
  }
  if (tail != head) drain(tail - head);
  const uint32_t vis = __reduce_add_sync(0xffffffffu, n_vis);
  const uint32_t inst = __reduce_add_sync(0xffffffffu, n_inst);
  if (lane == 0) {
    seg_count[w] = out_len;
    if (vis | inst) {
      atomicAdd(&err->n_visible, (unsigned long long)vis);
      atomicAdd(&err->n_instances, (unsigned long long)inst);
    }
    if (n_surv) atomicAdd(&err->n_precull, (unsigned long long)n_surv);
  }
}

// The same pass for SH degree 0 clouds with n % 4 == 0 and 16-byte aligned rows: lane l
// takes kRows consecutive rows (default 2: one 8-byte load per parameter row, 14 loads
// per lane in flight, 64 + registers at 6 CTAs/SM; 4 rows with 16-byte loads need 111
// registers, 4 CTAs/SM, and are 6 % slower at C5); the pre-cull runs on the
// loaded values, and each survivor is queued with its 14 parameters, so the exact path
// reads shared memory instead of re-gathering the row (scattered survivor rows would cost
// a 32-byte sector per 4-byte parameter). Survivors are queued in index order (a warp
// prefix sum over the lanes' counts); the group's cnt / sp_c are cleared with vector
// stores first (the exact path overwrites the survivors' after the __syncwarp).
#ifndef ODGS_BANDVEC_ROWS
#define ODGS_BANDVEC_ROWS 2
#endif
#ifndef ODGS_BANDVEC_MINB
#define ODGS_BANDVEC_MINB 6
#endif
constexpr int kBandVecWarps = 4;

// kRows consecutive rows per lane (float4: 4, float2: 2); the queue holds a warp's
// leftover survivors (< 32) plus one group of 32 kRows rows.
template <int kRows>
struct BandVec {
  static constexpr uint32_t kQueue = 32 + 32 * kRows;
  using V = typename std::conditional<kRows == 4, float4, typename std::conditional<kRows == 2, float2, float>::type>::type;
  __device__ static float el(const V& v, int u) {
    if constexpr (kRows == 4) return u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w;
    else if constexpr (kRows == 2) return u == 0 ? v.x : v.y;
    else return v;
  }
};

template <int kRows, int kMinBlocks>
__global__ void __launch_bounds__(kBandVecWarps * 32, kMinBlocks) k_band_preprocess_vec(
    int64_t n, const float* __restrict__ means, const float* __restrict__ rotations,
    const float* __restrict__ log_scales, const float* __restrict__ raw_opacities,
    const float* __restrict__ colors, DevCamera cam, DevSettings s, float4* __restrict__ sp_ab,
    float4* __restrict__ sp_c, float4* __restrict__ cov_out, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt, DevErrors* __restrict__ err,
    uint32_t* __restrict__ seg_keys, uint32_t* __restrict__ seg_vals, uint32_t* __restrict__ seg_count) {
  pdl_wait();
  using BV = BandVec<kRows>;
  using V = typename BV::V;
  constexpr uint32_t kQ = BV::kQueue;
  constexpr int kGroup = 32 * kRows;
  __shared__ uint32_t s_idx[kBandVecWarps][kQ];
  __shared__ float s_val[kBandVecWarps][14][kQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * kBandVecWarps + warp;
  const int64_t base = w * kBandWarpChunk;
  if (base >= n) return;
  const int64_t end = min(base + (int64_t)kBandWarpChunk, n);
  uint32_t head = 0, tail = 0;
  uint32_t out_len = 0, n_surv = 0, n_vis = 0, n_inst = 0;
  const uint32_t lt = (1u << lane) - 1u;
  const BandCull bc = make_band_cull(cam, s);
  auto drain = [&](uint32_t count) {
    bool visible = false, has = false;
    uint32_t key = 0, idx = 0;
    if (lane < count) {
      const uint32_t slot = (head + lane) % kQ;
      idx = s_idx[warp][slot];
      float v[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) v[k] = s_val[warp][k][slot];
      n_inst += preprocess_vals(idx, n, v, 0, nullptr, cam, s, sp_ab, sp_c, cov_out, keys, vals, cnt, err, &visible);
      has = cnt[idx] > 0;
      key = keys[idx];
    }
    head += count;
    n_vis += visible ? 1u : 0u;
    const uint32_t hb = __ballot_sync(0xffffffffu, has);
    if (has) {
      const int64_t o = base + out_len + __popc(hb & lt);
      seg_keys[o] = key;
      seg_vals[o] = idx;
    }
    out_len += __popc(hb);
  };
  const float* rows[14] = {means,     means + n,          means + 2 * n,      rotations,          rotations + n,
                           rotations + 2 * n, rotations + 3 * n, log_scales,  log_scales + n,     log_scales + 2 * n,
                           raw_opacities, colors,         colors + n,         colors + 2 * n};
  for (int64_t c = base; c < end; c += kGroup) {
    const int64_t i0 = c + kRows * lane;
    const bool any = i0 < end;  // end - base is a multiple of kRows
    V v[14];
#pragma unroll
    for (int k = 0; k < 14; ++k) v[k] = any ? __ldcs(reinterpret_cast<const V*>(rows[k] + i0)) : V{};
    uint32_t m = 0;
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      auto el = [&](int k) { return BV::el(v[k], u); };
      const float p[3] = {el(0), el(1), el(2)};
      const float qv[4] = {el(3), el(4), el(5), el(6)};
      const float ls[3] = {el(7), el(8), el(9)};
      // every parameter of the row: non-finite anywhere -> the exact path reports it
      const float fin = (((p[0] + p[1]) + (p[2] + qv[0])) + ((qv[1] + qv[2]) + (qv[3] + ls[0]))) +
                        ((ls[1] + ls[2]) + (el(10) + ((el(11) + el(12)) + el(13))));
      if (any && band_survives_v(p, qv, ls, fin, cam, s, bc)) m |= 1u << u;
    }
    if (any) {
      if constexpr (kRows == 4) reinterpret_cast<uint4*>(cnt + i0)[0] = make_uint4(0u, 0u, 0u, 0u);
      else if constexpr (kRows == 2) reinterpret_cast<uint2*>(cnt + i0)[0] = make_uint2(0u, 0u);
      else cnt[i0] = 0u;
#pragma unroll
      for (int u = 0; u < kRows; ++u) sp_c[i0 + u] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(0u));
    }
    const uint32_t cnt_l = __popc(m);
    uint32_t incl = cnt_l;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    uint32_t pos = tail + incl - cnt_l;
#pragma unroll
    for (int u = 0; u < kRows; ++u)
      if (m & (1u << u)) {
        const uint32_t slot = pos % kQ;
        s_idx[warp][slot] = (uint32_t)(i0 + u);
#pragma unroll
        for (int k = 0; k < 14; ++k) s_val[warp][k][slot] = BV::el(v[k], u);
        ++pos;
      }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    tail += total;
    n_surv += total;
    __syncwarp();
    while (tail - head >= 32) drain(32);
    __syncwarp();
  }
  if (tail != head) drain(tail - head);
  const uint32_t vis = __reduce_add_sync(0xffffffffu, n_vis);
  const uint32_t inst = __reduce_add_sync(0xffffffffu, n_inst);
  if (lane == 0) {
    seg_count[w] = out_len;
    if (vis | inst) {
      atomicAdd(&err->n_visible, (unsigned long long)vis);
      atomicAdd(&err->n_instances, (unsigned long long)inst);
    }
    if (n_surv) atomicAdd(&err->n_precull, (unsigned long long)n_surv);
  }
}

// Concatenates the warp segments (one warp per segment) at their scanned offsets.
__global__ void k_concat_segments(int64_t n_seg, const uint32_t* __restrict__ seg_count,
                                  const uint32_t* __restrict__ seg_off, const uint32_t* __restrict__ seg_keys,
                                  const uint32_t* __restrict__ seg_vals, uint32_t* __restrict__ keys_out,
                                  uint32_t* __restrict__ vals_out) {
  pdl_wait();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_seg) return;
  const uint32_t len = seg_count[w], off = seg_off[w];
  const int64_t src = w * kBandWarpChunk;
  for (uint32_t k = lane; k < len; k += 32) {
    keys_out[off + k] = seg_keys[src + k];
    vals_out[off + k] = seg_vals[src + k];
  }
}

int64_t band_segments(int64_t n) { return (n + kBandWarpChunk - 1) / kBandWarpChunk; }

void launch_band_preprocess(const PreprocessArgs& a, uint32_t* seg_keys, uint32_t* seg_vals, uint32_t* seg_count,
                            cudaStream_t stream) {
  if (a.n == 0) return;
  const int64_t n_seg = band_segments(a.n);
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = a.sh_degree == 0 && a.n % 4 == 0 && aligned(a.means) && aligned(a.rotations) &&
                   aligned(a.log_scales) && aligned(a.raw_opacities) && aligned(a.colors);
  if (vec) {
    launch_pdl(k_band_preprocess_vec<ODGS_BANDVEC_ROWS, ODGS_BANDVEC_MINB>,
               (unsigned)((n_seg + kBandVecWarps - 1) / kBandVecWarps), kBandVecWarps * 32, 0,
               stream, a.n, a.means, a.rotations, a.log_scales, a.raw_opacities, a.colors, a.cam, a.settings, a.sp_ab,
               a.sp_c, a.cov_out, a.keys, a.vals, a.cnt, a.err, seg_keys, seg_vals, seg_count);
    ++g_launches;
    return;
  }
  launch_pdl(k_band_preprocess, (unsigned)((n_seg + 7) / 8), 256, 0, stream, 
      a.n, a.means, a.rotations, a.log_scales, a.raw_opacities, a.colors, a.cam, a.settings, a.sp_ab, a.sp_c,
      a.cov_out, a.keys, a.vals, a.cnt, a.err, a.sh_degree, a.sh_rest, seg_keys, seg_vals, seg_count);
  ++g_launches;
}

void launch_concat_segments(int64_t n, const uint32_t* seg_count, const uint32_t* seg_off, const uint32_t* seg_keys,
                            const uint32_t* seg_vals, uint32_t* keys_out, uint32_t* vals_out, cudaStream_t stream) {
  const int64_t n_seg = band_segments(n);
  if (n_seg == 0) return;
  launch_pdl(k_concat_segments, (unsigned)((n_seg * 32 + 255) / 256), 256, 0, stream, n_seg, seg_count, seg_off, seg_keys,
                                                                               seg_vals, keys_out, vals_out);
  ++g_launches;
}

// ------------------------------------------------------------------ stream-ordered resets
// Kernels instead of memcpy / memset nodes, so they join the programmatic-launch chain.
// mode 0: everything; 1: the counters (sticky words kept); 2: the sticky words only.
__global__ void k_reset_errors(DevErrors* __restrict__ e, int mode) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  if (mode != 1) {
    e->nonfinite = kNoError;
    e->project = kNoError;
    e->bwd_domain = kNoError;
    e->bwd_nonfinite = kNoError;
    e->overflow = 0;
  }
  if (mode == 2) return;
  e->n_entries = 0;
  e->n_visible = 0;
  e->n_instances = 0;
  e->n_band = 0;
  e->n_precull = 0;
  e->k_sort = 0;
}

void launch_reset_errors(DevErrors* e, bool keep_sticky, cudaStream_t stream) {
  launch_pdl(k_reset_errors, 1, 32, 0, stream, e, keep_sticky ? 1 : 0);
  ++g_launches;
}

void launch_reset_sticky(DevErrors* e, cudaStream_t stream) {
  launch_pdl(k_reset_errors, 1, 32, 0, stream, e, 2);
  ++g_launches;
}

__global__ void k_zero_bytes(uint4* __restrict__ p, int64_t n16, uint8_t* __restrict__ tail, int n_tail) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) p[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x == 0 && (int)threadIdx.x < n_tail) tail[threadIdx.x] = 0;
}

void launch_zero_bytes(void* p, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return;
  // p is a cudaMalloc base (256-byte aligned)
  const int64_t n16 = (int64_t)(bytes / 16);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, 148 * 8));
  launch_pdl(k_zero_bytes, grid, 256, 0, stream, static_cast<uint4*>(p), n16,
             static_cast<uint8_t*>(p) + 16 * n16, (int)(bytes - 16 * (size_t)n16));
  ++g_launches;
}

// ------------------------------------------------------------------ emit tile entries
constexpr int kEmitWarps = 8;

__global__ void __launch_bounds__(kEmitWarps * 32) k_emit(
    int64_t n, const uint32_t* __restrict__ sorted_idx, const uint32_t* __restrict__ cnt_sorted,
    const uint32_t* __restrict__ off_sorted, const float4* __restrict__ sp_ab, const float4* __restrict__ sp_c,
    int width, int height, int tile_size, int tiles_x, int band_ty0, int band_ty1, uint32_t* __restrict__ out_keys,
    uint32_t* __restrict__ out_vals, uint32_t* __restrict__ ent_off_idx, const uint32_t* __restrict__ n_dev,
    const unsigned long long* __restrict__ k_total, uint32_t capacity, unsigned long long* __restrict__ k_sort,
    unsigned long long* __restrict__ overflow) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);  // depth-sorted ranks counted on the device
  if (k_sort && blockIdx.x == 0 && threadIdx.x == 0) {
    // Entries to sort / bin: all of them, or the capacity if they do not fit (the
    // overflow word then makes the host re-run the frame with enough room).
    const unsigned long long t = *k_total;
    *k_sort = t <= capacity ? t : capacity;
    if (t > capacity) atomicMax(overflow, t);
  }
  __shared__ int s_span[kEmitWarps][32][12];
  __shared__ uint32_t s_area[kEmitWarps][32][3];
  __shared__ uint32_t s_magic[kEmitWarps][32][3];  // ceil-ish 2^32 / span width (0: divide)
  __shared__ uint32_t s_excl[kEmitWarps][32];
  __shared__ uint32_t s_gid[kEmitWarps][32];
  __shared__ uint8_t s_nz[kEmitWarps][32];  // lanes with entries, by rank
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = ((int64_t)blockIdx.x * kEmitWarps + warp) * 32;
  if (base >= n) return;
  const int64_t r = base + lane;
  const bool valid = r < n;
  uint32_t c = 0, gid = 0, off = 0;
  if (valid) {
    c = cnt_sorted[r];
    gid = sorted_idx[r];
    off = off_sorted[r];
    ent_off_idx[gid] = off;
  }
  uint32_t areas[3] = {0, 0, 0};
  if (c > 0) {
    const float4 a = sp_ab[2 * (int64_t)gid];
    const float radius = sp_c[gid].z;
    for (int k = 0; k < 3; ++k) {
      int span[4];
      if (band_tiles(a.x, a.y, radius, k, width, height, tile_size, band_ty0, band_ty1, span)) {
        const uint32_t w = (uint32_t)(span[1] - span[0] + 1);
        areas[k] = w * (uint32_t)(span[3] - span[2] + 1);
        for (int q = 0; q < 4; ++q) s_span[warp][lane][4 * k + q] = span[q];
        // j / w == umulhi(j, m) for m = floor((2^32 - 1) / w) + 1 when j * w < 2^32.
        s_magic[warp][lane][k] = (uint64_t)areas[k] * w < (1ull << 32) ? 0xFFFFFFFFu / w + 1u : 0u;
      }
    }
  }
  s_area[warp][lane][0] = areas[0];
  s_area[warp][lane][1] = areas[1];
  s_area[warp][lane][2] = areas[2];
  s_gid[warp][lane] = gid;
  uint32_t incl = c;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const uint32_t excl = incl - c;
  s_excl[warp][lane] = excl;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t base_off = __shfl_sync(0xffffffffu, off, 0);
  const uint32_t lt = (1u << lane) - 1u, le = (2u << lane) - 1u;
  const uint32_t nz_mask = __ballot_sync(0xffffffffu, c > 0);
  if (c > 0) s_nz[warp][__popc(nz_mask & lt)] = (uint8_t)lane;
  __syncwarp();
  // Owner of entry p: the lanes with entries start their runs in increasing order, so
  // in each chunk of 32 entries the owner rank advances by the starts at or before p
  // (one OR-reduction of start bits per chunk instead of a binary search per entry).
  int rank = -1;  // owner rank of the entry before the chunk
  for (uint32_t P = 0; P < total; P += 32) {
    const uint32_t o = excl - P;
    const uint32_t bits = __reduce_or_sync(0xffffffffu, (c > 0 && o < 32u) ? (1u << o) : 0u);
    const int rk = rank + __popc(bits & le);
    rank += __popc(bits);
    const uint32_t p = P + lane;
    if (p < total) {
      const int lo = s_nz[warp][rk];
      uint32_t j = p - s_excl[warp][lo];
      int k = 0;
      while (j >= s_area[warp][lo][k]) {
        j -= s_area[warp][lo][k];
        ++k;
      }
      const int* span = s_span[warp][lo] + 4 * k;
      const uint32_t w = (uint32_t)(span[1] - span[0] + 1);
      const uint32_t m = s_magic[warp][lo][k];
      const uint32_t q = m ? __umulhi(j, m) : j / w;
      const int ty = span[2] + (int)q, tx = span[0] + (int)(j - q * w);
      if (base_off + p < capacity) {
        out_keys[base_off + p] = (uint32_t)(ty * tiles_x + tx);
        out_vals[base_off + p] = (s_gid[warp][lo] << 2) | (uint32_t)k;
      }
    }
  }
}

void launch_emit(const EmitArgs& a, cudaStream_t stream) {
  if (a.n == 0) return;
  const int64_t warps = (a.n + 31) / 32;
  const int64_t grid = (warps + kEmitWarps - 1) / kEmitWarps;
  launch_pdl(k_emit, (unsigned)grid, kEmitWarps * 32, 0, stream, a.n, a.sorted_idx, a.cnt_sorted, a.off_sorted, a.sp_ab,
             a.sp_c, a.width, a.height, a.tile_size, a.tiles_x, a.band_ty0, a.band_ty1, a.out_keys, a.out_vals,
             a.ent_off_idx, a.n_dev, a.total, a.capacity, a.k_sort, a.overflow);
  ++g_launches;
}

// ------------------------------------------------------------------ tile ranges
// offsets[t] = first entry of tile t (CSR, empty tiles included). Entries only fall in
// the band's tiles [t0, t1): thread e fills the tiles whose range starts at entry e
// (from the previous entry's tile + 1 up to its own), clamped to the band; the tiles
// outside the band (empty) are filled in parallel by k_fill_outside.
// Thread i covers entries 4i .. 4i+3 (one 16-byte key load; the sentinel position K
// belongs to the thread whose range contains it).
__global__ void k_tile_ranges(uint32_t k_entries, const uint32_t* __restrict__ keys, uint32_t t0, uint32_t t1,
                              int32_t* __restrict__ offsets, const uint32_t* __restrict__ k_dev) {
  pdl_wait();
  if (k_dev) k_entries = min(k_entries, *k_dev);  // capacity-sized launch, count on the device
  const uint32_t e_first = 4u * (blockIdx.x * blockDim.x + threadIdx.x);
  if (e_first > k_entries) return;
  uint32_t kv[4];
  if (e_first + 4u <= k_entries) {
    const uint4 q = *reinterpret_cast<const uint4*>(keys + e_first);
    kv[0] = q.x; kv[1] = q.y; kv[2] = q.z; kv[3] = q.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) kv[u] = e_first + u < k_entries ? keys[e_first + u] : t1;  // K: sentinel
  }
  uint32_t prev_key = e_first == 0 ? 0xFFFFFFFFu : keys[e_first - 1];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t e = e_first + u;
    if (e > k_entries) break;
    const uint32_t cur = kv[u];
    if (e == 0 || e == k_entries || prev_key != cur) {
      const uint32_t first = e == 0 ? t0 : prev_key + 1u;  // first tile whose range starts at e
      for (uint32_t t = first; t <= cur; ++t) offsets[t] = (int32_t)e;
    }
    prev_key = cur;
  }
}

__global__ void k_fill_outside(uint32_t k_entries, uint32_t n_tiles, uint32_t t0, uint32_t t1,
                               int32_t* __restrict__ offsets, const uint32_t* __restrict__ k_dev) {
  pdl_wait();
  if (k_dev) k_entries = min(k_entries, *k_dev);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < t0) offsets[t] = 0;
  else if (t > t1 && t <= n_tiles) offsets[t] = (int32_t)k_entries;
}

void launch_tile_ranges(uint32_t k_entries, const uint32_t* keys, uint32_t n_tiles, uint32_t t0, uint32_t t1,
                        int32_t* offsets, cudaStream_t stream, const uint32_t* k_dev) {
  if (k_entries == 0) {
    cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (n_tiles + 1), stream);
    return;
  }
  const uint32_t threads = k_entries / 4 + 1;
  launch_pdl(k_tile_ranges, (threads + 255) / 256, 256, 0, stream, k_entries, keys, t0, t1, offsets, k_dev);
  ++g_launches;
  if (t0 > 0 || t1 < n_tiles) {
    launch_pdl(k_fill_outside, (n_tiles + 1 + 255) / 256, 256, 0, stream, k_entries, n_tiles, t0, t1, offsets,
               k_dev);
    ++g_launches;
  }
}

// ------------------------------------------------------------------ tile order
// Launch order of the per-tile kernels (blend, backward raster): tiles by descending
// list length (quarter-octave buckets), so the few very long lists of the pole and
// seam tiles start first instead of trailing the grid. Per-tile results do not depend
// on the order (each CTA owns its tile), so the bucket-internal order — set by
// shared-memory atomics — is free.
constexpr int kOrderThreads = 1024;
constexpr int kOrderBuckets = 128;

__device__ __forceinline__ int order_bucket(int32_t len) {
  const uint32_t v = (uint32_t)len + 1u;
  const int b = 31 - __clz(v);                                  // floor(log2 v)
  const int frac = b >= 2 ? (int)((v >> (b - 2)) & 3u) : (int)((v << (2 - b)) & 3u);
  return kOrderBuckets - 1 - min(kOrderBuckets - 1, 4 * b + frac);  // longest first
}

__global__ void __launch_bounds__(kOrderThreads) k_tile_order(const int32_t* __restrict__ offsets, int tile_base,
                                                              int n, uint32_t* __restrict__ order) {
  pdl_wait();
  __shared__ __align__(16) uint32_t s_cnt[kOrderBuckets];
  for (int b = threadIdx.x; b < kOrderBuckets; b += kOrderThreads) s_cnt[b] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += kOrderThreads)
    atomicAdd(&s_cnt[order_bucket(offsets[tile_base + t + 1] - offsets[tile_base + t])], 1u);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the buckets: 4 per lane, then over the warp
    static_assert(kOrderBuckets == 128, "4 buckets per lane");
    const int lane = threadIdx.x;
    const uint4 c = *reinterpret_cast<const uint4*>(&s_cnt[4 * lane]);
    const uint32_t own = c.x + c.y + c.z + c.w;
    uint32_t incl = own;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const uint32_t e = incl - own;
    *reinterpret_cast<uint4*>(&s_cnt[4 * lane]) = make_uint4(e, e + c.x, e + c.x + c.y, e + c.x + c.y + c.z);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += kOrderThreads)
    order[atomicAdd(&s_cnt[order_bucket(offsets[tile_base + t + 1] - offsets[tile_base + t])], 1u)] = (uint32_t)t;
}

void launch_tile_order(const int32_t* offsets, int tile_base, int n, uint32_t* order, cudaStream_t stream) {
  if (n <= 0) return;
  launch_pdl(k_tile_order, 1, kOrderThreads, 0, stream, offsets, tile_base, n, order);
  ++g_launches;
}

// ------------------------------------------------------------------ blend
constexpr int kBlendThreads = 256;

template <int PPT>
__global__ void __launch_bounds__(kBlendThreads) k_blend(
    const int32_t* __restrict__ offsets, const uint32_t* __restrict__ vals, const float4* __restrict__ sp_ab,
    const float4* __restrict__ sp_c, int width, int height, int tile_size, int tiles_x, float alpha_clamp,
    float transmittance_floor, float cutoff2, float* __restrict__ image, float* __restrict__ trans_out,
    int32_t* __restrict__ walked_out, unsigned long long* __restrict__ work, int tile_base, PeerImages peers) {
  __shared__ float s_cx[kBlendThreads], s_cy[kBlendThreads], s_i00[kBlendThreads], s_i01x2[kBlendThreads],
      s_i11[kBlendThreads], s_op[kBlendThreads], s_r[kBlendThreads], s_g[kBlendThreads], s_b[kBlendThreads];
  const int tile = tile_base + blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int e0 = offsets[tile], e1 = offsets[tile + 1];
  const int tid = threadIdx.x;
  const int area = tile_size * tile_size;
  // Tiles larger than PPT * 256 pixels (tile_size > 64) are blended in pixel chunks,
  // each walking the tile's list again.
  for (int chunk = 0; chunk < area; chunk += PPT * kBlendThreads) {
  float px[PPT], py[PPT], t[PPT], cr[PPT], cg[PPT], cb[PPT];
  int walked[PPT];
  bool done[PPT];
  int64_t pix[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int lp = chunk + tid + q * kBlendThreads;
    // Column-major pixel order inside the tile so a warp writes runs of y (the
    // images are column-major, y + x*H).
    const int lx = lp / tile_size, ly = lp - lx * tile_size;
    const int x = tx * tile_size + lx, y = ty * tile_size + ly;
    const bool valid = lp < area && x < width && y < height;
    px[q] = (float)x + 0.5f;
    py[q] = (float)y + 0.5f;
    t[q] = 1.0f;
    cr[q] = cg[q] = cb[q] = 0.0f;
    walked[q] = e1 - e0;
    done[q] = !valid;
    pix[q] = valid ? (int64_t)x * height + y : -1;
  }

  const float W = (float)width;
  uint32_t contrib = 0;
  for (int base = e0; base < e1; base += kBlendThreads) {
    bool any_alive = false;
#pragma unroll
    for (int q = 0; q < PPT; ++q) any_alive |= !done[q];
    if (__syncthreads_count(any_alive) == 0) break;
    const int e = base + tid;
    if (e < e1) {
      const uint32_t v = vals[e];
      const uint32_t g = v >> 2;
      const int k = (int)(v & 3u);
      const float4 a = __ldg(sp_ab + 2 * (int64_t)g);
      const float4 b = __ldg(sp_ab + 2 * (int64_t)g + 1);
      const float c2 = __ldg(&sp_c[g].x);
      const float shift = k == 0 ? -W : (k == 1 ? 0.0f : W);
      s_cx[tid] = a.x + shift;
      s_cy[tid] = a.y;
      s_i00[tid] = a.z;
      s_i01x2[tid] = 2.0f * a.w;
      s_i11[tid] = b.x;
      s_op[tid] = b.y;
      s_r[tid] = b.z;
      s_g[tid] = b.w;
      s_b[tid] = c2;
    }
    __syncthreads();
    const int count = min(kBlendThreads, e1 - base);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (done[q]) continue;
      float tq = t[q], r = cr[q], gg = cg[q], bb = cb[q];
      const float x0 = px[q], y0 = py[q];
      int j = 0;
      for (; j < count; ++j) {
        const float dx = x0 - s_cx[j];
        const float dy = y0 - s_cy[j];
        const float d2 = s_i00[j] * dx * dx + s_i01x2[j] * dx * dy + s_i11[j] * dy * dy;
        if (d2 > cutoff2) continue;
        const float alpha = std_min(alpha_clamp, s_op[j] * pm_expf_blend(-d2 / 2.0f));
        const float t_next = tq * (1.0f - alpha);
        if (t_next < transmittance_floor) {
          walked[q] = base + j - e0;
          done[q] = true;
          break;
        }
        const float w = alpha * tq;
        ++contrib;
        r = r + s_r[j] * w;
        gg = gg + s_g[j] * w;
        bb = bb + s_b[j] * w;
        tq = t_next;
      }
      t[q] = tq;
      cr[q] = r;
      cg[q] = gg;
      cb[q] = bb;
    }
    __syncthreads();
  }

  const int64_t plane = (int64_t)width * height;
  // Work counters for the roofline: entries examined (walked, plus the terminating
  // entry when the walk stopped early) and entries composited.
  uint32_t exam = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q)
    if (pix[q] >= 0) exam += (uint32_t)min(walked[q] + 1, e1 - e0);
  const uint32_t w_exam = __reduce_add_sync(0xffffffffu, exam);
  const uint32_t w_contrib = __reduce_add_sync(0xffffffffu, contrib);
  if ((tid & 31) == 0 && work) {
    atomicAdd(work, (unsigned long long)w_exam);
    atomicAdd(work + 1, (unsigned long long)w_contrib);
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (pix[q] < 0) continue;
    image[pix[q]] = cr[q];
    image[plane + pix[q]] = cg[q];
    image[2 * plane + pix[q]] = cb[q];
    trans_out[pix[q]] = t[q];
    walked_out[pix[q]] = walked[q];
#pragma unroll
    for (int k = 0; k < kMaxPeers; ++k) {  // fused band all-gather, as in k_blend_cull
      if (k >= peers.n) break;
      float* o = peers.ptr[k];
      o[pix[q]] = cr[q];
      o[plane + pix[q]] = cg[q];
      o[2 * plane + pix[q]] = cb[q];
    }
  }
  __syncthreads();  // the next chunk restages the shared batch
  }
}

// ------------------------------------------------------------------ blend with warp culling
// 6 CTAs (48 warps) per SM: the walk is latency-bound on its dependent chains.
// kSmallCutoff: cutoff^2 <= 172, so every composited entry has -d2/2 >= -86 and the
// exponential's underflow branch is dead: pm_expf_blend(x) == pm_expf_blend_core(
// fminf(x, 88)) there, bit for bit, without a branch in the walk.
template <bool kSmallCutoff, bool kCount>
#ifndef ODGS_BLEND_MINB
#define ODGS_BLEND_MINB 7
#endif
__global__ void __launch_bounds__(kBlendThreads, ODGS_BLEND_MINB) k_blend_cull(
    const int32_t* __restrict__ offsets, const uint32_t* __restrict__ vals, const float4* __restrict__ sp_ab,
    const float4* __restrict__ sp_c, int width, int height, int tile_size, int tiles_x, float alpha_clamp,
    float transmittance_floor, float cutoff2, float* __restrict__ image, float* __restrict__ trans_out,
    int32_t* __restrict__ walked_out, unsigned long long* __restrict__ work, int tile_base,
    const uint32_t* __restrict__ order, PeerImages peers) {
  pdl_wait();
  constexpr int kWarps = kBlendThreads / 32;
  // One 48-byte record per staged entry: the walk addresses all three parts from one
  // base with immediate offsets (separate arrays cost an address computation each).
  struct alignas(16) Staged {
    float4 geo;  // cx, cy, i00, 2*i01
    float4 att;  // i11, opacity, r, g
    float4 b;    // b, -, -, -
  };
  __shared__ Staged s_ent[kBlendThreads];
  __shared__ uint8_t s_mask[kBlendThreads];
  // Per-warp lists of byte offsets into s_ent (the walk addresses a record without a
  // multiply).
  __shared__ uint16_t s_list[kWarps][kBlendThreads];
  __shared__ float4 s_wbox[kWarps];  // pixel-centre bbox of each warp: xmin, xmax, ymin, ymax

  const int tile = tile_base + (int)(order ? order[blockIdx.x] : blockIdx.x);
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int e0 = offsets[tile], e1 = offsets[tile + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // Pixel of this thread. 16x16 tiles: each warp owns an 8-wide x 4-tall block (lanes
  // run down a column in fours: the image is column-major). Wide blocks match the
  // horizontally stretched footprints of the ERP projection (sec(theta) in x), so the
  // warp culling below rejects more entries (measured: C3 blend 0.618 -> 0.563 ms vs
  // 4 x 8 blocks, 16 x 2 blocks 0.605 ms).
  int lx, ly;
  bool valid;
  if (tile_size == 16) {
    lx = (warp & 1) * 8 + (lane >> 2);
    ly = (warp >> 1) * 4 + (lane & 3);
    valid = true;
  } else {
    lx = tid / tile_size;
    ly = tid - lx * tile_size;
    valid = tid < tile_size * tile_size;
  }
  const int x = tx * tile_size + lx, y = ty * tile_size + ly;
  valid = valid && x < width && y < height;
  const float px = valid ? (float)x + 0.5f : -1.0f, py = (float)y + 0.5f;  // px < 0: no pixel
  {
    float xmin = valid ? px : INFINITY, xmax = valid ? px : -INFINITY;
    float ymin = valid ? py : INFINITY, ymax = valid ? py : -INFINITY;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      xmin = fminf(xmin, __shfl_xor_sync(0xffffffffu, xmin, d));
      xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, d));
      ymin = fminf(ymin, __shfl_xor_sync(0xffffffffu, ymin, d));
      ymax = fmaxf(ymax, __shfl_xor_sync(0xffffffffu, ymax, d));
    }
    if (lane == 0) s_wbox[warp] = make_float4(xmin, xmax, ymin, ymax);
  }

  float t = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
  int walked = e1 - e0;
  bool done = !valid;
  uint32_t contrib = 0;
  const float W = (float)width;
  const uint32_t lt_mask = (1u << lane) - 1u;

  for (int base = e0; base < e1; base += kBlendThreads) {
    if (__syncthreads_count(!done) == 0) break;  // also orders s_wbox / previous batch
    const int e = base + tid;
    uint32_t mask = 0;
    if (e < e1) {
      const uint32_t v = vals[e];
      const uint32_t g = v >> 2;
      const int k = (int)(v & 3u);
      const float4 a = __ldg(sp_ab + 2 * (int64_t)g);
      const float4 b = __ldg(sp_ab + 2 * (int64_t)g + 1);
      const float c2 = __ldg(&sp_c[g].x);
      const float cx = a.x + (k == 0 ? -W : (k == 1 ? 0.0f : W));
      const float cy = a.y;
      s_ent[tid].geo = make_float4(cx, cy, a.z, 2.0f * a.w);
      s_ent[tid].att = make_float4(b.x, b.y, b.z, b.w);
      s_ent[tid].b.x = c2;
      float ex, ey;
      if (!cull_extents(a.z, a.w, b.x, cutoff2, &ex, &ey)) {
        mask = 0xFFu;
      } else if (tile_size == 16) {
        // The warp boxes form a 2 (x) x 4 (y) grid of blocks: test the entry against the
        // two column and four row intervals (6 tests instead of 8 box tests). Warp w is
        // column w & 1, row w >> 1; its box's x part equals its column's (warp w & 1),
        // its y part its row's (warp w & ~1): same comparisons, same mask.
        const float4 c0 = s_wbox[0], c1 = s_wbox[1];
        const bool in0 = !((c0.x - cx > ex) || (c0.y - cx < -ex));
        const bool in1 = !((c1.x - cx > ex) || (c1.y - cx < -ex));
        uint32_t rows = 0;
#pragma unroll
        for (int wy = 0; wy < 4; ++wy) {
          const float4 r = s_wbox[2 * wy];
          rows |= ((r.z - cy > ey) || (r.w - cy < -ey)) ? 0u : (1u << (2 * wy));
        }
        mask = (in0 ? rows : 0u) | (in1 ? rows << 1 : 0u);
      } else {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const float4 bx = s_wbox[w];
          const bool out = (bx.x - cx > ex) || (bx.y - cx < -ex) || (bx.z - cy > ey) || (bx.w - cy < -ey);
          mask |= out ? 0u : (1u << w);
        }
      }
    }
    s_mask[tid] = (uint8_t)mask;
    __syncthreads();
    // Compact this warp's entries (in order) into its list.
    int n_list = 0;
#pragma unroll
    for (int c = 0; c < kBlendThreads / 32; ++c) {
      const bool mine = (s_mask[c * 32 + lane] >> warp) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, mine);
      if (mine) s_list[warp][n_list + __popc(bal & lt_mask)] = (uint16_t)((c * 32 + lane) * sizeof(Staged));
      n_list += __popc(bal);
    }
    __syncwarp();
    if (!done) {
      const char* ent_base = reinterpret_cast<const char*>(s_ent);
      for (const uint16_t *lp = s_list[warp], *lend = s_list[warp] + n_list; lp != lend; ++lp) {
        const Staged& ent = *reinterpret_cast<const Staged*>(ent_base + *lp);
        const float4 geo = ent.geo;
        const float dx = px - geo.x;
        const float dy = py - geo.y;
        const float4 att = ent.att;
        const float d2 = geo.z * dx * dx + geo.w * dx * dy + att.x * dy * dy;
        if (d2 > cutoff2) continue;
        const float x = -d2 / 2.0f;
        const float G = kSmallCutoff ? pm_expf_blend_core(fminf(x, 88.0f)) : pm_expf_blend(x);
        // fminf == std::min here: the product is never NaN or -0 for a projected splat.
        const float alpha = fminf(alpha_clamp, att.y * G);
        const float t_next = t * (1.0f - alpha);
        if (t_next < transmittance_floor) {
          walked = base + (int)(*lp / sizeof(Staged)) - e0;
          done = true;
          break;
        }
        const float wgt = alpha * t;
        if (kCount) ++contrib;
        cr = cr + att.z * wgt;
        cg = cg + att.w * wgt;
        cb = cb + ent.b.x * wgt;
        t = t_next;
      }
    }
  }

  // The pixel again from its centre (exact: coordinates < 2^23), so x, y and the valid
  // flag need no registers across the walk.
  const bool valid_px = px >= 0.0f;
  if (kCount) {
    const uint32_t exam = valid_px ? (uint32_t)min(walked + 1, e1 - e0) : 0u;
    const uint32_t w_exam = __reduce_add_sync(0xffffffffu, exam);
    const uint32_t w_contrib = __reduce_add_sync(0xffffffffu, contrib);
    if (lane == 0) {
      atomicAdd(work, (unsigned long long)w_exam);
      atomicAdd(work + 1, (unsigned long long)w_contrib);
    }
  }
  if (valid_px) {
    const int64_t plane = (int64_t)width * height;
    const int64_t p = (int64_t)(int)px * height + (int)py;
    image[p] = cr;
    image[plane + p] = cg;
    image[2 * plane + p] = cb;
    trans_out[p] = t;
    walked_out[p] = walked;
    // Fused all-gather: the same pixel into every peer's image. Unrolled, so the peer
    // pointers are read from the parameter bank (a runtime index would copy the array
    // to local memory).
#pragma unroll
    for (int k = 0; k < kMaxPeers; ++k) {
      if (k >= peers.n) break;
      float* q = peers.ptr[k];
      q[p] = cr;
      q[plane + p] = cg;
      q[2 * plane + p] = cb;
    }
  }
}

void launch_blend(const BlendArgs& a, cudaStream_t stream) {
  const int n_band_tiles = a.tiles_x * (a.band_ty1 - a.band_ty0);
  if (n_band_tiles <= 0) return;
  if (!a.plain && a.tile_size <= 16) {
    const float cutoff2 = a.cutoff_sigma * a.cutoff_sigma;
    // Work counters (examined / composited entries) only when the frame asks for them.
    auto kern = cutoff2 <= 172.0f ? (a.work ? k_blend_cull<true, true> : k_blend_cull<true, false>)
                                  : (a.work ? k_blend_cull<false, true> : k_blend_cull<false, false>);
    launch_pdl(kern, n_band_tiles, kBlendThreads, 0, stream, a.offsets, a.vals, a.sp_ab, a.sp_c, a.width, a.height,
                                                      a.tile_size, a.tiles_x, a.alpha_clamp, a.transmittance_floor,
                                                      cutoff2, a.image, a.transmittance, a.walked, a.work,
                                                      a.band_ty0 * a.tiles_x, a.order, a.peers);
    ++g_launches;
    return;
  }
  launch_blend_plain(a, stream);
}

void launch_blend_plain(const BlendArgs& a, cudaStream_t stream) {
  const int n_tiles = a.tiles_x * (a.band_ty1 - a.band_ty0);
  if (n_tiles <= 0) return;
  const float cutoff2 = a.cutoff_sigma * a.cutoff_sigma;
  const int area = a.tile_size * a.tile_size;
#define ODGS_BLEND(PPT)                                                                                          \
  k_blend<PPT><<<n_tiles, kBlendThreads, 0, stream>>>(a.offsets, a.vals, a.sp_ab, a.sp_c, a.width, a.height,    \
                                                      a.tile_size, a.tiles_x, a.alpha_clamp,                    \
                                                      a.transmittance_floor, cutoff2, a.image, a.transmittance, \
                                                      a.walked, a.work, a.band_ty0 * a.tiles_x, a.peers)
  if (area <= kBlendThreads) ODGS_BLEND(1);
  else if (area <= 4 * kBlendThreads) ODGS_BLEND(4);
  else ODGS_BLEND(16);
#undef ODGS_BLEND
  ++g_launches;
}

// ------------------------------------------------------------------ cull (rasterizer.hpp:15-28)
__global__ void k_cull(int64_t n, const float* __restrict__ means, DevCamera cam, float near_r, float far_r,
                       uint8_t* __restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float p[3] = {means[i], means[n + i], means[2 * n + i]};
  float mu[3];
  to_camera(cam, p, mu);
  const float d = sqrtf(sum3(mu[0] * mu[0], mu[1] * mu[1], mu[2] * mu[2]));
  keep[i] = (d >= near_r && d <= far_r) ? 1 : 0;
}

void launch_cull(int64_t n, const float* means, DevCamera cam, float near_r, float far_r, uint8_t* keep,
                 cudaStream_t stream) {
  if (n == 0) return;
  k_cull<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(n, means, cam, near_r, far_r, keep);
  ++g_launches;
}

}  // namespace odgs_b200
