// common.cuh — shared device code of the B200 ODGS rasterizer.
//
// Numerics contract: every translation unit of the rasterizer is compiled with
// --fmad=false (no contraction) and IEEE division/sqrt, and every operation below
// follows the reference's (and the oracle's) operation order, so a float render on
// the GPU is bit-identical to oracle::render<float, PortableMath>: splat records,
// instance order, tile CSR, walk lengths, transmittance and image.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "odgs_portable_math.h"

namespace odgs_b200 {
// Programmatic dependent launch (sm_90+): the kernel may be scheduled while its
// predecessor in the stream drains (hides the ~1.5 us launch gap between dependent
// kernels). Every kernel launched this way calls pdl_wait() first, before any global
// memory access, so its semantics equal a plain stream-ordered launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace odgs_b200

namespace odgs_b200 {

constexpr float kPiF = 3.14159274101257324f;  // std::numbers::pi_v<float>
constexpr uint32_t kCulledKey = 0xFFFFFFFFu;

// Per-call device error words. Each holds min over offenders of (index << 4 | code)
// so the lowest Gaussian index wins, as in the reference's serial loops.
//
// Two sections. The sticky words (errors, overflow) keep their first value across
// asynchronous operations until the host reads them at a check point; the counters are
// per render and reset by every render.
struct DevErrors {
  // -- sticky: reset only after the host has read them
  unsigned long long nonfinite;    // first_non_finite (rasterizer.hpp:134-136)
  unsigned long long project;      // project_gaussian throws (code 1 invalid_argument, 3 domain)
  unsigned long long bwd_domain;   // grad_position*/jacobian_omni_direct pole axis (backward.hpp:79-80)
  unsigned long long bwd_nonfinite;  // non-finite gradient (backward.hpp:440-446)
  unsigned long long overflow;     // max n_entries that exceeded the entry buffers' capacity, else 0
  // -- per-render counters
  unsigned long long n_entries;    // total tile entries K (written by the offsets scan)
  unsigned long long n_visible;    // projected splats (RenderOutput::splats.size())
  unsigned long long n_instances;  // seam instances (RenderOutput::instances.size())
  unsigned long long n_band;       // band renders: Gaussians with entries in the band
  unsigned long long n_precull;    // band renders: pre-cull survivors
  unsigned long long k_sort;       // tile entries sorted and binned: min(n_entries, capacity)
};
constexpr size_t kDevErrorsSticky = 5 * sizeof(unsigned long long);  // bytes of the sticky section
constexpr unsigned long long kNoError = ~0ull;

struct DevCamera {
  float R[3][3];
  float t[3];
  int width, height;
};

struct DevSettings {
  float near_radius, far_radius;
  int tile_size;
  float alpha_clamp, transmittance_floor, cutoff_sigma, lowpass_dilation, max_elevation;
  int band_ty0, band_ty1;  // tile rows [band_ty0, band_ty1) that get entries (row-band renders)
};

// Splat flags (sp_c.w as bits).
constexpr uint32_t kFlagVisible = 1u;
constexpr uint32_t kFlagClamped = 2u;
constexpr uint32_t kFlagShiftBase = 4u;  // bit (2 + k): instance for shift k in {-W, 0, +W} exists

// ------------------------------------------------------------------ small matrices
struct M2 { float a[2][2]; };
struct M3 { float a[3][3]; };
struct M23 { float a[2][3]; };

__host__ __device__ __forceinline__ float sum2(float a, float b) { return a + b; }
__host__ __device__ __forceinline__ float sum3(float a, float b, float c) { return a + (b + c); }
__host__ __device__ __forceinline__ float sum4(float a, float b, float c, float d) { return (a + b) + (c + d); }

// Lazy coefficient products with the halving sum order of the oracle (odgs_oracle.hpp mul()).
__device__ __forceinline__ M2 mul22(const M2& x, const M2& y) {
  M2 o;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) o.a[r][c] = sum2(x.a[r][0] * y.a[0][c], x.a[r][1] * y.a[1][c]);
  return o;
}
__device__ __forceinline__ M23 mul2_23(const M2& x, const M23& y) {
  M23 o;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) o.a[r][c] = sum2(x.a[r][0] * y.a[0][c], x.a[r][1] * y.a[1][c]);
  return o;
}
__device__ __forceinline__ M23 mul23_3(const M23& x, const M3& y) {
  M23 o;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      o.a[r][c] = sum3(x.a[r][0] * y.a[0][c], x.a[r][1] * y.a[1][c], x.a[r][2] * y.a[2][c]);
  return o;
}
__device__ __forceinline__ M3 mul33(const M3& x, const M3& y) {
  M3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      o.a[r][c] = sum3(x.a[r][0] * y.a[0][c], x.a[r][1] * y.a[1][c], x.a[r][2] * y.a[2][c]);
  return o;
}
// x * y^T for 2x3 x 2x3 -> 2x2.
__device__ __forceinline__ M2 mul23_32t(const M23& x, const M23& y) {
  M2 o;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c)
      o.a[r][c] = sum3(x.a[r][0] * y.a[c][0], x.a[r][1] * y.a[c][1], x.a[r][2] * y.a[c][2]);
  return o;
}
// m * m^T for 3x3.
__device__ __forceinline__ M3 mul33_t(const M3& m) {
  M3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      o.a[r][c] = sum3(m.a[r][0] * m.a[c][0], m.a[r][1] * m.a[c][1], m.a[r][2] * m.a[c][2]);
  return o;
}

// Eigen::Quaternion(w,x,y,z).toRotationMatrix() on a normalised quaternion (covariance.hpp:22).
__device__ __forceinline__ M3 quaternion_matrix(float w, float x, float y, float z) {
  const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
  const float twx = tx * w, twy = ty * w, twz = tz * w;
  const float txx = tx * x, txy = ty * x, txz = tz * x;
  const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r.a[0][0] = 1.0f - (tyy + tzz); r.a[0][1] = txy - twz;          r.a[0][2] = txz + twy;
  r.a[1][0] = txy + twz;          r.a[1][1] = 1.0f - (txx + tzz); r.a[1][2] = tyz - twx;
  r.a[2][0] = txz - twy;          r.a[2][1] = tyz + twx;          r.a[2][2] = 1.0f - (txx + tyy);
  return r;
}

__device__ __forceinline__ void to_camera(const DevCamera& cam, const float p[3], float mu[3]) {
  for (int r = 0; r < 3; ++r) mu[r] = sum3(cam.R[r][0] * p[0], cam.R[r][1] * p[1], cam.R[r][2] * p[2]) + cam.t[r];
}

// jacobian_omni_factored (projection.hpp:75-96) given the spherical angles and r.
__device__ __forceinline__ M23 jacobian_factored(float phi, float theta, float r, float W, float H,
                                                 float max_elevation, bool* clamped) {
  const bool clamp = fabsf(theta) > max_elevation;
  *clamped = clamp;
  float cp, sp, ct, st;
  pm_sincosf(phi, &sp, &cp);
  pm_sincosf(theta, &st, &ct);
  // pm_cosf is exactly even (sign-symmetric reduction and polynomials), so
  // cos(|theta|) == cos(theta) bit for bit (checked in oracle/ref_tests.cpp).
  const float sec = 1.0f / (clamp ? pm_cosf(max_elevation) : ct);
  M23 j_o;
  j_o.a[0][0] = 1.0f / r; j_o.a[0][1] = 0.0f; j_o.a[0][2] = 0.0f;
  j_o.a[1][0] = 0.0f; j_o.a[1][1] = 1.0f / r; j_o.a[1][2] = 0.0f;
  M2 q_o;
  q_o.a[0][0] = sec; q_o.a[0][1] = 0.0f; q_o.a[1][0] = 0.0f; q_o.a[1][1] = 1.0f;
  M2 s_o;
  s_o.a[0][0] = W / (2.0f * kPiF); s_o.a[0][1] = 0.0f; s_o.a[1][0] = 0.0f; s_o.a[1][1] = H / kPiF;
  M3 t_phi, t_theta;
  t_phi.a[0][0] = cp;   t_phi.a[0][1] = 0.0f; t_phi.a[0][2] = -sp;
  t_phi.a[1][0] = 0.0f; t_phi.a[1][1] = 1.0f; t_phi.a[1][2] = 0.0f;
  t_phi.a[2][0] = sp;   t_phi.a[2][1] = 0.0f; t_phi.a[2][2] = cp;
  t_theta.a[0][0] = 1.0f; t_theta.a[0][1] = 0.0f; t_theta.a[0][2] = 0.0f;
  t_theta.a[1][0] = 0.0f; t_theta.a[1][1] = ct;   t_theta.a[1][2] = st;
  t_theta.a[2][0] = 0.0f; t_theta.a[2][1] = -st;  t_theta.a[2][2] = ct;
  const M3 tmu = mul33(t_theta, t_phi);
  return mul23_3(mul2_23(mul22(s_o, q_o), j_o), tmu);
}

// Saturating floor-to-int (matches oracle::floor_to_int).
__device__ __forceinline__ int floor_to_int(float v) {
  float f = floorf(v);
  if (!(f >= -1073741824.0f)) f = -1073741824.0f;
  if (f > 1073741824.0f) f = 1073741824.0f;
  return (int)f;
}

// instance_box (rasterizer.hpp:107-122). Returns false if the clipped box is empty.
__device__ __forceinline__ bool instance_box(float mx, float my, float radius, float shift, int width, int height,
                                             int box[4]) {
  const float cx = mx + shift;
  const float cy = my;
  const int x0 = max(0, floor_to_int(cx - radius - 0.5f) + 1);
  const int x1 = min(width - 1, floor_to_int(cx + radius - 0.5f));
  const int y0 = max(0, floor_to_int(cy - radius - 0.5f) + 1);
  const int y1 = min(height - 1, floor_to_int(cy + radius - 0.5f));
  if (x0 > x1 || y0 > y1) return false;
  box[0] = x0; box[1] = x1; box[2] = y0; box[3] = y1;
  return true;
}

__device__ __forceinline__ float shift_of(int k, int width) {
  return k == 0 ? -(float)width : (k == 1 ? 0.0f : (float)width);
}

// x / d for 0 <= x < 2^32 / d (box coordinates: 0 <= x < image size), d >= 2, by a
// multiply-high with m = ceil(2^32 / d): x m / 2^32 = x / d + x e / 2^32 with
// 0 <= e < 1, and x / 2^32 < 1 / d keeps the floor exact. One integer division per
// thread (hoisted: d is a kernel argument) instead of one per coordinate.
__device__ __forceinline__ int div_tile(int x, int d) {
  if (d == 1) return x;
  const uint32_t m = 0xFFFFFFFFu / (uint32_t)d + 1u;
  return (int)__umulhi((uint32_t)x, m);
}

// Tile span of shift k of a splat (box / tile_size); false if no instance.
__device__ __forceinline__ bool instance_tiles(float mx, float my, float radius, int k, int width, int height,
                                               int tile_size, int span[4]) {
  int box[4];
  if (!instance_box(mx, my, radius, shift_of(k, width), width, height, box)) return false;
  for (int q = 0; q < 4; ++q) span[q] = div_tile(box[q], tile_size);
  return true;
}

// instance_tiles clipped to the tile rows of a row band; false if the instance has
// no tile inside the band (or does not exist).
__device__ __forceinline__ bool band_tiles(float mx, float my, float radius, int k, int width, int height,
                                           int tile_size, int band_ty0, int band_ty1, int span[4]) {
  if (!instance_tiles(mx, my, radius, k, width, height, tile_size, span)) return false;
  span[2] = max(span[2], band_ty0);
  span[3] = min(span[3], band_ty1 - 1);
  return span[2] <= span[3];
}

// Conservative half extents (ex, ey) of an entry's cutoff ellipse such that any pixel
// whose *computed* offset dx = fl(px - cx) satisfies |dx| > ex (or |dy| > ey) has a
// computed d2 > cutoff^2, so the reference loop would skip it (rasterizer.hpp:247).
//   exact:    min_dy Q(dx, dy) = dx^2 / Sigma00 with Sigma00 = i11 / det(conic);
//   rounding: |fl(d2) - Q| <= 4 eps (|t1|+|t2|+|t3|) <= 4 eps kappa Q with
//             kappa = (max(i00, i11) + |i01|) * (i00 + i11) / det(conic);
//   margin:   delta = 64 eps kappa covers that, and the rounding of det and Sigma00
//             (each <= 3 eps kappa); extents are inflated by (1 + 4 delta) in Q.
// Ill-conditioned entries (delta >= 0.25) are never culled.
// The reciprocal and square roots are the approximate MUFU ones (relative error a few
// 1e-7); the 2e-5 relative inflation of the extents covers them.
__device__ __forceinline__ bool cull_extents(float i00, float i01, float i11, float cutoff2, float* ex, float* ey) {
  const float det = i00 * i11 - i01 * i01;
  if (!(det > 0.0f) || !(i00 > 0.0f) || !(i11 > 0.0f)) return false;
  float rdet;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rdet) : "f"(det));
  const float kappa = (fmaxf(i00, i11) + fabsf(i01)) * (i00 + i11) * rdet;
  const float delta = 64.0f * 1.1920929e-7f * kappa;
  if (!(delta < 0.25f)) return false;
  const float f = cutoff2 * (1.0f + 4.0f * delta) * rdet;
  float sx, sy;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sx) : "f"(i11 * f));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sy) : "f"(i00 * f));
  *ex = sx * 1.00002f + 1e-4f;
  *ey = sy * 1.00002f + 1e-4f;
  return true;
}

// ------------------------------------------------------------------ SH colour (extension)
// Same basis, constants (double literals rounded to float, as the oracle's S(...))
// and operation order as oracle::sh_basis / sh_color.
__host__ __device__ __forceinline__ int sh_count(int degree) { return (degree + 1) * (degree + 1) - 1; }

__device__ __forceinline__ void sh_basis(int degree, float x, float y, float z, float Y[15]) {
  const float C1 = (float)0.4886025119029199;
  Y[0] = -C1 * y;
  Y[1] = C1 * z;
  Y[2] = -C1 * x;
  if (degree < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[3] = (float)1.0925484305920792 * xy;
  Y[4] = (float)-1.0925484305920792 * yz;
  Y[5] = (float)0.31539156525252005 * (2.0f * zz - xx - yy);
  Y[6] = (float)-1.0925484305920792 * xz;
  Y[7] = (float)0.5462742152960396 * (xx - yy);
  if (degree < 3) return;
  Y[8] = (float)-0.5900435899266435 * y * (3.0f * xx - yy);
  Y[9] = (float)2.890611442640554 * xy * z;
  Y[10] = (float)-0.4570457994644658 * y * (4.0f * zz - xx - yy);
  Y[11] = (float)0.3731763325901154 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  Y[12] = (float)-0.4570457994644658 * x * (4.0f * zz - xx - yy);
  Y[13] = (float)1.445305721320277 * z * (xx - yy);
  Y[14] = (float)-0.5900435899266435 * x * (xx - 3.0f * yy);
}

__device__ __forceinline__ void sh_basis_grad(int degree, float x, float y, float z, float dY[15][3]) {
  const float C1 = (float)0.4886025119029199;
  dY[0][0] = 0.0f; dY[0][1] = -C1; dY[0][2] = 0.0f;
  dY[1][0] = 0.0f; dY[1][1] = 0.0f; dY[1][2] = C1;
  dY[2][0] = -C1; dY[2][1] = 0.0f; dY[2][2] = 0.0f;
  if (degree < 2) return;
  const float C2[5] = {(float)1.0925484305920792, (float)-1.0925484305920792, (float)0.31539156525252005,
                       (float)-1.0925484305920792, (float)0.5462742152960396};
  const float xx = x * x, yy = y * y, zz = z * z;
  dY[3][0] = C2[0] * y; dY[3][1] = C2[0] * x; dY[3][2] = 0.0f;
  dY[4][0] = 0.0f; dY[4][1] = C2[1] * z; dY[4][2] = C2[1] * y;
  dY[5][0] = -2.0f * C2[2] * x; dY[5][1] = -2.0f * C2[2] * y; dY[5][2] = 4.0f * C2[2] * z;
  dY[6][0] = C2[3] * z; dY[6][1] = 0.0f; dY[6][2] = C2[3] * x;
  dY[7][0] = 2.0f * C2[4] * x; dY[7][1] = -2.0f * C2[4] * y; dY[7][2] = 0.0f;
  if (degree < 3) return;
  const float C3[7] = {(float)-0.5900435899266435, (float)2.890611442640554, (float)-0.4570457994644658,
                       (float)0.3731763325901154, (float)-0.4570457994644658, (float)1.445305721320277,
                       (float)-0.5900435899266435};
  dY[8][0] = 6.0f * C3[0] * x * y; dY[8][1] = C3[0] * (3.0f * xx - 3.0f * yy); dY[8][2] = 0.0f;
  dY[9][0] = C3[1] * y * z; dY[9][1] = C3[1] * x * z; dY[9][2] = C3[1] * x * y;
  dY[10][0] = -2.0f * C3[2] * x * y; dY[10][1] = C3[2] * (4.0f * zz - xx - 3.0f * yy); dY[10][2] = 8.0f * C3[2] * y * z;
  dY[11][0] = -6.0f * C3[3] * x * z; dY[11][1] = -6.0f * C3[3] * y * z;
  dY[11][2] = C3[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy);
  dY[12][0] = C3[4] * (4.0f * zz - 3.0f * xx - yy); dY[12][1] = -2.0f * C3[4] * x * y; dY[12][2] = 8.0f * C3[4] * x * z;
  dY[13][0] = 2.0f * C3[5] * x * z; dY[13][1] = -2.0f * C3[5] * y * z; dY[13][2] = C3[5] * (xx - yy);
  dY[14][0] = C3[6] * (3.0f * xx - 3.0f * yy); dY[14][1] = -6.0f * C3[6] * x * y; dY[14][2] = 0.0f;
}

// World-space unit view direction from the camera centre -R^T t to p (oracle::sh_direction).
__device__ __forceinline__ float sh_direction(const DevCamera& cam, const float p[3], float d[3]) {
  float v[3];
  for (int k = 0; k < 3; ++k) {
    const float cc = -sum3(cam.R[0][k] * cam.t[0], cam.R[1][k] * cam.t[1], cam.R[2][k] * cam.t[2]);
    v[k] = p[k] - cc;
  }
  const float len = sqrtf(sum3(v[0] * v[0], v[1] * v[1], v[2] * v[2]));
  for (int k = 0; k < 3; ++k) d[k] = len > 0.0f ? v[k] / len : 0.0f;
  return len;
}

__device__ __forceinline__ void atomic_min_error(unsigned long long* word, long long index, int code) {
  atomicMin(word, ((unsigned long long)index << 4) | (unsigned long long)code);
}

__device__ __forceinline__ float std_min(float a, float b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ float std_max(float a, float b) { return (a < b) ? b : a; }  // std::max

}  // namespace odgs_b200
