/*
 * odgs_portable_math.h — bit-reproducible transcendental functions shared by the
 * sm_100a kernels and the CPU oracle's `PortableMath` policy.
 *
 * Why this exists. The reference rasterizer calls libm `std::atan2`, `std::hypot`,
 * `std::sin`, `std::cos` and `std::exp` on float on the path to pixel means, radii
 * and per-pixel alphas (reference proj/include/odgs/projection.hpp:25-27,45-46,84-85,
 * covariance.hpp:35, types.hpp:30, rasterizer.hpp:249). Tile membership, tile ranges
 * and the per-pixel walk length depend on those bits, and CUDA's libdevice and
 * glibc round differently in the last place. Every function below is therefore built
 * only from IEEE-754 correctly rounded operations (+, -, *, /, sqrt, fma, integer
 * bit manipulation), so the host and the device produce the SAME bits.
 *
 * Precision:
 *   pm_expf, pm_sinf, pm_cosf, pm_atan2f, pm_hypotf evaluate in binary64 and round
 *   once to binary32: nearly always the correctly rounded float result (they agree
 *   with glibc's float functions except in rare last-place cases).
 *   pm_expf_blend evaluates in binary32 (degree-6 Horner), <= ~1 ulp, and is the
 *   per-pixel exponential of the blend and backward loops, where throughput matters.
 *
 * Build rules (both sides): no floating-point contraction — the host oracle is
 * compiled with -ffp-contract=off; on the device every operation here is an explicit
 * round-to-nearest intrinsic (__dmul_rn, __fadd_rn, ...) or an explicit fma, which
 * nvcc never re-associates or contracts. Round-to-nearest-even mode is assumed.
 */
#ifndef ODGS_PORTABLE_MATH_H
#define ODGS_PORTABLE_MATH_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PM_HD __host__ __device__ __forceinline__
#else
#define PM_HD static inline
#endif

/* Polynomial coefficient tables: on the device in constant memory, so each DFMA takes
   its coefficient as a constant-bank operand (64-bit immediates otherwise cost two
   uniform moves per coefficient); on the host a static array. Same values, same
   evaluation order on both sides. */
#if defined(__CUDACC__)
#define PM_TABLE(name, n, ...)                                   \
  static __constant__ double name##_dev[n] = {__VA_ARGS__};      \
  static const double name##_host[n] = {__VA_ARGS__};
#else
#define PM_TABLE(name, n, ...) static const double name##_host[n] = {__VA_ARGS__};
#endif
#if defined(__CUDA_ARCH__)
#define PM_COEF(name, k) (name##_dev[k])
#define PM_UNROLL _Pragma("unroll")
#else
#define PM_COEF(name, k) (name##_host[k])
#define PM_UNROLL
#endif

/* ---------------------------------------------------------------- primitives */

PM_HD double pm_dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
PM_HD double pm_dsub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
PM_HD double pm_dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
PM_HD double pm_ddiv(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
PM_HD double pm_dsqrt(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  return sqrt(a);
#endif
}
PM_HD double pm_dfma(double a, double b, double c) { return fma(a, b, c); }

PM_HD float pm_fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
PM_HD float pm_fsub(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fsub_rn(a, b);
#else
  return a - b;
#endif
}
PM_HD float pm_fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
PM_HD float pm_ffma(float a, float b, float c) { return fmaf(a, b, c); }

PM_HD float pm_d2f(double x) {
#if defined(__CUDA_ARCH__)
  return __double2float_rn(x);
#else
  return (float)x;
#endif
}

/* 2^k as a binary64, -1022 <= k <= 1023. */
PM_HD double pm_pow2i_d(int k) {
  const uint64_t bits = (uint64_t)(int64_t)(k + 1023) << 52;
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)bits);
#else
  double d;
  memcpy(&d, &bits, sizeof d);
  return d;
#endif
}

/* 2^k as a binary32, -126 <= k <= 127. */
PM_HD float pm_pow2i_f(int k) {
  const uint32_t bits = (uint32_t)(k + 127) << 23;
#if defined(__CUDA_ARCH__)
  return __uint_as_float(bits);
#else
  float f;
  memcpy(&f, &bits, sizeof f);
  return f;
#endif
}

PM_HD int pm_isnan_d(double x) { return x != x; }
PM_HD int pm_isinf_d(double x) { return x == x && (x - x) != (x - x); }

/* Round-to-nearest-even integer of |x| < 2^51, via the 1.5*2^52 shifter. */
PM_HD double pm_rint_d(double x) {
  const double shifter = 0x1.8p52;
  return pm_dsub(pm_dadd(x, shifter), shifter);
}

/* ---------------------------------------------------------------- exp */

/* e^x in binary64 for -745 < x < 709 (only used on float-derived arguments). */
PM_TABLE(pm_exp_tab, 14, 0x1.6124613a86d09p-33, 0x1.1eed8eff8d898p-29, 0x1.ae64567f544e4p-26, 0x1.27e4fb7789f5cp-22, 0x1.71de3a556c734p-19, 0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-13, 0x1.6c16c16c16c17p-10, 0x1.1111111111111p-7, 0x1.5555555555555p-5, 0x1.5555555555555p-3, 0x1.0p-1, 0x1.0p+0, 0x1.0p+0)

PM_HD double pm_exp_core_d(double x) {
  const double inv_ln2 = 0x1.71547652b82fep+0;
  const double ln2_hi = 0x1.62e42fefa39efp-1;
  const double ln2_lo = 0x1.abc9e3b39803fp-56;
  const double kd = pm_rint_d(pm_dmul(x, inv_ln2));
  double r = pm_dfma(-kd, ln2_hi, x);
  r = pm_dfma(-kd, ln2_lo, r);
  /* Taylor to degree 13 on |r| <= 0.347: truncation < 5e-18 relative. */
  double p = PM_COEF(pm_exp_tab, 0);
  PM_UNROLL
  for (int k_ = 1; k_ < 14; ++k_) p = pm_dfma(p, r, PM_COEF(pm_exp_tab, k_));
  return pm_dmul(p, pm_pow2i_d((int)kd));
}

/* expf(x), binary64 evaluation rounded once. */
PM_HD float pm_expf(float x) {
  if (x != x) return x;
  if (x < -104.0f) return 0.0f;          /* true value < half the least subnormal */
  if (x > 89.0f) return INFINITY;        /* true value > FLT_MAX */
  return pm_d2f(pm_exp_core_d((double)x));
}

/*
 * expf(x) in binary32 for the per-pixel loops (argument -d2/2 <= 0): n = rint(x/ln2)
 * via the 1.5*2^23 shifter, Cody-Waite reduction, a degree-6 near-minimax polynomial
 * on |r| <= ln2/2 (relative error 1.9e-9), and the scaling 2^n applied by adding n to
 * the exponent field (exact: for -86 <= x <= 88 the result is a normal float).
 * Results below e^-86 (x < -86) are flushed to +0 — the alpha they would produce is
 * < 1e-37 and can change neither the transmittance nor the colour. Arguments above 88
 * are evaluated at 88 (e^88 = 1.65e38): x = -d2/2 > 88 needs d2 < -176, which a
 * positive-definite form reaches only through rounding at |d| > ~8000 px, and the alpha
 * clamps there either way unless the opacity is below 6e-39.
 *
 * pm_expf_blend_core is the evaluation alone, valid for -86 <= x <= 88; pm_expf_blend
 * adds the special cases.
 */
PM_HD float pm_expf_blend_core(float x) {
  const float shifter = 12582912.0f; /* 1.5 * 2^23 */
  const float t = pm_ffma(x, 0x1.715476p+0f, shifter);
  const float n = pm_fsub(t, shifter);
  float r = pm_ffma(n, -0x1.62e400p-1f, x); /* n * ln2_hi is exact for |n| < 2^8 */
  r = pm_ffma(n, -0x1.7f7d1cp-20f, r);
  float p = 0x1.6ac294p-10f;
  p = pm_ffma(p, r, 0x1.126e46p-7f);
  p = pm_ffma(p, r, 0x1.55589p-5f);
  p = pm_ffma(p, r, 0x1.555408p-3f);
  p = pm_ffma(p, r, 0x1.fffffap-2f);
  p = pm_ffma(p, r, 0x1.0p+0f);
  p = pm_ffma(p, r, 0x1.0p+0f);
#if defined(__CUDA_ARCH__)
  const int32_t ni = __float_as_int(t) - __float_as_int(shifter);
  return __int_as_float(__float_as_int(p) + (int32_t)((uint32_t)ni << 23));
#else
  int32_t tb, sb, pb;
  memcpy(&tb, &t, 4);
  memcpy(&sb, &shifter, 4);
  memcpy(&pb, &p, 4);
  const int32_t ni = tb - sb;
  const int32_t rb = pb + (int32_t)((uint32_t)ni << 23);
  float res;
  memcpy(&res, &rb, 4);
  return res;
#endif
}

PM_HD float pm_expf_blend(float x) {
  if (!(x >= -86.0f)) return (x != x) ? x : 0.0f;
  return pm_expf_blend_core(fminf(x, 88.0f));
}

/* ---------------------------------------------------------------- sin / cos */

/* Reduces x to r in [-pi/4, pi/4] and the quadrant q = k mod 4 (|x| < 2^40). */
PM_HD double pm_reduce_pio2(double x, int* q) {
  const double two_over_pi = 0x1.45f306dc9c883p-1;
  const double p1 = 0x1.921fb54442d18p+0;
  const double p2 = 0x1.1a62633145c07p-54;
  const double p3 = -0x1.f1976b7ed8fbcp-110;
  const double kd = pm_rint_d(pm_dmul(x, two_over_pi));
  double r = pm_dfma(-kd, p1, x);
  r = pm_dfma(-kd, p2, r);
  r = pm_dfma(-kd, p3, r);
  *q = (int)((int64_t)kd & 3);
  return r;
}

PM_TABLE(pm_sin_tab, 8, 0x1.952c77030ad4ap-49, -0x1.ae7f3e733b81fp-41, 0x1.6124613a86d09p-33, -0x1.ae64567f544e4p-26, 0x1.71de3a556c734p-19, -0x1.a01a01a01a01ap-13, 0x1.1111111111111p-7, -0x1.5555555555555p-3)

PM_HD double pm_sin_poly(double r) {
  const double s = pm_dmul(r, r);
  double p = PM_COEF(pm_sin_tab, 0);
  PM_UNROLL
  for (int k_ = 1; k_ < 8; ++k_) p = pm_dfma(p, s, PM_COEF(pm_sin_tab, k_));
  return pm_dfma(pm_dmul(r, s), p, r);
}

PM_TABLE(pm_cos_tab, 9, -0x1.6827863b97d97p-53, 0x1.ae7f3e733b81fp-45, -0x1.93974a8c07c9dp-37, 0x1.1eed8eff8d898p-29, -0x1.27e4fb7789f5cp-22, 0x1.a01a01a01a01ap-16, -0x1.6c16c16c16c17p-10, 0x1.5555555555555p-5, -0x1.0p-1)

PM_HD double pm_cos_poly(double r) {
  const double s = pm_dmul(r, r);
  double p = PM_COEF(pm_cos_tab, 0);
  PM_UNROLL
  for (int k_ = 1; k_ < 9; ++k_) p = pm_dfma(p, s, PM_COEF(pm_cos_tab, k_));
  return pm_dfma(s, p, 1.0);
}

PM_HD float pm_sinf(float x) {
  if (x != x || x - x != 0.0f) return x - x; /* NaN for NaN and +-inf */
  int q;
  const double r = pm_reduce_pio2((double)x, &q);
  double v;
  switch (q) {
    case 0: v = pm_sin_poly(r); break;
    case 1: v = pm_cos_poly(r); break;
    case 2: v = -pm_sin_poly(r); break;
    default: v = -pm_cos_poly(r); break;
  }
  return pm_d2f(v);
}

PM_HD float pm_cosf(float x) {
  if (x != x || x - x != 0.0f) return x - x;
  int q;
  const double r = pm_reduce_pio2((double)x, &q);
  double v;
  switch (q) {
    case 0: v = pm_cos_poly(r); break;
    case 1: v = -pm_sin_poly(r); break;
    case 2: v = -pm_cos_poly(r); break;
    default: v = pm_sin_poly(r); break;
  }
  return pm_d2f(v);
}

/* sin and cos of the same argument with one range reduction; bit-identical to
   pm_sinf(x) and pm_cosf(x). */
PM_HD void pm_sincosf(float x, float* s, float* c) {
  if (x != x || x - x != 0.0f) {
    *s = x - x;
    *c = x - x;
    return;
  }
  int q;
  const double r = pm_reduce_pio2((double)x, &q);
  const double sp = pm_sin_poly(r), cp = pm_cos_poly(r);
  double vs, vc;
  switch (q) {
    case 0: vs = sp; vc = cp; break;
    case 1: vs = cp; vc = -sp; break;
    case 2: vs = -sp; vc = -cp; break;
    default: vs = -cp; vc = sp; break;
  }
  *s = pm_d2f(vs);
  *c = pm_d2f(vc);
}

/* ---------------------------------------------------------------- atan2 / hypot */

/* atan(t) for 0 <= t <= 1 in binary64. */
PM_TABLE(pm_atan_tab, 22, 0x1.6c16c16c16c17p-6, -0x1.7d05f417d05f4p-6, 0x1.8f9c18f9c18fap-6, -0x1.a41a41a41a41ap-6, 0x1.bacf914c1bad0p-6, -0x1.d41d41d41d41dp-6, 0x1.f07c1f07c1f08p-6, -0x1.0842108421084p-5, 0x1.1a7b9611a7b96p-5, -0x1.2f684bda12f68p-5, 0x1.47ae147ae147bp-5, -0x1.642c8590b2164p-5, 0x1.8618618618618p-5, -0x1.af286bca1af28p-5, 0x1.e1e1e1e1e1e1ep-5, -0x1.1111111111111p-4, 0x1.3b13b13b13b14p-4, -0x1.745d1745d1746p-4, 0x1.c71c71c71c71cp-4, -0x1.2492492492492p-3, 0x1.999999999999ap-3, -0x1.5555555555555p-2)

PM_HD double pm_atan_unit_d(double t) {
  const double tan_pi_8 = 0x1.a827999fcef32p-2;
  const double pi_4 = 0x1.921fb54442d18p-1;
  double base = 0.0, u = t;
  if (t > tan_pi_8) {
    u = pm_ddiv(pm_dsub(t, 1.0), pm_dadd(t, 1.0));
    base = pi_4;
  }
  /* Taylor in s = u^2 to u^45 on |u| <= tan(pi/8): truncation < 2e-19. */
  const double s = pm_dmul(u, u);
  double p = PM_COEF(pm_atan_tab, 0);
  PM_UNROLL
  for (int k_ = 1; k_ < 22; ++k_) p = pm_dfma(p, s, PM_COEF(pm_atan_tab, k_));
  return pm_dadd(base, pm_dfma(pm_dmul(u, s), p, u));
}

/* atan2f(y, x) with the C99 special-value conventions. */
PM_HD float pm_atan2f(float y, float x) {
  const double pi = 0x1.921fb54442d18p+1;
  const double pi_2 = 0x1.921fb54442d18p+0;
  const double pi_4 = 0x1.921fb54442d18p-1;
  if (x != x || y != y) return x + y;
  const int y_neg = signbit(y) != 0;
  const int x_neg = signbit(x) != 0;
  const double ax = fabs((double)x), ay = fabs((double)y);
  double a;
  if (ay == 0.0) {
    a = x_neg ? pi : 0.0;
  } else if (ax == 0.0) {
    a = pi_2;
  } else if (pm_isinf_d(ax) || pm_isinf_d(ay)) {
    if (pm_isinf_d(ax) && pm_isinf_d(ay))
      a = x_neg ? 3.0 * pi_4 : pi_4;
    else if (pm_isinf_d(ax))
      a = x_neg ? pi : 0.0;
    else
      a = pi_2;
  } else {
    if (ay <= ax)
      a = pm_atan_unit_d(pm_ddiv(ay, ax));
    else
      a = pm_dsub(pi_2, pm_atan_unit_d(pm_ddiv(ax, ay)));
    if (x_neg) a = pm_dsub(pi, a);
  }
  const float f = pm_d2f(a);
  return y_neg ? -f : f;
}

/* hypotf(x, y) as glibc computes it: sqrt(x*x + y*y) in binary64, rounded once. */
PM_HD float pm_hypotf(float x, float y) {
  const double ax = fabs((double)x), ay = fabs((double)y);
  if (pm_isinf_d(ax) || pm_isinf_d(ay)) return INFINITY;
  if (ax != ax || ay != ay) return x + y;
  return pm_d2f(pm_dsqrt(pm_dadd(pm_dmul(ax, ax), pm_dmul(ay, ay))));
}

/* ---------------------------------------------------------------- log */

/*
 * ln(x) for binary32 x, evaluated in binary64 and rounded once (logit, types.hpp:38,
 * and the split shrink log(1.6), densify.hpp:123). x = m 2^e with m in
 * [sqrt(1/2), sqrt(2)); ln m = 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, summed
 * to s^23 (truncation < 1e-19 relative); e ln2 in a hi/lo split.
 */
PM_HD float pm_logf(float x) {
  if (x != x || x < 0.0f) return NAN;
  if (x == 0.0f) return -INFINITY;
  if (x == INFINITY) return x;
  const double d = (double)x; /* exact; subnormal floats are normal doubles */
  uint64_t bits;
#if defined(__CUDA_ARCH__)
  bits = (uint64_t)__double_as_longlong(d);
#else
  memcpy(&bits, &d, sizeof bits);
#endif
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  uint64_t mb = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull; /* m in [1, 2) */
  if (mb > 0x3ff6a09e667f3bcdull) { /* m > sqrt(2): halve it (exact) */
    mb -= 0x0010000000000000ull;
    e += 1;
  }
  double m;
#if defined(__CUDA_ARCH__)
  m = __longlong_as_double((long long)mb);
#else
  memcpy(&m, &mb, sizeof m);
#endif
  const double s = pm_ddiv(pm_dsub(m, 1.0), pm_dadd(m, 1.0));
  const double z = pm_dmul(s, s);
  double p = 1.0 / 23.0;
  p = pm_dfma(p, z, 1.0 / 21.0);
  p = pm_dfma(p, z, 1.0 / 19.0);
  p = pm_dfma(p, z, 1.0 / 17.0);
  p = pm_dfma(p, z, 1.0 / 15.0);
  p = pm_dfma(p, z, 1.0 / 13.0);
  p = pm_dfma(p, z, 1.0 / 11.0);
  p = pm_dfma(p, z, 1.0 / 9.0);
  p = pm_dfma(p, z, 1.0 / 7.0);
  p = pm_dfma(p, z, 1.0 / 5.0);
  p = pm_dfma(p, z, 1.0 / 3.0);
  const double lm = pm_dmul(pm_dmul(2.0, s), pm_dfma(p, z, 1.0)); /* 2s (1 + z p) */
  const double ln2_hi = 0x1.62e42fefa39efp-1, ln2_lo = 0x1.abc9e3b39803fp-56;
  const double ed = (double)e;
  return pm_d2f(pm_dfma(ed, ln2_hi, pm_dfma(ed, ln2_lo, lm)));
}

#endif /* ODGS_PORTABLE_MATH_H */
