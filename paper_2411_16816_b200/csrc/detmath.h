// detmath.h — deterministic fp32 transcendentals shared by the sm_100a kernels
// and by the CPU oracle's fp32 instantiation.
//
// Why: BASELINE.json's north_star demands bit-exact tile lists, sorted keys and
// per-pixel contributor counts between the GPU path and the CPU oracle. Those
// integers are floor()/ceil()/threshold tests of values that went through
// exp / atan2 / asin (reference call sites: scene.hpp:194 `exp`, common.hpp:55-57
// `sigmoid`, projection.hpp:124 `atan2`/`asin`, SPEC.md:288 alpha). glibc's and
// CUDA's libm differ in the last ulp, so neither is used on the fp32 path:
// every function below is a fixed sequence of IEEE-754 binary32 add / mul / fma /
// div / sqrt operations, spelled with explicit round-to-nearest intrinsics on the
// device (never contracted, whatever --fmad says) and with plain operators on the
// host (the host build MUST use -ffp-contract=off; tests/test_detmath.py pins the
// bit patterns). Polynomials are the classic public-domain Cephes single-precision
// kernels (expf / atanf / asinf), accuracy <= 2 ulp, checked against libm in the
// CPU test-suite.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define DM_HD __host__ __device__ __forceinline__
#else
#define DM_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define DM_MUL(a, b) __fmul_rn((a), (b))
#define DM_ADD(a, b) __fadd_rn((a), (b))
#define DM_SUB(a, b) __fsub_rn((a), (b))
#define DM_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#define DM_DIV(a, b) __fdiv_rn((a), (b))
#define DM_SQRT(a) __fsqrt_rn((a))
#else
#define DM_MUL(a, b) ((a) * (b))
#define DM_ADD(a, b) ((a) + (b))
#define DM_SUB(a, b) ((a) - (b))
#define DM_FMA(a, b, c) __builtin_fmaf((a), (b), (c))
#define DM_DIV(a, b) ((a) / (b))
#define DM_SQRT(a) __builtin_sqrtf((a))
#endif

namespace detmath {

DM_HD float bits_to_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  std::memcpy(&f, &u, 4);
  return f;
#endif
}
DM_HD uint32_t float_to_bits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
#endif
}

DM_HD float fabs_(float x) { return bits_to_float(float_to_bits(x) & 0x7fffffffu); }

/// e^x. Cody-Waite reduction x = n ln2 + r, |r| <= ln2/2, degree-5 kernel,
/// result scaled by 2^n in two exact power-of-two multiplies. Inputs below
/// -87 flush to the smallest-normal neighbourhood (never denormal), inputs
/// above 88.7 return +inf. NaN propagates.
DM_HD float exp(float x) {
  if (!(x <= 88.72f)) return (x != x) ? x : bits_to_float(0x7f800000u);
  if (x < -87.0f) x = -87.0f;
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: add/sub rounds to nearest integer
  float n = DM_SUB(DM_ADD(DM_MUL(x, 1.44269504088896341f), kMagic), kMagic);
  float r = DM_FMA(n, -0.693359375f, x);        // ln2 high part (exact in 10 bits)
  r = DM_FMA(n, 2.12194440e-4f, r);             // minus ln2 low part
  float z = DM_MUL(r, r);
  float p = 1.9875691500e-4f;
  p = DM_FMA(p, r, 1.3981999507e-3f);
  p = DM_FMA(p, r, 8.3334519073e-3f);
  p = DM_FMA(p, r, 4.1665795894e-2f);
  p = DM_FMA(p, r, 1.6666665459e-1f);
  p = DM_FMA(p, r, 5.0000001201e-1f);
  p = DM_ADD(DM_FMA(p, z, r), 1.0f);
  int e = (int)n;            // in [-126, 128]
  int e1 = e >> 1;           // split so both factors are normal powers of two
  int e2 = e - e1;
  float s1 = bits_to_float((uint32_t)(e1 + 127) << 23);
  float s2 = bits_to_float((uint32_t)(e2 + 127) << 23);
  return DM_MUL(DM_MUL(p, s1), s2);
}

/// e^x for x <= 88 whose caller guarantees x >= -87 (the compositing kernels: x = -qf / 2 with qf <= qform_max).
/// Bit-identical to exp() on [-87, 88]: the same reduction and kernel; 2^n is then a normal number, so one exact
/// power-of-two multiply replaces the two-step scaling, the exponent comes from the low mantissa bits of the
/// magic-number sum instead of a float-to-int conversion, and both range branches go. Arguments above 88 (a
/// quadratic form below -176: not reachable with a positive-definite conic) evaluate as e^88, which the alpha clamp
/// treats like +inf.
DM_HD float exp_bounded(float x) {
  x = x < 88.0f ? x : 88.0f;
  const float kMagic = 12582912.0f;
  const float tmp = DM_ADD(DM_MUL(x, 1.44269504088896341f), kMagic);
  const float n = DM_SUB(tmp, kMagic);
  float r = DM_FMA(n, -0.693359375f, x);
  r = DM_FMA(n, 2.12194440e-4f, r);
  const float z = DM_MUL(r, r);
  float p = 1.9875691500e-4f;
  p = DM_FMA(p, r, 1.3981999507e-3f);
  p = DM_FMA(p, r, 8.3334519073e-3f);
  p = DM_FMA(p, r, 4.1665795894e-2f);
  p = DM_FMA(p, r, 1.6666665459e-1f);
  p = DM_FMA(p, r, 5.0000001201e-1f);
  p = DM_ADD(DM_FMA(p, z, r), 1.0f);
  const float s = bits_to_float((float_to_bits(tmp) << 23) + 0x3f800000u);  // 2^n, n in [-126, 127]
  return DM_MUL(p, s);
}

/// Numerically stable logistic, same branch structure as the reference
/// (common.hpp:54-58).
DM_HD float sigmoid(float x) {
  if (x >= 0.0f) return DM_DIV(1.0f, DM_ADD(1.0f, exp(-x)));
  float e = exp(x);
  return DM_DIV(e, DM_ADD(1.0f, e));
}

/// atan(t) for t >= 0 (t may be +inf). Cephes atanf reduction + degree-4 kernel in z = t^2.
DM_HD float atan_pos(float t) {
  float y0, x;
  if (t > 2.414213562373095f) {  // tan(3 pi / 8)
    y0 = 1.5707963267948966f;
    x = -DM_DIV(1.0f, t);
  } else if (t > 0.4142135623730950f) {  // tan(pi / 8)
    y0 = 0.7853981633974483f;
    x = DM_DIV(DM_SUB(t, 1.0f), DM_ADD(t, 1.0f));
  } else {
    y0 = 0.0f;
    x = t;
  }
  float z = DM_MUL(x, x);
  float p = 8.05374449538e-2f;
  p = DM_FMA(p, z, -1.38776856032e-1f);
  p = DM_FMA(p, z, 1.99777106478e-1f);
  p = DM_FMA(p, z, -3.33329491539e-1f);
  p = DM_FMA(DM_MUL(p, z), x, x);
  return DM_ADD(y0, p);
}

/// atan2(y, x) in (-pi, pi]; atan2(0, 0) = 0.
DM_HD float atan2(float y, float x) {
  float ax = fabs_(x), ay = fabs_(y);
  float r;
  if (ax == 0.0f && ay == 0.0f) {
    r = 0.0f;
  } else {
    r = atan_pos(DM_DIV(ay, ax));  // ay / 0 = +inf handled by the first branch
  }
  if (x < 0.0f) r = DM_SUB(3.14159265358979323846f, r);
  if (y < 0.0f) r = -r;
  return r;
}

/// asin(x), |x| <= 1 (values a hair above 1 clamp). Cephes asinf.
DM_HD float asin(float x) {
  float a = fabs_(x);
  if (a > 1.0f) a = 1.0f;
  float z, s;
  bool big = a > 0.5f;
  if (big) {
    z = DM_MUL(0.5f, DM_SUB(1.0f, a));
    s = DM_SQRT(z);
  } else {
    s = a;
    z = DM_MUL(a, a);
  }
  float p = 4.2163199048e-2f;
  p = DM_FMA(p, z, 2.4181311049e-2f);
  p = DM_FMA(p, z, 4.5470025998e-2f);
  p = DM_FMA(p, z, 7.4953002686e-2f);
  p = DM_FMA(p, z, 1.6666752422e-1f);
  p = DM_FMA(DM_MUL(p, z), s, s);
  if (big) p = DM_SUB(1.5707963267948966f, DM_ADD(p, p));
  return (x < 0.0f) ? -p : p;
}

}  // namespace detmath
