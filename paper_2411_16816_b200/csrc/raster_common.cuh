// raster_common.cuh — alpha evaluation shared by the forward and backward compositing kernels.
//
// SPEC.md:285-293 (Eq. 5/6): alpha = min(alpha_clamp, rho * exp(-qf/2)), rho = det_ratio * opacity,
// qf = d^T conic d with d = query - (mean2d + v t); skipped when qf > qform_max (projection.hpp:11)
// or alpha < alpha_min. Lidar azimuth differences are wrapped to (-pi, pi] (common.hpp:41-46).
//
// Written with explicit round-to-nearest intrinsics so that the forward and the backward kernels
// (which are compiled with different --fmad settings) and the CPU oracle take bit-identical skip
// decisions: contributor counts are a bit-exact parity gate, and the backward pass must revisit
// exactly the Gaussians the forward pass blended.
#pragma once

#include "splat_device.cuh"

namespace sb {

/// common.hpp:41-46. fmod is exact, so for |a| < 4 pi it is a compare + one exact subtraction.
__device__ __forceinline__ float wrap_pi(float a) {
  const float aa = fabsf(a);
  if (aa >= kTwoPi) {
    if (aa < 2.0f * kTwoPi) a = (a > 0.0f) ? __fsub_rn(a, kTwoPi) : __fadd_rn(a, kTwoPi);
    else a = fmodf(a, kTwoPi);
  }
  if (a > kPi) a = __fsub_rn(a, kTwoPi);
  if (a <= -kPi) a = __fadd_rn(a, kTwoPi);
  return a;
}

struct AlphaEval {
  float alpha, dx, dy, gauss;
  bool clamped;
};

template <bool kLidar>
__device__ __forceinline__ bool evaluate_alpha(const float4 gA /* mx my vx vy */, const float4 gB /* a b2 c rho */,
                                               float qx, float qy, float t, float qform_max, float alpha_clamp,
                                               float alpha_min, AlphaEval& o) {
  const float mx = __fmaf_rn(gA.z, t, gA.x);
  const float my = __fmaf_rn(gA.w, t, gA.y);
  float dx = __fsub_rn(qx, mx);
  if (kLidar) dx = wrap_pi(dx);
  const float dy = __fsub_rn(qy, my);
  const float qf = __fmaf_rn(gB.x, __fmul_rn(dx, dx), __fmaf_rn(gB.z, __fmul_rn(dy, dy), __fmul_rn(gB.y, __fmul_rn(dx, dy))));
  if (!(qf <= qform_max)) return false;
  const float gauss = detmath::exp(__fmul_rn(-0.5f, qf));
  float alpha = __fmul_rn(gB.w, gauss);
  const bool clamped = alpha > alpha_clamp;
  if (clamped) alpha = alpha_clamp;
  if (!(alpha >= alpha_min)) return false;
  o.alpha = alpha; o.dx = dx; o.dy = dy; o.gauss = gauss; o.clamped = clamped;
  return true;
}

}  // namespace sb
