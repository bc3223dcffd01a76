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

// L2 prefetch of a record the NEXT batch will stage: turns its DRAM round trip into an L2 hit (the compositing kernels
// are latency-bound: a batch is a chain of dependent global loads — list entry, record — in front of the compute)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ------------------------------------------------------------------------------------------------
// Shared-memory accesses by 32-bit window address. nvcc forms the address of a __shared__ array as
// (SR_CgaCtaId << 24) + offset (S2R + MOV + LEA) and, in the register-capped compositing loops, re-materialises it on
// every iteration instead of keeping it in a register: 6 of the ~33 instructions the camera forward spends per
// evaluated list entry. One base address is therefore pinned in a register (an opaque mov) and every array of the loop is
// addressed relative to it (the differences between the arrays' addresses are compile-time constants).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// the same address as an opaque register value: the compiler cannot re-derive it, so it stays in a register across a loop
__device__ __forceinline__ uint32_t smem_addr_pinned(const void* p) {
  uint32_t a = smem_addr(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

// ------------------------------------------------------------------------------------------------
// Packed fp32 pairs (sm_100a: FFMA2 / FMUL2 / FADD2 execute two IEEE-754 round-to-nearest operations per issue slot;
// each half is bit-identical to the scalar __f*_rn operation, so the parity contract is untouched). The compositing
// kernels are issue-bound, not FMA-pipe-bound: halving the fp32 instruction count of the inner loops is the point.
// ------------------------------------------------------------------------------------------------
typedef unsigned long long f32x2;  // .x in the low half
__device__ __forceinline__ f32x2 pack2(float x, float y) { f32x2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ void unpack2(f32x2 v, float& x, float& y) { asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v)); }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) { f32x2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) { f32x2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) { f32x2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) { f32x2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }

// alpha_qform without the azimuth wrap, on packed pairs: the same operations in the same order as the scalar form
// (mx my = fma(v, t, m); d = q - m; qf = fma(a, dx dx, fma(c, dy dy, b2 (dx dy)))), 7 issue slots instead of 10.
// m0 = (mean2d.x, mean2d.y), v = (vel.x, vel.y), q = (qx, qy), tt = (t, t).
__device__ __forceinline__ float alpha_qform_packed(f32x2 m0, f32x2 v, const float4 gB, f32x2 q, f32x2 tt, float& dx, float& dy) {
  const f32x2 d = sub2(q, fma2(v, tt, m0));
  const f32x2 dd = mul2(d, d);
  unpack2(d, dx, dy);
  float dxx, dyy;
  unpack2(dd, dxx, dyy);
  return __fmaf_rn(gB.x, dxx, __fmaf_rn(gB.z, dyy, __fmul_rn(gB.y, __fmul_rn(dx, dy))));
}

// 32 x 32 bit-matrix transpose across the warp: lane l passes row l, receives column l.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? (((y & ~m) >> s) | (x & ~m)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

struct AlphaEval {
  float alpha, dx, dy, gauss;
  bool clamped;
};

// Step 1 of evaluate_alpha: the offsets and the quadratic form (branch-free apart from the lidar wrap), so that two
// list entries can be evaluated side by side for instruction-level parallelism.
// `wrap` (lidar only, warp-uniform): false when the staging pass has certified |qx - mx| < pi for every query of the warp
// and every entry of the batch, so that wrap_pi would return its argument unchanged (see patch_mask).
template <bool kLidar>
__device__ __forceinline__ float alpha_qform(const float4 gA /* mx my vx vy */, const float4 gB /* a b2 c rho */, float qx,
                                             float qy, float t, float& dx, float& dy, bool wrap = true) {
  const float mx = __fmaf_rn(gA.z, t, gA.x);
  const float my = __fmaf_rn(gA.w, t, gA.y);
  dx = __fsub_rn(qx, mx);
  if (kLidar && wrap) dx = wrap_pi(dx);
  dy = __fsub_rn(qy, my);
  return __fmaf_rn(gB.x, __fmul_rn(dx, dx), __fmaf_rn(gB.z, __fmul_rn(dy, dy), __fmul_rn(gB.y, __fmul_rn(dx, dy))));
}

// Step 2: thresholds, exp, clamp. Returns false if the pair is skipped.
__device__ __forceinline__ bool alpha_finish(float qf, float rho, float dx, float dy, float qform_max, float alpha_clamp,
                                             float alpha_min, AlphaEval& o) {
  if (!(qf <= qform_max)) return false;
  // exp_bounded == detmath::exp on [-87, 88] (bit-identical, tests/test_oracle_kat.py). qf <= qform_max bounds the
  // argument from below; a numerically non-PSD conic can make qf hugely negative, so the argument is clamped at 88 from
  // above: there exp() is 1.65e38 (or inf beyond), rho * gauss exceeds alpha_clamp either way and the pair is blended
  // with the clamped alpha exactly as the oracle does (tests: test_near_singular_conics)
  const float gauss = detmath::exp_bounded(fminf(__fmul_rn(-0.5f, qf), 88.0f));
  float alpha = __fmul_rn(rho, gauss);
  const bool clamped = alpha > alpha_clamp;
  if (clamped) alpha = alpha_clamp;
  if (!(alpha >= alpha_min)) return false;
  o.alpha = alpha; o.dx = dx; o.dy = dy; o.gauss = gauss; o.clamped = clamped;
  return true;
}

template <bool kLidar>
__device__ __forceinline__ bool evaluate_alpha(const float4 gA /* mx my vx vy */, const float4 gB /* a b2 c rho */,
                                               float qx, float qy, float t, float qform_max, float alpha_clamp,
                                               float alpha_min, AlphaEval& o) {
  float dx, dy;
  const float qf = alpha_qform<kLidar>(gA, gB, qx, qy, t, dx, dy);
  return alpha_finish(qf, gB.w, dx, dy, qform_max, alpha_clamp, alpha_min, o);
}

// ------------------------------------------------------------------------------------------------
// Per-warp conservative culling (shared by the forward and backward compositing kernels).
//
// A CTA owns a tile; each of its 8 warps owns a compact PATCH of 32 queries (camera: 8x4 pixels; lidar:
// 32 rays consecutive in the per-tile azimuth-major order prepared at view creation, i.e. 4 azimuth
// bins x 8 beams on a grid sweep). When a batch of 256 Gaussians is staged, the staging thread tests its
// Gaussian against the 8 patch boxes and publishes an 8-bit mask; every warp then compacts the batch to
// the entries whose bit is set (order preserved) and walks only those.
//
// The test must NEVER drop a pair the exact per-query fp32 evaluation would blend, because contributor
// counts are a bit-exact parity gate. It is therefore a rigorous bound, not a heuristic:
//   * the set of fp32-computed offsets d = q - (m + v t) over the patch is enclosed in a box with centre
//     dc and half-extents H that include the rolling-shutter travel and the rounding of m + v t and q - m;
//   * the fp32 evaluation of Q differs from the exact one by at most ~4 ulp of the sum of term magnitudes
//     M <= a DX^2 + c DY^2 + |b2| DX DY; a margin of 2^-18 M (64 ulp) covers that, the cull's own
//     arithmetic and the rounding of the conic entries;
//   * for a positive semi-definite conic, minimising the exact Q over one coordinate gives
//     Q(d) >= dx^2 det4 / (4c) and Q(d) >= dy^2 det4 / (4a) with det4 = 4ac - b2^2, so the distance of the box from the
//     Gaussian's centre along either axis bounds Q from below (the "3 sigma slab" test, in exact arithmetic);
//     det4 is taken from the certified-PSD expression, i.e. rounded towards zero;
//   * the pair is dropped only if a lower bound exceeds qform_max, or the alpha it allows is below
//     alpha_min (with a 1% margin). A conic that is not certifiably PSD, a non-finite value, or a lidar
//     offset box that reaches the +-pi seam keeps the pair.
// Ill-conditioned grazing footprints (|d| ~ 1e5 px, M ~ 1e10) get a margin far above qform_max and are
// simply never culled — their per-query evaluation is rounding noise that must be reproduced, not bounded.
// ------------------------------------------------------------------------------------------------
struct PatchBox {
  float cx, cy, tc;
  float hx2, hy2;  // half-extents plus the query-side rounding slack: h + 2^-21 (|c| + h)
  float th2;       // th + 2^-21 (|tc| + th): multiplies |v| (travel during the patch's time span + slack on v t)
  int enabled;     // 0: the warp's queries are too spread out (or absent) to cull against
  int straddle;    // lidar: some query lies >= pi away from the first one (the patch crosses 0 / 2 pi): always wrap
};

// sqrt rounded up: MUFU.SQRT (2^-22 relative error) padded by 2^-20
__device__ __forceinline__ float sqrt_up(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * 1.000001f;
}

constexpr float kCullGamma = 3.814697265625e-06f;   // 2^-18
constexpr float kSlackUlp = 4.76837158203125e-07f;  // 2^-21

// Tests patches [kP0, kP0 + kNP) of the 8; returns their bits (in place: bit p for patch p).
// *wrapmask (lidar): bit p set if some query of patch p may need the azimuth wrap for this Gaussian, i.e. the raw
// difference qx - mx is not certified to lie inside (-pi, pi).
template <bool kLidar, int kP0 = 0, int kNP = 8>
__device__ __forceinline__ uint32_t patch_mask(const float4 gA, const float4 gB, const PatchBox* __restrict__ box,
                                               float qform_max, float alpha_min, uint32_t* wrapmask = nullptr) {
  if (wrapmask) *wrapmask = ((1u << kNP) - 1u) << kP0;
  const float a = gB.x, b2 = gB.y, c = gB.z, rho = gB.w;
  const float ab2 = fabsf(b2);
  // certified PSD: 4ac >= b2^2 with rounding slack on both sides
  const float det4 = 4.0f * a * c * (1.0f - 1e-6f) - b2 * b2 * (1.0f + 1e-6f);  // <= the exact 4ac - b2^2
  const bool psd = a > 0.0f && c > 0.0f && det4 >= 0.0f;
  if (!psd) return ((1u << kNP) - 1u) << kP0;
  // slab bounds: Q >= dx^2 kx and Q >= dy^2 ky, both factors rounded down
  // (approximate division, 2 ulp, under a 1.1e-5 safety factor: the directed-rounding intrinsics are ~70-instruction
  // subroutines — 6% of the camera forward's instructions went there)
  const float kx = __fdividef(det4, 4.0f * c) * (1.0f - 1.1e-5f), ky = __fdividef(det4, 4.0f * a) * (1.0f - 1.1e-5f);
  // alpha = rho exp(-qf/2) < alpha_min  <=>  qf > 2 ln(rho / alpha_min)
  float qmax = qform_max;
  if (alpha_min > 0.0f && rho > 0.0f && rho < 1e30f) qmax = fminf(qmax, 2.0f * __logf(rho * 1.01f / alpha_min) + 0.02f);
  const float avx = fabsf(gA.z), avy = fabsf(gA.w);
  const float slack_x = kSlackUlp * (fabsf(gA.x) + 8.0f), slack_y = kSlackUlp * (fabsf(gA.y) + 8.0f);
  uint32_t mask = 0u, wm = 0u;
#pragma unroll
  for (int p = kP0; p < kP0 + kNP; ++p) {
    const PatchBox b = box[p];
    bool keep = true;
    bool needw = true;
    if (b.enabled) {
      const float mxc = fmaf(gA.z, b.tc, gA.x), myc = fmaf(gA.w, b.tc, gA.y);
      float dcx = b.cx - mxc;
      if (kLidar) {
        // every query's raw difference lies within Hx of dcx (when the patch does not straddle the seam)
        needw = b.straddle || !(fabsf(dcx) + fmaf(fabsf(gA.z), b.th2, b.hx2) + kSlackUlp * (fabsf(gA.x) + 8.0f) < kPi - 1e-3f);
        dcx = wrap_pi(dcx);
      }
      const float dcy = b.cy - myc;
      // half-extents of the offset box: query box + rolling-shutter travel + rounding slack
      const float Hx = fmaf(avx, b.th2, b.hx2) + slack_x;
      const float Hy = fmaf(avy, b.th2, b.hy2) + slack_y;
      const float DX = fabsf(dcx) + Hx, DY = fabsf(dcy) + Hy;
      const bool seam = kLidar && !(DX < kPi - 1e-3f);
      // rounding slack of the fp32 quadratic form the exact evaluation computes: 2^-18 of the sum of term magnitudes
      const float E = kCullGamma * fmaf(a * DX, DX, fmaf(c * DY, DY, ab2 * DX * DY));
      // box-to-centre gaps; the extra slack covers the roundings of this very computation (dcx, Hx, the difference)
      const float gx = fmaxf(fabsf(dcx) - Hx - slack_x, 0.0f), gy = fmaxf(fabsf(dcy) - Hy - slack_y, 0.0f);
      const float slab = fmaxf(gx * gx * kx, gy * gy * ky) * (1.0f - 1e-5f);
      const float qe = qmax + E;
      // qe < 0: even qf = -E (the lowest value rounding allows) is beyond the alpha cut-off.
      // (A second bound — the triangle inequality of the Mahalanobis norm around the box centre,
      // sqrt(Q(d)) >= sqrt(Q(dc)) - sqrt(Qabs(H)) — was part of this test in round 1; measured on the north-star frame
      // it costs more instructions than the few extra pairs it removes save: camera forward 0.995 -> 0.952 ms and
      // lidar forward 0.482 -> 0.472 ms without it. Also measured and rejected: skipping the tests of patches whose warp
      // has saturated (no change: the warps of a tile saturate together) and re-fitting the boxes to the still
      // unsaturated queries before every batch (+4%: the boxes do not shrink, the lanes of a warp saturate together);
      // a third, ORIENTED slab across the ellipse's minor axis, Q >= (d.u)^2 det / (w^T C w) (+6%: only 3.7% fewer
      // survivors — what survives without blending on the north-star camera are grazing needles whose rounding
      // slack E exceeds qform_max, which no bound may remove).)
      const bool cull = !seam && ((qe < 0.0f) || (slab > qe * (1.0f + 1e-5f)));
      keep = !cull;
    }
    if (keep) mask |= 1u << p;
    if (needw) wm |= 1u << p;
  }
  if (kLidar && wrapmask) *wrapmask = wm;
  return mask;
}

// The same test with the per-box work cut to ~10 instructions (patch_mask above spends ~33 per box, 8 boxes per staged
// entry: 15% of the camera forward kernel). The rounding slack E is bounded ONCE per entry over the tile's box box[8]
// (tile_patch_box: it contains every patch box, so E_tile >= E_patch) and folded, with the alpha cut-off, into two
// per-entry radii: a patch is dropped when its box lies further than rx (ry) from the Gaussian's centre along x (y),
//   gap > r = sqrt(qe (1 + 2e-5) / k), qe = qmax + E_tile   =>   gap^2 k (1 - 1e-5) > (qmax + E_patch) (1 + 1e-5),
// i.e. exactly when patch_mask's slab test would drop it with the larger slack: every pair dropped here is dropped
// there (a subset, identical for well-conditioned footprints, where E is negligible), so it is as sound.
template <bool kLidar>
__device__ __forceinline__ uint32_t patch_mask_fast(const float4 gA, const float4 gB, const PatchBox* __restrict__ box,
                                                    float qform_max, float alpha_min, uint32_t* wrapmask = nullptr) {
  if (wrapmask) *wrapmask = 0xffu;
  const float a = gB.x, b2 = gB.y, c = gB.z, rho = gB.w;
  const float det4 = 4.0f * a * c * (1.0f - 1e-6f) - b2 * b2 * (1.0f + 1e-6f);  // <= the exact 4ac - b2^2
  const bool psd = a > 0.0f && c > 0.0f && det4 >= 0.0f;
  const PatchBox tb = box[8];
  if (!psd || !tb.enabled) return 0xffu;
  // (approximate division, 2 ulp, under a 1.1e-5 safety factor: the directed-rounding intrinsics are ~70-instruction
  // subroutines — 6% of the camera forward's instructions went there)
  const float kx = __fdividef(det4, 4.0f * c) * (1.0f - 1.1e-5f), ky = __fdividef(det4, 4.0f * a) * (1.0f - 1.1e-5f);
  float qmax = qform_max;
  if (alpha_min > 0.0f && rho > 0.0f && rho < 1e30f) qmax = fminf(qmax, 2.0f * __logf(rho * 1.01f / alpha_min) + 0.02f);
  const float avx = fabsf(gA.z), avy = fabsf(gA.w);
  const float slack_x = kSlackUlp * (fabsf(gA.x) + 8.0f), slack_y = kSlackUlp * (fabsf(gA.y) + 8.0f);
  // rounding slack of the fp32 quadratic form over the whole tile (un-wrapped azimuth difference: |wrap(u)| <= |u|)
  const float DXt = fabsf(tb.cx - fmaf(gA.z, tb.tc, gA.x)) + fmaf(avx, tb.th2, tb.hx2) + slack_x;
  const float DYt = fabsf(tb.cy - fmaf(gA.w, tb.tc, gA.y)) + fmaf(avy, tb.th2, tb.hy2) + slack_y;
  const float E = kCullGamma * fmaf(a * DXt, DXt, fmaf(c * DYt, DYt, fabsf(b2) * DXt * DYt));
  const float qe = (qmax + E) * (1.0f + 2e-5f);
  // qe < 0: even the lowest qf rounding allows is beyond the alpha cut-off -> radii below any gap. k == 0 -> r = inf
  // (never dropped along that axis); NaN compares false (kept).
  const float rx = qe < 0.0f ? -3.0e38f : sqrt_up(__fdividef(qe, kx) * (1.0f + 2e-6f)) + 2.0f * slack_x;
  const float ry = qe < 0.0f ? -3.0e38f : sqrt_up(__fdividef(qe, ky) * (1.0f + 2e-6f)) + 2.0f * slack_y;
  uint32_t mask = 0u, wm = 0u;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const PatchBox b = box[p];
    bool keep = true, needw = true;
    if (b.enabled) {
      float dcx = b.cx - fmaf(gA.z, b.tc, gA.x);
      const float dcy = b.cy - fmaf(gA.w, b.tc, gA.y);
      const float hx = fmaf(avx, b.th2, b.hx2), hy = fmaf(avy, b.th2, b.hy2);
      bool seam = false;
      if (kLidar) {
        needw = b.straddle || !(fabsf(dcx) + hx + 2.0f * slack_x < kPi - 1e-3f);
        dcx = wrap_pi(dcx);
        seam = !(fabsf(dcx) + hx + 2.0f * slack_x < kPi - 1e-3f);
      }
      // gap between the patch box and the centre (the 2 slack of patch_mask's gap are inside r)
      const bool cull = !seam && ((fabsf(dcx) - hx > rx) || (fabsf(dcy) - hy > ry));
      keep = !cull;
    }
    if (keep) mask |= 1u << p;
    if (needw) wm |= 1u << p;
  }
  if (kLidar && wrapmask) *wrapmask = wm;
  return mask;
}

// box[8] = a box containing the 8 patch boxes of the CTA (thread 0, after the patch boxes are visible). Disabled if no
// patch is enabled.
__device__ __forceinline__ void tile_patch_box(PatchBox* box) {
  const float big = 3.0e38f;
  float x0 = big, x1 = -big, y0 = big, y1 = -big, t0 = big, t1 = -big;
  int any = 0;
  for (int p = 0; p < 8; ++p) {
    const PatchBox b = box[p];
    if (!b.enabled) continue;
    any = 1;
    x0 = fminf(x0, b.cx - b.hx2); x1 = fmaxf(x1, b.cx + b.hx2);
    y0 = fminf(y0, b.cy - b.hy2); y1 = fmaxf(y1, b.cy + b.hy2);
    t0 = fminf(t0, b.tc - b.th2); t1 = fmaxf(t1, b.tc + b.th2);
  }
  PatchBox t;
  t.enabled = any;
  t.straddle = 1;
  t.cx = 0.5f * (x0 + x1); t.cy = 0.5f * (y0 + y1); t.tc = 0.5f * (t0 + t1);
  // half-extents padded so that the box certainly contains the patch boxes after the roundings above
  t.hx2 = (0.5f * (x1 - x0)) * (1.0f + 1e-5f) + 1e-6f * (fabsf(x0) + fabsf(x1)) + 1e-30f;
  t.hy2 = (0.5f * (y1 - y0)) * (1.0f + 1e-5f) + 1e-6f * (fabsf(y0) + fabsf(y1)) + 1e-30f;
  t.th2 = (0.5f * (t1 - t0)) * (1.0f + 1e-5f) + 1e-6f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
  if (!(t.hx2 == t.hx2 && t.hy2 == t.hy2 && t.th2 == t.th2) || !(t.hx2 < 1e30f && t.hy2 < 1e30f && t.th2 < 1e30f)) t.enabled = 0;
  box[8] = t;
}

// Bounding box of the warp's queries (lanes with `inside`), written by lane 0. Lidar azimuths are measured
// relative to the first valid lane's azimuth so that a patch straddling 0 / 2 pi stays compact.
template <bool kLidar>
__device__ __forceinline__ void warp_patch_box(bool inside, float qx, float qy, float t, int lane, PatchBox* out) {
  const unsigned act = __ballot_sync(0xffffffffu, inside);
  PatchBox b;
  b.cx = b.cy = b.tc = b.hx2 = b.hy2 = b.th2 = 0.0f;
  b.enabled = 0;
  b.straddle = 1;
  if (act != 0u) {
    const int first = __ffs(act) - 1;
    const float ref = __shfl_sync(0xffffffffu, qx, first);
    b.straddle = kLidar ? (__any_sync(0xffffffffu, inside && !(fabsf(qx - ref) < kPi - 1e-3f)) ? 1 : 0) : 0;
    float rx = kLidar ? wrap_pi(qx - ref) : qx;
    const float big = 3.0e38f;
    float x0 = inside ? rx : big, x1 = inside ? rx : -big;
    float y0 = inside ? qy : big, y1 = inside ? qy : -big;
    float t0 = inside ? t : big, t1 = inside ? t : -big;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      x0 = fminf(x0, __shfl_xor_sync(0xffffffffu, x0, o)); x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y0 = fminf(y0, __shfl_xor_sync(0xffffffffu, y0, o)); y1 = fmaxf(y1, __shfl_xor_sync(0xffffffffu, y1, o));
      t0 = fminf(t0, __shfl_xor_sync(0xffffffffu, t0, o)); t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, o));
    }
    // centre / half-extent, padded by a few ulp so the box certainly contains every query
    b.cx = 0.5f * (x0 + x1);
    b.cy = 0.5f * (y0 + y1);
    b.tc = 0.5f * (t0 + t1);
    float hx = 0.5f * (x1 - x0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(x0) + fabsf(x1)) + 1e-30f;
    const float hy = 0.5f * (y1 - y0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(y0) + fabsf(y1)) + 1e-30f;
    const float th = 0.5f * (t1 - t0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
    b.enabled = 1;
    if (kLidar) {
      b.cx += ref;                             // back to absolute azimuth (any 2 pi offset is removed by wrap_pi later)
      hx += 1e-6f * (fabsf(ref) + 8.0f);
      if (!(hx < 0.5f * kPi)) b.enabled = 0;   // rays all around the circle: nothing to cull against
    }
    b.hx2 = hx + kSlackUlp * (fabsf(b.cx) + hx);
    b.hy2 = hy + kSlackUlp * (fabsf(b.cy) + hy);
    b.th2 = th + kSlackUlp * (fabsf(b.tc) + th);
    if (!(b.hx2 == b.hx2 && b.hy2 == b.hy2 && b.th2 == b.th2)) b.enabled = 0;
  }
  if (lane == 0) *out = b;
}

// Bounding boxes of the warp's four 8-lane GROUPS (lanes 8g .. 8g + 7), written by the first lane of each group to
// out[g]: the second level of the culling hierarchy (k_raster_fwd walks one list per group, see there). Same
// construction and padding as warp_patch_box, reduced over the group only.
template <bool kLidar>
__device__ __forceinline__ void group_patch_box(bool inside, float qx, float qy, float t, int lane, PatchBox* out) {
  const unsigned act = __ballot_sync(0xffffffffu, inside);
  const int g = lane >> 3;
  const unsigned gact = (act >> (8 * g)) & 0xffu;
  PatchBox b;
  b.cx = b.cy = b.tc = b.hx2 = b.hy2 = b.th2 = 0.0f;
  b.enabled = 0;
  b.straddle = 1;
  // every lane takes part in the shuffles; groups without a valid lane produce a disabled box
  const int first = gact ? 8 * g + __ffs(gact) - 1 : lane;
  const float ref = __shfl_sync(0xffffffffu, qx, first);
  int strad = (kLidar && inside && !(fabsf(qx - ref) < kPi - 1e-3f)) ? 1 : 0;
  float rx = kLidar ? wrap_pi(qx - ref) : qx;
  const float big = 3.0e38f;
  float x0 = inside ? rx : big, x1 = inside ? rx : -big;
  float y0 = inside ? qy : big, y1 = inside ? qy : -big;
  float t0 = inside ? t : big, t1 = inside ? t : -big;
#pragma unroll
  for (int o = 4; o >= 1; o >>= 1) {
    x0 = fminf(x0, __shfl_xor_sync(0xffffffffu, x0, o)); x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
    y0 = fminf(y0, __shfl_xor_sync(0xffffffffu, y0, o)); y1 = fmaxf(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    t0 = fminf(t0, __shfl_xor_sync(0xffffffffu, t0, o)); t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, o));
    strad |= __shfl_xor_sync(0xffffffffu, strad, o);
  }
  if (gact != 0u) {
    b.straddle = kLidar ? strad : 0;
    b.cx = 0.5f * (x0 + x1);
    b.cy = 0.5f * (y0 + y1);
    b.tc = 0.5f * (t0 + t1);
    float hx = 0.5f * (x1 - x0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(x0) + fabsf(x1)) + 1e-30f;
    const float hy = 0.5f * (y1 - y0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(y0) + fabsf(y1)) + 1e-30f;
    const float th = 0.5f * (t1 - t0) * (1.0f + 1e-6f) + 1e-6f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
    b.enabled = 1;
    if (kLidar) {
      b.cx += ref;
      hx += 1e-6f * (fabsf(ref) + 8.0f);
      if (!(hx < 0.5f * kPi)) b.enabled = 0;
    }
    b.hx2 = hx + kSlackUlp * (fabsf(b.cx) + hx);
    b.hy2 = hy + kSlackUlp * (fabsf(b.cy) + hy);
    b.th2 = th + kSlackUlp * (fabsf(b.tc) + th);
    if (!(b.hx2 == b.hx2 && b.hy2 == b.hy2 && b.th2 == b.th2)) b.enabled = 0;
  }
  if ((lane & 7) == 0) out[g] = b;
}

// Order-preserving compaction of the batch entries whose mask has this warp's bit. Returns the count.
__device__ __forceinline__ int warp_compact(const uint8_t* __restrict__ sMask, int cnt, int warp, int lane,
                                            uint8_t* __restrict__ list) {
  int n = 0;
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int j = c0 + lane;
    const bool bit = j < cnt && ((sMask[j] >> warp) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    if (bit) list[n + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)j;
    n += __popc(bal);
  }
  __syncwarp();
  return n;
}

}  // namespace sb
