// splat_device.cuh — device-side types and the per-Gaussian forward math shared by the
// projection, binning and backward kernels of libsplat_b200.so.
//
// Reference semantics (paths under /root/reference/proj/include/splat/):
//   covariance_from_scale_quat  scene.hpp:190-196      compose_at_time   scene.hpp:273-308
//   project_camera              projection.hpp:88-118  project_lidar     projection.hpp:140-174
//   velocity / AABB / footprint projection.hpp:44-84   spherical map     projection.hpp:122-138
//
// Bit-exactness contract: the forward translation units are compiled with --fmad=false, so every
// `a * b + c` below is two IEEE-754 binary32 roundings in source order; the CPU oracle is built with
// -ffp-contract=off. Products are associated left to right exactly as the reference's Eigen
// expressions evaluate (`(R * S) * R^T`, `(J * C) * J^T`). Transcendentals come from detmath.h.
// Consequence: cull masks, AABBs, tile rectangles and sort keys are bit-identical to the oracle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "detmath.h"

namespace sb {

constexpr int kTile = 16;
constexpr int kNphi = 32;
constexpr int kNomega = 8;
constexpr int kMaxBoundaries = 63;  // supports up to 512 beams
constexpr int kChannels = 16;

constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 2.0f * 3.14159265358979323846f;

// Interpolated actor pose + effective body velocities at the query time (scene.hpp:238-258,
// 61-62), computed on the host in double and rounded once to float exactly like the
// reference's `cast<S>()`.
struct ActorState {
  float R[9];  // actor -> world, row-major
  float t[3];
  float w[3];  // effective_vel_ang
  float v[3];  // effective_vel_lin
};

// One sensor (camera or lidar) + RasterSettings + tile grid. Passed by value to kernels.
struct Sensor {
  int is_camera;
  float fx, fy, cx, cy;
  int width, height;
  float R[9], t[3], vel_lin[3], vel_ang[3];
  float shutter;      // camera shutter_duration / lidar scan_duration
  float time_offset;  // camera only
  float dilation;     // camera: settings.dilation; lidar: lidar.dilation() (projection.hpp:149)
  float near_plane, lidar_min_range;
  float elev_min, elev_max;
  float alpha_clamp, alpha_min, qform_max, transmittance_min;
  int tiles_x, tiles_y;
  float span, phi_max;  // lidar: N_phi * res_phi, M_phi * span
  int n_boundaries;
  float boundaries[kMaxBoundaries];
  int channels;  // camera 3 + d_f, lidar d_f
  int d_f;
};

struct SceneDev {
  int64_t n;
  int d_f;
  const float* mean;
  const float* scale_log;
  const float* quat;
  const float* opacity_logit;
  const float* color;
  const float* feature;
  const int32_t* actor_id;
  const ActorState* actors;  // n_actors entries (actor k at [k-1])
  int n_actors;
};

// Per-view projected state, indexed by SOURCE Gaussian index (no compaction on the hot path; the
// reference's compacted std::vector<ProjectedGaussian> order is recovered by a scan when asked).
struct ProjDev {
  float4* geomA;    // mean2d.x, mean2d.y, vel.x, vel.y
  float4* geomB;    // conic a, b2 = C01 + C10, c, rho = det_ratio * opacity
  float2* geomC;    // depth_key, vel.z (lidar v_r)
  float4* feat;     // 4 x float4 per Gaussian: camera rgb+feature, lidar feature (zero padded)
  int4* rect;       // x0, x1, y0, y1 (lidar x un-wrapped)
  uint32_t* count;  // tiles touched; 0 <=> culled
  uint32_t* dkey;   // fp32 bits of the (positive) depth key; 0xffffffff for culled Gaussians: the depth-sort key
  uint32_t* ccount; // two-level binning (camera): blocks of 2^cshift x 2^cshift tiles touched; null otherwise
  int cshift;
  int skip_feat;    // k_project leaves `feat` to k_pack_feat (geometry-first scene upload: colour / features still in flight)
};

__device__ __forceinline__ float wrap_two_pi(float a) {  // common.hpp:34-38
  a = fmodf(a, kTwoPi);
  if (a < 0.0f) a += kTwoPi;
  return a;
}

// 3x3 row-major helpers with the oracle's association: (a0*b0 + a1*b1) + a2*b2.
__device__ __forceinline__ float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
  return (a0 * b0 + a1 * b1) + a2 * b2;
}
__device__ __forceinline__ void mat_mul(const float* a, const float* b, float* c) {  // c = a b
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = dot3(a[3 * i], a[3 * i + 1], a[3 * i + 2], b[j], b[3 + j], b[6 + j]);
}
__device__ __forceinline__ void mat_mul_nt(const float* a, const float* b, float* c) {  // c = a b^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = dot3(a[3 * i], a[3 * i + 1], a[3 * i + 2], b[3 * j], b[3 * j + 1], b[3 * j + 2]);
}
__device__ __forceinline__ void mat_mul_tn(const float* a, const float* b, float* c) {  // c = a^T b
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = dot3(a[i], a[3 + i], a[6 + i], b[j], b[3 + j], b[6 + j]);
}
__device__ __forceinline__ void mat_vec(const float* a, const float* v, float* o) {  // o = a v
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = dot3(a[3 * i], a[3 * i + 1], a[3 * i + 2], v[0], v[1], v[2]);
}
__device__ __forceinline__ void mat_t_vec(const float* a, const float* v, float* o) {  // o = a^T v
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = dot3(a[i], a[3 + i], a[6 + i], v[0], v[1], v[2]);
}
__device__ __forceinline__ void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// Eigen::Quaternion(w,x,y,z).toRotationMatrix() (scene.hpp:193).
__device__ __forceinline__ void quat_to_rot(float w, float x, float y, float z, float* R) {
  const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
  const float twx = tx * w, twy = ty * w, twz = tz * w;
  const float txx = tx * x, txy = ty * x, txz = tz * x;
  const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1.0f - (tyy + tzz); R[1] = txy - twz;          R[2] = txz + twy;
  R[3] = txy + twz;          R[4] = 1.0f - (txx + tzz); R[5] = tyz - twx;
  R[6] = txz - twy;          R[7] = tyz + twx;          R[8] = 1.0f - (txx + tyy);
}

// Everything the forward pass knows about one Gaussian for one sensor.
struct Fwd {
  bool visible;
  bool dynamic;
  int actor;          // actor_id
  float q[4], qn;     // normalised quaternion, raw norm
  float Rq[9];        // R(q_hat)
  float s2[3];        // exp(2 scale_log)
  float cov_local[9];
  float mean_w[3], cov_w[9], vel_dyn_w[3];
  float opacity;
  float mu[3];        // sensor frame
  float cov_s[9];     // sensor-frame covariance R cov_w R^T
  float J[9];         // camera: rows 0-1 used, row 2 zero
  float mean2d[2], depth;
  float cov2d[4];
  float conic[4], det_ratio;
  float u[3];         // rel_vel_sensor
  float vel[3];
  float lo[2], hi[2];
};

// scene.hpp:190-196 + 273-308: world-frame mean / covariance / dynamic velocity / opacity.
__device__ __forceinline__ void compose_one(const SceneDev& sc, int64_t i, Fwd& f) {
  const float q0 = sc.quat[4 * i], q1 = sc.quat[4 * i + 1], q2 = sc.quat[4 * i + 2], q3 = sc.quat[4 * i + 3];
  f.qn = DM_SQRT(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
  f.q[0] = q0 / f.qn; f.q[1] = q1 / f.qn; f.q[2] = q2 / f.qn; f.q[3] = q3 / f.qn;
  quat_to_rot(f.q[0], f.q[1], f.q[2], f.q[3], f.Rq);
#pragma unroll
  for (int k = 0; k < 3; ++k) f.s2[k] = detmath::exp(2.0f * sc.scale_log[3 * i + k]);
  float RD[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) RD[3 * r + c] = f.Rq[3 * r + c] * f.s2[c];
  mat_mul_nt(RD, f.Rq, f.cov_local);
  f.opacity = detmath::sigmoid(sc.opacity_logit[i]);
  f.actor = sc.actor_id[i];
  f.dynamic = f.actor != 0;
  const float mb[3] = {sc.mean[3 * i], sc.mean[3 * i + 1], sc.mean[3 * i + 2]};
  if (!f.dynamic) {
#pragma unroll
    for (int k = 0; k < 3; ++k) { f.mean_w[k] = mb[k]; f.vel_dyn_w[k] = 0.0f; }
#pragma unroll
    for (int k = 0; k < 9; ++k) f.cov_w[k] = f.cov_local[k];
  } else {
    const ActorState& a = sc.actors[f.actor - 1];
    float Ra[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Ra[k] = a.R[k];
    float tmp[3];
    mat_vec(Ra, mb, tmp);
#pragma unroll
    for (int k = 0; k < 3; ++k) f.mean_w[k] = tmp[k] + a.t[k];
    float RC[9];
    mat_mul(Ra, f.cov_local, RC);
    mat_mul_nt(RC, Ra, f.cov_w);
    float wxm[3];
    cross3(a.w, mb, wxm);
    const float wb[3] = {wxm[0] + a.v[0], wxm[1] + a.v[1], wxm[2] + a.v[2]};
    mat_vec(Ra, wb, f.vel_dyn_w);
  }
}

// projection.hpp:75-84 with Eigen's closed-form 2x2 determinant / inverse.
__device__ __forceinline__ bool finalize_footprint(Fwd& f, float dilation) {
  const float det = f.cov2d[0] * f.cov2d[3] - f.cov2d[2] * f.cov2d[1];
  const float d00 = f.cov2d[0] + dilation, d11 = f.cov2d[3] + dilation, d01 = f.cov2d[1], d10 = f.cov2d[2];
  const float det_dilated = d00 * d11 - d10 * d01;
  if (!(det > 0.0f) || !(det_dilated > 0.0f)) return false;
  const float invdet = 1.0f / det_dilated;
  f.conic[0] = d11 * invdet;
  f.conic[1] = -d01 * invdet;
  f.conic[2] = -d10 * invdet;
  f.conic[3] = d00 * invdet;
  f.det_ratio = DM_SQRT(det / det_dilated);
  return true;
}

// projection.hpp:62-71
__device__ __forceinline__ void velocity_expanded_aabb(Fwd& f, float dilation, float shutter) {
  const float a0 = f.cov2d[0] + dilation, a1 = f.cov2d[3] + dilation;
  const float hx = 3.0f * DM_SQRT(0.0f < a0 ? a0 : 0.0f) + fabsf(f.vel[0]) * shutter / 2.0f;
  const float hy = 3.0f * DM_SQRT(0.0f < a1 ? a1 : 0.0f) + fabsf(f.vel[1]) * shutter / 2.0f;
  f.lo[0] = f.mean2d[0] - hx; f.lo[1] = f.mean2d[1] - hy;
  f.hi[0] = f.mean2d[0] + hx; f.hi[1] = f.mean2d[1] + hy;
}

// projection.hpp:44-48 with v_dyn rotated into the sensor frame (projection.hpp:110, 166)
__device__ __forceinline__ void relative_velocity(const Sensor& s, Fwd& f) {
  float c[3], vd[3];
  cross3(s.vel_ang, f.mu, c);
  mat_vec(s.R, f.vel_dyn_w, vd);
#pragma unroll
  for (int k = 0; k < 3; ++k) f.u[k] = (-c[k] - s.vel_lin[k]) + vd[k];
}

__device__ __forceinline__ void sensor_frame(const Sensor& s, Fwd& f) {
  float tmp[3];
  mat_vec(s.R, f.mean_w, tmp);
#pragma unroll
  for (int k = 0; k < 3; ++k) f.mu[k] = tmp[k] + s.t[k];
}

__device__ __forceinline__ void sensor_cov(const Sensor& s, Fwd& f) {
  float RC[9];
  mat_mul(s.R, f.cov_w, RC);
  mat_mul_nt(RC, s.R, f.cov_s);
}

// (J C) J^T for the first `rows` rows of J.
template <int ROWS>
__device__ __forceinline__ void jcjt(const float* J, const float* C, float* out /* ROWS x ROWS */) {
  float JC[ROWS * 3];
#pragma unroll
  for (int i = 0; i < ROWS; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) JC[3 * i + j] = dot3(J[3 * i], J[3 * i + 1], J[3 * i + 2], C[j], C[3 + j], C[6 + j]);
#pragma unroll
  for (int i = 0; i < ROWS; ++i)
#pragma unroll
    for (int j = 0; j < ROWS; ++j)
      out[ROWS * i + j] = dot3(JC[3 * i], JC[3 * i + 1], JC[3 * i + 2], J[3 * j], J[3 * j + 1], J[3 * j + 2]);
}

// projection.hpp:88-118 for one composed Gaussian.
__device__ __forceinline__ void project_camera_one(const Sensor& s, Fwd& f) {
  f.visible = false;
  sensor_frame(s, f);
  if (f.mu[2] <= s.near_plane) return;
  f.depth = f.mu[2];
  f.mean2d[0] = s.fx * f.mu[0] / f.mu[2] + s.cx;  // scene.hpp:109-111
  f.mean2d[1] = s.fy * f.mu[1] / f.mu[2] + s.cy;
  const float iz = 1.0f / f.mu[2];                // scene.hpp:112-117
  f.J[0] = s.fx * iz; f.J[1] = 0.0f; f.J[2] = -s.fx * f.mu[0] * iz * iz;
  f.J[3] = 0.0f; f.J[4] = s.fy * iz; f.J[5] = -s.fy * f.mu[1] * iz * iz;
  f.J[6] = f.J[7] = f.J[8] = 0.0f;
  sensor_cov(s, f);
  jcjt<2>(f.J, f.cov_s, f.cov2d);
  if (!finalize_footprint(f, s.dilation)) return;
  relative_velocity(s, f);
  f.vel[0] = dot3(f.J[0], f.J[1], f.J[2], f.u[0], f.u[1], f.u[2]);
  f.vel[1] = dot3(f.J[3], f.J[4], f.J[5], f.u[0], f.u[1], f.u[2]);
  f.vel[2] = 0.0f;
  velocity_expanded_aabb(f, s.dilation, s.shutter);
  const float W = (float)s.width, H = (float)s.height;  // projection.hpp:19-22, 114
  if (!(f.lo[0] < W && f.hi[0] > 0.0f && f.lo[1] < H && f.hi[1] > 0.0f)) return;
  f.visible = true;
}

// projection.hpp:127-138 (Eq. 11)
__device__ __forceinline__ void spherical_jacobian(const float* p, float* J) {
  const float x = p[0], y = p[1], z = p[2];
  const float d2 = x * x + y * y;
  const float d = DM_SQRT(d2);
  const float r2 = d2 + z * z;
  const float r = DM_SQRT(r2);
  J[0] = -y / d2; J[1] = x / d2; J[2] = 0.0f;
  J[3] = -x * z / (r2 * d); J[4] = -y * z / (r2 * d); J[5] = d / r2;
  J[6] = x / r; J[7] = y / r; J[8] = z / r;
}

// projection.hpp:140-174 for one composed Gaussian.
__device__ __forceinline__ void project_lidar_one(const Sensor& s, Fwd& f) {
  f.visible = false;
  sensor_frame(s, f);
  const float x = f.mu[0], y = f.mu[1], z = f.mu[2];
  const float d2 = x * x + y * y;
  if (d2 < s.lidar_min_range * s.lidar_min_range) return;
  const float r = DM_SQRT((x * x + y * y) + z * z);  // projection.hpp:122-125
  const float phi = wrap_two_pi(detmath::atan2(y, x));
  const float omega = detmath::asin(z / r);
  if (r < s.lidar_min_range) return;
  f.depth = r;
  f.mean2d[0] = phi; f.mean2d[1] = omega;
  spherical_jacobian(f.mu, f.J);
  sensor_cov(s, f);
  float c3[9];
  jcjt<3>(f.J, f.cov_s, c3);
  f.cov2d[0] = c3[0]; f.cov2d[1] = c3[1]; f.cov2d[2] = c3[3]; f.cov2d[3] = c3[4];
  if (!finalize_footprint(f, s.dilation)) return;
  relative_velocity(s, f);
#pragma unroll
  for (int k = 0; k < 3; ++k) f.vel[k] = dot3(f.J[3 * k], f.J[3 * k + 1], f.J[3 * k + 2], f.u[0], f.u[1], f.u[2]);
  velocity_expanded_aabb(f, s.dilation, s.shutter);
  if (f.hi[1] < s.elev_min || f.lo[1] > s.elev_max) return;
  f.visible = true;
}

// SPEC.md:190-198 image_tile_range
__device__ __forceinline__ int clamp_tile(float v, int m) {
  const float fm = (float)m;
  v = (v < 0.0f) ? 0.0f : v;  // std::max(v, 0)
  v = (fm < v) ? fm : v;      // std::min(v, m)
  return (int)v;
}
__device__ __forceinline__ int4 image_tile_range(const Fwd& f, int tiles_x, int tiles_y) {
  int4 r;
  r.x = clamp_tile(floorf(f.lo[0] / (float)kTile), tiles_x);
  r.y = clamp_tile(ceilf(f.hi[0] / (float)kTile), tiles_x);
  r.z = clamp_tile(floorf(f.lo[1] / (float)kTile), tiles_y);
  r.w = clamp_tile(ceilf(f.hi[1] / (float)kTile), tiles_y);
  return r;
}

// PAPER.md:466-490 / SPEC.md:200-218: azimuth columns (un-wrapped) and elevation rows.
__device__ __forceinline__ int4 lidar_tile_range(const Fwd& f, const Sensor& s) {
  const float lim = 4.0f * (float)s.tiles_x;
  float fl, fh;
  if (f.lo[0] >= 0.0f) fl = floorf(f.lo[0] / s.span);
  else fl = floorf(((f.lo[0] + kTwoPi) - s.phi_max) / s.span);
  if (f.hi[0] <= kTwoPi) fh = ceilf(f.hi[0] / s.span);
  else fh = ceilf(fmodf(f.hi[0], kTwoPi) / s.span) + (float)s.tiles_x;
  fl = fl < -lim ? -lim : fl; fl = lim < fl ? lim : fl;
  fh = fh < -lim ? -lim : fh; fh = lim < fh ? lim : fh;
  int4 r;
  r.x = (int)fl;
  r.y = (int)fh;
  if (r.y - r.x >= s.tiles_x) { r.x = 0; r.y = s.tiles_x; }
  r.z = 0;
  r.w = 1;
  for (int k = 0; k < s.n_boundaries; ++k) {
    if (s.boundaries[k] < f.lo[1]) r.z = k + 1;
    if (s.boundaries[k] <= f.hi[1]) r.w = k + 2;
  }
  return r;
}

}  // namespace sb
