// splat_oracle.hpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may use anything under oracle/. The product (libsplat_b200.so)
// never includes, links or calls it.
//
// What it is: a plain-struct (no Eigen) restatement of the reference's
//   scene-model  (/root/reference/proj/include/splat/scene.hpp)
//   projection   (/root/reference/proj/include/splat/projection.hpp)
//   math helpers (common.hpp, so3.hpp)
// templated on the scalar S in {float, double}, plus the FIRST implementation
// of the two modules the reference only specifies in prose:
//   tiling
//   rasterizer
// Every function cites the reference lines it follows.
//
// Pinning status: the reference ships no tests, goldens or fixtures.
// The oracle is pinned by (a) SPEC.md's worked examples KA1-KA16 and properties
// P1-P3 (tests/test_oracle_kat.py), (b) outputs of the UNMODIFIED reference
// headers compiled against a clean-room Eigen shim (oracle/_ref, compose +
// projection forward/backward; tests/test_oracle_vs_ref.py), (c) tiled ==
// brute-force and analytic == finite-difference self-consistency for the
// SPEC-only modules, for which no reference code exists ("parity unpinned"
// beyond SPEC's examples for tiling + rasterizer).
//
// fp32 instantiation: transcendental calls go through detmath.h (shared with
// the kernels) and the compositing inner loop spells its fused multiply-adds
// explicitly, so that a build with -ffp-contract=off executes the identical
// IEEE-754 operation sequence as the sm_100a kernels => integer outputs
// (cull mask, tile rectangles, sorted keys, contributor counts) are bit-exact.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../paper_2411_16816_b200/csrc/detmath.h"

namespace orc {

// ----------------------------------------------------------------------------
// scalar traits
// ----------------------------------------------------------------------------
template <class S> struct Sc;
template <> struct Sc<float> {
  static float exp(float x) { return detmath::exp(x); }
  static float sigmoid(float x) { return detmath::sigmoid(x); }
  static float atan2(float y, float x) { return detmath::atan2(y, x); }
  static float asin(float x) { return detmath::asin(x); }
  static float sqrt(float x) { return __builtin_sqrtf(x); }
  static float fma(float a, float b, float c) { return __builtin_fmaf(a, b, c); }
  static float fmod(float a, float b) { return std::fmod(a, b); }
  static float floor(float a) { return std::floor(a); }
  static float ceil(float a) { return std::ceil(a); }
  static float abs(float a) { return std::fabs(a); }
  static float cos(float a) { return std::cos(a); }   // decoder only (tolerance parity, no bit-exactness contract)
  static float sin(float a) { return std::sin(a); }
};
template <> struct Sc<double> {
  static double exp(double x) { return std::exp(x); }
  // common.hpp:54-58
  static double sigmoid(double x) {
    if (x >= 0) return 1.0 / (1.0 + std::exp(-x));
    double e = std::exp(x);
    return e / (1.0 + e);
  }
  static double atan2(double y, double x) { return std::atan2(y, x); }
  static double asin(double x) { return std::asin(x); }
  static double sqrt(double x) { return std::sqrt(x); }
  static double fma(double a, double b, double c) { return a * b + c; }
  static double fmod(double a, double b) { return std::fmod(a, b); }
  static double floor(double a) { return std::floor(a); }
  static double ceil(double a) { return std::ceil(a); }
  static double abs(double a) { return std::fabs(a); }
  static double cos(double a) { return std::cos(a); }
  static double sin(double a) { return std::sin(a); }
};

template <class S> constexpr S pi() { return static_cast<S>(3.14159265358979323846L); }  // common.hpp:30
template <class S> constexpr S two_pi() { return static_cast<S>(2) * pi<S>(); }          // common.hpp:31

/// common.hpp:34-38
template <class S> S wrap_two_pi(S a) {
  a = Sc<S>::fmod(a, two_pi<S>());
  if (a < S(0)) a += two_pi<S>();
  return a;
}
/// common.hpp:41-46
template <class S> S wrap_pi(S a) {
  a = Sc<S>::fmod(a, two_pi<S>());
  if (a > pi<S>()) a -= two_pi<S>();
  if (a <= -pi<S>()) a += two_pi<S>();
  return a;
}

// ----------------------------------------------------------------------------
// tiny fixed-size linear algebra, evaluation order spelled out
// ----------------------------------------------------------------------------
template <class S> struct V3 {
  S x = 0, y = 0, z = 0;
  V3() = default;
  V3(S a, S b, S c) : x(a), y(b), z(c) {}
  S operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  S& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
template <class S> V3<S> operator+(V3<S> a, V3<S> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class S> V3<S> operator-(V3<S> a, V3<S> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class S> V3<S> operator-(V3<S> a) { return {-a.x, -a.y, -a.z}; }
template <class S> V3<S> operator*(S s, V3<S> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class S> S dot(V3<S> a, V3<S> b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
template <class S> V3<S> cross(V3<S> a, V3<S> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

template <class S> struct M3 {
  S m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major
  S operator()(int r, int c) const { return m[3 * r + c]; }
  S& operator()(int r, int c) { return m[3 * r + c]; }
  static M3 identity() {
    M3 a;
    a(0, 0) = a(1, 1) = a(2, 2) = S(1);
    return a;
  }
  template <class T> M3<T> cast() const {
    M3<T> o;
    for (int i = 0; i < 9; ++i) o.m[i] = T(m[i]);
    return o;
  }
};
template <class S> M3<S> mul(const M3<S>& a, const M3<S>& b) {
  M3<S> c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
  return c;
}
/// a * b^T
template <class S> M3<S> mul_nt(const M3<S>& a, const M3<S>& b) {
  M3<S> c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(i, j) = (a(i, 0) * b(j, 0) + a(i, 1) * b(j, 1)) + a(i, 2) * b(j, 2);
  return c;
}
/// a^T * b
template <class S> M3<S> mul_tn(const M3<S>& a, const M3<S>& b) {
  M3<S> c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(i, j) = (a(0, i) * b(0, j) + a(1, i) * b(1, j)) + a(2, i) * b(2, j);
  return c;
}
template <class S> M3<S> transpose(const M3<S>& a) {
  M3<S> c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(i, j) = a(j, i);
  return c;
}
template <class S> M3<S> operator+(const M3<S>& a, const M3<S>& b) {
  M3<S> c;
  for (int i = 0; i < 9; ++i) c.m[i] = a.m[i] + b.m[i];
  return c;
}
template <class S> M3<S> operator-(const M3<S>& a, const M3<S>& b) {
  M3<S> c;
  for (int i = 0; i < 9; ++i) c.m[i] = a.m[i] - b.m[i];
  return c;
}
template <class S> M3<S> operator*(S s, const M3<S>& a) {
  M3<S> c;
  for (int i = 0; i < 9; ++i) c.m[i] = s * a.m[i];
  return c;
}
template <class S> V3<S> mul(const M3<S>& a, V3<S> v) {
  return {(a(0, 0) * v.x + a(0, 1) * v.y) + a(0, 2) * v.z, (a(1, 0) * v.x + a(1, 1) * v.y) + a(1, 2) * v.z,
          (a(2, 0) * v.x + a(2, 1) * v.y) + a(2, 2) * v.z};
}
template <class S> V3<S> mul_t(const M3<S>& a, V3<S> v) {  // a^T v
  return {(a(0, 0) * v.x + a(1, 0) * v.y) + a(2, 0) * v.z, (a(0, 1) * v.x + a(1, 1) * v.y) + a(2, 1) * v.z,
          (a(0, 2) * v.x + a(1, 2) * v.y) + a(2, 2) * v.z};
}
/// common.hpp:48-52
template <class S> M3<S> skew(V3<S> v) {
  M3<S> m;
  m(0, 1) = -v.z; m(0, 2) = v.y;
  m(1, 0) = v.z;  m(1, 2) = -v.x;
  m(2, 0) = -v.y; m(2, 1) = v.x;
  return m;
}
template <class S> S frob(const M3<S>& a, const M3<S>& b) {  // (a.array()*b.array()).sum()
  S s = 0;
  for (int i = 0; i < 9; ++i) s += a.m[i] * b.m[i];
  return s;
}

// ----------------------------------------------------------------------------
// so3.hpp (always evaluated in double: actor poses are per-actor host work)
// ----------------------------------------------------------------------------
using V3d = V3<double>;
using M3d = M3<double>;

/// so3.hpp:10-19
inline M3d so3_exp(V3d phi) {
  const double t2 = dot(phi, phi);
  const M3d K = skew(phi);
  if (t2 < 1e-16) return M3d::identity() + K + 0.5 * mul(K, K);
  const double t = std::sqrt(t2);
  return M3d::identity() + (std::sin(t) / t) * K + ((1.0 - std::cos(t)) / t2) * mul(K, K);
}
/// so3.hpp:21-38
inline V3d so3_log(const M3d& R) {
  const double tr = R(0, 0) + R(1, 1) + R(2, 2);
  const double c = std::clamp((tr - 1.0) / 2.0, -1.0, 1.0);
  const double t = std::acos(c);
  V3d w(R(2, 1) - R(1, 2), R(0, 2) - R(2, 0), R(1, 0) - R(0, 1));
  if (t < 1e-8) return 0.5 * w;
  if (t > pi<double>() - 1e-6) {
    M3d A = 0.5 * (R + M3d::identity());
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (A(i, i) > A(k, k)) k = i;
    V3d axis(A(0, k), A(1, k), A(2, k));
    axis = (1.0 / std::sqrt(A(k, k))) * axis;
    axis = (1.0 / std::sqrt(dot(axis, axis))) * axis;
    if (dot(w, axis) < 0) axis = -axis;
    return t * axis;
  }
  return (t / (2.0 * std::sin(t))) * w;
}
/// so3.hpp:41-50
inline M3d so3_right_jacobian(V3d phi) {
  const double t2 = dot(phi, phi);
  const M3d K = skew(phi);
  if (t2 < 1e-16) return M3d::identity() - 0.5 * K + (1.0 / 6.0) * mul(K, K);
  const double t = std::sqrt(t2);
  return M3d::identity() - ((1.0 - std::cos(t)) / t2) * K + ((t - std::sin(t)) / (t2 * t)) * mul(K, K);
}
/// so3.hpp:52-61
inline M3d so3_right_jacobian_inv(V3d phi) {
  const double t2 = dot(phi, phi);
  const M3d K = skew(phi);
  if (t2 < 1e-16) return M3d::identity() + 0.5 * K + (1.0 / 12.0) * mul(K, K);
  const double t = std::sqrt(t2);
  const double coeff = 1.0 / t2 - (1.0 + std::cos(t)) / (2.0 * t * std::sin(t));
  return M3d::identity() + 0.5 * K + coeff * mul(K, K);
}
/// so3.hpp:64-66
inline M3d so3_left_jacobian_inv(V3d phi) { return so3_right_jacobian_inv(-phi); }

/// so3.hpp:69-81
template <class S> struct SE3 {
  M3<S> R = M3<S>::identity();
  V3<S> t;
  V3<S> apply(V3<S> p) const { return mul(R, p) + t; }
};

// ----------------------------------------------------------------------------
// scene.hpp
// ----------------------------------------------------------------------------
/// scene.hpp:11-45. Columnar, Eigen column-major => xyz interleaved.
template <class S> struct GaussianSet {
  int64_t n = 0;
  int d_f = 0;
  std::vector<S> mean, scale_log, quat, opacity_logit, color, feature;
  std::vector<int32_t> actor_id;
  V3<S> mean_at(int64_t i) const { return {mean[3 * i], mean[3 * i + 1], mean[3 * i + 2]}; }
};

/// scene.hpp:50-96 (double storage, see header comment on so3)
struct ActorTrack {
  std::vector<double> stamps;
  std::vector<SE3<double>> poses;       // actor -> world
  std::vector<double> pose_offset;      // 6 x n col-major: rows 0-2 translation, 3-5 rotvec
  V3d vel_lin, vel_ang;
  double vel_offset[6] = {0, 0, 0, 0, 0, 0};
  int64_t pose_count() const { return (int64_t)poses.size(); }
  V3d effective_vel_lin() const { return {vel_lin.x + vel_offset[0], vel_lin.y + vel_offset[1], vel_lin.z + vel_offset[2]}; }
  V3d effective_vel_ang() const { return {vel_ang.x + vel_offset[3], vel_ang.y + vel_offset[4], vel_ang.z + vel_offset[5]}; }
  V3d off_t(int64_t i) const { return {pose_offset[6 * i], pose_offset[6 * i + 1], pose_offset[6 * i + 2]}; }
  V3d off_r(int64_t i) const { return {pose_offset[6 * i + 3], pose_offset[6 * i + 4], pose_offset[6 * i + 5]}; }
  /// scene.hpp:64-67
  SE3<double> corrected_pose(int64_t i) const {
    SE3<double> o;
    o.R = mul(poses[i].R, so3_exp(off_r(i)));
    o.t = poses[i].t + off_t(i);
    return o;
  }
  /// scene.hpp:70-83
  void init_velocity_from_poses() {
    vel_lin = V3d();
    vel_ang = V3d();
    const int64_t n = pose_count();
    if (n < 2) return;
    V3d v, w;
    for (int64_t i = 0; i + 1 < n; ++i) {
      const double dt = stamps[i + 1] - stamps[i];
      v = v + (1.0 / dt) * mul_t(poses[i].R, poses[i + 1].t - poses[i].t);
      w = w + (1.0 / dt) * so3_log(mul_tn(poses[i].R, poses[i + 1].R));
    }
    vel_lin = (1.0 / double(n - 1)) * v;
    vel_ang = (1.0 / double(n - 1)) * w;
  }
};

/// scene.hpp:98-137
template <class S> struct CameraModel {
  S fx = 100, fy = 100, cx = 50, cy = 50;
  int width = 100, height = 100;
  SE3<S> pose;  // world -> sensor
  V3<S> vel_lin, vel_ang;
  S shutter_duration = 0, time_offset = 0, timestamp = 0;
};
/// scene.hpp:139-168
template <class S> struct LidarModel {
  std::vector<S> elevation_channels;
  S azimuth_resolution = 0, scan_duration = 0, beam_divergence_h = 0, beam_divergence_v = 0;
  SE3<S> pose;
  V3<S> vel_lin, vel_ang;
  S timestamp = 0, max_range = 120;
  int beam_count() const { return (int)elevation_channels.size(); }
  S dilation() const { return beam_divergence_h * beam_divergence_v; }  // scene.hpp:152
};

/// scene.hpp:171-187
template <class S> struct SceneGraph {
  GaussianSet<S> gaussians;
  std::vector<ActorTrack> tracks;
};

/// Eigen::Quaternion(w,x,y,z).toRotationMatrix() — Eigen's published algorithm
/// (un-vendored dependency of scene.hpp:193; version unpinned, CMakeLists.txt:5).
template <class S> M3<S> quat_to_rot(S w, S x, S y, S z) {
  const S tx = S(2) * x, ty = S(2) * y, tz = S(2) * z;
  const S twx = tx * w, twy = ty * w, twz = tz * w;
  const S txx = tx * x, txy = ty * x, txz = tz * x;
  const S tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3<S> R;
  R(0, 0) = S(1) - (tyy + tzz); R(0, 1) = txy - twz;          R(0, 2) = txz + twy;
  R(1, 0) = txy + twz;          R(1, 1) = S(1) - (txx + tzz); R(1, 2) = tyz - twx;
  R(2, 0) = txz - twy;          R(2, 1) = tyz + twx;          R(2, 2) = S(1) - (txx + tyy);
  return R;
}

/// scene.hpp:190-196
template <class S> M3<S> covariance_from_scale_quat(V3<S> scale_log, const S* quat) {
  const S qn = Sc<S>::sqrt(((quat[0] * quat[0] + quat[1] * quat[1]) + quat[2] * quat[2]) + quat[3] * quat[3]);
  const S w = quat[0] / qn, x = quat[1] / qn, y = quat[2] / qn, z = quat[3] / qn;
  const M3<S> R = quat_to_rot<S>(w, x, y, z);
  const S s2[3] = {Sc<S>::exp(S(2) * scale_log.x), Sc<S>::exp(S(2) * scale_log.y), Sc<S>::exp(S(2) * scale_log.z)};
  M3<S> RD;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) RD(i, j) = R(i, j) * s2[j];
  return mul_nt(RD, R);
}

/// scene.hpp:200-226
template <class S>
void covariance_backward(V3<S> scale_log, const S* quat, const M3<S>& g_sigma_in, S* g_scale_log, S* g_quat) {
  const M3<S> G = S(0.5) * (g_sigma_in + transpose(g_sigma_in));
  const S qn = Sc<S>::sqrt(((quat[0] * quat[0] + quat[1] * quat[1]) + quat[2] * quat[2]) + quat[3] * quat[3]);
  const S q[4] = {quat[0] / qn, quat[1] / qn, quat[2] / qn, quat[3] / qn};
  const M3<S> R = quat_to_rot<S>(q[0], q[1], q[2], q[3]);
  const S s2[3] = {Sc<S>::exp(S(2) * scale_log.x), Sc<S>::exp(S(2) * scale_log.y), Sc<S>::exp(S(2) * scale_log.z)};
  const M3<S> M = mul(mul_tn(R, G), R);
  for (int k = 0; k < 3; ++k) g_scale_log[k] += M(k, k) * S(2) * s2[k];
  M3<S> GR = mul(G, R);
  M3<S> g_R;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) g_R(i, j) = S(2) * GR(i, j) * s2[j];
  const S w = q[0], x = q[1], y = q[2], z = q[3];
  const S dR[4][9] = {
      {S(0), -z, y, z, S(0), -x, -y, x, S(0)},
      {S(0), y, z, y, S(-2) * x, -w, z, w, S(-2) * x},
      {S(-2) * y, x, w, x, S(0), z, -w, z, S(-2) * y},
      {S(-2) * z, -w, x, w, S(-2) * z, y, x, y, S(0)}};
  S g_qhat[4];
  for (int k = 0; k < 4; ++k) {
    S s = 0;
    for (int e = 0; e < 9; ++e) s += g_R.m[e] * dR[k][e];
    g_qhat[k] = S(2) * s;
  }
  S qd = 0;
  for (int k = 0; k < 4; ++k) qd += q[k] * g_qhat[k];
  for (int k = 0; k < 4; ++k) g_quat[k] += (g_qhat[k] - q[k] * qd) / qn;
}

/// scene.hpp:231-258
struct InterpolatedPose {
  SE3<double> pose;
  int64_t i0 = 0, i1 = 0;
  double u = 0;
  V3d geo;
};
inline InterpolatedPose interpolate_pose(const ActorTrack& track, double t) {
  InterpolatedPose out;
  const int64_t n = track.pose_count();
  if (n == 0) throw std::runtime_error("actor track has no poses");
  if (n == 1) {
    out.pose = track.corrected_pose(0);
    return out;
  }
  int64_t i = 0;
  while (i + 2 < n && t >= track.stamps[i + 1]) ++i;
  out.i0 = i;
  out.i1 = i + 1;
  const double t0 = track.stamps[i], t1 = track.stamps[i + 1];
  out.u = (t - t0) / (t1 - t0);
  const SE3<double> a = track.corrected_pose(i), b = track.corrected_pose(i + 1);
  out.geo = so3_log(mul_tn(a.R, b.R));
  out.pose.R = mul(a.R, so3_exp(out.u * out.geo));
  out.pose.t = (1.0 - out.u) * a.t + out.u * b.t;
  return out;
}

/// scene.hpp:261-271
template <class S> struct ComposedScene {
  const SceneGraph<S>* graph = nullptr;
  S time = 0;
  std::vector<S> mean_w;   // 3N
  std::vector<M3<S>> cov_w;
  std::vector<S> vel_dyn_w;  // 3N
  std::vector<S> opacity;    // N
  std::vector<InterpolatedPose> actor_poses;
  int64_t size() const { return (int64_t)opacity.size(); }
  V3<S> mean_at(int64_t i) const { return {mean_w[3 * i], mean_w[3 * i + 1], mean_w[3 * i + 2]}; }
  V3<S> vel_at(int64_t i) const { return {vel_dyn_w[3 * i], vel_dyn_w[3 * i + 1], vel_dyn_w[3 * i + 2]}; }
};

template <class S> V3<S> cast3(V3d v) { return {S(v.x), S(v.y), S(v.z)}; }

/// Static chunked parallel map — restatement of common.hpp:72-90.
inline void parallel_chunks(int64_t count, int workers, const std::function<void(int, int64_t, int64_t)>& fn) {
  workers = std::max(1, workers);
  if (count <= 0) return;
  if (workers == 1 || count < 2 * workers) {
    fn(0, 0, count);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(workers);
  const int64_t chunk = (count + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int64_t b = std::min<int64_t>(count, w * chunk);
    const int64_t e = std::min<int64_t>(count, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, w, b, e] { fn(w, b, e); });
  }
  for (auto& t : pool) t.join();
}

/// scene.hpp:273-308. `workers` > 1 chunks the per-Gaussian loop (slots disjoint).
template <class S> ComposedScene<S> compose_at_time(const SceneGraph<S>& graph, S t, int workers = 1) {
  ComposedScene<S> out;
  out.graph = &graph;
  out.time = t;
  const int64_t n = graph.gaussians.n;
  out.mean_w.resize(3 * n);
  out.cov_w.resize(n);
  out.vel_dyn_w.assign(3 * n, S(0));
  out.opacity.resize(n);
  for (const auto& track : graph.tracks) out.actor_poses.push_back(interpolate_pose(track, (double)t));
  const auto& g = graph.gaussians;
  for (int64_t i = 0; i < n; ++i) {  // validation first so worker threads never throw
    const int aid = g.actor_id[i];
    if (aid < 0 || aid > (int)graph.tracks.size()) throw std::out_of_range("unknown actor_id " + std::to_string(aid));
  }
  parallel_chunks(n, workers, [&](int, int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      const V3<S> sl(g.scale_log[3 * i], g.scale_log[3 * i + 1], g.scale_log[3 * i + 2]);
      const M3<S> cov_local = covariance_from_scale_quat<S>(sl, &g.quat[4 * i]);
      const int aid = g.actor_id[i];
      out.opacity[i] = Sc<S>::sigmoid(g.opacity_logit[i]);
      if (aid == 0) {
        out.mean_w[3 * i] = g.mean[3 * i];
        out.mean_w[3 * i + 1] = g.mean[3 * i + 1];
        out.mean_w[3 * i + 2] = g.mean[3 * i + 2];
        out.cov_w[i] = cov_local;
        continue;
      }
      const auto& ip = out.actor_poses[aid - 1];
      const auto& track = graph.tracks[aid - 1];
      const M3<S> Ra = ip.pose.R.template cast<S>();
      const V3<S> ta = cast3<S>(ip.pose.t);
      const V3<S> mu_b = g.mean_at(i);
      const V3<S> mw = mul(Ra, mu_b) + ta;
      out.mean_w[3 * i] = mw.x; out.mean_w[3 * i + 1] = mw.y; out.mean_w[3 * i + 2] = mw.z;
      out.cov_w[i] = mul_nt(mul(Ra, cov_local), Ra);
      const V3<S> wa = cast3<S>(track.effective_vel_ang()), va = cast3<S>(track.effective_vel_lin());
      const V3<S> vd = mul(Ra, cross(wa, mu_b) + va);
      out.vel_dyn_w[3 * i] = vd.x; out.vel_dyn_w[3 * i + 1] = vd.y; out.vel_dyn_w[3 * i + 2] = vd.z;
    }
  });
  return out;
}

/// scene.hpp:313-323
template <class S> struct ComposeGrads {
  std::vector<S> g_mean_w;       // 3N
  std::vector<M3<S>> g_cov_w;    // N
  std::vector<S> g_vel_dyn_w;    // 3N
  void resize(int64_t n) {
    g_mean_w.assign(3 * n, S(0));
    g_cov_w.assign(n, M3<S>());
    g_vel_dyn_w.assign(3 * n, S(0));
  }
};

/// scene.hpp:325-363
template <class S> struct SceneParamGrads {
  std::vector<S> d_mean, d_scale_log, d_color, d_quat, d_opacity_logit, d_feature;
  struct ActorGrad {
    std::vector<double> d_pose_offset;  // 6 x poses
    double d_vel_offset[6] = {0, 0, 0, 0, 0, 0};
  };
  std::vector<ActorGrad> actors;
  void resize_like(const SceneGraph<S>& g) {
    const int64_t n = g.gaussians.n;
    d_mean.assign(3 * n, S(0));
    d_scale_log.assign(3 * n, S(0));
    d_color.assign(3 * n, S(0));
    d_quat.assign(4 * n, S(0));
    d_opacity_logit.assign(n, S(0));
    d_feature.assign((int64_t)g.gaussians.d_f * n, S(0));
    actors.assign(g.tracks.size(), ActorGrad());
    for (size_t a = 0; a < g.tracks.size(); ++a) actors[a].d_pose_offset.assign(6 * g.tracks[a].pose_count(), 0.0);
  }
  void add(const SceneParamGrads& o) {
    auto acc = [](std::vector<S>& a, const std::vector<S>& b) {
      for (size_t i = 0; i < a.size(); ++i) a[i] += b[i];
    };
    acc(d_mean, o.d_mean); acc(d_scale_log, o.d_scale_log); acc(d_color, o.d_color);
    acc(d_quat, o.d_quat); acc(d_opacity_logit, o.d_opacity_logit); acc(d_feature, o.d_feature);
    for (size_t a = 0; a < actors.size(); ++a) {
      for (size_t k = 0; k < actors[a].d_pose_offset.size(); ++k) actors[a].d_pose_offset[k] += o.actors[a].d_pose_offset[k];
      for (int k = 0; k < 6; ++k) actors[a].d_vel_offset[k] += o.actors[a].d_vel_offset[k];
    }
  }
};

/// scene.hpp:369-379
template <class S> V3<S> rotation_right_perturbation_grad(const M3<S>& R, const M3<S>& g_sigma, const M3<S>& sigma_local) {
  const M3<S> M = mul(mul_tn(R, S(0.5) * (g_sigma + transpose(g_sigma))), R);
  V3<S> g;
  for (int k = 0; k < 3; ++k) {
    V3<S> e;
    e[k] = S(1);
    const M3<S> E = skew(e);
    g[k] = frob(M, mul(E, sigma_local) + mul_nt(sigma_local, E));
  }
  return g;
}

/// scene.hpp:386-458. Actor slots are accumulated in double. `actors` is the shared-accumulator part
/// (scene.hpp:310-312): a threaded caller passes one per worker and reduces them in worker order.
template <class S>
void compose_backward(const ComposedScene<S>& scene, const ComposeGrads<S>& gin, const std::vector<S>& g_opacity,
                      SceneParamGrads<S>& out, std::vector<typename SceneParamGrads<S>::ActorGrad>& actors,
                      int64_t begin, int64_t end) {
  const SceneGraph<S>& graph = *scene.graph;
  const auto& gs = graph.gaussians;
  for (int64_t i = begin; i < end; ++i) {
    const int aid = gs.actor_id[i];
    const S o = scene.opacity[i];
    out.d_opacity_logit[i] += g_opacity[i] * o * (S(1) - o);
    const V3<S> sl(gs.scale_log[3 * i], gs.scale_log[3 * i + 1], gs.scale_log[3 * i + 2]);
    M3<S> g_cov_local;
    const V3<S> g_mu_w(gin.g_mean_w[3 * i], gin.g_mean_w[3 * i + 1], gin.g_mean_w[3 * i + 2]);
    if (aid == 0) {
      out.d_mean[3 * i] += g_mu_w.x; out.d_mean[3 * i + 1] += g_mu_w.y; out.d_mean[3 * i + 2] += g_mu_w.z;
      g_cov_local = gin.g_cov_w[i];
    } else {
      const auto& ip = scene.actor_poses[aid - 1];
      const auto& track = graph.tracks[aid - 1];
      auto& ag = actors[aid - 1];
      const M3<S> R = ip.pose.R.template cast<S>();
      const V3<S> mu_b = gs.mean_at(i);
      const M3<S> cov_local = covariance_from_scale_quat<S>(sl, &gs.quat[4 * i]);
      const V3<S> w_ang = cast3<S>(track.effective_vel_ang());
      const V3<S> w_body = cross(w_ang, mu_b) + cast3<S>(track.effective_vel_lin());
      // Mean (scene.hpp:412-414)
      const V3<S> Rt_g = mul_t(R, g_mu_w);
      V3<S> dm = Rt_g;
      V3<S> g_psi = cross(mu_b, Rt_g);
      // Covariance (416-418)
      g_cov_local = mul(mul_tn(R, gin.g_cov_w[i]), R);
      g_psi = g_psi + rotation_right_perturbation_grad<S>(R, gin.g_cov_w[i], cov_local);
      // Dynamic velocity (420-426)
      const V3<S> g_vw(gin.g_vel_dyn_w[3 * i], gin.g_vel_dyn_w[3 * i + 1], gin.g_vel_dyn_w[3 * i + 2]);
      const V3<S> g_w = mul_t(R, g_vw);
      g_psi = g_psi + cross(w_body, g_w);
      const V3<S> mxg = cross(mu_b, g_w);
      ag.d_vel_offset[0] += g_w.x; ag.d_vel_offset[1] += g_w.y; ag.d_vel_offset[2] += g_w.z;
      ag.d_vel_offset[3] += mxg.x; ag.d_vel_offset[4] += mxg.y; ag.d_vel_offset[5] += mxg.z;
      dm = dm + (-cross(w_ang, g_w));
      out.d_mean[3 * i] += dm.x; out.d_mean[3 * i + 1] += dm.y; out.d_mean[3 * i + 2] += dm.z;
      // Pose offsets (428-453), in double
      const V3d gmu((double)g_mu_w.x, (double)g_mu_w.y, (double)g_mu_w.z);
      const V3d gpsi((double)g_psi.x, (double)g_psi.y, (double)g_psi.z);
      auto add6 = [&](int64_t col, V3d tr, V3d rot) {
        double* p = &ag.d_pose_offset[6 * col];
        p[0] += tr.x; p[1] += tr.y; p[2] += tr.z; p[3] += rot.x; p[4] += rot.y; p[5] += rot.z;
      };
      if (track.pose_count() == 1) {
        const M3d Jr0 = so3_right_jacobian(track.off_r(0));
        add6(0, gmu, mul_t(Jr0, gpsi));
      } else {
        const double u = ip.u;
        const V3d phi = ip.geo;
        const M3d Jr_u = so3_right_jacobian(u * phi);
        const M3d B0 = transpose(so3_exp(u * phi)) - u * mul(Jr_u, so3_left_jacobian_inv(phi));
        const M3d B1 = u * mul(Jr_u, so3_right_jacobian_inv(phi));
        const M3d Jr0 = so3_right_jacobian(track.off_r(ip.i0));
        const M3d Jr1 = so3_right_jacobian(track.off_r(ip.i1));
        add6(ip.i0, (1.0 - u) * gmu, mul_t(Jr0, mul_t(B0, gpsi)));
        add6(ip.i1, u * gmu, mul_t(Jr1, mul_t(B1, gpsi)));
      }
    }
    covariance_backward<S>(sl, &gs.quat[4 * i], g_cov_local, &out.d_scale_log[3 * i], &out.d_quat[4 * i]);
  }
}

/// Reference signature (scene.hpp:386-389).
template <class S>
void compose_backward(const ComposedScene<S>& scene, const ComposeGrads<S>& gin, const std::vector<S>& g_opacity,
                      SceneParamGrads<S>& out, int64_t begin, int64_t end) {
  compose_backward<S>(scene, gin, g_opacity, out, out.actors, begin, end);
}

// ----------------------------------------------------------------------------
// projection.hpp
// ----------------------------------------------------------------------------
/// projection.hpp:7-15
template <class S> struct RasterSettings {
  S dilation = S(0.3);
  S alpha_clamp = S(0.999);
  S alpha_min = S(1) / S(255);
  S qform_max = S(9);
  S transmittance_min = S(1e-4);
  S near_plane = S(0.05);
  S lidar_min_range = S(0.25);
};

/// projection.hpp:28-40 (aabb = projection.hpp:17-23). cov2d/conic row-major 2x2.
template <class S> struct Projected {
  int64_t source_index = 0;
  S mean2d[2] = {0, 0};
  S depth_key = 0;
  S cov2d[4] = {0, 0, 0, 0};
  S velocity[3] = {0, 0, 0};
  S aabb_lo[2] = {0, 0}, aabb_hi[2] = {0, 0};
  S conic[4] = {0, 0, 0, 0};
  S det_ratio = 1;
  S mu_sensor[3] = {0, 0, 0};
  S rel_vel_sensor[3] = {0, 0, 0};
};

/// projection.hpp:44-48
template <class S> V3<S> relative_velocity_sensor(V3<S> mu, V3<S> vel_lin, V3<S> vel_ang, V3<S> v_dyn_sensor) {
  return (-cross(vel_ang, mu) - vel_lin) + v_dyn_sensor;
}

/// projection.hpp:62-71
template <class S> void velocity_expanded_aabb(Projected<S>& g, S dilation, S shutter) {
  const S hx = S(3) * Sc<S>::sqrt(std::max(S(0), g.cov2d[0] + dilation)) + Sc<S>::abs(g.velocity[0]) * shutter / S(2);
  const S hy = S(3) * Sc<S>::sqrt(std::max(S(0), g.cov2d[3] + dilation)) + Sc<S>::abs(g.velocity[1]) * shutter / S(2);
  g.aabb_lo[0] = g.mean2d[0] - hx; g.aabb_lo[1] = g.mean2d[1] - hy;
  g.aabb_hi[0] = g.mean2d[0] + hx; g.aabb_hi[1] = g.mean2d[1] + hy;
}

/// projection.hpp:75-84 (+ Eigen's closed-form 2x2 determinant / inverse)
template <class S> bool finalize_footprint(Projected<S>& g, S dilation) {
  const S det = g.cov2d[0] * g.cov2d[3] - g.cov2d[2] * g.cov2d[1];
  const S d00 = g.cov2d[0] + dilation, d11 = g.cov2d[3] + dilation, d01 = g.cov2d[1], d10 = g.cov2d[2];
  const S det_dilated = d00 * d11 - d10 * d01;
  if (!(det > S(0)) || !(det_dilated > S(0))) return false;
  const S invdet = S(1) / det_dilated;
  g.conic[0] = d11 * invdet;
  g.conic[1] = -d01 * invdet;
  g.conic[2] = -d10 * invdet;
  g.conic[3] = d00 * invdet;
  g.det_ratio = Sc<S>::sqrt(det / det_dilated);
  return true;
}

/// J (rows x 3) * C (3x3) * J^T, left to right, as Eigen evaluates `J * cov * J.transpose()`.
template <class S, int ROWS> void jcjt(const S J[ROWS][3], const M3<S>& C, S out[ROWS][ROWS]) {
  S JC[ROWS][3];
  for (int i = 0; i < ROWS; ++i)
    for (int j = 0; j < 3; ++j) JC[i][j] = (J[i][0] * C(0, j) + J[i][1] * C(1, j)) + J[i][2] * C(2, j);
  for (int i = 0; i < ROWS; ++i)
    for (int j = 0; j < ROWS; ++j) out[i][j] = (JC[i][0] * J[j][0] + JC[i][1] * J[j][1]) + JC[i][2] * J[j][2];
}

/// scene.hpp:112-117
template <class S> void camera_jacobian(const CameraModel<S>& cam, V3<S> p, S J[2][3]) {
  const S iz = S(1) / p.z;
  J[0][0] = cam.fx * iz; J[0][1] = S(0); J[0][2] = -cam.fx * p.x * iz * iz;
  J[1][0] = S(0); J[1][1] = cam.fy * iz; J[1][2] = -cam.fy * p.y * iz * iz;
}

/// projection.hpp:88-118 — one Gaussian; returns false when culled.
template <class S>
bool project_camera_one(const ComposedScene<S>& scene, const CameraModel<S>& cam, const RasterSettings<S>& st, int64_t i,
                        Projected<S>& g) {
  const M3<S>& R = cam.pose.R;
  const V3<S> mu_c = cam.pose.apply(scene.mean_at(i));
  if (mu_c.z <= st.near_plane) return false;
  g = Projected<S>();
  g.source_index = i;
  g.mu_sensor[0] = mu_c.x; g.mu_sensor[1] = mu_c.y; g.mu_sensor[2] = mu_c.z;
  g.depth_key = mu_c.z;
  g.mean2d[0] = cam.fx * mu_c.x / mu_c.z + cam.cx;  // scene.hpp:109-111
  g.mean2d[1] = cam.fy * mu_c.y / mu_c.z + cam.cy;
  S J[2][3];
  camera_jacobian(cam, mu_c, J);
  const M3<S> cov_c = mul_nt(mul(R, scene.cov_w[i]), R);
  S c2[2][2];
  jcjt<S, 2>(J, cov_c, c2);
  g.cov2d[0] = c2[0][0]; g.cov2d[1] = c2[0][1]; g.cov2d[2] = c2[1][0]; g.cov2d[3] = c2[1][1];
  if (!finalize_footprint(g, st.dilation)) return false;
  const V3<S> u = relative_velocity_sensor<S>(mu_c, cam.vel_lin, cam.vel_ang, mul(R, scene.vel_at(i)));
  g.rel_vel_sensor[0] = u.x; g.rel_vel_sensor[1] = u.y; g.rel_vel_sensor[2] = u.z;
  g.velocity[0] = (J[0][0] * u.x + J[0][1] * u.y) + J[0][2] * u.z;  // projection.hpp:50-53
  g.velocity[1] = (J[1][0] * u.x + J[1][1] * u.y) + J[1][2] * u.z;
  velocity_expanded_aabb(g, st.dilation, cam.shutter_duration);
  // projection.hpp:19-22, 114
  const S W = S(cam.width), H = S(cam.height);
  if (!(g.aabb_lo[0] < W && g.aabb_hi[0] > S(0) && g.aabb_lo[1] < H && g.aabb_hi[1] > S(0))) return false;
  return true;
}

template <class S>
std::vector<Projected<S>> project_camera(const ComposedScene<S>& scene, const CameraModel<S>& cam,
                                         const RasterSettings<S>& st, int workers = 1) {
  const int64_t n = scene.size();
  std::vector<std::vector<Projected<S>>> parts(std::max(1, workers));
  parallel_chunks(n, workers, [&](int w, int64_t b, int64_t e) {
    auto& out = parts[w];
    out.reserve(e - b);
    Projected<S> g;
    for (int64_t i = b; i < e; ++i)
      if (project_camera_one(scene, cam, st, i, g)) out.push_back(g);
  });
  std::vector<Projected<S>> out;
  for (auto& p : parts) out.insert(out.end(), p.begin(), p.end());  // worker order => ascending source_index
  return out;
}

/// projection.hpp:127-138 (Eq. 11)
template <class S> void spherical_jacobian(V3<S> p, S J[3][3]) {
  const S x = p.x, y = p.y, z = p.z;
  const S d2 = x * x + y * y;
  const S d = Sc<S>::sqrt(d2);
  const S r2 = d2 + z * z;
  const S r = Sc<S>::sqrt(r2);
  J[0][0] = -y / d2; J[0][1] = x / d2; J[0][2] = S(0);
  J[1][0] = -x * z / (r2 * d); J[1][1] = -y * z / (r2 * d); J[1][2] = d / r2;
  J[2][0] = x / r; J[2][1] = y / r; J[2][2] = z / r;
}

/// projection.hpp:140-174 — one Gaussian.
template <class S>
bool project_lidar_one(const ComposedScene<S>& scene, const LidarModel<S>& lidar, const RasterSettings<S>& st, int64_t i,
                       Projected<S>& g) {
  const M3<S>& R = lidar.pose.R;
  const S elev_min = lidar.elevation_channels.front();
  const S elev_max = lidar.elevation_channels.back();
  const S s = lidar.dilation();
  const V3<S> mu_l = lidar.pose.apply(scene.mean_at(i));
  const S d2 = mu_l.x * mu_l.x + mu_l.y * mu_l.y;
  if (d2 < st.lidar_min_range * st.lidar_min_range) return false;
  // spherical_of, projection.hpp:122-125
  const S r = Sc<S>::sqrt((mu_l.x * mu_l.x + mu_l.y * mu_l.y) + mu_l.z * mu_l.z);
  const S phi = wrap_two_pi(Sc<S>::atan2(mu_l.y, mu_l.x));
  const S omega = Sc<S>::asin(mu_l.z / r);
  if (r < st.lidar_min_range) return false;
  g = Projected<S>();
  g.source_index = i;
  g.mu_sensor[0] = mu_l.x; g.mu_sensor[1] = mu_l.y; g.mu_sensor[2] = mu_l.z;
  g.depth_key = r;
  g.mean2d[0] = phi; g.mean2d[1] = omega;
  S J[3][3];
  spherical_jacobian(mu_l, J);
  const M3<S> cov_l = mul_nt(mul(R, scene.cov_w[i]), R);
  S c3[3][3];
  jcjt<S, 3>(J, cov_l, c3);
  g.cov2d[0] = c3[0][0]; g.cov2d[1] = c3[0][1]; g.cov2d[2] = c3[1][0]; g.cov2d[3] = c3[1][1];
  if (!finalize_footprint(g, s)) return false;
  const V3<S> u = relative_velocity_sensor<S>(mu_l, lidar.vel_lin, lidar.vel_ang, mul(R, scene.vel_at(i)));
  g.rel_vel_sensor[0] = u.x; g.rel_vel_sensor[1] = u.y; g.rel_vel_sensor[2] = u.z;
  for (int k = 0; k < 3; ++k) g.velocity[k] = (J[k][0] * u.x + J[k][1] * u.y) + J[k][2] * u.z;
  velocity_expanded_aabb(g, s, lidar.scan_duration);
  if (g.aabb_hi[1] < elev_min || g.aabb_lo[1] > elev_max) return false;
  return true;
}

template <class S>
std::vector<Projected<S>> project_lidar(const ComposedScene<S>& scene, const LidarModel<S>& lidar,
                                        const RasterSettings<S>& st, int workers = 1) {
  const int64_t n = scene.size();
  std::vector<std::vector<Projected<S>>> parts(std::max(1, workers));
  parallel_chunks(n, workers, [&](int w, int64_t b, int64_t e) {
    auto& out = parts[w];
    out.reserve(e - b);
    Projected<S> g;
    for (int64_t i = b; i < e; ++i)
      if (project_lidar_one(scene, lidar, st, i, g)) out.push_back(g);
  });
  std::vector<Projected<S>> out;
  for (auto& p : parts) out.insert(out.end(), p.begin(), p.end());
  return out;
}

/// projection.hpp:178-205. All arrays are indexed by SOURCE Gaussian index
/// (the header's stated convention, projection.hpp:176-177; see DESIGN.md on
/// the k-vs-i inconsistency in the shipped consumers).
template <class S> struct ProjectedGrads {
  int64_t n = 0;
  int d_f = 0;
  std::vector<S> g_mean2d, g_range, g_cov2d, g_velocity, g_opacity, g_color, g_feature;
  void resize(int64_t n_, int d_f_) {
    n = n_; d_f = d_f_;
    g_mean2d.assign(2 * n, S(0)); g_range.assign(n, S(0)); g_cov2d.assign(4 * n, S(0));
    g_velocity.assign(3 * n, S(0)); g_opacity.assign(n, S(0)); g_color.assign(3 * n, S(0));
    g_feature.assign((int64_t)d_f * n, S(0));
  }
};

/// projection.hpp:207-222 (embedding grads belong to the decoder; out of scope)
template <class S> struct SensorGrads {
  S d_vel_lin[3] = {0, 0, 0};
  S d_vel_ang[3] = {0, 0, 0};
  S d_time_offset = 0;
};

/// projection.hpp:237-246
template <class S>
void velocity_chain_backward(V3<S> mu, V3<S> vel_ang, const M3<S>& R, V3<S> g_u, bool dynamic, V3<S>& g_mu,
                             SensorGrads<S>& sg, V3<S>* g_vel_dyn_w) {
  const V3<S> c = cross(mu, g_u);
  sg.d_vel_ang[0] += -c.x; sg.d_vel_ang[1] += -c.y; sg.d_vel_ang[2] += -c.z;
  sg.d_vel_lin[0] += -g_u.x; sg.d_vel_lin[1] += -g_u.y; sg.d_vel_lin[2] += -g_u.z;
  g_mu = g_mu + cross(vel_ang, g_u);
  if (dynamic && g_vel_dyn_w) *g_vel_dyn_w = *g_vel_dyn_w + mul_t(R, g_u);
}

/// projection.hpp:250-288
template <class S>
void project_camera_backward(const ComposedScene<S>& scene, const CameraModel<S>& cam,
                             const std::vector<Projected<S>>& projected, const ProjectedGrads<S>& gin,
                             ComposeGrads<S>& gscene, SensorGrads<S>& gsensor, int64_t begin, int64_t end) {
  const M3<S>& R = cam.pose.R;
  for (int64_t k = begin; k < end; ++k) {
    const auto& g = projected[k];
    const int64_t i = g.source_index;
    const bool dynamic = scene.graph->gaussians.actor_id[i] != 0;
    const V3<S> mu_c(g.mu_sensor[0], g.mu_sensor[1], g.mu_sensor[2]);
    S J[2][3];
    camera_jacobian(cam, mu_c, J);
    const M3<S> cov_c = mul_nt(mul(R, scene.cov_w[i]), R);
    const S* gc = &gin.g_cov2d[4 * i];
    const S G2[2][2] = {{gc[0], S(0.5) * (gc[1] + gc[2])}, {S(0.5) * (gc[1] + gc[2]), gc[3]}};
    const S gm[2] = {gin.g_mean2d[2 * i], gin.g_mean2d[2 * i + 1]};
    V3<S> g_mu_c(J[0][0] * gm[0] + J[1][0] * gm[1], J[0][1] * gm[0] + J[1][1] * gm[1], J[0][2] * gm[0] + J[1][2] * gm[1]);
    // g_cov_c = J^T G2 J
    S G2J[2][3];
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c) G2J[a][c] = G2[a][0] * J[0][c] + G2[a][1] * J[1][c];
    M3<S> g_cov_c;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) g_cov_c(a, c) = J[0][a] * G2J[0][c] + J[1][a] * G2J[1][c];
    const S gv[2] = {gin.g_velocity[3 * i], gin.g_velocity[3 * i + 1]};
    // g_J = 2 G2 J cov_c + g_v2d rel_vel^T
    S g_J[2][3];
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 3; ++c)
        g_J[a][c] = S(2) * ((G2J[a][0] * cov_c(0, c) + G2J[a][1] * cov_c(1, c)) + G2J[a][2] * cov_c(2, c)) +
                    gv[a] * g.rel_vel_sensor[c];
    const S z = mu_c.z, iz2 = S(1) / (z * z), iz3 = iz2 / z;
    g_mu_c.x += -cam.fx * iz2 * g_J[0][2];
    g_mu_c.y += -cam.fy * iz2 * g_J[1][2];
    g_mu_c.z += -cam.fx * iz2 * g_J[0][0] - cam.fy * iz2 * g_J[1][1] + S(2) * cam.fx * mu_c.x * iz3 * g_J[0][2] +
                S(2) * cam.fy * mu_c.y * iz3 * g_J[1][2];
    const V3<S> g_u(J[0][0] * gv[0] + J[1][0] * gv[1], J[0][1] * gv[0] + J[1][1] * gv[1], J[0][2] * gv[0] + J[1][2] * gv[1]);
    V3<S> g_vdyn;
    velocity_chain_backward<S>(mu_c, cam.vel_ang, R, g_u, dynamic, g_mu_c, gsensor, &g_vdyn);
    if (dynamic) {
      gscene.g_vel_dyn_w[3 * i] += g_vdyn.x; gscene.g_vel_dyn_w[3 * i + 1] += g_vdyn.y; gscene.g_vel_dyn_w[3 * i + 2] += g_vdyn.z;
    }
    const V3<S> gw = mul_t(R, g_mu_c);
    gscene.g_mean_w[3 * i] += gw.x; gscene.g_mean_w[3 * i + 1] += gw.y; gscene.g_mean_w[3 * i + 2] += gw.z;
    gscene.g_cov_w[i] = gscene.g_cov_w[i] + mul(mul_tn(R, g_cov_c), R);
  }
}

/// projection.hpp:294-318
template <class S> V3<S> spherical_jacobian_point_grad(V3<S> p, const S g_J[3][3]) {
  const S x = p.x, y = p.y, z = p.z;
  const S D2 = x * x + y * y;
  const S D = Sc<S>::sqrt(D2);
  const S D3 = D2 * D, D4 = D2 * D2;
  const S R2 = D2 + z * z;
  const S R1 = Sc<S>::sqrt(R2);
  const S R3 = R2 * R1, R4 = R2 * R2;
  const S dJx[9] = {S(2) * x * y / D4, (y * y - x * x) / D4, S(0),
                    z * (-D2 * R2 + S(2) * D2 * x * x + R2 * x * x) / (D3 * R4),
                    x * y * z * (S(3) * D2 + z * z) / (D3 * R4), x * (z * z - D2) / (D * R4),
                    (y * y + z * z) / R3, -x * y / R3, -x * z / R3};
  const S dJy[9] = {(y * y - x * x) / D4, S(-2) * x * y / D4, S(0),
                    x * y * z * (S(3) * D2 + z * z) / (D3 * R4),
                    z * (-D2 * R2 + S(2) * D2 * y * y + R2 * y * y) / (D3 * R4), y * (z * z - D2) / (D * R4),
                    -x * y / R3, (x * x + z * z) / R3, -y * z / R3};
  const S dJz[9] = {S(0), S(0), S(0), x * (z * z - D2) / (D * R4), y * (z * z - D2) / (D * R4),
                    S(-2) * D * z / R4, -x * z / R3, -y * z / R3, D2 / R3};
  V3<S> o;
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      o.x += g_J[a][c] * dJx[3 * a + c];
      o.y += g_J[a][c] * dJy[3 * a + c];
      o.z += g_J[a][c] * dJz[3 * a + c];
    }
  return o;
}

/// projection.hpp:322-357
template <class S>
void project_lidar_backward(const ComposedScene<S>& scene, const LidarModel<S>& lidar,
                            const std::vector<Projected<S>>& projected, const ProjectedGrads<S>& gin,
                            ComposeGrads<S>& gscene, SensorGrads<S>& gsensor, int64_t begin, int64_t end) {
  const M3<S>& R = lidar.pose.R;
  for (int64_t k = begin; k < end; ++k) {
    const auto& g = projected[k];
    const int64_t i = g.source_index;
    const bool dynamic = scene.graph->gaussians.actor_id[i] != 0;
    const V3<S> mu_l(g.mu_sensor[0], g.mu_sensor[1], g.mu_sensor[2]);
    S J[3][3];
    spherical_jacobian(mu_l, J);
    const M3<S> cov_l = mul_nt(mul(R, scene.cov_w[i]), R);
    const S* gc = &gin.g_cov2d[4 * i];
    S G3[3][3] = {{gc[0], S(0.5) * (gc[1] + gc[2]), S(0)}, {S(0.5) * (gc[1] + gc[2]), gc[3], S(0)}, {S(0), S(0), S(0)}};
    const S g_sph[3] = {gin.g_mean2d[2 * i], gin.g_mean2d[2 * i + 1], gin.g_range[i]};
    V3<S> g_mu_l;
    for (int c = 0; c < 3; ++c) g_mu_l[c] = (J[0][c] * g_sph[0] + J[1][c] * g_sph[1]) + J[2][c] * g_sph[2];
    S G3J[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) G3J[a][c] = (G3[a][0] * J[0][c] + G3[a][1] * J[1][c]) + G3[a][2] * J[2][c];
    M3<S> g_cov_l;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) g_cov_l(a, c) = (J[0][a] * G3J[0][c] + J[1][a] * G3J[1][c]) + J[2][a] * G3J[2][c];
    const S gv[3] = {gin.g_velocity[3 * i], gin.g_velocity[3 * i + 1], gin.g_velocity[3 * i + 2]};
    S g_J[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c)
        g_J[a][c] = S(2) * ((G3J[a][0] * cov_l(0, c) + G3J[a][1] * cov_l(1, c)) + G3J[a][2] * cov_l(2, c)) +
                    gv[a] * g.rel_vel_sensor[c];
    g_mu_l = g_mu_l + spherical_jacobian_point_grad<S>(mu_l, g_J);
    V3<S> g_u;
    for (int c = 0; c < 3; ++c) g_u[c] = (J[0][c] * gv[0] + J[1][c] * gv[1]) + J[2][c] * gv[2];
    V3<S> g_vdyn;
    velocity_chain_backward<S>(mu_l, lidar.vel_ang, R, g_u, dynamic, g_mu_l, gsensor, &g_vdyn);
    if (dynamic) {
      gscene.g_vel_dyn_w[3 * i] += g_vdyn.x; gscene.g_vel_dyn_w[3 * i + 1] += g_vdyn.y; gscene.g_vel_dyn_w[3 * i + 2] += g_vdyn.z;
    }
    const V3<S> gw = mul_t(R, g_mu_l);
    gscene.g_mean_w[3 * i] += gw.x; gscene.g_mean_w[3 * i + 1] += gw.y; gscene.g_mean_w[3 * i + 2] += gw.z;
    gscene.g_cov_w[i] = gscene.g_cov_w[i] + mul(mul_tn(R, g_cov_l), R);
  }
}

// ----------------------------------------------------------------------------
// tiling — no reference source exists
// ----------------------------------------------------------------------------
constexpr int kTile = 16;
constexpr int kNphi = 32;
constexpr int kNomega = 8;

struct TileRect {
  int x0 = 0, x1 = 0, y0 = 0, y1 = 0;  // inclusive-exclusive; lidar x may be negative / exceed M_phi before wrapping
  int64_t count() const { return (int64_t)std::max(0, x1 - x0) * std::max(0, y1 - y0); }
};

/// SPEC.md:190-198
template <class S> TileRect image_tile_range(const S lo[2], const S hi[2], int tiles_x, int tiles_y) {
  auto cl = [](S v, int m) { return (int)std::min(std::max(v, S(0)), S(m)); };
  TileRect r;
  r.x0 = cl(Sc<S>::floor(lo[0] / S(kTile)), tiles_x);
  r.x1 = cl(Sc<S>::ceil(hi[0] / S(kTile)), tiles_x);
  r.y0 = cl(Sc<S>::floor(lo[1] / S(kTile)), tiles_y);
  r.y1 = cl(Sc<S>::ceil(hi[1] / S(kTile)), tiles_y);
  return r;
}

/// Lidar tile grid, SPEC.md:181 / PAPER.md:446-452.
template <class S> struct LidarGrid {
  S span = 0;      // N_phi * res_phi
  S phi_max = 0;   // M_phi * span  (>= 2 pi)
  int m_phi = 0, m_omega = 0;
  std::vector<S> boundaries;  // m_omega - 1 interior row boundaries, midway between channels 8k-1 and 8k
};
template <class S> LidarGrid<S> make_lidar_grid(const LidarModel<S>& l) {
  LidarGrid<S> g;
  g.span = S(kNphi) * l.azimuth_resolution;
  // M_phi = ceil(360deg / span); evaluated in double with a 1e-4-tile guard so that
  // resolutions that divide the circle exactly do not spawn a sliver column from fp32 rounding of res_phi.
  g.m_phi = (int)std::ceil(6.283185307179586476925 / ((double)kNphi * (double)l.azimuth_resolution) - 1e-4);
  g.phi_max = S(g.m_phi) * g.span;
  const int nb = l.beam_count();
  g.m_omega = (nb + kNomega - 1) / kNomega;
  for (int k = 1; k < g.m_omega; ++k)
    g.boundaries.push_back(S(0.5) * (l.elevation_channels[kNomega * k - 1] + l.elevation_channels[kNomega * k]));
  return g;
}

/// PAPER.md:466-488. Returns [x0, x1) un-wrapped; emitted column = (x + M) mod M.
/// Full-circle AABBs (count >= M_phi) are capped to every column once (paper silent).
template <class S> void lidar_azimuth_tile_range(S phi_lo, S phi_hi, const LidarGrid<S>& g, int& x0, int& x1) {
  const S lim = S(4) * S(g.m_phi);  // clamp before int conversion
  S fl, fh;
  if (phi_lo >= S(0)) fl = Sc<S>::floor(phi_lo / g.span);
  else fl = Sc<S>::floor(((phi_lo + two_pi<S>()) - g.phi_max) / g.span);
  if (phi_hi <= two_pi<S>()) fh = Sc<S>::ceil(phi_hi / g.span);
  else fh = Sc<S>::ceil(Sc<S>::fmod(phi_hi, two_pi<S>()) / g.span) + S(g.m_phi);
  fl = std::min(std::max(fl, -lim), lim);
  fh = std::min(std::max(fh, -lim), lim);
  x0 = (int)fl;
  x1 = (int)fh;
  if (x1 - x0 >= g.m_phi) {
    x0 = 0;
    x1 = g.m_phi;
  }
}

/// PAPER.md:490. Rows r = [B_r, B_{r+1}) with B_0 = -inf, B_M = +inf.
template <class S> void lidar_elevation_tile_range(S om_lo, S om_hi, const LidarGrid<S>& g, int& y0, int& y1) {
  y0 = 0;
  y1 = 1;
  for (size_t k = 0; k < g.boundaries.size(); ++k) {
    if (g.boundaries[k] < om_lo) y0 = (int)k + 1;   // last boundary smaller than om_lo
    if (g.boundaries[k] <= om_hi) y1 = (int)k + 2;  // first boundary larger than om_hi is k+1 past these
  }
}

template <class S> TileRect lidar_tile_range(const S lo[2], const S hi[2], const LidarGrid<S>& g) {
  TileRect r;
  lidar_azimuth_tile_range(lo[0], hi[0], g, r.x0, r.x1);
  lidar_elevation_tile_range(lo[1], hi[1], g, r.y0, r.y1);
  return r;
}

// ----------------------------------------------------------------------------
// decode_lidar (§3.3, Appendix B) — no reference source exists
// ----------------------------------------------------------------------------
/// LidarHead: 2 layers, hidden 32, input = D_f blended features + 3 (ray direction in the sensor frame), outputs
/// intensity and ray-drop probability through logistic activations, rectified-linear inside.
/// Parameter block (row-major): W1 [32 x (d_f + 3)], b1 [32], W2 [2 x 32], b2 [2].
constexpr int kHeadHidden = 32;
inline int lidar_head_params(int d_f) { return kHeadHidden * (d_f + 3) + kHeadHidden + 2 * kHeadHidden + 2; }

template <class S> void ray_direction_sensor(S phi, S omega, S d[3]) {
  const S co = Sc<S>::cos(omega);
  d[0] = co * Sc<S>::cos(phi); d[1] = co * Sc<S>::sin(phi); d[2] = Sc<S>::sin(omega);
}

/// One ray. x = (features, direction); h = relu(W1 x + b1); y = sigmoid(W2 h + b2). Returns h for the backward.
template <class S> void lidar_head_forward_one(const S* w, int d_f, const S* feat, const S dir[3], S y[2], S h[kHeadHidden]) {
  const int in = d_f + 3;
  const S* W1 = w; const S* b1 = W1 + kHeadHidden * in; const S* W2 = b1 + kHeadHidden; const S* b2 = W2 + 2 * kHeadHidden;
  for (int j = 0; j < kHeadHidden; ++j) {
    S a = b1[j];
    for (int k = 0; k < d_f; ++k) a = Sc<S>::fma(W1[j * in + k], feat[k], a);
    for (int k = 0; k < 3; ++k) a = Sc<S>::fma(W1[j * in + d_f + k], dir[k], a);
    h[j] = a > S(0) ? a : S(0);
  }
  for (int o = 0; o < 2; ++o) {
    S a = b2[o];
    for (int j = 0; j < kHeadHidden; ++j) a = Sc<S>::fma(W2[o * kHeadHidden + j], h[j], a);
    y[o] = Sc<S>::sigmoid(a);
  }
}

/// Backward of one ray: accumulates the parameter gradients into gw (same layout as w) and returns dL/dfeat.
template <class S>
void lidar_head_backward_one(const S* w, int d_f, const S* feat, const S dir[3], const S g_y[2], S* gw, S* g_feat) {
  const int in = d_f + 3;
  const S* W1 = w; const S* b1 = W1 + kHeadHidden * in; const S* W2 = b1 + kHeadHidden;
  S* gW1 = gw; S* gb1 = gW1 + kHeadHidden * in; S* gW2 = gb1 + kHeadHidden; S* gb2 = gW2 + 2 * kHeadHidden;
  S y[2], h[kHeadHidden];
  lidar_head_forward_one<S>(w, d_f, feat, dir, y, h);
  S gp2[2];
  for (int o = 0; o < 2; ++o) {
    gp2[o] = g_y[o] * y[o] * (S(1) - y[o]);
    gb2[o] += gp2[o];
    for (int j = 0; j < kHeadHidden; ++j) gW2[o * kHeadHidden + j] += gp2[o] * h[j];
  }
  for (int k = 0; k < d_f; ++k) g_feat[k] = S(0);
  for (int j = 0; j < kHeadHidden; ++j) {
    if (!(h[j] > S(0))) continue;
    const S gp1 = W2[j] * gp2[0] + W2[kHeadHidden + j] * gp2[1];
    gb1[j] += gp1;
    for (int k = 0; k < d_f; ++k) { gW1[j * in + k] += gp1 * feat[k]; g_feat[k] += W1[j * in + k] * gp1; }
    for (int k = 0; k < 3; ++k) gW1[j * in + d_f + k] += gp1 * dir[k];
  }
}

// ----------------------------------------------------------------------------
// assign_points_to_tiles — no reference source exists
// ----------------------------------------------------------------------------
/// Result of mapping lidar returns to rasterization points. Per INPUT point: tile (-1 if rejected), spherical
/// coordinates relative to the sensor pose at the point's own capture time (Eq. 10 after ego-motion removal), the
/// capture-time offset t_l and the measured range. `order` lists the kept points tile-major (eval: ascending input
/// index inside a tile; train: ascending (hash, index), at most 256 per tile), `begin/end` are its per-tile slices.
template <class S> struct AssignedPoints {
  std::vector<int64_t> tile;
  std::vector<S> phi, omega, t_l, range;
  std::vector<int64_t> order, begin, end;
  int64_t rejected = 0, dropped = 0;
  int tiles_x = 0, tiles_y = 0;
};

/// The "seeded shuffle" of PAPER.md:512 (SPEC open question: tie-breaking undefined): a point keeps its place in a
/// full tile iff its hash is among the 256 smallest of the tile. Counter-based, so any implementation reproduces it.
inline uint32_t point_hash(uint32_t seed, uint32_t index) {
  uint32_t h = index * 0x9E3779B9u + seed;
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;  // murmur3 finaliser
  return h;
}

constexpr int kPointsPerTile = kNphi * kNomega;  // 256

/// One point: sensor-frame position at scan centre -> position at its own capture time under the constant-velocity
/// assumption (the same first-order motion model the rasterizer applies to Gaussians: u = -w x p - v,
/// projection.hpp:44-48) -> Eq. 10 (projection.hpp:122-125) -> the tile holding that zero-extent location
/// (column floor(phi / span); row = number of row boundaries below omega: a point on an edge belongs to the floor
/// tile). Returns false for non-finite input or a point at the sensor origin.
template <class S>
bool assign_one_point(const S* xyz_world, S stamp, const LidarModel<S>& lidar, const LidarGrid<S>& g, int64_t& tile, S& phi,
                      S& omega, S& t_l, S& range) {
  tile = -1; phi = omega = t_l = range = S(0);
  if (!(std::isfinite(xyz_world[0]) && std::isfinite(xyz_world[1]) && std::isfinite(xyz_world[2]) && std::isfinite(stamp)))
    return false;
  const V3<S> p0 = lidar.pose.apply(V3<S>{xyz_world[0], xyz_world[1], xyz_world[2]});
  t_l = stamp - lidar.timestamp;
  const V3<S> u = relative_velocity_sensor<S>(p0, lidar.vel_lin, lidar.vel_ang, V3<S>{S(0), S(0), S(0)});
  const V3<S> p{p0.x + u.x * t_l, p0.y + u.y * t_l, p0.z + u.z * t_l};
  const S r = Sc<S>::sqrt((p.x * p.x + p.y * p.y) + p.z * p.z);
  if (!(r > S(0)) || !std::isfinite(r)) return false;
  phi = wrap_two_pi(Sc<S>::atan2(p.y, p.x));
  omega = Sc<S>::asin(p.z / r);
  range = r;
  int col = (int)Sc<S>::floor(phi / g.span);
  col = std::min(std::max(col, 0), g.m_phi - 1);
  int row = 0;
  for (size_t k = 0; k < g.boundaries.size(); ++k)
    if (g.boundaries[k] < omega) row = (int)k + 1;
  tile = (int64_t)row * g.m_phi + col;
  return true;
}

template <class S>
AssignedPoints<S> assign_points_to_tiles(const S* xyz_world, const S* stamps, int64_t n, const LidarModel<S>& lidar,
                                         bool train, uint32_t seed) {
  AssignedPoints<S> a;
  const LidarGrid<S> g = make_lidar_grid<S>(lidar);
  a.tiles_x = g.m_phi; a.tiles_y = g.m_omega;
  const int64_t T = (int64_t)g.m_phi * g.m_omega;
  a.tile.resize(n); a.phi.resize(n); a.omega.resize(n); a.t_l.resize(n); a.range.resize(n);
  std::vector<std::vector<int64_t>> per_tile((size_t)T);
  for (int64_t i = 0; i < n; ++i) {
    if (assign_one_point<S>(xyz_world + 3 * i, stamps[i], lidar, g, a.tile[i], a.phi[i], a.omega[i], a.t_l[i], a.range[i]))
      per_tile[(size_t)a.tile[i]].push_back(i);
    else
      ++a.rejected;
  }
  a.begin.assign((size_t)T, 0); a.end.assign((size_t)T, 0);
  for (int64_t t = 0; t < T; ++t) {
    auto& v = per_tile[(size_t)t];
    if (train) {  // "shuffle points ... and discard any points beyond 256"
      std::stable_sort(v.begin(), v.end(), [&](int64_t x, int64_t y) {
        return point_hash(seed, (uint32_t)x) < point_hash(seed, (uint32_t)y);
      });
      if ((int64_t)v.size() > kPointsPerTile) {
        a.dropped += (int64_t)v.size() - kPointsPerTile;
        v.resize(kPointsPerTile);
      }
    }
    a.begin[(size_t)t] = (int64_t)a.order.size();
    a.order.insert(a.order.end(), v.begin(), v.end());
    a.end[(size_t)t] = (int64_t)a.order.size();
  }
  return a;
}

/// Sort key: tile id major, IEEE bits of the (positive) fp32 depth minor — the
/// 64-bit key the device radix sort uses. In fp64 mode the depth is compared as a double.
struct Isect {
  uint32_t tile;
  uint32_t depth_bits;  // fp32 mode
  double depth;         // ordering value
  int64_t src;          // source index
  int32_t pidx;         // position in projected list
};

struct Worklist {
  std::vector<Isect> items;            // sorted by (tile, depth, src)
  std::vector<int64_t> tile_begin, tile_end;
  int tiles_x = 0, tiles_y = 0;
};

/// stable sort on (tile_id, depth_key, source_index).
template <class S, class RectFn>
Worklist build_sorted_worklist(const std::vector<Projected<S>>& projected, int tiles_x, int tiles_y, bool wrap_x,
                               RectFn rect_of) {
  Worklist w;
  w.tiles_x = tiles_x; w.tiles_y = tiles_y;
  for (size_t k = 0; k < projected.size(); ++k) {
    const auto& g = projected[k];
    const TileRect r = rect_of(g);
    for (int y = r.y0; y < r.y1; ++y)
      for (int x = r.x0; x < r.x1; ++x) {
        const int xc = wrap_x ? ((x % tiles_x) + tiles_x) % tiles_x : x;
        Isect it;
        it.tile = (uint32_t)(y * tiles_x + xc);
        const float df = (float)g.depth_key;
        std::memcpy(&it.depth_bits, &df, 4);
        it.depth = (double)g.depth_key;
        it.src = g.source_index;
        it.pidx = (int32_t)k;
        w.items.push_back(it);
      }
  }
  std::stable_sort(w.items.begin(), w.items.end(), [](const Isect& a, const Isect& b) {
    if (a.tile != b.tile) return a.tile < b.tile;
    if (a.depth != b.depth) return a.depth < b.depth;
    return a.src < b.src;
  });
  const int T = tiles_x * tiles_y;
  w.tile_begin.assign(T, 0);
  w.tile_end.assign(T, 0);
  for (size_t i = 0; i < w.items.size(); ++i) {
    const uint32_t t = w.items[i].tile;
    if (i == 0 || w.items[i - 1].tile != t) w.tile_begin[t] = (int64_t)i;
    w.tile_end[t] = (int64_t)i + 1;
  }
  return w;
}

// ----------------------------------------------------------------------------
// rasterizer — no reference source exists
// ----------------------------------------------------------------------------
constexpr int kMaxChannels = 16;  // 3 colour + D_f <= 13 features

/// Per-Gaussian record the compositing loop reads (what the kernels stage in shared memory).
template <class S> struct Splat {
  S mx, my, vx, vy, vz;  // mean2d, sensor-space velocity
  S a, b2, c;            // conic: a = C00, b2 = C01 + C10, c = C11
  S rho;                 // det_ratio * opacity (Eq. 5 prefactor)
  S depth;               // z or range
  S f[kMaxChannels];     // camera: rgb + features; lidar: features
};

template <class S>
Splat<S> make_splat(const Projected<S>& g, const ComposedScene<S>& scene, bool camera) {
  Splat<S> s;
  const auto& gs = scene.graph->gaussians;
  const int64_t i = g.source_index;
  s.mx = g.mean2d[0]; s.my = g.mean2d[1];
  s.vx = g.velocity[0]; s.vy = g.velocity[1]; s.vz = g.velocity[2];
  s.a = g.conic[0]; s.b2 = g.conic[1] + g.conic[2]; s.c = g.conic[3];
  s.rho = g.det_ratio * scene.opacity[i];
  s.depth = g.depth_key;
  for (int k = 0; k < kMaxChannels; ++k) s.f[k] = S(0);
  int o = 0;
  if (camera) {
    for (int k = 0; k < 3; ++k) s.f[o++] = gs.color[3 * i + k];
  }
  for (int k = 0; k < gs.d_f; ++k) s.f[o++] = gs.feature[(int64_t)gs.d_f * i + k];
  return s;
}

/// SPEC.md:275-283 (Eq. 3) — p_v is the integer row index.
template <class S> S pixel_capture_offset(int p_v, int H, S t_rs, S time_offset) {
  return (S(p_v) / S(H) - S(0.5)) * t_rs + time_offset;
}

/// SPEC.md:285-293 (Eq. 5/6). Returns false when the contribution is skipped.
/// `wrap` = lidar azimuth difference wrapped to (-pi, pi] (common.hpp:41-46).
template <class S>
inline bool evaluate_alpha(const Splat<S>& g, S qx, S qy, S t, const RasterSettings<S>& st, bool wrap, S& alpha,
                           S& dx, S& dy, S& gauss, bool& clamped) {
  const S mx = Sc<S>::fma(g.vx, t, g.mx);
  const S my = Sc<S>::fma(g.vy, t, g.my);
  dx = qx - mx;
  if (wrap) dx = wrap_pi(dx);
  dy = qy - my;
  const S qf = Sc<S>::fma(g.a, dx * dx, Sc<S>::fma(g.c, dy * dy, g.b2 * (dx * dy)));
  if (!(qf <= st.qform_max)) return false;  // 3-sigma support bound (projection.hpp:11); also rejects NaN
  gauss = Sc<S>::exp(S(-0.5) * qf);
  alpha = g.rho * gauss;
  clamped = alpha > st.alpha_clamp;
  if (clamped) alpha = st.alpha_clamp;
  if (!(alpha >= st.alpha_min)) return false;
  return true;
}

template <class S> struct RasterOut {
  int64_t P = 0;
  bool camera = true;
  int channels = 0;                 // camera: 3 + d_f, lidar: d_f
  std::vector<S> blend;             // P x 16: camera rgb(3)+feat(13); lidar feat(13), [13]=expected, [14]=median, [15]=alpha
  std::vector<S> alpha;             // P  (accumulated opacity 1 - T)
  std::vector<S> t_final;           // P  saved terminal transmittance
  std::vector<S> range_blend;       // P  lidar: un-normalised sum w * r_rs
  std::vector<int32_t> n_contrib;   // P  number of blended Gaussians
  std::vector<int32_t> last_idx;    // P  list position (1-based, tile-local) of last blended Gaussian
  std::vector<S> los;               // P  lidar, optional: sum of alpha_i over blended Gaussians with r_i < r_p - eps
  int64_t nonfinite = 0;
};

template <class S> struct Ray { S phi, omega, t; };

/// Compositing of one query over one depth-ordered list. SPEC.md:295-313 (Eq. 4).
template <class S, class GetSplat>
inline void composite_one(int64_t count, GetSplat get, S qx, S qy, S t, bool lidar, const RasterSettings<S>& st, S* acc16,
                          S& T, S& range_acc, S& median, int32_t& n_contrib, int32_t& last_idx, int channels,
                          S los_cut = S(0), S* los = nullptr) {
  // los (lidar, optional): the line-of-sight accumulator of SPEC.md:427 / PAPER.md:532-536 — the sum of alpha_i over the
  // blended Gaussians whose rolling-shutter range lies in front of los_cut = r_p - eps ("penalizing opacity before the
  // ground truth lidar range"). It needs the per-Gaussian alphas, hence lives inside the compositing loop.
  if (los) *los = S(0);
  T = S(1);
  range_acc = S(0);
  median = S(0);
  bool med_found = false;
  n_contrib = 0;
  last_idx = 0;
  for (int k = 0; k < kMaxChannels; ++k) acc16[k] = S(0);
  for (int64_t j = 0; j < count; ++j) {
    const Splat<S>& g = get(j);
    S alpha, dx, dy, gauss;
    bool clamped;
    if (!evaluate_alpha(g, qx, qy, t, st, lidar, alpha, dx, dy, gauss, clamped)) continue;
    const S w = alpha * T;
    for (int k = 0; k < channels; ++k) acc16[k] = Sc<S>::fma(g.f[k], w, acc16[k]);
    T = T * (S(1) - alpha);
    ++n_contrib;
    last_idx = (int32_t)(j + 1);
    if (lidar) {
      const S r_rs = Sc<S>::fma(g.vz, t, g.depth);
      range_acc = Sc<S>::fma(r_rs, w, range_acc);
      if (los && r_rs < los_cut) *los += alpha;
      if (!med_found && T < S(0.5)) {
        median = r_rs;
        med_found = true;
      }
    }
    if (T < st.transmittance_min) break;
  }
}

/// Test-only introspection: the list positions (0-based, tile-local) a query blends, found by the very loop of
/// composite_one (same skip rules, same transmittance cut-off). Used by the gradient parity gate to find the
/// queries on which the fp32 and the fp64 forward passes take different discrete decisions, and the Gaussians those
/// queries touch.
template <class S, class GetSplat>
inline void contributors_one(int64_t count, GetSplat get, S qx, S qy, S t, bool lidar, const RasterSettings<S>& st,
                             std::vector<int32_t>& pos, std::vector<uint8_t>& was_clamped) {
  pos.clear();
  was_clamped.clear();
  S T = S(1);
  for (int64_t j = 0; j < count; ++j) {
    const Splat<S>& g = get(j);
    S alpha, dx, dy, gauss;
    bool clamped;
    if (!evaluate_alpha(g, qx, qy, t, st, lidar, alpha, dx, dy, gauss, clamped)) continue;
    T = T * (S(1) - alpha);
    pos.push_back((int32_t)j);
    was_clamped.push_back(clamped ? 1 : 0);
    if (T < st.transmittance_min) break;
  }
}

template <class S> void finish_lidar(S* px, S T, S range_acc, S median) {
  const S A = S(1) - T;
  px[13] = (A > S(1e-6)) ? range_acc / A : range_acc;
  px[14] = median;
  px[15] = A;
}

/// SPEC.md:295-303. One 16x16 tile per work unit; pixel centre (u+.5, v+.5) (scene.hpp:119-120).
template <class S>
RasterOut<S> rasterize_camera(const Worklist& wl, const std::vector<Projected<S>>& projected,
                              const ComposedScene<S>& scene, const CameraModel<S>& cam, const RasterSettings<S>& st,
                              int workers = 1) {
  RasterOut<S> out;
  const int W = cam.width, H = cam.height;
  out.P = (int64_t)W * H;
  out.camera = true;
  out.channels = 3 + scene.graph->gaussians.d_f;
  out.blend.assign(out.P * 16, S(0));
  out.alpha.assign(out.P, S(0));
  out.t_final.assign(out.P, S(1));
  out.n_contrib.assign(out.P, 0);
  out.last_idx.assign(out.P, 0);
  const int T = wl.tiles_x * wl.tiles_y;
  parallel_chunks(T, workers, [&](int, int64_t tb, int64_t te) {
    std::vector<Splat<S>> splats;
    for (int64_t tile = tb; tile < te; ++tile) {
      const int64_t b = wl.tile_begin[tile], e = wl.tile_end[tile];
      if (e <= b) continue;
      splats.resize(e - b);
      for (int64_t j = b; j < e; ++j) splats[j - b] = make_splat(projected[wl.items[j].pidx], scene, true);
      const int tx = (int)(tile % wl.tiles_x), ty = (int)(tile / wl.tiles_x);
      for (int py = ty * kTile; py < std::min(H, (ty + 1) * kTile); ++py) {
        const S t = pixel_capture_offset<S>(py, H, cam.shutter_duration, cam.time_offset);
        for (int px = tx * kTile; px < std::min(W, (tx + 1) * kTile); ++px) {
          const int64_t p = (int64_t)py * W + px;
          S Tt, ra, med;
          composite_one<S>(e - b, [&](int64_t j) -> const Splat<S>& { return splats[j]; }, S(px) + S(0.5),
                           S(py) + S(0.5), t, false, st, &out.blend[16 * p], Tt, ra, med, out.n_contrib[p],
                           out.last_idx[p], out.channels);
          out.t_final[p] = Tt;
          out.alpha[p] = S(1) - Tt;
        }
      }
    }
  });
  return out;
}

/// SPEC.md:305-313. Rays are grouped per tile: tile t owns rays [ray_begin[t], ray_end[t]) (<= 256 per pass).
template <class S>
RasterOut<S> rasterize_lidar(const Worklist& wl, const std::vector<Projected<S>>& projected,
                             const ComposedScene<S>& scene, const std::vector<Ray<S>>& rays,
                             const std::vector<int64_t>& ray_begin, const std::vector<int64_t>& ray_end,
                             const RasterSettings<S>& st, int workers = 1, const std::vector<S>* los_cut = nullptr) {
  RasterOut<S> out;
  out.P = (int64_t)rays.size();
  if (los_cut) out.los.assign(out.P, S(0));
  out.camera = false;
  out.channels = scene.graph->gaussians.d_f;
  out.blend.assign(out.P * 16, S(0));
  out.alpha.assign(out.P, S(0));
  out.t_final.assign(out.P, S(1));
  out.range_blend.assign(out.P, S(0));
  out.n_contrib.assign(out.P, 0);
  out.last_idx.assign(out.P, 0);
  const int T = wl.tiles_x * wl.tiles_y;
  parallel_chunks(T, workers, [&](int, int64_t tb, int64_t te) {
    std::vector<Splat<S>> splats;
    for (int64_t tile = tb; tile < te; ++tile) {
      const int64_t b = wl.tile_begin[tile], e = wl.tile_end[tile];
      splats.resize(std::max<int64_t>(0, e - b));
      for (int64_t j = b; j < e; ++j) splats[j - b] = make_splat(projected[wl.items[j].pidx], scene, false);
      for (int64_t p = ray_begin[tile]; p < ray_end[tile]; ++p) {
        S Tt, ra, med;
        composite_one<S>(std::max<int64_t>(0, e - b), [&](int64_t j) -> const Splat<S>& { return splats[j]; },
                         rays[p].phi, rays[p].omega, rays[p].t, true, st, &out.blend[16 * p], Tt, ra, med,
                         out.n_contrib[p], out.last_idx[p], out.channels, los_cut ? (*los_cut)[p] : S(0),
                         los_cut ? &out.los[p] : nullptr);
        out.t_final[p] = Tt;
        out.alpha[p] = S(1) - Tt;
        out.range_blend[p] = ra;
        finish_lidar(&out.blend[16 * p], Tt, ra, med);
      }
    }
  });
  return out;
}

/// every projected Gaussian against every query, global depth sort, no tiling,
/// no AABB. `early_exit` false disables the transmittance cut-off as SPEC describes.
template <class S>
RasterOut<S> brute_force(const std::vector<Projected<S>>& projected, const ComposedScene<S>& scene, bool camera,
                         const CameraModel<S>* cam, const std::vector<Ray<S>>* rays, RasterSettings<S> st,
                         bool early_exit) {
  if (!early_exit) st.transmittance_min = S(0);
  std::vector<int32_t> order(projected.size());
  for (size_t k = 0; k < order.size(); ++k) order[k] = (int32_t)k;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    if (projected[a].depth_key != projected[b].depth_key) return projected[a].depth_key < projected[b].depth_key;
    return projected[a].source_index < projected[b].source_index;
  });
  std::vector<Splat<S>> splats(order.size());
  for (size_t k = 0; k < order.size(); ++k) splats[k] = make_splat(projected[order[k]], scene, camera);
  RasterOut<S> out;
  out.camera = camera;
  const int d_f = scene.graph->gaussians.d_f;
  out.channels = camera ? 3 + d_f : d_f;
  out.P = camera ? (int64_t)cam->width * cam->height : (int64_t)rays->size();
  out.blend.assign(out.P * 16, S(0));
  out.alpha.assign(out.P, S(0));
  out.t_final.assign(out.P, S(1));
  out.range_blend.assign(out.P, S(0));
  out.n_contrib.assign(out.P, 0);
  out.last_idx.assign(out.P, 0);
  auto get = [&](int64_t j) -> const Splat<S>& { return splats[j]; };
  for (int64_t p = 0; p < out.P; ++p) {
    S Tt, ra, med;
    if (camera) {
      const int py = (int)(p / cam->width), px = (int)(p % cam->width);
      const S t = pixel_capture_offset<S>(py, cam->height, cam->shutter_duration, cam->time_offset);
      composite_one<S>((int64_t)splats.size(), get, S(px) + S(0.5), S(py) + S(0.5), t, false, st, &out.blend[16 * p], Tt,
                       ra, med, out.n_contrib[p], out.last_idx[p], out.channels);
    } else {
      composite_one<S>((int64_t)splats.size(), get, (*rays)[p].phi, (*rays)[p].omega, (*rays)[p].t, true, st,
                       &out.blend[16 * p], Tt, ra, med, out.n_contrib[p], out.last_idx[p], out.channels);
      finish_lidar(&out.blend[16 * p], Tt, ra, med);
      out.range_blend[p] = ra;
    }
    out.t_final[p] = Tt;
    out.alpha[p] = S(1) - Tt;
  }
  return out;
}

// ---- backward (derivation in DESIGN.md) ----------

/// Raw per-Gaussian sums the compositing backward produces (what the kernel's atomics accumulate),
/// indexed by source index.
template <class S> struct RasterGrads {
  int64_t n = 0;
  std::vector<S> g_conic;   // 3N: dL/dC as a symmetric matrix [Gaa, Gab, Gcc]
  std::vector<S> g_mean2d;  // 2N
  std::vector<S> g_vel;     // 3N
  std::vector<S> g_rho;     // N
  std::vector<S> g_range;   // N
  std::vector<S> g_f;       // 16N
  S d_time_offset = 0;
  void resize(int64_t n_) {
    n = n_;
    g_conic.assign(3 * n, S(0)); g_mean2d.assign(2 * n, S(0)); g_vel.assign(3 * n, S(0));
    g_rho.assign(n, S(0)); g_range.assign(n, S(0)); g_f.assign(16 * n, S(0));
    d_time_offset = S(0);
  }
  void add(const RasterGrads& o) {
    auto acc = [](std::vector<S>& a, const std::vector<S>& b) {
      for (size_t i = 0; i < a.size(); ++i) a[i] += b[i];
    };
    acc(g_conic, o.g_conic); acc(g_mean2d, o.g_mean2d); acc(g_vel, o.g_vel); acc(g_rho, o.g_rho);
    acc(g_range, o.g_range); acc(g_f, o.g_f);
    d_time_offset += o.d_time_offset;
  }
};

/// Back-to-front pass over one query. g_out16: upstream for the 16 blend slots
/// (camera: rgb+features; lidar: features, [13] = d/d expected). g_alpha: upstream of accumulated opacity.
template <class S, class GetSplat, class GetSrc>
inline void composite_one_backward(GetSplat get, GetSrc src_of, S qx, S qy, S t, bool lidar, const RasterSettings<S>& st,
                                   const S* g_out16, S g_alpha, S t_final, S range_blend, int32_t last_idx, int channels,
                                   RasterGrads<S>& out, S los_cut = S(0), S g_los = S(0), bool los = false) {
  if (last_idx <= 0) return;
  S g_acc = g_alpha;  // dL/dA, A = 1 - T_final
  S g_D = S(0);       // dL/d(range_blend)
  if (lidar) {
    const S A = S(1) - t_final;
    if (A > S(1e-6)) {  // expected = D / A
      g_D = g_out16[13] / A;
      g_acc += -g_out16[13] * (range_blend / A) / A;
    } else {
      g_D = g_out16[13];
    }
  }
  S T = t_final;
  S suffix[kMaxChannels];
  for (int k = 0; k < kMaxChannels; ++k) suffix[k] = S(0);
  S suffix_r = S(0);
  for (int64_t j = last_idx - 1; j >= 0; --j) {
    const Splat<S>& g = get(j);
    S alpha, dx, dy, gauss;
    bool clamped;
    if (!evaluate_alpha(g, qx, qy, t, st, lidar, alpha, dx, dy, gauss, clamped)) continue;
    const S one_m = S(1) - alpha;
    T = T / one_m;  // transmittance in front of this Gaussian
    const S w = alpha * T;
    const int64_t i = src_of(j);
    S g_a = S(0);
    for (int k = 0; k < channels; ++k) {
      out.g_f[16 * i + k] += w * g_out16[k];
      g_a += g_out16[k] * (g.f[k] * T - suffix[k] / one_m);
      suffix[k] += w * g.f[k];
    }
    if (lidar) {
      const S r_rs = Sc<S>::fma(g.vz, t, g.depth);
      out.g_range[i] += g_D * w;
      out.g_vel[3 * i + 2] += g_D * w * t;
      g_a += g_D * (r_rs * T - suffix_r / one_m);
      suffix_r += w * r_rs;
      if (los && r_rs < los_cut) g_a += g_los;  // d los / d alpha_i = 1 for the Gaussians in front of the cut
    }
    g_a += g_acc * t_final / one_m;
    if (clamped) continue;  // alpha == alpha_clamp is constant in every parameter
    const S g_sigma = -alpha * g_a;  // alpha = rho exp(-sigma), sigma = qf / 2
    out.g_rho[i] += gauss * g_a;
    const S gdx = g_sigma * (g.a * dx + S(0.5) * g.b2 * dy);
    const S gdy = g_sigma * (g.c * dy + S(0.5) * g.b2 * dx);
    out.g_conic[3 * i] += g_sigma * S(0.5) * dx * dx;
    out.g_conic[3 * i + 1] += g_sigma * S(0.5) * dx * dy;
    out.g_conic[3 * i + 2] += g_sigma * S(0.5) * dy * dy;
    out.g_mean2d[2 * i] += -gdx;
    out.g_mean2d[2 * i + 1] += -gdy;
    out.g_vel[3 * i] += -t * gdx;
    out.g_vel[3 * i + 1] += -t * gdy;
    out.d_time_offset += -(g.vx * gdx + g.vy * gdy);
  }
}

/// Per-Gaussian epilogue: raw sums -> reference-convention ProjectedGrads (projection.hpp:178-185):
/// g_cov2d w.r.t. cov2d (through conic and det_ratio), g_opacity w.r.t. activated opacity.
template <class S>
void raster_grads_to_projected_grads(const RasterGrads<S>& rg, const std::vector<Projected<S>>& projected,
                                     const ComposedScene<S>& scene, bool camera, ProjectedGrads<S>& pg) {
  const auto& gs = scene.graph->gaussians;
  pg.resize(gs.n, gs.d_f);
  for (const auto& g : projected) {
    const int64_t i = g.source_index;
    const S o = scene.opacity[i];
    const S g_rho = rg.g_rho[i];
    pg.g_opacity[i] = g.det_ratio * g_rho;
    const S g_dr = o * g_rho;
    // conic C (2x2, as stored) ; dL/dSigma' = -C^T Gc C^T with Gc symmetric
    const S C[2][2] = {{g.conic[0], g.conic[1]}, {g.conic[2], g.conic[3]}};
    const S Gc[2][2] = {{rg.g_conic[3 * i], rg.g_conic[3 * i + 1]}, {rg.g_conic[3 * i + 1], rg.g_conic[3 * i + 2]}};
    S CtG[2][2], M[2][2];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) CtG[a][b] = C[0][a] * Gc[0][b] + C[1][a] * Gc[1][b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) M[a][b] = -(CtG[a][0] * C[b][0] + CtG[a][1] * C[b][1]);
    // det_ratio = sqrt(|S| / |S + sI|): d/dS = (det_ratio / 2) (S^-T - C^T)
    const S det = g.cov2d[0] * g.cov2d[3] - g.cov2d[2] * g.cov2d[1];
    const S inv[2][2] = {{g.cov2d[3] / det, -g.cov2d[1] / det}, {-g.cov2d[2] / det, g.cov2d[0] / det}};
    const S k = g_dr * g.det_ratio * S(0.5);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) pg.g_cov2d[4 * i + 2 * a + b] = M[a][b] + k * (inv[b][a] - C[b][a]);
    pg.g_mean2d[2 * i] = rg.g_mean2d[2 * i];
    pg.g_mean2d[2 * i + 1] = rg.g_mean2d[2 * i + 1];
    pg.g_range[i] = rg.g_range[i];
    for (int c = 0; c < 3; ++c) pg.g_velocity[3 * i + c] = rg.g_vel[3 * i + c];
    int off = 0;
    if (camera)
      for (int c = 0; c < 3; ++c) pg.g_color[3 * i + c] = rg.g_f[16 * i + off++];
    for (int c = 0; c < gs.d_f; ++c) pg.g_feature[(int64_t)gs.d_f * i + c] = rg.g_f[16 * i + off++];
  }
}

/// SPEC.md:315-323. Tiles are independent; per-worker buffers reduced in worker order.
template <class S>
RasterGrads<S> rasterize_backward(const Worklist& wl, const std::vector<Projected<S>>& projected,
                                  const ComposedScene<S>& scene, bool camera, const CameraModel<S>* cam,
                                  const std::vector<Ray<S>>* rays, const std::vector<int64_t>* ray_begin,
                                  const std::vector<int64_t>* ray_end, const RasterSettings<S>& st,
                                  const RasterOut<S>& fwd, const std::vector<S>& g_blend16,
                                  const std::vector<S>& g_alpha, int workers = 1, const std::vector<S>* los_cut = nullptr,
                                  const std::vector<S>* g_los = nullptr) {
  const int64_t N = scene.size();
  const bool los = los_cut && g_los;
  const int T = wl.tiles_x * wl.tiles_y;
  workers = std::max(1, workers);
  std::vector<RasterGrads<S>> parts(workers);
  std::vector<char> used(workers, 0);
  parallel_chunks(T, workers, [&](int wk, int64_t tb, int64_t te) {
    auto& out = parts[wk];
    out.resize(N);
    used[wk] = 1;
    std::vector<Splat<S>> splats;
    for (int64_t tile = tb; tile < te; ++tile) {
      const int64_t b = wl.tile_begin[tile], e = wl.tile_end[tile];
      if (e <= b) continue;
      splats.resize(e - b);
      for (int64_t j = b; j < e; ++j) splats[j - b] = make_splat(projected[wl.items[j].pidx], scene, camera);
      auto get = [&](int64_t j) -> const Splat<S>& { return splats[j]; };
      auto src = [&](int64_t j) -> int64_t { return wl.items[b + j].src; };
      if (camera) {
        const int W = cam->width, H = cam->height;
        const int tx = (int)(tile % wl.tiles_x), ty = (int)(tile / wl.tiles_x);
        for (int py = ty * kTile; py < std::min(H, (ty + 1) * kTile); ++py) {
          const S t = pixel_capture_offset<S>(py, H, cam->shutter_duration, cam->time_offset);
          for (int px = tx * kTile; px < std::min(W, (tx + 1) * kTile); ++px) {
            const int64_t p = (int64_t)py * W + px;
            composite_one_backward<S>(get, src, S(px) + S(0.5), S(py) + S(0.5), t, false, st, &g_blend16[16 * p],
                                      g_alpha[p], fwd.t_final[p], S(0), fwd.last_idx[p], fwd.channels, out);
          }
        }
      } else {
        for (int64_t p = (*ray_begin)[tile]; p < (*ray_end)[tile]; ++p)
          composite_one_backward<S>(get, src, (*rays)[p].phi, (*rays)[p].omega, (*rays)[p].t, true, st,
                                    &g_blend16[16 * p], g_alpha[p], fwd.t_final[p], fwd.range_blend[p],
                                    fwd.last_idx[p], fwd.channels, out, los ? (*los_cut)[p] : S(0), los ? (*g_los)[p] : S(0),
                                    los);
      }
    }
  });
  RasterGrads<S> total;
  total.resize(N);
  for (int wk = 0; wk < workers; ++wk)
    if (used[wk]) total.add(parts[wk]);
  return total;
}

}  // namespace orc
