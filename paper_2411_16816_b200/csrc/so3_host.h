// so3_host.h — host-side (double) SO(3) helpers and actor pose interpolation for libsplat_b200.so.
//
// Actor tracks are per-actor work (tens of actors), so they stay on the host in double like the
// reference's test mode. Reference semantics: so3.hpp:10-66 (exp/log, right Jacobian family),
// scene.hpp:64-83 (corrected_pose, init_velocity_from_poses), scene.hpp:238-258 (interpolate_pose),
// scene.hpp:428-453 (pose-offset gradients).
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace sbh {

struct M3 {
  double a[9];
};
struct V3 {
  double a[3];
};

inline M3 eye() { return M3{{1, 0, 0, 0, 1, 0, 0, 0, 1}}; }
inline M3 hat(const V3& v) { return M3{{0, -v.a[2], v.a[1], v.a[2], 0, -v.a[0], -v.a[1], v.a[0], 0}}; }
inline M3 mm(const M3& x, const M3& y) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[3 * i + j] = x.a[3 * i] * y.a[j] + x.a[3 * i + 1] * y.a[3 + j] + x.a[3 * i + 2] * y.a[6 + j];
  return r;
}
inline M3 tr(const M3& x) { return M3{{x.a[0], x.a[3], x.a[6], x.a[1], x.a[4], x.a[7], x.a[2], x.a[5], x.a[8]}}; }
inline M3 lin(double ca, const M3& x, double cb, const M3& y, double cc, const M3& z) {
  M3 r;
  for (int i = 0; i < 9; ++i) r.a[i] = ca * x.a[i] + cb * y.a[i] + cc * z.a[i];
  return r;
}
inline V3 mv(const M3& x, const V3& v) {
  V3 r;
  for (int i = 0; i < 3; ++i) r.a[i] = x.a[3 * i] * v.a[0] + x.a[3 * i + 1] * v.a[1] + x.a[3 * i + 2] * v.a[2];
  return r;
}
inline V3 scale(double c, const V3& v) { return V3{{c * v.a[0], c * v.a[1], c * v.a[2]}}; }
inline double sqn(const V3& v) { return v.a[0] * v.a[0] + v.a[1] * v.a[1] + v.a[2] * v.a[2]; }

/// so3.hpp:10-19
inline M3 exp_so3(const V3& phi) {
  const double t2 = sqn(phi);
  const M3 K = hat(phi), K2 = mm(K, K);
  if (t2 < 1e-16) return lin(1.0, eye(), 1.0, K, 0.5, K2);
  const double t = std::sqrt(t2);
  return lin(1.0, eye(), std::sin(t) / t, K, (1.0 - std::cos(t)) / t2, K2);
}

/// so3.hpp:21-38
inline V3 log_so3(const M3& R) {
  const double c = std::clamp((R.a[0] + R.a[4] + R.a[8] - 1.0) / 2.0, -1.0, 1.0);
  const double t = std::acos(c);
  const V3 w{{R.a[7] - R.a[5], R.a[2] - R.a[6], R.a[3] - R.a[1]}};
  if (t < 1e-8) return scale(0.5, w);
  if (t > M_PI - 1e-6) {
    double A[9];
    for (int i = 0; i < 9; ++i) A[i] = 0.5 * (R.a[i] + (i % 4 == 0 ? 1.0 : 0.0));
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (A[4 * i] > A[4 * k]) k = i;
    V3 axis{{A[k], A[3 + k], A[6 + k]}};
    axis = scale(1.0 / std::sqrt(A[4 * k]), axis);
    axis = scale(1.0 / std::sqrt(sqn(axis)), axis);
    if (w.a[0] * axis.a[0] + w.a[1] * axis.a[1] + w.a[2] * axis.a[2] < 0) axis = scale(-1.0, axis);
    return scale(t, axis);
  }
  return scale(t / (2.0 * std::sin(t)), w);
}

/// so3.hpp:41-50
inline M3 right_jacobian(const V3& phi) {
  const double t2 = sqn(phi);
  const M3 K = hat(phi), K2 = mm(K, K);
  if (t2 < 1e-16) return lin(1.0, eye(), -0.5, K, 1.0 / 6.0, K2);
  const double t = std::sqrt(t2);
  return lin(1.0, eye(), -(1.0 - std::cos(t)) / t2, K, (t - std::sin(t)) / (t2 * t), K2);
}
/// so3.hpp:52-61
inline M3 right_jacobian_inv(const V3& phi) {
  const double t2 = sqn(phi);
  const M3 K = hat(phi), K2 = mm(K, K);
  if (t2 < 1e-16) return lin(1.0, eye(), 0.5, K, 1.0 / 12.0, K2);
  const double t = std::sqrt(t2);
  return lin(1.0, eye(), 0.5, K, 1.0 / t2 - (1.0 + std::cos(t)) / (2.0 * t * std::sin(t)), K2);
}
/// so3.hpp:64-66
inline M3 left_jacobian_inv(const V3& phi) { return right_jacobian_inv(scale(-1.0, phi)); }

/// scene.hpp:50-96
struct Track {
  std::vector<double> stamps, R, t, pose_offset;  // n, 9n, 3n, 6n
  double vel_lin[3] = {0, 0, 0}, vel_ang[3] = {0, 0, 0}, vel_offset[6] = {0, 0, 0, 0, 0, 0};
  int n_poses() const { return (int)stamps.size(); }
  M3 rot(int i) const {
    M3 m;
    std::copy(R.begin() + 9 * i, R.begin() + 9 * i + 9, m.a);
    return m;
  }
  V3 off_r(int i) const { return V3{{pose_offset[6 * i + 3], pose_offset[6 * i + 4], pose_offset[6 * i + 5]}}; }
  /// scene.hpp:64-67
  void corrected(int i, M3& Rc, V3& tc) const {
    Rc = mm(rot(i), exp_so3(off_r(i)));
    for (int k = 0; k < 3; ++k) tc.a[k] = t[3 * i + k] + pose_offset[6 * i + k];
  }
  /// scene.hpp:70-83
  void init_velocity_from_poses() {
    for (int k = 0; k < 3; ++k) vel_lin[k] = vel_ang[k] = 0.0;
    const int n = n_poses();
    if (n < 2) return;
    double v[3] = {0, 0, 0}, w[3] = {0, 0, 0};
    for (int i = 0; i + 1 < n; ++i) {
      const double dt = stamps[i + 1] - stamps[i];
      const V3 d{{t[3 * i + 3] - t[3 * i], t[3 * i + 4] - t[3 * i + 1], t[3 * i + 5] - t[3 * i + 2]}};
      const V3 lv = mv(tr(rot(i)), d);
      const V3 lw = log_so3(mm(tr(rot(i)), rot(i + 1)));
      for (int k = 0; k < 3; ++k) { v[k] += lv.a[k] / dt; w[k] += lw.a[k] / dt; }
    }
    for (int k = 0; k < 3; ++k) { vel_lin[k] = v[k] / double(n - 1); vel_ang[k] = w[k] / double(n - 1); }
  }
};

/// scene.hpp:231-258
struct Interp {
  M3 R = eye();
  V3 t{{0, 0, 0}};
  int i0 = 0, i1 = 0;
  double u = 0;
  V3 geo{{0, 0, 0}};
};
inline Interp interpolate_pose(const Track& tk, double time) {
  Interp o;
  const int n = tk.n_poses();
  if (n == 0) throw std::runtime_error("actor track has no poses");
  if (n == 1) {
    tk.corrected(0, o.R, o.t);
    return o;
  }
  int i = 0;
  while (i + 2 < n && time >= tk.stamps[i + 1]) ++i;
  o.i0 = i;
  o.i1 = i + 1;
  o.u = (time - tk.stamps[i]) / (tk.stamps[i + 1] - tk.stamps[i]);
  M3 Ra, Rb;
  V3 ta, tb;
  tk.corrected(i, Ra, ta);
  tk.corrected(i + 1, Rb, tb);
  o.geo = log_so3(mm(tr(Ra), Rb));
  o.R = mm(Ra, exp_so3(scale(o.u, o.geo)));
  for (int k = 0; k < 3; ++k) o.t.a[k] = (1.0 - o.u) * ta.a[k] + o.u * tb.a[k];
  return o;
}

/// scene.hpp:428-453: distribute the per-actor sums (sum of dL/d mean_w, sum of dL/d psi) onto the
/// per-stamp pose offsets. d_pose_offset: 6 x n_poses, stamp-major.
inline void pose_offset_backward(const Track& tk, const Interp& ip, const V3& g_mu, const V3& g_psi, double* d_pose_offset) {
  auto add = [&](int col, const V3& a, const V3& b) {
    for (int k = 0; k < 3; ++k) { d_pose_offset[6 * col + k] += a.a[k]; d_pose_offset[6 * col + 3 + k] += b.a[k]; }
  };
  if (tk.n_poses() == 1) {
    add(0, g_mu, mv(tr(right_jacobian(tk.off_r(0))), g_psi));
    return;
  }
  const double u = ip.u;
  const V3 uphi = scale(u, ip.geo);
  const M3 Jr_u = right_jacobian(uphi);
  const M3 zero{{0, 0, 0, 0, 0, 0, 0, 0, 0}};
  const M3 B0 = lin(1.0, tr(exp_so3(uphi)), -u, mm(Jr_u, left_jacobian_inv(ip.geo)), 0.0, zero);
  const M3 B1 = lin(u, mm(Jr_u, right_jacobian_inv(ip.geo)), 0.0, zero, 0.0, zero);
  add(ip.i0, scale(1.0 - u, g_mu), mv(tr(right_jacobian(tk.off_r(ip.i0))), mv(tr(B0), g_psi)));
  add(ip.i1, scale(u, g_mu), mv(tr(right_jacobian(tk.off_r(ip.i1))), mv(tr(B1), g_psi)));
}

}  // namespace sbh
