// ref_harness.cpp — C entry points over the UNMODIFIED reference headers, compiled where they lie
// (-I/root/reference/proj/include) against oracle/eigen_shim. TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/ref_build.sh into oracle/_ref/libsplat_ref.so (git-ignored; travels to the GPU box).
// Used by tests/test_oracle_vs_ref.py to pin the CPU oracle's restatement of
//   compose_at_time            scene.hpp:273-308        project_camera / project_lidar   projection.hpp:88-174
//   project_*_backward         projection.hpp:250-357   compose_backward                 scene.hpp:386-458
// and by scripts/make_golden.py to generate tests/golden/*.npz. No reference source is copied: this
// file only CALLS splat::* and moves plain arrays in and out.
//
// Packed sensor layouts are the oracle's (oracle_capi.cpp): cam[27], lidar[24], settings[7].
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "splat/projection.hpp"

namespace {

template <class S> struct RefH {
  splat::SceneGraph<S> graph;
  splat::ComposedScene<S> scene;
  bool camera = true;
  splat::CameraModel<S> cam;
  splat::LidarModel<S> lidar;
  splat::RasterSettings<S> st;
  std::vector<splat::ProjectedGaussian<S>> proj;
  splat::ComposeGrads<S> cg;
  splat::SensorGrads<S> sg;
  splat::SceneParamGrads<S> out;
  std::string error;
};

template <class S> void unpack_pose(const double* p, splat::SE3<S>& pose, splat::Vec3<S>& vl, splat::Vec3<S>& va) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) pose.R(r, c) = S(p[3 * r + c]);
  for (int k = 0; k < 3; ++k) { pose.t(k) = S(p[9 + k]); vl(k) = S(p[12 + k]); va(k) = S(p[15 + k]); }
}

template <class S> splat::RasterSettings<S> unpack_settings(const double* s) {
  splat::RasterSettings<S> st;
  st.dilation = S(s[0]); st.alpha_clamp = S(s[1]); st.alpha_min = S(s[2]); st.qform_max = S(s[3]);
  st.transmittance_min = S(s[4]); st.near_plane = S(s[5]); st.lidar_min_range = S(s[6]);
  return st;
}

template <class S>
void* scene_new(int64_t n, int d_f, const S* mean, const S* scale_log, const S* quat, const S* opacity_logit,
                const S* color, const S* feature, const int32_t* actor_id) {
  auto* h = new RefH<S>();
  auto& g = h->graph.gaussians;
  g.resize(n, d_f);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) {
      g.mean(k, i) = mean[3 * i + k];
      g.scale_log(k, i) = scale_log[3 * i + k];
      g.color(k, i) = color[3 * i + k];
    }
    for (int k = 0; k < 4; ++k) g.quat(k, i) = quat[4 * i + k];
    g.opacity_logit(0, i) = opacity_logit[i];
    for (int k = 0; k < d_f; ++k) g.feature(k, i) = feature[(int64_t)d_f * i + k];
    g.actor_id(i) = actor_id[i];
  }
  return h;
}

// Tracks arrive in double (like the oracle's) and are built as ActorTrack<double>, then cast<S>() —
// the reference's own conversion path (scene.hpp:85-96).
template <class S>
void add_track(void* hv, int n_poses, const double* stamps, const double* R, const double* t, const double* pose_offset,
               const double* vel_lin, const double* vel_ang, const double* vel_offset, int init_vel) {
  auto* h = (RefH<S>*)hv;
  splat::ActorTrack<double> tr;
  tr.pose_offset.setZero(6, n_poses);
  for (int i = 0; i < n_poses; ++i) {
    tr.stamps.push_back(stamps[i]);
    splat::SE3<double> p;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) p.R(r, c) = R[9 * i + 3 * r + c];
    for (int k = 0; k < 3; ++k) p.t(k) = t[3 * i + k];
    tr.poses.push_back(p);
    for (int k = 0; k < 6; ++k) tr.pose_offset(k, i) = pose_offset[6 * i + k];
  }
  if (init_vel) {
    tr.init_velocity_from_poses();
  } else {
    for (int k = 0; k < 3; ++k) { tr.vel_lin(k) = vel_lin[k]; tr.vel_ang(k) = vel_ang[k]; }
  }
  for (int k = 0; k < 6; ++k) tr.vel_offset(k) = vel_offset[k];
  h->graph.tracks.push_back(tr.template cast<S>());
}

template <class S> int64_t project(RefH<S>* h, double t_scene) {
  try {
    h->scene = splat::compose_at_time<S>(h->graph, S(t_scene));
    h->proj = h->camera ? splat::project_camera<S>(h->scene, h->cam, h->st) : splat::project_lidar<S>(h->scene, h->lidar, h->st);
  } catch (const std::exception& e) {
    h->error = e.what();
    return -1;
  }
  return (int64_t)h->proj.size();
}

template <class S> int64_t view_camera(void* hv, double t_scene, const double* c, const double* settings) {
  auto* h = (RefH<S>*)hv;
  h->camera = true;
  h->cam = splat::CameraModel<S>();
  h->cam.fx = S(c[0]); h->cam.fy = S(c[1]); h->cam.cx = S(c[2]); h->cam.cy = S(c[3]);
  h->cam.width = (int)c[4]; h->cam.height = (int)c[5];
  unpack_pose<S>(c + 6, h->cam.pose, h->cam.vel_lin, h->cam.vel_ang);
  h->cam.shutter_duration = S(c[24]); h->cam.time_offset = S(c[25]); h->cam.timestamp = S(c[26]);
  h->st = unpack_settings<S>(settings);
  return project(h, t_scene);
}

template <class S>
int64_t view_lidar(void* hv, double t_scene, const double* l, const double* elev, int n_beams, const double* settings) {
  auto* h = (RefH<S>*)hv;
  h->camera = false;
  h->lidar = splat::LidarModel<S>();
  h->lidar.azimuth_resolution = S(l[0]); h->lidar.scan_duration = S(l[1]);
  h->lidar.beam_divergence_h = S(l[2]); h->lidar.beam_divergence_v = S(l[3]);
  unpack_pose<S>(l + 4, h->lidar.pose, h->lidar.vel_lin, h->lidar.vel_ang);
  h->lidar.timestamp = S(l[22]); h->lidar.max_range = S(l[23]);
  for (int i = 0; i < n_beams; ++i) h->lidar.elevation_channels.push_back(S(elev[i]));
  h->st = unpack_settings<S>(settings);
  return project(h, t_scene);
}

// ProjectedGrads arrive indexed by SOURCE index (the header's stated convention, projection.hpp:176-177);
// the shipped consumers read the geometry groups by projected position k (projection.hpp:257-268, 329-344),
// so those groups are gathered through source_index here. See DESIGN.md "index convention".
template <class S>
int backward(void* hv, const S* g_mean2d, const S* g_range, const S* g_cov2d, const S* g_velocity, const S* g_opacity) {
  auto* h = (RefH<S>*)hv;
  const Eigen::Index n = h->graph.gaussians.size();
  const Eigen::Index V = (Eigen::Index)h->proj.size();
  splat::ProjectedGrads<S> gin;
  gin.resize(V, h->graph.gaussians.feature_dim());
  for (Eigen::Index k = 0; k < V; ++k) {
    const Eigen::Index i = h->proj[k].source_index;
    gin.g_mean2d(0, k) = g_mean2d[2 * i]; gin.g_mean2d(1, k) = g_mean2d[2 * i + 1];
    gin.g_range(0, k) = g_range[i];
    gin.g_cov2d[k](0, 0) = g_cov2d[4 * i]; gin.g_cov2d[k](0, 1) = g_cov2d[4 * i + 1];
    gin.g_cov2d[k](1, 0) = g_cov2d[4 * i + 2]; gin.g_cov2d[k](1, 1) = g_cov2d[4 * i + 3];
    for (int c = 0; c < 3; ++c) gin.g_velocity(c, k) = g_velocity[3 * i + c];
  }
  splat::MatRX<S, 1> g_op;
  g_op.setZero(1, n);
  for (Eigen::Index i = 0; i < n; ++i) g_op(0, i) = g_opacity[i];
  h->cg.resize(n);
  h->sg = splat::SensorGrads<S>();
  h->out.resize_like(h->graph);
  try {
    if (h->camera) splat::project_camera_backward<S>(h->scene, h->cam, h->proj, gin, h->cg, h->sg, 0, V);
    else splat::project_lidar_backward<S>(h->scene, h->lidar, h->proj, gin, h->cg, h->sg, 0, V);
    splat::compose_backward<S>(h->scene, h->cg, g_op, h->out, 0, n);
  } catch (const std::exception& e) {
    h->error = e.what();
    return -1;
  }
  return 0;
}

template <class S, class M> int64_t put_cols(const M& m, S* dst) {  // column-major kxN -> N rows of k
  if (dst)
    for (Eigen::Index j = 0; j < m.cols(); ++j)
      for (Eigen::Index i = 0; i < m.rows(); ++i) dst[j * m.rows() + i] = m(i, j);
  return (int64_t)(m.rows() * m.cols());
}

template <class S> int64_t array(void* hv, const char* name_c, void* dstv) {
  auto* h = (RefH<S>*)hv;
  const std::string name(name_c);
  S* dst = (S*)dstv;
  const int64_t n = h->graph.gaussians.size(), V = (int64_t)h->proj.size();
  auto mats = [&](const std::vector<splat::Mat3<S>>& v) -> int64_t {
    if (dst)
      for (size_t i = 0; i < v.size(); ++i)
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) dst[9 * i + 3 * r + c] = v[i](r, c);
    return 9 * (int64_t)v.size();
  };
  if (name == "mean_w") return put_cols<S>(h->scene.mean_w, dst);
  if (name == "vel_dyn_w") return put_cols<S>(h->scene.vel_dyn_w, dst);
  if (name == "opacity") return put_cols<S>(h->scene.opacity, dst);
  if (name == "cov_w") return mats(h->scene.cov_w);
  if (name == "source_index") {
    if (dstv) for (int64_t k = 0; k < V; ++k) ((int64_t*)dstv)[k] = (int64_t)h->proj[k].source_index;
    return V;
  }
  auto field = [&](int w, auto get) -> int64_t {
    if (dst)
      for (int64_t k = 0; k < V; ++k)
        for (int c = 0; c < w; ++c) dst[k * w + c] = get(h->proj[k], c);
    return V * w;
  };
  using PG = splat::ProjectedGaussian<S>;
  if (name == "mean2d") return field(2, [](const PG& g, int c) { return g.mean2d(c); });
  if (name == "depth_key") return field(1, [](const PG& g, int) { return g.depth_key; });
  if (name == "cov2d") return field(4, [](const PG& g, int c) { return g.cov2d(c / 2, c % 2); });
  if (name == "velocity") return field(3, [](const PG& g, int c) { return g.velocity(c); });
  if (name == "aabb") return field(4, [](const PG& g, int c) { return c < 2 ? g.aabb.lo(c) : g.aabb.hi(c - 2); });
  if (name == "conic") return field(4, [](const PG& g, int c) { return g.conic(c / 2, c % 2); });
  if (name == "det_ratio") return field(1, [](const PG& g, int) { return g.det_ratio; });
  if (name == "mu_sensor") return field(3, [](const PG& g, int c) { return g.mu_sensor(c); });
  if (name == "rel_vel_sensor") return field(3, [](const PG& g, int c) { return g.rel_vel_sensor(c); });
  if (name == "cg_mean_w") return put_cols<S>(h->cg.g_mean_w, dst);
  if (name == "cg_vel_dyn_w") return put_cols<S>(h->cg.g_vel_dyn_w, dst);
  if (name == "cg_cov_w") return mats(h->cg.g_cov_w);
  if (name == "d_mean") return put_cols<S>(h->out.d_mean, dst);
  if (name == "d_scale_log") return put_cols<S>(h->out.d_scale_log, dst);
  if (name == "d_quat") return put_cols<S>(h->out.d_quat, dst);
  if (name == "d_opacity_logit") return put_cols<S>(h->out.d_opacity_logit, dst);
  if (name == "sensor_grads") {
    if (dst) {
      for (int k = 0; k < 3; ++k) { dst[k] = h->sg.d_vel_lin(k); dst[3 + k] = h->sg.d_vel_ang(k); }
      dst[6] = h->sg.d_time_offset;
    }
    return 7;
  }
  if (name.rfind("actor_d_pose_offset:", 0) == 0) {
    const size_t a = (size_t)std::stoi(name.substr(20));
    if (a >= h->out.actors.size()) return -1;
    return put_cols<S>(h->out.actors[a].d_pose_offset, dst);
  }
  if (name.rfind("actor_d_vel_offset:", 0) == 0) {
    const size_t a = (size_t)std::stoi(name.substr(19));
    if (a >= h->out.actors.size()) return -1;
    return put_cols<S>(h->out.actors[a].d_vel_offset, dst);
  }
  if (name.rfind("actor_vel:", 0) == 0) {  // effective body velocities (lin 3, ang 3)
    const size_t a = (size_t)std::stoi(name.substr(10));
    if (a >= h->graph.tracks.size()) return -1;
    if (dst) {
      const auto vl = h->graph.tracks[a].effective_vel_lin(), va = h->graph.tracks[a].effective_vel_ang();
      for (int k = 0; k < 3; ++k) { dst[k] = vl(k); dst[3 + k] = va(k); }
    }
    return 6;
  }
  (void)n;
  return -1;
}

}  // namespace

#define REF_API(S, SUF)                                                                                                    \
  extern "C" void* ref_scene_new_##SUF(int64_t n, int d_f, const S* mean, const S* scale_log, const S* quat,               \
                                        const S* opacity_logit, const S* color, const S* feature, const int32_t* actor_id) { \
    return scene_new<S>(n, d_f, mean, scale_log, quat, opacity_logit, color, feature, actor_id);                           \
  }                                                                                                                        \
  extern "C" void ref_scene_add_track_##SUF(void* h, int n_poses, const double* stamps, const double* R, const double* t,  \
                                             const double* pose_offset, const double* vel_lin, const double* vel_ang,      \
                                             const double* vel_offset, int init_vel) {                                     \
    add_track<S>(h, n_poses, stamps, R, t, pose_offset, vel_lin, vel_ang, vel_offset, init_vel);                           \
  }                                                                                                                        \
  extern "C" void ref_scene_free_##SUF(void* h) { delete (RefH<S>*)h; }                                                    \
  extern "C" const char* ref_scene_error_##SUF(void* h) { return ((RefH<S>*)h)->error.c_str(); }                           \
  extern "C" int64_t ref_view_camera_##SUF(void* h, double t, const double* cam, const double* settings) {                 \
    return view_camera<S>(h, t, cam, settings);                                                                            \
  }                                                                                                                        \
  extern "C" int64_t ref_view_lidar_##SUF(void* h, double t, const double* lidar, const double* elev, int n_beams,         \
                                           const double* settings) {                                                       \
    return view_lidar<S>(h, t, lidar, elev, n_beams, settings);                                                            \
  }                                                                                                                        \
  extern "C" int ref_backward_##SUF(void* h, const S* g_mean2d, const S* g_range, const S* g_cov2d, const S* g_velocity,   \
                                     const S* g_opacity) {                                                                 \
    return backward<S>(h, g_mean2d, g_range, g_cov2d, g_velocity, g_opacity);                                              \
  }                                                                                                                        \
  extern "C" int64_t ref_array_##SUF(void* h, const char* name, void* dst) { return array<S>(h, name, dst); }              \
  extern "C" void ref_covariance_from_scale_quat_##SUF(const S* scale_log, const S* quat, S* out9) {                       \
    const splat::Mat3<S> c = splat::covariance_from_scale_quat<S>(splat::Vec3<S>(scale_log[0], scale_log[1], scale_log[2]), \
                                                                  splat::Vec4<S>(quat[0], quat[1], quat[2], quat[3]));     \
    for (int r = 0; r < 3; ++r)                                                                                            \
      for (int cc = 0; cc < 3; ++cc) out9[3 * r + cc] = c(r, cc);                                                          \
  }                                                                                                                        \
  extern "C" void ref_spherical_##SUF(const S* p, S* sph3, S* J9) {                                                        \
    const splat::Vec3<S> v(p[0], p[1], p[2]);                                                                              \
    const splat::Vec3<S> s = splat::spherical_of<S>(v);                                                                    \
    const splat::Mat3<S> J = splat::spherical_jacobian<S>(v);                                                              \
    for (int k = 0; k < 3; ++k) sph3[k] = s(k);                                                                            \
    for (int r = 0; r < 3; ++r)                                                                                            \
      for (int c = 0; c < 3; ++c) J9[3 * r + c] = J(r, c);                                                                 \
  }                                                                                                                        \
  extern "C" S ref_wrap_pi_##SUF(S a) { return splat::wrap_pi<S>(a); }                                                     \
  extern "C" S ref_wrap_two_pi_##SUF(S a) { return splat::wrap_two_pi<S>(a); }                                             \
  extern "C" S ref_sigmoid_##SUF(S a) { return splat::sigmoid<S>(a); }

REF_API(float, f32)
REF_API(double, f64)

extern "C" void ref_so3_roundtrip(const double* phi3, double* log_of_exp3, double* Jr9, double* Jrinv9) {
  const splat::Vec3<double> phi(phi3[0], phi3[1], phi3[2]);
  const splat::Vec3<double> l = splat::so3_log<double>(splat::so3_exp<double>(phi));
  const splat::Mat3<double> Jr = splat::so3_right_jacobian<double>(phi), Ji = splat::so3_right_jacobian_inv<double>(phi);
  for (int k = 0; k < 3; ++k) log_of_exp3[k] = l(k);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) { Jr9[3 * r + c] = Jr(r, c); Jrinv9[3 * r + c] = Ji(r, c); }
}
