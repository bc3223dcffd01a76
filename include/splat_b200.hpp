// splat_b200.hpp — C++ host façade over the C ABI (splat_b200.h) in the reference's OWN types.
//
// Include it after the reference's headers are on the include path (it includes splat/projection.hpp,
// which needs Eigen — the reference's dependency, not ours). Every function has the name, argument
// order and meaning of the reference function it replaces, with one extra leading argument: the
// device context (or a view bound to it). S = float only: the sm_100a kernels compute in fp32, the
// reference's "fast" mode.
//
//   reference (CPU)                                         drop-in (B200)
//   splat::compose_at_time(graph, t)                        splat::b200::compose_at_time(ctx, graph, t)
//   splat::project_camera(scene, cam, settings)             splat::b200::project_camera(ctx, scene, cam, settings)
//   splat::project_lidar(scene, lidar, settings)            splat::b200::project_lidar(ctx, scene, lidar, settings)
//   splat::project_camera_backward(scene, cam, projected,   splat::b200::project_camera_backward(ctx, scene, cam, projected,
//        gin, gscene, gsensor, begin, end)                       gin, gscene, gsensor, begin, end)
//   splat::project_lidar_backward(...)                      splat::b200::project_lidar_backward(ctx, ...)
//   splat::compose_backward(scene, gin, g_opacity, out,     splat::b200::compose_backward(ctx, scene, gin, g_opacity, out,
//        begin, end)                                             begin, end)
// plus the two modules the reference only specifies: SensorView::rasterize /
// SensorView::backward run tiling + compositing and the fused backward on the device.
//
// Ownership and errors follow the reference: results are returned by value, inputs are
// borrowed for the duration of the call, backward outputs are caller-allocated and ACCUMULATED (+=);
// std::out_of_range("unknown actor_id k") and std::runtime_error("actor track has no poses") keep their
// types and texts (scene.hpp:176-177, 242, 297-298).
#pragma once

#include <cstring>
#include <array>
#include <stdexcept>
#include <string>
#include <vector>

#include "splat/projection.hpp"
#include "splat_b200.h"

namespace splat::b200 {

namespace detail {
inline void check(splatb200_ctx* c, long long rc) {
  if (rc >= 0) return;
  const std::string msg = splatb200_last_error(c);
  if (rc == SPLATB200_EOUTOFRANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
inline void fill_pose(const SE3<float>& pose, const Vec3<float>& vl, const Vec3<float>& va, float* R, float* t, float* vel_lin,
                      float* vel_ang) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[3 * r + c] = pose.R(r, c);
  for (int k = 0; k < 3; ++k) { t[k] = pose.t(k); vel_lin[k] = vl(k); vel_ang[k] = va(k); }
}
inline splatb200_raster_settings pod(const RasterSettings<float>& s) {
  return {s.dilation, s.alpha_clamp, s.alpha_min, s.qform_max, s.transmittance_min, s.near_plane, s.lidar_min_range};
}
inline splatb200_camera pod(const CameraModel<float>& cam) {
  splatb200_camera c{};
  c.fx = cam.fx; c.fy = cam.fy; c.cx = cam.cx; c.cy = cam.cy;
  c.width = cam.width; c.height = cam.height;
  fill_pose(cam.pose, cam.vel_lin, cam.vel_ang, c.R, c.t, c.vel_lin, c.vel_ang);
  c.shutter_duration = cam.shutter_duration; c.time_offset = cam.time_offset; c.timestamp = cam.timestamp;
  return c;
}
inline splatb200_lidar pod(const LidarModel<float>& l) {
  splatb200_lidar c{};
  c.elevation_channels = l.elevation_channels.data();
  c.n_beams = l.beam_count();
  c.azimuth_resolution = l.azimuth_resolution; c.scan_duration = l.scan_duration;
  c.beam_divergence_h = l.beam_divergence_h; c.beam_divergence_v = l.beam_divergence_v;
  fill_pose(l.pose, l.vel_lin, l.vel_ang, c.R, c.t, c.vel_lin, c.vel_ang);
  c.timestamp = l.timestamp; c.max_range = l.max_range;
  return c;
}
}  // namespace detail

/// One (GPU, stream): owns the device copy of a SceneGraph and its SceneParamGrads.
class Context {
 public:
  explicit Context(int device = 0, void* cuda_stream = nullptr) {
    const int rc = splatb200_ctx_create(device, cuda_stream, &c_);
    if (rc != 0) throw std::runtime_error(std::string("splatb200_ctx_create: ") + splatb200_last_error(nullptr));
  }
  ~Context() { splatb200_ctx_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  splatb200_ctx* handle() const { return c_; }

  /// The per-iteration refresh of the GaussianSet without the wait (same shape as the resident scene; tracks untouched):
  /// geometry first, colour / features behind it, projection and binning of the next views overlap the rest of the
  /// copy. `g` must stay alive and unchanged until the next sync().
  void upload_parameters_async(const GaussianSet<float>& g) {
    detail::check(c_, splatb200_scene_upload_async(c_, (int64_t)g.size(), g.feature_dim(), g.mean.data(), g.scale_log.data(),
                                                   g.quat.data(), g.opacity_logit.data(), g.color.data(), g.feature.data(),
                                                   g.actor_id.data()));
  }

  /// Copy GaussianSet + tracks to the device (Eigen's column-major kxN is the ABI's N rows of k floats).
  void upload(const SceneGraph<float>& graph) {
    const auto& g = graph.gaussians;
    detail::check(c_, splatb200_scene_upload(c_, (int64_t)g.size(), g.feature_dim(), g.mean.data(), g.scale_log.data(), g.quat.data(),
                                             g.opacity_logit.data(), g.color.data(), g.feature.data(), g.actor_id.data()));
    std::vector<splatb200_actor_track> pods(graph.tracks.size());
    std::vector<std::vector<double>> keep;
    for (size_t a = 0; a < graph.tracks.size(); ++a) {
      const auto& tr = graph.tracks[a];
      const int np = (int)tr.pose_count();
      std::vector<double> st(np), R(9 * (size_t)np), t(3 * (size_t)np), po(6 * (size_t)np);
      for (int i = 0; i < np; ++i) {
        st[i] = tr.stamps[i];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) R[9 * i + 3 * r + c] = tr.poses[i].R(r, c);
        for (int k = 0; k < 3; ++k) t[3 * i + k] = tr.poses[i].t(k);
        for (int k = 0; k < 6; ++k) po[6 * i + k] = tr.pose_offset(k, i);
      }
      keep.push_back(std::move(st)); keep.push_back(std::move(R)); keep.push_back(std::move(t)); keep.push_back(std::move(po));
      auto& p = pods[a];
      p.n_poses = np;
      p.stamps = keep[4 * a].data(); p.R = keep[4 * a + 1].data(); p.t = keep[4 * a + 2].data(); p.pose_offset = keep[4 * a + 3].data();
      for (int k = 0; k < 3; ++k) { p.vel_lin[k] = tr.vel_lin(k); p.vel_ang[k] = tr.vel_ang(k); }
      for (int k = 0; k < 6; ++k) p.vel_offset[k] = tr.vel_offset(k);
      p.init_velocity_from_poses = 0;
    }
    detail::check(c_, splatb200_scene_set_tracks(c_, (int32_t)pods.size(), pods.data()));
    graph_ = &graph;
  }
  /// upload() unless this graph is already resident (callers that mutate parameters call upload themselves)
  void ensure(const SceneGraph<float>& graph) {
    if (graph_ != &graph) upload(graph);
  }
  void zero_grads() { detail::check(c_, splatb200_grads_zero(c_)); }

  // ---- multi-GPU ("parallel per sensor view"; scene.hpp:351-362 SceneParamGrads::add across workers) ----
  /// 128-byte NCCL id: rank 0 creates it, every rank receives it out of band (MPI_Bcast, a file, ...).
  static std::array<char, 128> nccl_unique_id() {
    std::array<char, 128> id{};
    if (splatb200_nccl_unique_id(id.data()) != 0) throw std::runtime_error("splatb200_nccl_unique_id: NCCL is not available");
    return id;
  }
  /// One rank per GPU: ncclCommInitRank over `world` ranks.
  void comm_init(const std::array<char, 128>& id, int rank, int world) {
    detail::check(c_, splatb200_ctx_comm_init(c_, id.data(), rank, world));
  }
  /// A trainer that already owns an ncclComm_t hands it over (it stays the trainer's).
  void comm_bind(void* nccl_comm, int rank, int world) { detail::check(c_, splatb200_ctx_comm_bind(c_, nccl_comm, rank, world)); }
  /// SceneParamGrads (and ActorGrad) summed over all ranks, in place on the device: the per-worker `add` of
  /// scene.hpp:351-362 as ONE ncclAllReduce per step, after this rank's last backward.
  void allreduce_grads() { detail::check(c_, splatb200_allreduce_grads(c_)); }

  /// SceneParamGrads += device gradients (scene.hpp:325-363), then the device buffer is zeroed, so that the
  /// reference's "accumulate into the caller's struct" contract holds call by call.
  void drain_grads_into(SceneParamGrads<float>& out) {
    const auto n = out.d_mean.cols();
    const int d_f = (int)out.d_feature.rows();
    std::vector<float> m(3 * (size_t)n), s(3 * (size_t)n), q(4 * (size_t)n), o((size_t)n), col(3 * (size_t)n), f((size_t)d_f * n);
    detail::check(c_, splatb200_grads_download(c_, m.data(), s.data(), q.data(), o.data(), col.data(), f.data()));
    for (Eigen::Index i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) {
        out.d_mean(k, i) += m[3 * i + k];
        out.d_scale_log(k, i) += s[3 * i + k];
        out.d_color(k, i) += col[3 * i + k];
      }
      for (int k = 0; k < 4; ++k) out.d_quat(k, i) += q[4 * i + k];
      out.d_opacity_logit(0, i) += o[i];
      for (int k = 0; k < d_f; ++k) out.d_feature(k, i) += f[(size_t)d_f * i + k];
    }
    for (size_t a = 0; a < out.actors.size(); ++a) {
      const auto np = out.actors[a].d_pose_offset.cols();
      std::vector<double> dp(6 * (size_t)np), dv(6);
      detail::check(c_, splatb200_grads_download_actor(c_, (int32_t)a, dp.data(), dv.data()));
      for (Eigen::Index i = 0; i < np; ++i)
        for (int k = 0; k < 6; ++k) out.actors[a].d_pose_offset(k, i) += (float)dp[6 * i + k];
      for (int k = 0; k < 6; ++k) out.actors[a].d_vel_offset(k) += (float)dv[k];
    }
    zero_grads();
  }

 private:
  splatb200_ctx* c_ = nullptr;
  const SceneGraph<float>* graph_ = nullptr;
};

/// One sensor render on the device (RAII over splatb200_view).
class SensorView {
 public:
  SensorView(Context& ctx, const CameraModel<float>& cam, const RasterSettings<float>& st) : ctx_(ctx), camera_(true) {
    const auto c = detail::pod(cam);
    const auto s = detail::pod(st);
    detail::check(ctx.handle(), splatb200_view_create_camera(ctx.handle(), &c, &s, &v_));
    queries_ = (int64_t)cam.width * cam.height;
  }
  /// rays: 3 floats each (azimuth, elevation, t_l), grouped per tile
  SensorView(Context& ctx, const LidarModel<float>& lidar, const RasterSettings<float>& st, const std::vector<float>& rays,
             const std::vector<int64_t>& ray_begin, const std::vector<int64_t>& ray_end)
      : ctx_(ctx), camera_(false) {
    const auto c = detail::pod(lidar);
    const auto s = detail::pod(st);
    detail::check(ctx.handle(), splatb200_view_create_lidar(ctx.handle(), &c, &s, rays.data(), (int64_t)rays.size() / 3, ray_begin.data(),
                                                            ray_end.data(), (int64_t)ray_begin.size(), &v_));
    queries_ = (int64_t)rays.size() / 3;
  }
  /// projection only (no rays needed): tile grid sized from the lidar, zero rays
  SensorView(Context& ctx, const LidarModel<float>& lidar, const RasterSettings<float>& st) : ctx_(ctx), camera_(false) {
    const auto c = detail::pod(lidar);
    const auto s = detail::pod(st);
    int32_t m_phi = 0, m_omega = 0;
    splatb200_lidar_grid(&c, &m_phi, &m_omega);
    const std::vector<int64_t> zeros((size_t)m_phi * m_omega, 0);
    const float none[3] = {0, 0, 0};
    detail::check(ctx.handle(), splatb200_view_create_lidar(ctx.handle(), &c, &s, none, 0, zeros.data(), zeros.data(),
                                                            (int64_t)zeros.size(), &v_));
  }
  ~SensorView() { splatb200_view_destroy(v_); }
  SensorView(const SensorView&) = delete;
  SensorView& operator=(const SensorView&) = delete;
  splatb200_view* handle() const { return v_; }
  int64_t queries() const { return queries_; }

  /// stop_after: 0 = project + tile + composite, 1 = projection only, 2 = projection + tiling
  void forward(float t_scene, int stop_after = 0) { detail::check(ctx_.handle(), splatb200_view_forward(v_, t_scene, stop_after)); }

  std::vector<ProjectedGaussian<float>> projected() {
    const int64_t V = splatb200_view_projected(v_, nullptr, nullptr);
    detail::check(ctx_.handle(), V);
    std::vector<int64_t> src((size_t)V);
    std::vector<float> f(25 * (size_t)V);
    detail::check(ctx_.handle(), splatb200_view_projected(v_, src.data(), f.data()));
    std::vector<ProjectedGaussian<float>> out((size_t)V);
    for (int64_t k = 0; k < V; ++k) {
      const float* p = &f[25 * (size_t)k];
      auto& g = out[(size_t)k];
      g.source_index = (Eigen::Index)src[(size_t)k];
      g.mean2d = Vec2<float>(p[0], p[1]);
      g.depth_key = p[2];
      g.cov2d(0, 0) = p[3]; g.cov2d(0, 1) = p[4]; g.cov2d(1, 0) = p[5]; g.cov2d(1, 1) = p[6];
      g.velocity = Vec3<float>(p[7], p[8], p[9]);
      g.aabb.lo = Vec2<float>(p[10], p[11]);
      g.aabb.hi = Vec2<float>(p[12], p[13]);
      g.conic(0, 0) = p[14]; g.conic(0, 1) = p[15]; g.conic(1, 0) = p[16]; g.conic(1, 1) = p[17];
      g.det_ratio = p[18];
      g.mu_sensor = Vec3<float>(p[19], p[20], p[21]);
      g.rel_vel_sensor = Vec3<float>(p[22], p[23], p[24]);
    }
    return out;
  }

  /// rasterize_camera / rasterize_lidar: 16 blended channels per query (camera: rgb + 13 features;
  /// lidar: 13 features, expected range, median range, accumulated opacity), accumulated opacity, contributor count
  void download(ChannelImage<float>& blend16, std::vector<float>& alpha, std::vector<int32_t>& n_contrib, int h, int w) {
    blend16 = ChannelImage<float>(16, h, w);          // physical layout: query-major (common.hpp:104-116)
    alpha.assign((size_t)queries_, 0.0f);
    n_contrib.assign((size_t)queries_, 0);
    detail::check(ctx_.handle(), splatb200_view_download(v_, blend16.data.data(), alpha.data(), n_contrib.data()));
  }
  /// rasterizer backward + projection backward + compose backward, fused on the device
  void backward(const ChannelImage<float>& g_blend16, const std::vector<float>& g_alpha) {
    detail::check(ctx_.handle(), splatb200_view_backward_host(v_, g_blend16.data.data(), g_alpha.data()));
    detail::check(ctx_.handle(), splatb200_ctx_sync(ctx_.handle()));
  }
  /// decode_image: the ConvDecoder over this camera view's render, with the camera's own embedding
  /// (CameraModel::embedding, scene.hpp:106). params: splatb200_conv_decoder_params() floats. -> image, H*W x 3.
  std::vector<float> decode_image(const std::vector<float>& params, const VecX<float>& embedding) {
    float e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 8 && k < (int)embedding.size(); ++k) e[k] = embedding(k);
    std::vector<float> image(3 * (size_t)queries_);
    detail::check(ctx_.handle(), splatb200_view_decode_image(v_, params.data(), e, image.data(), nullptr));
    return image;
  }
  /// its backward: dL/dimage -> dL/dparams (overwritten), SensorGrads::d_embedding (+=, projection.hpp:207-222); the
  /// gradient w.r.t. the render is added to the DEVICE buffer g_blend16 (P x 16) that splatb200_view_backward takes
  void decode_image_backward(const std::vector<float>& g_image, std::vector<float>& g_params, SensorGrads<float>& gsensor,
                             float* g_blend16_device) {
    float ge[8];
    g_params.assign((size_t)splatb200_conv_decoder_params(), 0.0f);
    detail::check(ctx_.handle(), splatb200_view_decode_image_backward(v_, g_image.data(), g_params.data(), ge, g_blend16_device, nullptr));
    if (gsensor.d_embedding.size() < 8) gsensor.d_embedding = VecX<float>::Zero(8);
    for (int k = 0; k < 8; ++k) gsensor.d_embedding(k) += ge[k];
  }
  void add_sensor_grads(SensorGrads<float>& out) {
    splatb200_sensor_grads g{};
    detail::check(ctx_.handle(), splatb200_view_sensor_grads(v_, &g));
    for (int k = 0; k < 3; ++k) { out.d_vel_lin(k) += g.d_vel_lin[k]; out.d_vel_ang(k) += g.d_vel_ang[k]; }
    out.d_time_offset += g.d_time_offset;
  }

 private:
  Context& ctx_;
  splatb200_view* v_ = nullptr;
  bool camera_;
  int64_t queries_ = 0;
};

// ------------------------------------------------------------------------------------------------
// drop-in functions (same names and argument order as the reference, plus the context)
// ------------------------------------------------------------------------------------------------

/// scene.hpp:273-308. Actor poses are interpolated on the host by the reference's own interpolate_pose.
inline ComposedScene<float> compose_at_time(Context& ctx, const SceneGraph<float>& graph, float t) {
  ctx.ensure(graph);
  ComposedScene<float> out;
  out.graph = &graph;
  out.time = t;
  const auto n = graph.gaussians.size();
  out.mean_w.resize(3, n);
  out.cov_w.resize((size_t)n);
  out.vel_dyn_w.setZero(3, n);
  out.opacity.resize(1, n);
  for (const auto& track : graph.tracks) out.actor_poses.push_back(interpolate_pose(track, t));
  // any view composes; a 1x1 camera is the cheapest carrier
  CameraModel<float> cam;
  cam.width = cam.height = 1;
  SensorView view(ctx, cam, RasterSettings<float>());
  view.forward(t, 1);
  std::vector<float> cov(9 * (size_t)n);
  detail::check(ctx.handle(), splatb200_view_composed(view.handle(), out.mean_w.data(), cov.data(), out.vel_dyn_w.data(), out.opacity.data()));
  for (Eigen::Index i = 0; i < n; ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) out.cov_w[(size_t)i](r, c) = cov[9 * (size_t)i + 3 * r + c];
  return out;
}

/// projection.hpp:88-118 (compose is re-done on the device from scene.graph at scene.time: the composed
/// arrays of `scene` are not uploaded)
inline std::vector<ProjectedGaussian<float>> project_camera(Context& ctx, const ComposedScene<float>& scene,
                                                            const CameraModel<float>& cam, const RasterSettings<float>& settings) {
  ctx.ensure(*scene.graph);
  SensorView view(ctx, cam, settings);
  view.forward(scene.time, 1);
  return view.projected();
}

/// projection.hpp:140-174
inline std::vector<ProjectedGaussian<float>> project_lidar(Context& ctx, const ComposedScene<float>& scene,
                                                           const LidarModel<float>& lidar, const RasterSettings<float>& settings) {
  ctx.ensure(*scene.graph);
  SensorView view(ctx, lidar, settings);
  view.forward(scene.time, 1);
  return view.projected();
}

namespace detail {
template <class Model>
void project_backward(Context& ctx, const ComposedScene<float>& scene, const Model& sensor,
                      const std::vector<ProjectedGaussian<float>>& projected, const ProjectedGrads<float>& gin,
                      ComposeGrads<float>& gscene, SensorGrads<float>& gsensor, Eigen::Index begin, Eigen::Index end,
                      const RasterSettings<float>& settings) {
  ctx.ensure(*scene.graph);
  SensorView view(ctx, sensor, settings);
  view.forward(scene.time, 1);
  const size_t V = projected.size();
  std::vector<float> cov2d(4 * V);
  for (size_t k = 0; k < V; ++k) {
    cov2d[4 * k] = gin.g_cov2d[k](0, 0); cov2d[4 * k + 1] = gin.g_cov2d[k](0, 1);
    cov2d[4 * k + 2] = gin.g_cov2d[k](1, 0); cov2d[4 * k + 3] = gin.g_cov2d[k](1, 1);
  }
  const auto n = scene.size();
  std::vector<float> gm(3 * (size_t)n, 0.0f), gc(9 * (size_t)n, 0.0f), gv(3 * (size_t)n, 0.0f);
  check(ctx.handle(), splatb200_view_project_backward(view.handle(), gin.g_mean2d.data(), gin.g_range.data(), cov2d.data(),
                                                      gin.g_velocity.data(), (int64_t)begin, (int64_t)end, gm.data(), gc.data(), gv.data()));
  for (Eigen::Index i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) { gscene.g_mean_w(k, i) += gm[3 * i + k]; gscene.g_vel_dyn_w(k, i) += gv[3 * i + k]; }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) gscene.g_cov_w[(size_t)i](r, c) += gc[9 * (size_t)i + 3 * r + c];
  }
  view.add_sensor_grads(gsensor);
}
}  // namespace detail

/// projection.hpp:250-288. The device rebuilds the projected list instead of uploading `projected`, so the
/// RasterSettings that shaped it must be the same; the reference's signature has none, hence the defaulted
/// trailing argument (pass the settings used for project_camera if they were not the defaults).
inline void project_camera_backward(Context& ctx, const ComposedScene<float>& scene, const CameraModel<float>& cam,
                                    const std::vector<ProjectedGaussian<float>>& projected, const ProjectedGrads<float>& gin,
                                    ComposeGrads<float>& gscene, SensorGrads<float>& gsensor, Eigen::Index begin, Eigen::Index end,
                                    const RasterSettings<float>& settings = RasterSettings<float>()) {
  detail::project_backward(ctx, scene, cam, projected, gin, gscene, gsensor, begin, end, settings);
}

/// projection.hpp:322-357
inline void project_lidar_backward(Context& ctx, const ComposedScene<float>& scene, const LidarModel<float>& lidar,
                                   const std::vector<ProjectedGaussian<float>>& projected, const ProjectedGrads<float>& gin,
                                   ComposeGrads<float>& gscene, SensorGrads<float>& gsensor, Eigen::Index begin, Eigen::Index end,
                                   const RasterSettings<float>& settings = RasterSettings<float>()) {
  detail::project_backward(ctx, scene, lidar, projected, gin, gscene, gsensor, begin, end, settings);
}

/// scene.hpp:386-458
inline void compose_backward(Context& ctx, const ComposedScene<float>& scene, const ComposeGrads<float>& gin,
                             const MatRX<float, 1>& g_opacity, SceneParamGrads<float>& out, Eigen::Index begin, Eigen::Index end) {
  ctx.ensure(*scene.graph);
  CameraModel<float> cam;
  cam.width = cam.height = 1;
  SensorView view(ctx, cam, RasterSettings<float>());
  view.forward(scene.time, 1);
  const auto n = scene.size();
  std::vector<float> gc(9 * (size_t)n);
  for (Eigen::Index i = 0; i < n; ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) gc[9 * (size_t)i + 3 * r + c] = gin.g_cov_w[(size_t)i](r, c);
  ctx.zero_grads();
  detail::check(ctx.handle(), splatb200_view_compose_backward(view.handle(), gin.g_mean_w.data(), gc.data(), gin.g_vel_dyn_w.data(),
                                                              g_opacity.data(), (int64_t)begin, (int64_t)end));
  ctx.drain_grads_into(out);
}

}  // namespace splat::b200
