// facade_test.cpp — a caller written against the REFERENCE's API (splat/scene.hpp, splat/projection.hpp)
// that runs every shipped function twice: the reference's CPU implementation and the drop-in from
// include/splat_b200.hpp (sm_100a kernels behind the C ABI), and compares them. Built in the container
// where /root/reference exists (tests/cpp/build.sh; the reference headers compile against
// oracle/eigen_shim); the binary travels to the GPU box and is run by tests/test_cpp_facade.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "splat_b200.hpp"

using namespace splat;

namespace {

int g_fail = 0;

struct Err {
  double worst = 0, q99 = 0;
};

// per-row relative error |a-b| / max(|b| row max, 1e-3 * global max)
Err row_err(const std::vector<std::vector<double>>& a, const std::vector<std::vector<double>>& b) {
  double gmax = 0;
  for (auto& r : b) for (double x : r) gmax = std::max(gmax, std::fabs(x));
  std::vector<double> e;
  for (size_t i = 0; i < a.size(); ++i) {
    double rmax = 1e-3 * gmax, d = 0;
    for (double x : b[i]) rmax = std::max(rmax, std::fabs(x));
    for (size_t k = 0; k < a[i].size(); ++k) d = std::max(d, std::fabs(a[i][k] - b[i][k]));
    e.push_back(rmax > 0 ? d / rmax : d);
  }
  Err out;
  if (e.empty()) return out;
  std::sort(e.begin(), e.end());
  out.worst = e.back();
  out.q99 = e[(size_t)(0.99 * (e.size() - 1))];
  return out;
}

void report(const char* what, Err e, double tol_q99, double tol_worst) {
  const bool ok = e.q99 <= tol_q99 && e.worst <= tol_worst;
  std::printf("  %-34s q99 %.2e  worst %.2e  %s\n", what, e.q99, e.worst, ok ? "ok" : "FAIL");
  if (!ok) ++g_fail;
}

template <class M> std::vector<std::vector<double>> rows_of(const M& m) {  // k x N -> N rows
  std::vector<std::vector<double>> out((size_t)m.cols());
  for (Eigen::Index j = 0; j < m.cols(); ++j)
    for (Eigen::Index i = 0; i < m.rows(); ++i) out[(size_t)j].push_back(m(i, j));
  return out;
}
template <class S> std::vector<std::vector<double>> rows_of(const std::vector<Mat3<S>>& v) {
  std::vector<std::vector<double>> out(v.size());
  for (size_t i = 0; i < v.size(); ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) out[i].push_back(v[i](r, c));
  return out;
}

std::vector<double> flat(const ProjectedGaussian<float>& g) {
  return {g.mean2d(0), g.mean2d(1), g.depth_key, g.cov2d(0, 0), g.cov2d(0, 1), g.cov2d(1, 0), g.cov2d(1, 1), g.velocity(0),
          g.velocity(1), g.velocity(2), g.aabb.lo(0), g.aabb.lo(1), g.aabb.hi(0), g.aabb.hi(1), g.conic(0, 0), g.conic(0, 1),
          g.conic(1, 0), g.conic(1, 1), g.det_ratio, g.mu_sensor(0), g.mu_sensor(1), g.mu_sensor(2), g.rel_vel_sensor(0),
          g.rel_vel_sensor(1), g.rel_vel_sensor(2)};
}

void compare_projected(const char* what, const std::vector<ProjectedGaussian<float>>& cpu, const std::vector<ProjectedGaussian<float>>& gpu) {
  // fp32 exp/atan2 differ in the last ulp between libm and the kernels' deterministic math: a borderline cull may flip
  size_t i = 0, j = 0, common = 0;
  static const char* names[9] = {"mean2d", "depth_key", "cov2d", "velocity", "aabb", "conic", "det_ratio", "mu_sensor", "rel_vel_sensor"};
  static const int off[10] = {0, 2, 3, 7, 10, 14, 18, 19, 22, 25};
  std::vector<std::vector<std::vector<double>>> a(9), b(9);
  while (i < cpu.size() && j < gpu.size()) {
    if (cpu[i].source_index < gpu[j].source_index) { ++i; continue; }
    if (cpu[i].source_index > gpu[j].source_index) { ++j; continue; }
    const auto fa = flat(gpu[j]), fb = flat(cpu[i]);
    for (int f = 0; f < 9; ++f) {
      a[f].emplace_back(fa.begin() + off[f], fa.begin() + off[f + 1]);
      b[f].emplace_back(fb.begin() + off[f], fb.begin() + off[f + 1]);
    }
    ++common; ++i; ++j;
  }
  std::printf("%s: V cpu %zu, gpu %zu, common %zu\n", what, cpu.size(), gpu.size(), common);
  if (common + 2 < 0.999 * cpu.size() || gpu.size() > cpu.size() * 1.001 + 2) { std::printf("  visible sets differ FAIL\n"); ++g_fail; }
  for (int f = 0; f < 9; ++f) report(names[f], row_err(a[f], b[f]), 1e-4, 5e-2);
}

SceneGraph<float> make_graph(int n, int n_actors, Rng& rng) {
  SceneGraph<double> g;
  g.gaussians.resize(n, 13);
  for (int i = 0; i < n; ++i) {
    const double r = uniform<double>(rng, 3.0, 40.0), th = uniform<double>(rng, 0.0, two_pi<double>());
    g.gaussians.mean(0, i) = r * std::cos(th);
    g.gaussians.mean(1, i) = r * std::sin(th);
    g.gaussians.mean(2, i) = uniform<double>(rng, -2.0, 6.0);
    for (int k = 0; k < 3; ++k) g.gaussians.scale_log(k, i) = normal<double>(rng, std::log(0.08), 0.5);
    for (int k = 0; k < 4; ++k) g.gaussians.quat(k, i) = normal<double>(rng);
    g.gaussians.opacity_logit(0, i) = normal<double>(rng, 0.0, 1.5);
    for (int k = 0; k < 3; ++k) g.gaussians.color(k, i) = uniform<double>(rng, 0.0, 1.0);
    for (int k = 0; k < 13; ++k) g.gaussians.feature(k, i) = normal<double>(rng);
    g.gaussians.actor_id(i) = 0;
  }
  for (int a = 0; a < n_actors; ++a) {
    ActorTrack<double> tr;
    tr.pose_offset.setZero(6, 3);
    const double yaw0 = uniform<double>(rng, 0.0, 6.28), rate = uniform<double>(rng, -0.3, 0.3), speed = uniform<double>(rng, 5.0, 20.0);
    for (int s = 0; s < 3; ++s) {
      const double t = -0.1 + 0.1 * s, yaw = yaw0 + rate * t;
      SE3<double> p;
      p.R << std::cos(yaw), -std::sin(yaw), 0.0, std::sin(yaw), std::cos(yaw), 0.0, 0.0, 0.0, 1.0;
      p.t = Vec3<double>(8.0 + 3.0 * a + speed * t * std::cos(yaw0), -3.0 + 2.0 * a + speed * t * std::sin(yaw0), 1.0);
      tr.stamps.push_back(t);
      tr.poses.push_back(p);
      for (int k = 0; k < 6; ++k) tr.pose_offset(k, s) = normal<double>(rng, 0.0, 0.01);
    }
    tr.init_velocity_from_poses();
    for (int k = 0; k < 6; ++k) tr.vel_offset(k) = normal<double>(rng, 0.0, 0.05);
    g.tracks.push_back(tr);
    for (int i = a; i < n; i += 10) {  // every 10th Gaussian rides an actor
      if (i % 10 != a) continue;
      g.gaussians.actor_id(i) = a + 1;
      g.gaussians.mean(0, i) = uniform<double>(rng, -2.25, 2.25);
      g.gaussians.mean(1, i) = uniform<double>(rng, -1.0, 1.0);
      g.gaussians.mean(2, i) = uniform<double>(rng, -0.8, 0.8);
    }
  }
  return g.cast<float>();
}

}  // namespace

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 20000;
  Rng rng(0x5eed0001);
  const SceneGraph<float> graph = make_graph(n, 3, rng);
  const float t = 0.03f;
  const RasterSettings<float> st;

  CameraModel<float> cam;
  cam.fx = cam.fy = 300.0f; cam.cx = 320.0f; cam.cy = 180.0f; cam.width = 640; cam.height = 360;
  cam.pose.R << 0, -1, 0, 0, 0, -1, 1, 0, 0;       // x right, y down, z forward  <-  world x forward, y left, z up
  cam.pose.t = Vec3<float>(0.0f, 1.5f, 0.0f);
  cam.vel_lin = Vec3<float>(0.0f, 0.0f, 15.0f);
  cam.vel_ang = Vec3<float>(0.0f, 0.1f, 0.0f);
  cam.shutter_duration = 0.03f;
  cam.time_offset = 0.002f;

  LidarModel<float> lidar;
  for (int k = 0; k < 64; ++k) lidar.elevation_channels.push_back((-25.0f + 40.0f * (float)k / 63.0f) * pi<float>() / 180.0f);
  lidar.azimuth_resolution = 0.2f * pi<float>() / 180.0f;
  lidar.scan_duration = 0.1f;
  lidar.beam_divergence_h = 3e-3f; lidar.beam_divergence_v = 1.5e-3f;
  lidar.pose.t = Vec3<float>(0.0f, 0.0f, -1.8f);
  lidar.vel_lin = Vec3<float>(12.0f, 1.0f, 0.0f);
  lidar.vel_ang = Vec3<float>(0.0f, 0.02f, 0.3f);

  b200::Context ctx(0);

  // ---- compose_at_time --------------------------------------------------------------------------
  const ComposedScene<float> cpu_scene = compose_at_time<float>(graph, t);
  const ComposedScene<float> gpu_scene = b200::compose_at_time(ctx, graph, t);
  std::printf("compose_at_time: N %ld\n", (long)cpu_scene.size());
  report("mean_w", row_err(rows_of(gpu_scene.mean_w), rows_of(cpu_scene.mean_w)), 1e-5, 1e-4);
  report("cov_w", row_err(rows_of(gpu_scene.cov_w), rows_of(cpu_scene.cov_w)), 1e-4, 1e-3);
  report("vel_dyn_w", row_err(rows_of(gpu_scene.vel_dyn_w), rows_of(cpu_scene.vel_dyn_w)), 1e-4, 1e-3);
  report("opacity", row_err(rows_of(gpu_scene.opacity), rows_of(cpu_scene.opacity)), 1e-5, 1e-4);

  // ---- project_camera / project_lidar -----------------------------------------------------------
  const auto cpu_cam = project_camera<float>(cpu_scene, cam, st);
  const auto gpu_cam = b200::project_camera(ctx, cpu_scene, cam, st);
  compare_projected("project_camera", cpu_cam, gpu_cam);
  const auto cpu_lid = project_lidar<float>(cpu_scene, lidar, st);
  const auto gpu_lid = b200::project_lidar(ctx, cpu_scene, lidar, st);
  compare_projected("project_lidar", cpu_lid, gpu_lid);

  // ---- project_*_backward + compose_backward ----------------------------------------------------
  for (int pass = 0; pass < 2; ++pass) {
    const bool is_cam = pass == 0;
    const auto& proj = is_cam ? gpu_cam : gpu_lid;   // the device's own list (identical up to borderline culls)
    const auto& cpu_proj = is_cam ? cpu_cam : cpu_lid;
    if (proj.size() != cpu_proj.size()) { std::printf("backward %s: skipped (visible sets differ by a borderline cull)\n", is_cam ? "camera" : "lidar"); continue; }
    const Eigen::Index V = (Eigen::Index)proj.size(), N = graph.gaussians.size();
    ProjectedGrads<float> gin;
    gin.resize(V, 13);
    for (Eigen::Index k = 0; k < V; ++k) {
      // well-scaled upstream gradients: d/d(mean2d) in 1/px (or 1/rad), d/d(cov2d) in 1/px^2
      const float s1 = is_cam ? 1.0f : 100.0f;
      gin.g_mean2d(0, k) = s1 * normal<float>(rng); gin.g_mean2d(1, k) = s1 * normal<float>(rng);
      gin.g_range(0, k) = is_cam ? 0.0f : normal<float>(rng);
      for (int r = 0; r < 2; ++r) for (int c = 0; c < 2; ++c) gin.g_cov2d[(size_t)k](r, c) = s1 * s1 * 0.1f * normal<float>(rng);
      for (int c = 0; c < 3; ++c) gin.g_velocity(c, k) = 0.01f * s1 * normal<float>(rng);
      if (is_cam) gin.g_velocity(2, k) = 0.0f;
    }
    MatRX<float, 1> g_op;
    g_op.setZero(1, N);
    for (Eigen::Index i = 0; i < N; ++i) g_op(0, i) = normal<float>(rng);

    ComposeGrads<float> cg_cpu, cg_gpu;
    cg_cpu.resize(N); cg_gpu.resize(N);
    SensorGrads<float> sg_cpu, sg_gpu;
    // the reference's chunked calling convention: two disjoint [begin, end) ranges
    const Eigen::Index mid = V / 3;
    if (is_cam) {
      project_camera_backward<float>(cpu_scene, cam, cpu_proj, gin, cg_cpu, sg_cpu, 0, mid);
      project_camera_backward<float>(cpu_scene, cam, cpu_proj, gin, cg_cpu, sg_cpu, mid, V);
      b200::project_camera_backward(ctx, cpu_scene, cam, proj, gin, cg_gpu, sg_gpu, 0, mid);
      b200::project_camera_backward(ctx, cpu_scene, cam, proj, gin, cg_gpu, sg_gpu, mid, V);
    } else {
      project_lidar_backward<float>(cpu_scene, lidar, cpu_proj, gin, cg_cpu, sg_cpu, 0, mid);
      project_lidar_backward<float>(cpu_scene, lidar, cpu_proj, gin, cg_cpu, sg_cpu, mid, V);
      b200::project_lidar_backward(ctx, cpu_scene, lidar, proj, gin, cg_gpu, sg_gpu, 0, mid);
      b200::project_lidar_backward(ctx, cpu_scene, lidar, proj, gin, cg_gpu, sg_gpu, mid, V);
    }
    std::printf("project_%s_backward: V %ld\n", is_cam ? "camera" : "lidar", (long)V);
    report("ComposeGrads.g_mean_w", row_err(rows_of(cg_gpu.g_mean_w), rows_of(cg_cpu.g_mean_w)), 1e-3, 0.5);
    report("ComposeGrads.g_cov_w", row_err(rows_of(cg_gpu.g_cov_w), rows_of(cg_cpu.g_cov_w)), 1e-3, 0.5);
    report("ComposeGrads.g_vel_dyn_w", row_err(rows_of(cg_gpu.g_vel_dyn_w), rows_of(cg_cpu.g_vel_dyn_w)), 1e-3, 0.5);
    double smax = 0, sdiff = 0;
    for (int k = 0; k < 3; ++k) {
      smax = std::max({smax, (double)std::fabs(sg_cpu.d_vel_lin(k)), (double)std::fabs(sg_cpu.d_vel_ang(k))});
      sdiff = std::max({sdiff, (double)std::fabs(sg_cpu.d_vel_lin(k) - sg_gpu.d_vel_lin(k)), (double)std::fabs(sg_cpu.d_vel_ang(k) - sg_gpu.d_vel_ang(k))});
    }
    std::printf("  %-34s rel %.2e  %s\n", "SensorGrads d_vel_lin/ang", sdiff / smax, sdiff <= 2e-2 * smax ? "ok" : "FAIL");
    if (sdiff > 2e-2 * smax) ++g_fail;

    SceneParamGrads<float> out_cpu, out_gpu;
    out_cpu.resize_like(graph); out_gpu.resize_like(graph);
    compose_backward<float>(cpu_scene, cg_cpu, g_op, out_cpu, 0, N);
    b200::compose_backward(ctx, cpu_scene, cg_cpu, g_op, out_gpu, 0, N);     // same ComposeGrads in
    std::printf("compose_backward:\n");
    report("d_mean", row_err(rows_of(out_gpu.d_mean), rows_of(out_cpu.d_mean)), 1e-3, 0.5);
    report("d_scale_log", row_err(rows_of(out_gpu.d_scale_log), rows_of(out_cpu.d_scale_log)), 1e-3, 0.5);
    report("d_quat", row_err(rows_of(out_gpu.d_quat), rows_of(out_cpu.d_quat)), 1e-3, 0.5);
    report("d_opacity_logit", row_err(rows_of(out_gpu.d_opacity_logit), rows_of(out_cpu.d_opacity_logit)), 1e-3, 0.5);
    for (size_t a = 0; a < graph.tracks.size(); ++a) {
      report("ActorGrad.d_pose_offset", row_err(rows_of(out_gpu.actors[a].d_pose_offset), rows_of(out_cpu.actors[a].d_pose_offset)), 5e-2, 5e-2);
      report("ActorGrad.d_vel_offset", row_err(rows_of(out_gpu.actors[a].d_vel_offset), rows_of(out_cpu.actors[a].d_vel_offset)), 5e-2, 5e-2);
    }
  }

  // ---- error behaviour (scene.hpp:297-298) -------------------------------------------------------
  {
    SceneGraph<float> bad = graph;
    bad.gaussians.actor_id(17) = 9;
    bool cpu_threw = false, gpu_threw = false;
    std::string cpu_msg, gpu_msg;
    try { compose_at_time<float>(bad, t); } catch (const std::out_of_range& e) { cpu_threw = true; cpu_msg = e.what(); }
    try { b200::compose_at_time(ctx, bad, t); } catch (const std::out_of_range& e) { gpu_threw = true; gpu_msg = e.what(); }
    const bool ok = cpu_threw && gpu_threw && cpu_msg == gpu_msg;
    std::printf("unknown actor id: cpu '%s' gpu '%s' %s\n", cpu_msg.c_str(), gpu_msg.c_str(), ok ? "ok" : "FAIL");
    if (!ok) ++g_fail;
  }

  // ---- the SPEC-only modules through the same façade: rasterize + fused backward ------------------
  {
    ctx.upload(graph);
    b200::SensorView view(ctx, cam, st);
    view.forward(t);
    ChannelImage<float> img;
    std::vector<float> alpha;
    std::vector<int32_t> nc;
    view.download(img, alpha, nc, cam.height, cam.width);
    double amin = 1e9, amax = -1e9;
    long contrib = 0;
    for (size_t k = 0; k < alpha.size(); ++k) { amin = std::min(amin, (double)alpha[k]); amax = std::max(amax, (double)alpha[k]); contrib += nc[k]; }
    const bool ok = amin >= 0.0 && amax <= 1.0 && contrib > 0;
    std::printf("rasterize_camera: alpha in [%.3f, %.3f], %ld blended pairs %s\n", amin, amax, contrib, ok ? "ok" : "FAIL");
    if (!ok) ++g_fail;
    ChannelImage<float> g(16, cam.height, cam.width);
    for (Eigen::Index k = 0; k < g.data.cols(); ++k) for (int c = 0; c < 16; ++c) g.data(c, k) = normal<float>(rng);
    std::vector<float> ga(alpha.size(), 0.5f);
    ctx.zero_grads();
    view.backward(g, ga);
    SceneParamGrads<float> out;
    out.resize_like(graph);
    ctx.drain_grads_into(out);
    double gsum = 0;
    for (Eigen::Index i = 0; i < out.d_mean.cols(); ++i) for (int k = 0; k < 3; ++k) gsum += std::fabs(out.d_mean(k, i));
    std::printf("fused backward: sum |d_mean| = %.4e %s\n", gsum, (gsum > 0 && std::isfinite(gsum)) ? "ok" : "FAIL");
    if (!(gsum > 0 && std::isfinite(gsum))) ++g_fail;
  }

  std::printf(g_fail ? "FACADE TEST FAILED (%d)\n" : "FACADE TEST PASSED\n", g_fail);
  return g_fail ? 1 : 0;
}
