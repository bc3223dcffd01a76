// oracle_capi.cpp — C entry points over splat_oracle.hpp for ctypes (tests/, bench.py cpu_baseline).
// TEST INFRASTRUCTURE ONLY; see the header of splat_oracle.hpp.
//
// Every function exists twice, suffixed _f32 and _f64 (SPEC.md:87 fast32 / test64).
// Sensor structs travel as packed double arrays:
//   cam[27]   = fx fy cx cy width height | R(9 row-major) | t(3) | vel_lin(3) | vel_ang(3) | shutter time_offset timestamp
//   lidar[24] = azimuth_res scan_duration div_h div_v | R(9) | t(3) | vel_lin(3) | vel_ang(3) | timestamp max_range
//   settings[7] = dilation alpha_clamp alpha_min qform_max transmittance_min near_plane lidar_min_range
#include <chrono>
#include <cstdio>
#include <map>

#include "splat_oracle.hpp"
#include "decoder_oracle.hpp"

using namespace orc;

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class S> struct SceneH {
  SceneGraph<S> graph;
  SceneParamGrads<S> grads;
  bool grads_ready = false;
  std::string error;
};

template <class S> struct ViewH {
  SceneH<S>* sh = nullptr;
  bool camera = true;
  CameraModel<S> cam;
  LidarModel<S> lidar;
  LidarGrid<S> grid;
  RasterSettings<S> st;
  ComposedScene<S> scene;
  std::vector<Projected<S>> proj;
  std::vector<TileRect> rects;
  Worklist wl;
  std::vector<Ray<S>> rays;
  std::vector<int64_t> ray_begin, ray_end;
  std::vector<S> los_cut, g_los;   // optional line-of-sight channel: per-ray cut r_p - eps, upstream gradient
  RasterOut<S> out;
  RasterGrads<S> rg;
  ProjectedGrads<S> pg;
  ComposeGrads<S> cg;
  SensorGrads<S> sg;
  double ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // compose, project, tiling, raster, raster_bwd, epilogue, project_bwd, compose_bwd
};

template <class S> RasterSettings<S> unpack_settings(const double* s) {
  RasterSettings<S> st;
  st.dilation = S(s[0]); st.alpha_clamp = S(s[1]); st.alpha_min = S(s[2]); st.qform_max = S(s[3]);
  st.transmittance_min = S(s[4]); st.near_plane = S(s[5]); st.lidar_min_range = S(s[6]);
  return st;
}
template <class S> void unpack_pose(const double* p, SE3<S>& pose, V3<S>& vl, V3<S>& va) {
  for (int i = 0; i < 9; ++i) pose.R.m[i] = S(p[i]);
  pose.t = V3<S>(S(p[9]), S(p[10]), S(p[11]));
  vl = V3<S>(S(p[12]), S(p[13]), S(p[14]));
  va = V3<S>(S(p[15]), S(p[16]), S(p[17]));
}
template <class S> CameraModel<S> unpack_camera(const double* c) {
  CameraModel<S> cam;
  cam.fx = S(c[0]); cam.fy = S(c[1]); cam.cx = S(c[2]); cam.cy = S(c[3]);
  cam.width = (int)c[4]; cam.height = (int)c[5];
  unpack_pose<S>(c + 6, cam.pose, cam.vel_lin, cam.vel_ang);
  cam.shutter_duration = S(c[24]); cam.time_offset = S(c[25]); cam.timestamp = S(c[26]);
  return cam;
}
template <class S> LidarModel<S> unpack_lidar(const double* l, const double* elev, int n_beams) {
  LidarModel<S> m;
  m.azimuth_resolution = S(l[0]); m.scan_duration = S(l[1]); m.beam_divergence_h = S(l[2]); m.beam_divergence_v = S(l[3]);
  unpack_pose<S>(l + 4, m.pose, m.vel_lin, m.vel_ang);
  m.timestamp = S(l[22]); m.max_range = S(l[23]);
  for (int i = 0; i < n_beams; ++i) m.elevation_channels.push_back(S(elev[i]));
  return m;
}

template <class S>
void* scene_new(int64_t n, int d_f, const S* mean, const S* scale_log, const S* quat, const S* opacity_logit,
                const S* color, const S* feature, const int32_t* actor_id) {
  auto* h = new SceneH<S>();
  auto& g = h->graph.gaussians;
  g.n = n; g.d_f = d_f;
  g.mean.assign(mean, mean + 3 * n);
  g.scale_log.assign(scale_log, scale_log + 3 * n);
  g.quat.assign(quat, quat + 4 * n);
  g.opacity_logit.assign(opacity_logit, opacity_logit + n);
  g.color.assign(color, color + 3 * n);
  g.feature.assign(feature, feature + (int64_t)d_f * n);
  g.actor_id.assign(actor_id, actor_id + n);
  return h;
}

template <class S>
void scene_add_track(void* hv, int n_poses, const double* stamps, const double* R, const double* t,
                     const double* pose_offset, const double* vel_lin, const double* vel_ang, const double* vel_offset,
                     int init_vel) {
  auto* h = (SceneH<S>*)hv;
  ActorTrack tr;
  for (int i = 0; i < n_poses; ++i) {
    tr.stamps.push_back(stamps[i]);
    SE3<double> p;
    for (int k = 0; k < 9; ++k) p.R.m[k] = R[9 * i + k];
    p.t = V3d(t[3 * i], t[3 * i + 1], t[3 * i + 2]);
    tr.poses.push_back(p);
  }
  tr.pose_offset.assign(pose_offset, pose_offset + 6 * n_poses);
  if (init_vel) {
    tr.init_velocity_from_poses();
  } else {
    tr.vel_lin = V3d(vel_lin[0], vel_lin[1], vel_lin[2]);
    tr.vel_ang = V3d(vel_ang[0], vel_ang[1], vel_ang[2]);
  }
  for (int k = 0; k < 6; ++k) tr.vel_offset[k] = vel_offset[k];
  h->graph.tracks.push_back(tr);
}

template <class S> void view_forward(ViewH<S>* v, double t_scene, int workers, int stop_after) {
  auto& h = *v->sh;
  double t0 = now_ms();
  v->scene = compose_at_time<S>(h.graph, S(t_scene), workers);
  double t1 = now_ms();
  v->ms[0] = t1 - t0;
  if (v->camera) v->proj = project_camera<S>(v->scene, v->cam, v->st, workers);
  else v->proj = project_lidar<S>(v->scene, v->lidar, v->st, workers);
  double t2 = now_ms();
  v->ms[1] = t2 - t1;
  if (stop_after == 1) return;
  int tx, ty;
  if (v->camera) {
    tx = (v->cam.width + kTile - 1) / kTile;
    ty = (v->cam.height + kTile - 1) / kTile;
  } else {
    v->grid = make_lidar_grid<S>(v->lidar);
    tx = v->grid.m_phi;
    ty = v->grid.m_omega;
  }
  v->rects.resize(v->proj.size());
  for (size_t k = 0; k < v->proj.size(); ++k)
    v->rects[k] = v->camera ? image_tile_range<S>(v->proj[k].aabb_lo, v->proj[k].aabb_hi, tx, ty)
                            : lidar_tile_range<S>(v->proj[k].aabb_lo, v->proj[k].aabb_hi, v->grid);
  size_t cursor = 0;
  v->wl = build_sorted_worklist<S>(v->proj, tx, ty, !v->camera, [&](const Projected<S>&) { return v->rects[cursor++]; });
  double t3 = now_ms();
  v->ms[2] = t3 - t2;
  if (stop_after == 2) return;
  if (v->camera) v->out = rasterize_camera<S>(v->wl, v->proj, v->scene, v->cam, v->st, workers);
  else v->out = rasterize_lidar<S>(v->wl, v->proj, v->scene, v->rays, v->ray_begin, v->ray_end, v->st, workers,
                                   v->los_cut.empty() ? nullptr : &v->los_cut);
  v->ms[3] = now_ms() - t3;
}

template <class S>
void* view_camera(void* sh, double t_scene, const double* cam, const double* settings, int workers, int stop_after) {
  auto* v = new ViewH<S>();
  v->sh = (SceneH<S>*)sh;
  v->camera = true;
  v->cam = unpack_camera<S>(cam);
  v->st = unpack_settings<S>(settings);
  try {
    view_forward(v, t_scene, workers, stop_after);
  } catch (const std::exception& e) {
    v->sh->error = e.what();
    delete v;
    return nullptr;
  }
  return v;
}

template <class S>
void* view_lidar(void* sh, double t_scene, const double* lidar, const double* elev, int n_beams, const double* settings,
                 const S* rays, int64_t n_rays, const int64_t* ray_begin, const int64_t* ray_end, int64_t n_tiles,
                 int workers, int stop_after) {
  auto* v = new ViewH<S>();
  v->sh = (SceneH<S>*)sh;
  v->camera = false;
  v->lidar = unpack_lidar<S>(lidar, elev, n_beams);
  v->st = unpack_settings<S>(settings);
  v->rays.resize(n_rays);
  for (int64_t p = 0; p < n_rays; ++p) v->rays[p] = Ray<S>{rays[3 * p], rays[3 * p + 1], rays[3 * p + 2]};
  v->ray_begin.assign(ray_begin, ray_begin + n_tiles);
  v->ray_end.assign(ray_end, ray_end + n_tiles);
  try {
    view_forward(v, t_scene, workers, stop_after);
  } catch (const std::exception& e) {
    v->sh->error = e.what();
    delete v;
    return nullptr;
  }
  return v;
}

template <class S> int view_backward(void* vv, const S* g_blend16, const S* g_alpha, int workers) {
  auto* v = (ViewH<S>*)vv;
  auto& h = *v->sh;
  const int64_t P = v->out.P;
  std::vector<S> gb(g_blend16, g_blend16 + 16 * P), ga(g_alpha, g_alpha + P);
  double t0 = now_ms();
  const bool los = !v->camera && !v->los_cut.empty() && v->g_los.size() == v->los_cut.size();
  v->rg = rasterize_backward<S>(v->wl, v->proj, v->scene, v->camera, &v->cam, &v->rays, &v->ray_begin, &v->ray_end,
                                v->st, v->out, gb, ga, workers, los ? &v->los_cut : nullptr, los ? &v->g_los : nullptr);
  double t1 = now_ms();
  v->ms[4] = t1 - t0;
  raster_grads_to_projected_grads<S>(v->rg, v->proj, v->scene, v->camera, v->pg);
  double t2 = now_ms();
  v->ms[5] = t2 - t1;
  const int64_t N = v->scene.size();
  const int64_t V = (int64_t)v->proj.size();
  // Per-worker buffers reduced in worker order (common.hpp:69-71). Per-Gaussian slots are disjoint, so the
  // shared ComposeGrads is written without per-worker copies; sensor slots are per-worker.
  v->cg.resize(N);
  v->sg = SensorGrads<S>();
  workers = std::max(1, workers);
  std::vector<SensorGrads<S>> sgs(workers);
  parallel_chunks(V, workers, [&](int w, int64_t b, int64_t e) {
    if (v->camera) project_camera_backward<S>(v->scene, v->cam, v->proj, v->pg, v->cg, sgs[w], b, e);
    else project_lidar_backward<S>(v->scene, v->lidar, v->proj, v->pg, v->cg, sgs[w], b, e);
  });
  for (auto& s : sgs) {
    for (int k = 0; k < 3; ++k) { v->sg.d_vel_lin[k] += s.d_vel_lin[k]; v->sg.d_vel_ang[k] += s.d_vel_ang[k]; }
  }
  v->sg.d_time_offset = v->camera ? v->rg.d_time_offset : S(0);
  double t3 = now_ms();
  v->ms[6] = t3 - t2;
  if (!h.grads_ready) {
    h.grads.resize_like(h.graph);
    h.grads_ready = true;
  }
  // compose_backward over the visible Gaussians only (all incoming grads of culled ones are zero).
  // Per-Gaussian slots are disjoint; actor slots are shared accumulators (scene.hpp:310-312) => one
  // actor-grad set per worker, reduced in worker order.
  using AG = typename SceneParamGrads<S>::ActorGrad;
  std::vector<AG> zero_actors(h.graph.tracks.size());
  for (size_t a = 0; a < zero_actors.size(); ++a) zero_actors[a].d_pose_offset.assign(6 * h.graph.tracks[a].pose_count(), 0.0);
  std::vector<std::vector<AG>> actor_parts(workers, zero_actors);
  const int d_f = h.graph.gaussians.d_f;
  parallel_chunks(V, workers, [&](int w, int64_t b, int64_t e) {
    for (int64_t k = b; k < e; ++k) {
      const int64_t i = v->proj[k].source_index;
      compose_backward<S>(v->scene, v->cg, v->pg.g_opacity, h.grads, actor_parts[w], i, i + 1);
      // appearance grads pass straight through (projection.hpp:183-185 -> scene.hpp:326-329)
      for (int c = 0; c < 3; ++c) h.grads.d_color[3 * i + c] += v->pg.g_color[3 * i + c];
      for (int c = 0; c < d_f; ++c) h.grads.d_feature[(int64_t)d_f * i + c] += v->pg.g_feature[(int64_t)d_f * i + c];
    }
  });
  for (auto& part : actor_parts)
    for (size_t a = 0; a < part.size(); ++a) {
      for (size_t k = 0; k < part[a].d_pose_offset.size(); ++k) h.grads.actors[a].d_pose_offset[k] += part[a].d_pose_offset[k];
      for (int k = 0; k < 6; ++k) h.grads.actors[a].d_vel_offset[k] += part[a].d_vel_offset[k];
    }
  v->ms[7] = now_ms() - t3;
  return 0;
}

template <class S> int64_t put(const std::vector<S>& src, void* dst) {
  if (dst) std::memcpy(dst, src.data(), src.size() * sizeof(S));
  return (int64_t)src.size();
}

template <class S> int64_t view_array(void* vv, const char* name_c, void* dst) {
  auto* v = (ViewH<S>*)vv;
  const std::string name(name_c);
  const size_t V = v->proj.size();
  auto proj_field = [&](int width, auto getter) -> int64_t {
    if (dst) {
      S* d = (S*)dst;
      for (size_t k = 0; k < V; ++k)
        for (int c = 0; c < width; ++c) d[k * width + c] = getter(v->proj[k], c);
    }
    return (int64_t)V * width;
  };
  auto ints = [&](size_t n, auto getter) -> int64_t {
    if (dst) {
      int64_t* d = (int64_t*)dst;
      for (size_t k = 0; k < n; ++k) d[k] = (int64_t)getter(k);
    }
    return (int64_t)n;
  };
  if (name == "source_index") return ints(V, [&](size_t k) { return v->proj[k].source_index; });
  if (name == "mean2d") return proj_field(2, [](const Projected<S>& g, int c) { return g.mean2d[c]; });
  if (name == "depth_key") return proj_field(1, [](const Projected<S>& g, int) { return g.depth_key; });
  if (name == "cov2d") return proj_field(4, [](const Projected<S>& g, int c) { return g.cov2d[c]; });
  if (name == "velocity") return proj_field(3, [](const Projected<S>& g, int c) { return g.velocity[c]; });
  if (name == "aabb") return proj_field(4, [](const Projected<S>& g, int c) { return c < 2 ? g.aabb_lo[c] : g.aabb_hi[c - 2]; });
  if (name == "conic") return proj_field(4, [](const Projected<S>& g, int c) { return g.conic[c]; });
  if (name == "det_ratio") return proj_field(1, [](const Projected<S>& g, int) { return g.det_ratio; });
  if (name == "mu_sensor") return proj_field(3, [](const Projected<S>& g, int c) { return g.mu_sensor[c]; });
  if (name == "rel_vel_sensor") return proj_field(3, [](const Projected<S>& g, int c) { return g.rel_vel_sensor[c]; });
  if (name == "rect")
    return ints(4 * v->rects.size(), [&](size_t k) {
      const TileRect& r = v->rects[k / 4];
      const int c = (int)(k % 4);
      return c == 0 ? r.x0 : (c == 1 ? r.x1 : (c == 2 ? r.y0 : r.y1));
    });
  if (name == "isect_tile") return ints(v->wl.items.size(), [&](size_t k) { return v->wl.items[k].tile; });
  if (name == "isect_depth_bits") return ints(v->wl.items.size(), [&](size_t k) { return v->wl.items[k].depth_bits; });
  if (name == "isect_src") return ints(v->wl.items.size(), [&](size_t k) { return v->wl.items[k].src; });
  if (name == "los") {
    if (dst) std::copy(v->out.los.begin(), v->out.los.end(), (S*)dst);
    return (int64_t)v->out.los.size();
  }
  if (name == "tile_begin") return ints(v->wl.tile_begin.size(), [&](size_t k) { return v->wl.tile_begin[k]; });
  if (name == "tile_end") return ints(v->wl.tile_end.size(), [&](size_t k) { return v->wl.tile_end[k]; });
  if (name == "grid") return ints(2, [&](size_t k) { return k == 0 ? v->wl.tiles_x : v->wl.tiles_y; });
  if (name == "n_contrib") return ints(v->out.n_contrib.size(), [&](size_t k) { return v->out.n_contrib[k]; });
  if (name == "last_idx") return ints(v->out.last_idx.size(), [&](size_t k) { return v->out.last_idx[k]; });
  if (name == "blend") return put(v->out.blend, dst);
  if (name == "alpha") return put(v->out.alpha, dst);
  if (name == "t_final") return put(v->out.t_final, dst);
  if (name == "range_blend") return put(v->out.range_blend, dst);
  if (name == "mean_w") return put(v->scene.mean_w, dst);
  if (name == "vel_dyn_w") return put(v->scene.vel_dyn_w, dst);
  if (name == "opacity") return put(v->scene.opacity, dst);
  if (name == "cov_w") {
    if (dst) {
      S* d = (S*)dst;
      for (size_t i = 0; i < v->scene.cov_w.size(); ++i)
        for (int e = 0; e < 9; ++e) d[9 * i + e] = v->scene.cov_w[i].m[e];
    }
    return (int64_t)v->scene.cov_w.size() * 9;
  }
  if (name == "rg_conic") return put(v->rg.g_conic, dst);
  if (name == "rg_mean2d") return put(v->rg.g_mean2d, dst);
  if (name == "rg_vel") return put(v->rg.g_vel, dst);
  if (name == "rg_rho") return put(v->rg.g_rho, dst);
  if (name == "rg_range") return put(v->rg.g_range, dst);
  if (name == "rg_f") return put(v->rg.g_f, dst);
  if (name == "pg_mean2d") return put(v->pg.g_mean2d, dst);
  if (name == "pg_range") return put(v->pg.g_range, dst);
  if (name == "pg_cov2d") return put(v->pg.g_cov2d, dst);
  if (name == "pg_velocity") return put(v->pg.g_velocity, dst);
  if (name == "pg_opacity") return put(v->pg.g_opacity, dst);
  if (name == "pg_color") return put(v->pg.g_color, dst);
  if (name == "pg_feature") return put(v->pg.g_feature, dst);
  if (name == "cg_mean_w") return put(v->cg.g_mean_w, dst);
  if (name == "cg_vel_dyn_w") return put(v->cg.g_vel_dyn_w, dst);
  if (name == "cg_cov_w") {
    if (dst) {
      S* d = (S*)dst;
      for (size_t i = 0; i < v->cg.g_cov_w.size(); ++i)
        for (int e = 0; e < 9; ++e) d[9 * i + e] = v->cg.g_cov_w[i].m[e];
    }
    return (int64_t)v->cg.g_cov_w.size() * 9;
  }
  if (name == "sensor_grads") {
    if (dst) {
      S* d = (S*)dst;
      for (int k = 0; k < 3; ++k) { d[k] = v->sg.d_vel_lin[k]; d[3 + k] = v->sg.d_vel_ang[k]; }
      d[6] = v->sg.d_time_offset;
    }
    return 7;
  }
  if (name == "ms") {
    if (dst) for (int k = 0; k < 8; ++k) ((S*)dst)[k] = S(v->ms[k]);
    return 8;
  }
  return -1;
}

template <class S> int64_t scene_array(void* hv, const char* name_c, void* dst) {
  auto* h = (SceneH<S>*)hv;
  const std::string name(name_c);
  if (!h->grads_ready) {
    h->grads.resize_like(h->graph);
    h->grads_ready = true;
  }
  if (name == "d_mean") return put(h->grads.d_mean, dst);
  if (name == "d_scale_log") return put(h->grads.d_scale_log, dst);
  if (name == "d_quat") return put(h->grads.d_quat, dst);
  if (name == "d_opacity_logit") return put(h->grads.d_opacity_logit, dst);
  if (name == "d_color") return put(h->grads.d_color, dst);
  if (name == "d_feature") return put(h->grads.d_feature, dst);
  if (name.rfind("actor_d_pose_offset:", 0) == 0) {
    const size_t a = (size_t)std::stoi(name.substr(20));
    if (a >= h->grads.actors.size()) return -1;
    return put(h->grads.actors[a].d_pose_offset, dst);  // double
  }
  if (name.rfind("actor_d_vel_offset:", 0) == 0) {
    const size_t a = (size_t)std::stoi(name.substr(19));
    if (a >= h->grads.actors.size()) return -1;
    if (dst) std::memcpy(dst, h->grads.actors[a].d_vel_offset, 6 * sizeof(double));
    return 6;
  }
  if (name.rfind("actor_vel:", 0) == 0) {  // effective body velocities (lin 3, ang 3), double
    const size_t a = (size_t)std::stoi(name.substr(10));
    if (a >= h->graph.tracks.size()) return -1;
    if (dst) {
      double* d = (double*)dst;
      const V3d l = h->graph.tracks[a].vel_lin, w = h->graph.tracks[a].vel_ang;
      d[0] = l.x; d[1] = l.y; d[2] = l.z; d[3] = w.x; d[4] = w.y; d[5] = w.z;
    }
    return 6;
  }
  return -1;
}

template <class S>
int view_brute(void* vv, int early_exit, S* blend16, S* alpha, int64_t* n_contrib) {
  auto* v = (ViewH<S>*)vv;
  RasterOut<S> o = brute_force<S>(v->proj, v->scene, v->camera, &v->cam, &v->rays, v->st, early_exit != 0);
  std::memcpy(blend16, o.blend.data(), o.blend.size() * sizeof(S));
  std::memcpy(alpha, o.alpha.data(), o.alpha.size() * sizeof(S));
  for (size_t p = 0; p < o.n_contrib.size(); ++p) n_contrib[p] = o.n_contrib[p];
  return 0;
}

// Contributor introspection for the gradient parity gate (tests only). For every query: the sequence of (source index,
// clamped) it blends. hash (P, optional): a 64-bit signature of that sequence. gauss_flag (N, optional): a query that
// blends a flagged Gaussian gets query_flag = 1. Every Gaussian blended by a query with query_flag = 1 is marked in
// gauss_mask (N, optional).
template <class S>
int view_contrib(void* vv, const uint8_t* gauss_flag, uint8_t* query_flag, uint8_t* gauss_mask, uint64_t* hash, int workers) {
  auto* v = (ViewH<S>*)vv;
  const Worklist& wl = v->wl;
  const int T = wl.tiles_x * wl.tiles_y;
  const bool camera = v->camera;
  const int W = camera ? v->cam.width : 0, H = camera ? v->cam.height : 0;
  parallel_chunks(T, workers, [&](int, int64_t tb, int64_t te) {
    std::vector<Splat<S>> splats;
    std::vector<int32_t> pos;
    std::vector<uint8_t> cl;
    for (int64_t tile = tb; tile < te; ++tile) {
      const int64_t b = wl.tile_begin[tile], e = std::max<int64_t>(wl.tile_begin[tile], wl.tile_end[tile]);
      splats.resize(e - b);
      for (int64_t j = b; j < e; ++j) splats[j - b] = make_splat(v->proj[wl.items[j].pidx], v->scene, camera);
      auto one = [&](int64_t p, S qx, S qy, S t) {
        contributors_one<S>(e - b, [&](int64_t j) -> const Splat<S>& { return splats[j]; }, qx, qy, t, !camera, v->st, pos, cl);
        uint64_t hsh = 0xcbf29ce484222325ull;
        bool flagged = query_flag && query_flag[p];
        for (size_t k = 0; k < pos.size(); ++k) {
          const int64_t src = wl.items[b + pos[k]].src;
          hsh = (hsh ^ (uint64_t)(2 * src + cl[k])) * 0x100000001b3ull;
          if (gauss_flag && gauss_flag[src]) flagged = true;
        }
        if (hash) hash[p] = hsh;
        if (flagged) {
          if (query_flag) query_flag[p] = 1;
          if (gauss_mask)
            for (size_t k = 0; k < pos.size(); ++k) gauss_mask[wl.items[b + pos[k]].src] = 1;
        }
      };
      if (camera) {
        const int tx = (int)(tile % wl.tiles_x), ty = (int)(tile / wl.tiles_x);
        for (int py = ty * kTile; py < std::min(H, (ty + 1) * kTile); ++py) {
          const S t = pixel_capture_offset<S>(py, H, v->cam.shutter_duration, v->cam.time_offset);
          for (int px = tx * kTile; px < std::min(W, (tx + 1) * kTile); ++px) one((int64_t)py * W + px, S(px) + S(0.5), S(py) + S(0.5), t);
        }
      } else {
        for (int64_t p = v->ray_begin[tile]; p < v->ray_end[tile]; ++p) one(p, v->rays[p].phi, v->rays[p].omega, v->rays[p].t);
      }
    }
  });
  return 0;
}

}  // namespace

#define ORC_API(SUF, S)                                                                                                  \
  extern "C" void* orc_scene_new_##SUF(int64_t n, int d_f, const S* mean, const S* scale_log, const S* quat,             \
                                       const S* opacity_logit, const S* color, const S* feature,                        \
                                       const int32_t* actor_id) {                                                        \
    return scene_new<S>(n, d_f, mean, scale_log, quat, opacity_logit, color, feature, actor_id);                         \
  }                                                                                                                      \
  extern "C" void orc_scene_add_track_##SUF(void* h, int n_poses, const double* stamps, const double* R,                 \
                                            const double* t, const double* pose_offset, const double* vel_lin,           \
                                            const double* vel_ang, const double* vel_offset, int init_vel) {             \
    scene_add_track<S>(h, n_poses, stamps, R, t, pose_offset, vel_lin, vel_ang, vel_offset, init_vel);                   \
  }                                                                                                                      \
  extern "C" void orc_scene_free_##SUF(void* h) { delete (SceneH<S>*)h; }                                                \
  extern "C" void orc_scene_zero_grads_##SUF(void* h) {                                                                  \
    ((SceneH<S>*)h)->grads.resize_like(((SceneH<S>*)h)->graph);                                                          \
    ((SceneH<S>*)h)->grads_ready = true;                                                                                 \
  }                                                                                                                      \
  extern "C" const char* orc_scene_error_##SUF(void* h) { return ((SceneH<S>*)h)->error.c_str(); }                       \
  extern "C" int64_t orc_scene_array_##SUF(void* h, const char* name, void* dst) { return scene_array<S>(h, name, dst); } \
  extern "C" void* orc_view_camera_##SUF(void* sh, double t_scene, const double* cam, const double* settings,            \
                                         int workers, int stop_after) {                                                  \
    return view_camera<S>(sh, t_scene, cam, settings, workers, stop_after);                                              \
  }                                                                                                                      \
  extern "C" void* orc_view_lidar_##SUF(void* sh, double t_scene, const double* lidar, const double* elev, int n_beams,  \
                                        const double* settings, const S* rays, int64_t n_rays,                          \
                                        const int64_t* ray_begin, const int64_t* ray_end, int64_t n_tiles, int workers,  \
                                        int stop_after) {                                                                \
    return view_lidar<S>(sh, t_scene, lidar, elev, n_beams, settings, rays, n_rays, ray_begin, ray_end, n_tiles,         \
                         workers, stop_after);                                                                           \
  }                                                                                                                      \
  extern "C" void orc_view_free_##SUF(void* v) { delete (ViewH<S>*)v; }                                                  \
  /* line-of-sight channel: sets the per-ray cut (r_p - eps) and re-runs the compositing so that array "los" exists */   \
  extern "C" void orc_view_set_los_##SUF(void* vv, const S* cut, int workers) {                                          \
    auto* v = (ViewH<S>*)vv;                                                                                             \
    v->los_cut.assign(cut, cut + v->rays.size());                                                                        \
    v->out = rasterize_lidar<S>(v->wl, v->proj, v->scene, v->rays, v->ray_begin, v->ray_end, v->st, workers, &v->los_cut); \
  }                                                                                                                      \
  extern "C" void orc_view_set_los_grad_##SUF(void* vv, const S* g) {                                                    \
    auto* v = (ViewH<S>*)vv;                                                                                             \
    v->g_los.assign(g, g + v->rays.size());                                                                              \
  }                                                  \
  extern "C" int orc_view_backward_##SUF(void* v, const S* g_blend16, const S* g_alpha, int workers) {                   \
    return view_backward<S>(v, g_blend16, g_alpha, workers);                                                             \
  }                                                                                                                      \
  extern "C" int64_t orc_view_array_##SUF(void* v, const char* name, void* dst) { return view_array<S>(v, name, dst); }  \
  extern "C" int orc_view_brute_##SUF(void* v, int early_exit, S* blend16, S* alpha, int64_t* n_contrib) {               \
    return view_brute<S>(v, early_exit, blend16, alpha, n_contrib);                                                      \
  }                                                                                                                      \
  extern "C" int orc_view_contrib_##SUF(void* v, const uint8_t* gauss_flag, uint8_t* query_flag, uint8_t* gauss_mask,     \
                                        uint64_t* hash, int workers) {                                                   \
    return view_contrib<S>(v, gauss_flag, query_flag, gauss_mask, hash, workers);                                        \
  }                                                                                                                      \
  /* ---- known-answer helpers (SPEC examples) ---- */                                                                   \
  extern "C" void orc_covariance_from_scale_quat_##SUF(const S* scale_log, const S* quat, S* out9) {                     \
    M3<S> c = covariance_from_scale_quat<S>(V3<S>(scale_log[0], scale_log[1], scale_log[2]), quat);                      \
    for (int i = 0; i < 9; ++i) out9[i] = c.m[i];                                                                        \
  }                                                                                                                      \
  extern "C" void orc_spherical_##SUF(const S* p, S* sph3, S* J9) {                                                      \
    S J[3][3];                                                                                                           \
    spherical_jacobian<S>(V3<S>(p[0], p[1], p[2]), J);                                                                   \
    for (int a = 0; a < 3; ++a)                                                                                          \
      for (int b = 0; b < 3; ++b) J9[3 * a + b] = J[a][b];                                                               \
    const S r = Sc<S>::sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);                                                  \
    sph3[0] = wrap_two_pi(Sc<S>::atan2(p[1], p[0]));                                                                     \
    sph3[1] = Sc<S>::asin(p[2] / r);                                                                                     \
    sph3[2] = r;                                                                                                         \
  }                                                                                                                      \
  extern "C" void orc_spherical_jacobian_point_grad_##SUF(const S* p, const S* gJ9, S* out3) {                           \
    S g[3][3];                                                                                                           \
    for (int a = 0; a < 3; ++a)                                                                                          \
      for (int b = 0; b < 3; ++b) g[a][b] = gJ9[3 * a + b];                                                              \
    V3<S> o = spherical_jacobian_point_grad<S>(V3<S>(p[0], p[1], p[2]), g);                                              \
    out3[0] = o.x; out3[1] = o.y; out3[2] = o.z;                                                                         \
  }                                                                                                                      \
  extern "C" void orc_image_tile_range_##SUF(const S* lo, const S* hi, int tiles_x, int tiles_y, int* out4) {            \
    TileRect r = image_tile_range<S>(lo, hi, tiles_x, tiles_y);                                                          \
    out4[0] = r.x0; out4[1] = r.x1; out4[2] = r.y0; out4[3] = r.y1;                                                      \
  }                                                                                                                      \
  extern "C" void orc_lidar_grid_##SUF(double az_res, const double* elev, int n_beams, S* span_phimax, int* m2,          \
                                       S* boundaries) {                                                                  \
    LidarModel<S> l;                                                                                                     \
    l.azimuth_resolution = S(az_res);                                                                                    \
    for (int i = 0; i < n_beams; ++i) l.elevation_channels.push_back(S(elev[i]));                                        \
    LidarGrid<S> g = make_lidar_grid<S>(l);                                                                              \
    span_phimax[0] = g.span; span_phimax[1] = g.phi_max;                                                                 \
    m2[0] = g.m_phi; m2[1] = g.m_omega;                                                                                  \
    for (size_t k = 0; k < g.boundaries.size(); ++k) boundaries[k] = g.boundaries[k];                                    \
  }                                                                                                                      \
  extern "C" void orc_lidar_tile_range_##SUF(double az_res, const double* elev, int n_beams, const S* lo, const S* hi,   \
                                             int* out4) {                                                                \
    LidarModel<S> l;                                                                                                     \
    l.azimuth_resolution = S(az_res);                                                                                    \
    for (int i = 0; i < n_beams; ++i) l.elevation_channels.push_back(S(elev[i]));                                        \
    LidarGrid<S> g = make_lidar_grid<S>(l);                                                                              \
    TileRect r = lidar_tile_range<S>(lo, hi, g);                                                                         \
    out4[0] = r.x0; out4[1] = r.x1; out4[2] = r.y0; out4[3] = r.y1;                                                      \
  }                                                                                                                      \
  extern "C" void orc_elevation_rows_##SUF(const S* boundaries, int nb, S lo, S hi, int* out2) {                         \
    LidarGrid<S> g;                                                                                                      \
    g.boundaries.assign(boundaries, boundaries + nb);                                                                    \
    g.m_omega = nb + 1;                                                                                                  \
    lidar_elevation_tile_range<S>(lo, hi, g, out2[0], out2[1]);                                                          \
  }                                                                                                                      \
  extern "C" S orc_pixel_capture_offset_##SUF(int p_v, int H, S t_rs, S off) {                                           \
    return pixel_capture_offset<S>(p_v, H, t_rs, off);                                                                   \
  }                                                                                                                      \
  extern "C" int orc_evaluate_alpha_##SUF(const S* splat10, S qx, S qy, S t, const double* settings, int wrap,           \
                                          S* alpha_out) {                                                                \
    Splat<S> g;                                                                                                          \
    g.mx = splat10[0]; g.my = splat10[1]; g.vx = splat10[2]; g.vy = splat10[3]; g.vz = splat10[4];                       \
    g.a = splat10[5]; g.b2 = splat10[6]; g.c = splat10[7]; g.rho = splat10[8]; g.depth = splat10[9];                     \
    RasterSettings<S> st = unpack_settings<S>(settings);                                                                 \
    S dx, dy, ga;                                                                                                        \
    bool cl;                                                                                                             \
    *alpha_out = S(0);                                                                                                   \
    return evaluate_alpha<S>(g, qx, qy, t, st, wrap != 0, *alpha_out, dx, dy, ga, cl) ? 1 : 0;                           \
  }                                                                                                                      \
  extern "C" int64_t orc_assign_points_##SUF(const double* lidar, const double* elev, int n_beams, const S* xyz,           \
                                             const S* stamps, int64_t n, int train, uint32_t seed, int64_t* tile,         \
                                             S* sph4 /* n x (phi, omega, t_l, range) */, int64_t* order,                  \
                                             int64_t* begin, int64_t* end, int64_t* counts3) {                           \
    const LidarModel<S> l = unpack_lidar<S>(lidar, elev, n_beams);                                                       \
    const AssignedPoints<S> a = assign_points_to_tiles<S>(xyz, stamps, n, l, train != 0, seed);                          \
    for (int64_t i = 0; i < n; ++i) {                                                                                    \
      tile[i] = a.tile[i];                                                                                               \
      sph4[4 * i] = a.phi[i]; sph4[4 * i + 1] = a.omega[i]; sph4[4 * i + 2] = a.t_l[i]; sph4[4 * i + 3] = a.range[i];    \
    }                                                                                                                    \
    for (size_t k = 0; k < a.order.size(); ++k) order[k] = a.order[k];                                                   \
    for (size_t t = 0; t < a.begin.size(); ++t) { begin[t] = a.begin[t]; end[t] = a.end[t]; }                            \
    counts3[0] = (int64_t)a.order.size(); counts3[1] = a.rejected; counts3[2] = a.dropped;                               \
    return (int64_t)a.begin.size();                                                                                      \
  }                                                                                                                      \
  /* decode_lidar: n rays; feat n x d_f, sph n x 2 (azimuth, elevation); y n x 2 (intensity, drop) */      \
  extern "C" void orc_lidar_head_forward_##SUF(const S* w, int d_f, int64_t n, const S* feat, const S* sph, S* y) {      \
    for (int64_t i = 0; i < n; ++i) {                                                                                    \
      S d[3], h[kHeadHidden];                                                                                            \
      ray_direction_sensor<S>(sph[2 * i], sph[2 * i + 1], d);                                                            \
      lidar_head_forward_one<S>(w, d_f, feat + (int64_t)d_f * i, d, y + 2 * i, h);                                       \
    }                                                                                                                    \
  }                                                                                                                      \
  extern "C" void orc_lidar_head_backward_##SUF(const S* w, int d_f, int64_t n, const S* feat, const S* sph,            \
                                                const S* g_y, S* gw, S* g_feat) {                                        \
    for (int k = 0; k < lidar_head_params(d_f); ++k) gw[k] = S(0);                                                       \
    for (int64_t i = 0; i < n; ++i) {                                                                                    \
      S d[3];                                                                                                            \
      ray_direction_sensor<S>(sph[2 * i], sph[2 * i + 1], d);                                                            \
      lidar_head_backward_one<S>(w, d_f, feat + (int64_t)d_f * i, d, g_y + 2 * i, gw, g_feat + (int64_t)d_f * i);        \
    }                                                                                                                    \
  }                                                                                                                      \
  extern "C" S orc_wrap_pi_##SUF(S a) { return wrap_pi<S>(a); }                                                          \
  extern "C" S orc_wrap_two_pi_##SUF(S a) { return wrap_two_pi<S>(a); }                                                  \
  extern "C" S orc_sigmoid_##SUF(S a) { return Sc<S>::sigmoid(a); }

ORC_API(f32, float)
ORC_API(f64, double)

// decode_image, decoder_oracle.hpp. rgb H x W x 3, feat H x W x d_f, intr = (fx, fy, cx, cy).
#define ORC_DECODER(SUF, S)                                                                                              \
  extern "C" void orc_decoder_forward_##SUF(const S* params, int H, int W, int d_f, const S* rgb, const S* feat,         \
                                            const S* intr, const S* emb, S* image, S* h2, int workers) {                              \
    DecoderState<S> st;                                                                                                  \
    decoder_forward<S>(params, H, W, d_f, rgb, feat, intr, emb, image, &st, workers);                                    \
    if (h2) std::copy(st.h2.begin(), st.h2.end(), h2);                                                                   \
  }                                                                                                                      \
  extern "C" void orc_decoder_backward_##SUF(const S* params, int H, int W, int d_f, const S* rgb, const S* feat,        \
                                             const S* intr, const S* emb, const S* g_image, S* g_params, S* g_rgb,       \
                                             S* g_feat, S* g_emb) {                                                      \
    DecoderState<S> st;                                                                                                  \
    std::vector<S> image((size_t)H * W * 3);                                                                             \
    decoder_forward<S>(params, H, W, d_f, rgb, feat, intr, emb, image.data(), &st);                                      \
    decoder_backward<S>(params, st, rgb, g_image, g_params, g_rgb, g_feat, g_emb);                                       \
  }
ORC_DECODER(f32, float)
// backward of the decode from SAVED activations (x0, h0, t1, h1, t2, h2: P x 32 each, e.g. those of the device path):
// the ReLU masks then are those of the forward that actually ran
extern "C" void orc_decoder_backward_state_f64(const double* params, int H, int W, int d_f, const double* rgb,
                                               const double* acts, const double* g_image, double* g_params, double* g_rgb,
                                               double* g_feat, double* g_emb) {
  DecoderState<double> st;
  st.H = H; st.W = W; st.d_f = d_f;
  const size_t n = (size_t)H * W * kDecWidth;
  std::vector<double>* dst[6] = {&st.x0, &st.h0, &st.t1, &st.h1, &st.t2, &st.h2};
  for (int k = 0; k < 6; ++k) dst[k]->assign(acts + k * n, acts + (k + 1) * n);
  decoder_backward<double>(params, st, rgb, g_image, g_params, g_rgb, g_feat, g_emb);
}
ORC_DECODER(f64, double)
extern "C" void orc_decoder_activations_f64(const double* params, int H, int W, int d_f, const double* rgb, const double* feat,
                                            const double* intr, const double* emb, double* acts) {
  DecoderState<double> st;
  std::vector<double> image((size_t)H * W * 3);
  decoder_forward<double>(params, H, W, d_f, rgb, feat, intr, emb, image.data(), &st);
  const size_t n = (size_t)H * W * kDecWidth;
  const std::vector<double>* src[6] = {&st.x0, &st.h0, &st.t1, &st.h1, &st.t2, &st.h2};
  for (int k = 0; k < 6; ++k) std::copy(src[k]->begin(), src[k]->end(), acts + k * n);
}
extern "C" int orc_decoder_params() { return kDecParams; }

// detmath bit-pattern probes (host build of the header the kernels use)
extern "C" void orc_detmath_eval(int fn, const float* x, const float* y, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    switch (fn) {
      case 0: out[i] = detmath::exp(x[i]); break;
      case 1: out[i] = detmath::sigmoid(x[i]); break;
      case 2: out[i] = detmath::atan2(y[i], x[i]); break;
      case 3: out[i] = detmath::asin(x[i]); break;
      case 4: out[i] = detmath::exp_bounded(x[i]); break;  // the compositing kernels' form of exp
      default: out[i] = 0.0f;
    }
  }
}

extern "C" void orc_so3_roundtrip(const double* phi3, double* log_of_exp3, double* Jr9, double* Jrinv9) {
  V3d p(phi3[0], phi3[1], phi3[2]);
  V3d q = so3_log(so3_exp(p));
  log_of_exp3[0] = q.x; log_of_exp3[1] = q.y; log_of_exp3[2] = q.z;
  M3d a = so3_right_jacobian(p), b = so3_right_jacobian_inv(p);
  for (int i = 0; i < 9; ++i) { Jr9[i] = a.m[i]; Jrinv9[i] = b.m[i]; }
}

extern "C" int orc_hardware_threads() { return (int)std::max(1u, std::thread::hardware_concurrency()); }
