// capi.cu — the C ABI of libsplat_b200.so (include/splat_b200.h): context, scene, views and the
// stream-ordered stage pipeline  project -> scan -> emit keys -> radix sort -> tile ranges ->
// composite, and its reverse. Host code only; the kernels live in forward.cu / binning.cu /
// raster_bwd.cu / project_bwd.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "../../include/splat_b200.h"
#include "kernels.h"
#include "so3_host.h"

using namespace sb;

namespace {
std::string g_create_error;

template <class T> void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}
struct DevScratch {  // a device allocation that lives for one call
  float* p = nullptr;
  ~DevScratch() { if (p) cudaFree(p); }
};
}  // namespace

struct splatb200_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::atomic<int64_t> launches{0};      // hand-written kernels (views may be driven from several host threads)
  int64_t lib_launches = 0;  // library kernels on the hot path (none since the radix sort is hand-written)
  bool profiling = false;
  bool view_streams = false;   // views run forward / backward on their own streams (splatb200_ctx_set_view_streams)
  // geometry-first upload (splatb200_scene_upload_async): colour / features follow on their own copy stream; a view's
  // forward waits for them only in front of its compositing kernel
  cudaStream_t s_app = nullptr;
  cudaEvent_t ev_geo = nullptr, ev_app = nullptr;
  bool app_pending = false;
  // Small transfers first (banded host-buffer calls). The copy engines were seen (CUPTI timeline of the north-star
  // frame, scripts/e2e_probe.py) to take a lidar view's one 15 MB download only after ALL ~150 MB of band copies a
  // camera view had queued — although it was submitted first and ready 3 ms earlier —, so the lidar's upload,
  // compositing backward and k_project_bwd ran alone at the end of the step. A single-band view therefore publishes
  // its pending download / upload event here, and a multi-band view lets it pass in front of its second band.
  std::mutex xfer_mu;  // views may be driven from several host threads
  cudaEvent_t yield_dl = nullptr, yield_ul = nullptr;
  int decoder_precise = 0;     // ConvDecoder convolutions in split-tf32 (three passes: fp32 accuracy) instead of plain tf32

  // scene
  int64_t n = 0;
  int d_f = 0;
  bool owns_scene = false;
  float *mean = nullptr, *scale_log = nullptr, *quat = nullptr, *opacity_logit = nullptr, *color = nullptr,
        *feature = nullptr;
  int32_t* actor_id = nullptr;
  std::map<int, int64_t> actor_first;  // distinct actor id -> first Gaussian using it (upload path)
  int bound_max_actor = 0;             // bind path
  std::vector<sbh::Track> tracks;

  // SceneParamGrads
  float* grads = nullptr;
  bool owns_grads = false;
  int64_t grads_floats = 0;
  std::vector<std::vector<double>> actor_d_pose;  // per track 6 x n_poses
  std::vector<std::vector<double>> actor_d_vel;   // per track 6
  std::vector<splatb200_view*> views;
  // optimizer state (splatb200_optimizer_step): Adam moments over the gradient buffer's layout, per-group skip flags
  float *adam_m = nullptr, *adam_v = nullptr;
  int64_t adam_floats = 0;
  int* adam_bad = nullptr;
  // NCCL communicator of the gradient all-reduce (splatb200_ctx_comm_init / _comm_bind); void*: ncclComm_t
  void* comm = nullptr;
  bool owns_comm = false;
  int comm_rank = 0, comm_world = 0;
  double* comm_stage = nullptr;  // device staging of the ActorGrad slots
  size_t comm_stage_bytes = 0;

  int fail(int code, const std::string& m) {
    err = m;
    return code;
  }
  ParamGradDev pg() const {
    ParamGradDev g;
    g.d_mean = grads;
    g.d_scale_log = grads + 3 * n;
    g.d_quat = grads + 6 * n;
    g.d_opacity_logit = grads + 10 * n;
    g.d_color = grads + 11 * n;
    g.d_feature = grads + 14 * n;
    return g;
  }
  SceneDev scene_dev(const ActorState* d_actors) const {
    SceneDev s;
    s.n = n; s.d_f = d_f; s.mean = mean; s.scale_log = scale_log; s.quat = quat; s.opacity_logit = opacity_logit;
    s.color = color; s.feature = feature; s.actor_id = actor_id; s.actors = d_actors; s.n_actors = (int)tracks.size();
    return s;
  }
};

struct splatb200_view {
  splatb200_ctx* ctx = nullptr;
  Sensor s;
  int64_t n_alloc = 0;  // Gaussians the per-source buffers are sized for
  ProjDev proj{};
  uint32_t* offsets = nullptr;  // n + 1: exclusive scan of the tile counts in depth order, [n] = total (mod 2^32)
  int64_t* d_total = nullptr;   // the number of intersections as counted from the tile rectangles (64-bit)
  void* tile_ws = nullptr;     // tile-rectangle difference array + digit histograms of the tile sort
  float* rg = nullptr;
  // intersections
  int64_t isect_cap = 0;
  uint32_t *keys0 = nullptr, *keys1 = nullptr;  // tile ids
  uint32_t *vals0 = nullptr, *vals1 = nullptr;  // source indices
  // depth sort of the Gaussians (N + 1 entries each; [n] is padding)
  uint32_t *dkey_alt = nullptr, *order0 = nullptr, *order1 = nullptr;
  void* dsort_temp = nullptr;
  size_t dsort_temp_bytes = 0;
  int order_sel = 0;
  void* sort_temp = nullptr;
  size_t sort_temp_bytes = 0;
  int sorted_sel = 0;
  uint32_t *tile_begin = nullptr, *tile_end = nullptr;
  // two-level binning (cameras): lists per block of 8 x 8 tiles first, expanded into the tile lists
  bool two_level = false;
  int stiles_x = 0, stiles_y = 0;
  uint32_t *super_begin = nullptr, *super_end = nullptr, *seg_first = nullptr;
  void* expand_temp = nullptr;
  void* tile_ws_c = nullptr;
  int64_t* d_total_c = nullptr;
  uint32_t* vals_fine = nullptr;  // the tile lists (two-level mode; otherwise the sorted vals0 / vals1)
  int64_t fine_cap = 0;
  int64_t hit_cap = 0;            // out.hit: one byte per tile-list entry
  bool multi_pass = false;        // some lidar tile holds more than 256 rays
  int64_t rows_cap = 0;           // out.hit_rows capacity in words (lidar v2 kernels)
  int64_t list_cap = 0;           // out.hit_list capacity in entries (shared backward kernel)
  // lidar: the v2 compositing kernels (raster_lidar.cu) unless a tile needs several ray passes or SPLATB200_LIDAR_V1 is set
  bool lidar_v2() const { static const bool off = std::getenv("SPLATB200_LIDAR_V1") != nullptr; return !s.is_camera && !multi_pass && !off; }
  int64_t I_sort = 0;             // entries the radix sort handles: block-level intersections, or I
  // queries
  int64_t P = 0, n_tiles = 0;
  int64_t P_cap = 0;   // queries the per-query buffers are sized for (lidar sweeps change size: view_set_rays)
  float *d_los_cut = nullptr, *d_los = nullptr, *d_g_los = nullptr;  // line-of-sight channel (lidar, optional)
  float *d_head_w = nullptr, *d_head_y = nullptr;                     // fused lidar head (optional)
  float* dec_act[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // ConvDecoder activations x0 h0 t1 h1 t2 h2 (lazy)
  float* dec_g[3] = {nullptr, nullptr, nullptr};                      // backward scratch, P x 32 each
  float *dec_gext = nullptr, *d_dec_gimage = nullptr, *d_dec_gparams = nullptr;  // (H+2)(W+2) x 32; P x 3; params + 8
  bool dec_ready = false;                                             // activations match the last forward + decode
  float *d_dec_image = nullptr, *d_dec_params = nullptr;              // decoded image P x 3; parameters + embedding
  int* d_dec_err = nullptr;
  float4* rays = nullptr;  // per ray POSITION: azimuth, elevation, t_l, bits of the original ray index (see create_lidar)
  int64_t *ray_begin = nullptr, *ray_end = nullptr;
  uint32_t* tile_order = nullptr;  // CTA -> tile permutation (longest worklists first), rebuilt every forward
  uint32_t* to_vals0 = nullptr;
  RasterOutDev out{};
  float *g_blend_stage = nullptr, *g_alpha_stage = nullptr;
  // overlapped host-buffer calls: forward done (compute -> d2h), download done, upload done, backward done
  cudaEvent_t ev_fwd = nullptr, ev_dl = nullptr, ev_up = nullptr, ev_bwd = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // this view's copy streams (views overlap each other's transfers)
  cudaStream_t vs = nullptr;       // this view's work stream (ctx->view_streams)
  cudaEvent_t ev_last = nullptr;   // last work enqueued on vs
  cudaEvent_t ev_ctx = nullptr;    // 'everything asked of the ctx stream so far', as seen at this view's last call
  bool busy = false;               // vs holds work the ctx stream has not been ordered after yet
  bool wait_up = false;            // the next backward waits for ev_up (overlapped upstream-gradient upload)
  // banded host transfers (forward_to_host / backward_from_host): the image is rendered and differentiated in bands of
  // tile rows, so that a band's download / upload runs beside the next band's kernels
  struct Band { int tile_first, tile_count; int64_t q0, q1; };
  std::vector<Band> bands;
  float* plan_blend = nullptr; float* plan_alpha = nullptr; int32_t* plan_ncontrib = nullptr;  // forward plan (host, pinned)
  bool plan_fwd = false;
  const float* plan_gb = nullptr; const float* plan_ga = nullptr;                              // backward plan (host, pinned)
  bool plan_bwd = false;
  bool band_dl_valid = false;      // ev_bdl[] hold this render's per-band downloads
  cudaEvent_t ev_bfwd[8] = {}, ev_bdl[8] = {}, ev_bup[8] = {};
  bool dl_pending = false, bwd_recorded = false;
  float* sensor_grads = nullptr;  // 6 + d_time_offset
  // actors
  ActorState* d_actors = nullptr;
  int d_actors_cap = 0;
  float* actor_acc = nullptr;
  int actor_acc_cap = 0;
  std::vector<sbh::Interp> poses;
  bool actor_pending = false;
  // state
  int64_t I = 0;
  int stage = 0;  // 0 nothing, 1 projected, 2 sorted, 3 rasterized
  float t_scene = 0.0f;
  int64_t* h_total = nullptr;  // pinned
  // per-stage CUDA events (ctx profiling): project, scan, emit_keys, sort, tile_ranges, raster_fwd, raster_bwd, project_bwd
  cudaEvent_t ev[8][2] = {};
  bool ev_valid[8] = {};   // recorded, not yet harvested
  double ev_sum_ms[8] = {};
  int64_t ev_count[8] = {};

  const uint32_t* order() const { return order_sel ? order1 : order0; }
  const uint32_t* vals() const { return two_level ? vals_fine : (sorted_sel ? vals1 : vals0); }
  const uint32_t* sorted_vals() const { return sorted_sel ? vals1 : vals0; }
};

#define CU_TRY(ctx, call)                                                                             \
  do {                                                                                                \
    cudaError_t e__ = (call);                                                                         \
    if (e__ != cudaSuccess)                                                                           \
      return (ctx)->fail(SPLATB200_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__));        \
  } while (0)

#define CHECK_LAUNCH(ctx, what)                                                                       \
  do {                                                                                                \
    cudaError_t e__ = cudaGetLastError();                                                             \
    if (e__ != cudaSuccess) return (ctx)->fail(SPLATB200_ECUDA, std::string(what) + ": " + cudaGetErrorString(e__)); \
  } while (0)

namespace {

void free_scene(splatb200_ctx* c) {
  if (c->owns_scene) {
    dfree(c->mean); dfree(c->scale_log); dfree(c->quat); dfree(c->opacity_logit); dfree(c->color); dfree(c->feature);
    dfree(c->actor_id);
  }
  c->mean = c->scale_log = c->quat = c->opacity_logit = c->color = c->feature = nullptr;
  c->actor_id = nullptr;
  c->owns_scene = false;
  if (c->owns_grads) dfree(c->grads);
  c->grads = nullptr;
  c->owns_grads = false;
  dfree(c->adam_m); dfree(c->adam_v); dfree(c->adam_bad);
  c->adam_floats = 0;
}

int alloc_grads(splatb200_ctx* c) {
  c->grads_floats = (int64_t)(14 + c->d_f) * c->n;
  CU_TRY(c, cudaMalloc(&c->grads, sizeof(float) * (size_t)std::max<int64_t>(1, c->grads_floats)));
  c->owns_grads = true;
  CU_TRY(c, cudaMemsetAsync(c->grads, 0, sizeof(float) * (size_t)c->grads_floats, c->stream));
  return SPLATB200_OK;
}

void reset_actor_grads(splatb200_ctx* c) {
  c->actor_d_pose.assign(c->tracks.size(), {});
  c->actor_d_vel.assign(c->tracks.size(), std::vector<double>(6, 0.0));
  for (size_t a = 0; a < c->tracks.size(); ++a) c->actor_d_pose[a].assign(6 * (size_t)c->tracks[a].n_poses(), 0.0);
}

// Fold a view's device-side per-actor sums into the host-side ActorGrad slots (scene.hpp:424-453).
int finalize_actor_grads(splatb200_view* v) {
  splatb200_ctx* c = v->ctx;
  if (!v->actor_pending) return SPLATB200_OK;
  const size_t na = c->tracks.size();
  std::vector<float> acc(kActorAccStride * na);
  CU_TRY(c, cudaMemcpyAsync(acc.data(), v->actor_acc, sizeof(float) * acc.size(), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  CU_TRY(c, cudaMemsetAsync(v->actor_acc, 0, sizeof(float) * acc.size(), c->stream));
  if (c->actor_d_pose.size() != na) reset_actor_grads(c);
  for (size_t a = 0; a < na && a < v->poses.size(); ++a) {
    const float* p = &acc[kActorAccStride * a];
    for (int k = 0; k < 6; ++k) c->actor_d_vel[a][k] += (double)p[6 + k];
    sbh::V3 g_mu{{p[0], p[1], p[2]}}, g_psi{{p[3], p[4], p[5]}};
    sbh::pose_offset_backward(c->tracks[a], v->poses[a], g_mu, g_psi, c->actor_d_pose[a].data());
  }
  v->actor_pending = false;
  return SPLATB200_OK;
}

void free_view_buffers(splatb200_view* v) {
  dfree(v->proj.geomA); dfree(v->proj.geomB); dfree(v->proj.geomC); dfree(v->proj.feat); dfree(v->proj.rect);
  dfree(v->proj.count); dfree(v->offsets); dfree(v->rg);
  dfree(v->proj.dkey); dfree(v->dkey_alt); dfree(v->order0); dfree(v->order1); dfree(v->dsort_temp);
  dfree(v->keys0); dfree(v->keys1); dfree(v->vals0); dfree(v->vals1); dfree(v->sort_temp);
  dfree(v->tile_begin); dfree(v->tile_end); dfree(v->rays); dfree(v->ray_begin); dfree(v->ray_end);
  dfree(v->to_vals0); dfree(v->tile_ws); dfree(v->d_total);
  dfree(v->super_begin); dfree(v->super_end); dfree(v->seg_first); dfree(v->expand_temp); dfree(v->tile_ws_c); dfree(v->d_total_c);
  dfree(v->vals_fine); dfree(v->proj.ccount);
  v->tile_order = nullptr;
  dfree(v->out.blend); dfree(v->out.alpha); dfree(v->out.t_final); dfree(v->out.range_blend);
  dfree(v->out.n_contrib); dfree(v->out.last_idx); dfree(v->out.hit); dfree(v->out.hit_list); dfree(v->out.hit_rows); dfree(v->out.stats); dfree(v->out.tile_wrap); dfree(v->d_los_cut); dfree(v->d_los); dfree(v->d_g_los); dfree(v->d_head_w); dfree(v->d_head_y); for (auto*& b : v->dec_act) dfree(b); for (auto*& b : v->dec_g) dfree(b); dfree(v->dec_gext); dfree(v->d_dec_gimage); dfree(v->d_dec_gparams); dfree(v->d_dec_image); dfree(v->d_dec_params); dfree(v->d_dec_err); dfree(v->g_blend_stage); dfree(v->g_alpha_stage);
  dfree(v->sensor_grads); dfree(v->actor_acc); dfree(v->d_actors);
  if (v->h_total) cudaFreeHost(v->h_total);
  v->h_total = nullptr;
  for (cudaEvent_t* e : {&v->ev_fwd, &v->ev_dl, &v->ev_up, &v->ev_bwd})
    if (*e) { cudaEventDestroy(*e); *e = nullptr; }
  for (cudaStream_t* q : {&v->s_h2d, &v->s_d2h, &v->vs})
    if (*q) { cudaStreamSynchronize(*q); cudaStreamDestroy(*q); *q = nullptr; }
  if (v->ev_last) { cudaEventDestroy(v->ev_last); v->ev_last = nullptr; }
  if (v->ev_ctx) { cudaEventDestroy(v->ev_ctx); v->ev_ctx = nullptr; }
  for (int b = 0; b < 8; ++b)
    for (cudaEvent_t* e : {&v->ev_bfwd[b], &v->ev_bdl[b], &v->ev_bup[b]})
      if (*e) { cudaEventDestroy(*e); *e = nullptr; }
  for (auto& e : v->ev)
    for (auto& x : e)
      if (x) { cudaEventDestroy(x); x = nullptr; }
}

// Fold every recorded-and-completed event pair into the running sums. Only called right after a
// stream synchronisation, so cudaEventElapsedTime never blocks and the timed region is not perturbed.
void harvest_stage_events(splatb200_view* v) {
  for (int k = 0; k < 8; ++k) {
    if (!v->ev_valid[k]) continue;
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, v->ev[k][0], v->ev[k][1]) == cudaSuccess) {
      v->ev_sum_ms[k] += ms;
      v->ev_count[k] += 1;
    }
    v->ev_valid[k] = false;
  }
}

// ---- view streams -----------------------------------------------------------------------------------
// With ctx->view_streams every view enqueues its forward / backward on its own stream, so that one sensor's
// latency-bound binning kernels and the tail of its compositing grid overlap another sensor's kernels. Ordering:
//   * a view's work is ordered after everything asked of the ctx stream before the call (scene upload, zero_grads);
//   * the ctx stream is ordered after the views' work at the ctx-level calls that consume it (zero_grads, uploads,
//     grads_download, ctx_sync, ctx_join) and at every other view-level call on that view.
cudaStream_t work_stream(splatb200_view* v) {
  splatb200_ctx* c = v->ctx;
  if (!c->view_streams) return c->stream;
  if (!v->vs) cudaStreamCreateWithFlags(&v->vs, cudaStreamNonBlocking);
  if (!v->ev_last) cudaEventCreateWithFlags(&v->ev_last, cudaEventDisableTiming);
  if (!v->ev_ctx) cudaEventCreateWithFlags(&v->ev_ctx, cudaEventDisableTiming);
  cudaEventRecord(v->ev_ctx, c->stream);
  cudaStreamWaitEvent(v->vs, v->ev_ctx, 0);
  return v->vs;
}
void mark_busy(splatb200_view* v, cudaStream_t st) {
  if (st == v->ctx->stream || !v->ev_last) return;
  cudaEventRecord(v->ev_last, st);
  v->busy = true;
}
void join_view(splatb200_view* v) {
  if (!v->busy) return;
  cudaStreamWaitEvent(v->ctx->stream, v->ev_last, 0);
  v->busy = false;
}
void join_all(splatb200_ctx* c) {
  for (auto* v : c->views) join_view(v);
}
// ctx-stream consumers of the colour / feature arrays order themselves after a geometry-first upload still in flight
void wait_appearance(splatb200_ctx* c) {
  if (c->app_pending) cudaStreamWaitEvent(c->stream, c->ev_app, 0);
}

struct StageTimer {
  splatb200_view* v;
  int stage;
  cudaStream_t s;
  StageTimer(splatb200_view* view, int st, cudaStream_t stream = nullptr) : v(view), stage(st), s(stream ? stream : view->ctx->stream) {
    if (!v->ctx->profiling) return;
    for (int k = 0; k < 2; ++k)
      if (!v->ev[stage][k]) cudaEventCreate(&v->ev[stage][k]);
    cudaEventRecord(v->ev[stage][0], s);
  }
  ~StageTimer() {
    if (!v->ctx->profiling) return;
    cudaEventRecord(v->ev[stage][1], s);
    v->ev_valid[stage] = true;
  }
};

int ensure_source_buffers(splatb200_view* v) {
  splatb200_ctx* c = v->ctx;
  if (v->n_alloc == c->n && v->proj.count) return SPLATB200_OK;
  dfree(v->proj.geomA); dfree(v->proj.geomB); dfree(v->proj.geomC); dfree(v->proj.feat); dfree(v->proj.rect);
  dfree(v->proj.count); dfree(v->offsets); dfree(v->rg);
  dfree(v->proj.dkey); dfree(v->dkey_alt); dfree(v->order0); dfree(v->order1); dfree(v->dsort_temp);
  const size_t n = (size_t)std::max<int64_t>(1, c->n);
  CU_TRY(c, cudaMalloc(&v->proj.geomA, sizeof(float4) * n));
  CU_TRY(c, cudaMalloc(&v->proj.geomB, sizeof(float4) * n));
  CU_TRY(c, cudaMalloc(&v->proj.geomC, sizeof(float2) * n));
  CU_TRY(c, cudaMalloc(&v->proj.feat, sizeof(float4) * 4 * n));
  CU_TRY(c, cudaMalloc(&v->proj.rect, sizeof(int4) * n));
  CU_TRY(c, cudaMalloc(&v->proj.count, sizeof(uint32_t) * (n + 1)));
  CU_TRY(c, cudaMemsetAsync(v->proj.count, 0, sizeof(uint32_t) * (n + 1), c->stream));
  dfree(v->proj.ccount);
  v->proj.cshift = 0;
  if (v->two_level) {
    CU_TRY(c, cudaMalloc(&v->proj.ccount, sizeof(uint32_t) * (n + 1)));
    v->proj.cshift = super_shift();
  }
  CU_TRY(c, cudaMalloc(&v->proj.dkey, sizeof(uint32_t) * (n + 1)));
  CU_TRY(c, cudaMalloc(&v->dkey_alt, sizeof(uint32_t) * (n + 1)));
  CU_TRY(c, cudaMalloc(&v->order0, sizeof(uint32_t) * (n + 1)));
  CU_TRY(c, cudaMalloc(&v->order1, sizeof(uint32_t) * (n + 1)));
  v->dsort_temp_bytes = depth_sort_temp_bytes((int64_t)n);
  CU_TRY(c, cudaMalloc(&v->dsort_temp, v->dsort_temp_bytes));
  CU_TRY(c, cudaMalloc(&v->offsets, sizeof(uint32_t) * (n + 1)));
  CU_TRY(c, cudaMalloc(&v->rg, sizeof(float) * kRasterGradStride * n));
  CU_TRY(c, cudaMemsetAsync(v->rg, 0, sizeof(float) * kRasterGradStride * n, c->stream));
  v->n_alloc = c->n;
  return SPLATB200_OK;
}

// n_sort: entries the radix sort handles (block-level intersections in two-level mode, else = n_fine)
int ensure_isect_capacity(splatb200_view* v, int64_t n_sort, int64_t n_fine) {
  splatb200_ctx* c = v->ctx;
  if (n_sort > v->isect_cap) {
    dfree(v->keys0); dfree(v->keys1); dfree(v->vals0); dfree(v->vals1); dfree(v->sort_temp);
    const int64_t cap = n_sort + n_sort / 4 + 1024;
    CU_TRY(c, cudaMalloc(&v->keys0, sizeof(uint32_t) * (size_t)cap));
    CU_TRY(c, cudaMalloc(&v->keys1, sizeof(uint32_t) * (size_t)cap));
    CU_TRY(c, cudaMalloc(&v->vals0, sizeof(uint32_t) * (size_t)cap));
    CU_TRY(c, cudaMalloc(&v->vals1, sizeof(uint32_t) * (size_t)cap));
    v->sort_temp_bytes = tile_sort_temp_bytes(cap, v->two_level ? (int64_t)v->stiles_x * v->stiles_y : v->n_tiles);
    CU_TRY(c, cudaMalloc(&v->sort_temp, v->sort_temp_bytes));
    if (v->two_level) {
      dfree(v->expand_temp);
      CU_TRY(c, cudaMalloc(&v->expand_temp, expand_temp_bytes(cap, v->stiles_x * v->stiles_y)));
    }
    v->isect_cap = cap;
  }
  if (n_fine > v->hit_cap) {
    dfree(v->out.hit);
    const int64_t cap = n_fine + n_fine / 4 + 2048;  // padded: the backward reads the hit bytes as aligned 4-byte words
    CU_TRY(c, cudaMalloc(&v->out.hit, (size_t)cap));
    v->hit_cap = cap;
  }
  if (n_fine > v->list_cap) {
    dfree(v->out.hit_list);
    const int64_t cap = n_fine + n_fine / 4 + 2048;
    CU_TRY(c, cudaMalloc(&v->out.hit_list, sizeof(uint32_t) * (size_t)cap));
    v->list_cap = cap;
  }
  if (v->lidar_v2()) {
    const int64_t need = (int64_t)lidar_hit_rows_words(n_fine, v->n_tiles);
    if (need > v->rows_cap) {
      dfree(v->out.hit_rows);
      const int64_t cap = need + need / 4;
      CU_TRY(c, cudaMalloc(&v->out.hit_rows, sizeof(uint32_t) * (size_t)cap));
      v->rows_cap = cap;
    }
  }
  if (v->two_level && n_fine > v->fine_cap) {
    dfree(v->vals_fine);
    const int64_t cap = n_fine + n_fine / 4 + 1024;
    CU_TRY(c, cudaMalloc(&v->vals_fine, sizeof(uint32_t) * (size_t)cap));
    v->fine_cap = cap;
  }
  return SPLATB200_OK;
}

void fill_settings(Sensor& s, const splatb200_raster_settings& st) {
  s.alpha_clamp = st.alpha_clamp; s.alpha_min = st.alpha_min; s.qform_max = st.qform_max;
  s.transmittance_min = st.transmittance_min; s.near_plane = st.near_plane; s.lidar_min_range = st.lidar_min_range;
}

void fill_pose(Sensor& s, const float* R, const float* t, const float* vl, const float* va) {
  for (int k = 0; k < 9; ++k) s.R[k] = R[k];
  for (int k = 0; k < 3; ++k) { s.t[k] = t[k]; s.vel_lin[k] = vl[k]; s.vel_ang[k] = va[k]; }
}

int alloc_query_buffers(splatb200_view* v) {
  splatb200_ctx* c = v->ctx;
  const size_t P = (size_t)std::max<int64_t>(1, v->P), T = (size_t)std::max<int64_t>(1, v->n_tiles);
  CU_TRY(c, cudaMalloc(&v->out.blend, sizeof(float) * 16 * P));
  CU_TRY(c, cudaMalloc(&v->out.alpha, sizeof(float) * P));
  CU_TRY(c, cudaMalloc(&v->out.t_final, sizeof(float) * P));
  CU_TRY(c, cudaMalloc(&v->out.range_blend, sizeof(float) * P));
  CU_TRY(c, cudaMalloc(&v->out.n_contrib, sizeof(int32_t) * P));
  CU_TRY(c, cudaMalloc(&v->out.last_idx, sizeof(int32_t) * P));
  CU_TRY(c, cudaMalloc(&v->tile_begin, sizeof(uint32_t) * T));
  CU_TRY(c, cudaMalloc(&v->tile_end, sizeof(uint32_t) * T));
  CU_TRY(c, cudaMalloc(&v->to_vals0, sizeof(uint32_t) * T));
  CU_TRY(c, cudaMalloc(&v->out.tile_wrap, 8 * T));  // per tile (shared kernels) or per (tile, warp) (lidar v2 kernels)
  CU_TRY(c, cudaMemsetAsync(v->out.tile_wrap, 1, 8 * T, c->stream));
  CU_TRY(c, cudaMalloc(&v->tile_ws, tile_hist_bytes(v->s.tiles_x, v->s.tiles_y)));
  CU_TRY(c, cudaMalloc(&v->d_total, sizeof(int64_t)));
  if (std::getenv("SPLATB200_STATS")) {  // debug counters of the compositing kernels (read through view_array "raster_stats")
    CU_TRY(c, cudaMalloc(&v->out.stats, sizeof(unsigned long long) * 8));
    CU_TRY(c, cudaMemsetAsync(v->out.stats, 0, sizeof(unsigned long long) * 8, c->stream));
  }
  if (v->two_level) {
    const int sh = super_shift();
    v->stiles_x = (v->s.tiles_x + (1 << sh) - 1) >> sh;
    v->stiles_y = (v->s.tiles_y + (1 << sh) - 1) >> sh;
    const size_t Ts = (size_t)std::max(1, v->stiles_x * v->stiles_y);
    CU_TRY(c, cudaMalloc(&v->super_begin, sizeof(uint32_t) * Ts));
    CU_TRY(c, cudaMalloc(&v->super_end, sizeof(uint32_t) * Ts));
    CU_TRY(c, cudaMalloc(&v->seg_first, sizeof(uint32_t) * (Ts + 1)));
    CU_TRY(c, cudaMalloc(&v->tile_ws_c, tile_hist_bytes(v->stiles_x, v->stiles_y)));
    CU_TRY(c, cudaMalloc(&v->d_total_c, sizeof(int64_t)));
  }
  CU_TRY(c, cudaMalloc(&v->sensor_grads, sizeof(float) * 8));
  CU_TRY(c, cudaMemsetAsync(v->sensor_grads, 0, sizeof(float) * 8, c->stream));
  CU_TRY(c, cudaMallocHost(&v->h_total, sizeof(int64_t) * 8));
  return SPLATB200_OK;
}

int lidar_grid_of(float az_res, int n_beams, int* m_phi, int* m_omega) {
  // M_phi = ceil(360deg / (N_phi res_phi)), evaluated in double with a 1e-4-tile guard so
  // that resolutions dividing the circle exactly do not spawn a sliver column from the fp32 rounding of res_phi.
  *m_phi = (int)std::ceil(6.283185307179586476925 / ((double)kNphi * (double)az_res) - 1e-4);
  *m_omega = (n_beams + kNomega - 1) / kNomega;
  return 0;
}

}  // namespace

// ---- context ------------------------------------------------------------------------------------
extern "C" int splatb200_ctx_create(int device, void* cuda_stream, splatb200_ctx** out) {
  if (!out) return SPLATB200_EINVAL;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    g_create_error = std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0") +
                     " (libsplat_b200 has no CPU fallback)";
    return SPLATB200_ECUDA;
  }
  if (device < 0 || device >= count) {
    g_create_error = "device index out of range";
    return SPLATB200_EINVAL;
  }
  e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    return SPLATB200_ECUDA;
  }
  auto* c = new splatb200_ctx();
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  *out = c;
  return SPLATB200_OK;
}

extern "C" void splatb200_ctx_destroy(splatb200_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->s_app) {
    cudaStreamSynchronize(c->s_app);
    cudaStreamDestroy(c->s_app);
    cudaEventDestroy(c->ev_geo);
    cudaEventDestroy(c->ev_app);
  }
  while (!c->views.empty()) splatb200_view_destroy(c->views.back());
  splatb200_ctx_comm_destroy(c);
  free_scene(c);
  delete c;
}

extern "C" const char* splatb200_last_error(const splatb200_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

extern "C" int splatb200_ctx_sync(splatb200_ctx* c) {
  join_all(c);
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->s_app) {
    CU_TRY(c, cudaStreamSynchronize(c->s_app));
    c->app_pending = false;
  }
  for (auto* v : c->views) {  // copy streams of the overlapped host-buffer calls
    if (v->s_h2d) CU_TRY(c, cudaStreamSynchronize(v->s_h2d));
    if (v->s_d2h) CU_TRY(c, cudaStreamSynchronize(v->s_d2h));
  }
  return SPLATB200_OK;
}

extern "C" int64_t splatb200_ctx_launch_count(const splatb200_ctx* c) { return c->launches; }

extern "C" int64_t splatb200_ctx_library_launch_count(const splatb200_ctx* c) { return c->lib_launches; }

extern "C" int splatb200_ctx_set_profiling(splatb200_ctx* c, int32_t on) {
  join_all(c);
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  c->profiling = on != 0;
  for (auto* v : c->views)
    for (int k = 0; k < 8; ++k) { v->ev_valid[k] = false; v->ev_sum_ms[k] = 0.0; v->ev_count[k] = 0; }
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_set_view_streams(splatb200_ctx* c, int32_t on) {
  join_all(c);
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  c->view_streams = on != 0;
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_join(splatb200_ctx* c) {
  join_all(c);
  return SPLATB200_OK;
}

extern "C" int splatb200_view_stage_ms(splatb200_view* v, float out_ms[8]) {
  splatb200_ctx* c = v->ctx;
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  harvest_stage_events(v);
  for (int k = 0; k < 8; ++k) out_ms[k] = v->ev_count[k] ? (float)(v->ev_sum_ms[k] / (double)v->ev_count[k]) : 0.0f;
  return SPLATB200_OK;
}

// ---- scene --------------------------------------------------------------------------------------
extern "C" int splatb200_scene_upload(splatb200_ctx* c, int64_t n, int32_t d_f, const float* mean, const float* scale_log,
                                      const float* quat, const float* opacity_logit, const float* color,
                                      const float* feature, const int32_t* actor_id) {
  join_all(c);
  if (n < 0 || d_f < 0 || d_f > 13) return c->fail(SPLATB200_EINVAL, "scene_upload: need n >= 0 and 0 <= d_f <= 13");
  CU_TRY(c, cudaSetDevice(c->device));
  if (c->s_app) {  // an asynchronous upload still in flight writes the same buffers
    CU_TRY(c, cudaStreamSynchronize(c->s_app));
    c->app_pending = false;
  }
  // Same shape as the resident scene (the per-iteration case: parameters change, sizes do not): keep the
  // device buffers and the SceneParamGrads buffer (owned or bound), only refresh the contents.
  const bool reuse = c->owns_scene && c->n == n && c->d_f == d_f && c->grads;
  if (!reuse) {
    CU_TRY(c, cudaStreamSynchronize(c->stream));
    free_scene(c);
    c->n = n;
    c->d_f = d_f;
    c->owns_scene = true;
  }
  const size_t m = (size_t)std::max<int64_t>(1, n);
  auto up = [&](float*& dst, const float* src, int width) -> cudaError_t {
    if (!reuse) {
      cudaError_t e = cudaMalloc(&dst, sizeof(float) * m * (size_t)std::max(1, width));
      if (e != cudaSuccess) return e;
    }
    if (n == 0 || width == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, sizeof(float) * (size_t)n * width, cudaMemcpyHostToDevice, c->stream);
  };
  CU_TRY(c, up(c->mean, mean, 3));
  CU_TRY(c, up(c->scale_log, scale_log, 3));
  CU_TRY(c, up(c->quat, quat, 4));
  CU_TRY(c, up(c->opacity_logit, opacity_logit, 1));
  CU_TRY(c, up(c->color, color, 3));
  CU_TRY(c, up(c->feature, feature, d_f));
  if (!reuse) CU_TRY(c, cudaMalloc(&c->actor_id, sizeof(int32_t) * m));
  if (n) CU_TRY(c, cudaMemcpyAsync(c->actor_id, actor_id, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  c->actor_first.clear();
  for (int64_t i = 0; i < n; ++i)
    if (actor_id[i] != 0) c->actor_first.emplace(actor_id[i], i);
  c->bound_max_actor = 0;
  // host arrays are borrowed for the duration of the call only (pageable or pinned)
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  for (auto* v : c->views) v->stage = 0;
  return reuse ? SPLATB200_OK : alloc_grads(c);
}

extern "C" int splatb200_scene_upload_async(splatb200_ctx* c, int64_t n, int32_t d_f, const float* mean, const float* scale_log,
                                            const float* quat, const float* opacity_logit, const float* color,
                                            const float* feature, const int32_t* actor_id) {
  // only the per-iteration case (same shape as the resident scene, buffers owned): anything else takes the blocking path
  if (!(c->owns_scene && c->n == n && c->d_f == d_f && c->grads) || n == 0)
    return splatb200_scene_upload(c, n, d_f, mean, scale_log, quat, opacity_logit, color, feature, actor_id);
  join_all(c);
  CU_TRY(c, cudaSetDevice(c->device));
  if (!c->s_app) {
    CU_TRY(c, cudaStreamCreateWithFlags(&c->s_app, cudaStreamNonBlocking));
    CU_TRY(c, cudaEventCreateWithFlags(&c->ev_geo, cudaEventDisableTiming));
    CU_TRY(c, cudaEventCreateWithFlags(&c->ev_app, cudaEventDisableTiming));
  }
  auto up = [&](void* dst, const void* src, size_t bytes, cudaStream_t st) { return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st); };
  const size_t fn = sizeof(float) * (size_t)n;
  // geometry (48 B per Gaussian) on the ctx stream: everything up to the tile lists needs nothing else
  CU_TRY(c, up(c->mean, mean, 3 * fn, c->stream));
  CU_TRY(c, up(c->scale_log, scale_log, 3 * fn, c->stream));
  CU_TRY(c, up(c->quat, quat, 4 * fn, c->stream));
  CU_TRY(c, up(c->opacity_logit, opacity_logit, fn, c->stream));
  CU_TRY(c, up(c->actor_id, actor_id, sizeof(int32_t) * (size_t)n, c->stream));
  CU_TRY(c, cudaEventRecord(c->ev_geo, c->stream));
  // appearance (12 + 4 d_f B per Gaussian) behind it on the link, but on its own stream: the views' projection and
  // binning kernels run while it is in flight
  CU_TRY(c, cudaStreamWaitEvent(c->s_app, c->ev_geo, 0));
  CU_TRY(c, up(c->color, color, 3 * fn, c->s_app));
  if (d_f) CU_TRY(c, up(c->feature, feature, (size_t)d_f * fn, c->s_app));
  CU_TRY(c, cudaEventRecord(c->ev_app, c->s_app));
  c->app_pending = true;
  c->actor_first.clear();
  for (int64_t i = 0; i < n; ++i)
    if (actor_id[i] != 0) c->actor_first.emplace(actor_id[i], i);
  c->bound_max_actor = 0;
  for (auto* v : c->views) v->stage = 0;
  return SPLATB200_OK;
}

extern "C" int splatb200_scene_bind_device(splatb200_ctx* c, int64_t n, int32_t d_f, const float* mean,
                                           const float* scale_log, const float* quat, const float* opacity_logit,
                                           const float* color, const float* feature, const int32_t* actor_id,
                                           int32_t max_actor_id) {
  join_all(c);
  if (n < 0 || d_f < 0 || d_f > 13) return c->fail(SPLATB200_EINVAL, "scene_bind_device: need n >= 0 and 0 <= d_f <= 13");
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  float* keep_grads = c->owns_grads ? nullptr : c->grads;
  const int64_t keep_floats = c->grads_floats;
  free_scene(c);
  c->n = n;
  c->d_f = d_f;
  c->mean = const_cast<float*>(mean); c->scale_log = const_cast<float*>(scale_log); c->quat = const_cast<float*>(quat);
  c->opacity_logit = const_cast<float*>(opacity_logit); c->color = const_cast<float*>(color);
  c->feature = const_cast<float*>(feature); c->actor_id = const_cast<int32_t*>(actor_id);
  c->actor_first.clear();
  c->bound_max_actor = max_actor_id;
  for (auto* v : c->views) v->stage = 0;
  if (n > 0 && actor_id) {
    // the caller's max_actor_id is a claim: ids outside [0, max_actor_id] would index the actor table out of bounds on
    // the device (scene_upload checks the same on the host)
    int h[2] = {0x7fffffff, -0x7fffffff - 1};
    int* d = nullptr;
    CU_TRY(c, cudaMalloc(&d, sizeof(h)));
    cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, c->stream);
    launch_actor_id_range(actor_id, n, d, c->stream);
    cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    cudaFree(d);
    if (e != cudaSuccess) return c->fail(SPLATB200_ECUDA, std::string("scene_bind_device: ") + cudaGetErrorString(e));
    c->launches += 1;
    if (h[0] < 0 || h[1] > max_actor_id)
      return c->fail(SPLATB200_EOUTOFRANGE, "scene_bind_device: actor_id values span [" + std::to_string(h[0]) + ", " +
                                                std::to_string(h[1]) + "], outside [0, max_actor_id = " + std::to_string(max_actor_id) + "]");
  }
  if (keep_grads && keep_floats == (int64_t)(14 + d_f) * n) {
    c->grads = keep_grads;
    c->grads_floats = keep_floats;
    return SPLATB200_OK;
  }
  return alloc_grads(c);
}

extern "C" int splatb200_scene_set_tracks(splatb200_ctx* c, int32_t n_tracks, const splatb200_actor_track* tracks) {
  if (n_tracks < 0) return c->fail(SPLATB200_EINVAL, "negative track count");
  for (auto* v : c->views) {
    int rc = finalize_actor_grads(v);
    if (rc) return rc;
    v->stage = 0;
  }
  c->tracks.clear();
  for (int a = 0; a < n_tracks; ++a) {
    const auto& t = tracks[a];
    sbh::Track tk;
    const int np = t.n_poses;
    tk.stamps.assign(t.stamps, t.stamps + np);
    tk.R.assign(t.R, t.R + 9 * np);
    tk.t.assign(t.t, t.t + 3 * np);
    if (t.pose_offset) tk.pose_offset.assign(t.pose_offset, t.pose_offset + 6 * np);
    else tk.pose_offset.assign(6 * (size_t)np, 0.0);
    for (int k = 0; k < 3; ++k) { tk.vel_lin[k] = t.vel_lin[k]; tk.vel_ang[k] = t.vel_ang[k]; }
    for (int k = 0; k < 6; ++k) tk.vel_offset[k] = t.vel_offset[k];
    if (t.init_velocity_from_poses) tk.init_velocity_from_poses();
    c->tracks.push_back(std::move(tk));
  }
  reset_actor_grads(c);
  return SPLATB200_OK;
}

extern "C" int splatb200_scene_actor_velocity(splatb200_ctx* c, int32_t track, double out6[6]) {
  if (track < 0 || track >= (int)c->tracks.size()) return c->fail(SPLATB200_EINVAL, "track index out of range");
  for (int k = 0; k < 3; ++k) { out6[k] = c->tracks[track].vel_lin[k]; out6[3 + k] = c->tracks[track].vel_ang[k]; }
  return SPLATB200_OK;
}

// ---- grads --------------------------------------------------------------------------------------
extern "C" int splatb200_grads_zero(splatb200_ctx* c) {
  join_all(c);
  if (c->grads) CU_TRY(c, cudaMemsetAsync(c->grads, 0, sizeof(float) * (size_t)c->grads_floats, c->stream));
  for (auto* v : c->views) {
    if (v->actor_pending) {
      CU_TRY(c, cudaMemsetAsync(v->actor_acc, 0, sizeof(float) * kActorAccStride * c->tracks.size(), c->stream));
      v->actor_pending = false;
    }
  }
  reset_actor_grads(c);
  return SPLATB200_OK;
}
extern "C" int64_t splatb200_grads_size(const splatb200_ctx* c) { return c->grads_floats; }
extern "C" float* splatb200_grads_device_ptr(splatb200_ctx* c) { return c->grads; }
extern "C" int splatb200_grads_bind_device(splatb200_ctx* c, float* dev, int64_t n_floats) {
  join_all(c);
  if (n_floats != (int64_t)(14 + c->d_f) * c->n) return c->fail(SPLATB200_EINVAL, "grads_bind_device: size must be (14 + d_f) * N floats");
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->owns_grads) dfree(c->grads);
  c->grads = dev;
  c->owns_grads = false;
  c->grads_floats = n_floats;
  return SPLATB200_OK;
}
extern "C" int splatb200_grads_download(splatb200_ctx* c, float* d_mean, float* d_scale_log, float* d_quat,
                                        float* d_opacity_logit, float* d_color, float* d_feature) {
  join_all(c);
  const ParamGradDev g = c->pg();
  const size_t n = (size_t)c->n;
  auto dl = [&](float* dst, const float* src, size_t w) -> cudaError_t {
    if (!dst || n * w == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, sizeof(float) * n * w, cudaMemcpyDeviceToHost, c->stream);
  };
  CU_TRY(c, dl(d_mean, g.d_mean, 3));
  CU_TRY(c, dl(d_scale_log, g.d_scale_log, 3));
  CU_TRY(c, dl(d_quat, g.d_quat, 4));
  CU_TRY(c, dl(d_opacity_logit, g.d_opacity_logit, 1));
  CU_TRY(c, dl(d_color, g.d_color, 3));
  CU_TRY(c, dl(d_feature, g.d_feature, (size_t)c->d_f));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}
extern "C" int splatb200_grads_download_actor(splatb200_ctx* c, int32_t track, double* d_pose_offset, double* d_vel_offset6) {
  join_all(c);
  if (track < 0 || track >= (int)c->tracks.size()) return c->fail(SPLATB200_EINVAL, "track index out of range");
  for (auto* v : c->views) {
    int rc = finalize_actor_grads(v);
    if (rc) return rc;
  }
  if (d_pose_offset) std::memcpy(d_pose_offset, c->actor_d_pose[track].data(), sizeof(double) * c->actor_d_pose[track].size());
  if (d_vel_offset6) std::memcpy(d_vel_offset6, c->actor_d_vel[track].data(), sizeof(double) * 6);
  return SPLATB200_OK;
}

// ---- views --------------------------------------------------------------------------------------
extern "C" int splatb200_view_set_camera(splatb200_view* v, const splatb200_camera* cam) {
  splatb200_ctx* c = v->ctx;
  if (!v->s.is_camera) return c->fail(SPLATB200_EINVAL, "view is not a camera");
  if (cam->width != v->s.width || cam->height != v->s.height) return c->fail(SPLATB200_EINVAL, "camera size is fixed per view");
  v->s.fx = cam->fx; v->s.fy = cam->fy; v->s.cx = cam->cx; v->s.cy = cam->cy;
  fill_pose(v->s, cam->R, cam->t, cam->vel_lin, cam->vel_ang);
  v->s.shutter = cam->shutter_duration;
  v->s.time_offset = cam->time_offset;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_set_lidar_pose(splatb200_view* v, const float R[9], const float t[3], const float vel_lin[3],
                                             const float vel_ang[3]) {
  if (v->s.is_camera) return v->ctx->fail(SPLATB200_EINVAL, "view is not a lidar");
  fill_pose(v->s, R, t, vel_lin, vel_ang);
  return SPLATB200_OK;
}

extern "C" int splatb200_view_create_camera(splatb200_ctx* c, const splatb200_camera* cam,
                                            const splatb200_raster_settings* st, splatb200_view** out) {
  if (!cam || !st || !out) return c->fail(SPLATB200_EINVAL, "null argument");
  if (cam->width < 1 || cam->height < 1) return c->fail(SPLATB200_EINVAL, "camera needs W, H >= 1");
  CU_TRY(c, cudaSetDevice(c->device));
  auto* v = new splatb200_view();
  v->ctx = c;
  std::memset(&v->s, 0, sizeof(Sensor));
  v->s.is_camera = 1;
  v->s.width = cam->width; v->s.height = cam->height;
  fill_settings(v->s, *st);
  v->s.dilation = st->dilation;
  v->s.tiles_x = (cam->width + kTile - 1) / kTile;
  v->s.tiles_y = (cam->height + kTile - 1) / kTile;
  v->P = (int64_t)cam->width * cam->height;
  v->n_tiles = (int64_t)v->s.tiles_x * v->s.tiles_y;
  v->two_level = std::getenv("SPLATB200_ONE_LEVEL") == nullptr;  // cameras bin in two levels (debug switch: one level)
  c->views.push_back(v);
  int rc = splatb200_view_set_camera(v, cam);
  if (!rc) rc = alloc_query_buffers(v);
  if (rc) {
    splatb200_view_destroy(v);
    return rc;
  }
  *out = v;
  return SPLATB200_OK;
}

extern "C" int splatb200_lidar_grid(const splatb200_lidar* l, int32_t* m_phi, int32_t* m_omega) {
  int a, b;
  lidar_grid_of(l->azimuth_resolution, l->n_beams, &a, &b);
  if (m_phi) *m_phi = a;
  if (m_omega) *m_omega = b;
  return SPLATB200_OK;
}

namespace {
// ---- warp patches of a lidar tile ----------------------------------------------------------------------------------
// 32 consecutive ray positions are one warp of the compositing kernels, and per-warp culling keeps a Gaussian for a warp
// when its footprint (diameter ~d) meets the bounding box of the warp's rays: the expected number of survivors is
// ~ (w + d)(h + d) for a w x h box. On a non-uniform elevation grid the best 32-ray shape differs from row to row: where
// beams are 0.13 degrees apart 4 azimuth bins x 8 beams is compact, where they are 0.8 degrees apart 32 bins x 1 beam
// is (a footprint of 0.5 degrees meets one beam, and 8 beams would span 6 degrees). The rays of a tile are therefore
// grouped by recursive bisection of the (relative azimuth, elevation) point set at multiples of 32 rays, choosing at
// every level the axis that minimises the summed (w + d)(h + d) of the leaves (exhaustive over the last three levels,
// i.e. one 256-ray pass; greedy above). Any ray set works; nothing assumes a lattice.
struct PatchRay { float x, y; int64_t r; };
float patch_leaf_cost(const PatchRay* p, int64_t n, float d) {
  float x0 = p[0].x, x1 = p[0].x, y0 = p[0].y, y1 = p[0].y;
  for (int64_t i = 1; i < n; ++i) { x0 = std::min(x0, p[i].x); x1 = std::max(x1, p[i].x); y0 = std::min(y0, p[i].y); y1 = std::max(y1, p[i].y); }
  return (x1 - x0 + d) * (y1 - y0 + d);
}
// inside one warp patch (n <= 32): consecutive 8-ray groups — the 8-lane groups of the forward compositing kernel —
// compact, by the same exhaustive bisection (at multiples of 8)
float group_order(PatchRay* p, int64_t n, float d) {
  if (n <= 8) return patch_leaf_cost(p, n, d);
  const int64_t half = (((n + 7) / 8 + 1) / 2) * 8;
  auto by_x = [](const PatchRay& a, const PatchRay& b) { return a.x < b.x || (a.x == b.x && (a.y < b.y || (a.y == b.y && a.r < b.r))); };
  auto by_y = [](const PatchRay& a, const PatchRay& b) { return a.y < b.y || (a.y == b.y && (a.x < b.x || (a.x == b.x && a.r < b.r))); };
  PatchRay alt[32];
  std::copy(p, p + n, alt);
  std::sort(p, p + n, by_x);
  const float cx = group_order(p, half, d) + group_order(p + half, n - half, d);
  std::sort(alt, alt + n, by_y);
  const float cy = group_order(alt, half, d) + group_order(alt + half, n - half, d);
  if (cy < cx) { std::copy(alt, alt + n, p); return cy; }
  return cx;
}
// orders p[0, n) in place so that consecutive 32-ray groups are compact patches; returns the summed leaf cost
float patch_order(PatchRay* p, int64_t n, float d) {
  if (n <= 32) {
    const float c = patch_leaf_cost(p, n, d);
    group_order(p, n, d);
    return c;
  }
  const int64_t groups = (n + 31) / 32;
  // passes of 256 rays stay compact too: above one pass, split at multiples of 8 groups
  const int64_t half = groups > 8 ? ((groups + 15) / 16) * 8 * 32 : ((groups + 1) / 2) * 32;
  auto by_x = [](const PatchRay& a, const PatchRay& b) { return a.x < b.x || (a.x == b.x && (a.y < b.y || (a.y == b.y && a.r < b.r))); };
  auto by_y = [](const PatchRay& a, const PatchRay& b) { return a.y < b.y || (a.y == b.y && (a.x < b.x || (a.x == b.x && a.r < b.r))); };
  if (groups > 8) {  // greedy: the longer axis
    float x0 = p[0].x, x1 = p[0].x, y0 = p[0].y, y1 = p[0].y;
    for (int64_t i = 1; i < n; ++i) { x0 = std::min(x0, p[i].x); x1 = std::max(x1, p[i].x); y0 = std::min(y0, p[i].y); y1 = std::max(y1, p[i].y); }
    if (x1 - x0 >= y1 - y0) std::sort(p, p + n, by_x); else std::sort(p, p + n, by_y);
    return patch_order(p, half, d) + patch_order(p + half, n - half, d);
  }
  std::vector<PatchRay> alt(p, p + n);
  std::sort(p, p + n, by_x);
  const float cx = patch_order(p, half, d) + patch_order(p + half, n - half, d);
  std::sort(alt.begin(), alt.end(), by_y);
  const float cy = patch_order(alt.data(), half, d) + patch_order(alt.data() + half, n - half, d);
  if (cy < cx) { std::copy(alt.begin(), alt.end(), p); return cy; }
  return cx;
}

// Packs and uploads a lidar view's rays (shared by view_create_lidar and view_set_rays). Within a tile the rays are
// re-ordered into compact 32-ray patches (patch_order above) that per-warp culling can exploit. The original index
// travels in .w; outputs keep the caller's ray order. Needs v->rays capacity >= n_rays (v->P_cap).
int upload_rays(splatb200_view* v, const float* rays, int64_t n_rays, const int64_t* ray_begin, const int64_t* ray_end) {
  splatb200_ctx* c = v->ctx;
  const int64_t n_tiles = v->n_tiles;
  if (n_rays > 0xffffffffLL) return c->fail(SPLATB200_EINVAL, "more than 2^32-1 rays in one view");
  if (n_rays > 0 && !rays) return c->fail(SPLATB200_EINVAL, "null rays");
  for (int64_t t = 0; t < n_tiles; ++t)
    if (ray_begin[t] < 0 || ray_end[t] < ray_begin[t] || ray_end[t] > n_rays)
      return c->fail(SPLATB200_EINVAL, "ray_begin/ray_end must delimit slices of the ray array");
  v->multi_pass = false;
  for (int64_t t = 0; t < n_tiles; ++t)
    if (ray_end[t] - ray_begin[t] > 256) v->multi_pass = true;  // several passes over a tile's list
  std::vector<float4> packed((size_t)std::max<int64_t>(1, n_rays));
  {
    // typical footprint diameter the grouping assumes (radians); SPLATB200_PATCH_D overrides, 0 = azimuth-major order
    float patch_d = 0.015f;
    if (const char* e = std::getenv("SPLATB200_PATCH_D")) patch_d = (float)std::atof(e);
    std::vector<PatchRay> keyed;
    for (int64_t t = 0; t < n_tiles; ++t) {
      const int64_t b = ray_begin[t], e = ray_end[t];
      if (e <= b) continue;
      keyed.clear();
      const float ref = rays[3 * b];
      for (int64_t r = b; r < e; ++r) {
        float rel = std::fmod(rays[3 * r] - ref, 6.283185307179586f);   // wrap to (-pi, pi] around the tile's first ray
        if (rel > 3.14159265358979f) rel -= 6.283185307179586f;
        if (rel <= -3.14159265358979f) rel += 6.283185307179586f;
        keyed.push_back({rel, rays[3 * r + 1], r});
      }
      if (patch_d > 0.0f) {
        patch_order(keyed.data(), (int64_t)keyed.size(), patch_d);
      } else {
        std::stable_sort(keyed.begin(), keyed.end(), [](const PatchRay& x, const PatchRay& y) { return x.x < y.x || (x.x == y.x && x.y < y.y); });
      }
      for (int64_t k = 0; k < e - b; ++k) {
        const int64_t r = keyed[(size_t)k].r;
        const uint32_t bits = (uint32_t)r;
        float w;
        std::memcpy(&w, &bits, 4);
        packed[(size_t)(b + k)] = make_float4(rays[3 * r], rays[3 * r + 1], rays[3 * r + 2], w);
      }
    }
  }
  if (!v->rays && cudaMalloc(&v->rays, sizeof(float4) * (size_t)v->P_cap) != cudaSuccess)
    return c->fail(SPLATB200_ENOMEM, "cudaMalloc rays");
  if (n_rays) cudaMemcpyAsync(v->rays, packed.data(), sizeof(float4) * (size_t)n_rays, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(v->ray_begin, ray_begin, sizeof(int64_t) * n_tiles, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(v->ray_end, ray_end, sizeof(int64_t) * n_tiles, cudaMemcpyHostToDevice, c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->fail(SPLATB200_ECUDA, "ray upload failed");
  v->P = n_rays;
  return SPLATB200_OK;
}
}  // namespace

extern "C" int splatb200_view_create_lidar(splatb200_ctx* c, const splatb200_lidar* l, const splatb200_raster_settings* st,
                                           const float* rays, int64_t n_rays, const int64_t* ray_begin,
                                           const int64_t* ray_end, int64_t n_tiles, splatb200_view** out) {
  if (!l || !st || !out || n_rays < 0) return c->fail(SPLATB200_EINVAL, "null argument");
  if (l->n_beams < 1 || !(l->azimuth_resolution > 0.0f)) return c->fail(SPLATB200_EINVAL, "lidar needs beams and res_phi > 0");
  CU_TRY(c, cudaSetDevice(c->device));
  int m_phi, m_omega;
  lidar_grid_of(l->azimuth_resolution, l->n_beams, &m_phi, &m_omega);
  if (m_omega - 1 > kMaxBoundaries) return c->fail(SPLATB200_EINVAL, "too many beams");
  if (n_tiles != (int64_t)m_phi * m_omega) return c->fail(SPLATB200_EINVAL, "n_tiles must equal M_phi * M_omega");
  auto* v = new splatb200_view();
  v->ctx = c;
  std::memset(&v->s, 0, sizeof(Sensor));
  v->s.is_camera = 0;
  fill_settings(v->s, *st);
  fill_pose(v->s, l->R, l->t, l->vel_lin, l->vel_ang);
  v->s.shutter = l->scan_duration;
  v->s.dilation = l->beam_divergence_h * l->beam_divergence_v;  // scene.hpp:152, projection.hpp:149
  v->s.elev_min = l->elevation_channels[0];
  v->s.elev_max = l->elevation_channels[l->n_beams - 1];
  v->s.tiles_x = m_phi;
  v->s.tiles_y = m_omega;
  v->s.span = (float)kNphi * l->azimuth_resolution;
  v->s.phi_max = (float)m_phi * v->s.span;
  v->s.n_boundaries = m_omega - 1;
  for (int k = 1; k < m_omega; ++k)  // midway between channels 8k-1 and 8k
    v->s.boundaries[k - 1] = 0.5f * (l->elevation_channels[kNomega * k - 1] + l->elevation_channels[kNomega * k]);
  v->P = n_rays;
  v->n_tiles = n_tiles;
  c->views.push_back(v);
  int rc = alloc_query_buffers(v);
  auto fin = [&](int code) {
    splatb200_view_destroy(v);
    return code;
  };
  if (rc) return fin(rc);
  if (cudaMalloc(&v->ray_begin, sizeof(int64_t) * n_tiles) != cudaSuccess || cudaMalloc(&v->ray_end, sizeof(int64_t) * n_tiles) != cudaSuccess)
    return fin(c->fail(SPLATB200_ENOMEM, "cudaMalloc ray slices"));
  v->P_cap = std::max<int64_t>(1, n_rays);
  rc = upload_rays(v, rays, n_rays, ray_begin, ray_end);
  if (rc) return fin(rc);
  *out = v;
  return SPLATB200_OK;
}

extern "C" void splatb200_view_destroy(splatb200_view* v) {
  if (v && v->vs) cudaStreamSynchronize(v->vs);
  if (!v) return;
  splatb200_ctx* c = v->ctx;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  finalize_actor_grads(v);
  {
    std::lock_guard<std::mutex> lk(c->xfer_mu);  // the yield slots may hold this view's events
    c->yield_dl = nullptr;
    c->yield_ul = nullptr;
  }
  free_view_buffers(v);
  for (size_t k = 0; k < c->views.size(); ++k)
    if (c->views[k] == v) {
      c->views.erase(c->views.begin() + k);
      break;
    }
  delete v;
}

// ---- optimizer step -----------------------------------------------------------------------
namespace {
int ensure_adam_state(splatb200_ctx* c) {
  const int64_t total = c->grads_floats;
  if (c->adam_floats == total && c->adam_m) return SPLATB200_OK;
  dfree(c->adam_m); dfree(c->adam_v); dfree(c->adam_bad);
  CU_TRY(c, cudaMalloc(&c->adam_m, sizeof(float) * (size_t)std::max<int64_t>(1, total)));
  CU_TRY(c, cudaMalloc(&c->adam_v, sizeof(float) * (size_t)std::max<int64_t>(1, total)));
  CU_TRY(c, cudaMalloc(&c->adam_bad, sizeof(int) * 6));
  CU_TRY(c, cudaMemsetAsync(c->adam_m, 0, sizeof(float) * (size_t)total, c->stream));
  CU_TRY(c, cudaMemsetAsync(c->adam_v, 0, sizeof(float) * (size_t)total, c->stream));
  c->adam_floats = total;
  return SPLATB200_OK;
}
AdamGroups adam_groups(const splatb200_ctx* c) {
  const int64_t width[6] = {3, 3, 4, 1, 3, c->d_f};
  AdamGroups gr;
  gr.begin[0] = 0;
  for (int k = 0; k < 6; ++k) gr.begin[k + 1] = gr.begin[k] + width[k] * c->n;
  return gr;
}
// flags the groups with a non-finite gradient inside [lo, hi) into c->adam_bad (device), after clearing it
int flag_nonfinite(splatb200_ctx* c, int64_t lo, int64_t hi) {
  AdamGroups gr = adam_groups(c);
  for (int k = 0; k <= 6; ++k) gr.begin[k] = std::min(std::max(gr.begin[k], lo), hi) - lo;  // slices relative to lo
  CU_TRY(c, cudaMemsetAsync(c->adam_bad, 0, sizeof(int) * 6, c->stream));
  launch_grad_finite(c->grads + lo, hi - lo, gr, c->adam_bad, c->stream);
  return SPLATB200_OK;
}
}  // namespace

extern "C" int splatb200_grads_nonfinite_range(splatb200_ctx* c, int64_t lo, int64_t hi, int32_t flags[6]) {
  if (!c->grads || !flags) return c->fail(SPLATB200_ERUNTIME, "grads_nonfinite_range without gradients");
  if (lo < 0 || hi < lo || hi > c->grads_floats) return c->fail(SPLATB200_EINVAL, "range outside the gradient buffer");
  CU_TRY(c, cudaSetDevice(c->device));
  join_all(c);
  int rc = ensure_adam_state(c);
  if (!rc) rc = flag_nonfinite(c, lo, hi);
  if (rc) return rc;
  int h[6];
  CU_TRY(c, cudaMemcpyAsync(h, c->adam_bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 6; ++k) flags[k] = h[k] != 0;
  return SPLATB200_OK;
}

extern "C" int splatb200_optimizer_step_range(splatb200_ctx* c, const splatb200_adam_config* cfg, int64_t step, int64_t lo,
                                              int64_t hi, const int32_t skip_groups[6], int32_t skipped[6]) {
  if (!cfg || step < 0) return c->fail(SPLATB200_EINVAL, "optimizer_step: bad arguments");
  if (!c->mean || !c->grads) return c->fail(SPLATB200_ERUNTIME, "optimizer_step without a scene");
  if (lo < 0 || hi < lo || hi > c->grads_floats) return c->fail(SPLATB200_EINVAL, "range outside the gradient buffer");
  CU_TRY(c, cudaSetDevice(c->device));
  join_all(c);
  wait_appearance(c);
  int rc = ensure_adam_state(c);
  if (!rc) rc = flag_nonfinite(c, lo, hi);
  if (rc) return rc;
  if (skip_groups) {  // groups another shard found non-finite
    int h[6], any = 0;
    for (int k = 0; k < 6; ++k) { h[k] = skip_groups[k] != 0; any |= h[k]; }
    if (any) {
      int cur[6];
      CU_TRY(c, cudaMemcpyAsync(cur, c->adam_bad, sizeof(cur), cudaMemcpyDeviceToHost, c->stream));
      CU_TRY(c, cudaStreamSynchronize(c->stream));
      for (int k = 0; k < 6; ++k) cur[k] |= h[k];
      CU_TRY(c, cudaMemcpy(c->adam_bad, cur, sizeof(cur), cudaMemcpyHostToDevice));
    }
  }
  for (int k = 0; k < 6; ++k) {  // lr_init == 0 freezes a group; anything else must be a valid exponential schedule
    if (!(cfg->lr_init[k] >= 0.0f) || (cfg->lr_init[k] > 0.0f && !(cfg->lr_final[k] > 0.0f)) || !std::isfinite(cfg->lr_init[k]) ||
        !std::isfinite(cfg->lr_final[k]))
      return c->fail(SPLATB200_EINVAL, "optimizer_step: group " + std::to_string(k) + " needs lr_init >= 0 and, unless frozen (lr_init == 0), lr_final > 0");
  }
  const AdamGroups gr = adam_groups(c);
  float* params[6] = {c->mean, c->scale_log, c->quat, c->opacity_logit, c->color, c->feature};
  const double t1 = (double)step + 1.0;
  const float bc1 = (float)(1.0 / (1.0 - std::pow(0.9, t1))), bc2 = (float)(1.0 / (1.0 - std::pow(0.999, t1)));
  int launched = 1;
  for (int k = 0; k < 6; ++k) {
    const int64_t a = std::max(gr.begin[k], lo), b = std::min(gr.begin[k + 1], hi);
    if (b <= a) continue;
    const double w = (double)cfg->warmup_steps[k];
    const double ramp = w > 0 ? std::min(1.0, (double)step / w) : 1.0;
    const double denom = (double)cfg->total_steps - w;
    const double t = denom > 0 ? std::min(1.0, std::max(0.0, ((double)step - w) / denom)) : 1.0;
    if (cfg->lr_init[k] == 0.0f) continue;  // frozen group: parameters and moments untouched
    const double lr = ramp * (double)cfg->lr_init[k] * std::pow((double)cfg->lr_final[k] / (double)cfg->lr_init[k], t);
    launch_adam(params[k] + (a - gr.begin[k]), c->grads + a, c->adam_m + a, c->adam_v + a, b - a, (float)lr, bc1, bc2,
                c->adam_bad + k, c->stream);
    ++launched;
  }
  CHECK_LAUNCH(c, "k_adam");
  c->launches += launched;
  if (skipped) {
    int h[6];
    CU_TRY(c, cudaMemcpyAsync(h, c->adam_bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CU_TRY(c, cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 6; ++k) skipped[k] = h[k] != 0;
  }
  for (auto* v : c->views) v->stage = 0;  // renders belong to the old parameters
  return SPLATB200_OK;
}

extern "C" int splatb200_optimizer_step(splatb200_ctx* c, const splatb200_adam_config* cfg, int64_t step, int32_t skipped[6]) {
  return splatb200_optimizer_step_range(c, cfg, step, 0, c->grads_floats, nullptr, skipped);
}

extern "C" int splatb200_optimizer_reset(splatb200_ctx* c) {
  // forget the Adam moments (a scene_upload of the same shape keeps them: that is the per-iteration parameter refresh)
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(c->adam_m); dfree(c->adam_v); dfree(c->adam_bad);
  c->adam_floats = 0;
  return SPLATB200_OK;
}

// ---- multi-GPU: NCCL all-reduce of SceneParamGrads (scene.hpp:351-362) ----------------------------------
// NCCL is bound at run time: a trainer (or torch) has its own libnccl.so.2 in the process, and a second copy linked into
// this library could not share its communicators.
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string why;
};
NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if (!api.h) api.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // the copy the process already uses
    for (const char* n : names)
      if (!api.h) api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) { api.why = std::string("libnccl.so.2 not found: ") + dlerror(); return; }
    auto sym = [&](const char* s) { void* p = dlsym(api.h, s); if (!p && api.why.empty()) api.why = std::string("missing NCCL symbol ") + s; return p; };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.Reduce = (decltype(api.Reduce))sym("ncclReduce");
    api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  });
  return api.why.empty() ? &api : nullptr;
}
#define NCCL_TRY(ctx, api, call)                                                                                   \
  do {                                                                                                             \
    ncclResult_t r__ = (call);                                                                                     \
    if (r__ != ncclSuccess) return (ctx)->fail(SPLATB200_ERUNTIME, std::string(#call) + ": " + (api)->GetErrorString(r__)); \
  } while (0)

// [lo, hi) of the flat gradient layout owned by `rank`: equal shards aligned to 4 floats (the last may be shorter)
void shard_of(int64_t total, int world, int rank, int64_t& lo, int64_t& hi) {
  int64_t per = (total + world - 1) / world;
  per = (per + 3) / 4 * 4;
  lo = std::min<int64_t>(total, (int64_t)rank * per);
  hi = std::min<int64_t>(total, lo + per);
}
}  // namespace

extern "C" int splatb200_nccl_unique_id(void* id128) {
  NcclApi* a = nccl_api();
  if (!a || !id128) return SPLATB200_ERUNTIME;
  ncclUniqueId id;
  if (a->GetUniqueId(&id) != ncclSuccess) return SPLATB200_ERUNTIME;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, 128);
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_comm_destroy(splatb200_ctx* c) {
  if (c->comm && c->owns_comm) {
    NcclApi* a = nccl_api();
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (a) a->CommDestroy((ncclComm_t)c->comm);
  }
  c->comm = nullptr;
  c->owns_comm = false;
  c->comm_rank = 0;
  c->comm_world = 0;
  dfree(c->comm_stage);
  c->comm_stage_bytes = 0;
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_comm_init(splatb200_ctx* c, const void* id128, int32_t rank, int32_t world) {
  NcclApi* a = nccl_api();
  if (!a) return c->fail(SPLATB200_ERUNTIME, "comm_init: libnccl.so.2 could not be bound at run time");
  if (!id128 || world < 1 || rank < 0 || rank >= world) return c->fail(SPLATB200_EINVAL, "comm_init: need 0 <= rank < world and an id");
  splatb200_ctx_comm_destroy(c);
  CU_TRY(c, cudaSetDevice(c->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclComm_t comm = nullptr;
  NCCL_TRY(c, a, a->CommInitRank(&comm, world, id, rank));
  c->comm = comm;
  c->owns_comm = true;
  c->comm_rank = rank;
  c->comm_world = world;
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_comm_bind(splatb200_ctx* c, void* nccl_comm, int32_t rank, int32_t world) {
  if (!nccl_api()) return c->fail(SPLATB200_ERUNTIME, "comm_bind: libnccl.so.2 could not be bound at run time");
  if (!nccl_comm || world < 1 || rank < 0 || rank >= world) return c->fail(SPLATB200_EINVAL, "comm_bind: need a communicator and 0 <= rank < world");
  splatb200_ctx_comm_destroy(c);
  c->comm = nccl_comm;
  c->owns_comm = false;
  c->comm_rank = rank;
  c->comm_world = world;
  return SPLATB200_OK;
}

extern "C" int splatb200_ctx_comm_info(const splatb200_ctx* c, int32_t* rank, int32_t* world) {
  if (rank) *rank = c->comm_rank;
  if (world) *world = c->comm ? c->comm_world : 0;
  return SPLATB200_OK;
}

// ActorGrad slots (host doubles) packed into one device buffer and summed over ranks with the same communicator
static int allreduce_actor_grads(splatb200_ctx* c, NcclApi* a) {
  const size_t na = c->tracks.size();
  if (na == 0) return SPLATB200_OK;
  for (auto* v : c->views) {
    int rc = finalize_actor_grads(v);
    if (rc) return rc;
  }
  if (c->actor_d_pose.size() != na) reset_actor_grads(c);
  std::vector<double> flat;
  for (size_t t = 0; t < na; ++t) {
    flat.insert(flat.end(), c->actor_d_pose[t].begin(), c->actor_d_pose[t].end());
    flat.insert(flat.end(), c->actor_d_vel[t].begin(), c->actor_d_vel[t].end());
  }
  if (c->comm_stage_bytes < flat.size() * sizeof(double)) {
    dfree(c->comm_stage);
    CU_TRY(c, cudaMalloc(&c->comm_stage, flat.size() * sizeof(double)));
    c->comm_stage_bytes = flat.size() * sizeof(double);
  }
  CU_TRY(c, cudaMemcpyAsync(c->comm_stage, flat.data(), flat.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, a, a->AllReduce(c->comm_stage, c->comm_stage, flat.size(), ncclDouble, ncclSum, (ncclComm_t)c->comm, c->stream));
  CU_TRY(c, cudaMemcpyAsync(flat.data(), c->comm_stage, flat.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  size_t o = 0;
  for (size_t t = 0; t < na; ++t) {
    std::copy(flat.begin() + o, flat.begin() + o + c->actor_d_pose[t].size(), c->actor_d_pose[t].begin());
    o += c->actor_d_pose[t].size();
    std::copy(flat.begin() + o, flat.begin() + o + 6, c->actor_d_vel[t].begin());
    o += 6;
  }
  return SPLATB200_OK;
}

extern "C" int splatb200_allreduce_grads(splatb200_ctx* c) {
  if (!c->comm) return c->fail(SPLATB200_ERUNTIME, "allreduce_grads without a communicator (splatb200_ctx_comm_init / _comm_bind)");
  NcclApi* a = nccl_api();
  if (!a) return c->fail(SPLATB200_ERUNTIME, "allreduce_grads: NCCL is not available");
  if (!c->grads) return c->fail(SPLATB200_ERUNTIME, "allreduce_grads without a scene");
  CU_TRY(c, cudaSetDevice(c->device));
  join_all(c);  // every view's backward (on its own stream) precedes the collective on the ctx stream
  if (c->grads_floats > 0)
    NCCL_TRY(c, a, a->AllReduce(c->grads, c->grads, (size_t)c->grads_floats, ncclFloat, ncclSum, (ncclComm_t)c->comm, c->stream));
  return allreduce_actor_grads(c, a);
}

extern "C" int splatb200_sharded_optimizer_step(splatb200_ctx* c, const splatb200_adam_config* cfg, int64_t step, int32_t skipped[6]) {
  if (!c->comm) return c->fail(SPLATB200_ERUNTIME, "sharded_optimizer_step without a communicator");
  NcclApi* a = nccl_api();
  if (!a) return c->fail(SPLATB200_ERUNTIME, "sharded_optimizer_step: NCCL is not available");
  if (!cfg || step < 0) return c->fail(SPLATB200_EINVAL, "optimizer_step: bad arguments");
  if (!c->mean || !c->grads) return c->fail(SPLATB200_ERUNTIME, "optimizer_step without a scene");
  CU_TRY(c, cudaSetDevice(c->device));
  join_all(c);
  const int world = c->comm_world, rank = c->comm_rank;
  const int64_t total = c->grads_floats;
  ncclComm_t comm = (ncclComm_t)c->comm;
  // (1) each shard is summed onto its owner (a reduce-scatter with ragged shards, one fused NCCL group)
  NCCL_TRY(c, a, a->GroupStart());
  for (int r = 0; r < world; ++r) {
    int64_t lo, hi;
    shard_of(total, world, r, lo, hi);
    if (hi > lo) NCCL_TRY(c, a, a->Reduce(c->grads + lo, c->grads + lo, (size_t)(hi - lo), ncclFloat, ncclSum, r, comm, c->stream));
  }
  NCCL_TRY(c, a, a->GroupEnd());
  // (2) groups to skip: a non-finite gradient in any shard skips the group on every rank
  int64_t lo, hi;
  shard_of(total, world, rank, lo, hi);
  int rc = ensure_adam_state(c);
  if (!rc) rc = flag_nonfinite(c, lo, hi);
  if (rc) return rc;
  NCCL_TRY(c, a, a->AllReduce(c->adam_bad, c->adam_bad, 6, ncclInt32, ncclMax, comm, c->stream));
  int h[6];
  CU_TRY(c, cudaMemcpyAsync(h, c->adam_bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  int32_t skip[6];
  for (int k = 0; k < 6; ++k) skip[k] = h[k] != 0;
  // (3) Adam on this rank's shard only
  rc = splatb200_optimizer_step_range(c, cfg, step, lo, hi, skip, skipped);
  if (rc) return rc;
  // (4) every owner broadcasts its updated slice of each parameter group (an all-gather with ragged shards)
  const AdamGroups gr = adam_groups(c);
  float* params[6] = {c->mean, c->scale_log, c->quat, c->opacity_logit, c->color, c->feature};
  NCCL_TRY(c, a, a->GroupStart());
  for (int r = 0; r < world; ++r) {
    int64_t rlo, rhi;
    shard_of(total, world, r, rlo, rhi);
    for (int k = 0; k < 6; ++k) {
      const int64_t b0 = std::max(gr.begin[k], rlo), b1 = std::min(gr.begin[k + 1], rhi);
      if (b1 <= b0) continue;
      float* ptr = params[k] + (b0 - gr.begin[k]);
      NCCL_TRY(c, a, a->Broadcast(ptr, ptr, (size_t)(b1 - b0), ncclFloat, r, comm, c->stream));
    }
  }
  NCCL_TRY(c, a, a->GroupEnd());
  if (skipped)
    for (int k = 0; k < 6; ++k) skipped[k] = skip[k];
  return SPLATB200_OK;
}

extern "C" int splatb200_scene_download(splatb200_ctx* c, float* mean, float* scale_log, float* quat, float* opacity_logit,
                                        float* color, float* feature) {
  if (!c->mean) return c->fail(SPLATB200_ERUNTIME, "no scene");
  join_all(c);
  wait_appearance(c);
  const size_t n = (size_t)c->n;
  float* dst[6] = {mean, scale_log, quat, opacity_logit, color, feature};
  const float* src[6] = {c->mean, c->scale_log, c->quat, c->opacity_logit, c->color, c->feature};
  const size_t width[6] = {3, 3, 4, 1, 3, (size_t)c->d_f};
  for (int k = 0; k < 6; ++k)
    if (dst[k] && n * width[k]) CU_TRY(c, cudaMemcpyAsync(dst[k], src[k], sizeof(float) * n * width[k], cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

// ---- lidar head ---------------------------------------------------------------------------
extern "C" int32_t splatb200_lidar_head_params(int32_t d_f) { return lidar_head_params(d_f); }

extern "C" int splatb200_view_set_lidar_head(splatb200_view* v, const float* weights) {
  splatb200_ctx* c = v->ctx;
  if (v->s.is_camera) return c->fail(SPLATB200_EINVAL, "the lidar head decodes a lidar view");
  join_view(v);
  if (!weights) {
    v->out.head_w = nullptr; v->out.head_y = nullptr;
    return SPLATB200_OK;
  }
  const int np = lidar_head_params(c->d_f);
  if (!v->d_head_w) CU_TRY(c, cudaMalloc(&v->d_head_w, sizeof(float) * 640));
  CU_TRY(c, cudaMemcpyAsync(v->d_head_w, weights, sizeof(float) * np, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  v->out.head_w = v->d_head_w;
  v->stage = std::min(v->stage, 2);
  return SPLATB200_OK;
}

extern "C" int splatb200_lidar_head_forward(splatb200_view* v, const float* weights, float* y) {
  splatb200_ctx* c = v->ctx;
  if (v->s.is_camera) return c->fail(SPLATB200_EINVAL, "the lidar head decodes a lidar view");
  if (!weights || !y) return c->fail(SPLATB200_EINVAL, "null argument");
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "lidar head before forward");
  join_view(v);
  const int np = lidar_head_params(c->d_f);
  DevScratch dw, dy;
  CU_TRY(c, cudaMalloc(&dw.p, sizeof(float) * np));
  CU_TRY(c, cudaMalloc(&dy.p, sizeof(float) * 2 * (size_t)std::max<int64_t>(1, v->P)));
  CU_TRY(c, cudaMemcpyAsync(dw.p, weights, sizeof(float) * np, cudaMemcpyHostToDevice, c->stream));
  launch_lidar_head_fwd(dw.p, c->d_f, v->P, v->rays, v->out.blend, dy.p, c->stream);
  CHECK_LAUNCH(c, "k_lidar_head_fwd");
  c->launches += v->P > 0;
  if (v->P) CU_TRY(c, cudaMemcpyAsync(y, dy.p, sizeof(float) * 2 * (size_t)v->P, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

extern "C" int splatb200_lidar_head_backward(splatb200_view* v, const float* weights, const float* g_y, float* g_weights,
                                             float* g_blend16) {
  splatb200_ctx* c = v->ctx;
  if (v->s.is_camera) return c->fail(SPLATB200_EINVAL, "the lidar head decodes a lidar view");
  if (!weights || !g_y || !g_weights || !g_blend16) return c->fail(SPLATB200_EINVAL, "null argument");
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "lidar head before forward");
  join_view(v);
  const int np = lidar_head_params(c->d_f);
  DevScratch dw, dgw, dgy;
  CU_TRY(c, cudaMalloc(&dw.p, sizeof(float) * np));
  CU_TRY(c, cudaMalloc(&dgw.p, sizeof(float) * np));
  CU_TRY(c, cudaMalloc(&dgy.p, sizeof(float) * 2 * (size_t)std::max<int64_t>(1, v->P)));
  CU_TRY(c, cudaMemcpyAsync(dw.p, weights, sizeof(float) * np, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(dgw.p, 0, sizeof(float) * np, c->stream));
  if (v->P) CU_TRY(c, cudaMemcpyAsync(dgy.p, g_y, sizeof(float) * 2 * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  launch_lidar_head_bwd(dw.p, c->d_f, v->P, v->rays, v->out.blend, dgy.p, g_blend16, dgw.p, c->stream);
  CHECK_LAUNCH(c, "k_lidar_head_bwd");
  c->launches += v->P > 0;
  CU_TRY(c, cudaMemcpyAsync(g_weights, dgw.p, sizeof(float) * np, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

// ---- camera ConvDecoder -------------------------------------------------------------------
extern "C" int32_t splatb200_conv_decoder_params(void) { return conv_decoder_params(); }

extern "C" int splatb200_ctx_set_decoder_precise(splatb200_ctx* c, int32_t on) {
  c->decoder_precise = on != 0;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_decode_image(splatb200_view* v, const float* params, const float* embedding, float* image,
                                           float* device_ms) {
  splatb200_ctx* c = v->ctx;
  if (!v->s.is_camera) return c->fail(SPLATB200_EINVAL, "decode_image decodes a camera view");
  if (!params || !embedding) return c->fail(SPLATB200_EINVAL, "null argument");
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "decode_image before forward");
  if (c->d_f + 11 > 32) return c->fail(SPLATB200_EINVAL, "decode_image: d_f + 3 + 8 input channels must fit the width of 32");
  if (v->s.width < 2 || v->s.height < 2) return c->fail(SPLATB200_EINVAL, "decode_image: reflect padding needs a 2 x 2 image");
  join_view(v);
  const int np = conv_decoder_params();
  const size_t P = (size_t)std::max<int64_t>(1, v->P);
  for (int k = 0; k < 6; ++k)
    if (!v->dec_act[k]) CU_TRY(c, cudaMalloc(&v->dec_act[k], sizeof(float) * 32 * P));
  if (!v->d_dec_image) CU_TRY(c, cudaMalloc(&v->d_dec_image, sizeof(float) * 3 * P));
  if (!v->d_dec_params) CU_TRY(c, cudaMalloc(&v->d_dec_params, sizeof(float) * (2 * 9248 + np + 8 + 2)));
  if (!v->d_dec_err) CU_TRY(c, cudaMalloc(&v->d_dec_err, sizeof(int)));
  float* d_emb = v->d_dec_params + ((np + 3) & ~3);
  CU_TRY(c, cudaMemcpyAsync(v->d_dec_params, params, sizeof(float) * np, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(d_emb, embedding, sizeof(float) * 8, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(v->d_dec_err, 0, sizeof(int), c->stream));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (device_ms) {
    CU_TRY(c, cudaEventCreate(&e0));
    CU_TRY(c, cudaEventCreate(&e1));
    CU_TRY(c, cudaEventRecord(e0, c->stream));
  }
  const int launched = launch_conv_decoder(v->d_dec_params, d_emb, v->s.height, v->s.width, c->d_f, v->s.fx, v->s.fy, v->s.cx,
                                           v->s.cy, v->out.blend, /*row pitch of the blend buffer*/ 16, v->dec_act, v->d_dec_image, v->d_dec_err,
                                           c->stream, c->decoder_precise);
  CHECK_LAUNCH(c, "k_conv3x3_tc");
  c->launches += launched;
  if (device_ms) CU_TRY(c, cudaEventRecord(e1, c->stream));
  int err = 0;
  CU_TRY(c, cudaMemcpyAsync(&err, v->d_dec_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (image && v->P) CU_TRY(c, cudaMemcpyAsync(image, v->d_dec_image, sizeof(float) * 3 * (size_t)v->P, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (device_ms) {
    CU_TRY(c, cudaEventElapsedTime(device_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (err) return c->fail(SPLATB200_ERUNTIME, "decode_image: tensor-core completion barrier timed out");
  v->dec_ready = true;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_decode_image_backward(splatb200_view* v, const float* g_image, float* g_params,
                                                    float* g_embedding, float* g_blend, float* device_ms) {
  splatb200_ctx* c = v->ctx;
  if (!v->s.is_camera) return c->fail(SPLATB200_EINVAL, "decode_image decodes a camera view");
  if (!g_image || !g_params || !g_embedding || !g_blend) return c->fail(SPLATB200_EINVAL, "null argument");
  if (!v->dec_ready || v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "decode_image backward without saved state");
  join_view(v);
  const int np = conv_decoder_params();
  const int H = v->s.height, W = v->s.width;
  const size_t P = (size_t)std::max<int64_t>(1, v->P);
  for (int k = 0; k < 3; ++k)
    if (!v->dec_g[k]) CU_TRY(c, cudaMalloc(&v->dec_g[k], sizeof(float) * 32 * P));
  if (!v->dec_gext) CU_TRY(c, cudaMalloc(&v->dec_gext, sizeof(float) * 32 * (size_t)(H + 2) * (W + 2)));
  if (!v->d_dec_gimage) CU_TRY(c, cudaMalloc(&v->d_dec_gimage, sizeof(float) * 3 * P));
  if (!v->d_dec_gparams) CU_TRY(c, cudaMalloc(&v->d_dec_gparams, sizeof(float) * (np + 8)));
  float* d_wt = v->d_dec_params + ((np + 3) & ~3) + 8;   // scratch behind the parameters and the embedding
  CU_TRY(c, cudaMemcpyAsync(v->d_dec_gimage, g_image, sizeof(float) * 3 * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(v->d_dec_gparams, 0, sizeof(float) * (np + 8), c->stream));
  CU_TRY(c, cudaMemsetAsync(v->d_dec_err, 0, sizeof(int), c->stream));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (device_ms) {
    CU_TRY(c, cudaEventCreate(&e0));
    CU_TRY(c, cudaEventCreate(&e1));
    CU_TRY(c, cudaEventRecord(e0, c->stream));
  }
  const int launched = launch_conv_decoder_backward(v->d_dec_params, H, W, c->d_f, v->out.blend, /*row pitch*/ 16, v->dec_act,
                                                    v->d_dec_gimage, v->dec_g, v->dec_gext, d_wt, v->d_dec_gparams,
                                                    v->d_dec_gparams + np, g_blend, v->d_dec_err, c->stream, c->decoder_precise);
  CHECK_LAUNCH(c, "conv decoder backward");
  c->launches += launched;
  if (device_ms) CU_TRY(c, cudaEventRecord(e1, c->stream));
  int err = 0;
  CU_TRY(c, cudaMemcpyAsync(&err, v->d_dec_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g_params, v->d_dec_gparams, sizeof(float) * np, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g_embedding, v->d_dec_gparams + np, sizeof(float) * 8, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (device_ms) {
    CU_TRY(c, cudaEventElapsedTime(device_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (err) return c->fail(SPLATB200_ERUNTIME, "decode_image backward: tensor-core completion barrier timed out");
  return SPLATB200_OK;
}

extern "C" int splatb200_debug_conv3x3_backward(splatb200_ctx* c, const float* x, int32_t H, int32_t W, const float* w,
                                                int32_t relu_in, const float* g_y, float* g_x, float* g_w) {
  if (!x || !w || !g_y || !g_x || !g_w || H < 2 || W < 2) return c->fail(SPLATB200_EINVAL, "bad argument");
  join_all(c);
  const size_t n = (size_t)H * W * 32, ne = (size_t)(H + 2) * (W + 2) * 32;
  DevScratch dx, dw, dwt, dgy, dgx, dgw, dge, de;
  CU_TRY(c, cudaMalloc(&dx.p, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&dgy.p, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&dgx.p, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&dge.p, sizeof(float) * ne));
  CU_TRY(c, cudaMalloc(&dw.p, sizeof(float) * 9248));
  CU_TRY(c, cudaMalloc(&dwt.p, sizeof(float) * 9248));
  CU_TRY(c, cudaMalloc(&dgw.p, sizeof(float) * 9248));
  CU_TRY(c, cudaMalloc(&de.p, sizeof(int)));
  CU_TRY(c, cudaMemcpyAsync(dx.p, x, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(dgy.p, g_y, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(dw.p, w, sizeof(float) * 9248, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(dgw.p, 0, sizeof(float) * 9248, c->stream));
  CU_TRY(c, cudaMemsetAsync(de.p, 0, sizeof(int), c->stream));
  launch_conv3x3_backward(dx.p, H, W, dw.p, relu_in, dgy.p, dwt.p, dge.p, dgx.p, dgw.p, (int*)de.p, c->stream, c->decoder_precise);
  CHECK_LAUNCH(c, "k_conv3x3_wgrad_tc");
  c->launches += 4;
  int err = 0;
  CU_TRY(c, cudaMemcpyAsync(&err, de.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g_x, dgx.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g_w, dgw.p, sizeof(float) * 9248, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (err) return c->fail(SPLATB200_ERUNTIME, "conv3x3 backward: tensor-core completion barrier timed out");
  return SPLATB200_OK;
}

extern "C" int splatb200_debug_conv3x3(splatb200_ctx* c, const float* x, int32_t H, int32_t W, const float* w, int32_t relu_in,
                                       const float* res, float* y) {
  if (!x || !w || !y || H < 2 || W < 2) return c->fail(SPLATB200_EINVAL, "bad argument");
  join_all(c);
  const size_t n = (size_t)H * W * 32;
  DevScratch dx, dw, dr, dy, de;
  CU_TRY(c, cudaMalloc(&dx.p, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&dy.p, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&dw.p, sizeof(float) * 9248));
  CU_TRY(c, cudaMalloc(&de.p, sizeof(int)));
  if (res) CU_TRY(c, cudaMalloc(&dr.p, sizeof(float) * n));
  CU_TRY(c, cudaMemcpyAsync(dx.p, x, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(dw.p, w, sizeof(float) * 9248, cudaMemcpyHostToDevice, c->stream));
  if (res) CU_TRY(c, cudaMemcpyAsync(dr.p, res, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(de.p, 0, sizeof(int), c->stream));
  CU_TRY(c, cudaMemsetAsync(dy.p, 0, sizeof(float) * n, c->stream));
  launch_conv3x3((const float*)dx.p, H, W, (const float*)dw.p, relu_in, (const float*)dr.p, (float*)dy.p, (int*)de.p, c->stream, c->decoder_precise);
  CHECK_LAUNCH(c, "k_conv3x3_tc");
  c->launches += 1;
  int err = 0;
  CU_TRY(c, cudaMemcpyAsync(&err, de.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaMemcpyAsync(y, dy.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (err) return c->fail(SPLATB200_ERUNTIME, "conv3x3: tensor-core completion barrier timed out");
  return SPLATB200_OK;
}

// ---- line-of-sight channel --------------------------------------------------------------------
extern "C" int splatb200_view_set_los(splatb200_view* v, const float* los_cut) {
  splatb200_ctx* c = v->ctx;
  if (v->s.is_camera) return c->fail(SPLATB200_EINVAL, "line of sight is a lidar channel");
  join_view(v);
  if (!los_cut) {
    v->out.los_cut = nullptr; v->out.los = nullptr; v->out.g_los = nullptr;
    return SPLATB200_OK;
  }
  const size_t cap = (size_t)std::max<int64_t>(1, std::max(v->P, v->P_cap));
  if (!v->d_los_cut) {
    CU_TRY(c, cudaMalloc(&v->d_los_cut, sizeof(float) * cap));
    CU_TRY(c, cudaMalloc(&v->d_los, sizeof(float) * cap));
    CU_TRY(c, cudaMalloc(&v->d_g_los, sizeof(float) * cap));
    CU_TRY(c, cudaMemsetAsync(v->d_g_los, 0, sizeof(float) * cap, c->stream));
  }
  if (v->P) CU_TRY(c, cudaMemcpyAsync(v->d_los_cut, los_cut, sizeof(float) * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemsetAsync(v->d_los, 0, sizeof(float) * cap, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));  // the host array is borrowed for the call only
  v->out.los_cut = v->d_los_cut; v->out.los = v->d_los; v->out.g_los = v->d_g_los;
  v->stage = std::min(v->stage, 2);  // the accumulator belongs to a forward with these cuts
  return SPLATB200_OK;
}

extern "C" int splatb200_view_set_los_grad(splatb200_view* v, const float* g_los) {
  splatb200_ctx* c = v->ctx;
  if (!v->out.los_cut) return c->fail(SPLATB200_ERUNTIME, "set_los_grad before set_los");
  if (!g_los) return c->fail(SPLATB200_EINVAL, "null gradient");
  join_view(v);
  if (v->P) CU_TRY(c, cudaMemcpyAsync(v->d_g_los, g_los, sizeof(float) * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

// A new sweep for an existing lidar view (the per-frame output of splatb200_assign_points): same tile grid, any number
// of rays. Buffers grow when the sweep is larger than any before.
extern "C" int splatb200_view_set_rays(splatb200_view* v, const float* rays, int64_t n_rays, const int64_t* ray_begin,
                                       const int64_t* ray_end, int64_t n_tiles) {
  splatb200_ctx* c = v->ctx;
  if (v->s.is_camera) return c->fail(SPLATB200_EINVAL, "view is not a lidar");
  if (n_rays < 0 || !ray_begin || !ray_end || n_tiles != v->n_tiles) return c->fail(SPLATB200_EINVAL, "set_rays: bad arguments");
  CU_TRY(c, cudaSetDevice(c->device));
  join_view(v);
  CU_TRY(c, cudaStreamSynchronize(c->stream));  // the previous sweep's kernels and copies are done with the buffers
  for (cudaStream_t q : {v->s_h2d, v->s_d2h})
    if (q) CU_TRY(c, cudaStreamSynchronize(q));
  v->dl_pending = false; v->band_dl_valid = false; v->bwd_recorded = false;
  if (n_rays > v->P_cap) {
    dfree(v->out.blend); dfree(v->out.alpha); dfree(v->out.t_final); dfree(v->out.range_blend); dfree(v->out.n_contrib);
    dfree(v->out.last_idx); dfree(v->g_blend_stage); dfree(v->g_alpha_stage); dfree(v->rays);
    dfree(v->d_los_cut); dfree(v->d_los); dfree(v->d_g_los); dfree(v->d_head_y);
    v->out.head_y = nullptr;
    const size_t cap = (size_t)(n_rays + n_rays / 8 + 256);
    CU_TRY(c, cudaMalloc(&v->out.blend, sizeof(float) * 16 * cap));
    CU_TRY(c, cudaMalloc(&v->out.alpha, sizeof(float) * cap));
    CU_TRY(c, cudaMalloc(&v->out.t_final, sizeof(float) * cap));
    CU_TRY(c, cudaMalloc(&v->out.range_blend, sizeof(float) * cap));
    CU_TRY(c, cudaMalloc(&v->out.n_contrib, sizeof(int32_t) * cap));
    CU_TRY(c, cudaMalloc(&v->out.last_idx, sizeof(int32_t) * cap));
    v->P_cap = (int64_t)cap;
  }
  v->stage = 0;
  v->bands.clear();
  v->out.los_cut = nullptr; v->out.los = nullptr; v->out.g_los = nullptr;  // cuts belong to a sweep: set them again
  return upload_rays(v, rays, n_rays, ray_begin, ray_end);
}

// compose_at_time's host part: actor validation (scene.hpp:297-298) and pose interpolation
// (scene.hpp:283-285), then the per-actor state upload.
static int prepare_actors(splatb200_view* v, float t_scene) {
  splatb200_ctx* c = v->ctx;
  const int na = (int)c->tracks.size();
  int rc = finalize_actor_grads(v);
  if (rc) return rc;
  v->poses.clear();
  try {
    for (const auto& tk : c->tracks) v->poses.push_back(sbh::interpolate_pose(tk, (double)t_scene));
  } catch (const std::runtime_error& e) {
    return c->fail(SPLATB200_ERUNTIME, e.what());
  }
  int bad = 0;
  int64_t bad_at = -1;
  for (const auto& kv : c->actor_first)
    if ((kv.first < 0 || kv.first > na) && (bad_at < 0 || kv.second < bad_at)) { bad = kv.first; bad_at = kv.second; }
  if (bad_at >= 0) return c->fail(SPLATB200_EOUTOFRANGE, "unknown actor_id " + std::to_string(bad));
  if (c->bound_max_actor > na) return c->fail(SPLATB200_EOUTOFRANGE, "unknown actor_id " + std::to_string(c->bound_max_actor));
  if (na == 0) return SPLATB200_OK;
  if (v->d_actors_cap < na) {
    dfree(v->d_actors);
    CU_TRY(c, cudaMalloc(&v->d_actors, sizeof(ActorState) * na));
    v->d_actors_cap = na;
  }
  if (v->actor_acc_cap < na) {
    dfree(v->actor_acc);
    CU_TRY(c, cudaMalloc(&v->actor_acc, sizeof(float) * kActorAccStride * na));
    CU_TRY(c, cudaMemsetAsync(v->actor_acc, 0, sizeof(float) * kActorAccStride * na, c->stream));
    v->actor_acc_cap = na;
  }
  std::vector<ActorState> st(na);
  for (int a = 0; a < na; ++a) {
    const auto& ip = v->poses[a];
    const auto& tk = c->tracks[a];
    for (int k = 0; k < 9; ++k) st[a].R[k] = (float)ip.R.a[k];
    for (int k = 0; k < 3; ++k) {
      st[a].t[k] = (float)ip.t.a[k];
      st[a].v[k] = (float)(tk.vel_lin[k] + tk.vel_offset[k]);      // scene.hpp:61
      st[a].w[k] = (float)(tk.vel_ang[k] + tk.vel_offset[3 + k]);  // scene.hpp:62
    }
  }
  // the previous frame's kernels may still read d_actors: order the overwrite after them
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (v->vs) CU_TRY(c, cudaStreamSynchronize(v->vs));
  CU_TRY(c, cudaMemcpy(v->d_actors, st.data(), sizeof(ActorState) * na, cudaMemcpyHostToDevice));
  return SPLATB200_OK;
}

extern "C" int splatb200_view_forward(splatb200_view* v, float t_scene, int32_t stop_after) {
  splatb200_ctx* c = v->ctx;
  CU_TRY(c, cudaSetDevice(c->device));
  if (!c->mean && c->n > 0) return c->fail(SPLATB200_EINVAL, "no scene uploaded");
  v->stage = 0;
  v->t_scene = t_scene;
  int rc = prepare_actors(v, t_scene);
  if (rc) return rc;
  rc = ensure_source_buffers(v);
  if (rc) return rc;
  v->s.d_f = c->d_f;
  v->s.channels = v->s.is_camera ? 3 + c->d_f : c->d_f;
  cudaStream_t st = work_stream(v);
  struct Busy { splatb200_view* v; cudaStream_t st; ~Busy() { mark_busy(v, st); } } busy_guard{v, st};
  const SceneDev sc = c->scene_dev(v->d_actors);
  CU_TRY(c, cudaMemsetAsync(v->sensor_grads, 0, sizeof(float) * 8, st));

  const bool late_app = c->app_pending;
  v->proj.skip_feat = late_app ? 1 : 0;
  {
    StageTimer tm(v, 0, st);
    launch_project(v->s, sc, v->proj, st);
  }
  CHECK_LAUNCH(c, "k_project");
  c->launches += c->n > 0;
  const int wrap_x = v->s.is_camera ? 0 : 1;
  const int sh = v->two_level ? super_shift() : 0;
  {
    // Per-tile list lengths straight from the tile rectangles (tile ranges, compositing CTA order, sort histograms).
    // (Independent of the depth sort; forking them onto a second stream was measured and gains nothing — both are
    // chains of small kernels and the fork/join events cost what the overlap saves. Overlap comes from running the
    // sensors of a frame on their own streams instead: splatb200_ctx_set_view_streams.)
    cudaStream_t ts = st;
    {
      StageTimer tm(v, 2, ts);
      c->launches += launch_tile_counts(c->n, v->proj, 0, v->s.tiles_x, v->s.tiles_y, wrap_x, v->tile_ws, v->tile_begin,
                                        v->tile_end, v->to_vals0, v->d_total, nullptr, ts, !v->two_level);
      v->tile_order = v->to_vals0;
      if (v->two_level)  // the same on the grid of 8 x 8-tile blocks: block ranges, list segments, sort histograms
        c->launches += launch_tile_counts(c->n, v->proj, sh, v->stiles_x, v->stiles_y, 0, v->tile_ws_c, v->super_begin,
                                          v->super_end, nullptr, v->d_total_c, v->seg_first, ts);
    }
    CHECK_LAUNCH(c, "k_tile_hist / k_tile_scan");
    {
      StageTimer tm(v, 1, st);
      // depth order of the Gaussians (stable: ties in ascending source index), then offsets in that order
      v->order_sel = 0;
      c->launches += launch_depth_sort_scan(v->proj.dkey, v->dkey_alt, v->order0, v->order1,
                                            v->two_level ? v->proj.ccount : v->proj.count, v->offsets, c->n, v->dsort_temp,
                                            v->dsort_temp_bytes, st);
    }
  }
  CHECK_LAUNCH(c, "depth sort + scan");
  for (int k = 1; k < 8; ++k) v->h_total[k] = 0;
  // look-back time-out flags (word 16 of each sort workspace): this frame's depth sort, the previous frame's tile sort
  // and expansion (their workspaces are only cleared when the next one is launched, after this sync)
  CU_TRY(c, cudaMemcpyAsync(v->h_total + 3, (const uint32_t*)v->dsort_temp + 16, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  if (v->sort_temp && v->I > 0) CU_TRY(c, cudaMemcpyAsync(v->h_total + 4, (const uint32_t*)v->sort_temp + 16, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  if (v->expand_temp && v->I > 0) CU_TRY(c, cudaMemcpyAsync(v->h_total + 5, (const uint32_t*)v->expand_temp + 16, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CU_TRY(c, cudaMemcpyAsync(v->h_total, v->d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CU_TRY(c, cudaMemcpyAsync(v->h_total + 1, v->offsets + c->n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  if (v->two_level) CU_TRY(c, cudaMemcpyAsync(v->h_total + 2, v->d_total_c, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CU_TRY(c, cudaStreamSynchronize(st));
  if (c->profiling) harvest_stage_events(v);  // previous step's events have all completed by now
  if (v->h_total[3] | v->h_total[4] | v->h_total[5])
    return c->fail(SPLATB200_ERUNTIME, "a decoupled look-back of the tile binning timed out (results of that render are invalid)");
  v->I = v->h_total[0];
  v->I_sort = v->two_level ? v->h_total[2] : v->I;
  v->stage = 1;
  if (stop_after == 1) return SPLATB200_OK;
  if (v->I >= (1LL << 30)) return c->fail(SPLATB200_ENOMEM, "2^30 or more intersections in one view");
  if ((int64_t)(uint32_t)v->h_total[1] != v->I_sort)
    return c->fail(SPLATB200_ERUNTIME, "tile histogram and count scan disagree on the number of intersections");
  rc = ensure_isect_capacity(v, v->I_sort, v->I);
  if (rc) return rc;

  v->sorted_sel = 0;
  if (v->I > 0) {
    StageTimer tm(v, 3, st);
    int nl = 0;
    if (!v->two_level) {
      v->sorted_sel = launch_tile_sort(c->n, v->I, v->offsets, v->order(), v->proj, 0, v->s.tiles_x, v->s.tiles_y, wrap_x,
                                       v->tile_ws, v->keys0, v->keys1, v->vals0, v->vals1, v->sort_temp, v->sort_temp_bytes, &nl, st);
    } else {
      v->sorted_sel = launch_tile_sort(c->n, v->I_sort, v->offsets, v->order(), v->proj, sh, v->stiles_x, v->stiles_y, 0,
                                       v->tile_ws_c, v->keys0, v->keys1, v->vals0, v->vals1, v->sort_temp, v->sort_temp_bytes, &nl, st);
      launch_expand(v->stiles_x, v->stiles_y, v->s.tiles_x, v->s.tiles_y, v->I_sort, v->super_begin, v->super_end, v->seg_first,
                    v->sorted_vals(), v->proj, v->tile_begin, v->expand_temp, v->vals_fine, st);
      ++nl;
    }
    CHECK_LAUNCH(c, "tile sort");
    c->launches += nl;
  }
  v->stage = 2;
  if (stop_after == 2) return SPLATB200_OK;

  if (v->dl_pending) {  // an overlapped download of the previous render still reads the output buffers
    CU_TRY(c, cudaStreamWaitEvent(st, v->ev_dl, 0));
    v->dl_pending = false;
  }
  if (late_app) {  // colour / features are needed from here on
    CU_TRY(c, cudaStreamWaitEvent(st, c->ev_app, 0));
    launch_pack_feat(v->s, sc, v->proj, st);
    CHECK_LAUNCH(c, "k_pack_feat");
    c->launches += c->n > 0;
  }
  v->out.hit_or = v->multi_pass ? 1 : 0;
  // hit bytes are OR-ed into: by the shared lidar kernel over several ray passes, by the lidar kernel pair one warp at a time
  if ((v->multi_pass || v->lidar_v2()) && v->I > 0) CU_TRY(c, cudaMemsetAsync(v->out.hit, 0, (size_t)v->I, st));
  if (v->out.head_w && !v->d_head_y)
    CU_TRY(c, cudaMalloc(&v->d_head_y, sizeof(float) * 2 * (size_t)std::max<int64_t>(1, std::max(v->P, v->P_cap))));
  v->out.head_y = v->out.head_w ? v->d_head_y : nullptr;
  v->band_dl_valid = false;
  if (!v->plan_fwd) {
    StageTimer tm(v, 5, st);
    if (v->lidar_v2())
      launch_raster_fwd_lidar(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end,
                              v->tile_order, v->out, st);
    else
      launch_raster_fwd(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, v->tile_order,
                        v->out, st);
    CHECK_LAUNCH(c, "k_raster_fwd");
    c->launches += 1;
  } else {
    // forward_to_host: band by band, each band's outputs leave on the view's device-to-host stream while the next band
    // is being composited
    v->plan_fwd = false;
    StageTimer tm(v, 5, st);
    for (size_t b = 0; b < v->bands.size(); ++b) {
      const auto& bd = v->bands[b];
      if (v->lidar_v2())
        launch_raster_fwd_lidar(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, nullptr,
                                v->out, st, bd.tile_first, bd.tile_count);
      else
        launch_raster_fwd(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, nullptr, v->out,
                          st, bd.tile_first, bd.tile_count);
      CHECK_LAUNCH(c, "k_raster_fwd (band)");
      c->launches += 1;
      CU_TRY(c, cudaEventRecord(v->ev_bfwd[b], st));
      CU_TRY(c, cudaStreamWaitEvent(v->s_d2h, v->ev_bfwd[b], 0));
      if (b >= 1 && !getenv("SPLATB200_NO_YIELD")) {  // small transfers first (splatb200_ctx::yield_dl)
        cudaEvent_t e = nullptr;
        {
          std::lock_guard<std::mutex> lk(c->xfer_mu);
          e = c->yield_dl;
          c->yield_dl = nullptr;
        }
        if (e) CU_TRY(c, cudaStreamWaitEvent(v->s_d2h, e, 0));
      }
      const size_t q0 = (size_t)bd.q0, nq = (size_t)(bd.q1 - bd.q0);
      if (nq) {
        if (v->plan_blend) CU_TRY(c, cudaMemcpyAsync(v->plan_blend + 16 * q0, v->out.blend + 16 * q0, sizeof(float) * 16 * nq, cudaMemcpyDeviceToHost, v->s_d2h));
        if (v->plan_alpha) CU_TRY(c, cudaMemcpyAsync(v->plan_alpha + q0, v->out.alpha + q0, sizeof(float) * nq, cudaMemcpyDeviceToHost, v->s_d2h));
        if (v->plan_ncontrib) CU_TRY(c, cudaMemcpyAsync(v->plan_ncontrib + q0, v->out.n_contrib + q0, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, v->s_d2h));
      }
      CU_TRY(c, cudaEventRecord(v->ev_bdl[b], v->s_d2h));
    }
    CU_TRY(c, cudaEventRecord(v->ev_dl, v->s_d2h));
    if (v->bands.size() == 1) {
      std::lock_guard<std::mutex> lk(c->xfer_mu);
      c->yield_dl = v->ev_dl;
    }
    v->dl_pending = true;
    v->band_dl_valid = true;
  }
  v->stage = 3;
  v->dec_ready = false;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_stats_get(splatb200_view* v, splatb200_view_stats* out) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "stats before forward");
  std::vector<uint32_t> cnt((size_t)c->n);
  if (c->n) CU_TRY(c, cudaMemcpyAsync(cnt.data(), v->proj.count, sizeof(uint32_t) * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  int64_t vis = 0;
  for (uint32_t x : cnt) vis += x != 0;
  out->n_gaussians = c->n;
  out->n_visible = vis;
  out->n_intersections = v->I;
  out->n_queries = v->P;
  out->tiles_x = v->s.tiles_x;
  out->tiles_y = v->s.tiles_y;
  return SPLATB200_OK;
}

extern "C" const float* splatb200_view_blend(splatb200_view* v) { return v->out.blend; }
extern "C" const float* splatb200_view_alpha(splatb200_view* v) { return v->out.alpha; }
extern "C" const int32_t* splatb200_view_n_contrib(splatb200_view* v) { return v->out.n_contrib; }

extern "C" int splatb200_view_backward(splatb200_view* v, const float* g_blend16, const float* g_alpha) {
  splatb200_ctx* c = v->ctx;
  CU_TRY(c, cudaSetDevice(c->device));
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  if (!g_blend16 || !g_alpha) return c->fail(SPLATB200_EINVAL, "null upstream gradient");
  cudaStream_t st = work_stream(v);
  struct Busy { splatb200_view* v; cudaStream_t st; ~Busy() { mark_busy(v, st); } } busy_guard{v, st};
  if (v->wait_up) {  // overlapped upload of the upstream gradients (backward_host_overlapped)
    CU_TRY(c, cudaStreamWaitEvent(st, v->ev_up, 0));
    v->wait_up = false;
  }
  RasterGradDev rg{v->rg};
  const ParamGradDev pg = c->pg();
  if (v->plan_bwd) {
    // backward_from_host: a band's upstream gradients are uploaded after that band's outputs have been downloaded (they
    // are a function of them) and its backward kernel starts as soon as they have arrived
    v->plan_bwd = false;
    StageTimer tm(v, 6, st);
    if (v->bwd_recorded) CU_TRY(c, cudaStreamWaitEvent(v->s_h2d, v->ev_bwd, 0));  // staging buffers still in use
    for (size_t b = 0; b < v->bands.size(); ++b) {
      const auto& bd = v->bands[b];
      const size_t q0 = (size_t)bd.q0, nq = (size_t)(bd.q1 - bd.q0);
      if (v->band_dl_valid) CU_TRY(c, cudaStreamWaitEvent(v->s_h2d, v->ev_bdl[b], 0));
      if (b >= 1 && !getenv("SPLATB200_NO_YIELD")) {  // small transfers first (splatb200_ctx::yield_ul)
        cudaEvent_t e = nullptr;
        {
          std::lock_guard<std::mutex> lk(c->xfer_mu);
          e = c->yield_ul;
          c->yield_ul = nullptr;
        }
        if (e) CU_TRY(c, cudaStreamWaitEvent(v->s_h2d, e, 0));
      }
      if (nq) {
        CU_TRY(c, cudaMemcpyAsync(v->g_blend_stage + 16 * q0, v->plan_gb + 16 * q0, sizeof(float) * 16 * nq, cudaMemcpyHostToDevice, v->s_h2d));
        CU_TRY(c, cudaMemcpyAsync(v->g_alpha_stage + q0, v->plan_ga + q0, sizeof(float) * nq, cudaMemcpyHostToDevice, v->s_h2d));
      }
      CU_TRY(c, cudaEventRecord(v->ev_bup[b], v->s_h2d));
      if (v->bands.size() == 1) {
        std::lock_guard<std::mutex> lk(c->xfer_mu);
        c->yield_ul = v->ev_bup[b];
      }
    }
    for (size_t b = 0; b < v->bands.size(); ++b) {
      const auto& bd = v->bands[b];
      CU_TRY(c, cudaStreamWaitEvent(st, v->ev_bup[b], 0));
      if (v->I > 0) {
        if (v->lidar_v2())
          launch_raster_bwd_lidar(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, nullptr,
                                  v->out, g_blend16, g_alpha, rg, pg, st, bd.tile_first, bd.tile_count);
        else
          launch_raster_bwd(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, nullptr, v->out,
                            g_blend16, g_alpha, rg, pg, v->sensor_grads + 6, st, bd.tile_first, bd.tile_count);
        CHECK_LAUNCH(c, "k_raster_bwd (band)");
        c->launches += 1;
      }
    }
  } else if (v->I > 0) {
    StageTimer tm(v, 6, st);
    if (v->lidar_v2())
      launch_raster_bwd_lidar(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end,
                              v->tile_order, v->out, g_blend16, g_alpha, rg, pg, st);
    else
      launch_raster_bwd(v->s, v->proj, v->vals(), v->tile_begin, v->tile_end, v->rays, v->ray_begin, v->ray_end, v->tile_order,
                        v->out, g_blend16, g_alpha, rg, pg, v->sensor_grads + 6, st);
    CHECK_LAUNCH(c, "k_raster_bwd");
    c->launches += 1;
  }
  {
    StageTimer tm(v, 7, st);
    launch_project_bwd(v->s, c->scene_dev(v->d_actors), v->proj, rg, pg, v->sensor_grads, v->actor_acc, st);
  }
  CHECK_LAUNCH(c, "k_project_bwd");
  c->launches += c->n > 0;
  if (!c->tracks.empty()) v->actor_pending = true;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_sensor_grads(splatb200_view* v, splatb200_sensor_grads* out) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  float h[8];
  CU_TRY(c, cudaMemcpyAsync(h, v->sensor_grads, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 3; ++k) { out->d_vel_lin[k] = h[k]; out->d_vel_ang[k] = h[3 + k]; }
  out->d_time_offset = h[6];
  return SPLATB200_OK;
}

extern "C" int splatb200_view_download(splatb200_view* v, float* blend16, float* alpha, int32_t* n_contrib) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "download before forward");
  const size_t P = (size_t)v->P;
  if (blend16 && P) CU_TRY(c, cudaMemcpyAsync(blend16, v->out.blend, sizeof(float) * 16 * P, cudaMemcpyDeviceToHost, c->stream));
  if (alpha && P) CU_TRY(c, cudaMemcpyAsync(alpha, v->out.alpha, sizeof(float) * P, cudaMemcpyDeviceToHost, c->stream));
  if (n_contrib && P) CU_TRY(c, cudaMemcpyAsync(n_contrib, v->out.n_contrib, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

extern "C" int splatb200_view_backward_host(splatb200_view* v, const float* g_blend16, const float* g_alpha) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  if (!g_blend16 || !g_alpha) return c->fail(SPLATB200_EINVAL, "null upstream gradient");
  const size_t P = (size_t)std::max<int64_t>(1, std::max(v->P, v->P_cap));  // lidar sweeps change size (view_set_rays)
  if (!v->g_blend_stage) {
    CU_TRY(c, cudaMalloc(&v->g_blend_stage, sizeof(float) * 16 * P));
    CU_TRY(c, cudaMalloc(&v->g_alpha_stage, sizeof(float) * P));
  }
  CU_TRY(c, cudaMemcpyAsync(v->g_blend_stage, g_blend16, sizeof(float) * 16 * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(v->g_alpha_stage, g_alpha, sizeof(float) * (size_t)v->P, cudaMemcpyHostToDevice, c->stream));
  return splatb200_view_backward(v, v->g_blend_stage, v->g_alpha_stage);
}

namespace {
int ensure_copy_events(splatb200_view* v) {
  splatb200_ctx* c = v->ctx;
  for (cudaEvent_t* e : {&v->ev_fwd, &v->ev_dl, &v->ev_up, &v->ev_bwd})
    if (!*e) CU_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaStream_t* q : {&v->s_h2d, &v->s_d2h})
    if (!*q) CU_TRY(c, cudaStreamCreateWithFlags(q, cudaStreamNonBlocking));
  return SPLATB200_OK;
}
}  // namespace

extern "C" int splatb200_view_download_async(splatb200_view* v, float* blend16, float* alpha, int32_t* n_contrib) {
  splatb200_ctx* c = v->ctx;
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "download before forward");
  int rc = ensure_copy_events(v);
  if (rc) return rc;
  const size_t P = (size_t)v->P;
  if (v->busy) {  // the forward ran on the view's own stream
    CU_TRY(c, cudaStreamWaitEvent(v->s_d2h, v->ev_last, 0));
  } else {
    CU_TRY(c, cudaEventRecord(v->ev_fwd, c->stream));
    CU_TRY(c, cudaStreamWaitEvent(v->s_d2h, v->ev_fwd, 0));
  }
  if (blend16 && P) CU_TRY(c, cudaMemcpyAsync(blend16, v->out.blend, sizeof(float) * 16 * P, cudaMemcpyDeviceToHost, v->s_d2h));
  if (alpha && P) CU_TRY(c, cudaMemcpyAsync(alpha, v->out.alpha, sizeof(float) * P, cudaMemcpyDeviceToHost, v->s_d2h));
  if (n_contrib && P) CU_TRY(c, cudaMemcpyAsync(n_contrib, v->out.n_contrib, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, v->s_d2h));
  CU_TRY(c, cudaEventRecord(v->ev_dl, v->s_d2h));
  v->dl_pending = true;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_backward_host_overlapped(splatb200_view* v, const float* g_blend16, const float* g_alpha) {
  splatb200_ctx* c = v->ctx;
  if (!g_blend16 || !g_alpha) return c->fail(SPLATB200_EINVAL, "null upstream gradient");
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  int rc = ensure_copy_events(v);
  if (rc) return rc;
  const size_t P = (size_t)std::max<int64_t>(1, std::max(v->P, v->P_cap));  // lidar sweeps change size (view_set_rays)
  if (!v->g_blend_stage) {
    CU_TRY(c, cudaMalloc(&v->g_blend_stage, sizeof(float) * 16 * P));
    CU_TRY(c, cudaMalloc(&v->g_alpha_stage, sizeof(float) * P));
  }
  // the upstream gradients are a function of the rendered outputs: their upload follows this view's download;
  // the staging buffers may still be read by this view's previous backward
  if (v->dl_pending) CU_TRY(c, cudaStreamWaitEvent(v->s_h2d, v->ev_dl, 0));
  if (v->bwd_recorded) CU_TRY(c, cudaStreamWaitEvent(v->s_h2d, v->ev_bwd, 0));
  CU_TRY(c, cudaMemcpyAsync(v->g_blend_stage, g_blend16, sizeof(float) * 16 * (size_t)v->P, cudaMemcpyHostToDevice, v->s_h2d));
  CU_TRY(c, cudaMemcpyAsync(v->g_alpha_stage, g_alpha, sizeof(float) * (size_t)v->P, cudaMemcpyHostToDevice, v->s_h2d));
  CU_TRY(c, cudaEventRecord(v->ev_up, v->s_h2d));
  v->wait_up = true;
  rc = splatb200_view_backward(v, v->g_blend_stage, v->g_alpha_stage);
  if (rc) return rc;
  CU_TRY(c, cudaEventRecord(v->ev_bwd, (c->view_streams && v->vs) ? v->vs : c->stream));
  v->bwd_recorded = true;
  return SPLATB200_OK;
}

// ---- fused host-buffer calls with banded, overlapped transfers ------------------------------------------------
namespace {
int make_bands(splatb200_view* v, int nb) {
  splatb200_ctx* c = v->ctx;
  int rc = ensure_copy_events(v);
  if (rc) return rc;
  if (nb <= 0) nb = v->s.is_camera ? 8 : 1;  // measured on the north-star frame: 2 bands 11.5 ms, 4 bands 10.6 ms, 8 bands 10.1 ms
  nb = std::min(nb, 8);
  v->bands.clear();
  if (v->s.is_camera) {
    const int rows = v->s.tiles_y, per = (rows + nb - 1) / nb;
    for (int r0 = 0; r0 < rows; r0 += per) {
      const int r1 = std::min(rows, r0 + per);
      const int64_t y0 = std::min<int64_t>(v->s.height, (int64_t)kTile * r0), y1 = std::min<int64_t>(v->s.height, (int64_t)kTile * r1);
      v->bands.push_back({r0 * v->s.tiles_x, (r1 - r0) * v->s.tiles_x, y0 * v->s.width, y1 * v->s.width});
    }
  } else {  // a lidar sweep is small (18 MB of outputs): one band
    v->bands.push_back({0, (int)v->n_tiles, 0, v->P});
  }
  for (size_t b = 0; b < v->bands.size(); ++b)
    for (cudaEvent_t* e : {&v->ev_bfwd[b], &v->ev_bdl[b], &v->ev_bup[b]})
      if (!*e) CU_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return SPLATB200_OK;
}
}  // namespace

extern "C" int splatb200_view_forward_to_host(splatb200_view* v, float t_scene, float* blend16, float* alpha, int32_t* n_contrib,
                                              int32_t bands) {
  int rc = make_bands(v, bands);
  if (rc) return rc;
  v->plan_blend = blend16; v->plan_alpha = alpha; v->plan_ncontrib = n_contrib;
  v->plan_fwd = true;
  rc = splatb200_view_forward(v, t_scene, 0);
  v->plan_fwd = false;
  return rc;
}

extern "C" int splatb200_view_backward_from_host(splatb200_view* v, const float* g_blend16, const float* g_alpha) {
  splatb200_ctx* c = v->ctx;
  if (!g_blend16 || !g_alpha) return c->fail(SPLATB200_EINVAL, "null upstream gradient");
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  if (v->bands.empty()) {
    int rc = make_bands(v, 0);
    if (rc) return rc;
  }
  const size_t P = (size_t)std::max<int64_t>(1, std::max(v->P, v->P_cap));  // lidar sweeps change size (view_set_rays)
  if (!v->g_blend_stage) {
    CU_TRY(c, cudaMalloc(&v->g_blend_stage, sizeof(float) * 16 * P));
    CU_TRY(c, cudaMalloc(&v->g_alpha_stage, sizeof(float) * P));
  }
  v->plan_gb = g_blend16; v->plan_ga = g_alpha;
  v->plan_bwd = true;
  int rc = splatb200_view_backward(v, v->g_blend_stage, v->g_alpha_stage);
  v->plan_bwd = false;
  if (rc) return rc;
  CU_TRY(c, cudaEventRecord(v->ev_bwd, (c->view_streams && v->vs) ? v->vs : c->stream));
  v->bwd_recorded = true;
  return SPLATB200_OK;
}

// ---- assign_points_to_tiles -----------------------------------------------------------------
// Device: per-point geometry + tile key (k_assign_points), stable radix sort by tile (and by shuffle hash first in
// training mode); host: the per-tile slices and the 256-point cap of the training mode (O(n) over the sorted keys).
extern "C" int splatb200_assign_points(splatb200_ctx* c, const splatb200_lidar* l, int64_t n, const float* points_xyz,
                                       const float* timestamps, int32_t train, uint32_t seed, int64_t* tile, float* sph,
                                       int64_t* order, int64_t* ray_begin, int64_t* ray_end, int64_t* counts) {
  if (!l || n < 0 || (n > 0 && (!points_xyz || !timestamps)) || !ray_begin || !ray_end || !counts)
    return c->fail(SPLATB200_EINVAL, "assign_points: null argument");
  if (l->n_beams < 1 || !(l->azimuth_resolution > 0.0f)) return c->fail(SPLATB200_EINVAL, "lidar needs beams and res_phi > 0");
  if (n >= (1LL << 30)) return c->fail(SPLATB200_EINVAL, "assign_points: too many points");
  CU_TRY(c, cudaSetDevice(c->device));
  int m_phi, m_omega;
  lidar_grid_of(l->azimuth_resolution, l->n_beams, &m_phi, &m_omega);
  if (m_omega - 1 > kMaxBoundaries) return c->fail(SPLATB200_EINVAL, "too many beams");
  const int64_t T = (int64_t)m_phi * m_omega;
  Sensor s;
  std::memset(&s, 0, sizeof(Sensor));
  fill_pose(s, l->R, l->t, l->vel_lin, l->vel_ang);
  s.tiles_x = m_phi; s.tiles_y = m_omega;
  s.span = (float)kNphi * l->azimuth_resolution;
  s.n_boundaries = m_omega - 1;
  for (int k = 1; k < m_omega; ++k)
    s.boundaries[k - 1] = 0.5f * (l->elevation_channels[kNomega * k - 1] + l->elevation_channels[kNomega * k]);
  for (int64_t t = 0; t < T; ++t) ray_begin[t] = ray_end[t] = 0;
  counts[0] = counts[1] = counts[2] = 0;
  if (n == 0) return SPLATB200_OK;

  const size_t m = (size_t)n;
  float *d_xyz = nullptr, *d_ts = nullptr;
  float4* d_sph = nullptr;
  uint32_t *d_key = nullptr, *d_hash = nullptr, *d_valid = nullptr, *k0 = nullptr, *k1 = nullptr, *o0 = nullptr, *o1 = nullptr,
           *oh = nullptr, *off = nullptr;
  void* temp = nullptr;
  const size_t temp_bytes = depth_sort_temp_bytes(n);
  auto fin = [&](int rc) {
    cudaFree(d_xyz); cudaFree(d_ts); cudaFree(d_sph); cudaFree(d_key); cudaFree(d_hash); cudaFree(d_valid); cudaFree(k0);
    cudaFree(k1); cudaFree(o0); cudaFree(o1); cudaFree(oh); cudaFree(off); cudaFree(temp);
    return rc;
  };
  if (cudaMalloc(&d_xyz, 12 * m) || cudaMalloc(&d_ts, 4 * m) || cudaMalloc(&d_sph, 16 * m) || cudaMalloc(&d_key, 4 * m) ||
      cudaMalloc(&d_hash, 4 * m) || cudaMalloc(&d_valid, 4 * m) || cudaMalloc(&k0, 4 * m) || cudaMalloc(&k1, 4 * m) ||
      cudaMalloc(&o0, 4 * m) || cudaMalloc(&o1, 4 * m) || cudaMalloc(&oh, 4 * m) || cudaMalloc(&off, 4 * (m + 1)) ||
      cudaMalloc(&temp, temp_bytes))
    return fin(c->fail(SPLATB200_ENOMEM, "assign_points: out of device memory"));
  cudaStream_t st = c->stream;
  cudaMemcpyAsync(d_xyz, points_xyz, 12 * m, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_ts, timestamps, 4 * m, cudaMemcpyHostToDevice, st);
  launch_assign_points(s, l->timestamp, n, d_xyz, d_ts, seed, d_key, d_sph, d_hash, d_valid, st);
  c->launches += 1;
  const uint32_t* final_order = o0;
  if (!train) {
    cudaMemcpyAsync(k0, d_key, 4 * m, cudaMemcpyDeviceToDevice, st);
    c->launches += launch_depth_sort_scan(k0, k1, o0, o1, d_valid, off, n, temp, temp_bytes, st);
  } else {  // LSD: by hash first, then (stably) by tile
    cudaMemcpyAsync(k0, d_hash, 4 * m, cudaMemcpyDeviceToDevice, st);
    c->launches += launch_depth_sort_scan(k0, k1, oh, o1, d_valid, off, n, temp, temp_bytes, st);
    launch_gather_u32(n, d_key, oh, k0, st);                       // keys in hash order
    c->launches += 1 + launch_depth_sort_scan(k0, k1, o0, o1, d_valid, off, n, temp, temp_bytes, st);
    launch_gather_u32(n, oh, o0, o1, st);                          // compose the two permutations
    c->launches += 1;
    final_order = o1;
  }
  std::vector<uint32_t> h_key(m), h_order(m);
  std::vector<float4> h_sph(m);
  cudaMemcpyAsync(h_key.data(), d_key, 4 * m, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_order.data(), final_order, 4 * m, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_sph.data(), d_sph, 16 * m, cudaMemcpyDeviceToHost, st);
  uint32_t err = 0;
  cudaMemcpyAsync(&err, (const uint32_t*)temp + 16, 4, cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fin(c->fail(SPLATB200_ECUDA, cudaGetErrorString(e)));
  if (err) return fin(c->fail(SPLATB200_ERUNTIME, "assign_points: look-back timed out"));
  int64_t kept = 0, rejected = 0, dropped = 0;
  for (size_t i = 0; i < m; ++i) {
    if (tile) tile[i] = h_key[i] == 0xffffffffu ? -1 : (int64_t)h_key[i];
    if (sph) { sph[4 * i] = h_sph[i].x; sph[4 * i + 1] = h_sph[i].y; sph[4 * i + 2] = h_sph[i].z; sph[4 * i + 3] = h_sph[i].w; }
    rejected += h_key[i] == 0xffffffffu;
  }
  // per-tile slices of the sorted order; training mode keeps the first 256 of a tile (smallest hashes)
  size_t k = 0;
  while (k < m) {
    const uint32_t t = h_key[h_order[k]];
    if (t == 0xffffffffu) break;  // rejected points sort last
    size_t e2 = k;
    while (e2 < m && h_key[h_order[e2]] == t) ++e2;
    size_t take = e2 - k;
    if (train && take > (size_t)(kNphi * kNomega)) { dropped += (int64_t)take - kNphi * kNomega; take = (size_t)(kNphi * kNomega); }
    ray_begin[t] = kept;
    for (size_t q = 0; q < take; ++q) {
      if (order) order[kept] = h_order[k + q];
      ++kept;
    }
    ray_end[t] = kept;
    k = e2;
  }
  counts[0] = kept; counts[1] = rejected; counts[2] = dropped;
  return fin(SPLATB200_OK);
}

// ---- test hook: the depth sort + count scan on caller data ----------------------------------------------
extern "C" int splatb200_debug_depth_sort(splatb200_ctx* c, int64_t n, const uint32_t* keys, const uint32_t* counts,
                                          uint32_t* order_out, uint32_t* offsets_out) {
  if (n < 0 || (n > 0 && (!keys || !counts))) return c->fail(SPLATB200_EINVAL, "debug_depth_sort: bad arguments");
  CU_TRY(c, cudaSetDevice(c->device));
  const size_t m = (size_t)std::max<int64_t>(1, n);
  uint32_t *k0 = nullptr, *k1 = nullptr, *o0 = nullptr, *o1 = nullptr, *cnt = nullptr, *off = nullptr;
  void* temp = nullptr;
  const size_t temp_bytes = depth_sort_temp_bytes(n);
  auto fin = [&](int rc) {
    cudaFree(k0); cudaFree(k1); cudaFree(o0); cudaFree(o1); cudaFree(cnt); cudaFree(off); cudaFree(temp);
    return rc;
  };
  if (cudaMalloc(&k0, 4 * m) || cudaMalloc(&k1, 4 * m) || cudaMalloc(&o0, 4 * m) || cudaMalloc(&o1, 4 * m) ||
      cudaMalloc(&cnt, 4 * m) || cudaMalloc(&off, 4 * (m + 1)) || cudaMalloc(&temp, temp_bytes))
    return fin(c->fail(SPLATB200_ENOMEM, "debug_depth_sort: out of device memory"));
  if (n) {
    cudaMemcpyAsync(k0, keys, 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(cnt, counts, 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream);
  }
  launch_depth_sort_scan(k0, k1, o0, o1, cnt, off, n, temp, temp_bytes, c->stream);
  if (n && order_out) cudaMemcpyAsync(order_out, o0, 4 * (size_t)n, cudaMemcpyDeviceToHost, c->stream);
  if (offsets_out) cudaMemcpyAsync(offsets_out, off, 4 * (size_t)(n + 1), cudaMemcpyDeviceToHost, c->stream);
  uint32_t err = 0;
  if (n) cudaMemcpyAsync(&err, (const uint32_t*)temp + 16, 4, cudaMemcpyDeviceToHost, c->stream);
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return fin(c->fail(SPLATB200_ECUDA, cudaGetErrorString(e)));
  if (err) return fin(c->fail(SPLATB200_ERUNTIME, "debug_depth_sort: look-back timed out"));
  return fin(SPLATB200_OK);
}

// ---- reference-granularity entry points ------------------------------------------------------------
// The functions the reference ships as code, one call each, HOST buffers in and out. Not the hot path
// (the fused forward/backward above is); these exist so that a caller written against
// splat/scene.hpp + splat/projection.hpp can switch function by function (include/splat_b200.hpp).
namespace {

int visible_list(splatb200_view* v, std::vector<int64_t>& vis) {
  splatb200_ctx* c = v->ctx;
  std::vector<uint32_t> cnt((size_t)c->n);
  if (c->n) CU_TRY(c, cudaMemcpyAsync(cnt.data(), v->proj.count, sizeof(uint32_t) * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  vis.clear();
  for (size_t i = 0; i < cnt.size(); ++i)
    if (cnt[i]) vis.push_back((int64_t)i);
  return SPLATB200_OK;
}

int run_dump(splatb200_view* v, std::vector<float>& h) {
  splatb200_ctx* c = v->ctx;
  const size_t N = (size_t)c->n;
  DevScratch d;
  CU_TRY(c, cudaMalloc(&d.p, sizeof(float) * kDumpStride * std::max<size_t>(1, N)));
  CU_TRY(c, cudaMemsetAsync(d.p, 0, sizeof(float) * kDumpStride * N, c->stream));
  launch_project_dump(v->s, c->scene_dev(v->d_actors), d.p, c->stream);
  CHECK_LAUNCH(c, "k_project_dump");
  h.resize((size_t)kDumpStride * N);
  if (N) CU_TRY(c, cudaMemcpyAsync(h.data(), d.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}

}  // namespace

extern "C" int splatb200_view_composed(splatb200_view* v, float* mean_w, float* cov_w, float* vel_dyn_w, float* opacity) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "view_composed before forward");
  std::vector<float> h;
  int rc = run_dump(v, h);
  if (rc) return rc;
  for (int64_t i = 0; i < c->n; ++i) {
    const float* o = &h[(size_t)kDumpStride * i];
    if (opacity) opacity[i] = o[26];
    for (int k = 0; k < 3; ++k) {
      if (mean_w) mean_w[3 * i + k] = o[27 + k];
      if (vel_dyn_w) vel_dyn_w[3 * i + k] = o[30 + k];
    }
    if (cov_w) for (int k = 0; k < 9; ++k) cov_w[9 * i + k] = o[33 + k];
  }
  return SPLATB200_OK;
}

extern "C" int64_t splatb200_view_projected(splatb200_view* v, int64_t* source_index, float* fields25) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "view_projected before forward");
  std::vector<int64_t> vis;
  int rc = visible_list(v, vis);
  if (rc) return rc;
  if (source_index) std::memcpy(source_index, vis.data(), sizeof(int64_t) * vis.size());
  if (fields25) {
    std::vector<float> h;
    rc = run_dump(v, h);
    if (rc) return rc;
    for (size_t k = 0; k < vis.size(); ++k) std::memcpy(fields25 + 25 * k, &h[(size_t)kDumpStride * vis[k] + 1], sizeof(float) * 25);
  }
  return (int64_t)vis.size();
}

namespace {

// scatter ProjectedGrads rows [begin, end) (indexed by projected position) to source index and upload
int upload_projected_grads(splatb200_view* v, const std::vector<int64_t>& vis, int64_t begin, int64_t end, const float* g_mean2d,
                           const float* g_range, const float* g_cov2d, const float* g_velocity, const float* g_opacity,
                           DevScratch& d) {
  splatb200_ctx* c = v->ctx;
  const size_t N = (size_t)c->n;
  std::vector<float> h((size_t)kProjGradStride * std::max<size_t>(1, N), 0.0f);
  for (int64_t k = begin; k < end; ++k) {
    float* q = &h[(size_t)kProjGradStride * vis[k]];
    if (g_mean2d) { q[0] = g_mean2d[2 * k]; q[1] = g_mean2d[2 * k + 1]; }
    if (g_range) q[2] = g_range[k];
    if (g_cov2d) for (int e = 0; e < 4; ++e) q[3 + e] = g_cov2d[4 * k + e];
    if (g_velocity) for (int e = 0; e < 3; ++e) q[7 + e] = g_velocity[3 * k + e];
  }
  if (g_opacity) for (size_t i = 0; i < N; ++i) h[(size_t)kProjGradStride * i + 10] = g_opacity[i];
  CU_TRY(c, cudaMalloc(&d.p, sizeof(float) * h.size()));
  CU_TRY(c, cudaMemcpyAsync(d.p, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));  // h is a local
  return SPLATB200_OK;
}

}  // namespace

extern "C" int splatb200_view_project_backward(splatb200_view* v, const float* g_mean2d, const float* g_range,
                                               const float* g_cov2d, const float* g_velocity, int64_t begin, int64_t end,
                                               float* g_mean_w, float* g_cov_w, float* g_vel_dyn_w) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  CU_TRY(c, cudaSetDevice(c->device));
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  std::vector<int64_t> vis;
  int rc = visible_list(v, vis);
  if (rc) return rc;
  if (begin < 0 || end > (int64_t)vis.size() || begin > end) return c->fail(SPLATB200_EINVAL, "project_backward: [begin, end) outside the projected list");
  if (begin == end) return SPLATB200_OK;
  DevScratch pgin, cg;
  rc = upload_projected_grads(v, vis, begin, end, g_mean2d, g_range, g_cov2d, g_velocity, nullptr, pgin);
  if (rc) return rc;
  const size_t N = (size_t)c->n;
  CU_TRY(c, cudaMalloc(&cg.p, sizeof(float) * kComposeGradStride * N));
  CU_TRY(c, cudaMemsetAsync(cg.p, 0, sizeof(float) * kComposeGradStride * N, c->stream));
  launch_project_bwd_mode(kProjOnly, v->s, c->scene_dev(v->d_actors), v->proj, c->pg(), v->sensor_grads, v->actor_acc, pgin.p,
                          cg.p, vis[begin], vis[end - 1] + 1, c->stream);
  CHECK_LAUNCH(c, "k_project_bwd<proj-only>");
  c->launches += 1;
  std::vector<float> h((size_t)kComposeGradStride * N);
  CU_TRY(c, cudaMemcpyAsync(h.data(), cg.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  for (int64_t k = begin; k < end; ++k) {  // accumulate (+=) like the reference (projection.hpp:283-286)
    const int64_t i = vis[k];
    const float* o = &h[(size_t)kComposeGradStride * i];
    for (int e = 0; e < 3; ++e) {
      if (g_mean_w) g_mean_w[3 * i + e] += o[e];
      if (g_vel_dyn_w) g_vel_dyn_w[3 * i + e] += o[12 + e];
    }
    if (g_cov_w) for (int e = 0; e < 9; ++e) g_cov_w[9 * i + e] += o[3 + e];
  }
  return SPLATB200_OK;
}

extern "C" int splatb200_view_compose_backward(splatb200_view* v, const float* g_mean_w, const float* g_cov_w,
                                               const float* g_vel_dyn_w, const float* g_opacity, int64_t begin, int64_t end) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  CU_TRY(c, cudaSetDevice(c->device));
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  if (begin < 0 || end > c->n || begin > end) return c->fail(SPLATB200_EINVAL, "compose_backward: [begin, end) outside the scene");
  if (begin == end) return SPLATB200_OK;
  const size_t N = (size_t)c->n;
  std::vector<float> hc((size_t)kComposeGradStride * N, 0.0f), hp((size_t)kProjGradStride * N, 0.0f);
  for (int64_t i = begin; i < end; ++i) {
    float* o = &hc[(size_t)kComposeGradStride * i];
    for (int e = 0; e < 3; ++e) {
      if (g_mean_w) o[e] = g_mean_w[3 * i + e];
      if (g_vel_dyn_w) o[12 + e] = g_vel_dyn_w[3 * i + e];
    }
    if (g_cov_w) for (int e = 0; e < 9; ++e) o[3 + e] = g_cov_w[9 * i + e];
    if (g_opacity) hp[(size_t)kProjGradStride * i + 10] = g_opacity[i];
  }
  DevScratch cg, pgin;
  CU_TRY(c, cudaMalloc(&cg.p, sizeof(float) * hc.size()));
  CU_TRY(c, cudaMalloc(&pgin.p, sizeof(float) * hp.size()));
  CU_TRY(c, cudaMemcpyAsync(cg.p, hc.data(), sizeof(float) * hc.size(), cudaMemcpyHostToDevice, c->stream));
  CU_TRY(c, cudaMemcpyAsync(pgin.p, hp.data(), sizeof(float) * hp.size(), cudaMemcpyHostToDevice, c->stream));
  launch_project_bwd_mode(kComposeOnly, v->s, c->scene_dev(v->d_actors), v->proj, c->pg(), v->sensor_grads, v->actor_acc,
                          pgin.p, cg.p, begin, end, c->stream);
  CHECK_LAUNCH(c, "k_project_bwd<compose-only>");
  c->launches += 1;
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (!c->tracks.empty()) v->actor_pending = true;
  return SPLATB200_OK;
}

extern "C" int splatb200_view_backward_projected(splatb200_view* v, const float* g_mean2d, const float* g_range,
                                                 const float* g_cov2d, const float* g_velocity, const float* g_opacity) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  CU_TRY(c, cudaSetDevice(c->device));
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "backward without saved forward state");
  if (c->n == 0) return SPLATB200_OK;
  std::vector<int64_t> vis;
  int rc = visible_list(v, vis);
  if (rc) return rc;
  DevScratch pgin;
  rc = upload_projected_grads(v, vis, 0, (int64_t)vis.size(), g_mean2d, g_range, g_cov2d, g_velocity, g_opacity, pgin);
  if (rc) return rc;
  launch_project_bwd_mode(kFromProjected, v->s, c->scene_dev(v->d_actors), v->proj, c->pg(), v->sensor_grads, v->actor_acc,
                          pgin.p, nullptr, 0, c->n, c->stream);
  CHECK_LAUNCH(c, "k_project_bwd<from-projected>");
  c->launches += 1;
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (!c->tracks.empty()) v->actor_pending = true;
  return SPLATB200_OK;
}

// ---- introspection ------------------------------------------------------------------------------
namespace {
template <class T> int fetch(splatb200_ctx* c, std::vector<T>& h, const T* d, size_t n) {
  h.resize(n);
  if (n) CU_TRY(c, cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return SPLATB200_OK;
}
}  // namespace

extern "C" int64_t splatb200_view_array(splatb200_view* v, const char* name_c, void* dst) {
  splatb200_ctx* c = v->ctx;
  join_view(v);  // order the ctx stream after the view's own stream
  const std::string name(name_c ? name_c : "");
  if (v->stage < 1) return c->fail(SPLATB200_ERUNTIME, "view_array before forward");
  const size_t N = (size_t)c->n;

  struct Field { const char* name; int off, width; };
  static const Field dump_fields[] = {{"mean2d", 1, 2}, {"depth_key", 3, 1}, {"cov2d", 4, 4}, {"velocity", 8, 3},
                                      {"aabb", 11, 4}, {"conic", 15, 4}, {"det_ratio", 19, 1}, {"mu_sensor", 20, 3},
                                      {"rel_vel_sensor", 23, 3}};
  static const Field scene_fields[] = {{"opacity", 26, 1}, {"mean_w", 27, 3}, {"vel_dyn_w", 30, 3}, {"cov_w", 33, 9}};
  const Field* df = nullptr;
  bool per_scene = false;
  for (const auto& f : dump_fields) if (name == f.name) df = &f;
  for (const auto& f : scene_fields) if (name == f.name) { df = &f; per_scene = true; }

  if (df || name == "source_index" || name == "rect") {
    std::vector<uint32_t> cnt;
    int rc = fetch(c, cnt, v->proj.count, N);
    if (rc) return rc;
    std::vector<int64_t> vis;
    for (size_t i = 0; i < N; ++i) if (cnt[i]) vis.push_back((int64_t)i);
    if (name == "source_index") {
      if (dst) std::memcpy(dst, vis.data(), sizeof(int64_t) * vis.size());
      return (int64_t)vis.size();
    }
    if (name == "rect") {
      std::vector<int4> r;
      rc = fetch(c, r, v->proj.rect, N);
      if (rc) return rc;
      if (dst) {
        int64_t* d = (int64_t*)dst;
        for (size_t k = 0; k < vis.size(); ++k) {
          const int4 q = r[vis[k]];
          d[4 * k] = q.x; d[4 * k + 1] = q.y; d[4 * k + 2] = q.z; d[4 * k + 3] = q.w;
        }
      }
      return (int64_t)vis.size() * 4;
    }
    const size_t rows = per_scene ? N : vis.size();
    if (!dst) return (int64_t)rows * df->width;
    float* dump = nullptr;
    CU_TRY(c, cudaMalloc(&dump, sizeof(float) * kDumpStride * std::max<size_t>(1, N)));
    cudaMemsetAsync(dump, 0, sizeof(float) * kDumpStride * N, c->stream);
    launch_project_dump(v->s, c->scene_dev(v->d_actors), dump, c->stream);
    std::vector<float> h;
    rc = fetch(c, h, dump, (size_t)kDumpStride * N);
    cudaFree(dump);
    if (rc) return rc;
    float* d = (float*)dst;
    for (size_t k = 0; k < rows; ++k) {
      const size_t i = per_scene ? k : (size_t)vis[k];
      for (int w = 0; w < df->width; ++w) d[k * df->width + w] = h[i * kDumpStride + df->off + w];
    }
    return (int64_t)rows * df->width;
  }

  if (name == "packed_record") {
    // what k_project STORED for the compositing kernels (not a recomputation): per visible Gaussian, in source order,
    // geomA (mean2d.xy, velocity.xy) | geomB (conic a, 2b, c, rho) | geomC (depth key, v_r) | the 16 channel slots
    std::vector<uint32_t> cnt;
    int rc = fetch(c, cnt, v->proj.count, N);
    if (rc) return rc;
    std::vector<size_t> vis;
    for (size_t i = 0; i < N; ++i) if (cnt[i]) vis.push_back(i);
    constexpr int kW = 26;
    if (!dst) return (int64_t)vis.size() * kW;
    std::vector<float4> gA, gB, gF;
    std::vector<float2> gC;
    rc = fetch(c, gA, (const float4*)v->proj.geomA, N);
    if (!rc) rc = fetch(c, gB, (const float4*)v->proj.geomB, N);
    if (!rc) rc = fetch(c, gC, (const float2*)v->proj.geomC, N);
    if (!rc) rc = fetch(c, gF, (const float4*)v->proj.feat, 4 * N);
    if (rc) return rc;
    float* d = (float*)dst;
    for (size_t k = 0; k < vis.size(); ++k) {
      const size_t i = vis[k];
      float* o = d + kW * k;
      o[0] = gA[i].x; o[1] = gA[i].y; o[2] = gA[i].z; o[3] = gA[i].w;
      o[4] = gB[i].x; o[5] = gB[i].y; o[6] = gB[i].z; o[7] = gB[i].w;
      o[8] = gC[i].x; o[9] = gC[i].y;
      for (int q = 0; q < 4; ++q) { o[10 + 4 * q] = gF[4 * i + q].x; o[11 + 4 * q] = gF[4 * i + q].y; o[12 + 4 * q] = gF[4 * i + q].z; o[13 + 4 * q] = gF[4 * i + q].w; }
    }
    return (int64_t)vis.size() * kW;
  }

  if (name == "isect_tile" || name == "isect_depth_bits" || name == "isect_src") {
    if (v->stage < 2) return c->fail(SPLATB200_ERUNTIME, "worklist not built");
    if (!dst) return v->I;
    int64_t* d = (int64_t*)dst;
    if (name == "isect_src") {
      std::vector<uint32_t> h;
      int rc = fetch(c, h, v->vals(), (size_t)v->I);
      if (rc) return rc;
      for (int64_t k = 0; k < v->I; ++k) d[k] = h[k];
    } else if (name == "isect_tile") {
      // the last sort pass writes source indices only; the tile of a list position follows from the tile ranges
      std::vector<uint32_t> tb, te;
      int rc = fetch(c, tb, v->tile_begin, (size_t)v->n_tiles);
      if (!rc) rc = fetch(c, te, v->tile_end, (size_t)v->n_tiles);
      if (rc) return rc;
      for (int64_t k = 0; k < v->I; ++k) d[k] = -1;
      for (int64_t t = 0; t < v->n_tiles; ++t)
        for (uint32_t k = tb[t]; k < te[t] && (int64_t)k < v->I; ++k) d[k] = t;
    } else {  // the depth half of the reference's sort key: fp32 bits of the owner's depth_key
      std::vector<uint32_t> h;
      std::vector<float2> gc;
      int rc = fetch(c, h, v->vals(), (size_t)v->I);
      if (!rc) rc = fetch(c, gc, (const float2*)v->proj.geomC, N);
      if (rc) return rc;
      for (int64_t k = 0; k < v->I; ++k) {
        uint32_t bits;
        std::memcpy(&bits, &gc[h[k]].x, 4);
        d[k] = bits;
      }
    }
    return v->I;
  }
  if (name == "tile_begin" || name == "tile_end") {
    if (v->stage < 2) return c->fail(SPLATB200_ERUNTIME, "worklist not built");
    if (!dst) return v->n_tiles;
    std::vector<uint32_t> h;
    int rc = fetch(c, h, name == "tile_begin" ? v->tile_begin : v->tile_end, (size_t)v->n_tiles);
    if (rc) return rc;
    for (int64_t k = 0; k < v->n_tiles; ++k) ((int64_t*)dst)[k] = h[k];
    return v->n_tiles;
  }
  if (name == "hit_bits") {  // per list entry: which warps of the tile's CTA blended it in the last forward (saved for the backward)
    if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "not rasterized");
    if (!dst) return v->I;
    std::vector<uint8_t> h;
    int rc = fetch(c, h, v->out.hit, (size_t)v->I);
    if (rc) return rc;
    for (int64_t k = 0; k < v->I; ++k) ((int64_t*)dst)[k] = h[k];
    return v->I;
  }
  if (name == "raster_stats") {  // cumulative since view creation; zeros unless SPLATB200_STATS is set
    if (dst) {
      // [0] staged entries, [1] per-warp survivors of the first-level cull, [2] shared lidar kernel: group-list entries;
      // lidar kernel pair: (entry, ray) candidates of the exact-qf prefilter, [3] shared lidar kernel: loop iterations (max
      // over the warp's groups); lidar kernel pair: phase-2 trips (longest lane per round), [4] staged entries with a
      // non-finite record
      unsigned long long h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (v->out.stats) {
        CU_TRY(c, cudaMemcpyAsync(h, v->out.stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CU_TRY(c, cudaStreamSynchronize(c->stream));
      }
      for (int k = 0; k < 8; ++k) ((int64_t*)dst)[k] = (int64_t)h[k];
    }
    return 8;
  }
  if (name == "grid") {
    if (dst) { ((int64_t*)dst)[0] = v->s.tiles_x; ((int64_t*)dst)[1] = v->s.tiles_y; }
    return 2;
  }
  if (v->stage < 3) return c->fail(SPLATB200_ERUNTIME, "not rasterized");
  const size_t P = (size_t)v->P;
  if (name == "n_contrib" || name == "last_idx") {
    if (!dst) return v->P;
    std::vector<int32_t> h;
    int rc = fetch(c, h, name == "n_contrib" ? v->out.n_contrib : v->out.last_idx, P);
    if (rc) return rc;
    for (size_t k = 0; k < P; ++k) ((int64_t*)dst)[k] = h[k];
    return v->P;
  }
  const float* src = nullptr;
  size_t cnt = P;
  if (name == "blend") { src = v->out.blend; cnt = 16 * P; }
  else if (name == "alpha") src = v->out.alpha;
  else if (name == "t_final") src = v->out.t_final;
  else if (name == "range_blend") src = v->out.range_blend;
  else if (name == "los") src = v->out.los;
  else if (name == "lidar_head") { src = v->out.head_y; cnt = 2 * P; }
  else if (name == "decoded") { src = v->d_dec_image; cnt = 3 * P; }
  else if (name.rfind("decoder_act", 0) == 0 && name.size() == 12 && name[11] >= '0' && name[11] <= '5') {
    src = v->dec_act[name[11] - '0']; cnt = 32 * P;   // x0, h0, t1, h1, t2, h2 of the last decode (P x 32)
  }
  if (!src) return c->fail(SPLATB200_EINVAL, "unknown array name " + name);
  if (dst && cnt) {
    CU_TRY(c, cudaMemcpyAsync(dst, src, sizeof(float) * cnt, cudaMemcpyDeviceToHost, c->stream));
    CU_TRY(c, cudaStreamSynchronize(c->stream));
  }
  return (int64_t)cnt;
}
