/* splat_b200.h — C ABI of libsplat_b200.so: the B200 (sm_100a) implementation of SplatAD's
 * differentiable camera + lidar Gaussian rasterizer hot path
 *     compose -> project -> tile-bin + sort -> composite   and the reverse.
 *
 * Plain pointers and sizes only; no C++/torch types. Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj/include/splat/, or SPEC.md for the
 * two modules the reference only specifies). INTEGRATION.md shows the reference-side binding.
 *
 * Conventions
 *  - All per-Gaussian arrays use the reference's physical layout (Eigen column-major kxN ==
 *    N rows of k contiguous floats): mean/scale_log/color 3 floats, quat 4 floats (w,x,y,z),
 *    feature d_f floats per Gaussian (scene.hpp:11-19).
 *  - Rotation matrices are 9 floats ROW-major.
 *  - Every call returns 0 on success or a negative SPLATB200_E* code; splatb200_last_error()
 *    gives the message. Errors the reference raises as C++ exceptions keep their text
 *    ("unknown actor_id 7" scene.hpp:176-177,297-298; "actor track has no poses" scene.hpp:242).
 *  - A ctx is bound to one device and one stream; calls on a ctx are stream-ordered and not
 *    thread-safe. Different ctxs are independent.
 *  - There is no CPU fallback: without a CUDA device ctx_create fails.
 */
#ifndef SPLAT_B200_H_
#define SPLAT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLATB200_OK 0
#define SPLATB200_EINVAL -1      /* bad argument */
#define SPLATB200_ECUDA -2       /* CUDA runtime error */
#define SPLATB200_EOUTOFRANGE -3 /* std::out_of_range in the reference (unknown actor_id) */
#define SPLATB200_ERUNTIME -4    /* std::runtime_error in the reference (empty track, backward without forward) */
#define SPLATB200_ENOMEM -5

#define SPLATB200_MAX_CHANNELS 16 /* 3 colour + D_f <= 13 features */
#define SPLATB200_TILE 16
#define SPLATB200_NPHI 32
#define SPLATB200_NOMEGA 8

typedef struct splatb200_ctx splatb200_ctx;
typedef struct splatb200_view splatb200_view;

/* projection.hpp:7-15 RasterSettings<float> */
typedef struct {
  float dilation, alpha_clamp, alpha_min, qform_max, transmittance_min, near_plane, lidar_min_range;
} splatb200_raster_settings;

/* scene.hpp:98-137 CameraModel<float> (embedding belongs to the decoder: out of scope) */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9], t[3];          /* pose: world -> sensor */
  float vel_lin[3], vel_ang[3];
  float shutter_duration, time_offset, timestamp;
} splatb200_camera;

/* scene.hpp:139-168 LidarModel<float> */
typedef struct {
  const float* elevation_channels; /* host pointer, n_beams strictly increasing radians */
  int32_t n_beams;
  float azimuth_resolution, scan_duration, beam_divergence_h, beam_divergence_v;
  float R[9], t[3];
  float vel_lin[3], vel_ang[3];
  float timestamp, max_range;
} splatb200_lidar;

/* scene.hpp:50-96 ActorTrack<double>: actor poses are per-actor host work and stay in double */
typedef struct {
  int32_t n_poses;
  const double* stamps;      /* n_poses, strictly increasing */
  const double* R;           /* n_poses x 9 row-major, actor -> world */
  const double* t;           /* n_poses x 3 */
  const double* pose_offset; /* n_poses x 6: translation (world) 0-2, rotvec (actor frame) 3-5 */
  double vel_lin[3], vel_ang[3];
  double vel_offset[6];
  int32_t init_velocity_from_poses; /* non-zero: ignore vel_lin/vel_ang, use scene.hpp:70-83 */
} splatb200_actor_track;

/* projection.hpp:207-222 SensorGrads<float> (d_embedding: decoder, out of scope) */
typedef struct {
  float d_vel_lin[3], d_vel_ang[3], d_time_offset;
} splatb200_sensor_grads;

/* counts of one forward pass */
typedef struct {
  int64_t n_gaussians;     /* N */
  int64_t n_visible;       /* V: |project_*()| */
  int64_t n_intersections; /* I: duplicated (Gaussian, tile) pairs */
  int64_t n_queries;       /* P: pixels or rays */
  int32_t tiles_x, tiles_y;
} splatb200_view_stats;

/* ---- context ------------------------------------------------------------------------------- */
int splatb200_ctx_create(int device, void* cuda_stream /* cudaStream_t or NULL */, splatb200_ctx** out);
void splatb200_ctx_destroy(splatb200_ctx* ctx);
const char* splatb200_last_error(const splatb200_ctx* ctx); /* ctx may be NULL: last create error */
int splatb200_ctx_sync(splatb200_ctx* ctx);
/* number of hand-written kernels launched by this ctx since creation (bench.py's gpu_launches), and the number of
 * library kernels launched beside them (always 0: the radix sorts and scans of the binning stage are hand-written) */
int64_t splatb200_ctx_launch_count(const splatb200_ctx* ctx);
int64_t splatb200_ctx_library_launch_count(const splatb200_ctx* ctx);
/* per-stage CUDA-event timing on the ctx stream (off by default). Stages: 0 project, 1 depth sort + scan, 2 tile counts
 * (tile ranges from the rectangles), 3 tile sort (duplication fused into its first pass), 4 unused, 5 raster_fwd, 6 raster_bwd, 7 project_bwd. set_profiling(1) resets the running
 * sums; stage_ms returns the MEAN milliseconds per launch of each stage over every forward / backward of
 * the view since then (syncs). Event pairs are folded into the sums at the forward pass's own
 * synchronisation point, so enabling profiling adds no host-device synchronisation to a timed region.
 * This is the measurement hook bench.py's roofline uses. */
int splatb200_ctx_set_profiling(splatb200_ctx* ctx, int32_t on);
/* View streams (off by default). On: every view enqueues its forward / backward on its own stream, so one sensor's
 * latency-bound binning kernels and the tail of its compositing grid overlap another sensor's kernels. A view's work is
 * ordered after everything asked of the ctx stream before the call; the ctx stream is ordered after the views' work by
 * zero / upload / download / sync calls, by every other call on that view, and by splatb200_ctx_join — call it before
 * work you enqueue yourself on the ctx stream (e.g. an NCCL all-reduce of the bound gradient buffer) reads the results.
 * Threads: with view streams on, DIFFERENT views of one ctx may be driven from different host threads (forward,
 * backward, download_async, backward_host_overlapped), so that one view's host sync — the worklist size, read once per
 * forward — does not delay another view's launches; ctx-level calls must not run concurrently with them. */
int splatb200_ctx_set_view_streams(splatb200_ctx* ctx, int32_t on);
int splatb200_ctx_join(splatb200_ctx* ctx);
int splatb200_view_stage_ms(splatb200_view* v, float out_ms[8]);

/* ---- multi-GPU: the one collective of the path ("parallel per sensor view" over an immutable scene,
 * SPEC.md:90; per-worker SceneParamGrads summed, scene.hpp:351-362 SceneParamGrads::add) ---------------------------
 * One process (and one ctx) per GPU; frames / sensors are sharded over ranks with the scene replicated; after a rank
 * has accumulated the gradients of its own work items, splatb200_allreduce_grads sums the contiguous
 * (14 + d_f) * N-float SceneParamGrads buffer (and the per-actor ActorGrad slots) over all ranks, in place, with NCCL.
 * NCCL is bound at run time from the process's own libnccl.so.2 (the one a trainer or torch already loaded), so the
 * library itself has no link-time NCCL dependency; without it these calls return SPLATB200_ERUNTIME.
 *   comm_init: rank 0 obtains a 128-byte id (splatb200_nccl_unique_id), every rank receives it out of band (MPI,
 *              torch.distributed, a file) and calls comm_init(ctx, id, rank, world) — ncclCommInitRank.
 *   comm_bind: a C++ trainer that already owns an ncclComm_t hands it over (not destroyed by the library).
 * allreduce_grads orders itself after every view stream (splatb200_ctx_join) and runs on the ctx stream. */
int splatb200_nccl_unique_id(void* id128);
int splatb200_ctx_comm_init(splatb200_ctx* ctx, const void* id128, int32_t rank, int32_t world);
int splatb200_ctx_comm_bind(splatb200_ctx* ctx, void* nccl_comm /* ncclComm_t */, int32_t rank, int32_t world);
int splatb200_ctx_comm_destroy(splatb200_ctx* ctx);
int splatb200_ctx_comm_info(const splatb200_ctx* ctx, int32_t* rank, int32_t* world); /* world = 0: no communicator */
int splatb200_allreduce_grads(splatb200_ctx* ctx);

/* ---- scene: GaussianSet + SceneGraph (scene.hpp:11-45, 171-187) ------------------------------ */
/* host arrays are copied to the device; actor_id is validated lazily against the tracks at
 * compose time exactly like scene.hpp:297-298 */
int splatb200_scene_upload(splatb200_ctx* ctx, int64_t n, int32_t d_f, const float* mean, const float* scale_log,
                           const float* quat, const float* opacity_logit, const float* color, const float* feature,
                           const int32_t* actor_id);
/* The per-iteration upload without the wait (a resident scene of the same shape; anything else takes the blocking path).
 * Geometry first: mean, scale_log, quat, opacity_logit and actor_id (48 B per Gaussian) go up on the ctx stream, colour
 * and features (12 + 4 d_f B) follow behind them on a copy stream of their own. A view's projection, depth sort and tile
 * binning need the geometry only and run while the appearance arrays are still in flight; its forward waits for them
 * in front of the compositing kernel. The host arrays must stay valid (and should be pinned) until the next
 * splatb200_ctx_sync. Same GaussianSet fields as scene.hpp:137-168. */
int splatb200_scene_upload_async(splatb200_ctx* ctx, int64_t n, int32_t d_f, const float* mean, const float* scale_log,
                                 const float* quat, const float* opacity_logit, const float* color, const float* feature,
                                 const int32_t* actor_id);
/* zero-copy variant: DEVICE pointers owned by the caller (e.g. optimiser state); must outlive use */
int splatb200_scene_bind_device(splatb200_ctx* ctx, int64_t n, int32_t d_f, const float* mean, const float* scale_log,
                                const float* quat, const float* opacity_logit, const float* color,
                                const float* feature, const int32_t* actor_id, int32_t max_actor_id);
/* SceneGraph::tracks; actor k (1-based) = tracks[k-1] */
int splatb200_scene_set_tracks(splatb200_ctx* ctx, int32_t n_tracks, const splatb200_actor_track* tracks);
/* ActorTrack::init_velocity_from_poses result / stored velocities (lin 3, ang 3; without vel_offset) */
int splatb200_scene_actor_velocity(splatb200_ctx* ctx, int32_t track, double out6[6]);

/* ---- SceneParamGrads (scene.hpp:325-363) ----------------------------------------------------- */
/* one contiguous device buffer of 27*N floats (d_f = 13):
 *   [d_mean 3N | d_scale_log 3N | d_quat 4N | d_opacity_logit N | d_color 3N | d_feature d_f*N]
 * backward ACCUMULATES (+=) like the reference (scene.hpp:394-456); zero explicitly. */
int splatb200_grads_zero(splatb200_ctx* ctx);
int64_t splatb200_grads_size(const splatb200_ctx* ctx);            /* number of floats */
float* splatb200_grads_device_ptr(splatb200_ctx* ctx);             /* for ncclAllReduce */
int splatb200_grads_bind_device(splatb200_ctx* ctx, float* dev, int64_t n_floats); /* caller-owned buffer */
int splatb200_grads_download(splatb200_ctx* ctx, float* d_mean, float* d_scale_log, float* d_quat,
                             float* d_opacity_logit, float* d_color, float* d_feature);
/* SceneParamGrads::ActorGrad: d_pose_offset (n_poses x 6) and d_vel_offset (6), double */
int splatb200_grads_download_actor(splatb200_ctx* ctx, int32_t track, double* d_pose_offset, double* d_vel_offset6);

/* ---- views: one sensor render ---------------------------------------------------------------- */
int splatb200_view_create_camera(splatb200_ctx* ctx, const splatb200_camera* cam,
                                 const splatb200_raster_settings* settings, splatb200_view** out);
/* rays: n_rays x 3 floats (azimuth in [0,2pi), elevation, capture-time offset t_l), grouped per
 * tile: tile t owns rays [ray_begin[t], ray_end[t]) (SPEC.md:230-238 assign_points_to_tiles
 * output); n_tiles must equal M_phi*M_omega. Host pointers, copied. */
int splatb200_view_create_lidar(splatb200_ctx* ctx, const splatb200_lidar* lidar,
                                const splatb200_raster_settings* settings, const float* rays, int64_t n_rays,
                                const int64_t* ray_begin, const int64_t* ray_end, int64_t n_tiles,
                                splatb200_view** out);
void splatb200_view_destroy(splatb200_view* v);
/* update sensor pose / velocities / time offset between frames without re-creating buffers */
int splatb200_view_set_camera(splatb200_view* v, const splatb200_camera* cam);
int splatb200_view_set_lidar_pose(splatb200_view* v, const float R[9], const float t[3], const float vel_lin[3],
                                  const float vel_ang[3]);
/* a new sweep for an existing lidar view — the per-frame output of splatb200_assign_points: same layout as the `rays`
 * of view_create_lidar, any number of rays (buffers grow as needed); n_tiles must equal the view's */
int splatb200_view_set_rays(splatb200_view* v, const float* rays, int64_t n_rays, const int64_t* ray_begin,
                            const int64_t* ray_end, int64_t n_tiles);
/* lidar tile grid: M_phi, M_omega */
int splatb200_lidar_grid(const splatb200_lidar* lidar, int32_t* m_phi, int32_t* m_omega);

/* compose_at_time (scene.hpp:273-308) + project_camera / project_lidar (projection.hpp:88-118,
 * 140-174) + image/lidar tile ranges and build_sorted_worklist +
 * rasterize_camera / rasterize_lidar, stream-ordered.
 * stop_after: 0 = everything, 1 = after projection, 2 = after tiling/sort. */
int splatb200_view_forward(splatb200_view* v, float t_scene, int32_t stop_after);
int splatb200_view_stats_get(splatb200_view* v, splatb200_view_stats* out); /* syncs */

/* Rendered outputs, DEVICE pointers valid until the next forward on this view.
 *   blend:  P x 16 floats, query-major (ChannelImage physical layout, common.hpp:104-116):
 *           camera: rgb(3) + feature(13); lidar: feature(13), [13] expected range, [14] median range,
 *           [15] accumulated opacity
 *   alpha:  P accumulated opacity (1 - T)
 *   n_contrib: P int32 number of blended Gaussians */
const float* splatb200_view_blend(splatb200_view* v);
const float* splatb200_view_alpha(splatb200_view* v);
const int32_t* splatb200_view_n_contrib(splatb200_view* v);

/* rasterizer backward + project_*_backward (projection.hpp:250-288, 322-357) +
 * compose_backward (scene.hpp:386-458). g_blend16: P x 16, g_alpha: P (DEVICE pointers).
 * Lidar: slots 14 (median) and 15 carry no gradient; the accumulated-opacity gradient is g_alpha.
 * Accumulates into the ctx's SceneParamGrads and this view's SensorGrads. */
int splatb200_view_backward(splatb200_view* v, const float* g_blend16, const float* g_alpha);
int splatb200_view_sensor_grads(splatb200_view* v, splatb200_sensor_grads* out); /* syncs */

/* Host-buffer convenience (the end-to-end path): upstream grads come from HOST memory, outputs go
 * to HOST memory; copies are issued on the ctx stream. Any pointer may be NULL to skip it. */
int splatb200_view_download(splatb200_view* v, float* blend16, float* alpha, int32_t* n_contrib);
int splatb200_view_backward_host(splatb200_view* v, const float* g_blend16, const float* g_alpha);
/* Overlapped variants of the two calls above for PINNED host buffers: the copies run on the view's own copy
 * streams (one per direction) beside the compute stream, ordered by events. download_async returns at once; the host buffers
 * are complete after splatb200_ctx_sync (or any later stream-ordered call that synchronises, e.g. grads_download of a
 * backward that depended on them). backward_host_overlapped uploads the upstream gradients on the host-to-device copy
 * stream — after this view's pending download_async, because upstream gradients are a function of the rendered
 * outputs — and runs the backward kernels once they have arrived; other views' kernels keep the GPU busy meanwhile. */
int splatb200_view_download_async(splatb200_view* v, float* blend16, float* alpha, int32_t* n_contrib);
int splatb200_view_backward_host_overlapped(splatb200_view* v, const float* g_blend16, const float* g_alpha);
/* Fused forms for PINNED host buffers: forward_to_host renders a camera image in `bands` bands of tile rows (0: default,
 * 4; at most 8; a lidar sweep is one band) and sends each band's outputs to the host on the view's copy stream while the
 * next band is being composited; backward_from_host uploads the upstream gradients band by band — a band's upload
 * follows that band's download, because upstream gradients are a function of the rendered outputs — and starts each
 * band's backward kernel as soon as its gradients have arrived. Host buffers are complete after splatb200_ctx_sync. */
int splatb200_view_forward_to_host(splatb200_view* v, float t_scene, float* blend16, float* alpha, int32_t* n_contrib,
                                   int32_t bands);
int splatb200_view_backward_from_host(splatb200_view* v, const float* g_blend16, const float* g_alpha);

/* ---- line-of-sight channel of a lidar view (SPEC.md:427 loss_total) -----
 * The one loss term that needs the compositing loop: los[q] = sum of alpha_i over the blended Gaussians whose
 * rolling-shutter range r_i lies in front of los_cut[q] = r_p - eps ("penalizing opacity before the ground truth lidar
 * range"; r_p is the `range` column splatb200_assign_points returns). set_los uploads the per-ray cuts (HOST, P floats;
 * NULL switches the channel off); the next forward fills the accumulator, read back with
 * splatb200_view_array(v, "los", dst). set_los_grad uploads dL/dlos (HOST, P floats) for the next backward, which adds
 * it to dL/dalpha_i of exactly those Gaussians. Both arrays are in the caller's ray order. */
int splatb200_view_set_los(splatb200_view* v, const float* los_cut);
int splatb200_view_set_los_grad(splatb200_view* v, const float* g_los);

/* ---- optimizer step (SPEC.md:439-444 optimizer_step) -------------------------
 * Adam (beta = 0.9 / 0.999, eps = 1e-15) with per-group scheduled learning rates, in place on the ctx's GaussianSet
 * (uploaded or bound device arrays), reading the ctx's SceneParamGrads buffer — i.e. what the backward passes, and on
 * several GPUs the all-reduce, left there. Groups: 0 mean, 1 scale_log, 2 quat, 3 opacity_logit, 4 color, 5 feature.
 * Learning rate of a group at `step` (0-based): min(1, step / warmup) * lr_init * (lr_final / lr_init)^t with
 * t = clamp((step - warmup) / (total_steps - warmup), 0, 1) — linear warm-up from 0, then exponential interpolation.
 * A group whose gradient holds a non-finite value is skipped (parameters and moments untouched); skipped[6] (may be NULL)
 * receives 1 for such groups. Moments live in the ctx and start at zero (reset by a scene upload of another size). */
typedef struct {
  float lr_init[6], lr_final[6];
  int64_t warmup_steps[6];
  int64_t total_steps;
} splatb200_adam_config;
int splatb200_optimizer_step(splatb200_ctx* ctx, const splatb200_adam_config* cfg, int64_t step, int32_t skipped[6]);
/* forget the Adam moments and step state (splatb200_scene_upload of the SAME shape keeps them — the per-iteration
 * parameter refresh —; a new shape or splatb200_scene_bind_device drops them) */
int splatb200_optimizer_reset(splatb200_ctx* ctx);
/* optimizer_step fused with the collective (every rank steps only its shard of the flat gradient layout):
 * reduce (sum) of each rank's shard to its owner, agreement on the groups to skip (a non-finite gradient anywhere skips
 * the group everywhere), Adam on the shard, broadcast of the updated parameters. Same bytes on the wire as the
 * all-reduce; optimizer work and state divide by the world size. */
int splatb200_sharded_optimizer_step(splatb200_ctx* ctx, const splatb200_adam_config* cfg, int64_t step, int32_t skipped[6]);
/* The same on the slice [lo, hi) of the gradient buffer's flat layout [mean 3N | scale_log 3N | quat 4N | opacity N |
 * color 3N | feature d_f N] only — a rank's shard after a reduce-scatter (paper_2411_16816_b200/dist.py
 * sharded_optimizer_step: reduce-scatter -> this -> all-gather of the parameters). skip_groups[6] (may be NULL): groups to
 * leave untouched, e.g. because ANOTHER rank's shard of the group held a non-finite gradient; skipped[6] reports the groups
 * whose gradient is non-finite inside [lo, hi). */
int splatb200_optimizer_step_range(splatb200_ctx* ctx, const splatb200_adam_config* cfg, int64_t step, int64_t lo, int64_t hi,
                                   const int32_t skip_groups[6], int32_t skipped[6]);
/* non-finite check alone, per group, inside [lo, hi) (sharded step: the flags are all-reduced before anyone steps) */
int splatb200_grads_nonfinite_range(splatb200_ctx* ctx, int64_t lo, int64_t hi, int32_t flags[6]);
/* current parameters back to HOST arrays (any pointer may be NULL) */
int splatb200_scene_download(splatb200_ctx* ctx, float* mean, float* scale_log, float* quat, float* opacity_logit, float* color,
                             float* feature);

/* ---- lidar head (SPEC.md:366-389 decode_lidar; section 3.3) ----------------------
 * A 2-layer perceptron (hidden 32, rectified-linear inside, logistic outputs) from the D_f blended features of a ray + its
 * direction in the sensor frame to (intensity, ray-drop probability). weights: HOST, splatb200_lidar_head_params(d_f)
 * floats, row-major W1 [32 x (d_f + 3)], b1 [32], W2 [2 x 32], b2 [2]. forward: after splatb200_view_forward of a lidar
 * view; y: HOST, P x 2 in the caller's ray order. backward: g_y HOST P x 2; g_weights HOST (overwritten with dL/dweights);
 * g_blend16: DEVICE, P x 16 — dL/dfeature is ADDED to slots [0, d_f) of each ray, so that the buffer (holding any other
 * upstream gradient of the render) can go straight into splatb200_view_backward. */
int32_t splatb200_lidar_head_params(int32_t d_f);
/* fused form of the forward: with weights set (HOST, copied; NULL switches it off) every splatb200_view_forward of the
 * lidar view also decodes the blended features in the compositing kernel's epilogue, while they are still in registers;
 * read the P x 2 result with splatb200_view_array(v, "lidar_head", dst). */
int splatb200_view_set_lidar_head(splatb200_view* v, const float* weights);
int splatb200_lidar_head_forward(splatb200_view* v, const float* weights, float* y);
int splatb200_lidar_head_backward(splatb200_view* v, const float* weights, const float* g_y, float* g_weights,
                                  float* g_blend16);

/* ---- camera ConvDecoder (SPEC.md:362-380 decode_image; Eq. 7-8; ray directions scene.hpp:119-122) ----
 * Maps a camera view's blended features (+ per-pixel ray direction + the camera's 8-d embedding, broadcast) to a
 * per-pixel affine colour correction: I = M . F_rgb + b with (M - 1, b) the 6 outputs of a small CNN — two residual
 * blocks of 3x3 convolutions at width 32 (ReLU inside, reflect padding) and a linear head. The reference ships no
 * decoder code; the concrete layer list and parameter packing are fixed in oracle/decoder_oracle.hpp:
 *   x0 = (feature[d_f], ray_direction[3], embedding[8], 0...) (32 ch);  h0 = conv0(x0);
 *   h1 = h0 + conv2(relu(conv1(relu(h0))));  h2 = h1 + conv4(relu(conv3(relu(h1))));  y = Wh h2 + bh;
 *   I_c = (1 + y_c) rgb_c + y_{3+c}.
 * params: HOST, splatb200_conv_decoder_params() floats: for l = 0..4 W_l[co 32][ky 3][kx 3][ci 32] then b_l[32]; then
 * Wh[6][32], bh[6]. embedding: HOST, 8 floats. image: HOST, P x 3 (may be NULL: read it with
 * splatb200_view_array(v, "decoded", dst)). device_ms (may be NULL): device time of the decode, CUDA events.
 * Call after splatb200_view_forward of a camera view. The convolutions run on the tensor cores (tcgen05, tf32 operands
 * rounded to nearest, fp32 accumulation): results agree with an fp32 evaluation to ~1e-3 relative. */
int32_t splatb200_conv_decoder_params(void);
/* Arithmetic of the decoder's convolutions (they run on the tf32 tensor cores). 0 (default): operands rounded to tf32,
 * fp32 accumulation — the image agrees with an fp32 evaluation to ~3e-3 of its scale. 1: split-tf32 ("3xTF32": every
 * convolution as three passes hi*hi + lo*hi + hi*lo accumulated in fp32) — fp32 accuracy (1e-4 against the fp32 reference
 * evaluation, gradients within 1e-3 of an fp64 backward) at three times the convolution time. Applies to
 * decode_image, its backward and the debug convolution hooks of this ctx. */
int splatb200_ctx_set_decoder_precise(splatb200_ctx* ctx, int32_t on);
int splatb200_view_decode_image(splatb200_view* v, const float* params, const float* embedding, float* image,
                                float* device_ms);
/* Backward of the decode ("Includes their backward passes"; gradient example SPEC.md:376). Needs the state
 * saved by the splatb200_view_decode_image call that followed the view's last forward (else SPLATB200_ERUNTIME, like
 * the rasterizer's backward without saved state). g_image: HOST, P x 3 = dL/dI. g_params: HOST,
 * splatb200_conv_decoder_params() floats, OVERWRITTEN with dL/dparams; g_embedding: HOST, 8 floats, overwritten
 * (SensorGrads::d_embedding, projection.hpp:207-222). g_blend: DEVICE, P x 16 (the blend buffer's row pitch: rgb, then d_f features) — dL/dF_rgb and
 * dL/dfeature are ADDED to it, so the buffer goes straight into splatb200_view_backward_device as the upstream gradient of the render.
 * Weight gradients and input gradients of the five convolutions run on the tensor cores as well. */
int splatb200_view_decode_image_backward(splatb200_view* v, const float* g_image, float* g_params, float* g_embedding,
                                         float* g_blend, float* device_ms);
/* test hook: one 3x3, 32 -> 32 convolution of the decoder on HOST arrays (x, y, res: H x W x 32 pixel-interleaved;
 * w: 9216 weights + 32 bias; res may be NULL). */
int splatb200_debug_conv3x3(splatb200_ctx* ctx, const float* x, int32_t H, int32_t W, const float* w, int32_t relu_in,
                            const float* res, float* y);
/* test hook: its gradients. g_y: H x W x 32 -> g_x (H x W x 32, masked by the ReLU of the input when relu_in),
 * g_w (9216 + 32, overwritten). */
int splatb200_debug_conv3x3_backward(splatb200_ctx* ctx, const float* x, int32_t H, int32_t W, const float* w,
                                     int32_t relu_in, const float* g_y, float* g_x, float* g_w);

/* ---- lidar returns -> rasterization points (SPEC.md:230-238 assign_points_to_tiles) ----
 * The producer of splatb200_view_create_lidar's `rays`. points_xyz: n x 3 world coordinates (ego-motion compensated),
 * timestamps: n capture times; HOST arrays. Each point is re-expressed relative to the sensor pose at its own capture
 * time (constant linear + angular velocity over the sweep), converted by Eq. 10 and mapped, with zero extent, to one
 * tile. Outputs (HOST, caller-allocated): tile[n] (-1: rejected — non-finite or at the sensor origin),
 * sph[n x 4] = (azimuth, elevation, t_l = timestamp - lidar.timestamp, range) per INPUT point, order[<= n] = the kept
 * points tile-major, ray_begin / ray_end [M_phi * M_omega] = its per-tile slices, counts[3] = kept, rejected, dropped.
 * train = 0 (evaluation): every valid point is kept, ascending input index inside a tile; tiles may hold more than
 * 256 points (rendered in additional passes). train = 1: a tile keeps the (at most) 256 points with the smallest
 * hash(seed, index), in (hash, index) order — the seeded shuffle-and-drop of PAPER.md:512. */
int splatb200_assign_points(splatb200_ctx* ctx, const splatb200_lidar* lidar, int64_t n, const float* points_xyz,
                            const float* timestamps, int32_t train, uint32_t seed, int64_t* tile, float* sph,
                            int64_t* order, int64_t* ray_begin, int64_t* ray_end, int64_t* counts);

/* ---- test hooks -----------------------------------------------------------------------------------
 * The hand-written depth sort + count scan of the binning stage on caller data (HOST arrays in and out): keys are
 * sorted as unsigned 32-bit integers, stably; order_out[k] = original position of the k-th smallest key;
 * offsets_out[k] = sum of counts[order_out[k']] over k' < k, k in [0, n] (mod 2^32). Exists so that the sort can be
 * tested on adversarial inputs (equal keys, partial tiles, n = 1) independently of the renderer. */
int splatb200_debug_depth_sort(splatb200_ctx* ctx, int64_t n, const uint32_t* keys, const uint32_t* counts,
                               uint32_t* order_out, uint32_t* offsets_out);

/* ---- reference-granularity entry points --------------------------------------------------------
 * One call per function the reference ships as code, HOST buffers in and out, for callers that switch
 * function by function (include/splat_b200.hpp wraps them in the reference's own types). All need a
 * forward(stop_after >= 1) on the view first; none is on the hot path. */
/* ComposedScene (scene.hpp:261-271) of compose_at_time (scene.hpp:273-308): N rows each, cov_w 9 floats
 * row-major; any pointer may be NULL */
int splatb200_view_composed(splatb200_view* v, float* mean_w, float* cov_w, float* vel_dyn_w, float* opacity);
/* std::vector<ProjectedGaussian> of project_camera / project_lidar (projection.hpp:28-40, 88-118, 140-174),
 * ascending source_index. Returns V (call with NULLs to size). fields25 per entry: mean2d 2, depth_key,
 * cov2d 4 row-major, velocity 3, aabb lo 2 + hi 2, conic 4 row-major, det_ratio, mu_sensor 3, rel_vel_sensor 3 */
int64_t splatb200_view_projected(splatb200_view* v, int64_t* source_index, float* fields25);
/* project_camera_backward / project_lidar_backward (projection.hpp:250-288, 322-357) over projected positions
 * [begin, end). g_mean2d (2), g_range (1), g_cov2d (4 row-major), g_velocity (3) have V rows indexed by projected
 * POSITION k, exactly what the shipped consumers read (projection.hpp:257-268, 329-344); NULL = zeros.
 * ComposeGrads (scene.hpp:313-323) g_mean_w (3), g_cov_w (9), g_vel_dyn_w (3) have N rows by source index and are
 * ACCUMULATED (+=); SensorGrads d_vel_lin / d_vel_ang accumulate in the view (splatb200_view_sensor_grads). */
int splatb200_view_project_backward(splatb200_view* v, const float* g_mean2d, const float* g_range, const float* g_cov2d,
                                    const float* g_velocity, int64_t begin, int64_t end, float* g_mean_w, float* g_cov_w,
                                    float* g_vel_dyn_w);
/* compose_backward (scene.hpp:386-458) over source indices [begin, end): ComposeGrads + g_opacity (activated,
 * N rows) in, accumulated into the ctx's SceneParamGrads (d_mean, d_scale_log, d_quat, d_opacity_logit, ActorGrad) */
int splatb200_view_compose_backward(splatb200_view* v, const float* g_mean_w, const float* g_cov_w, const float* g_vel_dyn_w,
                                    const float* g_opacity, int64_t begin, int64_t end);
/* both fused over the whole projected list: ProjectedGrads (projection.hpp:178-205) -> SceneParamGrads */
int splatb200_view_backward_projected(splatb200_view* v, const float* g_mean2d, const float* g_range, const float* g_cov2d,
                                      const float* g_velocity, const float* g_opacity);

/* Introspection for parity tests: copy a named intermediate to host. Returns the element count
 * (call with dst = NULL to size), or a negative error. int64 arrays: source_index, rect (x0,x1,y0,y1
 * per visible Gaussian, un-wrapped), isect_tile, isect_depth_bits, isect_src, tile_begin, tile_end,
 * n_contrib, last_idx. float arrays: mean2d(2), depth_key, cov2d(4), velocity(3), aabb(4), conic(4),
 * det_ratio, mu_sensor(3), rel_vel_sensor(3), blend(16), alpha, t_final, range_blend — projected
 * fields are compacted in ascending source_index like the reference's std::vector<ProjectedGaussian>
 * (projection.hpp:115,171). "packed_record" (26 floats per visible Gaussian, source order) is the record k_project
 * STORED for the compositing kernels, read back as it lies in HBM: mean2d.xy, velocity.xy | conic a, 2b, c,
 * rho = det_ratio * opacity | depth key, v_r | the 16 channel slots (camera: rgb + features; lidar: features). */
int64_t splatb200_view_array(splatb200_view* v, const char* name, void* dst);

#ifdef __cplusplus
}
#endif
#endif /* SPLAT_B200_H_ */
