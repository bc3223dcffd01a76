// kernels.h — host-callable launchers of the sm_100a kernels (one per stage of the hot path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "splat_device.cuh"

namespace sb {

// Per-device one-time setup of a kernel (cudaFuncSetAttribute is per device; a ctx may live on any GPU and views may be
// driven from several host threads): runs f() once for every device the calling site is reached on.
struct DeviceOnce {
  std::mutex m;
  uint64_t done[4] = {0, 0, 0, 0};  // up to 256 devices
  template <class F> void run(F&& f) {
    int d = 0;
    cudaGetDevice(&d);
    d &= 255;
    std::lock_guard<std::mutex> g(m);
    if (!((done[d >> 6] >> (d & 63)) & 1ull)) {
      f();
      done[d >> 6] |= 1ull << (d & 63);
    }
  }
};
// SM count of the current device (cached per device)
inline int device_sm_count() {
  static std::mutex m;
  static int sms[256] = {0};
  int d = 0;
  cudaGetDevice(&d);
  d &= 255;
  std::lock_guard<std::mutex> g(m);
  if (!sms[d]) cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d);
  return sms[d];
}

struct RasterOutDev {
  float* blend;        // P x 16
  float* alpha;        // P
  float* t_final;      // P  saved terminal transmittance
  float* range_blend;  // P  lidar: un-normalised sum w r_rs
  int32_t* n_contrib;  // P
  int32_t* last_idx;   // P  1-based tile-local list position of the last blended Gaussian
  uint8_t* hit;        // I  per list entry: bit w set if some query of warp w of the tile's CTA blended it (saved for
                       //    the backward pass, which then revisits only those entries)
  uint32_t* hit_list;  // I  scratch of the shared backward kernel: per tile the (position << 8 | hit byte) of its blended entries
  int hit_or;          // tiles with more than one ray pass: OR into (pre-zeroed) hit bytes instead of storing
  uint32_t* hit_rows;  // lidar v2 kernels (raster_lidar.cu), else null: the RAYS that blended each list entry, one 32-bit
                       //    word per (entry, warp of the tile's CTA) instead of the hit byte. One 2048-word block per 256
                       //    entries of a tile's list, block (tile_begin >> 8) + tile + (entry >> 8), laid out
                       //    [warp][entry & 255]; a word exists where bit `warp` of the entry's hit byte is set
  uint8_t* tile_wrap;  // T  lidar: 1 if some batch of the tile could not certify |azimuth difference| < pi (seam tiles);
                       //    the backward skips the wrap elsewhere. Written by the forward.
  // optional line-of-sight channel of a lidar view: los[q] = sum of alpha_i over the
  // blended Gaussians whose rolling-shutter range lies in front of los_cut[q] = r_p - eps; null = off
  const float* los_cut;  // P
  float* los;            // P
  const float* g_los;    // P  upstream gradient (backward)
  // optional fused lidar head: decode_lidar of the blended features as the compositing epilogue
  const float* head_w;   // lidar_head_params(d_f) parameters (device); null = off
  float* head_y;         // P x 2 (intensity, ray-drop probability)
  unsigned long long* stats;  // debug (SPLATB200_STATS=1), else null: 8 counters, see view_array "raster_stats"
};

// Raw per-Gaussian sums of the compositing backward, indexed by source index; consumed (and re-zeroed)
// by the projection backward. 12 floats = 48 bytes per Gaussian, in three 16-byte groups so that a warp sends each group
// as one vector RED and the projection backward reads / zeroes rows with 128-bit accesses:
//   [0..3] conic a, b, c; rho   [4..7] mean2d x, y; velocity x, y   [8..11] v_r, range (lidar), 2 pad
struct RasterGradDev {
  float* g;  // N x 12, zero between backward calls
};
constexpr int kRasterGradStride = 12;

// SceneParamGrads (scene.hpp:325-363) as one contiguous device buffer.
struct ParamGradDev {
  float* d_mean;
  float* d_scale_log;
  float* d_quat;
  float* d_opacity_logit;
  float* d_color;
  float* d_feature;
};

// Per-actor accumulators filled by the projection/compose backward, finished on the host with the
// SO(3) Jacobians (scene.hpp:428-453): g_mu_w (3), g_psi (3), d_vel_offset (6).
constexpr int kActorAccStride = 12;

// forward.cu
void launch_project(const Sensor& s, const SceneDev& sc, const ProjDev& p, cudaStream_t st);
// p.skip_feat = 1 in launch_project, then this once the colour / feature arrays are on the device
void launch_pack_feat(const Sensor& s, const SceneDev& sc, const ProjDev& p, cudaStream_t st);
// rays: one float4 per ray POSITION (azimuth, elevation, t_l, bit pattern of the original ray index), tile-major and
// azimuth-major inside a tile (prepared at view creation); tile_order: optional CTA -> tile permutation (longest
// worklists first), nullptr = identity
void launch_raster_fwd(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                       const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                       const uint32_t* tile_order, const RasterOutDev& out, cudaStream_t st, int tile_first = 0, int tile_count = -1);
// raster_lidar.cu: the lidar forward kernel, version 2 (lane = entry cull, bit transpose, lane = ray walk over its own
// candidates); needs out.hit_rows (lidar_hit_rows_words words) and tiles of at most 256 rays
size_t lidar_hit_rows_words(int64_t n_isect, int64_t n_tiles);
void launch_raster_fwd_lidar(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                             const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                             const uint32_t* tile_order, const RasterOutDev& out, cudaStream_t st, int tile_first = 0, int tile_count = -1);
constexpr int kDumpStride = 42;
void launch_project_dump(const Sensor& s, const SceneDev& sc, float* dump, cudaStream_t st);

// optim.cu (optimizer_step): Adam over the GaussianSet from the contiguous SceneParamGrads buffer
struct AdamGroups { int64_t begin[7]; };  // slices of the gradient buffer: mean, scale_log, quat, opacity_logit, color, feature
void launch_grad_finite(const float* g, int64_t n_floats, const AdamGroups& gr, int* bad6, cudaStream_t st);
void launch_actor_id_range(const int32_t* id, int64_t n, int* mn_mx /* device, preset to {INT_MAX, INT_MIN} */, cudaStream_t st);
void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float bc1, float bc2, const int* bad,
                 cudaStream_t st);

// decode.cu (decode_lidar): the lidar head over a view's blended features
int lidar_head_params(int d_f);
void launch_lidar_head_fwd(const float* w, int d_f, int64_t n_rays, const float4* rays, const float* blend16, float* y_out,
                           cudaStream_t st);
void launch_lidar_head_bwd(const float* w, int d_f, int64_t n_rays, const float4* rays, const float* blend16, const float* g_y,
                           float* g_blend16, float* g_w, cudaStream_t st);

// conv_decoder.cu (decode_image): the camera ConvDecoder on the tensor cores (tcgen05, tf32)
int conv_decoder_params();
// y = conv3x3(relu_in ? relu(x) : x; w[9216] + bias[32], reflect padding) (+ res); x, y, res: H x W x 32
// precise: split-tf32 ("3xTF32": hi hi + lo hi + hi lo in three passes) -> fp32 accuracy on the tf32 tensor cores
void launch_conv3x3(const float* x, int H, int W, const float* w, int relu_in, const float* res, float* y, int* err,
                    cudaStream_t st, int precise = 0);
// test hook: gradients of one convolution. gw (9248, +=), gx H x W x 32; wt: 9248 scratch, gext: (H+2)(W+2) x 32 scratch
void launch_conv3x3_backward(const float* x, int H, int W, const float* w, int relu_in, const float* gy, float* wt, float* gext,
                             float* gx, float* gw, int* err, cudaStream_t st, int precise = 0);
// blend (P x blend_stride: rgb, features) -> image P x 3; act: the six activations x0, h0, t1, h1, t2, h2 (P x 32 each,
// kept for the backward). Returns the launch count.
int launch_conv_decoder(const float* params, const float* emb, int H, int W, int d_f, float fx, float fy, float cx, float cy,
                        const float* blend, int blend_stride, float* const act[6], float* image, int* err, cudaStream_t st,
                        int precise = 0);
// g_image P x 3 -> g_params (+=), g_emb[8] (+=), g_blend P x blend_stride (+=: rgb and feature slots); g: three P x 32
// scratch buffers, gext: (H+2)(W+2) x 32, wt: 9248
int launch_conv_decoder_backward(const float* params, int H, int W, int d_f, const float* blend, int blend_stride,
                                 float* const act[6], const float* g_image, float* const g[3], float* gext, float* wt,
                                 float* g_params, float* g_emb, float* g_blend, int* err, cudaStream_t st, int precise = 0);

// assign.cu (assign_points_to_tiles): per-point tile key (0xffffffff = rejected), (phi, omega, t_l, range),
// shuffle hash, valid flag
void launch_assign_points(const Sensor& s, float timestamp, int64_t n, const float* xyz, const float* stamps, uint32_t seed,
                          uint32_t* key, float4* sph, uint32_t* hash, uint32_t* valid, cudaStream_t st);
void launch_gather_u32(int64_t n, const uint32_t* src, const uint32_t* idx, uint32_t* dst, cudaStream_t st);

// binning.cu (hand-written radix sort, scans, tile histogram — no library kernels)
size_t depth_sort_temp_bytes(int64_t n);
// stable sort of (dkey, position) by the 32-bit key; the sorted source indices land in order0 (dkey, dkey_alt, order1
// are scratch), then offsets[k] = sum_{k' < k} count[order0[k']] for k in [0, n]. Returns the number of kernels launched.
int launch_depth_sort_scan(uint32_t* dkey, uint32_t* dkey_alt, uint32_t* order0, uint32_t* order1, const uint32_t* count,
                           uint32_t* offsets, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st);
int super_shift();  // log2 of the block edge (in tiles) of the camera's two-level binning
size_t tile_hist_bytes(int tiles_x, int tiles_y);
// per-tile list lengths on the grid of 2^shift-tile blocks (shift 0: the tiles) from the tile rectangles ->
// tile_begin / tile_end (0, 0 for an empty tile), the CTA -> tile permutation (longest lists first; may be null),
// *total (device) and the digit histograms a sort by tile id needs (kept in tile_ws)
int launch_tile_counts(int64_t n, const ProjDev& p, int shift, int tiles_x, int tiles_y, int wrap_x, void* tile_ws,
                       uint32_t* tile_begin, uint32_t* tile_end, uint32_t* tile_order, int64_t* total, uint32_t* seg_first,
                       cudaStream_t st, bool want_hist = true);
size_t tile_sort_temp_bytes(int64_t cap, int64_t n_tiles);
// duplication (one (tile id, source index) pair per intersection, generated in depth order inside the first pass) +
// stable sort by tile id, on the grid of 2^shift-tile blocks. Returns which of vals0 / vals1 holds the sorted indices.
int launch_tile_sort(int64_t n, int64_t total, const uint32_t* offsets, const uint32_t* order, const ProjDev& p, int shift,
                     int tiles_x, int tiles_y, int wrap_x, const void* tile_ws, uint32_t* keys0, uint32_t* keys1, uint32_t* vals0,
                     uint32_t* vals1, void* temp, size_t temp_bytes, int* launches, cudaStream_t st);
// second level: block lists (sorted by block id, depth order inside), cut into segments (seg_first from
// launch_tile_counts on the block grid) -> tile lists
size_t expand_temp_bytes(int64_t cap_coarse, int n_super);
void launch_expand(int stiles_x, int stiles_y, int tiles_x, int tiles_y, int64_t n_coarse, const uint32_t* super_begin,
                   const uint32_t* super_end, const uint32_t* seg_first, const uint32_t* cvals, const ProjDev& p,
                   const uint32_t* tile_begin, void* temp, uint32_t* vals, cudaStream_t st);

// raster_bwd.cu
void launch_raster_bwd(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                       const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                       const uint32_t* tile_order, const RasterOutDev& fwd, const float* g_blend16, const float* g_alpha, const RasterGradDev& rg,
                       const ParamGradDev& pg, float* d_time_offset, cudaStream_t st, int tile_first = 0, int tile_count = -1);

// the lidar backward that pairs with launch_raster_fwd_lidar (reads fwd.hit_rows; tiles of at most 256 rays)
void launch_raster_bwd_lidar(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                             const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                             const uint32_t* tile_order, const RasterOutDev& fwd, const float* g_blend16, const float* g_alpha,
                             const RasterGradDev& rg, const ParamGradDev& pg, cudaStream_t st, int tile_first = 0, int tile_count = -1);

// project_bwd.cu
enum BwdMode { kFused = 0, kFromProjected = 1, kProjOnly = 2, kComposeOnly = 3 };
constexpr int kProjGradStride = 11;     // g_mean2d 2, g_range, g_cov2d 4, g_velocity 3, g_opacity
constexpr int kComposeGradStride = 15;  // g_mean_w 3, g_cov_w 9, g_vel_dyn_w 3
void launch_project_bwd_mode(int mode, const Sensor& s, const SceneDev& sc, const ProjDev& p, const ParamGradDev& pg,
                             float* sensor_grads6, float* actor_acc, const float* pgin, float* cg, int64_t i_lo,
                             int64_t i_hi, cudaStream_t st);
void launch_project_bwd(const Sensor& s, const SceneDev& sc, const ProjDev& p, const RasterGradDev& rg,
                        const ParamGradDev& pg, float* sensor_grads6, float* actor_acc, cudaStream_t st);

}  // namespace sb
