// raster_bwd.cu — compositing backward.
//
// One CTA per tile, the same query->thread mapping as the forward kernel. Each thread restarts from
// its saved terminal transmittance and walks the tile's list back to front, recomputing
// alpha with the very same instruction sequence as the forward pass (raster_common.cuh), so it
// revisits exactly the Gaussians that were blended.
//
// With w_i = alpha_i T_i, out_c = sum_i f_ic w_i, A = 1 - T_final:
//   dL/df_ic     = w_i g_c
//   dL/dalpha_i  = T_i sum_c g_c f_ic  -  (S_i - g_A T_final) / (1 - alpha_i),   S_i = sum_c g_c sum_{j>i} f_jc w_j
// S_i is carried as ONE scalar per thread (S += w_i * sum_c g_c f_ic), not one suffix per channel.
// For lidar the rolling-shutter range r_rs = r + v_r t is one more blended channel whose upstream is
// dL/d(range_blend); expected = range_blend / A feeds both.
//
// Reduction to per-Gaussian gradients (north_star (4): warp-aggregated atomics): the 26 per-pair
// values are reduced over the 32 lanes of a warp with a transposing butterfly (31 shuffles: after
// step k each lane keeps half of its values), which leaves value l on lane l; 26 lanes then issue
// ONE shared-memory atomic each into the batch's accumulator, and the accumulator is flushed to
// global memory with one RED per (tile, Gaussian, value) at the end of the batch. Warps in which no
// lane blends the Gaussian skip everything after the ballot.
#include "kernels.h"
#include "raster_common.cuh"

namespace sb {

constexpr int kRed = 26;  // 16 channel grads + conic 3 + mean2d 2 + vel 3 + rho + range

// In: v[0..31] per lane. Out: v[0] on lane l = sum over lanes of v[l].
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int k = 0; k < half; ++k) {
      const float send = hi ? v[k] : v[k + half];
      const float keep = hi ? v[k + half] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return v[0];
}

template <bool kCamera>
__global__ void __launch_bounds__(256, 2)
k_raster_bwd(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
             const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
             const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
             const uint32_t* __restrict__ tile_order, RasterOutDev fwd, const float* __restrict__ g_blend16,
             const float* __restrict__ g_alpha, RasterGradDev rg, ParamGradDev pg, float* __restrict__ d_time_offset) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* sA = reinterpret_cast<float4*>(smem_raw);  // 256
  float4* sB = sA + 256;                             // 256
  float4* sF = sB + 256;                             // 1024
  float2* sC = reinterpret_cast<float2*>(sF + 1024); // 256
  float* sG = reinterpret_cast<float*>(sC + 256);    // 256 * kRed
  uint32_t* sSrc = reinterpret_cast<uint32_t*>(sG + 256 * kRed);  // 256
  uint8_t* sMask = reinterpret_cast<uint8_t*>(sSrc + 256);        // 256
  uint8_t* sListAll = sMask + 256;                                // 8 x 256
  PatchBox* sBox = reinterpret_cast<PatchBox*>(sListAll + 8 * 256);  // 8
  __shared__ int s_max_last;
  __shared__ float s_dt[8];

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint8_t* sList = sListAll + 256 * warp;
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];
  if (le <= lb) return;

  for (int x = tid; x < 256 * kRed; x += 256) sG[x] = 0.0f;

  int64_t q_begin = 0, q_end = 1;
  if (!kCamera) { q_begin = ray_begin[tile]; q_end = ray_end[tile]; }
  float dt_local = 0.0f;

  for (int64_t q_base = q_begin; q_base < q_end; q_base += 256) {
    bool inside;
    int64_t pix;
    float qx, qy, t;
    if (kCamera) {  // same query -> thread mapping as the forward kernel
      const int px = (tile % s.tiles_x) * kTile + (warp & 1) * 8 + (lane & 7);
      const int py = (tile / s.tiles_x) * kTile + (warp >> 1) * 4 + (lane >> 3);
      inside = px < s.width && py < s.height;
      pix = (int64_t)py * s.width + px;
      qx = (float)px + 0.5f;
      qy = (float)py + 0.5f;
      t = __fadd_rn(__fmul_rn(__fsub_rn(__fdiv_rn((float)py, (float)s.height), 0.5f), s.shutter), s.time_offset);
    } else {
      const int64_t pos = q_base + tid;
      inside = pos < q_end;
      qx = qy = t = 0.0f;
      pix = 0;
      if (inside) {
        const float4 r = rays[pos];
        qx = r.x; qy = r.y; t = r.z;
        pix = (int64_t)__float_as_uint(r.w);
      }
    }
    warp_patch_box<!kCamera>(inside, qx, qy, t, lane, &sBox[warp]);

    int last = 0;
    float T = 1.0f, K = 0.0f, g_D = 0.0f;
    float g_out[kChannels];
#pragma unroll
    for (int k = 0; k < kChannels; ++k) g_out[k] = 0.0f;
    if (inside) {
      last = fwd.last_idx[pix];
      T = fwd.t_final[pix];
      const float4* g4 = reinterpret_cast<const float4*>(g_blend16 + 16 * pix);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 g = g4[k];
        g_out[4 * k] = g.x; g_out[4 * k + 1] = g.y; g_out[4 * k + 2] = g.z; g_out[4 * k + 3] = g.w;
      }
      float g_acc = g_alpha[pix];
      if (!kCamera) {
        const float A = 1.0f - T;
        if (A > 1e-6f) {  // expected = D / A
          g_D = g_out[13] / A;
          g_acc += -g_out[13] * (fwd.range_blend[pix] / A) / A;
        } else {
          g_D = g_out[13];
        }
      }
#pragma unroll
      for (int k = 0; k < kChannels; ++k)
        if (k >= s.channels) g_out[k] = 0.0f;
      K = g_acc * T;
    }
    float S = 0.0f;  // sum_c g_c * suffix_c (+ g_D * suffix_r)

    // warp and block maxima of `last`
    if (tid == 0) s_max_last = 0;
    __syncthreads();
    int warp_last = last;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) warp_last = max(warp_last, __shfl_xor_sync(0xffffffffu, warp_last, o));
    if (lane == 0 && warp_last > 0) atomicMax(&s_max_last, warp_last);
    __syncthreads();  // also publishes the patch boxes
    const int max_last = s_max_last;

    for (int batch = (max_last - 1) / 256; batch >= 0 && max_last > 0; --batch) {
      const int bstart = batch * 256;
      const int cnt = min(256, max_last - bstart);
      uint32_t mask = 0u;
      if (tid < cnt) {
        const uint32_t src = vals[lb + bstart + tid];
        const float4 gA = p.geomA[src], gB = p.geomB[src];
        mask = patch_mask<!kCamera>(gA, gB, sBox, s.qform_max, s.alpha_min);
        if (mask) {
          sSrc[tid] = src;
          sA[tid] = gA;
          sB[tid] = gB;
          if (!kCamera) sC[tid] = p.geomC[src];
#pragma unroll
          for (int k = 0; k < 4; ++k) sF[4 * tid + k] = p.feat[4 * (size_t)src + k];
        }
      }
      sMask[tid] = (uint8_t)mask;
      __syncthreads();

      bool touched = false;
      if (warp_last > bstart) {
        const int n_w = warp_compact(sMask, cnt, warp, lane, sList);
        for (int k = n_w - 1; k >= 0; --k) {
          const int jj = sList[k];
          const int pos = bstart + jj;
          AlphaEval ev;
          bool valid = false;
          float4 gA, gB;
          if (pos < last) {
            gA = sA[jj];
            gB = sB[jj];
            valid = evaluate_alpha<!kCamera>(gA, gB, qx, qy, t, s.qform_max, s.alpha_clamp, s.alpha_min, ev);
          }
          if (!__any_sync(0xffffffffu, valid)) continue;
          touched = true;

          float v[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0.0f;
          if (valid) {
            const float one_m = 1.0f - ev.alpha;
            const float inv = 1.0f / one_m;
            T = T * inv;  // transmittance in front of this Gaussian
            const float w = ev.alpha * T;
            float dotgf = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 f4 = sF[4 * jj + c];
              dotgf = fmaf(g_out[4 * c], f4.x, dotgf);
              dotgf = fmaf(g_out[4 * c + 1], f4.y, dotgf);
              dotgf = fmaf(g_out[4 * c + 2], f4.z, dotgf);
              dotgf = fmaf(g_out[4 * c + 3], f4.w, dotgf);
            }
#pragma unroll
            for (int c = 0; c < kChannels; ++c) v[c] = w * g_out[c];
            if (!kCamera) {
              const float2 c2 = sC[jj];
              const float r_rs = fmaf(c2.y, t, c2.x);
              dotgf = fmaf(g_D, r_rs, dotgf);
              v[25] = g_D * w;      // d/d range
              v[23] = g_D * w * t;  // d/d v_r
            }
            const float g_a = dotgf * T + (K - S) * inv;
            S = fmaf(w, dotgf, S);
            if (!ev.clamped) {  // alpha == alpha_clamp is constant in every parameter
              const float g_sigma = -ev.alpha * g_a;  // alpha = rho exp(-sigma), sigma = qf / 2
              const float gdx = g_sigma * (gB.x * ev.dx + 0.5f * gB.y * ev.dy);
              const float gdy = g_sigma * (gB.z * ev.dy + 0.5f * gB.y * ev.dx);
              v[16] = g_sigma * 0.5f * ev.dx * ev.dx;
              v[17] = g_sigma * 0.5f * ev.dx * ev.dy;
              v[18] = g_sigma * 0.5f * ev.dy * ev.dy;
              v[19] = -gdx;
              v[20] = -gdy;
              v[21] = -t * gdx;
              v[22] = -t * gdy;
              v[24] = ev.gauss * g_a;  // d/d rho
              dt_local -= gA.z * gdx + gA.w * gdy;
            }
          }
          const float r = warp_transpose_reduce(v, lane);
          if (lane < kRed && r != 0.0f) atomicAdd(&sG[jj * kRed + lane], r);
        }
      }
      // flush the batch accumulator: one RED per (tile, Gaussian, value); skipped when no warp blended anything
      if (__syncthreads_or(touched)) {
        for (int x = tid; x < cnt * kRed; x += 256) {
          const float val = sG[x];
          if (val != 0.0f) {
            const int jj = x / kRed, l = x - jj * kRed;
            const size_t src = sSrc[jj];
            float* dst;
            if (l >= 16) dst = rg.g + kRasterGradStride * src + (l - 16);
            else if (kCamera) dst = (l < 3) ? pg.d_color + 3 * src + l : pg.d_feature + (size_t)s.d_f * src + (l - 3);
            else dst = pg.d_feature + (size_t)s.d_f * src + l;
            atomicAdd(dst, val);
            sG[x] = 0.0f;
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();  // patch boxes / staging are reused by the next ray pass
  }

  if (kCamera) {  // SensorGrads.d_time_offset (projection.hpp:210)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) dt_local += __shfl_xor_sync(0xffffffffu, dt_local, o);
    if (lane == 0) s_dt[tid >> 5] = dt_local;
    __syncthreads();
    if (tid == 0) {
      float tot = 0.0f;
      for (int k = 0; k < 8; ++k) tot += s_dt[k];
      if (tot != 0.0f) atomicAdd(d_time_offset, tot);
    }
  }
}

constexpr size_t kBwdSmem = 256 * 16 * 2 + 1024 * 16 + 256 * 8 + 256 * kRed * 4 + 256 * 4 + 256 + 8 * 256 + 8 * sizeof(PatchBox);

void launch_raster_bwd(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                       const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                       const uint32_t* tile_order, const RasterOutDev& fwd, const float* g_blend16, const float* g_alpha,
                       const RasterGradDev& rg, const ParamGradDev& pg, float* d_time_offset, cudaStream_t st) {
  const int tiles = s.tiles_x * s.tiles_y;
  if (tiles == 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_raster_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
    cudaFuncSetAttribute(k_raster_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
    attr_set = true;
  }
  if (s.is_camera)
    k_raster_bwd<true><<<tiles, 256, kBwdSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                     fwd, g_blend16, g_alpha, rg, pg, d_time_offset);
  else
    k_raster_bwd<false><<<tiles, 256, kBwdSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                      fwd, g_blend16, g_alpha, rg, pg, d_time_offset);
}

}  // namespace sb
