// raster_lidar.cu — lidar forward compositing, version 2 (compiled with --fmad=false like forward.cu: exact IEEE
// operation sequence of the CPU oracle). SPEC.md:295-313 (Eq. 3-6).
//
// Why a second kernel. A lidar footprint (~0.5 deg) covers 6-7 of a tile's 256 rays, a camera footprint most of a
// tile's pixels. The shared kernel (forward.cu: lane = ray, one list entry per warp iteration) therefore runs the
// lidar with ~8 of 32 lanes blending per visited entry (profiles/README.md), and 75% of its evaluate + blend issue
// slots are masked off. Here the roles flip twice per round of 32 list entries:
//
//   phase 1 (lane = ENTRY): each lane takes one of the warp's surviving entries and evaluates the exact fp32
//     quadratic form against the warp's 32 rays (ray data read as shared-memory broadcasts): ~11 instructions per
//     (entry, ray) pair, all lanes busy, no exponential, no blend. It keeps a pair when qf <= min(qform_max, the qf
//     beyond which rho exp(-qf/2) < alpha_min) — a superset of the pairs the exact evaluation blends, computed from
//     the bit-identical qf;
//   a 32 x 32 bit transpose (5 shuffle stages) turns the per-entry ray masks into per-ray entry masks;
//   phase 2 (lane = RAY): each lane walks ITS OWN set bits front to back — different lanes are at different
//     entries — with the exact oracle sequence (alpha_qform + alpha_finish + blend), gathering the records from
//     shared memory. Per-ray blending order is unchanged, so contributor counts, last_idx and every blended value
//     are bit-identical to the shared kernel and to the oracle.
//
// The lanes that blended a list entry are saved as per-lane bit rows (RasterOutDev::hit_rows, 32 B per list entry,
// lane-major inside a 256-entry block) next to the per-entry hit byte: the lidar backward kernel (raster_bwd.cu,
// k_raster_bwd_lidar) walks exactly those bits, again one lane per ray.
//
// Tiles with more than 256 rays (several ray passes) stay on the shared kernel: the host picks.
#include "kernels.h"
#include "raster_common.cuh"
#include "decode_device.cuh"

namespace sb {

// 32 x 32 bit-matrix transpose across the warp: lane l passes row l, receives column l.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? (((y & ~m) >> s) | (x & ~m)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

template <bool kLos, bool kHead>
__global__ void __launch_bounds__(256, 3)
k_raster_fwd_lidar(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
                   const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
                   const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
                   const uint32_t* __restrict__ tile_order, int tile_first, RasterOutDev out) {
  __shared__ float4 sA[256];
  __shared__ float4 sB[256];
  __shared__ float2 sC[256];
  __shared__ float4 sF[4 * 256];   // PLANAR: sF[c * 256 + j] (phase 2 gathers: 16-byte stride between entries)
  __shared__ float4 sRay[256];     // azimuth, elevation, t of the tile's rays (phase 1 broadcasts)
  __shared__ uint8_t sMask[256];
  __shared__ uint8_t sList[8][256];
  __shared__ uint32_t sRow[8][8][32];  // [warp][word][lane]: bit (j & 31) of word (j >> 5) = this lane blended batch entry j
  __shared__ uint32_t sHitW[8][8];     // [warp][word]: OR of the warp's rows
  __shared__ PatchBox sBox[8];
  __shared__ float sHead[kHead ? 640 : 1];  // lidar head parameters (fused epilogue)

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : tile_first + (int)blockIdx.x;
  const int tid = threadIdx.x;
  if (kHead) {  // visible to everyone after the first barrier below
    const int np = headdev::kHid * (s.d_f + 3) + headdev::kHid + 2 * headdev::kHid + 2;
    for (int i = tid; i < np; i += 256) sHead[i] = out.head_w[i];
  }
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];
  const int64_t q_begin = ray_begin[tile], q_end = ray_end[tile];  // at most 256 rays (the host guarantees it)
  bool any_wrap = false;

  const int64_t pos = q_begin + tid;
  const bool inside = pos < q_end;
  float qx = 0.0f, qy = 0.0f, t = 0.0f;
  int64_t pix = 0;
  if (inside) {
    const float4 r = rays[pos];
    qx = r.x; qy = r.y; t = r.z;
    pix = (int64_t)__float_as_uint(r.w);  // original ray index
  }
  sRay[tid] = make_float4(qx, qy, t, t);
  warp_patch_box<true>(inside, qx, qy, t, lane, &sBox[warp]);

  float T = 1.0f, range_acc = 0.0f, median = 0.0f;
  float los = 0.0f, los_cut = 0.0f;
  if (kLos && inside) los_cut = out.los_cut[pix];
  bool med_found = false;
  int n_contrib = 0, last_idx = 0;
  f32x2 acc2[kChannels / 2];  // the 16 blended channels as packed pairs
#pragma unroll
  for (int k = 0; k < kChannels / 2; ++k) acc2[k] = pack2(0.0f, 0.0f);
  const f32x2 q2 = pack2(qx, qy), t2 = pack2(t, t);
  bool done = !inside;
  __syncthreads();  // patch boxes, rays visible

  // rows of hit bits: 2048 words per 256-entry batch, [warp][word][lane]; block index (lb >> 8) + tile + batch never
  // collides between tiles (a partial last batch still owns a whole block)
  uint32_t* const rows_tile = out.hit_rows + ((size_t)(lb >> 8) + (size_t)tile) * 2048u;

  int64_t pending = -1;  // list position of the batch whose hit bytes are still to be written (CTA-uniform)
  auto flush_hits = [&]() {
    if (pending >= 0 && (uint32_t)pending + tid < le) {
      uint32_t h = 0u;
#pragma unroll
      for (int w = 0; w < 8; ++w) h |= ((sHitW[w][tid >> 5] >> (tid & 31)) & 1u) << w;
      out.hit[pending + tid] = (uint8_t)h;
    }
    pending = -1;
  };
  unsigned long long st_cand = 0ull, st_iter = 0ull;
  for (uint32_t base = lb; base < le; base += 256) {
    const bool all_done = __syncthreads_and(done);
    flush_hits();
    if (all_done) break;
    const uint32_t idx = base + tid;
    uint32_t mask = 0u, wrapm = 0u;
    if (idx < le) {
      const uint32_t src = vals[idx];
      const float4 gA = p.geomA[src], gB = p.geomB[src];
      mask = patch_mask<true>(gA, gB, sBox, s.qform_max, s.alpha_min, &wrapm);
      if (out.stats && !(fabsf(gA.x) + fabsf(gA.y) + fabsf(gA.z) + fabsf(gA.w) + fabsf(gB.x) + fabsf(gB.y) + fabsf(gB.z) + fabsf(gB.w) < 3.0e38f))
        atomicAdd(&out.stats[4], 1ull);  // SPEC.md:289 non-finite record counter
      if (mask) {
        sA[tid] = gA;
        sB[tid] = gB;
        sC[tid] = p.geomC[src];
#pragma unroll
        for (int k = 0; k < 4; ++k) sF[k * 256 + tid] = p.feat[4 * (size_t)src + k];
      }
    }
    sMask[tid] = (uint8_t)mask;
    const bool wrap = __syncthreads_or((mask & wrapm) != 0u) != 0;
    any_wrap |= wrap;
#pragma unroll
    for (int w = 0; w < 8; ++w) sRow[warp][w][lane] = 0u;
    pending = (int64_t)base;
    const unsigned live = __ballot_sync(0xffffffffu, !done);
    if (live == 0u) {  // this warp's 32 rays have saturated
      if (lane < 8) sHitW[warp][lane] = 0u;
      continue;
    }
    const int cnt = min(256u, le - base);
    const int n_w = warp_compact(sMask, cnt, warp, lane, sList[warp]);
    const uint8_t* lst = sList[warp];
    const float4* wray = &sRay[32 * warp];
    for (int k0 = 0; k0 < n_w; k0 += 32) {
      // ---- phase 1: lane = entry -------------------------------------------------------------
      uint32_t m = 0u;
      const int k = k0 + lane;
      if (k < n_w) {
        const int j = lst[k];
        const float4 gA = sA[j], gB = sB[j];
        // alpha = rho exp(-qf/2) < alpha_min  <=>  qf > 2 ln(rho / alpha_min); margins: 1% on rho, 0.02 on qf (the
        // evaluation's exp and this log are accurate to ~1e-6)
        float qcut = s.qform_max;
        const float rho = gB.w;
        if (s.alpha_min > 0.0f && rho > 0.0f && rho < 1e30f) qcut = fminf(qcut, 2.0f * __logf(rho * 1.01f / s.alpha_min) + 0.02f);
        if (!wrap) {  // certified: no azimuth difference of this batch leaves (-pi, pi) — packed pairs, 10 issue slots per ray
          const f32x2 m0 = pack2(gA.x, gA.y), vv = pack2(gA.z, gA.w);
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const float4 ry = wray[r];  // qx qy t t
            float dx, dy;
            const float qf = alpha_qform_packed(m0, vv, gB, pack2(ry.x, ry.y), pack2(ry.z, ry.w), dx, dy);
            if (qf <= qcut) m |= 1u << r;
          }
        } else {
#pragma unroll 4
          for (int r = 0; r < 32; ++r) {
            const float4 ry = wray[r];
            float dx, dy;
            const float qf = alpha_qform<true>(gA, gB, ry.x, ry.y, ry.z, dx, dy, true);
            if (qf <= qcut) m |= 1u << r;
          }
        }
        m &= live;
      }
      uint32_t bits = transpose32(m, lane);  // bit kk: list entry k0 + kk may blend with MY ray
      if (done) bits = 0u;                   // saturated in an earlier round of this batch (`live` is per batch)
      if (out.stats) st_cand += __popc(bits);
      // ---- phase 2: lane = ray, every lane walks its own candidates front to back ------------
      int trips = 0;
      while (bits != 0u) {
        const int kk = __ffs(bits) - 1;
        bits &= bits - 1u;
        ++trips;
        const int j = lst[k0 + kk];
        const float4 gA = sA[j], gB = sB[j];
        float dx, dy;
        const float qf = wrap ? alpha_qform<true>(gA, gB, qx, qy, t, dx, dy, true)
                              : alpha_qform_packed(pack2(gA.x, gA.y), pack2(gA.z, gA.w), gB, q2, t2, dx, dy);
        AlphaEval ev;
        if (alpha_finish(qf, gB.w, dx, dy, s.qform_max, s.alpha_clamp, s.alpha_min, ev)) {
          const float w = __fmul_rn(ev.alpha, T);
          const f32x2 ww = pack2(w, w);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 f4 = sF[c * 256 + j];
            acc2[2 * c] = fma2(pack2(f4.x, f4.y), ww, acc2[2 * c]);
            acc2[2 * c + 1] = fma2(pack2(f4.z, f4.w), ww, acc2[2 * c + 1]);
          }
          T = __fmul_rn(T, __fsub_rn(1.0f, ev.alpha));
          ++n_contrib;
          last_idx = (int)(base - lb) + j + 1;
          sRow[warp][j >> 5][lane] |= 1u << (j & 31);
          const float2 c2 = sC[j];
          const float r_rs = __fmaf_rn(c2.y, t, c2.x);
          range_acc = __fmaf_rn(r_rs, w, range_acc);
          if (kLos && r_rs < los_cut) los = __fadd_rn(los, ev.alpha);  // opacity in front of the measured range
          if (!med_found && T < 0.5f) { median = r_rs; med_found = true; }
          if (T < s.transmittance_min) { done = true; bits = 0u; }
        }
      }
      if (out.stats) st_iter += (unsigned long long)__reduce_max_sync(0xffffffffu, trips);
      __syncwarp();
    }
    // the warp's rows of this batch -> global, their OR -> the hit bytes
    uint32_t* rows_b = rows_tile + (size_t)((base - lb) >> 8) * 2048u + warp * 256;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t v = sRow[warp][w][lane];
      const uint32_t o = __reduce_or_sync(0xffffffffu, v);
      if (o) rows_b[w * 32 + lane] = v;
      if (lane == 0) sHitW[warp][w] = o;
    }
    if (out.stats && lane == 0) {
      atomicAdd(&out.stats[1], (unsigned long long)n_w);
      if (warp == 0) atomicAdd(&out.stats[0], (unsigned long long)cnt);
    }
  }
  if (out.stats) {
    st_cand = __reduce_add_sync(0xffffffffu, (unsigned)st_cand);
    if (lane == 0) {
      atomicAdd(&out.stats[2], st_cand);
      atomicAdd(&out.stats[3], st_iter);
    }
  }

  if (inside) {
    float acc[kChannels];
#pragma unroll
    for (int k = 0; k < kChannels / 2; ++k) unpack2(acc2[k], acc[2 * k], acc[2 * k + 1]);
    const float A = __fsub_rn(1.0f, T);
    acc[13] = (A > 1e-6f) ? __fdiv_rn(range_acc, A) : range_acc;
    acc[14] = median;
    acc[15] = A;
    out.range_blend[pix] = range_acc;
    if (kLos) out.los[pix] = los;
    if (kHead) {  // decode_lidar on the blended features, while they are still in registers
      float x[headdev::kInMax], y[2], h[headdev::kHid];
#pragma unroll
      for (int k = 0; k < 13; ++k) x[k] = acc[k];
      headdev::ray_dir(qx, qy, x + s.d_f);
      headdev::head_forward(sHead, s.d_f + 3, x, y, h);
      out.head_y[2 * pix] = y[0];
      out.head_y[2 * pix + 1] = y[1];
    }
    float4* o4 = reinterpret_cast<float4*>(out.blend + 16 * pix);
#pragma unroll
    for (int k = 0; k < 4; ++k) o4[k] = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
    out.alpha[pix] = A;
    out.t_final[pix] = T;
    out.n_contrib[pix] = n_contrib;
    out.last_idx[pix] = last_idx;
  }
  __syncthreads();
  flush_hits();  // the last batch of a list that ended before every ray saturated
  if (tid == 0) out.tile_wrap[tile] = any_wrap ? 1 : 0;
}

size_t lidar_hit_rows_words(int64_t n_isect, int64_t n_tiles) { return (size_t)((n_isect >> 8) + n_tiles + 2) * 2048u; }

void launch_raster_fwd_lidar(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                             const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                             const uint32_t* tile_order, const RasterOutDev& out, cudaStream_t st, int tile_first, int tile_count) {
  const int tiles = tile_count < 0 ? s.tiles_x * s.tiles_y : tile_count;
  if (tiles <= 0) return;
  const uint32_t* order = tile_count < 0 ? tile_order : nullptr;
  if (tile_count < 0) tile_first = 0;
  if (out.los_cut && out.head_w)
    k_raster_fwd_lidar<true, true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.head_w)
    k_raster_fwd_lidar<false, true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.los_cut)
    k_raster_fwd_lidar<true, false><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else
    k_raster_fwd_lidar<false, false><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
}

}  // namespace sb
