// forward.cu — forward kernels of the hot path (compiled with --fmad=false, see splat_device.cuh).
//
//   k_project<camera|lidar>   compose_at_time + project_camera/project_lidar fused, one thread per
//                             Gaussian: scene.hpp:273-308, projection.hpp:88-118 / 140-174, plus the
//                             tile rectangle and the packed compositing record.
//   (tile binning — depth sort, duplication, tile sort, tile ranges — lives in binning.cu)
//   k_raster_fwd<camera|lidar> per-tile front-to-back compositing (Eq. 3-6).
#include <cstddef>

#include "kernels.h"
#include "raster_common.cuh"
#include "decode_device.cuh"

namespace sb {

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// ------------------------------------------------------------------------------------------------
// K1/K2: fused compose + projection + tile rectangle
// ------------------------------------------------------------------------------------------------
template <bool kCamera>
__device__ __forceinline__ void pack_channels(const SceneDev& sc, const ProjDev& p, int64_t i) {
  float ch[kChannels];
#pragma unroll
  for (int k = 0; k < kChannels; ++k) ch[k] = 0.0f;
  int o = 0;
  if (kCamera) {
#pragma unroll
    for (int k = 0; k < 3; ++k) ch[o++] = sc.color[3 * i + k];
  }
  for (int k = 0; k < sc.d_f; ++k) ch[o + k] = sc.feature[(int64_t)sc.d_f * i + k];
#pragma unroll
  for (int k = 0; k < 4; ++k) p.feat[4 * i + k] = make_float4(ch[4 * k], ch[4 * k + 1], ch[4 * k + 2], ch[4 * k + 3]);
}

template <bool kCamera>
__global__ void __launch_bounds__(256) k_project(const __grid_constant__ Sensor s, SceneDev sc, ProjDev p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sc.n) return;
  // every parameter row of this Gaussian is requested up front: the loads below sit at their first uses, spread over
  // the projection arithmetic, and would otherwise pay one L2 / DRAM round trip each
  prefetch_l1(sc.scale_log + 3 * i);
  prefetch_l1(sc.quat + 4 * i);
  prefetch_l1(sc.opacity_logit + i);
  prefetch_l1(sc.actor_id + i);
  Fwd f;
  compose_one(sc, i, f);
  if (kCamera) project_camera_one(s, f);
  else project_lidar_one(s, f);
  if (!f.visible) {
    p.count[i] = 0u;
    if (p.ccount) p.ccount[i] = 0u;
    p.dkey[i] = 0xffffffffu;
    return;
  }
  const int4 r = kCamera ? image_tile_range(f, s.tiles_x, s.tiles_y) : lidar_tile_range(f, s);
  const int w = r.y - r.x, h = r.w - r.z;
  const uint32_t cnt = (w > 0 && h > 0) ? (uint32_t)w * (uint32_t)h : 0u;
  p.count[i] = cnt;
  if (p.ccount) {  // blocks of 2^cshift x 2^cshift tiles the rectangle touches (first level of the two-level binning)
    const int up = (1 << p.cshift) - 1;
    const int cw = ((r.y + up) >> p.cshift) - (r.x >> p.cshift), ch = ((r.w + up) >> p.cshift) - (r.z >> p.cshift);
    p.ccount[i] = cnt ? (uint32_t)cw * (uint32_t)ch : 0u;
  }
  p.dkey[i] = cnt ? __float_as_uint(f.depth) : 0xffffffffu;  // depth > 0: the bit pattern orders like the value
  p.rect[i] = r;
  p.geomA[i] = make_float4(f.mean2d[0], f.mean2d[1], f.vel[0], f.vel[1]);
  p.geomB[i] = make_float4(f.conic[0], f.conic[1] + f.conic[2], f.conic[3], f.det_ratio * f.opacity);
  p.geomC[i] = make_float2(f.depth, f.vel[2]);
  if (!p.skip_feat) pack_channels<kCamera>(sc, p, i);
}

// The blended channels of one visible Gaussian (camera: rgb + features, lidar: features; zero padded to 16), packed next
// to its compositing record. Part of k_project, or on its own (k_pack_feat) when the scene's colour / feature arrays
// arrive after its geometry (splatb200_scene_upload_async).
template <bool kCamera>
__global__ void __launch_bounds__(256) k_pack_feat(SceneDev sc, ProjDev p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sc.n || p.count[i] == 0u) return;
  pack_channels<kCamera>(sc, p, i);
}

void launch_project(const Sensor& s, const SceneDev& sc, const ProjDev& p, cudaStream_t st) {
  if (sc.n == 0) return;
  const int threads = 256;
  const unsigned blocks = (unsigned)((sc.n + threads - 1) / threads);
  if (s.is_camera) k_project<true><<<blocks, threads, 0, st>>>(s, sc, p);
  else k_project<false><<<blocks, threads, 0, st>>>(s, sc, p);
}
void launch_pack_feat(const Sensor& s, const SceneDev& sc, const ProjDev& p, cudaStream_t st) {
  if (sc.n == 0) return;
  const unsigned blocks = (unsigned)((sc.n + 255) / 256);
  if (s.is_camera) k_pack_feat<true><<<blocks, 256, 0, st>>>(sc, p);
  else k_pack_feat<false><<<blocks, 256, 0, st>>>(sc, p);
}

// ------------------------------------------------------------------------------------------------
// K5/K6: forward compositing. One CTA of 256 threads per tile: 16x16 pixels, or up to 256 rays of a
// 32x8 lidar tile (more than 256 rays => additional passes over the list). Each warp owns
// a compact patch of 32 queries (camera: 8x4 pixels; lidar: 32 consecutive rays of the per-tile
// azimuth-major order, i.e. 4 azimuth bins x 8 beams of a grid sweep).
//
// Lidar culling is hierarchical. A warp's 32 rays form four GROUPS of 8 lanes (8 consecutive rays of the per-tile patch
// order, which the host makes compact). After the CTA-wide test against the 8 warp patches and the warp's compaction,
// every surviving entry is tested against the warp's four group boxes (same rigorous bound, one lane per entry) and
// appended to the lists of the groups that can see it; the four groups then walk their OWN lists in lock step — a lane
// reads the entry its group is at. The loop runs max(group list) iterations instead of the warp list's (1.39M instead
// of 2.38M per north-star sweep). The camera walks the warp list (measured: group lists cost it 35%).
//
// The tile's depth-sorted slice is staged through shared memory 256 Gaussians at a time. The staging
// thread tests its Gaussian against the 8 patch boxes (raster_common.cuh: a rigorous lower bound of the
// fp32 quadratic form, so no blended pair is ever dropped) and fetches the 112-byte record only if some
// patch can see it; every warp compacts the batch to its own visible entries with ballots and walks
// those front to back with broadcast shared-memory reads. The evaluation itself is the exact IEEE
// sequence of the oracle, so contributor counts stay bit-identical. The batch loop ends when every
// query of the tile has saturated (T < transmittance_min): one __syncthreads_and per batch; a warp whose
// 32 queries have all saturated stops evaluating on its own.
// ------------------------------------------------------------------------------------------------
template <bool kCamera, bool kLos = false, bool kHead = false>
__global__ void __launch_bounds__(256, kCamera ? 4 : 3)
k_raster_fwd(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
             const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
             const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
             const uint32_t* __restrict__ tile_order, int tile_first, RasterOutDev out) {
  // one struct: the camera's walk addresses every array relative to ONE pinned base register (raster_common.cuh: smem_addr)
  struct Staged {
    float4 sA[256];
    float4 sB[256];
    float4 sF[256 * 4];
    float2 sC[256];
    alignas(8) uint8_t sHit[8][256];  // [warp][batch entry]: some lane of the warp blended it
    uint8_t sList[8][256];
    uint8_t sMask[256];
  };
  __shared__ __align__(16) Staged sm;
  auto& sA = sm.sA;
  auto& sB = sm.sB;
  auto& sC = sm.sC;
  auto& sF = sm.sF;
  auto& sMask = sm.sMask;
  auto& sList = sm.sList;
  auto& sHit = sm.sHit;
  __shared__ uint8_t sSub[kCamera ? 1 : 8][4][kCamera ? 1 : 256];  // lidar, [warp][group]: the group's entries of the batch, in list order
  __shared__ PatchBox sBox[9];  // 8 warp patches + the tile's box (patch_mask_fast)
  __shared__ PatchBox sGBox[kCamera ? 1 : 8][4];                   // lidar: boxes of the 8-lane groups
  __shared__ float sHead[(!kCamera && kHead) ? 640 : 1];  // lidar head parameters (fused epilogue)

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : tile_first + (int)blockIdx.x;
  const int tid = threadIdx.x;
  if (!kCamera && kHead) {  // visible to everyone after the first barrier below
    const int np = headdev::kHid * (s.d_f + 3) + headdev::kHid + 2 * headdev::kHid + 2;
    for (int i = tid; i < np; i += 256) sHead[i] = out.head_w[i];
  }
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];

  int64_t q_begin = 0, q_end = 1;  // camera: single pass
  if (!kCamera) { q_begin = ray_begin[tile]; q_end = ray_end[tile]; }
  bool any_wrap = false;  // lidar, CTA-uniform: some batch needed the azimuth wrap

  for (int64_t q_base = q_begin; q_base < q_end; q_base += 256) {
    bool inside;
    int64_t pix;
    float qx, qy, t;
    if (kCamera) {
      const int px = (tile % s.tiles_x) * kTile + (warp & 1) * 8 + (lane & 7);
      const int py = (tile / s.tiles_x) * kTile + (warp >> 1) * 4 + (lane >> 3);
      inside = px < s.width && py < s.height;
      pix = (int64_t)py * s.width + px;
      qx = (float)px + 0.5f;
      qy = (float)py + 0.5f;
      t = ((float)py / (float)s.height - 0.5f) * s.shutter + s.time_offset;  // Eq. 3
    } else {
      const int64_t pos = q_base + tid;
      inside = pos < q_end;
      qx = qy = t = 0.0f;
      pix = 0;
      if (inside) {
        const float4 r = rays[pos];
        qx = r.x; qy = r.y; t = r.z;
        pix = (int64_t)__float_as_uint(r.w);  // original ray index
      }
    }
    warp_patch_box<!kCamera>(inside, qx, qy, t, lane, &sBox[warp]);
    bool group_live = true;
    if (!kCamera) {
      group_patch_box<true>(inside, qx, qy, t, lane, sGBox[warp]);
      group_live = ((__ballot_sync(0xffffffffu, inside) >> (lane & 24)) & 0xffu) != 0u;  // some ray in my group
    }

    float T = 1.0f, range_acc = 0.0f, median = 0.0f;
    constexpr bool los_on = !kCamera && kLos;  // a separate instantiation: the plain lidar kernel pays nothing for it
    float los = 0.0f, los_cut = 0.0f;
    if (los_on && inside) los_cut = out.los_cut[pix];
    bool med_found = false;
    int n_contrib = 0, last_idx = 0;
    f32x2 acc2[kChannels / 2];  // the 16 blended channels as packed pairs (FFMA2: two IEEE fmas per issue slot)
#pragma unroll
    for (int k = 0; k < kChannels / 2; ++k) acc2[k] = pack2(0.0f, 0.0f);
    const f32x2 q2 = pack2(qx, qy), t2 = pack2(t, t);
    bool done = !inside;
    __syncthreads();  // patch boxes visible
    if (tid == 0) tile_patch_box(sBox);  // published by the first barrier of the batch loop

    // the hit bytes of a batch are folded and written once every warp is through it, i.e. after the next barrier
    int64_t pending = -1;  // list position of the batch whose hit bytes are still in shared memory (CTA-uniform)
    auto flush_hits = [&]() {
      if (pending >= 0 && (uint32_t)pending + tid < le) {
        uint32_t h = 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) h |= (uint32_t)(sHit[w][tid] != 0) << w;
        uint8_t* dst = out.hit + pending + tid;
        *dst = out.hit_or ? (uint8_t)(*dst | h) : (uint8_t)h;
      }
      pending = -1;
    };
    for (uint32_t base = lb; base < le; base += 256) {
      const bool all_done = __syncthreads_and(done);
      flush_hits();
      if (all_done) break;
      const uint32_t idx = base + tid;
      uint32_t mask = 0u, wrapm = 0u;
      if (idx < le) {
        const uint32_t src = vals[idx];
        const float4 gA = p.geomA[src], gB = p.geomB[src];
        mask = patch_mask_fast<!kCamera>(gA, gB, sBox, s.qform_max, s.alpha_min, &wrapm);
        // SPEC.md:289 "non-finite alpha -> Gaussian skipped, counter incremented": a record with a non-finite field makes
        // every alpha it produces non-finite (skipped by the !(qf <= qform_max) / !(alpha >= alpha_min) tests); counted per
        // staged entry when the debug counters are on
        if (out.stats && !(fabsf(gA.x) + fabsf(gA.y) + fabsf(gA.z) + fabsf(gA.w) + fabsf(gB.x) + fabsf(gB.y) + fabsf(gB.z) + fabsf(gB.w) < 3.0e38f))
          atomicAdd(&out.stats[4], 1ull);
        if (mask) {
          sA[tid] = gA;
          sB[tid] = gB;
          if (!kCamera) sC[tid] = p.geomC[src];
#pragma unroll
          for (int k = 0; k < 4; ++k) sF[4 * tid + k] = p.feat[4 * (size_t)src + k];
        }
      }
      sMask[tid] = (uint8_t)mask;
      // lidar: does any (entry, patch) pair of this batch need the azimuth wrap? (rare: tiles at the seam)
      const bool wrap = kCamera ? (__syncthreads(), false) : __syncthreads_or((mask & wrapm) != 0u) != 0;
      any_wrap |= wrap;
      reinterpret_cast<uint2*>(sHit[warp])[lane] = make_uint2(0u, 0u);  // 256 bytes per warp
      pending = (int64_t)base;
      // (fetching the next batch's list entry one batch ahead and prefetching its records into L2 was measured: no
      // gain for the lidar, +4% on the issue-bound camera kernel; the backward kernels keep it, -3..4%)
      if (__all_sync(0xffffffffu, done)) continue;  // this warp's 32 queries have saturated
      __syncwarp();
      const int cnt = min(256u, le - base);
      const int n_w = warp_compact(sMask, cnt, warp, lane, sList[warp]);
      const uint8_t* lst = sList[warp];
      // second level (lidar): the warp's survivors against its four group boxes -> one list per group (order preserved)
      int n_g0 = 0, n_g1 = 0, n_g2 = 0, n_g3 = 0;
      for (int k0 = 0; !kCamera && k0 < n_w; k0 += 32) {
        const int k = k0 + lane;
        uint32_t gm = 0u;
        int j = 0;
        if (k < n_w) {
          j = lst[k];
          gm = patch_mask<!kCamera, 0, 4>(sA[j], sB[j], sGBox[warp], s.qform_max, s.alpha_min);
        }
        const unsigned lt = (1u << lane) - 1u;
        unsigned bal = __ballot_sync(0xffffffffu, gm & 1u);
        if (gm & 1u) sSub[warp][0][n_g0 + __popc(bal & lt)] = (uint8_t)j;
        n_g0 += __popc(bal);
        bal = __ballot_sync(0xffffffffu, gm & 2u);
        if (gm & 2u) sSub[warp][1][n_g1 + __popc(bal & lt)] = (uint8_t)j;
        n_g1 += __popc(bal);
        bal = __ballot_sync(0xffffffffu, gm & 4u);
        if (gm & 4u) sSub[warp][2][n_g2 + __popc(bal & lt)] = (uint8_t)j;
        n_g2 += __popc(bal);
        bal = __ballot_sync(0xffffffffu, gm & 8u);
        if (gm & 8u) sSub[warp][3][n_g3 + __popc(bal & lt)] = (uint8_t)j;
        n_g3 += __popc(bal);
      }
      __syncwarp();
      const int grp = lane >> 3;
      const int my_n = kCamera ? n_w : (group_live ? (grp == 0 ? n_g0 : grp == 1 ? n_g1 : grp == 2 ? n_g2 : n_g3) : 0);
      int max_n = my_n;
      if (!kCamera) {
#pragma unroll
        for (int o = 16; o >= 8; o >>= 1) max_n = max(max_n, __shfl_xor_sync(0xffffffffu, max_n, o));
      }
      const uint8_t* mine = kCamera ? lst : sSub[warp][grp];
      if (out.stats && lane == 0) {
        atomicAdd(&out.stats[1], (unsigned long long)n_w);
        atomicAdd(&out.stats[2], (unsigned long long)(n_g0 + n_g1 + n_g2 + n_g3));
        atomicAdd(&out.stats[3], (unsigned long long)max_n);
        if (warp == 0) atomicAdd(&out.stats[0], (unsigned long long)cnt);
      }
      auto blend = [&](int j, const AlphaEval& ev) {
        const float w = __fmul_rn(ev.alpha, T);
        const f32x2 ww = pack2(w, w);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 f4 = sF[4 * j + c];
          acc2[2 * c] = fma2(pack2(f4.x, f4.y), ww, acc2[2 * c]);
          acc2[2 * c + 1] = fma2(pack2(f4.z, f4.w), ww, acc2[2 * c + 1]);
        }
        T = __fmul_rn(T, __fsub_rn(1.0f, ev.alpha));
        ++n_contrib;
        last_idx = (int)(base - lb) + j + 1;
        sHit[warp][j] = 1;
        if (!kCamera) {
          const float2 c = sC[j];
          const float r_rs = __fmaf_rn(c.y, t, c.x);
          range_acc = __fmaf_rn(r_rs, w, range_acc);
          if (los_on && r_rs < los_cut) los = __fadd_rn(los, ev.alpha);  // opacity in front of the measured range
          if (!med_found && T < 0.5f) { median = r_rs; med_found = true; }
        }
        if (T < s.transmittance_min) done = true;
      };
      if (kCamera) {
        // the camera kernel is issue-bound: the plain loop has the fewest instructions
        // (group lists were measured on the camera as well: 0.98 -> 1.34 ms. Its footprints span the 8 x 4 patch, every
        // group keeps most entries, and the second-level cull is pure overhead: the camera walks the warp list)
        // Shared memory by window address (raster_common.cuh: smem_addr): no per-iteration address re-materialisation.
        const uint32_t aA = smem_addr_pinned(&sm);
        const uint32_t aB = aA + (uint32_t)offsetof(Staged, sB), aF = aA + (uint32_t)offsetof(Staged, sF);
        const uint32_t aL = aA + (uint32_t)offsetof(Staged, sList) + 256u * warp, aH = aA + (uint32_t)offsetof(Staged, sHit) + 256u * warp;
        for (int k = 0; k < n_w; ++k) {
          if ((k & 3) == 0 && __all_sync(0xffffffffu, done)) break;
          const uint32_t j = lds_u8(aL + k);
          const float4 gA = lds_f4(aA + 16u * j), gB = lds_f4(aB + 16u * j);
          float dx, dy;
          const float qf = alpha_qform_packed(pack2(gA.x, gA.y), pack2(gA.z, gA.w), gB, q2, t2, dx, dy);  // same operations, 7 issue slots
          AlphaEval ev;
          if (!done && alpha_finish(qf, gB.w, dx, dy, s.qform_max, s.alpha_clamp, s.alpha_min, ev)) {
            const float w = __fmul_rn(ev.alpha, T);
            const f32x2 ww = pack2(w, w);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 f4 = lds_f4(aF + 64u * j + 16u * c);
              acc2[2 * c] = fma2(pack2(f4.x, f4.y), ww, acc2[2 * c]);
              acc2[2 * c + 1] = fma2(pack2(f4.z, f4.w), ww, acc2[2 * c + 1]);
            }
            T = __fmul_rn(T, __fsub_rn(1.0f, ev.alpha));
            ++n_contrib;
            last_idx = (int)(base - lb) + (int)j + 1;
            sts_u8(aH + j, 1u);
            if (T < s.transmittance_min) done = true;
          }
        }
      } else {
        // the lidar kernel is latency-bound (wrap + fewer resident warps' worth of work per tile): two entries per
        // iteration with independent quadratic forms, next pair's records fetched before the current pair is blended
        const int last = max(my_n - 1, 0);
        int j0 = mine[0], j1 = mine[min(1, last)];
        float4 a0 = sA[j0], b0 = sB[j0], a1 = sA[j1], b1 = sB[j1];
        for (int k = 0; k < max_n; k += 2) {
          if ((k & 7) == 0 && !__any_sync(0xffffffffu, k < my_n && !done)) break;
          const bool has0 = k < my_n, has1 = k + 1 < my_n;
          const int jn0 = mine[min(k + 2, last)], jn1 = mine[min(k + 3, last)];  // clamped: always a slot of the list
          const float4 an0 = sA[jn0], bn0 = sB[jn0], an1 = sA[jn1], bn1 = sB[jn1];
          float dx0, dy0, dx1, dy1;
          const float qf0 = alpha_qform<true>(a0, b0, qx, qy, t, dx0, dy0, wrap);
          const float qf1 = alpha_qform<true>(a1, b1, qx, qy, t, dx1, dy1, wrap);
          AlphaEval ev;
          if (has0 && !done && alpha_finish(qf0, b0.w, dx0, dy0, s.qform_max, s.alpha_clamp, s.alpha_min, ev)) blend(j0, ev);
          if (has1 && !done && alpha_finish(qf1, b1.w, dx1, dy1, s.qform_max, s.alpha_clamp, s.alpha_min, ev)) blend(j1, ev);
          j0 = jn0; j1 = jn1; a0 = an0; b0 = bn0; a1 = an1; b1 = bn1;
        }
      }
    }

    if (inside) {
      float acc[kChannels];
#pragma unroll
      for (int k = 0; k < kChannels / 2; ++k) unpack2(acc2[k], acc[2 * k], acc[2 * k + 1]);
      const float A = __fsub_rn(1.0f, T);
      if (!kCamera) {
        acc[13] = (A > 1e-6f) ? __fdiv_rn(range_acc, A) : range_acc;
        acc[14] = median;
        acc[15] = A;
        out.range_blend[pix] = range_acc;
        if (los_on) out.los[pix] = los;
        if (kHead) {  // decode_lidar on the blended features, while they are still in registers
          float x[headdev::kInMax], y[2], h[headdev::kHid];
#pragma unroll
          for (int k = 0; k < 13; ++k) x[k] = acc[k];
          headdev::ray_dir(qx, qy, x + s.d_f);
          headdev::head_forward(sHead, s.d_f + 3, x, y, h);
          out.head_y[2 * pix] = y[0];
          out.head_y[2 * pix + 1] = y[1];
        }
      }
      float4* o4 = reinterpret_cast<float4*>(out.blend + 16 * pix);
#pragma unroll
      for (int k = 0; k < 4; ++k) o4[k] = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
      out.alpha[pix] = A;
      out.t_final[pix] = T;
      out.n_contrib[pix] = n_contrib;
      out.last_idx[pix] = last_idx;
    }
    __syncthreads();  // shared staging and patch boxes are reused by the next ray pass
    flush_hits();     // the last batch of a list that ended before every query saturated
  }
  if (!kCamera && tid == 0) out.tile_wrap[tile] = any_wrap ? 1 : 0;
}

void launch_raster_fwd(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                       const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                       const uint32_t* tile_order, const RasterOutDev& out, cudaStream_t st, int tile_first, int tile_count) {
  // tile_count < 0: the whole grid in tile_order; otherwise tiles [tile_first, tile_first + tile_count) in id order (a band)
  const int tiles = tile_count < 0 ? s.tiles_x * s.tiles_y : tile_count;
  if (tiles <= 0) return;
  const uint32_t* order = tile_count < 0 ? tile_order : nullptr;
  if (tile_count < 0) tile_first = 0;
  if (s.is_camera)
    k_raster_fwd<true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.los_cut && out.head_w)
    k_raster_fwd<false, true, true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.head_w)
    k_raster_fwd<false, false, true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.los_cut)
    k_raster_fwd<false, true><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else
    k_raster_fwd<false><<<tiles, 256, 0, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
}

// ------------------------------------------------------------------------------------------------
// Introspection (parity tests only, not on the hot path): the full ProjectedGaussian / ComposedScene
// record of every Gaussian, recomputed with the identical instruction sequence as k_project.
// Layout per Gaussian (kDumpStride floats): visible, mean2d 2, depth, cov2d 4, velocity 3, aabb 4,
// conic 4, det_ratio, mu_sensor 3, rel_vel_sensor 3, opacity, mean_w 3, vel_dyn_w 3, cov_w 9.
// ------------------------------------------------------------------------------------------------
template <bool kCamera>
__global__ void __launch_bounds__(256) k_project_dump(const __grid_constant__ Sensor s, SceneDev sc, float* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sc.n) return;
  Fwd f;
  compose_one(sc, i, f);
  if (kCamera) project_camera_one(s, f);
  else project_lidar_one(s, f);
  float* o = d + (size_t)kDumpStride * i;
  o[0] = f.visible ? 1.0f : 0.0f;
  o[26] = f.opacity;
  for (int k = 0; k < 3; ++k) { o[27 + k] = f.mean_w[k]; o[30 + k] = f.vel_dyn_w[k]; }
  for (int k = 0; k < 9; ++k) o[33 + k] = f.cov_w[k];
  if (!f.visible) return;
  o[1] = f.mean2d[0]; o[2] = f.mean2d[1]; o[3] = f.depth;
  for (int k = 0; k < 4; ++k) { o[4 + k] = f.cov2d[k]; o[15 + k] = f.conic[k]; }
  for (int k = 0; k < 3; ++k) { o[8 + k] = f.vel[k]; o[20 + k] = f.mu[k]; o[23 + k] = f.u[k]; }
  o[11] = f.lo[0]; o[12] = f.lo[1]; o[13] = f.hi[0]; o[14] = f.hi[1];
  o[19] = f.det_ratio;
}
void launch_project_dump(const Sensor& s, const SceneDev& sc, float* dump, cudaStream_t st) {
  if (sc.n == 0) return;
  const unsigned blocks = (unsigned)((sc.n + 255) / 256);
  if (s.is_camera) k_project_dump<true><<<blocks, 256, 0, st>>>(s, sc, dump);
  else k_project_dump<false><<<blocks, 256, 0, st>>>(s, sc, dump);
}

}  // namespace sb
