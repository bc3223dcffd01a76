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

constexpr int kSlots = 256 + 8 * 32;  // staged batch entries, then 32 carry slots per warp
constexpr int kListCap = 32 + 256;

// Batch staging is CTA-wide (thread = list entry: the record loads and the 8-box test are done once per entry); the
// walk is per warp in FULL rounds of 32 survivors: what is left of a batch (< 32 survivors) is copied to the warp's
// carry slots and opens the first round of the next batch, so only a list's very last round runs partially filled.
// (Measured alternatives: partial rounds per batch, 1.6 rounds per 32.4 survivors: 0.406 ms; every warp scanning the
// whole list on its own without CTA barriers: 0.62 ms — the 8-fold test work and the unhidden load chains cost more
// than the barriers.)
// The lanes that blended each entry leave as one 32-bit word per (entry, warp) in hit_rows[block][warp][entry & 255]
// (block = (tile_begin >> 8) + tile + (entry >> 8): never shared between tiles) — written only where some ray of the
// warp blended the entry, together with bit `warp` of the entry's hit byte (RasterOutDev::hit, zeroed by the host per
// forward): the same byte the shared kernels write, here it also says which words exist.
template <bool kLos, bool kHead>
__global__ void __launch_bounds__(256, 3)
k_raster_fwd_lidar(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
                   const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
                   const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
                   const uint32_t* __restrict__ tile_order, int tile_first, RasterOutDev out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* sA = reinterpret_cast<float4*>(smem_raw);              // kSlots: mean2d.xy, velocity.xy
  float4* sB = sA + kSlots;                                      // kSlots: conic a, 2b, c; rho
  float4* sF = sB + kSlots;                                      // 4 x kSlots, PLANAR (gathers by slot: 16-byte stride)
  float4* sRay = sF + 4 * kSlots;                                // 256: azimuth, elevation, t, t (phase 1 broadcasts)
  float2* sC = reinterpret_cast<float2*>(sRay + 256);            // kSlots: range, v_r
  uint32_t* sPos = reinterpret_cast<uint32_t*>(sC + kSlots);     // kSlots: tile-local list position
  uint16_t* sListAll = reinterpret_cast<uint16_t*>(sPos + kSlots);  // 8 x kListCap
  uint8_t* sMask = reinterpret_cast<uint8_t*>(sListAll + 8 * kListCap);  // 256
  __shared__ PatchBox sBox[9];  // 8 warp patches + the tile's box (patch_mask_fast)
  __shared__ float sHead[kHead ? 640 : 1];  // lidar head parameters (fused epilogue)

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : tile_first + (int)blockIdx.x;
  const int tid = threadIdx.x;
  if (kHead) {  // visible to everyone after the first barrier below
    const int np = headdev::kHid * (s.d_f + 3) + headdev::kHid + 2 * headdev::kHid + 2;
    for (int i = tid; i < np; i += 256) sHead[i] = out.head_w[i];
  }
  const int lane = tid & 31, warp = tid >> 5;
  uint16_t* lst = sListAll + kListCap * warp;
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];
  const int64_t q_begin = ray_begin[tile], q_end = ray_end[tile];  // at most 256 rays (the host guarantees it)

  const int64_t qpos = q_begin + tid;
  const bool inside = qpos < q_end;
  float qx = 0.0f, qy = 0.0f, t = 0.0f;
  int64_t pix = 0;
  if (inside) {
    const float4 r = rays[qpos];
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
  __syncthreads();  // patch boxes, rays, head parameters visible
  if (tid == 0) tile_patch_box(sBox);  // published by the first barrier of the batch loop

  uint32_t* const hitw = out.hit_rows + ((size_t)(lb >> 8) + (size_t)tile) * 2048u + warp * 256;
  uint32_t* const hit32 = reinterpret_cast<uint32_t*>(out.hit);  // hit bytes, four per word (cudaMalloc-aligned)
  const float4* wray = sRay + 32 * warp;
  const unsigned lt = (1u << lane) - 1u;
  const int carry0 = 256 + 32 * warp;  // this warp's carry slots
  int ncarry = 0;
  bool carry_wrap = false, any_wrap = false;
  unsigned live = __ballot_sync(0xffffffffu, !done);
  unsigned long long st_cand = 0ull, st_iter = 0ull;

  // one round: list entries k0 .. k0 + n - 1 (n <= 32); rw: some of them may need the azimuth wrap
  auto do_round = [&](int k0, int n, bool rw) {
    // ---- phase 1: lane = entry -----------------------------------------------------------------
    uint32_t m = 0u;
    int myslot = 0;
    if (lane < n) {
      myslot = lst[k0 + lane];
      const float4 gA = sA[myslot], gB = sB[myslot];
      // alpha = rho exp(-qf/2) < alpha_min  <=>  qf > 2 ln(rho / alpha_min); margins: 1% on rho, 0.02 on qf (the
      // evaluation's exp and this log are accurate to ~1e-6)
      float qcut = s.qform_max;
      const float rho = gB.w;
      if (s.alpha_min > 0.0f && rho > 0.0f && rho < 1e30f) qcut = fminf(qcut, 2.0f * __logf(rho * 1.01f / s.alpha_min) + 0.02f);
      if (!rw) {  // certified: no azimuth difference leaves (-pi, pi) — packed pairs, 10 issue slots per ray
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
    if (out.stats) st_cand += __popc(bits);
    // ---- phase 2: lane = ray, every lane walks its own candidates front to back ----------------
    uint32_t hitk = 0u;
    int trips = 0;
    // Two candidates per trip: the records are gathered and alpha evaluated for both first, branch-free (the same
    // operations as alpha_finish, the same decisions), so that the two chains interleave; then they are blended in order.
    auto eval = [&](int kk, int& slot, float& al, bool& ok) {
      slot = lst[k0 + kk];
      const float4 gA = sA[slot], gB = sB[slot];
      float dx, dy;
      const float qf = rw ? alpha_qform<true>(gA, gB, qx, qy, t, dx, dy, true)
                          : alpha_qform_packed(pack2(gA.x, gA.y), pack2(gA.z, gA.w), gB, q2, t2, dx, dy);
      const bool in = qf <= s.qform_max;
      const float gauss = detmath::exp_bounded(in ? fminf(__fmul_rn(-0.5f, qf), 88.0f) : 0.0f);
      al = __fmul_rn(gB.w, gauss);
      if (al > s.alpha_clamp) al = s.alpha_clamp;
      ok = in && (al >= s.alpha_min);
    };
    auto blend = [&](int slot, float al, uint32_t b) {
      const float w = __fmul_rn(al, T);
      const f32x2 ww = pack2(w, w);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 f4 = sF[c * kSlots + slot];
        acc2[2 * c] = fma2(pack2(f4.x, f4.y), ww, acc2[2 * c]);
        acc2[2 * c + 1] = fma2(pack2(f4.z, f4.w), ww, acc2[2 * c + 1]);
      }
      T = __fmul_rn(T, __fsub_rn(1.0f, al));
      ++n_contrib;
      last_idx = (int)sPos[slot] + 1;
      hitk |= b;
      const float2 c2 = sC[slot];
      const float r_rs = __fmaf_rn(c2.y, t, c2.x);
      range_acc = __fmaf_rn(r_rs, w, range_acc);
      if (kLos && r_rs < los_cut) los = __fadd_rn(los, al);  // opacity in front of the measured range
      if (!med_found && T < 0.5f) { median = r_rs; med_found = true; }
      if (T < s.transmittance_min) { done = true; bits = 0u; }
    };
    while (bits != 0u) {
      const uint32_t b0 = bits & (0u - bits);
      const int kk0 = __ffs(bits) - 1;
      bits ^= b0;
      const bool has1 = bits != 0u;
      const uint32_t b1 = bits & (0u - bits);
      const int kk1 = has1 ? __ffs(bits) - 1 : kk0;
      bits ^= b1;
      ++trips;
      int slot0, slot1;
      float al0, al1;
      bool ok0, ok1;
      eval(kk0, slot0, al0, ok0);
      eval(kk1, slot1, al1, ok1);
      if (ok0) blend(slot0, al0, b0);
      if (has1 && ok1 && !done) blend(slot1, al1, b1);
    }
    if (out.stats) st_iter += (unsigned long long)__reduce_max_sync(0xffffffffu, trips);
    // the rays that blended each entry: back to entry-major, one word per (entry, warp)
    const uint32_t hw = transpose32(hitk, lane);
    if (lane < n && hw != 0u) {
      const uint32_t ps = sPos[myslot];
      hitw[(size_t)(ps >> 8) * 2048u + (ps & 255u)] = hw;
      // ... and bit `warp` of the entry's hit byte (pre-zeroed by the host): the backward compacts the non-zero bytes
      // into a dense list and fetches exactly the words whose bit is set
      const uint32_t at = lb + ps;
      atomicOr(hit32 + (at >> 2), (1u << warp) << (8u * (at & 3u)));
    }
    live = __ballot_sync(0xffffffffu, !done);
  };
  auto copy_slot = [&](int from, int to) {
    sA[to] = sA[from];
    sB[to] = sB[from];
    sC[to] = sC[from];
    sPos[to] = sPos[from];
#pragma unroll
    for (int c = 0; c < 4; ++c) sF[c * kSlots + to] = sF[c * kSlots + from];
  };

  for (uint32_t base = lb; base < le; base += 256) {
    if (__syncthreads_and(done)) break;  // also: every warp is through with the staged batch
    const uint32_t idx = base + tid;
    uint32_t mask = 0u, wrapm = 0u;
    if (idx < le) {
      const uint32_t src = vals[idx];
      const float4 gA = p.geomA[src], gB = p.geomB[src];
      mask = patch_mask_fast<true>(gA, gB, sBox, s.qform_max, s.alpha_min, &wrapm);
      if (out.stats && !(fabsf(gA.x) + fabsf(gA.y) + fabsf(gA.z) + fabsf(gA.w) + fabsf(gB.x) + fabsf(gB.y) + fabsf(gB.z) + fabsf(gB.w) < 3.0e38f))
        atomicAdd(&out.stats[4], 1ull);  // SPEC.md:289 non-finite record counter
      if (mask) {
        sA[tid] = gA;
        sB[tid] = gB;
        sC[tid] = p.geomC[src];
        sPos[tid] = idx - lb;
#pragma unroll
        for (int k = 0; k < 4; ++k) sF[k * kSlots + tid] = p.feat[4 * (size_t)src + k];
      }
    }
    sMask[tid] = (uint8_t)mask;
    const bool wrap = __syncthreads_or((mask & wrapm) != 0u) != 0;
    any_wrap |= wrap;
    if (live == 0u) { ncarry = 0; continue; }  // this warp's 32 rays have saturated
    const int cnt = min(256u, le - base);
    // the warp's list: what the last batch left over, then this batch's survivors (order preserved)
    if (lane < ncarry) lst[lane] = (uint16_t)(carry0 + lane);
    int n = ncarry;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int j = c0 + lane;
      const bool bit = j < cnt && ((sMask[j] >> warp) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      if (bit) lst[n + __popc(bal & lt)] = (uint16_t)j;
      n += __popc(bal);
    }
    __syncwarp();
    if (out.stats && lane == 0) {
      atomicAdd(&out.stats[1], (unsigned long long)(n - ncarry));
      if (warp == 0) atomicAdd(&out.stats[0], (unsigned long long)cnt);
    }
    const bool rw = wrap || carry_wrap;
    int k0 = 0;
    for (; k0 + 32 <= n && live != 0u; k0 += 32) {
      do_round(k0, 32, rw);
      __syncwarp();
    }
    // what is left moves to the carry slots (it is either all new, or nothing was processed and the old carry stays)
    const int r = live != 0u ? n - k0 : 0;
    if (k0 == 0) {
      if (lane >= ncarry && lane < r) copy_slot(lst[lane], carry0 + lane);
      carry_wrap = r > 0 && rw;
    } else {
      if (lane < r) copy_slot(lst[k0 + lane], carry0 + lane);
      carry_wrap = r > 0 && wrap;
    }
    ncarry = r;
    __syncwarp();
  }
  if (ncarry > 0 && live != 0u) {  // the list's last, partial round
    if (lane < ncarry) lst[lane] = (uint16_t)(carry0 + lane);
    __syncwarp();
    do_round(0, ncarry, carry_wrap);
  }
  if (out.stats) {
    const unsigned tot = __reduce_add_sync(0xffffffffu, (unsigned)st_cand);
    if (lane == 0) {
      atomicAdd(&out.stats[2], (unsigned long long)tot);
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
  if (tid == 0) out.tile_wrap[tile] = any_wrap ? 1 : 0;  // CTA-uniform: the backward skips the wrap elsewhere
}

constexpr size_t kLidarFwdSmem = sizeof(float4) * (2 * kSlots + 4 * kSlots + 256) + sizeof(float2) * kSlots +
                                 sizeof(uint32_t) * kSlots + sizeof(uint16_t) * 8 * kListCap + 256;

size_t lidar_hit_rows_words(int64_t n_isect, int64_t n_tiles) { return (size_t)((n_isect >> 8) + n_tiles + 2) * 2048u; }

void launch_raster_fwd_lidar(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                             const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                             const uint32_t* tile_order, const RasterOutDev& out, cudaStream_t st, int tile_first, int tile_count) {
  const int tiles = tile_count < 0 ? s.tiles_x * s.tiles_y : tile_count;
  if (tiles <= 0) return;
  const uint32_t* order = tile_count < 0 ? tile_order : nullptr;
  if (tile_count < 0) tile_first = 0;
  constexpr size_t smem = kLidarFwdSmem;
  static DeviceOnce once;
  once.run([] {
    cudaFuncSetAttribute(k_raster_fwd_lidar<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_raster_fwd_lidar<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_raster_fwd_lidar<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_raster_fwd_lidar<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (out.los_cut && out.head_w)
    k_raster_fwd_lidar<true, true><<<tiles, 256, smem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.head_w)
    k_raster_fwd_lidar<false, true><<<tiles, 256, smem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else if (out.los_cut)
    k_raster_fwd_lidar<true, false><<<tiles, 256, smem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
  else
    k_raster_fwd_lidar<false, false><<<tiles, 256, smem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, order, tile_first, out);
}

}  // namespace sb
