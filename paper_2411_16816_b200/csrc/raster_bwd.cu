// raster_bwd.cu — compositing backward.
//
// One CTA per tile, the same query->thread mapping, per-warp patches and conservative culling as the
// forward kernel (raster_common.cuh). Each thread restarts from its saved terminal transmittance
// and walks its warp's compacted list back to front, recomputing alpha with the very same
// instruction sequence as the forward pass, so it revisits exactly the Gaussians that were blended.
//
// With w_i = alpha_i T_i, out_c = sum_i f_ic w_i, A = 1 - T_final:
//   dL/df_ic     = w_i g_c
//   dL/dalpha_i  = T_i sum_c g_c f_ic  -  (S_i - g_A T_final) / (1 - alpha_i),   S_i = sum_c g_c sum_{j>i} f_jc w_j
// S_i is carried as ONE scalar per thread (S += w_i * sum_c g_c f_ic), not one suffix per channel.
// For lidar the rolling-shutter range r_rs = r + v_r t is one more blended channel whose upstream is
// dL/d(range_blend); expected = range_blend / A feeds both.
//
// Reduction of the 26 per-pair values to per-Gaussian gradients, in two phases per warp:
//   A (lane = query): the sequential part. For every list entry that some lane blends, each lane computes
//     only TWO scalars — w and dL/dsigma (sigma = qf / 2) — and parks them in a [slot][lane] shared-memory
//     panel (strides 36 for w, 33 for dL/dsigma: conflict-free for these writes and for phase B's reads). Every other one of the 26 values is a product of one of
//     those scalars with per-query data (g_c, t, g_D) or per-Gaussian data (conic, mean, velocity); the
//     dL/drho term is -dL/dsigma / rho (alpha = rho exp(-sigma) when it is not clamped), so its sum over the
//     queries needs no panel of its own.
//   B: when the panel holds kChunk entries (or the batch ends) the roles flip. The 16 channel sums (for the lidar
//     13 features + range + v_r) are a dense (entries x queries) x (queries x channels) product and run as warp-level
//     tf32 MMAs with split operands (reduce_panel). For the eight geometric sums lanes are spread over the parked
//     entries (32 / E lanes per entry, E = capacity rounded up to a power of two), each lane loops over its share of
//     the 32 queries — query data is read as shared-memory broadcasts — and accumulates the sums of ITS Gaussian in
//     registers; log2(32 / E) shuffle steps join the lanes of one entry. This replaces a 31-shuffle transposing
//     butterfly per (warp, Gaussian) and costs about a third of the instructions.
// The panel carries its own copy of each parked Gaussian's record, so it survives batch boundaries and is
// (almost) always drained full. The 24-26 sums of a (warp, Gaussian) leave as fire-and-forget global REDs
// (north_star (4): warp-aggregated atomics — 32 queries are folded into one RED per value). Shared-memory
// float atomics are NOT used: on sm_100a they compile to a compare-and-swap spin loop (ATOMS.CAST.SPIN),
// which the first version of this kernel showed to be the bottleneck (profiles/).
#include <cstdlib>

#include "kernels.h"
#include "raster_common.cuh"

// Measured alternatives that lost (round 1, same box A/B): 3 CTAs/SM with 80 registers and smaller panels or half-size
// batches (4-15% slower); a sparse phase B over a saved ballot of the blending lanes (camera 4% slower); fully
// warp-private staging without any CTA barrier — each warp scanning the hit bytes and gathering its own entries 32 at a
// time (5% slower: the CTA-wide batch amortises one memory round trip over 256 list entries, the private ring pays one
// per 32).
namespace sb {

constexpr int kBatch = 256;  // list entries staged per batch
constexpr int kChunk = 16;   // panel capacity per warp (8 with 3 CTAs/SM was measured: 4-15% slower)
constexpr int kPanelStride = 33;  // dL/dsigma panel: read by the per-entry loop (lane = entry)
constexpr int kWStride = 36;      // w panel: read as the A fragments of the channel product (conflict-free: 4 gid + tig)
constexpr int kPxStride = 24;     // qx qy t g_D | G[16] | pad (24 tig + gid: conflict-free B fragments)

template <int kC>
struct WarpScratchT {
  float w[kC * kWStride];
  float gs[kC * kPanelStride];
  float px[32 * kPxStride];
  float4 gAB[2 * kC];  // the parked Gaussians' records: geomA | geomB
  uint32_t src[kC];
};
using WarpScratch = WarpScratchT<kChunk>;
constexpr int kChunkS = 8;  // panel capacity of the shared kernel (k_raster_bwd): 8 entries -> 75.8 KB per CTA, 3 CTAs per SM

// D += A B for one m16n8k8 tf32 tile (A row-major 16 x 8, B column-major 8 x 8, fp32 accumulators).
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
constexpr uint32_t kTf32Mask = 0xffffe000u;  // sign, exponent, 10 mantissa bits

// One 16-byte fire-and-forget reduction (REDG.E.ADD.F32x4): four adjacent floats of one row in ONE request. The raw
// geometric sums of an entry used to leave as eight scalar REDs issued value by value — eight instructions, each touching
// one 32-byte sector per entry (8 sectors per (warp, entry); measured with scripts/red_peak.cu the backward kernels ran
// at 46-59% of the GPU's RED sector ceiling). The scratch rows are laid out for this (kernels.h: kRasterGradStride).
__device__ __forceinline__ void red_add_v4(float* dst, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Phase B for `n` parked entries (1 <= n <= kChunk).
//
// The 16 channel sums are the one dense contraction of the path: dL/df[e][c] = sum_q w[e][q] G[q][c], a
// (16 entries x 32 queries) x (32 queries x 16 channels) product per drained panel. It runs as 8 warp-level
// m16n8k8 tiles with split operands (x = hi + lo, both exactly representable in tf32; hi hi + hi lo + lo hi, the
// "3xTF32" scheme: products exact, ~2^-21 relative error, fp32 accumulation), replacing 16 FMAs and four
// 128-bit shared loads per (entry, query) pair. Both operands are split on the fly: keeping pre-split G rows in
// shared memory was measured and lost (the 20 KB more per CTA push the carve-out to 228 KB and leave the lidar's
// gathers no L1: +5% on its kernel). For the lidar the two free columns carry g_D and g_D t, which yields d/d range and d/d v_r from the
// same product. tcgen05 does not fit here: the operand is produced in registers by this warp, 16 rows at a time.
// The eight geometric sums (conic 3, mean 2, velocity 2, rho) depend on the pair through Delta and stay on the
// fp32 pipe, lane = entry.
template <bool kCamera>
__device__ __forceinline__ void reduce_panel(const WarpScratch& ws, int n, int lane, int d_f, const RasterGradDev& rg,
                                             const ParamGradDev& pg, float& dt_local, bool wrap) {
  {  // channel product
    const int gid = lane >> 2, tig = lane & 3;
    float d[2][4], dlh[2][4], dhl[2][4];  // three accumulators per tile: six independent chains of four MMAs
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) d[nt][k] = dlh[nt][k] = dhl[nt][k] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int q = ks * 8 + tig;
      const float af[4] = {ws.w[gid * kWStride + q], ws.w[(gid + 8) * kWStride + q], ws.w[gid * kWStride + q + 4],
                           ws.w[(gid + 8) * kWStride + q + 4]};
      uint32_t ah[4], al[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ah[k] = __float_as_uint(af[k]) & kTf32Mask;
        al[k] = __float_as_uint(af[k] - __uint_as_float(ah[k])) & kTf32Mask;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const float* bp = &ws.px[q * kPxStride + 4 + nt * 8 + gid];
        const float bf0 = bp[0], bf1 = bp[4 * kPxStride];
        const uint32_t bh0 = __float_as_uint(bf0) & kTf32Mask, bh1 = __float_as_uint(bf1) & kTf32Mask;
        const uint32_t bl0 = __float_as_uint(bf0 - __uint_as_float(bh0)) & kTf32Mask;
        const uint32_t bl1 = __float_as_uint(bf1 - __uint_as_float(bh1)) & kTf32Mask;
        mma_tf32(dlh[nt], al, bh0, bh1);
        mma_tf32(dhl[nt], ah, bl0, bl1);
        mma_tf32(d[nt], ah, bh0, bh1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) d[nt][k] += dlh[nt][k] + dhl[nt][k];
    // lane holds rows gid, gid + 8 and columns nt * 8 + 2 tig, + 1: one RED per (warp, Gaussian, value)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = gid + 8 * h;
      if (e < n) {
        const size_t src = ws.src[e];
        float* f0 = kCamera ? pg.d_color + 3 * src : pg.d_feature + (size_t)d_f * src;
        float* f1 = pg.d_feature + (size_t)d_f * src - (kCamera ? 3 : 0);
        float* r0 = rg.g + kRasterGradStride * src - 16;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = nt * 8 + 2 * tig + j;
            const float v = d[nt][2 * h + j];
            if (v != 0.0f) {  // columns >= channels are exactly zero
              float* dst;
              if (kCamera) dst = c < 3 ? f0 + c : f1 + c;
              else dst = c < 13 ? f1 + c : (c == 13 ? r0 + 25 : r0 + 24);  // 13: d/d range (slot 9), 14: d/d v_r (slot 8)
              atomicAdd(dst, v);
            }
          }
      }
    }
  }
  int E = 1;  // capacity: smallest power of two >= n
  while (E < n) E <<= 1;
  const int e = lane & (E - 1);
  const int g = lane / E;  // which share of the queries
  const bool active = e < n;
  const float4 gA = ws.gAB[active ? e : 0], gB = ws.gAB[kChunk + (active ? e : 0)];
  // The eight geometric sums are linear in eight raw moments of g = dL/dsigma over the queries —
  // {1, dx, dy, dx dx, dx dy, dy dy, t dx, t dy} — so the loop accumulates those (14 fp32 instructions per pair) and
  // the conic / velocity factors are applied once per entry after the join.
  constexpr int kGeo = 8;
  float m[kGeo];  // S0 Sx Sy Sxx Sxy Syy Stx Sty
  const int row = e * kPanelStride;
  // (visiting only the queries that blended the entry — a divergent loop over a saved ballot — was measured: 2% faster
  // for the lidar, 4% slower for the camera, whose entries are blended by a third of the lanes; the dense loop stays)
  if (kCamera || !wrap) {
    // packed pairs (FFMA2 / FMUL2 / FADD2: two fp32 operations per issue slot): 9 issue slots per pair instead of 14
    const f32x2 m0 = pack2(gA.x, gA.y), vv = pack2(gA.z, gA.w);
    f32x2 sxy = pack2(0.0f, 0.0f), sq = sxy, st = sxy;  // (Sx, Sy), (Sxx, Syy), (Stx, Sty)
    float s0 = 0.0f, sxy_c = 0.0f;
#pragma unroll 4
    for (int pp = 0; pp < E; ++pp) {  // 32 / (32 / E) queries per lane
      const int q = g * E + pp;
      const float gs = ws.gs[row + q];
      const float4 q0 = *reinterpret_cast<const float4*>(&ws.px[q * kPxStride]);  // qx qy t g_D
      const f32x2 tt = pack2(q0.z, q0.z);
      const f32x2 d = sub2(pack2(q0.x, q0.y), fma2(vv, tt, m0));  // (dx, dy)
      const f32x2 ab = mul2(pack2(gs, gs), d);                     // (gs dx, gs dy)
      float dxs, dys, as, bs;
      unpack2(d, dxs, dys);
      unpack2(ab, as, bs);
      s0 += gs;
      sxy = add2(sxy, ab);
      sq = fma2(ab, d, sq);
      sxy_c = fmaf(as, dys, sxy_c);
      st = fma2(tt, ab, st);
    }
    m[0] = s0;
    unpack2(sxy, m[1], m[2]);
    unpack2(sq, m[3], m[5]);
    m[4] = sxy_c;
    unpack2(st, m[6], m[7]);
  } else {
#pragma unroll
    for (int c = 0; c < kGeo; ++c) m[c] = 0.0f;
#pragma unroll 4
    for (int pp = 0; pp < E; ++pp) {
      const int q = g * E + pp;
      const float gs = ws.gs[row + q];
      const float4 q0 = *reinterpret_cast<const float4*>(&ws.px[q * kPxStride]);  // qx qy t g_D
      const float t = q0.z;
      const float dx = wrap_pi(q0.x - fmaf(gA.z, t, gA.x));
      const float dy = q0.y - fmaf(gA.w, t, gA.y);
      const float a = gs * dx, b = gs * dy;
      m[0] += gs;
      m[1] += a;
      m[2] += b;
      m[3] = fmaf(a, dx, m[3]);
      m[4] = fmaf(a, dy, m[4]);
      m[5] = fmaf(b, dy, m[5]);
      m[6] = fmaf(t, a, m[6]);
      m[7] = fmaf(t, b, m[7]);
    }
  }
  // join the 32 / E lanes that worked on the same entry
  for (int o = E; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < kGeo; ++c) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
  }
  // after the butterfly every lane of an entry holds the full sums (at least two lanes per entry: E <= 16): lane g = 0
  // sends (conic, rho), lane g = 1 (mean2d, velocity.xy) — two 16-byte REDs per (warp, Gaussian) in one instruction
  if (active && g < 2) {
    const float hb = 0.5f * gB.y;
    float* r0 = rg.g + kRasterGradStride * (size_t)ws.src[e];
    if (g == 0) {
      const float a0 = 0.5f * m[3], a1 = 0.5f * m[4], a2 = 0.5f * m[5];  // dL/dconic
      const float a3 = __fdividef(-m[0], gB.w);  // dL/drho = -dL/dsigma / rho (rho > 0 for every blended entry)
      if (a0 != 0.0f || a1 != 0.0f || a2 != 0.0f || a3 != 0.0f) red_add_v4(r0, a0, a1, a2, a3);
    } else {
      const float gx = fmaf(hb, m[2], gB.x * m[1]), gy = fmaf(hb, m[1], gB.z * m[2]);     // sum of dL/dDelta
      const float gtx = fmaf(hb, m[7], gB.x * m[6]), gty = fmaf(hb, m[6], gB.z * m[7]);   // sum of t dL/dDelta
      if (kCamera) dt_local -= fmaf(gA.z, gx, gA.w * gy);  // SensorGrads.d_time_offset
      if (gx != 0.0f || gy != 0.0f || gtx != 0.0f || gty != 0.0f) red_add_v4(r0 + 4, -gx, -gy, -gtx, -gty);  // dL/dmean2d, dL/dvelocity.xy
    }
  }
  __syncwarp();
}

// Phase B for the n <= 8 entries of an 8-entry panel. The channel product is transposed — D[c][e] = sum_q G[q][c] w[e][q],
// M = 16 channels, N = 8 entries, K = 32 queries — so that an 8-entry panel fills the m16n8k8 tile: 12 split-tf32 MMAs
// and 12 accumulator registers (the 16-entry form: 24 and 24; half of its A rows would be empty here). Raw moments: 4
// lanes per entry, 8 queries each.
template <bool kCamera>
__device__ __forceinline__ void reduce_panel8(const WarpScratchT<kChunkS>& ws, int n, int lane, int d_f, const RasterGradDev& rg,
                                              const ParamGradDev& pg, float& dt_local, bool wrap) {
  {
    const int gid = lane >> 2, tig = lane & 3;
    float d[4], dlh[4], dhl[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = dlh[k] = dhl[k] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int q = ks * 8 + tig;
      // A[m = channel][k = query] = G[q][c]: rows gid, gid + 8; columns tig, tig + 4 (banks 24 tig + gid: conflict-free)
      const float* ap = &ws.px[q * kPxStride + 4 + gid];
      const float af[4] = {ap[0], ap[8], ap[4 * kPxStride], ap[4 * kPxStride + 8]};
      uint32_t ah[4], al[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ah[k] = __float_as_uint(af[k]) & kTf32Mask;
        al[k] = __float_as_uint(af[k] - __uint_as_float(ah[k])) & kTf32Mask;
      }
      // B[k = query][n = entry] = w[e][q]: rows tig, tig + 4; column gid (banks 4 gid + tig: conflict-free)
      const float bf0 = ws.w[gid * kWStride + q], bf1 = ws.w[gid * kWStride + q + 4];
      const uint32_t bh0 = __float_as_uint(bf0) & kTf32Mask, bh1 = __float_as_uint(bf1) & kTf32Mask;
      const uint32_t bl0 = __float_as_uint(bf0 - __uint_as_float(bh0)) & kTf32Mask;
      const uint32_t bl1 = __float_as_uint(bf1 - __uint_as_float(bh1)) & kTf32Mask;
      mma_tf32(dlh, al, bh0, bh1);
      mma_tf32(dhl, ah, bl0, bl1);
      mma_tf32(d, ah, bh0, bh1);
    }
    // lane holds channels gid, gid + 8 of entries 2 tig, 2 tig + 1: one RED per (warp, Gaussian, value)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int e = 2 * tig + j;
      if (e < n) {
        const size_t src = ws.src[e];
        float* f0 = kCamera ? pg.d_color + 3 * src : pg.d_feature + (size_t)d_f * src;
        float* f1 = pg.d_feature + (size_t)d_f * src - (kCamera ? 3 : 0);
        float* r0 = rg.g + kRasterGradStride * src - 16;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = gid + 8 * h;
          const float v = d[2 * h + j] + dlh[2 * h + j] + dhl[2 * h + j];
          if (v != 0.0f) {  // channels >= the sensor's are exactly zero
            float* dst;
            if (kCamera) dst = c < 3 ? f0 + c : f1 + c;
            else dst = c < 13 ? f1 + c : (c == 13 ? r0 + 25 : r0 + 24);  // 13: d/d range (slot 9), 14: d/d v_r (slot 8)
            atomicAdd(dst, v);
          }
        }
      }
    }
  }
  const int e = lane & 7, g = lane >> 3;
  const bool active = e < n;
  const float4 gA = ws.gAB[active ? e : 0], gB = ws.gAB[kChunkS + (active ? e : 0)];
  float m[8];  // S0 Sx Sy Sxx Sxy Syy Stx Sty
  const int row = e * kPanelStride;
  if (kCamera || !wrap) {
    const f32x2 m0 = pack2(gA.x, gA.y), vv = pack2(gA.z, gA.w);
    f32x2 sxy = pack2(0.0f, 0.0f), sq = sxy, st = sxy;  // (Sx, Sy), (Sxx, Syy), (Stx, Sty)
    float s0 = 0.0f, sxy_c = 0.0f;
#pragma unroll 4
    for (int pp = 0; pp < 8; ++pp) {
      const int q = g * 8 + pp;
      const float gs = ws.gs[row + q];
      const float4 q0 = *reinterpret_cast<const float4*>(&ws.px[q * kPxStride]);  // qx qy t g_D
      const f32x2 tt = pack2(q0.z, q0.z);
      const f32x2 dd = sub2(pack2(q0.x, q0.y), fma2(vv, tt, m0));  // (dx, dy)
      const f32x2 ab = mul2(pack2(gs, gs), dd);                     // (gs dx, gs dy)
      float dxs, dys, as, bs;
      unpack2(dd, dxs, dys);
      unpack2(ab, as, bs);
      s0 += gs;
      sxy = add2(sxy, ab);
      sq = fma2(ab, dd, sq);
      sxy_c = fmaf(as, dys, sxy_c);
      st = fma2(tt, ab, st);
    }
    m[0] = s0;
    unpack2(sxy, m[1], m[2]);
    unpack2(sq, m[3], m[5]);
    m[4] = sxy_c;
    unpack2(st, m[6], m[7]);
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) m[c] = 0.0f;
#pragma unroll 4
    for (int pp = 0; pp < 8; ++pp) {
      const int q = g * 8 + pp;
      const float gs = ws.gs[row + q];
      const float4 q0 = *reinterpret_cast<const float4*>(&ws.px[q * kPxStride]);
      const float t = q0.z;
      const float dx = wrap_pi(q0.x - fmaf(gA.z, t, gA.x));
      const float dy = q0.y - fmaf(gA.w, t, gA.y);
      const float a = gs * dx, b = gs * dy;
      m[0] += gs;
      m[1] += a;
      m[2] += b;
      m[3] = fmaf(a, dx, m[3]);
      m[4] = fmaf(a, dy, m[4]);
      m[5] = fmaf(b, dy, m[5]);
      m[6] = fmaf(t, a, m[6]);
      m[7] = fmaf(t, b, m[7]);
    }
  }
#pragma unroll
  for (int o = 8; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < 8; ++c) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
  }
  // after the butterfly every lane of an entry holds the full sums (four lanes per entry): lane g = 0
  // sends (conic, rho), lane g = 1 (mean2d, velocity.xy) — two 16-byte REDs per (warp, Gaussian) in one instruction
  if (active && g < 2) {
    const float hb = 0.5f * gB.y;
    float* r0 = rg.g + kRasterGradStride * (size_t)ws.src[e];
    if (g == 0) {
      const float a0 = 0.5f * m[3], a1 = 0.5f * m[4], a2 = 0.5f * m[5];  // dL/dconic
      const float a3 = __fdividef(-m[0], gB.w);  // dL/drho = -dL/dsigma / rho (rho > 0 for every blended entry)
      if (a0 != 0.0f || a1 != 0.0f || a2 != 0.0f || a3 != 0.0f) red_add_v4(r0, a0, a1, a2, a3);
    } else {
      const float gx = fmaf(hb, m[2], gB.x * m[1]), gy = fmaf(hb, m[1], gB.z * m[2]);     // sum of dL/dDelta
      const float gtx = fmaf(hb, m[7], gB.x * m[6]), gty = fmaf(hb, m[6], gB.z * m[7]);   // sum of t dL/dDelta
      if (kCamera) dt_local -= fmaf(gA.z, gx, gA.w * gy);  // SensorGrads.d_time_offset
      if (gx != 0.0f || gy != 0.0f || gtx != 0.0f || gty != 0.0f) red_add_v4(r0 + 4, -gx, -gy, -gtx, -gty);  // dL/dmean2d, dL/dvelocity.xy
    }
  }
  __syncwarp();
}

template <bool kCamera, bool kLos = false>
__global__ void __launch_bounds__(256, 3)
k_raster_bwd(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
             const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
             const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
             const uint32_t* __restrict__ tile_order, int tile_first, RasterOutDev fwd, const float* __restrict__ g_blend16,
             const float* __restrict__ g_alpha, RasterGradDev rg, ParamGradDev pg, float* __restrict__ d_time_offset) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* sA = reinterpret_cast<float4*>(smem_raw);                    // kBatch
  float4* sB = sA + kBatch;                                            // kBatch
  float4* sF = sB + kBatch;                                            // 4 kBatch
  float2* sC = reinterpret_cast<float2*>(sF + 4 * kBatch);             // kBatch
  uint32_t* sSrc = reinterpret_cast<uint32_t*>(sC + kBatch);           // kBatch
  uint32_t* sPos = sSrc + kBatch;                                      // kBatch: tile-local list position
  PatchBox* sBox = reinterpret_cast<PatchBox*>(sPos + kBatch);         // 8
  WarpScratchT<kChunkS>* sWs = reinterpret_cast<WarpScratchT<kChunkS>*>(sBox + 8);         // 8
  uint8_t* sMask = reinterpret_cast<uint8_t*>(sWs + 8);                // kBatch
  uint8_t* sListAll = sMask + kBatch;                                  // 8 x kBatch
  __shared__ int s_max_last;
  __shared__ int s_wcnt[8];
  __shared__ float s_dt[8];

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : tile_first + (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint8_t* sList = sListAll + kBatch * warp;
  WarpScratchT<kChunkS>& ws = sWs[warp];
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];
  if (le <= lb) return;
  // lidar: the forward pass certified, per tile, whether any azimuth difference can leave (-pi, pi) (raster_common.cuh)
  const bool wrap = kCamera ? false : fwd.tile_wrap[tile] != 0;
  // camera: a set hit bit means some lane of this warp blends the entry. (The same holds for lidar views without
  // multi-pass tiles, hit_or == 0, but skipping the vote there measured 1.5% SLOWER on the lidar kernel.)
  constexpr bool sure = kCamera;

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
    int last = 0;
    constexpr bool los_on = !kCamera && kLos;
    float los_cut = 0.0f, g_los = 0.0f;
    if (los_on && inside) { los_cut = fwd.los_cut[pix]; g_los = fwd.g_los[pix]; }
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
    f32x2 g2[kChannels / 2];  // the upstream gradient as packed pairs (phase A's dot product)
#pragma unroll
    for (int k = 0; k < kChannels / 2; ++k) g2[k] = pack2(g_out[2 * k], g_out[2 * k + 1]);

    // per-query data for phase B (read there as broadcasts)
    {
      float* row = &ws.px[lane * kPxStride];
      *reinterpret_cast<float4*>(row) = make_float4(qx, qy, t, g_D);
      // the B operand of the channel product (reduce_panel); lidar: columns 13, 14 = g_D, g_D t
      float gcol[kChannels];
#pragma unroll
      for (int k = 0; k < kChannels; ++k) gcol[k] = g_out[k];
      if (!kCamera) { gcol[13] = g_D; gcol[14] = g_D * t; gcol[15] = 0.0f; }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        *reinterpret_cast<float4*>(row + 4 + 4 * k) = make_float4(gcol[4 * k], gcol[4 * k + 1], gcol[4 * k + 2], gcol[4 * k + 3]);
    }

    // warp and block maxima of `last`
    if (tid == 0) s_max_last = 0;
    __syncthreads();
    int warp_last = last;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) warp_last = max(warp_last, __shfl_xor_sync(0xffffffffu, warp_last, o));
    if (lane == 0 && warp_last > 0) atomicMax(&s_max_last, warp_last);
    __syncthreads();  // also publishes the patch boxes and the per-query rows
    const int max_last = s_max_last;
    int n_slots = 0;  // parked entries (warp-uniform); the panel persists across batches
    unsigned long long jpack = 0ull;  // batch index of each parked slot (8 bits each)
    uint32_t pend = 0u;               // slots whose record has not been copied into the panel yet
    // records of the slots parked since the last copy: lane 8 w + e copies part w (geomA, geomB, index) of slot e
    auto copy_pending = [&]() {
      const int e = lane & 7, part = lane >> 3;
      if (part < 3 && ((pend >> e) & 1u)) {
        const int j = (int)((jpack >> (8 * e)) & 0xffull);
        if (part == 0) ws.gAB[e] = sA[j];
        else if (part == 1) ws.gAB[kChunkS + e] = sB[j];
        else ws.src[e] = sSrc[j];
      }
      pend = 0u;
      __syncwarp();
    };

    // Compact hit list. On the north-star camera 6% of the list entries a tile's forward pass visited were blended by
    // anyone (the rest are culled grazing footprints): walking the raw list in batches of 256 meant ~5 batches per tile
    // — two barriers and a chain of dependent loads each — for ~16 useful entries apiece. The CTA therefore first scans
    // its hit bytes (4 per thread and load, 1,024 per step) and writes (position << 8 | warp mask) of the entries that
    // were blended, in list order, to its slice of fwd.hit_list; the batches below are then dense.
    uint32_t* const hl = fwd.hit_list + lb;
    int n_hit = 0;  // CTA-uniform
    {
      const uint32_t w0 = lb >> 2;  // absolute 4-byte word of the tile's first hit byte (the buffer is padded)
      const uint32_t* hit4 = reinterpret_cast<const uint32_t*>(fwd.hit);
      for (uint32_t wbase = w0; 4u * wbase < lb + (uint32_t)max_last; wbase += 256u) {
        const uint32_t word = hit4[wbase + tid];
        const int pos0 = (int)(4u * (wbase + tid)) - (int)lb;  // tile-local position of the word's first byte
        uint32_t ent[4];
        int c4 = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t m = (word >> (8 * i)) & 0xffu;
          const int ps = pos0 + i;
          if (m != 0u && ps >= 0 && ps < max_last) ent[c4++] = ((uint32_t)ps << 8) | m;
        }
        int incl = c4;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (lane == 31) s_wcnt[warp] = incl;
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int c = s_wcnt[w];
          if (w < warp) before += c;
          total += c;
        }
        uint32_t* dst = hl + n_hit + before + (incl - c4);
        for (int i = 0; i < c4; ++i) dst[i] = ent[i];
        n_hit += total;
        __syncthreads();  // s_wcnt is reused; after the last step: the list is visible to the whole CTA
      }
    }

    // list entry and record index of a batch are fetched one batch ahead and its records prefetched into L2: a batch's
    // staging then starts with the record loads instead of a chain of dependent global loads
    uint32_t ent_next = 0u, src_next = 0u;
    const int nbat = (n_hit + kBatch - 1) / kBatch;
    if (nbat > 0) {
      const int i0 = (nbat - 1) * kBatch + tid;
      if (i0 < n_hit) {
        ent_next = hl[i0];
        src_next = vals[lb + (ent_next >> 8)];
      }
    }
    for (int batch = nbat - 1; batch >= 0; --batch) {
      const int cnt = min(kBatch, n_hit - batch * kBatch);
      {
        const uint32_t ent = ent_next;
        const uint32_t src = src_next;
        ent_next = 0u;
        if (batch > 0) {  // the batch in front of this one is always full
          ent_next = hl[(batch - 1) * kBatch + tid];
          src_next = vals[lb + (ent_next >> 8)];
        }
        if (tid < cnt) {
          sSrc[tid] = src;
          sPos[tid] = ent >> 8;
          sA[tid] = p.geomA[src];
          sB[tid] = p.geomB[src];
          if (!kCamera) sC[tid] = p.geomC[src];
#pragma unroll
          for (int k = 0; k < 4; ++k) sF[4 * tid + k] = p.feat[4 * (size_t)src + k];
        }
        sMask[tid] = tid < cnt ? (uint8_t)(ent & 0xffu) : (uint8_t)0;
      }
      __syncthreads();

      if ((uint32_t)warp_last > sPos[0]) {  // the batch's first entry is its closest
        const int n_w = warp_compact(sMask, cnt, warp, lane, sList);
        // park one list entry (phase A); `valid`: this lane blended it in the forward pass
        auto park = [&](int jj, bool valid, const AlphaEval& ev) {
          float w = 0.0f, g_sigma = 0.0f;
          if (valid) {
            const float one_m = 1.0f - ev.alpha;
            // 1 - alpha lies in [1 - alpha_clamp, 1]: MUFU.RCP alone (1 ulp, no range fix-up) is within the 1e-3 gradient
            // tolerance by four orders of magnitude even compounded over a pixel's whole list
            float inv;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(one_m));
            T = T * inv;  // transmittance in front of this Gaussian
            w = ev.alpha * T;
            // four partial sums: a 16-long dependent FMA chain is 64 cycles of latency in a latency-bound loop
            f32x2 d01 = pack2(0.0f, 0.0f), d23 = d01;  // packed pairs: 8 FFMA2 instead of 16 FFMA
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 f4 = sF[4 * jj + c];
              d01 = fma2(g2[2 * c], pack2(f4.x, f4.y), d01);
              d23 = fma2(g2[2 * c + 1], pack2(f4.z, f4.w), d23);
            }
            float d0, d1, d2, d3;
            unpack2(d01, d0, d1);
            unpack2(d23, d2, d3);
            float dotgf = (d0 + d1) + (d2 + d3);
            float g_extra = 0.0f;
            if (!kCamera) {
              const float2 c2 = sC[jj];
              const float r_rs = fmaf(c2.y, t, c2.x);  // r_rs = r + v_r t
              dotgf = fmaf(g_D, r_rs, dotgf);
              if (los_on && r_rs < los_cut) g_extra = g_los;  // d los / d alpha_i = 1 in front of the cut
            }
            const float g_a = dotgf * T + (K - S) * inv + g_extra;
            S = fmaf(w, dotgf, S);
            if (!ev.clamped) g_sigma = -ev.alpha * g_a;  // alpha = rho exp(-sigma), sigma = qf / 2; clamped: constant
          }
          ws.w[n_slots * kWStride + lane] = w;
          ws.gs[n_slots * kPanelStride + lane] = g_sigma;
          // the record travels with the entry — copied for all pending slots at once (copy_pending: 24 lanes, one
          // record part each) when the panel is full or the batch ends, instead of by three lanes per entry
          jpack |= (unsigned long long)jj << (8 * n_slots);
          pend |= 1u << n_slots;
          if (++n_slots == kChunkS) {
            copy_pending();
            reduce_panel8<kCamera>(ws, n_slots, lane, s.d_f, rg, pg, dt_local, wrap);
            n_slots = 0;
            jpack = 0ull;
          }
        };
        // two entries per iteration: independent quadratic forms (ILP), parked in back-to-front order; the camera
        // parks without the vote (-3% on its kernel)
        for (int k = n_w - 1; k >= 0; k -= 2) {
          const bool has1 = k >= 1;
          const int j0 = sList[k], j1 = sList[has1 ? k - 1 : k];
          const float4 a0 = sA[j0], b0 = sB[j0], a1 = sA[j1], b1 = sB[j1];
          float dx0, dy0, dx1, dy1;
          const float qf0 = kCamera ? alpha_qform_packed(pack2(a0.x, a0.y), pack2(a0.z, a0.w), b0, pack2(qx, qy), pack2(t, t), dx0, dy0)
                                    : alpha_qform<!kCamera>(a0, b0, qx, qy, t, dx0, dy0, wrap);
          const float qf1 = kCamera ? alpha_qform_packed(pack2(a1.x, a1.y), pack2(a1.z, a1.w), b1, pack2(qx, qy), pack2(t, t), dx1, dy1)
                                    : alpha_qform<!kCamera>(a1, b1, qx, qy, t, dx1, dy1, wrap);
          AlphaEval ev;
          bool valid = ((int)sPos[j0] < last) && alpha_finish(qf0, b0.w, dx0, dy0, s.qform_max, s.alpha_clamp, s.alpha_min, ev);
          if (sure || __any_sync(0xffffffffu, valid)) park(j0, valid, ev);
          valid = has1 && ((int)sPos[j1] < last) && alpha_finish(qf1, b1.w, dx1, dy1, s.qform_max, s.alpha_clamp, s.alpha_min, ev);
          if ((sure && has1) || __any_sync(0xffffffffu, valid)) park(j1, valid, ev);
        }
      }
      if (pend) copy_pending();  // the staged records go away with the batch
      if (batch > 0) {  // next batch's records -> L2
        prefetch_l2(&p.geomA[src_next]);
        prefetch_l2(&p.geomB[src_next]);
        prefetch_l2(&p.feat[4 * (size_t)src_next]);
        if (!kCamera) prefetch_l2(&p.geomC[src_next]);
      }
      __syncthreads();  // every warp is done with the staged batch
    }
    if (n_slots > 0) {  // drain what is left of this pass
      __syncwarp();
      reduce_panel8<kCamera>(ws, n_slots, lane, s.d_f, rg, pg, dt_local, wrap);
      n_slots = 0;
    }
    jpack = 0ull;
    __syncthreads();  // patch boxes / staging / per-query rows are reused by the next ray pass
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

// ------------------------------------------------------------------------------------------------
// Lidar compositing backward, version 2 (pairs with raster_lidar.cu's forward).
//
// A lidar list entry is blended by ~8 of a warp's 32 rays and needed by 1.06 of the tile's 8 warps. The shared kernel
// above walks a warp's hit entries one at a time with all 32 lanes (phase A: ~140 instructions per entry for ~8 useful
// lanes) behind CTA-wide staging barriers. Here
//   * every warp works on its own: it reads ITS hit words (one per list entry: the rays that blended it, saved by the
//     forward), fetches the records of the entries it blended into a private ring — no CTA barrier anywhere;
//   * phase A is lane-divergent: a lane walks only the entries ITS ray blended (bits of the hit words, kept per lane in
//     ring order), back to front, so different lanes are at different entries of the 16-entry chunk — about half the
//     trips of the entry-by-entry walk — and parks (w, dL/dsigma) in the [slot][lane] panel (zero-filled first);
//   * phase B (channel product as split-tf32 MMAs, raw moments, REDs) is reduce_panel above, unchanged.
// ------------------------------------------------------------------------------------------------
template <bool kLos>
__global__ void __launch_bounds__(256, 2)
k_raster_bwd_lidar(const __grid_constant__ Sensor s, ProjDev p, const uint32_t* __restrict__ vals,
                   const uint32_t* __restrict__ tile_begin, const uint32_t* __restrict__ tile_end,
                   const float4* __restrict__ rays, const int64_t* __restrict__ ray_begin, const int64_t* __restrict__ ray_end,
                   const uint32_t* __restrict__ tile_order, int tile_first, RasterOutDev fwd, const float* __restrict__ g_blend16,
                   const float* __restrict__ g_alpha, RasterGradDev rg, ParamGradDev pg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* sA = reinterpret_cast<float4*>(smem_raw);                    // kBatch
  float4* sB = sA + kBatch;                                            // kBatch
  float4* sF = sB + kBatch;                                            // 4 kBatch, PLANAR: sF[c * kBatch + j]
  float2* sC = reinterpret_cast<float2*>(sF + 4 * kBatch);             // kBatch
  uint32_t* sSrc = reinterpret_cast<uint32_t*>(sC + kBatch);           // kBatch
  uint32_t* sHw = sSrc + kBatch;                                       // 8 x kBatch: [warp][entry] hit words of the batch
  WarpScratch* sWs = reinterpret_cast<WarpScratch*>(sHw + 8 * kBatch); // 8
  uint8_t* sListAll = reinterpret_cast<uint8_t*>(sWs + 8);             // 8 x kBatch
  __shared__ int s_max_last;
  __shared__ int s_wcnt[8];

  const int tile = tile_order ? (int)tile_order[blockIdx.x] : tile_first + (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint8_t* sList = sListAll + kBatch * warp;
  const uint32_t* myHw = sHw + kBatch * warp;
  WarpScratch& ws = sWs[warp];
  const uint32_t lb = tile_begin[tile], le = tile_end[tile];
  if (le <= lb) return;
  const bool wrap = fwd.tile_wrap[tile] != 0;  // certified per tile by the forward (raster_common.cuh)
  const int64_t qpos = ray_begin[tile] + tid;
  const bool inside = qpos < ray_end[tile];
  float qx = 0.0f, qy = 0.0f, t = 0.0f;
  int64_t pix = 0;
  if (inside) {
    const float4 r = rays[qpos];
    qx = r.x; qy = r.y; t = r.z;
    pix = (int64_t)__float_as_uint(r.w);
  }
  int last = 0;
  float los_cut = 0.0f, g_los = 0.0f;
  if (kLos && inside) { los_cut = fwd.los_cut[pix]; g_los = fwd.g_los[pix]; }
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
    const float A = 1.0f - T;
    if (A > 1e-6f) {  // expected = D / A
      g_D = g_out[13] / A;
      g_acc += -g_out[13] * (fwd.range_blend[pix] / A) / A;
    } else {
      g_D = g_out[13];
    }
#pragma unroll
    for (int k = 0; k < kChannels; ++k)
      if (k >= s.channels) g_out[k] = 0.0f;
    K = g_acc * T;
  }
  float S = 0.0f;  // sum_c g_c * suffix_c + g_D * suffix_r
  f32x2 g2[kChannels / 2];  // the upstream gradient as packed pairs (phase A's dot product)
#pragma unroll
  for (int k = 0; k < kChannels / 2; ++k) g2[k] = pack2(g_out[2 * k], g_out[2 * k + 1]);
  {  // per-query data for phase B (read there as broadcasts)
    float* row = &ws.px[lane * kPxStride];
    *reinterpret_cast<float4*>(row) = make_float4(qx, qy, t, g_D);
    float gcol[kChannels];
#pragma unroll
    for (int k = 0; k < kChannels; ++k) gcol[k] = g_out[k];
    gcol[13] = g_D; gcol[14] = g_D * t; gcol[15] = 0.0f;  // columns 13, 14 of the channel product: d/d range, d/d v_r
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<float4*>(row + 4 + 4 * k) = make_float4(gcol[4 * k], gcol[4 * k + 1], gcol[4 * k + 2], gcol[4 * k + 3]);
  }
  auto zero_panel = [&]() {  // lanes that did not blend an entry contribute nothing
    float4* w4 = reinterpret_cast<float4*>(ws.w);
    float4* g4 = reinterpret_cast<float4*>(ws.gs);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = lane; i < kChunk * kWStride / 4; i += 32) w4[i] = z;
    for (int i = lane; i < kChunk * kPanelStride / 4; i += 32) g4[i] = z;
  };
  zero_panel();
  if (tid == 0) s_max_last = 0;
  __syncthreads();
  int warp_last = last;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) warp_last = max(warp_last, __shfl_xor_sync(0xffffffffu, warp_last, o));
  if (lane == 0 && warp_last > 0) atomicMax(&s_max_last, warp_last);
  __syncthreads();
  const int max_last = s_max_last;
  if (max_last == 0) return;

  const uint32_t* const hitw = fwd.hit_rows + ((size_t)(lb >> 8) + (size_t)tile) * 2048u;  // [block][warp][entry & 255]
  int n_slots = 0;  // parked entries (warp-uniform); the panel persists across batches
  float dt_unused = 0.0f;

  // Compact hit list (as in k_raster_bwd): half of a lidar tile's entries were blended by some warp. The CTA scans its
  // hit bytes (bit w: warp w has a hit word for the entry), 1,024 per step, and keeps (position << 8 | byte) of the
  // non-zero ones, in list order; the batches below are dense.
  uint32_t* const hl = fwd.hit_list + lb;
  int n_hit = 0;  // CTA-uniform
  {
    const uint32_t w0 = lb >> 2;
    const uint32_t* hit4 = reinterpret_cast<const uint32_t*>(fwd.hit);
    for (uint32_t wbase = w0; 4u * wbase < lb + (uint32_t)max_last; wbase += 256u) {
      const uint32_t word = hit4[wbase + tid];
      const int pos0 = (int)(4u * (wbase + tid)) - (int)lb;
      uint32_t ent[4];
      int c4 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t m = (word >> (8 * i)) & 0xffu;
        const int ps = pos0 + i;
        if (m != 0u && ps >= 0 && ps < max_last) ent[c4++] = ((uint32_t)ps << 8) | m;
      }
      int incl = c4;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wcnt[warp] = incl;
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int c = s_wcnt[w];
        if (w < warp) before += c;
        total += c;
      }
      uint32_t* dst = hl + n_hit + before + (incl - c4);
      for (int i = 0; i < c4; ++i) dst[i] = ent[i];
      n_hit += total;
      __syncthreads();  // s_wcnt is reused; after the last step: the list is visible to the whole CTA
    }
  }

  // a batch's list entries, hit words and record indices are fetched one batch ahead and its records prefetched into
  // L2: staging then starts with the record loads instead of a chain of dependent global loads
  uint32_t hw_next[8], ent_next = 0u, src_next = 0u;
  auto fetch = [&](int i) {  // compact entry i of this thread's next batch
    ent_next = hl[i];
    const uint32_t ps = ent_next >> 8;
    src_next = vals[lb + ps];
#pragma unroll
    for (int w = 0; w < 8; ++w)
      hw_next[w] = ((ent_next >> w) & 1u) ? hitw[(size_t)(ps >> 8) * 2048u + w * 256 + (ps & 255u)] : 0u;
  };
#pragma unroll
  for (int w = 0; w < 8; ++w) hw_next[w] = 0u;
  const int nbat = (n_hit + kBatch - 1) / kBatch;
  if (nbat > 0 && (nbat - 1) * kBatch + tid < n_hit) fetch((nbat - 1) * kBatch + tid);
  for (int batch = nbat - 1; batch >= 0; --batch) {
    const int cnt = min(kBatch, n_hit - batch * kBatch);
    // thread = compact entry: the hit words of the warps that blended it, its record
    {
      uint32_t hwv[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) hwv[w] = hw_next[w];
      const uint32_t src = src_next;
      if (batch > 0) fetch((batch - 1) * kBatch + tid);  // the batch in front of this one is always full
      if (tid < cnt) {
#pragma unroll
        for (int w = 0; w < 8; ++w) sHw[w * kBatch + tid] = hwv[w];
        sSrc[tid] = src;
        sA[tid] = p.geomA[src];
        sB[tid] = p.geomB[src];
        sC[tid] = p.geomC[src];
#pragma unroll
        for (int k = 0; k < 4; ++k) sF[k * kBatch + tid] = p.feat[4 * (size_t)src + k];
      }
    }
    __syncthreads();

    {
      // the warp's hit entries of this batch, back to front
      int n_w = 0;
      for (int c0 = (cnt - 1) & ~31; c0 >= 0; c0 -= 32) {
        const int j = c0 + (31 - lane);  // lane 0 takes the highest entry: ballot ranks are back-to-front ranks
        const bool bit = j < cnt && myHw[j] != 0u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        if (bit) sList[n_w + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)j;
        n_w += __popc(bal);
      }
      __syncwarp();
      for (int k0 = 0; k0 < n_w;) {
        const int g = min(kChunk - n_slots, n_w - k0);
        // my ray's bit of each of the g entries; their records for phase B
        uint32_t hw_e = 0u;
        if (lane < g) {
          const int j = sList[k0 + lane];
          hw_e = myHw[j];
          ws.gAB[n_slots + lane] = sA[j];
          ws.gAB[kChunk + n_slots + lane] = sB[j];
          ws.src[n_slots + lane] = sSrc[j];
        }
        uint32_t mybits = transpose32(hw_e, lane);  // bit e: my ray blended entry k0 + e
        // ---- phase A: every lane walks the entries ITS ray blended, back to front ---------------
        // Two hits per trip: alpha, 1 / (1 - alpha) and the dot product with the upstream gradient do not depend on the
        // walk and are evaluated for both first, branch-free, so that the two chains of gathers and arithmetic
        // interleave (the kernel is latency-bound); the walk itself (T, the suffix scalar) is a few dependent operations.
        auto eval = [&](int e, float& al, float& inv, float& dot, float& gext, bool& ok, bool& clampd) {
          const int j = sList[k0 + e];
          const float4 gA = sA[j], gB = sB[j];
          float dx, dy;
          const float qf = alpha_qform<true>(gA, gB, qx, qy, t, dx, dy, wrap);
          // alpha_finish without its early exits (same operations, same decisions)
          const float gauss = detmath::exp_bounded((qf <= s.qform_max) ? fminf(__fmul_rn(-0.5f, qf), 88.0f) : 0.0f);
          al = __fmul_rn(gB.w, gauss);
          clampd = al > s.alpha_clamp;
          if (clampd) al = s.alpha_clamp;
          ok = (qf <= s.qform_max) && (al >= s.alpha_min);  // (the bit says blended)
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(1.0f - al));  // [1 - alpha_clamp, 1]: 1 ulp, no range fix-up needed
          f32x2 d01 = pack2(0.0f, 0.0f), d23 = d01;  // packed pairs: 8 FFMA2 instead of 16 FFMA
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 f4 = sF[c * kBatch + j];
            d01 = fma2(g2[2 * c], pack2(f4.x, f4.y), d01);
            d23 = fma2(g2[2 * c + 1], pack2(f4.z, f4.w), d23);
          }
          float d0, d1, d2, d3;
          unpack2(d01, d0, d1);
          unpack2(d23, d2, d3);
          const float2 c2 = sC[j];
          const float r_rs = fmaf(c2.y, t, c2.x);  // r_rs = r + v_r t
          dot = fmaf(g_D, r_rs, (d0 + d1) + (d2 + d3));
          gext = (kLos && r_rs < los_cut) ? g_los : 0.0f;  // d los / d alpha_i = 1 in front of the cut
        };
        auto apply = [&](int e, float al, float inv, float dot, float gext, bool clampd) {
          T = T * inv;  // transmittance in front of this Gaussian
          const float w = al * T;
          const float g_a = dot * T + (K - S) * inv + gext;
          S = fmaf(w, dot, S);
          ws.w[(n_slots + e) * kWStride + lane] = w;
          if (!clampd) ws.gs[(n_slots + e) * kPanelStride + lane] = -al * g_a;  // alpha = rho exp(-sigma); clamped: constant
        };
        while (mybits != 0u) {
          const int e0 = __ffs(mybits) - 1;
          mybits &= mybits - 1u;
          const bool has1 = mybits != 0u;
          const int e1 = has1 ? __ffs(mybits) - 1 : e0;
          mybits &= mybits - 1u;  // (0 stays 0)
          float al0, inv0, dot0, gx0, al1, inv1, dot1, gx1;
          bool ok0, ok1, cl0, cl1;
          eval(e0, al0, inv0, dot0, gx0, ok0, cl0);
          eval(e1, al1, inv1, dot1, gx1, ok1, cl1);
          if (ok0) apply(e0, al0, inv0, dot0, gx0, cl0);
          if (has1 && ok1) apply(e1, al1, inv1, dot1, gx1, cl1);
        }
        n_slots += g;
        k0 += g;
        __syncwarp();
        if (n_slots == kChunk) {
          reduce_panel<false>(ws, n_slots, lane, s.d_f, rg, pg, dt_unused, wrap);
          zero_panel();
          __syncwarp();
          n_slots = 0;
        }
      }
    }
    if (batch > 0) {  // next batch's records -> L2
      prefetch_l2(&p.geomA[src_next]);
      prefetch_l2(&p.geomB[src_next]);
      prefetch_l2(&p.geomC[src_next]);
      prefetch_l2(&p.feat[4 * (size_t)src_next]);
    }
    __syncthreads();  // every warp is done with the staged batch
  }
  if (n_slots > 0) {
    __syncwarp();
    reduce_panel<false>(ws, n_slots, lane, s.d_f, rg, pg, dt_unused, wrap);
  }
}

constexpr size_t kBwdLidarSmem = kBatch * 16 * 2 + 4 * kBatch * 16 + kBatch * 8 + kBatch * 4 + 8 * kBatch * 4 + 8 * sizeof(WarpScratch) + 8 * kBatch;

void launch_raster_bwd_lidar(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                             const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                             const uint32_t* tile_order, const RasterOutDev& fwd, const float* g_blend16, const float* g_alpha,
                             const RasterGradDev& rg, const ParamGradDev& pg, cudaStream_t st, int tile_first, int tile_count) {
  const int tiles = tile_count < 0 ? s.tiles_x * s.tiles_y : tile_count;
  if (tiles <= 0) return;
  if (tile_count < 0) tile_first = 0;
  else tile_order = nullptr;
  static DeviceOnce once;
  once.run([] {
    cudaFuncSetAttribute(k_raster_bwd_lidar<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdLidarSmem);
    cudaFuncSetAttribute(k_raster_bwd_lidar<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdLidarSmem);
  });
  if (fwd.los_cut && fwd.g_los)
    k_raster_bwd_lidar<true><<<tiles, 256, kBwdLidarSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                               tile_first, fwd, g_blend16, g_alpha, rg, pg);
  else
    k_raster_bwd_lidar<false><<<tiles, 256, kBwdLidarSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                                tile_first, fwd, g_blend16, g_alpha, rg, pg);
}

constexpr size_t kBwdSmem = kBatch * 16 * 2 + 4 * kBatch * 16 + kBatch * 8 + kBatch * 4 * 2 + 8 * sizeof(PatchBox) +
                            8 * sizeof(WarpScratchT<kChunkS>) + kBatch + 8 * kBatch;

void launch_raster_bwd(const Sensor& s, const ProjDev& p, const uint32_t* vals, const uint32_t* tile_begin,
                       const uint32_t* tile_end, const float4* rays, const int64_t* ray_begin, const int64_t* ray_end,
                       const uint32_t* tile_order, const RasterOutDev& fwd, const float* g_blend16, const float* g_alpha,
                       const RasterGradDev& rg, const ParamGradDev& pg, float* d_time_offset, cudaStream_t st, int tile_first,
                       int tile_count) {
  const int tiles = tile_count < 0 ? s.tiles_x * s.tiles_y : tile_count;
  if (tiles <= 0) return;
  if (tile_count < 0) tile_first = 0;
  else tile_order = nullptr;
  static DeviceOnce once;
  once.run([] {
    cudaFuncSetAttribute(k_raster_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
    cudaFuncSetAttribute(k_raster_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
    cudaFuncSetAttribute(k_raster_bwd<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
  });
  if (s.is_camera)
    k_raster_bwd<true><<<tiles, 256, kBwdSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                     tile_first, fwd, g_blend16, g_alpha, rg, pg, d_time_offset);
  else if (fwd.los_cut && fwd.g_los)
    k_raster_bwd<false, true><<<tiles, 256, kBwdSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                            tile_first, fwd, g_blend16, g_alpha, rg, pg, d_time_offset);
  else
    k_raster_bwd<false><<<tiles, 256, kBwdSmem, st>>>(s, p, vals, tile_begin, tile_end, rays, ray_begin, ray_end, tile_order,
                                                      tile_first, fwd, g_blend16, g_alpha, rg, pg, d_time_offset);
}

}  // namespace sb
