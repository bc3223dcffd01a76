// decode_image — the camera ConvDecoder (Eq. 7-8).
//
// The only dense contraction of the system, so the only kernel here that runs on the tensor cores: every 3x3, 32 -> 32
// convolution is an implicit GEMM issued as tcgen05.mma (kind::tf32, M = 128 pixels, N = 32 or 64 output channels —
// two stacked taps —, K = 8 input channels per instruction) with the accumulator in tensor memory.
//
// Layer list (the reference ships no decoder; SPEC fixes width, depth, kernel size, padding and the output map, the
// rest is fixed in oracle/decoder_oracle.hpp's header and mirrored here):
//   x0 = (feature[d_f], ray_direction(u, v) [scene.hpp:119-122], embedding[8], 0 ...)        32 channels
//   h0 = conv0(x0); h1 = h0 + conv2(relu(conv1(relu(h0)))); h2 = h1 + conv4(relu(conv3(relu(h1))))
//   y = Wh h2 + bh;  I_c = (1 + y_c) rgb_c + y_{3+c}
//
// Activations are pixel-interleaved, 32 floats = 128 B per pixel. One CTA tile = 2 image rows x 128 pixels. The tile's
// halo (4 rows x 130 pixels, reflect padding resolved while loading) is staged in shared memory as eight planes of
// 16-byte units, plane c holding channels 4c..4c+3 of every halo pixel: unit (c, row, px) = c * kCPlane + row * 130 + px.
// That is exactly the tensor core's no-swizzle K-major operand layout (8 rows x 16 B core matrices, consecutive rows
// 16 B apart, 8-row groups 128 B apart, the two 16-byte K chunks of one instruction one plane apart), and in it a
// filter tap (ky, kx) is nothing but a different start address — the nine taps of a convolution read the one staged
// halo, no im2col copy, no per-tap reload. The weights of a layer (9 taps x 32 x 32, 36 KB) are staged once per CTA
// in the same layout; CTAs are persistent (one per SM) and warp-specialised: producer warps stage the next tile while
// one lane issues the current tile's MMAs and the epilogue warps drain the previous one (k_conv3x3_tc below).
// Operands are rounded to tf32 (round-to-nearest) while staging; accumulation is fp32.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace sb {
namespace {

constexpr int kCTW = 128;                      // tile width in pixels = M of one MMA
constexpr int kCTR = 2;                        // tile rows (one accumulator of 32 TMEM columns each)
constexpr int kCHW = kCTW + 2, kCHR = kCTR + 2;
constexpr int kCPlane = kCHR * kCHW + 1;       // 521 units of 16 B; odd, so staging stores are bank-conflict free
constexpr int kCXUnits = 8 * kCPlane;          // halo: 66,688 B
constexpr int kCWUnits = 9 * 8 * 32;           // weights: 36,864 B
constexpr int kCThreads = 256;                 // warp w: tile row w / 4, TMEM lanes 32 (w % 4) ..
constexpr int kCTmemCols = 32 * kCTR;          // 64
constexpr int kCTries = 1 << 18;                // bounded wait on the MMA completion barrier

// tcgen05 instruction descriptor: D = f32 (bits 4-5 = 1), A = B = tf32 (bits 7-9, 10-12 = 2), both K-major (bits 15,
// 16 = 0), N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor, no swizzle: start address, leading (K chunk) and stride (8-row group) byte offsets
// in 16-byte units, descriptor version 1 at bit 46
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// Split-tf32 ("3xTF32") operands for the precise mode: part 0 = hi = tf32(x), part 1 = lo = tf32(x - hi). A product
// x w = hi hi + lo hi + hi lo + O(2^-22 |x w|): three passes of the same kernel, accumulated in fp32 through the
// residual input, reach fp32 accuracy on the tf32 tensor cores.
__device__ __forceinline__ float tf32_part(float x, int part) {
  const float hi = to_tf32(x);
  return part ? to_tf32(x - hi) : hi;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate) : "memory");
}

__device__ __forceinline__ void tmem_load32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, "
      "%24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ int reflect_clamped(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * (n - 1) - i;
  return min(max(i, 0), n - 1);
}

struct ConvArgs {
  const float* x;        // H x W x 32
  const float* w;        // 9216 weights [co][ky][kx][ci] + 32 bias
  const float* res;      // residual added to the output (null: none)
  float* y;              // H x W x 32 (unused by the head variant)
  int H, W;
  int relu_in;
  int ext;               // 0: y = conv(x), reflect padding, H x W. 1 (input-gradient form): zero padding and the output
                         // domain grown by one pixel on every side, y is (H + 2) x (W + 2) — see k_dec_fold
  // head variant: h2 = res + conv -> y6 = Wh h2 + bh -> image = (1 + y[0:3]) * rgb + y[3:6]
  const float* head;     // 192 + 6
  const float* blend;    // P x blend_stride, rgb first
  int blend_stride;
  float* image;          // P x 3
  float* h2;             // trunk output kept for the backward (may be null)
  int* err;              // set to 1 if a pipeline barrier timed out
  int xpart, wpart;      // which tf32 part of the activations / weights is staged (0 hi, 1 lo; tf32_part)
  int no_bias;           // passes 2 and 3 of the precise mode: the bias went in with pass 1
};

// ---- mbarrier helpers (bounded waits: a protocol mistake must not hang the device) ----
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 t;\n\tmbarrier.arrive.shared::cta.b64 t, [%0];\n\t}\n" :: "r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (int tries = 0; tries < kCTries && !done; ++tries)   // try_wait suspends the warp: no issue slots burnt
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  return done != 0;
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(bar) : "memory");
}

// Warp-specialised, persistent, one CTA per SM. Three roles run a tile apart from each other:
//   warps 8..15  producers: stage tile i+1's halo into the other halo buffer          (full[s] / empty[s])
//   warp 16      one lane issues tile i's 72 MMAs into accumulator set i & 1          (tfull[s] / tempty[s])
//   warps 0..7   epilogue of tile i-1: TMEM -> registers -> shared-memory transpose -> coalesced global stores
#ifndef SB_PROD_WARPS
#define SB_PROD_WARPS 6
#endif
constexpr int kWsEpiWarps = 8, kWsProdWarps = SB_PROD_WARPS;   // epilogue warp w: tile row w / 4, TMEM lanes 32 (w % 4) ..
constexpr int kWsThreads = 32 * (kWsEpiWarps + kWsProdWarps + 1);   // 416
constexpr int kWsEpiFloats = 32 * 32;                               // per epilogue warp: 32 pixels x 32 channels
constexpr int kWsSmemBytes = (2 * kCXUnits + kCWUnits) * 16 + kWsEpiWarps * kWsEpiFloats * 4 + 32 * 4 + 256 * 4 + 128;

template <bool kHead>
__global__ void __launch_bounds__(kWsThreads, 1) k_conv3x3_tc(ConvArgs a) {
  static_assert(kWsEpiWarps == 4 * kCTR, "one epilogue warp per (tile row, TMEM lane quarter)");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* sX = reinterpret_cast<float4*>(smem_raw);              // two halo buffers
  float4* sW = sX + 2 * kCXUnits;
  float* sEpi = reinterpret_cast<float*>(sW + kCWUnits);         // [4 warps][32 px][32 ch], 16-byte units XOR-swizzled
  float* sBias = sEpi + kWsEpiWarps * kWsEpiFloats;
  float* sHead = sBias + 32;                                     // 198 used
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sHead + 256);     // full[2], empty[2], tfull[2], tempty[2]
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBar + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Ho = a.H + 2 * a.ext, Wo = a.W + 2 * a.ext;  // output domain
  const int tiles_x = (Wo + kCTW - 1) / kCTW, tiles_y = (Ho + kCTR - 1) / kCTR;
  const int n_tiles = tiles_x * tiles_y;
  const uint32_t bar0 = smem_u32(sBar);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 16u + 8u * s; };
  auto tfull = [&](int s) { return bar0 + 32u + 8u * s; };
  auto tempty = [&](int s) { return bar0 + 48u + 8u * s; };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(sTmem)), "r"(2 * kCTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(full(s), 32 * kWsProdWarps);
      mbar_init(empty(s), 1);
      mbar_init(tfull(s), 1);
      mbar_init(tempty(s), 32 * kWsEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the layer's weights, once per CTA: unit (((kx * 8 + c) * 3 + (2 - ky)) * 32 + co) = W[co][ky][kx][4c .. 4c+3]: for a
  // filter column kx and K chunk c the rows of ky = 2, 1, 0 follow each other, so 64 consecutive rows are the taps
  // (ky, ky - 1) — the two taps that read the SAME halo row for the tile's two output rows (see the MMA loop)
  {
    const float4* gw = reinterpret_cast<const float4*>(a.w);
    for (int i = tid; i < kCWUnits; i += kWsThreads) {
      const int co = i / 72, rem = i - co * 72, tap = rem >> 3, c = rem & 7;
      const int ky = tap / 3, kx = tap - 3 * ky;
      float4 v = __ldg(gw + i);
      v.x = tf32_part(v.x, a.wpart); v.y = tf32_part(v.y, a.wpart); v.z = tf32_part(v.z, a.wpart); v.w = tf32_part(v.w, a.wpart);
      sW[((kx * 8 + c) * 3 + (2 - ky)) * 32 + co] = v;
    }
    if (tid < 32) sBias[tid] = a.no_bias ? 0.f : __ldg(a.w + 9216 + tid);
    if (kHead)
      for (int i = tid; i < 198; i += kWsThreads) sHead[i] = __ldg(a.head + i);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *sTmem;
  bool ok = true;

  if (warp >= kWsEpiWarps && warp < kWsEpiWarps + kWsProdWarps) {
    // =============================== producers ===============================
    const int t = tid - 32 * kWsEpiWarps;
    const int c = t & 7, pl = t >> 3;
    const float relu_floor = a.relu_in ? 0.f : -INFINITY;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int s = it & 1;
      const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
      const int x0 = tx * kCTW, y0 = ty * kCTR;
      if (!mbar_wait(empty(s), ((it >> 1) & 1) ^ 1)) { ok = false; break; }
      float4* dstX = sX + s * kCXUnits;
      constexpr int kPl = 4 * kWsProdWarps;                 // pixel lanes
      constexpr int kPxIters = (kCHW + kPl - 1) / kPl;
      // two halo rows (12 loads) in flight per thread. (cp.async straight into the planes + a fix-up pass for ReLU and
      // rounding was measured 9% slower.)
#pragma unroll
      for (int r0 = 0; r0 < kCHR; r0 += 2) {
        float4 v[2][kPxIters];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          int gy = y0 - 1 + r0 + rr - a.ext;
          const bool row_out = a.ext && (gy < 0 || gy >= a.H);
          gy = reflect_clamped(gy, a.H);
          const float4* rowp = reinterpret_cast<const float4*>(a.x + (int64_t)gy * a.W * 32) + c;
#pragma unroll
          for (int k = 0; k < kPxIters; ++k) {
            const int px = pl + kPl * k;
            int gx = x0 - 1 + px - a.ext;
            const bool out = row_out || (a.ext && (gx < 0 || gx >= a.W));
            gx = reflect_clamped(gx, a.W);
            v[rr][k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (px < kCHW && !out) v[rr][k] = __ldg(rowp + gx * 8);
          }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
          for (int k = 0; k < kPxIters; ++k) {
            const int px = pl + kPl * k;
            if (px < kCHW) {
              float4 q = v[rr][k];
              q.x = tf32_part(fmaxf(q.x, relu_floor), a.xpart); q.y = tf32_part(fmaxf(q.y, relu_floor), a.xpart);
              q.z = tf32_part(fmaxf(q.z, relu_floor), a.xpart); q.w = tf32_part(fmaxf(q.w, relu_floor), a.xpart);
              dstX[c * kCPlane + (r0 + rr) * kCHW + px] = q;
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy stores -> tensor-core reads
      mbar_arrive(full(s));
    }
  } else if (warp == kWsEpiWarps + kWsProdWarps) {
    // =============================== MMA issuer (one lane) ===============================
    if (lane == 0) {
      const uint32_t w_addr = smem_u32(sW);
      constexpr uint32_t a_lbo = (uint32_t)kCPlane * 16u, a_sbo = 128u, b_lbo = 3u * 512u, b_sbo = 128u;
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        const uint32_t par = (it >> 1) & 1;
        if (!mbar_wait(tempty(s), par ^ 1) || !mbar_wait(full(s), par)) { ok = false; break; }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t x_addr = smem_u32(sX + s * kCXUnits);
        const uint32_t d_addr = tmem_base + (uint32_t)(s * kCTmemCols);
        // Halo row h feeds output row r through tap ky = h - r. Rows h = 1, 2 feed BOTH output rows: one N = 64
        // instruction (weights of ky = h and ky = h - 1 stacked, accumulator columns of r = 0 and r = 1 adjacent)
        // instead of two N = 32 ones — 48 instructions per tile instead of 72, a third less operand traffic.
        // The accumulate flag covers the whole instruction, so each output row is first touched (and cleared) by the
        // halo row that feeds it alone: h = 0 for row 0, h = 3 for row 1; the shared rows h = 1, 2 then accumulate.
#pragma unroll
        for (int hh = 0; hh < kCHR; ++hh) {
          const int h = hh == 0 ? 0 : (hh == 1 ? 3 : hh - 1);
          const int r_lo = h >= 3 ? 1 : 0;                       // first output row fed
          const int n_rows = (h == 0 || h == 3) ? 1 : 2;         // output rows fed
          const int ky_hi = h - r_lo;                            // tap of the first one (the second: ky_hi - 1)
          const uint32_t idesc = (kIdesc & ~(0x3Fu << 17)) | ((uint32_t)(32 * n_rows >> 3) << 17);
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint32_t aa = x_addr + (uint32_t)((2 * ks) * kCPlane + h * kCHW + kx) * 16u;
              const uint32_t bb = w_addr + (uint32_t)(((kx * 8 + 2 * ks) * 3 + (2 - ky_hi)) * 32) * 16u;
              const uint32_t acc_flag = ((h == 0 || h == 3) && kx == 0 && ks == 0) ? 0u : 1u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                  :: "r"(d_addr + (uint32_t)(r_lo * 32)), "l"(smem_desc(aa, a_lbo, a_sbo)), "l"(smem_desc(bb, b_lbo, b_sbo)),
                     "r"(idesc), "r"(acc_flag) : "memory");
            }
          }
        }
        umma_commit(empty(s));    // halo buffer s may be refilled once these MMAs have read it
        umma_commit(tfull(s));    // accumulator set s is complete
      }
    }
    __syncwarp();
  } else if (warp < kWsEpiWarps) {
    // =============================== epilogue ===============================
    float* my = sEpi + warp * kWsEpiFloats;
    const int cq = lane & 7, pq = lane >> 3;      // coalesced phase: 16-byte unit, pixel within a group of 4
    const float4 bias4 = reinterpret_cast<const float4*>(sBias)[cq];
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int s = it & 1;
      const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
      const int x0 = tx * kCTW, y0 = ty * kCTR;
      if (!mbar_wait(tfull(s), (it >> 1) & 1)) { ok = false; break; }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      {
        const int r = warp >> 2, wq = warp & 3;
        float acc[32];
        tmem_load32(tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(s * kCTmemCols + r * 32), acc);
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(tempty(s));   // the accumulators are in registers: hand the set back
        // lane = pixel -> shared memory (unit c of pixel l at c ^ (l & 7)) -> lane = (pixel group, unit)
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c)
          reinterpret_cast<float4*>(my)[lane * 8 + (c ^ (lane & 7))] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
        __syncwarp();
        const int gy = y0 + r;
        const int gx0 = x0 + wq * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int l = 4 * k + pq;
          float4 v = reinterpret_cast<float4*>(my)[l * 8 + (cq ^ (l & 7))];
          v.x += bias4.x; v.y += bias4.y; v.z += bias4.z; v.w += bias4.w;
          const int gx = gx0 + l;
          const bool live = gx < Wo && gy < Ho;
          const int64_t p = (int64_t)gy * Wo + gx;
          if (live && a.res) {
            const float4 q = *(reinterpret_cast<const float4*>(a.res + p * 32) + cq);  // plain load: res may alias y (precise mode)
            v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
          }
          if (kHead) {
            if (live && a.h2) reinterpret_cast<float4*>(a.h2 + p * 32)[cq] = v;
            reinterpret_cast<float4*>(my)[l * 8 + (cq ^ (l & 7))] = v;   // back for the per-pixel head
          } else if (live) {
            reinterpret_cast<float4*>(a.y + p * 32)[cq] = v;
          }
        }
        if (kHead) {
          __syncwarp();
          const int gx = gx0 + lane;
          if (gx < Wo && gy < Ho) {
            const int64_t p = (int64_t)gy * Wo + gx;
            float y6[6];
#pragma unroll
            for (int o = 0; o < 6; ++o) y6[o] = sHead[192 + o];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 h = reinterpret_cast<float4*>(my)[lane * 8 + (c ^ (lane & 7))];
#pragma unroll
              for (int o = 0; o < 6; ++o) {
                const float4 w4 = reinterpret_cast<const float4*>(sHead + o * 32)[c];
                y6[o] = fmaf(w4.x, h.x, fmaf(w4.y, h.y, fmaf(w4.z, h.z, fmaf(w4.w, h.w, y6[o]))));
              }
            }
            const float* rgb = a.blend + p * a.blend_stride;
#pragma unroll
            for (int c = 0; c < 3; ++c) a.image[3 * p + c] = fmaf(1.f + y6[c], __ldg(rgb + c), y6[3 + c]);
          }
        }
      }
    }
  }
  if (!ok && a.err) *a.err = 1;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem_base), "r"(2 * kCTmemCols) : "memory");
}

// x0 = (feature, ray direction, embedding, 0 ...): one thread per (pixel, 16-byte unit)
__global__ void __launch_bounds__(256) k_decoder_input(int H, int W, int d_f, float fx, float fy, float cx, float cy,
                                                        const float* __restrict__ blend, int blend_stride,
                                                        const float* __restrict__ emb, float* __restrict__ x0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t P = (int64_t)H * W;
  if (i >= P * 8) return;
  const int64_t p = i >> 3;
  const int c = (int)(i & 7);
  const int v = (int)(p / W), u = (int)(p - (int64_t)v * W);
  // scene.hpp:119-122 (only the units that hold a direction channel pay for it)
  float da = 0.f, db = 0.f, inv = 0.f;
  if (4 * c + 3 >= d_f && 4 * c < d_f + 3) {
    da = (float(u) + 0.5f - cx) / fx; db = (float(v) + 0.5f - cy) / fy;
    inv = 1.f / sqrtf(da * da + db * db + 1.f);
  }
  float out[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = 4 * c + j;
    float val = 0.f;
    if (k < d_f) val = __ldg(blend + p * blend_stride + 3 + k);
    else if (k == d_f) val = da * inv;
    else if (k == d_f + 1) val = db * inv;
    else if (k == d_f + 2) val = inv;
    else if (k < d_f + 11) val = __ldg(emb + (k - d_f - 3));
    out[j] = val;
  }
  reinterpret_cast<float4*>(x0)[i] = make_float4(out[0], out[1], out[2], out[3]);
}

int conv_grid(int H, int W) {
  const int sms = device_sm_count();
  const int tiles = ((W + kCTW - 1) / kCTW) * ((H + kCTR - 1) / kCTR);
  return tiles < sms ? tiles : sms;
}

template <bool kHead> void launch_conv(const ConvArgs& a, cudaStream_t st) {
  static DeviceOnce once;
  once.run([] { cudaFuncSetAttribute(k_conv3x3_tc<kHead>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmemBytes); });
  k_conv3x3_tc<kHead><<<conv_grid(a.H + 2 * a.ext, a.W + 2 * a.ext), kWsThreads, kWsSmemBytes, st>>>(a);
}


// precise mode: three passes (hi hi, lo hi, hi lo), accumulated in fp32 through the residual input. The head variant
// runs its first two passes as plain convolutions into h2 and applies the head in the third.
template <bool kHead> void launch_conv_p(const ConvArgs& a, int precise, cudaStream_t st) {
  if (!precise) { launch_conv<kHead>(a, st); return; }
  float* acc = kHead ? a.h2 : a.y;
  ConvArgs p = a;
  p.y = acc; p.xpart = 0; p.wpart = 0; p.no_bias = 0;
  launch_conv<false>(p, st);
  p.res = acc; p.no_bias = 1; p.xpart = 1; p.wpart = 0;
  launch_conv<false>(p, st);
  p.xpart = 0; p.wpart = 1;
  if (kHead) {
    ConvArgs q = a;
    q.res = acc; q.no_bias = 1; q.xpart = 0; q.wpart = 1;
    launch_conv<true>(q, st);
  } else {
    launch_conv<false>(p, st);
  }
}

// ================================================ backward ====================================================
// weight gradient of one convolution on the tensor cores:
//   g_w[co][ky][kx][ci] = sum_p g_y[p][co] * xr[reflect(p + (ky-1, kx-1))][ci],  xr = relu_in ? relu(x) : x.
// The reduction runs over pixels, so pixels are the K dimension: both operands are transposed while they are staged
// (channel rows, 4 consecutive pixels per 16-byte unit — K-major again; the MN-major operand forms returned zeros for
// tf32 on this part, measured with either swizzle mode). One tile = 64 pixels of two image rows y0, y0+1:
//   A [(h, ci) 128 rows][q 72]   = halo row h = 0..3 (image row y0-1+h), halo pixel q (x0-1+q)
//   B_r,kx [co 32][q 72]         = g_y[row y0+r][pixel q - kx][co]   — per output row three shifted copies (filter column)
//   D_r,kx[(h, ci)][co] += A . B_r,kx^T   — 9 instructions of 128 x 32 x 8 each; halo row h is tap ky = h - r of row r,
//                                            so three of the four 32-row groups of every D are weight gradients
// The six D stay in tensor memory across all the tiles of the persistent CTA (6 x 32 columns) and are added to global
// memory once, at the end (g_w[ky] = D_0[h = ky] + D_1[h = ky + 1]).
constexpr int kWT = 64;                              // tile width (pixels)
constexpr int kWQC = (kWT + 2 + 7) / 8 * 2;          // 18 K chunks of 4 pixels (72 halo pixels, the last 6 zero)
constexpr int kWXChunk = 128 * 4 + 4;                // floats per K chunk of A (+16 B: conflict-free transposed stores)
constexpr int kWGChunk = 64 * 4 + 4;                 // floats per K chunk of B (64 rows: output row r, channel co)
constexpr int kWXFloats = kWQC * kWXChunk;           // 37,152 B
constexpr int kWGFloats = kWQC * kWGChunk;           // 18,720 B per shifted copy (both output rows)
constexpr int kWSmemBytes = (kWXFloats + 3 * kWGFloats) * 4 + 8 * 32 * 4 + 64;   // 94 KB: two CTAs per SM
constexpr int kWTmemCols = 256;                      // 6 x 32 used

struct WgradArgs {
  const float* x;      // H x W x 32, input of the convolution
  const float* gy;     // H x W x 32, gradient of its output
  float* gw;           // 9216 + 32, accumulated (+=)
  int H, W, relu_in;
  int* err;
  int xpart, gpart;    // tf32 parts staged (precise mode: three passes, see tf32_part)
  int no_bias;         // passes 2 and 3: the bias gradient went in with pass 1
};

__global__ void __launch_bounds__(kCThreads, 2) k_conv3x3_wgrad_tc(WgradArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sX = reinterpret_cast<float*>(smem_raw);
  float* sG = sX + kWXFloats;
  float* sRed = sG + 3 * kWGFloats;                            // [8 warps][32]
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sRed + 256);
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles_x = (a.W + kWT - 1) / kWT;
  const int n_tiles = tiles_x * ((a.H + 1) / 2);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(sTmem)), "r"(kWTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(sBar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = tid; i < kWXFloats + 3 * kWGFloats; i += kCThreads) sX[i] = 0.f;   // pads
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *sTmem;
  const uint32_t x_addr = smem_u32(sX), g_addr = smem_u32(sG), bar_addr = smem_u32(sBar);
  uint32_t phase = 0, accumulate = 0;
  float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);   // bias gradient of channel unit 2 (warp & 3) + (tid & 1)
  bool ok = true;

  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int ty = tile / tiles_x;
    const int y0 = 2 * ty, x0 = (tile - ty * tiles_x) * kWT;
    // halo rows y0-1 .. y0+2, pixels x0-1 .. x0+64, transposed: float (q / 4, h * 32 + ci, q % 4). A warp covers
    // 2 channel units x 16 pixels: 32-byte sectors from global memory, 32 distinct banks per transposed store.
    {
      constexpr int kItems = 4 * 5 * 128;   // rows x (5 x 16 pixels, 66 used) x (16 px x 8 units): 10 per thread
      float4 v[10];
#pragma unroll
      for (int u = 0; u < 10; ++u) {
        const int i = tid + u * kCThreads;
        const int c = ((i >> 5) & 3) * 2 + (i & 1), blk = i >> 7;
        const int row = blk / 5, q = (blk - row * 5) * 16 + ((i >> 1) & 15);
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < kItems && q < kWT + 2) {
          const int gy = reflect_clamped(y0 - 1 + row, a.H), gx = reflect_clamped(x0 - 1 + q, a.W);
          v[u] = __ldg(reinterpret_cast<const float4*>(a.x + ((int64_t)gy * a.W + gx) * 32) + c);
        }
      }
#pragma unroll
      for (int u = 0; u < 10; ++u) {
        const int i = tid + u * kCThreads;
        const int c = ((i >> 5) & 3) * 2 + (i & 1), blk = i >> 7;
        const int row = blk / 5, q = (blk - row * 5) * 16 + ((i >> 1) & 15);
        if (i < kItems && q < kWT + 2) {
          float4 t = v[u];
          if (a.relu_in) { t.x = fmaxf(t.x, 0.f); t.y = fmaxf(t.y, 0.f); t.z = fmaxf(t.z, 0.f); t.w = fmaxf(t.w, 0.f); }
          float* dst = sX + (q >> 2) * kWXChunk + (row * 32 + 4 * c) * 4 + (q & 3);
          dst[0] = tf32_part(t.x, a.xpart); dst[4] = tf32_part(t.y, a.xpart); dst[8] = tf32_part(t.z, a.xpart); dst[12] = tf32_part(t.w, a.xpart);
        }
      }
    }
    {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = tid + u * kCThreads;
        const int c = ((i >> 5) & 3) * 2 + (i & 1), px = ((i >> 7) & 3) * 16 + ((i >> 1) & 15), r = i >> 9;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (x0 + px < a.W && y0 + r < a.H) v[u] = __ldg(reinterpret_cast<const float4*>(a.gy + ((int64_t)(y0 + r) * a.W + x0 + px) * 32) + c);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = tid + u * kCThreads;
        const int c = ((i >> 5) & 3) * 2 + (i & 1), px = ((i >> 7) & 3) * 16 + ((i >> 1) & 15), r = i >> 9;
        float4 t = v[u];
        if (!a.no_bias) { bsum.x += t.x; bsum.y += t.y; bsum.z += t.z; bsum.w += t.w; }
        t.x = tf32_part(t.x, a.gpart); t.y = tf32_part(t.y, a.gpart); t.z = tf32_part(t.z, a.gpart); t.w = tf32_part(t.w, a.gpart);
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const int q = px + kx;
          float* dst = sG + kx * kWGFloats + (q >> 2) * kWGChunk + (r * 32 + 4 * c) * 4 + (q & 3);
          dst[0] = t.x; dst[4] = t.y; dst[8] = t.z; dst[12] = t.w;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
      for (int ks = 0; ks < kWQC / 2; ++ks) {
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {   // one N = 64 instruction per filter column: both output rows' dL/dy stacked
          const uint32_t aa = x_addr + (uint32_t)(2 * ks * kWXChunk * 4);
          const uint32_t bb = g_addr + (uint32_t)(kx * kWGFloats * 4) + (uint32_t)(2 * ks * kWGChunk * 4);
          constexpr uint32_t idesc64 = (kIdesc & ~(0x3Fu << 17)) | ((64u >> 3) << 17);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
              :: "r"(tmem_base + (uint32_t)(kx * 64)), "l"(smem_desc(aa, kWXChunk * 4u, 128u)), "l"(smem_desc(bb, kWGChunk * 4u, 128u)),
                 "r"(idesc64), "r"(accumulate | (uint32_t)ks) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(bar_addr) : "memory");
    }
    accumulate = 1;
    {
      uint32_t done = 0;
      for (int tries = 0; tries < kCTries && !done; ++tries)   // try_wait suspends the warp: no issue slots burnt
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done) : "r"(bar_addr), "r"(phase) : "memory");
      if (!__syncthreads_and((int)done)) {
        if (tid == 0 && a.err) *a.err = 1;
        ok = false;
        break;
      }
      phase ^= 1u;
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // ---- weights: warp h (0..3) holds halo row h (lanes = ci); 6 x 32 columns = (r, kx, co); tap ky = h - r ----
  if (ok && accumulate && warp < 4) {
#pragma unroll 1
    for (int rk = 0; rk < 6; ++rk) {
      float acc[32];
      const int kx = rk >> 1, r = rk & 1, ky = warp - r;   // columns: (kx, r, co)
      tmem_load32(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(rk * 32), acc);
      if (ky >= 0 && ky < 3) {
#pragma unroll
        for (int co = 0; co < 32; ++co) atomicAdd(a.gw + ((co * 3 + ky) * 3 + kx) * 32 + lane, acc[co]);
      }
    }
  }
  // ---- bias: sum the per-thread partials of each channel unit (lanes of equal parity, then warps w and w + 4) ----
  {
    float4 t = bsum;
#pragma unroll
    for (int m = 2; m < 32; m <<= 1) {
      t.x += __shfl_xor_sync(0xffffffffu, t.x, m); t.y += __shfl_xor_sync(0xffffffffu, t.y, m);
      t.z += __shfl_xor_sync(0xffffffffu, t.z, m); t.w += __shfl_xor_sync(0xffffffffu, t.w, m);
    }
    if (lane < 2) reinterpret_cast<float4*>(sRed)[warp * 2 + lane] = t;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (ok && tid < 32) {
    const int c = tid >> 2;   // channel unit: warps (c >> 1) and (c >> 1) + 4, lane c & 1
    const float t = sRed[(((c >> 1) * 2 + (c & 1)) << 2) + (tid & 3)] + sRed[((((c >> 1) + 4) * 2 + (c & 1)) << 2) + (tid & 3)];
    atomicAdd(a.gw + 9216 + tid, t);
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem_base), "r"(kWTmemCols) : "memory");
}

// weights of the input-gradient convolution: Wt[ci][ky][kx][co] = W[co][2-ky][2-kx][ci], zero bias
__global__ void k_dec_transpose_w(const float* __restrict__ w, float* __restrict__ wt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 9216) {
    const int co = i & 31, t = (i >> 5) % 9, ci = i / 288;
    wt[i] = w[(co * 9 + (8 - t)) * 32 + ci];
  } else if (i < 9248) {
    wt[i] = 0.f;
  }
}

// Folds the extended-domain result of the zero-padded transposed convolution back onto the image (the adjoint of
// reflect padding: what landed on row -1 belongs to row 1, on row H to row H-2, same for columns; both when H == 3).
__device__ __forceinline__ float4 fold_sum(const float* __restrict__ gext, int H, int W, int y, int x, int c) {
  const int We = W + 2;
  constexpr int kNone = -9;
  const int yc[3] = {y, y == 1 ? -1 : kNone, y == H - 2 ? H : kNone};
  const int xc[3] = {x, x == 1 ? -1 : kNone, x == W - 2 ? W : kNone};
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (yc[a] == kNone) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (xc[b] == kNone) continue;
      const float4 t = __ldg(reinterpret_cast<const float4*>(gext + ((int64_t)(yc[a] + 1) * We + (xc[b] + 1)) * 32) + c);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
  }
  return s;
}

// g_x = mask(x) . fold(gext) + add. One thread per (pixel, 16-byte unit).
__global__ void __launch_bounds__(256) k_dec_fold(int H, int W, const float* __restrict__ gext, const float* __restrict__ x_mask,
                                                   const float* __restrict__ add, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)H * W * 8) return;
  const int64_t p = i >> 3;
  const int c = (int)(i & 7);
  const int y = (int)(p / W), x = (int)(p - (int64_t)y * W);
  float4 s = fold_sum(gext, H, W, y, x, c);
  if (x_mask) {
    const float4 m = __ldg(reinterpret_cast<const float4*>(x_mask + p * 32) + c);
    if (!(m.x > 0.f)) s.x = 0.f;
    if (!(m.y > 0.f)) s.y = 0.f;
    if (!(m.z > 0.f)) s.z = 0.f;
    if (!(m.w > 0.f)) s.w = 0.f;
  }
  if (add) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(add + p * 32) + c);
    s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
  }
  reinterpret_cast<float4*>(out)[i] = s;
}

// The stem's fold, fused with the gradient of the decoder input: feature slots are added to the blend gradient, the
// embedding slots are summed over all pixels (registers over the grid-stride loop -> warp -> block -> one atomic).
__global__ void __launch_bounds__(256) k_dec_fold_input(int H, int W, int d_f, const float* __restrict__ gext,
                                                         float* __restrict__ g_blend, int blend_stride, float* __restrict__ g_emb) {
  __shared__ float sEmb[8];
  if (threadIdx.x < 8) sEmb[threadIdx.x] = 0.f;
  __syncthreads();
  const int c = threadIdx.x & 7;
  const int64_t n = (int64_t)H * W * 8;
  float e[4] = {0.f, 0.f, 0.f, 0.f};   // channels 4c .. 4c+3 of this thread's unit
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i >> 3;
    const int y = (int)(p / W), x = (int)(p - (int64_t)y * W);
    const float4 s = fold_sum(gext, H, W, y, x, c);
    const float v[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 4 * c + j;
      if (k < d_f) g_blend[p * blend_stride + 3 + k] += v[j];
      e[j] += v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float t = e[j];
    t += __shfl_xor_sync(0xffffffffu, t, 8);
    t += __shfl_xor_sync(0xffffffffu, t, 16);
    const int k = 4 * c + j - d_f - 3;   // embedding slot
    if ((threadIdx.x & 31) < 8 && k >= 0 && k < 8) atomicAdd(&sEmb[k], t);
  }
  __syncthreads();
  if (threadIdx.x < 8) atomicAdd(g_emb + threadIdx.x, sEmb[threadIdx.x]);
}

// head backward, 8 threads per pixel (thread = one 16-byte channel unit): from dL/dimage, dL/drgb (added to the blend
// gradient), dL/dh2, and the head's parameter gradients (kept in registers over the grid-stride loop, then reduced)
__global__ void __launch_bounds__(256) k_dec_head_bwd(int64_t P, const float* __restrict__ h2, const float* __restrict__ head,
                                                       const float* __restrict__ blend, int blend_stride,
                                                       const float* __restrict__ g_image, float* __restrict__ g_blend,
                                                       float* __restrict__ g_h2, float* __restrict__ g_head) {
  __shared__ float sAcc[198];
  for (int i = threadIdx.x; i < 198; i += blockDim.x) sAcc[i] = 0.f;
  __syncthreads();
  const int c = threadIdx.x & 7;
  float wh[6][4], bh[3], wacc[6][4], bacc[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    bacc[q] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) { wh[q][j] = __ldg(head + q * 32 + 4 * c + j); wacc[q][j] = 0.f; }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) bh[q] = __ldg(head + 192 + q);
  const int64_t n_groups = (P + 31) / 32;
  for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const int64_t p = grp * 32 + (threadIdx.x >> 3);
    const bool live = p < P;
    float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) h = __ldg(reinterpret_cast<const float4*>(h2 + p * 32) + c);
    float gy[6];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float y = wh[q][0] * h.x + wh[q][1] * h.y + wh[q][2] * h.z + wh[q][3] * h.w;
      y += __shfl_xor_sync(0xffffffffu, y, 1);
      y += __shfl_xor_sync(0xffffffffu, y, 2);
      y += __shfl_xor_sync(0xffffffffu, y, 4);
      y += bh[q];
      const float g = live ? __ldg(g_image + 3 * p + q) : 0.f;
      if (live && c == q) g_blend[p * blend_stride + q] += g * (1.f + y);
      gy[q] = live ? g * __ldg(blend + p * blend_stride + q) : 0.f;
      gy[3 + q] = g;
    }
    if (live) {
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < 6; ++q) t = fmaf(gy[q], wh[q][j], t);
        o[j] = t;
      }
      reinterpret_cast<float4*>(g_h2 + p * 32)[c] = make_float4(o[0], o[1], o[2], o[3]);
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      wacc[q][0] = fmaf(gy[q], h.x, wacc[q][0]); wacc[q][1] = fmaf(gy[q], h.y, wacc[q][1]);
      wacc[q][2] = fmaf(gy[q], h.z, wacc[q][2]); wacc[q][3] = fmaf(gy[q], h.w, wacc[q][3]);
      bacc[q] += gy[q];
    }
  }
  // lanes of equal channel unit (xor 8, 16), then the block, then one atomic per parameter and CTA
#pragma unroll
  for (int q = 0; q < 6; ++q) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float t = wacc[q][j];
      t += __shfl_xor_sync(0xffffffffu, t, 8);
      t += __shfl_xor_sync(0xffffffffu, t, 16);
      if ((threadIdx.x & 31) < 8) atomicAdd(&sAcc[q * 32 + 4 * c + j], t);
    }
    float t = bacc[q];
    t += __shfl_xor_sync(0xffffffffu, t, 8);
    t += __shfl_xor_sync(0xffffffffu, t, 16);
    if ((threadIdx.x & 31) == 0) atomicAdd(&sAcc[192 + q], t);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 198; i += blockDim.x) atomicAdd(g_head + i, sAcc[i]);
}

int sm_count() { return device_sm_count(); }

void launch_wgrad(const float* x, const float* gy, float* gw, int H, int W, int relu_in, int* err, cudaStream_t st, int precise) {
  static DeviceOnce once;
  once.run([] { cudaFuncSetAttribute(k_conv3x3_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmemBytes); });
  const int tiles = ((W + kWT - 1) / kWT) * ((H + 1) / 2);
  const int grid = tiles < 2 * sm_count() ? tiles : 2 * sm_count();
  WgradArgs a{x, gy, gw, H, W, relu_in, err, 0, 0, 0};
  k_conv3x3_wgrad_tc<<<grid, kCThreads, kWSmemBytes, st>>>(a);
  if (precise) {  // + lo(x) hi(g) + hi(x) lo(g), accumulated by the kernel's own +=
    a.no_bias = 1; a.xpart = 1; a.gpart = 0;
    k_conv3x3_wgrad_tc<<<grid, kCThreads, kWSmemBytes, st>>>(a);
    a.xpart = 0; a.gpart = 1;
    k_conv3x3_wgrad_tc<<<grid, kCThreads, kWSmemBytes, st>>>(a);
  }
}

// g_x = mask(x) . fold(convT(g_y)) + add: transposed weights -> tensor-core convolution on the grown domain -> fold
void launch_dgrad_conv(const float* gy, const float* w, float* wt, float* gext, int H, int W, int* err, cudaStream_t st, int precise) {
  k_dec_transpose_w<<<(9248 + 255) / 256, 256, 0, st>>>(w, wt);
  ConvArgs a{};
  a.x = gy; a.w = wt; a.y = gext; a.H = H; a.W = W; a.ext = 1; a.err = err;
  launch_conv_p<false>(a, precise, st);
}

void launch_dgrad(const float* gy, const float* w, float* wt, float* gext, const float* x_mask, const float* add, float* gx,
                  int H, int W, int* err, cudaStream_t st, int precise) {
  launch_dgrad_conv(gy, w, wt, gext, H, W, err, st, precise);
  const int64_t units = (int64_t)H * W * 8;
  k_dec_fold<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(H, W, gext, x_mask, add, gx);
}

}  // namespace

int conv_decoder_params() { return 5 * 9248 + 198; }

void launch_conv3x3(const float* x, int H, int W, const float* w, int relu_in, const float* res, float* y, int* err,
                    cudaStream_t st, int precise) {
  if (H <= 0 || W <= 0) return;
  ConvArgs a{};
  a.x = x; a.w = w; a.res = res; a.y = y; a.H = H; a.W = W; a.relu_in = relu_in; a.err = err;
  launch_conv_p<false>(a, precise, st);
}

void launch_conv3x3_backward(const float* x, int H, int W, const float* w, int relu_in, const float* gy, float* wt, float* gext,
                             float* gx, float* gw, int* err, cudaStream_t st, int precise) {
  if (H <= 0 || W <= 0) return;
  launch_wgrad(x, gy, gw, H, W, relu_in, err, st, precise);
  launch_dgrad(gy, w, wt, gext, relu_in ? x : nullptr, nullptr, gx, H, W, err, st, precise);
}

int launch_conv_decoder(const float* params, const float* emb, int H, int W, int d_f, float fx, float fy, float cx, float cy,
                        const float* blend, int blend_stride, float* const act[6], float* image, int* err, cudaStream_t st,
                        int precise) {
  if (H <= 0 || W <= 0) return 0;
  const int64_t units = (int64_t)H * W * 8;
  float *x0 = act[0], *h0 = act[1], *t1 = act[2], *h1 = act[3], *t2 = act[4], *h2 = act[5];
  k_decoder_input<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(H, W, d_f, fx, fy, cx, cy, blend, blend_stride, emb, x0);
  ConvArgs a{};
  a.H = H; a.W = W; a.err = err;
  a.x = x0; a.w = params; a.res = nullptr; a.y = h0; a.relu_in = 0;
  launch_conv_p<false>(a, precise, st);
  a.x = h0; a.w = params + 9248; a.y = t1; a.relu_in = 1;
  launch_conv_p<false>(a, precise, st);
  a.x = t1; a.w = params + 2 * 9248; a.res = h0; a.y = h1;                            // h1 = h0 + conv2(relu(t1))
  launch_conv_p<false>(a, precise, st);
  a.x = h1; a.w = params + 3 * 9248; a.res = nullptr; a.y = t2;
  launch_conv_p<false>(a, precise, st);
  a.x = t2; a.w = params + 4 * 9248; a.res = h1; a.y = nullptr;                       // h2 = h1 + conv4(relu(t2)) -> head
  a.head = params + 5 * 9248; a.blend = blend; a.blend_stride = blend_stride; a.image = image; a.h2 = h2;
  launch_conv_p<true>(a, precise, st);
  return precise ? 16 : 6;
}

int launch_conv_decoder_backward(const float* params, int H, int W, int d_f, const float* blend, int blend_stride,
                                 float* const act[6], const float* g_image, float* const g[3], float* gext, float* wt,
                                 float* g_params, float* g_emb, float* g_blend, int* err, cudaStream_t st, int precise) {
  if (H <= 0 || W <= 0) return 0;
  const int64_t P = (int64_t)H * W;
  const float *x0 = act[0], *h0 = act[1], *t1 = act[2], *h1 = act[3], *t2 = act[4], *h2 = act[5];
  float *g0 = g[0], *g1 = g[1], *g2 = g[2];
  const int grid = 4 * sm_count();
  k_dec_head_bwd<<<grid, 256, 0, st>>>(P, h2, params + 5 * 9248, blend, blend_stride, g_image, g_blend, g0, g_params + 5 * 9248);
  // block 2: h2 = h1 + conv4(relu(t2)), t2 = conv3(relu(h1));  g0 = dL/dh2
  launch_wgrad(t2, g0, g_params + 4 * 9248, H, W, 1, err, st, precise);
  launch_dgrad(g0, params + 4 * 9248, wt, gext, t2, nullptr, g1, H, W, err, st, precise);      // g1 = dL/dt2
  launch_wgrad(h1, g1, g_params + 3 * 9248, H, W, 1, err, st, precise);
  launch_dgrad(g1, params + 3 * 9248, wt, gext, h1, g0, g2, H, W, err, st, precise);           // g2 = dL/dh1
  // block 1: h1 = h0 + conv2(relu(t1)), t1 = conv1(relu(h0))
  launch_wgrad(t1, g2, g_params + 2 * 9248, H, W, 1, err, st, precise);
  launch_dgrad(g2, params + 2 * 9248, wt, gext, t1, nullptr, g1, H, W, err, st, precise);      // g1 = dL/dt1
  launch_wgrad(h0, g1, g_params + 9248, H, W, 1, err, st, precise);
  launch_dgrad(g1, params + 9248, wt, gext, h0, g2, g0, H, W, err, st, precise);               // g0 = dL/dh0
  // stem: h0 = conv0(x0)
  launch_wgrad(x0, g0, g_params, H, W, 0, err, st, precise);
  launch_dgrad_conv(g0, params, wt, gext, H, W, err, st, precise);                             // dL/dx0 on the grown domain
  k_dec_fold_input<<<grid, 256, 0, st>>>(H, W, d_f, gext, g_blend, blend_stride, g_emb);
  return precise ? 1 + 5 * 8 : 1 + 5 * 4;
}

}  // namespace sb
