// decode_image — the camera ConvDecoder (Eq. 7-8).
//
// The only dense contraction of the system, so the only kernel here that runs on the tensor cores: every 3x3, 32 -> 32
// convolution is an implicit GEMM issued as tcgen05.mma (kind::tf32, M = 128 pixels, N = 32 output channels, K = 8
// input channels per instruction) with the accumulator in tensor memory.
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
// in the same layout; CTAs are persistent (two per SM, so one stages while the other's MMAs and epilogue run).
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
constexpr int kCSmemBytes = (kCXUnits + kCWUnits) * 16 + 32 * 4 + 256 * 4 + 64;
constexpr int kCSpin = 1 << 22;

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
  // head variant: h2 = res + conv -> y6 = Wh h2 + bh -> image = (1 + y[0:3]) * rgb + y[3:6]
  const float* head;     // 192 + 6
  const float* blend;    // P x blend_stride, rgb first
  int blend_stride;
  float* image;          // P x 3
  int* err;              // set to 1 if the MMA completion barrier timed out
};

template <bool kHead>
__global__ void __launch_bounds__(kCThreads, 2) k_conv3x3_tc(ConvArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* sX = reinterpret_cast<float4*>(smem_raw);
  float4* sW = sX + kCXUnits;
  float* sBias = reinterpret_cast<float*>(sW + kCWUnits);
  float* sHead = sBias + 32;                                    // 198 used
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sHead + 256);
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles_x = (a.W + kCTW - 1) / kCTW, tiles_y = (a.H + kCTR - 1) / kCTR;
  const int n_tiles = tiles_x * tiles_y;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(sTmem)), "r"(kCTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(sBar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the layer's weights, once per CTA: unit ((tap * 8 + c) * 32 + co) = W[co][tap][4c .. 4c+3]
  {
    const float4* gw = reinterpret_cast<const float4*>(a.w);
    for (int i = tid; i < kCWUnits; i += kCThreads) {
      const int co = i / 72, rem = i - co * 72, tap = rem >> 3, c = rem & 7;
      float4 v = __ldg(gw + i);
      v.x = to_tf32(v.x); v.y = to_tf32(v.y); v.z = to_tf32(v.z); v.w = to_tf32(v.w);
      sW[(tap * 8 + c) * 32 + co] = v;
    }
    if (tid < 32) sBias[tid] = __ldg(a.w + 9216 + tid);
    if (kHead)
      for (int i = tid; i < 198; i += kCThreads) sHead[i] = __ldg(a.head + i);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *sTmem;
  const uint32_t x_addr = smem_u32(sX), w_addr = smem_u32(sW), bar_addr = smem_u32(sBar);
  // K-major, no swizzle: leading offset = distance between the two 16-byte K chunks, stride offset = 8-row groups
  constexpr uint32_t a_lbo = (uint32_t)kCPlane * 16u, a_sbo = 128u;
  constexpr uint32_t b_lbo = 512u, b_sbo = 128u;
  uint32_t phase = 0;

  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int x0 = tx * kCTW, y0 = ty * kCTR;
    // ---- stage the halo: 4 rows x 130 pixels x 8 units, reflect padding, optional ReLU, tf32 rounding ----
    for (int i = tid; i < kCHR * kCHW * 8; i += kCThreads) {
      const int c = i & 7, hp = i >> 3;
      const int row = hp / kCHW, px = hp - row * kCHW;
      const int gy = reflect_clamped(y0 - 1 + row, a.H), gx = reflect_clamped(x0 - 1 + px, a.W);
      float4 v = __ldg(reinterpret_cast<const float4*>(a.x + ((int64_t)gy * a.W + gx) * 32) + c);
      if (a.relu_in) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
      v.x = to_tf32(v.x); v.y = to_tf32(v.y); v.z = to_tf32(v.z); v.w = to_tf32(v.w);
      sX[c * kCPlane + hp] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy stores -> tensor-core reads
    __syncthreads();
    // ---- one thread issues the tile's 2 x 9 x 4 MMAs (128 x 32 x 8 each) and commits them to the barrier ----
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int r = 0; r < kCTR; ++r) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int ky = tap / 3, kx = tap - 3 * ky;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t aa = x_addr + (uint32_t)((2 * ks) * kCPlane + (r + ky) * kCHW + kx) * 16u;
            const uint32_t bb = w_addr + (uint32_t)((tap * 8 + 2 * ks) * 32) * 16u;
            mma_tf32(tmem_base + (uint32_t)(r * 32), smem_desc(aa, a_lbo, a_sbo), smem_desc(bb, b_lbo, b_sbo),
                     (tap | ks) != 0);
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(bar_addr) : "memory");
    }
    // ---- wait for the MMAs (bounded: a descriptor mistake must not hang the device) ----
    {
      uint32_t done = 0;
      for (int spin = 0; spin < kCSpin && !done; ++spin)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done) : "r"(bar_addr), "r"(phase) : "memory");
      if (!__syncthreads_and((int)done)) {
        if (tid == 0 && a.err) *a.err = 1;
        break;
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // ---- epilogue: warp w reads row w / 4, pixels 32 (w % 4) + lane; one pixel's 32 channels per thread ----
    {
      const int r = warp >> 2, q = warp & 3;
      float acc[32];
      tmem_load32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(r * 32), acc);
      const int gx = x0 + q * 32 + lane, gy = y0 + r;
      if (gx < a.W && gy < a.H) {
        const int64_t p = (int64_t)gy * a.W + gx;
#pragma unroll
        for (int k = 0; k < 32; ++k) acc[k] += sBias[k];
        if (a.res) {
          const float4* rp = reinterpret_cast<const float4*>(a.res + p * 32);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 t = __ldg(rp + c);
            acc[4 * c] += t.x; acc[4 * c + 1] += t.y; acc[4 * c + 2] += t.z; acc[4 * c + 3] += t.w;
          }
        }
        if (kHead) {
          float y6[6];
#pragma unroll
          for (int o = 0; o < 6; ++o) {
            float s = sHead[192 + o];
#pragma unroll
            for (int k = 0; k < 32; ++k) s = fmaf(sHead[o * 32 + k], acc[k], s);
            y6[o] = s;
          }
          const float* rgb = a.blend + p * a.blend_stride;
#pragma unroll
          for (int c = 0; c < 3; ++c) a.image[3 * p + c] = fmaf(1.f + y6[c], __ldg(rgb + c), y6[3 + c]);
        } else {
          float4* yp = reinterpret_cast<float4*>(a.y + p * 32);
#pragma unroll
          for (int c = 0; c < 8; ++c) yp[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // accumulators read and halo consumed: both free for the next tile
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem_base), "r"(kCTmemCols) : "memory");
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
  // scene.hpp:119-122
  const float da = (float(u) + 0.5f - cx) / fx, db = (float(v) + 0.5f - cy) / fy;
  const float inv = 1.f / sqrtf(da * da + db * db + 1.f);
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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = ((W + kCTW - 1) / kCTW) * ((H + kCTR - 1) / kCTR);
  return tiles < 2 * sms ? tiles : 2 * sms;
}

template <bool kHead> void launch_conv(const ConvArgs& a, cudaStream_t st) {
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(k_conv3x3_tc<kHead>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmemBytes);
    once = true;
  }
  k_conv3x3_tc<kHead><<<conv_grid(a.H, a.W), kCThreads, kCSmemBytes, st>>>(a);
}

}  // namespace

int conv_decoder_params() { return 5 * 9248 + 198; }

void launch_conv3x3(const float* x, int H, int W, const float* w, int relu_in, const float* res, float* y, int* err,
                    cudaStream_t st) {
  if (H <= 0 || W <= 0) return;
  ConvArgs a{};
  a.x = x; a.w = w; a.res = res; a.y = y; a.H = H; a.W = W; a.relu_in = relu_in; a.err = err;
  launch_conv<false>(a, st);
}

int launch_conv_decoder(const float* params, const float* emb, int H, int W, int d_f, float fx, float fy, float cx, float cy,
                        const float* blend, int blend_stride, float* buf_a, float* buf_b, float* buf_c, float* image,
                        int* err, cudaStream_t st) {
  if (H <= 0 || W <= 0) return 0;
  const int64_t units = (int64_t)H * W * 8;
  k_decoder_input<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(H, W, d_f, fx, fy, cx, cy, blend, blend_stride, emb, buf_a);
  ConvArgs a{};
  a.H = H; a.W = W; a.err = err;
  a.x = buf_a; a.w = params; a.res = nullptr; a.y = buf_b; a.relu_in = 0;             // h0 (b)
  launch_conv<false>(a, st);
  a.x = buf_b; a.w = params + 9248; a.y = buf_c; a.relu_in = 1;                       // t1 (c)
  launch_conv<false>(a, st);
  a.x = buf_c; a.w = params + 2 * 9248; a.res = buf_b; a.y = buf_a;                   // h1 = h0 + conv2 (a)
  launch_conv<false>(a, st);
  a.x = buf_a; a.w = params + 3 * 9248; a.res = nullptr; a.y = buf_c;                 // t2 (c)
  launch_conv<false>(a, st);
  a.x = buf_c; a.w = params + 4 * 9248; a.res = buf_a; a.y = nullptr;                 // h2 = h1 + conv4 -> head -> image
  a.head = params + 5 * 9248; a.blend = blend; a.blend_stride = blend_stride; a.image = image;
  launch_conv<true>(a, st);
  return 6;
}

}  // namespace sb
