// decode.cu — decode_lidar (section 3.3, Appendix B): the lidar head, SURVEY 8(f) rank 1.
// A 2-layer perceptron (hidden 32, rectified-linear inside, logistic outputs) maps the D_f blended features of a ray
// plus its direction in the sensor frame to intensity and ray-drop probability. Parameter block (row-major):
// W1 [32 x (d_f + 3)], b1 [32], W2 [2 x 32], b2 [2].
//
//   k_lidar_head_fwd   one thread per ray, parameters in shared memory.
//   k_lidar_head_bwd   persistent CTAs. Each thread back-propagates its ray (hidden layer recomputed), adds dL/dfeature
//                      to the ray's slots of the compositing kernels' upstream buffer (P x 16), and parks its
//                      pre-activation gradients and inputs in a per-warp shared-memory tile; the warp then accumulates
//                      the weight gradients as a 32-ray outer-product sum — every lane owns fixed entries of W1 / W2 /
//                      biases and keeps running sums in registers across the CTA's rays — so the 610 sums leave as
//                      ONE atomic per entry and CTA, not one per ray.
#include "kernels.h"
#include "decode_device.cuh"

namespace sb {

namespace {
using namespace headdev;
}  // namespace

__global__ void __launch_bounds__(256)
k_lidar_head_fwd(const float* __restrict__ w, int n_params, int d_f, int64_t n_rays, const float4* __restrict__ rays,
                 const float* __restrict__ blend16, float* __restrict__ y_out /* P x 2, caller's ray order */) {
  extern __shared__ float sw[];
  for (int i = threadIdx.x; i < n_params; i += 256) sw[i] = w[i];
  __syncthreads();
  const int64_t pos = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (pos >= n_rays) return;
  const float4 r = rays[pos];
  const int64_t q = (int64_t)__float_as_uint(r.w);
  float x[kInMax], y[2], h[kHid];
  for (int k = 0; k < d_f; ++k) x[k] = blend16[16 * q + k];
  ray_dir(r.x, r.y, x + d_f);
  head_forward(sw, d_f + 3, x, y, h);
  y_out[2 * q] = y[0];
  y_out[2 * q + 1] = y[1];
}

__global__ void __launch_bounds__(256)
k_lidar_head_bwd(const float* __restrict__ w, int n_params, int d_f, int64_t n_rays, const float4* __restrict__ rays,
                 const float* __restrict__ blend16, const float* __restrict__ g_y /* P x 2 */,
                 float* __restrict__ g_blend16 /* P x 16, += on slots [0, d_f) */, float* __restrict__ g_w /* n_params, += */) {
  extern __shared__ float smem[];
  float* sw = smem;                                   // n_params (<= 610)
  float* tiles = smem + ((n_params + 3) & ~3);        // per warp: A [32 x 33], X [32 x 17]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* A = tiles + warp * (32 * 33 + 32 * 17);      // pre-activation gradients of layer 1 (then: hidden activations)
  float* X = A + 32 * 33;                             // inputs (then: pre-activation gradients of layer 2)
  for (int i = tid; i < n_params; i += 256) sw[i] = w[i];
  __syncthreads();
  const int in = d_f + 3;
  const float* W1 = sw; const float* W2 = sw + kHid * in + kHid;
  // fixed ownership: lane owns W1 entries lane + 32 m (m < 16; entry e = j * in + k), W2 entries lane and lane + 32,
  // b1[lane], and (lanes 0, 1) b2[lane]
  float aW1[16], aW2[2] = {0.0f, 0.0f}, ab1 = 0.0f, ab2 = 0.0f;
#pragma unroll
  for (int m = 0; m < 16; ++m) aW1[m] = 0.0f;
  const int n_w1 = kHid * in;
  for (int64_t base = (int64_t)blockIdx.x * 256; base < n_rays; base += (int64_t)gridDim.x * 256) {
    const int64_t pos = base + tid;
    const bool live = pos < n_rays;
    float x[kInMax], y[2], h[kHid], gp2[2] = {0.0f, 0.0f};
    for (int k = 0; k < kInMax; ++k) x[k] = 0.0f;
    for (int j = 0; j < kHid; ++j) h[j] = 0.0f;
    int64_t q = 0;
    if (live) {
      const float4 r = rays[pos];
      q = (int64_t)__float_as_uint(r.w);
      for (int k = 0; k < d_f; ++k) x[k] = blend16[16 * q + k];
      ray_dir(r.x, r.y, x + d_f);
      head_forward(sw, in, x, y, h);
      gp2[0] = g_y[2 * q] * y[0] * (1.0f - y[0]);
      gp2[1] = g_y[2 * q + 1] * y[1] * (1.0f - y[1]);
    }
    // layer 1 pre-activation gradients, dL/dfeature
    float gf[kInMax];
    for (int k = 0; k < kInMax; ++k) gf[k] = 0.0f;
#pragma unroll 4
    for (int j = 0; j < kHid; ++j) {
      const float gp1 = h[j] > 0.0f ? fmaf(W2[j], gp2[0], W2[kHid + j] * gp2[1]) : 0.0f;
      A[lane * 33 + j] = gp1;
      for (int k = 0; k < d_f; ++k) gf[k] = fmaf(W1[j * in + k], gp1, gf[k]);
    }
    for (int k = 0; k < in; ++k) X[lane * 17 + k] = x[k];
    if (live)
      for (int k = 0; k < d_f; ++k) g_blend16[16 * q + k] += gf[k];
    __syncwarp();
    // W1 / b1: sums over the warp's 32 rays
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = lane + 32 * m;
      if (e < n_w1) {
        const int j = e / in, k = e - j * in;
        float s = 0.0f;
#pragma unroll 8
        for (int t = 0; t < 32; ++t) s = fmaf(A[t * 33 + j], X[t * 17 + k], s);
        aW1[m] += s;
      }
    }
    {
      float s = 0.0f;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) s += A[t * 33 + lane];
      ab1 += s;
    }
    __syncwarp();
    // W2 / b2: hidden activations and layer-2 pre-activation gradients through the same tiles
#pragma unroll 4
    for (int j = 0; j < kHid; ++j) A[lane * 33 + j] = h[j];
    X[lane * 17] = gp2[0]; X[lane * 17 + 1] = gp2[1];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int e = lane + 32 * m, o = e / kHid, j = e - o * kHid;
      float s = 0.0f;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) s = fmaf(X[t * 17 + o], A[t * 33 + j], s);
      aW2[m] += s;
    }
    if (lane < 2) {
      float s = 0.0f;
      for (int t = 0; t < 32; ++t) s += X[t * 17 + lane];
      ab2 += s;
    }
    __syncwarp();
  }
  // one atomic per entry and warp (8 per CTA; CTAs are persistent: a few hundred per entry in total)
  float* gW1 = g_w; float* gb1 = gW1 + n_w1; float* gW2 = gb1 + kHid; float* gb2 = gW2 + 2 * kHid;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int e = lane + 32 * m;
    if (e < n_w1 && aW1[m] != 0.0f) atomicAdd(&gW1[e], aW1[m]);
  }
  if (ab1 != 0.0f) atomicAdd(&gb1[lane], ab1);
#pragma unroll
  for (int m = 0; m < 2; ++m)
    if (aW2[m] != 0.0f) atomicAdd(&gW2[lane + 32 * m], aW2[m]);
  if (lane < 2 && ab2 != 0.0f) atomicAdd(&gb2[lane], ab2);
}

int lidar_head_params(int d_f) { return kHid * (d_f + 3) + kHid + 2 * kHid + 2; }

void launch_lidar_head_fwd(const float* w, int d_f, int64_t n_rays, const float4* rays, const float* blend16, float* y_out,
                           cudaStream_t st) {
  if (n_rays <= 0) return;
  const int np = lidar_head_params(d_f);
  k_lidar_head_fwd<<<(unsigned)((n_rays + 255) / 256), 256, sizeof(float) * np, st>>>(w, np, d_f, n_rays, rays, blend16, y_out);
}

void launch_lidar_head_bwd(const float* w, int d_f, int64_t n_rays, const float4* rays, const float* blend16, const float* g_y,
                           float* g_blend16, float* g_w, cudaStream_t st) {
  if (n_rays <= 0) return;
  const int np = lidar_head_params(d_f);
  const size_t smem = sizeof(float) * (((np + 3) & ~3) + 8 * (32 * 33 + 32 * 17));
  // opt in once per device to the largest size any d_f needs (kInMax inputs), not to the first call's
  constexpr size_t smem_max = sizeof(float) * (((kHid * kInMax + kHid + 2 * kHid + 2 + 3) & ~3) + 8 * (32 * 33 + 32 * 17));
  static DeviceOnce once;
  once.run([] { cudaFuncSetAttribute(k_lidar_head_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max); });
  const unsigned blocks = (unsigned)std::min<int64_t>(2 * (int64_t)device_sm_count(), (n_rays + 255) / 256);
  k_lidar_head_bwd<<<blocks, 256, smem, st>>>(w, np, d_f, n_rays, rays, blend16, g_y, g_blend16, g_w);
}

}  // namespace sb
