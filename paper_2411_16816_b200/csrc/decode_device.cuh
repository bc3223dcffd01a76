// decode_device.cuh — device functions of the lidar head, shared by decode.cu and the fused epilogue
// of the lidar compositing kernel (forward.cu).
#pragma once

#include <cuda_runtime.h>

namespace sb {
namespace headdev {
constexpr int kHid = 32;
constexpr int kInMax = 16;  // d_f + 3 <= 16

__device__ __forceinline__ float sigmoidf_(float a) {
  if (a >= 0.0f) return 1.0f / (1.0f + __expf(-a));
  const float e = __expf(a);
  return e / (1.0f + e);
}
__device__ __forceinline__ void ray_dir(float phi, float omega, float d[3]) {
  float so, co, sp, cp;
  sincosf(omega, &so, &co);
  sincosf(phi, &sp, &cp);
  d[0] = co * cp; d[1] = co * sp; d[2] = so;
}
__device__ __forceinline__ void head_forward(const float* __restrict__ sw, int in, const float x[kInMax], float y[2], float h[kHid]) {
  const float* W1 = sw; const float* b1 = W1 + kHid * in; const float* W2 = b1 + kHid; const float* b2 = W2 + 2 * kHid;
#pragma unroll 4
  for (int j = 0; j < kHid; ++j) {
    float a = b1[j];
    for (int k = 0; k < in; ++k) a = fmaf(W1[j * in + k], x[k], a);
    h[j] = fmaxf(a, 0.0f);
  }
  float a0 = b2[0], a1 = b2[1];
#pragma unroll
  for (int j = 0; j < kHid; ++j) { a0 = fmaf(W2[j], h[j], a0); a1 = fmaf(W2[kHid + j], h[j], a1); }
  y[0] = sigmoidf_(a0); y[1] = sigmoidf_(a1);
}
}  // namespace headdev
}  // namespace sb
