// optim.cu — optimizer_step: Adam with per-group scheduled learning rates over
// the GaussianSet, in place on the device, straight from the contiguous SceneParamGrads buffer the backward pass (and
// the all-reduce) leaves behind. beta = (0.9, 0.999), eps = 1e-15; a group whose gradient holds a
// non-finite value is skipped and reported.
//
//   k_grad_finite   per group: does the gradient slice hold a non-finite value?  (one read of the gradients)
//   k_adam          one thread per 4 elements (128-bit accesses): g, m, v, p in; m, v, p out — 28 B per element, purely
//                   HBM-bound.
#include "kernels.h"

namespace sb {

__global__ void __launch_bounds__(256) k_grad_finite(const float* __restrict__ g, int64_t n_floats, AdamGroups gr,
                                                     int* __restrict__ bad /* 6 */) {
  const int64_t stride = (int64_t)gridDim.x * 256;
  int local = 0;  // bit per group
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n_floats; i += stride) {
    if (!isfinite(g[i])) {
#pragma unroll
      for (int k = 0; k < 6; ++k)
        if (i >= gr.begin[k] && i < gr.begin[k + 1]) local |= 1 << k;
    }
  }
  if (local)
    for (int k = 0; k < 6; ++k)
      if (local & (1 << k)) atomicOr(&bad[k], 1);
}

__global__ void __launch_bounds__(256)
k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
       float bc1 /* 1 / (1 - beta1^t) */, float bc2 /* 1 / (1 - beta2^t) */, const int* __restrict__ bad) {
  if (*bad) return;  // non-finite gradient: the group keeps its parameters and moments
  constexpr float b1 = 0.9f, b2 = 0.999f, eps = 1e-15f;
  const int64_t i4 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
  if (i4 >= n) return;
  auto one = [&](float& pp, float gg, float& mm, float& vv) {
    mm = fmaf(b1, mm, (1.0f - b1) * gg);
    vv = fmaf(b2, vv, (1.0f - b2) * gg * gg);
    pp -= lr * (mm * bc1) / (sqrtf(vv * bc2) + eps);
  };
  const bool vec = i4 + 4 <= n && ((reinterpret_cast<uintptr_t>(p + i4) | reinterpret_cast<uintptr_t>(g + i4) |
                                    reinterpret_cast<uintptr_t>(m + i4) | reinterpret_cast<uintptr_t>(v + i4)) & 15u) == 0;
  if (vec) {
    float4 P = *reinterpret_cast<float4*>(p + i4), M = *reinterpret_cast<float4*>(m + i4), V = *reinterpret_cast<float4*>(v + i4);
    const float4 G = *reinterpret_cast<const float4*>(g + i4);
    one(P.x, G.x, M.x, V.x); one(P.y, G.y, M.y, V.y); one(P.z, G.z, M.z, V.z); one(P.w, G.w, M.w, V.w);
    *reinterpret_cast<float4*>(p + i4) = P; *reinterpret_cast<float4*>(m + i4) = M; *reinterpret_cast<float4*>(v + i4) = V;
  } else {
    for (int64_t i = i4; i < n && i < i4 + 4; ++i) one(p[i], g[i], m[i], v[i]);
  }
}

// min / max of a bound actor_id array (scene_bind_device validates what scene_upload checks on the host)
__global__ void __launch_bounds__(256) k_actor_id_range(const int32_t* __restrict__ id, int64_t n, int* __restrict__ mn_mx) {
  int lo = 0x7fffffff, hi = -0x7fffffff - 1;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    const int v = id[i];
    lo = min(lo, v); hi = max(hi, v);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { atomicMin(&mn_mx[0], lo); atomicMax(&mn_mx[1], hi); }
}
void launch_actor_id_range(const int32_t* id, int64_t n, int* mn_mx, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>(148 * 4, (n + 255) / 256);
  k_actor_id_range<<<blocks, 256, 0, st>>>(id, n, mn_mx);
}

void launch_grad_finite(const float* g, int64_t n_floats, const AdamGroups& gr, int* bad, cudaStream_t st) {
  if (n_floats <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>(148 * 8, (n_floats + 255) / 256);
  k_grad_finite<<<blocks, 256, 0, st>>>(g, n_floats, gr, bad);
}
void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float bc1, float bc2, const int* bad,
                 cudaStream_t st) {
  if (n <= 0) return;
  k_adam<<<(unsigned)((n + 1023) / 1024), 256, 0, st>>>(p, g, m, v, n, lr, bc1, bc2, bad);
}

}  // namespace sb
