// assign.cu — assign_points_to_tiles: lidar returns -> rasterization points.
// Compiled with --fmad=false like forward.cu: the per-point arithmetic is the exact IEEE sequence of the CPU oracle
// (its assign_one_point), so tile ids and ray coordinates are bit-identical.
//
//   k_assign_points   one thread per point: non-finite -> rejected; sensor-frame position at scan centre ->
//                     position at the point's own capture time under the constant-velocity assumption (the motion
//                     model the rasterizer applies to Gaussians, u = -w x p - v, projection.hpp:44-48) -> Eq. 10
//                     (projection.hpp:122-125) -> the tile holding that zero-extent location; sort key = tile id
//                     (0xffffffff if rejected), plus the shuffle hash of the training mode.
// The stable sort by tile is the binning stage's hand-written radix sort (binning.cu).
#include "kernels.h"

namespace sb {

__device__ __forceinline__ uint32_t point_hash(uint32_t seed, uint32_t index) {
  uint32_t h = index * 0x9E3779B9u + seed;
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;  // murmur3 finaliser
  return h;
}

__global__ void __launch_bounds__(256)
k_assign_points(const __grid_constant__ Sensor s, float timestamp, int64_t n, const float* __restrict__ xyz,
                const float* __restrict__ stamps, uint32_t seed, uint32_t* __restrict__ key, float4* __restrict__ sph,
                uint32_t* __restrict__ hash, uint32_t* __restrict__ valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float pw[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  const float stamp = stamps[i];
  uint32_t k = 0xffffffffu;
  float4 o = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (isfinite(pw[0]) && isfinite(pw[1]) && isfinite(pw[2]) && isfinite(stamp)) {
    float tmp[3], p0[3], c[3];
    mat_vec(s.R, pw, tmp);
#pragma unroll
    for (int a = 0; a < 3; ++a) p0[a] = tmp[a] + s.t[a];
    const float t_l = stamp - timestamp;
    cross3(s.vel_ang, p0, c);
    float p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float u = (-c[a] - s.vel_lin[a]) + 0.0f;
      p[a] = p0[a] + u * t_l;
    }
    const float r = DM_SQRT((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
    if (r > 0.0f && isfinite(r)) {
      const float phi = wrap_two_pi(detmath::atan2(p[1], p[0]));
      const float omega = detmath::asin(p[2] / r);
      int col = (int)floorf(phi / s.span);
      col = min(max(col, 0), s.tiles_x - 1);
      int row = 0;
      for (int b = 0; b < s.n_boundaries; ++b)
        if (s.boundaries[b] < omega) row = b + 1;
      k = (uint32_t)(row * s.tiles_x + col);
      o = make_float4(phi, omega, t_l, r);
    }
  }
  key[i] = k;
  sph[i] = o;
  hash[i] = point_hash(seed, (uint32_t)i);
  valid[i] = k != 0xffffffffu ? 1u : 0u;
}

__global__ void __launch_bounds__(256) k_gather_u32(int64_t n, const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                                                    uint32_t* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

void launch_assign_points(const Sensor& s, float timestamp, int64_t n, const float* xyz, const float* stamps, uint32_t seed,
                          uint32_t* key, float4* sph, uint32_t* hash, uint32_t* valid, cudaStream_t st) {
  if (n <= 0) return;
  k_assign_points<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, timestamp, n, xyz, stamps, seed, key, sph, hash, valid);
}
void launch_gather_u32(int64_t n, const uint32_t* src, const uint32_t* idx, uint32_t* dst, cudaStream_t st) {
  if (n <= 0) return;
  k_gather_u32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, src, idx, dst);
}

}  // namespace sb
