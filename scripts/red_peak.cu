// red_peak.cu — measured ceiling of fire-and-forget global float atomics (RED.E.ADD.F32) on this GPU, the denominator of
// the "atomic throughput" the compositing / projection backward kernels are quoted against (bench.py: roofline.atomic).
// Patterns (all over a 27M-float buffer, the size of SceneParamGrads at 1M Gaussians, i.e. 108 MB — inside the 126 MB L2):
//   coalesced : a warp adds to 32 consecutive floats (4 sectors per instruction), grid-stride sweeps
//   rows26    : the backward kernels' pattern — lanes 0..25 of a warp add to the 13 + 3 + 10 floats of one pseudo-random
//               Gaussian's rows (feature, colour, raw geometric sums: three row starts, ~5 sectors per instruction)
//   scattered : every lane adds to its own pseudo-random float (32 sectors per instruction)
//   one_line  : every warp adds to the same 32 floats (same-address contention: what L2 serialises)
// Build (sm_100a): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_bin/red_peak scripts/red_peak.cu
// Run on the GPU box: scripts/_bin/red_peak > gpurun_out/red_peak.json
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int kPattern>
__global__ void __launch_bounds__(256) k_red(float* __restrict__ buf, uint32_t n_floats, uint32_t n_rows, int iters) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int it = 0; it < iters; ++it) {
    const uint32_t w = gwarp + (uint32_t)it * nwarps;
    if (kPattern == 0) {
      const uint32_t at = (uint32_t)(((uint64_t)w * 32u) % (n_floats - 32u));
      atomicAdd(buf + at + lane, 1.0f);
    } else if (kPattern == 1) {
      const uint32_t g = mix(w) % n_rows;  // one Gaussian per warp instruction
      // [d_feature 13 n | d_color 3 n | raw sums 10 n] laid out as three arrays
      float* dst = lane < 13 ? buf + 13u * g + lane : lane < 16 ? buf + 13u * n_rows + 3u * g + (lane - 13u)
                                                                : buf + 16u * n_rows + 10u * g + (lane - 16u);
      if (lane < 26) atomicAdd(dst, 1.0f);
    } else if (kPattern == 2) {
      atomicAdd(buf + mix(w * 32u + lane) % n_floats, 1.0f);
    } else {
      atomicAdd(buf + lane, 1.0f);
    }
  }
}

template <int kPattern>
static void run(const char* name, float* buf, uint32_t n_floats, uint32_t n_rows, double sectors_per_inst, int lanes, bool last) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, iters = kPattern == 3 ? 64 : 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(buf, 0, sizeof(float) * (size_t)n_floats);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_red<kPattern><<<blocks, 256>>>(buf, n_floats, n_rows, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double insts = (double)blocks * 8.0 * iters;
  printf("  \"%s\": {\"ms\": %.4f, \"warp_instructions\": %.0f, \"g_red_ops_per_s\": %.2f, \"g_sectors_per_s\": %.2f, \"sectors_per_instruction\": %.1f}%s\n",
         name, best, insts, insts * lanes / best / 1e6, insts * sectors_per_inst / best / 1e6, sectors_per_inst, last ? "" : ",");
}

int main() {
  const uint32_t n_rows = 1000000u, n_floats = 27u * n_rows;
  float* buf = nullptr;
  if (cudaMalloc(&buf, sizeof(float) * (size_t)n_floats) != cudaSuccess) { fprintf(stderr, "no CUDA device\n"); return 1; }
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\n  \"device\": \"%s\", \"sms\": %d, \"buffer_bytes\": %zu,\n", p.name, p.multiProcessorCount, sizeof(float) * (size_t)n_floats);
  run<0>("coalesced", buf, n_floats, n_rows, 4.0, 32, false);
  run<1>("rows26", buf, n_floats, n_rows, 5.25, 26, false);  // 13 floats ~2.6 sectors, 3 floats ~1.3, 10 floats ~2.2 (unaligned rows) -> counted exactly by ncu; nominal here
  run<2>("scattered", buf, n_floats, n_rows, 32.0, 32, false);
  run<3>("one_line", buf, n_floats, n_rows, 4.0, 32, true);
  printf("}\n");
  cudaFree(buf);
  return 0;
}
