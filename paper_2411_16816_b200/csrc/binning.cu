// binning.cu — device-wide scan and radix sort used by the tile binning stage (SPEC.md:220-228,
// "Paper inherits 3DGS's global radix sort").
//
// Two narrow stable LSD radix sorts give the reference's (tile_id, depth_key, source_index) order: the
// Gaussians by the IEEE bits of their positive fp32 depth (N entries, 32 bits; the input is in ascending
// source index, which supplies the third criterion), then the duplicated intersections — emitted in that
// depth order — by tile id alone (ceil(log2 T) bits). See forward.cu K3.
#include <cub/cub.cuh>

#include "kernels.h"

namespace sb {

// count of the k-th Gaussian in depth order, widened to int64 (I can exceed 2^31 at 3M Gaussians x 6 cameras)
struct PermutedCount {
  const uint32_t* count;
  const uint32_t* order;
  __host__ __device__ __forceinline__ int64_t operator()(const int64_t& k) const { return (int64_t)count[order[k]]; }
};
using CountIt = cub::TransformInputIterator<int64_t, PermutedCount, cub::CountingInputIterator<int64_t>>;

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  CountIt it(cub::CountingInputIterator<int64_t>(0), PermutedCount{nullptr, nullptr});
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int64_t*)nullptr, n + 1);
  return bytes + 256;
}

// offsets[0..n]: exclusive scan of count[order[k]] with the total in offsets[n]. count and order must have n + 1
// readable entries (the caller keeps one padding element: count[n] = 0, order[n] = n).
void launch_scan_counts(const uint32_t* count, const uint32_t* order, int64_t* offsets, int64_t n, void* temp,
                        size_t temp_bytes, cudaStream_t st) {
  CountIt it(cub::CountingInputIterator<int64_t>(0), PermutedCount{count, order});
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, it, offsets, n + 1, st);
}

void launch_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n + 1, st);
}

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, n, 0, 32);
  return bytes + 256;
}

int launch_sort_pairs(uint32_t* keys0, uint32_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t n, int key_bits,
                      void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DoubleBuffer<uint32_t> k(keys0, keys1);
  cub::DoubleBuffer<uint32_t> v(vals0, vals1);
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, n, 0, key_bits, st);
  return k.selector;
}

}  // namespace sb
