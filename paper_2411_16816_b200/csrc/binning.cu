// binning.cu — device-wide scan and radix sort used by the tile binning stage (SPEC.md:220-228,
// "Paper inherits 3DGS's global radix sort").
//
// The sort key is tile_id << 32 | IEEE bits of the positive fp32 depth, so an LSD radix sort over
// the live bits [0, 32 + ceil(log2(tiles))) orders by (tile, depth); LSD radix sort is stable, and
// the key stream is emitted in ascending source index, which supplies the reference's third sort
// criterion (source_index) for free.
#include <cub/cub.cuh>

#include "kernels.h"

namespace sb {

struct U32ToI64 {
  __host__ __device__ __forceinline__ int64_t operator()(const uint32_t& v) const { return (int64_t)v; }
};

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::TransformInputIterator<int64_t, U32ToI64, const uint32_t*> it(nullptr, U32ToI64());
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int64_t*)nullptr, n + 1);
  return bytes + 256;
}

// offsets[0..n]: exclusive scan of count[0..n) with the total in offsets[n]. count must have n + 1
// readable entries with count[n] ignored (the caller keeps one padding element set to 0).
void launch_scan_counts(const uint32_t* count, int64_t* offsets, int64_t n, void* temp, size_t temp_bytes,
                        cudaStream_t st) {
  cub::TransformInputIterator<int64_t, U32ToI64, const uint32_t*> it(count, U32ToI64());
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, it, offsets, n + 1, st);
}

void launch_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n + 1, st);
}

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint64_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, n, 0, 64);
  return bytes + 256;
}

int launch_sort_pairs(uint64_t* keys0, uint64_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t n, int key_bits,
                      void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DoubleBuffer<uint64_t> k(keys0, keys1);
  cub::DoubleBuffer<uint32_t> v(vals0, vals1);
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, n, 0, key_bits, st);
  return k.selector;
}

}  // namespace sb
