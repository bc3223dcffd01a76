// binning.cu — hand-written device radix sort, scans and tile histogram of the tile binning stage
// ("Paper inherits 3DGS's global radix sort"). No library kernels.
//
// The worklist order the reference specifies is (tile_id, depth_key, source_index). It is produced by two narrow
// stable LSD radix sorts instead of one wide one:
//   1. the Gaussians are sorted by the IEEE bits of their positive fp32 depth (N entries, 4 x 8 bits; the input is in
//      ascending source index, which supplies the third criterion; culled Gaussians carry 0xffffffff and end up
//      behind every visible one)                                         k_radix_hist + 4 x k_radix_pass;
//   2. an exclusive scan of the tile counts in that order gives every Gaussian's first intersection
//                                                                       k_count_scan (single pass, look-back);
//   3. the per-tile list lengths do not need the list: every visible Gaussian adds its tile rectangle to a 2-D
//      difference array (4 REDs), whose 2-D prefix sum is the number of Gaussians per tile; one more scan gives
//      tile_begin/tile_end, the digit histograms of step 4 and the longest-first CTA order of the compositing kernels
//                                                                       k_tile_hist + k_tile_scan;
//   4. the intersections are sorted by tile id alone — ceil(log2 T) bits in ceil(bits / 8) passes. The first pass
//      GENERATES its input (each Gaussian's tiles in row-major order, Gaussians in depth order) instead of reading it,
//      the last pass writes source indices only: 20 B of traffic per intersection for a 1080p image where
//      emit + library sort + range extraction moved 52 B.             k_radix_pass<emit>, k_radix_pass<vals only>
//
// k_radix_pass is a onesweep pass (one read, one write per pass): CTAs take 4,096-item tiles in ticket order, rank
// their items per digit with warp match ballots (stable), publish per-digit counts and resolve their global offsets by
// decoupled look-back over the preceding tiles' counts, then scatter through shared memory so that global writes
// are runs of equal digits.
#include "kernels.h"

namespace sb {

namespace {

constexpr int kRThreads = 512;
constexpr int kRItems = 8;
constexpr int kRTile = kRThreads * kRItems;  // 4,096 items per CTA
constexpr int kRWarps = kRThreads / 32;
constexpr int kRMaxBins = 256;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1u;
constexpr uint32_t kSpinLimit = 1u << 24;  // look-back polls before giving up (a lost predecessor must not hang the GPU)

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }
__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile64(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// Exclusive scan of one value per thread over a 256-thread CTA; `total` receives the CTA sum. s_warp: 8 words.
template <int kWarps = kRWarps>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __syncthreads();  // s_warp may still be read from a previous call
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t base = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = s_warp[w];
    if (w < warp) base += c;
    tot += c;
  }
  total = tot;
  return base + inc - v;
}

// tile rectangle -> rectangle on the grid of 2^shift x 2^shift-tile blocks
__device__ __forceinline__ int4 coarse_rect(int4 r, int shift) {
  const int up = (1 << shift) - 1;
  return make_int4(r.x >> shift, (r.y + up) >> shift, r.z >> shift, (r.w + up) >> shift);
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// Digit histograms of 32-bit keys, all four 8-bit digits in one read.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s[4 * 256];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * 256; i += 256) s[i] = 0u;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * 256 * 4;
  for (int64_t i = ((int64_t)blockIdx.x * 256 + tid) * 4; i < n; i += stride) {
    uint32_t k[4];
    int m = 4;
    if (i + 4 <= n) {
      const uint4 q = *reinterpret_cast<const uint4*>(keys + i);
      k[0] = q.x; k[1] = q.y; k[2] = q.z; k[3] = q.w;
    } else {
      m = (int)(n - i);
      for (int u = 0; u < m; ++u) k[u] = keys[i + u];
    }
    for (int u = 0; u < m; ++u) {
#pragma unroll
      for (int p = 0; p < 4; ++p) atomicAdd(&s[p * 256 + ((k[u] >> (8 * p)) & 255u)], 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < 4 * 256; i += 256)
    if (s[i]) atomicAdd(&hist[i], s[i]);
}

// ------------------------------------------------------------------------------------------------
// One onesweep pass. kSrc: 0 = (keys, vals) from memory; 1 = keys from memory, vals = position (first pass of the
// depth sort: no iota buffer); 2 = the duplication step itself — item e of the input is the e-th (tile id, source
// index) pair of the emitted stream, generated from the depth-ordered offsets and the tile rectangles.
// ------------------------------------------------------------------------------------------------
struct EmitSrc {
  int64_t n;               // Gaussians
  const uint32_t* offsets; // n + 1, exclusive scan of the tile counts over the depth-sorted order (I < 2^30)
  const uint32_t* order;   // depth-sorted position -> source index
  const int4* rect;
  int tiles_x, wrap_x;     // grid the keys are generated on (the coarse grid if shift > 0)
  int shift;
};

constexpr int kStagePad = kRTile + kRTile / 16;  // staging index x + (x >> 4): conflict-free blocked writes, striped reads
constexpr size_t kRadixSmem = sizeof(uint32_t) * (2 * kStagePad + (kRTile + 2));

template <int kSrc, bool kWriteKeys>
__global__ void __launch_bounds__(kRThreads, 2)
k_radix_pass(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
             uint32_t* __restrict__ vals_out, int64_t n, int shift, int bits, const uint32_t* __restrict__ hist,
             uint32_t* __restrict__ state, uint32_t* __restrict__ ticket, uint32_t* __restrict__ err, EmitSrc em) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* s_keys = smem;                  // kStagePad
  uint32_t* s_vals = smem + kStagePad;      // kStagePad
  uint32_t* s_u = smem + 2 * kStagePad;     // kRTile + 2: emit offsets, then the per-warp digit counters (8 x 256)
  __shared__ uint32_t s_cstart[kRMaxBins], s_gbase[kRMaxBins], s_warp[kRWarps];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = 1 << bits;
  const uint32_t dmask = (uint32_t)nb - 1u;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t e0 = (int64_t)tile * kRTile;
  const int cnt = (int)min((int64_t)kRTile, n - e0);

  uint32_t key[kRItems], val[kRItems];
  if (kSrc == 2) {
    // (a) owner of the tile's first intersection: 256-ary search, offsets[k0] <= e0 < offsets[k0 + 1]
    int64_t lo = 0, hi = em.n;
    while (hi - lo > 1) {
      const int64_t step = (hi - lo + kRThreads - 1) / kRThreads;
      const int64_t idx = lo + (int64_t)(tid + 1) * step;
      const int c = __syncthreads_count(idx < hi && (int64_t)em.offsets[idx] <= e0);
      lo += (int64_t)c * step;
      hi = min(hi, lo + step);
    }
    const int64_t k0 = lo;
    // (b) the offsets of the <= 4,097 Gaussians the tile spans, relative to e0 (every entry in front of the culled tail
    //     owns >= 1 intersection)
    int* s_off = reinterpret_cast<int*>(s_u);
    const int span = (int)min((int64_t)(kRTile + 2), em.n + 1 - k0);
    for (int x = tid; x < span; x += kRThreads)
      s_off[x] = (int)min((int64_t)em.offsets[k0 + x] - e0, (int64_t)(kRTile + 1));
    __syncthreads();
    // (c) 16 consecutive intersections per thread: one binary search, then a walk through the owners' rectangles
    const int x0 = tid * kRItems;
    if (x0 < cnt) {
      int l = 0, h = span - 1;  // s_off[l] <= x0 < s_off[h]
      while (h - l > 1) {
        const int mid = (l + h) >> 1;
        if (s_off[mid] <= x0) l = mid;
        else h = mid;
      }
      uint32_t src = em.order[k0 + l];
      int4 r = coarse_rect(em.rect[src], em.shift);
      int w = r.y - r.x;
      int next = s_off[l + 1];
      const int local = x0 - s_off[l];
      int ly = local / w, lx = local - ly * w;
      const int tx = em.tiles_x;
      auto wrapped = [&](int x) { return em.wrap_x ? ((x % tx) + tx) % tx : x; };
      int xw = wrapped(r.x + lx);
#pragma unroll
      for (int u = 0; u < kRItems; ++u) {
        const int x = x0 + u;
        if (x < cnt) {
          while (x >= next) {
            ++l;
            next = s_off[l + 1];
            src = em.order[k0 + l];
            r = coarse_rect(em.rect[src], em.shift);
            w = r.y - r.x;
            lx = 0; ly = 0;
            xw = wrapped(r.x);
          }
          const int p = x + (x >> 4);
          s_keys[p] = (uint32_t)((r.z + ly) * tx + xw);
          s_vals[p] = src;
          ++lx; ++xw;
          if (xw == tx && em.wrap_x) xw = 0;
          if (lx == w) { lx = 0; ++ly; xw = wrapped(r.x); }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
      const int x = warp * (kRItems * 32) + i * 32 + lane;
      const int p = x + (x >> 4);
      key[i] = s_keys[p];
      val[i] = s_vals[p];
    }
    __syncthreads();  // staging and s_off are reused below
  } else {
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
      const int x = warp * (kRItems * 32) + i * 32 + lane;
      key[i] = 0u; val[i] = 0u;
      if (x < cnt) {
        key[i] = keys_in[e0 + x];
        val[i] = kSrc == 1 ? (uint32_t)(e0 + x) : vals_in[e0 + x];
      }
    }
  }

  // ---- stable ranks inside the warp's 512 items (item order: round i, then lane) --------------------------------
  uint32_t* s_wcnt = s_u + warp * kRMaxBins;
  for (int b = lane; b < nb; b += 32) s_wcnt[b] = 0u;
  __syncwarp();
  // matches first: 16 independent MATCH instructions in flight, then the (short) sequential walk over the counters
  uint32_t rank[kRItems];  // holds the peer mask until the walk replaces it
  const uint32_t lt = (1u << lane) - 1u;
  const bool full = cnt == kRTile;
  if (full) {
#pragma unroll
    for (int i = 0; i < kRItems; ++i) rank[i] = __match_any_sync(0xffffffffu, (key[i] >> shift) & dmask);
  } else {
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
      const bool valid = warp * (kRItems * 32) + i * 32 + lane < cnt;
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      rank[i] = 0u;
      if (valid) rank[i] = __match_any_sync(vm, (key[i] >> shift) & dmask);
    }
  }
#pragma unroll
  for (int i = 0; i < kRItems; ++i) {
    const uint32_t peers = rank[i];
    const uint32_t d = (key[i] >> shift) & dmask;
    const int leader = peers ? __ffs(peers) - 1 : 0;
    uint32_t pre = 0u;
    if (peers && lane == leader) {
      pre = s_wcnt[d];
      s_wcnt[d] = pre + __popc(peers);
    }
    __syncwarp();  // this round's counter updates are visible to the next round's leaders
    pre = __shfl_sync(0xffffffffu, pre, leader);
    rank[i] = pre + __popc(peers & lt);
  }
  __syncthreads();

  // ---- per-digit counts of the CTA, their offsets across warps, and the look-back ------------------------------
  uint32_t cta_count = 0u;
  if (tid < nb) {
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
      const uint32_t c = s_u[w * kRMaxBins + tid];
      s_u[w * kRMaxBins + tid] = cta_count;
      cta_count += c;
    }
    st_volatile(&state[(size_t)tile * nb + tid], (tile == 0 ? kFlagPrefix : kFlagAgg) | cta_count);
  }
  uint32_t dummy;
  const uint32_t cstart = block_excl_scan(cta_count, s_warp, dummy);
  const uint32_t ghist = block_excl_scan(tid < nb ? hist[tid] : 0u, s_warp, dummy);
  if (tid < nb) {
    uint32_t excl = 0u;
    if (tile > 0) {
      // look back over the preceding tiles' counts, 8 tiles per step (independent loads), until an inclusive prefix
      int64_t t = (int64_t)tile - 1;
      uint32_t spins = 0u;
      bool done = false;
      while (!done) {
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = (t - u >= 0) ? ld_volatile(&state[(size_t)(t - u) * nb + tid]) : kFlagPrefix;
        bool stall = false;
        int used = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!done && !stall) {
            const uint32_t f = w[u] >> 30;
            if (f == 0u) stall = true;
            else { excl += w[u] & kValMask; ++used; done = f != 1u; }
          }
        }
        t -= used;
        if (stall && ++spins > kSpinLimit) { *err = 1u; done = true; }
      }
      st_volatile(&state[(size_t)tile * nb + tid], kFlagPrefix | (excl + cta_count));
    }
    s_cstart[tid] = cstart;
    s_gbase[tid] = ghist + excl - cstart;  // + position in the CTA's sorted buffer = global position
  }
  __syncthreads();

  // ---- scatter to the sorted order in shared memory, then write runs of equal digits ---------------------------
#pragma unroll
  for (int i = 0; i < kRItems; ++i) {
    const int x = warp * (kRItems * 32) + i * 32 + lane;
    if (x < cnt) {
      const uint32_t d = (key[i] >> shift) & dmask;
      // consecutive tile ids land a whole bin apart: XOR-swizzle the position so that they hit different banks
      uint32_t pos = s_cstart[d] + s_wcnt[d] + rank[i];
      pos ^= (pos >> 5) & 31u;
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  __syncthreads();
  for (int j = tid; j < cnt; j += kRThreads) {
    const int js = j ^ ((j >> 5) & 31);
    const uint32_t k = s_keys[js];
    const uint32_t g = s_gbase[(k >> shift) & dmask] + (uint32_t)j;
    if (kWriteKeys) keys_out[g] = k;
    vals_out[g] = s_vals[js];
  }
}

// ------------------------------------------------------------------------------------------------
// offsets[k] = sum_{k' < k} count[order[k']] for k in [0, n], one pass with decoupled look-back. 32-bit: a view holds
// fewer than 2^30 intersections (the host checks the 64-bit total of k_tile_scan before anything reads the offsets).
// ------------------------------------------------------------------------------------------------
constexpr int kSItems = 8;
constexpr int kSTile = 256 * kSItems;

__global__ void __launch_bounds__(256)
k_count_scan(const uint32_t* __restrict__ count, const uint32_t* __restrict__ order, int64_t n, uint32_t* __restrict__ offsets,
             uint32_t* __restrict__ state, uint32_t* __restrict__ ticket, uint32_t* __restrict__ err) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_tile, s_base;
  __shared__ uint32_t s_out[kSTile + kSTile / 8];  // index j + (j >> 3): blocked writes, striped reads, no conflicts
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base_k = (int64_t)tile * kSTile;
  const int64_t k0 = base_k + (int64_t)tid * kSItems;
  uint32_t o[kSItems], c[kSItems];
  if (k0 + kSItems <= n) {  // two 128-bit loads of the order, then the gathers
    const uint4 a = *reinterpret_cast<const uint4*>(order + k0), b = *reinterpret_cast<const uint4*>(order + k0 + 4);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
#pragma unroll
    for (int u = 0; u < kSItems; ++u) c[u] = count[o[u]];
  } else {
#pragma unroll
    for (int u = 0; u < kSItems; ++u) c[u] = (k0 + u < n) ? count[order[k0 + u]] : 0u;
  }
  uint32_t mine = 0u;
#pragma unroll
  for (int u = 0; u < kSItems; ++u) mine += c[u];
  uint32_t total;
  const uint32_t excl_in_tile = block_excl_scan<8>(mine, s_warp, total);
  if (tid < 32) {
    // Look-back by one WARP, 32 predecessors per step (one load per lane, ballots, one warp sum). Every tile of the scan
    // is resident at once (489 at 1M Gaussians), so a late tile sums most of its predecessors' aggregates: one thread
    // reading 8 per step left the other 255 threads of every CTA at the barrier below (ncu: 41 barrier-stall cycles
    // per issued instruction).
    const int lane = tid;
    uint32_t excl = 0u;
    if (lane == 0) st_volatile(&state[tile], (tile == 0 ? kFlagPrefix : kFlagAgg) | total);
    int64_t t = (int64_t)tile - 1;
    uint32_t spins = 0u;
    bool done = tile == 0;
    while (!done) {
      const int64_t idx = t - lane;
      const uint32_t w = idx >= 0 ? ld_volatile(&state[idx]) : kFlagPrefix;
      const uint32_t f = w >> 30;
      const unsigned notready = __ballot_sync(0xffffffffu, f == 0u);
      const unsigned pref = __ballot_sync(0xffffffffu, f != 0u && f != 1u);
      const int fp = pref ? __ffs(pref) - 1 : 31;              // lanes 0 .. fp are needed
      const unsigned need = fp >= 31 ? 0xffffffffu : ((2u << fp) - 1u);
      if (notready & need) {                                     // a needed predecessor has not published yet
        if (++spins > kSpinLimit) { if (lane == 0) *err = 1u; done = true; }
        continue;
      }
      excl += __reduce_add_sync(0xffffffffu, ((need >> lane) & 1u) ? (w & kValMask) : 0u);
      if (pref) done = true;
      else t -= 32;
    }
    if (lane == 0) {
      if (tile != 0) st_volatile(&state[tile], kFlagPrefix | ((excl + total) & kValMask));
      s_base = excl;
    }
  }
  __syncthreads();
  uint32_t run = s_base + excl_in_tile;
#pragma unroll
  for (int u = 0; u < kSItems; ++u) {
    const int j = tid * kSItems + u;
    s_out[j + (j >> 3)] = run;
    run += c[u];
  }
  __syncthreads();
  for (int j = tid; j < kSTile; j += 256)
    if (base_k + j <= n) offsets[base_k + j] = s_out[j + (j >> 3)];  // k == n: the grand total
}

// ------------------------------------------------------------------------------------------------
// Per-tile list lengths without the list. Every visible Gaussian either increments the tiles of a small rectangle
// directly or adds a large rectangle to a 2-D difference array (4 REDs); k_tile_scan prefix-sums the latter and adds
// the two. Each tile's two counters live in their own 128-byte line (kTileStride ints): L2 serialises atomics per line,
// and 1,000 lidar tiles packed into 32 lines made this kernel 0.6 ms.
// `shift` > 0 counts on the coarse grid of 2^shift x 2^shift tiles (the first level of the camera's two-level binning).
// ------------------------------------------------------------------------------------------------
constexpr int kTileStride = 32;  // ints per tile slot: [0] difference array, [1] direct count
constexpr int kDirectMax = 4;    // rectangles of up to this many tiles are counted directly

__global__ void __launch_bounds__(256)
k_tile_hist(int64_t n, const uint32_t* __restrict__ count, const int4* __restrict__ rect, int shift, int tiles_x, int wrap_x,
            int* __restrict__ slots /* (tiles_y + 1) x (tiles_x + 1) x kTileStride */) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (count[i] == 0u) return;
  const int4 r = coarse_rect(rect[i], shift);
  const int W = tiles_x + 1;
  const int w = r.y - r.x;
  const uint32_t cnt = (uint32_t)w * (uint32_t)(r.w - r.z);
  const int x0 = wrap_x ? ((r.x % tiles_x) + tiles_x) % tiles_x : r.x;  // lidar: columns are x mod M_phi, width <= M_phi
  if (cnt <= (uint32_t)kDirectMax) {
    for (int y = r.z; y < r.w; ++y) {
      int x = x0;
      for (int k = 0; k < w; ++k) {
        atomicAdd(&slots[(size_t)(y * W + x) * kTileStride + 1], 1);
        if (++x == tiles_x) x = 0;  // only a wrapped lidar rectangle gets here
      }
    }
    return;
  }
  auto add = [&](int xa, int xb) {
    atomicAdd(&slots[(size_t)(r.z * W + xa) * kTileStride], 1);
    atomicAdd(&slots[(size_t)(r.z * W + xb) * kTileStride], -1);
    atomicAdd(&slots[(size_t)(r.w * W + xa) * kTileStride], -1);
    atomicAdd(&slots[(size_t)(r.w * W + xb) * kTileStride], 1);
  };
  if (x0 + w <= tiles_x) add(x0, x0 + w);
  else { add(x0, tiles_x); add(0, x0 + w - tiles_x); }
}

// The same counts through a per-CTA shared-memory copy of the slot grid (small grids: the lidar's tiles, the camera's
// 8 x 8-tile blocks). On the camera's 135-block grid every visible Gaussian's increments land on 135 cache lines and L2
// serialises atomics per line (36 us for 248k Gaussians); here a CTA accumulates ~1,700 Gaussians in shared memory
// (integer shared atomics are native) and flushes its non-zero counters: one global atomic per (CTA, slot).
constexpr int kHistSmemSlots = 2048;
__global__ void __launch_bounds__(256)
k_tile_hist_smem(int64_t n, const uint32_t* __restrict__ count, const int4* __restrict__ rect, int shift, int tiles_x, int tiles_y,
                 int wrap_x, int* __restrict__ slots) {
  __shared__ int s_diff[kHistSmemSlots], s_dir[kHistSmemSlots];
  const int W = tiles_x + 1, S = W * (tiles_y + 1);
  for (int k = threadIdx.x; k < S; k += 256) { s_diff[k] = 0; s_dir[k] = 0; }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    if (count[i] == 0u) continue;
    const int4 r = coarse_rect(rect[i], shift);
    const int w = r.y - r.x;
    const uint32_t cnt = (uint32_t)w * (uint32_t)(r.w - r.z);
    const int x0 = wrap_x ? ((r.x % tiles_x) + tiles_x) % tiles_x : r.x;
    if (cnt <= (uint32_t)kDirectMax) {
      for (int y = r.z; y < r.w; ++y) {
        int x = x0;
        for (int k = 0; k < w; ++k) {
          atomicAdd(&s_dir[y * W + x], 1);
          if (++x == tiles_x) x = 0;
        }
      }
      continue;
    }
    auto add = [&](int xa, int xb) {
      atomicAdd(&s_diff[r.z * W + xa], 1);
      atomicAdd(&s_diff[r.z * W + xb], -1);
      atomicAdd(&s_diff[r.w * W + xa], -1);
      atomicAdd(&s_diff[r.w * W + xb], 1);
    };
    if (x0 + w <= tiles_x) add(x0, x0 + w);
    else { add(x0, tiles_x); add(0, x0 + w - tiles_x); }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < S; k += 256) {
    const int d = s_diff[k], c = s_dir[k];
    if (d) atomicAdd(&slots[(size_t)k * kTileStride], d);
    if (c) atomicAdd(&slots[(size_t)k * kTileStride + 1], c);
  }
}

// One CTA: gathers the slots into a compact array (shared memory when the grid fits, a global scratch otherwise),
// 2-D prefix sum of the difference array, exclusive scan over the tiles -> tile_begin / tile_end (0, 0 for an empty
// tile, like the oracle), the digit histograms of the tile sort's passes, the total, and the CTA -> tile permutation of
// the compositing kernels (longest lists first: counting sort over 256 length buckets).
struct TilePasses {
  int n_pass;
  int shift[4], bits[4];
};

__global__ void __launch_bounds__(1024)
k_tile_scan(int tiles_x, int tiles_y, const int* __restrict__ slots, int* __restrict__ gscratch /* 2 T ints or null */,
            uint32_t* __restrict__ tile_begin, uint32_t* __restrict__ tile_end, uint32_t* __restrict__ hist /* n_pass x 256 or null */,
            TilePasses tp, uint32_t* __restrict__ tile_order /* or null */, int64_t* __restrict__ total_out,
            uint32_t* __restrict__ seg_first /* T + 1 or null: exclusive scan of ceil(length / seg_len) */, int seg_len) {
  extern __shared__ int s_dyn[];
  __shared__ unsigned long long s_wsum[32];
  __shared__ uint32_t s_hist[4 * kRMaxBins];
  __shared__ unsigned s_max;
  __shared__ unsigned s_len[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = tiles_x + 1;
  const int T = tiles_x * tiles_y;
  int* a = gscratch ? gscratch : s_dyn;  // T: difference array -> list lengths
  int* dir = a + T;                       // T: directly counted rectangles
  for (int i = tid; i < 4 * kRMaxBins; i += 1024) s_hist[i] = 0u;
  if (tid < 256) s_len[tid] = 0u;
  if (tid == 0) s_max = 1u;
  for (int t = tid; t < T; t += 1024) {
    const size_t g = (size_t)((t / tiles_x) * W + (t % tiles_x)) * kTileStride;
    a[t] = slots[g];
    dir[t] = slots[g + 1];
  }
  __syncthreads();
  // rows: a warp per row, 32 columns per step
  for (int y = warp; y < tiles_y; y += 32) {
    int carry = 0;
    for (int xb = 0; xb < tiles_x; xb += 32) {
      const int x = xb + lane;
      int v = x < tiles_x ? a[y * tiles_x + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      v += carry;
      if (x < tiles_x) a[y * tiles_x + x] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // columns: a warp per column, 32 rows per step; the directly counted rectangles are folded in on the way
  for (int x = warp; x < tiles_x; x += 32) {
    int carry = 0;
    for (int yb = 0; yb < tiles_y; yb += 32) {
      const int y = yb + lane;
      int v = y < tiles_y ? a[y * tiles_x + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      v += carry;
      if (y < tiles_y) a[y * tiles_x + x] = v + dir[y * tiles_x + x];
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // exclusive scan over the tiles (row-major ids): each thread owns a run of consecutive tiles
  const int per = (T + 1023) / 1024;
  const int t0 = tid * per, t1 = min(T, t0 + per);
  unsigned long long mine = 0ull;
  unsigned mx = 0u;
  for (int t = t0; t < t1; ++t) {
    const unsigned c = (unsigned)a[t];
    mine += c;
    mx = max(mx, c);
  }
  unsigned long long inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 31) s_wsum[warp] = inc;
  if (lane == 0) atomicMax(&s_max, mx);
  __syncthreads();
  unsigned long long base = 0ull, total = 0ull;
  for (int w = 0; w < 32; ++w) {
    const unsigned long long v = s_wsum[w];
    if (w < warp) base += v;
    total += v;
  }
  if (tid == 0) *total_out = (int64_t)total;
  if (seg_first) {  // segments of the lists (two-level binning): a second scan over the same runs
    __syncthreads();
    unsigned long long segs = 0ull;
    for (int t = t0; t < t1; ++t) segs += ((unsigned)a[t] + (unsigned)seg_len - 1u) / (unsigned)seg_len;
    unsigned long long sinc = segs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, sinc, o);
      if (lane >= o) sinc += u;
    }
    if (lane == 31) s_wsum[warp] = sinc;
    __syncthreads();
    unsigned long long sbase = 0ull, stotal = 0ull;
    for (int w = 0; w < 32; ++w) {
      const unsigned long long v = s_wsum[w];
      if (w < warp) sbase += v;
      stotal += v;
    }
    unsigned long long srun = sbase + sinc - segs;
    for (int t = t0; t < t1; ++t) {
      seg_first[t] = (uint32_t)srun;
      srun += ((unsigned)a[t] + (unsigned)seg_len - 1u) / (unsigned)seg_len;
    }
    if (tid == 0) seg_first[T] = (uint32_t)stotal;
  }
  const float scale = 255.0f / (float)s_max;
  unsigned long long run = base + inc - mine;
  for (int t = t0; t < t1; ++t) {
    const unsigned c = (unsigned)a[t];
    tile_begin[t] = c ? (uint32_t)run : 0u;
    tile_end[t] = c ? (uint32_t)(run + c) : 0u;
    run += c;
    if (c && hist) {
      for (int p = 0; p < tp.n_pass; ++p)
        atomicAdd(&s_hist[p * kRMaxBins + (((uint32_t)t >> tp.shift[p]) & ((1u << tp.bits[p]) - 1u))], c);
    }
    atomicAdd(&s_len[255 - (int)((float)c * scale)], 1u);
  }
  __syncthreads();
  if (hist)
    for (int i = tid; i < tp.n_pass * kRMaxBins; i += 1024) hist[i] = s_hist[i];
  if (!tile_order) return;
  if (tid == 0) {  // exclusive scan of the 256 length buckets
    unsigned r = 0u;
    for (int b = 0; b < 256; ++b) { const unsigned c = s_len[b]; s_len[b] = r; r += c; }
  }
  __syncthreads();
  for (int t = t0; t < t1; ++t)
    tile_order[atomicAdd(&s_len[255 - (int)((float)(unsigned)a[t] * scale)], 1u)] = (uint32_t)t;
}

// ------------------------------------------------------------------------------------------------
// Second level of the camera's binning: the depth-ordered list of every 8 x 8-tile block (the output of the coarse
// sort) is cut into segments of 1,024 entries; one CTA per segment appends its Gaussians to the lists of the tiles
// their rectangles cover. A Gaussian covering all 8,160 tiles of a 1080p image costs 135 coarse entries + 8,160
// four-byte stores instead of 8,160 sorted key-value pairs.
//   1. gather (source index -> rectangle) and turn each rectangle into a 64-bit tile mask of the block;
//   2. count the segment's entries per tile (per-lane adds, one warp reduction per tile);
//   3. publish the 64 counts and look back over the preceding segments of the same block (decoupled look-back)
//      -> the segment's first position in each of the 64 tile lists;
//   4. warp w owns tile row w: ballot ranks keep the list order, every store instruction writes a run of
//      consecutive positions of one tile list.
// ------------------------------------------------------------------------------------------------
constexpr int kSuperShift = 3;
constexpr int kSuper = 1 << kSuperShift;
constexpr int kSeg = 1024;

__global__ void __launch_bounds__(256)
k_expand(int stiles_x, int n_super, int tiles_x, int tiles_y, const uint32_t* __restrict__ super_begin,
         const uint32_t* __restrict__ super_end, const uint32_t* __restrict__ seg_first /* n_super + 1 */,
         const uint32_t* __restrict__ cvals, const int4* __restrict__ rect, const uint32_t* __restrict__ tile_begin,
         uint32_t* __restrict__ state /* segments x 64 */, uint32_t* __restrict__ ticket, uint32_t* __restrict__ err,
         uint32_t* __restrict__ vals) {
  __shared__ uint32_t s_src[kSeg];
  __shared__ unsigned long long s_mask[kSeg];
  __shared__ uint32_t s_cnt[64], s_cursor[64];
  __shared__ uint32_t s_seg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_seg = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t seg = s_seg;
  if (seg >= seg_first[n_super]) return;
  // block owning this segment: seg_first[st] <= seg < seg_first[st + 1] (256-ary search)
  int lo = 0, hi = n_super;
  while (hi - lo > 1) {
    const int step = (hi - lo + 255) / 256;
    const int idx = lo + (tid + 1) * step;
    const int c = __syncthreads_count(idx < hi && seg_first[idx] <= seg);
    lo += c * step;
    hi = min(hi, lo + step);
  }
  const int st = lo;
  const uint32_t j = seg - seg_first[st];  // segment index inside the block's list
  const uint32_t lb = super_begin[st] + j * kSeg;
  const int cnt = (int)min((uint32_t)kSeg, super_end[st] - lb);
  const int bx = (st % stiles_x) * kSuper, by = (st / stiles_x) * kSuper;

  // 1. gather + masks
#pragma unroll
  for (int u = 0; u < kSeg / 256; ++u) {
    const int e = u * 256 + tid;
    uint32_t src = 0u;
    unsigned long long m = 0ull;
    if (e < cnt) {
      src = cvals[lb + e];
      const int4 r = rect[src];
      const int xlo = max(r.x - bx, 0), xhi = min(r.y - bx, kSuper);
      const int ylo = max(r.z - by, 0), yhi = min(r.w - by, kSuper);
      if (xlo < xhi && ylo < yhi) {
        const unsigned long long xbits = ((1u << xhi) - 1u) & ~((1u << xlo) - 1u);
        const unsigned long long rows_hi = yhi >= kSuper ? ~0ull : ((1ull << (8 * yhi)) - 1ull);
        const unsigned long long rows_lo = (1ull << (8 * ylo)) - 1ull;
        m = (xbits * 0x0101010101010101ull) & rows_hi & ~rows_lo;
      }
    }
    s_src[e] = src;
    s_mask[e] = m;
  }
  __syncthreads();

  // 2. per-tile counts of the segment: warp w counts tile row w
  const int ksteps = (cnt + 31) >> 5;
  {
    uint32_t acc[kSuper];
#pragma unroll
    for (int c = 0; c < kSuper; ++c) acc[c] = 0u;
    for (int k = 0; k < ksteps; ++k) {
      const uint32_t m8 = (uint32_t)(s_mask[k * 32 + lane] >> (8 * warp)) & 0xffu;
#pragma unroll
      for (int c = 0; c < kSuper; ++c) acc[c] += (m8 >> c) & 1u;
    }
#pragma unroll
    for (int c = 0; c < kSuper; ++c) {
      const uint32_t tot = __reduce_add_sync(0xffffffffu, acc[c]);
      if (lane == c) s_cnt[warp * kSuper + c] = tot;
    }
  }
  __syncthreads();

  // 3. first position of the segment in each tile list
  if (tid < 64) {
    const uint32_t mine = s_cnt[tid];
    uint32_t excl = 0u;
    if (j == 0) {
      st_volatile(&state[(size_t)seg * 64 + tid], kFlagPrefix | mine);
    } else {
      st_volatile(&state[(size_t)seg * 64 + tid], kFlagAgg | mine);
      int64_t t = (int64_t)seg - 1;
      const int64_t t_first = (int64_t)seg - (int64_t)j;  // first segment of this block
      uint32_t spins = 0u;
      bool done = false;
      while (!done) {
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = (t - u >= t_first) ? ld_volatile(&state[(size_t)(t - u) * 64 + tid]) : kFlagPrefix;
        bool stall = false;
        int used = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!done && !stall) {
            const uint32_t f = w[u] >> 30;
            if (f == 0u) stall = true;
            else { excl += w[u] & kValMask; ++used; done = f != 1u; }
          }
        }
        t -= used;
        if (stall && ++spins > kSpinLimit) { *err = 1u; done = true; }
      }
      st_volatile(&state[(size_t)seg * 64 + tid], kFlagPrefix | (excl + mine));
    }
    const int tx = bx + (tid & 7), ty = by + (tid >> 3);
    s_cursor[tid] = excl + ((tx < tiles_x && ty < tiles_y) ? tile_begin[ty * tiles_x + tx] : 0u);
  }
  __syncthreads();

  // 4. append: warp w walks the segment for tile row w
  uint32_t pos[kSuper];
#pragma unroll
  for (int c = 0; c < kSuper; ++c) pos[c] = s_cursor[warp * kSuper + c];
  const uint32_t lt = (1u << lane) - 1u;
  for (int k = 0; k < ksteps; ++k) {
    const int e = k * 32 + lane;
    const uint32_t m8 = (uint32_t)(s_mask[e] >> (8 * warp)) & 0xffu;  // 0 beyond cnt
    const uint32_t src = s_src[e];
#pragma unroll
    for (int c = 0; c < kSuper; ++c) {
      const uint32_t bit = (m8 >> c) & 1u;
      const unsigned b = __ballot_sync(0xffffffffu, bit != 0u);
      const uint32_t rank = __popc(b & lt);
      if (bit) vals[pos[c] + rank] = src;
      pos[c] += __shfl_sync(0xffffffffu, rank + bit, 31);  // = popc(b), without a second trip through the XU pipe
    }
  }
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
namespace {
inline int64_t radix_tiles(int64_t n) { return (n + kRTile - 1) / kRTile; }
constexpr size_t kHdrWords = 64;  // tickets [0..15], error flag [16]

template <int kSrc, bool kWriteKeys>
void launch_pass(const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo, int64_t n, int shift, int bits,
                 const uint32_t* hist, uint32_t* state, uint32_t* ticket, uint32_t* err, const EmitSrc& em, cudaStream_t st) {
  static DeviceOnce once;
  once.run([] { cudaFuncSetAttribute(k_radix_pass<kSrc, kWriteKeys>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRadixSmem); });
  k_radix_pass<kSrc, kWriteKeys><<<(unsigned)radix_tiles(n), kRThreads, kRadixSmem, st>>>(ki, vi, ko, vo, n, shift, bits, hist,
                                                                                          state, ticket, err, em);
}

// passes of a tile-id sort: ceil(bits / 8) passes of (almost) equal width
TilePasses tile_passes(int64_t n_tiles) {
  int bits = 1;
  while ((1LL << bits) < n_tiles) ++bits;
  TilePasses tp{};
  tp.n_pass = (bits + 7) / 8;
  int shift = 0;
  for (int p = 0; p < tp.n_pass; ++p) {
    const int b = (bits - shift + (tp.n_pass - p) - 1) / (tp.n_pass - p);
    tp.shift[p] = shift;
    tp.bits[p] = b;
    shift += b;
  }
  return tp;
}

constexpr size_t kScanSmemMax = 200 * 1024;
}  // namespace

// workspace of the depth sort + count scan over n Gaussians
size_t depth_sort_temp_bytes(int64_t n) {
  const size_t tiles = (size_t)radix_tiles(std::max<int64_t>(n, 1));
  const size_t scan_tiles = (size_t)((std::max<int64_t>(n, 1) + 1 + kSTile - 1) / kSTile);
  return sizeof(uint32_t) * (kHdrWords + 4 * 256 + 4 * tiles * 256 + scan_tiles + 1) + 64;
}

// Sorts (dkey, position) by the 32-bit key, stable; the sorted source indices end up in order0 (dkey / dkey_alt and
// order1 are scratch), then offsets[k] = exclusive scan of count[order0[k]], k in [0, n].
int launch_depth_sort_scan(uint32_t* dkey, uint32_t* dkey_alt, uint32_t* order0, uint32_t* order1, const uint32_t* count,
                           uint32_t* offsets, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st) {
  if (n <= 0) {
    cudaMemsetAsync(offsets, 0, sizeof(uint32_t), st);
    return 0;
  }
  const size_t tiles = (size_t)radix_tiles(n);
  cudaMemsetAsync(temp, 0, temp_bytes, st);
  uint32_t* hdr = (uint32_t*)temp;
  uint32_t* hist = hdr + kHdrWords;
  uint32_t* state = hist + 4 * 256;
  uint32_t* scan_state = state + 4 * tiles * 256;
  const int hist_blocks = (int)std::min<int64_t>(148 * 4, (n + 1023) / 1024);
  k_radix_hist<<<hist_blocks, 256, 0, st>>>(dkey, n, hist);
  const EmitSrc none{};
  launch_pass<1, true>(dkey, nullptr, dkey_alt, order1, n, 0, 8, hist, state, hdr + 0, hdr + 16, none, st);
  launch_pass<0, true>(dkey_alt, order1, dkey, order0, n, 8, 8, hist + 256, state + tiles * 256, hdr + 1, hdr + 16, none, st);
  launch_pass<0, true>(dkey, order0, dkey_alt, order1, n, 16, 8, hist + 512, state + 2 * tiles * 256, hdr + 2, hdr + 16, none, st);
  launch_pass<0, false>(dkey_alt, order1, dkey, order0, n, 24, 8, hist + 768, state + 3 * tiles * 256, hdr + 3, hdr + 16, none, st);
  const unsigned scan_blocks = (unsigned)((n + 1 + kSTile - 1) / kSTile);
  k_count_scan<<<scan_blocks, 256, 0, st>>>(count, order0, n, offsets, scan_state, hdr + 4, hdr + 16);
  return 6;  // kernels launched
}

int super_shift() { return kSuperShift; }

// Workspace of launch_tile_counts for a grid of tiles_x x tiles_y tiles: padded slots, compact scratch, histograms.
static size_t tile_slot_bytes(int tiles_x, int tiles_y) {
  return sizeof(int) * kTileStride * (size_t)(tiles_x + 1) * (size_t)(tiles_y + 1);
}
static size_t tile_scratch_bytes(int tiles_x, int tiles_y) { return sizeof(int) * 2 * (size_t)tiles_x * (size_t)tiles_y; }
size_t tile_hist_bytes(int tiles_x, int tiles_y) {
  return tile_slot_bytes(tiles_x, tiles_y) + tile_scratch_bytes(tiles_x, tiles_y) + sizeof(uint32_t) * 4 * 256 + 64;
}
static const uint32_t* tile_ws_hist(const void* ws, int tiles_x, int tiles_y) {
  return (const uint32_t*)((const char*)ws + tile_slot_bytes(tiles_x, tiles_y) + tile_scratch_bytes(tiles_x, tiles_y));
}

// Per-tile list lengths on the grid of 2^shift-tile blocks (shift 0: the tiles themselves) from the tile rectangles
// -> tile_begin / tile_end (0, 0 for an empty tile), the CTA -> tile permutation (longest lists first; optional),
// *total (device) and the digit histograms a sort by tile id needs (kept in tile_ws).
int launch_tile_counts(int64_t n, const ProjDev& p, int shift, int tiles_x, int tiles_y, int wrap_x, void* tile_ws,
                       uint32_t* tile_begin, uint32_t* tile_end, uint32_t* tile_order, int64_t* total, uint32_t* seg_first,
                       cudaStream_t st, bool want_hist) {
  const size_t slot_bytes = tile_slot_bytes(tiles_x, tiles_y);
  cudaMemsetAsync(tile_ws, 0, slot_bytes, st);
  int* slots = (int*)tile_ws;
  int* scratch = (int*)((char*)tile_ws + slot_bytes);
  uint32_t* hist = (uint32_t*)tile_ws_hist(tile_ws, tiles_x, tiles_y);
  int launches = 0;
  if (n > 0) {
    if ((tiles_x + 1) * (tiles_y + 1) <= kHistSmemSlots) {
      const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 4 * (int64_t)device_sm_count());
      k_tile_hist_smem<<<blocks, 256, 0, st>>>(n, p.count, p.rect, shift, tiles_x, tiles_y, wrap_x, slots);
    } else {
      k_tile_hist<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, p.count, p.rect, shift, tiles_x, wrap_x, slots);
    }
    ++launches;
  }
  const size_t smem = tile_scratch_bytes(tiles_x, tiles_y);
  const bool in_smem = smem <= kScanSmemMax;
  static DeviceOnce once;
  once.run([] { cudaFuncSetAttribute(k_tile_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmemMax); });
  if (!want_hist) hist = nullptr;  // the grid is not sorted on (two-level binning sorts blocks, not tiles)
  k_tile_scan<<<1, 1024, in_smem ? smem : 0, st>>>(tiles_x, tiles_y, slots, in_smem ? nullptr : scratch, tile_begin, tile_end, hist,
                                                   tile_passes((int64_t)tiles_x * tiles_y), tile_order, total, seg_first, kSeg);
  return launches + 1;
}

size_t tile_sort_temp_bytes(int64_t cap, int64_t n_tiles) {
  const TilePasses tp = tile_passes(n_tiles);
  size_t words = kHdrWords;
  for (int p = 0; p < tp.n_pass; ++p) words += (size_t)radix_tiles(std::max<int64_t>(cap, 1)) << tp.bits[p];
  return sizeof(uint32_t) * words + 64;
}

// Emits the (tile id, source index) stream in depth order and sorts it by tile id (stable), on the grid of
// 2^shift-tile blocks. Returns which of vals0 / vals1 holds the sorted source indices (0 / 1); *launches receives the
// kernel count. tile_ws: the workspace launch_tile_counts filled for the same grid.
int launch_tile_sort(int64_t n, int64_t total, const uint32_t* offsets, const uint32_t* order, const ProjDev& p, int shift,
                     int tiles_x, int tiles_y, int wrap_x, const void* tile_ws, uint32_t* keys0, uint32_t* keys1, uint32_t* vals0,
                     uint32_t* vals1, void* temp, size_t temp_bytes, int* launches, cudaStream_t st) {
  *launches = 0;
  if (total <= 0) return 0;
  const TilePasses tp = tile_passes((int64_t)tiles_x * tiles_y);
  const uint32_t* hist = tile_ws_hist(tile_ws, tiles_x, tiles_y);
  const size_t tiles = (size_t)radix_tiles(total);
  size_t words = kHdrWords;
  for (int q = 0; q < tp.n_pass; ++q) words += tiles << tp.bits[q];
  cudaMemsetAsync(temp, 0, std::min(temp_bytes, sizeof(uint32_t) * words), st);
  uint32_t* hdr = (uint32_t*)temp;
  uint32_t* state = hdr + kHdrWords;
  EmitSrc em{n, offsets, order, p.rect, tiles_x, wrap_x, shift};
  uint32_t* k[2] = {keys0, keys1};
  uint32_t* v[2] = {vals0, vals1};
  int cur = 0;  // buffer holding the current pass's input (pass 0 has none)
  for (int q = 0; q < tp.n_pass; ++q) {
    const bool last = q == tp.n_pass - 1;
    const uint32_t* h = hist + 256 * q;
    if (q == 0) {
      if (last) launch_pass<2, false>(nullptr, nullptr, k[0], v[0], total, tp.shift[q], tp.bits[q], h, state, hdr + q, hdr + 16, em, st);
      else launch_pass<2, true>(nullptr, nullptr, k[0], v[0], total, tp.shift[q], tp.bits[q], h, state, hdr + q, hdr + 16, em, st);
      cur = 0;
    } else {
      if (last) launch_pass<0, false>(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], total, tp.shift[q], tp.bits[q], h, state, hdr + q, hdr + 16, em, st);
      else launch_pass<0, true>(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], total, tp.shift[q], tp.bits[q], h, state, hdr + q, hdr + 16, em, st);
      cur ^= 1;
    }
    state += tiles << tp.bits[q];
    ++*launches;
  }
  return cur;
}

// Second level of the two-level binning: expands the block lists (cvals, sorted by block) into the tile lists.
// n_coarse: block-level intersections (bounds the number of segments); state: expand_temp_bytes().
size_t expand_temp_bytes(int64_t cap_coarse, int n_super) {
  return sizeof(uint32_t) * (kHdrWords + 64 * (size_t)(cap_coarse / kSeg + n_super + 1));
}
void launch_expand(int stiles_x, int stiles_y, int tiles_x, int tiles_y, int64_t n_coarse, const uint32_t* super_begin,
                   const uint32_t* super_end, const uint32_t* seg_first, const uint32_t* cvals, const ProjDev& p,
                   const uint32_t* tile_begin, void* temp, uint32_t* vals, cudaStream_t st) {
  const int n_super = stiles_x * stiles_y;
  if (n_super <= 0 || n_coarse <= 0) return;
  const int64_t max_segs = n_coarse / kSeg + n_super;
  cudaMemsetAsync(temp, 0, sizeof(uint32_t) * (kHdrWords + 64 * (size_t)max_segs), st);
  uint32_t* hdr = (uint32_t*)temp;
  k_expand<<<(unsigned)max_segs, 256, 0, st>>>(stiles_x, n_super, tiles_x, tiles_y, super_begin, super_end, seg_first, cvals, p.rect,
                                               tile_begin, hdr + kHdrWords, hdr, hdr + 16, vals);
}

}  // namespace sb
