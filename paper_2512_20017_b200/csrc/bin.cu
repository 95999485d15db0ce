// K2 tile binning ("sorts these view-dependent splats by their
// distance to the camera plane").
//
//  1. bs_bin_depth_keys : key = (slot << 32) | f32bits(depth), value = row.
//     depth > 0 (near plane) so the IEEE bits order like the floats.
//  2. (caller) stable radix sort of those keys -> per-slot depth order, ties
//     in input row order (ascending point index within a source shard).
//  3. bs_bin_count      : tiles per splat in that order + inclusive scan.
//  4. bs_bin_emit       : (slot*tiles + tile, row) instances in depth order.
//  5. (caller) stable radix sort on the bucket id -> per-tile lists that
//     stay depth-sorted (stability), i.e. exactly the order of a stable sort
//     on the 64-bit key ((slot, tile) << 32 | depth).
//  6. bs_tile_ranges    : [start, end) of every bucket.
//
// Tile rectangles: tile.cuh.  The training step uses the bucket + per-tile
// sort pipeline of bin_tiles.cu; this radix-sort pipeline is kept as an
// alternative ABI (and cross-check) producing the identical lists.
#include "tile.cuh"

namespace bs {
namespace {

__global__ void depth_keys_kernel(const float* __restrict__ sp, int64_t n, const int64_t* __restrict__ seg_row0,
                                  const int32_t* __restrict__ seg_slot, int n_segs, uint64_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    // segment of row r: last s with seg_row0[s] <= r
    int lo = 0, hi = n_segs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg_row0[mid] <= r) lo = mid;
      else hi = mid - 1;
    }
    const uint32_t slot = (uint32_t)seg_slot[lo];
    const float depth = sp[r * BS_SP_FLOATS + 9];
    keys[r] = ((uint64_t)slot << 32) | (uint64_t)__float_as_uint(depth);
    vals[r] = (uint32_t)r;
  }
}

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_inclusive_scan(int64_t v, int64_t* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_w[lane] = t;
  }
  __syncthreads();
  const int64_t r = (w ? s_w[w - 1] : 0) + x;
  return r;
}

// Pass 1: tiles per sorted splat; per-block totals.
__global__ void __launch_bounds__(kScanThreads) count_kernel(const float* __restrict__ sp,
                                                             const uint32_t* __restrict__ rows, int64_t n,
                                                             const uint64_t* __restrict__ skeys,
                                                             const bs_camera* __restrict__ cams,
                                                             int64_t* __restrict__ offsets,
                                                             int64_t* __restrict__ block_sums) {
  __shared__ int64_t s_w[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t c[kScanItems];
  int64_t local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    c[k] = 0;
    if (i < n) {
      const int slot = (int)(skeys[i] >> 32);
      int x0, x1, y0, y1;
      c[k] = tile_rect(sp + (int64_t)rows[i] * BS_SP_FLOATS, cams[slot].width, cams[slot].height, x0, x1, y0, y1);
    }
    local += c[k];
  }
  const int64_t incl = block_inclusive_scan(local, s_w);
  int64_t run = incl - local;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    run += c[k];
    if (base + k < n) offsets[base + k] = run;
  }
  if (threadIdx.x == kScanThreads - 1) block_sums[blockIdx.x] = incl;
}

// Pass 2: exclusive scan of block sums (single CTA) + total.
__global__ void __launch_bounds__(kScanThreads) block_sums_kernel(int64_t* __restrict__ block_sums, int nb,
                                                                  int64_t* __restrict__ total) {
  __shared__ int64_t s_w[32];
  int64_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int i = b0 + threadIdx.x;
    const int64_t v = i < nb ? block_sums[i] : 0;
    const int64_t incl = block_inclusive_scan(v, s_w);
    if (i < nb) block_sums[i] = carry + incl - v;
    const int64_t tot = s_w[31];
    __syncthreads();
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// Pass 3: add block offsets.
__global__ void add_offsets_kernel(int64_t* __restrict__ offsets, int64_t n, const int64_t* __restrict__ block_sums) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) offsets[i] += block_sums[i / kScanTile];
}

__global__ void emit_kernel(const float* __restrict__ sp, const uint32_t* __restrict__ rows, int64_t n,
                            const uint64_t* __restrict__ skeys, const bs_camera* __restrict__ cams,
                            int tiles_per_slot, const int64_t* __restrict__ offsets, uint32_t* __restrict__ ikeys,
                            uint32_t* __restrict__ irows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(skeys[i] >> 32);
    const uint32_t row = rows[i];
    const int W = cams[slot].width, H = cams[slot].height;
    int x0, x1, y0, y1;
    const int cnt = tile_rect(sp + (int64_t)row * BS_SP_FLOATS, W, H, x0, x1, y0, y1);
    if (cnt == 0) continue;
    const int tx = (W + BS_TILE - 1) / BS_TILE;
    int64_t o = offsets[i] - cnt;
    const uint32_t sbase = (uint32_t)slot * (uint32_t)tiles_per_slot;
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) {
        ikeys[o] = sbase + (uint32_t)(y * tx + x);
        irows[o] = row;
        ++o;
      }
  }
}

__global__ void ranges_kernel(const uint32_t* __restrict__ keys, const int64_t* n_dev, int64_t n_host,
                              int2* __restrict__ ranges) {
  const int64_t n = n_dev ? *n_dev : n_host;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) ranges[k].x = (int)i;
    if (i == n - 1 || keys[i + 1] != k) ranges[k].y = (int)(i + 1);
  }
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_bin_depth_keys(const float* sp_rows, int64_t n_rows, const int64_t* seg_row0,
                                     const int32_t* seg_slot, int32_t n_segs, uint64_t* keys, uint32_t* vals,
                                     void* stream) {
  BS_REQUIRE(n_segs >= 1, BS_ERR_PARAMETER, "bin: need at least one segment");
  if (n_rows == 0) return BS_OK;
  depth_keys_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(sp_rows, n_rows, seg_row0, seg_slot,
                                                                          n_segs, keys, vals);
  BS_LAUNCH_CHECK("depth_keys_kernel");
  return BS_OK;
}

extern "C" size_t bs_bin_count_workspace(int64_t n_rows) {
  return sizeof(int64_t) * (size_t)((n_rows + kScanTile - 1) / kScanTile + 1);
}

extern "C" int32_t bs_bin_count(const float* sp_rows, const uint32_t* sorted_rows, int64_t n_rows,
                                const uint64_t* sorted_keys, const bs_camera* slot_cams, int64_t* offsets,
                                int64_t* total_dev, void* ws, size_t ws_bytes, void* stream) {
  BS_REQUIRE(ws_bytes >= bs_bin_count_workspace(n_rows), BS_ERR_CAPACITY, "bin_count workspace too small");
  cudaStream_t s = as_stream(stream);
  if (n_rows == 0) {
    cudaMemsetAsync(total_dev, 0, sizeof(int64_t), s);
    return BS_OK;
  }
  const int nb = (int)((n_rows + kScanTile - 1) / kScanTile);
  int64_t* bsums = static_cast<int64_t*>(ws);
  count_kernel<<<nb, kScanThreads, 0, s>>>(sp_rows, sorted_rows, n_rows, sorted_keys, slot_cams, offsets, bsums);
  BS_LAUNCH_CHECK("bin count_kernel");
  block_sums_kernel<<<1, kScanThreads, 0, s>>>(bsums, nb, total_dev);
  BS_LAUNCH_CHECK("bin block_sums_kernel");
  add_offsets_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(offsets, n_rows, bsums);
  BS_LAUNCH_CHECK("bin add_offsets_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_emit(const float* sp_rows, const uint32_t* sorted_rows, int64_t n_rows,
                               const uint64_t* sorted_keys, const bs_camera* slot_cams, int32_t tiles_per_slot,
                               const int64_t* offsets, uint32_t* inst_keys, uint32_t* inst_rows, void* stream) {
  if (n_rows == 0) return BS_OK;
  emit_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(sp_rows, sorted_rows, n_rows, sorted_keys,
                                                                    slot_cams, tiles_per_slot, offsets, inst_keys,
                                                                    inst_rows);
  BS_LAUNCH_CHECK("bin emit_kernel");
  return BS_OK;
}

extern "C" int32_t bs_tile_ranges(const uint32_t* inst_keys, const int64_t* n_dev, int64_t n_host,
                                  int32_t n_buckets, int32_t* ranges, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(ranges, 0, sizeof(int32_t) * 2 * (size_t)n_buckets, s) != cudaSuccess)
    return set_error(BS_ERR_CUDA, "tile_ranges memset failed");
  if (n_host == 0) return BS_OK;
  ranges_kernel<<<grid_for(n_host, 256), 256, 0, s>>>(inst_keys, n_dev, n_host, reinterpret_cast<int2*>(ranges));
  BS_LAUNCH_CHECK("ranges_kernel");
  return BS_OK;
}
