// K2 tile binning, bucket pipeline ("sorts these
// view-dependent splats by their distance to the camera plane").
//
//  1. bs_bin_tiles_count   per (row, covered tile): atomicAdd on the
//                          (slot, tile) bucket counter
//  2. bs_bin_tiles_offsets one-CTA exclusive scan -> ranges [start, end),
//                          scatter cursors, total and largest bucket
//  3. bs_bin_tiles_scatter per (row, tile): key = (f32bits(depth) << 32) | row
//                          written at an atomically claimed slot of the bucket
//                          (arbitrary order inside the bucket)
//  4. bs_bin_tiles_sort    one CTA per bucket: bitonic sort of the bucket's
//                          keys in shared memory; the row (low 32 bits) of
//                          the sorted keys is the tile list
// Every key is unique (rows are), so the per-tile order -- ascending depth,
// ties by ascending row -- is a total order: deterministic and identical to
// a stable depth sort of the rows followed by a stable tile sort (bin.cu),
// without any full-length radix pass.  Depth > 0 (near plane), so the IEEE
// bits order like the floats.  Buckets larger than the shared-memory
// capacity are left to the caller (radix sort of that slice + bs_keys_low32).
#include "tile.cuh"

namespace bs {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortCap = 4096;  // keys per bucket sorted in shared memory (32 KB)

struct BinGeom {
  const float* sp;
  int64_t n;
  const int64_t* seg_row0;
  const int32_t* seg_slot;
  int n_segs;
  const bs_camera* cams;
  int tiles_per_slot;
};

__global__ void count_tiles_kernel(BinGeom g, int32_t* __restrict__ counts) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < g.n; r += (int64_t)gridDim.x * blockDim.x) {
    const int slot = g.seg_slot[segment_of(g.seg_row0, g.n_segs, r)];
    const int W = g.cams[slot].width, H = g.cams[slot].height;
    int x0, x1, y0, y1;
    if (!tile_rect(g.sp + r * BS_SP_FLOATS, W, H, x0, x1, y0, y1)) continue;
    const int tx = (W + BS_TILE - 1) / BS_TILE;
    int32_t* base = counts + (int64_t)slot * g.tiles_per_slot;
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) atomicAdd(base + y * tx + x, 1);
  }
}

__global__ void __launch_bounds__(1024) offsets_kernel(const int32_t* __restrict__ counts, int nb,
                                                       int2* __restrict__ ranges, int32_t* __restrict__ cursor,
                                                       int64_t* __restrict__ stats) {
  __shared__ int64_t s_w[32];
  __shared__ int s_mx[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // each thread owns a contiguous run of buckets: one block-wide scan total
  const int per = (nb + 1023) / 1024;
  const int b_lo = min(nb, tid * per), b_hi = min(nb, b_lo + per);
  int64_t local = 0;
  int mx = 0;
  for (int i = b_lo; i < b_hi; ++i) {
    const int v = counts[i];
    local += v;
    mx = max(mx, v);
  }
  int64_t x = local;
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
  int64_t start = (w ? s_w[w - 1] : 0) + x - local;
  for (int i = b_lo; i < b_hi; ++i) {
    const int v = counts[i];
    ranges[i] = make_int2((int)start, (int)(start + v));
    cursor[i] = (int)start;
    start += v;
  }
  const int64_t carry = s_w[31];
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_mx[w] = mx;
  __syncthreads();
  if (tid == 0) {
    int m = 0;
    for (int k = 0; k < 32; ++k) m = max(m, s_mx[k]);
    stats[0] = carry;
    stats[1] = m;
  }
}

__global__ void scatter_tiles_kernel(BinGeom g, int32_t* __restrict__ cursor, uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < g.n; r += (int64_t)gridDim.x * blockDim.x) {
    const int slot = g.seg_slot[segment_of(g.seg_row0, g.n_segs, r)];
    const int W = g.cams[slot].width, H = g.cams[slot].height;
    const float* row = g.sp + r * BS_SP_FLOATS;
    int x0, x1, y0, y1;
    if (!tile_rect(row, W, H, x0, x1, y0, y1)) continue;
    const int tx = (W + BS_TILE - 1) / BS_TILE;
    const uint64_t key = ((uint64_t)__float_as_uint(row[9]) << 32) | (uint64_t)(uint32_t)r;
    int32_t* base = cursor + (int64_t)slot * g.tiles_per_slot;
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) keys[atomicAdd(base + y * tx + x, 1)] = key;
  }
}

// Small buckets (n <= kWarpCap): one warp per bucket, bitonic network over
// the padded power of two in warp-private shared memory, every lane owning
// whole compare-exchange pairs (no idle half, only __syncwarp).
constexpr int kWarpCap = 1024;
constexpr int kSortWarpsPerCta = 8;

__global__ void __launch_bounds__(32 * kSortWarpsPerCta) sort_tiles_warp_kernel(const uint64_t* __restrict__ keys,
                                                                                 const int2* __restrict__ ranges,
                                                                                 int nb, int cap,
                                                                                 uint32_t* __restrict__ rows) {
  extern __shared__ uint64_t s_all[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kSortWarpsPerCta + w;
  if (b >= nb) return;
  const int2 rg = ranges[b];
  const int n = rg.y - rg.x;
  if (n <= 0 || n > cap || n > kWarpCap) return;
  if (n == 1) {
    if (lane == 0) rows[rg.x] = (uint32_t)keys[rg.x];
    return;
  }
  uint64_t* s = s_all + w * kWarpCap;
  int m = 2;
  while (m < n) m <<= 1;
  for (int i = lane; i < m; i += 32) s[i] = i < n ? keys[rg.x + i] : ~0ull;
  __syncwarp();
  const int half = m >> 1;
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int p = lane; p < half; p += 32) {
        const int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));  // bit log2(j) of i is 0
        const int ixj = i | j;
        const uint64_t a = s[i], c = s[ixj];
        if ((a > c) == ((i & k) == 0)) {
          s[i] = c;
          s[ixj] = a;
        }
      }
      __syncwarp();
    }
  }
  for (int i = lane; i < n; i += 32) rows[rg.x + i] = (uint32_t)s[i];
}

// Buckets with kWarpCap < n <= cap: one CTA each.
__global__ void __launch_bounds__(kSortThreads) sort_tiles_kernel(const uint64_t* __restrict__ keys,
                                                                  const int2* __restrict__ ranges, int cap,
                                                                  uint32_t* __restrict__ rows) {
  __shared__ uint64_t s[kSortCap];
  const int2 rg = ranges[blockIdx.x];
  const int n = rg.y - rg.x;
  if (n <= kWarpCap || n > cap) return;
  if (n == 1) {
    if (threadIdx.x == 0) rows[rg.x] = (uint32_t)keys[rg.x];
    return;
  }
  int m = 2;
  while (m < n) m <<= 1;
  for (int i = threadIdx.x; i < m; i += kSortThreads) s[i] = i < n ? keys[rg.x + i] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += kSortThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s[i], b = s[ixj];
          if (((i & k) == 0) ? (a > b) : (a < b)) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += kSortThreads) rows[rg.x + i] = (uint32_t)s[i];
}

__global__ void low32_kernel(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)keys[i];
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_bin_tiles_count(const float* sp_rows, int64_t n_rows, const int64_t* seg_row0,
                                      const int32_t* seg_slot, int32_t n_segs, const bs_camera* slot_cams,
                                      int32_t tiles_per_slot, int32_t n_buckets, int32_t* bucket_counts,
                                      void* stream) {
  BS_REQUIRE(n_segs >= 1 && n_buckets >= 1, BS_ERR_PARAMETER, "bin: bad segment/bucket counts");
  BS_REQUIRE(n_rows < (1ll << 32), BS_ERR_PARAMETER, "bin: too many rows for 32-bit row ids");
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(bucket_counts, 0, sizeof(int32_t) * (size_t)n_buckets, s) != cudaSuccess)
    return set_error(BS_ERR_CUDA, "bin: memset failed");
  if (n_rows == 0) return BS_OK;
  BinGeom g{sp_rows, n_rows, seg_row0, seg_slot, n_segs, slot_cams, tiles_per_slot};
  count_tiles_kernel<<<grid_for(n_rows, 256), 256, 0, s>>>(g, bucket_counts);
  BS_LAUNCH_CHECK("count_tiles_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_offsets(const int32_t* bucket_counts, int32_t n_buckets, int32_t* ranges,
                                        int32_t* cursor, int64_t* stats, void* stream) {
  BS_REQUIRE(n_buckets >= 1, BS_ERR_PARAMETER, "bin: bad bucket count");
  offsets_kernel<<<1, 1024, 0, as_stream(stream)>>>(bucket_counts, n_buckets, reinterpret_cast<int2*>(ranges),
                                                    cursor, stats);
  BS_LAUNCH_CHECK("offsets_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_scatter(const float* sp_rows, int64_t n_rows, const int64_t* seg_row0,
                                        const int32_t* seg_slot, int32_t n_segs, const bs_camera* slot_cams,
                                        int32_t tiles_per_slot, int32_t* cursor, uint64_t* inst_keys,
                                        void* stream) {
  BS_REQUIRE(n_segs >= 1, BS_ERR_PARAMETER, "bin: need at least one segment");
  if (n_rows == 0) return BS_OK;
  BinGeom g{sp_rows, n_rows, seg_row0, seg_slot, n_segs, slot_cams, tiles_per_slot};
  scatter_tiles_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(g, cursor, inst_keys);
  BS_LAUNCH_CHECK("scatter_tiles_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_sort(const uint64_t* inst_keys, const int32_t* ranges, int32_t n_buckets,
                                     int32_t smem_cap, uint32_t* inst_rows, void* stream) {
  BS_REQUIRE(smem_cap >= 1 && smem_cap <= kSortCap, BS_ERR_PARAMETER, "bin: smem_cap must be in [1, %d]",
             kSortCap);
  if (n_buckets == 0) return BS_OK;
  cudaStream_t s = as_stream(stream);
  const size_t wsmem = sizeof(uint64_t) * kWarpCap * kSortWarpsPerCta;
  cudaFuncSetAttribute(sort_tiles_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem);
  sort_tiles_warp_kernel<<<(n_buckets + kSortWarpsPerCta - 1) / kSortWarpsPerCta, 32 * kSortWarpsPerCta, wsmem, s>>>(
      inst_keys, reinterpret_cast<const int2*>(ranges), n_buckets, smem_cap, inst_rows);
  BS_LAUNCH_CHECK("sort_tiles_warp_kernel");
  if (smem_cap > kWarpCap) {
    sort_tiles_kernel<<<n_buckets, kSortThreads, 0, s>>>(inst_keys, reinterpret_cast<const int2*>(ranges), smem_cap,
                                                         inst_rows);
    BS_LAUNCH_CHECK("sort_tiles_kernel");
  }
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_max_sort(void) { return kSortCap; }

extern "C" int32_t bs_keys_low32(const uint64_t* keys, int64_t n, uint32_t* out, void* stream) {
  if (n == 0) return BS_OK;
  low32_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(keys, n, out);
  BS_LAUNCH_CHECK("low32_kernel");
  return BS_OK;
}
