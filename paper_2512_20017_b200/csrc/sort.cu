// Stable LSD radix sort of (key, u32 value) pairs, 8-bit digits.
//
// Used for the Z-order permutation (np.argsort(kind="stable") on Morton
// codes, visibility.py:122), the per-view depth order and the tile
// bucketing of the binning stage.  Three kernels per pass:
//   upsweep   per-tile digit histogram (warp-aggregated smem counters)
//   scan      one CTA per digit: exclusive scan of that digit's tile counts
//   downsweep per-tile stable ranking (__match_any_sync peers, warp-private
//             running counters -> warp prefix), local reorder in smem, then
//             coalesced runs written to the global digit buckets
// The element count may live in device memory (n_dev) so binning never
// needs a host round trip to size the grid.
#include "common.cuh"

namespace bs {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItems = 16;                        // per thread
constexpr int kTile = kSortThreads * kItems;      // 4096 keys per tile
constexpr int kWarpSpan = kTile / kSortWarps;     // 512 keys per warp
constexpr int kRadix = 256;

__device__ __forceinline__ int64_t load_n(const int64_t* n_dev, int64_t n_host) {
  return n_dev ? *n_dev : n_host;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift, uint32_t mask) {
  return static_cast<uint32_t>(k >> shift) & mask;
}

// Block-wide exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t block_exscan_256(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < kSortWarps ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < kSortWarps; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kSortWarps) s_warp[lane] = t;
  }
  __syncthreads();
  const uint32_t warp_prefix = w ? s_warp[w - 1] : 0;
  if (total) *total = s_warp[kSortWarps - 1];
  return warp_prefix + x - v;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) upsweep_kernel(const K* __restrict__ keys, const int64_t* n_dev,
                                                               int64_t n_host, int shift, uint32_t mask,
                                                               uint32_t* __restrict__ hist, int num_tiles) {
  __shared__ uint32_t s_h[kSortWarps][kRadix];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&s_h[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = load_n(n_dev, n_host);
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * kWarpSpan;
#pragma unroll 4
  for (int r = 0; r < kWarpSpan / 32; ++r) {
    const int64_t i = base + r * 32 + lane;
    const uint32_t d = i < n ? digit_of(keys[i], shift, mask) : kRadix;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d < kRadix && (__ffs(peers) - 1) == lane) s_h[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kSortWarps; ++j) sum += s_h[j][tid];
  hist[(size_t)tid * num_tiles + blockIdx.x] = sum;
}

// One CTA per digit: exclusive scan of hist[d][0..num_tiles) in place.
__global__ void __launch_bounds__(1024) scan_digit_kernel(uint32_t* __restrict__ hist, int num_tiles,
                                                          uint32_t* __restrict__ totals) {
  __shared__ uint32_t s_w[32];
  uint32_t* row = hist + (size_t)blockIdx.x * num_tiles;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t carry = 0;
  for (int base = 0; base < num_tiles; base += 1024) {
    const int i = base + tid;
    const uint32_t v = i < num_tiles ? row[i] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t t = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      s_w[lane] = t;
    }
    __syncthreads();
    const uint32_t pre = (w ? s_w[w - 1] : 0) + x - v;
    if (i < num_tiles) row[i] = carry + pre;
    const uint32_t chunk_total = s_w[31];
    __syncthreads();
    carry += chunk_total;
  }
  if (tid == 0) totals[blockIdx.x] = carry;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) downsweep_kernel(const K* __restrict__ keys_in,
                                                                 const uint32_t* __restrict__ vals_in,
                                                                 K* __restrict__ keys_out,
                                                                 uint32_t* __restrict__ vals_out,
                                                                 const int64_t* n_dev, int64_t n_host, int shift,
                                                                 uint32_t mask, const uint32_t* __restrict__ hist,
                                                                 const uint32_t* __restrict__ totals,
                                                                 int num_tiles) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* s_keys = reinterpret_cast<K*>(smem);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kTile);
  __shared__ uint32_t s_wcnt[kSortWarps][kRadix];
  __shared__ uint32_t s_doff[kRadix];
  __shared__ uint32_t s_gbase[kRadix];
  __shared__ uint32_t s_scan[kSortWarps];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t n = load_n(n_dev, n_host);
  const int64_t tile_base = (int64_t)blockIdx.x * kTile;
  if (tile_base >= n) return;
  const int64_t rem = n - tile_base;
  const int tile_n = rem < kTile ? (int)rem : kTile;

  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&s_wcnt[0][0])[i] = 0;
  {
    // global base of every digit for this tile
    const uint32_t dbase = block_exscan_256(totals[tid], s_scan, nullptr);
    s_gbase[tid] = dbase + hist[(size_t)tid * num_tiles + blockIdx.x];
  }
  __syncthreads();

  K k[kItems];
  uint32_t v[kItems], d[kItems], rank[kItems];
  const int64_t wbase = tile_base + (int64_t)w * kWarpSpan;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool ok = i < n;
    k[r] = ok ? keys_in[i] : K(0);
    v[r] = ok ? vals_in[i] : 0u;
    d[r] = ok ? digit_of(k[r], shift, mask) : (uint32_t)kRadix;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[r]);
    uint32_t old = 0;
    if (d[r] < kRadix) old = s_wcnt[w][d[r]];
    rank[r] = old + __popc(peers & lt);
    __syncwarp();
    if (d[r] < kRadix && (__ffs(peers) - 1) == lane) s_wcnt[w][d[r]] = old + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kSortWarps; ++j) {
      const uint32_t t = s_wcnt[j][tid];
      s_wcnt[j][tid] = run;
      run += t;
    }
    const uint32_t doff = block_exscan_256(run, s_scan, nullptr);
    s_doff[tid] = doff;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (d[r] < kRadix) {
      const uint32_t lp = s_doff[d[r]] + s_wcnt[w][d[r]] + rank[r];
      s_keys[lp] = k[r];
      s_vals[lp] = v[r];
    }
  }
  __syncthreads();
  for (int j = tid; j < tile_n; j += kSortThreads) {
    const K kk = s_keys[j];
    const uint32_t dd = digit_of(kk, shift, mask);
    const int64_t out = (int64_t)s_gbase[dd] + (j - (int64_t)s_doff[dd]);
    keys_out[out] = kk;
    vals_out[out] = s_vals[j];
  }
}

template <typename K>
int32_t radix_sort(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n_host,
                   const int64_t* n_dev, int begin_bit, int end_bit, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
  BS_REQUIRE(begin_bit >= 0 && end_bit <= (int)(8 * sizeof(K)) && begin_bit <= end_bit, BS_ERR_PARAMETER,
             "radix sort: bad bit range [%d, %d)", begin_bit, end_bit);
  BS_REQUIRE(n_host >= 0 && n_host < (1ll << 32), BS_ERR_PARAMETER, "radix sort: capacity out of range");
  if (n_host == 0 || begin_bit == end_bit) return BS_OK;
  const int num_tiles = (int)((n_host + kTile - 1) / kTile);
  const size_t need = sizeof(uint32_t) * ((size_t)kRadix * num_tiles + kRadix);
  BS_REQUIRE(ws_bytes >= need, BS_ERR_CAPACITY, "radix sort workspace too small (%zu < %zu)", ws_bytes, need);
  uint32_t* hist = static_cast<uint32_t*>(ws);
  uint32_t* totals = hist + (size_t)kRadix * num_tiles;
  const size_t smem = (sizeof(K) + sizeof(uint32_t)) * kTile;
  cudaFuncSetAttribute(downsweep_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  K* kin = keys;
  uint32_t* vin = vals;
  K* kout = keys_alt;
  uint32_t* vout = vals_alt;
  int passes = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8, ++passes) {
    const int nbits = min(8, end_bit - shift);
    const uint32_t mask = (1u << nbits) - 1u;
    upsweep_kernel<K><<<num_tiles, kSortThreads, 0, s>>>(kin, n_dev, n_host, shift, mask, hist, num_tiles);
    BS_LAUNCH_CHECK("radix upsweep");
    scan_digit_kernel<<<kRadix, 1024, 0, s>>>(hist, num_tiles, totals);
    BS_LAUNCH_CHECK("radix scan");
    downsweep_kernel<K><<<num_tiles, kSortThreads, smem, s>>>(kin, vin, kout, vout, n_dev, n_host, shift, mask,
                                                              hist, totals, num_tiles);
    BS_LAUNCH_CHECK("radix downsweep");
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  if (passes & 1) {
    if (cudaMemcpyAsync(keys, kin, sizeof(K) * n_host, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(vals, vin, sizeof(uint32_t) * n_host, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return set_error(BS_ERR_CUDA, "radix sort: copy-back failed");
  }
  return BS_OK;
}

}  // namespace
}  // namespace bs

extern "C" size_t bs_radix_sort_workspace(int64_t capacity) {
  const int64_t tiles = (capacity + bs::kTile - 1) / bs::kTile;
  return sizeof(uint32_t) * ((size_t)bs::kRadix * (tiles > 0 ? tiles : 1) + bs::kRadix);
}

extern "C" int32_t bs_radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                                     int64_t n_host, const int64_t* n_dev, int32_t begin_bit, int32_t end_bit,
                                     void* ws, size_t ws_bytes, void* stream) {
  return bs::radix_sort<uint64_t>(keys, vals, keys_alt, vals_alt, n_host, n_dev, begin_bit, end_bit, ws, ws_bytes,
                                  bs::as_stream(stream));
}

extern "C" int32_t bs_radix_sort_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                                     int64_t n_host, const int64_t* n_dev, int32_t begin_bit, int32_t end_bit,
                                     void* ws, size_t ws_bytes, void* stream) {
  return bs::radix_sort<uint32_t>(keys, vals, keys_alt, vals_alt, n_host, n_dev, begin_bit, end_bit, ws, ws_bytes,
                                  bs::as_stream(stream));
}
