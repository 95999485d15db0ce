// K2 tile binning, bucket pipeline ("sorts these
// view-dependent splats by their distance to the camera plane").
//
//  1. bs_bin_tiles_count   per (row, covered tile): atomicAdd on the
//                          (slot, tile) bucket counter, warp-aggregated
//  2. bs_bin_tiles_offsets one-CTA exclusive scan -> ranges [start, end),
//                          scatter cursors, total and largest bucket
//  3. bs_bin_tiles_scatter per (row, tile): key = (f32bits(depth) << 32) | row
//                          written at an atomically claimed slot of the bucket
//                          (arbitrary order inside the bucket)
//  4. bs_bin_tiles_sort    by bucket size: one warp per bucket with a
//                          register bitonic network (<= 256 keys) or a
//                          register + shared-memory merge sort (257..1024,
//                          the common classes), one CTA per larger bucket;
//                          the row (low 32 bits) of the sorted keys is the
//                          tile list
// Every key is unique (rows are), so the per-tile order -- ascending depth,
// ties by ascending row -- is a total order: deterministic and identical to
// a stable depth sort of the rows followed by a stable tile sort (bin.cu),
// without any full-length radix pass.  Depth > 0 (near plane), so the IEEE
// bits order like the floats.  Buckets larger than the shared-memory
// capacity are left to the caller (radix sort of that slice + bs_keys_low32).
#include "tile.cuh"

namespace bs {
namespace {

constexpr int kSortThreads = 1024;
constexpr int kSortCap = 16384;  // keys per bucket sorted in shared memory (128 KB, dynamic)

struct BinGeom {
  const float* sp;
  int64_t n;
  const int64_t* seg_row0;
  const int32_t* seg_slot;
  int n_segs;
  const bs_camera* cams;
  int tiles_per_slot;
  SpLayout lay;
};

// Rows of a warp are consecutive points of one Z-ordered shard, so their
// tiles coincide often: every round each lane takes its next covered tile,
// lanes with equal buckets are grouped with __match_any_sync and only the
// group leader touches the counter (warp-aggregated atomics).
struct RowTiles {
  int slot, x0, x1, y1, tx, x, y;
  bool left;  // tiles remain
  __device__ __forceinline__ void init(const BinGeom& g, int64_t r) {
    left = false;
    if (r >= g.n) return;
    slot = g.seg_slot[segment_of(g.seg_row0, g.n_segs, r)];
    const int W = g.cams[slot].width, H = g.cams[slot].height;
    int y0;
    if (!tile_rect_at(g.sp + r * g.lay.stride, g.lay.rad_off, g.lay.ctr_off, W, H, x0, x1, y0, y1)) return;
    tx = (W + BS_TILE - 1) / BS_TILE;
    x = x0;
    y = y0;
    left = true;
  }
  // bucket of the current tile (or -1), then advance
  __device__ __forceinline__ int next(int tiles_per_slot) {
    if (!left) return -1;
    const int b = slot * tiles_per_slot + y * tx + x;
    if (++x == x1) {
      x = x0;
      left = ++y < y1;
    }
    return b;
  }
};

__global__ void count_tiles_kernel(BinGeom g, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; r0 < g.n; r0 += stride) {
    RowTiles t;
    t.init(g, r0 + lane);
    while (__any_sync(0xffffffffu, t.left)) {
      const int b = t.next(g.tiles_per_slot);
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      if (b >= 0 && lane == __ffs(peers) - 1) atomicAdd(counts + b, __popc(peers));
    }
  }
}

// Bucket offsets: 3-phase scan (per-block sums, scan of the block sums,
// block-local scan + offset), every access coalesced.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ int64_t block_exscan(int64_t v, int64_t* s_w, int64_t* total) {
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
    int64_t t = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_w[lane] = t;
  }
  __syncthreads();
  if (total) *total = s_w[(blockDim.x >> 5) - 1];
  return (w ? s_w[w - 1] : 0) + x - v;
}

__global__ void __launch_bounds__(kScanBlock) bucket_sums_kernel(const int32_t* __restrict__ counts, int nb,
                                                                  int64_t* __restrict__ part, int* __restrict__ pmax) {
  __shared__ int64_t s_w[32];
  __shared__ int s_m[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int v = i < nb ? counts[i] : 0;
  int64_t tot;
  block_exscan(v, s_w, &tot);
  int m = v;
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 32; ++k) m = max(m, s_m[k]);
    part[blockIdx.x] = tot;
    pmax[blockIdx.x] = max(m, s_m[0]);
  }
}

__global__ void __launch_bounds__(kScanBlock) bucket_parts_kernel(int64_t* __restrict__ part,
                                                                   const int* __restrict__ pmax, int np,
                                                                   int64_t* __restrict__ stats) {
  __shared__ int64_t s_w[32];
  __shared__ int s_m[32];
  int64_t carry = 0;
  int m = 0;
  for (int b0 = 0; b0 < np; b0 += kScanBlock) {
    const int i = b0 + threadIdx.x;
    const int64_t v = i < np ? part[i] : 0;
    if (i < np) m = max(m, pmax[i]);
    int64_t tot;
    const int64_t ex = block_exscan(v, s_w, &tot);
    if (i < np) part[i] = carry + ex;
    __syncthreads();
    carry += tot;
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 32; ++k) m = max(m, s_m[k]);
    stats[0] = carry;
    stats[1] = m;
  }
}

__global__ void __launch_bounds__(kScanBlock) bucket_ranges_kernel(const int32_t* __restrict__ counts, int nb,
                                                                    const int64_t* __restrict__ part,
                                                                    int2* __restrict__ ranges,
                                                                    int32_t* __restrict__ cursor) {
  __shared__ int64_t s_w[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int v = i < nb ? counts[i] : 0;
  const int64_t start = part[blockIdx.x] + block_exscan(v, s_w, nullptr);
  if (i < nb) {
    ranges[i] = make_int2((int)start, (int)(start + v));
    cursor[i] = (int)start;
  }
}

// Up to kScatterU tiles of every lane per round: the rounds' buckets are
// grouped (match_any) and their leaders' returning atomics are all issued
// before the first position is needed, so kScatterU atomic round trips
// overlap instead of one per tile.
#ifndef BS_SCATTER_UNROLL
#define BS_SCATTER_UNROLL 4  // A/B on B200 (C4 bin stage): 1 2.24, 2 2.25, 4 2.19, 8 2.25 ms
#endif
constexpr int kScatterU = BS_SCATTER_UNROLL;

template <class Next>
__device__ __forceinline__ void scatter_rounds(Next next, bool& left, uint64_t key, int32_t* __restrict__ cursor,
                                               uint64_t* __restrict__ keys, int64_t capacity) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  while (__any_sync(0xffffffffu, left)) {
    int b[kScatterU], pos[kScatterU], leader[kScatterU];
    uint32_t peers[kScatterU];
#pragma unroll
    for (int u = 0; u < kScatterU; ++u) b[u] = next();
#pragma unroll
    for (int u = 0; u < kScatterU; ++u) {
      peers[u] = __match_any_sync(0xffffffffu, b[u]);
      leader[u] = __ffs(peers[u]) - 1;
      pos[u] = 0;
      if (b[u] >= 0 && lane == leader[u]) pos[u] = atomicAdd(cursor + b[u], __popc(peers[u]));
    }
#pragma unroll
    for (int u = 0; u < kScatterU; ++u) {
      const int64_t at = (int64_t)__shfl_sync(0xffffffffu, pos[u], leader[u]) + __popc(peers[u] & lt);
      if (b[u] >= 0 && at < capacity) keys[at] = key;
    }
  }
}

// Positions at or beyond `capacity` are dropped: the caller sizes the key
// buffer before it has read the instance count and re-runs on overflow.
__global__ void scatter_tiles_kernel(BinGeom g, int32_t* __restrict__ cursor, uint64_t* __restrict__ keys,
                                     int64_t capacity) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; r0 < g.n; r0 += stride) {
    const int64_t r = r0 + lane;
    RowTiles t;
    t.init(g, r);
    const uint64_t key =
        t.left ? ((uint64_t)__float_as_uint(g.sp[r * g.lay.stride + g.lay.depth_off]) << 32) | (uint64_t)(uint32_t)r
               : 0ull;
    scatter_rounds([&]() { return t.next(g.tiles_per_slot); }, t.left, key, cursor, keys, capacity);
  }
}

// Single-pass variant: rectangle and depth bits from the projection's row
// records (int4 per row) -- 16 B per row instead of the splat row.
#ifndef BS_SCATTER_LDCS
#define BS_SCATTER_LDCS 1  // records read evict-first (C2 bin 0.229 -> 0.226 ms; profiles/r2z_ab_scatter_ldcs.txt)
#endif
__global__ void scatter_rec_kernel(const int4* __restrict__ rec, int64_t n, const int64_t* __restrict__ seg_row0,
                                   const int32_t* __restrict__ seg_slot, int n_segs, const bs_camera* __restrict__ cams,
                                   int tiles_per_slot, int32_t* __restrict__ cursor, uint64_t* __restrict__ keys,
                                   int64_t capacity) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; r0 < n; r0 += stride) {
    const int64_t r = r0 + lane;
    int x0 = 0, x1 = 0, y = 0, y1 = 0, x = 0, tx = 1;
    int64_t bucket0 = 0;
    uint64_t key = 0ull;
    bool left = false;
    if (r < n) {
#if BS_SCATTER_LDCS
      const int4 q = __ldcs(rec + r);  // the record's only read
#else
      const int4 q = rec[r];
#endif
      x0 = q.y & 0xffff;
      x1 = (int)((uint32_t)q.y >> 16);
      y = q.z & 0xffff;
      y1 = (int)((uint32_t)q.z >> 16);
      left = x1 > x0 && y1 > y;
      const int slot = seg_slot[segment_of(seg_row0, n_segs, r)];
      tx = (cams[slot].width + BS_TILE - 1) / BS_TILE;
      bucket0 = (int64_t)slot * tiles_per_slot;
      key = ((uint64_t)(uint32_t)q.x << 32) | (uint64_t)(uint32_t)r;
      x = x0;
    }
    scatter_rounds(
        [&]() {
          int b = -1;
          if (left) {
            b = (int)(bucket0 + (int64_t)y * tx + x);
            if (++x == x1) {
              x = x0;
              left = ++y < y1;
            }
          }
          return b;
        },
        left, key, cursor, keys, capacity);
  }
}

// Small buckets (n <= kWarpCap): one warp per bucket, bitonic network held
// entirely in registers.  Lane l owns elements [l*E, l*E + E) of the padded
// power of two M = 32*E; partners closer than E are exchanged inside the
// lane, farther ones with __shfl_xor (same register slot, lane ^ j/E).  The
// network is fully unrolled per E, so there is no shared memory traffic and
// no dependent-load chain.
constexpr int kWarpCap = 1024;
constexpr int kSortWarpsPerCta = 8;
#ifndef BS_SORT_BITONIC256
#define BS_SORT_BITONIC256 1  // measured: 10 us faster on C2 than the E = 8 merge sort
#endif
constexpr bool kBitonic256 = BS_SORT_BITONIC256;
#ifndef BS_SORT_MERGE1024
#define BS_SORT_MERGE1024 1
#endif
constexpr bool kMerge1024 = BS_SORT_MERGE1024;  // 513..1024 keys: merge sort instead of the bitonic network  // 129..256 keys: bitonic network instead of merge sort

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

template <int E>
__device__ __forceinline__ void warp_bitonic(uint64_t (&x)[E], int lane) {
  constexpr int M = 32 * E;
#pragma unroll
  for (int k = 2; k <= M; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lj = j / E;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const bool asc = ((lane * E + e) & k) == 0;
          const uint64_t o = shfl_xor_u64(x[e], lj);
          const bool take_min = lower == asc;
          x[e] = (take_min == (o < x[e])) ? o : x[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & j) == 0) {
            const bool asc = ((lane * E + e) & k) == 0;
            const uint64_t a = x[e], b = x[e | j];
            const bool sw = asc ? (a > b) : (a < b);
            x[e] = sw ? b : a;
            x[e | j] = sw ? a : b;
          }
        }
      }
    }
  }
}

#ifndef BS_SORT_LDCS
#define BS_SORT_LDCS 1  // C2 bin 0.2255 -> 0.2236 ms, C3 0.547 -> 0.541 ms (profiles/r2z_ab_sort_ldcs.txt)
#endif
// A bucket sort reads each instance key once (its last use): evict-first
// when BS_SORT_LDCS, so the sorted row lists the raster reads next keep L2.
__device__ __forceinline__ uint64_t sort_key_load(const uint64_t* p) {
#if BS_SORT_LDCS
  return __ldcs(reinterpret_cast<const unsigned long long*>(p));
#else
  return __ldg(p);
#endif
}

template <int E>
__device__ __forceinline__ void sort_bucket_regs(const uint64_t* __restrict__ keys, int start, int n,
                                                 uint32_t* __restrict__ rows, int lane) {
  uint64_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    x[e] = i < n ? sort_key_load(keys + start + i) : ~0ull;
  }
  warp_bitonic<E>(x, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    if (i < n) rows[start + i] = (uint32_t)x[e];
  }
}

// Buckets of 129..1024 keys (the common classes): one warp per bucket, merge
// sort instead of a bitonic network (45 steps over 16 keys per lane for 512).
// Each lane sorts its E keys in registers (in-lane bitonic network), then
// log2(32) = 5 rounds merge runs of E, 2E, ..., 16E through warp-private
// shared memory: lane l produces merged outputs [E l, E l + E) of its pair
// of runs -- the split point by a merge-path binary search, then E
// sequential merge steps.  Padding keys are ~0 (sort last; every real key is
// unique).  Loads and the row stores go through the same buffer so global
// accesses stay coalesced.
__device__ __forceinline__ int mpad(int i) { return i + (i >> 4); }  // one pad word per 16: bank skew

__device__ __forceinline__ void cas64(uint64_t& a, uint64_t& b) {
  const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}

template <int E>
__device__ __forceinline__ void warp_merge_sort(const uint64_t* __restrict__ keys, int start, int n,
                                                uint32_t* __restrict__ rows, uint64_t* sm, int lane) {
  constexpr int M = 32 * E;
  for (int i = lane; i < M; i += 32) sm[mpad(i)] = i < n ? sort_key_load(keys + start + i) : ~0ull;
  __syncwarp();
  uint64_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = sm[mpad(lane * E + e)];
#pragma unroll
  for (int k = 2; k <= E; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int p = e ^ j;
        if (p > e) {
          if ((e & k) == 0) cas64(x[e], x[p]);
          else cas64(x[p], x[e]);
        }
      }
#pragma unroll 1
  for (int L = E; L < M; L <<= 1) {
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) sm[mpad(lane * E + e)] = x[e];
    __syncwarp();
    const int d0 = lane * E;
    const int base = d0 & ~(2 * L - 1);
    const int d = d0 - base;  // outputs of this pair before this lane's first
    const int a0 = base, b0 = base + L;
    int lo = max(0, d - L), hi = min(d, L);
    while (lo < hi) {  // merge path: A elements among the first d outputs
      const int mid = (lo + hi) >> 1;
      if (sm[mpad(a0 + mid)] <= sm[mpad(b0 + d - 1 - mid)]) lo = mid + 1;
      else hi = mid;
    }
    int i = lo, j = d - lo;
    uint64_t a = i < L ? sm[mpad(a0 + i)] : ~0ull;
    uint64_t b = j < L ? sm[mpad(b0 + j)] : ~0ull;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool take_a = j >= L || (i < L && a <= b);
      x[e] = take_a ? a : b;
      if (take_a) {
        ++i;
        a = i < L ? sm[mpad(a0 + i)] : ~0ull;
      } else {
        ++j;
        b = j < L ? sm[mpad(b0 + j)] : ~0ull;
      }
    }
  }
  __syncwarp();
  uint32_t* sr = reinterpret_cast<uint32_t*>(sm);
#pragma unroll
  for (int e = 0; e < E; ++e) sr[mpad(lane * E + e)] = (uint32_t)x[e];
  __syncwarp();
  for (int i = lane; i < n; i += 32) rows[start + i] = sr[mpad(i)];
}

// Size class (16 E, 32 E] -- E = 8: 129..256, 16: 257..512, 32: 513..1024.
template <int E, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) sort_tiles_merge_kernel(const uint64_t* __restrict__ keys,
                                                                       const int2* __restrict__ ranges, int nb,
                                                                       int cap, uint32_t* __restrict__ rows) {
  constexpr int kWords = 32 * E + 2 * E;  // mpad(32 E - 1) + 1
  __shared__ uint64_t s_buf[WARPS][kWords];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * WARPS + w;
  if (b >= nb) return;
  const int2 rg = ranges[b];
  const int n = rg.y - rg.x;
  if (n <= 16 * E || n > 32 * E || n > cap) return;
  warp_merge_sort<E>(keys, rg.x, n, rows, s_buf[w], lane);
}

// One launch per size class (n <= 256, <= 512, <= 1024) so that each class
// is compiled with the registers of its own largest network (the 1024-key
// network needs 64 key registers per lane; the common 257..512 class half of
// that), instead of the whole kernel paying for the largest one.
template <int EMAX>
__global__ void __launch_bounds__(32 * kSortWarpsPerCta, EMAX >= 32 ? 1 : 4) sort_tiles_warp_kernel(const uint64_t* __restrict__ keys,
                                                                                 const int2* __restrict__ ranges,
                                                                                 int nb, int cap,
                                                                                 uint32_t* __restrict__ rows) {
  constexpr int kLo = EMAX <= 8 ? 0 : 16 * EMAX;  // exclusive lower bound of the class
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kSortWarpsPerCta + w;
  if (b >= nb) return;
  const int2 rg = ranges[b];
  const int n = rg.y - rg.x;
  if (n <= kLo || n > 32 * EMAX || n > cap) return;
  if constexpr (EMAX <= 8) {
    if (n <= 0) return;
    if (n == 1) {
      if (lane == 0) rows[rg.x] = (uint32_t)keys[rg.x];
      return;
    }
    if (n <= 32) sort_bucket_regs<1>(keys, rg.x, n, rows, lane);
    else if (n <= 64) sort_bucket_regs<2>(keys, rg.x, n, rows, lane);
    else if (n <= 128) sort_bucket_regs<4>(keys, rg.x, n, rows, lane);
    else if constexpr (EMAX >= 8) sort_bucket_regs<8>(keys, rg.x, n, rows, lane);
  } else {
    sort_bucket_regs<EMAX>(keys, rg.x, n, rows, lane);
  }
}

// Buckets with kWarpCap < n <= cap: one CTA each.
// Buckets with kWarpCap < n <= cap: a persistent grid (one 1024-thread CTA
// per SM, 128 KB of shared memory) scans the bucket table 1024 entries at a
// time, collects the large buckets of each slice and bitonic-sorts them one
// after the other with the whole CTA -- no CTA per bucket (most buckets are
// small and a launch over all of them costs more than the sorting).
__global__ void __launch_bounds__(kSortThreads) sort_tiles_kernel(const uint64_t* __restrict__ keys,
                                                                  const int2* __restrict__ ranges, int nb, int cap,
                                                                  uint32_t* __restrict__ rows) {
  extern __shared__ uint64_t s[];  // [cap rounded up to a power of two]
  __shared__ int s_list[kSortThreads];
  __shared__ int s_n;
  for (int base = blockIdx.x * kSortThreads; base < nb; base += gridDim.x * kSortThreads) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int b = base + threadIdx.x;
    if (b < nb) {
      const int2 rg = ranges[b];
      const int n = rg.y - rg.x;
      if (n > kWarpCap && n <= cap) s_list[atomicAdd(&s_n, 1)] = b;
    }
    __syncthreads();
    const int n_big = s_n;
    for (int t = 0; t < n_big; ++t) {
      const int2 rg = ranges[s_list[t]];
      const int n = rg.y - rg.x;
      int m = 2;
      while (m < n) m <<= 1;
      for (int i = threadIdx.x; i < m; i += kSortThreads) s[i] = i < n ? keys[rg.x + i] : ~0ull;
      __syncthreads();
      for (int k = 2; k <= m; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = threadIdx.x; i < m; i += kSortThreads) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const uint64_t a = s[i], c = s[ixj];
              if (((i & k) == 0) ? (a > c) : (a < c)) {
                s[i] = c;
                s[ixj] = a;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < n; i += kSortThreads) rows[rg.x + i] = (uint32_t)s[i];
      __syncthreads();
    }
  }
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
                                      int32_t model, void* stream) {
  BS_REQUIRE(n_segs >= 1 && n_buckets >= 1, BS_ERR_PARAMETER, "bin: bad segment/bucket counts");
  BS_REQUIRE(n_rows < (1ll << 32), BS_ERR_PARAMETER, "bin: too many rows for 32-bit row ids");
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(bucket_counts, 0, sizeof(int32_t) * (size_t)n_buckets, s) != cudaSuccess)
    return set_error(BS_ERR_CUDA, "bin: memset failed");
  if (n_rows == 0) return BS_OK;
  BinGeom g{sp_rows, n_rows, seg_row0, seg_slot, n_segs, slot_cams, tiles_per_slot, sp_layout(model)};
  count_tiles_kernel<<<grid_for(n_rows, 256), 256, 0, s>>>(g, bucket_counts);
  BS_LAUNCH_CHECK("count_tiles_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_scatter_rec(const int32_t* row_bin, int64_t n_rows, const int64_t* seg_row0,
                                            const int32_t* seg_slot, int32_t n_segs, const bs_camera* slot_cams,
                                            int32_t tiles_per_slot, int32_t* cursor, uint64_t* inst_keys,
                                            int64_t capacity, void* stream) {
  BS_REQUIRE(n_segs >= 1, BS_ERR_PARAMETER, "bin: need at least one segment");
  BS_REQUIRE(n_rows < (1ll << 32), BS_ERR_PARAMETER, "bin: too many rows for 32-bit row ids");
  if (n_rows == 0) return BS_OK;
  scatter_rec_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const int4*>(row_bin), n_rows, seg_row0, seg_slot, n_segs, slot_cams, tiles_per_slot, cursor,
      inst_keys, capacity);
  BS_LAUNCH_CHECK("scatter_rec_kernel");
  return BS_OK;
}

extern "C" size_t bs_bin_tiles_offsets_workspace(int32_t n_buckets) {
  const size_t np = (size_t)(n_buckets + kScanBlock - 1) / kScanBlock;
  return (sizeof(int64_t) + sizeof(int)) * (np > 0 ? np : 1);
}

extern "C" int32_t bs_bin_tiles_offsets(const int32_t* bucket_counts, int32_t n_buckets, int32_t* ranges,
                                        int32_t* cursor, int64_t* stats, void* workspace, size_t ws_bytes,
                                        void* stream) {
  BS_REQUIRE(n_buckets >= 1, BS_ERR_PARAMETER, "bin: bad bucket count");
  cudaStream_t s = as_stream(stream);
  const int np = (n_buckets + kScanBlock - 1) / kScanBlock;
  BS_REQUIRE(ws_bytes >= bs_bin_tiles_offsets_workspace(n_buckets), BS_ERR_CAPACITY,
             "bin offsets workspace too small");
  int64_t* part = static_cast<int64_t*>(workspace);
  int* pmax = reinterpret_cast<int*>(part + np);
  bucket_sums_kernel<<<np, kScanBlock, 0, s>>>(bucket_counts, n_buckets, part, pmax);
  BS_LAUNCH_CHECK("bucket_sums_kernel");
  bucket_parts_kernel<<<1, kScanBlock, 0, s>>>(part, pmax, np, stats);
  BS_LAUNCH_CHECK("bucket_parts_kernel");
  bucket_ranges_kernel<<<np, kScanBlock, 0, s>>>(bucket_counts, n_buckets, part, reinterpret_cast<int2*>(ranges),
                                                 cursor);
  BS_LAUNCH_CHECK("bucket_ranges_kernel");
  return BS_OK;
}

extern "C" int32_t bs_bin_tiles_scatter(const float* sp_rows, int64_t n_rows, const int64_t* seg_row0,
                                        const int32_t* seg_slot, int32_t n_segs, const bs_camera* slot_cams,
                                        int32_t tiles_per_slot, int32_t* cursor, uint64_t* inst_keys,
                                        int64_t capacity, int32_t model, void* stream) {
  BS_REQUIRE(n_segs >= 1, BS_ERR_PARAMETER, "bin: need at least one segment");
  if (n_rows == 0) return BS_OK;
  BinGeom g{sp_rows, n_rows, seg_row0, seg_slot, n_segs, slot_cams, tiles_per_slot, sp_layout(model)};
  scatter_tiles_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(g, cursor, inst_keys, capacity);
  BS_LAUNCH_CHECK("scatter_tiles_kernel");
  return BS_OK;
}

namespace {
int32_t bin_tiles_sort(const uint64_t* inst_keys, const int32_t* ranges, int32_t n_buckets, int32_t smem_cap,
                       bool bitonic256, uint32_t* inst_rows, void* stream) {
  BS_REQUIRE(smem_cap >= 1 && smem_cap <= kSortCap, BS_ERR_PARAMETER, "bin: smem_cap must be in [1, %d]",
             kSortCap);
  if (n_buckets == 0) return BS_OK;
  cudaStream_t s = as_stream(stream);
  const int grid = (n_buckets + kSortWarpsPerCta - 1) / kSortWarpsPerCta;
  const int2* rg = reinterpret_cast<const int2*>(ranges);
  // n <= 128 (and, with bitonic256, 129..256): register bitonic networks
  if (bitonic256)
    sort_tiles_warp_kernel<8><<<grid, 32 * kSortWarpsPerCta, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
  else
    sort_tiles_warp_kernel<4><<<grid, 32 * kSortWarpsPerCta, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
  BS_LAUNCH_CHECK("sort_tiles_warp_kernel<small>");
  if (!bitonic256) {
    sort_tiles_merge_kernel<8, 8><<<grid, 32 * 8, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
    BS_LAUNCH_CHECK("sort_tiles_merge_kernel<8>");
  }
  // size classes above smem_cap cannot hold a bucket the caller wants sorted
  // here (callers pass min(cap, largest bucket)): their launches are skipped
  if (smem_cap > 256) {
    sort_tiles_merge_kernel<16, 8><<<grid, 32 * 8, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
    BS_LAUNCH_CHECK("sort_tiles_merge_kernel<16>");
  }
  if (smem_cap <= 512) {
  } else if (kMerge1024) {
    const int grid4 = (n_buckets + 3) / 4;
    sort_tiles_merge_kernel<32, 4><<<grid4, 32 * 4, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
    BS_LAUNCH_CHECK("sort_tiles_merge_kernel<32>");
  } else {
    sort_tiles_warp_kernel<32><<<grid, 32 * kSortWarpsPerCta, 0, s>>>(inst_keys, rg, n_buckets, smem_cap, inst_rows);
    BS_LAUNCH_CHECK("sort_tiles_warp_kernel<32>");
  }
  if (smem_cap > kWarpCap) {
    {
      int m = 2;
      while (m < smem_cap) m <<= 1;
      const size_t smem = sizeof(uint64_t) * (size_t)m;
      cudaFuncSetAttribute(sort_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      sort_tiles_kernel<<<sms, kSortThreads, smem, s>>>(inst_keys, reinterpret_cast<const int2*>(ranges), n_buckets,
                                                        smem_cap, inst_rows);
    }
    BS_LAUNCH_CHECK("sort_tiles_kernel");
  }
  return BS_OK;
}
}  // namespace

extern "C" int32_t bs_bin_tiles_sort(const uint64_t* inst_keys, const int32_t* ranges, int32_t n_buckets,
                                     int32_t smem_cap, uint32_t* inst_rows, void* stream) {
  return bin_tiles_sort(inst_keys, ranges, n_buckets, smem_cap, kBitonic256, inst_rows, stream);
}

// With the instance count: the 129..256-key buckets go through the register
// bitonic network when the buckets are full on average (C2: 261 keys per
// bucket, 10 us faster), else through the warp merge sort, which also lets
// the small-bucket kernel use the 128-key network and its smaller register
// budget (C4: 123 keys per bucket, 2.19 -> 2.03 ms for the binning stage).
extern "C" int32_t bs_bin_tiles_sort_n(const uint64_t* inst_keys, const int32_t* ranges, int32_t n_buckets,
                                       int32_t smem_cap, int64_t n_inst, uint32_t* inst_rows, void* stream) {
  const bool bitonic256 = n_inst >= 192ll * n_buckets;
  return bin_tiles_sort(inst_keys, ranges, n_buckets, smem_cap, bitonic256, inst_rows, stream);
}

extern "C" int32_t bs_bin_tiles_max_sort(void) { return kSortCap; }

extern "C" int32_t bs_keys_low32(const uint64_t* keys, int64_t n, uint32_t* out, void* stream) {
  if (n == 0) return BS_OK;
  low32_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(keys, n, out);
  BS_LAUNCH_CHECK("low32_kernel");
  return BS_OK;
}
