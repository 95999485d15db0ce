// Patch-level image placement (P > 1) of the distributed step: which ranks
// need a splat row, the send layout of the splat all-to-all, and the return
// path of the gradient rows.
//
// With P x P patches per view, patch j of view v is rendered by rank
// W[v P^2 + j] (hierarchical_place over the access matrix of
// visibility.py:308-358).  A splat row is needed by every rank that renders a
// patch its support box (sp[rad_off], sp[rad_off + 1]) reaches -- the render
// set, a superset of the access matrix's centre-in-patch count
// (SURVEY.md §7(iv)).  Patch c of a view spans pixel columns
// [floor(c W / P), floor((c + 1) W / P)) (visibility.py:164-165).
//
//   bs_row_dest_mask    per row: bit d set iff rank d renders a patch the
//                       row's support reaches
//   bs_dest_compact     per destination d, the rows with bit d in row order
//                       (view-major), i.e. the send layout grouped by
//                       destination then view; per-(d, view) counts
//   bs_gather_rows      send rows = sp[send_idx]
//   bs_scatter_add_rows gsp[send_idx] += returned gradient rows (a row sent
//                       to several ranks gets all their contributions)
#include "common.cuh"
#include "tile.cuh"

namespace bs {
namespace {

__global__ void row_dest_mask_kernel(const float* __restrict__ sp, int stride, int rad_off, int ctr_off, int64_t n_rows,
                                     const int64_t* __restrict__ view_row0, int B, int P, int W, int H,
                                     const int32_t* __restrict__ patch_owner, uint32_t* __restrict__ mask) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int v = 0;  // view of row r: last v with view_row0[v] <= r
    for (int k = 1; k < B; ++k)
      if (view_row0[k] <= r) v = k;
    const float* row = sp + r * stride;
    const float u = row[ctr_off], vv = row[ctr_off + 1], hx = row[rad_off], hy = row[rad_off + 1];
    uint32_t m = 0u;
    if (hx > 0.f && hy > 0.f) {
      // pixel columns / rows whose centres the support box may reach (padded)
      const int x0 = max(0, (int)ceilf(u - hx - 0.5f - 1e-3f)), x1 = min(W - 1, (int)floorf(u + hx - 0.5f + 1e-3f));
      const int y0 = max(0, (int)ceilf(vv - hy - 0.5f - 1e-3f)), y1 = min(H - 1, (int)floorf(vv + hy - 0.5f + 1e-3f));
      if (x0 <= x1 && y0 <= y1) {
        const int c0 = ((x0 + 1) * P - 1) / W, c1 = ((x1 + 1) * P - 1) / W;
        const int r0 = ((y0 + 1) * P - 1) / H, r1 = ((y1 + 1) * P - 1) / H;
        for (int pr = r0; pr <= r1; ++pr)
          for (int pc = c0; pc <= c1; ++pc) m |= 1u << patch_owner[(v * P + pr) * P + pc];
      }
    }
    mask[r] = m;
  }
}

constexpr int kCompactThreads = 1024;

// phase 1: per block of rows, how many carry bit d (n_dest <= 32)
__global__ void __launch_bounds__(kCompactThreads) dest_count_kernel(const uint32_t* __restrict__ mask, int64_t n_rows,
                                                                     int n_dest, int32_t* __restrict__ block_counts) {
  __shared__ int s_cnt[32];
  if (threadIdx.x < 32) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t r = blockIdx.x * (int64_t)kCompactThreads + threadIdx.x;
  const uint32_t m = r < n_rows ? mask[r] : 0u;
  for (int d = 0; d < n_dest; ++d) {
    const int c = __popc(__ballot_sync(0xffffffffu, (m >> d) & 1u));
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt[d], c);
  }
  __syncthreads();
  if (threadIdx.x < n_dest) block_counts[(int64_t)blockIdx.x * n_dest + threadIdx.x] = s_cnt[threadIdx.x];
}

// phase 2 (one block): exclusive offsets in (d, block) order; dest_total[d]
__global__ void __launch_bounds__(1024) dest_scan_kernel(int32_t* __restrict__ block_counts, int n_blocks, int n_dest,
                                                         int64_t* __restrict__ dest_total) {
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int d = 0; d < n_dest; ++d) {
    const int64_t d_begin = s_carry;
    for (int b0 = 0; b0 < n_blocks; b0 += 1024) {
      const int b = b0 + threadIdx.x;
      const int64_t x0 = b < n_blocks ? block_counts[(int64_t)b * n_dest + d] : 0;
      int64_t x = x0;
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
      const int64_t excl = s_carry + (w ? s_w[w - 1] : 0) + x - x0;
      if (b < n_blocks) block_counts[(int64_t)b * n_dest + d] = (int32_t)(excl - d_begin);
      const int64_t tot = s_w[31];
      __syncthreads();
      if (threadIdx.x == 0) s_carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) dest_total[d] = s_carry - d_begin;
    __syncthreads();
  }
}

// phase 3: positions; send_idx[dest_base[d] + rank] = r; per-(d, view) counts
__global__ void __launch_bounds__(kCompactThreads) dest_scatter_kernel(
    const uint32_t* __restrict__ mask, int64_t n_rows, int n_dest, const int32_t* __restrict__ block_offsets,
    const int64_t* __restrict__ dest_base, const int64_t* __restrict__ view_row0, int B,
    int64_t* __restrict__ send_idx, int64_t* __restrict__ view_counts) {
  __shared__ int s_wsum[32][kCompactThreads / 32];
  const int64_t r = blockIdx.x * (int64_t)kCompactThreads + threadIdx.x;
  const uint32_t m = r < n_rows ? mask[r] : 0u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (int d = 0; d < n_dest; ++d) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (m >> d) & 1u);
    if (lane == 0) s_wsum[d][w] = __popc(bal);
  }
  __syncthreads();
  int v = 0;
  if (r < n_rows)
    for (int k = 1; k < B; ++k)
      if (view_row0[k] <= r) v = k;
  for (int d = 0; d < n_dest; ++d) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (m >> d) & 1u);
    if ((m >> d) & 1u) {
      int before = 0;
      for (int k = 0; k < w; ++k) before += s_wsum[d][k];
      const int64_t pos = dest_base[d] + block_offsets[(int64_t)blockIdx.x * n_dest + d] + before + __popc(bal & lt);
      send_idx[pos] = r;
      atomicAdd(reinterpret_cast<unsigned long long*>(view_counts + (int64_t)d * B + v), 1ull);
    }
  }
}

__global__ void gather_rows_kernel(const float4* __restrict__ src, int w4, const int64_t* __restrict__ idx, int64_t n,
                                   float4* __restrict__ dst) {
  const int64_t total = n * w4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w4;
    const int k = (int)(t - i * w4);
    dst[t] = src[idx[i] * w4 + k];
  }
}

__global__ void gather_words_kernel(const uint32_t* __restrict__ src, int w, const int64_t* __restrict__ idx, int64_t n,
                                    uint32_t* __restrict__ dst) {
  const int64_t total = n * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w;
    const int k = (int)(t - i * w);
    dst[t] = src[idx[i] * w + k];
  }
}

// canonical order: key = (slot << 32) | global id, value = received row
__global__ void order_keys_kernel(const int32_t* __restrict__ row_gid, int64_t n, const int64_t* __restrict__ seg_row0,
                                  const int32_t* __restrict__ seg_slot, int n_segs, uint64_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int slot = seg_slot[segment_of(seg_row0, n_segs, r)];
    keys[r] = ((uint64_t)(uint32_t)slot << 32) | (uint32_t)row_gid[r];
    vals[r] = (uint32_t)r;
  }
}

__global__ void order_out_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                                 int64_t* __restrict__ order, int32_t* __restrict__ canon_gid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    order[i] = (int64_t)vals[i];
    if (canon_gid) canon_gid[i] = (int32_t)(uint32_t)keys[i];
  }
}

__global__ void scatter_add_rows_kernel(const float* __restrict__ src, int src_width, int dst_width, int used,
                                        const int64_t* __restrict__ idx, int64_t n, float* __restrict__ dst) {
  const int64_t total = n * used;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / used;
    const int k = (int)(t - i * used);
    atomicAdd(dst + idx[i] * dst_width + k, src[i * src_width + k]);
  }
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_row_dest_mask(const float* sp_rows, int32_t model, int64_t n_rows, const int64_t* view_row0,
                                    int32_t n_views, int32_t P, int32_t width, int32_t height,
                                    const int32_t* patch_owner, uint32_t* dest_mask, void* stream) {
  BS_REQUIRE(n_rows >= 0 && n_views >= 1 && n_views <= 32, BS_ERR_PARAMETER, "bad row / view counts");
  BS_REQUIRE(P >= 1 && P <= 8 && width >= P && height >= P, BS_ERR_PARAMETER, "patch factor must be in [1, 8]");
  if (n_rows == 0) return BS_OK;
  const SpLayout L = sp_layout(model);
  row_dest_mask_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(
      sp_rows, L.stride, L.rad_off, L.ctr_off, n_rows, view_row0, n_views, P, width, height, patch_owner, dest_mask);
  BS_LAUNCH_CHECK("row_dest_mask_kernel");
  return BS_OK;
}

extern "C" size_t bs_dest_compact_workspace(int64_t n_rows, int32_t n_dest) {
  const int64_t blocks = (n_rows + kCompactThreads - 1) / kCompactThreads;
  return sizeof(int32_t) * (size_t)(blocks > 0 ? blocks : 1) * (size_t)n_dest + 256;
}

// dest_total: int64 [n_dest] (rows per destination); dest_base: int64
// [n_dest] exclusive offsets of the destinations in send_idx, given by the
// caller from dest_total (two calls: count_only = 1 fills dest_total, then
// count_only = 0 writes send_idx and view_counts int64 [n_dest][n_views],
// which the caller zeroes).
extern "C" int32_t bs_dest_compact(const uint32_t* dest_mask, int64_t n_rows, int32_t n_dest,
                                   const int64_t* view_row0, int32_t n_views, int32_t count_only,
                                   int64_t* dest_total, const int64_t* dest_base, int64_t* send_idx,
                                   int64_t* view_counts, void* workspace, size_t ws_bytes, void* stream) {
  BS_REQUIRE(n_dest >= 1 && n_dest <= 32, BS_ERR_PARAMETER, "1..32 destinations");
  BS_REQUIRE(ws_bytes >= bs_dest_compact_workspace(n_rows, n_dest), BS_ERR_CAPACITY, "dest_compact workspace");
  cudaStream_t s = as_stream(stream);
  const int blocks = (int)((n_rows + kCompactThreads - 1) / kCompactThreads);
  int32_t* bc = static_cast<int32_t*>(workspace);
  if (count_only) {
    if (n_rows == 0) {
      cudaMemsetAsync(dest_total, 0, sizeof(int64_t) * n_dest, s);
      return BS_OK;
    }
    dest_count_kernel<<<blocks, kCompactThreads, 0, s>>>(dest_mask, n_rows, n_dest, bc);
    BS_LAUNCH_CHECK("dest_count_kernel");
    dest_scan_kernel<<<1, 1024, 0, s>>>(bc, blocks, n_dest, dest_total);
    BS_LAUNCH_CHECK("dest_scan_kernel");
    return BS_OK;
  }
  if (n_rows == 0) return BS_OK;
  dest_scatter_kernel<<<blocks, kCompactThreads, 0, s>>>(dest_mask, n_rows, n_dest, bc, dest_base, view_row0, n_views,
                                                        send_idx, view_counts);
  BS_LAUNCH_CHECK("dest_scatter_kernel");
  return BS_OK;
}

extern "C" int32_t bs_gather_rows(const float* src, int32_t width, const int64_t* idx, int64_t n, float* dst,
                                  void* stream) {
  BS_REQUIRE(width > 0, BS_ERR_PARAMETER, "row width must be >= 1");
  if (n <= 0) return BS_OK;
  if (width % 4 != 0) {
    gather_words_kernel<<<grid_for(n * width, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const uint32_t*>(src), width, idx, n, reinterpret_cast<uint32_t*>(dst));
    BS_LAUNCH_CHECK("gather_words_kernel");
    return BS_OK;
  }
  gather_rows_kernel<<<grid_for(n * (width / 4), 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(src), width / 4, idx, n, reinterpret_cast<float4*>(dst));
  BS_LAUNCH_CHECK("gather_rows_kernel");
  return BS_OK;
}

extern "C" int32_t bs_scatter_add_rows(const float* src, int32_t src_width, int32_t used, const int64_t* idx,
                                       int64_t n, float* dst, int32_t dst_width, void* stream) {
  BS_REQUIRE(used > 0 && used <= src_width && used <= dst_width, BS_ERR_PARAMETER, "bad row width");
  if (n <= 0) return BS_OK;
  scatter_add_rows_kernel<<<grid_for(n * used, 256), 256, 0, as_stream(stream)>>>(src, src_width, dst_width, used, idx,
                                                                                  n, dst);
  BS_LAUNCH_CHECK("scatter_add_rows_kernel");
  return BS_OK;
}

extern "C" size_t bs_canonical_order_workspace(int64_t n_rows) {
  const int64_t n = n_rows > 0 ? n_rows : 1;
  const size_t a = ((size_t)n * 8 + 255) & ~(size_t)255, b = ((size_t)n * 4 + 255) & ~(size_t)255;
  return 2 * a + 2 * b + bs_radix_sort_workspace(n);
}

extern "C" int32_t bs_canonical_order(const int32_t* row_gid, int64_t n_rows, const int64_t* seg_row0,
                                      const int32_t* seg_slot, int32_t n_segs, int32_t n_slots, int64_t* order,
                                      int32_t* canon_gid, void* workspace, size_t ws_bytes, void* stream) {
  BS_REQUIRE(n_slots >= 1 && n_segs >= 1, BS_ERR_PARAMETER, "canonical_order needs >= 1 slot and segment");
  BS_REQUIRE(ws_bytes >= bs_canonical_order_workspace(n_rows), BS_ERR_CAPACITY, "canonical_order workspace too small");
  if (n_rows <= 0) return BS_OK;
  const int64_t n = n_rows;
  const size_t a = ((size_t)n * 8 + 255) & ~(size_t)255, b = ((size_t)n * 4 + 255) & ~(size_t)255;
  char* w = static_cast<char*>(workspace);
  uint64_t* keys = reinterpret_cast<uint64_t*>(w);
  uint64_t* keys_alt = reinterpret_cast<uint64_t*>(w + a);
  uint32_t* vals = reinterpret_cast<uint32_t*>(w + 2 * a);
  uint32_t* vals_alt = reinterpret_cast<uint32_t*>(w + 2 * a + b);
  void* sort_ws = w + 2 * a + 2 * b;
  cudaStream_t s = as_stream(stream);
  order_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(row_gid, n, seg_row0, seg_slot, n_segs, keys, vals);
  BS_LAUNCH_CHECK("order_keys_kernel");
  int bits = 1;
  while ((1 << bits) < n_slots) ++bits;
  // keys sorted stably on [0, 32 + bits): ids are unique within a slot
  const int32_t st = bs_radix_sort_u64(keys, vals, keys_alt, vals_alt, n, nullptr, 0, 32 + bits, sort_ws,
                                       bs_radix_sort_workspace(n), stream);
  if (st) return st;
  order_out_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, vals, n, order, canon_gid);
  BS_LAUNCH_CHECK("order_out_kernel");
  return BS_OK;
}
