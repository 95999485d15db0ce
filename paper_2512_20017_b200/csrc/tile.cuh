// Tile geometry shared by the binning kernels.
#pragma once
#include "common.cuh"

namespace bs {

// Tile rectangle of a splat (integer-exact on host and device), support box
// centre (u, v) and half-widths (rx, ry) (3DGS: mean, sp[10], sp[11]):
//   x0 = clamp(floor((u - rx) / 16), 0, tiles_x), x1 = clamp(floor((u + rx) / 16) + 1, 0, tiles_x)
// (and the same in y with ry): the tiles whose pixel span meets the box.
__device__ __forceinline__ int tile_rect_vals(float u, float v, float rx, float ry, int W, int H, int& x0, int& x1,
                                              int& y0, int& y1) {
  if (!(rx > 0.f) || !(ry > 0.f)) {
    x0 = x1 = y0 = y1 = 0;
    return 0;
  }
  const int tx = (W + BS_TILE - 1) / BS_TILE, ty = (H + BS_TILE - 1) / BS_TILE;
  const float inv = 1.0f / BS_TILE;  // exact power of two
  x0 = (int)fminf(fmaxf(floorf(fmul(fsub(u, rx), inv)), 0.f), (float)tx);
  x1 = (int)fminf(fmaxf(fadd(floorf(fmul(fadd(u, rx), inv)), 1.f), 0.f), (float)tx);
  y0 = (int)fminf(fmaxf(floorf(fmul(fsub(v, ry), inv)), 0.f), (float)ty);
  y1 = (int)fminf(fmaxf(fadd(floorf(fmul(fadd(v, ry), inv)), 1.f), 0.f), (float)ty);
  if (x1 <= x0 || y1 <= y0) return 0;
  return (x1 - x0) * (y1 - y0);
}

__device__ __forceinline__ int tile_rect_at(const float* __restrict__ row, int rad_off, int ctr_off, int W, int H,
                                            int& x0, int& x1, int& y0, int& y1) {
  return tile_rect_vals(row[ctr_off], row[ctr_off + 1], row[rad_off], row[rad_off + 1], W, H, x0, x1, y0, y1);
}

// Tile counting of one row's rectangle into (slot, tile) buckets,
// warp-aggregated over the lanes active here (equal buckets -> one atomic).
#ifndef BS_COUNT_PLAIN_ATOMICS
#define BS_COUNT_PLAIN_ATOMICS 0
#endif
__device__ __forceinline__ void count_rect(int32_t* __restrict__ counts, int64_t bucket0, int tx, int x0, int x1,
                                           int y0, int y1) {
#if BS_COUNT_PLAIN_ATOMICS
  for (int y = y0; y < y1; ++y)
    for (int x = x0; x < x1; ++x) atomicAdd(counts + bucket0 + (int64_t)y * tx + x, 1);
  return;
#endif
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  int x = x0, y = y0;
  bool left = x1 > x0 && y1 > y0;
  while (__any_sync(act, left)) {
    int64_t b = -1;
    if (left) {
      b = bucket0 + (int64_t)y * tx + x;
      if (++x == x1) {
        x = x0;
        left = ++y < y1;
      }
    }
    const unsigned peers = __match_any_sync(act, (unsigned long long)b);
    if (b >= 0 && lane == __ffs(peers) - 1) atomicAdd(counts + b, __popc(peers));
  }
}

// 3DGS rows keep the radii at floats 10, 11 (2DGS rows: 16, 17).
__device__ __forceinline__ int tile_rect(const float* __restrict__ row, int W, int H, int& x0, int& x1, int& y0,
                                         int& y1) {
  return tile_rect_at(row, 10, 0, W, H, x0, x1, y0, y1);
}

// Row geometry of the splat-state layouts (include/splat_b200.h).
// Support box: centre (row[ctr_off], row[ctr_off + 1]), half-widths
// (row[rad_off], row[rad_off + 1]); 3DGS centres it on the splat's mean.
struct SpLayout {
  int stride, rad_off, depth_off, ctr_off;
};
__host__ __device__ __forceinline__ SpLayout sp_layout(int model) {
  return model == BS_MODEL_2DGS ? SpLayout{BS_SP2_FLOATS, 16, 15, 22} : SpLayout{BS_SP_FLOATS, 10, 9, 0};
}

// Segment (render slot run) of row r: last s with seg_row0[s] <= r.
__device__ __forceinline__ int segment_of(const int64_t* __restrict__ seg_row0, int n_segs, int64_t r) {
  int lo = 0, hi = n_segs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_row0[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

}  // namespace bs
