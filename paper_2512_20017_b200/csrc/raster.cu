// K3 forward alpha compositing (image_render), the mean-L1
// loss (loss_fn) and K4 backward (image_render.backward,
// PAPER.md:503).
//
// One CTA of 256 threads per 16x16 tile; one pixel per thread (pixel centre
// (x + 0.5, y + 0.5)).  Splats of the tile's depth-sorted instance range are
// staged through shared memory in batches of 256 (one gathered SP row per
// thread), then every thread blends the batch front to back:
//   power = -0.5 (A dx^2 + C dy^2) - B dx dy,  dx = u - px
//   alpha = min(0.99, opacity * exp(power)); skipped if power > 0 or
//   alpha < 1/255; the pixel stops before the splat that would bring its
//   transmittance below 1e-4 (standard 3DGS conventions).
// The CTA leaves the loop when every pixel is done (__syncthreads_count).
// The backward kernel walks the same range back to front, reconstructing
// T by division, and reduces each splat's 9 gradient terms over the warp
// (shuffles) before one atomicAdd per term per warp.
#include "common.cuh"

namespace bs {
namespace {

constexpr int kRastThreads = BS_TILE * BS_TILE;  // 256
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kAlphaMax = 0.99f;
constexpr float kTMin = 1e-4f;

struct RastArgs {
  int n_slots, tiles_per_slot, W, H, tiles_x;
  float bg[3];
  int loss_fused;
  float inv_norm;  // 1 / (H * W * 3)
};

// Bit-identical in both kernels (explicit round-to-nearest intrinsics).
// a = (u, v, conic_a, conic_b), cconic = conic_c.
__device__ __forceinline__ float splat_power(float4 a, float cconic, float px, float py, float& dx, float& dy) {
  dx = __fsub_rn(a.x, px);
  dy = __fsub_rn(a.y, py);
  const float q = __fmaf_rn(a.z, __fmul_rn(dx, dx), __fmul_rn(cconic, __fmul_rn(dy, dy)));
  return __fmaf_rn(-0.5f, q, -__fmul_rn(a.w, __fmul_rn(dx, dy)));
}

// smem staging: sa = (u, v, A, B), sb = (C, opacity, r, g), sc = b
struct SplatSmem {
  float4 a[kRastThreads];
  float4 b[kRastThreads];
  float c[kRastThreads];
  uint32_t row[kRastThreads];
};

__device__ __forceinline__ void stage_splat(SplatSmem& s, int j, const float* __restrict__ sp, uint32_t row) {
  const float4* r4 = reinterpret_cast<const float4*>(sp + (int64_t)row * BS_SP_FLOATS);
  const float4 p0 = __ldg(r4);      // u v opac A
  const float4 p1 = __ldg(r4 + 1);  // B C r g
  const float b = __ldg(sp + (int64_t)row * BS_SP_FLOATS + 8);
  s.a[j] = make_float4(p0.x, p0.y, p0.w, p1.x);
  s.b[j] = make_float4(p1.y, p0.z, p1.z, p1.w);
  s.c[j] = b;
  s.row[j] = row;
}

__global__ void __launch_bounds__(kRastThreads) raster_fwd_kernel(RastArgs a, const float* __restrict__ sp,
                                                                  const uint32_t* __restrict__ inst_rows,
                                                                  const int2* __restrict__ ranges,
                                                                  float* __restrict__ image,
                                                                  float* __restrict__ final_T,
                                                                  int32_t* __restrict__ n_contrib,
                                                                  const uint8_t* __restrict__ gt,
                                                                  const int32_t* __restrict__ gt_view,
                                                                  float* __restrict__ loss_tiles) {
  __shared__ SplatSmem s;
  __shared__ float s_red[kRastThreads / 32];
  const int slot = blockIdx.z;
  const int tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int px = blockIdx.x * BS_TILE + (threadIdx.x % BS_TILE);
  const int py = blockIdx.y * BS_TILE + (threadIdx.x / BS_TILE);
  const bool inside = px < a.W && py < a.H;
  const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  int contrib = 0;
  bool done = !inside;
  for (int b0 = rg.x; b0 < rg.y; b0 += kRastThreads) {
    if (__syncthreads_count(done) == kRastThreads) break;
    const int idx = b0 + threadIdx.x;
    if (idx < rg.y) stage_splat(s, threadIdx.x, sp, inst_rows[idx]);
    __syncthreads();
    const int nb = min(kRastThreads, rg.y - b0);
    for (int j = 0; j < nb && !done; ++j) {
      const float4 sa = s.a[j];
      const float4 sb = s.b[j];
      float dx, dy;
      const float power = splat_power(sa, sb.x, pxf, pyf, dx, dy);
      if (power > 0.f) continue;
      const float alpha = fminf(kAlphaMax, __fmul_rn(sb.y, __expf(power)));
      if (alpha < kAlphaMin) continue;
      const float nT = __fmul_rn(T, __fsub_rn(1.f, alpha));
      if (nT < kTMin) {
        done = true;
        break;
      }
      const float w = __fmul_rn(alpha, T);
      C0 = __fmaf_rn(sb.z, w, C0);
      C1 = __fmaf_rn(sb.w, w, C1);
      C2 = __fmaf_rn(s.c[j], w, C2);
      T = nT;
      contrib = b0 + j + 1 - rg.x;
    }
  }
  float l = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    const float o0 = C0 + T * a.bg[0], o1 = C1 + T * a.bg[1], o2 = C2 + T * a.bg[2];
    image[3 * pix] = o0;
    image[3 * pix + 1] = o1;
    image[3 * pix + 2] = o2;
    final_T[pix] = T;
    n_contrib[pix] = contrib;
    if (a.loss_fused) {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
      const float g0 = gp[0] * (1.f / 255.f), g1 = gp[1] * (1.f / 255.f), g2 = gp[2] * (1.f / 255.f);
      l = fabsf(o0 - g0) + fabsf(o1 - g1) + fabsf(o2 - g2);
    }
  }
  if (a.loss_fused) {
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int k = 0; k < kRastThreads / 32; ++k) t += s_red[k];
      loss_tiles[(int64_t)slot * a.tiles_per_slot + tile] = t;
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kRastThreads) raster_bwd_kernel(
    RastArgs a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    const float* __restrict__ image, const float* __restrict__ final_T, const int32_t* __restrict__ n_contrib,
    const float* __restrict__ grad_image, const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view,
    float* __restrict__ g_sp) {
  __shared__ SplatSmem s;
  __shared__ int s_max[kRastThreads / 32];
  const int slot = blockIdx.z;
  const int tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int px = blockIdx.x * BS_TILE + (threadIdx.x % BS_TILE);
  const int py = blockIdx.y * BS_TILE + (threadIdx.x / BS_TILE);
  const bool inside = px < a.W && py < a.H;
  const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  const int lane = threadIdx.x & 31;

  float T = 1.f, dC0 = 0.f, dC1 = 0.f, dC2 = 0.f;
  int my_n = 0;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    T = final_T[pix];
    my_n = n_contrib[pix];
    if (grad_image) {
      dC0 = grad_image[3 * pix];
      dC1 = grad_image[3 * pix + 1];
      dC2 = grad_image[3 * pix + 2];
    } else {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
      const float d0 = image[3 * pix] - gp[0] * (1.f / 255.f);
      const float d1 = image[3 * pix + 1] - gp[1] * (1.f / 255.f);
      const float d2 = image[3 * pix + 2] - gp[2] * (1.f / 255.f);
      dC0 = (d0 > 0.f ? 1.f : (d0 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      dC1 = (d1 > 0.f ? 1.f : (d1 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      dC2 = (d2 > 0.f ? 1.f : (d2 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    }
  }
  // deepest contributing splat over the tile
  int mx = my_n;
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  int tile_n = 0;
  for (int k = 0; k < kRastThreads / 32; ++k) tile_n = max(tile_n, s_max[k]);
  const float T_final = T;
  const float bgdot = a.bg[0] * dC0 + a.bg[1] * dC1 + a.bg[2] * dC2;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;          // colour behind the current splat
  float last_alpha = 0.f, lc0 = 0.f, lc1 = 0.f, lc2 = 0.f;
  const int end = rg.x + tile_n;
  for (int bend = end; bend > rg.x; bend -= kRastThreads) {
    const int bstart = max(rg.x, bend - kRastThreads);
    const int nb = bend - bstart;
    __syncthreads();
    if ((int)threadIdx.x < nb) stage_splat(s, threadIdx.x, sp, inst_rows[bend - 1 - threadIdx.x]);
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      const int rel = bend - 1 - j - rg.x;  // range-relative index of this splat
      bool valid = inside && rel < my_n;
      float g[9];
      const float4 sa = s.a[j];
      const float4 sb = s.b[j];
      const float cb = s.c[j];
      float dx = 0.f, dy = 0.f, power = 0.f, alpha = 0.f, ex = 0.f;
      if (valid) {
        power = splat_power(sa, sb.x, pxf, pyf, dx, dy);
        valid = power <= 0.f;
        if (valid) {
          ex = __expf(power);
          const float raw = __fmul_rn(sb.y, ex);
          alpha = fminf(kAlphaMax, raw);
          valid = alpha >= kAlphaMin;
          if (valid) {
            const float ra = 1.f / (1.f - alpha);
            T = T * ra;
            const float fac = alpha * T;
            g[6] = fac * dC0;
            g[7] = fac * dC1;
            g[8] = fac * dC2;
            acc0 = last_alpha * lc0 + (1.f - last_alpha) * acc0;
            acc1 = last_alpha * lc1 + (1.f - last_alpha) * acc1;
            acc2 = last_alpha * lc2 + (1.f - last_alpha) * acc2;
            last_alpha = alpha;
            lc0 = sb.z;
            lc1 = sb.w;
            lc2 = cb;
            float dL_dalpha = T * ((sb.z - acc0) * dC0 + (sb.w - acc1) * dC1 + (cb - acc2) * dC2);
            dL_dalpha -= T_final * ra * bgdot;
            const bool clamped = raw > kAlphaMax;
            const float dL_dpow = clamped ? 0.f : dL_dalpha * alpha;
            g[2] = clamped ? 0.f : dL_dalpha * ex;
            g[3] = -0.5f * dx * dx * dL_dpow;
            g[4] = -dx * dy * dL_dpow;
            g[5] = -0.5f * dy * dy * dL_dpow;
            g[0] = -(sa.z * dx + sa.w * dy) * dL_dpow;
            g[1] = -(sa.w * dx + sb.x * dy) * dL_dpow;
          }
        }
      }
      if (!__any_sync(0xffffffffu, valid)) continue;
      if (!valid)
#pragma unroll
        for (int k = 0; k < 9; ++k) g[k] = 0.f;
#pragma unroll
      for (int k = 0; k < 9; ++k) g[k] = warp_sum(g[k]);
      if (lane == 0) {
        float* dst = g_sp + (int64_t)s.row[j] * BS_GSP_FLOATS;
#pragma unroll
        for (int k = 0; k < 9; ++k) atomicAdd(dst + k, g[k]);
      }
    }
  }
}

__global__ void l1_loss_kernel(const float* __restrict__ img, const uint8_t* __restrict__ gt, int n_slots,
                               int64_t per_slot, float* __restrict__ partial, float* __restrict__ grad,
                               float inv_norm) {
  // grid: (blocks_per_slot, n_slots); deterministic partial per block
  __shared__ float s_red[8];
  const int slot = blockIdx.y;
  float l = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_slot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = slot * per_slot + i;
    const float d = img[k] - gt[k] * (1.f / 255.f);
    l += fabsf(d);
    if (grad) grad[k] = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_norm;
  }
  l = warp_sum(l);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_red[k];
    partial[slot * gridDim.x + blockIdx.x] = t;
  }
}

// loss[s] = sum(partial[s, :]) * inv_norm, fixed order (deterministic).
__global__ void reduce_partials_kernel(const float* __restrict__ partial, int n_slots, int per, float inv_norm,
                                       float* __restrict__ loss) {
  __shared__ float s_red[32];
  const int slot = blockIdx.x;
  float l = 0.f;
  for (int i = threadIdx.x; i < per; i += blockDim.x) l += partial[(int64_t)slot * per + i];
  l = warp_sum(l);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_red[k];
    loss[slot] = t * inv_norm;
  }
}

int32_t make_args(const bs_raster_desc* d, RastArgs& a) {
  BS_REQUIRE(d != nullptr, BS_ERR_PARAMETER, "null raster descriptor");
  BS_REQUIRE(d->width >= 1 && d->height >= 1, BS_ERR_PARAMETER, "image size must be >= 1 pixel");
  BS_REQUIRE(d->n_slots >= 1 && d->n_slots <= 65535, BS_ERR_PARAMETER, "bad slot count");
  a.n_slots = d->n_slots;
  a.W = d->width;
  a.H = d->height;
  a.tiles_x = (d->width + BS_TILE - 1) / BS_TILE;
  const int tiles_y = (d->height + BS_TILE - 1) / BS_TILE;
  BS_REQUIRE(d->tiles_per_slot >= a.tiles_x * tiles_y, BS_ERR_PARAMETER, "tiles_per_slot too small");
  a.tiles_per_slot = d->tiles_per_slot;
  a.bg[0] = d->bg[0];
  a.bg[1] = d->bg[1];
  a.bg[2] = d->bg[2];
  a.loss_fused = d->loss_fused;
  a.inv_norm = (float)(1.0 / (3.0 * (double)d->width * (double)d->height));
  return BS_OK;
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_raster_fwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                 const int32_t* ranges, float* image, float* final_T, int32_t* n_contrib,
                                 const uint8_t* gt, const int32_t* gt_slot_view, float* loss_tiles,
                                 void* stream) {
  RastArgs a;
  int32_t st = make_args(d, a);
  if (st) return st;
  BS_REQUIRE(!a.loss_fused || (gt && loss_tiles), BS_ERR_PARAMETER, "fused loss needs gt and loss_tiles");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  raster_fwd_kernel<<<grid, kRastThreads, 0, as_stream(stream)>>>(a, sp_rows, inst_rows,
                                                                  reinterpret_cast<const int2*>(ranges), image,
                                                                  final_T, n_contrib, gt, gt_slot_view, loss_tiles);
  BS_LAUNCH_CHECK("raster_fwd_kernel");
  return BS_OK;
}

extern "C" int32_t bs_raster_bwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                 const int32_t* ranges, const float* image, const float* final_T,
                                 const int32_t* n_contrib, const float* grad_image, const uint8_t* gt,
                                 const int32_t* gt_slot_view, float* g_sp, void* stream) {
  RastArgs a;
  int32_t st = make_args(d, a);
  if (st) return st;
  BS_REQUIRE(grad_image || (image && gt), BS_ERR_PARAMETER, "raster_bwd needs grad_image or (image, gt)");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  raster_bwd_kernel<<<grid, kRastThreads, 0, as_stream(stream)>>>(a, sp_rows, inst_rows,
                                                                  reinterpret_cast<const int2*>(ranges), image,
                                                                  final_T, n_contrib, grad_image, gt, gt_slot_view, g_sp);
  BS_LAUNCH_CHECK("raster_bwd_kernel");
  return BS_OK;
}

extern "C" size_t bs_l1_loss_workspace(int32_t n_slots) { return sizeof(float) * 64 * (size_t)n_slots; }

extern "C" int32_t bs_l1_loss(const float* image, const uint8_t* gt, int32_t n_slots, int32_t height, int32_t width,
                              float* loss, float* grad, void* ws, size_t ws_bytes, void* stream) {
  BS_REQUIRE(n_slots >= 1 && height >= 1 && width >= 1, BS_ERR_PARAMETER, "bad image shape");
  BS_REQUIRE(ws_bytes >= bs_l1_loss_workspace(n_slots), BS_ERR_CAPACITY, "l1_loss workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t per = 3ll * height * width;
  const int blocks = 64;
  float* partial = static_cast<float*>(ws);
  const float inv_norm = (float)(1.0 / (double)per);
  l1_loss_kernel<<<dim3(blocks, n_slots), 256, 0, s>>>(image, gt, n_slots, per, partial, grad, inv_norm);
  BS_LAUNCH_CHECK("l1_loss_kernel");
  reduce_partials_kernel<<<n_slots, 64, 0, s>>>(partial, n_slots, blocks, inv_norm, loss);
  BS_LAUNCH_CHECK("reduce_partials_kernel");
  return BS_OK;
}

extern "C" int32_t bs_reduce_loss_tiles(const float* loss_tiles, int32_t n_slots, int32_t tiles_per_slot,
                                        int32_t height, int32_t width, float* loss, void* stream) {
  BS_REQUIRE(n_slots >= 1, BS_ERR_PARAMETER, "bad slot count");
  const float inv_norm = (float)(1.0 / (3.0 * (double)height * (double)width));
  reduce_partials_kernel<<<n_slots, 256, 0, as_stream(stream)>>>(loss_tiles, n_slots, tiles_per_slot, inv_norm,
                                                                 loss);
  BS_LAUNCH_CHECK("reduce_partials_kernel");
  return BS_OK;
}
