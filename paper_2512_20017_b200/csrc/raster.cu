// K3 forward alpha compositing (image_render), the mean-L1
// loss (loss_fn) and K4 backward (image_render.backward,
// PAPER.md:503).
//
// One CTA per 16x16 tile.  With PPL pixels per lane (default 1) a warp owns
// an 8 x 4*PPL pixel region and a tile holds 8 / PPL such warps.  The warps
// of a tile never synchronise with each other: each walks the tile's
// depth-sorted instance range in chunks of 32 on its own, gathering one SP
// row per lane (the next chunk is prefetched into registers while the
// current one is blended), keeps only the splats whose support box (the
// projection's per-axis extents sp[10], sp[11]) can reach its region,
// compacts them with a ballot into warp-private shared memory and blends
// them in depth order.  Per pixel (centre (x + 0.5, y + 0.5)):
//   power = -0.5 q = -0.5 (A dx^2 + C dy^2) - B dx dy,  dx = u - px
//   alpha = min(0.99, opacity * exp(power)); the pair contributes iff
//   q <= k, k = min(9, 2 ln(255 opacity)) -- the 3-sigma cut and the
//   alpha >= 1/255 test as ONE threshold on the exponent, per splat from the
//   shared deterministic log (support_k), so the decision never depends on
//   the exp approximation and is the oracle's bit for bit; a pixel stops
//   before the splat that would bring its transmittance below 1e-4
//   (standard 3DGS conventions; deviations from gsplat
//   v1.4.0 in DESIGN.md §3).
// The conic is staged pre-scaled by -log2(e)/2 (B by -log2(e)) so the
// exponent is one ex2.approx; forward and backward evaluate alpha with the
// same instructions, so their skip / stop decisions agree exactly.
// The support filter only drops splats that are skipped at every pixel of
// the region, so the blend equals walking the whole list.
//
// Backward: each warp walks its own range back to front from the deepest
// contributor of its pixels (T recovered by division).  Per splat the lanes
// that contribute are counted with a ballot: up to kSparseLanes (10) of them
// add their 9 gradient terms with direct REDs (two 128-bit + one 32-bit RED
// into the 16-byte aligned G_SP row); otherwise the warp reduce-scatters the
// 9 sums in 12 shuffles and 9 lanes issue one RED each.
#include "common.cuh"
#include "packed.cuh"

namespace bs {
namespace {

constexpr float kAlphaMax = 0.99f;
constexpr float kTMin = 1e-4f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kHalfLog2e = -0.5f * kLog2e;  // p2 = power * log2(e) = q * kHalfLog2e
#ifndef BS_SPARSE_LANES
// swept on B200 (C2, 128-bit REDs; round 2, 48-byte staged records): 6 1.974, 8 1.937,
// 10 1.931, 12 1.958, 16 2.118 ms (round 1, separate arrays: 12 best at 2.06)
#define BS_SPARSE_LANES 10
#endif
constexpr int kSparseLanes = BS_SPARSE_LANES;

#ifdef BS_RASTER_STATS
// tuning instrumentation (never in the product build; tools/raster_stats.py):
// [0] bwd warp-chunks, [1] bwd kept iterations, [2] of them with no
// contributing lane, [3] sparse, [4] dense, [5] sum of contributing lanes,
// [6] sum of live lanes, [8..40] histogram of contributing lanes; [48] fwd
// warp-chunks, [49] fwd kept iterations, [50] fwd lanes past the support test
__device__ unsigned long long g_rstats[64];
#endif

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct RastArgs {
  int n_slots, tiles_per_slot, W, H, tiles_x;
  float bg[3];
  int loss_fused;
  float inv_norm;                // 1 / (H * W * 3)
  int patch_P;
  const uint64_t* slot_patches;  // NULL: every pixel
  const float* support;          // per-row support threshold (bs_row_support) or NULL
};

// Patch restriction (P > 1): does this slot render pixel (x, y)?  Patch c of
// an image side spans [floor(c W / P), floor((c + 1) W / P)).
__device__ __forceinline__ bool slot_pixel(const uint64_t* slot_patches, int P, int W, int H, int slot, int x, int y) {
  if (x >= W || y >= H) return false;
  if (slot_patches == nullptr) return true;
  const int pc = ((x + 1) * P - 1) / W, pr = ((y + 1) * P - 1) / H;
  return (slot_patches[slot] >> (pr * P + pc)) & 1ull;
}


// packed FP32 pairs: csrc/packed.cuh

// log2(e) * power at a pixel from the pre-scaled conic:
// uv = (u, v), k = (kA, kC), kb: kA = -log2(e) A / 2, kC = -log2(e) C / 2,
// kb = -log2(e) B; npx = -(px, py).  d = (dx, dy) = uv - pixel.
//   power2 = fma(kb, dx dy, kA dx^2) + kC dy^2
// Explicit round-to-nearest ops in a fixed order: identical in both kernels.
__device__ __forceinline__ float splat_power2(F2 uv, F2 k, float kb, F2 npx, F2& d) {
  d = add2(uv, npx);
  const float2 dd = unf2(d);
  const float2 t = unf2(mul2(mul2(d, d), k));
  return __fadd_rn(__fmaf_rn(kb, __fmul_rn(dd.x, dd.y), t.x), t.y);
}

// Warp-private staging, one 48-byte record per splat (one address, three
// broadcast LDS.128): a = (u, v, kA, kC), b = (kB, opacity, r, g),
// c = (b-channel, th2, row bits, -): th2 = the exponent threshold k * (-log2(e) / 2)
struct Staged {
  float4 a, b, c;
};
struct WarpSmem {
  Staged s[32];
};
// forward staging (no row needed): arrays, conflict-free 16-byte stores
struct WarpSmemF {
  float4 a[32];
  float4 b[32];
  float2 c[32];
};

// Lowest log2-exponent of the splat's support: p2 >= th2 <=> q <= k.
__device__ __forceinline__ float support_p2(float opacity) { return __fmul_rn(support_k(opacity), kHalfLog2e); }

// One gathered splat (register prefetch of the next chunk).
struct Splat {
  float4 p0, p1;  // (u v opac A), (B C r g)
  float b;
  float2 h;       // support half-widths (hx, hy) = sp[10], sp[11]
  float th2;      // support threshold (per-row array; else computed at staging)
  uint32_t row;
  bool ok;
};

__device__ __forceinline__ void fetch_row_data(Splat& f, const float* __restrict__ sp, const float* __restrict__ sup,
                                               uint32_t row, bool ok) {
  f.ok = ok;
  if (ok) {
    f.row = row;
    const float4* r4 = reinterpret_cast<const float4*>(sp + (int64_t)row * BS_SP_FLOATS);
    f.p0 = __ldg(r4);
    f.p1 = __ldg(r4 + 1);
    f.b = __ldg(sp + (int64_t)row * BS_SP_FLOATS + 8);
    f.h = __ldg(reinterpret_cast<const float2*>(sp + (int64_t)row * BS_SP_FLOATS + 10));
    if (sup) f.th2 = __ldg(sup + row);
  }
}

__device__ __forceinline__ void fetch_splat(Splat& f, const float* __restrict__ sp, const float* __restrict__ sup,
                                            const uint32_t* __restrict__ inst_rows, int idx, bool ok) {
  fetch_row_data(f, sp, sup, ok ? __ldg(inst_rows + idx) : 0u, ok);
}

// Row index of instance idx (prefetched one chunk ahead of its SP row so the
// two dependent gathers never sit back to back).
__device__ __forceinline__ uint32_t fetch_row(const uint32_t* __restrict__ inst_rows, int idx, bool ok) {
  return ok ? __ldg(inst_rows + idx) : 0u;
}

// Can this splat's support (the box of half-widths hx = sp[10], hy = sp[11]
// around (u, v), written by the projection; 0 = never contributes) reach a
// pixel centre of [x0,x1] x [y0,y1]?  Padded by 1e-3 px + 1e-4 relative so
// pairs on the box edge are left to the per-pixel test.
__device__ __forceinline__ bool reaches(const Splat& f, float x0, float x1, float y0, float y1) {
  const float u = f.p0.x, v = f.p0.y, hx = f.h.x, hy = f.h.y;
  if (!f.ok || !(hx > 0.f)) return false;
  return fabsf(u - fminf(fmaxf(u, x0), x1)) <= fmaf(hx, 1.0001f, 1e-3f) &&
         fabsf(v - fminf(fmaxf(v, y0), y1)) <= fmaf(hy, 1.0001f, 1e-3f);
}

__device__ __forceinline__ void stage(WarpSmemF& s, int lane, const Splat& f, bool have_support) {
  s.a[lane] = make_float4(f.p0.x, f.p0.y, __fmul_rn(f.p0.w, kHalfLog2e), __fmul_rn(f.p1.y, kHalfLog2e));
  s.b[lane] = make_float4(__fmul_rn(f.p1.x, -kLog2e), f.p0.z, f.p1.z, f.p1.w);
  s.c[lane] = make_float2(f.b, have_support ? f.th2 : support_p2(f.p0.z));
}

__device__ __forceinline__ void stage(WarpSmem& s, int lane, const Splat& f, bool have_support) {
  Staged& t = s.s[lane];
  t.a = make_float4(f.p0.x, f.p0.y, __fmul_rn(f.p0.w, kHalfLog2e), __fmul_rn(f.p1.y, kHalfLog2e));
  t.b = make_float4(__fmul_rn(f.p1.x, -kLog2e), f.p0.z, f.p1.z, f.p1.w);
  t.c = make_float4(f.b, have_support ? f.th2 : support_p2(f.p0.z), __uint_as_float(f.row), 0.f);
}

// Pixel region of a warp: 8 x (4 * PPL) pixels, PPL vertically adjacent
// pixels per lane; a 16x16 tile holds 8 / PPL such regions (one per warp).
template <int PPL>
struct Region {
  static constexpr int kH = 4 * PPL;
  static constexpr int kWarps = (BS_TILE * BS_TILE) / (32 * PPL);
  static constexpr int kThreads = 32 * kWarps;
  int px, py0;           // lane's pixels: (px, py0 + k), k < PPL
  float x0, x1, y0, y1;  // pixel-centre extent of the warp's region
  __device__ __forceinline__ Region(int tile_x, int tile_y) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rx = tile_x * BS_TILE + (w & 1) * 8, ry = tile_y * BS_TILE + (w >> 1) * kH;
    px = rx + (lane & 7);
    py0 = ry + PPL * (lane >> 3);
    x0 = (float)rx + 0.5f;
    x1 = x0 + 7.f;
    y0 = (float)ry + 0.5f;
    y1 = y0 + (float)(kH - 1);
  }
};

struct PixelFwd {
  F2 c01;  // (r, g) accumulated
  float T, c2;
  int contrib;
  bool done;
};

__device__ __forceinline__ void blend(PixelFwd& p, const float4& sa, const float4& sb, float cb, float th2, F2 npx,
                                      int rel) {
  F2 d;
  const float power2 = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, npx, d);
  if (power2 > 0.f || power2 < th2) return;
  const float alpha = fminf(kAlphaMax, __fmul_rn(sb.y, ex2_approx(power2)));
  const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
  if (nT < kTMin) {
    p.done = true;
    return;
  }
  const float w = __fmul_rn(alpha, p.T);
  p.c01 = fma2(f2(sb.z, sb.w), bcast(w), p.c01);
  p.c2 = __fmaf_rn(cb, w, p.c2);
  p.T = nT;
  p.contrib = rel + 1;
}

// blend() with one early-out (the support test, mostly warp-uniform) and
// selects for the rest; same arithmetic as blend().
__device__ __forceinline__ bool blend_sel(PixelFwd& p, const float4& sa, const float4& sb, float cb, float th2, F2 npx,
                                          int rel) {
  F2 d;
  const float power2 = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, npx, d);
  if (power2 > 0.f || power2 < th2) return false;
  const float alpha = fminf(kAlphaMax, __fmul_rn(sb.y, ex2_approx(power2)));
  const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
  const bool fin = nT < kTMin;
  const bool c = !fin;
  const float w = __fmul_rn(alpha, p.T);
  const F2 c01 = fma2(f2(sb.z, sb.w), bcast(w), p.c01);
  const float c2 = __fmaf_rn(cb, w, p.c2);
  p.done = p.done || fin;
  p.c01 = c ? c01 : p.c01;
  p.c2 = c ? c2 : p.c2;
  p.T = c ? nT : p.T;
  p.contrib = c ? rel + 1 : p.contrib;
  return c;
}

// blend_sel without any branch (done pixels and pairs outside the support
// keep their state through selects); same arithmetic for a blended pair.
__device__ __forceinline__ bool blend_pred(PixelFwd& p, const float4& sa, const float4& sb, float cb, float th2, F2 npx,
                                           int rel) {
  F2 d;
  const float power2 = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, npx, d);
  const bool in = !p.done && !(power2 > 0.f || power2 < th2);
  const float alpha = fminf(kAlphaMax, __fmul_rn(sb.y, ex2_approx(fminf(power2, 0.f))));
  const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
  const bool fin = nT < kTMin;
  const bool c = in && !fin;
  const float w = __fmul_rn(alpha, p.T);
  const F2 c01 = fma2(f2(sb.z, sb.w), bcast(w), p.c01);
  const float c2 = __fmaf_rn(cb, w, p.c2);
  p.done = p.done || (in && fin);
  p.c01 = c ? c01 : p.c01;
  p.c2 = c ? c2 : p.c2;
  p.T = c ? nT : p.T;
  p.contrib = c ? rel + 1 : p.contrib;
  return c;
}

template <int PPL>
__device__ __forceinline__ bool all_done(const PixelFwd (&p)[PPL]) {
  bool d = true;
#pragma unroll
  for (int k = 0; k < PPL; ++k) d = d && p[k].done;
  return d;
}

template <int PPL, bool kPatches, bool kSup>
__global__ void __launch_bounds__(Region<PPL>::kThreads) raster_fwd_kernel(
    RastArgs a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    float* __restrict__ image, float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
    const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view, float* __restrict__ loss_tiles) {
  constexpr int kW = Region<PPL>::kWarps;
  __shared__ WarpSmemF smem[kW];
  __shared__ float s_red[kW];
  const int slot = blockIdx.z;
  const int tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmemF& s = smem[w];
  const Region<PPL> q(blockIdx.x, blockIdx.y);
  const float pxf = (float)q.px + 0.5f;
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  PixelFwd p[PPL];
#pragma unroll
  for (int k = 0; k < PPL; ++k)
    p[k] = PixelFwd{f2(0.f, 0.f), 1.f, 0.f, 0,
                    !(kPatches ? slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, q.px, q.py0 + k)
                               : (q.px < a.W && q.py0 + k < a.H))};
  Splat f;
  const float* sup = kSup ? a.support : nullptr;  // kSup: per-row support thresholds given
  fetch_splat(f, sp, sup, inst_rows, rg.x + lane, rg.x + lane < rg.y);
  uint32_t row_next = fetch_row(inst_rows, rg.x + 32 + lane, rg.x + 32 + lane < rg.y);
#ifdef BS_RASTER_STATS
  unsigned long long fst[3] = {0, 0, 0};
#endif
  for (int b0 = rg.x; b0 < rg.y; b0 += 32) {
    if (__all_sync(0xffffffffu, all_done<PPL>(p))) break;
    const bool keep = reaches(f, q.x0, q.x1, q.y0, q.y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
#ifdef BS_RASTER_STATS
    fst[0]++;
    fst[1] += __popc(bits);
#endif
    if (keep) stage(s, lane, f, kSup);
    fetch_row_data(f, sp, sup, row_next, b0 + 32 + lane < rg.y);
    row_next = fetch_row(inst_rows, b0 + 64 + lane, b0 + 64 + lane < rg.y);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      const float4 sa = s.a[j];
      const float4 sb = s.b[j];
      const float2 sc = s.c[j];
      const int rel = b0 + j - rg.x;
      if constexpr (PPL == 1) {
#ifdef BS_RASTER_STATS
        {
          F2 dd;
          const float pw = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, f2(-pxf, -((float)q.py0 + 0.5f)), dd);
          fst[2] += __popc(__ballot_sync(__activemask(), !p[0].done && !(pw > 0.f || pw < sc.y)));
        }
#endif
        if (!p[0].done) blend_sel(p[0], sa, sb, sc.x, sc.y, f2(-pxf, -((float)q.py0 + 0.5f)), rel);
      } else {
#pragma unroll
        for (int k = 0; k < PPL; ++k)
          if (!p[k].done) blend(p[k], sa, sb, sc.x, sc.y, f2(-pxf, -((float)(q.py0 + k) + 0.5f)), rel);
      }
    }
    __syncwarp();
  }
#ifdef BS_RASTER_STATS
  if (lane == 0)
    for (int k = 0; k < 3; ++k) atomicAdd(&g_rstats[48 + k], fst[k]);
#endif
  float l = 0.f;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    if (!(kPatches ? slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, q.px, q.py0 + k)
                   : (q.px < a.W && q.py0 + k < a.H)))
      continue;
    const int64_t pix = ((int64_t)slot * a.H + q.py0 + k) * a.W + q.px;
    const float2 c01 = unf2(p[k].c01);
    const float o0 = c01.x + p[k].T * a.bg[0], o1 = c01.y + p[k].T * a.bg[1], o2 = p[k].c2 + p[k].T * a.bg[2];
    image[3 * pix] = o0;
    image[3 * pix + 1] = o1;
    image[3 * pix + 2] = o2;
    final_T[pix] = p[k].T;
    n_contrib[pix] = p[k].contrib;
    if (a.loss_fused) {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + q.py0 + k) * a.W + q.px);
      l += fabsf(o0 - gp[0] * (1.f / 255.f)) + fabsf(o1 - gp[1] * (1.f / 255.f)) + fabsf(o2 - gp[2] * (1.f / 255.f));
    }
  }
  if (a.loss_fused) {
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) s_red[w] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int k = 0; k < kW; ++k) t += s_red[k];
      loss_tiles[(int64_t)slot * a.tiles_per_slot + tile] = t;
    }
  }
}

// Reduce-scatter of 9 per-lane values over the warp in 12 shuffles.  Returns
// the full warp sum of value `out_idx` in lanes where out_idx >= 0 (even
// lanes; every index 0..8 appears in exactly one even lane).
__device__ __forceinline__ float warp_reduce9(const float v[9], int& out_idx) {
  const int lane = threadIdx.x & 31;
  // step 1 (xor 16): lower half keeps values 0..4, upper half 5..8 (+pad)
  const bool u16 = lane & 16;
  float a[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const float hi = i < 4 ? v[5 + i] : 0.f;
    const float send = u16 ? v[i] : hi;
    const float mine = u16 ? hi : v[i];
    a[i] = mine + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  // step 2 (xor 8): positions 0..2 | 3..4
  const bool u8 = lane & 8;
  float b[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float hi = i < 2 ? a[3 + i] : 0.f;
    const float send = u8 ? a[i] : hi;
    const float mine = u8 ? hi : a[i];
    b[i] = mine + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  // step 3 (xor 4): positions 0..1 | 2
  const bool u4 = lane & 4;
  float c[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float hi = i < 1 ? b[2 + i] : 0.f;
    const float send = u4 ? b[i] : hi;
    const float mine = u4 ? hi : b[i];
    c[i] = mine + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  // step 4 (xor 2): position 0 | 1
  const bool u2 = lane & 2;
  const float send = u2 ? c[0] : c[1];
  const float mine = u2 ? c[1] : c[0];
  float d = mine + __shfl_xor_sync(0xffffffffu, send, 2);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  // lane bits (b4 b3 b2 b1) -> value index (see the split sequence above)
  constexpr uint64_t kMap = 0xFFF8F765FF43F210ull;  // nibble per (lane >> 1); F = none
  const int nib = (int)((kMap >> (4 * (lane >> 1))) & 0xF);
  out_idx = ((lane & 1) == 0 && nib != 0xF) ? nib : -1;
  return d;
}

struct PixelBwd {
  float2 acc01;  // colour behind the current splat (r, g), normalised
  F2 dC01;       // dL/dC (r, g)
  float T, T_final, dC2, acc2, bgdot;
  int n;
};

// Gradient contribution of one splat at one pixel.  kAssign: writes all 9
// terms of g when it returns true (g untouched otherwise); else adds into g.
// acc = colour blended behind this splat, normalised by the transmittance
// in front of it: acc' = acc + alpha (c - acc) after the splat.  kBg: the
// background is not black (adds its transmittance term to dL/dalpha).
template <bool kAssign, bool kBg>
__device__ __forceinline__ bool pixel_grad(PixelBwd& p, const float4& sa, const float4& sb, float cb, float th2, F2 npx,
                                           float g[9]) {
  F2 d;
  const float power2 = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, npx, d);
  if (power2 > 0.f || power2 < th2) return false;
  const float ex = ex2_approx(power2);
  const float raw = __fmul_rn(sb.y, ex);
  const float alpha = fminf(kAlphaMax, raw);
  const float ra = rcp_approx(1.f - alpha);  // alpha <= 0.99
  p.T = p.T * ra;
  const float fac = alpha * p.T;
  const F2 e01 = add2(f2(sb.z, sb.w), f2(-p.acc01.x, -p.acc01.y));
  const float e2 = cb - p.acc2;
  const float2 ed = unf2(mul2(e01, p.dC01));
  float dL_dalpha = p.T * fmaf(e2, p.dC2, ed.x + ed.y);
  if (kBg) dL_dalpha -= p.T_final * ra * p.bgdot;
  p.acc01 = unf2(fma2(bcast(alpha), e01, f2(p.acc01.x, p.acc01.y)));
  p.acc2 = fmaf(alpha, e2, p.acc2);
  // clamped alpha (raw > 0.99): colour gradient only.  G_SP carries the
  // moments of dL/dpower (power = -q/2) over the pixels; the projection
  // backward applies the conic (include/splat_b200.h, G_SP row).
  const float dpow = raw > kAlphaMax ? 0.f : dL_dalpha * alpha;  // dL / d power
  const float2 t01 = unf2(mul2(bcast(dpow), d));     // dpow (dx, dy)
  const float2 t34 = unf2(mul2(bcast(t01.x), d));    // dpow dx (dx, dy)
  const float2 t67 = unf2(mul2(bcast(fac), p.dC01));
  float t[9];
  t[0] = t01.x;
  t[1] = t01.y;
  t[2] = raw > kAlphaMax ? 0.f : dL_dalpha * ex;
  t[3] = t34.x;
  t[4] = t34.y;
  t[5] = t01.y * unf2(d).y;
  t[6] = t67.x;
  t[7] = t67.y;
  t[8] = fac * p.dC2;
#pragma unroll
  for (int k = 0; k < 9; ++k) g[k] = kAssign ? t[k] : g[k] + t[k];
  return true;
}

// pixel_grad<true, kBg> without branches (one pixel per lane): every lane
// runs the whole sequence and the pixels the splat does not touch (or that lie
// past their last contributor: live == false) keep their state through
// selects and return zero terms.  The arithmetic of a contributing pixel is
// the same instruction sequence as pixel_grad's, so the results are identical;
// what goes is the divergent-branch bookkeeping (BSSY/BSYNC, three branches
// and their reconvergence stalls) in the hottest loop of the backward.
// The per-pair math in two halves: pair_front depends only on the splat
// and the pixel (independent of the back-to-front recurrence, so a loop can
// evaluate the next splat's front while the current one's tail and
// reduction run); pair_back advances the pixel's T / acc and writes the 9
// gradient terms.  pixel_grad_sel = front + support test + back.
struct PairFront {
  F2 d;
  float power2, ex, raw, alpha, ra;
};

__device__ __forceinline__ void pair_front(PairFront& f, const float4& sa, const float4& sb, F2 npx) {
  f.power2 = splat_power2(f2(sa.x, sa.y), f2(sa.z, sa.w), sb.x, npx, f.d);
  f.ex = ex2_approx(fminf(f.power2, 0.f));
  f.raw = __fmul_rn(sb.y, f.ex);
  f.alpha = fminf(kAlphaMax, f.raw);
  f.ra = rcp_approx(1.f - f.alpha);  // alpha <= 0.99
}

template <bool kBg>
__device__ __forceinline__ void pair_back(PixelBwd& p, const PairFront& f, const float4& sb, float cb, bool ok,
                                          float g[9]) {
  const float T = p.T * f.ra;
  const float fac = f.alpha * T;
  const F2 e01 = add2(f2(sb.z, sb.w), f2(-p.acc01.x, -p.acc01.y));
  const float e2 = cb - p.acc2;
  const float2 ed = unf2(mul2(e01, p.dC01));
  float dL_dalpha = T * fmaf(e2, p.dC2, ed.x + ed.y);
  if (kBg) dL_dalpha -= p.T_final * f.ra * p.bgdot;
  const float2 acc01 = unf2(fma2(bcast(f.alpha), e01, f2(p.acc01.x, p.acc01.y)));
  const float acc2 = fmaf(f.alpha, e2, p.acc2);
  p.T = ok ? T : p.T;
  p.acc01 = ok ? acc01 : p.acc01;
  p.acc2 = ok ? acc2 : p.acc2;
  const bool grad = ok && !(f.raw > kAlphaMax);
  const float dpow = grad ? dL_dalpha * f.alpha : 0.f;  // dL / d power
  const float2 t01 = unf2(mul2(bcast(dpow), f.d));
  const float2 t34 = unf2(mul2(bcast(t01.x), f.d));
  const float2 t67 = unf2(mul2(bcast(ok ? fac : 0.f), p.dC01));
  g[0] = t01.x;
  g[1] = t01.y;
  g[2] = grad ? dL_dalpha * f.ex : 0.f;
  g[3] = t34.x;
  g[4] = t34.y;
  g[5] = t01.y * unf2(f.d).y;
  g[6] = t67.x;
  g[7] = t67.y;
  g[8] = (ok ? fac : 0.f) * p.dC2;
}

template <bool kBg>
__device__ __forceinline__ bool pixel_grad_sel(PixelBwd& p, const float4& sa, const float4& sb, float cb, float th2,
                                               F2 npx, bool live, float g[9]) {
  PairFront f;
  pair_front(f, sa, sb, npx);
  const bool ok = live && !(f.power2 > 0.f || f.power2 < th2);
  pair_back<kBg>(p, f, sb, cb, ok, g);
  return ok;
}

__device__ __forceinline__ void init_pixel_bwd(PixelBwd& q, const RastArgs& a, int slot, int px, int py, bool inside,
                                               const float* __restrict__ image, const float* __restrict__ final_T,
                                               const int32_t* __restrict__ n_contrib,
                                               const float* __restrict__ grad_image, const uint8_t* __restrict__ gt,
                                               const int32_t* __restrict__ gt_view) {
  q.T = 1.f;
  q.n = 0;
  float dC0 = 0.f, dC1 = 0.f;
  q.dC2 = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    q.T = final_T[pix];
    q.n = n_contrib[pix];
    if (grad_image) {
      dC0 = grad_image[3 * pix];
      dC1 = grad_image[3 * pix + 1];
      q.dC2 = grad_image[3 * pix + 2];
    } else {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
      const float d0 = image[3 * pix] - gp[0] * (1.f / 255.f);
      const float d1 = image[3 * pix + 1] - gp[1] * (1.f / 255.f);
      const float d2 = image[3 * pix + 2] - gp[2] * (1.f / 255.f);
      dC0 = (d0 > 0.f ? 1.f : (d0 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      dC1 = (d1 > 0.f ? 1.f : (d1 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      q.dC2 = (d2 > 0.f ? 1.f : (d2 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    }
  }
  q.T_final = q.T;
  q.dC01 = f2(dC0, dC1);
  q.bgdot = a.bg[0] * dC0 + a.bg[1] * dC1 + a.bg[2] * q.dC2;
  q.acc01 = make_float2(0.f, 0.f);
  q.acc2 = 0.f;
}

template <int PPL, bool kBg, bool kSup>
__global__ void __launch_bounds__(Region<PPL>::kThreads, (PPL == 1 ? 1024 : 768) / Region<PPL>::kThreads) raster_bwd_kernel(
    RastArgs a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    const float* __restrict__ image, const float* __restrict__ final_T, const int32_t* __restrict__ n_contrib,
    const float* __restrict__ grad_image, const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view,
    float* __restrict__ g_sp) {
  constexpr int kW = Region<PPL>::kWarps;
  __shared__ WarpSmem smem[kW];
  const int slot = blockIdx.z;
  const int tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem& s = smem[w];
  const Region<PPL> q(blockIdx.x, blockIdx.y);
  const float pxf = (float)q.px + 0.5f;
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  PixelBwd p[PPL];
  int warp_n = 0;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    init_pixel_bwd(p[k], a, slot, q.px, q.py0 + k,
                   slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, q.px, q.py0 + k), image, final_T, n_contrib,
                   grad_image, gt, gt_view);
    warp_n = max(warp_n, p[k].n);
  }
  for (int o = 16; o > 0; o >>= 1) warp_n = max(warp_n, __shfl_xor_sync(0xffffffffu, warp_n, o));
  const int end = rg.x + warp_n;  // deepest contributor of this warp's pixels
  Splat f;
  const float* sup = kSup ? a.support : nullptr;  // kSup: per-row support thresholds given
  fetch_splat(f, sp, sup, inst_rows, end - 1 - lane, end - 1 - lane >= rg.x);
  uint32_t row_next = fetch_row(inst_rows, end - 33 - lane, end - 33 - lane >= rg.x);
  // chunks back to front; within a chunk lane j holds instance cend - 1 - j
#ifdef BS_RASTER_STATS
  unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long hist[33];
  for (int k = 0; k < 33; ++k) hist[k] = 0;
#endif
  for (int cend = end; cend > rg.x; cend -= 32) {
    const bool keep = reaches(f, q.x0, q.x1, q.y0, q.y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
#ifdef BS_RASTER_STATS
    st[0]++;
    st[1] += __popc(bits);
#endif
    if (keep) stage(s, lane, f, kSup);
    fetch_row_data(f, sp, sup, row_next, cend - 33 - lane >= rg.x);
    row_next = fetch_row(inst_rows, cend - 65 - lane, cend - 65 - lane >= rg.x);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      const int rel = cend - 1 - j - rg.x;  // range-relative index of this splat
      float g[9];
      const float4 sa = s.s[j].a;
      const float4 sb = s.s[j].b;
      const float4 sc = s.s[j].c;
      bool any = false;
      if constexpr (PPL == 1) {
        any = pixel_grad_sel<kBg>(p[0], sa, sb, sc.x, sc.y, f2(-pxf, -((float)q.py0 + 0.5f)), rel < p[0].n, g);
      } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) g[k] = 0.f;
#pragma unroll
        for (int k = 0; k < PPL; ++k)
          if (rel < p[k].n)
            any |= pixel_grad<false, kBg>(p[k], sa, sb, sc.x, sc.y, f2(-pxf, -((float)(q.py0 + k) + 0.5f)), g);
      }
      const uint32_t who = __ballot_sync(0xffffffffu, any);
#ifdef BS_RASTER_STATS
      st[2] += who == 0u;
      st[3] += who != 0u && __popc(who) <= kSparseLanes;
      st[4] += __popc(who) > kSparseLanes;
      st[5] += __popc(who);
      st[6] += __popc(__ballot_sync(0xffffffffu, rel < p[0].n));
      hist[__popc(who)]++;
#endif
      if (who == 0u) continue;
      float* dst = g_sp + (int64_t)__float_as_uint(sc.z) * BS_GSP_FLOATS;
#ifdef BS_BWD_NO_REDUCE
      // tuning probe only (tools/gpu_probe_reduce.sh): the gradient terms are
      // computed but not reduced -- the upper bound of any reduction scheme
      if (g[0] + g[1] + g[2] + g[3] + g[4] + g[5] + g[6] + g[7] + g[8] == 1.2345e-30f) atomicAdd(dst, 1.f);
      continue;
#endif
      if (__popc(who) <= kSparseLanes) {
        if (any) {
#if BS_GSP_FLOATS == 12
          // 16-byte aligned rows: two 128-bit REDs + one scalar
          atomicAdd(reinterpret_cast<float4*>(dst), make_float4(g[0], g[1], g[2], g[3]));
          atomicAdd(reinterpret_cast<float4*>(dst + 4), make_float4(g[4], g[5], g[6], g[7]));
          atomicAdd(dst + 8, g[8]);
#else
#pragma unroll
          for (int k = 0; k < 9; ++k) atomicAdd(dst + k, g[k]);
#endif
        }
      } else {  // g is zero in the lanes without a contribution
        int idx;
        const float r = warp_reduce9(g, idx);
        if (idx >= 0) atomicAdd(dst + idx, r);
      }
    }
    __syncwarp();
  }
#ifdef BS_RASTER_STATS
  if (lane == 0) {
    for (int k = 0; k < 7; ++k) atomicAdd(&g_rstats[k], st[k]);
    for (int k = 0; k < 33; ++k)
      if (hist[k]) atomicAdd(&g_rstats[8 + k], hist[k]);
  }
#endif
}

// ---- K3 + L + K4 in one kernel (the mean-L1 training step) ----------------
//
// raster_fwd_kernel and raster_bwd_kernel walk the same depth-sorted tile
// list with the same per-warp support filter; the backward repeats the
// forward's chunk work (row gathers, support test, ballot, staging) and
// re-reads every pixel's T, n_contrib, colour and ground truth.  Fused, each
// warp stages the forward's kept splats as 48-byte records in a warp-private
// shared-memory list, blends them (predicated, no branch per pair), stores
// in each record the ballot of the lanes it was blended into, drops the
// records blended into no pixel after every chunk, turns its pixels' final
// colours straight into dL/dC (L1 sign), and walks the list back to front,
// two records per iteration, the mask standing in for the support and
// contributor tests: no gathers, no per-pixel reloads.  A warp that keeps
// more than kKeep splats (the list overflows) falls back to the backward's
// own chunked walk over global memory.  Per pair the arithmetic is
// raster_fwd_kernel's / raster_bwd_kernel's, so the image is identical and
// the gradients differ only by atomic order.
#ifndef BS_FUSED_KEEP
#define BS_FUSED_KEEP 128  // swept on B200 (C2 raster ms): 64 2.93, 128 2.61, 256 (2 CTAs) 5.5; separate kernels 2.93
#endif
#ifndef BS_FUSED_CTAS
#define BS_FUSED_CTAS 4
#endif
#ifndef BS_FUSED_PAIR_MERGE
#define BS_FUSED_PAIR_MERGE 1  // A/B on B200 (C2 raster): 0 2.474, 1 (sparse pairs) 2.443, 2 (all disjoint pairs) 2.456 ms;
                               // the record of each lane's splat re-read per lane instead of selected: 2.464
#endif
#ifndef BS_FUSED_FWD_SEL
#define BS_FUSED_FWD_SEL 1  // A/B on B200 (C2 raster): branchy 2.545, predicated 2.484 ms
#endif
constexpr int kKeep = BS_FUSED_KEEP;  // kept-splat records per warp (48 B each)

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

struct KeptRec {
  float4 a, b, c;  // as Staged; c.w = the lanes the forward blended the splat into (written after its blend)
};

// the reduction of one splat's 9 terms over the warp into its G_SP row:
// `who` = the contributing lanes (non-zero), `any` = this lane's bit
__device__ __forceinline__ void reduce_splat(const float g[9], uint32_t who, bool any, float* __restrict__ dst) {
  if (__popc(who) <= kSparseLanes) {
    if (any) {
      atomicAdd(reinterpret_cast<float4*>(dst), make_float4(g[0], g[1], g[2], g[3]));
      atomicAdd(reinterpret_cast<float4*>(dst + 4), make_float4(g[4], g[5], g[6], g[7]));
      atomicAdd(dst + 8, g[8]);
    }
  } else {
    int idx;
    const float r = warp_reduce9(g, idx);
    if (idx >= 0) atomicAdd(dst + idx, r);
  }
}

// one kept splat of the fused backward from its record (c.w = the lanes the
// forward blended it into, never 0 in the compacted list)
template <bool kBg>
__device__ __forceinline__ void bwd_rec(PixelBwd& p, const PairFront& fr, const float4& sb, const float4& sc,
                                        float* __restrict__ g_sp) {
  const uint32_t who = __float_as_uint(sc.w);
  const bool any = (who >> (threadIdx.x & 31)) & 1u;
  float g[9];
  pair_back<kBg>(p, fr, sb, sc.x, any, g);
  reduce_splat(g, who, any, g_sp + (int64_t)__float_as_uint(sc.z) * BS_GSP_FLOATS);
}

// one splat of the backward for one warp: pixel gradient + warp reduction + REDs
template <bool kBg>
__device__ __forceinline__ void bwd_splat(PixelBwd& p, const float4& sa, const float4& sb, const float4& sc, int rel,
                                          F2 npx, float* __restrict__ g_sp) {
  float g[9];
  const bool any = pixel_grad_sel<kBg>(p, sa, sb, sc.x, sc.y, npx, rel < p.n, g);
  const uint32_t who = __ballot_sync(0xffffffffu, any);
  if (who == 0u) return;
  float* dst = g_sp + (int64_t)__float_as_uint(sc.z) * BS_GSP_FLOATS;
  if (__popc(who) <= kSparseLanes) {
    if (any) {
      atomicAdd(reinterpret_cast<float4*>(dst), make_float4(g[0], g[1], g[2], g[3]));
      atomicAdd(reinterpret_cast<float4*>(dst + 4), make_float4(g[4], g[5], g[6], g[7]));
      atomicAdd(dst + 8, g[8]);
    }
  } else {
    int idx;
    const float r = warp_reduce9(g, idx);
    if (idx >= 0) atomicAdd(dst + idx, r);
  }
}

template <bool kBg, bool kSup>
__global__ void __launch_bounds__(256, BS_FUSED_CTAS) raster_fused_kernel(
    RastArgs a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    float* __restrict__ image, float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
    const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view, float* __restrict__ loss_tiles,
    float* __restrict__ g_sp) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  __shared__ float s_red[8];
  const int slot = blockIdx.z;
  const int tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  KeptRec* kept = reinterpret_cast<KeptRec*>(s_dyn) + w * kKeep;
  const Region<1> q(blockIdx.x, blockIdx.y);
  const float pxf = (float)q.px + 0.5f;
  const F2 npx = f2(-pxf, -((float)q.py0 + 0.5f));
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  const bool inside = slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, q.px, q.py0);
  // ---------------- forward: blend front to back, appending the kept splats
  PixelFwd pf{f2(0.f, 0.f), 1.f, 0.f, 0, !inside};
  Splat f;
  const float* sup = kSup ? a.support : nullptr;
  fetch_splat(f, sp, sup, inst_rows, rg.x + lane, rg.x + lane < rg.y);
  uint32_t row_next = fetch_row(inst_rows, rg.x + 32 + lane, rg.x + 32 + lane < rg.y);
  int nk = 0;  // kept records appended (warp-uniform)
  for (int b0 = rg.x; b0 < rg.y; b0 += 32) {
    if (__all_sync(0xffffffffu, pf.done)) break;
    const bool keep = reaches(f, q.x0, q.x1, q.y0, q.y1);
    const uint32_t bits = __ballot_sync(0xffffffffu, keep);
    const int nb = __popc(bits);
    // records of a chunk are contiguous: a list that would run past kKeep is
    // abandoned (the backward falls back) and its chunks are staged at 0
    KeptRec* const rk = kept + (nk + nb <= kKeep ? nk : 0);
    if (keep) {
      KeptRec& r = rk[__popc(bits & ((1u << lane) - 1u))];
      r.a = make_float4(f.p0.x, f.p0.y, __fmul_rn(f.p0.w, kHalfLog2e), __fmul_rn(f.p1.y, kHalfLog2e));
      r.b = make_float4(__fmul_rn(f.p1.x, -kLog2e), f.p0.z, f.p1.z, f.p1.w);
      r.c = make_float4(f.b, kSup ? f.th2 : support_p2(f.p0.z), __uint_as_float(f.row), 0.f);  // c.w: the mask
    }
    fetch_row_data(f, sp, sup, row_next, b0 + 32 + lane < rg.y);
    row_next = fetch_row(inst_rows, b0 + 64 + lane, b0 + 64 + lane < rg.y);
    __syncwarp();
    // explicit shared-space addresses: the three record loads stay together
    // ahead of the per-pixel branch, and the address is one add per splat
    uint32_t ra = (uint32_t)__cvta_generic_to_shared(rk);
    uint32_t rest = bits;  // staging lanes of the records still to blend: record k came from lane ffs(rest) - 1
    for (int k = 0; k < nb; ++k, ra += (uint32_t)sizeof(KeptRec)) {
      // c.w is not read here: lane 0 writes the record's mask into it below
      const float4 sa = lds128(ra), sb = lds128(ra + 16);
      const float2 sc = lds64(ra + 32);
      const int rel = b0 + __ffs(rest) - 1 - rg.x;  // range-relative index of the splat
      rest &= rest - 1u;
#if BS_FUSED_FWD_SEL
      const bool blended = blend_pred(pf, sa, sb, sc.x, sc.y, npx, rel);
#else
      bool blended = false;
      if (!pf.done) blended = blend_sel(pf, sa, sb, sc.x, sc.y, npx, rel);
#endif
      // the pixels this splat was blended into: exactly the pairs the backward
      // differentiates (rel < n_contrib and inside the support).  (Keeping
      // the masks in registers until the chunk ends measured slower: spills.)
      const uint32_t who = __ballot_sync(0xffffffffu, blended);
      if (lane == 0) sts32(ra + 44, who);
    }
    __syncwarp();
    if (nk + nb <= kKeep) {
      // drop the chunk's records blended into no pixel: the backward's list
      // holds contributing splats only (lane j moves record j)
      KeptRec r;
      if (lane < nb) r = rk[lane];
      const bool live = lane < nb && __float_as_uint(r.c.w) != 0u;
      const uint32_t lb = __ballot_sync(0xffffffffu, live);
      __syncwarp();
      if (live) rk[__popc(lb & ((1u << lane) - 1u))] = r;
      nk += __popc(lb);
      __syncwarp();
    } else {
      nk = kKeep + 1;  // the list overflowed: the backward takes the chunked walk
    }
  }
  // outputs + loss partial + this pixel's L1 gradient
  float l = 0.f;
  PixelBwd p;
  p.T = 1.f;
  p.n = 0;
  float dC0 = 0.f, dC1 = 0.f;
  p.dC2 = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + q.py0) * a.W + q.px;
    const float2 c01 = unf2(pf.c01);
    const float o0 = c01.x + pf.T * a.bg[0], o1 = c01.y + pf.T * a.bg[1], o2 = pf.c2 + pf.T * a.bg[2];
    image[3 * pix] = o0;
    image[3 * pix + 1] = o1;
    image[3 * pix + 2] = o2;
    if (final_T) final_T[pix] = pf.T;
    if (n_contrib) n_contrib[pix] = pf.contrib;
    const int gv = gt_view ? gt_view[slot] : slot;
    const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + q.py0) * a.W + q.px);
    const float d0 = o0 - gp[0] * (1.f / 255.f), d1 = o1 - gp[1] * (1.f / 255.f), d2 = o2 - gp[2] * (1.f / 255.f);
    l = fabsf(d0) + fabsf(d1) + fabsf(d2);
    dC0 = (d0 > 0.f ? 1.f : (d0 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    dC1 = (d1 > 0.f ? 1.f : (d1 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    p.dC2 = (d2 > 0.f ? 1.f : (d2 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    p.T = pf.T;
    p.n = pf.contrib;
  }
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) s_red[w] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += s_red[k];
    loss_tiles[(int64_t)slot * a.tiles_per_slot + tile] = t;
  }
  p.T_final = p.T;
  p.dC01 = f2(dC0, dC1);
  p.bgdot = a.bg[0] * dC0 + a.bg[1] * dC1 + a.bg[2] * p.dC2;
  p.acc01 = make_float2(0.f, 0.f);
  p.acc2 = 0.f;
#ifdef BS_RASTER_STATS
  if (lane == 0) {  // [56] lists that wrapped, [57] warps, [58] kept records, [59] > 192, [60] > 256
    atomicAdd(&g_rstats[56], (unsigned long long)(nk > kKeep));
    atomicAdd(&g_rstats[57], 1ull);
    atomicAdd(&g_rstats[58], (unsigned long long)nk);
    atomicAdd(&g_rstats[59], (unsigned long long)(nk > 192));
    atomicAdd(&g_rstats[60], (unsigned long long)(nk > 256));
  }
#endif
  // ---------------- backward: back to front from the deepest contributor
  if (nk <= kKeep) {
    // two records per iteration: the front half of the shallower splat's
    // pair math does not depend on the deeper one's, so it overlaps the
    // deeper splat's tail and reduction
    int k = nk - 1;
    for (; k >= 1; k -= 2) {
      const KeptRec& r1 = kept[k];
      const KeptRec& r0 = kept[k - 1];
      const float4 a1 = r1.a, b1 = r1.b, c1 = r1.c;
      const float4 a0 = r0.a, b0 = r0.b, c0 = r0.c;
#if BS_FUSED_PAIR_MERGE
      const uint32_t m1 = __float_as_uint(c1.w), m0 = __float_as_uint(c0.w);
#if BS_FUSED_PAIR_MERGE >= 2
      if ((m1 & m0) == 0u) {
#else
      if ((m1 & m0) == 0u && __popc(m1) <= kSparseLanes && __popc(m0) <= kSparseLanes) {
#endif
        // two splats on disjoint pixels: one pass of the pair math, each
        // lane on the splat that covers its pixel (the other does not touch
        // the pixel, so their order does not matter for it)
        const bool in1 = (m1 >> lane) & 1u, in0 = (m0 >> lane) & 1u;
        const bool any = in1 || in0;
        const float4 a = in1 ? a1 : a0, b = in1 ? b1 : b0;
        const float cb = in1 ? c1.x : c0.x;
        PairFront f;
        pair_front(f, a, b, npx);
        float g[9];
        pair_back<kBg>(p, f, b, cb, any, g);
#if BS_FUSED_PAIR_MERGE >= 2
        if (__popc(m1) <= kSparseLanes && __popc(m0) <= kSparseLanes) {
#endif
          if (any) {
            float* dst = g_sp + (int64_t)__float_as_uint(in1 ? c1.z : c0.z) * BS_GSP_FLOATS;
            atomicAdd(reinterpret_cast<float4*>(dst), make_float4(g[0], g[1], g[2], g[3]));
            atomicAdd(reinterpret_cast<float4*>(dst + 4), make_float4(g[4], g[5], g[6], g[7]));
            atomicAdd(dst + 8, g[8]);
          }
#if BS_FUSED_PAIR_MERGE >= 2
        } else {
          // each splat's own lanes (a dense one reduces the others' as zero)
          float gm[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) gm[t] = in1 ? g[t] : 0.f;
          reduce_splat(gm, m1, in1, g_sp + (int64_t)__float_as_uint(c1.z) * BS_GSP_FLOATS);
#pragma unroll
          for (int t = 0; t < 9; ++t) gm[t] = in0 ? g[t] : 0.f;
          reduce_splat(gm, m0, in0, g_sp + (int64_t)__float_as_uint(c0.z) * BS_GSP_FLOATS);
        }
#endif
        continue;
      }
#endif
      PairFront f1, f0;
      pair_front(f1, a1, b1, npx);
      pair_front(f0, a0, b0, npx);
      bwd_rec<kBg>(p, f1, b1, c1, g_sp);
      bwd_rec<kBg>(p, f0, b0, c0, g_sp);
    }
    if (k == 0) {
      const KeptRec& r = kept[0];
      const float4 a0 = r.a, b0 = r.b;
      PairFront f0;
      pair_front(f0, a0, b0, npx);
      bwd_rec<kBg>(p, f0, b0, r.c, g_sp);
    }
    return;
  }
  // the list wrapped: the backward's own chunked walk over global memory
  WarpSmem& s = *reinterpret_cast<WarpSmem*>(kept);
  __syncwarp();
  int warp_n = p.n;
  for (int o = 16; o > 0; o >>= 1) warp_n = max(warp_n, __shfl_xor_sync(0xffffffffu, warp_n, o));
  const int end = rg.x + warp_n;
  fetch_splat(f, sp, sup, inst_rows, end - 1 - lane, end - 1 - lane >= rg.x);
  row_next = fetch_row(inst_rows, end - 33 - lane, end - 33 - lane >= rg.x);
  for (int cend = end; cend > rg.x; cend -= 32) {
    const bool keep = reaches(f, q.x0, q.x1, q.y0, q.y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if (keep) stage(s, lane, f, kSup);
    fetch_row_data(f, sp, sup, row_next, cend - 33 - lane >= rg.x);
    row_next = fetch_row(inst_rows, cend - 65 - lane, cend - 65 - lane >= rg.x);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      bwd_splat<kBg>(p, s.s[j].a, s.s[j].b, s.s[j].c, cend - 1 - j - rg.x, npx, g_sp);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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
  a.patch_P = d->patch_P > 0 ? d->patch_P : 1;
  a.slot_patches = d->slot_patches;
  a.support = d->row_support;
  BS_REQUIRE(a.slot_patches == nullptr || (a.patch_P >= 1 && a.patch_P <= 8 && a.W >= a.patch_P && a.H >= a.patch_P),
             BS_ERR_PARAMETER, "patch_P must be in [1, 8] with slot_patches");
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
  auto launch = [&](auto kern, int threads) {
    kern<<<grid, threads, 0, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges), image,
                                                  final_T, n_contrib, gt, gt_slot_view, loss_tiles);
  };
  const bool patches = a.slot_patches != nullptr, sup = a.support != nullptr;
  if (d->pixels_per_lane == 1) {
    if (sup)
      patches ? launch(raster_fwd_kernel<1, true, true>, Region<1>::kThreads)
              : launch(raster_fwd_kernel<1, false, true>, Region<1>::kThreads);
    else
      patches ? launch(raster_fwd_kernel<1, true, false>, Region<1>::kThreads)
              : launch(raster_fwd_kernel<1, false, false>, Region<1>::kThreads);
  } else {
    patches ? launch(raster_fwd_kernel<2, true, false>, Region<2>::kThreads)
            : launch(raster_fwd_kernel<2, false, false>, Region<2>::kThreads);
  }
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
  const bool bg = a.bg[0] != 0.f || a.bg[1] != 0.f || a.bg[2] != 0.f;
  auto launch = [&](auto kern, int threads) {
    kern<<<grid, threads, 0, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges), image,
                                                  final_T, n_contrib, grad_image, gt, gt_slot_view, g_sp);
  };
  const bool sup = a.support != nullptr;
  if (d->pixels_per_lane == 1) {
    if (sup)
      bg ? launch(raster_bwd_kernel<1, true, true>, Region<1>::kThreads)
         : launch(raster_bwd_kernel<1, false, true>, Region<1>::kThreads);
    else
      bg ? launch(raster_bwd_kernel<1, true, false>, Region<1>::kThreads)
         : launch(raster_bwd_kernel<1, false, false>, Region<1>::kThreads);
  } else {
    bg ? launch(raster_bwd_kernel<2, true, false>, Region<2>::kThreads)
       : launch(raster_bwd_kernel<2, false, false>, Region<2>::kThreads);
  }
  BS_LAUNCH_CHECK("raster_bwd_kernel");
  return BS_OK;
}

#ifdef BS_RASTER_STATS
extern "C" int32_t bs_debug_raster_stats(unsigned long long* out, int32_t reset) {
  cudaMemcpyFromSymbol(out, g_rstats, sizeof(g_rstats));
  if (reset) {
    unsigned long long z[64] = {0};
    cudaMemcpyToSymbol(g_rstats, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" int32_t bs_raster_fwd_bwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                     const int32_t* ranges, float* image, float* final_T, int32_t* n_contrib,
                                     const uint8_t* gt, const int32_t* gt_slot_view, float* loss_tiles, float* g_sp,
                                     void* stream) {
  RastArgs a;
  int32_t st = make_args(d, a);
  if (st) return st;
  BS_REQUIRE(gt && loss_tiles && g_sp, BS_ERR_PARAMETER, "raster_fwd_bwd needs gt, loss_tiles and g_sp");
  BS_REQUIRE(d->pixels_per_lane == 1, BS_ERR_PARAMETER, "raster_fwd_bwd: 1 pixel per lane");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  const bool bg = a.bg[0] != 0.f || a.bg[1] != 0.f || a.bg[2] != 0.f;
  const size_t smem = sizeof(KeptRec) * kKeep * 8;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges), image,
                                                 final_T, n_contrib, gt, gt_slot_view, loss_tiles, g_sp);
  };
  const bool sup = a.support != nullptr;
  if (sup)
    bg ? launch(raster_fused_kernel<true, true>) : launch(raster_fused_kernel<false, true>);
  else
    bg ? launch(raster_fused_kernel<true, false>) : launch(raster_fused_kernel<false, false>);
  BS_LAUNCH_CHECK("raster_fused_kernel");
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
  reduce_partials_kernel<<<n_slots, 1024, 0, as_stream(stream)>>>(loss_tiles, n_slots, tiles_per_slot, inv_norm,
                                                                 loss);
  BS_LAUNCH_CHECK("reduce_partials_kernel");
  return BS_OK;
}
