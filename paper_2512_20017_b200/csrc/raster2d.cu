// 2DGS rasterisation (surfel ray-splat intersection, splat2d_math.cuh):
// forward alpha compositing + fused mean-L1 partials, and the backward.
// Same execution scheme as the 3DGS kernels (raster.cu, 1 pixel per lane):
// 16x16 tiles, 8 independent warps per tile each owning an 8x4 pixel
// region, chunks of 32 gathered instances with a register prefetch, a
// per-warp footprint filter, ballot compaction into warp-private shared
// memory.  Per pixel (centre x + 0.5, y + 0.5):
//   h_x = M_row0 - x M_row2, h_y = M_row1 - y M_row2, zeta = h_x x h_y,
//   (u, v) = zeta.xy / zeta.z,  g3 = u^2 + v^2,  g2 = 2 |mean2d - pixel|^2,
//   alpha = min(0.99, opacity exp(-0.5 min(g3, g2))); the pair contributes
// iff min(g3, g2) <= k, k = min(9, 2 ln(255 opacity)) (the 3-sigma cut and
// alpha >= 1/255 as one threshold, as in 3DGS), decided WITHOUT the division:
// g3 <= k <=> zx^2 + zy^2 <= k zz^2, and the disk branch of the min iff
// zx^2 + zy^2 <= g2 zz^2 -- explicit round-to-nearest ops, so the decisions
// are the oracle's bit for bit while u, v use one approximate reciprocal.
// Same stop rule as 3DGS.  Footprint filter: the projection's support box
// (see reaches2).
// Per pixel zeta is affine in the pixel (staging computes it at the region
// origin and its two increments), so the backward accumulates the moments of
// dL/dzeta instead of dL/dM (include/splat_b200.h, 2DGS G_SP row).
// Backward: 15 gradient terms per splat; up to 12 contributing lanes add them
// with four 128-bit REDs each (64-byte aligned G_SP rows), otherwise they are reduce-scattered over the warp in 16
// shuffles and one RED per term is issued per (region, splat).  exp is one
// ex2.approx in both kernels (identical skip / stop decisions).
#include "splat2d_math.cuh"
#include "packed.cuh"

namespace bs {
namespace {

constexpr int kW2 = 8;  // warps per 16x16 tile (8x4 region each)
constexpr int kT2 = 32 * kW2;
constexpr float kAMax = 0.99f;
constexpr float kTStop = 1e-4f;
constexpr float kLog2e2 = 1.4426950408889634f;
#ifndef BS_SPARSE2_LANES
#define BS_SPARSE2_LANES 9  // re-swept on the fused kernel (C3 raster ms): 5 6.73, 7 6.53, 9 6.50, 12 6.57, 16 6.84
#endif
#ifndef BS_R2_FWD_CTAS
#define BS_R2_FWD_CTAS 4
#endif
#ifndef BS_R2_BWD_CTAS
#define BS_R2_BWD_CTAS 3
#endif
constexpr int kSparse2 = BS_SPARSE2_LANES;  // contributing lanes handled with direct REDs

__device__ __forceinline__ float ex2a(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rcpa(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct R2Args {
  int n_slots, tiles_per_slot, W, H, tiles_x;
  float bg[3];
  int loss_fused;
  float inv_norm;
  int patch_P;
  const uint64_t* slot_patches;  // NULL: every pixel
  const float* support;          // per-row support threshold k (bs_row_support) or NULL
};

// Patch restriction (P > 1): does this slot render pixel (x, y)?  Patch c of
// an image side spans [floor(c W / P), floor((c + 1) W / P)).
__device__ __forceinline__ bool slot_pixel(const uint64_t* slot_patches, int P, int W, int H, int slot, int x, int y) {
  if (x >= W || y >= H) return false;
  if (slot_patches == nullptr) return true;
  const int pc = ((x + 1) * P - 1) / W, pr = ((y + 1) * P - 1) / H;
  return (slot_patches[slot] >> (pr * P + pc)) & 1ull;
}


// staged splat: a = (u, v, opac, M0), b = (M1..M4), c = (M5..M8), d = (r, g, b, -)
struct Warp2 {
  float4 a[32], b[32], c[32], d[32];
  uint32_t row[32];
};

struct Splat2 {
  float4 p[4];   // SP floats 0..15
  float2 h, c;   // support box half-widths (16, 17) and centre (22, 23)
  float k;       // support threshold (per-row array; else computed at staging)
  uint32_t row;
  bool ok;
};

__device__ __forceinline__ void fetch2_row(Splat2& f, const float* __restrict__ sp, const float* __restrict__ sup,
                                           uint32_t row, bool ok) {
  f.ok = ok;
  if (ok) {
    f.row = row;
    if (sup) f.k = __ldg(sup + row);
    const float4* r4 = reinterpret_cast<const float4*>(sp + (int64_t)row * kSP2);
#pragma unroll
    for (int k = 0; k < 4; ++k) f.p[k] = __ldg(r4 + k);
    f.h = __ldg(reinterpret_cast<const float2*>(sp + (int64_t)row * kSP2 + 16));
    f.c = __ldg(reinterpret_cast<const float2*>(sp + (int64_t)row * kSP2 + 22));
  }
}

__device__ __forceinline__ void fetch2(Splat2& f, const float* __restrict__ sp, const float* __restrict__ sup,
                                       const uint32_t* __restrict__ rows, int idx, bool ok) {
  fetch2_row(f, sp, sup, ok ? __ldg(rows + idx) : 0u, ok);
}

// row index prefetched one chunk ahead of its SP row (no back-to-back dependent gathers)
__device__ __forceinline__ uint32_t row2(const uint32_t* __restrict__ rows, int idx, bool ok) {
  return ok ? __ldg(rows + idx) : 0u;
}

// M rows from the staged layout: r0 = (M0, M1, M2), r1 = (M3, M4, M5), r2 = (M6, M7, M8)
__device__ __forceinline__ void m_rows(const float4& a, const float4& b, const float4& c, float r0[3], float r1[3],
                                       float r2[3]) {
  r0[0] = a.w; r0[1] = b.x; r0[2] = b.y;
  r1[0] = b.z; r1[1] = b.w; r1[2] = c.x;
  r2[0] = c.y; r2[1] = c.z; r2[2] = c.w;
}

// Can the splat's support box (written by the projection: the union of the
// image of the disk u^2 + v^2 <= k and the low-pass circle, k = min(9,
// 2 ln(255 o)); half-widths 0 = never contributes) reach a pixel centre of
// [x0,x1] x [y0,y1]?  Padded like the 3DGS test.
__device__ __forceinline__ bool reaches2(const Splat2& f, float x0, float x1, float y0, float y1) {
  if (!f.ok || !(f.h.x > 0.f)) return false;
  return fabsf(f.c.x - fminf(fmaxf(f.c.x, x0), x1)) <= fmaf(f.h.x, 1.0001f, 1e-3f) &&
         fabsf(f.c.y - fminf(fmaxf(f.c.y, y0), y1)) <= fmaf(f.h.y, 1.0001f, 1e-3f);
}

// Staging: zeta = h_x x h_y is affine in the pixel (h_x = r0 - px r2,
// h_y = r1 - py r2, and r2 x r2 = 0).  Each warp stages zeta at its region
// origin (X, Y) (the per-pixel formula evaluated once, z0 = hx0 x hy0) and
// the increments zb = hy0 x r2, zc = r2 x hx0 of the origin-shifted rows, so
// a pixel needs zeta = z0 + zb ox + zc oy with small exact integer offsets.
// staged (x/y components in aligned register pairs for packed FP32):
//   a = (u, v, opac, z0.z), b = (z0.x, z0.y, zb.x, zb.y),
//   c = (zc.x, zc.y, zb.z, zc.z), d = (r, g, b, -)
__device__ __forceinline__ void cross3(const float a[3], const float b[3], float o[3]) {
  o[0] = __fsub_rn(__fmul_rn(a[1], b[2]), __fmul_rn(a[2], b[1]));
  o[1] = __fsub_rn(__fmul_rn(a[2], b[0]), __fmul_rn(a[0], b[2]));
  o[2] = __fsub_rn(__fmul_rn(a[0], b[1]), __fmul_rn(a[1], b[0]));
}

// stage2's record as four float4 (the fused kernel's kept list)
__device__ __forceinline__ void stage2_rec(const Splat2& f, float X, float Y, bool have_support, float4 (&r)[4]) {
  float r0[3], r1[3], r2[3];
  m_rows(f.p[0], f.p[1], f.p[2], r0, r1, r2);
  float hx[3], hy[3], z0[3], zb[3], zc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    hx[k] = __fsub_rn(r0[k], __fmul_rn(X, r2[k]));
    hy[k] = __fsub_rn(r1[k], __fmul_rn(Y, r2[k]));
  }
  cross3(hx, hy, z0);
  cross3(hy, r2, zb);
  cross3(r2, hx, zc);
  r[0] = make_float4(f.p[0].x, f.p[0].y, f.p[0].z, z0[2]);
  r[1] = make_float4(z0[0], z0[1], zb[0], zb[1]);
  r[2] = make_float4(zc[0], zc[1], zb[2], zc[2]);
  r[3] = make_float4(f.p[3].x, f.p[3].y, f.p[3].z, have_support ? f.k : support_k(f.p[0].z));
}

__device__ __forceinline__ void stage2(Warp2& s, int lane, const Splat2& f, float X, float Y, bool have_support) {
  float r0[3], r1[3], r2[3];
  m_rows(f.p[0], f.p[1], f.p[2], r0, r1, r2);
  float hx[3], hy[3], z0[3], zb[3], zc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    hx[k] = __fsub_rn(r0[k], __fmul_rn(X, r2[k]));
    hy[k] = __fsub_rn(r1[k], __fmul_rn(Y, r2[k]));
  }
  // increments from the origin-shifted rows (small, like the per-pixel
  // formula's operands): (hx - ox r2) x (hy - oy r2) = z0 + ox (hy x r2) + oy (r2 x hx)
  cross3(hx, hy, z0);
  cross3(hy, r2, zb);
  cross3(r2, hx, zc);
  s.a[lane] = make_float4(f.p[0].x, f.p[0].y, f.p[0].z, z0[2]);
  s.b[lane] = make_float4(z0[0], z0[1], zb[0], zb[1]);
  s.c[lane] = make_float4(zc[0], zc[1], zb[2], zc[2]);
  s.d[lane] = make_float4(f.p[3].x, f.p[3].y, f.p[3].z, have_support ? f.k : support_k(f.p[0].z));  // (r, g, b, k)
  s.row[lane] = f.row;
}

struct Eval2 {
  float z[3], iz, u, v, g3, dx, dy, g2, pw2;
  bool ok, in, disk;  // z.z != 0; min(g3, g2) <= k; g3 <= g2 (division-free, exact)
};

// Bit-identical in forward and backward (explicit round-to-nearest ops).
// (ox, oy): the pixel's offset from the region origin (small integers).
__device__ __forceinline__ void eval2(const float4& a, const float4& b, const float4& c, float k, float px, float py,
                                      float ox, float oy, Eval2& e) {
  // (z.x, z.y) as a packed pair; each lane is the same FMA chain as z.z
  const float2 zxy = unf2(fma2(f2(c.x, c.y), bcast(oy), fma2(f2(b.z, b.w), bcast(ox), f2(b.x, b.y))));
  e.z[0] = zxy.x;
  e.z[1] = zxy.y;
  e.z[2] = __fmaf_rn(c.w, oy, __fmaf_rn(c.z, ox, a.w));
  e.ok = e.z[2] != 0.f;
  // one approximate reciprocal (both kernels evaluate it identically); the
  // rest is evaluated for every pixel and discarded when !ok
  e.iz = rcpa(e.ok ? e.z[2] : 1.f);
  const float2 uv = unf2(mul2(f2(e.z[0], e.z[1]), bcast(e.iz)));
  e.u = uv.x;
  e.v = uv.y;
  e.g3 = __fmaf_rn(e.u, e.u, __fmul_rn(e.v, e.v));
  const float2 dd = unf2(add2(f2(a.x, a.y), f2(-px, -py)));
  e.dx = dd.x;
  e.dy = dd.y;
  e.g2 = __fmul_rn(2.f, __fmaf_rn(e.dx, e.dx, __fmul_rn(e.dy, e.dy)));
  // log2 exponent -0.5 log2(e) min(g3, g2): one rounding, the same value as
  // (-0.5 min) * log2(e) (the 0.5 scaling is exact)
  e.pw2 = __fmul_rn(fminf(e.g3, e.g2), -0.5f * kLog2e2);
  const float n3 = __fmaf_rn(e.z[0], e.z[0], __fmul_rn(e.z[1], e.z[1])), zz = __fmul_rn(e.z[2], e.z[2]);
  e.in = e.ok && (n3 <= __fmul_rn(k, zz) || e.g2 <= k);
  e.disk = n3 <= __fmul_rn(e.g2, zz);
}

struct Px2 {
  float T, c0, c1, c2;
  int contrib;
  bool done;
};

__global__ void __launch_bounds__(kT2, BS_R2_FWD_CTAS) raster2d_fwd_kernel(R2Args a, const float* __restrict__ sp,
                                                            const uint32_t* __restrict__ inst_rows,
                                                            const int2* __restrict__ ranges, float* __restrict__ image,
                                                            float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
                                                            const uint8_t* __restrict__ gt,
                                                            const int32_t* __restrict__ gt_view,
                                                            float* __restrict__ loss_tiles) {
  __shared__ Warp2 smem[kW2];
  __shared__ float s_red[kW2];
  const int slot = blockIdx.z, tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Warp2& s = smem[w];
  const int rx = blockIdx.x * BS_TILE + (w & 1) * 8, ry = blockIdx.y * BS_TILE + (w >> 1) * 4;
  const int px = rx + (lane & 7), py = ry + (lane >> 3);
  const float x0 = rx + 0.5f, x1 = x0 + 7.f, y0 = ry + 0.5f, y1 = y0 + 3.f;
  const float pxf = px + 0.5f, pyf = py + 0.5f;
  const float oxf = (float)(lane & 7), oyf = (float)(lane >> 3);  // offset from the region origin (x0, y0)
  const bool inside = slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, px, py);
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  Px2 p{1.f, 0.f, 0.f, 0.f, 0, !inside};
  Splat2 f;
  fetch2(f, sp, a.support, inst_rows, rg.x + lane, rg.x + lane < rg.y);
  uint32_t row_next = row2(inst_rows, rg.x + 32 + lane, rg.x + 32 + lane < rg.y);
  for (int b0 = rg.x; b0 < rg.y; b0 += 32) {
    if (__all_sync(0xffffffffu, p.done)) break;
    const bool keep = reaches2(f, x0, x1, y0, y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if (keep) stage2(s, lane, f, x0, y0, a.support != nullptr);
    fetch2_row(f, sp, a.support, row_next, b0 + 32 + lane < rg.y);
    row_next = row2(inst_rows, b0 + 64 + lane, b0 + 64 + lane < rg.y);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      if (p.done) continue;
      Eval2 e;
      const float4 sa = s.a[j];
      const float4 col = s.d[j];
      eval2(sa, s.b[j], s.c[j], col.w, pxf, pyf, oxf, oyf, e);
      if (!e.in) continue;  // min(g3, g2) > k: outside the support
      // past the support test: selects instead of branches
      const float alpha = fminf(kAMax, __fmul_rn(sa.z, ex2a(e.pw2)));
      const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
      const bool fin = nT < kTStop;
      const bool c = !fin;
      const float wgt = __fmul_rn(alpha, p.T);
      p.done = p.done || fin;
      p.c0 = c ? __fmaf_rn(col.x, wgt, p.c0) : p.c0;
      p.c1 = c ? __fmaf_rn(col.y, wgt, p.c1) : p.c1;
      p.c2 = c ? __fmaf_rn(col.z, wgt, p.c2) : p.c2;
      p.T = c ? nT : p.T;
      p.contrib = c ? b0 + j + 1 - rg.x : p.contrib;
    }
    __syncwarp();
  }
  float l = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    const float o0 = p.c0 + p.T * a.bg[0], o1 = p.c1 + p.T * a.bg[1], o2 = p.c2 + p.T * a.bg[2];
    image[3 * pix] = o0;
    image[3 * pix + 1] = o1;
    image[3 * pix + 2] = o2;
    final_T[pix] = p.T;
    n_contrib[pix] = p.contrib;
    if (a.loss_fused) {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
      l = fabsf(o0 - gp[0] * (1.f / 255.f)) + fabsf(o1 - gp[1] * (1.f / 255.f)) + fabsf(o2 - gp[2] * (1.f / 255.f));
    }
  }
  if (a.loss_fused) {
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) s_red[w] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int k = 0; k < kW2; ++k) t += s_red[k];
      loss_tiles[(int64_t)slot * a.tiles_per_slot + tile] = t;
    }
  }
}

// Reduce-scatter of 16 per-lane values (index 15 padding) in 16 shuffles;
// even lane L ends with the warp sum of value L >> 1.
__device__ __forceinline__ float warp_reduce16(float v[16]) {
  const int lane = threadIdx.x & 31;
  float a[8], b[4], c[2];
  const bool u16 = lane & 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float send = u16 ? v[i] : v[8 + i];
    const float mine = u16 ? v[8 + i] : v[i];
    a[i] = mine + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  const bool u8 = lane & 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = u8 ? a[i] : a[4 + i];
    const float mine = u8 ? a[4 + i] : a[i];
    b[i] = mine + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool u4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = u4 ? b[i] : b[2 + i];
    const float mine = u4 ? b[2 + i] : b[i];
    c[i] = mine + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const bool u2 = lane & 2;
  const float send = u2 ? c[0] : c[1];
  const float mine = u2 ? c[1] : c[0];
  float d = mine + __shfl_xor_sync(0xffffffffu, send, 2);
  return d + __shfl_xor_sync(0xffffffffu, d, 1);
}

struct PxB2 {
  float T, T_final, dC0, dC1, dC2, acc0, acc1, acc2, bgdot;
  int n;
};

// One splat of the 2DGS backward for one warp, in two halves: bwd2_front
// depends only on the splat and the pixel (a loop can evaluate the next
// splat's front while the current one's tail and reduction run);
// bwd2_back advances the pixel's T / acc and writes the 16 gradient terms
// (selects instead of branches: every lane runs the whole sequence, pixels
// without a contribution keep their state and produce zero terms -- the same
// arithmetic as a branchy version for the contributing ones).
struct Front2 {
  Eval2 e;
  float ex, raw, alpha, ra;
};

__device__ __forceinline__ void bwd2_front(Front2& f, const float4& sa, const float4& sb, const float4& sc, float k,
                                           float pxf, float pyf, float oxf, float oyf) {
  eval2(sa, sb, sc, k, pxf, pyf, oxf, oyf, f.e);
  f.ex = ex2a(fminf(f.e.pw2, 0.f));
  f.raw = __fmul_rn(sa.z, f.ex);
  f.alpha = fminf(kAMax, f.raw);
  f.ra = rcpa(1.f - f.alpha);  // alpha <= 0.99
}

template <bool kBg>
__device__ __forceinline__ void bwd2_back(PxB2& q, const Front2& f, const float4& col, bool any, float pxf, float pyf,
                                          float g[16]) {
  {
    const float ra = f.ra;
    const float T = q.T * ra;
    const float fac = any ? f.alpha * T : 0.f;
    g[12] = fac * q.dC0;
    g[13] = fac * q.dC1;
    g[14] = fac * q.dC2;
    g[15] = 0.f;
    // acc = colour behind this splat (normalised); acc' = acc + f.alpha (c - acc)
    const float e0 = col.x - q.acc0, e1 = col.y - q.acc1, e2 = col.z - q.acc2;
    float dLda = T * (e0 * q.dC0 + e1 * q.dC1 + e2 * q.dC2);
    if (kBg) dLda -= q.T_final * ra * q.bgdot;
    q.acc0 = any ? fmaf(f.alpha, e0, q.acc0) : q.acc0;
    q.acc1 = any ? fmaf(f.alpha, e1, q.acc1) : q.acc1;
    q.acc2 = any ? fmaf(f.alpha, e2, q.acc2) : q.acc2;
    q.T = any ? T : q.T;
    const bool grad = any && f.raw <= kAMax;
    const float dpow = dLda * f.alpha;
    g[11] = grad ? dLda * f.ex : 0.f;
    // disk term: power = -0.5 (u^2 + v^2), (u, v) = zeta.xy / zeta.z; G_SP2
    // carries the moments sum gz, sum gz px, sum gz py of dL/dzeta (the
    // projection backward applies the M rows)
    const bool disk = grad && f.e.disk;
    const F2 guv = mul2(f2(f.e.u, f.e.v), bcast(-dpow));  // dL/d(u, v)
    const float2 g_uv = unf2(guv);
    const float iz = f.e.iz;
    const F2 gz01 = mul2(guv, bcast(iz));
    const float gz2 = -(g_uv.x * f.e.u + g_uv.y * f.e.v) * iz;
    const float2 z01 = unf2(gz01);
    const float2 zx = unf2(mul2(gz01, bcast(pxf)));
    const float2 zy = unf2(mul2(gz01, bcast(pyf)));
    g[2] = disk ? z01.x : 0.f;
    g[3] = disk ? z01.y : 0.f;
    g[4] = disk ? gz2 : 0.f;
    g[5] = disk ? zx.x : 0.f;
    g[6] = disk ? zx.y : 0.f;
    g[7] = disk ? gz2 * pxf : 0.f;
    g[8] = disk ? zy.x : 0.f;
    g[9] = disk ? zy.y : 0.f;
    g[10] = disk ? gz2 * pyf : 0.f;
    // low-pass term: power = -(dx^2 + dy^2), dx = u - px
    const bool lp = grad && !disk;
    g[0] = lp ? -2.f * f.e.dx * dpow : 0.f;
    g[1] = lp ? -2.f * f.e.dy * dpow : 0.f;
  }
}

// the reduction of one splat's 15 terms into its G_SP row (`who` non-zero)
__device__ __forceinline__ void reduce2(const float g[16], uint32_t who, bool any, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  if (__popc(who) <= kSparse2) {
    if (any) {
      // 64-byte aligned rows: four 128-bit REDs (the 16th float is padding, g[15] = 0)
#pragma unroll
      for (int k = 0; k < 16; k += 4)
        atomicAdd(reinterpret_cast<float4*>(dst + k), make_float4(g[k], g[k + 1], g[k + 2], g[k + 3]));
    }
  } else {
    const float r = warp_reduce16(const_cast<float*>(g));
    const int idx = lane >> 1;
    if ((lane & 1) == 0 && idx < kGSP2Used) atomicAdd(dst + idx, r);
  }
}

template <bool kBg>
__device__ __forceinline__ void bwd2_splat(PxB2& q, const float4& sa, const float4& sb, const float4& sc,
                                           const float4& col, uint32_t row, int rel, float pxf, float pyf, float oxf,
                                           float oyf, float* __restrict__ g_sp) {
  Front2 f;
  bwd2_front(f, sa, sb, sc, col.w, pxf, pyf, oxf, oyf);
  const bool any = rel < q.n && f.e.in;
  float g[16];
  bwd2_back<kBg>(q, f, col, any, pxf, pyf, g);
  const uint32_t who = __ballot_sync(0xffffffffu, any);
  if (who == 0u) return;
  reduce2(g, who, any, g_sp + (int64_t)row * kGSP2);
}

template <bool kBg>
__global__ void __launch_bounds__(kT2, BS_R2_BWD_CTAS) raster2d_bwd_kernel(
    R2Args a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    const float* __restrict__ image, const float* __restrict__ final_T, const int32_t* __restrict__ n_contrib,
    const float* __restrict__ grad_image, const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view,
    float* __restrict__ g_sp) {
  __shared__ Warp2 smem[kW2];
  const int slot = blockIdx.z, tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Warp2& s = smem[w];
  const int rx = blockIdx.x * BS_TILE + (w & 1) * 8, ry = blockIdx.y * BS_TILE + (w >> 1) * 4;
  const int px = rx + (lane & 7), py = ry + (lane >> 3);
  const float x0 = rx + 0.5f, x1 = x0 + 7.f, y0 = ry + 0.5f, y1 = y0 + 3.f;
  const float pxf = px + 0.5f, pyf = py + 0.5f;
  const float oxf = (float)(lane & 7), oyf = (float)(lane >> 3);  // offset from the region origin (x0, y0)
  const bool inside = slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, px, py);
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  PxB2 q;
  q.T = 1.f;
  q.n = 0;
  q.dC0 = q.dC1 = q.dC2 = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    q.T = final_T[pix];
    q.n = n_contrib[pix];
    if (grad_image) {
      q.dC0 = grad_image[3 * pix];
      q.dC1 = grad_image[3 * pix + 1];
      q.dC2 = grad_image[3 * pix + 2];
    } else {
      const int gv = gt_view ? gt_view[slot] : slot;
      const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
      const float d0 = image[3 * pix] - gp[0] * (1.f / 255.f);
      const float d1 = image[3 * pix + 1] - gp[1] * (1.f / 255.f);
      const float d2 = image[3 * pix + 2] - gp[2] * (1.f / 255.f);
      q.dC0 = (d0 > 0.f ? 1.f : (d0 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      q.dC1 = (d1 > 0.f ? 1.f : (d1 < 0.f ? -1.f : 0.f)) * a.inv_norm;
      q.dC2 = (d2 > 0.f ? 1.f : (d2 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    }
  }
  q.T_final = q.T;
  q.bgdot = a.bg[0] * q.dC0 + a.bg[1] * q.dC1 + a.bg[2] * q.dC2;
  q.acc0 = q.acc1 = q.acc2 = 0.f;
  int warp_n = q.n;
  for (int o = 16; o > 0; o >>= 1) warp_n = max(warp_n, __shfl_xor_sync(0xffffffffu, warp_n, o));
  const int end = rg.x + warp_n;
  Splat2 f;
  fetch2(f, sp, a.support, inst_rows, end - 1 - lane, end - 1 - lane >= rg.x);
  uint32_t row_next = row2(inst_rows, end - 33 - lane, end - 33 - lane >= rg.x);
  for (int cend = end; cend > rg.x; cend -= 32) {
    const bool keep = reaches2(f, x0, x1, y0, y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if (keep) stage2(s, lane, f, x0, y0, a.support != nullptr);
    fetch2_row(f, sp, a.support, row_next, cend - 33 - lane >= rg.x);
    row_next = row2(inst_rows, cend - 65 - lane, cend - 65 - lane >= rg.x);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      const int rel = cend - 1 - j - rg.x;
      bwd2_splat<kBg>(q, s.a[j], s.b[j], s.c[j], s.d[j], s.row[j], rel, pxf, pyf, oxf, oyf, g_sp);
    }
    __syncwarp();
  }
}

// ---- K3 + L + K4 in one kernel (2DGS; see raster_fused_kernel in raster.cu)
#ifndef BS_FUSED2_KEEP
#define BS_FUSED2_KEEP 128  // swept on B200 (C3 raster ms, before the list compaction): 32 (4 CTAs) 7.80, 64 7.29, 128 7.16; separate kernels 7.32
#endif
#ifndef BS_FUSED2_CTAS
#define BS_FUSED2_CTAS 3
#endif
#ifndef BS_FUSED2_PAIR_MERGE
#define BS_FUSED2_PAIR_MERGE 2  // A/B on B200 (C3 raster): 0 6.500, 1 (sparse pairs) 6.303, 2 (all disjoint pairs) 6.242 ms
#endif
constexpr int kKeep2 = BS_FUSED2_KEEP;  // kept-splat records per warp

struct Kept2 {
  float4 rec[kKeep2][4];  // staged a, b, c, d (stage2 layout)
  int2 idx[kKeep2];       // (G_SP row, mask of the lanes the splat was blended into)
};

template <bool kBg>
__global__ void __launch_bounds__(kT2, BS_FUSED2_CTAS) raster2d_fused_kernel(
    R2Args a, const float* __restrict__ sp, const uint32_t* __restrict__ inst_rows, const int2* __restrict__ ranges,
    float* __restrict__ image, float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
    const uint8_t* __restrict__ gt, const int32_t* __restrict__ gt_view, float* __restrict__ loss_tiles,
    float* __restrict__ g_sp) {
  extern __shared__ __align__(16) unsigned char s_dyn2[];
  __shared__ float s_red[kW2];
  const int slot = blockIdx.z, tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Kept2& kp = reinterpret_cast<Kept2*>(s_dyn2)[w];
  const int rx = blockIdx.x * BS_TILE + (w & 1) * 8, ry = blockIdx.y * BS_TILE + (w >> 1) * 4;
  const int px = rx + (lane & 7), py = ry + (lane >> 3);
  const float x0 = rx + 0.5f, x1 = x0 + 7.f, y0 = ry + 0.5f, y1 = y0 + 3.f;
  const float pxf = px + 0.5f, pyf = py + 0.5f;
  const float oxf = (float)(lane & 7), oyf = (float)(lane >> 3);
  const bool inside = slot_pixel(a.slot_patches, a.patch_P, a.W, a.H, slot, px, py);
  const int2 rg = ranges[(int64_t)slot * a.tiles_per_slot + tile];
  // ---------------- forward (raster2d_fwd_kernel's blend), appending the kept splats
  Px2 p{1.f, 0.f, 0.f, 0.f, 0, !inside};
  Splat2 f;
  fetch2(f, sp, a.support, inst_rows, rg.x + lane, rg.x + lane < rg.y);
  uint32_t row_next = row2(inst_rows, rg.x + 32 + lane, rg.x + 32 + lane < rg.y);
  int nk = 0;  // kept records (warp-uniform); kKeep2 + 1 once the list overflowed
  for (int b0 = rg.x; b0 < rg.y; b0 += 32) {
    if (__all_sync(0xffffffffu, p.done)) break;
    const bool keep = reaches2(f, x0, x1, y0, y1);
    const uint32_t bits = __ballot_sync(0xffffffffu, keep);
    const int nb = __popc(bits);
    // a chunk's records are contiguous; a chunk that does not fit is staged
    // at 0 and the backward takes the chunked walk
    const int base = nk + nb <= kKeep2 ? nk : 0;
    if (keep) {
      const int pos = base + __popc(bits & ((1u << lane) - 1u));
      stage2_rec(f, x0, y0, a.support != nullptr, kp.rec[pos]);
      kp.idx[pos] = make_int2((int)f.row, 0);  // .y: the mask, written after the blend
    }
    fetch2_row(f, sp, a.support, row_next, b0 + 32 + lane < rg.y);
    row_next = row2(inst_rows, b0 + 64 + lane, b0 + 64 + lane < rg.y);
    __syncwarp();
    uint32_t rest = bits;  // staging lanes of the records still to blend
    for (int k = 0; k < nb; ++k) {
      const int pos = base + k;
      const int rel = b0 + __ffs(rest) - 1 - rg.x;  // range-relative index (idx.y is not read here)
      rest &= rest - 1u;
      Eval2 e;
      const float4 sa = kp.rec[pos][0];
      const float4 col = kp.rec[pos][3];
      eval2(sa, kp.rec[pos][1], kp.rec[pos][2], col.w, pxf, pyf, oxf, oyf, e);
      // predicated (no branch): pixels done or outside the support keep their state
      const bool in = !p.done && e.in;
      const float alpha = fminf(kAMax, __fmul_rn(sa.z, ex2a(fminf(e.pw2, 0.f))));
      const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
      const bool fin = nT < kTStop;
      const bool c = in && !fin;
      const float wgt = __fmul_rn(alpha, p.T);
      p.done = p.done || (in && fin);
      p.c0 = c ? __fmaf_rn(col.x, wgt, p.c0) : p.c0;
      p.c1 = c ? __fmaf_rn(col.y, wgt, p.c1) : p.c1;
      p.c2 = c ? __fmaf_rn(col.z, wgt, p.c2) : p.c2;
      p.T = c ? nT : p.T;
      p.contrib = c ? rel + 1 : p.contrib;
      // the lanes this splat was blended into = the pairs the backward
      // differentiates (written after every lane's last read of the record)
      const uint32_t who = __ballot_sync(0xffffffffu, c);
      if (lane == 0) kp.idx[pos].y = (int)who;
    }
    __syncwarp();
    if (nk + nb <= kKeep2) {
      // keep only the records blended into some pixel (lane j moves record j)
      float4 r[4];
      int2 id = make_int2(0, 0);
      if (lane < nb) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) r[q4] = kp.rec[base + lane][q4];
        id = kp.idx[base + lane];
      }
      const bool live = lane < nb && id.y != 0;
      const uint32_t lb = __ballot_sync(0xffffffffu, live);
      __syncwarp();
      if (live) {
        const int dst = base + __popc(lb & ((1u << lane) - 1u));
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) kp.rec[dst][q4] = r[q4];
        kp.idx[dst] = id;
      }
      nk += __popc(lb);
      __syncwarp();
    } else {
      nk = kKeep2 + 1;
    }
  }
  // outputs, loss partial, this pixel's L1 gradient
  float l = 0.f;
  PxB2 q;
  q.T = 1.f;
  q.n = 0;
  q.dC0 = q.dC1 = q.dC2 = 0.f;
  if (inside) {
    const int64_t pix = ((int64_t)slot * a.H + py) * a.W + px;
    const float o0 = p.c0 + p.T * a.bg[0], o1 = p.c1 + p.T * a.bg[1], o2 = p.c2 + p.T * a.bg[2];
    image[3 * pix] = o0;
    image[3 * pix + 1] = o1;
    image[3 * pix + 2] = o2;
    if (final_T) final_T[pix] = p.T;
    if (n_contrib) n_contrib[pix] = p.contrib;
    const int gv = gt_view ? gt_view[slot] : slot;
    const uint8_t* gp = gt + 3 * (((int64_t)gv * a.H + py) * a.W + px);
    const float d0 = o0 - gp[0] * (1.f / 255.f), d1 = o1 - gp[1] * (1.f / 255.f), d2 = o2 - gp[2] * (1.f / 255.f);
    l = fabsf(d0) + fabsf(d1) + fabsf(d2);
    q.dC0 = (d0 > 0.f ? 1.f : (d0 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    q.dC1 = (d1 > 0.f ? 1.f : (d1 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    q.dC2 = (d2 > 0.f ? 1.f : (d2 < 0.f ? -1.f : 0.f)) * a.inv_norm;
    q.T = p.T;
    q.n = p.contrib;
  }
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) s_red[w] = l;
  __syncthreads();  // (an arrival counter without the barrier measured no faster)
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < kW2; ++k) t += s_red[k];
    loss_tiles[(int64_t)slot * a.tiles_per_slot + tile] = t;
  }
  q.T_final = q.T;
  q.bgdot = a.bg[0] * q.dC0 + a.bg[1] * q.dC1 + a.bg[2] * q.dC2;
  q.acc0 = q.acc1 = q.acc2 = 0.f;
  // ---------------- backward: the kept list back to front, two records per
  // iteration (the shallower splat's front half overlaps the deeper one's
  // tail and reduction)
  if (nk <= kKeep2) {
    int k = nk - 1;
    for (; k >= 1; k -= 2) {
      const int2 id1 = kp.idx[k], id0 = kp.idx[k - 1];
#if BS_FUSED2_PAIR_MERGE
      const uint32_t m1 = (uint32_t)id1.y, m0 = (uint32_t)id0.y;
#if BS_FUSED2_PAIR_MERGE >= 2
      if ((m1 & m0) == 0u && (__popc(m1) > kSparse2 || __popc(m0) > kSparse2)) {
        // disjoint with a dense one: one pass, then each surfel's own lanes
        // reduced (the other surfel's lanes as zero)
        const bool in1 = (m1 >> lane) & 1u, in0 = (m0 >> lane) & 1u;
        const int kk = in1 ? k : k - 1;
        const float4 cc = kp.rec[kk][3];
        Front2 f;
        bwd2_front(f, kp.rec[kk][0], kp.rec[kk][1], kp.rec[kk][2], cc.w, pxf, pyf, oxf, oyf);
        float g[16], gm[16];
        bwd2_back<kBg>(q, f, cc, in1 || in0, pxf, pyf, g);
#pragma unroll
        for (int t = 0; t < 16; ++t) gm[t] = in1 ? g[t] : 0.f;
        reduce2(gm, m1, in1, g_sp + (int64_t)(uint32_t)id1.x * kGSP2);
#pragma unroll
        for (int t = 0; t < 16; ++t) gm[t] = in0 ? g[t] : 0.f;
        reduce2(gm, m0, in0, g_sp + (int64_t)(uint32_t)id0.x * kGSP2);
        continue;
      }
#endif
      if ((m1 & m0) == 0u && __popc(m1) <= kSparse2 && __popc(m0) <= kSparse2) {
        // two sparse surfels on disjoint pixels: one pass, each lane reading
        // the record of the surfel that covers its pixel (see raster.cu)
        const bool in1 = (m1 >> lane) & 1u;
        const bool any = in1 || ((m0 >> lane) & 1u);
        const int kk = in1 ? k : k - 1;
        const float4 cc = kp.rec[kk][3];
        Front2 f;
        bwd2_front(f, kp.rec[kk][0], kp.rec[kk][1], kp.rec[kk][2], cc.w, pxf, pyf, oxf, oyf);
        float g[16];
        bwd2_back<kBg>(q, f, cc, any, pxf, pyf, g);
        if (any) {
          float* dst = g_sp + (int64_t)(uint32_t)(in1 ? id1.x : id0.x) * kGSP2;
#pragma unroll
          for (int t = 0; t < 16; t += 4)
            atomicAdd(reinterpret_cast<float4*>(dst + t), make_float4(g[t], g[t + 1], g[t + 2], g[t + 3]));
        }
        continue;
      }
#endif
      const float4 c1 = kp.rec[k][3], c0 = kp.rec[k - 1][3];
      Front2 f1, f0;
      bwd2_front(f1, kp.rec[k][0], kp.rec[k][1], kp.rec[k][2], c1.w, pxf, pyf, oxf, oyf);
      bwd2_front(f0, kp.rec[k - 1][0], kp.rec[k - 1][1], kp.rec[k - 1][2], c0.w, pxf, pyf, oxf, oyf);
      float g[16];
      const bool any1 = ((uint32_t)id1.y >> lane) & 1u;
      bwd2_back<kBg>(q, f1, c1, any1, pxf, pyf, g);
      reduce2(g, (uint32_t)id1.y, any1, g_sp + (int64_t)(uint32_t)id1.x * kGSP2);
      const bool any0 = ((uint32_t)id0.y >> lane) & 1u;
      bwd2_back<kBg>(q, f0, c0, any0, pxf, pyf, g);
      reduce2(g, (uint32_t)id0.y, any0, g_sp + (int64_t)(uint32_t)id0.x * kGSP2);
    }
    if (k == 0) {
      const int2 id = kp.idx[0];
      const float4 c0 = kp.rec[0][3];
      Front2 f0;
      bwd2_front(f0, kp.rec[0][0], kp.rec[0][1], kp.rec[0][2], c0.w, pxf, pyf, oxf, oyf);
      float g[16];
      const bool any = ((uint32_t)id.y >> lane) & 1u;
      bwd2_back<kBg>(q, f0, c0, any, pxf, pyf, g);
      reduce2(g, (uint32_t)id.y, any, g_sp + (int64_t)(uint32_t)id.x * kGSP2);
    }
    return;
  }
  // the list wrapped: chunked walk over global memory (raster2d_bwd_kernel's)
  Warp2& s = *reinterpret_cast<Warp2*>(&kp);
  __syncwarp();
  int warp_n = q.n;
  for (int o = 16; o > 0; o >>= 1) warp_n = max(warp_n, __shfl_xor_sync(0xffffffffu, warp_n, o));
  const int end = rg.x + warp_n;
  fetch2(f, sp, a.support, inst_rows, end - 1 - lane, end - 1 - lane >= rg.x);
  row_next = row2(inst_rows, end - 33 - lane, end - 33 - lane >= rg.x);
  for (int cend = end; cend > rg.x; cend -= 32) {
    const bool keep = reaches2(f, x0, x1, y0, y1);
    uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if (keep) stage2(s, lane, f, x0, y0, a.support != nullptr);
    fetch2_row(f, sp, a.support, row_next, cend - 33 - lane >= rg.x);
    row_next = row2(inst_rows, cend - 65 - lane, cend - 65 - lane >= rg.x);
    __syncwarp();
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      bwd2_splat<kBg>(q, s.a[j], s.b[j], s.c[j], s.d[j], s.row[j], cend - 1 - j - rg.x, pxf, pyf, oxf, oyf, g_sp);
    }
    __syncwarp();
  }
}

int32_t make_r2(const bs_raster_desc* d, R2Args& a) {
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

extern "C" int32_t bs_raster2d_fwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                   const int32_t* ranges, float* image, float* final_T, int32_t* n_contrib,
                                   const uint8_t* gt, const int32_t* gt_slot_view, float* loss_tiles, void* stream) {
  R2Args a;
  int32_t st = make_r2(d, a);
  if (st) return st;
  BS_REQUIRE(!a.loss_fused || (gt && loss_tiles), BS_ERR_PARAMETER, "fused loss needs gt and loss_tiles");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  raster2d_fwd_kernel<<<grid, kT2, 0, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges),
                                                          image, final_T, n_contrib, gt, gt_slot_view, loss_tiles);
  BS_LAUNCH_CHECK("raster2d_fwd_kernel");
  return BS_OK;
}

extern "C" int32_t bs_raster2d_fwd_bwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                       const int32_t* ranges, float* image, float* final_T, int32_t* n_contrib,
                                       const uint8_t* gt, const int32_t* gt_slot_view, float* loss_tiles,
                                       float* g_sp, void* stream) {
  R2Args a;
  int32_t st = make_r2(d, a);
  if (st) return st;
  BS_REQUIRE(gt && loss_tiles && g_sp, BS_ERR_PARAMETER, "raster2d_fwd_bwd needs gt, loss_tiles and g_sp");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  const bool bg = a.bg[0] != 0.f || a.bg[1] != 0.f || a.bg[2] != 0.f;
  auto kern = bg ? raster2d_fused_kernel<true> : raster2d_fused_kernel<false>;
  const size_t smem = sizeof(Kept2) * kW2;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kT2, smem, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges), image,
                                               final_T, n_contrib, gt, gt_slot_view, loss_tiles, g_sp);
  BS_LAUNCH_CHECK("raster2d_fused_kernel");
  return BS_OK;
}

extern "C" int32_t bs_raster2d_bwd(const bs_raster_desc* d, const float* sp_rows, const uint32_t* inst_rows,
                                   const int32_t* ranges, const float* image, const float* final_T,
                                   const int32_t* n_contrib, const float* grad_image, const uint8_t* gt,
                                   const int32_t* gt_slot_view, float* g_sp, void* stream) {
  R2Args a;
  int32_t st = make_r2(d, a);
  if (st) return st;
  BS_REQUIRE(grad_image || (image && gt), BS_ERR_PARAMETER, "raster_bwd needs grad_image or (image, gt)");
  const dim3 grid(a.tiles_x, (a.H + BS_TILE - 1) / BS_TILE, a.n_slots);
  const bool bg = a.bg[0] != 0.f || a.bg[1] != 0.f || a.bg[2] != 0.f;
  auto kern = bg ? raster2d_bwd_kernel<true> : raster2d_bwd_kernel<false>;
  kern<<<grid, kT2, 0, as_stream(stream)>>>(a, sp_rows, inst_rows, reinterpret_cast<const int2*>(ranges), image,
                                            final_T, n_contrib, grad_image, gt, gt_slot_view, g_sp);
  BS_LAUNCH_CHECK("raster2d_bwd_kernel");
  return BS_OK;
}
