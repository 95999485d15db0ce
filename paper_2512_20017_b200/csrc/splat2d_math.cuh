// 2D Gaussian splatting (2DGS, surfel ray-splat intersection; PAPER.md:
// 773-777, state table) -- projection, its analytic
// backward, and the per-pixel evaluation shared by the raster kernels.
//
// A point is an oriented disk: centre p, tangent axes R(q)[:,0]*s_u and
// R(q)[:,1]*s_v (s = exp(log_scale.xy)), normal R(q)[:,2].  With camera-frame
// columns c0 = K Rcw t_u, c1 = K Rcw t_v, c2 = K Rcw (p - campos) the
// homogeneous image of the local point (u, v) is M (u, v, 1)^T, M = [c0 c1 c2]
// ("ray transform", stored row-major -- the KWH matrix of the state table).
// For a pixel centre (x, y) the ray meets the disk at
//   h_x = M_row0 - x M_row2,  h_y = M_row1 - y M_row2,  zeta = h_x x h_y,
//   (u, v) = (zeta.x, zeta.y) / zeta.z,
// and, with the screen-space low-pass of 2DGS (sigma_f = 1/sqrt 2 px),
//   power = -0.5 min(u^2 + v^2, 2 |mean2d - pixel|^2).
// mean2d = c2.xy / c2.z (projected centre); per-axis radii bound the image of
// the 3-sigma disk u^2 + v^2 = 9 (exact bounding box of that conic from its
// dual C* = M diag(9, 9, -1) M^T), measured from mean2d.
//
// Forward: explicit round-to-nearest ops (bit-identical to the CPU oracle).
#pragma once
#include "splat_math.cuh"

namespace bs {

// SP row of a 2DGS splat (24 floats, 96 B):
//   0 u  1 v  2 opacity  3..11 M (row-major)  12 r 13 g 14 b  15 depth
//   16 radius_x  17 radius_y (half-widths of the support box)  18..20 normal
//   (camera frame)  21 pad  22 box centre x  23 box centre y
constexpr int kSP2 = 24;
// G_SP row of a 2DGS splat (16 floats, 64-byte aligned; 15 used): d u, d v,
// d M[9], d opacity, d rgb, pad
constexpr int kGSP2 = 16;
constexpr int kGSP2Used = 15;

// View-independent part of a surfel projection (once per point): rotation of
// the quaternion, the two tangent scales, activated opacity.
struct Pre2D {
  float Rq[9], s[2], opac;
};

__device__ __forceinline__ void point_pre2(const PointIn& pt, Pre2D& r) {
  QuatFrame q;
  quat_frame(pt, 2, q);
#pragma unroll
  for (int k = 0; k < 9; ++k) r.Rq[k] = q.Rq[k];
  r.s[0] = q.s[0];
  r.s[1] = q.s[1];
  r.opac = det_sigmoid(pt.op_logit);
}

// dL/dRq accumulated over views (G, row-major) -> quaternion (g[8..11]).
__device__ __forceinline__ void point_pre2_backward(const PointIn& pt, const float G[9], float* g) {
  QuatFrame q;
  quat_frame(pt, 2, q);
  float gq[4];
  quat_backward(q, G, gq);
#pragma unroll
  for (int k = 0; k < 4; ++k) g[8 + k] += gq[k];
}

struct Proj2D {
  float d[3], qc[3], Rc[9];
  float c0[3], c1[3], c2[3];  // M columns
  float u, v, depth, radius_x, radius_y, normal[3];
  float support_k;  // k = min(9, 2 ln(255 o)) of the support (box, rasteriser threshold)
  float box_cx, box_cy;  // centre of the support box (half-widths radius_x / radius_y)
  float len, dir[3], Y[16], col_raw[3], col[3], opac;
  bool valid;
};

__device__ __forceinline__ void kmul(const bs_camera& c, const float x[3], float out[3]) {
  out[0] = fadd(fmul(c.fx, x[0]), fmul(c.cx, x[2]));
  out[1] = fadd(fmul(c.fy, x[1]), fmul(c.cy, x[2]));
  out[2] = x[2];
}

template <class SH>
__device__ __forceinline__ void project2d_forward(const PointIn& pt, const Pre2D& pre, const SH& sh,
                                                  const bs_camera& c, int n_sh, Proj2D& f,
                                                  const float* gcol = nullptr, float* wk = nullptr) {
#pragma unroll
  for (int k = 0; k < 3; ++k) f.d[k] = fsub(pt.p[k], c.pos[k]);
  const float* W = c.rot_cw;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    f.qc[k] = fadd(fadd(fmul(W[3 * k], f.d[0]), fmul(W[3 * k + 1], f.d[1])), fmul(W[3 * k + 2], f.d[2]));
  // Rc = Rcw Rq
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      f.Rc[3 * i + j] =
          fadd(fadd(fmul(W[3 * i], pre.Rq[j]), fmul(W[3 * i + 1], pre.Rq[3 + j])), fmul(W[3 * i + 2], pre.Rq[6 + j]));
  float tu[3], tv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    tu[i] = fmul(f.Rc[3 * i], pre.s[0]);
    tv[i] = fmul(f.Rc[3 * i + 1], pre.s[1]);
  }
  kmul(c, tu, f.c0);
  kmul(c, tv, f.c1);
  kmul(c, f.qc, f.c2);
  const float z = f.qc[2];
  f.depth = z;
  f.u = fdiv(f.c2[0], f.c2[2]);
  f.v = fdiv(f.c2[1], f.c2[2]);
  // Dual conics of the disk images, in image coordinates CENTRED on (u, v):
  // x - u = (p.x - u p.z) / p.z for p = c0 s + c1 t + c2, so the columns are
  // shifted to c_i' = (c_i.x - u c_i.z, c_i.y - v c_i.z, c_i.z) (c2' ~ (0, 0, z)).
  // In absolute pixel coordinates the box half-width comes out of
  // bx^2 - C*00 / C*22 with bx ~ u ~ 10^3 px: a float cancellation of
  // ~0.1 px.  C*_ij = s (c0'_i c0'_j + c1'_i c1'_j) - c2'_i c2'_j.
  float a0[3], a1[3], a2[3];
  a0[0] = fsub(f.c0[0], fmul(f.u, f.c0[2]));
  a0[1] = fsub(f.c0[1], fmul(f.v, f.c0[2]));
  a0[2] = f.c0[2];
  a1[0] = fsub(f.c1[0], fmul(f.u, f.c1[2]));
  a1[1] = fsub(f.c1[1], fmul(f.v, f.c1[2]));
  a1[2] = f.c1[2];
  a2[0] = fsub(f.c2[0], fmul(f.u, f.c2[2]));
  a2[1] = fsub(f.c2[1], fmul(f.v, f.c2[2]));
  a2[2] = f.c2[2];
  // the 3-sigma disk (s = 9) images to a bounded ellipse
  const float c22 = fsub(fmul(9.f, fadd(fmul(a0[2], a0[2]), fmul(a1[2], a1[2]))), fmul(a2[2], a2[2]));
  const float c02 = fsub(fmul(9.f, fadd(fmul(a0[0], a0[2]), fmul(a1[0], a1[2]))), fmul(a2[0], a2[2]));
  const float c12 = fsub(fmul(9.f, fadd(fmul(a0[1], a0[2]), fmul(a1[1], a1[2]))), fmul(a2[1], a2[2]));
  const float c00 = fsub(fmul(9.f, fadd(fmul(a0[0], a0[0]), fmul(a1[0], a1[0]))), fmul(a2[0], a2[0]));
  const float c11 = fsub(fmul(9.f, fadd(fmul(a0[1], a0[1]), fmul(a1[1], a1[1]))), fmul(a2[1], a2[1]));
  f.valid = c22 < 0.f;
  f.radius_x = f.radius_y = 0.f;
  if (f.valid) {
    const float bx = fdiv(c02, c22), by = fdiv(c12, c22);
    const float ex = fsub(fmul(bx, bx), fdiv(c00, c22));
    const float ey = fsub(fmul(by, by), fdiv(c11, c22));
    f.valid = ex >= 0.f && ey >= 0.f;
  }
  f.box_cx = f.u;
  f.box_cy = f.v;
  const float k = support_k(pre.opac);
  f.support_k = k;
  if (f.valid && k > 0.f) {
    // support {min(g3, g2) <= k}, k = min(9, 2 ln(255 o)): the image of the
    // disk u^2 + v^2 <= k (dual conic, bounded since the 9-disk's is) united
    // with the low-pass circle |mean2d - pixel| <= sqrt(k / 2)
    const float k22 = fsub(fmul(k, fadd(fmul(a0[2], a0[2]), fmul(a1[2], a1[2]))), fmul(a2[2], a2[2]));
    const float k02 = fsub(fmul(k, fadd(fmul(a0[0], a0[2]), fmul(a1[0], a1[2]))), fmul(a2[0], a2[2]));
    const float k12 = fsub(fmul(k, fadd(fmul(a0[1], a0[2]), fmul(a1[1], a1[2]))), fmul(a2[1], a2[2]));
    const float k00 = fsub(fmul(k, fadd(fmul(a0[0], a0[0]), fmul(a1[0], a1[0]))), fmul(a2[0], a2[0]));
    const float k11 = fsub(fmul(k, fadd(fmul(a0[1], a0[1]), fmul(a1[1], a1[1]))), fmul(a2[1], a2[1]));
    const float bx = fdiv(k02, k22), by = fdiv(k12, k22);  // ellipse centre - (u, v)
    const float hx = fsqrt(fmaxf(fsub(fmul(bx, bx), fdiv(k00, k22)), 0.f));
    const float hy = fsqrt(fmaxf(fsub(fmul(by, by), fdiv(k11, k22)), 0.f));
    const float rc = fsqrt(fmul(0.5f, k));
    const float x0 = fminf(fsub(bx, hx), -rc), x1 = fmaxf(fadd(bx, hx), rc);
    const float y0 = fminf(fsub(by, hy), -rc), y1 = fmaxf(fadd(by, hy), rc);
    f.box_cx = fadd(f.u, fmul(0.5f, fadd(x0, x1)));
    f.box_cy = fadd(f.v, fmul(0.5f, fadd(y0, y1)));
    f.radius_x = fmul(0.5f, fsub(x1, x0));
    f.radius_y = fmul(0.5f, fsub(y1, y0));
  }
  // camera-frame normal, oriented towards the camera
  float n0 = f.Rc[2], n1 = f.Rc[5], n2 = f.Rc[8];
  const float facing = fadd(fadd(fmul(n0, f.qc[0]), fmul(n1, f.qc[1])), fmul(n2, f.qc[2]));
  if (facing > 0.f) {
    n0 = -n0;
    n1 = -n1;
    n2 = -n2;
  }
  f.normal[0] = n0;
  f.normal[1] = n1;
  f.normal[2] = n2;
  // view-dependent colour and opacity (as 3DGS)
  f.len = fsqrt(fadd(fadd(fmul(f.d[0], f.d[0]), fmul(f.d[1], f.d[1])), fmul(f.d[2], f.d[2])));
#pragma unroll
  for (int k = 0; k < 3; ++k) f.dir[k] = fdiv(f.d[k], f.len);
  sh_basis(f.dir, n_sh, f.Y);
  sh_colour(sh, n_sh, f.Y, f.col_raw, f.col, gcol, wk);
  f.opac = pre.opac;
}

__device__ __forceinline__ void write_sp2_row(float* __restrict__ row, const Proj2D& f) {
  float4* r4 = reinterpret_cast<float4*>(row);
  // rows of M: (c0.x c1.x c2.x) (c0.y c1.y c2.y) (c0.z c1.z c2.z)
  r4[0] = make_float4(f.u, f.v, f.opac, f.c0[0]);
  r4[1] = make_float4(f.c1[0], f.c2[0], f.c0[1], f.c1[1]);
  r4[2] = make_float4(f.c2[1], f.c0[2], f.c1[2], f.c2[2]);
  r4[3] = make_float4(f.col[0], f.col[1], f.col[2], f.depth);
  r4[4] = make_float4(f.valid ? f.radius_x : 0.f, f.valid ? f.radius_y : 0.f, f.normal[0], f.normal[1]);
  r4[5] = make_float4(f.normal[2], 0.f, f.box_cx, f.box_cy);
}

// G_SP2 rows from the rasteriser carry, in entries 2..10, the moments
// Ga = sum dL/dzeta, Gb = sum px dL/dzeta, Gc = sum py dL/dzeta of the
// per-pixel zeta = r0 x r1 + px (r1 x r2) + py (r2 x r0) (r_i: rows of M).
// dL/dr0 = r1 x Ga + Gc x r2, dL/dr1 = Ga x r0 + r2 x Gb,
// dL/dr2 = Gb x r1 + r0 x Gc  ->  entries 2..10 become dL/dM (row-major).
__device__ __forceinline__ void cross3f(const float a[3], const float b[3], float o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

__device__ __forceinline__ void gsp2_from_moments(const Proj2D& f, float* gs) {
  const float r0[3] = {f.c0[0], f.c1[0], f.c2[0]};
  const float r1[3] = {f.c0[1], f.c1[1], f.c2[1]};
  const float r2[3] = {f.c0[2], f.c1[2], f.c2[2]};
  const float Ga[3] = {gs[2], gs[3], gs[4]}, Gb[3] = {gs[5], gs[6], gs[7]}, Gc[3] = {gs[8], gs[9], gs[10]};
  float t0[3], t1[3];
  cross3f(r1, Ga, t0);
  cross3f(Gc, r2, t1);
#pragma unroll
  for (int k = 0; k < 3; ++k) gs[2 + k] = t0[k] + t1[k];
  cross3f(Ga, r0, t0);
  cross3f(r2, Gb, t1);
#pragma unroll
  for (int k = 0; k < 3; ++k) gs[5 + k] = t0[k] + t1[k];
  cross3f(Gb, r1, t0);
  cross3f(r0, Gc, t1);
#pragma unroll
  for (int k = 0; k < 3; ++k) gs[8 + k] = t0[k] + t1[k];
}

// Accumulate the parameter gradient of one (point, view) pair.
// gsp = (du, dv, dM[9] row-major, dopacity, dr, dg, db).
// GR accumulates dL/dRq (row-major) for point_pre2_backward.
template <class SH, class ShAdd>
__device__ __forceinline__ void project2d_backward(const PointIn& pt, const Pre2D& pre, const SH& sh,
                                                   const bs_camera& c, int n_sh, const Proj2D& f,
                                                   const float gsp[15], float* g, float GR[9], ShAdd& sh_add,
                                                   const float* wk_pre = nullptr) {
  if (!f.valid) return;
  // ---- colour -> sh, dir (as 3DGS)
  float wk[16];
  sh_colour_backward(sh, n_sh, f.Y, f.col_raw, gsp + 12, wk_pre, wk, sh_add);
  float gdir[3];
  sh_dir_grad(f.dir, n_sh, wk, gdir);
  const float dd = f.dir[0] * gdir[0] + f.dir[1] * gdir[1] + f.dir[2] * gdir[2];
  float gp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) gp[k] = (gdir[k] - f.dir[k] * dd) / f.len;
  // ---- opacity
  g[3] += gsp[11] * pre.opac * (1.f - pre.opac);
  // ---- M rows -> columns c0, c1, c2; mean2d = c2.xy / c2.z
  const float* gm = gsp + 2;  // row-major 3x3
  float gc0[3] = {gm[0], gm[3], gm[6]};
  float gc1[3] = {gm[1], gm[4], gm[7]};
  float gc2[3] = {gm[2], gm[5], gm[8]};
  const float iz = 1.f / f.c2[2];
  gc2[0] += gsp[0] * iz;
  gc2[1] += gsp[1] * iz;
  gc2[2] += -(gsp[0] * f.c2[0] + gsp[1] * f.c2[1]) * iz * iz;
  // c = K x  ->  dL/dx = (fx gc.x, fy gc.y, cx gc.x + cy gc.y + gc.z)
  auto kback = [&](const float gcv[3], float gx[3]) {
    gx[0] = c.fx * gcv[0];
    gx[1] = c.fy * gcv[1];
    gx[2] = c.cx * gcv[0] + c.cy * gcv[1] + gcv[2];
  };
  float gtu[3], gtv[3], gq[3];
  kback(gc0, gtu);
  kback(gc1, gtv);
  kback(gc2, gq);
  // ---- q = Rcw (p - campos)
  const float* W = c.rot_cw;
#pragma unroll
  for (int k = 0; k < 3; ++k) gp[k] += W[k] * gq[0] + W[3 + k] * gq[1] + W[6 + k] * gq[2];
  g[0] += gp[0];
  g[1] += gp[1];
  g[2] += gp[2];
  // ---- tu = Rc[:,0] s_u, tv = Rc[:,1] s_v
  float gs0 = 0.f, gs1 = 0.f;
  float gRc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    gs0 += f.Rc[3 * i] * gtu[i];
    gs1 += f.Rc[3 * i + 1] * gtv[i];
    gRc[3 * i] = gtu[i] * pre.s[0];
    gRc[3 * i + 1] = gtv[i] * pre.s[1];
    gRc[3 * i + 2] = 0.f;  // the normal column carries no loss gradient
  }
  g[4] += gs0 * pre.s[0];
  g[5] += gs1 * pre.s[1];
  // ---- Rc = Rcw Rq  ->  dL/dRq = Rcw^T dL/dRc
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) GR[3 * i + j] += W[i] * gRc[j] + W[3 + i] * gRc[3 + j] + W[6 + i] * gRc[6 + j];
}

}  // namespace bs
