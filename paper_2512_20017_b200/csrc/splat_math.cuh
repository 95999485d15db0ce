// 3DGS projection math (pts_splatting) and its
// analytic backward (pts_splatting.backward).
//
// Forward: every arithmetic op is an explicit round-to-nearest intrinsic
// (bs::fmul/fadd/...), so the splat state is bit-identical to the CPU
// oracle (oracle/splat_oracle.c, same op sequence, -ffp-contract=off).
// Backward: ordinary float arithmetic (contraction allowed); compared to the
// oracle within the fp32 tolerance stated in tests/test_gpu_parity.py.
//
// Conventions (builder-chosen standard 3DGS, frozen here):
//   EWA dilation 0.3 px^2, Jacobian clamp |x/z| <= 1.3 tan(fov/2),
//   support of a splat = {q <= 9} (3-sigma ellipse) intersected with
//   {alpha >= 1/255}; radii = float half-widths sqrt(k cov2d_xx),
//   sqrt(k cov2d_yy), k = min(9, 2 ln(255 o)): the tight bounding box of the
//   support (opacity-aware; 0 when o < 1/255), SH degree <= 3 with colour
//   max(sum + 0.5, 0), opacity = sigmoid(logit), scale = exp(log_scale).
#pragma once
#include "common.cuh"

namespace bs {

constexpr float kSH_C0 = 0.28209479177387814f;
constexpr float kSH_C1 = 0.4886025119029199f;
constexpr float kSH_C2_0 = 1.0925484305920792f;
constexpr float kSH_C2_1 = -1.0925484305920792f;
constexpr float kSH_C2_2 = 0.31539156525252005f;
constexpr float kSH_C2_3 = -1.0925484305920792f;
constexpr float kSH_C2_4 = 0.5462742152960396f;
constexpr float kSH_C3_0 = -0.5900435899266435f;
constexpr float kSH_C3_1 = 2.890611442640554f;
constexpr float kSH_C3_2 = -0.4570457994644658f;
constexpr float kSH_C3_3 = 0.3731763325901154f;
constexpr float kSH_C3_4 = -0.4570457994644658f;
constexpr float kSH_C3_5 = 1.445305721320277f;
constexpr float kSH_C3_6 = -0.5900435899266435f;
constexpr float kDilation = 0.3f;

struct PointIn {
  float p[3];
  float op_logit;
  float ls[3];
  float q[4];
  float sh[48];
};

struct ProjFwd {
  float d[3];      // p - campos
  float qc[3];     // camera-frame position
  float Sc[6];     // camera-frame covariance (00 01 02 11 12 22)
  float J00, J02, J11, J12;
  bool clamp_x, clamp_y;
  float tx, ty;
  float a, b, c, det;  // dilated 2D covariance
  float conic[3];
  float radius_x, radius_y;
  float support_k;  // k = min(9, 2 ln(255 o)) of the support (extents, rasteriser threshold)
  float u, v, depth;
  float len, dir[3];
  float Y[16];
  float col_raw[3], col[3];
  float opac;
  bool valid;
};

__device__ __forceinline__ void load_point(const float4* __restrict__ params, int64_t S, int64_t i,
                                           int n_sh, PointIn& pt) {
  const float4 a = params[i];
  const float4 b = params[S + i];
  const float4 q = params[2 * S + i];
  pt.p[0] = a.x; pt.p[1] = a.y; pt.p[2] = a.z; pt.op_logit = a.w;
  pt.ls[0] = b.x; pt.ls[1] = b.y; pt.ls[2] = b.z;
  pt.q[0] = q.x; pt.q[1] = q.y; pt.q[2] = q.z; pt.q[3] = q.w;
  const int planes = (3 * n_sh + 3) / 4;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    if (k < planes) {
      const float4 t = params[(3 + k) * S + i];
      pt.sh[4 * k] = t.x; pt.sh[4 * k + 1] = t.y; pt.sh[4 * k + 2] = t.z; pt.sh[4 * k + 3] = t.w;
    } else {
      pt.sh[4 * k] = pt.sh[4 * k + 1] = pt.sh[4 * k + 2] = pt.sh[4 * k + 3] = 0.f;
    }
  }
}

__device__ __forceinline__ void sh_basis(const float dir[3], int n_sh, float Y[16]) {
  const float x = dir[0], y = dir[1], z = dir[2];
  Y[0] = kSH_C0;
#pragma unroll
  for (int k = 1; k < 16; ++k) Y[k] = 0.f;
  if (n_sh > 1) {
    Y[1] = fmul(-kSH_C1, y);
    Y[2] = fmul(kSH_C1, z);
    Y[3] = fmul(-kSH_C1, x);
  }
  if (n_sh > 4) {
    const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(z, z);
    const float xy = fmul(x, y), yz = fmul(y, z), xz = fmul(x, z);
    Y[4] = fmul(kSH_C2_0, xy);
    Y[5] = fmul(kSH_C2_1, yz);
    Y[6] = fmul(kSH_C2_2, fsub(fsub(fmul(2.f, zz), xx), yy));
    Y[7] = fmul(kSH_C2_3, xz);
    Y[8] = fmul(kSH_C2_4, fsub(xx, yy));
    if (n_sh > 9) {
      Y[9] = fmul(fmul(kSH_C3_0, y), fsub(fmul(3.f, xx), yy));
      Y[10] = fmul(fmul(kSH_C3_1, xy), z);
      Y[11] = fmul(fmul(kSH_C3_2, y), fsub(fsub(fmul(4.f, zz), xx), yy));
      Y[12] = fmul(fmul(kSH_C3_3, z), fsub(fsub(fmul(2.f, zz), fmul(3.f, xx)), fmul(3.f, yy)));
      Y[13] = fmul(fmul(kSH_C3_4, x), fsub(fsub(fmul(4.f, zz), xx), yy));
      Y[14] = fmul(fmul(kSH_C3_5, z), fsub(xx, yy));
      Y[15] = fmul(fmul(kSH_C3_6, x), fsub(xx, fmul(3.f, yy)));
    }
  }
}

// SH coefficient accessors: from the registers of a loaded point, or straight
// from the plane-major parameters (L1-resident) to keep 48 registers free.
// load4(q): coefficients 4q .. 4q + 3 (one float4 plane entry).
struct ShRegs {
  const float* sh;
  __device__ __forceinline__ float operator()(int f) const { return sh[f]; }
  __device__ __forceinline__ float4 load4(int q) const {
    return make_float4(sh[4 * q], sh[4 * q + 1], sh[4 * q + 2], sh[4 * q + 3]);
  }
};
struct ShPlanes {
  const float* params;  // plane-major float4 planes as floats
  int64_t S, i;
  __device__ __forceinline__ float operator()(int f) const {
    return __ldg(params + ((int64_t)(3 + (f >> 2)) * S + i) * 4 + (f & 3));
  }
  __device__ __forceinline__ float4 load4(int q) const {
    return __ldg(reinterpret_cast<const float4*>(params) + (int64_t)(3 + q) * S + i);
  }
};

// SH coefficients of one point staged in shared memory as float4 entries
// [q][kProjThreads] (s = &entry[0][thread]; stride 256 float4 between q).
struct ShSmem {
  const float4* s;
  __device__ __forceinline__ float4 load4(int q) const { return s[q * 256]; }
  __device__ __forceinline__ float operator()(int f) const {
    const float4 v = s[(f >> 2) * 256];
    return (f & 3) == 0 ? v.x : (f & 3) == 1 ? v.y : (f & 3) == 2 ? v.z : v.w;
  }
};

// View-dependent colour from the SH coefficients (flat index f = 3k + ch):
// each channel sums Y_k sh_{k,ch} in k order (round-to-nearest, as the
// reference); coefficients are read as float4 plane entries.  With gcol
// (the colour gradient of this view) it also returns the direction weights
// wk[k] = sum_ch gcol[ch] sh_{k,ch} the backward needs when no channel is
// clamped, so the backward does not read the coefficients a second time.
template <class SH>
__device__ __forceinline__ void sh_colour(const SH& sh, int n_sh, const float Y[16], float col_raw[3], float col[3],
                                          const float* gcol, float* wk) {
  float acc[3] = {0.f, 0.f, 0.f};
  if (wk) {
#pragma unroll
    for (int k = 0; k < 16; ++k) wk[k] = 0.f;
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    if (4 * q >= 3 * n_sh) break;
    const float4 v4 = sh.load4(q);
    const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int f = 4 * q + e, k = f / 3, ch = f % 3;
      if (k < n_sh) {
        const float t = fmul(Y[k], v[e]);
        acc[ch] = k == 0 ? t : fadd(acc[ch], t);
        if (wk) wk[k] = __fmaf_rn(gcol[ch], v[e], wk[k]);
      }
    }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    col_raw[ch] = fadd(acc[ch], 0.5f);
    col[ch] = fmaxf(col_raw[ch], 0.f);
  }
}

// Backward of the colour clamp into the SH coefficients and the direction
// weights wk (see sh_colour; wk_pre is used when no channel was clamped).
// The coefficient gradients go out as float4 plane entries:
// sh_add.add4(q, (dL/dsh_f for f = 4q .. 4q + 3)), f = 3k + channel.
template <class SH, class ShAdd>
__device__ __forceinline__ void sh_colour_backward(const SH& sh, int n_sh, const float Y[16], const float col_raw[3],
                                                   const float gcol[3], const float* wk_pre, float wk[16],
                                                   ShAdd& sh_add) {
  float dc[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) dc[ch] = col_raw[ch] >= 0.f ? gcol[ch] : 0.f;
  const bool fast = wk_pre != nullptr && col_raw[0] >= 0.f && col_raw[1] >= 0.f && col_raw[2] >= 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) wk[k] = fast ? wk_pre[k] : 0.f;
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    if (4 * q >= 3 * n_sh) break;
    float v[4];
    float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!fast) c4 = sh.load4(q);
    const float c[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int f = 4 * q + e, k = f / 3, ch = f % 3;
      v[e] = k < n_sh ? Y[k] * dc[ch] : 0.f;
      if (!fast && k < n_sh) wk[k] = __fmaf_rn(dc[ch], c[e], wk[k]);
    }
    sh_add.add4(q, make_float4(v[0], v[1], v[2], v[3]));
  }
}

// Scales, normalised quaternion and its rotation matrix of a point (shared by
// the 3DGS and 2DGS models; explicit round-to-nearest ops).
struct QuatFrame {
  float s[3], qn[4], qnorm, Rq[9];
};

__device__ __forceinline__ void quat_frame(const PointIn& pt, int n_scales, QuatFrame& r) {
#pragma unroll
  for (int k = 0; k < 3; ++k) r.s[k] = k < n_scales ? det_expf(pt.ls[k]) : 0.f;
  const float nn = fadd(fadd(fadd(fmul(pt.q[0], pt.q[0]), fmul(pt.q[1], pt.q[1])), fmul(pt.q[2], pt.q[2])),
                        fmul(pt.q[3], pt.q[3]));
  r.qnorm = fsqrt(nn);
#pragma unroll
  for (int k = 0; k < 4; ++k) r.qn[k] = fdiv(pt.q[k], r.qnorm);
  const float w = r.qn[0], x = r.qn[1], y = r.qn[2], zq = r.qn[3];
  const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(zq, zq);
  const float xy = fmul(x, y), xz = fmul(x, zq), yz = fmul(y, zq);
  const float wx = fmul(w, x), wy = fmul(w, y), wz = fmul(w, zq);
  r.Rq[0] = fsub(1.f, fmul(2.f, fadd(yy, zz)));
  r.Rq[1] = fmul(2.f, fsub(xy, wz));
  r.Rq[2] = fmul(2.f, fadd(xz, wy));
  r.Rq[3] = fmul(2.f, fadd(xy, wz));
  r.Rq[4] = fsub(1.f, fmul(2.f, fadd(xx, zz)));
  r.Rq[5] = fmul(2.f, fsub(yz, wx));
  r.Rq[6] = fmul(2.f, fsub(xz, wy));
  r.Rq[7] = fmul(2.f, fadd(yz, wx));
  r.Rq[8] = fsub(1.f, fmul(2.f, fadd(xx, yy)));
}

// dL/d(raw quaternion) from dL/dRq (G, row-major), through the normalisation.
__device__ __forceinline__ void quat_backward(const QuatFrame& r, const float G[9], float gq[4]) {
  const float w = r.qn[0], x = r.qn[1], y = r.qn[2], zq = r.qn[3];
  float gqn[4];
  gqn[0] = 2.f * (-zq * G[1] + y * G[2] + zq * G[3] - x * G[5] - y * G[6] + x * G[7]);
  gqn[1] = 2.f * (y * G[1] + zq * G[2] + y * G[3] - 2.f * x * G[4] - w * G[5] + zq * G[6] + w * G[7] - 2.f * x * G[8]);
  gqn[2] = 2.f * (-2.f * y * G[0] + x * G[1] + w * G[2] + x * G[3] + zq * G[5] - w * G[6] + zq * G[7] - 2.f * y * G[8]);
  gqn[3] = 2.f * (-2.f * zq * G[0] - w * G[1] + x * G[2] + w * G[3] - 2.f * zq * G[4] + y * G[5] + x * G[6] + y * G[7]);
  const float dq = w * gqn[0] + x * gqn[1] + y * gqn[2] + zq * gqn[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) gq[k] = (gqn[k] - r.qn[k] * dq) / r.qnorm;
}

// View-independent part of a 3DGS projection, computed once per point and
// reused for all its views: world covariance Sg = (Rq S)(Rq S)^T (00 01 02 11
// 12 22) and the activated opacity.
struct PointPre {
  float Sg[6];
  float opac;
};

__device__ __forceinline__ void point_pre(const PointIn& pt, PointPre& r) {
  QuatFrame q;
  quat_frame(pt, 3, q);
  float M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[3 * i + j] = fmul(q.Rq[3 * i + j], q.s[j]);
  int k = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j)
      r.Sg[k++] = fadd(fadd(fmul(M[3 * i], M[3 * j]), fmul(M[3 * i + 1], M[3 * j + 1])), fmul(M[3 * i + 2], M[3 * j + 2]));
  r.opac = det_sigmoid(pt.op_logit);
}

// Gradient of the view-independent part: dL/dSg (accumulated over views,
// 6 unique entries) -> log scales (g[4..6]) and quaternion (g[8..11]).
__device__ __forceinline__ void point_pre_backward(const PointIn& pt, const float gS[6], float* g) {
  QuatFrame q;
  quat_frame(pt, 3, q);
  const float gSg[9] = {gS[0], gS[1], gS[2], gS[1], gS[3], gS[4], gS[2], gS[4], gS[5]};
  float M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[3 * i + j] = q.Rq[3 * i + j] * q.s[j];
  // Sg = M M^T, M = Rq S  ->  g_M = 2 g_Sg M
  float gM[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      gM[3 * i + j] = 2.f * (gSg[3 * i] * M[j] + gSg[3 * i + 1] * M[3 + j] + gSg[3 * i + 2] * M[6 + j]);
  float G[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float gs = q.Rq[j] * gM[j] + q.Rq[3 + j] * gM[3 + j] + q.Rq[6 + j] * gM[6 + j];
    g[4 + j] += gs * q.s[j];
#pragma unroll
    for (int i = 0; i < 3; ++i) G[3 * i + j] = gM[3 * i + j] * q.s[j];
  }
  float gq[4];
  quat_backward(q, G, gq);
#pragma unroll
  for (int k = 0; k < 4; ++k) g[8 + k] += gq[k];
}

template <class SH>
__device__ __forceinline__ void project_forward_t(const PointIn& pt, const PointPre& pre, const SH& sh,
                                                  const bs_camera& c, int n_sh, ProjFwd& f,
                                                  const float* gcol = nullptr, float* wk = nullptr) {
  // camera frame: q = Rcw (p - pos)
#pragma unroll
  for (int k = 0; k < 3; ++k) f.d[k] = fsub(pt.p[k], c.pos[k]);
#pragma unroll
  for (int k = 0; k < 3; ++k)
    f.qc[k] = fadd(fadd(fmul(c.rot_cw[3 * k], f.d[0]), fmul(c.rot_cw[3 * k + 1], f.d[1])),
                   fmul(c.rot_cw[3 * k + 2], f.d[2]));
  const float z = f.qc[2];
  const float Sg[9] = {pre.Sg[0], pre.Sg[1], pre.Sg[2], pre.Sg[1], pre.Sg[3], pre.Sg[4],
                       pre.Sg[2], pre.Sg[4], pre.Sg[5]};
  // Sc = W Sg W^T
  const float* W = c.rot_cw;
  float T[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      T[3 * i + j] = fadd(fadd(fmul(W[3 * i], Sg[j]), fmul(W[3 * i + 1], Sg[3 + j])), fmul(W[3 * i + 2], Sg[6 + j]));
  float Sc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const float v =
          fadd(fadd(fmul(T[3 * i], W[3 * j]), fmul(T[3 * i + 1], W[3 * j + 1])), fmul(T[3 * i + 2], W[3 * j + 2]));
      Sc[3 * i + j] = v;
      Sc[3 * j + i] = v;
    }
  f.Sc[0] = Sc[0]; f.Sc[1] = Sc[1]; f.Sc[2] = Sc[2]; f.Sc[3] = Sc[4]; f.Sc[4] = Sc[5]; f.Sc[5] = Sc[8];
  // EWA Jacobian with the usual clamp of x/z, y/z
  const float xr = fdiv(f.qc[0], z), yr = fdiv(f.qc[1], z);
  f.clamp_x = (xr < -c.lim_x) || (xr > c.lim_x);
  f.clamp_y = (yr < -c.lim_y) || (yr > c.lim_y);
  f.tx = fmul(fminf(c.lim_x, fmaxf(-c.lim_x, xr)), z);
  f.ty = fmul(fminf(c.lim_y, fmaxf(-c.lim_y, yr)), z);
  const float z2 = fmul(z, z);
  f.J00 = fdiv(c.fx, z);
  f.J11 = fdiv(c.fy, z);
  f.J02 = -fdiv(fmul(c.fx, f.tx), z2);
  f.J12 = -fdiv(fmul(c.fy, f.ty), z2);
  float U0[3], U1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    U0[j] = fadd(fmul(f.J00, Sc[j]), fmul(f.J02, Sc[6 + j]));
    U1[j] = fadd(fmul(f.J11, Sc[3 + j]), fmul(f.J12, Sc[6 + j]));
  }
  f.a = fadd(fadd(fmul(U0[0], f.J00), fmul(U0[2], f.J02)), kDilation);
  f.b = fadd(fmul(U0[1], f.J11), fmul(U0[2], f.J12));
  f.c = fadd(fadd(fmul(U1[1], f.J11), fmul(U1[2], f.J12)), kDilation);
  f.det = fsub(fmul(f.a, f.c), fmul(f.b, f.b));
  f.valid = f.det > 0.f;
  f.support_k = support_k(pre.opac);
  if (f.valid) {
    f.conic[0] = fdiv(f.c, f.det);
    f.conic[1] = fdiv(-f.b, f.det);
    f.conic[2] = fdiv(f.a, f.det);
    // per-axis extents = the tight bounding box of the support ellipse
    // q <= k, k = min(9, 2 ln(255 o)) (half-widths sqrt(k cov_xx), sqrt(k cov_yy))
    const float k = f.support_k;
    f.radius_x = k > 0.f ? fsqrt(fmul(k, f.a)) : 0.f;
    f.radius_y = k > 0.f ? fsqrt(fmul(k, f.c)) : 0.f;
  } else {
    f.conic[0] = f.conic[1] = f.conic[2] = 0.f;
    f.radius_x = f.radius_y = 0.f;
  }
  f.u = fadd(fmul(c.fx, xr), c.cx);
  f.v = fadd(fmul(c.fy, yr), c.cy);
  f.depth = z;
  // view-dependent colour
  f.len = fsqrt(fadd(fadd(fmul(f.d[0], f.d[0]), fmul(f.d[1], f.d[1])), fmul(f.d[2], f.d[2])));
#pragma unroll
  for (int k = 0; k < 3; ++k) f.dir[k] = fdiv(f.d[k], f.len);
  sh_basis(f.dir, n_sh, f.Y);
  sh_colour(sh, n_sh, f.Y, f.col_raw, f.col, gcol, wk);
  f.opac = pre.opac;
}

__device__ __forceinline__ void write_sp_row(float* __restrict__ row, const ProjFwd& f) {
  float4* r4 = reinterpret_cast<float4*>(row);
  r4[0] = make_float4(f.u, f.v, f.opac, f.conic[0]);
  r4[1] = make_float4(f.conic[1], f.conic[2], f.col[0], f.col[1]);
  r4[2] = make_float4(f.col[2], f.depth, f.valid ? f.radius_x : 0.f, f.valid ? f.radius_y : 0.f);
}

// G_SP rows from the rasteriser hold moments of dL/dpower over the pixels,
// power = -q/2, d = (u - px, v - py): M1 = sum dpow dx, M2 = sum dpow dy,
// M3..M5 = sum dpow (dx^2, dx dy, dy^2).  With conic (A, B, C):
// dL/du = -(A M1 + B M2), dL/dv = -(B M1 + C M2), dL/dA = -M3/2,
// dL/dB = -M4, dL/dC = -M5/2 (entries 2, 6..8 are already dL/dSP).
__device__ __forceinline__ void gsp_from_moments(const float conic[3], float* gs) {
  const float m1 = gs[0], m2 = gs[1];
  gs[0] = -(conic[0] * m1 + conic[1] * m2);
  gs[1] = -(conic[1] * m1 + conic[2] * m2);
  gs[3] = -0.5f * gs[3];
  gs[4] = -gs[4];
  gs[5] = -0.5f * gs[5];
}

// Gradient of the 60-float parameter row of one point (plane layout order:
// mean xyz, opacity logit, log scales xyz, pad, quat wxyz, sh[48]).
struct PointGrad {
  float g[60];
};

// dY_k/d(dir) accumulated against per-coefficient weights wk[k] = sum_ch dc*sh.
__device__ __forceinline__ void sh_dir_grad(const float dir[3], int n_sh, const float* wk, float gd[3]) {
  const float x = dir[0], y = dir[1], z = dir[2];
  gd[0] = gd[1] = gd[2] = 0.f;
  if (n_sh > 1) {
    gd[1] += -kSH_C1 * wk[1];
    gd[2] += kSH_C1 * wk[2];
    gd[0] += -kSH_C1 * wk[3];
  }
  if (n_sh > 4) {
    const float xx = x * x, yy = y * y, zz = z * z;
    gd[0] += kSH_C2_0 * y * wk[4];
    gd[1] += kSH_C2_0 * x * wk[4];
    gd[1] += kSH_C2_1 * z * wk[5];
    gd[2] += kSH_C2_1 * y * wk[5];
    gd[0] += -2.f * kSH_C2_2 * x * wk[6];
    gd[1] += -2.f * kSH_C2_2 * y * wk[6];
    gd[2] += 4.f * kSH_C2_2 * z * wk[6];
    gd[0] += kSH_C2_3 * z * wk[7];
    gd[2] += kSH_C2_3 * x * wk[7];
    gd[0] += 2.f * kSH_C2_4 * x * wk[8];
    gd[1] += -2.f * kSH_C2_4 * y * wk[8];
    if (n_sh > 9) {
      gd[0] += kSH_C3_0 * 6.f * x * y * wk[9];
      gd[1] += kSH_C3_0 * (3.f * xx - 3.f * yy) * wk[9];
      gd[0] += kSH_C3_1 * y * z * wk[10];
      gd[1] += kSH_C3_1 * x * z * wk[10];
      gd[2] += kSH_C3_1 * x * y * wk[10];
      gd[0] += kSH_C3_2 * (-2.f * x * y) * wk[11];
      gd[1] += kSH_C3_2 * (4.f * zz - xx - 3.f * yy) * wk[11];
      gd[2] += kSH_C3_2 * 8.f * y * z * wk[11];
      gd[0] += kSH_C3_3 * (-6.f * x * z) * wk[12];
      gd[1] += kSH_C3_3 * (-6.f * y * z) * wk[12];
      gd[2] += kSH_C3_3 * (6.f * zz - 3.f * xx - 3.f * yy) * wk[12];
      gd[0] += kSH_C3_4 * (4.f * zz - 3.f * xx - yy) * wk[13];
      gd[1] += kSH_C3_4 * (-2.f * x * y) * wk[13];
      gd[2] += kSH_C3_4 * 8.f * x * z * wk[13];
      gd[0] += kSH_C3_5 * 2.f * x * z * wk[14];
      gd[1] += kSH_C3_5 * (-2.f * y * z) * wk[14];
      gd[2] += kSH_C3_5 * (xx - yy) * wk[14];
      gd[0] += kSH_C3_6 * (3.f * xx - 3.f * yy) * wk[15];
      gd[1] += kSH_C3_6 * (-6.f * x * y) * wk[15];
    }
  }
}

// Accumulate d L / d params of one (point, view) pair: the 12 geometry
// floats (plane 0..2 order) into g, the SH coefficient gradients through
// sh_add(flat index f = 3k + channel, value).
// gsp = (du, dv, dopac, dA, dB, dC, dr, dg, db).
// gS accumulates dL/dSg (6 unique entries) for point_pre_backward.
template <class SH, class ShAdd>
__device__ __forceinline__ void project_backward_t(const PointIn& pt, const PointPre& pre, const SH& sh,
                                                   const bs_camera& c, int n_sh, const ProjFwd& f,
                                                   const float gsp[9], float* g, float gS[6], ShAdd& sh_add,
                                                   const float* wk_pre = nullptr) {
  if (!f.valid) return;
  // ---- colour -> sh, dir
  float wk[16];
  sh_colour_backward(sh, n_sh, f.Y, f.col_raw, gsp + 6, wk_pre, wk, sh_add);
  float gdir[3];
  sh_dir_grad(f.dir, n_sh, wk, gdir);
  const float dd = f.dir[0] * gdir[0] + f.dir[1] * gdir[1] + f.dir[2] * gdir[2];
  float gp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) gp[k] = (gdir[k] - f.dir[k] * dd) / f.len;
  // ---- opacity
  g[3] += gsp[2] * pre.opac * (1.f - pre.opac);
  // ---- means2d -> camera point
  const float z = f.qc[2], iz = 1.f / z, iz2 = iz * iz;
  float gq[3];
  gq[0] = gsp[0] * c.fx * iz;
  gq[1] = gsp[1] * c.fy * iz;
  gq[2] = -(gsp[0] * c.fx * f.qc[0] + gsp[1] * c.fy * f.qc[1]) * iz2;
  // ---- conic -> dilated 2D covariance
  const float A = gsp[3], Bg = gsp[4], Cg = gsp[5];
  const float a = f.a, b = f.b, cc = f.c;
  const float id2 = 1.f / (f.det * f.det);
  const float ga = (-cc * cc * A + b * cc * Bg - b * b * Cg) * id2;
  const float gb = (2.f * b * cc * A - (a * cc + b * b) * Bg + 2.f * a * b * Cg) * id2;
  const float gc = (-b * b * A + a * b * Bg - a * a * Cg) * id2;
  // ---- cov2d = J Sc J^T
  const float J0[3] = {f.J00, 0.f, f.J02};
  const float J1[3] = {0.f, f.J11, f.J12};
  const float Sc[9] = {f.Sc[0], f.Sc[1], f.Sc[2], f.Sc[1], f.Sc[3], f.Sc[4], f.Sc[2], f.Sc[4], f.Sc[5]};
  float gSc[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      gSc[3 * i + j] = ga * J0[i] * J0[j] + 0.5f * gb * (J0[i] * J1[j] + J1[i] * J0[j]) + gc * J1[i] * J1[j];
  float GJ0[3], GJ1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    GJ0[k] = ga * J0[k] + 0.5f * gb * J1[k];
    GJ1[k] = 0.5f * gb * J0[k] + gc * J1[k];
  }
  // g_J = 2 (Gm J) Sc
  float gJ00 = 0.f, gJ02 = 0.f, gJ11 = 0.f, gJ12 = 0.f;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    gJ00 += 2.f * GJ0[m] * Sc[3 * m + 0];
    gJ02 += 2.f * GJ0[m] * Sc[3 * m + 2];
    gJ11 += 2.f * GJ1[m] * Sc[3 * m + 1];
    gJ12 += 2.f * GJ1[m] * Sc[3 * m + 2];
  }
  // ---- J -> camera point
  gq[2] += -c.fx * iz2 * gJ00 - c.fy * iz2 * gJ11;
  if (!f.clamp_x) {
    gq[0] += -c.fx * iz2 * gJ02;
    gq[2] += 2.f * c.fx * f.qc[0] * iz2 * iz * gJ02;
  } else {
    gq[2] += c.fx * f.tx * iz2 * iz * gJ02;
  }
  if (!f.clamp_y) {
    gq[1] += -c.fy * iz2 * gJ12;
    gq[2] += 2.f * c.fy * f.qc[1] * iz2 * iz * gJ12;
  } else {
    gq[2] += c.fy * f.ty * iz2 * iz * gJ12;
  }
  // ---- camera point -> world mean: g_p += W^T g_q
  const float* W = c.rot_cw;
#pragma unroll
  for (int k = 0; k < 3; ++k) gp[k] += W[k] * gq[0] + W[3 + k] * gq[1] + W[6 + k] * gq[2];
  g[0] += gp[0];
  g[1] += gp[1];
  g[2] += gp[2];
  // ---- Sc = W Sg W^T  ->  g_Sg = W^T g_Sc W
  float tmp[9], gSg[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) tmp[3 * i + j] = W[i] * gSc[j] + W[3 + i] * gSc[3 + j] + W[6 + i] * gSc[6 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) gSg[3 * i + j] = tmp[3 * i] * W[j] + tmp[3 * i + 1] * W[3 + j] + tmp[3 * i + 2] * W[6 + j];
  gS[0] += gSg[0];
  gS[1] += gSg[1];
  gS[2] += gSg[2];
  gS[3] += gSg[4];
  gS[4] += gSg[5];
  gS[5] += gSg[8];
}

}  // namespace bs
