/*
 * CPU oracle of the PBDR training-step hot path (test infrastructure; see
 * splat_oracle.h).  Build: gcc -O2 -fopenmp -ffp-contract=off (no FMA
 * contraction: every float op rounds separately, so the projection below
 * performs exactly the op sequence of the sm_100a kernel and reproduces its
 * splat state bit-for-bit).
 *
 * Reference citations (/root/reference):
 *   culling / access counts  pkg/src/splatsched/visibility.py:153-161,
 *                            237-252, 263-292, 308-358
 *   Morton codes             visibility.py:33-62
 *   training step            PAPER.md:465-518 (Alg. 1), rendering outline
 *                            PAPER.md:264, splat state PAPER.md:1192-1200
 */
#include "splat_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16
#define SPF 12
#define GSPF 9

/* ------------------------------------------------------------------------ */
/* culling (visibility.py)                                                  */

/* p @ planes[:, :3].T + planes[:, 3] as OpenBLAS evaluates it for >= 2 rows
 * (visibility.py:155-156; order measured in SURVEY.md §0.6). */
static double pdist(const double* pl, double x, double y, double z) {
  return fma(z, pl[2], fma(y, pl[1], x * pl[0])) + pl[3];
}

/* d[i][k] for n points against m planes (exposed for the BLAS-order check) */
void or_plane_distances(const double* pts, int64_t n, const double* planes, int32_t m, double* out) {
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) out[i * m + k] = pdist(planes + 4 * k, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

/* plane pointer of a view block: 0 near, 1 far, 2+c x-edge c, 3+P+r y-edge r */
static const double* vplane(const double* vp, int k) { return vp + 4 * k; }

/* cull_group (visibility.py:263-276) for patch (r, c); 1 = OUTSIDE. */
static int group_outside(const double* vp, int P, int r, int c, const float* box) {
  const double* pl[6] = {vplane(vp, 0), vplane(vp, 1), vplane(vp, 2 + c), vplane(vp, 2 + c + 1),
                         vplane(vp, 3 + P + r), vplane(vp, 3 + P + r + 1)};
  const int neg[6] = {0, 0, 0, 1, 0, 1};
  for (int k = 0; k < 6; ++k) {
    int all = 1;
    for (int i = 0; i < 2 && all; ++i)
      for (int j = 0; j < 2 && all; ++j)
        for (int l = 0; l < 2 && all; ++l) {
          const double d = pdist(pl[k], (double)box[3 * i + 0], (double)box[3 * j + 1], (double)box[3 * l + 2]);
          /* the exclusive plane is the negation: -d < 0  <=>  d > 0 */
          all = neg[k] ? (d > 0.0) : (d < 0.0);
        }
    if (all) return 1;
  }
  return 0;
}

/* Frustum.contains for patch (r, c) (visibility.py:158-161). */
static int in_patch(const double* vp, int P, int r, int c, double x, double y, double z) {
  if (!(pdist(vplane(vp, 0), x, y, z) >= 0.0)) return 0;
  if (!(pdist(vplane(vp, 1), x, y, z) >= 0.0)) return 0;
  if (!(pdist(vplane(vp, 2 + c), x, y, z) >= 0.0)) return 0;
  if (!(-pdist(vplane(vp, 2 + c + 1), x, y, z) > 0.0)) return 0;
  if (!(pdist(vplane(vp, 3 + P + r), x, y, z) >= 0.0)) return 0;
  if (!(-pdist(vplane(vp, 3 + P + r + 1), x, y, z) > 0.0)) return 0;
  return 1;
}

void or_access_matrix(const float* pos, int64_t n, const int32_t* gb, const float* aabb, int32_t ng,
                      const double* planes, int32_t B, int32_t P, const int32_t* point_gpu, int32_t N, int32_t mode,
                      const float* presence, const float* view_times, int64_t* out) {
  (void)n;
  const int npl = 2 + 2 * (P + 1);
  memset(out, 0, sizeof(int64_t) * (size_t)B * P * P * N);
  for (int v = 0; v < B; ++v) {
    const double* vp = planes + (size_t)v * npl * 4;
    for (int r = 0; r < P; ++r)
      for (int c = 0; c < P; ++c) {
        int64_t* row = out + ((size_t)v * P * P + r * P + c) * N;
        for (int g = 0; g < ng; ++g) {
          if (aabb && group_outside(vp, P, r, c, aabb + 6 * (size_t)g)) continue; /* _candidate_indices */
          for (int i = gb[g]; i < gb[g + 1]; ++i) {
            int ok = 1;
            if (mode == 0) {
              ok = in_patch(vp, P, r, c, pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]);
              if (ok && presence) {
                const float t = view_times[v]; /* f32 compare (visibility.py:251) */
                ok = (presence[2 * (size_t)i] <= t) && (t <= presence[2 * (size_t)i + 1]);
              }
            }
            if (ok) row[point_gpu ? point_gpu[i] : 0] += 1;
          }
        }
      }
  }
}

void or_visibility_mask(const float* pos, int64_t n, const int32_t* gb, const float* aabb, int32_t ng,
                        const double* planes, int32_t B, uint32_t* mask) {
  memset(mask, 0, sizeof(uint32_t) * (size_t)n);
  const int npl = 6;
  for (int v = 0; v < B; ++v) {
    const double* vp = planes + (size_t)v * npl * 4;
    for (int g = 0; g < ng; ++g) {
      if (aabb && group_outside(vp, 1, 0, 0, aabb + 6 * (size_t)g)) continue;
      for (int i = gb[g]; i < gb[g + 1]; ++i)
        if (in_patch(vp, 1, 0, 0, pos[3 * (size_t)i], pos[3 * (size_t)i + 1], pos[3 * (size_t)i + 2]))
          mask[i] |= 1u << v;
    }
  }
}

/* _quantize + _interleave3 (visibility.py:33-52) */
void or_morton(const float* pos, int64_t n, const float* bbox, int32_t bits, uint64_t* codes) {
  const double scale = (double)((1ull << bits) - 1);
  double mn[3], ext[3];
  for (int k = 0; k < 3; ++k) {
    mn[k] = (double)bbox[k];
    ext[k] = (double)bbox[3 + k] - mn[k];
    if (ext[k] == 0.0) ext[k] = 1.0;
  }
  for (int64_t i = 0; i < n; ++i) {
    uint64_t q[3];
    for (int k = 0; k < 3; ++k) {
      double t = floor(((double)pos[3 * i + k] - mn[k]) / ext[k] * scale);
      if (t < 0) t = 0;
      if (t > scale) t = scale;
      q[k] = (uint64_t)t;
    }
    uint64_t code = 0;
    for (int b = 0; b < bits; ++b) {
      code |= ((q[0] >> b) & 1ull) << (3 * b);
      code |= ((q[1] >> b) & 1ull) << (3 * b + 1);
      code |= ((q[2] >> b) & 1ull) << (3 * b + 2);
    }
    codes[i] = code;
  }
}

/* ------------------------------------------------------------------------ */
/* projection (pts_splatting) -- same op sequence as csrc/splat_math.cuh     */

static const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
static const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                            -1.0925484305920792f, 0.5462742152960396f};
static const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                            0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                            -0.5900435899266435f};

typedef union {
  float f;
  uint32_t u;
} fbits;

float or_det_expf(float x) {
  x = fminf(fmaxf(x, -80.0f), 80.0f);
  const float n = rintf(x * 0x1.715476p+0f);
  float r = x - n * 0x1.62e400p-1f;
  r = r - n * 0x1.7f7d1cp-20f;
  float p = 0x1.6c16c2p-10f;
  p = p * r + 0x1.111112p-7f;
  p = p * r + 0x1.555556p-5f;
  p = p * r + 0x1.555556p-3f;
  p = p * r + 0x1.000000p-1f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  fbits s;
  s.u = (uint32_t)((int)n + 127) << 23;
  return p * s.f;
}

/* ln(x), same op sequence as csrc/common.cuh det_logf */
float or_det_logf(float x) {
  if (!(x >= 1.17549435e-38f)) return -87.5f;
  fbits b;
  b.f = x;
  int e = (int)(b.u >> 23) - 127;
  fbits mb;
  mb.u = (b.u & 0x7fffffu) | 0x3f800000u;
  float m = mb.f;
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e += 1;
  }
  const float s = (m - 1.0f) / (m + 1.0f);
  const float s2 = s * s;
  float p = 0x1.c71c72p-4f;
  p = p * s2 + 0x1.249250p-3f;
  p = p * s2 + 0x1.99999ap-3f;
  p = p * s2 + 0x1.555556p-2f;
  p = p * s2 + 1.0f;
  const float lnm = (2.0f * s) * p;
  const float fe = (float)e;
  return fe * 0x1.62e400p-1f + (lnm + fe * 0x1.7f7d1cp-20f);
}

typedef struct {
  float p[3], op, ls[3], q[4], sh[48];
} opoint;

typedef struct {
  float d[3], qc[3], s[3], qn[4], qnorm, Rq[9], Sc[9];
  float J00, J02, J11, J12, tx, ty;
  int clamp_x, clamp_y;
  float a, b, c, det, conic[3], radius_x, radius_y, u, v, depth, len, dir[3], Y[16], col_raw[3], col[3], opac;
  int valid;
} oproj;

static void load_opoint(const float* params, int64_t S, int64_t i, opoint* pt) {
  const float* p0 = params + 4 * i;
  const float* p1 = params + 4 * (S + i);
  const float* p2 = params + 4 * (2 * S + i);
  for (int k = 0; k < 3; ++k) pt->p[k] = p0[k];
  pt->op = p0[3];
  for (int k = 0; k < 3; ++k) pt->ls[k] = p1[k];
  for (int k = 0; k < 4; ++k) pt->q[k] = p2[k];
  for (int f = 0; f < 48; ++f) pt->sh[f] = params[4 * ((3 + f / 4) * S + i) + (f % 4)];
}

static void sh_basis(const float* dir, int n_sh, float* Y) {
  const float x = dir[0], y = dir[1], z = dir[2];
  for (int k = 0; k < 16; ++k) Y[k] = 0.f;
  Y[0] = C0;
  if (n_sh > 1) {
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
  }
  if (n_sh > 4) {
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = C2[0] * xy;
    Y[5] = C2[1] * yz;
    Y[6] = C2[2] * ((2.f * zz - xx) - yy);
    Y[7] = C2[3] * xz;
    Y[8] = C2[4] * (xx - yy);
    if (n_sh > 9) {
      Y[9] = (C3[0] * y) * (3.f * xx - yy);
      Y[10] = (C3[1] * xy) * z;
      Y[11] = (C3[2] * y) * ((4.f * zz - xx) - yy);
      Y[12] = (C3[3] * z) * ((2.f * zz - 3.f * xx) - 3.f * yy);
      Y[13] = (C3[4] * x) * ((4.f * zz - xx) - yy);
      Y[14] = (C3[5] * z) * (xx - yy);
      Y[15] = (C3[6] * x) * (xx - 3.f * yy);
    }
  }
}

static void proj_fwd(const opoint* pt, const or_camera* c, int n_sh, oproj* f) {
  for (int k = 0; k < 3; ++k) f->d[k] = pt->p[k] - c->pos[k];
  for (int k = 0; k < 3; ++k)
    f->qc[k] = (c->rot_cw[3 * k] * f->d[0] + c->rot_cw[3 * k + 1] * f->d[1]) + c->rot_cw[3 * k + 2] * f->d[2];
  const float z = f->qc[2];
  for (int k = 0; k < 3; ++k) f->s[k] = or_det_expf(pt->ls[k]);
  const float nn = ((pt->q[0] * pt->q[0] + pt->q[1] * pt->q[1]) + pt->q[2] * pt->q[2]) + pt->q[3] * pt->q[3];
  f->qnorm = sqrtf(nn);
  for (int k = 0; k < 4; ++k) f->qn[k] = pt->q[k] / f->qnorm;
  const float w = f->qn[0], x = f->qn[1], y = f->qn[2], zq = f->qn[3];
  const float xx = x * x, yy = y * y, zz = zq * zq, xy = x * y, xz = x * zq, yz = y * zq;
  const float wx = w * x, wy = w * y, wz = w * zq;
  float* R = f->Rq;
  R[0] = 1.f - 2.f * (yy + zz);
  R[1] = 2.f * (xy - wz);
  R[2] = 2.f * (xz + wy);
  R[3] = 2.f * (xy + wz);
  R[4] = 1.f - 2.f * (xx + zz);
  R[5] = 2.f * (yz - wx);
  R[6] = 2.f * (xz - wy);
  R[7] = 2.f * (yz + wx);
  R[8] = 1.f - 2.f * (xx + yy);
  float M[9], Sg[9], T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M[3 * i + j] = R[3 * i + j] * f->s[j];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      const float v = (M[3 * i] * M[3 * j] + M[3 * i + 1] * M[3 * j + 1]) + M[3 * i + 2] * M[3 * j + 2];
      Sg[3 * i + j] = v;
      Sg[3 * j + i] = v;
    }
  const float* W = c->rot_cw;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = (W[3 * i] * Sg[j] + W[3 * i + 1] * Sg[3 + j]) + W[3 * i + 2] * Sg[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      const float v = (T[3 * i] * W[3 * j] + T[3 * i + 1] * W[3 * j + 1]) + T[3 * i + 2] * W[3 * j + 2];
      f->Sc[3 * i + j] = v;
      f->Sc[3 * j + i] = v;
    }
  const float* Sc = f->Sc;
  const float xr = f->qc[0] / z, yr = f->qc[1] / z;
  f->clamp_x = (xr < -c->lim_x) || (xr > c->lim_x);
  f->clamp_y = (yr < -c->lim_y) || (yr > c->lim_y);
  f->tx = fminf(c->lim_x, fmaxf(-c->lim_x, xr)) * z;
  f->ty = fminf(c->lim_y, fmaxf(-c->lim_y, yr)) * z;
  const float z2 = z * z;
  f->J00 = c->fx / z;
  f->J11 = c->fy / z;
  f->J02 = -((c->fx * f->tx) / z2);
  f->J12 = -((c->fy * f->ty) / z2);
  float U0[3], U1[3];
  for (int j = 0; j < 3; ++j) {
    U0[j] = f->J00 * Sc[j] + f->J02 * Sc[6 + j];
    U1[j] = f->J11 * Sc[3 + j] + f->J12 * Sc[6 + j];
  }
  f->a = (U0[0] * f->J00 + U0[2] * f->J02) + 0.3f;
  f->b = U0[1] * f->J11 + U0[2] * f->J12;
  f->c = (U1[1] * f->J11 + U1[2] * f->J12) + 0.3f;
  f->det = f->a * f->c - f->b * f->b;
  f->valid = f->det > 0.f;
  if (f->valid) {
    f->conic[0] = f->c / f->det;
    f->conic[1] = (-f->b) / f->det;
    f->conic[2] = f->a / f->det;
    /* support box: q <= k, k = min(9, 2 ln(255 o)) (csrc/common.cuh support_k) */
    const float o = 1.f / (1.f + or_det_expf(-pt->op));
    const float k = fminf(9.0f, 2.0f * or_det_logf(255.0f * o));
    f->radius_x = k > 0.f ? sqrtf(k * f->a) : 0.f;
    f->radius_y = k > 0.f ? sqrtf(k * f->c) : 0.f;
  } else {
    f->conic[0] = f->conic[1] = f->conic[2] = 0.f;
    f->radius_x = f->radius_y = 0.f;
  }
  f->u = c->fx * xr + c->cx;
  f->v = c->fy * yr + c->cy;
  f->depth = z;
  f->len = sqrtf((f->d[0] * f->d[0] + f->d[1] * f->d[1]) + f->d[2] * f->d[2]);
  for (int k = 0; k < 3; ++k) f->dir[k] = f->d[k] / f->len;
  sh_basis(f->dir, n_sh, f->Y);
  for (int ch = 0; ch < 3; ++ch) {
    float acc = f->Y[0] * pt->sh[ch];
    for (int k = 1; k < n_sh; ++k) acc = acc + f->Y[k] * pt->sh[3 * k + ch];
    f->col_raw[ch] = acc + 0.5f;
    f->col[ch] = fmaxf(f->col_raw[ch], 0.f);
  }
  f->opac = 1.f / (1.f + or_det_expf(-pt->op));
}

void or_project(const float* params, int64_t S, const int64_t* idx, int64_t m, const or_camera* c, int32_t sh_degree,
                float* sp) {
  const int n_sh = (sh_degree + 1) * (sh_degree + 1);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k) {
    opoint pt;
    oproj f;
    load_opoint(params, S, idx[k], &pt);
    proj_fwd(&pt, c, n_sh, &f);
    float* r = sp + k * SPF;
    r[0] = f.u;
    r[1] = f.v;
    r[2] = f.opac;
    r[3] = f.conic[0];
    r[4] = f.conic[1];
    r[5] = f.conic[2];
    r[6] = f.col[0];
    r[7] = f.col[1];
    r[8] = f.col[2];
    r[9] = f.depth;
    r[10] = f.valid ? f.radius_x : 0.f;
    r[11] = f.valid ? f.radius_y : 0.f;
  }
}

/* Analytic backward of proj_fwd (chain rule written out independently of the
 * CUDA file; checked against float64 autograd in tests). */
static void proj_bwd(const opoint* pt, const or_camera* c, int n_sh, const oproj* f, const float* gsp_m, float* g) {
  if (!f->valid) return;
  /* G_SP moments -> dL/d(u, v, opacity, conic, rgb) with this view's conic */
  float gsp[9];
  for (int k = 0; k < 9; ++k) gsp[k] = gsp_m[k];
  gsp[0] = -(f->conic[0] * gsp_m[0] + f->conic[1] * gsp_m[1]);
  gsp[1] = -(f->conic[1] * gsp_m[0] + f->conic[2] * gsp_m[1]);
  gsp[3] = -0.5f * gsp_m[3];
  gsp[4] = -gsp_m[4];
  gsp[5] = -0.5f * gsp_m[5];
  float dc[3];
  for (int ch = 0; ch < 3; ++ch) dc[ch] = f->col_raw[ch] >= 0.f ? gsp[6 + ch] : 0.f;
  float wk[16] = {0};
  for (int k = 0; k < n_sh; ++k)
    for (int ch = 0; ch < 3; ++ch) {
      g[12 + 3 * k + ch] += f->Y[k] * dc[ch];
      wk[k] += dc[ch] * pt->sh[3 * k + ch];
    }
  /* gradient of sum_k wk[k] Y_k(dir) w.r.t. dir */
  const float x = f->dir[0], y = f->dir[1], z = f->dir[2];
  float gd[3] = {0, 0, 0};
  if (n_sh > 1) {
    gd[1] -= C1 * wk[1];
    gd[2] += C1 * wk[2];
    gd[0] -= C1 * wk[3];
  }
  if (n_sh > 4) {
    gd[0] += C2[0] * y * wk[4];
    gd[1] += C2[0] * x * wk[4];
    gd[1] += C2[1] * z * wk[5];
    gd[2] += C2[1] * y * wk[5];
    gd[0] -= 2.f * C2[2] * x * wk[6];
    gd[1] -= 2.f * C2[2] * y * wk[6];
    gd[2] += 4.f * C2[2] * z * wk[6];
    gd[0] += C2[3] * z * wk[7];
    gd[2] += C2[3] * x * wk[7];
    gd[0] += 2.f * C2[4] * x * wk[8];
    gd[1] -= 2.f * C2[4] * y * wk[8];
  }
  if (n_sh > 9) {
    const float xx = x * x, yy = y * y, zz = z * z;
    /* Y9 = C3_0 (3 x^2 y - y^3) */
    gd[0] += C3[0] * 6.f * x * y * wk[9];
    gd[1] += C3[0] * 3.f * (xx - yy) * wk[9];
    /* Y10 = C3_1 x y z */
    gd[0] += C3[1] * y * z * wk[10];
    gd[1] += C3[1] * x * z * wk[10];
    gd[2] += C3[1] * x * y * wk[10];
    /* Y11 = C3_2 (4 y z^2 - x^2 y - y^3) */
    gd[0] += C3[2] * (-2.f * x * y) * wk[11];
    gd[1] += C3[2] * (4.f * zz - xx - 3.f * yy) * wk[11];
    gd[2] += C3[2] * (8.f * y * z) * wk[11];
    /* Y12 = C3_3 (2 z^3 - 3 x^2 z - 3 y^2 z) */
    gd[0] += C3[3] * (-6.f * x * z) * wk[12];
    gd[1] += C3[3] * (-6.f * y * z) * wk[12];
    gd[2] += C3[3] * (6.f * zz - 3.f * xx - 3.f * yy) * wk[12];
    /* Y13 = C3_4 (4 x z^2 - x^3 - x y^2) */
    gd[0] += C3[4] * (4.f * zz - 3.f * xx - yy) * wk[13];
    gd[1] += C3[4] * (-2.f * x * y) * wk[13];
    gd[2] += C3[4] * (8.f * x * z) * wk[13];
    /* Y14 = C3_5 (x^2 z - y^2 z) */
    gd[0] += C3[5] * (2.f * x * z) * wk[14];
    gd[1] += C3[5] * (-2.f * y * z) * wk[14];
    gd[2] += C3[5] * (xx - yy) * wk[14];
    /* Y15 = C3_6 (x^3 - 3 x y^2) */
    gd[0] += C3[6] * 3.f * (xx - yy) * wk[15];
    gd[1] += C3[6] * (-6.f * x * y) * wk[15];
  }
  const float dd = x * gd[0] + y * gd[1] + z * gd[2];
  float gp[3];
  for (int k = 0; k < 3; ++k) gp[k] = (gd[k] - f->dir[k] * dd) / f->len;
  g[3] += gsp[2] * f->opac * (1.f - f->opac);
  const float zc = f->qc[2];
  float gq[3];
  gq[0] = gsp[0] * c->fx / zc;
  gq[1] = gsp[1] * c->fy / zc;
  gq[2] = -(gsp[0] * c->fx * f->qc[0] + gsp[1] * c->fy * f->qc[1]) / (zc * zc);
  /* conic = inv(cov2d): d conic / d (a, b, c) */
  const float A = gsp[3], Bg = gsp[4], Cg = gsp[5];
  const float a = f->a, b = f->b, cc = f->c, det2 = f->det * f->det;
  const float ga = (-cc * cc * A + b * cc * Bg - b * b * Cg) / det2;
  const float gb = (2.f * b * cc * A - (a * cc + b * b) * Bg + 2.f * a * b * Cg) / det2;
  const float gc = (-b * b * A + a * b * Bg - a * a * Cg) / det2;
  /* cov2d = J Sc J^T with J = [[J00, 0, J02], [0, J11, J12]] */
  const float J[2][3] = {{f->J00, 0.f, f->J02}, {0.f, f->J11, f->J12}};
  const float Gm[2][2] = {{ga, 0.5f * gb}, {0.5f * gb, gc}};
  float gSc[9] = {0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int r = 0; r < 2; ++r)
        for (int s = 0; s < 2; ++s) gSc[3 * i + j] += J[r][i] * Gm[r][s] * J[s][j];
  float gJ[2][3] = {{0}};
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 3; ++k)
      for (int s = 0; s < 2; ++s)
        for (int m = 0; m < 3; ++m) gJ[r][k] += 2.f * Gm[r][s] * J[s][m] * f->Sc[3 * m + k];
  const float iz2 = 1.f / (zc * zc), iz3 = iz2 / zc;
  gq[2] += -c->fx * iz2 * gJ[0][0] - c->fy * iz2 * gJ[1][1];
  if (!f->clamp_x) {
    gq[0] += -c->fx * iz2 * gJ[0][2];
    gq[2] += 2.f * c->fx * f->qc[0] * iz3 * gJ[0][2];
  } else {
    gq[2] += c->fx * f->tx * iz3 * gJ[0][2];
  }
  if (!f->clamp_y) {
    gq[1] += -c->fy * iz2 * gJ[1][2];
    gq[2] += 2.f * c->fy * f->qc[1] * iz3 * gJ[1][2];
  } else {
    gq[2] += c->fy * f->ty * iz3 * gJ[1][2];
  }
  const float* W = c->rot_cw;
  for (int k = 0; k < 3; ++k) g[k] += gp[k] + W[k] * gq[0] + W[3 + k] * gq[1] + W[6 + k] * gq[2];
  /* Sc = W Sg W^T */
  float gSg[9] = {0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) gSg[3 * i + j] += W[3 * r + i] * gSc[3 * r + s] * W[3 * s + j];
  /* Sg = M M^T, M = R diag(s) */
  float M[9], gM[9] = {0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M[3 * i + j] = f->Rq[3 * i + j] * f->s[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k) gM[3 * i + j] += (gSg[3 * i + k] + gSg[3 * k + i]) * M[3 * k + j];
  float G[9];
  for (int j = 0; j < 3; ++j) {
    float gs = 0.f;
    for (int i = 0; i < 3; ++i) {
      gs += f->Rq[3 * i + j] * gM[3 * i + j];
      G[3 * i + j] = gM[3 * i + j] * f->s[j];
    }
    g[4 + j] += gs * f->s[j];
  }
  const float w = f->qn[0], qx = f->qn[1], qy = f->qn[2], qz = f->qn[3];
  float gqn[4];
  gqn[0] = 2.f * (-qz * G[1] + qy * G[2] + qz * G[3] - qx * G[5] - qy * G[6] + qx * G[7]);
  gqn[1] = 2.f * (qy * G[1] + qz * G[2] + qy * G[3] - 2.f * qx * G[4] - w * G[5] + qz * G[6] + w * G[7] - 2.f * qx * G[8]);
  gqn[2] = 2.f * (-2.f * qy * G[0] + qx * G[1] + w * G[2] + qx * G[3] + qz * G[5] - w * G[6] + qz * G[7] - 2.f * qy * G[8]);
  gqn[3] = 2.f * (-2.f * qz * G[0] - w * G[1] + qx * G[2] + w * G[3] - 2.f * qz * G[4] + qy * G[5] + qx * G[6] + qy * G[7]);
  const float dq = w * gqn[0] + qx * gqn[1] + qy * gqn[2] + qz * gqn[3];
  for (int k = 0; k < 4; ++k) g[8 + k] += (gqn[k] - f->qn[k] * dq) / f->qnorm;
}

void or_project_bwd(const float* params, int64_t S, const int64_t* idx, int64_t m, const or_camera* c,
                    int32_t sh_degree, const float* gsp, float* grad_params) {
  const int n_sh = (sh_degree + 1) * (sh_degree + 1);
  for (int64_t k = 0; k < m; ++k) {
    opoint pt;
    oproj f;
    float g[60] = {0};
    const int64_t i = idx[k];
    load_opoint(params, S, i, &pt);
    proj_fwd(&pt, c, n_sh, &f);
    proj_bwd(&pt, c, n_sh, &f, gsp + k * GSPF, g);
    for (int p = 0; p < 15; ++p)
      for (int l = 0; l < 4; ++l) grad_params[4 * (p * S + i) + l] += g[4 * p + l];
  }
}

/* ------------------------------------------------------------------------ */
/* binning + rasterisation                                                   */

typedef struct {
  uint32_t tile, depth_bits, row;
} oinst;

static int inst_cmp(const void* pa, const void* pb) {
  const oinst* a = (const oinst*)pa;
  const oinst* b = (const oinst*)pb;
  if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
  if (a->depth_bits != b->depth_bits) return a->depth_bits < b->depth_bits ? -1 : 1;
  return a->row < b->row ? -1 : (a->row > b->row);
}

/* tiles whose span meets [u - r, u + r] of the support box centred at
 * (row[ctr], row[ctr + 1]) (same f32 ops as csrc/tile.cuh) */
static int tile_rect_at(const float* row, int rad, int ctr, int W, int H, int* x0, int* x1, int* y0, int* y1) {
  const float u = row[ctr], v = row[ctr + 1], rx = row[rad], ry = row[rad + 1];
  if (!(rx > 0.f) || !(ry > 0.f)) return 0;
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  *x0 = (int)fminf(fmaxf(floorf((u - rx) * 0.0625f), 0.f), (float)tx);
  *x1 = (int)fminf(fmaxf(floorf((u + rx) * 0.0625f) + 1.f, 0.f), (float)tx);
  *y0 = (int)fminf(fmaxf(floorf((v - ry) * 0.0625f), 0.f), (float)ty);
  *y1 = (int)fminf(fmaxf(floorf((v + ry) * 0.0625f) + 1.f, 0.f), (float)ty);
  if (*x1 <= *x0 || *y1 <= *y0) return 0;
  return (*x1 - *x0) * (*y1 - *y0);
}

/* row geometry: 3DGS rows {12 floats, radii at 10, depth at 9}, 2DGS {24, 16, 15} */
typedef struct {
  int stride, rad, depth, ctr;
} olayout;
static const olayout LAY3 = {SPF, 10, 9, 0};
static const olayout LAY2 = {24, 16, 15, 22};

static oinst* bin_view_l(const float* sp, int64_t m, int W, int H, olayout L, int64_t* n_out, int32_t* ranges) {
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  int64_t total = 0;
  int x0, x1, y0, y1;
  for (int64_t k = 0; k < m; ++k) total += tile_rect_at(sp + k * L.stride, L.rad, L.ctr, W, H, &x0, &x1, &y0, &y1);
  oinst* inst = (oinst*)malloc(sizeof(oinst) * (size_t)(total > 0 ? total : 1));
  int64_t o = 0;
  for (int64_t k = 0; k < m; ++k) {
    const float* r = sp + k * L.stride;
    if (!tile_rect_at(r, L.rad, L.ctr, W, H, &x0, &x1, &y0, &y1)) continue;
    fbits db;
    db.f = r[L.depth];
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) {
        inst[o].tile = (uint32_t)(y * tx + x);
        inst[o].depth_bits = db.u;
        inst[o].row = (uint32_t)k;
        ++o;
      }
  }
  qsort(inst, (size_t)total, sizeof(oinst), inst_cmp);
  for (int t = 0; t < tx * ty; ++t) ranges[2 * t] = ranges[2 * t + 1] = 0;
  for (int64_t i = 0; i < total; ++i) {
    const uint32_t t = inst[i].tile;
    if (i == 0 || inst[i - 1].tile != t) ranges[2 * t] = (int32_t)i;
    if (i == total - 1 || inst[i + 1].tile != t) ranges[2 * t + 1] = (int32_t)(i + 1);
  }
  *n_out = total;
  return inst;
}

static oinst* bin_view(const float* sp, int64_t m, int W, int H, int64_t* n_out, int32_t* ranges) {
  return bin_view_l(sp, m, W, H, LAY3, n_out, ranges);
}

/* Per-pixel exponent in log2 units, in the op order of csrc/raster.cu
 * (stage + splat_power2): the conic pre-scaled by -log2(e)/2 (B by -log2(e)),
 * d = (u - px, v - py), p2 = fma(kB, dx dy, kA dx^2) + kC dy^2.  Bit-identical
 * to the kernels, so every keep/skip decision is the same. */
#define LOG2E_F 1.4426950408889634f
static float splat_p2(const float* r, float px, float py, float* dx, float* dy) {
  const float kA = r[3] * (-0.5f * LOG2E_F), kC = r[5] * (-0.5f * LOG2E_F), kB = r[4] * -LOG2E_F;
  *dx = r[0] + (-px);
  *dy = r[1] + (-py);
  const float tx = ((*dx) * (*dx)) * kA, ty = ((*dy) * (*dy)) * kC;
  return fmaf(kB, (*dx) * (*dy), tx) + ty;
}

/* Support of a splat at a pixel: q <= k, k = min(9, 2 ln(255 o)) (the
 * alpha >= 1/255 test and the 3-sigma cut as one threshold on the exponent,
 * computed with the shared deterministic log: csrc/raster.cu support_p2) */
static float support_p2(float o) {
  const float k = fminf(9.0f, 2.0f * or_det_logf(255.0f * o));
  return k * (-0.5f * LOG2E_F);
}

/* the support threshold of every row, computed once (bs_row_support):
 * 3DGS the log2-exponent threshold, 2DGS k; opacity is float 2 of both rows */
static float* row_support(const float* sp, int64_t m, int stride, int two_d) {
  float* out = (float*)malloc(sizeof(float) * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k) {
    const float o = sp[k * stride + 2];
    out[k] = two_d ? fminf(9.0f, 2.0f * or_det_logf(255.0f * o)) : support_p2(o);
  }
  return out;
}

int32_t or_render(const float* sp, int64_t m, int32_t W, int32_t H, const float* bg, float* image, float* final_T,
                  int32_t* n_contrib, uint32_t* tile_lists, int64_t* n_inst, int32_t* tile_ranges) {
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  int32_t* ranges = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)tx * ty);
  int64_t total = 0;
  oinst* inst = bin_view(sp, m, W, H, &total, ranges);
  if (tile_lists) {
    if (*n_inst < total) {
      *n_inst = total;
      free(inst);
      free(ranges);
      return 1;
    }
    for (int64_t i = 0; i < total; ++i) tile_lists[i] = inst[i].row;
    memcpy(tile_ranges, ranges, sizeof(int32_t) * 2 * (size_t)tx * ty);
  }
  if (n_inst) *n_inst = total;
  float* sup = row_support(sp, m, SPF, 0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int t = 0; t < tx * ty; ++t) {
    const int bx = t % tx, by = t / tx;
    for (int ly = 0; ly < TILE; ++ly)
      for (int lx = 0; lx < TILE; ++lx) {
        const int px = bx * TILE + lx, py = by * TILE + ly;
        if (px >= W || py >= H) continue;
        const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
        float T = 1.f, C[3] = {0, 0, 0};
        int contrib = 0;
        for (int i = ranges[2 * t]; i < ranges[2 * t + 1]; ++i) {
          const float* r = sp + (int64_t)inst[i].row * SPF;
          float dx, dy;
          const float p2 = splat_p2(r, pxf, pyf, &dx, &dy);
          if (p2 > 0.f || p2 < sup[inst[i].row]) continue; /* outside the support (q > k) */
          const float alpha = fminf(0.99f, r[2] * exp2f(p2));
          const float nT = T * (1.f - alpha);
          if (nT < 1e-4f) break;
          const float w = alpha * T;
          for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(r[6 + ch], w, C[ch]);
          T = nT;
          contrib = i + 1 - ranges[2 * t];
        }
        const int64_t pix = (int64_t)py * W + px;
        for (int ch = 0; ch < 3; ++ch) image[3 * pix + ch] = C[ch] + T * bg[ch];
        final_T[pix] = T;
        n_contrib[pix] = contrib;
      }
  }
  free(inst);
  free(sup);
  free(ranges);
  return 0;
}

int32_t or_render_bwd(const float* sp, int64_t m, int32_t W, int32_t H, const float* bg, const float* final_T,
                      const int32_t* n_contrib, const float* grad_image, float* gsp) {
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  int32_t* ranges = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)tx * ty);
  int64_t total = 0;
  oinst* inst = bin_view(sp, m, W, H, &total, ranges);
  float* sup = row_support(sp, m, SPF, 0);
  memset(gsp, 0, sizeof(float) * GSPF * (size_t)m);
  /* serial over tiles: gradient sums are order-sensitive only at fp32 level */
  for (int t = 0; t < tx * ty; ++t) {
    const int bx = t % tx, by = t / tx;
    for (int ly = 0; ly < TILE; ++ly)
      for (int lx = 0; lx < TILE; ++lx) {
        const int px = bx * TILE + lx, py = by * TILE + ly;
        if (px >= W || py >= H) continue;
        const int64_t pix = (int64_t)py * W + px;
        const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
        const float* dC = grad_image + 3 * pix;
        const float T_final = final_T[pix];
        const float bgdot = bg[0] * dC[0] + bg[1] * dC[1] + bg[2] * dC[2];
        float T = T_final, acc[3] = {0, 0, 0}, last_alpha = 0.f, lc[3] = {0, 0, 0};
        const int r0 = ranges[2 * t];
        for (int i = r0 + n_contrib[pix] - 1; i >= r0; --i) {
          const int64_t row = inst[i].row;
          const float* r = sp + row * SPF;
          float dx, dy;
          const float p2 = splat_p2(r, pxf, pyf, &dx, &dy);
          if (p2 > 0.f || p2 < sup[row]) continue; /* outside the support (q > k) */
          const float ex = exp2f(p2);
          const float raw = r[2] * ex;
          const float alpha = fminf(0.99f, raw);
          const float ra = 1.f / (1.f - alpha);
          T = T * ra;
          float* g = gsp + row * GSPF;
          const float fac = alpha * T;
          for (int ch = 0; ch < 3; ++ch) g[6 + ch] += fac * dC[ch];
          for (int ch = 0; ch < 3; ++ch) acc[ch] = last_alpha * lc[ch] + (1.f - last_alpha) * acc[ch];
          last_alpha = alpha;
          for (int ch = 0; ch < 3; ++ch) lc[ch] = r[6 + ch];
          float dL_da = 0.f;
          for (int ch = 0; ch < 3; ++ch) dL_da += (r[6 + ch] - acc[ch]) * dC[ch];
          dL_da = T * dL_da - T_final * ra * bgdot;
          if (raw > 0.99f) continue; /* clamped alpha: no gradient to opacity/geometry */
          /* G_SP: moments of dpow = dL/dpower (include/splat_b200.h) */
          const float dpow = dL_da * alpha;
          g[2] += dL_da * ex;
          g[0] += dpow * dx;
          g[1] += dpow * dy;
          g[3] += dpow * dx * dx;
          g[4] += dpow * dx * dy;
          g[5] += dpow * dy * dy;
        }
      }
  }
  free(inst);
  free(sup);
  free(ranges);
  return 0;
}

double or_l1_loss(const float* image, const uint8_t* gt, int64_t n, float* grad) {
  double s = 0.0;
  const float inv = (float)(1.0 / (double)n);
  for (int64_t i = 0; i < n; ++i) {
    const float d = image[i] - gt[i] * (1.f / 255.f);
    s += fabsf(d);
    if (grad) grad[i] = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv;
  }
  return s / (double)n;
}

/* torch.optim.Adam single-tensor arithmetic */
void or_adam(float* p, const float* g, float* m, float* v, int64_t n, const float* lr60, int64_t S, float beta1,
             float beta2, float eps, int32_t step) {
  const double bc1 = 1.0 - pow((double)beta1, (double)step);
  const double bc2 = 1.0 - pow((double)beta2, (double)step);
  const float scale = (float)(1.0 / bc1), bc2s = (float)sqrt(bc2);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    const int64_t plane = (t / 4) / S;
    const int lane = (int)(t % 4);
    m[t] = m[t] + (1.f - beta1) * (g[t] - m[t]);
    v[t] = beta2 * v[t] + (1.f - beta2) * g[t] * g[t];
    const float denom = sqrtf(v[t]) / bc2s + eps;
    p[t] = p[t] - (lr60[4 * plane + lane] * scale) * m[t] / denom;
  }
}

double or_train_step(float* params, float* exp_avg, float* exp_avg_sq, int64_t S, const double* planes,
                     const or_camera* cams, int32_t B, const uint8_t* gt, int32_t sh_degree, const float* lr60,
                     float beta1, float beta2, float eps, int32_t step, int32_t n_threads) {
  return or_train_step_model(params, exp_avg, exp_avg_sq, S, planes, cams, B, gt, sh_degree, lr60, beta1, beta2, eps,
                             step, n_threads, 0);
}

/* ------------------------------------------------------------------------ */
/* 2DGS (surfel) variant: PAPER.md:773-777 and the 20-element state of       */
/* PAPER.md:1217-1226.  Rows: SP2F = 24 floats                               */
/*   u v opac M[9] (row-major ray transform) r g b depth rx ry normal[3] pad  */
/* and G_SP2F = 15 floats (du dv dM[9] dopac dr dg db).  The paper's 2DGS    */
/* kernels (gsplat) are not in /root/reference: parity for this half is      */
/* pinned by the float64 autograd restatement in tests/test_oracle_2d.py.    */

#define SP2F 24
#define GSP2F 15

typedef struct {
  float d[3], qc[3], s[2], qn[4], qnorm, Rq[9], Rc[9];
  float c0[3], c1[3], c2[3];
  float u, v, depth, radius_x, radius_y, box_cx, box_cy, normal[3];
  float len, dir[3], Y[16], col_raw[3], col[3], opac;
  int valid;
} oproj2;

/* homogeneous image of a camera-frame vector: K x (no division) */
static void kapply(const or_camera* c, const float* x, float* out) {
  out[0] = c->fx * x[0] + c->cx * x[2];
  out[1] = c->fy * x[1] + c->cy * x[2];
  out[2] = x[2];
}

static void quat_rot(const float* qn, float* R) {
  const float w = qn[0], x = qn[1], y = qn[2], z = qn[3];
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  const float wx = w * x, wy = w * y, wz = w * z;
  R[0] = 1.f - 2.f * (yy + zz);
  R[1] = 2.f * (xy - wz);
  R[2] = 2.f * (xz + wy);
  R[3] = 2.f * (xy + wz);
  R[4] = 1.f - 2.f * (xx + zz);
  R[5] = 2.f * (yz - wx);
  R[6] = 2.f * (xz - wy);
  R[7] = 2.f * (yz + wx);
  R[8] = 1.f - 2.f * (xx + yy);
}

static void proj2_fwd(const opoint* pt, const or_camera* c, int n_sh, oproj2* f) {
  const float* W = c->rot_cw;
  for (int k = 0; k < 3; ++k) f->d[k] = pt->p[k] - c->pos[k];
  for (int k = 0; k < 3; ++k) f->qc[k] = (W[3 * k] * f->d[0] + W[3 * k + 1] * f->d[1]) + W[3 * k + 2] * f->d[2];
  f->s[0] = or_det_expf(pt->ls[0]);
  f->s[1] = or_det_expf(pt->ls[1]);
  const float nn = ((pt->q[0] * pt->q[0] + pt->q[1] * pt->q[1]) + pt->q[2] * pt->q[2]) + pt->q[3] * pt->q[3];
  f->qnorm = sqrtf(nn);
  for (int k = 0; k < 4; ++k) f->qn[k] = pt->q[k] / f->qnorm;
  quat_rot(f->qn, f->Rq);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      f->Rc[3 * i + j] = (W[3 * i] * f->Rq[j] + W[3 * i + 1] * f->Rq[3 + j]) + W[3 * i + 2] * f->Rq[6 + j];
  float tu[3], tv[3];
  for (int i = 0; i < 3; ++i) {
    tu[i] = f->Rc[3 * i] * f->s[0];
    tv[i] = f->Rc[3 * i + 1] * f->s[1];
  }
  kapply(c, tu, f->c0);
  kapply(c, tv, f->c1);
  kapply(c, f->qc, f->c2);
  f->depth = f->qc[2];
  f->u = f->c2[0] / f->c2[2];
  f->v = f->c2[1] / f->c2[2];
  /* dual conics of the disk images in image coordinates centred on (u, v)
   * (csrc/splat2d_math.cuh: the columns shifted to c' = (c.x - u c.z,
   * c.y - v c.z, c.z), which avoids the ~0.1 px float cancellation of the
   * absolute-coordinate box); same op sequence as the kernel */
  float a[3], b[3], e[3];
  a[0] = f->c0[0] - f->u * f->c0[2];
  a[1] = f->c0[1] - f->v * f->c0[2];
  a[2] = f->c0[2];
  b[0] = f->c1[0] - f->u * f->c1[2];
  b[1] = f->c1[1] - f->v * f->c1[2];
  b[2] = f->c1[2];
  e[0] = f->c2[0] - f->u * f->c2[2];
  e[1] = f->c2[1] - f->v * f->c2[2];
  e[2] = f->c2[2];
  /* the image of the disk u^2 + v^2 <= 9 is a bounded ellipse */
  const float d22 = 9.f * (a[2] * a[2] + b[2] * b[2]) - e[2] * e[2];
  const float d02 = 9.f * (a[0] * a[2] + b[0] * b[2]) - e[0] * e[2];
  const float d12 = 9.f * (a[1] * a[2] + b[1] * b[2]) - e[1] * e[2];
  const float d00 = 9.f * (a[0] * a[0] + b[0] * b[0]) - e[0] * e[0];
  const float d11 = 9.f * (a[1] * a[1] + b[1] * b[1]) - e[1] * e[1];
  f->valid = d22 < 0.f;
  f->radius_x = f->radius_y = 0.f;
  if (f->valid) {
    const float bx = d02 / d22, by = d12 / d22;
    const float ex = bx * bx - d00 / d22, ey = by * by - d11 / d22;
    f->valid = ex >= 0.f && ey >= 0.f;
  }
  /* support box (csrc/splat2d_math.cuh): image of the disk u^2 + v^2 <= k
   * united with the low-pass circle of radius sqrt(k / 2), k = min(9, 2 ln(255 o)) */
  f->box_cx = f->u;
  f->box_cy = f->v;
  {
    const float o = 1.f / (1.f + or_det_expf(-pt->op));
    const float k = fminf(9.0f, 2.0f * or_det_logf(255.0f * o));
    if (f->valid && k > 0.f) {
      const float k22 = k * (a[2] * a[2] + b[2] * b[2]) - e[2] * e[2];
      const float k02 = k * (a[0] * a[2] + b[0] * b[2]) - e[0] * e[2];
      const float k12 = k * (a[1] * a[2] + b[1] * b[2]) - e[1] * e[2];
      const float k00 = k * (a[0] * a[0] + b[0] * b[0]) - e[0] * e[0];
      const float k11 = k * (a[1] * a[1] + b[1] * b[1]) - e[1] * e[1];
      const float bx = k02 / k22, by = k12 / k22;
      const float hx = sqrtf(fmaxf(bx * bx - k00 / k22, 0.f));
      const float hy = sqrtf(fmaxf(by * by - k11 / k22, 0.f));
      const float rc = sqrtf(0.5f * k);
      const float x0 = fminf(bx - hx, -rc), x1 = fmaxf(bx + hx, rc);
      const float y0 = fminf(by - hy, -rc), y1 = fmaxf(by + hy, rc);
      f->box_cx = f->u + 0.5f * (x0 + x1);
      f->box_cy = f->v + 0.5f * (y0 + y1);
      f->radius_x = 0.5f * (x1 - x0);
      f->radius_y = 0.5f * (y1 - y0);
    }
  }
  float n[3] = {f->Rc[2], f->Rc[5], f->Rc[8]};
  const float facing = (n[0] * f->qc[0] + n[1] * f->qc[1]) + n[2] * f->qc[2];
  for (int k = 0; k < 3; ++k) f->normal[k] = facing > 0.f ? -n[k] : n[k];
  f->len = sqrtf((f->d[0] * f->d[0] + f->d[1] * f->d[1]) + f->d[2] * f->d[2]);
  for (int k = 0; k < 3; ++k) f->dir[k] = f->d[k] / f->len;
  sh_basis(f->dir, n_sh, f->Y);
  for (int ch = 0; ch < 3; ++ch) {
    float acc = f->Y[0] * pt->sh[ch];
    for (int k = 1; k < n_sh; ++k) acc = acc + f->Y[k] * pt->sh[3 * k + ch];
    f->col_raw[ch] = acc + 0.5f;
    f->col[ch] = fmaxf(f->col_raw[ch], 0.f);
  }
  f->opac = 1.f / (1.f + or_det_expf(-pt->op));
}

void or_project2d(const float* params, int64_t S, const int64_t* idx, int64_t m, const or_camera* c,
                  int32_t sh_degree, float* sp) {
  const int n_sh = (sh_degree + 1) * (sh_degree + 1);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k) {
    opoint pt;
    oproj2 f;
    load_opoint(params, S, idx[k], &pt);
    proj2_fwd(&pt, c, n_sh, &f);
    float* r = sp + k * SP2F;
    r[0] = f.u;
    r[1] = f.v;
    r[2] = f.opac;
    for (int i = 0; i < 3; ++i) {
      r[3 + 3 * i + 0] = f.c0[i];
      r[3 + 3 * i + 1] = f.c1[i];
      r[3 + 3 * i + 2] = f.c2[i];
    }
    for (int ch = 0; ch < 3; ++ch) r[12 + ch] = f.col[ch];
    r[15] = f.depth;
    r[16] = f.valid ? f.radius_x : 0.f;
    r[17] = f.valid ? f.radius_y : 0.f;
    for (int k2 = 0; k2 < 3; ++k2) r[18 + k2] = f.normal[k2];
    r[21] = 0.f;
    r[22] = f.box_cx;
    r[23] = f.box_cy;
  }
}

/* gradient of sum_k wk[k] Y_k(dir) w.r.t. dir (same basis as sh_basis) */
static void sh_dir_grad_o(const float* dir, int n_sh, const float* wk, float* gd) {
  const float x = dir[0], y = dir[1], z = dir[2];
  gd[0] = gd[1] = gd[2] = 0.f;
  if (n_sh > 1) {
    gd[1] -= C1 * wk[1];
    gd[2] += C1 * wk[2];
    gd[0] -= C1 * wk[3];
  }
  if (n_sh > 4) {
    gd[0] += C2[0] * y * wk[4];
    gd[1] += C2[0] * x * wk[4];
    gd[1] += C2[1] * z * wk[5];
    gd[2] += C2[1] * y * wk[5];
    gd[0] -= 2.f * C2[2] * x * wk[6];
    gd[1] -= 2.f * C2[2] * y * wk[6];
    gd[2] += 4.f * C2[2] * z * wk[6];
    gd[0] += C2[3] * z * wk[7];
    gd[2] += C2[3] * x * wk[7];
    gd[0] += 2.f * C2[4] * x * wk[8];
    gd[1] -= 2.f * C2[4] * y * wk[8];
  }
  if (n_sh > 9) {
    const float xx = x * x, yy = y * y, zz = z * z;
    gd[0] += C3[0] * 6.f * x * y * wk[9];
    gd[1] += C3[0] * 3.f * (xx - yy) * wk[9];
    gd[0] += C3[1] * y * z * wk[10];
    gd[1] += C3[1] * x * z * wk[10];
    gd[2] += C3[1] * x * y * wk[10];
    gd[0] += C3[2] * (-2.f * x * y) * wk[11];
    gd[1] += C3[2] * (4.f * zz - xx - 3.f * yy) * wk[11];
    gd[2] += C3[2] * (8.f * y * z) * wk[11];
    gd[0] += C3[3] * (-6.f * x * z) * wk[12];
    gd[1] += C3[3] * (-6.f * y * z) * wk[12];
    gd[2] += C3[3] * (6.f * zz - 3.f * xx - 3.f * yy) * wk[12];
    gd[0] += C3[4] * (4.f * zz - 3.f * xx - yy) * wk[13];
    gd[1] += C3[4] * (-2.f * x * y) * wk[13];
    gd[2] += C3[4] * (8.f * x * z) * wk[13];
    gd[0] += C3[5] * (2.f * x * z) * wk[14];
    gd[1] += C3[5] * (-2.f * y * z) * wk[14];
    gd[2] += C3[5] * (xx - yy) * wk[14];
    gd[0] += C3[6] * 3.f * (xx - yy) * wk[15];
    gd[1] += C3[6] * (-6.f * x * y) * wk[15];
  }
}

static void cross3o(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

static void proj2_bwd(const opoint* pt, const or_camera* c, int n_sh, const oproj2* f, const float* gsp_m, float* g) {
  if (!f->valid) return;
  /* G_SP2 moments (Ga, Gb, Gc of dL/dzeta) -> dL/dM rows:
   * dL/dr0 = r1 x Ga + Gc x r2, dL/dr1 = Ga x r0 + r2 x Gb, dL/dr2 = Gb x r1 + r0 x Gc */
  float gsp[15];
  for (int k = 0; k < 15; ++k) gsp[k] = gsp_m[k];
  {
    const float r0[3] = {f->c0[0], f->c1[0], f->c2[0]}, r1[3] = {f->c0[1], f->c1[1], f->c2[1]},
                r2[3] = {f->c0[2], f->c1[2], f->c2[2]};
    const float* Ga = gsp_m + 2;
    const float* Gb = gsp_m + 5;
    const float* Gc = gsp_m + 8;
    float t0[3], t1[3];
    cross3o(r1, Ga, t0);
    cross3o(Gc, r2, t1);
    for (int k = 0; k < 3; ++k) gsp[2 + k] = t0[k] + t1[k];
    cross3o(Ga, r0, t0);
    cross3o(r2, Gb, t1);
    for (int k = 0; k < 3; ++k) gsp[5 + k] = t0[k] + t1[k];
    cross3o(Gb, r1, t0);
    cross3o(r0, Gc, t1);
    for (int k = 0; k < 3; ++k) gsp[8 + k] = t0[k] + t1[k];
  }
  float dc[3], wk[16] = {0}, gd[3];
  for (int ch = 0; ch < 3; ++ch) dc[ch] = f->col_raw[ch] >= 0.f ? gsp[12 + ch] : 0.f;
  for (int k = 0; k < n_sh; ++k)
    for (int ch = 0; ch < 3; ++ch) {
      g[12 + 3 * k + ch] += f->Y[k] * dc[ch];
      wk[k] += dc[ch] * pt->sh[3 * k + ch];
    }
  sh_dir_grad_o(f->dir, n_sh, wk, gd);
  const float dd = f->dir[0] * gd[0] + f->dir[1] * gd[1] + f->dir[2] * gd[2];
  float gpos[3];
  for (int k = 0; k < 3; ++k) gpos[k] = (gd[k] - f->dir[k] * dd) / f->len;
  g[3] += gsp[11] * f->opac * (1.f - f->opac);
  /* M = [c0 c1 c2] (columns); dL/dc_j = column j of dL/dM, plus the mean2d term on c2 */
  float gcol[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) gcol[j][i] = gsp[2 + 3 * i + j];
  const float z = f->c2[2];
  gcol[2][0] += gsp[0] / z;
  gcol[2][1] += gsp[1] / z;
  gcol[2][2] -= (gsp[0] * f->c2[0] + gsp[1] * f->c2[1]) / (z * z);
  /* back through K: x -> (fx x0 + cx x2, fy x1 + cy x2, x2) */
  float gx[3][3];
  for (int j = 0; j < 3; ++j) {
    gx[j][0] = c->fx * gcol[j][0];
    gx[j][1] = c->fy * gcol[j][1];
    gx[j][2] = c->cx * gcol[j][0] + c->cy * gcol[j][1] + gcol[j][2];
  }
  /* qc = W (p - campos): dL/dp = W^T dL/dqc */
  const float* W = c->rot_cw;
  for (int k = 0; k < 3; ++k) g[k] += gpos[k] + W[k] * gx[2][0] + W[3 + k] * gx[2][1] + W[6 + k] * gx[2][2];
  /* t_u = Rc[:,0] s_u, t_v = Rc[:,1] s_v */
  float gRc[9] = {0};
  float gsu = 0.f, gsv = 0.f;
  for (int i = 0; i < 3; ++i) {
    gsu += gx[0][i] * f->Rc[3 * i];
    gsv += gx[1][i] * f->Rc[3 * i + 1];
    gRc[3 * i] = gx[0][i] * f->s[0];
    gRc[3 * i + 1] = gx[1][i] * f->s[1];
  }
  g[4] += gsu * f->s[0];
  g[5] += gsv * f->s[1];
  /* Rc = W Rq: dL/dRq = W^T dL/dRc */
  float G[9] = {0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int r = 0; r < 3; ++r) G[3 * i + j] += W[3 * r + i] * gRc[3 * r + j];
  const float w = f->qn[0], qx = f->qn[1], qy = f->qn[2], qz = f->qn[3];
  float gqn[4];
  gqn[0] = 2.f * (-qz * G[1] + qy * G[2] + qz * G[3] - qx * G[5] - qy * G[6] + qx * G[7]);
  gqn[1] = 2.f * (qy * G[1] + qz * G[2] + qy * G[3] - 2.f * qx * G[4] - w * G[5] + qz * G[6] + w * G[7] - 2.f * qx * G[8]);
  gqn[2] = 2.f * (-2.f * qy * G[0] + qx * G[1] + w * G[2] + qx * G[3] + qz * G[5] - w * G[6] + qz * G[7] - 2.f * qy * G[8]);
  gqn[3] = 2.f * (-2.f * qz * G[0] - w * G[1] + qx * G[2] + w * G[3] - 2.f * qz * G[4] + qy * G[5] + qx * G[6] + qy * G[7]);
  const float dq = w * gqn[0] + qx * gqn[1] + qy * gqn[2] + qz * gqn[3];
  for (int k = 0; k < 4; ++k) g[8 + k] += (gqn[k] - f->qn[k] * dq) / f->qnorm;
}

void or_project2d_bwd(const float* params, int64_t S, const int64_t* idx, int64_t m, const or_camera* c,
                      int32_t sh_degree, const float* gsp, float* grad_params) {
  const int n_sh = (sh_degree + 1) * (sh_degree + 1);
  for (int64_t k = 0; k < m; ++k) {
    opoint pt;
    oproj2 f;
    float g[60] = {0};
    const int64_t i = idx[k];
    load_opoint(params, S, i, &pt);
    proj2_fwd(&pt, c, n_sh, &f);
    proj2_bwd(&pt, c, n_sh, &f, gsp + k * GSP2F, g);
    for (int p = 0; p < 15; ++p)
      for (int l = 0; l < 4; ++l) grad_params[4 * (p * S + i) + l] += g[4 * p + l];
  }
}

/* ray-splat intersection of pixel centre (px, py) with a 2DGS row */
typedef struct {
  float hx[3], hy[3], z[3], u, v, g3, dx, dy, g2, power;
  int ok, in, disk;
} oeval2;

static void cross3e(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* zeta = h_x x h_y is affine in the pixel; it is evaluated, as in the kernels
 * (csrc/raster2d.cu stage2/eval2), from the pixel's 8x4 region origin (X, Y):
 * zeta = z0 + ox (hy0 x r2) + oy (r2 x hx0), z0 = hx0 x hy0, with the
 * origin-shifted rows hx0 = r0 - X r2, hy0 = r1 - Y r2 and the pixel's integer
 * offsets (ox, oy) from the origin. */
static void eval2_o(const float* r, float k, float px, float py, oeval2* e) {
  const float* M = r + 3;
  const int x = (int)px, y = (int)py; /* pixel centre = integer + 0.5 */
  const int rx = (x / 8) * 8, ry = (y / 4) * 4;
  const float X = (float)rx + 0.5f, Y = (float)ry + 0.5f, ox = (float)(x - rx), oy = (float)(y - ry);
  float z0[3], zb[3], zc[3];
  for (int k = 0; k < 3; ++k) {
    e->hx[k] = M[k] - X * M[6 + k];
    e->hy[k] = M[3 + k] - Y * M[6 + k];
  }
  cross3e(e->hx, e->hy, z0);
  cross3e(e->hy, M + 6, zb);
  cross3e(M + 6, e->hx, zc);
  for (int k = 0; k < 3; ++k) e->z[k] = fmaf(zc[k], oy, fmaf(zb[k], ox, z0[k]));
  e->ok = e->z[2] != 0.f;
  e->in = e->disk = 0;
  if (!e->ok) return;
  e->u = e->z[0] / e->z[2];
  e->v = e->z[1] / e->z[2];
  e->g3 = fmaf(e->u, e->u, e->v * e->v);
  e->dx = r[0] + (-px);
  e->dy = r[1] + (-py);
  e->g2 = 2.f * fmaf(e->dx, e->dx, e->dy * e->dy);
  e->power = -0.5f * fminf(e->g3, e->g2);
  /* decisions without the division (csrc/raster2d.cu eval2, bit-identical):
   * g3 <= k  <=>  zx^2 + zy^2 <= k zz^2, k = min(9, 2 ln(255 o)); the disk
   * branch of min(g3, g2) iff zx^2 + zy^2 <= g2 zz^2 */
  const float n3 = fmaf(e->z[0], e->z[0], e->z[1] * e->z[1]), zz = e->z[2] * e->z[2];
  e->in = (n3 <= k * zz) || (e->g2 <= k);
  e->disk = n3 <= e->g2 * zz;
}

int32_t or_render2d(const float* sp, int64_t m, int32_t W, int32_t H, const float* bg, float* image, float* final_T,
                    int32_t* n_contrib, uint32_t* tile_lists, int64_t* n_inst, int32_t* tile_ranges) {
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  int32_t* ranges = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)tx * ty);
  int64_t total = 0;
  oinst* inst = bin_view_l(sp, m, W, H, LAY2, &total, ranges);
  float* sup = row_support(sp, m, SP2F, 1);
  if (tile_lists) {
    if (*n_inst < total) {
      *n_inst = total;
      free(inst);
      free(sup);
      free(ranges);
      return 1;
    }
    for (int64_t i = 0; i < total; ++i) tile_lists[i] = inst[i].row;
    memcpy(tile_ranges, ranges, sizeof(int32_t) * 2 * (size_t)tx * ty);
  }
  if (n_inst) *n_inst = total;
#pragma omp parallel for schedule(dynamic, 4)
  for (int t = 0; t < tx * ty; ++t) {
    const int bx = t % tx, by = t / tx;
    for (int ly = 0; ly < TILE; ++ly)
      for (int lx = 0; lx < TILE; ++lx) {
        const int px = bx * TILE + lx, py = by * TILE + ly;
        if (px >= W || py >= H) continue;
        const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
        float T = 1.f, C[3] = {0, 0, 0};
        int contrib = 0;
        for (int i = ranges[2 * t]; i < ranges[2 * t + 1]; ++i) {
          const float* r = sp + (int64_t)inst[i].row * SP2F;
          oeval2 e;
          eval2_o(r, sup[inst[i].row], pxf, pyf, &e);
          if (!e.ok || !e.in) continue; /* outside the support: min(g3, g2) > k */
          const float alpha = fminf(0.99f, r[2] * expf(e.power));
          const float nT = T * (1.f - alpha);
          if (nT < 1e-4f) break;
          const float w = alpha * T;
          for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(r[12 + ch], w, C[ch]);
          T = nT;
          contrib = i + 1 - ranges[2 * t];
        }
        const int64_t pix = (int64_t)py * W + px;
        for (int ch = 0; ch < 3; ++ch) image[3 * pix + ch] = C[ch] + T * bg[ch];
        final_T[pix] = T;
        n_contrib[pix] = contrib;
      }
  }
  free(inst);
  free(sup);
  free(ranges);
  return 0;
}

int32_t or_render2d_bwd(const float* sp, int64_t m, int32_t W, int32_t H, const float* bg, const float* final_T,
                        const int32_t* n_contrib, const float* grad_image, float* gsp) {
  const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
  int32_t* ranges = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)tx * ty);
  int64_t total = 0;
  oinst* inst = bin_view_l(sp, m, W, H, LAY2, &total, ranges);
  float* sup = row_support(sp, m, SP2F, 1);
  memset(gsp, 0, sizeof(float) * GSP2F * (size_t)m);
  for (int t = 0; t < tx * ty; ++t) {
    const int bx = t % tx, by = t / tx;
    for (int ly = 0; ly < TILE; ++ly)
      for (int lx = 0; lx < TILE; ++lx) {
        const int px = bx * TILE + lx, py = by * TILE + ly;
        if (px >= W || py >= H) continue;
        const int64_t pix = (int64_t)py * W + px;
        const float pxf = (float)px + 0.5f, pyf = (float)py + 0.5f;
        const float* dC = grad_image + 3 * pix;
        const float T_final = final_T[pix];
        const float bgdot = bg[0] * dC[0] + bg[1] * dC[1] + bg[2] * dC[2];
        float T = T_final, acc[3] = {0, 0, 0}, last_alpha = 0.f, lc[3] = {0, 0, 0};
        const int r0 = ranges[2 * t];
        for (int i = r0 + n_contrib[pix] - 1; i >= r0; --i) {
          const int64_t row = inst[i].row;
          const float* r = sp + row * SP2F;
          oeval2 e;
          eval2_o(r, sup[inst[i].row], pxf, pyf, &e);
          if (!e.ok || !e.in) continue; /* outside the support: min(g3, g2) > k */
          const float ex = expf(e.power);
          const float raw = r[2] * ex;
          const float alpha = fminf(0.99f, raw);
          const float ra = 1.f / (1.f - alpha);
          T = T * ra;
          float* g = gsp + row * GSP2F;
          const float fac = alpha * T;
          for (int ch = 0; ch < 3; ++ch) g[12 + ch] += fac * dC[ch];
          for (int ch = 0; ch < 3; ++ch) acc[ch] = last_alpha * lc[ch] + (1.f - last_alpha) * acc[ch];
          last_alpha = alpha;
          for (int ch = 0; ch < 3; ++ch) lc[ch] = r[12 + ch];
          float dL_da = 0.f;
          for (int ch = 0; ch < 3; ++ch) dL_da += (r[12 + ch] - acc[ch]) * dC[ch];
          dL_da = T * dL_da - T_final * ra * bgdot;
          if (raw > 0.99f) continue;
          const float dpow = dL_da * alpha;
          g[11] += dL_da * ex;
          if (e.disk) {
            /* power = -(u^2 + v^2) / 2, (u, v) = zeta.xy / zeta.z, zeta = hx x hy */
            const float gu = -e.u * dpow, gv = -e.v * dpow;
            const float gz[3] = {gu / e.z[2], gv / e.z[2], -(gu * e.z[0] + gv * e.z[1]) / (e.z[2] * e.z[2])};
            /* G_SP2 moments of dL/dzeta: sum gz, sum gz px, sum gz py
             * (zeta = r0 x r1 + px (r1 x r2) + py (r2 x r0); include/splat_b200.h) */
            for (int k = 0; k < 3; ++k) {
              g[2 + k] += gz[k];
              g[5 + k] += gz[k] * pxf;
              g[8 + k] += gz[k] * pyf;
            }
          } else {
            /* low-pass branch: power = -(dx^2 + dy^2) */
            g[0] += -2.f * e.dx * dpow;
            g[1] += -2.f * e.dy * dpow;
          }
        }
      }
  }
  free(inst);
  free(sup);
  free(ranges);
  return 0;
}

double or_train_step_model(float* params, float* exp_avg, float* exp_avg_sq, int64_t S, const double* planes,
                           const or_camera* cams, int32_t B, const uint8_t* gt, int32_t sh_degree, const float* lr60,
                           float beta1, float beta2, float eps, int32_t step, int32_t n_threads, int32_t model) {
  (void)n_threads;
  const int64_t NP = 60 * S;
  float* grads = (float*)calloc((size_t)NP, sizeof(float));
  float* pos = (float*)malloc(sizeof(float) * 3 * (size_t)S);
  for (int64_t i = 0; i < S; ++i)
    for (int k = 0; k < 3; ++k) pos[3 * i + k] = params[4 * i + k];
  double loss = 0.0;
  for (int v = 0; v < B; ++v) {
    const or_camera* c = cams + v;
    const double* vp = planes + (size_t)v * 24;
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S > 0 ? S : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < S; ++i)
      if (in_patch(vp, 1, 0, 0, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2])) idx[m++] = i;
    const int spf = model ? SP2F : SPF, gspf = model ? GSP2F : GSPF;
    float* sp = (float*)malloc(sizeof(float) * spf * (size_t)(m > 0 ? m : 1));
    if (model)
      or_project2d(params, S, idx, m, c, sh_degree, sp);
    else
      or_project(params, S, idx, m, c, sh_degree, sp);
    const int W = c->width, H = c->height;
    const int64_t npx = (int64_t)W * H;
    float* img = (float*)malloc(sizeof(float) * 3 * (size_t)npx);
    float* fT = (float*)malloc(sizeof(float) * (size_t)npx);
    int32_t* nc = (int32_t*)malloc(sizeof(int32_t) * (size_t)npx);
    float* gimg = (float*)malloc(sizeof(float) * 3 * (size_t)npx);
    const float bg[3] = {0, 0, 0};
    if (model)
      or_render2d(sp, m, W, H, bg, img, fT, nc, NULL, NULL, NULL);
    else
      or_render(sp, m, W, H, bg, img, fT, nc, NULL, NULL, NULL);
    loss += or_l1_loss(img, gt + (size_t)v * 3 * npx, 3 * npx, gimg);
    float* gsp = (float*)malloc(sizeof(float) * gspf * (size_t)(m > 0 ? m : 1));
    if (model) {
      or_render2d_bwd(sp, m, W, H, bg, fT, nc, gimg, gsp);
      or_project2d_bwd(params, S, idx, m, c, sh_degree, gsp, grads);
    } else {
      or_render_bwd(sp, m, W, H, bg, fT, nc, gimg, gsp);
      or_project_bwd(params, S, idx, m, c, sh_degree, gsp, grads);
    }
    free(idx);
    free(sp);
    free(img);
    free(fT);
    free(nc);
    free(gimg);
    free(gsp);
  }
  or_adam(params, grads, exp_avg, exp_avg_sq, NP, lr60, S, beta1, beta2, eps, step);
  free(grads);
  free(pos);
  return loss;
}


/* ---- densification (restates csrc/densify.cu; include/splat_b200.h
 * bs_densify_* semantics: 3DGS clone / split / prune) ------ */
static uint64_t so_splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static float so_split_normal(uint64_t base, int child, int axis) {
  uint32_t sum = 0;
  for (int j = 0; j < 12; ++j) sum += (uint32_t)(so_splitmix64(base + (uint64_t)(child * 36 + axis * 12 + j + 1)) >> 40);
  return (float)sum * 0x1p-24f - 6.0f;
}

/* action per point (0 prune, 1 keep, 2 clone, 3 split) and output count per
 * group; stats float2 per point or NULL */
void so_densify_mark(const float* params, int64_t S, const float* stats, const int32_t* group_begin, int32_t ng,
                     float grad_threshold, float split_scale, float min_opacity, float max_scale, int32_t* action,
                     int32_t* group_out) {
  for (int32_t g = 0; g < ng; ++g) {
    int32_t cnt = 0;
    for (int32_t i = group_begin[g]; i < group_begin[g + 1]; ++i) {
      const float* p0 = params + 4 * i;
      const float* p1 = params + 4 * (S + i);
      const float o = 1.f / (1.f + or_det_expf(-p0[3]));
      const float smax = fmaxf(fmaxf(or_det_expf(p1[0]), or_det_expf(p1[1])), or_det_expf(p1[2]));
      const float sx = stats ? stats[2 * i] : 0.f, sy = stats ? stats[2 * i + 1] : 0.f;
      int a;
      if (o < min_opacity || (max_scale > 0.f && smax > max_scale)) {
        a = 0;
      } else {
        const float avg = sy > 0.f ? sx / sy : 0.f;
        a = (sy > 0.f && avg >= grad_threshold) ? (smax > split_scale ? 3 : 2) : 1;
      }
      action[i] = a;
      cnt += a == 0 ? 0 : (a == 1 ? 1 : 2);
    }
    group_out[g] = cnt;
  }
}

/* new shard (plane layout [15][S_new][4]) from the actions; new_begin the
 * exclusive scan of group_out; gid NULL = local index */
void so_densify_apply(const float* params, const float* m, const float* v, int64_t S, const int32_t* action,
                      const int32_t* group_begin, const int32_t* new_begin, int32_t ng, const int32_t* gid,
                      uint32_t seed, float* params_new, float* m_new, float* v_new, int64_t S_new,
                      int32_t* src_index) {
  const float kLogSplit = 0x1.e148a2p-2f;
  for (int32_t g = 0; g < ng; ++g) {
    int64_t j = new_begin[g];
    for (int32_t i = group_begin[g]; i < group_begin[g + 1]; ++i) {
      const int a = action[i];
      if (a == 0) continue;
      if (a == 3) {
        const float* p0 = params + 4 * i;
        const float* p1 = params + 4 * (S + i);
        const float* q = params + 4 * (2 * S + i);
        float s[3], qn[4], R[9];
        for (int k = 0; k < 3; ++k) s[k] = or_det_expf(p1[k]);
        const float nn = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
        const float qnorm = sqrtf(nn);
        for (int k = 0; k < 4; ++k) qn[k] = q[k] / qnorm;
        quat_rot(qn, R);
        const uint32_t id = gid ? (uint32_t)gid[i] : (uint32_t)i;
        const uint64_t base = so_splitmix64(((uint64_t)seed << 32) | id);
        for (int ch = 0; ch < 2; ++ch, ++j) {
          float l[3];
          for (int k = 0; k < 3; ++k) l[k] = s[k] * so_split_normal(base, ch, k);
          float* o0 = params_new + 4 * j;
          for (int r = 0; r < 3; ++r) o0[r] = p0[r] + ((R[3 * r] * l[0] + R[3 * r + 1] * l[1]) + R[3 * r + 2] * l[2]);
          o0[3] = p0[3];
          float* o1 = params_new + 4 * (S_new + j);
          for (int k = 0; k < 3; ++k) o1[k] = p1[k] - kLogSplit;
          o1[3] = p1[3];
          for (int pl = 2; pl < 15; ++pl)
            for (int e = 0; e < 4; ++e) params_new[4 * (pl * S_new + j) + e] = params[4 * (pl * S + i) + e];
          for (int pl = 0; pl < 15; ++pl)
            for (int e = 0; e < 4; ++e) m_new[4 * (pl * S_new + j) + e] = v_new[4 * (pl * S_new + j) + e] = 0.f;
          src_index[j] = i;
        }
      } else {
        for (int rep = 0; rep < (a == 2 ? 2 : 1); ++rep, ++j) {
          for (int pl = 0; pl < 15; ++pl)
            for (int e = 0; e < 4; ++e) {
              params_new[4 * (pl * S_new + j) + e] = params[4 * (pl * S + i) + e];
              m_new[4 * (pl * S_new + j) + e] = rep ? 0.f : m[4 * (pl * S + i) + e];
              v_new[4 * (pl * S_new + j) + e] = rep ? 0.f : v[4 * (pl * S + i) + e];
            }
          src_index[j] = i;
        }
      }
    }
  }
}

/* min/max of the means of each group (empty group: zeros) */
void so_group_aabb_ranges(const float* params, const int32_t* group_begin, int32_t ng, float* aabb) {
  for (int32_t g = 0; g < ng; ++g) {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int32_t i = group_begin[g]; i < group_begin[g + 1]; ++i)
      for (int k = 0; k < 3; ++k) {
        mn[k] = fminf(mn[k], params[4 * i + k]);
        mx[k] = fmaxf(mx[k], params[4 * i + k]);
      }
    const int empty = group_begin[g + 1] <= group_begin[g];
    for (int k = 0; k < 3; ++k) {
      aabb[6 * g + k] = empty ? 0.f : mn[k];
      aabb[6 * g + 3 + k] = empty ? 0.f : mx[k];
    }
  }
}
