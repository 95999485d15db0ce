/*
 * CPU oracle for the PBDR training-step hot path.  TEST INFRASTRUCTURE ONLY:
 * imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg, never by the product path.
 *
 * Integer half (culling, access counts, Morton codes) restates
 * /root/reference/pkg/src/splatsched/visibility.py and is pinned against
 * golden vectors produced by the reference itself (tests/golden/).
 * Floating-point half (projection, binning, rasterisation, loss, backward,
 * Adam) has NO reference implementation in /root/reference (SPEC.md:8
 * excludes it; the paper's gsplat v1.4.0 kernels are not vendored):
 * parity for it is "unpinned" against the reference and is instead pinned
 * by an independent float64 torch-autograd restatement (tests/test_oracle_*).
 */
#ifndef SPLAT_ORACLE_H
#define SPLAT_ORACLE_H
#include <stdint.h>

typedef struct {
  float rot_cw[9];
  float pos[3];
  float fx, fy, cx, cy;
  float lim_x, lim_y;
  float near_plane, far_plane;
  int32_t width, height;
} or_camera; /* same layout as bs_camera */

/* access counts per (view, patch, gpu): out int64 [B*P*P][N] (zeroed here).
 * mode 0 exact, 1 group approx.  planes as in bs_cull_count. */
void or_access_matrix(const float* pos, int64_t n, const int32_t* group_begin,
                      const float* aabb, int32_t ng, const double* planes,
                      int32_t B, int32_t P, const int32_t* point_gpu,
                      int32_t N, int32_t mode, const float* presence,
                      const float* view_times, int64_t* out);
/* per-point visibility bitmask for B <= 32 full-view frusta (P = 1). */
void or_visibility_mask(const float* pos, int64_t n, const int32_t* group_begin,
                        const float* aabb, int32_t ng, const double* planes,
                        int32_t B, uint32_t* mask);
void or_morton(const float* pos, int64_t n, const float* bbox, int32_t bits,
               uint64_t* codes);
float or_det_expf(float x);
float or_det_logf(float x);

/* params: plane layout [15][S][4].  Projects points idx[0..m) for camera c
 * into sp rows [m][12]. */
void or_project(const float* params, int64_t S, const int64_t* idx, int64_t m,
                const or_camera* c, int32_t sh_degree, float* sp);
/* Accumulates d/dparams (plane layout) of m projected points given their
 * G_SP rows [m][9]. */
void or_project_bwd(const float* params, int64_t S, const int64_t* idx,
                    int64_t m, const or_camera* c, int32_t sh_degree,
                    const float* gsp, float* grad_params);

/* Renders one view from m sp rows (depth-sort + tile binning + blend).
 * image [H][W][3], final_T [H][W], n_contrib [H][W].  If tile_lists is not
 * NULL it receives the sorted row indices per tile (concatenated, tile
 * major) and tile_ranges [tiles][2]; capacity in *n_inst (updated). */
int32_t or_render(const float* sp, int64_t m, int32_t W, int32_t H,
                  const float* bg, float* image, float* final_T,
                  int32_t* n_contrib, uint32_t* tile_lists, int64_t* n_inst,
                  int32_t* tile_ranges);
/* d/d sp rows (gsp [m][9], zeroed here) given dL/dimage. */
int32_t or_render_bwd(const float* sp, int64_t m, int32_t W, int32_t H,
                      const float* bg, const float* final_T,
                      const int32_t* n_contrib, const float* grad_image,
                      float* gsp);
/* mean-L1 vs u8 ground truth; grad may be NULL. */
double or_l1_loss(const float* image, const uint8_t* gt, int64_t n,
                  float* grad);
void or_adam(float* p, const float* g, float* m, float* v, int64_t n,
             const float* lr_per_lane60, int64_t S, float beta1, float beta2,
             float eps, int32_t step);

/* One full training step over B views on the CPU (OpenMP): cull, project,
 * render, L1 loss, backward, projection backward, Adam.  Returns the sum of
 * the per-view losses.  gt: u8 [B][H][W][3]. */
double or_train_step(float* params, float* exp_avg, float* exp_avg_sq,
                     int64_t S, const double* planes, const or_camera* cams,
                     int32_t B, const uint8_t* gt, int32_t sh_degree,
                     const float* lr60, float beta1, float beta2, float eps,
                     int32_t step, int32_t n_threads);

/* 2DGS (surfel) variants: rows [m][24] / gradient rows [m][15]
 * (include/splat_b200.h BS_SP2_FLOATS / BS_GSP2_FLOATS). */
void or_project2d(const float* params, int64_t S, const int64_t* idx, int64_t m,
                  const or_camera* c, int32_t sh_degree, float* sp);
void or_project2d_bwd(const float* params, int64_t S, const int64_t* idx,
                      int64_t m, const or_camera* c, int32_t sh_degree,
                      const float* gsp, float* grad_params);
int32_t or_render2d(const float* sp, int64_t m, int32_t W, int32_t H,
                    const float* bg, float* image, float* final_T,
                    int32_t* n_contrib, uint32_t* tile_lists, int64_t* n_inst,
                    int32_t* tile_ranges);
int32_t or_render2d_bwd(const float* sp, int64_t m, int32_t W, int32_t H,
                        const float* bg, const float* final_T,
                        const int32_t* n_contrib, const float* grad_image,
                        float* gsp);
/* or_train_step for model 0 (3DGS) or 1 (2DGS). */
double or_train_step_model(float* params, float* exp_avg, float* exp_avg_sq,
                           int64_t S, const double* planes,
                           const or_camera* cams, int32_t B, const uint8_t* gt,
                           int32_t sh_degree, const float* lr60, float beta1,
                           float beta2, float eps, int32_t step,
                           int32_t n_threads, int32_t model);

/* densification (csrc/densify.cu semantics, include/splat_b200.h
 * bs_densify_*): actions + per-group output counts, the new shard, and the
 * AABBs of variable-size groups. */
void so_densify_mark(const float* params, int64_t S, const float* stats, const int32_t* group_begin, int32_t ng,
                     float grad_threshold, float split_scale, float min_opacity, float max_scale, int32_t* action,
                     int32_t* group_out);
void so_densify_apply(const float* params, const float* m, const float* v, int64_t S, const int32_t* action,
                      const int32_t* group_begin, const int32_t* new_begin, int32_t ng, const int32_t* gid,
                      uint32_t seed, float* params_new, float* m_new, float* v_new, int64_t S_new,
                      int32_t* src_index);
void so_group_aabb_ranges(const float* params, const int32_t* group_begin, int32_t ng, float* aabb);

#endif
