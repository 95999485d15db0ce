/*
 * splat_b200.h — C ABI of the B200-native point-based differentiable
 * rendering (PBDR) training step (Algorithm 1 of arxiv 2512.20017,
 * PAPER.md:465-518).
 *
 * Every entry point is a stateless, asynchronous launch on the caller's
 * CUDA stream.  All pointers are DEVICE pointers unless the parameter name
 * ends in `_host`.  The caller owns all memory (torch tensors on the Python
 * side); the library never allocates.  Return value: 0 on success, otherwise
 * a bs_status code whose meaning maps 1:1 onto the reference's exception
 * classes (pkg/src/splatsched/errors.py:8-51); the message is available
 * from bs_last_error() (thread-local).
 *
 * Interfaces replaced (reference file:line, /root/reference/pkg/src/splatsched):
 *   bs_cull_count      visibility.py:237-252 cull_points, 263-276 cull_group,
 *                      283-292 _candidate_indices, 308-358 build_access_matrix,
 *                      partition.py:65-97 build_bipartite_graph (edge mode),
 *                      PAPER.md:474-483 pts_culling + C[v]_k (mask mode)
 *   bs_bbox            scene.py:109-112 PointCloud.bbox
 *   bs_morton_codes    visibility.py:33-62 _quantize/_interleave3/morton_codes
 *   bs_radix_sort_*    visibility.py:122 np.argsort(kind="stable")
 *   bs_group_aabb      visibility.py:127-133 (group AABBs of zorder_group)
 *   bs_scan_counts     (row layout of SP[v]_k)
 *   bs_project_fwd     PAPER.md:418,452 pts_splatting (3DGS, 11-element SP,
 *                      PAPER.md:1192-1200)
 *   bs_bin_*           PAPER.md:264 "sorts ... splats by their distance"
 *   bs_raster_fwd      PAPER.md:264,494 image_render forward
 *   bs_l1_loss         PAPER.md:495 loss_fn
 *   bs_raster_bwd      PAPER.md:503 image_render.backward
 *   bs_project_bwd     PAPER.md:513-514 pts_splatting.backward
 *   bs_adam_step       PAPER.md:517 AdamUpdate
 *   bs_project_bwd_adam  PAPER.md:511-517 (lines 23-27 of Alg. 1 fused)
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:8-51) ------------------------------------ */
enum {
  BS_OK = 0,
  BS_ERR_PARAMETER = 1,     /* ParameterError     errors.py:12-13 */
  BS_ERR_CONFIGURATION = 2, /* ConfigurationError errors.py:16-17 */
  BS_ERR_CONSISTENCY = 3,   /* ConsistencyError   errors.py:20-21 */
  BS_ERR_CONSTRAINT = 4,    /* ConstraintError    errors.py:24-25 */
  BS_ERR_CUDA = 5,          /* CUDA runtime failure (no reference analogue) */
  BS_ERR_CAPACITY = 6       /* caller buffer too small (ParameterError) */
};

const char* bs_last_error(void);
int32_t bs_abi_version(void);
/* Number of kernel launches issued by this library since load (for the
 * bench's gpu_launches claim). */
int64_t bs_launch_count(void);

/* ---- parameter layout --------------------------------------------------
 * A shard of S points is stored as BS_PARAM_PLANES planes of float4, plane
 * p at float offset p*S*4:
 *   plane 0  : mean.x mean.y mean.z opacity_logit
 *   plane 1  : log_scale.x log_scale.y log_scale.z 0      (2DGS: .z unused)
 *   plane 2  : quat.w quat.x quat.y quat.z
 *   plane 3+ : SH coefficients, flat index f = 3*k + channel (k = 0..15),
 *              plane 3 + f/4, lane f%4
 * 59 live floats per point ("59 attributes") + 1 pad. */
#define BS_PARAM_PLANES 15
#define BS_PARAM_FLOATS 60
/* splat-state row (SP): 12 floats, 48 B; the 11 elements of PAPER.md
 * Table tab:states-3dgs + 1 pad:
 *   0 u  1 v  2 opacity  3 conic_a  4 conic_b  5 conic_c
 *   6 r  7 g  8 b        9 depth    10 radius_x  11 radius_y
 * (the paper's single "radii" element is stored per axis as float
 * half-widths: the tight box of the splat's support q <= min(9, 2 ln(255 o)),
 * i.e. the 3-sigma ellipse cut by alpha >= 1/255; 0 = never contributes) */
#define BS_SP_FLOATS 12
/* gradient row (G_SP): 12 floats (48 B, 16-byte aligned so the rasteriser
 * adds with 128-bit REDs), 9 used + 3 pad, as written by bs_raster_bwd -- moments of
 * dL/dpower over the pixels (power = -q/2, dx = u - px, dy = v - py):
 *   0 sum dpow dx  1 sum dpow dy  2 dL/dopacity  3 sum dpow dx^2
 *   4 sum dpow dx dy  5 sum dpow dy^2  6..8 dL/drgb
 * The projection backward, which has the conic (A, B, C), turns them into
 * dL/du = -(A m0 + B m1), dL/dv = -(B m0 + C m1), dL/dA = -m3/2,
 * dL/dB = -m4, dL/dC = -m5/2 (bs_proj_desc.gsp_form = 1 accepts plain
 * dL/dSP instead: d u, d v, d opacity, d conic a/b/c, d rgb). */
#define BS_GSP_FLOATS 12
#define BS_TILE 16

/* Camera of one view, float32, as consumed by the projection and raster
 * kernels.  Convention of CameraView (scene.py:126-131): +x right, +y down,
 * +z forward; rot_cw = rotation^T maps world to camera; pixel x of a
 * camera-frame point q is fx*q.x/q.z + cx (test_visibility.py:204-215). */
typedef struct {
  float rot_cw[9]; /* row-major world->camera rotation */
  float pos[3];    /* camera centre, world */
  float fx, fy, cx, cy;
  float lim_x, lim_y; /* 1.3 * tan(fov/2): EWA Jacobian clamp */
  float near_plane, far_plane;
  int32_t width, height;
} bs_camera;

/* ---- per-step view rows and small host transfers (csrc/views.cu) -------
 * The batch's per-view rows (cameras, frustum planes, view times, ground-truth
 * indices; the reference selects views by index, visibility.py:308-358) are
 * gathered with the view ids passed as kernel parameters (`ids` is a HOST
 * array, n <= 32), and the step's few host-bound integers are stored by a
 * kernel into mapped pinned memory: neither waits on the copy engines behind
 * the caller's bulk uploads.  dst[k] = src[ids[k]], rows of row_bytes (a
 * multiple of 4). */
int32_t bs_select_rows(const int32_t* ids, int32_t n, const void* src,
                       int64_t n_src_rows, int64_t row_bytes, void* dst,
                       void* stream);
/* n_bytes (a multiple of 4) of host memory (any: read at the call) into
 * device memory, as kernel parameters, stream-ordered: the step's small
 * per-step tables (row offsets, slot lists, owners) without a copy engine
 * or a stream synchronisation */
int32_t bs_upload(const void* host, int64_t n_bytes, void* dst, void* stream);
/* n_bytes (a multiple of 4) from device memory into pinned host memory
 * (cudaHostAlloc / torch pin_memory), stream-ordered */
int32_t bs_copy_to_host(const void* src, int64_t n_bytes, void* dst_pinned,
                        void* stream);

/* ---- K0: culling / access counts --------------------------------------- */
enum {
  BS_CULL_ACCESS_EXACT = 0,  /* out0: int64 [B*P*P, n_gpus] (build_access_matrix EXACT) */
  BS_CULL_ACCESS_GROUP = 1,  /* out0: int64 [B*P*P, n_gpus] (GROUP_APPROX) */
  BS_CULL_EDGES = 2,         /* out0: int32 [n_groups, B] per-(group,view) counts */
  BS_CULL_MASK = 3           /* out0: uint32 [n] view bitmask (B<=32),
                                out1: int32 [n_groups, B] counts,
                                out2: int64 [B*P*P] per-patch counts (may be NULL) */
};

typedef struct {
  int32_t mode;
  int32_t n_views;    /* B */
  int32_t P;          /* patch factor >= 1 */
  int32_t n_gpus;     /* columns of the access matrix (ACCESS modes) */
  int32_t temporal;   /* 1: also test presence[i,0] <= t <= presence[i,1] in f32 */
  int32_t pos_stride; /* floats between consecutive positions: 3 or 4 */
  int32_t max_chunks; /* BS_CULL_MASK with chunk_prefix: chunks of 256 points
                         per group slot, ceil(max_group_points / 256) */
  int32_t* chunk_prefix; /* BS_CULL_MASK, optional: int32 [n_groups][max_chunks][B],
                            visible points of view v in the group's chunks
                            before chunk c (the per-point projection kernels
                            then start each 256-point CTA at its row offset
                            instead of re-counting the group's earlier chunks) */
} bs_cull_desc;

/* Visible-chunk work list from a BS_CULL_MASK launch's counts (out1) and
 * chunk_prefix: work_list (int32 [n_groups * max_chunks]) receives
 * g * max_chunks + c for every 256-point chunk with a visible point, in no
 * particular order, and *work_count their number; the projection kernels
 * then visit only those chunks (bs_proj_desc.work_list). */
int32_t bs_list_chunks(const int32_t* counts, const int32_t* chunk_prefix,
                       const int32_t* group_begin, int32_t n_groups,
                       int32_t max_chunks, int32_t n_views,
                       int32_t* work_list, int32_t* work_count,
                       void* stream);

/* planes: float64 [B][2 + 2*(P+1)][4]: near, far, x-edges c=0..P,
 *   y-edges r=0..P, each (nx, ny, nz, offset) exactly as numpy computes
 *   them in frustum_from_view (visibility.py:168-217).  Patch (r,c) of a
 *   view holds p iff near>=0, far>=0, xe[c]>=0, xe[c+1]<0, ye[r]>=0,
 *   ye[r+1]<0 with d = fma(z,nz,fma(y,ny,x*nx)) + offset in f64.
 * group_begin: int32 [n_groups+1] point offsets; group_aabb: float32
 *   [n_groups][2][3] (min; max) or NULL (no AABB early-out; ACCESS_GROUP
 *   requires it).  point_gpu: int32 [n] or NULL (all points -> column 0).
 * presence: float32 [n][2] or NULL; view_times: float32 [B] or NULL. */
int32_t bs_cull_count(const bs_cull_desc* desc_host, const float* positions,
                      int64_t n_points, const float* presence,
                      const int32_t* group_begin, const float* group_aabb,
                      int32_t n_groups, const double* planes,
                      const float* view_times, const int32_t* point_gpu,
                      void* out0, void* out1, void* out2, void* stream);

/* ---- Morton codes / grouping ------------------------------------------ */
/* bbox_out: float32 [2][3] (min; max) of positions (exact reduction). */
int32_t bs_bbox(const float* positions, int64_t n, int32_t pos_stride,
                float* bbox_out, void* workspace, size_t ws_bytes,
                void* stream);
size_t bs_bbox_workspace(int64_t n);
/* codes[i] = interleave(clip(floor((p - min)/extent*(2^b-1)))) in f64. */
int32_t bs_morton_codes(const float* positions, int64_t n, int32_t pos_stride,
                        const float* bbox, int32_t bits_per_axis,
                        uint64_t* codes, void* stream);
/* AABB of each group of G consecutive points (last group may be short). */
int32_t bs_group_aabb(const float* positions, int64_t n, int32_t pos_stride,
                      int32_t G, float* aabb_out, void* stream);
/* out[i, :] = in[idx[i], :] for rows of `row_floats` floats (float4-aligned
 * plane layout aware: in/out are plane-major with n_in / n_out rows). */
int32_t bs_gather_planes(const float* in, int64_t n_in, const int64_t* idx,
                         int64_t n_out, int32_t n_planes, float* out,
                         void* stream);

/* ---- radix sort (stable LSD, 8-bit digits) ----------------------------- */
/* Sorts (keys, vals) by bits [begin_bit, end_bit).  n is read from
 * n_dev (device int64) when non-NULL, else n_host.  Result is in keys/vals;
 * keys_alt/vals_alt are scratch of the same capacity. */
size_t bs_radix_sort_workspace(int64_t capacity);
int32_t bs_radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt,
                          uint32_t* vals_alt, int64_t n_host,
                          const int64_t* n_dev, int32_t begin_bit,
                          int32_t end_bit, void* workspace, size_t ws_bytes,
                          void* stream);
int32_t bs_radix_sort_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt,
                          uint32_t* vals_alt, int64_t n_host,
                          const int64_t* n_dev, int32_t begin_bit,
                          int32_t end_bit, void* workspace, size_t ws_bytes,
                          void* stream);

/* ---- row layout of the splat state ------------------------------------ */
/* counts: int32 [n_groups][B] (from BS_CULL_MASK).  view_order: int32 [B]
 * host array (NULL = identity); rows are laid out view-major in this order.
 * Outputs: base: int32 [n_groups][B] first row of (group, view) relative to
 * the view's first row; view_rows: int64 [B] visible points per view;
 * view_row0: int64 [B] first row of each view. */
int32_t bs_scan_counts(const int32_t* counts, int32_t n_groups,
                       int32_t n_views, const int32_t* view_order_host,
                       int32_t* base, int64_t* view_rows, int64_t* view_row0,
                       void* stream);

/* ---- K1: projection (pts_splatting) ------------------------------------ */
enum { BS_MODEL_3DGS = 0, BS_MODEL_2DGS = 1 };
/* 2DGS splat-state row (BS_SP2_FLOATS = 24 floats, 96 B): the 20 elements of
 * PAPER.md Table tab:states-2dgs -- 0 u 1 v 2 opacity 3..11 ray transform M
 * (row-major KWH) 12..14 rgb 15 depth 16 radius_x 17 radius_y 18..20 normal
 * -- + 21 pad, 22..23 centre of the support box whose half-widths are
 * radius_x/y (the image of the disk u^2 + v^2 <= k united with the low-pass
 * circle, k = min(9, 2 ln(255 o)); 0 = never contributes).  G_SP row: 16 floats (64-byte aligned for 128-bit REDs):
 * d u, d v, then the moments Ga = sum dL/dzeta, Gb = sum px dL/dzeta,
 * Gc = sum py dL/dzeta of the per-pixel zeta = r0 x r1 + px (r1 x r2) +
 * py (r2 x r0) (r_i rows of M), d opacity, d rgb, pad.  The projection
 * backward turns the moments into dL/dM (dL/dr0 = r1 x Ga + Gc x r2,
 * dL/dr1 = Ga x r0 + r2 x Gb, dL/dr2 = Gb x r1 + r0 x Gc); gsp_form = 1
 * accepts plain dL/dM instead. */
#define BS_SP2_FLOATS 24
#define BS_GSP2_FLOATS 16
typedef struct {
  int32_t n_views;
  int32_t sh_degree; /* 0..3 */
  int32_t tiles_x_max, tiles_y_max;
  int32_t model;     /* BS_MODEL_3DGS (default) or BS_MODEL_2DGS */
  int32_t max_group_points; /* largest group size; > 0 lets the per-point
                               kernels split a group over several CTAs (one
                               per 256 points), 0 = one CTA per group */
  int32_t gsp_form;  /* 3DGS G_SP rows given to the projection backward:
                        0 = raster moments (bs_raster_bwd output, default),
                        1 = plain dL/dSP (d u, d v, d opacity, d conic, d rgb) */
  const int32_t* chunk_prefix; /* optional: bs_cull_count's chunk_prefix for the
                                  same mask, max_chunks = ceil(max_group_points / 256) */
  float* gsp_zero;             /* optional (bs_project_fwd): G_SP rows (BS_GSP_FLOATS /
                                  BS_GSP2_FLOATS floats) cleared at the index of every SP
                                  row written -- the accumulator of a single-rank step,
                                  cleared without a separate pass */
  const int32_t* point_gid;    /* optional (bs_project_fwd): global id of every local
                                  point (NULL: the local index) */
  int32_t* row_gid;            /* optional (bs_project_fwd): int32 per SP row, the
                                  global id of the row's point -- the canonical
                                  tie order of the receiving rank (bs_canonical_order) */
  float* row_support;          /* optional (bs_project_fwd): f32 per SP row, the
                                  support threshold the rasterisers test (see
                                  bs_row_support), computed with the extents */
  float* const* view_sp;       /* optional (bs_project_fwd): device array [n_views] of
                                  row-0 pointers -- view v's rows go to
                                  view_sp[v] + k * row floats instead of sp_rows at
                                  view_row0[v] + k (peer receive buffers: the forward
                                  all-to-all fused into the projection) */
  int32_t* const* view_gid;    /* optional, with view_sp and row_gid semantics: the
                                  rows' global ids at view_gid[v] + k */
  int32_t* bucket_counts;      /* optional (bs_project_fwd, single-pass binning): the
                                  (view, tile) bucket counters [n_views][tiles_per_slot]
                                  (zeroed by the caller), incremented per covered tile
                                  of every row as bs_bin_tiles_count would */
  int32_t* row_bin;            /* with bucket_counts: int32x4 per SP row, (depth bits,
                                  x0 | x1 << 16, y0 | y1 << 16, 0) -- the row's tile
                                  rectangle for bs_bin_tiles_scatter_rec */
  int32_t tiles_per_slot;      /* bucket stride of bucket_counts */
  float* densify_stats;        /* optional (bs_project_bwd_adam, 3DGS): float2 per local
                                  point, (sum over views of |dL/d mean2d| in NDC units,
                                  number of views with a valid splat) ACCUMULATED --
                                  the densification statistic (bs_densify_mark) */
  const int32_t* work_list;    /* optional, with chunk_prefix: bs_list_chunks' list of
                                  the chunks with a visible point and its device count
                                  (work_count); bs_project_fwd, and bs_project_bwd_adam
                                  with selective Adam, then run a grid-stride loop over
                                  those chunks instead of one CTA per (group, chunk) --
                                  at C4 (~2 % of the points visible per view) the empty
                                  CTAs cost more than the work.  Same results (rows are
                                  placed by chunk_prefix, points update independently) */
  const int32_t* work_count;
} bs_proj_desc;
int32_t bs_project_fwd(const bs_proj_desc* desc_host, const float* params,
                       int64_t n_points, const uint32_t* vis_mask,
                       const int32_t* group_begin, int32_t n_groups,
                       const int32_t* base, const int64_t* view_row0,
                       const bs_camera* cams, float* sp_rows, void* stream);

/* ---- K2: tile binning ------------------------------------------------- */
/* Rows [seg_row0[s], seg_row0[s+1]) belong to render slot seg_slot[s].
 * Step 1: depth keys ((slot<<32)|f32bits(depth)) for every row. */
int32_t bs_bin_depth_keys(const float* sp_rows, int64_t n_rows,
                          const int64_t* seg_row0, const int32_t* seg_slot,
                          int32_t n_segs, uint64_t* keys, uint32_t* vals,
                          void* stream);
/* Step 2: per depth-sorted row, number of tiles (reads sp row radius/uv);
 * writes int64 inclusive prefix counts into offsets [n_rows] and the total
 * into total_dev[0]. */
int32_t bs_bin_count(const float* sp_rows, const uint32_t* sorted_rows,
                     int64_t n_rows, const uint64_t* sorted_keys,
                     const bs_camera* slot_cams, int64_t* offsets,
                     int64_t* total_dev, void* workspace, size_t ws_bytes,
                     void* stream);
size_t bs_bin_count_workspace(int64_t n_rows);
/* Step 3: emit (slot*tiles_per_slot + tile, row) instances in depth order. */
int32_t bs_bin_emit(const float* sp_rows, const uint32_t* sorted_rows,
                    int64_t n_rows, const uint64_t* sorted_keys,
                    const bs_camera* slot_cams, int32_t tiles_per_slot,
                    const int64_t* offsets, uint32_t* inst_keys,
                    uint32_t* inst_rows, void* stream);
/* Step 4: ranges int32 [n_slots*tiles_per_slot][2] = [start, end). */
int32_t bs_tile_ranges(const uint32_t* inst_keys, const int64_t* n_dev,
                       int64_t n_host, int32_t n_buckets, int32_t* ranges,
                       void* stream);

/* ---- K2, bucket pipeline (used by the training step) --------------------
 * Same per-tile lists as the pipeline above (ascending depth, ties by row),
 * without full-length radix passes:
 *   count   -> bucket_counts int32 [n_buckets] (zeroed inside)
 *   offsets -> ranges int32 [n_buckets][2], cursor int32 [n_buckets],
 *              stats int64 [2] = {total instances, largest bucket}
 *   scatter -> inst_keys u64 [total] = (f32bits(depth) << 32) | row, grouped
 *              by bucket (unordered inside)
 *   sort    -> inst_rows u32 [total]: per bucket, rows in key order; buckets
 *              with more than smem_cap (<= bs_bin_tiles_max_sort()) keys are
 *              skipped -- sort that slice with bs_radix_sort_u64 and take
 *              bs_keys_low32.  Passing min(cap, largest bucket) (the
 *              offsets' stats[1]) skips the launches of empty size classes. */
int32_t bs_bin_tiles_count(const float* sp_rows, int64_t n_rows,
                           const int64_t* seg_row0, const int32_t* seg_slot,
                           int32_t n_segs, const bs_camera* slot_cams,
                           int32_t tiles_per_slot, int32_t n_buckets,
                           int32_t* bucket_counts, int32_t model, void* stream);
int32_t bs_bin_tiles_offsets(const int32_t* bucket_counts, int32_t n_buckets,
                             int32_t* ranges, int32_t* cursor, int64_t* stats,
                             void* workspace, size_t ws_bytes, void* stream);
size_t bs_bin_tiles_offsets_workspace(int32_t n_buckets);
int32_t bs_bin_tiles_scatter(const float* sp_rows, int64_t n_rows,
                             const int64_t* seg_row0, const int32_t* seg_slot,
                             int32_t n_segs, const bs_camera* slot_cams,
                             int32_t tiles_per_slot, int32_t* cursor,
                             uint64_t* inst_keys, int64_t capacity,
                             int32_t model, void* stream);
/* (keys at positions >= capacity are dropped, so the key buffer can be
 * sized before the instance count reaches the host; re-run offsets + scatter
 * with a larger buffer when the count exceeds it) */
/* Single-pass variant of bs_bin_tiles_scatter: the rows' tile rectangles and
 * depth bits come from the projection's row_bin records (16 B per row)
 * instead of a second read of the splat rows; same keys, same positions. */
int32_t bs_bin_tiles_scatter_rec(const int32_t* row_bin, int64_t n_rows, const int64_t* seg_row0,
                                 const int32_t* seg_slot, int32_t n_segs, const bs_camera* slot_cams,
                                 int32_t tiles_per_slot, int32_t* cursor, uint64_t* inst_keys,
                                 int64_t capacity, void* stream);
int32_t bs_bin_tiles_sort(const uint64_t* inst_keys, const int32_t* ranges,
                          int32_t n_buckets, int32_t smem_cap,
                          uint32_t* inst_rows, void* stream);
/* bs_bin_tiles_sort choosing the 129..256-key method from the average bucket
 * occupancy n_inst / n_buckets (the register bitonic network for full
 * buckets, the warp merge sort for sparse ones); same lists. */
int32_t bs_bin_tiles_sort_n(const uint64_t* inst_keys, const int32_t* ranges,
                            int32_t n_buckets, int32_t smem_cap, int64_t n_inst,
                            uint32_t* inst_rows, void* stream);
int32_t bs_bin_tiles_max_sort(void);
int32_t bs_keys_low32(const uint64_t* keys, int64_t n, uint32_t* out,
                      void* stream);

/* ---- K3/L/K4: rasterisation ------------------------------------------- */
typedef struct {
  int32_t n_slots;
  int32_t tiles_per_slot; /* bucket stride (max tiles_x*tiles_y) */
  int32_t width, height;  /* common image size of all slots */
  float bg[3];
  int32_t loss_fused;     /* 1: gt given, fwd writes L1 partials per tile */
  int32_t pixels_per_lane;/* 1: 8x4 pixel region per warp, 2 (default, 0): 8x8 */
  int32_t patch_P;        /* patches per image side (P > 1 with slot_patches) */
  const uint64_t* slot_patches; /* device uint64 [n_slots] or NULL: bit
                           (r P + c) set = this slot renders patch (r, c); the
                           other pixels are neither rendered nor in the loss
                           (the view's loss normalisation is unchanged) */
  const float* row_support; /* optional: f32 per SP row (bs_row_support); NULL =
                           computed per staged splat (same values) */
} bs_raster_desc;
/* image: f32 [n_slots][H][W][3]; final_T: f32 [n_slots][H][W];
 * n_contrib: int32 [n_slots][H][W] (range-relative end of the blend);
 * gt: u8 [*][H][W][3] or NULL, image of slot s at gt_slot_view[s] (NULL =
 * identity); loss_tiles: f32 [n_slots][tiles]. */
int32_t bs_raster_fwd(const bs_raster_desc* desc_host, const float* sp_rows,
                      const uint32_t* inst_rows, const int32_t* ranges,
                      float* image, float* final_T, int32_t* n_contrib,
                      const uint8_t* gt, const int32_t* gt_slot_view,
                      float* loss_tiles, void* stream);
/* mean-L1 loss per slot: loss[s] = mean|img - gt/255|; grad = d loss/d img
 * (grad may be NULL).  The fused training step instead reduces the per-tile
 * partials of bs_raster_fwd with bs_reduce_loss_tiles. */
int32_t bs_l1_loss(const float* image, const uint8_t* gt, int32_t n_slots,
                   int32_t height, int32_t width, float* loss, float* grad,
                   void* workspace, size_t ws_bytes, void* stream);
size_t bs_l1_loss_workspace(int32_t n_slots);
int32_t bs_reduce_loss_tiles(const float* loss_tiles, int32_t n_slots,
                             int32_t tiles_per_slot, int32_t height,
                             int32_t width, float* loss, void* stream);
/* dL/dimage either given (grad_image f32 [n_slots][H][W][3]) or, when NULL,
 * the mean-L1 gradient recomputed from image and gt.  g_sp: f32 [n_rows][9]
 * accumulated with atomics (caller zeroes it). */
int32_t bs_raster_bwd(const bs_raster_desc* desc_host, const float* sp_rows,
                      const uint32_t* inst_rows, const int32_t* ranges,
                      const float* image, const float* final_T,
                      const int32_t* n_contrib, const float* grad_image,
                      const uint8_t* gt, const int32_t* gt_slot_view,
                      float* g_sp, void* stream);

/* K3 + L + K4 of the mean-L1 training step in one launch (1 pixel per lane):
 * the forward's outputs and loss partials of bs_raster_fwd (loss fused, gt
 * required) and the G_SP of bs_raster_bwd with grad_image == NULL, without
 * re-walking the tile lists from global memory (each warp keeps its
 * forward's filtered splat list in shared memory; see csrc/raster.cu).
 * final_T and n_contrib may be NULL (the fused backward does not read them;
 * the training step skips their 8 B per pixel unless asked to keep them). */
int32_t bs_raster_fwd_bwd(const bs_raster_desc* desc_host, const float* sp_rows,
                          const uint32_t* inst_rows, const int32_t* ranges,
                          float* image, float* final_T, int32_t* n_contrib,
                          const uint8_t* gt, const int32_t* gt_slot_view,
                          float* loss_tiles, float* g_sp, void* stream);

/* 2DGS (surfel) variants: same arguments, BS_SP2_FLOATS rows in, BS_GSP2_FLOATS
 * gradient rows out (config 3; reference: the 2DGS state of PAPER.md:1217-1226,
 * the paper's 2DGS renderer is gsplat's and absent from /root/reference).  Pixel weight exp(-0.5 min(u^2+v^2,
 * 2|mean2d - pixel|^2)) with (u, v) the ray-splat intersection. */
int32_t bs_raster2d_fwd(const bs_raster_desc* desc_host, const float* sp_rows,
                        const uint32_t* inst_rows, const int32_t* ranges,
                        float* image, float* final_T, int32_t* n_contrib,
                        const uint8_t* gt, const int32_t* gt_slot_view,
                        float* loss_tiles, void* stream);
int32_t bs_raster2d_bwd(const bs_raster_desc* desc_host, const float* sp_rows,
                        const uint32_t* inst_rows, const int32_t* ranges,
                        const float* image, const float* final_T,
                        const int32_t* n_contrib, const float* grad_image,
                        const uint8_t* gt, const int32_t* gt_slot_view,
                        float* g_sp, void* stream);
/* 2DGS K3 + L + K4 in one launch (bs_raster_fwd_bwd semantics). */
int32_t bs_raster2d_fwd_bwd(const bs_raster_desc* desc_host, const float* sp_rows,
                            const uint32_t* inst_rows, const int32_t* ranges,
                            float* image, float* final_T, int32_t* n_contrib,
                            const uint8_t* gt, const int32_t* gt_slot_view,
                            float* loss_tiles, float* g_sp, void* stream);

/* ---- densification ("periodic densification"; standard 3DGS
 * clone / split / prune) ------------------------------- */
/* Per point (3DGS): o = sigmoid(opacity logit), smax = max_k exp(log_scale_k),
 * avg = stats.x / stats.y (0 when stats.y == 0):
 *   PRUNE (0 outputs)  o < min_opacity, or max_scale > 0 and smax > max_scale
 *   SPLIT (2 outputs)  else avg >= grad_threshold and smax >  split_scale
 *   CLONE (2 outputs)  else avg >= grad_threshold (and smax <= split_scale)
 *   KEEP  (1 output)   otherwise
 * Outputs stay in the point's group, in point order: KEEP copies the point
 * and its Adam moments; CLONE writes the point (with its moments) then an
 * exact copy with zero moments; SPLIT writes two children with zero moments,
 * log scales minus ln(1.6) and means mu + R(q) (s * eps), eps ~ N(0, 1) per
 * axis by the Irwin-Hall sum of 12 uniforms from splitmix64(seed, global id,
 * child, axis) -- every op a round-to-nearest float op, so the outputs are
 * bit-exact against the CPU oracle (oracle/splat_oracle.c so_densify). */
#define BS_DENSIFY_PRUNE 0
#define BS_DENSIFY_KEEP 1
#define BS_DENSIFY_CLONE 2
#define BS_DENSIFY_SPLIT 3
typedef struct {
  int32_t model;          /* BS_MODEL_3DGS */
  float grad_threshold;   /* on the mean NDC-space |dL/d mean2d| (3DGS: 2e-4) */
  float split_scale;      /* split above / clone at or below this max world scale */
  float min_opacity;      /* prune below (3DGS: 0.005) */
  float max_scale;        /* prune above this max world scale; <= 0: off */
  uint32_t seed;          /* split samples */
} bs_densify_desc;
/* action: int32 [n_points] (BS_DENSIFY_*); group_out: int32 [n_groups], the
 * number of output points of each group (its new size). */
int32_t bs_densify_mark(const bs_densify_desc* desc_host, const float* params, int64_t n_points,
                        const float* stats, const int32_t* group_begin, int32_t n_groups,
                        int32_t* action, int32_t* group_out, void* stream);
/* new_group_begin: int32 [n_groups + 1], the exclusive scan of group_out;
 * point_gid: global id per old point (NULL = local index) for the split
 * samples; outputs params_new / exp_avg_new / exp_avg_sq_new (plane layout,
 * n_new points) and src_index int32 [n_new] (the old point each new point
 * comes from). */
int32_t bs_densify_apply(const bs_densify_desc* desc_host, const float* params, const float* exp_avg,
                         const float* exp_avg_sq, int64_t n_points, const int32_t* action,
                         const int32_t* group_begin, const int32_t* new_group_begin, int32_t n_groups,
                         const int32_t* point_gid, float* params_new, float* exp_avg_new,
                         float* exp_avg_sq_new, int64_t n_new, int32_t* src_index, void* stream);
/* aabb_out f32 [n_groups][6] (min xyz, max xyz) of each group's means --
 * visibility.py:127-133 for groups of any size. */
int32_t bs_group_aabb_ranges(const float* params, int64_t n_points, const int32_t* group_begin,
                             int32_t n_groups, float* aabb_out, void* stream);

/* ---- K1b + K5 ---------------------------------------------------------- */
/* grad_params: plane layout like params, ACCUMULATED (caller zeroes). */
int32_t bs_project_bwd(const bs_proj_desc* desc_host, const float* params,
                       int64_t n_points, const uint32_t* vis_mask,
                       const int32_t* group_begin, int32_t n_groups,
                       const int32_t* base, const int64_t* view_row0,
                       const bs_camera* cams, const float* g_sp,
                       float* grad_params, void* stream);

typedef struct {
  float lr[BS_PARAM_FLOATS]; /* per (plane, lane) learning rate */
  float beta1, beta2, eps;
  int32_t step;       /* 1-based step count for bias correction */
  int32_t selective;  /* 1: skip points with vis_mask == 0 */
} bs_adam_desc;
int32_t bs_adam_step(const bs_adam_desc* desc_host, float* params,
                     const float* grads, float* exp_avg, float* exp_avg_sq,
                     int64_t n_points, const uint32_t* vis_mask, void* stream);
/* Fused: projection backward over all views of each point followed by the
 * Adam update of that point; no grad_params round trip through HBM. */
int32_t bs_project_bwd_adam(const bs_proj_desc* pdesc_host,
                            const bs_adam_desc* adesc_host, float* params,
                            float* exp_avg, float* exp_avg_sq,
                            int64_t n_points, const uint32_t* vis_mask,
                            const int32_t* group_begin, int32_t n_groups,
                            const int32_t* base, const int64_t* view_row0,
                            const bs_camera* cams, const float* g_sp,
                            void* stream);

/* ---- patch placement (P > 1): render sets and the exchange layout ------
 * Patch j of view v is rendered by rank patch_owner[v P^2 + j] (W of
 * hierarchical_place, placement.py:316-361).  Replace the reference's
 * transfer accounting by the rows actually moved (simulator.py:134-183 counts
 * the access matrix; the render set adds the splats whose support crosses
 * a patch border). */
/* dest_mask[r]: bit d set iff rank d renders a patch the support box of row r
 * reaches.  Rows view-major from view_row0 (ascending). */
int32_t bs_row_dest_mask(const float* sp_rows, int32_t model, int64_t n_rows,
                         const int64_t* view_row0, int32_t n_views, int32_t P,
                         int32_t width, int32_t height,
                         const int32_t* patch_owner, uint32_t* dest_mask,
                         void* stream);
/* Send layout grouped by destination, then view, rows ascending:
 * count_only = 1 -> dest_total[d]; then count_only = 0 with dest_base (the
 * exclusive scan of dest_total) -> send_idx[dest_base[d] + k] = row and
 * view_counts[d][v] (caller zeroes it). */
size_t bs_dest_compact_workspace(int64_t n_rows, int32_t n_dest);
int32_t bs_dest_compact(const uint32_t* dest_mask, int64_t n_rows, int32_t n_dest,
                        const int64_t* view_row0, int32_t n_views, int32_t count_only,
                        int64_t* dest_total, const int64_t* dest_base, int64_t* send_idx,
                        int64_t* view_counts, void* workspace, size_t ws_bytes,
                        void* stream);
/* dst[i] = src[idx[i]] (rows of `width` 32-bit words; float4 copies when
 * width % 4 == 0) */
int32_t bs_gather_rows(const float* src, int32_t width, const int64_t* idx, int64_t n,
                       float* dst, void* stream);
/* dst[idx[i]][k] += src[i][k], k < used (atomic: rows sent to several ranks);
 * row strides src_width / dst_width floats */
int32_t bs_scatter_add_rows(const float* src, int32_t src_width, int32_t used,
                            const int64_t* idx, int64_t n, float* dst, int32_t dst_width,
                            void* stream);

/* Canonical row order of a receiving rank (stable order
 * contract of visibility.py:122): the rows of every render slot sorted by the
 * global id of their point, so that the per-tile lists (ties in depth broken
 * by row) are the same on 1 or N ranks.  Replaces nothing in the reference
 * (it has no receive side); called by the executor between the splat
 * all-to-all and the binning.
 * row_gid[r] (int32 >= 0) of received row r, segments [seg_row0[s], next)
 * rendered in slot seg_slot[s].  Outputs: order[i] = received row placed at
 * canonical position i (slot-major, ascending global id), canon_gid[i] (optional)
 * its global id. */
/* ---- peer-memory exchange (csrc/peer.cu; replaces the all-to-alls of
 * counted by the reference in simulator.py:134-183) ----
 * One IPC-exported allocation per rank, mapped by the others; completion by
 * stream-ordered flags.  bs_ipc_alloc: cudaMalloc + handle (bs_ipc_handle_bytes
 * bytes), zero-filled; bs_ipc_open / close / free.  bs_stream_signal: after
 * all prior work of `stream`, *flag = value (system-scope fence first);
 * bs_stream_wait: later work of `stream` waits until *flag >= value. */
size_t bs_ipc_handle_bytes(void);
int32_t bs_ipc_alloc(size_t bytes, void** ptr, uint8_t* handle);
int32_t bs_ipc_open(const uint8_t* handle, void** ptr);
int32_t bs_ipc_close(void* ptr);
int32_t bs_ipc_free(void* ptr);
int32_t bs_stream_signal(void* stream, uint32_t* flag, uint32_t value);
int32_t bs_stream_wait(void* stream, const uint32_t* flag, uint32_t value);
/* Gradient rows back to their owners: the first `width` floats of canonical
 * row i (stride src_width; received row order[i], in segment s = (source
 * seg_src[s], view), segment start seg_row0[s]) are copied to
 * dst[seg_src[s]] + (seg_dst0[s] + order[i] - seg_row0[s]) * dst_width
 * (dst: device array [n_ranks] of the owners' G_SP send-layout buffers). */
int32_t bs_return_rows(const float* src, int32_t src_width, int32_t width, const int64_t* order, int64_t n,
                       const int64_t* seg_row0, const int32_t* seg_src, const int64_t* seg_dst0,
                       int32_t n_segs, float* const* dst, int32_t dst_width, void* stream);

/* Per-row support threshold of the rasterisers: a pixel pair contributes
 * iff q <= k, k = min(9, 2 ln(255 o)) (include/ header notes);
 * 3DGS rows store k * (-log2(e) / 2) (the threshold on the log2 exponent),
 * 2DGS rows k.  Computed once per row (the projection writes it through
 * bs_proj_desc.row_support; this entry recomputes it for received rows)
 * instead of once per (warp, staged splat). */
int32_t bs_row_support(const float* sp_rows, int32_t model, int64_t n_rows, float* out, void* stream);
size_t bs_canonical_order_workspace(int64_t n_rows);
int32_t bs_canonical_order(const int32_t* row_gid, int64_t n_rows, const int64_t* seg_row0,
                           const int32_t* seg_slot, int32_t n_segs, int32_t n_slots,
                           int64_t* order, int32_t* canon_gid, void* workspace, size_t ws_bytes,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLAT_B200_H */
