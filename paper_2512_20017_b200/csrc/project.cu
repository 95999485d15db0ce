// K1 projection (pts_splatting), K1b projection backward, K5 Adam, and the
// fused K1b+K5 per-point kernel (Alg. 1 lines 23-27).
//
// Row layout: the splat state of view v is a contiguous run of rows in the
// order of ascending local point index; runs are concatenated in the
// caller's view order (destination order for the all-to-all).
// The row of (point i in group g, view v) is
//     view_row0[v] + base[g][v] + #{visible points of v in g before i}
// recomputed identically by every per-point kernel with warp ballots, so no
// per-(view, point) index table is ever materialised.
#include "splat2d_math.cuh"
#include "tile.cuh"

namespace bs {
namespace {

constexpr int kProjThreads = 256;
#ifndef BS_ADAM_BATCH
#define BS_ADAM_BATCH 3
#endif
constexpr int kAdamBatch = BS_ADAM_BATCH;
#ifndef BS_ADAM_SMEM_PARAMS
#define BS_ADAM_SMEM_PARAMS 1
#endif  // parameter planes per batch of Adam loads in the fused kernel
#ifndef BS_GSP_LDCS
#define BS_GSP_LDCS 1
#endif  // 1: G_SP rows read evict-first (ld.global.cs) by the projection backward: their
        // last use before the next step's projection clears them (C2 0.366 -> 0.360 ms,
        // DRAM reads 1.025 -> 0.982 GB; C3 0.787 -> 0.755 ms)
#ifndef BS_ADAM_STREAM
#define BS_ADAM_STREAM 2
#endif  // 2: parameters and moments written evict-first (st.global.cs): the lines are
        // dead to this kernel after the update, so L2 keeps the bulk prefetches of
        // the planes still to come (C2: 0.376 -> 0.366 ms, C3: 0.787 -> 0.779 ms);
        // 1: also the moment loads (ld.global.cs; 0.368 ms); 0: no hints
constexpr int kProjWarps = kProjThreads / 32;
#ifndef BS_SH_EVICT_FIRST
#define BS_SH_EVICT_FIRST 1
#endif  // 1: the projection kernels stage SH coefficients with an L2 evict-first policy
        // (with BS_GSP_ZERO_CS: C2 projection 0.167 -> 0.165 ms, fused Adam 0.362 -> 0.356 ms;
        // C3 fused Adam 0.759 -> 0.748 ms; profiles/r2z_ab_proj_hints.txt)
#ifndef BS_GSP_ZERO_CS
#define BS_GSP_ZERO_CS 1
#endif  // 1: the projection clears G_SP rows with evict-first stores

// 16-byte global -> shared copy of one SH float4 (L2::cache_hint with an
// evict-first policy when BS_SH_EVICT_FIRST: the coefficients are read once
// per kernel, so their lines should not displace the kernel's outputs in L2)
__device__ __forceinline__ void sh_copy16(uint32_t dst, const void* src) {
#if BS_SH_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#endif
}

constexpr int kMaxViews = 32;

// Per-round in-group ranks of the set view bits of every thread.
struct RowRanker {
  uint32_t* s_bal;  // [kProjWarps][kMaxViews]
  int* s_run;       // [kMaxViews]

  // Call with all threads of the CTA.  Returns nothing; rows are obtained by
  // row_of() for set bits until the next advance().
  // kSparse (the visible-chunk kernels): ballots only for the views some
  // lane of the warp sees (a sparse step's chunk is usually visible in one
  // or two of the batch's views); the other views' entries are zero
  template <bool kSparse = false>
  __device__ void round(uint32_t mask, int B) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if constexpr (kSparse) {
      const uint32_t seen = __reduce_or_sync(0xffffffffu, mask);
      if (lane < B && !((seen >> lane) & 1u)) s_bal[w * kMaxViews + lane] = 0u;
      for (uint32_t rest = seen; rest; rest &= rest - 1u) {
        const int v = __ffs(rest) - 1;
        const uint32_t bal = __ballot_sync(0xffffffffu, (mask >> v) & 1u);
        if (lane == 0) s_bal[w * kMaxViews + v] = bal;
      }
    } else {
      for (int v = 0; v < B; ++v) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (mask >> v) & 1u);
        if (lane == 0) s_bal[w * kMaxViews + v] = bal;
      }
    }
    __syncthreads();
  }
  __device__ int row_offset(int v) const {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int pre = s_run[v];
    for (int j = 0; j < w; ++j) pre += __popc(s_bal[j * kMaxViews + v]);
    return pre + __popc(s_bal[w * kMaxViews + v] & ((1u << lane) - 1u));
  }
  __device__ void advance(int B) {
    __syncthreads();
    if (threadIdx.x < B) {
      int add = 0;
      for (int j = 0; j < kProjWarps; ++j) add += __popc(s_bal[j * kMaxViews + threadIdx.x]);
      s_run[threadIdx.x] += add;
    }
    __syncthreads();
  }
};

// Point range of this CTA.  gridDim.y == 1: the whole group g.  Otherwise
// chunk blockIdx.y (kProjThreads points) of g, with the ranker's running
// per-view counts advanced over the group's earlier chunks first.  Returns
// false (uniformly over the CTA) when the chunk lies past the group's end.
__device__ __forceinline__ bool chunk_range(const int32_t* __restrict__ group_begin, const uint32_t* __restrict__ mask,
                                            const int32_t* __restrict__ chunk_prefix, RowRanker& rk, int g, int cy,
                                            int ny, int B, int& lo, int& hi) {
  const int begin = group_begin[g], end = group_begin[g + 1];
  if (ny == 1) {
    lo = begin;
    hi = end;
    return true;
  }
  lo = begin + cy * kProjThreads;
  if (lo >= end) return false;
  hi = min(end, lo + kProjThreads);
  if (chunk_prefix) {  // counted by the culling kernel
    if (threadIdx.x < B) rk.s_run[threadIdx.x] = chunk_prefix[((size_t)g * ny + cy) * B + threadIdx.x];
    __syncthreads();
    return true;
  }
  for (int b = begin; b < lo; b += kProjThreads) {
    rk.round(mask[b + threadIdx.x], B);
    rk.advance(B);
  }
  return true;
}

struct ProjArgs {
  int B, n_sh;
  const float4* params;
  int64_t S;
  const uint32_t* mask;
  const int32_t* group_begin;
  const int32_t* base;  // [ng][B]
  const int64_t* view_row0;
  const bs_camera* cams;
  int gsp_standard;  // 3DGS G_SP rows: 0 = raster moments (default), 1 = dL/dSP
  const int32_t* chunk_prefix;  // [ng][gridDim.y][B] rows before each chunk, or NULL
  float* gsp_zero;              // G_SP rows cleared alongside the SP rows (project_fwd), or NULL
  const int32_t* point_gid;     // global id per local point (project_fwd), or NULL (= local index)
  int32_t* row_gid;             // per SP row: global id of its point (project_fwd), or NULL
  float* row_support;           // per SP row: the rasteriser's support threshold (project_fwd), or NULL
  float* const* view_sp;        // per view: row-0 pointer of its rows (peer receive buffers), or NULL
  int32_t* const* view_gid;     // per view: row-0 pointer of its global ids, or NULL
  int32_t* bucket_counts;       // single-pass binning: (view, tile) counters, or NULL
  int4* row_bin;                // with bucket_counts: per-row (depth bits, x0|x1<<16, y0|y1<<16, 0)
  int tiles_per_slot;
  float2* densify_stats;        // (bs_project_bwd_adam, 3DGS): per point (sum |dL/d mean2d| NDC, views), or NULL
  // visible-chunk work list (bs_cull_count): g * max_chunks + c per entry, or NULL
  const int32_t* work_list;
  const int32_t* work_count;
  int max_chunks;
};

// Splat models: 3DGS (EWA Gaussians, 12-float SP rows) and 2DGS (surfels,
// 24-float SP rows, splat2d_math.cuh).
// Per point: pre() once (view-independent work), forward()/backward() per
// view, finish() once to push the accumulated view-independent gradient
// (Acc) through the scales and the quaternion.
struct Model3 {
  using F = ProjFwd;
  using Pre = PointPre;
  static constexpr int kSP = BS_SP_FLOATS, kGSP = BS_GSP_FLOATS, kAcc = 6;
  static constexpr bool k2D = false;
  __device__ static void pre(const PointIn& pt, Pre& r) { point_pre(pt, r); }
  static constexpr int kGcol = 6;  // colour gradient inside a G_SP row
  static constexpr bool kFuseWk = false;
  template <class SH>
  __device__ static void forward(const PointIn& pt, const Pre& r, const SH& sh, const bs_camera& c, int n_sh, F& f,
                                 const float* gcol = nullptr, float* wk = nullptr) {
    project_forward_t(pt, r, sh, c, n_sh, f, gcol, wk);
  }
  __device__ static void write(float* row, const F& f) { write_sp_row(row, f); }
  // support box and depth exactly as written into the row (floats 0, 1, 10, 11, 9)
  __device__ static void box(const F& f, float& u, float& v, float& rx, float& ry, float& depth) {
    u = f.u;
    v = f.v;
    rx = f.valid ? f.radius_x : 0.f;
    ry = f.valid ? f.radius_y : 0.f;
    depth = f.depth;
  }
  template <class SH, class A>
  __device__ static void backward(const PointIn& pt, const Pre& r, const SH& sh, const bs_camera& c, int n_sh,
                                  const F& f, const float* gs, float* g, float* acc, A& add,
                                  const float* wk_pre = nullptr) {
    project_backward_t(pt, r, sh, c, n_sh, f, gs, g, acc, add, wk_pre);
  }
  __device__ static void finish(const PointIn& pt, const float* acc, float* g) { point_pre_backward(pt, acc, g); }
  // raster moments (M1..M5 of dL/dpower) -> dL/d(u, v, conic a, b, c)
  __device__ static void from_moments(const F& f, float* gs) { gsp_from_moments(f.conic, gs); }
};

struct Model2 {
  using F = Proj2D;
  using Pre = Pre2D;
  static constexpr int kSP = kSP2, kGSP = kGSP2, kAcc = 9;
  static constexpr bool k2D = true;
  __device__ static void pre(const PointIn& pt, Pre& r) { point_pre2(pt, r); }
  static constexpr int kGcol = 12;
  static constexpr bool kFuseWk = true;
  template <class SH>
  __device__ static void forward(const PointIn& pt, const Pre& r, const SH& sh, const bs_camera& c, int n_sh, F& f,
                                 const float* gcol = nullptr, float* wk = nullptr) {
    project2d_forward(pt, r, sh, c, n_sh, f, gcol, wk);
  }
  __device__ static void write(float* row, const F& f) { write_sp2_row(row, f); }
  // support box and depth exactly as written into the row (floats 22, 23, 16, 17, 15)
  __device__ static void box(const F& f, float& u, float& v, float& rx, float& ry, float& depth) {
    u = f.box_cx;
    v = f.box_cy;
    rx = f.valid ? f.radius_x : 0.f;
    ry = f.valid ? f.radius_y : 0.f;
    depth = f.depth;
  }
  template <class SH, class A>
  __device__ static void backward(const PointIn& pt, const Pre& r, const SH& sh, const bs_camera& c, int n_sh,
                                  const F& f, const float* gs, float* g, float* acc, A& add,
                                  const float* wk_pre = nullptr) {
    project2d_backward(pt, r, sh, c, n_sh, f, gs, g, acc, add, wk_pre);
  }
  __device__ static void finish(const PointIn& pt, const float* acc, float* g) { point_pre2_backward(pt, acc, g); }
  // raster moments of dL/dzeta -> dL/dM rows
  __device__ static void from_moments(const F& f, float* gs) { gsp2_from_moments(f, gs); }
};

template <class M, bool kWork>
#ifndef BS_PROJ_FWD_CTAS
#define BS_PROJ_FWD_CTAS 4  // CTAs per SM the projection's register budget is sized for
#endif
__device__ __forceinline__ void project_fwd_chunk(const ProjArgs& a, float* __restrict__ sp, int g, int cy, int ny) {
  // each thread's SH coefficients, staged by cp.async (no registers held for
  // them across the view loop): [12][kProjThreads] float4
  extern __shared__ float4 s_sh4f[];
  __shared__ uint32_t s_bal[kProjWarps * kMaxViews];
  __shared__ int s_run[kMaxViews];
  __shared__ bs_camera s_cam[kMaxViews];
  __shared__ int64_t s_row0[kMaxViews];
  const int B = a.B;
  if (threadIdx.x < B) {
    s_run[threadIdx.x] = 0;
    s_cam[threadIdx.x] = a.cams[threadIdx.x];
    s_row0[threadIdx.x] = a.view_row0[threadIdx.x] + a.base[(size_t)g * B + threadIdx.x];
  }
  __syncthreads();
  RowRanker rk{s_bal, s_run};
  int lo, end;
  if (!chunk_range(a.group_begin, a.mask, a.chunk_prefix, rk, g, cy, ny, B, lo, end)) return;
  for (int b0 = lo; b0 < end; b0 += kProjThreads) {
    const int i = b0 + threadIdx.x;
    const uint32_t mask = i < end ? a.mask[i] : 0u;
    // a round without a visible point writes no row and advances no count
    if (!__syncthreads_or(mask != 0u)) continue;
    if (mask) {
      const int sh_q = (3 * a.n_sh + 3) / 4;
      for (int q = 0; q < sh_q; ++q) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_sh4f + q * kProjThreads + threadIdx.x);
        sh_copy16(dst, a.params + (int64_t)(3 + q) * a.S + i);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    rk.template round<kWork>(mask, B);
    if (mask) {
      PointIn pt;
      load_point(a.params, a.S, i, 0, pt);  // geometry planes; SH from shared memory
      typename M::Pre pre;
      M::pre(pt, pre);
      asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own column
      const ShSmem sh{s_sh4f + threadIdx.x};
      uint32_t m = mask;
      while (m) {
        const int v = __ffs(m) - 1;
        m &= m - 1;
        typename M::F f;
        M::forward(pt, pre, sh, s_cam[v], a.n_sh, f);
        const int64_t row = s_row0[v] + rk.row_offset(v);
        if (a.view_sp) {
          // the row of this view lands in its renderer's receive buffer
          const int64_t k = row - a.view_row0[v];
          M::write(a.view_sp[v] + k * M::kSP, f);
          if (a.view_gid) a.view_gid[v][k] = a.point_gid ? a.point_gid[i] : i;
        } else {
          M::write(sp + row * M::kSP, f);
          if (a.row_gid) a.row_gid[row] = a.point_gid ? a.point_gid[i] : i;
        }
        if (a.bucket_counts) {
          // single-pass binning: this row's tile rectangle is counted here and
          // recorded for the scatter, which then never re-reads the row
          float bu, bv, brx, bry, bd;
          M::box(f, bu, bv, brx, bry, bd);
          const int Wv = s_cam[v].width, Hv = s_cam[v].height;
          int x0, x1, y0, y1;
          tile_rect_vals(bu, bv, brx, bry, Wv, Hv, x0, x1, y0, y1);
          a.row_bin[row] = make_int4((int)__float_as_uint(bd), x0 | (x1 << 16), y0 | (y1 << 16), 0);
          count_rect(a.bucket_counts, (int64_t)v * a.tiles_per_slot, (Wv + BS_TILE - 1) / BS_TILE, x0, x1, y0, y1);
        }
        if (a.row_support) a.row_support[row] = row_support_from_k(f.support_k, M::k2D);
        if (a.gsp_zero) {
          float4* z = reinterpret_cast<float4*>(a.gsp_zero + row * M::kGSP);
#pragma unroll
          for (int k = 0; k < M::kGSP / 4; ++k) {
#if BS_GSP_ZERO_CS
            __stcs(z + k, make_float4(0.f, 0.f, 0.f, 0.f));
#else
            z[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
          }
        }
      }
    }
    if (b0 + kProjThreads < end) rk.advance(B);  // (a chunk's single round needs no advance)
  }
}

// One CTA per (group, chunk), or -- with a visible-chunk work list -- a
// grid-stride loop over the listed chunks (empty chunks cost no CTA).
// (kWork: separate instantiations, so the one-CTA-per-chunk kernel keeps
// its own register allocation)
template <class M, bool kWork>
__global__ void __launch_bounds__(kProjThreads, BS_PROJ_FWD_CTAS) project_fwd_kernel(ProjArgs a, float* __restrict__ sp) {
  if constexpr (!kWork) {
    project_fwd_chunk<M, false>(a, sp, blockIdx.x, blockIdx.y, gridDim.y);
    return;
  }
  const int n = *a.work_count;
  for (int w = blockIdx.x; w < n; w += gridDim.x) {
    const int item = __ldg(a.work_list + w);
    project_fwd_chunk<M, true>(a, sp, item / a.max_chunks, item % a.max_chunks, a.max_chunks);
    __syncthreads();  // the chunk's shared-memory state is rebuilt by the next
  }
}

// Accumulate the parameter gradient of one point over all its views:
// geometry (12 floats) into g, SH coefficients through sh_add.
template <class M, class SH, class ShAdd>
__device__ __forceinline__ void point_backward(const ProjArgs& a, const bs_camera* s_cam, const int64_t* s_row0,
                                               const RowRanker& rk, uint32_t mask, const PointIn& pt, const SH& sh,
                                               const float* __restrict__ gsp, float* g, ShAdd& sh_add,
                                               float2* dstat = nullptr) {
  typename M::Pre pre;
  M::pre(pt, pre);
  float acc[M::kAcc];
#pragma unroll
  for (int k = 0; k < M::kAcc; ++k) acc[k] = 0.f;
  uint32_t m = mask;
  while (m) {
    const int v = __ffs(m) - 1;
    m &= m - 1;
    const int64_t row = s_row0[v] + rk.row_offset(v);
    float gs[M::kGSP];
    const float* src = gsp + row * M::kGSP;
#if BS_GSP_LDCS
    // the row's last use before the next step's projection clears it: evict-first
#pragma unroll
    for (int k = 0; k < M::kGSP / 4; ++k) {
      const float4 t = __ldcs(reinterpret_cast<const float4*>(src) + k);
      gs[4 * k] = t.x, gs[4 * k + 1] = t.y, gs[4 * k + 2] = t.z, gs[4 * k + 3] = t.w;
    }
#else
#pragma unroll
    for (int k = 0; k < M::kGSP; ++k) gs[k] = src[k];
#endif
    typename M::F f;
    float wk[16];  // SH direction weights, computed with the colour (one pass over the coefficients)
    M::forward(pt, pre, sh, s_cam[v], a.n_sh, f, M::kFuseWk ? gs + M::kGcol : nullptr, M::kFuseWk ? wk : nullptr);
    if (!a.gsp_standard) M::from_moments(f, gs);
    if constexpr (!M::k2D) {
      // densification statistic: |dL/d mean2d| in NDC units (u = (x_ndc + 1) W / 2), views with a valid splat
      if (dstat && f.valid) {
        const float gx = gs[0] * (0.5f * (float)s_cam[v].width), gy = gs[1] * (0.5f * (float)s_cam[v].height);
        dstat->x += sqrtf(gx * gx + gy * gy);
        dstat->y += 1.f;
      }
    }
    M::backward(pt, pre, sh, s_cam[v], a.n_sh, f, gs, g, acc, sh_add, M::kFuseWk ? wk : nullptr);
  }
  M::finish(pt, acc, g);
}

// SH gradient accumulators (sh_colour_backward's add4): registers, or this
// thread's float4 column of shared memory ([12][kProjThreads] float4)
struct ShAccRegs {
  float* g;
  __device__ __forceinline__ void add4(int q, float4 v) {
    g[4 * q] += v.x;
    g[4 * q + 1] += v.y;
    g[4 * q + 2] += v.z;
    g[4 * q + 3] += v.w;
  }
};
struct ShAccSmem {
  float4* col;  // &entry[0][thread]
  __device__ __forceinline__ void add4(int q, float4 v) {
    float4 t = col[q * kProjThreads];
    t.x += v.x;
    t.y += v.y;
    t.z += v.z;
    t.w += v.w;
    col[q * kProjThreads] = t;
  }
};

template <class M>
__global__ void __launch_bounds__(kProjThreads) project_bwd_kernel(ProjArgs a, const float* __restrict__ gsp,
                                                                   float4* __restrict__ gparams) {
  __shared__ uint32_t s_bal[kProjWarps * kMaxViews];
  __shared__ int s_run[kMaxViews];
  __shared__ bs_camera s_cam[kMaxViews];
  __shared__ int64_t s_row0[kMaxViews];
  const int g = blockIdx.x, B = a.B;
  if (threadIdx.x < B) {
    s_run[threadIdx.x] = 0;
    s_cam[threadIdx.x] = a.cams[threadIdx.x];
    s_row0[threadIdx.x] = a.view_row0[threadIdx.x] + a.base[(size_t)g * B + threadIdx.x];
  }
  __syncthreads();
  RowRanker rk{s_bal, s_run};
  int lo, end;
  if (!chunk_range(a.group_begin, a.mask, a.chunk_prefix, rk, g, blockIdx.y, gridDim.y, B, lo, end)) return;
  for (int b0 = lo; b0 < end; b0 += kProjThreads) {
    const int i = b0 + threadIdx.x;
    const uint32_t mask = i < end ? a.mask[i] : 0u;
    if (!__syncthreads_or(mask != 0u)) continue;  // no visible point: no row, no gradient
    rk.round(mask, B);
    if (mask) {
      PointIn pt;
      load_point(a.params, a.S, i, a.n_sh, pt);
      PointGrad gr;
#pragma unroll
      for (int k = 0; k < 60; ++k) gr.g[k] = 0.f;
      ShAccRegs acc{gr.g + 12};
      point_backward<M>(a, s_cam, s_row0, rk, mask, pt, ShRegs{pt.sh}, gsp, gr.g, acc);
#pragma unroll
      for (int p = 0; p < BS_PARAM_PLANES; ++p) {
        float4 acc = gparams[p * a.S + i];
        acc.x += gr.g[4 * p];
        acc.y += gr.g[4 * p + 1];
        acc.z += gr.g[4 * p + 2];
        acc.w += gr.g[4 * p + 3];
        gparams[p * a.S + i] = acc;
      }
    }
    if (b0 + kProjThreads < end) rk.advance(B);  // (a chunk's single round needs no advance)
  }
}

struct AdamConsts {
  float step[BS_PARAM_FLOATS];  // lr / (1 - beta1^t) per lane
  float beta1, beta2, eps, inv_bc2_sqrt;
  int selective;
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// torch.optim.Adam (foreach=False) update on one float4 of a plane:
//   m += (1 - b1)(g - m);  v = b2 v + (1 - b2) g^2
//   p -= lr / bc1 * m / (sqrt(v) / sqrt(bc2) + eps)
// with the square root and the two divisions as MUFU approximations
// (~1e-7 relative on the update; tests compare with torch at rtol 1e-5):
// the IEEE-exact sequence cost ~40 instructions per scalar, 30% of the
// fused projection-backward + Adam kernel.
__device__ __forceinline__ void adam4(float4& p, float4 g, float4& m, float4& v, const AdamConsts& c, int plane) {
  float* pp = &p.x;
  float* gg = &g.x;
  float* mm = &m.x;
  float* vv = &v.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mm[k] = mm[k] + (1.f - c.beta1) * (gg[k] - mm[k]);
    vv[k] = c.beta2 * vv[k] + (1.f - c.beta2) * gg[k] * gg[k];
    const float denom = sqrt_approx(vv[k]) * c.inv_bc2_sqrt + c.eps;
    pp[k] = pp[k] - __fdividef(c.step[4 * plane + k] * mm[k], denom);
  }
}

__global__ void __launch_bounds__(256) adam_kernel(AdamConsts c, float4* __restrict__ params,
                                                   const float4* __restrict__ grads, float4* __restrict__ m,
                                                   float4* __restrict__ v, int64_t S,
                                                   const uint32_t* __restrict__ mask) {
  const int64_t total = S * BS_PARAM_PLANES;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(t / S);
    const int64_t i = t - plane * S;
    if (c.selective && mask && mask[i] == 0u) continue;
    float4 p = params[t], mm = m[t], vv = v[t];
    adam4(p, grads[t], mm, vv, c, plane);
    params[t] = p;
    m[t] = mm;
    v[t] = vv;
  }
}

template <class M, bool kWork>
__device__ __forceinline__ void project_bwd_adam_chunk(const ProjArgs& a, const AdamConsts& c,
                                                       const float* __restrict__ gsp, float4* params,
                                                       float4* __restrict__ m, float4* __restrict__ v, int g, int cy,
                                                       int ny) {
  // [12][kProjThreads] float4 SH gradients, then [12][kProjThreads] float4 SH values
  extern __shared__ float4 s_gsh4[];
  float4* s_sh4 = s_gsh4 + 12 * kProjThreads;
  __shared__ uint32_t s_bal[kProjWarps * kMaxViews];
  __shared__ int s_run[kMaxViews];
  __shared__ bs_camera s_cam[kMaxViews];
  __shared__ int64_t s_row0[kMaxViews];
  const int B = a.B;
  if (threadIdx.x < B) {
    s_run[threadIdx.x] = 0;
    s_cam[threadIdx.x] = a.cams[threadIdx.x];
    s_row0[threadIdx.x] = a.view_row0[threadIdx.x] + a.base[(size_t)g * B + threadIdx.x];
  }
  __syncthreads();
  RowRanker rk{s_bal, s_run};
  int lo, end;
  if (!chunk_range(a.group_begin, a.mask, a.chunk_prefix, rk, g, cy, ny, B, lo, end)) return;
  for (int b0 = lo; b0 < end; b0 += kProjThreads) {
    const int i = b0 + threadIdx.x;
    const bool ok = i < end;
    const uint32_t mask = ok ? a.mask[i] : 0u;
    // selective Adam: a round without a visible point updates nothing (and
    // its rows advance no view's count) -- skip it before any traffic
    if (c.selective && !__syncthreads_or(mask != 0u)) continue;
    // Copies that cost no registers: the block's parameter and moment planes
    // into L2 by the bulk-copy engine (one contiguous request per (array,
    // plane)) for the Adam update, and this point's SH coefficients into its
    // own shared-memory column (cp.async) for the per-view math, which then
    // reads them at shared-memory latency instead of one dependent global
    // load per float4.
    if (threadIdx.x < 3 * BS_PARAM_PLANES) {
      const int arr = threadIdx.x / BS_PARAM_PLANES, pl = threadIdx.x % BS_PARAM_PLANES;
      const float4* base4 = arr == 0 ? params : (arr == 1 ? m : v);
      const uint32_t bytes = 16u * (uint32_t)min(kProjThreads, end - b0);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base4 + (int64_t)pl * a.S + b0), "r"(bytes)
                   : "memory");
    }
    const int sh_q = (3 * a.n_sh + 3) / 4;  // float4 entries holding this degree's coefficients
    // only visible points stage their coefficients: every copy issued here is
    // waited for below (cp.async.wait_all inside `if (mask)`), so no copy is
    // left in flight into the column when the next round reuses it
    if (mask) {
      for (int q = 0; q < sh_q; ++q) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_sh4 + q * kProjThreads + threadIdx.x);
        sh_copy16(dst, params + (int64_t)(3 + q) * a.S + i);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    rk.template round<kWork>(mask, B);
    if (ok && !(c.selective && mask == 0u)) {
      // geometry gradient in registers, the 48 SH gradients in this thread's
      // shared-memory column (keeps the register peak below the
      // 2-CTAs-per-SM budget)
      float g12[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) g12[k] = 0.f;
      float4* my_sh = s_gsh4 + threadIdx.x;
#pragma unroll
      for (int q = 0; q < 12; ++q) my_sh[q * kProjThreads] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (mask) {
        PointIn pt;
        load_point(a.params, a.S, i, 0, pt);  // geometry planes only; SH from shared memory
        asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own column
        const ShSmem sh{s_sh4 + threadIdx.x};
        ShAccSmem acc{my_sh};
        if (a.densify_stats != nullptr && !M::k2D) {
          float2 ds = make_float2(0.f, 0.f);
          point_backward<M>(a, s_cam, s_row0, rk, mask, pt, sh, gsp, g12, acc, &ds);
          float2 t = a.densify_stats[i];
          a.densify_stats[i] = make_float2(t.x + ds.x, t.y + ds.y);
        } else {
          point_backward<M>(a, s_cam, s_row0, rk, mask, pt, sh, gsp, g12, acc);
        }
      }
      // Adam over the 15 planes, 3 planes per batch: all 15 loads of a batch
      // are issued before its first store (memory-level parallelism)
#pragma unroll
      for (int p0 = 0; p0 < BS_PARAM_PLANES; p0 += kAdamBatch) {
        float4 pp[kAdamBatch], mm[kAdamBatch], vv[kAdamBatch];
#pragma unroll
        for (int k = 0; k < kAdamBatch; ++k) {
          const int64_t t = (p0 + k) * a.S + i;
#if BS_ADAM_SMEM_PARAMS
          // SH planes of a visible point: already in this thread's shared column
          const int q = p0 + k - 3;
          pp[k] = (q >= 0 && q < sh_q && mask) ? s_sh4[q * kProjThreads + threadIdx.x] : params[t];
#else
          pp[k] = params[t];
#endif
#if BS_ADAM_STREAM == 1
          mm[k] = __ldcs(m + t);
          vv[k] = __ldcs(v + t);
#else
          mm[k] = m[t];
          vv[k] = v[t];
#endif
        }
#pragma unroll
        for (int k = 0; k < kAdamBatch; ++k) {
          const int p = p0 + k;
          const int64_t t = p * a.S + i;
          const float4 gg = p < 3 ? make_float4(g12[4 * p], g12[4 * p + 1], g12[4 * p + 2], g12[4 * p + 3])
                                  : my_sh[(p - 3) * kProjThreads];
          adam4(pp[k], gg, mm[k], vv[k], c, p);
#if BS_ADAM_STREAM
          __stcs(params + t, pp[k]);
          __stcs(m + t, mm[k]);
          __stcs(v + t, vv[k]);
#else
          params[t] = pp[k];
          m[t] = mm[k];
          v[t] = vv[k];
#endif
        }
      }
    }
    if (b0 + kProjThreads < end) rk.advance(B);  // (a chunk's single round needs no advance)
  }
}

template <class M, bool kWork>
__global__ void __launch_bounds__(kProjThreads, 2) project_bwd_adam_kernel(ProjArgs a, AdamConsts c,
                                                                           const float* __restrict__ gsp,
                                                                           float4* params,
                                                                           float4* __restrict__ m,
                                                                           float4* __restrict__ v) {
  if constexpr (!kWork) {
    project_bwd_adam_chunk<M, false>(a, c, gsp, params, m, v, blockIdx.x, blockIdx.y, gridDim.y);
    return;
  }
  // selective Adam over the visible chunks only (the launcher passes the list
  // only then: dense Adam updates every point)
  const int n = *a.work_count;
  for (int w = blockIdx.x; w < n; w += gridDim.x) {
    const int item = __ldg(a.work_list + w);
    project_bwd_adam_chunk<M, true>(a, c, gsp, params, m, v, item / a.max_chunks, item % a.max_chunks, a.max_chunks);
    __syncthreads();
  }
}

// ---- row layout ------------------------------------------------------------

__global__ void __launch_bounds__(1024) scan_counts_kernel(const int32_t* __restrict__ counts, int ng, int B,
                                                           int32_t* __restrict__ base, int64_t* __restrict__ rows) {
  __shared__ int s_w[32];
  const int v = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < ng; b0 += 1024) {
    const int gi = b0 + tid;
    const int x0 = gi < ng ? counts[(size_t)gi * B + v] : 0;
    int x = x0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      s_w[lane] = t;
    }
    __syncthreads();
    if (gi < ng) base[(size_t)gi * B + v] = carry + (w ? s_w[w - 1] : 0) + x - x0;
    const int tot = s_w[31];
    __syncthreads();
    carry += tot;
  }
  if (tid == 0) rows[v] = carry;
}

struct ViewOrder {
  int order[kMaxViews];
};

__global__ void view_row0_kernel(const int64_t* __restrict__ rows, ViewOrder o, int B, int64_t* __restrict__ row0) {
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int k = 0; k < B; ++k) {
      row0[o.order[k]] = acc;
      acc += rows[o.order[k]];
    }
  }
}

__global__ void row_support_kernel(const float* __restrict__ sp, int stride, bool two_d, int64_t n,
                                   float* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    out[r] = row_support_value(sp[r * stride + 2], two_d);  // opacity: float 2 of both row layouts
}

int32_t check_proj(const bs_proj_desc* d) {
  BS_REQUIRE(d != nullptr, BS_ERR_PARAMETER, "null projection descriptor");
  BS_REQUIRE(d->n_views >= 1 && d->n_views <= kMaxViews, BS_ERR_PARAMETER, "projection supports 1..32 views");
  BS_REQUIRE(d->sh_degree >= 0 && d->sh_degree <= 3, BS_ERR_PARAMETER, "sh_degree must be in [0, 3]");
  BS_REQUIRE(d->max_group_points >= 0 && d->max_group_points <= (1 << 24), BS_ERR_PARAMETER,
             "max_group_points must be in [0, 2^24]");
  return BS_OK;
}

dim3 proj_grid(const bs_proj_desc* d, int n_groups) {
  const int chunks = d->max_group_points > 0 ? (d->max_group_points + kProjThreads - 1) / kProjThreads : 1;
  return dim3(n_groups, chunks);
}

// The visible-chunk work list applies when the chunk prefixes it indexes are
// given; the grid-stride launch then uses up to 8 x `ctas_per_sm` CTAs per
// SM (so a step whose chunks are all visible keeps one CTA per chunk).
bool use_work(const bs_proj_desc* d) { return d->work_list && d->max_group_points > 0 && d->chunk_prefix; }

void set_work(ProjArgs& a, const bs_proj_desc* d, int n_groups, bool on) {
  a.max_chunks = (int)proj_grid(d, n_groups).y;
  a.work_list = on ? d->work_list : nullptr;
  a.work_count = on ? d->work_count : nullptr;
}

dim3 work_grid(const bs_proj_desc* d, int n_groups, int ctas_per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const dim3 full = proj_grid(d, n_groups);
  const long long total = (long long)full.x * full.y;
  return dim3((unsigned)std::min<long long>(total, 8ll * ctas_per_sm * sms), 1);
}

AdamConsts make_adam(const bs_adam_desc* d) {
  AdamConsts c;
  const double bc1 = 1.0 - pow((double)d->beta1, (double)d->step);
  const double bc2 = 1.0 - pow((double)d->beta2, (double)d->step);
  for (int k = 0; k < BS_PARAM_FLOATS; ++k) c.step[k] = (float)((double)d->lr[k] / bc1);
  c.beta1 = d->beta1;
  c.beta2 = d->beta2;
  c.eps = d->eps;
  c.inv_bc2_sqrt = (float)(1.0 / sqrt(bc2));
  c.selective = d->selective;
  return c;
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_scan_counts(const int32_t* counts, int32_t n_groups, int32_t n_views,
                                  const int32_t* view_order_host, int32_t* base, int64_t* view_rows,
                                  int64_t* view_row0, void* stream) {
  BS_REQUIRE(n_views >= 1 && n_views <= kMaxViews, BS_ERR_PARAMETER, "scan_counts supports 1..32 views");
  ViewOrder o;
  bool seen[kMaxViews] = {false};
  for (int k = 0; k < n_views; ++k) {
    const int v = view_order_host ? view_order_host[k] : k;
    BS_REQUIRE(v >= 0 && v < n_views && !seen[v], BS_ERR_PARAMETER, "view_order must be a permutation");
    seen[v] = true;
    o.order[k] = v;
  }
  cudaStream_t s = as_stream(stream);
  if (n_groups > 0) {
    scan_counts_kernel<<<n_views, 1024, 0, s>>>(counts, n_groups, n_views, base, view_rows);
    BS_LAUNCH_CHECK("scan_counts_kernel");
  } else {
    cudaMemsetAsync(view_rows, 0, sizeof(int64_t) * n_views, s);
  }
  view_row0_kernel<<<1, 32, 0, s>>>(view_rows, o, n_views, view_row0);
  BS_LAUNCH_CHECK("view_row0_kernel");
  return BS_OK;
}

extern "C" int32_t bs_project_fwd(const bs_proj_desc* d, const float* params, int64_t n_points,
                                  const uint32_t* vis_mask, const int32_t* group_begin, int32_t n_groups,
                                  const int32_t* base, const int64_t* view_row0, const bs_camera* cams,
                                  float* sp_rows, void* stream) {
  int32_t st = check_proj(d);
  if (st) return st;
  if (n_groups == 0) return BS_OK;
  const int n_sh = (d->sh_degree + 1) * (d->sh_degree + 1);
  ProjArgs a{d->n_views, n_sh, reinterpret_cast<const float4*>(params), n_points, vis_mask, group_begin, base,
             view_row0, cams, d->gsp_form, d->max_group_points > 0 ? d->chunk_prefix : nullptr, d->gsp_zero,
             d->point_gid, d->row_gid, d->row_support, d->view_sp, d->view_gid, d->bucket_counts,
             reinterpret_cast<int4*>(d->row_bin), d->tiles_per_slot};
  const bool work = use_work(d);
  set_work(a, d, n_groups, work);
  const dim3 grid = work ? work_grid(d, n_groups, BS_PROJ_FWD_CTAS) : proj_grid(d, n_groups);
  const size_t smem = sizeof(float4) * 12 * kProjThreads;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, kProjThreads, smem, as_stream(stream)>>>(a, sp_rows);
  };
  if (d->model == BS_MODEL_2DGS) work ? launch(project_fwd_kernel<Model2, true>) : launch(project_fwd_kernel<Model2, false>);
  else work ? launch(project_fwd_kernel<Model3, true>) : launch(project_fwd_kernel<Model3, false>);
  BS_LAUNCH_CHECK("project_fwd_kernel");
  return BS_OK;
}

extern "C" int32_t bs_project_bwd(const bs_proj_desc* d, const float* params, int64_t n_points,
                                  const uint32_t* vis_mask, const int32_t* group_begin, int32_t n_groups,
                                  const int32_t* base, const int64_t* view_row0, const bs_camera* cams,
                                  const float* g_sp, float* grad_params, void* stream) {
  int32_t st = check_proj(d);
  if (st) return st;
  if (n_groups == 0) return BS_OK;
  const int n_sh = (d->sh_degree + 1) * (d->sh_degree + 1);
  ProjArgs a{d->n_views, n_sh, reinterpret_cast<const float4*>(params), n_points, vis_mask, group_begin, base,
             view_row0, cams, d->gsp_form, d->max_group_points > 0 ? d->chunk_prefix : nullptr, nullptr,
             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  set_work(a, d, n_groups, false);
  const dim3 grid = proj_grid(d, n_groups);
  if (d->model == BS_MODEL_2DGS)
    project_bwd_kernel<Model2><<<grid, kProjThreads, 0, as_stream(stream)>>>(
        a, g_sp, reinterpret_cast<float4*>(grad_params));
  else
    project_bwd_kernel<Model3><<<grid, kProjThreads, 0, as_stream(stream)>>>(
        a, g_sp, reinterpret_cast<float4*>(grad_params));
  BS_LAUNCH_CHECK("project_bwd_kernel");
  return BS_OK;
}

extern "C" int32_t bs_adam_step(const bs_adam_desc* d, float* params, const float* grads, float* exp_avg,
                                float* exp_avg_sq, int64_t n_points, const uint32_t* vis_mask, void* stream) {
  BS_REQUIRE(d != nullptr && d->step >= 1, BS_ERR_PARAMETER, "adam: step must be >= 1");
  BS_REQUIRE(!d->selective || vis_mask, BS_ERR_PARAMETER, "selective adam needs the visibility mask");
  if (n_points == 0) return BS_OK;
  AdamConsts c = make_adam(d);
  adam_kernel<<<grid_for(n_points * BS_PARAM_PLANES, 256), 256, 0, as_stream(stream)>>>(
      c, reinterpret_cast<float4*>(params), reinterpret_cast<const float4*>(grads),
      reinterpret_cast<float4*>(exp_avg), reinterpret_cast<float4*>(exp_avg_sq), n_points, vis_mask);
  BS_LAUNCH_CHECK("adam_kernel");
  return BS_OK;
}

extern "C" int32_t bs_project_bwd_adam(const bs_proj_desc* pd, const bs_adam_desc* ad, float* params,
                                       float* exp_avg, float* exp_avg_sq, int64_t n_points,
                                       const uint32_t* vis_mask, const int32_t* group_begin, int32_t n_groups,
                                       const int32_t* base, const int64_t* view_row0, const bs_camera* cams,
                                       const float* g_sp, void* stream) {
  int32_t st = check_proj(pd);
  if (st) return st;
  BS_REQUIRE(ad != nullptr && ad->step >= 1, BS_ERR_PARAMETER, "adam: step must be >= 1");
  if (n_groups == 0) return BS_OK;
  const int n_sh = (pd->sh_degree + 1) * (pd->sh_degree + 1);
  ProjArgs a{pd->n_views, n_sh, reinterpret_cast<const float4*>(params), n_points, vis_mask, group_begin, base,
             view_row0, cams, pd->gsp_form, pd->max_group_points > 0 ? pd->chunk_prefix : nullptr, nullptr,
             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
             reinterpret_cast<float2*>(pd->densify_stats)};
  AdamConsts c = make_adam(ad);
  // dense Adam updates every point: the visible-chunk list only with selective Adam
  const bool work = use_work(pd) && c.selective;
  set_work(a, pd, n_groups, work);
  const dim3 grid = work ? work_grid(pd, n_groups, 2) : proj_grid(pd, n_groups);
  const size_t smem = sizeof(float4) * 24 * kProjThreads;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, kProjThreads, smem, as_stream(stream)>>>(a, c, g_sp, reinterpret_cast<float4*>(params),
                                                             reinterpret_cast<float4*>(exp_avg),
                                                             reinterpret_cast<float4*>(exp_avg_sq));
  };
  if (pd->model == BS_MODEL_2DGS)
    work ? launch(project_bwd_adam_kernel<Model2, true>) : launch(project_bwd_adam_kernel<Model2, false>);
  else work ? launch(project_bwd_adam_kernel<Model3, true>) : launch(project_bwd_adam_kernel<Model3, false>);
  BS_LAUNCH_CHECK("project_bwd_adam_kernel");
  return BS_OK;
}

extern "C" int32_t bs_row_support(const float* sp_rows, int32_t model, int64_t n_rows, float* out, void* stream) {
  BS_REQUIRE(model == BS_MODEL_3DGS || model == BS_MODEL_2DGS, BS_ERR_PARAMETER, "unknown splat model");
  if (n_rows <= 0) return BS_OK;
  const bool two_d = model == BS_MODEL_2DGS;
  row_support_kernel<<<grid_for(n_rows, 256), 256, 0, as_stream(stream)>>>(sp_rows, two_d ? kSP2 : BS_SP_FLOATS, two_d,
                                                                          n_rows, out);
  BS_LAUNCH_CHECK("row_support_kernel");
  return BS_OK;
}
