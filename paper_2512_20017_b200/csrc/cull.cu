// K0: frustum culling + access counting, Morton codes, grouping helpers.
//
// Semantics follow /root/reference/pkg/src/splatsched/visibility.py:
//   * signed distance d = p . n + off in float64, OpenBLAS order
//     (visibility.py:155-156) -> bs::plane_dist
//   * inside iff d >= 0 on inclusive planes, d > 0 on exclusive ones
//     (visibility.py:158-161); the exclusive right/bottom plane of a patch
//     is the exact negation of the next patch's left/top plane
//     (visibility.py:196-208), so "-d > 0" is evaluated as "d < 0" on the
//     shared plane.
//   * a group is skipped for a patch iff some plane of that patch has all
//     8 AABB corners strictly outside (visibility.py:263-276), and only
//     points of non-skipped groups are counted (visibility.py:283-292,
//     337-357) -- applied per patch exactly like _candidate_indices.
//   * temporal presence compared in float32 (visibility.py:251 under
//     NumPy-2 weak-scalar promotion).
#include "common.cuh"

namespace bs {
namespace {

constexpr int kCullThreads = 256;
constexpr int kMaxPatchCountsSmem = 8192;  // ints of smem histogram

struct CullArgs {
  int mode, B, P, N, temporal, stride;
  const float* pos;
  const float* presence;
  const int32_t* group_begin;
  const float* aabb;
  int n_groups;
  const double* planes;  // [B][npl][4]
  const float* view_times;
  const int32_t* point_gpu;
  void* out0;
  void* out1;
  void* out2;
  int max_chunks;
  int32_t* chunk_prefix;  // MASK: [n_groups][max_chunks][B] or NULL
};
static_assert(kCullThreads == 256, "chunk_prefix counts 256-point chunks (the projection CTA size)");

// Plane indices inside one view's block: 0 near, 1 far, 2..2+P x-edges,
// 3+P..3+2P y-edges.
__device__ __forceinline__ int npl_of(int P) { return 2 + 2 * (P + 1); }

// True iff some plane of patch (r, c) puts all 8 corners strictly outside.
__device__ bool aabb_outside(const double* vp, int P, int r, int c, const double lo[3],
                             const double hi[3]) {
  // plane list of the patch: near, far, xe[c], -xe[c+1], ye[r], -ye[r+1]
  const double* pl[6] = {vp, vp + 4, vp + 4 * (2 + c), vp + 4 * (2 + c + 1),
                         vp + 4 * (3 + P + r), vp + 4 * (3 + P + r + 1)};
  const bool neg[6] = {false, false, false, true, false, true};
  for (int k = 0; k < 6; ++k) {
    bool all_out = true;
    for (int i = 0; i < 8 && all_out; ++i) {
      const double x = (i & 4) ? hi[0] : lo[0];
      const double y = (i & 2) ? hi[1] : lo[1];
      const double z = (i & 1) ? hi[2] : lo[2];
      const double d = plane_dist(pl[k], x, y, z);
      all_out = neg[k] ? (d > 0.0) : (d < 0.0);
    }
    if (all_out) return true;
  }
  return false;
}

template <int MODE>
__global__ void __launch_bounds__(kCullThreads) cull_kernel(CullArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = a.P, B = a.B, PP = P * P, N = a.N;
  const int npl = npl_of(P);
  double* s_planes = reinterpret_cast<double*>(smem_raw);            // B*npl*4
  uint8_t* s_live = reinterpret_cast<uint8_t*>(s_planes + B * npl * 4);  // B*PP
  int* s_cnt = reinterpret_cast<int*>(s_live + ((B * PP + 15) & ~15));
  __shared__ int s_any_live;
  __shared__ uint8_t s_view_live[1024];

  const int g = blockIdx.x;
  const int begin = a.group_begin[g], end = a.group_begin[g + 1];
  const int tid = threadIdx.x;

  for (int i = tid; i < B * npl * 4; i += blockDim.x) s_planes[i] = a.planes[i];
  int n_cnt = 0;
  if (MODE == BS_CULL_ACCESS_EXACT || MODE == BS_CULL_ACCESS_GROUP) n_cnt = B * PP * N;
  if (MODE == BS_CULL_EDGES) n_cnt = B;
  if (MODE == BS_CULL_MASK) n_cnt = B + B * PP;
  const bool smem_cnt = n_cnt <= kMaxPatchCountsSmem;
  const int zero_n = smem_cnt ? n_cnt : ((MODE == BS_CULL_MASK || MODE == BS_CULL_EDGES) ? B : 0);
  for (int i = tid; i < zero_n; i += blockDim.x) s_cnt[i] = 0;
  if (tid == 0) s_any_live = 0;
  __syncthreads();

  // ---- group AABB early-out per (view, patch) --------------------------
  for (int j = tid; j < B * PP; j += blockDim.x) {
    uint8_t live = 1;
    if (a.aabb != nullptr) {
      const float* bx = a.aabb + 6 * (size_t)g;
      const double lo[3] = {bx[0], bx[1], bx[2]};
      const double hi[3] = {bx[3], bx[4], bx[5]};
      const int v = j / PP, rc = j % PP;
      live = aabb_outside(s_planes + (size_t)v * npl * 4, P, rc / P, rc % P, lo, hi) ? 0 : 1;
    }
    s_live[j] = live;
    if (live) s_any_live = 1;
  }
  __syncthreads();
  for (int v = tid; v < B && v < 1024; v += blockDim.x) {
    uint8_t any = 0;
    for (int j = 0; j < PP; ++j) any |= s_live[v * PP + j];
    s_view_live[v] = any;
  }
  __syncthreads();
  // MASK mode (B <= 32): the group's live views as a bit set, so the
  // per-point loop visits only them (a group is usually live in 1-3 of the
  // batch's views)
  uint32_t live_bits = 0;
  if (MODE == BS_CULL_MASK)
    for (int v = 0; v < B && v < 32; ++v) live_bits |= (uint32_t)s_view_live[v] << v;

  if (MODE == BS_CULL_ACCESS_GROUP) {
    // Every point of a non-culled group counts (GROUP_APPROX).
    for (int i = begin + tid; i < end; i += blockDim.x) {
      const int gpu = a.point_gpu ? a.point_gpu[i] : 0;
      for (int j = 0; j < B * PP; ++j)
        if (s_live[j]) {
          if (smem_cnt) atomicAdd(&s_cnt[j * N + gpu], 1);
          else atomicAdd(reinterpret_cast<unsigned long long*>(a.out0) + (size_t)j * N + gpu, 1ull);
        }
    }
  } else if (MODE == BS_CULL_MASK && !s_any_live) {
    // the group is outside every batch frustum (CTA-uniform; at C4 ~98 % of
    // the groups): zero masks and chunk prefixes, no per-point plane tests
    for (int i = begin + tid; i < end; i += blockDim.x) static_cast<uint32_t*>(a.out0)[i] = 0u;
    if (a.chunk_prefix) {
      const int n_chunks = (end - begin + kCullThreads - 1) / kCullThreads;
      for (int t = tid; t < n_chunks * B; t += blockDim.x)
        a.chunk_prefix[((size_t)g * a.max_chunks + t / B) * B + t % B] = 0;
    }
  } else if (s_any_live) {
    const int lane = tid & 31;
    for (int base = begin; base < end; base += blockDim.x) {
      if (MODE == BS_CULL_MASK && a.chunk_prefix) {
        // counts of the chunks before this one (all of them are in s_cnt)
        __syncthreads();
        if (tid < B)
          a.chunk_prefix[((size_t)g * a.max_chunks + (base - begin) / kCullThreads) * B + tid] = s_cnt[tid];
        __syncthreads();
      }
      const int i = base + tid;
      const bool valid = i < end;
      double x = 0, y = 0, z = 0;
      float t0 = 0.f, t1 = 0.f;
      int gpu = 0;
      if (valid && s_any_live) {
        const float* p = a.pos + (size_t)i * a.stride;
        x = p[0];
        y = p[1];
        z = p[2];
        if (a.temporal) {
          t0 = a.presence[2 * (size_t)i];
          t1 = a.presence[2 * (size_t)i + 1];
        }
        if (MODE == BS_CULL_ACCESS_EXACT && a.point_gpu) gpu = a.point_gpu[i];
      }
      uint32_t mask = 0;
      uint32_t todo = live_bits;
      for (int v = 0; MODE == BS_CULL_MASK ? todo != 0u : v < B; ++v) {
        if (MODE == BS_CULL_MASK) {  // next live view (CTA-uniform)
          v = __ffs(todo) - 1;
          todo &= todo - 1;
        }
        bool vis_view = false;
        // any live patch for this view? (uniform across the CTA)
        if (s_view_live[v] && valid) {
          const double* vp = s_planes + (size_t)v * npl * 4;
          bool in_time = true;
          if (a.temporal) {
            const float tv = a.view_times[v];
            in_time = (t0 <= tv) && (tv <= t1);
          }
          if (in_time && plane_dist(vp, x, y, z) >= 0.0 && plane_dist(vp + 4, x, y, z) >= 0.0) {
            // column / row membership from the shared edge planes
            double dprev = plane_dist(vp + 8, x, y, z);
            for (int c = 0; c < P; ++c) {
              const double dnext = plane_dist(vp + 4 * (2 + c + 1), x, y, z);
              if (dprev >= 0.0 && dnext < 0.0) {
                double eprev = plane_dist(vp + 4 * (3 + P), x, y, z);
                for (int r = 0; r < P; ++r) {
                  const double enext = plane_dist(vp + 4 * (3 + P + r + 1), x, y, z);
                  if (eprev >= 0.0 && enext < 0.0 && s_live[v * PP + r * P + c]) {
                    const int j = v * PP + r * P + c;
                    vis_view = true;
                    if (MODE == BS_CULL_ACCESS_EXACT) {
                      if (smem_cnt) atomicAdd(&s_cnt[j * N + gpu], 1);
                      else
                        atomicAdd(reinterpret_cast<unsigned long long*>(a.out0) + (size_t)j * N + gpu,
                                  1ull);
                    } else if (MODE == BS_CULL_MASK && a.out2) {
                      if (smem_cnt) atomicAdd(&s_cnt[B + j], 1);
                      else atomicAdd(reinterpret_cast<unsigned long long*>(a.out2) + j, 1ull);
                    }
                  }
                  eprev = enext;
                }
              }
              dprev = dnext;
            }
          }
        }
        if ((MODE == BS_CULL_EDGES || MODE == BS_CULL_MASK) && s_view_live[v]) {  // CTA-uniform
          const unsigned bal = __ballot_sync(0xffffffffu, vis_view);
          if (lane == 0 && bal) atomicAdd(&s_cnt[v], __popc(bal));
          if (vis_view) mask |= 1u << (v & 31);
        }
      }
      if (MODE == BS_CULL_MASK && valid) static_cast<uint32_t*>(a.out0)[i] = mask;
    }
  }
  __syncthreads();

  // ---- flush ----------------------------------------------------------------
  if (MODE == BS_CULL_ACCESS_EXACT || MODE == BS_CULL_ACCESS_GROUP) {
    if (smem_cnt)
      for (int i = tid; i < n_cnt; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(reinterpret_cast<unsigned long long*>(a.out0) + i, (unsigned long long)s_cnt[i]);
  } else if (MODE == BS_CULL_EDGES) {
    for (int v = tid; v < B; v += blockDim.x) static_cast<int32_t*>(a.out0)[(size_t)g * B + v] = s_cnt[v];
  } else if (MODE == BS_CULL_MASK) {
    for (int v = tid; v < B; v += blockDim.x) static_cast<int32_t*>(a.out1)[(size_t)g * B + v] = s_cnt[v];
    if (a.out2 && smem_cnt)
      for (int j = tid; j < B * PP; j += blockDim.x)
        if (s_cnt[B + j])
          atomicAdd(reinterpret_cast<unsigned long long*>(a.out2) + j, (unsigned long long)s_cnt[B + j]);
  }
}

// ---------------------------------------------------------------------------
// bbox (exact min/max) -- scene.py:109-112

__global__ void bbox_partial_kernel(const float* __restrict__ pos, int64_t n, int stride,
                                    float* __restrict__ part) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float* p = pos + i * stride;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mn[k] = fminf(mn[k], p[k]);
      mx[k] = fmaxf(mx[k], p[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    for (int o = 16; o > 0; o >>= 1) {
      mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
      mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
    }
  __shared__ float s[32][6];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 3; ++k) {
      s[w][k] = mn[k];
      s[w][3 + k] = mx[k];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    float r = s[0][threadIdx.x];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
      r = threadIdx.x < 3 ? fminf(r, s[j][threadIdx.x]) : fmaxf(r, s[j][threadIdx.x]);
    part[blockIdx.x * 6 + threadIdx.x] = r;
  }
}

__global__ void bbox_final_kernel(const float* __restrict__ part, int nparts, float* __restrict__ out) {
  const int k = threadIdx.x;
  if (k < 6) {
    float r = part[k];
    for (int j = 1; j < nparts; ++j) r = k < 3 ? fminf(r, part[j * 6 + k]) : fmaxf(r, part[j * 6 + k]);
    out[k] = r;
  }
}

constexpr int kBboxBlocks = 512;

// ---------------------------------------------------------------------------
// Morton codes -- visibility.py:33-62

__device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__global__ void morton_kernel(const float* __restrict__ pos, int64_t n, int stride,
                              const float* __restrict__ bbox, int bits, uint64_t* __restrict__ codes) {
  const double scale = (double)((1ull << bits) - 1);
  double mn[3], ext[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = (double)bbox[k];
    const double e = __dsub_rn((double)bbox[3 + k], mn[k]);
    ext[k] = e == 0.0 ? 1.0 : e;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double t = floor(__dmul_rn(__ddiv_rn(__dsub_rn((double)pos[i * stride + k], mn[k]), ext[k]), scale));
      t = fmin(fmax(t, 0.0), scale);
      q[k] = (uint64_t)t;
    }
    codes[i] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
  }
}

// One warp per group of G consecutive points.
__global__ void group_aabb_kernel(const float* __restrict__ pos, int64_t n, int stride, int G,
                                  int64_t n_groups, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const int64_t b = g * G, e = min(b + G, n);
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = b + lane; i < e; i += 32)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float v = pos[i * stride + k];
      mn[k] = fminf(mn[k], v);
      mx[k] = fmaxf(mx[k], v);
    }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    for (int o = 16; o > 0; o >>= 1) {
      mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
      mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
    }
  if (lane < 3) out[g * 6 + lane] = mn[lane];
  else if (lane < 6) out[g * 6 + lane] = mx[lane - 3];
}

__global__ void gather_planes_kernel(const float4* __restrict__ in, int64_t n_in,
                                     const int64_t* __restrict__ idx, int64_t n_out, int n_planes,
                                     float4* __restrict__ out) {
  const int64_t total = n_out * n_planes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / n_out, i = t - p * n_out;
    out[p * n_out + i] = in[p * n_in + idx[i]];
  }
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_cull_count(const bs_cull_desc* d, const float* positions, int64_t n_points,
                                 const float* presence, const int32_t* group_begin, const float* group_aabb,
                                 int32_t n_groups, const double* planes, const float* view_times,
                                 const int32_t* point_gpu, void* out0, void* out1, void* out2, void* stream) {
  BS_REQUIRE(d != nullptr, BS_ERR_PARAMETER, "bs_cull_count: null descriptor");
  BS_REQUIRE(d->P >= 1 && d->P <= 64, BS_ERR_PARAMETER, "patch factor P must be >= 1 (got %d)", d->P);
  BS_REQUIRE(d->n_views >= 1, BS_ERR_PARAMETER, "need at least one view");
  BS_REQUIRE(d->pos_stride >= 3, BS_ERR_PARAMETER, "pos_stride must be >= 3");
  BS_REQUIRE(n_points >= 0 && n_points < (1ll << 31), BS_ERR_PARAMETER, "n_points out of range");
  BS_REQUIRE(group_begin != nullptr && n_groups >= 0, BS_ERR_PARAMETER, "group offsets required");
  BS_REQUIRE(out0 != nullptr, BS_ERR_PARAMETER, "out0 required");
  BS_REQUIRE(!d->temporal || (presence && view_times), BS_ERR_CONFIGURATION,
             "temporal culling requested without timestamps");
  const int mode = d->mode;
  if (mode == BS_CULL_MASK) {
    BS_REQUIRE(d->n_views <= 32, BS_ERR_PARAMETER, "mask mode supports at most 32 views per launch");
    BS_REQUIRE(out1 != nullptr, BS_ERR_PARAMETER, "mask mode needs out1 (counts)");
  }
  if (mode == BS_CULL_ACCESS_GROUP)
    BS_REQUIRE(group_aabb != nullptr, BS_ERR_PARAMETER, "GROUP_APPROX needs group AABBs");
  if (mode == BS_CULL_ACCESS_EXACT || mode == BS_CULL_ACCESS_GROUP)
    BS_REQUIRE(d->n_gpus >= 1, BS_ERR_PARAMETER, "n_gpus must be >= 1");
  cudaStream_t s = as_stream(stream);
  const int B = d->n_views, P = d->P, PP = P * P;
  if (mode == BS_CULL_ACCESS_EXACT || mode == BS_CULL_ACCESS_GROUP) {
    if (cudaMemsetAsync(out0, 0, sizeof(int64_t) * (size_t)B * PP * d->n_gpus, s) != cudaSuccess)
      return set_error(BS_ERR_CUDA, "memset out0 failed");
  }
  if (mode == BS_CULL_MASK && out2) {
    if (cudaMemsetAsync(out2, 0, sizeof(int64_t) * (size_t)B * PP, s) != cudaSuccess)
      return set_error(BS_ERR_CUDA, "memset out2 failed");
  }
  if (n_groups == 0) return BS_OK;
  const int npl = 2 + 2 * (P + 1);
  int n_cnt = 0;
  if (mode == BS_CULL_ACCESS_EXACT || mode == BS_CULL_ACCESS_GROUP) n_cnt = B * PP * d->n_gpus;
  if (mode == BS_CULL_EDGES) n_cnt = B;
  if (mode == BS_CULL_MASK) n_cnt = B + B * PP;
  if (n_cnt > kMaxPatchCountsSmem) {
    BS_REQUIRE(mode != BS_CULL_EDGES && !(mode == BS_CULL_MASK && B > kMaxPatchCountsSmem), BS_ERR_PARAMETER,
               "too many views per launch");
    n_cnt = (mode == BS_CULL_MASK) ? B : 0;
  }
  const size_t smem = sizeof(double) * B * npl * 4 + ((B * PP + 15) & ~15) + sizeof(int) * (size_t)n_cnt;
  BS_REQUIRE(smem <= 200 * 1024, BS_ERR_PARAMETER, "too many views/patches for one launch (%zu B smem)", smem);
  if (mode == BS_CULL_MASK && d->chunk_prefix)
    BS_REQUIRE(d->max_chunks >= 1, BS_ERR_PARAMETER, "chunk_prefix needs max_chunks >= 1");
  CullArgs a{mode, B, P, d->n_gpus, d->temporal, d->pos_stride, positions, presence, group_begin,
             group_aabb, n_groups, planes, view_times, point_gpu, out0, out1, out2,
             d->max_chunks, mode == BS_CULL_MASK ? d->chunk_prefix : nullptr};
  auto launch = [&](auto kern) -> int32_t {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<n_groups, kCullThreads, smem, s>>>(a);
    return check_launch("cull_kernel");
  };
  switch (mode) {
    case BS_CULL_ACCESS_EXACT: return launch(cull_kernel<BS_CULL_ACCESS_EXACT>);
    case BS_CULL_ACCESS_GROUP: return launch(cull_kernel<BS_CULL_ACCESS_GROUP>);
    case BS_CULL_EDGES: return launch(cull_kernel<BS_CULL_EDGES>);
    case BS_CULL_MASK: return launch(cull_kernel<BS_CULL_MASK>);
  }
  return set_error(BS_ERR_PARAMETER, "unknown cull mode %d", mode);
}

extern "C" size_t bs_bbox_workspace(int64_t) { return sizeof(float) * 6 * kBboxBlocks; }

extern "C" int32_t bs_bbox(const float* positions, int64_t n, int32_t stride, float* bbox_out, void* ws,
                           size_t ws_bytes, void* stream) {
  BS_REQUIRE(n >= 1, BS_ERR_PARAMETER, "point cloud must be non-empty");
  BS_REQUIRE(ws_bytes >= bs_bbox_workspace(n), BS_ERR_CAPACITY, "bbox workspace too small");
  cudaStream_t s = as_stream(stream);
  const int blocks = (int)std::min<int64_t>(kBboxBlocks, (n + 255) / 256);
  bbox_partial_kernel<<<blocks, 256, 0, s>>>(positions, n, stride, static_cast<float*>(ws));
  BS_LAUNCH_CHECK("bbox_partial_kernel");
  bbox_final_kernel<<<1, 32, 0, s>>>(static_cast<float*>(ws), blocks, bbox_out);
  BS_LAUNCH_CHECK("bbox_final_kernel");
  return BS_OK;
}

extern "C" int32_t bs_morton_codes(const float* positions, int64_t n, int32_t stride, const float* bbox,
                                   int32_t bits, uint64_t* codes, void* stream) {
  BS_REQUIRE(bits >= 1 && bits <= 21, BS_ERR_PARAMETER, "bits_per_axis must be in [1, 21]");
  if (n == 0) return BS_OK;
  morton_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(positions, n, stride, bbox, bits, codes);
  BS_LAUNCH_CHECK("morton_kernel");
  return BS_OK;
}

extern "C" int32_t bs_group_aabb(const float* positions, int64_t n, int32_t stride, int32_t G, float* out,
                                 void* stream) {
  BS_REQUIRE(G >= 1, BS_ERR_PARAMETER, "group size G must be >= 1");
  if (n == 0) return BS_OK;
  const int64_t ng = (n + G - 1) / G;
  const int64_t blocks = (ng + 7) / 8;
  group_aabb_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(positions, n, stride, G, ng, out);
  BS_LAUNCH_CHECK("group_aabb_kernel");
  return BS_OK;
}

extern "C" int32_t bs_gather_planes(const float* in, int64_t n_in, const int64_t* idx, int64_t n_out,
                                    int32_t n_planes, float* out, void* stream) {
  if (n_out == 0) return BS_OK;
  gather_planes_kernel<<<grid_for(n_out * n_planes, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(in), n_in, idx, n_out, n_planes, reinterpret_cast<float4*>(out));
  BS_LAUNCH_CHECK("gather_planes_kernel");
  return BS_OK;
}

// ---------------------------------------------------------------------------
// Visible-chunk work list from the culling's counts: chunk c of group g has a
// visible point iff some view's running count grows over it (chunk_prefix
// of chunk c + 1, or the group's total for the last chunk, minus chunk c's).
// The projection kernels then loop over the listed chunks only (at C4 ~2 %
// of the points are visible per view; one CTA per (group, chunk) would mostly
// launch empty CTAs).  Warp-aggregated appends, in no particular order.

namespace bs {
namespace {

__global__ void list_chunks_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ chunk_prefix,
                                   const int32_t* __restrict__ group_begin, int n_groups, int max_chunks, int B,
                                   int32_t* __restrict__ work_list, int32_t* __restrict__ work_count) {
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)n_groups * max_chunks;
  for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x; t0 < total; t0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    bool vis = false;
    if (t < total) {
      const int g = (int)(t / max_chunks), c = (int)(t - (int64_t)g * max_chunks);
      const int size = group_begin[g + 1] - group_begin[g];
      if (c * kCullThreads < size) {
        const bool last = (c + 1) * kCullThreads >= size;
        const int32_t* p0 = chunk_prefix + ((int64_t)g * max_chunks + c) * B;
        const int32_t* p1 = last ? counts + (int64_t)g * B : p0 + B;
        for (int v = 0; v < B && !vis; ++v) vis = p1[v] > p0[v];
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, vis);
    if (bal == 0u) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(work_count, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (vis) work_list[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)t;
  }
}

}  // namespace
}  // namespace bs

extern "C" int32_t bs_list_chunks(const int32_t* counts, const int32_t* chunk_prefix, const int32_t* group_begin,
                                  int32_t n_groups, int32_t max_chunks, int32_t n_views, int32_t* work_list,
                                  int32_t* work_count, void* stream) {
  BS_REQUIRE(max_chunks >= 1 && n_views >= 1 && n_groups >= 0, BS_ERR_PARAMETER, "list_chunks: bad sizes");
  BS_REQUIRE((int64_t)n_groups * max_chunks < (1ll << 31), BS_ERR_PARAMETER, "list_chunks: too many chunks");
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(work_count, 0, sizeof(int32_t), s) != cudaSuccess)
    return set_error(BS_ERR_CUDA, "list_chunks: memset failed");
  const int64_t total = (int64_t)n_groups * max_chunks;
  if (total == 0) return BS_OK;
  list_chunks_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 2048), 256, 0, s>>>(
      counts, chunk_prefix, group_begin, n_groups, max_chunks, n_views, work_list, work_count);
  BS_LAUNCH_CHECK("list_chunks_kernel");
  return BS_OK;
}
