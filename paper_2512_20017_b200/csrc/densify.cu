// Periodic densification of the point shard (standard 3DGS
// clone / split / prune) and the AABBs of variable-size
// point groups.
//
// The shard keeps its layout contract: points stay in their Z-order group
// (outputs of a point follow it inside the group, in point order), so the
// group table, the culling and the row layout of the next step work
// unchanged on the new shard; only the group boundaries move.  Two passes,
// one CTA per group: bs_densify_mark decides every point's action and counts
// each group's outputs; the caller scans the counts into the new group table;
// bs_densify_apply block-scans the per-point output counts and writes the
// new plane-major parameters and Adam moments.  The split samples are an
// Irwin-Hall sum of 12 splitmix64 uniforms per axis and every float op is an
// explicit round-to-nearest intrinsic, so the new shard is bit-exact against
// the C oracle (so_densify, compiled with -ffp-contract=off).
#include "splat_math.cuh"

namespace bs {
namespace {

constexpr int kDensThreads = 256;
constexpr float kLogSplit = 0x1.e148a2p-2f;  // ln(1.6) = ln(0.8 * 2): 3DGS's split scale factor

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// N(0, 1) sample (Irwin-Hall, 12 uniforms of 24 bits) for (child, axis)
__device__ __forceinline__ float split_normal(uint64_t base, int child, int axis) {
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < 12; ++j) sum += (uint32_t)(splitmix64(base + (uint64_t)(child * 36 + axis * 12 + j + 1)) >> 40);
  return fsub(fmul(__uint2float_rn(sum), 0x1p-24f), 6.0f);
}

struct DensArgs {
  float grad_threshold, split_scale, min_opacity, max_scale;
  uint32_t seed;
};

__device__ __forceinline__ int point_action(const DensArgs& a, float4 p0, float4 p1, float2 st) {
  const float o = det_sigmoid(p0.w);
  const float smax = fmaxf(fmaxf(det_expf(p1.x), det_expf(p1.y)), det_expf(p1.z));
  if (o < a.min_opacity || (a.max_scale > 0.f && smax > a.max_scale)) return BS_DENSIFY_PRUNE;
  const float avg = st.y > 0.f ? fdiv(st.x, st.y) : 0.f;
  if (st.y > 0.f && avg >= a.grad_threshold) return smax > a.split_scale ? BS_DENSIFY_SPLIT : BS_DENSIFY_CLONE;
  return BS_DENSIFY_KEEP;
}

__device__ __forceinline__ int n_out(int action) {
  return action == BS_DENSIFY_PRUNE ? 0 : (action == BS_DENSIFY_KEEP ? 1 : 2);
}

// inclusive block scan of one int per thread (kDensThreads threads); returns
// the inclusive prefix, total in *total
__device__ __forceinline__ int block_scan(int x, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) s_warp[w] = v;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < kDensThreads / 32; ++k) {
    const int t = s_warp[k];
    pre += k < w ? t : 0;
    tot += t;
  }
  __syncthreads();
  *total = tot;
  return pre + v;
}

__global__ void __launch_bounds__(kDensThreads) densify_mark_kernel(DensArgs a, const float4* __restrict__ params,
                                                                    int64_t S, const float2* __restrict__ stats,
                                                                    const int32_t* __restrict__ group_begin,
                                                                    int32_t* __restrict__ action,
                                                                    int32_t* __restrict__ group_out) {
  __shared__ int s_warp[kDensThreads / 32];
  const int g = blockIdx.x;
  const int lo = group_begin[g], hi = group_begin[g + 1];
  int count = 0;
  for (int b0 = lo; b0 < hi; b0 += kDensThreads) {
    const int i = b0 + threadIdx.x;
    int c = 0;
    if (i < hi) {
      const int act = point_action(a, params[i], params[S + i], stats ? stats[i] : make_float2(0.f, 0.f));
      action[i] = act;
      c = n_out(act);
    }
    int tot;
    block_scan(c, s_warp, &tot);
    count += tot;
  }
  if (threadIdx.x == 0) group_out[g] = count;
}

__global__ void __launch_bounds__(kDensThreads) densify_apply_kernel(
    DensArgs a, const float4* __restrict__ params, const float4* __restrict__ m, const float4* __restrict__ v,
    int64_t S, const int32_t* __restrict__ action, const int32_t* __restrict__ group_begin,
    const int32_t* __restrict__ new_begin, const int32_t* __restrict__ point_gid, float4* __restrict__ params_new,
    float4* __restrict__ m_new, float4* __restrict__ v_new, int64_t S_new, int32_t* __restrict__ src_index) {
  __shared__ int s_warp[kDensThreads / 32];
  const int g = blockIdx.x;
  const int lo = group_begin[g], hi = group_begin[g + 1];
  int64_t out0 = new_begin[g];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b0 = lo; b0 < hi; b0 += kDensThreads) {
    const int i = b0 + threadIdx.x;
    const int act = i < hi ? action[i] : BS_DENSIFY_PRUNE;
    const int c = n_out(act);
    int tot;
    const int incl = block_scan(c, s_warp, &tot);
    const int64_t j = out0 + incl - c;  // first output of point i
    out0 += tot;
    if (c == 0) continue;
    if (act == BS_DENSIFY_SPLIT) {
      PointIn pt;
      const float4 p0 = params[i], p1 = params[S + i], q4 = params[2 * S + i];
      pt.p[0] = p0.x; pt.p[1] = p0.y; pt.p[2] = p0.z; pt.op_logit = p0.w;
      pt.ls[0] = p1.x; pt.ls[1] = p1.y; pt.ls[2] = p1.z;
      pt.q[0] = q4.x; pt.q[1] = q4.y; pt.q[2] = q4.z; pt.q[3] = q4.w;
      QuatFrame q;
      quat_frame(pt, 3, q);
      const uint32_t gid = point_gid ? (uint32_t)point_gid[i] : (uint32_t)i;
      const uint64_t base = splitmix64(((uint64_t)a.seed << 32) | gid);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        float l[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) l[k] = fmul(q.s[k], split_normal(base, ch, k));
        float mu[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
          mu[r] = fadd(pt.p[r], fadd(fadd(fmul(q.Rq[3 * r], l[0]), fmul(q.Rq[3 * r + 1], l[1])), fmul(q.Rq[3 * r + 2], l[2])));
        const int64_t o = j + ch;
        params_new[o] = make_float4(mu[0], mu[1], mu[2], p0.w);
        params_new[S_new + o] = make_float4(fsub(p1.x, kLogSplit), fsub(p1.y, kLogSplit), fsub(p1.z, kLogSplit), p1.w);
        for (int p = 2; p < BS_PARAM_PLANES; ++p) params_new[p * S_new + o] = params[p * S + i];
        for (int p = 0; p < BS_PARAM_PLANES; ++p) {
          m_new[p * S_new + o] = zero;
          v_new[p * S_new + o] = zero;
        }
        src_index[o] = i;
      }
    } else {
      for (int p = 0; p < BS_PARAM_PLANES; ++p) {
        const float4 x = params[p * S + i];
        params_new[p * S_new + j] = x;
        m_new[p * S_new + j] = m[p * S + i];
        v_new[p * S_new + j] = v[p * S + i];
        if (act == BS_DENSIFY_CLONE) {
          params_new[p * S_new + j + 1] = x;
          m_new[p * S_new + j + 1] = zero;
          v_new[p * S_new + j + 1] = zero;
        }
      }
      src_index[j] = i;
      if (act == BS_DENSIFY_CLONE) src_index[j + 1] = i;
    }
  }
}

__global__ void __launch_bounds__(kDensThreads) group_aabb_ranges_kernel(const float4* __restrict__ params,
                                                                         const int32_t* __restrict__ group_begin,
                                                                         float* __restrict__ aabb) {
  __shared__ float s_red[6][kDensThreads / 32];
  const int g = blockIdx.x;
  const int lo = group_begin[g], hi = group_begin[g + 1];
  const float inf = __int_as_float(0x7f800000);
  float mn[3] = {inf, inf, inf}, mx[3] = {-inf, -inf, -inf};
  for (int i = lo + threadIdx.x; i < hi; i += kDensThreads) {
    const float4 p = params[i];
    mn[0] = fminf(mn[0], p.x); mn[1] = fminf(mn[1], p.y); mn[2] = fminf(mn[2], p.z);
    mx[0] = fmaxf(mx[0], p.x); mx[1] = fmaxf(mx[1], p.y); mx[2] = fmaxf(mx[2], p.z);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
      mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
    }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int k = 0; k < 3; ++k) {
      s_red[k][w] = mn[k];
      s_red[3 + k][w] = mx[k];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int k = threadIdx.x;
    float r = k < 3 ? inf : -inf;
    for (int j = 0; j < kDensThreads / 32; ++j) r = k < 3 ? fminf(r, s_red[k][j]) : fmaxf(r, s_red[k][j]);
    // an empty group (every point pruned) gets the degenerate box at the origin
    aabb[(int64_t)g * 6 + k] = hi > lo ? r : 0.f;
  }
}

int32_t dens_args(const bs_densify_desc* d, DensArgs& a) {
  BS_REQUIRE(d != nullptr, BS_ERR_PARAMETER, "null densify descriptor");
  BS_REQUIRE(d->model == BS_MODEL_3DGS, BS_ERR_PARAMETER, "densification is implemented for the 3DGS model");
  BS_REQUIRE(d->grad_threshold >= 0.f && d->split_scale >= 0.f && d->min_opacity >= 0.f, BS_ERR_PARAMETER,
             "densify thresholds must be non-negative");
  a = DensArgs{d->grad_threshold, d->split_scale, d->min_opacity, d->max_scale, d->seed};
  return BS_OK;
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_densify_mark(const bs_densify_desc* d, const float* params, int64_t n_points, const float* stats,
                                   const int32_t* group_begin, int32_t n_groups, int32_t* action,
                                   int32_t* group_out, void* stream) {
  DensArgs a;
  int32_t st = dens_args(d, a);
  if (st) return st;
  BS_REQUIRE(n_groups >= 0 && n_points >= 0 && n_points < (1ll << 31), BS_ERR_PARAMETER, "bad shard size");
  if (n_groups == 0) return BS_OK;
  densify_mark_kernel<<<n_groups, kDensThreads, 0, as_stream(stream)>>>(
      a, reinterpret_cast<const float4*>(params), n_points, reinterpret_cast<const float2*>(stats), group_begin,
      action, group_out);
  BS_LAUNCH_CHECK("densify_mark_kernel");
  return BS_OK;
}

extern "C" int32_t bs_densify_apply(const bs_densify_desc* d, const float* params, const float* exp_avg,
                                    const float* exp_avg_sq, int64_t n_points, const int32_t* action,
                                    const int32_t* group_begin, const int32_t* new_group_begin, int32_t n_groups,
                                    const int32_t* point_gid, float* params_new, float* exp_avg_new,
                                    float* exp_avg_sq_new, int64_t n_new, int32_t* src_index, void* stream) {
  DensArgs a;
  int32_t st = dens_args(d, a);
  if (st) return st;
  BS_REQUIRE(n_groups >= 0 && n_new >= 0 && n_new < (1ll << 31), BS_ERR_PARAMETER, "bad shard size");
  if (n_groups == 0) return BS_OK;
  densify_apply_kernel<<<n_groups, kDensThreads, 0, as_stream(stream)>>>(
      a, reinterpret_cast<const float4*>(params), reinterpret_cast<const float4*>(exp_avg),
      reinterpret_cast<const float4*>(exp_avg_sq), n_points, action, group_begin, new_group_begin, point_gid,
      reinterpret_cast<float4*>(params_new), reinterpret_cast<float4*>(exp_avg_new),
      reinterpret_cast<float4*>(exp_avg_sq_new), n_new, src_index);
  BS_LAUNCH_CHECK("densify_apply_kernel");
  return BS_OK;
}

extern "C" int32_t bs_group_aabb_ranges(const float* params, int64_t n_points, const int32_t* group_begin,
                                        int32_t n_groups, float* aabb_out, void* stream) {
  BS_REQUIRE(n_groups >= 0 && n_points >= 0, BS_ERR_PARAMETER, "bad shard size");
  if (n_groups == 0) return BS_OK;
  group_aabb_ranges_kernel<<<n_groups, kDensThreads, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(params),
                                                                             group_begin, aabb_out);
  BS_LAUNCH_CHECK("group_aabb_ranges_kernel");
  return BS_OK;
}
