// Shared helpers for the sm_100a kernels behind include/splat_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include "../../include/splat_b200.h"

namespace bs {

// ---------------------------------------------------------------------------
// status / error plumbing (thread-local message, errors.py:8-51 codes)

int32_t set_error(int32_t code, const char* fmt, ...);
std::atomic<int64_t>& launch_counter();

inline void count_launch(int64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

inline int32_t check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(BS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  count_launch();
  return BS_OK;
}

#define BS_REQUIRE(cond, code, ...)            \
  do {                                         \
    if (!(cond)) return bs::set_error(code, __VA_ARGS__); \
  } while (0)

#define BS_LAUNCH_CHECK(what)                  \
  do {                                         \
    int32_t _st = bs::check_launch(what);      \
    if (_st != BS_OK) return _st;              \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

inline int grid_for(int64_t n, int block, int max_blocks = kNumSMs * 16) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// Deterministic float32 arithmetic.  Every op on a path that feeds an
// integer output (radius, tile rect, depth key) is an explicit IEEE
// round-to-nearest intrinsic so ptxas cannot contract it into an FMA; the
// CPU oracle (oracle/splat_oracle.c, -ffp-contract=off) performs the same
// op sequence and therefore produces bit-identical splat state.

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }

// exp(x) by Cody-Waite reduction + degree-6 Horner polynomial; only exact
// IEEE ops, so host and device agree bit-for-bit.  Input clamped to
// [-80, 80] (no subnormal results).
__device__ __forceinline__ float det_expf(float x) {
  x = fminf(fmaxf(x, -80.0f), 80.0f);
  const float n = rintf(fmul(x, 0x1.715476p+0f));
  float r = fsub(x, fmul(n, 0x1.62e400p-1f));
  r = fsub(r, fmul(n, 0x1.7f7d1cp-20f));
  float p = 0x1.6c16c2p-10f;                   // 1/720
  p = fadd(fmul(p, r), 0x1.111112p-7f);        // 1/120
  p = fadd(fmul(p, r), 0x1.555556p-5f);        // 1/24
  p = fadd(fmul(p, r), 0x1.555556p-3f);        // 1/6
  p = fadd(fmul(p, r), 0x1.000000p-1f);        // 1/2
  p = fadd(fmul(p, r), 1.0f);
  p = fadd(fmul(p, r), 1.0f);
  const int e = static_cast<int>(n) + 127;
  return fmul(p, __int_as_float(e << 23));
}

// ln(x) for normal x > 0: x = m 2^e with m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh(s), s = (m - 1) / (m + 1), odd series to s^9 (|s| <= 0.172,
// truncation < 1e-9).  Exact IEEE ops only (host oracle: or_det_logf).
// Non-positive or subnormal input returns -87.5 (below ln(FLT_MIN)).
__device__ __forceinline__ float det_logf(float x) {
  if (!(x >= 1.17549435e-38f)) return -87.5f;
  const uint32_t ix = __float_as_uint(x);
  int e = (int)(ix >> 23) - 127;
  float m = __uint_as_float((ix & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) {
    m = fmul(m, 0.5f);
    e += 1;
  }
  const float s = fdiv(fsub(m, 1.0f), fadd(m, 1.0f));
  const float s2 = fmul(s, s);
  float p = 0x1.c71c72p-4f;              // 1/9
  p = fadd(fmul(p, s2), 0x1.249250p-3f);  // 1/7
  p = fadd(fmul(p, s2), 0x1.99999ap-3f);  // 1/5
  p = fadd(fmul(p, s2), 0x1.555556p-2f);  // 1/3
  p = fadd(fmul(p, s2), 1.0f);
  const float lnm = fmul(fmul(2.0f, s), p);
  const float fe = (float)e;
  return fadd(fmul(fe, 0x1.62e400p-1f), fadd(lnm, fmul(fe, 0x1.7f7d1cp-20f)));
}

// Squared Mahalanobis extent of a 3DGS splat's support: the blend keeps a
// pair iff q <= 9 (3-sigma ellipse) and alpha = o exp(-q/2) >= 1/255, i.e.
// q <= min(9, 2 ln(255 o)).  <= 0: the splat can never contribute.
__device__ __forceinline__ float support_k(float opac) {
  return fminf(9.0f, fmul(2.0f, det_logf(fmul(255.0f, opac))));
}

// Rasteriser support threshold of a row with opacity o (bs_row_support):
// 3DGS the log2-exponent threshold k * (-log2(e) / 2), 2DGS k itself.
constexpr float kHalfLog2eNeg = -0.5f * 1.4426950408889634f;
__device__ __forceinline__ float row_support_from_k(float k, bool two_d) { return two_d ? k : fmul(k, kHalfLog2eNeg); }
__device__ __forceinline__ float row_support_value(float opac, bool two_d) {
  return row_support_from_k(support_k(opac), two_d);
}

__device__ __forceinline__ float det_sigmoid(float x) {
  return fdiv(1.0f, fadd(1.0f, det_expf(-x)));
}

// f64 signed distance in the order OpenBLAS evaluates
// `p @ planes[:, :3].T + planes[:, 3]` (visibility.py:155-156).
__device__ __forceinline__ double plane_dist(const double* pl, double x, double y, double z) {
  return __dadd_rn(__fma_rn(z, pl[2], __fma_rn(y, pl[1], __dmul_rn(x, pl[0]))), pl[3]);
}

}  // namespace bs
