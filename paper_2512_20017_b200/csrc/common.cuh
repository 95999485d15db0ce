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

__device__ __forceinline__ float det_sigmoid(float x) {
  return fdiv(1.0f, fadd(1.0f, det_expf(-x)));
}

// f64 signed distance in the order OpenBLAS evaluates
// `p @ planes[:, :3].T + planes[:, 3]` (visibility.py:155-156).
__device__ __forceinline__ double plane_dist(const double* pl, double x, double y, double z) {
  return __dadd_rn(__fma_rn(z, pl[2], __fma_rn(y, pl[1], __dmul_rn(x, pl[0]))), pl[3]);
}

}  // namespace bs
