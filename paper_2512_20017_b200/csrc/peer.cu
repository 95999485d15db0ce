// Peer-memory exchange of the distributed step (Alg. 1 lines 9 and 21,
// PAPER.md:488, 508) without a collective library: every rank exports one
// device allocation (cudaIpcGetMemHandle), the others map it
// (cudaIpcOpenMemHandle; NVLink / NVSwitch P2P between GPUs, plain device
// memory between processes sharing one GPU), and
//   * the projection writes each splat row straight into the receive buffer
//     of the rank that renders its view (bs_proj_desc.view_sp / view_gid:
//     one row-0 pointer per view) -- the forward all-to-all fused into K1;
//   * the gradient rows go back the same way: bs_return_rows writes every
//     G_SP row of the canonical order into its owner's send-layout slot
//     (the backward all-to-all fused into the un-permutation);
//   * completion travels as stream-ordered 32-bit flags: the producer's
//     stream writes (flag := epoch) into the consumer's flag word after its
//     kernel (cuStreamWriteValue32, with a system-scope fence before the
//     write), the consumer's stream waits for (flag >= epoch)
//     (cuStreamWaitValue32) before its next kernel.  No host round trip, no
//     spinning kernel.
// The driver entry points are resolved at run time (cudaGetDriverEntryPoint),
// so the library keeps its runtime-only link.
#include <cuda.h>

#include "common.cuh"
#include "tile.cuh"

namespace bs {
namespace {

__global__ void return_rows_kernel(const float* __restrict__ src, int src_width, int width,
                                   const int64_t* __restrict__ order, int64_t n, const int64_t* __restrict__ seg_row0,
                                   const int32_t* __restrict__ seg_src, const int64_t* __restrict__ seg_dst0, int n_segs,
                                   float* const* __restrict__ dst, int dst_width) {
  // one thread per (canonical row, float) -- `width` used floats of the row
  const int64_t total = n * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / width;
    const int k = (int)(t - i * width);
    const int64_t r = order[i];                     // received row of canonical position i
    const int s = segment_of(seg_row0, n_segs, r);  // (source, view) segment of the received row
    dst[seg_src[s]][(seg_dst0[s] + (r - seg_row0[s])) * dst_width + k] = src[i * src_width + k];
  }
}

typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <class F>
int32_t driver_fn(const char* name, F& fn) {
  if (fn) return BS_OK;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  BS_REQUIRE(e == cudaSuccess && q == cudaDriverEntryPointSuccess && p, BS_ERR_CUDA,
             "driver entry point %s unavailable", name);
  fn = reinterpret_cast<F>(p);
  return BS_OK;
}

WriteValueFn g_write = nullptr;
WaitValueFn g_wait = nullptr;

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_ipc_alloc(size_t bytes, void** ptr, uint8_t* handle) {
  BS_REQUIRE(bytes > 0 && ptr && handle, BS_ERR_PARAMETER, "ipc_alloc: bad arguments");
  cudaError_t e = cudaMalloc(ptr, bytes);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_alloc: cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_alloc: cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle, &h, sizeof(h));
  e = cudaMemset(*ptr, 0, bytes);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_alloc: memset: %s", cudaGetErrorString(e));
  return BS_OK;
}

extern "C" int32_t bs_ipc_open(const uint8_t* handle, void** ptr) {
  BS_REQUIRE(handle && ptr, BS_ERR_PARAMETER, "ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_open: %s", cudaGetErrorString(e));
  return BS_OK;
}

extern "C" int32_t bs_ipc_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_close: %s", cudaGetErrorString(e));
  return BS_OK;
}

extern "C" int32_t bs_ipc_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  BS_REQUIRE(e == cudaSuccess, BS_ERR_CUDA, "ipc_free: %s", cudaGetErrorString(e));
  return BS_OK;
}

extern "C" size_t bs_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

extern "C" int32_t bs_stream_signal(void* stream, uint32_t* flag, uint32_t value) {
  int32_t st = driver_fn("cuStreamWriteValue32", g_write);
  if (st) return st;
  // default flags: a fence (system scope) orders every prior write of the
  // stream before the flag write
  const CUresult r = g_write(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0);
  BS_REQUIRE(r == CUDA_SUCCESS, BS_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  return BS_OK;
}

extern "C" int32_t bs_stream_wait(void* stream, const uint32_t* flag, uint32_t value) {
  int32_t st = driver_fn("cuStreamWaitValue32", g_wait);
  if (st) return st;
  const CUresult r = g_wait(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                            CU_STREAM_WAIT_VALUE_GEQ);
  BS_REQUIRE(r == CUDA_SUCCESS, BS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return BS_OK;
}

extern "C" int32_t bs_return_rows(const float* src, int32_t src_width, int32_t width, const int64_t* order, int64_t n,
                                  const int64_t* seg_row0, const int32_t* seg_src, const int64_t* seg_dst0,
                                  int32_t n_segs, float* const* dst, int32_t dst_width, void* stream) {
  BS_REQUIRE(width > 0 && width <= src_width && width <= dst_width, BS_ERR_PARAMETER, "return_rows: bad row widths");
  BS_REQUIRE(n_segs >= 1, BS_ERR_PARAMETER, "return_rows: no segments");
  if (n <= 0) return BS_OK;
  return_rows_kernel<<<grid_for(n * width, 256), 256, 0, as_stream(stream)>>>(
      src, src_width, width, order, n, seg_row0, seg_src, seg_dst0, n_segs, dst, dst_width);
  BS_LAUNCH_CHECK("return_rows_kernel");
  return BS_OK;
}
