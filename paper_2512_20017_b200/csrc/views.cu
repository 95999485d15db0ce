// Per-step view selection and the step's small host transfers, without the
// copy engines (and without the stream synchronisation a pageable
// host-to-device copy implies).  A step needs a handful of per-view rows on the device (the
// batch's cameras, frustum planes, view times, ground-truth indices; Alg. 1
// line 3) and returns a few integers to the host (the per-view
// row counts C[v]_k that size the render buffers, the instance count).  As
// cudaMemcpyAsync transfers these queue on the copy engines behind any bulk
// H2D traffic the caller runs beside the step (the ground-truth upload of the
// next batch): a 16-byte copy then waits for a 6 MB one.  Here the batch's
// view ids travel as kernel parameters and the results are stored straight
// into mapped pinned host memory by a kernel (UVA: every cudaHostAlloc
// allocation is device-accessible at its host address).
#include "common.cuh"

namespace bs {
namespace {

constexpr int kMaxSel = 32;

struct SelIds {
  int32_t n;
  int32_t ids[kMaxSel];
};

// dst[k][w] = src[ids[k]][w], 32-bit words
__global__ void select_rows_kernel(SelIds s, const uint32_t* __restrict__ src, int64_t row_words,
                                   uint32_t* __restrict__ dst) {
  const int64_t total = (int64_t)s.n * row_words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / row_words, w = t - k * row_words;
    dst[t] = src[(int64_t)s.ids[k] * row_words + w];
  }
}

// A small host array as a kernel parameter (kUploadWords words per launch).
constexpr int kUploadWords = 512;  // 2 KB: inside the classic 4 KB parameter limit
struct UploadBlob {
  uint32_t w[kUploadWords];
};

__global__ void upload_kernel(UploadBlob b, int n_words, uint32_t* __restrict__ dst) {
  for (int t = threadIdx.x; t < n_words; t += blockDim.x) dst[t] = b.w[t];
}

__global__ void copy_words_kernel(const uint32_t* __restrict__ src, int64_t n_words, uint32_t* dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_words; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t];
}

}  // namespace
}  // namespace bs

using namespace bs;

extern "C" int32_t bs_select_rows(const int32_t* ids, int32_t n, const void* src, int64_t n_src_rows,
                                  int64_t row_bytes, void* dst, void* stream) {
  BS_REQUIRE(n >= 0 && n <= kMaxSel, BS_ERR_PARAMETER, "select_rows: 0..%d rows", kMaxSel);
  BS_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0, BS_ERR_PARAMETER, "select_rows: row size must be a multiple of 4");
  if (n == 0) return BS_OK;
  BS_REQUIRE(ids != nullptr && src != nullptr && dst != nullptr, BS_ERR_PARAMETER, "select_rows: null pointer");
  SelIds s;
  s.n = n;
  for (int k = 0; k < n; ++k) {
    BS_REQUIRE(ids[k] >= 0 && ids[k] < n_src_rows, BS_ERR_PARAMETER, "select_rows: id %d out of range [0, %lld)",
               ids[k], (long long)n_src_rows);
    s.ids[k] = ids[k];
  }
  const int64_t words = row_bytes / 4, total = words * n;
  select_rows_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 1024), 256, 0, as_stream(stream)>>>(
      s, static_cast<const uint32_t*>(src), words, static_cast<uint32_t*>(dst));
  BS_LAUNCH_CHECK("select_rows_kernel");
  return BS_OK;
}

extern "C" int32_t bs_copy_to_host(const void* src, int64_t n_bytes, void* dst_pinned, void* stream) {
  BS_REQUIRE(n_bytes >= 0 && n_bytes % 4 == 0, BS_ERR_PARAMETER, "copy_to_host: size must be a multiple of 4");
  if (n_bytes == 0) return BS_OK;
  cudaPointerAttributes at;
  BS_REQUIRE(cudaPointerGetAttributes(&at, dst_pinned) == cudaSuccess && at.type == cudaMemoryTypeHost &&
                 at.devicePointer != nullptr,
             BS_ERR_PARAMETER, "copy_to_host: destination must be mapped pinned host memory");
  const int64_t words = n_bytes / 4;
  copy_words_kernel<<<(int)std::min<int64_t>((words + 255) / 256, 1024), 256, 0, as_stream(stream)>>>(
      static_cast<const uint32_t*>(src), words, static_cast<uint32_t*>(at.devicePointer));
  BS_LAUNCH_CHECK("copy_words_kernel");
  return BS_OK;
}

extern "C" int32_t bs_upload(const void* host, int64_t n_bytes, void* dst, void* stream) {
  BS_REQUIRE(n_bytes >= 0 && n_bytes % 4 == 0, BS_ERR_PARAMETER, "upload: size must be a multiple of 4");
  BS_REQUIRE(n_bytes == 0 || (host != nullptr && dst != nullptr), BS_ERR_PARAMETER, "upload: null pointer");
  const uint32_t* src = static_cast<const uint32_t*>(host);
  uint32_t* out = static_cast<uint32_t*>(dst);
  for (int64_t w0 = 0; w0 < n_bytes / 4; w0 += kUploadWords) {
    const int n = (int)std::min<int64_t>(kUploadWords, n_bytes / 4 - w0);
    UploadBlob b;
    memcpy(b.w, src + w0, sizeof(uint32_t) * n);
    upload_kernel<<<1, 256, 0, as_stream(stream)>>>(b, n, out + w0);
    BS_LAUNCH_CHECK("upload_kernel");
  }
  return BS_OK;
}
