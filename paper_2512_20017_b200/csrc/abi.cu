// ABI housekeeping: thread-local error message, version, launch counter.
#include <stdarg.h>

#include "common.cuh"

namespace bs {

static thread_local char g_last_error[1024] = "";

int32_t set_error(int32_t code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> counter{0};
  return counter;
}

}  // namespace bs

extern "C" const char* bs_last_error(void) { return bs::g_last_error; }
extern "C" int32_t bs_abi_version(void) { return 1; }
extern "C" int64_t bs_launch_count(void) { return bs::launch_counter().load(); }
