// Library-wide state: last-error message, launch counter, device query.
#include <atomic>
#include <cstring>

#include "tl_common.cuh"

namespace tl {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      cached = 148;
  }
  return cached;
}

}  // namespace tl

extern "C" const char* tl_last_error(void) { return tl::g_err; }
extern "C" int tl_abi_version(void) { return TL_ABI_VERSION; }
extern "C" int64_t tl_launch_count(void) { return tl::g_launches.load(); }
