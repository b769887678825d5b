// Library-wide state: last-error message, launch counter, device query.
#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

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

// SM count of the current device (cached per device id).
int num_sms() {
  constexpr int kMax = 64;
  static std::atomic<int> cached[kMax];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMax) return 148;
  int n = cached[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// ---------------------------------------------------------- profiling ----
namespace {
struct ProfRec {
  int cat;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_pool;
const char* kProfNames[PROF_N] = {"pack",     "advantage", "loss",     "reduce",
                                  "gather",   "gemm_fwd",  "combine",  "gemm_dsoftmax",
                                  "gemm_dh",  "gemm_dw",   "gemm_other", "dsoftmax",
                                  "rescale"};

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(int c, cudaStream_t s) : cat(c), st(s) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ev0 = take_event();
  cudaEventRecord(ev0, st);
}

ProfScope::~ProfScope() {
  if (!ev0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t ev1 = take_event();
  cudaEventRecord(ev1, st);
  g_prof.push_back({cat, ev0, ev1});
}

}  // namespace tl

extern "C" int tl_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(tl::g_prof_mu);
  for (auto& r : tl::g_prof) {
    tl::g_pool.push_back(r.a);
    tl::g_pool.push_back(r.b);
  }
  tl::g_prof.clear();
  tl::g_prof_on.store(on != 0);
  return TL_OK;
}

extern "C" int tl_profile_read(double* ms, int64_t* counts, int32_t n_cat) {
  std::lock_guard<std::mutex> lk(tl::g_prof_mu);
  for (int i = 0; i < n_cat; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  for (auto& r : tl::g_prof) {
    TL_CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0.f;
    TL_CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.cat < n_cat) {
      ms[r.cat] += t;
      counts[r.cat] += 1;
    }
  }
  return TL_OK;
}

extern "C" const char* tl_profile_category(int32_t i) {
  return (i >= 0 && i < tl::PROF_N) ? tl::kProfNames[i] : "";
}

extern "C" const char* tl_last_error(void) { return tl::g_err; }
extern "C" int tl_abi_version(void) { return TL_ABI_VERSION; }
extern "C" int64_t tl_launch_count(void) { return tl::g_launches.load(); }
