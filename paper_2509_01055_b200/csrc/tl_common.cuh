// Shared host/device utilities for the toolloop-b200 C-ABI library.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/toolloop_b200.h"

namespace tl {

// Thread-local last-error message (tl_last_error()).
void set_error(const char* fmt, ...);

#define TL_CUDA_TRY(expr)                                                      \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::tl::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                      cudaGetErrorString(_e));                                 \
      return TL_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

#define TL_LAUNCH_CHECK()                                                      \
  do {                                                                         \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::tl::set_error("%s:%d launch: %s", __FILE__, __LINE__,                  \
                      cudaGetErrorString(_e));                                 \
      return TL_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

#define TL_REQUIRE(cond, code, ...)                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::tl::set_error(__VA_ARGS__);                                            \
      return (code);                                                           \
    }                                                                          \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-owned workspace (the library never allocates
// device memory on the hot path).
struct Workspace {
  char* base;
  size_t cap;
  size_t used = 0;
  template <class T>
  T* take(size_t n) {
    used = align_up(used, 256);
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += n * sizeof(T);
    return p;
  }
  bool ok() const { return used <= cap; }
};

int num_sms();

// CUDA-event launch counter: every kernel the library launches bumps it so
// bench.py can report `gpu_launches` from the library itself.
void count_launch(int n = 1);

// Optional per-category device timing (tl_profile_enable): a ProfScope
// records a CUDA event pair on the launching stream around the kernels it
// encloses; tl_profile_read() resolves and sums them.  Disabled = no-op.
enum ProfCat {
  PROF_PACK = 0,
  PROF_ADV,
  PROF_LOSS,
  PROF_REDUCE,
  PROF_GATHER,
  PROF_GEMM_FWD,
  PROF_COMBINE,
  PROF_GEMM_DS,
  PROF_GEMM_DH,
  PROF_GEMM_DW,
  PROF_GEMM_OTHER,
  PROF_DSOFTMAX,
  PROF_RESCALE,
  PROF_N
};
struct ProfScope {
  int cat;
  cudaStream_t st;
  cudaEvent_t ev0 = nullptr;
  ProfScope(int c, cudaStream_t s);
  ~ProfScope();
};

}  // namespace tl
