// Internal entry points shared between the standalone loss (loss.cu) and the
// fused LM-head step (lmhead.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tl_common.cuh"

namespace tl {
// Scratch of the deterministic trajectory -> group -> report reductions
// (loss.cu): per-unit partials, per-trajectory / per-group rows, arrival
// counters.
struct ReduceWs {
  double* unit_out;
  double* traj_out;
  double* group_out;
  int* ctr;
};
ReduceWs carve_reduce(Workspace& w, long long n_tokens, int n_traj, int n_groups);
// Per-token terms written by the fused log-prob epilogue -> report.
int launch_reductions(const float* term, const float* k3o, const uint8_t* flags, const float* ent,
                      const uint8_t* mask, int use_mask, const int32_t* cu, const int32_t* group_off,
                      int n_traj, int n_groups, long long n_tokens, int agg, const ReduceWs& r,
                      double* report, cudaStream_t st);
}  // namespace tl
