// Internal entry points shared between the standalone loss (loss.cu) and the
// fused LM-head step (lmhead.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tl {
// Deterministic reductions of per-token terms: trajectory -> group -> report.
// traj_out [n_traj * 8], group_out [n_groups * TL_GROUP_OUT_LEN].
int launch_reductions(const float* term, const float* k3o, const uint8_t* flags, const float* ent,
                      const uint8_t* mask, int use_mask, const int32_t* cu, const int32_t* group_off,
                      int n_traj, int n_groups, int agg, double* traj_out, double* group_out,
                      double* report, cudaStream_t st);
}  // namespace tl
