// K2 — GRPO group-normalised advantages (rl/loss.py:103-116).
//
// One warp per group (a group is a contiguous run of trajectories sharing a
// prompt).  The two math.fsum reductions are reproduced exactly with a
// lane-distributed superaccumulator (exact_fp64.cuh): every lane adds the
// digits of each reward that fall into its limbs, lane 0 carry-propagates and
// rounds once.  Then, as in the reference:
//   mean = fsum(R) / G
//   var  = fsum((R - mean)^2) / G        (squares as IEEE x*x)
//   A_i  = (R_i - mean) / max(sqrt(var), std_floor)
// All fp64 operations are the IEEE round-to-nearest ones of CPython, in the
// same order, with FMA contraction disabled via __d*_rn intrinsics.
// The warp also writes the per-trajectory gradient weight of the fused loss
// (reference aggregation cli.py:317-344 or DAPO token-mean) and the
// trajectory -> group map.
#include "exact_fp64.cuh"
#include "tl_common.cuh"

namespace tl {
namespace {

constexpr int kAdvWarps = 4;

__global__ void __launch_bounds__(kAdvWarps * 32)
    group_adv_kernel(const double* __restrict__ rewards, const int32_t* __restrict__ group_off,
                     int n_groups, double std_floor, const int32_t* __restrict__ act_off, int agg,
                     double norm_groups, double norm_tokens, double* __restrict__ adv64,
                     float* __restrict__ adv32, float* __restrict__ traj_w,
                     int32_t* __restrict__ traj_group) {
  __shared__ long long limbs[kAdvWarps][96];
  __shared__ double bcast[kAdvWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * kAdvWarps + w;
  if (g >= n_groups) return;
  const int b0 = group_off[g], b1 = group_off[g + 1], G = b1 - b0;
  long long* L = limbs[w];

  double mean = 0.0, div = 1.0;
  if (G >= 2) {
    // ---- mean = fsum(R) / G
    SuperAccLane acc;
    acc.clear();
    for (int i = 0; i < G; ++i) acc.add(rewards[b0 + i]);
#pragma unroll
    for (int j = 0; j < 3; ++j) L[lane + 32 * j] = acc.limb[j];
    __syncwarp();
    if (lane == 0) bcast[w] = __ddiv_rn(superacc_finalize(L), static_cast<double>(G));
    __syncwarp();
    mean = bcast[w];
    // ---- var = fsum((R - mean)^2) / G
    acc.clear();
    for (int i = 0; i < G; ++i) {
      const double d = __dadd_rn(rewards[b0 + i], -mean);
      acc.add(__dmul_rn(d, d));
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 3; ++j) L[lane + 32 * j] = acc.limb[j];
    __syncwarp();
    if (lane == 0) {
      const double var = __ddiv_rn(superacc_finalize(L), static_cast<double>(G));
      const double sd = __dsqrt_rn(var);
      bcast[w] = sd > std_floor ? sd : std_floor;  // max(std, floor)
    }
    __syncwarp();
    div = bcast[w];
  }
  for (int i = lane; i < G; i += 32) {
    const int b = b0 + i;
    // GroupTooSmall is raised on host before launch; NaN marks misuse.
    const double a = G >= 2 ? __ddiv_rn(__dadd_rn(rewards[b], -mean), div) : __longlong_as_double(0x7ff8000000000000LL);
    if (adv64) adv64[b] = a;
    if (adv32) adv32[b] = static_cast<float>(a);
    if (traj_group) traj_group[b] = g;
    if (traj_w) {
      float wt = 0.f;
      const int n = act_off ? act_off[b + 1] - act_off[b] : 1;
      if (n > 0) {
        wt = agg == 1 ? static_cast<float>(1.0 / norm_tokens)
                      : static_cast<float>(1.0 / (static_cast<double>(n) * G * norm_groups));
      }
      traj_w[b] = wt;
    }
  }
}

}  // namespace
}  // namespace tl

extern "C" int tl_group_advantages(const double* rewards, const int32_t* group_off,
                                   int32_t n_groups, int32_t n_traj, double std_floor,
                                   const int32_t* act_off, int32_t agg, double norm_groups,
                                   double norm_tokens, double* adv64, float* adv32, float* traj_w,
                                   int32_t* traj_group, tl_stream_t stream) {
  TL_REQUIRE(n_groups >= 0 && n_traj >= 0, TL_ERR_INVALID_ARG, "negative sizes");
  TL_REQUIRE(std_floor > 0.0, TL_ERR_INVALID_ARG, "std_floor must be positive");
  TL_REQUIRE(agg == 0 || agg == 1, TL_ERR_INVALID_ARG, "agg must be 0 or 1");
  if (traj_w) {
    TL_REQUIRE(agg == 1 ? norm_tokens > 0 : norm_groups > 0, TL_ERR_INVALID_ARG,
               "normaliser must be positive");
  }
  if (n_groups == 0) return TL_OK;
  const int grid = (n_groups + tl::kAdvWarps - 1) / tl::kAdvWarps;
  tl::ProfScope prof(tl::PROF_ADV, static_cast<cudaStream_t>(stream));
  tl::group_adv_kernel<<<grid, tl::kAdvWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      rewards, group_off, n_groups, std_floor, act_off, agg, norm_groups, norm_tokens, adv64,
      adv32, traj_w, traj_group);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}
