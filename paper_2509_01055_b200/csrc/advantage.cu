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

// F2 — verifiable rewards (rl/rewards.py:15-68) from per-trajectory signals,
// evaluated inside the advantage warp so the group RaPR (fraction of the
// group's responses that invoked a tool, rewards.py:43-63) is a warp ballot.
struct RewardSpec {
  tl_reward_params p;
  const uint8_t* correct;      // matcher result / terminated_ok (swe)
  const uint8_t* tool_called;  // invoked_tool / tool_called
  const int32_t* n_vo;         // tool invocations (visual reasoner)
  const double* r_acc;         // accuracy term (visual reasoner)
  const uint8_t* tests_pass;   // swe
  double* rewards_out;         // [B]
  double* rapr_out;            // [n_groups] (nullable)
  const double* rapr_in;       // [n_groups] override (nullable)
};

__device__ double reward_of(const RewardSpec& rs, int b, double rapr) {
  const tl_reward_params& p = rs.p;
  const bool ok = rs.correct && rs.correct[b];
  switch (p.kind) {
    case TL_REWARD_MATCH: return ok ? 1.0 : -1.0;
    case TL_REWARD_MATH: return ok ? 1.0 : __dadd_rn(-1.0, -0.25);
    case TL_REWARD_DEEPSEARCH:
      return __dadd_rn(ok ? 1.0 : -1.0, rs.tool_called[b] ? 0.1 : 0.0);
    case TL_REWARD_VISUAL_REASONER: {
      const double gap = __dadd_rn(p.h, -rapr);
      const double cur = rs.tool_called[b] ? __dmul_rn(p.alpha, 0.0 > gap ? 0.0 : gap) : 0.0;
      const int over = p.n - rs.n_vo[b];
      const double pen = __dmul_rn(p.beta, static_cast<double>(over < 0 ? over : 0));
      return __dadd_rn(__dadd_rn(rs.r_acc[b], cur), pen);
    }
    case TL_REWARD_SWE: return (ok && rs.tests_pass[b]) ? 1.0 : 0.0;
    default: return __longlong_as_double(0x7ff8000000000000LL);
  }
}

__global__ void __launch_bounds__(kAdvWarps * 32)
    group_adv_kernel(const double* rewards, const int32_t* __restrict__ group_off,
                     int n_groups, double std_floor, const int32_t* __restrict__ act_off, int agg,
                     double norm_groups, double norm_tokens, double* __restrict__ adv64,
                     float* __restrict__ adv32, float* __restrict__ traj_w,
                     int32_t* __restrict__ traj_group, RewardSpec rs) {
  __shared__ long long limbs[kAdvWarps][96];
  __shared__ double bcast[kAdvWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * kAdvWarps + w;
  if (g >= n_groups) return;
  const int b0 = group_off[g], b1 = group_off[g + 1], G = b1 - b0;
  long long* L = limbs[w];

  if (rs.p.kind >= 0) {
    double rapr = 0.0;
    if (rs.rapr_in) {
      rapr = rs.rapr_in[g];
    } else if (rs.tool_called) {
      int invoked = 0;
      for (int i0 = 0; i0 < G; i0 += 32) {
        const bool t = i0 + lane < G && rs.tool_called[b0 + i0 + lane];
        invoked += __popc(__ballot_sync(0xffffffffu, t));
      }
      rapr = G ? __ddiv_rn(static_cast<double>(invoked), static_cast<double>(G)) : 0.0;
    }
    for (int i = lane; i < G; i += 32) rs.rewards_out[b0 + i] = reward_of(rs, b0 + i, rapr);
    if (rs.rapr_out && lane == 0) rs.rapr_out[g] = rapr;
    __threadfence_block();
    __syncwarp();
    rewards = rs.rewards_out;
  }

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
  tl::RewardSpec rs{};
  rs.p.kind = -1;
  tl::group_adv_kernel<<<grid, tl::kAdvWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      rewards, group_off, n_groups, std_floor, act_off, agg, norm_groups, norm_tokens, adv64,
      adv32, traj_w, traj_group, rs);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}

extern "C" int tl_group_rewards_advantages(
    const tl_reward_params* params, const uint8_t* correct, const uint8_t* tool_called,
    const int32_t* n_vo, const double* r_acc, const uint8_t* tests_pass, const int32_t* group_off,
    int32_t n_groups, int32_t n_traj, double std_floor, const double* rapr_in,
    double* rewards_out, double* rapr_out, double* adv64, float* adv32, tl_stream_t stream) {
  TL_REQUIRE(params && rewards_out, TL_ERR_INVALID_ARG, "params / rewards_out required");
  TL_REQUIRE(params->kind >= TL_REWARD_MATCH && params->kind <= TL_REWARD_SWE, TL_ERR_INVALID_ARG,
             "unknown reward kind %d", params->kind);
  TL_REQUIRE(std_floor > 0.0, TL_ERR_INVALID_ARG, "std_floor must be positive");
  const int k = params->kind;
  TL_REQUIRE(k == TL_REWARD_VISUAL_REASONER || correct, TL_ERR_INVALID_ARG, "correct[] required");
  TL_REQUIRE((k != TL_REWARD_DEEPSEARCH && k != TL_REWARD_VISUAL_REASONER) || tool_called,
             TL_ERR_INVALID_ARG, "tool_called[] required");
  TL_REQUIRE(k != TL_REWARD_VISUAL_REASONER || (n_vo && r_acc), TL_ERR_INVALID_ARG,
             "n_vo[] and r_acc[] required");
  TL_REQUIRE(k != TL_REWARD_SWE || tests_pass, TL_ERR_INVALID_ARG, "tests_pass[] required");
  (void)n_traj;
  if (n_groups == 0) return TL_OK;
  const int grid = (n_groups + tl::kAdvWarps - 1) / tl::kAdvWarps;
  tl::ProfScope prof(tl::PROF_ADV, static_cast<cudaStream_t>(stream));
  tl::RewardSpec rs{*params,    correct,     tool_called, n_vo,    r_acc,
                    tests_pass, rewards_out, rapr_out,    rapr_in};
  tl::group_adv_kernel<<<grid, tl::kAdvWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      rewards_out, group_off, n_groups, std_floor, nullptr, 0, 1.0, 1.0, adv64, adv32, nullptr,
      nullptr, rs);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}
